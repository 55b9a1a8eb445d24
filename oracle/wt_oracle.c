/*
 * wt_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded CPU construction of the levelwise wavelet
 * tree of arXiv 1407.8142 ("Parallel Wavelet Tree Construction").  It exists
 * to prove the CUDA path right.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load it.  The product
 * (paper_1407_8142_b200/) never links, imports or calls anything here, and
 * this file shares no code, header, table or constant with it.
 *
 * What it computes (all citations are PAPER.md line numbers):
 *   - L = ceil(log2 sigma); the root represents [0, 2^L - 1]          :217-218
 *   - a node [a..b] has bit 0 for symbols in the lower half, 1 otherwise;
 *     children are the two halves; stop when no symbols             :219-226
 *   - levelWT, Fig. 1 (:330-380): per level, per node, mask
 *     2^(L-(l+1)) (:333) selects the bit; X[i] = 1 for "left" symbols,
 *     X = exclusive prefix sum, X_s its total (:347-352); a "right"
 *     symbol goes to start + X_s + i - X[i], a "left" one to
 *     start + X[i] (:353-360); children (start, X_s, 2id+1) and
 *     (start + X_s, len - X_s, 2id+2) when non-empty (:363-371).
 *     The recursion below visits nodes depth first, left before right,
 *     so each level's node list comes out in ascending key order;
 *     Fig. 1 builds the same lists breadth first (the filter of :375).
 *   - node key p at level l: heap id 2^l - 1 + p (:418-420, :509, :536-539)
 *   - rank directory: a prefix count of the level bitmap sampled at
 *     two granularities (Jacobson, :805-814); reading R-9 fixes
 *     the sampling: 512-bit blocks (u16, relative to the superblock) and
 *     65536-bit superblocks (u64, absolute), plus the level total.
 *   - access / rank_c by top-down descent (:204-211), using rank1 from the
 *     directory above, so that brute-force query tests also pin the
 *     directory.
 *
 * Parity status: every output array is pinned by tests/test_oracle_pins.py
 * (closed forms, brute force, exhaustive tiny inputs); see DESIGN.md.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_EINVAL (-1)
#define OR_ESYMBOL (-2)
#define OR_ENOMEM (-3)

typedef struct {
  uint64_t n;
  uint64_t sigma;
  uint32_t levels;
  uint32_t elem_bytes;
  uint64_t words_per_level;
  uint64_t *bits;           /* levels * words_per_level, LSB-first       */
  uint64_t *level_node_ptr; /* levels + 1, CSR offsets into node arrays  */
  uint32_t *node_key;       /* top-l-bit prefix p of each non-empty node */
  uint32_t *node_start;     /* first position of the node at its level   */
  uint64_t total_nodes;
  uint64_t blocks_per_level; /* ceil(n / 512)                            */
  uint64_t supers_per_level; /* ceil(n / 65536) + 1                      */
  uint16_t *rank_block;      /* levels * blocks_per_level                 */
  uint64_t *rank_super;      /* levels * supers_per_level                 */
} oracle_tree;

/* growable (key, start) list for one level */
typedef struct {
  uint32_t *key;
  uint32_t *start;
  uint64_t len, cap;
} node_list;

typedef struct {
  uint32_t L;
  uint64_t wpl;
  uint64_t *bits;
  uint32_t *A;  /* the level's sequence S (Fig. 1 "S")   */
  uint32_t *T;  /* the next level's sequence (Fig. 1 "S'") */
  uint32_t *X;  /* prefix-sum array X of Fig. 1 l.12-14 (n < 2^32) */
  node_list *nodes;
  int oom;
} builder;

static int push_node(node_list *nl, uint32_t key, uint32_t start) {
  if (nl->len == nl->cap) {
    uint64_t nc = nl->cap ? nl->cap * 2 : 16;
    uint32_t *k = (uint32_t *)realloc(nl->key, nc * sizeof(uint32_t));
    if (!k) return -1;
    nl->key = k;
    uint32_t *s = (uint32_t *)realloc(nl->start, nc * sizeof(uint32_t));
    if (!s) return -1;
    nl->start = s;
    nl->cap = nc;
  }
  nl->key[nl->len] = key;
  nl->start[nl->len] = start;
  nl->len++;
  return 0;
}

/* visit(l, p, s, e): node with key p at level l covering positions [s, e). */
static void visit(builder *b, uint32_t l, uint32_t p, uint64_t s, uint64_t e) {
  if (b->oom) return;
  if (s == e || l == b->L) return; /* no symbols, or below the last level */
  if (push_node(&b->nodes[l], p, (uint32_t)s)) { b->oom = 1; return; }
  uint32_t mask_shift = b->L - (l + 1);          /* mask = 2^(L-(l+1)), :333 */
  uint64_t len = e - s;
  uint64_t *B = b->bits + (uint64_t)l * b->wpl;  /* this level's bitmap     */
  /* Fig. 1 l.12-13: X[i] = 1 if the symbol goes left (bit is 0) */
  /* Fig. 1 l.14: exclusive prefix sum; X_s = total */
  uint64_t Xs = 0;
  for (uint64_t i = 0; i < len; i++) {
    uint32_t left = ((b->A[s + i] >> mask_shift) & 1u) == 0;
    b->X[s + i] = (uint32_t)Xs;
    Xs += left;
  }
  /* Fig. 1 l.15-17: set the bit and move the symbol to S' */
  for (uint64_t i = 0; i < len; i++) {
    uint32_t sym = b->A[s + i];
    if ((sym >> mask_shift) & 1u) {
      uint64_t pos = s + i;
      B[pos >> 6] |= (uint64_t)1 << (pos & 63);
      b->T[s + Xs + i - b->X[s + i]] = sym;
    } else {
      b->T[s + b->X[s + i]] = sym;
    }
  }
  memcpy(b->A + s, b->T + s, len * sizeof(uint32_t)); /* swap(S, S'), l.21 */
  /* Fig. 1 l.18-19: children, ids 2id+1 / 2id+2 <=> keys 2p / 2p+1 */
  if (Xs > 0) visit(b, l + 1, 2 * p, s, s + Xs);
  if (len - Xs > 0) visit(b, l + 1, 2 * p + 1, s + Xs, e);
}

static uint32_t bitlen_minus1(uint64_t sigma) {
  /* L = ceil(log2 sigma) = bit length of sigma - 1 (sigma >= 1) */
  uint64_t v = sigma - 1;
  uint32_t L = 0;
  while (v) { L++; v >>= 1; }
  return L;
}

static uint32_t popcount64(uint64_t w) { return (uint32_t)__builtin_popcountll(w); }

/* rank directory (:805-814 with reading R-9): walk the 512-bit blocks of each
 * level; block entries count the ones before the block inside its
 * superblock, superblock entries the ones before the superblock, and the
 * last superblock entry is the level total. */
static void rank_directory(const uint64_t *bits, uint32_t L, uint64_t wpl, uint64_t bpl, uint64_t spl,
                           uint16_t *rank_block, uint64_t *rank_super) {
  for (uint32_t l = 0; l < L; l++) {
    const uint64_t *B = bits + (uint64_t)l * wpl;
    uint16_t *blk = rank_block + (uint64_t)l * bpl;
    uint64_t *sup = rank_super + (uint64_t)l * spl;
    uint64_t ones = 0, base = 0;
    for (uint64_t k = 0; k < bpl; k++) {
      if (k % 128 == 0) { sup[k / 128] = ones; base = ones; }
      blk[k] = (uint16_t)(ones - base);
      for (int w = 0; w < 8; w++) ones += popcount64(B[k * 8 + w]);
    }
    sup[spl - 1] = ones; /* the level total */
  }
}

void oracle_free(oracle_tree *t) {
  if (!t) return;
  free(t->bits);
  free(t->level_node_ptr);
  free(t->node_key);
  free(t->node_start);
  free(t->rank_block);
  free(t->rank_super);
  free(t);
}

uint32_t oracle_levels(uint64_t sigma) { return sigma ? bitlen_minus1(sigma) : 0; }

int oracle_build(const void *seq, uint64_t n, uint32_t elem_bytes, uint64_t sigma,
                 oracle_tree **out) {
  if (!out) return OR_EINVAL;
  *out = NULL;
  if ((n > 0 && !seq) || (elem_bytes != 1 && elem_bytes != 2 && elem_bytes != 4))
    return OR_EINVAL;
  if (sigma < 1 || sigma > ((uint64_t)1 << (8 * elem_bytes)) || n >= ((uint64_t)1 << 32))
    return OR_EINVAL;
  uint32_t L = bitlen_minus1(sigma);

  /* validation: every symbol must be < sigma (R-11) */
  uint32_t *A = (uint32_t *)malloc((n ? n : 1) * sizeof(uint32_t));
  if (!A) return OR_ENOMEM;
  for (uint64_t i = 0; i < n; i++) {
    uint32_t v;
    if (elem_bytes == 1) v = ((const uint8_t *)seq)[i];
    else if (elem_bytes == 2) v = ((const uint16_t *)seq)[i];
    else v = ((const uint32_t *)seq)[i];
    if ((uint64_t)v >= sigma) { free(A); return OR_ESYMBOL; }
    A[i] = v;
  }

  oracle_tree *t = (oracle_tree *)calloc(1, sizeof(oracle_tree));
  if (!t) { free(A); return OR_ENOMEM; }
  t->n = n;
  t->sigma = sigma;
  t->levels = L;
  t->elem_bytes = elem_bytes;
  t->words_per_level = ((n + 511) / 512) * 8;
  t->blocks_per_level = (n + 511) / 512;
  t->supers_per_level = (n + 65535) / 65536 + 1;
  uint64_t nbits = (uint64_t)L * t->words_per_level;
  t->bits = (uint64_t *)calloc(nbits ? nbits : 1, sizeof(uint64_t));
  t->level_node_ptr = (uint64_t *)calloc(L + 1, sizeof(uint64_t));
  t->rank_block = (uint16_t *)calloc(L * t->blocks_per_level + 1, sizeof(uint16_t));
  t->rank_super = (uint64_t *)calloc(L * t->supers_per_level + 1, sizeof(uint64_t));
  builder b;
  memset(&b, 0, sizeof(b));
  b.L = L;
  b.wpl = t->words_per_level;
  b.bits = t->bits;
  b.A = A;
  b.T = (uint32_t *)malloc((n ? n : 1) * sizeof(uint32_t));
  b.X = (uint32_t *)malloc((n ? n : 1) * sizeof(uint32_t));
  b.nodes = (node_list *)calloc(L ? L : 1, sizeof(node_list));
  if (!t->bits || !t->level_node_ptr || !t->rank_block || !t->rank_super || !b.T || !b.X ||
      !b.nodes) {
    free(A); free(b.T); free(b.X); free(b.nodes); oracle_free(t);
    return OR_ENOMEM;
  }

  /* levelWT: A = {(0, n, 0, 2^L)} (Fig. 1 l.2) */
  visit(&b, 0, 0, 0, n);
  free(b.T);
  free(b.X);
  free(A);
  if (b.oom) {
    for (uint32_t l = 0; l < L; l++) { free(b.nodes[l].key); free(b.nodes[l].start); }
    free(b.nodes);
    oracle_free(t);
    return OR_ENOMEM;
  }

  /* concatenate the per-level node lists (CSR) */
  uint64_t total = 0;
  for (uint32_t l = 0; l < L; l++) {
    t->level_node_ptr[l] = total;
    total += b.nodes[l].len;
  }
  t->level_node_ptr[L] = total;
  t->total_nodes = total;
  t->node_key = (uint32_t *)malloc((total ? total : 1) * sizeof(uint32_t));
  t->node_start = (uint32_t *)malloc((total ? total : 1) * sizeof(uint32_t));
  if (!t->node_key || !t->node_start) {
    for (uint32_t l = 0; l < L; l++) { free(b.nodes[l].key); free(b.nodes[l].start); }
    free(b.nodes);
    oracle_free(t);
    return OR_ENOMEM;
  }
  for (uint32_t l = 0; l < L; l++) {
    uint64_t off = t->level_node_ptr[l];
    if (b.nodes[l].len) {
      memcpy(t->node_key + off, b.nodes[l].key, b.nodes[l].len * sizeof(uint32_t));
      memcpy(t->node_start + off, b.nodes[l].start, b.nodes[l].len * sizeof(uint32_t));
    }
    free(b.nodes[l].key);
    free(b.nodes[l].start);
  }
  free(b.nodes);

  rank_directory(t->bits, L, t->words_per_level, t->blocks_per_level, t->supers_per_level, t->rank_block,
                 t->rank_super);
  *out = t;
  return OR_OK;
}

/* rank1(l, i) = number of 1 bits of level l in positions [0, i) */
static uint64_t rank1(const oracle_tree *t, uint32_t l, uint64_t i) {
  if (i >= t->n) return t->rank_super[(uint64_t)l * t->supers_per_level + t->supers_per_level - 1];
  const uint64_t *B = t->bits + (uint64_t)l * t->words_per_level;
  uint64_t r = t->rank_super[(uint64_t)l * t->supers_per_level + (i >> 16)];
  r += t->rank_block[(uint64_t)l * t->blocks_per_level + (i >> 9)];
  uint64_t w0 = (i >> 9) * 8;
  for (uint64_t w = w0; w < (i >> 6); w++) r += popcount64(B[w]);
  if (i & 63) r += popcount64(B[i >> 6] & (((uint64_t)1 << (i & 63)) - 1));
  return r;
}

uint64_t oracle_rank1(const oracle_tree *t, uint32_t level, uint64_t i) {
  if (!t || level >= t->levels || i > t->n) return UINT64_MAX;
  return rank1(t, level, i);
}

/* access(S, i) (:204-205): descend, remapping i into the child's range */
uint32_t oracle_access(const oracle_tree *t, uint64_t i) {
  if (!t || i >= t->n) return UINT32_MAX;
  uint64_t s = 0, e = t->n;
  uint32_t sym = 0;
  for (uint32_t l = 0; l < t->levels; l++) {
    uint64_t r1s = rank1(t, l, s), r1e = rank1(t, l, e), r1i = rank1(t, l, i);
    uint64_t z = (e - s) - (r1e - r1s); /* zeros in the node = left child size */
    const uint64_t *B = t->bits + (uint64_t)l * t->words_per_level;
    uint32_t bit = (uint32_t)((B[i >> 6] >> (i & 63)) & 1u);
    sym = (sym << 1) | bit;
    if (bit) {
      i = s + z + (r1i - r1s);
      s = s + z;
    } else {
      i = s + ((i - s) - (r1i - r1s));
      e = s + z;
    }
  }
  return sym;
}

/* rank_c(S, i) (:205-206): occurrences of c in positions 0..i inclusive */
uint64_t oracle_rank(const oracle_tree *t, uint32_t c, uint64_t i) {
  if (!t || i >= t->n || (uint64_t)c >= t->sigma) return UINT64_MAX;
  uint64_t s = 0, e = t->n, r = i + 1; /* r = count of the prefix [s, s+r) */
  for (uint32_t l = 0; l < t->levels; l++) {
    uint64_t r1s = rank1(t, l, s), r1e = rank1(t, l, e), r1p = rank1(t, l, s + r);
    uint64_t z = (e - s) - (r1e - r1s);
    uint32_t bit = (c >> (t->levels - 1 - l)) & 1u;
    if (bit) {
      r = r1p - r1s;
      s = s + z;
    } else {
      r = r - (r1p - r1s);
      e = s + z;
    }
    if (r == 0) return 0;
  }
  return r;
}


/* ======================================================================
 * Wavelet matrix (§7 "Extensions").
 *
 *   "on level l, all symbols with a 0 as their l'th highest bit are
 *    represented on the left side of the level's bitmap and all symbols
 *    with a 1 ... on the right.  Each level stores the number of 0's on the
 *    level.  The bitmap is filled based on the l+1'st highest bit" (:911-916)
 *   "we proceed level-by-level and stably reorder S based on the l'th
 *    highest bit of the symbols using ... prefix sum (similar to levelWT)
 *    ... which also gives the number of 0's on the level" (:917-921)
 *
 * So: A_0 = S; level l's bitmap holds bit (L-1-l) of A_l[i] (the (l+1)'st
 * highest); zeros[l] = number of 0 bits of level l; A_{l+1} = A_l stably
 * reordered by that bit, zeros first, with the prefix sum of levelWT's
 * Fig. 1 l.12-17 over the whole level (one node).  Same bit layout and rank
 * directory as the tree above.
 * ====================================================================== */
typedef struct {
  uint64_t n;
  uint64_t sigma;
  uint32_t levels;
  uint32_t elem_bytes;
  uint64_t words_per_level;
  uint64_t *bits;            /* levels * words_per_level, LSB-first      */
  uint64_t *zeros;           /* levels: number of 0 bits of each level   */
  uint64_t blocks_per_level;
  uint64_t supers_per_level;
  uint16_t *rank_block;
  uint64_t *rank_super;
} oracle_wm;

void oracle_wm_free(oracle_wm *m) {
  if (!m) return;
  free(m->bits);
  free(m->zeros);
  free(m->rank_block);
  free(m->rank_super);
  free(m);
}

int oracle_wm_build(const void *seq, uint64_t n, uint32_t elem_bytes, uint64_t sigma, oracle_wm **out) {
  if (!out) return OR_EINVAL;
  *out = NULL;
  if ((n > 0 && !seq) || (elem_bytes != 1 && elem_bytes != 2 && elem_bytes != 4))
    return OR_EINVAL;
  if (sigma < 1 || sigma > ((uint64_t)1 << (8 * elem_bytes)) || n >= ((uint64_t)1 << 32))
    return OR_EINVAL;
  uint32_t L = bitlen_minus1(sigma);
  uint32_t *A = (uint32_t *)malloc((n ? n : 1) * sizeof(uint32_t));
  uint32_t *T = (uint32_t *)malloc((n ? n : 1) * sizeof(uint32_t));
  uint32_t *X = (uint32_t *)malloc((n ? n : 1) * sizeof(uint32_t));
  if (!A || !T || !X) { free(A); free(T); free(X); return OR_ENOMEM; }
  for (uint64_t i = 0; i < n; i++) {
    uint32_t v;
    if (elem_bytes == 1) v = ((const uint8_t *)seq)[i];
    else if (elem_bytes == 2) v = ((const uint16_t *)seq)[i];
    else v = ((const uint32_t *)seq)[i];
    if ((uint64_t)v >= sigma) { free(A); free(T); free(X); return OR_ESYMBOL; }
    A[i] = v;
  }
  oracle_wm *m = (oracle_wm *)calloc(1, sizeof(oracle_wm));
  if (!m) { free(A); free(T); free(X); return OR_ENOMEM; }
  m->n = n;
  m->sigma = sigma;
  m->levels = L;
  m->elem_bytes = elem_bytes;
  m->words_per_level = ((n + 511) / 512) * 8;
  m->blocks_per_level = (n + 511) / 512;
  m->supers_per_level = (n + 65535) / 65536 + 1;
  uint64_t nbits = (uint64_t)L * m->words_per_level;
  m->bits = (uint64_t *)calloc(nbits ? nbits : 1, sizeof(uint64_t));
  m->zeros = (uint64_t *)calloc(L ? L : 1, sizeof(uint64_t));
  m->rank_block = (uint16_t *)calloc(L * m->blocks_per_level + 1, sizeof(uint16_t));
  m->rank_super = (uint64_t *)calloc(L * m->supers_per_level + 1, sizeof(uint64_t));
  if (!m->bits || !m->zeros || !m->rank_block || !m->rank_super) {
    free(A); free(T); free(X); oracle_wm_free(m);
    return OR_ENOMEM;
  }
  for (uint32_t l = 0; l < L; l++) {
    uint32_t shift = L - (l + 1); /* the (l+1)'st highest bit (:915-916) */
    uint64_t *B = m->bits + (uint64_t)l * m->words_per_level;
    /* X[i] = 1 for a 0 bit; exclusive prefix sum X, total X_s = zeros (Fig. 1 l.12-14) */
    uint64_t Xs = 0;
    for (uint64_t i = 0; i < n; i++) {
      X[i] = (uint32_t)Xs;
      Xs += ((A[i] >> shift) & 1u) == 0;
    }
    m->zeros[l] = Xs;
    /* fill the bitmap and reorder stably, zeros first (Fig. 1 l.15-17, one node) */
    for (uint64_t i = 0; i < n; i++) {
      if ((A[i] >> shift) & 1u) {
        B[i >> 6] |= (uint64_t)1 << (i & 63);
        T[Xs + i - X[i]] = A[i];
      } else {
        T[X[i]] = A[i];
      }
    }
    uint32_t *tmp = A; A = T; T = tmp; /* swap(S, S') */
  }
  free(A); free(T); free(X);
  rank_directory(m->bits, L, m->words_per_level, m->blocks_per_level, m->supers_per_level, m->rank_block,
                 m->rank_super);
  *out = m;
  return OR_OK;
}

static uint64_t wm_rank1(const oracle_wm *m, uint32_t l, uint64_t i) {
  if (i >= m->n) return m->rank_super[(uint64_t)l * m->supers_per_level + m->supers_per_level - 1];
  const uint64_t *B = m->bits + (uint64_t)l * m->words_per_level;
  uint64_t r = m->rank_super[(uint64_t)l * m->supers_per_level + (i >> 16)];
  r += m->rank_block[(uint64_t)l * m->blocks_per_level + (i >> 9)];
  for (uint64_t w = (i >> 9) * 8; w < (i >> 6); w++) r += popcount64(B[w]);
  if (i & 63) r += popcount64(B[i >> 6] & (((uint64_t)1 << (i & 63)) - 1));
  return r;
}

/* access(i): the bit at i selects the side; a 0 moves to rank0(i), a 1 to
 * zeros[l] + rank1(i) (the reorder of :917-921 applied to one position) */
uint32_t oracle_wm_access(const oracle_wm *m, uint64_t i) {
  if (!m || i >= m->n) return UINT32_MAX;
  uint32_t sym = 0;
  for (uint32_t l = 0; l < m->levels; l++) {
    const uint64_t *B = m->bits + (uint64_t)l * m->words_per_level;
    uint32_t bit = (uint32_t)((B[i >> 6] >> (i & 63)) & 1u);
    uint64_t r1 = wm_rank1(m, l, i);
    sym = (sym << 1) | bit;
    i = bit ? m->zeros[l] + r1 : i - r1;
  }
  return sym;
}

/* rank_c(i), inclusive (:205-206): track the range [s, e) of the positions
 * 0..i that share c's leading bits, level by level */
uint64_t oracle_wm_rank(const oracle_wm *m, uint32_t c, uint64_t i) {
  if (!m || i >= m->n || (uint64_t)c >= m->sigma) return UINT64_MAX;
  uint64_t s = 0, e = i + 1;
  for (uint32_t l = 0; l < m->levels; l++) {
    uint64_t r1s = wm_rank1(m, l, s), r1e = wm_rank1(m, l, e);
    if ((c >> (m->levels - 1 - l)) & 1u) {
      s = m->zeros[l] + r1s;
      e = m->zeros[l] + r1e;
    } else {
      s = s - r1s;
      e = e - r1e;
    }
    if (s == e) return 0;
  }
  return e - s;
}

/* ======================================================================
 * Select (§6 :827-845).
 *
 * select_c(S, k) = position of the k'th occurrence of c (k >= 1, 0-based
 * positions; UINT64_MAX when k == 0, k > the count of c, or c >= sigma).
 *
 * Select directory (Clark's first level, :827-829, with DESIGN.md reading
 * R-14 fixing the sampling): per level, the positions of all 1 bits (and of
 * all 0 bits) are computed "using a prefix sum and filter" (:839-841) and
 * every 4096'th is kept: sel1[l*SPS + j] = position of the (4096 j)'th 1 bit
 * (0-based count), sel0 likewise for 0 bits; SPS = ceil(n / 4096) + 1 and
 * entries past the last sample are n.
 *
 * select_b(l, k) on a level bitmap scans forward from the sample of the
 * k'th b-bit; select_c descends top-down to find c's node (tree) or class
 * start (matrix) at every level, then climbs back up with select_b.
 * ====================================================================== */
#define OR_SEL_SAMPLE 4096u

static uint64_t sel_per_level(uint64_t n) { return (n + OR_SEL_SAMPLE - 1) / OR_SEL_SAMPLE + 1; }

/* filter the positions of the b-bits of one level, keep every 4096'th */
static void select_samples(const uint64_t *B, uint64_t n, uint32_t b, uint32_t *out, uint64_t sps) {
  uint64_t cnt = 0, j = 0;
  for (uint64_t i = 0; i < n; i++) {
    uint32_t bit = (uint32_t)((B[i >> 6] >> (i & 63)) & 1u);
    if (bit == b) {
      if (cnt % OR_SEL_SAMPLE == 0) out[j++] = (uint32_t)i;
      cnt++;
    }
  }
  for (; j < sps; j++) out[j] = (uint32_t)n;
}

/* select_b(l, k): position of the k'th (1-based) b-bit of a level; n if none */
static uint64_t level_select(const uint64_t *B, uint64_t n, const uint32_t *samples, uint32_t b, uint64_t k) {
  if (k == 0) return n;
  uint64_t j = (k - 1) / OR_SEL_SAMPLE;
  uint64_t i = samples[j];
  if (i >= n) return n;
  uint64_t need = (k - 1) % OR_SEL_SAMPLE; /* b-bits still to skip after the sample */
  for (; i < n; i++) {
    uint32_t bit = (uint32_t)((B[i >> 6] >> (i & 63)) & 1u);
    if (bit == b) {
      if (need == 0) return i;
      need--;
    }
  }
  return n;
}

/* --- tree --- */
int oracle_select_dir(const oracle_tree *t, uint32_t **sel0, uint32_t **sel1, uint64_t *sps_out) {
  if (!t || !sel0 || !sel1 || !sps_out) return OR_EINVAL;
  uint64_t sps = sel_per_level(t->n);
  uint32_t *s0 = (uint32_t *)malloc((t->levels * sps + 1) * sizeof(uint32_t));
  uint32_t *s1 = (uint32_t *)malloc((t->levels * sps + 1) * sizeof(uint32_t));
  if (!s0 || !s1) { free(s0); free(s1); return OR_ENOMEM; }
  for (uint32_t l = 0; l < t->levels; l++) {
    const uint64_t *B = t->bits + (uint64_t)l * t->words_per_level;
    select_samples(B, t->n, 0, s0 + (uint64_t)l * sps, sps);
    select_samples(B, t->n, 1, s1 + (uint64_t)l * sps, sps);
  }
  *sel0 = s0; *sel1 = s1; *sps_out = sps;
  return OR_OK;
}

void oracle_free_buf(void *p) { free(p); }

/* select_c(S, k) on the tree: top-down node ranges [s_l, e_l) of c's prefix
 * (as rank does), then bottom-up: the offset p inside the level-(l+1) child
 * becomes select_b(level l, rank_b(s_l) + p + 1) - s_l. */
uint64_t oracle_select(const oracle_tree *t, const uint32_t *sel0, const uint32_t *sel1, uint64_t sps, uint32_t c,
                       uint64_t k) {
  if (!t || (uint64_t)c >= t->sigma || k == 0 || k > t->n) return UINT64_MAX;
  uint32_t L = t->levels;
  uint64_t s[33], e[33];
  s[0] = 0; e[0] = t->n;
  for (uint32_t l = 0; l < L; l++) {
    uint64_t r1s = rank1(t, l, s[l]), r1e = rank1(t, l, e[l]);
    uint64_t z = (e[l] - s[l]) - (r1e - r1s);
    if ((c >> (L - 1 - l)) & 1u) { s[l + 1] = s[l] + z; e[l + 1] = e[l]; }
    else { s[l + 1] = s[l]; e[l + 1] = s[l] + z; }
  }
  if (k > e[L] - s[L]) return UINT64_MAX; /* fewer than k occurrences of c */
  uint64_t p = k - 1;                      /* offset inside c's range at level L */
  for (uint32_t l = L; l-- > 0;) {
    const uint64_t *B = t->bits + (uint64_t)l * t->words_per_level;
    uint32_t b = (c >> (L - 1 - l)) & 1u;
    uint64_t before = b ? rank1(t, l, s[l]) : s[l] - rank1(t, l, s[l]);
    uint64_t q = level_select(B, t->n, (b ? sel1 : sel0) + (uint64_t)l * sps, b, before + p + 1);
    p = q - s[l];
  }
  return p;
}

/* --- matrix --- */
int oracle_wm_select_dir(const oracle_wm *m, uint32_t **sel0, uint32_t **sel1, uint64_t *sps_out) {
  if (!m || !sel0 || !sel1 || !sps_out) return OR_EINVAL;
  uint64_t sps = sel_per_level(m->n);
  uint32_t *s0 = (uint32_t *)malloc((m->levels * sps + 1) * sizeof(uint32_t));
  uint32_t *s1 = (uint32_t *)malloc((m->levels * sps + 1) * sizeof(uint32_t));
  if (!s0 || !s1) { free(s0); free(s1); return OR_ENOMEM; }
  for (uint32_t l = 0; l < m->levels; l++) {
    const uint64_t *B = m->bits + (uint64_t)l * m->words_per_level;
    select_samples(B, m->n, 0, s0 + (uint64_t)l * sps, sps);
    select_samples(B, m->n, 1, s1 + (uint64_t)l * sps, sps);
  }
  *sel0 = s0; *sel1 = s1; *sps_out = sps;
  return OR_OK;
}

/* select_c on the matrix: c's class start at every level top-down
 * (s_{l+1} = b ? zeros[l] + rank1(s_l) : rank0(s_l)), then bottom-up
 * p_l = select_b(level l, rank_b(s_l) + (p_{l+1} - s_{l+1}) + 1). */
uint64_t oracle_wm_select(const oracle_wm *m, const uint32_t *sel0, const uint32_t *sel1, uint64_t sps, uint32_t c,
                          uint64_t k) {
  if (!m || (uint64_t)c >= m->sigma || k == 0 || k > m->n) return UINT64_MAX;
  uint32_t L = m->levels;
  uint64_t s[33], e[33];
  s[0] = 0; e[0] = m->n;
  for (uint32_t l = 0; l < L; l++) {
    uint64_t r1s = wm_rank1(m, l, s[l]), r1e = wm_rank1(m, l, e[l]);
    if ((c >> (L - 1 - l)) & 1u) { s[l + 1] = m->zeros[l] + r1s; e[l + 1] = m->zeros[l] + r1e; }
    else { s[l + 1] = s[l] - r1s; e[l + 1] = e[l] - r1e; }
  }
  if (k > e[L] - s[L]) return UINT64_MAX;
  uint64_t p = s[L] + k - 1; /* position at the (virtual) level L */
  for (uint32_t l = L; l-- > 0;) {
    const uint64_t *B = m->bits + (uint64_t)l * m->words_per_level;
    uint32_t b = (c >> (L - 1 - l)) & 1u;
    uint64_t r1s = wm_rank1(m, l, s[l]);
    uint64_t before = b ? r1s : s[l] - r1s;
    uint64_t off = p - s[l + 1];
    p = level_select(B, m->n, (b ? sel1 : sel0) + (uint64_t)l * sps, b, before + off + 1);
  }
  return p;
}
