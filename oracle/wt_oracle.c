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
#define OR_EUNSUPPORTED (-5)

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

/* ======================================================================
 * Huffman-shaped wavelet tree (§7 "Extensions"; SURVEY
 * §8(f) f3).
 *
 *   "each node is placed at a level proportional to the length of its
 *    Huffman code" (:855-856); "we first compute the Huffman tree and
 *    prefix codes" (:858-859); "We map each symbol to an integer
 *    corresponding to the location of its leaf in an in-order traversal of
 *    the Huffman tree ... At each internal node ... we store the highest
 *    mapped integer of nodes in its left sub-tree ... the decision of how to
 *    set the bitmap and where to place the symbol in S' can be made with a
 *    single comparison with the mapped integers.  The rest of the
 *    computation follows the logic of levelWT." (:862-873)
 *
 * Readings (R-17..R-20):
 *   R-17 Huffman tree: the textbook two-queue construction over the symbols
 *        that occur, leaves ordered by (frequency, symbol) ascending; each
 *        step removes the two lightest items, a leaf before an internal
 *        node of equal weight.  Code lengths = leaf depths.
 *   R-18 Codes: canonical codes for those lengths (symbols ordered by
 *        (length, symbol); the first code is all zeros; each next code is
 *        (previous + 1) shifted left by the length increase).  The
 *        wavelet tree has the shape of the canonical code trie; a 0 code
 *        bit goes left (:220-224).
 *   R-19 Levels: level l holds, for every element still inside an internal
 *        node at depth l, its code bit l; elements whose leaf is reached
 *        leave the sequence (levelWT's S' keeps only internal children).
 *        Nodes in each level in left-to-right (key) order; node key = the
 *        l-bit code prefix.  Each level's bitmap, directory and node list
 *        use the same per-level layout as the balanced tree, with levels
 *        concatenated (word/block/super offsets per level).
 *   R-20 Fewer than two distinct symbols: the root is a leaf, 0 levels.
 * ====================================================================== */
typedef struct {
  uint64_t n;
  uint64_t sigma;
  uint32_t levels;          /* h = longest code length                     */
  uint32_t elem_bytes;
  uint64_t *level_len;      /* levels: n_l = elements inside depth-l nodes */
  uint64_t *level_word_ptr; /* levels + 1: ceil(n_l/512)*8 words per level  */
  uint64_t *level_block_ptr;/* levels + 1: ceil(n_l/512) blocks per level   */
  uint64_t *level_super_ptr;/* levels + 1: ceil(n_l/65536)+1 per level      */
  uint64_t *bits;
  uint16_t *rank_block;
  uint64_t *rank_super;
  uint64_t *level_node_ptr; /* levels + 1 */
  uint32_t *node_key;       /* l-bit code prefix of the internal node      */
  uint32_t *node_start;     /* first position of the node in its level     */
  uint64_t total_nodes;
  uint32_t *code;           /* sigma: canonical code (right-aligned)       */
  uint8_t *code_len;        /* sigma: code length, 0 = symbol absent       */
  uint32_t only_symbol;     /* levels == 0 and n > 0: the one symbol (R-20) */
} oracle_hwt;

/* explicit binary tree node (Huffman tree, then the canonical trie) */
typedef struct {
  uint64_t weight;
  int32_t child[2];  /* -1 for a leaf */
  int32_t sym;       /* leaf symbol, -1 for internal */
  uint32_t thr;      /* internal: highest mapped integer of the left subtree */
  uint64_t start;    /* internal: first position at its level */
} or_hnode;

void oracle_hwt_free(oracle_hwt *t) {
  if (!t) return;
  free(t->level_len); free(t->level_word_ptr); free(t->level_block_ptr); free(t->level_super_ptr);
  free(t->bits); free(t->rank_block); free(t->rank_super);
  free(t->level_node_ptr); free(t->node_key); free(t->node_start);
  free(t->code); free(t->code_len);
  free(t);
}

static int cmp_leaf(const void *a, const void *b) {
  /* (frequency, symbol) ascending; entries are (freq << 32 | sym) */
  uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* depth of every leaf under node v (recursive walk) */
static void leaf_depths(const or_hnode *T, int32_t v, uint32_t d, uint8_t *len, uint32_t *maxd) {
  if (T[v].sym >= 0) {
    len[T[v].sym] = (uint8_t)(d > 255 ? 255 : d);
    if (d > *maxd) *maxd = d;
    return;
  }
  leaf_depths(T, T[v].child[0], d + 1, len, maxd);
  leaf_depths(T, T[v].child[1], d + 1, len, maxd);
}

/* R-17: two-queue Huffman construction; writes len[sym] (0 = absent) and
 * returns the longest length.  m = number of occurring symbols. */
static int huffman_lengths(const uint64_t *freq, uint64_t sigma, uint8_t *len, uint32_t *h_out) {
  uint64_t m = 0;
  for (uint64_t c = 0; c < sigma; c++) m += freq[c] > 0;
  memset(len, 0, sigma);
  *h_out = 0;
  if (m < 2) return 0; /* R-20 */
  uint64_t *leaf = (uint64_t *)malloc(m * sizeof(uint64_t));
  or_hnode *T = (or_hnode *)malloc((2 * m) * sizeof(or_hnode));
  if (!leaf || !T) { free(leaf); free(T); return -1; }
  uint64_t k = 0;
  for (uint64_t c = 0; c < sigma; c++)
    if (freq[c]) leaf[k++] = (freq[c] << 32) | c;
  qsort(leaf, m, sizeof(uint64_t), cmp_leaf);
  for (uint64_t i = 0; i < m; i++) {
    T[i].weight = leaf[i] >> 32;
    T[i].sym = (int32_t)(leaf[i] & 0xffffffffu);
    T[i].child[0] = T[i].child[1] = -1;
  }
  /* queue 1 = leaves [lq, m); queue 2 = internal nodes [iq, nint) */
  uint64_t lq = 0, iq = m, nint = m;
  for (uint64_t step = 0; step + 1 < m; step++) {
    int32_t pick[2];
    for (int j = 0; j < 2; j++) {
      int take_leaf;
      if (lq >= m) take_leaf = 0;
      else if (iq >= nint) take_leaf = 1;
      else take_leaf = T[lq].weight <= T[iq].weight; /* a leaf first on ties */
      pick[j] = (int32_t)(take_leaf ? lq++ : iq++);
    }
    T[nint].weight = T[pick[0]].weight + T[pick[1]].weight;
    T[nint].child[0] = pick[0];
    T[nint].child[1] = pick[1];
    T[nint].sym = -1;
    nint++;
  }
  leaf_depths(T, (int32_t)(nint - 1), 0, len, h_out);
  free(leaf);
  free(T);
  return 0;
}

/* R-18: canonical codes from the lengths */
static void canonical_codes(const uint8_t *len, uint64_t sigma, uint32_t h, uint32_t *code) {
  memset(code, 0, sigma * sizeof(uint32_t));
  uint64_t cur = 0;
  uint32_t prev = 0;
  int first = 1;
  for (uint32_t L = 1; L <= h; L++) {
    for (uint64_t c = 0; c < sigma; c++) {
      if (len[c] != L) continue;
      if (first) { cur = 0; first = 0; }
      else cur = (cur + 1) << (L - prev);
      prev = L;
      code[c] = (uint32_t)cur;
    }
  }
}

/* in-order numbering of the trie: leaves get 0, 1, 2, ...; every internal
 * node records the highest number in its left subtree (:864-869) */
static uint32_t inorder_map(or_hnode *T, int32_t v, uint32_t next, uint32_t *map) {
  if (T[v].sym >= 0) { map[T[v].sym] = next; return next + 1; }
  next = inorder_map(T, T[v].child[0], next, map);
  T[v].thr = next - 1;
  return inorder_map(T, T[v].child[1], next, map);
}

int oracle_hwt_build(const void *seq, uint64_t n, uint32_t elem_bytes, uint64_t sigma, oracle_hwt **out) {
  if (!out) return OR_EINVAL;
  *out = NULL;
  if ((n > 0 && !seq) || (elem_bytes != 1 && elem_bytes != 2 && elem_bytes != 4))
    return OR_EINVAL;
  if (sigma < 1 || sigma > ((uint64_t)1 << (8 * elem_bytes)) || sigma > 65536 || n >= ((uint64_t)1 << 32))
    return OR_EINVAL;
  uint32_t *S = (uint32_t *)malloc((n ? n : 1) * sizeof(uint32_t));
  uint64_t *freq = (uint64_t *)calloc(sigma, sizeof(uint64_t));
  if (!S || !freq) { free(S); free(freq); return OR_ENOMEM; }
  for (uint64_t i = 0; i < n; i++) {
    uint32_t v;
    if (elem_bytes == 1) v = ((const uint8_t *)seq)[i];
    else if (elem_bytes == 2) v = ((const uint16_t *)seq)[i];
    else v = ((const uint32_t *)seq)[i];
    if ((uint64_t)v >= sigma) { free(S); free(freq); return OR_ESYMBOL; }
    S[i] = v;
    freq[v]++;
  }
  oracle_hwt *t = (oracle_hwt *)calloc(1, sizeof(oracle_hwt));
  if (!t) { free(S); free(freq); return OR_ENOMEM; }
  t->n = n;
  t->sigma = sigma;
  t->elem_bytes = elem_bytes;
  t->code = (uint32_t *)calloc(sigma, sizeof(uint32_t));
  t->code_len = (uint8_t *)calloc(sigma, 1);
  uint32_t h = 0;
  if (!t->code || !t->code_len || huffman_lengths(freq, sigma, t->code_len, &h)) {
    free(S); free(freq); oracle_hwt_free(t);
    return OR_ENOMEM;
  }
  if (h > 32) { free(S); free(freq); oracle_hwt_free(t); return OR_EUNSUPPORTED; }
  canonical_codes(t->code_len, sigma, h, t->code);
  t->levels = h;
  for (uint64_t c = 0; c < sigma; c++)
    if (freq[c]) { t->only_symbol = (uint32_t)c; break; }

  /* the canonical trie: insert every code; node 0 is the root */
  uint64_t m = 0;
  for (uint64_t c = 0; c < sigma; c++) m += t->code_len[c] > 0;
  uint64_t cap = 2 * (m ? m : 1);
  or_hnode *T = (or_hnode *)calloc(cap, sizeof(or_hnode));
  uint32_t *map = (uint32_t *)calloc(sigma, sizeof(uint32_t));
  if (!T || !map) { free(T); free(map); free(S); free(freq); oracle_hwt_free(t); return OR_ENOMEM; }
  uint64_t nn = 1;
  T[0].child[0] = T[0].child[1] = -1;
  T[0].sym = -1;
  for (uint64_t c = 0; c < sigma && h > 0; c++) {
    uint32_t L = t->code_len[c];
    if (!L) continue;
    int32_t v = 0;
    for (uint32_t d = 0; d < L; d++) {
      uint32_t b = (t->code[c] >> (L - 1 - d)) & 1u;
      if (T[v].child[b] < 0) {
        T[nn].child[0] = T[nn].child[1] = -1;
        T[nn].sym = -1;
        T[v].child[b] = (int32_t)nn++;
      }
      v = T[v].child[b];
    }
    T[v].sym = (int32_t)c;
  }
  if (h > 0) inorder_map(T, 0, 0, map);

  /* levelWT over the Huffman shape (:870-873, R-19): breadth first, level by level */
  t->level_len = (uint64_t *)calloc(h ? h : 1, sizeof(uint64_t));
  t->level_word_ptr = (uint64_t *)calloc(h + 1, sizeof(uint64_t));
  t->level_block_ptr = (uint64_t *)calloc(h + 1, sizeof(uint64_t));
  t->level_super_ptr = (uint64_t *)calloc(h + 1, sizeof(uint64_t));
  t->level_node_ptr = (uint64_t *)calloc(h + 1, sizeof(uint64_t));
  uint32_t *A = (uint32_t *)malloc((n ? n : 1) * sizeof(uint32_t)); /* mapped integers of level l */
  uint32_t *Anext = (uint32_t *)malloc((n ? n : 1) * sizeof(uint32_t));
  uint32_t *X = (uint32_t *)malloc((n ? n : 1) * sizeof(uint32_t));
  int32_t *cur = (int32_t *)malloc(cap * sizeof(int32_t)), *nxt = (int32_t *)malloc(cap * sizeof(int32_t));
  uint32_t *ckey = (uint32_t *)malloc(cap * sizeof(uint32_t)), *nkey = (uint32_t *)malloc(cap * sizeof(uint32_t));
  uint64_t *clen = (uint64_t *)malloc(cap * sizeof(uint64_t)), *nlen = (uint64_t *)malloc(cap * sizeof(uint64_t));
  node_list *nodes = (node_list *)calloc(h ? h : 1, sizeof(node_list));
  uint64_t **lbits = (uint64_t **)calloc(h ? h : 1, sizeof(uint64_t *));
  int oom = !t->level_len || !t->level_word_ptr || !t->level_block_ptr || !t->level_super_ptr ||
            !t->level_node_ptr || !A || !Anext || !X || !cur || !nxt || !ckey || !nkey || !clen || !nlen ||
            !nodes || !lbits;
  uint64_t ncur = 0, nl = n;
  if (!oom && h > 0 && n > 0) {
    for (uint64_t i = 0; i < n; i++) A[i] = map[S[i]];
    cur[0] = 0; ckey[0] = 0; clen[0] = n; ncur = 1;
  }
  for (uint32_t l = 0; l < h && !oom; l++) {
    t->level_len[l] = nl;
    uint64_t wl = (nl + 511) / 512 * 8;
    lbits[l] = (uint64_t *)calloc(wl ? wl : 1, sizeof(uint64_t));
    if (!lbits[l]) { oom = 1; break; }
    uint64_t pos = 0, nnext = 0, nout = 0;
    for (uint64_t j = 0; j < ncur; j++) {
      const or_hnode *v = &T[cur[j]];
      uint64_t s = pos, len = clen[j];
      if (push_node(&nodes[l], ckey[j], (uint32_t)s)) { oom = 1; break; }
      T[cur[j]].start = s;
      /* Fig. 1 l.12-14 with the comparison of :870-872: X[i] = 1 when the
       * mapped integer is at most thr (the symbol is in the left subtree) */
      uint64_t Xs = 0;
      for (uint64_t i = 0; i < len; i++) {
        X[s + i] = (uint32_t)Xs;
        Xs += A[s + i] <= v->thr;
      }
      /* children (Fig. 1 l.18-19): only internal children continue to level l+1 */
      const int32_t cl = v->child[0], cr = v->child[1];
      const int keep_l = T[cl].sym < 0 && Xs > 0, keep_r = T[cr].sym < 0 && len - Xs > 0;
      const uint64_t lbase = nout, rbase = nout + (keep_l ? Xs : 0);
      /* Fig. 1 l.15-17: set the bit; a left symbol goes to X[i], a right one to X_s + i - X[i] */
      for (uint64_t i = 0; i < len; i++) {
        uint32_t a = A[s + i];
        if (a > v->thr) {
          lbits[l][(s + i) >> 6] |= (uint64_t)1 << ((s + i) & 63);
          if (keep_r) Anext[rbase + i - X[s + i]] = a;
        } else if (keep_l) {
          Anext[lbase + X[s + i]] = a;
        }
      }
      if (keep_l) { nxt[nnext] = cl; nkey[nnext] = 2 * ckey[j]; nlen[nnext] = Xs; nnext++; }
      if (keep_r) { nxt[nnext] = cr; nkey[nnext] = 2 * ckey[j] + 1; nlen[nnext] = len - Xs; nnext++; }
      nout += (keep_l ? Xs : 0) + (keep_r ? len - Xs : 0);
      pos += len;
    }
    { uint32_t *tmp = A; A = Anext; Anext = tmp; }
    { int32_t *tmp = cur; cur = nxt; nxt = tmp; }
    { uint32_t *tmp = ckey; ckey = nkey; nkey = tmp; }
    { uint64_t *tmp = clen; clen = nlen; nlen = tmp; }
    ncur = nnext;
    nl = nout;
  }
  free(A); free(Anext); free(X); free(cur); free(nxt); free(ckey); free(nkey); free(clen); free(nlen);
  free(S); free(freq); free(map); free(T);

  if (!oom) {
    for (uint32_t l = 0; l < h; l++) {
      uint64_t nlv = t->level_len[l];
      t->level_word_ptr[l + 1] = t->level_word_ptr[l] + (nlv + 511) / 512 * 8;
      t->level_block_ptr[l + 1] = t->level_block_ptr[l] + (nlv + 511) / 512;
      t->level_super_ptr[l + 1] = t->level_super_ptr[l] + (nlv + 65535) / 65536 + 1;
      t->level_node_ptr[l + 1] = t->level_node_ptr[l] + nodes[l].len;
    }
    t->total_nodes = t->level_node_ptr[h];
    t->bits = (uint64_t *)calloc(t->level_word_ptr[h] + 1, sizeof(uint64_t));
    t->rank_block = (uint16_t *)calloc(t->level_block_ptr[h] + 1, sizeof(uint16_t));
    t->rank_super = (uint64_t *)calloc(t->level_super_ptr[h] + 1, sizeof(uint64_t));
    t->node_key = (uint32_t *)malloc((t->total_nodes + 1) * sizeof(uint32_t));
    t->node_start = (uint32_t *)malloc((t->total_nodes + 1) * sizeof(uint32_t));
    oom = !t->bits || !t->rank_block || !t->rank_super || !t->node_key || !t->node_start;
  }
  for (uint32_t l = 0; l < h; l++) {
    if (!oom) {
      uint64_t wl = t->level_word_ptr[l + 1] - t->level_word_ptr[l];
      if (wl) memcpy(t->bits + t->level_word_ptr[l], lbits[l], wl * sizeof(uint64_t));
      uint64_t off = t->level_node_ptr[l];
      if (nodes[l].len) {
        memcpy(t->node_key + off, nodes[l].key, nodes[l].len * sizeof(uint32_t));
        memcpy(t->node_start + off, nodes[l].start, nodes[l].len * sizeof(uint32_t));
      }
      rank_directory(t->bits + t->level_word_ptr[l], 1, wl, t->level_block_ptr[l + 1] - t->level_block_ptr[l],
                     t->level_super_ptr[l + 1] - t->level_super_ptr[l], t->rank_block + t->level_block_ptr[l],
                     t->rank_super + t->level_super_ptr[l]);
    }
    free(lbits[l]);
    free(nodes[l].key);
    free(nodes[l].start);
  }
  free(lbits);
  free(nodes);
  if (oom) { oracle_hwt_free(t); return OR_ENOMEM; }
  *out = t;
  return OR_OK;
}

/* rank1 of level l of the Huffman-shaped tree: ones in [0, i) */
static uint64_t hwt_rank1(const oracle_hwt *t, uint32_t l, uint64_t i) {
  const uint64_t nl = t->level_len[l];
  const uint64_t *sup = t->rank_super + t->level_super_ptr[l];
  if (i >= nl) return sup[t->level_super_ptr[l + 1] - t->level_super_ptr[l] - 1];
  const uint64_t *B = t->bits + t->level_word_ptr[l];
  uint64_t r = sup[i >> 16] + t->rank_block[t->level_block_ptr[l] + (i >> 9)];
  for (uint64_t w = (i >> 9) * 8; w < (i >> 6); w++) r += popcount64(B[w]);
  if (i & 63) r += popcount64(B[i >> 6] & (((uint64_t)1 << (i & 63)) - 1));
  return r;
}

/* node of level l with key p: (start, end) by a linear scan of the level's list */
static int hwt_node(const oracle_hwt *t, uint32_t l, uint32_t p, uint64_t *s, uint64_t *e) {
  for (uint64_t j = t->level_node_ptr[l]; j < t->level_node_ptr[l + 1]; j++) {
    if (t->node_key[j] == p) {
      *s = t->node_start[j];
      *e = j + 1 < t->level_node_ptr[l + 1] ? t->node_start[j + 1] : t->level_len[l];
      return 1;
    }
  }
  return 0;
}

/* the symbol whose code is the l-bit value p, or -1 */
static int64_t hwt_leaf(const oracle_hwt *t, uint32_t l, uint32_t p) {
  for (uint64_t c = 0; c < t->sigma; c++)
    if (t->code_len[c] == l && t->code[c] == p) return (int64_t)c;
  return -1;
}

/* access(i): descend; a 0 bit keeps rank0 within the node, a 1 bit rank1;
 * stop when the code read so far is a leaf */
uint32_t oracle_hwt_access(const oracle_hwt *t, uint64_t i) {
  if (!t || i >= t->n) return UINT32_MAX;
  if (t->levels == 0) return t->only_symbol; /* R-20: the root is the leaf */
  uint32_t p = 0;
  uint64_t s = 0, e = t->n;
  for (uint32_t l = 0; l < t->levels; l++) {
    const uint64_t *B = t->bits + t->level_word_ptr[l];
    uint32_t bit = (uint32_t)((B[i >> 6] >> (i & 63)) & 1u);
    uint64_t r1s = hwt_rank1(t, l, s), r1i = hwt_rank1(t, l, i);
    uint64_t r = bit ? r1i - r1s : (i - s) - (r1i - r1s); /* rank within the node */
    p = 2 * p + bit;
    int64_t sym = hwt_leaf(t, l + 1, p);
    if (sym >= 0) return (uint32_t)sym;
    if (!hwt_node(t, l + 1, p, &s, &e)) return UINT32_MAX;
    i = s + r;
  }
  return UINT32_MAX;
}

/* rank_c(i), inclusive: follow c's code, counting within each node */
uint64_t oracle_hwt_rank(const oracle_hwt *t, uint32_t c, uint64_t i) {
  if (!t || i >= t->n || (uint64_t)c >= t->sigma) return UINT64_MAX;
  uint32_t L = t->code_len[c];
  if (t->levels == 0) return c == t->only_symbol ? i + 1 : 0; /* R-20 */
  if (L == 0) return 0;
  uint64_t s = 0, e = t->n, r = i + 1;
  uint32_t p = 0;
  for (uint32_t l = 0; l < L; l++) {
    uint32_t bit = (t->code[c] >> (L - 1 - l)) & 1u;
    uint64_t r1s = hwt_rank1(t, l, s), r1p = hwt_rank1(t, l, s + r);
    r = bit ? r1p - r1s : r - (r1p - r1s);
    if (r == 0) return 0;
    p = 2 * p + bit;
    if (l + 1 == L) break;
    if (!hwt_node(t, l + 1, p, &s, &e)) return UINT64_MAX;
  }
  (void)e;
  return r;
}

/* select_c(S, k) on the Huffman-shaped tree (PAPER.md:207-208 with the tree
 * walk of :204-206): descend along c's code to find the node of every level,
 * then climb from the deepest node -- the k'th occurrence of c is the k'th
 * bit equal to c's last code bit inside that node, and at every level above
 * the r'th position of the child is the r'th bit equal to the level's code
 * bit inside the parent.  Bits are found by a plain scan of the level. */
static uint64_t hwt_select_bit(const oracle_hwt *t, uint32_t l, uint64_t s, uint64_t e, uint32_t b, uint64_t j) {
  const uint64_t *B = t->bits + t->level_word_ptr[l];
  for (uint64_t i = s; i < e; i++) {
    if ((uint32_t)((B[i >> 6] >> (i & 63)) & 1u) == b) {
      if (--j == 0) return i;
    }
  }
  return UINT64_MAX;
}

uint64_t oracle_hwt_select(const oracle_hwt *t, uint32_t c, uint64_t k) {
  if (!t || (uint64_t)c >= t->sigma || k == 0) return UINT64_MAX;
  if (t->levels == 0) return (t->n && c == t->only_symbol && k <= t->n) ? k - 1 : UINT64_MAX;
  uint32_t L = t->code_len[c];
  if (L == 0) return UINT64_MAX;
  uint64_t s[64], e[64];
  s[0] = 0;
  e[0] = t->level_len[0];
  uint32_t p = 0;
  for (uint32_t l = 0; l + 1 < L; l++) {
    p = 2 * p + ((t->code[c] >> (L - 1 - l)) & 1u);
    if (!hwt_node(t, l + 1, p, &s[l + 1], &e[l + 1])) return UINT64_MAX;
  }
  uint64_t r = k;  /* 1-based rank inside the node of level l */
  for (int l = (int)L - 1; l >= 0; l--) {
    uint32_t b = (t->code[c] >> (L - 1 - (uint32_t)l)) & 1u;
    uint64_t pos = hwt_select_bit(t, (uint32_t)l, s[l], e[l], b, r);
    if (pos == UINT64_MAX) return UINT64_MAX;
    r = pos - s[l] + 1;
  }
  return r - 1;
}
