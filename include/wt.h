/*
 * wt.h -- C ABI of the B200 (sm_100a) levelwise wavelet-tree builder.
 *
 * The operation is the construction of arXiv 1407.8142 ("Parallel Wavelet
 * Tree Construction"), levelWT (Fig. 1): for an
 * integer sequence S of length n over the alphabet [0, sigma) (PAPER.md:
 * 201-203), L = ceil(log2 sigma) levels; level l
 * stores, for every element of S_l = S stably sorted by its top l bits
 * (PAPER.md:468-475), the element's (l+1)'st highest bit (mask
 * 2^(L-(l+1))); each node's sub-sequence is stably
 * split by that bit; the level's non-empty nodes
 * and a two-level rank directory are
 * emitted.  Queries follow PAPER.md:204-208.
 *
 * All pointers in this header are plain pointers; no C++ or torch types.
 * "Device pointer" means CUDA global memory of the current device.  Streams
 * are passed as `void*` holding a cudaStream_t (NULL = legacy default stream).
 *
 * Normative output layout ("Output layout"):
 *   bits      u64[levels * words_per_level], words_per_level = ceil(n/512)*8.
 *             Bit i of level l = (bits[l*WPL + (i>>6)] >> (i & 63)) & 1
 *             (LSB first, reading R-1).  Padding bits are 0.
 *   nodes     CSR over levels: level_node_ptr u64[levels+1]; entries
 *             j in [ptr[l], ptr[l+1]) are the level's non-empty nodes in
 *             ascending key order: node_key[j] = p (the node's top-l-bit
 *             prefix; heap id 2^l - 1 + p),
 *             node_start[j] = position of its first element at level l.
 *             A node's length is the next start (or n) minus its start.
 *   rank      blocks_per_level = ceil(n/512), supers_per_level =
 *             ceil(n/65536) + 1.  rank_super[l*SPL + s] = number of 1 bits
 *             of level l in [0, min(s*65536, n)) (last entry = level total);
 *             rank_block[l*BPL + b] = number of 1 bits in
 *             [floor(b/128)*65536, b*512) (always < 65536).
 *             rank1(l, i) = super[i>>16] + block[i>>9]
 *                         + popc(words of the block before word i>>6)
 *                         + popc(bits[i>>6] & ((1<<(i&63)) - 1)).
 */
#ifndef WT_B200_H
#define WT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Return codes. */
#define WT_OK 0
#define WT_EINVAL (-1)      /* null pointer, bad elem_bytes/sigma, n out of range   */
#define WT_ESYMBOL (-2)     /* some S[i] >= sigma; no tree is produced              */
#define WT_ENOMEM (-3)      /* device (or pinned host) allocation failed            */
#define WT_ECUDA (-4)       /* a CUDA runtime call or kernel launch failed          */
#define WT_EUNSUPPORTED (-5)/* reserved: valid input this build cannot handle        */

/* Read-only view of a built tree.  Every array pointer is a DEVICE pointer
 * owned by the library; it stays valid until wt_free(). */
typedef struct wt_tree {
  uint64_t n;                 /* sequence length                              */
  uint64_t sigma;             /* alphabet size                                */
  uint32_t levels;            /* L = ceil(log2 sigma) (0 when sigma == 1)     */
  uint32_t elem_bytes;        /* bytes per input symbol: 1, 2 or 4            */
  uint64_t words_per_level;   /* ceil(n/512) * 8                              */
  uint64_t *bits;             /* u64[levels * words_per_level]                */
  uint64_t *level_node_ptr;   /* u64[levels + 1]                              */
  uint32_t *node_key;         /* u32[total_nodes]                             */
  uint32_t *node_start;       /* u32[total_nodes]                             */
  uint64_t total_nodes;       /* level_node_ptr[levels]                       */
  uint64_t blocks_per_level;  /* ceil(n/512)                                  */
  uint64_t supers_per_level;  /* ceil(n/65536) + 1                            */
  uint16_t *rank_block;       /* u16[levels * blocks_per_level]               */
  uint64_t *rank_super;       /* u64[levels * supers_per_level]               */
  uint64_t select_per_level;  /* ceil(n/4096) + 1 (0 until wt_select_index)   */
  uint32_t *select0;          /* u32[levels * select_per_level] or NULL       */
  uint32_t *select1;          /* u32[levels * select_per_level] or NULL       */
  void *internal;             /* library bookkeeping; do not touch            */
} wt_tree;

/*
 * wt_build -- build the wavelet tree of S (Fig. 1; SURVEY §8(a)
 * steps A1-A7).
 *   d_seq      DEVICE pointer to n symbols of elem_bytes bytes each
 *              (little-endian unsigned).  Caller-owned, read-only, not
 *              retained after return.  Any alignment is accepted.
 *   n          sequence length, 0 <= n < 2^32.
 *   elem_bytes 1, 2 or 4.
 *   sigma      alphabet size, 1 <= sigma <= 2^(8*elem_bytes) (so up to 2^32,
 *              L = ceil(log2 sigma) <= 32 levels).
 *   stream     cudaStream_t (as void*) on which all work is enqueued.
 *   out        receives the tree on success, NULL on any error.
 * Work is enqueued on `stream`, which is then synchronised ONCE to read the
 * error flag and the per-level node counts; on WT_OK the tree is complete
 * and immutable.  Output memory is stream-ordered device memory owned by the
 * library and released only by wt_free().  On error nothing leaks.
 * n == 0 gives empty levels; sigma == 1 gives a tree with 0 levels.
 */
int wt_build(const void *d_seq, uint64_t n, uint32_t elem_bytes, uint64_t sigma,
             void *stream, wt_tree **out);

/*
 * wt_build_host -- as wt_build, but h_seq is a HOST pointer (pinned memory
 * gives full PCIe bandwidth; pageable memory is accepted).  The host->device
 * copy is enqueued on `stream` inside the call; everything else is identical
 * (the end-to-end path measured by bench.py's "e2e").
 */
int wt_build_host(const void *h_seq, uint64_t n, uint32_t elem_bytes, uint64_t sigma,
                  void *stream, wt_tree **out);

/* wt_free -- release everything owned by t: stream-ordered frees on the
 * build stream, after the work already enqueued on it and on every stream that
 * a query (wt_access / wt_rank / wt_select) or wt_select_index of this tree
 * used (the build stream waits for an event recorded on each).  Does not
 * synchronise the host.  NULL is a no-op.  Returns WT_ECUDA if a free failed. */
int wt_free(wt_tree *t);

/*
 * wt_access -- batched access(S, i) (batched queries
 * PAPER.md:275-277).  d_pos: DEVICE u64[q] positions; d_out: DEVICE u32[q]
 * receives S[pos[k]], or UINT32_MAX when pos[k] >= n.  Asynchronous on
 * `stream`; caller owns both buffers.  WT_EINVAL on null t, or null buffers
 * with q > 0.
 */
int wt_access(const wt_tree *t, const uint64_t *d_pos, uint64_t q, uint32_t *d_out,
              void *stream);

/*
 * wt_rank -- batched rank_c(S, i) = #{ j <= i : S[j] == c } (inclusive,
 * PAPER.md:205-206).  d_sym: DEVICE u32[q] symbols c; d_pos: DEVICE u64[q];
 * d_out: DEVICE u64[q], UINT64_MAX when pos >= n or c >= sigma.
 * Asynchronous; errors as wt_access.
 */
int wt_rank(const wt_tree *t, const uint32_t *d_sym, const uint64_t *d_pos, uint64_t q,
            uint64_t *d_out, void *stream);

/* ---- wavelet matrix ----
 *
 * Level l's bitmap holds the (l+1)'st highest bit of A_l, where A_0 = S and
 * A_{l+1} is A_l stably reordered by level l's bit, zeros first (:911-921);
 * equivalently A_l is S stably sorted by the reverse of its top l bits
 * (:924-925).  Each level stores its number of 0 bits (:914).  Bits, padding
 * and rank directory use exactly the layout of wt_tree above; there is no
 * node table (a level is one sequence).
 */
typedef struct wm_matrix {
  uint64_t n;                 /* sequence length                              */
  uint64_t sigma;             /* alphabet size                                */
  uint32_t levels;            /* L = ceil(log2 sigma)                         */
  uint32_t elem_bytes;        /* bytes per input symbol                       */
  uint64_t words_per_level;   /* ceil(n/512) * 8                              */
  uint64_t *bits;             /* u64[levels * words_per_level] (device)       */
  uint64_t *zeros;            /* u64[levels]: 0 bits of each level (device)   */
  uint64_t blocks_per_level;  /* ceil(n/512)                                  */
  uint64_t supers_per_level;  /* ceil(n/65536) + 1                            */
  uint16_t *rank_block;       /* u16[levels * blocks_per_level] (device)      */
  uint64_t *rank_super;       /* u64[levels * supers_per_level] (device)      */
  uint64_t select_per_level;  /* as wt_tree                                   */
  uint32_t *select0;
  uint32_t *select1;
  void *internal;             /* library bookkeeping; do not touch            */
} wm_matrix;

/* wm_build -- build the wavelet matrix of S.  Arguments, stream semantics,
 * ownership and errors exactly as wt_build (WT_ESYMBOL for S[i] >= sigma,
 * WT_EINVAL for bad arguments, one stream synchronisation at the end). */
int wm_build(const void *d_seq, uint64_t n, uint32_t elem_bytes, uint64_t sigma,
             void *stream, wm_matrix **out);
/* wm_free -- release everything owned by m; NULL is a no-op.  Ordered like
 * wt_free (after the build stream and every stream a query of m used). */
int wm_free(wm_matrix *m);
/* wm_access / wm_rank -- batched access(S, i) and inclusive rank_c(S, i)
 * on the matrix: a 0 bit at level l maps i to rank0(i),
 * a 1 bit to zeros[l] + rank1(i).  Buffers, sentinels and errors exactly as
 * wt_access / wt_rank. */
int wm_access(const wm_matrix *m, const uint64_t *d_pos, uint64_t q, uint32_t *d_out, void *stream);
int wm_rank(const wm_matrix *m, const uint32_t *d_sym, const uint64_t *d_pos, uint64_t q,
            uint64_t *d_out, void *stream);

/* ---- select ----
 *
 * Select directory (Clark's first level; DESIGN.md reading
 * R-14): per level, the positions of every 4096'th 0 bit and 1 bit --
 * select1[l*SPS + j] = position of the (4096 j)'th 1 bit of level l (0-based
 * count), select0 likewise for 0 bits, SPS = ceil(n/4096) + 1, entries past
 * the last sample are n.  Built on demand (the paper times construction
 * without rank/select, :649-651) by *_select_index, asynchronously on
 * `stream`, owned by the tree / matrix and released with it; idempotent.
 *
 * wt_select / wm_select -- batched select_c(S, k) = position of the k'th
 * (k >= 1) occurrence of symbol c.  d_sym: DEVICE u32[q]; d_k: DEVICE
 * u64[q]; d_out: DEVICE u64[q] receives the 0-based position, or UINT64_MAX
 * when k == 0, k exceeds the count of c, or c >= sigma.  Asynchronous on
 * `stream`.  WT_EINVAL on null pointers (q > 0) or when the select index
 * has not been built.
 */
int wt_select_index(wt_tree *t, void *stream);
int wt_select(const wt_tree *t, const uint32_t *d_sym, const uint64_t *d_k, uint64_t q, uint64_t *d_out,
              void *stream);
int wm_select_index(wm_matrix *m, void *stream);
int wm_select(const wm_matrix *m, const uint32_t *d_sym, const uint64_t *d_k, uint64_t q, uint64_t *d_out,
              void *stream);

/* ---- Huffman-shaped wavelet tree ----
 *
 * "each node is placed at a level proportional to the length of its Huffman
 * code" (:855-856).  Readings (R-17..R-20):
 *   - Huffman tree by the two-queue method over the occurring symbols,
 *     leaves ordered by (frequency, symbol), a leaf before an internal node
 *     of equal weight; code length = leaf depth (R-17).
 *   - canonical codes: first code of length L is (first(L-1) + count(L-1))
 *     << 1, symbols of one length numbered in symbol order (R-18); a 0 bit
 *     goes left.  code[c] is right-aligned; code_len[c] = 0 for a symbol
 *     that does not occur.
 *   - level l holds, for every element whose code is longer than l, its code
 *     bit l, in levelWT order (stable per node, nodes left to right); the
 *     elements that reach a leaf leave the sequence (R-19).  n_l =
 *     level_len[l]; sum_l n_l = sum_c freq(c) * code_len[c].
 *   - fewer than two distinct symbols: 0 levels; only_symbol is the symbol
 *     (R-20).  Codes longer than 32 bits: WT_EUNSUPPORTED.
 * Layout: the levels are concatenated; level l occupies
 *   bits       [level_word_ptr[l],  level_word_ptr[l+1])   ceil(n_l/512)*8 words
 *   rank_block [level_block_ptr[l], level_block_ptr[l+1])  ceil(n_l/512)
 *   rank_super [level_super_ptr[l], level_super_ptr[l+1])  ceil(n_l/65536)+1
 * with the per-level meaning of wt_tree (LSB-first bits, zero padding,
 * relative u16 block counts, absolute u64 super counts, last = level total).
 * Nodes: CSR level_node_ptr[levels+1] over node_key (the l-bit code prefix
 * of the internal node) and node_start (its first position in level l), in
 * ascending key order.  Every array pointer is a DEVICE pointer owned by the
 * library until hwt_free().
 */
typedef struct hwt_tree {
  uint64_t n;                 /* sequence length                              */
  uint64_t sigma;             /* alphabet size (<= 65536)                     */
  uint32_t levels;            /* h = longest code length                      */
  uint32_t elem_bytes;        /* bytes per input symbol                       */
  uint64_t *level_len;        /* u64[levels]: n_l                             */
  uint64_t *level_word_ptr;   /* u64[levels+1]                                */
  uint64_t *level_block_ptr;  /* u64[levels+1]                                */
  uint64_t *level_super_ptr;  /* u64[levels+1]                                */
  uint64_t *bits;             /* u64[level_word_ptr[levels]]                  */
  uint16_t *rank_block;       /* u16[level_block_ptr[levels]]                 */
  uint64_t *rank_super;       /* u64[level_super_ptr[levels]]                 */
  uint64_t *level_node_ptr;   /* u64[levels+1]                                */
  uint32_t *node_key;         /* u32[total_nodes]                             */
  uint32_t *node_start;       /* u32[total_nodes]                             */
  uint64_t total_nodes;       /* internal nodes of the Huffman tree           */
  uint32_t *code;             /* u32[sigma] canonical code (right-aligned)    */
  uint8_t *code_len;          /* u8[sigma], 0 = symbol absent                 */
  uint32_t only_symbol;       /* levels == 0 && n > 0: the single symbol      */
  uint32_t stages;            /* padded-code passes used by the build (diagnostic) */
  uint64_t total_bits;        /* sum of level_len                             */
  void *internal;             /* library bookkeeping; do not touch            */
} hwt_tree;

/* hwt_build -- build the Huffman-shaped wavelet tree of S.  Arguments as
 * wt_build with sigma <= 65536 (WT_EINVAL otherwise).  Work is enqueued on
 * `stream`; the call synchronises it three times (after the code lengths,
 * inside the balanced pass over the padded codes, after the node
 * compaction).  Errors: WT_EINVAL, WT_ESYMBOL, WT_ENOMEM, WT_ECUDA,
 * WT_EUNSUPPORTED (a code longer than 32 bits); on error *out = NULL and
 * nothing leaks. */
int hwt_build(const void *d_seq, uint64_t n, uint32_t elem_bytes, uint64_t sigma,
              void *stream, hwt_tree **out);
/* hwt_free -- release everything owned by t; NULL is a no-op.  Ordered like
 * wt_free (after the build stream and every stream a query of t used). */
int hwt_free(hwt_tree *t);
/* hwt_access / hwt_rank -- batched access(S, i) and inclusive rank_c(S, i)
 * by descent along the code; rank_c of an absent symbol
 * c < sigma is 0.  Buffers, sentinels and errors exactly as wt_access /
 * wt_rank. */
int hwt_access(const hwt_tree *t, const uint64_t *d_pos, uint64_t q, uint32_t *d_out, void *stream);
int hwt_rank(const hwt_tree *t, const uint32_t *d_sym, const uint64_t *d_pos, uint64_t q,
             uint64_t *d_out, void *stream);
/* hwt_select -- batched select_c(S, k): descent along c's
 * code to the deepest node, then bit selects climbing back up (binary
 * searches over each level's rank directory; no select index is needed).
 * Buffers, sentinels (UINT64_MAX for k == 0, k > count of c, c >= sigma or
 * c absent) and errors as wt_select. */
int hwt_select(const hwt_tree *t, const uint32_t *d_sym, const uint64_t *d_k, uint64_t q, uint64_t *d_out,
               void *stream);

/* ---- sharded build helpers (orchestrated by the Python
 * module paper_1407_8142_b200/dist.py over torch.distributed / NCCL) ----
 *
 * With S split into contiguous chunks, one per GPU, levels 0..tau-1 of the
 * tree are runs of each chunk placed at global offsets, and levels >= tau
 * are built by the owner of each top-tau digit range from S_tau restricted
 * to that range (S_tau = S stably sorted by its top tau bits, PAPER.md:
 * 468-475); see DESIGN.md §8.
 *
 * wt_digit_counts -- d_counts[d] (DEVICE u64[2^tau]) = number of i with
 *   ((S[i] >> shift) & (2^tau - 1)) == d, 1 <= tau <= 8.  Validates
 *   S[i] < sigma (WT_ESYMBOL).  Synchronises `stream` once.
 * wt_digits -- d_out[i] (DEVICE u8) = (S[i] >> shift) & (2^tau - 1).  Async.
 * wt_partition -- d_out (DEVICE, n symbols of elem_bytes, caller-owned,
 *   must not alias d_in) = d_in stably sorted by ((x >> shift) & (2^tau-1)).
 *   Asynchronous on `stream`.
 * wt_gather_bits -- DEVICE u64 d_dst[0, dst_words) = bits gathered from the
 *   LSB-first bit array d_src by nseg segments d_segs[3k..3k+2] = (dst_bit,
 *   src_bit, len) (DEVICE u64), sorted by dst_bit and disjoint; bits no
 *   segment covers are 0.  Asynchronous.
 * wt_create -- allocate a wt_tree for n symbols over sigma with total_nodes
 *   node entries; bits are zeroed, every other array is left for the caller
 *   to fill through its device pointers (level_node_ptr, node_key,
 *   node_start), then wt_finish computes the rank directory from the bits
 *   and synchronises.  Released by wt_free.  Errors as wt_build.
 */
int wt_digit_counts(const void *d_seq, uint64_t n, uint32_t elem_bytes, uint64_t sigma, uint32_t shift,
                    uint32_t tau, uint64_t *d_counts, void *stream);
int wt_digits(const void *d_seq, uint64_t n, uint32_t elem_bytes, uint32_t shift, uint32_t tau, uint8_t *d_out,
              void *stream);
int wt_partition(const void *d_in, uint64_t n, uint32_t elem_bytes, uint32_t shift, uint32_t tau, void *d_out,
                 void *stream);
int wt_gather_bits(const uint64_t *d_src, const uint64_t *d_segs, uint64_t nseg, uint64_t *d_dst,
                   uint64_t dst_words, void *stream);
int wt_create(uint64_t n, uint64_t sigma, uint32_t elem_bytes, uint64_t total_nodes, void *stream,
              wt_tree **out);
int wt_finish(wt_tree *t, void *stream);

/* ---- measurement hooks (used by bench.py; no effect on results) ---- */

#define WT_PROF_MAX 32
typedef struct wt_prof_entry {
  char name[40];          /* kernel name                                    */
  float ms;               /* summed device time of its launches (CUDA events
                             recorded on the launch stream)                 */
  uint32_t launches;      /* launches in the last profiled build            */
  uint32_t pad;
  uint64_t algo_bytes;    /* algorithmic bytes moved by those launches
                                             */
} wt_prof_entry;

typedef struct wt_profile {
  uint32_t count;               /* valid entries                            */
  uint32_t total_launches;      /* all kernel launches of the last build    */
  wt_prof_entry e[WT_PROF_MAX];
} wt_profile;

/* Enable (1) / disable (0) per-kernel event timing in subsequent builds;
 * enabling also resets the total of wt_profile_total. */
int wt_profile_enable(int on);
/* Copy the per-kernel record of the most recent build (profiled or not:
 * launches and total_launches are always filled, ms only when enabled). */
int wt_last_profile(wt_profile *out);
/* The per-kernel record summed over every build since profiling was last
 * enabled (bench.py reads it once after the timed steps). */
int wt_profile_total(wt_profile *out);
/* Version string of the library. */
const char *wt_version(void);

#ifdef __cplusplus
}
#endif
#endif /* WT_B200_H */
