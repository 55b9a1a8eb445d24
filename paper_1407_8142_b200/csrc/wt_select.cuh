// wt_select.cuh -- select directory and batched select_c (PAPER.md:207-208,
// §6 :827-845).
//
// Directory (Clark's first level, :827-829, sampled every SEL_SAMPLE = 4096
// occurrences, reading R-14): for every 512-bit block of a level the
// rank directory gives the 1s (and 0s) before it; a block holds fewer than
// 4096 bits, so it contains at most one sampled 1 and one sampled 0 -- one
// thread per block finds them ("prefix sum and filter", :839-841).
//
// select_b(l, k): from the k'th b-bit's sample, binary search over the
// superblocks and blocks of the rank directory, then popcounts over <= 8 words
// and a select inside one word.  select_c descends top-down to find c's node
// (tree) or class start (matrix) per level, then climbs back up with select_b.
#pragma once
#include "wt_common.cuh"
#include "wt_rank.cuh"

namespace wtb {

constexpr uint32_t SEL_SAMPLE = 4096;

static __global__ void k_fill_u32(uint32_t *__restrict__ a, uint64_t cnt, uint32_t v) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (uint64_t)gridDim.x * blockDim.x)
    a[i] = v;
}

// b-bits of level l before position p (p a multiple of 512, p <= n rounded)
__device__ __forceinline__ uint64_t d_cnt_block(const TreeView &t, uint32_t l, uint64_t blk, uint32_t b) {
  const uint64_t ones = t.rank_super[(uint64_t)l * t.spl + (blk >> 7)] + t.rank_block[(uint64_t)l * t.bpl + blk];
  return b ? ones : blk * 512 - ones;
}

// position of the j'th (0-based) set bit of w (j < popc(w))
__device__ __forceinline__ uint32_t select_in_word(uint64_t w, uint32_t j) {
  const uint32_t lo = (uint32_t)w, plo = __popc(lo);
  if (j < plo) return __fns(lo, 0, (int)j + 1);
  return 32 + __fns((uint32_t)(w >> 32), 0, (int)(j - plo) + 1);
}

static __global__ void k_select_dir(TreeView t, uint32_t *__restrict__ sel0, uint32_t *__restrict__ sel1, uint64_t sps) {
  const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (uint64_t)t.L * t.bpl) return;
  const uint32_t l = (uint32_t)(gid / t.bpl);
  const uint64_t blk = gid % t.bpl;
  const uint64_t *B = t.bits + (uint64_t)l * t.wpl + blk * 8;
  const uint64_t o_before = d_cnt_block(t, l, blk, 1);
  const uint64_t nb = (t.n - blk * 512) < 512 ? (t.n - blk * 512) : 512;  // bits of this block inside [0, n)
  uint64_t w[8];
  uint32_t ones = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) {
    w[i] = B[i];
    ones += __popcll(w[i]);
  }
  const uint64_t z_before = blk * 512 - o_before;
  const uint32_t zeros = (uint32_t)nb - ones;
#pragma unroll
  for (int b = 0; b < 2; b++) {
    const uint64_t before = b ? o_before : z_before;
    const uint32_t cnt = b ? ones : zeros;
    const uint64_t m = (before + SEL_SAMPLE - 1) / SEL_SAMPLE;  // first sample index >= before
    if (cnt == 0 || m * SEL_SAMPLE >= before + cnt) continue;
    uint32_t need = (uint32_t)(m * SEL_SAMPLE - before);  // b-bits of the block before the sampled one
    for (int i = 0; i < 8; i++) {
      uint64_t v = b ? w[i] : ~w[i];
      if (blk * 512 + i * 64 + 64 > t.n) {  // mask padding past n
        const uint64_t valid = t.n > blk * 512 + i * 64 ? t.n - (blk * 512 + i * 64) : 0;
        v &= valid >= 64 ? ~0ull : ((1ull << valid) - 1ull);
      }
      const uint32_t pc = __popcll(v);
      if (need < pc) {
        (b ? sel1 : sel0)[(uint64_t)l * sps + m] = (uint32_t)(blk * 512 + i * 64 + select_in_word(v, need));
        break;
      }
      need -= pc;
    }
  }
}

// position of the k'th (1-based) b-bit of level l, or n
static __device__ uint64_t d_select_b(const TreeView &t, const uint32_t *sel, uint64_t sps, uint32_t l, uint32_t b,
                               uint64_t k) {
  if (k == 0) return t.n;
  const uint64_t j = (k - 1) / SEL_SAMPLE;
  const uint64_t p0 = sel[(uint64_t)l * sps + j];
  if (p0 >= t.n) return t.n;
  const uint64_t p1 = sel[(uint64_t)l * sps + j + 1];
  const uint64_t target = k - 1;  // b-bits before the answer
  // block: largest blk in [p0/512, p1/512] with cnt_b(blk) <= target (binary search over blocks)
  uint64_t lo = p0 >> 9, hi = ((p1 < t.n ? p1 : t.n - 1) >> 9) + 1;
  while (hi - lo > 1) {
    const uint64_t mid = (lo + hi) >> 1;
    if (d_cnt_block(t, l, mid, b) <= target) lo = mid;
    else hi = mid;
  }
  uint64_t need = target - d_cnt_block(t, l, lo, b);
  const uint64_t *B = t.bits + (uint64_t)l * t.wpl + lo * 8;
  for (int i = 0; i < 8; i++) {
    uint64_t v = b ? B[i] : ~B[i];
    const uint64_t base = lo * 512 + i * 64;
    if (base + 64 > t.n) {
      const uint64_t valid = t.n > base ? t.n - base : 0;
      v &= valid >= 64 ? ~0ull : ((1ull << valid) - 1ull);
    }
    const uint32_t pc = __popcll(v);
    if (need < pc) return base + select_in_word(v, (uint32_t)need);
    need -= pc;
  }
  return t.n;
}

__device__ __forceinline__ uint64_t d_rank_b(const TreeView &t, uint32_t l, uint64_t i, uint32_t b) {
  const uint64_t r1 = d_rank1(t, l, i);
  return b ? r1 : (i < t.n ? i : t.n) - r1;
}

// tree: top-down node ranges of c's prefix, then bottom-up selects
static __global__ void k_wt_select(TreeView t, const uint32_t *__restrict__ sel0, const uint32_t *__restrict__ sel1,
                            uint64_t sps, uint64_t sigma, const uint32_t *__restrict__ sym,
                            const uint64_t *__restrict__ kk, uint64_t q, uint64_t *__restrict__ out) {
  const uint64_t id = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= q) return;
  const uint32_t c = sym[id];
  const uint64_t k = kk[id];
  if ((uint64_t)c >= sigma || k == 0 || k > t.n) { out[id] = ~0ull; return; }
  uint64_t s[33];
  uint64_t sl = 0, el = t.n;
  for (uint32_t l = 0; l < t.L; l++) {
    s[l] = sl;
    const uint64_t r1s = d_rank1(t, l, sl), r1e = d_rank1(t, l, el);
    const uint64_t z = (el - sl) - (r1e - r1s);
    if ((c >> (t.L - 1 - l)) & 1u) sl += z;
    else el = sl + z;
  }
  if (k > el - sl) { out[id] = ~0ull; return; }
  uint64_t p = k - 1;
  for (uint32_t l = t.L; l-- > 0;) {
    const uint32_t b = (c >> (t.L - 1 - l)) & 1u;
    const uint64_t before = d_rank_b(t, l, s[l], b);
    p = d_select_b(t, b ? sel1 : sel0, sps, l, b, before + p + 1) - s[l];
  }
  out[id] = p;
}

// matrix: class starts top-down, then bottom-up selects
static __global__ void k_wm_select(TreeView t, const uint64_t *__restrict__ zeros, const uint32_t *__restrict__ sel0,
                            const uint32_t *__restrict__ sel1, uint64_t sps, uint64_t sigma,
                            const uint32_t *__restrict__ sym, const uint64_t *__restrict__ kk, uint64_t q,
                            uint64_t *__restrict__ out) {
  const uint64_t id = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= q) return;
  const uint32_t c = sym[id];
  const uint64_t k = kk[id];
  if ((uint64_t)c >= sigma || k == 0 || k > t.n) { out[id] = ~0ull; return; }
  uint64_t s[33];
  uint64_t sl = 0, el = t.n;
  for (uint32_t l = 0; l < t.L; l++) {
    s[l] = sl;
    const uint64_t r1s = d_rank1(t, l, sl), r1e = d_rank1(t, l, el);
    if ((c >> (t.L - 1 - l)) & 1u) { sl = zeros[l] + r1s; el = zeros[l] + r1e; }
    else { sl -= r1s; el -= r1e; }
  }
  s[t.L] = sl;
  if (k > el - sl) { out[id] = ~0ull; return; }
  uint64_t p = sl + k - 1;
  for (uint32_t l = t.L; l-- > 0;) {
    const uint32_t b = (c >> (t.L - 1 - l)) & 1u;
    const uint64_t before = d_rank_b(t, l, s[l], b);
    p = d_select_b(t, b ? sel1 : sel0, sps, l, b, before + (p - s[l + 1]) + 1);
  }
  out[id] = p;
}

}  // namespace wtb
