// wt_rank.cuh -- A7 rank-directory finalize and A8 batched queries.
//
// Directory (reading R-9): per level, u16
// rank_block[b] = ones in [floor(b/128)*65536, b*512) and u64 rank_super[s] =
// ones in [0, min(s*65536, n)).  k_rank_local popcounts the finished bitmaps
// block by block; k_rank_super scans the superblock totals.
#pragma once
#include "wt_common.cuh"

namespace wtb {

// ---------------------------------------------------------------------------
// A7 finalize: rank_block (u16, relative to the superblock) and rank_super.
// k_rank_local: one warp per (level, superblock); k_rank_super: one CTA per level.
// ---------------------------------------------------------------------------
static __global__ void k_rank_local(const uint64_t *__restrict__ bits, uint64_t wpl, uint64_t bpl, uint64_t nsup_data,
                             uint32_t lbeg, uint32_t nl, uint16_t *__restrict__ rank_block,
                             uint64_t *__restrict__ suptot, const uint32_t *err) {
  // One warp per (level, superblock) of levels [lbeg, lbeg+nl): popcount of its
  // <= 128 blocks of 8 words (a streaming read of the finished bitmaps), then
  // the in-superblock scan.
  if (*err) return;
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= (uint64_t)nl * nsup_data) return;
  const uint32_t l = lbeg + (uint32_t)(gw / nsup_data);
  const uint64_t s = gw % nsup_data;
  const uint64_t b0 = s * 128;
  const uint64_t *B = bits + (uint64_t)l * wpl;
  uint32_t v[4], sum = 0;
#pragma unroll
  for (int i = 0; i < 4; i++) {
    const uint64_t b = b0 + lane * 4 + i;
    uint32_t c = 0;
    if (b < bpl) {
      const ulonglong2 *w = reinterpret_cast<const ulonglong2 *>(B + b * 8);
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const ulonglong2 x = __ldcs(w + k);
        c += __popcll(x.x) + __popcll(x.y);
      }
    }
    v[i] = c;
    sum += c;
  }
  const uint32_t incl = warp_incl_scan(sum, lane);
  uint32_t run = incl - sum;
#pragma unroll
  for (int i = 0; i < 4; i++) {
    const uint64_t b = b0 + lane * 4 + i;
    if (b < bpl) rank_block[(uint64_t)l * bpl + b] = (uint16_t)run;
    run += v[i];
  }
  if (lane == 31) suptot[(uint64_t)l * nsup_data + s] = incl;
}

// A7 finalize from the block popcounts the group pass accumulated (fused A7):
// blkcnt[l*bpl + b] = ones of block b of level l.  One warp per (level, superblock).
static __global__ void k_rank_counts(const uint32_t *__restrict__ blkcnt, uint64_t bpl, uint64_t nsup_data,
                                     uint32_t lbeg, uint32_t nl, uint16_t *__restrict__ rank_block,
                                     uint64_t *__restrict__ suptot, const uint32_t *err) {
  if (*err) return;
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= (uint64_t)nl * nsup_data) return;
  const uint32_t l = lbeg + (uint32_t)(gw / nsup_data);
  const uint64_t s = gw % nsup_data;
  const uint64_t b0 = s * 128 + lane * 4;
  uint32_t v[4] = {0, 0, 0, 0}, sum = 0;
  if (b0 + 4 <= bpl && (((uint64_t)l * bpl + b0) & 3) == 0) {
    const uint4 q = *reinterpret_cast<const uint4 *>(blkcnt + (uint64_t)l * bpl + b0);
    v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
  } else {
#pragma unroll
    for (int i = 0; i < 4; i++) v[i] = (b0 + i < bpl) ? blkcnt[(uint64_t)l * bpl + b0 + i] : 0u;
  }
#pragma unroll
  for (int i = 0; i < 4; i++) sum += v[i];
  const uint32_t incl = warp_incl_scan(sum, lane);
  uint32_t run = incl - sum;
#pragma unroll
  for (int i = 0; i < 4; i++) {
    if (b0 + i < bpl) rank_block[(uint64_t)l * bpl + b0 + i] = (uint16_t)run;
    run += v[i];
  }
  if (lane == 31) suptot[(uint64_t)l * nsup_data + s] = incl;
}

static __global__ void __launch_bounds__(1024) k_rank_super(const uint64_t *__restrict__ suptot, uint64_t nsup_data,
                                                    uint64_t spl, uint64_t *__restrict__ rank_super,
                                                    const uint32_t *err) {
  __shared__ unsigned long long warp_tot[33];
  if (*err) return;
  const uint32_t l = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long carry = 0;
  for (uint64_t base = 0; base < spl; base += blockDim.x) {
    const uint64_t s = base + threadIdx.x;
    unsigned long long v = (s < nsup_data) ? suptot[(uint64_t)l * nsup_data + s] : 0ull;
    unsigned long long incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long t = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      unsigned long long w = warp_tot[lane];
      unsigned long long wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        unsigned long long t = __shfl_up_sync(FULL, wi, o);
        if (lane >= o) wi += t;
      }
      warp_tot[lane] = wi - w;
      if (lane == 31) warp_tot[32] = wi;
    }
    __syncthreads();
    if (s < spl) rank_super[(uint64_t)l * spl + s] = carry + warp_tot[warp] + incl - v;
    carry += warp_tot[32];
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// A8 batched queries (verification path): top-down descent with rank1 from
// the directory.
// ---------------------------------------------------------------------------
struct TreeView {
  uint64_t n, wpl, bpl, spl;
  uint32_t L;
  const uint64_t *bits;
  const uint16_t *rank_block;
  const uint64_t *rank_super;
};

__device__ __forceinline__ uint64_t d_rank1(const TreeView &t, uint32_t l, uint64_t i) {
  if (i >= t.n) return t.rank_super[(uint64_t)l * t.spl + t.spl - 1];
  const uint64_t *B = t.bits + (uint64_t)l * t.wpl;
  uint64_t r = t.rank_super[(uint64_t)l * t.spl + (i >> 16)] + t.rank_block[(uint64_t)l * t.bpl + (i >> 9)];
  for (uint64_t w = (i >> 9) * 8; w < (i >> 6); w++) r += __popcll(B[w]);
  if (i & 63) r += __popcll(B[i >> 6] & ((1ull << (i & 63)) - 1ull));
  return r;
}

static __global__ void k_access(TreeView t, const uint64_t *__restrict__ pos, uint64_t q, uint32_t *__restrict__ out) {
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= q) return;
  uint64_t i = pos[k];
  if (i >= t.n) { out[k] = 0xffffffffu; return; }
  uint64_t s = 0, e = t.n;
  uint32_t sym = 0;
  for (uint32_t l = 0; l < t.L; l++) {
    const uint64_t r1s = d_rank1(t, l, s), r1e = d_rank1(t, l, e), r1i = d_rank1(t, l, i);
    const uint64_t z = (e - s) - (r1e - r1s);
    const uint32_t bit = (uint32_t)((t.bits[(uint64_t)l * t.wpl + (i >> 6)] >> (i & 63)) & 1ull);
    sym = (sym << 1) | bit;
    if (bit) { i = s + z + (r1i - r1s); s += z; }
    else { i = s + (i - s) - (r1i - r1s); e = s + z; }
  }
  out[k] = sym;
}

static __global__ void k_rank_query(TreeView t, uint64_t sigma, const uint32_t *__restrict__ sym,
                             const uint64_t *__restrict__ pos, uint64_t q, uint64_t *__restrict__ out) {
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= q) return;
  const uint64_t i = pos[k];
  const uint32_t c = sym[k];
  if (i >= t.n || (uint64_t)c >= sigma) { out[k] = ~0ull; return; }
  uint64_t s = 0, e = t.n, r = i + 1;
  for (uint32_t l = 0; l < t.L && r; l++) {
    const uint64_t r1s = d_rank1(t, l, s), r1e = d_rank1(t, l, e), r1p = d_rank1(t, l, s + r);
    const uint64_t z = (e - s) - (r1e - r1s);
    if ((c >> (t.L - 1 - l)) & 1u) { r = r1p - r1s; s += z; }
    else { r = r - (r1p - r1s); e = s + z; }
  }
  out[k] = r;
}

}  // namespace wtb
