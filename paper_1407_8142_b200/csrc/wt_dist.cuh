// wt_dist.cuh -- kernels of the sharded (multi-GPU) build, SURVEY §8(e) / f4.
//
// One process per GPU holds a contiguous chunk S_r of S.  The build needs,
// besides the single-GPU passes:
//   * per-chunk counts of the top-tau digit (validation included): the
//     exchange step's metadata (PAPER.md:266-273 split-then-merge, with the
//     merge replaced by placing runs at global offsets);
//   * a stable partition of a chunk by that digit (MSD radix step) before
//     and after the all-to-all, so that every owner receives S_tau restricted
//     to its digit range (S_l is S stably sorted by its top
//     l bits);
//   * a bit-range gather that places the runs of every rank at their global
//     positions (levels < tau: per-(rank, class) runs; levels >= tau: one run
//     per owner).
// The orchestration (collectives over torch.distributed / NCCL) is in
// paper_1407_8142_b200/dist.py.
#pragma once
#include "wt_common.cuh"

namespace wtb {

constexpr uint32_t PART_TILE = 4096;  // elements per CTA tile of the partition
constexpr uint32_t PART_THREADS = 256, PART_PER = PART_TILE / PART_THREADS;

// d[i] = (S[i] >> shift) & dmask as a byte (the chunk's top-tau digits).
template <typename T>
__global__ void k_digits(const T *__restrict__ keys, uint64_t n, uint32_t shift, uint32_t dmask,
                         uint8_t *__restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = (uint8_t)(((uint32_t)keys[i] >> shift) & dmask);
}

// Per-tile digit counts, stored digit-major: thT[d * ntiles + tile].
template <typename T>
__global__ void __launch_bounds__(PART_THREADS) k_part_hist(const T *__restrict__ keys, uint64_t n, uint64_t sigma,
                                                            uint32_t shift, uint32_t ndig, uint32_t ntiles,
                                                            uint32_t *__restrict__ thT, uint32_t *err) {
  __shared__ uint32_t h[4][256];
  const uint32_t dmask = ndig - 1u;
  bool bad = false;
  for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    for (uint32_t i = threadIdx.x; i < 4 * 256; i += blockDim.x) (&h[0][0])[i] = 0;
    __syncthreads();
    const uint64_t b = (uint64_t)t * PART_TILE;
    for (uint32_t i = threadIdx.x; i < PART_TILE; i += blockDim.x) {
      const uint64_t j = b + i;
      if (j < n) {
        const uint32_t v = (uint32_t)keys[j];
        if ((uint64_t)v >= sigma) bad = true;
        atomicAdd(&h[threadIdx.x & 3][(v >> shift) & dmask], 1u);
      }
    }
    __syncthreads();
    for (uint32_t d = threadIdx.x; d < ndig; d += blockDim.x)
      thT[(uint64_t)d * ntiles + t] = h[0][d] + h[1][d] + h[2][d] + h[3][d];
    __syncthreads();
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0 && err) atomicOr(err, 1u);
}

// One CTA per digit: exclusive scan of its tile counts in place; tot[d] = total.
static __global__ void __launch_bounds__(1024) k_part_scan(uint32_t *__restrict__ thT, uint32_t ntiles,
                                                   uint64_t *__restrict__ tot) {
  __shared__ uint32_t shm[33];
  uint32_t *row = thT + (uint64_t)blockIdx.x * ntiles;
  uint32_t carry = 0;
  for (uint32_t t0 = 0; t0 < ntiles; t0 += blockDim.x) {
    const uint32_t t = t0 + threadIdx.x;
    const uint32_t v = t < ntiles ? row[t] : 0u;
    uint32_t total;
    const uint32_t ex = block_exscan(v, shm, &total);
    if (t < ntiles) row[t] = carry + ex;
    carry += total;
  }
  if (threadIdx.x == 0) tot[blockIdx.x] = carry;
}

// Stable scatter of one tile: element j of digit d goes to
//   base(d) + (same-digit elements of earlier tiles) + (earlier in this tile).
// Each warp owns PART_PER chunks of 32 consecutive elements; ranks inside a
// chunk come from tau ballots (lanes whose digit bits all agree).
template <typename T>
__global__ void __launch_bounds__(PART_THREADS) k_part_scatter(const T *__restrict__ keys, uint64_t n, uint32_t shift,
                                                               uint32_t tau, uint32_t ntiles,
                                                               const uint32_t *__restrict__ thT,
                                                               const uint64_t *__restrict__ tot, T *__restrict__ out) {
  constexpr uint32_t NW = PART_THREADS / 32;
  __shared__ uint32_t cw[NW][256];
  __shared__ unsigned long long base[256];
  const uint32_t ndig = 1u << tau, dmask = ndig - 1u;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t t = blockIdx.x;
  for (uint32_t i = threadIdx.x; i < NW * 256; i += blockDim.x) (&cw[0][0])[i] = 0;
  if (threadIdx.x == 0) {
    unsigned long long acc = 0;
    for (uint32_t d = 0; d < ndig; d++) { base[d] = acc; acc += tot[d]; }
  }
  __syncthreads();
  const uint64_t wb = (uint64_t)t * PART_TILE + (uint64_t)warp * PART_PER * 32;
  T v[PART_PER];
  uint32_t rk[PART_PER];
#pragma unroll
  for (uint32_t c = 0; c < PART_PER; c++) {
    const uint64_t j = wb + c * 32 + lane;
    const bool ok = j < n;
    v[c] = ok ? keys[j] : T(0);
    const uint32_t d = ((uint32_t)v[c] >> shift) & dmask;
    uint32_t peers = __ballot_sync(FULL, ok);
    for (uint32_t b = 0; b < tau; b++) {
      const uint32_t m = __ballot_sync(FULL, (d >> b) & 1u);
      peers &= ((d >> b) & 1u) ? m : ~m;
    }
    rk[c] = cw[warp][d] + __popc(peers & lanemask_lt());
    __syncwarp();
    if (ok && (peers & lanemask_lt()) == 0) cw[warp][d] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // exclusive scan of the warp counts per digit
  for (uint32_t d = threadIdx.x; d < ndig; d += blockDim.x) {
    uint32_t acc = 0;
    for (uint32_t w = 0; w < NW; w++) { const uint32_t x = cw[w][d]; cw[w][d] = acc; acc += x; }
  }
  __syncthreads();
#pragma unroll
  for (uint32_t c = 0; c < PART_PER; c++) {
    const uint64_t j = wb + c * 32 + lane;
    if (j < n) {
      const uint32_t d = ((uint32_t)v[c] >> shift) & dmask;
      out[base[d] + thT[(uint64_t)d * ntiles + t] + cw[warp][d] + rk[c]] = v[c];
    }
  }
}

// ---------------------------------------------------------------------------
// Bit-range gather: dst bits [0, 64 * dst_words) from segments (dst_bit,
// src_bit, len) sorted by dst_bit and disjoint; uncovered bits are 0.  A CTA
// owns GB_WORDS * GB_WPT output words: warp 0 finds the covering segments,
// stages them in shared memory when they fit.
// ---------------------------------------------------------------------------
constexpr uint32_t GB_WORDS = 256, GB_WPT = 8, GB_SEGS = 1024;

static __global__ void __launch_bounds__(GB_WORDS) k_gather_bits(const uint64_t *__restrict__ src,
                                                          const uint64_t *__restrict__ segs, uint64_t nseg,
                                                          uint64_t *__restrict__ dst, uint64_t dst_words) {
  __shared__ unsigned long long s_d[GB_SEGS], s_s[GB_SEGS], s_l[GB_SEGS];
  __shared__ uint64_t s_k0, s_k1;
  const uint64_t w0 = (uint64_t)blockIdx.x * GB_WORDS * GB_WPT;
  if (w0 >= dst_words) return;
  const uint64_t bit0 = w0 * 64, bit1 = min(w0 + GB_WORDS * GB_WPT, dst_words) * 64;
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    // k0 = first segment ending after bit0; k1 = first segment starting at or after bit1
    uint64_t lo = 0, hi = nseg;
    while (hi - lo > 32) {
      const uint64_t step = (hi - lo + 31) / 32, p = lo + lane * step;
      const bool le = p < hi && segs[3 * p] + segs[3 * p + 2] <= bit0;
      const uint32_t c = __popc(__ballot_sync(FULL, le));
      if (c == 0) { hi = lo; break; }
      const uint64_t nlo = lo + (c - 1) * step + 1;
      hi = min(hi, lo + c * step);
      lo = nlo;
    }
    {
      const bool le = lo + lane < hi && segs[3 * (lo + lane)] + segs[3 * (lo + lane) + 2] <= bit0;
      lo += __popc(__ballot_sync(FULL, le));
    }
    const uint64_t k0 = lo;
    lo = k0;
    hi = nseg;
    while (hi - lo > 32) {
      const uint64_t step = (hi - lo + 31) / 32, p = lo + lane * step;
      const bool le = p < hi && segs[3 * p] < bit1;
      const uint32_t c = __popc(__ballot_sync(FULL, le));
      if (c == 0) { hi = lo; break; }
      const uint64_t nlo = lo + (c - 1) * step + 1;
      hi = min(hi, lo + c * step);
      lo = nlo;
    }
    {
      const bool le = lo + lane < hi && segs[3 * (lo + lane)] < bit1;
      lo += __popc(__ballot_sync(FULL, le));
    }
    if (lane == 0) { s_k0 = k0; s_k1 = lo; }
  }
  __syncthreads();
  const uint64_t k0 = s_k0, cnt = s_k1 - s_k0;
  const bool staged = cnt <= GB_SEGS;
  if (staged) {
    for (uint64_t i = threadIdx.x; i < cnt; i += blockDim.x) {
      s_d[i] = segs[3 * (k0 + i)];
      s_s[i] = segs[3 * (k0 + i) + 1];
      s_l[i] = segs[3 * (k0 + i) + 2];
    }
  }
  __syncthreads();
  auto SD = [&](uint64_t k) -> uint64_t { return staged ? s_d[k] : segs[3 * (k0 + k)]; };
  auto SS = [&](uint64_t k) -> uint64_t { return staged ? s_s[k] : segs[3 * (k0 + k) + 1]; };
  auto SL = [&](uint64_t k) -> uint64_t { return staged ? s_l[k] : segs[3 * (k0 + k) + 2]; };
  for (uint32_t r = 0; r < GB_WPT; r++) {
    const uint64_t w = w0 + r * GB_WORDS + threadIdx.x;
    if (w >= dst_words) break;
    const uint64_t b0 = w * 64, b1 = b0 + 64;
    // first segment ending after b0
    uint64_t a = 0, z = cnt;
    while (a < z) {
      const uint64_t mid = (a + z) >> 1;
      if (SD(mid) + SL(mid) <= b0) a = mid + 1; else z = mid;
    }
    uint64_t res = 0;
    for (uint64_t k = a; k < cnt; k++) {
      const uint64_t d0 = SD(k);
      if (d0 >= b1) break;
      const uint64_t s = d0 > b0 ? d0 : b0, e = min(d0 + SL(k), b1);
      if (e <= s) continue;
      const uint64_t take = e - s, sb = SS(k) + (s - d0);
      const uint64_t wi = sb >> 6, o = sb & 63;
      uint64_t v = src[wi] >> o;
      if (o && o + take > 64) v |= src[wi + 1] << (64 - o);
      if (take < 64) v &= (1ull << take) - 1ull;
      res |= v << (s - b0);
    }
    dst[w] = res;
  }
}

}  // namespace wtb
