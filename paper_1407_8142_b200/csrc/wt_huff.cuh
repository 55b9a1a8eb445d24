// wt_huff.cuh -- Huffman-shaped wavelet tree.
//
// The paper builds the Huffman tree and codes (:858-860), maps every symbol
// to its leaf and then "follows the logic of levelWT" (:870-873).  On the
// GPU the same result is reached in four steps:
//
//   H1 k_sym_hist      symbol histogram + validation (one read of S)
//   H2 k_huff_codes    one CTA: sort the occurring symbols by (freq, sym),
//                      two-queue Huffman code lengths in parallel rounds
//                      (reading R-17), canonical codes (R-18) and the
//                      per-level element counts n_l
//   H3 k_huff_map      S -> padded code (code << (h - len)), an h-bit key
//   H4 the balanced levelWT pass (k_group) over the padded keys, then
//      k_hwt_segments / k_hwt_bits: level l of the Huffman-shaped tree is
//      level l of the padded tree with the nodes that are already Huffman
//      leaves (code length <= l) cut out (R-19).  A padded key shares its
//      top-l bits with no key of a longer code (prefix-free codes), so those
//      nodes hold exactly the elements that left the sequence, and the
//      surviving nodes keep levelWT's stable order.
#pragma once
#include "wt_common.cuh"

namespace wtb {

constexpr uint32_t HUFF_MAXLEN = 32;  // longest supported code (R-20)

// Canonical-code tables shared by the segment pass and the queries.
struct HuffCanon {
  uint32_t first[HUFF_MAXLEN + 2];   // first canonical code of each length
  uint32_t count[HUFF_MAXLEN + 2];   // symbols of each length
  uint32_t offset[HUFF_MAXLEN + 2];  // index of the first such symbol in sym_sorted
};

// ---------------------------------------------------------------------------
// H1: histogram of S over [0, sigma) (sigma <= 65536) with validation, in
// shared memory per CTA, flushed once per CTA with global atomics.
// ---------------------------------------------------------------------------
// Visit S warp-uniformly: 16-byte vectors (E symbols per lane), then the
// scalar tail; f(v, valid) is called by all 32 lanes together.
template <typename InT, typename F>
__device__ __forceinline__ void visit_warp(const InT *__restrict__ S, uint64_t n, uint64_t gwarp, uint64_t nwarps,
                                           int lane, F f) {
  constexpr uint32_t E = 16 / sizeof(InT);
  const uint64_t nv = ((uintptr_t)S % 16 == 0) ? n / E : 0;
  const uint4 *SV = reinterpret_cast<const uint4 *>(S);
  for (uint64_t base = gwarp * 32; base < nv; base += nwarps * 32) {
    const uint64_t vi = base + lane;
    const bool ok = vi < nv;
    const uint4 q = ok ? __ldcs(SV + vi) : make_uint4(0, 0, 0, 0);
    const InT *e = reinterpret_cast<const InT *>(&q);
#pragma unroll
    for (uint32_t k = 0; k < E; k++) f((uint32_t)e[k], ok);
  }
  for (uint64_t base = nv * E + gwarp * 32; base < n; base += nwarps * 32) {
    const uint64_t i = base + lane;
    f(i < n ? (uint32_t)S[i] : 0u, i < n);
  }
}

// add one warp's 32 symbols into bins: lanes holding equal values combine
// first (match.any), taken only when some lane repeats its neighbour's value
// (a skewed input), so a hot symbol does not serialise on one counter
template <typename AddF>
__device__ __forceinline__ void warp_hist_add(uint32_t v, bool ok, int lane, AddF add) {
  const bool rep = v == __shfl_sync(FULL, v, (lane + 1) & 31);
  if (__any_sync(FULL, rep && ok)) {
    const uint32_t peers = __match_any_sync(FULL, ok ? v : 0xffffffffu);
    if (ok && lane == __ffs(peers) - 1) add(v, (uint32_t)__popc(peers));
  } else if (ok) {
    add(v, 1u);
  }
}

// sigma <= 256: one sub-histogram per warp (16 x 256 bins)
template <typename InT>
__global__ void __launch_bounds__(512) k_sym_hist_small(const InT *__restrict__ S, uint64_t n, uint32_t sigma,
                                                        uint32_t *__restrict__ hist, uint32_t *err) {
  __shared__ uint32_t h[16][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (uint32_t b = threadIdx.x; b < 16 * 256; b += blockDim.x) (&h[0][0])[b] = 0;
  __syncthreads();
  bool bad = false;
  uint32_t *hw = h[warp];
  visit_warp(S, n, (uint64_t)blockIdx.x * 16 + warp, (uint64_t)gridDim.x * 16, lane, [&](uint32_t v, bool ok) {
    if (ok) {
      if (v < sigma) atomicAdd(&hw[v], 1u);
      else bad = true;
    }
  });
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(err, 1u);
  for (uint32_t b = threadIdx.x; b < sigma; b += blockDim.x) {
    uint32_t t = 0;
#pragma unroll
    for (int w = 0; w < 16; w++) t += h[w][b];
    if (t) atomicAdd(&hist[b], t);
  }
}

// 256 < sigma <= 65536: bins in parts of HIST_PART (128 KB of shared memory);
// CTA b counts part b % nparts over its share of S (every element is read
// once per part)
constexpr uint32_t HIST_PART = 32768;
template <typename InT>
__global__ void __launch_bounds__(1024) k_sym_hist(const InT *__restrict__ S, uint64_t n, uint32_t sigma,
                                                   uint32_t nparts, uint32_t *__restrict__ hist, uint32_t *err) {
  extern __shared__ uint32_t hs[];
  const uint32_t part = blockIdx.x % nparts, idx = blockIdx.x / nparts, nblk = gridDim.x / nparts;
  const uint32_t lo = part * HIST_PART, cnt = min(HIST_PART, sigma - lo);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
  for (uint32_t b = threadIdx.x; b < cnt; b += blockDim.x) hs[b] = 0;
  __syncthreads();
  bool bad = false;
  visit_warp(S, n, (uint64_t)idx * wpb + warp, (uint64_t)nblk * wpb, lane, [&](uint32_t v, bool ok) {
    if (ok && v >= sigma) bad = true;
    const uint32_t r = v - lo;
    warp_hist_add(r, ok && r < cnt, lane, [&](uint32_t x, uint32_t c) { atomicAdd(&hs[x], c); });
  });
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(err, 1u);
  for (uint32_t b = threadIdx.x; b < cnt; b += blockDim.x)
    if (hs[b]) atomicAdd(&hist[lo + b], hs[b]);
}

// ---------------------------------------------------------------------------
// H2: code lengths, canonical codes and level sizes (one CTA of 1024 threads).
//   keys     scratch u64[P], P = next power of two >= max(sigma, 2)
//   scr      scratch u32[6 * sigma]
//   info     u64[4 + HUFF_MAXLEN]: [0] h, [1] m (occurring symbols), [2] the
//            only symbol when m == 1, [3] 1 when a code is longer than 32,
//            [4 + l] n_l = elements whose code is longer than l.
//
// Code lengths (R-17) by the two-queue method, run in rounds: with s the sum
// of the two lightest items, every item of weight <= s (in queue order,
// leaves before internal nodes of equal weight) would be paired off in that
// order by the sequential method before any new node (weight >= s) is
// consumed, so a round pairs all of them at once (an odd last item waits).
// Depths follow from the parent links, round by round in reverse.
// ---------------------------------------------------------------------------
constexpr uint32_t SORT_CH = 2048;  // bitonic keys per shared-memory chunk

// first index in [lo, hi) whose weight exceeds s (weights nondecreasing); one warp
template <typename F>
__device__ __forceinline__ uint32_t warp_upper(F w, uint32_t lo, uint32_t hi, uint64_t s, int lane) {
  while (hi - lo > 32) {
    const uint32_t step = (hi - lo + 31) / 32;
    const uint32_t p = lo + lane * step;
    const bool le = p < hi && w(p) <= s;
    const uint32_t c = __popc(__ballot_sync(FULL, le));
    if (c == 0) return lo;
    const uint32_t nlo = lo + (c - 1) * step + 1;
    hi = min(hi, lo + c * step);
    lo = nlo;
  }
  const bool le = lo + lane < hi && w(lo + lane) <= s;
  return lo + __popc(__ballot_sync(FULL, le));
}

__device__ __forceinline__ void bitonic_chunk(uint64_t *sk, uint32_t base, uint32_t cnt, uint32_t k, uint32_t jmax) {
  for (uint32_t j = jmax; j > 0; j >>= 1) {
    for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) {
      const uint32_t x = i ^ j;
      if (x > i) {
        const uint64_t a = sk[i], b = sk[x];
        const bool up = ((base + i) & k) == 0;
        if ((a > b) == up) { sk[i] = b; sk[x] = a; }
      }
    }
    __syncthreads();
  }
}

// compact the occurring symbols as keys (freq << 32 | sym) in symbol order,
// padded with UINT64_MAX to P; info[1] = m (one CTA)
static __global__ void __launch_bounds__(1024) k_huff_compact(const uint32_t *__restrict__ hist, uint32_t sigma,
                                                       uint64_t *__restrict__ keys, uint32_t P,
                                                       uint64_t *__restrict__ info) {
  __shared__ uint32_t shm[33];
  uint32_t base = 0;
  for (uint32_t c0 = 0; c0 < P; c0 += blockDim.x) {
    const uint32_t c = c0 + threadIdx.x;
    const uint32_t f = c < sigma ? hist[c] : 0u;
    uint32_t total;
    const uint32_t ex = block_exscan(f ? 1u : 0u, shm, &total);
    if (f) keys[base + ex] = ((uint64_t)f << 32) | c;
    base += total;
  }
  for (uint32_t i = base + threadIdx.x; i < P; i += blockDim.x) keys[i] = ~0ull;
  if (threadIdx.x == 0) info[1] = base;
}

// bitonic sort of keys[0, P), P a power of two: chunks of SORT_CH keys in
// shared memory (one CTA each) for the strides < SORT_CH, one
// compare-exchange per thread for the larger strides.
// k == 0: sort each chunk completely (k = 2 .. CH); else strides CH/2 .. 1 of stage k.
static __global__ void __launch_bounds__(1024) k_bitonic_chunk(uint64_t *__restrict__ keys, uint32_t P, uint32_t k) {
  __shared__ uint64_t sk[SORT_CH];
  const uint32_t CH = P < SORT_CH ? P : SORT_CH;
  const uint32_t c0 = blockIdx.x * CH;
  for (uint32_t i = threadIdx.x; i < CH; i += blockDim.x) sk[i] = keys[c0 + i];
  __syncthreads();
  if (k == 0) {
    for (uint32_t kk = 2; kk <= CH; kk <<= 1) bitonic_chunk(sk, c0, CH, kk, kk >> 1);
  } else {
    bitonic_chunk(sk, c0, CH, k, CH >> 1);
  }
  for (uint32_t i = threadIdx.x; i < CH; i += blockDim.x) keys[c0 + i] = sk[i];
}

static __global__ void k_bitonic_step(uint64_t *__restrict__ keys, uint32_t P, uint32_t j, uint32_t k) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;  // pair index
  if (t >= P / 2) return;
  const uint32_t i = ((t & ~(j - 1)) << 1) | (t & (j - 1)), x = i | j;
  const uint64_t a = keys[i], b = keys[x];
  if ((a > b) == ((i & k) == 0)) { keys[i] = b; keys[x] = a; }
}

static __global__ void __launch_bounds__(1024) k_huff_codes(const uint64_t *__restrict__ keys, uint32_t sigma,
                                                     uint32_t *__restrict__ scr, uint8_t *__restrict__ code_len,
                                                     uint32_t *__restrict__ code, uint32_t *__restrict__ pad,
                                                     uint32_t *__restrict__ sym_sorted, HuffCanon *canon,
                                                     uint64_t *__restrict__ info) {
  __shared__ uint32_t cnt[HUFF_MAXLEN + 2], first[HUFF_MAXLEN + 2], offs[HUFF_MAXLEN + 2];
  __shared__ unsigned long long tot[HUFF_MAXLEN + 2];
  __shared__ uint32_t s_lh, s_ih, s_ic, s_kl, s_ki, s_done, s_nph, s_h;
  const uint32_t tid = threadIdx.x;
  // phase stamps (globaltimer ns) in info[40..46] and the round count in info[39] (diagnostics)
#define HUFF_STAMP(i)                                                                          \
  if (tid == 0) {                                                                              \
    unsigned long long t_;                                                                     \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                     \
    info[40 + (i)] = t_;                                                                       \
  }
  const int lane = tid & 31, warp = tid >> 5;
  uint32_t *iw = scr, *lpar = scr + sigma, *ipar = scr + 2 * sigma, *phase_end = scr + 3 * sigma;
  uint32_t *dep = scr + 4 * sigma, *slot = scr + 5 * sigma;
  const uint32_t m = (uint32_t)info[1];
  if (tid < HUFF_MAXLEN + 2) { cnt[tid] = 0; tot[tid] = 0; }
  HUFF_STAMP(0)
  HUFF_STAMP(1)
  HUFF_STAMP(2)
  // ---- code lengths: rounds of the two-queue method ----
  auto lwt = [&](uint32_t i) -> uint64_t { return keys[i] >> 32; };
  auto iwt = [&](uint32_t j) -> uint64_t { return iw[j]; };
  if (tid == 0) { s_lh = 0; s_ih = 0; s_ic = 0; s_nph = 0; s_done = m < 2; }
  __syncthreads();
  while (!s_done) {
    const uint32_t lh = s_lh, ih = s_ih, ic = s_ic;
    if (warp == 0) {
      // the two lightest items (a leaf first on equal weight)
      uint64_t w2[2];
      uint32_t a = lh, b = ih;
      for (int t = 0; t < 2; t++) {
        const bool leaf = a < m && (b >= ic || lwt(a) <= iwt(b));
        w2[t] = leaf ? lwt(a++) : iwt(b++);
      }
      const uint64_t sw = w2[0] + w2[1];
      uint32_t kl = warp_upper(lwt, lh, m, sw, lane) - lh;
      uint32_t ki = warp_upper(iwt, ih, ic, sw, lane) - ih;
      if ((kl + ki) & 1u) {  // the last item in queue order waits for the next round
        if (ki > 0 && (kl == 0 || iwt(ih + ki - 1) >= lwt(lh + kl - 1))) ki--;
        else kl--;
      }
      if (lane == 0) { s_kl = kl; s_ki = ki; }
    }
    __syncthreads();
    const uint32_t kl = s_kl, ki = s_ki, k = kl + ki;
    // queue-order rank of every item of the round (binary search in the other queue)
    for (uint32_t a = tid; a < kl; a += blockDim.x) {
      const uint64_t w = lwt(lh + a);
      uint32_t lo = 0, hi = ki;  // internal items strictly lighter come first
      while (lo < hi) { const uint32_t md = (lo + hi) >> 1; if (iwt(ih + md) < w) lo = md + 1; else hi = md; }
      slot[a + lo] = lh + a;
    }
    for (uint32_t b = tid; b < ki; b += blockDim.x) {
      const uint64_t w = iwt(ih + b);
      uint32_t lo = 0, hi = kl;  // leaves of equal weight come first
      while (lo < hi) { const uint32_t md = (lo + hi) >> 1; if (lwt(lh + md) <= w) lo = md + 1; else hi = md; }
      slot[b + lo] = 0x80000000u | (ih + b);
    }
    __syncthreads();
    for (uint32_t r = tid; r < k / 2; r += blockDim.x) {
      const uint32_t x = slot[2 * r], y = slot[2 * r + 1], node = ic + r;
      const uint64_t wx = (x >> 31) ? iwt(x & 0x7fffffffu) : lwt(x);
      const uint64_t wy = (y >> 31) ? iwt(y & 0x7fffffffu) : lwt(y);
      iw[node] = (uint32_t)(wx + wy);
      if (x >> 31) ipar[x & 0x7fffffffu] = node; else lpar[x] = node;
      if (y >> 31) ipar[y & 0x7fffffffu] = node; else lpar[y] = node;
    }
    __syncthreads();
    if (tid == 0) {
      s_lh = lh + kl;
      s_ih = ih + ki;
      s_ic = ic + k / 2;
      phase_end[s_nph++] = ic + k / 2;
      s_done = (m - s_lh) + (s_ic - s_ih) <= 1;
    }
    __syncthreads();
  }
  HUFF_STAMP(3)
  if (tid == 0) info[39] = s_nph;
  // depths of internal nodes, rounds in reverse (a parent is made in a later round)
  if (m >= 2) {
    const uint32_t root = m - 2;
    for (int ph = (int)s_nph - 1; ph >= 0; ph--) {
      const uint32_t lo = ph ? phase_end[ph - 1] : 0u, hi = phase_end[ph];
      for (uint32_t j = lo + tid; j < hi; j += blockDim.x) dep[j] = j == root ? 0u : dep[ipar[j]] + 1;
      __syncthreads();
    }
  }
  uint32_t hloc = 0;
  for (uint32_t i = tid; i < m && m >= 2; i += blockDim.x) hloc = max(hloc, dep[lpar[i]] + 1);
  for (int o = 16; o; o >>= 1) hloc = max(hloc, __shfl_xor_sync(FULL, hloc, o));
  if (tid == 0) s_h = 0;
  __syncthreads();
  if (lane == 0) atomicMax(&s_h, hloc);
  __syncthreads();
  const uint32_t h = s_h;
  if (tid == 0) {
    info[0] = h;
    info[1] = m;
    info[2] = m == 1 ? (uint32_t)(keys[0] & 0xffffffffu) : 0u;
    info[3] = h > HUFF_MAXLEN ? 1u : 0u;
  }
  if (h > HUFF_MAXLEN) return;

  HUFF_STAMP(4)
  // scatter the lengths to symbols; per-length symbol and element totals
  for (uint32_t c = tid; c < sigma; c += blockDim.x) code_len[c] = 0;
  __syncthreads();
  for (uint32_t i0 = 0; i0 < m && m >= 2; i0 += blockDim.x) {
    const uint32_t i = i0 + tid;
    const bool ok = i < m;
    const uint64_t kv = ok ? keys[i] : 0ull;
    const uint32_t L = ok ? dep[lpar[i]] + 1 : 0u, f = (uint32_t)(kv >> 32);
    if (ok) code_len[(uint32_t)(kv & 0xffffffffu)] = (uint8_t)L;
    const uint32_t peers = __match_any_sync(FULL, L);
    const uint32_t fs = __reduce_add_sync(peers, f);  // < n < 2^32
    if (ok && lane == __ffs(peers) - 1) {
      atomicAdd(&cnt[L], (uint32_t)__popc(peers));
      atomicAdd(&tot[L], (unsigned long long)fs);
    }
  }
  __syncthreads();
  // canonical first codes (R-18): code(L) = (code(L-1) + count(L-1)) << 1
  if (tid == 0) {
    uint32_t c = 0, o = 0;
    first[0] = 0;
    offs[0] = 0;
    for (uint32_t L = 1; L <= HUFF_MAXLEN + 1; L++) {
      c = (c + cnt[L - 1]) << 1;
      first[L] = c;
      offs[L] = o;
      o += L <= h ? cnt[L] : 0u;
    }
    cnt[0] = 0;
    for (uint32_t L = 0; L < HUFF_MAXLEN + 2; L++) {
      canon->first[L] = first[L];
      canon->count[L] = L <= h ? cnt[L] : 0u;
      canon->offset[L] = offs[L];
    }
    unsigned long long above = 0;  // elements with code length > l
    for (int l = (int)HUFF_MAXLEN; l >= 0; l--) {
      if (l < (int)HUFF_MAXLEN) info[4 + l] = above;
      above += (l >= 1 && (uint32_t)l <= h) ? tot[l] : 0ull;
    }
  }
  __syncthreads();
  HUFF_STAMP(5)
  // codes in symbol order within each length: chunks of 1024 symbols; the
  // rank among equal lengths = earlier chunks + earlier warps + earlier lanes
  {
    __shared__ uint32_t wcnt[32][HUFF_MAXLEN + 1];
    __shared__ uint32_t run[HUFF_MAXLEN + 1];
    if (tid <= HUFF_MAXLEN) run[tid] = 0;
    for (uint32_t c0 = 0; c0 < sigma; c0 += blockDim.x) {
      const uint32_t c = c0 + tid;
      const uint32_t L = c < sigma ? code_len[c] : 0u;
      const uint32_t peers = __match_any_sync(FULL, L);
      const uint32_t rin = __popc(peers & lanemask_lt());
      for (uint32_t k = lane; k <= HUFF_MAXLEN; k += 32) wcnt[warp][k] = 0;
      __syncwarp();
      if (rin == 0) wcnt[warp][L] = __popc(peers);
      __syncthreads();
      if (tid <= HUFF_MAXLEN) {  // exclusive scan over warps for length tid
        uint32_t acc = run[tid];
        for (int w = 0; w < 32; w++) { const uint32_t x = wcnt[w][tid]; wcnt[w][tid] = acc; acc += x; }
        run[tid] = acc;
      }
      __syncthreads();
      if (L) {
        const uint32_t r = wcnt[warp][L] + rin;
        const uint32_t cd = first[L] + r;
        code[c] = cd;
        pad[c] = h == L ? cd : (cd << (h - L));
        sym_sorted[offs[L] + r] = c;
      }
      __syncthreads();
    }
  }
  HUFF_STAMP(6)
  for (uint32_t c = tid; c < sigma; c += blockDim.x)
    if (code_len[c] == 0) { code[c] = 0; pad[c] = 0; }
}

// ---------------------------------------------------------------------------
// H3: X[i] = padded code of S[i].
// ---------------------------------------------------------------------------
template <typename InT, typename OutT, bool SMEM>
__global__ void __launch_bounds__(512) k_huff_map(const InT *__restrict__ S, uint64_t n, uint32_t sigma,
                                                  const uint32_t *__restrict__ pad, OutT *__restrict__ X) {
  extern __shared__ __align__(16) unsigned char map_smem[];
  OutT *tab = reinterpret_cast<OutT *>(map_smem);
  if constexpr (SMEM) {
    for (uint32_t c = threadIdx.x; c < sigma; c += blockDim.x) tab[c] = (OutT)pad[c];
    __syncthreads();
  }
  auto look = [&](uint32_t v) -> OutT { return SMEM ? tab[v] : (OutT)__ldg(pad + v); };
  // 16-byte vectors of S (E symbols each), U vectors in flight per thread;
  // S from the CUDA allocator is 256-byte aligned, the tail runs scalar
  constexpr uint32_t E = 16 / sizeof(InT), U = 4;
  const uint64_t nv = ((uintptr_t)S % 16 == 0) ? n / E : 0;
  const uint4 *SV = reinterpret_cast<const uint4 *>(S);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * U;
  for (uint64_t v0 = (uint64_t)blockIdx.x * blockDim.x * U + threadIdx.x; v0 < nv; v0 += stride) {
    uint4 q[U];
#pragma unroll
    for (uint32_t u = 0; u < U; u++) {
      const uint64_t vi = v0 + (uint64_t)u * blockDim.x;
      q[u] = vi < nv ? __ldcs(SV + vi) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (uint32_t u = 0; u < U; u++) {
      const uint64_t vi = v0 + (uint64_t)u * blockDim.x;
      if (vi >= nv) break;
      const InT *e = reinterpret_cast<const InT *>(&q[u]);
      OutT o[E];
#pragma unroll
      for (uint32_t k = 0; k < E; k++) o[k] = look((uint32_t)e[k]);
      OutT *dst = X + vi * E;
      if constexpr (E * sizeof(OutT) == 16) *reinterpret_cast<uint4 *>(dst) = *reinterpret_cast<const uint4 *>(o);
      else if constexpr (E * sizeof(OutT) == 8) *reinterpret_cast<uint2 *>(dst) = *reinterpret_cast<const uint2 *>(o);
      else if constexpr (E * sizeof(OutT) == 32) {
        reinterpret_cast<uint4 *>(dst)[0] = reinterpret_cast<const uint4 *>(o)[0];
        reinterpret_cast<uint4 *>(dst)[1] = reinterpret_cast<const uint4 *>(o)[1];
      } else {
#pragma unroll
        for (uint32_t k = 0; k < E; k++) dst[k] = o[k];
      }
    }
  }
  for (uint64_t i = nv * E + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    X[i] = look((uint32_t)S[i]);
}

// ---------------------------------------------------------------------------
// H4a: per level (one CTA each), the padded tree's nodes that are still
// internal Huffman nodes, in order, with their source and destination starts.
//   seg_* are laid out like the padded node table (offset level_node_ptr[l]);
//   alive[l] = number of surviving nodes; err |= 2 when their total length
//   differs from n_l.
// ---------------------------------------------------------------------------
static __global__ void __launch_bounds__(1024) k_hwt_segments(const uint64_t *__restrict__ pptr, const uint32_t *__restrict__ pkey,
                                                       const uint32_t *__restrict__ pstart, uint64_t n,
                                                       const HuffCanon *__restrict__ canon, const uint64_t *__restrict__ info,
                                                       uint32_t *__restrict__ seg_src, uint32_t *__restrict__ seg_dst,
                                                       uint32_t *__restrict__ seg_key, uint32_t *__restrict__ alive,
                                                       uint32_t *err, uint32_t lbase) {
  __shared__ uint32_t shm[33];
  const uint32_t l = lbase + blockIdx.x;
  const uint64_t lo = pptr[l], hi = pptr[l + 1];
  uint32_t nalive = 0, dst = 0;
  for (uint64_t j0 = lo; j0 < hi; j0 += blockDim.x) {
    const uint64_t j = j0 + threadIdx.x;
    uint32_t len = 0, live = 0, p = 0, st = 0;
    if (j < hi) {
      p = pkey[j];
      st = pstart[j];
      const uint64_t en = j + 1 < hi ? pstart[j + 1] : n;
      len = (uint32_t)(en - st);
      live = 1;
      // a leaf of length L <= l whose code is the top L bits of p kills the node
      for (uint32_t L = 1; L <= l; L++) {
        const uint32_t q = p >> (l - L);
        if (q - canon->first[L] < canon->count[L]) { live = 0; break; }
      }
    }
    uint32_t tl, tc;
    const uint32_t ex_len = block_exscan(live ? len : 0u, shm, &tl);
    const uint32_t ex_cnt = block_exscan(live, shm, &tc);
    if (live) {
      seg_src[lo + nalive + ex_cnt] = st;
      seg_dst[lo + nalive + ex_cnt] = dst + ex_len;
      seg_key[lo + nalive + ex_cnt] = p;
    }
    nalive += tc;
    dst += tl;
  }
  if (threadIdx.x == 0) {
    alive[l] = nalive;
    if ((uint64_t)dst != info[4 + l]) atomicOr(err, 2u);
  }
}

// ---------------------------------------------------------------------------
// Staged mode (skewed codes): the keys of stage g are the padded codes,
// truncated to their top `hi` bits, of the elements whose code is longer than
// `lo` (they alone reach level lo), in S order -- a stable compaction.
// k_hwt_alive_count: per tile of PART_TILE elements, the number alive.
// k_hwt_alive_scatter: after the scan of the tile counts, each warp ranks its
// 16 chunks of 32 with ballots.
// ---------------------------------------------------------------------------
constexpr uint32_t HA_TILE = 4096, HA_THREADS = 256, HA_PER = HA_TILE / HA_THREADS;

template <typename InT>
__global__ void __launch_bounds__(HA_THREADS) k_hwt_alive_count(const InT *__restrict__ S, uint64_t n,
                                                               const uint8_t *__restrict__ code_len, uint32_t lo,
                                                               uint32_t ntiles, uint32_t *__restrict__ tcount) {
  __shared__ uint32_t c;
  if (threadIdx.x == 0) c = 0;
  __syncthreads();
  const uint64_t b = (uint64_t)blockIdx.x * HA_TILE;
  uint32_t mine = 0;
  for (uint32_t i = threadIdx.x; i < HA_TILE; i += blockDim.x)
    if (b + i < n && code_len[(uint32_t)S[b + i]] > lo) mine++;
  mine = __reduce_add_sync(FULL, mine);
  if ((threadIdx.x & 31) == 0) atomicAdd(&c, mine);
  __syncthreads();
  if (threadIdx.x == 0) tcount[blockIdx.x] = c;
}

template <typename InT, typename OutT>
__global__ void __launch_bounds__(HA_THREADS) k_hwt_alive_scatter(const InT *__restrict__ S, uint64_t n,
                                                                 const uint8_t *__restrict__ code_len,
                                                                 const uint32_t *__restrict__ pad, uint32_t lo,
                                                                 uint32_t shift, const uint32_t *__restrict__ toff,
                                                                 OutT *__restrict__ out) {
  constexpr uint32_t NW = HA_THREADS / 32;
  __shared__ uint32_t wc[NW];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t wb = (uint64_t)blockIdx.x * HA_TILE + (uint64_t)warp * HA_PER * 32;
  uint32_t key[HA_PER], m[HA_PER], cnt = 0;
#pragma unroll
  for (uint32_t c = 0; c < HA_PER; c++) {
    const uint64_t j = wb + c * 32 + lane;
    uint32_t sym = j < n ? (uint32_t)S[j] : 0u;
    const bool ok = j < n && code_len[sym] > lo;
    key[c] = ok ? pad[sym] >> shift : 0u;
    m[c] = __ballot_sync(FULL, ok);
    cnt += __popc(m[c]);
  }
  if (lane == 0) wc[warp] = cnt;
  __syncthreads();
  uint32_t off = toff[blockIdx.x];
  for (int w = 0; w < warp; w++) off += wc[w];
#pragma unroll
  for (uint32_t c = 0; c < HA_PER; c++) {
    if ((m[c] >> lane) & 1u) out[off + __popc(m[c] & lanemask_lt())] = (OutT)key[c];
    off += __popc(m[c]);
  }
}

// Per-level bookkeeping passed by value (host knows it after H2).
struct HwtLevels {
  uint32_t h;
  uint32_t lbase;                   // first level of the current stage (blockIdx.y = level - lbase)
  uint64_t nl[HUFF_MAXLEN];
  uint64_t wptr[HUFF_MAXLEN + 1];   // output word offset of each level
  uint64_t segbase[HUFF_MAXLEN];    // padded node-table offset of the level
  uint32_t nseg[HUFF_MAXLEN];       // surviving nodes of the level
};

// ---------------------------------------------------------------------------
// H4b: gather the surviving bit ranges of each padded level (funnel-shifted
// 64-bit windows).  A CTA owns 256 consecutive output words of one level
// (blockIdx.y = level): warp 0 finds the segments that cover the CTA's bit
// range with one 32-ary search, stages up to HB_SEGS of them in shared
// memory, and every thread then locates its word's first segment there.
// ---------------------------------------------------------------------------
constexpr uint32_t HB_WORDS = 256, HB_WPT = 8, HB_SEGS = 2048;

static __global__ void __launch_bounds__(HB_WORDS) k_hwt_bits(HwtLevels lv, const uint64_t *__restrict__ pbits, uint64_t pwpl,
                                                       const uint32_t *__restrict__ seg_src,
                                                       const uint32_t *__restrict__ seg_dst, uint64_t *__restrict__ out) {
  __shared__ uint32_t s_dst[HB_SEGS + 1], s_src[HB_SEGS];
  __shared__ uint32_t s_k0, s_k1;
  const uint32_t l = lv.lbase + blockIdx.y;
  const uint64_t nw = lv.wptr[l + 1] - lv.wptr[l];
  const uint64_t w0 = (uint64_t)blockIdx.x * HB_WORDS * HB_WPT;
  if (w0 >= nw) return;
  const uint64_t nl = lv.nl[l];
  const uint32_t *sd = seg_dst + lv.segbase[l];
  const uint32_t *ss = seg_src + lv.segbase[l];
  const uint32_t ns = lv.nseg[l];
  const uint64_t bit0 = w0 * 64, bit1 = min((w0 + HB_WORDS * HB_WPT) * 64, nl);
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    auto dstw = [&](uint32_t k) -> uint64_t { return sd[k]; };
    // k0 = last segment with dst <= bit0; k1 = first segment with dst >= bit1
    const uint32_t k0 = bit0 < nl ? warp_upper(dstw, 0, ns, bit0, lane) - 1 : 0u;
    const uint32_t k1 = bit0 < nl ? warp_upper(dstw, k0, ns, bit1 - 1, lane) : 0u;
    if (lane == 0) { s_k0 = k0; s_k1 = k1; }
  }
  __syncthreads();
  const uint32_t k0 = s_k0, k1 = s_k1, cnt = k1 - k0;
  const bool staged = cnt <= HB_SEGS;
  if (staged) {
    for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) { s_dst[i] = sd[k0 + i]; s_src[i] = ss[k0 + i]; }
    if (threadIdx.x == 0) s_dst[cnt] = k1 < ns ? sd[k1] : (uint32_t)nl;
  }
  __syncthreads();
  const uint64_t *P = pbits + (uint64_t)l * pwpl;
  for (uint32_t r = 0; r < HB_WPT; r++) {
    const uint64_t w = w0 + r * HB_WORDS + threadIdx.x;
    if (w >= nw) break;
    const uint64_t b0 = w * 64;
    uint64_t res = 0;
    if (b0 < nl) {
      const uint64_t b1 = b0 + 64 < nl ? b0 + 64 : nl;
      // the segment (relative to k0) holding bit b0
      uint32_t a = 0, z = cnt;
      while (z - a > 1) {
        const uint32_t mid = (a + z) >> 1;
        if ((staged ? s_dst[mid] : sd[k0 + mid]) <= b0) a = mid; else z = mid;
      }
      uint64_t pos = b0;
      for (uint32_t k = a; pos < b1 && k < cnt; k++) {
        const uint64_t dk = staged ? s_dst[k] : sd[k0 + k];
        const uint64_t dend = staged ? s_dst[k + 1] : (k0 + k + 1 < ns ? sd[k0 + k + 1] : nl);
        if (dend <= pos) continue;
        const uint64_t take = (dend < b1 ? dend : b1) - pos;
        const uint64_t src = (staged ? s_src[k] : ss[k0 + k]) + (pos - dk);
        const uint64_t wi = src >> 6, o = src & 63;
        uint64_t v = P[wi] >> o;
        if (o && o + take > 64) v |= P[wi + 1] << (64 - o);
        if (take < 64) v &= (1ull << take) - 1ull;
        res |= v << (pos - b0);
        pos += take;
      }
    }
    out[lv.wptr[l] + w] = res;
  }
}

// Rank directory of all levels in two launches (per-level offsets by value).
struct HwtRankLv {
  uint32_t h;
  uint64_t nl[HUFF_MAXLEN];
  uint64_t wptr[HUFF_MAXLEN + 1], bptr[HUFF_MAXLEN + 1], sptr[HUFF_MAXLEN + 1];
  uint64_t soff[HUFF_MAXLEN + 1];  // cumulative superblocks holding data
};

// one warp per (level, data superblock): popcounts of its <= 128 blocks and
// the in-superblock scan (the per-level layout of k_rank_local)
static __global__ void k_hwt_rank_local(HwtRankLv r, const uint64_t *__restrict__ bits, uint16_t *__restrict__ rank_block,
                                 uint64_t *__restrict__ suptot) {
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= r.soff[r.h]) return;
  uint32_t l = 0;
  while (r.soff[l + 1] <= gw) l++;
  const uint64_t sidx = gw - r.soff[l];
  const uint64_t bpl = r.bptr[l + 1] - r.bptr[l];
  const uint64_t *B = bits + r.wptr[l];
  uint32_t v[4], sum = 0;
#pragma unroll
  for (int i = 0; i < 4; i++) {
    const uint64_t b = sidx * 128 + lane * 4 + i;
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
    const uint64_t b = sidx * 128 + lane * 4 + i;
    if (b < bpl) rank_block[r.bptr[l] + b] = (uint16_t)run;
    run += v[i];
  }
  if (lane == 31) suptot[gw] = incl;
}

// one CTA per level: exclusive scan of the superblock totals (+ the total)
static __global__ void __launch_bounds__(1024) k_hwt_rank_super(HwtRankLv r, const uint64_t *__restrict__ suptot,
                                                        uint64_t *__restrict__ rank_super) {
  __shared__ unsigned long long warp_tot[33];
  const uint32_t l = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t nsd = r.soff[l + 1] - r.soff[l], spl = r.sptr[l + 1] - r.sptr[l];
  const uint64_t *st = suptot + r.soff[l];
  uint64_t *rs = rank_super + r.sptr[l];
  unsigned long long carry = 0;
  for (uint64_t base = 0; base < spl; base += blockDim.x) {
    const uint64_t si = base + threadIdx.x;
    const unsigned long long v = si < nsd ? st[si] : 0ull;
    unsigned long long incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long t = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const unsigned long long w = warp_tot[lane];
      unsigned long long wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long t = __shfl_up_sync(FULL, wi, o);
        if (lane >= o) wi += t;
      }
      warp_tot[lane] = wi - w;
      if (lane == 31) warp_tot[32] = wi;
    }
    __syncthreads();
    if (si < spl) rs[si] = carry + warp_tot[warp] + incl - v;
    carry += warp_tot[32];
    __syncthreads();
  }
}

// Node table of the Huffman-shaped tree from the surviving segments.
static __global__ void k_hwt_nodes(HwtLevels lv, const uint64_t *__restrict__ optr, const uint32_t *__restrict__ seg_key,
                            const uint32_t *__restrict__ seg_dst, uint32_t *__restrict__ node_key,
                            uint32_t *__restrict__ node_start) {
  const uint32_t l = lv.lbase + blockIdx.y;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < lv.nseg[l]; j += gridDim.x * blockDim.x) {
    node_key[optr[l] + j] = seg_key[lv.segbase[l] + j];
    node_start[optr[l] + j] = seg_dst[lv.segbase[l] + j];
  }
}

// ---------------------------------------------------------------------------
// Queries (verification path, PAPER.md:204-206 on the Huffman shape).
// ---------------------------------------------------------------------------
struct HwtView {
  uint64_t n;
  uint32_t h, only_symbol;
  uint64_t sigma;
  const uint64_t *level_len, *wptr, *bptr, *sptr, *node_ptr;
  const uint64_t *bits;
  const uint16_t *rank_block;
  const uint64_t *rank_super;
  const uint32_t *node_key, *node_start, *code, *sym_sorted;
  const uint8_t *code_len;
  const HuffCanon *canon;
};

__device__ __forceinline__ uint64_t hwt_rank1(const HwtView &t, uint32_t l, uint64_t i) {
  const uint64_t nl = t.level_len[l];
  const uint64_t *sup = t.rank_super + t.sptr[l];
  if (i >= nl) return sup[t.sptr[l + 1] - t.sptr[l] - 1];
  const uint64_t *B = t.bits + t.wptr[l];
  uint64_t r = sup[i >> 16] + t.rank_block[t.bptr[l] + (i >> 9)];
  for (uint64_t w = (i >> 9) * 8; w < (i >> 6); w++) r += __popcll(B[w]);
  if (i & 63) r += __popcll(B[i >> 6] & ((1ull << (i & 63)) - 1ull));
  return r;
}

// start of node (l, p), binary search over the level's sorted keys
__device__ __forceinline__ bool hwt_node_start(const HwtView &t, uint32_t l, uint32_t p, uint64_t *s) {
  uint64_t a = t.node_ptr[l], z = t.node_ptr[l + 1];
  while (a < z) {
    const uint64_t mid = (a + z) >> 1;
    if (t.node_key[mid] < p) a = mid + 1; else z = mid;
  }
  if (a < t.node_ptr[l + 1] && t.node_key[a] == p) { *s = t.node_start[a]; return true; }
  return false;
}

static __global__ void k_hwt_access(HwtView t, const uint64_t *__restrict__ pos, uint64_t q, uint32_t *__restrict__ out) {
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= q) return;
  uint64_t i = pos[k];
  if (i >= t.n) { out[k] = 0xffffffffu; return; }
  if (t.h == 0) { out[k] = t.only_symbol; return; }
  uint64_t s = 0;
  uint32_t p = 0, res = 0xffffffffu;
  for (uint32_t l = 0; l < t.h; l++) {
    const uint32_t bit = (uint32_t)((t.bits[t.wptr[l] + (i >> 6)] >> (i & 63)) & 1ull);
    const uint64_t r1s = hwt_rank1(t, l, s), r1i = hwt_rank1(t, l, i);
    const uint64_t r = bit ? r1i - r1s : (i - s) - (r1i - r1s);
    p = 2 * p + bit;
    const uint32_t L = l + 1;
    if (p - t.canon->first[L] < t.canon->count[L]) { res = t.sym_sorted[t.canon->offset[L] + p - t.canon->first[L]]; break; }
    if (!hwt_node_start(t, L, p, &s)) break;
    i = s + r;
  }
  out[k] = res;
}

static __global__ void k_hwt_rank(HwtView t, const uint32_t *__restrict__ sym, const uint64_t *__restrict__ pos, uint64_t q,
                           uint64_t *__restrict__ out) {
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= q) return;
  const uint64_t i = pos[k];
  const uint32_t c = sym[k];
  if (i >= t.n || (uint64_t)c >= t.sigma) { out[k] = ~0ull; return; }
  if (t.h == 0) { out[k] = c == t.only_symbol ? i + 1 : 0ull; return; }
  const uint32_t L = t.code_len[c];
  if (L == 0) { out[k] = 0; return; }
  const uint32_t cd = t.code[c];
  uint64_t s = 0, r = i + 1;
  uint32_t p = 0;
  for (uint32_t l = 0; l < L; l++) {
    const uint32_t bit = (cd >> (L - 1 - l)) & 1u;
    const uint64_t r1s = hwt_rank1(t, l, s), r1p = hwt_rank1(t, l, s + r);
    r = bit ? r1p - r1s : r - (r1p - r1s);
    if (r == 0) break;
    p = 2 * p + bit;
    if (l + 1 < L && !hwt_node_start(t, l + 1, p, &s)) { r = ~0ull; break; }
  }
  out[k] = r;
}

// select_c on the Huffman-shaped tree: descend along c's
// code for the node of every level, then climb from the deepest node with
// select_b inside each node; select_b by binary searches over the level's
// superblocks, blocks and words (no select directory for ragged levels).
__device__ __forceinline__ uint32_t hwt_select_in_word(uint64_t v, uint32_t r) {  // r'th (0-based) set bit
  for (uint32_t i = 0; i < r; i++) v &= v - 1;
  return (uint32_t)__ffsll((long long)v) - 1u;
}

// position of the T'th (1-based) b-bit of level l, or UINT64_MAX
__device__ __forceinline__ uint64_t hwt_select_b(const HwtView &t, uint32_t l, uint32_t b, uint64_t T) {
  const uint64_t nl = t.level_len[l];
  const uint64_t nsd = t.sptr[l + 1] - t.sptr[l] - 1;  // superblocks holding data
  const uint64_t *sup = t.rank_super + t.sptr[l];
  const uint16_t *blk = t.rank_block + t.bptr[l];
  const uint64_t *B = t.bits + t.wptr[l];
  auto before_sup = [&](uint64_t i) -> uint64_t {  // b-bits in [0, min(i*65536, nl))
    const uint64_t p = i * 65536 < nl ? i * 65536 : nl;
    return b ? sup[i] : p - sup[i];
  };
  if (T == 0 || before_sup(nsd) < T) return ~0ull;
  uint64_t lo = 0, hi = nsd;  // last superblock with before < T
  while (hi - lo > 1) {
    const uint64_t mid = (lo + hi) >> 1;
    if (before_sup(mid) < T) lo = mid; else hi = mid;
  }
  const uint64_t base_s = before_sup(lo);
  const uint64_t nblk = t.bptr[l + 1] - t.bptr[l];
  uint64_t blo = lo * 128, bhi = (lo * 128 + 128 < nblk ? lo * 128 + 128 : nblk);
  auto before_blk = [&](uint64_t j) -> uint64_t {
    const uint64_t ones = blk[j];
    return base_s + (b ? ones : (j * 512 - lo * 65536) - ones);
  };
  while (bhi - blo > 1) {
    const uint64_t mid = (blo + bhi) >> 1;
    if (before_blk(mid) < T) blo = mid; else bhi = mid;
  }
  uint64_t need = T - 1 - before_blk(blo);
  for (int i = 0; i < 8; i++) {
    const uint64_t base = blo * 512 + i * 64;
    if (base >= nl) break;
    uint64_t v = b ? B[blo * 8 + i] : ~B[blo * 8 + i];
    if (base + 64 > nl) v &= (1ull << (nl - base)) - 1ull;
    const uint32_t pc = __popcll(v);
    if (need < pc) return base + hwt_select_in_word(v, (uint32_t)need);
    need -= pc;
  }
  return ~0ull;
}

__device__ __forceinline__ uint64_t hwt_rank_b(const HwtView &t, uint32_t l, uint64_t i, uint32_t b) {
  const uint64_t r1 = hwt_rank1(t, l, i);
  return b ? r1 : i - r1;
}

static __global__ void k_hwt_select(HwtView t, const uint32_t *__restrict__ sym, const uint64_t *__restrict__ kk,
                                    uint64_t q, uint64_t *__restrict__ out) {
  const uint64_t qi = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (qi >= q) return;
  const uint32_t c = sym[qi];
  const uint64_t K = kk[qi];
  uint64_t res = ~0ull;
  if ((uint64_t)c < t.sigma && K > 0) {
    if (t.h == 0) {
      if (t.n && c == t.only_symbol && K <= t.n) res = K - 1;
    } else if (t.code_len[c]) {
      const uint32_t L = t.code_len[c], cd = t.code[c];
      uint64_t st[HUFF_MAXLEN];
      st[0] = 0;
      uint32_t p = 0;
      bool ok = true;
      for (uint32_t l = 0; l + 1 < L && ok; l++) {
        p = 2 * p + ((cd >> (L - 1 - l)) & 1u);
        ok = hwt_node_start(t, l + 1, p, &st[l + 1]);
      }
      if (ok) {
        uint64_t r = K;  // 1-based rank inside the node of level l
        for (int l = (int)L - 1; l >= 0 && r != ~0ull; l--) {
          const uint32_t b = (cd >> (L - 1 - (uint32_t)l)) & 1u;
          const uint64_t pos = hwt_select_b(t, (uint32_t)l, b, hwt_rank_b(t, (uint32_t)l, st[l], b) + r);
          // the answer must lie inside the node: its b-bits before pos, counted from the node start, are r - 1
          r = pos == ~0ull ? ~0ull : pos - st[l] + 1;
          if (r != ~0ull && l == (int)L - 1) {
            // node end at the deepest level: the next node's start (or the level end)
            uint64_t a = t.node_ptr[l], z = t.node_ptr[l + 1], e = t.level_len[l];
            while (a < z) {
              const uint64_t mid = (a + z) >> 1;
              if (t.node_key[mid] <= p) a = mid + 1; else z = mid;
            }
            if (a < t.node_ptr[l + 1]) e = t.node_start[a];
            if (pos >= e) r = ~0ull;
          }
        }
        if (r != ~0ull) res = r - 1;
      }
    }
  }
  out[qi] = res;
}

}  // namespace wtb
