// wt_prep.cuh -- A1 (validation, digit histograms), A4 (node table) and the
// chain bookkeeping of the group passes.
//
// Terms:
//  * group g: levels l0 .. l0+tau-1 built by one k_group pass; the digit of a
//    key is its tau level bits, taken from the top.
//  * row: a non-empty node of level l0 (the root for g = 0).  Its digit
//    histogram, exclusive-scanned, is Cseg[row][0..2^tau]; node (P:q) of level
//    l0+k starts at row_start[row] + Cseg[row][q << (tau-k)] (PAPER.md:468-475:
//    a level-l node is the run of S_l whose symbols share the top l bits; nodes
//    are laid out in prefix order, Fig. 2 l.11-13).
//  * chain: <= CH consecutive positions of one row, processed tile by tile by
//    one warp.  E[d][c] (exclusive scan over chains of the per-chain digit
//    counts) gives every chain the number of same-row elements with digit d
//    ahead of it: E[d][c] - E[d][first chain of the row].
#pragma once
#include "wt_common.cuh"

namespace wtb {

// ---------------------------------------------------------------------------
// Chain geometry.  Group 0: K equal chunks of the root.  Group g >= 1: every
// row (non-empty node of level l0, from the node table) split into pieces of
// <= CH positions.  One CTA of 1024 threads for g >= 1.
// ---------------------------------------------------------------------------
static __global__ void k_chains_root(uint64_t n, uint64_t CH, uint32_t K, uint32_t *__restrict__ chain_begin,
                              uint32_t *__restrict__ chain_end, uint32_t *__restrict__ chain_row,
                              uint32_t *__restrict__ row_first, uint32_t *__restrict__ row_start,
                              uint32_t *__restrict__ row_key, uint32_t *__restrict__ counts, const uint32_t *err) {
  if (*err) return;
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < K) {
    const uint64_t b = (uint64_t)c * CH, e = b + CH < n ? b + CH : n;
    chain_begin[c] = (uint32_t)b;
    chain_end[c] = (uint32_t)e;
    chain_row[c] = 0;
  }
  if (c == 0) {
    row_first[0] = 0;
    row_first[1] = K;
    row_start[0] = 0;
    row_key[0] = 0;
    counts[0] = K;  // chains
    counts[1] = 1;  // rows
  }
}

static __global__ void __launch_bounds__(1024) k_chains_from_nodes(
    const uint64_t *__restrict__ level_node_ptr, const uint32_t *__restrict__ ncount, uint32_t l0,
    const uint32_t *__restrict__ node_key, const uint32_t *__restrict__ node_start, uint64_t n, uint64_t CH,
    uint32_t *__restrict__ chain_begin, uint32_t *__restrict__ chain_end, uint32_t *__restrict__ chain_row,
    uint32_t *__restrict__ row_first, uint32_t *__restrict__ row_start, uint32_t *__restrict__ row_key,
    uint32_t *__restrict__ counts, const uint32_t *err) {
  __shared__ uint32_t shm[33];
  if (*err) return;
  // level l0's nodes were emitted by the previous group: base and count are final
  const uint64_t p0 = level_node_ptr[l0];
  const uint32_t nr = ncount[l0];
  uint32_t carry = 0;
  for (uint32_t b0 = 0; b0 < nr; b0 += blockDim.x) {
    const uint32_t r = b0 + threadIdx.x;
    uint32_t beg = 0, end = 0, nc = 0;
    if (r < nr) {
      beg = node_start[p0 + r];
      end = (r + 1 < nr) ? node_start[p0 + r + 1] : (uint32_t)n;
      nc = (uint32_t)((end - beg + CH - 1) / CH);
    }
    uint32_t tot;
    const uint32_t off = block_exscan(nc, shm, &tot) + carry;
    if (r < nr) {
      row_first[r] = off;
      row_start[r] = beg;
      row_key[r] = node_key[p0 + r];
      for (uint32_t i = 0; i < nc; i++) {
        const uint64_t b = beg + (uint64_t)i * CH;
        chain_begin[off + i] = (uint32_t)b;
        chain_end[off + i] = (uint32_t)(b + CH < end ? b + CH : end);
        chain_row[off + i] = r;
      }
    }
    carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    row_first[nr] = carry;
    counts[0] = carry;
    counts[1] = nr;
  }
}

// ---------------------------------------------------------------------------
// A1 / per-chain digit histogram: one CTA per chain; 16-byte streaming loads;
// for the root pass also validates S[i] < sigma.
// histT[d][c] = count of digit d in chain c (transposed for the scans).
// Shared counters are lane-major, h[d * 32 + lane]: every lane of a warp owns
// its own bank, so the per-element atomics are free of bank conflicts (with
// bins shared by the lanes the random digits of a warp collide in ~3.5-way
// bank conflicts and the atomics replay).  The reduction reads column
// (j + d) mod 32 so that consecutive digits hit distinct banks.
// ---------------------------------------------------------------------------
template <typename T, bool VALIDATE>
__global__ void __launch_bounds__(512) k_chain_hist(const T *__restrict__ keys, uint64_t sigma, uint32_t shift,
                                                   uint32_t ndig, const uint32_t *__restrict__ chain_begin,
                                                   const uint32_t *__restrict__ chain_end,
                                                   const uint32_t *__restrict__ counts, uint32_t stride,
                                                   uint32_t *__restrict__ histT, uint32_t *err) {
  __shared__ uint32_t h[NDIG * 32];
  if (!VALIDATE && ld_relaxed(err)) return;
  const uint32_t nchains = counts[0];
  const uint32_t lane = threadIdx.x & 31;
  bool bad = false;
  for (uint32_t c = blockIdx.x; c < nchains; c += gridDim.x) {
  for (uint32_t i = threadIdx.x; i < 32 * ndig; i += blockDim.x) h[i] = 0;
  __syncthreads();
  uint32_t *hs = h + lane;
  const uint32_t dmask = ndig - 1u;
  auto add = [&](uint32_t v) {
    if (VALIDATE && (uint64_t)v >= sigma) {
      bad = true;
      return;
    }
    atomicAdd(&hs[((v >> shift) & dmask) << 5], 1u);
  };
  const uint32_t beg = chain_begin[c], end = chain_end[c];
  constexpr int PER = 16 / sizeof(T);
  const uintptr_t sb = reinterpret_cast<uintptr_t>(keys + beg);
  const uintptr_t ab = sb & ~(uintptr_t)15;
  const int head = (int)((sb - ab) / sizeof(T));
  const uint4 *V = reinterpret_cast<const uint4 *>(ab);
  const uint32_t len = end - beg;
  const uint32_t nv = (uint32_t)(((uint64_t)head + len + PER - 1) / PER);
  // vectors [1, nfull) lie wholly inside the chain: no per-element bounds
  // checks there, two 16-byte loads in flight per thread; the (at most two)
  // partial vectors at the ends take the checked path
  const uint32_t nfull = (uint32_t)(((uint64_t)head + len) / PER);
  auto vec_checked = [&](uint32_t i) {
    const uint4 q = __ldcs(V + i);
    const T *e = reinterpret_cast<const T *>(&q);
#pragma unroll
    for (int k = 0; k < PER; k++) {
      const int64_t pos = (int64_t)i * PER + k - head;
      if (pos >= 0 && pos < (int64_t)len) add((uint32_t)e[k]);
    }
  };
  auto vec_all = [&](const uint4 &q) {
    const T *e = reinterpret_cast<const T *>(&q);
#pragma unroll
    for (int k = 0; k < PER; k++) add((uint32_t)e[k]);
  };
  if (threadIdx.x == 0) vec_checked(0);
  if (nfull < nv && threadIdx.x == (nfull % blockDim.x) && nfull > 0) vec_checked(nfull);
  uint32_t i = 1 + threadIdx.x;
  for (; i + blockDim.x < nfull; i += 2 * blockDim.x) {
    const uint4 q0 = __ldcs(V + i), q1 = __ldcs(V + i + blockDim.x);
    vec_all(q0);
    vec_all(q1);
  }
  if (i < nfull) vec_all(__ldcs(V + i));
  __syncthreads();
  for (uint32_t d = threadIdx.x; d < ndig; d += blockDim.x) {
    uint32_t sum = 0;
#pragma unroll 8
    for (uint32_t j = 0; j < 32; j++) sum += h[(d << 5) + ((j + d) & 31u)];
    histT[(uint64_t)d * stride + c] = sum;
  }
  __syncthreads();
  }
  if (VALIDATE && __any_sync(FULL, bad) && (threadIdx.x & 31) == 0) atomicOr(err, 1u);
}

// E[d][c] = sum_{c' < c} histT[d][c'] (in place), E[d][nchains] = total; one CTA per digit.
static __global__ void __launch_bounds__(1024) k_chain_scan(uint32_t *__restrict__ histT, uint32_t stride,
                                                    const uint32_t *__restrict__ counts, const uint32_t *err) {
  __shared__ uint32_t shm[33];
  if (*err) return;
  const uint32_t nc = counts[0];
  uint32_t *row = histT + (uint64_t)blockIdx.x * stride;
  uint32_t carry = 0;
  for (uint32_t b0 = 0; b0 <= nc; b0 += blockDim.x) {
    const uint32_t c = b0 + threadIdx.x;
    const uint32_t v = c < nc ? row[c] : 0u;
    uint32_t tot;
    const uint32_t ex = block_exscan(v, shm, &tot);
    if (c <= nc) row[c] = carry + ex;
    carry += tot;
    __syncthreads();
  }
}

// V[c][d] = E[d][c] - E[d][first chain of c's row]: the chain's starting digit
// counts inside its row, chain-major (one 1 KB vector per chain, bulk-copied by
// k_wgroup together with the chain's first tile).  One warp per chain.
static __global__ void k_chain_vec(const uint32_t *__restrict__ E, uint32_t stride, const uint32_t *__restrict__ chain_row,
                                   const uint32_t *__restrict__ row_first, const uint32_t *__restrict__ counts,
                                   uint32_t ndig, uint32_t *__restrict__ V, const uint32_t *err) {
  if (*err) return;
  const uint32_t c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (c >= counts[0]) return;
  const uint32_t f = row_first[chain_row[c]];
  uint32_t *out = V + (uint64_t)c * 256;
  for (uint32_t d = lane; d < 256; d += 32)
    out[d] = d < ndig ? E[(uint64_t)d * stride + c] - E[(uint64_t)d * stride + f] : 0u;
}

// Cseg[r][0..ndig] = exclusive scan over d of the row's digit totals
// E[d][row_first[r+1]] - E[d][row_first[r]].  One warp per row.
static __global__ void k_row_scan(const uint32_t *__restrict__ E, uint32_t stride, const uint32_t *__restrict__ row_first,
                           const uint32_t *__restrict__ counts, uint32_t ndig, uint32_t *__restrict__ Cseg,
                           const uint32_t *err) {
  if (*err) return;
  const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= counts[1]) return;
  const uint32_t f0 = row_first[w], f1 = row_first[w + 1];
  uint32_t *out = Cseg + (uint64_t)w * (ndig + 1);
  const uint32_t per = (ndig + 31) >> 5;
  uint32_t v[NDIG / 32], s = 0;
#pragma unroll
  for (int i = 0; i < NDIG / 32; i++) {
    const uint32_t d = lane * per + i;
    v[i] = (i < (int)per && d < ndig) ? E[(uint64_t)d * stride + f1] - E[(uint64_t)d * stride + f0] : 0u;
    s += v[i];
  }
  const uint32_t incl = warp_incl_scan(s, lane);
  uint32_t run = incl - s;
#pragma unroll
  for (int i = 0; i < NDIG / 32; i++) {
    const uint32_t d = lane * per + i;
    if (i < (int)per && d < ndig) out[d] = run;
    run += v[i];
  }
  if (lane == 31) out[ndig] = incl;
}

// ---------------------------------------------------------------------------
// A4: non-empty nodes of the group's levels l0+k (k = k_lo .. k_hi).  Node
// (P << k | q) of row r is non-empty iff its count is > 0 (Fig. 1 l.18-20);
// rows are in key order, so the CSR order is (level, row, q).  Three steps,
// all multi-CTA so that millions of rows scale:
//   k_row_nodes_count  rowcnt[k][r] = non-empty q of row r at level l0+k
//                      (from Cseg, chain mode)
//   k_scan_rows        exclusive scan of rowcnt per level (two-level scan),
//                      ncount[l0+k] = level total, level_node_ptr
//   k_row_nodes_emit   writes (key, start) at base + rowoff + local rank
// ---------------------------------------------------------------------------
static __global__ void k_row_nodes_count(const uint32_t *__restrict__ Cseg, const uint32_t *__restrict__ counts,
                                  uint32_t tau, uint32_t k_lo, uint32_t nk, uint64_t rstride,
                                  uint32_t *__restrict__ rowcnt, const uint32_t *err) {
  // one warp per (row, level): lanes test 32 prefixes q at a time
  if (*err) return;
  const uint32_t nr = counts[1], ndig = 1u << tau;
  const int lane = threadIdx.x & 31;
  const uint64_t items = (uint64_t)nr * nk;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t it = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < items; it += nwarps) {
    const uint32_t r = (uint32_t)(it % nr), kk = (uint32_t)(it / nr);
    const uint32_t k = k_lo + kk, sh = tau - k;
    const uint32_t *row = Cseg + (uint64_t)r * (ndig + 1);
    uint32_t c = 0;
    for (uint32_t q0 = 0; q0 < (1u << k); q0 += 32) {
      const uint32_t q = q0 + lane;
      const bool ne = q < (1u << k) && row[(q + 1) << sh] > row[q << sh];
      c += __popc(__ballot_sync(FULL, ne));
    }
    if (lane == 0) rowcnt[(uint64_t)kk * rstride + r] = c;
  }
}

constexpr int SCAN_BLK = 2048;  // rows per scan block

// pass 1: per (level, block) sums.  grid (nblocks, nk), 1024 threads.
static __global__ void __launch_bounds__(1024) k_scan_rows_1(const uint32_t *__restrict__ rowcnt, uint64_t rstride,
                                                     const uint32_t *__restrict__ counts, uint32_t *__restrict__ bsum,
                                                     uint32_t bstride, const uint32_t *err) {
  __shared__ uint32_t shm[33];
  if (*err) return;
  const uint32_t nr = counts[1];
  const uint64_t b0 = (uint64_t)blockIdx.x * SCAN_BLK;
  if (b0 >= nr) return;
  const uint32_t *rc = rowcnt + (uint64_t)blockIdx.y * rstride;
  uint32_t s = 0;
  for (uint64_t r = b0 + threadIdx.x; r < b0 + SCAN_BLK && r < nr; r += blockDim.x) s += rc[r];
  uint32_t tot;
  block_exscan(s, shm, &tot);
  if (threadIdx.x == 0) bsum[(uint64_t)blockIdx.y * bstride + blockIdx.x] = tot;
}

// pass 2: per level, exclusive scan of the block sums (one CTA per level);
// also the level totals, their CSR bases and level_node_ptr.
static __global__ void __launch_bounds__(1024) k_scan_rows_2(uint32_t *__restrict__ bsum, uint32_t bstride,
                                                     const uint32_t *__restrict__ counts, uint32_t l0, uint32_t k_lo,
                                                     uint32_t nk, uint32_t L, uint32_t *__restrict__ ncount,
                                                     uint64_t *__restrict__ level_node_ptr, const uint32_t *err) {
  __shared__ uint32_t shm[33];
  if (*err) return;
  const uint32_t nr = counts[1];
  const uint32_t nb = (nr + SCAN_BLK - 1) / SCAN_BLK;
  uint32_t *bs = bsum + (uint64_t)blockIdx.x * bstride;
  uint32_t carry = 0;
  for (uint32_t b0 = 0; b0 < nb; b0 += blockDim.x) {
    const uint32_t b = b0 + threadIdx.x;
    const uint32_t v = b < nb ? bs[b] : 0u;
    uint32_t tot;
    const uint32_t ex = block_exscan(v, shm, &tot);
    if (b < nb) bs[b] = carry + ex;
    carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) ncount[l0 + k_lo + blockIdx.x] = carry;
}

// Node table of group 0 (one row: the root, l0 = 0) in one warp: levels
// k_lo .. k_lo+nk-1 in order, non-empty classes of the root's digit scan
// Cseg[0] (Fig. 1 l.18-20); also ncount[] and level_node_ptr[] of those
// levels.  Replaces the count / scan / emit passes of the general case.
static __global__ void k_root_nodes(const uint32_t *__restrict__ Cseg, uint32_t tau, uint32_t k_lo, uint32_t nk,
                                    uint32_t L, uint32_t *__restrict__ ncount, uint64_t *__restrict__ level_node_ptr,
                                    uint32_t *__restrict__ node_key, uint32_t *__restrict__ node_start,
                                    const uint32_t *err) {
  if (*err || blockIdx.x || threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  const uint32_t lt = lanemask_lt();
  uint64_t j = 0;
  for (uint32_t kk = 0; kk < nk; kk++) {
    const uint32_t k = k_lo + kk, sh = tau - k;
    if (lane == 0) level_node_ptr[k] = j;
    uint32_t c = 0;
    for (uint32_t q0 = 0; q0 < (1u << k); q0 += 32) {
      const uint32_t q = q0 + lane;
      uint32_t a = 0, b = 0;
      if (q < (1u << k)) {
        a = Cseg[q << sh];
        b = Cseg[(q + 1) << sh];
      }
      const uint32_t bm = __ballot_sync(FULL, b > a);
      if (b > a) {
        node_key[j + __popc(bm & lt)] = q;
        node_start[j + __popc(bm & lt)] = a;
      }
      j += __popc(bm);
      c += __popc(bm);
    }
    if (lane == 0) {
      ncount[k] = c;
      if (k + 1 == L) level_node_ptr[L] = j;
    }
  }
}

// Level CSR bases: level_node_ptr[lev] for the group's levels (runs after pass 2).
static __global__ void k_level_ptr(const uint32_t *__restrict__ ncount, uint32_t l0, uint32_t k_lo, uint32_t nk, uint32_t L,
                            uint64_t *__restrict__ level_node_ptr, const uint32_t *err) {
  if (*err) return;
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (uint32_t kk = 0; kk < nk; kk++) {
    const uint32_t lev = l0 + k_lo + kk;
    uint64_t base = 0;
    for (uint32_t l = 0; l < lev; l++) base += ncount[l];
    level_node_ptr[lev] = base;
    if (lev + 1 == L) level_node_ptr[L] = base + ncount[lev];
  }
}

// pass 3: rowoff[k][r] = exclusive prefix within the level (in place over rowcnt).
static __global__ void __launch_bounds__(1024) k_scan_rows_3(uint32_t *__restrict__ rowcnt, uint64_t rstride,
                                                     const uint32_t *__restrict__ counts,
                                                     const uint32_t *__restrict__ bsum, uint32_t bstride,
                                                     const uint32_t *err) {
  __shared__ uint32_t shm[33];
  if (*err) return;
  const uint32_t nr = counts[1];
  const uint64_t b0 = (uint64_t)blockIdx.x * SCAN_BLK;
  if (b0 >= nr) return;
  uint32_t *rc = rowcnt + (uint64_t)blockIdx.y * rstride;
  uint32_t carry = bsum[(uint64_t)blockIdx.y * bstride + blockIdx.x];
  for (uint64_t base = b0; base < b0 + SCAN_BLK && base < nr; base += blockDim.x) {
    const uint64_t r = base + threadIdx.x;
    const bool in = r < b0 + SCAN_BLK && r < nr;
    const uint32_t v = in ? rc[r] : 0u;
    uint32_t tot;
    const uint32_t ex = block_exscan(v, shm, &tot);
    if (in) rc[r] = carry + ex;
    carry += tot;
    __syncthreads();
  }
}

static __global__ void k_row_nodes_emit(const uint32_t *__restrict__ Cseg, const uint32_t *__restrict__ counts, uint32_t tau,
                                 uint32_t l0, uint32_t k_lo, uint32_t nk, uint64_t rstride,
                                 const uint32_t *__restrict__ rowoff, const uint64_t *__restrict__ level_node_ptr,
                                 const uint32_t *__restrict__ row_key, const uint32_t *__restrict__ row_start,
                                 uint32_t *__restrict__ node_key, uint32_t *__restrict__ node_start,
                                 const uint32_t *err) {
  // one warp per (row, level); node j = level base + row offset + rank among the row's non-empty q
  if (*err) return;
  const uint32_t nr = counts[1], ndig = 1u << tau;
  const int lane = threadIdx.x & 31;
  const uint32_t lt = lanemask_lt();
  const uint64_t items = (uint64_t)nr * nk;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t it = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < items; it += nwarps) {
    const uint32_t r = (uint32_t)(it % nr), kk = (uint32_t)(it / nr);
    const uint32_t k = k_lo + kk, sh = tau - k;
    const uint32_t *row = Cseg + (uint64_t)r * (ndig + 1);
    uint64_t j = level_node_ptr[l0 + k] + rowoff[(uint64_t)kk * rstride + r];
    const uint32_t P = row_key[r], rs = row_start[r];
    for (uint32_t q0 = 0; q0 < (1u << k); q0 += 32) {
      const uint32_t q = q0 + lane;
      uint32_t a = 0, b = 0;
      if (q < (1u << k)) {
        a = row[q << sh];
        b = row[(q + 1) << sh];
      }
      const uint32_t bm = __ballot_sync(FULL, b > a);
      if (b > a) {
        const uint64_t jj = j + __popc(bm & lt);
        node_key[jj] = (P << k) | q;
        node_start[jj] = rs + a;
      }
      j += __popc(bm);
    }
  }
}

// Occupancy of the 2^tau digits of a row as 8 words (bit i of word j = digit
// 32j + i), reduced level by level: a level-(k-1) prefix is non-empty iff one
// of its two children is.  Returns the occupancy popcount per level in cnt[k].
__device__ __forceinline__ uint32_t gather_pairs(uint32_t w) {  // OR bit pairs, pack 16 bits
  w = (w | (w >> 1)) & 0x55555555u;
  w = (w | (w >> 1)) & 0x33333333u;
  w = (w | (w >> 2)) & 0x0f0f0f0fu;
  w = (w | (w >> 4)) & 0x00ff00ffu;
  w = (w | (w >> 8)) & 0x0000ffffu;
  return w;
}

// Local mode (rows small enough for one tile): per-row node counts straight
// from the row's keys.  One warp per row; a row larger than TW sets err |= 2
// (the host then rebuilds with chain mode).
template <typename KeyT>
__global__ void __launch_bounds__(256) k_local_count(const KeyT *__restrict__ keys, uint32_t pbits, uint32_t tau,
                                                    uint32_t nk, const uint32_t *__restrict__ chain_begin,
                                                    const uint32_t *__restrict__ chain_end,
                                                    const uint32_t *__restrict__ counts, uint64_t rstride,
                                                    uint32_t *__restrict__ rowcnt, uint32_t *err) {
  __shared__ uint32_t h[8][NDIG];
  if (ld_relaxed(err)) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t nr = counts[1], ndig = 1u << tau;
  for (uint32_t r = blockIdx.x * 8 + warp; r < nr; r += gridDim.x * 8) {
    const uint32_t beg = chain_begin[r], end = chain_end[r];
    if (end - beg > (uint32_t)TW) {
      if (lane == 0) atomicOr(err, 2u);
      return;
    }
#pragma unroll
    for (int i = 0; i < NDIG / 32; i++) h[warp][lane + 32 * i] = 0;
    __syncwarp();
    for (uint32_t i = beg + lane; i < end; i += 32) h[warp][((uint32_t)keys[i] >> pbits) & (ndig - 1u)] = 1u;
    __syncwarp();
    uint32_t w[NDIG / 32];
#pragma unroll
    for (int j = 0; j < NDIG / 32; j++) w[j] = __ballot_sync(FULL, h[warp][32 * j + lane] != 0);
    // level k = tau: w holds 2^tau bits; reduce to k = tau-1, ..., 1
    uint32_t nbits = ndig;
    for (int k = (int)tau; k >= 1; k--) {
      if ((uint32_t)k <= nk && lane == 0) {
        uint32_t c = 0;
#pragma unroll
        for (int j = 0; j < NDIG / 32; j++) c += (32u * j < nbits) ? __popc(w[j]) : 0u;
        rowcnt[(uint64_t)(k - 1) * rstride + r] = c;
      }
      // halve: word j' = pairs of words 2j', 2j'+1
      uint32_t nw[NDIG / 32];
#pragma unroll
      for (int j = 0; j < NDIG / 64; j++) nw[j] = gather_pairs(w[2 * j]) | (gather_pairs(w[2 * j + 1]) << 16);
#pragma unroll
      for (int j = NDIG / 64; j < NDIG / 32; j++) nw[j] = 0;
      if (nbits <= 32) nw[0] = gather_pairs(w[0]);
#pragma unroll
      for (int j = 0; j < NDIG / 32; j++) w[j] = nw[j];
      nbits >>= 1;
    }
    __syncwarp();
  }
}

}  // namespace wtb
