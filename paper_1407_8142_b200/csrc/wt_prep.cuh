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
__global__ void k_chains_root(uint64_t n, uint64_t CH, uint32_t K, uint32_t *__restrict__ chain_begin,
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

__global__ void __launch_bounds__(1024) k_chains_from_nodes(
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
// ---------------------------------------------------------------------------
template <typename T, bool VALIDATE>
__global__ void __launch_bounds__(512) k_chain_hist(const T *__restrict__ keys, uint64_t sigma, uint32_t shift,
                                                   uint32_t ndig, const uint32_t *__restrict__ chain_begin,
                                                   const uint32_t *__restrict__ chain_end,
                                                   const uint32_t *__restrict__ counts, uint32_t stride,
                                                   uint32_t *__restrict__ histT, uint32_t *err) {
  __shared__ uint32_t h[NDIG * 4];  // 4 sub-histograms spread same-bin contention
  if (!VALIDATE && ld_relaxed(err)) return;
  const uint32_t nchains = counts[0];
  bool bad = false;
  for (uint32_t c = blockIdx.x; c < nchains; c += gridDim.x) {
  for (uint32_t i = threadIdx.x; i < 4 * NDIG; i += blockDim.x) h[i] = 0;
  __syncthreads();
  uint32_t *hs = h + (threadIdx.x & 3) * NDIG;
  const uint32_t dmask = ndig - 1u;
  auto add = [&](uint32_t v) {
    if (VALIDATE && (uint64_t)v >= sigma) {
      bad = true;
      return;
    }
    atomicAdd(&hs[(v >> shift) & dmask], 1u);
  };
  const uint32_t beg = chain_begin[c], end = chain_end[c];
  constexpr int PER = 16 / sizeof(T);
  const uintptr_t sb = reinterpret_cast<uintptr_t>(keys + beg);
  const uintptr_t ab = sb & ~(uintptr_t)15;
  const int head = (int)((sb - ab) / sizeof(T));
  const uint4 *V = reinterpret_cast<const uint4 *>(ab);
  const uint32_t len = end - beg;
  const uint32_t nv = (head + len + PER - 1) / PER;
  for (uint32_t i = threadIdx.x; i < nv; i += blockDim.x) {
    const uint4 q = __ldcs(V + i);
    const T *e = reinterpret_cast<const T *>(&q);
#pragma unroll
    for (int k = 0; k < PER; k++) {
      const int pos = (int)(i * PER + k) - head;
      if (pos >= 0 && pos < (int)len) add((uint32_t)e[k]);
    }
  }
  __syncthreads();
  for (uint32_t d = threadIdx.x; d < ndig; d += blockDim.x)
    histT[(uint64_t)d * stride + c] = h[d] + h[NDIG + d] + h[2 * NDIG + d] + h[3 * NDIG + d];
  __syncthreads();
  }
  if (VALIDATE && __any_sync(FULL, bad) && (threadIdx.x & 31) == 0) atomicOr(err, 1u);
}

// E[d][c] = sum_{c' < c} histT[d][c'] (in place), E[d][nchains] = total; one CTA per digit.
__global__ void __launch_bounds__(1024) k_chain_scan(uint32_t *__restrict__ histT, uint32_t stride,
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

// Cseg[r][0..ndig] = exclusive scan over d of the row's digit totals
// E[d][row_first[r+1]] - E[d][row_first[r]].  One warp per row.
__global__ void k_row_scan(const uint32_t *__restrict__ E, uint32_t stride, const uint32_t *__restrict__ row_first,
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
// A4: non-empty nodes of levels l0+k (k = k_lo .. k_hi) from the rows' Cseg.
// Node (P << k | q) is non-empty iff Cseg[r][(q+1) << (tau-k)] > Cseg[r][q << (tau-k)]
// (Fig. 1 l.18-20).  One CTA per level; rows in order, so keys ascend.
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool node_nonempty(const uint32_t *Cs, uint32_t ndig, uint32_t r, uint32_t q,
                                              uint32_t sh) {
  const uint32_t *row = Cs + (uint64_t)r * (ndig + 1);
  return row[(q + 1) << sh] > row[q << sh];
}

__global__ void __launch_bounds__(1024) k_nodes_count(const uint32_t *__restrict__ Cseg,
                                                     const uint32_t *__restrict__ counts, uint32_t tau, uint32_t l0,
                                                     uint32_t k_lo, uint32_t *__restrict__ ncount,
                                                     const uint32_t *err) {
  __shared__ uint32_t shm[33];
  if (*err) return;
  const uint32_t k = k_lo + blockIdx.x;
  const uint32_t nr = counts[1], nq = 1u << k, sh = tau - k, ndig = 1u << tau;
  const uint64_t tot_items = (uint64_t)nr * nq;
  uint32_t c = 0;
  for (uint64_t f = threadIdx.x; f < tot_items; f += blockDim.x)
    c += node_nonempty(Cseg, ndig, (uint32_t)(f >> k), (uint32_t)(f & (nq - 1)), sh);
  uint32_t tot;
  block_exscan(c, shm, &tot);
  if (threadIdx.x == 0) ncount[l0 + k] = tot;
}

__global__ void __launch_bounds__(1024) k_nodes_emit(const uint32_t *__restrict__ Cseg,
                                                    const uint32_t *__restrict__ counts, uint32_t tau, uint32_t l0,
                                                    uint32_t k_lo, uint32_t L, const uint32_t *__restrict__ row_key,
                                                    const uint32_t *__restrict__ row_start,
                                                    const uint32_t *__restrict__ ncount,
                                                    uint64_t *__restrict__ level_node_ptr,
                                                    uint32_t *__restrict__ node_key,
                                                    uint32_t *__restrict__ node_start, const uint32_t *err) {
  __shared__ uint32_t shm[33];
  if (*err) return;
  const uint32_t k = k_lo + blockIdx.x;
  const uint32_t lev = l0 + k;
  uint64_t base = 0;
  for (uint32_t l = 0; l < lev; l++) base += ncount[l];
  if (threadIdx.x == 0) {
    level_node_ptr[lev] = base;
    if (lev + 1 == L) level_node_ptr[L] = base + ncount[lev];
  }
  const uint32_t nr = counts[1], nq = 1u << k, sh = tau - k, ndig = 1u << tau;
  const uint64_t tot_items = (uint64_t)nr * nq;
  uint64_t carry = 0;
  for (uint64_t f0 = 0; f0 < tot_items; f0 += blockDim.x) {
    const uint64_t f = f0 + threadIdx.x;
    const uint32_t r = (uint32_t)(f >> k), q = (uint32_t)(f & (nq - 1));
    const bool ne = f < tot_items && node_nonempty(Cseg, ndig, r, q, sh);
    uint32_t tot;
    const uint32_t off = block_exscan(ne ? 1u : 0u, shm, &tot);
    if (ne) {
      const uint64_t j = base + carry + off;
      node_key[j] = (row_key[r] << k) | q;
      node_start[j] = row_start[r] + Cseg[(uint64_t)r * (ndig + 1) + (q << sh)];
    }
    carry += tot;
    __syncthreads();
  }
}

}  // namespace wtb
