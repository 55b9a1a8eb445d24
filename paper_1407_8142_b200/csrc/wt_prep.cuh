// wt_prep.cuh -- A1 (validation, histograms), A4 (node table) and the
// bookkeeping that lets the group passes run (chains, claim order).
//
// Terms:
//  * group g: levels l0 .. l0+tau-1 built by one k_group pass; digit = the
//    tau level bits of a key, taken from its top.
//  * row: a level-l0 node ("segment") of group g, with its digit histogram
//    scanned into Cseg[row][0..2^tau]: the start of node (P:q) at level l0+k
//    is row_start[row] + Cseg[row][q << (tau-k)]  (Fig. 2 l.13 / PAPER.md
//    468-475: a level-l node is the set of symbols sharing the top l bits,
//    laid out in prefix order).
//  * chain: a run of consecutive warp tiles whose lookback is sequential.
//    Group 0 splits S into K chunks (chains) whose starting counts come from
//    the chunked A1 histogram; group g >= 1 uses one chain per row.
#pragma once
#include "wt_common.cuh"

namespace wtb {

// ---------------------------------------------------------------------------
// A1: validate S[i] < sigma and histogram the top tau0 bits, one CTA per
// chunk of CH symbols.  partial[c][d] = count of digit d in chunk c.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(1024) k_hist(const T *__restrict__ S, uint64_t n, uint64_t sigma,
                                              uint32_t shift, uint32_t ndig, uint64_t CH,
                                              uint32_t *__restrict__ partial, uint32_t *err) {
  __shared__ uint32_t h[NDIG * 4];  // 4 sub-histograms to spread contention
  for (uint32_t i = threadIdx.x; i < 4 * NDIG; i += blockDim.x) h[i] = 0;
  __syncthreads();
  uint32_t *hs = h + (threadIdx.x & 3) * NDIG;
  bool bad = false;
  auto add = [&](uint32_t v) {
    if ((uint64_t)v >= sigma) {
      bad = true;
      return;
    }
    atomicAdd(&hs[v >> shift], 1u);
  };
  const uint64_t lo = (uint64_t)blockIdx.x * CH;
  const uint64_t hi = lo + CH < n ? lo + CH : n;
  const T *base = S + lo;
  const uint64_t cnt = hi > lo ? hi - lo : 0;
  constexpr int PER = 16 / sizeof(T);
  if ((reinterpret_cast<uintptr_t>(base) & 15) == 0) {
    const uint4 *V = reinterpret_cast<const uint4 *>(base);
    const uint64_t nv = cnt / PER;
    uint64_t i = threadIdx.x;
    for (; i + 3 * blockDim.x < nv; i += 4 * blockDim.x) {
      uint4 q[4];
#pragma unroll
      for (int u = 0; u < 4; u++) q[u] = __ldcs(V + i + u * blockDim.x);
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const T *e = reinterpret_cast<const T *>(&q[u]);
#pragma unroll
        for (int k = 0; k < PER; k++) add((uint32_t)e[k]);
      }
    }
    for (; i < nv; i += blockDim.x) {
      const uint4 q = __ldcs(V + i);
      const T *e = reinterpret_cast<const T *>(&q);
#pragma unroll
      for (int k = 0; k < PER; k++) add((uint32_t)e[k]);
    }
    for (uint64_t j = nv * PER + threadIdx.x; j < cnt; j += blockDim.x) add((uint32_t)base[j]);
  } else {
    for (uint64_t j = threadIdx.x; j < cnt; j += blockDim.x) add((uint32_t)base[j]);
  }
  if (__any_sync(FULL, bad) && (threadIdx.x & 31) == 0) atomicOr(err, 1u);
  __syncthreads();
  for (uint32_t d = threadIdx.x; d < ndig; d += blockDim.x)
    partial[(uint64_t)blockIdx.x * ndig + d] = h[d] + h[NDIG + d] + h[2 * NDIG + d] + h[3 * NDIG + d];
}

// Group 0 chains = A1 chunks.  One CTA of NDIG threads:
//   chain_prefix[c][d] = sum_{c' < c} partial[c'][d]   (counts ahead of chunk c)
//   Cseg row 0 = exclusive scan over d of the global digit histogram
// plus the chain geometry arrays.
__global__ void __launch_bounds__(NDIG) k_chunk_scan(const uint32_t *__restrict__ partial, uint32_t K,
                                                    uint32_t ndig, uint64_t n, uint64_t CH,
                                                    uint32_t *__restrict__ chain_prefix,
                                                    uint32_t *__restrict__ Cseg, uint32_t *__restrict__ row_start,
                                                    uint32_t *__restrict__ chain_begin,
                                                    uint32_t *__restrict__ chain_end,
                                                    uint32_t *__restrict__ chain_key,
                                                    uint32_t *__restrict__ chain_row, uint32_t *nchains,
                                                    const uint32_t *err) {
  __shared__ uint32_t shm[33];
  if (*err) return;
  const uint32_t d = threadIdx.x;
  uint32_t run = 0;
  if (d < ndig) {
    for (uint32_t c = 0; c < K; c++) {
      chain_prefix[(uint64_t)c * ndig + d] = run;
      run += partial[(uint64_t)c * ndig + d];
    }
  }
  uint32_t tot;
  const uint32_t ex = block_exscan(d < ndig ? run : 0u, shm, &tot);
  if (d < ndig) Cseg[d] = ex;
  if (d == 0) {
    Cseg[ndig] = tot;
    row_start[0] = 0;
    *nchains = K;
  }
  for (uint32_t c = d; c < K; c += blockDim.x) {
    const uint64_t b = (uint64_t)c * CH, e = b + CH < n ? b + CH : n;
    chain_begin[c] = (uint32_t)b;
    chain_end[c] = (uint32_t)e;
    chain_key[c] = 0;
    chain_row[c] = 0;
  }
}

// Group g >= 1 chains = rows = the non-empty nodes of level l0 (their CSR
// slice of the node table).  Grid-stride over rows.
__global__ void k_chains_from_nodes(const uint64_t *__restrict__ level_node_ptr,
                                    const uint32_t *__restrict__ ncount, uint32_t l0,
                                    const uint32_t *__restrict__ node_key,
                                    const uint32_t *__restrict__ node_start, uint64_t n,
                                    uint32_t *__restrict__ chain_begin, uint32_t *__restrict__ chain_end,
                                    uint32_t *__restrict__ chain_key, uint32_t *__restrict__ chain_row,
                                    uint32_t *__restrict__ row_start, uint32_t *nchains, const uint32_t *err) {
  if (*err) return;
  // level l0's nodes were emitted by the previous group: base and count are final
  const uint64_t p0 = level_node_ptr[l0];
  const uint32_t nr = ncount[l0];
  if (blockIdx.x == 0 && threadIdx.x == 0) *nchains = nr;
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < nr; r += gridDim.x * blockDim.x) {
    const uint32_t b = node_start[p0 + r];
    chain_begin[r] = b;
    chain_end[r] = (r + 1 < nr) ? node_start[p0 + r + 1] : (uint32_t)n;
    chain_key[r] = node_key[p0 + r];
    chain_row[r] = r;
    row_start[r] = b;
  }
}

// ---------------------------------------------------------------------------
// Claim order.  Tiles are numbered chain-major for the lookback state
// (tile_base[c] + j) but CLAIMED round-robin across chains: round r holds
// tile j = r of every chain with more than r tiles, chains ordered by tile
// count (descending).  Tile (c, j-1) is always claimed before (c, j), so the
// lookback makes progress, and concurrently running tiles belong to many
// independent chains, so a lookback rarely waits.
// One CTA of 1024 threads.  hnt/tie must be zeroed (size >= maxtiles + 2).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_claims(const uint32_t *__restrict__ chain_begin,
                                                const uint32_t *__restrict__ chain_end,
                                                const uint32_t *nchains_p, uint32_t *__restrict__ tile_base,
                                                uint32_t *__restrict__ hnt, uint32_t *__restrict__ cum,
                                                uint32_t *__restrict__ tie, uint2 *__restrict__ claim,
                                                uint32_t *total_tiles, const uint32_t *err) {
  __shared__ uint32_t shm[33];
  __shared__ uint32_t s_maxnt;
  if (*err) return;
  const uint32_t nc = *nchains_p;
  if (threadIdx.x == 0) s_maxnt = 0;
  __syncthreads();
  // 1. tile counts, chain-major bases, histogram of tile counts
  uint32_t carry = 0;
  for (uint32_t b0 = 0; b0 < nc; b0 += blockDim.x) {
    const uint32_t c = b0 + threadIdx.x;
    uint32_t nt = 0;
    if (c < nc) nt = (chain_end[c] - chain_begin[c] + TW - 1) / TW;
    uint32_t tot;
    const uint32_t off = block_exscan(nt, shm, &tot);
    if (c < nc) {
      tile_base[c] = carry + off;
      if (nt) {
        atomicAdd(&hnt[nt], 1u);
        atomicMax(&s_maxnt, nt);
      }
    }
    carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total_tiles = carry;
  __syncthreads();
  const uint32_t maxnt = s_maxnt;
  // 2. cnt_r = #{c : nt_c > r} (suffix sums of hnt), cum[r] = sum_{r' < r} cnt_r'.
  //    Process r descending in blocks; keep cnt in cum[] first, then scan.
  uint32_t suffix = 0;
  for (int64_t top = (int64_t)maxnt; top >= 1; top -= blockDim.x) {
    // v = hnt[top - tid] for indices top, top-1, ...
    const int64_t v_idx = top - (int64_t)threadIdx.x;
    const uint32_t v = v_idx >= 1 ? hnt[v_idx] : 0u;
    uint32_t tot;
    const uint32_t ex = block_exscan(v, shm, &tot);  // sum of hnt over (v_idx, top]
    // cnt_{v_idx - 1} = #{nt > v_idx - 1} = #{nt >= v_idx} = suffix + ex + v
    if (v_idx >= 1) cum[v_idx - 1] = suffix + ex + v;
    suffix += tot;
    __syncthreads();
  }
  __syncthreads();
  // exclusive scan of cnt over r = 0..maxnt-1 into cum (in place), cum[maxnt] = total
  uint32_t run = 0;
  for (uint32_t b0 = 0; b0 < maxnt; b0 += blockDim.x) {
    const uint32_t r = b0 + threadIdx.x;
    const uint32_t v = r < maxnt ? cum[r] : 0u;
    uint32_t tot;
    const uint32_t ex = block_exscan(v, shm, &tot);
    if (r < maxnt) cum[r] = run + ex;
    run += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) cum[maxnt] = run;
  // cnt_r again needed for the sort position: #{c : nt_c > nt} = cum[nt+1] - cum[nt] for rounds...
  // position of chain c among chains sorted by nt descending:
  //   #{c' : nt_c' > nt_c} + tie index.  #{nt_c' > x} = cnt_x = cum[x+1] - cum[x].
  __syncthreads();
  for (uint32_t c = threadIdx.x; c < nc; c += blockDim.x) {
    const uint32_t nt = (chain_end[c] - chain_begin[c] + TW - 1) / TW;
    if (!nt) continue;
    const uint32_t greater = (nt < maxnt) ? (cum[nt + 1] - cum[nt]) : 0u;
    const uint32_t k = greater + atomicAdd(&tie[nt], 1u);
    for (uint32_t j = 0; j < nt; j++) claim[cum[j] + k] = make_uint2(c, j);
  }
}

// ---------------------------------------------------------------------------
// Group g >= 1: per-row digit histogram of the group's input keys (A1 for the
// deeper levels), then per-row exclusive scan -> Cseg.
// ---------------------------------------------------------------------------
template <typename KeyT>
__global__ void __launch_bounds__(256) k_seg_hist(const KeyT *__restrict__ keys, uint32_t dshift, uint32_t ndig,
                                                 const uint2 *__restrict__ claim, const uint32_t *total_tiles,
                                                 const uint32_t *__restrict__ chain_begin,
                                                 const uint32_t *__restrict__ chain_end,
                                                 const uint32_t *__restrict__ chain_row,
                                                 uint32_t *__restrict__ seghist, const uint32_t *err) {
  __shared__ uint32_t h[8][NDIG];
  if (*err) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t T = *total_tiles;
  for (uint32_t t = blockIdx.x * 8 + warp; t < T; t += gridDim.x * 8) {
    for (uint32_t d = lane; d < ndig; d += 32) h[warp][d] = 0;
    __syncwarp();
    const uint2 cj = claim[t];
    const uint32_t start = chain_begin[cj.x] + cj.y * TW;
    const uint32_t end = min(start + (uint32_t)TW, chain_end[cj.x]);
    for (uint32_t i = start + lane; i < end; i += 32)
      atomicAdd(&h[warp][((uint32_t)keys[i] >> dshift) & (ndig - 1u)], 1u);
    __syncwarp();
    uint32_t *row = seghist + (uint64_t)chain_row[cj.x] * (ndig + 1);
    for (uint32_t d = lane; d < ndig; d += 32)
      if (h[warp][d]) atomicAdd(&row[d], h[warp][d]);
    __syncwarp();
  }
}

// Cseg[r][0..ndig] = exclusive scan of seghist[r][0..ndig) (in place); one warp per row.
__global__ void k_seg_scan(uint32_t *__restrict__ seghist, const uint32_t *nrows_p, uint32_t ndig,
                           const uint32_t *err) {
  if (*err) return;
  const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= *nrows_p) return;
  uint32_t *row = seghist + (uint64_t)w * (ndig + 1);
  const uint32_t per = (ndig + 31) >> 5;
  uint32_t v[8], s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) {
    const uint32_t d = lane * per + i;
    v[i] = (i < (int)per && d < ndig) ? row[d] : 0u;
    s += v[i];
  }
  const uint32_t incl = warp_incl_scan(s, lane);
  uint32_t run = incl - s;
#pragma unroll
  for (int i = 0; i < 8; i++) {
    const uint32_t d = lane * per + i;
    if (i < (int)per && d < ndig) row[d] = run;
    run += v[i];
  }
  if (lane == 31) row[ndig] = incl;
}

// ---------------------------------------------------------------------------
// A4: non-empty nodes of the group's levels l0+k (k = k_lo .. k_hi), from the
// rows' Cseg.  Node (P << k | q) is non-empty iff its count
// Cseg[r][(q+1) << (tau-k)] - Cseg[r][q << (tau-k)] > 0 (Fig. 1 l.18-20).
// One CTA per level; rows visited in order, so keys ascend.
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool node_nonempty(const uint32_t *Cs, uint32_t ndig, uint32_t r, uint32_t q,
                                              uint32_t sh) {
  const uint32_t *row = Cs + (uint64_t)r * (ndig + 1);
  return row[(q + 1) << sh] > row[q << sh];
}

__global__ void __launch_bounds__(1024) k_nodes_count(const uint32_t *__restrict__ Cseg, const uint32_t *nrows_p,
                                                     uint32_t tau, uint32_t l0, uint32_t k_lo,
                                                     uint32_t *__restrict__ ncount, const uint32_t *err) {
  __shared__ uint32_t shm[33];
  if (*err) return;
  const uint32_t k = k_lo + blockIdx.x;
  const uint32_t nr = *nrows_p, nq = 1u << k, sh = tau - k, ndig = 1u << tau;
  const uint64_t tot_items = (uint64_t)nr * nq;
  uint32_t c = 0;
  for (uint64_t f = threadIdx.x; f < tot_items; f += blockDim.x)
    c += node_nonempty(Cseg, ndig, (uint32_t)(f >> k), (uint32_t)(f & (nq - 1)), sh);
  uint32_t tot;
  block_exscan(c, shm, &tot);
  if (threadIdx.x == 0) ncount[l0 + k] = tot;
}

__global__ void __launch_bounds__(1024) k_nodes_emit(const uint32_t *__restrict__ Cseg, const uint32_t *nrows_p,
                                                    uint32_t tau, uint32_t l0, uint32_t k_lo, uint32_t L,
                                                    const uint32_t *__restrict__ chain_key,
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
  const uint32_t nr = *nrows_p, nq = 1u << k, sh = tau - k, ndig = 1u << tau;
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
      node_key[j] = (chain_key[r] << k) | q;
      node_start[j] = row_start[r] + Cseg[(uint64_t)r * (ndig + 1) + (q << sh)];
    }
    carry += tot;
    __syncthreads();
  }
}

}  // namespace wtb
