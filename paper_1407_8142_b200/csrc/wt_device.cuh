// wt_device.cuh -- sm_100a kernels of the levelwise wavelet-tree build.
//
// Citations are PAPER.md line numbers (arXiv 1407.8142) and SURVEY.md §8 rows.
// Pipeline of one wt_build:
//   k_hist        A1  validate S, per-CTA symbol histogram of the top Lh bits
//   k_hist_reduce A1  sum the per-CTA partials
//   k_scan_hist   A1  exclusive scan -> Hx; C_l(p) = Hx[p << (Lh - l)] is the
//                     start of node p at level l
//   k_node_count/ k_node_emit   A4  non-empty nodes per level (Fig. 1 l.18-20)
//   k_segments    A4  tiles of the level-l0 nodes for groups g >= 1
//   k_group       A2+A3+A5+A6+A7  tau levels per HBM pass (the hot kernel)
//   k_rank_local / k_rank_super  A7  two-level rank directory
//   k_access / k_rank_query      A8  batched queries
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace wtb {

constexpr uint32_t FULL = 0xffffffffu;
constexpr int TW = 4096;               // elements per warp tile
constexpr int NCH = TW / 32;           // 32-element chunks per tile
constexpr int TAU_MAX = 8;             // levels fused per HBM pass
constexpr int NDIG = 1 << TAU_MAX;     // digit values per pass
constexpr uint32_t FLAG_AGG = 1u << 30;  // lookback: tile aggregate published
constexpr uint32_t FLAG_INC = 2u << 30;  // lookback: inclusive prefix published
constexpr uint32_t VAL_MASK = (1u << 30) - 1;

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ uint32_t ld_volatile(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_volatile(uint32_t *p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Warp-cooperative exclusive scan of a[0..cnt) into out[0..cnt], out[cnt] = total.
// a and out live in shared memory; they may alias.
__device__ __forceinline__ void warp_exscan(const uint32_t *a, int cnt, uint32_t *out, int lane) {
  const int per = (cnt + 31) >> 5;
  const int lo = lane * per;
  const int hi = min(lo + per, cnt);
  uint32_t s = 0;
  for (int i = lo; i < hi; i++) s += a[i];
  uint32_t incl = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t v = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += v;
  }
  uint32_t run = incl - s;
  uint32_t total = __shfl_sync(FULL, incl, 31);
  __syncwarp();
  for (int i = lo; i < hi; i++) {
    uint32_t v = a[i];
    out[i] = run;
    run += v;
  }
  if (lane == 0) out[cnt] = total;
  __syncwarp();
}

// Bits [base, base+64) of a little-endian bit array stored as nw u32 words;
// bits outside [0, 32*nw) read as 0.  base may be negative (> -64).
__device__ __forceinline__ uint64_t extract64(const uint32_t *w, int base, int nw) {
  int b = base < 0 ? 0 : base;
  int wi = b >> 5, sh = b & 31;
  uint32_t x0 = wi < nw ? w[wi] : 0u;
  uint32_t x1 = wi + 1 < nw ? w[wi + 1] : 0u;
  uint32_t x2 = wi + 2 < nw ? w[wi + 2] : 0u;
  uint64_t v = (((uint64_t)x1 << 32) | x0) >> sh;
  if (sh) v |= (uint64_t)x2 << (64 - sh);
  if (base < 0) v <<= (-base);
  return v;
}

// ---------------------------------------------------------------------------
// A1: validation + histogram of the top Lh bits of every symbol.
// PAIR16: bins are u16 pairs packed in u32 words (Lh = 16 does not fit u32
// bins in shared memory); a wrap of a 16-bit half is detected from the
// returned old word and compensated in `adj` (global, exact).
// ---------------------------------------------------------------------------
template <typename T, bool PAIR16>
__global__ void __launch_bounds__(1024) k_hist(const T *__restrict__ S, uint64_t n, uint64_t sigma,
                                              uint32_t shift, uint32_t nbins,
                                              uint32_t *__restrict__ partial,
                                              uint32_t *__restrict__ adj, uint32_t *err) {
  extern __shared__ uint32_t h[];
  const uint32_t nw = PAIR16 ? nbins / 2 : nbins;
  for (uint32_t i = threadIdx.x; i < nw; i += blockDim.x) h[i] = 0;
  __syncthreads();
  bool bad = false;
  auto add = [&](uint32_t v) {
    if ((uint64_t)v >= sigma) { bad = true; return; }
    uint32_t b = v >> shift;
    if (!PAIR16) {
      atomicAdd(&h[b], 1u);
    } else {
      uint32_t hi = b & 1u;
      uint32_t old = atomicAdd(&h[b >> 1], hi ? 0x10000u : 1u);
      if (!hi) {
        if ((old & 0xffffu) == 0xffffu) {       // low half wrapped, carried into high
          atomicAdd(&adj[b], 0x10000u);
          atomicAdd(&adj[b | 1u], 0xffffffffu);  // -1: the spurious carry
          if ((old >> 16) == 0xffffu) atomicAdd(&adj[b | 1u], 0x10000u);  // carry wrapped high
        }
      } else if ((old >> 16) == 0xffffu) {
        atomicAdd(&adj[b], 0x10000u);
      }
    }
  };
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
  constexpr int PER = 16 / sizeof(T);
  if ((reinterpret_cast<uintptr_t>(S) & 15) == 0) {
    const uint4 *V = reinterpret_cast<const uint4 *>(S);
    const uint64_t nv = n / PER;
    uint64_t i = tid;
    for (; i + 3 * nth < nv; i += 4 * nth) {
      uint4 q[4];
#pragma unroll
      for (int u = 0; u < 4; u++) q[u] = __ldcs(V + i + u * nth);
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const T *e = reinterpret_cast<const T *>(&q[u]);
#pragma unroll
        for (int k = 0; k < PER; k++) add((uint32_t)e[k]);
      }
    }
    for (; i < nv; i += nth) {
      uint4 q = __ldcs(V + i);
      const T *e = reinterpret_cast<const T *>(&q);
#pragma unroll
      for (int k = 0; k < PER; k++) add((uint32_t)e[k]);
    }
    for (uint64_t j = nv * PER + tid; j < n; j += nth) add((uint32_t)S[j]);
  } else {
    for (uint64_t j = tid; j < n; j += nth) add((uint32_t)S[j]);
  }
  if (__any_sync(FULL, bad) && (threadIdx.x & 31) == 0) atomicOr(err, 1u);
  __syncthreads();
  uint32_t *out = partial + (uint64_t)blockIdx.x * nbins;
  if (!PAIR16) {
    for (uint32_t i = threadIdx.x; i < nbins; i += blockDim.x) out[i] = h[i];
  } else {
    for (uint32_t i = threadIdx.x; i < nw; i += blockDim.x) {
      uint32_t w = h[i];
      out[2 * i] = w & 0xffffu;
      out[2 * i + 1] = w >> 16;
    }
  }
}

// hist[b] = sum over CTAs of partial[c][b] + adj[b]
__global__ void k_hist_reduce(const uint32_t *__restrict__ partial, uint32_t nparts, uint32_t nbins,
                              const uint32_t *__restrict__ adj, uint32_t *__restrict__ hist) {
  uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nbins) return;
  uint32_t s = adj[b];
  for (uint32_t c = 0; c < nparts; c++) s += partial[(uint64_t)c * nbins + b];
  hist[b] = s;
}

// Hx[b] = sum_{b' < b} hist[b'] for b in [0, nbins]; one CTA of 1024 threads.
__global__ void __launch_bounds__(1024) k_scan_hist(const uint32_t *__restrict__ hist, uint32_t nbins,
                                                   uint32_t *__restrict__ Hx, const uint32_t *err) {
  __shared__ uint32_t warp_tot[32];
  if (*err) return;
  const uint32_t per = (nbins + blockDim.x - 1) / blockDim.x;
  const uint32_t lo = min(threadIdx.x * per, nbins), hi = min(lo + per, nbins);
  uint32_t s = 0;
  for (uint32_t i = lo; i < hi; i++) s += hist[i];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t v = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0u;
    uint32_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t v = __shfl_up_sync(FULL, wi, o);
      if (lane >= o) wi += v;
    }
    warp_tot[lane] = wi - w;
  }
  __syncthreads();
  uint32_t run = warp_tot[warp] + incl - s;
  for (uint32_t i = lo; i < hi; i++) {
    Hx[i] = run;
    run += hist[i];
  }
  if (threadIdx.x == blockDim.x - 1) Hx[nbins] = warp_tot[warp] + incl;
}

// Block-wide exclusive scan helper (blockDim.x == 1024): returns the exclusive
// prefix of v and writes the block total to *total.
__device__ __forceinline__ uint32_t block_exscan(uint32_t v, uint32_t *shm32, uint32_t *total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += t;
  }
  __syncthreads();
  if (lane == 31) shm32[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < (int)(blockDim.x >> 5) ? shm32[lane] : 0u;
    uint32_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t t = __shfl_up_sync(FULL, wi, o);
      if (lane >= o) wi += t;
    }
    shm32[lane] = wi - w;
    if (lane == 31) shm32[32] = wi;
  }
  __syncthreads();
  uint32_t r = shm32[warp] + incl - v;
  *total = shm32[32];
  return r;
}

// A4: number of non-empty nodes of level l (one CTA per level, blockDim 1024).
// Node p of level l is non-empty iff C_l(p+1) > C_l(p)  (Fig. 1 l.18-20).
__global__ void __launch_bounds__(1024) k_node_count(const uint32_t *__restrict__ Hx, uint32_t Lh,
                                                    uint32_t *__restrict__ ncount, const uint32_t *err) {
  __shared__ uint32_t shm[33];
  if (*err) return;
  const uint32_t l = blockIdx.x;
  const uint32_t np = 1u << l, sh = Lh - l;
  uint32_t c = 0;
  for (uint32_t p = threadIdx.x; p < np; p += blockDim.x)
    c += Hx[(uint64_t)(p + 1) << sh] > Hx[(uint64_t)p << sh];
  uint32_t tot;
  block_exscan(c, shm, &tot);
  if (threadIdx.x == 0) ncount[l] = tot;
}

__global__ void __launch_bounds__(1024) k_node_emit(const uint32_t *__restrict__ Hx, uint32_t Lh, uint32_t L,
                                                   const uint32_t *__restrict__ ncount,
                                                   uint64_t *__restrict__ level_node_ptr,
                                                   uint32_t *__restrict__ node_key,
                                                   uint32_t *__restrict__ node_start, const uint32_t *err) {
  __shared__ uint32_t shm[33];
  if (*err) return;
  const uint32_t l = blockIdx.x;
  uint64_t base = 0;
  for (uint32_t k = 0; k < l; k++) base += ncount[k];
  if (l == 0 && threadIdx.x <= L) {
    uint64_t acc = 0;
    for (uint32_t k = 0; k < threadIdx.x; k++) acc += ncount[k];
    level_node_ptr[threadIdx.x] = acc;
  }
  const uint32_t np = 1u << l, sh = Lh - l;
  const uint32_t per = (np + blockDim.x - 1) / blockDim.x;
  const uint32_t lo = min(threadIdx.x * per, np), hi = min(lo + per, np);
  uint32_t c = 0;
  for (uint32_t p = lo; p < hi; p++) c += Hx[(uint64_t)(p + 1) << sh] > Hx[(uint64_t)p << sh];
  uint32_t tot;
  uint32_t off = block_exscan(c, shm, &tot);
  for (uint32_t p = lo; p < hi; p++) {
    uint32_t s0 = Hx[(uint64_t)p << sh], s1 = Hx[(uint64_t)(p + 1) << sh];
    if (s1 > s0) {
      node_key[base + off] = p;
      node_start[base + off] = s0;
      off++;
    }
  }
}

// Tiles of the segments (= non-empty nodes of level l0) for a group g >= 1.
// One CTA (1024 threads).  Segment s covers [node_start[s], next start or n);
// it gets ceil(len / TW) warp tiles; tile_seg maps tile -> segment.
__global__ void __launch_bounds__(1024) k_segments(const uint64_t *__restrict__ level_node_ptr, uint32_t l0,
                                                  const uint32_t *__restrict__ node_start, uint64_t n,
                                                  uint32_t *__restrict__ seg_tile_base,
                                                  uint32_t *__restrict__ tile_seg,
                                                  uint32_t *__restrict__ total_tiles, const uint32_t *err) {
  __shared__ uint32_t shm[33];
  if (*err) return;
  const uint64_t p0 = level_node_ptr[l0], p1 = level_node_ptr[l0 + 1];
  const uint32_t nseg = (uint32_t)(p1 - p0);
  const uint32_t *st = node_start + p0;
  uint32_t carry = 0;
  for (uint32_t base = 0; base < nseg; base += blockDim.x) {
    uint32_t s = base + threadIdx.x;
    uint32_t nt = 0;
    if (s < nseg) {
      uint64_t e = (s + 1 < nseg) ? st[s + 1] : n;
      nt = (uint32_t)((e - st[s] + TW - 1) / TW);
    }
    uint32_t tot;
    uint32_t off = block_exscan(nt, shm, &tot) + carry;
    if (s < nseg) {
      seg_tile_base[s] = off;
      for (uint32_t j = 0; j < nt; j++) tile_seg[off + j] = s;
    }
    carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total_tiles = carry;
}

// ---------------------------------------------------------------------------
// The hot kernel: one pass over HBM builds tau consecutive levels l0..l0+tau-1
// (SURVEY §8(a) A2, A3, A5, A6, A7).
//
// Work unit: a warp tile of <= TW consecutive positions of S_{l0} lying inside
// one level-l0 node ("segment", key P).  Per tile:
//  1. load keys (coalesced), record = (digit << pbits) | payload, where digit
//     = the tau level bits and payload = the bits below; per-tile digit
//     histogram; publish it as the tile aggregate (decoupled lookback).
//  2. tau stable 1-bit splits in shared memory (Fig. 1 l.12-17): at local level
//     k the tile is in S_{l0+k} order; a warp ballot of the level bit gives 32
//     bitmap bits (A2); an element's destination is
//        bit 0: O(gs) + (pos - O(pos))      bit 1: (ge - O(ge)) + O(pos)
//     where O(x) = ones before position x and [gs, ge) is its group; the
//     group terms come from the digit histogram (table T_k), O(pos) from a
//     running popcount.
//  3. lookback over preceding tiles of the same segment -> before[d], the
//     number of elements with digit d ahead of this tile in the segment;
//     publish the inclusive prefix.
//  4. global placement.  Level l0+k bits of prefix q form one run starting at
//        G = C_{l0+k}((P << k) | q) + sum_{d in q} before[d];
//     words fully inside the run are stored, shared edge words are OR-ed
//     atomically into the zero-initialised bitmap (A5).
//     Rank-directory block counts are accumulated per 512-bit block (A7).
//     Keys narrowed to the payload are written at their S_{l0+tau} position
//     (A6; the short-list idea of PAPER.md:26-34) for the next pass.
// ---------------------------------------------------------------------------
struct GroupParams {
  const void *keys_in;
  uint8_t *keys_out;
  uint64_t n;
  uint32_t Lh, l0, tau, pbits;
  const uint32_t *Hx;
  uint32_t single_seg;
  uint32_t ntiles_single;
  const uint64_t *level_node_ptr;
  const uint32_t *node_key;
  const uint32_t *node_start;
  const uint32_t *tile_seg;
  const uint32_t *seg_tile_base;
  const uint32_t *total_tiles;
  uint32_t *tile_counter;
  uint32_t *state;
  uint64_t *bits;
  uint64_t wpl;
  uint32_t *blkcnt;
  uint64_t bpl;
  const uint32_t *err;
};

template <typename RecT>
struct WarpSmem {
  alignas(16) RecT buf[2][TW];
  uint32_t LB[TAU_MAX][NCH];   // ballot words of each local level
  uint32_t hist[NDIG];         // digit counts; later before[]; later key bases
  uint32_t Hl[NDIG + 1];       // exclusive scan of hist (local group starts)
  uint32_t BX[NDIG + 1];       // exclusive scan of before[]
  uint16_t T[2 * NDIG];        // per-level split tables, level k at 2^(k+1)-2
  uint32_t RG[NDIG / 2 + 1];   // run global start
  uint32_t RL[NDIG / 2 + 1];   // run local start
  uint32_t RC[NDIG / 2 + 1];   // run length
  uint32_t RW[NDIG / 2 + 2];   // run word-count scan
};

template <typename InT, typename RecT, bool HAS_OUT>
__global__ void __launch_bounds__(128) k_group(GroupParams p) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WarpSmem<RecT> &ws = *reinterpret_cast<WarpSmem<RecT> *>(smem_raw + warp * sizeof(WarpSmem<RecT>));
  if (ld_volatile(p.err)) return;
  const InT *keys = reinterpret_cast<const InT *>(p.keys_in);
  const uint32_t tau = p.tau, pbits = p.pbits;
  const uint32_t ndig = 1u << tau;
  const uint32_t pmask = (1u << pbits) - 1u;
  const uint32_t total_tiles = p.single_seg ? p.ntiles_single : ld_volatile(p.total_tiles);
  const uint32_t lt = lanemask_lt();

  while (true) {
    uint32_t t = 0;
    if (lane == 0) t = atomicAdd(p.tile_counter, 1u);
    t = __shfl_sync(FULL, t, 0);
    if (t >= total_tiles) break;

    // ---- tile geometry ----
    uint32_t seg = 0, j = t, P = 0;
    uint64_t seg_begin = 0, seg_end = p.n;
    if (!p.single_seg) {
      const uint64_t p0 = p.level_node_ptr[p.l0], p1 = p.level_node_ptr[p.l0 + 1];
      seg = p.tile_seg[t];
      j = t - p.seg_tile_base[seg];
      seg_begin = p.node_start[p0 + seg];
      seg_end = (p0 + seg + 1 < p1) ? p.node_start[p0 + seg + 1] : p.n;
      P = p.node_key[p0 + seg];
    }
    const uint64_t start = seg_begin + (uint64_t)j * TW;
    const uint64_t rem = seg_end - start;
    const uint32_t len = rem < (uint64_t)TW ? (uint32_t)rem : (uint32_t)TW;
    const uint32_t nch = (len + 31) >> 5;

    // ---- 1. load, records, histogram, publish aggregate ----
    for (uint32_t d = lane; d < ndig; d += 32) ws.hist[d] = 0;
    __syncwarp();
    RecT *b0 = ws.buf[0];
    const InT *src_keys = keys + start;
    constexpr int PER = 16 / sizeof(InT);  // symbols per 16-byte load
    if (len == TW && (reinterpret_cast<uintptr_t>(src_keys) & 15) == 0) {
      // full, aligned tile: 16-byte streaming loads, records stored as a vector
      const uint4 *v = reinterpret_cast<const uint4 *>(src_keys);
#pragma unroll 4
      for (int i = lane; i < TW / PER; i += 32) {
        const uint4 q = __ldcs(v + i);
        const InT *e = reinterpret_cast<const InT *>(&q);
        RecT r[PER];
#pragma unroll
        for (int k = 0; k < PER; k++) {
          const uint32_t key = (uint32_t)e[k];
          const uint32_t dig = (key >> pbits) & (ndig - 1u);
          r[k] = (RecT)((dig << pbits) | (key & pmask));
          atomicAdd(&ws.hist[dig], 1u);
        }
        if constexpr (PER * sizeof(RecT) == 16) {
          *reinterpret_cast<uint4 *>(b0 + i * PER) = *reinterpret_cast<const uint4 *>(r);
        } else if constexpr (PER * sizeof(RecT) == 8) {
          *reinterpret_cast<uint2 *>(b0 + i * PER) = *reinterpret_cast<const uint2 *>(r);
        } else {
#pragma unroll
          for (int k = 0; k < PER; k++) b0[i * PER + k] = r[k];
        }
      }
    } else {
      for (uint32_t c = 0; c < nch; c++) {
        uint32_t pos = c * 32 + lane;
        if (pos < len) {
          uint32_t key = (uint32_t)src_keys[pos];
          uint32_t dig = (key >> pbits) & (ndig - 1u);
          b0[pos] = (RecT)((dig << pbits) | (key & pmask));
          atomicAdd(&ws.hist[dig], 1u);
        }
      }
    }
    __syncwarp();
    uint32_t *st = p.state + (uint64_t)t * NDIG;
    for (uint32_t d = lane; d < ndig; d += 32) st_volatile(st + d, (j == 0 ? FLAG_INC : FLAG_AGG) | ws.hist[d]);

    // ---- 2. lookback, per digit (lane handles digits lane, lane+32, ...).
    //      Done before the local splits so that the inclusive prefix is
    //      published early and successors' walks stay short. ----
    if (j == 0) {
      for (uint32_t d = lane; d < ndig; d += 32) ws.BX[d] = 0;  // before[d]
    } else {
      constexpr int DPL = NDIG / 32;
      uint32_t acc[DPL];
      uint32_t done = 0, need = 0;
#pragma unroll
      for (int i = 0; i < DPL; i++) {
        acc[i] = 0;
        if (lane + 32u * i < ndig) need |= 1u << i;
      }
      uint32_t u = t - 1;
      while (done != need) {
        uint32_t v[DPL];
        bool ready = true;
#pragma unroll
        for (int i = 0; i < DPL; i++) {
          v[i] = 0;
          if ((need & ~done) & (1u << i)) {
            v[i] = ld_volatile(p.state + (uint64_t)u * NDIG + lane + 32u * i);
            if ((v[i] & ~VAL_MASK) == 0) ready = false;
          }
        }
        if (!ready) continue;  // predecessor has not published yet: spin
#pragma unroll
        for (int i = 0; i < DPL; i++) {
          if ((need & ~done) & (1u << i)) {
            acc[i] += v[i] & VAL_MASK;
            if ((v[i] & ~VAL_MASK) == FLAG_INC) done |= 1u << i;
          }
        }
        u--;
      }
#pragma unroll
      for (int i = 0; i < DPL; i++) {
        uint32_t d = lane + 32u * i;
        if (d < ndig) {
          st_volatile(st + d, FLAG_INC | (acc[i] + ws.hist[d]));
          ws.BX[d] = acc[i];
        }
      }
    }
    __syncwarp();
    // ---- 3. local tables and tau stable splits ----
    warp_exscan(ws.hist, ndig, ws.Hl, lane);
    // hist[] <- before[]; BX <- exclusive scan of before[]
    for (uint32_t d = lane; d < ndig; d += 32) ws.hist[d] = ws.BX[d];
    __syncwarp();
    warp_exscan(ws.hist, ndig, ws.BX, lane);
    for (uint32_t k = 0; k < tau; k++) {
      const uint32_t nq = 1u << k, sh = tau - k;
      uint16_t *Tk = ws.T + (2u << k) - 2u;
      // ones(q) = count of digits with prefix (q:1); O(q) = exclusive scan
      const uint32_t per = (nq + 31) >> 5;
      const uint32_t lo = min(lane * per, nq), hi = min(lo + per, nq);
      uint32_t s = 0;
      for (uint32_t q = lo; q < hi; q++)
        s += ws.Hl[(2 * q + 2) << (sh - 1)] - ws.Hl[(2 * q + 1) << (sh - 1)];
      uint32_t incl = s;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t v = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += v;
      }
      uint32_t O = incl - s;
      for (uint32_t q = lo; q < hi; q++) {
        uint32_t ones = ws.Hl[(2 * q + 2) << (sh - 1)] - ws.Hl[(2 * q + 1) << (sh - 1)];
        Tk[2 * q] = (uint16_t)O;                                   // O(gs)
        Tk[2 * q + 1] = (uint16_t)(ws.Hl[(q + 1) << sh] - (O + ones));  // ge - O(ge)
        O += ones;
      }
    }
    __syncwarp();
    for (uint32_t k = 0; k < tau; k++) {
      const uint32_t bitsh = pbits + tau - 1u - k;
      const uint16_t *Tk = ws.T + (2u << k) - 2u;
      const RecT *src = ws.buf[k & 1];
      RecT *dst = ws.buf[(k + 1) & 1];
      uint32_t Orun = 0;
      for (uint32_t c = 0; c < nch; c++) {
        const uint32_t pos = c * 32 + lane;
        const bool valid = pos < len;
        const uint32_t r = valid ? (uint32_t)src[pos] : 0u;
        const uint32_t tag = r >> bitsh;
        const bool P1 = valid && (tag & 1u);
        const uint32_t m = __ballot_sync(FULL, P1);
        if (lane == 0) ws.LB[k][c] = m;
        const uint32_t c1 = __popc(m & lt);
        const uint32_t tb = Tk[tag];
        const uint32_t d = P1 ? (tb + Orun + c1) : (tb + pos - Orun - c1);
        if (valid) dst[d] = (RecT)r;
        Orun += __popc(m);
      }
      __syncwarp();
    }
    const RecT *fin = ws.buf[tau & 1];

    // ---- 4a. narrowed keys at their S_{l0+tau} position (A6) ----
    const uint32_t lastlev = p.l0 + tau;
    if (HAS_OUT) {
      for (uint32_t d = lane; d < ndig; d += 32) {
        uint32_t pref = (P << tau) | d;
        uint32_t C = p.Hx[(uint64_t)pref << (p.Lh - lastlev)];
        ws.hist[d] = C + ws.hist[d] - ws.Hl[d];  // key base per digit
      }
      __syncwarp();
      for (uint32_t c = 0; c < nch; c++) {
        uint32_t pos = c * 32 + lane;
        if (pos < len) {
          uint32_t r = fin[pos];
          uint32_t d = r >> pbits;
          p.keys_out[ws.hist[d] + pos] = (uint8_t)(r & pmask);
        }
      }
    }

    // ---- 4b. bitmap runs + rank block counts (A2, A5, A7) ----
    for (uint32_t k = 0; k < tau; k++) {
      const uint32_t lev = p.l0 + k;
      const uint32_t nq = 1u << k, sh = tau - k;
      for (uint32_t q = lane; q < nq; q += 32) {
        uint32_t ls = ws.Hl[q << sh];
        uint32_t cnt = ws.Hl[(q + 1) << sh] - ls;
        uint32_t pref = (P << k) | q;
        uint32_t G = p.Hx[(uint64_t)pref << (p.Lh - lev)] + (ws.BX[(q + 1) << sh] - ws.BX[q << sh]);
        ws.RG[q] = G;
        ws.RL[q] = ls;
        ws.RC[q] = cnt;
        ws.RW[q] = cnt ? (uint32_t)(((uint64_t)G + cnt - 1) >> 6) - (G >> 6) + 1u : 0u;
      }
      __syncwarp();
      warp_exscan(ws.RW, nq, ws.RW, lane);
      const uint32_t total_w = ws.RW[nq];
      uint64_t *B = p.bits + (uint64_t)lev * p.wpl;
      uint32_t *BC = p.blkcnt + (uint64_t)lev * p.bpl;
      uint32_t q = 0;
      for (uint32_t i0 = 0; i0 < total_w; i0 += 32) {
        const uint32_t i = i0 + lane;
        const bool act = i < total_w;
        const uint32_t amask = __ballot_sync(FULL, act);
        if (act) {
          while (ws.RW[q + 1] <= i) q++;
          const uint32_t G = ws.RG[q], ls = ws.RL[q], cnt = ws.RC[q];
          const uint64_t gw = (G >> 6) + (i - ws.RW[q]);
          const uint64_t lo = gw * 64;
          const int base = (int)((int64_t)ls + (int64_t)lo - (int64_t)G);
          uint64_t val = extract64(ws.LB[k], base, NCH);
          const uint64_t s0 = ((uint64_t)G > lo ? (uint64_t)G : lo) - lo;
          const uint64_t gend = (uint64_t)G + cnt;
          const uint64_t e0 = (gend < lo + 64 ? gend : lo + 64) - lo;
          const uint64_t mask = (e0 - s0 == 64) ? ~0ull : (((1ull << (e0 - s0)) - 1ull) << s0);
          val &= mask;
          const uint64_t hi_clip = (lo + 64 < p.n) ? lo + 64 : p.n;
          const bool owned = (G <= lo) && ((uint64_t)G + cnt >= hi_clip);
          if (owned) B[gw] = val;
          else if (val) atomicOr(reinterpret_cast<unsigned long long *>(&B[gw]), (unsigned long long)val);
          const uint32_t blk = (uint32_t)(gw >> 3);
          const uint32_t peers = __match_any_sync(amask, blk);
          const uint32_t sum = __reduce_add_sync(peers, (uint32_t)__popcll(val));
          if (sum && lane == (__ffs(peers) - 1)) atomicAdd(&BC[blk], sum);
        }
      }
      __syncwarp();
    }
  }
}

// ---------------------------------------------------------------------------
// A7 finalize: rank_block (u16, relative to the superblock) and rank_super.
// k_rank_local: one warp per (level, superblock); k_rank_super: one CTA per level.
// ---------------------------------------------------------------------------
__global__ void k_rank_local(const uint32_t *__restrict__ blkcnt, uint64_t bpl, uint64_t nsup_data,
                             uint32_t L, uint16_t *__restrict__ rank_block, uint64_t *__restrict__ suptot,
                             const uint32_t *err) {
  if (*err) return;
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (gw >= (uint64_t)L * nsup_data) return;
  const uint32_t l = (uint32_t)(gw / nsup_data);
  const uint64_t s = gw % nsup_data;
  const uint64_t b0 = s * 128;
  uint32_t v[4], sum = 0;
#pragma unroll
  for (int i = 0; i < 4; i++) {
    uint64_t b = b0 + lane * 4 + i;
    v[i] = b < bpl ? blkcnt[(uint64_t)l * bpl + b] : 0u;
    sum += v[i];
  }
  uint32_t incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += t;
  }
  uint32_t run = incl - sum;
#pragma unroll
  for (int i = 0; i < 4; i++) {
    uint64_t b = b0 + lane * 4 + i;
    if (b < bpl) rank_block[(uint64_t)l * bpl + b] = (uint16_t)run;
    run += v[i];
  }
  if (lane == 31) suptot[(uint64_t)l * nsup_data + s] = incl;
}

__global__ void __launch_bounds__(1024) k_rank_super(const uint64_t *__restrict__ suptot, uint64_t nsup_data,
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

__global__ void k_access(TreeView t, const uint64_t *__restrict__ pos, uint64_t q, uint32_t *__restrict__ out) {
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

__global__ void k_rank_query(TreeView t, uint64_t sigma, const uint32_t *__restrict__ sym,
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
