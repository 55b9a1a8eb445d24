// wt_wm.cuh -- wavelet matrix: the group
// pass and the batched queries.
//
// Definition: A_0 = S; level l's bitmap holds the
// (l+1)'st highest bit of A_l; A_{l+1} = A_l stably reordered by that bit,
// zeros first; each level stores its number of 0 bits.  Equivalently A_l is
// S stably sorted by the reverse of its top l bits (:924-925).
//
// Fused pass over tau levels l0 .. l0+tau-1 (same chains, tiles, carries and
// run placement as the tree's k_group, one warp per chain): the input is
// A_{l0}; with d the tau-bit digit of a key (its next tau bits, MSB first),
// the order of A_{l0+k} restricted to one tile is the tile stably sorted by
// the WM class c = reverse of the top k bits of d (class_k(d) = the low k
// bits of rev_tau(d)), and A_{l0+k+1} is obtained from A_{l0+k} by ONE
// stable zeros-first split of the whole tile by bit k of d (the new bit
// becomes the most significant of the class).  So every split is a
// single-class split (no table), and level l0+k's bits of class c form one
// run in the tile, placed at
//     G = #{all elements of the sequence with a smaller class}     (global)
//       + #{class-c elements in earlier tiles}                     (before)
// -- class counts are sums of digit counts over the contiguous digit range
// of the prefix t = reverse_k(c).
#pragma once
#include "wt_common.cuh"
#include "wt_group.cuh"

namespace wtb {

#ifndef WT_WMTW
#define WT_WMTW 2048
#endif
template <typename RecT>
struct WmTile {
  static constexpr int TW = sizeof(RecT) == 1 ? 2 * WT_WMTW : (sizeof(RecT) == 2 ? WT_WMTW : WT_WMTW / 2);
};

template <typename RecT, bool HAS_OUT>
struct WmSmem {
  static constexpr int TWT = WmTile<RecT>::TW;
  alignas(16) RecT buf[2][TWT + 16 / sizeof(RecT)];
  alignas(16) uint32_t H[NDIG + 4];        // tile digit counts, then exclusive scan (digit order)
  alignas(16) uint32_t BX[NDIG + 4];       // same-sequence elements ahead of the tile, exclusive over digits
  alignas(16) uint32_t CR[NDIG + 4];       // whole-sequence exclusive digit scan (Cseg[0])
  alignas(16) unsigned long long CW[NDIG]; // carried partial word of run slot (1 << k) + c
  alignas(16) uint32_t LB[TWT / 32 + 8];   // ballot words of the current level
  alignas(16) uint32_t KB[HAS_OUT ? NDIG : 4];
  alignas(16) uint32_t RS[NDIG + 4];       // per class of the current level: tile-local start
  alignas(16) uint32_t GS[NDIG + 4];       // per class: global start of this tile's run
  alignas(16) uint16_t RO[NDIG + 8];
  alignas(16) uint8_t CF[NDIG];
  uint32_t zt;                             // zeros of the level bit in the tile
};

__device__ __forceinline__ uint32_t rev_bits(uint32_t c, uint32_t k) { return k ? __brev(c) >> (32 - k) : 0u; }

// Classes of local level k (one warp): RS[c] = tile-local start, GS[c] =
// global start of the tile's class-c run, RS[2^k] = len; when k < tau also
// s.zt = zeros of the level bit in the tile.
template <typename SM>
__device__ __forceinline__ void wm_classes(SM &s, uint32_t k, uint32_t tau, int lane) {
  const uint32_t nq = 1u << k, sh = tau - k;
  const uint32_t per = (nq + 31) >> 5;
  const uint32_t lo = min(lane * per, nq), hi = min(lo + per, nq);
  uint32_t tcv[NDIG / 32], gcv[NDIG / 32];
  uint32_t st = 0, sg = 0, zs = 0;
#pragma unroll
  for (int i = 0; i < NDIG / 32; i++) {
    const uint32_t c = lo + i;
    tcv[i] = gcv[i] = 0;
    if (c < hi) {
      const uint32_t t = rev_bits(c, k);
      tcv[i] = s.H[(t + 1) << sh] - s.H[t << sh];
      gcv[i] = s.CR[(t + 1) << sh] - s.CR[t << sh];
      if (k < tau) zs += s.H[(2 * t + 1) << (sh - 1)] - s.H[(2 * t) << (sh - 1)];
    }
    st += tcv[i];
    sg += gcv[i];
  }
  const uint32_t it = warp_incl_scan(st, lane), ig = warp_incl_scan(sg, lane);
  uint32_t rt = it - st, rg = ig - sg;
#pragma unroll
  for (int i = 0; i < NDIG / 32; i++) {
    const uint32_t c = lo + i;
    if (c < hi) {
      const uint32_t t = rev_bits(c, k);
      s.RS[c] = rt;
      s.GS[c] = rg + (s.BX[(t + 1) << sh] - s.BX[t << sh]);
    }
    rt += tcv[i];
    rg += gcv[i];
  }
  if (lane == 31) s.RS[nq] = it;
  const uint32_t z = __reduce_add_sync(FULL, zs);
  if (lane == 0) s.zt = z;
}

// One warp: stable zeros-first split of the whole tile by bit `bitsh` of the
// records (src -> dst), the level's ballot words into LB.
template <typename RecT, bool DO_SPLIT>
__device__ __forceinline__ void wm_split(uint32_t srcA, uint32_t dstA, uint32_t zt, uint32_t len, uint32_t bitsh,
                                         uint32_t *LB, int lane, uint32_t lt) {
  constexpr uint32_t RB = sizeof(RecT);
  uint32_t bitmask = 1u << bitsh;
  asm("" : "+r"(bitmask));
  const uint32_t sA = srcA + lane * RB;
  const uint32_t a1 = dstA + RB * zt;
  const uint32_t LA = smem_u32(LB);
  uint32_t Orun = 0;
  const uint32_t full = len / (32 * U);
  for (uint32_t b = 0; b < full; b++) {
    const uint32_t cb = b * (32 * U);
    uint32_t r[U], m[U];
#pragma unroll
    for (int u = 0; u < U; u++) r[u] = lds<RecT>(sA + (cb + u * 32) * RB);
#pragma unroll
    for (int u = 0; u < U; u++) {
      const bool P = (r[u] & bitmask) != 0;
      m[u] = __ballot_sync(FULL, P);
      if constexpr (DO_SPLIT) {
        const uint32_t O = Orun + __popc(m[u] & lt);
        const uint32_t Z = cb + u * 32 + lane - O;
        sts<RecT>(P ? a1 + RB * O : dstA + RB * Z, r[u]);
        Orun += __popc(m[u]);
      }
    }
    if (lane == 0) {
#pragma unroll
      for (int u = 0; u < U; u += 4) sts_v4(LA + b * (4 * U) + 4 * u, m[u], m[u + 1], m[u + 2], m[u + 3]);
    }
  }
  const uint32_t nch = (len + 31) >> 5;
  for (uint32_t ci = full * U; ci < nch; ci++) {
    const uint32_t x = ci * 32 + lane;
    const bool valid = x < len;
    const uint32_t r = valid ? lds<RecT>(sA + ci * 32 * RB) : 0u;
    const bool P = valid && (r & bitmask);
    const uint32_t m = __ballot_sync(FULL, P);
    if (lane == 0) LB[ci] = m;
    if constexpr (DO_SPLIT) {
      const uint32_t O = Orun + __popc(m & lt);
      if (valid) sts<RecT>(P ? a1 + RB * O : dstA + RB * (x - O), r);
      Orun += __popc(m);
    }
  }
}

template <typename InT, typename RecT, typename OutT, bool HAS_OUT>
__global__ void __launch_bounds__(32) k_wm_group(GroupParams p) {
  using SM = WmSmem<RecT, HAS_OUT>;
  constexpr int TWT = SM::TWT;
  constexpr int NW = TWT / 32 + 8;
  constexpr uint32_t RB = sizeof(RecT);
  __shared__ SM s;
  const int lane = threadIdx.x;
  if (ld_relaxed(p.err)) return;
  const InT *keys = reinterpret_cast<const InT *>(p.keys_in);
  const uint32_t tau = p.tau, pbits = p.pbits;
  const uint32_t ndig = 1u << tau;
  const uint32_t pmask = (1u << pbits) - 1u;
  const uint32_t nchains = p.counts[0];
  const uint32_t lt = lanemask_lt();
  for (uint32_t d = lane; d <= ndig; d += 32) s.CR[d] = p.Cseg[d];  // one row: the whole sequence

  while (true) {
    uint32_t c = 0;
    if (lane == 0) c = atomicAdd(p.chain_counter, 1u);
    c = __shfl_sync(FULL, c, 0);
    if (c >= nchains) break;
    const uint32_t cbeg = p.chain_begin[c], cend = p.chain_end[c];
    for (uint32_t d = lane; d < ndig; d += 32) s.BX[d] = p.E[(uint64_t)d * p.estride + c];
    for (uint32_t i = lane; i < NDIG / 4; i += 32) reinterpret_cast<uint32_t *>(s.CF)[i] = 0u;
    __syncwarp();
    digit_exscan(s.BX, ndig, lane);
    __syncwarp();

    for (uint64_t start64 = cbeg; start64 < cend; start64 += TWT) {  // 64-bit: cend may be near 2^32
      const uint32_t start = (uint32_t)start64;
      const uint32_t rem = cend - start;
      const uint32_t len = rem < (uint32_t)TWT ? rem : (uint32_t)TWT;
      for (uint32_t d = lane; d < NDIG; d += 32) s.H[d] = 0u;
      __syncwarp();
      // ---- load, records, digit counts ----
      uint32_t head0 = 0;
      {
        constexpr int PER = 16 / sizeof(InT);
        const uintptr_t sb = reinterpret_cast<uintptr_t>(keys + start);
        const uintptr_t ab = sb & ~(uintptr_t)15;
        const int head = (int)((sb - ab) / sizeof(InT));
        const uint4 *v = reinterpret_cast<const uint4 *>(ab);
        RecT *b0 = s.buf[0];
        if (sizeof(InT) == sizeof(RecT) || (head == 0 && len == (uint32_t)TWT)) {
          if constexpr (sizeof(InT) == sizeof(RecT)) head0 = (uint32_t)head;
          const int nv = (head + (int)len + PER - 1) / PER;
          for (int i = lane; i < nv; i += 32) {
            const uint4 q = __ldcs(v + i);
            const InT *e = reinterpret_cast<const InT *>(&q);
            if constexpr (sizeof(InT) == sizeof(RecT)) *reinterpret_cast<uint4 *>(b0 + i * PER) = q;
#pragma unroll
            for (int k = 0; k < PER; k++) {
              const int pos = i * PER + k - head;
              const bool in = (unsigned)pos < len;
              if constexpr (sizeof(InT) != sizeof(RecT)) {
                if (in) b0[pos] = (RecT)(uint32_t)e[k];
              }
              atomicAdd(&s.H[in ? (((uint32_t)e[k] >> pbits) & (ndig - 1u)) : (uint32_t)TRASH], 1u);
            }
          }
        } else {  // unaligned or ragged tile with a width conversion: element by element
          for (uint32_t i = lane; i < len; i += 32) {
            const uint32_t key = (uint32_t)keys[start + i];
            b0[i] = (RecT)key;
            atomicAdd(&s.H[(key >> pbits) & (ndig - 1u)], 1u);
          }
        }
      }
      __syncwarp();
      digit_exscan(s.H, ndig, lane);
      __syncwarp();
      if constexpr (HAS_OUT) {  // final order: class rev_tau(d); KB[d] = global start - local start
        wm_classes(s, tau, tau, lane);
        __syncwarp();
        for (uint32_t cc = lane; cc < ndig; cc += 32) {
          const uint32_t d = rev_bits(cc, tau);
          s.KB[d] = s.GS[cc] - s.RS[cc];
        }
        __syncwarp();
      }
      // ---- levels ----
      for (uint32_t k = 0; k < tau; k++) {
        const bool do_split = HAS_OUT || (k + 1 < tau);
        const uint32_t bitsh = pbits + tau - 1u - k;
        const uint32_t srcA = smem_u32(s.buf[k & 1]) + (k == 0 ? head0 * RB : 0u);
        const uint32_t dstA = smem_u32(s.buf[(k + 1) & 1]);
        wm_classes(s, k, tau, lane);
        __syncwarp();
        if (do_split) wm_split<RecT, true>(srcA, dstA, s.zt, len, bitsh, s.LB, lane, lt);
        else wm_split<RecT, false>(srcA, dstA, 0, len, bitsh, s.LB, lane, lt);
        __syncwarp();
        // runs: class c's bits are LB bits [RS[c], RS[c+1]) -> global [GS[c], ...)
        uint64_t *B = p.bits + (uint64_t)(p.l0 + k) * p.wpl;
        const uint32_t nq = 1u << k;
        uint32_t Ni = 0;
        for (uint32_t j0 = 0; j0 < nq; j0 += 32) {
          const uint32_t q = j0 + lane;
          uint32_t ni = 0;
          if (q < nq) {
            const uint32_t ls = s.RS[q], cnt = s.RS[q + 1] - ls;
            if (cnt) {
              const uint32_t G = s.GS[q];
              const uint32_t gw0 = G >> 6, gw1 = (uint32_t)(((uint64_t)G + cnt - 1) >> 6);
              ni = gw1 > gw0 + 1 ? gw1 - gw0 - 1 : 0u;
              run_ends(s, s.LB, NW, nq + q, B, p.n, G, ls, cnt);
            }
          }
          const uint32_t incl = warp_incl_scan(ni, lane);
          if (q < nq) s.RO[q] = (uint16_t)(Ni + incl - ni);
          Ni += __shfl_sync(FULL, incl, 31);
        }
        __syncwarp();
        for (uint32_t j = lane; j < Ni; j += 32) {
          uint32_t lo = 0, hi = nq;
          while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (s.RO[mid] <= j) lo = mid;
            else hi = mid;
          }
          const uint32_t ls = s.RS[lo], G = s.GS[lo];
          const uint32_t gw = (G >> 6) + 1 + (j - s.RO[lo]);
          B[gw] = extract64(s.LB, (int)(ls + gw * 64u - G), NW);
        }
        __syncwarp();
      }
      // ---- narrowed keys for the next pass (A_{l0+tau} order) ----
      if constexpr (HAS_OUT) {
        OutT *ko = reinterpret_cast<OutT *>(p.keys_out);
        const RecT *fin = s.buf[tau & 1];
        for (uint32_t i = lane; i < len; i += 32) {
          const uint32_t r = fin[i];
          ko[s.KB[r >> pbits] + i] = (OutT)(r & pmask);
        }
      }
      for (uint32_t d = lane; d <= ndig; d += 32) s.BX[d] += s.H[d];
      __syncwarp();
    }
    // ---- chain end: flush carried words at the runs' end positions ----
    for (uint32_t k = 0; k < tau; k++) {
      wm_classes(s, k, tau, lane);  // GS = global end of this chain's runs (BX is past the last tile)
      __syncwarp();
      for (uint32_t q = lane; q < (1u << k); q += 32) {
        const uint32_t slot = (1u << k) + q;
        if (s.CF[slot] & CF_VALID) {
          uint64_t *B = p.bits + (uint64_t)(p.l0 + k) * p.wpl;
          atomicOr(reinterpret_cast<unsigned long long *>(&B[s.GS[q] >> 6]), s.CW[slot]);
        }
      }
      __syncwarp();
    }
  }
}

// ===========================================================================
// CTA version (WPB warps, the tile of the tree's k_group): per level, warp 0
// derives the classes (RS, GS, ZP) from the tile histogram; levels 0..J0-1
// split the whole tile cooperatively (quarters, ones of each quarter from a
// ballot pass); deeper levels give every warp a contiguous range of whole
// classes, whose zeros / ones bases follow from the histogram alone (class
// c's zeros count is a digit-range sum), so no counting pass is needed.
// ===========================================================================
template <typename RecT, bool HAS_OUT>
struct WmSmem4 {
  static constexpr int TT = GroupTile<RecT>::TT;
  static constexpr int NLB = TT / 32 + 8 * WPB;
  alignas(16) RecT buf[2][TT + 16 / sizeof(RecT)];
  alignas(16) uint32_t H[NDIG + 4];
  alignas(16) uint32_t BX[NDIG + 4];
  alignas(16) uint32_t CR[NDIG + 4];
  alignas(16) unsigned long long CW[NDIG];
  alignas(16) uint32_t LB[NLB];
  alignas(16) uint32_t KB[HAS_OUT ? NDIG : 4];
  alignas(16) uint32_t RS[NDIG + 4];       // class c of the level: tile-local start (RS[nq] = len)
  alignas(16) uint32_t GS[NDIG + 4];       // global start of the tile's class-c run
  alignas(16) uint32_t ZP[NDIG + 4];       // zeros of the level bit in classes < c
  alignas(16) uint16_t RO[WPB][NDIG / 2 + 8];  // a warp may own every class of a level (small tiles)
  alignas(16) uint8_t CF[NDIG];
  uint32_t onesW[WPB];
  uint32_t wr[WPB + 1];                    // first class of each warp's range (deep levels)
  uint32_t zt;
  uint32_t chain;
};

// wm_classes plus ZP (one warp); k < tau.
template <typename SM>
__device__ __forceinline__ void wm_classes4(SM &s, uint32_t k, uint32_t tau, int lane) {
  const uint32_t nq = 1u << k, sh = tau - k;
  const uint32_t per = (nq + 31) >> 5;
  const uint32_t lo = min(lane * per, nq), hi = min(lo + per, nq);
  uint32_t st = 0, sg = 0, sz = 0;
  for (uint32_t c = lo; c < hi; c++) {
    const uint32_t t = rev_bits(c, k);
    st += s.H[(t + 1) << sh] - s.H[t << sh];
    sg += s.CR[(t + 1) << sh] - s.CR[t << sh];
    sz += s.H[(2 * t + 1) << (sh - 1)] - s.H[t << sh];
  }
  const uint32_t it = warp_incl_scan(st, lane), ig = warp_incl_scan(sg, lane), iz = warp_incl_scan(sz, lane);
  uint32_t rt = it - st, rg = ig - sg, rz = iz - sz;
  for (uint32_t c = lo; c < hi; c++) {
    const uint32_t t = rev_bits(c, k);
    s.RS[c] = rt;
    s.GS[c] = rg + (s.BX[(t + 1) << sh] - s.BX[t << sh]);
    s.ZP[c] = rz;
    rt += s.H[(t + 1) << sh] - s.H[t << sh];
    rg += s.CR[(t + 1) << sh] - s.CR[t << sh];
    rz += s.H[(2 * t + 1) << (sh - 1)] - s.H[t << sh];
  }
  if (lane == 31) {
    s.RS[nq] = it;
    s.ZP[nq] = iz;
    s.zt = iz;
  }
}

// Stable zeros-first split of tile positions [p0, p0+wl) by bit `bitsh`
// (one warp): a zero goes to Z0 + (zeros before it in the range), a one to
// O0 + (ones before it in the range).  STORE_LB: ballot words to LB (bit x =
// position p0 + x, LB 16-byte aligned).  Returns the range's ones.
template <typename RecT, bool DO_SPLIT, bool STORE_LB>
__device__ __forceinline__ uint32_t wm_split_range(uint32_t srcA, uint32_t dstA, uint32_t p0, uint32_t wl,
                                                   uint32_t Z0, uint32_t O0, uint32_t bitsh, uint32_t *LB,
                                                   int lane, uint32_t lt) {
  constexpr uint32_t RB = sizeof(RecT);
  uint32_t bitmask = 1u << bitsh;
  uint32_t LA = smem_u32(LB), xl = (uint32_t)lane;
  asm("" : "+r"(bitmask), "+r"(LA), "+r"(xl));
  const uint32_t sA = srcA + (p0 + xl) * RB;
  const uint32_t a1 = dstA + RB * O0, a0 = dstA + RB * (Z0 + xl);
  uint32_t Orun = 0;
  const uint32_t full = wl / (32 * U);
  for (uint32_t b = 0; b < full; b++) {
    const uint32_t cb = b * (32 * U);
    uint32_t r[U], m[U];
#pragma unroll
    for (int u = 0; u < U; u++) r[u] = lds<RecT>(sA + (cb + u * 32) * RB);
#pragma unroll
    for (int u = 0; u < U; u++) {
      const bool P = (r[u] & bitmask) != 0;
      m[u] = __ballot_sync(FULL, P);
      if constexpr (DO_SPLIT) {
        const uint32_t O = Orun + __popc(m[u] & lt);
        sts<RecT>(P ? a1 + RB * O : a0 + RB * (cb + u * 32 - O), r[u]);
      }
      Orun += __popc(m[u]);
    }
    if (STORE_LB && lane == 0) {
#pragma unroll
      for (int u = 0; u < U; u += 4) sts_v4(LA + b * (4 * U) + 4 * u, m[u], m[u + 1], m[u + 2], m[u + 3]);
    }
  }
  const uint32_t nch = (wl + 31) >> 5;
  for (uint32_t ci = full * U; ci < nch; ci++) {
    const uint32_t x = ci * 32 + lane;
    const bool valid = x < wl;
    const uint32_t r = valid ? lds<RecT>(sA + ci * 32 * RB) : 0u;
    const bool P = valid && (r & bitmask);
    const uint32_t m = __ballot_sync(FULL, P);
    if (STORE_LB && lane == 0) LB[ci] = m;
    if constexpr (DO_SPLIT) {
      const uint32_t O = Orun + __popc(m & lt);
      if (valid) sts<RecT>(P ? a1 + RB * O : dstA + RB * (Z0 + x - O), r);
    }
    Orun += __popc(m);
  }
  return Orun;
}

// Runs of classes [qa, qb) of level k: class q's bits are LB bits
// [RS[q] - A, ...) (local to LB), placed at GS[q].  Edge words by the lanes of
// the edge warp, interior words by nthr threads after `sync`.
template <typename SM, typename Sync>
__device__ __forceinline__ void wm_emit(SM &s, uint16_t *RO, const uint32_t *LB, int nw, uint32_t k, uint32_t qa,
                                        uint32_t qb, uint32_t A, uint64_t *B, uint64_t n, bool edge_warp, int lane,
                                        int tid0, int nthr, Sync sync) {
  const uint32_t nq = qb - qa;
  if (edge_warp) {
    uint32_t Ni = 0;
    for (uint32_t j0 = 0; j0 < nq; j0 += 32) {
      const uint32_t q = qa + j0 + lane;
      uint32_t ni = 0;
      if (q < qb) {
        const uint32_t ls = s.RS[q] - A, cnt = s.RS[q + 1] - s.RS[q];
        if (cnt) {
          const uint32_t G = s.GS[q];
          const uint32_t gw0 = G >> 6, gw1 = (uint32_t)(((uint64_t)G + cnt - 1) >> 6);
          ni = gw1 > gw0 + 1 ? gw1 - gw0 - 1 : 0u;
          run_ends(s, LB, nw, (1u << k) + q, B, n, G, ls, cnt);
        }
      }
      const uint32_t incl = warp_incl_scan(ni, lane);
      if (q < qb) RO[q - qa] = (uint16_t)(Ni + incl - ni);
      Ni += __shfl_sync(FULL, incl, 31);
    }
    if (lane == 0) RO[nq] = (uint16_t)Ni;
  }
  sync();
  const uint32_t Ni = RO[nq];
  for (uint32_t j = tid0; j < Ni; j += nthr) {
    uint32_t lo = 0, hi = nq;
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (RO[mid] <= j) lo = mid;
      else hi = mid;
    }
    const uint32_t q = qa + lo;
    const uint32_t ls = s.RS[q] - A, G = s.GS[q];
    const uint32_t gw = (G >> 6) + 1 + (j - RO[lo]);
    B[gw] = extract64(LB, (int)(ls + gw * 64u - G), nw);
  }
}

template <typename InT, typename RecT, typename OutT, bool HAS_OUT>
__global__ void __launch_bounds__(WPB * 32, 4) k_wm_group4(GroupParams p) {
  using SM = WmSmem4<RecT, HAS_OUT>;
  constexpr int TT = SM::TT;
  constexpr int QL = TT / WPB;
  constexpr uint32_t RB = sizeof(RecT);
  __shared__ SM s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (ld_relaxed(p.err)) return;
  const InT *keys = reinterpret_cast<const InT *>(p.keys_in);
  const uint32_t tau = p.tau, pbits = p.pbits;
  const uint32_t ndig = 1u << tau;
  const uint32_t pmask = (1u << pbits) - 1u;
  const uint32_t nchains = p.counts[0];
  const uint32_t lt = lanemask_lt();
  const uint32_t jc = tau < (uint32_t)J0 ? tau : (uint32_t)J0;
  auto csync = [] { __syncthreads(); };
  auto wsync = [] { __syncwarp(); };
  for (uint32_t d = tid; d <= ndig; d += WPB * 32) s.CR[d] = p.Cseg[d];  // one row: the whole sequence

  while (true) {
    if (tid == 0) s.chain = atomicAdd(p.chain_counter, 1u);
    __syncthreads();
    const uint32_t c = s.chain;
    if (c >= nchains) break;
    const uint32_t cbeg = p.chain_begin[c], cend = p.chain_end[c];
    for (uint32_t d = tid; d < ndig; d += WPB * 32) s.BX[d] = p.E[(uint64_t)d * p.estride + c];
    for (uint32_t i = tid; i < NDIG / 4; i += WPB * 32) reinterpret_cast<uint32_t *>(s.CF)[i] = 0u;
    __syncthreads();
    if (warp == 0) digit_exscan(s.BX, ndig, lane);

    for (uint64_t start64 = cbeg; start64 < cend; start64 += TT) {  // 64-bit: cend may be near 2^32
      const uint32_t start = (uint32_t)start64;
      const uint32_t rem = cend - start;
      const uint32_t len = rem < (uint32_t)TT ? rem : (uint32_t)TT;
      for (uint32_t d = tid; d < NDIG; d += WPB * 32) s.H[d] = 0u;
      __syncthreads();
      // ---- load, records, digit counts (all threads) ----
      uint32_t head0 = 0;
      {
        constexpr int PER = 16 / sizeof(InT);
        const uintptr_t sb = reinterpret_cast<uintptr_t>(keys + start);
        const uintptr_t ab = sb & ~(uintptr_t)15;
        const int head = (int)((sb - ab) / sizeof(InT));
        const uint4 *v = reinterpret_cast<const uint4 *>(ab);
        RecT *b0 = s.buf[0];
        if (sizeof(InT) == sizeof(RecT) || (head == 0 && len == (uint32_t)TT)) {
          if constexpr (sizeof(InT) == sizeof(RecT)) head0 = (uint32_t)head;
          const int nv = (head + (int)len + PER - 1) / PER;
          for (int i = tid; i < nv; i += WPB * 32) {
            const uint4 q = __ldcs(v + i);
            const InT *e = reinterpret_cast<const InT *>(&q);
            if constexpr (sizeof(InT) == sizeof(RecT)) *reinterpret_cast<uint4 *>(b0 + i * PER) = q;
#pragma unroll
            for (int k = 0; k < PER; k++) {
              const int pos = i * PER + k - head;
              const bool in = (unsigned)pos < len;
              if constexpr (sizeof(InT) != sizeof(RecT)) {
                if (in) b0[pos] = (RecT)(uint32_t)e[k];
              }
              atomicAdd(&s.H[in ? (((uint32_t)e[k] >> pbits) & (ndig - 1u)) : (uint32_t)TRASH], 1u);
            }
          }
        } else {
          for (uint32_t i = tid; i < len; i += WPB * 32) {
            const uint32_t key = (uint32_t)keys[start + i];
            b0[i] = (RecT)key;
            atomicAdd(&s.H[(key >> pbits) & (ndig - 1u)], 1u);
          }
        }
      }
      __syncthreads();
      if (warp == 0) {
        digit_exscan(s.H, ndig, lane);
        __syncwarp();
        if constexpr (HAS_OUT) {  // final order: class rev_tau(d); KB[d] = global start - local start
          wm_classes(s, tau, tau, lane);
          __syncwarp();
          for (uint32_t cc = lane; cc < ndig; cc += 32) {
            const uint32_t d = rev_bits(cc, tau);
            s.KB[d] = s.GS[cc] - s.RS[cc];
          }
        }
      }
      __syncthreads();

      for (uint32_t k = 0; k < tau; k++) {
        const bool do_split = HAS_OUT || (k + 1 < tau);
        const uint32_t bitsh = pbits + tau - 1u - k;
        const uint32_t srcA = smem_u32(s.buf[k & 1]) + (k == 0 ? head0 * RB : 0u);
        const uint32_t dstA = smem_u32(s.buf[(k + 1) & 1]);
        const uint32_t nq = 1u << k;
        uint64_t *B = p.bits + (uint64_t)(p.l0 + k) * p.wpl;
        if (warp == 0) wm_classes4(s, k, tau, lane);
        if (k < jc) {
          // ---- cooperative level: quarters, ones per quarter from a ballot pass ----
          const uint32_t qlo = min((uint32_t)(warp * QL), len), qhi = min((uint32_t)((warp + 1) * QL), len);
          const uint32_t ones = wm_split_range<RecT, false, true>(srcA, dstA, qlo, qhi - qlo, 0, 0, bitsh,
                                                                  s.LB + qlo / 32, lane, lt);
          if (lane == 0) s.onesW[warp] = ones;
          __syncthreads();
          uint32_t Ob = 0;
          for (int w = 0; w < warp; w++) Ob += s.onesW[w];
          if (do_split)
            wm_split_range<RecT, true, false>(srcA, dstA, qlo, qhi - qlo, qlo - Ob, s.zt + Ob, bitsh,
                                              s.LB + qlo / 32, lane, lt);
          __syncthreads();
          wm_emit(s, s.RO[0], s.LB, SM::NLB, k, 0, nq, 0, B, p.n, warp == 0, lane, tid, WPB * 32, csync);
          __syncthreads();
        } else {
          // ---- deeper level: each warp a contiguous range of whole classes ----
          __syncthreads();
          if (warp == 0 && lane <= WPB) {  // wr[w] = first class whose start >= w * len / WPB
            const uint32_t target = (uint32_t)(((uint64_t)len * lane) / WPB);
            uint32_t lo = 0, hi = nq;
            while (lo < hi) {
              const uint32_t mid = (lo + hi) >> 1;
              if (s.RS[mid] < target) lo = mid + 1;
              else hi = mid;
            }
            s.wr[lane] = lane == WPB ? nq : (lane == 0 ? 0u : lo);
          }
          __syncthreads();
          const uint32_t qa = s.wr[warp], qb = max(s.wr[warp + 1], qa);
          const uint32_t A = s.RS[qa], wl = s.RS[qb] - A;
          uint32_t lbo = 0;
          for (int w = 0; w < warp; w++) lbo += ((s.RS[s.wr[w + 1]] - s.RS[s.wr[w]] + 127) / 128) * 4;
          uint32_t *LBw = s.LB + lbo;
          if (wl) {
            const uint32_t Z0 = s.ZP[qa], O0 = s.zt + A - s.ZP[qa];
            if (do_split) wm_split_range<RecT, true, true>(srcA, dstA, A, wl, Z0, O0, bitsh, LBw, lane, lt);
            else wm_split_range<RecT, false, true>(srcA, dstA, A, wl, Z0, O0, bitsh, LBw, lane, lt);
            __syncwarp();
            wm_emit(s, s.RO[warp], LBw, (int)((wl + 31) / 32), k, qa, qb, A, B, p.n, true, lane, lane, 32, wsync);
          }
          __syncthreads();
        }
      }
      // ---- narrowed keys for the next pass (A_{l0+tau} order) ----
      if constexpr (HAS_OUT) {
        OutT *ko = reinterpret_cast<OutT *>(p.keys_out);
        const RecT *fin = s.buf[tau & 1];
        for (uint32_t i = tid; i < len; i += WPB * 32) {
          const uint32_t r = fin[i];
          ko[s.KB[r >> pbits] + i] = (OutT)(r & pmask);
        }
      }
      for (uint32_t d = tid; d <= ndig; d += WPB * 32) s.BX[d] += s.H[d];
      __syncthreads();
    }
    // ---- chain end: flush carried words at the runs' end positions ----
    for (uint32_t k = 0; k < tau; k++) {
      if (warp == 0) wm_classes4(s, k, tau, lane);  // GS = global end of this chain's runs
      __syncthreads();
      for (uint32_t q = tid; q < (1u << k); q += WPB * 32) {
        const uint32_t slot = (1u << k) + q;
        if (s.CF[slot] & CF_VALID) {
          uint64_t *B = p.bits + (uint64_t)(p.l0 + k) * p.wpl;
          atomicOr(reinterpret_cast<unsigned long long *>(&B[s.GS[q] >> 6]), s.CW[slot]);
        }
      }
      __syncthreads();
    }
  }
}

// zeros[l] = n - (ones of level l), from the rank directory's level totals.
static __global__ void k_wm_zeros(const uint64_t *__restrict__ rank_super, uint64_t spl, uint32_t L, uint64_t n,
                           uint64_t *__restrict__ zeros, const uint32_t *err) {
  if (*err) return;
  const uint32_t l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l < L) zeros[l] = n - rank_super[(uint64_t)l * spl + spl - 1];
}

// Batched queries: a 0 bit at level l maps i -> rank0(i),
// a 1 bit maps i -> zeros[l] + rank1(i).
static __global__ void k_wm_access(TreeView t, const uint64_t *__restrict__ zeros, const uint64_t *__restrict__ pos,
                            uint64_t q, uint32_t *__restrict__ out) {
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= q) return;
  uint64_t i = pos[k];
  if (i >= t.n) { out[k] = 0xffffffffu; return; }
  uint32_t sym = 0;
  for (uint32_t l = 0; l < t.L; l++) {
    const uint32_t bit = (uint32_t)((t.bits[(uint64_t)l * t.wpl + (i >> 6)] >> (i & 63)) & 1ull);
    const uint64_t r1 = d_rank1(t, l, i);
    sym = (sym << 1) | bit;
    i = bit ? zeros[l] + r1 : i - r1;
  }
  out[k] = sym;
}

static __global__ void k_wm_rank(TreeView t, const uint64_t *__restrict__ zeros, uint64_t sigma,
                          const uint32_t *__restrict__ sym, const uint64_t *__restrict__ pos, uint64_t q,
                          uint64_t *__restrict__ out) {
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= q) return;
  const uint64_t i = pos[k];
  const uint32_t c = sym[k];
  if (i >= t.n || (uint64_t)c >= sigma) { out[k] = ~0ull; return; }
  uint64_t s = 0, e = i + 1;
  for (uint32_t l = 0; l < t.L && s < e; l++) {
    const uint64_t r1s = d_rank1(t, l, s), r1e = d_rank1(t, l, e);
    if ((c >> (t.L - 1 - l)) & 1u) {
      s = zeros[l] + r1s;
      e = zeros[l] + r1e;
    } else {
      s -= r1s;
      e -= r1e;
    }
  }
  out[k] = e - s;
}

}  // namespace wtb
