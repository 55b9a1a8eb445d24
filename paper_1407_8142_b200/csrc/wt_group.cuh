// wt_group.cuh -- the hot kernel: one HBM pass builds tau consecutive levels
// l0 .. l0+tau-1 of the levelwise wavelet tree.
//
// Work unit: a chain (<= CH consecutive positions of S_{l0} inside one
// level-l0 node, its "row"), processed by ONE warp (one warp per CTA, static
// shared memory, so every buffer has a compile-time address) as a sequence
// of tiles of <= GTW positions.  BX[d] = exclusive prefix over digits of the
// same-row elements ahead of the tile (chain prefix from the per-chain
// histograms, then a running sum).  Per tile:
//  1. load keys (16-byte vector loads); the record is the (narrowed) key
//     itself: its top tau bits are the digit, the rest the payload; digit
//     counts H (shared-memory atomics), then H := exclusive scan of H.
//  2. tau stable 1-bit splits in shared memory (Fig. 1 l.12-17): at
//     local level k the tile is in S_{l0+k} order; a warp ballot of the level
//     bit gives 32 bitmap bits in order (A2); an element's destination is
//        bit 0: T[2q]   + (pos - O(pos))      T[2q]   = O(gs)
//        bit 1: T[2q+1] + O(pos)              T[2q+1] = gm - O(gs)
//     where O(x) = ones before position x in the tile, [gs, ge) the element's
//     class q (its k-bit prefix) and gm the start of its right child: the
//     prefix sums X / X_s of Fig. 1 l.14 restated for all classes of the tile
//     at once; T is indexed by the top k+1 digit bits (q << 1 | bit).
//  3. global placement: level l0+k bits of class q form one run starting at
//        G = row_start + Cseg[row][q << (tau-k)] + sum_{d in q} before[d];
//     words fully inside a run are stored; the partial last word of a run is
//     carried to the next tile of the chain (runs of consecutive tiles are
//     adjacent), so only words shared with another chain or node are OR-ed
//     atomically into the zero-initialised bitmap (A5; at
//     most 2 shared words per node).
//  4. keys narrowed to the payload are written, per digit run, at their
//     S_{l0+tau} position for the next pass (A6; the short lists of
//     PAPER.md:26-34) -- coalesced runs from the final shared-memory order.
#pragma once
#include "wt_common.cuh"

namespace wtb {

struct GroupParams {
  const void *keys_in;
  void *keys_out;
  uint64_t n;
  uint32_t l0, tau, pbits;
  const uint32_t *counts;  // [0] chains, [1] rows
  const uint32_t *chain_begin;
  const uint32_t *chain_end;
  const uint32_t *chain_row;
  const uint32_t *row_first;  // first chain of each row
  const uint32_t *E;          // E[d][c]: same-row elements with digit d ahead of chain c (+ row offset)
  uint32_t estride;
  const uint32_t *Cseg;       // [row][ndig + 1]
  const uint32_t *row_start;
  uint32_t *chain_counter;
  uint64_t *bits;
  uint64_t wpl;
  uint32_t *err;
};

#ifndef WT_GTW
#define WT_GTW 2048
#endif
// tile width of the group kernel (positions per tile): 8 KB of records per
// buffer whatever the record width (u8: 2*GTW, u16: GTW, u32: GTW/2)
template <typename RecT>
struct GroupTile {
  static constexpr int TW = sizeof(RecT) == 1 ? 2 * WT_GTW : (sizeof(RecT) == 2 ? WT_GTW : WT_GTW / 2);
};

constexpr uint8_t CF_VALID = 1, CF_SHARED = 2;
constexpr int TRASH = NDIG + 2;  // histogram bin of the load cover's out-of-tile records

template <typename RecT, bool HAS_OUT>
struct GroupSmem {
  static constexpr int TWT = GroupTile<RecT>::TW;
  alignas(16) RecT buf[2][TWT + 16 / sizeof(RecT)];  // records, ping-pong between levels (+ load head)
  alignas(16) uint32_t H[NDIG + 4];        // tile digit counts, then their exclusive scan (H[ndig] = len)
  alignas(16) uint32_t BX[NDIG + 4];       // exclusive prefix over digits of same-row elements ahead of the tile
  alignas(16) uint32_t CR[NDIG + 4];       // the chain's row: start of each digit (Cseg[row])
  alignas(16) unsigned long long CW[NDIG]; // carried partial word of run slot (1 << k) + q
  alignas(16) uint32_t LB[TWT / 32];       // ballot words of the current level
  alignas(16) uint32_t KB[HAS_OUT ? NDIG : 4];  // per-digit base of the narrowed-key output
  alignas(16) uint16_t T[NDIG];            // split table of the current level (destination addresses)
  uint16_t FB[TWT / 256 + 2];              // per batch of 256 positions: its class if it lies in one
  alignas(16) uint8_t CF[NDIG];            // carry flags of each slot
};

// Bits of run [G, G+cnt) (local bits [ls, ls+cnt) of LB) that fall in global word gw.
template <int NW>
__device__ __forceinline__ uint64_t run_word(const uint32_t *LB, uint32_t G, uint32_t ls, uint32_t cnt, uint32_t gw) {
  const uint64_t lo = (uint64_t)gw * 64, gend = (uint64_t)G + cnt;
  uint64_t v = extract64(LB, (int)((int64_t)ls + (int64_t)lo - (int64_t)G), NW);
  const uint32_t s0 = (uint64_t)G > lo ? (uint32_t)(G - lo) : 0u;
  const uint32_t e0 = gend < lo + 64 ? (uint32_t)(gend - lo) : 64u;
  const uint64_t mask = (e0 - s0 == 64) ? ~0ull : (((1ull << (e0 - s0)) - 1ull) << s0);
  return v & mask;
}

// First and last word of a run, with the carry of slot `slot` (one lane).
template <typename SM>
__device__ __forceinline__ void run_ends(SM &s, uint32_t slot, uint64_t *B, uint64_t n, uint32_t G, uint32_t ls,
                                         uint32_t cnt) {
  constexpr int NW = SM::TWT / 32;
  const uint32_t gw0 = G >> 6, gw1 = (uint32_t)(((uint64_t)G + cnt - 1) >> 6);
  const uint64_t gend = (uint64_t)G + cnt;
  uint64_t v = run_word<NW>(s.LB, G, ls, cnt, gw0);
  const uint32_t f = s.CF[slot];
  bool shared;
  if (f & CF_VALID) {  // the word holds earlier bits of this run (previous tiles of the chain)
    v |= s.CW[slot];
    shared = (f & CF_SHARED) != 0;
  } else {
    shared = (G & 63u) != 0;  // its low bits belong to another chain or node
  }
  const uint64_t end0 = ((uint64_t)gw0 * 64 + 64 < n) ? (uint64_t)gw0 * 64 + 64 : n;
  if (gw0 == gw1 && gend < end0) {  // the word stays open: carry it to the next tile
    s.CW[slot] = v;
    s.CF[slot] = CF_VALID | (shared ? CF_SHARED : 0);
    return;
  }
  if (shared) atomicOr(reinterpret_cast<unsigned long long *>(&B[gw0]), (unsigned long long)v);
  else B[gw0] = v;
  s.CF[slot] = 0;
  if (gw1 > gw0) {
    const uint64_t v1 = run_word<NW>(s.LB, G, ls, cnt, gw1);
    const uint64_t end1 = ((uint64_t)gw1 * 64 + 64 < n) ? (uint64_t)gw1 * 64 + 64 : n;
    if (gend >= end1) {
      B[gw1] = v1;
    } else {
      s.CW[slot] = v1;
      s.CF[slot] = CF_VALID;
    }
  }
}

// Warp-cooperative exclusive scan over digits of a[0..nd) (in place, u32),
// a[nd] = total; lane owns PER = ceil(nd/32) consecutive digits.
__device__ __forceinline__ void digit_exscan(uint32_t *a, uint32_t nd, int lane) {
  const uint32_t per = (nd + 31) >> 5;
  const uint32_t lo = min(lane * per, nd), hi = min(lo + per, nd);
  uint32_t v[NDIG / 32], sum = 0;
#pragma unroll
  for (int i = 0; i < NDIG / 32; i++) {
    v[i] = (lo + i < hi) ? a[lo + i] : 0u;
    sum += v[i];
  }
  const uint32_t incl = warp_incl_scan(sum, lane);
  uint32_t run = incl - sum;
  __syncwarp();
#pragma unroll
  for (int i = 0; i < NDIG / 32; i++) {
    if (lo + i < hi) a[lo + i] = run;
    run += v[i];
  }
  if (lane == 31) a[nd] = incl;
}

constexpr int U = 8;  // chunks per software-pipelined batch

template <typename InT, typename RecT, typename OutT, bool HAS_OUT>
__global__ void __launch_bounds__(32) k_group(GroupParams p) {
  using SM = GroupSmem<RecT, HAS_OUT>;
  constexpr int TWT = SM::TWT;
  constexpr int NW = TWT / 32;
  __shared__ SM s;
  const int lane = threadIdx.x;
  if (ld_relaxed(p.err)) return;
  const InT *keys = reinterpret_cast<const InT *>(p.keys_in);
  const uint32_t tau = p.tau, pbits = p.pbits;
  const uint32_t ndig = 1u << tau;
  const uint32_t pmask = (1u << pbits) - 1u;
  const uint32_t nchains = p.counts[0];
  const uint32_t lt = lanemask_lt();

  while (true) {
    uint32_t c = 0;
    if (lane == 0) c = atomicAdd(p.chain_counter, 1u);
    c = __shfl_sync(FULL, c, 0);
    if (c >= nchains) break;

    // ---- chain geometry and its starting counts ----
    const uint32_t row = p.chain_row[c];
    const uint32_t cbeg = p.chain_begin[c], cend = p.chain_end[c];
    const uint32_t rstart = p.row_start[row];
    const uint32_t *Crow = s.CR;
    {
      const uint32_t *Cg = p.Cseg + (uint64_t)row * (ndig + 1);
      for (uint32_t d = lane; d <= ndig; d += 32) s.CR[d] = Cg[d];
      const uint32_t cfirst = p.row_first[row];
      for (uint32_t d = lane; d < ndig; d += 32)
        s.BX[d] = p.E[(uint64_t)d * p.estride + c] - p.E[(uint64_t)d * p.estride + cfirst];
      for (uint32_t i = lane; i < NDIG / 4; i += 32) reinterpret_cast<uint32_t *>(s.CF)[i] = 0u;
      __syncwarp();
      digit_exscan(s.BX, ndig, lane);
      __syncwarp();
    }

    for (uint32_t start = cbeg; start < cend; start += TWT) {
      const uint32_t rem = cend - start;
      const uint32_t len = rem < (uint32_t)TWT ? rem : (uint32_t)TWT;
      const uint32_t nch = (len + 31) >> 5;

      // ---- 1. load, records, digit counts ----
      for (uint32_t d = lane; d < NDIG; d += 32) s.H[d] = 0u;
      __syncwarp();
      const RecT *src0 = s.buf[0];  // level-l0 order of the tile
      {
        constexpr int PER = 16 / sizeof(InT);
        const uintptr_t sb = reinterpret_cast<uintptr_t>(keys + start);
        const uintptr_t ab = sb & ~(uintptr_t)15;
        const int head = (int)((sb - ab) / sizeof(InT));
        const uint4 *v = reinterpret_cast<const uint4 *>(ab);
        const int nv = (head + (int)len + PER - 1) / PER;
        if constexpr (sizeof(InT) == sizeof(RecT)) {
          // records are the keys: copy the aligned cover of the tile, the
          // tile starts `head` records into buf[0]
          RecT *b0 = s.buf[0];
          src0 = b0 + head;
          constexpr int VB = 8;  // vectors in flight per lane
          for (int i0 = 0; i0 < nv; i0 += 32 * VB) {
            uint4 q[VB];
#pragma unroll
            for (int j = 0; j < VB; j++) {
              const int i = i0 + lane + 32 * j;
              if (i < nv) q[j] = __ldcs(v + i);
            }
#pragma unroll
            for (int j = 0; j < VB; j++) {
              const int i = i0 + lane + 32 * j;
              if (i < nv) {
                *reinterpret_cast<uint4 *>(b0 + i * PER) = q[j];
                const InT *e = reinterpret_cast<const InT *>(&q[j]);
                const int p0 = i * PER - head;
                if (p0 >= 0 && p0 + PER <= (int)len) {
#pragma unroll
                  for (int k = 0; k < PER; k++) atomicAdd(&s.H[((uint32_t)e[k] >> pbits) & (ndig - 1u)], 1u);
                } else {
#pragma unroll
                  for (int k = 0; k < PER; k++) {
                    const bool in = (unsigned)(p0 + k) < len;
                    atomicAdd(&s.H[in ? (((uint32_t)e[k] >> pbits) & (ndig - 1u)) : (uint32_t)TRASH], 1u);
                  }
                }
              }
            }
          }
        } else {
          RecT *b0 = s.buf[0];
          if (head == 0 && len == (uint32_t)TWT) {
            constexpr int VB = 8;
            static_assert((TWT / PER) % (32 * VB) == 0, "tile = whole rounds of vectors");
#pragma unroll 1
            for (int i0 = 0; i0 < TWT / PER; i0 += 32 * VB) {
            uint4 qv[VB];
#pragma unroll
            for (int j = 0; j < VB; j++) qv[j] = __ldcs(v + i0 + lane + 32 * j);
#pragma unroll
            for (int j = 0; j < VB; j++) {
              const int i = i0 + lane + 32 * j;
              const uint4 q = qv[j];
              const InT *e = reinterpret_cast<const InT *>(&q);
              alignas(16) RecT r[PER];
#pragma unroll
              for (int k = 0; k < PER; k++) {
                const uint32_t key = (uint32_t)e[k];
                r[k] = (RecT)key;
                atomicAdd(&s.H[(key >> pbits) & (ndig - 1u)], 1u);
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
            }
          } else {  // ragged or unaligned tile (rare): element by element
            for (uint32_t i = lane; i < len; i += 32) {
              const uint32_t key = (uint32_t)keys[start + i];
              b0[i] = (RecT)key;
              atomicAdd(&s.H[(key >> pbits) & (ndig - 1u)], 1u);
            }
          }
        }
      }
      __syncwarp();
      digit_exscan(s.H, ndig, lane);  // H[d] = local start of digit d, H[ndig] = len
      __syncwarp();
      if constexpr (HAS_OUT) {  // key position = KB[digit] + final local position (A6)
        for (uint32_t d = lane; d < ndig; d += 32)
          s.KB[d] = rstart + Crow[d] + (s.BX[d + 1] - s.BX[d]) - s.H[d];
      }

      // ---- 2./3. per level: table, split (or ballot only), bitmap runs ----
      for (uint32_t k = 0; k < tau; k++) {
        const uint32_t nq = 1u << k, sh = tau - k;
        const bool do_split = HAS_OUT || (k + 1 < tau);
        const uint32_t bitsh = pbits + tau - 1u - k;
        const uint32_t bitmask = 1u << bitsh;
        const RecT *__restrict__ src = k == 0 ? src0 : s.buf[k & 1];
        RecT *__restrict__ dst = s.buf[(k + 1) & 1];
        constexpr uint32_t RB = sizeof(RecT);
        const uint32_t dstA = smem_u32(dst);
        const uint32_t full = len / (32 * U);
        if (do_split) {
          // split table T_k as destination byte addresses:
          //   T[2q] = &dst[O(gs)],  T[2q+1] = &dst[gm - O(gs)]
          const uint32_t per = (nq + 31) >> 5;
          const uint32_t lo = min(lane * per, nq), hi = min(lo + per, nq);
          uint32_t sum = 0;
          for (uint32_t q = lo; q < hi; q++) sum += s.H[(q + 1) << sh] - s.H[(2 * q + 1) << (sh - 1)];
          const uint32_t incl = warp_incl_scan(sum, lane);
          uint32_t O = incl - sum;
          for (uint32_t q = lo; q < hi; q++) {
            const uint32_t gm = s.H[(2 * q + 1) << (sh - 1)];
            s.T[2 * q] = (uint16_t)(dstA + RB * O);
            s.T[2 * q + 1] = (uint16_t)(dstA + RB * (gm - O));
            O += s.H[(q + 1) << sh] - gm;
          }
          // batches lying inside one class take the uniform path: FB[b] = class or NONE
          if (lane < (int)full) {
            const uint32_t x = (uint32_t)lane * (32 * U);
            uint32_t qlo = 0, qhi = nq;
            while (qhi - qlo > 1) {
              const uint32_t mid = (qlo + qhi) >> 1;
              if (s.H[mid << sh] <= x) qlo = mid;
              else qhi = mid;
            }
            s.FB[lane] = s.H[(qlo + 1) << sh] >= x + 32 * U ? (uint16_t)qlo : (uint16_t)0xffffu;
          }
        }
        __syncwarp();
        uint32_t Orun = 0;
        const uint32_t srcA = smem_u32(src) + lane * RB;
        const uint32_t TA = smem_u32(s.T);
        if (do_split) {
          for (uint32_t b = 0; b < full; b++) {
            const uint32_t cb = b * (32 * U);
            const uint32_t fq = s.FB[b];
            uint32_t r[U], m[U];
#pragma unroll
            for (int u = 0; u < U; u++) r[u] = lds<RecT>(srcA + (cb + u * 32) * RB);
#pragma unroll
            for (int u = 0; u < U; u++) m[u] = __ballot_sync(FULL, r[u] & bitmask);
            if (fq != 0xffffu) {  // one class: uniform destinations
              const uint32_t a0 = s.T[2 * fq], a1 = s.T[2 * fq + 1];
#pragma unroll
              for (int u = 0; u < U; u++) {
                const uint32_t O = Orun + __popc(m[u] & lt);
                const uint32_t Z = cb + u * 32 + lane - O;
                const uint32_t x1 = a1 + RB * O, x0 = a0 + RB * Z;
                sts<RecT>((r[u] & bitmask) ? x1 : x0, r[u]);
                Orun += __popc(m[u]);
              }
            } else {
              uint32_t t[U];
#pragma unroll
              for (int u = 0; u < U; u++) t[u] = lds<uint16_t>(TA + 2 * (r[u] >> bitsh));
#pragma unroll
              for (int u = 0; u < U; u++) {
                const uint32_t O = Orun + __popc(m[u] & lt);
                const uint32_t Z = cb + u * 32 + lane - O;
                sts<RecT>(t[u] + RB * ((r[u] & bitmask) ? O : Z), r[u]);
                Orun += __popc(m[u]);
              }
            }
            if (lane == 0) {
              uint4 *lb = reinterpret_cast<uint4 *>(&s.LB[b * U]);
              lb[0] = make_uint4(m[0], m[1], m[2], m[3]);
              lb[1] = make_uint4(m[4], m[5], m[6], m[7]);
            }
          }
        } else {
          for (uint32_t b = 0; b < full; b++) {
            const uint32_t cb = b * (32 * U);
            uint32_t m[U];
#pragma unroll
            for (int u = 0; u < U; u++) m[u] = __ballot_sync(FULL, lds<RecT>(srcA + (cb + u * 32) * RB) & bitmask);
            if (lane == 0) {
              uint4 *lb = reinterpret_cast<uint4 *>(&s.LB[b * U]);
              lb[0] = make_uint4(m[0], m[1], m[2], m[3]);
              lb[1] = make_uint4(m[4], m[5], m[6], m[7]);
            }
          }
        }
        for (uint32_t ci = full * U; ci < nch; ci++) {  // ragged tail, one chunk at a time
          const uint32_t pos = ci * 32 + lane;
          const bool valid = pos < len;
          const uint32_t r = valid ? (uint32_t)src[pos] : 0u;
          const bool P1 = valid && (r & bitmask);
          const uint32_t m = __ballot_sync(FULL, P1);
          if (lane == 0) s.LB[ci] = m;
          if (do_split) {
            const uint32_t O = Orun + __popc(m & lt);
            const uint32_t t = s.T[r >> bitsh];
            if (valid) sts<RecT>(t + RB * (P1 ? O : pos - O), r);
            Orun += __popc(m);
          }
        }
        __syncwarp();

        // ---- bitmap runs of level l0+k -> global (A2, A5) ----
        // (a) lane per run: edge words with carries; RO[q] = exclusive scan
        //     of the runs' interior word counts (kept in T, free after the split)
        uint64_t *B = p.bits + (uint64_t)(p.l0 + k) * p.wpl;
        uint16_t *RO = s.T;
        uint32_t Ni = 0;
        for (uint32_t q0 = 0; q0 < nq; q0 += 32) {
          const uint32_t q = q0 + lane;
          uint32_t ni = 0;
          if (q < nq) {
            const uint32_t ls = s.H[q << sh], cnt = s.H[(q + 1) << sh] - ls;
            if (cnt) {
              const uint32_t G = rstart + Crow[q << sh] + (s.BX[(q + 1) << sh] - s.BX[q << sh]);
              const uint32_t gw0 = G >> 6, gw1 = (uint32_t)(((uint64_t)G + cnt - 1) >> 6);
              ni = gw1 > gw0 + 1 ? gw1 - gw0 - 1 : 0u;
              run_ends(s, nq + q, B, p.n, G, ls, cnt);
            }
          }
          const uint32_t incl = warp_incl_scan(ni, lane);
          if (q < nq) RO[q] = (uint16_t)(Ni + incl - ni);
          Ni += __shfl_sync(FULL, incl, 31);
        }
        __syncwarp();
        // (b) interior words (Ni <= len/64): word j belongs to the last run q
        //     with RO[q] <= j (binary search), it is fully covered: plain store
        for (uint32_t j = lane; j < Ni; j += 32) {
          uint32_t lo = 0, hi = nq;
          while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (RO[mid] <= j) lo = mid;
            else hi = mid;
          }
          const uint32_t q = lo;
          const uint32_t ls = s.H[q << sh];
          const uint32_t G = rstart + Crow[q << sh] + (s.BX[(q + 1) << sh] - s.BX[q << sh]);
          const uint32_t gw = (G >> 6) + 1 + (j - RO[q]);
          B[gw] = extract64(s.LB, (int)(ls + gw * 64u - G), NW);
        }
        __syncwarp();
      }

      // ---- 4. narrowed keys, digit run by digit run (A6) ----
      if constexpr (HAS_OUT) {
        OutT *ko = reinterpret_cast<OutT *>(p.keys_out);
        const RecT *fin = s.buf[tau & 1];
#pragma unroll 4
        for (uint32_t i = lane; i < len; i += 32) {
          const uint32_t r = fin[i];
          ko[s.KB[r >> pbits] + i] = (OutT)(r & pmask);
        }
      }
      // ---- 5. running counts for the next tile of the chain ----
      for (uint32_t d = lane; d <= ndig; d += 32) s.BX[d] += s.H[d];
      __syncwarp();
    }
    // ---- chain end: flush carried words (shared with the next chain or row) ----
    for (uint32_t slot = 1 + lane; slot < ndig; slot += 32) {
      if (s.CF[slot] & CF_VALID) {
        const uint32_t k = 31 - __clz(slot), q = slot - (1u << k), sh = tau - k;
        const uint32_t Gend = rstart + Crow[q << sh] + (s.BX[(q + 1) << sh] - s.BX[q << sh]);
        uint64_t *B = p.bits + (uint64_t)(p.l0 + k) * p.wpl;
        atomicOr(reinterpret_cast<unsigned long long *>(&B[Gend >> 6]), s.CW[slot]);
      }
    }
    __syncwarp();
  }
}

}  // namespace wtb
