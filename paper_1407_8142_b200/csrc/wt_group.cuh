// wt_group.cuh -- the hot kernel: one HBM pass builds tau consecutive levels
// l0 .. l0+tau-1 of the levelwise wavelet tree.
//
// Work unit: a chain (<= CH consecutive positions of S_{l0} inside one
// level-l0 node, its "row"), processed by one warp as a sequence of tiles of
// <= TW positions.  before[d] = the number of same-row elements with digit d
// ahead of the tile (chain prefix from the per-chain histograms, then a
// running sum).  Per tile:
//  1. load keys (16-byte vector loads), record = (digit << pbits) | payload,
//     digit = the tau level bits, payload = the bits below them; digit counts.
//  3. tau stable 1-bit splits in shared memory (Fig. 1 l.12-17): at
//     local level k the tile is in S_{l0+k} order; a warp ballot of the level
//     bit gives 32 bitmap bits in order (A2); an element's destination is
//        bit 0: O(gs) + (pos - O(pos))        bit 1: (ge - O(ge)) + O(pos)
//     where O(x) = ones before position x and [gs, ge) is its group (the
//     prefix sum X / X_s of Fig. 1 l.14 restated per group); the group terms
//     come from the tile digit histogram (table T_k), O(pos) from a running
//     popcount.  Chunks are processed in batches of 8 so that shared-memory
//     loads of a batch overlap.
//  4. global placement: level l0+k bits of prefix q form one run starting at
//        G = row_start + Cseg[row][q << (tau-k)] + sum_{d in q} before[d];
//     words fully inside the run are stored; the partial last word of a run is
//     carried to the next tile of the chain (runs of consecutive tiles are
//     adjacent), so only words shared with another chain or row are OR-ed
//     atomically into the zero-initialised bitmap (A5; at
//     most 2 shared words per node).  Keys narrowed to the
//     payload are written at their S_{l0+tau} position (A6; the short lists
//     of PAPER.md:26-34) for the next pass.
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
  // local mode (one tile per row; the row's own counts give its node starts)
  uint32_t nk;                     // levels l0+1 .. l0+nk get their nodes emitted here
  uint64_t rstride;
  const uint32_t *rowoff;          // [k-1][row] exclusive prefix of node counts
  const uint64_t *level_node_ptr;
  const uint32_t *row_key;
  uint32_t *node_key;
  uint32_t *node_start;
};

constexpr uint32_t NO_CARRY = 0xffffffffu;
constexpr uint32_t CARRY_SHARED = 0x80000000u;  // the word's low part belongs to another chain/run

template <typename RecT>
struct WarpSmem {
  alignas(16) RecT buf[2][TW];
  alignas(16) unsigned long long CW[NDIG];  // carried partial word per run (k,q): slot 2^k - 1 + q
  alignas(16) uint32_t LB[NCH];            // ballot words of the current local level
  uint32_t CI[NDIG];                       // carried word index | CARRY_SHARED, or NO_CARRY
  uint32_t hist2[NDIG / 2];                // digit counts as u16 pairs (<= TW < 2^16)
  uint32_t before[NDIG];                   // running same-row count ahead of the tile, per digit
  uint32_t BX[NDIG + 1];                   // exclusive scan of before[]
  uint32_t KB[NDIG];                       // per-digit base of the narrowed-key output
  uint32_t RG[NDIG / 2 + 1];               // run global start
  uint16_t Hl[NDIG + 2];                   // exclusive scan of the counts (local group starts)
  uint16_t T[NDIG];                        // split table of the current level
};

#ifndef WT_GROUP_WARPS
#define WT_GROUP_WARPS 2
#endif
constexpr int GROUP_WARPS = WT_GROUP_WARPS;
constexpr int U = 8;  // chunks per software-pipelined batch

__device__ __forceinline__ uint32_t hcount(const uint32_t *hist2, uint32_t d) {
  return (hist2[d >> 1] >> ((d & 1u) << 4)) & 0xffffu;
}

// Bits of run [G, G+cnt) (local bits [ls, ls+cnt) of LB) that fall in word gw.
__device__ __forceinline__ uint64_t run_word(const uint32_t *LB, uint32_t G, uint32_t ls, uint32_t cnt, uint64_t gw) {
  const uint64_t lo = gw * 64, gend = (uint64_t)G + cnt;
  uint64_t v = extract64(LB, (int)((int64_t)ls + (int64_t)lo - (int64_t)G), NCH);
  const uint64_t s0 = ((uint64_t)G > lo ? (uint64_t)G : lo) - lo;
  const uint64_t e0 = (gend < lo + 64 ? gend : lo + 64) - lo;
  const uint64_t mask = (e0 - s0 == 64) ? ~0ull : (((1ull << (e0 - s0)) - 1ull) << s0);
  return v & mask;
}

// First and last word of a run, with the carry of run slot `slot` (one lane).
template <typename RecT>
__device__ __forceinline__ void run_ends(WarpSmem<RecT> &ws, uint32_t slot, uint64_t *B, uint64_t n, uint32_t G,
                                         uint32_t ls, uint32_t cnt) {
  const uint64_t gw0 = G >> 6, gw1 = ((uint64_t)G + cnt - 1) >> 6;
  const uint64_t gend = (uint64_t)G + cnt;
  // first word
  uint64_t v = run_word(ws.LB, G, ls, cnt, gw0);
  bool shared;
  const uint32_t ci = ws.CI[slot];
  if (ci != NO_CARRY) {
    v |= ws.CW[slot];
    shared = (ci & CARRY_SHARED) != 0;
  } else {
    shared = (G & 63u) != 0;
  }
  const uint64_t end0 = (gw0 * 64 + 64 < n) ? gw0 * 64 + 64 : n;
  if (gw0 == gw1 && gend < end0) {  // the word stays open: carry it to the next tile
    ws.CW[slot] = v;
    ws.CI[slot] = (uint32_t)gw0 | (shared ? CARRY_SHARED : 0u);
    return;
  }
  if (shared) atomicOr(reinterpret_cast<unsigned long long *>(&B[gw0]), (unsigned long long)v);
  else B[gw0] = v;
  ws.CI[slot] = NO_CARRY;
  if (gw1 > gw0) {
    const uint64_t v1 = run_word(ws.LB, G, ls, cnt, gw1);
    const uint64_t end1 = (gw1 * 64 + 64 < n) ? gw1 * 64 + 64 : n;
    if (gend >= end1) {
      B[gw1] = v1;
    } else {
      ws.CW[slot] = v1;
      ws.CI[slot] = (uint32_t)gw1;
    }
  }
}

template <typename InT, typename RecT, typename OutT, bool HAS_OUT>
__global__ void __launch_bounds__(GROUP_WARPS * 32) k_group(GroupParams p) {
  constexpr bool LOCAL = false;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WarpSmem<RecT> &ws = *reinterpret_cast<WarpSmem<RecT> *>(smem_raw + warp * sizeof(WarpSmem<RecT>));
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
    const uint32_t *Crow = LOCAL ? nullptr : p.Cseg + (uint64_t)row * (ndig + 1);
    if (LOCAL && cend - cbeg > (uint32_t)TW) {  // not a one-tile row: the host falls back to chain mode
      if (lane == 0) atomicOr(p.err, 2u);
      continue;
    }
    if (LOCAL) {
      for (uint32_t d = lane; d < ndig; d += 32) ws.before[d] = 0;
    } else {
      const uint32_t cfirst = p.row_first[row];
      for (uint32_t d = lane; d < ndig; d += 32)
        ws.before[d] = p.E[(uint64_t)d * p.estride + c] - p.E[(uint64_t)d * p.estride + cfirst];
    }
    for (uint32_t i = lane; i < NDIG; i += 32) ws.CI[i] = NO_CARRY;
    __syncwarp();

    for (uint64_t start64 = cbeg; start64 < cend; start64 += TW) {
      const uint32_t start = (uint32_t)start64;
      const uint32_t rem = cend - start;
      const uint32_t len = rem < (uint32_t)TW ? rem : (uint32_t)TW;
      const uint32_t nch = (len + 31) >> 5;

      // ---- 1. load, records, digit counts ----
      for (uint32_t d = lane; d < NDIG / 2; d += 32) ws.hist2[d] = 0;
      __syncwarp();
      {
        RecT *b0 = ws.buf[0];
        constexpr int PER = 16 / sizeof(InT);
        const uintptr_t sb = reinterpret_cast<uintptr_t>(keys + start);
        const uintptr_t ab = sb & ~(uintptr_t)15;
        const int head = (int)((sb - ab) / sizeof(InT));
        const uint4 *v = reinterpret_cast<const uint4 *>(ab);
        const int nv = (head + (int)len + PER - 1) / PER;
        if (head == 0 && len == TW) {
#pragma unroll 4
          for (int i = lane; i < TW / PER; i += 32) {
            const uint4 q = __ldcs(v + i);
            const InT *e = reinterpret_cast<const InT *>(&q);
            alignas(16) RecT r[PER];
#pragma unroll
            for (int k = 0; k < PER; k++) {
              const uint32_t key = (uint32_t)e[k];
              const uint32_t dig = (key >> pbits) & (ndig - 1u);
              r[k] = (RecT)((dig << pbits) | (key & pmask));
              atomicAdd(&ws.hist2[dig >> 1], 1u << ((dig & 1u) << 4));
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
#pragma unroll 2
          for (int i = lane; i < nv; i += 32) {
            const uint4 q = __ldcs(v + i);
            const InT *e = reinterpret_cast<const InT *>(&q);
#pragma unroll
            for (int k = 0; k < PER; k++) {
              const int pos = i * PER + k - head;
              if (pos >= 0 && pos < (int)len) {
                const uint32_t key = (uint32_t)e[k];
                const uint32_t dig = (key >> pbits) & (ndig - 1u);
                b0[pos] = (RecT)((dig << pbits) | (key & pmask));
                atomicAdd(&ws.hist2[dig >> 1], 1u << ((dig & 1u) << 4));
              }
            }
          }
        }
      }
      __syncwarp();

      // ---- 2. Hl = exclusive scan of the counts, BX = exclusive scan of before ----
      {
        const uint32_t per = (ndig + 31) >> 5;
        const uint32_t lo = min(lane * per, ndig), hi = min(lo + per, ndig);
        uint32_t s1 = 0, s2 = 0;
        for (uint32_t d = lo; d < hi; d++) {
          s1 += hcount(ws.hist2, d);
          s2 += ws.before[d];
        }
        const uint32_t i1 = warp_incl_scan(s1, lane), i2 = warp_incl_scan(s2, lane);
        uint32_t r1 = i1 - s1, r2 = i2 - s2;
        for (uint32_t d = lo; d < hi; d++) {
          ws.Hl[d] = (uint16_t)r1;
          ws.BX[d] = r2;
          r1 += hcount(ws.hist2, d);
          r2 += ws.before[d];
        }
        if (lane == 31) {
          ws.Hl[ndig] = (uint16_t)i1;
          ws.BX[ndig] = i2;
        }
        __syncwarp();
      }

      if constexpr (HAS_OUT) {  // key position = KB[digit] + final local position (A6)
        for (uint32_t d = lane; d < ndig; d += 32)
          ws.KB[d] = LOCAL ? rstart : rstart + Crow[d] + ws.before[d] - ws.Hl[d];
        __syncwarp();
      }
      if constexpr (LOCAL) {  // A4: this row's nodes of levels l0+1 .. l0+nk (Fig. 1 l.18-20)
        const uint32_t P = p.row_key[row];
        for (uint32_t k = 1; k <= p.nk; k++) {
          const uint32_t nq = 1u << k, sh = tau - k;
          uint64_t j = p.level_node_ptr[p.l0 + k] + p.rowoff[(uint64_t)(k - 1) * p.rstride + row];
          for (uint32_t q0 = 0; q0 < nq; q0 += 32) {
            const uint32_t q = q0 + lane;
            const bool ne = q < nq && ws.Hl[(q + 1) << sh] > ws.Hl[q << sh];
            const uint32_t bm = __ballot_sync(FULL, ne);
            if (ne) {
              const uint64_t jj = j + __popc(bm & lt);
              p.node_key[jj] = (P << k) | q;
              p.node_start[jj] = rstart + ws.Hl[q << sh];
            }
            j += __popc(bm);
          }
        }
      }
      OutT *ko = reinterpret_cast<OutT *>(p.keys_out);

      // ---- 3. per level: table, split (or ballot only), bitmap runs ----
      for (uint32_t k = 0; k < tau; k++) {
        const uint32_t nq = 1u << k, sh = tau - k;
        const bool do_split = HAS_OUT || (k + 1 < tau);
        const bool to_global = HAS_OUT && (k + 1 == tau);  // last split scatters the keys to HBM
        const uint32_t bitmask = 1u << (pbits + tau - 1u - k);
        const uint32_t bitsh = pbits + tau - 1u - k;
        const RecT *__restrict__ src = ws.buf[k & 1];
        RecT *__restrict__ dst = ws.buf[(k + 1) & 1];
        {  // split table T_k and run starts of level l0+k
          const uint32_t per = (nq + 31) >> 5;
          const uint32_t lo = min(lane * per, nq), hi = min(lo + per, nq);
          uint32_t s = 0;
          for (uint32_t q = lo; q < hi; q++) s += ws.Hl[(2 * q + 2) << (sh - 1)] - ws.Hl[(2 * q + 1) << (sh - 1)];
          const uint32_t incl = warp_incl_scan(s, lane);
          uint32_t O = incl - s;
          for (uint32_t q = lo; q < hi; q++) {
            const uint32_t ge = ws.Hl[(q + 1) << sh];
            const uint32_t ones = ws.Hl[(2 * q + 2) << (sh - 1)] - ws.Hl[(2 * q + 1) << (sh - 1)];
            ws.T[2 * q] = (uint16_t)O;                    // O(gs)
            ws.T[2 * q + 1] = (uint16_t)(ge - (O + ones));  // ge - O(ge)
            O += ones;
            ws.RG[q] = LOCAL ? rstart + ws.Hl[q << sh]
                             : rstart + Crow[q << sh] + (ws.BX[(q + 1) << sh] - ws.BX[q << sh]);
          }
        }
        __syncwarp();
        const uint16_t *__restrict__ Tk = ws.T;
        uint32_t Orun = 0;
        const uint32_t full = len / (32 * U);
        for (uint32_t b = 0; b < full; b++) {
          const uint32_t cbase = b * (32 * U) + lane;
          uint32_t r[U], m[U];
#pragma unroll
          for (int u = 0; u < U; u++) r[u] = (uint32_t)src[cbase + u * 32];
          if (do_split) {
            uint32_t tb[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
              m[u] = __ballot_sync(FULL, r[u] & bitmask);
              tb[u] = Tk[r[u] >> bitsh];
            }
            uint32_t pc[U], ob[U];
#pragma unroll
            for (int u = 0; u < U; u++) pc[u] = __popc(m[u]);
            ob[0] = Orun;
            ob[1] = Orun + pc[0];
            const uint32_t p01 = pc[0] + pc[1], p23 = pc[2] + pc[3], p45 = pc[4] + pc[5];
            ob[2] = Orun + p01;
            ob[3] = ob[2] + pc[2];
            ob[4] = ob[2] + p23;
            ob[5] = ob[4] + pc[4];
            ob[6] = ob[4] + p45;
            ob[7] = ob[6] + pc[6];
            Orun = ob[7] + pc[7];
            if (to_global) {
              uint32_t kb[U];
#pragma unroll
              for (int u = 0; u < U; u++) kb[u] = ws.KB[r[u] >> pbits];
#pragma unroll
              for (int u = 0; u < U; u++) {
                const uint32_t Y = ob[u] + __popc(m[u] & lt);
                const uint32_t d = (r[u] & bitmask) ? tb[u] + Y : tb[u] + (cbase + u * 32) - Y;
                ko[kb[u] + d] = (OutT)(r[u] & pmask);
              }
            } else {
#pragma unroll
              for (int u = 0; u < U; u++) {
                const uint32_t Y = ob[u] + __popc(m[u] & lt);
                const uint32_t d = (r[u] & bitmask) ? tb[u] + Y : tb[u] + (cbase + u * 32) - Y;
                dst[d] = (RecT)r[u];
              }
            }
          } else {
#pragma unroll
            for (int u = 0; u < U; u++) m[u] = __ballot_sync(FULL, r[u] & bitmask);
          }
          if (lane == 0) {
            uint4 *lb = reinterpret_cast<uint4 *>(&ws.LB[b * U]);
            lb[0] = make_uint4(m[0], m[1], m[2], m[3]);
            lb[1] = make_uint4(m[4], m[5], m[6], m[7]);
          }
        }
        for (uint32_t ci = full * U; ci < nch; ci++) {  // ragged tail, one chunk at a time
          const uint32_t pos = ci * 32 + lane;
          const bool valid = pos < len;
          const uint32_t r = valid ? (uint32_t)src[pos] : 0u;
          const bool P1 = valid && (r & bitmask);
          const uint32_t m = __ballot_sync(FULL, P1);
          if (lane == 0) ws.LB[ci] = m;
          if (do_split) {
            const uint32_t Y = Orun + __popc(m & lt);
            const uint32_t tb = Tk[r >> bitsh];
            const uint32_t d = P1 ? tb + Y : tb + pos - Y;
            if (valid) {
              if (to_global) ko[ws.KB[r >> pbits] + d] = (OutT)(r & pmask);
              else dst[d] = (RecT)r;
            }
            Orun += __popc(m);
          }
        }
        __syncwarp();

        // ---- bitmap runs of level l0+k -> global (A2, A5) ----
        uint64_t *B = p.bits + (uint64_t)(p.l0 + k) * p.wpl;
        const uint32_t slot0 = nq - 1u;
        if (nq >= 32) {
          for (uint32_t q = lane; q < nq; q += 32) {  // one lane per run
            const uint32_t ls = ws.Hl[q << sh], cnt = ws.Hl[(q + 1) << sh] - ls;
            if (!cnt) continue;
            const uint32_t G = ws.RG[q];
            const uint64_t gw0 = G >> 6, gw1 = ((uint64_t)G + cnt - 1) >> 6;
            for (uint64_t gw = gw0 + 1; gw < gw1; gw++) B[gw] = run_word(ws.LB, G, ls, cnt, gw);
            run_ends(ws, slot0 + q, B, p.n, G, ls, cnt);
          }
        } else {
          for (uint32_t q = 0; q < nq; q++) {  // lanes split a run's interior words
            const uint32_t ls = ws.Hl[q << sh], cnt = ws.Hl[(q + 1) << sh] - ls;
            if (!cnt) continue;
            const uint32_t G = ws.RG[q];
            const uint64_t gw0 = G >> 6, gw1 = ((uint64_t)G + cnt - 1) >> 6;
            for (uint64_t gw = gw0 + 1 + lane; gw < gw1; gw += 32) B[gw] = run_word(ws.LB, G, ls, cnt, gw);
          }
          if (lane < nq) {  // first/last words of all runs in parallel (lane = run)
            const uint32_t q = lane;
            const uint32_t ls = ws.Hl[q << sh], cnt = ws.Hl[(q + 1) << sh] - ls;
            if (cnt) run_ends(ws, slot0 + q, B, p.n, ws.RG[q], ls, cnt);
          }
        }
        __syncwarp();
      }
      // ---- 5. running counts for the next tile of the chain ----
      for (uint32_t d = lane; d < ndig; d += 32) ws.before[d] += hcount(ws.hist2, d);
      __syncwarp();
    }
    // ---- chain end: flush carried words (shared with the next chain or row) ----
    for (uint32_t i = lane; i < (1u << tau) - 1u; i += 32) {
      const uint32_t ci = ws.CI[i];
      if (ci != NO_CARRY) {
        const uint32_t k = 31 - __clz(i + 1);  // slot i = 2^k - 1 + q
        uint64_t *B = p.bits + (uint64_t)(p.l0 + k) * p.wpl;
        atomicOr(reinterpret_cast<unsigned long long *>(&B[ci & ~CARRY_SHARED]), ws.CW[i]);
      }
    }
    __syncwarp();
  }
}

}  // namespace wtb
