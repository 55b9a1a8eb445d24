// wt_group.cuh -- the hot kernel: one HBM pass builds tau consecutive levels
// l0 .. l0+tau-1 of the levelwise wavelet tree.
//
// Work unit: a warp tile of <= TW consecutive positions of S_{l0} inside one
// level-l0 node (its "row", key P).  Per tile:
//  1. load keys (16-byte vector loads), record = (digit << pbits) | payload,
//     digit = the tau level bits, payload = the bits below them; per-tile digit
//     histogram; publish it as the tile aggregate (decoupled lookback).
//  2. lookback over the preceding tiles of the same chain -> before[d] = the
//     number of same-node elements with digit d ahead of this tile; publish
//     the inclusive prefix at once.
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
//     words fully inside the run are stored, shared edge words are OR-ed
//     atomically into the zero-initialised bitmap (A5; only
//     the <= 2 boundary words of a run are shared).  Rank-directory block
//     counts are accumulated per 512-bit block (A7).  Keys narrowed to the
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
  const uint2 *claim;
  const uint32_t *total_tiles;
  const uint32_t *tile_base;
  const uint32_t *chain_begin;
  const uint32_t *chain_end;
  const uint32_t *chain_key;
  const uint32_t *chain_row;
  const uint32_t *chain_prefix;  // [chain][ndig] or null
  const uint32_t *Cseg;          // [row][ndig + 1]
  const uint32_t *row_start;
  uint32_t *tile_counter;
  uint32_t *state;               // [tile][NDIG]
  uint64_t *bits;
  uint64_t wpl;
  uint32_t *blkcnt;
  uint64_t bpl;
  const uint32_t *err;
};

template <typename RecT>
struct WarpSmem {
  alignas(16) RecT buf[2][TW];
  alignas(16) uint32_t LB[NCH];  // ballot words of the current local level
  uint32_t hist[NDIG];           // digit counts; then before[]; then key bases
  uint32_t Hl[NDIG + 1];         // exclusive scan of hist (local group starts)
  uint32_t BX[NDIG + 1];         // exclusive scan of before[]
  uint16_t T[NDIG];              // split table of the current level (2^(k+1) entries)
  uint32_t RG[NDIG / 2 + 1];     // run global start
};

constexpr int GROUP_WARPS = 2;
constexpr int U = 8;  // chunks per software-pipelined batch

// Write the bits of one run [G, G+cnt) <- local bits [ls, ls+cnt) of LB
// for words gw in [w_lo, w_hi) of the run; accumulate the rank-directory block
// counts of the words this lane writes (A7) into BC with one red per block.
__device__ __forceinline__ void put_run_words(const uint32_t *LB, uint64_t *B, uint32_t *BC, uint64_t n,
                                              uint32_t G, uint32_t ls, uint32_t cnt, uint64_t gw_begin,
                                              uint64_t gw_end) {
  const uint64_t gend = (uint64_t)G + cnt;
  uint32_t acc = 0;
  uint64_t cur_blk = gw_begin >> 3;
  for (uint64_t gw = gw_begin; gw < gw_end; gw++) {
    const uint64_t lo = gw * 64;
    const int base = (int)((int64_t)ls + (int64_t)lo - (int64_t)G);
    uint64_t val = extract64(LB, base, NCH);
    const uint64_t s0 = ((uint64_t)G > lo ? (uint64_t)G : lo) - lo;
    const uint64_t e0 = (gend < lo + 64 ? gend : lo + 64) - lo;
    const uint64_t mask = (e0 - s0 == 64) ? ~0ull : (((1ull << (e0 - s0)) - 1ull) << s0);
    val &= mask;
    const uint64_t hi_clip = (lo + 64 < n) ? lo + 64 : n;
    if ((uint64_t)G <= lo && gend >= hi_clip) B[gw] = val;
    else if (val) atomicOr(reinterpret_cast<unsigned long long *>(&B[gw]), (unsigned long long)val);
    if ((gw >> 3) != cur_blk) {
      if (acc) atomicAdd(&BC[cur_blk], acc);
      acc = 0;
      cur_blk = gw >> 3;
    }
    acc += (uint32_t)__popcll(val);
  }
  if (acc) atomicAdd(&BC[cur_blk], acc);
}

template <typename InT, typename RecT, typename OutT, bool HAS_OUT>
__global__ void __launch_bounds__(GROUP_WARPS * 32) k_group(GroupParams p) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WarpSmem<RecT> &ws = *reinterpret_cast<WarpSmem<RecT> *>(smem_raw + warp * sizeof(WarpSmem<RecT>));
  if (ld_relaxed(p.err)) return;
  const InT *keys = reinterpret_cast<const InT *>(p.keys_in);
  const uint32_t tau = p.tau, pbits = p.pbits;
  const uint32_t ndig = 1u << tau;
  const uint32_t pmask = (1u << pbits) - 1u;
  const uint32_t total_tiles = ld_relaxed(p.total_tiles);
  const uint32_t lt = lanemask_lt();

  while (true) {
    uint32_t t = 0;
    if (lane == 0) t = atomicAdd(p.tile_counter, 1u);
    t = __shfl_sync(FULL, t, 0);
    if (t >= total_tiles) break;

    // ---- tile geometry ----
    const uint2 cj = p.claim[t];
    const uint32_t ch = cj.x, j = cj.y;
    const uint32_t start = p.chain_begin[ch] + j * TW;
    const uint32_t rem = p.chain_end[ch] - start;
    const uint32_t len = rem < (uint32_t)TW ? rem : (uint32_t)TW;
    const uint32_t nch = (len + 31) >> 5;
    const uint32_t row = p.chain_row[ch];
    const uint32_t rstart = p.row_start[row];
    const uint32_t *Crow = p.Cseg + (uint64_t)row * (ndig + 1);
    uint32_t *st = p.state + (uint64_t)(p.tile_base[ch] + j) * NDIG;

    // ---- 1. load, records, histogram ----
    for (uint32_t d = lane; d < ndig; d += 32) ws.hist[d] = 0;
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
              atomicAdd(&ws.hist[dig], 1u);
            }
          }
        }
      }
    }
    __syncwarp();

    // ---- 2. publish + lookback (lane handles digits lane, lane+32, ...) ----
    constexpr int DPL = NDIG / 32;
    if (j == 0) {
      for (uint32_t d = lane; d < ndig; d += 32) {
        const uint32_t pre = p.chain_prefix ? p.chain_prefix[(uint64_t)ch * ndig + d] : 0u;
        st_relaxed(st + d, FLAG_INC | (pre + ws.hist[d]));
        ws.BX[d] = pre;  // before[d]
      }
    } else {
      for (uint32_t d = lane; d < ndig; d += 32) st_relaxed(st + d, FLAG_AGG | ws.hist[d]);
      uint32_t acc[DPL];
      uint32_t done = 0, need = 0;
#pragma unroll
      for (int i = 0; i < DPL; i++) {
        acc[i] = 0;
        if (lane + 32u * i < ndig) need |= 1u << i;
      }
      const uint32_t *pst = st;
      while (done != need) {
        pst -= NDIG;
        uint32_t v[DPL];
        while (true) {  // spin until the predecessor has published
          bool ready = true;
#pragma unroll
          for (int i = 0; i < DPL; i++) {
            v[i] = 0;
            if ((need & ~done) & (1u << i)) {
              v[i] = ld_relaxed(pst + lane + 32u * i);
              if ((v[i] & ~VAL_MASK) == 0) ready = false;
            }
          }
          if (ready) break;
        }
#pragma unroll
        for (int i = 0; i < DPL; i++) {
          if ((need & ~done) & (1u << i)) {
            acc[i] += v[i] & VAL_MASK;
            if ((v[i] & ~VAL_MASK) == FLAG_INC) done |= 1u << i;
          }
        }
      }
#pragma unroll
      for (int i = 0; i < DPL; i++) {
        const uint32_t d = lane + 32u * i;
        if (d < ndig) {
          st_relaxed(st + d, FLAG_INC | (acc[i] + ws.hist[d]));
          ws.BX[d] = acc[i];
        }
      }
    }
    __syncwarp();
    warp_exscan(ws.hist, ndig, ws.Hl, lane);
    for (uint32_t d = lane; d < ndig; d += 32) ws.hist[d] = ws.BX[d];  // hist <- before
    __syncwarp();
    warp_exscan(ws.hist, ndig, ws.BX, lane);

    // ---- 3. per level: table, split (or ballot only), bitmap runs ----
    for (uint32_t k = 0; k < tau; k++) {
      const uint32_t nq = 1u << k, sh = tau - k;
      const bool do_split = HAS_OUT || (k + 1 < tau);
      const uint32_t bitsh = pbits + tau - 1u - k;
      const RecT *__restrict__ src = ws.buf[k & 1];
      RecT *__restrict__ dst = ws.buf[(k + 1) & 1];
      // run descriptors of level l0+k (and the split table T_k)
      {
        const uint32_t per = (nq + 31) >> 5;
        const uint32_t lo = min(lane * per, nq), hi = min(lo + per, nq);
        uint32_t s = 0;
        for (uint32_t q = lo; q < hi; q++) s += ws.Hl[(2 * q + 2) << (sh - 1)] - ws.Hl[(2 * q + 1) << (sh - 1)];
        const uint32_t incl = warp_incl_scan(s, lane);
        uint32_t O = incl - s;
        for (uint32_t q = lo; q < hi; q++) {
          const uint32_t gs = ws.Hl[q << sh], ge = ws.Hl[(q + 1) << sh];
          const uint32_t ones = ws.Hl[(2 * q + 2) << (sh - 1)] - ws.Hl[(2 * q + 1) << (sh - 1)];
          ws.T[2 * q] = (uint16_t)O;                    // O(gs)
          ws.T[2 * q + 1] = (uint16_t)(ge - (O + ones));  // ge - O(ge)
          O += ones;
          (void)gs;
          ws.RG[q] = rstart + Crow[q << sh] + (ws.BX[(q + 1) << sh] - ws.BX[q << sh]);
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
            const uint32_t tag = r[u] >> bitsh;
            m[u] = __ballot_sync(FULL, tag & 1u);
            tb[u] = Tk[tag];
          }
          uint32_t pc[U], ob[U];
#pragma unroll
          for (int u = 0; u < U; u++) pc[u] = __popc(m[u]);
          // ones before chunk u of the batch: short dependency tree, not a chain
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
#pragma unroll
          for (int u = 0; u < U; u++) {
            const uint32_t Y = ob[u] + __popc(m[u] & lt);
            const uint32_t d = ((r[u] >> bitsh) & 1u) ? tb[u] + Y : tb[u] + (cbase + u * 32) - Y;
            dst[d] = (RecT)r[u];
          }
        } else {
#pragma unroll
          for (int u = 0; u < U; u++) m[u] = __ballot_sync(FULL, (r[u] >> bitsh) & 1u);
        }
        if (lane == 0) {
          uint4 *lb = reinterpret_cast<uint4 *>(&ws.LB[b * U]);
          lb[0] = make_uint4(m[0], m[1], m[2], m[3]);
          lb[1] = make_uint4(m[4], m[5], m[6], m[7]);
        }
      }
      for (uint32_t c = full * U; c < nch; c++) {  // ragged tail, one chunk at a time
        const uint32_t pos = c * 32 + lane;
        const bool valid = pos < len;
        const uint32_t r = valid ? (uint32_t)src[pos] : 0u;
        const uint32_t tag = r >> bitsh;
        const bool P1 = valid && (tag & 1u);
        const uint32_t m = __ballot_sync(FULL, P1);
        if (lane == 0) ws.LB[c] = m;
        if (do_split) {
          const uint32_t Y = Orun + __popc(m & lt);
          const uint32_t d = P1 ? Tk[tag] + Y : Tk[tag] + pos - Y;
          if (valid) dst[d] = (RecT)r;
          Orun += __popc(m);
        }
      }
      __syncwarp();
      // bitmap runs of level l0+k -> global (A2, A5) + rank block counts (A7)
      uint64_t *B = p.bits + (uint64_t)(p.l0 + k) * p.wpl;
      uint32_t *BC = p.blkcnt + (uint64_t)(p.l0 + k) * p.bpl;
      if (nq >= 32) {
        for (uint32_t q = lane; q < nq; q += 32) {  // one lane per run
          const uint32_t ls = ws.Hl[q << sh], cnt = ws.Hl[(q + 1) << sh] - ls;
          if (cnt) {
            const uint32_t G = ws.RG[q];
            put_run_words(ws.LB, B, BC, p.n, G, ls, cnt, G >> 6, (((uint64_t)G + cnt - 1) >> 6) + 1);
          }
        }
      } else {
        for (uint32_t q = 0; q < nq; q++) {  // lanes split a run's words
          const uint32_t ls = ws.Hl[q << sh], cnt = ws.Hl[(q + 1) << sh] - ls;
          if (!cnt) continue;
          const uint32_t G = ws.RG[q];
          const uint64_t w0 = G >> 6, w1 = (((uint64_t)G + cnt - 1) >> 6) + 1;
          const uint64_t nw = w1 - w0;
          const uint64_t per = (nw + 31) / 32;
          // lane takes a contiguous slice of words, aligned to 512-bit blocks when long
          uint64_t a = w0 + lane * per, e = a + per;
          if (a > w1) a = w1;
          if (e > w1) e = w1;
          if (a < e) put_run_words(ws.LB, B, BC, p.n, G, ls, cnt, a, e);
        }
      }
      __syncwarp();
    }
    const RecT *fin = ws.buf[tau & 1];

    // ---- 4. narrowed keys at their S_{l0+tau} position (A6) ----
    if constexpr (HAS_OUT) {
      OutT *ko = reinterpret_cast<OutT *>(p.keys_out);
      for (uint32_t d = lane; d < ndig; d += 32)
        ws.hist[d] = rstart + Crow[d] + ws.hist[d] - ws.Hl[d];  // key base per digit
      __syncwarp();
      for (uint32_t c0 = 0; c0 < nch; c0 += U) {
        uint32_t r[U], kb[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
          const uint32_t pos = (c0 + u) * 32 + lane;
          r[u] = pos < len ? (uint32_t)fin[pos] : 0u;
        }
#pragma unroll
        for (int u = 0; u < U; u++) kb[u] = ws.hist[r[u] >> pbits];
#pragma unroll
        for (int u = 0; u < U; u++) {
          const uint32_t pos = (c0 + u) * 32 + lane;
          if (pos < len) ko[kb[u] + pos] = (OutT)(r[u] & pmask);
        }
      }
      __syncwarp();
    }
  }
}

}  // namespace wtb
