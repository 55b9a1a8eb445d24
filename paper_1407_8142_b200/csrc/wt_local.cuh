// wt_local.cuh -- the deep-level pass for groups whose level-l0 nodes are small
// (local mode; config 5 levels 24..31: ~16.7M nodes of ~32 symbols).
//
// The subtree of a level-l0 node ("row") occupies the same contiguous range
// [row_start, row_end) at every deeper level (a node's
// children partition its symbols), so a row can be finished entirely inside
// one warp, with no global counts: the row's own digit histogram gives every
// node start below it.  A warp takes a BATCH of consecutive rows (those whose
// start lies in one TW-sized window of positions); the batch covers a
// contiguous range [A, B) at each of the tau levels, so each level's bits are
// assembled word by word as the rows arrive (lane k owns level k's word) and
// written with only the two edge words shared (A5).
//
// Per row:
//  * <= 32 symbols: register path, one symbol per lane, no data movement: the
//    position of a symbol at local level k is
//        pos_k = #{row symbols whose k-bit prefix is smaller}
//              + #{earlier row symbols with the same k-bit prefix}
//    (the stable order of Fig. 1 / PAPER.md:468-475), maintained with two lane
//    masks (lt: smaller prefix, eq: same prefix) updated by one ballot per
//    level; the level's bits are one warp OR-reduction of (bit << pos_k).
//  * 33..64 symbols: the same with two symbols per lane and 64-bit masks
//    (config 5: ~45 % of the level-24 nodes).  The next row's start, key and
//    first 64 symbols are loaded while the current row is processed.
//  * larger rows: the tile path of k_group (shared-memory stable splits with
//    the row's split tables), bits copied into the batch staging.
// Node tables (A4): pass 1 (LM_COUNT) counts each batch's nodes per level;
// after a scan over batches, pass 2 (LM_BUILD) writes them in (level, row,
// prefix) order, and pass 3 (LM_BIG) finishes the rows longer than LT that
// pass 2 deferred (their node offsets recorded, their bits OR-ed in).
#pragma once
#include "wt_common.cuh"

namespace wtb {

struct LocalParams {
  const void *keys_in;
  void *keys_out;
  uint64_t n;
  uint32_t l0, tau, pbits, nk;  // nodes of levels l0+1 .. l0+nk are emitted here
  uint32_t nbatch;
  const uint32_t *batch_first;  // first row of each batch, [nbatch + 1]
  const uint32_t *counts;       // [1] = rows
  const uint32_t *row_start;    // start of each row (level-l0 node)
  const uint32_t *row_key;      // its key (top-l0-bit prefix)
  uint32_t *batch_counter;
  uint32_t *batchcnt;           // [k-1][nbatch]: pass 1 counts, then exclusive offsets
  const uint64_t *level_node_ptr;
  uint32_t *node_key;
  uint32_t *node_start;
  uint64_t *bits;
  uint64_t wpl;
  uint32_t *err;
  uint32_t *defer;        // rows longer than LT left by the build pass: [row, nodeoff x 8] each
  uint32_t *defer_count;  // entries in defer
};

// Passes of the local mode: node counts, the build of every row up to LT
// symbols, and the build of the longer rows the build pass deferred (one
// "batch" per such row).  Splitting off the rare long rows keeps the build
// pass's per-warp shared memory small (occupancy: it is latency-bound).
enum : int { LM_COUNT = 0, LM_BUILD = 1, LM_BIG = 2 };
constexpr uint32_t LT = 1024;
constexpr uint32_t DEFER_W = 1 + TAU_MAX;  // u32 per deferred row

// Per-warp shared memory; the counting pass needs no records, staging or level bits.
template <typename RecT, int MODE>
struct LocalSmem {
  static constexpr uint32_t BUFN = MODE == LM_COUNT ? 1 : (MODE == LM_BUILD ? LT : TW);
  alignas(16) RecT buf[2][BUFN];
  unsigned long long acc[TAU_MAX];  // per level: the output word being assembled ...
  uint32_t accw[TAU_MAX];           // ... and its index (rows arrive in position order)
  alignas(16) uint32_t LB[MODE == LM_COUNT ? 1 : BUFN / 32];
  uint32_t hist2[NDIG / 2];
  uint32_t pres[NDIG / 32];  // counting pass: the digits present in a row (bit set)
  uint16_t Hl[NDIG + 2];
  uint16_t T[NDIG];
};

constexpr int LOCAL_WARPS = 2;

// Level-bit output of a batch [A, Bend): bits arrive in position order and are
// assembled word by word per level; a word that lies wholly inside the batch
// is stored, a word shared with a neighbouring batch (or with a row the build
// pass deferred) is OR-ed in (A5: only edge words are shared).
__device__ __forceinline__ void acc_flush(unsigned long long v, uint32_t gw, uint64_t *Bw, uint32_t A, uint32_t Bend,
                                          uint64_t n) {
  if (gw == 0xffffffffu) return;
  const uint64_t lo = (uint64_t)gw * 64, hi = lo + 64, hic = hi < n ? hi : n;
  if ((uint64_t)A <= lo && (uint64_t)Bend >= hic) Bw[gw] = v;
  else if (v) atomicOr(reinterpret_cast<unsigned long long *>(&Bw[gw]), v);
}

// append nb (<= 32) bits v (zero above nb) at global bit g of level k
template <typename WS>
__device__ __forceinline__ void acc_put(WS &ws, uint32_t k, uint32_t g, uint32_t v, uint32_t nb, uint64_t *Bw,
                                        uint32_t A, uint32_t Bend, uint64_t n) {
  if (!nb) return;
  const uint32_t gw = g >> 6, sh = g & 63;
  unsigned long long a = ws.acc[k];
  uint32_t w = ws.accw[k];
  if (gw != w) {
    acc_flush(a, w, Bw, A, Bend, n);
    a = 0;
    w = gw;
  }
  a |= (unsigned long long)v << sh;
  if (sh + nb > 64) {
    acc_flush(a, w, Bw, A, Bend, n);
    a = (unsigned long long)v >> (64 - sh);
    w = gw + 1;
  }
  ws.acc[k] = a;
  ws.accw[k] = w;
}

template <typename InT, typename RecT, typename OutT, bool HAS_OUT, int MODE>
__global__ void __launch_bounds__(LOCAL_WARPS * 32) k_local(LocalParams p) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  constexpr bool COUNT = MODE == LM_COUNT;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  LocalSmem<RecT, MODE> &ws =
      *reinterpret_cast<LocalSmem<RecT, MODE> *>(smem_raw + warp * sizeof(LocalSmem<RecT, MODE>));
  if (ld_relaxed(p.err)) return;
  const InT *keys = reinterpret_cast<const InT *>(p.keys_in);
  OutT *ko = reinterpret_cast<OutT *>(p.keys_out);
  const uint32_t tau = p.tau, pbits = p.pbits, ndig = 1u << tau;
  const uint32_t pmask = (1u << pbits) - 1u;
  const uint32_t nrows = p.counts[1];
  const uint32_t nk = p.nk;
  const uint32_t lt = lanemask_lt();

  while (true) {
    uint32_t b = 0;
    if (lane == 0) b = atomicAdd(p.batch_counter, 1u);
    b = __shfl_sync(FULL, b, 0);
    const uint32_t nb = MODE == LM_BIG ? ld_relaxed(p.defer_count) : p.nbatch;
    if (b >= nb) break;
    const uint32_t r0 = MODE == LM_BIG ? p.defer[(uint64_t)b * DEFER_W] : p.batch_first[b];
    const uint32_t r1 = MODE == LM_BIG ? r0 + 1 : p.batch_first[b + 1];
    if (r0 >= r1) {  // no row starts in this window: it contributes no nodes
      if (COUNT && lane < (int)p.nk) p.batchcnt[(uint64_t)lane * p.nbatch + b] = 0;
      continue;
    }
    const uint32_t A = p.row_start[r0];
    const uint32_t Bend = r1 < nrows ? p.row_start[r1] : (uint32_t)p.n;
    if (Bend - A > 2u * TW) {  // a row larger than TW: the host falls back to chain mode
      if (lane == 0) atomicOr(p.err, 2u);
      continue;
    }
    uint64_t *Bl = p.bits + (uint64_t)(p.l0 + (lane < (int)tau ? lane : 0)) * p.wpl;  // lane k: level l0+k
    if constexpr (!COUNT) {
      if (lane < (int)tau) {
        ws.acc[lane] = 0;
        ws.accw[lane] = 0xffffffffu;
      }
    }
    // running node offsets (lane kk holds level l0+1+kk), from the batch scan
    uint32_t nodeoff = 0;
    if (lane < (int)p.nk)
      nodeoff = COUNT ? 0u : (MODE == LM_BIG ? p.defer[(uint64_t)b * DEFER_W + 1 + lane]
                                             : p.batchcnt[(uint64_t)lane * p.nbatch + b]);
    // lane kk (< nk): the global index of the next node of level l0+1+kk
    uint64_t gn = 0;
    if (!COUNT && lane < (int)p.nk) gn = p.level_node_ptr[p.l0 + 1 + lane] + nodeoff;
    uint32_t gn_lo = (uint32_t)gn, gn_hi = (uint32_t)(gn >> 32);
    auto node_add = [&](uint32_t c) {  // lane kk: c more nodes of level l0+1+kk
      if (lane < (int)nk) {
        nodeoff += c;
        if (!COUNT) {
          gn += c;
          gn_lo = (uint32_t)gn;
          gn_hi = (uint32_t)(gn >> 32);
        }
      }
    };
    __syncwarp();

    // the next row's start, key and first 64 symbols are loaded one row ahead
    uint32_t rs_n = A, re_n = r0 + 1 < nrows ? p.row_start[r0 + 1] : (uint32_t)p.n, P_n = p.row_key[r0];
    uint32_t kA_n = (uint64_t)rs_n + lane < p.n ? (uint32_t)keys[(uint64_t)rs_n + lane] : 0u;
    uint32_t kB_n = (uint64_t)rs_n + 32 + lane < p.n ? (uint32_t)keys[(uint64_t)rs_n + 32 + lane] : 0u;
    for (uint32_t r = r0; r < r1; r++) {
      const uint32_t rs = rs_n, re = re_n, P = P_n, kA0 = kA_n, kB0 = kB_n;
      const uint32_t len = re - rs;
      if (r + 1 < r1) {
        rs_n = re;
        re_n = r + 2 < nrows ? p.row_start[r + 2] : (uint32_t)p.n;
        P_n = p.row_key[r + 1];
        kA_n = (uint64_t)rs_n + lane < p.n ? (uint32_t)keys[(uint64_t)rs_n + lane] : 0u;
        kB_n = (uint64_t)rs_n + 32 + lane < p.n ? (uint32_t)keys[(uint64_t)rs_n + 32 + lane] : 0u;
      }
      if (COUNT && len <= 64) {
        // ---------------- counting pass, rows of <= 64 symbols ----------------
        // nodes of level l0+k = the distinct k-bit digit prefixes of the row (Fig. 1
        // l.18-20): with the row's digit set as a bitmap (one shared-memory OR per
        // symbol), a k-bit prefix is a group of 2^(tau-k) consecutive bits, and the
        // count is the number of non-empty groups (bit folds + POPC per word)
        const uint32_t nw = (ndig + 31) >> 5;
        if (lane < (int)nw) ws.pres[lane] = 0;
        __syncwarp();
        const uint32_t dA = (kA0 >> pbits) & (ndig - 1u), dB = (kB0 >> pbits) & (ndig - 1u);
        if ((uint32_t)lane < len) atomicOr(&ws.pres[dA >> 5], 1u << (dA & 31u));
        if ((uint32_t)lane + 32u < len) atomicOr(&ws.pres[dB >> 5], 1u << (dB & 31u));
        __syncwarp();
        uint32_t y = lane < (int)nw ? ws.pres[lane] : 0u;
        const uint32_t wm = __ballot_sync(FULL, y != 0);  // non-empty 32-digit words
        // c_G = non-empty groups of 2^G digits, G = 0..5, per word; three 10-bit fields per sum
        uint32_t c012 = __popc(y);
        y |= y >> 1;
        c012 |= __popc(y & 0x55555555u) << 10;
        y |= y >> 2;
        c012 |= __popc(y & 0x11111111u) << 20;
        y |= y >> 4;
        uint32_t c345 = __popc(y & 0x01010101u);
        y |= y >> 8;
        c345 |= __popc(y & 0x00010001u) << 10;
        y |= y >> 16;
        c345 |= (y & 1u) << 20;
        c012 = __reduce_add_sync(FULL, c012);
        c345 = __reduce_add_sync(FULL, c345);
        // lane j: level l0+1+j, groups of 2^G digits with G = tau - 1 - j
        const int G = (int)tau - 1 - lane;
        uint32_t cnt = 0;
        if (G >= 0 && G <= 2) cnt = (c012 >> (10 * G)) & 1023u;
        else if (G >= 3 && G <= 5) cnt = (c345 >> (10 * (G - 3))) & 1023u;
        else if (G >= 6) {  // groups of 2^(G-5) words
          const uint32_t gw = 1u << (G - 5);
          uint32_t m = wm;
          for (uint32_t sh = 1; sh < gw; sh <<= 1) m |= m >> sh;
          cnt = __popc(m & (gw == 2 ? 0x55u : (gw == 4 ? 0x11u : 0x01u)));
        }
        node_add(cnt);
        __syncwarp();
        continue;
      }
      if (len <= 32) {
        // ---------------- register path ----------------
        // rd: the symbol's tau digit bits reversed, so that local level k's bit
        // (the (k+1)'st highest) is rd bit k; the loop is unrolled
        // over k (constant shifts, constant lane selects)
        const bool valid = (uint32_t)lane < len;
        const uint32_t key = valid ? kA0 : 0u;
        const uint32_t dig = (key >> pbits) & (ndig - 1u);
        const uint32_t rd = __brev(dig) >> (32u - tau);
        uint32_t eq = __ballot_sync(FULL, valid), ltm = 0;  // same prefix / smaller prefix (this row)
        uint32_t myw = 0;                                    // lane k: the row's word of level l0+k
        uint32_t cpk0 = 0, cpk1 = 0;                         // node counts of levels l0+1.., 8 bits each
#pragma unroll
        for (uint32_t k = 0; k < TAU_MAX; k++) {
          if (k >= tau) break;
          const uint32_t bit = (rd >> k) & 1u;
          const uint32_t m = __ballot_sync(FULL, valid && bit);
          if (!COUNT) {
            const uint32_t pos = __popc(ltm) + __popc(eq & lt);  // position at level l0+k
            const uint32_t word = __reduce_or_sync(FULL, valid && bit ? (1u << pos) : 0u);
            if (lane == (int)k) myw = word;
          }
          // refine to the (k+1)-bit prefix: same group and same bit; smaller if bit 0 vs my 1
          if (bit) {
            ltm |= eq & ~m;
            eq &= m;
          } else {
            eq &= ~m;
          }
          if (k + 1 <= nk) {  // nodes of level l0+k+1 = distinct (k+1)-bit prefixes
            const bool first = valid && (eq & lt) == 0;
            const uint32_t fm = __ballot_sync(FULL, first);
            if (!COUNT) {
              const uint64_t j0 = ((uint64_t)__shfl_sync(FULL, gn_hi, k) << 32) | __shfl_sync(FULL, gn_lo, k);
              if (first) {
                const uint64_t j = j0 + __popc(fm & ltm);  // leaders with a smaller prefix
                p.node_key[j] = (P << (k + 1)) | (dig >> (tau - 1u - k));
                p.node_start[j] = rs + __popc(ltm);
              }
            }
            if (k < 4) cpk0 += __popc(fm) << (8 * k);
            else cpk1 += __popc(fm) << (8 * (k - 4));
          }
        }
        node_add(((lane & 4) ? cpk1 : cpk0) >> (8 * (lane & 3)) & 0xffu);
        if (HAS_OUT && !COUNT && valid) ko[rs + __popc(ltm) + __popc(eq & lt)] = (OutT)(key & pmask);
        if (!COUNT && lane < (int)tau) acc_put(ws, lane, rs, myw, len, Bl, A, Bend, p.n);
        __syncwarp();
        continue;
      }
      if (len <= 64) {
        // ---------------- register path, two symbols per lane ----------------
        // symbols x = lane (A) and x = 32 + lane (B); 64-bit masks over the row:
        // eq = same prefix as x, ltm = smaller prefix than x, before = index < x.
        const bool vB = (uint32_t)lane + 32u < len;
        const uint32_t kA = kA0;
        const uint32_t kB = vB ? kB0 : 0u;
        const uint32_t dA = (kA >> pbits) & (ndig - 1u), dB = (kB >> pbits) & (ndig - 1u);
        const uint32_t rA = __brev(dA) >> (32u - tau), rB = __brev(dB) >> (32u - tau);
        const uint64_t valid64 = ((uint64_t)__ballot_sync(FULL, vB) << 32) | 0xffffffffull;
        const uint64_t befA = (uint64_t)lt, befB = 0xffffffffull | ((uint64_t)lt << 32);
        uint64_t eqA = valid64, eqB = valid64, ltA = 0, ltB = 0;
        uint32_t mylo = 0, myhi = 0;  // lane k: the row's words of level l0+k
        uint32_t cpk0 = 0, cpk1 = 0;
#pragma unroll
        for (uint32_t k = 0; k < TAU_MAX; k++) {
          if (k >= tau) break;
          const uint32_t bA = (rA >> k) & 1u, bB = (rB >> k) & 1u;
          const uint64_t M = ((uint64_t)__ballot_sync(FULL, vB && bB) << 32) | __ballot_sync(FULL, bA);
          if (!COUNT) {
            const uint32_t pA = __popcll(ltA) + __popcll(eqA & befA);
            const uint32_t pB = __popcll(ltB) + __popcll(eqB & befB);
            const uint32_t oA = bA ? 1u << (pA & 31u) : 0u, oB = (vB && bB) ? 1u << (pB & 31u) : 0u;
            const uint32_t lo = __reduce_or_sync(FULL, (pA < 32 ? oA : 0u) | (pB < 32 ? oB : 0u));
            const uint32_t hi = __reduce_or_sync(FULL, (pA < 32 ? 0u : oA) | (pB < 32 ? 0u : oB));
            if (lane == (int)k) { mylo = lo; myhi = hi; }
          }
          if (bA) { ltA |= eqA & ~M; eqA &= M; } else { eqA &= ~M; }
          if (bB) { ltB |= eqB & ~M; eqB &= M; } else { eqB &= ~M; }
          if (k + 1 <= nk) {  // nodes of level l0+k+1 = distinct (k+1)-bit prefixes
            const bool fA = (eqA & befA) == 0, fB = vB && (eqB & befB) == 0;
            const uint64_t F = ((uint64_t)__ballot_sync(FULL, fB) << 32) | __ballot_sync(FULL, fA);
            if (!COUNT) {
              const uint64_t j0 = ((uint64_t)__shfl_sync(FULL, gn_hi, k) << 32) | __shfl_sync(FULL, gn_lo, k);
              if (fA) {
                p.node_key[j0 + __popcll(F & ltA)] = (P << (k + 1)) | (dA >> (tau - 1u - k));
                p.node_start[j0 + __popcll(F & ltA)] = rs + __popcll(ltA);
              }
              if (fB) {
                p.node_key[j0 + __popcll(F & ltB)] = (P << (k + 1)) | (dB >> (tau - 1u - k));
                p.node_start[j0 + __popcll(F & ltB)] = rs + __popcll(ltB);
              }
            }
            if (k < 4) cpk0 += __popcll(F) << (8 * k);
            else cpk1 += __popcll(F) << (8 * (k - 4));
          }
        }
        node_add(((lane & 4) ? cpk1 : cpk0) >> (8 * (lane & 3)) & 0xffu);
        if (HAS_OUT && !COUNT) {
          ko[rs + __popcll(ltA) + __popcll(eqA & befA)] = (OutT)(kA & pmask);
          if (vB) ko[rs + __popcll(ltB) + __popcll(eqB & befB)] = (OutT)(kB & pmask);
        }
        if (!COUNT && lane < (int)tau) {
          acc_put(ws, lane, rs, mylo, 32, Bl, A, Bend, p.n);
          acc_put(ws, lane, rs + 32, myhi, len - 32, Bl, A, Bend, p.n);
        }
        __syncwarp();
        continue;
      }
      // ---------------- tile path (64 < len <= TW) ----------------
      if (len > (uint32_t)TW) {
        if (lane == 0) atomicOr(p.err, 2u);
        break;
      }
      // the build pass leaves rows longer than its buffers to the LM_BIG pass:
      // record where their nodes go, count them, emit nothing
      bool emit = !COUNT;
      if (MODE == LM_BUILD && len > LT) {
        uint32_t e = 0;
        if (lane == 0) e = atomicAdd(p.defer_count, 1u);
        e = __shfl_sync(FULL, e, 0);
        if (lane == 0) p.defer[(uint64_t)e * DEFER_W] = r;
        if (lane < (int)p.nk) p.defer[(uint64_t)e * DEFER_W + 1 + lane] = nodeoff;
        emit = false;
      }
      const uint32_t nch = (len + 31) >> 5;
      for (uint32_t d = lane; d < NDIG / 2; d += 32) ws.hist2[d] = 0;
      __syncwarp();
      for (uint32_t pos = lane; pos < len; pos += 32) {
        const uint32_t key = (uint32_t)keys[rs + pos];
        const uint32_t dig = (key >> pbits) & (ndig - 1u);
        if (!COUNT && emit) ws.buf[0][pos] = (RecT)((dig << pbits) | (key & pmask));
        atomicAdd(&ws.hist2[dig >> 1], 1u << ((dig & 1u) << 4));
      }
      __syncwarp();
      {  // Hl = exclusive scan of the row's digit counts
        const uint32_t per = (ndig + 31) >> 5;
        const uint32_t lo = min(lane * per, ndig), hi = min(lo + per, ndig);
        uint32_t s1 = 0;
        for (uint32_t d = lo; d < hi; d++) s1 += (ws.hist2[d >> 1] >> ((d & 1u) << 4)) & 0xffffu;
        const uint32_t i1 = warp_incl_scan(s1, lane);
        uint32_t r1v = i1 - s1;
        for (uint32_t d = lo; d < hi; d++) {
          ws.Hl[d] = (uint16_t)r1v;
          r1v += (ws.hist2[d >> 1] >> ((d & 1u) << 4)) & 0xffffu;
        }
        if (lane == 31) ws.Hl[ndig] = (uint16_t)i1;
        __syncwarp();
      }
      // nodes of levels l0+1 .. l0+nk (Fig. 1 l.18-20)
      for (uint32_t k = 1; k <= p.nk; k++) {
        const uint32_t nq = 1u << k, sh = tau - k;
        uint32_t base = __shfl_sync(FULL, nodeoff, k - 1);
        for (uint32_t q0 = 0; q0 < nq; q0 += 32) {
          const uint32_t q = q0 + lane;
          const bool ne = q < nq && ws.Hl[(q + 1) << sh] > ws.Hl[q << sh];
          const uint32_t bm = __ballot_sync(FULL, ne);
          if (emit && ne) {
            const uint64_t j = p.level_node_ptr[p.l0 + k] + base + __popc(bm & lt);
            p.node_key[j] = (P << k) | q;
            p.node_start[j] = rs + ws.Hl[q << sh];
          }
          base += __popc(bm);
        }
        if (lane == (int)(k - 1)) nodeoff = base;
      }
      if (!COUNT && lane < (int)nk) {  // keep the node cursors of the register paths in step
        gn = p.level_node_ptr[p.l0 + 1 + lane] + nodeoff;
        gn_lo = (uint32_t)gn;
        gn_hi = (uint32_t)(gn >> 32);
      }
      if (!COUNT && emit) {
      for (uint32_t k = 0; k < tau; k++) {
        const uint32_t nq = 1u << k, sh = tau - k;
        const bool do_split = HAS_OUT || (k + 1 < tau);
        const uint32_t bitmask = 1u << (pbits + tau - 1u - k);
        const uint32_t bitsh = pbits + tau - 1u - k;
        const RecT *src = ws.buf[k & 1];
        RecT *dst = ws.buf[(k + 1) & 1];
        {  // split table T_k of the row
          const uint32_t per = (nq + 31) >> 5;
          const uint32_t lo = min(lane * per, nq), hi = min(lo + per, nq);
          uint32_t sacc = 0;
          for (uint32_t q = lo; q < hi; q++) sacc += ws.Hl[(2 * q + 2) << (sh - 1)] - ws.Hl[(2 * q + 1) << (sh - 1)];
          const uint32_t incl = warp_incl_scan(sacc, lane);
          uint32_t O = incl - sacc;
          for (uint32_t q = lo; q < hi; q++) {
            const uint32_t ge = ws.Hl[(q + 1) << sh];
            const uint32_t ones = ws.Hl[(2 * q + 2) << (sh - 1)] - ws.Hl[(2 * q + 1) << (sh - 1)];
            ws.T[2 * q] = (uint16_t)O;
            ws.T[2 * q + 1] = (uint16_t)(ge - (O + ones));
            O += ones;
          }
        }
        __syncwarp();
        uint32_t Orun = 0;
        for (uint32_t ci = 0; ci < nch; ci++) {
          const uint32_t pos = ci * 32 + lane;
          const bool valid = pos < len;
          const uint32_t rr = valid ? (uint32_t)src[pos] : 0u;
          const bool P1 = valid && (rr & bitmask);
          const uint32_t m = __ballot_sync(FULL, P1);
          if (lane == 0) ws.LB[ci] = m;
          if (do_split) {
            const uint32_t Y = Orun + __popc(m & lt);
            const uint32_t tb = ws.T[rr >> bitsh];
            const uint32_t d = P1 ? tb + Y : tb + pos - Y;
            if (valid) {
              if (HAS_OUT && k + 1 == tau) ko[rs + d] = (OutT)(rr & pmask);
              else dst[d] = (RecT)rr;
            }
            Orun += __popc(m);
          }
        }
        __syncwarp();
        // the row's level bits are LB[0..len) in order: append them to level k's output
        if (lane == 0) {
          uint64_t *Bk = p.bits + (uint64_t)(p.l0 + k) * p.wpl;
          for (uint32_t ci = 0; ci < nch; ci++) {
            const uint32_t nb = min(32u, len - ci * 32);
            const uint32_t v = nb == 32 ? ws.LB[ci] : (ws.LB[ci] & ((1u << nb) - 1u));
            acc_put(ws, k, rs + ci * 32, v, nb, Bk, A, Bend, p.n);
          }
        }
        __syncwarp();
      }
      }
    }
    if (COUNT) {
      if (lane < (int)p.nk) p.batchcnt[(uint64_t)lane * p.nbatch + b] = nodeoff;
      continue;
    }
    __syncwarp();
    // ---- the last assembled word of each level ----
    if (lane < (int)tau) acc_flush(ws.acc[lane], ws.accw[lane], Bl, A, Bend, p.n);
    __syncwarp();
  }
}

// Batches: batch b = the rows whose start lies in [b*TW, (b+1)*TW).
// batch_first[b] = lower_bound(row_start, b*TW), b = 0..nbatch.
static __global__ void k_batches(const uint32_t *__restrict__ row_start, const uint32_t *__restrict__ counts,
                          uint32_t nbatch, uint32_t *__restrict__ batch_first, uint32_t *__restrict__ bcounts,
                          const uint32_t *err) {
  if (*err) return;
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b == 0) bcounts[1] = nbatch;  // "rows" of the batch-count scan
  if (b > nbatch) return;
  const uint32_t nr = counts[1];
  const uint64_t key = (uint64_t)b * TW;
  uint32_t lo = 0, hi = nr;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (row_start[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  batch_first[b] = b == nbatch ? nr : lo;
}

// Rows of a local-mode group = the non-empty nodes of level l0 (grid-stride).
static __global__ void k_rows_from_nodes(const uint64_t *__restrict__ level_node_ptr, const uint32_t *__restrict__ ncount,
                                  uint32_t l0, const uint32_t *__restrict__ node_key,
                                  const uint32_t *__restrict__ node_start, uint32_t *__restrict__ row_start,
                                  uint32_t *__restrict__ row_key, uint32_t *__restrict__ counts, const uint32_t *err) {
  if (*err) return;
  const uint64_t p0 = level_node_ptr[l0];
  const uint32_t nr = ncount[l0];
  if (blockIdx.x == 0 && threadIdx.x == 0) counts[1] = nr;
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < nr; r += gridDim.x * blockDim.x) {
    row_start[r] = node_start[p0 + r];
    row_key[r] = node_key[p0 + r];
  }
}

}  // namespace wtb
