// wt_group.cuh -- the hot kernel: one HBM pass builds tau consecutive levels
// l0 .. l0+tau-1 of the levelwise wavelet tree.
//
// Work unit: a chain (<= CH consecutive positions of S_{l0} inside one
// level-l0 node, its "row"), processed by one CTA of WPB warps as a sequence
// of tiles of <= TT positions.  BX[d] = exclusive prefix over digits of the
// same-row elements ahead of the tile (chain prefix from the per-chain
// histograms, then a running sum).  Per tile:
//  1. load keys (16-byte vector loads, warp w loads quarter w); the record is
//     the (narrowed) key itself: its top tau bits are the digit, the rest the
//     payload; digit counts H (shared-memory atomics), then H := exclusive
//     scan of H, so class q of local level k spans [H[q<<(tau-k)], H[(q+1)<<(tau-k)]).
//  2. tau stable 1-bit splits in shared memory (Fig. 1 l.12-17): at
//     local level k the tile is in S_{l0+k} order; a warp ballot of the level
//     bit gives 32 bitmap bits in order (A2); an element's destination is
//        bit 0: T[2q]   + (pos - O(pos))      T[2q]   = O(gs)
//        bit 1: T[2q+1] + O(pos)              T[2q+1] = gm - O(gs)
//     where O(x) = ones before position x (counted from the start of the
//     range being split), [gs, ge) the element's class q and gm the start of
//     its right child: the prefix sums X / X_s of Fig. 1 l.14 restated for all
//     classes of a range at once (T holds destination addresses).
//     Levels 0 .. J0-1 are split by the whole CTA (each warp a quarter; the
//     quarter's ones counts come from the load for level 0 and from a ballot
//     pass for level 1); from level J0 on, warp w owns class w of level J0 --
//     a contiguous range that contains all its descendants
//     -- and finishes the remaining levels of that range alone.
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
  const uint32_t *V;          // [chain][256]: same-row elements with digit d ahead of the chain (k_wgroup)
  const uint32_t *row_start;
  uint32_t *chain_counter;
  uint64_t *bits;
  uint64_t wpl;
  uint32_t *err;
  uint32_t *blkcnt;  // [level][bpl]: ones per 512-bit block, accumulated by k_wgroup (fused A7)
  uint64_t bpl;
};

#ifdef WT_PHASES
static __device__ unsigned long long g_ph[16];
#define PH_DECL                            \
  unsigned long long ph_t = clock64();     \
  unsigned long long ph_acc[12];           \
  for (int i = 0; i < 12; i++) ph_acc[i] = 0;
#define PH(i)                                           \
  do {                                                  \
    if (threadIdx.x == 0) {                             \
      const unsigned long long t_ = clock64();          \
      ph_acc[i] += t_ - ph_t;                           \
      ph_t = t_;                                        \
    }                                                   \
  } while (0)
#define PH_FLUSH \
  if (threadIdx.x == 0) for (int i = 0; i < 12; i++) atomicAdd(&g_ph[i], ph_acc[i]);
#else
#define PH_DECL
#define PH(i) \
  do {        \
  } while (0)
#define PH_FLUSH
#endif

constexpr int WPB = 4;  // warps per CTA
constexpr int J0 = 2;   // levels split by the whole CTA (log2 WPB)
#ifndef WT_GMINB
#define WT_GMINB 5
#endif
#ifndef WT_GTT
#define WT_GTT 8192
#endif
// tile width (positions per tile): WT_GTT * 2 bytes of records per buffer
template <typename RecT>
struct GroupTile {
  static constexpr int TT = sizeof(RecT) == 1 ? 2 * WT_GTT : (sizeof(RecT) == 2 ? WT_GTT : (WT_GTT / 2) / 1024 * 1024);
  static_assert(TT % (WPB * 256) == 0, "quarters are whole batches");
};

constexpr uint8_t CF_VALID = 1, CF_SHARED = 2;
constexpr int TRASH = NDIG + 2;  // histogram bin of the load cover's out-of-tile records
constexpr uint16_t FB_NONE = 0xffffu;
#ifndef WT_U
#define WT_U 8
#endif
// running ones count of a chunk: WT_CNT_REDUX=1 uses the warp reduction (a
// uniform result, off the MIO pipe that POPC shares with shared memory)
#ifndef WT_CNT_REDUX
#define WT_CNT_REDUX 0
#endif
__device__ __forceinline__ uint32_t chunk_ones(uint32_t m, bool P) {
#if WT_CNT_REDUX
  return __reduce_add_sync(0xffffffffu, P ? 1u : 0u);
#else
  return __popc(m);
#endif
}
constexpr int U = WT_U;  // chunks per software-pipelined batch

template <typename RecT, bool HAS_OUT>
struct GroupSmem {
  static constexpr int TT = GroupTile<RecT>::TT;
  static constexpr int NLB = TT / 32 + 8 * WPB;
  static constexpr int NFB = TT / 128 + 2 * WPB;  // batches of >= 4 chunks
  alignas(16) RecT buf[2][TT + 16 / sizeof(RecT)];  // records, ping-pong between levels (+ load head)
  alignas(16) uint32_t H[NDIG + 4];        // tile digit counts, then their exclusive scan (H[ndig] = len)
  alignas(16) uint32_t BX[NDIG + 4];       // exclusive prefix over digits of same-row elements ahead of the tile
  alignas(16) uint32_t CR[NDIG + 4];       // the chain's row: start of each digit (Cseg[row])
  alignas(16) unsigned long long CW[NDIG]; // carried partial word of run slot (1 << k) + q
  alignas(16) uint32_t LB[NLB];            // ballot words of the current level
  alignas(16) uint32_t KB[HAS_OUT ? NDIG : 4];  // per-digit base of the narrowed-key output
  alignas(16) uint16_t T[2 * NDIG];        // split tables (destination addresses); level k at [2^(k+1)-2, ..)
  alignas(16) uint16_t RO[WPB][NDIG / 4 + 8];  // per warp: exclusive scan of its runs' interior word counts
  alignas(16) uint16_t FB[NFB];            // per batch of 256 positions: its class if it lies in one
  alignas(16) uint8_t CF[NDIG];            // carry flags of each slot
  uint32_t onesW[WPB];                     // ones of the current level in each warp's quarter
  uint32_t chain;
};

// Bits of run [G, G+cnt) (local bits [ls, ls+cnt) of LB) that fall in global word gw.
__device__ __forceinline__ uint64_t run_word(const uint32_t *LB, int nw, uint32_t G, uint32_t ls, uint32_t cnt,
                                             uint32_t gw) {
  const uint64_t lo = (uint64_t)gw * 64, gend = (uint64_t)G + cnt;
  uint64_t v = extract64(LB, (int)((int64_t)ls + (int64_t)lo - (int64_t)G), nw);
  const uint32_t s0 = (uint64_t)G > lo ? (uint32_t)(G - lo) : 0u;
  const uint32_t e0 = gend < lo + 64 ? (uint32_t)(gend - lo) : 64u;
  const uint64_t mask = (e0 - s0 == 64) ? ~0ull : (((1ull << (e0 - s0)) - 1ull) << s0);
  return v & mask;
}

// First and last word of a run, with the carry of slot `slot` (one lane).
template <typename SM>
__device__ __forceinline__ void run_ends(SM &s, const uint32_t *LB, int nw, uint32_t slot, uint64_t *B, uint64_t n,
                                         uint32_t G, uint32_t ls, uint32_t cnt) {
  const uint32_t gw0 = G >> 6, gw1 = (uint32_t)(((uint64_t)G + cnt - 1) >> 6);
  const uint64_t gend = (uint64_t)G + cnt;
  uint64_t v = run_word(LB, nw, G, ls, cnt, gw0);
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
  WT_CHECK(gend <= n, 101);
  if (shared) atomicOr(reinterpret_cast<unsigned long long *>(&B[gw0]), (unsigned long long)v);
  else B[gw0] = v;
  s.CF[slot] = 0;
  if (gw1 > gw0) {
    const uint64_t v1 = run_word(LB, nw, G, ls, cnt, gw1);
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

// Split table of level k for classes [qa, qb) (one warp), destinations in dst:
//   T[2q] = &dst[O(gs_q)], T[2q+1] = &dst[gm_q - O(gs_q)], O counted from class qa.
// Each level has its own slice of s.T (warps run through levels independently).
__device__ __forceinline__ uint32_t table_off(uint32_t k) { return (2u << k) - 2u; }
template <typename SM>
__device__ __forceinline__ void build_table(SM &s, uint16_t *T, uint32_t qa, uint32_t qb, uint32_t sh, uint32_t dstA,
                                            uint32_t RB, int lane) {
  const uint32_t nq = qb - qa;
  const uint32_t per = (nq + 31) >> 5;
  const uint32_t lo = qa + min(lane * per, nq), hi = qa + min(lane * per + per, nq);
  uint32_t sum = 0;
  for (uint32_t q = lo; q < hi; q++) sum += s.H[(q + 1) << sh] - s.H[(2 * q + 1) << (sh - 1)];
  const uint32_t incl = warp_incl_scan(sum, lane);
  uint32_t O = incl - sum;
  for (uint32_t q = lo; q < hi; q++) {
    const uint32_t gm = s.H[(2 * q + 1) << (sh - 1)];
    T[2 * q] = (uint16_t)(dstA + RB * O);
    T[2 * q + 1] = (uint16_t)(dstA + RB * (gm - O));
    O += s.H[(q + 1) << sh] - gm;
  }
}

// Per batch of 256 positions of the range [A, A+wl): its class in [qa, qb) if
// the batch lies inside one class, else FB_NONE (one warp).
template <typename SM>
__device__ __forceinline__ void build_fb(SM &s, uint16_t *FB, uint32_t qa, uint32_t qb, uint32_t sh, uint32_t A,
                                         uint32_t wl, int lane) {
  const uint32_t nb = wl / (32 * U);
  if (wl < (qb - qa) * (32 * U)) {  // classes shorter than a batch on average: table path throughout
    for (uint32_t b = lane; b < nb; b += 32) FB[b] = FB_NONE;
    return;
  }
  for (uint32_t b = lane; b < nb; b += 32) {
    const uint32_t x = A + b * (32 * U);
    uint32_t qlo = qa, qhi = qb;
    while (qhi - qlo > 1) {
      const uint32_t mid = (qlo + qhi) >> 1;
      if (s.H[mid << sh] <= x) qlo = mid;
      else qhi = mid;
    }
    FB[b] = s.H[(qlo + 1) << sh] >= x + 32 * U ? (uint16_t)qlo : FB_NONE;
  }
}

// One warp splits positions [A, A+wl) of level k (src -> dst through T),
// writing the level's ballot words to LB[0 ..) (bit x = position A + x; LB is
// 16-byte aligned) when STORE_LB; Orun starts at Obase (ones before A in the
// counted range).
template <typename RecT, bool DO_SPLIT, bool STORE_LB>
__device__ __forceinline__ uint32_t split_range(const uint16_t *T, const uint16_t *FB, uint32_t *LB, uint32_t srcA,
                                            uint32_t A, uint32_t wl, uint32_t Obase, uint32_t bitsh, int lane,
                                            uint32_t lt) {
  constexpr uint32_t RB = sizeof(RecT);
  uint32_t bitmask = 1u << bitsh;
  asm("" : "+r"(bitmask));  // opaque: test the bit with one LOP3 instead of shift+mask+compare
  // opaque copies: keep these in registers instead of recomputing them from
  // special registers / kernel parameters inside the loop
  uint32_t TA = smem_u32(T), LA = smem_u32(LB), Al = A + lane;
  asm("" : "+r"(TA), "+r"(LA), "+r"(Al), "+r"(bitsh));
  const uint32_t sA = srcA + Al * RB;
  uint32_t Orun = Obase;
  const uint32_t full = wl / (32 * U);
  for (uint32_t b = 0; b < full; b++) {
    const uint32_t cb = b * (32 * U);
    uint32_t r[U], m[U];
#pragma unroll
    for (int u = 0; u < U; u++) r[u] = lds<RecT>(sA + (cb + u * 32) * RB);
    if constexpr (DO_SPLIT) {
      const uint32_t fq = FB[b];
      const uint32_t pb = Al + cb;
      if (fq != FB_NONE) {  // one class: uniform destinations
        const uint32_t a01 = lds<uint32_t>(TA + 4 * fq);
        const uint32_t a0 = __byte_perm(a01, 0, 0x4410), a1 = __byte_perm(a01, 0, 0x4432);
#pragma unroll
        for (int u = 0; u < U; u++) {
          const bool P = (r[u] & bitmask) != 0;
          m[u] = __ballot_sync(FULL, P);
          const uint32_t O = Orun + __popc(m[u] & lt);
          const uint32_t Z = pb + u * 32 - O;
          sts<RecT>(P ? a1 + RB * O : a0 + RB * Z, r[u]);
          Orun += chunk_ones(m[u], P);
        }
      } else {
        uint32_t t[U];
#pragma unroll
        for (int u = 0; u < U; u++) t[u] = lds<uint16_t>(TA + 2 * (r[u] >> bitsh));
#pragma unroll
        for (int u = 0; u < U; u++) {
          const bool P = (r[u] & bitmask) != 0;
          m[u] = __ballot_sync(FULL, P);
          const uint32_t O = Orun + __popc(m[u] & lt);
          const uint32_t Z = pb + u * 32 - O;
          sts<RecT>(t[u] + RB * (P ? O : Z), r[u]);
          Orun += chunk_ones(m[u], P);
        }
      }
    } else {
#pragma unroll
      for (int u = 0; u < U; u++) {
        m[u] = __ballot_sync(FULL, r[u] & bitmask);
        Orun += __popc(m[u]);
      }
    }
    if (STORE_LB && lane == 0) {
#pragma unroll
      for (int u = 0; u < U; u += 4) sts_v4(LA + b * (4 * U) + 4 * u, m[u], m[u + 1], m[u + 2], m[u + 3]);
    }
  }
  const uint32_t nch = (wl + 31) >> 5;
  for (uint32_t ci = full * U; ci < nch; ci++) {  // ragged tail, one chunk at a time
    const uint32_t x = ci * 32 + lane;
    const bool valid = x < wl;
    const uint32_t r = valid ? lds<RecT>(sA + ci * 32 * RB) : 0u;
    const bool P1 = valid && (r & bitmask);
    const uint32_t m = __ballot_sync(FULL, P1);
    if (STORE_LB && lane == 0) LB[ci] = m;
    if constexpr (DO_SPLIT) {
      const uint32_t O = Orun + __popc(m & lt);
      const uint32_t t = lds<uint16_t>(TA + 2 * (r >> bitsh));
      if (valid) sts<RecT>(t + RB * (P1 ? O : A + x - O), r);
    }
    Orun += __popc(m);
  }
  return Orun - Obase;
}

// Runs of level k for classes [qa, qb): bits of class q are LB bits
// [H[q<<sh] - A, ...).  Edge words by the lanes of the edge warp (lane per
// run); interior words by a team of nthr threads (thread index tid0), after
// `sync` publishes RO (exclusive scan of the runs' interior word counts).
template <typename SM, typename Sync>
__device__ __forceinline__ void emit_runs(SM &s, uint16_t *RO, const uint32_t *LB, int nw, uint32_t k, uint32_t qa,
                                          uint32_t qb, uint32_t sh, uint32_t A, uint32_t rstart, uint64_t *B,
                                          uint64_t n, bool edge_warp, int lane, int tid0, int nthr, Sync sync) {
  const uint32_t nq = qb - qa;
  if (edge_warp) {
    uint32_t Ni = 0;
    for (uint32_t j0 = 0; j0 < nq; j0 += 32) {
      const uint32_t q = qa + j0 + lane;
      uint32_t ni = 0;
      if (q < qb) {
        const uint32_t ls = s.H[q << sh] - A, cnt = s.H[(q + 1) << sh] - s.H[q << sh];
        if (cnt) {
          const uint32_t G = rstart + s.CR[q << sh] + (s.BX[(q + 1) << sh] - s.BX[q << sh]);
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
    const uint32_t ls = s.H[q << sh] - A;
    const uint32_t G = rstart + s.CR[q << sh] + (s.BX[(q + 1) << sh] - s.BX[q << sh]);
    const uint32_t gw = (G >> 6) + 1 + (j - RO[lo]);
    WT_CHECK((uint64_t)gw * 64 + 64 <= n, 102);
    WT_CHECK(ls + gw * 64u - G + 64 <= (uint32_t)nw * 32u, 103);
    B[gw] = extract64(LB, (int)(ls + gw * 64u - G), nw);
  }
}

template <typename InT, typename RecT, typename OutT, bool HAS_OUT>
__global__ void __launch_bounds__(WPB * 32, WT_GMINB) k_group(GroupParams p) {
  using SM = GroupSmem<RecT, HAS_OUT>;
  constexpr int TT = SM::TT;
  constexpr int QL = TT / WPB;  // quarter length
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
  const uint32_t jc = tau < (uint32_t)J0 ? tau : (uint32_t)J0;  // levels split by the whole CTA
  auto csync = [] { __syncthreads(); };
  auto wsync = [] { __syncwarp(); };
  PH_DECL

  while (true) {
    if (tid == 0) s.chain = atomicAdd(p.chain_counter, 1u);
    __syncthreads();
    const uint32_t c = s.chain;
    if (c >= nchains) break;

    // ---- chain geometry and its starting counts ----
    const uint32_t row = p.chain_row[c];
    const uint32_t cbeg = p.chain_begin[c], cend = p.chain_end[c];
    const uint32_t rstart = p.row_start[row];
    {
      const uint32_t *Cg = p.Cseg + (uint64_t)row * (ndig + 1);
      for (uint32_t d = tid; d <= ndig; d += WPB * 32) s.CR[d] = Cg[d];
      const uint32_t cfirst = p.row_first[row];
      for (uint32_t d = tid; d < ndig; d += WPB * 32)
        s.BX[d] = p.E[(uint64_t)d * p.estride + c] - p.E[(uint64_t)d * p.estride + cfirst];
      for (uint32_t i = tid; i < NDIG / 4; i += WPB * 32) reinterpret_cast<uint32_t *>(s.CF)[i] = 0u;
      __syncthreads();
      if (warp == 0) digit_exscan(s.BX, ndig, lane);
    }

    for (uint64_t start64 = cbeg; start64 < cend; start64 += TT) {  // 64-bit: cend may be near 2^32
      const uint32_t start = (uint32_t)start64;
      PH(0);
      const uint32_t rem = cend - start;
      const uint32_t len = rem < (uint32_t)TT ? rem : (uint32_t)TT;
      WT_CHECK(cend <= p.n && cbeg <= cend, 108);
      for (uint32_t d = tid; d < NDIG; d += WPB * 32) s.H[d] = 0u;
      __syncthreads();

      // ---- 1. load (warp w: quarter [qlo, qhi)), records, digit counts,
      //         ones of level l0 in the quarter ----
      const uint32_t qlo = min((uint32_t)(warp * QL), len), qhi = min((uint32_t)((warp + 1) * QL), len);
      const uint32_t b0bit = pbits + tau - 1u;  // level-l0 bit of a key
      uint32_t ones0 = 0;
      // the level-l0 bit of every InT lane of a 32-bit word (records = keys in the copy path)
      const uint32_t onesmask = (sizeof(InT) == 1 ? 0x01010101u : (sizeof(InT) == 2 ? 0x00010001u : 1u)) << b0bit;
      const bool full_digit = sizeof(InT) == 1 && pbits == 0 && ndig == 256;
      uint32_t head0;
      {
        constexpr int PER = 16 / sizeof(InT);
        const uintptr_t sb = reinterpret_cast<uintptr_t>(keys + start);
        const uintptr_t ab = sb & ~(uintptr_t)15;
        const int head = (int)((sb - ab) / sizeof(InT));
        const uint4 *v = reinterpret_cast<const uint4 *>(ab);
        RecT *b0 = s.buf[0];
        if constexpr (sizeof(InT) == sizeof(RecT)) {
          // records are the keys: copy the aligned cover; the tile starts
          // `head` records into buf[0]
          head0 = (uint32_t)head;
          const int i_lo = (head + (int)qlo) / PER, i_hi = (head + (int)qhi + PER - 1) / PER;
          constexpr int VB = 8;
          for (int i0 = i_lo; i0 < i_hi; i0 += 32 * VB) {
            uint4 q[VB];
#pragma unroll
            for (int j = 0; j < VB; j++) {
              const int i = i0 + lane + 32 * j;
              if (i < i_hi) q[j] = __ldcs(v + i);
            }
#pragma unroll
            for (int j = 0; j < VB; j++) {
              const int i = i0 + lane + 32 * j;
              if (i < i_hi) {
                *reinterpret_cast<uint4 *>(b0 + i * PER) = q[j];
                const InT *e = reinterpret_cast<const InT *>(&q[j]);
                const int p0 = i * PER - head;
                if (p0 >= (int)qlo && p0 + PER <= (int)qhi) {
                  if (full_digit) {  // the record is the digit (u8 keys, last group): no shift or mask
#pragma unroll
                    for (int k = 0; k < PER; k++) atomicAdd(&s.H[(uint32_t)e[k]], 1u);
                  } else {
#pragma unroll
                    for (int k = 0; k < PER; k++) atomicAdd(&s.H[((uint32_t)e[k] >> pbits) & (ndig - 1u)], 1u);
                  }
                  // level-l0 ones of the 16 bytes: one masked popcount per 32-bit word
                  ones0 += __popc(q[j].x & onesmask) + __popc(q[j].y & onesmask) + __popc(q[j].z & onesmask) +
                           __popc(q[j].w & onesmask);
                } else {
#pragma unroll
                  for (int k = 0; k < PER; k++) {
                    const bool in = (unsigned)(p0 + k - (int)qlo) < qhi - qlo;
                    atomicAdd(&s.H[in ? (((uint32_t)e[k] >> pbits) & (ndig - 1u)) : (uint32_t)TRASH], 1u);
                    ones0 += in ? (((uint32_t)e[k] >> b0bit) & 1u) : 0u;
                  }
                }
              }
            }
          }
        } else {
          head0 = 0;
          if (head == 0 && len == (uint32_t)TT) {
            constexpr int VB = 8;
            const int i_lo = (int)qlo / PER, i_hi = (int)qhi / PER;
            for (int i0 = i_lo; i0 < i_hi; i0 += 32 * VB) {
              uint4 qv[VB];
#pragma unroll
              for (int j = 0; j < VB; j++) {
                const int i = i0 + lane + 32 * j;
                if (i < i_hi) qv[j] = __ldcs(v + i);
              }
#pragma unroll
              for (int j = 0; j < VB; j++) {
                const int i = i0 + lane + 32 * j;
                if (i < i_hi) {
                  const InT *e = reinterpret_cast<const InT *>(&qv[j]);
                  alignas(16) RecT r[PER];
#pragma unroll
                  for (int k = 0; k < PER; k++) {
                    const uint32_t key = (uint32_t)e[k];
                    r[k] = (RecT)key;
                    atomicAdd(&s.H[(key >> pbits) & (ndig - 1u)], 1u);
                    ones0 += (key >> b0bit) & 1u;
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
            }
          } else {  // ragged or unaligned tile (rare): element by element
            for (uint32_t i = qlo + lane; i < qhi; i += 32) {
              const uint32_t key = (uint32_t)keys[start + i];
              b0[i] = (RecT)key;
              atomicAdd(&s.H[(key >> pbits) & (ndig - 1u)], 1u);
              ones0 += (key >> b0bit) & 1u;
            }
          }
        }
      }
      {
        const uint32_t w1 = __reduce_add_sync(FULL, ones0);
        if (lane == 0) s.onesW[warp] = w1;
      }
      __syncthreads();
      PH(1);
      if (warp == 0) {
        digit_exscan(s.H, ndig, lane);  // H[d] = local start of digit d, H[ndig] = len
        __syncwarp();
        WT_CHECK(s.H[ndig] == len, 109);
        WT_CHECK(s.BX[ndig] + len <= p.n, 110);
        if constexpr (HAS_OUT) {  // key position = KB[digit] + final local position (A6)
          for (uint32_t d = lane; d < ndig; d += 32)
            s.KB[d] = rstart + s.CR[d] + (s.BX[d + 1] - s.BX[d]) - s.H[d];
        }
      }
      __syncthreads();
      PH(2);

      // ---- 2a. levels l0 .. l0+jc-1: the CTA splits the whole tile ----
      for (uint32_t k = 0; k < jc; k++) {
        const uint32_t nq = 1u << k, sh = tau - k;
        const bool do_split = HAS_OUT || (k + 1 < tau);
        const uint32_t bitsh = pbits + tau - 1u - k;
        const uint32_t srcA = smem_u32(s.buf[k & 1]) + (k == 0 ? head0 * RB : 0u);
        const uint32_t dstA = smem_u32(s.buf[(k + 1) & 1]);
        uint32_t *LBq = s.LB + qlo / 32;
        uint16_t *FBq = s.FB + warp * (QL / (32 * U));
        if (k > 0) {  // ones of the quarter at this level: a ballot pass (also the level's bitmap words)
          const uint32_t ones =
              split_range<RecT, false, true>(s.T, FBq, LBq, srcA, qlo, qhi - qlo, 0, bitsh, lane, lt);
          if (lane == 0) s.onesW[warp] = ones;
        }
        if (do_split && warp == 0) build_table(s, s.T + table_off(k), 0, nq, sh, dstA, RB, lane);
        if (do_split) build_fb(s, FBq, 0, nq, sh, qlo, qhi - qlo, lane);
        __syncthreads();
        uint32_t Obase = 0;
        for (int w = 0; w < warp; w++) Obase += s.onesW[w];
        if (do_split) {
          if (k == 0) split_range<RecT, true, true>(s.T + table_off(k), FBq, LBq, srcA, qlo, qhi - qlo, Obase, bitsh, lane, lt);
          else split_range<RecT, true, false>(s.T + table_off(k), FBq, LBq, srcA, qlo, qhi - qlo, Obase, bitsh, lane, lt);
        } else if (k == 0) {
          split_range<RecT, false, true>(s.T + table_off(k), FBq, LBq, srcA, qlo, qhi - qlo, Obase, bitsh, lane, lt);
        }
        __syncthreads();
        uint64_t *B = p.bits + (uint64_t)(p.l0 + k) * p.wpl;
        emit_runs(s, s.RO[0], s.LB, SM::NLB, k, 0, nq, sh, 0, rstart, B, p.n, warp == 0, lane, tid, WPB * 32,
                  csync);
        __syncthreads();
        PH(3 + (k > 0));
      }

      // ---- 2b. levels l0+jc .. l0+tau-1: warp w finishes class w of level l0+jc ----
      if (tau > jc) {
        const uint32_t shJ = tau - jc;
        const uint32_t A = s.H[(uint32_t)warp << shJ], wl = s.H[(uint32_t)(warp + 1) << shJ] - A;
        // this warp's slices of the LB / FB pools (prefix over the warps before it)
        uint32_t lbo = 0, fbo = 0;
        for (int w = 0; w < warp; w++) {
          const uint32_t l = s.H[(uint32_t)(w + 1) << shJ] - s.H[(uint32_t)w << shJ];
          lbo += ((l + 127) / 128) * 4;  // 16-byte aligned slices
          fbo += l / (32 * U);
        }
        uint32_t *LBw = s.LB + lbo;
        uint16_t *FBw = s.FB + fbo;
        for (uint32_t k = jc; k < tau && wl; k++) {
          const uint32_t sh = tau - k, kk = k - jc;
          const uint32_t qa = (uint32_t)warp << kk, qb = (uint32_t)(warp + 1) << kk;
          const bool do_split = HAS_OUT || (k + 1 < tau);
          const uint32_t bitsh = pbits + tau - 1u - k;
          const uint32_t srcA = smem_u32(s.buf[k & 1]);
          const uint32_t dstA = smem_u32(s.buf[(k + 1) & 1]);
          if (do_split) {
            build_table(s, s.T + table_off(k), qa, qb, sh, dstA, RB, lane);
            build_fb(s, FBw, qa, qb, sh, A, wl, lane);
            __syncwarp();
            PH(5);
            split_range<RecT, true, true>(s.T + table_off(k), FBw, LBw, srcA, A, wl, 0, bitsh, lane, lt);
          } else {
            split_range<RecT, false, true>(s.T + table_off(k), FBw, LBw, srcA, A, wl, 0, bitsh, lane, lt);
          }
          __syncwarp();
          PH(6);
          uint64_t *B = p.bits + (uint64_t)(p.l0 + k) * p.wpl;
          emit_runs(s, s.RO[warp], LBw, (int)((wl + 31) / 32), k, qa, qb, sh, A, rstart, B, p.n, true, lane, lane,
                    32, wsync);
          __syncwarp();
          PH(7);
        }
      }
      __syncthreads();
      PH(8);

      // ---- 3. narrowed keys, digit run by digit run (A6) ----
      if constexpr (HAS_OUT) {
        OutT *ko = reinterpret_cast<OutT *>(p.keys_out);
        const RecT *fin = s.buf[tau & 1];
#pragma unroll 4
        for (uint32_t i = tid; i < len; i += WPB * 32) {
          const uint32_t r = fin[i];
          WT_CHECK(s.KB[r >> pbits] + i < p.n, 104);
          ko[s.KB[r >> pbits] + i] = (OutT)(r & pmask);
        }
      }
      // ---- 4. running counts for the next tile of the chain ----
      for (uint32_t d = tid; d <= ndig; d += WPB * 32) s.BX[d] += s.H[d];
      __syncthreads();
      PH(9);
    }
    // ---- chain end: flush carried words (shared with the next chain or row) ----
    for (uint32_t slot = 1 + tid; slot < ndig; slot += WPB * 32) {
      if (s.CF[slot] & CF_VALID) {
        const uint32_t k = 31 - __clz(slot), q = slot - (1u << k), sh = tau - k;
        const uint32_t Gend = rstart + s.CR[q << sh] + (s.BX[(q + 1) << sh] - s.BX[q << sh]);
        uint64_t *B = p.bits + (uint64_t)(p.l0 + k) * p.wpl;
        WT_CHECK(Gend <= p.n, 105);
        atomicOr(reinterpret_cast<unsigned long long *>(&B[Gend >> 6]), s.CW[slot]);
      }
    }
    __syncthreads();
    PH(10);
  }
  PH_FLUSH
}

}  // namespace wtb
