// wt_wgroup.cuh -- the hot kernel, round 2: one HBM pass builds tau <= 8
// consecutive levels l0 .. l0+tau-1 of the levelwise wavelet tree (SURVEY
// §8(a) A2, A3, A5, A6, and A7's block counts), one CTA of CT_WARPS warps per
// tile, persistent over chains.
//
// What a CTA computes (Fig. 1 l.12-17, restated for a tile): a chain
// is <= CH consecutive positions of S_{l0} inside one level-l0 node (its
// "row"); it is processed in tiles of <= T positions held in shared memory.
// Inside a tile the CTA keeps the records in the tile's *wavelet-matrix
// order* M_k (the tile stably sorted by the reversed top-k digit bits,
// PAPER.md:911-925): going from M_k to M_{k+1} is ONE stable zeros-first
// split of the whole tile by bit k, so no per-node (per-class) split tables
// are needed.  A class of level k (the elements of one level-(l0+k) node,
// PAPER.md:213-226) is a contiguous run of M_k in original order -- the same
// run it forms in S_{l0+k} -- so level l0+k's bitmap is
// M_k's bitmap with the class runs placed at their tree positions.  Warp w
// splits quarter w of the tile; the quarters' ones counts (onesW, from a
// counting pass over the next bit) give each warp its zeros/ones bases, so a
// level costs two CTA barriers.
//
// Records: rec = bit-reverse of the top kb = min(L - l0, tau) key bits, plus
// the remaining (payload) key bits above them in natural order, so the
// level-(l0+k) bit (the (l+1)'st highest bit) is rec bit k, the
// reversed digit rd = rec & (2^tau - 1) is the class index r of level tau in
// M_tau order, and rec >> tau is the key narrowed for the next group.
//
// The split (per level, per 32*E-position "superchunk", E = 8 (u8, u16
// records) or 4 (u32)): lane l holds E consecutive records (one LDS.64 /
// LDS.128); the level bits t_j, their exclusive in-lane prefix (SWAR: one IMAD
// per 4 bytes), the lane's count and the cross-lane exclusive prefix O
// (ballots of the count's bits + POPC) give every element its rank in its own
// stream; the destination is
//     bit 0: dst + zeros_before(superchunk) + (E*lane - O) + (j - pre_j)
//     bit 1: dst + Z + ones_before(superchunk) + O + pre_j
// (Fig. 1 l.15-17: zeros to start + X[i], ones to start + X_s + i - X[i]),
// evaluated for two elements at a time with one dp2a each.  The level's
// bitmap bytes and the ones before every 32-bit word (a word-grain rank
// directory of the tile) are written to shared memory; class counts of level
// k+1 follow from rank queries at the class boundaries of level k, so no
// per-tile digit histogram is built.  Padding records (all ones) fill the
// last superchunk: they are ones at every level and stay at the end.
//
// Staging (north_star (2)): the TMA unit moves the next tile while the current
// one is split.  Two forms, chosen per input width at compile time
// (WT_WG_STAGE8/16/32): (a) staged -- tile i+1's raw input is fetched by one
// cp.async.bulk into `stage`, completing on an mbarrier; (b) unstaged (the
// default for every width since the end of round 2) -- the next tile is bulk-
// prefetched into L2 (cp.async.bulk.prefetch.L2) and the load step reads it
// with 16-byte loads; the stage's 1-4 B per position of shared memory buy a
// sixth CTA per SM (8-bit inputs: k_group1 1.255 -> 1.197 ms on cfg4,
// profiles/r02s5/tune_tiles8b.log) or larger tiles (16/32-bit inputs).  The
// next chain's starting digit counts V always arrive by cp.async.bulk on the
// mbarrier.
//
// Global placement (A5): class r of level k goes to the
// running position pos[slot], slot = 2^k + r, initialised per chain from V
// and the row's digit scan (Cseg of wt_prep.cuh); words inside a run are
// stored, the partial last word of a run is carried to the next tile of the
// chain, words shared with another chain or node get the writer's bits by an
// atomic OR and an atomic AND confined to them (put_shared_word), so the
// bitmap needs no zero initialisation (only its padding words are zeroed).  Each run also adds its ones to the 512-bit
// blocks it overlaps (red.add into blkcnt; fused A7), so the
// rank directory needs no second read of the bitmaps (k_rank_counts).
#pragma once
#include "wt_common.cuh"
#include "wt_group.cuh"  // GroupParams, CF_VALID / CF_SHARED

namespace wtb {

#ifndef WT_CT_WARPS
#define WT_CT_WARPS 4
#endif
constexpr int CT_WARPS = WT_CT_WARPS;  // warps of a CTA; they share one tile, each splits a quarter
// cross-lane prefix of the split by a packed shfl.up scan over two superchunks
// (8-bit records: measured faster; 16-bit: slower, the ballots stay)
#ifndef WT_WG_SCAN
#define WT_WG_SCAN 1
#endif
#ifndef WT_WG_SCAN16
#define WT_WG_SCAN16 0
#endif
#ifndef WT_WG_PIPE
#define WT_WG_PIPE 1
#endif
#ifndef WT_WG_UNROLL
#define WT_WG_UNROLL 2
#endif
constexpr int WG_UNROLL = WT_WG_UNROLL;  // superchunks of the split loop unrolled

// 32-bit records per lane per superchunk: 4 (one LDS.128; a third ballot of the
// lane count, but half the cross-lane prefixes per record) or 2 (one LDS.64)
#ifndef WT_WG_E32
#define WT_WG_E32 4
#endif
template <typename RecT>
struct WGTile {
  static constexpr int E = sizeof(RecT) == 4 ? WT_WG_E32 : 8;  // records per lane per superchunk (one LDS)
  static constexpr int SC = 32 * E;                      // positions per superchunk
};

#ifndef WT_WG_STAGE32
#define WT_WG_STAGE32 0
#endif
// whether tiles of this input width are prefetched into shared memory by a bulk
// copy (else the load step reads them from global memory directly)
#ifndef WT_WG_STAGE16
#define WT_WG_STAGE16 0
#endif
#ifndef WT_WG_STAGE8
#define WT_WG_STAGE8 0
#endif
template <typename InT>
struct WGStage {
  static constexpr bool on = sizeof(InT) == 1 ? WT_WG_STAGE8 : sizeof(InT) == 2 ? WT_WG_STAGE16 : WT_WG_STAGE32;
};

#ifndef WT_CT_TB
#define WT_CT_TB 8192
#endif
#ifndef WT_CT_TB16
#define WT_CT_TB16 6144
#endif
#ifndef WT_CT_TB16NS
#define WT_CT_TB16NS 12288
#endif
#ifndef WT_CT_TB32NS
#define WT_CT_TB32NS 8192
#endif
// records per tile: WT_CT_TB bytes of records (WT_CT_TB16 for 16-bit records of a staged
// input); unstaged inputs use the stage's shared memory for larger tiles: 6144
// 16-bit records of a 32-bit input, 4096 of a 16-bit input, 2048 32-bit records
// (tools/tune.py).  8-bit inputs keep 8192-record tiles (larger
// unstaged tiles lose the sixth CTA per SM: 10240 -> 1.254 ms, 12288 -> 1.309 ms).
template <typename InT, typename RecT>
struct WGSize {
  static constexpr int RB = sizeof(RecT);
#ifndef WT_CT_TBNS
#define WT_CT_TBNS WT_CT_TB
#endif
#ifndef WT_CT_TB16NS16
#define WT_CT_TB16NS16 8192
#endif
  static constexpr int BYTES = RB == 2 ? (WGStage<InT>::on ? WT_CT_TB16 : sizeof(InT) == 2 ? WT_CT_TB16NS16 : WT_CT_TB16NS)
                                       : RB == 4 ? (WGStage<InT>::on ? WT_CT_TB : WT_CT_TB32NS)
                                                 : (WGStage<InT>::on ? WT_CT_TB : WT_CT_TBNS);
  static constexpr int T = BYTES / RB;
  static constexpr int SPW = T / WGTile<RecT>::SC / CT_WARPS;  // superchunks per warp
  static_assert(SPW >= 1 && T % (WGTile<RecT>::SC * CT_WARPS) == 0, "whole superchunks per warp");
};

template <typename InT, typename RecT, bool HAS_OUT>
struct WGSmem {
  static constexpr int T = WGSize<InT, RecT>::T;
  static constexpr int LBB = T / 8 + 16;  // bytes per level bitmap (+ slack for 3-word reads)
  static constexpr int RPW = T / 32 + 2;  // word ranks per level (+ the padded end)
  alignas(16) RecT rec[2][T];
  alignas(16) uint8_t stage[WGStage<InT>::on ? T * sizeof(InT) + 32 : 16];  // raw input of the next tile (TMA bulk copy)
  alignas(16) uint8_t LB[TAU_MAX][LBB];  // level bitmaps of the tile (M_k order)
  alignas(16) uint16_t RP[TAU_MAX][RPW]; // ones of the level before each 32-bit word of LB
  alignas(16) uint32_t V[256];           // chain's starting digit counts (bulk copy, next chain's)
  alignas(16) uint32_t pos[256];         // running global bit position of slot 2^k + r
  alignas(16) uint32_t kpos[HAS_OUT ? 256 : 1];  // running key position per (true) digit
  alignas(16) unsigned long long CW[256];        // carried partial word per slot (chain setup: scratch)
  alignas(16) uint16_t C[512];           // class counts (real) of slot 2^k + r, k <= tau
  alignas(16) uint16_t S[512];           // class starts (tile positions in M_k)
  alignas(16) uint32_t Zs[TAU_MAX + 2];  // zeros of each level's bit (real elements)
  alignas(16) uint32_t onesW[CT_WARPS];  // ones of the current bit in each warp's quarter
  alignas(16) unsigned long long bar;    // mbarrier of the bulk copy
  uint32_t chain, cnext;
  alignas(16) uint8_t CF[256];           // carry flags per slot
};

__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ uint2 lds64(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts8(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void sts16(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void sts64(uint32_t a, uint32_t x, uint32_t y) {
  asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(a), "r"(x), "r"(y) : "memory");
}
// ballot of (v & m) != 0
__device__ __forceinline__ uint32_t ballot_m(uint32_t v, uint32_t m) {
  uint32_t r;
  asm(
      "{.reg .pred p; .reg .b32 t; and.b32 t, %1, %2; setp.ne.u32 p, t, 0; vote.sync.ballot.b32 %0, p, 0xffffffff;}"
      : "=r"(r)
      : "r"(v), "r"(m));
  return r;
}
// one step of an inclusive warp scan: v + (the value of lane - d, if it exists)
__device__ __forceinline__ uint32_t shfl_up_add(uint32_t v, uint32_t d) {
  asm volatile(
      "{.reg .pred p; .reg .b32 t; shfl.sync.up.b32 t|p, %0, %1, 0, 0xffffffff; @p add.u32 %0, %0, t;}"
      : "+r"(v)
      : "r"(d));
  return v;
}
__device__ __forceinline__ uint32_t rev_bits(uint32_t x, uint32_t nb) { return nb ? __brev(x) >> (32u - nb) : 0u; }

// ---------------------------------------------------------------------------
// One level of one sub-tile: the level's bitmap (LB, M_k order) and the ones
// before every 32-bit word of it (RP), optionally the stable split src -> dst
// (byte addresses), and the ones of bit k+1 (returned, padding included).
// nsc superchunks; Z = zeros of bit k.
// ---------------------------------------------------------------------------
template <typename RecT, bool MOVE>
__device__ __forceinline__ void wg_split(uint8_t *LB, uint16_t *RP, uint32_t src, uint32_t dst, uint32_t c0,
                                         uint32_t c1, uint32_t nsc, uint32_t k, uint32_t Z, uint32_t SP0, int lane,
                                         uint32_t lt) {
  constexpr uint32_t E = WGTile<RecT>::E, SC = WGTile<RecT>::SC, RB = sizeof(RecT);
  constexpr uint32_t LANEB = E * RB;                // record bytes per lane per superchunk
  const uint32_t lbA = smem_u32(LB), rpA = smem_u32(RP);
  const uint32_t sA = src + lane * LANEB;
  uint32_t SP = SP0;                                // ones before the superchunk (level k)
  uint32_t Bo = dst + (Z + SP0) * RB;               // ones region + ones so far
  uint32_t Bz = dst + (c0 * SC - SP0) * RB + lane * LANEB;  // zeros so far + this lane's first slot
  if constexpr (RB <= 2) {
    // 8 records per lane: their digit bytes d (8-bit records: the records; 16-bit:
    // the low bytes gathered by two PRMT), the level bits t, the exclusive in-lane
    // prefix pre (SWAR: one IMAD per 4 bytes) and the lane's ones count (0..8)
    struct Sw {
      uint32_t t_lo, t_hi, pre_lo, pre_hi, cnt;
    };
    auto swar = [&](uint32_t d_lo, uint32_t d_hi) {
      Sw w;
      w.t_lo = (d_lo >> k) & 0x01010101u;
      w.t_hi = (d_hi >> k) & 0x01010101u;
      w.pre_lo = w.t_lo * 0x01010100u;
      const uint32_t inc_lo = w.pre_lo + w.t_lo;
      w.pre_hi = w.t_hi * 0x01010100u + __byte_perm(inc_lo, 0, 0x3333);
      w.cnt = (w.pre_hi + w.t_hi) >> 24;
      return w;
    };
    // superchunk c with the lane's exclusive cross-lane prefix O and the superchunk's ones Sc:
    // word ranks, the level's bitmap byte, and (MOVE) the stable split of the records
    auto emit = [&](uint32_t c, const Sw &w, uint32_t O, uint32_t Sc, uint32_t r0, uint32_t r1, uint32_t r2,
                    uint32_t r3) {
      if (!(lane & 3)) sts16(rpA + (c * 8u + (lane >> 2)) * 2u, SP + O);
      // bits 24..27 <- elements 0..3, bits 28..31 <- elements 4..7 (disjoint products, no carries)
      sts8(lbA + c * 32u + lane, (w.t_lo * 0x01020408u + w.t_hi * 0x10204080u) >> 24);
      if constexpr (MOVE) {
        const uint32_t D0 = Bz - RB * O;
        const uint32_t A = (Bo + RB * O - D0) | (RB << 16);
        WT_CHECK(D0 >= dst && Bo + RB * O <= dst + nsc * SC * RB, 201);
        const uint32_t M_lo = w.t_lo * 0xffu, M_hi = w.t_hi * 0xffu;
        const uint32_t q_lo = (w.pre_lo & M_lo) | ((0x03020100u - w.pre_lo) & ~M_lo);
        const uint32_t q_hi = (w.pre_hi & M_hi) | ((0x07060504u - w.pre_hi) & ~M_hi);
        const uint32_t tq0 = __byte_perm(w.t_lo, q_lo, 0x5140), tq1 = __byte_perm(w.t_lo, q_lo, 0x7362);
        const uint32_t tq2 = __byte_perm(w.t_hi, q_hi, 0x5140), tq3 = __byte_perm(w.t_hi, q_hi, 0x7362);
        if constexpr (RB == 1) {
          sts8(__dp2a_lo(A, tq0, D0), r0);
          sts8(__dp2a_hi(A, tq0, D0), __byte_perm(r0, 0, 0x1));
          sts8(__dp2a_lo(A, tq1, D0), __byte_perm(r0, 0, 0x2));
          sts8(__dp2a_hi(A, tq1, D0), __byte_perm(r0, 0, 0x3));
          sts8(__dp2a_lo(A, tq2, D0), r1);
          sts8(__dp2a_hi(A, tq2, D0), __byte_perm(r1, 0, 0x1));
          sts8(__dp2a_lo(A, tq3, D0), __byte_perm(r1, 0, 0x2));
          sts8(__dp2a_hi(A, tq3, D0), __byte_perm(r1, 0, 0x3));
        } else {
          sts16(__dp2a_lo(A, tq0, D0), r0);
          sts16(__dp2a_hi(A, tq0, D0), r0 >> 16);
          sts16(__dp2a_lo(A, tq1, D0), r1);
          sts16(__dp2a_hi(A, tq1, D0), r1 >> 16);
          sts16(__dp2a_lo(A, tq2, D0), r2);
          sts16(__dp2a_hi(A, tq2, D0), r2 >> 16);
          sts16(__dp2a_lo(A, tq3, D0), r3);
          sts16(__dp2a_hi(A, tq3, D0), r3 >> 16);
        }
      }
      SP += Sc;
      Bo += RB * Sc;
      Bz += RB * (SC - Sc);
    };
    auto load = [&](uint32_t c, uint32_t &r0, uint32_t &r1, uint32_t &r2, uint32_t &r3) {
      if constexpr (RB == 1) {
        const uint2 x = lds64(sA + c * (SC * RB));
        r0 = x.x; r1 = x.y; r2 = r3 = 0u;
      } else {
        const uint4 x = lds128(sA + c * (SC * RB));
        r0 = x.x; r1 = x.y; r2 = x.z; r3 = x.w;
      }
    };
    auto digits_lo = [&](uint32_t r0, uint32_t r1) { return RB == 1 ? r0 : __byte_perm(r0, r1, 0x6420); };
    auto digits_hi = [&](uint32_t r1, uint32_t r2, uint32_t r3) { return RB == 1 ? r1 : __byte_perm(r2, r3, 0x6420); };
    uint32_t c = c0;
    if constexpr ((RB == 1 && WT_WG_SCAN) || (RB == 2 && WT_WG_SCAN16)) {
    // two superchunks per cross-lane prefix: the lanes' counts packed in 16-bit
    // fields, one 5-step shfl.up scan (two instructions a step) for both
    for (; c + 1 < c1; c += 2) {
      uint32_t a0, a1, a2, a3, b0, b1, b2, b3;
      load(c, a0, a1, a2, a3);
      load(c + 1, b0, b1, b2, b3);
      const Sw wa = swar(digits_lo(a0, a1), digits_hi(a1, a2, a3));
      const Sw wb = swar(digits_lo(b0, b1), digits_hi(b1, b2, b3));
      const uint32_t own = wa.cnt | (wb.cnt << 16);
      uint32_t incl = own;
#pragma unroll
      for (uint32_t d = 1; d < 32; d <<= 1) incl = shfl_up_add(incl, d);
      const uint32_t ex = incl - own, tot = __shfl_sync(FULL, incl, 31);
      emit(c, wa, ex & 0xffffu, tot & 0xffffu, a0, a1, a2, a3);
      emit(c + 1, wb, ex >> 16, tot >> 16, b0, b1, b2, b3);
    }
    }
    // one superchunk at a time: the cross-lane prefix from ballots of the count's bits;
    // software pipelined (the next superchunk's load is issued before this one is processed)
    uint32_t n0 = 0, n1 = 0, n2 = 0, n3 = 0;
    if (WT_WG_PIPE && c < c1) load(c, n0, n1, n2, n3);
#pragma unroll(WG_UNROLL)
    for (; c < c1; c++) {
      uint32_t a0, a1, a2, a3;
      if (WT_WG_PIPE) {
        a0 = n0; a1 = n1; a2 = n2; a3 = n3;
        if (c + 1 < c1) load(c + 1, n0, n1, n2, n3);
      } else {
        load(c, a0, a1, a2, a3);
      }
      const Sw w = swar(digits_lo(a0, a1), digits_hi(a1, a2, a3));
      const uint32_t inc = w.cnt << 24;
      const uint32_t O = __popc(ballot_m(inc, 1u << 24) & lt) + 2 * __popc(ballot_m(inc, 2u << 24) & lt) +
                         4 * __popc(ballot_m(inc, 4u << 24) & lt) + 8 * __popc(ballot_m(inc, 8u << 24) & lt);
      const uint32_t Sc = __shfl_sync(FULL, O + w.cnt, 31);
      emit(c, w, O, Sc, a0, a1, a2, a3);
    }
  } else if constexpr (E == 4) {
    // 32-bit records, four per lane: lane count 0..4 (three ballots), the lane's
    // nibble of level bits paired with its neighbour's into one bitmap byte
#pragma unroll 2
    for (uint32_t c = c0; c < c1; c++) {
      const uint4 x = lds128(sA + c * (SC * RB));
      const uint32_t t0 = (x.x >> k) & 1u, t1 = (x.y >> k) & 1u, t2 = (x.z >> k) & 1u, t3 = (x.w >> k) & 1u;
      const uint32_t p2 = t0 + t1, p3 = p2 + t2, tot = p3 + t3;
      const uint32_t O = __popc(ballot_m(tot, 1u) & lt) + 2 * __popc(ballot_m(tot, 2u) & lt) +
                         4 * __popc(ballot_m(tot, 4u) & lt);
      const uint32_t Sc = __shfl_sync(FULL, O + tot, 31);
      uint32_t v = t0 | (t1 << 1) | (t2 << 2) | (t3 << 3);
      v |= __shfl_down_sync(FULL, v, 1) << 4;
      if (!(lane & 7)) sts16(rpA + (c * 4u + (lane >> 3)) * 2u, SP + O);
      if (!(lane & 1)) sts8(lbA + c * 16u + (lane >> 1), v);
      if constexpr (MOVE) {
        const uint32_t D0 = Bz - 4u * O, D1 = Bo + 4u * O;  // the lane's first zero / one slot
        WT_CHECK(D0 >= dst && D1 <= dst + nsc * SC * RB, 201);
        sts<uint32_t>(t0 ? D1 : D0, x.x);
        sts<uint32_t>(t1 ? D1 + 4u * t0 : D0 + 4u * (1u - t0), x.y);
        sts<uint32_t>(t2 ? D1 + 4u * p2 : D0 + 4u * (2u - p2), x.z);
        sts<uint32_t>(t3 ? D1 + 4u * p3 : D0 + 4u * (3u - p3), x.w);
      }
      SP += Sc;
      Bo += 4u * Sc;
      Bz += 4u * (SC - Sc);
    }
  } else {
#pragma unroll 2
    for (uint32_t c = c0; c < c1; c++) {
      const uint2 x = lds64(sA + c * (SC * RB));
      const uint32_t t0 = (x.x >> k) & 1u, t1 = (x.y >> k) & 1u;
      const uint32_t tot = t0 + t1;
      const uint32_t O = __popc(ballot_m(tot, 1u) & lt) + 2 * __popc(ballot_m(tot, 2u) & lt);
      const uint32_t Sc = __shfl_sync(FULL, O + tot, 31);
      uint32_t v = t0 | (t1 << 1);
      v |= __shfl_down_sync(FULL, v, 1) << 2;
      v |= __shfl_down_sync(FULL, v, 2) << 4;
      if (!(lane & 15)) sts16(rpA + (c * 2u + (lane >> 4)) * 2u, SP + O);
      if (!(lane & 3)) sts8(lbA + c * 8u + (lane >> 2), v);
      if constexpr (MOVE) {
        const uint32_t D0 = Bz - 4u * O, D1 = Bo + 4u * O;
        sts<uint32_t>(t0 ? D1 : D0, x.x);
        sts<uint32_t>(t1 ? D1 + 4u * t0 : D0 + 4u * (1u - t0), x.y);
      }
      SP += Sc;
      Bo += 4u * Sc;
      Bz += 4u * (SC - Sc);
    }
  }
  if (lane == 0 && c1 == nsc && c0 < c1) RP[nsc * SC / 32] = (uint16_t)SP;  // rank at the padded end
}

// ones of bit k over superchunks [c0, c1) of the tile (padding included), warp-reduced
template <typename RecT>
__device__ __forceinline__ uint32_t wg_count(uint32_t src, uint32_t c0, uint32_t c1, uint32_t k, int lane) {
  constexpr uint32_t E = WGTile<RecT>::E, SC = WGTile<RecT>::SC, RB = sizeof(RecT);
  const uint32_t sA = src + lane * (E * RB);
  uint32_t acc = 0;
#pragma unroll 4
  for (uint32_t c = c0; c < c1; c++) {
    if constexpr (RB == 1) {
      const uint2 x = lds64(sA + c * (SC * RB));
      acc += ((x.x >> k) & 0x01010101u) + ((x.y >> k) & 0x01010101u);
    } else if constexpr (RB == 2) {
      const uint4 x = lds128(sA + c * (SC * RB));
      acc += ((__byte_perm(x.x, x.y, 0x6420) >> k) & 0x01010101u) + ((__byte_perm(x.z, x.w, 0x6420) >> k) & 0x01010101u);
    } else if constexpr (E == 4) {
      const uint4 x = lds128(sA + c * (SC * RB));
      acc += ((x.x >> k) & 1u) + ((x.y >> k) & 1u) + ((x.z >> k) & 1u) + ((x.w >> k) & 1u);
    } else {
      const uint2 x = lds64(sA + c * (SC * RB));
      acc += ((x.x >> k) & 1u) + ((x.y >> k) & 1u);
    }
  }
  if constexpr (RB <= 2) acc = (acc * 0x01010101u) >> 24;  // bytes <= 2 per superchunk: no overflow
  return __reduce_add_sync(FULL, acc);
}

// ones of the level before sub-tile position p (p <= padded length)
__device__ __forceinline__ uint32_t wg_rank1(const uint32_t *LBw, const uint16_t *RP, uint32_t p) {
  const uint32_t w = p >> 5;
  return RP[w] + __popc(LBw[w] & ((1u << (p & 31u)) - 1u));
}

// bits [pos, pos + nb) of a tile bitmap (u32 words), 1 <= nb <= 64, LSB first
__device__ __forceinline__ uint64_t lb_bits(const uint32_t *LBw, uint32_t pos, uint32_t nb) {
  const uint32_t w = pos >> 5, sh = pos & 31u;
  const uint32_t x0 = LBw[w], x1 = LBw[w + 1], x2 = LBw[w + 2];
  uint32_t lo = __funnelshift_r(x0, x1, sh), hi = __funnelshift_r(x1, x2, sh);
  if (nb < 32) {
    lo &= (1u << nb) - 1u;
    hi = 0;
  } else if (nb < 64) {
    hi &= (1u << (nb - 32)) - 1u;
  }
  return ((uint64_t)hi << 32) | lo;
}

#ifndef WT_WG_INLANE
#define WT_WG_INLANE 3
#endif
// One run (one thread): tile bitmap bits [ls, ls+cnt) -> global bits
// [G, G+cnt) of B (cnt > 0, G + cnt <= n < 2^32).  The first word takes the
// carried bits of the slot; it is OR-ed atomically when its low bits belong to
// another chain or node, stored otherwise; an unfinished last word (the run
// ends inside it before n) is carried to the next tile of the chain.  Interior
// words are stored here when few, else their count is returned for the
// cooperative pass.
// fused A7: a run [G, G+cnt) placed from tile bits
// [ls, ls+cnt) adds, to every 512-bit block it overlaps, the ones of the
// overlap -- two rank queries on the tile bitmap (bits are counted where they
// come from, independent of when their word is committed)
__device__ __forceinline__ void run_blocks(uint32_t *bc, const uint32_t *LBw, const uint16_t *RP, uint32_t G,
                                           uint32_t ls, uint32_t cnt, uint32_t b_lo, uint32_t b_hi, uint32_t step) {
  const uint32_t e = G + cnt;
  for (uint32_t b = b_lo; b <= b_hi; b += step) {
    const uint32_t lo = max(G, b << 9), hi = min(e, (b << 9) + 512u);
    const uint32_t c = wg_rank1(LBw, RP, ls + (hi - G)) - wg_rank1(LBw, RP, ls + (lo - G));
    WT_CHECK(lo < hi && c <= hi - lo, 206);
    if (c) atomicAdd(bc + b, c);
  }
}
// A5 without a zero-initialised bitmap (PAPER.md:430-439 CASes the <= 2
// shared words of a node; here two order-independent atomics): a word shared
// with other chains or nodes gets this writer's bits m set to v -- OR sets its
// ones, AND clears its zeros, neither touches bits outside m -- so whatever
// the word held before and in whatever order its writers come, every bit ends
// as its owner wrote it.  Words a run owns entirely are stored; only the
// level's padding words (beyond the last word holding a position < n) are
// zeroed separately (k_zero_pad).  With WT_BITS_MEMSET the bitmap is zeroed
// first and one atomicOr suffices.
#ifndef WT_BITS_MEMSET
#define WT_BITS_MEMSET 0
#endif
__device__ __forceinline__ void put_shared_word(uint64_t *w, uint64_t v, uint64_t m) {
  atomicOr(reinterpret_cast<unsigned long long *>(w), (unsigned long long)v);
  if (!WT_BITS_MEMSET) atomicAnd(reinterpret_cast<unsigned long long *>(w), (unsigned long long)(v | ~m));
}
constexpr uint32_t CF_LO_SHIFT = 2;  // carry flags: bits 2..7 = the chain's first bit in the carried word

// zero the padding words [n64, wpl) of levels l0 .. l0+nl-1 (one block per level)
static __global__ void k_zero_pad(uint64_t *bits, uint64_t wpl, uint64_t n64, uint32_t l0) {
  uint64_t *B = bits + (uint64_t)(l0 + blockIdx.x) * wpl;
  for (uint64_t w = n64 + threadIdx.x; w < wpl; w += blockDim.x) B[w] = 0;
}

// `ones` returns the ones of the run's own bits when every word of it was
// handled here (ni == 0), else ~0u (the caller falls back to rank queries)
__device__ __forceinline__ uint32_t wg_run(unsigned long long &cw, uint8_t &cf, const uint32_t *LBw, uint64_t *B,
                                           uint32_t n32, uint32_t G, uint32_t ls, uint32_t cnt, uint32_t &ones) {
  const uint32_t g0 = G & 63u, e = G + cnt;
  const uint32_t gw0 = G >> 6, gwl = (e - 1u) >> 6;
  WT_CHECK(cnt > 0 && (uint64_t)G + cnt <= n32, 203);
  const uint32_t hb = min(cnt, 64u - g0);
  const uint64_t hbits = lb_bits(LBw, ls, hb);
  uint32_t c = __popcll(hbits);
  uint64_t head = hbits << g0;
  const uint32_t f = cf;
  bool shared = g0 != 0;
  uint32_t lo = g0;  // the word's bits from lo up belong to this chain and slot
  if (f & CF_VALID) {
    head |= cw;
    shared = (f & CF_SHARED) != 0;
    lo = f >> CF_LO_SHIFT;
  }
  const bool open_end = (e & 63u) != 0 && e != n32;  // the run's last word is unfinished
  if (gw0 == gwl && open_end) {
    cw = head;
    cf = CF_VALID | (shared ? CF_SHARED : 0) | (lo << CF_LO_SHIFT);
    ones = c;
    return 0u;
  }
  // a written first word is ours from bit lo to 64 (a run ending inside it ends at n:
  // the bits above n are zero padding, also ours)
  if (shared) put_shared_word(&B[gw0], head, ~0ull << lo);
  else B[gw0] = head;
  cf = 0;
  if (gw0 == gwl) {
    ones = c;
    return 0u;
  }
  const uint32_t tb = e - (gwl << 6);  // 1..64 bits in the last word
  const uint64_t tail = lb_bits(LBw, ls + cnt - tb, tb);
  c += __popcll(tail);
  if (open_end) {
    cw = tail;
    cf = CF_VALID;
  } else {
    B[gwl] = tail;
  }
  const uint32_t ni = gwl - gw0 - 1u;
  if (ni <= WT_WG_INLANE) {
    for (uint32_t w = 0; w < ni; w++) {
      const uint64_t x = lb_bits(LBw, ls + hb + 64u * w, 64);
      c += __popcll(x);
      B[gw0 + 1u + w] = x;
    }
    ones = c;
    return 0u;
  }
  ones = ~0u;
  return ni;
}

// ---- TMA bulk copy (cp.async.bulk) of the raw input of one sub-tile ----
__device__ __forceinline__ void bar_init(uint32_t bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// lane 0: the aligned 16-byte cover of [src, src + bytes) into dst; returns the head offset
__device__ __forceinline__ void bulk_load(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(src);
  const uintptr_t a0 = a & ~(uintptr_t)15, a1 = (a + bytes + 15) & ~(uintptr_t)15;
  const uint32_t sz = (uint32_t)(a1 - a0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(sz) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(a0), "r"(sz), "r"(bar)
               : "memory");
}
// lane 0: as bulk_load, plus a second 16-byte-aligned copy (bytes2 % 16 == 0) on the same barrier
__device__ __forceinline__ void bulk_load2(uint32_t dst, const void *src, uint32_t bytes, uint32_t dst2,
                                           const void *src2, uint32_t bytes2, uint32_t bar) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(src);
  const uintptr_t a0 = a & ~(uintptr_t)15, a1 = (a + bytes + 15) & ~(uintptr_t)15;
  const uint32_t sz = (uint32_t)(a1 - a0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(sz + bytes2) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(a0), "r"(sz), "r"(bar)
               : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst2),
               "l"(src2), "r"(bytes2), "r"(bar)
               : "memory");
}
// bulk prefetch of [src, src + bytes) into L2 (TMA unit; the 16-byte-aligned cover)
__device__ __forceinline__ void prefetch_l2(const void *src, uint32_t bytes) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(src);
  const uintptr_t a0 = a & ~(uintptr_t)15, a1 = (a + bytes + 15) & ~(uintptr_t)15;
  if (a1 > a0)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"((uint32_t)(a1 - a0)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint32_t bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p;}"
        : "=r"(done)
        : "r"(bar), "r"(phase)
        : "memory");
  }
}

// raw 32-bit words of one 16-byte record group from the staging buffer:
// in[0 .. 4*NV) = bytes [h + 16*NV*g, +16*NV) (h = head offset < 16, uniform)
template <uint32_t NV>
__device__ __forceinline__ void stage_words(const uint8_t *stg, uint32_t g, uint32_t h, uint32_t *in) {
  const uint4 *V = reinterpret_cast<const uint4 *>(stg) + NV * g;
  uint32_t raw[4 * NV + 4];
#pragma unroll
  for (uint32_t q = 0; q < NV; q++) {
    const uint4 u = V[q];
    raw[4 * q] = u.x; raw[4 * q + 1] = u.y; raw[4 * q + 2] = u.z; raw[4 * q + 3] = u.w;
  }
  if (h == 0) {
#pragma unroll
    for (uint32_t q = 0; q < 4 * NV; q++) in[q] = raw[q];
    return;
  }
  {
    const uint4 u = V[NV];
    raw[4 * NV] = u.x; raw[4 * NV + 1] = u.y; raw[4 * NV + 2] = u.z; raw[4 * NV + 3] = u.w;
  }
  const uint32_t hb = 8u * (h & 3u);
#define WG_SHIFT(H)                                                                                             \
  case H:                                                                                                       \
    _Pragma("unroll") for (uint32_t q = 0; q < 4 * NV; q++) in[q] = __funnelshift_r(raw[q + H], raw[q + H + 1], hb); \
    break;
  switch (h >> 2) { WG_SHIFT(0) WG_SHIFT(1) WG_SHIFT(2) WG_SHIFT(3) }
#undef WG_SHIFT
}

// as stage_words, from global memory (V = the 16-byte-aligned cover of the tile)
template <uint32_t NV>
__device__ __forceinline__ void global_words(const uint4 *V0, uint32_t g, uint32_t h, uint32_t *in) {
  const uint4 *V = V0 + NV * g;
  uint32_t raw[4 * NV + 4];
#pragma unroll
  for (uint32_t q = 0; q < NV; q++) {
    const uint4 u = __ldcs(V + q);
    raw[4 * q] = u.x; raw[4 * q + 1] = u.y; raw[4 * q + 2] = u.z; raw[4 * q + 3] = u.w;
  }
  if (h == 0) {
#pragma unroll
    for (uint32_t q = 0; q < 4 * NV; q++) in[q] = raw[q];
    return;
  }
  {
    const uint4 u = __ldcs(V + NV);
    raw[4 * NV] = u.x; raw[4 * NV + 1] = u.y; raw[4 * NV + 2] = u.z; raw[4 * NV + 3] = u.w;
  }
  const uint32_t hb = 8u * (h & 3u);
#define WG_SHIFT(H)                                                                                             \
  case H:                                                                                                       \
    _Pragma("unroll") for (uint32_t q = 0; q < 4 * NV; q++) in[q] = __funnelshift_r(raw[q + H], raw[q + H + 1], hb); \
    break;
  switch (h >> 2) { WG_SHIFT(0) WG_SHIFT(1) WG_SHIFT(2) WG_SHIFT(3) }
#undef WG_SHIFT
}

template <typename InT, typename RecT, typename OutT, bool HAS_OUT>
__global__ void __launch_bounds__(CT_WARPS * 32) k_wgroup(GroupParams p) {
  using SM = WGSmem<InT, RecT, HAS_OUT>;
  constexpr uint32_t T = SM::T, SC = WGTile<RecT>::SC, SPW = WGSize<InT, RecT>::SPW, RB = sizeof(RecT),
                     IB = sizeof(InT);
  constexpr uint32_t PER = 16 / RB, NV = PER * IB / 16;  // records per 16-byte group, input uint4 per group
  constexpr uint32_t NT = CT_WARPS * 32;
  constexpr bool STAGE = WGStage<InT>::on;
  extern __shared__ __align__(16) uint8_t wg_raw[];
  SM &s = *reinterpret_cast<SM *>(wg_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (ld_relaxed(p.err)) return;
  const uint32_t lt = lanemask_lt();
  const uint32_t tau = p.tau, pbits = p.pbits, kb = tau + pbits;
  const uint32_t ndig = 1u << tau, dmask = ndig - 1u;
  const uint32_t pmask = pbits >= 32 ? 0xffffffffu : (1u << pbits) - 1u;
  const uint32_t nchains = p.counts[0];
  const uint32_t n32 = (uint32_t)p.n;  // n < 2^32 (wt_build's contract)
  const InT *keys = reinterpret_cast<const InT *>(p.keys_in);
  const uint32_t bar = smem_u32(&s.bar), stg = smem_u32(s.stage), vA = smem_u32(s.V);
  // thread 0: claim a chain and start the bulk copy of its first tile and its digit vector
  auto claim = [&]() {
    const uint32_t c = atomicAdd(p.chain_counter, 1u);
    if (c < nchains) {
      const uint32_t b = p.chain_begin[c], e = p.chain_end[c];
      if constexpr (STAGE) {
        bulk_load2(stg, keys + b, min(e - b, T) * IB, vA, p.V + (uint64_t)c * 256, 1024u, bar);
      } else {
        bulk_load(vA, p.V + (uint64_t)c * 256, 1024u, bar);
        prefetch_l2(keys + b, min(e - b, T) * IB);  // the chain's first tile, read at its start
      }
    }
    return c;
  };
  if (tid == 0) {
    bar_init(bar);
    s.chain = claim();
  }
  __syncthreads();
  uint32_t phase = 0;
  uint32_t c = s.chain;

  while (c < nchains) {
    // ---- chain setup: running positions of every class slot and digit ----
    const uint32_t row = p.chain_row[c];
    const uint32_t cbeg = p.chain_begin[c], cend = p.chain_end[c];
    const uint32_t rstart = p.row_start[row];
    const uint32_t *Cg = p.Cseg + (uint64_t)row * (ndig + 1);
    uint32_t *X = reinterpret_cast<uint32_t *>(s.CW);  // scratch until the carries start
    bar_wait(bar, phase);  // the chain's digit vector (and first tile) have landed
    if constexpr (!STAGE) phase ^= 1u;  // one bulk copy (V) per chain
    if (warp == 0) {
      // X[d] = exclusive scan over digits of the same-row elements ahead of the chain
      uint32_t v[8], sum = 0;
      const uint32_t per = (ndig + 31) >> 5, lo = min(lane * per, ndig), hi = min(lo + per, ndig);
#pragma unroll
      for (int i = 0; i < 8; i++) {
        const uint32_t d = lo + i;
        v[i] = (d < hi) ? s.V[d] : 0u;
        sum += v[i];
      }
      const uint32_t incl = warp_incl_scan(sum, lane);
      uint32_t run = incl - sum;
#pragma unroll
      for (int i = 0; i < 8; i++) {
        const uint32_t d = lo + i;
        if (d < hi) {
          if constexpr (HAS_OUT) s.kpos[d] = rstart + Cg[d] + v[i];
          X[d] = run;
          run += v[i];
        }
      }
      if (lane == 31) X[ndig] = incl;
    }
    __syncthreads();
    // slot 2^k + r, class q = rev_k(r): rstart + Cseg[q << (tau-k)] + (X[(q+1) << (tau-k)] - X[q << (tau-k)])
    for (uint32_t slot = 1 + tid; slot < ndig; slot += NT) {
      const uint32_t k = 31 - __clz(slot), r = slot - (1u << k);
      const uint32_t q = rev_bits(r, k), sh = tau - k;
      s.pos[slot] = rstart + Cg[q << sh] + (X[(q + 1) << sh] - X[q << sh]);
      WT_CHECK(s.pos[slot] <= n32, 205);
    }
    __syncthreads();
    for (uint32_t i = tid; i < 256; i += NT) s.CF[i] = 0;

    for (uint64_t start64 = cbeg; start64 < cend; start64 += T) {
      const uint32_t start = (uint32_t)start64;
      const uint32_t rem = cend - start;
      const uint32_t len = rem < T ? rem : T;
      const uint32_t nsc = (len + SC - 1) / SC, ntot = nsc * SC;
      const uint32_t c0 = min((uint32_t)warp * SPW, nsc), c1 = min(c0 + SPW, nsc);  // this warp's quarter

      // ---- 1. records from the staged input + ones of bit 0 per quarter ----
      // record = (payload << tau) | reversed digit: level l0+k's bit (the (k+1)'st highest
      // bit of the key) is record bit k; the payload keeps its natural order
      if constexpr (STAGE) {
        if (start64 != cbeg) bar_wait(bar, phase);
        phase ^= 1u;
      }
      {
        const uint32_t h = (uint32_t)(reinterpret_cast<uintptr_t>(keys + start) & 15u);
        RecT *R = s.rec[0];
        uint32_t ones0 = 0;
        for (uint32_t g = c0 * (SC / PER) + lane; g < c1 * (SC / PER); g += 32) {
          const uint32_t i0 = g * PER;
          uint32_t in[4 * NV], w[4];
          if constexpr (STAGE) stage_words<NV>(s.stage, g, h, in);
          else global_words<NV>(reinterpret_cast<const uint4 *>(reinterpret_cast<uintptr_t>(keys + start) & ~(uintptr_t)15), g, h, in);
          if constexpr (IB == 1 && RB == 1) {
#pragma unroll
            for (int q = 0; q < 4; q++) {
              uint32_t x = __byte_perm(__brev(in[q]), 0, 0x0123);  // every byte bit-reversed
              if (kb < 8) x = (x >> (8u - kb)) & (((1u << kb) - 1u) * 0x01010101u);
              w[q] = x;
            }
          } else if (IB == 4 && RB == 2 && kb == 16 && tau == 8) {
            // key = digit << 8 | payload (< 2^16): record bytes {rev8(digit), payload}
#pragma unroll
            for (int q = 0; q < 4; q++) {
              const uint32_t r0 = __byte_perm(__brev(in[2 * q]), in[2 * q], 0x0042);
              const uint32_t r1 = __byte_perm(__brev(in[2 * q + 1]), in[2 * q + 1], 0x0042);
              w[q] = __byte_perm(r0, r1, 0x5410);
            }
          } else {
#pragma unroll
            for (int q = 0; q < 4; q++) w[q] = 0u;
#pragma unroll
            for (uint32_t e = 0; e < PER; e++) {
              uint32_t key;
              if constexpr (IB == 1) key = (in[e >> 2] >> (8 * (e & 3))) & 0xffu;
              else if constexpr (IB == 2) key = (in[e >> 1] >> (16 * (e & 1))) & 0xffffu;
              else key = in[e];
              const uint32_t r = ((__brev(key) >> (32u - kb)) & dmask) | ((key & pmask) << tau);
              w[(e * RB) >> 2] |= r << (8u * ((e * RB) & 3u));
            }
          }
          if (i0 + PER > len) {  // padding records (all ones: a one at every level, they stay last)
#pragma unroll
            for (uint32_t e = 0; e < PER; e++) {
              if (i0 + e >= len) {
                if constexpr (RB == 4) w[e] = 0xffffffffu;
                else w[(e * RB) >> 2] |= ((1u << (8 * RB)) - 1u) << (8u * ((e * RB) & 3u));
              }
            }
          }
          if constexpr (RB == 1) {
            ones0 += __popc((w[0] & 0x01010101u)) + __popc(w[1] & 0x01010101u) + __popc(w[2] & 0x01010101u) +
                     __popc(w[3] & 0x01010101u);
          } else if constexpr (RB == 2) {
            ones0 += __popc((w[0] & 0x00010001u)) + __popc(w[1] & 0x00010001u) + __popc(w[2] & 0x00010001u) +
                     __popc(w[3] & 0x00010001u);
          } else {
            ones0 += (w[0] & 1u) + (w[1] & 1u) + (w[2] & 1u) + (w[3] & 1u);
          }
          *reinterpret_cast<uint4 *>(R + i0) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        ones0 = __reduce_add_sync(FULL, ones0);
        if (lane == 0) s.onesW[warp] = ones0;
      }
      if (tid == 0) {
        s.C[1] = (uint16_t)len;  // slot 1: the one class of level 0
        s.S[1] = 0;
      }
      __syncthreads();
      // the staging buffer is free: prefetch the next tile of the chain, or the next chain's first
      if (tid == 0) {
        if (!STAGE) {  // the next tile of the chain into L2 while this one is split
          if (start64 + T < cend) prefetch_l2(keys + start + T, min(cend - (start + T), T) * IB);
          else s.cnext = claim();
        } else if (start64 + T < cend) {
          bulk_load(stg, keys + start + T, min(cend - (start + T), T) * IB, bar);
        } else {
          s.cnext = claim();
        }
      }

      // ---- 2. tau levels of splits (bitmaps and word ranks kept per level) ----
      for (uint32_t k = 0; k < tau; k++) {
        uint32_t before = 0, tot = 0;
        const uint32_t *cnts = s.onesW;
#pragma unroll
        for (int w = 0; w < CT_WARPS; w++) {
          const uint32_t o = cnts[w];
          before += w < warp ? o : 0u;
          tot += o;
        }
        const uint32_t Z = ntot - tot;  // zeros of bit k (padding records are ones)
        if (tid == 0) s.Zs[k] = Z;
        const uint32_t src = smem_u32(s.rec[k & 1u]), dst = smem_u32(s.rec[(k & 1u) ^ 1u]);
        const bool move = HAS_OUT || k + 1 < tau;
        if (c0 < c1) {
          if (move) wg_split<RecT, true>(s.LB[k], s.RP[k], src, dst, c0, c1, nsc, k, Z, before, lane, lt);
          else wg_split<RecT, false>(s.LB[k], s.RP[k], src, dst, c0, c1, nsc, k, Z, before, lane, lt);
        }
        __syncthreads();
        if (k + 1 < tau) {
          const uint32_t o = c0 < c1 ? wg_count<RecT>(dst, c0, c1, k + 1, lane) : 0u;
          if (lane == 0) s.onesW[warp] = o;
          __syncthreads();
        }
      }

      // ---- 3. classes of every level: M_{k+1} = the zeros of M_k, then its ones ----
      // slot 2^k + r holds class r of level k (r = reversed k-bit prefix)
#ifdef WT_WG_DIAG_NORUNS
      const uint32_t kmax = 0;
#else
      const uint32_t kmax = HAS_OUT ? tau : tau - 1u;  // deepest level whose classes are needed
#endif
      auto classes_of = [&](uint32_t k) {
        const uint32_t nk = 1u << k;
        const uint32_t *LBw = reinterpret_cast<const uint32_t *>(s.LB[k]);
        const uint32_t Zk = s.Zs[k];
        for (uint32_t r = tid; r < nk; r += NT) {
          const uint32_t st = s.S[nk + r], cn = s.C[nk + r];
          const uint32_t a = wg_rank1(LBw, s.RP[k], st), b = wg_rank1(LBw, s.RP[k], st + cn);
          WT_CHECK(st + cn <= len && b >= a && b - a <= cn && a <= st, 202);
          s.C[2 * nk + r] = (uint16_t)(cn - (b - a));
          s.C[3 * nk + r] = (uint16_t)(b - a);
          s.S[2 * nk + r] = (uint16_t)(st - a);
          s.S[3 * nk + r] = (uint16_t)(Zk + a);
        }
      };
      if (warp == 0) {  // levels with <= 16 classes: warp 0 alone (warp-synchronous)
        for (uint32_t k = 0; k < min(kmax, 5u); k++) {
          classes_of(k);
          __syncwarp();
        }
      }
      __syncthreads();
      for (uint32_t k = 5; k < kmax; k++) {
        classes_of(k);
        __syncthreads();
      }
#ifdef WT_DEBUG
      if (tid == 0) {
        for (uint32_t k = 0; k <= kmax; k++) {
          uint32_t sum = 0;
          for (uint32_t r = 0; r < (1u << k); r++) sum += s.C[(1u << k) + r];
          WT_CHECK(sum == len, 207);
        }
      }
      __syncthreads();
#endif

      // ---- 4. runs of every level (thread per class), long runs' interior words by the warp ----
#ifdef WT_WG_DIAG_NORUNS
      for (uint32_t s0 = 1; s0 < 0; s0 += NT) {
#else
      for (uint32_t s0 = 1; s0 < ndig; s0 += NT) {
#endif
        const uint32_t slot = s0 + lane * CT_WARPS + warp;  // interleaved: long runs spread over the warps
        uint32_t ni = 0, gwA = 0, lsA = 0, kk = 0, Gr = 0, lsr = 0, cnr = 0;
        if (slot < ndig) {
          const uint32_t cn = s.C[slot];
          if (cn) {
            kk = 31 - __clz(slot);
            const uint32_t G = s.pos[slot], ls = s.S[slot];
            uint64_t *B = p.bits + (uint64_t)(p.l0 + kk) * p.wpl;
            uint32_t ones;
            ni = wg_run(s.CW[slot], s.CF[slot], reinterpret_cast<const uint32_t *>(s.LB[kk]), B, n32, G, ls, cn, ones);
            gwA = (G >> 6) + 1;
            lsA = ls + min(cn, 64u - (G & 63u));
            s.pos[slot] = G + cn;
            Gr = G; lsr = ls; cnr = cn;
            // fused A7: a run inside one 512-bit block adds the ones wg_run counted; other
            // short runs count their blocks here, long ones below (lane per block)
            if ((G >> 9) == ((G + cn - 1u) >> 9) && ones != ~0u) {
              if (ones) atomicAdd(p.blkcnt + (uint64_t)(p.l0 + kk) * p.bpl + (G >> 9), ones);
            } else if ((((G + cn - 1u) >> 9) - (G >> 9)) < 4u)
              run_blocks(p.blkcnt + (uint64_t)(p.l0 + kk) * p.bpl, reinterpret_cast<const uint32_t *>(s.LB[kk]),
                         s.RP[kk], G, ls, cn, G >> 9, (G + cn - 1u) >> 9, 1u);
          }
        }
        uint32_t m = __ballot_sync(FULL, ni != 0);
        while (m) {
          const int src_l = __ffs(m) - 1;
          m &= m - 1;
          const uint32_t g = __shfl_sync(FULL, gwA, src_l), l0 = __shfl_sync(FULL, lsA, src_l),
                         nn = __shfl_sync(FULL, ni, src_l), k2 = __shfl_sync(FULL, kk, src_l);
          uint64_t *B = p.bits + (uint64_t)(p.l0 + k2) * p.wpl;
          const uint32_t *LBw = reinterpret_cast<const uint32_t *>(s.LB[k2]);
          for (uint32_t w = lane; w < nn; w += 32) B[g + w] = lb_bits(LBw, l0 + 64u * w, 64);
        }
        m = __ballot_sync(FULL, cnr != 0 && (((Gr + cnr - 1u) >> 9) - (Gr >> 9)) >= 4u);
        while (m) {
          const int src_l = __ffs(m) - 1;
          m &= m - 1;
          const uint32_t G = __shfl_sync(FULL, Gr, src_l), ls = __shfl_sync(FULL, lsr, src_l),
                         cn = __shfl_sync(FULL, cnr, src_l), k2 = __shfl_sync(FULL, kk, src_l);
          run_blocks(p.blkcnt + (uint64_t)(p.l0 + k2) * p.bpl, reinterpret_cast<const uint32_t *>(s.LB[k2]), s.RP[k2],
                     G, ls, cn, (G >> 9) + lane, (G + cn - 1u) >> 9, 32u);
        }
      }

      // ---- 5. narrowed keys at their S_{l0+tau} position (A6) ----
#ifdef WT_WG_DIAG_NORUNS
      if constexpr (false) {
#else
      if constexpr (HAS_OUT) {
#endif
        const uint32_t fin = tau & 1u;
        uint32_t *KB = reinterpret_cast<uint32_t *>(s.rec[fin ^ 1u]);  // free after the last split
        for (uint32_t r = tid; r < ndig; r += NT) {
          const uint32_t d = rev_bits(r, tau);
          const uint32_t kp = s.kpos[d];
          KB[r] = kp - s.S[ndig + r];
          s.kpos[d] = kp + s.C[ndig + r];
        }
        __syncthreads();
        OutT *ko = reinterpret_cast<OutT *>(p.keys_out);
        const RecT *R = s.rec[fin];
#pragma unroll 4
        for (uint32_t i = tid; i < len; i += NT) {
          const uint32_t r = R[i];
          WT_CHECK((uint64_t)(uint32_t)(KB[r & dmask] + i) < p.n, 204);  // KB is a wrapped 32-bit base
          ko[KB[r & dmask] + i] = (OutT)(r >> tau);
        }
      }
      __syncthreads();
    }
    // ---- chain end: flush carried words (shared with the next chain or row) ----
    for (uint32_t slot = 1 + tid; slot < ndig; slot += NT) {
      if (s.CF[slot] & CF_VALID) {
        const uint32_t l = p.l0 + (31 - __clz(slot)), gw = s.pos[slot] >> 6;
        uint64_t *B = p.bits + (uint64_t)l * p.wpl;
        // the carried word holds this chain's bits [lo, pos & 63) (pos & 63 != 0: open end)
        const uint32_t lo = s.CF[slot] >> CF_LO_SHIFT, hi = s.pos[slot] & 63u;
        put_shared_word(&B[gw], s.CW[slot], (~0ull << lo) & ((1ull << hi) - 1ull));
      }
    }
    __syncthreads();
    c = s.cnext;
    __syncthreads();
  }
}

}  // namespace wtb
