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

    for (uint32_t start = cbeg; start < cend; start += TWT) {
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

// zeros[l] = n - (ones of level l), from the rank directory's level totals.
__global__ void k_wm_zeros(const uint64_t *__restrict__ rank_super, uint64_t spl, uint32_t L, uint64_t n,
                           uint64_t *__restrict__ zeros, const uint32_t *err) {
  if (*err) return;
  const uint32_t l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l < L) zeros[l] = n - rank_super[(uint64_t)l * spl + spl - 1];
}

// Batched queries: a 0 bit at level l maps i -> rank0(i),
// a 1 bit maps i -> zeros[l] + rank1(i).
__global__ void k_wm_access(TreeView t, const uint64_t *__restrict__ zeros, const uint64_t *__restrict__ pos,
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

__global__ void k_wm_rank(TreeView t, const uint64_t *__restrict__ zeros, uint64_t sigma,
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
