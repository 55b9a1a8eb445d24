// wt_small.cuh -- trees of one or two levels over byte symbols (sigma <= 4:
// DNA-like inputs), built without the fused group pass.
//
// Level 0 is the top bit of S in S order (Fig. 1 l.4 on the root).
// With two levels, level 1 holds the low bit of the symbols whose top bit is
// 0, in S order, followed by the low bit of those whose top bit is 1 (the
// stable split of the root, Fig. 1 l.12-17): two compacted bit streams.
// Each lane takes 16 consecutive bytes and works on them as packed words:
// the level bits of 4 bytes come from one multiply (bit i of byte i lands in
// bit 24+i), the compaction of the low bits by side uses a 256-entry nibble
// table (pext of 4 bits by a 4-bit mask), a warp scan places every lane's
// bits in its warp's part of the stream, staged in shared memory; the
// streams' offsets come from per-tile zero counts (k_small_count) and their
// scan.  Only the first and last word of each warp's part are shared.
#pragma once
#include "wt_common.cuh"

namespace wtb {

constexpr uint32_t SMALL_WARPS = 8, SMALL_BYTES = 16, SMALL_ITERS = 8;
constexpr uint32_t SMALL_WARP_SPAN = 32 * SMALL_BYTES * SMALL_ITERS;   // 4096 symbols per warp
constexpr uint32_t SMALL_TILE = SMALL_WARPS * SMALL_WARP_SPAN;          // 32768 symbols per CTA

// bits b of the 4 bytes of w, in byte order (bit i <- byte i)
__device__ __forceinline__ uint32_t small_movemask4(uint32_t w, uint32_t b) {
  return (((w >> b) & 0x01010101u) * 0x01020408u) >> 24;
}

// the 16 symbols of lane `lane` in iteration `it` of a warp: bit masks of the
// top bit (m1), the low bit (m0) and of the symbols inside [0, n) (vm);
// bad |= a symbol >= sigma
__device__ __forceinline__ void small_load16(const uint8_t *__restrict__ S, uint64_t n, uint64_t e0, uint32_t sigma,
                                             uint32_t topbit, uint32_t &m1, uint32_t &m0, uint32_t &vm, bool &bad) {
  uint32_t w[4] = {0u, 0u, 0u, 0u};
  if (e0 + SMALL_BYTES <= n) {
    const uint4 q = __ldcs(reinterpret_cast<const uint4 *>(S + e0));
    w[0] = q.x; w[1] = q.y; w[2] = q.z; w[3] = q.w;
    vm = 0xFFFFu;
  } else {
    vm = 0;
    for (uint32_t i = 0; i < SMALL_BYTES; i++)
      if (e0 + i < n) {
        w[i >> 2] |= (uint32_t)S[e0 + i] << (8 * (i & 3));
        vm |= 1u << i;
      }
  }
  m1 = m0 = 0;
#pragma unroll
  for (int k = 0; k < 4; k++) {
    // byte >= sigma (sigma <= 4 < 128): bit 7 of (byte | 0x80) - sigma, per byte, no borrows
    const uint32_t ge = ((w[k] | 0x80808080u) - sigma * 0x01010101u) & 0x80808080u;
    const uint32_t vk = (vm >> (4 * k)) & 0xFu;
    bad |= (small_movemask4(ge, 7) & vk) != 0;
    m1 |= small_movemask4(w[k], topbit) << (4 * k);
    m0 |= small_movemask4(w[k], 0) << (4 * k);
  }
  m1 &= vm;
  m0 &= vm;
}

// zeros of the top bit per tile (zc[tile]); validation S[i] < sigma
static __global__ void __launch_bounds__(SMALL_WARPS * 32)
    k_small_count(const uint8_t *__restrict__ S, uint64_t n, uint32_t sigma, uint32_t topbit,
                  uint32_t *__restrict__ zc, uint32_t *err) {
  __shared__ uint32_t tz;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) tz = 0;
  __syncthreads();
  const uint64_t wb = (uint64_t)blockIdx.x * SMALL_TILE + (uint64_t)warp * SMALL_WARP_SPAN;
  uint32_t z = 0;
  bool bad = false;
#pragma unroll
  for (uint32_t it = 0; it < SMALL_ITERS; it++) {
    const uint64_t e0 = wb + ((uint64_t)it * 32 + lane) * SMALL_BYTES;
    uint32_t m1, m0, vm;
    small_load16(S, n, e0, sigma, topbit, m1, m0, vm, bad);
    z += __popc(vm & ~m1);
  }
  z = __reduce_add_sync(FULL, z);
  if (lane == 0) atomicAdd(&tz, z);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(err, 1u);
  if (threadIdx.x == 0) zc[blockIdx.x] = tz;
}

// OR a word of a warp's stream part [rs, re) into the level (plain store when
// the word lies wholly inside the part)
__device__ __forceinline__ void small_out(uint32_t *B32, uint64_t gw, uint32_t v, uint64_t rs, uint64_t re) {
  const uint64_t lo = gw * 32;
  if (rs <= lo && lo + 32 <= re) B32[gw] = v;
  else if (v) atomicOr(&B32[gw], v);
}

static __global__ void __launch_bounds__(SMALL_WARPS * 32)
    k_small_write(const uint8_t *__restrict__ S, uint64_t n, uint32_t L, const uint32_t *__restrict__ zoff,
                  const uint64_t *__restrict__ ztot, uint64_t *__restrict__ bits, uint64_t wpl) {
  __shared__ uint8_t lut[256];                     // pext of a nibble x by a nibble mask: lut[mask << 4 | x]
  __shared__ uint32_t wz[SMALL_WARPS];
  __shared__ uint32_t stage[SMALL_WARPS][2][SMALL_WARP_SPAN / 32 + 2];  // per warp: zero-side, one-side bits
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t lt = lanemask_lt();
  const uint32_t topbit = L - 1;
  {
    const uint32_t mk = threadIdx.x >> 4, x = threadIdx.x & 15;
    uint32_t r = 0, c = 0;
    for (uint32_t i = 0; i < 4; i++)
      if ((mk >> i) & 1u) r |= ((x >> i) & 1u) << c++;
    lut[threadIdx.x] = (uint8_t)r;
  }
  for (uint32_t i = lane; i < 2 * (SMALL_WARP_SPAN / 32 + 2); i += 32) (&stage[warp][0][0])[i] = 0;
  const uint64_t wb = (uint64_t)blockIdx.x * SMALL_TILE + (uint64_t)warp * SMALL_WARP_SPAN;
  uint16_t *B0 = reinterpret_cast<uint16_t *>(bits);
  uint32_t m1s[SMALL_ITERS], m0s[SMALL_ITERS], vms[SMALL_ITERS];
  uint32_t z = 0;
  bool bad = false;
#pragma unroll
  for (uint32_t it = 0; it < SMALL_ITERS; it++) {
    const uint64_t e0 = wb + ((uint64_t)it * 32 + lane) * SMALL_BYTES;
    small_load16(S, n, e0, 4, topbit, m1s[it], m0s[it], vms[it], bad);
    if (e0 < n) B0[e0 >> 4] = (uint16_t)m1s[it];  // level 0: 16 aligned bits per lane
    z += __popc(vms[it] & ~m1s[it]);
  }
  if (L < 2) return;
  z = __reduce_add_sync(FULL, z);
  if (lane == 0) wz[warp] = z;
  __syncthreads();  // lut, wz
  uint64_t zb = zoff[blockIdx.x];
  for (int w = 0; w < warp; w++) zb += wz[w];
  // per lane: compacted low bits of each side, placed by a warp scan into the staging
  uint32_t zpos = 0, opos = 0;  // running bits of this warp's parts
#pragma unroll
  for (uint32_t it = 0; it < SMALL_ITERS; it++) {
    const uint32_t m1 = m1s[it], m0 = m0s[it], vm = vms[it];
    const uint32_t zmask = vm & ~m1;
    uint32_t zbits = 0, obits = 0, zc = 0, oc = 0;
#pragma unroll
    for (uint32_t k = 0; k < 4; k++) {
      const uint32_t x = (m0 >> (4 * k)) & 15u, zm = (zmask >> (4 * k)) & 15u, om = (m1 >> (4 * k)) & 15u;
      zbits |= (uint32_t)lut[(zm << 4) | x] << zc;
      zc += __popc(zm);
      obits |= (uint32_t)lut[(om << 4) | x] << oc;
      oc += __popc(om);
    }
    const uint32_t zi = warp_incl_scan(zc, lane), oi = warp_incl_scan(oc, lane);
    const uint32_t zo = zpos + zi - zc, oo = opos + oi - oc;
    if (zc) {
      atomicOr(&stage[warp][0][zo >> 5], zbits << (zo & 31));
      if ((zo & 31) + zc > 32) atomicOr(&stage[warp][0][(zo >> 5) + 1], zbits >> (32 - (zo & 31)));
    }
    if (oc) {
      atomicOr(&stage[warp][1][oo >> 5], obits << (oo & 31));
      if ((oo & 31) + oc > 32) atomicOr(&stage[warp][1][(oo >> 5) + 1], obits >> (32 - (oo & 31)));
    }
    zpos += __shfl_sync(FULL, zi, 31);
    opos += __shfl_sync(FULL, oi, 31);
  }
  __syncwarp();
  // copy the warp's two parts out: zero side at zb, one side at Z + (ones before)
  const uint64_t Z = *ztot;
  const uint64_t ob = Z + (wb < n ? wb : n) - zb;
  uint32_t *B1 = reinterpret_cast<uint32_t *>(bits + wpl);
#pragma unroll
  for (int side = 0; side < 2; side++) {
    const uint64_t g = side ? ob : zb;
    const uint32_t cnt = side ? opos : zpos;
    if (!cnt) continue;
    const uint32_t *st = stage[warp][side];
    const uint64_t w0 = g >> 5, w1 = (g + cnt - 1) >> 5;
    const uint32_t sh = (uint32_t)(g & 31);
    for (uint64_t gw = w0 + lane; gw <= w1; gw += 32) {
      const uint32_t j = (uint32_t)(gw - w0);  // output word j takes staging bits [32j - sh, 32j - sh + 32)
      const uint32_t lo = j > 0 ? st[j - 1] : 0u, hi = st[j];
      const uint32_t v = sh ? ((hi << sh) | (lo >> (32 - sh))) : hi;
      small_out(B1, gw, v, g, g + cnt);
    }
  }
}

// node table of a one- or two-level tree (n > 0)
static __global__ void k_small_nodes(uint32_t L, uint64_t n, const uint64_t *__restrict__ ztot,
                                     uint64_t *__restrict__ ptr, uint32_t *__restrict__ key,
                                     uint32_t *__restrict__ start) {
  if (threadIdx.x || blockIdx.x) return;
  ptr[0] = 0;
  ptr[1] = 1;
  key[0] = 0;
  start[0] = 0;
  if (L == 2) {
    const uint64_t Z = *ztot;
    uint32_t j = 1;
    if (Z > 0) { key[j] = 0; start[j] = 0; j++; }
    if (n > Z) { key[j] = 1; start[j] = (uint32_t)Z; j++; }
    ptr[2] = j;
  }
}

}  // namespace wtb
