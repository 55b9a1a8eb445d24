// wt_common.cuh -- constants and warp/block helpers shared by the kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace wtb {

constexpr uint32_t FULL = 0xffffffffu;
#ifndef WT_TW
#define WT_TW 4096
#endif
constexpr int TW = WT_TW;                // elements per warp tile
constexpr int NCH = TW / 32;             // 32-element chunks per tile
constexpr int TAU_MAX = 8;               // levels fused per HBM pass
constexpr int NDIG = 1 << TAU_MAX;       // digit values per pass

#ifdef WT_DEBUG
static __device__ uint32_t g_wt_dbg[4];
#define WT_CHECK(cond, code)                                                        \
  do {                                                                              \
    if (!(cond)) {                                                                  \
      if (atomicCAS(&::wtb::g_wt_dbg[0], 0u, (uint32_t)(code)) == 0u) {             \
        ::wtb::g_wt_dbg[1] = blockIdx.x;                                            \
        ::wtb::g_wt_dbg[2] = threadIdx.x;                                           \
      }                                                                             \
    }                                                                               \
  } while (0)
#else
#define WT_CHECK(cond, code) \
  do {                       \
  } while (0)
#endif

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t *p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(FULL, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// Warp-cooperative exclusive scan of a[0..cnt) into out[0..cnt], out[cnt] = total.
// a and out live in shared memory; they may alias.
__device__ __forceinline__ void warp_exscan(const uint32_t *a, int cnt, uint32_t *out, int lane) {
  const int per = (cnt + 31) >> 5;
  const int lo = min(lane * per, cnt);
  const int hi = min(lo + per, cnt);
  uint32_t s = 0;
  for (int i = lo; i < hi; i++) s += a[i];
  const uint32_t incl = warp_incl_scan(s, lane);
  uint32_t run = incl - s;
  const uint32_t total = __shfl_sync(FULL, incl, 31);
  __syncwarp();
  for (int i = lo; i < hi; i++) {
    uint32_t v = a[i];
    out[i] = run;
    run += v;
  }
  if (lane == 0) out[cnt] = total;
  __syncwarp();
}

// Block-wide exclusive scan (any blockDim multiple of 32, <= 1024); shm needs
// 33 words.  Returns the exclusive prefix of v; *total = block sum.
__device__ __forceinline__ uint32_t block_exscan(uint32_t v, uint32_t *shm, uint32_t *total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t incl = warp_incl_scan(v, lane);
  __syncthreads();
  if (lane == 31) shm[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < (int)(blockDim.x >> 5) ? shm[lane] : 0u;
    uint32_t wi = warp_incl_scan(w, lane);
    shm[lane] = wi - w;
    if (lane == 31) shm[32] = wi;
  }
  __syncthreads();
  *total = shm[32];
  return shm[warp] + incl - v;
}

// Explicit shared-memory (state space .shared) accesses by 32-bit byte address.
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <typename T>
__device__ __forceinline__ uint32_t lds(uint32_t a) {
  uint32_t v;
  if constexpr (sizeof(T) == 1) asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
  else if constexpr (sizeof(T) == 2) asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(a));
  else asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
template <typename T>
__device__ __forceinline__ void sts(uint32_t a, uint32_t v) {
  if constexpr (sizeof(T) == 1) asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v) : "memory");
  else if constexpr (sizeof(T) == 2) asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "r"(v) : "memory");
  else asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

__device__ __forceinline__ void sts_v4(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}

// Bits [base, base+64) of a little-endian bit array of nw u32 words; bits
// outside [0, 32*nw) read as 0.  base may be negative (> -64).
__device__ __forceinline__ uint64_t extract64(const uint32_t *w, int base, int nw) {
  const int b = base < 0 ? 0 : base;
  const int wi = b >> 5, sh = b & 31;
  const uint32_t x0 = wi < nw ? w[wi] : 0u;
  const uint32_t x1 = wi + 1 < nw ? w[wi + 1] : 0u;
  const uint32_t x2 = wi + 2 < nw ? w[wi + 2] : 0u;
  uint64_t v = (((uint64_t)x1 << 32) | x0) >> sh;
  if (sh) v |= (uint64_t)x2 << (64 - sh);
  if (base < 0) v <<= (-base);
  return v;
}

}  // namespace wtb
