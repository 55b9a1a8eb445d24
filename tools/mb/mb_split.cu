// Microbenchmark: per-warp tiles, in-tile wavelet-matrix order (every split is
// one tile-wide stable split), 8 levels of u8 records.  Measures the floor of
// the element-moving split loop on B200 (no run output, bits written densely).
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr uint32_t FULL = 0xffffffffu;
__device__ __forceinline__ uint32_t lanemask_lt() { uint32_t m; asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m)); return m; }
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t lds8(uint32_t a) { uint32_t v; asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a)); return v; }
__device__ __forceinline__ void sts8(uint32_t a, uint32_t v) { asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v) : "memory"); }

#ifndef MB_T
#define MB_T 4096
#endif
#ifndef MB_U
#define MB_U 8
#endif
#ifndef MB_NW
#define MB_NW 4
#endif
constexpr int T = MB_T, U = MB_U, NW = MB_NW;

struct WS {
  alignas(16) uint8_t a[T];
  alignas(16) uint8_t b[T];
  alignas(16) uint32_t LB[T / 32];
  uint32_t H[256];
};

__global__ void __launch_bounds__(NW * 32) k_mb(const uint8_t *__restrict__ in, uint64_t n, uint32_t *__restrict__ out,
                                               uint32_t *counter) {
  extern __shared__ __align__(16) uint8_t smraw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WS &s = reinterpret_cast<WS *>(smraw)[warp];
  const uint32_t lt = lanemask_lt();
  const uint64_t ntiles = n / T;
  while (true) {
    uint32_t tile = 0;
    if (lane == 0) tile = atomicAdd(counter, 1u);
    tile = __shfl_sync(FULL, tile, 0);
    if (tile >= ntiles) break;
    for (int i = lane; i < 256; i += 32) s.H[i] = 0;
    __syncwarp();
    const uint4 *v = reinterpret_cast<const uint4 *>(in + (uint64_t)tile * T);
#pragma unroll
    for (int j = 0; j < T / 512; j++) {
      const uint4 q = __ldcs(v + lane + 32 * j);
      reinterpret_cast<uint4 *>(s.a)[lane + 32 * j] = q;
      const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int t = 0; t < 4; t++)
#pragma unroll
        for (int b = 0; b < 4; b++) atomicAdd(&s.H[(w[t] >> (8 * b)) & 255u], 1u);
    }
    __syncwarp();
    // zeros of each bit over the whole tile
    uint32_t zb[8];
#pragma unroll
    for (int b = 0; b < 8; b++) zb[b] = 0;
    for (int d = lane; d < 256; d += 32) {
      const uint32_t h = s.H[d];
#pragma unroll
      for (int b = 0; b < 8; b++) zb[b] += ((d >> b) & 1) ? 0u : h;
    }
#pragma unroll
    for (int b = 0; b < 8; b++) zb[b] = __reduce_add_sync(FULL, zb[b]);
    uint32_t src = smem_u32(s.a), dst = smem_u32(s.b);
#pragma unroll 1
    for (int k = 0; k < 8; k++) {
      const int bit = 7 - k;
      uint32_t bitmask = 1u << bit;
      asm("" : "+r"(bitmask));
      uint32_t Zk = 0;
#pragma unroll
      for (int b = 0; b < 8; b++) if (b == bit) Zk = zb[b];
      // dest bases: ones at dst + Zk + Orun + o ; zeros at dst + pos - Orun - o
      uint32_t B1 = dst + Zk;            // + Orun (uniform)
      uint32_t B0 = dst + lane;          // + pos base - Orun
      const uint32_t sA = src + lane;
      const bool mv = k < 7;
#pragma unroll 1
      for (int c = 0; c < T / 32; c += U) {
        uint32_t r[U], m[U];
#pragma unroll
        for (int u = 0; u < U; u++) r[u] = lds8(sA + (c + u) * 32);
#pragma unroll
        for (int u = 0; u < U; u++) {
          const bool P = (r[u] & bitmask) != 0;
          m[u] = __ballot_sync(FULL, P);
          if (mv) {
            const uint32_t o = __popc(m[u] & lt);
            sts8(P ? B1 + o : B0 - o, r[u]);
          }
          const uint32_t cnt = __popc(m[u]);
          B1 += cnt;
          B0 += 32 - cnt;
        }
        if (lane < U) {
          uint32_t mm = m[0];
#pragma unroll
          for (int u = 1; u < U; u++) if (lane == u) mm = m[u];
          s.LB[c + lane] = mm;
        }
      }
      __syncwarp();
      uint32_t *o = out + ((uint64_t)tile * 8 + k) * (T / 32);
      for (int i = lane; i < T / 32; i += 32) o[i] = s.LB[i];
      __syncwarp();
      const uint32_t t = src; src = dst; dst = t;
    }
  }
}

__global__ void k_fill(uint8_t *p, uint64_t n, uint64_t seed) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull; z ^= z >> 31;
    p[i] = (uint8_t)(z >> 56);
  }
}

int main(int argc, char **argv) {
  const uint64_t n = 1ull << 28;
  uint8_t *in; uint32_t *out, *cnt;
  cudaMalloc(&in, n); cudaMalloc(&out, n); cudaMalloc(&cnt, 4);
  k_fill<<<4096, 256>>>(in, n, 4);
  const size_t smem = NW * sizeof(WS);
  cudaFuncSetAttribute(k_mb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0, nsm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mb, NW * 32, smem);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9;
  for (int it = 0; it < 6; it++) {
    cudaMemsetAsync(cnt, 0, 4);
    cudaEventRecord(e0);
    k_mb<<<nsm * per_sm, NW * 32, smem>>>(in, n, out, cnt);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (it) best = ms < best ? ms : best;
  }
  printf("T=%d U=%d NW=%d smem/CTA=%zu CTAs/SM=%d warps/SM=%d : %.3f ms for 2^28 x 8 levels  -> %.2f SMSP-cycles/chunk-level @1.965GHz, err=%s\n",
         T, U, NW, smem, per_sm, per_sm * NW, best, best * 1e-3 * 1.965e9 * nsm * 4 / (n / 32.0 * 8),
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
