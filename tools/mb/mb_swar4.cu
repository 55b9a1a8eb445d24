// Microbenchmark 2: SWAR lane-major split.  Lane l holds 8 consecutive u8
// records of a 256-record superchunk (LDS.64); in-lane exclusive prefix of the
// level bits by IMAD (bytes), cross-lane prefix of the lane totals (0..8) by 4
// ballots + 4 POPC.  Per-warp tiles, in-tile wavelet-matrix order.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr uint32_t FULL = 0xffffffffu;
__device__ __forceinline__ uint32_t lanemask_lt() { uint32_t m; asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m)); return m; }
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void sts8(uint32_t a, uint32_t v) { asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v) : "memory"); }
__device__ __forceinline__ uint32_t ballot_bit(uint32_t v, uint32_t m) {
  uint32_t r;
  asm volatile("{.reg .pred p; .reg .b32 t; and.b32 t, %1, %2; setp.ne.u32 p, t, 0; vote.sync.ballot.b32 %0, p, 0xffffffff;}"
               : "=r"(r) : "r"(v), "r"(m));
  return r;
}
__device__ __forceinline__ uint2 lds64(uint32_t a) { uint2 v; asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a)); return v; }

#ifndef MB_T
#define MB_T 4096
#endif
#ifndef MB_NW
#define MB_NW 4
#endif
#ifndef MB_SHFL
#define MB_SHFL 1
#endif
constexpr int T = MB_T, NW = MB_NW;

struct WS {
  alignas(16) uint8_t a[T];
  alignas(16) uint8_t b[T];
  alignas(16) uint8_t LB[T / 8];
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
      uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int t = 0; t < 4; t++) w[t] = __byte_perm(__brev(w[t]), 0, 0x0123);
      reinterpret_cast<uint4 *>(s.a)[lane + 32 * j] = make_uint4(w[0], w[1], w[2], w[3]);
#pragma unroll
      for (int t = 0; t < 4; t++)
#pragma unroll
        for (int b = 0; b < 4; b++) atomicAdd(&s.H[(w[t] >> (8 * b)) & 255u], 1u);
    }
    __syncwarp();
    uint32_t zb[8];
#pragma unroll
    for (int b = 0; b < 8; b++) zb[b] = 0;
    for (int d = lane; d < 256; d += 32) {
      const uint32_t h = s.H[d];
#pragma unroll
      for (int b = 0; b < 8; b++) zb[b] += ((d >> (7 - b)) & 1) ? 0u : h;
    }
#pragma unroll
    for (int b = 0; b < 8; b++) zb[b] = __reduce_add_sync(FULL, zb[b]);
    uint32_t src = smem_u32(s.a), dst = smem_u32(s.b);
    const uint32_t lbA = smem_u32(s.LB) + lane;
#pragma unroll 1
    for (int k = 0; k < 8; k++) {
      const int bit = 7 - k;  // zb indexed by the original bit
      uint32_t Zk = 0;
#pragma unroll
      for (int b = 0; b < 8; b++) if (b == bit) Zk = zb[b];
      uint32_t B1 = dst + Zk, B0 = dst;
      const uint32_t sA = src + 8 * lane;
      const bool mv = k < 7;
#pragma unroll 2
      for (int c = 0; c < T / 256; c++) {
        const uint2 xx = lds64(sA + 256 * c);
        const uint32_t t_lo = xx.x & 0x01010101u, t_hi = xx.y & 0x01010101u;
        const uint32_t pre_lo = t_lo * 0x01010100u;
        const uint32_t inc_lo = pre_lo + t_lo;                 // byte 3: ones in lo 4
        const uint32_t pre_hi = t_hi * 0x01010100u + __umulhi(inc_lo, 0x100u) * 0x01010101u;
        const uint32_t inc = pre_hi + t_hi;                    // byte 3: lane total (0..8)
        const uint32_t v0 = ballot_bit(inc, 1u << 24), v1 = ballot_bit(inc, 2u << 24),
                       v2 = ballot_bit(inc, 4u << 24), v3 = ballot_bit(inc, 8u << 24);
        const uint32_t O = __popc(v0 & lt) + 2 * __popc(v1 & lt) + 4 * __popc(v2 & lt) + 8 * __popc(v3 & lt);
        const uint32_t S = __shfl_sync(FULL, O + __umulhi(inc, 0x100u), 31);
        if (mv) {
          const uint32_t D0 = B0 + 8 * lane - O;                // zeros of this lane start here
          const uint32_t A = (B1 + O - D0) | 0x10000u;          // {h0 = ones-minus-zeros base, h1 = 1}
          const uint32_t M_lo = t_lo * 0xffu, M_hi = t_hi * 0xffu;
          const uint32_t q_lo = (pre_lo & M_lo) | ((0x03020100u - pre_lo) & ~M_lo);
          const uint32_t q_hi = (pre_hi & M_hi) | ((0x07060504u - pre_hi) & ~M_hi);
          const uint32_t xs_lo = xx.x >> 1, xs_hi = xx.y >> 1;
#pragma unroll
          for (int w = 0; w < 2; w++) {
            const uint32_t q = w ? q_hi : q_lo, t = w ? t_hi : t_lo, xs = w ? xs_hi : xs_lo;
            const uint32_t tq0 = __byte_perm(t, q, 0x5140), tq1 = __byte_perm(t, q, 0x7362);
            sts8(__dp2a_lo(A, tq0, D0), xs);
            sts8(__dp2a_hi(A, tq0, D0), __byte_perm(xs, 0, 0x1));
            sts8(__dp2a_lo(A, tq1, D0), __byte_perm(xs, 0, 0x2));
            sts8(__dp2a_hi(A, tq1, D0), __byte_perm(xs, 0, 0x3));
          }
        }
        const uint32_t byte = __umulhi(t_lo * 0x01020408u, 0x100u) | (__umulhi(t_hi * 0x01020408u, 0x100u) << 4);
        sts8(lbA + 32 * c, byte);
        B1 += S;
        B0 += 256 - S;
      }
      __syncwarp();
      uint32_t *o = out + ((uint64_t)tile * 8 + k) * (T / 32);
      for (int i = lane; i < T / 32; i += 32) o[i] = reinterpret_cast<const uint32_t *>(s.LB)[i];
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

// CPU check of one tile: level-k bits in matrix order
static void check(const uint8_t *h_in, const uint32_t *h_out, int tile) {
  uint8_t A[T], B[T];
  for (int i = 0; i < T; i++) A[i] = h_in[(size_t)tile * T + i];
  int bad = 0;
  for (int k = 0; k < 8; k++) {
    const int bit = 7 - k;
    for (int i = 0; i < T; i++) {
      const uint32_t got = (h_out[((size_t)tile * 8 + k) * (T / 32) + i / 32] >> (i % 32)) & 1u;
      if (got != ((A[i] >> bit) & 1u)) bad++;
    }
    int z = 0;
    for (int i = 0; i < T; i++) if (!((A[i] >> bit) & 1)) B[z++] = A[i];
    for (int i = 0; i < T; i++) if ((A[i] >> bit) & 1) B[z++] = A[i];
    for (int i = 0; i < T; i++) A[i] = B[i];
  }
  printf("check tile %d: %s (%d bad bits)\n", tile, bad ? "FAIL" : "ok", bad);
}

int main() {
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
  printf("SWAR T=%d NW=%d SHFL=%d smem/CTA=%zu CTAs/SM=%d warps/SM=%d : %.3f ms -> %.2f SMSP-cycles/chunk-level, err=%s\n",
         T, NW, MB_SHFL, smem, per_sm, per_sm * NW, best, best * 1e-3 * 1.965e9 * nsm * 4 / (n / 32.0 * 8),
         cudaGetErrorString(cudaGetLastError()));
  uint8_t *h_in = (uint8_t *)malloc(3 * T);
  uint32_t *h_out = (uint32_t *)malloc((size_t)3 * 8 * T / 8);
  cudaMemcpy(h_in, in, 3 * T, cudaMemcpyDeviceToHost);
  cudaMemcpy(h_out, out, (size_t)3 * 8 * T / 8, cudaMemcpyDeviceToHost);
  for (int t = 0; t < 3; t++) check(h_in, h_out, t);
  return 0;
}
