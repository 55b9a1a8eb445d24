// Throughput of match.any.sync (MATCH.ANY) vs an 8-ballot peer mask, per SM.
#include <cstdio>
#include <cstdint>
__global__ void k_match(const uint32_t *in, uint32_t *out, int iters) {
  uint32_t x = in[blockIdx.x * blockDim.x + threadIdx.x], acc = 0;
  for (int i = 0; i < iters; i++) {
    const uint32_t m = __match_any_sync(0xffffffffu, x & 255u);
    acc += __popc(m & ((1u << (threadIdx.x & 31)) - 1u));
    x = x * 1664525u + 1013904223u;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_ballot8(const uint32_t *in, uint32_t *out, int iters) {
  uint32_t x = in[blockIdx.x * blockDim.x + threadIdx.x], acc = 0;
  for (int i = 0; i < iters; i++) {
    const uint32_t d = x & 255u;
    uint32_t peers = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < 8; b++) {
      const uint32_t v = __ballot_sync(0xffffffffu, (d >> b) & 1u);
      peers &= ((d >> b) & 1u) ? v : ~v;
    }
    acc += __popc(peers & ((1u << (threadIdx.x & 31)) - 1u));
    x = x * 1664525u + 1013904223u;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  const int nb = 148 * 8, nt = 256, iters = 4096;
  uint32_t *in, *out;
  cudaMalloc(&in, nb * nt * 4); cudaMalloc(&out, nb * nt * 4);
  cudaMemset(in, 7, nb * nt * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int v = 0; v < 2; v++) {
    float best = 1e9;
    for (int r = 0; r < 4; r++) {
      cudaEventRecord(e0);
      if (v == 0) k_match<<<nb, nt>>>(in, out, iters); else k_ballot8<<<nb, nt>>>(in, out, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (r) best = ms < best ? ms : best;
    }
    const double warp_ops = (double)nb * nt / 32 * iters;
    printf("%s: %.3f ms, %.2f SM-cycles per warp-op (incl. popc + lcg)\n", v ? "8 ballots" : "match.any", best,
           best * 1e-3 * 1.965e9 * 148 / warp_ops);
  }
  return 0;
}
