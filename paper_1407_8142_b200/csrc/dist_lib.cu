// dist_lib.cu -- extern "C" helpers of the sharded build (
// orchestration in paper_1407_8142_b200/dist.py): wt_digit_counts, wt_digits,
// wt_partition, wt_gather_bits, wt_create, wt_finish of include/wt.h.
#include "wt_host.cuh"
#include "wt_dist.cuh"
#include "wt_rank.cuh"

using namespace wtb;
using namespace wthost;

// ============ sharded build helpers (orchestration in dist.py) ============
namespace {

template <typename T>
int partition_impl(const void *d_in, uint64_t n, uint64_t sigma, uint32_t shift, uint32_t tau, void *d_out,
                   uint64_t *d_counts, bool validate, cudaStream_t s) {
  const uint32_t ndig = 1u << tau;
  const uint32_t ntiles = (uint32_t)((n + PART_TILE - 1) / PART_TILE);
  Allocs A{s};
  uint32_t *thT = A.alloc<uint32_t>((uint64_t)ndig * std::max<uint32_t>(ntiles, 1), false);
  uint64_t *tot = d_counts ? d_counts : A.alloc<uint64_t>(ndig, false);
  uint32_t *err = A.alloc<uint32_t>(1, false);
  if (A.fail) { A.free_scratch(); return WT_ENOMEM; }
  cudaError_t ce = cudaMemsetAsync(err, 0, sizeof(uint32_t), s);
  if (ntiles) {
    const unsigned g = (unsigned)std::min<uint64_t>(ntiles, 8ull * num_sms());
    k_part_hist<T><<<g, PART_THREADS, 0, s>>>((const T *)d_in, n, sigma, shift, ndig, ntiles, thT, err);
    k_part_scan<<<ndig, 1024, 0, s>>>(thT, ntiles, tot);
    if (d_out) k_part_scatter<T><<<ntiles, PART_THREADS, 0, s>>>((const T *)d_in, n, shift, tau, ntiles, thT, tot, (T *)d_out);
  } else if (ce == cudaSuccess) {
    ce = cudaMemsetAsync(tot, 0, ndig * sizeof(uint64_t), s);
  }
  if (ce == cudaSuccess) ce = cudaGetLastError();
  uint32_t h_err = 0;
  if (validate && ce == cudaSuccess) ce = cudaMemcpyAsync(&h_err, err, sizeof(uint32_t), cudaMemcpyDeviceToHost, s);
  A.free_scratch();
  if (validate && ce == cudaSuccess) ce = cudaStreamSynchronize(s);
  if (ce != cudaSuccess) return WT_ECUDA;
  return h_err ? WT_ESYMBOL : WT_OK;
}

int partition_dispatch(const void *d_in, uint64_t n, uint32_t eb, uint64_t sigma, uint32_t shift, uint32_t tau,
                       void *d_out, uint64_t *d_counts, bool validate, void *stream) {
  if ((n > 0 && !d_in) || (eb != 1 && eb != 2 && eb != 4) || tau < 1 || tau > 8 || shift >= 32) return WT_EINVAL;
  if (sigma < 1 || sigma > (1ull << (8 * eb)) || n >= (1ull << 32)) return WT_EINVAL;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  configure_pool_once();
  if (eb == 1) return partition_impl<uint8_t>(d_in, n, sigma, shift, tau, d_out, d_counts, validate, s);
  if (eb == 2) return partition_impl<uint16_t>(d_in, n, sigma, shift, tau, d_out, d_counts, validate, s);
  return partition_impl<uint32_t>(d_in, n, sigma, shift, tau, d_out, d_counts, validate, s);
}

}  // namespace

extern "C" {

int wt_digit_counts(const void *d_seq, uint64_t n, uint32_t elem_bytes, uint64_t sigma, uint32_t shift, uint32_t tau,
                    uint64_t *d_counts, void *stream) {
  if (!d_counts) return WT_EINVAL;
  return partition_dispatch(d_seq, n, elem_bytes, sigma, shift, tau, nullptr, d_counts, true, stream);
}

int wt_partition(const void *d_in, uint64_t n, uint32_t elem_bytes, uint32_t shift, uint32_t tau, void *d_out,
                 void *stream) {
  if (n > 0 && !d_out) return WT_EINVAL;
  return partition_dispatch(d_in, n, elem_bytes, 1ull << (8 * elem_bytes), shift, tau, d_out, nullptr, false, stream);
}

int wt_digits(const void *d_seq, uint64_t n, uint32_t elem_bytes, uint32_t shift, uint32_t tau, uint8_t *d_out,
              void *stream) {
  if ((n > 0 && (!d_seq || !d_out)) || (elem_bytes != 1 && elem_bytes != 2 && elem_bytes != 4) || tau < 1 ||
      tau > 8 || shift >= 32)
    return WT_EINVAL;
  if (!n) return WT_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const unsigned g = (unsigned)std::min<uint64_t>((n + 255) / 256, 8ull * num_sms());
  const uint32_t m = (1u << tau) - 1u;
  if (elem_bytes == 1) k_digits<uint8_t><<<g, 256, 0, s>>>((const uint8_t *)d_seq, n, shift, m, d_out);
  else if (elem_bytes == 2) k_digits<uint16_t><<<g, 256, 0, s>>>((const uint16_t *)d_seq, n, shift, m, d_out);
  else k_digits<uint32_t><<<g, 256, 0, s>>>((const uint32_t *)d_seq, n, shift, m, d_out);
  return cudaGetLastError() == cudaSuccess ? WT_OK : WT_ECUDA;
}

int wt_gather_bits(const uint64_t *d_src, const uint64_t *d_segs, uint64_t nseg, uint64_t *d_dst, uint64_t dst_words,
                   void *stream) {
  if ((dst_words && !d_dst) || (nseg && (!d_segs || !d_src))) return WT_EINVAL;
  if (!dst_words) return WT_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint64_t per = (uint64_t)GB_WORDS * GB_WPT;
  k_gather_bits<<<(unsigned)((dst_words + per - 1) / per), GB_WORDS, 0, s>>>(d_src, d_segs, nseg, d_dst, dst_words);
  return cudaGetLastError() == cudaSuccess ? WT_OK : WT_ECUDA;
}

int wt_create(uint64_t n, uint64_t sigma, uint32_t elem_bytes, uint64_t total_nodes, void *stream, wt_tree **out) {
  if (!out) return WT_EINVAL;
  *out = nullptr;
  if (elem_bytes != 1 && elem_bytes != 2 && elem_bytes != 4) return WT_EINVAL;
  if (sigma < 1 || sigma > (1ull << (8 * elem_bytes)) || n >= (1ull << 32)) return WT_EINVAL;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  configure_pool_once();
  const uint32_t L = levels_of(sigma);
  Allocs A{s};
  wt_tree *t = new wt_tree();
  memset(t, 0, sizeof(*t));
  t->n = n;
  t->sigma = sigma;
  t->levels = L;
  t->elem_bytes = elem_bytes;
  t->words_per_level = ((n + 511) / 512) * 8;
  t->blocks_per_level = (n + 511) / 512;
  t->supers_per_level = (n + 65535) / 65536 + 1;
  t->total_nodes = total_nodes;
  t->bits = A.alloc<uint64_t>(L * t->words_per_level, true);
  t->level_node_ptr = A.alloc<uint64_t>(L + 1, true);
  t->node_key = A.alloc<uint32_t>(total_nodes, true);
  t->node_start = A.alloc<uint32_t>(total_nodes, true);
  t->rank_block = A.alloc<uint16_t>(L * t->blocks_per_level, true);
  t->rank_super = A.alloc<uint64_t>(L * t->supers_per_level, true);
  cudaError_t ce = cudaSuccess;
  if (!A.fail && L * t->words_per_level)
    ce = cudaMemsetAsync(t->bits, 0, L * t->words_per_level * sizeof(uint64_t), s);
  if (A.fail || ce != cudaSuccess) {
    A.free_outputs();
    cudaStreamSynchronize(s);
    delete t;
    return A.fail ? WT_ENOMEM : WT_ECUDA;
  }
  Internal *in = new Internal();
  in->stream = s;
  in->outputs = A.outputs;
  t->internal = in;
  *out = t;
  return WT_OK;
}

int wt_finish(wt_tree *t, void *stream) {
  if (!t || !t->internal) return WT_EINVAL;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint32_t L = t->levels;
  const uint64_t n = t->n, WPL = t->words_per_level, BPL = t->blocks_per_level, SPL = t->supers_per_level;
  const uint64_t NSD = SPL - 1;
  cudaError_t ce = cudaSuccess;
  if (L && n) {
    uint64_t *suptot = nullptr;
    ce = cudaMallocAsync(&suptot, L * NSD * sizeof(uint64_t), s);
    if (ce != cudaSuccess) return WT_ENOMEM;
    uint32_t *err = nullptr;
    ce = cudaMallocAsync(&err, sizeof(uint32_t), s);
    if (ce == cudaSuccess) ce = cudaMemsetAsync(err, 0, sizeof(uint32_t), s);
    if (ce == cudaSuccess) {
      const uint64_t warps = (uint64_t)L * NSD;
      k_rank_local<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, s>>>(t->bits, WPL, BPL, NSD, 0, L, t->rank_block,
                                                                         suptot, err);
      k_rank_super<<<L, 1024, 0, s>>>(suptot, NSD, SPL, t->rank_super, err);
      ce = cudaGetLastError();
    }
    cudaFreeAsync(suptot, s);
    if (err) cudaFreeAsync(err, s);
  } else if (L) {
    ce = cudaMemsetAsync(t->rank_super, 0, L * SPL * sizeof(uint64_t), s);
  }
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
  return ce == cudaSuccess ? WT_OK : WT_ECUDA;
}

}  // extern "C"
