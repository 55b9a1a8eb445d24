// hwt_lib.cu -- host orchestration of the Huffman-shaped wavelet tree
// and its extern "C" entry points hwt_build /
// hwt_free / hwt_access / hwt_rank of include/wt.h.
#include "wt_host.cuh"
#include "wt_dist.cuh"
#include "wt_huff.cuh"

using namespace wtb;
using namespace wthost;

// ============ Huffman-shaped wavelet tree ============
namespace {

struct HwtInternal {
  cudaStream_t stream;
  std::vector<void *> outputs;
  TouchSet touched;
  uint32_t *sym_sorted = nullptr;
  HuffCanon *canon = nullptr;
};

uint64_t *hwt_stage() {  // pinned staging for the host reads of hwt_build (one per host thread)
  static thread_local uint64_t *st = nullptr;
  if (!st && cudaMallocHost(&st, 256 * sizeof(uint64_t)) != cudaSuccess) st = nullptr;
  return st;
}

template <typename InT>
void launch_sym_hist(const void *S, uint64_t n, uint32_t sigma, uint32_t *hist, uint32_t *err, cudaStream_t s) {
  if (sigma <= 256) {
    const unsigned grid = (unsigned)std::min<uint64_t>((n + 8191) / 8192, 4ull * num_sms());
    k_sym_hist_small<InT><<<grid, 512, 0, s>>>((const InT *)S, n, sigma, hist, err);
  } else {
    static PerDevice<int> attr;
    attr.get([](int &) {
      cudaFuncSetAttribute(k_sym_hist<InT>, cudaFuncAttributeMaxDynamicSharedMemorySize, HIST_PART * 4);
    });
    const uint32_t nparts = (sigma + HIST_PART - 1) / HIST_PART;
    const uint32_t bins = std::min<uint32_t>(sigma, HIST_PART);
    const uint32_t per = std::max<uint32_t>(1, (uint32_t)std::min<uint64_t>((n + 16383) / 16384, 2ull * num_sms() / nparts));
    k_sym_hist<InT><<<per * nparts, 1024, bins * 4, s>>>((const InT *)S, n, sigma, nparts, hist, err);
  }
}

template <typename InT, typename OutT>
void launch_map_t(const void *S, uint64_t n, uint32_t sigma, const uint32_t *pad, void *X, cudaStream_t s) {
  const size_t tab = (size_t)sigma * sizeof(OutT);
  const unsigned grid = (unsigned)std::min<uint64_t>((n + 2047) / 2048, 4ull * num_sms());
  if (tab <= 160 * 1024) {
    static PerDevice<int> attr;
    attr.get([](int &) {
      cudaFuncSetAttribute(k_huff_map<InT, OutT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    });
    k_huff_map<InT, OutT, true><<<grid, 512, tab, s>>>((const InT *)S, n, sigma, pad, (OutT *)X);
  } else {
    k_huff_map<InT, OutT, false><<<grid, 512, 0, s>>>((const InT *)S, n, sigma, pad, (OutT *)X);
  }
}

template <typename InT>
void launch_map(const void *S, uint64_t n, uint32_t sigma, const uint32_t *pad, void *X, uint32_t xw, cudaStream_t s) {
  if (xw == 1) launch_map_t<InT, uint8_t>(S, n, sigma, pad, X, s);
  else if (xw == 2) launch_map_t<InT, uint16_t>(S, n, sigma, pad, X, s);
  else launch_map_t<InT, uint32_t>(S, n, sigma, pad, X, s);
}

int hwt_build_impl(const void *d_seq, uint64_t n, uint32_t eb, uint64_t sigma, void *stream_v, hwt_tree **out) {
  if (!out) return WT_EINVAL;
  *out = nullptr;
  if (eb != 1 && eb != 2 && eb != 4) return WT_EINVAL;
  if (sigma < 1 || sigma > (1ull << (8 * eb)) || sigma > 65536) return WT_EINVAL;
  if (n >= (1ull << 32)) return WT_EINVAL;
  if (n > 0 && !d_seq) return WT_EINVAL;
  cudaStream_t s = static_cast<cudaStream_t>(stream_v);
  configure_pool_once();
  uint64_t *stage = hwt_stage();
  if (!stage) return WT_ENOMEM;
  Allocs A{s};
  const uint32_t sg = (uint32_t)sigma;
  uint32_t P = 2;
  while (P < sg) P <<= 1;

  hwt_tree *t = new hwt_tree();
  memset(t, 0, sizeof(*t));
  t->n = n;
  t->sigma = sigma;
  t->elem_bytes = eb;
  uint32_t *hist = A.alloc<uint32_t>(sg, false);
  uint32_t *err = A.alloc<uint32_t>(4, false);
  uint64_t *keys = A.alloc<uint64_t>(P, false);
  uint32_t *scr = A.alloc<uint32_t>(6ull * sg, false);
  uint32_t *pad = A.alloc<uint32_t>(sg, false);
  uint64_t *info = A.alloc<uint64_t>(48, false);
  t->code_len = A.alloc<uint8_t>(sg, true);
  t->code = A.alloc<uint32_t>(sg, true);
  uint32_t *sym_sorted = A.alloc<uint32_t>(sg, true);
  HuffCanon *canon = A.alloc<HuffCanon>(1, true);
  auto fail = [&](int rc) {
    A.free_scratch();
    A.free_outputs();
    cudaStreamSynchronize(s);
    delete t;
    return rc;
  };
  if (A.fail) return fail(WT_ENOMEM);
  cudaError_t ce = cudaSuccess;
  auto chk = [&](cudaError_t e) {
    if (e != cudaSuccess && ce == cudaSuccess) ce = e;
  };

  // ---- H1 + H2: histogram, code lengths, canonical codes, level sizes ----
  chk(cudaMemsetAsync(hist, 0, sg * sizeof(uint32_t), s));
  chk(cudaMemsetAsync(err, 0, 4 * sizeof(uint32_t), s));
  if (n) {
    if (eb == 1) launch_sym_hist<uint8_t>(d_seq, n, sg, hist, err, s);
    else if (eb == 2) launch_sym_hist<uint16_t>(d_seq, n, sg, hist, err, s);
    else launch_sym_hist<uint32_t>(d_seq, n, sg, hist, err, s);
    chk(cudaGetLastError());
  }
  k_huff_compact<<<1, 1024, 0, s>>>(hist, sg, keys, P, info);
  {  // bitonic sort of the (freq, sym) keys
    const uint32_t CH = std::min<uint32_t>(P, SORT_CH);
    k_bitonic_chunk<<<P / CH, 1024, 0, s>>>(keys, P, 0);
    for (uint32_t k = 2 * CH; k <= P; k <<= 1) {
      for (uint32_t j = k >> 1; j >= CH; j >>= 1)
        k_bitonic_step<<<(P / 2 + 255) / 256, 256, 0, s>>>(keys, P, j, k);
      k_bitonic_chunk<<<P / CH, 1024, 0, s>>>(keys, P, k);
    }
  }
  k_huff_codes<<<1, 1024, 0, s>>>(keys, sg, scr, t->code_len, t->code, pad, sym_sorted, canon, info);
  chk(cudaGetLastError());
  chk(cudaMemcpyAsync(stage, info, (4 + HUFF_MAXLEN) * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
  chk(cudaMemcpyAsync(stage + 64, err, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  chk(cudaStreamSynchronize(s));
  if (ce != cudaSuccess) return fail(WT_ECUDA);
  if ((uint32_t)stage[64]) return fail(WT_ESYMBOL);
  if (stage[3]) return fail(WT_EUNSUPPORTED);
  const uint32_t h = (uint32_t)stage[0];
  if (getenv("WT_HUFF_TIMING")) {
    uint64_t tm[8];
    cudaMemcpy(tm, info + 39, sizeof(tm), cudaMemcpyDeviceToHost);
    fprintf(stderr,
            "k_huff_codes: rounds %llu; compact %.1f us, sort %.1f, rounds %.1f, depths %.1f, lengths %.1f, "
            "codes %.1f\n",
            (unsigned long long)tm[0], (tm[2] - tm[1]) / 1e3, (tm[3] - tm[2]) / 1e3, (tm[4] - tm[3]) / 1e3,
            (tm[5] - tm[4]) / 1e3, (tm[6] - tm[5]) / 1e3, (tm[7] - tm[6]) / 1e3);
  }
  t->levels = h;
  t->only_symbol = (uint32_t)stage[2];
  HwtLevels lv;
  memset(&lv, 0, sizeof(lv));
  lv.h = h;
  std::vector<uint64_t> host(5 * (HUFF_MAXLEN + 1), 0);  // len | wptr | bptr | sptr | node ptr
  uint64_t *h_len = host.data(), *h_wp = h_len + (HUFF_MAXLEN + 1), *h_bp = h_wp + (HUFF_MAXLEN + 1);
  uint64_t *h_sp = h_bp + (HUFF_MAXLEN + 1), *h_np = h_sp + (HUFF_MAXLEN + 1);
  for (uint32_t l = 0; l < h; l++) {
    const uint64_t nl = stage[4 + l];
    h_len[l] = lv.nl[l] = nl;
    h_wp[l + 1] = h_wp[l] + (nl + 511) / 512 * 8;
    h_bp[l + 1] = h_bp[l] + (nl + 511) / 512;
    h_sp[l + 1] = h_sp[l] + (nl + 65535) / 65536 + 1;
    t->total_bits += nl;
  }
  for (uint32_t l = 0; l <= h; l++) lv.wptr[l] = h_wp[l];
  t->level_len = A.alloc<uint64_t>(h, true);
  t->level_word_ptr = A.alloc<uint64_t>(h + 1, true);
  t->level_block_ptr = A.alloc<uint64_t>(h + 1, true);
  t->level_super_ptr = A.alloc<uint64_t>(h + 1, true);
  t->level_node_ptr = A.alloc<uint64_t>(h + 1, true);
  t->bits = A.alloc<uint64_t>(h_wp[h], true);
  t->rank_block = A.alloc<uint16_t>(h_bp[h], true);
  t->rank_super = A.alloc<uint64_t>(h_sp[h], true);
  if (A.fail) return fail(WT_ENOMEM);
  chk(cudaMemcpyAsync(t->level_len, h_len, h * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
  chk(cudaMemcpyAsync(t->level_word_ptr, h_wp, (h + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
  chk(cudaMemcpyAsync(t->level_block_ptr, h_bp, (h + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
  chk(cudaMemcpyAsync(t->level_super_ptr, h_sp, (h + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, s));

  if (h > 0) {
    // ---- H4: balanced levelWT over the padded codes, in stages ----
    // Stage [lo, hi) builds the tree of the elements whose code is longer than
    // lo (the only ones that reach level lo), keyed by the top hi bits of the
    // padded code, and keeps its levels lo .. hi-1.  One stage [0, h) when
    // most codes are long; 8-level stages while at least half of the elements
    // leave the sequence within the stage (skewed codes: work ~ sum of n_lo).
    // Plan by a cost model in element-group passes: a stage [lo, hi) costs
    // n_lo * ceil(hi / 8) plus ~0.3 n for its compaction (two reads of S)
    // unless it is the single stage [0, h); best[lo] = cheapest finish from lo.
    std::vector<std::pair<uint32_t, uint32_t>> stg;
    {
      const uint32_t nb = (h + TAU_MAX - 1) / TAU_MAX;
      std::vector<double> best(nb + 1, 0.0);
      std::vector<uint32_t> cut(nb + 1, h);
      auto nlo = [&](uint32_t lo) { return (double)(lo ? h_len[lo] : n); };
      for (int bi = (int)nb - 1; bi >= 0; bi--) {
        const uint32_t lo = (uint32_t)bi * TAU_MAX;
        const double ov = lo ? 0.3 * (double)n : 0.0;
        double c = nlo(lo) * nb + ov;  // one stage to the end
        cut[bi] = h;
        if (lo + TAU_MAX < h) {
          const double c2 = nlo(lo) * (bi + 1) + 0.3 * (double)n + best[bi + 1];
          if (c2 < c) { c = c2; cut[bi] = lo + TAU_MAX; }
        }
        best[bi] = c;
      }
      for (uint32_t lo = 0; lo < h; lo = cut[lo / TAU_MAX]) stg.push_back({lo, cut[lo / TAU_MAX]});
    }
    t->stages = (uint32_t)stg.size();
    // ---- H3: padded codes (single stage; a staged build compacts per stage) ----
    void *X = nullptr;
    if (stg.size() == 1) {
      const uint32_t xw = width_of(h);
      X = A.alloc<uint8_t>(n * xw, false);
      if (A.fail) return fail(WT_ENOMEM);
      if (eb == 1) launch_map<uint8_t>(d_seq, n, sg, pad, X, xw, s);
      else if (eb == 2) launch_map<uint16_t>(d_seq, n, sg, pad, X, xw, s);
      else launch_map<uint32_t>(d_seq, n, sg, pad, X, xw, s);
      chk(cudaGetLastError());
    }
    struct StageSegs { uint32_t lo, hi; uint32_t *key, *dst; uint64_t base[HUFF_MAXLEN]; uint32_t cnt[HUFF_MAXLEN]; };
    std::vector<StageSegs> done;
    uint32_t maxseg = 1;
    for (const auto &st : stg) {
      const uint32_t lo = st.first, hi = st.second;
      const uint64_t ng = lo ? h_len[lo] : n;
      const uint32_t kw = width_of(hi);
      void *Xg = X;
      if (lo > 0 || hi < h) {  // stage keys: alive elements, top hi bits of the padded code, S order
        Xg = A.alloc<uint8_t>(ng * kw, false);
        const uint32_t ntiles = (uint32_t)((n + HA_TILE - 1) / HA_TILE);
        uint32_t *tc = A.alloc<uint32_t>(ntiles, false);
        uint64_t *tt = A.alloc<uint64_t>(1, false);
        if (A.fail) return fail(WT_ENOMEM);
        auto run = [&](auto in_tag, auto out_tag) {
          using IT = decltype(in_tag);
          using OT = decltype(out_tag);
          k_hwt_alive_count<IT><<<ntiles, HA_THREADS, 0, s>>>((const IT *)d_seq, n, t->code_len, lo, ntiles, tc);
          k_part_scan<<<1, 1024, 0, s>>>(tc, ntiles, tt);
          k_hwt_alive_scatter<IT, OT><<<ntiles, HA_THREADS, 0, s>>>((const IT *)d_seq, n, t->code_len, pad, lo,
                                                                    h - hi, tc, (OT *)Xg);
        };
        auto run_in = [&](auto in_tag) {
          if (kw == 1) run(in_tag, uint8_t{});
          else if (kw == 2) run(in_tag, uint16_t{});
          else run(in_tag, uint32_t{});
        };
        if (eb == 1) run_in(uint8_t{});
        else if (eb == 2) run_in(uint16_t{});
        else run_in(uint32_t{});
        chk(cudaGetLastError());
      }
      wt_tree *pt = nullptr;
      const int rc = build_impl(Xg, nullptr, false, ng, kw, 1ull << hi, stream_v, &pt, false);
      if (rc != WT_OK) return fail(rc);
      StageSegs sg_{lo, hi, nullptr, nullptr, {}, {}};
      uint32_t *seg_src = A.alloc<uint32_t>(pt->total_nodes, false);
      sg_.dst = A.alloc<uint32_t>(pt->total_nodes, false);
      sg_.key = A.alloc<uint32_t>(pt->total_nodes, false);
      uint32_t *alive = A.alloc<uint32_t>(h, false);
      if (A.fail) { wt_free(pt); return fail(WT_ENOMEM); }
      k_hwt_segments<<<hi - lo, 1024, 0, s>>>(pt->level_node_ptr, pt->node_key, pt->node_start, ng, canon, info,
                                              seg_src, sg_.dst, sg_.key, alive, err, lo);
      chk(cudaGetLastError());
      chk(cudaMemcpyAsync(stage, pt->level_node_ptr, (hi + 1) * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
      chk(cudaMemcpyAsync(stage + 64, err, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
      chk(cudaMemcpyAsync(stage + 128, alive + lo, (hi - lo) * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
      chk(cudaStreamSynchronize(s));
      if (ce != cudaSuccess || (uint32_t)stage[64]) { wt_free(pt); return fail(WT_ECUDA); }
      const uint32_t *h_alive = reinterpret_cast<const uint32_t *>(stage + 128);
      lv.lbase = lo;
      uint64_t maxw = 0;
      for (uint32_t l = lo; l < hi; l++) {
        lv.segbase[l] = sg_.base[l] = stage[l];
        lv.nseg[l] = sg_.cnt[l] = h_alive[l - lo];
        h_np[l + 1] = h_alive[l - lo];  // counts for now, prefix-summed below
        maxseg = std::max(maxseg, h_alive[l - lo]);
        maxw = std::max(maxw, h_wp[l + 1] - h_wp[l]);
      }
      if (maxw) {
        const uint64_t per = (uint64_t)HB_WORDS * HB_WPT;
        k_hwt_bits<<<dim3((unsigned)((maxw + per - 1) / per), hi - lo), HB_WORDS, 0, s>>>(
            lv, pt->bits, pt->words_per_level, seg_src, sg_.dst, t->bits);
        chk(cudaGetLastError());
      }
      done.push_back(sg_);
      const int frc = wt_free(pt);  // stream-ordered after the kernels above (same stream)
      if (frc != WT_OK) return fail(WT_ECUDA);
    }
    for (uint32_t l = 0; l < h; l++) h_np[l + 1] += h_np[l];
    t->total_nodes = h_np[h];
    t->node_key = A.alloc<uint32_t>(t->total_nodes, true);
    t->node_start = A.alloc<uint32_t>(t->total_nodes, true);
    if (A.fail) return fail(WT_ENOMEM);
    chk(cudaMemcpyAsync(t->level_node_ptr, h_np, (h + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
    for (const auto &d : done) {
      lv.lbase = d.lo;
      for (uint32_t l = d.lo; l < d.hi; l++) { lv.segbase[l] = d.base[l]; lv.nseg[l] = d.cnt[l]; }
      k_hwt_nodes<<<dim3(std::min<uint32_t>((maxseg + 255) / 256, 1024), d.hi - d.lo), 256, 0, s>>>(
          lv, t->level_node_ptr, d.key, d.dst, t->node_key, t->node_start);
      chk(cudaGetLastError());
    }
    // ---- rank directory of all levels ----
    HwtRankLv rk;
    memset(&rk, 0, sizeof(rk));
    rk.h = h;
    for (uint32_t l = 0; l <= h; l++) { rk.wptr[l] = h_wp[l]; rk.bptr[l] = h_bp[l]; rk.sptr[l] = h_sp[l]; }
    for (uint32_t l = 0; l < h; l++) { rk.nl[l] = h_len[l]; rk.soff[l + 1] = rk.soff[l] + (h_len[l] + 65535) / 65536; }
    uint64_t *suptot = A.alloc<uint64_t>(rk.soff[h], false);
    if (A.fail) return fail(WT_ENOMEM);
    if (rk.soff[h]) {
      k_hwt_rank_local<<<(unsigned)((rk.soff[h] * 32 + 255) / 256), 256, 0, s>>>(rk, t->bits, t->rank_block, suptot);
      chk(cudaGetLastError());
    }
    k_hwt_rank_super<<<h, 1024, 0, s>>>(rk, suptot, t->rank_super);
    chk(cudaGetLastError());
  } else {
    chk(cudaMemcpyAsync(t->level_node_ptr, h_np, sizeof(uint64_t), cudaMemcpyHostToDevice, s));
  }
  A.free_scratch();
  chk(cudaStreamSynchronize(s));
  if (ce != cudaSuccess) return fail(WT_ECUDA);
  HwtInternal *in = new HwtInternal();
  in->stream = s;
  in->outputs = A.outputs;
  in->sym_sorted = sym_sorted;
  in->canon = canon;
  t->internal = in;
  *out = t;
  return WT_OK;
}

HwtView view_of_hwt(const hwt_tree *t) {
  const HwtInternal *in = static_cast<const HwtInternal *>(t->internal);
  HwtView v;
  v.n = t->n;
  v.h = t->levels;
  v.only_symbol = t->only_symbol;
  v.sigma = t->sigma;
  v.level_len = t->level_len;
  v.wptr = t->level_word_ptr;
  v.bptr = t->level_block_ptr;
  v.sptr = t->level_super_ptr;
  v.node_ptr = t->level_node_ptr;
  v.bits = t->bits;
  v.rank_block = t->rank_block;
  v.rank_super = t->rank_super;
  v.node_key = t->node_key;
  v.node_start = t->node_start;
  v.code = t->code;
  v.sym_sorted = in->sym_sorted;
  v.code_len = t->code_len;
  v.canon = in->canon;
  return v;
}

}  // namespace

extern "C" {

int hwt_build(const void *d_seq, uint64_t n, uint32_t elem_bytes, uint64_t sigma, void *stream, hwt_tree **out) {
  return hwt_build_impl(d_seq, n, elem_bytes, sigma, stream, out);
}

int hwt_free(hwt_tree *t) {
  if (!t) return WT_OK;
  HwtInternal *in = static_cast<HwtInternal *>(t->internal);
  cudaError_t e = cudaSuccess;
  if (in) {  // stream-ordered, after the build stream and every stream a query used (as wt_free)
    e = in->touched.order_before(in->stream);
    for (void *p : in->outputs) {
      cudaError_t e2 = cudaFreeAsync(p, in->stream);
      if (e2 != cudaSuccess) e = e2;
    }
    delete in;
  }
  delete t;
  return e == cudaSuccess ? WT_OK : WT_ECUDA;
}

static void touch_hwt(const hwt_tree *t, void *stream) {
  HwtInternal *in = static_cast<HwtInternal *>(t->internal);
  in->touched.add(static_cast<cudaStream_t>(stream), in->stream);
}

int hwt_access(const hwt_tree *t, const uint64_t *d_pos, uint64_t q, uint32_t *d_out, void *stream) {
  if (!t || !t->internal || (q > 0 && (!d_pos || !d_out))) return WT_EINVAL;
  if (q == 0) return WT_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  touch_hwt(t, stream);
  k_hwt_access<<<(unsigned)((q + 255) / 256), 256, 0, s>>>(view_of_hwt(t), d_pos, q, d_out);
  return cudaGetLastError() == cudaSuccess ? WT_OK : WT_ECUDA;
}

int hwt_rank(const hwt_tree *t, const uint32_t *d_sym, const uint64_t *d_pos, uint64_t q, uint64_t *d_out,
             void *stream) {
  if (!t || !t->internal || (q > 0 && (!d_sym || !d_pos || !d_out))) return WT_EINVAL;
  if (q == 0) return WT_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  touch_hwt(t, stream);
  k_hwt_rank<<<(unsigned)((q + 255) / 256), 256, 0, s>>>(view_of_hwt(t), d_sym, d_pos, q, d_out);
  return cudaGetLastError() == cudaSuccess ? WT_OK : WT_ECUDA;
}

int hwt_select(const hwt_tree *t, const uint32_t *d_sym, const uint64_t *d_k, uint64_t q, uint64_t *d_out,
               void *stream) {
  if (!t || !t->internal || (q > 0 && (!d_sym || !d_k || !d_out))) return WT_EINVAL;
  if (q == 0) return WT_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  touch_hwt(t, stream);
  k_hwt_select<<<(unsigned)((q + 127) / 128), 128, 0, s>>>(view_of_hwt(t), d_sym, d_k, q, d_out);
  return cudaGetLastError() == cudaSuccess ? WT_OK : WT_ECUDA;
}

}  // extern "C"

