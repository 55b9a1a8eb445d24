// wm_lib.cu -- host orchestration of the wavelet matrix
// and its extern "C" entry points wm_build / wm_free / wm_access / wm_rank /
// wm_select* of include/wt.h.
#include "wt_host.cuh"
#include "wt_prep.cuh"
#include "wt_rank.cuh"
#include "wt_select.cuh"
#include "wt_wm.cuh"

using namespace wtb;
using namespace wthost;

namespace {

// ===================== wavelet matrix =====================
struct WmLaunch {
  void (*kern)(GroupParams) = nullptr;
  int grid = 0, block = 32;
  uint32_t tile = 0;
};

template <typename InT, typename RecT, typename OutT, bool HAS_OUT>
WmLaunch wm_launch() {
  static PerDevice<WmLaunch> pd_;
  return pd_.get([](WmLaunch &wl) {
#ifdef WT_WM_WARP  // the one-warp pass (kept for comparison)
    wl.kern = k_wm_group<InT, RecT, OutT, HAS_OUT>;
    wl.tile = WmTile<RecT>::TW;
    wl.block = 32;
#else
    wl.kern = k_wm_group4<InT, RecT, OutT, HAS_OUT>;
    wl.tile = WmSmem4<RecT, HAS_OUT>::TT;
    wl.block = WPB * 32;
#endif
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, wl.kern, wl.block, 0);
    wl.grid = num_sms() * (per_sm < 1 ? 1 : per_sm);
  });
}

WmLaunch pick_wm(uint32_t inw, uint32_t recw, uint32_t outw, bool has_out) {
  if (!has_out) {
    if (recw == 1) {
      if (inw == 1) return wm_launch<uint8_t, uint8_t, uint8_t, false>();
      if (inw == 2) return wm_launch<uint16_t, uint8_t, uint8_t, false>();
      return wm_launch<uint32_t, uint8_t, uint8_t, false>();
    }
    return WmLaunch{};
  }
  if (recw == 2) {
    if (inw == 2) return wm_launch<uint16_t, uint16_t, uint8_t, true>();
    return wm_launch<uint32_t, uint16_t, uint8_t, true>();
  }
  if (outw == 2) return wm_launch<uint32_t, uint32_t, uint16_t, true>();
  return wm_launch<uint32_t, uint32_t, uint32_t, true>();
}

struct WmInternal {
  cudaStream_t stream;
  std::vector<void *> outputs;
  TouchSet touched;
};

int wm_build_impl(const void *d_seq, uint64_t n, uint32_t eb, uint64_t sigma, void *stream_v, wm_matrix **out) {
  if (!out) return WT_EINVAL;
  *out = nullptr;
  if (eb != 1 && eb != 2 && eb != 4) return WT_EINVAL;
  if (sigma < 1 || sigma > (1ull << (8 * eb))) return WT_EINVAL;
  if (n >= (1ull << 32)) return WT_EINVAL;
  if (n > 0 && !d_seq) return WT_EINVAL;
  const uint32_t L = levels_of(sigma);
  cudaStream_t s = static_cast<cudaStream_t>(stream_v);
  configure_pool_once();
  Allocs A{s};
  const uint64_t WPL = ((n + 511) / 512) * 8, BPL = (n + 511) / 512, SPL = (n + 65535) / 65536 + 1, NSD = SPL - 1;
  wm_matrix *m = new wm_matrix();
  memset(m, 0, sizeof(*m));
  m->n = n;
  m->sigma = sigma;
  m->levels = L;
  m->elem_bytes = eb;
  m->words_per_level = WPL;
  m->blocks_per_level = BPL;
  m->supers_per_level = SPL;
  A.use_arena();
  A.alloc_outputs({{(void **)&m->bits, L * WPL * 8}, {(void **)&m->zeros, L * 8}, {(void **)&m->rank_block, L * BPL * 2},
                   {(void **)&m->rank_super, L * SPL * 8}});
  uint32_t *err = A.alloc<uint32_t>(4, false);
  uint64_t *suptot = A.alloc<uint64_t>(L * NSD, false);
  const uint32_t NG = (L + TAU_MAX - 1) / TAU_MAX;
  struct Grp {
    uint32_t l0, tau, pbits, ndig, inw, recw, outw;
    WmLaunch wl;
    uint64_t CH, K;
    void *keys_out;
  } G[4];
  uint64_t maxK = 1;
  for (uint32_t g = 0; g < NG; g++) {
    Grp &gr = G[g];
    gr.l0 = g * TAU_MAX;
    gr.tau = std::min<uint32_t>(TAU_MAX, L - gr.l0);
    gr.pbits = L - gr.l0 - gr.tau;
    gr.ndig = 1u << gr.tau;
    gr.inw = g == 0 ? eb : width_of(L - gr.l0);
    gr.recw = width_of(L - gr.l0);
    gr.outw = width_of(gr.pbits);
    gr.wl = pick_wm(gr.inw, gr.recw, gr.outw, g + 1 < NG);
    if (!gr.wl.kern) {
      A.free_scratch();
      A.free_outputs();
      cudaStreamSynchronize(s);
      delete m;
      return WT_EUNSUPPORTED;
    }
    const uint64_t tt = gr.wl.tile;
    const uint64_t target = (n + 16 * (uint64_t)gr.wl.grid - 1) / (16 * (uint64_t)gr.wl.grid);
    gr.CH = std::max<uint64_t>(tt, ((target + tt - 1) / tt) * tt);
    gr.K = std::max<uint64_t>((n + gr.CH - 1) / gr.CH, 1);
    maxK = std::max(maxK, gr.K);
    gr.keys_out = g + 1 < NG ? A.alloc<uint8_t>(n * gr.outw, false) : nullptr;
  }
  // sigma == 1 (no group): validation in chains of 2^24 symbols (32-bit chain arithmetic)
  constexpr uint64_t VCH = 1ull << 24;
  if (!NG) maxK = std::max<uint64_t>((n + VCH - 1) / VCH, 1);
  // chain tables (reused by every group: one row, the whole sequence)
  uint32_t *cb = A.alloc<uint32_t>(maxK, false), *ce_ = A.alloc<uint32_t>(maxK, false);
  uint32_t *cr = A.alloc<uint32_t>(maxK, false), *rf = A.alloc<uint32_t>(2, false);
  uint32_t *rs = A.alloc<uint32_t>(1, false), *rk = A.alloc<uint32_t>(1, false);
  uint32_t *E = A.alloc<uint32_t>(NDIG * (maxK + 1), false), *Cseg = A.alloc<uint32_t>(NDIG + 1, false);
  uint32_t *cnt = A.alloc<uint32_t>(4 * (NG ? NG : 1), false);
  if (A.fail) {
    A.free_scratch();
    A.free_outputs();
    cudaStreamSynchronize(s);
    delete m;
    return WT_ENOMEM;
  }
  cudaError_t ce = cudaSuccess;
  auto chk = [&](cudaError_t e) {
    if (e != cudaSuccess && ce == cudaSuccess) ce = e;
  };
  chk(cudaMemsetAsync(err, 0, 4 * sizeof(uint32_t), s));
  chk(cudaMemsetAsync(cnt, 0, 4 * (NG ? NG : 1) * sizeof(uint32_t), s));
  if (L && n) chk(cudaMemsetAsync(m->bits, 0, L * WPL * sizeof(uint64_t), s));
  cudaStream_t side = side_stream();
  bool side_used = false;
  const void *keys_in = d_seq;
  if (n && !NG) {  // sigma == 1: validation only (every symbol must be 0)
    const uint32_t K = (uint32_t)maxK, st = K + 1;
    const unsigned hg = std::min<uint32_t>(K, 4 * num_sms());
    k_chains_root<<<(K + 255) / 256, 256, 0, s>>>(n, VCH, K, cb, ce_, cr, rf, rs, rk, cnt, err);
    if (eb == 1) k_chain_hist<uint8_t, true><<<hg, 512, 0, s>>>((const uint8_t *)d_seq, sigma, 0, 1, cb, ce_, cnt, st, E, err);
    else if (eb == 2) k_chain_hist<uint16_t, true><<<hg, 512, 0, s>>>((const uint16_t *)d_seq, sigma, 0, 1, cb, ce_, cnt, st, E, err);
    else k_chain_hist<uint32_t, true><<<hg, 512, 0, s>>>((const uint32_t *)d_seq, sigma, 0, 1, cb, ce_, cnt, st, E, err);
    chk(cudaGetLastError());
  }
  for (uint32_t g = 0; g < NG && n; g++) {
    Grp &gr = G[g];
    uint32_t *gc = cnt + 4 * g;
    const uint32_t K = (uint32_t)gr.K, stride = (uint32_t)gr.K + 1;
    k_chains_root<<<(K + 255) / 256, 256, 0, s>>>(n, gr.CH, K, cb, ce_, cr, rf, rs, rk, gc, err);
    const unsigned hgrid = std::min<uint32_t>(K, 4 * num_sms());
    if (g == 0) {
      if (eb == 1) k_chain_hist<uint8_t, true><<<hgrid, 512, 0, s>>>((const uint8_t *)keys_in, sigma, gr.pbits, gr.ndig, cb, ce_, gc, stride, E, err);
      else if (eb == 2) k_chain_hist<uint16_t, true><<<hgrid, 512, 0, s>>>((const uint16_t *)keys_in, sigma, gr.pbits, gr.ndig, cb, ce_, gc, stride, E, err);
      else k_chain_hist<uint32_t, true><<<hgrid, 512, 0, s>>>((const uint32_t *)keys_in, sigma, gr.pbits, gr.ndig, cb, ce_, gc, stride, E, err);
    } else {
      if (gr.inw == 1) k_chain_hist<uint8_t, false><<<hgrid, 512, 0, s>>>((const uint8_t *)keys_in, sigma, gr.pbits, gr.ndig, cb, ce_, gc, stride, E, err);
      else if (gr.inw == 2) k_chain_hist<uint16_t, false><<<hgrid, 512, 0, s>>>((const uint16_t *)keys_in, sigma, gr.pbits, gr.ndig, cb, ce_, gc, stride, E, err);
      else k_chain_hist<uint32_t, false><<<hgrid, 512, 0, s>>>((const uint32_t *)keys_in, sigma, gr.pbits, gr.ndig, cb, ce_, gc, stride, E, err);
    }
    chk(cudaGetLastError());
    k_chain_scan<<<gr.ndig, 1024, 0, s>>>(E, stride, gc, err);
    k_row_scan<<<1, 32, 0, s>>>(E, stride, rf, gc, gr.ndig, Cseg, err);
    chk(cudaGetLastError());
    GroupParams gp{};
    gp.keys_in = keys_in;
    gp.keys_out = gr.keys_out;
    gp.n = n;
    gp.l0 = gr.l0;
    gp.tau = gr.tau;
    gp.pbits = gr.pbits;
    gp.counts = gc;
    gp.chain_begin = cb;
    gp.chain_end = ce_;
    gp.chain_row = cr;
    gp.row_first = rf;
    gp.E = E;
    gp.estride = stride;
    gp.Cseg = Cseg;
    gp.row_start = rs;
    gp.chain_counter = gc + 2;
    gp.bits = m->bits;
    gp.wpl = WPL;
    gp.err = err;
    gr.wl.kern<<<gr.wl.grid, gr.wl.block, 0, s>>>(gp);
    chk(cudaGetLastError());
    if (NSD) {  // rank block counts of this group's levels on the side stream
      cudaEvent_t ev;
      chk(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      chk(cudaEventRecord(ev, s));
      chk(cudaStreamWaitEvent(side, ev, 0));
      cudaEventDestroy(ev);
      const uint64_t warps = (uint64_t)gr.tau * NSD;
      k_rank_local<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, side>>>(m->bits, WPL, BPL, NSD, gr.l0, gr.tau,
                                                                             m->rank_block, suptot, err);
      chk(cudaGetLastError());
      side_used = true;
    }
    keys_in = gr.keys_out;
  }
  cudaEvent_t ev_side = nullptr;
  if (side_used) {
    chk(cudaEventCreateWithFlags(&ev_side, cudaEventDisableTiming));
    chk(cudaEventRecord(ev_side, side));
    chk(cudaStreamWaitEvent(s, ev_side, 0));
  }
  if (L > 0) {
    if (n > 0) k_rank_super<<<L, 1024, 0, s>>>(suptot, NSD, SPL, m->rank_super, err);
    else chk(cudaMemsetAsync(m->rank_super, 0, L * SPL * sizeof(uint64_t), s));
    k_wm_zeros<<<(L + 31) / 32, 32, 0, s>>>(m->rank_super, SPL, L, n, m->zeros, err);
    chk(cudaGetLastError());
  }
  static thread_local uint32_t *h_err = nullptr;  // pinned, one per host thread
  if (!h_err && cudaMallocHost(&h_err, sizeof(uint32_t) * 4) != cudaSuccess) h_err = nullptr;
  if (!h_err) {
    A.free_scratch();
    A.free_outputs();
    cudaStreamSynchronize(s);
    delete m;
    return WT_ENOMEM;
  }
  chk(cudaMemcpyAsync(h_err, err, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  A.free_scratch();
  chk(cudaStreamSynchronize(s));
  if (ev_side) cudaEventDestroy(ev_side);
  if (ce != cudaSuccess || (*h_err & 1u)) {
    const bool sym = ce == cudaSuccess;
    A.free_outputs();
    cudaStreamSynchronize(s);
    delete m;
    return sym ? WT_ESYMBOL : WT_ECUDA;
  }
  WmInternal *in = new WmInternal();
  in->stream = s;
  in->outputs = A.outputs;
  m->internal = in;
  *out = m;
  return WT_OK;
}

}  // namespace

extern "C" {

int wm_build(const void *d_seq, uint64_t n, uint32_t elem_bytes, uint64_t sigma, void *stream, wm_matrix **out) {
  return wm_build_impl(d_seq, n, elem_bytes, sigma, stream, out);
}

int wm_free(wm_matrix *m) {
  if (!m) return WT_OK;
  WmInternal *in = static_cast<WmInternal *>(m->internal);
  cudaError_t e = cudaSuccess;
  if (in) {  // stream-ordered, after the build stream and every stream a query used (as wt_free)
    e = in->touched.order_before(in->stream);
    for (void *p : in->outputs) {
      const cudaError_t e2 = cudaFreeAsync(p, in->stream);
      if (e2 != cudaSuccess) e = e2;
    }
    delete in;
  }
  delete m;
  return e == cudaSuccess ? WT_OK : WT_ECUDA;
}

static void touch_wm(const wm_matrix *m, void *stream) {
  if (m && m->internal) {
    WmInternal *in = static_cast<WmInternal *>(m->internal);
    in->touched.add(static_cast<cudaStream_t>(stream), in->stream);
  }
}

static TreeView view_of_wm(const wm_matrix *m) {
  TreeView v;
  v.n = m->n;
  v.wpl = m->words_per_level;
  v.bpl = m->blocks_per_level;
  v.spl = m->supers_per_level;
  v.L = m->levels;
  v.bits = m->bits;
  v.rank_block = m->rank_block;
  v.rank_super = m->rank_super;
  return v;
}

int wm_access(const wm_matrix *m, const uint64_t *d_pos, uint64_t q, uint32_t *d_out, void *stream) {
  if (!m || (q > 0 && (!d_pos || !d_out))) return WT_EINVAL;
  if (q == 0) return WT_OK;
  touch_wm(m, stream);
  k_wm_access<<<(unsigned)((q + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(view_of_wm(m), m->zeros,
                                                                                           d_pos, q, d_out);
  return cudaGetLastError() == cudaSuccess ? WT_OK : WT_ECUDA;
}

int wm_select_index(wm_matrix *m, void *stream) {
  if (!m || !m->internal) return WT_EINVAL;
  WmInternal *in = static_cast<WmInternal *>(m->internal);
  touch_wm(m, stream);
  return select_index_impl(view_of_wm(m), &m->select_per_level, &m->select0, &m->select1, in->outputs,
                           static_cast<cudaStream_t>(stream));
}

int wm_select(const wm_matrix *m, const uint32_t *d_sym, const uint64_t *d_k, uint64_t q, uint64_t *d_out,
              void *stream) {
  if (!m || (q > 0 && (!d_sym || !d_k || !d_out)) || !m->select_per_level) return WT_EINVAL;
  if (q == 0) return WT_OK;
  touch_wm(m, stream);
  k_wm_select<<<(unsigned)((q + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      view_of_wm(m), m->zeros, m->select0, m->select1, m->select_per_level, m->sigma, d_sym, d_k, q, d_out);
  return cudaGetLastError() == cudaSuccess ? WT_OK : WT_ECUDA;
}

int wm_rank(const wm_matrix *m, const uint32_t *d_sym, const uint64_t *d_pos, uint64_t q, uint64_t *d_out,
            void *stream) {
  if (!m || (q > 0 && (!d_sym || !d_pos || !d_out))) return WT_EINVAL;
  if (q == 0) return WT_OK;
  touch_wm(m, stream);
  k_wm_rank<<<(unsigned)((q + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      view_of_wm(m), m->zeros, m->sigma, d_sym, d_pos, q, d_out);
  return cudaGetLastError() == cudaSuccess ? WT_OK : WT_ECUDA;
}

}  // extern "C"
