// wt_lib.cu -- host orchestration and the extern "C" entry points of include/wt.h.
//
// One wt_build = A1 (validate + histogram), A4 (node table), then one k_group
// pass per group of <= 8 levels (A2/A3/A5/A6/A7 fused), then the A7 finalize.
// The stream is synchronised exactly once, at the end, to read the error flag
// and the node counts.
#include "wt.h"
#include "wt_device.cuh"

#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

using namespace wtb;

namespace {

struct Prof {
  bool enabled = false;
  wt_profile last{};
  std::mutex mu;
};
Prof g_prof;

struct Launch {
  std::string name;
  uint64_t algo_bytes;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
};

// Per-build recorder of kernel launches (optionally timed with events).
struct Recorder {
  cudaStream_t s;
  bool timed;
  std::vector<Launch> launches;
  explicit Recorder(cudaStream_t st, bool t) : s(st), timed(t) {}
  void begin(const char *name, uint64_t bytes) {
    Launch L;
    L.name = name;
    L.algo_bytes = bytes;
    if (timed) {
      cudaEventCreate(&L.e0);
      cudaEventCreate(&L.e1);
      cudaEventRecord(L.e0, s);
    }
    launches.push_back(L);
  }
  void end() {
    if (timed) cudaEventRecord(launches.back().e1, s);
  }
  void publish() {  // after the stream has been synchronised
    wt_profile p{};
    p.total_launches = (uint32_t)launches.size();
    for (auto &L : launches) {
      float ms = 0.f;
      if (timed) {
        cudaEventElapsedTime(&ms, L.e0, L.e1);
        cudaEventDestroy(L.e0);
        cudaEventDestroy(L.e1);
      }
      int k = -1;
      for (uint32_t i = 0; i < p.count; i++)
        if (L.name == p.e[i].name) k = (int)i;
      if (k < 0 && p.count < WT_PROF_MAX) {
        k = (int)p.count++;
        snprintf(p.e[k].name, sizeof(p.e[k].name), "%s", L.name.c_str());
      }
      if (k >= 0) {
        p.e[k].ms += ms;
        p.e[k].launches += 1;
        p.e[k].algo_bytes += L.algo_bytes;
      }
    }
    std::lock_guard<std::mutex> g(g_prof.mu);
    g_prof.last = p;
  }
  void discard() {
    if (timed)
      for (auto &L : launches) {
        cudaEventDestroy(L.e0);
        cudaEventDestroy(L.e1);
      }
  }
};

struct Internal {
  cudaStream_t stream;
  std::vector<void *> outputs;
};

uint32_t levels_of(uint64_t sigma) {
  uint64_t v = sigma - 1;
  uint32_t L = 0;
  while (v) { L++; v >>= 1; }
  return L;
}

int g_num_sms = 0;
int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

void configure_pool_once() {
  static std::once_flag f;
  std::call_once(f, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  });
}

// Stream-ordered allocations that are released together on error.
struct Allocs {
  cudaStream_t s;
  std::vector<void *> scratch, outputs;
  bool fail = false;
  template <typename T>
  T *alloc(size_t count, bool output) {
    if (count == 0) count = 1;
    void *p = nullptr;
    if (cudaMallocAsync(&p, count * sizeof(T), s) != cudaSuccess) {
      fail = true;
      return nullptr;
    }
    (output ? outputs : scratch).push_back(p);
    return static_cast<T *>(p);
  }
  void free_scratch() {
    for (void *p : scratch) cudaFreeAsync(p, s);
    scratch.clear();
  }
  void free_outputs() {
    for (void *p : outputs) cudaFreeAsync(p, s);
    outputs.clear();
  }
};

template <typename InT, typename RecT, bool HAS_OUT>
cudaError_t launch_group(const GroupParams &gp, cudaStream_t s, int grid) {
  const size_t smem = 4 * sizeof(WarpSmem<RecT>);
  auto kern = k_group<InT, RecT, HAS_OUT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, 128, smem, s>>>(gp);
  return cudaGetLastError();
}

template <typename RecT>
int group_grid() {
  const size_t smem = 4 * sizeof(WarpSmem<RecT>);
  int per_sm = (int)((227 * 1024) / (smem + 1024));
  if (per_sm < 1) per_sm = 1;
  return num_sms() * per_sm;
}

int build_impl(const void *d_seq, const void *h_seq, bool from_host, uint64_t n, uint32_t eb,
               uint64_t sigma, void *stream_v, wt_tree **out) {
  if (!out) return WT_EINVAL;
  *out = nullptr;
  if (eb != 1 && eb != 2 && eb != 4) return WT_EINVAL;
  if (sigma < 1 || sigma > (1ull << (8 * eb))) return WT_EINVAL;
  if (n >= (1ull << 32)) return WT_EINVAL;
  if (n > 0 && !(from_host ? h_seq : d_seq)) return WT_EINVAL;
  const uint32_t L = levels_of(sigma);
  if (L > 16 || n >= (1ull << 30)) return WT_EUNSUPPORTED;
  cudaStream_t s = static_cast<cudaStream_t>(stream_v);
  configure_pool_once();

  bool timed;
  {
    std::lock_guard<std::mutex> g(g_prof.mu);
    timed = g_prof.enabled;
  }
  Recorder rec(s, timed);
  Allocs A{s};

  const uint64_t WPL = ((n + 511) / 512) * 8;
  const uint64_t BPL = (n + 511) / 512;
  const uint64_t SPL = (n + 65535) / 65536 + 1;
  const uint64_t NSD = SPL - 1;  // superblocks holding data
  uint64_t max_nodes = 0;
  for (uint32_t l = 0; l < L; l++) max_nodes += std::min<uint64_t>(1ull << l, n);

  wt_tree *t = new wt_tree();
  memset(t, 0, sizeof(*t));
  t->n = n;
  t->sigma = sigma;
  t->levels = L;
  t->elem_bytes = eb;
  t->words_per_level = WPL;
  t->blocks_per_level = BPL;
  t->supers_per_level = SPL;
  t->bits = A.alloc<uint64_t>(L * WPL, true);
  t->level_node_ptr = A.alloc<uint64_t>(L + 1, true);
  t->node_key = A.alloc<uint32_t>(max_nodes, true);
  t->node_start = A.alloc<uint32_t>(max_nodes, true);
  t->rank_block = A.alloc<uint16_t>(L * BPL, true);
  t->rank_super = A.alloc<uint64_t>(L * SPL, true);

  // scratch
  const void *seq = d_seq;
  if (from_host) {
    void *d = A.alloc<uint8_t>(n * eb, false);
    if (!A.fail && n) {
      if (cudaMemcpyAsync(d, h_seq, n * eb, cudaMemcpyHostToDevice, s) != cudaSuccess) A.fail = true;
    }
    seq = d;
  }
  const uint32_t Lh = L;  // L <= 16: the histogram covers every level
  const uint32_t nbins = 1u << Lh;
  const bool pair16 = Lh > 15;
  const int hist_ctas = num_sms() * (pair16 ? 1 : 2);
  uint32_t *err = A.alloc<uint32_t>(4, false);
  uint32_t *partial = A.alloc<uint32_t>((uint64_t)hist_ctas * nbins, false);
  uint32_t *adj = A.alloc<uint32_t>(nbins, false);
  uint32_t *hist = A.alloc<uint32_t>(nbins, false);
  uint32_t *Hx = A.alloc<uint32_t>(nbins + 1, false);
  uint32_t *ncount = A.alloc<uint32_t>(L + 1, false);
  uint32_t *blkcnt = A.alloc<uint32_t>(L * BPL, false);
  uint64_t *suptot = A.alloc<uint64_t>(L * NSD, false);
  const uint32_t tau0 = L < 8 ? L : 8;
  const uint32_t tau1 = L - tau0;
  const uint64_t max_tiles0 = (n + TW - 1) / TW;
  const uint64_t max_tiles1 = tau1 ? (n + TW - 1) / TW + std::min<uint64_t>(1ull << tau0, n) : 0;
  const uint64_t max_tiles = std::max(max_tiles0, max_tiles1);
  uint32_t *state = A.alloc<uint32_t>(max_tiles * NDIG, false);
  uint32_t *counters = A.alloc<uint32_t>(4, false);
  uint8_t *keys1 = tau1 ? A.alloc<uint8_t>(n, false) : nullptr;
  uint32_t *tile_seg = tau1 ? A.alloc<uint32_t>(max_tiles1, false) : nullptr;
  uint32_t *seg_tile_base = tau1 ? A.alloc<uint32_t>(std::min<uint64_t>(1ull << tau0, n) + 1, false) : nullptr;
  uint32_t *total_tiles = counters + 2;

  static uint64_t *h_stage = nullptr;  // pinned staging for the single D2H
  static std::mutex stage_mu;
  {
    std::lock_guard<std::mutex> g(stage_mu);
    if (!h_stage && cudaMallocHost(&h_stage, 64 * sizeof(uint64_t)) != cudaSuccess) A.fail = true;
  }

  auto fail_out = [&](int code) {
    A.free_scratch();
    A.free_outputs();
    cudaStreamSynchronize(s);
    rec.discard();
    delete t;
    return code;
  };
  if (A.fail) return fail_out(WT_ENOMEM);

  cudaError_t ce = cudaSuccess;
  auto chk = [&](cudaError_t e) { if (e != cudaSuccess && ce == cudaSuccess) ce = e; };

  chk(cudaMemsetAsync(err, 0, 4 * sizeof(uint32_t), s));
  chk(cudaMemsetAsync(counters, 0, 4 * sizeof(uint32_t), s));
  chk(cudaMemsetAsync(adj, 0, nbins * sizeof(uint32_t), s));
  chk(cudaMemsetAsync(t->level_node_ptr, 0, (L + 1) * sizeof(uint64_t), s));
  if (L) {
    chk(cudaMemsetAsync(t->bits, 0, L * WPL * sizeof(uint64_t), s));
    chk(cudaMemsetAsync(blkcnt, 0, L * BPL * sizeof(uint32_t), s));
    if (max_tiles) chk(cudaMemsetAsync(state, 0, max_tiles * NDIG * sizeof(uint32_t), s));
  }

  // ---- A1: validate + histogram ----
  {
    const uint32_t shift = L - Lh;
    const size_t smem = (pair16 ? nbins / 2 : nbins) * sizeof(uint32_t);
    rec.begin("k_hist", n * eb);
#define HIST_LAUNCH(T, PAIR)                                                                          \
  do {                                                                                                \
    cudaFuncSetAttribute(k_hist<T, PAIR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);    \
    k_hist<T, PAIR><<<hist_ctas, 1024, smem, s>>>((const T *)seq, n, sigma, shift, nbins, partial, adj, \
                                                   err);                                              \
  } while (0)
    if (eb == 1) HIST_LAUNCH(uint8_t, false);
    else if (eb == 2) { if (pair16) HIST_LAUNCH(uint16_t, true); else HIST_LAUNCH(uint16_t, false); }
    else { if (pair16) HIST_LAUNCH(uint32_t, true); else HIST_LAUNCH(uint32_t, false); }
#undef HIST_LAUNCH
    chk(cudaGetLastError());
    rec.end();
    rec.begin("k_hist_reduce", (uint64_t)hist_ctas * nbins * 4);
    k_hist_reduce<<<(nbins + 255) / 256, 256, 0, s>>>(partial, hist_ctas, nbins, adj, hist);
    chk(cudaGetLastError());
    rec.end();
    rec.begin("k_scan_hist", (uint64_t)nbins * 8);
    k_scan_hist<<<1, 1024, 0, s>>>(hist, nbins, Hx, err);
    chk(cudaGetLastError());
    rec.end();
  }

  if (L > 0 && n > 0) {
    // ---- A4: node table ----
    rec.begin("k_node_count", 0);
    k_node_count<<<L, 1024, 0, s>>>(Hx, Lh, ncount, err);
    chk(cudaGetLastError());
    rec.end();
    rec.begin("k_node_emit", max_nodes * 8);
    k_node_emit<<<L, 1024, 0, s>>>(Hx, Lh, L, ncount, t->level_node_ptr, t->node_key, t->node_start, err);
    chk(cudaGetLastError());
    rec.end();

    // ---- group 0: levels 0..tau0-1 over S ----
    GroupParams gp{};
    gp.keys_in = seq;
    gp.keys_out = keys1;
    gp.n = n;
    gp.Lh = Lh;
    gp.l0 = 0;
    gp.tau = tau0;
    gp.pbits = L - tau0;
    gp.Hx = Hx;
    gp.single_seg = 1;
    gp.ntiles_single = (uint32_t)max_tiles0;
    gp.level_node_ptr = t->level_node_ptr;
    gp.node_key = t->node_key;
    gp.node_start = t->node_start;
    gp.tile_counter = counters;
    gp.state = state;
    gp.bits = t->bits;
    gp.wpl = WPL;
    gp.blkcnt = blkcnt;
    gp.bpl = BPL;
    gp.err = err;
    const uint64_t g0_bytes = n * eb + (tau1 ? n : 0) + (uint64_t)tau0 * n / 8;
    rec.begin("k_group0", g0_bytes);
    if (tau1 == 0) {
      if (eb == 1) chk(launch_group<uint8_t, uint8_t, false>(gp, s, group_grid<uint8_t>()));
      else if (eb == 2) chk(launch_group<uint16_t, uint8_t, false>(gp, s, group_grid<uint8_t>()));
      else chk(launch_group<uint32_t, uint8_t, false>(gp, s, group_grid<uint8_t>()));
    } else {
      if (eb == 2) chk(launch_group<uint16_t, uint16_t, true>(gp, s, group_grid<uint16_t>()));
      else chk(launch_group<uint32_t, uint16_t, true>(gp, s, group_grid<uint16_t>()));
    }
    rec.end();

    if (tau1) {
      // ---- group 1: levels tau0..L-1 over the narrowed keys, per level-tau0 node ----
      rec.begin("k_segments", 0);
      k_segments<<<1, 1024, 0, s>>>(t->level_node_ptr, tau0, t->node_start, n, seg_tile_base, tile_seg,
                                    total_tiles, err);
      chk(cudaGetLastError());
      rec.end();
      chk(cudaMemsetAsync(state, 0, max_tiles1 * NDIG * sizeof(uint32_t), s));
      GroupParams g1 = gp;
      g1.keys_in = keys1;
      g1.keys_out = nullptr;
      g1.l0 = tau0;
      g1.tau = tau1;
      g1.pbits = 0;
      g1.single_seg = 0;
      g1.tile_seg = tile_seg;
      g1.seg_tile_base = seg_tile_base;
      g1.total_tiles = total_tiles;
      g1.tile_counter = counters + 1;
      rec.begin("k_group1", n + (uint64_t)tau1 * n / 8);
      chk(launch_group<uint8_t, uint8_t, false>(g1, s, group_grid<uint8_t>()));
      rec.end();
    }

    // ---- A7 finalize ----
    if (NSD) {
      const uint64_t warps = (uint64_t)L * NSD;
      rec.begin("k_rank_local", L * BPL * 6 + L * NSD * 8);
      k_rank_local<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, s>>>(blkcnt, BPL, NSD, L, t->rank_block,
                                                                        suptot, err);
      chk(cudaGetLastError());
      rec.end();
    }
    rec.begin("k_rank_super", L * SPL * 16);
    k_rank_super<<<L, 1024, 0, s>>>(suptot, NSD, SPL, t->rank_super, err);
    chk(cudaGetLastError());
    rec.end();
  } else if (L > 0) {
    // n == 0: empty levels, one (zero) super entry per level
    chk(cudaMemsetAsync(t->rank_super, 0, L * SPL * sizeof(uint64_t), s));
  }

  // ---- the single host sync: error flag + node counts ----
  chk(cudaMemcpyAsync(h_stage, err, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  if (L) chk(cudaMemcpyAsync(h_stage + 1, t->level_node_ptr + L, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
  A.free_scratch();
  chk(cudaStreamSynchronize(s));
  if (ce != cudaSuccess) {
    A.free_outputs();
    cudaStreamSynchronize(s);
    rec.discard();
    delete t;
    return WT_ECUDA;
  }
  const uint32_t errflag = (uint32_t)(h_stage[0] & 0xffffffffu);
  t->total_nodes = L ? h_stage[1] : 0;
  rec.publish();
  if (errflag) {
    A.free_outputs();
    cudaStreamSynchronize(s);
    delete t;
    return WT_ESYMBOL;
  }
  Internal *in = new Internal();
  in->stream = s;
  in->outputs = A.outputs;  // released by wt_free
  t->internal = in;
  *out = t;
  return WT_OK;
}

}  // namespace

extern "C" {

int wt_build(const void *d_seq, uint64_t n, uint32_t elem_bytes, uint64_t sigma, void *stream, wt_tree **out) {
  return build_impl(d_seq, nullptr, false, n, elem_bytes, sigma, stream, out);
}

int wt_build_host(const void *h_seq, uint64_t n, uint32_t elem_bytes, uint64_t sigma, void *stream,
                  wt_tree **out) {
  return build_impl(nullptr, h_seq, true, n, elem_bytes, sigma, stream, out);
}

int wt_free(wt_tree *t) {
  if (!t) return WT_OK;
  Internal *in = static_cast<Internal *>(t->internal);
  cudaError_t e = cudaSuccess;
  if (in) {
    for (void *p : in->outputs) {
      cudaError_t e2 = cudaFreeAsync(p, in->stream);
      if (e2 != cudaSuccess) e = e2;
    }
    cudaError_t e3 = cudaStreamSynchronize(in->stream);
    if (e3 != cudaSuccess) e = e3;
    delete in;
  }
  delete t;
  return e == cudaSuccess ? WT_OK : WT_ECUDA;
}

static TreeView view_of(const wt_tree *t) {
  TreeView v;
  v.n = t->n;
  v.wpl = t->words_per_level;
  v.bpl = t->blocks_per_level;
  v.spl = t->supers_per_level;
  v.L = t->levels;
  v.bits = t->bits;
  v.rank_block = t->rank_block;
  v.rank_super = t->rank_super;
  return v;
}

int wt_access(const wt_tree *t, const uint64_t *d_pos, uint64_t q, uint32_t *d_out, void *stream) {
  if (!t || (q > 0 && (!d_pos || !d_out))) return WT_EINVAL;
  if (q == 0) return WT_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  k_access<<<(unsigned)((q + 255) / 256), 256, 0, s>>>(view_of(t), d_pos, q, d_out);
  return cudaGetLastError() == cudaSuccess ? WT_OK : WT_ECUDA;
}

int wt_rank(const wt_tree *t, const uint32_t *d_sym, const uint64_t *d_pos, uint64_t q, uint64_t *d_out,
            void *stream) {
  if (!t || (q > 0 && (!d_sym || !d_pos || !d_out))) return WT_EINVAL;
  if (q == 0) return WT_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  k_rank_query<<<(unsigned)((q + 255) / 256), 256, 0, s>>>(view_of(t), t->sigma, d_sym, d_pos, q, d_out);
  return cudaGetLastError() == cudaSuccess ? WT_OK : WT_ECUDA;
}

int wt_profile_enable(int on) {
  std::lock_guard<std::mutex> g(g_prof.mu);
  g_prof.enabled = on != 0;
  return WT_OK;
}

int wt_last_profile(wt_profile *out) {
  if (!out) return WT_EINVAL;
  std::lock_guard<std::mutex> g(g_prof.mu);
  *out = g_prof.last;
  return WT_OK;
}

const char *wt_version(void) { return "wt-b200 0.1 (sm_100a)"; }

}  // extern "C"
