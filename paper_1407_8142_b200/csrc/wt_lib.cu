// wt_lib.cu -- host orchestration and the extern "C" entry points of include/wt.h.
//
// One wt_build = A1 (validate + histogram), A4 (node table), then one k_group
// pass per group of <= 8 levels (A2/A3/A5/A6/A7 fused), then the A7 finalize.
// The stream is synchronised exactly once, at the end, to read the error flag
// and the node counts.
#include "wt.h"
#include "wt_group.cuh"
#include "wt_local.cuh"
#include "wt_prep.cuh"
#include "wt_rank.cuh"
#include "wt_wm.cuh"
#include "wt_select.cuh"
#include "wt_huff.cuh"
#include "wt_dist.cuh"

#include <cstdio>
#include <algorithm>
#include <cstdlib>
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
  cudaStream_t cur = nullptr;
  void begin(const char *name, uint64_t bytes, cudaStream_t on = nullptr) {
    Launch L;
    L.name = name;
    L.algo_bytes = bytes;
    cur = on ? on : s;
    if (timed) {
      cudaEventCreate(&L.e0);
      cudaEventCreate(&L.e1);
      cudaEventRecord(L.e0, cur);
    }
    launches.push_back(L);
  }
  void end() {
    if (timed) cudaEventRecord(launches.back().e1, cur);
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

// A second stream of the same device for the rank directory of finished
// level groups, so that it overlaps the next group pass (created once).
cudaStream_t side_stream() {
  static cudaStream_t side = nullptr;
  static std::once_flag f;
  std::call_once(f, [] { cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking); });
  return side;
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

// Launch configuration of one k_group instantiation (persistent, occupancy-sized grid).
struct GroupLaunch {
  void (*kern)(GroupParams) = nullptr;
  size_t smem = 0;
  int grid = 0;
  uint32_t tile = 0;  // positions per tile (chains are cut at multiples of it)
};

template <typename InT, typename RecT, typename OutT, bool HAS_OUT>
GroupLaunch group_launch() {
  static GroupLaunch gl;
  static std::once_flag f;
  std::call_once(f, [] {
    gl.kern = k_group<InT, RecT, OutT, HAS_OUT>;
    gl.smem = 0;  // static shared memory
    gl.tile = GroupTile<RecT>::TT;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gl.kern, WPB * 32, 0);
    gl.grid = num_sms() * (per_sm < 1 ? 1 : per_sm);
  });
  return gl;
}

struct LocalLaunch {
  void (*count)(LocalParams) = nullptr;
  void (*build)(LocalParams) = nullptr;
  void (*big)(LocalParams) = nullptr;
  size_t smem = 0, smem_count = 0, smem_big = 0;
  int grid = 0, grid_count = 0, grid_big = 0;
};

template <typename InT, typename RecT, typename OutT, bool HAS_OUT>
LocalLaunch local_launch() {
  static LocalLaunch ll;
  static std::once_flag f;
  std::call_once(f, [] {
    ll.count = k_local<InT, RecT, OutT, HAS_OUT, LM_COUNT>;
    ll.build = k_local<InT, RecT, OutT, HAS_OUT, LM_BUILD>;
    ll.big = k_local<InT, RecT, OutT, HAS_OUT, LM_BIG>;
    ll.smem_count = LOCAL_WARPS * sizeof(LocalSmem<RecT, LM_COUNT>);
    ll.smem = LOCAL_WARPS * sizeof(LocalSmem<RecT, LM_BUILD>);
    ll.smem_big = LOCAL_WARPS * sizeof(LocalSmem<RecT, LM_BIG>);
    auto setup = [](void (*f)(LocalParams), size_t smem, int *grid) {
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, LOCAL_WARPS * 32, smem);
      *grid = num_sms() * (per_sm < 1 ? 1 : per_sm);
    };
    setup(ll.count, ll.smem_count, &ll.grid_count);
    setup(ll.build, ll.smem, &ll.grid);
    setup(ll.big, ll.smem_big, &ll.grid_big);
  });
  return ll;
}

LocalLaunch pick_local(uint32_t inw, uint32_t recw, uint32_t outw, bool has_out) {
  if (!has_out) {
    if (recw == 1) {
      if (inw == 1) return local_launch<uint8_t, uint8_t, uint8_t, false>();
      if (inw == 2) return local_launch<uint16_t, uint8_t, uint8_t, false>();
      return local_launch<uint32_t, uint8_t, uint8_t, false>();
    }
    return LocalLaunch{};
  }
  if (recw == 2) {
    if (inw == 2) return local_launch<uint16_t, uint16_t, uint8_t, true>();
    return local_launch<uint32_t, uint16_t, uint8_t, true>();
  }
  if (outw == 2) return local_launch<uint32_t, uint32_t, uint16_t, true>();
  return local_launch<uint32_t, uint32_t, uint32_t, true>();
}

// bytes of an unsigned integer holding `bits` bits
uint32_t width_of(uint32_t bits) { return bits <= 8 ? 1u : (bits <= 16 ? 2u : 4u); }

// k_group instantiation for (input width, record width, output width, local?)
GroupLaunch pick_group_mode(uint32_t inw, uint32_t recw, uint32_t outw, bool has_out) {
  if (!has_out) {
    if (recw == 1) {
      if (inw == 1) return group_launch<uint8_t, uint8_t, uint8_t, false>();
      if (inw == 2) return group_launch<uint16_t, uint8_t, uint8_t, false>();
      return group_launch<uint32_t, uint8_t, uint8_t, false>();
    }
    return GroupLaunch{};  // the last group always has <= 8 bits per record
  }
  if (recw == 2) {
    if (inw == 2) return group_launch<uint16_t, uint16_t, uint8_t, true>();
    return group_launch<uint32_t, uint16_t, uint8_t, true>();
  }
  // recw == 4
  if (outw == 2) return group_launch<uint32_t, uint32_t, uint16_t, true>();
  return group_launch<uint32_t, uint32_t, uint32_t, true>();
}

// Per-group scratch: chains, rows, digit tables, node-count scans.
struct GroupBufs {
  uint32_t tau = 0, l0 = 0, pbits = 0, ndig = 0, nk = 0, k_lo = 0;
  uint32_t inw = 0, recw = 0, outw = 0;
  bool local = false;
  uint64_t CH = TW, max_chains = 0, max_rows = 0;
  GroupLaunch gl;
  LocalLaunch ll;
  uint32_t nbatch = 0;
  uint32_t *batch_first = nullptr, *bcounts = nullptr;  // bcounts: [0] claim counter, [1] batches, [2] deferred rows
  uint64_t ndefer = 0;
  uint32_t *defer = nullptr;
  void *keys_out = nullptr;
  uint32_t *chain_begin = nullptr, *chain_end = nullptr, *chain_row = nullptr;
  uint32_t *row_first = nullptr, *row_start = nullptr, *row_key = nullptr;
  uint32_t *E = nullptr, *Cseg = nullptr;
  uint32_t *rowcnt = nullptr, *bsum = nullptr;
  uint32_t nblk = 0;
  uint32_t *counts = nullptr;  // [0] chains, [1] rows, [2] chain claim counter
  void alloc(Allocs &A) {
    chain_begin = A.alloc<uint32_t>(max_chains, false);
    chain_end = A.alloc<uint32_t>(max_chains, false);
    chain_row = A.alloc<uint32_t>(max_chains, false);
    row_first = A.alloc<uint32_t>(max_rows + 1, false);
    row_start = A.alloc<uint32_t>(max_rows, false);
    row_key = A.alloc<uint32_t>(max_rows, false);
    if (!local) {
      E = A.alloc<uint32_t>((uint64_t)ndig * (max_chains + 1), false);
      Cseg = A.alloc<uint32_t>(max_rows * (ndig + 1), false);
    }
    const uint64_t nunits = local ? nbatch : max_rows;  // node counts per batch (local) or row
    nblk = (uint32_t)((nunits + SCAN_BLK - 1) / SCAN_BLK);
    if (nk) {
      rowcnt = A.alloc<uint32_t>((uint64_t)nk * nunits, false);
      bsum = A.alloc<uint32_t>((uint64_t)nk * nblk, false);
    }
    if (local) {
      batch_first = A.alloc<uint32_t>(nbatch + 1, false);
      bcounts = A.alloc<uint32_t>(4, false);
      defer = A.alloc<uint32_t>(ndefer * DEFER_W, false);
    }
    counts = A.alloc<uint32_t>(4, false);
  }
};

int build_impl(const void *d_seq, const void *h_seq, bool from_host, uint64_t n, uint32_t eb,
               uint64_t sigma, void *stream_v, wt_tree **out, bool force_chain) {
  if (!out) return WT_EINVAL;
  *out = nullptr;
  if (eb != 1 && eb != 2 && eb != 4) return WT_EINVAL;
  if (sigma < 1 || sigma > (1ull << (8 * eb))) return WT_EINVAL;
  if (n >= (1ull << 32)) return WT_EINVAL;
  if (n > 0 && !(from_host ? h_seq : d_seq)) return WT_EINVAL;
  const uint32_t L = levels_of(sigma);
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

  const void *seq = d_seq;
  if (from_host) {
    void *d = A.alloc<uint8_t>(n * eb, false);
    if (!A.fail && n) {
      if (cudaMemcpyAsync(d, h_seq, n * eb, cudaMemcpyHostToDevice, s) != cudaSuccess) A.fail = true;
    }
    seq = d;
  }

  // ---- plan: groups of <= 8 levels ----
  const uint32_t NG = (L + TAU_MAX - 1) / TAU_MAX;
  GroupBufs G[4];
  for (uint32_t g = 0; g < NG; g++) {
    GroupBufs &gb = G[g];
    gb.l0 = g * TAU_MAX;
    gb.tau = std::min<uint32_t>(TAU_MAX, L - gb.l0);
    gb.pbits = L - gb.l0 - gb.tau;
    gb.ndig = 1u << gb.tau;
    gb.k_lo = g == 0 ? 0u : 1u;
    gb.inw = g == 0 ? eb : width_of(L - gb.l0);
    gb.recw = width_of(L - gb.l0);
    gb.outw = width_of(gb.pbits);
    const bool has_out = g + 1 < NG;
    gb.max_rows = g == 0 ? 1 : std::min<uint64_t>(1ull << gb.l0, std::max<uint64_t>(n, 1));
    // local mode when level-l0 nodes are small on average (one tile per row)
    gb.local = !force_chain && g > 0 && n / gb.max_rows <= (uint64_t)TW / 8;
    const uint32_t k_hi = std::min<uint32_t>(gb.tau, L - 1 - gb.l0);
    gb.nk = k_hi >= gb.k_lo ? k_hi - gb.k_lo + 1 : 0;
    if (gb.local) gb.ll = pick_local(gb.inw, gb.recw, gb.outw, has_out);
    else gb.gl = pick_group_mode(gb.inw, gb.recw, gb.outw, has_out);
    if (gb.local ? !gb.ll.build : !gb.gl.kern) {
      A.free_scratch();
      A.free_outputs();
      cudaStreamSynchronize(s);
      delete t;
      return WT_EUNSUPPORTED;
    }
    if (gb.local) {
      gb.nbatch = (uint32_t)((n + TW - 1) / TW);
      gb.ndefer = n / (LT + 1) + 1;
      gb.max_chains = 1;
    } else {
      const uint64_t warps = (uint64_t)gb.gl.grid;  // CTAs (one chain at a time each)
      static const uint64_t cpw =
          getenv("WT_CHAINS_PER_WARP") ? strtoull(getenv("WT_CHAINS_PER_WARP"), 0, 10) : 16;
      const uint64_t target = (n + cpw * warps - 1) / (cpw * warps);
      const uint64_t tt = gb.gl.tile;
      gb.CH = std::max<uint64_t>(tt, ((target + tt - 1) / tt) * tt);
      gb.max_chains = g == 0 ? std::max<uint64_t>((n + gb.CH - 1) / gb.CH, 1)
                             : (n + gb.CH - 1) / gb.CH + gb.max_rows;
    }
    gb.alloc(A);
    if (has_out) gb.keys_out = A.alloc<uint8_t>(n * gb.outw, false);
  }
  uint32_t *err = A.alloc<uint32_t>(4, false);
  uint32_t *ncount = A.alloc<uint32_t>(L + 1, false);
  uint64_t *suptot = A.alloc<uint64_t>(L * NSD, false);

  // pinned staging for the single D2H; one per host thread, so that builds
  // issued concurrently from several threads do not share it
  static thread_local uint64_t *h_stage = nullptr;
  if (!h_stage && cudaMallocHost(&h_stage, 64 * sizeof(uint64_t)) != cudaSuccess) A.fail = true;
  if (A.fail) {
    A.free_scratch();
    A.free_outputs();
    cudaStreamSynchronize(s);
    rec.discard();
    delete t;
    return WT_ENOMEM;
  }

  cudaError_t ce = cudaSuccess;
  auto chk = [&](cudaError_t e) {
    if (e != cudaSuccess && ce == cudaSuccess) ce = e;
  };

  chk(cudaMemsetAsync(err, 0, 4 * sizeof(uint32_t), s));
  chk(cudaMemsetAsync(t->level_node_ptr, 0, (L + 1) * sizeof(uint64_t), s));
  if (L && n) chk(cudaMemsetAsync(t->bits, 0, L * WPL * sizeof(uint64_t), s));
  for (uint32_t g = 0; g < NG; g++) chk(cudaMemsetAsync(G[g].counts, 0, 4 * sizeof(uint32_t), s));

  // A7 per level group, on the side stream once the group's bitmaps are final
  cudaStream_t side = side_stream();
  cudaEvent_t ev_side = nullptr;
  bool side_used = false;
  auto rank_levels = [&](uint32_t lbeg, uint32_t nl) {
    if (!NSD || !nl || !n) return;
    cudaEvent_t ev;
    chk(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    chk(cudaEventRecord(ev, s));
    chk(cudaStreamWaitEvent(side, ev, 0));
    cudaEventDestroy(ev);
    const uint64_t warps = (uint64_t)nl * NSD;
    rec.begin("k_rank_local", nl * WPL * 8 + nl * BPL * 2 + nl * NSD * 8, side);
    k_rank_local<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, side>>>(t->bits, WPL, BPL, NSD, lbeg, nl,
                                                                           t->rank_block, suptot, err);
    chk(cudaGetLastError());
    rec.end();
    side_used = true;
  };

  const void *keys_in = seq;
  for (uint32_t g = 0; g < NG || (g == 0 && L == 0); g++) {
    // ---- chains of this group + their digit histograms (A1 for g = 0) ----
    if (g == 0) {
      const uint64_t CH0 = NG ? G[0].CH : std::max<uint64_t>(n, 1);
      const uint32_t K = NG ? (uint32_t)G[0].max_chains : (uint32_t)((n + CH0 - 1) / CH0);
      const uint32_t tau0 = NG ? G[0].tau : 0;
      const uint32_t ndig0 = 1u << tau0;
      uint32_t *cb, *ce_, *cr, *rf, *rs, *rk, *E, *cnt;
      uint32_t stride;
      if (NG) {
        GroupBufs &gb = G[0];
        cb = gb.chain_begin; ce_ = gb.chain_end; cr = gb.chain_row; rf = gb.row_first; rs = gb.row_start;
        rk = gb.row_key; E = gb.E; cnt = gb.counts; stride = (uint32_t)gb.max_chains + 1;
      } else {  // sigma == 1: validation only
        cb = A.alloc<uint32_t>(K, false); ce_ = A.alloc<uint32_t>(K, false); cr = A.alloc<uint32_t>(K, false);
        rf = A.alloc<uint32_t>(2, false); rs = A.alloc<uint32_t>(1, false); rk = A.alloc<uint32_t>(1, false);
        E = A.alloc<uint32_t>(K + 1, false); cnt = A.alloc<uint32_t>(4, false); stride = K + 1;
        if (A.fail) { ce = cudaErrorMemoryAllocation; break; }
      }
      if (n) {
        k_chains_root<<<(K + 255) / 256, 256, 0, s>>>(n, CH0, K, cb, ce_, cr, rf, rs, rk, cnt, err);
        chk(cudaGetLastError());
        rec.begin("k_hist", n * eb);
        const uint32_t shift = L - tau0;
        const unsigned grid = std::min<uint32_t>(K, 4 * num_sms());
        if (eb == 1)
          k_chain_hist<uint8_t, true><<<grid, 512, 0, s>>>((const uint8_t *)seq, sigma, shift, ndig0, cb, ce_, cnt, stride, E, err);
        else if (eb == 2)
          k_chain_hist<uint16_t, true><<<grid, 512, 0, s>>>((const uint16_t *)seq, sigma, shift, ndig0, cb, ce_, cnt, stride, E, err);
        else
          k_chain_hist<uint32_t, true><<<grid, 512, 0, s>>>((const uint32_t *)seq, sigma, shift, ndig0, cb, ce_, cnt, stride, E, err);
        chk(cudaGetLastError());
        rec.end();
      }
      if (!NG || !n) break;
    } else if (G[g].local) {
      // ======== local mode: batches of small level-l0 nodes, finished per warp ========
      GroupBufs &gb = G[g];
      rec.begin("k_rows", gb.max_rows * 8);
      k_rows_from_nodes<<<(unsigned)std::min<uint64_t>((gb.max_rows + 255) / 256, 65535), 256, 0, s>>>(
          t->level_node_ptr, ncount, gb.l0, t->node_key, t->node_start, gb.row_start, gb.row_key, gb.counts, err);
      k_batches<<<(gb.nbatch + 256) / 256, 256, 0, s>>>(gb.row_start, gb.counts, gb.nbatch, gb.batch_first,
                                                         gb.bcounts, err);
      chk(cudaGetLastError());
      chk(cudaMemsetAsync(gb.bcounts, 0, sizeof(uint32_t), s));  // [0] = batch claim counter
      rec.end();
      LocalParams lp{};
      lp.keys_in = keys_in;
      lp.keys_out = gb.keys_out;
      lp.n = n;
      lp.l0 = gb.l0;
      lp.tau = gb.tau;
      lp.pbits = gb.pbits;
      lp.nk = gb.nk;
      lp.nbatch = gb.nbatch;
      lp.batch_first = gb.batch_first;
      lp.counts = gb.counts;
      lp.row_start = gb.row_start;
      lp.row_key = gb.row_key;
      lp.batch_counter = gb.bcounts;
      lp.batchcnt = gb.rowcnt;
      lp.level_node_ptr = t->level_node_ptr;
      lp.node_key = t->node_key;
      lp.node_start = t->node_start;
      lp.bits = t->bits;
      lp.wpl = WPL;
      lp.err = err;
      lp.defer = gb.defer;
      lp.defer_count = gb.bcounts + 2;
      chk(cudaMemsetAsync(gb.bcounts + 2, 0, sizeof(uint32_t), s));
      if (gb.nk) {
        // A4 pass 1: node counts per batch and level, then their scan (CSR offsets)
        rec.begin("k_local_count", n * gb.inw);
        gb.ll.count<<<gb.ll.grid_count, LOCAL_WARPS * 32, gb.ll.smem_count, s>>>(lp);
        chk(cudaGetLastError());
        k_scan_rows_1<<<dim3(gb.nblk, gb.nk), 1024, 0, s>>>(gb.rowcnt, gb.nbatch, gb.bcounts, gb.bsum, gb.nblk, err);
        k_scan_rows_2<<<gb.nk, 1024, 0, s>>>(gb.bsum, gb.nblk, gb.bcounts, gb.l0, gb.k_lo, gb.nk, L, ncount,
                                             t->level_node_ptr, err);
        k_scan_rows_3<<<dim3(gb.nblk, gb.nk), 1024, 0, s>>>(gb.rowcnt, gb.nbatch, gb.bcounts, gb.bsum, gb.nblk, err);
        k_level_ptr<<<1, 32, 0, s>>>(ncount, gb.l0, gb.k_lo, gb.nk, L, t->level_node_ptr, err);
        chk(cudaMemsetAsync(gb.bcounts, 0, sizeof(uint32_t), s));
        chk(cudaGetLastError());
        rec.end();
      }
      const bool has_out = g + 1 < NG;
      char name[32];
      snprintf(name, sizeof(name), "k_group%u", g);
      rec.begin(name, n * gb.inw + (has_out ? n * gb.outw : 0) + (uint64_t)gb.tau * n / 8);
      gb.ll.build<<<gb.ll.grid, LOCAL_WARPS * 32, gb.ll.smem, s>>>(lp);
      chk(cudaGetLastError());
      chk(cudaMemsetAsync(gb.bcounts, 0, sizeof(uint32_t), s));  // claim counter for the deferred rows
      gb.ll.big<<<gb.ll.grid_big, LOCAL_WARPS * 32, gb.ll.smem_big, s>>>(lp);
      chk(cudaGetLastError());
      rec.end();
      rank_levels(gb.l0, gb.tau);
      keys_in = gb.keys_out;
      continue;
    } else {
      GroupBufs &gb = G[g];
      rec.begin("k_chains", gb.max_chains * 12);
      k_chains_from_nodes<<<1, 1024, 0, s>>>(t->level_node_ptr, ncount, gb.l0, t->node_key, t->node_start, n,
                                             gb.CH, gb.chain_begin, gb.chain_end, gb.chain_row, gb.row_first,
                                             gb.row_start, gb.row_key, gb.counts, err);
      chk(cudaGetLastError());
      rec.end();
      rec.begin("k_seg_hist", n * gb.inw);
      const unsigned grid = (unsigned)std::min<uint64_t>(gb.max_chains, 4 * num_sms());
      const uint32_t estr = (uint32_t)gb.max_chains + 1;
      if (gb.inw == 1)
        k_chain_hist<uint8_t, false><<<grid, 512, 0, s>>>((const uint8_t *)keys_in, sigma, gb.pbits, gb.ndig,
                                                          gb.chain_begin, gb.chain_end, gb.counts, estr, gb.E, err);
      else if (gb.inw == 2)
        k_chain_hist<uint16_t, false><<<grid, 512, 0, s>>>((const uint16_t *)keys_in, sigma, gb.pbits, gb.ndig,
                                                           gb.chain_begin, gb.chain_end, gb.counts, estr, gb.E, err);
      else
        k_chain_hist<uint32_t, false><<<grid, 512, 0, s>>>((const uint32_t *)keys_in, sigma, gb.pbits, gb.ndig,
                                                           gb.chain_begin, gb.chain_end, gb.counts, estr, gb.E, err);
      chk(cudaGetLastError());
      rec.end();
    }
    // ======== chain mode ========
    GroupBufs &gb = G[g];
    const uint32_t stride = (uint32_t)gb.max_chains + 1;
    rec.begin("k_chain_scan", (uint64_t)gb.ndig * gb.max_chains * 8);
    k_chain_scan<<<gb.ndig, 1024, 0, s>>>(gb.E, stride, gb.counts, err);
    chk(cudaGetLastError());
    rec.end();
    rec.begin("k_row_scan", gb.max_rows * (gb.ndig + 1) * 4);
    k_row_scan<<<(unsigned)((gb.max_rows * 32 + 255) / 256), 256, 0, s>>>(gb.E, stride, gb.row_first, gb.counts,
                                                                          gb.ndig, gb.Cseg, err);
    chk(cudaGetLastError());
    rec.end();
    // ---- A4: node table of this group's levels l0+k_lo .. l0+k_lo+nk-1 ----
    if (gb.nk) {
      const uint64_t rstride = gb.max_rows;
      const unsigned cgrid = (unsigned)std::min<uint64_t>((gb.max_rows * gb.nk * 32 + 255) / 256, 65535);
      rec.begin("k_nodes_count", 0);
      k_row_nodes_count<<<cgrid, 256, 0, s>>>(gb.Cseg, gb.counts, gb.tau, gb.k_lo, gb.nk, rstride, gb.rowcnt, err);
      chk(cudaGetLastError());
      k_scan_rows_1<<<dim3(gb.nblk, gb.nk), 1024, 0, s>>>(gb.rowcnt, rstride, gb.counts, gb.bsum, gb.nblk, err);
      k_scan_rows_2<<<gb.nk, 1024, 0, s>>>(gb.bsum, gb.nblk, gb.counts, gb.l0, gb.k_lo, gb.nk, L, ncount,
                                           t->level_node_ptr, err);
      k_scan_rows_3<<<dim3(gb.nblk, gb.nk), 1024, 0, s>>>(gb.rowcnt, rstride, gb.counts, gb.bsum, gb.nblk, err);
      k_level_ptr<<<1, 32, 0, s>>>(ncount, gb.l0, gb.k_lo, gb.nk, L, t->level_node_ptr, err);
      chk(cudaGetLastError());
      rec.end();
      rec.begin("k_nodes_emit", 0);
      k_row_nodes_emit<<<cgrid, 256, 0, s>>>(gb.Cseg, gb.counts, gb.tau, gb.l0, gb.k_lo, gb.nk, rstride, gb.rowcnt,
                                             t->level_node_ptr, gb.row_key, gb.row_start, t->node_key,
                                             t->node_start, err);
      chk(cudaGetLastError());
      rec.end();
    }
    // ---- the fused tau-level pass ----
    GroupParams gp{};
    gp.keys_in = keys_in;
    gp.keys_out = gb.keys_out;
    gp.n = n;
    gp.l0 = gb.l0;
    gp.tau = gb.tau;
    gp.pbits = gb.pbits;
    gp.counts = gb.counts;
    gp.chain_begin = gb.chain_begin;
    gp.chain_end = gb.chain_end;
    gp.chain_row = gb.chain_row;
    gp.row_first = gb.row_first;
    gp.E = gb.E;
    gp.estride = stride;
    gp.Cseg = gb.Cseg;
    gp.row_start = gb.row_start;
    gp.chain_counter = gb.counts + 2;
    gp.bits = t->bits;
    gp.wpl = WPL;
    gp.err = err;
    const bool has_out = g + 1 < NG;
    char name[32];
    snprintf(name, sizeof(name), "k_group%u", g);
    rec.begin(name, n * gb.inw + (has_out ? n * gb.outw : 0) + (uint64_t)gb.tau * n / 8);
    gb.gl.kern<<<gb.gl.grid, WPB * 32, 0, s>>>(gp);
    chk(cudaGetLastError());
    rec.end();
    rank_levels(gb.l0, gb.tau);
    keys_in = gb.keys_out;
  }

  if (L > 0 && n > 0) {
    // ---- A7: rank directory (per-group block counts ran on the side stream) ----
    if (side_used) {
      chk(cudaEventCreateWithFlags(&ev_side, cudaEventDisableTiming));
      chk(cudaEventRecord(ev_side, side));
      chk(cudaStreamWaitEvent(s, ev_side, 0));
    }
    rec.begin("k_rank_super", L * SPL * 16);
    k_rank_super<<<L, 1024, 0, s>>>(suptot, NSD, SPL, t->rank_super, err);
    chk(cudaGetLastError());
    rec.end();
  } else if (L > 0) {
    // n == 0: empty levels, one (zero) super entry per level
    chk(cudaMemsetAsync(t->rank_super, 0, L * SPL * sizeof(uint64_t), s));
  }

  if (ev_side) cudaEventDestroy(ev_side);
  // ---- the single host sync: error flag + node count ----
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
    if (errflag & 1u) return WT_ESYMBOL;
    // a level-l0 node too large for local mode: rebuild with chain mode everywhere
    return force_chain ? WT_ECUDA : build_impl(d_seq, h_seq, from_host, n, eb, sigma, stream_v, out, true);
  }
  Internal *in = new Internal();
  in->stream = s;
  in->outputs = A.outputs;  // released by wt_free
  t->internal = in;
  *out = t;
  return WT_OK;
}


// ===================== wavelet matrix =====================
struct WmLaunch {
  void (*kern)(GroupParams) = nullptr;
  int grid = 0, block = 32;
  uint32_t tile = 0;
};

template <typename InT, typename RecT, typename OutT, bool HAS_OUT>
WmLaunch wm_launch() {
  static WmLaunch wl;
  static std::once_flag f;
  std::call_once(f, [] {
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
  return wl;
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
  m->bits = A.alloc<uint64_t>(L * WPL, true);
  m->zeros = A.alloc<uint64_t>(L, true);
  m->rank_block = A.alloc<uint16_t>(L * BPL, true);
  m->rank_super = A.alloc<uint64_t>(L * SPL, true);
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
    const uint64_t CH = std::max<uint64_t>(n, 1);
    k_chains_root<<<1, 256, 0, s>>>(n, CH, 1, cb, ce_, cr, rf, rs, rk, cnt, err);
    if (eb == 1) k_chain_hist<uint8_t, true><<<1, 512, 0, s>>>((const uint8_t *)d_seq, sigma, 0, 1, cb, ce_, cnt, 2, E, err);
    else if (eb == 2) k_chain_hist<uint16_t, true><<<1, 512, 0, s>>>((const uint16_t *)d_seq, sigma, 0, 1, cb, ce_, cnt, 2, E, err);
    else k_chain_hist<uint32_t, true><<<1, 512, 0, s>>>((const uint32_t *)d_seq, sigma, 0, 1, cb, ce_, cnt, 2, E, err);
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

int wt_build(const void *d_seq, uint64_t n, uint32_t elem_bytes, uint64_t sigma, void *stream, wt_tree **out) {
  return build_impl(d_seq, nullptr, false, n, elem_bytes, sigma, stream, out, false);
}

int wt_build_host(const void *h_seq, uint64_t n, uint32_t elem_bytes, uint64_t sigma, void *stream,
                  wt_tree **out) {
  return build_impl(nullptr, h_seq, true, n, elem_bytes, sigma, stream, out, false);
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

// select directory of one structure (bits + rank directory in `v`), stream-ordered
static int select_index_impl(const TreeView &v, uint64_t *sps_out, uint32_t **s0, uint32_t **s1,
                             std::vector<void *> &owned, cudaStream_t s) {
  if (*sps_out) return WT_OK;  // already built
  const uint64_t sps = (v.n + SEL_SAMPLE - 1) / SEL_SAMPLE + 1;
  const uint64_t cnt = (uint64_t)v.L * sps;
  uint32_t *a = nullptr, *b = nullptr;
  if (cnt) {
    if (cudaMallocAsync(&a, cnt * sizeof(uint32_t), s) != cudaSuccess) return WT_ENOMEM;
    if (cudaMallocAsync(&b, cnt * sizeof(uint32_t), s) != cudaSuccess) {
      cudaFreeAsync(a, s);
      return WT_ENOMEM;
    }
    const unsigned fg = (unsigned)std::min<uint64_t>((cnt + 255) / 256, 65535);
    k_fill_u32<<<fg, 256, 0, s>>>(a, cnt, (uint32_t)v.n);
    k_fill_u32<<<fg, 256, 0, s>>>(b, cnt, (uint32_t)v.n);
    const uint64_t items = (uint64_t)v.L * v.bpl;
    if (items) k_select_dir<<<(unsigned)((items + 255) / 256), 256, 0, s>>>(v, a, b, sps);
    if (cudaGetLastError() != cudaSuccess) {
      cudaFreeAsync(a, s);
      cudaFreeAsync(b, s);
      return WT_ECUDA;
    }
    owned.push_back(a);
    owned.push_back(b);
  }
  *s0 = a;
  *s1 = b;
  *sps_out = sps;
  return WT_OK;
}

int wt_select_index(wt_tree *t, void *stream) {
  if (!t || !t->internal) return WT_EINVAL;
  Internal *in = static_cast<Internal *>(t->internal);
  return select_index_impl(view_of(t), &t->select_per_level, &t->select0, &t->select1, in->outputs,
                           static_cast<cudaStream_t>(stream));
}

int wt_select(const wt_tree *t, const uint32_t *d_sym, const uint64_t *d_k, uint64_t q, uint64_t *d_out,
              void *stream) {
  if (!t || (q > 0 && (!d_sym || !d_k || !d_out)) || !t->select_per_level) return WT_EINVAL;
  if (q == 0) return WT_OK;
  k_wt_select<<<(unsigned)((q + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      view_of(t), t->select0, t->select1, t->select_per_level, t->sigma, d_sym, d_k, q, d_out);
  return cudaGetLastError() == cudaSuccess ? WT_OK : WT_ECUDA;
}

int wm_build(const void *d_seq, uint64_t n, uint32_t elem_bytes, uint64_t sigma, void *stream, wm_matrix **out) {
  return wm_build_impl(d_seq, n, elem_bytes, sigma, stream, out);
}

int wm_free(wm_matrix *m) {
  if (!m) return WT_OK;
  WmInternal *in = static_cast<WmInternal *>(m->internal);
  cudaError_t e = cudaSuccess;
  if (in) {
    for (void *p : in->outputs) {
      const cudaError_t e2 = cudaFreeAsync(p, in->stream);
      if (e2 != cudaSuccess) e = e2;
    }
    const cudaError_t e3 = cudaStreamSynchronize(in->stream);
    if (e3 != cudaSuccess) e = e3;
    delete in;
  }
  delete m;
  return e == cudaSuccess ? WT_OK : WT_ECUDA;
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
  k_wm_access<<<(unsigned)((q + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(view_of_wm(m), m->zeros,
                                                                                           d_pos, q, d_out);
  return cudaGetLastError() == cudaSuccess ? WT_OK : WT_ECUDA;
}

int wm_select_index(wm_matrix *m, void *stream) {
  if (!m || !m->internal) return WT_EINVAL;
  WmInternal *in = static_cast<WmInternal *>(m->internal);
  return select_index_impl(view_of_wm(m), &m->select_per_level, &m->select0, &m->select1, in->outputs,
                           static_cast<cudaStream_t>(stream));
}

int wm_select(const wm_matrix *m, const uint32_t *d_sym, const uint64_t *d_k, uint64_t q, uint64_t *d_out,
              void *stream) {
  if (!m || (q > 0 && (!d_sym || !d_k || !d_out)) || !m->select_per_level) return WT_EINVAL;
  if (q == 0) return WT_OK;
  k_wm_select<<<(unsigned)((q + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      view_of_wm(m), m->zeros, m->select0, m->select1, m->select_per_level, m->sigma, d_sym, d_k, q, d_out);
  return cudaGetLastError() == cudaSuccess ? WT_OK : WT_ECUDA;
}

int wm_rank(const wm_matrix *m, const uint32_t *d_sym, const uint64_t *d_pos, uint64_t q, uint64_t *d_out,
            void *stream) {
  if (!m || (q > 0 && (!d_sym || !d_pos || !d_out))) return WT_EINVAL;
  if (q == 0) return WT_OK;
  k_wm_rank<<<(unsigned)((q + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      view_of_wm(m), m->zeros, m->sigma, d_sym, d_pos, q, d_out);
  return cudaGetLastError() == cudaSuccess ? WT_OK : WT_ECUDA;
}

#ifdef WT_PHASES
int wt_phases(unsigned long long *out16) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out16, wtb::g_ph, 16 * sizeof(unsigned long long));
  unsigned long long z[16] = {0};
  cudaMemcpyToSymbol(wtb::g_ph, z, sizeof(z));
  return WT_OK;
}
#endif

#ifdef WT_DEBUG
int wt_debug_code(uint32_t *out4) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out4, wtb::g_wt_dbg, 4 * sizeof(uint32_t));
  return WT_OK;
}
#endif

}  // extern "C"


// ============ Huffman-shaped wavelet tree ============
namespace {

struct HwtInternal {
  cudaStream_t stream;
  std::vector<void *> outputs;
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
    static std::once_flag f;
    std::call_once(f, [] {
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
    static std::once_flag f;
    std::call_once(f, [] {
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
      const int frc = wt_free(pt);  // stream-ordered after the kernels above; synchronises
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

int hwt_access(const hwt_tree *t, const uint64_t *d_pos, uint64_t q, uint32_t *d_out, void *stream) {
  if (!t || !t->internal || (q > 0 && (!d_pos || !d_out))) return WT_EINVAL;
  if (q == 0) return WT_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  k_hwt_access<<<(unsigned)((q + 255) / 256), 256, 0, s>>>(view_of_hwt(t), d_pos, q, d_out);
  return cudaGetLastError() == cudaSuccess ? WT_OK : WT_ECUDA;
}

int hwt_rank(const hwt_tree *t, const uint32_t *d_sym, const uint64_t *d_pos, uint64_t q, uint64_t *d_out,
             void *stream) {
  if (!t || !t->internal || (q > 0 && (!d_sym || !d_pos || !d_out))) return WT_EINVAL;
  if (q == 0) return WT_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  k_hwt_rank<<<(unsigned)((q + 255) / 256), 256, 0, s>>>(view_of_hwt(t), d_sym, d_pos, q, d_out);
  return cudaGetLastError() == cudaSuccess ? WT_OK : WT_ECUDA;
}

}  // extern "C"


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
