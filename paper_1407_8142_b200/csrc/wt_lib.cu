// wt_lib.cu -- host orchestration of the tree and the extern "C" entry points
// wt_build / wt_free / wt_access / wt_rank / wt_select* / profiling hooks of
// include/wt.h.
//
// One wt_build = A1 (validate + histogram), A4 (node table), then one k_group
// pass per group of <= 8 levels (A2/A3/A5/A6 fused), then the A7 finalize.
// The stream is synchronised exactly once, at the end, to read the error flag
// and the node counts.
#include "wt_host.cuh"
#include "wt_group.cuh"
#include "wt_wgroup.cuh"
#include "wt_local.cuh"
#include "wt_prep.cuh"
#include "wt_rank.cuh"
#include "wt_select.cuh"
#include "wt_small.cuh"
#include "wt_dist.cuh"

using namespace wtb;
using namespace wthost;

namespace {

// Launch configuration of one k_group instantiation (persistent, occupancy-sized grid).
struct GroupLaunch {
  void (*kern)(GroupParams) = nullptr;
  size_t smem = 0;
  int grid = 0;
  int threads = 0;
  int workers = 0;    // independent chain workers (CTAs, or warps for k_wgroup)
  uint32_t tile = 0;  // positions per tile (chains are cut at multiples of it)
};

template <typename InT, typename RecT, typename OutT, bool HAS_OUT>
GroupLaunch group_launch() {
  static PerDevice<GroupLaunch> pd_;
  return pd_.get([](GroupLaunch &gl) {
    gl.kern = k_group<InT, RecT, OutT, HAS_OUT>;
    gl.smem = 0;  // static shared memory
    gl.tile = GroupTile<RecT>::TT;
    gl.threads = WPB * 32;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gl.kern, WPB * 32, 0);
    gl.grid = num_sms() * (per_sm < 1 ? 1 : per_sm);
    gl.workers = gl.grid;
  });
}

// k_wgroup: one chain per CTA at a time, dynamic shared memory
template <typename InT, typename RecT, typename OutT, bool HAS_OUT>
GroupLaunch wgroup_launch() {
  static PerDevice<GroupLaunch> pd_;
  return pd_.get([](GroupLaunch &gl) {
    gl.kern = k_wgroup<InT, RecT, OutT, HAS_OUT>;
    gl.smem = sizeof(WGSmem<InT, RecT, HAS_OUT>);
    gl.tile = WGSize<InT, RecT>::T;
    gl.threads = CT_WARPS * 32;
    cudaFuncSetAttribute(gl.kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gl.smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gl.kern, gl.threads, gl.smem);
    gl.grid = num_sms() * (per_sm < 1 ? 1 : per_sm);
    gl.workers = gl.grid;  // one chain per CTA at a time
  });
}

inline bool use_old_group() {
  static const bool old = getenv("WT_OLD_GROUP") != nullptr;
  return old;
}

template <typename InT, typename RecT, typename OutT, bool HAS_OUT>
GroupLaunch any_group_launch() {
  return use_old_group() ? group_launch<InT, RecT, OutT, HAS_OUT>() : wgroup_launch<InT, RecT, OutT, HAS_OUT>();
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
  static PerDevice<LocalLaunch> pd_;
  return pd_.get([](LocalLaunch &ll) {
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
    if (outw == 2) return LocalLaunch{};  // not instantiated (WT_TAUS splits only): build reports WT_EUNSUPPORTED
    if (inw == 2) return local_launch<uint16_t, uint16_t, uint8_t, true>();
    return local_launch<uint32_t, uint16_t, uint8_t, true>();
  }
  if (outw == 2) return local_launch<uint32_t, uint32_t, uint16_t, true>();
  return local_launch<uint32_t, uint32_t, uint32_t, true>();
}


// k_group instantiation for (input width, record width, output width, local?)
GroupLaunch pick_group_mode(uint32_t inw, uint32_t recw, uint32_t outw, bool has_out) {
  if (!has_out) {
    if (recw == 1) {
      if (inw == 1) return any_group_launch<uint8_t, uint8_t, uint8_t, false>();
      if (inw == 2) return any_group_launch<uint16_t, uint8_t, uint8_t, false>();
      return any_group_launch<uint32_t, uint8_t, uint8_t, false>();
    }
    return GroupLaunch{};  // the last group always has <= 8 bits per record
  }
  if (recw == 1) return GroupLaunch{};  // 8-bit records with a payload: not instantiated (WT_TAUS splits only)
  if (recw == 2) {
    if (outw == 2) {  // tau < 8 with a payload of 9..15 bits (WT_TAUS splits)
      if (inw == 2) return wgroup_launch<uint16_t, uint16_t, uint16_t, true>();
      return wgroup_launch<uint32_t, uint16_t, uint16_t, true>();
    }
    if (inw == 2) return any_group_launch<uint16_t, uint16_t, uint8_t, true>();
    return any_group_launch<uint32_t, uint16_t, uint8_t, true>();
  }
  // recw == 4
  if (outw == 2) return any_group_launch<uint32_t, uint32_t, uint16_t, true>();
  return any_group_launch<uint32_t, uint32_t, uint32_t, true>();
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
  uint32_t *E = nullptr, *Cseg = nullptr, *V = nullptr;
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
      if (!use_old_group()) V = A.alloc<uint32_t>((uint64_t)max_chains * 256, false);
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

}  // namespace

namespace wthost {

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
  A.use_arena();
  A.alloc_outputs({{(void **)&t->bits, L * WPL * 8}, {(void **)&t->level_node_ptr, (L + 1) * 8},
                   {(void **)&t->node_key, max_nodes * 4}, {(void **)&t->node_start, max_nodes * 4},
                   {(void **)&t->rank_block, L * BPL * 2}, {(void **)&t->rank_super, L * SPL * 8}});

  const void *seq = d_seq;
  if (from_host) {
    void *d = A.alloc<uint8_t>(n * eb, false);
    if (!A.fail && n) {
      if (cudaMemcpyAsync(d, h_seq, n * eb, cudaMemcpyHostToDevice, s) != cudaSuccess) A.fail = true;
    }
    seq = d;
  }

  // ---- plan: groups of <= 8 levels ----
  // one or two levels (sigma <= 4): the direct kernels of wt_small.cuh
  const bool small = (L == 1 || L == 2) && n > 0 && eb == 1 && !getenv("WT_NO_SMALL") &&
                     (from_host || reinterpret_cast<uintptr_t>(d_seq) % 16 == 0);
  // levels per group: tau = 8 except the first group (it takes the rest); WT_TAUS="a,b,..."
  // (developer knob, used only when the list sums to L) overrides the split
  uint32_t taus[8] = {0}, NG = 0;
  if (!small) {
    if (const char *e = getenv("WT_TAUS")) {
      uint32_t sum = 0, k = 0;
      for (const char *c = e; *c && k < 8;) {
        const uint32_t v = (uint32_t)strtoul(c, (char **)&c, 10);
        if (v < 1 || v > TAU_MAX) { k = 0; break; }
        taus[k++] = v;
        sum += v;
        if (*c == ',') c++;
        else break;
      }
      if (sum == L && k) NG = k;
    }
    if (!NG) {
      // the FIRST group takes the remainder L - 8 (NG - 1): the records narrow to a
      // multiple of 8 bits as early as possible (32-bit records cost ~2x, 16-bit ~1.4x
      // an 8-bit level).  WT_TAUS_TAIL=1: the remainder goes last.
      NG = (L + TAU_MAX - 1) / TAU_MAX;
      static const bool tail = getenv("WT_TAUS_TAIL") != nullptr;
      for (uint32_t g = 0; g < NG; g++) taus[g] = TAU_MAX;
      if (NG) taus[tail ? NG - 1 : 0] = L - (NG - 1) * TAU_MAX;
    }
  }
  GroupBufs G[8];
  for (uint32_t g = 0, l0 = 0; g < NG; l0 += taus[g], g++) {
    GroupBufs &gb = G[g];
    gb.l0 = l0;
    gb.tau = taus[g];
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
      const uint64_t warps = (uint64_t)gb.gl.workers;  // chain workers (one chain at a time each)
      static const uint64_t cpw = getenv("WT_CHAINS_PER_WARP") ? strtoull(getenv("WT_CHAINS_PER_WARP"), 0, 10)
                                                              : 16;
      const uint64_t target = (n + cpw * warps - 1) / (cpw * warps);
      const uint64_t tt = gb.gl.tile;
      gb.CH = std::max<uint64_t>(tt, ((target + tt - 1) / tt) * tt);
      // one-tile chains pay the chain setup and the carried-word flush per tile: two tiles
      // per chain while that still leaves >= 4 chains per worker (n = 10^8, 888 workers)
      if (gb.CH == tt && n >= 8 * tt * warps) gb.CH = 2 * tt;
      gb.max_chains = g == 0 ? std::max<uint64_t>((n + gb.CH - 1) / gb.CH, 1)
                             : (n + gb.CH - 1) / gb.CH + gb.max_rows;
    }
    gb.alloc(A);
    if (has_out) gb.keys_out = A.alloc<uint8_t>(n * gb.outw, false);
  }
  uint32_t *err = A.alloc<uint32_t>(4, false);
  uint32_t *ncount = A.alloc<uint32_t>(L + 1, false);
  uint64_t *suptot = A.alloc<uint64_t>(L * NSD, false);
  // fused A7: block popcounts accumulated by the k_wgroup passes (chain-mode groups)
  bool any_chain = false;
  for (uint32_t g = 0; g < NG; g++) any_chain |= !G[g].local;
  uint32_t *blkcnt = (any_chain && !use_old_group() && n) ? A.alloc<uint32_t>((uint64_t)L * BPL, false) : nullptr;
  const uint32_t small_tiles = small ? (uint32_t)((n + SMALL_TILE - 1) / SMALL_TILE) : 0u;
  uint32_t *small_zc = small ? A.alloc<uint32_t>(small_tiles, false) : nullptr;
  uint64_t *small_tot = small ? A.alloc<uint64_t>(1, false) : nullptr;

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
  for (uint32_t g = 0; g < NG; g++) chk(cudaMemsetAsync(G[g].counts, 0, 4 * sizeof(uint32_t), s));
  cudaStream_t side = side_stream();
  // Zeroing of the bitmaps (and of the fused-A7 block counts): with level groups, one
  // memset per group on the side stream, so that it overlaps the prep kernels and the
  // earlier (compute-bound) group passes; group g's first bitmap writer waits for
  // ev_zero[g].  The side stream first waits for this stream (the allocations).
  cudaEvent_t ev_zero[8] = {};
  bool zeroed[8] = {};
  const bool zero_side = L && n && NG > 0;
  // group g's levels: zeroed on the side stream once this stream reaches this point
  auto zero_group = [&](uint32_t g) {
    if (!zero_side || g >= NG || zeroed[g]) return;
    zeroed[g] = true;
    cudaEvent_t ev0;
    chk(cudaEventCreateWithFlags(&ev0, cudaEventDisableTiming));
    chk(cudaEventRecord(ev0, s));
    chk(cudaStreamWaitEvent(side, ev0, 0));
    cudaEventDestroy(ev0);
    if (!G[g].local && !use_old_group() && !WT_BITS_MEMSET)
      // k_wgroup writes every word of its levels (put_shared_word): only the padding
      k_zero_pad<<<G[g].tau, 32, 0, side>>>(t->bits, WPL, (n + 63) / 64, G[g].l0);
    else
      chk(cudaMemsetAsync(t->bits + (uint64_t)G[g].l0 * WPL, 0, (uint64_t)G[g].tau * WPL * sizeof(uint64_t), side));
    if (blkcnt)
      chk(cudaMemsetAsync(blkcnt + (uint64_t)G[g].l0 * BPL, 0, (uint64_t)G[g].tau * BPL * sizeof(uint32_t), side));
    chk(cudaEventCreateWithFlags(&ev_zero[g], cudaEventDisableTiming));
    chk(cudaEventRecord(ev_zero[g], side));
  };
  if (zero_side) {
    // all groups now: the memsets overlap A1 and the chain setup (measured: a memset
    // running next to a persistent group pass takes its SM slots and slows it more)
    for (uint32_t g = 0; g < NG; g++) zero_group(g);
  } else {
    if (L && n) chk(cudaMemsetAsync(t->bits, 0, L * WPL * sizeof(uint64_t), s));
    if (blkcnt) chk(cudaMemsetAsync(blkcnt, 0, (uint64_t)L * BPL * sizeof(uint32_t), s));
  }
  auto wait_zero = [&](uint32_t g) {
    if (g < NG) zero_group(g);  // (no-op when already enqueued)
    if (g < 8 && ev_zero[g]) {
      chk(cudaStreamWaitEvent(s, ev_zero[g], 0));
      cudaEventDestroy(ev_zero[g]);
      ev_zero[g] = nullptr;
    }
  };

  // A7 per level group, on the side stream once the group's bitmaps are final
  cudaEvent_t ev_side = nullptr;
  bool side_used = false;
  // (the last group's directory has no later pass to overlap: main stream)
  auto rank_levels = [&](uint32_t lbeg, uint32_t nl) {
    if (!NSD || !nl || !n) return;
    const bool last = lbeg + nl >= L;
    cudaStream_t rs = last ? s : side;
    if (!last) {
      cudaEvent_t ev;
      chk(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      chk(cudaEventRecord(ev, s));
      chk(cudaStreamWaitEvent(side, ev, 0));
      cudaEventDestroy(ev);
      side_used = true;
    }
    const uint64_t warps = (uint64_t)nl * NSD;
    rec.begin("k_rank_local", nl * WPL * 8 + nl * BPL * 2 + nl * NSD * 8, rs);
    k_rank_local<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, rs>>>(t->bits, WPL, BPL, NSD, lbeg, nl,
                                                                         t->rank_block, suptot, err);
    chk(cudaGetLastError());
    rec.end();
  };

  // Work nothing on this stream waits for until the end of the build (the node tables of
  // a group's levels, the block entries of a finished group) goes to the side stream:
  // fork_side() orders the side stream after this stream's work so far; join_side()
  // makes this stream wait for the node tables enqueued there so far (before the next
  // group reads them); the end of the build waits for the whole side stream.  WT_NO_SIDE_A4: everything on this stream.
  // Not while kernel events are recorded (wt_profile_enable): a side-stream interval would
  // include the wait for SM slots behind the persistent group pass, not the kernel's time.
  static const bool side_a4_env = getenv("WT_NO_SIDE_A4") == nullptr;
  const bool side_a4 = side_a4_env && !rec.timed;
  cudaEvent_t ev_a4 = nullptr;  // the side stream's node tables so far
  auto fork_side = [&]() {
    cudaEvent_t ev;
    chk(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    chk(cudaEventRecord(ev, s));
    chk(cudaStreamWaitEvent(side, ev, 0));
    cudaEventDestroy(ev);
    side_used = true;
  };
  auto join_side = [&]() {
    if (!ev_a4) return;
    chk(cudaStreamWaitEvent(s, ev_a4, 0));
    cudaEventDestroy(ev_a4);
    ev_a4 = nullptr;
  };

  if (small) {
    // ---- sigma <= 4: level 0 by ballots, level 1 as two compacted bit streams ----
    rec.begin("k_small_count", n * eb);
    k_small_count<<<small_tiles, SMALL_WARPS * 32, 0, s>>>((const uint8_t *)seq, n, (uint32_t)sigma, L - 1,
                                                           small_zc, err);
    k_part_scan<<<1, 1024, 0, s>>>(small_zc, small_tiles, small_tot);
    chk(cudaGetLastError());
    rec.end();
    rec.begin("k_small_write", n * eb + (uint64_t)L * n / 8);
    k_small_write<<<small_tiles, SMALL_WARPS * 32, 0, s>>>((const uint8_t *)seq, n, L, small_zc, small_tot, t->bits,
                                                           WPL);
    k_small_nodes<<<1, 32, 0, s>>>(L, n, small_tot, t->level_node_ptr, t->node_key, t->node_start);
    chk(cudaGetLastError());
    rec.end();
    rec.begin("k_rank_local", (uint64_t)L * (WPL * 8 + BPL * 2 + NSD * 8));
    k_rank_local<<<(unsigned)(((uint64_t)L * NSD * 32 + 255) / 256), 256, 0, s>>>(t->bits, WPL, BPL, NSD, 0, L,
                                                                                     t->rank_block, suptot, err);
    chk(cudaGetLastError());
    rec.end();
  }

  const void *keys_in = seq;
  for (uint32_t g = 0; g < NG || (g == 0 && L == 0); g++) {
    // ---- chains of this group + their digit histograms (A1 for g = 0) ----
    if (g == 0) {
      // sigma == 1 (no group): validation in chains of 2^24 symbols (32-bit chain arithmetic)
      const uint64_t CH0 = NG ? G[0].CH : (1ull << 24);
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
      join_side();  // the node tables of level l0
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
      rec.begin(name, (uint64_t)gb.tau * WPL * 8);  // algorithmic: the group's bitmap levels
      wait_zero(g);
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
      join_side();  // the node tables of level l0
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
    if (gb.V) {
      rec.begin("k_chain_vec", gb.max_chains * 256 * 12);
      k_chain_vec<<<(unsigned)((gb.max_chains * 32 + 255) / 256), 256, 0, s>>>(gb.E, stride, gb.chain_row,
                                                                              gb.row_first, gb.counts, gb.ndig, gb.V,
                                                                              err);
      chk(cudaGetLastError());
      rec.end();
    }
    // ---- A4: node table of this group's levels l0+k_lo .. l0+k_lo+nk-1 ----
    if (gb.nk && g == 0) {
      rec.begin("k_nodes_count", 0);
      k_root_nodes<<<1, 32, 0, s>>>(gb.Cseg, gb.tau, gb.k_lo, gb.nk, L, ncount, t->level_node_ptr, t->node_key,
                                    t->node_start, err);
      chk(cudaGetLastError());
      rec.end();
    } else if (gb.nk) {
      // (side stream: it needs Cseg and the rows, and only the next group's chain setup
      // and the end of the build need it; it overlaps k_chain_vec and the group pass)
      const uint64_t rstride = gb.max_rows;
      const unsigned cgrid = (unsigned)std::min<uint64_t>((gb.max_rows * gb.nk * 32 + 255) / 256, 65535);
      cudaStream_t a4 = s;
      if (side_a4) {
        fork_side();
        a4 = side;
      }
      rec.begin("k_nodes_count", 0, a4);
      k_row_nodes_count<<<cgrid, 256, 0, a4>>>(gb.Cseg, gb.counts, gb.tau, gb.k_lo, gb.nk, rstride, gb.rowcnt, err);
      chk(cudaGetLastError());
      k_scan_rows_1<<<dim3(gb.nblk, gb.nk), 1024, 0, a4>>>(gb.rowcnt, rstride, gb.counts, gb.bsum, gb.nblk, err);
      k_scan_rows_2<<<gb.nk, 1024, 0, a4>>>(gb.bsum, gb.nblk, gb.counts, gb.l0, gb.k_lo, gb.nk, L, ncount,
                                            t->level_node_ptr, err);
      k_scan_rows_3<<<dim3(gb.nblk, gb.nk), 1024, 0, a4>>>(gb.rowcnt, rstride, gb.counts, gb.bsum, gb.nblk, err);
      k_level_ptr<<<1, 32, 0, a4>>>(ncount, gb.l0, gb.k_lo, gb.nk, L, t->level_node_ptr, err);
      chk(cudaGetLastError());
      rec.end();
      rec.begin("k_nodes_emit", 0, a4);
      k_row_nodes_emit<<<cgrid, 256, 0, a4>>>(gb.Cseg, gb.counts, gb.tau, gb.l0, gb.k_lo, gb.nk, rstride, gb.rowcnt,
                                              t->level_node_ptr, gb.row_key, gb.row_start, t->node_key,
                                              t->node_start, err);
      chk(cudaGetLastError());
      rec.end();
      if (a4 == side) {
        if (ev_a4) cudaEventDestroy(ev_a4);
        chk(cudaEventCreateWithFlags(&ev_a4, cudaEventDisableTiming));
        chk(cudaEventRecord(ev_a4, side));
      }
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
    gp.V = gb.V;
    gp.row_start = gb.row_start;
    gp.chain_counter = gb.counts + 2;
    gp.bits = t->bits;
    gp.wpl = WPL;
    gp.err = err;
    gp.blkcnt = blkcnt;
    gp.bpl = BPL;
    const bool has_out = g + 1 < NG;
    char name[32];
    snprintf(name, sizeof(name), "k_group%u", g);
    // algorithmic bytes: S read once (group 0) + the group's bitmap
    // levels; the narrowed keys between groups are overhead, not counted
    rec.begin(name, (g == 0 ? n * eb : 0) + (uint64_t)gb.tau * WPL * 8);
    wait_zero(g);
    gb.gl.kern<<<gb.gl.grid, gb.gl.threads, gb.gl.smem, s>>>(gp);
    chk(cudaGetLastError());
    rec.end();
    if (blkcnt) {
      // fused A7: the pass accumulated the block popcounts; scan them per superblock
      if (NSD) {
        cudaStream_t rs = s;
        if (side_a4 && has_out) {  // a later group follows: overlap its chain setup
          fork_side();
          rs = side;
        }
        rec.begin("k_rank_counts", (uint64_t)gb.tau * (BPL * 4 + BPL * 2 + NSD * 8), rs);
        const uint64_t warps = (uint64_t)gb.tau * NSD;
        k_rank_counts<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, rs>>>(blkcnt, BPL, NSD, gb.l0, gb.tau,
                                                                             t->rank_block, suptot, err);
        chk(cudaGetLastError());
        rec.end();
      }
    } else {
      rank_levels(gb.l0, gb.tau);
    }
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
  if (ev_a4) cudaEventDestroy(ev_a4);
  for (uint32_t g = 0; g < 8; g++) {  // groups that never launched (errors): keep s ordered
    if (ev_zero[g]) {
      chk(cudaStreamWaitEvent(s, ev_zero[g], 0));
      cudaEventDestroy(ev_zero[g]);
    }
  }
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


}  // namespace wthost

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
    // stream-ordered: after the work queued on the build stream and on every
    // stream a query or select index of this tree used
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

static void touch(const wt_tree *t, void *stream) {
  if (t && t->internal) {
    Internal *in = static_cast<Internal *>(t->internal);
    in->touched.add(static_cast<cudaStream_t>(stream), in->stream);
  }
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
  touch(t, stream);
  k_access<<<(unsigned)((q + 255) / 256), 256, 0, s>>>(view_of(t), d_pos, q, d_out);
  return cudaGetLastError() == cudaSuccess ? WT_OK : WT_ECUDA;
}

int wt_rank(const wt_tree *t, const uint32_t *d_sym, const uint64_t *d_pos, uint64_t q, uint64_t *d_out,
            void *stream) {
  if (!t || (q > 0 && (!d_sym || !d_pos || !d_out))) return WT_EINVAL;
  if (q == 0) return WT_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  touch(t, stream);
  k_rank_query<<<(unsigned)((q + 255) / 256), 256, 0, s>>>(view_of(t), t->sigma, d_sym, d_pos, q, d_out);
  return cudaGetLastError() == cudaSuccess ? WT_OK : WT_ECUDA;
}

int wt_profile_enable(int on) {
  std::lock_guard<std::mutex> g(g_prof.mu);
  g_prof.enabled = on != 0;
  if (on) g_prof.total = wt_profile{};
  return WT_OK;
}

int wt_profile_total(wt_profile *out) {
  if (!out) return WT_EINVAL;
  std::lock_guard<std::mutex> g(g_prof.mu);
  *out = g_prof.total;
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

// select directory of one structure (bits + rank directory in `v`), stream-ordered
int wthost::select_index_impl(const TreeView &v, uint64_t *sps_out, uint32_t **s0, uint32_t **s1,
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

extern "C" {

int wt_select_index(wt_tree *t, void *stream) {
  if (!t || !t->internal) return WT_EINVAL;
  Internal *in = static_cast<Internal *>(t->internal);
  touch(t, stream);
  return select_index_impl(view_of(t), &t->select_per_level, &t->select0, &t->select1, in->outputs,
                           static_cast<cudaStream_t>(stream));
}

int wt_select(const wt_tree *t, const uint32_t *d_sym, const uint64_t *d_k, uint64_t q, uint64_t *d_out,
              void *stream) {
  if (!t || (q > 0 && (!d_sym || !d_k || !d_out)) || !t->select_per_level) return WT_EINVAL;
  if (q == 0) return WT_OK;
  touch(t, stream);
  k_wt_select<<<(unsigned)((q + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      view_of(t), t->select0, t->select1, t->select_per_level, t->sigma, d_sym, d_k, q, d_out);
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
