// wt_lib.cu -- host orchestration and the extern "C" entry points of include/wt.h.
//
// One wt_build = A1 (validate + histogram), A4 (node table), then one k_group
// pass per group of <= 8 levels (A2/A3/A5/A6/A7 fused), then the A7 finalize.
// The stream is synchronised exactly once, at the end, to read the error flag
// and the node counts.
#include "wt.h"
#include "wt_group.cuh"
#include "wt_prep.cuh"
#include "wt_rank.cuh"

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

template <typename InT, typename RecT, typename OutT, bool HAS_OUT>
cudaError_t launch_group(const GroupParams &gp, cudaStream_t s) {
  const size_t smem = GROUP_WARPS * sizeof(WarpSmem<RecT>);
  auto kern = k_group<InT, RecT, OutT, HAS_OUT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, GROUP_WARPS * 32, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  kern<<<num_sms() * per_sm, GROUP_WARPS * 32, smem, s>>>(gp);
  return cudaGetLastError();
}

// Per-group scratch: chains, claim order, digit tables.
struct GroupBufs {
  uint32_t tau = 0, l0 = 0, pbits = 0, ndig = 0;
  uint64_t max_chains = 0, max_tiles = 0, max_rows = 0;
  uint32_t *chain_begin = nullptr, *chain_end = nullptr, *chain_key = nullptr, *chain_row = nullptr;
  uint32_t *row_start = nullptr, *chain_prefix = nullptr, *tile_base = nullptr;
  uint32_t *hnt = nullptr, *tie = nullptr, *cum = nullptr, *Cseg = nullptr;
  uint32_t *scalars = nullptr;  // [0] nchains, [1] total tiles, [2] tile counter, [3] nrows
  uint2 *claim = nullptr;
  void alloc(Allocs &A) {
    chain_begin = A.alloc<uint32_t>(max_chains, false);
    chain_end = A.alloc<uint32_t>(max_chains, false);
    chain_key = A.alloc<uint32_t>(max_chains, false);
    chain_row = A.alloc<uint32_t>(max_chains, false);
    row_start = A.alloc<uint32_t>(max_rows, false);
    tile_base = A.alloc<uint32_t>(max_chains, false);
    hnt = A.alloc<uint32_t>(max_tiles + 2, false);
    tie = A.alloc<uint32_t>(max_tiles + 2, false);
    cum = A.alloc<uint32_t>(max_tiles + 2, false);
    Cseg = A.alloc<uint32_t>(max_rows * (ndig + 1), false);
    scalars = A.alloc<uint32_t>(4, false);
    claim = A.alloc<uint2>(max_tiles, false);
  }
};

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

  const void *seq = d_seq;
  if (from_host) {
    void *d = A.alloc<uint8_t>(n * eb, false);
    if (!A.fail && n) {
      if (cudaMemcpyAsync(d, h_seq, n * eb, cudaMemcpyHostToDevice, s) != cudaSuccess) A.fail = true;
    }
    seq = d;
  }

  // ---- plan: groups of <= 8 levels; A1 chunks are the group-0 chains ----
  const uint32_t NG = (L + TAU_MAX - 1) / TAU_MAX;
  GroupBufs G[2];
  const uint64_t ntiles_n = std::max<uint64_t>((n + TW - 1) / TW, 1);
  uint32_t K = (uint32_t)std::min<uint64_t>((uint64_t)num_sms() * 2, ntiles_n);
  const uint64_t CH = ((ntiles_n + K - 1) / K) * TW;
  K = (uint32_t)std::max<uint64_t>((n + CH - 1) / CH, 1);
  for (uint32_t g = 0; g < NG; g++) {
    GroupBufs &gb = G[g];
    gb.l0 = g * TAU_MAX;
    gb.tau = std::min<uint32_t>(TAU_MAX, L - gb.l0);
    gb.pbits = L - gb.l0 - gb.tau;
    gb.ndig = 1u << gb.tau;
    if (g == 0) {
      gb.max_chains = K;
      gb.max_rows = 1;
      gb.max_tiles = ntiles_n + 1;
    } else {
      gb.max_chains = std::min<uint64_t>(1ull << gb.l0, std::max<uint64_t>(n, 1));
      gb.max_rows = gb.max_chains;
      gb.max_tiles = ntiles_n + gb.max_chains + 1;
    }
    gb.alloc(A);
  }
  uint32_t *err = A.alloc<uint32_t>(4, false);
  uint32_t *partial = A.alloc<uint32_t>((uint64_t)K * NDIG, false);
  if (NG) G[0].chain_prefix = A.alloc<uint32_t>((uint64_t)K * NDIG, false);
  uint32_t *ncount = A.alloc<uint32_t>(L + 1, false);
  uint32_t *blkcnt = A.alloc<uint32_t>(L * BPL, false);
  uint64_t *suptot = A.alloc<uint64_t>(L * NSD, false);
  uint64_t max_tiles = 1;
  for (uint32_t g = 0; g < NG; g++) max_tiles = std::max(max_tiles, G[g].max_tiles);
  uint32_t *state = A.alloc<uint32_t>(max_tiles * NDIG, false);
  void *keys1 = NG > 1 ? (void *)A.alloc<uint8_t>(n, false) : nullptr;

  static uint64_t *h_stage = nullptr;  // pinned staging for the single D2H
  static std::mutex stage_mu;
  {
    std::lock_guard<std::mutex> g(stage_mu);
    if (!h_stage && cudaMallocHost(&h_stage, 64 * sizeof(uint64_t)) != cudaSuccess) A.fail = true;
  }
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
  if (L && n) {
    chk(cudaMemsetAsync(t->bits, 0, L * WPL * sizeof(uint64_t), s));
    chk(cudaMemsetAsync(blkcnt, 0, L * BPL * sizeof(uint32_t), s));
  }
  for (uint32_t g = 0; g < NG && n; g++) {
    chk(cudaMemsetAsync(G[g].scalars, 0, 4 * sizeof(uint32_t), s));
    chk(cudaMemsetAsync(G[g].hnt, 0, (G[g].max_tiles + 2) * sizeof(uint32_t), s));
    chk(cudaMemsetAsync(G[g].tie, 0, (G[g].max_tiles + 2) * sizeof(uint32_t), s));
    if (g > 0) chk(cudaMemsetAsync(G[g].Cseg, 0, G[g].max_rows * (G[g].ndig + 1) * sizeof(uint32_t), s));
  }

  // ---- A1: validate + chunked digit histogram of the top tau0 bits ----
  {
    const uint32_t tau0 = NG ? G[0].tau : 0;
    const uint32_t shift = L - tau0;
    rec.begin("k_hist", n * eb);
    if (eb == 1)
      k_hist<uint8_t><<<K, 1024, 0, s>>>((const uint8_t *)seq, n, sigma, shift, 1u << tau0, CH, partial, err);
    else if (eb == 2)
      k_hist<uint16_t><<<K, 1024, 0, s>>>((const uint16_t *)seq, n, sigma, shift, 1u << tau0, CH, partial, err);
    else
      k_hist<uint32_t><<<K, 1024, 0, s>>>((const uint32_t *)seq, n, sigma, shift, 1u << tau0, CH, partial, err);
    chk(cudaGetLastError());
    rec.end();
  }

  if (L > 0 && n > 0) {
    for (uint32_t g = 0; g < NG; g++) {
      GroupBufs &gb = G[g];
      // ---- chains + digit table (Cseg) of this group ----
      if (g == 0) {
        rec.begin("k_chunk_scan", (uint64_t)K * gb.ndig * 8);
        k_chunk_scan<<<1, NDIG, 0, s>>>(partial, K, gb.ndig, n, CH, gb.chain_prefix, gb.Cseg, gb.row_start,
                                        gb.chain_begin, gb.chain_end, gb.chain_key, gb.chain_row, gb.scalars, err);
        chk(cudaGetLastError());
        rec.end();
        chk(cudaMemsetAsync(gb.scalars + 3, 0, sizeof(uint32_t), s));
        static const uint32_t one = 1;
        chk(cudaMemcpyAsync(gb.scalars + 3, &one, sizeof(uint32_t), cudaMemcpyHostToDevice, s));
      } else {
        rec.begin("k_chains", gb.max_chains * 24);
        k_chains_from_nodes<<<(unsigned)std::min<uint64_t>((gb.max_chains + 255) / 256, 4096), 256, 0, s>>>(
            t->level_node_ptr, ncount, gb.l0, t->node_key, t->node_start, n, gb.chain_begin, gb.chain_end, gb.chain_key,
            gb.chain_row, gb.row_start, gb.scalars, err);
        chk(cudaGetLastError());
        rec.end();
        chk(cudaMemcpyAsync(gb.scalars + 3, gb.scalars, sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
      }
      // ---- claim order ----
      rec.begin("k_claims", gb.max_tiles * 8);
      k_claims<<<1, 1024, 0, s>>>(gb.chain_begin, gb.chain_end, gb.scalars, gb.tile_base, gb.hnt, gb.cum, gb.tie,
                                  gb.claim, gb.scalars + 1, err);
      chk(cudaGetLastError());
      rec.end();
      if (g > 0) {
        // per-row digit histogram of the narrowed keys -> Cseg
        rec.begin("k_seg_hist", n);
        k_seg_hist<uint8_t><<<num_sms() * 8, 256, 0, s>>>((const uint8_t *)keys1, gb.pbits, gb.ndig, gb.claim,
                                                          gb.scalars + 1, gb.chain_begin, gb.chain_end,
                                                          gb.chain_row, gb.Cseg, err);
        chk(cudaGetLastError());
        rec.end();
        rec.begin("k_seg_scan", gb.max_rows * (gb.ndig + 1) * 8);
        k_seg_scan<<<(unsigned)((gb.max_rows * 32 + 255) / 256), 256, 0, s>>>(gb.Cseg, gb.scalars + 3, gb.ndig, err);
        chk(cudaGetLastError());
        rec.end();
      }
      // ---- A4: node table of this group's levels ----
      {
        const uint32_t k_lo = g == 0 ? 0u : 1u;
        const uint32_t k_hi = std::min<uint32_t>(gb.tau, L - 1 - gb.l0);  // inclusive
        if (k_hi >= k_lo) {
          rec.begin("k_nodes_count", 0);
          k_nodes_count<<<k_hi - k_lo + 1, 1024, 0, s>>>(gb.Cseg, gb.scalars + 3, gb.tau, gb.l0, k_lo, ncount, err);
          chk(cudaGetLastError());
          rec.end();
          rec.begin("k_nodes_emit", 0);
          k_nodes_emit<<<k_hi - k_lo + 1, 1024, 0, s>>>(gb.Cseg, gb.scalars + 3, gb.tau, gb.l0, k_lo, L,
                                                        gb.chain_key, gb.row_start, ncount, t->level_node_ptr,
                                                        t->node_key, t->node_start, err);
          chk(cudaGetLastError());
          rec.end();
        }
      }
      // ---- the fused tau-level pass ----
      if (g > 0) chk(cudaMemsetAsync(state, 0, gb.max_tiles * NDIG * sizeof(uint32_t), s));
      else chk(cudaMemsetAsync(state, 0, max_tiles * NDIG * sizeof(uint32_t), s));
      GroupParams gp{};
      gp.keys_in = g == 0 ? seq : keys1;
      gp.keys_out = (g + 1 < NG) ? keys1 : nullptr;
      gp.n = n;
      gp.l0 = gb.l0;
      gp.tau = gb.tau;
      gp.pbits = gb.pbits;
      gp.claim = gb.claim;
      gp.total_tiles = gb.scalars + 1;
      gp.tile_base = gb.tile_base;
      gp.chain_begin = gb.chain_begin;
      gp.chain_end = gb.chain_end;
      gp.chain_key = gb.chain_key;
      gp.chain_row = gb.chain_row;
      gp.chain_prefix = gb.chain_prefix;
      gp.Cseg = gb.Cseg;
      gp.row_start = gb.row_start;
      gp.tile_counter = gb.scalars + 2;
      gp.state = state;
      gp.bits = t->bits;
      gp.wpl = WPL;
      gp.blkcnt = blkcnt;
      gp.bpl = BPL;
      gp.err = err;
      const bool has_out = g + 1 < NG;
      const uint64_t in_bytes = g == 0 ? n * eb : n;
      char name[32];
      snprintf(name, sizeof(name), "k_group%u", g);
      rec.begin(name, in_bytes + (has_out ? n : 0) + (uint64_t)gb.tau * n / 8);
      if (g > 0) {
        chk(launch_group<uint8_t, uint8_t, uint8_t, false>(gp, s));
      } else if (!has_out) {
        if (eb == 1) chk(launch_group<uint8_t, uint8_t, uint8_t, false>(gp, s));
        else if (eb == 2) chk(launch_group<uint16_t, uint8_t, uint8_t, false>(gp, s));
        else chk(launch_group<uint32_t, uint8_t, uint8_t, false>(gp, s));
      } else {
        if (eb == 2) chk(launch_group<uint16_t, uint16_t, uint8_t, true>(gp, s));
        else chk(launch_group<uint32_t, uint16_t, uint8_t, true>(gp, s));
      }
      rec.end();
    }

    // ---- A7 finalize ----
    if (NSD) {
      const uint64_t warps = (uint64_t)L * NSD;
      rec.begin("k_rank_local", L * BPL * 6 + L * NSD * 8);
      k_rank_local<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, s>>>(blkcnt, BPL, NSD, L, t->rank_block, suptot,
                                                                        err);
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
