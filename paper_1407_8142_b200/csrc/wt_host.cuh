// wt_host.cuh -- host-side helpers shared by the translation units of
// libwt_b200.so (wt_lib.cu: the tree; wm_lib.cu: the matrix; hwt_lib.cu: the
// Huffman-shaped tree; dist_lib.cu: the sharded-build helpers): per-build
// launch recorder, stream-ordered allocations, device queries.
#pragma once
#include "wt.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

namespace wtb {
struct TreeView;
}

namespace wthost {

struct Prof {
  bool enabled = false;
  wt_profile last{}, total{};  // the last build; all builds since profiling was enabled
  std::mutex mu;
};
inline Prof g_prof;

struct Launch {
  std::string name;
  uint64_t algo_bytes;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
};

// Per-build recorder of kernel launches (optionally timed with events).
// timing events are recycled per host thread (creating events per build
// would add host latency between the builds being timed)
inline std::vector<cudaEvent_t> &event_pool() {
  static thread_local std::vector<cudaEvent_t> pool;
  return pool;
}
inline cudaEvent_t event_get() {
  auto &pool = event_pool();
  if (pool.empty()) {
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
  }
  cudaEvent_t e = pool.back();
  pool.pop_back();
  return e;
}
inline void event_put(cudaEvent_t e) {
  if (e) event_pool().push_back(e);
}

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
      L.e0 = event_get();
      L.e1 = event_get();
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
        event_put(L.e0);
        event_put(L.e1);
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
    wt_profile &T = g_prof.total;  // accumulate by kernel name
    T.total_launches += p.total_launches;
    for (uint32_t i = 0; i < p.count; i++) {
      int k = -1;
      for (uint32_t j = 0; j < T.count; j++)
        if (!strcmp(T.e[j].name, p.e[i].name)) k = (int)j;
      if (k < 0 && T.count < WT_PROF_MAX) {
        k = (int)T.count++;
        memcpy(T.e[k].name, p.e[i].name, sizeof(T.e[k].name));
      }
      if (k >= 0) {
        T.e[k].ms += p.e[i].ms;
        T.e[k].launches += p.e[i].launches;
        T.e[k].algo_bytes += p.e[i].algo_bytes;
      }
    }
  }
  void discard() {
    if (timed)
      for (auto &L : launches) {
        event_put(L.e0);
        event_put(L.e1);
      }
  }
};

// Streams other than the build stream on which queries / select indexes of a
// structure were enqueued: its free waits for them (an event per stream)
// before releasing the memory on the build stream.
struct TouchSet {
  std::mutex mu;
  std::vector<cudaStream_t> streams;
  void add(cudaStream_t s, cudaStream_t build) {
    if (s == build) return;
    std::lock_guard<std::mutex> g(mu);
    for (cudaStream_t x : streams)
      if (x == s) return;
    streams.push_back(s);
  }
  cudaError_t order_before(cudaStream_t build) {  // build stream waits for every touched stream
    std::lock_guard<std::mutex> g(mu);
    cudaError_t e = cudaSuccess;
    for (cudaStream_t x : streams) {
      cudaEvent_t ev;
      if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) return cudaErrorUnknown;
      if (cudaEventRecord(ev, x) != cudaSuccess || cudaStreamWaitEvent(build, ev, 0) != cudaSuccess)
        e = cudaErrorUnknown;
      cudaEventDestroy(ev);
    }
    return e;
  }
};

struct Internal {
  cudaStream_t stream;
  std::vector<void *> outputs;
  TouchSet touched;
};

inline uint32_t levels_of(uint64_t sigma) {
  uint64_t v = sigma - 1;
  uint32_t L = 0;
  while (v) { L++; v >>= 1; }
  return L;
}

// Per-device lazily initialised state: a process may drive several GPUs, so
// launch configurations, function attributes, side streams and pool settings
// are kept per device (the current device of the calling thread).
constexpr int MAX_DEV = 64;
inline int cur_device() {
  int d = 0;
  cudaGetDevice(&d);
  return (d < 0 || d >= MAX_DEV) ? 0 : d;
}
template <typename T>
struct PerDevice {
  T v[MAX_DEV]{};
  std::once_flag f[MAX_DEV];
  template <typename Init>
  T &get(Init init) {
    const int d = cur_device();
    std::call_once(f[d], [&] { init(v[d]); });
    return v[d];
  }
};

// A second stream of the same device for the rank directory of finished
// level groups, so that it overlaps the next group pass (created once per device).
inline cudaStream_t side_stream() {
  static PerDevice<cudaStream_t> side;
  return side.get([](cudaStream_t &st) { cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking); });
}

inline int num_sms() {
  static PerDevice<int> sms;
  return sms.get([](int &v) {
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, cur_device());
    if (v <= 0) v = 148;
  });
}

inline void configure_pool_once() {
  static PerDevice<int> done;
  done.get([](int &) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, cur_device()) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  });
}

// Stream-ordered allocations that are released together on error.
// Per-thread scratch arena: reused by consecutive builds of one host thread
// (every build synchronises its stream before returning), so that a small
// build makes no allocation calls for its scratch.  Capped at ARENA_MAX;
// larger needs fall back to stream-ordered allocations.
struct Arena {
  char *base = nullptr;
  size_t cap = 0, used = 0, want = 0;
  bool busy = false;
};
inline Arena &thread_arena() {  // per host thread and device (the arena's memory lives on that device)
  static thread_local Arena a[MAX_DEV];
  return a[cur_device()];
}
constexpr size_t ARENA_MAX = 64ull << 20;

// Stream-ordered allocations that are released together on error.
struct Allocs {
  cudaStream_t s;
  std::vector<void *> scratch, outputs;
  bool fail = false;
  Arena *ar = nullptr;  // scratch is carved from the thread's arena while set
  template <typename T>
  T *alloc(size_t count, bool output) {
    if (count == 0) count = 1;
    const size_t bytes = (count * sizeof(T) + 255) & ~(size_t)255;
    if (!output && ar) {
      ar->want += bytes;
      if (ar->used + bytes <= ar->cap) {
        void *p = ar->base + ar->used;
        ar->used += bytes;
        return static_cast<T *>(p);
      }
    }
    void *p = nullptr;
    if (cudaMallocAsync(&p, count * sizeof(T), s) != cudaSuccess) {
      fail = true;
      return nullptr;
    }
    (output ? outputs : scratch).push_back(p);
    return static_cast<T *>(p);
  }
  // several outputs in one allocation (released together by the owner's free)
  bool alloc_outputs(std::initializer_list<std::pair<void **, size_t>> items) {
    size_t total = 0;
    for (const auto &it : items) total += (it.second + 255) & ~(size_t)255;
    void *p = nullptr;
    if (cudaMallocAsync(&p, total ? total : 256, s) != cudaSuccess) {
      fail = true;
      for (const auto &it : items) *it.first = nullptr;
      return false;
    }
    outputs.push_back(p);
    char *c = static_cast<char *>(p);
    for (const auto &it : items) {
      *it.first = c;
      c += (it.second + 255) & ~(size_t)255;
    }
    return true;
  }
  void use_arena() {  // not for nested builds (the arena is then busy)
    Arena &a = thread_arena();
    if (a.busy) return;
    a.busy = true;
    a.used = a.want = 0;
    ar = &a;
  }
  void free_scratch() {
    for (void *p : scratch) cudaFreeAsync(p, s);
    scratch.clear();
  }
  void free_outputs() {
    for (void *p : outputs) cudaFreeAsync(p, s);
    outputs.clear();
  }
  // after the build's stream is synchronised: release (and grow) the arena
  ~Allocs() {
    if (!ar) return;
    if (ar->want > ar->cap && ar->want <= ARENA_MAX) {
      if (ar->base) cudaFree(ar->base);
      ar->base = nullptr;
      ar->cap = 0;
      if (cudaMalloc(&ar->base, ar->want) == cudaSuccess) ar->cap = ar->want;
    }
    ar->used = 0;
    ar->busy = false;
  }
};

// bytes of an unsigned integer holding `bits` bits
inline uint32_t width_of(uint32_t bits) { return bits <= 8 ? 1u : (bits <= 16 ? 2u : 4u); }

// Defined in wt_lib.cu.  build_impl: the whole wt_build (the Huffman-shaped
// build runs it on padded codes); select_index_impl: the select directory of
// one structure (tree or matrix).
int build_impl(const void *d_seq, const void *h_seq, bool from_host, uint64_t n, uint32_t eb, uint64_t sigma,
               void *stream_v, wt_tree **out, bool force_chain);
int select_index_impl(const wtb::TreeView &v, uint64_t *sps_out, uint32_t **s0, uint32_t **s1,
                      std::vector<void *> &owned, cudaStream_t s);

}  // namespace wthost
