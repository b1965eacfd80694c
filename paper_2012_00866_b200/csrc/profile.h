// profile.h -- per-stage launch accounting for libhusky.
//
// Every kernel launch of the library goes through a Scope, which (a) always
// counts the launch and (b) when profiling is enabled records a CUDA event
// pair around it on the launching stream.  Elapsed times are harvested at the
// library's synchronisation points (events already complete).  This is the
// T1/T2/T3 split of PAPER.md:238-245 measured per kernel family.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

namespace husky {

enum Stage : int {
  ST_ENCODE = 0, ST_HIST_SCAN, ST_RADIX, ST_RUNS_SCAN, ST_CLASSIFY, ST_FIX_SMALL, ST_FIX_MEDIUM,
  ST_REFINE, ST_GATHER, ST_MULTI, ST_COUNT
};

struct Profiler {
  std::mutex mu;
  int on = 0;  // 0 off, 1 an event pair per launch, 2 event pairs per GroupScope only
  struct Pending { int stage; cudaEvent_t a, b; uint64_t elems; };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> pool;
  double ms[ST_COUNT] = {};
  uint64_t launches[ST_COUNT] = {};
  uint64_t elems[ST_COUNT] = {};
  uint64_t total_launches = 0;  // always counted
  // mode 1: every harvested launch in order (stage, elements, ms), bounded
  struct Rec { int stage; uint64_t elems; double ms; };
  std::vector<Rec> log;
  static constexpr size_t kLogMax = 1 << 16;

  cudaEvent_t get() {
    if (!pool.empty()) { cudaEvent_t e = pool.back(); pool.pop_back(); return e; }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  // harvest every pending pair (call after a stream synchronisation)
  void flush() {
    std::lock_guard<std::mutex> g(mu);
    for (auto &p : pending) {
      float t = 0.f;
      if (cudaEventSynchronize(p.b) == cudaSuccess && cudaEventElapsedTime(&t, p.a, p.b) == cudaSuccess) {
        ms[p.stage] += t;
        if (on == 1 && log.size() < kLogMax) log.push_back({p.stage, p.elems, (double)t});
      }
      pool.push_back(p.a);
      pool.push_back(p.b);
    }
    pending.clear();
  }
};

Profiler &profiler();

inline bool debug_sync() {
  static const bool on = [] {
    const char *v = getenv("HUSKY_DEBUG_SYNC");
    return v && v[0] == '1';
  }();
  return on;
}

struct Scope {
  int stage;
  cudaStream_t s;
  uint64_t elems;
  cudaEvent_t a = nullptr;
  Scope(int st, cudaStream_t str, uint64_t m) : stage(st), s(str), elems(m) {
    Profiler &P = profiler();
    std::lock_guard<std::mutex> g(P.mu);
    P.total_launches++;
    P.launches[stage]++;
    P.elems[stage] += m;
    if (P.on == 1) {
      a = P.get();
      cudaEventRecord(a, s);
    }
  }
  ~Scope() {
    if (debug_sync()) {  // HUSKY_DEBUG_SYNC=1: localise device faults per launch
      cudaError_t e = cudaStreamSynchronize(s);
      if (e == cudaSuccess) e = cudaGetLastError();
      if (e != cudaSuccess)
        fprintf(stderr, "[husky] device error after stage %d launch (%llu elems): %s\n", stage,
                (unsigned long long)elems, cudaGetErrorString(e));
    }
    if (!a) return;
    Profiler &P = profiler();
    std::lock_guard<std::mutex> g(P.mu);
    cudaEvent_t b = P.get();
    cudaEventRecord(b, s);
    P.pending.push_back({stage, a, b, elems});
  }
};

// Profiler mode 2: one event pair around a group of launches of one stage (e.g.
// all radix passes of a sort), so the timed region carries two event records
// per group instead of two per launch.  Adds the group's time to the stage.
struct GroupScope {
  int stage;
  cudaStream_t s;
  cudaEvent_t a = nullptr;
  GroupScope(int st, cudaStream_t str) : stage(st), s(str) {
    Profiler &P = profiler();
    std::lock_guard<std::mutex> g(P.mu);
    if (P.on == 2) {
      a = P.get();
      cudaEventRecord(a, s);
    }
  }
  ~GroupScope() {
    if (!a) return;
    Profiler &P = profiler();
    std::lock_guard<std::mutex> g(P.mu);
    cudaEvent_t b = P.get();
    cudaEventRecord(b, s);
    P.pending.push_back({stage, a, b, 0});
  }
};

#define HUSKY_CAT2(a, b) a##b
#define HUSKY_CAT(a, b) HUSKY_CAT2(a, b)
#define HUSKY_SCOPE(stage, stream, elems) ::husky::Scope HUSKY_CAT(husky_scope_, __COUNTER__)(stage, stream, elems)

}  // namespace husky
