// prof.h — per-kernel live profile of the PISO step (the
// "kernels" table of bench.py; north star: "achieved HBM GB/s reported
// against B200 peak for every kernel").
//
// In profile mode every kernel launch of the step is followed by a CUDA
// event on the launching stream and tagged with its kernel name, AMG level
// and algorithmic bytes; a launch's time is the interval from
// the previous launch's event (or, at the start of a sequence, a fresh start
// event) to its own, so the rows add up to the profiled time of the
// sequences and each kernel carries its own launch gap (what a launch costs
// the step, the point in the latency-bound AMG levels).  Krylov kernels also carry their
// iteration index within the enqueued chunk; after the chunk's control-block
// read-back the harvest attributes the launches of iterations the device
// skipped (solve already converged: the kernel exits on the done flag) to a
// separate "no-op" row with zero bytes, so GB/s is computed over launches
// that did the work.  Chunks with small (AMG coarse-level) kernels are
// captured into a CUDA graph and replayed, so a host slower than the GPU
// never opens a gap inside an event pair.
#pragma once
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

#include "dev.cuh"

namespace dfvm {

struct Prof {
  struct Stat { const char* name; int lvl; int64_t n; double ms, bytes; };
  struct Rec { int stat; double bytes; int iter, post; cudaEvent_t a, b; };
  bool on = false;
  std::vector<Stat> stats;
  std::vector<Rec> recs;             // enqueued, not yet harvested
  std::vector<cudaEvent_t> pool;
  int iter = -1;                     // Krylov iteration within the current chunk (-1: not iterative)
  int post = 0;                      // 1: launched after the iteration's convergence check
  cudaEvent_t last = nullptr;        // the previous launch's end event in the current sequence

  ~Prof() {
    for (auto e : pool) cudaEventDestroy(e);
    for (auto& r : recs) cudaEventDestroy(r.b);
    for (auto e : starts) cudaEventDestroy(e);
  }
  // a new sequence (host synchronisation, start / end of a graph capture):
  // the next launch starts from a fresh event
  void cut() { last = nullptr; }
  void clear() {
    last = nullptr;
    stats.clear();
    for (auto& r : recs) pool.push_back(r.b);
    for (auto e : starts) pool.push_back(e);
    starts.clear();
    recs.clear();
  }
  int stat_index(const char* name, int lvl) {
    for (size_t i = 0; i < stats.size(); ++i)
      if (stats[i].lvl == lvl && std::strcmp(stats[i].name, name) == 0) return (int)i;
    stats.push_back(Stat{name, lvl, 0, 0.0, 0.0});
    return (int)stats.size() - 1;
  }
  cudaEvent_t get() {
    if (!pool.empty()) { cudaEvent_t e = pool.back(); pool.pop_back(); return e; }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
  }
  cudaEvent_t begin(cudaStream_t s) {
    if (last) return last;
    cudaEvent_t a = get();
    record_event(a, s);
    starts.push_back(a);
    return a;
  }
  void end(cudaEvent_t a, const char* name, int lvl, double bytes, cudaStream_t s) {
    cudaEvent_t b = get();
    record_event(b, s);
    recs.push_back(Rec{stat_index(name, lvl), bytes, iter, post, a, b});
    last = b;
  }
  std::vector<cudaEvent_t> starts;   // fresh start events of the sequences (returned at harvest)
  // after the stream has synchronised: `ran` iterations of the chunk did
  // work, the last one stopped after its check when `done_last`
  void harvest(int ran = 1 << 30, bool done_last = false) {
    for (auto& r : recs) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, r.a, r.b);
      const bool noop = r.iter >= 0 && (r.iter >= ran || (r.post && done_last && r.iter == ran - 1));
      Stat& st = stats[noop ? stat_index("(no-op launches after convergence)", -1) : r.stat];
      st.n++;
      st.ms += ms;
      if (!noop) st.bytes += r.bytes;
      pool.push_back(r.b);            // every event is some record's end, or a sequence start
    }
    for (auto e : starts) pool.push_back(e);
    starts.clear();
    recs.clear();
    last = nullptr;
    cudaGetLastError();
  }
};

// launch bracketed by profile events (no-op when P is null or off)
#define PLAUNCH(P, NAME, LVL, BYTES, S, ...)                                      \
  do {                                                                            \
    ::dfvm::Prof* p_ = (P);                                                       \
    cudaEvent_t pa_ = (p_ && p_->on) ? p_->begin(S) : nullptr;                   \
    __VA_ARGS__;                                                                  \
    if (pa_) p_->end(pa_, NAME, LVL, (double)(BYTES), S);                         \
  } while (0)

}  // namespace dfvm
