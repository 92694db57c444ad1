// Live kernel timing for bench.py's roofline figure: when enabled, every GEMM
// launch is bracketed by CUDA events recorded on the stream it is launched on;
// collect() sums durations and the algorithmic FLOPs of the launches.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <utility>
#include <vector>

#include "../../include/adaptra.h"
#include "prof.h"
#include "util.h"

namespace adaptra {
namespace {
struct Rec {
  int kind;
  cudaEvent_t a, b;
  double flops, bytes;
};
std::mutex g_mu;
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool;
bool g_on = false;

cudaEvent_t take() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

bool prof_on() { return g_on; }

static std::atomic<long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
long long launch_count() { return g_launches.load(); }

void* prof_begin(cudaStream_t st) {
  std::lock_guard<std::mutex> lk(g_mu);
  cudaEvent_t e = take();
  cudaEventRecord(e, st);
  return e;
}

void prof_end(void* begin, cudaStream_t st, int kind, double flops, double bytes) {
  std::lock_guard<std::mutex> lk(g_mu);
  cudaEvent_t e = take();
  cudaEventRecord(e, st);
  g_recs.push_back(Rec{kind, (cudaEvent_t)begin, e, flops, bytes});
}
}  // namespace adaptra

using namespace adaptra;

extern "C" int64_t adaptra_launch_count(void) { return (int64_t)launch_count(); }

extern "C" int adaptra_prof_enable(int32_t on) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_on = on != 0;
  return ADAPTRA_OK;
}

extern "C" int adaptra_prof_collect(int32_t kind, int64_t* n_launches, double* sum_ms, double* flops,
                                    double* bytes) {
  std::lock_guard<std::mutex> lk(g_mu);
  int64_t n = 0;
  double ms = 0, fl = 0, by = 0;
  std::vector<Rec> keep;
  for (auto& r : g_recs) {
    if (r.kind != kind) {
      keep.push_back(r);
      continue;
    }
    cudaEventSynchronize(r.b);
    float t = 0.f;
    if (cudaEventElapsedTime(&t, r.a, r.b) == cudaSuccess) {
      ms += t;
      fl += r.flops;
      by += r.bytes;
      n++;
    }
    g_pool.push_back(r.a);
    g_pool.push_back(r.b);
  }
  g_recs.swap(keep);
  cudaGetLastError();
  if (n_launches) *n_launches = n;
  if (sum_ms) *sum_ms = ms;
  if (flops) *flops = fl;
  if (bytes) *bytes = by;
  return ADAPTRA_OK;
}

extern "C" int adaptra_prof_collect_ex(int32_t kind, int64_t* n_launches, double* sum_ms, double* union_ms,
                                       double* flops, double* bytes) {
  std::lock_guard<std::mutex> lk(g_mu);
  int64_t n = 0;
  double ms = 0, fl = 0, by = 0;
  std::vector<Rec> keep;
  std::vector<std::pair<float, float>> iv;
  cudaEvent_t base = nullptr;
  for (auto& r : g_recs) {
    if (r.kind != kind) {
      keep.push_back(r);
      continue;
    }
    cudaEventSynchronize(r.b);
    if (!base) base = r.a;
    float t = 0.f, t0 = 0.f, t1 = 0.f;
    if (cudaEventElapsedTime(&t, r.a, r.b) == cudaSuccess && cudaEventElapsedTime(&t0, base, r.a) == cudaSuccess &&
        cudaEventElapsedTime(&t1, base, r.b) == cudaSuccess) {
      ms += t;
      fl += r.flops;
      by += r.bytes;
      iv.emplace_back(t0, t1);
      n++;
    }
  }
  // union of the launch intervals (every stream of this device shares the base event's clock)
  std::sort(iv.begin(), iv.end());
  double u = 0;
  float cs = 0.f, ce = 0.f;
  bool open = false;
  for (auto& p : iv) {
    if (!open || p.first > ce) {
      if (open) u += ce - cs;
      cs = p.first;
      ce = p.second;
      open = true;
    } else {
      ce = std::max(ce, p.second);
    }
  }
  if (open) u += ce - cs;
  for (auto& r : g_recs) {
    if (r.kind == kind) {
      g_pool.push_back(r.a);
      g_pool.push_back(r.b);
    }
  }
  g_recs.swap(keep);
  cudaGetLastError();
  if (n_launches) *n_launches = n;
  if (sum_ms) *sum_ms = ms;
  if (union_ms) *union_ms = u;
  if (flops) *flops = fl;
  if (bytes) *bytes = by;
  return ADAPTRA_OK;
}
