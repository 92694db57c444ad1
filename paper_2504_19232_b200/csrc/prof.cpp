// Live kernel timing for bench.py's roofline figure: when enabled, every GEMM
// launch is bracketed by CUDA events recorded on the stream it is launched on;
// collect() sums durations and the algorithmic FLOPs of the launches.
#include <cuda_runtime.h>

#include <atomic>
#include <mutex>
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
