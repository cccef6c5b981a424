// profile.cu — optional per-kernel CUDA-event timing (bench.py's roofline).
// Disabled by default; when enabled every launch of a kernel class is
// bracketed by events on its own stream, so the kernel's duration is measured
// where it runs, without a profiler.
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "kernels.h"

namespace sparcml {

namespace {
struct Rec {
  cudaEvent_t a, b;
};
std::mutex g_mu;
bool g_on = false;
std::string g_only;   // empty: every kernel class
std::map<std::string, std::vector<Rec>> g_recs;
std::vector<cudaEvent_t> g_pool;

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

ProfScope::ProfScope(const char* name, cudaStream_t s) : name_(name), s_(s), a_(nullptr) {
  if (!g_on) return;
  std::lock_guard<std::mutex> l(g_mu);
  if (!g_only.empty() && g_only != name) return;
  a_ = take();
  cudaEventRecord(static_cast<cudaEvent_t>(a_), s_);
}

ProfScope::~ProfScope() {
  if (!a_) return;
  std::lock_guard<std::mutex> l(g_mu);
  cudaEvent_t b = take();
  cudaEventRecord(b, s_);
  g_recs[name_].push_back(Rec{static_cast<cudaEvent_t>(a_), b});
}

}  // namespace sparcml

using namespace sparcml;

extern "C" {

void sparcml_profile_enable(int on) {
  std::lock_guard<std::mutex> l(g_mu);
  g_on = on != 0;
}

void sparcml_profile_only(const char* name) {
  std::lock_guard<std::mutex> l(g_mu);
  g_only = name ? name : "";
}

void sparcml_profile_reset(void) {
  std::lock_guard<std::mutex> l(g_mu);
  for (auto& kv : g_recs)
    for (auto& r : kv.second) {
      g_pool.push_back(r.a);
      g_pool.push_back(r.b);
    }
  g_recs.clear();
}

sparcml_status sparcml_profile_read(const char* name, uint64_t* launches, double* total_ms) {
  if (!name || !launches || !total_ms) return SPARCML_ERR_INVALID_ARG;
  std::lock_guard<std::mutex> l(g_mu);
  *launches = 0;
  *total_ms = 0.0;
  auto it = g_recs.find(name);
  if (it == g_recs.end()) return SPARCML_OK;
  for (auto& r : it->second) {
    if (cudaEventSynchronize(r.b) != cudaSuccess) return SPARCML_ERR_CUDA;
    float ms = 0.0f;
    if (cudaEventElapsedTime(&ms, r.a, r.b) != cudaSuccess) return SPARCML_ERR_CUDA;
    *total_ms += ms;
    ++*launches;
  }
  return SPARCML_OK;
}

}  // extern "C"
