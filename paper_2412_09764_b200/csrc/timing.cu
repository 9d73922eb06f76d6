// Optional per-launch timing with CUDA events recorded on the launch stream.
// When enabled (ml_timing_enable(1)), every kernel launch, cuBLASLt GEMM and
// memset of the library records an event after it; API entry points record a
// start marker.  A launch's duration is the time between its event and the
// previous event on the same stream (kernels on one stream serialise), which
// bench.py aggregates per kernel name over the timed region.
#include "internal.cuh"

#include <map>
#include <mutex>
#include <vector>

namespace ml {
namespace {
struct Mark {
  const char* name;
  cudaEvent_t ev;
  cudaStream_t s;
};
std::mutex g_mu;
bool g_on = false;
std::vector<Mark> g_marks;
std::vector<cudaEvent_t> g_pool;
size_t g_pool_used = 0;
}  // namespace

void timing_mark(const char* name, cudaStream_t s) {
  if (!g_on) return;
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_pool_used == g_pool.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    g_pool.push_back(e);
  }
  cudaEvent_t e = g_pool[g_pool_used++];
  cudaEventRecord(e, s);
  g_marks.push_back({name, e, s});
}

}  // namespace ml

using namespace ml;

extern "C" {

void ml_timing_enable(int on) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_on = on != 0;
}

void ml_timing_reset(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_marks.clear();
  g_pool_used = 0;
}

// Writes "name count total_ms\n" lines (aggregated over all recorded
// launches) into buf; returns the number of bytes needed (incl. NUL).
size_t ml_timing_report(char* buf, size_t len) {
  std::lock_guard<std::mutex> lk(g_mu);
  std::map<std::string, std::pair<long, double>> agg;
  std::map<cudaStream_t, cudaEvent_t> last;
  for (const Mark& m : g_marks) {
    auto it = last.find(m.s);
    if (m.name && it != last.end()) {
      cudaEventSynchronize(m.ev);
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, it->second, m.ev) == cudaSuccess) {
        auto& a = agg[m.name];
        a.first += 1;
        a.second += ms;
      }
    }
    last[m.s] = m.ev;
  }
  std::string out;
  char line[256];
  for (auto& kv : agg) {
    snprintf(line, sizeof(line), "%s %ld %.6f\n", kv.first.c_str(), kv.second.first, kv.second.second);
    out += line;
  }
  if (buf && len) {
    size_t n = out.size() < len - 1 ? out.size() : len - 1;
    memcpy(buf, out.data(), n);
    buf[n] = 0;
  }
  return out.size() + 1;
}

}  // extern "C"
