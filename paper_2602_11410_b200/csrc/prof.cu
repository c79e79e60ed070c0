#include <atomic>
#include <mutex>
#include <vector>

#include "../../include/cadet.h"
#include "prof.cuh"

namespace cadet {
namespace {
std::atomic<long long> g_launches{0};
std::mutex g_mu;
int g_classes = 0;
int g_max = 0;
std::vector<cudaEvent_t> g_ev;   // 2 per pair
std::vector<int> g_cls;
int g_used = 0;
}  // namespace

void note_launches(int n) { g_launches += n; }

// Inside stream capture a plain cudaEventRecord only adds a capture dependency; an external
// event-record node is needed for the event to be re-recorded by every graph replay.
static void record(cudaEvent_t ev, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  if (cs == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal);
  else
    cudaEventRecord(ev, st);
}

int prof_begin(int cls, cudaStream_t st) {
  if (!g_classes) return -1;
  std::lock_guard<std::mutex> lk(g_mu);
  if (!(g_classes & (1 << cls)) || g_used >= g_max) return -1;
  const int slot = g_used++;
  g_cls[slot] = cls;
  record(g_ev[2 * slot], st);
  return slot;
}

void prof_end(int slot, cudaStream_t st) {
  if (slot < 0) return;
  record(g_ev[2 * slot + 1], st);
}
}  // namespace cadet

using namespace cadet;

extern "C" {
int64_t cadet_launch_count(void) { return g_launches.load(); }

cadet_status cadet_prof_enable(int32_t classes, int32_t max_pairs) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (max_pairs < 0) return CADET_E_ARG;
  if ((int)g_ev.size() < 2 * max_pairs) {
    const size_t old = g_ev.size();
    g_ev.resize(2 * (size_t)max_pairs);
    for (size_t i = old; i < g_ev.size(); ++i)
      if (cudaEventCreate(&g_ev[i]) != cudaSuccess) return CADET_E_CUDA;
    g_cls.resize(max_pairs);
  }
  g_max = max_pairs;
  g_used = 0;
  g_classes = classes;
  return CADET_OK;
}

cadet_status cadet_prof_read(double* ms, int64_t* launches) {
  std::lock_guard<std::mutex> lk(g_mu);
  for (int c = 0; c < 4; ++c) {
    if (ms) ms[c] = 0.0;
    if (launches) launches[c] = 0;
  }
  for (int i = 0; i < g_used; ++i) {
    if (cudaEventSynchronize(g_ev[2 * i + 1]) != cudaSuccess) return CADET_E_CUDA;
    float t = 0.f;
    cudaEventElapsedTime(&t, g_ev[2 * i], g_ev[2 * i + 1]);
    if (ms) ms[g_cls[i]] += t;
    if (launches) launches[g_cls[i]] += 1;
  }
  g_classes = 0;
  g_used = 0;
  return CADET_OK;
}
}
