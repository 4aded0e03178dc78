// Runtime plumbing of libfm_gpu.so: stream selection, error mapping, the
// launch counter and the constant-memory filter banks.
#include <atomic>
#include <cstdio>
#include <cstring>

#include "fm_device.cuh"
#include "fm_internal.hpp"

namespace fmh {

namespace {
std::atomic<int64_t> g_launches{0};
thread_local cudaStream_t g_stream = nullptr;
thread_local int g_banks_device = -1;
}  // namespace

void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e == cudaSuccess) return;
  char buf[512];
  std::snprintf(buf, sizeof(buf), "CUDA error %s (%s) in %s at %s:%d", cudaGetErrorName(e),
                cudaGetErrorString(e), what, file, line);
  throw Error(FM_ERR_CUDA, buf);
}

void count_launch(const char* file, int line) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) cuda_check(e, "kernel launch", file, line);
}

int64_t launches() { return g_launches.load(); }
void count_graph_launches(int64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// The library's own non-blocking stream (one per thread and device) unless the
// caller routed work onto theirs with fm_set_stream.  A non-default stream is
// required for CUDA-graph capture of the step loop.
cudaStream_t stream() {
  static thread_local cudaStream_t own[64] = {};
  if (g_stream) return g_stream;
  int dev = 0;
  FM_CUDA(cudaGetDevice(&dev));
  if (!own[dev]) {
    FM_CUDA(cudaStreamCreateWithFlags(&own[dev], cudaStreamNonBlocking));
    // keep freed blocks in the stream-ordered pool: the pyramids of repeated
    // MRA / adapt passes are re-allocated without new page mappings
    cudaMemPool_t pool;
    FM_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t keep = UINT64_MAX;
    FM_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  }
  return own[dev];
}
void set_stream(cudaStream_t s) { g_stream = s; }

double elapsed_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  FM_CUDA(cudaEventElapsedTime(&ms, a, b));
  return double(ms);
}

const char* kernel_family_name(int f) {
  static const char* names[KF_COUNT] = {"k_head_friction", "k_stage<1>",     "k_stage<2>",
                                        "k_commit",        "k_acc_faces",    "k_acc_leaves",
                                        "k_uni_head",      "k_uni_stage<1>", "k_uni_stage<2>",
                                        "k_seg<1>",        "k_seg<2>",       "k_decide"};
  return f >= 0 && f < KF_COUNT ? names[f] : "?";
}

KTimer& ktimer() {
  static thread_local KTimer t;
  return t;
}
void kt_begin(int fam) {
  KTimer& t = ktimer();
  if (!t.on) return;
  cudaEvent_t e;
  FM_CUDA(cudaEventCreate(&e));
  FM_CUDA(cudaEventRecord(e, stream()));
  t.fam.push_back(fam);
  t.a.push_back(e);
}
void kt_end() {
  KTimer& t = ktimer();
  if (!t.on) return;
  cudaEvent_t e;
  FM_CUDA(cudaEventCreate(&e));
  FM_CUDA(cudaEventRecord(e, stream()));
  t.b.push_back(e);
}

// The filter banks are compile-time constants (fmd::tap); nothing to upload.
void upload_banks() {}

}  // namespace fmh
