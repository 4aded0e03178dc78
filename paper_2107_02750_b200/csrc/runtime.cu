// Runtime plumbing of libfm_gpu.so: stream selection, error mapping, the
// launch counter and the constant-memory filter banks.
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>

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
                                        "k_uni_head",      "k_uni_march<1>", "k_uni_march<2>",
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

// ---- device allocations and the FM_GUARD checker --------------------------
namespace {
constexpr size_t kGuard = 256;  // bytes of pattern before and after (keeps 256 B alignment)
constexpr unsigned char kGuardByte = 0xA5;
bool guard_on() {
  static const bool on = [] {
    const char* e = std::getenv("FM_GUARD");
    return e && e[0] == '1';
  }();
  return on;
}
struct GuardReg {
  std::mutex mu;
  std::unordered_map<void*, size_t> live;  // user pointer -> user bytes
  unsigned long long* bad = nullptr;       // device: overrun count
  int64_t checked = 0;
};
GuardReg& guard_reg() {
  static GuardReg* r = new GuardReg();  // never destroyed (frees may run at exit)
  return *r;
}
__global__ void k_guard_check(const unsigned char* base, size_t bytes, unsigned long long* bad) {
  // the band before (base .. base + kGuard) and after (base + kGuard + bytes ..);
  // one count per damaged buffer
  int hit = 0;
  for (size_t q = threadIdx.x; q < 2 * kGuard; q += blockDim.x) {
    const size_t at = q < kGuard ? q : kGuard + bytes + (q - kGuard);
    hit |= base[at] != kGuardByte;
  }
  if (__syncthreads_or(hit) && threadIdx.x == 0) atomicAdd(bad, 1ull);
}
void guard_check_async(void* user, size_t bytes) {
  GuardReg& r = guard_reg();
  k_guard_check<<<1, 128, 0, stream()>>>(static_cast<unsigned char*>(user) - kGuard, bytes, r.bad);
  r.checked += 1;
}
void* raw_alloc(size_t bytes) {
  void* p = nullptr;
#ifdef FM_PLAIN_MALLOC
  FM_CUDA(cudaStreamSynchronize(stream()));
  FM_CUDA(cudaMalloc(&p, bytes));
#else
  FM_CUDA(cudaMallocAsync(&p, bytes, stream()));
#endif
  return p;
}
void raw_free(void* p) {
#ifdef FM_PLAIN_MALLOC
  cudaStreamSynchronize(stream());
  cudaFree(p);
#else
  cudaFreeAsync(p, stream());
#endif
}
}  // namespace

void* dev_alloc(size_t bytes) {
  if (!guard_on()) return raw_alloc(bytes);
  GuardReg& r = guard_reg();
  std::lock_guard<std::mutex> lk(r.mu);
  if (!r.bad) {
    FM_CUDA(cudaMalloc(&r.bad, sizeof(unsigned long long)));
    FM_CUDA(cudaMemset(r.bad, 0, sizeof(unsigned long long)));
  }
  unsigned char* base = static_cast<unsigned char*>(raw_alloc(bytes + 2 * kGuard));
  FM_CUDA(cudaMemsetAsync(base, kGuardByte, kGuard, stream()));
  FM_CUDA(cudaMemsetAsync(base + kGuard + bytes, kGuardByte, kGuard, stream()));
  r.live[base + kGuard] = bytes;
  return base + kGuard;
}

void dev_free(void* p, size_t bytes) {
  if (!p) return;
  if (!guard_on()) {
    raw_free(p);
    return;
  }
  GuardReg& r = guard_reg();
  std::lock_guard<std::mutex> lk(r.mu);
  auto it = r.live.find(p);
  if (it != r.live.end()) {
    bytes = it->second;
    r.live.erase(it);
  }
  guard_check_async(p, bytes);
  raw_free(static_cast<unsigned char*>(p) - kGuard);
}

bool guard_enabled() { return guard_on(); }

// Checks every live allocation's bands and reports the totals (checks done
// so far, overruns found); no-op counts when FM_GUARD is off.
void guard_report(int64_t* checked, int64_t* overruns) {
  int64_t c = 0, o = 0;
  if (guard_on()) {
    GuardReg& r = guard_reg();
    std::lock_guard<std::mutex> lk(r.mu);
    for (const auto& kv : r.live) guard_check_async(kv.first, kv.second);
    unsigned long long h = 0;
    if (r.bad) {
      FM_CUDA(cudaMemcpyAsync(&h, r.bad, sizeof(h), cudaMemcpyDeviceToHost, stream()));
      FM_CUDA(cudaStreamSynchronize(stream()));
    }
    c = r.checked;
    o = int64_t(h);
  }
  if (checked) *checked = c;
  if (overruns) *overruns = o;
}

// The filter banks are compile-time constants (fmd::tap); nothing to upload.
void upload_banks() {}

}  // namespace fmh
