// Host-side internals of libfm_gpu.so: device buffers, error plumbing and
// the grid / sim objects behind the opaque C handles of include/fm_gpu.h.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/fm_gpu.h"

#include <nvtx3/nvToolsExt.h>

namespace fmh {

struct NvtxRange {
  explicit NvtxRange(const char* n) { nvtxRangePushA(n); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};


struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void cuda_check(cudaError_t e, const char* what, const char* file, int line);
#define FM_CUDA(x) ::fmh::cuda_check((x), #x, __FILE__, __LINE__)
#define FM_LAUNCHED() ::fmh::count_launch(__FILE__, __LINE__)
// NVTX ranges around the library's phases (no-ops unless a profiler such as
// Nsight Systems attaches; header-only NVTX v3 from the CUDA toolkit)
#define FM_RANGE(name) ::fmh::NvtxRange fm_nvtx_range_(name)
void count_launch(const char* file, int line);
int64_t launches();
void count_graph_launches(int64_t n);  // kernels replayed by a graph launch

cudaStream_t stream();
void set_stream(cudaStream_t s);
void upload_banks();  // fills fmd::c_bank once per device

// Device allocation (stream-ordered pool; FM_PLAIN_MALLOC: cudaMalloc).
// FM_GUARD=1 in the environment: every allocation carries guard bands of a
// known byte pattern before and after it, checked on the device when it is
// freed and for every live allocation by fm_debug_guard_report: an
// out-of-bounds write past either end of a buffer is counted (runtime.cu).
void* dev_alloc(size_t bytes);
void dev_free(void* p, size_t bytes);
void guard_report(int64_t* checked, int64_t* overruns);
bool guard_enabled();

// Owning device buffer.
template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  size_t cap = 0;  // elements allocated (>= n)
  DBuf() = default;
  explicit DBuf(size_t count) { alloc(count); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), cap(o.cap) {
    o.p = nullptr;
    o.n = 0;
    o.cap = 0;
  }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      n = o.n;
      cap = o.cap;
      o.p = nullptr;
      o.n = 0;
      o.cap = 0;
    }
    return *this;
  }
  ~DBuf() { release(); }
  // Logical size `count`, keeping the allocation when it holds count
  // elements (re-gridded sims: no free / malloc per adapt); grows by 1/4.
  void ensure(size_t count) {
    if (p && count <= cap) {
      n = count;
      return;
    }
    const size_t c = count + count / 4;
    alloc(c);
    n = count;
  }
  void alloc(size_t count) {
    if (count == n && p) return;
    release();
    n = count;
    cap = count;
    if (count) p = static_cast<T*>(dev_alloc(count * sizeof(T)));
  }
  void release() {
    if (p) dev_free(p, cap * sizeof(T));
    p = nullptr;
    n = 0;
    cap = 0;
  }
  void zero() {
    if (n) FM_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), stream()));
  }
  void fill_bytes(int v) {
    if (n) FM_CUDA(cudaMemsetAsync(p, v, n * sizeof(T), stream()));
  }
  void upload(const T* h, size_t count) {
    alloc(count);
    if (count)
      FM_CUDA(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, stream()));
  }
  void download(T* h, size_t count) const {
    if (count)
      FM_CUDA(cudaMemcpyAsync(h, p, count * sizeof(T), cudaMemcpyDeviceToHost, stream()));
  }
  std::vector<T> to_host() const {
    std::vector<T> v(n);
    download(v.data(), n);
    FM_CUDA(cudaStreamSynchronize(stream()));
    return v;
  }
};

// Device-resident static MRA result (the NonUniformGrid of quadgrid.hpp:117-120
// plus the DetailTree of detail_tree.hpp:13-30), in block-Morton layout.
struct Grid {
  int L = 0, M = 1, N = 1, kind = 0;
  double R = 1, x0 = 0, y0 = 0, eps = 0, field_norm = 0;
  bool graded = true;
  // the topography may hold |z| > 1e300 (or came from a leaf list): its decode
  // keeps every filter tap (dkind)
  bool big = true;
  int dkind() const { return kind | (big ? 0 : 2); }
  // deferred significance (mra_encode's defer_sig): max |d| per node of the
  // levels > sig_done, d_hat = max|d| / sig_den >= eps taken by the grading
  std::vector<DBuf<double>> dmx;
  int sig_done = -1;
  double sig_den = 1.0;
  int64_t nleaves = 0;
  std::vector<DBuf<double>> det;   // [L] x 9 doubles per node
  std::vector<DBuf<uint8_t>> flag; // [L] final (closed, graded) flags
  std::vector<DBuf<int32_t>> cnt;  // [L] leaf count of each node's subtree
  std::vector<DBuf<int32_t>> off;  // [L] first leaf index of each active node
  DBuf<double> coarse;             // M*N x 3: level-0 scaling
  // leaves in device (Morton) order
  DBuf<int8_t> lf_l;
  DBuf<int32_t> lf_i, lf_j;
  DBuf<double> lf_z;  // 3 per leaf
  std::vector<DBuf<double>> zs;  // build_leaves' decoded-plane scratch per level
  double mra_ms = 0, mra_bytes = 0;
  uint64_t nodes(int l) const { return uint64_t(M) * N << (2 * l); }
};

Grid* mra_static(const fm_raster* dem, int L, double eps, bool graded, int kind);
// A grid from a leaf list + topography (read_nug / make_quadgrid), static sims only.
Grid* grid_from_leaves(int L, int M, int N, double R, double x0, double y0, int64_t n, const int32_t* lv,
                       const int32_t* li, const int32_t* lj, const double* topo3);
// The stages of mra_static, reused by the adaptive solver.
// defer_sig: leave the significance of the levels with more than 256 nodes
// to the grading pass, which forms it from the encode's max |d| (g.dmx)
void mra_encode(const fm_raster* dem, int L, double eps, int kind, Grid& g, double* ms, bool defer_sig = false);
// ring (optional, per level): take each node's own flag as the same-level
// 8-neighbour dilation of ring[l] (buffer_ring) instead of g.flag[l]
void grade_count_levels(Grid& g, bool graded, const std::vector<const uint8_t*>* ring = nullptr);
// Shared by the static and the adaptive pipelines: from final per-level flags
// (already in g.flag) compute counts, offsets, then decode topography details
// top-down into the leaf arrays.  Returns the leaf count.
int64_t build_leaves(Grid& g);
void build_leaves_device(Grid& g, long long* total);
// grade_count_levels(g, true, ring) then build_leaves_device(g, total), the
// small levels of both in one launch (the adapt's prefix)
void grade_and_build_leaves_device(Grid& g, const std::vector<const uint8_t*>* ring, long long* total);
// Permutation device-order -> reference (level, j, i) order, computed on the host.
std::vector<int64_t> reference_order(const Grid& g, std::vector<int8_t>* l = nullptr,
                                     std::vector<int32_t>* i = nullptr,
                                     std::vector<int32_t>* j = nullptr);

double elapsed_ms(cudaEvent_t a, cudaEvent_t b);

// A pair of timing events, destroyed on every exit path.
struct EventPair {
  cudaEvent_t a = nullptr, b = nullptr;
  EventPair() {
    FM_CUDA(cudaEventCreate(&a));
    FM_CUDA(cudaEventCreate(&b));
  }
  EventPair(const EventPair&) = delete;
  EventPair& operator=(const EventPair&) = delete;
  ~EventPair() {
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
  }
  double ms() const { return elapsed_ms(a, b); }
};

// Launch helper for the step chain (a plain launch + error check).
template <typename... KArgs, typename... Args>
void launch_k(void (*k)(KArgs...), dim3 grid, dim3 block, cudaStream_t st, Args... args) {
  k<<<grid, block, 0, st>>>(static_cast<KArgs>(args)...);
  FM_CUDA(cudaGetLastError());
}

// Optional per-launch timing for fm_sim_profile: when on, every kernel launch
// of a step is bracketed by CUDA events on the library stream.
enum KernelFamily {
  KF_HEAD = 0,    // step head + friction (DG2/FV1)
  KF_STAGE1,      // RK stage 1 (FV1: the whole update)
  KF_STAGE2,      // RK stage 2 + fused epilogue
  KF_COMMIT,      // (unused: the clock needs no commit kernel)
  KF_ACC_FACES,   // ACC face discharges + step head
  KF_ACC_LEAVES,  // ACC leaf update + fused epilogue
  KF_UNI_HEAD,    // uniform raster: head + friction
  KF_UNI_STAGE1,  // uniform raster: stage 1
  KF_UNI_STAGE2,  // uniform raster: stage 2
  KF_SEG1,        // segment states, stage 1
  KF_SEG2,        // segment states, stage 2
  KF_DECIDE,      // the one-thread step decision
  KF_COUNT
};
const char* kernel_family_name(int f);
struct KTimer {
  bool on = false;
  std::vector<int> fam;
  std::vector<cudaEvent_t> a, b;
};
KTimer& ktimer();
void kt_begin(int fam);
void kt_end();

// ancestor_closure + grade_flags on host flags (levels back to back, row-major).
void grade_flags_host(int L, int M, int N, bool graded, uint8_t* flags);

// Level-L planes (3 per node, block-Morton order) of a vertex raster, padded
// and nodata-walled as project_raster does (field.cpp:64-117).
void project_planes(const fm_raster* r, int L, int M, int N, DBuf<double>& out);
// Parent scaling of every level l = L-1..0 from the level-L planes
// (encode rows 0-2, wavelets.cpp:77-86); sc[l] holds 3 doubles per node.
void scaling_pyramid(DBuf<double>&& level_L, int L, int M, int N, int kind,
                     std::vector<DBuf<double>>& sc);

}  // namespace fmh
