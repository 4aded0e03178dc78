// The reference leaf order on the device.
//
// The reference stores leaves sorted by (level, j, i) (make_quadgrid,
// quadgrid.cpp:94-98); the device keeps them in Morton order.  Host-facing
// downloads/uploads permute between the two.  Sorting 2.3 M leaves and
// scattering 200 MB of state on the host cost ~0.4 s per download for
// config 4; here the leaf keys (level << 58 | j << 29 | i, the reference's
// own leaf_key layout) are radix-sorted on the device once per leaf set, and
// every transfer is a device gather/scatter plus one contiguous copy (into
// page-locked host memory the gather writes the host rows directly).
#include <cub/device/device_radix_sort.cuh>

#include "fm_device.cuh"
#include "fm_sim.hpp"

namespace fmh {

namespace {

inline unsigned nblk(uint64_t n, int t) { return unsigned((n + t - 1) / t); }

__global__ void k_keys(int64_t n, const int8_t* __restrict__ lvl, const int32_t* __restrict__ li,
                       const int32_t* __restrict__ lj, unsigned long long* __restrict__ key,
                       int32_t* __restrict__ idx) {
  const int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (k >= n) return;
  key[k] = (static_cast<unsigned long long>(lvl[k]) << 58) |
           (static_cast<unsigned long long>(lj[k]) << 29) | static_cast<unsigned long long>(li[k]);
  idx[k] = int32_t(k);
}

// dst[r] = src[perm[r]] for rows of `width` elements
template <typename T>
__global__ void k_gather(int64_t n, int width, const int32_t* __restrict__ perm, const T* __restrict__ src,
                         T* __restrict__ dst) {
  const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (t >= n * width) return;
  const int64_t r = t / width, q = t % width;
  dst[t] = src[int64_t(perm[r]) * width + q];
}

// dst[perm[r]] = src[r]
template <typename T>
__global__ void k_scatter(int64_t n, int width, const int32_t* __restrict__ perm, const T* __restrict__ src,
                          T* __restrict__ dst) {
  const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (t >= n * width) return;
  const int64_t r = t / width, q = t % width;
  dst[int64_t(perm[r]) * width + q] = src[t];
}

// dst[r] = src[perm[r] * stride + col]
__global__ void k_gather_col(int64_t n, int stride, int col, const int32_t* __restrict__ perm,
                             const double* __restrict__ src, double* __restrict__ dst) {
  const int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (r < n) dst[r] = src[int64_t(perm ? perm[r] : r) * stride + col];
}

__global__ void k_widen(int64_t n, const int32_t* __restrict__ perm, const int8_t* __restrict__ lvl,
                        int32_t* __restrict__ out) {
  const int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (r < n) out[r] = lvl[perm[r]];
}

// The device view of a page-locked host buffer (cudaHostAlloc / registered,
// mapped under unified addressing), or nullptr for pageable memory.  A gather
// into such a buffer writes the host rows straight over PCIe: no staging
// buffer to allocate and no separate copy.
template <typename T>
T* mapped_host(T* host) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, host) != cudaSuccess) {
    (void)cudaGetLastError();
    return nullptr;
  }
  return a.type == cudaMemoryTypeHost ? static_cast<T*>(a.devicePointer) : nullptr;
}

// Device scratch a caller lends to the gathers (the sim's idle U* buffer),
// so a download to pageable memory needs no allocation.
struct Stage {
  void* p = nullptr;
  size_t bytes = 0;
};
thread_local Stage g_stage;

template <typename T>
T* staging(size_t count) {
  return g_stage.p && count * sizeof(T) <= g_stage.bytes ? static_cast<T*>(g_stage.p) : nullptr;
}

}  // namespace

StageScope::StageScope(void* p, size_t bytes) { g_stage = Stage{p, bytes}; }
StageScope::~StageScope() { g_stage = Stage{}; }

// Runs every kernel of this file once on two elements, so their module is
// loaded at fm_init and not (lazily, with a variable cost measured up to
// 0.1-0.3 s on B200 boxes) inside the first download or sim setup.
void order_preload() {
  cudaStream_t st = stream();
  const int64_t n = 2;
  DBuf<int8_t> lvl(n);
  DBuf<int32_t> li(n), lj(n), idx(n), perm(n), i32(n);
  DBuf<unsigned long long> k0(n), k1(n);
  DBuf<double> a(3 * n), b(3 * n);
  lvl.zero();
  li.zero();
  lj.zero();
  k_keys<<<1, 32, 0, st>>>(n, lvl.p, li.p, lj.p, k0.p, idx.p);
  size_t tmp_bytes = 0;
  FM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k0.p, k1.p, idx.p, perm.p, int(n), 0, 62, st));
  DBuf<unsigned char> tmp(std::max<size_t>(tmp_bytes, 1));
  FM_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, k0.p, k1.p, idx.p, perm.p, int(n), 0, 62, st));
  a.zero();
  k_gather<double><<<1, 32, 0, st>>>(n, 3, perm.p, a.p, b.p);
  k_scatter<double><<<1, 32, 0, st>>>(n, 3, perm.p, a.p, b.p);
  k_gather<int32_t><<<1, 32, 0, st>>>(n, 1, perm.p, li.p, i32.p);
  k_widen<<<1, 32, 0, st>>>(n, perm.p, lvl.p, i32.p);
  k_gather_col<<<1, 32, 0, st>>>(n, 3, 0, perm.p, a.p, b.p);
  FM_CUDA(cudaGetLastError());
  FM_CUDA(cudaStreamSynchronize(st));
}

const int32_t* sim_ref_perm(Sim& s) {
  if (s.uniform) return nullptr;  // j * nx + i is already the reference order
  if (s.ref_perm_ok && s.ref_perm.n == size_t(s.n)) return s.ref_perm.p;
  cudaStream_t st = stream();
  const int64_t n = s.n;
  DBuf<unsigned long long> k0(std::max<int64_t>(n, 1)), k1(std::max<int64_t>(n, 1));
  DBuf<int32_t> i0(std::max<int64_t>(n, 1));
  s.ref_perm.alloc(std::max<int64_t>(n, 1));
  k_keys<<<nblk(n, 256), 256, 0, st>>>(n, s.lvl.p, s.li.p, s.lj.p, k0.p, i0.p);
  FM_LAUNCHED();
  size_t tmp_bytes = 0;
  FM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k0.p, k1.p, i0.p, s.ref_perm.p, int(n), 0,
                                          62, st));
  DBuf<unsigned char> tmp(std::max<size_t>(tmp_bytes, 1));
  FM_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, k0.p, k1.p, i0.p, s.ref_perm.p, int(n), 0,
                                          62, st));
  FM_LAUNCHED();
  s.ref_perm_ok = true;
  return s.ref_perm.p;
}

void gather_rows(const int32_t* perm, int64_t n, int width, const double* src, double* host_dst) {
  cudaStream_t st = stream();
  if (!perm) {
    FM_CUDA(cudaMemcpyAsync(host_dst, src, size_t(n) * width * sizeof(double), cudaMemcpyDeviceToHost, st));
    return;
  }
  if (double* d = mapped_host(host_dst)) {
    k_gather<double><<<nblk(n * width, 256), 256, 0, st>>>(n, width, perm, src, d);
    FM_LAUNCHED();
    FM_CUDA(cudaStreamSynchronize(st));
    return;
  }
  DBuf<double> tmp;
  double* buf = staging<double>(size_t(n) * width);
  if (!buf) {
    tmp.alloc(std::max<int64_t>(n * width, 1));
    buf = tmp.p;
  }
  k_gather<double><<<nblk(n * width, 256), 256, 0, st>>>(n, width, perm, src, buf);
  FM_LAUNCHED();
  FM_CUDA(cudaMemcpyAsync(host_dst, buf, size_t(n) * width * sizeof(double), cudaMemcpyDeviceToHost, st));
  FM_CUDA(cudaStreamSynchronize(st));
}

void gather_i32(const int32_t* perm, int64_t n, const int32_t* src, int32_t* host_dst) {
  cudaStream_t st = stream();
  if (!perm) {
    FM_CUDA(cudaMemcpyAsync(host_dst, src, size_t(n) * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    return;
  }
  if (int32_t* d = mapped_host(host_dst)) {
    k_gather<int32_t><<<nblk(n, 256), 256, 0, st>>>(n, 1, perm, src, d);
    FM_LAUNCHED();
    FM_CUDA(cudaStreamSynchronize(st));
    return;
  }
  DBuf<int32_t> tmp;
  int32_t* buf = staging<int32_t>(size_t(n));
  if (!buf) {
    tmp.alloc(std::max<int64_t>(n, 1));
    buf = tmp.p;
  }
  k_gather<int32_t><<<nblk(n, 256), 256, 0, st>>>(n, 1, perm, src, buf);
  FM_LAUNCHED();
  FM_CUDA(cudaMemcpyAsync(host_dst, buf, size_t(n) * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  FM_CUDA(cudaStreamSynchronize(st));
}

void gather_levels(const int32_t* perm, int64_t n, const int8_t* lvl, int32_t* host_dst) {
  cudaStream_t st = stream();
  if (int32_t* d = perm ? mapped_host(host_dst) : nullptr) {
    k_widen<<<nblk(n, 256), 256, 0, st>>>(n, perm, lvl, d);
    FM_LAUNCHED();
    FM_CUDA(cudaStreamSynchronize(st));
    return;
  }
  DBuf<int32_t> tmp;
  int32_t* buf = staging<int32_t>(size_t(n));
  if (!buf) {
    tmp.alloc(std::max<int64_t>(n, 1));
    buf = tmp.p;
  }
  if (perm) {
    k_widen<<<nblk(n, 256), 256, 0, st>>>(n, perm, lvl, buf);
    FM_LAUNCHED();
  } else {
    FM_CUDA(cudaMemsetAsync(buf, 0, size_t(n) * sizeof(int32_t), st));
  }
  FM_CUDA(cudaMemcpyAsync(host_dst, buf, size_t(n) * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  FM_CUDA(cudaStreamSynchronize(st));
}

void gather_col(const int32_t* perm, int64_t n, int stride, int col, const double* src, double* host_dst) {
  cudaStream_t st = stream();
  DBuf<double> tmp(std::max<int64_t>(n, 1));
  k_gather_col<<<nblk(n, 256), 256, 0, st>>>(n, stride, col, perm, src, tmp.p);
  FM_LAUNCHED();
  FM_CUDA(cudaMemcpyAsync(host_dst, tmp.p, size_t(n) * sizeof(double), cudaMemcpyDeviceToHost, st));
  FM_CUDA(cudaStreamSynchronize(st));
}

void scatter_rows(const int32_t* perm, int64_t n, int width, const double* host_src, double* dst) {
  cudaStream_t st = stream();
  if (!perm) {
    FM_CUDA(cudaMemcpyAsync(dst, host_src, size_t(n) * width * sizeof(double), cudaMemcpyHostToDevice, st));
    FM_CUDA(cudaStreamSynchronize(st));
    return;
  }
  DBuf<double> tmp;
  tmp.upload(host_src, size_t(n) * width);
  k_scatter<double><<<nblk(n * width, 256), 256, 0, st>>>(n, width, perm, tmp.p, dst);
  FM_LAUNCHED();
  FM_CUDA(cudaStreamSynchronize(st));
}

}  // namespace fmh
