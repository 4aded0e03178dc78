// Output sampling on the device: the drive<Sim> loop's gauge samples and
// raster dumps (run.cpp:56-74).
//
//   k_leaf_start   first fine cell of each leaf on the block-Morton curve
//   k_raster_nu    sample_to_raster (quadgrid.cpp:262-285) of leaf_raster
//                  (solver_nonuniform.cpp:508-519): every fine cell finds its
//                  leaf by binary search over the leaf starts (leaves tile the
//                  fine Morton curve in order) and evaluates the leaf's plane
//                  at the cell centre; one thread per output value, row-major,
//                  so the stores are coalesced.
//   k_raster_uni   field_raster (solver_uniform.cpp:501-516): c0 per cell.
//   k_gauges       NonUniformSim::sample_gauge (solver_nonuniform.cpp:489-506)
//                  / UniformSim::sample_gauge (solver_uniform.cpp:480-498).
//   k_extent       extent_metrics (metrics.cpp:51-73): hit / miss / false-alarm
//                  counts of two depth rasters, warp-reduced, one atomic each.
//
// The reference probes a hash map per fine cell (QuadGrid::find_containing,
// quadgrid.cpp:61-68) on one host thread: 67M probes for config 4.
#include "fm_device.cuh"
#include "fm_sim.hpp"
#include "step_common.cuh"

using namespace fmd;

namespace fmh {

namespace {

inline unsigned nblk(uint64_t n, int t) { return unsigned((n + t - 1) / t); }

__global__ void k_leaf_start(long long n, int L, int M, const int8_t* __restrict__ lvl,
                             const int32_t* __restrict__ li, const int32_t* __restrict__ lj,
                             unsigned long long* __restrict__ start) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int l = lvl[k];
  start[k] = node_index(l, li[k], lj[k], M) << (2 * (L - l));
}

// Leaf containing fine cell (fi, fj): the last leaf whose start is <= its
// Morton position (QuadGrid::find_containing, quadgrid.cpp:61-68).
__device__ __forceinline__ long long containing(const unsigned long long* __restrict__ start,
                                                long long n, unsigned long long m) {
  long long lo = 0, hi = n - 1;
  while (lo < hi) {
    const long long mid = (lo + hi + 1) >> 1;
    if (start[mid] <= m)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

// Whether Morton position m lies inside the leaves this sim owns: a sharded
// non-uniform sim owns one contiguous Morton range [start[0], end of its last
// leaf); every other fine cell belongs to another rank (NaN there, like the
// uniform band path).
__device__ __forceinline__ bool owned(const unsigned long long* __restrict__ start,
                                      const int8_t* __restrict__ lvl, long long n, int L,
                                      unsigned long long m) {
  return n > 0 && m >= start[0] && m < start[n - 1] + (1ull << (2 * (L - lvl[n - 1])));
}

__global__ void k_raster_nu(NuView v, const unsigned long long* __restrict__ start,
                            const double* __restrict__ u, int which, double* __restrict__ out) {
  const int nc = v.M << v.L, nr = v.N << v.L;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)nc * nr) return;
  const int row = int(t / nc), fi = int(t % nc);
  const int fj = nr - 1 - row;
  const unsigned long long m = node_index(v.L, fi, fj, v.M);
  if (!owned(start, v.lvl, v.n, v.L, m)) {
    out[t] = nan("");
    return;
  }
  const long long k = containing(start, v.n, m);
  const int l = v.lvl[k];
  const double x = v.x0 + (fi + 0.5) * v.R;
  const double y = v.y0 + (fj + 0.5) * v.R;
  const double* p = u + 9 * k + 3 * which;
  out[t] = eval_plane(P3{p[0], p[1], p[2]}, lcen(v.x0, v, l, v.li[k]), lcen(v.y0, v, l, v.lj[k]),
                      lsize(v, l), x, y);
}

__global__ void k_raster_uni(int nx, int ny, const double* __restrict__ u, int which,
                             double* __restrict__ out) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)nx * ny) return;
  const int row = int(t / nx), i = int(t % nx);
  const int j = ny - 1 - row;
  out[t] = u[9 * ((long long)j * nx + i) + 3 * which];
}

struct GaugeGeom {
  bool uniform, dg2;
  int nx, ny;
  int gy0, nyg;  // a raster band: its first global row, the global row count
};

__global__ void k_gauges(NuView v, GaugeGeom gg, const unsigned long long* __restrict__ start,
                         const double* __restrict__ u, int n, const double* __restrict__ xy,
                         double* __restrict__ out4) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n) return;
  const double x = xy[2 * g], y = xy[2 * g + 1];
  long long k;
  double cx, cy, sz;
  if (gg.uniform) {
    // UniformSim::sample_gauge (solver_uniform.cpp:480-483)
    const int i = min(max(int(floor((x - v.x0) / v.R)), 0), gg.nx - 1);
    const int j = min(max(int(floor((y - v.y0) / v.R)), 0), gg.nyg - 1);
    if (j < gg.gy0 || j >= gg.gy0 + gg.ny) {  // another band's cell
      for (int q = 0; q < 4; ++q) out4[4 * g + q] = nan("");
      return;
    }
    k = (long long)(j - gg.gy0) * gg.nx + i;
    cx = v.x0 + (i + 0.5) * v.R;
    cy = v.y0 + (j + 0.5) * v.R;
    sz = v.R;
  } else {
    // QuadGrid::find_point (quadgrid.cpp:70-74)
    const int fi = min(max(int(floor((x - v.x0) / v.R)), 0), (v.M << v.L) - 1);
    const int fj = min(max(int(floor((y - v.y0) / v.R)), 0), (v.N << v.L) - 1);
    const unsigned long long m = node_index(v.L, fi, fj, v.M);
    if (!owned(start, v.lvl, v.n, v.L, m)) {  // another shard's leaf
      for (int q = 0; q < 4; ++q) out4[4 * g + q] = nan("");
      return;
    }
    k = containing(start, v.n, m);
    const int l = v.lvl[k];
    cx = lcen(v.x0, v, l, v.li[k]);
    cy = lcen(v.y0, v, l, v.lj[k]);
    sz = lsize(v, l);
  }
  const double* s = u + 9 * k;
  const double* z = v.z + 3 * k;
  double h, zv, qx, qy;
  if (gg.dg2) {
    h = smax(0.0, eval_plane(P3{s[0], s[1], s[2]}, cx, cy, sz, x, y));
    zv = eval_plane(P3{z[0], z[1], z[2]}, cx, cy, sz, x, y);
    qx = eval_plane(P3{s[3], s[4], s[5]}, cx, cy, sz, x, y);
    qy = eval_plane(P3{s[6], s[7], s[8]}, cx, cy, sz, x, y);
  } else {
    h = s[0];
    zv = z[0];
    qx = s[3];
    qy = s[6];
  }
  out4[4 * g] = h;
  out4[4 * g + 1] = h + zv;
  out4[4 * g + 2] = vel(h, qx, v.hdry);
  out4[4 * g + 3] = vel(h, qy, v.hdry);
}

__global__ void k_extent(long long n, const double* __restrict__ test, const double* __restrict__ ref,
                         double nd_test, double nd_ref, double wet, unsigned long long* __restrict__ cnt) {
  unsigned long long h = 0, m = 0, f = 0;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n;
       k += (long long)gridDim.x * blockDim.x) {
    const double a = test[k], b = ref[k];
    if (a == nd_test || b == nd_ref) continue;
    const bool wt = a >= wet, wr = b >= wet;
    h += wt && wr;
    m += !wt && wr;
    f += wt && !wr;
  }
  for (int o = 16; o; o >>= 1) {
    h += __shfl_xor_sync(0xffffffffu, h, o);
    m += __shfl_xor_sync(0xffffffffu, m, o);
    f += __shfl_xor_sync(0xffffffffu, f, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (h) atomicAdd(&cnt[0], h);
    if (m) atomicAdd(&cnt[1], m);
    if (f) atomicAdd(&cnt[2], f);
  }
}

void leaf_starts(Sim& s, DBuf<unsigned long long>& start) {
  start.alloc(size_t(s.n));
  k_leaf_start<<<nblk(s.n, 256), 256, 0, stream()>>>(s.n, s.L, s.M, s.lvl.p, s.li.p, s.lj.p,
                                                      start.p);
  FM_LAUNCHED();
}

}  // namespace

void sim_raster_shape(const Sim& s, int32_t* nc, int32_t* nr, double* xll, double* yll, double* cs,
                      double* nodata) {
  if (s.uniform) {
    *nc = s.nx, *nr = s.ny;  // a band's own rows when sharded
  } else {
    *nc = s.M << s.L, *nr = s.N << s.L;
  }
  *xll = s.x0, *yll = s.y0 + s.gy0 * s.R, *cs = s.R, *nodata = -9999.0;
}

void sim_raster(Sim& s, int which, double* out, bool on_device) {
  if (which < 0 || which > 2)
    throw Error(FM_ERR_CONFIG, "raster: which must be 0 (h), 1 (qx) or 2 (qy)");
  sim_sync_u(s);
  int32_t nc, nr;
  double a, b, c, d;
  sim_raster_shape(s, &nc, &nr, &a, &b, &c, &d);
  const size_t cells = size_t(nc) * nr;
  DBuf<double> tmp;
  double* dst = out;
  if (!on_device) {
    tmp.alloc(cells);
    dst = tmp.p;
  }
  cudaStream_t st = stream();
  if (s.uniform) {
    k_raster_uni<<<nblk(cells, 256), 256, 0, st>>>(s.nx, s.ny, s.u.p, which, dst);
    FM_LAUNCHED();
  } else {
    DBuf<unsigned long long> start;
    leaf_starts(s, start);
    k_raster_nu<<<nblk(cells, 256), 256, 0, st>>>(s.view(), start.p, s.u.p, which, dst);
    FM_LAUNCHED();
  }
  if (!on_device) tmp.download(out, cells);
  FM_CUDA(cudaStreamSynchronize(st));
}

void sim_sample_gauges(Sim& s, int n, const double* x, const double* y, double* out4) {
  if (n <= 0) return;
  sim_sync_u(s);
  std::vector<double> xy(2 * size_t(n));
  for (int g = 0; g < n; ++g) xy[2 * g] = x[g], xy[2 * g + 1] = y[g];
  DBuf<double> dxy, dout(4 * size_t(n));
  dxy.upload(xy.data(), xy.size());
  DBuf<unsigned long long> start;
  if (!s.uniform) leaf_starts(s, start);
  GaugeGeom gg{s.uniform, s.scheme == FM_DG2, s.nx, s.ny, s.gy0, s.nyg ? s.nyg : s.ny};
  k_gauges<<<nblk(n, 64), 64, 0, stream()>>>(s.view(), gg, start.p, s.u.p, n, dxy.p, dout.p);
  FM_LAUNCHED();
  dout.download(out4, 4 * size_t(n));
  FM_CUDA(cudaStreamSynchronize(stream()));
}

// extent_metrics (metrics.cpp:51-73) of two rasters, host or device resident.
void extent_metrics(const fm_raster* test, const fm_raster* ref, double wet, int64_t* counts,
                    double* rates) {
  if (!test || !ref) throw Error(FM_ERR_CONFIG, "extent_metrics: null raster");
  if (test->ncols != ref->ncols || test->nrows != ref->nrows || test->xll != ref->xll ||
      test->yll != ref->yll || test->cellsize != ref->cellsize)
    throw Error(FM_ERR_IO, "extent_metrics: raster geometries do not match");
  const long long n = (long long)ref->ncols * ref->nrows;
  cudaStream_t st = stream();
  DBuf<double> ta, tb;
  const double* a = test->values;
  const double* b = ref->values;
  if (!test->on_device) {
    ta.upload(test->values, n);
    a = ta.p;
  }
  if (!ref->on_device) {
    tb.upload(ref->values, n);
    b = tb.p;
  }
  DBuf<unsigned long long> c(3);
  c.zero();
  k_extent<<<148 * 8, 256, 0, st>>>(n, a, b, test->nodata, ref->nodata, wet, c.p);
  FM_LAUNCHED();
  unsigned long long h[3];
  c.download(h, 3);
  FM_CUDA(cudaStreamSynchronize(st));
  const long long hits = (long long)h[0], misses = (long long)h[1], fa = (long long)h[2];
  if (counts) counts[0] = hits, counts[1] = misses, counts[2] = fa;
  if (rates) {
    rates[0] = (hits + misses) > 0 ? double(hits) / double(hits + misses) : 1.0;
    rates[1] = (hits + fa) > 0 ? double(fa) / double(hits + fa) : 0.0;
    const long long denom = hits + misses + fa;
    rates[2] = denom > 0 ? double(hits) / double(denom) : 1.0;
  }
}

}  // namespace fmh
