// Per-node bodies of the level passes shared by the static MRA (mra.cu) and
// the adaptive re-grid (adaptive.cu): grading + subtree leaf counts
// (grade_flags, detail_tree.cpp:97-113, with buffer_ring's dilation) and the
// top-down decode into the leaf list (assemble_grid, detail_tree.cpp:132-164).
#pragma once

#include "fm_device.cuh"

namespace fmh {
namespace {

using namespace fmd;

// Final flags and subtree leaf counts, one level per launch, fine -> coarse.
// G(l) = sig(l) | any G(l+1) child | (graded) any G(l+1) node edge-adjacent to
// the 2x2 child block.  This single gather equals the reference's closure +
// sequential grading sweep (detail_tree.cpp:56-64, 97-113): a level-(l+1)
// flagged node flags the parents of its four edge neighbours, i.e. the
// parent P gets flagged iff a flagged level-(l+1) node is a child of P or
// edge-adjacent to P's child block, and G(l+1) is final before level l is
// visited in both formulations.  (Verified against the oracle on random trees
// in tests/test_mra_gpu.py.)
// ring (adaptive re-grid): the node's own flag is buffer_ring's dilation
// (solver_adaptive.cpp:75-94) of the closed flags `ring` of its level, taken
// here rather than in a separate pass: any flagged node in the same-level
// 8-neighbourhood (or itself)
// The neighbour flags below are loaded together (predicated on lying inside
// the domain) and then combined, once the node's own flags leave the answer
// open: the grading pass is a chain of levels, and a load-test-branch
// sequence per neighbour put up to 17 dependent round trips on a node's
// critical path.  Same results as the early-exit form.
__device__ __forceinline__ int ring_flag(const uint8_t* __restrict__ ring, int l, int M, int N, uint64_t n) {
  if (ring[n]) return 1;
  int i, j;
  node_ij(l, n, M, i, j);
  const int w = M << l, h = N << l;
  int any = 0;
#pragma unroll
  for (int q = 0; q < 9; ++q) {
    if (q == 4) continue;
    const int ni = i + q % 3 - 1, nj = j + q / 3 - 1;
    const bool in = ni >= 0 && nj >= 0 && ni < w && nj < h;
    any |= in ? ring[node_index(l, in ? ni : i, in ? nj : j, M)] : 0;
  }
  return any ? 1 : 0;
}

__device__ __forceinline__ void grade_count_node(uint8_t* __restrict__ fl, const uint8_t* __restrict__ fl1,
                                                 int32_t* __restrict__ cnt, const int32_t* __restrict__ cnt1,
                                                 int l, int L, int M, int N, uint64_t n, int graded,
                                                 const uint8_t* __restrict__ ring = nullptr) {
  int g = ring ? ring_flag(ring, l, M, N, n) : fl[n];
  int c = 1;
  if (l + 1 < L) {
    const uint32_t kids = *reinterpret_cast<const uint32_t*>(fl1 + 4 * n);
    // 2:1 grading: a flagged level-(l+1) node edge-adjacent to the child block
    int nbr = 0;
    if (graded && !kids && !g) {
      int i, j;
      node_ij(l, n, M, i, j);
      const int w = M << (l + 1), h = N << (l + 1);
      const int ci = 2 * i, cj = 2 * j;
      const int ri[8] = {ci - 1, ci - 1, ci + 2, ci + 2, ci, ci + 1, ci, ci + 1};
      const int rj[8] = {cj, cj + 1, cj, cj + 1, cj - 1, cj - 1, cj + 2, cj + 2};
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const bool in = ri[q] >= 0 && rj[q] >= 0 && ri[q] < w && rj[q] < h;
        nbr |= in ? fl1[node_index(l + 1, in ? ri[q] : ci, in ? rj[q] : cj, M)] : 0;
      }
    }
    if (kids || nbr) g = 1;
    if (g) {
      const int4 cc = *reinterpret_cast<const int4*>(cnt1 + 4 * n);
      c = cc.x + cc.y + cc.z + cc.w;
    }
  } else if (g) {
    c = 4;
  }
  fl[n] = uint8_t(g);
  cnt[n] = c;
}
struct LeafOut {
  int8_t* l;
  int32_t* i;
  int32_t* j;
  double* z;
};

__device__ __forceinline__ void emit_leaf(const LeafOut& o, int l, uint64_t node, int M, int32_t at,
                                          const P3& z) {
  int i, j;
  node_ij(l, node, M, i, j);
  o.l[at] = int8_t(l);
  o.i[at] = i;
  o.j[at] = j;
  o.z[3 * at] = z.c0;
  o.z[3 * at + 1] = z.cx;
  o.z[3 * at + 2] = z.cy;
}

// Top-down decode of one level (detail_tree.cpp:132-164): an active flagged
// node decodes its stored details into its four children; children that are
// leaves are emitted at their final index, the others pass their plane and
// offset down through the level-(l+1) scratch.
__device__ __forceinline__ void topdown_node(const uint8_t* __restrict__ flp, const uint8_t* __restrict__ fl,
                                             const uint8_t* __restrict__ fl1, const int32_t* __restrict__ cnt1,
                                             const int32_t* __restrict__ off, int32_t* __restrict__ off1,
                                             const double* __restrict__ zin, double* __restrict__ zout,
                                             const double* __restrict__ det, int l, int L, int M, int kind,
                                             uint64_t n, const LeafOut& out) {
  if (l > 0 && !flp[n >> 2]) return;
  const P3 z{zin[3 * n], zin[3 * n + 1], zin[3 * n + 2]};
  const int32_t o = off[n];
  if (!fl[n]) {
    if (l == 0) emit_leaf(out, 0, n, M, o, z);
    return;
  }
  double d[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) d[q] = det[9 * n + q];
  P3 kids[4];
  decode(z, d, kind, kids);
  int32_t run = o;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint64_t c = 4 * n + k;
    if (l + 1 == L) {
      emit_leaf(out, L, c, M, run, kids[k]);
      run += 1;
    } else if (!fl1[c]) {
      emit_leaf(out, l + 1, c, M, run, kids[k]);
      off1[c] = run;
      run += 1;
    } else {
      zout[3 * c] = kids[k].c0;
      zout[3 * c + 1] = kids[k].cx;
      zout[3 * c + 2] = kids[k].cy;
      off1[c] = run;
      run += cnt1[c];
    }
  }
}
// Exclusive scan of cnt[0..n) into off by the calling CTA (any block size
// that is a multiple of 32); the total lands in *total.
__device__ __forceinline__ void cta_exclusive_scan(const int32_t* __restrict__ cnt, int32_t* __restrict__ off,
                                                   int64_t n, long long* total) {
  __shared__ long long wsum[32];
  __shared__ long long base;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int64_t b0 = 0; b0 < n; b0 += blockDim.x) {
    const int64_t k = b0 + threadIdx.x;
    const long long v = k < n ? cnt[k] : 0;
    long long x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
      long long s = lane < nw ? wsum[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += y;
      }
      if (lane < nw) wsum[lane] = s;  // inclusive over warps
    }
    __syncthreads();
    const long long incl = x + (w ? wsum[w - 1] : 0);
    if (k < n) off[k] = int32_t(base + incl - v);
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) base += incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = base;
}

}  // namespace
}  // namespace fmh
