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
// grade_count_node for the four siblings 4m..4m+3 of level l >= 1 (children
// of level-(l-1) node m) in one thread: the flags and counts of a sibling
// quad are contiguous (block-Morton), so its own flags, its children's flags
// and counts, and the neighbours' flags come as a few 4 / 16 B words from
// the 3 x 3 level-(l-1) parents around m instead of ~17 byte loads per node,
// each behind its own index computation.  The same flags and counts as four
// grade_count_node calls.
__device__ __forceinline__ void grade_count_quad(uint8_t* __restrict__ fl, const uint8_t* __restrict__ fl1,
                                                 int32_t* __restrict__ cnt, const int32_t* __restrict__ cnt1,
                                                 int l, int L, int M, int N, uint64_t m, int graded,
                                                 const uint8_t* __restrict__ ring,
                                                 const uint32_t* own_sig = nullptr) {
  // the 3 x 3 parents' node indices (-1: outside the domain), needed for the
  // ring and the graded neighbours only
  long long par[3][3];
  if (ring || (graded && l + 1 < L)) {
    int I, J;
    node_ij(l - 1, m, M, I, J);
    const int wp = M << (l - 1), hp = N << (l - 1);  // level-(l-1) extent
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
      for (int dx = -1; dx <= 1; ++dx) {
        const int pi = I + dx, pj = J + dy;
        const bool in = pi >= 0 && pj >= 0 && pi < wp && pj < hp;
        par[dy + 1][dx + 1] = in ? (long long)node_index(l - 1, pi, pj, M) : -1;
      }
  }
  // own flags (or the ring's dilation of its closed flags)
  int g[4];
  if (ring) {
    // the 4 x 4 window of level-l nodes around the quad, bit (4y + x) for
    // node (2I - 1 + x, 2J - 1 + y), from the parents' sibling words
    uint32_t w[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b)
        w[a][b] = par[a][b] >= 0 ? *reinterpret_cast<const uint32_t*>(ring + 4 * par[a][b]) : 0u;
    unsigned win = 0;
#pragma unroll
    for (int y = 0; y < 4; ++y)
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        const int pa = y == 0 ? 0 : y == 3 ? 2 : 1, pb = x == 0 ? 0 : x == 3 ? 2 : 1;
        const int cx = (x == 0 || x == 2) ? 1 : 0, cy = (y == 0 || y == 2) ? 1 : 0;
        const unsigned byte = (w[pa][pb] >> (8 * (cx | (cy << 1)))) & 0xffu;
        win |= (byte ? 1u : 0u) << (4 * y + x);
      }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int x = 1 + (c & 1), y = 1 + (c >> 1);  // the node's window position
      const unsigned nb3 = (0x7u << (x - 1)) * 0x111u << (4 * (y - 1));  // its 3 x 3 block
      g[c] = (win & nb3) ? 1 : 0;
    }
  } else {
    // own flags: fl's (or, deferred significance, the caller's)
    const uint32_t own = own_sig ? *own_sig : *reinterpret_cast<const uint32_t*>(fl + 4 * m);
#pragma unroll
    for (int c = 0; c < 4; ++c) g[c] = int((own >> (8 * c)) & 0xffu);
  }
  int cn[4] = {1, 1, 1, 1};
  if (l + 1 < L) {
    // the children's flags of the quad's nodes (node c: word c)
    const uint4 k4 = *reinterpret_cast<const uint4*>(fl1 + 16 * m);
    const uint32_t kids[4] = {k4.x, k4.y, k4.z, k4.w};
    bool any_g = false;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      int nbr = 0;
      if (graded && !kids[c] && !g[c]) {
        // the level-(l+1) nodes edge-adjacent to node c's child block: the
        // facing children of its W E S N level-l neighbours, each either a
        // sibling in this quad or a node of a side parent
        const int cx = c & 1, cy = c >> 1;
        auto childw = [&](int nx, int ny) -> uint32_t {  // window coords of a level-l node, 0..3
          const int pa = ny == 0 ? 0 : ny == 3 ? 2 : 1, pb = nx == 0 ? 0 : nx == 3 ? 2 : 1;
          const long long p = par[pa][pb];
          if (p < 0) return 0u;
          const int cc = (nx == 0 || nx == 2 ? 1 : 0) | ((ny == 0 || ny == 2 ? 1 : 0) << 1);
          return *reinterpret_cast<const uint32_t*>(fl1 + 4 * (4 * p + cc));
        };
        const int x = 1 + cx, y = 1 + cy;
        const uint32_t W = cx ? kids[c - 1] : childw(x - 1, y);
        const uint32_t E = cx ? childw(x + 1, y) : kids[c + 1];
        const uint32_t S = cy ? kids[c - 2] : childw(x, y - 1);
        const uint32_t Nn = cy ? childw(x, y + 1) : kids[c + 2];
        // facing children: W's east column (bytes 1, 3), E's west (0, 2),
        // S's north row (2, 3), N's south row (0, 1)
        nbr = ((W & 0xff00ff00u) | (E & 0x00ff00ffu) | (S & 0xffff0000u) | (Nn & 0x0000ffffu)) ? 1 : 0;
      }
      if (kids[c] || nbr) g[c] = 1;
      any_g |= g[c] != 0;
    }
    if (any_g) {
      const int4* cc = reinterpret_cast<const int4*>(cnt1 + 16 * m);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (g[c]) {
          const int4 v = cc[c];
          cn[c] = v.x + v.y + v.z + v.w;
        }
      }
    }
  } else {
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (g[c]) cn[c] = 4;
  }
  *reinterpret_cast<uint32_t*>(fl + 4 * m) =
      uint32_t(uint8_t(g[0])) | (uint32_t(uint8_t(g[1])) << 8) | (uint32_t(uint8_t(g[2])) << 16) |
      (uint32_t(uint8_t(g[3])) << 24);
  *reinterpret_cast<int4*>(cnt + 4 * m) = make_int4(cn[0], cn[1], cn[2], cn[3]);
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
