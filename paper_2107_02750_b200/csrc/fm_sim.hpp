// Device views and the host Sim object behind fm_sim* (the drive<Sim> duck
// type of run.cpp:35-141 implemented on the device).
#pragma once

#include <memory>

#include "fm_internal.hpp"

namespace fmh {

constexpr int kMaxInflows = 8;
constexpr int kMaxHydroSamples = 4096;

// Device copy of the EventClock (sim_common.hpp:31-45) plus the per-step
// control block written by the step-decision kernel.  clk[1] is the published
// state: k_decide reads it as the step-start state and replaces it with the
// step in flight, which is the next step's start state.  clk[0] is unused.
struct DevClock {
  double end_time, out_int, gauge_int, now;
  long long next_out, next_gauge;
  double dt, t0;         // this step
  long long steps, max_steps;
  int active, stop_at_events, event_due, finished;
  int blew_up, had_step, pad0, pad1;
  double dt_min, dt_max, vol_in, blow_t;
  unsigned long long bad_key;     // reported key of the first non-finite cell
  double per_cell[kMaxInflows];   // Q(t0) dt / region_cells, or 0 when Q <= 0
  int on[kMaxInflows];
};

// Per-step reductions, double-buffered by step parity.
struct DevRed {
  unsigned long long dtmin;   // DG2/FV1: min size/max(sx,sy); ACC: min wet size
  unsigned long long hmaxc;   // ACC: ~bits of the max wet h (min-reduced like the
                              // other fields, so a slot reduces across ranks with one min)
  unsigned long long badkey;  // min (level<<58 | j<<29 | i) of non-finite cells
  unsigned long long pad;
};

struct Hydro {
  int off[kMaxInflows + 1];
  int n;
  long long region[kMaxInflows];
  double t[kMaxHydroSamples], q[kMaxHydroSamples];
};

// Everything a non-uniform leaf kernel needs (POD, passed by value).
struct NuView {
  int L, M, N, scheme, adaptive, ninflow, libm;
  double R, x0, y0, g, hdry, courant;
  int bc[4];
  long long n;
  // per level: element size R * 2^(L-l) and its reciprocal (host-computed,
  // the same IEEE values as the device expressions they replace)
  double lsz[16], linv[16];
  const int8_t* lvl;
  const int32_t* li;
  const int32_t* lj;
  const double* z;      // 3 per leaf
  const double* nman;
  const int32_t* nb;    // 8 per leaf: 2 per side (N,E,S,W)
  const uint8_t* sk;    // 2 bits per side: 0 boundary, 1 coarser, 2 same, 3 finer
  const double* zpair;  // adaptive: per leaf-side z* partner (4 per leaf) or null
  const int32_t* infc;  // ninflow x n fine-cell counts per leaf
  // ACC
  const int32_t* seg_l;
  const int32_t* seg_r;
  const uint8_t* seg_geo;  // per segment: x-normal + limit-point offsets (k_seg_geo)
  const double2* segz;     // P2: per segment, both leaves' z at its centre (k_seg_z)
  const double* zside;     // P2: per leaf, z at its four side midpoints N E S W (k_seg_z)
  const int32_t* sid;   // 8 per leaf: segment ids of the sub-faces per side
  const double* segst;  // 6 per segment: HLL flux (m n t), z*, h*L, h*R
  long long nseg;
  // adaptive sims: the segment count lives on the device (the host launches
  // with an upper bound, see build_topology); null for static sims
  const long long* nseg_dev;
};

// Operations of one step (nu_step_ops in nu_flow.cu).
enum StepOp { OP_HEAD, OP_EXCH_U, OP_STAGE1, OP_EXCH_US, OP_STAGE2, OP_ACC, OP_REDUCE };

struct Comm;  // shard.cu: the transport between the ranks of a sharded sim

// A sim restricted to a contiguous Morton range of the global leaves plus a
// halo of remote neighbours (shard.cu).  Local leaf arrays hold the `n` owned
// leaves first, then the halo grouped by owner rank; segments are the global
// segments with at least one owned leaf, in global order.
struct Shard {
  Comm* comm = nullptr;
  int rank = 0, nranks = 1;
  int64_t first = 0, n_global = 0, n_halo = 0;
  std::vector<int> peers;                 // ranks exchanged with, ascending
  std::vector<int64_t> soff, scnt;        // per peer: slice of send_idx / send_buf
  std::vector<int64_t> hoff, hcnt;        // per peer: slice of the halo (local n + hoff)
  DBuf<int32_t> send_idx;                 // local indices of the owned leaves sent
  DBuf<double> send_buf;                  // 9 doubles per sent leaf
  // NCCL: the exchange runs on a side stream (fork/join through events, also
  // under graph capture) while the segments that need no halo are computed
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  bool pending = false;
  // the stage split (DG2 stage 1): the owned leaves some peer needs (each
  // once, ascending) and the rest; stage 1 runs the first list, starts the
  // U* exchange (NCCL) and runs the rest while it is in flight
  DBuf<int32_t> stage_first, stage_rest;
  int64_t n_first = 0, n_rest = 0;
  bool us_started = false;  // this step's U* exchange was started inside stage 1
  ~Shard();
};

struct Sim {
  int solver = 0, scheme = 0, libm = 0;
  bool adaptive = false, uniform = false;
  double g = 9.80665, hdry = 1e-6, courant = 0.33;
  int bc[4] = {0, 0, 0, 0};
  // geometry
  int L = 0, M = 1, N = 1;
  double R = 1, x0 = 0, y0 = 0;
  int nx = 0, ny = 0;  // uniform raster (ny: owned rows of a band)
  int gy0 = 0, nyg = 0;        // band: first global row, global row count (0: unsharded)
  int ghost_s = 0, ghost_n = 0;  // band: ghost rows stored after the owned ones
  // Power-of-two element sizes with exactly representable coordinates: the
  // stage kernels evaluate planes at exact offsets and replace divisions by
  // the element size with exact reciprocal multiplies (bit-identical).
  bool p2 = false;
  int64_t n = 0, nseg = 0;
  // adaptive sims: the re-grid's topology build does not wait for the
  // segment count; nseg is then an upper bound (4 n) for launch sizes, the
  // true count is nseg_dev[0] on the device and lands in host->nseg (page-
  // locked) at the next host sync, when nseg_lazy is cleared
  DBuf<long long> nseg_dev;
  bool nseg_lazy = false;
  DBuf<int32_t> topo_owned, topo_base;  // adaptive: build_topology's scratch, kept
  DBuf<long long> topo_sums;
  // page-locked host slots for readbacks that ride on one sync: the clock,
  // the new leaf count of an adapt, the segment count
  struct HostSlots {
    DevClock clk;
    long long n_new, nseg;
  };
  HostSlots* host = nullptr;
  HostSlots& slots();
  void settle_nseg() {  // after a host sync
    if (nseg_lazy) {
      nseg = host->nseg;
      nseg_lazy = false;
    }
  }
  int64_t nseg_inner = 0;  // shards: leading local segments with both leaves owned
  // leaves (device Morton order) and state
  DBuf<int8_t> lvl;
  DBuf<int32_t> li, lj;
  DBuf<double> u, us, z, nman, zpair;
  DBuf<int32_t> nb, sid, seg_l, seg_r;
  DBuf<uint8_t> sk, seg_geo;
  DBuf<double> segz;        // P2: 2 per segment (static topography limits)
  DBuf<double> zside;       // P2: 4 per leaf (static topography side limits)
  DBuf<double> segst;       // DG2/FV1 segment states (6 per segment)
  DBuf<double> accq, accqb;  // ACC: per segment, per leaf-side (4 per leaf)
  DBuf<double> aqx, aqy;     // uniform ACC faces
  DBuf<int32_t> infc;        // per inflow per leaf counts
  int ninflow = 0;
  std::vector<std::vector<double>> hy_t, hy_q;
  std::vector<long long> region;
  std::vector<int> rect;     // 4 per inflow (i0 j0 i1 j1)
  DBuf<Hydro> hydro;
  DBuf<DevClock> clk;        // [2]
  DBuf<DevRed> red;          // [2]
  DBuf<int> errflag;         // device error bits (negative depth into HLL)
  bool fv1_in_star = false;
  // ACC's compact state while the device loop runs (nu_flow.cu): h (owned +
  // halo), qx, qy (owned), z.c0 (owned + halo) and the minimum key of a leaf
  // with a non-finite slope; acc_soa: the compact arrays hold the state and
  // the c0 columns of U are stale (the slopes in U never change under ACC)
  DBuf<double> ch, cqx, cqy, czc;
  DBuf<unsigned long long> cbad;
  bool acc_soa = false;
  // FV1's compact state (nu_flow.cu): rows of 3 (h, qx, qy means) for U
  // (owned + halo) and U*; fv1c: the state is there (between steps in cs3),
  // the slopes in U are +0 exactly (checked when the state moves in)
  DBuf<double> cu3, cs3;
  bool fv1c = false;
  // device-side checkpoint (fm_sim_snapshot / fm_sim_restore)
  DBuf<double> snap_u, snap_us, snap_q, snap_qb, snap_aqx, snap_aqy;
  int64_t snap_n = -1;
  // bumped whenever the leaf set changes (adaptive re-grid): a snapshot only
  // restores onto the leaf set it was taken from
  uint64_t leaf_gen = 0, snap_gen = ~0ull;
  bool snap_fv1 = false;
  double last_run_ms = 0.0;
  // Manning raster (kept for adaptive remaps)
  DBuf<double> mr;
  const double* mr_ext = nullptr;  // the caller's raster, read in place during creation only
  int mr_ncols = 0, mr_nrows = 0;
  double mr_xll = 0, mr_yll = 0, mr_cs = 1, manning = 0;
  bool has_mr = false;
  // adaptive state
  std::unique_ptr<Grid> grid;      // current grid pyramids (flags/off) + topo details
  struct AdaptState* ad = nullptr;  // owned; freed by adaptive_destroy
  int adapt_every = 1;
  int64_t since_adapt = 0;
  std::vector<std::pair<double, int64_t>> element_log;
  // CUDA graphs of 32, 8 and 1 device-loop steps (sim_run)
  cudaGraphExec_t gexec[3] = {nullptr, nullptr, nullptr};
  int64_t gkern[3] = {0, 0, 0};
  int g_layout = 0;  // the state layout the graphs were captured with
  std::unique_ptr<Shard> shard;  // set for a sharded (multi-rank) static sim
  // device order -> reference (level, j, i) order, cached per leaf set (order.cu)
  DBuf<int32_t> ref_perm;
  bool ref_perm_ok = false;
  ~Sim();

  NuView view() const;
};

Sim* sim_create(const fm_sim_desc* d, const fm_raster* dem, const Grid* grid);
double sim_compute_dt(Sim& s);
void sim_step(Sim& s, double dt);
double sim_apply_inflows(Sim& s, double t, double dt);
void sim_adapt(Sim& s, double t);
double sim_volume(Sim& s);
bool sim_finite(Sim& s, double* bx, double* by);
void sim_download(Sim& s, int32_t* l, int32_t* i, int32_t* j, double* u9, double* z3);
void sim_upload(Sim& s, const double* u9);
void sim_run(Sim& s, fm_clock* clk, int64_t max_steps, int stop_at_events, fm_run_result* out);
void sim_profile(Sim& s, int64_t steps, double* ms, int64_t* counts, int cap, int* nfam);
void sim_snapshot(Sim& s);
void adaptive_stats(Sim& s, int64_t* n_enc, int64_t* n_int);
void sim_checkpoint(Sim& s, const char* path);
void sim_resume(Sim& s, const char* path);
void sim_sync_u(Sim& s);  // FV1: move the staged post-step state back into u
// reference-order transfers (order.cu); perm == nullptr means identity
const int32_t* sim_ref_perm(Sim& s);
void order_preload();
// Lends device scratch to the gathers below for the scope's lifetime.
struct StageScope {
  StageScope(void* p, size_t bytes);
  ~StageScope();
};
void gather_rows(const int32_t* perm, int64_t n, int width, const double* src, double* host_dst);
void gather_i32(const int32_t* perm, int64_t n, const int32_t* src, int32_t* host_dst);
void gather_levels(const int32_t* perm, int64_t n, const int8_t* lvl, int32_t* host_dst);
void gather_col(const int32_t* perm, int64_t n, int stride, int col, const double* src, double* host_dst);
void scatter_rows(const int32_t* perm, int64_t n, int width, const double* host_src, double* dst);
// output sampling (output.cu)
void sim_raster_shape(const Sim& s, int32_t* nc, int32_t* nr, double* xll, double* yll, double* cs,
                      double* nodata);
void sim_raster(Sim& s, int which, double* out, bool on_device);
void sim_sample_gauges(Sim& s, int n, const double* x, const double* y, double* out4);
void extent_metrics(const fm_raster* test, const fm_raster* ref, double wet, int64_t* counts,
                    double* rates);
void sim_restore(Sim& s);

// step operations (nu_flow.cu) and the shard layer (shard.cu)
std::vector<int> nu_step_ops(const Sim& s, bool manual);
void nu_step_op(Sim& s, int op, bool manual, double mdt, int* err);
void un_step_op(Sim& s, int op, bool manual, double mdt, int* err);
inline void step_op(Sim& s, int op, bool manual, double mdt, int* err) {
  if (s.uniform)
    un_step_op(s, op, manual, mdt, err);
  else
    nu_step_op(s, op, manual, mdt, err);
}
void shard_op(Sim& s, int op);  // exchange / reduce for a sharded sim (NCCL)
void shard_finish(Sim& s);      // join an exchange started by shard_op
void shard_stage_lists(Sim& s);  // the stage split's leaf lists (after send_idx)
struct ShardPlan {
  int64_t first = 0, count = 0;
  std::vector<int64_t> segs;              // global ids of the local segments, ascending
  std::vector<int64_t> halo;              // global ids of the halo leaves, ascending
  std::vector<int> halo_owner;            // owner rank of each halo leaf (ascending)
  std::vector<std::vector<int64_t>> send; // per rank: owned global ids it needs, ascending
};
int64_t shard_first(int64_t n, int nranks, int r);
ShardPlan shard_plan(int64_t n, int64_t nseg, const int32_t* seg_l, const int32_t* seg_r, int nranks,
                     int rank);
Comm* comm_create_local(int nranks);
Comm* comm_create_nccl(int nranks, int rank, const uint8_t* id);
Comm* comm_create_host(int nranks, int rank, const char* name);
bool shard_eager(const Sim& s);  // the step cannot be graph-captured (host transport)
bool shard_nccl(const Sim& s);   // a shard on an NCCL communicator
void comm_unique_id(uint8_t* out);
void comm_destroy(Comm* c);
void comm_forget(Comm* c, Sim* s);
Sim* sim_create_shard(const fm_sim_desc* d, const fm_raster* dem, const Grid* grid, Comm* comm, int rank);
double* exch_array(Sim& s, int op, int* w);
void shard_pack(Sim& s, const double* arr, int w);
void shard_local_recv(Sim& s, double* arr, int w);
void shard_local_reduce(const std::vector<Sim*>& sims);
void shard_allreduce_u64_min(Sim& s, unsigned long long* dev, int count);
double shard_allreduce_sum(Sim& s, double v);
void group_run(const std::vector<Sim*>& sims, fm_clock* clk, int64_t max_steps, int stop_at_events,
               fm_run_result* out);
// topology (topo.cu)
// zp (adaptive re-grids): the z encode-up pyramid per level; the segment
// pass then also writes the segment statics, side limits and z* partners
void build_topology(Sim& s, const Grid& g, const double* const* zp = nullptr);
void build_seg_geo(Sim& s);  // after seg_l / seg_r and the leaf keys are final
void build_seg_z(Sim& s);    // after build_seg_geo and the final topography z
void resolve_inflows(Sim& s, const Grid& g);
void resolve_manning(Sim& s);
int64_t scan_exclusive(const int32_t* in, int32_t* out, int64_t n);

// adaptive (adaptive.cu)
void adaptive_init(Sim& s, const fm_sim_desc* d, const fm_raster* dem);
void adaptive_adapt(Sim& s, double t);
// adaptive_adapt in two halves around one host sync: the device-sized prefix
// (its new leaf count copied to s.slots().n_new), then, after the caller's
// sync, the transfer and the topology of the new leaf set
void adaptive_adapt_begin(Sim& s);
void adaptive_adapt_finish(Sim& s, double t);

// uniform (uniform.cu)
void uniform_init(Sim& s, const fm_sim_desc* d, const fm_raster* dem);

}  // namespace fmh
