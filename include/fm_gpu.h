/*
 * fm_gpu.h — C ABI of the B200-native floodmra hot path (libfm_gpu.so).
 *
 * This is the drop-in boundary.  Each entry point replaces one seam of the
 * reference C++ library (`/root/reference/proj/core`, namespace floodmra);
 * the interface it stands in for is cited beside it.  Plain pointers and
 * sizes only: no C++ types, no torch types, no exceptions cross this line.
 * Every call returns an `int` status (FM_OK = 0); on failure
 * `fm_last_error()` returns a thread-local message and the status maps onto
 * the reference exception types (errors.hpp:9-37) and CLI exit codes
 * (tools/floodmra.cpp:171-186):
 *
 *   FM_ERR_CONFIG    ConfigError      (exit 2)
 *   FM_ERR_IO        IoError/ParseError (exit 3)
 *   FM_ERR_BLOWUP    BlowUpError      (exit 4; fm_run_result.blow_up_time = t)
 *   FM_ERR_STRUCTURE StructureError   (exit 1)
 *   FM_ERR_DOMAIN    DomainError      (exit 1)
 *   FM_ERR_CUDA      CUDA runtime / no device (exit 1) — there is no CPU fallback
 *
 * Units, layouts and orders follow the reference:
 *   - rasters are ESRI-style, row 0 = north (raster.hpp:8-26);
 *   - a DEM of n x m cells is an (n+1) x (m+1) VERTEX raster (field.hpp:93-98);
 *   - leaf arrays returned "in reference order" are sorted by (level, j, i)
 *     exactly as make_quadgrid sorts them (quadgrid.cpp:94-98);
 *   - flow coefficients per cell are 9 doubles
 *       [h.c0 h.c1x h.c1y qx.c0 qx.c1x qx.c1y qy.c0 qy.c1x qy.c1y]
 *     (FlowCoeffs, field.hpp:49-67) and topography 3 doubles [c0 c1x c1y].
 */
#ifndef FM_GPU_H
#define FM_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
enum {
  FM_OK = 0,
  FM_ERR_OTHER = 1,
  FM_ERR_CONFIG = 2,
  FM_ERR_IO = 3,
  FM_ERR_BLOWUP = 4,
  FM_ERR_STRUCTURE = 5,
  FM_ERR_DOMAIN = 6,
  FM_ERR_CUDA = 7
};

/* SolverKind (config.hpp:9) */
enum { FM_DG2 = 0, FM_FV1 = 1, FM_ACC = 2, FM_MWDG2 = 3, FM_HWFV1 = 4 };
/* WaveletKind (wavelets.hpp:9) */
enum { FM_MW = 0, FM_HW = 1 };
/* BoundaryKind (config.hpp:11) */
enum { FM_REFLECTIVE = 0, FM_OPEN = 1 };
/* Side (config.hpp:12) */
enum { FM_NORTH = 0, FM_EAST = 1, FM_SOUTH = 2, FM_WEST = 3 };
/* leaf orders for fm_grid_leaves / fm_sim_download */
enum { FM_ORDER_REFERENCE = 0, FM_ORDER_DEVICE = 1 };
/* fm_sim_desc.libm */
enum { FM_LIBM_NATIVE = 0, FM_LIBM_PORTABLE = 1 };

/* Raster (raster.hpp:10-26).  `values` is ncols*nrows doubles, row 0 north.
 * `on_device` != 0 means `values` is a CUDA device pointer already resident
 * in HBM (used by the bench's kernel-only leg); 0 means host memory. */
typedef struct fm_raster {
  const double* values;
  int32_t ncols, nrows;
  double xll, yll, cellsize, nodata;
  int32_t on_device;
} fm_raster;

/* InflowSpec + Hydrograph (config.hpp:15-18, hydrograph.hpp:10-16): an
 * inclusive fine-cell rectangle receiving a t,Q hydrograph as a depth source. */
typedef struct fm_inflow {
  const double* t;
  const double* q;
  int32_t nsamples;
  int32_t i0, j0, i1, j1;
} fm_inflow;

/* The subset of ScenarioConfig (config.hpp:29-69) the solvers read. */
typedef struct fm_sim_desc {
  int32_t solver;          /* FM_DG2 .. FM_HWFV1 */
  double g, h_dry;         /* 9.80665, 1e-6 */
  double courant;          /* <= 0: per-solver default (config.cpp:37-47) */
  int32_t bc[4];           /* N, E, S, W : FM_REFLECTIVE / FM_OPEN */
  double manning;          /* uniform Manning n */
  const fm_raster* manning_raster;      /* optional, CELL-centred n x m */
  const fm_raster* initial_depth_raster; /* optional, same geometry as DEM */
  int32_t has_initial_surface;
  double initial_surface;
  double initial_depth;
  const fm_inflow* inflows;
  int32_t n_inflows;
  double epsilon;          /* adaptive solvers */
  int32_t max_level;       /* adaptive solvers */
  int32_t adapt_every;     /* adaptive solvers, >= 1 */
  /* libm used by friction (cbrt) and ACC (pow(h, 7/3)):
   *   FM_LIBM_NATIVE   the platform's (CUDA on the GPU, glibc in the reference);
   *   FM_LIBM_PORTABLE a deterministic +,-,*,/ implementation that the CPU
   *                    oracle reproduces bit-for-bit (parity harness only). */
  int32_t libm;
} fm_sim_desc;

/* EventClock (sim_common.hpp:31-45) state. */
typedef struct fm_clock {
  double end_time, output_interval, gauge_interval, now;
  int64_t next_output, next_gauge;
} fm_clock;

/* What one call of the device-resident drive loop did (run.cpp:80-111). */
typedef struct fm_run_result {
  int64_t steps;
  double dt_min, dt_max;
  double volume_inflow;
  int32_t blew_up;
  double blow_up_time;
  double bad_x, bad_y;
  int32_t finished;       /* clock.now >= end_time */
  int32_t event_due;      /* stopped because a gauge/output event was reached */
} fm_run_result;

typedef struct fm_grid fm_grid;
typedef struct fm_sim fm_sim;

/* ---- runtime ------------------------------------------------------------ */
const char* fm_last_error(void);
/* Select the CUDA device for this thread's subsequent calls (one rank per GPU). */
int fm_init(int32_t device);
/* Route all library work onto `stream` (a cudaStream_t; NULL = library stream). */
int fm_set_stream(void* stream);
int fm_synchronize(void);
/* Number of kernels this library has launched since load (evidence counter). */
int64_t fm_launch_count(void);
/* Device self-checks of the arithmetic building blocks against IEEE:
 * which = 0: the inlined division vs `/` on n seeded random operand pairs;
 * which = 1: the constant-divisor division of project4 (a / (4 sqrt3)) vs `/`;
 * which = 2: the shared-divisor division of zdiv2 (nvcc's fast-path sequence
 *            with the reciprocal computed once) vs `a == 0 ? a : a / b`;
 * spanning the fast-path exponent window and its edges.  *failures counts
 * bit mismatches.  which = 3 (FM_GUARD=1 only): one deliberate write past a
 * buffer's end, *failures = the overruns fm_debug_guard_report then finds
 * (the checker's positive control; n and seed unused). */
int fm_selftest(int32_t which, int64_t n, uint64_t seed, int64_t* failures);
/* Out-of-bounds write check (this pool refuses compute-sanitizer): with
 * FM_GUARD=1 in the environment when the library loads, every device
 * allocation carries 256 B guard bands of a known pattern on both sides,
 * verified on the device when the buffer is freed and, here, for every live
 * buffer.  *checked: band checks so far; *overruns: bands found modified.
 * Both 0 when FM_GUARD is off. */
int fm_debug_guard_report(int64_t* checked, int64_t* overruns);

/* The libm building blocks as the device evaluates them, for tests:
 * fn 0 = pow(x, 7/3) (FM_LIBM_NATIVE: correctly rounded in double-double,
 * fp32 correction terms), 1 = cbrt(x) (native), 2 = CUDA's pow(x, 7.0/3.0),
 * 3 = pow(x, 7/3) with the portable cube root, 4 = the all-fp64
 * double-double evaluation (the check for fn 0). */
int fm_eval_libm(int32_t fn, int64_t n, const double* x, double* out);

/* ---- static MRA --------------------------------------------------------- */
/* generate_static_grid(dem, eps, L, graded, kind)  — detail_tree.hpp:55-56,
 * detail_tree.cpp:172-178.  Pipeline: project_raster (field.cpp:106-117) ->
 * build_detail_tree (detail_tree.cpp:10-54) -> flag_significant
 * (:66-74) -> grade_flags (:97-113) -> assemble_grid (:132-164). */
int fm_mra_static(const fm_raster* dem, int32_t L, double eps, int32_t graded, int32_t kind,
                  fm_grid** out);
/* A grid from a leaf list and its topography: read_nug's construction
 * (quadgrid.cpp:310-327) via make_quadgrid (quadgrid.cpp:85-110), e.g. for
 * run_scenario's grid_file path (run.cpp:150-153).  Leaves in any order;
 * StructureError when they leave the domain, do not tile it or overlap.
 * Flags / details of an imported grid: flags = internal nodes, details 0. */
int fm_grid_import(int32_t L, int32_t M, int32_t N, double Rfine, double x0, double y0, int64_t n,
                   const int32_t* level, const int32_t* i, const int32_t* j, const double* topo3,
                   fm_grid** out);
int fm_grid_destroy(fm_grid* g);
int64_t fm_grid_num_leaves(const fm_grid* g);
/* QuadGrid scalars (quadgrid.hpp:54-60) plus DetailTree::field_norm. */
int fm_grid_info(const fm_grid* g, int32_t* L, int32_t* M, int32_t* N, double* Rfine, double* x0,
                 double* y0, double* field_norm);
/* Leaves + topography (NonUniformGrid, quadgrid.hpp:117-120).  Any output
 * pointer may be NULL.  topo3 is 3 doubles per leaf. */
int fm_grid_leaves(const fm_grid* g, int32_t order, int32_t* level, int32_t* i, int32_t* j,
                   double* topo3);
/* DetailTree::flags[level] (detail_tree.hpp:23), row-major j*(M<<level)+i. */
int fm_grid_flags(const fm_grid* g, int32_t level, uint8_t* out);
/* Per-node normalised details d_hat of DetailTree level `level`, row-major. */
int fm_grid_dhat(const fm_grid* g, int32_t level, double* out);
/* Count of nodes with |d_hat - eps| <= rel*eps. */
int fm_grid_near_threshold(const fm_grid* g, double rel, int64_t* count);
/* Device time of the last MRA pipeline's kernels (ms) and algorithmic bytes. */
int fm_grid_timing(const fm_grid* g, double* ms, double* bytes);
/* ancestor_closure (detail_tree.cpp:56-64) followed, when `graded`, by
 * grade_flags (detail_tree.cpp:97-113) on caller-supplied flags: `flags` holds
 * levels 0..L-1 back to back, each row-major j*(M<<l)+i; updated in place. */
int fm_grade_flags(int32_t L, int32_t M, int32_t N, int32_t graded, uint8_t* flags);

/* ---- simulations (drive<Sim> duck type, run.cpp:35-141) ----------------- */
/* run_scenario's dispatch (run.cpp:145-164): adaptive solvers build an
 * AdaptiveSim from the DEM (solver_adaptive.cpp:209-236); otherwise a
 * non-NULL grid gives make_nonuniform_sim (solver_nonuniform.cpp:558-636) and
 * a NULL grid gives make_uniform_sim (solver_uniform.cpp:522-601). */
int fm_sim_create(const fm_sim_desc* desc, const fm_raster* dem, const fm_grid* grid,
                  fm_sim** out);
int fm_sim_destroy(fm_sim* s);
int64_t fm_sim_num_cells(const fm_sim* s);
/* The sim's QuadGrid geometry (quadgrid.hpp:54-60): finest level L, coarse
 * blocks M x N, finest element size Rfine and the domain origin (x0, y0).
 * Uniform sims report L = 0 with M x N the raster's cells. */
int fm_sim_geometry(const fm_sim* s, int32_t* L, int32_t* M, int32_t* N, double* Rfine, double* x0,
                    double* y0);
int64_t fm_sim_num_segments(const fm_sim* s);
/* Sim::compute_dt (solver_nonuniform.cpp:427-449, solver_uniform.cpp:424-442). */
int fm_sim_compute_dt(fm_sim* s, double* dt);
/* Sim::step (solver_nonuniform.cpp:420-425, solver_uniform.cpp:417-422). */
int fm_sim_step(fm_sim* s, double dt);
/* Sim::apply_inflows (solver_nonuniform.cpp:451-465). */
int fm_sim_apply_inflows(fm_sim* s, double t, double dt, double* added);
/* AdaptiveSim::adapt (solver_adaptive.cpp:136-171); FM_ERR_CONFIG for static sims. */
int fm_sim_adapt(fm_sim* s, double t);
/* Sim::volume (solver_nonuniform.cpp:467-477). */
int fm_sim_volume(fm_sim* s, double* v);
/* Sim::finite_state (solver_nonuniform.cpp:479-487). */
int fm_sim_finite(fm_sim* s, int32_t* ok, double* bad_x, double* bad_y);
/* State in reference order ((level,j,i) for leaves, j*nx+i for rasters).
 * Any pointer may be NULL.  u9: 9 doubles per cell, z3: 3 per cell. */
int fm_sim_download(fm_sim* s, int32_t* level, int32_t* i, int32_t* j, double* u9, double* z3);
/* Overwrite the flow state (reference order) — lockstep re-seeding. */
int fm_sim_upload(fm_sim* s, const double* u9);
/* Geometry of the rasters below: depth_raster()/qx_raster()/qy_raster() of
 * NonUniformSim (fine grid, (N<<L) x (M<<L), quadgrid.cpp:266-272) and
 * UniformSim (ny x nx, solver_uniform.cpp:503-509). */
int fm_sim_raster_shape(fm_sim* s, int32_t* ncols, int32_t* nrows, double* xll, double* yll,
                        double* cellsize, double* nodata);
/* Sim::depth_raster / qx_raster / qy_raster (which = 0 / 1 / 2): non-uniform
 * sims sample every leaf plane at the fine-cell centres (sample_to_raster,
 * quadgrid.cpp:262-285, via solver_nonuniform.cpp:508-519), uniform sims copy
 * c0 (solver_uniform.cpp:501-520).  Row 0 north, ncols*nrows doubles into
 * `out` (a CUDA device pointer when out_on_device != 0).  The caller applies
 * crop_and_mask (sim_common.cpp:133-151) as drive<Sim> does. */
int fm_sim_raster(fm_sim* s, int32_t which, double* out, int32_t out_on_device);
/* Sim::sample_gauge (solver_nonuniform.cpp:489-506, solver_uniform.cpp:480-498)
 * at n points: out4 = n x GaugeValue {h, eta, u, v} (sim_common.hpp:47-49). */
int fm_sim_sample_gauges(fm_sim* s, int32_t n, const double* x, const double* y, double* out4);
/* Device-side checkpoint of the flow state (U, U*, ACC discharges) and
 * its restore, without host traffic; restore fails if the leaf set changed
 * since the snapshot (adaptive re-gridding). */
int fm_sim_snapshot(fm_sim* s);
/* The last adapt's sizes (adaptive sims): parents encoded by encode_up
 * (solver_adaptive.cpp:16-57) and the pyramid's internal nodes, for the
 * SURVEY §8 d4 adapt byte count. */
int fm_sim_adapt_stats(fm_sim* s, int64_t* n_encoded, int64_t* n_internal);
/* Binary checkpoint / restart (the reference has none): the leaf
 * keys and topography in the reference order, the flow state, and ACC's
 * face discharges.  Resume requires the same scenario and leaf set (keys
 * and topography bit for bit; FM_ERR_CONFIG otherwise); the EventClock
 * stays with the caller.  I/O errors: FM_ERR_IO. */
int fm_sim_checkpoint(fm_sim* s, const char* path);
int fm_sim_resume(fm_sim* s, const char* path);
int fm_sim_restore(fm_sim* s);
/* UniformSim's ACC face discharges acc_qx ((nx+1) x ny, row-major j*(nx+1)+i)
 * and acc_qy (nx x (ny+1)) (solver_uniform.hpp:53-54), read into get_x/get_y
 * and/or overwritten from set_x/set_y (any pointer may be NULL); the tests of
 * test_solver_uniform.cpp:303-326 set and read them directly.  Uniform ACC
 * sims only (FM_ERR_CONFIG otherwise). */
int fm_sim_acc_faces(fm_sim* s, double* get_x, double* get_y, const double* set_x, const double* set_y);
/* AdaptiveSim::element_log (solver_adaptive.hpp:23): number of entries, and copy. */
int64_t fm_sim_element_log(fm_sim* s, double* t, int64_t* count, int64_t cap);
/* The drive<Sim> loop body (run.cpp:80-111) resident on the device:
 * dt = clip(compute_dt) ; step ; apply_inflows ; advance ; adapt ; finite.
 * Runs until `max_steps`, the end time, a blow-up, or (stop_at_events != 0)
 * a gauge/output event time is reached.  `clk` is updated in place. */
int fm_sim_run(fm_sim* s, fm_clock* clk, int64_t max_steps, int32_t stop_at_events,
               fm_run_result* out);
/* Device time (ms) of the last fm_sim_run's kernels, measured with CUDA events. */
int fm_sim_last_run_ms(fm_sim* s, double* ms);
/* Per-kernel timing: runs `steps` device-loop steps launching each kernel
 * individually between CUDA events on the library stream; writes per kernel
 * family the summed milliseconds and launch counts (family names via
 * fm_sim_kernel_name).  Returns the number of families in *n. */
int fm_sim_profile(fm_sim* s, int64_t steps, double* ms, int64_t* launches, int32_t cap,
                   int32_t* n);
const char* fm_sim_kernel_name(fm_sim* s, int32_t family);

/* extent_metrics (metrics.cpp:51-73): a cell is inundated iff depth >=
 * wet_threshold, nodata cells of either raster are skipped.  counts =
 * {hits, misses, false_alarms}, rates = {hit_rate, false_alarm, csi}.  Either
 * raster may be device resident (e.g. from fm_sim_raster(..., out_on_device=1)).
 * Mismatched geometries: FM_ERR_IO (ParseError). */
/* rmse (metrics.cpp:32-46) of two gauge series (t strictly increasing): the
 * test series linearly interpolated at the reference's sample times inside
 * the overlap, the reference's summation order.  Host-side: gauge series are
 * hundreds of samples.  Empty or non-overlapping series: FM_ERR_IO. */
int fm_rmse(const double* test_t, const double* test_v, int64_t n_test, const double* ref_t,
            const double* ref_v, int64_t n_ref, double* out);
int fm_extent_metrics(const fm_raster* test, const fm_raster* ref, double wet_threshold,
                      int64_t* counts, double* rates);

/* ---- file formats either side of the path -------------
 * Host-side; the text formats are the reference's, byte for byte, and each
 * has a binary side format (magic "FMRB1" / "FMNG1", little-endian raw
 * fields) that the readers recognise by its magic.
 *
 * fm_raster_read: read_ascii_grid (raster.cpp:22-79) — six keyword/value
 * header lines in any order, keywords case-insensitive, then ncols*nrows
 * whitespace-separated values; the body is parsed by all host threads.  On
 * success out->values is library-owned host memory (page-locked when a device
 * is present, so it uploads at the link's rate), out->on_device = 0; free it
 * with fm_raster_release.  Unopenable file, malformed header or a value count
 * other than ncols*nrows: FM_ERR_IO (IoError / ParseError). */
int fm_raster_read(const char* path, fm_raster* out);
int fm_raster_release(fm_raster* r);
/* write_ascii_grid (raster.cpp:81-96) when binary == 0 ("%.17g" values, one
 * raster row per line), else the binary side format.  Host rasters only. */
int fm_raster_write(const fm_raster* r, const char* path, int32_t binary);
/* write_nug (quadgrid.cpp:287-302): "nug L M N Rfine x0 y0" then one
 * "level i j c0 c1x c1y" line per leaf in the reference's leaf order
 * (binary != 0: the same fields raw). */
int fm_grid_write(const fm_grid* g, const char* path, int32_t binary);
/* read_nug (quadgrid.cpp:304-327): records up to the first that does not
 * parse, then fm_grid_import's construction and checks (StructureError for
 * leaves that do not tile the domain, ParseError for a malformed header). */
int fm_grid_read(const char* path, fm_grid** out);

/* ---- multi-GPU: Morton-range shards of a static non-uniform sim ----------
 * (the reference is single-process.)  Rank r of R owns the
 * contiguous range [floor(n r / R), floor(n (r+1) / R)) of the Morton-ordered
 * leaves plus a halo of remote neighbours; per DG2 step two halo exchanges
 * and one min-allreduce, so every shard's state equals the unsharded sim's
 * bit for bit.  Adaptive and uniform sims do not shard (replicas). */
typedef struct fm_comm fm_comm;
/* NCCL transport, one process per GPU: rank 0 makes the id, the host
 * broadcasts it, every rank creates its communicator. */
int fm_comm_unique_id(uint8_t id[128]);
int fm_comm_create_nccl(int32_t nranks, int32_t rank, const uint8_t id[128], fm_comm** out);
/* Local group: all ranks as shards in this process on this device, stepped
 * together by fm_group_run (single-GPU check of the partition logic). */
int fm_comm_create_local(int32_t nranks, fm_comm** out);
/* A host transport: one process per rank (any devices, one GPU included),
 * halo slices and reduction slots staged through the POSIX shared-memory
 * segment `name` ("/..."; every rank passes the same name, rank 0 unlinks it
 * on destroy) with a process-shared barrier.  Steps are not graph-captured
 * on this transport.  Collective: every rank must call it. */
int fm_comm_create_host(int32_t nranks, int32_t rank, const char* name, fm_comm** out);
int fm_comm_destroy(fm_comm* c);
/* make_nonuniform_sim (solver_nonuniform.cpp:558-636) restricted to this
 * rank's shard.  fm_sim_run / step / compute_dt / finite / volume on an NCCL
 * shard are collective over the ranks; download / rasters return the shard's
 * own leaves. */
int fm_sim_create_shard(const fm_sim_desc* desc, const fm_raster* dem, const fm_grid* grid,
                        fm_comm* comm, int32_t rank, fm_sim** out);
int fm_sim_shard_info(const fm_sim* s, int32_t* rank, int32_t* nranks, int64_t* first,
                      int64_t* owned, int64_t* halo, int64_t* n_global);
/* The drive loop (run.cpp:80-111) over all shards of a local group. */
int fm_group_run(fm_sim* const* sims, int32_t n, fm_clock* clk, int64_t max_steps,
                 int32_t stop_at_events, fm_run_result* out);
/* The partition plan on the host (no device needed): owned range, local
 * segment count, halo (ascending global ids, their owner ranks) and the
 * owned leaves each rank needs (send_counts[nranks], concatenated ascending
 * lists in `send`).  Call with halo = send = NULL for the sizes. */
int fm_shard_plan(int64_t n_leaves, int64_t n_segments, const int32_t* seg_l,
                  const int32_t* seg_r, int32_t nranks, int32_t rank, int64_t* first,
                  int64_t* count, int64_t* n_local_segments, int64_t* n_halo, int64_t* halo,
                  int32_t* halo_owner, int64_t* send_counts, int64_t* send);
/* A sim's leaves and interior segments in device (Morton) order:
 * level/i/j per leaf (n), seg_l/seg_r per segment (W/S leaf, E/N leaf). */
int fm_sim_topology(fm_sim* s, int32_t* level, int32_t* i, int32_t* j, int32_t* seg_l,
                    int32_t* seg_r);

#ifdef __cplusplus
}
#endif

#endif /* FM_GPU_H */
