/*
 * ncsg.h -- C ABI of the B200-native NCS (near-circulant splitting) hot path.
 *
 * Drop-in boundary for the reference's CPU operator/solver path
 * (arXiv 1810.13100 reference `ncstomo`, paths relative to
 * /root/reference/proj).  Plain pointers and sizes only; no C++ exceptions
 * cross this boundary.  Every function returns an ncsg_status; the message of
 * the last failure on the calling thread is available from
 * ncsg_last_error().  Status codes mirror the reference's exception classes
 * and CLI exit codes (tools/main.cpp:588-603):
 *   NCSG_INVALID   <- std::invalid_argument   (e.g. radon.cpp:37-42)
 *   NCSG_DIVERGED  <- DivergenceError          (solvers.hpp:101-105)
 *   NCSG_CUDA      <- device / runtime failure (no CPU fallback exists)
 *
 * All compute is fp32 on the device; host-facing *_host entry points take
 * and return fp64 like the reference's std::span<const double> signatures and
 * convert at the boundary.  Device entry points take device pointers and a
 * cudaStream_t passed as void* (NULL = the handle's own stream).
 */
#ifndef NCSG_H
#define NCSG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  NCSG_OK = 0,
  NCSG_INVALID = 2,
  NCSG_RUNTIME = 3,
  NCSG_DIVERGED = 4,
  NCSG_CUDA = 5
} ncsg_status;

/* Message of the last failing call on this thread ("" if none). */
const char* ncsg_last_error(void);
/* Library version "major.minor.patch". */
const char* ncsg_version(void);
/* Number of visible CUDA devices (0 when none: every compute entry point then
 * fails with NCSG_CUDA -- there is no CPU fallback). */
int ncsg_device_count(void);

/* ------------------------------------------------------------------ geometry
 * Replaces ncstomo::default_detector_count (radon.cpp:10-13). */
int ncsg_default_detector_count(int n);

/* Parallel-beam projector handle.  Replaces RadonMap::RadonMap(n, n_angles,
 * n_det) (radon.hpp:16-36, radon.cpp:35-72): same validation (n >= 2,
 * n_angles >= 1, odd n_det covering the diagonal) and the same sample set --
 * the reference's fp64 ray table and per-sample box check are replayed on the
 * host when the handle is created and uploaded as per-ray valid intervals. */
typedef struct ncsg_radon ncsg_radon;
ncsg_status ncsg_radon_create(int n, int n_angles, int n_det, int device, ncsg_radon** out);
ncsg_status ncsg_radon_destroy(ncsg_radon* r);
/* domain_size() == n*n, range_size() == n_angles*n_det (radon.cpp:74-80). */
size_t ncsg_radon_domain_size(const ncsg_radon* r);
size_t ncsg_radon_range_size(const ncsg_radon* r);
/* Number of valid bilinear samples per application (= sum of R(1)). */
int64_t ncsg_radon_sample_count(const ncsg_radon* r);

/* RadonMap::forward (radon.cpp:82-102) on `batch` images laid out back to
 * back (stride n*n) into `batch` sinograms (stride n_angles*n_det), angle-
 * major [t][d] (image.hpp:23-36).  Device pointers. */
ncsg_status ncsg_radon_forward(const ncsg_radon* r, const float* x, float* out, int batch,
                               void* stream);
/* RadonMap::adjoint (radon.cpp:104-127): exact transpose of forward; `out` is
 * overwritten (the reference zero-fills first, radon.cpp:107). */
ncsg_status ncsg_radon_adjoint(const ncsg_radon* r, const float* u, float* out, int batch,
                               void* stream);
/* Host fp64 wrappers with the reference's span<const double> semantics. */
ncsg_status ncsg_radon_forward_host(const ncsg_radon* r, const double* x, double* out,
                                    int batch);
ncsg_status ncsg_radon_adjoint_host(const ncsg_radon* r, const double* u, double* out,
                                    int batch);

/* ------------------------------------------------------- sparse / fan beam
 * SparseMap (sparse.hpp:21-43): CSR over sinogram bins (view-major) with the
 * stored transpose for the adjoint (deterministic, exact to the matrix). */
typedef struct ncsg_sparse ncsg_sparse;

/* build_fanbeam(n, FanBeamGeometry{views, rays, source_radius, fan_angle})
 * (fanbeam.cpp:43-111, Siddon lengths in fp64 on the host), same validation
 * messages; the matrix is uploaded as fp32 values / int32 indices. */
ncsg_status ncsg_fanbeam_create(int n, int views, int rays, double source_radius,
                                double fan_angle, int device, ncsg_sparse** out);
/* FanBeamGeometry::defaults (fanbeam.cpp:10-17): radius n, fan covering the
 * corner circle. */
ncsg_status ncsg_fan_defaults(int n, double* source_radius, double* fan_angle);
/* SparseMap(n, views, rays, triplets) (sparse.cpp:9-45) from COO triplets. */
ncsg_status ncsg_sparse_create(int n, int views, int rays, int64_t nnz, const int64_t* rows,
                               const int64_t* cols, const double* vals, int device,
                               ncsg_sparse** out);
ncsg_status ncsg_sparse_destroy(ncsg_sparse* a);
int64_t ncsg_sparse_nnz(const ncsg_sparse* a);
/* SparseMap::forward / adjoint (sparse.cpp:55-71) on device arrays (batch
 * back to back) or fp64 host spans. */
ncsg_status ncsg_sparse_forward(const ncsg_sparse* a, const float* x, float* out, int batch,
                                void* stream);
ncsg_status ncsg_sparse_adjoint(const ncsg_sparse* a, const float* u, float* out, int batch,
                                void* stream);
ncsg_status ncsg_sparse_forward_host(const ncsg_sparse* a, const double* x, double* out,
                                     int batch);
ncsg_status ncsg_sparse_adjoint_host(const ncsg_sparse* a, const double* u, double* out,
                                     int batch);

/* GradMap::forward / adjoint (grad.hpp:17-28, grad.cpp:53-84): range layout is
 * the N x (N-1) horizontal block followed by the (N-1) x N vertical block. */
ncsg_status ncsg_grad_forward(int n, const float* x, float* out, int batch, void* stream);
ncsg_status ncsg_grad_adjoint(int n, const float* g, float* out, int batch, void* stream);
ncsg_status ncsg_grad_forward_host(int n, const double* x, double* out, int batch);
ncsg_status ncsg_grad_adjoint_host(int n, const double* g, double* out, int batch);

/* MaskApplier::apply (circulant.hpp:31-42, circulant.cpp:27-37):
 * out = Re(F^-1 (h .* F x)) for real N x N images; `mask` is the interleaved
 * complex N x N SpectralMask in DFT-bin order (circulant.hpp:16-25).  x and
 * out may alias.  Host fp64 in/out, device fp32 compute. */
ncsg_status ncsg_mask_apply_host(int n, const double* mask, const double* x, double* out,
                                 int batch, int device);

/* -------------------------------------------------------------------- solver
 * Problem + solver-configuration handle: the device-resident Engine of
 * solvers.cpp:84-265.  Problem kinds:
 *   NCSG_CT       blocks {1, R, QuadraticConj, b}, {beta/alpha, D,
 *                 ScaledL1Conj(lambda*alpha/beta)} -- assemble_problem
 *                 (pipeline.cpp:69-98)
 *   NCSG_DENOISE  blocks {1, I, QuadraticConj, b}, {beta/alpha, D, ...}
 *                 (the SplitProblem built in test_solvers.cpp:646-664)
 *   NCSG_PET      blocks {1, R, PoissonConj(counts = b, alpha), 0},
 *                 {beta/alpha, D, ...} -- assemble_problem with model "pet"
 *                 (pipeline.cpp:84-89; prox.cpp:9-13, 47-74)
 * With positivity != 0 a third block {1, I, NonnegConj} is appended
 * (pipeline.cpp:93-96).  `mask` (nullable) is the SolverConfig::mask -- the
 * metric surrogate C; NULL selects M = gamma I, i.e. pdhg_solve
 * (solvers.cpp:428-433).  The engine applies pinv(gamma + alpha*C) with
 * cfg.pinv_rel_tol (solvers.cpp:93-99).  `b` holds `batch` offsets back to
 * back (m each). */
typedef enum { NCSG_CT = 0, NCSG_DENOISE = 1, NCSG_PET = 2 } ncsg_kind;

typedef struct {
  int kind;          /* ncsg_kind */
  int n;             /* image side N */
  int n_angles;      /* CT only */
  int n_det;         /* CT only */
  int batch;         /* independent problems sharing geometry and mask */
  int positivity;    /* append {1, I, NonnegConj} */
  double alpha;      /* SolverConfig::alpha, also ModelParams::alpha */
  double beta;       /* ModelParams::beta: D-block weight beta/alpha */
  double lambda;     /* TV weight: ScaledL1Conj bound lambda*alpha/beta */
  double gamma;      /* SolverConfig::gamma */
  double pinv_rel_tol; /* SolverConfig::pinv_rel_tol (1e-12 by default) */
  const double* mask;  /* interleaved complex N*N, nullable (PDHG) */
  const double* b;     /* batch * m offsets (m = angles*det or N*N) */
  int angle_begin;   /* angle shard [angle_begin, angle_end) of this rank; */
  int angle_end;     /* 0,0 = all angles (single GPU) */
  int device;
  /* CT / PET data block on an explicit SparseMap (fan beam) instead of the
   * parallel-beam RadonMap (nullable; n_angles / n_det then come from it).
   * The handle must outlive the problem (the reference's shared_ptr). */
  const struct ncsg_sparse* sparse;
  /* Orbit sharding (shard_count > 1, n_angles % 4 == 0, angle_end == 0):
   * this rank owns the dihedral angle orbits whose representative index is
   * == shard_rank mod shard_count, so every shard keeps the orbit forward.
   * 0, 0 = off (contiguous angle_begin/angle_end sharding or none). */
  int shard_rank;
  int shard_count;
  /* SolverConfig::m_pinv_override / m_override (solvers.hpp:70-71) as
   * circulant operators: interleaved complex N*N symbols, nullable.  m_pinv
   * set selects the reference's Override mode (mode_from, solvers.cpp:75-79;
   * it wins over `mask`): the x-update applies Re(F^-1 (m_pinv . F A^T u))
   * as given (no gamma, no pseudoinverse), and M in the step seminorm and the
   * step-condition screen is the m_symbol circulant (required there, as
   * Engine::apply_m requires m_override, solvers.cpp:193-197). */
  const double* m_pinv;
  const double* m_symbol;
} ncsg_problem_desc;

typedef struct ncsg_problem ncsg_problem;

ncsg_status ncsg_problem_create(const ncsg_problem_desc* desc, ncsg_problem** out);
ncsg_status ncsg_problem_destroy(ncsg_problem* p);
/* SplitProblem::domain_size/range_size (solvers.hpp:28-29), per problem. */
size_t ncsg_problem_domain_size(const ncsg_problem* p);
size_t ncsg_problem_range_size(const ncsg_problem* p);
/* The handle's CUDA stream (cudaStream_t as void*). */
void* ncsg_problem_stream(const ncsg_problem* p);

/* SolverState{x, u, iter} (solvers.hpp:74-78) in/out, fp64 host arrays of
 * batch*N*N and batch*range_size.  NULL x or u means zeros (make_state,
 * solvers.cpp:406-411).  set_state also runs Engine::init (ax = A x,
 * solvers.cpp:118-122). */
ncsg_status ncsg_set_state(ncsg_problem* p, const double* x, const double* u, int64_t iter);
ncsg_status ncsg_get_state(ncsg_problem* p, double* x, double* u, int64_t* iter);
/* Device views of the state (fp32, batch-major) for zero-copy callers.
 * Writing u through the view: fetch it again (or ncsg_set_state) after the
 * write and before the next step -- the call marks the engine's derived copy
 * of u stale. */
float* ncsg_state_x(ncsg_problem* p);
float* ncsg_state_u(ncsg_problem* p);

/* `iters` x Engine::step (solvers.cpp:124-161), asynchronous on the handle's
 * stream; no host synchronisation.  Divergence (check_finite,
 * solvers.cpp:248-255) is flagged on the device and reported by the next
 * synchronising call. */
ncsg_status ncsg_step(ncsg_problem* p, int iters);
/* Same, replayed through a captured CUDA graph of `iters` steps. */
ncsg_status ncsg_step_graph(ncsg_problem* p, int iters);
/* Synchronise; returns NCSG_DIVERGED (and *iter, nullable) if any step so far
 * left the finite range. */
ncsg_status ncsg_sync(ncsg_problem* p, int64_t* diverged_iter);

/* Engine::objective = objective_from_ax(ax) (solvers.cpp:163,362-381), one
 * value per problem (out[batch]). */
ncsg_status ncsg_objective(ncsg_problem* p, double* out);
/* Engine::step_seminorm (solvers.cpp:166-202) of (dx, du) = (x_k - x_{k-1},
 * u_k - u_{k-1}) for the last step; NaN where the radicand is negative beyond
 * roundoff (solvers.cpp:305-316). */
ncsg_status ncsg_last_seminorm(ncsg_problem* p, double* out);

/* ConvergenceRecord row (solvers.hpp:82-86). */
typedef struct {
  int64_t iter;
  double objective;
  double rel_subopt;
  double seminorm_step;
  double wall_ms;
} ncsg_record_row;

/* ncs_solve / pdhg_solve (solvers.cpp:267-337, 423-433): max_iters steps from
 * the current state (reset iter to 0), recording every `record_every` steps
 * and at the end.  rows: capacity max_rows per problem, problem-major
 * (row r of problem q at rows[q*max_rows + r]); *n_rows = rows per problem.
 * f_star (nullable, one per problem) anchors rel_subopt as in the reference.
 * check_step_condition runs the 40-step power-method screen with `seed`
 * (SolverConfig::seed; solvers.cpp:206-245, 278) and writes its estimate into
 * *screen_est (nullable; NaN when not run).  As in the reference a positive
 * estimate is a warning for the caller, not an error. */
ncsg_status ncsg_solve(ncsg_problem* p, int max_iters, int record_every,
                       int check_step_condition, uint64_t seed, const double* f_star,
                       ncsg_record_row* rows, int max_rows, int* n_rows, double* screen_est);

/* admm_cg_solve (solvers.cpp:435-440): n_cg > 0 switches the x-update to
 * w = (1/alpha) cg(A^T A, A^T u, n_cg) (solvers.cpp:138-145, 442-463;
 * NormalMap, linear_map.cpp:57-61) -- M = alpha A^T A, so the problem must
 * have no mask; record iterations are scaled by n_cg (solvers.cpp:279) and
 * the step-condition screen is skipped (solvers.cpp:207).  Batch 1,
 * unsharded.  n_cg = 0 restores the circulant / PDHG x-update. */
ncsg_status ncsg_set_cg(ncsg_problem* p, int n_cg);

/* ------------------------------------------------------------- setup path
 * (the GPU versions of the reference's CPU setup.) */

/* calibrate_scale(NormalMap(R), radon_mask(N, 1, 1), n_samples, seed)
 * (circulant.cpp:142-169) -- the least-squares scale of the R^T R template
 * that measurement_mask (pipeline.cpp:100-110) passes to radon_mask for
 * parallel-beam geometry.  Probes are the reference's RngStream(seed, s)
 * normals (circulant.cpp:89-94), drawn on the host bit-for-bit. */
ncsg_status ncsg_calibrate_scale(const ncsg_radon* r, int n_samples, uint64_t seed,
                                 double* scale);

/* measurement_mask for a non-parallel geometry (pipeline.cpp:100-110):
 * empirical_mask(NormalMap(A), N, n_samples, seed).mask
 * (circulant.cpp:98-140) of a SparseMap, written as interleaved complex N*N
 * (the SpectralMask layout); *n_dead (nullable) = bins no probe resolved. */
ncsg_status ncsg_sparse_empirical_mask(const ncsg_sparse* a, int n_samples, uint64_t seed,
                                       double* mask, int* n_dead);

/* DC response of R^T R, <1, R^T R 1>/N^2: the dc value of radon_mask under the
 * rule the configs pin. */
ncsg_status ncsg_radon_dc_response(const ncsg_radon* r, double* dc);

/* Engine::screen_step_condition (solvers.cpp:206-245): `iters` steps of
 * power_method (solvers.cpp:466-484, start vector RngStream(seed, 0)) on
 * alpha A^T A - M + shift I, shift = gamma + alpha max|h| (gamma without a
 * mask).  *est = the estimated largest eigenvalue of alpha A^T A - M (the
 * reference warns when est > 1e-8 max(1, shift)); *shift (nullable).  With
 * gamma = 0 this is alpha * lambda_max(A^T A - C), the gamma rule of the
 * configs.  Unsharded problems only. */
ncsg_status ncsg_screen_step_condition(ncsg_problem* p, uint64_t seed, int iters, double* est,
                                       double* shift);

/* -------------------------------------------------------- multi-GPU phases
 * One NCS step split at its exchange points for angle-sharded execution
 * (SURVEY.md §8e): phase A computes this rank's partial A^T u (own angles of
 * R^T u_s, plus the D^T u_g / identity terms on rank 0 only) into the device
 * buffer returned by ncsg_atu_buffer(); the caller all-reduces that buffer
 * (NCCL over NVLink) and runs phase B, which applies M^+ (replicated FFT),
 * updates x, projects the own angles and updates the own dual blocks. */
ncsg_status ncsg_step_phase_a(ncsg_problem* p);
float* ncsg_atu_buffer(ncsg_problem* p);
/* Use a caller-owned device buffer (batch*N*N floats, e.g. a torch tensor that
 * NCCL all-reduces) as the A^T u exchange buffer; NULL reverts to internal. */
ncsg_status ncsg_set_atu_buffer(ncsg_problem* p, float* dev_ptr);
ncsg_status ncsg_step_phase_b(ncsg_problem* p);

/* ------------------------------------------------------------ measurement
 * Phase timing for bench.py: while profiling, every step records CUDA events
 * on the handle's stream between its phases (adjoint, FFT rows r2c + combine,
 * FFT columns, FFT rows c2r + x update, member images for the orbit forward,
 * forward, dual update);
 * ncsg_profile_end synchronises and returns the summed milliseconds per phase
 * and the number of profiled steps. */
ncsg_status ncsg_profile_begin(ncsg_problem* p);
ncsg_status ncsg_profile_end(ncsg_problem* p, double* phase_ms, int n_phase, int* steps);
/* ------------------------------------------------------------ multi-GPU
 * Communicator of a sharded problem.  A problem created with
 * an angle or orbit shard (angle_begin/angle_end, shard_rank/shard_count)
 * holds only its rank's rows of R; with a communicator attached, ncsg_step /
 * ncsg_step_graph* / ncsg_solve run the whole sharded iteration
 * (Engine::step, solvers.cpp:124-161, with the StackedMap::adjoint sum of
 * linear_map.cpp:47-55 across ranks):
 *   NCSG_XCHG_SLAB       partial A^T u -> reduce-scatter into N/P-row slabs ->
 *                        slab row FFT -> all-to-all -> column FFT . filter .
 *                        inverse -> all-to-all -> slab inverse rows + x update
 *                        -> all-gather of x (N % P == 0);
 *   NCSG_XCHG_ALLREDUCE  one all-reduce of the partial A^T u, replicated
 *                        circulant solve on every rank (latency-bound sizes);
 *   NCSG_XCHG_P2P        the slab step with every exchange fused into the
 *                        producing kernel over peer memory (NVLink: CUDA IPC
 *                        mappings of the peers' buffers): the A^T u assembly
 *                        stores each row into its owner's slot (reduce-
 *                        scatter), the row FFT stores each bin block into its
 *                        column owner (all-to-all), the column pass stores
 *                        back, the x update stores its rows into every rank's
 *                        image (all-gather); a stream-ordered barrier between
 *                        the kernels (NCCL or local transport, <= 8 ranks).
 * Objective / seminorm records and the divergence flags are reduced across
 * ranks.  (* graph capture only with the NCCL transport.)
 * Transports: NCCL (one communicator per rank, from a unique id shared by
 * the caller -- MPI, torch.distributed, a file), caller callbacks, or an
 * in-process group of ranks driven by host threads (tests, one GPU). */
typedef struct ncsg_comm ncsg_comm;
typedef enum { NCSG_F32 = 0, NCSG_F64 = 1, NCSG_I32 = 2 } ncsg_dtype;
typedef enum { NCSG_SUM = 0, NCSG_MIN = 1, NCSG_MAX = 2 } ncsg_redop;
typedef enum { NCSG_XCHG_ALLREDUCE = 0, NCSG_XCHG_SLAB = 1, NCSG_XCHG_P2P = 2 } ncsg_exchange;
/* Callback transport: device pointers; the library synchronises `stream`
 * before each call and expects the result complete in device memory on
 * return (a pageable H2D cudaMemcpy alone is not: synchronise after it, or
 * copy on `stream` and synchronise that); 0 = success. */
typedef struct ncsg_comm_ops {
  void* ctx;
  int rank, nranks;
  int (*all_reduce)(void* ctx, void* buf, size_t count, int dtype, int op, void* stream);
  int (*reduce_scatter)(void* ctx, const float* send, float* recv, size_t count, void* stream);
  int (*all_gather)(void* ctx, const float* send, float* recv, size_t count, void* stream);
  int (*all_to_all)(void* ctx, const float* send, float* recv, size_t count, void* stream);
} ncsg_comm_ops;
ncsg_status ncsg_nccl_unique_id(unsigned char id[128]);
ncsg_status ncsg_comm_create_nccl(const unsigned char id[128], int rank, int nranks, int device,
                                  ncsg_comm** out);
ncsg_status ncsg_comm_create_callbacks(const ncsg_comm_ops* ops, ncsg_comm** out);
/* nranks communicators of one in-process group (out[r] = rank r). */
ncsg_status ncsg_comm_create_local(int nranks, ncsg_comm** out);
/* A rank of a communicator whose collectives do nothing: times one rank's
 * kernels of the sharded step on one GPU (scaling projections; results are
 * meaningless). */
ncsg_status ncsg_comm_create_null(int rank, int nranks, ncsg_comm** out);
ncsg_status ncsg_comm_destroy(ncsg_comm* c);
/* Attach (or with NULL detach) the communicator; `exchange` = ncsg_exchange.
 * The communicator must outlive the problem's use of it. */
ncsg_status ncsg_problem_set_comm(ncsg_problem* p, ncsg_comm* c, int exchange);

/* The live plan of a problem (bench.py's roofline: the partial-sum counts
 * and sample count the per-kernel byte models use). */
typedef struct ncsg_plan_info {
  int orbit_forward;  /* 1: dihedral-orbit forward (fp_orbit_kernel) */
  int gather_adjoint; /* 1: pixel-driven orbit gather adjoint (bp_gather_kernel) */
  int fp_slots;       /* forward partial slots per ray summed by the dual update */
  int bp_partials;    /* adjoint partial images summed by the FFT row pass */
  int n_orbits;       /* dihedral orbits of the (own) angle set */
  int transposed_copy;/* 1: the x update also writes x^T (per-angle class-H forward) */
  int64_t samples;    /* bilinear samples per R application (own angles) */
  int64_t m0, g, range, batch;
  int dual_fused;     /* 1: the whole dual update runs in the inverse row pass (DENOISE) */
  int64_t adjoint_table_bytes; /* gather adjoint's window-weight table streamed per R^T
                                  application (8 B per (pixel, orbit)); 0: windows evaluated
                                  every step (NCSG_GA_WTAB=0, over NCSG_GA_WTAB_MAX_GB, or no
                                  memory) */
} ncsg_plan_info;
ncsg_status ncsg_problem_plan(const ncsg_problem* p, ncsg_plan_info* out);
/* Kernel launches issued by this library since load. */
int64_t ncsg_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* NCSG_H */
