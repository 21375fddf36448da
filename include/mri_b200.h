/*
 * mri_b200.h -- C-ABI of the B200-native MRI slow step (libmri_b200.so).
 *
 * Drop-in boundary for the data-parallel work inside one explicit MRI-GARK
 * slow step of the reference multirate toolkit.  Every entry point replaces a
 * reference interface, cited as proj/<file>:<line> under /root/reference:
 *
 *   mr_mri_step / mr_mri_integrate   <- multirate::mri_step / mri_integrate
 *                                       (include/multirate/mri.hpp:117-133,
 *                                        src/mri.cpp:323-435, :524-540)
 *   mr_coupling_load                 <- MriCoupling + finalize()/import_coupling
 *                                       (mri.hpp:32-62, mri.cpp:59-167, :590-626)
 *   mr_table_load                    <- ButcherTable (butcher.hpp:16-27) used by
 *                                       erk_step (erk.cpp:9-38)
 *   mr_fast_* / mr_slow_*            <- PartitionedSystem::f_fast / f_explicit
 *                                       (partitioned_system.hpp:25-61); the RHS
 *                                       callbacks become device "plugins"
 *   mr_fast_rhs / mr_slow_rhs        <- one RhsFn call (partitioned_system.hpp:17)
 *   mr_slow_implicit_diffusion       <- PartitionedSystem::f_implicit + the
 *                                       ImplicitStageSolver of IMEX couplings
 *                                       (partitioned_system.hpp:25-61,
 *                                        mri.cpp:378-421, solvers.cpp:34-208)
 *   mr_wrms_norm ... mr_all_finite   <- state_vector.hpp:119-176
 *   status codes                     <- ContractError / IntegrationError
 *                                       (state_vector.hpp:22-36)
 *
 * Conventions: plain pointers and sizes, no exceptions across the ABI, no
 * torch types.  Host state buffers use exactly the reference's species-major
 * layout Y[comp * ncell + cell], cell = (i * n1 + j) * n2 + k (axis 2
 * fastest), so a multirate::StateVector::data() can be passed directly.
 * Counters are uint64_t[8] in EvalCounters field order
 * (partitioned_system.hpp:66-79) and are ACCUMULATED like the reference's
 * by-reference EvalCounters.  Functions are synchronous on the context's
 * stream unless stated otherwise.
 */
#ifndef MRI_B200_H_
#define MRI_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mr_ctx mr_ctx;

/* status codes */
#define MR_OK 0
#define MR_CONTRACT 1    /* multirate::ContractError */
#define MR_INTEGRATION 2 /* multirate::IntegrationError (see fail_stage) */
#define MR_CUDA 3        /* CUDA / NCCL failure */

/* StageKind (mri.hpp:23) */
#define MR_STAGE_FAST_IVP 0
#define MR_STAGE_IMPLICIT_SOLVE 1
#define MR_STAGE_EXPLICIT_UPDATE 2

/* counters index (EvalCounters field order) */
#define MR_CNT_FAST_EVALS 0
#define MR_CNT_IMPLICIT_EVALS 1
#define MR_CNT_EXPLICIT_EVALS 2
#define MR_CNT_IMPLICIT_SOLVES 3
#define MR_CNT_NONLINEAR_ITERS 4
#define MR_CNT_LINEAR_ITERS 5
#define MR_CNT_PRECOND_SOLVES 6
#define MR_CNT_FAST_IVPS 7

/* ---------------- context / grid ---------------- */
int mr_ctx_create(int device, mr_ctx** out);
/* One process, several GPUs (the reference's single-threaded caller driving a
 * multi-GPU run): a DOMAIN context owning one slab context per listed device
 * (a device may repeat).  mr_grid_set on it (i0 = 0, n0_local = n0) splits
 * axis 0 into equal slabs in device order; every setup call is applied to all
 * slabs; upload/download scatter/gather the reference's species-major host
 * layout; a step runs the stage plan on every device, each slab on its own
 * stream, with the ghost planes copied peer-to-peer (cudaMemcpyPeerAsync over
 * NVLink, ordered by events) and the IMEX dot products summed in slab order --
 * bitwise the result of the same slabs as in-process virtual ranks.  Not
 * available on a domain: mr_state_device_ptr, the device-pointer reductions,
 * mr_mri_step_async, mr_comm_init.  mr_ctx_destroy frees the slabs. */
int mr_ctx_create_multi(const int* devices, int n, mr_ctx** out);
void mr_ctx_destroy(mr_ctx* ctx);
const char* mr_last_error(const mr_ctx* ctx);
int mr_version(void);

/* Grid of n0 x n1 x n2 global cells with n_comp components per cell.  This
 * context owns the slab of planes [i0, i0 + n0_local) along axis 0 (the
 * slowest axis); a single-GPU run passes i0 = 0, n0_local = n0. */
int mr_grid_set(mr_ctx* ctx, int n0, int n1, int n2, int n_comp, double length,
                int i0, int n0_local);

/* ---------------- method data ---------------- */
/* Raw coupling tables as in the v1 audit format (mri.cpp:560-626): c[s],
 * kind[s], gamma[n_deg][s][s], omega[n_deg][s][s].  Validated and finalized
 * with the reference's rules (mri.cpp:59-167). */
int mr_coupling_load(mr_ctx* ctx, int s, int n_deg, const double* c, const int* kind,
                     const double* gamma, const double* omega);
/* Same, from the reference's v1 text (export_coupling output). */
int mr_coupling_load_text(mr_ctx* ctx, const char* text);
/* Explicit inner table A[s][s], b[s], c[s] (s <= 6). */
int mr_table_load(mr_ctx* ctx, int s, const double* A, const double* b, const double* c);
/* MriMethodConfig::m (mri.hpp:64-68) */
int mr_set_substeps(mr_ctx* ctx, int m);

/* ---------------- physics plugins (PartitionedSystem) ---------------- */
/* fast = per-cell Arrhenius chemistry (n_comp must be S + 1, energy last).
 * species[S*5] = {W, a, b, h0, s0}; reactions[R*3] = {lnA, beta, Ea/Rc};
 * rspecies[R*4] = {r1, r2, p1, p2} (-1 = absent).  DESIGN.md "Physics". */
int mr_fast_chemistry(mr_ctx* ctx, int S, int R, double rho, const double* species,
                      const double* reactions, const int* rspecies);
/* fast = per-cell linear map f = A v, A[n_comp][n_comp] (test plugin; the
 * reference's LinearTwoRateOde, models.cpp:47-63, applied per cell) */
int mr_fast_linear(mr_ctx* ctx, const double* A);
int mr_fast_none(mr_ctx* ctx); /* f_fast absent */
/* slow = 3D periodic centred advection-diffusion, order 2/4/8.  vel_prof ==
 * NULL: uniform velocity u[3]; else tabulated profiles [3][2][nmax] with
 * u_d = P[d][0][coord of lower other axis] + P[d][1][coord of upper one]. */
int mr_slow_stencil(mr_ctx* ctx, int order, double diffusion, const double* u,
                    const double* vel_prof, int nmax);
int mr_slow_linear(mr_ctx* ctx, const double* A);
int mr_slow_none(mr_ctx* ctx);
/* IMEX split of the slow partition (call after mr_slow_stencil): adds
 * f_implicit = d_impl * L7 y (7-point periodic Laplacian, every component) and
 * solves the ImplicitSolve stages (I - gamma f_implicit) Y = known with
 * cg_iters iterations of Jacobi-preconditioned CG started at Y = known.
 * Required by couplings with ImplicitSolve stages or gamma terms; explicit
 * couplings on a split system are a ContractError (mri.cpp:310-319). */
int mr_slow_implicit_diffusion(mr_ctx* ctx, double d_impl, int cg_iters);
/* ImplicitStageSolver (mri.hpp:84-95) of the ImplicitSolve stages: the
 * NewtonConfig (solvers.hpp:19-23; defaults 1e-10, 0.1, 10) and the WRMS
 * weights (local slab, dof doubles, host; NULL = unit weights, freed when the
 * grid changes).  Newton runs as newton_solve (solvers.cpp:150-208) with the
 * fixed-iteration PCG in place of GMRES. */
int mr_newton_config(mr_ctx* ctx, double tolerance, double safety, int max_iters,
                     const double* weights);

/* ---------------- state ---------------- */
int mr_state_upload(mr_ctx* ctx, const double* host);   /* local slab, species-major */
int mr_state_download(mr_ctx* ctx, double* host);
/* device pointer of the current state (valid until the next step; NULL while
 * an asynchronous step is pending) */
double* mr_state_device_ptr(mr_ctx* ctx);
size_t mr_state_dof(const mr_ctx* ctx);

/* ---------------- stepping ---------------- */
/* One slow step t -> t+H of the device-resident state.  On MR_INTEGRATION the
 * state is unchanged and *fail_stage is the reference's
 * IntegrationError::stage_index (inner ERK stage index for a fast-IVP
 * failure, MRI stage index otherwise); counters then hold the reference's
 * partial counts up to the failure. */
int mr_mri_step(mr_ctx* ctx, double t, double H, uint64_t* counters, int* fail_stage);
int mr_mri_integrate(mr_ctx* ctx, double t0, double tf, double H, uint64_t* counters,
                     int* fail_stage);
/* Asynchronous step: enqueued on the context's stream after the work already
 * queued on `stream` (a cudaStream_t; NULL = the legacy default stream), and
 * `stream` is made to wait for it; returns without waiting.  The failure key,
 * the counters (accumulated into `counters`) and the state commit happen in
 * mr_mri_step_wait, which returns what mr_mri_step would have.  Until then the
 * context rejects state-touching calls with MR_CONTRACT.  IMEX couplings still
 * synchronise inside the step (host Newton decisions).  The result is
 * reachable (mr_state_device_ptr, mr_state_download) only after
 * mr_mri_step_wait: the commit is a host-side buffer swap. */
int mr_mri_step_async(mr_ctx* ctx, double t, double H, void* stream);
int mr_mri_step_wait(mr_ctx* ctx, uint64_t* counters, int* fail_stage);
/* End-to-end variant with HOST buffers: H2D of y_in, the step, D2H of y_out.
 * Where the plan allows (single slab, chemistry + order-8 stencil, n >= 64)
 * the copies are pipelined with the step's first and last ops in plane chunks
 * (pinned buffers overlap; results bitwise equal to mr_mri_step).  On failure
 * y_out keeps its previous contents (it is saved on the device first and
 * written back) and the device state is y_in. */
int mr_mri_step_host(mr_ctx* ctx, double t, double H, const double* y_in, double* y_out,
                     uint64_t* counters, int* fail_stage);
/* Host<->device bytes the last mr_mri_step_host moved (the pipelined step also
 * saves y_out to the device: 2 x state H2D). */
int mr_last_host_step_bytes(const mr_ctx* ctx, uint64_t* h2d, uint64_t* d2h);
/* ark_imex_step / ark_imex_integrate (proj/src/mri.cpp:437-557): the
 * single-rate ARK4(3)6L[2]SA IMEX pair (butcher.cpp:362-427) on the same
 * plugins -- explicit part f_fast + f_explicit, implicit f_implicit solved
 * by the device Newton-PCG (mr_slow_implicit_diffusion, mr_newton_config).
 * Counters accumulate like EvalCounters; state unchanged on failure. */
int mr_ark_imex_step(mr_ctx* ctx, double t, double H, uint64_t* counters, int* fail_stage);
int mr_ark_imex_integrate(mr_ctx* ctx, double t0, double tf, double H, uint64_t* counters,
                          int* fail_stage);
/* reference_solution (proj/src/erk.cpp:59-75): single-rate cash-karp5
 * (erk_integrate, :40-57) of the summed right-hand side f_fast + f_implicit +
 * f_explicit (partitioned_system.hpp:41-48) from t0 to tf with step h_ref, on
 * the device-resident state (the reference solution of the convergence /
 * efficiency studies, harness.cpp:411-429).  No counters.  On MR_INTEGRATION
 * the state is unchanged and *fail_stage is erk_step's stage index. */
int mr_reference_solution(mr_ctx* ctx, double t0, double tf, double h_ref, int* fail_stage);
/* erk_integrate (proj/src/erk.cpp:40-57) with an explicit table A[s][s]
 * (row-major), b[s], c[s] (s <= 12) on the summed right-hand side -- the
 * harness's "erk-<table>" method family (harness.cpp:346-355).  Adds one to
 * *n_explicit_evals per stage evaluation (erk.cpp:28; may be NULL).  On
 * MR_INTEGRATION the state is unchanged, *fail_stage is erk_step's stage index
 * and the count stops where erk_step threw. */
int mr_erk_integrate(mr_ctx* ctx, int s, const double* A, const double* b, const double* c,
                     double t0, double tf, double h, uint64_t* n_explicit_evals,
                     int* fail_stage);

/* Spectral deferred corrections on the device plugins (proj/src/sdc.cpp).
 * mr_sdc_integrate: sdc_integrate (sdc.cpp:267-281) of sum_rhs with an
 *   n-node rule -- nodes[n] on [0,1] and the integration matrix S[(n-1)*n]
 *   of lobatto_nodes(n) (sdc.hpp:17-27) -- and n_sweeps correction sweeps;
 *   evaluations counted into *n_evals like harness.cpp:356-366.
 * mr_mrsdc_load + mr_mrsdc_integrate: mrsdc_integrate (sdc.cpp:283-301) with
 *   the scheme of build_scheme(X, Y, Z, n_sweeps) (sdc.hpp:29-55) flattened:
 *   coarse_nodes[X], fine_nodes[n_fine], coarse_of_fine[n_fine],
 *   coarse_index_of_fine[n_fine] (-1: no coarse node), fine_row[(n_fine-1)*Y],
 *   application_offset[n_fine-1], coarse_row[(n_fine-1)*X]; counters
 *   (EvalCounters order) accumulate n_fast_evals / n_explicit_evals.
 * A non-finite node update fails with MR_INTEGRATION, fail_stage = the node
 * (the reference's IntegrationError stage_index), the state restored to the
 * call's input and the counters as far as the reference had counted.  The
 * node caches need 2 n_fine + 2 X + 5 state-sized buffers (MR_CUDA when the
 * device runs out of memory). */
int mr_sdc_integrate(mr_ctx* ctx, int n_nodes, const double* nodes, const double* S, int n_sweeps,
                     double t0, double tf, double H, uint64_t* n_evals, int* fail_stage);
int mr_mrsdc_load(mr_ctx* ctx, int X, int Y, int n_fine, int n_sweeps, const double* coarse_nodes,
                  const double* fine_nodes, const int* coarse_of_fine,
                  const int* coarse_index_of_fine, const double* fine_row,
                  const int* application_offset, const double* coarse_row);
int mr_mrsdc_integrate(mr_ctx* ctx, double t0, double tf, double H, uint64_t* counters,
                       int* fail_stage);
/* The reference's node sets, built on the host with its arithmetic (bitwise
 * equal): lobatto_nodes(n) (sdc.cpp:60-80; nodes[n], S[(n-1)*n]) and
 * build_scheme(X, Y, Z, .) (sdc.cpp:82-153; *n_fine = capacity in / count
 * out, all array pointers NULL = size query).  mr_mrsdc_build = build_scheme
 * + mr_mrsdc_load.  No device work: callable without a GPU. */
int mr_lobatto_rule(int n, double* nodes, double* S);
int mr_mrsdc_scheme(int X, int Y, int Z, int* n_fine, double* coarse_nodes, double* fine_nodes,
                    int* coarse_of_fine, int* coarse_index_of_fine, double* fine_row,
                    int* application_offset, double* coarse_row);
int mr_mrsdc_build(mr_ctx* ctx, int X, int Y, int Z, int n_sweeps);
/* Location of the last failure: MRI stage, fast substep, inner stage. */
int mr_last_failure(const mr_ctx* ctx, int* mri_stage, int* substep, int* inner_stage);

/* Single RHS evaluations ("Mode A": a reference RhsFn backed by the GPU).
 * Host buffers, local slab; slow evaluation exchanges halos when sharded. */
int mr_fast_rhs(mr_ctx* ctx, double t, const double* y, double* out);
int mr_slow_rhs(mr_ctx* ctx, double t, const double* y, double* out);
int mr_implicit_rhs(mr_ctx* ctx, double t, const double* y, double* out);

/* ---------------- reductions (device pointers, this context's stream) ---------------- */
int mr_wrms_norm(mr_ctx* ctx, const double* x, const double* w, size_t n, double* out);
int mr_two_norm(mr_ctx* ctx, const double* x, size_t n, double* out);
int mr_dot(mr_ctx* ctx, const double* x, const double* y, size_t n, double* out);
int mr_max_norm(mr_ctx* ctx, const double* x, size_t n, double* out);
int mr_max_norm_component(mr_ctx* ctx, const double* x, size_t n, size_t offset,
                          size_t count, double* out);
int mr_all_finite(mr_ctx* ctx, const double* x, size_t n, int* out);

/* ---------------- multi-GPU (slab decomposition over NCCL) ---------------- */
/* id128: ncclUniqueId bytes from rank 0 (broadcast by the caller).  Call before
 * mr_grid_set; the context then owns the slab [i0, i0 + n0_local) of its rank and
 * exchanges g = order/2 ghost planes per slow evaluation with grouped
 * ncclSend/ncclRecv.  nranks == 1 builds no communicator (periodic single
 * slab). */
int mr_nccl_unique_id(char* id128);
int mr_comm_init(mr_ctx* ctx, int nranks, int rank, const char* id128);
/* A one-rank NCCL communicator: the rank's whole NCCL code path (halo
 * send/recv to itself overlapped with the interior stencil, all-reduced
 * failure key, all-gathered CG dot products) on one GPU. */
int mr_comm_init_loopback(mr_ctx* ctx);

/* In-process "virtual ranks" (one GPU, several slab contexts sharing the
 * device): the same slab code path with halos copied device-to-device. */
int mr_group_step(mr_ctx** ctxs, int n, double t, double H, uint64_t* counters,
                  int* fail_stage);

/* ---------------- host-side generators (seeded, bit-reproducible) ---------------- */
int mr_mechanism_generate(uint64_t seed, int S, int R, double* species, double* reactions,
                          int* rspecies);
/* initial condition of the local slab [i0, i0+n0_local) of an n0 x n1 x n2 grid */
int mr_initial_condition(uint64_t seed, int S, double rho, const double* species, int n0,
                         int n1, int n2, double length, int i0, int n0_local, double* Y,
                         int threads);
int mr_velocity_profiles(uint64_t seed, int n0, int n1, int n2, double length, double* prof);

/* ---------------- host-only method inspection (no GPU needed) ---------------- */
/* Parse + finalize a v1 coupling text with the reference's rules; fills the
 * stage count, kinds, slow-evaluation schedule and substeps per stage for m.
 * Returns MR_CONTRACT with the reference's message in err on violation. */
int mr_coupling_inspect(const char* text, int m, int* s, int* kinds, int* eval_at, int* n_sub,
                        char* err, size_t errlen);
/* EvalCounters increments of one successful slow step (plan of the device
 * stage loop) for an inner table of s_f stages. */
int mr_step_counts(const char* text, int s_f, int m, int fast_present, int slow_present,
                   uint64_t* counters, char* err, size_t errlen);

/* ---------------- instrumentation ---------------- */
/* cudaStream_t of the context (for event timing by the caller) */
void* mr_stream(mr_ctx* ctx);
/* number of kernels this context launched since creation */
uint64_t mr_launch_count(const mr_ctx* ctx);
/* fp64 work accounting of one chemistry RHS evaluation */
double mr_chem_flops_per_eval(const mr_ctx* ctx);
/* measured fp64 FMA peak of this GPU (DFMA chain microbenchmark), TFLOP/s */
int mr_fp64_peak(mr_ctx* ctx, double* tflops);
/* record CUDA events around every launch class of a step (default off) */
int mr_set_profiling(mr_ctx* ctx, int enable);
/* per-kernel-class device time of the last step (ms), from CUDA events */
int mr_last_step_profile(const mr_ctx* ctx, double* chem_ms, double* slow_ms, double* other_ms);

#ifdef __cplusplus
}
#endif
#endif
