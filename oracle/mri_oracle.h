/*
 * oracle/mri_oracle.h -- CPU ORACLE (test infrastructure only).
 *
 * This is the checker, never the product: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The
 * product path (paper_2211_03293_b200/) never links or calls anything here.
 *
 * Contents:
 *   1. A plain-C restatement of the reference's explicit MRI slow step
 *      (/root/reference/proj/src/mri.cpp, erk.cpp, butcher.cpp,
 *      include/multirate/state_vector.hpp), each function citing the
 *      reference file:line it follows.  Operation order is kept identical so
 *      that, built with -ffp-contract=off, it reproduces the reference
 *      stepper bit-for-bit (checked against oracle/_ref, which is the
 *      reference's own sources compiled by oracle/Makefile).
 *   2. The builder-defined physics plugged into the reference's
 *      PartitionedSystem callbacks (the reference ships only a Brusselator
 *      surrogate, proj/src/models.cpp:112-274): seeded synthetic Arrhenius
 *      mechanism, per-cell chemistry RHS with temperature from energy,
 *      3D periodic 2/4/8-order advection-diffusion stencil, seeded initial
 *      condition and velocity field.  DESIGN.md section "Physics" is the
 *      normative statement of these formulas; this file is their executable
 *      CPU form.  Parity of the physics is pinned by this oracle (there is
 *      no reference implementation of it -- SURVEY.md 8(c)); parity of the
 *      stepper is pinned by the compiled reference (oracle/_ref).
 */
#ifndef MRI_ORACLE_H_
#define MRI_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MAX_STAGES 16
#define ORC_MAX_DEG 4
#define ORC_MAX_TABLE 8

/* status codes (mirror the reference's exception classes) */
#define ORC_OK 0
#define ORC_CONTRACT 1     /* ContractError, state_vector.hpp:22-25 */
#define ORC_INTEGRATION 2  /* IntegrationError, state_vector.hpp:30-36 */

/* StageKind, mri.hpp:23 */
#define ORC_FAST_IVP 0
#define ORC_IMPLICIT_SOLVE 1
#define ORC_EXPLICIT_UPDATE 2

/* ButcherTable, butcher.hpp:16-27 (explicit tables only on this path) */
typedef struct {
  int s;
  int order;
  int is_explicit;
  double A[ORC_MAX_TABLE][ORC_MAX_TABLE];
  double b[ORC_MAX_TABLE];
  double c[ORC_MAX_TABLE];
} orc_table;

/* MriCoupling, mri.hpp:32-62 */
typedef struct {
  char name[64];
  int s;
  int ndeg_gamma, ndeg_omega; /* gamma.size(), omega.size() */
  int order;
  double c[ORC_MAX_STAGES];
  int kind[ORC_MAX_STAGES];
  double gamma[ORC_MAX_DEG][ORC_MAX_STAGES][ORC_MAX_STAGES];
  double omega[ORC_MAX_DEG][ORC_MAX_STAGES][ORC_MAX_STAGES];
  /* derived by finalize (mri.cpp:59-167) */
  double gbar[ORC_MAX_STAGES][ORC_MAX_STAGES];
  double wbar[ORC_MAX_STAGES][ORC_MAX_STAGES];
  int eval_explicit_at[ORC_MAX_STAGES];
  int fI_referenced[ORC_MAX_STAGES];
} orc_coupling;

/* EvalCounters, partitioned_system.hpp:66-79 (same field order) */
typedef struct {
  uint64_t n_fast_evals, n_implicit_evals, n_explicit_evals, n_implicit_solves,
      n_nonlinear_iters, n_linear_iters, n_precond_solves, n_fast_ivps;
} orc_counters;

/* ---------------- physics: mechanism ---------------- */
/* Packed mechanism, identical to the product C-ABI (include/mri_b200.h):
 *   species[S*5]   = {W, a, b, h0, s0}          per species
 *   reactions[R*3] = {lnA, beta, EaR}           per reaction (EaR = Ea/Rc [K])
 *   rspecies[R*4]  = {r1, r2, p1, p2}           species index or -1        */
typedef struct {
  int S, R;
  double rho;
  double *species, *reactions;
  int *rspecies;
  /* derived (orc_mech_derive) */
  double *rhoW, *Wrho, *c0, *c1, *c2, *hb;
  int *dnu;
  int *csr_off, *csr_rxn, *csr_sgn; /* species <- reaction incidence, j ascending */
} orc_mech;

int orc_mech_generate(uint64_t seed, int S, int R, double* species,
                      double* reactions, int* rspecies);
int orc_mech_init(orc_mech* m, int S, int R, double rho, const double* species,
                  const double* reactions, const int* rspecies);
void orc_mech_free(orc_mech* m);

/* per-cell chemistry RHS on a species-major state with ncomp = S+1 (energy last) */
void orc_chem_rhs(const orc_mech* m, size_t ncell, const double* Y, double* out);
double orc_temperature(const orc_mech* m, const double* v, size_t stride);

/* ---------------- physics: grid, stencil, IC ---------------- */
typedef struct {
  int n0, n1, n2;  /* cells per axis; axis 2 fastest (cell=(i*n1+j)*n2+k) */
  double length;   /* cube side L (dx = L/n per axis) */
  int ncomp;
  int order;       /* 2, 4 or 8 */
  double diffusion;
  int vel_kind;    /* 0 uniform, 1 tabulated profiles */
  double u_const[3];
  /* vel_kind 1: u_d(cell) = P[d][0][coord of axis a0(d)] + P[d][1][coord of axis a1(d)],
   * a0 < a1 the two axes != d; profile arrays of length n_axis */
  const double* prof[3][2];
  /* IMEX split (config C5): f_explicit = advection only (diffusion above must be
   * 0), f_implicit = d_impl * L7 (7-point Laplacian); ImplicitSolve stages
   * run newton_solve's iteration (solvers.cpp:150-208, unit weights) with
   * cg_iters iterations of Jacobi-preconditioned CG as the linear solver */
  int imex;
  double d_impl;
  int cg_iters;
  double newton_tol;     /* NewtonConfig (solvers.hpp:19-23) */
  double newton_safety;
  int newton_max_iters;
  const double* newton_w; /* ImplicitStageSolver::weights (mri.hpp:84-95); NULL = unit */
} orc_grid;

void orc_stencil_rhs(const orc_grid* g, const double* Y, double* out);
int orc_velocity_profiles(uint64_t seed, int n0, int n1, int n2, double length,
                          double* prof /* [3][2][nmax] with nmax=max(n) */);
void orc_initial_condition(uint64_t seed, const orc_mech* m, int n0, int n1, int n2,
                           double length, int i0_global, int n0_global, double* Y);

/* ---------------- stepper ---------------- */
int orc_table_lookup(const char* name, orc_table* t);
int orc_coupling_finalize(orc_coupling* cp, char* err, size_t errlen);
int orc_coupling_from_mis(const char* name, const orc_table* base, int order,
                          int split_widest, orc_coupling* out);
int orc_coupling_import(const char* text, orc_coupling* out, char* err, size_t errlen);
int orc_coupling_export(const orc_coupling* cp, char* buf, size_t buflen);
int orc_coupling_register(const char* name, orc_coupling* out);

/* problem = PartitionedSystem analogue with builder plugins */
#define ORC_FAST_NONE 0
#define ORC_FAST_CHEM 1
#define ORC_FAST_LINEAR 2
#define ORC_SLOW_NONE 0
#define ORC_SLOW_STENCIL 1
#define ORC_SLOW_LINEAR 2
typedef struct {
  size_t ncell;
  int ncomp;
  int fast_kind, slow_kind;
  const orc_mech* mech;
  const orc_grid* grid;
  const double* fast_A; /* ncomp x ncomp, applied per cell */
  const double* slow_A;
  int threads;          /* >1: OpenMP-free pthread split of the RHS loops */
} orc_problem;

void orc_fast_rhs(const orc_problem* p, double t, const double* y, double* out);
void orc_implicit_rhs(const orc_problem* p, double t, const double* y, double* out);
void orc_slow_rhs(const orc_problem* p, double t, const double* y, double* out);

int orc_mri_step(const orc_coupling* cp, const orc_table* fast, int m,
                 const orc_problem* p, double t, double* y, double H,
                 orc_counters* cnt, int* fail_stage, char* err, size_t errlen);
int orc_mri_integrate(const orc_coupling* cp, const orc_table* fast, int m,
                      const orc_problem* p, double t0, double tf, double H,
                      double* y, orc_counters* cnt, int* fail_stage, char* err,
                      size_t errlen);

/* ---------------- flat session API (ctypes-friendly) ---------------- */
typedef struct {
  int n0, n1, n2;        /* local grid (slab) */
  int n0_global, i0_global;
  int ncomp;
  double length;
  int fast_kind, slow_kind;
  int S, R;
  double rho;
  const double* species;
  const double* reactions;
  const int* rspecies;
  const double* fast_A;
  const double* slow_A;
  int order;
  double diffusion;
  int vel_kind;
  double u_const[3];
  const double* prof;    /* [3][2][prof_nmax] */
  int prof_nmax;
  int threads;
  int imex;              /* 1: f_implicit = d_impl * L7, f_explicit = advection */
  double d_impl;
  int cg_iters;
  double newton_tol;
  double newton_safety;
  int newton_max_iters;
  const double* newton_w;
} orc_sys_cfg;

typedef struct orc_sys orc_sys;
orc_sys* orc_sys_create(const orc_sys_cfg* cfg);
void orc_sys_destroy(orc_sys* s);
const orc_problem* orc_sys_problem(const orc_sys* s);
void orc_sys_set_threads(orc_sys* s, int threads);
int orc_sys_fast_rhs(orc_sys* s, double t, const double* y, double* out);
int orc_sys_slow_rhs(orc_sys* s, double t, const double* y, double* out);
int orc_sys_implicit_rhs(orc_sys* s, double t, const double* y, double* out);
int orc_sys_initial_condition(orc_sys* s, uint64_t seed, double* Y);
/* coupling: registered name ("mis-kw3") or v1 audit text; fast table by name */
int orc_sys_mri_step(orc_sys* s, const char* coupling, const char* fast_table, int m,
                     double t, double H, double* y, uint64_t* counters, int* fail_stage,
                     char* err, size_t errlen);
/* ark_imex_step / ark_imex_integrate (proj/src/mri.cpp:437-557), ARK4(3)6L[2]SA */
int orc_ark_imex_step(const orc_problem* p, double t, double* y, double H, orc_counters* cnt,
                      int* fail_stage, char* err, size_t errlen);
int orc_ark_imex_integrate(const orc_problem* p, double t0, double tf, double H, double* y,
                           orc_counters* cnt, int* fail_stage, char* err, size_t errlen);
int orc_sys_ark_imex_integrate(orc_sys* s, double t0, double tf, double H, double* y,
                               uint64_t* counters, int* fail_stage, char* err, size_t errlen);
/* erk_integrate (proj/src/erk.cpp:40-57) of a named explicit table on sum_rhs;
   *evals += stage evaluations (erk.cpp:28) */
int orc_erk_integrate(const orc_problem* p, const char* table, double t0, double tf, double h,
                      double* y, uint64_t* evals, int* fail_stage, char* err, size_t errlen);
int orc_sys_erk_integrate(orc_sys* s, const char* table, double t0, double tf, double h, double* y,
                          uint64_t* evals, int* fail_stage, char* err, size_t errlen);
/* reference_solution (proj/src/erk.cpp:59-75): cash-karp5 on sum_rhs */
int orc_reference_solution(const orc_problem* p, double t0, double tf, double h, double* y,
                           int* fail_stage, char* err, size_t errlen);
int orc_sys_reference_solution(orc_sys* s, double t0, double tf, double h, double* y,
                               int* fail_stage, char* err, size_t errlen);
int orc_sys_mri_integrate(orc_sys* s, const char* coupling, const char* fast_table, int m,
                          double t0, double tf, double H, double* y, uint64_t* counters,
                          int* fail_stage, char* err, size_t errlen);
int orc_coupling_load(const char* spec, orc_coupling* out, char* err, size_t errlen);

/* ---------------- vector contract, state_vector.hpp:119-176 ---------------- */
double orc_wrms_norm(const double* x, const double* w, size_t n);
double orc_two_norm(const double* x, size_t n);
double orc_dot(const double* x, const double* y, size_t n);
double orc_max_norm(const double* x, size_t n);
double orc_max_norm_component(const double* x, size_t offset, size_t count);
int orc_all_finite(const double* x, size_t n);

/* splitmix64 helpers shared by the generators */
uint64_t orc_splitmix64_next(uint64_t* state);
uint64_t orc_mix64(uint64_t z);

#ifdef __cplusplus
}
#endif
#endif
