// mri_b200.cu -- host side of libmri_b200.so: context, method data, the MRI
// slow-step stage loop and the C-ABI (include/mri_b200.h).
//
// The stage loop mirrors multirate::mri_step (proj/src/mri.cpp:323-435) for
// fully explicit couplings, but instead of one full-vector pass per vector op
// it compiles the coupling into a short plan of fused device launches:
//
//   SLOW(j)   K2 stencil: fE_j = f_slow(Y_j)        (eval_slow_at, mri.cpp:339-349)
//   CHAIN     K1: maximal run of cell-local stages between two slow evaluations
//             (fast IVPs with their forcing, explicit updates, finite checks)
//   UPDATE    K3: explicit update when a run holds no fast IVP
//
// Counters follow the reference's increment rules exactly (mri.cpp:342, :347,
// :378; erk.cpp:28), including partial counts on an IntegrationError.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: no-ops unless a tool attaches
#include "nccl_shim.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/mri_b200.h"
#include "common.cuh"

namespace {

constexpr double kRu = 8.31446261815324e7;  // erg/(mol K)
constexpr double kPatm = 1.01325e6;         // dyn/cm^2
constexpr double kConsistencyTol = 1.0e-12; // mri.cpp:14
constexpr int kMaxStages = 16;

struct Coupling {
  std::string name;
  int s = 0;
  int ndeg_g = 0, ndeg_o = 0;
  double c[kMaxStages] = {};
  int kind[kMaxStages] = {};
  std::vector<double> gamma, omega;  // [deg][s][s]
  double gbar[kMaxStages][kMaxStages] = {};
  double wbar[kMaxStages][kMaxStages] = {};
  bool eval_at[kMaxStages] = {};
  bool fE_ref[kMaxStages] = {};
  bool fI_ref[kMaxStages] = {};
  bool implicit = false;
  double G(int k, int i, int j) const { return gamma[((size_t)k * s + i) * s + j]; }
  double W(int k, int i, int j) const { return omega[((size_t)k * s + i) * s + j]; }
  int degrees() const { return std::max(ndeg_g, ndeg_o); }
};

// MriCoupling::finalize (proj/src/mri.cpp:59-167): validation + derived data
bool finalize(Coupling& cp, std::string& err)
{
  const int s = cp.s;
  auto bad = [&](const std::string& m) {
    err = "MriCoupling " + cp.name + ": " + m;
    return false;
  };
  if (s < 2 || s > kMaxStages) return bad("inconsistent sizes");
  if (std::fabs(cp.c[0]) > 0.0 || std::fabs(cp.c[s - 1] - 1.0) > kConsistencyTol)
    return bad("need c[0]=0 and c[s-1]=1");
  for (int i = 1; i < s; ++i)
    if (cp.c[i] < cp.c[i - 1] - kConsistencyTol) return bad("abscissae decrease");
  for (int pass = 0; pass < 2; ++pass) {
    const int nd = pass == 0 ? cp.ndeg_g : cp.ndeg_o;
    for (int k = 0; k < nd; ++k)
      for (int i = 0; i < s; ++i)
        for (int j = i; j < s; ++j) {
          const double v = pass == 0 ? cp.G(k, i, j) : cp.W(k, i, j);
          const bool diag_ok = pass == 0 && j == i && cp.kind[i] == MR_STAGE_IMPLICIT_SOLVE;
          if (v != 0.0 && !diag_ok)
            return bad(std::string(pass == 0 ? "gamma" : "omega") +
                       " not lower triangular at stage " + std::to_string(i));
        }
  }
  std::memset(cp.gbar, 0, sizeof(cp.gbar));
  std::memset(cp.wbar, 0, sizeof(cp.wbar));
  for (int k = 0; k < cp.ndeg_g; ++k) {
    const double w = 1.0 / static_cast<double>(k + 1);
    for (int i = 0; i < s; ++i)
      for (int j = 0; j < s; ++j) cp.gbar[i][j] += w * cp.G(k, i, j);
  }
  for (int k = 0; k < cp.ndeg_o; ++k) {
    const double w = 1.0 / static_cast<double>(k + 1);
    for (int i = 0; i < s; ++i)
      for (int j = 0; j < s; ++j) cp.wbar[i][j] += w * cp.W(k, i, j);
  }
  bool has_g = false, has_o = false;
  for (double v : cp.gamma) has_g |= v != 0.0;
  for (double v : cp.omega) has_o |= v != 0.0;
  cp.implicit = has_g;
  for (int i = 1; i < s; ++i) {
    const double dc = cp.c[i] - cp.c[i - 1];
    if (cp.kind[i] == MR_STAGE_FAST_IVP) {
      if (dc <= 0.0) return bad("fast-ivp stage " + std::to_string(i) + " has dc <= 0");
    } else {
      if (dc > kConsistencyTol)
        return bad("stage " + std::to_string(i) + " solves/updates with dc > 0");
      if (cp.kind[i] == MR_STAGE_IMPLICIT_SOLVE && cp.gbar[i][i] == 0.0)
        return bad("implicit stage " + std::to_string(i) + " has zero diagonal");
    }
    for (int pass = 0; pass < 2; ++pass) {
      const bool used = pass == 0 ? has_g : has_o;
      if (!used) continue;
      const int nd = pass == 0 ? cp.ndeg_g : cp.ndeg_o;
      double bar_sum = 0.0;
      for (int k = 0; k < nd; ++k) {
        double rk = 0.0;
        for (int j = 0; j < s; ++j) rk += pass == 0 ? cp.G(k, i, j) : cp.W(k, i, j);
        bar_sum += rk / static_cast<double>(k + 1);
        if (k >= 1 && std::fabs(rk) > kConsistencyTol)
          return bad("degree-" + std::to_string(k) + " row sum nonzero at stage " +
                     std::to_string(i));
      }
      if (std::fabs(bar_sum - dc) > kConsistencyTol)
        return bad("row integral != dc at stage " + std::to_string(i));
    }
  }
  for (int i = 0; i < s; ++i) cp.fI_ref[i] = cp.fE_ref[i] = false;
  for (int k = 0; k < cp.ndeg_g; ++k)
    for (int i = 0; i < s; ++i)
      for (int j = 0; j < i; ++j)
        if (cp.G(k, i, j) != 0.0) cp.fI_ref[j] = true;
  for (int k = 0; k < cp.ndeg_o; ++k)
    for (int i = 0; i < s; ++i)
      for (int j = 0; j < i; ++j)
        if (cp.W(k, i, j) != 0.0) cp.fE_ref[j] = true;
  for (int i = 0; i < s; ++i) cp.eval_at[i] = cp.fE_ref[i];
  if (!has_g && has_o) cp.eval_at[s - 1] = true;  // mri.cpp:162-166
  return true;
}

// ---------------------------------------------------------------------------
struct Op {
  enum Type { SLOW = 0, COUNT_SLOW = 1, CHAIN = 2, UPDATE = 3, MISSING = 4, IMPL = 5, SOLVE = 6 } type;
  int stage = 0;
  std::vector<int> stages;  // CHAIN
};

struct Plan {
  std::vector<Op> ops;
  int slot_of[kMaxStages];   // fE_j
  int islot_of[kMaxStages];  // fI_j (IMEX couplings)
  int nslots = 0;
};

}  // namespace

#ifndef MR_HEAD_CHUNKS
#define MR_HEAD_CHUNKS 32  // measured (C4 e2e over the device step): 16 -> 66 ms, 32 -> 42 ms, 64 -> 79 ms
#endif
constexpr int kHeadChunks = MR_HEAD_CHUNKS;  // plane chunks of a pipelined host-buffer step

struct mr_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  // grid
  bool has_grid = false;
  int n0 = 0, n1 = 0, n2 = 0, ncomp = 0, i0 = 0, n0l = 0;
  double length = 1.0;
  size_t plane = 0, ncell = 0, dof = 0;
  // method
  bool has_coupling = false, has_table = false;
  Coupling cp;
  TableDev tab{};
  int m = 1;
  // plugins
  int fast_kind = -1, slow_kind = -1;
  int S = 0, R = 0;
  double rho = 0.0;
  ChemParams* chemP = nullptr;  // host copy, passed by value to the kernels
  double chem_flops = 0.0;
  std::vector<void*> chem_bufs;
  LinDev fastA{}, slowA{};
  int order = 2, M = 1;
  double D = 0.0;
  double u[3] = {0, 0, 0};
  int vel_kind = 0;
  double* d_prof = nullptr;
  int nmax = 0;
  // IMEX implicit partition: f_I = d_impl L7, fixed-iteration PCG solves
  bool imex = false;
  double d_impl = 0.0;
  int cg_iters = 0;
  double *cg_known = nullptr, *cg_r = nullptr, *cg_z = nullptr, *cg_p = nullptr, *cg_q = nullptr;
  double* cg_part = nullptr;    // block partials of a dot product
  double* cg_part2 = nullptr;   // second set (the residual kernel reduces two sums)
  double* cg_sc = nullptr;      // [0] rz, [1] pAp, [2] rz_new, [3] sum (G w)^2
  double* cg_gather = nullptr;  // [nranks] for the cross-rank fixed-order sum
  double* newton_w = nullptr;   // ImplicitStageSolver::weights (local slab); null = unit
  std::vector<double*> rs_bufs;  // reference solution: k[6], stage, f_fast, f_implicit
  std::vector<double*> sdc_bufs; // (multirate) SDC: caches, node states, scratch, backup
  struct SdcScheme {             // mr_mrsdc_load: the reference's MrsdcScheme, flattened
    bool loaded = false;
    int X = 0, Y = 0, n_fine = 0, n_sweeps = 0;
    std::vector<double> coarse_nodes, fine_nodes, fine_row, coarse_row;
    std::vector<int> coarse_of_fine, coarse_index_of_fine, application_offset;
  } mrsdc;
  std::vector<double*> ark_bufs; // ARK-IMEX: fE[6], fI[6], f_fast
  double newton_tol = 1.0e-10;  // NewtonConfig defaults (solvers.hpp:19-23)
  double newton_safety = 0.1;
  int newton_max = 10;
  int solve_evals[kMaxStages] = {};  // this step: residual evaluations per solve stage
  int solve_nl[kMaxStages] = {};     // this step: Newton iterations per solve stage
  // buffers
  double* y_state = nullptr;
  double* y_work = nullptr;
  std::vector<double*> slots;
  double *send_lo = nullptr, *send_hi = nullptr, *recv_lo = nullptr, *recv_hi = nullptr;
  size_t halo_elems = 0;
  double *scr_in = nullptr, *scr_out = nullptr;
  double* y_backup = nullptr;  // state at the start of an integrate call (restored on failure)
  unsigned long long* d_fail = nullptr;
  unsigned long long* h_fail = nullptr;
  double* d_red = nullptr;  // partials + out
  double* h_red = nullptr;
  bool state_valid = false;
  // comm
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
  // mr_mri_step_host: the upload of the caller's state rides on the step's
  // first stencil + fused chain, plane chunk by plane chunk (domain_step)
  const double* host_in = nullptr;
  double* host_out = nullptr;  // ... and the result streams out during its last ops
  bool out_streamed = false;   // y_out was backed up to y_backup and is being written
  bool pipeline_nccl = false;  // pipelined host step also on an NCCL rank (mr_debug_pipeline_nccl)
  uint64_t host_h2d = 0, host_d2h = 0;  // bytes the last host-buffer step moved
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_copy[kHeadChunks + 1] = {};
  cudaStream_t comm_stream = nullptr;  // halo exchange overlapped with the interior stencil
  cudaEvent_t ev_pack = nullptr, ev_halo = nullptr;
  // instrumentation
  uint64_t launches = 0;
  bool profile = false;
  double prof_chem = 0, prof_slow = 0, prof_other = 0;
  std::vector<cudaEvent_t> ev_pool;
  int fail_mri = -1, fail_sub = -1, fail_inner = -1;
  // mr_mri_step_async: everything mr_mri_step_wait needs to finish the step
  struct Pending {
    bool active = false;
    Plan plan;
    double t = 0.0, H = 0.0;
    int missing_stage = -1;
    unsigned long long host_key = 0;
    std::vector<std::pair<int, size_t>> timed;
    const double* ycur = nullptr;
  } pending;
  cudaEvent_t ev_async_in = nullptr, ev_async_out = nullptr;
  // multi-device domain (mr_ctx_create_multi): a domain context owns one slab
  // context per device, slabs along axis 0 in device order.  A slab of a
  // domain launches on its own stream and device; its neighbours' copies of
  // its ghost planes and the slab-ordered dot products are ordered by events.
  std::vector<mr_ctx*> slabs;
  bool in_domain = false;
  cudaEvent_t ev_send = nullptr;  // this slab's ghost planes are packed
  cudaEvent_t ev_recv = nullptr;  // this slab has copied its neighbours' planes
  cudaEvent_t ev_dot = nullptr;   // this slab's dot-product partial is final
  bool recv_recorded = false;
};

namespace {

int set_err(mr_ctx* c, int code, const std::string& msg)
{
  if (c) c->err = msg;
  return code;
}

// NVTX range for the host-side stage loop (nsys / ncu --nvtx show the MRI
// stage structure of a step; free when no tool is attached)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  NvtxRange(const char* kind, int a, int b = -1)
  {
    char buf[64];
    if (b >= 0)
      std::snprintf(buf, sizeof(buf), "%s %d..%d", kind, a, b);
    else
      std::snprintf(buf, sizeof(buf), "%s %d", kind, a);
    nvtxRangePushA(buf);
  }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// stream / device of slab c inside a step whose shared stream is st: the slabs
// of a multi-device domain each run on their own stream and device, the
// in-process virtual ranks of one device share the first slab's stream
inline cudaStream_t sst(const mr_ctx* c, cudaStream_t st) { return c->in_domain ? c->stream : st; }
inline void sdev(const mr_ctx* c)
{
  if (c->in_domain) cudaSetDevice(c->device);
}

#define MR_CUDA_TRY(ctx, call)                                                            \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return set_err(ctx, MR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));    \
  } while (0)

#define MR_NCCL_TRY(ctx, call)                                                            \
  do {                                                                                     \
    if (!nccl_api().ok) return set_err(ctx, MR_CUDA, "NCCL (libnccl.so.2) not available");  \
    ncclResult_t r_ = (nccl_api().call);                                                   \
    if (r_ != ncclSuccess)                                                                 \
      return set_err(ctx, MR_CUDA, std::string(#call) + ": " + nccl_api().GetErrorString(r_)); \
  } while (0)

void free_dev(void*& p)
{
  if (p) cudaFree(p);
  p = nullptr;
}

template <class T>
void free_dev_t(T*& p)
{
  void* q = p;
  free_dev(q);
  p = nullptr;
}

void free_state(mr_ctx* c)
{
  free_dev_t(c->y_state);
  free_dev_t(c->y_work);
  for (auto& p : c->slots) free_dev_t(p);
  c->slots.clear();
  free_dev_t(c->send_lo);
  free_dev_t(c->send_hi);
  free_dev_t(c->recv_lo);
  free_dev_t(c->recv_hi);
  free_dev_t(c->scr_in);
  free_dev_t(c->scr_out);
  free_dev_t(c->y_backup);
  free_dev_t(c->cg_known);
  free_dev_t(c->cg_r);
  free_dev_t(c->cg_z);
  free_dev_t(c->cg_p);
  free_dev_t(c->cg_q);
  free_dev_t(c->newton_w);  // weights are per grid
  for (auto& p : c->rs_bufs) free_dev_t(p);
  c->rs_bufs.clear();
  for (auto& p : c->sdc_bufs) free_dev_t(p);
  c->sdc_bufs.clear();
  for (auto& p : c->ark_bufs) free_dev_t(p);
  c->ark_bufs.clear();
  c->halo_elems = 0;
  c->state_valid = false;
}

int ensure_cg(mr_ctx* c)
{
  double** bufs[5] = {&c->cg_known, &c->cg_r, &c->cg_z, &c->cg_p, &c->cg_q};
  for (double** b : bufs)
    if (!*b) MR_CUDA_TRY(c, cudaMalloc(b, c->dof * sizeof(double)));
  if (!c->cg_part) MR_CUDA_TRY(c, cudaMalloc(&c->cg_part, sizeof(double) * lap_blocks()));
  if (!c->cg_part2) MR_CUDA_TRY(c, cudaMalloc(&c->cg_part2, sizeof(double) * lap_blocks()));
  if (!c->cg_sc) MR_CUDA_TRY(c, cudaMalloc(&c->cg_sc, sizeof(double) * 8));
  if (!c->cg_gather) MR_CUDA_TRY(c, cudaMalloc(&c->cg_gather, sizeof(double) * 64));
  return MR_OK;
}

int ensure_state(mr_ctx* c)
{
  if (!c->has_grid) return set_err(c, MR_CONTRACT, "grid not set (mr_grid_set)");
  if (!c->y_state) {
    MR_CUDA_TRY(c, cudaMalloc(&c->y_state, c->dof * sizeof(double)));
    MR_CUDA_TRY(c, cudaMemsetAsync(c->y_state, 0, c->dof * sizeof(double), c->stream));
  }
  if (!c->y_work) MR_CUDA_TRY(c, cudaMalloc(&c->y_work, c->dof * sizeof(double)));
  return MR_OK;
}

int ensure_slots(mr_ctx* c, int n)
{
  while ((int)c->slots.size() < n) {
    double* p = nullptr;
    MR_CUDA_TRY(c, cudaMalloc(&p, c->dof * sizeof(double)));
    c->slots.push_back(p);
  }
  return MR_OK;
}

int ensure_halo(mr_ctx* c)
{
  const size_t need = (size_t)c->ncomp * c->M * c->plane;
  if (c->halo_elems == need) return MR_OK;
  free_dev_t(c->send_lo);
  free_dev_t(c->send_hi);
  free_dev_t(c->recv_lo);
  free_dev_t(c->recv_hi);
  MR_CUDA_TRY(c, cudaMalloc(&c->send_lo, need * sizeof(double)));
  MR_CUDA_TRY(c, cudaMalloc(&c->send_hi, need * sizeof(double)));
  if (c->comm) {
    MR_CUDA_TRY(c, cudaMalloc(&c->recv_lo, need * sizeof(double)));
    MR_CUDA_TRY(c, cudaMalloc(&c->recv_hi, need * sizeof(double)));
  }
  c->halo_elems = need;
  return MR_OK;
}

bool fast_present(const mr_ctx* c) { return c->fast_kind != FK_NONE; }
bool slow_present(const mr_ctx* c) { return c->slow_kind != SK_NONE; }

int check_ready(mr_ctx* c)
{
  if (!c->has_grid) return set_err(c, MR_CONTRACT, "grid not set (mr_grid_set)");
  if (!c->has_coupling) return set_err(c, MR_CONTRACT, "coupling not loaded");
  if (!c->has_table) return set_err(c, MR_CONTRACT, "fast table not loaded");
  if (c->fast_kind < 0 || c->slow_kind < 0)
    return set_err(c, MR_CONTRACT, "PartitionedSystem: fast/slow plugins not configured");
  if (c->fast_kind == FK_NONE && c->slow_kind == SK_NONE)
    return set_err(c, MR_CONTRACT, "PartitionedSystem: at least one partition required");
  if (c->cp.implicit && !(c->slow_kind == SK_STENCIL && c->imex))
    return set_err(c, MR_CONTRACT, "mri_step: coupling needs f_implicit");
  if (!c->cp.implicit && c->imex)
    return set_err(c, MR_CONTRACT,
                   "mri_step: explicit coupling on a split slow partition (f_I + f_E)");
  if (c->imex && c->nranks > 16)
    return set_err(c, MR_CONTRACT, "IMEX solves support at most 16 slabs per process group");
  if (c->fast_kind == FK_CHEM && c->ncomp != c->S + 1)
    return set_err(c, MR_CONTRACT, "chemistry plugin needs n_comp == S + 1");
  if ((c->fast_kind == FK_LINEAR && c->fastA.n != c->ncomp) ||
      (c->slow_kind == SK_LINEAR && c->slowA.n != c->ncomp))
    return set_err(c, MR_CONTRACT, "linear plugin size != n_comp");
  if (c->slow_kind == SK_STENCIL && c->n0l < c->M)
    return set_err(c, MR_CONTRACT, "slab thinner than the stencil ghost width");
  return MR_OK;
}

Plan build_plan(const mr_ctx* c)
{
  const Coupling& cp = c->cp;
  const int s = cp.s;
  Plan p;
  for (int i = 0; i < kMaxStages; ++i) p.slot_of[i] = p.islot_of[i] = -1;
  const bool slow = slow_present(c);
  const bool imp = cp.implicit;  // check_ready guarantees the implicit plugin
  for (int j = 0; j < s; ++j)
    if (slow && cp.eval_at[j] && cp.fE_ref[j]) p.slot_of[j] = p.nslots++;
  for (int j = 0; j < s; ++j)
    if (imp && cp.fI_ref[j]) p.islot_of[j] = p.nslots++;
  // eval_slow_at (mri.cpp:339-349): f_E where scheduled, f_I where referenced
  // (not at solve stages, whose f_I is recovered from the solve)
  auto eval_ops = [&](int j) {
    if (slow && cp.eval_at[j]) {
      Op o;
      o.type = p.slot_of[j] >= 0 ? Op::SLOW : Op::COUNT_SLOW;  // unreferenced: count only
      o.stage = j;
      p.ops.push_back(o);
    }
    if (imp && cp.fI_ref[j] && cp.kind[j] != MR_STAGE_IMPLICIT_SOLVE) {
      Op o;
      o.type = Op::IMPL;
      o.stage = j;
      p.ops.push_back(o);
    }
  };
  auto evals_at = [&](int j) {
    return (slow && cp.eval_at[j]) ||
           (imp && cp.fI_ref[j] && cp.kind[j] != MR_STAGE_IMPLICIT_SOLVE);
  };
  eval_ops(0);
  std::vector<int> run;
  auto flush = [&]() {
    if (run.empty()) return;
    bool has_ivp = false;
    for (int i : run) has_ivp |= cp.kind[i] == MR_STAGE_FAST_IVP;
    if (!has_ivp) {
      for (int i : run) {
        Op o;
        o.type = Op::UPDATE;
        o.stage = i;
        p.ops.push_back(o);
      }
    } else {
      for (size_t a = 0; a < run.size(); a += MR_MAXCHAIN) {
        Op o;
        o.type = Op::CHAIN;
        for (size_t b = a; b < std::min(run.size(), a + MR_MAXCHAIN); ++b) o.stages.push_back(run[b]);
        p.ops.push_back(o);
      }
    }
    run.clear();
  };
  for (int i = 1; i < s; ++i) {
    // a stage referencing a slow value that is never evaluated: the reference
    // fails inside build_forcing / axpy_into at that stage (mri.cpp:288-296)
    bool missing = false;
    for (int j = 0; j < i; ++j) {
      bool refE = false, refI = false;
      if (cp.kind[i] == MR_STAGE_FAST_IVP) {
        for (int k = 0; k < cp.ndeg_o; ++k) refE |= cp.W(k, i, j) != 0.0;
        for (int k = 0; k < cp.ndeg_g; ++k) refI |= cp.G(k, i, j) != 0.0;
      } else {
        refE = cp.wbar[i][j] != 0.0;
        refI = cp.gbar[i][j] != 0.0;
      }
      if ((refE && p.slot_of[j] < 0) || (refI && p.islot_of[j] < 0)) missing = true;
    }
    if (missing) {
      flush();
      Op o;
      o.type = Op::MISSING;
      o.stage = i;
      p.ops.push_back(o);
      return p;
    }
    if (cp.kind[i] == MR_STAGE_IMPLICIT_SOLVE) {
      flush();
      Op o;
      o.type = Op::SOLVE;
      o.stage = i;
      p.ops.push_back(o);
      eval_ops(i);
      continue;
    }
    run.push_back(i);
    if (evals_at(i) || i == s - 1) {
      flush();
      eval_ops(i);
    }
  }
  return p;
}

// per-stage IVP schedule (mri.cpp:358-377)
struct IvpSched {
  int n_sub;
  double t_start, span, h_sub, dc;
};

IvpSched ivp_sched(const mr_ctx* c, int i, double t, double H)
{
  const Coupling& cp = c->cp;
  IvpSched r;
  r.dc = cp.c[i] - cp.c[i - 1];
  r.span = r.dc * H;
  r.n_sub = static_cast<int>(std::max(1L, std::lround(static_cast<double>(c->m) * r.dc)));
  r.t_start = t + cp.c[i - 1] * H;
  r.h_sub = r.span / r.n_sub;
  return r;
}

int ndeg_of(const mr_ctx* c) { return std::max(c->cp.degrees(), 1); }

void fill_chain_stage(const mr_ctx* c, int i, double t, double H, const Plan& p,
                      ChainStageDev& st)
{
  const Coupling& cp = c->cp;
  std::memset(&st, 0, sizeof(st));
  st.mri_stage = i;
  if (cp.kind[i] == MR_STAGE_FAST_IVP) {
    const IvpSched sc = ivp_sched(c, i, t, H);
    st.kind = 0;
    st.n_sub = sc.n_sub;
    st.t_start = sc.t_start;
    st.span = sc.span;
    st.h_sub = sc.h_sub;
    // build_forcing order (mri.cpp:285-301): gamma over fI, then omega over fE
    for (int pass = 0; pass < 2; ++pass) {
      const int nd = pass == 0 ? cp.ndeg_g : cp.ndeg_o;
      for (int j = 0; j < i; ++j) {
        bool refd = false;
        for (int k = 0; k < nd; ++k) refd |= (pass == 0 ? cp.G(k, i, j) : cp.W(k, i, j)) != 0.0;
        if (!refd) continue;
        const int r = st.nref++;
        st.ref_slot[r] = pass == 0 ? p.islot_of[j] : p.slot_of[j];
        for (int k = 0; k < MR_MAXDEG; ++k)
          st.coef[k][r] = k < nd ? (pass == 0 ? cp.G(k, i, j) : cp.W(k, i, j)) / sc.dc : 0.0;
      }
    }
  } else {
    // known = Y + sum_j H (gbar_ij fI_j + wbar_ij fE_j), j ascending (mri.cpp:380-384)
    st.kind = 2;
    for (int j = 0; j < i; ++j) {
      if (cp.gbar[i][j] != 0.0) {
        const int r = st.nref++;
        st.ref_slot[r] = p.islot_of[j];
        st.coef[0][r] = H * cp.gbar[i][j];
      }
      if (cp.wbar[i][j] != 0.0) {
        const int r = st.nref++;
        st.ref_slot[r] = p.slot_of[j];
        st.coef[0][r] = H * cp.wbar[i][j];
      }
    }
  }
}

// Per-evaluation tau of a chain's FastIvp stages, in the kernels' evaluation
// order and with their operations (dadd/dmul/ddiv in IEEE double: the host
// values are bitwise the device's); too many evaluations: ntau = 0.
void fill_chain_taus(const mr_ctx* c, ChainArgs& a)
{
  a.ntau = 0;
  int e = 0;
  for (int si = 0; si < a.nst; ++si) {
    const ChainStageDev& st = a.st[si];
    if (st.kind != 0) continue;
    if (e + st.n_sub * c->tab.s > MR_MAXTAU) return;
    for (int sub = 0; sub < st.n_sub; ++sub) {
      const double t0 = st.t_start + (double)sub * st.h_sub;
      for (int j = 0; j < c->tab.s; ++j) {
        const double theta = t0 + c->tab.c[j] * st.h_sub;
        a.tau[e++] = (theta + -st.t_start) / st.span;
      }
    }
  }
  a.ntau = e;
}

cudaEvent_t pool_event(mr_ctx* c, size_t idx)
{
  while (c->ev_pool.size() <= idx) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    c->ev_pool.push_back(e);
  }
  return c->ev_pool[idx];
}

// grouped send/recv of the packed ghost planes with the periodic neighbours
// (r - 1) mod P and (r + 1) mod P (a one-rank communicator sends to itself)
int nccl_halo_exchange(mr_ctx* c, cudaStream_t st)
{
  const int left = (c->rank - 1 + c->nranks) % c->nranks;
  const int right = (c->rank + 1) % c->nranks;
  MR_NCCL_TRY(c, GroupStart());
  MR_NCCL_TRY(c, Send(c->send_lo, c->halo_elems, ncclDouble, left, c->comm, st));
  MR_NCCL_TRY(c, Recv(c->recv_hi, c->halo_elems, ncclDouble, right, c->comm, st));
  MR_NCCL_TRY(c, Send(c->send_hi, c->halo_elems, ncclDouble, right, c->comm, st));
  MR_NCCL_TRY(c, Recv(c->recv_lo, c->halo_elems, ncclDouble, left, c->comm, st));
  MR_NCCL_TRY(c, GroupEnd());
  return MR_OK;
}

// ---------------------------------------------------------------------------
// halo exchange for the stencil: fills halo pointers of every context
// ---------------------------------------------------------------------------
int exchange_halos(mr_ctx** cs, int n, const double* const* ycur, const double** lo,
                   const double** hi, cudaStream_t st)
{
  const bool dom = cs[0]->in_domain && n > 1;
  for (int r = 0; r < n; ++r) {
    mr_ctx* c = cs[r];
    sdev(c);
    int rc = ensure_halo(c);
    if (rc) return rc;
    if (dom && cs[(r + n - 1) % n]->recv_recorded) {
      // the neighbours' copies of this slab's previous planes are done
      MR_CUDA_TRY(c, cudaStreamWaitEvent(c->stream, cs[(r + n - 1) % n]->ev_recv, 0));
      MR_CUDA_TRY(c, cudaStreamWaitEvent(c->stream, cs[(r + 1) % n]->ev_recv, 0));
    }
    MR_CUDA_TRY(c, launch_halo_pack(ycur[r], c->send_lo, c->send_hi, c->ncomp, c->n0l, c->plane,
                                    c->M, sst(c, st)));
    c->launches++;
    if (dom) MR_CUDA_TRY(c, cudaEventRecord(c->ev_send, c->stream));
  }
  if (n == 1 && !cs[0]->comm) {  // periodic single slab: own planes wrap around
    lo[0] = cs[0]->send_hi;
    hi[0] = cs[0]->send_lo;
    return MR_OK;
  }
  if (n == 1) {  // NCCL ring of slabs
    mr_ctx* c = cs[0];
    int rc = nccl_halo_exchange(c, st);
    if (rc) return rc;
    lo[0] = c->recv_lo;
    hi[0] = c->recv_hi;
    return MR_OK;
  }
  // several slabs in one process: each slab copies its neighbours' packed
  // planes -- peer-to-peer over NVLink between the GPUs of a multi-device
  // domain (after the neighbours' pack events), device-to-device on the one
  // shared stream of in-process virtual ranks
  for (int r = 0; r < n; ++r) {
    mr_ctx* c = cs[r];
    sdev(c);
    if (!c->recv_lo) {
      MR_CUDA_TRY(c, cudaMalloc(&c->recv_lo, c->halo_elems * sizeof(double)));
      MR_CUDA_TRY(c, cudaMalloc(&c->recv_hi, c->halo_elems * sizeof(double)));
    }
  }
  for (int r = 0; r < n; ++r) {
    mr_ctx* c = cs[r];
    mr_ctx* L = cs[(r - 1 + n) % n];
    mr_ctx* Rr = cs[(r + 1) % n];
    sdev(c);
    const cudaStream_t s2 = sst(c, st);
    const size_t bytes = c->halo_elems * sizeof(double);
    if (dom) {
      MR_CUDA_TRY(c, cudaStreamWaitEvent(s2, L->ev_send, 0));
      MR_CUDA_TRY(c, cudaStreamWaitEvent(s2, Rr->ev_send, 0));
      MR_CUDA_TRY(c, cudaMemcpyPeerAsync(c->recv_lo, c->device, L->send_hi, L->device, bytes, s2));
      MR_CUDA_TRY(c, cudaMemcpyPeerAsync(c->recv_hi, c->device, Rr->send_lo, Rr->device, bytes, s2));
      MR_CUDA_TRY(c, cudaEventRecord(c->ev_recv, s2));
      c->recv_recorded = true;
    } else {
      MR_CUDA_TRY(c, cudaMemcpyAsync(c->recv_lo, L->send_hi, bytes, cudaMemcpyDeviceToDevice, s2));
      MR_CUDA_TRY(c, cudaMemcpyAsync(c->recv_hi, Rr->send_lo, bytes, cudaMemcpyDeviceToDevice, s2));
    }
    lo[r] = c->recv_lo;
    hi[r] = c->recv_hi;
  }
  return MR_OK;
}

StencilArgs stencil_args(const mr_ctx* c, const double* y, double* out, const double* lo,
                         const double* hi)
{
  StencilArgs a{};
  a.y = y;
  a.out = out;
  a.halo_lo = lo;
  a.halo_hi = hi;
  a.n0l = c->n0l;
  a.n1 = c->n1;
  a.n2 = c->n2;
  a.ncomp = c->ncomp;
  a.M = c->M;
  a.i0 = c->i0;
  a.i_lo = 0;
  a.i_hi = c->n0l;
  for (int i = 0; i < 5; ++i) a.a[i] = a.b[i] = 0.0;
  if (c->order == 2) {
    a.a[1] = 1.0 / 2.0;
    a.b[0] = -2.0; a.b[1] = 1.0;
  } else if (c->order == 4) {
    a.a[1] = 2.0 / 3.0; a.a[2] = -1.0 / 12.0;
    a.b[0] = -5.0 / 2.0; a.b[1] = 4.0 / 3.0; a.b[2] = -1.0 / 12.0;
  } else {
    a.a[1] = 4.0 / 5.0; a.a[2] = -1.0 / 5.0; a.a[3] = 4.0 / 105.0; a.a[4] = -1.0 / 280.0;
    a.b[0] = -205.0 / 72.0; a.b[1] = 8.0 / 5.0; a.b[2] = -1.0 / 5.0; a.b[3] = 8.0 / 315.0;
    a.b[4] = -1.0 / 560.0;
  }
  const int ng[3] = {c->n0, c->n1, c->n2};
  for (int d = 0; d < 3; ++d) {
    const double dx = c->length / ng[d];
    a.inv_dx[d] = 1.0 / dx;
    a.inv_dx2[d] = 1.0 / (dx * dx);
  }
  a.D = c->D;
  a.vel_kind = c->vel_kind;
  for (int d = 0; d < 3; ++d) a.u[d] = c->u[d];
  a.prof = c->d_prof;
  a.nmax = c->nmax;
  return a;
}

// slow RHS of every context's current state into `outs`
int eval_slow(mr_ctx** cs, int n, const double* const* ycur, double* const* outs,
              cudaStream_t st)
{
  if (cs[0]->slow_kind == SK_LINEAR) {
    for (int r = 0; r < n; ++r) {
      sdev(cs[r]);
      MR_CUDA_TRY(cs[r], launch_slow_linear(ycur[r], outs[r], cs[r]->ncell, cs[r]->slowA,
                                            sst(cs[r], st)));
      cs[r]->launches++;
    }
    return MR_OK;
  }
  if (n == 1 && cs[0]->comm) {
    // NCCL rank: the halo exchange runs on the comm stream while the interior
    // planes [M, n0l - M) -- which read no ghost plane -- are computed; the
    // boundary planes follow once the halos have landed
    mr_ctx* c = cs[0];
    StencilArgs a = stencil_args(c, ycur[0], outs[0], nullptr, nullptr);
    if (stencil_plane_ranges(a) && c->n0l >= 2 * c->M + 1) {
      int rc = ensure_halo(c);
      if (rc) return rc;
      if (!c->comm_stream) {
        MR_CUDA_TRY(c, cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
        MR_CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_pack, cudaEventDisableTiming));
        MR_CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_halo, cudaEventDisableTiming));
      }
      MR_CUDA_TRY(c, launch_halo_pack(ycur[0], c->send_lo, c->send_hi, c->ncomp, c->n0l, c->plane,
                                      c->M, st));
      c->launches++;
      MR_CUDA_TRY(c, cudaEventRecord(c->ev_pack, st));
      MR_CUDA_TRY(c, cudaStreamWaitEvent(c->comm_stream, c->ev_pack, 0));
      rc = nccl_halo_exchange(c, c->comm_stream);
      if (rc) return rc;
      MR_CUDA_TRY(c, cudaEventRecord(c->ev_halo, c->comm_stream));
      a.halo_lo = c->recv_lo;
      a.halo_hi = c->recv_hi;
      a.i_lo = c->M;
      a.i_hi = c->n0l - c->M;
      MR_CUDA_TRY(c, launch_stencil(a, st));  // interior
      MR_CUDA_TRY(c, cudaStreamWaitEvent(st, c->ev_halo, 0));
      a.i_lo = 0;
      a.i_hi = c->M;
      MR_CUDA_TRY(c, launch_stencil(a, st));  // first ghost-dependent planes
      a.i_lo = c->n0l - c->M;
      a.i_hi = c->n0l;
      MR_CUDA_TRY(c, launch_stencil(a, st));  // last ghost-dependent planes
      c->launches += 3;
      return MR_OK;
    }
  }
  std::vector<const double*> lo(n), hi(n);
  int rc = exchange_halos(cs, n, ycur, lo.data(), hi.data(), st);
  if (rc) return rc;
  for (int r = 0; r < n; ++r) {
    sdev(cs[r]);
    MR_CUDA_TRY(cs[r], launch_stencil(stencil_args(cs[r], ycur[r], outs[r], lo[r], hi[r]),
                                      sst(cs[r], st)));
    cs[r]->launches++;
  }
  return MR_OK;
}

void add_solve_counts(const mr_ctx* c, int stage, uint64_t* cnt)
{
  // newton_solve (solvers.cpp:150-208): one implicit eval per residual, one
  // nonlinear iteration per update; each linear solve = cg_iters CG
  // iterations (one matvec each) and cg_iters + 1 Jacobi applications
  const uint64_t nl = (uint64_t)c->solve_nl[stage];
  cnt[MR_CNT_IMPLICIT_EVALS] += (uint64_t)c->solve_evals[stage];
  cnt[MR_CNT_NONLINEAR_ITERS] += nl;
  cnt[MR_CNT_LINEAR_ITERS] += nl * (uint64_t)c->cg_iters;
  cnt[MR_CNT_PRECOND_SOLVES] += nl * ((uint64_t)c->cg_iters + 1);
  cnt[MR_CNT_IMPLICIT_SOLVES] += 1;
}

void add_counts_full(const mr_ctx* c, const Plan& p, double t, double H, uint64_t* cnt)
{
  for (const Op& o : p.ops) {
    if (o.type == Op::SLOW || o.type == Op::COUNT_SLOW) cnt[MR_CNT_EXPLICIT_EVALS]++;
    if (o.type == Op::IMPL) cnt[MR_CNT_IMPLICIT_EVALS]++;
    if (o.type == Op::SOLVE) add_solve_counts(c, o.stage, cnt);
    if (o.type == Op::CHAIN)
      for (int i : o.stages)
        if (c->cp.kind[i] == MR_STAGE_FAST_IVP) {
          if (fast_present(c))
            cnt[MR_CNT_FAST_EVALS] += (uint64_t)ivp_sched(c, i, t, H).n_sub * c->tab.s;
          cnt[MR_CNT_FAST_IVPS]++;
        }
  }
}

// counts up to a failure at (stage, sub, inner) -- what the reference's
// by-reference EvalCounters hold when mri_step throws.  For a solve stage,
// inner 0 = non-finite stage data (before the solve), 1 = non-finite state
// after it, 2 = Newton did not converge.
void add_counts_partial(const mr_ctx* c, const Plan& p, double t, double H, int fs, int fsub,
                        int finner, uint64_t* cnt)
{
  for (const Op& o : p.ops) {
    if ((o.type == Op::SLOW || o.type == Op::COUNT_SLOW) && o.stage < fs)
      cnt[MR_CNT_EXPLICIT_EVALS]++;
    if (o.type == Op::IMPL && o.stage < fs) cnt[MR_CNT_IMPLICIT_EVALS]++;
    if (o.type == Op::SOLVE && (o.stage < fs || (o.stage == fs && finner >= 1)))
      add_solve_counts(c, o.stage, cnt);
    if (o.type == Op::CHAIN)
      for (int i : o.stages) {
        if (c->cp.kind[i] != MR_STAGE_FAST_IVP || i > fs) continue;
        const int ns = ivp_sched(c, i, t, H).n_sub;
        if (i < fs) {
          if (fast_present(c)) cnt[MR_CNT_FAST_EVALS] += (uint64_t)ns * c->tab.s;
          cnt[MR_CNT_FAST_IVPS]++;
        } else if (fast_present(c)) {
          cnt[MR_CNT_FAST_EVALS] += (uint64_t)fsub * c->tab.s + (uint64_t)finner;
        }
      }
  }
}

LapArgs lap_args(const mr_ctx* c, double gamma)
{
  LapArgs a{};
  a.n0l = c->n0l;
  a.n1 = c->n1;
  a.n2 = c->n2;
  a.ncomp = c->ncomp;
  a.M = c->M;
  const int ng[3] = {c->n0, c->n1, c->n2};
  double sdx = 0.0;
  for (int d = 0; d < 3; ++d) {
    const double dx = c->length / ng[d];
    a.inv_dx2[d] = 1.0 / (dx * dx);
    sdx += 2.0 / (dx * dx);
  }
  a.D = c->d_impl;
  a.gamma = gamma;
  a.dg = 1.0 + gamma * (c->d_impl * sdx);
  return a;
}

// f_I = d_impl L7 y of every context's current state into `outs`
int eval_implicit(mr_ctx** cs, int n, const double* const* ycur, double* const* outs,
                  cudaStream_t st)
{
  std::vector<const double*> lo(n), hi(n);
  int rc = exchange_halos(cs, n, ycur, lo.data(), hi.data(), st);
  if (rc) return rc;
  for (int r = 0; r < n; ++r) {
    sdev(cs[r]);
    MR_CUDA_TRY(cs[r], launch_lap7(0, lap_args(cs[r], 0.0), ycur[r], lo[r], hi[r], nullptr,
                                   nullptr, outs[r], nullptr, nullptr, nullptr, nullptr,
                                   sst(cs[r], st)));
    cs[r]->launches++;
  }
  return MR_OK;
}

// global dot product: block partials -> per-slab value -> sum over slabs
// (in-process, slab order) or ranks (NCCL all-gather, rank order)
int dot_finalize(mr_ctx** cs, int n, int slot, cudaStream_t st, bool second = false)
{
  for (int r = 0; r < n; ++r) {
    sdev(cs[r]);
    MR_CUDA_TRY(cs[r], launch_part_sum(second ? cs[r]->cg_part2 : cs[r]->cg_part, cs[r]->cg_sc,
                                       slot, sst(cs[r], st)));
    cs[r]->launches++;
  }
  if (n > 1 && cs[0]->in_domain) {
    // multi-device: gather the slab values on the first slab's device, sum
    // them in slab order there (the order of scalar_combine_kernel, so the
    // result is bitwise that of the virtual ranks) and copy the sum back
    mr_ctx* c0 = cs[0];
    for (int r = 0; r < n; ++r) {
      sdev(cs[r]);
      MR_CUDA_TRY(cs[r], cudaEventRecord(cs[r]->ev_dot, cs[r]->stream));
    }
    sdev(c0);
    for (int r = 0; r < n; ++r) {
      MR_CUDA_TRY(c0, cudaStreamWaitEvent(c0->stream, cs[r]->ev_dot, 0));
      MR_CUDA_TRY(c0, cudaMemcpyPeerAsync(c0->cg_gather + r, c0->device, cs[r]->cg_sc + slot,
                                          cs[r]->device, sizeof(double), c0->stream));
    }
    MR_CUDA_TRY(c0, launch_gathered_sum(c0->cg_gather, n, c0->cg_sc, slot, c0->stream));
    c0->launches++;
    MR_CUDA_TRY(c0, cudaEventRecord(c0->ev_dot, c0->stream));
    for (int r = 1; r < n; ++r) {
      sdev(cs[r]);
      MR_CUDA_TRY(cs[r], cudaStreamWaitEvent(cs[r]->stream, c0->ev_dot, 0));
      MR_CUDA_TRY(cs[r], cudaMemcpyPeerAsync(cs[r]->cg_sc + slot, cs[r]->device, c0->cg_sc + slot,
                                             c0->device, sizeof(double), cs[r]->stream));
    }
    return MR_OK;
  }
  if (n > 1) {
    std::vector<double*> scs(n);
    for (int r = 0; r < n; ++r) scs[r] = cs[r]->cg_sc;
    MR_CUDA_TRY(cs[0], launch_scalar_combine(scs.data(), n, slot, st));
    cs[0]->launches++;
  } else if (cs[0]->comm) {
    mr_ctx* c = cs[0];
    MR_NCCL_TRY(c, AllGather(c->cg_sc + slot, c->cg_gather, 1, ncclDouble, c->comm, st));
    MR_CUDA_TRY(c, launch_gathered_sum(c->cg_gather, c->nranks, c->cg_sc, slot, st));
    c->launches++;
  }
  return MR_OK;
}

// newton_solve (solvers.cpp:150-208) on G(Y) = Y - gamma f_I(Y) - known with
// known in cg_known and Y (initialised by the caller, = known) in y_work; the
// linear solve is the fixed-iteration PCG (same iteration as oracle
// newton_pcg_stage).  Convergence is a host decision on the globally reduced
// WRMS (one 8-byte read per Newton iteration; every slab and rank sees the
// same value).  On success fI = (Y - known)/gamma (mri.cpp:418-421) goes to
// fI_out[r]; on failure *host_key = (stage, 0, 2).  Counts go to
// solve_evals[i] / solve_nl[i].
int newton_pcg(mr_ctx** cs, int n, int i, double gamma, double* const* fI_out,
               unsigned long long* host_key, cudaStream_t st)
{
  mr_ctx* c0 = cs[0];
  const double target = c0->newton_safety * c0->newton_tol;
  const double nglob = (double)c0->n0 * c0->n1 * c0->n2 * c0->ncomp;
  std::vector<const double*> lo(n), hi(n), src(n);
  for (int r = 0; r < n; ++r) {
    cs[r]->solve_evals[i] = 0;
    cs[r]->solve_nl[i] = 0;
  }
  bool converged = false;
  for (int iter = 0; iter <= c0->newton_max; ++iter) {
    // residual G(Y) at Y = y_work; r = -G, z = r/dg, p = z
    for (int r = 0; r < n; ++r) src[r] = cs[r]->y_work;
    int rc = exchange_halos(cs, n, src.data(), lo.data(), hi.data(), st);
    if (rc) return rc;
    for (int r = 0; r < n; ++r) {
      mr_ctx* c = cs[r];
      sdev(c);
      MR_CUDA_TRY(c, launch_lap7(1, lap_args(c, gamma), c->y_work, lo[r], hi[r], c->cg_known,
                                 c->newton_w, c->cg_r, c->cg_z, c->cg_p, c->cg_part, c->cg_part2,
                                 sst(c, st)));
      c->launches++;
      c->solve_evals[i]++;
    }
    rc = dot_finalize(cs, n, 3, st);
    if (rc) return rc;
    sdev(c0);
    MR_CUDA_TRY(c0, cudaMemcpyAsync(c0->h_red, c0->cg_sc + 3, sizeof(double),
                                    cudaMemcpyDeviceToHost, sst(c0, st)));
    MR_CUDA_TRY(c0, cudaStreamSynchronize(sst(c0, st)));
    const double wrms = std::sqrt(c0->h_red[0] / nglob);
    if (!std::isfinite(wrms)) break;
    if (wrms <= target) {
      converged = true;
      break;
    }
    if (iter == c0->newton_max) break;
    rc = dot_finalize(cs, n, 0, st, true);  // rz
    if (rc) return rc;
    for (int it = 0; it < c0->cg_iters; ++it) {
      for (int r = 0; r < n; ++r) src[r] = cs[r]->cg_p;
      rc = exchange_halos(cs, n, src.data(), lo.data(), hi.data(), st);
      if (rc) return rc;
      for (int r = 0; r < n; ++r) {
        mr_ctx* c = cs[r];
        sdev(c);
        MR_CUDA_TRY(c, launch_lap7(2, lap_args(c, gamma), c->cg_p, lo[r], hi[r], nullptr, nullptr,
                                   c->cg_q, nullptr, nullptr, c->cg_part, nullptr, sst(c, st)));
        c->launches++;
      }
      rc = dot_finalize(cs, n, 1, st);  // pAp
      if (rc) return rc;
      for (int r = 0; r < n; ++r) {
        mr_ctx* c = cs[r];
        sdev(c);
        MR_CUDA_TRY(c, launch_cg_update(c->dof, lap_args(c, gamma).dg, c->cg_sc, c->y_work,
                                        c->cg_r, c->cg_z, c->cg_p, c->cg_q, c->cg_part, sst(c, st)));
        c->launches++;
      }
      rc = dot_finalize(cs, n, 2, st);  // rz_new
      if (rc) return rc;
      for (int r = 0; r < n; ++r) {
        mr_ctx* c = cs[r];
        sdev(c);
        MR_CUDA_TRY(c, launch_cg_p(c->dof, c->cg_sc, c->cg_p, c->cg_z, sst(c, st)));
        MR_CUDA_TRY(c, launch_scalar_copy(c->cg_sc, 0, 2, sst(c, st)));
        c->launches += 2;
      }
    }
    for (int r = 0; r < n; ++r) cs[r]->solve_nl[i]++;
  }
  if (!converged) {
    *host_key = mr_fail_key(i, 0, 2);
    return MR_OK;
  }
  for (int r = 0; r < n; ++r) {
    mr_ctx* c = cs[r];
    sdev(c);
    MR_CUDA_TRY(c, launch_recover_fi(c->dof, gamma, c->y_work, c->cg_known, fI_out[r], i, c->d_fail,
                                     sst(c, st)));
    c->launches++;
  }
  return MR_OK;
}

// ImplicitSolve stage i (mri.cpp:378-421): known, then newton_pcg from
// Y = known.  *host_key is set when Newton fails.
int solve_stage(mr_ctx** cs, int n, int i, double t, double H, const Plan& plan,
                std::vector<const double*>& ycur, cudaStream_t st, unsigned long long* host_key)
{
  const double gamma = H * cs[0]->cp.gbar[i][i];
  for (int r = 0; r < n; ++r) {
    mr_ctx* c = cs[r];
    sdev(c);
    int rc = ensure_cg(c);
    if (rc) return rc;
    ChainStageDev sd;
    fill_chain_stage(c, i, t, H, plan, sd);
    const double* f[MR_MAXREF];
    for (int q = 0; q < sd.nref; ++q) f[q] = c->slots[sd.ref_slot[q]];
    MR_CUDA_TRY(c, launch_update(ycur[r], c->cg_known, sd.nref, f, sd.coef[0], c->dof, i,
                                 c->d_fail, sst(c, st)));
    MR_CUDA_TRY(c, cudaMemcpyAsync(c->y_work, c->cg_known, c->dof * sizeof(double),
                                   cudaMemcpyDeviceToDevice, sst(c, st)));
    c->launches++;
    ycur[r] = c->y_work;
  }
  std::vector<double*> fI_out(n);
  for (int r = 0; r < n; ++r)
    fI_out[r] = plan.islot_of[i] >= 0 ? cs[r]->slots[plan.islot_of[i]] : cs[r]->cg_q;
  return newton_pcg(cs, n, i, gamma, fI_out.data(), host_key, st);
}

// One slow step over a domain of slab contexts sharing a device stream (n > 1)
// or one context (n == 1, possibly an NCCL rank).
int domain_finish(mr_ctx** cs, int n, const Plan& plan, double t, double H, int missing_stage,
                  unsigned long long host_key, const std::vector<std::pair<int, size_t>>& timed,
                  const double* const* ycur, uint64_t* counters, int* fail_stage);

// async: enqueue only (n == 1); the step is finished by domain_finish from
// mr_mri_step_wait with the state kept in ctx->pending
// ---- pipelined host-buffer step (mr_mri_step_host) ----
// The state travels in K plane chunks (>= M planes each) on a copy stream
// while the step computes: the upload rides on the step's first two ops (the
// stage-0 slow evaluation and the first fused chain), the download on its
// last three (the last fused chain, the last slow evaluation and the final
// explicit update).  Those ops run chunk by chunk on the compute stream, in an
// order that respects the stencil's +-M-plane reach; every kernel computes
// exactly what the whole-grid op computes (bitwise equal results), only the
// PCIe copies now hide behind the chemistry.
int host_chunks(const mr_ctx* c, int* pb)
{
  const int K = std::min(kHeadChunks, c->M > 0 ? c->n0l / c->M : 0);
  for (int q = 0; q <= K && K > 0; ++q) pb[q] = (int)((long long)q * c->n0l / K);
  return K;
}

bool pipeline_ok(const mr_ctx* c, const Plan& plan)
{
  int pb[kHeadChunks + 1];
  // Not on NCCL ranks: the chunked schedule works there (the end chunks wait
  // for the exchanged ghosts; tests/test_gpu_nccl.py with MR_PIPELINE_NCCL),
  // but through the one-GPU loopback communicator it measured no better than
  // the plain copies (705-744 vs 712 ms per slab step, the exchange kernels
  // queue behind the chemistry), so ranks keep the plain upload/download until
  // it can be measured on the 8-GPU box.  Not the in-process domains either.
  if ((c->comm && !c->pipeline_nccl) || c->in_domain || c->profile || c->fast_kind != FK_CHEM ||
      c->slow_kind != SK_STENCIL || c->imex || host_chunks(c, pb) < 3 || plan.ops.size() < 2)
    return false;
  return stencil_plane_ranges(stencil_args(c, c->y_state, nullptr, nullptr, nullptr));
}

int ensure_copy_stream(mr_ctx* c)
{
  if (!c->copy_stream) {
    MR_CUDA_TRY(c, cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    for (cudaEvent_t& e : c->ev_copy)
      MR_CUDA_TRY(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  return MR_OK;
}

void fill_chain_args(mr_ctx* c, const Op& o, const Plan& plan, double t, double H,
                     const double* yin, ChainArgs& a)
{
  std::memset(&a, 0, sizeof(a));
  a.nst = (int)o.stages.size();
  a.ndeg = ndeg_of(c);
  for (int q = 0; q < a.nst; ++q) fill_chain_stage(c, o.stages[q], t, H, plan, a.st[q]);
  a.tab = c->tab;
  a.y_in = yin;
  a.y_out = c->y_work;
  for (int q = 0; q < (int)c->slots.size() && q < MR_MAXSLOT; ++q) a.fE[q] = c->slots[q];
  a.ncell = c->ncell;
  a.ncomp = c->ncomp;
  a.fail = c->d_fail;
  fill_chain_taus(c, a);
}

// chunked copy of planes [pb[q], pb[q+1]) of every component
cudaError_t copy_chunk(mr_ctx* c, double* dst, const double* src, const int* pb, int q,
                       cudaMemcpyKind kind)
{
  const size_t off = (size_t)pb[q] * c->plane, pitch = c->ncell * sizeof(double);
  return cudaMemcpy2DAsync(dst + off, pitch, src + off, pitch,
                           (size_t)(pb[q + 1] - pb[q]) * c->plane * sizeof(double), c->ncomp,
                           kind, c->copy_stream);
}

// Ghost planes of a chunked slow evaluation of `y`: the first and last M
// planes packed on `st`; on an NCCL rank they are then exchanged with the
// neighbours on the comm stream (ev_halo marks their arrival), on a single
// periodic slab the packed planes are the ghosts themselves.
int chunk_halos(mr_ctx* c, const double* y, cudaStream_t st, StencilArgs& sa)
{
  MR_CUDA_TRY(c, launch_halo_pack(y, c->send_lo, c->send_hi, c->ncomp, c->n0l, c->plane, c->M, st));
  c->launches++;
  if (!c->comm) {
    sa.halo_lo = c->send_hi;
    sa.halo_hi = c->send_lo;
    return MR_OK;
  }
  if (!c->comm_stream) {
    MR_CUDA_TRY(c, cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
    MR_CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_pack, cudaEventDisableTiming));
    MR_CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_halo, cudaEventDisableTiming));
  }
  MR_CUDA_TRY(c, cudaEventRecord(c->ev_pack, st));
  MR_CUDA_TRY(c, cudaStreamWaitEvent(c->comm_stream, c->ev_pack, 0));
  int rc = nccl_halo_exchange(c, c->comm_stream);
  if (rc) return rc;
  MR_CUDA_TRY(c, cudaEventRecord(c->ev_halo, c->comm_stream));
  sa.halo_lo = c->recv_lo;
  sa.halo_hi = c->recv_hi;
  return MR_OK;
}

// Upload + ops[0] (SLOW 0) + ops[1] (CHAIN).  Chunks are copied in the order
// K-1, 0, 1, ..., K-2 (the end chunks hold the slab's ghost-source planes);
// the stencil + chain of chunk q go as soon as chunks q-1..q+1 have landed --
// on an NCCL rank the two end chunks last, after the exchanged ghosts.
// *nops = 2 when done, 0 when the plan does not start that way.
int head_upload(mr_ctx* c, const double* hin, const Plan& plan, double t, double H,
                const ChemCfg& ccfg, cudaStream_t st, int* nops)
{
  *nops = 0;
  if (plan.ops[0].type != Op::SLOW || plan.ops[0].stage != 0 || plan.ops[1].type != Op::CHAIN)
    return MR_OK;
  int pb[kHeadChunks + 1];
  const int K = host_chunks(c, pb);
  int rc = ensure_halo(c);
  if (rc) return rc;
  rc = ensure_copy_stream(c);
  if (rc) return rc;
  // the copies start after whatever the compute stream still does with y_state
  MR_CUDA_TRY(c, cudaEventRecord(c->ev_copy[kHeadChunks], st));
  MR_CUDA_TRY(c, cudaStreamWaitEvent(c->copy_stream, c->ev_copy[kHeadChunks], 0));
  auto pos = [&](int q) { return q == K - 1 ? 0 : q + 1; };  // place in the copy order
  for (int i = 0; i < K; ++i) {
    const int q = (i + K - 1) % K;  // K-1, 0, 1, ..., K-2
    MR_CUDA_TRY(c, copy_chunk(c, c->y_state, hin, pb, q, cudaMemcpyHostToDevice));
    MR_CUDA_TRY(c, cudaEventRecord(c->ev_copy[q], c->copy_stream));
  }
  StencilArgs sa = stencil_args(c, c->y_state, c->slots[plan.slot_of[0]], nullptr, nullptr);
  MR_CUDA_TRY(c, cudaStreamWaitEvent(st, c->ev_copy[0], 0));  // chunks K-1 and 0
  rc = chunk_halos(c, c->y_state, st, sa);
  if (rc) return rc;
  const Op& o = plan.ops[1];
  ChainArgs a;
  fill_chain_args(c, o, plan, t, H, c->y_state, a);
  const NvtxRange r0("slow f_E", 0, -1);
  const NvtxRange r1("fast IVP chain", o.stages.front(), o.stages.back());
  auto chunk = [&](int q) -> int {
    // one copy event covers chunks q-1..q+1: the latest of them in copy order
    int last = q;
    if (q > 0 && pos(q - 1) > pos(last)) last = q - 1;
    if (q + 1 < K && pos(q + 1) > pos(last)) last = q + 1;
    MR_CUDA_TRY(c, cudaStreamWaitEvent(st, c->ev_copy[last], 0));
    sa.i_lo = pb[q];
    sa.i_hi = pb[q + 1];
    MR_CUDA_TRY(c, launch_stencil(sa, st));
    a.cell0 = (size_t)pb[q] * c->plane;
    a.cell1 = (size_t)pb[q + 1] * c->plane;
    MR_CUDA_TRY(c, launch_chem_chain(ccfg, a, *c->chemP, st));
    c->launches += 2;
    return MR_OK;
  };
  if (!c->comm) {
    for (int q = 0; q < K; ++q)
      if ((rc = chunk(q))) return rc;
  } else {
    for (int q = 1; q + 1 < K; ++q)
      if ((rc = chunk(q))) return rc;
    MR_CUDA_TRY(c, cudaStreamWaitEvent(st, c->ev_halo, 0));
    if ((rc = chunk(0))) return rc;
    if ((rc = chunk(K - 1))) return rc;
  }
  *nops = 2;
  return MR_OK;
}

// Index of the final UPDATE of a plan ending CHAIN, SLOW(j), UPDATE(s-1)
// (+ unreferenced COUNT_SLOW), or -1.
int tail_index(const Plan& plan, size_t first_op)
{
  size_t L = plan.ops.size();
  while (L > 0 && plan.ops[L - 1].type == Op::COUNT_SLOW) --L;
  if (L < 3 || L - 3 < first_op) return -1;
  const Op& oc = plan.ops[L - 3];
  const Op& os = plan.ops[L - 2];
  const Op& ou = plan.ops[L - 1];
  if (oc.type != Op::CHAIN || os.type != Op::SLOW || plan.slot_of[os.stage] < 0 ||
      ou.type != Op::UPDATE)
    return -1;
  return (int)(L - 1);
}

// ops[L-2..L]: the last chain, slow evaluation and explicit update, chunk by
// chunk, each finished chunk of the result streaming to hout.  Chain chunks in
// the order K-1, 0, 1, ..., K-2; the stencil of chunk q once the chains of
// q-1..q+1 (or the ghosts, for the end chunks) are done; the in-place update
// of chunk q once every stencil reading its planes (q-1..q+1) is done; then
// its download.  An NCCL rank exchanges the ghosts once its end chunks are
// final and runs the end chunks' stencils after they arrive.
int tail_download(mr_ctx* c, const Plan& plan, int L, double t, double H, const ChemCfg& ccfg,
                  const double* yin, double* hout, cudaStream_t st)
{
  int pb[kHeadChunks + 1];
  const int K = host_chunks(c, pb);
  int rc = ensure_halo(c);
  if (rc) return rc;
  const Op& oc = plan.ops[L - 2];
  const Op& os = plan.ops[L - 1];
  const Op& ou = plan.ops[L];
  ChainArgs a;
  fill_chain_args(c, oc, plan, t, H, yin, a);
  StencilArgs sa = stencil_args(c, c->y_work, c->slots[plan.slot_of[os.stage]], nullptr, nullptr);
  ChainStageDev sd;
  fill_chain_stage(c, ou.stage, t, H, plan, sd);
  const NvtxRange r0("fast IVP chain", oc.stages.front(), oc.stages.back());
  const NvtxRange r1("slow f_E", os.stage, -1);
  const NvtxRange r2("explicit update", ou.stage, -1);
  std::vector<char> chained(K, 0), stenciled(K, 0), updated(K, 0);
  bool ghosts = false;
  auto stencil_ready = [&](int q) {
    return chained[q] && (q == 0 ? ghosts : chained[q - 1] != 0) &&
           (q == K - 1 ? ghosts : chained[q + 1] != 0);
  };
  auto update_ready = [&](int q) {
    return stenciled[q] && (q == 0 || stenciled[q - 1]) && (q == K - 1 || stenciled[q + 1]);
  };
  auto advance = [&]() -> int {  // everything whose inputs are enqueued
    for (int q = 0; q < K; ++q)
      if (!stenciled[q] && stencil_ready(q)) {
        sa.i_lo = pb[q];
        sa.i_hi = pb[q + 1];
        MR_CUDA_TRY(c, launch_stencil(sa, st));
        c->launches++;
        stenciled[q] = 1;
      }
    for (int q = 0; q < K; ++q)
      if (!updated[q] && update_ready(q)) {
        const size_t off = (size_t)pb[q] * c->plane;
        const double* f[MR_MAXREF];
        for (int r = 0; r < sd.nref; ++r) f[r] = c->slots[sd.ref_slot[r]] + off;
        MR_CUDA_TRY(c, launch_update_rows(c->y_work + off, c->y_work + off, sd.nref, f, sd.coef[0],
                                          (size_t)(pb[q + 1] - pb[q]) * c->plane, c->ncomp,
                                          c->ncell, ou.stage, c->d_fail, st));
        c->launches++;
        MR_CUDA_TRY(c, cudaEventRecord(c->ev_copy[q], st));
        MR_CUDA_TRY(c, cudaStreamWaitEvent(c->copy_stream, c->ev_copy[q], 0));
        MR_CUDA_TRY(c, copy_chunk(c, hout, c->y_work, pb, q, cudaMemcpyDeviceToHost));
        updated[q] = 1;
      }
    return MR_OK;
  };
  for (int i = 0; i < K; ++i) {
    const int q = (i + K - 1) % K;  // K-1, 0, 1, ..., K-2
    a.cell0 = (size_t)pb[q] * c->plane;
    a.cell1 = (size_t)pb[q + 1] * c->plane;
    MR_CUDA_TRY(c, launch_chem_chain(ccfg, a, *c->chemP, st));
    c->launches++;
    chained[q] = 1;
    if (q == 0) {  // both end chunks are final: their ghost-source planes go out
      rc = chunk_halos(c, c->y_work, st, sa);
      if (rc) return rc;
      ghosts = !c->comm;
    }
    if ((rc = advance())) return rc;
  }
  if (c->comm) {
    // the exchanged ghosts, waited for only after the last chain chunk: the
    // exchange kernels find SMs between the chain launches, and an earlier
    // wait was measured to stall the compute stream (slab 1/8: 723 vs 705 ms)
    MR_CUDA_TRY(c, cudaStreamWaitEvent(st, c->ev_halo, 0));
    ghosts = true;
    if ((rc = advance())) return rc;
  }
  for (int q = 0; q < K; ++q)
    if (!updated[q]) return set_err(c, MR_CUDA, "tail_download: chunk schedule incomplete");
  return MR_OK;
}

int domain_step(mr_ctx** cs, int n, double t, double H, uint64_t* counters, int* fail_stage,
                bool async = false)
{
  mr_ctx* c0 = cs[0];
  if (fail_stage) *fail_stage = -1;
  if (!(H > 0.0)) return set_err(c0, MR_CONTRACT, "mri_step: H must be positive");
  for (int r = 0; r < n; ++r) {
    sdev(cs[r]);
    int rc = check_ready(cs[r]);
    if (rc) return rc;
    rc = ensure_state(cs[r]);
    if (rc) return rc;
  }
  const Plan plan = build_plan(c0);
  if (plan.nslots > MR_MAXSLOT)
    return set_err(c0, MR_CONTRACT, "coupling stores more slow stage values than the device plan holds");
  for (int i = 1; i < c0->cp.s; ++i) {
    int nref = 0;
    const Coupling& cp = c0->cp;
    for (int j = 0; j < i; ++j) {
      bool g = false, w = false;
      for (int k = 0; k < cp.ndeg_g; ++k) g |= cp.G(k, i, j) != 0.0;
      for (int k = 0; k < cp.ndeg_o; ++k) w |= cp.W(k, i, j) != 0.0;
      if (cp.kind[i] != MR_STAGE_FAST_IVP) {
        g = cp.gbar[i][j] != 0.0;
        w = cp.wbar[i][j] != 0.0;
      }
      nref += (int)g + (int)w;
    }
    if (nref > MR_MAXREF)
      return set_err(c0, MR_CONTRACT, "coupling stage references more slow values than the device plan holds");
  }
  for (int r = 0; r < n; ++r) {
    sdev(cs[r]);
    int rc = ensure_slots(cs[r], plan.nslots);
    if (rc) return rc;
  }
  cudaStream_t st = c0->stream;
  ChainCfg cfg;
  ChemCfg ccfg;
  if (c0->fast_kind == FK_CHEM) {
    if (chem_pick(&ccfg, c0->ncomp, c0->S, c0->R, c0->tab, ndeg_of(c0)))
      return set_err(c0, MR_CONTRACT, "unsupported mechanism size / table for the chemistry kernel");
  } else if (chain_pick(&cfg, c0->fast_kind, c0->ncomp, c0->tab.s, ndeg_of(c0))) {
    return set_err(c0, MR_CONTRACT, "unsupported component count / table for the fused IVP kernel");
  }
  for (int r = 0; r < n; ++r) {
    sdev(cs[r]);
    MR_CUDA_TRY(cs[r], cudaMemsetAsync(cs[r]->d_fail, 0xFF, sizeof(unsigned long long),
                                       sst(cs[r], st)));
  }

  std::vector<const double*> ycur(n);
  std::vector<double*> outs(n);
  for (int r = 0; r < n; ++r) ycur[r] = cs[r]->y_state;
  size_t ev = 0;
  std::vector<std::pair<int, size_t>> timed;  // (class, event index)
  int missing_stage = -1;
  unsigned long long host_key = MR_NO_FAIL;  // Newton failure (host decision)

  NvtxRange step_range("mri_step");
  size_t first_op = 0, end_op = plan.ops.size();
  int tail_L = -1;
  double* hout = nullptr;
  if (n == 1 && c0->host_in) {  // host-buffer step: pipelined upload / download
    const double* hin = c0->host_in;
    hout = c0->host_out;
    c0->host_in = nullptr;
    c0->host_out = nullptr;
    const bool pipe = !async && pipeline_ok(c0, plan);
    int nops = 0;
    if (pipe) {
      int rc = head_upload(c0, hin, plan, t, H, ccfg, st, &nops);
      if (rc) return rc;
    }
    if (nops == 0) {
      MR_CUDA_TRY(c0, cudaMemcpyAsync(c0->y_state, hin, c0->dof * sizeof(double),
                                      cudaMemcpyHostToDevice, st));
    } else {
      ycur[0] = c0->y_work;
      first_op = (size_t)nops;
    }
    if (pipe && hout) tail_L = tail_index(plan, first_op);
    if (tail_L >= 0) {
      // the caller's y_out is saved first (behind the upload on the copy
      // stream): a failing step restores it, so no partial result survives
      int rc = ensure_copy_stream(c0);
      if (rc) return rc;
      if (!c0->y_backup) MR_CUDA_TRY(c0, cudaMalloc(&c0->y_backup, c0->dof * sizeof(double)));
      if (nops == 0) {
        MR_CUDA_TRY(c0, cudaEventRecord(c0->ev_copy[kHeadChunks], st));
        MR_CUDA_TRY(c0, cudaStreamWaitEvent(c0->copy_stream, c0->ev_copy[kHeadChunks], 0));
      }
      MR_CUDA_TRY(c0, cudaMemcpyAsync(c0->y_backup, hout, c0->dof * sizeof(double),
                                      cudaMemcpyHostToDevice, c0->copy_stream));
      c0->out_streamed = true;
      end_op = (size_t)tail_L - 2;
    }
  }
  for (size_t oi = first_op; oi < end_op; ++oi) {
    const Op& o = plan.ops[oi];
    if (o.type == Op::COUNT_SLOW) continue;
    if (o.type == Op::MISSING) {
      missing_stage = o.stage;
      break;
    }
    // one NVTX range per stage-plan op: slow evaluation f_E(j), implicit
    // evaluation f_I(j), implicit solve of stage i, explicit update of stage
    // i, fused chain of cell-local stages i..k
    const NvtxRange op_range(o.type == Op::SLOW     ? "slow f_E"
                             : o.type == Op::IMPL   ? "implicit f_I"
                             : o.type == Op::SOLVE  ? "implicit solve"
                             : o.type == Op::UPDATE ? "explicit update"
                                                    : "fast IVP chain",
                             o.type == Op::CHAIN ? o.stages.front() : o.stage,
                             o.type == Op::CHAIN ? o.stages.back() : -1);
    // profile classes: 0 fused fast IVPs, 1 explicit slow RHS (stencil),
    // 2 everything else (updates, implicit evaluations and solves)
    const int cls = o.type == Op::CHAIN ? 0 : (o.type == Op::SLOW ? 1 : 2);
    if (c0->profile) {
      cudaEventRecord(pool_event(c0, ev), st);
      timed.push_back({cls, ev});
      ev += 2;
    }
    if (o.type == Op::SLOW) {
      for (int r = 0; r < n; ++r) outs[r] = cs[r]->slots[plan.slot_of[o.stage]];
      int rc = eval_slow(cs, n, ycur.data(), outs.data(), st);
      if (rc) return rc;
    } else if (o.type == Op::IMPL) {
      for (int r = 0; r < n; ++r) outs[r] = cs[r]->slots[plan.islot_of[o.stage]];
      int rc = eval_implicit(cs, n, ycur.data(), outs.data(), st);
      if (rc) return rc;
    } else if (o.type == Op::SOLVE) {
      int rc = solve_stage(cs, n, o.stage, t, H, plan, ycur, st, &host_key);
      if (rc) return rc;
      if (host_key != MR_NO_FAIL) {
        if (c0->profile) cudaEventRecord(pool_event(c0, timed.back().second + 1), st);
        break;
      }
    } else if (o.type == Op::UPDATE) {
      for (int r = 0; r < n; ++r) {
        mr_ctx* c = cs[r];
        sdev(c);
        ChainStageDev sd;
        fill_chain_stage(c, o.stage, t, H, plan, sd);
        const double* f[MR_MAXREF];
        for (int q = 0; q < sd.nref; ++q) f[q] = c->slots[sd.ref_slot[q]];
        MR_CUDA_TRY(c, launch_update(ycur[r], c->y_work, sd.nref, f, sd.coef[0], c->dof, o.stage,
                                     c->d_fail, sst(c, st)));
        c->launches++;
        ycur[r] = c->y_work;
      }
    } else {  // CHAIN
      for (int r = 0; r < n; ++r) {
        mr_ctx* c = cs[r];
        ChainArgs a;
        std::memset(&a, 0, sizeof(a));
        a.nst = (int)o.stages.size();
        a.ndeg = ndeg_of(c);
        for (int q = 0; q < a.nst; ++q) fill_chain_stage(c, o.stages[q], t, H, plan, a.st[q]);
        a.tab = c->tab;
        a.y_in = ycur[r];
        a.y_out = c->y_work;
        for (int q = 0; q < (int)c->slots.size() && q < MR_MAXSLOT; ++q) a.fE[q] = c->slots[q];
        a.ncell = c->ncell;
        a.ncomp = c->ncomp;
        a.fail = c->d_fail;
        if (c->fast_kind == FK_CHEM) fill_chain_taus(c, a);
        sdev(c);
        if (c->fast_kind == FK_CHEM)
          MR_CUDA_TRY(c, launch_chem_chain(ccfg, a, *c->chemP, sst(c, st)));
        else
          MR_CUDA_TRY(c, launch_chain(cfg, a, c->fastA, sst(c, st)));
        c->launches++;
        ycur[r] = c->y_work;
      }
    }
    if (c0->profile) cudaEventRecord(pool_event(c0, timed.back().second + 1), st);
  }
  if (tail_L >= 0 && missing_stage < 0 && host_key == MR_NO_FAIL) {
    int rc = tail_download(c0, plan, tail_L, t, H, ccfg, ycur[0], hout, st);
    if (rc) return rc;
    ycur[0] = c0->y_work;
  }

  // combine failure keys (min over slabs / ranks)
  if (n == 1 && c0->comm) {
    MR_NCCL_TRY(c0, AllReduce(c0->d_fail, c0->d_fail, 1, ncclUint64, ncclMin, c0->comm, st));
  }
  for (int r = 0; r < n; ++r) {
    sdev(cs[r]);
    MR_CUDA_TRY(cs[r], cudaMemcpyAsync(cs[r]->h_fail, cs[r]->d_fail, sizeof(unsigned long long),
                                       cudaMemcpyDeviceToHost, sst(cs[r], st)));
  }
  if (async) {
    mr_ctx::Pending& pd = c0->pending;
    pd.active = true;
    pd.plan = plan;
    pd.t = t;
    pd.H = H;
    pd.missing_stage = missing_stage;
    pd.host_key = host_key;
    pd.timed = timed;
    pd.ycur = ycur[0];
    return MR_OK;
  }
  return domain_finish(cs, n, plan, t, H, missing_stage, host_key, timed, ycur.data(), counters,
                       fail_stage);
}

// waits for the enqueued step, decodes the failure key, adds the counters and
// commits the state (domain_step's second half)
int domain_finish(mr_ctx** cs, int n, const Plan& plan, double t, double H, int missing_stage,
                  unsigned long long host_key, const std::vector<std::pair<int, size_t>>& timed,
                  const double* const* ycur, uint64_t* counters, int* fail_stage)
{
  mr_ctx* c0 = cs[0];
  if (fail_stage) *fail_stage = -1;
  for (int r = 0; r < n; ++r) {
    if (!cs[r]->in_domain && r > 0) break;  // virtual ranks share the first slab's stream
    sdev(cs[r]);
    MR_CUDA_TRY(c0, cudaStreamSynchronize(cs[r]->stream));
  }
  unsigned long long key = MR_NO_FAIL;
  for (int r = 0; r < n; ++r) key = std::min(key, *cs[r]->h_fail);
  key = std::min(key, host_key);

  if (c0->profile) {
    c0->prof_chem = c0->prof_slow = c0->prof_other = 0.0;
    for (auto& tv : timed) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, c0->ev_pool[tv.second], c0->ev_pool[tv.second + 1]);
      (tv.first == 0 ? c0->prof_chem : tv.first == 1 ? c0->prof_slow : c0->prof_other) += ms;
    }
  }

  if (missing_stage >= 0 && key == MR_NO_FAIL) {
    // stages before the missing reference ran; count them, report the failure
    const Coupling& cp = c0->cp;
    uint64_t part[8] = {};
    add_counts_partial(c0, plan, t, H, missing_stage, 0, 0, part);
    if (counters)
      for (int q = 0; q < 8; ++q) counters[q] += part[q];
    for (int r = 0; r < n; ++r) {
      cs[r]->fail_mri = missing_stage;
      cs[r]->fail_sub = cs[r]->fail_inner = -1;
    }
    if (cp.kind[missing_stage] == MR_STAGE_FAST_IVP) {
      if (fail_stage) *fail_stage = missing_stage;
      return set_err(c0, MR_INTEGRATION,
                     "build_forcing: missing explicit value at stage " + std::to_string(missing_stage));
    }
    return set_err(c0, MR_CONTRACT, "axpy_into: length mismatch");
  }

  if (key != MR_NO_FAIL) {
    const int fs = (int)(key >> 40);
    const int fsub = (int)((key >> 8) & 0xFFFFFFFFull);
    const int finner = (int)(key & 0xFFull);
    uint64_t part[8] = {};
    const bool ivp = c0->cp.kind[fs] == MR_STAGE_FAST_IVP;
    add_counts_partial(c0, plan, t, H, fs, ivp ? fsub : 0, finner, part);
    if (counters)
      for (int q = 0; q < 8; ++q) counters[q] += part[q];
    for (int r = 0; r < n; ++r) {
      cs[r]->fail_mri = fs;
      cs[r]->fail_sub = ivp ? fsub : -1;
      cs[r]->fail_inner = ivp ? finner : -1;
    }
    if (fail_stage) *fail_stage = ivp ? finner : fs;
    if (ivp)
      return set_err(c0, MR_INTEGRATION,
                     finner == c0->tab.s ? "erk_step: non-finite result"
                                         : "erk_step: non-finite stage value");
    if (c0->cp.kind[fs] == MR_STAGE_IMPLICIT_SOLVE && finner == 0)
      return set_err(c0, MR_INTEGRATION,
                     "mri_step: non-finite stage data at stage " + std::to_string(fs));
    if (c0->cp.kind[fs] == MR_STAGE_IMPLICIT_SOLVE && finner == 2)
      return set_err(c0, MR_INTEGRATION,
                     "mri_step: nonlinear solve failed at stage " + std::to_string(fs));
    return set_err(c0, MR_INTEGRATION, "mri_step: non-finite state at stage " + std::to_string(fs));
  }
  if (counters) add_counts_full(c0, plan, t, H, counters);
  for (int r = 0; r < n; ++r) {
    mr_ctx* c = cs[r];
    if (ycur[r] == c->y_work) std::swap(c->y_state, c->y_work);
    c->fail_mri = c->fail_sub = c->fail_inner = -1;
  }
  return MR_OK;
}

int read_coupling_text(const char* text, Coupling& cp, std::string& err)
{
  std::istringstream in(text);
  std::string magic, version, name, sf, df;
  in >> magic >> version >> name >> sf >> df;
  if (magic != "mri-coupling" || version != "v1" || sf.rfind("s=", 0) != 0 ||
      df.rfind("degrees=", 0) != 0) {
    err = "import_coupling: bad header";
    return MR_CONTRACT;
  }
  cp = Coupling();
  cp.name = name;
  cp.s = std::atoi(sf.c_str() + 2);
  const int d = std::atoi(df.c_str() + 8);
  if (cp.s < 2 || d < 1 || cp.s > kMaxStages) {
    err = "import_coupling: bad dimensions";
    return MR_CONTRACT;
  }
  for (int i = 0; i < cp.s; ++i) in >> cp.c[i];
  for (int i = 0; i < cp.s; ++i) {
    std::string tok;
    in >> tok;
    if (tok == "fast-ivp") cp.kind[i] = MR_STAGE_FAST_IVP;
    else if (tok == "implicit-solve") cp.kind[i] = MR_STAGE_IMPLICIT_SOLVE;
    else if (tok == "explicit-update") cp.kind[i] = MR_STAGE_EXPLICIT_UPDATE;
    else {
      err = "import_coupling: unknown stage kind '" + tok + "'";
      return MR_CONTRACT;
    }
  }
  cp.ndeg_g = cp.ndeg_o = d;
  cp.gamma.assign((size_t)d * cp.s * cp.s, 0.0);
  cp.omega.assign((size_t)d * cp.s * cp.s, 0.0);
  for (auto& v : cp.gamma) in >> v;
  for (auto& v : cp.omega) in >> v;
  if (!in) {
    err = "import_coupling: truncated input";
    return MR_CONTRACT;
  }
  return finalize(cp, err) ? MR_OK : MR_CONTRACT;
}

}  // namespace

// a context with an asynchronous step in flight accepts only mr_mri_step_wait
// (and the read-only queries): every entry point that touches the state, the
// buffers or the configuration calls this first
static int pending_guard(mr_ctx* c)
{
  if (c && c->pending.active)
    return set_err(c, MR_CONTRACT, "an asynchronous step is in flight: call mr_mri_step_wait first");
  return MR_OK;
}


// ---------------------------------------------------------------------------
// multi-device domain helpers (mr_ctx_create_multi)
// ---------------------------------------------------------------------------
// f applied to every slab of a domain; the first failure's message becomes the
// domain's
template <class F>
static int for_slabs(mr_ctx* d, F&& f)
{
  for (mr_ctx* sl : d->slabs) {
    const int rc = f(sl);
    if (rc) return set_err(d, rc, sl->err);
  }
  return MR_OK;
}

// after a multi-slab call: the first slab carries the step's error message
static int domain_rc(mr_ctx* d, int rc)
{
  if (rc) d->err = d->slabs[0]->err;
  return rc;
}

// host <-> slab copies of a domain-wide species-major buffer
// Y[comp][global cell]: slab r's component k is one contiguous chunk at
// comp * ncell_global + i0 * plane, so each slab is one 2D copy (ncomp rows)
static int domain_copy(mr_ctx* d, const double* host_in, double* host_out, double* const* dev_bufs,
                bool to_dev)
{
  const size_t gpitch = d->ncell * sizeof(double);
  for (size_t r = 0; r < d->slabs.size(); ++r) {
    mr_ctx* sl = d->slabs[r];
    cudaSetDevice(sl->device);
    const size_t lpitch = sl->ncell * sizeof(double);
    const size_t off = (size_t)sl->i0 * sl->plane;
    if (to_dev)
      MR_CUDA_TRY(d, cudaMemcpy2DAsync(dev_bufs[r], lpitch, host_in + off, gpitch, lpitch,
                                       (size_t)sl->ncomp, cudaMemcpyHostToDevice, sl->stream));
    else
      MR_CUDA_TRY(d, cudaMemcpy2DAsync(host_out + off, gpitch, dev_bufs[r], lpitch, lpitch,
                                       (size_t)sl->ncomp, cudaMemcpyDeviceToHost, sl->stream));
  }
  for (mr_ctx* sl : d->slabs) {
    cudaSetDevice(sl->device);
    MR_CUDA_TRY(d, cudaStreamSynchronize(sl->stream));
  }
  return MR_OK;
}

// a slab's share of a domain-wide host array (species-major), as a vector
static std::vector<double> domain_slice(const mr_ctx* d, const mr_ctx* sl, const double* host)
{
  std::vector<double> v(sl->dof);
  const size_t off = (size_t)sl->i0 * sl->plane;
  for (int k = 0; k < sl->ncomp; ++k)
    std::memcpy(v.data() + (size_t)k * sl->ncell, host + (size_t)k * d->ncell + off,
                sl->ncell * sizeof(double));
  return v;
}

// the contexts a step runs over: the slabs of a domain, or the context itself
static std::vector<mr_ctx*> members(mr_ctx* c)
{
  return c->slabs.empty() ? std::vector<mr_ctx*>{c} : c->slabs;
}

// one RHS of a domain-wide host vector: scatter into each slab's scratch,
// evaluate (kind 0 fast, 1 slow, 2 implicit), gather (Mode A, multi-GPU)
// one fast-partition RHS evaluation between device buffers
static int eval_fast_dev(mr_ctx* c, const double* in, double* out, cudaStream_t st)
{
  if (c->fast_kind == FK_CHEM) {
    ChemCfg ccfg;
    TableDev t4{};
    t4.s = 4;
    if (chem_pick(&ccfg, c->ncomp, c->S, c->R, t4, 1))
      return set_err(c, MR_CONTRACT, "unsupported mechanism size");
    MR_CUDA_TRY(c, launch_chem_rhs(ccfg, in, out, c->ncell, c->ncomp, *c->chemP, st));
  } else {
    ChainCfg cfg;
    if (chain_pick(&cfg, c->fast_kind, c->ncomp, 4, 1))
      return set_err(c, MR_CONTRACT, "unsupported component count");
    MR_CUDA_TRY(c, launch_fast_rhs(cfg, in, out, c->ncell, c->ncomp, c->fastA, st));
  }
  c->launches++;
  return MR_OK;
}
static int domain_rhs(mr_ctx* d, int kind, const double* y, double* out)
{
  const int n = (int)d->slabs.size();
  std::vector<double*> in(n), o(n);
  std::vector<const double*> ci(n);
  for (int r = 0; r < n; ++r) {
    mr_ctx* sl = d->slabs[r];
    cudaSetDevice(sl->device);
    if (!sl->scr_in) MR_CUDA_TRY(d, cudaMalloc(&sl->scr_in, sl->dof * sizeof(double)));
    if (!sl->scr_out) MR_CUDA_TRY(d, cudaMalloc(&sl->scr_out, sl->dof * sizeof(double)));
    in[r] = sl->scr_in;
    ci[r] = sl->scr_in;
    o[r] = sl->scr_out;
  }
  int rc = domain_copy(d, y, nullptr, in.data(), true);
  if (rc) return rc;
  if (kind == 0) {
    for (int r = 0; r < n; ++r) {
      cudaSetDevice(d->slabs[r]->device);
      rc = eval_fast_dev(d->slabs[r], in[r], o[r], d->slabs[r]->stream);
      if (rc) return domain_rc(d, rc);
    }
  } else if (kind == 1) {
    rc = eval_slow(d->slabs.data(), n, ci.data(), o.data(), d->slabs[0]->stream);
    if (rc) return domain_rc(d, rc);
  } else {
    rc = eval_implicit(d->slabs.data(), n, ci.data(), o.data(), d->slabs[0]->stream);
    if (rc) return domain_rc(d, rc);
  }
  return domain_copy(d, nullptr, out, o.data(), false);
}

#define MR_FORWARD(c, expr)                                            \
  do {                                                                 \
    if ((c) && !(c)->slabs.empty()) return for_slabs((c), [&](mr_ctx* sl_) { return (expr); }); \
  } while (0)
#define MR_NOT_ON_DOMAIN(c, what)                                                          \
  do {                                                                                     \
    if ((c) && !(c)->slabs.empty())                                                        \
      return set_err((c), MR_CONTRACT, std::string(what) + ": not available on a multi-device domain"); \
  } while (0)

// ===========================================================================
// C-ABI
// ===========================================================================
extern "C" {

int mr_version(void) { return 1; }

int mr_ctx_create(int device, mr_ctx** out)
{
  if (!out) return MR_CONTRACT;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return MR_CUDA;
  if (device < 0 || device >= ndev) return MR_CONTRACT;
  if (cudaSetDevice(device) != cudaSuccess) return MR_CUDA;
  mr_ctx* c = new mr_ctx();
  c->device = device;
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMalloc(&c->d_fail, sizeof(unsigned long long)) != cudaSuccess ||
      cudaMallocHost(&c->h_fail, sizeof(unsigned long long)) != cudaSuccess ||
      cudaMalloc(&c->d_red, sizeof(double) * (reduce_blocks() + 8)) != cudaSuccess ||
      cudaMallocHost(&c->h_red, sizeof(double) * 8) != cudaSuccess) {
    delete c;
    return MR_CUDA;
  }
  *out = c;
  return MR_OK;
}

// one process, several GPUs (SURVEY.md 8(b) mr_ctx_create(devices, n)): a
// domain context owning one slab context per listed device
int mr_ctx_create_multi(const int* devices, int n, mr_ctx** out)
{
  if (!out || !devices || n < 1) return MR_CONTRACT;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return MR_CUDA;
  for (int i = 0; i < n; ++i)
    if (devices[i] < 0 || devices[i] >= ndev) return MR_CONTRACT;
  mr_ctx* d = new mr_ctx();
  d->device = devices[0];
  for (int i = 0; i < n; ++i) {
    mr_ctx* sl = nullptr;
    const int rc = mr_ctx_create(devices[i], &sl);
    if (rc) {
      mr_ctx_destroy(d);
      return rc;
    }
    d->slabs.push_back(sl);
    sl->in_domain = true;
    cudaSetDevice(sl->device);
    if (cudaEventCreateWithFlags(&sl->ev_send, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&sl->ev_recv, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&sl->ev_dot, cudaEventDisableTiming) != cudaSuccess) {
      mr_ctx_destroy(d);
      return MR_CUDA;
    }
  }
  d->stream = d->slabs[0]->stream;  // mr_stream(): the first slab's stream
  // direct NVLink copies between the GPUs that exchange ghost planes (ring
  // neighbours) and dot-product scalars (with the first slab's GPU)
  for (int i = 0; i < n; ++i)
    for (int j : {(i + 1) % n, (i + n - 1) % n, 0}) {
      const int a = devices[i], b = devices[j];
      int ok = 0;
      if (a == b || cudaDeviceCanAccessPeer(&ok, a, b) != cudaSuccess || !ok) continue;
      cudaSetDevice(a);
      if (cudaDeviceEnablePeerAccess(b, 0) != cudaSuccess) cudaGetLastError();  // already enabled
    }
  cudaSetDevice(devices[0]);
  *out = d;
  return MR_OK;
}

void mr_ctx_destroy(mr_ctx* c)
{
  if (!c) return;
  if (!c->slabs.empty() || (!c->stream && !c->in_domain)) {  // a domain: its slabs own everything
    for (mr_ctx* sl : c->slabs) mr_ctx_destroy(sl);
    delete c;
    return;
  }
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  free_state(c);
  for (void*& p : c->chem_bufs) free_dev(p);
  delete c->chemP;
  free_dev_t(c->d_prof);
  free_dev_t(c->d_fail);
  free_dev_t(c->d_red);
  free_dev_t(c->cg_part);
  free_dev_t(c->cg_part2);
  free_dev_t(c->cg_sc);
  free_dev_t(c->cg_gather);
  if (c->h_fail) cudaFreeHost(c->h_fail);
  if (c->h_red) cudaFreeHost(c->h_red);
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  if (c->comm && nccl_api().ok) nccl_api().CommDestroy(c->comm);
  cudaStreamDestroy(c->stream);
  if (c->ev_async_in) cudaEventDestroy(c->ev_async_in);
  if (c->ev_async_out) cudaEventDestroy(c->ev_async_out);
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  for (cudaEvent_t e : c->ev_copy)
    if (e) cudaEventDestroy(e);
  if (c->ev_pack) cudaEventDestroy(c->ev_pack);
  if (c->ev_halo) cudaEventDestroy(c->ev_halo);
  if (c->ev_send) cudaEventDestroy(c->ev_send);
  if (c->ev_recv) cudaEventDestroy(c->ev_recv);
  if (c->ev_dot) cudaEventDestroy(c->ev_dot);
  delete c;
}

const char* mr_last_error(const mr_ctx* c) { return c ? c->err.c_str() : "null context"; }

int mr_grid_set(mr_ctx* c, int n0, int n1, int n2, int n_comp, double length, int i0, int n0_local)
{
  if (!c) return MR_CONTRACT;
  if (int g = pending_guard(c)) return g;
  if (n0 < 1 || n1 < 1 || n2 < 1 || n_comp < 1 || !(length > 0.0) || i0 < 0 || n0_local < 1 ||
      i0 + n0_local > n0)
    return set_err(c, MR_CONTRACT, "mr_grid_set: bad grid");
  if (!c->slabs.empty()) {  // a domain owns the whole grid; equal slabs in device order
    const int P = (int)c->slabs.size();
    if (i0 != 0 || n0_local != n0 || n0 < P)
      return set_err(c, MR_CONTRACT,
                     "mr_grid_set: a multi-device domain owns the whole grid (i0 = 0, n0_local = n0 >= devices)");
    const int base = n0 / P, rem = n0 % P;
    for (int r = 0; r < P; ++r) {
      const int rc = mr_grid_set(c->slabs[r], n0, n1, n2, n_comp, length, r * base + std::min(r, rem),
                                 base + (r < rem ? 1 : 0));
      if (rc) return set_err(c, rc, c->slabs[r]->err);
    }
  }
  cudaSetDevice(c->device);
  free_state(c);
  c->n0 = n0; c->n1 = n1; c->n2 = n2; c->ncomp = n_comp; c->length = length;
  c->i0 = i0; c->n0l = n0_local;
  c->plane = (size_t)n1 * n2;
  c->ncell = c->plane * n0_local;
  c->dof = c->ncell * n_comp;
  c->has_grid = true;
  return MR_OK;
}

int mr_coupling_load(mr_ctx* c, int s, int n_deg, const double* cc, const int* kind,
                     const double* gamma, const double* omega)
{
  if (int g = pending_guard(c)) return g;
  MR_FORWARD(c, mr_coupling_load(sl_, s, n_deg, cc, kind, gamma, omega));
  if (!c || !cc || !kind || s < 2 || s > kMaxStages || n_deg < 1 || n_deg > 8)
    return set_err(c, MR_CONTRACT, "mr_coupling_load: bad arguments");
  Coupling cp;
  cp.name = "loaded";
  cp.s = s;
  cp.ndeg_g = gamma ? n_deg : 0;
  cp.ndeg_o = omega ? n_deg : 0;
  for (int i = 0; i < s; ++i) {
    cp.c[i] = cc[i];
    cp.kind[i] = kind[i];
  }
  if (gamma) cp.gamma.assign(gamma, gamma + (size_t)n_deg * s * s);
  if (omega) cp.omega.assign(omega, omega + (size_t)n_deg * s * s);
  std::string err;
  if (!finalize(cp, err)) return set_err(c, MR_CONTRACT, err);
  if (std::max(cp.degrees(), 1) > MR_MAXDEG)
    return set_err(c, MR_CONTRACT, "forcing polynomial degree > 2 not supported");
  c->cp = cp;
  c->has_coupling = true;
  return MR_OK;
}

int mr_coupling_load_text(mr_ctx* c, const char* text)
{
  if (!c || !text) return MR_CONTRACT;
  if (int g = pending_guard(c)) return g;
  MR_FORWARD(c, mr_coupling_load_text(sl_, text));
  Coupling cp;
  std::string err;
  int rc = read_coupling_text(text, cp, err);
  if (rc) return set_err(c, rc, err);
  if (std::max(cp.degrees(), 1) > MR_MAXDEG)
    return set_err(c, MR_CONTRACT, "forcing polynomial degree > 2 not supported");
  c->cp = cp;
  c->has_coupling = true;
  return MR_OK;
}

int mr_table_load(mr_ctx* c, int s, const double* A, const double* b, const double* cc)
{
  if (int g = pending_guard(c)) return g;
  MR_FORWARD(c, mr_table_load(sl_, s, A, b, cc));
  if (!c || !A || !b || !cc || s < 1 || s > MR_MAXS)
    return set_err(c, MR_CONTRACT, "mr_table_load: bad arguments");
  TableDev t{};
  t.s = s;
  for (int i = 0; i < s; ++i) {
    for (int j = 0; j < s; ++j) {
      t.A[i][j] = A[i * s + j];
      if (j >= i && A[i * s + j] != 0.0)
        return set_err(c, MR_CONTRACT, "erk_step: table must be explicit");
    }
    t.b[i] = b[i];
    t.c[i] = cc[i];
  }
  c->tab = t;
  c->has_table = true;
  return MR_OK;
}

int mr_set_substeps(mr_ctx* c, int m)
{
  if (int g = pending_guard(c)) return g;
  MR_FORWARD(c, mr_set_substeps(sl_, m));
  if (!c || m < 1) return set_err(c, MR_CONTRACT, "m must be >= 1");
  c->m = m;
  return MR_OK;
}

int mr_fast_chemistry(mr_ctx* c, int S, int R, double rho, const double* species,
                      const double* reactions, const int* rspecies)
{
  if (int g = pending_guard(c)) return g;
  MR_FORWARD(c, mr_fast_chemistry(sl_, S, R, rho, species, reactions, rspecies));
  if (!c || S < 1 || R < 1 || !(rho > 0.0) || !species || !reactions || !rspecies)
    return set_err(c, MR_CONTRACT, "mr_fast_chemistry: bad arguments");
  cudaSetDevice(c->device);
  for (void*& p : c->chem_bufs) free_dev(p);
  c->chem_bufs.clear();
  const int Sp = (S + 1 + 31) / 32 * 32;
  std::vector<double> sp(9 * (size_t)Sp, 0.0);
  for (int k = 0; k < S; ++k) {
    const double W = species[5 * k], a = species[5 * k + 1], b = species[5 * k + 2];
    const double h0 = species[5 * k + 3], s0 = species[5 * k + 4];
    const double rW = kRu / W;
    sp[0 * Sp + k] = h0;
    sp[1 * Sp + k] = a;
    sp[2 * Sp + k] = 0.5 * b;
    sp[3 * Sp + k] = s0;
    sp[4 * Sp + k] = rho / W;
    sp[5 * Sp + k] = W / rho;
    sp[6 * Sp + k] = rW * h0;
    sp[7 * Sp + k] = rW * (a - 1.0);
    sp[8 * Sp + k] = rW * (0.5 * b);
  }
  std::vector<double4> rx(R);
  std::vector<int4> rs(R);
  std::vector<int> cnt(S + 1, 0);
  for (int j = 0; j < R; ++j) {
    int q[4];
    for (int t = 0; t < 4; ++t) {
      q[t] = rspecies[4 * j + t];
      if (q[t] >= S || (q[t] < 0 && (t == 0 || t == 2)))
        return set_err(c, MR_CONTRACT, "mr_fast_chemistry: bad species index");
      if (q[t] >= 0) cnt[q[t] + 1]++;
    }
    const int nr = 1 + (q[1] >= 0), np = 1 + (q[3] >= 0);
    rx[j] = make_double4(reactions[3 * j], reactions[3 * j + 1], reactions[3 * j + 2],
                         (double)(np - nr));
    rs[j] = make_int4(q[0], q[1] < 0 ? S : q[1], q[2], q[3] < 0 ? S : q[3]);
  }
  for (int k = 0; k < S; ++k) cnt[k + 1] += cnt[k];
  std::vector<int> ent(std::max(cnt[S], 1));
  std::vector<int> fill(S, 0);
  for (int j = 0; j < R; ++j)
    for (int t = 0; t < 4; ++t) {
      const int k = rspecies[4 * j + t];
      if (k < 0) continue;
      ent[cnt[k] + fill[k]++] = 2 * j + (t >= 2 ? 1 : 0);
    }
  auto up = [&](const void* h, size_t bytes) -> void* {
    void* d = nullptr;
    if (cudaMalloc(&d, bytes) != cudaSuccess) return nullptr;
    cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice);
    c->chem_bufs.push_back(d);
    return d;
  };
  // chemistry kernel parameters: per-species data in the constant bank,
  // reaction records + production lists in a blob staged into shared memory
  if (S + 1 > MR_CHEM_MAXS || R > MR_CHEM_MAXR)
    return set_err(c, MR_CONTRACT, "mechanism too large for the chemistry kernel (S<=63)");
  if (!c->chemP) c->chemP = new ChemParams();
  ChemParams& P = *c->chemP;
  std::memset(&P, 0, sizeof(P));
  P.S = S;
  P.R = R;
  P.RuP = kRu / kPatm;
#ifdef MR_PHASE_PROF
  {
    unsigned long long* pp = nullptr;
    MR_CUDA_TRY(c, cudaMalloc(&pp, 8 * sizeof(unsigned long long)));
    MR_CUDA_TRY(c, cudaMemset(pp, 0, 8 * sizeof(unsigned long long)));
    c->chem_bufs.push_back(pp);
    P.prof = pp;
  }
#endif
  for (int k = 0; k < S; ++k) {
    P.h0[k] = sp[0 * Sp + k]; P.a[k] = sp[1 * Sp + k]; P.hb[k] = sp[2 * Sp + k];
    P.s0[k] = sp[3 * Sp + k]; P.rhoW[k] = sp[4 * Sp + k]; P.Wrho[k] = sp[5 * Sp + k];
    P.c0[k] = sp[6 * Sp + k]; P.c1[k] = sp[7 * Sp + k]; P.c2[k] = sp[8 * Sp + k];
  }
  {
    ChemCfg lay;
    TableDev t4{};
    t4.s = 4;
    const int nnz = cnt[S];
    // blob bound: records + entries + per-list padding (<= 3 per list)
    const size_t blob_bound = (size_t)R * sizeof(ChemRec) +
                              4 * ((size_t)nnz + 2 * 3 * (size_t)S * MR_CHEM_MAXCHUNK) + 16;
    int rcz = 0, nch = 0;
    if (chem_pick(&lay, S + 1, S, R, t4, 1) ||
        chem_chunking(lay, S, R, blob_bound, &rcz, &nch))
      return set_err(c, MR_CONTRACT, "mechanism too large for the chemistry kernel's shared memory");
    P.rc = rcz;
    P.nchunk = nch;
    std::vector<ChemRec> recs(R);
    for (int j = 0; j < R; ++j) {
      ChemRec& r = recs[j];
      std::memset(&r, 0, sizeof(r));
      r.lnA = rx[j].x; r.beta = rx[j].y; r.EaR = rx[j].z;
      r.r1o = (unsigned)rs[j].x * 512u; r.r2o = (unsigned)rs[j].y * 512u;
      r.p1o = (unsigned)rs[j].z * 256u; r.p2o = (unsigned)rs[j].w * 256u;
    }
    const unsigned qrow = 256u;
    const unsigned zero_off = (unsigned)rcz * qrow;  // all-zero row right after q
    std::vector<unsigned> ents;
    for (int k = 0; k < S; ++k)
      for (int ch2 = 0; ch2 < nch; ++ch2) {
        unsigned short st4[2], n4[2];
        for (int sign = 0; sign < 2; ++sign) {  // 0: producing (+), 1: consuming (-)
          while (ents.size() % 4) ents.push_back(zero_off);
          st4[sign] = (unsigned short)(ents.size() / 4);
          size_t n0 = ents.size();
          for (int q2 = cnt[k]; q2 < cnt[k + 1]; ++q2) {
            const int j = ent[q2] >> 1, prod = ent[q2] & 1;
            if ((prod == 1) != (sign == 0)) continue;
            if (j < ch2 * rcz || j >= (ch2 + 1) * rcz) continue;
            ents.push_back((unsigned)(j - ch2 * rcz) * qrow);
          }
          while ((ents.size() - n0) % 4) ents.push_back(zero_off);
          n4[sign] = (unsigned short)((ents.size() - n0) / 4);
        }
        P.lst[k][ch2] = make_ushort4(st4[0], n4[0], st4[1], n4[1]);
      }
    while (ents.size() % 4) ents.push_back(zero_off);
    // every shared-memory offset the kernel will add to a lane address stays
    // inside its table (compute-sanitizer is not available on the GPU pool:
    // the bounds of all data-dependent shared accesses are checked here)
    for (const ChemRec& r : recs)
      if (r.r1o >= (unsigned)(S + 1) * 512u || r.r2o >= (unsigned)(S + 1) * 512u ||
          r.p1o >= (unsigned)(S + 1) * 256u || r.p2o >= (unsigned)(S + 1) * 256u)
        return set_err(c, MR_CONTRACT, "mr_fast_chemistry: species offset outside its table");
    for (unsigned e : ents)
      if (e > zero_off || e % 256u)
        return set_err(c, MR_CONTRACT, "mr_fast_chemistry: production entry outside the rate buffer");
    for (int k = 0; k < S; ++k)
      for (int ch2 = 0; ch2 < nch; ++ch2) {
        const ushort4 L = P.lst[k][ch2];
        if ((size_t)(L.x + L.y) * 4 > ents.size() || (size_t)(L.z + L.w) * 4 > ents.size())
          return set_err(c, MR_CONTRACT, "mr_fast_chemistry: production list outside the blob");
      }
    const size_t rec_bytes = (size_t)R * sizeof(ChemRec);
    const size_t blob_bytes = rec_bytes + ents.size() * 4;
    if (blob_bytes > blob_bound)
      return set_err(c, MR_CONTRACT, "chemistry blob exceeds its shared-memory budget");
    std::vector<unsigned char> blob(blob_bytes);
    std::memcpy(blob.data(), recs.data(), rec_bytes);
    std::memcpy(blob.data() + rec_bytes, ents.data(), ents.size() * 4);
    P.blob = (const uint4*)up(blob.data(), blob_bytes);
    if (!P.blob) return set_err(c, MR_CUDA, "mr_fast_chemistry: device allocation failed");
    P.blob_words = (int)(blob_bytes / 16);
    P.ent_base = (int)(rec_bytes / 16);
  }
  c->S = S;
  c->R = R;
  c->rho = rho;
  c->fast_kind = FK_CHEM;
  // fp64 work per RHS evaluation + its RK4/forcing arithmetic (DESIGN.md
  // "Roofline accounting"): FMA = 2, + - * / = 1, exp = 34 (the branch-free
  // sequence of kernels_chem.cuh: 15 FMA + 1 add + 1 mul), log = 40.
  const double ce = 34.0, cl = 40.0;
  double f = 0.0;
  f += 8.0 + cl + 3.0;                      // T(e) root, log T, 1/T, RT/P, P/RT
  f += S * (6.0 + 6.0 + ce + 5.0 + 1.0);    // e(T) sums, g, exp, C/E'/D', W/rho
  for (int j = 0; j < R; ++j) {              // kf exponent, exp, forward/reverse, q:
    const int nr = 1 + (rspecies[4 * j + 1] >= 0), np = 1 + (rspecies[4 * j + 3] >= 0);
    f += 4.0 + ce + 2.0 + 2.0 * (nr - 1) + (np - 1);  // products of present operands only
  }
  f += cnt[S];                              // production sums
  f += (S + 1) * 7.0;                       // forcing Horner + f + r, stage, out
  c->chem_flops = f;
  return MR_OK;
}

int mr_fast_linear(mr_ctx* c, const double* A)
{
  if (int g = pending_guard(c)) return g;
  MR_FORWARD(c, mr_fast_linear(sl_, A));
  if (!c || !A || !c->has_grid || c->ncomp > MR_MAXLIN)
    return set_err(c, MR_CONTRACT, "mr_fast_linear: needs grid with n_comp <= 8");
  c->fastA.n = c->ncomp;
  for (int i = 0; i < c->ncomp * c->ncomp; ++i) c->fastA.A[i] = A[i];
  c->fast_kind = FK_LINEAR;
  return MR_OK;
}

int mr_fast_none(mr_ctx* c)
{
  if (!c) return MR_CONTRACT;
  if (int g = pending_guard(c)) return g;
  MR_FORWARD(c, mr_fast_none(sl_));
  c->fast_kind = FK_NONE;
  return MR_OK;
}

int mr_slow_stencil(mr_ctx* c, int order, double diffusion, const double* u, const double* prof,
                    int nmax)
{
  if (int g = pending_guard(c)) return g;
  MR_FORWARD(c, mr_slow_stencil(sl_, order, diffusion, u, prof, nmax));
  if (!c || !c->has_grid || (order != 2 && order != 4 && order != 8) || diffusion < 0.0)
    return set_err(c, MR_CONTRACT, "mr_slow_stencil: bad arguments (order 2/4/8, grid first)");
  cudaSetDevice(c->device);
  free_dev_t(c->d_prof);
  c->order = order;
  c->M = order / 2;
  c->D = diffusion;
  if (prof) {
    if (nmax < std::max(c->n0, std::max(c->n1, c->n2)))
      return set_err(c, MR_CONTRACT, "mr_slow_stencil: profile length < grid size");
    MR_CUDA_TRY(c, cudaMalloc(&c->d_prof, sizeof(double) * 6 * nmax));
    MR_CUDA_TRY(c, cudaMemcpy(c->d_prof, prof, sizeof(double) * 6 * nmax, cudaMemcpyHostToDevice));
    c->vel_kind = 1;
    c->nmax = nmax;
  } else {
    if (!u) return set_err(c, MR_CONTRACT, "mr_slow_stencil: need u or profiles");
    for (int d = 0; d < 3; ++d) c->u[d] = u[d];
    c->vel_kind = 0;
  }
  c->slow_kind = SK_STENCIL;
  c->imex = false;  // mr_slow_implicit_diffusion adds the implicit partition
  c->halo_elems = 0;
  free_dev_t(c->send_lo);
  free_dev_t(c->send_hi);
  free_dev_t(c->recv_lo);
  free_dev_t(c->recv_hi);
  return MR_OK;
}

static int ensure_scratch(mr_ctx* c);

int mr_slow_implicit_diffusion(mr_ctx* c, double d_impl, int cg_iters)
{
  if (int g = pending_guard(c)) return g;
  MR_FORWARD(c, mr_slow_implicit_diffusion(sl_, d_impl, cg_iters));
  if (!c || c->slow_kind != SK_STENCIL || !(d_impl >= 0.0) || cg_iters < 0)
    return set_err(c, MR_CONTRACT,
                   "mr_slow_implicit_diffusion: needs the stencil plugin, d_impl >= 0, cg_iters >= 0");
  c->imex = true;
  c->d_impl = d_impl;
  c->cg_iters = cg_iters;
  return MR_OK;
}

int mr_newton_config(mr_ctx* c, double tolerance, double safety, int max_iters,
                     const double* weights)
{
  if (int g = pending_guard(c)) return g;
  if (!c->slabs.empty()) {
    if (weights && !c->has_grid) return set_err(c, MR_CONTRACT, "grid not set (mr_grid_set)");
    return for_slabs(c, [&](mr_ctx* sl_) {
      if (!weights) return mr_newton_config(sl_, tolerance, safety, max_iters, nullptr);
      const std::vector<double> w = domain_slice(c, sl_, weights);
      return mr_newton_config(sl_, tolerance, safety, max_iters, w.data());
    });
  }
  if (!c || !(tolerance > 0.0) || !(safety > 0.0) || safety > 1.0 || max_iters < 0)
    return set_err(c, MR_CONTRACT, "newton_solve: bad NewtonConfig");
  if (weights && !c->has_grid) return set_err(c, MR_CONTRACT, "grid not set (mr_grid_set)");
  cudaSetDevice(c->device);
  c->newton_tol = tolerance;
  c->newton_safety = safety;
  c->newton_max = max_iters;
  free_dev_t(c->newton_w);
  if (weights) {
    MR_CUDA_TRY(c, cudaMalloc(&c->newton_w, c->dof * sizeof(double)));
    MR_CUDA_TRY(c, cudaMemcpy(c->newton_w, weights, c->dof * sizeof(double), cudaMemcpyHostToDevice));
  }
  return MR_OK;
}

int mr_implicit_rhs(mr_ctx* c, double t, const double* y, double* out)
{
  (void)t;
  if (!c || !y || !out) return MR_CONTRACT;
  if (int g = pending_guard(c)) return g;
  if (!c->slabs.empty()) {
    if (!c->slabs[0]->imex)
      return set_err(c, MR_CONTRACT, "mr_implicit_rhs: no implicit partition configured");
    return domain_rhs(c, 2, y, out);
  }
  if (!c->imex) return set_err(c, MR_CONTRACT, "mr_implicit_rhs: no implicit partition configured");
  cudaSetDevice(c->device);
  int rc = ensure_scratch(c);
  if (rc) return rc;
  MR_CUDA_TRY(c, cudaMemcpyAsync(c->scr_in, y, c->dof * sizeof(double), cudaMemcpyHostToDevice,
                                 c->stream));
  const double* ycur = c->scr_in;
  double* o = c->scr_out;
  rc = eval_implicit(&c, 1, &ycur, &o, c->stream);
  if (rc) return rc;
  MR_CUDA_TRY(c, cudaMemcpyAsync(out, c->scr_out, c->dof * sizeof(double), cudaMemcpyDeviceToHost,
                                 c->stream));
  MR_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return MR_OK;
}

int mr_slow_linear(mr_ctx* c, const double* A)
{
  if (int g = pending_guard(c)) return g;
  MR_FORWARD(c, mr_slow_linear(sl_, A));
  if (!c || !A || !c->has_grid || c->ncomp > MR_MAXLIN)
    return set_err(c, MR_CONTRACT, "mr_slow_linear: needs grid with n_comp <= 8");
  c->imex = false;
  c->slowA.n = c->ncomp;
  for (int i = 0; i < c->ncomp * c->ncomp; ++i) c->slowA.A[i] = A[i];
  c->slow_kind = SK_LINEAR;
  return MR_OK;
}

int mr_slow_none(mr_ctx* c)
{
  if (!c) return MR_CONTRACT;
  if (int g = pending_guard(c)) return g;
  MR_FORWARD(c, mr_slow_none(sl_));
  c->slow_kind = SK_NONE;
  c->imex = false;
  return MR_OK;
}

int mr_state_upload(mr_ctx* c, const double* host)
{
  if (!c || !host) return MR_CONTRACT;
  if (int g = pending_guard(c)) return g;
  if (!c->slabs.empty()) {
    if (!c->has_grid) return set_err(c, MR_CONTRACT, "grid not set (mr_grid_set)");
    std::vector<double*> bufs;
    for (mr_ctx* sl : c->slabs) {
      cudaSetDevice(sl->device);
      if (int rc = ensure_state(sl)) return set_err(c, rc, sl->err);
      bufs.push_back(sl->y_state);
    }
    const int rc = domain_copy(c, host, nullptr, bufs.data(), true);
    for (mr_ctx* sl : c->slabs) sl->state_valid = rc == MR_OK;
    return rc;
  }
  cudaSetDevice(c->device);
  int rc = ensure_state(c);
  if (rc) return rc;
  MR_CUDA_TRY(c, cudaMemcpyAsync(c->y_state, host, c->dof * sizeof(double),
                                 cudaMemcpyHostToDevice, c->stream));
  MR_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  c->state_valid = true;
  return MR_OK;
}

int mr_state_download(mr_ctx* c, double* host)
{
  if (!c || !host) return MR_CONTRACT;
  if (int g = pending_guard(c)) return g;
  if (!c->slabs.empty()) {
    std::vector<double*> bufs;
    for (mr_ctx* sl : c->slabs) {
      if (!sl->y_state) return set_err(c, MR_CONTRACT, "no state");
      bufs.push_back(sl->y_state);
    }
    return domain_copy(c, nullptr, host, bufs.data(), false);
  }
  if (!c->y_state) return set_err(c, MR_CONTRACT, "no state");
  cudaSetDevice(c->device);
  MR_CUDA_TRY(c, cudaMemcpyAsync(host, c->y_state, c->dof * sizeof(double),
                                 cudaMemcpyDeviceToHost, c->stream));
  MR_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return MR_OK;
}

// the result of an asynchronous step becomes the state at mr_mri_step_wait
// (the commit is a host-side buffer swap): no pointer while one is pending
double* mr_state_device_ptr(mr_ctx* c)
{
  if (!c || pending_guard(c)) return nullptr;
  if (!c->slabs.empty()) {  // one buffer per GPU: no single pointer
    set_err(c, MR_CONTRACT, "mr_state_device_ptr: not available on a multi-device domain");
    return nullptr;
  }
  if (ensure_state(c)) return nullptr;
  return c->y_state;
}

size_t mr_state_dof(const mr_ctx* c) { return c ? c->dof : 0; }

int mr_mri_step(mr_ctx* c, double t, double H, uint64_t* counters, int* fail_stage)
{
  if (!c) return MR_CONTRACT;
  if (int g = pending_guard(c)) return g;
  if (!c->slabs.empty())
    return domain_rc(c, domain_step(c->slabs.data(), (int)c->slabs.size(), t, H, counters,
                                    fail_stage));
  cudaSetDevice(c->device);
  mr_ctx* cs[1] = {c};
  return domain_step(cs, 1, t, H, counters, fail_stage);
}

int mr_mri_step_async(mr_ctx* c, double t, double H, void* stream)
{
  if (!c) return MR_CONTRACT;
  if (int g = pending_guard(c)) return g;
  MR_NOT_ON_DOMAIN(c, "mr_mri_step_async");
  cudaSetDevice(c->device);
  if (!c->ev_async_in) {
    MR_CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_async_in, cudaEventDisableTiming));
    MR_CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_async_out, cudaEventDisableTiming));
  }
  cudaStream_t us = static_cast<cudaStream_t>(stream);
  MR_CUDA_TRY(c, cudaEventRecord(c->ev_async_in, us));  // after the caller's queued work
  MR_CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->ev_async_in, 0));
  mr_ctx* cs[1] = {c};
  const int rc = domain_step(cs, 1, t, H, nullptr, nullptr, true);
  // the caller's stream follows whatever was enqueued, also when the enqueue
  // failed part-way (kernels already queued keep reading the state)
  const cudaError_t e1 = cudaEventRecord(c->ev_async_out, c->stream);
  const cudaError_t e2 = cudaStreamWaitEvent(us, c->ev_async_out, 0);
  if (rc) {
    cudaStreamSynchronize(c->stream);
    c->pending = mr_ctx::Pending{};
    return rc;
  }
  if (e1 != cudaSuccess || e2 != cudaSuccess) {
    c->pending = mr_ctx::Pending{};
    return set_err(c, MR_CUDA, std::string("mr_mri_step_async: ") +
                                   cudaGetErrorString(e1 != cudaSuccess ? e1 : e2));
  }
  return MR_OK;
}

int mr_mri_step_wait(mr_ctx* c, uint64_t* counters, int* fail_stage)
{
  if (!c) return MR_CONTRACT;
  if (!c->pending.active) return set_err(c, MR_CONTRACT, "mr_mri_step_wait: no step in flight");
  cudaSetDevice(c->device);
  mr_ctx::Pending pd = std::move(c->pending);
  c->pending = mr_ctx::Pending{};
  mr_ctx* cs[1] = {c};
  const double* yc[1] = {pd.ycur};
  return domain_finish(cs, 1, pd.plan, pd.t, pd.H, pd.missing_stage, pd.host_key, pd.timed, yc,
                       counters, fail_stage);
}

// mri_integrate, proj/src/mri.cpp:524-540 (state unchanged on failure)
int mr_mri_integrate(mr_ctx* c, double t0, double tf, double H, uint64_t* counters,
                     int* fail_stage)
{
  if (!c) return MR_CONTRACT;
  if (int g = pending_guard(c)) return g;
  if (fail_stage) *fail_stage = -1;
  if (!(tf > t0)) return set_err(c, MR_CONTRACT, "mri_integrate: tf must exceed t0");
  const std::vector<mr_ctx*> ms = members(c);
  for (mr_ctx* m : ms) {
    cudaSetDevice(m->device);
    if (int rc = ensure_state(m)) return set_err(c, rc, m->err);
  }
  const long n_steps = static_cast<long>(std::ceil((tf - t0) / H - 1e-12));
  const bool backup = n_steps > 1;
  if (backup)  // allocated once per grid, reused by every integrate call
    for (mr_ctx* m : ms) {
      cudaSetDevice(m->device);
      if (!m->y_backup) MR_CUDA_TRY(c, cudaMalloc(&m->y_backup, m->dof * sizeof(double)));
      MR_CUDA_TRY(c, cudaMemcpyAsync(m->y_backup, m->y_state, m->dof * sizeof(double),
                                     cudaMemcpyDeviceToDevice, m->stream));
    }
  double t = t0;
  int rc = MR_OK;
  for (long i = 0; i < n_steps; ++i) {
    const double step = (i == n_steps - 1) ? (tf - t) : H;
    rc = mr_mri_step(c, t, step, counters, fail_stage);
    if (rc) break;
    t = (i == n_steps - 1) ? tf : t0 + static_cast<double>(i + 1) * H;
  }
  if (backup)
    for (mr_ctx* m : ms) {
      cudaSetDevice(m->device);
      if (rc)
        cudaMemcpyAsync(m->y_state, m->y_backup, m->dof * sizeof(double), cudaMemcpyDeviceToDevice,
                        m->stream);
      cudaStreamSynchronize(m->stream);
    }
  return rc;
}


// ---------------------------------------------------------------------------
// ARK-IMEX: ark_imex_step (mri.cpp:437-522) with the
// ARK4(3)6L[2]SA pair (butcher.cpp:362-427) on the same device plugins --
// combined explicit part f_fast + f_explicit, implicit f_implicit solved by
// newton_pcg (the stage solver of the IMEX MRI path).
// ---------------------------------------------------------------------------
namespace {
struct Ark436 {
  double AE[6][6] = {}, AI[6][6] = {}, b[6] = {}, c[6] = {};
  Ark436()
  {
    c[1] = 0.5; c[2] = 83.0 / 250.0; c[3] = 31.0 / 50.0; c[4] = 17.0 / 20.0; c[5] = 1.0;
    AE[1][0] = 0.5;
    AE[2][0] = 13861.0 / 62500.0; AE[2][1] = 6889.0 / 62500.0;
    AE[3][0] = -116923316275.0 / 2393684061468.0;
    AE[3][1] = -2731218467317.0 / 15368042101831.0;
    AE[3][2] = 9408046702089.0 / 11113171139209.0;
    AE[4][0] = -451086348788.0 / 2902428689909.0;
    AE[4][1] = -2682348792572.0 / 7519795681897.0;
    AE[4][2] = 12662868775082.0 / 11960479115383.0;
    AE[4][3] = 3355817975965.0 / 11060851509271.0;
    AE[5][0] = 647845179188.0 / 3216320057751.0;
    AE[5][1] = 73281519250.0 / 8382639484533.0;
    AE[5][2] = 552539513391.0 / 3454668386233.0;
    AE[5][3] = 3354512671639.0 / 8306763924573.0;
    AE[5][4] = 4040.0 / 17871.0;
    b[0] = 82889.0 / 524892.0; b[2] = 15625.0 / 83664.0; b[3] = 69875.0 / 102672.0;
    b[4] = -2260.0 / 8211.0; b[5] = 0.25;
    AI[1][0] = 0.25; AI[1][1] = 0.25;
    AI[2][0] = 8611.0 / 62500.0; AI[2][1] = -1743.0 / 31250.0; AI[2][2] = 0.25;
    AI[3][0] = 5012029.0 / 34652500.0; AI[3][1] = -654441.0 / 2922500.0;
    AI[3][2] = 174375.0 / 388108.0; AI[3][3] = 0.25;
    AI[4][0] = 15267082809.0 / 155376265600.0; AI[4][1] = -71443401.0 / 120774400.0;
    AI[4][2] = 730878875.0 / 902184768.0; AI[4][3] = 2285395.0 / 8070912.0; AI[4][4] = 0.25;
    AI[5][0] = 82889.0 / 524892.0; AI[5][2] = 15625.0 / 83664.0; AI[5][3] = 69875.0 / 102672.0;
    AI[5][4] = -2260.0 / 8211.0; AI[5][5] = 0.25;
  }
};

// combined_explicit (mri.cpp:450-456) of every context's `in` into `out`
int ark_explicit(mr_ctx** cs, int n, double* const* in, double* const* out, cudaStream_t st)
{
  const bool fast = cs[0]->fast_kind != FK_NONE, slow = cs[0]->slow_kind != SK_NONE;
  for (int r = 0; r < n && fast; ++r) {
    sdev(cs[r]);
    int rc = eval_fast_dev(cs[r], in[r], cs[r]->ark_bufs[12], sst(cs[r], st));
    if (rc) return rc;
  }
  if (slow) {
    std::vector<const double*> yc(in, in + n);
    int rc = eval_slow(cs, n, yc.data(), out, st);
    if (rc) return rc;
  }
  for (int r = 0; r < n; ++r) {
    sdev(cs[r]);
    MR_CUDA_TRY(cs[r], launch_add2(cs[r]->dof, fast ? cs[r]->ark_bufs[12] : nullptr,
                                   slow ? out[r] : nullptr, out[r], sst(cs[r], st)));
    cs[r]->launches++;
  }
  return MR_OK;
}

int ark_domain_step(mr_ctx** cs, int n, double t, double H, uint64_t* counters, int* fail_stage)
{
  const NvtxRange range("ark_imex_step");
  mr_ctx* c0 = cs[0];
  if (fail_stage) *fail_stage = -1;
  if (!(H > 0.0)) return set_err(c0, MR_CONTRACT, "ark_imex_step: H must be positive");
  for (int r = 0; r < n; ++r) {
    mr_ctx* c = cs[r];
    sdev(c);
    if (!c->has_grid) return set_err(c0, MR_CONTRACT, "grid not set (mr_grid_set)");
    if (c->fast_kind < 0 || c->slow_kind < 0)
      return set_err(c0, MR_CONTRACT, "PartitionedSystem: fast/slow plugins not configured");
    if (!(c->slow_kind == SK_STENCIL && c->imex))
      return set_err(c0, MR_CONTRACT, "ark_imex_step: f_implicit required");
    int rc = ensure_state(c);
    if (rc) return rc;
    rc = ensure_cg(c);
    if (rc) return rc;
    while ((int)c->ark_bufs.size() < 13) {
      double* p = nullptr;
      MR_CUDA_TRY(c, cudaMalloc(&p, c->dof * sizeof(double)));
      c->ark_bufs.push_back(p);
    }
    MR_CUDA_TRY(c, cudaMemsetAsync(c->d_fail, 0xFF, sizeof(unsigned long long), sst(c, c0->stream)));
  }
  static const Ark436 tb;
  const int s = 6;
  cudaStream_t st = c0->stream;
  std::vector<double*> in(n), out(n);
  uint64_t cnt[8] = {}, snap[7][8] = {};
  unsigned long long host_key = MR_NO_FAIL;
  // stage 0: fE_0 = combined(y), fI_0 = f_I(y)
  for (int r = 0; r < n; ++r) {
    in[r] = cs[r]->y_state;
    out[r] = cs[r]->ark_bufs[0];
  }
  int rc = ark_explicit(cs, n, in.data(), out.data(), st);
  if (rc) return rc;
  cnt[MR_CNT_EXPLICIT_EVALS]++;
  {
    std::vector<const double*> yc(n);
    for (int r = 0; r < n; ++r) {
      yc[r] = cs[r]->y_state;
      out[r] = cs[r]->ark_bufs[6];
    }
    rc = eval_implicit(cs, n, yc.data(), out.data(), st);
    if (rc) return rc;
  }
  cnt[MR_CNT_IMPLICIT_EVALS]++;
  for (int i = 1; i < s; ++i) {
    std::memcpy(snap[i], cnt, sizeof(cnt));
    // known = y + sum_j H (AE_ij fE_j, then AI_ij fI_j)   (mri.cpp:467-471)
    for (int r = 0; r < n; ++r) {
      mr_ctx* c = cs[r];
      sdev(c);
      const double* f[MR_MAXREF];
      double cf[MR_MAXREF];
      int nref = 0;
      for (int j = 0; j < i; ++j) {
        if (tb.AE[i][j] != 0.0) { f[nref] = c->ark_bufs[j]; cf[nref++] = H * tb.AE[i][j]; }
        if (tb.AI[i][j] != 0.0) { f[nref] = c->ark_bufs[6 + j]; cf[nref++] = H * tb.AI[i][j]; }
      }
      MR_CUDA_TRY(c, launch_update(c->y_state, c->cg_known, nref, f, cf, c->dof, i, c->d_fail,
                                   sst(c, st)));
      MR_CUDA_TRY(c, cudaMemcpyAsync(c->y_work, c->cg_known, c->dof * sizeof(double),
                                     cudaMemcpyDeviceToDevice, sst(c, st)));
      c->launches++;
      out[r] = c->ark_bufs[6 + i];
    }
    rc = newton_pcg(cs, n, i, H * tb.AI[i][i], out.data(), &host_key, st);
    if (rc) return rc;
    const uint64_t nl = (uint64_t)c0->solve_nl[i];
    cnt[MR_CNT_IMPLICIT_EVALS] += (uint64_t)c0->solve_evals[i];
    cnt[MR_CNT_NONLINEAR_ITERS] += nl;
    cnt[MR_CNT_LINEAR_ITERS] += nl * (uint64_t)c0->cg_iters;
    cnt[MR_CNT_PRECOND_SOLVES] += nl * ((uint64_t)c0->cg_iters + 1);
    cnt[MR_CNT_IMPLICIT_SOLVES]++;
    if (host_key != MR_NO_FAIL) break;
    // fE_i = combined(t + c_i H, Y)
    for (int r = 0; r < n; ++r) {
      in[r] = cs[r]->y_work;
      out[r] = cs[r]->ark_bufs[i];
    }
    rc = ark_explicit(cs, n, in.data(), out.data(), st);
    if (rc) return rc;
    cnt[MR_CNT_EXPLICIT_EVALS]++;
  }
  if (host_key == MR_NO_FAIL) {
    // out = y + sum_j H b_j (fE_j, then fI_j)   (mri.cpp:510-516)
    for (int r = 0; r < n; ++r) {
      mr_ctx* c = cs[r];
      sdev(c);
      const double* f[MR_MAXREF];
      double cf[MR_MAXREF];
      int nref = 0;
      for (int j = 0; j < s; ++j)
        if (tb.b[j] != 0.0) {
          f[nref] = c->ark_bufs[j]; cf[nref++] = H * tb.b[j];
          f[nref] = c->ark_bufs[6 + j]; cf[nref++] = H * tb.b[j];
        }
      MR_CUDA_TRY(c, launch_update(c->y_state, c->y_work, nref, f, cf, c->dof, s, c->d_fail,
                                   sst(c, st)));
      c->launches++;
    }
  }
  unsigned long long key = MR_NO_FAIL;
  if (n == 1 && c0->comm)
    MR_NCCL_TRY(c0, AllReduce(c0->d_fail, c0->d_fail, 1, ncclUint64, ncclMin, c0->comm, st));
  for (int r = 0; r < n; ++r) {
    sdev(cs[r]);
    MR_CUDA_TRY(cs[r], cudaMemcpyAsync(cs[r]->h_fail, cs[r]->d_fail, sizeof(unsigned long long),
                                       cudaMemcpyDeviceToHost, sst(cs[r], st)));
  }
  for (int r = 0; r < n; ++r) {
    if (!cs[r]->in_domain && r > 0) break;
    sdev(cs[r]);
    MR_CUDA_TRY(c0, cudaStreamSynchronize(sst(cs[r], st)));
  }
  for (int r = 0; r < n; ++r) key = std::min(key, *cs[r]->h_fail);
  key = std::min(key, host_key);
  if (key != MR_NO_FAIL) {
    const int fs = (int)(key >> 40), inner = (int)(key & 0xFFull);
    const uint64_t* part = (fs < s && inner == 0) ? snap[fs] : cnt;
    if (counters)
      for (int q = 0; q < 8; ++q) counters[q] += part[q];
    if (fail_stage) *fail_stage = fs;
    if (fs == s) return set_err(c0, MR_INTEGRATION, "ark_imex_step: non-finite result");
    if (inner == 0)
      return set_err(c0, MR_INTEGRATION,
                     "ark_imex_step: non-finite stage data at stage " + std::to_string(fs));
    return set_err(c0, MR_INTEGRATION,
                   "ark_imex_step: nonlinear solve failed at stage " + std::to_string(fs));
  }
  if (counters)
    for (int q = 0; q < 8; ++q) counters[q] += cnt[q];
  for (int r = 0; r < n; ++r) std::swap(cs[r]->y_state, cs[r]->y_work);
  return MR_OK;
}
}  // namespace

int mr_ark_imex_step(mr_ctx* c, double t, double H, uint64_t* counters, int* fail_stage)
{
  if (!c) return MR_CONTRACT;
  if (int g = pending_guard(c)) return g;
  if (!c->slabs.empty())
    return domain_rc(c, ark_domain_step(c->slabs.data(), (int)c->slabs.size(), t, H, counters,
                                        fail_stage));
  cudaSetDevice(c->device);
  return ark_domain_step(&c, 1, t, H, counters, fail_stage);
}

int mr_ark_imex_integrate(mr_ctx* c, double t0, double tf, double H, uint64_t* counters,
                          int* fail_stage)
{
  if (!c) return MR_CONTRACT;
  if (int g = pending_guard(c)) return g;
  if (fail_stage) *fail_stage = -1;
  if (!(tf > t0)) return set_err(c, MR_CONTRACT, "ark_imex_integrate: tf must exceed t0");
  const std::vector<mr_ctx*> ms = members(c);
  for (mr_ctx* m : ms) {
    cudaSetDevice(m->device);
    if (int rc = ensure_state(m)) return set_err(c, rc, m->err);
  }
  const long n_steps = static_cast<long>(std::ceil((tf - t0) / H - 1e-12));
  const bool backup = n_steps > 1;
  if (backup)
    for (mr_ctx* m : ms) {
      cudaSetDevice(m->device);
      if (!m->y_backup) MR_CUDA_TRY(c, cudaMalloc(&m->y_backup, m->dof * sizeof(double)));
      MR_CUDA_TRY(c, cudaMemcpyAsync(m->y_backup, m->y_state, m->dof * sizeof(double),
                                     cudaMemcpyDeviceToDevice, m->stream));
    }
  double t = t0;
  int rc = MR_OK;
  for (long i = 0; i < n_steps; ++i) {
    const double step = (i == n_steps - 1) ? (tf - t) : H;
    rc = mr_ark_imex_step(c, t, step, counters, fail_stage);
    if (rc) break;
    t = (i == n_steps - 1) ? tf : t0 + static_cast<double>(i + 1) * H;
  }
  if (backup)
    for (mr_ctx* m : ms) {
      cudaSetDevice(m->device);
      if (rc)
        cudaMemcpyAsync(m->y_state, m->y_backup, m->dof * sizeof(double), cudaMemcpyDeviceToDevice,
                        m->stream);
      cudaStreamSynchronize(m->stream);
    }
  return rc;
}

int mr_mri_step_host(mr_ctx* c, double t, double H, const double* y_in, double* y_out,
                     uint64_t* counters, int* fail_stage)
{
  if (!c || !y_in || !y_out) return MR_CONTRACT;
  if (int g = pending_guard(c)) return g;
  if (!c->slabs.empty()) {
    int rc = mr_state_upload(c, y_in);
    if (rc) return rc;
    rc = mr_mri_step(c, t, H, counters, fail_stage);
    if (rc) return rc;
    return mr_state_download(c, y_out);
  }
  cudaSetDevice(c->device);
  int rc = ensure_state(c);
  if (rc) return rc;
  // the step itself moves the data (domain_step: head_upload / tail_download)
  const uint64_t bytes = (uint64_t)c->dof * sizeof(double);
  c->host_in = y_in;
  c->host_out = y_out;
  c->out_streamed = false;
  c->host_h2d = bytes;  // y_in
  c->host_d2h = 0;
  rc = mr_mri_step(c, t, H, counters, fail_stage);
  c->host_in = nullptr;
  c->host_out = nullptr;
  if (c->out_streamed) {  // y_out was saved (H2D) and written by the step's last ops
    c->out_streamed = false;
    c->host_h2d += bytes;
    c->host_d2h = bytes;
    MR_CUDA_TRY(c, cudaStreamSynchronize(c->copy_stream));
    if (rc) {  // no partial result: the caller's buffer as it was
      cudaMemcpy(y_out, c->y_backup, c->dof * sizeof(double), cudaMemcpyDeviceToHost);
      c->host_d2h += bytes;
      return rc;
    }
    return MR_OK;
  }
  if (rc) return rc;
  c->host_d2h = bytes;
  MR_CUDA_TRY(c, cudaMemcpyAsync(y_out, c->y_state, c->dof * sizeof(double),
                                 cudaMemcpyDeviceToHost, c->stream));
  MR_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return MR_OK;
}

int mr_last_host_step_bytes(const mr_ctx* c, uint64_t* h2d, uint64_t* d2h)
{
  if (!c || !h2d || !d2h) return MR_CONTRACT;
  uint64_t a = c->host_h2d, b = c->host_d2h;
  for (const mr_ctx* sl : c->slabs) {
    a += sl->host_h2d;
    b += sl->host_d2h;
  }
  *h2d = a;
  *d2h = b;
  return MR_OK;
}

int mr_last_failure(const mr_ctx* c, int* mri_stage, int* substep, int* inner_stage)
{
  if (!c) return MR_CONTRACT;
  if (!c->slabs.empty()) c = c->slabs[0];
  if (mri_stage) *mri_stage = c->fail_mri;
  if (substep) *substep = c->fail_sub;
  if (inner_stage) *inner_stage = c->fail_inner;
  return MR_OK;
}

static int ensure_scratch(mr_ctx* c)
{
  if (!c->scr_in) MR_CUDA_TRY(c, cudaMalloc(&c->scr_in, c->dof * sizeof(double)));
  if (!c->scr_out) MR_CUDA_TRY(c, cudaMalloc(&c->scr_out, c->dof * sizeof(double)));
  return MR_OK;
}

int mr_fast_rhs(mr_ctx* c, double t, const double* y, double* out)
{
  (void)t;
  if (!c || !y || !out) return MR_CONTRACT;
  if (int g = pending_guard(c)) return g;
  if (!c->slabs.empty()) {
    if (!c->has_grid || c->slabs[0]->fast_kind < 0)
      return set_err(c, MR_CONTRACT, "fast plugin not set");
    return domain_rhs(c, 0, y, out);
  }
  if (!c->has_grid || c->fast_kind < 0) return set_err(c, MR_CONTRACT, "fast plugin not set");
  if (c->fast_kind == FK_CHEM && c->ncomp != c->S + 1)
    return set_err(c, MR_CONTRACT, "chemistry plugin needs n_comp == S + 1");
  cudaSetDevice(c->device);
  int rc = ensure_scratch(c);
  if (rc) return rc;
  MR_CUDA_TRY(c, cudaMemcpyAsync(c->scr_in, y, c->dof * sizeof(double), cudaMemcpyHostToDevice,
                                 c->stream));
  if (c->fast_kind == FK_CHEM) {
    ChemCfg ccfg;
    TableDev t4{};
    t4.s = 4;
    if (chem_pick(&ccfg, c->ncomp, c->S, c->R, t4, 1))
      return set_err(c, MR_CONTRACT, "unsupported mechanism size");
    MR_CUDA_TRY(c, launch_chem_rhs(ccfg, c->scr_in, c->scr_out, c->ncell, c->ncomp, *c->chemP,
                                   c->stream));
  } else {
    ChainCfg cfg;
    if (chain_pick(&cfg, c->fast_kind, c->ncomp, 4, 1))
      return set_err(c, MR_CONTRACT, "unsupported component count");
    MR_CUDA_TRY(c, launch_fast_rhs(cfg, c->scr_in, c->scr_out, c->ncell, c->ncomp, c->fastA,
                                   c->stream));
  }
  c->launches++;
  MR_CUDA_TRY(c, cudaMemcpyAsync(out, c->scr_out, c->dof * sizeof(double), cudaMemcpyDeviceToHost,
                                 c->stream));
  MR_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return MR_OK;
}



// erk_integrate (erk.cpp:40-57) of an explicit table on sum_rhs
// (partitioned_system.hpp:41-48) over the device-resident state: erk_step's
// stage loop, finite checks (:24-36) and per-stage evaluation count (:28).
// On failure the state is restored to its value at entry (the reference's
// input is const) and the count stops where erk_step threw.
static int erk_integrate_dev(mr_ctx** cs, int n, int s, const double* A, const double* b,
                             double t0, double tf, double h, uint64_t* evals, int* fail_stage)
{
  if (fail_stage) *fail_stage = -1;
  mr_ctx* c0 = cs[0];
  if (!c0->has_grid) return set_err(c0, MR_CONTRACT, "grid not set (mr_grid_set)");
  if (c0->fast_kind < 0 || c0->slow_kind < 0)
    return set_err(c0, MR_CONTRACT, "PartitionedSystem: fast/slow plugins not configured");
  if (c0->fast_kind == FK_NONE && c0->slow_kind == SK_NONE)
    return set_err(c0, MR_CONTRACT, "PartitionedSystem: at least one partition required");
  if (!(tf > t0)) return set_err(c0, MR_CONTRACT, "erk_integrate: tf must exceed t0");
  if (!(h > 0.0)) return set_err(c0, MR_CONTRACT, "erk_integrate: h must be positive");
  if (s < 1 || s > MR_MAXREF) return set_err(c0, MR_CONTRACT, "erk_integrate: 1 <= stages <= 12");
  for (int i = 0; i < s; ++i)
    for (int j = i; j < s; ++j)
      if (A[i * s + j] != 0.0) return set_err(c0, MR_CONTRACT, "erk_step: table must be explicit");
  for (int r = 0; r < n; ++r) {
    mr_ctx* c = cs[r];
    if (c->slow_kind == SK_STENCIL && c->n0l < c->M)
      return set_err(c0, MR_CONTRACT, "slab thinner than the stencil ghost width");
    cudaSetDevice(c->device);
    int rc = ensure_state(c);
    if (rc) return rc;
    // buffers: k[0..s-1], stage, f_fast, f_implicit, entry backup
    while ((int)c->rs_bufs.size() < s + 4) {
      double* p = nullptr;
      MR_CUDA_TRY(c, cudaMalloc(&p, c->dof * sizeof(double)));
      c->rs_bufs.push_back(p);
    }
  }
  const bool fast = c0->fast_kind != FK_NONE, slow = c0->slow_kind != SK_NONE;
  const bool imp = c0->slow_kind == SK_STENCIL && c0->imex;
  cudaStream_t st = c0->stream;
  auto buf = [&](int r, int q) { return cs[r]->rs_bufs[q]; };  // k_q (q < s), stage, f_F, f_I, backup
  for (int r = 0; r < n; ++r) {
    sdev(cs[r]);
    MR_CUDA_TRY(cs[r], cudaMemcpyAsync(buf(r, s + 3), cs[r]->y_state, cs[r]->dof * sizeof(double),
                                       cudaMemcpyDeviceToDevice, sst(cs[r], st)));
  }
  std::vector<const double*> yc(n);
  std::vector<double*> oc(n);
  const long n_steps = (long)std::ceil((tf - t0) / h - 1e-12);
  double t = t0;
  for (long ns = 0; ns < n_steps; ++ns) {
    const double step = (ns == n_steps - 1) ? (tf - t) : h;
    for (int r = 0; r < n; ++r) {
      sdev(cs[r]);
      MR_CUDA_TRY(cs[r], cudaMemsetAsync(cs[r]->d_fail, 0xFF, sizeof(unsigned long long),
                                         sst(cs[r], st)));
    }
    for (int i = 0; i < s; ++i) {
      for (int r = 0; r < n; ++r) {
        mr_ctx* c = cs[r];
        sdev(c);
        const double* f[MR_MAXREF];
        double cf[MR_MAXREF];
        int nref = 0;
        for (int j = 0; j < i; ++j)
          if (A[i * s + j] != 0.0) {
            f[nref] = buf(r, j);
            cf[nref++] = step * A[i * s + j];
          }
        MR_CUDA_TRY(c, launch_update(c->y_state, buf(r, s), nref, f, cf, c->dof, i, c->d_fail,
                                     sst(c, st)));
        c->launches++;
        if (fast) {
          int rc = eval_fast_dev(c, buf(r, s), buf(r, s + 1), sst(c, st));
          if (rc) return rc;
        }
      }
      for (int r = 0; r < n; ++r) yc[r] = buf(r, s);
      if (imp) {
        for (int r = 0; r < n; ++r) oc[r] = buf(r, s + 2);
        int rc = eval_implicit(cs, n, yc.data(), oc.data(), st);
        if (rc) return rc;
      }
      if (slow) {
        for (int r = 0; r < n; ++r) oc[r] = buf(r, i);
        int rc = eval_slow(cs, n, yc.data(), oc.data(), st);
        if (rc) return rc;
      }
      for (int r = 0; r < n; ++r) {
        mr_ctx* c = cs[r];
        sdev(c);
        MR_CUDA_TRY(c, launch_sum_rhs(c->dof, fast ? buf(r, s + 1) : nullptr,
                                      imp ? buf(r, s + 2) : nullptr, slow ? buf(r, i) : nullptr,
                                      buf(r, i), sst(c, st)));
        c->launches++;
      }
    }
    for (int r = 0; r < n; ++r) {
      mr_ctx* c = cs[r];
      sdev(c);
      const double* f[MR_MAXREF];
      double cf[MR_MAXREF];
      int nref = 0;
      for (int i = 0; i < s; ++i)
        if (b[i] != 0.0) {
          f[nref] = buf(r, i);
          cf[nref++] = step * b[i];
        }
      MR_CUDA_TRY(c, launch_update(c->y_state, c->y_work, nref, f, cf, c->dof, s, c->d_fail,
                                   sst(c, st)));
      c->launches++;
      if (c->comm)
        MR_NCCL_TRY(c, AllReduce(c->d_fail, c->d_fail, 1, ncclUint64, ncclMin, c->comm, sst(c, st)));
      MR_CUDA_TRY(c, cudaMemcpyAsync(c->h_fail, c->d_fail, sizeof(unsigned long long),
                                     cudaMemcpyDeviceToHost, sst(c, st)));
    }
    unsigned long long key = MR_NO_FAIL;
    for (int r = 0; r < n; ++r) {
      sdev(cs[r]);
      MR_CUDA_TRY(cs[r], cudaStreamSynchronize(sst(cs[r], st)));
      key = std::min(key, *cs[r]->h_fail);
    }
    if (key != MR_NO_FAIL) {
      const int fs = (int)(key >> 40);
      if (fail_stage) *fail_stage = fs;
      if (evals) *evals += (uint64_t)(fs < s ? fs : s);  // stages evaluated before the throw
      for (int r = 0; r < n; ++r) {
        sdev(cs[r]);
        MR_CUDA_TRY(cs[r], cudaMemcpyAsync(cs[r]->y_state, buf(r, s + 3),
                                           cs[r]->dof * sizeof(double), cudaMemcpyDeviceToDevice,
                                           sst(cs[r], st)));
        MR_CUDA_TRY(cs[r], cudaStreamSynchronize(sst(cs[r], st)));
      }
      return set_err(c0, MR_INTEGRATION,
                     fs == s ? "erk_step: non-finite result" : "erk_step: non-finite stage value");
    }
    if (evals) *evals += (uint64_t)s;
    for (int r = 0; r < n; ++r) std::swap(cs[r]->y_state, cs[r]->y_work);
    t = (ns == n_steps - 1) ? tf : t0 + (double)(ns + 1) * h;
  }
  return MR_OK;
}

int mr_erk_integrate(mr_ctx* c, int s, const double* A, const double* b, const double* cvec,
                     double t0, double tf, double h, uint64_t* n_explicit_evals, int* fail_stage)
{
  (void)cvec;  // sum_rhs of the plugins is autonomous: t + c_i h is not consumed
  if (!c || !A || !b) return MR_CONTRACT;
  if (int g = pending_guard(c)) return g;
  if (!c->slabs.empty())
    return domain_rc(c, erk_integrate_dev(c->slabs.data(), (int)c->slabs.size(), s, A, b, t0, tf,
                                          h, n_explicit_evals, fail_stage));
  return erk_integrate_dev(&c, 1, s, A, b, t0, tf, h, n_explicit_evals, fail_stage);
}

// ---- spectral deferred corrections (proj/src/sdc.cpp) ----
// One engine for both of the reference's SDC drivers:
//   * multirate (mrsdc_step, sdc.cpp:233-265, sweep :155-199): f_fast cached at
//     the n_fine fine nodes, slow_rhs = f_implicit + f_explicit at the X coarse
//     nodes, each sweep a forward-Euler correction node by node;
//   * single rate (sdc_step, :201-231): the same sweep with X = 0, one rule
//     (fine_row = the integration matrix S, offset 0) and f_total = sum_rhs in
//     the fine-node cache.
// Per node the update is one fused multi-operand axpy in the reference's
// order (quadrature of the previous iterate, fine then coarse, then the four
// forward-Euler terms), its finite check keyed (sweep, node) so the first
// failure in execution order is the one reported.  The plugins are autonomous
// (no t dependence), so the initial caches -- the same state at every node --
// are evaluated once and copied; they are counted like the reference's
// separate evaluations.  Cache slots are pointer-swapped between sweeps (the
// reference copies the k-th iterate's caches).
namespace {
struct SdcRun {
  bool single;  // sdc_step on sum_rhs
  int X, Y, nf, sweeps;
  const double *coarse_nodes, *fine_nodes, *fine_row, *coarse_row;
  const int *coarse_of_fine, *coarse_index_of_fine, *application_offset;
};
}  // namespace

static int sdc_integrate_dev(mr_ctx** cs, int n, const SdcRun& R, double t0, double tf, double H,
                             uint64_t* cnt_fast, uint64_t* cnt_slow, int* fail_stage)
{
  if (fail_stage) *fail_stage = -1;
  mr_ctx* c0 = cs[0];
  const char* who = R.single ? "sdc_integrate" : "mrsdc_integrate";
  if (!c0->has_grid) return set_err(c0, MR_CONTRACT, "grid not set (mr_grid_set)");
  if (c0->fast_kind < 0 || c0->slow_kind < 0)
    return set_err(c0, MR_CONTRACT, "PartitionedSystem: fast/slow plugins not configured");
  if (!(tf > t0)) return set_err(c0, MR_CONTRACT, std::string(who) + ": tf must exceed t0");
  if (!(H > 0.0)) return set_err(c0, MR_CONTRACT, std::string(who) + ": H must be positive");
  const int nf = R.nf, X = R.single ? 0 : R.X;
  const int nbuf = 2 * nf + 2 * X + 5;  // f caches x2, slow caches x2, node states x2, scratch x2, backup
  for (int r = 0; r < n; ++r) {
    mr_ctx* c = cs[r];
    if (c->slow_kind == SK_STENCIL && c->n0l < c->M)
      return set_err(c0, MR_CONTRACT, "slab thinner than the stencil ghost width");
    cudaSetDevice(c->device);
    int rc = ensure_state(c);
    if (rc) return rc;
    while ((int)c->sdc_bufs.size() < nbuf) {
      double* p = nullptr;
      if (cudaMalloc(&p, c->dof * sizeof(double)) != cudaSuccess) {
        cudaGetLastError();
        return set_err(c0, MR_CUDA, std::string(who) + ": device memory for the " +
                                        std::to_string(nbuf) + " node caches exhausted");
      }
      c->sdc_bufs.push_back(p);
    }
  }
  const bool fast = c0->fast_kind != FK_NONE, slow = c0->slow_kind != SK_NONE;
  const bool imp = c0->slow_kind == SK_STENCIL && c0->imex;
  cudaStream_t st = c0->stream;
  // per slab: cache pointers (cur / spare) into sdc_bufs
  std::vector<std::vector<double*>> fcur(n), fspare(n), scur(n), sspare(n);
  for (int r = 0; r < n; ++r) {
    auto& B = cs[r]->sdc_bufs;
    for (int q = 0; q < nf; ++q) {
      fcur[r].push_back(B[q]);
      fspare[r].push_back(B[nf + q]);
    }
    for (int p = 0; p < X; ++p) {
      scur[r].push_back(B[2 * nf + p]);
      sspare[r].push_back(B[2 * nf + X + p]);
    }
  }
  auto node = [&](int r, int q) -> double* {  // state of fine node q >= 1
    return cs[r]->sdc_bufs[2 * nf + 2 * X + (q & 1)];
  };
  auto scrF = [&](int r) { return cs[r]->sdc_bufs[2 * nf + 2 * X + 2]; };
  auto scrI = [&](int r) { return cs[r]->sdc_bufs[2 * nf + 2 * X + 3]; };
  auto backup = [&](int r) { return cs[r]->sdc_bufs[2 * nf + 2 * X + 4]; };
  std::vector<const double*> yc(n);
  std::vector<double*> oc(n);
  // f_total (sum_rhs order: fast, implicit, explicit) or the fast part alone
  auto eval_fine = [&](const std::vector<const double*>& in, const std::vector<double*>& out) -> int {
    if (!R.single) {
      for (int r = 0; r < n; ++r) {
        mr_ctx* c = cs[r];
        sdev(c);
        if (fast) {
          int rc = eval_fast_dev(c, in[r], out[r], sst(c, st));
          if (rc) return rc;
        } else {
          MR_CUDA_TRY(c, cudaMemsetAsync(out[r], 0, c->dof * sizeof(double), sst(c, st)));
        }
      }
      return MR_OK;
    }
    for (int r = 0; r < n; ++r)
      if (fast) {
        sdev(cs[r]);
        int rc = eval_fast_dev(cs[r], in[r], scrF(r), sst(cs[r], st));
        if (rc) return rc;
      }
    std::vector<double*> oi(n);
    for (int r = 0; r < n; ++r) oi[r] = scrI(r);
    if (imp) {
      int rc = eval_implicit(cs, n, in.data(), oi.data(), st);
      if (rc) return rc;
    }
    if (slow) {
      int rc = eval_slow(cs, n, in.data(), out.data(), st);
      if (rc) return rc;
    }
    for (int r = 0; r < n; ++r) {
      mr_ctx* c = cs[r];
      sdev(c);
      MR_CUDA_TRY(c, launch_sum_rhs(c->dof, fast ? scrF(r) : nullptr, imp ? scrI(r) : nullptr,
                                    slow ? out[r] : nullptr, out[r], sst(c, st)));
      c->launches++;
    }
    return MR_OK;
  };
  // slow_rhs (partitioned_system.hpp:54-60): implicit then explicit
  auto eval_coarse = [&](const std::vector<const double*>& in, const std::vector<double*>& out) -> int {
    std::vector<double*> oi(n);
    for (int r = 0; r < n; ++r) oi[r] = scrI(r);
    if (imp) {
      int rc = eval_implicit(cs, n, in.data(), oi.data(), st);
      if (rc) return rc;
    }
    if (slow) {
      int rc = eval_slow(cs, n, in.data(), out.data(), st);
      if (rc) return rc;
    }
    for (int r = 0; r < n; ++r) {
      mr_ctx* c = cs[r];
      sdev(c);
      MR_CUDA_TRY(c, launch_sum_rhs(c->dof, nullptr, imp ? scrI(r) : nullptr,
                                    slow ? out[r] : nullptr, out[r], sst(c, st)));
      c->launches++;
    }
    return MR_OK;
  };
  // evaluations of one sweep (and of the coarse nodes it reaches before node k)
  int coarse_hits = 0;
  for (int q = 1; q < nf; ++q) coarse_hits += !R.single && R.coarse_index_of_fine[q] >= 0;
  for (int r = 0; r < n; ++r) {
    sdev(cs[r]);
    MR_CUDA_TRY(cs[r], cudaMemcpyAsync(backup(r), cs[r]->y_state, cs[r]->dof * sizeof(double),
                                       cudaMemcpyDeviceToDevice, sst(cs[r], st)));
  }
  const long n_steps = (long)std::ceil((tf - t0) / H - 1e-12);
  double t = t0;
  for (long ns = 0; ns < n_steps; ++ns) {
    const double step = (ns == n_steps - 1) ? (tf - t) : H;
    for (int r = 0; r < n; ++r) {
      sdev(cs[r]);
      MR_CUDA_TRY(cs[r], cudaMemsetAsync(cs[r]->d_fail, 0xFF, sizeof(unsigned long long),
                                         sst(cs[r], st)));
    }
    // initial caches: the step's state at every node
    for (int r = 0; r < n; ++r) {
      yc[r] = cs[r]->y_state;
      oc[r] = fcur[r][0];
    }
    int rc = eval_fine(yc, oc);
    if (rc) return rc;
    if (X > 0) {
      for (int r = 0; r < n; ++r) oc[r] = scur[r][0];
      rc = eval_coarse(yc, oc);
      if (rc) return rc;
    }
    for (int r = 0; r < n; ++r) {
      mr_ctx* c = cs[r];
      sdev(c);
      const size_t bytes = c->dof * sizeof(double);
      for (int q = 1; q < nf; ++q)
        MR_CUDA_TRY(c, cudaMemcpyAsync(fcur[r][q], fcur[r][0], bytes, cudaMemcpyDeviceToDevice, sst(c, st)));
      for (int p = 1; p < X; ++p)
        MR_CUDA_TRY(c, cudaMemcpyAsync(scur[r][p], scur[r][0], bytes, cudaMemcpyDeviceToDevice, sst(c, st)));
    }
    for (int sw = 0; sw < R.sweeps; ++sw) {
      // the k-th iterate's caches (read) and fresh slots for the (k+1)-th
      std::vector<std::vector<double*>> fold = fcur, sold = scur;
      for (int q = 0; q < nf - 1; ++q) {
        const double hq = (R.fine_nodes[q + 1] - R.fine_nodes[q]) * step;
        const int p = R.single ? 0 : R.coarse_of_fine[q];
        const int key_stage = sw * 4096 + q + 1;
        for (int r = 0; r < n; ++r) {
          mr_ctx* c = cs[r];
          sdev(c);
          const double* f[2 * MR_MAXREF];
          double cf[2 * MR_MAXREF];
          int nt = 0;
          const int Yn = R.single ? nf : R.Y;
          const int off = R.single ? 0 : R.application_offset[q];
          for (int j = 0; j < Yn; ++j) {
            const double w = R.fine_row[(size_t)q * Yn + j];
            if (w != 0.0) { f[nt] = fold[r][off + j]; cf[nt++] = step * w; }
          }
          for (int j = 0; j < X; ++j) {
            const double w = R.coarse_row[(size_t)q * X + j];
            if (w != 0.0) { f[nt] = sold[r][j]; cf[nt++] = step * w; }
          }
          f[nt] = fcur[r][q]; cf[nt++] = hq;
          f[nt] = fold[r][q]; cf[nt++] = -hq;
          if (X > 0) {
            f[nt] = scur[r][p]; cf[nt++] = hq;
            f[nt] = sold[r][p]; cf[nt++] = -hq;
          }
          const double* src = q == 0 ? c->y_state : node(r, q);
          double* dst = node(r, q + 1);
          // the terms in order, in launches of at most MR_MAXREF (sequential adds)
          for (int a = 0; a < nt; a += MR_MAXREF) {
            const int na = std::min(MR_MAXREF, nt - a);
            MR_CUDA_TRY(c, launch_update(a == 0 ? src : dst, dst, na, f + a, cf + a, c->dof,
                                         key_stage, c->d_fail, sst(c, st)));
            c->launches++;
          }
          yc[r] = dst;
          oc[r] = fspare[r][q + 1];
        }
        rc = eval_fine(yc, oc);
        if (rc) return rc;
        for (int r = 0; r < n; ++r) std::swap(fcur[r][q + 1], fspare[r][q + 1]);
        const int cp = R.single ? -1 : R.coarse_index_of_fine[q + 1];
        if (cp >= 0) {
          for (int r = 0; r < n; ++r) oc[r] = sspare[r][cp];
          rc = eval_coarse(yc, oc);
          if (rc) return rc;
          for (int r = 0; r < n; ++r) std::swap(scur[r][cp], sspare[r][cp]);
        }
      }
    }
    // failure key of this step (min over slabs / ranks)
    for (int r = 0; r < n; ++r) {
      mr_ctx* c = cs[r];
      sdev(c);
      if (c->comm)
        MR_NCCL_TRY(c, AllReduce(c->d_fail, c->d_fail, 1, ncclUint64, ncclMin, c->comm, sst(c, st)));
      MR_CUDA_TRY(c, cudaMemcpyAsync(c->h_fail, c->d_fail, sizeof(unsigned long long),
                                     cudaMemcpyDeviceToHost, sst(c, st)));
    }
    unsigned long long key = MR_NO_FAIL;
    for (int r = 0; r < n; ++r) {
      sdev(cs[r]);
      MR_CUDA_TRY(cs[r], cudaStreamSynchronize(sst(cs[r], st)));
      key = std::min(key, *cs[r]->h_fail);
    }
    const uint64_t per_fast = (uint64_t)(nf - 1), per_slow = (uint64_t)coarse_hits;
    if (key != MR_NO_FAIL) {
      const int m = (int)(key >> 40), sw = m / 4096, k = m % 4096;  // node k failed in sweep sw
      int hits = 0;
      for (int q = 1; q < k; ++q) hits += !R.single && R.coarse_index_of_fine[q] >= 0;
      if (cnt_fast && (fast || R.single)) *cnt_fast += (uint64_t)nf + (uint64_t)sw * per_fast + (uint64_t)(k - 1);
      if (cnt_slow && !R.single) *cnt_slow += (uint64_t)X + (uint64_t)sw * per_slow + (uint64_t)hits;
      if (fail_stage) *fail_stage = k;
      for (int r = 0; r < n; ++r) {
        sdev(cs[r]);
        MR_CUDA_TRY(cs[r], cudaMemcpyAsync(cs[r]->y_state, backup(r), cs[r]->dof * sizeof(double),
                                           cudaMemcpyDeviceToDevice, sst(cs[r], st)));
        MR_CUDA_TRY(cs[r], cudaStreamSynchronize(sst(cs[r], st)));
      }
      return set_err(c0, MR_INTEGRATION,
                     std::string(R.single ? "sdc_step" : "mrsdc_sweep") +
                         ": non-finite update at node " + std::to_string(k));
    }
    if (cnt_fast && (fast || R.single)) *cnt_fast += (uint64_t)nf + (uint64_t)R.sweeps * per_fast;
    if (cnt_slow && !R.single) *cnt_slow += (uint64_t)X + (uint64_t)R.sweeps * per_slow;
    // the last fine node is the step's result
    for (int r = 0; r < n; ++r) {
      mr_ctx* c = cs[r];
      sdev(c);
      if (R.sweeps > 0) {
        MR_CUDA_TRY(c, cudaMemcpyAsync(c->y_work, node(r, nf - 1), c->dof * sizeof(double),
                                       cudaMemcpyDeviceToDevice, sst(c, st)));
        std::swap(c->y_state, c->y_work);
      }
    }
    t = (ns == n_steps - 1) ? tf : t0 + (double)(ns + 1) * H;
  }
  return MR_OK;
}

// ---- SDC node sets (restated from proj/src/sdc.cpp:14-150 with the same
// arithmetic order, so the tables are bitwise the reference's) ----
namespace {
// integral over [a, b] of the Lagrange basis polynomial j of `x` (sdc.cpp:14-41):
// the monomial coefficients of prod_{m != j} (t - x_m), integrated term by
// term, divided by prod_{m != j} (x_j - x_m)
double lagrange_basis_integral(const std::vector<double>& x, int j, double a, double b)
{
  std::vector<double> c{1.0};
  double den = 1.0;
  for (int m = 0; m < (int)x.size(); ++m) {
    if (m == j) continue;
    std::vector<double> nc(c.size() + 1, 0.0);
    for (size_t k = 0; k < c.size(); ++k) {
      nc[k + 1] += c[k];
      nc[k] -= x[m] * c[k];
    }
    c.swap(nc);
    den *= x[j] - x[m];
  }
  double sum = 0.0, bk = b, ak = a;
  for (size_t k = 0; k < c.size(); ++k) {
    sum += c[k] * (bk - ak) / (double)(k + 1);
    bk *= b;
    ak *= a;
  }
  return sum / den;
}

// Gauss-Lobatto nodes on [0, 1] (n = 3 or 5) and S[q][j] = integral of basis
// j over [x_q, x_{q+1}] (sdc.cpp:60-80)
bool lobatto_rule(int n, std::vector<double>& x, std::vector<double>& S)
{
  if (n == 3) {
    x = {0.0, 0.5, 1.0};
  } else if (n == 5) {
    const double r = std::sqrt(3.0 / 7.0);
    x = {0.0, 0.5 * (1.0 - r), 0.5, 0.5 * (1.0 + r), 1.0};
  } else {
    return false;
  }
  S.assign((size_t)(n - 1) * n, 0.0);
  for (int q = 0; q + 1 < n; ++q)
    for (int j = 0; j < n; ++j) S[(size_t)q * n + j] = lagrange_basis_integral(x, j, x[q], x[q + 1]);
  return true;
}

constexpr double kSdcNodeTol = 1.0e-12;  // sdc.cpp:10

// build_scheme(X, Y, Z, n_sweeps) (sdc.cpp:82-153): X coarse Lobatto nodes,
// each coarse interval split into Z applications of the Y-node rule, the
// shared junction nodes merged
int mrsdc_tables(int X, int Y, int Z, mr_ctx::SdcScheme& M)
{
  if ((X != 3 && X != 5) || (Y != 3 && Y != 5) || Z < 1) return 1;
  std::vector<double> xc, Sc, xf, Sf;
  lobatto_rule(X, xc, Sc);
  lobatto_rule(Y, xf, Sf);
  std::vector<double> start, width;
  for (int p = 0; p + 1 < X; ++p) {
    const double w = (xc[p + 1] - xc[p]) / Z;
    for (int z = 0; z < Z; ++z) {
      start.push_back(xc[p] + z * w);
      width.push_back(w);
    }
  }
  M.fine_nodes.assign(1, 0.0);
  std::vector<int> first;
  for (size_t a = 0; a < start.size(); ++a) {
    first.push_back((int)M.fine_nodes.size() - 1);
    for (int j = 1; j < Y; ++j) M.fine_nodes.push_back(start[a] + xf[j] * width[a]);
  }
  const int nf = (int)M.fine_nodes.size();
  if (nf != X + (X - 1) * (Z - 1) + (X - 1) * (Y - 2) * Z) return 1;
  M.X = X;
  M.Y = Y;
  M.n_fine = nf;
  M.coarse_nodes = xc;
  M.fine_row.assign((size_t)(nf - 1) * Y, 0.0);
  M.application_offset.assign(nf - 1, 0);
  M.coarse_row.assign((size_t)(nf - 1) * X, 0.0);
  int app = 0;
  for (int q = 0; q + 1 < nf; ++q) {
    while (app + 1 < (int)start.size() && M.fine_nodes[q] >= start[app + 1] - kSdcNodeTol) ++app;
    const int local = q - first[app];
    for (int j = 0; j < Y; ++j) M.fine_row[(size_t)q * Y + j] = width[app] * Sf[(size_t)local * Y + j];
    M.application_offset[q] = first[app];
    for (int j = 0; j < X; ++j)
      M.coarse_row[(size_t)q * X + j] =
          lagrange_basis_integral(xc, j, M.fine_nodes[q], M.fine_nodes[q + 1]);
  }
  M.coarse_of_fine.assign(nf, 0);
  M.coarse_index_of_fine.assign(nf, -1);
  for (int q = 0; q < nf; ++q) {
    int p = 0;
    for (int j = 0; j < X; ++j)
      if (xc[j] <= M.fine_nodes[q] + kSdcNodeTol) p = j;
    M.coarse_of_fine[q] = p;
    if (std::fabs(xc[p] - M.fine_nodes[q]) < kSdcNodeTol) M.coarse_index_of_fine[q] = p;
  }
  return 0;
}
}  // namespace

int mr_lobatto_rule(int n, double* nodes, double* S)
{
  std::vector<double> x, s;
  if (!nodes || !S || !lobatto_rule(n, x, s)) return MR_CONTRACT;
  std::memcpy(nodes, x.data(), x.size() * sizeof(double));
  std::memcpy(S, s.data(), s.size() * sizeof(double));
  return MR_OK;
}

int mr_mrsdc_scheme(int X, int Y, int Z, int* n_fine, double* coarse_nodes, double* fine_nodes,
                    int* coarse_of_fine, int* coarse_index_of_fine, double* fine_row,
                    int* application_offset, double* coarse_row)
{
  mr_ctx::SdcScheme M;
  if (!n_fine || mrsdc_tables(X, Y, Z, M)) return MR_CONTRACT;
  const int nf = M.n_fine;
  const bool want = coarse_nodes && fine_nodes && coarse_of_fine && coarse_index_of_fine &&
                    fine_row && application_offset && coarse_row;
  if (want && *n_fine < nf) return MR_CONTRACT;
  *n_fine = nf;
  if (!want) return MR_OK;  // size query
  std::memcpy(coarse_nodes, M.coarse_nodes.data(), X * sizeof(double));
  std::memcpy(fine_nodes, M.fine_nodes.data(), nf * sizeof(double));
  std::memcpy(coarse_of_fine, M.coarse_of_fine.data(), nf * sizeof(int));
  std::memcpy(coarse_index_of_fine, M.coarse_index_of_fine.data(), nf * sizeof(int));
  std::memcpy(fine_row, M.fine_row.data(), M.fine_row.size() * sizeof(double));
  std::memcpy(application_offset, M.application_offset.data(), (nf - 1) * sizeof(int));
  std::memcpy(coarse_row, M.coarse_row.data(), M.coarse_row.size() * sizeof(double));
  return MR_OK;
}

int mr_mrsdc_build(mr_ctx* c, int X, int Y, int Z, int n_sweeps)
{
  if (!c) return MR_CONTRACT;
  if (int g = pending_guard(c)) return g;
  MR_FORWARD(c, mr_mrsdc_build(sl_, X, Y, Z, n_sweeps));
  mr_ctx::SdcScheme M;
  if (n_sweeps < 1 || mrsdc_tables(X, Y, Z, M))
    return set_err(c, MR_CONTRACT, "build_scheme: need X,Y in {3,5}, Z >= 1, sweeps >= 1");
  M.n_sweeps = n_sweeps;
  M.loaded = true;
  c->mrsdc = M;
  return MR_OK;
}

int mr_sdc_integrate(mr_ctx* c, int n_nodes, const double* nodes, const double* S, int n_sweeps,
                     double t0, double tf, double H, uint64_t* n_evals, int* fail_stage)
{
  if (!c) return MR_CONTRACT;
  if (int g = pending_guard(c)) return g;
  if (!nodes || !S || n_nodes < 2 || n_nodes > MR_MAXREF - 2 || n_sweeps < 0)
    return set_err(c, MR_CONTRACT, "sdc_integrate: 2 <= nodes <= 10, S[(n-1) x n], sweeps >= 0");
  SdcRun R{};
  R.single = true;
  R.nf = n_nodes;
  R.Y = n_nodes;
  R.sweeps = n_sweeps;
  R.fine_nodes = nodes;
  R.fine_row = S;
  if (!c->slabs.empty())
    return domain_rc(c, sdc_integrate_dev(c->slabs.data(), (int)c->slabs.size(), R, t0, tf, H,
                                          n_evals, nullptr, fail_stage));
  return sdc_integrate_dev(&c, 1, R, t0, tf, H, n_evals, nullptr, fail_stage);
}

int mr_mrsdc_load(mr_ctx* c, int X, int Y, int n_fine, int n_sweeps, const double* coarse_nodes,
                  const double* fine_nodes, const int* coarse_of_fine,
                  const int* coarse_index_of_fine, const double* fine_row,
                  const int* application_offset, const double* coarse_row)
{
  if (!c) return MR_CONTRACT;
  if (int g = pending_guard(c)) return g;
  MR_FORWARD(c, mr_mrsdc_load(sl_, X, Y, n_fine, n_sweeps, coarse_nodes, fine_nodes,
                              coarse_of_fine, coarse_index_of_fine, fine_row, application_offset,
                              coarse_row));
  if (X < 2 || Y < 2 || n_fine < 2 || n_fine > 4095 || n_sweeps < 0 || Y + X + 4 > 2 * MR_MAXREF ||
      !coarse_nodes || !fine_nodes || !coarse_of_fine || !coarse_index_of_fine || !fine_row ||
      !application_offset || !coarse_row)
    return set_err(c, MR_CONTRACT, "mr_mrsdc_load: bad scheme");
  mr_ctx::SdcScheme M;  // validated before it replaces the loaded scheme
  M.X = X;
  M.Y = Y;
  M.n_fine = n_fine;
  M.n_sweeps = n_sweeps;
  M.coarse_nodes.assign(coarse_nodes, coarse_nodes + X);
  M.fine_nodes.assign(fine_nodes, fine_nodes + n_fine);
  M.coarse_of_fine.assign(coarse_of_fine, coarse_of_fine + n_fine);
  M.coarse_index_of_fine.assign(coarse_index_of_fine, coarse_index_of_fine + n_fine);
  M.fine_row.assign(fine_row, fine_row + (size_t)(n_fine - 1) * Y);
  M.application_offset.assign(application_offset, application_offset + (n_fine - 1));
  M.coarse_row.assign(coarse_row, coarse_row + (size_t)(n_fine - 1) * X);
  for (int q = 0; q < n_fine; ++q)
    if (M.coarse_of_fine[q] < 0 || M.coarse_of_fine[q] >= X || M.coarse_index_of_fine[q] >= X)
      return set_err(c, MR_CONTRACT, "mr_mrsdc_load: coarse index out of range");
  for (int q = 0; q + 1 < n_fine; ++q)
    if (M.application_offset[q] < 0 || M.application_offset[q] + Y > n_fine)
      return set_err(c, MR_CONTRACT, "mr_mrsdc_load: application offset out of range");
  M.loaded = true;
  c->mrsdc = std::move(M);
  return MR_OK;
}

int mr_mrsdc_integrate(mr_ctx* c, double t0, double tf, double H, uint64_t* counters,
                       int* fail_stage)
{
  if (!c) return MR_CONTRACT;
  if (int g = pending_guard(c)) return g;
  mr_ctx* m = c->slabs.empty() ? c : c->slabs[0];
  if (!m->mrsdc.loaded) return set_err(c, MR_CONTRACT, "mrsdc_integrate: no scheme (mr_mrsdc_load)");
  const auto& M = m->mrsdc;
  SdcRun R{};
  R.single = false;
  R.X = M.X;
  R.Y = M.Y;
  R.nf = M.n_fine;
  R.sweeps = M.n_sweeps;
  R.coarse_nodes = M.coarse_nodes.data();
  R.fine_nodes = M.fine_nodes.data();
  R.fine_row = M.fine_row.data();
  R.coarse_row = M.coarse_row.data();
  R.coarse_of_fine = M.coarse_of_fine.data();
  R.coarse_index_of_fine = M.coarse_index_of_fine.data();
  R.application_offset = M.application_offset.data();
  uint64_t* cf = counters ? counters + MR_CNT_FAST_EVALS : nullptr;
  uint64_t* cx = counters ? counters + MR_CNT_EXPLICIT_EVALS : nullptr;
  if (!c->slabs.empty())
    return domain_rc(c, sdc_integrate_dev(c->slabs.data(), (int)c->slabs.size(), R, t0, tf, H, cf,
                                          cx, fail_stage));
  return sdc_integrate_dev(&c, 1, R, t0, tf, H, cf, cx, fail_stage);
}

// reference_solution (erk.cpp:59-75): erk_integrate of cash-karp5
// (butcher.cpp:305-321, written exactly as there), no counters.
int mr_reference_solution(mr_ctx* c, double t0, double tf, double h, int* fail_stage)
{
  if (!c) return MR_CONTRACT;
  if (int g = pending_guard(c)) return g;
  double A[6][6] = {{0}}, b[6] = {0};
  A[1][0] = 1.0 / 5.0;
  A[2][0] = 3.0 / 40.0; A[2][1] = 9.0 / 40.0;
  A[3][0] = 3.0 / 10.0; A[3][1] = -9.0 / 10.0; A[3][2] = 6.0 / 5.0;
  A[4][0] = -11.0 / 54.0; A[4][1] = 5.0 / 2.0; A[4][2] = -70.0 / 27.0; A[4][3] = 35.0 / 27.0;
  A[5][0] = 1631.0 / 55296.0; A[5][1] = 175.0 / 512.0; A[5][2] = 575.0 / 13824.0;
  A[5][3] = 44275.0 / 110592.0; A[5][4] = 253.0 / 4096.0;
  b[0] = 37.0 / 378.0; b[2] = 250.0 / 621.0; b[3] = 125.0 / 594.0; b[5] = 512.0 / 1771.0;
  if (!c->slabs.empty())
    return domain_rc(c, erk_integrate_dev(c->slabs.data(), (int)c->slabs.size(), 6, &A[0][0], b,
                                          t0, tf, h, nullptr, fail_stage));
  return erk_integrate_dev(&c, 1, 6, &A[0][0], b, t0, tf, h, nullptr, fail_stage);
}

int mr_slow_rhs(mr_ctx* c, double t, const double* y, double* out)
{
  (void)t;
  if (!c || !y || !out) return MR_CONTRACT;
  if (int g = pending_guard(c)) return g;
  if (!c->slabs.empty()) {
    if (!c->has_grid || c->slabs[0]->slow_kind < 0)
      return set_err(c, MR_CONTRACT, "slow plugin not set");
    if (c->slabs[0]->slow_kind == SK_NONE) {
      std::memset(out, 0, c->dof * sizeof(double));
      return MR_OK;
    }
    for (mr_ctx* sl : c->slabs)
      if (sl->slow_kind == SK_STENCIL && sl->n0l < sl->M)
        return set_err(c, MR_CONTRACT, "slab thinner than the stencil ghost width");
    return domain_rhs(c, 1, y, out);
  }
  if (!c->has_grid || c->slow_kind < 0) return set_err(c, MR_CONTRACT, "slow plugin not set");
  if (c->slow_kind == SK_STENCIL && c->n0l < c->M)
    return set_err(c, MR_CONTRACT, "slab thinner than the stencil ghost width");
  cudaSetDevice(c->device);
  int rc = ensure_scratch(c);
  if (rc) return rc;
  MR_CUDA_TRY(c, cudaMemcpyAsync(c->scr_in, y, c->dof * sizeof(double), cudaMemcpyHostToDevice,
                                 c->stream));
  if (c->slow_kind == SK_NONE) {
    MR_CUDA_TRY(c, cudaMemsetAsync(c->scr_out, 0, c->dof * sizeof(double), c->stream));
  } else {
    mr_ctx* cs[1] = {c};
    const double* yc[1] = {c->scr_in};
    double* oc[1] = {c->scr_out};
    rc = eval_slow(cs, 1, yc, oc, c->stream);
    if (rc) return rc;
  }
  MR_CUDA_TRY(c, cudaMemcpyAsync(out, c->scr_out, c->dof * sizeof(double), cudaMemcpyDeviceToHost,
                                 c->stream));
  MR_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return MR_OK;
}

// ---------------- reductions ----------------
static int reduce(mr_ctx* c, int kind, const double* x, const double* w, size_t n, double* out)
{
  if (!c || !x || !out) return MR_CONTRACT;
  if (int g = pending_guard(c)) return g;
  MR_NOT_ON_DOMAIN(c, "device-pointer reductions");
  cudaSetDevice(c->device);
  const int nb = reduce_blocks();
  double* part = c->d_red;
  double* dout = c->d_red + nb;
  MR_CUDA_TRY(c, launch_reduce(kind, x, w, n, part, nb, dout, c->stream));
  c->launches += 2;
  MR_CUDA_TRY(c, cudaMemcpyAsync(c->h_red, dout, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  MR_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  *out = c->h_red[0];
  return MR_OK;
}

int mr_wrms_norm(mr_ctx* c, const double* x, const double* w, size_t n, double* out)
{
  if (n == 0) return set_err(c, MR_CONTRACT, "wrms_norm: empty vector");
  if (!w) return set_err(c, MR_CONTRACT, "wrms_norm: weights required");
  return reduce(c, RED_WRMS, x, w, n, out);
}

int mr_two_norm(mr_ctx* c, const double* x, size_t n, double* out)
{
  if (n == 0) { if (out) *out = 0.0; return MR_OK; }
  return reduce(c, RED_TWO, x, nullptr, n, out);
}

int mr_dot(mr_ctx* c, const double* x, const double* y, size_t n, double* out)
{
  if (n == 0) { if (out) *out = 0.0; return MR_OK; }
  if (!y) return set_err(c, MR_CONTRACT, "dot: null vector");
  return reduce(c, RED_DOT, x, y, n, out);
}

int mr_max_norm(mr_ctx* c, const double* x, size_t n, double* out)
{
  if (n == 0) return set_err(c, MR_CONTRACT, "max_norm: empty vector");
  return reduce(c, RED_MAX, x, nullptr, n, out);
}

int mr_max_norm_component(mr_ctx* c, const double* x, size_t n, size_t offset, size_t count,
                          double* out)
{
  if (count == 0 || offset + count > n)
    return set_err(c, MR_CONTRACT, "max_norm_component: bad slice");
  return reduce(c, RED_MAX, x + offset, nullptr, count, out);
}

int mr_all_finite(mr_ctx* c, const double* x, size_t n, int* out)
{
  if (!out) return MR_CONTRACT;
  if (n == 0) { *out = 1; return MR_OK; }
  double bad = 0.0;
  int rc = reduce(c, RED_NONFINITE, x, nullptr, n, &bad);
  if (rc) return rc;
  *out = bad == 0.0 ? 1 : 0;
  return MR_OK;
}

// ---------------- multi-GPU ----------------
int mr_nccl_unique_id(char* id128)
{
  if (!id128) return MR_CONTRACT;
  ncclUniqueId id;
  if (!nccl_api().ok || nccl_api().GetUniqueId(&id) != ncclSuccess) return MR_CUDA;
  std::memcpy(id128, id.internal, NCCL_UNIQUE_ID_BYTES);
  return MR_OK;
}

static int comm_init_nccl(mr_ctx* c, int nranks, int rank, const char* id128)
{
  ncclUniqueId id;
  std::memcpy(id.internal, id128, NCCL_UNIQUE_ID_BYTES);
  MR_NCCL_TRY(c, CommInitRank(&c->comm, nranks, id, rank));
  c->nranks = nranks;
  c->rank = rank;
  c->halo_elems = 0;  // reallocate halos with receive buffers
  return MR_OK;
}

int mr_comm_init(mr_ctx* c, int nranks, int rank, const char* id128)
{
  if (!c || nranks < 1 || rank < 0 || rank >= nranks || !id128) return MR_CONTRACT;
  if (int g = pending_guard(c)) return g;
  MR_NOT_ON_DOMAIN(c, "mr_comm_init");
  if (c->comm) return set_err(c, MR_CONTRACT, "mr_comm_init: communicator already set");
  cudaSetDevice(c->device);
  if (nranks == 1) {  // no communicator: the periodic single-slab path
    c->nranks = 1;
    c->rank = 0;
    return MR_OK;
  }
  return comm_init_nccl(c, nranks, rank, id128);
}

// one-rank NCCL communicator: the whole NCCL path (halo send/recv to itself,
// failure-key all-reduce, all-gathered CG dot products) on one GPU, so tests
// and the benchmark can compare it with the plain single-slab path
int mr_comm_init_loopback(mr_ctx* c)
{
  if (!c) return MR_CONTRACT;
  if (int g = pending_guard(c)) return g;
  MR_NOT_ON_DOMAIN(c, "mr_comm_init_loopback");
  if (c->comm) return set_err(c, MR_CONTRACT, "mr_comm_init_loopback: communicator already set");
  cudaSetDevice(c->device);
  ncclUniqueId id;
  if (!nccl_api().ok) return set_err(c, MR_CUDA, "NCCL (libnccl.so.2) not available");
  if (nccl_api().GetUniqueId(&id) != ncclSuccess) return set_err(c, MR_CUDA, "ncclGetUniqueId failed");
  return comm_init_nccl(c, 1, 0, reinterpret_cast<const char*>(id.internal));
}

int mr_group_step(mr_ctx** cs, int n, double t, double H, uint64_t* counters, int* fail_stage)
{
  if (!cs || n < 1) return MR_CONTRACT;
  for (int r = 0; r < n; ++r) {
    if (!cs[r] || cs[r]->device != cs[0]->device || cs[r]->nranks != 1 || cs[r]->comm ||
        !cs[r]->slabs.empty() || cs[r]->in_domain)
      return set_err(cs[0], MR_CONTRACT, "mr_group_step: contexts must share one device");
    if (cs[r]->pending.active)
      return set_err(cs[0], MR_CONTRACT, "an asynchronous step is in flight: call mr_mri_step_wait first");
  }
  cudaSetDevice(cs[0]->device);
  // order all slabs on the first context's stream
  for (int r = 1; r < n; ++r) cudaStreamSynchronize(cs[r]->stream);
  int rc = domain_step(cs, n, t, H, counters, fail_stage);
  if (rc)
    for (int r = 1; r < n; ++r) cs[r]->err = cs[0]->err;
  return rc;
}

// ---------------- host-only inspection ----------------
int mr_coupling_inspect(const char* text, int m, int* s, int* kinds, int* eval_at, int* n_sub,
                        char* err, size_t errlen)
{
  if (!text) return MR_CONTRACT;
  Coupling cp;
  std::string e;
  const int rc = read_coupling_text(text, cp, e);
  if (rc) {
    if (err && errlen) std::snprintf(err, errlen, "%s", e.c_str());
    return rc;
  }
  if (s) *s = cp.s;
  for (int i = 0; i < cp.s; ++i) {
    if (kinds) kinds[i] = cp.kind[i];
    if (eval_at) eval_at[i] = cp.eval_at[i] ? 1 : 0;
    if (n_sub) {
      n_sub[i] = 0;
      if (i > 0 && cp.kind[i] == MR_STAGE_FAST_IVP)
        n_sub[i] = (int)std::max(1L, std::lround((double)m * (cp.c[i] - cp.c[i - 1])));
    }
  }
  return MR_OK;
}

int mr_step_counts(const char* text, int s_f, int m, int fast_present, int slow_present,
                   uint64_t* counters, char* err, size_t errlen)
{
  if (!text || !counters || s_f < 1 || m < 1) return MR_CONTRACT;
  mr_ctx tmp;
  std::string e;
  const int rc = read_coupling_text(text, tmp.cp, e);
  if (rc) {
    if (err && errlen) std::snprintf(err, errlen, "%s", e.c_str());
    return rc;
  }
  tmp.has_coupling = true;
  tmp.tab.s = s_f;
  tmp.m = m;
  tmp.fast_kind = fast_present ? FK_LINEAR : FK_NONE;
  tmp.slow_kind = slow_present ? SK_LINEAR : SK_NONE;
  for (int i = 0; i < kMaxStages; ++i) {  // solves: one Newton iteration (linear stage problem)
    tmp.solve_evals[i] = 2;
    tmp.solve_nl[i] = 1;
  }
  const Plan p = build_plan(&tmp);
  for (const Op& o : p.ops)
    if (o.type == Op::MISSING) {
      if (err && errlen) std::snprintf(err, errlen, "missing slow value at stage %d", o.stage);
      return MR_INTEGRATION;
    }
  add_counts_full(&tmp, p, 0.0, 1.0, counters);
  return MR_OK;
}

// ---------------- instrumentation ----------------
// Debug (not part of include/mri_b200.h): HBM throughput of the vector
// kernels (K3 update, sum/add combines, K5 IMEX kernels, K4 reductions) on
// this context's state-sized buffers.  out[2*q] = ms per launch, out[2*q+1] =
// algorithmic GB/s; returns the number of kernels measured.
int mr_debug_vector_bench(mr_ctx* c, double* out, int maxn)
{
  if (!c || !c->has_grid || c->slow_kind != SK_STENCIL) return -1;
  cudaSetDevice(c->device);
  if (ensure_state(c) || ensure_slots(c, 3) || ensure_cg(c) || ensure_halo(c)) return -1;
  cudaStream_t st = c->stream;
  const size_t n = c->dof;
  const double B = 8.0 * (double)n;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int q = 0;
  auto timeit = [&](double bytes, auto&& launch) {
    launch();
    cudaEventRecord(e0, st);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) launch();
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (q < maxn) {
      out[2 * q] = ms / reps;
      out[2 * q + 1] = bytes / (ms / reps * 1e-3) / 1e9;
    }
    ++q;
  };
  double* y = c->y_state;
  double* o = c->y_work;
  double** sl = c->slots.data();
  const double* f3[3] = {sl[0], sl[1], sl[2]};
  const double cf3[3] = {1e-3, 2e-3, 3e-3};
  cudaMemsetAsync(c->d_fail, 0xFF, sizeof(unsigned long long), st);
  timeit(3 * B, [&] { launch_update(y, o, 1, f3, cf3, n, 0, c->d_fail, st); });
  timeit(5 * B, [&] { launch_update(y, o, 3, f3, cf3, n, 0, c->d_fail, st); });
  timeit(4 * B, [&] { launch_sum_rhs(n, sl[0], sl[1], sl[2], o, st); });
  const double* lo = c->send_hi;
  const double* hi = c->send_lo;
  launch_halo_pack(y, c->send_lo, c->send_hi, c->ncomp, c->n0l, c->plane, c->M, st);
  LapArgs la = lap_args(c, 1e-3);
  timeit(2 * B, [&] { launch_lap7(0, la, y, lo, hi, nullptr, nullptr, o, nullptr, nullptr, nullptr, nullptr, st); });
  timeit(5 * B, [&] { launch_lap7(1, la, y, lo, hi, c->cg_known, nullptr, c->cg_r, c->cg_z, c->cg_p, c->cg_part, c->cg_part2, st); });
  timeit(2 * B, [&] { launch_lap7(2, la, c->cg_p, lo, hi, nullptr, nullptr, c->cg_q, nullptr, nullptr, c->cg_part, nullptr, st); });
  cudaMemsetAsync(c->cg_sc, 0, 8 * sizeof(double), st);
  timeit(7 * B, [&] { launch_cg_update(n, la.dg, c->cg_sc, o, c->cg_r, c->cg_z, c->cg_p, c->cg_q, c->cg_part, st); });
  timeit(3 * B, [&] { launch_cg_p(n, c->cg_sc, c->cg_p, c->cg_z, st); });
  timeit(3 * B, [&] { launch_recover_fi(n, 1.0, o, c->cg_known, c->cg_q, 0, c->d_fail, st); });
  const int nb = reduce_blocks();
  timeit(2 * B, [&] { launch_reduce(RED_WRMS, y, o, n, c->d_red, nb, c->d_red + nb, st); });
  timeit(2 * B, [&] { launch_reduce(RED_DOT, y, o, n, c->d_red, nb, c->d_red + nb, st); });
  timeit(1 * B, [&] { launch_reduce(RED_MAX, y, nullptr, n, c->d_red, nb, c->d_red + nb, st); });
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return q;
}

// Debug (not part of include/mri_b200.h): let the pipelined host-buffer step
// run on an NCCL rank (off by default, see pipeline_ok)
int mr_debug_pipeline_nccl(mr_ctx* c, int on)
{
  if (!c) return MR_CONTRACT;
  c->pipeline_nccl = on != 0;
  return MR_OK;
}

// Debug (not part of include/mri_b200.h): chemistry phase cycles of an
// MR_PHASE_PROF build, summed over blocks; out[7] = blocks.  reset zeroes them.
int mr_debug_chem_phases(mr_ctx* c, uint64_t* out, int reset)
{
  if (!c || !c->chemP || !c->chemP->prof) return MR_CONTRACT;
  cudaSetDevice(c->device);
  MR_CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (out)
    MR_CUDA_TRY(c, cudaMemcpy(out, c->chemP->prof, 8 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  if (reset) MR_CUDA_TRY(c, cudaMemset(c->chemP->prof, 0, 8 * sizeof(uint64_t)));
  return MR_OK;
}

void* mr_stream(mr_ctx* c) { return c ? (void*)c->stream : nullptr; }
uint64_t mr_launch_count(const mr_ctx* c)
{
  if (!c) return 0;
  uint64_t n = c->launches;
  for (const mr_ctx* sl : c->slabs) n += sl->launches;
  return n;
}
double mr_chem_flops_per_eval(const mr_ctx* c)
{
  if (c && !c->slabs.empty()) c = c->slabs[0];
  return c ? c->chem_flops : 0.0;
}

int mr_fp64_peak(mr_ctx* c, double* tflops)
{
  if (!c || !tflops) return MR_CONTRACT;
  if (!c->slabs.empty()) c = c->slabs[0];
  cudaSetDevice(c->device);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  double best = 0.0;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(a, c->stream);
    MR_CUDA_TRY(c, launch_fp64_peak(c->d_red, blocks, threads, iters, c->stream));
    cudaEventRecord(b, c->stream);
    MR_CUDA_TRY(c, cudaEventSynchronize(b));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    const double flops = 2.0 * 64.0 * (double)iters * blocks * threads;
    if (rep > 0) best = std::max(best, flops / (ms * 1e-3) / 1e12);
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  *tflops = best;
  return MR_OK;
}

int mr_set_profiling(mr_ctx* c, int enable)
{
  if (!c) return MR_CONTRACT;
  if (int g = pending_guard(c)) return g;
  MR_FORWARD(c, mr_set_profiling(sl_, enable));
  c->profile = enable != 0;
  return MR_OK;
}

int mr_last_step_profile(const mr_ctx* c, double* chem_ms, double* slow_ms, double* other_ms)
{
  if (!c) return MR_CONTRACT;
  if (!c->slabs.empty()) c = c->slabs[0];
  if (chem_ms) *chem_ms = c->prof_chem;
  if (slow_ms) *slow_ms = c->prof_slow;
  if (other_ms) *other_ms = c->prof_other;
  return MR_OK;
}

}  // extern "C"
