// kernels_chain.cu -- K1: fused cell-local MRI stage chain.
//
// One launch runs a maximal run of cell-local MRI stages (fast IVPs and
// explicit updates with no slow evaluation in between) for every cell:
//
//   build_forcing        proj/src/mri.cpp:266-303   (coefficients in registers)
//   n_sub x erk_step     proj/src/erk.cpp:9-38      (stage values in registers)
//   fast_rhs lambda      proj/src/mri.cpp:364-371   (f_fast + Horner forcing,
//                                                    proj/include/multirate/mri.hpp:98-107)
//   explicit update      proj/src/mri.cpp:380-384, :422-424
//   all_finite checks    proj/src/erk.cpp:24-26, :34-36, proj/src/mri.cpp:427-431
//
// Y and the referenced slow-stage values fE_j are read once and Y written once
// per chain (bytes = 8*ncomp*ncell*(2 + n_ref)); everything in
// between stays on chip.  The stepper arithmetic (stage sums, forcing, Horner,
// tau) uses __dmul_rn/__dadd_rn in the reference's exact order, so it is bit
// identical to the reference wherever the RHS is (the linear test plugins).
//
// This generic kernel serves the linear test plugin (LinearTwoRateOde per
// cell) and an absent fast partition; the chemistry plugin has its own block
// kernel (kernels_chem.cuh).  Thread mapping: G lanes cooperate on one cell
// (CPW = 32/G cells per warp, lane = cw + CPW*lg); lane lg owns components
// lg + G*t (t < SPL).
#include <cuda_runtime.h>

#include "common.cuh"

namespace {

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
// per-cell linear map (G == 1): f_a = sum_b A[a][b] v_b in mat_apply order
// (proj/src/models.cpp:30-34)
template <int SPL>
__device__ __forceinline__ void lin_eval(const LinDev& L, const double (&v)[SPL], double (&f)[SPL])
{
#pragma unroll
  for (int a = 0; a < SPL; ++a) {
    double acc = 0.0;
    if (a < L.n) {
      acc = dmul(L.A[a * L.n], v[0]);
#pragma unroll
      for (int b = 1; b < SPL; ++b)
        if (b < L.n) acc = dadd(acc, dmul(L.A[a * L.n + b], v[b]));
    }
    f[a] = acc;
  }
}

template <int FK, int SPL>
__device__ __forceinline__ void fast_eval(const LinDev& lin, const double (&v)[SPL],
                                          double (&f)[SPL])
{
  static_assert(FK == FK_LINEAR || FK == FK_NONE, "chemistry runs in kernels_chem.cuh");
  if constexpr (FK == FK_LINEAR) {
    lin_eval<SPL>(lin, v, f);
  } else {
#pragma unroll
    for (int t = 0; t < SPL; ++t) f[t] = 0.0;  // StateVector(v.size())
  }
}

template <int FK, int G, int SPL, int MAXS, int NDEG>
__global__ void __launch_bounds__(128) chain_kernel(const ChainArgs a, const LinDev lin)
{
  constexpr int CPW = 32 / G;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cw = lane % CPW, lg = lane / CPW;
  const size_t warp_cell0 = ((size_t)blockIdx.x * (blockDim.x >> 5) + warp) * CPW;
  if (warp_cell0 >= a.ncell) return;  // whole warp idle
  const size_t cell = warp_cell0 + cw;
  const bool active = cell < a.ncell;
  const size_t nc = a.ncell;
  const int ncomp = a.ncomp;

  double y[SPL];
#pragma unroll
  for (int t = 0; t < SPL; ++t) {
    const int comp = lg + G * t;
    y[t] = (active && comp < ncomp) ? a.y_in[(size_t)comp * nc + cell] : 0.0;
  }
  bool failed = !active;

  for (int si = 0; si < a.nst; ++si) {
    const ChainStageDev& st = a.st[si];
    if (st.kind != 0) {
      // ExplicitUpdate: known = Y + sum_j (H*wbar_ij) fE_j, j ascending
      for (int r = 0; r < st.nref; ++r) {
        const double cf = st.coef[0][r];
        if (cf == 0.0) continue;
        const double* __restrict__ fv = a.fE[st.ref_slot[r]];
#pragma unroll
        for (int t = 0; t < SPL; ++t) {
          const int comp = lg + G * t;
          if (active && comp < ncomp) y[t] = dadd(y[t], dmul(cf, fv[(size_t)comp * nc + cell]));
        }
      }
      if (!failed) {
        bool bad = false;
#pragma unroll
        for (int t = 0; t < SPL; ++t)
          if (lg + G * t < ncomp && !isfinite(y[t])) bad = true;
        if (bad) {
          atomicMin(a.fail, mr_fail_key(st.mri_stage, 0, 0));
          failed = true;
        }
      }
      continue;
    }

    // FastIvp: forcing coefficients r_k = sum_j (omega[k][i][j]/dc) fE_j
    double rc[NDEG][SPL];
#pragma unroll
    for (int k = 0; k < NDEG; ++k)
#pragma unroll
      for (int t = 0; t < SPL; ++t) rc[k][t] = 0.0;
    for (int r = 0; r < st.nref; ++r) {
      const double* __restrict__ fv = a.fE[st.ref_slot[r]];
#pragma unroll
      for (int t = 0; t < SPL; ++t) {
        const int comp = lg + G * t;
        const double x = (active && comp < ncomp) ? fv[(size_t)comp * nc + cell] : 0.0;
#pragma unroll
        for (int k = 0; k < NDEG; ++k) {
          const double cf = st.coef[k][r];
          if (cf != 0.0) rc[k][t] = dadd(rc[k][t], dmul(cf, x));
        }
      }
    }

    const double h = st.h_sub;
    const int s = a.tab.s;
    for (int sub = 0; sub < st.n_sub; ++sub) {
      const double t0 = dadd(st.t_start, dmul((double)sub, h));
      double pre[MAXS][SPL];
      double out[SPL];
#pragma unroll
      for (int i = 0; i < MAXS; ++i)
#pragma unroll
        for (int t = 0; t < SPL; ++t) pre[i][t] = y[t];
#pragma unroll
      for (int t = 0; t < SPL; ++t) out[t] = y[t];

      for (int j = 0; j < s; ++j) {
        double stg[SPL];
#pragma unroll
        for (int t = 0; t < SPL; ++t) stg[t] = pre[0][t];
#pragma unroll
        for (int i = 1; i < MAXS; ++i)
          if (i == j) {
#pragma unroll
            for (int t = 0; t < SPL; ++t) stg[t] = pre[i][t];
          }
        if (!failed) {
          bool bad = false;
#pragma unroll
          for (int t = 0; t < SPL; ++t)
            if (lg + G * t < ncomp && !isfinite(stg[t])) bad = true;
          if (bad) {
            atomicMin(a.fail, mr_fail_key(st.mri_stage, sub, j));
            failed = true;
          }
        }
        const double theta = dadd(t0, dmul(a.tab.c[j], h));
        const double tau = __ddiv_rn(dadd(theta, -st.t_start), st.span);
        double f[SPL];
        fast_eval<FK, SPL>(lin, stg, f);
        const double hb = dmul(h, a.tab.b[j]);
        const bool use_b = a.tab.b[j] != 0.0;
#pragma unroll
        for (int t = 0; t < SPL; ++t) {
          double fr = rc[NDEG - 1][t];
#pragma unroll
          for (int k = NDEG - 2; k >= 0; --k) fr = dadd(dmul(fr, tau), rc[k][t]);
          const double kj = dadd(f[t], fr);
#pragma unroll
          for (int i = 1; i < MAXS; ++i) {
            if (i > j && i < s) {
              const double Aij = a.tab.A[i][j];
              if (Aij != 0.0) pre[i][t] = dadd(pre[i][t], dmul(dmul(h, Aij), kj));
            }
          }
          if (use_b) out[t] = dadd(out[t], dmul(hb, kj));
        }
      }
      if (!failed) {
        bool bad = false;
#pragma unroll
        for (int t = 0; t < SPL; ++t)
          if (lg + G * t < ncomp && !isfinite(out[t])) bad = true;
        if (bad) {
          atomicMin(a.fail, mr_fail_key(st.mri_stage, sub, s));
          failed = true;
        }
      }
#pragma unroll
      for (int t = 0; t < SPL; ++t) y[t] = out[t];
    }
  }

#pragma unroll
  for (int t = 0; t < SPL; ++t) {
    const int comp = lg + G * t;
    if (active && comp < ncomp) a.y_out[(size_t)comp * nc + cell] = y[t];
  }
}

// single fast-RHS evaluation (Mode A: reference RhsFn backed by the GPU)
template <int FK, int G, int SPL>
__global__ void __launch_bounds__(128) fast_rhs_kernel(const double* __restrict__ yin,
                                                       double* __restrict__ fout, size_t nc,
                                                       int ncomp, const LinDev lin)
{
  constexpr int CPW = 32 / G;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cw = lane % CPW, lg = lane / CPW;
  const size_t warp_cell0 = ((size_t)blockIdx.x * (blockDim.x >> 5) + warp) * CPW;
  if (warp_cell0 >= nc) return;
  const size_t cell = warp_cell0 + cw;
  const bool active = cell < nc;
  double v[SPL], f[SPL];
#pragma unroll
  for (int t = 0; t < SPL; ++t) {
    const int comp = lg + G * t;
    v[t] = (active && comp < ncomp) ? yin[(size_t)comp * nc + cell] : 0.0;
  }
  fast_eval<FK, SPL>(lin, v, f);
#pragma unroll
  for (int t = 0; t < SPL; ++t) {
    const int comp = lg + G * t;
    if (active && comp < ncomp) fout[(size_t)comp * nc + cell] = f[t];
  }
}

constexpr int kBlock = 128;

template <int FK, int G, int SPL, int MAXS, int NDEG>
cudaError_t run_chain(const ChainArgs& a, const LinDev& lin, cudaStream_t st)
{
  constexpr int CPB = (kBlock / 32) * (32 / G);
  const size_t blocks = (a.ncell + CPB - 1) / CPB;
  chain_kernel<FK, G, SPL, MAXS, NDEG><<<(unsigned)blocks, kBlock, 0, st>>>(a, lin);
  return cudaGetLastError();
}

template <int FK, int G, int SPL>
cudaError_t run_rhs(const double* y, double* out, size_t nc, int ncomp, const LinDev& lin,
                    cudaStream_t st)
{
  constexpr int CPB = (kBlock / 32) * (32 / G);
  const size_t blocks = (nc + CPB - 1) / CPB;
  fast_rhs_kernel<FK, G, SPL><<<(unsigned)blocks, kBlock, 0, st>>>(y, out, nc, ncomp, lin);
  return cudaGetLastError();
}

}  // namespace

// (G, SPL) layouts of the absent fast partition (lanes per cell grow with the
// component count so a thread carries at most 3 components)
#define MR_NONE_LAYOUTS(X) X(4, 3) X(8, 2) X(8, 3) X(16, 2) X(32, 2)

int chain_pick(ChainCfg* cfg, int fast_kind, int ncomp, int s_f, int ndeg)
{
  cfg->fast_kind = fast_kind;
  cfg->maxs = s_f <= 4 ? 4 : 6;
  cfg->ndeg = ndeg;
  if (s_f > MR_MAXS || ndeg < 1 || ndeg > MR_MAXDEG) return 1;
  if (fast_kind == FK_LINEAR) {
    cfg->G = 1;
    cfg->SPL = ncomp <= 2 ? 2 : ncomp <= 4 ? 4 : 8;
    return ncomp <= MR_MAXLIN ? 0 : 1;
  }
  if (fast_kind != FK_NONE) return 1;
  if (ncomp <= 12) { cfg->G = 4; cfg->SPL = 3; }
  else if (ncomp <= 16) { cfg->G = 8; cfg->SPL = 2; }
  else if (ncomp <= 24) { cfg->G = 8; cfg->SPL = 3; }
  else if (ncomp <= 32) { cfg->G = 16; cfg->SPL = 2; }
  else if (ncomp <= 64) { cfg->G = 32; cfg->SPL = 2; }
  else return 1;
  return 0;
}

cudaError_t launch_chain(const ChainCfg& cfg, const ChainArgs& a, const LinDev& lin,
                         cudaStream_t st)
{
#define MR_DISPATCH_MS(FK, GG, SS)                                                    \
  if (cfg.maxs == 4 && cfg.ndeg == 1) return run_chain<FK, GG, SS, 4, 1>(a, lin, st); \
  if (cfg.maxs == 4 && cfg.ndeg == 2) return run_chain<FK, GG, SS, 4, 2>(a, lin, st); \
  if (cfg.maxs == 6 && cfg.ndeg == 1) return run_chain<FK, GG, SS, 6, 1>(a, lin, st); \
  if (cfg.maxs == 6 && cfg.ndeg == 2) return run_chain<FK, GG, SS, 6, 2>(a, lin, st);
#define MR_NONE_CASE(GG, SS) \
  if (cfg.G == GG && cfg.SPL == SS) { MR_DISPATCH_MS(FK_NONE, GG, SS) }
  if (cfg.fast_kind == FK_NONE) { MR_NONE_LAYOUTS(MR_NONE_CASE) }
  else if (cfg.fast_kind == FK_LINEAR) {
    if (cfg.SPL == 2) { MR_DISPATCH_MS(FK_LINEAR, 1, 2) }
    if (cfg.SPL == 4) { MR_DISPATCH_MS(FK_LINEAR, 1, 4) }
    if (cfg.SPL == 8) { MR_DISPATCH_MS(FK_LINEAR, 1, 8) }
  }
#undef MR_NONE_CASE
#undef MR_DISPATCH_MS
  return cudaErrorInvalidConfiguration;
}

cudaError_t launch_fast_rhs(const ChainCfg& cfg, const double* y, double* out, size_t ncell,
                            int ncomp, const LinDev& lin, cudaStream_t st)
{
#define MR_RHS_NONE(GG, SS) \
  if (cfg.G == GG && cfg.SPL == SS) return run_rhs<FK_NONE, GG, SS>(y, out, ncell, ncomp, lin, st);
  if (cfg.fast_kind == FK_NONE) { MR_NONE_LAYOUTS(MR_RHS_NONE) }
  else if (cfg.fast_kind == FK_LINEAR) {
    if (cfg.SPL == 2) return run_rhs<FK_LINEAR, 1, 2>(y, out, ncell, ncomp, lin, st);
    if (cfg.SPL == 4) return run_rhs<FK_LINEAR, 1, 4>(y, out, ncell, ncomp, lin, st);
    if (cfg.SPL == 8) return run_rhs<FK_LINEAR, 1, 8>(y, out, ncell, ncomp, lin, st);
  }
#undef MR_RHS_NONE
  return cudaErrorInvalidConfiguration;
}
