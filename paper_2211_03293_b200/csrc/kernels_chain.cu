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
// Thread mapping: G lanes cooperate on one cell (CPW = 32/G cells per warp,
// lane = cw + CPW*lg); lane lg owns components lg + G*t (t < SPL).  For the
// chemistry the G lanes split the reactions (j = lg + G*t) and the species;
// per-cell scratch (C, exp(g/RT), exp(-g/RT), rates of progress q) lives in
// shared memory laid out [item][CPW] so a warp's species-phase accesses are
// 32 consecutive doubles.  All cross-lane combines are butterflies or fixed
// CSR orders, so results are bitwise run-to-run deterministic.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace {

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
// (used by the generic kernel's chemistry branch, instantiated only when the
// block chemistry kernel cannot take a mechanism)
[[maybe_unused]] __device__ __forceinline__ double4 ldg4(const double4* p)
{
  const double2 lo = __ldg(reinterpret_cast<const double2*>(p));
  const double2 hi = __ldg(reinterpret_cast<const double2*>(p) + 1);
  return make_double4(lo.x, lo.y, hi.x, hi.y);
}

// ---------------------------------------------------------------------------
// Per-cell synthetic Arrhenius chemistry (CPU form in
// oracle/mri_oracle.c chem_cell).  v/f: this lane's components.
// ---------------------------------------------------------------------------
template <int G, int SPL>
__device__ __forceinline__ void chem_eval(const ChemDev& ch, const double (&v)[SPL],
                                          double (&f)[SPL], double* sm, int lg)
{
  constexpr int CPW = 32 / G;
  const int S = ch.S, S1 = ch.S + 1, Sp = ch.Spad;
  const double* __restrict__ sp = ch.sp;

  // temperature from energy: e(T) = E0 + E1 T + E2 T^2, closed-form root
  double p0 = 0.0, p1 = 0.0, p2 = 0.0, e = 0.0;
#pragma unroll
  for (int t = 0; t < SPL; ++t) {
    const int comp = lg + G * t;
    if (comp < S) {
      p0 += v[t] * __ldg(sp + 6 * Sp + comp);
      p1 += v[t] * __ldg(sp + 7 * Sp + comp);
      p2 += v[t] * __ldg(sp + 8 * Sp + comp);
    } else if (comp == S) {
      e = v[t];
    }
  }
#pragma unroll
  for (int o = CPW; o < 32; o <<= 1) {  // butterfly: every lane ends bitwise equal
    p0 += __shfl_xor_sync(0xffffffffu, p0, o);
    p1 += __shfl_xor_sync(0xffffffffu, p1, o);
    p2 += __shfl_xor_sync(0xffffffffu, p2, o);
    e += __shfl_xor_sync(0xffffffffu, e, o);
  }
  const double de = e - p0;
  const double T = (2.0 * de) / (p1 + sqrt(p1 * p1 + 4.0 * p2 * de));
  const double lnT = log(T);
  const double invT = 1.0 / T;

  // species: concentrations and exp(+-g_k/RT)
#pragma unroll
  for (int t = 0; t < SPL; ++t) {
    const int comp = lg + G * t;
    if (comp < S) {
      const double g = __ldg(sp + comp) * invT + __ldg(sp + Sp + comp) * (1.0 - lnT) -
                       __ldg(sp + 2 * Sp + comp) * T - __ldg(sp + 3 * Sp + comp);
      const double Ek = exp(g);
      sm[comp * CPW] = __ldg(sp + 4 * Sp + comp) * v[t];
      sm[(S1 + comp) * CPW] = Ek;
      sm[(2 * S1 + comp) * CPW] = 1.0 / Ek;
    }
  }
  __syncwarp();
  const double RTP = ch.RuP * T;
  const double iRTP = 1.0 / RTP;
  const double* C = sm;
  const double* E = sm + S1 * CPW;
  const double* Ei = sm + 2 * S1 * CPW;
  double* q = sm + 3 * S1 * CPW;
  // reactions: rates of progress
  for (int j = lg; j < ch.R; j += G) {
    const double4 p = ldg4(ch.rxn + j);
    const int4 s = __ldg(ch.rsp + j);
    const double kf = exp(p.x + p.y * lnT - p.z * invT);
    double kr = kf * E[s.z * CPW] * E[s.w * CPW] * Ei[s.x * CPW] * Ei[s.y * CPW];
    kr = kr * (p.w > 0.5 ? RTP : (p.w < -0.5 ? iRTP : 1.0));
    q[j * CPW] = kf * C[s.x * CPW] * C[s.y * CPW] - kr * C[s.z * CPW] * C[s.w * CPW];
  }
  __syncwarp();
  // species production, fixed CSR order (reaction ascending)
#pragma unroll
  for (int t = 0; t < SPL; ++t) {
    const int comp = lg + G * t;
    double w = 0.0;
    if (comp < S) {
      const int b = __ldg(ch.csr_off + comp), en = __ldg(ch.csr_off + comp + 1);
      for (int pp = b; pp < en; ++pp) {
        const int ent = __ldg(ch.csr_ent + pp);
        const double qq = q[(ent >> 1) * CPW];
        w = (ent & 1) ? w + qq : w - qq;
      }
      w = __ldg(sp + 5 * Sp + comp) * w;
    }
    f[t] = w;  // energy (comp == S): de/dt = 0, constant-volume adiabatic
  }
}

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

template <int FK, int G, int SPL>
__device__ __forceinline__ void fast_eval(const ChemDev& ch, const LinDev& lin,
                                          const double (&v)[SPL], double (&f)[SPL], double* sm,
                                          int lg)
{
  if constexpr (FK == FK_CHEM) {
    chem_eval<G, SPL>(ch, v, f, sm, lg);
  } else if constexpr (FK == FK_LINEAR) {
    lin_eval<SPL>(lin, v, f);
  } else {
#pragma unroll
    for (int t = 0; t < SPL; ++t) f[t] = 0.0;  // StateVector(v.size())
  }
}

template <int FK, int G>
__device__ __forceinline__ double* chem_scratch(const ChemDev& ch, int warp, int cw, int lg)
{
  extern __shared__ double smem[];
  if constexpr (FK != FK_CHEM) {
    return nullptr;
  } else {
    constexpr int CPW = 32 / G;
    const int items = 3 * (ch.S + 1) + ch.R;
    double* sm = smem + (size_t)warp * CPW * items + cw;
    if (lg == 0) {  // absent-reactant dummy slot: C = E = Ei = 1
      sm[ch.S * CPW] = 1.0;
      sm[(2 * ch.S + 1) * CPW] = 1.0;
      sm[(3 * ch.S + 2) * CPW] = 1.0;
    }
    return sm;
  }
}

template <int FK, int G, int SPL, int MAXS, int NDEG>
__global__ void __launch_bounds__(128) chain_kernel(const ChainArgs a, const ChemDev ch,
                                                    const LinDev lin)
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
  double* sm = chem_scratch<FK, G>(ch, warp, cw, lg);

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
        fast_eval<FK, G, SPL>(ch, lin, stg, f, sm, lg);
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
                                                       int ncomp, const ChemDev ch,
                                                       const LinDev lin)
{
  constexpr int CPW = 32 / G;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cw = lane % CPW, lg = lane / CPW;
  const size_t warp_cell0 = ((size_t)blockIdx.x * (blockDim.x >> 5) + warp) * CPW;
  if (warp_cell0 >= nc) return;
  const size_t cell = warp_cell0 + cw;
  const bool active = cell < nc;
  double* sm = chem_scratch<FK, G>(ch, warp, cw, lg);
  double v[SPL], f[SPL];
#pragma unroll
  for (int t = 0; t < SPL; ++t) {
    const int comp = lg + G * t;
    v[t] = (active && comp < ncomp) ? yin[(size_t)comp * nc + cell] : 0.0;
  }
  fast_eval<FK, G, SPL>(ch, lin, v, f, sm, lg);
#pragma unroll
  for (int t = 0; t < SPL; ++t) {
    const int comp = lg + G * t;
    if (active && comp < ncomp) fout[(size_t)comp * nc + cell] = f[t];
  }
}

constexpr int kBlock = 128;

template <int FK, int G, int SPL, int MAXS, int NDEG>
cudaError_t run_chain(const ChainArgs& a, const ChemDev& ch, const LinDev& lin, size_t smem,
                      cudaStream_t st)
{
  constexpr int CPB = (kBlock / 32) * (32 / G);
  const size_t blocks = (a.ncell + CPB - 1) / CPB;
  auto k = chain_kernel<FK, G, SPL, MAXS, NDEG>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k<<<(unsigned)blocks, kBlock, smem, st>>>(a, ch, lin);
  return cudaGetLastError();
}

template <int FK, int G, int SPL>
cudaError_t run_rhs(const double* y, double* out, size_t nc, int ncomp, const ChemDev& ch,
                    const LinDev& lin, size_t smem, cudaStream_t st)
{
  constexpr int CPB = (kBlock / 32) * (32 / G);
  const size_t blocks = (nc + CPB - 1) / CPB;
  auto k = fast_rhs_kernel<FK, G, SPL>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k<<<(unsigned)blocks, kBlock, smem, st>>>(y, out, nc, ncomp, ch, lin);
  return cudaGetLastError();
}

}  // namespace

// (G, SPL) layouts instantiated for the chemistry / none plugins
#define MR_CHEM_LAYOUTS(X) X(4, 3) X(8, 2) X(8, 3) X(16, 2) X(16, 4) X(32, 2)

int chain_pick(ChainCfg* cfg, int fast_kind, int ncomp, int S, int R, int s_f, int ndeg)
{
  (void)S;
  (void)R;
  cfg->fast_kind = fast_kind;
  cfg->maxs = s_f <= 4 ? 4 : 6;
  cfg->ndeg = ndeg;
  if (s_f > MR_MAXS || ndeg < 1 || ndeg > MR_MAXDEG) return 1;
  if (fast_kind == FK_LINEAR) {
    cfg->G = 1;
    cfg->SPL = ncomp <= 2 ? 2 : ncomp <= 4 ? 4 : 8;
    return ncomp <= MR_MAXLIN ? 0 : 1;
  }
  // chemistry / none: lanes per cell grow with the component count
  if (ncomp <= 12) { cfg->G = 4; cfg->SPL = 3; }
  else if (ncomp <= 16) { cfg->G = 8; cfg->SPL = 2; }
  else if (ncomp <= 24) { cfg->G = 8; cfg->SPL = 3; }
  else if (ncomp <= 32) { cfg->G = 16; cfg->SPL = 2; }
  else if (ncomp <= 64) { cfg->G = 32; cfg->SPL = 2; }
  else return 1;
  // experiment hook: MR_CHEM_LAYOUT="G,SPL" forces an instantiated layout
  if (const char* env = getenv("MR_CHEM_LAYOUT")) {
    int g = 0, spl = 0;
    if (sscanf(env, "%d,%d", &g, &spl) == 2 && g * spl >= ncomp) {
      bool known = false;
#define MR_KNOWN(GG, SS) known |= (g == GG && spl == SS);
      MR_CHEM_LAYOUTS(MR_KNOWN)
#undef MR_KNOWN
      if (known) { cfg->G = g; cfg->SPL = spl; }
    }
  }
  return 0;
}

size_t chain_smem_bytes(const ChainCfg& cfg, int S, int R, int block)
{
  if (cfg.fast_kind != FK_CHEM) return 0;
  const int warps = block / 32;
  return sizeof(double) * (size_t)warps * (32 / cfg.G) * (size_t)(3 * (S + 1) + R);
}

cudaError_t launch_chain(const ChainCfg& cfg, const ChainArgs& a, const ChemDev& ch,
                         const LinDev& lin, cudaStream_t st)
{
  const size_t smem = chain_smem_bytes(cfg, ch.S, ch.R, kBlock);
#define MR_DISPATCH_MS(FK, GG, SS)                                                       \
  if (cfg.maxs == 4 && cfg.ndeg == 1) return run_chain<FK, GG, SS, 4, 1>(a, ch, lin, smem, st); \
  if (cfg.maxs == 4 && cfg.ndeg == 2) return run_chain<FK, GG, SS, 4, 2>(a, ch, lin, smem, st); \
  if (cfg.maxs == 6 && cfg.ndeg == 1) return run_chain<FK, GG, SS, 6, 1>(a, ch, lin, smem, st); \
  if (cfg.maxs == 6 && cfg.ndeg == 2) return run_chain<FK, GG, SS, 6, 2>(a, ch, lin, smem, st);
#define MR_CHEM_CASE(GG, SS) \
  if (cfg.G == GG && cfg.SPL == SS) { MR_DISPATCH_MS(FK_CHEM, GG, SS) }
#define MR_NONE_CASE(GG, SS) \
  if (cfg.G == GG && cfg.SPL == SS) { MR_DISPATCH_MS(FK_NONE, GG, SS) }
  if (cfg.fast_kind == FK_NONE) { MR_CHEM_LAYOUTS(MR_NONE_CASE) }
  else if (cfg.fast_kind == FK_LINEAR) {
    if (cfg.SPL == 2) { MR_DISPATCH_MS(FK_LINEAR, 1, 2) }
    if (cfg.SPL == 4) { MR_DISPATCH_MS(FK_LINEAR, 1, 4) }
    if (cfg.SPL == 8) { MR_DISPATCH_MS(FK_LINEAR, 1, 8) }
  }
  return cudaErrorInvalidConfiguration;
}

cudaError_t launch_fast_rhs(const ChainCfg& cfg, const double* y, double* out, size_t ncell,
                            int ncomp, const ChemDev& ch, const LinDev& lin, cudaStream_t st)
{
  const size_t smem = chain_smem_bytes(cfg, ch.S, ch.R, kBlock);
#define MR_RHS_CHEM(GG, SS) \
  if (cfg.G == GG && cfg.SPL == SS) return run_rhs<FK_CHEM, GG, SS>(y, out, ncell, ncomp, ch, lin, smem, st);
#define MR_RHS_NONE(GG, SS) \
  if (cfg.G == GG && cfg.SPL == SS) return run_rhs<FK_NONE, GG, SS>(y, out, ncell, ncomp, ch, lin, smem, st);
  if (cfg.fast_kind == FK_NONE) { MR_CHEM_LAYOUTS(MR_RHS_NONE) }
  else if (cfg.fast_kind == FK_LINEAR) {
    if (cfg.SPL == 2) return run_rhs<FK_LINEAR, 1, 2>(y, out, ncell, ncomp, ch, lin, smem, st);
    if (cfg.SPL == 4) return run_rhs<FK_LINEAR, 1, 4>(y, out, ncell, ncomp, ch, lin, smem, st);
    if (cfg.SPL == 8) return run_rhs<FK_LINEAR, 1, 8>(y, out, ncell, ncomp, ch, lin, smem, st);
  }
  return cudaErrorInvalidConfiguration;
}
