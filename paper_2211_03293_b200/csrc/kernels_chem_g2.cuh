// kernels_chem_g2.cuh -- K1 for the large mechanisms (C4/C5: 53 species,
// 325 reactions): two cell groups per 1024-thread block that take turns on
// ONE rate-of-progress buffer.
//
// The single-group kernel (kernels_chem.cuh) runs every RHS evaluation as
// barrier-separated phases: energy partial sums -> one warp solves T ->
// species rows -> reactions -> production -> RK bookkeeping.  The reaction
// and production phases (~68% of the time) keep the shared-memory pipe ~85%
// busy; the other phases are latency-bound and leave the SM mostly idle
// (DESIGN.md section 4).  Here a block holds two independent groups of 32
// cells (16 warps x 4 components each).  The full rate buffer q[R][32] is
// shared and handed back and forth with named barriers, so the groups are
// forced half a cycle apart: while group A runs reactions + production, group
// B runs its serial phases (temperature, species rows, RK update) and waits
// for the buffer; then they swap.  Only one copy of the 83 KB buffer is
// needed, which is what lets both groups keep the whole mechanism resident
// (an earlier two-group variant gave each group its own buffer, had to chunk
// it, and let the groups run free -- slower, DESIGN.md experiment (r)).
//
//   bar 1+g  group g internal (512 threads)
//   bar 3+g  "rate buffer free for group g": group g syncs (its species rows
//            are complete), the other group arrives after its production
//
// The forcing-polynomial coefficients of a FastIvp stage are written once to
// a per-cell scratch (a.rcs, [ndeg][ncomp][ncell]) and read back per
// evaluation -- the wave's working set stays in L2 and the reads sit in the
// latency-tolerant RK phase -- which keeps the RK state of 4 components per
// thread inside the 64-register budget of a 1024-thread block.
//
// Arithmetic per cell is that of kernels_chem.cuh (same rows, records, exp,
// production order); only the association of the energy partial sums
// differs (16 warps x 4 slots instead of 32 x 2).
#pragma once
#include "kernels_chem.cuh"

namespace mrchem {

#ifndef MR_G2_UNROLL
#define MR_G2_UNROLL 2
#endif
constexpr int kG2Unroll = MR_G2_UNROLL;

__device__ __forceinline__ void nbar_sync(int id, int n)
{
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void nbar_arrive(int id, int n)
{
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// shared memory, in this order:
//   q    double  [rc][32]   rates of progress (shared by both groups)
//   zero double  [32]       padding target of the production lists
//   blob uint4   [words]    ChemRec[R] + production lists
//   spc  double2 [S1][5]    per-species constants
//   per group g: CE double2 [S1][32], D double [S1][32], tinf double [3][32]
//   (the energy partials part[4][NW][32] alias the group's CE rows: they are
//    written after the group's production, when the rows are dead, and read
//    before the species phase rewrites them)
__host__ __device__ inline size_t g2_group_bytes(int S1) { return (size_t)S1 * 768 + 3 * 256; }
__host__ __device__ inline size_t g2_smem_bytes(int S1, int rc, int blob_words)
{
  return (size_t)rc * 256 + 256 + (size_t)blob_words * 16 + (size_t)S1 * 80 + 2 * g2_group_bytes(S1);
}

__device__ __forceinline__ Smem stage_g2(char* base, const ChemParams& P, int g, int c, int w)
{
  const int S1 = P.S + 1;
  char* q = base;
  char* zero = q + P.rc * 256;
  uint4* blob = reinterpret_cast<uint4*>(zero + 256);
  double2* spc = reinterpret_cast<double2*>(blob + P.blob_words);
  char* grp = reinterpret_cast<char*>(spc + S1 * 5) + (size_t)g * g2_group_bytes(S1);
  Smem m;
  m.q = q;
  m.rec = reinterpret_cast<const char*>(blob);
  m.ent = blob + P.ent_base;
  m.spc = spc;
  m.CE = grp;
  m.D = grp + S1 * 512;
  m.tinf = reinterpret_cast<double*>(m.D + S1 * 256);
  m.part = reinterpret_cast<double*>(m.CE);
  for (int i = threadIdx.x; i < P.S; i += blockDim.x) {
    spc[i * 5 + 0] = make_double2(P.c0[i], P.c1[i]);
    spc[i * 5 + 1] = make_double2(P.c2[i], P.h0[i]);
    spc[i * 5 + 2] = make_double2(P.a[i], P.hb[i]);
    spc[i * 5 + 3] = make_double2(P.s0[i], P.rhoW[i]);
    spc[i * 5 + 4] = make_double2(P.Wrho[i], 0.0);
  }
  for (int i = threadIdx.x; i < P.blob_words; i += blockDim.x) blob[i] = __ldg(P.blob + i);
  if (w == 0) {
    if (g == 0) reinterpret_cast<double*>(zero)[c] = 0.0;
    // absent-species dummy rows: C = E' = D' = 1 (never overwritten: the
    // energy partials alias rows < 4*NW*32*8 / 512 only)
    *reinterpret_cast<double2*>(m.CE + P.S * 512 + c * 16) = make_double2(1.0, 1.0);
    *reinterpret_cast<double*>(m.D + P.S * 256 + c * 8) = 1.0;
  }
  __syncthreads();
  return m;
}

// One RHS evaluation for group g's 32 cells (all 512 threads of the group).
template <int NW, int SPL>
__device__ __forceinline__ void chem_group_eval(const ChemParams& P, const Smem& m, int g, int w,
                                                int c, const int (&kk)[SPL],
                                                const double (&v)[SPL], double (&f)[SPL])
{
  constexpr int GT = NW * 32;  // threads per group
  const int S = P.S;
  const unsigned lane8 = (unsigned)c * 8u, lane16 = (unsigned)c * 16u;
  {
    double p0 = 0.0, p1 = 0.0, p2 = 0.0, e = 0.0;
#pragma unroll
    for (int t = 0; t < SPL; ++t) {
      const int k = kk[t];
      if (k < S) {
        const double2 c01 = m.spc[k * 5 + 0];
        p0 += v[t] * c01.x;
        p1 += v[t] * c01.y;
        p2 += v[t] * m.spc[k * 5 + 1].x;
      } else if (k == S) {
        e = v[t];
      }
    }
    m.part[(0 * NW + w) * 32 + c] = p0;
    m.part[(1 * NW + w) * 32 + c] = p1;
    m.part[(2 * NW + w) * 32 + c] = p2;
    m.part[(3 * NW + w) * 32 + c] = e;
  }
  nbar_sync(1 + g, GT);
  if (w == 0) {
    double E0 = 0.0, E1 = 0.0, E2 = 0.0, ee = 0.0;
#pragma unroll
    for (int q = 0; q < NW; ++q) {
      E0 += m.part[(0 * NW + q) * 32 + c];
      E1 += m.part[(1 * NW + q) * 32 + c];
      E2 += m.part[(2 * NW + q) * 32 + c];
      ee += m.part[(3 * NW + q) * 32 + c];
    }
    const double de = ee - E0;
    const double T = (2.0 * de) / (E1 + sqrt(E1 * E1 + 4.0 * E2 * de));
    m.tinf[0 * 32 + c] = T;
    m.tinf[1 * 32 + c] = log(T);
    m.tinf[2 * 32 + c] = 1.0 / T;
  }
  nbar_sync(1 + g, GT);
  const double T = m.tinf[0 * 32 + c];
  const double lnT = m.tinf[1 * 32 + c];
  const double invT = m.tinf[2 * 32 + c];
  {
    const double RTP = P.RuP * T;
    const double iRTP = 1.0 / RTP;
#pragma unroll
    for (int t = 0; t < SPL; ++t) {
      const int k = kk[t];
      if (k < S) {
        const double2 c2h0 = m.spc[k * 5 + 1], ahb = m.spc[k * 5 + 2], s0rw = m.spc[k * 5 + 3];
        const double gk = c2h0.y * invT + ahb.x * (1.0 - lnT) - ahb.y * T - s0rw.x;
        const double E = mr_exp(gk);
        const double Ei = 1.0 / E;
        const double Ck = s0rw.y * v[t];
        *reinterpret_cast<double2*>(m.CE + k * 512 + lane16) = make_double2(Ck, Ei * iRTP);
        *reinterpret_cast<double*>(m.D + k * 256 + lane8) = (E * Ck) * RTP;
      }
    }
  }
  // species rows complete AND the other group has released the rate buffer
  nbar_sync(3 + g, 2 * GT);

  const int R = P.R;
  const char* CEl = m.CE + lane16;
  const char* Dl = m.D + lane8;
  const char* ql = m.q + lane8;
  {
    char* qw = m.q + lane8 + (unsigned)w * 256u;
    const char* rp = m.rec + w * (int)sizeof(ChemRec);
#pragma unroll kG2Unroll
    for (int j = w; j < R; j += NW) {
      const double2 ab = *reinterpret_cast<const double2*>(rp);
      const uint4 er = *reinterpret_cast<const uint4*>(rp + 16);
      const uint2 pp = *reinterpret_cast<const uint2*>(rp + 32);
      const double EaR = __hiloint2double((int)er.y, (int)er.x);
      const double kf = mr_exp(fma(-EaR, invT, fma(ab.y, lnT, ab.x)));
      const double2 a1 = at<double2>(CEl, er.z);
      const double2 a2 = at<double2>(CEl, er.w);
      const double d1 = at<double>(Dl, pp.x);
      const double d2 = at<double>(Dl, pp.y);
      const double fwd = a1.x * a2.x;
      const double rev = (d1 * d2) * (a1.y * a2.y);
      *reinterpret_cast<double*>(qw) = kf * (fwd - rev);
      qw += NW * 256;
      rp += NW * (int)sizeof(ChemRec);
    }
  }
  nbar_sync(1 + g, GT);
  double acc[SPL];
#pragma unroll
  for (int t = 0; t < SPL; ++t) {
    const int k = kk[t];
    double s_ = 0.0;
    if (k < S) {
      const ushort4 L = P.lst[k][0];
      for (int i = 0; i < L.y; ++i) {
        const uint4 e = m.ent[L.x + i];
        s_ += at<double>(ql, e.x);
        s_ += at<double>(ql, e.y);
        s_ += at<double>(ql, e.z);
        s_ += at<double>(ql, e.w);
      }
      for (int i = 0; i < L.w; ++i) {
        const uint4 e = m.ent[L.z + i];
        s_ -= at<double>(ql, e.x);
        s_ -= at<double>(ql, e.y);
        s_ -= at<double>(ql, e.z);
        s_ -= at<double>(ql, e.w);
      }
    }
    acc[t] = s_;
  }
  // hand the rate buffer to the other group
  nbar_arrive(3 + (1 - g), 2 * GT);
#pragma unroll
  for (int t = 0; t < SPL; ++t) {
    const int k = kk[t];
    f[t] = k < S ? m.spc[k * 5 + 4].x * acc[t] : 0.0;  // energy: de/dt = 0
  }
}

template <int NW, int SPL, bool SUBDIAG, int MAXS, int NDEG>
__global__ void __launch_bounds__(2 * NW * 32, 1)
    chem_chain_g2_kernel(const __grid_constant__ ChainArgs a, const __grid_constant__ ChemParams P)
{
  extern __shared__ __align__(16) double smem_raw[];
  const int c = threadIdx.x & 31;
  const int g = (int)(threadIdx.x >> 5) / NW;
  const int w = (int)(threadIdx.x >> 5) - g * NW;
  const size_t cell = ((size_t)blockIdx.x * 2 + g) * 32 + c;
  const bool active = cell < a.ncell;
  const size_t nc = a.ncell;
  const int ncomp = a.ncomp;
  const Smem m = stage_g2(reinterpret_cast<char*>(smem_raw), P, g, c, w);
  // the rate buffer starts out free for group 0
  if (g == 1) nbar_arrive(3, 2 * NW * 32);
  int kk[SPL];
#pragma unroll
  for (int t = 0; t < SPL; ++t) kk[t] = P.perm[w + NW * t];

  double y[SPL];
#pragma unroll
  for (int t = 0; t < SPL; ++t) {
    const int k = kk[t];
    y[t] = (active && k < ncomp) ? a.y_in[(size_t)k * nc + cell] : 0.0;
  }
  bool failed = !active;

  for (int si = 0; si < a.nst; ++si) {
    const ChainStageDev& st = a.st[si];
    if (st.kind != 0) {  // ExplicitUpdate: Y += sum_j (H wbar_ij) fE_j
      for (int r = 0; r < st.nref; ++r) {
        const double cf = st.coef[0][r];
        if (cf == 0.0) continue;
        const double* __restrict__ fv = a.fE[st.ref_slot[r]];
#pragma unroll
        for (int t = 0; t < SPL; ++t) {
          const int k = kk[t];
          if (active && k < ncomp) y[t] = dadd(y[t], dmul(cf, fv[(size_t)k * nc + cell]));
        }
      }
      if (!failed) {
        bool bad = false;
#pragma unroll
        for (int t = 0; t < SPL; ++t)
          if (kk[t] < ncomp && !isfinite(y[t])) bad = true;
        if (bad) {
          atomicMin(a.fail, mr_fail_key(st.mri_stage, 0, 0));
          failed = true;
        }
      }
      continue;
    }

    // FastIvp: forcing coefficients r_k = sum_j (omega[k][i][j]/dc) fE_j,
    // summed in build_forcing's order and parked in the per-cell scratch
#pragma unroll
    for (int t = 0; t < SPL; ++t) {
      const int kc = kk[t];
      if (!(active && kc < ncomp)) continue;
      double rcv[NDEG];
#pragma unroll
      for (int k = 0; k < NDEG; ++k) rcv[k] = 0.0;
      for (int r = 0; r < st.nref; ++r) {
        const double x = a.fE[st.ref_slot[r]][(size_t)kc * nc + cell];
#pragma unroll
        for (int k = 0; k < NDEG; ++k) {
          const double cf = st.coef[k][r];
          if (cf != 0.0) rcv[k] = dadd(rcv[k], dmul(cf, x));
        }
      }
#pragma unroll
      for (int k = 0; k < NDEG; ++k) a.rcs[((size_t)k * ncomp + kc) * nc + cell] = rcv[k];
    }

    const double h = st.h_sub;
    const int sf = a.tab.s;
    for (int sub = 0; sub < st.n_sub; ++sub) {
      const double t0 = dadd(st.t_start, dmul((double)sub, h));
      constexpr int NPRE = SUBDIAG ? 1 : MAXS;
      double pre[NPRE][SPL];
      double out[SPL];
#pragma unroll
      for (int i = 0; i < NPRE; ++i)
#pragma unroll
        for (int t = 0; t < SPL; ++t) pre[i][t] = y[t];
#pragma unroll
      for (int t = 0; t < SPL; ++t) out[t] = y[t];

      for (int j = 0; j < sf; ++j) {
        double stg[SPL];
#pragma unroll
        for (int t = 0; t < SPL; ++t) stg[t] = pre[0][t];
        if constexpr (!SUBDIAG) {
#pragma unroll
          for (int i = 1; i < NPRE; ++i)
            if (i == j) {
#pragma unroll
              for (int t = 0; t < SPL; ++t) stg[t] = pre[i][t];
            }
        }
        if (!failed) {
          bool bad = false;
#pragma unroll
          for (int t = 0; t < SPL; ++t)
            if (kk[t] < ncomp && !isfinite(stg[t])) bad = true;
          if (bad) {
            atomicMin(a.fail, mr_fail_key(st.mri_stage, sub, j));
            failed = true;
          }
        }
        const double theta = dadd(t0, dmul(a.tab.c[j], h));
        const double tau = __ddiv_rn(dadd(theta, -st.t_start), st.span);
        double f[SPL];
        chem_group_eval<NW, SPL>(P, m, g, w, c, kk, stg, f);
        const double hb = dmul(h, a.tab.b[j]);
        const bool use_b = a.tab.b[j] != 0.0;
        double hA_next = 0.0;
        bool useA = false;
        if constexpr (SUBDIAG) {
          useA = j + 1 < sf && a.tab.A[j + 1][j] != 0.0;
          if (useA) hA_next = dmul(h, a.tab.A[j + 1][j]);
        }
#pragma unroll
        for (int t = 0; t < SPL; ++t) {
          const int kc = kk[t];
          double fr = 0.0;
          if (active && kc < ncomp) {
            fr = a.rcs[((size_t)(NDEG - 1) * ncomp + kc) * nc + cell];
#pragma unroll
            for (int k = NDEG - 2; k >= 0; --k)
              fr = dadd(dmul(fr, tau), a.rcs[((size_t)k * ncomp + kc) * nc + cell]);
          }
          const double kj = dadd(f[t], fr);
          if constexpr (SUBDIAG) {
            if (j + 1 < sf) pre[0][t] = useA ? dadd(y[t], dmul(hA_next, kj)) : y[t];
          } else {
#pragma unroll
            for (int i = 1; i < NPRE; ++i) {
              if (i > j && i < sf) {
                const double Aij = a.tab.A[i][j];
                if (Aij != 0.0) pre[i][t] = dadd(pre[i][t], dmul(dmul(h, Aij), kj));
              }
            }
          }
          if (use_b) out[t] = dadd(out[t], dmul(hb, kj));
        }
      }
      if (!failed) {
        bool bad = false;
#pragma unroll
        for (int t = 0; t < SPL; ++t)
          if (kk[t] < ncomp && !isfinite(out[t])) bad = true;
        if (bad) {
          atomicMin(a.fail, mr_fail_key(st.mri_stage, sub, sf));
          failed = true;
        }
      }
#pragma unroll
      for (int t = 0; t < SPL; ++t) y[t] = out[t];
    }
  }
  // consume group 1's last release so every barrier generation completes
  if (g == 0) nbar_sync(3, 2 * NW * 32);

#pragma unroll
  for (int t = 0; t < SPL; ++t) {
    const int k = kk[t];
    if (active && k < ncomp) a.y_out[(size_t)k * nc + cell] = y[t];
  }
}

template <int NW, int SPL, bool SUBDIAG, int MAXS, int NDEG>
cudaError_t run_chem_chain_g2(const ChainArgs& a, const ChemParams& P, cudaStream_t st)
{
  const size_t smem = g2_smem_bytes(P.S + 1, P.rc, P.blob_words);
  auto k = chem_chain_g2_kernel<NW, SPL, SUBDIAG, MAXS, NDEG>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const size_t blocks = (a.ncell + 63) / 64;
  k<<<(unsigned)blocks, 2 * NW * 32, smem, st>>>(a, P);
  return cudaGetLastError();
}

}  // namespace mrchem
