// kernels_chem2.cuh -- K1 for the large mechanisms (C4/C5: 53 species, 325
// reactions): the fused fast-IVP chain with the Arrhenius RHS, TWO cells per
// thread.
//
// Same data flow and arithmetic as kernels_chem.cuh (one block owns a set of
// cells, warp w owns components w + NW*t, reactions j = w (mod NW) and, in the
// production phase, its own species; every mechanism index is warp-uniform),
// but a block owns 64 cells and lane l computes cells 2l and 2l+1.  Every
// per-reaction and per-species instruction that is not cell arithmetic --
// the broadcast record loads, the operand address adds, the loop control,
// the production-list walk, the per-eval stage bookkeeping -- is therefore
// issued once per TWO cells, and each shared-memory row access is one
// conflict-free LDS.128/STS.128 (512 B per warp).  The round-1 capture of the
// one-cell kernel showed those instructions at ~45% of all issue slots
// (profiles/r01/chem_chain_c4_256_summary.txt); halving them is the point.
//
// Shared memory (bytes; rows are [64 cells] of doubles, 512 B):
//   C    [S1][64]  C_k = rho Y_k / W_k            (row S: 1.0, absent operand)
//   E    [S1][64]  E'_k = (P/RT) / E_k            (row S: 1.0)
//   D    [S1][64]  D'_k = E_k C_k RT/P            (row S: 1.0)
//   q    [rc][64]  rates of progress of one chunk, then one all-zero row
//   blob           ChemRec[R] + production lists (offsets scaled to 512-B rows)
//   tinf [3][64]   T, ln T, 1/T
//   spc  [S1][5]   double2 per-species constants (as kernels_chem.cuh)
//   part [4][NW][64] energy partial sums, ALIASED onto the E and D tables:
//                  they are dead from the last reaction chunk of one
//                  evaluation to the species phase of the next, and the
//                  species phase rewrites their dummy rows every evaluation.
// The E and D tables are reached from a C-row address with a uniform-register
// offset ([R + UR] addressing), so an operand pair costs one address add.
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels_chem.cuh"

namespace mrchem {

constexpr int kC2Cells = 64;  // cells per block
constexpr unsigned kC2Row = 512u;

__host__ __device__ inline size_t smem2_bytes(int NW, int S1, int rc, int blob_words)
{
  const size_t tables = 3 * (size_t)S1 * kC2Row;
  (void)NW;  // the partial sums live in the E and D tables (4 NW <= 2 S1 rows)
  return tables + (size_t)rc * kC2Row + kC2Row + (size_t)blob_words * 16 + 3 * kC2Row +
         (size_t)S1 * 80;
}

struct Smem2 {
  char* C;         // table bases
  unsigned dE;     // E table - C table (bytes)
  unsigned dD;     // D table - C table
  char* q;
  const char* rec;
  const uint4* ent;
  double* part;    // == E table
  double* tinf;
  const double2* spc;
};

__device__ __forceinline__ Smem2 stage2(char* base, const ChemParams& P, int lane)
{
  const int S1 = P.S + 1;
  Smem2 m;
  m.C = base;
  m.dE = (unsigned)S1 * kC2Row;
  m.dD = 2u * (unsigned)S1 * kC2Row;
  m.part = reinterpret_cast<double*>(base + m.dE);
  m.q = base + 3 * (size_t)S1 * kC2Row;
  char* zero = m.q + (size_t)P.rc * kC2Row;
  uint4* blob = reinterpret_cast<uint4*>(zero + kC2Row);
  m.rec = reinterpret_cast<const char*>(blob);
  m.ent = blob + P.ent_base;
  m.tinf = reinterpret_cast<double*>(blob + P.blob_words);
  double2* spc = reinterpret_cast<double2*>(m.tinf + 3 * kC2Cells);
  m.spc = spc;
  for (int i = threadIdx.x; i < P.S; i += blockDim.x) {
    spc[i * 5 + 0] = make_double2(P.c0[i], P.c1[i]);
    spc[i * 5 + 1] = make_double2(P.c2[i], P.h0[i]);
    spc[i * 5 + 2] = make_double2(P.a[i], P.hb[i]);
    spc[i * 5 + 3] = make_double2(P.s0[i], P.rhoW[i]);
    spc[i * 5 + 4] = make_double2(P.Wrho[i], 0.0);
  }
  for (int i = threadIdx.x; i < P.blob_words; i += blockDim.x) blob[i] = __ldg(P.blob + i);
  if (threadIdx.x < 32) {
    reinterpret_cast<double2*>(zero)[lane] = make_double2(0.0, 0.0);
    *reinterpret_cast<double2*>(m.C + P.S * kC2Row + lane * 16) = make_double2(1.0, 1.0);
  }
  __syncthreads();
  return m;
}

__device__ __forceinline__ double2 lds2(const char* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ void sts2(char* p, double a, double b)
{
  *reinterpret_cast<double2*>(p) = make_double2(a, b);
}

// One chemistry RHS evaluation for the block's 64 cells (all threads call it).
// v[t] / f[t]: this thread's component kk[t] at its two cells (.x, .y).
template <int NW, int SPL>
__device__ __forceinline__ void chem2_block_eval(const ChemParams& P, const Smem2& m, int w,
                                                 int lane, const int (&kk)[SPL],
                                                 const double2 (&v)[SPL], double2 (&f)[SPL])
{
  const int S = P.S;
  const unsigned l16 = (unsigned)lane * 16u;
  // ---- temperature from energy: partial sums of e(T) = E0 + E1 T + E2 T^2
  {
    double2 p0 = make_double2(0.0, 0.0), p1 = p0, p2 = p0, e = p0;
#pragma unroll
    for (int t = 0; t < SPL; ++t) {
      const int k = kk[t];
      if (k < S) {
        const double2 c01 = m.spc[k * 5 + 0];
        const double c2 = m.spc[k * 5 + 1].x;
        p0.x += v[t].x * c01.x;
        p0.y += v[t].y * c01.x;
        p1.x += v[t].x * c01.y;
        p1.y += v[t].y * c01.y;
        p2.x += v[t].x * c2;
        p2.y += v[t].y * c2;
      } else if (k == S) {
        e = v[t];
      }
    }
    char* pr = reinterpret_cast<char*>(m.part) + l16;
    *reinterpret_cast<double2*>(pr + (0 * NW + w) * kC2Row) = p0;
    *reinterpret_cast<double2*>(pr + (1 * NW + w) * kC2Row) = p1;
    *reinterpret_cast<double2*>(pr + (2 * NW + w) * kC2Row) = p2;
    *reinterpret_cast<double2*>(pr + (3 * NW + w) * kC2Row) = e;
  }
  __syncthreads();
  if (w == 0) {
    const char* pr = reinterpret_cast<const char*>(m.part) + l16;
    double2 E0 = make_double2(0.0, 0.0), E1 = E0, E2 = E0, ee = E0;
#pragma unroll 6
    for (int q = 0; q < NW; ++q) {
      const double2 a = lds2(pr + (0 * NW + q) * kC2Row);
      const double2 b = lds2(pr + (1 * NW + q) * kC2Row);
      const double2 c = lds2(pr + (2 * NW + q) * kC2Row);
      const double2 d = lds2(pr + (3 * NW + q) * kC2Row);
      E0.x += a.x; E0.y += a.y;
      E1.x += b.x; E1.y += b.y;
      E2.x += c.x; E2.y += c.y;
      ee.x += d.x; ee.y += d.y;
    }
    const double dex = ee.x - E0.x, dey = ee.y - E0.y;
    const double Tx = (2.0 * dex) / (E1.x + sqrt(E1.x * E1.x + 4.0 * E2.x * dex));
    const double Ty = (2.0 * dey) / (E1.y + sqrt(E1.y * E1.y + 4.0 * E2.y * dey));
    char* ti = reinterpret_cast<char*>(m.tinf) + l16;
    sts2(ti, Tx, Ty);
    sts2(ti + kC2Row, log(Tx), log(Ty));
    sts2(ti + 2 * kC2Row, 1.0 / Tx, 1.0 / Ty);
  }
  __syncthreads();
  const char* ti = reinterpret_cast<const char*>(m.tinf) + l16;
  const double2 T = lds2(ti);
  const double2 lnT = lds2(ti + kC2Row);
  const double2 invT = lds2(ti + 2 * kC2Row);

  // ---- species rows: C_k, (1/E_k)(P/RT), (E_k C_k)(RT/P); dummy rows of
  //      the E and D tables (overwritten by the partial sums) restored
  {
    const double RTPx = P.RuP * T.x, RTPy = P.RuP * T.y;
    const double iRTPx = 1.0 / RTPx, iRTPy = 1.0 / RTPy;
#pragma unroll
    for (int t = 0; t < SPL; ++t) {
      const int k = kk[t];
      if (k < S) {
        const double2 c2h0 = m.spc[k * 5 + 1], ahb = m.spc[k * 5 + 2], s0rw = m.spc[k * 5 + 3];
        const double gx = c2h0.y * invT.x + ahb.x * (1.0 - lnT.x) - ahb.y * T.x - s0rw.x;
        const double gy = c2h0.y * invT.y + ahb.x * (1.0 - lnT.y) - ahb.y * T.y - s0rw.x;
        const double Ex = mr_exp(gx), Ey = mr_exp(gy);
        const double Eix = 1.0 / Ex, Eiy = 1.0 / Ey;
        const double Ckx = s0rw.y * v[t].x, Cky = s0rw.y * v[t].y;
        char* row = m.C + (unsigned)k * kC2Row + l16;
        sts2(row, Ckx, Cky);
        sts2(row + m.dE, Eix * iRTPx, Eiy * iRTPy);
        sts2(row + m.dD, (Ex * Ckx) * RTPx, (Ey * Cky) * RTPy);
      } else if (k == S) {
        char* row = m.C + (unsigned)k * kC2Row + l16;
        sts2(row + m.dE, 1.0, 1.0);
        sts2(row + m.dD, 1.0, 1.0);
      }
    }
  }
  __syncthreads();

  double2 acc[SPL];
#pragma unroll
  for (int t = 0; t < SPL; ++t) acc[t] = make_double2(0.0, 0.0);
  const int R = P.R;
  const char* Cl = m.C + l16;
  const char* ql = m.q + l16;
  const unsigned dE = m.dE, dD = m.dD;
  for (int ch = 0; ch < P.nchunk; ++ch) {
    const int j0 = ch * P.rc;
    const int j1 = min(R, j0 + P.rc);
    // ---- reactions of this chunk (both cells):
    //      q = kf (C_r1 C_r2 - (D'_p1 D'_p2)(E'_r1 E'_r2)), kf = exp(lnA + beta lnT - EaR/T)
    char* qw = m.q + l16 + (unsigned)w * kC2Row;
    const char* rp = m.rec + (j0 + w) * (int)sizeof(ChemRec);
#pragma unroll kRxUnroll
    for (int j = j0 + w; j < j1; j += NW) {
      const double2 ab = *reinterpret_cast<const double2*>(rp);
      const uint4 er = *reinterpret_cast<const uint4*>(rp + 16);
      const uint2 pp = *reinterpret_cast<const uint2*>(rp + 32);
      const double EaR = __hiloint2double((int)er.y, (int)er.x);
      const double kfx = mr_exp(fma(-EaR, invT.x, fma(ab.y, lnT.x, ab.x)));
      const double kfy = mr_exp(fma(-EaR, invT.y, fma(ab.y, lnT.y, ab.x)));
      const char* r1 = Cl + er.z;
      const char* r2 = Cl + er.w;
      const double2 c1 = lds2(r1), c2 = lds2(r2);
      const double2 e1 = lds2(r1 + dE), e2 = lds2(r2 + dE);
      const double2 d1 = lds2(Cl + pp.x + dD), d2 = lds2(Cl + pp.y + dD);
      const double fx = c1.x * c2.x, fy = c1.y * c2.y;
      const double rx = (d1.x * d2.x) * (e1.x * e2.x);
      const double ry = (d1.y * d2.y) * (e1.y * e2.y);
      sts2(qw, kfx * (fx - rx), kfy * (fy - ry));
      qw += NW * kC2Row;
      rp += NW * (int)sizeof(ChemRec);
    }
    __syncthreads();
    // ---- production: w_k += sum_(producing) q - sum_(consuming) q, reaction
    //      ascending, four entries per broadcast LDS.128 (padding -> zero row)
#pragma unroll
    for (int t = 0; t < SPL; ++t) {
      const int k = kk[t];
      if (k < S) {
        const ushort4 L = P.lst[k][ch];
        double2 s_ = acc[t];
        for (int i = 0; i < L.y; ++i) {
          const uint4 e = m.ent[L.x + i];
          const double2 a = lds2(ql + e.x), b = lds2(ql + e.y), c = lds2(ql + e.z), d = lds2(ql + e.w);
          s_.x += a.x; s_.y += a.y;
          s_.x += b.x; s_.y += b.y;
          s_.x += c.x; s_.y += c.y;
          s_.x += d.x; s_.y += d.y;
        }
        for (int i = 0; i < L.w; ++i) {
          const uint4 e = m.ent[L.z + i];
          const double2 a = lds2(ql + e.x), b = lds2(ql + e.y), c = lds2(ql + e.z), d = lds2(ql + e.w);
          s_.x -= a.x; s_.y -= a.y;
          s_.x -= b.x; s_.y -= b.y;
          s_.x -= c.x; s_.y -= c.y;
          s_.x -= d.x; s_.y -= d.y;
        }
        acc[t] = s_;
      }
    }
    if (ch + 1 < P.nchunk) __syncthreads();  // q is overwritten by the next chunk
  }
#pragma unroll
  for (int t = 0; t < SPL; ++t) {
    const int k = kk[t];
    if (k < S) {
      const double wr = m.spc[k * 5 + 4].x;
      f[t] = make_double2(wr * acc[t].x, wr * acc[t].y);
    } else {
      f[t] = make_double2(0.0, 0.0);  // energy: de/dt = 0
    }
  }
}

// global y/fE access of the thread's two cells (cell0 even; either may be
// past the end of the grid)
__device__ __forceinline__ double2 ldg_pair(const double* __restrict__ p, size_t cell0, size_t nc)
{
  double2 r;
  r.x = cell0 < nc ? p[cell0] : 0.0;
  r.y = cell0 + 1 < nc ? p[cell0 + 1] : 0.0;
  return r;
}

// all_finite over this thread's components at its active cells
template <int SPL>
__device__ __forceinline__ bool all_finite2(const double2 (&x)[SPL], const int (&kk)[SPL], int ncomp,
                                            bool act0, bool act1)
{
  bool ok = true;
#pragma unroll
  for (int t = 0; t < SPL; ++t)
    if (kk[t] < ncomp) ok = ok && (!act0 || isfinite(x[t].x)) && (!act1 || isfinite(x[t].y));
  return ok;
}

template <int NW, int SPL, bool SUBDIAG, int MAXS, int NDEG>
__global__ void __launch_bounds__(NW * 32, 1)
    chem2_chain_kernel(const __grid_constant__ ChainArgs a, const __grid_constant__ ChemParams P)
{
  extern __shared__ __align__(16) double smem_raw[];
  const int lane = threadIdx.x & 31;
  const int w = (int)(threadIdx.x >> 5);
  const size_t cell0 = (size_t)blockIdx.x * kC2Cells + 2 * lane;
  const size_t nc = a.ncell;
  const int ncomp = a.ncomp;
  const bool act0 = cell0 < nc, act1 = cell0 + 1 < nc;
  const Smem2 m = stage2(reinterpret_cast<char*>(smem_raw), P, lane);
  int kk[SPL];
#pragma unroll
  for (int t = 0; t < SPL; ++t) kk[t] = w + NW * t;

  double2 y[SPL];
#pragma unroll
  for (int t = 0; t < SPL; ++t) {
    const int k = kk[t];
    y[t] = k < ncomp ? ldg_pair(a.y_in + (size_t)k * nc, cell0, nc) : make_double2(0.0, 0.0);
  }
  // an idle cell (past the grid) never reports a failure
  bool failed = !act0 && !act1;
#define finite2(x) all_finite2<SPL>(x, kk, ncomp, act0, act1)

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
          if (k < ncomp) {
            const double2 x = ldg_pair(fv + (size_t)k * nc, cell0, nc);
            y[t].x = dadd(y[t].x, dmul(cf, x.x));
            y[t].y = dadd(y[t].y, dmul(cf, x.y));
          }
        }
      }
      if (!failed && !finite2(y)) {
        atomicMin(a.fail, mr_fail_key(st.mri_stage, 0, 0));
        failed = true;
      }
      continue;
    }

    // FastIvp: forcing coefficients r_k = sum_j (omega[k][i][j]/dc) fE_j
    double2 rc[NDEG][SPL];
#pragma unroll
    for (int k = 0; k < NDEG; ++k)
#pragma unroll
      for (int t = 0; t < SPL; ++t) rc[k][t] = make_double2(0.0, 0.0);
    for (int r = 0; r < st.nref; ++r) {
      const double* __restrict__ fv = a.fE[st.ref_slot[r]];
#pragma unroll
      for (int t = 0; t < SPL; ++t) {
        const int kc = kk[t];
        const double2 x = kc < ncomp ? ldg_pair(fv + (size_t)kc * nc, cell0, nc) : make_double2(0.0, 0.0);
#pragma unroll
        for (int k = 0; k < NDEG; ++k) {
          const double cf = st.coef[k][r];
          if (cf != 0.0) {
            rc[k][t].x = dadd(rc[k][t].x, dmul(cf, x.x));
            rc[k][t].y = dadd(rc[k][t].y, dmul(cf, x.y));
          }
        }
      }
    }

    const double h = st.h_sub;
    const int sf = a.tab.s;
    for (int sub = 0; sub < st.n_sub; ++sub) {
      const double t0 = dadd(st.t_start, dmul((double)sub, h));
      constexpr int NPRE = SUBDIAG ? 1 : MAXS;
      double2 pre[NPRE][SPL];
      double2 out[SPL];
#pragma unroll
      for (int i = 0; i < NPRE; ++i)
#pragma unroll
        for (int t = 0; t < SPL; ++t) pre[i][t] = y[t];
#pragma unroll
      for (int t = 0; t < SPL; ++t) out[t] = y[t];

      for (int j = 0; j < sf; ++j) {
        double2 stg[SPL];
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
        if (!failed && !finite2(stg)) {
          atomicMin(a.fail, mr_fail_key(st.mri_stage, sub, j));
          failed = true;
        }
        const double theta = dadd(t0, dmul(a.tab.c[j], h));
        const double tau = __ddiv_rn(dadd(theta, -st.t_start), st.span);
        double2 f[SPL];
        chem2_block_eval<NW, SPL>(P, m, w, lane, kk, stg, f);
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
          double frx = rc[NDEG - 1][t].x, fry = rc[NDEG - 1][t].y;
#pragma unroll
          for (int k = NDEG - 2; k >= 0; --k) {
            frx = dadd(dmul(frx, tau), rc[k][t].x);
            fry = dadd(dmul(fry, tau), rc[k][t].y);
          }
          const double kjx = dadd(f[t].x, frx), kjy = dadd(f[t].y, fry);
          if constexpr (SUBDIAG) {
            // stage_{j+1} = y + (h A[j+1][j]) k_j, the only nonzero entry
            if (j + 1 < sf) {
              pre[0][t].x = useA ? dadd(y[t].x, dmul(hA_next, kjx)) : y[t].x;
              pre[0][t].y = useA ? dadd(y[t].y, dmul(hA_next, kjy)) : y[t].y;
            }
          } else {
#pragma unroll
            for (int i = 1; i < NPRE; ++i) {
              if (i > j && i < sf) {
                const double Aij = a.tab.A[i][j];
                if (Aij != 0.0) {
                  const double hA = dmul(h, Aij);
                  pre[i][t].x = dadd(pre[i][t].x, dmul(hA, kjx));
                  pre[i][t].y = dadd(pre[i][t].y, dmul(hA, kjy));
                }
              }
            }
          }
          if (use_b) {
            out[t].x = dadd(out[t].x, dmul(hb, kjx));
            out[t].y = dadd(out[t].y, dmul(hb, kjy));
          }
        }
      }
      if (!failed && !finite2(out)) {
        atomicMin(a.fail, mr_fail_key(st.mri_stage, sub, sf));
        failed = true;
      }
#pragma unroll
      for (int t = 0; t < SPL; ++t) y[t] = out[t];
    }
  }

#pragma unroll
  for (int t = 0; t < SPL; ++t) {
    const int k = kk[t];
    if (k < ncomp) {
      double* o = a.y_out + (size_t)k * nc;
      if (act0) o[cell0] = y[t].x;
      if (act1) o[cell0 + 1] = y[t].y;
    }
  }
#undef finite2
}

template <int NW, int SPL>
__global__ void __launch_bounds__(NW * 32, 1) chem2_rhs_kernel(const double* __restrict__ yin,
                                                              double* __restrict__ fout, size_t nc,
                                                              int ncomp,
                                                              const __grid_constant__ ChemParams P)
{
  extern __shared__ __align__(16) double smem_raw[];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const size_t cell0 = (size_t)blockIdx.x * kC2Cells + 2 * lane;
  const Smem2 m = stage2(reinterpret_cast<char*>(smem_raw), P, lane);
  int kk[SPL];
#pragma unroll
  for (int t = 0; t < SPL; ++t) kk[t] = w + NW * t;
  double2 v[SPL], f[SPL];
#pragma unroll
  for (int t = 0; t < SPL; ++t)
    v[t] = kk[t] < ncomp ? ldg_pair(yin + (size_t)kk[t] * nc, cell0, nc) : make_double2(0.0, 0.0);
  chem2_block_eval<NW, SPL>(P, m, w, lane, kk, v, f);
#pragma unroll
  for (int t = 0; t < SPL; ++t) {
    const int k = kk[t];
    if (k < ncomp) {
      if (cell0 < nc) fout[(size_t)k * nc + cell0] = f[t].x;
      if (cell0 + 1 < nc) fout[(size_t)k * nc + cell0 + 1] = f[t].y;
    }
  }
}

template <int NW, int SPL, bool SUBDIAG, int MAXS, int NDEG>
cudaError_t run_chem2_chain(const ChainArgs& a, const ChemParams& P, cudaStream_t st)
{
  const size_t smem = smem2_bytes(NW, P.S + 1, P.rc, P.blob_words);
  auto k = chem2_chain_kernel<NW, SPL, SUBDIAG, MAXS, NDEG>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const size_t blocks = (a.ncell + kC2Cells - 1) / kC2Cells;
  k<<<(unsigned)blocks, NW * 32, smem, st>>>(a, P);
  return cudaGetLastError();
}

template <int NW, int SPL>
cudaError_t run_chem2_rhs(const double* y, double* out, size_t nc, int ncomp, const ChemParams& P,
                          cudaStream_t st)
{
  const size_t smem = smem2_bytes(NW, P.S + 1, P.rc, P.blob_words);
  auto k = chem2_rhs_kernel<NW, SPL>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k<<<(unsigned)((nc + kC2Cells - 1) / kC2Cells), NW * 32, smem, st>>>(y, out, nc, ncomp, P);
  return cudaGetLastError();
}

}  // namespace mrchem
