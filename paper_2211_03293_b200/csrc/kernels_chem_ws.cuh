// kernels_chem_ws.cuh -- K1 for the large mechanisms (C4/C5: 53 species,
// 325 reactions): a warp-specialised chemistry chain over two cell groups.
//
// The single-group kernel (kernels_chem.cuh) runs each RHS evaluation as
// block-barrier phases: energy partial sums -> one warp solves T -> species
// rows -> reactions -> production -> RK update.  The temperature and species
// phases are latency-bound (one warp, or one exp per thread) and ~20% of the
// time (a build that skips them runs 572 vs 687 ms per C4 step at 128^3,
// DESIGN.md section 4).  Here a 1024-thread block holds two groups of 32
// cells (A, B) and its warps specialise:
//
//   * NW = 32 - NS WORKER warps run reactions, production and the RK update
//     of one group while the serial warps prepare the other one.  Worker w
//     owns the components perm[w + NW t] (t < 2) of both groups, the
//     reactions j = w (mod NW), and writes the stage values of the next
//     evaluation into the group's D rows;
//   * the NS SERIAL warps (lane = cell) read those rows, sum e(T) = E0 +
//     E1 T + E2 T^2 in species order, solve T, and write the species rows
//     (C, E') and D' that the reactions gather (species split among them).
//
// Workers:  ... | react A  prod A  RK A -> rows A' | react B  prod B  RK B -> rows B' | react A' ...
// Serial:   ... |      species rows B (from B)      |      species rows A'            | ...
//
//   bar 1+X  "stage values of group X written": workers arrive, serial warps sync
//   bar 3+X  "species rows of group X ready": serial warps arrive, workers sync
//            (all workers sync, so every worker has also finished the
//             previous group's production: the rate buffer is free)
//   bar 5    workers only: every rate of progress written
//   bar 6    serial warps only: the stage values are read before the species
//            rows overwrite them (NS > 1)
//
// One rate buffer q[R][32] serves both groups (they take turns), so both
// keep the whole mechanism resident.  The forcing coefficients of a FastIvp
// stage go to a per-cell scratch (a.rcs, [ndeg][ncomp][ncell], written once
// per stage, read per evaluation from L2) to keep the RK state of two
// groups x two components inside the 64 registers of a 1024-thread block.
//
// Arithmetic per cell is that of kernels_chem.cuh (rows, records, exp,
// production order); e(T)'s sums run in species order.
#pragma once
#include "kernels_chem.cuh"

namespace mrchem {

#ifndef MR_WS_SERIAL
#define MR_WS_SERIAL 2
#endif
constexpr int kWsSerial = MR_WS_SERIAL;      // serial warps (the last ones of the block)
constexpr int kWsWorkers = 32 - kWsSerial;   // worker warps

__device__ __forceinline__ void nbar_sync(int id, int n)
{
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void nbar_arrive(int id, int n)
{
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// shared memory, in this order:
//   q    double  [rc][32]   rates of progress (the groups take turns)
//   zero double  [32]       padding target of the production lists
//   blob uint4   [words]    ChemRec[R] + production lists
//   spc  double2 [S1][5]    per-species constants
//   per group X: CE double2 [S1][32] (C, E'), D double [S1][32] (stage
//   values Y_k from the workers, then D' from the serial warp), e [32]
//   (energy stage value), tinf [3][32] (T, ln T, 1/T)
__host__ __device__ inline size_t ws_group_bytes(int S1) { return (size_t)S1 * 768 + 256 + 768; }
__host__ __device__ inline size_t ws_smem_bytes(int S1, int rc, int blob_words)
{
  return (size_t)rc * 256 + 256 + (size_t)blob_words * 16 + (size_t)S1 * 80 + 2 * ws_group_bytes(S1);
}

struct WsSmem {
  char* q;
  const char* rec;
  const uint4* ent;
  const double2* spc;
  char* CE[2];
  char* D[2];
  double* e[2];
  double* tinf[2];
};

__device__ __forceinline__ WsSmem stage_ws(char* base, const ChemParams& P, int c, int wid)
{
  const int S1 = P.S + 1;
  WsSmem m;
  m.q = base;
  char* zero = m.q + P.rc * 256;
  uint4* blob = reinterpret_cast<uint4*>(zero + 256);
  double2* spc = reinterpret_cast<double2*>(blob + P.blob_words);
  m.rec = reinterpret_cast<const char*>(blob);
  m.ent = blob + P.ent_base;
  m.spc = spc;
  char* grp = reinterpret_cast<char*>(spc + S1 * 5);
  for (int X = 0; X < 2; ++X) {
    m.CE[X] = grp;
    m.D[X] = grp + S1 * 512;
    m.e[X] = reinterpret_cast<double*>(m.D[X] + S1 * 256);
    m.tinf[X] = m.e[X] + 32;
    grp += ws_group_bytes(S1);
  }
  for (int i = threadIdx.x; i < P.S; i += blockDim.x) {
    spc[i * 5 + 0] = make_double2(P.c0[i], P.c1[i]);
    spc[i * 5 + 1] = make_double2(P.c2[i], P.h0[i]);
    spc[i * 5 + 2] = make_double2(P.a[i], P.hb[i]);
    spc[i * 5 + 3] = make_double2(P.s0[i], P.rhoW[i]);
    spc[i * 5 + 4] = make_double2(P.Wrho[i], 0.0);
  }
  for (int i = threadIdx.x; i < P.blob_words; i += blockDim.x) blob[i] = __ldg(P.blob + i);
  if (wid == 0) {
    reinterpret_cast<double*>(zero)[c] = 0.0;
    // absent-species dummy rows: C = E' = D' = 1 (row S: never written)
    for (int X = 0; X < 2; ++X) {
      *reinterpret_cast<double2*>(m.CE[X] + P.S * 512 + c * 16) = make_double2(1.0, 1.0);
      *reinterpret_cast<double*>(m.D[X] + P.S * 256 + c * 8) = 1.0;
    }
  }
  __syncthreads();
  return m;
}

// The serial warps' part of one evaluation of group X (lane = cell): every
// serial warp sums e(T) and solves T (redundantly: no barrier among them),
// serial warp sw then writes the species rows k = sw (mod kWsSerial), four
// species at a time (loads first, four independent exp / reciprocal chains).
__device__ __forceinline__ void ws_species_rows(const ChemParams& P, const WsSmem& m, int X, int c,
                                                int sw)
{
  const int S = P.S;
  const unsigned lane8 = (unsigned)c * 8u, lane16 = (unsigned)c * 16u;
  const char* Dl = m.D[X] + lane8;
  double E0 = 0.0, E1 = 0.0, E2 = 0.0;
#pragma unroll 4
  for (int k = 0; k < S; ++k) {
    const double v = at<double>(Dl, (unsigned)k * 256u);
    const double2 c01 = m.spc[k * 5 + 0];
    E0 += v * c01.x;
    E1 += v * c01.y;
    E2 += v * m.spc[k * 5 + 1].x;
  }
  // every serial warp has read the stage values before any overwrites them
  if constexpr (kWsSerial > 1) nbar_sync(6, kWsSerial * 32);
  const double de = m.e[X][c] - E0;
  const double T = (2.0 * de) / (E1 + sqrt(E1 * E1 + 4.0 * E2 * de));
  const double lnT = log(T);
  const double invT = 1.0 / T;
  if (sw == 0) {
    m.tinf[X][0 * 32 + c] = T;
    m.tinf[X][1 * 32 + c] = lnT;
    m.tinf[X][2 * 32 + c] = invT;
  }
  const double RTP = P.RuP * T;
  const double iRTP = 1.0 / RTP;
  const double omlnT = 1.0 - lnT;
  constexpr int B = 4;
  for (int k0 = sw; k0 < S; k0 += B * kWsSerial) {
    double Y[B], E[B];
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int k = min(k0 + u * kWsSerial, S - 1);
      Y[u] = at<double>(Dl, (unsigned)k * 256u);
    }
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int k = min(k0 + u * kWsSerial, S - 1);
      const double2 c2h0 = m.spc[k * 5 + 1], ahb = m.spc[k * 5 + 2];
      const double g = c2h0.y * invT + ahb.x * omlnT - ahb.y * T - m.spc[k * 5 + 3].x;
      E[u] = mr_exp(g);
    }
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int k = k0 + u * kWsSerial;
      if (k < S) {
        const double Ck = m.spc[k * 5 + 3].y * Y[u];
        const double Ei = 1.0 / E[u];
        *reinterpret_cast<double2*>(m.CE[X] + k * 512 + lane16) = make_double2(Ck, Ei * iRTP);
        *reinterpret_cast<double*>(m.D[X] + k * 256 + lane8) = (E[u] * Ck) * RTP;
      }
    }
  }
}

// Workers: reactions and production of group X (all workers), returns the
// production rates of the thread's two components in mass-fraction units.
template <int SPL>
__device__ __forceinline__ void ws_react_produce(const ChemParams& P, const WsSmem& m, int X, int w,
                                                 int c, const int (&kk)[SPL], double (&f)[SPL])
{
  constexpr int NW = kWsWorkers;
  const int S = P.S;
  const unsigned lane8 = (unsigned)c * 8u, lane16 = (unsigned)c * 16u;
  nbar_sync(3 + X, 32 * 32);  // species rows of X ready; rate buffer free
  const double lnT = m.tinf[X][1 * 32 + c];
  const double invT = m.tinf[X][2 * 32 + c];
  const int R = P.R;
  const char* CEl = m.CE[X] + lane16;
  const char* Dl = m.D[X] + lane8;
  const char* ql = m.q + lane8;
  {
    char* qw = m.q + lane8 + (unsigned)w * 256u;
    const char* rp = m.rec + w * (int)sizeof(ChemRec);
#pragma unroll kRxUnroll
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
  nbar_sync(5, NW * 32);  // every rate of progress of X written
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
      s_ *= m.spc[k * 5 + 4].x;
    }
    f[t] = s_;  // energy (k == S) and idle slots: 0
  }
}

// Position of one RHS evaluation in the chain: stage, substep, inner stage.
struct WsPos {
  int si, sub, j;
};

// first evaluation at or after stage s0 (FastIvp stages with n_sub >= 1)
__device__ __forceinline__ bool ws_first(const ChainArgs& a, int s0, WsPos& p)
{
  for (int s = s0; s < a.nst; ++s)
    if (a.st[s].kind == 0 && a.st[s].n_sub > 0) {
      p.si = s;
      p.sub = 0;
      p.j = 0;
      return true;
    }
  return false;
}
__device__ __forceinline__ bool ws_next(const ChainArgs& a, const WsPos& p, WsPos& n)
{
  n = p;
  if (p.j + 1 < a.tab.s) {
    n.j = p.j + 1;
    return true;
  }
  n.j = 0;
  if (p.sub + 1 < a.st[p.si].n_sub) {
    n.sub = p.sub + 1;
    return true;
  }
  return ws_first(a, p.si + 1, n);
}

template <int SPL, bool SUBDIAG, int MAXS>
struct WsGroup {
  static constexpr int NPRE = SUBDIAG ? 1 : MAXS;
  double y[SPL], out[SPL], pre[NPRE][SPL];
};

template <int SPL, bool SUBDIAG, int MAXS, int NDEG>
struct WsWorker {
  const ChainArgs& a;
  const ChemParams& P;
  const WsSmem& m;
  int w, c;
  int kk[SPL];
  size_t cell[2];
  bool active[2];
  bool failed[2];

  __device__ __forceinline__ bool mine(int X, int t) const { return active[X] && kk[t] < a.ncomp; }

  // ExplicitUpdate stage s on group X: Y += sum_j (H wbar_ij) fE_j
  __device__ __forceinline__ void update(int X, WsGroup<SPL, SUBDIAG, MAXS>& G, int s)
  {
    const ChainStageDev& st = a.st[s];
    const size_t nc = a.ncell;
    for (int r = 0; r < st.nref; ++r) {
      const double cf = st.coef[0][r];
      if (cf == 0.0) continue;
      const double* __restrict__ fv = a.fE[st.ref_slot[r]];
#pragma unroll
      for (int t = 0; t < SPL; ++t)
        if (mine(X, t)) G.y[t] = dadd(G.y[t], dmul(cf, fv[(size_t)kk[t] * nc + cell[X]]));
    }
    if (!failed[X]) {
      bool bad = false;
#pragma unroll
      for (int t = 0; t < SPL; ++t)
        if (kk[t] < a.ncomp && !isfinite(G.y[t])) bad = true;
      if (bad) {
        atomicMin(a.fail, mr_fail_key(st.mri_stage, 0, 0));
        failed[X] = true;
      }
    }
  }

  // FastIvp stage s begins on group X: forcing coefficients r_k = sum_j
  // (omega[k][i][j]/dc) fE_j (build_forcing's order) into the scratch
  __device__ __forceinline__ void begin_stage(int X, int s)
  {
    const ChainStageDev& st = a.st[s];
    const size_t nc = a.ncell;
#pragma unroll
    for (int t = 0; t < SPL; ++t) {
      if (!mine(X, t)) continue;
      const int kc = kk[t];
      double rcv[NDEG];
#pragma unroll
      for (int k = 0; k < NDEG; ++k) rcv[k] = 0.0;
      for (int r = 0; r < st.nref; ++r) {
        const double x = a.fE[st.ref_slot[r]][(size_t)kc * nc + cell[X]];
#pragma unroll
        for (int k = 0; k < NDEG; ++k) {
          const double cf = st.coef[k][r];
          if (cf != 0.0) rcv[k] = dadd(rcv[k], dmul(cf, x));
        }
      }
#pragma unroll
      for (int k = 0; k < NDEG; ++k) a.rcs[((size_t)k * a.ncomp + kc) * nc + cell[X]] = rcv[k];
    }
  }

  // stage values of the evaluation at p: finite check (erk_step's stage
  // check), then into the group's D rows / energy row for the serial warp
  __device__ __forceinline__ void publish(int X, const double (&stg)[SPL], const WsPos& p)
  {
    if (!failed[X]) {
      bool bad = false;
#pragma unroll
      for (int t = 0; t < SPL; ++t)
        if (kk[t] < a.ncomp && !isfinite(stg[t])) bad = true;
      if (bad) {
        atomicMin(a.fail, mr_fail_key(a.st[p.si].mri_stage, p.sub, p.j));
        failed[X] = true;
      }
    }
    const int S = P.S;
#pragma unroll
    for (int t = 0; t < SPL; ++t) {
      const int k = kk[t];
      if (k < S)
        *reinterpret_cast<double*>(m.D[X] + k * 256 + c * 8) = stg[t];
      else if (k == S)
        m.e[X][c] = stg[t];
    }
    nbar_arrive(1 + X, 32 * 32);
  }

  __device__ __forceinline__ void start_substep(WsGroup<SPL, SUBDIAG, MAXS>& G)
  {
#pragma unroll
    for (int i = 0; i < G.NPRE; ++i)
#pragma unroll
      for (int t = 0; t < SPL; ++t) G.pre[i][t] = G.y[t];
#pragma unroll
    for (int t = 0; t < SPL; ++t) G.out[t] = G.y[t];
  }

  // RK accumulation of the evaluation at p with production rates f, then
  // everything up to the next evaluation n (substep/stage ends, explicit
  // updates, forcing of the next FastIvp stage) and its stage values.
  __device__ __forceinline__ void finish(int X, WsGroup<SPL, SUBDIAG, MAXS>& G, const WsPos& p,
                                         const double (&f)[SPL], bool more, const WsPos& n)
  {
    const ChainStageDev& st = a.st[p.si];
    const double h = st.h_sub;
    const int sf = a.tab.s;
    const int j = p.j;
    const double t0 = dadd(st.t_start, dmul((double)p.sub, h));
    const double theta = dadd(t0, dmul(a.tab.c[j], h));
    const double tau = __ddiv_rn(dadd(theta, -st.t_start), st.span);
    const double hb = dmul(h, a.tab.b[j]);
    const bool use_b = a.tab.b[j] != 0.0;
    double hA_next = 0.0;
    bool useA = false;
    if constexpr (SUBDIAG) {
      useA = j + 1 < sf && a.tab.A[j + 1][j] != 0.0;
      if (useA) hA_next = dmul(h, a.tab.A[j + 1][j]);
    }
    const size_t nc = a.ncell;
#pragma unroll
    for (int t = 0; t < SPL; ++t) {
      const int kc = kk[t];
      double fr = 0.0;
      if (mine(X, t)) {
        fr = a.rcs[((size_t)(NDEG - 1) * a.ncomp + kc) * nc + cell[X]];
#pragma unroll
        for (int k = NDEG - 2; k >= 0; --k)
          fr = dadd(dmul(fr, tau), a.rcs[((size_t)k * a.ncomp + kc) * nc + cell[X]]);
      }
      const double kj = dadd(f[t], fr);
      if constexpr (SUBDIAG) {
        if (j + 1 < sf) G.pre[0][t] = useA ? dadd(G.y[t], dmul(hA_next, kj)) : G.y[t];
      } else {
#pragma unroll
        for (int i = 1; i < G.NPRE; ++i) {
          if (i > j && i < sf) {
            const double Aij = a.tab.A[i][j];
            if (Aij != 0.0) G.pre[i][t] = dadd(G.pre[i][t], dmul(dmul(h, Aij), kj));
          }
        }
      }
      if (use_b) G.out[t] = dadd(G.out[t], dmul(hb, kj));
    }
    double stg[SPL];
    if (j + 1 < sf) {  // next inner stage of this substep
#pragma unroll
      for (int t = 0; t < SPL; ++t) stg[t] = G.pre[0][t];
      if constexpr (!SUBDIAG) {
#pragma unroll
        for (int i = 1; i < G.NPRE; ++i)
          if (i == j + 1) {
#pragma unroll
            for (int t = 0; t < SPL; ++t) stg[t] = G.pre[i][t];
          }
      }
      publish(X, stg, n);
      return;
    }
    // substep end
    if (!failed[X]) {
      bool bad = false;
#pragma unroll
      for (int t = 0; t < SPL; ++t)
        if (kk[t] < a.ncomp && !isfinite(G.out[t])) bad = true;
      if (bad) {
        atomicMin(a.fail, mr_fail_key(st.mri_stage, p.sub, sf));
        failed[X] = true;
      }
    }
#pragma unroll
    for (int t = 0; t < SPL; ++t) G.y[t] = G.out[t];
    if (!more || n.si != p.si) {  // stage end: explicit updates up to the next FastIvp stage
      const int s_end = more ? n.si : a.nst;
      for (int s = p.si + 1; s < s_end; ++s)
        if (a.st[s].kind != 0) update(X, G, s);
      if (!more) return;
      begin_stage(X, n.si);
    }
    start_substep(G);
#pragma unroll
    for (int t = 0; t < SPL; ++t) stg[t] = G.y[t];
    publish(X, stg, n);
  }
};

template <int SPL, bool SUBDIAG, int MAXS, int NDEG>
__global__ void __launch_bounds__(1024, 1)
    chem_chain_ws_kernel(const __grid_constant__ ChainArgs a, const __grid_constant__ ChemParams P)
{
  extern __shared__ __align__(16) double smem_raw[];
  const int c = threadIdx.x & 31;
  const int wid = (int)(threadIdx.x >> 5);
  const WsSmem m = stage_ws(reinterpret_cast<char*>(smem_raw), P, c, wid);
  WsPos pos;
  bool more = ws_first(a, 0, pos);

  if (wid >= kWsWorkers) {  // ---------------- serial warps
    while (more) {
#pragma unroll 1
      for (int X = 0; X < 2; ++X) {
        nbar_sync(1 + X, 32 * 32);
        ws_species_rows(P, m, X, c, wid - kWsWorkers);
        nbar_arrive(3 + X, 32 * 32);
      }
      WsPos nx;
      more = ws_next(a, pos, nx);
      pos = nx;
    }
    return;
  }

  // ---------------- worker warps
  WsWorker<SPL, SUBDIAG, MAXS, NDEG> W{a, P, m, wid, c, {}, {}, {}, {}};
#pragma unroll
  for (int t = 0; t < SPL; ++t) W.kk[t] = P.perm[wid + kWsWorkers * t];
  WsGroup<SPL, SUBDIAG, MAXS> G[2];
#pragma unroll
  for (int X = 0; X < 2; ++X) {
    W.cell[X] = ((size_t)blockIdx.x * 2 + X) * 32 + c;
    W.active[X] = W.cell[X] < a.ncell;
    W.failed[X] = !W.active[X];
#pragma unroll
    for (int t = 0; t < SPL; ++t)
      G[X].y[t] = W.mine(X, t) ? a.y_in[(size_t)W.kk[t] * a.ncell + W.cell[X]] : 0.0;
  }
  // leading explicit updates, then the first evaluation's stage values
#pragma unroll
  for (int X = 0; X < 2; ++X) {
    const int s_end = more ? pos.si : a.nst;
    for (int s = 0; s < s_end; ++s)
      if (a.st[s].kind != 0) W.update(X, G[X], s);
    if (more) {
      W.begin_stage(X, pos.si);
      W.start_substep(G[X]);
      W.publish(X, G[X].y, pos);
    }
  }
  while (more) {
    WsPos nx;
    const bool nmore = ws_next(a, pos, nx);
#pragma unroll
    for (int X = 0; X < 2; ++X) {
      double f[SPL];
      ws_react_produce<SPL>(P, m, X, wid, c, W.kk, f);
      W.finish(X, G[X], pos, f, nmore, nx);
    }
    pos = nx;
    more = nmore;
  }
#pragma unroll
  for (int X = 0; X < 2; ++X)
#pragma unroll
    for (int t = 0; t < SPL; ++t)
      if (W.mine(X, t)) a.y_out[(size_t)W.kk[t] * a.ncell + W.cell[X]] = G[X].y[t];
}

template <int SPL, bool SUBDIAG, int MAXS, int NDEG>
cudaError_t run_chem_chain_ws(const ChainArgs& a, const ChemParams& P, cudaStream_t st)
{
  const size_t smem = ws_smem_bytes(P.S + 1, P.rc, P.blob_words);
  auto k = chem_chain_ws_kernel<SPL, SUBDIAG, MAXS, NDEG>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const size_t blocks = (a.ncell + 63) / 64;
  k<<<(unsigned)blocks, 1024, smem, st>>>(a, P);
  return cudaGetLastError();
}

}  // namespace mrchem
