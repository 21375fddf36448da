// common.cuh -- shared device-side structures of libmri_b200.so.
//
// Layout in HBM: every state-sized vector is
// species-major, Y[comp * ncell + cell], cell = (i * n1 + j) * n2 + k over the
// local slab (axis 0 sharded), exactly the reference's host layout
// (proj/src/models.cpp:117-125, :155-157) so uploads are a single memcpy.
#pragma once

#include <cstddef>
#include <cstdint>

#define MR_MAXS 6      // inner ERK stages (butcher tables up to cash-karp5)
#define MR_MAXDEG 2    // forcing-polynomial coefficients (gark4 uses 2)
#define MR_MAXREF 12   // referenced slow-RHS stage values per MRI stage
#define MR_MAXCHAIN 6  // cell-local MRI stages fused into one launch
#define MR_MAXSLOT 24 // stored slow-RHS stage values
#define MR_MAXLIN 8    // components of the linear test plugins
#define MR_MAXTAU 1024 // per-evaluation tau values carried by a chain launch

// Explicit Butcher table (butcher.hpp:16-27)
struct TableDev {
  int s;
  double A[MR_MAXS][MR_MAXS];
  double b[MR_MAXS];
  double c[MR_MAXS];
};

// One cell-local MRI stage inside a fused chain (mri.cpp:354-426):
//  kind 0 = FastIvp: build_forcing + n_sub inner ERK steps
//  kind 2 = ExplicitUpdate: Y += sum_j (H wbar_ij) fE_j
struct ChainStageDev {
  int kind;
  int mri_stage;
  int n_sub;
  int nref;
  double t_start, span, h_sub;
  int ref_slot[MR_MAXREF];
  // FastIvp: coef[k][r] = omega[k][i][j_r] / dc (0 => term skipped, as
  // build_forcing's `if (coef == 0.0) continue`); Update: coef[0][r] = H*wbar
  double coef[MR_MAXDEG][MR_MAXREF];
};

struct ChainArgs {
  int nst;
  int ndeg;  // r.coeffs.size() = max(degrees, 1)
  ChainStageDev st[MR_MAXCHAIN];
  TableDev tab;
  const double* y_in;
  double* y_out;
  const double* fE[MR_MAXSLOT];
  size_t ncell;  // cells of the slab (the stride of a component)
  int ncomp;
  unsigned long long* fail;
  // tau = (theta - t_start) / span of every inner stage of the chain's FastIvp
  // stages in evaluation order (uniform scalars computed once on the host
  // with the same IEEE operations; ntau = 0: the kernel computes them)
  int ntau;
  double tau[MR_MAXTAU];
  size_t cell0, cell1;  // cells [cell0, cell1) this launch advances (chemistry
                        // chain; cell1 == 0: all), e.g. the plane chunks of a
                        // host-buffer step whose upload is still in flight
};

// Mechanism for the chemistry kernel.  Scalars and per-species data travel
// in the kernel parameter space (constant bank); the per-reaction records and
// the production lists live in a device blob that every block stages into
// shared memory once per launch, so the hot loops read them with broadcast
// LDS.128 (no per-thread constant indexing, no index decoding).
#define MR_CHEM_MAXS 64    // species + 1 (absent-reactant dummy slot)
#define MR_CHEM_MAXR 1024
#define MR_CHEM_MAXCHUNK 6
struct ChemRec {           // 48 B, one per reaction
  double lnA, beta, EaR;
  unsigned r1o, r2o;       // byte offsets of the reactant rows in the (C, E') double2 table
  unsigned p1o, p2o;       // byte offsets of the product rows in the D' table (absent: dummy row)
  unsigned pad0, pad1;
};
struct ChemParams {
  int S, R;
  int rc, nchunk;          // reactions per rate-buffer chunk, number of chunks
  double RuP;
  const uint4* blob;       // [R ChemRec][production entries], 16-B aligned
  int blob_words;          // size of the blob in uint4
  int ent_base;            // first entry word (uint4 index) of the production lists
  double h0[MR_CHEM_MAXS], a[MR_CHEM_MAXS], hb[MR_CHEM_MAXS], s0[MR_CHEM_MAXS];
  double rhoW[MR_CHEM_MAXS], Wrho[MR_CHEM_MAXS];
  double c0[MR_CHEM_MAXS], c1[MR_CHEM_MAXS], c2[MR_CHEM_MAXS];
  // species k, chunk ch: {plus start, plus count, minus start, minus count}
  // in uint4 words relative to ent_base; entries are byte offsets of q rows
  // (chunk-local), lists padded to 4 with the offset of an all-zero row
  ushort4 lst[MR_CHEM_MAXS][MR_CHEM_MAXCHUNK];
  unsigned long long* prof;  // phase-cycle accumulators (MR_PHASE_PROF builds only)
};

struct ChemCfg {
  int NW, SPL;  // warps per block (slots), components per thread
  bool subdiag;
  int nstage;  // inner table stages (non-subdiagonal tables: stage accumulators)
  int ndeg;
};

struct LinDev {
  int n;
  double A[MR_MAXLIN * MR_MAXLIN];
};

// Slow RHS (stencil) arguments
struct StencilArgs {
  const double* y;
  double* out;
  const double* halo_lo;  // [comp][g][n1*n2]: planes i0-g .. i0-1
  const double* halo_hi;  // [comp][g][n1*n2]: planes i0+n0l .. i0+n0l+g-1
  int n0l, n1, n2, ncomp, M;
  int i0;                 // global index of the first local plane
  int i_lo, i_hi;         // local planes [i_lo, i_hi) this launch writes (ring kernel; others: all)
  double a[5], b[5];
  double inv_dx[3], inv_dx2[3];
  double D;
  int vel_kind;
  double u[3];
  const double* prof;     // [3][2][nmax]
  int nmax;
};

// 7-point Laplacian of the IMEX implicit partition (f_I = D L7 y)
struct LapArgs {
  int n0l, n1, n2, ncomp, M;  // M = halo depth of the exchanged planes
  double inv_dx2[3];
  double D;
  double gamma, dg;           // stage gamma and the Jacobi diagonal 1 + gamma D sum 2/dx^2
};

enum FastKind { FK_NONE = 0, FK_CHEM = 1, FK_LINEAR = 2 };
enum SlowKind { SK_NONE = 0, SK_STENCIL = 1, SK_LINEAR = 2 };

// failure key, ordered like the reference's execution order
__host__ __device__ inline unsigned long long mr_fail_key(int mri_stage, int sub, int inner)
{
  return ((unsigned long long)mri_stage << 40) | ((unsigned long long)sub << 8) |
         (unsigned long long)inner;
}
#define MR_NO_FAIL 0xFFFFFFFFFFFFFFFFull

// ---------------- launchers (defined in the .cu files) ----------------
#include <cuda_runtime.h>

// chain kernel configuration chosen by the host
struct ChainCfg {
  int fast_kind;
  int G;     // lanes per cell
  int SPL;   // components per lane
  int maxs;  // 4 or 6
  int ndeg;  // 1 or 2
};
int chain_pick(ChainCfg* cfg, int fast_kind, int ncomp, int s_f, int ndeg);
cudaError_t launch_chain(const ChainCfg& cfg, const ChainArgs& a, const LinDev& lin,
                         cudaStream_t st);
cudaError_t launch_fast_rhs(const ChainCfg& cfg, const double* y, double* out, size_t ncell,
                            int ncomp, const LinDev& lin, cudaStream_t st);

int chem_pick(ChemCfg* cfg, int ncomp, int S, int R, const TableDev& tab, int ndeg);
int chem_chunking(const ChemCfg& cfg, int S, int R, size_t blob_bytes, int* rc, int* nchunk);
cudaError_t launch_chem_chain(const ChemCfg& cfg, const ChainArgs& a, const ChemParams& P,
                              cudaStream_t st);
cudaError_t launch_chem_rhs(const ChemCfg& cfg, const double* y, double* out, size_t ncell,
                            int ncomp, const ChemParams& P, cudaStream_t st);

cudaError_t launch_update(const double* y_in, double* y_out, int nref, const double* const* f,
                          const double* coef, size_t n, int mri_stage,
                          unsigned long long* fail, cudaStream_t st);
cudaError_t launch_update_rows(const double* y_in, double* y_out, int nref, const double* const* f,
                               const double* coef, size_t row_len, int rows, size_t row_stride,
                               int mri_stage, unsigned long long* fail, cudaStream_t st);
cudaError_t launch_stencil(const StencilArgs& a, cudaStream_t st);
bool stencil_plane_ranges(const StencilArgs& a);  // launch_stencil accepts [i_lo, i_hi) < all planes
cudaError_t launch_slow_linear(const double* y, double* out, size_t ncell, const LinDev& lin,
                               cudaStream_t st);
cudaError_t launch_halo_pack(const double* y, double* send_lo, double* send_hi, int ncomp,
                             int n0l, size_t plane, int g, cudaStream_t st);

// reductions: result written to *d_out (device); fixed-order two-pass
enum RedKind { RED_WRMS = 0, RED_TWO = 1, RED_DOT = 2, RED_MAX = 3, RED_NONFINITE = 4 };
cudaError_t launch_reduce(int kind, const double* x, const double* w, size_t n, double* d_part,
                          int nblocks, double* d_out, cudaStream_t st);
int reduce_blocks();

int lap_blocks();
cudaError_t launch_lap7(int mode, const LapArgs& a, const double* y, const double* lo,
                        const double* hi, const double* known, const double* w, double* o1,
                        double* o2, double* o3, double* part, double* part2, cudaStream_t st);
cudaError_t launch_cg_update(size_t n, double dg, const double* sc, double* Y, double* r, double* z,
                             const double* p, const double* q, double* part, cudaStream_t st);
cudaError_t launch_cg_p(size_t n, const double* sc, double* p, const double* z, cudaStream_t st);
cudaError_t launch_part_sum(const double* part, double* sc, int slot, cudaStream_t st);
cudaError_t launch_scalar_combine(double* const* scs, int n, int slot, cudaStream_t st);
cudaError_t launch_gathered_sum(const double* g, int n, double* sc, int slot, cudaStream_t st);
cudaError_t launch_scalar_copy(double* sc, int dst, int src, cudaStream_t st);
cudaError_t launch_sum_rhs(size_t n, const double* ff, const double* fi, const double* fe,
                           double* out, cudaStream_t st);
cudaError_t launch_add2(size_t n, const double* a, const double* b, double* out, cudaStream_t st);
cudaError_t launch_recover_fi(size_t n, double gamma, const double* Y, const double* known,
                              double* fI, int mri_stage, unsigned long long* fail,
                              cudaStream_t st);

cudaError_t launch_fp64_peak(double* sink, int blocks, int threads, int iters, cudaStream_t st);
