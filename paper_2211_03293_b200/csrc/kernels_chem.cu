// kernels_chem.cu -- host side of K1 for the chemistry plugin: layout
// choice, rate-buffer chunking and dispatch to the per-layout instantiations
// (kernels_chem_nw*.cu).  Kernel design: kernels_chem.cuh.
#include <cuda_runtime.h>

#include "kernels_chem.cuh"

namespace mrchem {
#define MR_DECL(A, B)                                                                      \
  extern template cudaError_t run_chem_chain<A, B, true, 4, 1>(const ChainArgs&, const ChemParams&, cudaStream_t);  \
  extern template cudaError_t run_chem_chain<A, B, true, 4, 2>(const ChainArgs&, const ChemParams&, cudaStream_t);  \
  extern template cudaError_t run_chem_chain<A, B, false, 6, 1>(const ChainArgs&, const ChemParams&, cudaStream_t); \
  extern template cudaError_t run_chem_chain<A, B, false, 6, 2>(const ChainArgs&, const ChemParams&, cudaStream_t); \
  extern template cudaError_t run_chem_rhs<A, B>(const double*, double*, size_t, int, const ChemParams&, cudaStream_t);
MR_DECL(4, 3)
MR_DECL(8, 3)
MR_DECL(32, 2)
#undef MR_DECL
extern template cudaError_t run_chem_chain<32, 2, false, 3, 1>(const ChainArgs&, const ChemParams&, cudaStream_t);
extern template cudaError_t run_chem_chain<32, 2, false, 3, 2>(const ChainArgs&, const ChemParams&, cudaStream_t);
}  // namespace mrchem

// (NW warps = slots, SPL components per thread) layouts: C1/C2 (10
// components), C3 (22), C4/C5 (54); DESIGN.md section 4 for the measurements
#define MR_CHEM_BLOCK_LAYOUTS(X) X(4, 3) X(8, 3) X(32, 2)

int chem_pick(ChemCfg* cfg, int ncomp, int S, int R, const TableDev& tab, int ndeg)
{
  (void)R;
  if (S + 1 > MR_CHEM_MAXS || ndeg < 1 || ndeg > MR_MAXDEG || tab.s > MR_MAXS) return 1;
  bool subdiag = true;
  for (int i = 0; i < tab.s; ++i)
    for (int j = 0; j < i - 1; ++j)
      if (tab.A[i][j] != 0.0) subdiag = false;
  cfg->subdiag = subdiag;
  cfg->nstage = tab.s;
  cfg->ndeg = ndeg;
  if (ncomp <= 12) { cfg->NW = 4; cfg->SPL = 3; }
  else if (ncomp <= 24) { cfg->NW = 8; cfg->SPL = 3; }
  else if (ncomp <= 64) { cfg->NW = 32; cfg->SPL = 2; }
  else return 1;
  return 0;
}

// rate-buffer chunking: largest chunk (multiple of NW) such that two blocks
// fit the 227 KB shared memory of an SM for NW <= 8 (one 1024-thread block
// for NW = 32)
int chem_chunking(const ChemCfg& cfg, int S, int R, size_t blob_bytes, int* rc, int* nchunk)
{
  const int NW = cfg.NW;
  const size_t budget = (size_t)(NW <= 8 ? 113 : 227) * 1024;
  const int words = (int)((blob_bytes + 15) / 16);
  const size_t fixed = mrchem::smem_bytes(NW, S + 1, 0, words);
  const size_t row = 256;
  if (fixed >= budget) return 1;
  int cap = (int)((budget - fixed) / row);
  cap -= cap % NW;
  if (cap < NW) return 1;
  int n = (R + cap - 1) / cap;
  if (n > MR_CHEM_MAXCHUNK) return 1;
  int size = (R + n - 1) / n;
  size = (size + NW - 1) / NW * NW;
  *rc = size;
  *nchunk = n;
  return 0;
}

cudaError_t launch_chem_chain(const ChemCfg& cfg, const ChainArgs& a, const ChemParams& P,
                              cudaStream_t st)
{
#define MR_CHEM_DISPATCH(A, B)                                                              \
  if (cfg.NW == A && cfg.SPL == B) {                                                        \
    if (cfg.subdiag && cfg.ndeg == 1) return mrchem::run_chem_chain<A, B, true, 4, 1>(a, P, st);   \
    if (cfg.subdiag && cfg.ndeg == 2) return mrchem::run_chem_chain<A, B, true, 4, 2>(a, P, st);   \
    if (!cfg.subdiag && cfg.ndeg == 1) return mrchem::run_chem_chain<A, B, false, 6, 1>(a, P, st); \
    if (!cfg.subdiag && cfg.ndeg == 2) return mrchem::run_chem_chain<A, B, false, 6, 2>(a, P, st); \
  }
  if (cfg.NW == 32 && cfg.SPL == 2 && !cfg.subdiag && cfg.nstage <= 3) {
    if (cfg.ndeg == 1) return mrchem::run_chem_chain<32, 2, false, 3, 1>(a, P, st);
    if (cfg.ndeg == 2) return mrchem::run_chem_chain<32, 2, false, 3, 2>(a, P, st);
  }
  MR_CHEM_BLOCK_LAYOUTS(MR_CHEM_DISPATCH)
#undef MR_CHEM_DISPATCH
  return cudaErrorInvalidConfiguration;
}

cudaError_t launch_chem_rhs(const ChemCfg& cfg, const double* y, double* out, size_t ncell,
                            int ncomp, const ChemParams& P, cudaStream_t st)
{
#define MR_CHEM_RHS(A, B) \
  if (cfg.NW == A && cfg.SPL == B) return mrchem::run_chem_rhs<A, B>(y, out, ncell, ncomp, P, st);
  MR_CHEM_BLOCK_LAYOUTS(MR_CHEM_RHS)
#undef MR_CHEM_RHS
  return cudaErrorInvalidConfiguration;
}

