// kernels_chem_nw16s4g2.cu -- instantiation of the chemistry kernel for two
// 32-cell groups per block, 16 warps x 4 components per thread in each group
// (named barriers per group; see kernels_chem.cuh).
#include "kernels_chem.cuh"

namespace mrchem {
template cudaError_t run_chem_chain<16, 4, true, 4, 1, 2>(const ChainArgs&, const ChemParams&, cudaStream_t);
template cudaError_t run_chem_chain<16, 4, true, 4, 2, 2>(const ChainArgs&, const ChemParams&, cudaStream_t);
template cudaError_t run_chem_chain<16, 4, false, 6, 1, 2>(const ChainArgs&, const ChemParams&, cudaStream_t);
template cudaError_t run_chem_chain<16, 4, false, 6, 2, 2>(const ChainArgs&, const ChemParams&, cudaStream_t);
}  // namespace mrchem
