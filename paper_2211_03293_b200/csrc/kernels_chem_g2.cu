// kernels_chem_g2.cu -- instantiation of the two-group chemistry kernel
// (16 warps x 4 components per cell group, two groups per block; see
// kernels_chem_g2.cuh).
#include "kernels_chem_g2.cuh"

namespace mrchem {
template cudaError_t run_chem_chain_g2<16, 4, true, 4, 1>(const ChainArgs&, const ChemParams&, cudaStream_t);
template cudaError_t run_chem_chain_g2<16, 4, true, 4, 2>(const ChainArgs&, const ChemParams&, cudaStream_t);
template cudaError_t run_chem_chain_g2<16, 4, false, 6, 1>(const ChainArgs&, const ChemParams&, cudaStream_t);
template cudaError_t run_chem_chain_g2<16, 4, false, 6, 2>(const ChainArgs&, const ChemParams&, cudaStream_t);
// three-stage non-subdiagonal tables (kutta3, C5): fewer stage accumulators
template cudaError_t run_chem_chain_g2<16, 4, false, 3, 1>(const ChainArgs&, const ChemParams&, cudaStream_t);
template cudaError_t run_chem_chain_g2<16, 4, false, 3, 2>(const ChainArgs&, const ChemParams&, cudaStream_t);
}  // namespace mrchem
