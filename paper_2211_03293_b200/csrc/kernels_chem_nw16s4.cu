// kernels_chem_nw16s4.cu -- instantiation of the chemistry kernel for
// 16 warps per block x 4 components per thread (see kernels_chem.cuh).
#include "kernels_chem.cuh"

namespace mrchem {
template cudaError_t run_chem_chain<16, 4, true, 4, 1>(const ChainArgs&, const ChemParams&, cudaStream_t);
template cudaError_t run_chem_chain<16, 4, true, 4, 2>(const ChainArgs&, const ChemParams&, cudaStream_t);
template cudaError_t run_chem_chain<16, 4, false, 6, 1>(const ChainArgs&, const ChemParams&, cudaStream_t);
template cudaError_t run_chem_chain<16, 4, false, 6, 2>(const ChainArgs&, const ChemParams&, cudaStream_t);
template cudaError_t run_chem_rhs<16, 4>(const double*, double*, size_t, int, const ChemParams&, cudaStream_t);
}  // namespace mrchem
