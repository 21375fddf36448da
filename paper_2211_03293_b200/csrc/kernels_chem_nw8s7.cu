// kernels_chem_nw8s7.cu -- instantiation of the chemistry kernel for
// 8 warps per block x 7 components per thread (see kernels_chem.cuh).
#include "kernels_chem.cuh"

namespace mrchem {
template cudaError_t run_chem_chain<8, 7, true, 4, 1>(const ChainArgs&, const ChemParams&, cudaStream_t);
template cudaError_t run_chem_chain<8, 7, true, 4, 2>(const ChainArgs&, const ChemParams&, cudaStream_t);
template cudaError_t run_chem_chain<8, 7, false, 6, 1>(const ChainArgs&, const ChemParams&, cudaStream_t);
template cudaError_t run_chem_chain<8, 7, false, 6, 2>(const ChainArgs&, const ChemParams&, cudaStream_t);
template cudaError_t run_chem_rhs<8, 7>(const double*, double*, size_t, int, const ChemParams&, cudaStream_t);
}  // namespace mrchem
