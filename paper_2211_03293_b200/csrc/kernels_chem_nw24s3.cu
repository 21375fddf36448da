// kernels_chem_nw24s3.cu -- instantiation of the chemistry kernel for
// 24 warps per block x 3 components per thread (see kernels_chem.cuh).
#include "kernels_chem.cuh"

namespace mrchem {
template cudaError_t run_chem_chain<24, 3, true, 4, 1>(const ChainArgs&, const ChemParams&, cudaStream_t);
template cudaError_t run_chem_chain<24, 3, true, 4, 2>(const ChainArgs&, const ChemParams&, cudaStream_t);
template cudaError_t run_chem_chain<24, 3, false, 6, 1>(const ChainArgs&, const ChemParams&, cudaStream_t);
template cudaError_t run_chem_chain<24, 3, false, 6, 2>(const ChainArgs&, const ChemParams&, cudaStream_t);
template cudaError_t run_chem_rhs<24, 3>(const double*, double*, size_t, int, const ChemParams&, cudaStream_t);
}  // namespace mrchem
