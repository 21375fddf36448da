// kernels_chem_nw32s2.cu -- instantiation of the chemistry kernel for
// 32 warps per block x 2 components per thread (see kernels_chem.cuh).
#include "kernels_chem.cuh"

namespace mrchem {
template cudaError_t run_chem_chain<32, 2, true, 4, 1>(const ChainArgs&, const ChemParams&, cudaStream_t);
template cudaError_t run_chem_chain<32, 2, true, 4, 2>(const ChainArgs&, const ChemParams&, cudaStream_t);
template cudaError_t run_chem_chain<32, 2, false, 6, 1>(const ChainArgs&, const ChemParams&, cudaStream_t);
template cudaError_t run_chem_chain<32, 2, false, 6, 2>(const ChainArgs&, const ChemParams&, cudaStream_t);
// three-stage non-subdiagonal tables (kutta3, C5): fewer stage accumulators
template cudaError_t run_chem_chain<32, 2, false, 3, 1>(const ChainArgs&, const ChemParams&, cudaStream_t);
template cudaError_t run_chem_chain<32, 2, false, 3, 2>(const ChainArgs&, const ChemParams&, cudaStream_t);
template cudaError_t run_chem_rhs<32, 2>(const double*, double*, size_t, int, const ChemParams&, cudaStream_t);
}  // namespace mrchem
