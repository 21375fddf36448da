// kernels_chem2_nw18s3.cu -- instantiation of the two-cells-per-thread
// chemistry kernel (kernels_chem2.cuh) for 18 warps x 3 components per
// thread: the 54 components of the 53-species mechanisms (C4, C5).
#include "kernels_chem2.cuh"

namespace mrchem {
template cudaError_t run_chem2_chain<18, 3, true, 4, 1>(const ChainArgs&, const ChemParams&, cudaStream_t);
template cudaError_t run_chem2_chain<18, 3, true, 4, 2>(const ChainArgs&, const ChemParams&, cudaStream_t);
template cudaError_t run_chem2_chain<18, 3, false, 6, 1>(const ChainArgs&, const ChemParams&, cudaStream_t);
template cudaError_t run_chem2_chain<18, 3, false, 6, 2>(const ChainArgs&, const ChemParams&, cudaStream_t);
// three-stage non-subdiagonal tables (kutta3, C5): fewer stage accumulators
template cudaError_t run_chem2_chain<18, 3, false, 3, 1>(const ChainArgs&, const ChemParams&, cudaStream_t);
template cudaError_t run_chem2_chain<18, 3, false, 3, 2>(const ChainArgs&, const ChemParams&, cudaStream_t);
template cudaError_t run_chem2_rhs<18, 3>(const double*, double*, size_t, int, const ChemParams&, cudaStream_t);
}  // namespace mrchem
