// kernels_chem_ws.cu -- instantiation of the warp-specialised chemistry
// chain (31 worker warps x 2 components, one serial warp, two cell groups
// per block; see kernels_chem_ws.cuh).
#include "kernels_chem_ws.cuh"

namespace mrchem {
template cudaError_t run_chem_chain_ws<2, true, 4, 1>(const ChainArgs&, const ChemParams&, cudaStream_t);
template cudaError_t run_chem_chain_ws<2, true, 4, 2>(const ChainArgs&, const ChemParams&, cudaStream_t);
template cudaError_t run_chem_chain_ws<2, false, 6, 1>(const ChainArgs&, const ChemParams&, cudaStream_t);
template cudaError_t run_chem_chain_ws<2, false, 6, 2>(const ChainArgs&, const ChemParams&, cudaStream_t);
// three-stage non-subdiagonal tables (kutta3, C5): fewer stage accumulators
template cudaError_t run_chem_chain_ws<2, false, 3, 1>(const ChainArgs&, const ChemParams&, cudaStream_t);
template cudaError_t run_chem_chain_ws<2, false, 3, 2>(const ChainArgs&, const ChemParams&, cudaStream_t);
}  // namespace mrchem
