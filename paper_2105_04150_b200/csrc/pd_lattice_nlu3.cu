// pd_lattice_nlu3.cu -- the unrolled n-linear lattice kernel for integrator
// mode 3 (pd_lattice_nlu.cuh).
#include "pd_lattice_nlu.cuh"

namespace pdb {
cudaError_t launch_nlu_m3(const DevArgs& A, const LatticeArgs& L, cudaStream_t st) {
    return launch_nlu_impl<3>(A, L, st);
}
void preload_nlu_m3() { preload_nlu_impl<3>(); }
} // namespace pdb
