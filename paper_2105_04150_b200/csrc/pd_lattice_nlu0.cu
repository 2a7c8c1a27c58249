// pd_lattice_nlu0.cu -- the unrolled n-linear lattice kernel for integrator
// mode 0 (pd_lattice_nlu.cuh).
#include "pd_lattice_nlu.cuh"

namespace pdb {
cudaError_t launch_nlu_m0(const DevArgs& A, const LatticeArgs& L, cudaStream_t st) {
    return launch_nlu_impl<0>(A, L, st);
}
void preload_nlu_m0() { preload_nlu_impl<0>(); }
} // namespace pdb
