// pd_lattice_nlu2.cu -- the unrolled n-linear lattice kernel for integrator
// mode 2 (pd_lattice_nlu.cuh).
#include "pd_lattice_nlu.cuh"

namespace pdb {
cudaError_t launch_nlu_m2(const DevArgs& A, const LatticeArgs& L, cudaStream_t st) {
    return launch_nlu_impl<2>(A, L, st);
}
void preload_nlu_m2() { preload_nlu_impl<2>(); }
} // namespace pdb
