// pd_lattice_nlu1.cu -- the unrolled n-linear lattice kernel for integrator
// mode 1 (pd_lattice_nlu.cuh).
#include "pd_lattice_nlu.cuh"

namespace pdb {
cudaError_t launch_nlu_m1(const DevArgs& A, const LatticeArgs& L, cudaStream_t st) {
    return launch_nlu_impl<1>(A, L, st);
}
void preload_nlu_m1() { preload_nlu_impl<1>(); }
} // namespace pdb
