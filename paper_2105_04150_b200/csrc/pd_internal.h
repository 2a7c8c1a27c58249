// pd_internal.h -- host-side launcher declarations shared by the .cu units.
#pragma once

#include <cuda_runtime.h>

#include "pd_device.cuh"

namespace pdb {

// pd_host.cu: record the message pd_last_error() returns; returns code.
int set_error(int code, const char* msg);

// pd_exact.cu
void exact_set_laws(const DevLaw* laws, int n, cudaStream_t stream);
cudaError_t launch_exact(const DevArgs& A, int mode, bool node_sum, cudaStream_t st);

// pd_aux.cu
void launch_pack_xv(const double* coords, const double* volume, long long n, double4* xv,
                    cudaStream_t st);
void launch_pack_u(const double* u, const uint8_t* nofail, long long n, double4* out,
                   cudaStream_t st);
void launch_unpack_u(const double4* u, long long n, double* out, cudaStream_t st);
void launch_init_alive(const int32_t* entries, long long n, int N, int W, uint32_t* alive,
                       cudaStream_t st);
void launch_validate_entries(const int32_t* entries, long long n, int N,
                             unsigned long long* bad_row, cudaStream_t st);
void launch_vv_prologue(const DevArgs& A, cudaStream_t st);
void launch_check_finite(const double4* u, long long begin, long long end, long long step,
                         long long* err, cudaStream_t st);
void launch_materialize_entries(const int32_t* entries, const uint32_t* alive, long long n, int N,
                                int W, int32_t* out, cudaStream_t st);
void launch_damage(const int32_t* n_neigh, const int32_t* initial, long long n, double* phi,
                   cudaStream_t st);
void launch_sum(const int32_t* x, long long n, unsigned long long* out, cudaStream_t st);
void launch_tips(const double4* u, const double* v, const double* a, const double4* xv,
                 const double* body, const double* ext, int n_sets, const long long* offsets,
                 const long long* nodes, long long step, pd_tip_record* out, cudaStream_t st);

} // namespace pdb
