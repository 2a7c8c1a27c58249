// pd_exact.cu -- fp64 "parity" kernels: bitwise equal to the reference CPU path.
//
// Compiled with -fmad=false and written with explicit __d*_rn intrinsics so
// no multiply-add is ever contracted: every slot evaluates exactly the
// reference's IEEE expression sequence.
//
// Mapping (one fused launch per time step):
//   * a group of G = min(N, 32) lanes owns one node i; lane l owns slots
//     k = l + G*m, m < M = N/G (M <= 8, so N <= 256);
//   * each lane evaluates its slots like bond_contribution (engine.cpp:53-109):
//     stretch, law, fused break into the alive bitmask (+ n_neigh), history;
//   * the group sums the N contributions with reduce_group's halving-stride
//     tree (engine.cpp:11-19): strides >= G are lane-local, strides < G are
//     __shfl_down steps -- the same pairs in the same order, so the body force
//     is bit-identical to compute_forces_bond_parallel.  The node_parallel
//     variant is a serial in-order sum (engine.cpp:152-158) via broadcasts;
//   * lane 0 then runs the node's integrator epilogue in the reference's order:
//     velocity-Verlet kick + displacement kinematics (engine.cpp:235-252,
//     274-286) and the NEXT step's drift + prescribed positions (engine.cpp:
//     221-233, 262-272) into the other u buffer; or Euler / Euler-Cromer
//     (engine.cpp:187-219) with positions + kinematics of step s+1.
//   Double-buffered u removes the read/write race the paper cites as the
//   reason integration cannot be fused.
#include <cuda_runtime.h>

#include "pd_device.cuh"
#include "pd_internal.h"

namespace pdb {

__constant__ DevLaw c_laws[PD_MAX_LAWS];

void exact_set_laws(const DevLaw* laws, int n, cudaStream_t stream) {
    cudaMemcpyToSymbolAsync(c_laws, laws, sizeof(DevLaw) * size_t(n), 0,
                            cudaMemcpyHostToDevice, stream);
}

namespace {

constexpr unsigned FULL = 0xffffffffu;

// envelope_force / secant_stiffness (formulas.hpp:77-96)
__device__ __forceinline__ double envelope_force(const DevLaw& law, double s) {
    double s_prev = 0.0, f_prev = 0.0;
    for (int k = 0; k < law.nbp; ++k) {
        const double s_k = law.bp[k];
        if (s < s_k || k + 1 == law.nbp) {
            const double t = __ddiv_rn(__dsub_rn(s, s_prev), __dsub_rn(s_k, s_prev));
            return __dadd_rn(f_prev, __dmul_rn(t, __dsub_rn(law.f[k], f_prev)));
        }
        s_prev = s_k;
        f_prev = law.f[k];
    }
    return __dmul_rn(law.c, s);
}

__device__ __forceinline__ double secant_stiffness(const DevLaw& law, double h) {
    if (h <= 0.0)
        return law.c;
    return __ddiv_rn(envelope_force(law, h), h);
}

__device__ __forceinline__ double norm3(double x, double y, double z) {
    return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z)));
}

struct Contribution {
    double x, y, z;
};

// One slot of bond_contribution (engine.cpp:53-109).  Returns the slot's
// contribution; clears `alive` on a break.
// j is loaded (and its records prefetched into L1) by the caller before any
// slot is evaluated.
__device__ __forceinline__ Contribution slot_contribution(const DevArgs& A, long long idx, int j,
                                                          const double4& xi, const double4& ui,
                                                          bool i_no_fail, bool& alive,
                                                          int& broke) {
    Contribution c{0.0, 0.0, 0.0};
    if (!alive)
        return c;
    const double4 xj = A.xv[j];
    const double4 uj = A.u_in[j];
    const double rx = __dsub_rn(xj.x, xi.x), ry = __dsub_rn(xj.y, xi.y), rz = __dsub_rn(xj.z, xi.z);
    const double cx = __dadd_rn(rx, __dsub_rn(uj.x, ui.x));
    const double cy = __dadd_rn(ry, __dsub_rn(uj.y, ui.y));
    const double cz = __dadd_rn(rz, __dsub_rn(uj.z, ui.z));
    const double ref_len = norm3(rx, ry, rz);
    const double cur_len = norm3(cx, cy, cz);
    const double s = __ddiv_rn(__dsub_rn(cur_len, ref_len), ref_len);

    const DevLaw& law = c_laws[A.btype ? int(__ldg(A.btype + idx)) : 0];
    double f;
    const bool no_fail = i_no_fail || uj.w != 0.0;
    if (no_fail) {
        f = __dmul_rn(law.c, s);
    } else if (law.nbp == 1) {
        if (s >= law.bp[0]) {
            alive = false;
            ++broke;
            return c;
        }
        f = __dmul_rn(law.c, s);
    } else {
        const double s_c = law.bp[law.nbp - 1];
        const double h = A.hist[idx];
        if (s > h)
            A.hist[idx] = s;
        if (h >= s_c || s >= s_c) {
            alive = false;
            ++broke;
            return c;
        }
        f = (s >= h) ? envelope_force(law, s) : __dmul_rn(secant_stiffness(law, h), s);
    }
    if (cur_len < 1e-30)
        return c;
    double scale = __dmul_rn(f, xj.w);
    if (A.lambda)
        scale = __dmul_rn(scale, __ldg(A.lambda + idx));
    if (A.beta)
        scale = __dmul_rn(scale, __ldg(A.beta + idx));
    const double q = __ddiv_rn(scale, cur_len);
    c.x = __dmul_rn(cx, q);
    c.y = __dmul_rn(cy, q);
    c.z = __dmul_rn(cz, q);
    return c;
}

// 4 CTAs of 256 per SM (64 registers, small spill): 16.6 ms/step at 10M against 18.6 ms at
// the compiler's 80 registers (3 CTAs) -- the kernel is gather-latency bound
// (PD_EXACT_MINB for experiments)
#ifndef PD_EXACT_MINB
#define PD_EXACT_MINB 4
#endif
// MODE: 0 = force pass only (compute_forces), 1 = velocity-Verlet step,
//       2 = Euler step, 3 = Euler-Cromer step.
template <int MODE, int M, bool NODE_SUM>
__global__ void __launch_bounds__(256, PD_EXACT_MINB) exact_step_kernel(DevArgs A) {
    if (MODE != 0 && *(volatile long long*)A.err_step != kNoError)
        return; // a previous step saw non-finite u: the reference threw there
    const int G = (M > 1) ? 32 : (A.N < 32 ? A.N : 32);
    const int lane = threadIdx.x & 31;
    const int sub = lane / G;
    const int gl = lane - sub * G;
    const long long warp = (long long)(blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long i = A.begin + warp * (32 / G) + sub;
    const bool valid = i < A.end;
    const int N = A.N;

    double4 xi = make_double4(0, 0, 0, 0), ui = make_double4(0, 0, 0, 0);
    if (valid) {
        xi = A.xv[i];
        ui = A.u_in[i];
    }
    const bool i_no_fail = ui.w != 0.0;

    Contribution c[M];
    uint32_t old_words[M];
    bool alive[M];
    int broke = 0;
    // every live slot's neighbour index first, and its x and u records
    // prefetched into L1 (no registers held), before the first slot's long
    // fp64 evaluation chain: otherwise each slot's gather waits on L2 in turn
    int jm[M];
#pragma unroll
    for (int m = 0; m < M; ++m) {
        const int k = gl + G * m;
        old_words[m] = valid ? A.alive[i * A.W + (k >> 5)] : 0u;
        alive[m] = valid && ((old_words[m] >> (k & 31)) & 1u);
        jm[m] = alive[m] ? __ldg(A.entries + i * N + k) : 0;
    }
#pragma unroll
    for (int m = 1; m < M; ++m)
        if (alive[m]) {
            asm volatile("prefetch.global.L1 [%0];" ::"l"(A.xv + jm[m]));
            asm volatile("prefetch.global.L1 [%0];" ::"l"(A.u_in + jm[m]));
        }
#pragma unroll
    for (int m = 0; m < M; ++m) {
        const int k = gl + G * m;
        c[m] = slot_contribution(A, i * N + k, jm[m], xi, ui, i_no_fail, alive[m], broke);
    }

    // fused break bookkeeping: alive words and n_neigh (engine.cpp:93-96)
#pragma unroll
    for (int m = 0; m < M; ++m) {
        uint32_t word = __ballot_sync(FULL, alive[m]);
        if (G < 32)
            word = (word >> (sub * G)) & (0xffffffffu >> (32 - G));
        if (valid && gl == 0 && word != old_words[m])
            A.alive[i * A.W + m] = word;
    }
    if (__any_sync(FULL, broke != 0)) {
        for (int off = G / 2; off > 0; off /= 2)
            broke += __shfl_down_sync(FULL, broke, off, G);
        if (valid && gl == 0 && broke)
            A.n_neigh[i] -= broke;
    }

    double fx, fy, fz;
    if (!NODE_SUM) {
        // reduce_group (engine.cpp:11-19): strides N/2 .. G lane-local ...
#pragma unroll
        for (int h = M / 2; h >= 1; h /= 2)
#pragma unroll
            for (int mm = 0; mm < h; ++mm) {
                c[mm].x = __dadd_rn(c[mm].x, c[mm + h].x);
                c[mm].y = __dadd_rn(c[mm].y, c[mm + h].y);
                c[mm].z = __dadd_rn(c[mm].z, c[mm + h].z);
            }
        // ... strides G/2 .. 1 across lanes: c[k] += c[k + stride]
        for (int st = G / 2; st >= 1; st /= 2) {
            const double ox = __shfl_down_sync(FULL, c[0].x, st, G);
            const double oy = __shfl_down_sync(FULL, c[0].y, st, G);
            const double oz = __shfl_down_sync(FULL, c[0].z, st, G);
            c[0].x = __dadd_rn(c[0].x, ox);
            c[0].y = __dadd_rn(c[0].y, oy);
            c[0].z = __dadd_rn(c[0].z, oz);
        }
        fx = c[0].x;
        fy = c[0].y;
        fz = c[0].z;
    } else {
        // compute_forces_node_parallel: serial left-to-right sum over slots
        fx = fy = fz = 0.0;
#pragma unroll
        for (int m = 0; m < M; ++m)
            for (int l = 0; l < G; ++l) {
                fx = __dadd_rn(fx, __shfl_sync(FULL, c[m].x, l, G));
                fy = __dadd_rn(fy, __shfl_sync(FULL, c[m].y, l, G));
                fz = __dadd_rn(fz, __shfl_sync(FULL, c[m].z, l, G));
            }
    }
    if (!valid || gl != 0)
        return;

    if (MODE == 0) {
        A.body_force[3 * i] = fx;
        A.body_force[3 * i + 1] = fy;
        A.body_force[3 * i + 2] = fz;
        return;
    }
    node_epilogue<MODE>(A, i, ui, fx, fy, fz);
}

template <int MODE, bool NODE_SUM>
cudaError_t launch_m(const DevArgs& A, int M, dim3 grid, cudaStream_t st) {
    switch (M) {
    case 1:
        t_last_kernel = kernel_name<0, MODE, 1, NODE_SUM>("exact_step_kernel");
        exact_step_kernel<MODE, 1, NODE_SUM><<<grid, 256, 0, st>>>(A);
        break;
    case 2:
        t_last_kernel = kernel_name<0, MODE, 2, NODE_SUM>("exact_step_kernel");
        exact_step_kernel<MODE, 2, NODE_SUM><<<grid, 256, 0, st>>>(A);
        break;
    case 4:
        t_last_kernel = kernel_name<0, MODE, 4, NODE_SUM>("exact_step_kernel");
        exact_step_kernel<MODE, 4, NODE_SUM><<<grid, 256, 0, st>>>(A);
        break;
    case 8:
        t_last_kernel = kernel_name<0, MODE, 8, NODE_SUM>("exact_step_kernel");
        exact_step_kernel<MODE, 8, NODE_SUM><<<grid, 256, 0, st>>>(A);
        break;
    default:
        return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

template <bool NODE_SUM>
cudaError_t launch_mode(const DevArgs& A, int mode, int M, dim3 grid, cudaStream_t st) {
    switch (mode) {
    case 0:
        return launch_m<0, NODE_SUM>(A, M, grid, st);
    case 1:
        return launch_m<1, NODE_SUM>(A, M, grid, st);
    case 2:
        return launch_m<2, NODE_SUM>(A, M, grid, st);
    default:
        return launch_m<3, NODE_SUM>(A, M, grid, st);
    }
}

} // namespace

template <class K> static void preload(K k) {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, reinterpret_cast<const void*>(k));
}

template <int MODE> static void preload_mode() {
    preload(exact_step_kernel<MODE, 1, false>);
    preload(exact_step_kernel<MODE, 2, false>);
    preload(exact_step_kernel<MODE, 4, false>);
    preload(exact_step_kernel<MODE, 8, false>);
    preload(exact_step_kernel<MODE, 1, true>);
    preload(exact_step_kernel<MODE, 2, true>);
    preload(exact_step_kernel<MODE, 4, true>);
    preload(exact_step_kernel<MODE, 8, true>);
}

void preload_exact() {
    preload_mode<0>();
    preload_mode<1>();
    preload_mode<2>();
    preload_mode<3>();
}

cudaError_t launch_exact(const DevArgs& A, int mode, bool node_sum, cudaStream_t st) {
    const long long nodes = A.end - A.begin;
    if (nodes <= 0)
        return cudaSuccess;
    const int G = A.N < 32 ? A.N : 32;
    const int M = A.N / G;
    const long long per_warp = 32 / G;
    const long long warps = (nodes + per_warp - 1) / per_warp;
    const dim3 grid(unsigned((warps * 32 + 255) / 256));
    return node_sum ? launch_mode<true>(A, mode, M, grid, st)
                    : launch_mode<false>(A, mode, M, grid, st);
}

} // namespace pdb
