// pd_exact.cu -- fp64 "parity" kernels: bitwise equal to the reference CPU path.
//
// Compiled with -fmad=false and written with explicit __d*_rn intrinsics so
// no multiply-add is ever contracted: every slot evaluates exactly the
// reference's IEEE expression sequence.
//
// Mapping (one fused launch per time step):
//   * a group of G lanes owns one node i (G = N for N < 32, 16 for the
//     N = 128 lattice ball -- two nodes per warp share the per-node prologue
//     and epilogue -- else 32); lane l owns slots k = l + G*m, m < M = N/G
//     (N <= 1024);
//   * one PMB law without bond types or corrections (the bench lattice)
//     takes a specialised slot body with the law in registers (slot_pmb);
//   * each lane evaluates its slots like bond_contribution (engine.cpp:53-109):
//     stretch, law, fused break into the alive bitmask (+ n_neigh), history;
//   * the group sums the N contributions with reduce_group's halving-stride
//     tree (engine.cpp:11-19): strides >= G are lane-local (evaluated in tree
//     order, tree_sum), strides < G are __shfl_down steps -- the same pairs in
//     the same order, so the body force
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

#include <cstdlib>

#include "pd_device.cuh"
#include "pd_internal.h"

namespace pdb {


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

    // the law table lives in global memory (up to 256 laws of 32 breakpoints:
    // too large for the constant bank); a warp's reads of one type broadcast
    const DevLaw& law = A.laws[A.btype ? int(__ldg(A.btype + idx)) : 0];
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

// The single-PMB-law model with no bond types and no corrections (the bench
// lattice): bond_contribution (engine.cpp:53-109) with the law constants in
// registers and no law-table, history or correction branches -- the same
// IEEE operations in the same order, so the same bits.
__device__ __forceinline__ Contribution slot_pmb(const DevArgs& A, int j, const double4& xi,
                                                 const double4& ui, bool i_no_fail, bool& alive,
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
    // no-fail bonds never break (engine.cpp:83-86); PMB breaks at s >= s_c (:93-98)
    if (!(i_no_fail || uj.w != 0.0) && s >= A.pmb_sc) {
        alive = false;
        ++broke;
        return c;
    }
    const double f = __dmul_rn(A.pmb_c, s);
    if (cur_len < 1e-30)
        return c;
    const double q = __ddiv_rn(__dmul_rn(f, xj.w), cur_len);
    c.x = __dmul_rn(cx, q);
    c.y = __dmul_rn(cy, q);
    c.z = __dmul_rn(cz, q);
    return c;
}

// reduce_group's lane-local strides (N/2 .. G: c[m] += c[m + h] for h = M/2 .. 1)
// evaluated in tree order: the sum over slots {OFF, OFF + STRIDE, ...} is the
// sum of its even half and its odd half, each formed the same way -- the same
// pairs in the same order as the stride loop, but each slot's contribution is
// added as soon as its partner exists, so at most log2(M) + 1 triples are live
// instead of M.
template <int M, int OFF, int STRIDE, class F>
__device__ __forceinline__ Contribution tree_sum(F& eval) {
    if constexpr (M == 1) {
        return eval(OFF);
    } else {
        const Contribution l = tree_sum<M / 2, OFF, 2 * STRIDE>(eval);
        const Contribution r = tree_sum<M / 2, OFF + STRIDE, 2 * STRIDE>(eval);
        return Contribution{__dadd_rn(l.x, r.x), __dadd_rn(l.y, r.y), __dadd_rn(l.z, r.z)};
    }
}

// 4 CTAs of 256 per SM (64 registers)
#ifndef PD_EXACT_MINB
#define PD_EXACT_MINB 4
#endif
#ifndef PD_EXACT_PF
#define PD_EXACT_PF 2
#endif
// MODE: 0 = force pass only (compute_forces), 1 = velocity-Verlet step,
//       2 = Euler step, 3 = Euler-Cromer step.
// GT lanes own one node (GT = 0: G = N < 32 at run time, M = 1); lane l of a
// node owns slots l + G m, m < M = N / G.  Several nodes per warp (G < 32)
// share the warp's per-node prologue and integrator epilogue; reduce_group's
// strides >= G stay lane-local (tree_sum), strides < G are shuffles within
// the node's G lanes -- the reference's pairs for every G.
template <int MODE, int GT, int M, bool NODE_SUM, bool PMB>
__global__ void __launch_bounds__(256, PD_EXACT_MINB) exact_step_kernel(DevArgs A) {
    if (MODE != 0 && *(volatile long long*)A.err_step != kNoError)
        return; // a previous step saw non-finite u: the reference threw there
    const int G = GT > 0 ? GT : (A.N < 32 ? A.N : 32);
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

    // this lane's slots: live bits (from the row's alive words) and indices
    constexpr int WMAX = GT > 0 ? (GT * M + 31) / 32 : 1;  // alive words per row
    uint32_t old_words[WMAX];
#pragma unroll
    for (int w = 0; w < WMAX; ++w)
        old_words[w] = valid && w < A.W ? A.alive[i * A.W + w] : 0u;
    uint32_t live = 0;  // bit m: slot gl + G m is alive
    int jm[M];
#pragma unroll
    for (int m = 0; m < M; ++m) {
        const int k = gl + G * m;
        const bool al = valid && ((old_words[k >> 5] >> (k & 31)) & 1u);
        live |= (al ? 1u : 0u) << m;
        jm[m] = al ? __ldg(A.entries + i * N + k) : 0;
    }
    // live slots' x and u records prefetched into L1 (no registers held)
    // ahead of their long fp64 evaluation chains: all at once (PD_EXACT_PF =
    // 0), or PD_EXACT_PF slots ahead in evaluation order (the tree order is
    // the bit reversal of 0 .. M-1)
    auto prefetch = [&](int m) {
        if ((live >> m) & 1u) {
            asm volatile("prefetch.global.L1 [%0];" ::"l"(A.xv + jm[m]));
            asm volatile("prefetch.global.L1 [%0];" ::"l"(A.u_in + jm[m]));
        }
    };
    constexpr int PF = PD_EXACT_PF;
    constexpr int LOGM = M >= 32 ? 5 : M >= 16 ? 4 : M >= 8 ? 3 : M >= 4 ? 2 : M >= 2 ? 1 : 0;
    auto bitrev = [](int x) {
        int r = 0;
#pragma unroll
        for (int b = 0; b < LOGM; ++b)
            r |= ((x >> b) & 1) << (LOGM - 1 - b);
        return r;
    };
    if (PF == 0 || NODE_SUM) {
#pragma unroll
        for (int m = 1; m < M; ++m)
            prefetch(m);
    } else {
#pragma unroll
        for (int p = 1; p < PF && p < M; ++p)
            prefetch(bitrev(p));
    }
    int broke = 0;
    auto eval = [&](int m) -> Contribution {
        if (PF > 0 && !NODE_SUM && bitrev(m) + PF < M)
            prefetch(bitrev(bitrev(m) + PF));  // the slot PF positions later
        const int k = gl + G * m;
        bool al = (live >> m) & 1u;
        const Contribution c =
            PMB ? slot_pmb(A, jm[m], xi, ui, i_no_fail, al, broke)
                : slot_contribution(A, i * N + k, jm[m], xi, ui, i_no_fail, al, broke);
        if (!al)
            live &= ~(1u << m);
        return c;
    };
    Contribution c0{};
    Contribution c[NODE_SUM ? M : 1];
    if (!NODE_SUM) {
        c0 = tree_sum<M, 0, 1>(eval);  // reduce_group's lane-local strides
    } else {
#pragma unroll
        for (int m = 0; m < M; ++m)
            c[m] = eval(m);
    }

    // fused break bookkeeping: alive words and n_neigh (engine.cpp:93-96).
    // Word w holds slots 32w .. 32w+31 = lanes gl of sub-slots m = w R + j
    // (R = 32 / G), bit gl + G j.
    const uint32_t gmask = G >= 32 ? 0xffffffffu : ((1u << G) - 1u);
    constexpr int R = GT > 0 && GT < 32 ? 32 / GT : 1;
#pragma unroll
    for (int w = 0; w < WMAX; ++w) {
        uint32_t word = 0;
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const int m = w * R + j;
            if (m < M) {
                const uint32_t b = __ballot_sync(FULL, (live >> m) & 1u);
                word |= (G >= 32 ? b : ((b >> (sub * G)) & gmask)) << (G * j);
            }
        }
        if (valid && gl == 0 && w < A.W && word != old_words[w])
            A.alive[i * A.W + w] = word;
    }
    if (__any_sync(FULL, broke != 0)) {
        for (int off = G / 2; off > 0; off /= 2)
            broke += __shfl_down_sync(FULL, broke, off, G);
        if (valid && gl == 0 && broke)
            A.n_neigh[i] -= broke;
    }

    double fx, fy, fz;
    if (!NODE_SUM) {
        // reduce_group (engine.cpp:11-19) strides G/2 .. 1 across lanes:
        // c[k] += c[k + stride]
        for (int st = G / 2; st >= 1; st /= 2) {
            const double ox = __shfl_down_sync(FULL, c0.x, st, G);
            const double oy = __shfl_down_sync(FULL, c0.y, st, G);
            const double oz = __shfl_down_sync(FULL, c0.z, st, G);
            c0.x = __dadd_rn(c0.x, ox);
            c0.y = __dadd_rn(c0.y, oy);
            c0.z = __dadd_rn(c0.z, oz);
        }
        fx = c0.x;
        fy = c0.y;
        fz = c0.z;
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

template <int MODE, int GT, int M, bool NODE_SUM, bool PMB>
cudaError_t launch_gm(const DevArgs& A, dim3 grid, cudaStream_t st) {
    t_last_kernel = kernel_name<0, MODE, GT, M, NODE_SUM, PMB>("exact_step_kernel");
    exact_step_kernel<MODE, GT, M, NODE_SUM, PMB><<<grid, 256, 0, st>>>(A);
    return cudaGetLastError();
}

// lanes per node: N < 32 -> G = N (M = 1); N = 32, 64 -> G = 32; N = 128 ->
// G = 16 (two nodes per warp, 8 slots per lane); N = 256 .. 1024 -> G = 32
template <int MODE, bool NODE_SUM, bool PMB>
cudaError_t launch_m(const DevArgs& A, int G, int M, dim3 grid, cudaStream_t st) {
    if (G < 32 && M == 1)
        return launch_gm<MODE, 0, 1, NODE_SUM, PMB>(A, grid, st);
    switch (G * 1000 + M) {
    case 32001: return launch_gm<MODE, 32, 1, NODE_SUM, PMB>(A, grid, st);
    case 32002: return launch_gm<MODE, 32, 2, NODE_SUM, PMB>(A, grid, st);
    case 32004: return launch_gm<MODE, 32, 4, NODE_SUM, PMB>(A, grid, st);
    case 16008: return launch_gm<MODE, 16, 8, NODE_SUM, PMB>(A, grid, st);
    case 8016: return launch_gm<MODE, 8, 16, NODE_SUM, PMB>(A, grid, st);
    case 32008: return launch_gm<MODE, 32, 8, NODE_SUM, PMB>(A, grid, st);
    case 32016: return launch_gm<MODE, 32, 16, NODE_SUM, PMB>(A, grid, st);
    case 32032: return launch_gm<MODE, 32, 32, NODE_SUM, PMB>(A, grid, st);
    default: return cudaErrorInvalidValue;
    }
}

template <bool NODE_SUM, bool PMB>
cudaError_t launch_mode(const DevArgs& A, int mode, int G, int M, dim3 grid, cudaStream_t st) {
    switch (mode) {
    case 0:
        return launch_m<0, NODE_SUM, PMB>(A, G, M, grid, st);
    case 1:
        return launch_m<1, NODE_SUM, PMB>(A, G, M, grid, st);
    case 2:
        return launch_m<2, NODE_SUM, PMB>(A, G, M, grid, st);
    default:
        return launch_m<3, NODE_SUM, PMB>(A, G, M, grid, st);
    }
}

} // namespace

template <class K> static void preload(K k) {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, reinterpret_cast<const void*>(k));
}

template <int MODE, bool NS, bool PMB> static void preload_ns() {
    preload(exact_step_kernel<MODE, 0, 1, NS, PMB>);
    preload(exact_step_kernel<MODE, 32, 1, NS, PMB>);
    preload(exact_step_kernel<MODE, 32, 2, NS, PMB>);
    preload(exact_step_kernel<MODE, 32, 4, NS, PMB>);
    preload(exact_step_kernel<MODE, 16, 8, NS, PMB>);
    preload(exact_step_kernel<MODE, 8, 16, NS, PMB>);
    preload(exact_step_kernel<MODE, 32, 8, NS, PMB>);
    preload(exact_step_kernel<MODE, 32, 16, NS, PMB>);
    preload(exact_step_kernel<MODE, 32, 32, NS, PMB>);
}

template <int MODE> static void preload_mode() {
    preload_ns<MODE, false, false>();
    preload_ns<MODE, true, false>();
    preload_ns<MODE, false, true>();
    preload_ns<MODE, true, true>();
}

void preload_exact() {
    preload_mode<0>();
    preload_mode<1>();
    preload_mode<2>();
    preload_mode<3>();
}

cudaError_t launch_exact(const DevArgs& A, int mode, bool node_sum, bool pmb, cudaStream_t st) {
    const long long nodes = A.end - A.begin;
    if (nodes <= 0)
        return cudaSuccess;
    int G = A.N < 32 ? A.N : 32;
    // N = 128 (the 3dx / pi dx lattice ball): two nodes per warp.  PD_EXACT_G
    // overrides (8, 16, 32) for experiments.
    if (A.N == 128)
        G = 16;
    if (const char* e = std::getenv("PD_EXACT_G")) {
        const int g = std::atoi(e);
        if ((g == 8 || g == 16 || g == 32) && A.N == 128)
            G = g;
    }
    const int M = A.N / G;
    const long long per_warp = 32 / G;
    const long long warps = (nodes + per_warp - 1) / per_warp;
    const dim3 grid(unsigned((warps * 32 + 255) / 256));
    if (pmb)
        return node_sum ? launch_mode<true, true>(A, mode, G, M, grid, st)
                        : launch_mode<false, true>(A, mode, G, M, grid, st);
    return node_sum ? launch_mode<true, false>(A, mode, G, M, grid, st)
                    : launch_mode<false, false>(A, mode, G, M, grid, st);
}

} // namespace pdb
