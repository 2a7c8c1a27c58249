// pd_lattice_nlu.cuh -- the unrolled n-linear lattice kernel, instantiated per
// integrator in pd_lattice_nlu<MODE>.cu (four translation units, so the
// heavily unrolled instantiations compile in parallel).
#pragma once
#include "pd_lattice.cuh"

namespace pdb {
namespace {

// ---- the unrolled NL kernel: one register law of <= 3 breakpoints --------------
//
// The 122 slots unrolled like the PMB kernel (compile-time offsets, length
// classes).  The per-bond streams (stretch history, lambda * beta) are read
// through a ring of ND registers: slot K's values are loaded ND slots ahead at
// a compile-time offset of the thread's brick-major base (pd_lattice.cuh
// slot_base).  The loads are not predicated on the live bit: a dead slot's
// value is never used, and an interior node has every slot live.
//
// The law is branch free:
//   e   = max(s, h, tiny)                        (h: stretch history)
//   env = op1(l_0(e), op2(l_1(e), l_2(e)))       (l_k(e) = a_k + sl_k e: segment
//                                                 k of envelope_force; op = min
//                                                 at a concave kink, max at a
//                                                 convex one -- the piecewise-
//                                                 linear envelope exactly)
//   f   = env * (s / e)                          (= env(s) when s >= h, else
//                                                 secant(h) s = env(h) / h * s,
//                                                 which is c s while h < bp_0;
//                                                 tiny stands in for h = 0, where
//                                                 the secant is c, formulas.hpp:92-96)
// History is written (s > h) before the break test e >= s_c, as
// bond_contribution does (engine.cpp:88-92); no-failure pairs take c s with
// no history and no break (engine.cpp:79-88).  Breaks are detected as in the
// PMB kernel: every live slot adds its force and the largest breakable e is
// tracked; a node whose bonds break is recomputed without them.

// store s when the slot is live (on != 0), breakable (w >= thr) and s > hh as
// one predicated instruction; volatile: kept in program order with the other
// volatile asm, so the slow path (behind a compiler barrier) reads it back
template <bool NF>
__device__ __forceinline__ void stg_hist_if(float* p, unsigned on, float w, float thr, float s,
                                            float hh) {
    if (NF)
        asm volatile("{\n\t.reg .pred q, r, t;\n\t"
                     "setp.ne.u32 q, %1, 0;\n\t"
                     "setp.ge.and.f32 r, %2, %3, q;\n\t"
                     "setp.gt.and.f32 t, %4, %5, r;\n\t"
                     "@t st.global.f32 [%0], %4;\n\t}"
                     :: "l"(p), "r"(on), "f"(w), "f"(thr), "f"(s), "f"(hh));
    else
        asm volatile("{\n\t.reg .pred q, t;\n\t"
                     "setp.ne.u32 q, %1, 0;\n\t"
                     "setp.gt.and.f32 t, %2, %3, q;\n\t"
                     "@t st.global.f32 [%0], %2;\n\t}"
                     :: "l"(p), "r"(on), "f"(s), "f"(hh));
}

#ifndef PD_NLU_PRED
#define PD_NLU_PRED 1
#endif
// a ring load predicated on the slot's live bit (a dead slot keeps the
// register's previous, finite, value: its result is never used).  volatile:
// it stays ND slots ahead of its use, between the (volatile) history stores
// of its neighbouring slots -- the compiler would otherwise sink the load
// toward its use to save registers and expose the HBM latency.
__device__ __forceinline__ void ldg_keep_if(float& v, const float* p, unsigned on) {
    asm volatile("{\n\t.reg .pred q;\n\t"
        "setp.ne.u32 q, %2, 0;\n\t"
        "@q ld.global.f32 %0, [%1];\n\t}"
        : "+f"(v) : "l"(p), "r"(on));
}

#ifndef PD_NLU_PFD
#define PD_NLU_PFD 24
#endif
__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" :: "l"(p));
}

// typed (several laws): store the history word (s with the bond type in its
// low 3 bits) when the slot is live, breakable, of a law with history
// (hflag > 0) and s > hh
template <bool NF>
__device__ __forceinline__ void stg_typed_if(float* p, unsigned on, float w, float thr, float hflag,
                                             float s, float hh, unsigned word) {
    if (NF)
        asm volatile("{\n\t.reg .pred q, r, t, u;\n\t"
                     "setp.ne.u32 q, %1, 0;\n\t"
                     "setp.ge.and.f32 r, %2, %3, q;\n\t"
                     "setp.gt.and.f32 u, %4, 0f00000000, r;\n\t"
                     "setp.gt.and.f32 t, %5, %6, u;\n\t"
                     "@t st.global.b32 [%0], %7;\n\t}"
                     :: "l"(p), "r"(on), "f"(w), "f"(thr), "f"(hflag), "f"(s), "f"(hh), "r"(word));
    else
        asm volatile("{\n\t.reg .pred q, t, u;\n\t"
                     "setp.ne.u32 q, %1, 0;\n\t"
                     "setp.gt.and.f32 u, %2, 0f00000000, q;\n\t"
                     "setp.gt.and.f32 t, %3, %4, u;\n\t"
                     "@t st.global.b32 [%0], %5;\n\t}"
                     :: "l"(p), "r"(on), "f"(hflag), "f"(s), "f"(hh), "r"(word));
}

__device__ __forceinline__ void bulk_prefetch_l2(const void* p, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(p), "r"(bytes) : "memory");
}

struct AccN {
    float2 gxy;
    float gz;
    float2 fxy;
    float fz;
    float emax;  // largest e over live breakable slots
};

#ifndef PD_NLU_ND
#define PD_NLU_ND 8
#endif
constexpr int ND = PD_NLU_ND;  // ring depth (slots of history / lambda loads in flight)

// f for stretch s and history hh (hh ignored for NBP = 1); e is the stretch
// the break test uses (max(s, h))
// several laws (NBP = 0): the bond's law from the per-type table, three
// segment lines (a law with fewer breakpoints repeats its last line);
// p0 = (c, sl_1, a_1, +-s_c: + when the law keeps history), p1 = (sl_2, a_2,
// +1 convex first kink / -1, +1 convex second kink / -1)
__device__ __forceinline__ float nl_law_typed(const float4& p0, const float4& p1, float s, float hh,
                                              float& e) {
    e = fmax_nan3(s, hh, 1e-30f);
    const float l0 = p0.x * e, l1 = fmaf(p0.y, e, p0.z), l2 = fmaf(p1.x, e, p1.y);
    const float t = p1.w > 0.f ? fmaxf(l1, l2) : fminf(l1, l2);
    const float env = p1.z > 0.f ? fmaxf(l0, t) : fminf(l0, t);
    return env * (s * rcp_approx(e));
}

template <int NBP>
__device__ __forceinline__ float nl_law(const NlRegLaw& R, float s, float hh, float& e) {
    if (NBP == 1) {
        e = s;
        return R.c * s;
    }
    e = fmax_nan3(s, hh, 1e-30f);
    const float l0 = R.sl0 * e, l1 = fmaf(R.sl1, e, R.a1), l2 = fmaf(R.sl2, e, R.a2);
    const float t = R.cvx2 ? fmaxf(l1, l2) : fminf(l1, l2);
    const float env = R.cvx1 ? fmaxf(l0, t) : fminf(l0, t);
    return env * (s * rcp_approx(e));
}

template <int K, int NBP, bool LAM, bool NF, int NB>
__device__ __forceinline__ void nl_slot(const float4* own, const float4& ri, const uint4& m,
                                        float* hb, const float* lb, float nfthr,
                                        const NlRegLaw& R, const float4* tab, float (&hr)[ND],
                                        float (&lr)[ND], AccN& acc) {
    constexpr int C = kOrder.slot[K];
    constexpr int dx = pat(C, 0), dy = pat(C, 1), dz = pat(C, 2);
    constexpr int off = dx + HX * (dy + HY * dz);
    constexpr unsigned bit = 1u << (C & 31);
    constexpr int word = C >> 5;
    const unsigned mw = word == 0 ? m.x : (word == 1 ? m.y : (word == 2 ? m.z : m.w));
    const bool live = (mw & bit) != 0u;
    // this slot's streamed values; refill the ring ND slots ahead
    float hh = NBP != 1 ? hr[K % ND] : 0.f;
    const float lam = LAM ? lr[K % ND] : 1.f;
    // typed: the ring holds history words (bond type in the low 3 bits)
    unsigned ty = 0u;
    float4 p0, p1;
    if (NBP == 0) {
        const unsigned bits = __float_as_uint(hh);
        ty = bits & 7u;
        hh = __uint_as_float(bits & ~7u);
        p0 = tab[2 * ty];
        p1 = tab[2 * ty + 1];
        if (!(p0.w > 0.f))
            hh = 0.f;  // a law without history (PMB) never reads one (engine.cpp:84-87)
    }
    if constexpr (K + ND < NPAT) {
        constexpr int CN = kOrder.slot[K + ND];
#if PD_NLU_PRED
        constexpr unsigned nbit = 1u << (CN & 31);
        constexpr int nword = CN >> 5;
        const unsigned nmw = nword == 0 ? m.x : (nword == 1 ? m.y : (nword == 2 ? m.z : m.w));
        if (NBP != 1)
            ldg_keep_if(hr[K % ND], hb + CN * NB, nmw & nbit);
        if (LAM)
            ldg_keep_if(lr[K % ND], lb + CN * NB, nmw & nbit);
#else
        if (NBP != 1)
            ldg_keep_if(hr[K % ND], hb + CN * NB, 1u);
        if (LAM)
            ldg_keep_if(lr[K % ND], lb + CN * NB, 1u);
#endif
    }
#if PD_NLU_PFD > 0
    // L2 prefetch PD_NLU_PFD slots ahead (no register): the ring load then
    // waits on L2, not HBM
    if constexpr (K + PD_NLU_PFD < NPAT) {
        constexpr int CP = kOrder.slot[K + PD_NLU_PFD];
        if (NBP != 1)
            prefetch_l2(hb + CP * NB);
        if (LAM)
            prefetch_l2(lb + CP * NB);
    }
#endif
    const float4 rj = own[off];
    float s, a, cz;
    float2 cxy;
    stretch_c<dx, dy, dz>(rj, ri, s, a, cxy, cz);
    // breakable: live and neither end no-failure (nfthr = +inf for a
    // no-failure node; rj.w < 0 for a no-failure neighbour)
    const bool brk_ok = live && (!NF || rj.w >= nfthr);
    float e;
    float f;
    if (NBP == 0) {
        f = nl_law_typed(p0, p1, s, hh, e);
        if (NF && !brk_ok)
            f = p0.x * s;
        stg_typed_if<NF>(hb + C * NB, mw & bit, rj.w, nfthr, p0.w, s, hh,
                         (__float_as_uint(s) & ~7u) | ty);
        if (brk_ok)  // e >= s_c of the bond's own law <=> e - |s_c| >= 0 (exact sign)
            acc.emax = fmax_nan(acc.emax, e - fabsf(p0.w));
    } else {
        f = nl_law<NBP>(R, s, hh, e);
        if (NF && !brk_ok)
            f = R.c * s;
        if (NBP > 1)
            stg_hist_if<NF>(hb + C * NB, mw & bit, rj.w, nfthr, s, hh);
        if (brk_ok)
            acc.emax = fmax_nan(acc.emax, e);
    }
    float scale = f * a;
    if (NF)
        scale *= fabsf(rj.w);
    if (LAM)
        scale *= lam;
    if (live) {
        acc.gxy = __ffma2_rn(cxy, make_float2(scale, scale), acc.gxy);
        acc.gz = fmaf(cz, scale, acc.gz);
    }
    if constexpr (kOrder.last[K]) {
        constexpr float len = root(dx * dx + dy * dy + dz * dz);
        acc.fxy = __ffma2_rn(acc.gxy, make_float2(len, len), acc.fxy);
        acc.fz = fmaf(acc.gz, len, acc.fz);
        acc.gxy = make_float2(0.f, 0.f);
        acc.gz = 0.f;
    }
}

template <int K, int NBP, bool LAM, int NB>
__device__ __forceinline__ void nl_ring_one(const float* hb, const float* lb, float (&hr)[ND],
                                            float (&lr)[ND]) {
    constexpr int C = kOrder.slot[K];
    hr[K] = NBP != 1 ? hb[C * NB] : 0.f;
    lr[K] = LAM ? __ldcs(lb + C * NB) : 1.f;
}

template <int NBP, bool LAM, int NB, int... K>
__device__ __forceinline__ void nl_ring_init(std::integer_sequence<int, K...>, const float* hb,
                                             const float* lb, float (&hr)[ND], float (&lr)[ND]) {
    (nl_ring_one<K, NBP, LAM, NB>(hb, lb, hr, lr), ...);
}

template <int NBP, bool LAM, bool NF, int NB, int... K>
__device__ __forceinline__ void nl_all_slots(std::integer_sequence<int, K...>, const float4* own,
                                             const float4& ri, const uint4& m, float* hb,
                                             const float* lb, float nfthr, const NlRegLaw& R,
                                             const float4* tab, float (&hr)[ND], float (&lr)[ND],
                                             AccN& acc) {
    (nl_slot<K, NBP, LAM, NF, NB>(own, ri, m, hb, lb, nfthr, R, tab, hr, lr, acc), ...);
}

// the rare pass for a node that loses bonds: the history is already updated,
// which leaves e and f of every slot unchanged (e = max(s, h_old) = max(s, h_new))
template <int NBP, bool LAM, bool NF, int NB>
__device__ __forceinline__ uint4 nl_slow_node(const LatticeArgs& L, const float4* own,
                                              const float4 ri, const uint4 m, const float* hb,
                                              const float* lb, float nfthr, const NlRegLaw& R,
                                              const float4* tab, float sc, float3& fo) {
    unsigned dead[4] = {0u, 0u, 0u, 0u};
    const unsigned w[4] = {m.x, m.y, m.z, m.w};
    float fx = 0.f, fy = 0.f, fz = 0.f;
#pragma unroll 1
    for (int c = 0; c < NPAT; ++c) {
        if (!((w[c >> 5] >> (c & 31)) & 1u))
            continue;
        const int dx = L.pat[c][0], dy = L.pat[c][1], dz = L.pat[c][2];
        const float4 rj = own[dx + HX * (dy + HY * dz)];
        float a;
        const float s = stretch_r(rj, ri, dx, dy, dz, a);
        // collapsed (|xi + eta| = 0 or below fp32's normal range, a = +inf):
        // the reference's s = -1 updates no history, never breaks and adds 0
        // (engine.cpp:61-65, 88-101); the unrolled pass stored no history for
        // it either (NaN > h is false)
        if (a == __int_as_float(0x7f800000))
            continue;
        const bool brk_ok = !NF || rj.w >= nfthr;
        float e, f, c_lin = R.c, s_c = sc;
        if (NBP == 0) {
            const unsigned bits = __float_as_uint(hb[c * NB]);
            const float4 p0 = tab[2 * (bits & 7u)], p1 = tab[2 * (bits & 7u) + 1];
            const float hh = p0.w > 0.f ? __uint_as_float(bits & ~7u) : 0.f;
            f = nl_law_typed(p0, p1, s, hh, e);
            c_lin = p0.x;
            s_c = fabsf(p0.w);
        } else {
            f = nl_law<NBP>(R, s, NBP > 1 ? hb[c * NB] : 0.f, e);
        }
        if (brk_ok && !(e < s_c)) {
            dead[c >> 5] |= 1u << (c & 31);
            continue;
        }
        if (!brk_ok)
            f = c_lin * s;
        float scale = f * a * sqrtf(float(L.pat[c][3]));  // |d| (= root(r2), correctly rounded)
        if (NF)
            scale *= fabsf(rj.w);
        if (LAM)
            scale *= lb[c * NB];
        fx = fmaf(rj.x - ri.x + float(dx), scale, fx);
        fy = fmaf(rj.y - ri.y + float(dy), scale, fy);
        fz = fmaf(rj.z - ri.z + float(dz), scale, fz);
    }
    fo = make_float3(fx, fy, fz);
    return make_uint4(dead[0], dead[1], dead[2], dead[3]);
}

template <int MODE, bool BC, int NBP, bool LAM, bool NF, int BZT>
__global__ void __launch_bounds__(BX * BY * BZT, 16 / BZT) lattice_nlu_kernel(DevArgs A,
                                                                              LatticeArgs L) {
    constexpr int NB = BX * BY * BZT;  // nodes of the brick: the per-bond slot stride
    constexpr long long kBrickSlots = (long long)NPAT * NB;
    if (MODE != 0 && *(volatile long long*)A.err_step != kNoError)
        return;
    extern __shared__ float4 rec[];
    const int gx0 = blockIdx.x * BX, gy0 = blockIdx.y * BY, gz0 = L.z0 + blockIdx.z * BZT;
    const int tx = threadIdx.x % BX, ty = (threadIdx.x / BX) % BY, tz = threadIdx.x / (BX * BY);
    const int gx = gx0 + tx, gy = gy0 + ty, gz = gz0 + tz;
    const bool active = gx < L.nx && gy < L.ny && gz < L.z0 + L.nz_own;
    const long long plane = (long long)L.nx * L.ny;
    const long long i = gx + (long long)L.nx * gy + plane * gz;
    const uint4 m = active ? __ldcs(L.mask + i) : make_uint4(0, 0, 0, 0);
    const long long sb = (blockIdx.x + (long long)gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z)) *
                             kBrickSlots + threadIdx.x;  // == slot_base(L, i)
    float* hb = NBP != 1 ? L.hist + sb : nullptr;
    __shared__ float4 tab[2 * 8];  // typed: per-type law lines (LatticeArgs::tl)
    if (NBP == 0 && threadIdx.x < 2 * 8)
        tab[threadIdx.x] = L.tl[threadIdx.x];
    const float* lb = LAM ? L.lam + sb : nullptr;
    // Opt-in (PD_NLU_PF=1): the brick's per-bond streams are contiguous
    // (kBrickSlots values), so one thread can ask L2 for all of them up front.
    // Measured slower than the per-slot prefetch below.
    if (L.prefetch && threadIdx.x == 0) {
        const long long base = sb - threadIdx.x;
        if (NBP != 1)
            bulk_prefetch_l2(L.hist + base, unsigned(kBrickSlots * sizeof(float)));
        if (LAM)
            bulk_prefetch_l2(L.lam + base, unsigned(kBrickSlots * sizeof(float)));
    }
    // the first ring of streamed values is in flight while the halo is staged
    float hr[ND], lr[ND];
    nl_ring_init<NBP, LAM, NB>(std::make_integer_sequence<int, ND>{}, hb, lb, hr, lr);
    const double4 U0 = A.u_in[gx0 + (long long)L.nx * gy0 + plane * gz0];
    stage_box<BZT, NF>(A, L, rec, gx0, gy0, gz0, U0);
    __syncthreads();
    if (!active)
        return;

    const float4* own = rec + (tx + 3) + HX * ((ty + 3) + HY * (tz + 3));
    const float4 ri = *own;
    const float inf = __int_as_float(0x7f800000);
    const float nfthr = (NF && ri.w < 0.f) ? inf : 0.f;
    const NlRegLaw& R = L.rl;
    AccN acc{make_float2(0.f, 0.f), 0.f, make_float2(0.f, 0.f), 0.f, -inf};
    nl_all_slots<NBP, LAM, NF, NB>(std::make_integer_sequence<int, NPAT>{}, own, ri, m, hb, lb,
                               nfthr, R, tab, hr, lr, acc);
    // a live bond breaks (or overflowed), or a collapsed bond made the force NaN
    if (!(acc.emax < (NBP == 0 ? 0.f : R.sc)) || isnan(acc.fxy.x + acc.fxy.y + acc.fz)) {
        asm volatile("" ::: "memory");  // after this node's history stores
        float3 f;
        const uint4 d = nl_slow_node<NBP, LAM, NF, NB>(L, own, ri, m, hb, lb, nfthr, R, tab, R.sc, f);
        L.mask[i] = make_uint4(m.x & ~d.x, m.y & ~d.y, m.z & ~d.z, m.w & ~d.w);
        A.n_neigh[i] -= __popc(d.x) + __popc(d.y) + __popc(d.z) + __popc(d.w);
        acc.fxy = make_float2(f.x, f.y);
        acc.fz = f.z;
    }
    const double Fx = double(acc.fxy.x * L.cv), Fy = double(acc.fxy.y * L.cv),
                 Fz = double(acc.fz * L.cv);
    if (MODE == 0) {
        A.body_force[3 * i] = Fx;
        A.body_force[3 * i + 1] = Fy;
        A.body_force[3 * i + 2] = Fz;
        return;
    }
    node_epilogue<MODE, BC>(A, i, A.u_in[i], Fx, Fy, Fz);
}

template <int MODE, bool BC, int NBP, bool LAM, bool NF, int BZT>
cudaError_t launch_nlu6(const DevArgs& A, const LatticeArgs& L, cudaStream_t st) {
    const int nbx = (L.nx + BX - 1) / BX, nby = (L.ny + BY - 1) / BY,
              nbz = (L.nz_own + BZT - 1) / BZT;
    if (nbx * nby * nbz == 0)
        return cudaSuccess;
    const int smem = int(sizeof(float4)) * nrec<BZT>();
    const cudaError_t e = smem_optin<lattice_nlu_kernel<MODE, BC, NBP, LAM, NF, BZT>>(smem);
    if (e != cudaSuccess)
        return e;
    t_last_kernel = kernel_name<3, MODE, BC, NBP, LAM, NF, BZT>("lattice_nlu_kernel");
    lattice_nlu_kernel<MODE, BC, NBP, LAM, NF, BZT>
        <<<dim3(unsigned(nbx), unsigned(nby), unsigned(nbz)), BX * BY * BZT, smem, st>>>(A, L);
    return cudaGetLastError();
}

// the brick depth of the per-bond layout (L.nlbz, fixed at upload)
template <int MODE, bool BC, int NBP, bool LAM, bool NF>
cudaError_t launch_nlu5(const DevArgs& A, const LatticeArgs& L, cudaStream_t st) {
    return L.nlbz == 4 ? launch_nlu6<MODE, BC, NBP, LAM, NF, 4>(A, L, st)
                       : launch_nlu6<MODE, BC, NBP, LAM, NF, 8>(A, L, st);
}

template <int MODE, bool BC, int NBP>
cudaError_t launch_nlu3(const DevArgs& A, const LatticeArgs& L, cudaStream_t st) {
    if (L.lam)
        return L.nf ? launch_nlu5<MODE, BC, NBP, true, true>(A, L, st)
                    : launch_nlu5<MODE, BC, NBP, true, false>(A, L, st);
    return L.nf ? launch_nlu5<MODE, BC, NBP, false, true>(A, L, st)
                : launch_nlu5<MODE, BC, NBP, false, false>(A, L, st);
}

// one register law: NBP = 1 (no history) or 3 (two breakpoints: the third
// segment repeats the second)
// ... or several laws by bond type (NBP = 0, L.typed)
template <int MODE> cudaError_t launch_nlu_impl(const DevArgs& A, const LatticeArgs& L,
                                                cudaStream_t st) {
    if (A.bc_kind)
        return L.typed         ? launch_nlu3<MODE, true, 0>(A, L, st)
               : L.rl.nbp == 1 ? launch_nlu3<MODE, true, 1>(A, L, st)
                               : launch_nlu3<MODE, true, 3>(A, L, st);
    return L.typed         ? launch_nlu3<MODE, false, 0>(A, L, st)
           : L.rl.nbp == 1 ? launch_nlu3<MODE, false, 1>(A, L, st)
                           : launch_nlu3<MODE, false, 3>(A, L, st);
}

template <auto Kernel, int BZT> void nlu_preload_fn() {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, reinterpret_cast<const void*>(Kernel));
    smem_optin<Kernel>(int(sizeof(float4)) * nrec<BZT>());
}

template <int MODE, bool BC, int NBP> void preload_nlu3() {
    nlu_preload_fn<lattice_nlu_kernel<MODE, BC, NBP, true, true, 4>, 4>();
    nlu_preload_fn<lattice_nlu_kernel<MODE, BC, NBP, true, true, 8>, 8>();
    nlu_preload_fn<lattice_nlu_kernel<MODE, BC, NBP, true, false, 4>, 4>();
    nlu_preload_fn<lattice_nlu_kernel<MODE, BC, NBP, true, false, 8>, 8>();
    nlu_preload_fn<lattice_nlu_kernel<MODE, BC, NBP, false, true, 4>, 4>();
    nlu_preload_fn<lattice_nlu_kernel<MODE, BC, NBP, false, true, 8>, 8>();
    nlu_preload_fn<lattice_nlu_kernel<MODE, BC, NBP, false, false, 4>, 4>();
    nlu_preload_fn<lattice_nlu_kernel<MODE, BC, NBP, false, false, 8>, 8>();
}

template <int MODE> void preload_nlu_impl() {
    preload_nlu3<MODE, true, 0>();
    preload_nlu3<MODE, false, 0>();
    preload_nlu3<MODE, true, 1>();
    preload_nlu3<MODE, true, 3>();
    preload_nlu3<MODE, false, 1>();
    preload_nlu3<MODE, false, 3>();
}

} // namespace
} // namespace pdb
