// pd_lattice.cu -- the fast path on structured lattices (grid_coordinates,
// geometry.cpp:25-38): implicit connectivity.
//
// On a lattice every family row is a subset of ONE neighbour pattern: the
// integer offsets d with 0 < |d|^2 <= 9 (122 offsets; delta / spacing in
// [3, sqrt 10), which covers the reference's delta = 3 dx and pi dx), in the
// rows' own ascending-index order (dz, dy, dx).  So a row is stored as a
// 128-bit mask over that pattern (bit c = "offset c is a live bond"; a break
// clears the bit, like writing -1 into entries, engine.cpp:93-96) and the
// neighbour of slot c is found by address arithmetic, not by an index load:
//
//   * a CTA owns a brick of 16 x 4 x 8 lattice nodes (one thread each) and
//     stages the displacement of its 22 x 10 x 14 halo box into shared memory
//     once per step as fp32 (u - U_brick) / spacing -- 16 B per record, read
//     with one conflict-free LDS.128 per slot at a compile-time offset;
//   * xi = d (in spacings) and |xi|, 1/|xi| are compile-time constants of the
//     fully unrolled slot sequence, so only eta is arithmetic:
//       s = eta.(2d + eta) / (|d| (|d + eta| + |d|))   (cancellation free)
//     with MUFU rsqrt / rcp, exactly as the general fast path;
//   * the integrator epilogue is the shared fp64 node_epilogue.
// HBM per step: the 16-byte mask (read; written only on a break) plus the
// node arrays -- no per-bond index stream at all.
//
// Used for KernelVariant fast when the model is a lattice with one PMB law,
// uniform volumes and no per-bond data (pd_host.cu decides); everything else
// takes the general tile layout (pd_fast.cu).
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <utility>
#include <vector>
#include <algorithm>

#include "pd_device.cuh"
#include "pd_fast.cuh"
#include "pd_internal.h"
#include "pd_lattice.cuh"

namespace pdb {

namespace {
struct Acc {
    float2 gxy;  // sum over the current length class of c * s / (|c| |d|), x and y lanes
    float gz;
    float2 fxy;  // sum over finished classes (times |d|): the node's force / (c V)
    float fz;
    float smax;  // largest stretch over the live breakable slots
};

// NF (no-failure nodes and/or per-node volumes present): a record's w holds
// V_j / V_0, negated for a no-failure node; the bond never breaks when either
// end is no-failure (engine.cpp:79-80, 86-88: the node's own flag lifts s_c
// to +inf) and its force carries V_j (engine.cpp:103).
template <int K, bool NF>
__device__ __forceinline__ void slot(const float4* own, const float4& ri, const uint4& m, Acc& acc) {
    constexpr int C = kOrder.slot[K];
    constexpr int dx = pat(C, 0), dy = pat(C, 1), dz = pat(C, 2);
    constexpr int off = dx + HX * (dy + HY * dz);
    constexpr int word = C >> 5;
    constexpr unsigned bit = 1u << (C & 31);
    const unsigned mw = word == 0 ? m.x : (word == 1 ? m.y : (word == 2 ? m.z : m.w));
    // branch free: a dead slot's record may be anything finite (an
    // out-of-domain box record is 0); its contribution is predicated away
    const float4 rj = own[off];
    float s, a, cz;
    float2 cxy;
    stretch_c<dx, dy, dz>(rj, ri, s, a, cxy, cz);
    // Every live slot adds its force and raises smax; a live slot that
    // breaks (s >= s_c, bond_contribution's PMB test, engine.cpp:90-98) makes
    // smax >= s_c, and the node is then recomputed without its broken bonds
    // (slow_node) -- so the common no-break slot has no break test at all.
    // A no-failure neighbour's bond (NF: rj.w < 0) never breaks: no smax.
    const bool live = (mw & bit) != 0u;
    const float scale = NF ? s * a * fabsf(rj.w) : s * a;
    if (live) {
        acc.gxy = __ffma2_rn(cxy, make_float2(scale, scale), acc.gxy);
        acc.gz = fmaf(cz, scale, acc.gz);
        if (!NF || rj.w >= 0.f)
            acc.smax = fmax_nan(acc.smax, s);
    }
    if constexpr (kOrder.last[K]) {  // close the class: times |d|
        constexpr float len = root(dx * dx + dy * dy + dz * dz);
        acc.fxy = __ffma2_rn(acc.gxy, make_float2(len, len), acc.fxy);
        acc.fz = fmaf(acc.gz, len, acc.fz);
        acc.gxy = make_float2(0.f, 0.f);
        acc.gz = 0.f;
    }
}

__constant__ signed char c_pat[NPAT][4];  // dx, dy, dz, |d|^2
__constant__ signed char c_slot[343];     // (dz+3)*49 + (dy+3)*7 + (dx+3) -> slot, -1 outside
__constant__ float c_len[NPAT];           // |d|


// The rare pass for a node that loses bonds this step: recompute each live
// slot's stretch (the unrolled slots' arithmetic, so the same s), return the
// broken bits and the force of the slots that stay.
// (Inlined: a noinline call would pass m and ri through the stack, a local
// store on every node.)
template <bool NF>
__device__ __forceinline__ uint4 slow_node(const float4* own, const float4 ri, const uint4 m,
                                           float sc, float3& f) {
    unsigned w[4] = {m.x, m.y, m.z, m.w};
    unsigned dead[4] = {0u, 0u, 0u, 0u};
    float fx = 0.f, fy = 0.f, fz = 0.f;
#pragma unroll 1
    for (int c = 0; c < NPAT; ++c) {
        if (!((w[c >> 5] >> (c & 31)) & 1u))
            continue;
        const int dx = c_pat[c][0], dy = c_pat[c][1], dz = c_pat[c][2];
        const float4 rj = own[dx + HX * (dy + HY * dz)];
        float a;
        const float s = stretch_r(rj, ri, dx, dy, dz, a);
        // a collapsed bond (|xi + eta| = 0, or below fp32's normal range: the
        // approximate rsqrt flushes it and a = +inf) keeps its bit and adds
        // nothing: the reference's stretch is -1 < s_c there and its
        // contribution 0 (engine.cpp:61-65, 100-101)
        if (a == __int_as_float(0x7f800000))
            continue;
        if (!(s < sc) && !(rj.w < 0.f)) {  // a no-failure neighbour keeps the bond
            dead[c >> 5] |= 1u << (c & 31);
            continue;
        }
        const float scale = s * a * (NF ? fabsf(rj.w) : 1.f) * c_len[c];
        fx = fmaf(rj.x - ri.x + float(dx), scale, fx);
        fy = fmaf(rj.y - ri.y + float(dy), scale, fy);
        fz = fmaf(rj.z - ri.z + float(dz), scale, fz);
    }
    f = make_float3(fx, fy, fz);
    return make_uint4(dead[0], dead[1], dead[2], dead[3]);
}

template <bool NF, int... K>
__device__ __forceinline__ void all_slots(std::integer_sequence<int, K...>, const float4* own,
                                          const float4& ri, const uint4& m, Acc& a) {
    (slot<K, NF>(own, ri, m, a), ...);
}


template <int MODE, int BZT, int MINB, bool BC, bool NF>
__global__ void __launch_bounds__(BX * BY * BZT, MINB) lattice_step_kernel(DevArgs A,
                                                                           LatticeArgs L) {
    constexpr int TT = BX * BY * BZT, HZ = BZT + 6;
    if (MODE != 0 && *(volatile long long*)A.err_step != kNoError)
        return;
    extern __shared__ float4 rec[];  // HX * HY * HZ records (dynamic: > 48 KB for BZT = 8)
    // grid = (bricks in x, bricks in y, bricks in z over the owned planes)
    const int gx0 = blockIdx.x * BX, gy0 = blockIdx.y * BY, gz0 = L.z0 + blockIdx.z * BZT;
    const int tx = threadIdx.x % BX, ty = (threadIdx.x / BX) % BY, tz = threadIdx.x / (BX * BY);
    const int gx = gx0 + tx, gy = gy0 + ty, gz = gz0 + tz;
    const bool active = gx < L.nx && gy < L.ny && gz < L.z0 + L.nz_own;
    const long long plane = (long long)L.nx * L.ny;
    const long long i = gx + (long long)L.nx * gy + plane * gz;
    // the row mask streams in while the halo is staged
    uint4 m = active ? __ldcs(L.mask + i) : make_uint4(0, 0, 0, 0);

    // 1. stage the halo box
    const double4 U0 = A.u_in[gx0 + (long long)L.nx * gy0 + plane * gz0];
    stage_box<BZT, NF>(A, L, rec, gx0, gy0, gz0, U0);
    __syncthreads();
    if (!active)
        return;

    // 2. the node's bonds: 122 pattern slots, unrolled at compile time
    const float4* own = rec + (tx + 3) + HX * ((ty + 3) + HY * (tz + 3));  // HY pitch is the same
    const float4 ri = *own;
    // a no-failure node's own bonds never break
    const float sc = (NF && ri.w < 0.f) ? __int_as_float(0x7f800000) : L.sc;
    Acc a{make_float2(0.f, 0.f), 0.f, make_float2(0.f, 0.f), 0.f, -__int_as_float(0x7f800000)};
    all_slots<NF>(std::make_integer_sequence<int, NPAT>{}, own, ri, m, a);
    // some live bond breaks this step (or its stretch overflowed), or a
    // collapsed bond (|xi + eta| = 0: NaN stretch) made the force NaN -- rare
    // cases, recomputed slot by slot with the reference's semantics
    if (!(a.smax < sc) || isnan(a.fxy.x + a.fxy.y + a.fz)) {
        float3 f;
        const uint4 d = slow_node<NF>(own, ri, m, sc, f);
        L.mask[i] = make_uint4(m.x & ~d.x, m.y & ~d.y, m.z & ~d.z, m.w & ~d.w);
        A.n_neigh[i] -= __popc(d.x) + __popc(d.y) + __popc(d.z) + __popc(d.w);
        a.fxy = make_float2(f.x, f.y);
        a.fz = f.z;
    }
    const double fx = double(a.fxy.x * L.cv), fy = double(a.fxy.y * L.cv), fz = double(a.fz * L.cv);

    // 3. fp64 epilogue
    if (MODE == 0) {
        A.body_force[3 * i] = fx;
        A.body_force[3 * i + 1] = fy;
        A.body_force[3 * i + 2] = fz;
        return;
    }
    node_epilogue<MODE, BC>(A, i, A.u_in[i], fx, fy, fz);
}

// ---- small models: one persistent launch for a run of steps -------------------
//
// A model of a few thousand nodes (cfg1's 9,800-node beam) is a latency chain,
// not a throughput problem: one thread per node walking 122 slots, a fresh
// launch every step (profiles/r02_small_cfg1_ncu.md).  Here one cooperative
// launch advances all the steps between two host events (write steps,
// snapshots, the end of the run):
//   * a CTA owns an SBX x 4 x 1 brick; each node's 122 slots are split over
//     SPN = 8 warps, one per half of a 32-bit word of the row mask (4 with
//     16-wide bricks: a word each; warp w runs part w % SPN, so the warps of
//     one part share a scheduler);
//   * each word is walked as a rolled loop over the slots some lane of the
//     warp still has (rolled_word): a few hundred bytes of code, so the
//     kernel stays in the SM's instruction cache (the unrolled slot parts,
//     55 KB, streamed from L2 every step and measured no faster);
//   * the words' forces meet in shared memory and are summed in word order
//     (deterministic) by the node's word-0 thread, which keeps u, v, a and
//     1/rho of its node in registers (the boundary conditions in shared
//     memory) across the steps and runs the shared fp64 epilogue
//     (node_epilogue) exactly as the one-step kernels do;
//   * steps are separated by a grid barrier: an arrival counter in global
//     memory (release add, acquire poll); u written by other CTAs is read
//     with ld.global.cg, so no stale L1 line survives a step.
// Co-residency is guaranteed by cudaLaunchCooperativeKernel; the host takes
// this path only when the grid fits (lattice_small_fits).  A barrier that
// never completes (impossible under a cooperative launch) ends the run after
// a timeout with kBarrierTimeout instead of hanging the device.
constexpr int kSmallMaxRamps = 32;  // ramp table of the small kernel (one per lane of a warp)

inline int sm_count_small() {
    static const int n = [] {
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        return cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0
                   ? v
                   : 148;
    }();
    return n;
}

// The rolled walk of one mask word (slots 32 word .. 32 word + 31): only the
// slots some lane of the warp still has (a warp-uniform bit loop, four slots
// per iteration for ILP), each with bond_contribution's break test directly
// (engine.cpp:90-98) -- no re-walk -- and slow_node's semantics for collapsed
// and no-failure bonds.
struct SlotGeo {
    float4 d;  // dx, dy, dz, |d|^2
    float4 e;  // |d|^4, |d|, record offset in the staged box (int bits), 0
};

template <bool NF>
__device__ __forceinline__ void rolled_word(const float4* own, const float4& ri, unsigned mw, int gbase,
                                            float sc, const SlotGeo* geo, float3& f, unsigned& dead) {
    unsigned todo = __reduce_or_sync(0xffffffffu, mw);
    float fx = 0.f, fy = 0.f, fz = 0.f;
    unsigned dd = 0u;
    while (todo) {
        // four slots per iteration, branch free (a missing fourth slot
        // re-reads slot b = 0 and is predicated away), so the scheduler can
        // interleave their dependency chains
        int b[4];
        unsigned v = 0u;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            b[q] = todo != 0u ? __ffs(todo) - 1 : 0;
            v |= (todo != 0u ? 1u : 0u) << q;
            todo &= todo - 1u;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const SlotGeo g = geo[gbase + b[q]];
            const float4 rj = own[__float_as_int(g.e.z)];
            // stretch_c's arithmetic with the offset from the table
            const float2 dxy = make_float2(g.d.x, g.d.y);
            const float2 hxy = __fadd2_rn(make_float2(rj.x, rj.y), make_float2(-ri.x, -ri.y));
            const float hz = rj.z - ri.z;
            const float2 cxy = __fadd2_rn(hxy, dxy);
            const float2 txy = __fadd2_rn(cxy, dxy);
            const float cz = hz + g.d.z, tz = cz + g.d.z;
            const float2 pxy = __fmul2_rn(hxy, txy);
            float num = __fadd_rn(pxy.x, pxy.y);
            num = fmaf(hz, tz, num);
            const float w = fmaf(num, g.d.w, g.e.x);
            const float a = rsqrt_approx(w);
            const float st = num * rcp_approx(fmaf(w, a, g.d.w));
            // live, and not collapsed (|xi + eta| = 0: a = +inf, kept with no
            // force as in slow_node, engine.cpp:61-65, 100-101)
            const bool live = ((v >> q) & 1u) && ((mw >> b[q]) & 1u) && a != __int_as_float(0x7f800000);
            // breaks unless a no-failure neighbour keeps it
            const bool brk = live && !(st < sc) && !(rj.w < 0.f);
            dd |= brk ? 1u << b[q] : 0u;
            // selected, not multiplied by 0: a dead slot's record may be
            // non-finite (fp32 overflow of a huge displacement)
            const bool use = live && !brk;
            const float scale = st * a * (NF ? fabsf(rj.w) : 1.f) * g.e.y;
            fx = use ? fmaf(cxy.x, scale, fx) : fx;
            fy = use ? fmaf(cxy.y, scale, fy) : fy;
            fz = use ? fmaf(cz, scale, fz) : fz;
        }
    }
    f = make_float3(fx, fy, fz);
    dead = dd;
}

__device__ __forceinline__ double4 ldcg4(const double4* p) {
    const double2 a = __ldcg(reinterpret_cast<const double2*>(p));
    const double2 b = __ldcg(reinterpret_cast<const double2*>(p) + 1);
    return make_double4(a.x, a.y, b.x, b.y);
}

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// The gate at the top of step s (= the launch's first step + k).  For k > 0,
// arrive (release: this CTA's u / v / a stores, ordered before thread 0 by
// the CTA barrier, become visible with the count) and wait until the count
// reaches target (acquire: every other CTA's step s - 1 stores are visible).
// Then stop if a step before s saw non-finite u (err_step <= s; a concurrent
// step-s epilogue elsewhere can only write s + 1) or the barrier timed out.
// Thread 0 decides for the whole CTA.
__device__ __forceinline__ bool step_gate(bool wait, unsigned long long* count,
                                          unsigned long long target, long long* err_step,
                                          long long s) {
    __shared__ int go;
    __syncthreads();
    if (threadIdx.x == 0) {
        bool ok = true;
        if (wait) {
            asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(count) : "memory");
            const unsigned long long t0 = globaltimer();
            for (;;) {
                unsigned long long c;
                asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(c) : "l"(count) : "memory");
                if (c >= target)
                    break;
                if (globaltimer() - t0 > 4000000000ull) {  // 4 s: never under a cooperative launch
                    *(volatile long long*)err_step = kBarrierTimeout;
                    ok = false;
                    break;
                }
            }
        }
        go = ok && !(*(volatile long long*)err_step <= s);
    }
    __syncthreads();
    return go != 0;
}

// SPN slot parts per node: 4 (a mask word each) or 8 (half a word each)
template <int MODE, bool BC, bool NF, int SBX, int SPN>
__global__ void __launch_bounds__(SBX * BY * SPN, SPN == 8 ? 3 : 512 / (SBX * BY * SPN))
    lattice_small_kernel(DevArgs A, LatticeArgs L, SmallArgs S) {
    constexpr int NB = SBX * BY;               // nodes per brick
    constexpr int NT = NB * SPN;               // threads
    constexpr int SHX = SBX + 6;               // halo box: SHX x HY x 7
    constexpr int NR = SHX * HY * 7;
    constexpr int NRT = (NR + NT - 1) / NT;    // records staged per thread
    static_assert(NB % 32 == 0, "a warp holds 32 nodes of one brick");
    __shared__ float4 rec[NR];
    __shared__ float4 part_f[SPN - 1][NB];
    __shared__ unsigned part_d[SPN - 1][NB];  // broken bits of the part, relative to its first slot
    __shared__ uint4 smask[NB];
    __shared__ SlotGeo geo[128];
    __shared__ AxisBc sbc[BC ? NB : 1][3];    // the nodes' boundary conditions, loaded once
    // the ramp values of steps k (srv[k & 1]) and k + 1, per ramp (the host
    // takes this kernel only for at most kSmallMaxRamps ramps)
    __shared__ RampVals srv[2][BC ? kSmallMaxRamps : 1];
    __shared__ double4 sU0;                    // the brick origin's u: the staging reference
    const int t = threadIdx.x, wid = t / 32;
    const int p = wid % SPN;                   // the slot part of this warp (warp-uniform)
    const int node = (wid / SPN) * 32 + t % 32;
    const int pword = SPN == 4 ? p : p / 2;    // its mask word
    const int pshift = SPN == 4 ? 0 : 16 * (p % 2);
    if (t < 128) {
        SlotGeo g{};
        if (t < NPAT) {
            const int dx = c_pat[t][0], dy = c_pat[t][1], dz = c_pat[t][2], r2 = c_pat[t][3];
            g.d = make_float4(float(dx), float(dy), float(dz), float(r2));
            g.e = make_float4(float(r2 * r2), c_len[t], __int_as_float(dx + SHX * (dy + HY * dz)), 0.f);
        }
        geo[t] = g;
    }
    const int tx = node % SBX, ty = node / SBX;
    const int gx0 = blockIdx.x * SBX, gy0 = blockIdx.y * BY, gz0 = L.z0 + blockIdx.z;
    const int gx = gx0 + tx, gy = gy0 + ty;
    const bool active = gx < L.nx && gy < L.ny;
    const long long plane = (long long)L.nx * L.ny;
    const long long i = gx + (long long)L.nx * gy + plane * gz0;
    // the node's state only its word-0 thread touches stays in registers
    // across the steps: u, v, a, 1/rho (and the BCs in shared memory)
    NodeIn nin{};
    double4 ui = make_double4(0.0, 0.0, 0.0, 0.0);
    if (p == 0) {
        smask[node] = active ? L.mask[i] : make_uint4(0, 0, 0, 0);
        if (active) {
            nin = load_node_in(A, i);
            ui = ldcg4(S.u[0] + i);
            if (BC)
                for (int ax = 0; ax < 3; ++ax)
                    sbc[node][ax] = load_axis_bc(A, i, ax);
        }
        if (node == 0)
            sU0 = ui;  // node 0 of a brick is always inside the lattice
    }
    if (BC && wid == 1 && t % 32 < S.n_ramps)  // step 0's ramp values (read after the first gate)
        srv[0][t % 32] = ramp_vals(A.ramps[t % 32], A.step);
    const unsigned long long nblocks = (unsigned long long)gridDim.x * gridDim.y * gridDim.z;
    const float ih = float(L.inv_h);
    // the records this thread stages: their source node and (NF) the constant
    // signed volume ratio, computed once
    // (-1: a record outside the lattice, staged as 0; measured faster than
    // branch-free loads of a clamped neighbour, which load every record)
    long long src[NRT];
    float wv[NRT];
#pragma unroll
    for (int q = 0; q < NRT; ++q) {
        const int r = t + q * NT;
        const int pz = r / (SHX * HY), rr = r % (SHX * HY);
        const int X = gx0 - 3 + rr % SHX, Y = gy0 - 3 + rr / SHX, Z = gz0 - 3 + pz;
        const bool ok = r < NR && X >= 0 && X < L.nx && Y >= 0 && Y < L.ny && Z >= 0 && Z < L.nz_local;
        src[q] = ok ? X + (long long)L.nx * Y + plane * Z : -1;
        wv[q] = 0.f;
        if (NF && ok) {
            const float vf = L.vol_varies ? float(A.xv[src[q]].w * L.inv_v0) : 1.f;
            wv[q] = S.u[0][src[q]].w != 0.0 ? -vf : vf;  // the no-failure flag rides in u.w
        }
    }
    double4* const u0 = S.u[0];
    double4* const u1 = S.u[1];
    const float4* own = rec + (tx + 3) + SHX * ((ty + 3) + HY * 3);
#ifdef PD_SMALL_PROF
    long long pc[6] = {0, 0, 0, 0, 0, 0}, pt = clock64();
#define PD_PROF_MARK(q) do { const long long n_ = clock64(); if (k > 0) pc[q] += n_ - pt; pt = n_; } while (0)
#else
#define PD_PROF_MARK(q) do { } while (0)
#endif
    for (int k = 0; k < S.steps; ++k) {
        PD_PROF_MARK(3);
        if (!step_gate(k > 0, S.bar, S.bar_base + nblocks * (unsigned long long)k, A.err_step,
                       A.step + k))
            return;
        PD_PROF_MARK(0);
        const double4* uin = (k & 1) ? u1 : u0;
        double4* uout = (k & 1) ? u0 : u1;
        // every record's load in flight at once (no dependent load: the
        // reference u of the brick origin is already in shared memory)
        const double4 U0 = sU0;
        double2 uxy[NRT];
        double uz[NRT];
#pragma unroll
        for (int q = 0; q < NRT; ++q) {
            uxy[q] = make_double2(0.0, 0.0);
            uz[q] = 0.0;
            if (src[q] >= 0) {
                uxy[q] = __ldcg(reinterpret_cast<const double2*>(uin + src[q]));
                uz[q] = __ldcg(&uin[src[q]].z);
            }
        }
#pragma unroll
        for (int q = 0; q < NRT; ++q) {
            const int r = t + q * NT;
            if (r < NR)
                rec[r] = src[q] >= 0 ? make_float4(float(uxy[q].x - U0.x) * ih, float(uxy[q].y - U0.y) * ih,
                                                   float(uz[q] - U0.z) * ih, wv[q])
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        __syncthreads();
        PD_PROF_MARK(1);
        const float4 ri = *own;
        const uint4 m = smask[node];
        const float sc = (NF && ri.w < 0.f) ? __int_as_float(0x7f800000) : L.sc;
        const unsigned mw = pword == 0 ? m.x : (pword == 1 ? m.y : (pword == 2 ? m.z : m.w));
        float3 f;
        unsigned dw;
        rolled_word<NF>(own, ri, SPN == 4 ? mw : (mw >> pshift) & 0xffffu, 32 * pword + pshift, sc, geo,
                        f, dw);
        if (p > 0) {
            part_f[p - 1][node] = make_float4(f.x, f.y, f.z, 0.f);
            part_d[p - 1][node] = dw;
        }
        __syncthreads();
        PD_PROF_MARK(2);
        if (p != 0 || !active) {
            // warp 1 evaluates the next step's ramps while warp 0 integrates
            if (BC && wid == 1 && t % 32 < S.n_ramps && k + 1 < S.steps)
                srv[(k + 1) & 1][t % 32] = ramp_vals(A.ramps[t % 32], A.step + k + 1);
            continue;
        }
        unsigned dd[4] = {dw, 0u, 0u, 0u};
#pragma unroll
        for (int q = 1; q < SPN; ++q) {  // part order: the same sum every run
            const float4 g = part_f[q - 1][node];
            f.x += g.x;
            f.y += g.y;
            f.z += g.z;
            dd[SPN == 4 ? q : q / 2] |= part_d[q - 1][node] << (SPN == 4 ? 0 : 16 * (q % 2));
        }
        const uint4 dead = make_uint4(dd[0], dd[1], dd[2], dd[3]);
        if (dead.x | dead.y | dead.z | dead.w) {
            const uint4 nm = make_uint4(m.x & ~dead.x, m.y & ~dead.y, m.z & ~dead.z, m.w & ~dead.w);
            smask[node] = nm;
            L.mask[i] = nm;
            A.n_neigh[i] -= __popc(dead.x) + __popc(dead.y) + __popc(dead.z) + __popc(dead.w);
        }
        const double fx = double(f.x * L.cv), fy = double(f.y * L.cv), fz = double(f.z * L.cv);
        PD_PROF_MARK(4);
        DevArgs Ak = A;
        Ak.u_in = uin;
        Ak.u_out = uout;
        Ak.step = A.step + k;
        const bool last = k + 1 == S.steps;
        Ak.store_forces = last ? S.store_last : 0;
        Ak.do_drift = last ? S.drift_last : 1;
        node_epilogue<MODE, BC, true>(Ak, i, ui, fx, fy, fz, nin, BC ? sbc[node] : nullptr, &nin, &ui,
                                      srv[k & 1]);
        PD_PROF_MARK(5);
        if (node == 0)
            sU0 = ui;  // read by the next step's staging, after its gate
    }
#ifdef PD_SMALL_PROF
    if (t == 0 && (blockIdx.x == 0 || blockIdx.x == 2) && blockIdx.y == 0 && blockIdx.z % 4 == 2)
        printf("small prof cta x=%d z=%d steps=%d cycles/step gate %lld stage %lld slots %lld combine %lld "
               "epilogue %lld tail %lld\n",
               blockIdx.x, blockIdx.z, S.steps, pc[0] / (S.steps - 1), pc[1] / (S.steps - 1), pc[2] / (S.steps - 1),
               pc[4] / (S.steps - 1), pc[5] / (S.steps - 1), pc[3] / (S.steps - 1));
#endif
#undef PD_PROF_MARK
}

// Brick width of the small kernel: the per-step critical path is the SM with
// the most CTAs, so take the width with the fewest brick-columns on the
// busiest SM (cfg1's 50 x 14 x 14 beam: 224 16-wide CTAs put two on 76 SMs,
// 392 8-wide ones three on some: 32 vs 24 columns).  PD_SMALL_BX = 8 / 16
// forces one.
inline int small_bx(const LatticeArgs& L) {
    if (const char* e = std::getenv("PD_SMALL_BX")) {
        const int v = std::atoi(e);
        if (v == 8 || v == 16)
            return v;
    }
    const long long sms = sm_count_small();
    long long best = -1;
    int bx = 16;
    for (int w : {16, 8}) {
        const long long ctas = (long long)((L.nx + w - 1) / w) * ((L.ny + BY - 1) / BY) * L.nz_own;
        const long long cost = (ctas + sms - 1) / sms * w;
        if (best < 0 || cost < best) {
            best = cost;
            bx = w;
        }
    }
    return bx;
}

// Slot parts per node: 8 (half a mask word per warp) with 8-wide bricks,
// else 4.  PD_SMALL_P = 4 / 8 forces one (8 only with 8-wide bricks).
inline int small_parts(int bx) {
    if (const char* e = std::getenv("PD_SMALL_P")) {
        const int v = std::atoi(e);
        if (v == 4 || (v == 8 && bx == 8))
            return v;
    }
    return bx == 8 ? 8 : 4;
}

template <int MODE, bool BC, bool NF, int SBX, int SPN>
cudaError_t launch_small_w(const DevArgs& A, const LatticeArgs& L, const SmallArgs& S, cudaStream_t st) {
    const dim3 grid{unsigned((L.nx + SBX - 1) / SBX), unsigned((L.ny + BY - 1) / BY), unsigned(L.nz_own)};
    t_last_kernel = kernel_name<3, MODE, BC, NF, SBX, SPN>("lattice_small_kernel");
    DevArgs a = A;
    LatticeArgs l = L;
    SmallArgs s = S;
    void* args[] = {&a, &l, &s};
    return cudaLaunchCooperativeKernel(
        reinterpret_cast<const void*>(lattice_small_kernel<MODE, BC, NF, SBX, SPN>), grid,
        dim3(SBX * BY * SPN), args, 0, st);
}

template <int MODE, bool BC, bool NF>
cudaError_t launch_small_t(const DevArgs& A, const LatticeArgs& L, const SmallArgs& S, cudaStream_t st) {
    const int bx = small_bx(L);
    if (bx == 16)
        return launch_small_w<MODE, BC, NF, 16, 4>(A, L, S, st);
    return small_parts(8) == 8 ? launch_small_w<MODE, BC, NF, 8, 8>(A, L, S, st)
                               : launch_small_w<MODE, BC, NF, 8, 4>(A, L, S, st);
}

template <auto Kernel> int occupancy(int threads) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, Kernel, threads, 0) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return per_sm;
}

template <int MODE, bool BC, bool NF> int small_capacity(int bx) {
    if (bx == 16)
        return occupancy<lattice_small_kernel<MODE, BC, NF, 16, 4>>(16 * BY * 4);
    return small_parts(8) == 8 ? occupancy<lattice_small_kernel<MODE, BC, NF, 8, 8>>(8 * BY * 8)
                               : occupancy<lattice_small_kernel<MODE, BC, NF, 8, 4>>(8 * BY * 4);
}

template <int MODE> int small_capacity_mode(bool bc, bool nf, int bx) {
    return bc ? (nf ? small_capacity<MODE, true, true>(bx) : small_capacity<MODE, true, false>(bx))
              : (nf ? small_capacity<MODE, false, true>(bx) : small_capacity<MODE, false, false>(bx));
}

template <int MODE>
cudaError_t launch_small_mode(const DevArgs& A, const LatticeArgs& L, const SmallArgs& S, cudaStream_t st) {
    if (L.nf)
        return A.bc_kind ? launch_small_t<MODE, true, true>(A, L, S, st)
                         : launch_small_t<MODE, false, true>(A, L, S, st);
    return A.bc_kind ? launch_small_t<MODE, true, false>(A, L, S, st)
                     : launch_small_t<MODE, false, false>(A, L, S, st);
}

// ---- n-linear laws, bond types, lambda / beta on the lattice (NL) -------------
//
// The general NL kernel (more than 8 laws or more than 3 breakpoints; the
// unrolled kernels of pd_lattice_nlu.cuh take every other n-linear model).
// The per-bond data live in the brick-major arrays (pd_lattice.cuh
// slot_base): fp32 stretch history, u8 bond type, fp32 lambda * beta.  The
// slot loop is a runtime loop with the laws in constant memory.  Semantics are
// bond_contribution's (engine.cpp:53-109), in fp32 like the tile kernel.

__constant__ FastLaw c_llaws[PD_MAX_LAWS];
// per slot (padded to 128; slots 122..127 never have a mask bit):
// (dx, dy, dz, |d|^2), (|d|, 1/|d|) and the box record offset
__constant__ float4 c_geo[128];
__constant__ float2 c_geo2[128];
__constant__ int c_goff[128];

// envelope_force of the single register law: the same segment arithmetic as
// fast_envelope (f_{k-1} + (e - bp_{k-1}) sl_k), branch free
__device__ __forceinline__ float reg_envelope(const NlRegLaw& R, float e) {
    const bool k1 = e >= R.bp0, k2 = e >= R.bp1;
    const float bs = k2 ? R.bp1 : (k1 ? R.bp0 : 0.f);
    const float bf = k2 ? R.f1 : (k1 ? R.f0 : 0.f);
    const float sl = k2 ? R.sl2 : (k1 ? R.sl1 : R.sl0);
    return bf + (e - bs) * sl;
}

// MULTI = false: one law of at most three breakpoints, held in registers (the
// bond type, if any, can only name it).  MULTI = true: per-bond law from
// constant memory, any number of breakpoints.
template <int MODE, bool BC, bool MULTI, int BZT>
__global__ void __launch_bounds__(BX * BY * BZT, 16 / BZT) lattice_nl_kernel(DevArgs A,
                                                                            LatticeArgs L) {
    constexpr int NLB = BX * BY * BZT;
    constexpr long long kBrickSlots = (long long)NPAT * NLB;
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
    const double4 U0 = A.u_in[gx0 + (long long)L.nx * gy0 + plane * gz0];
    stage_box<BZT, true>(A, L, rec, gx0, gy0, gz0, U0);
    __syncthreads();
    if (!active)
        return;

    const float4* own = rec + (tx + 3) + HX * ((ty + 3) + HY * (tz + 3));
    const float4 ri = *own;
    const bool nfi = ri.w < 0.f;
    const long long sb = (blockIdx.x + (long long)gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z)) *
                             kBrickSlots + threadIdx.x;  // == slot_base(L, i)
    const NlRegLaw R = L.rl;
    float fx = 0.f, fy = 0.f, fz = 0.f;
    unsigned d0 = 0u, d1 = 0u, d2 = 0u, d3 = 0u;
    // groups of 8 slots (never straddling a mask word); the next group's
    // history loads are issued before the current group is evaluated so the
    // history stream keeps several loads in flight per thread
    constexpr int G = 8;
    float* hp = L.hist ? L.hist + sb : nullptr;  // slot c at hp[c * NLB]
    float hnext[G];
#pragma unroll
    for (int q = 0; q < G; ++q)
        hnext[q] = hp ? hp[q * NLB] : 0.f;
#pragma unroll 1
    for (int c0 = 0; c0 < NPAT; c0 += G) {
        float hcur[G];
#pragma unroll
        for (int q = 0; q < G; ++q) {
            hcur[q] = hnext[q];
            hnext[q] = (hp && c0 + G + q < NPAT) ? hp[(c0 + G + q) * NLB] : 0.f;
        }
        const int word = c0 >> 5;
        const unsigned mword = word == 0 ? m.x : (word == 1 ? m.y : (word == 2 ? m.z : m.w));
        const unsigned mw8 = (mword >> (c0 & 31)) & 0xffu;
        if (mw8 == 0u)
            continue;
        const long long sbase = (long long)c0 * NLB + sb;
        float lam[G];  // lambda * beta
        int bt[G];
#pragma unroll
        for (int q = 0; q < G; ++q) {
            const bool ok = ((mw8 >> q) & 1u) != 0u;
            lam[q] = (L.lam && ok) ? L.lam[sbase + q * NLB] : 1.f;
            bt[q] = (MULTI && L.btype && ok) ? int(L.btype[sbase + q * NLB]) : 0;
        }
        unsigned dg = 0u;
#pragma unroll
        for (int q = 0; q < G; ++q) {
            if (!((mw8 >> q) & 1u))
                continue;
            const float4 g1 = c_geo[c0 + q];
            const float2 g2 = c_geo2[c0 + q];
            const float4 rj = own[c_goff[c0 + q]];
            float s, rc, cx, cy, cz;
            stretch(rj, ri, g1.x, g1.y, g1.z, g1.w, g2.x, g2.y, s, rc, cx, cy, cz);
            if (rc == __int_as_float(0x7f800000))
                continue;  // collapsed (|xi + eta| = 0): s = -1 in the reference, no break, 0
            const float hh = hcur[q];
            float f;
            bool brk = false;
            if (MULTI) {
                const FastLaw& law = c_llaws[bt[q]];
                if (nfi || rj.w < 0.f) {
                    f = law.c * s;  // a no-failure end: never breaks, no history
                } else if (law.nbp == 1) {
                    brk = !(s < law.bp[0]);
                    f = law.c * s;
                } else {
                    const float s_c = law.bp[law.nbp - 1];
                    if (s > hh)
                        hp[(c0 + q) * NLB] = s;  // history before the break test (engine.cpp:88-92)
                    brk = hh >= s_c || !(s < s_c);
                    f = (s >= hh) ? fast_envelope(law, s)
                                  : (hh < law.bp[0] ? law.sl[0] : fast_envelope(law, hh) * rcp_approx(hh)) * s;
                }
            } else {
                if (nfi || rj.w < 0.f) {
                    f = R.c * s;
                } else if (!R.hist) {
                    brk = !(s < R.sc);
                    f = R.c * s;
                } else {
                    if (s > hh)
                        hp[(c0 + q) * NLB] = s;
                    const float e = fmaxf(s, hh);
                    brk = !(e < R.sc) || !(s < R.sc);
                    const float env = reg_envelope(R, e);
                    f = (s >= hh) ? env : (hh < R.bp0 ? R.sl0 : env * rcp_approx(hh)) * s;
                }
            }
            if (brk) {
                dg |= 1u << q;
                continue;
            }
            const float scale = f * lam[q] * fabsf(rj.w) * rc;
            fx = fmaf(cx, scale, fx);
            fy = fmaf(cy, scale, fy);
            fz = fmaf(cz, scale, fz);
        }
        if (dg) {
            const unsigned sh = dg << (c0 & 31);
            if (word == 0)
                d0 |= sh;
            else if (word == 1)
                d1 |= sh;
            else if (word == 2)
                d2 |= sh;
            else
                d3 |= sh;
        }
    }
    const int broke = __popc(d0) + __popc(d1) + __popc(d2) + __popc(d3);
    if (broke) {
        L.mask[i] = make_uint4(m.x & ~d0, m.y & ~d1, m.z & ~d2, m.w & ~d3);
        A.n_neigh[i] -= broke;
    }
    const double Fx = double(fx * L.cv), Fy = double(fy * L.cv), Fz = double(fz * L.cv);
    if (MODE == 0) {
        A.body_force[3 * i] = Fx;
        A.body_force[3 * i + 1] = Fy;
        A.body_force[3 * i + 2] = Fz;
        return;
    }
    node_epilogue<MODE, BC>(A, i, A.u_in[i], Fx, Fy, Fz);
}

// row -> mask: bit c set for every live entry whose offset is pattern slot c;
// *bad = 1 when a row holds a bond outside the pattern
__global__ void lattice_coords_kernel(const double4* xv, long long n, LatticeArgs L, int* bad) {
    const long long i = blockIdx.x * 256LL + threadIdx.x;
    if (i >= n)
        return;
    const long long plane = (long long)L.nx * L.ny;
    const double tol = 1e-9 * L.h;
    const double4 x = xv[i];
    if (fabs(x.x - (L.ox + double(i % L.nx) * L.h)) > tol ||
        fabs(x.y - (L.oy + double((i / L.nx) % L.ny) * L.h)) > tol ||
        fabs(x.z - (L.oz + double(i / plane) * L.h)) > tol)
        atomicExch(bad, 1);
}

struct SlotSrc {  // reference-layout per-slot arrays (n x N) to scatter into [c][node]
    const double* hist;
    const uint8_t* btype;
    const double* lambda;
    const double* beta;
};

// One warp per row: lane l reads slots l, l + 32, ... (coalesced), decodes each
// live entry to its pattern slot, scatters the per-bond values to the
// brick-major arrays, and the row's mask is the warp's OR.
__global__ void lattice_mask_kernel(const int32_t* entries, long long begin, long long end, int N,
                                    int nx, int ny, uint4* mask, int* bad, SlotSrc src,
                                    LatticeArgs L) {
    const long long i = begin + (blockIdx.x * 256LL + threadIdx.x) / 32;
    const int lane = threadIdx.x & 31;
    if (i >= end)  // warp-uniform
        return;
    const long long plane = (long long)nx * ny;
    const int ix = int(i % nx), iy = int((i / nx) % ny), iz = int(i / plane);
    // decode d = j - i = dx + nx dy + plane dz by rounding with fp32
    // reciprocals (no integer division per entry): exact whenever |dx|, |dy|
    // <= 3 and nx, ny >= 8 (|dx + nx dy| < plane / 2, |dx| < nx / 2); the
    // decoded offset is then checked against the pattern box and the lattice
    // bounds, so a wrong decode can only flag a row as off-pattern
    const float inv_plane = 1.0f / float(plane), inv_nx = 1.0f / float(nx);
    const bool fast_decode = nx >= 8 && ny >= 8 && plane < (1LL << 22);
    const long long sb = slot_base(L, i);
    unsigned w[4] = {0u, 0u, 0u, 0u};
    bool off = false;
    for (int k = lane; k < N; k += 32) {
        const int32_t j = entries[i * N + k];
        if (j < 0)
            continue;
        int dx, dy, dz;
        if (fast_decode) {
            const long long dl = (long long)j - i;
            const int d = int(max(min(dl, 4 * plane), -4 * plane));
            dz = __float2int_rn(float(d) * inv_plane);
            const int r = d - dz * int(plane);
            dy = __float2int_rn(float(r) * inv_nx);
            dx = r - dy * nx;
            if (dl != d || ix + dx < 0 || ix + dx >= nx || iy + dy < 0 || iy + dy >= ny ||
                iz + dz < 0 || iz + dz >= L.nz_local) {
                off = true;
                continue;
            }
        } else {
            dx = int(j % nx) - ix;
            dy = int((j / nx) % ny) - iy;
            dz = int(j / plane) - iz;
        }
        const int c = (dx < -3 || dx > 3 || dy < -3 || dy > 3 || dz < -3 || dz > 3)
                          ? -1
                          : int(c_slot[(dz + 3) * 49 + (dy + 3) * 7 + (dx + 3)]);
        if (c < 0) {
            off = true;
            continue;
        }
        w[c >> 5] |= 1u << (c & 31);
        const long long sidx = sb + (long long)c * (64 * L.nlbz), idx = i * N + k;
        if (L.typed) {  // history word: fp32 history, bond type in the low 3 bits
            const unsigned h = src.hist ? __float_as_uint(float(src.hist[idx])) & ~7u : 0u;
            L.hist[sidx] = __uint_as_float(h | (src.btype ? unsigned(src.btype[idx]) & 7u : 0u));
        } else if (L.hist && src.hist) {
            L.hist[sidx] = float(src.hist[idx]);
        }
        if (L.btype)
            L.btype[sidx] = src.btype[idx];
        if (L.lam)  // lambda * beta in one stream (engine.cpp:103-107)
            L.lam[sidx] = float((src.lambda ? src.lambda[idx] : 1.0) *
                                (src.beta ? src.beta[idx] : 1.0));
    }
    if (off)
        atomicExch(bad, 1);
    const uint4 m = make_uint4(__reduce_or_sync(0xffffffffu, w[0]), __reduce_or_sync(0xffffffffu, w[1]),
                               __reduce_or_sync(0xffffffffu, w[2]), __reduce_or_sync(0xffffffffu, w[3]));
    if (lane == 0)
        mask[i] = m;
}

// entries in the reference layout: the uploaded row with -1 where the mask bit
// of the slot's offset is clear
__global__ void lattice_materialize_kernel(const int32_t* entries0, const uint4* mask,
                                           long long begin, long long end, long long n, int N,
                                           LatticeArgs L, int32_t* out, double* hist_out) {
    const int nx = L.nx, ny = L.ny;
    const float* hist = L.hist;
    const long long i = blockIdx.x * 256LL + threadIdx.x;
    if (i >= n)
        return;
    const bool owned = i >= begin && i < end;
    const long long plane = (long long)nx * ny;
    const int ix = int(i % nx), iy = int((i / nx) % ny), iz = int(i / plane);
    const uint4 m = owned ? mask[i] : make_uint4(~0u, ~0u, ~0u, ~0u);
    const unsigned w[4] = {m.x, m.y, m.z, m.w};
    for (int k = 0; k < N; ++k) {
        const int32_t j = entries0[i * N + k];
        int32_t v = j;
        if (j >= 0 && owned) {
            const int dx = int(j % nx) - ix, dy = int((j / nx) % ny) - iy,
                      dz = int(j / plane) - iz;
            const int c = int(c_slot[(dz + 3) * 49 + (dy + 3) * 7 + (dx + 3)]);
            if (!((w[c >> 5] >> (c & 31)) & 1u))
                v = -1;
            if (hist_out) {  // broken bonds keep their last history (engine.cpp:88-92)
                float h = hist[slot_base(L, i) + (long long)c * (64 * L.nlbz)];
                if (L.typed)
                    h = __uint_as_float(__float_as_uint(h) & ~7u);
                hist_out[i * N + k] = double(h);
            }
        }
        if (out)
            out[i * N + k] = v;
    }
}

template <class K> void preload_fn(K k) {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, reinterpret_cast<const void*>(k));
}

// the dynamic shared-memory opt-in is per device: a process may drive
// several GPUs (slab ranks as threads)
template <int MODE, int BZT, int MINB, bool BC, bool NF> cudaError_t configure_one() {
    static std::atomic<bool> done[64];
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess)
        return e;
    if (dev < 64 && done[dev].load(std::memory_order_acquire))
        return cudaSuccess;
    e = cudaFuncSetAttribute(lattice_step_kernel<MODE, BZT, MINB, BC, NF>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(sizeof(float4)) * nrec<BZT>());
    if (e == cudaSuccess && dev < 64)
        done[dev].store(true, std::memory_order_release);
    return e;
}

template <int MODE, int BZT, int MINB, bool BC, bool NF>
cudaError_t launch_cfg(const DevArgs& A, const LatticeArgs& L, cudaStream_t st) {
    const int nbx = (L.nx + BX - 1) / BX, nby = (L.ny + BY - 1) / BY,
              nbz = (L.nz_own + BZT - 1) / BZT;
    if (nbx * nby * nbz == 0)
        return cudaSuccess;
    const cudaError_t e = configure_one<MODE, BZT, MINB, BC, NF>();
    if (e != cudaSuccess)
        return e;
    t_last_kernel = kernel_name<1, MODE, BZT, MINB, BC, NF>("lattice_step_kernel");
    lattice_step_kernel<MODE, BZT, MINB, BC, NF>
        <<<dim3(unsigned(nbx), unsigned(nby), unsigned(nbz)), BX * BY * BZT,
           sizeof(float4) * nrec<BZT>(), st>>>(A, L);
    return cudaGetLastError();
}

// Brick shape and CTAs per SM (register budget).  Measured at 10M nodes
// (profiles/): 16x4x4 bricks at 5 CTAs/SM (48 registers, 40 warps/SM) beat
// 16x4x8 at 2 (64 registers) by 15 %; 16x4x2 bricks lose to the halo overhead
// (13.8 staged records per node).  Without boundary conditions the epilogue
// is lighter and 6 CTAs/SM (40 registers) fit.  PD_LAT_CFG selects
// alternatives for the bench configuration: 1 = 16x4x8 x3, 2 = 16x4x4 x4,
// 3 = 16x4x8 x2, 4 = 16x4x4 x5, 9 = 16x4x9 x2, 10 = 16x4x9 x3.
int sm_count() {
    static const int n = [] {
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        return cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0
                   ? v
                   : 148;
    }();
    return n;
}

template <int MODE, bool BC, bool NF>
cudaError_t launch_bc(const DevArgs& A, const LatticeArgs& L, cudaStream_t st) {
    // Small models (fewer 16x4x4 bricks than two per SM, e.g. cfg1's beam):
    // the step is one latency chain per thread, so use 16x4x1 bricks (more
    // CTAs over the SMs) and the full register file (the compiler can overlap
    // several slots).  PD_LAT_CFG = 5 forces it; any other
    // nonzero value forbids it (6: the large-model rule below without its
    // brick-depth waste test, i.e. 16x4x4 bricks; 1-4, 7, 8: fixed shapes).
    const long long bricks4 = (long long)((L.nx + 15) / 16) * ((L.ny + 3) / 4) * ((L.nz_own + 3) / 4);
    if (L.cfg == 5 || (L.cfg == 0 && bricks4 < 2LL * sm_count()))
        return launch_cfg<MODE, 1, 1, BC, NF>(A, L, st);
    if constexpr (!NF && !BC) {
        switch (L.cfg) {
        case 1: return launch_cfg<MODE, 8, 3, BC, NF>(A, L, st);
        case 2: return launch_cfg<MODE, 4, 4, BC, NF>(A, L, st);
        case 3: return launch_cfg<MODE, 8, 2, BC, NF>(A, L, st);
        case 4: return launch_cfg<MODE, 4, 5, BC, NF>(A, L, st);
        case 7: return launch_cfg<MODE, 6, 4, BC, NF>(A, L, st);
        case 8: return launch_cfg<MODE, 12, 2, BC, NF>(A, L, st);
        case 9: return launch_cfg<MODE, 9, 2, BC, NF>(A, L, st);
        case 10: return launch_cfg<MODE, 9, 3, BC, NF>(A, L, st);
        default: break;
        }
    }
    // Without BC code, 16x4x8 bricks at 3 CTAs/SM (40 registers) stage 6.0
    // halo records per node against 8.6 for 16x4x4 and measured 5 % faster
    // at 10M (profiles/) -- unless the owned planes
    // leave a much emptier last z-brick (e.g. 27-plane slabs of 216 over 8
    // GPUs), where 16x4x4 bricks waste less.
    // 16x4x9 bricks (2 CTAs/SM) fit plane counts that are multiples of 9 but
    // not of 8: a 27-plane slab (216 over 8 GPUs) takes 0.154 ms against
    // 0.166 ms with 16x4x4 bricks; on 216 planes 16x4x8 stays faster (1.111
    // against 1.122 ms).
    if constexpr (!BC) {
        const int nz = L.nz_own;
        const double waste8 = double((nz + 7) / 8 * 8 - nz) / nz;
        const double waste9 = double((nz + 8) / 9 * 9 - nz) / nz;
        const double waste4 = double((nz + 3) / 4 * 4 - nz) / nz;
        if (L.cfg == 0 && waste8 - waste4 < 0.04)
            return launch_cfg<MODE, 8, 3, BC, NF>(A, L, st);
        if (L.cfg == 0 && waste9 <= waste4)
            return launch_cfg<MODE, 9, 2, BC, NF>(A, L, st);
    }
    return launch_cfg<MODE, 4, BC ? 5 : 6, BC, NF>(A, L, st);
}

template <int MODE> cudaError_t launch_mode(const DevArgs& A, const LatticeArgs& L, cudaStream_t st) {
    if (L.nf)
        return A.bc_kind ? launch_bc<MODE, true, true>(A, L, st)
                         : launch_bc<MODE, false, true>(A, L, st);
    return A.bc_kind ? launch_bc<MODE, true, false>(A, L, st)
                     : launch_bc<MODE, false, false>(A, L, st);
}

template <int MODE, bool BC, bool NF> void preload_bc() {
    preload_fn(lattice_step_kernel<MODE, 4, BC ? 5 : 6, BC, NF>);
    configure_one<MODE, 4, BC ? 5 : 6, BC, NF>();
    if constexpr (!BC) {
        preload_fn(lattice_step_kernel<MODE, 8, 3, BC, NF>);
        configure_one<MODE, 8, 3, BC, NF>();
        preload_fn(lattice_step_kernel<MODE, 9, 2, BC, NF>);
        configure_one<MODE, 9, 2, BC, NF>();
    }
    preload_fn(lattice_step_kernel<MODE, 1, 1, BC, NF>);
    configure_one<MODE, 1, 1, BC, NF>();
    if constexpr (!NF && !BC) {
        preload_fn(lattice_step_kernel<MODE, 8, 2, BC, NF>);
        preload_fn(lattice_step_kernel<MODE, 8, 3, BC, NF>);
        preload_fn(lattice_step_kernel<MODE, 4, 4, BC, NF>);
        preload_fn(lattice_step_kernel<MODE, 4, 5, BC, NF>);
        preload_fn(lattice_step_kernel<MODE, 6, 4, BC, NF>);
        preload_fn(lattice_step_kernel<MODE, 12, 2, BC, NF>);
        configure_one<MODE, 6, 4, BC, NF>();
        configure_one<MODE, 12, 2, BC, NF>();
        preload_fn(lattice_step_kernel<MODE, 9, 2, BC, NF>);
        preload_fn(lattice_step_kernel<MODE, 9, 3, BC, NF>);
        configure_one<MODE, 9, 2, BC, NF>();
        configure_one<MODE, 9, 3, BC, NF>();
        configure_one<MODE, 8, 2, BC, NF>();
        configure_one<MODE, 8, 3, BC, NF>();
        configure_one<MODE, 4, 4, BC, NF>();
        configure_one<MODE, 4, 5, BC, NF>();
    }
}

template <int MODE, bool BC, bool NF> void preload_small() {
    preload_fn(lattice_small_kernel<MODE, BC, NF, 16, 4>);
    preload_fn(lattice_small_kernel<MODE, BC, NF, 8, 4>);
    preload_fn(lattice_small_kernel<MODE, BC, NF, 8, 8>);
}

template <int MODE> void preload_mode() {
    if constexpr (MODE != 0) {
        preload_small<MODE, true, true>();
        preload_small<MODE, true, false>();
        preload_small<MODE, false, true>();
        preload_small<MODE, false, false>();
    }
    preload_bc<MODE, true, false>();
    preload_bc<MODE, false, false>();
    preload_bc<MODE, true, true>();
    preload_bc<MODE, false, true>();
}

} // namespace

long long lattice_slot_count(const LatticeArgs& L) {
    const long long nbx = (L.nx + 15) / 16, nby = (L.ny + 3) / 4,
                    nbz = (L.nz_own + L.nlbz - 1) / L.nlbz;
    return nbx * nby * nbz * (long long)NPAT * (64 * L.nlbz);
}

bool lattice_detect(const double* coords, long long n, long long own_begin, long long own_end,
                    LatticeArgs& L) {
    if (n < 2)
        return false;
    const double ox = coords[0], oy = coords[1], oz = coords[2];
    long long nx = 1;
    while (nx < n && coords[3 * nx + 1] == oy && coords[3 * nx + 2] == oz)
        ++nx;
    if (nx < 2)
        return false;
    const double h = coords[3] - ox;
    if (!(h > 0))
        return false;
    long long ny = 1;
    while (ny * nx < n && coords[3 * (ny * nx) + 2] == oz)
        ++ny;
    const long long plane = nx * ny;
    if (n % plane != 0)
        return false;
    const long long nz = n / plane;
    // every node is checked against origin + k h on the device
    // (lattice_build_masks), together with the rows
    if (own_begin % plane != 0 || own_end % plane != 0)
        return false;  // owned range of a slab: whole planes
    for (int c = 0; c < NPAT; ++c) {
        L.pat[c][0] = (signed char)pat(c, 0);
        L.pat[c][1] = (signed char)pat(c, 1);
        L.pat[c][2] = (signed char)pat(c, 2);
        L.pat[c][3] = (signed char)(pat(c, 0) * pat(c, 0) + pat(c, 1) * pat(c, 1) + pat(c, 2) * pat(c, 2));
    }
    L.nx = int(nx);
    L.ny = int(ny);
    L.nz_local = int(nz);
    L.z0 = int(own_begin / plane);
    L.nz_own = int((own_end - own_begin) / plane);
    L.h = h;
    L.inv_h = 1.0 / h;
    L.ox = ox;
    L.oy = oy;
    L.oz = oz;
    return true;
}

cudaError_t lattice_build_masks(const double4* xv, long long n, const int32_t* entries,
                                long long begin, long long end, int N, const LatticeArgs& L,
                                uint4* mask, int* bad, const double* hist, const uint8_t* btype,
                                const double* lambda, const double* beta, cudaStream_t st) {
    if (n > 0)
        lattice_coords_kernel<<<unsigned((n + 255) / 256), 256, 0, st>>>(xv, n, L, bad);
    signed char tab[NPAT][4];
    for (int c = 0; c < NPAT; ++c) {
        tab[c][0] = (signed char)pat(c, 0);
        tab[c][1] = (signed char)pat(c, 1);
        tab[c][2] = (signed char)pat(c, 2);
        tab[c][3] = (signed char)(tab[c][0] * tab[c][0] + tab[c][1] * tab[c][1] +
                                  tab[c][2] * tab[c][2]);
    }
    signed char slot_of[343];
    for (int k = 0; k < 343; ++k)
        slot_of[k] = -1;
    for (int c = 0; c < NPAT; ++c)
        slot_of[(tab[c][2] + 3) * 49 + (tab[c][1] + 3) * 7 + (tab[c][0] + 3)] = (signed char)c;
    cudaError_t e = cudaMemcpyToSymbolAsync(c_pat, tab, sizeof tab, 0, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess)
        e = cudaMemcpyToSymbolAsync(c_slot, slot_of, sizeof slot_of, 0, cudaMemcpyHostToDevice, st);
    float lens[NPAT];
    for (int c = 0; c < NPAT; ++c)
        lens[c] = root(int(tab[c][3]));
    if (e == cudaSuccess)
        e = cudaMemcpyToSymbolAsync(c_len, lens, sizeof lens, 0, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess)
        return e;
    {
        float4 geo[128];
        float2 geo2[128];
        int goff[128];
        for (int c = 0; c < 128; ++c) {
            geo[c] = make_float4(0.f, 0.f, 0.f, 0.f);
            geo2[c] = make_float2(0.f, 0.f);
            goff[c] = 0;
            if (c >= NPAT)
                continue;
            const int r2 = int(tab[c][3]);
            geo[c] = make_float4(float(tab[c][0]), float(tab[c][1]), float(tab[c][2]), float(r2));
            geo2[c] = make_float2(root(r2), 1.0f / root(r2));
            goff[c] = tab[c][0] + HX * (tab[c][1] + HY * tab[c][2]);
        }
        e = cudaMemcpyToSymbolAsync(c_geo, geo, sizeof geo, 0, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess)
            e = cudaMemcpyToSymbolAsync(c_geo2, geo2, sizeof geo2, 0, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess)
            e = cudaMemcpyToSymbolAsync(c_goff, goff, sizeof goff, 0, cudaMemcpyHostToDevice, st);
        if (e != cudaSuccess)
            return e;
    }
    SlotSrc src{hist, btype, lambda, beta};
    if (end > begin)
        lattice_mask_kernel<<<unsigned((end - begin + 7) / 8), 256, 0, st>>>(
            entries, begin, end, N, L.nx, L.ny, mask, bad, src, L);
    return cudaGetLastError();
}

template <int MODE, bool BC, int BZT>
cudaError_t launch_nl_loop(const DevArgs& A, const LatticeArgs& L, cudaStream_t st) {
    const int nbx = (L.nx + BX - 1) / BX, nby = (L.ny + BY - 1) / BY,
              nbz = (L.nz_own + BZT - 1) / BZT;
    if (nbx * nby * nbz == 0)
        return cudaSuccess;
    const dim3 grid{unsigned(nbx), unsigned(nby), unsigned(nbz)};
    const size_t smem = sizeof(float4) * nrec<BZT>();
    const cudaError_t e = smem_optin<lattice_nl_kernel<MODE, BC, true, BZT>>(int(smem));
    if (e != cudaSuccess)
        return e;
    t_last_kernel = kernel_name<2, MODE, BC, 1, BZT>("lattice_nl_kernel");
    lattice_nl_kernel<MODE, BC, true, BZT><<<grid, BX * BY * BZT, smem, st>>>(A, L);
    return cudaGetLastError();
}

template <int MODE, bool BC>
cudaError_t launch_nl(const DevArgs& A, const LatticeArgs& L, cudaStream_t st) {
    if (L.multi && !L.typed)  // the loop kernel (also forced by PD_LAT_NL_LOOP at setup)
        return L.nlbz == 4 ? launch_nl_loop<MODE, BC, 4>(A, L, st)
                           : launch_nl_loop<MODE, BC, 8>(A, L, st);
    return MODE == 0   ? launch_nlu_m0(A, L, st)
           : MODE == 1 ? launch_nlu_m1(A, L, st)
           : MODE == 2 ? launch_nlu_m2(A, L, st)
                       : launch_nlu_m3(A, L, st);
}

template <int MODE> cudaError_t launch_nl_mode(const DevArgs& A, const LatticeArgs& L,
                                               cudaStream_t st) {
    return A.bc_kind ? launch_nl<MODE, true>(A, L, st) : launch_nl<MODE, false>(A, L, st);
}

cudaError_t launch_lattice(const DevArgs& A, const LatticeArgs& L, int mode, cudaStream_t st) {
    if (L.nl) {
        switch (mode) {
        case 0: return launch_nl_mode<0>(A, L, st);
        case 1: return launch_nl_mode<1>(A, L, st);
        case 2: return launch_nl_mode<2>(A, L, st);
        default: return launch_nl_mode<3>(A, L, st);
        }
    }
    switch (mode) {
    case 0: return launch_mode<0>(A, L, st);
    case 1: return launch_mode<1>(A, L, st);
    case 2: return launch_mode<2>(A, L, st);
    default: return launch_mode<3>(A, L, st);
    }
}

long long lattice_small_ctas(const LatticeArgs& L) {
    if (L.nl || L.cfg != 0)  // PD_LAT_CFG = 5 forces the one-step small-brick kernel
        return 0;
    const long long bricks4 = (long long)((L.nx + 15) / 16) * ((L.ny + 3) / 4) * ((L.nz_own + 3) / 4);
    if (bricks4 >= 2LL * sm_count())
        return 0;
    const int bx = small_bx(L);
    return (long long)((L.nx + bx - 1) / bx) * ((L.ny + BY - 1) / BY) * L.nz_own;
}

bool lattice_small_fits(const LatticeArgs& L, int mode, bool bc) {
    const long long ctas = lattice_small_ctas(L);
    if (ctas <= 0)
        return false;
    const bool nf = L.nf != 0;
    const int bx = small_bx(L);
    const int per_sm = mode == 1 ? small_capacity_mode<1>(bc, nf, bx)
                     : mode == 2 ? small_capacity_mode<2>(bc, nf, bx)
                                 : small_capacity_mode<3>(bc, nf, bx);
    return ctas <= (long long)per_sm * sm_count();
}

cudaError_t launch_lattice_small(const DevArgs& A, const LatticeArgs& L, int mode, const SmallArgs& S,
                                 cudaStream_t st) {
    switch (mode) {
    case 1: return launch_small_mode<1>(A, L, S, st);
    case 2: return launch_small_mode<2>(A, L, S, st);
    case 3: return launch_small_mode<3>(A, L, S, st);
    default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_lattice_materialize(const int32_t* entries0, const uint4* mask, long long begin,
                                       long long end, long long n, int N, const LatticeArgs& L,
                                       int32_t* out, double* hist_out, cudaStream_t st) {
    if (n > 0)
        lattice_materialize_kernel<<<unsigned((n + 255) / 256), 256, 0, st>>>(
            entries0, mask, begin, end, n, N, L, out, hist_out);
    return cudaGetLastError();
}

bool lattice_minmax_ok(const double* bp, const double* f, int nbp) {
    if (nbp <= 2)
        return nbp >= 1;  // one line, or two lines meeting at bp_0: always max/min of them
    if (nbp > 3)
        return false;
    // the kernels' lines in fp64 (lattice_set_laws): l_0 = sl_0 e, l_k = a_k + sl_k e
    const double sl0 = f[0] / bp[0];
    const double sl1 = (f[1] - f[0]) / (bp[1] - bp[0]), a1 = f[0] - bp[0] * sl1;
    const double sl2 = (f[2] - f[1]) / (bp[2] - bp[1]), a2 = f[1] - bp[1] * sl2;
    const bool cvx1 = sl1 > sl0, cvx2 = sl2 > sl1;
    const double sl[3] = {sl0, sl1, sl2}, a[3] = {0.0, a1, a2};
    auto comp = [&](double e) {
        const double l0 = sl0 * e, l1 = a1 + sl1 * e, l2 = a2 + sl2 * e;
        const double t = cvx2 ? std::max(l1, l2) : std::min(l1, l2);
        return cvx1 ? std::max(l0, t) : std::min(l0, t);
    };
    auto env = [&](double e) {  // envelope_force: the segment whose end exceeds e
        const int k = e < bp[0] ? 0 : (e < bp[1] ? 1 : 2);
        return a[k] + sl[k] * e;
    };
    // both sides are piecewise linear with kinks only at the breakpoints and
    // where two lines cross: equal at every such point (and at 0) => equal on
    // [0, s_c]
    std::vector<double> pts = {0.0, bp[0], bp[1], bp[2]};
    for (int p = 0; p < 3; ++p)
        for (int q = p + 1; q < 3; ++q)
            if (sl[p] != sl[q]) {
                const double e = (a[q] - a[p]) / (sl[p] - sl[q]);
                if (e > 0.0 && e < bp[2])
                    pts.push_back(e);
            }
    double scale = 0.0;
    for (int k = 0; k < 3; ++k)
        scale = std::max(scale, std::fabs(f[k]));
    scale = std::max(scale, std::fabs(sl0 * bp[0]));
    for (double e : pts)
        if (std::fabs(comp(e) - env(e)) > 1e-9 * scale)
            return false;
    return true;
}

void lattice_set_laws(const DevLaw* laws, int n, LatticeArgs& L, cudaStream_t st) {
    FastLaw f[PD_MAX_LAWS];
    for (int k = 0; k < n; ++k)
        fast_law_from(f[k], laws[k].c, laws[k].nbp, laws[k].bp, laws[k].f);
    cudaMemcpyToSymbolAsync(c_llaws, f, sizeof(FastLaw) * size_t(n), 0, cudaMemcpyHostToDevice, st);
    // one law of <= 3 breakpoints: registers (bp1 = +inf for two breakpoints)
    L.multi = !(n == 1 && f[0].nbp >= 1 && f[0].nbp <= 3);
    const FastLaw& a = f[0];
    const float inf = std::numeric_limits<float>::infinity();
    L.rl.c = a.c;
    L.rl.hist = a.nbp > 1;
    L.rl.sc = a.bp[a.nbp - 1];
    L.rl.bp0 = a.nbp > 1 ? a.bp[0] : inf;
    L.rl.bp1 = a.nbp > 2 ? a.bp[1] : inf;
    L.rl.f0 = a.f[0];
    L.rl.f1 = a.nbp > 2 ? a.f[1] : 0.f;
    L.rl.sl0 = a.sl[0];
    L.rl.sl1 = a.nbp > 1 ? a.sl[1] : 0.f;
    L.rl.sl2 = a.nbp > 2 ? a.sl[2] : 0.f;
    L.rl.nbp = a.nbp;
    if (L.typed) {  // per-type segment lines in fp64 -> fp32 (pd_lattice_nlu.cuh nl_law_typed)
        for (int k = 0; k < 8; ++k) {
            L.tl[2 * k] = make_float4(0.f, 0.f, 0.f, 1.f);
            L.tl[2 * k + 1] = make_float4(0.f, 0.f, -1.f, -1.f);
        }
        for (int k = 0; k < n && k < 8; ++k) {
            const DevLaw& d = laws[k];
            const double c = d.c, sl0 = d.f[0] / d.bp[0];
            double sl1 = sl0, a1 = 0.0, sl2 = sl0, a2 = 0.0;
            if (d.nbp >= 2) {
                sl1 = (d.f[1] - d.f[0]) / (d.bp[1] - d.bp[0]);
                a1 = d.f[0] - d.bp[0] * sl1;
                sl2 = sl1;
                a2 = a1;
            }
            if (d.nbp >= 3) {
                sl2 = (d.f[2] - d.f[1]) / (d.bp[2] - d.bp[1]);
                a2 = d.f[1] - d.bp[1] * sl2;
            }
            const float sc = float(d.bp[d.nbp - 1]);
            L.tl[2 * k] = make_float4(float(d.nbp == 1 ? c : sl0), float(sl1), float(a1),
                                      d.nbp > 1 ? sc : -sc);
            L.tl[2 * k + 1] = make_float4(float(sl2), float(a2), sl1 > sl0 ? 1.f : -1.f,
                                          sl2 > sl1 ? 1.f : -1.f);
        }
    }
    if (n >= 1 && laws[0].nbp >= 2) {  // a_k = f_{k-1} - bp_{k-1} sl_k in fp64
        const DevLaw& d = laws[0];
        const double sl0 = d.f[0] / d.bp[0];
        const double sl1 = (d.f[1] - d.f[0]) / (d.bp[1] - d.bp[0]);
        L.rl.a1 = float(d.f[0] - d.bp[0] * sl1);
        L.rl.cvx1 = sl1 > sl0;
        if (d.nbp >= 3) {
            const double sl2 = (d.f[2] - d.f[1]) / (d.bp[2] - d.bp[1]);
            L.rl.a2 = float(d.f[1] - d.bp[1] * sl2);
            L.rl.cvx2 = sl2 > sl1;
        } else {  // two breakpoints: the third segment repeats the second
            L.rl.a2 = L.rl.a1;
            L.rl.sl2 = L.rl.sl1;
        }
    }
}

template <int MODE> void preload_nl() {
    preload_fn(lattice_nl_kernel<MODE, true, true, 4>);
    preload_fn(lattice_nl_kernel<MODE, false, true, 4>);
    preload_fn(lattice_nl_kernel<MODE, true, true, 8>);
    preload_fn(lattice_nl_kernel<MODE, false, true, 8>);
    smem_optin<lattice_nl_kernel<MODE, true, true, 8>>(int(sizeof(float4)) * nrec<8>());
    smem_optin<lattice_nl_kernel<MODE, false, true, 8>>(int(sizeof(float4)) * nrec<8>());
}

void preload_lattice() {
    preload_nlu_m0();
    preload_nlu_m1();
    preload_nlu_m2();
    preload_nlu_m3();
    preload_nl<0>();
    preload_nl<1>();
    preload_nl<2>();
    preload_nl<3>();
    preload_mode<0>();
    preload_mode<1>();
    preload_mode<2>();
    preload_mode<3>();
    preload_fn(lattice_mask_kernel);
    preload_fn(lattice_coords_kernel);
    preload_fn(lattice_materialize_kernel);
}

} // namespace pdb
