// pd_device.cuh -- device-side layouts shared by the B200 kernels.
//
// HBM layout of one resident model (one pd_ctx), n nodes, group size N:
//   xv       double4[n]   {x, y, z, V_j}            gathered per live slot (32 B, LDG.256)
//   u[2]     double4[n]   {ux, uy, uz, no_fail_j}   double-buffered displacement; the
//                                                   4th lane carries the node's no-failure
//                                                   flag so the per-slot gather needs no
//                                                   extra load (engine.cpp:79-80)
//   v, a     double[3n]   per-node streams (reference flat layout)
//   rho      double[n]
//   entries  int32[n*N]   the row list as uploaded (never rewritten; breaks live in alive)
//   alive    uint32[n*W]  W = max(1, N/32); bit k of row i == (entries[i*N+k] != -1)
//                         in the reference's mutable list (engine.cpp:81-83, 93-96)
//   hist     double[n*N]  only for n-linear laws (types.hpp:120)
//   btype    uint8[n*N]   optional bond types (types.hpp:71)
//   lambda, beta double[n*N] optional (types.hpp:161-165)
//   bc_*     per node-axis boundary arrays (types.hpp:145-155), NULL when all free
#pragma once

#include <cstdint>

#include "../../include/pd_b200.h"

namespace pdb {

struct DevLaw {
    double c;
    int nbp;
    int pad_;
    double bp[PD_MAX_BREAKPOINTS];
    double f[PD_MAX_BREAKPOINTS];
};

struct DevRamp {
    int kind;
    int pad_;
    long long rise;
    double target;
};

constexpr long long kNoError = 0x7fffffffffffffffLL;

struct DevArgs {
    long long n;        // nodes in this context (owned + ghost)
    long long begin;    // first node this launch computes
    long long end;      // one past the last node this launch computes
    int N;              // group size
    int log2N;
    int W;              // alive words per row
    int n_laws;
    const double4* xv;
    const double4* u_in;
    double4* u_out;
    double* v;
    double* a;
    const double* rho;
    const double* inv_rho;    // 1/rho, precomputed once (Real(1) / density[i], engine.cpp:244)
    const int32_t* entries;
    uint32_t* alive;
    int32_t* n_neigh;         // live count per row, decremented on breaks
    double* hist;
    const uint8_t* btype;
    const double* lambda;
    const double* beta;
    const uint8_t* bc_kind;   // 3n or NULL
    const double* bc_mag;     // 3n
    const uint8_t* bc_ramp;   // 3n
    const DevRamp* ramps;
    double* body_force;       // 3n, stored when store_forces
    double* ext_force;        // 3n, stored when store_forces
    long long* err_step;      // first step whose force pass sees non-finite u
    long long step;           // the step s this launch advances (s -> s+1)
    double dt;
    double half_dt;           // dt / 2   (host-computed, same IEEE result)
    double half_dt2;          // dt * dt / 2
    double dt2;               // dt * dt
    double damping;
    double pmb_c, pmb_sc;     // the single-PMB-law model (exact kernel specialisation)
    const DevLaw* laws;       // the law table (exact kernel)
    int store_forces;
    int do_drift;             // VV: produce next step's drifted u into u_out
    // multi-GPU slabs: owned nodes that are ghosts on the neighbouring ranks
    // also store their new u into those ranks' u buffers (same parity as
    // u_out) over NVLink; xfer[i] = {row on rank lo, row on rank hi} or -1
    const int2* xfer;         // NULL on one GPU
    double4* peer_lo;
    double4* peer_hi;
};

constexpr long long kPeerTimeout = -2;  // err_step value: a peer rank never arrived
constexpr long long kBarrierTimeout = -3;  // err_step value: a persistent launch's grid barrier timed out

// Store an owned node's new displacement into the ghost rows of the
// neighbouring ranks (peer memory) and make it visible system-wide before the
// step's sync kernel publishes the step.  One system fence per warp, not per
// node: the converged lanes meet at __syncwarp (which orders their stores
// before the leader's) and the leader's fence.sc.sys is cumulative over them.
__device__ __forceinline__ void push_ghost(const DevArgs& A, long long i, const double4& un) {
    if (!A.xfer)
        return;
    const int2 t = A.xfer[i];
    if (t.x >= 0)
        A.peer_lo[t.x] = un;
    if (t.y >= 0)
        A.peer_hi[t.y] = un;
    const unsigned act = __activemask();
    const unsigned pushed = __ballot_sync(act, t.x >= 0 || t.y >= 0);
    if (pushed) {
        __syncwarp(act);
        if ((threadIdx.x & 31) == unsigned(__ffs(act) - 1))
            __threadfence_system();
    }
}

// RampProfile::scale/rate/accel (types.cpp:119-169); same operation order, so
// with FMA contraction disabled the device values equal the host's bit for bit.
// Not inlined: only boundary-condition node-axes call them, and three inlined
// axes of fp64 divisions cost the unrolled kernels ~9 KB of instruction cache.
#ifdef PD_RAMP_INLINE
#define PD_RAMP_FN __forceinline__
#else
#define PD_RAMP_FN __noinline__
#endif
static __device__ PD_RAMP_FN double ramp_scale(const DevRamp& r, long long step) {
    if (r.kind == PD_RAMP_CONSTANT)
        return r.target;
    if (r.rise <= 0 || step >= r.rise)
        return r.target;
    if (r.kind == PD_RAMP_LINEAR)
        return __ddiv_rn(__dmul_rn(r.target, (double)step), (double)r.rise);
    const double t = __ddiv_rn((double)step, (double)r.rise);
    // target * t * t * t * (10 + t * (-15 + 6 * t))
    const double inner = __dadd_rn(10.0, __dmul_rn(t, __dadd_rn(-15.0, __dmul_rn(6.0, t))));
    return __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(r.target, t), t), t), inner);
}

static __device__ PD_RAMP_FN double ramp_rate(const DevRamp& r, long long step) {
    if (r.kind == PD_RAMP_CONSTANT)
        return 0.0;
    if (r.rise <= 0 || step >= r.rise)
        return 0.0;
    if (r.kind == PD_RAMP_LINEAR)
        return __ddiv_rn(r.target, (double)r.rise);
    const double t = __ddiv_rn((double)step, (double)r.rise);
    // target * 30 * t * t * (t - 1) * (t - 1) / rise
    double x = __dmul_rn(r.target, 30.0);
    x = __dmul_rn(x, t);
    x = __dmul_rn(x, t);
    x = __dmul_rn(x, __dsub_rn(t, 1.0));
    x = __dmul_rn(x, __dsub_rn(t, 1.0));
    return __ddiv_rn(x, (double)r.rise);
}

static __device__ PD_RAMP_FN double ramp_accel(const DevRamp& r, long long step) {
    if (r.kind != PD_RAMP_QUINTIC)
        return 0.0;
    if (r.rise <= 0 || step >= r.rise)
        return 0.0;
    const double t = __ddiv_rn((double)step, (double)r.rise);
    // target * 60 * t * (2 * t - 1) * (t - 1) / (rise * rise)
    double x = __dmul_rn(r.target, 60.0);
    x = __dmul_rn(x, t);
    x = __dmul_rn(x, __dsub_rn(__dmul_rn(2.0, t), 1.0));
    x = __dmul_rn(x, __dsub_rn(t, 1.0));
    return __ddiv_rn(x, __dmul_rn((double)r.rise, (double)r.rise));
}

// x / d for d > 0 (dt, dt^2) in the persistent small-model kernel, where the
// supports' divisions are the per-step critical path: a zero numerator (a
// fixed support: magnitude 0) gives the signed zero IEEE division gives with
// no division at all (__ddiv_rn takes its slow path for zero numerators, and
// an inlined one is speculated past a test), others call it out of line.
// The one-step kernels keep the plain inline division: an out-of-line call
// costs the big unrolled kernels registers around the call site (cfg2's
// n-linear step: 87 -> 112 us).
static __device__ __noinline__ double div_call(double x, double d) { return __ddiv_rn(x, d); }

__device__ __forceinline__ double div_pos(double x, double d) {
    if (x == 0.0 && d > 0.0)
        return x;
    return div_call(x, d);
}

__device__ __forceinline__ bool finite3(double x, double y, double z) {
    return isfinite(x) && isfinite(y) && isfinite(z);
}

// Per-node integrator epilogue shared by every force kernel.  fp64 with
// explicit round-to-nearest intrinsics (never contracted), so the exact and
// fast paths integrate identically given the same body force.
//   MODE 1: verlet_kick + apply_displacement_kinematics(s+1)  (engine.cpp:235-252, 274-286)
//           then verlet_drift + apply_displacement_positions(s+2) for the next
//           step into u_out (engine.cpp:221-233, 262-272; driver order :397-404)
//   MODE 2: step_euler (engine.cpp:187-202), MODE 3: step_euler_cromer (:204-219),
//           then positions + kinematics of step s+1 (driver order :405-415)
// External force: external_force.assign(0) then += mag * scale (engine.cpp:288-297),
// evaluated at s+1 (Verlet) or s (Euler).
// Per-node integrator inputs; loaded right before the epilogue, or early
// (before a kernel's bond loop) so their latency overlaps the bond work.
struct NodeIn {
    double v[3], a[3], inv_rho;
};

__device__ __forceinline__ NodeIn load_node_in(const DevArgs& A, long long i) {
    NodeIn r;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        r.v[ax] = A.v[3 * i + ax];
        r.a[ax] = A.a[3 * i + ax];
    }
    r.inv_rho = A.inv_rho[i];
    return r;
}

// One node-axis's boundary condition (types.hpp:145-155): its kind, and for
// a prescribed axis the magnitude and the ramp record.
struct AxisBc {
    int kind;
    int rid;  // ramp id
    double mag;
    DevRamp ramp;
};

__device__ __forceinline__ AxisBc load_axis_bc(const DevArgs& A, long long i, int ax) {
    AxisBc b{PD_BC_FREE, 0, 0.0, DevRamp{}};
    b.kind = A.bc_kind ? int(A.bc_kind[3 * i + ax]) : PD_BC_FREE;
    if (b.kind != PD_BC_FREE) {
        b.mag = A.bc_mag[3 * i + ax];
        b.rid = A.bc_ramp[3 * i + ax];
        b.ramp = A.ramps[b.rid];
    }
    return b;
}

// The ramp values one step s needs (node_epilogue): scale(s), scale(s + 1),
// scale(s + 2), rate(s + 1), accel(s + 1) -- the same calls, so the same bits.
// A kernel that runs many nodes per step can evaluate them once per ramp.
struct RampVals {
    double sc0, sc1, sc2, rate1, acc1;
};

__device__ __forceinline__ RampVals ramp_vals(const DevRamp& r, long long s) {
    return RampVals{ramp_scale(r, s), ramp_scale(r, s + 1), ramp_scale(r, s + 2), ramp_rate(r, s + 1),
                    ramp_accel(r, s + 1)};
}

// BC = false: the caller guarantees A.bc_kind == NULL (no boundary conditions),
// so the ramp code is compiled out (fewer registers in the fused kernels).
// KEEP = true (the persistent small-model kernel, which owns its nodes across
// steps): bc holds the node's three AxisBc (shared memory), rv this step's
// RampVals per ramp id, and next / u_next receive the node's new v, a (and
// 1/rho) and the u written to u_out (the next step's u_in), so nothing is
// reloaded; zero-numerator divisions skip the division (div_pos).  KEEP =
// false compiles to the one-step kernels' original code (the extra state
// cost the exact kernel 3 % at 216^3 in registers and spills).
template <int MODE, bool BC = true, bool KEEP = false>
__device__ __forceinline__ void node_epilogue(const DevArgs& A, long long i, const double4& ui,
                                              double fx, double fy, double fz, const NodeIn& in,
                                              const AxisBc* bc = nullptr, NodeIn* next = nullptr,
                                              double4* u_next = nullptr, const RampVals* rv = nullptr) {
    const double Fb[3] = {fx, fy, fz};
    const double u0[3] = {ui.x, ui.y, ui.z};
    const long long s = A.step;
    const double dt = A.dt;
    const double inv = in.inv_rho;
    double v[3], a[3], un[3], Fe[3];
    // each axis is independent; processing one axis at a time keeps the ramp
    // records out of local memory
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        int kind = PD_BC_FREE, rid = 0;
        double mag = 0.0;
        DevRamp ramp{};
        if constexpr (KEEP) {
            if constexpr (BC) {
                kind = bc[ax].kind;
                mag = bc[ax].mag;
                rid = bc[ax].rid;
            }
        } else {
            kind = (BC && A.bc_kind) ? int(A.bc_kind[3 * i + ax]) : PD_BC_FREE;
            if (kind != PD_BC_FREE) {
                mag = A.bc_mag[3 * i + ax];
                ramp = A.ramps[A.bc_ramp[3 * i + ax]];
            }
        }
        // RampProfile values at s + ds: this step's table (KEEP), else evaluated here
        auto scale_at = [&](int ds) {
            if constexpr (KEEP)
                return ds == 0 ? rv[rid].sc0 : ds == 1 ? rv[rid].sc1 : rv[rid].sc2;
            else
                return ramp_scale(ramp, s + ds);
        };
        auto rate1 = [&] {
            if constexpr (KEEP)
                return rv[rid].rate1;
            else
                return ramp_rate(ramp, s + 1);
        };
        auto accel1 = [&] {
            if constexpr (KEEP)
                return rv[rid].acc1;
            else
                return ramp_accel(ramp, s + 1);
        };
        auto div = [&](double x, double d) {
            if constexpr (KEEP)
                return div_pos(x, d);
            else
                return __ddiv_rn(x, d);
        };
        Fe[ax] = kind == PD_BC_FORCE ? __dadd_rn(0.0, __dmul_rn(mag, scale_at(MODE == 1 ? 1 : 0))) : 0.0;
        if (MODE == 1) {
            const double vh = __dadd_rn(in.v[ax], __dmul_rn(in.a[ax], A.half_dt));
            double an = __dmul_rn(__dsub_rn(__dadd_rn(Fb[ax], Fe[ax]), __dmul_rn(vh, A.damping)), inv);
            double vn = __dadd_rn(vh, __dmul_rn(an, A.half_dt));
            if (kind == PD_BC_DISPLACEMENT) {
                vn = div(__dmul_rn(mag, rate1()), dt);
                an = div(__dmul_rn(mag, accel1()), A.dt2);
            }
            v[ax] = vn;
            a[ax] = an;
            un[ax] = __dadd_rn(__dadd_rn(u0[ax], __dmul_rn(vn, dt)), __dmul_rn(an, A.half_dt2));
            if (kind == PD_BC_DISPLACEMENT)
                un[ax] = __dmul_rn(mag, scale_at(2));
        } else {
            const double acc = __dmul_rn(__dadd_rn(Fb[ax], Fe[ax]), inv);
            const double v_old = in.v[ax];
            const double v_new = __dadd_rn(v_old, __dmul_rn(acc, dt));
            a[ax] = acc;
            v[ax] = v_new;
            un[ax] = __dadd_rn(u0[ax], __dmul_rn(MODE == 2 ? v_old : v_new, dt));
            if (kind == PD_BC_DISPLACEMENT) {
                un[ax] = __dmul_rn(mag, scale_at(1));
                v[ax] = div(__dmul_rn(mag, rate1()), dt);
                a[ax] = div(__dmul_rn(mag, accel1()), A.dt2);
            }
        }
    }
    const bool write_u = MODE != 1 || A.do_drift != 0;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        A.v[3 * i + ax] = v[ax];
        A.a[3 * i + ax] = a[ax];
    }
    if constexpr (KEEP) {
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
            next->v[ax] = v[ax];
            next->a[ax] = a[ax];
        }
        next->inv_rho = in.inv_rho;
    }
    if (A.store_forces) {
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
            A.body_force[3 * i + ax] = Fb[ax];
            A.ext_force[3 * i + ax] = Fe[ax];
        }
    }
    if (write_u) {
        const double4 unew = make_double4(un[0], un[1], un[2], ui.w);
        A.u_out[i] = unew;
        if constexpr (KEEP)
            *u_next = unew;
        push_ghost(A, i, unew);
        if (!finite3(un[0], un[1], un[2]))
            atomicMin((unsigned long long*)A.err_step, (unsigned long long)(s + 1));
    } else if constexpr (KEEP) {
        *u_next = ui;
    }
}

template <int MODE, bool BC = true>
__device__ __forceinline__ void node_epilogue(const DevArgs& A, long long i, const double4& ui,
                                              double fx, double fy, double fz) {
    node_epilogue<MODE, BC>(A, i, ui, fx, fy, fz, load_node_in(A, i));
}

} // namespace pdb
