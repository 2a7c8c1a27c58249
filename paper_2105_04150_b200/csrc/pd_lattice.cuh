// pd_lattice.cuh -- device helpers shared by the lattice kernels (pd_lattice.cu
// and the per-integrator pd_lattice_nlu*.cu units): the 122-offset neighbour
// pattern, the fp32 stretch arithmetic, the length-class slot order, the
// brick-major per-bond layout and the halo staging.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <utility>

#include "pd_device.cuh"
#include "pd_fast.cuh"
#include "pd_internal.h"

namespace pdb {
namespace {

// brick = 16 x 4 x BZT nodes (one thread each); halo box HX x HY x (BZT + 6)
constexpr int BX = 16, BY = 4;
constexpr int HX = BX + 6, HY = BY + 6;
constexpr int NPAT = 122;
template <int BZT> constexpr int nrec() { return HX * HY * (BZT + 6); }

// offset c of the pattern, components 0/1/2 = dx/dy/dz, in (dz, dy, dx)
// lexicographic order = ascending reference index order of a row
__host__ __device__ constexpr int pat(int c, int which) {
    int k = 0;
    for (int dz = -3; dz <= 3; ++dz)
        for (int dy = -3; dy <= 3; ++dy)
            for (int dx = -3; dx <= 3; ++dx) {
                const int r2 = dx * dx + dy * dy + dz * dz;
                if (r2 == 0 || r2 > 9)
                    continue;
                if (k == c)
                    return which == 0 ? dx : (which == 1 ? dy : dz);
                ++k;
            }
    return 0;
}

__host__ __device__ constexpr float root(int r2) {
    return r2 == 1 ? 1.0f
         : r2 == 2 ? 1.41421356237f
         : r2 == 3 ? 1.73205080757f
         : r2 == 4 ? 2.0f
         : r2 == 5 ? 2.2360679775f
         : r2 == 6 ? 2.44948974278f
         : r2 == 8 ? 2.82842712475f
         : 3.0f;
}

__device__ __forceinline__ float rsqrt_approx(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}


// The n-linear kernel's stretch (runtime offsets): s and 1/|xi + eta|.
__device__ __forceinline__ void stretch(const float4& rj, const float4& ri, float dx, float dy,
                                        float dz, float r2, float len, float rr, float& s,
                                        float& rc, float& cx, float& cy, float& cz) {
    const float2 hxy = __fadd2_rn(make_float2(rj.x, rj.y), make_float2(-ri.x, -ri.y));
    const float hx = hxy.x, hy = hxy.y, hz = rj.z - ri.z;  // eta / spacing
    cx = hx + dx;
    cy = hy + dy;
    cz = hz + dz;
    // eta.(2 xi + eta), cancellation free
    float num = hz * (hz + (dz + dz));
    num = fmaf(hy, hy + (dy + dy), num);
    num = fmaf(hx, hx + (dx + dx), num);
    const float cur2 = num + r2;
    rc = rsqrt_approx(cur2);
    s = num * rr * rcp_approx(fmaf(cur2, rc, len));
}

// The PMB kernel's stretch.  With w = |xi + eta|^2 |xi|^2 (one FMA from num),
//   a = rsqrt(w) = 1 / (|d| |c|),   s = num / (|d| (|c| + |d|)) = num * rcp(w a + |d|^2)
// so the 1/|d| of s and of the force direction cost no multiply; the caller
// scales each length class's sum by |d| once.  Zero components of d add
// nothing (a compile-time fold the compiler may not do: h + 0.0f != h for
// h = -0.0f).  The unrolled slots (compile-time d) and the break pass
// (runtime d, zero components added as +0) give bit-identical s: they differ
// at most in the sign of a zero term, which cannot change the sum unless
// num = +-0, and then s = +-0 tests the same against s_c.
template <int DX, int DY, int DZ>
__device__ __forceinline__ void stretch_c(const float4& rj, const float4& ri, float& s, float& a,
                                          float2& cxy, float& cz) {
    constexpr int R2 = DX * DX + DY * DY + DZ * DZ;
    // x and y lanes packed (FADD2 / FMUL2; the offset pair comes from a
    // uniform register): eta, xi + eta and xi + eta + d
    const float2 hxy = __fadd2_rn(make_float2(rj.x, rj.y), make_float2(-ri.x, -ri.y));
    const float hz = rj.z - ri.z;  // eta / spacing
    float2 txy;
    if (DX != 0 || DY != 0) {
        const float2 d = make_float2(float(DX), float(DY));
        cxy = __fadd2_rn(hxy, d);
        txy = __fadd2_rn(cxy, d);
    } else {
        cxy = txy = hxy;
    }
    cz = DZ ? hz + float(DZ) : hz;
    const float tz = DZ ? cz + float(DZ) : hz;
    // eta.(2 xi + eta), cancellation free
    const float2 pxy = __fmul2_rn(hxy, txy);
    float num = __fadd_rn(pxy.x, pxy.y);
    num = fmaf(hz, tz, num);
    const float w = fmaf(num, float(R2), float(R2 * R2));
    a = rsqrt_approx(w);
    s = num * rcp_approx(fmaf(w, a, float(R2)));
}

// the same arithmetic with a runtime offset (the rare recompute passes): no
// contraction, lane by lane as the packed instructions round
__device__ __forceinline__ float stretch_r(const float4& rj, const float4& ri, int dx, int dy,
                                           int dz, float& a) {
    const int r2 = dx * dx + dy * dy + dz * dz;
    const float2 hxy = __fadd2_rn(make_float2(rj.x, rj.y), make_float2(-ri.x, -ri.y));
    const float hx = hxy.x, hy = hxy.y, hz = __fsub_rn(rj.z, ri.z);
    const float tx = __fadd_rn(__fadd_rn(hx, float(dx)), float(dx));
    const float ty = __fadd_rn(__fadd_rn(hy, float(dy)), float(dy));
    const float tz = __fadd_rn(__fadd_rn(hz, float(dz)), float(dz));
    float num = __fadd_rn(__fmul_rn(hx, tx), __fmul_rn(hy, ty));
    num = fmaf(hz, tz, num);
    const float w = fmaf(num, float(r2), float(r2 * r2));
    a = rsqrt_approx(w);
    return __fmul_rn(num, rcp_approx(fmaf(w, a, float(r2))));
}

// max that propagates NaN (max.NaN.f32, one FMNMX): an fp32 stretch that
// overflowed (|xi + eta|^2 beyond fp32 range gives inf * 0 in the cancellation-
// free form) is NaN, and a NaN stretch breaks its bond as the reference's
// +inf stretch does (engine.cpp:90-98); breaks are tested as !(s < s_c)
__device__ __forceinline__ float fmax_nan(float a, float b) {
    float r;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float fmax_nan3(float a, float b, float c) {  // one FMNMX3
    float r;
    asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

// Slots are evaluated grouped by length class |d|^2 (1, 2, 3, 4, 5, 6, 8, 9),
// pattern order within a class; K is the position in that order.
struct ClassOrder {
    int slot[NPAT];   // K -> pattern slot
    bool last[NPAT];  // K closes its length class
};
constexpr ClassOrder make_class_order() {
    ClassOrder o{};
    int r2s[NPAT] = {};
    int k = 0;
    for (int dz = -3; dz <= 3; ++dz)
        for (int dy = -3; dy <= 3; ++dy)
            for (int dx = -3; dx <= 3; ++dx) {
                const int r2 = dx * dx + dy * dy + dz * dz;
                if (r2 != 0 && r2 <= 9)
                    r2s[k++] = r2;
            }
    k = 0;
    for (int r2 = 1; r2 <= 9; ++r2)
        for (int c = 0; c < NPAT; ++c)
            if (r2s[c] == r2)
                o.slot[k++] = c;
    for (int q = 0; q < NPAT; ++q)
        o.last[q] = q == NPAT - 1 || r2s[o.slot[q]] != r2s[o.slot[q + 1]];
    return o;
}
constexpr ClassOrder kOrder = make_class_order();

// The dynamic shared-memory opt-in above 48 KB, once per kernel and device
// (a process may drive several GPUs: slab ranks as threads).
template <auto Kernel> cudaError_t smem_optin(int bytes) {
    static std::atomic<unsigned long long> done{0};  // bit d: set on device d
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess)
        return e;
    const unsigned long long bit = dev < 64 ? (1ull << dev) : 0ull;
    if (done.load(std::memory_order_acquire) & bit)
        return cudaSuccess;
    e = cudaFuncSetAttribute(reinterpret_cast<const void*>(Kernel),
                             cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess)
        done.fetch_or(bit, std::memory_order_acq_rel);
    return e;
}

// Per-bond (slot) arrays of the NL path are brick-major: the node at lane t
// (= tx + 16 ty + 64 tz) of 16 x 4 x L.nlbz brick b keeps slot c at
// b * 122 * NB + c * NB + t, NB = 64 L.nlbz the brick's node count.  A step
// thread reads slot c at a compile-time offset from its own base, and a
// warp's access is one 128-byte line.  Bricks tile the owned planes only
// (ghost rows carry no bond state).  The depth (4 or 8 planes) is chosen at
// upload: 8 stages fewer halo records per node, 4 wastes less on thin models.
__host__ __device__ inline long long slot_base(const LatticeArgs& L, long long i) {
    const long long plane = (long long)L.nx * L.ny;
    const int ix = int(i % L.nx), iy = int((i / L.nx) % L.ny), iz = int(i / plane) - L.z0;
    const long long nbx = (L.nx + 15) / 16, nby = (L.ny + 3) / 4;
    const int bz = L.nlbz;
    const long long b = ix / 16 + nbx * (iy / 4 + nby * (iz / bz));
    return b * (long long)NPAT * (64 * bz) + (ix % 16) + 16 * (iy % 4) + 64 * (iz % bz);
}

// Stage the halo box of the brick at (gx0, gy0, gz0) plane by plane
// (HX x HY = 220 records; thread t owns record t % 220 of plane t / 220 of
// each pass): fp32 (u - U_brick) / spacing, plus for NF the signed V_j / V_0.
// Planes are loaded PL at a time so several L2/HBM round trips are in flight.
template <int BZT, bool NF>
__device__ __forceinline__ void stage_box(const DevArgs& A, const LatticeArgs& L, float4* rec,
                                          int gx0, int gy0, int gz0, const double4& U0) {
    constexpr int TT = BX * BY * BZT, HZ = BZT + 6;
    const long long plane = (long long)L.nx * L.ny;
    const float ih = float(L.inv_h);
#ifndef PD_STAGE_FLAT
#define PD_STAGE_FLAT 0
#endif
    if constexpr (TT < HX * HY || PD_STAGE_FLAT) {
        // small bricks (fewer threads than a box plane has records): record r
        // of the box at r = t, t + TT, ..., four in flight per thread
        constexpr int NR = HX * HY * HZ, PL = 4;
        for (int r0 = threadIdx.x; r0 < NR; r0 += TT * PL) {
            double4 u[PL];
            bool ok[PL];
            float wv[PL];
#pragma unroll
            for (int k = 0; k < PL; ++k) {
                const int r = r0 + k * TT;
                const int pz = r / (HX * HY), q = r % (HX * HY);
                const int X = gx0 - 3 + q % HX, Y = gy0 - 3 + q / HX, Z = gz0 - 3 + pz;
                ok[k] = r < NR && X >= 0 && X < L.nx && Y >= 0 && Y < L.ny && Z >= 0 &&
                        Z < L.nz_local;
                u[k] = make_double4(0.0, 0.0, 0.0, 0.0);
                wv[k] = 0.f;
                if (ok[k]) {
                    const long long j = X + (long long)L.nx * Y + plane * Z;
                    u[k] = A.u_in[j];
                    if (NF) {
                        const float vf = L.vol_varies ? float(A.xv[j].w * L.inv_v0) : 1.f;
                        wv[k] = u[k].w != 0.0 ? -vf : vf;
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < PL; ++k) {
                const int r = r0 + k * TT;
                if (r < NR)
                    rec[r] = ok[k] ? make_float4(float(u[k].x - U0.x) * ih, float(u[k].y - U0.y) * ih,
                                                 float(u[k].z - U0.z) * ih, wv[k])
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
        return;
    }
    {
        constexpr int PREC = HX * HY;          // records per box plane
        constexpr int PPASS = TT / PREC;       // planes per pass (1 or 2)
#ifndef PD_LAT_PL
#define PD_LAT_PL 2
#endif
        constexpr int PL = PD_LAT_PL;          // passes in flight
        const int t = threadIdx.x;
        const int q = t % PREC, pp = t / PREC;
        const int px = q % HX, py = q / HX;
        const int X = gx0 - 3 + px, Y = gy0 - 3 + py;
        const bool xy_ok = pp < PPASS && X >= 0 && X < L.nx && Y >= 0 && Y < L.ny;
        const double4* src = A.u_in + (X + (long long)L.nx * Y);
        float4* dst = rec + q + PREC * pp;
        for (int pz0 = 0; pz0 < HZ; pz0 += PPASS * PL) {
            double ux[PL], uy[PL], uz[PL];
            float wv[PL];
            bool ok[PL];
#pragma unroll
            for (int k = 0; k < PL; ++k) {
                const int pz = pz0 + pp + PPASS * k;
                const int Z = gz0 - 3 + pz;
                ok[k] = xy_ok && pz < HZ && Z >= 0 && Z < L.nz_local;
                ux[k] = uy[k] = uz[k] = 0.0;
                wv[k] = 0.f;
                if (ok[k]) {
                    const double4* pu = src + plane * Z;
                    const double2 xy = *reinterpret_cast<const double2*>(pu);
                    ux[k] = xy.x;
                    uy[k] = xy.y;
                    if (NF) {
                        const double2 zw = reinterpret_cast<const double2*>(pu)[1];
                        uz[k] = zw.x;
                        // V_j / V_0 (1 with uniform volumes), negative for a no-failure node
                        const float vf =
                            L.vol_varies ? float(A.xv[(pu - A.u_in)].w * L.inv_v0) : 1.f;
                        wv[k] = zw.y != 0.0 ? -vf : vf;
                    } else {
                        uz[k] = reinterpret_cast<const double*>(pu)[2];
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < PL; ++k) {
                const int pz = pz0 + pp + PPASS * k;
                if (pp < PPASS && pz < HZ)
                    dst[PREC * (pz - pp)] =
                        ok[k] ? make_float4(float(ux[k] - U0.x) * ih, float(uy[k] - U0.y) * ih,
                                            float(uz[k] - U0.z) * ih, wv[k])
                              : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
    }
}

} // namespace
} // namespace pdb
