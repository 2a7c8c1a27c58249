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

#include <cmath>
#include <utility>

#include "pd_device.cuh"
#include "pd_internal.h"

namespace pdb {

namespace {

constexpr int BX = 16, BY = 4, BZ = 8;                // brick (threads)
constexpr int HX = BX + 6, HY = BY + 6, HZ = BZ + 6;  // halo box (records)
constexpr int NREC = HX * HY * HZ;                    // 3080
constexpr int TT = BX * BY * BZ;                      // 512
constexpr int NPAT = 122;

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

struct Acc {
    float fx, fy, fz;
    unsigned dead[4];
};

template <int C>
__device__ __forceinline__ void slot(const float4* own, const float4& ri, const uint4& m, float sc,
                                     Acc& a) {
    constexpr int dx = pat(C, 0), dy = pat(C, 1), dz = pat(C, 2);
    constexpr int r2 = dx * dx + dy * dy + dz * dz;
    constexpr float len = root(r2);
    constexpr float rr = 1.0f / root(r2);
    constexpr int off = dx + HX * (dy + HY * dz);
    constexpr int word = C >> 5;
    constexpr unsigned bit = 1u << (C & 31);
    const unsigned mw = word == 0 ? m.x : (word == 1 ? m.y : (word == 2 ? m.z : m.w));
    const bool live = (mw & bit) != 0;
    // branch free: a dead slot's record may be anything finite (an
    // out-of-domain box record is 0); its contribution is selected away
    const float4 rj = own[off];
    const float hx = rj.x - ri.x, hy = rj.y - ri.y, hz = rj.z - ri.z;  // eta / spacing
    const float cx = hx + float(dx), cy = hy + float(dy), cz = hz + float(dz);
    // eta.(2 xi + eta), cancellation free
    float num = hz * (hz + float(2 * dz));
    num = fmaf(hy, hy + float(2 * dy), num);
    num = fmaf(hx, hx + float(2 * dx), num);
    const float cur2 = num + float(r2);
    const float rc = rsqrt_approx(cur2);
    const float s = num * rr * rcp_approx(fmaf(cur2, rc, len));
    const float scale = s * rc;
    // predicated tail: live = bit set; break = live && s >= s_c (bond_contribution's
    // PMB break, engine.cpp:90-98) clears the bit; otherwise a live slot adds its force
    unsigned& dead = a.dead[word];
    asm("{\n\t.reg .pred pl, pb, pc;\n\t"
        "setp.ne.u32 pl, %4, 0;\n\t"
        "setp.ge.and.f32 pb, %5, %6, pl;\n\t"
        "setp.lt.and.f32 pc, %5, %6, pl;\n\t"
        "@pb or.b32 %0, %0, %7;\n\t"
        "@pc fma.rn.f32 %1, %8, %11, %1;\n\t"
        "@pc fma.rn.f32 %2, %9, %11, %2;\n\t"
        "@pc fma.rn.f32 %3, %10, %11, %3;\n\t}"
        : "+r"(dead), "+f"(a.fx), "+f"(a.fy), "+f"(a.fz)
        : "r"(mw & bit), "f"(s), "f"(sc), "r"(bit), "f"(cx), "f"(cy), "f"(cz), "f"(scale));
    (void)live;
}

template <int... C>
__device__ __forceinline__ void all_slots(std::integer_sequence<int, C...>, const float4* own,
                                          const float4& ri, const uint4& m, float sc, Acc& a) {
    (slot<C>(own, ri, m, sc, a), ...);
}

template <int MODE>
__global__ void __launch_bounds__(TT, 2) lattice_step_kernel(DevArgs A, LatticeArgs L) {
    if (MODE != 0 && *(volatile long long*)A.err_step != kNoError)
        return;
    extern __shared__ float4 rec[];  // NREC records (49 KB: dynamic)
    const int nbx = (L.nx + BX - 1) / BX, nby = (L.ny + BY - 1) / BY;
    const int b = blockIdx.x;
    const int bxi = b % nbx, byi = (b / nbx) % nby, bzi = b / (nbx * nby);
    const int gx0 = bxi * BX, gy0 = byi * BY, gz0 = L.z0 + bzi * BZ;
    const int tx = threadIdx.x % BX, ty = (threadIdx.x / BX) % BY, tz = threadIdx.x / (BX * BY);
    const int gx = gx0 + tx, gy = gy0 + ty, gz = gz0 + tz;
    const bool active = gx < L.nx && gy < L.ny && gz < L.z0 + L.nz_own;
    const long long plane = (long long)L.nx * L.ny;
    const long long i = gx + (long long)L.nx * gy + plane * gz;
    // the row mask streams in while the halo is staged
    uint4 m = active ? __ldcs(L.mask + i) : make_uint4(0, 0, 0, 0);

    // 1. stage the halo box: fp32 (u - U_brick) / spacing
    const double4 U0 = A.u_in[gx0 + (long long)L.nx * gy0 + plane * gz0];
    const double ih = L.inv_h;
    for (int p = threadIdx.x; p < NREC; p += TT) {
        const int px = p % HX, py = (p / HX) % HY, pz = p / (HX * HY);
        const int X = gx0 - 3 + px, Y = gy0 - 3 + py, Z = gz0 - 3 + pz;
        float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
        if (X >= 0 && X < L.nx && Y >= 0 && Y < L.ny && Z >= 0 && Z < L.nz_local) {
            const double4 u = A.u_in[X + (long long)L.nx * Y + plane * Z];
            r = make_float4(float((u.x - U0.x) * ih), float((u.y - U0.y) * ih),
                            float((u.z - U0.z) * ih), 0.f);
        }
        rec[p] = r;
    }
    __syncthreads();
    if (!active)
        return;

    // 2. the node's bonds: 122 pattern slots, unrolled at compile time
    const float4* own = rec + (tx + 3) + HX * ((ty + 3) + HY * (tz + 3));
    const float4 ri = *own;
    Acc a{0.f, 0.f, 0.f, {0u, 0u, 0u, 0u}};
    all_slots(std::make_integer_sequence<int, NPAT>{}, own, ri, m, L.sc, a);
    const unsigned d0 = a.dead[0], d1 = a.dead[1], d2 = a.dead[2], d3 = a.dead[3];
    if (d0 | d1 | d2 | d3) {
        L.mask[i] = make_uint4(m.x & ~d0, m.y & ~d1, m.z & ~d2, m.w & ~d3);
        A.n_neigh[i] -= __popc(d0) + __popc(d1) + __popc(d2) + __popc(d3);
    }
    const double fx = double(a.fx * L.cv), fy = double(a.fy * L.cv), fz = double(a.fz * L.cv);

    // 3. fp64 epilogue
    if (MODE == 0) {
        A.body_force[3 * i] = fx;
        A.body_force[3 * i + 1] = fy;
        A.body_force[3 * i + 2] = fz;
        return;
    }
    node_epilogue<MODE>(A, i, A.u_in[i], fx, fy, fz);
}

// row -> mask: bit c set for every live entry whose offset is pattern slot c;
// *bad = 1 when a row holds a bond outside the pattern
__global__ void lattice_mask_kernel(const int32_t* entries, long long begin, long long end, int N,
                                    int nx, int ny, uint4* mask, int* bad) {
    const long long i = begin + blockIdx.x * 256LL + threadIdx.x;
    if (i >= end)
        return;
    const long long plane = (long long)nx * ny;
    const int ix = int(i % nx), iy = int((i / nx) % ny), iz = int(i / plane);
    unsigned w[4] = {0u, 0u, 0u, 0u};
    for (int k = 0; k < N; ++k) {
        const int32_t j = entries[i * N + k];
        if (j < 0)
            continue;
        const int dx = int(j % nx) - ix, dy = int((j / nx) % ny) - iy, dz = int(j / plane) - iz;
        const int r2 = dx * dx + dy * dy + dz * dz;
        if (r2 == 0 || r2 > 9) {
            atomicExch(bad, 1);
            return;
        }
        // slot index of (dx, dy, dz): count pattern offsets before it
        int c = 0;
        for (int z = -3; z <= 3; ++z)
            for (int y = -3; y <= 3; ++y)
                for (int x = -3; x <= 3; ++x) {
                    const int q = x * x + y * y + z * z;
                    if (q == 0 || q > 9)
                        continue;
                    if (z < dz || (z == dz && (y < dy || (y == dy && x < dx))))
                        ++c;
                }
        w[c >> 5] |= 1u << (c & 31);
    }
    mask[i] = make_uint4(w[0], w[1], w[2], w[3]);
}

// entries in the reference layout: the uploaded row with -1 where the mask bit
// of the slot's offset is clear
__global__ void lattice_materialize_kernel(const int32_t* entries0, const uint4* mask,
                                           long long begin, long long end, long long n, int N,
                                           int nx, int ny, int32_t* out) {
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
            int c = 0;
            for (int z = -3; z <= 3; ++z)
                for (int y = -3; y <= 3; ++y)
                    for (int x = -3; x <= 3; ++x) {
                        const int q = x * x + y * y + z * z;
                        if (q == 0 || q > 9)
                            continue;
                        if (z < dz || (z == dz && (y < dy || (y == dy && x < dx))))
                            ++c;
                    }
            if (!((w[c >> 5] >> (c & 31)) & 1u))
                v = -1;
        }
        out[i * N + k] = v;
    }
}

template <class K> void preload_fn(K k) {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, reinterpret_cast<const void*>(k));
}

// the halo box exceeds the 48 KB default: lift the limit once per process
cudaError_t configure_smem() {
    static bool done = false;
    if (done)
        return cudaSuccess;
    const int smem = int(sizeof(float4) * NREC);
    cudaError_t e = cudaSuccess;
    for (const void* k : {reinterpret_cast<const void*>(lattice_step_kernel<0>),
                          reinterpret_cast<const void*>(lattice_step_kernel<1>),
                          reinterpret_cast<const void*>(lattice_step_kernel<2>),
                          reinterpret_cast<const void*>(lattice_step_kernel<3>)})
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    done = e == cudaSuccess;
    return e;
}

} // namespace

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
    const double tol = 1e-9 * h;
    for (long long i = 0; i < n; ++i) {
        const long long kx = i % nx, ky = (i / nx) % ny, kz = i / plane;
        if (std::fabs(coords[3 * i] - (ox + double(kx) * h)) > tol ||
            std::fabs(coords[3 * i + 1] - (oy + double(ky) * h)) > tol ||
            std::fabs(coords[3 * i + 2] - (oz + double(kz) * h)) > tol)
            return false;
    }
    if (own_begin % plane != 0 || own_end % plane != 0)
        return false;  // owned range of a slab: whole planes
    L.nx = int(nx);
    L.ny = int(ny);
    L.nz_local = int(nz);
    L.z0 = int(own_begin / plane);
    L.nz_own = int((own_end - own_begin) / plane);
    L.h = h;
    L.inv_h = 1.0 / h;
    return true;
}

cudaError_t lattice_build_masks(const int32_t* entries, long long begin, long long end, int N,
                                const LatticeArgs& L, uint4* mask, int* bad, cudaStream_t st) {
    if (end > begin)
        lattice_mask_kernel<<<unsigned((end - begin + 255) / 256), 256, 0, st>>>(
            entries, begin, end, N, L.nx, L.ny, mask, bad);
    return cudaGetLastError();
}

cudaError_t launch_lattice(const DevArgs& A, const LatticeArgs& L, int mode, cudaStream_t st) {
    const int nbx = (L.nx + BX - 1) / BX, nby = (L.ny + BY - 1) / BY, nbz = (L.nz_own + BZ - 1) / BZ;
    const unsigned blocks = unsigned(nbx * nby * nbz);
    if (blocks == 0)
        return cudaSuccess;
    cudaError_t e = configure_smem();
    if (e != cudaSuccess)
        return e;
    const size_t smem = sizeof(float4) * NREC;
    switch (mode) {
    case 0: lattice_step_kernel<0><<<blocks, TT, smem, st>>>(A, L); break;
    case 1: lattice_step_kernel<1><<<blocks, TT, smem, st>>>(A, L); break;
    case 2: lattice_step_kernel<2><<<blocks, TT, smem, st>>>(A, L); break;
    default: lattice_step_kernel<3><<<blocks, TT, smem, st>>>(A, L); break;
    }
    return cudaGetLastError();
}

cudaError_t launch_lattice_materialize(const int32_t* entries0, const uint4* mask, long long begin,
                                       long long end, long long n, int N, const LatticeArgs& L,
                                       int32_t* out, cudaStream_t st) {
    if (n > 0)
        lattice_materialize_kernel<<<unsigned((n + 255) / 256), 256, 0, st>>>(
            entries0, mask, begin, end, n, N, L.nx, L.ny, out);
    return cudaGetLastError();
}

void preload_lattice() {
    preload_fn(lattice_step_kernel<0>);
    preload_fn(lattice_step_kernel<1>);
    preload_fn(lattice_step_kernel<2>);
    preload_fn(lattice_step_kernel<3>);
    preload_fn(lattice_mask_kernel);
    preload_fn(lattice_materialize_kernel);
    configure_smem();
}

} // namespace pdb
