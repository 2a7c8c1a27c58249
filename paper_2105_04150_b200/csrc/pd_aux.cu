// pd_aux.cu -- small per-node kernels around the fused step: layout packing,
// the Verlet prologue drift, finite checks, connectivity materialisation,
// damage (K3) and tip reductions (K6).  fp64 arithmetic uses explicit __d*_rn
// intrinsics so results are bitwise equal to the reference.
#include <cuda_runtime.h>

#include "pd_device.cuh"
#include "pd_internal.h"

namespace pdb {
namespace {

constexpr int TPB = 256;

inline dim3 grid_for(long long n) { return dim3(unsigned((n + TPB - 1) / TPB)); }

__global__ void pack_xv_kernel(const double* coords, const double* volume, long long n,
                               double4* xv) {
    const long long i = blockIdx.x * (long long)TPB + threadIdx.x;
    if (i < n)
        xv[i] = make_double4(coords[3 * i], coords[3 * i + 1], coords[3 * i + 2], volume[i]);
}

__global__ void pack_u_kernel(const double* u, const uint8_t* nofail, long long n, double4* out) {
    const long long i = blockIdx.x * (long long)TPB + threadIdx.x;
    if (i < n)
        out[i] = make_double4(u[3 * i], u[3 * i + 1], u[3 * i + 2],
                              (nofail && nofail[i]) ? 1.0 : 0.0);
}

__global__ void unpack_u_kernel(const double4* u, long long n, double* out) {
    const long long i = blockIdx.x * (long long)TPB + threadIdx.x;
    if (i < n) {
        const double4 x = u[i];
        out[3 * i] = x.x;
        out[3 * i + 1] = x.y;
        out[3 * i + 2] = x.z;
    }
}

// alive bit k of row i <=> entries[i*N+k] >= 0 (engine.cpp:56-58 skips j < 0)
__global__ void init_alive_kernel(const int32_t* entries, long long n, int N, int W,
                                  uint32_t* alive) {
    const long long w = blockIdx.x * (long long)TPB + threadIdx.x;
    if (w >= n * W)
        return;
    const long long i = w / W;
    const int base = int(w - i * W) * 32;
    const int cnt = N < 32 ? N : 32;
    uint32_t word = 0;
    for (int b = 0; b < cnt; ++b)
        if (entries[i * N + base + b] >= 0)
            word |= 1u << b;
    alive[w] = word;
}

// Memory safety: any live entry must index a node of this context.
__global__ void validate_entries_kernel(const int32_t* entries, long long n, int N,
                                        unsigned long long* bad_row) {
    const long long idx = blockIdx.x * (long long)TPB + threadIdx.x;
    if (idx >= n * N)
        return;
    const int32_t j = entries[idx];
    if (j >= n || (j < 0 && j != -1))
        atomicMin(bad_row, (unsigned long long)(idx / N));
}

// verlet_drift (engine.cpp:221-233) + apply_displacement_positions(s+1)
// (engine.cpp:262-272) ahead of the first fused step of a run.
__global__ void vv_prologue_kernel(DevArgs A) {
    const long long i = A.begin + blockIdx.x * (long long)TPB + threadIdx.x;
    if (i >= A.end)
        return;
    const double dt = A.dt;
    const double half_dt2 = A.half_dt2;
    const double4 u = A.u_in[i];
    const double u0[3] = {u.x, u.y, u.z};
    double un[3];
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        un[ax] = __dadd_rn(__dadd_rn(u0[ax], __dmul_rn(A.v[3 * i + ax], dt)),
                           __dmul_rn(A.a[3 * i + ax], half_dt2));
        if (A.bc_kind && A.bc_kind[3 * i + ax] == PD_BC_DISPLACEMENT)
            un[ax] = __dmul_rn(A.bc_mag[3 * i + ax], ramp_scale(A.ramps[A.bc_ramp[3 * i + ax]],
                                                                A.step + 1));
    }
    const double4 unew = make_double4(un[0], un[1], un[2], u.w);
    A.u_out[i] = unew;
    push_ghost(A, i, unew);
    if (!finite3(un[0], un[1], un[2]))
        atomicMin((unsigned long long*)A.err_step, (unsigned long long)A.step);
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Slab barrier after a step (one thread): publish this rank's non-finite flag
// and the epoch to every rank's sync words, wait until every rank has
// published the epoch, then adopt the smallest flag so all ranks stop at the
// same step (the reference throws in the force pass of that step).
// sync words of a rank: [0, PD_MAX_RANKS) epochs, [PD_MAX_RANKS, 2*PD_MAX_RANKS) flags.
__global__ void slab_sync_kernel(SyncArgs S) {
    if (threadIdx.x != 0 || blockIdx.x != 0)
        return;
    const long long mine = *(volatile long long*)S.err_step;
    __threadfence_system();
    for (int p = 0; p < S.world; ++p)
        *(volatile unsigned long long*)(S.peer_sync[p] + PD_MAX_RANKS + S.rank) =
            (unsigned long long)mine;
    __threadfence_system();
    for (int p = 0; p < S.world; ++p)
        st_release_sys(S.peer_sync[p] + S.rank, S.epoch);
    const unsigned long long t0 = globaltimer();
    long long merged = mine;
    for (int q = 0; q < S.world; ++q) {
        while (ld_acquire_sys(S.my_sync + q) < S.epoch) {
            if (globaltimer() - t0 > (unsigned long long)S.timeout_ns) {
                *(volatile long long*)S.err_step = kPeerTimeout;
                return;
            }
            __nanosleep(200);
        }
        const long long e = (long long)ld_acquire_sys(S.my_sync + PD_MAX_RANKS + q);
        merged = e < merged ? e : merged;
    }
    if (merged != mine)
        *(volatile long long*)S.err_step = merged;
}

// check_state_finite (engine.cpp:23-28)
__global__ void check_finite_kernel(const double4* u, long long begin, long long end,
                                    long long step, long long* err) {
    const long long i = begin + blockIdx.x * (long long)TPB + threadIdx.x;
    if (i >= end)
        return;
    const double4 x = u[i];
    if (!finite3(x.x, x.y, x.z))
        atomicMin((unsigned long long*)err, (unsigned long long)step);
}

__global__ void materialize_entries_kernel(const int32_t* entries, const uint32_t* alive,
                                           long long n, int N, int W, int32_t* out) {
    const long long idx = blockIdx.x * (long long)TPB + threadIdx.x;
    if (idx >= n * N)
        return;
    const long long i = idx / N;
    const int k = int(idx - i * N);
    const uint32_t word = alive[i * W + (k >> 5)];
    out[idx] = ((word >> (k & 31)) & 1u) ? entries[idx] : -1;
}

// local_damage via make_snapshot (formulas.hpp:49-55, io.cpp:243-247)
__global__ void damage_kernel(const int32_t* n_neigh, const int32_t* initial, long long n,
                              double* phi) {
    const long long i = blockIdx.x * (long long)TPB + threadIdx.x;
    if (i >= n)
        return;
    const int32_t init = initial[i];
    phi[i] = init > 0 ? __dsub_rn(1.0, __ddiv_rn((double)n_neigh[i], (double)init)) : 0.0;
}

__global__ void inv_kernel(const double* x, long long n, double* out) {
    const long long i = blockIdx.x * (long long)TPB + threadIdx.x;
    if (i < n)
        out[i] = __ddiv_rn(1.0, x[i]);
}

__global__ void sum_kernel(const int32_t* x, long long n, unsigned long long* out) {
    __shared__ unsigned long long part[TPB / 32];
    unsigned long long acc = 0;
    for (long long i = blockIdx.x * (long long)TPB + threadIdx.x; i < n;
         i += (long long)gridDim.x * TPB)
        acc += (unsigned long long)x[i];
    for (int o = 16; o > 0; o /= 2)
        acc += __shfl_down_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0)
        part[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int w = 0; w < TPB / 32; ++w)
            t += part[w];
        atomicAdd(out, t);
    }
}

// record_tips (engine.cpp:349-370): one thread per tip set, sequential sums
// in set order so the result matches the reference bit for bit.
__global__ void tips_kernel(const double4* u, const double* v, const double* a, const double4* xv,
                            const double* body, const double* ext, int n_sets,
                            const long long* offsets, const long long* nodes, long long step,
                            pd_tip_record* out) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_sets)
        return;
    pd_tip_record r;
    r.step = step;
    for (int ax = 0; ax < 3; ++ax)
        r.mean_u[ax] = r.mean_v[ax] = r.mean_a[ax] = r.body_force_sum[ax] =
            r.external_force_sum[ax] = 0.0;
    const long long b = offsets[s], e = offsets[s + 1];
    for (long long t = b; t < e; ++t) {
        const long long i = nodes[t];
        const double4 ui = u[i];
        const double uu[3] = {ui.x, ui.y, ui.z};
        const double vol = xv[i].w;
        for (int ax = 0; ax < 3; ++ax) {
            r.mean_u[ax] = __dadd_rn(r.mean_u[ax], uu[ax]);
            r.mean_v[ax] = __dadd_rn(r.mean_v[ax], v[3 * i + ax]);
            r.mean_a[ax] = __dadd_rn(r.mean_a[ax], a[3 * i + ax]);
            r.body_force_sum[ax] = __dadd_rn(r.body_force_sum[ax], __dmul_rn(body[3 * i + ax], vol));
            r.external_force_sum[ax] =
                __dadd_rn(r.external_force_sum[ax], __dmul_rn(ext[3 * i + ax], vol));
        }
    }
    if (e > b) {
        const double inv = __ddiv_rn(1.0, (double)(e - b));
        for (int ax = 0; ax < 3; ++ax) {
            r.mean_u[ax] = __dmul_rn(r.mean_u[ax], inv);
            r.mean_v[ax] = __dmul_rn(r.mean_v[ax], inv);
            r.mean_a[ax] = __dmul_rn(r.mean_a[ax], inv);
        }
    }
    out[s] = r;
}

// u, v, a and force x volume of listed rows (multi-rank tip records; the
// products are record_tips' own, engine.cpp:357-360)
__global__ void node_values_kernel(const double4* u, const double* v, const double* a,
                                   const double4* xv, const double* body, const double* ext,
                                   const long long* rows, long long count, double* out) {
    const long long k = blockIdx.x * (long long)TPB + threadIdx.x;
    if (k >= count)
        return;
    const long long i = rows[k];
    const double4 ui = u[i];
    const double vol = xv[i].w;
    double* o = out + 15 * k;
    o[0] = ui.x;
    o[1] = ui.y;
    o[2] = ui.z;
    for (int ax = 0; ax < 3; ++ax) {
        o[3 + ax] = v[3 * i + ax];
        o[6 + ax] = a[3 * i + ax];
        o[9 + ax] = __dmul_rn(body[3 * i + ax], vol);
        o[12 + ax] = __dmul_rn(ext[3 * i + ax], vol);
    }
}

// rows whose materialised entries differ from the uploaded ones (unordered list)
__global__ void changed_rows_kernel(const int32_t* cur, const int32_t* orig, long long n, int N,
                                    int* list, unsigned long long* count) {
    const long long i = blockIdx.x * (long long)TPB + threadIdx.x;
    if (i >= n)
        return;
    for (int k = 0; k < N; ++k)
        if (cur[i * N + k] != orig[i * N + k]) {
            list[atomicAdd(count, 1ull)] = int(i);
            return;
        }
}

__global__ void gather_list_rows_kernel(const int32_t* cur, const int* list, long long m, int N,
                                        int32_t* out) {
    const long long r = blockIdx.x;
    if (r >= m)
        return;
    const long long i = list[r];
    for (int k = threadIdx.x; k < N; k += blockDim.x)
        out[r * N + k] = cur[i * N + k];
}

// The reference's stand-alone integrators over flat n x 3 host-layout arrays
// (engine.cpp:187-252), in its expression order (-fmad=false):
//   op 0 verlet_drift:   u = u + v dt + a (dt dt / 2)
//   op 1 verlet_kick:    v_half = v + a (dt/2); a = (F - v_half eta) (1/rho);
//                        v = v_half + a (dt/2)
//   op 2 step_euler:     a = F (1/rho); v = v_old + a dt; u = u + v_old dt
//   op 3 step_euler_cromer: a = F (1/rho); v = v + a dt; u = u + v_new dt
// with F = body_force + external_force (engine.cpp:173-175).
__global__ void integrate_kernel(IntegrateArgs I) {
    const long long i = blockIdx.x * (long long)TPB + threadIdx.x;
    if (i >= I.n)
        return;
    const double dt = I.dt;
    const double inv = I.op == 0 ? 0.0 : __ddiv_rn(1.0, I.density[i]);
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        const long long k = 3 * i + ax;
        if (I.op == 0) {
            I.u[k] = __dadd_rn(__dadd_rn(I.u[k], __dmul_rn(I.v[k], dt)),
                               __dmul_rn(I.a[k], __ddiv_rn(__dmul_rn(dt, dt), 2.0)));
            continue;
        }
        const double F = __dadd_rn(I.body[k], I.ext[k]);
        if (I.op == 1) {
            const double half = __ddiv_rn(dt, 2.0);
            const double vh = __dadd_rn(I.v[k], __dmul_rn(I.a[k], half));
            const double an = __dmul_rn(__dsub_rn(F, __dmul_rn(vh, I.damping)), inv);
            I.a[k] = an;
            I.v[k] = __dadd_rn(vh, __dmul_rn(an, half));
        } else {
            const double acc = __dmul_rn(F, inv);
            const double v_old = I.v[k];
            const double v_new = __dadd_rn(v_old, __dmul_rn(acc, dt));
            I.a[k] = acc;
            I.v[k] = v_new;
            I.u[k] = __dadd_rn(I.u[k], __dmul_rn(I.op == 2 ? v_old : v_new, dt));
        }
    }
}

// apply_displacement_positions / _kinematics and accumulate_external_force
// (engine.cpp:262-297) over the node-axes, selected by the bits of B.ops
__global__ void boundary_kernel(BoundaryArgs B) {
    const long long k = blockIdx.x * (long long)TPB + threadIdx.x;
    if (k >= 3 * B.n)
        return;
    const int kind = B.kind[k];
    if (kind == PD_BC_FREE)
        return;
    const DevRamp r = B.ramps[B.ramp_id[k]];
    const double mag = B.mag[k];
    if (kind == PD_BC_DISPLACEMENT) {
        if (B.ops & 1)
            B.u[k] = __dmul_rn(mag, ramp_scale(r, B.step));
        if (B.ops & 2) {
            B.v[k] = __ddiv_rn(__dmul_rn(mag, ramp_rate(r, B.step)), B.dt);
            B.a[k] = __ddiv_rn(__dmul_rn(mag, ramp_accel(r, B.step)), __dmul_rn(B.dt, B.dt));
        }
    } else if (kind == PD_BC_FORCE && (B.ops & 4)) {
        B.ext[k] = __dadd_rn(B.ext[k], __dmul_rn(mag, ramp_scale(r, B.step)));
    }
}

} // namespace

void launch_changed_rows(const int32_t* cur, const int32_t* orig, long long n, int N, int* list,
                         unsigned long long* count, cudaStream_t st) {
    if (n > 0)
        changed_rows_kernel<<<grid_for(n), TPB, 0, st>>>(cur, orig, n, N, list, count);
}

void launch_gather_list_rows(const int32_t* cur, const int* list, long long m, int N, int32_t* out,
                             cudaStream_t st) {
    if (m > 0)
        gather_list_rows_kernel<<<unsigned(m), 128, 0, st>>>(cur, list, m, N, out);
}

void launch_node_values(const double4* u, const double* v, const double* a, const double4* xv,
                        const double* body, const double* ext, const long long* rows,
                        long long count, double* out, cudaStream_t st) {
    if (count > 0)
        node_values_kernel<<<grid_for(count), TPB, 0, st>>>(u, v, a, xv, body, ext, rows, count,
                                                            out);
}

void launch_pack_xv(const double* coords, const double* volume, long long n, double4* xv,
                    cudaStream_t st) {
    if (n > 0)
        pack_xv_kernel<<<grid_for(n), TPB, 0, st>>>(coords, volume, n, xv);
}

void launch_pack_u(const double* u, const uint8_t* nofail, long long n, double4* out,
                   cudaStream_t st) {
    if (n > 0)
        pack_u_kernel<<<grid_for(n), TPB, 0, st>>>(u, nofail, n, out);
}

void launch_unpack_u(const double4* u, long long n, double* out, cudaStream_t st) {
    if (n > 0)
        unpack_u_kernel<<<grid_for(n), TPB, 0, st>>>(u, n, out);
}

void launch_init_alive(const int32_t* entries, long long n, int N, int W, uint32_t* alive,
                       cudaStream_t st) {
    if (n > 0)
        init_alive_kernel<<<grid_for(n * W), TPB, 0, st>>>(entries, n, N, W, alive);
}

void launch_validate_entries(const int32_t* entries, long long n, int N,
                             unsigned long long* bad_row, cudaStream_t st) {
    if (n > 0)
        validate_entries_kernel<<<grid_for(n * N), TPB, 0, st>>>(entries, n, N, bad_row);
}

// Force the (lazily loaded) module functions of this unit in now: with CUDA
// lazy loading the first launch of a kernel may wait for the whole device,
// which deadlocks against a peer rank's spinning slab_sync_kernel.
template <class K> static void preload(K k) {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, reinterpret_cast<const void*>(k));
}

void preload_aux() {
    preload(pack_xv_kernel);
    preload(pack_u_kernel);
    preload(unpack_u_kernel);
    preload(init_alive_kernel);
    preload(validate_entries_kernel);
    preload(vv_prologue_kernel);
    preload(slab_sync_kernel);
    preload(check_finite_kernel);
    preload(materialize_entries_kernel);
    preload(damage_kernel);
    preload(inv_kernel);
    preload(sum_kernel);
    preload(tips_kernel);
    preload(node_values_kernel);
    preload(changed_rows_kernel);
    preload(gather_list_rows_kernel);
}

void launch_slab_sync(const SyncArgs& S, cudaStream_t st) {
    slab_sync_kernel<<<1, 32, 0, st>>>(S);
}

void launch_vv_prologue(const DevArgs& A, cudaStream_t st) {
    if (A.end > A.begin)
        vv_prologue_kernel<<<grid_for(A.end - A.begin), TPB, 0, st>>>(A);
}

void launch_check_finite(const double4* u, long long begin, long long end, long long step,
                         long long* err, cudaStream_t st) {
    if (end > begin)
        check_finite_kernel<<<grid_for(end - begin), TPB, 0, st>>>(u, begin, end, step, err);
}

void launch_materialize_entries(const int32_t* entries, const uint32_t* alive, long long n, int N,
                                int W, int32_t* out, cudaStream_t st) {
    if (n > 0)
        materialize_entries_kernel<<<grid_for(n * N), TPB, 0, st>>>(entries, alive, n, N, W, out);
}

void launch_damage(const int32_t* n_neigh, const int32_t* initial, long long n, double* phi,
                   cudaStream_t st) {
    if (n > 0)
        damage_kernel<<<grid_for(n), TPB, 0, st>>>(n_neigh, initial, n, phi);
}

void launch_inv(const double* x, long long n, double* out, cudaStream_t st) {
    if (n > 0)
        inv_kernel<<<grid_for(n), TPB, 0, st>>>(x, n, out);
}

void launch_sum(const int32_t* x, long long n, unsigned long long* out, cudaStream_t st) {
    long long blocks = (n + TPB - 1) / TPB;
    if (blocks > 148 * 8)
        blocks = 148 * 8;
    if (n > 0)
        sum_kernel<<<unsigned(blocks), TPB, 0, st>>>(x, n, out);
}

void launch_tips(const double4* u, const double* v, const double* a, const double4* xv,
                 const double* body, const double* ext, int n_sets, const long long* offsets,
                 const long long* nodes, long long step, pd_tip_record* out, cudaStream_t st) {
    if (n_sets > 0)
        tips_kernel<<<(n_sets + 63) / 64, 64, 0, st>>>(u, v, a, xv, body, ext, n_sets, offsets,
                                                       nodes, step, out);
}

void launch_integrate(const IntegrateArgs& I, cudaStream_t st) {
    if (I.n > 0)
        integrate_kernel<<<grid_for(I.n), TPB, 0, st>>>(I);
}

void launch_boundary(const BoundaryArgs& B, cudaStream_t st) {
    if (B.n > 0)
        boundary_kernel<<<grid_for(3 * B.n), TPB, 0, st>>>(B);
}

} // namespace pdb
