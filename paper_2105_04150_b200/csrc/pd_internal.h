// pd_internal.h -- host-side launcher declarations shared by the .cu units.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdio>
#include <string>
#include <vector>

#include "pd_device.cuh"
#include "pd_fast.cuh"

namespace pdb {

// The step kernel the last launch on this host thread ran, as
// "<family><template values>" (pd_ctx_kernel; the parity tests assert which
// instantiation they exercised).
inline thread_local const char* t_last_kernel = "";
template <int Family, int... V> const char* kernel_name(const char* base) {
    static const std::string s = [base] {
        std::string r = base;
        r += '<';
        ((r += std::to_string(V) + ","), ...);
        r.back() = '>';
        return r;
    }();
    return s.c_str();
}

// pd_xfer.cpp: large host <-> device copies through pinned bounce buffers
// (synchronous with respect to the host on return)
cudaError_t h2d_large(void* dev, const void* host, size_t bytes, cudaStream_t s);
cudaError_t d2h_large(void* host, const void* dev, size_t bytes, cudaStream_t s);

// pd_io.cpp: binary container writer (reference io.cpp BinWriter), host or
// device sections
struct StreamWriter {
    FILE* f = nullptr;
    std::string path;
    void* bounce = nullptr;
    bool failed = false;
    ~StreamWriter();
    int open(const char* p);
    int bytes(const void* data, uint64_t len);
    template <class T> int pod(T v) { return bytes(&v, sizeof(T)); }
    int section_host(uint32_t id, const void* data, uint64_t len);
    int section_device(uint32_t id, const void* dev, uint64_t len, cudaStream_t s);
    int close();
};

// pd_xfer.cpp: process-wide cache of device blocks.  Contexts of the same
// model size (the calibration outer loop, repeated simulate() calls) reuse
// mapped memory instead of paying cudaFree/cudaMalloc of ~10 GB each time.
cudaError_t dev_alloc(void** p, size_t bytes);
void dev_free(void* p, size_t bytes);
void release_cached_blocks();

// pd_io.cpp: the pdsnap text writer (multi-threaded formatting, in-order write)
int write_snapshot_file(const char* path, int64_t step, int64_t n, const double* coords,
                        const double* u, const double* v, const double* phi);

// Owning device buffer, resized on demand.
template <class T> struct DevBuf {
    T* p = nullptr;
    size_t count = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p)
            dev_free(p, count * sizeof(T));
        p = nullptr;
        count = 0;
    }
    cudaError_t alloc(size_t n) {
        if (n == count && p)
            return cudaSuccess;
        release();
        if (n == 0)
            return cudaSuccess;
        void* q = nullptr;
        const cudaError_t e = dev_alloc(&q, n * sizeof(T));
        if (e == cudaSuccess) {
            p = static_cast<T*>(q);
            count = n;
        }
        return e;
    }
    cudaError_t upload(const T* host, size_t n, cudaStream_t st) {
        cudaError_t e = alloc(n);
        if (e != cudaSuccess || n == 0)
            return e;
        return h2d_large(p, host, n * sizeof(T), st);
    }
};

// pd_host.cu: record the message pd_last_error() returns; returns code.
int set_error(int code, const char* msg);

// pd_layout.cu -- the fast path tile layout (pd_fast.cuh), built on the device
struct FastLayoutDev {
    int T = 0, n_tiles = 0, max_halo = 0;
    long long total_slots = 0;
    DevBuf<int> perm, inv, tile_of, tile_start, kmax8, wgroups, halo, nf_start;
    DevBuf<unsigned short> own_slot, lidx;
    DevBuf<unsigned short> origk;  // Morton tiles: a compact slot's position in the original row
    DevBuf<long long> halo_off, slot_off;
    DevBuf<float> hist32, lambda32, beta32;
    DevBuf<uint8_t> btype_c;
    std::vector<int> inv_host;  // local node -> internal row
};
struct FastLayoutIn {
    long long n = 0, own_begin = 0, own_end = 0;
    int N = 0, T = 0;
    bool history = false;
    const double4* xv = nullptr;     // local order
    const int32_t* entries = nullptr;
    const uint8_t* nofail = nullptr;
    const double* hist = nullptr;
    const uint8_t* btype = nullptr;
    const double* lambda = nullptr;
    const double* beta = nullptr;
};
// *error = 1 when a tile's neighbourhood exceeds FAST_MAX_HALO records
cudaError_t gpu_build_layout(FastLayoutDev& L, const FastLayoutIn& in, int* error,
                             cudaStream_t s);


void fast_set_laws(const DevLaw* laws, int n, cudaStream_t stream);
cudaError_t launch_fast(const DevArgs& A, const FastDev& F, int mode, int kind, int tiles,
                        cudaStream_t st);
template <class T, int W>
void launch_gather_rows(const T* in, T* out, const int* map, long long n, cudaStream_t st);
void launch_fast_materialize(const unsigned short* origk, const int32_t* entries0, const int* inv,
                             const int* tile_of,
                             const int* tile_start, const long long* slot_off, int T,
                             const unsigned short* lidx, const float* hist32, long long n, int N,
                             int32_t* entries_out, double* hist_out, cudaStream_t st);

// every kernel of the library loaded up front (multi-GPU runs, see pd_aux.cu)
void preload_aux();
void preload_exact();
void preload_fast();

// pd_lattice.cu -- the fast path on structured lattices (implicit connectivity)
struct NlRegLaw {  // one n-linear law of <= 3 breakpoints, fp32 (pd_lattice.cu)
    float c = 0.f, sc = 0.f, bp0 = 0.f, bp1 = 0.f, f0 = 0.f, f1 = 0.f;
    float sl0 = 0.f, sl1 = 0.f, sl2 = 0.f;
    float a1 = 0.f, a2 = 0.f;  // segment k as a_k + sl_k s (a_0 = 0), from fp64 on the host
    int cvx1 = 0, cvx2 = 0;    // kink k convex (slope rises): the envelope takes max there
    int nbp = 1;
    int hist = 0;
};
struct LatticeArgs {
    int nx = 0, ny = 0, nz_local = 0;  // local lattice (x fastest, z slowest)
    int z0 = 0, nz_own = 0;            // owned planes [z0, z0 + nz_own)
    double h = 1.0, inv_h = 1.0;       // spacing
    double ox = 0, oy = 0, oz = 0;     // origin
    float sc = 0.f, cv = 0.f;          // PMB critical stretch, c * V
    int cfg = 0;                       // brick / occupancy configuration (PD_LAT_CFG)
    int nf = 0;                        // no-failure nodes or per-node volumes present
    int vol_varies = 0;                // volumes differ (records carry V_j / V_0)
    double inv_v0 = 1.0;               // 1 / V_0 (node 0's volume)
    uint4* mask = nullptr;             // per node: live bonds over the 122-offset pattern
    // NL (n-linear laws / bond types / lambda / beta): brick-major slot arrays
    // (pd_lattice.cu slot_base)
    int nl = 0;
    long long n_local = 0;
    float* hist = nullptr;
    uint8_t* btype = nullptr;
    float* lam = nullptr;  // lambda * beta (either may be absent)
    int multi = 1;   // per-bond laws from constant memory; else the register law rl
    NlRegLaw rl;
    signed char pat[128][4];  // the offset pattern (dx, dy, dz, |d|^2): the rare slow paths
    // typed: several laws (<= 8, <= 3 breakpoints each) chosen by bond type on
    // the unrolled kernel; the history words carry the type in their low 3
    // bits and tl holds per type (c, sl_1, a_1, +-s_c), (sl_2, a_2, cvx_1, cvx_2)
    int typed = 0;
    int nlbz = 8;  // z planes of the NL bricks: the per-bond layout (pd_lattice.cuh slot_base)
    float4 tl[16];
    int prefetch = 0;         // NL: bulk L2 prefetch of a brick's per-bond streams (PD_NLU_PF=1; measured slower than the per-slot prefetch)
};
bool lattice_detect(const double* coords, long long n, long long own_begin, long long own_end,
                    LatticeArgs& L);
cudaError_t lattice_build_masks(const double4* xv, long long n, const int32_t* entries,
                                long long begin, long long end, int N, const LatticeArgs& L,
                                uint4* mask, int* bad, const double* hist, const uint8_t* btype,
                                const double* lambda, const double* beta, cudaStream_t st);
void lattice_set_laws(const DevLaw* laws, int n, LatticeArgs& L, cudaStream_t st);
long long lattice_slot_count(const LatticeArgs& L);  // length of the brick-major slot arrays
// true when the unrolled lattice kernels' branch-free envelope
// op1(l_0, op2(l_1, l_2)) (pd_lattice_nlu.cuh nl_law) reproduces
// envelope_force (formulas.hpp:77-89) of this law on [0, s_c]; false for
// more than 3 breakpoints and for shapes such as hardening-then-softening
bool lattice_minmax_ok(const double* bp, const double* f, int nbp);
cudaError_t launch_lattice(const DevArgs& A, const LatticeArgs& L, int mode, cudaStream_t st);
// Small lattice models: one cooperative launch advancing `steps` steps
// (pd_lattice.cu lattice_small_kernel).  Step k reads u[k & 1] and writes
// u[(k & 1) ^ 1]; forces are stored and the next drift done (VV) as
// store_last / drift_last say on the last step only, every other step drifts
// and stores nothing.  bar counts CTA arrivals: step k waits for
// bar_base + k * CTAs.
struct SmallArgs {
    double4* u[2];
    unsigned long long* bar;
    unsigned long long bar_base;
    int steps;
    int store_last;
    int drift_last;
    int n_ramps;  // ramp table length, <= 32 (the kernel evaluates each ramp once per step)
};
// CTAs the small kernel needs (0: not applicable) and whether they are all
// co-resident for this mode / BC / NF combination
long long lattice_small_ctas(const LatticeArgs& L);
bool lattice_small_fits(const LatticeArgs& L, int mode, bool bc);
cudaError_t launch_lattice_small(const DevArgs& A, const LatticeArgs& L, int mode, const SmallArgs& S,
                                 cudaStream_t st);
cudaError_t launch_lattice_materialize(const int32_t* entries0, const uint4* mask, long long begin,
                                       long long end, long long n, int N, const LatticeArgs& L,
                                       int32_t* out, double* hist_out, cudaStream_t st);
void preload_lattice();
// pd_lattice_nlu<M>.cu: the unrolled n-linear kernel per integrator mode
cudaError_t launch_nlu_m0(const DevArgs& A, const LatticeArgs& L, cudaStream_t st);
cudaError_t launch_nlu_m1(const DevArgs& A, const LatticeArgs& L, cudaStream_t st);
cudaError_t launch_nlu_m2(const DevArgs& A, const LatticeArgs& L, cudaStream_t st);
cudaError_t launch_nlu_m3(const DevArgs& A, const LatticeArgs& L, cudaStream_t st);
void preload_nlu_m0();
void preload_nlu_m1();
void preload_nlu_m2();
void preload_nlu_m3();

// pd_exact.cu
// pmb: one PMB law, no bond types, no lambda / beta (A.pmb_c, A.pmb_sc set)
cudaError_t launch_exact(const DevArgs& A, int mode, bool node_sum, bool pmb, cudaStream_t st);

// pd_aux.cu
struct SyncArgs {
    unsigned long long* peer_sync[PD_MAX_RANKS];  // every rank's sync words (own included)
    unsigned long long* my_sync;
    long long* err_step;
    int rank, world;
    unsigned long long epoch;
    long long timeout_ns;
};
void launch_slab_sync(const SyncArgs& S, cudaStream_t st);

// stand-alone integrators and boundary passes (pd_aux.cu; C ABI in pd_host.cu)
struct IntegrateArgs {
    double* u;
    double* v;
    double* a;
    const double* body;
    const double* ext;
    const double* density;
    long long n;
    double dt, damping;
    int op;  // 0 verlet_drift, 1 verlet_kick, 2 step_euler, 3 step_euler_cromer
};
struct BoundaryArgs {
    double* u;
    double* v;
    double* a;
    double* ext;
    const uint8_t* kind;
    const double* mag;
    const uint8_t* ramp_id;
    const DevRamp* ramps;
    long long n, step;
    double dt;
    int ops;  // bit 0 positions, bit 1 kinematics, bit 2 external force
};
void launch_integrate(const IntegrateArgs& I, cudaStream_t st);
void launch_boundary(const BoundaryArgs& B, cudaStream_t st);
void launch_changed_rows(const int32_t* cur, const int32_t* orig, long long n, int N, int* list,
                         unsigned long long* count, cudaStream_t st);
void launch_gather_list_rows(const int32_t* cur, const int* list, long long m, int N, int32_t* out,
                             cudaStream_t st);
void launch_node_values(const double4* u, const double* v, const double* a, const double4* xv,
                        const double* body, const double* ext, const long long* rows,
                        long long count, double* out, cudaStream_t st);
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
void launch_inv(const double* x, long long n, double* out, cudaStream_t st);
void launch_tips(const double4* u, const double* v, const double* a, const double4* xv,
                 const double* body, const double* ext, int n_sets, const long long* offsets,
                 const long long* nodes, long long step, pd_tip_record* out, cudaStream_t st);

} // namespace pdb
