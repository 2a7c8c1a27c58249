// pd_host.cu -- the C ABI (include/pd_b200.h): validation with the reference's
// error types and messages, device residency, the per-step launch loop, and
// the host views handed to write hooks.
//
// Reference contracts followed here:
//   ModelBundle::validate            engine.cpp:335-341 -> types.cpp:6-21, 92-99, 181-196
//   check_force_inputs               engine.cpp:30-49
//   compute_forces (dispatcher)      engine.cpp:163-169
//   simulate (loop, cadence, tips)   engine.cpp:374-425, record_tips :349-370
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <memory>
#include <deque>
#include <mutex>
#include <thread>
#include <mutex>
#include <unistd.h>
#include <string>
#include <vector>

#include "pd_device.cuh"
#include "pd_internal.h"

using namespace pdb;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

int ok() {
    g_err.clear();
    return PD_OK;
}

// PD_TIMING=1: host wall time of the setup / run / download phases on stderr
struct PhaseTimer {
    bool on = std::getenv("PD_TIMING") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void mark(const char* what) {
        if (!on)
            return;
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[pd timing] %-28s %9.3f ms\n", what,
                     std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};

} // namespace

int pdb::set_error(int code, const char* msg) {
    g_err = msg;
    return code;
}

namespace {

#define PD_CK(expr)                                                                              \
    do {                                                                                         \
        cudaError_t e_ = (expr);                                                                 \
        if (e_ != cudaSuccess)                                                                   \
            return fail(PD_E_CUDA, "CUDA error %s at %s:%d (%s)", cudaGetErrorString(e_),        \
                        __FILE__, __LINE__, #expr);                                              \
    } while (0)

#define PD_TRY(expr)                                                                             \
    do {                                                                                         \
        int rc_ = (expr);                                                                        \
        if (rc_ != PD_OK)                                                                        \
            return rc_;                                                                          \
    } while (0)

// ---- validation with the reference's messages -----------------------------

int law_validate(const pd_law& l) {
    if (!(l.stiffness > 0))
        return fail(PD_E_INVALID_ARGUMENT, "DamageLaw: stiffness must be positive");
    if (l.n_breakpoints < 1)
        return fail(PD_E_INVALID_ARGUMENT,
                    "DamageLaw: breakpoints and forces must match and be non-empty");
    if (l.n_breakpoints > PD_MAX_BREAKPOINTS)
        return fail(PD_E_INVALID_ARGUMENT, "DamageLaw: more than %d breakpoints is not supported",
                    PD_MAX_BREAKPOINTS);
    double prev = 0;
    for (int k = 0; k < l.n_breakpoints; ++k) {
        if (!(l.breakpoints[k] > prev))
            return fail(PD_E_INVALID_ARGUMENT,
                        "DamageLaw: breakpoints must be strictly increasing and positive");
        prev = l.breakpoints[k];
    }
    const double f0 = l.stiffness * l.breakpoints[0];
    if (std::abs(l.forces[0] - f0) > 1e-9 * std::max(std::abs(f0), 1.0))
        return fail(PD_E_INVALID_ARGUMENT, "DamageLaw: envelope must leave the origin with slope c");
    return PD_OK;
}

int model_validate(const pd_damage_model& m) {
    if (m.n_laws < 1 || !m.laws)
        return fail(PD_E_INVALID_ARGUMENT, "DamageModel: no laws defined");
    if (m.n_laws > PD_MAX_LAWS)
        return fail(PD_E_INVALID_ARGUMENT, "DamageModel: more than %d laws", PD_MAX_LAWS);
    for (int k = 0; k < m.n_laws; ++k)
        PD_TRY(law_validate(m.laws[k]));
    if (m.damping < 0)
        return fail(PD_E_INVALID_ARGUMENT, "DamageModel: negative damping");
    return PD_OK;
}

bool needs_history(const pd_damage_model& m) {
    for (int k = 0; k < m.n_laws; ++k)
        if (m.laws[k].n_breakpoints > 1)
            return true;
    return false;
}

// fn(b, e) over [0, n) in chunks on several host threads
template <class Fn> void par_for(int64_t n, Fn fn) {
    const int64_t parts = std::min<int64_t>(std::max(1u, std::thread::hardware_concurrency()),
                                            n / (int64_t(1) << 16) + 1);
    if (parts <= 1) {
        fn(int64_t(0), n);
        return;
    }
    std::vector<std::thread> th;
    const int64_t step = (n + parts - 1) / parts;
    for (int64_t p = 0; p < parts; ++p)
        th.emplace_back([&, p] { fn(p * step, std::min(n, (p + 1) * step)); });
    for (auto& t : th)
        t.join();
}

// true when pred(k) holds for some k in [0, n): chunks on several host threads
// (the validation scans are O(n) over 10M-node arrays); the callers rescan
// serially only on failure, to report the first failing index
template <class Pred> bool par_any(int64_t n, Pred pred) {
    const int64_t parts = std::min<int64_t>(std::max(1u, std::thread::hardware_concurrency()),
                                            n / (int64_t(1) << 20) + 1);
    if (parts <= 1) {
        for (int64_t k = 0; k < n; ++k)
            if (pred(k))
                return true;
        return false;
    }
    std::atomic<bool> hit{false};
    std::vector<std::thread> th;
    const int64_t step = (n + parts - 1) / parts;
    for (int64_t p = 0; p < parts; ++p)
        th.emplace_back([&, p] {
            const int64_t b = p * step, e = std::min(n, b + step);
            for (int64_t k = b; k < e && !hit.load(std::memory_order_relaxed); ++k)
                if (pred(k)) {
                    hit = true;
                    return;
                }
        });
    for (auto& t : th)
        t.join();
    return hit;
}

int particles_validate(const pd_particles& p) {
    const int64_t n = p.n;
    if (n < 1)
        return fail(PD_E_INVALID_ARGUMENT, "ParticleSet: empty");
    if (p.coords_size != 3 * n || p.density_size != n)
        return fail(PD_E_INVALID_ARGUMENT, "ParticleSet: field lengths differ");
    if (!par_any(n, [&](int64_t i) { return !(p.volume[i] > 0) || !(p.density[i] > 0); }))
        return PD_OK;
    for (int64_t i = 0; i < n; ++i) {
        if (!(p.volume[i] > 0))
            return fail(PD_E_INVALID_ARGUMENT, "ParticleSet: non-positive volume at node %lld",
                        (long long)i);
        if (!(p.density[i] > 0))
            return fail(PD_E_INVALID_ARGUMENT, "ParticleSet: non-positive density at node %lld",
                        (long long)i);
    }
    return PD_OK;
}

int bc_validate(const pd_boundary& bc, int64_t n) {
    if (bc.kind_size != 3 * n || bc.magnitude_size != 3 * n || bc.ramp_id_size != 3 * n ||
        bc.no_failure_size != n)
        return fail(PD_E_INVALID_ARGUMENT,
                    "BoundaryConditions: field lengths do not match node count");
    if (bc.n_ramps < 1)
        return fail(PD_E_INVALID_ARGUMENT, "BoundaryConditions: no ramp profiles");
    if (par_any(3 * n, [&](int64_t k) { return bc.ramp_id[k] >= bc.n_ramps; }))
        return fail(PD_E_INVALID_ARGUMENT, "BoundaryConditions: ramp id out of range");
    for (int32_t s = 0; s < bc.n_tip_sets; ++s)
        for (int64_t t = bc.tip_offsets[s]; t < bc.tip_offsets[s + 1]; ++t)
            if (bc.tip_nodes[t] < 0 || bc.tip_nodes[t] >= n)
                return fail(PD_E_INVALID_ARGUMENT,
                            "BoundaryConditions: tip set #%d has an invalid node index", s);
    return PD_OK;
}

int group_validate(int64_t N) {
    if (N < 1 || (N & (N - 1)) != 0)
        return fail(PD_E_INVALID_ARGUMENT, "NeighborList: group size must be a power of two");
    // the device family builder sorts rows of up to 1024 members
    // (pd_family.cu); the exact kernel gives each of 32 lanes N / 32 slots
    if (N > 1024)
        return fail(PD_E_INVALID_ARGUMENT,
                    "NeighborList: group size %lld exceeds the supported maximum of 1024",
                    (long long)N);
    return PD_OK;
}

} // namespace

// ---- the resident context ---------------------------------------------------

struct pd_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    int64_t launches = 0;
    const char* kernel = "";  // the step kernel instantiation last launched

    int64_t n = 0;
    int N = 0, W = 0, log2N = 0;
    double horizon = 0;
    int variant = PD_BOND_PARALLEL;
    bool history = false;
    bool has_bc = false;
    int n_laws = 0;
    bool exact_pmb = false;  // one PMB law: the specialised exact kernel (pd_exact.cu slot_pmb)
    double exact_c = 0, exact_sc = 0;
    double damping = 0, dt = 0;
    int64_t step = 0;
    int cur = 0;

    DevBuf<double4> xv, u[2];
    DevBuf<double> v, a, rho, inv_rho, hist, hist_keep, lambda, beta, body, ext;
    DevBuf<int32_t> entries, n_neigh, initial, scratch_i32;
    DevBuf<uint32_t> alive;
    DevBuf<uint8_t> btype, bc_kind, bc_ramp, nofail;
    DevBuf<double> bc_mag, scratch_f64;
    DevBuf<DevRamp> ramps;
    DevBuf<DevLaw> laws;  // the exact kernel's law table
    DevBuf<long long> err, tip_offsets, tip_nodes;
    DevBuf<unsigned long long> counter;
    DevBuf<pd_tip_record> tips;
    int n_tip_sets = 0;
    bool forces_valid = false;

    // the range of device rows this context integrates (all rows on one GPU;
    // the owned rows of a multi-GPU slab)
    int64_t comp_begin = 0, comp_end = 0;
    int64_t own_begin = 0, own_end = 0;  // owned LOCAL node ids
    bool partial = false;                // uploaded by pd_ctx_upload_part
    bool dst_has_upload = false;         // download target = the uploaded host arrays
    // multi-GPU slab world (pd_ctx_connect)
    int rank = 0, world = 1;
    DevBuf<unsigned long long> sync;     // 2 * PD_MAX_RANKS words (epochs, flags)
    DevBuf<unsigned long long> bar;      // arrival counter of the persistent small-model launch
    unsigned long long epoch = 0;
    DevBuf<int2> xfer;
    double4* peer_u[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // [lo/hi][parity]
    unsigned long long* peer_sync[PD_MAX_RANKS] = {};
    std::vector<void*> ipc_opened;
    std::vector<int> inv_host;           // local node -> device row (PD_FAST)

    // fast path (PD_FAST): internal brick order + tile layout (pd_fast.cuh)
    bool fast = false;
    int kind = 2;  // fast kernel specialisation (pd_fast.cu)
    float pmb_c = 0, pmb_sc = 0, pmb_cv = 0;
    int fast_T = FAST_T, fast_cfg = 0;
    FastLayoutDev lay;  // built on the device (pd_layout.cu)
    // PD_FAST on a structured lattice: implicit connectivity (pd_lattice.cu),
    // node arrays stay in the reference order
    bool lattice = false;
    LatticeArgs lat;
    DevBuf<uint4> lmask;
    DevBuf<float> lhist, llam;  // NL: brick-major per-bond arrays (llam = lambda * beta)
    DevBuf<uint8_t> lbtype;
    bool permuted() const { return fast && !lattice; }
    // async snapshots (pd_ctx_snapshot_every)
    int64_t snap_every = 0;
    std::string snap_pattern;
    struct SnapJob {
        int slot;
        int64_t step;
    };
    DevBuf<double> snap_dev[2];
    cudaEvent_t snap_ready[2] = {nullptr, nullptr};
    bool snap_busy[2] = {false, false};
    std::mutex snap_mu;
    std::condition_variable snap_cv;
    std::deque<SnapJob> snap_jobs;
    std::thread snap_thread;
    bool snap_stop = false;
    std::string snap_error;
    cudaStream_t snap_stream = nullptr;
    int64_t row_of(int64_t local) const {
        return permuted() ? int64_t(lay.inv_host[size_t(local)]) : local;
    }
    DevBuf<double4> scratch_d4;
    DevBuf<int32_t> scratch_n;
    DevBuf<uint8_t> scratch_u8;

    FastDev fast_args() const {
        FastDev F{};
        F.T = fast_T;
        F.cap = (lay.max_halo + 1 + 31) / 32 * 32;
        F.cfg = fast_cfg;
        F.n_tiles = lay.n_tiles;
        F.tile0 = 0;
        F.tile_start = lay.tile_start.p;
        F.halo_off = lay.halo_off.p;
        F.halo = lay.halo.p;
        F.slot_off = lay.slot_off.p;
        F.kmax8 = lay.kmax8.p;
        F.wgroups = lay.wgroups.p;
        F.own_slot = lay.own_slot.p;
        F.nf_start = lay.nf_start.p;
        F.lidx = lay.lidx.p;
        F.hist = lay.hist32.p;
        F.btype = lay.btype_c.p;
        F.lambda = lay.lambda32.p;
        F.beta = lay.beta32.p;
        F.pmb_c = pmb_c;
        F.pmb_sc = pmb_sc;
        F.pmb_cv = pmb_cv;
        return F;
    }

    DevArgs args() const {
        DevArgs A{};
        A.n = n;
        A.begin = comp_begin;
        A.end = comp_end;
        A.N = N;
        A.log2N = log2N;
        A.W = W;
        A.n_laws = n_laws;
        A.xv = xv.p;
        A.u_in = u[cur].p;
        A.u_out = u[cur ^ 1].p;
        A.v = v.p;
        A.a = a.p;
        A.rho = rho.p;
        A.inv_rho = inv_rho.p;
        A.entries = entries.p;
        A.alive = alive.p;
        A.n_neigh = n_neigh.p;
        A.hist = hist.p;
        A.btype = btype.p;
        A.lambda = lambda.p;
        A.beta = beta.p;
        A.bc_kind = has_bc ? bc_kind.p : nullptr;
        A.bc_mag = bc_mag.p;
        A.bc_ramp = bc_ramp.p;
        A.ramps = ramps.p;
        A.body_force = body.p;
        A.ext_force = ext.p;
        A.err_step = err.p;
        A.step = step;
        A.dt = dt;
        A.half_dt = dt / 2;
        A.half_dt2 = dt * dt / 2;
        A.dt2 = dt * dt;
        A.damping = damping;
        A.pmb_c = exact_c;
        A.pmb_sc = exact_sc;
        A.laws = laws.p;
        A.store_forces = 0;
        A.do_drift = 0;
        A.xfer = world > 1 ? xfer.p : nullptr;
        A.peer_lo = peer_u[0][cur ^ 1];
        A.peer_hi = peer_u[1][cur ^ 1];
        return A;
    }
};

namespace {

int select_device(pd_ctx* ctx) {
    PD_CK(cudaSetDevice(ctx->device));
    return PD_OK;
}

int upload_laws(pd_ctx* ctx, const pd_damage_model& m) {
    std::vector<DevLaw> laws(size_t(m.n_laws));
    for (int k = 0; k < m.n_laws; ++k) {
        DevLaw& d = laws[size_t(k)];
        std::memset(&d, 0, sizeof d);
        d.c = m.laws[k].stiffness;
        d.nbp = m.laws[k].n_breakpoints;
        for (int b = 0; b < d.nbp; ++b) {
            d.bp[b] = m.laws[k].breakpoints[b];
            d.f[b] = m.laws[k].forces[b];
        }
    }
    PD_CK(ctx->laws.upload(laws.data(), laws.size(), ctx->stream));
    ctx->n_laws = m.n_laws;
    ctx->exact_pmb = m.n_laws == 1 && m.laws[0].n_breakpoints == 1;
    ctx->exact_c = m.laws[0].stiffness;
    ctx->exact_sc = m.laws[0].breakpoints[0];
    ctx->damping = m.damping;
    ctx->history = needs_history(m);
    return PD_OK;
}

// Geometry, connectivity, corrections and the mutable state.  Validation of
// the caller's sizes is done by the callers (they differ between
// compute_forces and simulate, as in the reference).
int upload_common(pd_ctx* ctx, const pd_particles& p, const pd_state& st,
                  const pd_damage_model& m, const pd_corrections& corr,
                  const uint8_t* nofail, int64_t nofail_size) {
    cudaStream_t s = ctx->stream;
    const int64_t n = st.connectivity.n;
    const int64_t N = st.connectivity.group_size;
    PD_TRY(group_validate(N));
    ctx->fast = false;
    ctx->lattice = false;
    if (p.coords_size != 3 * n || !p.coords || !p.volume)
        return fail(PD_E_INVALID_ARGUMENT, "ParticleSet: field lengths differ");
    ctx->n = n;
    ctx->N = int(N);
    ctx->horizon = st.connectivity.horizon;
    ctx->W = N < 32 ? 1 : int(N / 32);
    ctx->log2N = 0;
    while ((int64_t(1) << ctx->log2N) < N)
        ++ctx->log2N;
    const int64_t slots = n * N;

    // bond types must index a law (out of range is UB in the reference)
    if (st.connectivity.bond_type_size != 0) {
        if (st.connectivity.bond_type_size != slots)
            return fail(PD_E_INVALID_ARGUMENT, "NeighborList: bond_type size mismatch");
        const auto bad_type = [&](int64_t k) {
            return st.connectivity.entries[k] >= 0 && st.connectivity.bond_type[k] >= m.n_laws;
        };
        if (par_any(slots, bad_type))
            for (int64_t k = 0; k < slots; ++k)
                if (bad_type(k))
                    return fail(PD_E_INVALID_ARGUMENT, "DamageModel: unknown bond type %d",
                                int(st.connectivity.bond_type[k]));
    }
    PD_TRY(upload_laws(ctx, m));

    // xv = {x, y, z, V}
    PD_CK(ctx->scratch_f64.upload(p.coords, size_t(3 * n), s));
    PD_CK(ctx->rho.alloc(size_t(n)));
    // pageable host arrays go through the pinned bounce pipeline (pd_xfer.cpp):
    // a direct cudaMemcpyAsync from pageable memory runs at ~6 GB/s
    PD_CK(h2d_large(ctx->rho.p, p.volume, sizeof(double) * n, s));
    PD_CK(ctx->xv.alloc(size_t(n)));
    launch_pack_xv(ctx->scratch_f64.p, ctx->rho.p, n, ctx->xv.p, s);
    ++ctx->launches;
    if (p.density && p.density_size == n)
        PD_CK(h2d_large(ctx->rho.p, p.density, sizeof(double) * n, s));
    PD_CK(ctx->inv_rho.alloc(size_t(n)));
    launch_inv(ctx->rho.p, n, ctx->inv_rho.p, s);  // Real(1) / density[i] (engine.cpp:244)
    ++ctx->launches;

    // u = {ux, uy, uz, no_failure}
    PD_CK(ctx->scratch_f64.upload(st.u, size_t(3 * n), s));
    PD_CK(ctx->nofail.alloc(size_t(n)));
    if (nofail && nofail_size == n)
        PD_CK(h2d_large(ctx->nofail.p, nofail, size_t(n), s));
    else
        PD_CK(cudaMemsetAsync(ctx->nofail.p, 0, size_t(n), s));
    PD_CK(ctx->u[0].alloc(size_t(n)));
    PD_CK(ctx->u[1].alloc(size_t(n)));
    ctx->cur = 0;
    launch_pack_u(ctx->scratch_f64.p, ctx->nofail.p, n, ctx->u[0].p, s);
    ++ctx->launches;

    PD_CK(ctx->v.alloc(size_t(3 * n)));
    PD_CK(ctx->a.alloc(size_t(3 * n)));
    if (st.v)
        PD_CK(h2d_large(ctx->v.p, st.v, sizeof(double) * 3 * n, s));
    else
        PD_CK(cudaMemsetAsync(ctx->v.p, 0, sizeof(double) * 3 * n, s));
    if (st.a)
        PD_CK(h2d_large(ctx->a.p, st.a, sizeof(double) * 3 * n, s));
    else
        PD_CK(cudaMemsetAsync(ctx->a.p, 0, sizeof(double) * 3 * n, s));

    // connectivity: immutable row list + alive mask + counts
    PD_CK(ctx->entries.upload(st.connectivity.entries, size_t(slots), s));
    PD_CK(ctx->n_neigh.upload(st.connectivity.n_neigh, size_t(n), s));
    PD_CK(ctx->initial.upload(st.connectivity.initial_n_neigh, size_t(n), s));
    PD_CK(ctx->alive.alloc(size_t(n * ctx->W)));
    PD_CK(ctx->counter.alloc(1));
    const unsigned long long none = ~0ull;
    PD_CK(cudaMemcpyAsync(ctx->counter.p, &none, sizeof none, cudaMemcpyHostToDevice, s));
    launch_validate_entries(ctx->entries.p, n, ctx->N, ctx->counter.p, s);
    launch_init_alive(ctx->entries.p, n, ctx->N, ctx->W, ctx->alive.p, s);
    ctx->launches += 2;
    unsigned long long bad = 0;
    PD_CK(cudaMemcpyAsync(&bad, ctx->counter.p, sizeof bad, cudaMemcpyDeviceToHost, s));
    PD_CK(cudaStreamSynchronize(s));
    if (bad != none)
        return fail(PD_E_INVALID_ARGUMENT, "NeighborList: entry out of range in row %llu", bad);

    if (st.connectivity.bond_type_size != 0)
        PD_CK(ctx->btype.upload(st.connectivity.bond_type, size_t(slots), s));
    else
        ctx->btype.release();
    if (ctx->history) {
        if (st.bond_history && st.bond_history_size == slots)
            PD_CK(ctx->hist.upload(st.bond_history, size_t(slots), s));
        else {
            PD_CK(ctx->hist.alloc(size_t(slots)));
            PD_CK(cudaMemsetAsync(ctx->hist.p, 0, sizeof(double) * slots, s));
        }
        ctx->hist_keep.release();
    } else {
        ctx->hist.release();
        // a state that carries bond_history under a model without n-linear
        // laws: the reference keeps it untouched and save_state still writes
        // it (io.cpp section 10), so it is kept on the device unchanged
        if (st.bond_history && st.bond_history_size == slots)
            PD_CK(ctx->hist_keep.upload(st.bond_history, size_t(slots), s));
        else
            ctx->hist_keep.release();
    }
    if (corr.lambda_size != 0)
        PD_CK(ctx->lambda.upload(corr.lambda, size_t(slots), s));
    else
        ctx->lambda.release();
    if (corr.beta_size != 0)
        PD_CK(ctx->beta.upload(corr.beta, size_t(slots), s));
    else
        ctx->beta.release();

    PD_CK(ctx->err.alloc(1));
    PD_CK(ctx->body.alloc(size_t(3 * n)));
    PD_CK(ctx->ext.alloc(size_t(3 * n)));
    PD_CK(cudaMemsetAsync(ctx->body.p, 0, sizeof(double) * 3 * n, s));
    PD_CK(cudaMemsetAsync(ctx->ext.p, 0, sizeof(double) * 3 * n, s));
    ctx->forces_valid = false;
    ctx->step = st.step;
    if (!ctx->partial) {
        ctx->own_begin = 0;
        ctx->own_end = n;
    }
    ctx->comp_begin = ctx->own_begin;
    ctx->comp_end = ctx->own_end;
    ctx->scratch_f64.release();
    PD_CK(cudaStreamSynchronize(s));
    return PD_OK;
}

int upload_bc(pd_ctx* ctx, const pd_boundary& bc) {
    cudaStream_t s = ctx->stream;
    const int64_t n = ctx->n;
    const bool any = par_any(3 * n, [&](int64_t k) { return bc.kind[k] != PD_BC_FREE; });
    ctx->has_bc = any;
    if (any) {
        PD_CK(ctx->bc_kind.upload(bc.kind, size_t(3 * n), s));
        PD_CK(ctx->bc_mag.upload(bc.magnitude, size_t(3 * n), s));
        PD_CK(ctx->bc_ramp.upload(bc.ramp_id, size_t(3 * n), s));
    }
    std::vector<DevRamp> ramps(size_t(bc.n_ramps));
    for (int k = 0; k < bc.n_ramps; ++k) {
        ramps[size_t(k)].kind = bc.ramps[k].kind;
        ramps[size_t(k)].pad_ = 0;
        ramps[size_t(k)].rise = bc.ramps[k].rise_steps;
        ramps[size_t(k)].target = bc.ramps[k].target_scale;
    }
    PD_CK(ctx->ramps.upload(ramps.data(), ramps.size(), s));
    ctx->n_tip_sets = bc.n_tip_sets;
    if (bc.n_tip_sets > 0) {
        std::vector<long long> off(size_t(bc.n_tip_sets + 1));
        for (int k = 0; k <= bc.n_tip_sets; ++k)
            off[size_t(k)] = bc.tip_offsets[k];
        PD_CK(ctx->tip_offsets.upload(off.data(), off.size(), s));
        const int64_t total = bc.tip_offsets[bc.n_tip_sets];
        std::vector<long long> nodes(size_t(std::max<int64_t>(total, 1)), 0);
        for (int64_t t = 0; t < total; ++t)
            nodes[size_t(t)] = bc.tip_nodes[t];
        PD_CK(ctx->tip_nodes.upload(nodes.data(), nodes.size(), s));
    }
    PD_CK(cudaStreamSynchronize(s));
    return PD_OK;
}

// Copy selected resident fields into host arrays of `st` / `forces` (in the
// reference's node order; the fast path gathers out of its brick order).
int download(pd_ctx* ctx, pd_state* st, pd_force_field* forces, int32_t fields) {
    cudaStream_t s = ctx->stream;
    const int64_t n = ctx->n;
    const int64_t slots = n * ctx->N;
    const int* inv = ctx->permuted() ? ctx->lay.inv.p : nullptr;
    auto vec3_out = [&](const double* dev, double* host) -> int {
        const double* src = dev;
        if (inv) {
            PD_CK(ctx->scratch_f64.alloc(size_t(3 * n)));
            launch_gather_rows<double, 3>(dev, ctx->scratch_f64.p, inv, n, s);
            ++ctx->launches;
            src = ctx->scratch_f64.p;
        }
        PD_CK(d2h_large(host, src, sizeof(double) * 3 * n, s));
        return PD_OK;
    };
    if ((fields & PD_FIELD_U) && st && st->u) {
        const double4* src = ctx->u[ctx->cur].p;
        if (inv) {
            PD_CK(ctx->scratch_d4.alloc(size_t(n)));
            launch_gather_rows<double4, 1>(src, ctx->scratch_d4.p, inv, n, s);
            ++ctx->launches;
            src = ctx->scratch_d4.p;
        }
        PD_CK(ctx->scratch_f64.alloc(size_t(3 * n)));
        launch_unpack_u(src, n, ctx->scratch_f64.p, s);
        ++ctx->launches;
        PD_CK(d2h_large(st->u, ctx->scratch_f64.p, sizeof(double) * 3 * n, s));
    }
    if ((fields & PD_FIELD_V) && st && st->v)
        PD_TRY(vec3_out(ctx->v.p, st->v));
    if ((fields & PD_FIELD_A) && st && st->a)
        PD_TRY(vec3_out(ctx->a.p, st->a));
    const bool want_hist = (fields & PD_FIELD_HISTORY) && st && st->bond_history &&
                           (ctx->history || ctx->hist_keep.p);
    if (want_hist && st->bond_history_size != slots)
        return fail(PD_E_INVALID_ARGUMENT, "download: bond_history must be sized n x N");
    if ((fields & PD_FIELD_CONNECTIVITY) && st) {
        if (st->connectivity.entries) {
            PD_CK(ctx->scratch_i32.alloc(size_t(slots)));
            if (ctx->lattice)
                PD_CK(launch_lattice_materialize(ctx->entries.p, ctx->lmask.p, ctx->own_begin,
                                                 ctx->own_end, n, ctx->N, ctx->lat,
                                                 ctx->scratch_i32.p, nullptr, s));
            else if (ctx->fast)
                launch_fast_materialize(ctx->lay.origk.p, ctx->entries.p, ctx->lay.inv.p, ctx->lay.tile_of.p,
                                        ctx->lay.tile_start.p, ctx->lay.slot_off.p, ctx->fast_T, ctx->lay.lidx.p,
                                        nullptr, n, ctx->N, ctx->scratch_i32.p, nullptr, s);
            else
                launch_materialize_entries(ctx->entries.p, ctx->alive.p, n, ctx->N, ctx->W,
                                           ctx->scratch_i32.p, s);
            ++ctx->launches;
            if (ctx->dst_has_upload) {
                // the destination still holds the uploaded rows (one-shot
                // simulate writes back into the caller's array): move only
                // the rows that changed
                PD_CK(ctx->counter.alloc(1));
                PD_CK(ctx->scratch_n.alloc(size_t(n)));
                PD_CK(cudaMemsetAsync(ctx->counter.p, 0, sizeof(unsigned long long), s));
                launch_changed_rows(ctx->scratch_i32.p, ctx->entries.p, n, ctx->N,
                                    ctx->scratch_n.p, ctx->counter.p, s);
                unsigned long long m = 0;
                PD_CK(cudaMemcpyAsync(&m, ctx->counter.p, sizeof m, cudaMemcpyDeviceToHost, s));
                PD_CK(cudaStreamSynchronize(s));
                ctx->launches += 1;
                if (m > 0 && 4 * (long long)m > n) {
                    // most rows changed (a fracturing run): the whole array in
                    // one pinned, multi-threaded copy beats a gather + scatter
                    PD_CK(d2h_large(st->connectivity.entries, ctx->scratch_i32.p,
                                    sizeof(int32_t) * slots, s));
                } else if (m > 0) {
                    DevBuf<int32_t> rows;
                    const size_t N = size_t(ctx->N);
                    PD_CK(rows.alloc(size_t(m) * N));
                    launch_gather_list_rows(ctx->scratch_i32.p, ctx->scratch_n.p, (long long)m,
                                            ctx->N, rows.p, s);
                    ++ctx->launches;
                    std::unique_ptr<int[]> list(new int[size_t(m)]);
                    std::unique_ptr<int32_t[]> host_rows(new int32_t[size_t(m) * N]);  // no zero fill
                    PD_CK(d2h_large(list.get(), ctx->scratch_n.p, sizeof(int) * m, s));
                    PD_CK(d2h_large(host_rows.get(), rows.p, sizeof(int32_t) * size_t(m) * N, s));
                    int32_t* dst = st->connectivity.entries;
                    const int32_t* src = host_rows.get();
                    const int* rl = list.get();
                    par_for((int64_t)m, [&](int64_t b, int64_t e) {
                        for (int64_t r = b; r < e; ++r)
                            std::memcpy(dst + size_t(rl[r]) * N, src + size_t(r) * N,
                                        sizeof(int32_t) * N);
                    });
                }
            } else {
                PD_CK(d2h_large(st->connectivity.entries, ctx->scratch_i32.p,
                                sizeof(int32_t) * slots, s));
            }
        }
        if (st->connectivity.n_neigh) {
            const int32_t* src = ctx->n_neigh.p;
            if (inv) {
                PD_CK(ctx->scratch_n.alloc(size_t(n)));
                launch_gather_rows<int32_t, 1>(src, ctx->scratch_n.p, inv, n, s);
                ++ctx->launches;
                src = ctx->scratch_n.p;
            }
            PD_CK(d2h_large(st->connectivity.n_neigh, src, sizeof(int32_t) * n, s));
        }
        PD_CK(cudaStreamSynchronize(s));
    }
    if (want_hist) {
        if (ctx->history && ctx->lattice) {
            PD_CK(launch_lattice_materialize(ctx->entries.p, ctx->lmask.p, ctx->own_begin,
                                             ctx->own_end, n, ctx->N, ctx->lat, nullptr,
                                             ctx->hist.p, s));
            ++ctx->launches;
        } else if (ctx->history && ctx->permuted()) {
            launch_fast_materialize(ctx->lay.origk.p, ctx->entries.p, ctx->lay.inv.p, ctx->lay.tile_of.p, ctx->lay.tile_start.p,
                                    ctx->lay.slot_off.p, ctx->fast_T, ctx->lay.lidx.p, ctx->lay.hist32.p, n,
                                    ctx->N, nullptr, ctx->hist.p, s);
            ++ctx->launches;
        }
        PD_CK(d2h_large(st->bond_history, ctx->history ? ctx->hist.p : ctx->hist_keep.p,
                        sizeof(double) * slots, s));
    }
    if ((fields & PD_FIELD_FORCES) && forces) {
        if (forces->body_force)
            PD_TRY(vec3_out(ctx->body.p, forces->body_force));
        if (forces->external_force)
            PD_TRY(vec3_out(ctx->ext.p, forces->external_force));
    }
    if (st)
        st->step = ctx->step;
    PD_CK(cudaStreamSynchronize(s));
    return PD_OK;
}

// Renumber the resident node arrays into the fast path's brick order and
// build its tile layout from the host copies of the rows.
// PD_FAST on a lattice: implicit connectivity (pd_lattice.cu).  One PMB law
// runs the unrolled kernel (no-failure nodes and per-node volumes ride in the
// staged records); n-linear laws, bond types and lambda / beta run the NL
// kernels with brick-major per-bond arrays.  Returns false (and
// leaves the context untouched) when the model does not qualify;
// PD_FAST_LAYOUT=general forces the general tile layout.
// the fast kernels keep their laws in 8-breakpoint tables
int fast_laws_ok(const pd_damage_model& m) {
    for (int k = 0; k < m.n_laws; ++k)
        if (m.laws[k].n_breakpoints > 8)
            return fail(PD_E_INVALID_ARGUMENT,
                        "fast variant: law %d has %d breakpoints; the fast kernels take at most 8 "
                        "(the exact variants take up to %d)",
                        k, m.laws[k].n_breakpoints, PD_MAX_BREAKPOINTS);
    return PD_OK;
}

int try_lattice(pd_ctx* ctx, const pd_particles& p, const pd_state& st, const pd_damage_model& m,
                const pd_corrections& corr, const uint8_t* nofail, int64_t nofail_size,
                bool* used) {
    *used = false;
    if (const char* e = std::getenv("PD_FAST_LAYOUT"))
        if (std::strcmp(e, "general") == 0)
            return PD_OK;
    const int64_t n = ctx->n;
    // n-linear laws, several laws, bond types or lambda / beta: the NL kernels
    // with brick-major per-bond arrays
    const bool nl = m.n_laws != 1 || m.laws[0].n_breakpoints != 1 || ctx->history ||
                    st.connectivity.bond_type_size != 0 || corr.lambda_size != 0 ||
                    corr.beta_size != 0;
    const bool any_nf = nofail && nofail_size == n &&
                        par_any(n, [&](int64_t i) { return nofail[i] != 0; });
    const bool vol_varies = par_any(n, [&](int64_t i) { return p.volume[i] != p.volume[0]; });
    LatticeArgs L;
    if (!lattice_detect(p.coords, n, ctx->own_begin, ctx->own_end, L))
        return PD_OK;
    cudaStream_t s = ctx->stream;
    PD_CK(ctx->lmask.alloc(size_t(n)));
    L.n_local = n;
    L.nl = nl ? 1 : 0;
    // NL brick depth: 8 planes unless the owned planes leave a much emptier last
    // brick than 4 would (thin plates, 27-plane slabs); PD_NL_BZ=4|8 forces it
    {
        const int nz = L.nz_own > 0 ? L.nz_own : 1;
        const double waste8 = double((nz + 7) / 8 * 8 - nz) / nz;
        const double waste4 = double((nz + 3) / 4 * 4 - nz) / nz;
        L.nlbz = waste8 - waste4 < 0.04 ? 8 : 4;
        if (const char* e = std::getenv("PD_NL_BZ"))
            L.nlbz = std::atoi(e) == 4 ? 4 : 8;
    }
    const size_t pslots = size_t(lattice_slot_count(L));
    // several laws (<= 8, <= 3 breakpoints each): the typed unrolled kernel,
    // with the bond type in the history words (PD_LAT_NL_LOOP: the loop kernel)
    // The unrolled kernels evaluate each law's envelope as min/max of its
    // segment lines; laws where that composition is not the envelope
    // (e.g. hardening then softening) take the loop kernel's segment selection
    bool minmax_ok = true;
    for (int k = 0; k < m.n_laws && minmax_ok; ++k)
        minmax_ok = lattice_minmax_ok(m.laws[k].breakpoints, m.laws[k].forces,
                                      m.laws[k].n_breakpoints);
    bool small_laws = m.n_laws >= 2 && m.n_laws <= 8 && minmax_ok;
    for (int k = 0; k < m.n_laws && small_laws; ++k)
        small_laws = m.laws[k].n_breakpoints <= 3;
    L.typed = (nl && small_laws && !std::getenv("PD_LAT_NL_LOOP")) ? 1 : 0;
    if (L.typed) {
        PD_CK(ctx->lhist.alloc(pslots));
        PD_CK(cudaMemsetAsync(ctx->lhist.p, 0, sizeof(float) * pslots, s));
        L.hist = ctx->lhist.p;
    } else if (nl && ctx->history) {
        PD_CK(ctx->lhist.alloc(pslots));
        PD_CK(cudaMemsetAsync(ctx->lhist.p, 0, sizeof(float) * pslots, s));
        L.hist = ctx->lhist.p;
    }
    if (nl && !L.typed && st.connectivity.bond_type_size != 0) {
        PD_CK(ctx->lbtype.alloc(pslots));
        PD_CK(cudaMemsetAsync(ctx->lbtype.p, 0, pslots, s));
        L.btype = ctx->lbtype.p;
    }
    if (nl && (corr.lambda_size != 0 || corr.beta_size != 0)) {
        PD_CK(ctx->llam.alloc(pslots));  // lambda * beta
        L.lam = ctx->llam.p;
    }
    PD_CK(ctx->counter.alloc(1));
    PD_CK(cudaMemsetAsync(ctx->counter.p, 0, sizeof(unsigned long long), s));
    int* bad = reinterpret_cast<int*>(ctx->counter.p);
    PD_CK(lattice_build_masks(ctx->xv.p, n, ctx->entries.p, ctx->own_begin, ctx->own_end,
                              ctx->N, L, ctx->lmask.p, bad, ctx->history ? ctx->hist.p : nullptr,
                              ctx->btype.p, ctx->lambda.p, ctx->beta.p, s));
    int bad_h = 0;
    PD_CK(cudaMemcpyAsync(&bad_h, bad, sizeof bad_h, cudaMemcpyDeviceToHost, s));
    PD_CK(cudaStreamSynchronize(s));
    if (bad_h) {
        ctx->lmask.release();
        ctx->lhist.release();
        ctx->lbtype.release();
        ctx->llam.release();
        return PD_OK;
    }
    if (nl) {
        // laws in constant memory; forces carry V_0 (c and V_j / V_0 are per bond)
        std::vector<DevLaw> laws(size_t(m.n_laws));
        for (int k = 0; k < m.n_laws; ++k) {
            std::memset(&laws[size_t(k)], 0, sizeof(DevLaw));
            laws[size_t(k)].c = m.laws[k].stiffness;
            laws[size_t(k)].nbp = m.laws[k].n_breakpoints;
            for (int b = 0; b < laws[size_t(k)].nbp; ++b) {
                laws[size_t(k)].bp[b] = m.laws[k].breakpoints[b];
                laws[size_t(k)].f[b] = m.laws[k].forces[b];
            }
        }
        lattice_set_laws(laws.data(), m.n_laws, L, s);
        PD_CK(cudaGetLastError());
        if (std::getenv("PD_LAT_NL_LOOP") || !minmax_ok)  // the runtime-loop kernel
            L.multi = 1;
    }
    L.sc = float(m.laws[0].breakpoints[0]);
    L.cv = nl ? float(p.volume[0]) : float(m.laws[0].stiffness * p.volume[0]);
    L.nf = (any_nf || vol_varies) ? 1 : 0;
    L.vol_varies = vol_varies ? 1 : 0;
    L.inv_v0 = 1.0 / p.volume[0];
    L.mask = ctx->lmask.p;
    if (const char* e = std::getenv("PD_LAT_CFG"))
        L.cfg = std::atoi(e);
    if (const char* e = std::getenv("PD_NLU_PF"))
        L.prefetch = std::atoi(e);
    ctx->lat = L;
    ctx->lattice = true;
    ctx->fast = true;
    *used = true;
    return PD_OK;
}

int setup_fast(pd_ctx* ctx, const pd_particles& p, const pd_state& st,
               const pd_damage_model& m, const pd_corrections& corr, const uint8_t* nofail,
               int64_t nofail_size, pd_boundary* bc_tips) {
    cudaStream_t s = ctx->stream;
    const int64_t n = ctx->n;
    // PD_FAST_CFG selects a tile configuration (pd_fast.cu launch_one); the
    // default is 512-node tiles
    ctx->fast_cfg = 0;
    if (const char* e = std::getenv("PD_FAST_CFG"))
        ctx->fast_cfg = std::atoi(e);
    ctx->fast_T = (ctx->fast_cfg == 1 || ctx->fast_cfg == 2) ? 256 : 512;
    PhaseTimer tm;
    FastLayoutIn in;
    in.n = n;
    in.own_begin = ctx->own_begin;
    in.own_end = ctx->own_end;
    in.N = ctx->N;
    in.T = ctx->fast_T;
    in.history = ctx->history;
    in.xv = ctx->xv.p;
    in.entries = ctx->entries.p;
    bool any_nf = false;
    for (int64_t i = 0; nofail && nofail_size == n && i < n && !any_nf; ++i)
        any_nf = nofail[i] != 0;
    in.nofail = any_nf ? ctx->nofail.p : nullptr;
    in.hist = ctx->history ? ctx->hist.p : nullptr;
    in.btype = st.connectivity.bond_type_size ? ctx->btype.p : nullptr;
    in.lambda = corr.lambda_size ? ctx->lambda.p : nullptr;
    in.beta = corr.beta_size ? ctx->beta.p : nullptr;
    int too_big = 0;
    PD_CK(gpu_build_layout(ctx->lay, in, &too_big, s));
    if (too_big)
        return fail(PD_E_INVALID_ARGUMENT,
                    "PD_FAST: a tile neighbourhood exceeds %d nodes of shared memory; use "
                    "PD_BOND_PARALLEL for this mesh", FAST_MAX_HALO);
    tm.mark("fast: device layout build");
    ctx->comp_begin = 0;  // owned nodes come first in the internal order
    ctx->comp_end = ctx->own_end - ctx->own_begin;
    // permute node arrays into internal order
    const int* perm = ctx->lay.perm.p;
    PD_CK(ctx->scratch_d4.alloc(size_t(n)));
    launch_gather_rows<double4, 1>(ctx->xv.p, ctx->scratch_d4.p, perm, n, s);
    PD_CK(cudaMemcpyAsync(ctx->xv.p, ctx->scratch_d4.p, sizeof(double4) * n,
                          cudaMemcpyDeviceToDevice, s));
    launch_gather_rows<double4, 1>(ctx->u[ctx->cur].p, ctx->scratch_d4.p, perm, n, s);
    PD_CK(cudaMemcpyAsync(ctx->u[ctx->cur].p, ctx->scratch_d4.p, sizeof(double4) * n,
                          cudaMemcpyDeviceToDevice, s));
    PD_CK(ctx->scratch_f64.alloc(size_t(3 * n)));
    for (double* arr : {ctx->v.p, ctx->a.p}) {
        launch_gather_rows<double, 3>(arr, ctx->scratch_f64.p, perm, n, s);
        PD_CK(cudaMemcpyAsync(arr, ctx->scratch_f64.p, sizeof(double) * 3 * n,
                              cudaMemcpyDeviceToDevice, s));
    }
    launch_gather_rows<double, 1>(ctx->rho.p, ctx->scratch_f64.p, perm, n, s);
    PD_CK(cudaMemcpyAsync(ctx->rho.p, ctx->scratch_f64.p, sizeof(double) * n,
                          cudaMemcpyDeviceToDevice, s));
    launch_inv(ctx->rho.p, n, ctx->inv_rho.p, s);
    PD_CK(ctx->scratch_n.alloc(size_t(n)));
    for (int32_t* arr : {ctx->n_neigh.p, ctx->initial.p}) {
        launch_gather_rows<int32_t, 1>(arr, ctx->scratch_n.p, perm, n, s);
        PD_CK(cudaMemcpyAsync(arr, ctx->scratch_n.p, sizeof(int32_t) * n,
                              cudaMemcpyDeviceToDevice, s));
    }
    if (ctx->has_bc) {
        PD_CK(ctx->scratch_u8.alloc(size_t(3 * n)));
        for (uint8_t* arr : {ctx->bc_kind.p, ctx->bc_ramp.p}) {
            launch_gather_rows<uint8_t, 3>(arr, ctx->scratch_u8.p, perm, n, s);
            PD_CK(cudaMemcpyAsync(arr, ctx->scratch_u8.p, 3 * n, cudaMemcpyDeviceToDevice, s));
        }
        launch_gather_rows<double, 3>(ctx->bc_mag.p, ctx->scratch_f64.p, perm, n, s);
        PD_CK(cudaMemcpyAsync(ctx->bc_mag.p, ctx->scratch_f64.p, sizeof(double) * 3 * n,
                              cudaMemcpyDeviceToDevice, s));
    }
    ctx->launches += 10;
    // tip sets refer to reference node numbers
    if (bc_tips && ctx->n_tip_sets > 0) {
        const int64_t total = bc_tips->tip_offsets[bc_tips->n_tip_sets];
        std::vector<long long> nodes(size_t(std::max<int64_t>(total, 1)), 0);
        for (int64_t t = 0; t < total; ++t)
            nodes[size_t(t)] = ctx->lay.inv_host[size_t(bc_tips->tip_nodes[t])];
        PD_CK(ctx->tip_nodes.upload(nodes.data(), nodes.size(), s));
    }
    // the single-PMB-law specialisation needs no per-slot law data
    const bool general = m.n_laws > 1 || ctx->history || ctx->lay.btype_c.p ||
                         ctx->lay.lambda32.p || ctx->lay.beta32.p;
    bool uniform = true;
    for (int64_t i = 1; i < n && uniform; ++i)
        uniform = p.volume[i] == p.volume[0];
    bool any_nofail = false;
    for (int64_t i = 0; i < n && nofail_size == n && !any_nofail; ++i)
        any_nofail = nofail[i] != 0;
    ctx->kind = general ? 2 : ((uniform && !any_nofail) ? 0 : 1);
    ctx->pmb_c = float(m.laws[0].stiffness);
    ctx->pmb_sc = float(m.laws[0].breakpoints[0]);
    ctx->pmb_cv = float(m.laws[0].stiffness * p.volume[0]);
    std::vector<DevLaw> laws(size_t(m.n_laws));
    for (int k = 0; k < m.n_laws; ++k) {
        std::memset(&laws[size_t(k)], 0, sizeof(DevLaw));
        laws[size_t(k)].c = m.laws[k].stiffness;
        laws[size_t(k)].nbp = m.laws[k].n_breakpoints;
        for (int b = 0; b < laws[size_t(k)].nbp; ++b) {
            laws[size_t(k)].bp[b] = m.laws[k].breakpoints[b];
            laws[size_t(k)].f[b] = m.laws[k].forces[b];
        }
    }
    fast_set_laws(laws.data(), m.n_laws, s);
    PD_CK(cudaGetLastError());
    ctx->fast = true;
    PD_CK(cudaStreamSynchronize(s));
    return PD_OK;
}

int launch_step(pd_ctx* ctx, DevArgs& A, int mode) {
    if (ctx->lattice)
        PD_CK(launch_lattice(A, ctx->lat, mode, ctx->stream));
    else if (ctx->fast)
        PD_CK(launch_fast(A, ctx->fast_args(), mode, ctx->kind, ctx->lay.n_tiles, ctx->stream));
    else
        PD_CK(launch_exact(A, mode, ctx->variant == PD_NODE_PARALLEL, ctx->exact_pmb && !A.btype &&
                                                                   !A.lambda && !A.beta,
                           ctx->stream));
    ctx->kernel = t_last_kernel;
    ++ctx->launches;
    return PD_OK;
}

// x, u, v (n x 3 each) and phi (n) of the resident state, reference node
// order, into dev[10 n] (make_snapshot, io.cpp:235-249).
int snapshot_fields(pd_ctx* ctx, double* dev, cudaStream_t s) {
    const int64_t n = ctx->n;
    const int* inv = ctx->permuted() ? ctx->lay.inv.p : nullptr;
    DevBuf<double4> t4;
    DevBuf<int32_t> t1, t2;
    const double4* xv = ctx->xv.p;
    const double4* u = ctx->u[ctx->cur].p;
    const double* v = ctx->v.p;
    const int32_t* nn = ctx->n_neigh.p;
    const int32_t* ini = ctx->initial.p;
    if (inv) {
        PD_CK(t4.alloc(size_t(2 * n)));
        launch_gather_rows<double4, 1>(xv, t4.p, inv, n, s);
        launch_gather_rows<double4, 1>(u, t4.p + n, inv, n, s);
        xv = t4.p;
        u = t4.p + n;
        launch_gather_rows<double, 3>(v, dev + 6 * n, inv, n, s);
        v = nullptr;
        PD_CK(t1.alloc(size_t(n)));
        PD_CK(t2.alloc(size_t(n)));
        launch_gather_rows<int32_t, 1>(nn, t1.p, inv, n, s);
        launch_gather_rows<int32_t, 1>(ini, t2.p, inv, n, s);
        nn = t1.p;
        ini = t2.p;
    }
    launch_unpack_u(xv, n, dev, s);
    launch_unpack_u(u, n, dev + 3 * n, s);
    if (v)
        PD_CK(cudaMemcpyAsync(dev + 6 * n, v, sizeof(double) * 3 * n, cudaMemcpyDeviceToDevice, s));
    launch_damage(nn, ini, n, dev + 9 * n, s);
    ctx->launches += inv ? 9 : 3;
    PD_CK(cudaGetLastError());
    if (inv)
        PD_CK(cudaStreamSynchronize(s));  // the temporaries are released on return
    return PD_OK;
}

void snapshot_worker(pd_ctx* ctx) {
    cudaSetDevice(ctx->device);
    std::vector<double> h;
    for (;;) {
        pd_ctx::SnapJob job;
        {
            std::unique_lock<std::mutex> lk(ctx->snap_mu);
            ctx->snap_cv.wait(lk, [&] { return ctx->snap_stop || !ctx->snap_jobs.empty(); });
            if (ctx->snap_jobs.empty())
                return;
            job = ctx->snap_jobs.front();
            ctx->snap_jobs.pop_front();
        }
        const int64_t n = ctx->n;
        h.resize(size_t(10 * n + 1));
        std::string err;
        if (cudaStreamWaitEvent(ctx->snap_stream, ctx->snap_ready[job.slot], 0) != cudaSuccess ||
            d2h_large(h.data(), ctx->snap_dev[job.slot].p, sizeof(double) * h.size(),
                      ctx->snap_stream) != cudaSuccess) {
            err = "snapshot download failed";
        } else if (long long e; std::memcpy(&e, h.data() + 10 * n, sizeof e), e < job.step) {
            // the run failed at step e before this write step: the reference
            // throws inside step e's force pass and never writes this file
        } else {
            char path[4096];
            std::snprintf(path, sizeof path, ctx->snap_pattern.c_str(), (long long)job.step);
            if (write_snapshot_file(path, job.step, n, h.data(), h.data() + 3 * n,
                                    h.data() + 6 * n, h.data() + 9 * n) != PD_OK)
                err = pd_last_error();
        }
        std::lock_guard<std::mutex> lk(ctx->snap_mu);
        ctx->snap_busy[job.slot] = false;
        if (!err.empty() && ctx->snap_error.empty())
            ctx->snap_error = err;
        ctx->snap_cv.notify_all();
    }
}

// Queue the state of the step just finished for an asynchronous snapshot.
int snapshot_async(pd_ctx* ctx, int64_t step) {
    if (!ctx->snap_thread.joinable()) {
        ctx->snap_stop = false;
        ctx->snap_error.clear();
        if (!ctx->snap_stream)
            PD_CK(cudaStreamCreateWithFlags(&ctx->snap_stream, cudaStreamNonBlocking));
        for (int k = 0; k < 2; ++k)
            if (!ctx->snap_ready[k])
                PD_CK(cudaEventCreateWithFlags(&ctx->snap_ready[k], cudaEventDisableTiming));
        ctx->snap_thread = std::thread(snapshot_worker, ctx);
    }
    int slot = -1;
    {
        std::unique_lock<std::mutex> lk(ctx->snap_mu);
        ctx->snap_cv.wait(lk, [&] { return !ctx->snap_busy[0] || !ctx->snap_busy[1]; });
        slot = ctx->snap_busy[0] ? 1 : 0;
        ctx->snap_busy[slot] = true;
    }
    PD_CK(ctx->snap_dev[slot].alloc(size_t(10 * ctx->n + 1)));
    PD_TRY(snapshot_fields(ctx, ctx->snap_dev[slot].p, ctx->stream));
    // the first failed step rides along, so the writer can drop snapshots
    // queued past a non-finite error (the later step kernels returned early)
    PD_CK(cudaMemcpyAsync(ctx->snap_dev[slot].p + 10 * ctx->n, ctx->err.p, sizeof(long long),
                          cudaMemcpyDeviceToDevice, ctx->stream));
    PD_CK(cudaEventRecord(ctx->snap_ready[slot], ctx->stream));
    {
        std::lock_guard<std::mutex> lk(ctx->snap_mu);
        ctx->snap_jobs.push_back({slot, step});
    }
    ctx->snap_cv.notify_all();
    return PD_OK;
}

// Wait until every queued snapshot is written; report the first failure.
int snapshot_flush(pd_ctx* ctx) {
    if (!ctx->snap_thread.joinable())
        return PD_OK;
    {
        std::unique_lock<std::mutex> lk(ctx->snap_mu);
        ctx->snap_cv.wait(lk, [&] {
            return ctx->snap_jobs.empty() && !ctx->snap_busy[0] && !ctx->snap_busy[1];
        });
        if (!ctx->snap_error.empty()) {
            const std::string e = ctx->snap_error;
            ctx->snap_error.clear();
            return fail(PD_E_RUNTIME, "%s", e.c_str());
        }
    }
    return PD_OK;
}

void snapshot_stop(pd_ctx* ctx) {
    if (!ctx->snap_thread.joinable())
        return;
    {
        std::lock_guard<std::mutex> lk(ctx->snap_mu);
        ctx->snap_stop = true;
    }
    ctx->snap_cv.notify_all();
    ctx->snap_thread.join();
    for (int k = 0; k < 2; ++k)
        if (ctx->snap_ready[k])
            cudaEventDestroy(ctx->snap_ready[k]);
    if (ctx->snap_stream)
        cudaStreamDestroy(ctx->snap_stream);
}

// Slab barrier after a launch that wrote peer ghost rows (no-op on one GPU).
int slab_sync(pd_ctx* ctx) {
    if (ctx->world <= 1)
        return PD_OK;
    SyncArgs S{};
    for (int p = 0; p < ctx->world; ++p)
        S.peer_sync[p] = ctx->peer_sync[p];
    S.my_sync = ctx->sync.p;
    S.err_step = ctx->err.p;
    S.rank = ctx->rank;
    S.world = ctx->world;
    S.epoch = ++ctx->epoch;
    S.timeout_ns = 120LL * 1000 * 1000 * 1000;
    launch_slab_sync(S, ctx->stream);
    ++ctx->launches;
    PD_CK(cudaGetLastError());
    return PD_OK;
}

// Host view of the hook's state: the caller's arrays when the run is a
// one-shot simulate (state is mutated in place like the reference), else the
// staging vectors below.
struct HookStage {
    std::vector<double> u, v, a, hist, body, ext;
    std::vector<int32_t> entries, n_neigh;
};

thread_local bool t_in_batch = false;  // a pd_simulate_batch worker thread

int run_loop(pd_ctx* ctx, const pd_options& opt, pd_write_hook hook, void* user,
             int32_t hook_fields, pd_state* hook_state, pd_tip_record* tips_out,
             int64_t tips_capacity, int64_t* n_tips_out) {
    cudaStream_t s = ctx->stream;
    if (n_tips_out)
        *n_tips_out = 0;
    if (opt.steps < 1)
        return fail(PD_E_INVALID_ARGUMENT, "simulate: steps must be >= 1");
    if (opt.integrator < PD_VELOCITY_VERLET || opt.integrator > PD_EULER_CROMER)
        return fail(PD_E_INVALID_ARGUMENT, "simulate: unknown integrator");
    const int64_t first = opt.first_step, last = opt.first_step + opt.steps;
    int64_t writes = 0;
    if (opt.write_every > 0)
        for (int64_t w = (first / opt.write_every + 1) * opt.write_every; w <= last;
             w += opt.write_every)
            if (w > first)
                ++writes;
    const int64_t n_records = writes * ctx->n_tip_sets;
    if (n_records > tips_capacity)
        return fail(PD_E_INVALID_ARGUMENT, "simulate: tips_out capacity too small");
    if (n_records > 0)
        PD_CK(ctx->tips.alloc(size_t(n_records)));

    if ((opt.variant == PD_FAST) != ctx->fast)
        return fail(PD_E_INVALID_ARGUMENT,
                    "simulate: the variant must match the one the model was uploaded for");
    if (opt.variant != PD_FAST)
        ctx->variant = opt.variant;
    const bool vv = opt.integrator == PD_VELOCITY_VERLET;
    const int mode = vv ? 1 : (opt.integrator == PD_EULER ? 2 : 3);
    const long long none = kNoError;
    PD_CK(cudaMemcpyAsync(ctx->err.p, &none, sizeof none, cudaMemcpyHostToDevice, s));
    ctx->step = first;
    const int cur0 = ctx->cur;
    DevArgs A = ctx->args();
    A.step = first;
    if (vv) {
        launch_vv_prologue(A, s);
        ctx->cur ^= 1;
    } else {
        launch_check_finite(ctx->u[ctx->cur].p, ctx->comp_begin, ctx->comp_end, first,
                            ctx->err.p, s);
    }
    ++ctx->launches;
    PD_TRY(slab_sync(ctx));

    HookStage stage;
    int64_t rec = 0;
    int rc = PD_OK;
    int64_t failed_at = -1;
    // Small lattice models on one GPU: every run of steps without host work
    // in between (write steps, snapshots, the end) is one persistent launch
    // (pd_lattice.cu lattice_small_kernel).  PD_LAT_PERSIST=0 turns it off.
    // (not inside pd_simulate_batch: its models run concurrently on several
    // streams, where one-step launches interleave and cooperative grids of
    // several models would compete for residency)
    const char* persist_var = std::getenv("PD_LAT_PERSIST");
    const bool persist_env = !(persist_var && std::atoi(persist_var) == 0) && !t_in_batch;
    const bool persist = persist_env && ctx->lattice && ctx->world <= 1 &&
                         (!ctx->has_bc || ctx->ramps.count <= 32) &&
                         lattice_small_fits(ctx->lat, mode, ctx->has_bc);
    const unsigned long long small_ctas = persist ? (unsigned long long)lattice_small_ctas(ctx->lat) : 0;
    unsigned long long bar_base = 0;
    int64_t chunk_left = 0;
    if (persist) {
        PD_CK(ctx->bar.alloc(1));
        PD_CK(cudaMemsetAsync(ctx->bar.p, 0, sizeof(unsigned long long), s));
    }
    auto store_at = [&](int64_t st) {
        // forces are kept at write steps and at the end of every run (so a
        // download after the run sees the last step's force field)
        const bool is_write = opt.write_every > 0 && (st + 1) % opt.write_every == 0;
        return (is_write && (ctx->n_tip_sets > 0 || hook)) || st + 1 == last;
    };
    for (int64_t st = first; st < last; ++st) {
        const bool is_write = opt.write_every > 0 && (st + 1) % opt.write_every == 0;
        A = ctx->args();
        A.step = st;
        A.store_forces = store_at(st);
        A.do_drift = st + 1 < last;
        if (persist) {
            if (chunk_left == 0) {
                int64_t e = st;  // the chunk's last step: host work follows it
                while (e + 1 < last && !(opt.write_every > 0 && (e + 1) % opt.write_every == 0) &&
                       !(ctx->snap_every > 0 && (e + 1) % ctx->snap_every == 0))
                    ++e;
                SmallArgs S{};
                S.u[0] = ctx->u[ctx->cur].p;
                S.u[1] = ctx->u[ctx->cur ^ 1].p;
                S.bar = ctx->bar.p;
                S.bar_base = bar_base;
                S.steps = int(std::min<int64_t>(e - st + 1, 1 << 30));
                e = st + S.steps - 1;
                S.store_last = store_at(e);
                S.drift_last = e + 1 < last;
                S.n_ramps = int(ctx->ramps.count);
                PD_CK(launch_lattice_small(A, ctx->lat, mode, S, s));
                ctx->kernel = t_last_kernel;
                ++ctx->launches;
                bar_base += small_ctas * (unsigned long long)(S.steps - 1);
                chunk_left = S.steps;
            }
            --chunk_left;
        } else {
            PD_TRY(launch_step(ctx, A, mode));
            PD_TRY(slab_sync(ctx));
        }
        if (!vv)
            ctx->cur ^= 1;
        if (ctx->snap_every > 0 && (st + 1) % ctx->snap_every == 0) {
            const int64_t saved = ctx->step;
            ctx->step = st + 1;
            const int rs = snapshot_async(ctx, st + 1);
            ctx->step = saved;
            if (rs != PD_OK)
                return rs;
        }
        if (is_write) {
            if (ctx->n_tip_sets > 0) {
                launch_tips(ctx->u[ctx->cur].p, ctx->v.p, ctx->a.p, ctx->xv.p, ctx->body.p,
                            ctx->ext.p, ctx->n_tip_sets, ctx->tip_offsets.p, ctx->tip_nodes.p,
                            st + 1, ctx->tips.p + rec, s);
                ++ctx->launches;
                rec += ctx->n_tip_sets;
            }
            if (hook) {
                long long err = none;
                PD_CK(cudaMemcpyAsync(&err, ctx->err.p, sizeof err, cudaMemcpyDeviceToHost, s));
                PD_CK(cudaStreamSynchronize(s));
                if (err == kPeerTimeout)
                    return fail(PD_E_CUDA, "slab sync: a peer rank did not reach step %lld",
                                (long long)(st + 1));
                if (err == kBarrierTimeout)
                    return fail(PD_E_CUDA, "persistent step launch: grid barrier timeout");
                if (err <= st) {
                    failed_at = err;
                    break;
                }
                const int64_t saved = ctx->step;
                ctx->step = st + 1;
                pd_force_field ff{nullptr, nullptr};
                pd_state view{};
                if (hook_state) {
                    view = *hook_state;
                } else {
                    const int64_t n = ctx->n, slots = n * ctx->N;
                    view.connectivity.n = n;
                    view.connectivity.group_size = ctx->N;
                    if (hook_fields & PD_FIELD_U)
                        stage.u.resize(size_t(3 * n)), view.u = stage.u.data();
                    if (hook_fields & PD_FIELD_V)
                        stage.v.resize(size_t(3 * n)), view.v = stage.v.data();
                    if (hook_fields & PD_FIELD_A)
                        stage.a.resize(size_t(3 * n)), view.a = stage.a.data();
                    if (hook_fields & PD_FIELD_CONNECTIVITY) {
                        stage.entries.resize(size_t(slots));
                        stage.n_neigh.resize(size_t(n));
                        view.connectivity.entries = stage.entries.data();
                        view.connectivity.n_neigh = stage.n_neigh.data();
                    }
                    if ((hook_fields & PD_FIELD_HISTORY) && ctx->history) {
                        stage.hist.resize(size_t(slots));
                        view.bond_history = stage.hist.data();
                        view.bond_history_size = slots;
                    }
                }
                if (hook_fields & PD_FIELD_FORCES) {
                    stage.body.resize(size_t(3 * ctx->n));
                    stage.ext.resize(size_t(3 * ctx->n));
                    ff.body_force = stage.body.data();
                    ff.external_force = stage.ext.data();
                }
                PD_TRY(download(ctx, &view, &ff, hook_fields));
                ctx->step = saved;
                if (hook(user, &view, &ff) != 0) {
                    rc = fail(PD_E_RUNTIME, "simulate: write hook failed at step %lld",
                              (long long)(st + 1));
                    ctx->step = st + 1;
                    break;
                }
            }
        }
        if (vv && st + 1 < last)
            ctx->cur ^= 1;
        ctx->step = st + 1;
    }
    long long err = none;
    PD_CK(cudaMemcpyAsync(&err, ctx->err.p, sizeof err, cudaMemcpyDeviceToHost, s));
    PD_CK(cudaStreamSynchronize(s));
    PD_TRY(snapshot_flush(ctx));
    if (err == kPeerTimeout)
        return fail(PD_E_CUDA, "slab sync: a peer rank did not arrive (timeout)");
    if (err == kBarrierTimeout)
        return fail(PD_E_CUDA, "persistent step launch: grid barrier timeout");
    if (failed_at < 0 && err < last)
        failed_at = err;
    int64_t keep = rec;
    if (failed_at >= 0) {
        // The reference threw inside the force pass of step `failed_at`: the
        // state is the one that force pass saw.
        const int64_t e = failed_at;
        ctx->cur = vv ? (cur0 ^ 1 ^ int((e - first) & 1)) : (cur0 ^ int((e - first) & 1));
        ctx->step = e;
        keep = 0;
        if (opt.write_every > 0)
            for (int64_t w = first + 1; w <= e; ++w)
                if (w % opt.write_every == 0)
                    keep += ctx->n_tip_sets;
        rc = fail(PD_E_RUNTIME, "compute_forces: non-finite displacement at step %lld",
                  (long long)e);
    }
    keep = std::min(keep, rec);
    if (keep > 0 && tips_out)
        PD_CK(cudaMemcpy(tips_out, ctx->tips.p, sizeof(pd_tip_record) * keep,
                         cudaMemcpyDeviceToHost));
    if (n_tips_out)
        *n_tips_out = keep;
    ctx->forces_valid = true;
    return rc;
}

} // namespace

namespace {
int upload_impl(pd_ctx* ctx, const pd_bundle* b, const pd_state* st, int32_t variant);
}

// ---- C ABI ------------------------------------------------------------------

extern "C" {

int pd_abi_version(void) { return PD_ABI_VERSION; }

const char* pd_last_error(void) { return g_err.c_str(); }

int pd_device_count(void) {
    // the visible devices do not change within a process: count them once
    // (cheap attribute queries, not cudaGetDeviceProperties)
    static const int usable = [] {
        int count = 0;
        if (cudaGetDeviceCount(&count) != cudaSuccess) {
            cudaGetLastError();
            return 0;
        }
        int n = 0;
        for (int d = 0; d < count; ++d) {
            int major = 0;
            if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, d) ==
                    cudaSuccess &&
                major >= 10)
                ++n;
        }
        return n;
    }();
    return usable;
}

int pd_ctx_create(int device, pd_ctx** out) {
    *out = nullptr;
    if (pd_device_count() == 0)
        return fail(PD_E_NO_DEVICE, "no sm_100 (B200) device is visible to the CUDA runtime");
    auto* ctx = new pd_ctx;
    ctx->device = device;
    if (select_device(ctx) != PD_OK) {
        delete ctx;
        return PD_E_CUDA;
    }
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
        delete ctx;
        return fail(PD_E_CUDA, "cudaStreamCreate failed");
    }
    *out = ctx;
    return ok();
}

void pd_ctx_destroy(pd_ctx* ctx) {
    if (!ctx)
        return;
    PhaseTimer tm;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    tm.mark("destroy: sync");
    snapshot_stop(ctx);
    for (void* p : ctx->ipc_opened)
        cudaIpcCloseMemHandle(p);
    cudaStreamDestroy(ctx->stream);
    tm.mark("destroy: stream");
    delete ctx;
    tm.mark("destroy: buffers");
}

void* pd_ctx_stream(pd_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

int64_t pd_ctx_launch_count(pd_ctx* ctx) { return ctx ? ctx->launches : 0; }

int pd_ctx_save_state(pd_ctx* ctx, const char* path) {
    PD_TRY(select_device(ctx));
    if (ctx->world > 1 || ctx->partial)
        return fail(PD_E_INVALID_ARGUMENT, "save_state: a slab context holds a local model only");
    cudaStream_t s = ctx->stream;
    const int64_t n = ctx->n, N = ctx->N, slots = n * N;
    const int* inv = ctx->permuted() ? ctx->lay.inv.p : nullptr;
    StreamWriter w;
    PD_TRY(w.open(path));
    w.bytes("PDST", 4);
    w.pod(uint32_t(1));
    w.pod(uint64_t(n));
    w.pod(uint64_t(N));
    w.pod(uint64_t(ctx->step));
    w.pod(double(ctx->horizon));
    // u (double4 {u, no_fail} in device-row order -> flat n x 3, reference order)
    const double4* u = ctx->u[ctx->cur].p;
    if (inv) {
        PD_CK(ctx->scratch_d4.alloc(size_t(n)));
        launch_gather_rows<double4, 1>(u, ctx->scratch_d4.p, inv, n, s);
        u = ctx->scratch_d4.p;
    }
    PD_CK(ctx->scratch_f64.alloc(size_t(3 * n)));
    launch_unpack_u(u, n, ctx->scratch_f64.p, s);
    PD_TRY(w.section_device(7, ctx->scratch_f64.p, 24 * uint64_t(n), s));
    for (int f = 0; f < 2; ++f) {
        const double* src = f == 0 ? ctx->v.p : ctx->a.p;
        if (inv) {
            launch_gather_rows<double, 3>(src, ctx->scratch_f64.p, inv, n, s);
            src = ctx->scratch_f64.p;
        }
        PD_TRY(w.section_device(f == 0 ? 8 : 9, src, 24 * uint64_t(n), s));
    }
    PD_CK(ctx->scratch_i32.alloc(size_t(slots)));
    if (ctx->lattice)
        PD_CK(launch_lattice_materialize(ctx->entries.p, ctx->lmask.p, ctx->own_begin,
                                         ctx->own_end, n, ctx->N, ctx->lat, ctx->scratch_i32.p,
                                         nullptr, s));
    else if (ctx->fast)
        launch_fast_materialize(ctx->lay.origk.p, ctx->entries.p, ctx->lay.inv.p, ctx->lay.tile_of.p,
                                ctx->lay.tile_start.p, ctx->lay.slot_off.p, ctx->fast_T,
                                ctx->lay.lidx.p, nullptr, n, ctx->N, ctx->scratch_i32.p, nullptr, s);
    else
        launch_materialize_entries(ctx->entries.p, ctx->alive.p, n, ctx->N, ctx->W,
                                   ctx->scratch_i32.p, s);
    PD_TRY(w.section_device(1, ctx->scratch_i32.p, 4 * uint64_t(slots), s));
    PD_CK(ctx->scratch_n.alloc(size_t(n)));
    for (int f = 0; f < 2; ++f) {
        const int32_t* src = f == 0 ? ctx->n_neigh.p : ctx->initial.p;
        if (inv) {
            launch_gather_rows<int32_t, 1>(src, ctx->scratch_n.p, inv, n, s);
            src = ctx->scratch_n.p;
        }
        PD_TRY(w.section_device(f == 0 ? 2 : 6, src, 4 * uint64_t(n), s));
    }
    if (ctx->btype.p)
        PD_TRY(w.section_device(5, ctx->btype.p, uint64_t(slots), s));
    if (ctx->history) {
        if (ctx->lattice)
            PD_CK(launch_lattice_materialize(ctx->entries.p, ctx->lmask.p, ctx->own_begin,
                                             ctx->own_end, n, ctx->N, ctx->lat, nullptr,
                                             ctx->hist.p, s));
        else if (ctx->permuted())
            launch_fast_materialize(ctx->lay.origk.p, ctx->entries.p, ctx->lay.inv.p, ctx->lay.tile_of.p,
                                    ctx->lay.tile_start.p, ctx->lay.slot_off.p, ctx->fast_T,
                                    ctx->lay.lidx.p, ctx->lay.hist32.p, n, ctx->N, nullptr,
                                    ctx->hist.p, s);
        PD_TRY(w.section_device(10, ctx->hist.p, 8 * uint64_t(slots), s));
    } else if (ctx->hist_keep.p) {
        PD_TRY(w.section_device(10, ctx->hist_keep.p, 8 * uint64_t(slots), s));
    }
    ctx->launches += 8;
    PD_TRY(w.close());
    return ok();
}

int pd_ctx_write_snapshot(pd_ctx* ctx, const char* path) {
    PD_TRY(select_device(ctx));
    if (ctx->world > 1 || ctx->partial)
        return fail(PD_E_INVALID_ARGUMENT, "write_snapshot: a slab context holds a local model only");
    DevBuf<double> buf;
    PD_CK(buf.alloc(size_t(10 * ctx->n)));
    PD_TRY(snapshot_fields(ctx, buf.p, ctx->stream));
    std::vector<double> h(size_t(10 * ctx->n));
    PD_CK(d2h_large(h.data(), buf.p, sizeof(double) * h.size(), ctx->stream));
    const int64_t n = ctx->n;
    PD_TRY(write_snapshot_file(path, ctx->step, n, h.data(), h.data() + 3 * n, h.data() + 6 * n,
                               h.data() + 9 * n));
    return ok();
}

int pd_ctx_snapshot_every(pd_ctx* ctx, int64_t every, const char* pattern) {
    PD_TRY(select_device(ctx));
    if (every < 0)
        return fail(PD_E_INVALID_ARGUMENT, "snapshot_every: negative cadence");
    if (every > 0 && (ctx->world > 1 || ctx->partial))
        return fail(PD_E_INVALID_ARGUMENT, "snapshot_every: a slab context holds a local model only");
    ctx->snap_every = every;
    ctx->snap_pattern = pattern ? pattern : "";
    return ok();
}

const char* pd_ctx_kernel(pd_ctx* ctx) { return ctx ? ctx->kernel : ""; }

int pd_ctx_layout(pd_ctx* ctx) {
    if (!ctx || !ctx->fast)
        return PD_LAYOUT_EXACT;
    return ctx->lattice ? PD_LAYOUT_LATTICE : PD_LAYOUT_TILES;
}

int pd_ctx_upload(pd_ctx* ctx, const pd_bundle* b, const pd_state* st, int32_t variant) {
    ctx->partial = false;
    return upload_impl(ctx, b, st, variant);
}

int pd_ctx_upload_part(pd_ctx* ctx, const pd_bundle* b, const pd_state* st, int32_t variant,
                       int64_t own_begin, int64_t own_end) {
    if (own_begin < 0 || own_end < own_begin || own_end > b->particles.n)
        return fail(PD_E_INVALID_ARGUMENT, "slab: owned range [%lld, %lld) outside the %lld local nodes",
                    (long long)own_begin, (long long)own_end, (long long)b->particles.n);
    ctx->partial = true;
    ctx->own_begin = own_begin;
    ctx->own_end = own_end;
    const int rc = upload_impl(ctx, b, st, variant);
    return rc;
}

int pd_ctx_internal_index(pd_ctx* ctx, const int64_t* local, int64_t count, int64_t* out) {
    for (int64_t k = 0; k < count; ++k) {
        if (local[k] < 0 || local[k] >= ctx->n)
            return fail(PD_E_INVALID_ARGUMENT, "internal_index: node %lld out of range",
                        (long long)local[k]);
        out[k] = ctx->row_of(local[k]);
    }
    return ok();
}

int pd_ctx_export(pd_ctx* ctx, pd_peer_handle* out) {
    PD_TRY(select_device(ctx));
    std::memset(out, 0, sizeof *out);
    if (!ctx->sync.p) {
        PD_CK(ctx->sync.alloc(2 * PD_MAX_RANKS));
        PD_CK(cudaMemset(ctx->sync.p, 0, sizeof(unsigned long long) * 2 * PD_MAX_RANKS));
        PD_CK(cudaDeviceSynchronize());
    }
    if (!ctx->u[0].p || !ctx->u[1].p)
        return fail(PD_E_INVALID_ARGUMENT, "export: upload the model first");
    out->device = ctx->device;
    out->pid = int32_t(getpid());
    cudaIpcMemHandle_t h;
    PD_CK(cudaIpcGetMemHandle(&h, ctx->u[0].p));
    std::memcpy(out->ipc_u0, &h, sizeof h);
    PD_CK(cudaIpcGetMemHandle(&h, ctx->u[1].p));
    std::memcpy(out->ipc_u1, &h, sizeof h);
    PD_CK(cudaIpcGetMemHandle(&h, ctx->sync.p));
    std::memcpy(out->ipc_sync, &h, sizeof h);
    out->u0 = uint64_t(reinterpret_cast<uintptr_t>(ctx->u[0].p));
    out->u1 = uint64_t(reinterpret_cast<uintptr_t>(ctx->u[1].p));
    out->sync = uint64_t(reinterpret_cast<uintptr_t>(ctx->sync.p));
    return ok();
}

int pd_ctx_connect(pd_ctx* ctx, int32_t rank, int32_t world, const pd_peer_handle* peers,
                   int32_t lo, int32_t hi, const int64_t* send_lo, const int64_t* send_hi) {
    PD_TRY(select_device(ctx));
    if (world < 1 || world > PD_MAX_RANKS || rank < 0 || rank >= world)
        return fail(PD_E_INVALID_ARGUMENT, "connect: rank %d of %d (at most %d ranks)", rank,
                    world, PD_MAX_RANKS);
    if ((lo >= world) || (hi >= world) || (lo == rank && lo >= 0) || (hi == rank && hi >= 0))
        return fail(PD_E_INVALID_ARGUMENT, "connect: bad neighbour ranks %d / %d", lo, hi);
    if (!ctx->sync.p)
        return fail(PD_E_INVALID_ARGUMENT, "connect: export this context first");
    // every kernel a run may launch is loaded now: under CUDA lazy loading a
    // first launch can wait for the whole device, which would deadlock
    // against a peer rank's spinning sync kernel (callers barrier after
    // connect, so no rank spins before every rank has loaded).  Modules load
    // per device, so each device is preloaded once (thread ranks on several
    // GPUs of one process each load their own device)
    static std::once_flag loaded[64];
    if (ctx->device < 0 || ctx->device >= 64)
        return fail(PD_E_INVALID_ARGUMENT, "connect: device ordinal %d out of range", ctx->device);
    std::call_once(loaded[ctx->device], [] {
        preload_aux();
        preload_exact();
        preload_fast();
        preload_lattice();
    });
    PD_CK(cudaGetLastError());
    const int me = int(getpid());
    // map every peer's u buffers and sync words
    void* mapped[PD_MAX_RANKS][3] = {};
    for (int p = 0; p < world; ++p) {
        if (p == rank) {
            mapped[p][0] = ctx->u[0].p;
            mapped[p][1] = ctx->u[1].p;
            mapped[p][2] = ctx->sync.p;
            continue;
        }
        const pd_peer_handle& h = peers[p];
        if (h.pid == me) {
            if (h.device != ctx->device) {
                const cudaError_t e = cudaDeviceEnablePeerAccess(h.device, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
                    PD_CK(e);
                cudaGetLastError();
            }
            mapped[p][0] = reinterpret_cast<void*>(uintptr_t(h.u0));
            mapped[p][1] = reinterpret_cast<void*>(uintptr_t(h.u1));
            mapped[p][2] = reinterpret_cast<void*>(uintptr_t(h.sync));
        } else {
            const uint8_t* src[3] = {h.ipc_u0, h.ipc_u1, h.ipc_sync};
            for (int k = 0; k < 3; ++k) {
                cudaIpcMemHandle_t ih;
                std::memcpy(&ih, src[k], sizeof ih);
                PD_CK(cudaIpcOpenMemHandle(&mapped[p][k], ih, cudaIpcMemLazyEnablePeerAccess));
                ctx->ipc_opened.push_back(mapped[p][k]);
            }
        }
    }
    ctx->rank = rank;
    ctx->world = world;
    ctx->epoch = 0;
    for (int p = 0; p < world; ++p)
        ctx->peer_sync[p] = static_cast<unsigned long long*>(mapped[p][2]);
    for (int side = 0; side < 2; ++side) {
        const int r = side == 0 ? lo : hi;
        for (int par = 0; par < 2; ++par)
            ctx->peer_u[side][par] = r >= 0 ? static_cast<double4*>(mapped[r][par]) : nullptr;
    }
    // per device row: the peer rows this owned node's u goes to
    std::vector<int2> x(size_t(ctx->n), make_int2(-1, -1));
    for (int64_t i = ctx->own_begin; i < ctx->own_end; ++i) {
        const int64_t row = ctx->row_of(i);
        const int64_t a = (lo >= 0 && send_lo) ? send_lo[i] : -1;
        const int64_t b = (hi >= 0 && send_hi) ? send_hi[i] : -1;
        if (a >= INT32_MAX || b >= INT32_MAX)
            return fail(PD_E_INVALID_ARGUMENT, "connect: peer row index out of range");
        x[size_t(row)] = make_int2(int(a), int(b));
    }
    PD_CK(ctx->xfer.upload(x.data(), x.size(), ctx->stream));
    PD_CK(cudaStreamSynchronize(ctx->stream));
    return ok();
}

int pd_ctx_node_values(pd_ctx* ctx, const int64_t* local, int64_t count, double* out) {
    PD_TRY(select_device(ctx));
    std::vector<long long> rows(size_t(std::max<int64_t>(count, 1)), 0);
    for (int64_t k = 0; k < count; ++k) {
        if (local[k] < 0 || local[k] >= ctx->n)
            return fail(PD_E_INVALID_ARGUMENT, "node_values: node %lld out of range",
                        (long long)local[k]);
        rows[size_t(k)] = ctx->row_of(local[k]);
    }
    if (count == 0)
        return ok();
    cudaStream_t s = ctx->stream;
    DevBuf<long long> d_rows;
    DevBuf<double> d_out;
    PD_CK(d_rows.upload(rows.data(), size_t(count), s));
    PD_CK(d_out.alloc(size_t(15 * count)));
    launch_node_values(ctx->u[ctx->cur].p, ctx->v.p, ctx->a.p, ctx->xv.p, ctx->body.p, ctx->ext.p,
                       d_rows.p, count, d_out.p, s);
    ++ctx->launches;
    PD_CK(cudaMemcpyAsync(out, d_out.p, sizeof(double) * 15 * count, cudaMemcpyDeviceToHost, s));
    PD_CK(cudaStreamSynchronize(s));
    return ok();
}

} // extern "C"

namespace {

int upload_impl(pd_ctx* ctx, const pd_bundle* b, const pd_state* st, int32_t variant) {
    PD_TRY(select_device(ctx));
    PhaseTimer tm;
    if (variant < PD_BOND_PARALLEL || variant > PD_FAST)
        return fail(PD_E_INVALID_ARGUMENT, "unknown kernel variant %d", variant);
    // ModelBundle::validate (engine.cpp:335-341)
    PD_TRY(particles_validate(b->particles));
    PD_TRY(model_validate(b->model));
    PD_TRY(bc_validate(b->bc, b->particles.n));
    if (!(b->dt > 0))
        return fail(PD_E_INVALID_ARGUMENT, "ModelBundle: dt must be positive");
    if (st->connectivity.n != b->particles.n)
        return fail(PD_E_INVALID_ARGUMENT, "simulate: state does not match the bundle");
    tm.mark("upload: validate");
    // simulate: corr.no_failure = bc.no_failure (engine.cpp:386-387)
    PD_TRY(upload_common(ctx, b->particles, *st, b->model, b->corrections, b->bc.no_failure,
                         b->bc.no_failure_size));
    tm.mark("upload: common");
    const int64_t slots = ctx->n * ctx->N;
    if (b->corrections.lambda_size != 0 && b->corrections.lambda_size != slots)
        return fail(PD_E_INVALID_ARGUMENT, "compute_forces: lambda size mismatch");
    if (b->corrections.beta_size != 0 && b->corrections.beta_size != slots)
        return fail(PD_E_INVALID_ARGUMENT, "compute_forces: beta size mismatch");
    PD_TRY(upload_bc(ctx, b->bc));
    tm.mark("upload: bc");
    if (variant == PD_FAST) {
        bool lattice = false;
        PD_TRY(fast_laws_ok(b->model));
        PD_TRY(try_lattice(ctx, b->particles, *st, b->model, b->corrections, b->bc.no_failure,
                           b->bc.no_failure_size, &lattice));
        if (!lattice) {
            pd_boundary bc = b->bc;
            PD_TRY(setup_fast(ctx, b->particles, *st, b->model, b->corrections, b->bc.no_failure,
                              b->bc.no_failure_size, &bc));
        }
        tm.mark(lattice ? "upload: lattice masks" : "upload: fast layout");
    }
    ctx->variant = variant;
    ctx->dt = b->dt;
    return ok();
}

} // namespace

extern "C" {

int pd_ctx_run(pd_ctx* ctx, const pd_options* options, pd_write_hook on_write, void* user,
               int32_t hook_fields, pd_tip_record* tips_out, int64_t tips_capacity,
               int64_t* n_tips_out) {
    PD_TRY(select_device(ctx));
    const int rc = run_loop(ctx, *options, on_write, user, hook_fields, nullptr, tips_out,
                            tips_capacity, n_tips_out);
    return rc == PD_OK ? ok() : rc;
}

int pd_ctx_compute_forces(pd_ctx* ctx) {
    PD_TRY(select_device(ctx));
    cudaStream_t s = ctx->stream;
    const long long none = kNoError;
    PD_CK(cudaMemcpyAsync(ctx->err.p, &none, sizeof none, cudaMemcpyHostToDevice, s));
    launch_check_finite(ctx->u[ctx->cur].p, 0, ctx->n, ctx->step, ctx->err.p, s);
    ++ctx->launches;
    long long err = none;
    PD_CK(cudaMemcpyAsync(&err, ctx->err.p, sizeof err, cudaMemcpyDeviceToHost, s));
    PD_CK(cudaStreamSynchronize(s));
    if (err != none)
        return fail(PD_E_RUNTIME, "compute_forces: non-finite displacement at step %lld",
                    (long long)ctx->step);
    DevArgs A = ctx->args();
    PD_TRY(launch_step(ctx, A, 0));
    PD_CK(cudaStreamSynchronize(s));
    ctx->forces_valid = true;
    return ok();
}

int pd_ctx_download(pd_ctx* ctx, pd_state* state, pd_force_field* forces, int32_t fields) {
    PD_TRY(select_device(ctx));
    PD_TRY(download(ctx, state, forces, fields));
    return ok();
}

int pd_ctx_damage(pd_ctx* ctx, double* phi_out) {
    PD_TRY(select_device(ctx));
    cudaStream_t s = ctx->stream;
    PD_CK(ctx->scratch_f64.alloc(size_t(2 * ctx->n)));
    launch_damage(ctx->n_neigh.p, ctx->initial.p, ctx->n, ctx->scratch_f64.p, s);
    ++ctx->launches;
    const double* phi = ctx->scratch_f64.p;
    if (ctx->permuted()) {
        launch_gather_rows<double, 1>(phi, ctx->scratch_f64.p + ctx->n, ctx->lay.inv.p, ctx->n, s);
        ++ctx->launches;
        phi = ctx->scratch_f64.p + ctx->n;
    }
    PD_CK(cudaMemcpyAsync(phi_out, phi, sizeof(double) * ctx->n, cudaMemcpyDeviceToHost, s));
    PD_CK(cudaStreamSynchronize(s));
    return ok();
}

int64_t pd_ctx_live_bonds(pd_ctx* ctx) {
    if (select_device(ctx) != PD_OK)
        return -1;
    cudaStream_t s = ctx->stream;
    if (ctx->counter.alloc(1) != cudaSuccess)
        return -1;
    cudaMemsetAsync(ctx->counter.p, 0, sizeof(unsigned long long), s);
    launch_sum(ctx->n_neigh.p, ctx->n, ctx->counter.p, s);
    ++ctx->launches;
    unsigned long long total = 0;
    cudaMemcpyAsync(&total, ctx->counter.p, sizeof total, cudaMemcpyDeviceToHost, s);
    if (cudaStreamSynchronize(s) != cudaSuccess)
        return -1;
    return int64_t(total);
}

int pd_compute_forces(int32_t variant, pd_state* state, const pd_particles* particles,
                      const pd_damage_model* model, const pd_corrections* corr,
                      pd_force_field* out) {
    // check_force_inputs (engine.cpp:30-49), in the reference's order
    const int64_t n = state->connectivity.n;
    if (particles->n != n)
        return fail(PD_E_INVALID_ARGUMENT, "compute_forces: particle set does not match state");
    const int64_t slots = n * state->connectivity.group_size;
    if (corr->lambda_size != 0 && corr->lambda_size != slots)
        return fail(PD_E_INVALID_ARGUMENT, "compute_forces: lambda size mismatch");
    if (corr->beta_size != 0 && corr->beta_size != slots)
        return fail(PD_E_INVALID_ARGUMENT, "compute_forces: beta size mismatch");
    if (corr->no_failure_size != 0 && corr->no_failure_size != n)
        return fail(PD_E_INVALID_ARGUMENT, "compute_forces: no_failure size mismatch");
    if (model->n_laws >= 1 && needs_history(*model) && state->bond_history_size != slots)
        return fail(PD_E_INVALID_ARGUMENT, "compute_forces: model needs per-bond history");
    if (state->connectivity.bond_type_size != 0 && model->n_laws < 2 &&
        state->connectivity.bond_type_size != slots)
        return fail(PD_E_INVALID_ARGUMENT, "compute_forces: bond_type size mismatch");
    PD_TRY(model_validate(*model));
    for (int64_t k = 0; k < 3 * n; ++k)
        if (!std::isfinite(state->u[k]))
            return fail(PD_E_RUNTIME, "compute_forces: non-finite displacement at step %lld",
                        (long long)state->step);
    if (variant < PD_BOND_PARALLEL || variant > PD_FAST)
        return fail(PD_E_INVALID_ARGUMENT, "unknown kernel variant %d", variant);
    if (n == 0)
        return ok();

    pd_ctx* ctx = nullptr;
    PD_TRY(pd_ctx_create(0, &ctx));
    struct Guard {
        pd_ctx* c;
        ~Guard() { pd_ctx_destroy(c); }
    } guard{ctx};
    pd_state st = *state;
    st.v = nullptr;
    st.a = nullptr;
    PD_TRY(upload_common(ctx, *particles, st, *model, *corr, corr->no_failure,
                         corr->no_failure_size));
    if (variant == PD_FAST) {
        bool lattice = false;
        PD_TRY(fast_laws_ok(*model));
        PD_TRY(try_lattice(ctx, *particles, st, *model, *corr, corr->no_failure,
                           corr->no_failure_size, &lattice));
        if (!lattice)
            PD_TRY(setup_fast(ctx, *particles, st, *model, *corr, corr->no_failure,
                              corr->no_failure_size, nullptr));
    }
    ctx->variant = variant;
    DevArgs A = ctx->args();
    PD_TRY(launch_step(ctx, A, 0));
    pd_force_field ff{out->body_force, nullptr};
    PD_TRY(download(ctx, state, &ff,
                    PD_FIELD_CONNECTIVITY | PD_FIELD_HISTORY | PD_FIELD_FORCES));
    return ok();
}

int pd_simulate(const pd_bundle* bundle, pd_state* state, const pd_options* options,
                pd_write_hook on_write, void* user, pd_tip_record* tips_out,
                int64_t tips_capacity, int64_t* n_tips_out) {
    if (n_tips_out)
        *n_tips_out = 0;
    if (options->steps < 1)
        return fail(PD_E_INVALID_ARGUMENT, "simulate: steps must be >= 1");
    if (bundle->model.n_laws >= 1 && needs_history(bundle->model) &&
        state->bond_history_size != state->connectivity.n * state->connectivity.group_size)
        return fail(PD_E_INVALID_ARGUMENT, "simulate: bond_history must be sized n x N");
    PhaseTimer tm;
    pd_ctx* ctx = nullptr;
    PD_TRY(pd_ctx_create(0, &ctx));
    struct Guard {
        pd_ctx* c;
        PhaseTimer* t;
        ~Guard() {
            pd_ctx_destroy(c);
            t->mark("simulate: destroy");
        }
    } guard{ctx, &tm};
    tm.mark("simulate: create");
    PD_TRY(pd_ctx_upload(ctx, bundle, state, options->variant));
    PD_CK(cudaStreamSynchronize(ctx->stream));
    tm.mark("simulate: upload");
    // every download of this call writes into the caller's own arrays, which
    // hold the uploaded rows until the first download rewrites changed rows
    ctx->dst_has_upload = true;
    int rc = run_loop(ctx, *options, on_write, user, PD_FIELD_ALL, state, tips_out, tips_capacity,
                      n_tips_out);
    PD_CK(cudaStreamSynchronize(ctx->stream));
    tm.mark("simulate: run");
    // the state is the caller's in every outcome, as the reference mutates in place
    const int rc2 = download(ctx, state, nullptr,
                             PD_FIELD_U | PD_FIELD_V | PD_FIELD_A | PD_FIELD_CONNECTIVITY |
                                 PD_FIELD_HISTORY);
    tm.mark("simulate: download");
    if (rc != PD_OK)
        return rc;
    if (rc2 != PD_OK)
        return rc2;
    return ok();
}

int pd_simulate_batch(int32_t k, const pd_bundle* bundles, pd_state* states,
                      const pd_options* options, pd_tip_record* tips_out,
                      const int64_t* tips_offset, int64_t* n_tips_out, int32_t* status,
                      int32_t threads) {
    if (k < 0)
        return fail(PD_E_INVALID_ARGUMENT, "simulate_batch: negative model count");
    if (threads <= 0)
        threads = int32_t(std::min<unsigned>(8u, std::max(1u, std::thread::hardware_concurrency())));
    threads = std::min<int32_t>(threads, std::max<int32_t>(k, 1));
    std::vector<std::string> msgs(static_cast<size_t>(k));
    std::atomic<int32_t> next{0};
    auto worker = [&] {
        t_in_batch = true;
        for (;;) {
            const int32_t m = next.fetch_add(1);
            if (m >= k)
                return;
            pd_tip_record* tips = nullptr;
            int64_t cap = 0;
            if (tips_out && tips_offset) {
                tips = tips_out + tips_offset[m];
                cap = tips_offset[m + 1] - tips_offset[m];
            }
            int64_t got = 0;
            const int rc = pd_simulate(&bundles[m], &states[m], &options[m], nullptr, nullptr, tips,
                                       cap, &got);
            status[m] = rc;
            if (n_tips_out)
                n_tips_out[m] = got;
            if (rc != PD_OK)
                msgs[size_t(m)] = pd_last_error();
        }
    };
    std::vector<std::thread> pool;
    for (int32_t t = 0; t < threads; ++t)
        pool.emplace_back(worker);
    for (auto& th : pool)
        th.join();
    for (int32_t m = 0; m < k; ++m)
        if (status[m] != PD_OK)
            return fail(status[m], "simulate_batch: model %d: %s", m, msgs[size_t(m)].c_str());
    return ok();
}

int pd_damage(const pd_neighbor_list* family, double* phi) {
    // local_damage's range check (formulas.hpp:49-55) on the inputs, then K3 on the device
    const int64_t n = family->n;
    for (int64_t i = 0; i < n; ++i) {
        const int32_t init = family->initial_n_neigh[i];
        const int32_t cur = family->n_neigh[i];
        if (init > 0 && (cur < 0 || cur > init))
            return fail(PD_E_DOMAIN, "local_damage: current count out of range");
    }
    if (n == 0)
        return ok();
    pd_ctx* ctx = nullptr;
    PD_TRY(pd_ctx_create(0, &ctx));
    struct Guard {
        pd_ctx* c;
        ~Guard() { pd_ctx_destroy(c); }
    } guard{ctx};
    cudaStream_t s = ctx->stream;
    ctx->n = n;
    PD_CK(ctx->n_neigh.upload(family->n_neigh, size_t(n), s));
    PD_CK(ctx->initial.upload(family->initial_n_neigh, size_t(n), s));
    return pd_ctx_damage(ctx, phi);
}


// ---- the reference's stand-alone integrators and boundary passes ----------
// (engine.hpp:38-78, engine.cpp:187-305) on the device over host buffers:
// each call uploads the arrays it reads, runs one kernel with the reference's
// expression order (pd_aux.cu, -fmad=false) and writes back the arrays the
// reference writes, so hand-composed steps (test_engine.cpp:196-357) give the
// reference's bits.

static int integrate_host(const char* who, int op, pd_state* st, const pd_force_field* f,
                          double dt, double damping, const double* density, int64_t density_size) {
    if (!(dt > 0))
        return fail(PD_E_DOMAIN, "%s: dt must be positive", who);
    const int64_t n = st->connectivity.n;
    if (op != 0) {  // check_density (engine.cpp:177-183)
        if (density_size != n)
            return fail(PD_E_INVALID_ARGUMENT,
                        "integrator: density array does not match node count");
        if (par_any(n, [&](int64_t i) { return !(density[i] > 0); }))
            return fail(PD_E_DOMAIN, "integrator: density must be positive");
    }
    if (n == 0)
        return ok();
    pd_ctx* ctx = nullptr;
    PD_TRY(pd_ctx_create(0, &ctx));
    struct Guard {
        pd_ctx* c;
        ~Guard() { pd_ctx_destroy(c); }
    } guard{ctx};
    cudaStream_t s = ctx->stream;
    const size_t n3 = size_t(3 * n);
    DevBuf<double> u, v, a, body, ext, rho;
    PD_CK(v.upload(st->v, n3, s));
    PD_CK(a.upload(st->a, n3, s));
    if (op != 1)
        PD_CK(u.upload(st->u, n3, s));
    if (op != 0) {
        PD_CK(body.upload(f->body_force, n3, s));
        PD_CK(ext.upload(f->external_force, n3, s));
        PD_CK(rho.upload(density, size_t(n), s));
    }
    IntegrateArgs I{u.p, v.p, a.p, body.p, ext.p, rho.p, (long long)n, dt, damping, op};
    launch_integrate(I, s);
    PD_CK(cudaGetLastError());
    if (op != 1)
        PD_CK(cudaMemcpyAsync(st->u, u.p, sizeof(double) * n3, cudaMemcpyDeviceToHost, s));
    if (op != 0) {
        PD_CK(cudaMemcpyAsync(st->v, v.p, sizeof(double) * n3, cudaMemcpyDeviceToHost, s));
        PD_CK(cudaMemcpyAsync(st->a, a.p, sizeof(double) * n3, cudaMemcpyDeviceToHost, s));
    }
    PD_CK(cudaStreamSynchronize(s));
    return ok();
}

static int boundary_host(int ops, pd_state* st, const pd_boundary* bc, int64_t step, double dt,
                         pd_force_field* out, int64_t n) {
    if (n == 0)
        return ok();
    // the device reads kind / magnitude / ramp_id for all 3n node-axes and
    // the ramp each names: sizes and ids are checked first (the reference
    // indexes them unchecked outside apply_boundary)
    if (bc->kind_size != 3 * n || bc->magnitude_size != 3 * n || bc->ramp_id_size != 3 * n)
        return fail(PD_E_INVALID_ARGUMENT,
                    "BoundaryConditions: field lengths do not match node count");
    if (bc->n_ramps < 1 || par_any(3 * n, [&](int64_t k) { return bc->ramp_id[k] >= bc->n_ramps; }))
        return fail(PD_E_INVALID_ARGUMENT, "BoundaryConditions: ramp id out of range");
    pd_ctx* ctx = nullptr;
    PD_TRY(pd_ctx_create(0, &ctx));
    struct Guard {
        pd_ctx* c;
        ~Guard() { pd_ctx_destroy(c); }
    } guard{ctx};
    cudaStream_t s = ctx->stream;
    const size_t n3 = size_t(3 * n);
    std::vector<DevRamp> ramps(size_t(bc->n_ramps));
    for (int k = 0; k < bc->n_ramps; ++k)
        ramps[size_t(k)] = DevRamp{bc->ramps[k].kind, 0, bc->ramps[k].rise_steps,
                                   bc->ramps[k].target_scale};
    DevBuf<double> u, v, a, ext, mag;
    DevBuf<uint8_t> kind, rid;
    DevBuf<DevRamp> dr;
    PD_CK(kind.upload(bc->kind, n3, s));
    PD_CK(mag.upload(bc->magnitude, n3, s));
    PD_CK(rid.upload(bc->ramp_id, n3, s));
    PD_CK(dr.upload(ramps.data(), ramps.size(), s));
    if (ops & 1)
        PD_CK(u.upload(st->u, n3, s));
    if (ops & 2) {
        PD_CK(v.upload(st->v, n3, s));
        PD_CK(a.upload(st->a, n3, s));
    }
    if (ops & 4)
        PD_CK(ext.upload(out->external_force, n3, s));
    BoundaryArgs B{u.p, v.p, a.p, ext.p, kind.p, mag.p, rid.p, dr.p, (long long)n,
                   (long long)step, dt, ops};
    launch_boundary(B, s);
    PD_CK(cudaGetLastError());
    if (ops & 1)
        PD_CK(cudaMemcpyAsync(st->u, u.p, sizeof(double) * n3, cudaMemcpyDeviceToHost, s));
    if (ops & 2) {
        PD_CK(cudaMemcpyAsync(st->v, v.p, sizeof(double) * n3, cudaMemcpyDeviceToHost, s));
        PD_CK(cudaMemcpyAsync(st->a, a.p, sizeof(double) * n3, cudaMemcpyDeviceToHost, s));
    }
    if (ops & 4)
        PD_CK(cudaMemcpyAsync(out->external_force, ext.p, sizeof(double) * n3,
                              cudaMemcpyDeviceToHost, s));
    PD_CK(cudaStreamSynchronize(s));
    return ok();
}

int pd_verlet_drift(pd_state* state, double dt) {
    return integrate_host("verlet_drift", 0, state, nullptr, dt, 0.0, nullptr, 0);
}

int pd_verlet_kick(pd_state* state, const pd_force_field* forces, double dt, double damping,
                   const double* density, int64_t density_size) {
    return integrate_host("verlet_kick", 1, state, forces, dt, damping, density, density_size);
}

int pd_step_euler(pd_state* state, const pd_force_field* forces, double dt, const double* density,
                  int64_t density_size) {
    return integrate_host("step_euler", 2, state, forces, dt, 0.0, density, density_size);
}

int pd_step_euler_cromer(pd_state* state, const pd_force_field* forces, double dt,
                         const double* density, int64_t density_size) {
    return integrate_host("step_euler_cromer", 3, state, forces, dt, 0.0, density, density_size);
}

int pd_step_velocity_verlet(pd_state* state, pd_force_eval forces, void* user,
                            pd_force_field* scratch, double dt, double damping,
                            const double* density, int64_t density_size) {
    // step_velocity_verlet (engine.cpp:254-260): drift, forces at the advanced
    // positions (the caller's ForceEval, e.g. pd_compute_forces), kick
    PD_TRY(pd_verlet_drift(state, dt));
    if (forces && forces(user, state, scratch) != 0)
        return fail(PD_E_RUNTIME, "step_velocity_verlet: force evaluation failed");
    PD_TRY(pd_verlet_kick(state, scratch, dt, damping, density, density_size));
    state->step += 1;
    return ok();
}

int pd_apply_displacement_positions(pd_state* state, const pd_boundary* bc, int64_t step) {
    return boundary_host(1, state, bc, step, 1.0, nullptr, state->connectivity.n);
}

int pd_apply_displacement_kinematics(pd_state* state, const pd_boundary* bc, int64_t step,
                                     double dt) {
    return boundary_host(2, state, bc, step, dt, nullptr, state->connectivity.n);
}

int pd_accumulate_external_force(const pd_boundary* bc, int64_t step, pd_force_field* out,
                                 int64_t n) {
    return boundary_host(4, nullptr, bc, step, 1.0, out, n);
}

int pd_apply_boundary(pd_state* state, const pd_boundary* bc, int64_t step, double dt,
                      pd_force_field* out) {
    // apply_boundary (engine.cpp:299-305): validate, positions, kinematics, forces
    PD_TRY(bc_validate(*bc, state->connectivity.n));
    return boundary_host(7, state, bc, step, dt, out, state->connectivity.n);
}

} // extern "C"

