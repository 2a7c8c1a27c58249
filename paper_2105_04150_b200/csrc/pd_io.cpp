// pd_io.cpp -- the reference's binary containers (io.cpp:297-564), byte for
// byte: PDST (restart state) and PDNL (family cache).
//
//   "PDST" u32 version=1, u64 n, u64 N, u64 step, f64 horizon, then sections
//   "PDNL" u32 version=1, u64 n, u64 N,           f64 horizon, then sections
//   section = u32 id, u64 byte length, payload; Real arrays widened to f64.
//   Section order on write follows save_state / save_cache exactly, so files
//   written here are identical to the reference's (tests/test_io_formats.py).
//
// Host entry points read and write caller-owned arrays; pd_ctx_save_state
// (pd_host.cu) streams a resident state straight from HBM through the same
// writer (StreamWriter::section_device), so a 10-30M-node restart file never
// needs a host-size copy of the state.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "pd_internal.h"

namespace pdb {

namespace {

enum : uint32_t {
    sec_entries = 1,
    sec_n_neigh = 2,
    sec_lambda = 3,
    sec_beta = 4,
    sec_bond_type = 5,
    sec_initial_n_neigh = 6,
    sec_u = 7,
    sec_v = 8,
    sec_a = 9,
    sec_history = 10,
};
constexpr uint32_t kVersion = 1;

int io_fail(const std::string& path, const std::string& what) {
    return set_error(PD_E_RUNTIME, (path + ": " + what).c_str());  // IoError (io.cpp:24-26)
}

struct Reader {
    FILE* f = nullptr;
    std::string path;
    uint64_t remaining = 0;
    ~Reader() {
        if (f)
            std::fclose(f);
    }
    int open(const char* p) {
        path = p;
        f = std::fopen(p, "rb");
        if (!f)
            return io_fail(path, "cannot open file");
        std::fseek(f, 0, SEEK_END);
        remaining = uint64_t(std::ftell(f));
        std::fseek(f, 0, SEEK_SET);
        return PD_OK;
    }
    int bytes(void* dst, uint64_t len) {
        if (len > remaining)
            return io_fail(path, "truncated file");
        if (len && std::fread(dst, 1, size_t(len), f) != size_t(len))
            return io_fail(path, "truncated file");
        remaining -= len;
        return PD_OK;
    }
    int skip(uint64_t len) {
        if (len > remaining)
            return io_fail(path, "truncated file");
        std::fseek(f, long(len), SEEK_CUR);
        remaining -= len;
        return PD_OK;
    }
    template <class T> int pod(T& v) { return bytes(&v, sizeof(T)); }
};

#define IO_TRY(expr)                                                                             \
    do {                                                                                         \
        const int rc_ = (expr);                                                                  \
        if (rc_ != PD_OK)                                                                        \
            return rc_;                                                                          \
    } while (0)

int check_magic(Reader& r, const char expect[4]) {
    char magic[4];
    IO_TRY(r.bytes(magic, 4));
    if (std::memcmp(magic, expect, 4) != 0)
        return io_fail(r.path, std::string("bad magic, not a ") + std::string(expect, 4) + " file");
    uint32_t version = 0;
    IO_TRY(r.pod(version));
    if (version != kVersion)
        return io_fail(r.path, "unsupported version " + std::to_string(version));
    return PD_OK;
}

// read_section_payload (io.cpp:383-393): the declared length must match
int payload(Reader& r, void* dst, uint64_t expected_bytes) {
    uint64_t len = 0;
    IO_TRY(r.pod(len));
    if (len != expected_bytes)
        return io_fail(r.path, "section length " + std::to_string(len) +
                                   " does not match expected " + std::to_string(expected_bytes) +
                                   " bytes");
    return dst ? r.bytes(dst, len) : r.skip(len);
}

bool pow2(uint64_t v) { return v && !(v & (v - 1)); }

// NeighborList::validate (types.cpp:23-48)
int validate_rows(const int32_t* entries, const int32_t* n_neigh, const int32_t* initial, int64_t n,
                  int64_t N) {
    if (N < 1 || !pow2(uint64_t(N)))
        return set_error(PD_E_INVALID_ARGUMENT, "NeighborList: group size must be a power of two");
    if (!initial && n > 0)
        return set_error(PD_E_INVALID_ARGUMENT, "NeighborList: initial counts missing");
    for (int64_t i = 0; i < n; ++i) {
        int32_t live = 0;
        for (int64_t k = 0; k < N; ++k) {
            const int32_t j = entries[i * N + k];
            if (j == -1)
                continue;
            if (j < 0 || j >= n) {
                const std::string m = "NeighborList: entry out of range in row " + std::to_string(i);
                return set_error(PD_E_INVALID_ARGUMENT, m.c_str());
            }
            if (j == i) {
                const std::string m =
                    "NeighborList: node " + std::to_string(i) + " bonded to itself";
                return set_error(PD_E_INVALID_ARGUMENT, m.c_str());
            }
            ++live;
        }
        if (live != n_neigh[i]) {
            const std::string m = "NeighborList: count mismatch in row " + std::to_string(i);
            return set_error(PD_E_INVALID_ARGUMENT, m.c_str());
        }
    }
    return PD_OK;
}

} // namespace

// ---- writer -----------------------------------------------------------------

int StreamWriter::open(const char* p) {
    path = p;
    f = std::fopen(p, "wb");
    if (!f)
        return io_fail(path, "cannot open for writing");
    return PD_OK;
}

StreamWriter::~StreamWriter() {
    if (bounce)
        cudaFreeHost(bounce);
    if (f)
        std::fclose(f);
}

int StreamWriter::bytes(const void* data, uint64_t len) {
    if (len && std::fwrite(data, 1, size_t(len), f) != size_t(len))
        failed = true;
    return PD_OK;
}

int StreamWriter::section_host(uint32_t id, const void* data, uint64_t len) {
    pod(id);
    pod(len);
    return bytes(data, len);
}

int StreamWriter::section_device(uint32_t id, const void* dev, uint64_t len, cudaStream_t s) {
    pod(id);
    pod(len);
    // through a pinned chunk: D2H then fwrite (the disk is the bottleneck)
    constexpr uint64_t kChunk = uint64_t(32) << 20;
    if (!bounce) {
        if (cudaHostAlloc(&bounce, kChunk, cudaHostAllocDefault) != cudaSuccess) {
            bounce = nullptr;
            return set_error(PD_E_CUDA, "pinned staging allocation failed");
        }
    }
    for (uint64_t off = 0; off < len; off += kChunk) {
        const uint64_t n = std::min(kChunk, len - off);
        if (cudaMemcpyAsync(bounce, static_cast<const char*>(dev) + off, size_t(n),
                            cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess)
            return set_error(PD_E_CUDA, "device read for the state file failed");
        bytes(bounce, n);
    }
    return PD_OK;
}

int StreamWriter::close() {
    if (bounce)
        cudaFreeHost(bounce);
    bounce = nullptr;
    const bool bad = failed || std::fflush(f) != 0 || std::ferror(f);
    std::fclose(f);
    f = nullptr;
    if (bad)
        return io_fail(path, "write failed");
    return PD_OK;
}

} // namespace pdb

using namespace pdb;

extern "C" {

// save_state (io.cpp:485-505)
int pd_save_state(const pd_state* st, const char* path) {
    const pd_neighbor_list& c = st->connectivity;
    IO_TRY(validate_rows(c.entries, c.n_neigh, c.initial_n_neigh, c.n, c.group_size));
    if (c.bond_type_size != 0 && c.bond_type_size != c.n * c.group_size)
        return set_error(PD_E_INVALID_ARGUMENT, "NeighborList: bond_type size mismatch");
    StreamWriter w;
    IO_TRY(w.open(path));
    const uint64_t n = uint64_t(c.n), N = uint64_t(c.group_size);
    w.bytes("PDST", 4);
    w.pod(kVersion);
    w.pod(n);
    w.pod(N);
    w.pod(uint64_t(st->step));
    w.pod(double(c.horizon));
    w.section_host(sec_u, st->u, 8 * 3 * n);
    w.section_host(sec_v, st->v, 8 * 3 * n);
    w.section_host(sec_a, st->a, 8 * 3 * n);
    w.section_host(sec_entries, c.entries, 4 * n * N);
    w.section_host(sec_n_neigh, c.n_neigh, 4 * n);
    w.section_host(sec_initial_n_neigh, c.initial_n_neigh, 4 * n);
    if (c.bond_type_size)
        w.section_host(sec_bond_type, c.bond_type, n * N);
    if (st->bond_history && st->bond_history_size)
        w.section_host(sec_history, st->bond_history, 8 * uint64_t(st->bond_history_size));
    IO_TRY(w.close());
    return set_error(PD_OK, "");
}

int pd_state_file_header(const char* path, pd_file_header* out) {
    std::memset(out, 0, sizeof *out);
    Reader r;
    IO_TRY(r.open(path));
    IO_TRY(check_magic(r, "PDST"));
    uint64_t n = 0, N = 0, step = 0;
    double horizon = 0;
    IO_TRY(r.pod(n));
    IO_TRY(r.pod(N));
    IO_TRY(r.pod(step));
    IO_TRY(r.pod(horizon));
    if (n == 0 || N == 0 || !pow2(N))
        return io_fail(r.path, "corrupt header");
    out->n = int64_t(n);
    out->group_size = int64_t(N);
    out->step = int64_t(step);
    out->horizon = horizon;
    // the same sequential checks load_state makes (io.cpp:521-557), so a bad
    // file fails here with the reference's message
    const uint64_t slots = n * N;
    while (r.remaining) {
        uint32_t id = 0;
        IO_TRY(r.pod(id));
        uint64_t expect = 0;
        switch (id) {
        case sec_u: case sec_v: case sec_a: expect = 24 * n; break;
        case sec_entries: expect = 4 * slots; break;
        case sec_n_neigh: case sec_initial_n_neigh: expect = 4 * n; break;
        case sec_bond_type: expect = slots; out->has_bond_type = 1; break;
        case sec_history: expect = 8 * slots; out->has_history = 1; break;
        default: return io_fail(r.path, "unknown section id " + std::to_string(id));
        }
        IO_TRY(payload(r, nullptr, expect));
    }
    return set_error(PD_OK, "");
}

// load_state (io.cpp:507-562) into caller arrays sized from pd_state_file_header
int pd_load_state(const char* path, pd_state* st) {
    Reader r;
    IO_TRY(r.open(path));
    IO_TRY(check_magic(r, "PDST"));
    uint64_t n = 0, N = 0, step = 0;
    double horizon = 0;
    IO_TRY(r.pod(n));
    IO_TRY(r.pod(N));
    IO_TRY(r.pod(step));
    IO_TRY(r.pod(horizon));
    if (n == 0 || N == 0 || !pow2(N))
        return io_fail(r.path, "corrupt header");
    pd_neighbor_list& c = st->connectivity;
    if (uint64_t(c.n) != n || uint64_t(c.group_size) != N)
        return set_error(PD_E_INVALID_ARGUMENT, "load_state: arrays do not match the file");
    const uint64_t slots = n * N;
    int required = 0;
    while (r.remaining) {
        uint32_t id = 0;
        IO_TRY(r.pod(id));
        switch (id) {
        case sec_u: IO_TRY(payload(r, st->u, 8 * 3 * n)); ++required; break;
        case sec_v: IO_TRY(payload(r, st->v, 8 * 3 * n)); ++required; break;
        case sec_a: IO_TRY(payload(r, st->a, 8 * 3 * n)); ++required; break;
        case sec_entries: IO_TRY(payload(r, c.entries, 4 * slots)); ++required; break;
        case sec_n_neigh: IO_TRY(payload(r, c.n_neigh, 4 * n)); ++required; break;
        case sec_initial_n_neigh:
            IO_TRY(payload(r, const_cast<int32_t*>(c.initial_n_neigh), 4 * n));
            ++required;
            break;
        case sec_bond_type:
            IO_TRY(payload(r, c.bond_type_size ? const_cast<uint8_t*>(c.bond_type) : nullptr,
                           slots));
            break;
        case sec_history:
            IO_TRY(payload(r, st->bond_history_size ? st->bond_history : nullptr, 8 * slots));
            break;
        default: return io_fail(r.path, "unknown section id " + std::to_string(id));
        }
    }
    if (required != 6)
        return io_fail(r.path, "missing required sections");
    st->step = int64_t(step);
    c.horizon = horizon;
    IO_TRY(validate_rows(c.entries, c.n_neigh, c.initial_n_neigh, c.n, c.group_size));
    return set_error(PD_OK, "");
}

// save_cache (io.cpp:416-434)
int pd_save_cache(const pd_neighbor_list* c, const pd_corrections* corr, const char* path) {
    IO_TRY(validate_rows(c->entries, c->n_neigh, c->initial_n_neigh, c->n, c->group_size));
    StreamWriter w;
    IO_TRY(w.open(path));
    const uint64_t n = uint64_t(c->n), N = uint64_t(c->group_size);
    w.bytes("PDNL", 4);
    w.pod(kVersion);
    w.pod(n);
    w.pod(N);
    w.pod(double(c->horizon));
    w.section_host(sec_entries, c->entries, 4 * n * N);
    w.section_host(sec_n_neigh, c->n_neigh, 4 * n);
    w.section_host(sec_initial_n_neigh, c->initial_n_neigh, 4 * n);
    if (c->bond_type_size)
        w.section_host(sec_bond_type, c->bond_type, n * N);
    if (corr && corr->lambda_size)
        w.section_host(sec_lambda, corr->lambda, 8 * uint64_t(corr->lambda_size));
    if (corr && corr->beta_size)
        w.section_host(sec_beta, corr->beta, 8 * uint64_t(corr->beta_size));
    IO_TRY(w.close());
    return set_error(PD_OK, "");
}

int pd_cache_file_header(const char* path, pd_file_header* out) {
    std::memset(out, 0, sizeof *out);
    Reader r;
    IO_TRY(r.open(path));
    IO_TRY(check_magic(r, "PDNL"));
    uint64_t n = 0, N = 0;
    double horizon = 0;
    IO_TRY(r.pod(n));
    IO_TRY(r.pod(N));
    IO_TRY(r.pod(horizon));
    if (n == 0 || N == 0 || !pow2(N))
        return io_fail(r.path, "corrupt header");
    out->n = int64_t(n);
    out->group_size = int64_t(N);
    out->horizon = horizon;
    const uint64_t slots = n * N;
    while (r.remaining) {
        uint32_t id = 0;
        IO_TRY(r.pod(id));
        uint64_t expect = 0;
        switch (id) {
        case sec_entries: expect = 4 * slots; break;
        case sec_n_neigh: case sec_initial_n_neigh: expect = 4 * n; break;
        case sec_bond_type: expect = slots; out->has_bond_type = 1; break;
        case sec_lambda: expect = 8 * slots; out->has_lambda = 1; break;
        case sec_beta: expect = 8 * slots; out->has_beta = 1; break;
        default: return io_fail(r.path, "unknown section id " + std::to_string(id));
        }
        IO_TRY(payload(r, nullptr, expect));
    }
    return set_error(PD_OK, "");
}

// load_cache (io.cpp:436-483)
int pd_load_cache(const char* path, pd_neighbor_list* c, pd_corrections* corr) {
    Reader r;
    IO_TRY(r.open(path));
    IO_TRY(check_magic(r, "PDNL"));
    uint64_t n = 0, N = 0;
    double horizon = 0;
    IO_TRY(r.pod(n));
    IO_TRY(r.pod(N));
    IO_TRY(r.pod(horizon));
    if (n == 0 || N == 0 || !pow2(N))
        return io_fail(r.path, "corrupt header");
    if (uint64_t(c->n) != n || uint64_t(c->group_size) != N)
        return set_error(PD_E_INVALID_ARGUMENT, "load_cache: arrays do not match the file");
    const uint64_t slots = n * N;
    bool have_entries = false, have_counts = false, have_initial = false;
    while (r.remaining) {
        uint32_t id = 0;
        IO_TRY(r.pod(id));
        switch (id) {
        case sec_entries: IO_TRY(payload(r, c->entries, 4 * slots)); have_entries = true; break;
        case sec_n_neigh: IO_TRY(payload(r, c->n_neigh, 4 * n)); have_counts = true; break;
        case sec_initial_n_neigh:
            IO_TRY(payload(r, const_cast<int32_t*>(c->initial_n_neigh), 4 * n));
            have_initial = true;
            break;
        case sec_bond_type:
            IO_TRY(payload(r, c->bond_type_size ? const_cast<uint8_t*>(c->bond_type) : nullptr,
                           slots));
            break;
        case sec_lambda:
            IO_TRY(payload(r, corr && corr->lambda_size ? const_cast<double*>(corr->lambda)
                                                        : nullptr,
                           8 * slots));
            break;
        case sec_beta:
            IO_TRY(payload(r, corr && corr->beta_size ? const_cast<double*>(corr->beta) : nullptr,
                           8 * slots));
            break;
        default: return io_fail(r.path, "unknown section id " + std::to_string(id));
        }
    }
    if (!have_entries || !have_counts || !have_initial)
        return io_fail(r.path, "missing required sections");
    c->horizon = horizon;
    IO_TRY(validate_rows(c->entries, c->n_neigh, c->initial_n_neigh, c->n, c->group_size));
    return set_error(PD_OK, "");
}

} // extern "C"

// ---- ASCII snapshots (io.cpp:235-269) ---------------------------------------
//
//   pdsnap 1 <step>
//   <n>
//   x y z ux uy uz vx vy vz phi        "%.17g" each (format_real, io.cpp:16-20)
//
// The lines are formatted by several host threads into per-thread buffers and
// written in node order, so the bytes equal write_snapshot(make_snapshot(...)).

namespace pdb {

int write_snapshot_file(const char* path, int64_t step, int64_t n, const double* coords,
                        const double* u, const double* v, const double* phi) {
    FILE* f = std::fopen(path, "wb");
    if (!f) {
        const std::string m = std::string(path) + ": cannot open for writing (step " +
                              std::to_string(step) + ")";
        return set_error(PD_E_RUNTIME, m.c_str());
    }
    std::fprintf(f, "pdsnap 1 %lld\n%lld\n", (long long)step, (long long)n);
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const int64_t block = 1 << 16;  // nodes per formatting task
    const int64_t nblocks = (n + block - 1) / block;
    const int64_t threads = std::min<int64_t>(int64_t(std::min(16u, hw)), std::max<int64_t>(1, nblocks));
    bool bad = false;
    // rounds of `threads` blocks: format in parallel, write in order
    std::vector<std::string> out(static_cast<size_t>(threads));
    for (int64_t b0 = 0; b0 < nblocks && !bad; b0 += threads) {
        std::vector<std::thread> pool;
        for (int64_t t = 0; t < threads && b0 + t < nblocks; ++t)
            pool.emplace_back([&, t] {
                std::string& s = out[size_t(t)];
                s.clear();
                const int64_t i0 = (b0 + t) * block, i1 = std::min(n, i0 + block);
                s.reserve(size_t(i1 - i0) * 240);
                char buf[40];
                auto put = [&](double x, char sep) {
                    const int len = std::snprintf(buf, sizeof buf, "%.17g", x);
                    s.append(buf, size_t(len));
                    s.push_back(sep);
                };
                for (int64_t i = i0; i < i1; ++i) {
                    put(coords[3 * i], ' ');
                    put(coords[3 * i + 1], ' ');
                    put(coords[3 * i + 2], ' ');
                    put(u[3 * i], ' ');
                    put(u[3 * i + 1], ' ');
                    put(u[3 * i + 2], ' ');
                    put(v[3 * i], ' ');
                    put(v[3 * i + 1], ' ');
                    put(v[3 * i + 2], ' ');
                    put(phi[i], '\n');
                }
            });
        for (auto& th : pool)
            th.join();
        for (int64_t t = 0; t < threads && b0 + t < nblocks; ++t)
            if (std::fwrite(out[size_t(t)].data(), 1, out[size_t(t)].size(), f) !=
                out[size_t(t)].size())
                bad = true;
    }
    bad = bad || std::fflush(f) != 0 || std::ferror(f);
    std::fclose(f);
    if (bad) {
        const std::string m =
            std::string(path) + ": write failed (step " + std::to_string(step) + ")";
        return set_error(PD_E_RUNTIME, m.c_str());
    }
    return PD_OK;
}

} // namespace pdb

extern "C" int pd_write_snapshot(const pd_state* st, const pd_particles* p, const char* path) {
    const int64_t n = st->connectivity.n;
    if (p->n != n || p->coords_size != 3 * n)
        return set_error(PD_E_INVALID_ARGUMENT, "write_snapshot: particle set does not match state");
    std::vector<double> phi(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
        const int32_t init = st->connectivity.initial_n_neigh[i];
        const int32_t cur = st->connectivity.n_neigh[i];
        if (init > 0 && (cur < 0 || cur > init))
            return set_error(PD_E_DOMAIN, "local_damage: current count out of range");
        phi[size_t(i)] = init > 0 ? 1.0 - double(cur) / double(init) : 0.0;  // make_snapshot
    }
    const int rc = pdb::write_snapshot_file(path, st->step, n, p->coords, st->u, st->v, phi.data());
    return rc == PD_OK ? set_error(PD_OK, "") : rc;
}
