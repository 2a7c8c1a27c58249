// pd_layout.cu -- the fast path's tile layout (pd_fast.cuh), built on the device.
//
// Same result as the layout a host would build from the rows: nodes renumbered
// into spatial bricks (lattices) or along a Morton curve (other meshes), tiles
// of <= T consecutive internal nodes, per tile a halo of every node its rows
// touch (no-failure nodes last; ascending reference order on bricks, internal
// order on Morton tiles), and per live slot the index of the neighbour's
// shared-memory record.  All passes are sorts, scans and
// per-node kernels over data already resident for the step, so setting up a
// 10M-node model costs milliseconds instead of seconds of host work:
//
//   1. per axis: sort the coordinates, count distinct values (<= 4096: a
//      lattice axis on all three: bricks of 16 x 4 x T/64 grid planes; else
//      a Morton curve of mean-spacing cells); brick / Morton key per owned
//      node; stable radix sort of the owned nodes by key -> perm; run lengths
//      -> balanced tiles of <= T nodes (host, one value per brick; the Morton
//      curve is one run) -> perm / inv.  A warp's nodes stay spatial
//      neighbours, so its shared-memory reads of one slot hit nearby records
//      (ordering a tile's nodes by row length instead scattered them over the
//      banks: 20 % slower on a jittered lattice);
//   2. live count per row -> kmax8 per tile -> slot offsets (host scan of one
//      value per tile);
//   3. one 64-bit key (tile, no-failure flag, node) per live slot and per
//      owned node; radix sort + unique -> every tile's halo as a contiguous
//      sorted segment;
//   4. per owned node: binary-search each live neighbour in its tile's
//      segment -> 16-bit slot offsets; compact history / bond types /
//      corrections alongside.
#include <cuda_runtime.h>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_run_length_encode.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include <algorithm>
#include <cmath>
#include <vector>

#include "pd_device.cuh"
#include "pd_internal.h"

namespace pdb {
namespace {

constexpr int TPB = 256;

inline unsigned blocks_for(long long n) { return unsigned((n + TPB - 1) / TPB); }

#define LY_CK(expr)                                                                              \
    do {                                                                                         \
        cudaError_t e_ = (expr);                                                                 \
        if (e_ != cudaSuccess)                                                                   \
            return e_;                                                                           \
    } while (0)

// scratch allocation released at scope exit
struct Scratch {
    std::vector<void*> ptrs;
    ~Scratch() {
        for (void* p : ptrs)
            cudaFree(p);
    }
    template <class T> cudaError_t get(T** out, size_t count) {
        void* p = nullptr;
        cudaError_t e = cudaMalloc(&p, std::max<size_t>(1, count) * sizeof(T));
        if (e == cudaSuccess)
            ptrs.push_back(p);
        *out = static_cast<T*>(p);
        return e;
    }
};

__global__ void axis_kernel(const double4* xv, long long n, int axis, double* out) {
    const long long i = blockIdx.x * (long long)TPB + threadIdx.x;
    if (i < n) {
        const double4 x = xv[i];
        out[i] = axis == 0 ? x.x : (axis == 1 ? x.y : x.z);
    }
}

struct BrickGrid {
    int lattice[3];
    const double* uniq[3];  // sorted distinct values of a lattice axis
    int n_uniq[3];
    long long kbrick[3];
    double lo[3], len[3];
    long long nb[3];
    int morton;      // not a lattice on every axis: Morton order of h-cells
    double inv_h;
};

__device__ __forceinline__ unsigned long long spread3(unsigned long long v) {  // 21 bits -> 63
    v &= 0x1fffffull;
    v = (v | v << 32) & 0x1f00000000ffffull;
    v = (v | v << 16) & 0x1f0000ff0000ffull;
    v = (v | v << 8) & 0x100f00f00f00f00full;
    v = (v | v << 4) & 0x10c30c30c30c30c3ull;
    v = (v | v << 2) & 0x1249249249249249ull;
    return v;
}

__device__ __forceinline__ long long lower_bound_d(const double* a, int n, double v) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] < v)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

__global__ void brick_key_kernel(const double4* xv, long long begin, long long count, BrickGrid g,
                                 unsigned long long* keys, int* vals) {
    const long long k = blockIdx.x * (long long)TPB + threadIdx.x;
    if (k >= count)
        return;
    const long long i = begin + k;
    const double4 x = xv[i];
    const double c3[3] = {x.x, x.y, x.z};
    if (g.morton) {
        unsigned long long key = 0;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            const double q = floor((c3[d] - g.lo[d]) * g.inv_h);
            const unsigned long long c = q < 0 ? 0ull : (q > 2097151.0 ? 2097151ull
                                                                        : (unsigned long long)q);
            key |= spread3(c) << d;
        }
        keys[k] = key;
        vals[k] = int(i);
        return;
    }
    long long b[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        long long c;
        if (g.lattice[d])
            c = lower_bound_d(g.uniq[d], g.n_uniq[d], c3[d]) / g.kbrick[d];
        else
            c = g.len[d] > 0 ? (long long)floor((c3[d] - g.lo[d]) / g.len[d]) : 0;
        b[d] = c < 0 ? 0 : (c > g.nb[d] - 1 ? g.nb[d] - 1 : c);
    }
    keys[k] = (unsigned long long)((b[2] * g.nb[1] + b[1]) * g.nb[0] + b[0]);
    vals[k] = int(i);
}

// lexicographic key of a node's mean-spacing cell (z, y, x): the order a
// lattice's reference numbering has, computed from the coordinates so Morton
// tiles get it whatever the input numbering
__global__ void lex_key_kernel(const double4* xv, long long n, BrickGrid g,
                               unsigned long long* keys, int* vals) {
    const long long i = blockIdx.x * (long long)TPB + threadIdx.x;
    if (i >= n)
        return;
    const double4 x = xv[i];
    const double c3[3] = {x.x, x.y, x.z};
    unsigned long long q[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const double v = floor((c3[d] - g.lo[d]) * g.inv_h);
        q[d] = v < 0 ? 0ull : (v > 2097151.0 ? 2097151ull : (unsigned long long)v);
    }
    keys[i] = (q[2] << 42) | (q[1] << 21) | q[0];
    vals[i] = int(i);
}

__global__ void rank_kernel(const int* sorted_ids, long long n, int* rank) {
    const long long r = blockIdx.x * (long long)TPB + threadIdx.x;
    if (r < n)
        rank[sorted_ids[r]] = int(r);
}

__global__ void tile_lex_key_kernel(const int* perm, const int* tile_of, const int* lexrank,
                                    long long n_own, unsigned long long* keys) {
    const long long ii = blockIdx.x * (long long)TPB + threadIdx.x;
    if (ii < n_own)
        keys[ii] = ((unsigned long long)tile_of[ii] << 32) | (unsigned)lexrank[perm[ii]];
}

__global__ void compose_kernel(const int* inv, const int* sorted_ids, long long n, int* out) {
    const long long r = blockIdx.x * (long long)TPB + threadIdx.x;
    if (r < n)
        out[r] = inv[sorted_ids[r]];
}

// perm[n_own + k] = k-th ghost (local order); inv = perm^-1
__global__ void perm_tail_kernel(int* perm, long long n, long long own_begin, long long own_end) {
    const long long k = blockIdx.x * (long long)TPB + threadIdx.x;
    const long long n_own = own_end - own_begin;
    if (k >= n - n_own)
        return;
    perm[n_own + k] = int(k < own_begin ? k : k - own_begin + own_end);
}

__global__ void inv_kernel(const int* perm, long long n, int* inv) {
    const long long ii = blockIdx.x * (long long)TPB + threadIdx.x;
    if (ii < n)
        inv[perm[ii]] = int(ii);
}

__global__ void tile_of_kernel(const int* tile_start, int n_tiles, int* tile_of) {
    const int t = blockIdx.x;
    if (t >= n_tiles)
        return;
    for (int ii = tile_start[t] + threadIdx.x; ii < tile_start[t + 1]; ii += blockDim.x)
        tile_of[ii] = t;
}

__global__ void live_kernel(const int32_t* entries, const int* perm, const int* tile_of,
                            long long n_own, int N, int* live, int* kmax) {
    const long long ii = blockIdx.x * (long long)TPB + threadIdx.x;
    if (ii >= n_own)
        return;
    const long long i = perm[ii];
    int c = 0;
    for (int k = 0; k < N; ++k)
        c += entries[i * N + k] >= 0;
    live[ii] = c + 1;  // + the node itself (pair keys)
    atomicMax(kmax + tile_of[ii], c);
}

// halo key of node j (reference id) in tile `tile`: a tile's halo is sorted by
// (no-failure flag, order id) so that the records a warp's neighbours read at
// one slot sit close together, as the warp's own nodes do (few bank
// conflicts): the reference id on lattice bricks (x-fastest runs), the
// internal (Morton) id on irregular meshes (inv != NULL)
__device__ __forceinline__ unsigned long long pair_key(int tile, const uint8_t* nofail,
                                                       const int* inv, int j) {
    const unsigned long long nf = (nofail && nofail[j]) ? 1ull : 0ull;
    const unsigned o = unsigned(inv ? inv[j] : j);
    return ((unsigned long long)tile << 33) | (nf << 32) | (unsigned long long)o;
}

__global__ void pair_keys_kernel(const int32_t* entries, const int* perm, const int* inv,
                                 const int* tile_of,
                                 const uint8_t* nofail, const long long* off, long long n_own,
                                 int N, unsigned long long* keys) {
    const long long ii = blockIdx.x * (long long)TPB + threadIdx.x;
    if (ii >= n_own)
        return;
    const long long i = perm[ii];
    const int t = tile_of[ii];
    long long o = off[ii];
    keys[o++] = pair_key(t, nofail, inv, int(i));
    for (int k = 0; k < N; ++k) {
        const int32_t j = entries[i * N + k];
        if (j >= 0)
            keys[o++] = pair_key(t, nofail, inv, j);
    }
}

// halo_off[t] = first key of tile t; halo[k] = internal id of the key's node
__global__ void halo_kernel(const unsigned long long* hk, long long H, const int* inv,
                            long long* halo_off, int* halo) {
    const long long k = blockIdx.x * (long long)TPB + threadIdx.x;
    if (k >= H)
        return;
    const unsigned long long key = hk[k];
    const int t = int(key >> 33);
    if (k == 0 || int(hk[k - 1] >> 33) != t)
        halo_off[t] = k;
    const int o = int(unsigned(key & 0xffffffffull));
    halo[k] = inv ? inv[o] : o;
}

// nf_start[t] = position of the first no-failure key + 1 (its shared-memory
// record index), found per key
__global__ void nf_start_kernel(const unsigned long long* hk, long long H, const long long* halo_off,
                                int* nf_start) {
    const long long k = blockIdx.x * (long long)TPB + threadIdx.x;
    if (k >= H)
        return;
    const unsigned long long key = hk[k];
    if (!((key >> 32) & 1ull))
        return;
    const int t = int(key >> 33);
    const bool first = k == halo_off[t] || !((hk[k - 1] >> 32) & 1ull);
    if (first)
        nf_start[t] = int(k - halo_off[t] + 1);
}

__device__ __forceinline__ long long lower_bound_u64(const unsigned long long* a, long long lo,
                                                     long long hi, unsigned long long v) {
    while (lo < hi) {
        const long long mid = (lo + hi) >> 1;
        if (a[mid] < v)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

struct SlotArgs {
    const int32_t* entries;
    const int* perm;
    const int* inv;
    const int* tile_of;
    const int* tile_start;
    const long long* slot_off;
    const long long* halo_off;
    const unsigned long long* hk;
    const uint8_t* nofail;
    const double* hist;
    const uint8_t* btype;
    const double* lambda;
    const double* beta;
    long long n_own;
    int N, T;
    unsigned short* lidx;
    unsigned short* own_slot;
    unsigned short* origk;
    int* wgroups;
    float* hist32;
    uint8_t* btype_c;
    float* lambda32;
    float* beta32;
};

__global__ void slot_kernel(SlotArgs S) {
    const long long ii = blockIdx.x * (long long)TPB + threadIdx.x;
    if (ii >= S.n_own)
        return;
    const long long i = S.perm[ii];
    const int t = S.tile_of[ii];
    const long long h0 = S.halo_off[t], h1 = S.halo_off[t + 1];
    const long long base = S.slot_off[t] + (long long)(ii - S.tile_start[t]) * 8;
    const long long own = lower_bound_u64(S.hk, h0, h1, pair_key(t, S.nofail, S.inv, int(i))) - h0;
    const bool nfi = S.nofail && S.nofail[i];
    S.own_slot[ii] = (unsigned short)((own + 1) | (nfi ? 0x8000 : 0));
    int c = 0;
    for (int k = 0; k < S.N; ++k) {
        const long long idx = i * S.N + k;
        const int32_t j = S.entries[idx];
        if (j < 0)
            continue;
        const long long pos = lower_bound_u64(S.hk, h0, h1, pair_key(t, S.nofail, S.inv, j)) - h0;
        const long long s = base + (long long)(c >> 3) * S.T * 8 + (c & 7);
        S.lidx[s] = (unsigned short)(pos + 1);
        if (S.origk)
            S.origk[s] = (unsigned short)k;
        if (S.hist32)
            S.hist32[s] = S.hist ? float(S.hist[idx]) : 0.f;
        if (S.btype_c)
            S.btype_c[s] = S.btype[idx];
        if (S.lambda32)
            S.lambda32[s] = float(S.lambda[idx]);
        if (S.beta32)
            S.beta32[s] = float(S.beta[idx]);
        ++c;
    }
    // per warp of tile threads: the 8-slot groups its longest row needs
    if (c > 0)
        atomicMax(S.wgroups + (long long)t * (S.T / 32) + (ii - S.tile_start[t]) / 32, (c + 7) / 8);
}

// Morton tiles: each node's compact slots re-ordered by halo record index, so
// that at one slot the 32 lanes of a warp (Morton-consecutive nodes) read
// records that sit close together in shared memory -- rows in the reference
// order against a Morton-ordered halo scatter them over the banks (2x the
// shared-memory wavefronts on a jittered lattice).  One warp per node: keys
// (record << 10 | compact slot) bitonic-sorted in shared memory, then every
// per-slot array gathered from a copy of the unsorted layout.
struct SortArgs {
    const int* live;  // compact row length + 1, per owned node (internal order)
    const int* tile_of;
    const int* tile_start;
    const long long* slot_off;
    long long n_own;
    int T;
    const unsigned short *lidx0, *origk0;
    const float *hist0, *lambda0, *beta0;
    const uint8_t* btype0;
    unsigned short *lidx, *origk;
    float *hist, *lambda, *beta;
    uint8_t* btype;
};

constexpr int SORT_WARPS = 4;
constexpr int SORT_MAX = 1024;

__global__ void __launch_bounds__(SORT_WARPS * 32) sort_rows_kernel(SortArgs S) {
    __shared__ unsigned keys[SORT_WARPS][SORT_MAX];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long ii = blockIdx.x * (long long)SORT_WARPS + w;
    if (ii >= S.n_own)
        return;
    const int L = S.live[ii] - 1;
    if (L <= 1)
        return;
    const int t = S.tile_of[ii];
    const long long base = S.slot_off[t] + (long long)(ii - S.tile_start[t]) * 8;
    auto slot = [&](int c) { return base + (long long)(c >> 3) * S.T * 8 + (c & 7); };
    int P = 32;
    while (P < L)
        P <<= 1;
    unsigned* k = keys[w];
    for (int c = lane; c < P; c += 32)
        k[c] = c < L ? (unsigned(S.lidx0[slot(c)]) << 10) | unsigned(c) : 0xffffffffu;
    __syncwarp();
    for (int size = 2; size <= P; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int c = lane; c < P; c += 32) {
                const int o = c ^ stride;
                if (o > c) {
                    const bool up = (c & size) == 0;
                    const unsigned a = k[c], b = k[o];
                    if ((a > b) == up) {
                        k[c] = b;
                        k[o] = a;
                    }
                }
            }
            __syncwarp();
        }
    for (int r = lane; r < L; r += 32) {
        const int c = int(k[r] & 1023u);
        const long long sn = slot(r), so = slot(c);
        S.lidx[sn] = S.lidx0[so];
        S.origk[sn] = S.origk0[so];
        if (S.hist)
            S.hist[sn] = S.hist0[so];
        if (S.btype)
            S.btype[sn] = S.btype0[so];
        if (S.lambda)
            S.lambda[sn] = S.lambda0[so];
        if (S.beta)
            S.beta[sn] = S.beta0[so];
    }
}

template <class T> __global__ void fill_kernel(T* p, long long n, T v) {
    const long long k = blockIdx.x * (long long)TPB + threadIdx.x;
    if (k < n)
        p[k] = v;
}

template <class T> cudaError_t fill(T* p, long long n, T v, cudaStream_t s) {
    if (n > 0)
        fill_kernel<T><<<blocks_for(n), TPB, 0, s>>>(p, n, v);
    return cudaGetLastError();
}

int bits_for(unsigned long long v) {
    int b = 0;
    while (b < 64 && (v >> b) != 0)
        ++b;
    return std::max(b, 1);
}

} // namespace

cudaError_t gpu_build_layout(FastLayoutDev& L, const FastLayoutIn& in, int* error,
                             cudaStream_t s) {
    *error = 0;
    const long long n = in.n, ob = in.own_begin, oe = in.own_end, n_own = oe - ob;
    const int N = in.N, T = in.T;
    Scratch tmp;
    void* cub_tmp = nullptr;
    size_t cub_bytes = 0;
    auto cub_reserve = [&](size_t need) -> cudaError_t {
        if (need <= cub_bytes)
            return cudaSuccess;
        if (cub_tmp)
            cudaFree(cub_tmp);
        cub_tmp = nullptr;
        cub_bytes = need;
        return cudaMalloc(&cub_tmp, need);
    };
    struct CubFree {
        void** p;
        ~CubFree() {
            if (*p)
                cudaFree(*p);
        }
    } cub_free{&cub_tmp};

    // ---- 1. bricks -------------------------------------------------------
    BrickGrid g{};
    const long long kBrick[3] = {16, 4, T / 64};
    double lo[3], hi[3];
    std::vector<double> uniq_host[3];
    {
        double *ax, *ax_sorted, *uniq;
        int* n_uniq_d;
        LY_CK(tmp.get(&ax, size_t(n)));
        LY_CK(tmp.get(&ax_sorted, size_t(n)));
        LY_CK(tmp.get(&n_uniq_d, 1));
        for (int d = 0; d < 3; ++d) {
            axis_kernel<<<blocks_for(n), TPB, 0, s>>>(in.xv, n, d, ax);
            size_t need = 0;
            LY_CK(cub::DeviceRadixSort::SortKeys(nullptr, need, ax, ax_sorted, int(n), 0, 64, s));
            LY_CK(cub_reserve(need));
            LY_CK(cub::DeviceRadixSort::SortKeys(cub_tmp, cub_bytes, ax, ax_sorted, int(n), 0, 64,
                                                 s));
            LY_CK(cudaMemcpyAsync(&lo[d], ax_sorted, sizeof(double), cudaMemcpyDeviceToHost, s));
            LY_CK(cudaMemcpyAsync(&hi[d], ax_sorted + n - 1, sizeof(double), cudaMemcpyDeviceToHost,
                                  s));
            LY_CK(tmp.get(&uniq, size_t(n)));
            need = 0;
            LY_CK(cub::DeviceSelect::Unique(nullptr, need, ax_sorted, uniq, n_uniq_d, int(n), s));
            LY_CK(cub_reserve(need));
            LY_CK(cub::DeviceSelect::Unique(cub_tmp, cub_bytes, ax_sorted, uniq, n_uniq_d, int(n),
                                            s));
            int nu = 0;
            LY_CK(cudaMemcpyAsync(&nu, n_uniq_d, sizeof(int), cudaMemcpyDeviceToHost, s));
            LY_CK(cudaStreamSynchronize(s));
            g.lattice[d] = nu <= 4096;
            g.uniq[d] = uniq;
            g.n_uniq[d] = nu;
        }
    }
    double ext[3], prod = 1.0;
    int dims = 0;
    for (int d = 0; d < 3; ++d) {
        ext[d] = hi[d] - lo[d];
        if (ext[d] > 0) {
            prod *= ext[d];
            ++dims;
        }
    }
    const double h = dims == 0 ? 1.0 : std::pow(prod / double(n), 1.0 / dims);
    for (int d = 0; d < 3; ++d) {
        g.kbrick[d] = kBrick[d];
        g.lo[d] = lo[d];
        if (g.lattice[d]) {
            g.nb[d] = (g.n_uniq[d] + kBrick[d] - 1) / kBrick[d];
            g.len[d] = 1.0;
        } else {
            g.nb[d] = 1;
            g.len[d] = ext[d] > 0 ? ext[d] / double(g.nb[d]) : 1.0;
        }
    }
    // irregular meshes: tiles are runs of T nodes along a Morton curve of
    // mean-spacing cells (compact, nearly cubic, all but the last full)
    g.morton = !(g.lattice[0] && g.lattice[1] && g.lattice[2]);
    g.inv_h = 1.0 / h;
    const unsigned long long nbricks = (unsigned long long)(g.nb[0] * g.nb[1] * g.nb[2]);
    LY_CK(L.perm.alloc(size_t(n)));
    LY_CK(L.inv.alloc(size_t(n)));
    std::vector<int> tile_start;
    if (n_own > 0) {
        unsigned long long *keys, *keys_sorted, *rle_keys;
        int *vals, *rle_counts, *n_runs_d;
        LY_CK(tmp.get(&keys, size_t(n_own)));
        LY_CK(tmp.get(&keys_sorted, size_t(n_own)));
        LY_CK(tmp.get(&vals, size_t(n_own)));
        brick_key_kernel<<<blocks_for(n_own), TPB, 0, s>>>(in.xv, ob, n_own, g, keys, vals);
        LY_CK(cudaGetLastError());
        const int kb = g.morton ? 63 : bits_for(nbricks);
        size_t need = 0;
        LY_CK(cub::DeviceRadixSort::SortPairs(nullptr, need, keys, keys_sorted, vals, L.perm.p,
                                              int(n_own), 0, kb, s));
        LY_CK(cub_reserve(need));
        LY_CK(cub::DeviceRadixSort::SortPairs(cub_tmp, cub_bytes, keys, keys_sorted, vals, L.perm.p,
                                              int(n_own), 0, kb, s));
        LY_CK(tmp.get(&rle_keys, size_t(n_own)));
        LY_CK(tmp.get(&rle_counts, size_t(n_own)));
        LY_CK(tmp.get(&n_runs_d, 1));
        need = 0;
        LY_CK(cub::DeviceRunLengthEncode::Encode(nullptr, need, keys_sorted, rle_keys, rle_counts,
                                                 n_runs_d, int(n_own), s));
        LY_CK(cub_reserve(need));
        LY_CK(cub::DeviceRunLengthEncode::Encode(cub_tmp, cub_bytes, keys_sorted, rle_keys,
                                                 rle_counts, n_runs_d, int(n_own), s));
        int runs = 0;
        LY_CK(cudaMemcpyAsync(&runs, n_runs_d, sizeof(int), cudaMemcpyDeviceToHost, s));
        LY_CK(cudaStreamSynchronize(s));
        std::vector<int> counts(static_cast<size_t>(runs));
        LY_CK(cudaMemcpyAsync(counts.data(), rle_counts, sizeof(int) * size_t(runs),
                              cudaMemcpyDeviceToHost, s));
        LY_CK(cudaStreamSynchronize(s));
        if (g.morton)  // one run: the whole curve is cut into T-node pieces
            counts.assign(1, int(n_own));
        // a brick of c nodes becomes ceil(c / T) tiles of balanced size (a
        // 530-node bin is two 265-node tiles, not 512 + 18)
        long long at = 0;
        for (int c : counts) {
            const long long nt = (c + T - 1) / T;
            for (long long q = 0; q < nt; ++q)
                tile_start.push_back(int(at + q * c / nt));
            at += c;
        }
    }
    tile_start.push_back(int(n_own));
    const int tiles = int(tile_start.size()) - 1;
    L.T = T;
    L.n_tiles = tiles;
    LY_CK(L.tile_start.upload(tile_start.data(), tile_start.size(), s));
    LY_CK(L.tile_of.alloc(size_t(n)));
    LY_CK(cudaMemsetAsync(L.tile_of.p, 0xff, sizeof(int) * size_t(n), s));
    if (tiles > 0)
        tile_of_kernel<<<unsigned(tiles), TPB, 0, s>>>(L.tile_start.p, tiles, L.tile_of.p);
    // Morton tiles: order each tile's nodes, and every halo, lexicographically
    // by mean-spacing cell (lexrank), as a lattice's reference numbering is,
    // so a warp's nodes are x-runs and the records its lanes read at one slot
    // sit side by side in shared memory (rows are then sorted by record,
    // sort_rows_kernel)
    int *lexrank = nullptr, *lex_ids = nullptr, *lex_to_internal = nullptr;
    if (g.morton && n > 0) {
        unsigned long long *lk, *lk_sorted;
        int* iota;
        LY_CK(tmp.get(&lk, size_t(n)));
        LY_CK(tmp.get(&lk_sorted, size_t(n)));
        LY_CK(tmp.get(&iota, size_t(n)));
        LY_CK(tmp.get(&lex_ids, size_t(n)));
        LY_CK(tmp.get(&lexrank, size_t(n)));
        LY_CK(tmp.get(&lex_to_internal, size_t(n)));
        lex_key_kernel<<<blocks_for(n), TPB, 0, s>>>(in.xv, n, g, lk, iota);
        size_t need = 0;
        LY_CK(cub::DeviceRadixSort::SortPairs(nullptr, need, lk, lk_sorted, iota, lex_ids, int(n),
                                              0, 63, s));
        LY_CK(cub_reserve(need));
        LY_CK(cub::DeviceRadixSort::SortPairs(cub_tmp, cub_bytes, lk, lk_sorted, iota, lex_ids,
                                              int(n), 0, 63, s));
        rank_kernel<<<blocks_for(n), TPB, 0, s>>>(lex_ids, n, lexrank);
        if (n_own > 0) {
            int* perm2;
            LY_CK(tmp.get(&perm2, size_t(n_own)));
            tile_lex_key_kernel<<<blocks_for(n_own), TPB, 0, s>>>(L.perm.p, L.tile_of.p, lexrank,
                                                                 n_own, lk);
            const int kb = 32 + bits_for((unsigned long long)std::max(tiles, 1));
            need = 0;
            LY_CK(cub::DeviceRadixSort::SortPairs(nullptr, need, lk, lk_sorted, L.perm.p, perm2,
                                                  int(n_own), 0, kb, s));
            LY_CK(cub_reserve(need));
            LY_CK(cub::DeviceRadixSort::SortPairs(cub_tmp, cub_bytes, lk, lk_sorted, L.perm.p,
                                                  perm2, int(n_own), 0, kb, s));
            LY_CK(cudaMemcpyAsync(L.perm.p, perm2, sizeof(int) * size_t(n_own),
                                  cudaMemcpyDeviceToDevice, s));
        }
    }
    if (n > n_own)
        perm_tail_kernel<<<blocks_for(n - n_own), TPB, 0, s>>>(L.perm.p, n, ob, oe);
    inv_kernel<<<blocks_for(n), TPB, 0, s>>>(L.perm.p, n, L.inv.p);
    if (g.morton && n > 0)
        compose_kernel<<<blocks_for(n), TPB, 0, s>>>(L.inv.p, lex_ids, n, lex_to_internal);
    LY_CK(cudaGetLastError());

    // halo order: reference ids on bricks, lexicographic cell rank on Morton tiles
    const int* halo_key_inv = g.morton ? lexrank : nullptr;            // key -> order id
    const int* halo_by_ref = g.morton ? lex_to_internal : L.inv.p;     // order id -> internal id

    // ---- 2. slot offsets -------------------------------------------------
    int *live, *kmax;
    long long* pair_off;
    LY_CK(tmp.get(&live, size_t(n_own)));
    LY_CK(tmp.get(&kmax, size_t(tiles)));
    LY_CK(tmp.get(&pair_off, size_t(n_own)));
    LY_CK(cudaMemsetAsync(kmax, 0, sizeof(int) * size_t(std::max(tiles, 1)), s));
    if (n_own > 0)
        live_kernel<<<blocks_for(n_own), TPB, 0, s>>>(in.entries, L.perm.p, L.tile_of.p, n_own, N,
                                                      live, kmax);
    LY_CK(cudaGetLastError());
    std::vector<int> kmax_h(static_cast<size_t>(tiles));
    LY_CK(cudaMemcpyAsync(kmax_h.data(), kmax, sizeof(int) * size_t(tiles), cudaMemcpyDeviceToHost,
                          s));
    {
        size_t need = 0;
        LY_CK(cub::DeviceScan::ExclusiveSum(nullptr, need, live, pair_off, int(n_own), s));
        LY_CK(cub_reserve(need));
        LY_CK(cub::DeviceScan::ExclusiveSum(cub_tmp, cub_bytes, live, pair_off, int(n_own), s));
    }
    long long last_off = 0;
    int last_live = 0;
    if (n_own > 0) {
        LY_CK(cudaMemcpyAsync(&last_off, pair_off + n_own - 1, sizeof(long long),
                              cudaMemcpyDeviceToHost, s));
        LY_CK(cudaMemcpyAsync(&last_live, live + n_own - 1, sizeof(int), cudaMemcpyDeviceToHost, s));
    }
    LY_CK(cudaStreamSynchronize(s));
    const long long n_pairs = last_off + last_live;
    std::vector<int> kmax8(static_cast<size_t>(tiles));
    std::vector<long long> slot_off(static_cast<size_t>(tiles));
    long long slots = 0;
    for (int t = 0; t < tiles; ++t) {
        kmax8[size_t(t)] = (kmax_h[size_t(t)] + 7) / 8 * 8;
        slot_off[size_t(t)] = slots;
        slots += (long long)kmax8[size_t(t)] * T;
    }
    L.total_slots = slots;
    LY_CK(L.kmax8.upload(kmax8.data(), kmax8.size(), s));
    LY_CK(L.slot_off.upload(slot_off.data(), slot_off.size(), s));

    // ---- 3. halos --------------------------------------------------------
    unsigned long long *pk, *pk_sorted, *hk;
    long long* n_uniq_d;
    LY_CK(tmp.get(&pk, size_t(n_pairs)));
    LY_CK(tmp.get(&pk_sorted, size_t(n_pairs)));
    LY_CK(tmp.get(&n_uniq_d, 1));
    if (n_own > 0)
        pair_keys_kernel<<<blocks_for(n_own), TPB, 0, s>>>(in.entries, L.perm.p, halo_key_inv, L.tile_of.p,
                                                           in.nofail, pair_off, n_own, N, pk);
    LY_CK(cudaGetLastError());
    const int key_bits = 33 + bits_for((unsigned long long)std::max(tiles, 1));
    {
        size_t need = 0;
        LY_CK(cub::DeviceRadixSort::SortKeys(nullptr, need, pk, pk_sorted, n_pairs, 0, key_bits,
                                             s));
        LY_CK(cub_reserve(need));
        LY_CK(cub::DeviceRadixSort::SortKeys(cub_tmp, cub_bytes, pk, pk_sorted, n_pairs, 0,
                                             key_bits, s));
    }
    hk = pk;  // the unsorted keys are dead: reuse their storage for the unique list
    {
        size_t need = 0;
        LY_CK(cub::DeviceSelect::Unique(nullptr, need, pk_sorted, hk, n_uniq_d, n_pairs, s));
        LY_CK(cub_reserve(need));
        LY_CK(cub::DeviceSelect::Unique(cub_tmp, cub_bytes, pk_sorted, hk, n_uniq_d, n_pairs, s));
    }
    long long H = 0;
    LY_CK(cudaMemcpyAsync(&H, n_uniq_d, sizeof(long long), cudaMemcpyDeviceToHost, s));
    LY_CK(cudaStreamSynchronize(s));
    LY_CK(L.halo_off.alloc(size_t(tiles + 1)));
    LY_CK(L.halo.alloc(size_t(std::max(H, 1LL))));
    LY_CK(L.nf_start.alloc(size_t(std::max(tiles, 1))));
    LY_CK(fill<int>(L.nf_start.p, tiles, 0x7fffffff, s));
    LY_CK(cudaMemcpyAsync(L.halo_off.p + tiles, &H, sizeof(long long), cudaMemcpyHostToDevice, s));
    if (H > 0) {
        halo_kernel<<<blocks_for(H), TPB, 0, s>>>(hk, H, halo_by_ref, L.halo_off.p, L.halo.p);
        nf_start_kernel<<<blocks_for(H), TPB, 0, s>>>(hk, H, L.halo_off.p, L.nf_start.p);
    }
    LY_CK(cudaGetLastError());
    std::vector<long long> halo_off(static_cast<size_t>(tiles + 1));
    LY_CK(cudaMemcpyAsync(halo_off.data(), L.halo_off.p, sizeof(long long) * size_t(tiles + 1),
                          cudaMemcpyDeviceToHost, s));
    LY_CK(cudaStreamSynchronize(s));
    L.max_halo = 0;
    for (int t = 0; t < tiles; ++t)
        L.max_halo = std::max(L.max_halo, int(halo_off[size_t(t + 1)] - halo_off[size_t(t)]));
    if (L.max_halo > FAST_MAX_HALO) {
        *error = 1;
        return cudaSuccess;
    }

    // ---- 4. slots --------------------------------------------------------
    LY_CK(L.lidx.alloc(size_t(std::max(slots, 1LL))));
    LY_CK(cudaMemsetAsync(L.lidx.p, 0, sizeof(unsigned short) * size_t(std::max(slots, 1LL)), s));
    LY_CK(L.own_slot.alloc(size_t(n)));
    LY_CK(cudaMemsetAsync(L.own_slot.p, 0, sizeof(unsigned short) * size_t(n), s));
    SlotArgs S{};
    if (in.history) {
        LY_CK(L.hist32.alloc(size_t(std::max(slots, 1LL))));
        LY_CK(cudaMemsetAsync(L.hist32.p, 0, sizeof(float) * size_t(std::max(slots, 1LL)), s));
        S.hist32 = L.hist32.p;
    } else {
        L.hist32.release();
    }
    if (in.btype) {
        LY_CK(L.btype_c.alloc(size_t(std::max(slots, 1LL))));
        LY_CK(cudaMemsetAsync(L.btype_c.p, 0, size_t(std::max(slots, 1LL)), s));
        S.btype_c = L.btype_c.p;
    } else {
        L.btype_c.release();
    }
    if (in.lambda) {
        LY_CK(L.lambda32.alloc(size_t(std::max(slots, 1LL))));
        LY_CK(fill<float>(L.lambda32.p, slots, 1.f, s));
        S.lambda32 = L.lambda32.p;
    } else {
        L.lambda32.release();
    }
    if (in.beta) {
        LY_CK(L.beta32.alloc(size_t(std::max(slots, 1LL))));
        LY_CK(fill<float>(L.beta32.p, slots, 1.f, s));
        S.beta32 = L.beta32.p;
    } else {
        L.beta32.release();
    }
    S.entries = in.entries;
    S.perm = L.perm.p;
    S.inv = halo_key_inv;
    S.tile_of = L.tile_of.p;
    S.tile_start = L.tile_start.p;
    S.slot_off = L.slot_off.p;
    S.halo_off = L.halo_off.p;
    S.hk = hk;
    S.nofail = in.nofail;
    S.hist = in.hist;
    S.btype = in.btype;
    S.lambda = in.lambda;
    S.beta = in.beta;
    S.n_own = n_own;
    S.N = N;
    S.T = T;
    S.lidx = L.lidx.p;
    S.own_slot = L.own_slot.p;
    LY_CK(L.wgroups.alloc(size_t(std::max(tiles, 1)) * size_t(T / 32)));
    LY_CK(cudaMemsetAsync(L.wgroups.p, 0, sizeof(int) * size_t(std::max(tiles, 1)) * size_t(T / 32), s));
    S.wgroups = L.wgroups.p;
    if (g.morton) {
        LY_CK(L.origk.alloc(size_t(std::max(slots, 1LL))));
        S.origk = L.origk.p;
    } else {
        L.origk.release();
    }
    if (n_own > 0)
        slot_kernel<<<blocks_for(n_own), TPB, 0, s>>>(S);
    LY_CK(cudaGetLastError());
    if (g.morton && n_own > 0 && slots > 0) {
        // rows by halo record (sort_rows_kernel): sort from copies of the
        // unsorted per-slot arrays
        const size_t ns = size_t(slots);
        unsigned short *lidx0, *origk0;
        LY_CK(tmp.get(&lidx0, ns));
        LY_CK(tmp.get(&origk0, ns));
        LY_CK(cudaMemcpyAsync(lidx0, L.lidx.p, 2 * ns, cudaMemcpyDeviceToDevice, s));
        LY_CK(cudaMemcpyAsync(origk0, L.origk.p, 2 * ns, cudaMemcpyDeviceToDevice, s));
        SortArgs R{};
        R.live = live;
        R.tile_of = L.tile_of.p;
        R.tile_start = L.tile_start.p;
        R.slot_off = L.slot_off.p;
        R.n_own = n_own;
        R.T = T;
        R.lidx0 = lidx0;
        R.origk0 = origk0;
        R.lidx = L.lidx.p;
        R.origk = L.origk.p;
        auto copy_f = [&](float* a, const float** a0, float** out) -> cudaError_t {
            if (!a)
                return cudaSuccess;
            float* c0;
            cudaError_t e = tmp.get(&c0, ns);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(c0, a, 4 * ns, cudaMemcpyDeviceToDevice, s);
            *a0 = c0;
            *out = a;
            return e;
        };
        LY_CK(copy_f(L.hist32.p, &R.hist0, &R.hist));
        LY_CK(copy_f(L.lambda32.p, &R.lambda0, &R.lambda));
        LY_CK(copy_f(L.beta32.p, &R.beta0, &R.beta));
        if (L.btype_c.p) {
            uint8_t* b0;
            LY_CK(tmp.get(&b0, ns));
            LY_CK(cudaMemcpyAsync(b0, L.btype_c.p, ns, cudaMemcpyDeviceToDevice, s));
            R.btype0 = b0;
            R.btype = L.btype_c.p;
        }
        sort_rows_kernel<<<unsigned((n_own + SORT_WARPS - 1) / SORT_WARPS), SORT_WARPS * 32, 0, s>>>(R);
        LY_CK(cudaGetLastError());
    }
    L.inv_host.resize(size_t(n));
    LY_CK(cudaMemcpyAsync(L.inv_host.data(), L.inv.p, sizeof(int) * size_t(n),
                          cudaMemcpyDeviceToHost, s));
    LY_CK(cudaStreamSynchronize(s));
    return cudaSuccess;
}

} // namespace pdb
