// pd_family.cu -- family construction on the device.
//
// Reproduces build_family (geometry.cpp:97-211) bit for bit:
//   * the same uniform cell index of side delta, with the same origin (grid
//     hint or coordinate bounding box), the same floor((x - o) / cell) and
//     clamping (geometry.cpp:86-129) -- fp64 IEEE on the device equals the host;
//   * the same membership test r2 = dx*dx + dy*dy + dz*dz <= delta^2 over the
//     27 surrounding cells, with the coincident-node error for r2 < 1e-24;
//   * rows sorted ascending and padded with -1 to N = bit_ceil(max |H_i|)
//     (pack_rows, geometry.cpp:131-161).
// Pipeline: cell keys -> CUB radix sort (node order stable within a cell) ->
// cell start table -> one warp per node counts, then fills its row in shared
// memory and bitonic-sorts it.
#include <cuda_runtime.h>
#include <cub/device/device_radix_sort.cuh>

#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "pd_device.cuh"
#include "pd_internal.h"

namespace pdb {
namespace {

constexpr int MAX_ROW = 1024;     // per-node neighbours the builder can sort
constexpr int WARPS = 4;          // warps per block in the row kernels

struct CellGrid {
    double ox, oy, oz, cell;
    long long nx, ny, nz;
};

__device__ __forceinline__ long long clamp_coord(double x, double o, double cell, long long count) {
    long long c = (long long)floor(__ddiv_rn(__dsub_rn(x, o), cell));
    c = c < 0 ? 0 : c;
    return c > count - 1 ? count - 1 : c;
}

__global__ void cell_key_kernel(const double* coords, long long n, CellGrid g,
                                unsigned long long* keys, int* vals) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n)
        return;
    const long long cx = clamp_coord(coords[3 * i], g.ox, g.cell, g.nx);
    const long long cy = clamp_coord(coords[3 * i + 1], g.oy, g.cell, g.ny);
    const long long cz = clamp_coord(coords[3 * i + 2], g.oz, g.cell, g.nz);
    keys[i] = (unsigned long long)((cz * g.ny + cy) * g.nx + cx);
    vals[i] = int(i);
}

// start[c] = first sorted position of cell c (dense table), start[ncells] = n
__global__ void cell_start_kernel(const unsigned long long* sorted, long long n, long long ncells,
                                  long long* start) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t > n)
        return;
    const long long prev = t == 0 ? -1 : (long long)sorted[t - 1];
    const long long here = t == n ? ncells : (long long)sorted[t];
    for (long long c = prev + 1; c <= here; ++c)
        start[c] = t;
}

__device__ __forceinline__ void cell_range(const unsigned long long* sorted, const long long* start,
                                           long long n, long long id, long long& b, long long& e) {
    if (start) {
        b = start[id];
        e = start[id + 1];
        return;
    }
    long long lo = 0, hi = n;
    while (lo < hi) {
        const long long mid = (lo + hi) >> 1;
        if ((long long)sorted[mid] < id)
            lo = mid + 1;
        else
            hi = mid;
    }
    b = lo;
    hi = n;
    while (lo < hi) {
        const long long mid = (lo + hi) >> 1;
        if ((long long)sorted[mid] <= id)
            lo = mid + 1;
        else
            hi = mid;
    }
    e = lo;
}

struct RowArgs {
    const double* coords;
    long long n;
    double h2;
    CellGrid g;
    const unsigned long long* sorted;
    const int* order;
    const long long* start;
    int* counts;
    int* entries;       // fill pass only
    int group;          // fill pass only
    unsigned long long* coincident; // (i << 32 | j) of the first coincident pair
};

template <bool FILL>
__global__ void __launch_bounds__(WARPS * 32) row_kernel(RowArgs R) {
    __shared__ int buf[WARPS][MAX_ROW];
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    const long long i = (long long)blockIdx.x * WARPS + w;
    if (i >= R.n)
        return;
    const double xi = R.coords[3 * i], yi = R.coords[3 * i + 1], zi = R.coords[3 * i + 2];
    const long long cx = clamp_coord(xi, R.g.ox, R.g.cell, R.g.nx);
    const long long cy = clamp_coord(yi, R.g.oy, R.g.cell, R.g.ny);
    const long long cz = clamp_coord(zi, R.g.oz, R.g.cell, R.g.nz);
    int count = 0;
    for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                const long long ccx = cx + dx, ccy = cy + dy, ccz = cz + dz;
                if (ccx < 0 || ccy < 0 || ccz < 0 || ccx >= R.g.nx || ccy >= R.g.ny ||
                    ccz >= R.g.nz)
                    continue;
                long long b, e;
                cell_range(R.sorted, R.start, R.n, (ccz * R.g.ny + ccy) * R.g.nx + ccx, b, e);
                for (long long t0 = b; t0 < e; t0 += 32) {
                    const long long t = t0 + lane;
                    bool hit = false;
                    int j = -1;
                    if (t < e) {
                        j = R.order[t];
                        if ((long long)j != i) {
                            const double d0 = __dsub_rn(R.coords[3 * (long long)j], xi);
                            const double d1 = __dsub_rn(R.coords[3 * (long long)j + 1], yi);
                            const double d2 = __dsub_rn(R.coords[3 * (long long)j + 2], zi);
                            const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)),
                                                        __dmul_rn(d2, d2));
                            hit = r2 <= R.h2;
                            if (hit && r2 < 1e-24)
                                atomicMin(R.coincident,
                                          ((unsigned long long)i << 32) | (unsigned long long)j);
                        }
                    }
                    const unsigned mask = __ballot_sync(0xffffffffu, hit);
                    if (FILL && hit) {
                        const int pos = count + __popc(mask & ((1u << lane) - 1u));
                        if (pos < MAX_ROW)
                            buf[w][pos] = j;
                    }
                    count += __popc(mask);
                }
            }
    if (!FILL) {
        if (lane == 0)
            R.counts[i] = count;
        return;
    }
    // bitonic sort of the row in shared memory (padding = INT_MAX sorts last)
    int len = 1;
    while (len < count)
        len <<= 1;
    for (int t = count + lane; t < len; t += 32)
        buf[w][t] = 0x7fffffff;
    __syncwarp();
    for (int k = 2; k <= len; k <<= 1)
        for (int jj = k >> 1; jj > 0; jj >>= 1) {
            for (int t = lane; t < len; t += 32) {
                const int p = t ^ jj;
                if (p > t) {
                    const int a = buf[w][t], bb = buf[w][p];
                    const bool up = (t & k) == 0;
                    if ((a > bb) == up) {
                        buf[w][t] = bb;
                        buf[w][p] = a;
                    }
                }
            }
            __syncwarp();
        }
    int* row = R.entries + i * (long long)R.group;
    for (int t = lane; t < R.group; t += 32)
        row[t] = t < count ? buf[w][t] : -1;
}

__global__ void max_kernel(const int* x, long long n, int* out) {
    int m = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        m = max(m, x[i]);
    for (int o = 16; o > 0; o /= 2)
        m = max(m, __shfl_down_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0)
        atomicMax(out, m);
}

int ffail(int code, const std::string& msg) { return set_error(code, msg.c_str()); }

} // namespace
} // namespace pdb

struct pd_family {
    long long n = 0;
    int group = 0;
    int* entries = nullptr;
    int* counts = nullptr;
};

using namespace pdb;

#define PF_CK(expr)                                                                              \
    do {                                                                                         \
        cudaError_t e_ = (expr);                                                                 \
        if (e_ != cudaSuccess) {                                                                 \
            rc = ffail(PD_E_CUDA, std::string("CUDA error in build_family: ") +                 \
                                      cudaGetErrorString(e_));                                   \
            goto done;                                                                           \
        }                                                                                        \
    } while (0)

extern "C" {

// build_family(coords, horizon, grid_hint) (geometry.hpp:60-62).  grid_hint =
// {ox, oy, oz, spacing, nx, ny, nz} or NULL.  The rows stay on the device in
// *out until pd_family_download / pd_family_free.
int pd_build_family(const double* coords, int64_t n, double horizon, const double* grid_hint,
                    struct pd_family** out, int64_t* group_size_out) {
    *out = nullptr;
    if (!(horizon > 0))
        return ffail(PD_E_DOMAIN, "build_family: horizon must be positive");
    if (n < 1 || !coords)
        return ffail(PD_E_INVALID_ARGUMENT, "build_family: bad coordinate array");
    int rc = PD_OK;
    // make_cell_index (geometry.cpp:97-129): origin and extent on the host
    double lo[3], hi[3];
    if (grid_hint && grid_hint[3] > 0) {
        for (int d = 0; d < 3; ++d) {
            lo[d] = grid_hint[d];
            hi[d] = grid_hint[d] + double((long long)grid_hint[4 + d] - 1) * grid_hint[3];
        }
    } else {
        for (int d = 0; d < 3; ++d)
            lo[d] = hi[d] = coords[d];
        for (int64_t i = 1; i < n; ++i)
            for (int d = 0; d < 3; ++d) {
                lo[d] = std::min(lo[d], coords[3 * i + d]);
                hi[d] = std::max(hi[d], coords[3 * i + d]);
            }
    }
    CellGrid g;
    g.ox = lo[0];
    g.oy = lo[1];
    g.oz = lo[2];
    g.cell = horizon;
    long long cnt[3];
    for (int d = 0; d < 3; ++d)
        cnt[d] = std::max(1LL, (long long)std::floor((hi[d] - lo[d]) / horizon) + 1);
    g.nx = cnt[0];
    g.ny = cnt[1];
    g.nz = cnt[2];
    const long long ncells = g.nx * g.ny * g.nz;

    double* d_coords = nullptr;
    unsigned long long *keys = nullptr, *keys_sorted = nullptr, *coincident = nullptr;
    int *vals = nullptr, *order = nullptr, *d_max = nullptr;
    long long* start = nullptr;
    void* temp = nullptr;
    size_t temp_bytes = 0;
    pd_family* fam = new pd_family;
    fam->n = n;
    int max_count = 0;
    unsigned long long first_coincident = ~0ull;
    RowArgs R{};
    const unsigned blocks = unsigned((n + 255) / 256);
    const unsigned row_blocks = unsigned((n + WARPS - 1) / WARPS);
    int end_bit = 1;
    while (end_bit < 64 && (1ull << end_bit) < (unsigned long long)ncells)
        ++end_bit;

    PF_CK(cudaMalloc(&d_coords, sizeof(double) * 3 * n));
    PF_CK(cudaMemcpy(d_coords, coords, sizeof(double) * 3 * n, cudaMemcpyHostToDevice));
    PF_CK(cudaMalloc(&keys, sizeof(unsigned long long) * n));
    PF_CK(cudaMalloc(&keys_sorted, sizeof(unsigned long long) * n));
    PF_CK(cudaMalloc(&vals, sizeof(int) * n));
    PF_CK(cudaMalloc(&order, sizeof(int) * n));
    PF_CK(cudaMalloc(&coincident, sizeof(unsigned long long)));
    PF_CK(cudaMemset(coincident, 0xff, sizeof(unsigned long long)));
    PF_CK(cudaMalloc(&d_max, sizeof(int)));
    PF_CK(cudaMemset(d_max, 0, sizeof(int)));
    cell_key_kernel<<<blocks, 256>>>(d_coords, n, g, keys, vals);
    PF_CK(cudaGetLastError());
    PF_CK(cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, keys, keys_sorted, vals, order,
                                          int(n), 0, end_bit));
    PF_CK(cudaMalloc(&temp, temp_bytes));
    PF_CK(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys, keys_sorted, vals, order, int(n),
                                          0, end_bit));
    if (ncells <= 8 * n + 4096) {
        PF_CK(cudaMalloc(&start, sizeof(long long) * (ncells + 1)));
        cell_start_kernel<<<unsigned((n + 1 + 255) / 256), 256>>>(keys_sorted, n, ncells, start);
        PF_CK(cudaGetLastError());
    }
    PF_CK(cudaMalloc(&fam->counts, sizeof(int) * n));
    R.coords = d_coords;
    R.n = n;
    R.h2 = horizon * horizon;
    R.g = g;
    R.sorted = keys_sorted;
    R.order = order;
    R.start = start;
    R.counts = fam->counts;
    R.coincident = coincident;
    row_kernel<false><<<row_blocks, WARPS * 32>>>(R);
    PF_CK(cudaGetLastError());
    PF_CK(cudaMemcpy(&first_coincident, coincident, sizeof first_coincident,
                     cudaMemcpyDeviceToHost));
    if (first_coincident != ~0ull) {
        rc = ffail(PD_E_INVALID_ARGUMENT,
                   "build_family: coincident nodes " + std::to_string(first_coincident >> 32) +
                       " and " + std::to_string(first_coincident & 0xffffffffull));
        goto done;
    }
    max_kernel<<<std::min(blocks, 148u * 8u), 256>>>(fam->counts, n, d_max);
    PF_CK(cudaGetLastError());
    PF_CK(cudaMemcpy(&max_count, d_max, sizeof(int), cudaMemcpyDeviceToHost));
    if (max_count > MAX_ROW) {
        rc = ffail(PD_E_INVALID_ARGUMENT, "build_family: a family has " +
                                              std::to_string(max_count) +
                                              " members; the device builder supports 1024");
        goto done;
    }
    fam->group = 1;
    while (fam->group < std::max(max_count, 1))
        fam->group <<= 1;
    PF_CK(cudaMalloc(&fam->entries, sizeof(int) * size_t(n) * size_t(fam->group)));
    R.entries = fam->entries;
    R.group = fam->group;
    row_kernel<true><<<row_blocks, WARPS * 32>>>(R);
    PF_CK(cudaGetLastError());
    PF_CK(cudaDeviceSynchronize());
done:
    cudaFree(d_coords);
    cudaFree(keys);
    cudaFree(keys_sorted);
    cudaFree(vals);
    cudaFree(order);
    cudaFree(coincident);
    cudaFree(d_max);
    cudaFree(start);
    cudaFree(temp);
    if (rc != PD_OK) {
        cudaFree(fam->entries);
        cudaFree(fam->counts);
        delete fam;
        return rc;
    }
    *out = fam;
    *group_size_out = fam->group;
    return set_error(PD_OK, "");
}

// Copy the rows (n x N), n_neigh and initial_n_neigh (both = |H_i|) to the host.
int pd_family_download(struct pd_family* fam, int32_t* entries, int32_t* n_neigh,
                       int32_t* initial) {
    int rc = PD_OK;
    if (entries)
        PF_CK(cudaMemcpy(entries, fam->entries, sizeof(int) * size_t(fam->n) * size_t(fam->group),
                         cudaMemcpyDeviceToHost));
    if (n_neigh)
        PF_CK(cudaMemcpy(n_neigh, fam->counts, sizeof(int) * size_t(fam->n),
                         cudaMemcpyDeviceToHost));
    if (initial)
        PF_CK(cudaMemcpy(initial, fam->counts, sizeof(int) * size_t(fam->n),
                         cudaMemcpyDeviceToHost));
done:
    return rc;
}

void pd_family_free(struct pd_family* fam) {
    if (!fam)
        return;
    cudaFree(fam->entries);
    cudaFree(fam->counts);
    delete fam;
}

} // extern "C"
