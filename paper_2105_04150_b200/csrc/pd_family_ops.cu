// pd_family_ops.cu -- setup-time operations on a family list, on the device
// (SURVEY.md section 8(f), row 1), bit for bit with the reference:
//
//   pd_classify_bonds              build_family's BondClassifier pass (pack_rows,
//                                  geometry.cpp:131-161; geometry.hpp:45-54) for
//                                  a rule-table classifier: every node gets a
//                                  class from region rules, the slot (i, j) the
//                                  type table[class_i][class_j]
//   pd_neighborhood_volumes        neighborhood_volumes (geometry.cpp:238-252):
//                                  per node an in-order fp64 sum over its live
//                                  slots, so the sum is the reference's bits
//   pd_surface_correction_factors  surface_correction_factors (geometry.cpp:263-283):
//                                  lambda = 2 V0 / (V_i + V_j), 1 on padding
//   pd_break_initial_bonds         break_initial_bonds with plane_crossing_predicate
//                                  or notch_predicate (geometry.cpp:285-319)
//
// Compiled with -fmad=false and written with __d*_rn: every value is the
// reference's IEEE expression.  The host arrays are uploaded, processed and
// downloaded per call (setup time, not the time step).
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "pd_b200.h"
#include "pd_internal.h"

namespace pdb {
namespace {

constexpr int TPB = 256;

inline unsigned blocks_for(long long n) { return unsigned((n + TPB - 1) / TPB); }

// one region rule: box (inclusive bounds) or cylinder about an axis
__device__ __forceinline__ bool in_region(const pd_region& r, double x, double y, double z) {
    const double p[3] = {x, y, z};
    if (r.kind == PD_REGION_BOX) {
        for (int d = 0; d < 3; ++d)
            if (!(p[d] >= r.lo[d] && p[d] <= r.hi[d]))
                return false;
        return true;
    }
    // cylinder: axis a, centre (c0, c1) in the two other axes (ascending
    // order), radius r, extent [lo[a], hi[a]] along the axis
    const int a = r.axis;
    const int b0 = a == 0 ? 1 : 0, b1 = a == 2 ? 1 : 2;
    if (!(p[a] >= r.lo[a] && p[a] <= r.hi[a]))
        return false;
    const double d0 = __dsub_rn(p[b0], r.c[0]), d1 = __dsub_rn(p[b1], r.c[1]);
    return __dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)) <= __dmul_rn(r.radius, r.radius);
}

// node classes: the last matching region wins, else default_class
__global__ void node_class_kernel(const double* coords, long long n, const pd_region* regions,
                                  int n_regions, int default_class, int* cls) {
    const long long i = blockIdx.x * (long long)TPB + threadIdx.x;
    if (i >= n)
        return;
    int c = default_class;
    for (int k = 0; k < n_regions; ++k)
        if (in_region(regions[k], coords[3 * i], coords[3 * i + 1], coords[3 * i + 2]))
            c = regions[k].cls;
    cls[i] = c;
}

__global__ void bond_type_kernel(const int32_t* entries, long long n, int N, const int* cls,
                                 const uint8_t* table, int n_classes, uint8_t* out) {
    const long long idx = blockIdx.x * (long long)TPB + threadIdx.x;
    if (idx >= n * N)
        return;
    const int32_t j = entries[idx];
    // pack_rows assigns a type to every member slot (padding keeps 0)
    out[idx] = j < 0 ? uint8_t(0) : table[cls[idx / N] * n_classes + cls[j]];
}

// neighborhood_volumes: sum += volumes[j] over the row in slot order
__global__ void nbhd_kernel(const int32_t* entries, long long n, int N, const double* vol,
                            double* out) {
    const long long i = blockIdx.x * (long long)TPB + threadIdx.x;
    if (i >= n)
        return;
    double sum = 0.0;
    for (int k = 0; k < N; ++k) {
        const int32_t j = entries[i * N + k];
        if (j != -1)
            sum = __dadd_rn(sum, vol[j]);
    }
    out[i] = sum;
}

__global__ void lambda_kernel(const int32_t* entries, long long n, int N, const double* nbhd,
                              double two_v0, double* lambda, unsigned long long* first_bad) {
    const long long idx = blockIdx.x * (long long)TPB + threadIdx.x;
    if (idx >= n * N)
        return;
    const int32_t j = entries[idx];
    if (j == -1) {
        lambda[idx] = 1.0;
        return;
    }
    const double denom = __dadd_rn(nbhd[idx / N], nbhd[j]);
    if (!(denom > 0.0)) {
        atomicMin(first_bad, (unsigned long long)idx);
        lambda[idx] = 1.0;
        return;
    }
    lambda[idx] = __ddiv_rn(two_v0, denom);
}

// break_initial_bonds: entries[idx] = -1 where the predicate holds; the row's
// count drops (the reference decrements n_neigh per zapped slot)
__global__ void break_kernel(int32_t* entries, int32_t* n_neigh, long long n, int N,
                             const double* coords, pd_bond_predicate P) {
    const long long idx = blockIdx.x * (long long)TPB + threadIdx.x;
    if (idx >= n * N)
        return;
    const int32_t j = entries[idx];
    if (j == -1)
        return;
    const long long i = idx / N;
    const double* a = coords + 3 * i;
    const double* b = coords + 3 * (long long)j;
    const double da = __dsub_rn(a[P.axis], P.position), db = __dsub_rn(b[P.axis], P.position);
    bool hit;
    if (P.kind == PD_PREDICATE_PLANE) {
        hit = __dmul_rn(da, db) < 0.0;
    } else {
        hit = false;
        if (!(__dmul_rn(da, db) >= 0.0)) {
            const double t = __ddiv_rn(da, __dsub_rn(da, db));
            const double cross = __dadd_rn(a[P.sweep_axis],
                                           __dmul_rn(t, __dsub_rn(b[P.sweep_axis], a[P.sweep_axis])));
            hit = cross <= P.depth;
        }
    }
    if (hit) {
        entries[idx] = -1;
        atomicSub(n_neigh + i, 1);
    }
}

// entries must name nodes of the list (or -1): a bad index would read past
// the per-node arrays; the first offending row is reported
__global__ void entry_range_kernel(const int32_t* entries, long long n, int N,
                                   unsigned long long* first_bad) {
    const long long idx = blockIdx.x * (long long)TPB + threadIdx.x;
    if (idx >= n * N)
        return;
    const int32_t j = entries[idx];
    if (j < -1 || j >= n)
        atomicMin(first_bad, (unsigned long long)(idx / N));
}

// RAII device buffer for this translation unit
template <class T> struct Buf {
    T* p = nullptr;
    ~Buf() { cudaFree(p); }
    cudaError_t alloc(size_t count) { return cudaMalloc(&p, sizeof(T) * (count ? count : 1)); }
    cudaError_t up(const T* h, size_t count) {
        cudaError_t e = alloc(count);
        if (e == cudaSuccess && count)
            e = cudaMemcpy(p, h, sizeof(T) * count, cudaMemcpyHostToDevice);
        return e;
    }
};

#define FO_CK(expr)                                                                              \
    do {                                                                                         \
        cudaError_t e_ = (expr);                                                                 \
        if (e_ != cudaSuccess)                                                                   \
            return set_error(PD_E_CUDA, (std::string("CUDA error in ") + __func__ + ": " +      \
                                         cudaGetErrorString(e_)).c_str());                       \
    } while (0)

int entries_in_range(const int32_t* dev_entries, long long n, int N, const char* who) {
    Buf<unsigned long long> bad;
    FO_CK(bad.alloc(1));
    FO_CK(cudaMemset(bad.p, 0xff, sizeof(unsigned long long)));
    if (n > 0)
        entry_range_kernel<<<blocks_for(n * N), TPB>>>(dev_entries, n, N, bad.p);
    FO_CK(cudaGetLastError());
    unsigned long long first = 0;
    FO_CK(cudaMemcpy(&first, bad.p, sizeof first, cudaMemcpyDeviceToHost));
    if (first != ~0ull)
        return set_error(PD_E_INVALID_ARGUMENT,
                         (std::string(who) + ": NeighborList entry out of range in row " +
                          std::to_string(first)).c_str());
    return PD_OK;
}

int check_family(const pd_neighbor_list* f, const char* who) {
    if (!f || f->n < 0 || f->group_size < 1 || (f->n > 0 && (!f->entries || !f->n_neigh)))
        return set_error(PD_E_INVALID_ARGUMENT, (std::string(who) + ": bad family").c_str());
    return PD_OK;
}

template <class T> struct Buf;

int device_ok() {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count < 1) {
        cudaGetLastError();
        return set_error(PD_E_NO_DEVICE, "no sm_100 (B200) device is visible to the CUDA runtime");
    }
    return PD_OK;
}

int neighborhood_volumes_dev(const pd_neighbor_list* f, const double* volumes, Buf<int32_t>& ent,
                             Buf<double>& nbhd) {
    const long long n = f->n, N = f->group_size;
    Buf<double> vol;
    FO_CK(ent.up(f->entries, size_t(n * N)));
    if (entries_in_range(ent.p, n, int(N), "neighborhood_volumes") != PD_OK)
        return PD_E_INVALID_ARGUMENT;
    FO_CK(vol.up(volumes, size_t(n)));
    FO_CK(nbhd.alloc(size_t(n)));
    if (n > 0)
        nbhd_kernel<<<blocks_for(n), TPB>>>(ent.p, n, int(N), vol.p, nbhd.p);
    FO_CK(cudaGetLastError());
    return PD_OK;
}

} // namespace
} // namespace pdb

using namespace pdb;

extern "C" {

int pd_classify_bonds(const double* coords, const pd_neighbor_list* family,
                      const pd_classifier* cls, uint8_t* bond_type_out) {
    if (check_family(family, "classify_bonds") != PD_OK)
        return PD_E_INVALID_ARGUMENT;
    if (!cls || cls->n_classes < 1 || cls->n_classes > 256 || !cls->type_table ||
        cls->n_regions < 0 || (cls->n_regions > 0 && !cls->regions) ||
        cls->default_class < 0 || cls->default_class >= cls->n_classes)
        return set_error(PD_E_INVALID_ARGUMENT, "classify_bonds: bad classifier");
    for (int k = 0; k < cls->n_regions; ++k) {
        const pd_region& r = cls->regions[k];
        if (r.cls < 0 || r.cls >= cls->n_classes || (r.kind != PD_REGION_BOX &&
                                                     r.kind != PD_REGION_CYLINDER) ||
            r.axis < 0 || r.axis > 2)
            return set_error(PD_E_INVALID_ARGUMENT, "classify_bonds: bad region rule");
    }
    // the reference requires a symmetric classifier (geometry.hpp:50-52)
    const int nc = cls->n_classes;
    for (int a = 0; a < nc; ++a)
        for (int b = 0; b < a; ++b)
            if (cls->type_table[a * nc + b] != cls->type_table[b * nc + a])
                return set_error(PD_E_INVALID_ARGUMENT,
                                 "classify_bonds: the type table must be symmetric");
    if (device_ok() != PD_OK)
        return PD_E_NO_DEVICE;
    const long long n = family->n, N = family->group_size;
    Buf<double> xyz;
    Buf<pd_region> regions;
    Buf<int> node_cls;
    Buf<uint8_t> table, out;
    Buf<int32_t> ent;
    FO_CK(xyz.up(coords, size_t(3 * n)));
    FO_CK(regions.up(cls->regions, size_t(cls->n_regions)));
    FO_CK(table.up(cls->type_table, size_t(nc * nc)));
    FO_CK(ent.up(family->entries, size_t(n * N)));
    if (entries_in_range(ent.p, n, int(N), "classify_bonds") != PD_OK)
        return PD_E_INVALID_ARGUMENT;
    FO_CK(node_cls.alloc(size_t(n)));
    FO_CK(out.alloc(size_t(n * N)));
    if (n > 0) {
        node_class_kernel<<<blocks_for(n), TPB>>>(xyz.p, n, regions.p, cls->n_regions,
                                                  cls->default_class, node_cls.p);
        bond_type_kernel<<<blocks_for(n * N), TPB>>>(ent.p, n, int(N), node_cls.p, table.p, nc,
                                                     out.p);
    }
    FO_CK(cudaGetLastError());
    FO_CK(cudaMemcpy(bond_type_out, out.p, size_t(n * N), cudaMemcpyDeviceToHost));
    return set_error(PD_OK, "");
}

int pd_neighborhood_volumes(const double* volumes, const pd_neighbor_list* family, double* out) {
    if (check_family(family, "neighborhood_volumes") != PD_OK)
        return PD_E_INVALID_ARGUMENT;
    if (device_ok() != PD_OK)
        return PD_E_NO_DEVICE;
    Buf<int32_t> ent;
    Buf<double> nbhd;
    const int rc = neighborhood_volumes_dev(family, volumes, ent, nbhd);
    if (rc != PD_OK)
        return rc;
    FO_CK(cudaMemcpy(out, nbhd.p, sizeof(double) * size_t(family->n), cudaMemcpyDeviceToHost));
    return set_error(PD_OK, "");
}

int pd_surface_correction_factors(const double* volumes, const pd_neighbor_list* family,
                                  double v0, double* lambda_out) {
    if (!(v0 > 0))
        return set_error(PD_E_DOMAIN, "surface_correction_factors: V0 must be positive");
    if (check_family(family, "surface_correction_factors") != PD_OK)
        return PD_E_INVALID_ARGUMENT;
    if (device_ok() != PD_OK)
        return PD_E_NO_DEVICE;
    const long long n = family->n, N = family->group_size;
    Buf<int32_t> ent;
    Buf<double> nbhd, lambda;
    Buf<unsigned long long> bad;
    int rc = neighborhood_volumes_dev(family, volumes, ent, nbhd);
    if (rc != PD_OK)
        return rc;
    FO_CK(lambda.alloc(size_t(n * N)));
    FO_CK(bad.alloc(1));
    FO_CK(cudaMemset(bad.p, 0xff, sizeof(unsigned long long)));
    if (n > 0)
        lambda_kernel<<<blocks_for(n * N), TPB>>>(ent.p, n, int(N), nbhd.p, 2.0 * v0,
                                                  lambda.p, bad.p);
    FO_CK(cudaGetLastError());
    unsigned long long first = 0;
    FO_CK(cudaMemcpy(&first, bad.p, sizeof first, cudaMemcpyDeviceToHost));
    if (first != ~0ull) {
        const long long i = (long long)(first / (unsigned long long)N);
        return set_error(PD_E_DOMAIN,
                         ("surface_correction_factors: zero neighborhood volume for bond " +
                          std::to_string(i) + "-" + std::to_string(family->entries[first]))
                             .c_str());
    }
    FO_CK(cudaMemcpy(lambda_out, lambda.p, sizeof(double) * size_t(n * N),
                     cudaMemcpyDeviceToHost));
    return set_error(PD_OK, "");
}

int pd_break_initial_bonds(pd_neighbor_list* family, const double* coords,
                           const pd_bond_predicate* predicate) {
    if (check_family(family, "break_initial_bonds") != PD_OK)
        return PD_E_INVALID_ARGUMENT;
    if (!predicate)
        return set_error(PD_OK, "");  // an empty predicate breaks nothing (geometry.cpp:287-288)
    const pd_bond_predicate& P = *predicate;
    if ((P.kind != PD_PREDICATE_PLANE && P.kind != PD_PREDICATE_NOTCH) || P.axis < 0 ||
        P.axis > 2 || (P.kind == PD_PREDICATE_NOTCH && (P.sweep_axis < 0 || P.sweep_axis > 2)))
        return set_error(PD_E_INVALID_ARGUMENT, "break_initial_bonds: bad predicate");
    if (device_ok() != PD_OK)
        return PD_E_NO_DEVICE;
    const long long n = family->n, N = family->group_size;
    Buf<int32_t> ent, nn;
    Buf<double> xyz;
    FO_CK(ent.up(family->entries, size_t(n * N)));
    if (entries_in_range(ent.p, n, int(N), "break_initial_bonds") != PD_OK)
        return PD_E_INVALID_ARGUMENT;
    FO_CK(nn.up(family->n_neigh, size_t(n)));
    FO_CK(xyz.up(coords, size_t(3 * n)));
    if (n > 0)
        break_kernel<<<blocks_for(n * N), TPB>>>(ent.p, nn.p, n, int(N), xyz.p, P);
    FO_CK(cudaGetLastError());
    FO_CK(cudaMemcpy(family->entries, ent.p, sizeof(int32_t) * size_t(n * N),
                     cudaMemcpyDeviceToHost));
    FO_CK(cudaMemcpy(family->n_neigh, nn.p, sizeof(int32_t) * size_t(n), cudaMemcpyDeviceToHost));
    return set_error(PD_OK, "");
}

} // extern "C"
