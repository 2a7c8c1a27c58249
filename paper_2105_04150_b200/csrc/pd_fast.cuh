// pd_fast.cuh -- layout of the fast (tolerance-bound) path.
//
// Nodes are renumbered into spatial bricks (internal order); a tile is up to
// T = 512 consecutive internal nodes of one brick and is processed by one CTA
// with one thread per node.  Each tile owns:
//   halo[halo_off[t] .. halo_off[t+1])  internal ids of every node its rows
//                                       reference (owned nodes included), staged
//                                       into shared memory once per step as
//                                       fp32 {x - O_t, V} and {u - U_t, no_fail}
//   lidx   uint16 per live slot          index p of the neighbour's shared-memory
//                                       record (halo position + 1; the records
//                                       are sA[p] float4, sB[p] float2, sV[p]);
//                                       0 = broken or padding (record 0 is a
//                                       dummy that adds 0).  No-failure
//                                       neighbours are staged last in the halo,
//                                       so p >= nf_start[tile] flags them.  Slot
//                                       c of tile-thread t lives at
//                                       slot_off[t] + (c/8)*T*8 + t*8 + c%8, so
//                                       one 16-byte load fetches 8 slots and a
//                                       warp's loads are contiguous.
// Rows are compacted (live slots in the reference's slot order); the original
// slot positions are recovered at download by walking the uploaded row.
#pragma once

#include <cstdint>

namespace pdb {

constexpr int FAST_T = 512;           // default threads (= owned nodes) per tile
constexpr int FAST_MAX_HALO = 7000;   // (7000 + 1) * 28 B = 196 KB of shared memory; 8*(7000+1) < 65536

struct FastDev {
    int T;                     // threads (= owned nodes) per tile: 512 or 256
    int cap;                   // shared-memory records reserved per array (max halo + 1)
    int cfg;                   // kernel configuration (pd_fast.cu launch_one)
    int n_tiles;
    int tile0;                 // first tile of this launch
    const int* tile_start;     // n_tiles + 1 internal node ids
    const long long* halo_off; // n_tiles + 1
    const int* halo;           // internal ids
    const long long* slot_off; // n_tiles
    const int* kmax8;          // per tile, multiple of 8
    const int* wgroups;        // per (tile, warp): 8-slot groups of the warp's longest row
    const unsigned short* own_slot; // shared-memory position of each (internal) node in its tile,
                                    // bit 15 = the node is a no-failure node
    const int* nf_start;       // per tile: first record index that is a no-failure node
    unsigned short* lidx;
    float* hist;               // compact fp32 history (n-linear laws)
    const uint8_t* btype;      // compact bond types or NULL
    const float* lambda;       // compact or NULL
    const float* beta;         // compact or NULL
    float pmb_c, pmb_sc;       // the single-PMB-law specialisation
    float pmb_cv;              // c * V when every volume is equal (KIND 0)
};

struct FastLaw {
    float c;
    int nbp;
    float bp[8];
    float f[8];
    float sl[8];  // segment slopes (f_k - f_{k-1}) / (bp_k - bp_{k-1}), from fp64 on the host
};

// envelope_force (formulas.hpp:77-89) in fp32 with the host-computed slopes:
// f_{k-1} + (s - bp_{k-1}) * sl_k on the first segment whose end exceeds s
// (the last segment also beyond its end); no division on the device.
// The secant stiffness env(h) / h (formulas.hpp:92-96) is sl_0 exactly while h
// lies on the first segment (h <= 0 included: c = f_0 / bp_0 for a validated
// law); the kernels take that branch instead of env(h) * rcp(h), which would
// turn a subnormal h (a wave front's leading edge) into 0 * inf.
__host__ __device__ __forceinline__ float fast_envelope(const FastLaw& law, float s) {
    float s_prev = 0.f, f_prev = 0.f;
    for (int k = 0; k < law.nbp; ++k) {
        if (s < law.bp[k] || k + 1 == law.nbp)
            return f_prev + (s - s_prev) * law.sl[k];
        s_prev = law.bp[k];
        f_prev = law.f[k];
    }
    return law.c * s;
}

inline void fast_law_from(FastLaw& out, double c, int nbp, const double* bp, const double* f) {
    out = FastLaw{};
    out.c = float(c);
    out.nbp = nbp;
    double s_prev = 0.0, f_prev = 0.0;
    for (int b = 0; b < nbp && b < 8; ++b) {
        out.bp[b] = float(bp[b]);
        out.f[b] = float(f[b]);
        out.sl[b] = float((f[b] - f_prev) / (bp[b] - s_prev));
        s_prev = bp[b];
        f_prev = f[b];
    }
}

} // namespace pdb
