// pd_fast.cuh -- layout of the fast (tolerance-bound) path.
//
// Nodes are renumbered into spatial bricks (internal order); a tile is up to
// T = 512 consecutive internal nodes of one brick and is processed by one CTA
// with one thread per node.  Each tile owns:
//   halo[halo_off[t] .. halo_off[t+1])  internal ids of every node its rows
//                                       reference (owned nodes included), staged
//                                       into shared memory once per step as
//                                       fp32 {x - O_t, V} and {u - U_t, no_fail}
//   lidx   uint16 per live slot          bits 0-14: shared-memory index of the
//                                       neighbour (halo position + 1); 0 = broken
//                                       or padding (a dummy record that adds 0);
//                                       bit 15: the neighbour is a no-fail node.  Slot c of
//                                       tile-thread t lives at
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
    const unsigned short* own_slot; // shared-memory position of each (internal) node in its tile,
                                    // bit 15 = the node is a no-failure node
    const int* nf_start;       // per tile: first slot offset that names a no-failure node
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
};

} // namespace pdb
