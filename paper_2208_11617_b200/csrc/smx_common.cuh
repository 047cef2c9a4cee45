// Shared device-side definitions for the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "smx_b200.h"
#include "smx_maps.hpp"

namespace smx {

// Everything a kernel needs to know about one launch, passed by value.
struct Geom {
    int kind;   // SMX_BB / SMX_H2D / SMX_H3D
    int dims;   // 2 or 3
    int n;      // map parameter
    int rho;    // tile edge
    int ex, ey, ez;
    int strict;           // h2d/h3d emit the strict view: data row = y - 1
    int side;             // cell side S
    const unsigned long long* prefix;  // 3-D: tet_layer_prefix(S, z), z = 0..S+1
    trapezoid<int> trap;  // SMX_TRAP: the band this launch covers (one launch per band)
    int wy0;              // first grid row of this launch (row-range shards: wy = wy0 + blockIdx.y)
    int ty0, ty1;         // x-run 2-D kernels: only tiles whose data tile row is in [ty0, ty1)
                          // (ty1 == 0: no filter) — one chunk of a pipelined host-buffer call
    const int2* order;    // ACCUM x-run: CTA i takes strip group order[i] = (x group, grid row)
    int norder;           // (a launch order sorted by data tile row; nullptr: blockIdx order)
};

// strict_view (maps.hpp:35-38): outputs in { x < y }, shifted y - 1 by the sweep
__host__ __device__ constexpr bool strict_kind(int k) { return k == SMX_H2D || k == SMX_PADDED || k == SMX_TRAP || k == SMX_H3D; }

// The raw map_outcome of one block (maps.hpp), per kind.
template <int KIND>
__device__ __forceinline__ outcome<int> map_raw(const Geom& g, int wx, int wy, int wz) {
    if (KIND == SMX_H2D) return map_h2d<int>(wx, wy);
    if (KIND == SMX_H3D) return map_h3d<int>(wx, wy, wz, g.n);
    if (KIND == SMX_PADDED) return map_h2d_padded<int>(wx, wy, g.n);
    if (KIND == SMX_TRAP) return map_h2d_trapezoid<int>(wx, wy, g.trap);
    if (KIND == SMX_RB) return map_rb<int>(wx, wy, g.n);
    if (KIND == SMX_LAMBDA) return map_lambda<int>(uint64_t(wx));
    return map_bb<int>(wx, wy, wz, g.n, g.dims);
}

// Per-block map dispatch; returns the with-diagonal tile coordinate (strict
// shift already applied, simulator.hpp:202).
template <int KIND>
__device__ __forceinline__ outcome<int> map_block(const Geom& g, int wx, int wy, int wz) {
    outcome<int> o = map_raw<KIND>(g, wx, wy, wz);
    if (strict_kind(KIND)) o.y -= 1;
    return o;
}

__device__ __forceinline__ unsigned long long tri_idx(long long x, long long y) {
    return (unsigned long long)(y) * (unsigned long long)(y + 1) / 2ull + (unsigned long long)x;
}

// Counter slots: atomics are spread over NSLOT addresses to avoid a single
// hot L2 line; the host sums them.
constexpr int NSLOT = 64;
struct DevCounters {
    unsigned long long blocks_void[NSLOT];
    unsigned long long threads_useful[NSLOT];
};

}  // namespace smx

