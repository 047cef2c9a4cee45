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
};

// Per-block map dispatch; returns the with-diagonal tile coordinate (strict
// shift already applied, simulator.hpp:202).
template <int KIND>
__device__ __forceinline__ outcome<int> map_block(const Geom& g, int wx, int wy, int wz) {
    outcome<int> o;
    if (KIND == SMX_H2D) o = map_h2d<int>(wx, wy);
    else if (KIND == SMX_H3D) o = map_h3d<int>(wx, wy, wz, g.n);
    else o = map_bb<int>(wx, wy, wz, g.n, g.dims);
    if (KIND != SMX_BB) o.y -= 1;
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

