// smx_maps.hpp — the block-space map arithmetic, written ONCE and compiled for
// both sides of the boundary: nvcc inlines it into the sm_100a kernels
// (paper_2208_11617_b200/csrc/*.cu) and g++ uses it for the host drop-in
// (include/simplexmap_b200.hpp). Integer type I is int32_t on the device (every
// BASELINE grid keeps block and tile coordinates < 2^17) and int64_t on the host,
// matching the reference's i64 API.
//
// Semantics restated from the reference (arXiv 2208.11617 `simplexmap`):
//   floor_log2            bits.hpp:22-25
//   tri/tet membership    core.hpp:63-69
//   packed linearisers    core.hpp:136-149
//   map_bb                maps.hpp:107-116
//   map_h2d               maps.hpp:200-207
//   map_h3d               maps.hpp:302-337
// Argument validation (the reference's std::invalid_argument paths) lives in
// the callers: the C ABI validates grids once per launch; kernels only ever see
// in-range block coordinates.
#pragma once

#include <stdint.h>

#if defined(__CUDACC__)
#define SMX_HD __host__ __device__ __forceinline__
#else
#define SMX_HD inline
#endif

namespace smx {

template <class I>
struct outcome {
    I is_void;
    I x, y, z;     // target block (strict view for h2d/h3d: y is one above the
                   // with-diagonal row; the launch engine applies y-1)
    I level_b;     // stack level b (power of two)
    I index_q;     // orthotope index q at level b
};

SMX_HD int floor_log2_u32(uint32_t v) {
#if defined(__CUDA_ARCH__)
    return 31 - __clz(v);  // one FLO.U32
#else
    return 31 - __builtin_clz(v);
#endif
}

SMX_HD int floor_log2_u64(uint64_t v) {
#if defined(__CUDA_ARCH__)
    return 63 - __clzll(v);
#else
    return 63 - __builtin_clzll(v);
#endif
}

template <class I>
SMX_HD int floor_log2(I v) {
    if (sizeof(I) <= 4) return floor_log2_u32(uint32_t(v));
    return floor_log2_u64(uint64_t(v));
}

SMX_HD bool is_pow2(uint64_t v) { return v != 0 && (v & (v - 1)) == 0; }

// ---- geometry ----
template <class I>
SMX_HD bool tri_contains(I side, I x, I y) { return 0 <= x && x <= y && y <= side - 1; }
template <class I>
SMX_HD bool tet_contains(I side, I x, I y, I z) {
    return 0 <= x && x <= y && z >= 0 && y <= side - 1 - z;
}

SMX_HD uint64_t tri_cells(int64_t side) {
    return side < 1 ? 0 : uint64_t(side) * uint64_t(side + 1) / 2;
}
SMX_HD uint64_t tet_cells(int64_t side) {
    if (side < 1) return 0;
    uint64_t a = uint64_t(side), b = a + 1, c = a + 2;
    if (a % 2 == 0) a /= 2; else b /= 2;
    if (a % 3 == 0) a /= 3; else if (b % 3 == 0) b /= 3; else c /= 3;
    return a * b * c;
}
SMX_HD uint64_t tri_index(int64_t x, int64_t y) {
    return uint64_t(y) * uint64_t(y + 1) / 2 + uint64_t(x);
}
// tet_layer_prefix(S, z) = tet(S) - tet(S - z): the packed offset of layer z.
SMX_HD uint64_t tet_layer_prefix(int64_t side, int64_t z) {
    if (z <= 0) return 0;
    return tet_cells(side) - (z >= side ? 0 : tet_cells(side - z));
}
SMX_HD uint64_t tet_index(int64_t side, int64_t x, int64_t y, int64_t z) {
    return tet_layer_prefix(side, z) + tri_index(x, y);
}

// ---- maps ----

// BB: the n^m box; blocks outside the with-diagonal view are Void.
template <class I>
SMX_HD outcome<I> map_bb(I wx, I wy, I wz, I n, int m) {
    bool member = m == 2 ? tri_contains<I>(n, wx, wy) : tet_contains<I>(n, wx, wy, wz);
    if (!member) return {1, 0, 0, 0, 1, 0};
    return {0, wx, wy, wz, 1, 0};
}

// H, 2-simplex: b = 2^floor(log2(wy+1)), q = wx >> log2 b,
// target (wx + q b, wy + 2 q b + 1) in the strict view. Never Void.
template <class I>
SMX_HD outcome<I> map_h2d(I wx, I wy) {
    const int lg = floor_log2<I>(wy + 1);
    const I q = wx >> lg;
    return {0, wx + (q << lg), wy + (q << (lg + 1)) + 1, 0, I(1) << lg, q};
}

// H, 3-simplex (n a power of two >= 4). Grid (n/2, n/2, ceil(3(n-1)/4)).
// (i) wz < n/2: the major cube of side s = n/2, displaced one row up
//     (anchor = 1); (ii) wz >= n/2: slab level s = 2^floor(log2(wy+1)),
//     Void when s > n/4 or wz - n/2 >= s; q-th replica along x at a = 2qs;
// (iii) images deeper than 2s-1 fold: the anchored cube's facet layer lands
//     on the wall plane y = a + s, everything else transposes through the
//     hinge (a + ly + lz - s, a + lz, s - lz + lx).
template <class I>
SMX_HD outcome<I> map_h3d(I wx, I wy, I wz, I n) {
    const I nh = n >> 1;
    I s, a, q, lx, ly, lz, anchor;
    if (wz < nh) {
        s = nh; a = 0; q = 0; lx = wx; ly = wy; lz = wz; anchor = 1;
    } else {
        const int lg = floor_log2<I>(wy + 1);
        s = I(1) << lg;
        lz = wz - nh;
        if (s > (n >> 2) || lz >= s) return {1, 0, 0, 0, 1, 0};
        q = wx >> lg;
        a = q << (lg + 1);
        lx = wx - (q << lg);
        ly = wy - (s - 1);
        anchor = 0;
    }
    const I x = a + lx, y = a + s + anchor + ly, z = lz;
    const I depth = (y - a) + z;
    if (depth <= 2 * s - 1) return {0, x, y, z, s, q};
    if (anchor == 1 && depth == 2 * s) return {0, x, a + s, z, s, q};
    return {0, a + ly + lz - s, a + lz, s - lz + lx, s, q};
}

}  // namespace smx
