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
//   map_rb_2d             maps.hpp:120-141       (comparison map)
//   map_lambda_2d         maps.hpp:145-159, core.hpp:151-156 (comparison map)
//   map_h2d_padded        maps.hpp:209-222       (general n)
//   decompose_trapezoids  maps.hpp:224-267, map_h2d_trapezoid :269-281
// Argument validation (the reference's std::invalid_argument paths) lives in
// the callers: the C ABI validates grids once per launch; kernels only ever see
// in-range block coordinates.
#pragma once

#include <math.h>
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

// ---- general-n and comparison 2-D maps ----

SMX_HD uint64_t pow2_floor(uint64_t v) { return uint64_t(1) << floor_log2_u64(v); }
SMX_HD int ceil_log2_u64(uint64_t v) { return v == 1 ? 0 : floor_log2_u64(v - 1) + 1; }
SMX_HD uint64_t pow2_ceil(uint64_t v) { return uint64_t(1) << ceil_log2_u64(v); }

// RB: the rectangle (n/2, n+1) for even n, ((n+1)/2, n) for odd n, folded onto
// T(n) (with-diagonal view): the point-reflected upper part, and for even n the
// extra column w_y = n onto the main diagonal's tail. Never Void.
template <class I>
SMX_HD outcome<I> map_rb(I wx, I wy, I n) {
    if (n % 2 == 0 && wy == n) return {0, n / 2, n / 2 + wx, 0, 1, 0};
    if (wx <= wy) return {0, wx, wy, 0, 1, 0};
    return {0, n - wx, n - 1 - wy, 0, 1, 0};
}

// lambda: the linear block index of T(n) -> (x, y) by the quadratic root with
// an exact integer fix-up (core.hpp:151-156). Never Void.
SMX_HD void tri_coord_at(uint64_t index, int64_t* x, int64_t* y) {
    int64_t r = int64_t((sqrt(8.0 * double(index) + 1.0) - 1.0) / 2.0);
    while (r > 0 && tri_index(0, r) > index) --r;
    while (tri_index(0, r + 1) <= index) ++r;
    *x = int64_t(index - tri_index(0, r));
    *y = r;
}
template <class I>
SMX_HD outcome<I> map_lambda(uint64_t index) {
    int64_t x, y;
    tri_coord_at(index, &x, &y);
    return {0, I(x), I(y), 0, 1, 0};
}

// H padded from above: the power-of-two grid h2d(2^ceil(log2 n)); blocks whose
// strict-view row is beyond n - 1 are Void.
template <class I>
SMX_HD outcome<I> map_h2d_padded(I wx, I wy, I n) {
    outcome<I> o = map_h2d<I>(wx, wy);
    if (o.y > n - 1) return {1, 0, 0, 0, 1, 0};
    return o;
}

// One band of the concurrent-trapezoid scheme (trapezoid_params, maps.hpp:49-60).
template <class I>
struct trapezoid {
    I delta_x, delta_y;
    I band;        // power-of-two triangle side of this band
    I h1, h2;      // last unfolded row; rows of the band-wide box
    I grid_width;  // band / 2
    I valid_side;  // rows beyond are Void (final padded band only)
    I ext_x, ext_y;
};

// decompose_trapezoids (maps.hpp:228-257): greedy peel of power-of-two bands
// from the left; the last remainder is padded from above once the padding
// drops below T. Writes at most `max` bands, returns the count (or -1 when
// more would be needed; never for n < 2^63). Requires n >= 2, T >= 1.
SMX_HD int decompose_trapezoids(int64_t n, int64_t T, trapezoid<int64_t>* out, int max) {
    int cnt = 0;
    int64_t c = 0, r = n;
    while (r >= 2) {
        const int64_t pad = int64_t(pow2_ceil(uint64_t(r))) - r;
        trapezoid<int64_t> t;
        t.delta_x = t.delta_y = c;
        if (pad < T) {
            t.band = int64_t(pow2_ceil(uint64_t(r)));
            t.h2 = 0;
            t.valid_side = r;
        } else {
            t.band = int64_t(pow2_floor(uint64_t(r)));
            t.h2 = r - t.band;
            t.valid_side = t.band;
        }
        t.h1 = t.band + t.h2 - 2;
        t.grid_width = t.band / 2;
        t.ext_x = t.grid_width;
        t.ext_y = t.band - 1 + 2 * t.h2;
        if (cnt == max) return -1;
        out[cnt++] = t;
        if (pad < T) break;
        c += t.band;
        r -= t.band;
    }
    return cnt;
}

// map_h2d_trapezoid (maps.hpp:269-281): the H2D map of the band's triangle,
// rows beyond h1 fold the band-wide box's second half (k = 1) beside the first.
template <class I>
SMX_HD outcome<I> map_h2d_trapezoid(I wx, I wy, const trapezoid<I>& p) {
    const int lg = floor_log2<I>(wy + 1);
    const I q = wx >> lg;
    const I k = wy > p.h1 ? 1 : 0;
    const I x = p.delta_x + wx + (q << lg) + k * p.grid_width;
    const I y = p.delta_y + wy - k * p.h2 + (q << (lg + 1)) + 1;
    if (p.h2 == 0 && y - p.delta_y > p.valid_side - 1) return {1, 0, 0, 0, 1, 0};
    return {0, x, y, 0, I(1) << lg, q};
}

}  // namespace smx
