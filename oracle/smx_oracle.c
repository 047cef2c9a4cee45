/*
 * TEST INFRASTRUCTURE ONLY — the CPU checker. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load this library; the product
 * (paper_2208_11617_b200/, include/) never links, loads or calls it.
 *
 * A plain-C restatement of the reference's hot path (arXiv 2208.11617 reference,
 * /root/reference/proj/include/simplexmap/{bits,core,maps,simulator}.hpp). Each function cites the
 * reference lines it restates. It exists for two reasons:
 *   1. a second, independently written implementation of the map arithmetic,
 *      pinned against the reference itself (oracle/_ref, built from the
 *      unmodified headers) and the golden vectors in tests/golden/;
 *   2. a FAST multithreaded 3-D Life oracle: the reference's kernel_ca_run runs
 *      at ~0.25 M cell-steps/s (each neighbour read recomputes tet layer
 *      prefixes through 128-bit divisions, core.hpp:140-149 -> :81-97), which
 *      makes the BASELINE configs C4 (100 steps, 179 M cells) and C5 (1.4 G
 *      cells) infeasible. The row-sweep restatement below is bit-identical to
 *      kernel_ca_run (checked in tests/test_oracle.py at sides 7..255 against
 *      oracle/_ref and against the SURVEY Appendix-A hashes).
 *
 * Status codes: 0 ok, 1 invalid argument (the reference throws
 * std::invalid_argument), 2 overflow.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef uint64_t u64;
typedef int64_t i64;
typedef uint32_t u32;
typedef uint8_t u8;

enum { K_BB = 0, K_RB = 1, K_LAMBDA = 2, K_H2D = 3, K_TRAP = 4, K_PADDED = 5, K_H3D = 6 };

/* bits.hpp:22-25 — floor(log2 v) = 63 - clz(v); v >= 1 */
static int floor_log2(u64 v) { return 63 - __builtin_clzll(v); }
/* bits.hpp:42-44 */
static int is_pow2(u64 v) { return v != 0 && (v & (v - 1)) == 0; }

/* core.hpp:105-114 / :125-133 — C(n+m-1, m) for m = 2, 3 in exact u64 (the
 * reference uses a 192-bit mul-div; every side used here keeps the products
 * well inside 64 bits). */
u64 orc_tri_cells(i64 side) { return side < 1 ? 0 : (u64)side * (u64)(side + 1) / 2; }
u64 orc_tet_cells(i64 side) {
    if (side < 1) return 0;
    u64 a = (u64)side, b = (u64)side + 1, c = (u64)side + 2;
    /* a*b*c is divisible by 6; divide early to stay inside 64 bits */
    if (a % 2 == 0) a /= 2; else b /= 2;
    if (a % 3 == 0) a /= 3; else if (b % 3 == 0) b /= 3; else c /= 3;
    return a * b * c;
}
/* core.hpp:136-149 */
static u64 tri_index(i64 x, i64 y) { return (u64)y * (u64)(y + 1) / 2 + (u64)x; }
u64 orc_tet_layer_prefix(i64 side, i64 z) {
    if (z == 0) return 0;
    u64 full = orc_tet_cells(side);
    u64 rest = z >= side ? 0 : orc_tet_cells(side - z);
    return full - rest;
}
/* core.hpp:63-69 */
static int tri_contains(i64 side, i64 x, i64 y) { return 0 <= x && x <= y && y <= side - 1; }
static int tet_contains(i64 side, i64 x, i64 y, i64 z) {
    return 0 <= x && x <= y && z >= 0 && y <= side - 1 - z;
}

/* ---- grids: maps.hpp:96-105 (bb), :188-198 (h2d), :285-295 (h3d) ---- */
int orc_grid(int kind, int m, i64 n, i64* ext3) {
    if (kind == K_BB) {
        if (m != 2 && m != 3) return 1;
        if (n < 1) return 1;
        ext3[0] = n; ext3[1] = n; ext3[2] = m == 3 ? n : 1;
        return 0;
    }
    if (kind == K_H2D) {
        if (m != 2 || n < 2 || !is_pow2((u64)n)) return 1;
        ext3[0] = n / 2; ext3[1] = n - 1; ext3[2] = 1;
        return 0;
    }
    if (kind == K_H3D) {
        if (m != 3 || n < 4 || !is_pow2((u64)n)) return 1;
        ext3[0] = n / 2; ext3[1] = n / 2; ext3[2] = (3 * (n - 1) + 3) / 4;
        return 0;
    }
    return 1;
}

/* grid_spec::domain_side (maps.hpp:91): strict views (h2d, h3d) cover side n-1 */
i64 orc_domain_side(int kind, i64 n) { return kind == K_BB ? n : n - 1; }

/* out6 = {is_void, x, y, z, level_b, index_q} — map_outcome (maps.hpp:40-47) */
static void put(i64* o, i64 v, i64 x, i64 y, i64 z, i64 b, i64 q) {
    o[0] = v; o[1] = x; o[2] = y; o[3] = z; o[4] = b; o[5] = q;
}

/* maps.hpp:107-116 */
int orc_map_bb(i64 x, i64 y, i64 z, i64 n, int m, i64* o) {
    if (m != 2 && m != 3) return 1;
    int in = x >= 0 && x < n && y >= 0 && y < n && (m == 2 ? z == 0 : (z >= 0 && z < n));
    if (!in) return 1;
    int member = m == 2 ? tri_contains(n, x, y) : tet_contains(n, x, y, z);
    if (!member) put(o, 1, 0, 0, 0, 1, 0);
    else put(o, 0, x, y, z, 1, 0);
    return 0;
}

/* maps.hpp:200-207 */
int orc_map_h2d(i64 x, i64 y, i64* o) {
    if (x < 0 || y < 0) return 1;
    int lg = floor_log2((u64)y + 1);
    i64 b = (i64)1 << lg;
    i64 q = x >> lg;
    put(o, 0, x + (q << lg), y + (q << (lg + 1)) + 1, 0, b, q);
    return 0;
}

/* maps.hpp:302-337 — restated case by case: (i) displaced major cube,
 * (ii) power-of-two slab levels with the two Void rules, (iii) the fold:
 * wall plane for the anchored cube's facet layer, hinge transpose otherwise. */
int orc_map_h3d(i64 wx, i64 wy, i64 wz, i64 n, i64* o) {
    if (n < 4 || !is_pow2((u64)n)) return 1;
    if (wx < 0 || wx >= n / 2 || wy < 0 || wy >= n / 2 || wz < 0 || wz >= (3 * (n - 1) + 3) / 4)
        return 1;
    const i64 nh = n / 2;
    i64 s, a, q, lx, ly, lz, anchor;
    if (wz < nh) {
        s = nh; a = 0; q = 0; lx = wx; ly = wy; lz = wz; anchor = 1;
    } else {
        int lg = floor_log2((u64)wy + 1);
        s = (i64)1 << lg;
        if (s > n / 4 || wz - nh >= s) { put(o, 1, 0, 0, 0, 1, 0); return 0; }
        q = wx >> lg;
        a = q << (lg + 1);
        lx = wx - (q << lg);
        ly = wy - (s - 1);
        lz = wz - nh;
        anchor = 0;
    }
    i64 x = a + lx, y = a + s + anchor + ly, z = lz;
    i64 depth = (y - a) + z;
    if (depth <= 2 * s - 1) put(o, 0, x, y, z, s, q);
    else if (anchor == 1 && depth == 2 * s) put(o, 0, x, a + s, z, s, q);
    else put(o, 0, a + ly + lz - s, a + lz, s - lz + lx, s, q);
    return 0;
}

static int map_any(int kind, int m, i64 n, i64 x, i64 y, i64 z, i64* o) {
    if (kind == K_BB) return orc_map_bb(x, y, z, n, m, o);
    if (kind == K_H2D) return orc_map_h2d(x, y, o);
    if (kind == K_H3D) return orc_map_h3d(x, y, z, n, o);
    return 1;
}

/* All block outcomes in natural z, y, x order (simulator.hpp:113-118). */
int orc_map_outcomes(int kind, int m, i64 n, i64* out, u64 count) {
    i64 e[3];
    if (orc_grid(kind, m, n, e)) return 1;
    if ((u64)(e[0] * e[1] * e[2]) != count) return 1;
    u64 i = 0;
    for (i64 z = 0; z < e[2]; ++z)
        for (i64 y = 0; y < e[1]; ++y)
            for (i64 x = 0; x < e[0]; ++x)
                if (map_any(kind, m, n, x, y, z, out + 6 * i++)) return 1;
    return 0;
}

/* detail::sweep (simulator.hpp:177-218) restated: block walk -> map -> Void
 * filter -> strict y-1 shift -> rho^m local cells -> membership -> packed index.
 * coverage (nullable) gets ++ per useful cell (simulator.hpp:290-294); cells32
 * (nullable) gets ++ per useful cell (launch_accum, :320-323).
 * counters: {blocks, void, threads, useful}. */
int orc_sweep(int kind, int m, i64 n, i64 rho, u32* coverage, u32* cells32, u64* counters) {
    i64 e[3];
    if (rho < 1 || orc_grid(kind, m, n, e)) return 1;
    const int is3d = m == 3;
    const int strict = kind != K_BB;
    const i64 side = orc_domain_side(kind, n) * rho;
    const u64 tpb = is3d ? (u64)(rho * rho * rho) : (u64)(rho * rho);
    u64 c[4] = {0, 0, 0, 0};
    for (i64 wz = 0; wz < e[2]; ++wz)
        for (i64 wy = 0; wy < e[1]; ++wy)
            for (i64 wx = 0; wx < e[0]; ++wx) {
                i64 o[6];
                if (map_any(kind, m, n, wx, wy, wz, o)) return 1;
                c[0]++;
                c[2] += tpb;
                if (o[0]) { c[1]++; continue; }
                i64 dx = o[1], dy = o[2] - (strict ? 1 : 0), dz = o[3];
                for (i64 lz = 0; lz < (is3d ? rho : 1); ++lz)
                    for (i64 ly = 0; ly < rho; ++ly)
                        for (i64 lx = 0; lx < rho; ++lx) {
                            i64 cx = dx * rho + lx, cy = dy * rho + ly, cz = dz * rho + lz;
                            int member = is3d ? tet_contains(side, cx, cy, cz)
                                              : tri_contains(side, cx, cy);
                            if (!member) continue;
                            u64 idx = (is3d ? orc_tet_layer_prefix(side, cz) : 0) + tri_index(cx, cy);
                            c[3]++;
                            if (coverage) coverage[idx]++;
                            if (cells32) cells32[idx]++;
                        }
            }
    if (counters) memcpy(counters, c, sizeof c);
    return 0;
}

/* ---- general-n and comparison 2-D maps ---- */

/* bits.hpp:28-40 */
static u64 pow2_floor(u64 v) { return (u64)1 << floor_log2(v); }
static u64 pow2_ceil(u64 v) { return v == 1 ? 1 : (u64)1 << (floor_log2(v - 1) + 1); }

/* trapezoid_params (maps.hpp:49-60) */
typedef struct { i64 dx, dy, band, h1, h2, gw, vside, ex, ey; } trap_t;

/* decompose_trapezoids (maps.hpp:228-257): peel the largest power-of-two band
 * from the left while padding the remainder from above would cost >= T rows;
 * then pad the last remainder. */
static int decompose(i64 n, i64 T, trap_t* t, int max) {
    if (n < 2 || T < 1) return -1;
    int cnt = 0;
    i64 c = 0, r = n;
    while (r >= 2) {
        i64 pad = (i64)pow2_ceil((u64)r) - r;
        trap_t b;
        b.dx = b.dy = c;
        if (pad < T) { b.band = (i64)pow2_ceil((u64)r); b.h2 = 0; b.vside = r; }
        else { b.band = (i64)pow2_floor((u64)r); b.h2 = r - b.band; b.vside = b.band; }
        b.h1 = b.band + b.h2 - 2;
        b.gw = b.band / 2;
        b.ex = b.gw;
        b.ey = b.band - 1 + 2 * b.h2;
        if (cnt == max) return -1;
        t[cnt++] = b;
        if (pad < T) break;
        c += b.band;
        r -= b.band;
    }
    return cnt;
}

int orc_decompose_trapezoids(i64 n, i64 T, i64* out9, int max, int* count) {
    trap_t t[64];
    int c = decompose(n, T, t, 64);
    if (c < 0) return 1;
    *count = c;
    for (int i = 0; i < c && i < max; ++i) {
        i64* r = out9 + 9 * i;
        r[0] = t[i].dx; r[1] = t[i].dy; r[2] = t[i].band; r[3] = t[i].h1; r[4] = t[i].h2;
        r[5] = t[i].gw; r[6] = t[i].vside; r[7] = t[i].ex; r[8] = t[i].ey;
    }
    return 0;
}

/* maps.hpp:133-141 — fold of the (n/2 x n+1) or ((n+1)/2 x n) rectangle onto T(n) */
int orc_map_rb(i64 x, i64 y, i64 n, i64* o) {
    if (n < 1) return 1;
    i64 ex = n % 2 == 0 ? n / 2 : (n + 1) / 2, ey = n % 2 == 0 ? n + 1 : n;
    if (x < 0 || x >= ex || y < 0 || y >= ey) return 1;
    if (n % 2 == 0 && y == n) put(o, 0, n / 2, n / 2 + x, 0, 1, 0);
    else if (x <= y) put(o, 0, x, y, 0, 1, 0);
    else put(o, 0, n - x, n - 1 - y, 0, 1, 0);
    return 0;
}

/* integer floor(sqrt(v)) by Newton steps (independent of the reference's
 * floating-point root + fix-up, core.hpp:151-156; same result for all v) */
static u64 isqrt_u64(u64 v) {
    if (v < 2) return v;
    u64 r = (u64)1 << ((64 - __builtin_clzll(v) + 1) / 2);
    for (;;) {
        u64 nr = (r + v / r) / 2;
        if (nr >= r) break;
        r = nr;
    }
    while (r * r > v) --r;
    while ((r + 1) * (r + 1) <= v) ++r;
    return r;
}

/* maps.hpp:156-159 — linear block index -> (x, y): y = floor((isqrt(8i+1)-1)/2) */
int orc_map_lambda(u64 index, i64 n, i64* o) {
    if (index >= orc_tri_cells(n)) return 1;
    i64 y = (i64)((isqrt_u64(8 * index + 1) - 1) / 2);
    put(o, 0, (i64)(index - tri_index(0, y)), y, 0, 1, 0);
    return 0;
}

/* maps.hpp:219-222 — h2d of the power-of-two cover, rows beyond n-1 Void */
int orc_map_padded(i64 x, i64 y, i64 n, i64* o) {
    if (orc_map_h2d(x, y, o)) return 1;
    if (o[2] > n - 1) put(o, 1, 0, 0, 0, 1, 0);
    return 0;
}

/* maps.hpp:269-281 */
static int map_trap(i64 x, i64 y, const trap_t* p, i64* o) {
    if (x < 0 || x >= p->ex || y < 0 || y >= p->ey) return 1;
    int lg = floor_log2((u64)y + 1);
    i64 b = (i64)1 << lg, q = x >> lg, k = y > p->h1 ? 1 : 0;
    i64 tx = p->dx + x + (q << lg) + k * p->gw;
    i64 ty = p->dy + y - k * p->h2 + (q << (lg + 1)) + 1;
    if (p->h2 == 0 && ty - p->dy > p->vside - 1) put(o, 1, 0, 0, 0, 1, 0);
    else put(o, 0, tx, ty, 0, b, q);
    return 0;
}

int orc_map_trapezoid(i64 n, i64 T, int band, i64 x, i64 y, i64* o) {
    trap_t t[64];
    int c = decompose(n, T, t, 64);
    if (c < 0 || band < 0 || band >= c) return 1;
    return map_trap(x, y, &t[band], o);
}

/* A grid as the reference walks it (simulator.hpp:109-158): one sub-grid, or
 * one per trapezoid band in order. */
typedef struct { i64 e[3]; int band; } sub_t;

static int subs_of(int kind, int m, i64 n, i64 T, sub_t* s, trap_t* t, int* ns) {
    if (kind == K_TRAP) {
        if (m != 2) return 1;
        int c = decompose(n, T, t, 64);
        if (c < 0) return 1;
        for (int i = 0; i < c; ++i) { s[i].e[0] = t[i].ex; s[i].e[1] = t[i].ey; s[i].e[2] = 1; s[i].band = i; }
        *ns = c;
        return 0;
    }
    s[0].band = -1;
    *ns = 1;
    if (kind == K_RB) {          /* maps.hpp:120-128 */
        if (m != 2 || n < 1) return 1;
        s[0].e[0] = n % 2 == 0 ? n / 2 : (n + 1) / 2; s[0].e[1] = n % 2 == 0 ? n + 1 : n; s[0].e[2] = 1;
        return 0;
    }
    if (kind == K_LAMBDA) {      /* maps.hpp:145-152 */
        if (m != 2 || n < 1) return 1;
        s[0].e[0] = (i64)orc_tri_cells(n); s[0].e[1] = 1; s[0].e[2] = 1;
        return 0;
    }
    if (kind == K_PADDED) {      /* maps.hpp:211-217 */
        if (m != 2 || n < 2) return 1;
        i64 p2 = (i64)pow2_ceil((u64)n);
        s[0].e[0] = p2 / 2; s[0].e[1] = p2 - 1; s[0].e[2] = 1;
        return 0;
    }
    return orc_grid(kind, m, n, s[0].e);
}

static int strict_kind(int kind) { return kind == K_H2D || kind == K_TRAP || kind == K_PADDED || kind == K_H3D; }

static int map_at(int kind, int m, i64 n, const trap_t* t, int band, i64 x, i64 y, i64 z, i64* o) {
    switch (kind) {
        case K_RB: return orc_map_rb(x, y, n, o);
        case K_LAMBDA: return orc_map_lambda((u64)x, n, o);
        case K_PADDED: return orc_map_padded(x, y, n, o);
        case K_TRAP: return map_trap(x, y, &t[band], o);
        default: return map_any(kind, m, n, x, y, z, o);
    }
}

u64 orc_grid_blocks(int kind, int m, i64 n, i64 T) {
    sub_t s[64]; trap_t t[64]; int ns = 0;
    if (subs_of(kind, m, n, T, s, t, &ns)) return 0;
    u64 b = 0;
    for (int i = 0; i < ns; ++i) b += (u64)(s[i].e[0] * s[i].e[1] * s[i].e[2]);
    return b;
}

/* every block of any grid kind in the reference's emission order */
int orc_map_outcomes_t(int kind, int m, i64 n, i64 T, i64* out, u64 count) {
    sub_t s[64]; trap_t t[64]; int ns = 0;
    if (subs_of(kind, m, n, T, s, t, &ns)) return 1;
    u64 i = 0;
    for (int k = 0; k < ns; ++k)
        for (i64 z = 0; z < s[k].e[2]; ++z)
            for (i64 y = 0; y < s[k].e[1]; ++y)
                for (i64 x = 0; x < s[k].e[0]; ++x) {
                    if (i >= count) return 1;
                    if (map_at(kind, m, n, t, s[k].band, x, y, z, out + 6 * i++)) return 1;
                }
    return i == count ? 0 : 1;
}

/* detail::sweep (simulator.hpp:177-218) for any 2-D/3-D grid kind (see orc_sweep) */
int orc_sweep_t(int kind, int m, i64 n, i64 rho, i64 T, u32* coverage, u32* cells32, u64* counters) {
    sub_t s[64]; trap_t t[64]; int ns = 0;
    if (rho < 1 || subs_of(kind, m, n, T, s, t, &ns)) return 1;
    const int is3d = m == 3;
    const int strict = strict_kind(kind);
    const i64 side = (strict ? n - 1 : n) * rho;
    const u64 tpb = is3d ? (u64)(rho * rho * rho) : (u64)(rho * rho);
    u64 c[4] = {0, 0, 0, 0};
    for (int k = 0; k < ns; ++k)
        for (i64 wz = 0; wz < s[k].e[2]; ++wz)
            for (i64 wy = 0; wy < s[k].e[1]; ++wy)
                for (i64 wx = 0; wx < s[k].e[0]; ++wx) {
                    i64 o[6];
                    if (map_at(kind, m, n, t, s[k].band, wx, wy, wz, o)) return 1;
                    c[0]++;
                    c[2] += tpb;
                    if (o[0]) { c[1]++; continue; }
                    i64 dx = o[1], dy = o[2] - (strict ? 1 : 0), dz = o[3];
                    for (i64 lz = 0; lz < (is3d ? rho : 1); ++lz)
                        for (i64 ly = 0; ly < rho; ++ly)
                            for (i64 lx = 0; lx < rho; ++lx) {
                                i64 cx = dx * rho + lx, cy = dy * rho + ly, cz = dz * rho + lz;
                                int member = is3d ? tet_contains(side, cx, cy, cz) : tri_contains(side, cx, cy);
                                if (!member) continue;
                                u64 idx = (is3d ? orc_tet_layer_prefix(side, cz) : 0) + tri_index(cx, cy);
                                c[3]++;
                                if (coverage) coverage[idx]++;
                                if (cells32) cells32[idx]++;
                            }
                }
    if (counters) memcpy(counters, c, sizeof c);
    return 0;
}

/* bits.hpp:84-89, :96-109 */
static u64 splitmix64(u64* s) {
    u64 z = (*s += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
static u64 fnv1a_u64(u64 h, u64 v) {
    for (int i = 0; i < 8; ++i) {
        h ^= (v >> (8 * i)) & 0xffu; /* little-endian byte order of the u64 */
        h *= 0x100000001b3ull;
    }
    return h;
}

/* simulator.hpp:68-73 — FNV-1a over u64 m, u64 side, then the raw cell bytes */
u64 orc_state_hash(int m, i64 side, const void* bytes, u64 nbytes) {
    u64 h = 0xcbf29ce484222325ull;
    h = fnv1a_u64(h, (u64)m);
    h = fnv1a_u64(h, (u64)side);
    const u8* p = (const u8*)bytes;
    for (u64 i = 0; i < nbytes; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ull;
    }
    return h;
}

/* ---------------- threaded helpers ---------------- */

typedef struct {
    void (*fn)(void* ctx, i64 item);
    void* ctx;
    i64 count;
    i64 next; /* atomically claimed */
} pool_t;

static void* pool_worker(void* arg) {
    pool_t* p = (pool_t*)arg;
    for (;;) {
        i64 it = __atomic_fetch_add(&p->next, 1, __ATOMIC_RELAXED);
        if (it >= p->count) break;
        p->fn(p->ctx, it);
    }
    return NULL;
}

static void run_pool(void (*fn)(void*, i64), void* ctx, i64 count, int nthreads) {
    pool_t p = {fn, ctx, count, 0};
    if (nthreads <= 1 || count <= 1) {
        for (i64 i = 0; i < count; ++i) fn(ctx, i);
        return;
    }
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    int started = 0;
    for (int t = 0; t < nthreads; ++t)
        if (pthread_create(&th[t], NULL, pool_worker, &p) == 0) ++started;
    if (started == 0) pool_worker(&p);
    for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
}

/* make_life_state (simulator.hpp:390-398): alive iff
 * splitmix64(fnv1a_append_u64(seed, i)) >> 62 == 0, keyed by packed index i. */
typedef struct { u64 seed; u8* out; u64 n; u64 chunk; } life_ctx;
static void life_chunk(void* vc, i64 it) {
    life_ctx* c = (life_ctx*)vc;
    u64 lo = (u64)it * c->chunk, hi = lo + c->chunk;
    if (hi > c->n) hi = c->n;
    for (u64 i = lo; i < hi; ++i) {
        u64 key = fnv1a_u64(c->seed, i);
        c->out[i] = (splitmix64(&key) >> 62) == 0 ? 1 : 0;
    }
}
int orc_make_life_state(int m, i64 side, u64 seed, u8* out, u64 ncells, int nthreads) {
    if ((m != 2 && m != 3) || side < 1) return 1;
    u64 want = m == 2 ? orc_tri_cells(side) : orc_tet_cells(side);
    if (want != ncells) return 1;
    life_ctx c = {seed, out, ncells, 1u << 20};
    run_pool(life_chunk, &c, (i64)((ncells + c.chunk - 1) / c.chunk), nthreads);
    return 0;
}

/* life_next (simulator.hpp:220-223): B3/S23 */
static u8 life_next(u8 alive, int nb) {
    if (alive) return (nb == 2 || nb == 3) ? 1 : 0;
    return nb == 3 ? 1 : 0;
}

/* Literal per-cell restatement of alive_neighbors_3d_dead (simulator.hpp:242-253)
 * driven by kernel_ca_run's z, y, x loop (:417-422). Slow; used to pin the fast
 * row sweep below on small sides. */
int orc_ca3d_run_literal(i64 side, i64 steps, u8* cells, u64 ncells) {
    if (side < 1 || steps < 0 || orc_tet_cells(side) != ncells) return 1;
    u8* next = (u8*)calloc(ncells ? ncells : 1, 1);
    if (!next) return 2;
    for (i64 st = 0; st < steps; ++st) {
        for (i64 z = 0; z < side; ++z)
            for (i64 y = 0; y + z < side; ++y)
                for (i64 x = 0; x <= y; ++x) {
                    int count = 0;
                    for (i64 dz = -1; dz <= 1; ++dz)
                        for (i64 dy = -1; dy <= 1; ++dy)
                            for (i64 dx = -1; dx <= 1; ++dx) {
                                if (!dx && !dy && !dz) continue;
                                i64 nx = x + dx, ny = y + dy, nz = z + dz;
                                if (tet_contains(side, nx, ny, nz))
                                    count += cells[orc_tet_layer_prefix(side, nz) + tri_index(nx, ny)];
                            }
                    u64 idx = orc_tet_layer_prefix(side, z) + tri_index(x, y);
                    next[idx] = life_next(cells[idx], count);
                }
        memcpy(cells, next, ncells);
    }
    free(next);
    return 0;
}

/* Fast restatement: the same neighbour set, evaluated row by row. For output
 * row (y, z) the 9 source rows (y+dy, z+dz) exist iff tet_contains admits some
 * x there (z' >= 0, y' >= 0, y' + z' <= side-1); inside a source row the
 * admissible x' are [0, y'] — exactly tet_contains (core.hpp:67-69). The
 * centre is included in the 27-sum and subtracted again. */
typedef struct { i64 side; const u8* cur; u8* next; const u64* prefix; } ca_ctx;
static void ca_layer(void* vc, i64 z) {
    ca_ctx* c = (ca_ctx*)vc;
    const i64 S = c->side;
    int cnt[1 << 16];
    int* count = (S + 2 <= (1 << 16)) ? cnt : (int*)malloc(sizeof(int) * (size_t)(S + 2));
    for (i64 y = 0; y + z < S; ++y) {
        for (i64 x = 0; x <= y; ++x) count[x] = 0;
        for (i64 dz = -1; dz <= 1; ++dz) {
            i64 zz = z + dz;
            if (zz < 0 || zz >= S) continue;
            for (i64 dy = -1; dy <= 1; ++dy) {
                i64 yy = y + dy;
                if (yy < 0 || yy + zz > S - 1) continue;
                const u8* r = c->cur + c->prefix[zz] + tri_index(0, yy);
                for (i64 x = 0; x <= y; ++x) {
                    int s = 0;
                    if (x - 1 >= 0 && x - 1 <= yy) s += r[x - 1];
                    if (x <= yy) s += r[x];
                    if (x + 1 <= yy) s += r[x + 1];
                    count[x] += s;
                }
            }
        }
        const u8* me = c->cur + c->prefix[z] + tri_index(0, y);
        u8* out = c->next + c->prefix[z] + tri_index(0, y);
        for (i64 x = 0; x <= y; ++x) out[x] = life_next(me[x], count[x] - me[x]);
    }
    if (count != cnt) free(count);
}

int orc_ca3d_run(i64 side, i64 steps, u8* cells, u64 ncells, int nthreads) {
    if (side < 1 || steps < 0 || orc_tet_cells(side) != ncells) return 1;
    u8* next = (u8*)malloc(ncells ? ncells : 1);
    u64* prefix = (u64*)malloc(sizeof(u64) * (size_t)(side + 1));
    if (!next || !prefix) { free(next); free(prefix); return 2; }
    for (i64 z = 0; z <= side; ++z) prefix[z] = orc_tet_layer_prefix(side, z);
    u8* cur = cells;
    for (i64 st = 0; st < steps; ++st) {
        ca_ctx c = {side, cur, next, prefix};
        run_pool(ca_layer, &c, side, nthreads);
        u8* t = cur; cur = next; next = t;
    }
    if (cur != cells) { /* odd step count: result lives in the scratch buffer */
        memcpy(cells, cur, ncells);
        next = cur;
    }
    free(next);
    free(prefix);
    return 0;
}

/* kernel_accum (simulator.hpp:329-331) */
void orc_kernel_accum(u32* cells, u64 n) { for (u64 i = 0; i < n; ++i) cells[i] += 1; }

/* verify_exact_cover (simulator.hpp:467-478): first cell with multiplicity != 1,
 * converted back to (x, y, z) through tri_coord_at/tet_coord_at (core.hpp:151-164). */
int orc_first_defect(int m, i64 side, const u32* cov, u64 n, i64* w3, u64* mult) {
    for (u64 i = 0; i < n; ++i) {
        if (cov[i] == 1) continue;
        i64 z = 0;
        u64 rem = i;
        if (m == 3) {
            while (z + 1 < side && orc_tet_layer_prefix(side, z + 1) <= i) ++z;
            rem = i - orc_tet_layer_prefix(side, z);
        }
        i64 y = 0;
        while (tri_index(0, y + 1) <= rem) ++y;
        w3[0] = (i64)(rem - tri_index(0, y));
        w3[1] = y;
        w3[2] = z;
        *mult = cov[i];
        return 0; /* not exact */
    }
    return 1; /* exact */
}

/* ---- EDM and the periodic 2-D Life ---- */

/* make_edm_points (simulator.hpp:333-343) + splitmix64_unit (bits.hpp:92-94) */
void orc_make_edm_points(i64 count, u64 seed, double* out) {
    u64 st = seed;
    for (i64 i = 0; i < 2 * count; ++i) out[i] = (double)(splitmix64(&st) >> 11) * 0x1.0p-53;
}

/* kernel_edm (simulator.hpp:375-386) with edm_distance (:345-350): mul, mul,
 * add, sqrt, each rounded (this file is built with -ffp-contract=off) */
void orc_kernel_edm(i64 side, const double* pts, double* cells) {
    for (i64 y = 0; y < side; ++y)
        for (i64 x = 0; x <= y; ++x) {
            double dx = pts[2 * x] - pts[2 * y], dy = pts[2 * x + 1] - pts[2 * y + 1];
            cells[tri_index(x, y)] = sqrt(dx * dx + dy * dy);
        }
}

/* kernel_ca_run m = 2 (simulator.hpp:409-425) with alive_neighbors_2d_periodic
 * (:227-239): Moore neighbourhood wrapped modulo the side, x > y reads dead */
int orc_ca2d_run(i64 side, i64 steps, u8* cells, u64 ncells) {
    if (ncells != orc_tri_cells(side) || steps < 0) return 1;
    u8* next = (u8*)malloc(ncells ? ncells : 1);
    if (!next) return 2;
    for (i64 st = 0; st < steps; ++st) {
        for (i64 y = 0; y < side; ++y)
            for (i64 x = 0; x <= y; ++x) {
                int count = 0;
                for (i64 dy = -1; dy <= 1; ++dy)
                    for (i64 dx = -1; dx <= 1; ++dx) {
                        if (!dx && !dy) continue;
                        i64 nx = x + dx, ny = y + dy;
                        if (nx < 0) nx += side; else if (nx >= side) nx -= side;
                        if (ny < 0) ny += side; else if (ny >= side) ny -= side;
                        if (nx <= ny) count += cells[tri_index(nx, ny)];
                    }
                next[tri_index(x, y)] = life_next(cells[tri_index(x, y)], count);
            }
        memcpy(cells, next, ncells);
    }
    free(next);
    return 0;
}
