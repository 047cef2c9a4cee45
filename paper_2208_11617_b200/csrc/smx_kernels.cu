// sm_100a kernels for the H-map hot path: block-outcome dump, the paper's MAP
// kernel, ACCUM (block and x-run schemes), Life init, 3-D Life (block scheme)
// and the tile pack/unpack used by the multi-GPU halo exchange.
//
// Reference semantics: detail::sweep (simulator.hpp:177-218) — map -> Void ->
// strict y-1 -> rho^m cells -> membership -> packed index -> body.
#include "smx_common.cuh"
#include <algorithm>
#include <cstdlib>

#include "smx_launch.hpp"
#include "smx_runs.cuh"

namespace smx {

#define FULL_MASK 0xffffffffu

// ---------------------------------------------------------------------------
// Block outcome dump: one thread per block, raw map_outcome (no strict shift),
// natural z, y, x order (simulator.hpp:113-118).
template <int KIND>
__global__ void k_outcomes(Geom g, smx_outcome* out, unsigned long long count) {
    const unsigned long long exy = (unsigned long long)g.ex * (unsigned long long)g.ey;
    for (unsigned long long b = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; b < count;
         b += (unsigned long long)gridDim.x * blockDim.x) {
        const int wz = int(b / exy);
        const unsigned long long r = b - (unsigned long long)wz * exy;
        const int wy = int(r / (unsigned long long)g.ex);
        const int wx = int(r - (unsigned long long)wy * g.ex);
        const outcome<int> o = map_raw<KIND>(g, wx, wy, wz);
        int4* dst = reinterpret_cast<int4*>(out + b);
        dst[0] = make_int4(o.is_void, o.x, o.y, o.z);
        dst[1] = make_int4(o.level_b, o.index_q, 0, 0);
    }
}

// ---------------------------------------------------------------------------
// Block scheme helpers. CTA = one map block; blockDim = (min(rho,1024),
// min(rho, 1024/bx), ...) and threads loop over the remaining local extent.
// The map is evaluated once per warp (lane 0) and broadcast with shuffles.
struct BlockTarget {
    int is_void, x, y, z;
};

template <int KIND>
__device__ __forceinline__ BlockTarget warp_map(const Geom& g, int wx, int wy, int wz) {
    const unsigned m = __activemask();
    const int lane = (threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z)) & 31;
    outcome<int> o{0, 0, 0, 0, 1, 0};
    const int leader = __ffs(m) - 1;
    if (lane == leader) o = map_block<KIND>(g, wx, wy, wz);
    BlockTarget t;
    t.is_void = __shfl_sync(m, o.is_void, leader);
    t.x = __shfl_sync(m, o.x, leader);
    t.y = __shfl_sync(m, o.y, leader);
    t.z = __shfl_sync(m, o.z, leader);
    return t;
}

__device__ __forceinline__ int flat_tid() {
    return threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
}

// MODE bit 0: coverage atomics; bit 1: counters; MODE 0: checksum sink only
// (the paper's MAP kernel for timing).
template <int KIND, int MODE>
__global__ void k_map_block(Geom g, int wz0, uint32_t* __restrict__ cov, DevCounters* cnt,
                            unsigned* sink) {
    const int wx = blockIdx.x, wy = g.wy0 + blockIdx.y, wz = blockIdx.z + wz0;
    const BlockTarget t = warp_map<KIND>(g, wx, wy, wz);
    const int slot = (wx + 7 * wy + 13 * wz) & (NSLOT - 1);
    if (t.is_void) {
        if ((MODE & 2) && flat_tid() == 0) atomicAdd(&cnt->blocks_void[slot], 1ull);
        return;
    }
    const int rho = g.rho, S = g.side;
    const int zext = g.dims == 3 ? rho : 1;
    unsigned acc = 0;
    unsigned useful = 0;
    for (int lz = threadIdx.z; lz < zext; lz += blockDim.z)
        for (int ly = threadIdx.y; ly < rho; ly += blockDim.y)
            for (int lx = threadIdx.x; lx < rho; lx += blockDim.x) {
                const int cx = t.x * rho + lx, cy = t.y * rho + ly, cz = t.z * rho + lz;
                const bool member = g.dims == 3 ? tet_contains<int>(S, cx, cy, cz)
                                                : tri_contains<int>(S, cx, cy);
                if (!member) continue;
                unsigned long long idx = tri_idx(cx, cy);
                if (g.dims == 3) idx += g.prefix[cz];
                ++useful;
                acc ^= unsigned(idx) * 0x9E3779B1u;
                if (MODE & 1) atomicAdd(&cov[idx], 1u);
            }
    if (MODE & 2) {
        const unsigned m = __activemask();
        unsigned s = __reduce_add_sync(m, useful);
        if ((flat_tid() & 31) == __ffs(m) - 1) atomicAdd(&cnt->threads_useful[slot], (unsigned long long)s);
    }
    if (MODE == 0 && acc == 0x5bd1e995u) sink[0] = acc;  // keeps the map live, never true in practice
}

// ---------------------------------------------------------------------------
// ACCUM, block scheme (the paper's launch model): ++cells[idx] per useful thread.
template <int KIND>
__global__ void k_accum_block(Geom g, uint32_t* __restrict__ cells) {
    const int wx = blockIdx.x, wy = g.wy0 + blockIdx.y;
    const BlockTarget t = warp_map<KIND>(g, wx, wy, 0);
    if (t.is_void) return;
    const int rho = g.rho, S = g.side;
    for (int ly = threadIdx.y; ly < rho; ly += blockDim.y)
        for (int lx = threadIdx.x; lx < rho; lx += blockDim.x) {
            const int cx = t.x * rho + lx, cy = t.y * rho + ly;
            if (!tri_contains<int>(S, cx, cy)) continue;
            cells[tri_idx(cx, cy)] += 1u;
        }
}

// ---------------------------------------------------------------------------
// ACCUM, x-run scheme. CTA (256 threads) = KX (32) consecutive map blocks of one
// grid row. Warp 0 maps them lane-parallel; tiles whose predecessor lane maps to
// the x-adjacent tile join one run (H2D: every q-run of length b; BB: the row
// segment left of the diagonal). Each run is then streamed row by row with
// 128-bit loads/stores over its 16-byte-aligned interior and scalar head/tail.
constexpr int ACC_THREADS = 256;

// RR rows per warp batch, each [e0, e1): the interior 16-byte vectors of all RR
// rows are loaded before any store, so a lane keeps up to RR * NV 16-byte loads
// in flight (the in-place read-modify-write is HBM-latency bound otherwise).
template <int RR, int NV>
__device__ __forceinline__ void accum_rows(uint32_t* __restrict__ cells, const unsigned long long (&e)[RR][2],
                                           int lane) {
    unsigned long long a0[RR], a1[RR];
    uint4 v[RR][NV];
#pragma unroll
    for (int r = 0; r < RR; ++r) {
        a0[r] = (e[r][0] + 3) & ~3ull;
        a1[r] = e[r][1] & ~3ull;
        if (a0[r] > a1[r]) a0[r] = a1[r] = e[r][1];  // short row: all scalar
    }
#pragma unroll
    for (int r = 0; r < RR; ++r)
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const unsigned long long p = a0[r] + 4ull * (lane + 32 * k);
            if (p < a1[r]) v[r][k] = *reinterpret_cast<const uint4*>(cells + p);
        }
#pragma unroll
    for (int r = 0; r < RR; ++r)
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const unsigned long long p = a0[r] + 4ull * (lane + 32 * k);
            if (p < a1[r]) {
                uint4 t = v[r][k];
                t.x += 1u; t.y += 1u; t.z += 1u; t.w += 1u;
                *reinterpret_cast<uint4*>(cells + p) = t;
            }
        }
#pragma unroll
    for (int r = 0; r < RR; ++r) {
        // long rows beyond the unrolled window
        for (unsigned long long p = a0[r] + 4ull * (lane + 32 * NV); p < a1[r]; p += 128ull) {
            uint4 t = *reinterpret_cast<const uint4*>(cells + p);
            t.x += 1u; t.y += 1u; t.z += 1u; t.w += 1u;
            *reinterpret_cast<uint4*>(cells + p) = t;
        }
        // scalar head [e0, a0) and tail [a1, e1): at most 3 + 3 cells, or a short row
        const unsigned long long nh = a0[r] - e[r][0];
        for (unsigned long long i = lane; i < nh; i += 32) cells[e[r][0] + i] += 1u;
        const unsigned long long nt = e[r][1] - a1[r];
        for (unsigned long long i = lane; i < nt; i += 32) cells[a1[r] + i] += 1u;
    }
}

template <int KIND, int KX, int RR, int NV, int KS = 1>
__global__ void __launch_bounds__(ACC_THREADS, 4) k_accum_runs(Geom g, uint32_t* __restrict__ cells) {
    // KS strips of KX blocks per CTA, mapped concurrently by warps 0 .. KS-1
    __shared__ int s_run[KS * KX][3];
    __shared__ int s_nrun[KS];
    __shared__ int s_total;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // consecutive CTAs take consecutive strips of a grid row: their cells are
    // consecutive segments of the same data rows (a launch order with
    // consecutive grid rows per strip column measured slower for both maps:
    // C3 H 5800 vs 6335 GB/s, profiles/r2/accum_order.txt)
    int xs = blockIdx.x, wy = g.wy0 + blockIdx.y;
    if (g.order) {
        const int2 o = g.order[blockIdx.x];
        xs = o.x, wy = o.y;
    }
    strips_runs<KIND, KX, KS>(g, xs, wy, s_run, s_nrun, &s_total);
    const int nruns = s_total;
    const int rho = g.rho, S = g.side;
    const int rows = nruns * rho;
    constexpr int NW = ACC_THREADS / 32;
    // short run rows (< 128 cells: H2D's first grid rows, level b < KX, runs
    // of b tiles each in another data row; every row at rho <= 2): the CTA's
    // threads tile the rows as W-lane slots (W = the power of two >= the
    // widest row), one cell per thread and row, four rows in flight per
    // thread — instead of a warp per row of a few vectors (at C1 those CTAs
    // held SM slots ~100 us) or a lane per row (rho 2: 16 of 256 threads busy)
    int wmax = 0;
    for (int r = 0; r < nruns; ++r) wmax = max(wmax, s_run[r][2]);
    if (wmax * rho < 128) {
        int lgW = 4;
        while ((1 << lgW) < wmax * rho) ++lgW;
        const int P = ACC_THREADS >> lgW, sub = threadIdx.x >> lgW, col = threadIdx.x & ((1 << lgW) - 1);
        const bool p2 = (rho & (rho - 1)) == 0;
        const int lr = __ffs(rho) - 1;
        for (int rr0 = 0; rr0 < rows; rr0 += 4 * P) {
            uint32_t* ptr[4];
            uint32_t v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                ptr[u] = nullptr;
                const int rr = rr0 + u * P + sub;
                if (rr < rows) {
                    const int r = p2 ? rr >> lr : rr / rho, ly = rr - r * rho;
                    const int cy = s_run[r][1] * rho + ly;
                    const int x = s_run[r][0] * rho + col;
                    const int xhi = min((s_run[r][0] + s_run[r][2]) * rho, cy + 1);  // tri_contains: x <= y
                    if (cy <= S - 1 && x < xhi) ptr[u] = cells + tri_idx(x, cy);
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (ptr[u]) v[u] = *ptr[u];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (ptr[u]) *ptr[u] = v[u] + 1u;
        }
        return;
    }
    for (int row = warp; row < rows; row += RR * NW) {
        unsigned long long e[RR][2];
#pragma unroll
        for (int h = 0; h < RR; ++h) {
            e[h][0] = e[h][1] = 0;
            const int rr = row + h * NW;
            if (rr >= rows) continue;
            const int r = rr / rho, ly = rr - r * rho;
            const int cy = s_run[r][1] * rho + ly;
            const int xlo = s_run[r][0] * rho;
            int xhi = (s_run[r][0] + s_run[r][2]) * rho;
            if (xhi > cy + 1) xhi = cy + 1;  // tri_contains: x <= y
            if (cy > S - 1 || xlo >= xhi) continue;
            const unsigned long long base = tri_idx(0, cy);
            e[h][0] = base + xlo;
            e[h][1] = base + xhi;
        }
        accum_rows<RR, NV>(cells, e, lane);
    }
}

// ---------------------------------------------------------------------------
// make_life_state (simulator.hpp:390-398): alive iff
// splitmix64(fnv1a_append_u64(seed, i)) >> 62 == 0 (bits.hpp:84-109).
__device__ __forceinline__ unsigned char life_bit(unsigned long long seed, unsigned long long i) {
    unsigned long long h = seed;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        h ^= (i >> (8 * k)) & 0xffull;
        h *= 0x100000001b3ull;
    }
    unsigned long long z = h + 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z ^= z >> 31;
    return (z >> 62) == 0 ? 1 : 0;
}

__global__ void k_life_init(unsigned long long seed, uint8_t* __restrict__ cells, unsigned long long n) {
    const unsigned long long nvec = n / 16;
    for (unsigned long long v = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; v < nvec;
         v += (unsigned long long)gridDim.x * blockDim.x) {
        uint32_t w[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            uint32_t acc = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b) acc |= uint32_t(life_bit(seed, v * 16 + 4 * j + b)) << (8 * b);
            w[j] = acc;
        }
        reinterpret_cast<uint4*>(cells)[v] = make_uint4(w[0], w[1], w[2], w[3]);
    }
    if (blockIdx.x == 0 && threadIdx.x < 16) {
        const unsigned long long i = nvec * 16 + threadIdx.x;
        if (i < n) cells[i] = life_bit(seed, i);
    }
}

// kernel_accum (simulator.hpp:329-331), the sequential reference's "one visit
// per cell": no block map, every u32 of the packed state += 1. 16-byte vectors
// over the 16-byte-aligned interior, scalar head / tail; grid-stride.
__global__ void __launch_bounds__(256) k_increment_all(uint32_t* __restrict__ cells, unsigned long long n) {
    const unsigned long long head = ((16u - (reinterpret_cast<uintptr_t>(cells) & 15u)) & 15u) / 4u;
    const unsigned long long h = head < n ? head : n;
    const unsigned long long nvec = (n - h) / 4;
    uint4* v4 = reinterpret_cast<uint4*>(cells + h);
    // 4 vectors per thread in flight (loads before stores)
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long v = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; v < nvec; v += 4 * stride) {
        uint4 x[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (v + k * stride < nvec) x[k] = v4[v + k * stride];
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (v + k * stride < nvec) {
                x[k].x += 1u, x[k].y += 1u, x[k].z += 1u, x[k].w += 1u;
                v4[v + k * stride] = x[k];
            }
    }
    if (blockIdx.x == 0 && threadIdx.x < 8) {
        const unsigned long long t = threadIdx.x;
        if (t < h) cells[t] += 1u;                                           // head (< 4)
        const unsigned long long i = h + nvec * 4 + t;                       // tail (< 4)
        if (t < 4 && i < n) cells[i] += 1u;
    }
}

// ---------------------------------------------------------------------------
// 3-D Life, block scheme: one CTA per map block, one thread per cell; the 26
// neighbours are read through the packed index with the tetrahedron membership
// filter (alive_neighbors_3d_dead, simulator.hpp:242-253), life_next :220-223.
__device__ __forceinline__ int life_rule(int alive, int nb) {
    return alive ? (nb == 2 || nb == 3) : (nb == 3);
}

template <int KIND>
__global__ void k_ca_block(Geom g, int wz0, const uint8_t* __restrict__ cur, uint8_t* __restrict__ next) {
    const int wx = blockIdx.x, wy = blockIdx.y, wz = blockIdx.z + wz0;
    const BlockTarget t = warp_map<KIND>(g, wx, wy, wz);
    if (t.is_void) return;
    const int rho = g.rho, S = g.side;
    const unsigned long long* __restrict__ P = g.prefix;
    for (int lz = threadIdx.z; lz < rho; lz += blockDim.z)
        for (int ly = threadIdx.y; ly < rho; ly += blockDim.y)
            for (int lx = threadIdx.x; lx < rho; lx += blockDim.x) {
                const int cx = t.x * rho + lx, cy = t.y * rho + ly, cz = t.z * rho + lz;
                if (!tet_contains<int>(S, cx, cy, cz)) continue;
                int count = 0;
#pragma unroll
                for (int dz = -1; dz <= 1; ++dz) {
                    const int zz = cz + dz;
                    if (zz < 0 || zz > S - 1) continue;
                    const unsigned long long pz = __ldg(P + zz);
#pragma unroll
                    for (int dy = -1; dy <= 1; ++dy) {
                        const int yy = cy + dy;
                        if (yy < 0 || yy + zz > S - 1) continue;
                        const uint8_t* row = cur + pz + tri_idx(0, yy);
#pragma unroll
                        for (int dx = -1; dx <= 1; ++dx) {
                            const int xx = cx + dx;
                            if (xx >= 0 && xx <= yy) count += __ldg(row + xx);
                        }
                    }
                }
                const unsigned long long idx = P[cz] + tri_idx(cx, cy);
                const int me = cur[idx];
                next[idx] = (uint8_t)life_rule(me, count - me);
            }
}

// ---------------------------------------------------------------------------
// Halo tile pack/unpack (multi-GPU exchange): tile k occupies rho^3 bytes of
// the buffer in lz, ly, lx order; cells outside the tetrahedron pack as 0 and
// are skipped on unpack.
__global__ void k_tiles_pack(Geom g, const uint8_t* __restrict__ cells, const int* __restrict__ tiles,
                             uint8_t* __restrict__ out) {
    const int k = blockIdx.x;
    const int X = tiles[3 * k], Y = tiles[3 * k + 1], Z = tiles[3 * k + 2];
    const int rho = g.rho, S = g.side, r3 = rho * rho * rho;
    for (int t = threadIdx.x; t < r3; t += blockDim.x) {
        const int lx = t % rho, ly = (t / rho) % rho, lz = t / (rho * rho);
        const int cx = X * rho + lx, cy = Y * rho + ly, cz = Z * rho + lz;
        uint8_t v = 0;
        if (tet_contains<int>(S, cx, cy, cz)) v = cells[g.prefix[cz] + tri_idx(cx, cy)];
        out[(unsigned long long)k * r3 + t] = v;
    }
}

__global__ void k_tiles_unpack(Geom g, uint8_t* __restrict__ cells, const int* __restrict__ tiles,
                               const uint8_t* __restrict__ in) {
    const int k = blockIdx.x;
    const int X = tiles[3 * k], Y = tiles[3 * k + 1], Z = tiles[3 * k + 2];
    const int rho = g.rho, S = g.side, r3 = rho * rho * rho;
    for (int t = threadIdx.x; t < r3; t += blockDim.x) {
        const int lx = t % rho, ly = (t / rho) % rho, lz = t / (rho * rho);
        const int cx = X * rho + lx, cy = Y * rho + ly, cz = Z * rho + lz;
        if (tet_contains<int>(S, cx, cy, cz))
            cells[g.prefix[cz] + tri_idx(cx, cy)] = in[(unsigned long long)k * r3 + t];
    }
}

// ---------------------------------------------------------------------------
// verify_exact_cover on the device (simulator.hpp:467-478): the first packed
// index whose multiplicity is not 1 (ncells when the cover is exact).
__global__ void k_first_defect(const uint32_t* __restrict__ cov, unsigned long long n,
                               unsigned long long* __restrict__ first) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        if (__ldg(cov + i) != 1u) {
            atomicMin(first, i);
            return;  // later indices of this thread cannot be smaller
        }
    }
}

void launch_first_defect(const uint32_t* cov, unsigned long long n, unsigned long long* first, cudaStream_t s) {
    unsigned long long blocks = (n + 255) / 256;
    if (blocks > 148ull * 16) blocks = 148ull * 16;
    if (blocks == 0) blocks = 1;
    k_first_defect<<<(unsigned)blocks, 256, 0, s>>>(cov, n, first);
}

// ---------------------------------------------------------------------------
// Launchers.
static dim3 block_shape(const Geom& g) {
    const int bx = g.rho < 1024 ? g.rho : 1024;
    int by = 1024 / bx;
    if (by > g.rho) by = g.rho;
    int bz = 1;
    if (g.dims == 3) {
        bz = 1024 / (bx * by);
        if (bz > g.rho) bz = g.rho;
        if (bz < 1) bz = 1;
    }
    return dim3(bx, by, bz);
}

#define SMX_DISPATCH_KIND(kind, F, ...)                             \
    do {                                                            \
        switch (kind) {                                             \
            case SMX_H2D: F<SMX_H2D>(__VA_ARGS__); break;           \
            case SMX_H3D: F<SMX_H3D>(__VA_ARGS__); break;           \
            case SMX_PADDED: F<SMX_PADDED>(__VA_ARGS__); break;     \
            case SMX_TRAP: F<SMX_TRAP>(__VA_ARGS__); break;         \
            case SMX_RB: F<SMX_RB>(__VA_ARGS__); break;             \
            case SMX_LAMBDA: F<SMX_LAMBDA>(__VA_ARGS__); break;     \
            default: F<SMX_BB>(__VA_ARGS__); break;                 \
        }                                                           \
    } while (0)

template <int KIND>
static void launch_outcomes_k(const Geom& g, smx_outcome* out, unsigned long long count, cudaStream_t s) {
    const int threads = 256;
    unsigned long long blocks = (count + threads - 1) / threads;
    if (blocks > 148ull * 64) blocks = 148ull * 64;
    if (blocks == 0) blocks = 1;
    k_outcomes<KIND><<<(unsigned)blocks, threads, 0, s>>>(g, out, count);
}
void launch_outcomes(const Geom& g, smx_outcome* out, unsigned long long count, cudaStream_t s) {
    SMX_DISPATCH_KIND(g.kind, launch_outcomes_k, g, out, count, s);
}

template <int KIND>
static void launch_map_block_k(const Geom& g, int wz0, int wz1, uint32_t* cov, DevCounters* cnt,
                               unsigned* sink, cudaStream_t s) {
    const dim3 grid(g.ex, g.ey, wz1 - wz0), blk = block_shape(g);
    const int mode = (cov ? 1 : 0) | (cnt ? 2 : 0);
    switch (mode) {
        case 0: k_map_block<KIND, 0><<<grid, blk, 0, s>>>(g, wz0, cov, cnt, sink); break;
        case 1: k_map_block<KIND, 1><<<grid, blk, 0, s>>>(g, wz0, cov, cnt, sink); break;
        case 2: k_map_block<KIND, 2><<<grid, blk, 0, s>>>(g, wz0, cov, cnt, sink); break;
        default: k_map_block<KIND, 3><<<grid, blk, 0, s>>>(g, wz0, cov, cnt, sink); break;
    }
}
void launch_map_block(const Geom& g, uint32_t* cov, DevCounters* cnt, unsigned* sink, cudaStream_t s) {
    SMX_DISPATCH_KIND(g.kind, launch_map_block_k, g, 0, g.ez, cov, cnt, sink, s);
}

template <int KIND, int KX, int RR, int NV, int KS = 1>
static void launch_runs_t(const Geom& g, uint32_t* cells, cudaStream_t s) {
    const dim3 grid = g.order ? dim3(unsigned(g.norder), 1, 1) : dim3((g.ex + KX * KS - 1) / (KX * KS), g.ey, 1);
    k_accum_runs<KIND, KX, RR, NV, KS><<<grid, ACC_THREADS, 0, s>>>(g, cells);
}

template <int KIND>
static void launch_accum_k(const Geom& g, uint32_t* cells, int exec, cudaStream_t s) {
    if (exec == SMX_EXEC_BLOCK) {
        k_accum_block<KIND><<<dim3(g.ex, g.ey, 1), block_shape(g), 0, s>>>(g, cells);
        return;
    }
    // 32 blocks per CTA strip, 2 rows x 4 vectors in flight per lane, 4 CTAs
    // per SM (<= 64 registers): C3 at 0.85 of the HBM peak
    // (profiles/r1/accum_sweep.txt; 3 CTAs: 0.78, 5 CTAs: spills, 0.60)
    // (a warp-persistent variant — each warp maps and streams its own strips,
    // no CTA barrier — measured slower on B200: C3 3.28 vs 3.04 ms, BB 3.86 vs
    // 3.03 ms; tools/accum_ceiling.py)
    // two 32-block strips per CTA (mapped concurrently by warps 0 and 1), one
    // row per warp at a time with 4 x 16-byte vectors per lane: consecutive
    // warps stream consecutive cell rows. Measured at C3 (tools/accum_ceiling.py,
    // profiles/r2/accum_shapes.txt; GB/s H / BB): 1 strip, 2 rows x 4 vectors
    // 5645 / 5686; 2 strips, 2 x 4: 6102 / 6261; 2 strips, 1 x 8: 6267 / 6503;
    // 2 strips, 1 x 4: 6338 / 6596; 4 strips, 1 x 4: 6254 / 6444.
    // small tiles: eight strips per CTA, so a CTA still streams ~16 K cells
    // (rho = 8: 256 blocks x 64 cells) instead of a few thousand per map pass,
    // and several short rows in flight per warp. Side ~65.5 K, Gcells/s H / BB
    // (profiles/r2/accum_rho_sweep.txt): rho 8: 563 / 524 -> 770 / 752 (0.94
    // of HBM); rho 4: 247 / 200 -> 484 / 411; rho 2: 45 / 40 -> 236 / 175
    if (g.rho >= 16) launch_runs_t<KIND, 32, 1, 4, 2>(g, cells, s);
    else if (g.rho >= 8) launch_runs_t<KIND, 32, 2, 2, 8>(g, cells, s);  // 256-cell rows: 2 rows x 2 vectors
    else launch_runs_t<KIND, 32, 4, 1, 8>(g, cells, s);  // 128-cell rows: 4 rows x 1 vector (rho <= 2: a row per lane)
}
int accum_strip_blocks(int rho) { return 32 * (rho >= 16 ? 2 : 8); }  // map blocks per x-run CTA
void launch_accum(const Geom& g, uint32_t* cells, int exec, cudaStream_t s) {
    SMX_DISPATCH_KIND(g.kind, launch_accum_k, g, cells, exec, s);
}

void launch_life_init(unsigned long long seed, uint8_t* cells, unsigned long long n, cudaStream_t s) {
    const int threads = 256;
    unsigned long long blocks = (n / 16 + threads - 1) / threads;
    if (blocks > 148ull * 32) blocks = 148ull * 32;
    if (blocks == 0) blocks = 1;
    k_life_init<<<(unsigned)blocks, threads, 0, s>>>(seed, cells, n);
}

void launch_increment(uint32_t* cells, unsigned long long n, cudaStream_t s) {
    if (n == 0) return;
    const int threads = 256;
    unsigned long long blocks = (n / 16 + threads - 1) / threads;
    if (blocks > 148ull * 8) blocks = 148ull * 8;
    if (blocks == 0) blocks = 1;
    k_increment_all<<<(unsigned)blocks, threads, 0, s>>>(cells, n);
}

template <int KIND>
static void launch_ca_k(const Geom& g, int wz0, int wz1, const uint8_t* cur, uint8_t* next, cudaStream_t s) {
    if (wz1 <= wz0) return;
    k_ca_block<KIND><<<dim3(g.ex, g.ey, wz1 - wz0), block_shape(g), 0, s>>>(g, wz0, cur, next);
}
// block scheme only; the x-run scheme is driven by the C ABI (pack + k_ca_bits)
void launch_ca(const Geom& g, int wz0, int wz1, const uint8_t* cur, uint8_t* next, int exec, cudaStream_t s) {
    (void)exec;  // the block scheme is the only per-cell CA kernel here
    if (g.kind == SMX_H3D) launch_ca_k<SMX_H3D>(g, wz0, wz1, cur, next, s);
    else launch_ca_k<SMX_BB>(g, wz0, wz1, cur, next, s);
}

void launch_tiles_pack(const Geom& g, const uint8_t* cells, const int* tiles, unsigned long long ntiles,
                       uint8_t* out, cudaStream_t s) {
    if (ntiles == 0) return;
    k_tiles_pack<<<(unsigned)ntiles, 256, 0, s>>>(g, cells, tiles, out);
}
void launch_tiles_unpack(const Geom& g, uint8_t* cells, const int* tiles, unsigned long long ntiles,
                         const uint8_t* in, cudaStream_t s) {
    if (ntiles == 0) return;
    k_tiles_unpack<<<(unsigned)ntiles, 256, 0, s>>>(g, cells, tiles, in);
}

}  // namespace smx
