// sm_100a kernels for the other two 2-simplex workloads of the reference
// (SURVEY 8(f) #2, #3), through every 2-D map (bb, rb, lambda, h2d,
// h2d-padded, trapezoid bands):
//
//  * EDM (launch_edm, simulator.hpp:345-372): cell (x, y) = the Euclidean
//    distance between points x and y, f64, written once per cell. Bit-exact
//    with the reference (whose g++ build does not contract to FMA): explicit
//    round-to-nearest mul / add / sqrt intrinsics, one fixed expression order
//    (edm_distance, simulator.hpp:345-350).
//  * 2-D Life with the periodic boundary (launch_ca m = 2, simulator.hpp:
//    227-239, 431-463): Moore neighbourhood wrapped modulo the side, wrapped
//    coordinates outside T(S) (x > y) read as dead; B3/S23.
//
// Each in two execution schemes: BLOCK (the paper's launch model: one CTA per
// map block, rho^2 threads) and RUNS (a warp maps 32 blocks and merges
// x-adjacent tiles into runs; EDM streams whole cell rows of the runs with
// lane-consecutive 8-byte stores, Life cuts them into 32-cell bit-sliced items
// whose neighbourhoods come from a bit triangle of the state, packed first).
#include "smx_common.cuh"
#include <algorithm>
#include <cstdlib>

#include "smx_launch.hpp"
#include "smx_ca_common.cuh"
#include "smx_runs.cuh"

namespace smx {

namespace {

constexpr int T2_THREADS = 256;
constexpr int T2_KX = 32;

// edm_distance (simulator.hpp:345-350): dx*dx + dy*dy, then sqrt, each
// correctly rounded (no FMA contraction)
__device__ __forceinline__ double edm_dist(double2 a, double2 b) {
    const double dx = __dsub_rn(a.x, b.x), dy = __dsub_rn(a.y, b.y);
    return __dsqrt_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
}

// alive_neighbors_2d_periodic (simulator.hpp:227-239) + life_next (:220-223)
__device__ __forceinline__ uint8_t life2d_cell(const uint8_t* __restrict__ cur, int S, int x, int y) {
    int count = 0;
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy) {
        int ny = y + dy;
        ny = ny < 0 ? ny + S : (ny >= S ? ny - S : ny);
        const unsigned long long row = tri_idx(0, ny);
#pragma unroll
        for (int dx = -1; dx <= 1; ++dx) {
            if (dx == 0 && dy == 0) continue;
            int nx = x + dx;
            nx = nx < 0 ? nx + S : (nx >= S ? nx - S : nx);
            if (nx <= ny) count += __ldg(cur + row + nx);
        }
    }
    const int me = cur[tri_idx(x, y)];
    return (uint8_t)(me ? (count == 2 || count == 3) : (count == 3));
}

template <int KIND>
__global__ void k_edm_block(Geom g, const double2* __restrict__ pts, double* __restrict__ cells) {
    const int wx = blockIdx.x, wy = blockIdx.y;
    __shared__ outcome<int> s_o;
    if (threadIdx.x == 0 && threadIdx.y == 0) s_o = map_block<KIND>(g, wx, wy, 0);
    __syncthreads();
    const outcome<int> o = s_o;
    if (o.is_void) return;
    const int rho = g.rho, S = g.side;
    for (int ly = threadIdx.y; ly < rho; ly += blockDim.y)
        for (int lx = threadIdx.x; lx < rho; lx += blockDim.x) {
            const int cx = o.x * rho + lx, cy = o.y * rho + ly;
            if (!tri_contains<int>(S, cx, cy)) continue;
            cells[tri_idx(cx, cy)] = edm_dist(pts[cx], pts[cy]);
        }
}

// (two strips per CTA with paired 16-byte stores measured slower here: 591 vs
// 633 Gcells/s at C1; the write-only stream prefers one strip and lane-strided
// 8-byte stores)
template <int KIND, int EDM_ILP>
__global__ void __launch_bounds__(T2_THREADS) k_edm_runs(Geom g, const double2* __restrict__ pts,
                                                         double* __restrict__ cells) {
    __shared__ int s_run[T2_KX][3];
    __shared__ int s_nruns;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (warp == 0) strip_runs<KIND, T2_KX>(g, blockIdx.x * T2_KX, blockIdx.y, s_run, &s_nruns);
    __syncthreads();
    const int rows = s_nruns * g.rho;
    for (int rr = warp; rr < rows; rr += T2_THREADS / 32) {
        int cy, xlo, xhi;
        if (!run_row(s_run, rr, g.rho, g.side, &cy, &xlo, &xhi)) continue;
        const double2 py = pts[cy];
        double* row = cells + tri_idx(0, cy);
        if (EDM_ILP > 1) {
            // EDM_ILP cells per lane in flight: the point loads of all of them
            // issue before the first distance
            int x = xlo + lane;
            for (; x + 32 * (EDM_ILP - 1) < xhi; x += 32 * EDM_ILP) {
                double2 p[EDM_ILP];
#pragma unroll
                for (int k = 0; k < EDM_ILP; ++k) p[k] = __ldg(pts + x + 32 * k);
#pragma unroll
                for (int k = 0; k < EDM_ILP; ++k) row[x + 32 * k] = edm_dist(p[k], py);
            }
            for (; x < xhi; x += 32) row[x] = edm_dist(__ldg(pts + x), py);
        } else {
            for (int x = xlo + lane; x < xhi; x += 32) row[x] = edm_dist(__ldg(pts + x), py);
        }
    }
}

template <int KIND>
__global__ void k_ca2d_block(Geom g, const uint8_t* __restrict__ cur, uint8_t* __restrict__ next) {
    const int wx = blockIdx.x, wy = blockIdx.y;
    __shared__ outcome<int> s_o;
    if (threadIdx.x == 0 && threadIdx.y == 0) s_o = map_block<KIND>(g, wx, wy, 0);
    __syncthreads();
    const outcome<int> o = s_o;
    if (o.is_void) return;
    const int rho = g.rho, S = g.side;
    for (int ly = threadIdx.y; ly < rho; ly += blockDim.y)
        for (int lx = threadIdx.x; lx < rho; lx += blockDim.x) {
            const int cx = o.x * rho + lx, cy = o.y * rho + ly;
            if (!tri_contains<int>(S, cx, cy)) continue;
            next[tri_idx(cx, cy)] = life2d_cell(cur, S, cx, cy);
        }
}

// The bit-sliced 2-D Life kernel indexes the packed state with IDX: int when
// T(S) < 2^31 (every 2-D configuration up to side ~65K), else long long.

// 16 cells of a u8 state at 16-aligned packed index q. GUARD: zero outside
// [0, ncells) (bytes past the last cell are not state), for windows that run
// off either end of the array.
template <bool GUARD, typename IDX>
__device__ __forceinline__ uint4 load_cells16(const uint8_t* __restrict__ cur, IDX q, IDX ncells) {
    if (GUARD) {
        if (q < 0 || q >= ncells) return make_uint4(0, 0, 0, 0);
        uint4 v = __ldg(reinterpret_cast<const uint4*>(cur + q));
        if (q + 16 > ncells) {
            const int keep = int(ncells - q);
            uint32_t* w = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int k = keep - 4 * i;
                w[i] = k >= 4 ? w[i] : (k <= 0 ? 0u : (w[i] & (0xffffffffu >> (32 - 8 * k))));
            }
        }
        return v;
    }
    return __ldg(reinterpret_cast<const uint4*>(cur + q));
}

// ---- the bit triangle: bit i of word i / 32 = packed cell i (0 / 1) ----
// The x-run step reads its 3 x 34-cell neighbourhood windows from it: three
// words per row instead of 64 bytes, no byte -> bit packing per chunk, and
// the 1/8-size triangle stays in L2 while the u8 state streams once through
// the pack and once as the step's stores.

// words i and i + 1 of the triangle at a signed word index (0 before the
// start; the buffer ends with zero words, so reads past the last cell are 0)
template <bool GUARD, typename IDX>
__device__ __forceinline__ uint32_t tri_word(const uint32_t* __restrict__ bits, IDX w) {
    if (GUARD && w < 0) return 0u;
    return __ldg(bits + w);
}

// row_hsum from the bit triangle: cells x0 - 1 .. x0 + 32 of the row starting
// at packed index Rr with len cells
// (MASK = false: the window lies inside the row, 1 <= x0 and x0 + 32 < len)
template <bool GUARD, bool MASK, typename IDX>
__device__ __forceinline__ void row_hsum_bits(const uint32_t* __restrict__ bits, IDX Rr, int len, int x0,
                                              uint32_t& s0, uint32_t& s1, uint32_t* centre) {
    const IDX p = Rr + x0 - 1;
    const IDX w = p >> 5;  // floor (arithmetic shift)
    const int d = int(p & 31);
    const uint32_t lo = tri_word<GUARD>(bits, w), hi = tri_word<GUARD>(bits, w + 1), hi2 = __ldg(bits + w + 2);
    uint32_t M = __funnelshift_r(lo, hi, d);           // bit j = cell x0 - 1 + j
    uint32_t T = __funnelshift_r(hi, hi2, d) & 3u;     // cells x0 + 31, x0 + 32
    if (MASK) {
        M &= ca::range_mask(1 - x0, len - x0);
        T &= ((x0 + 31 >= 0 && x0 + 31 < len) ? 1u : 0u) | ((x0 + 32 >= 0 && x0 + 32 < len) ? 2u : 0u);
    }
    const uint32_t l = M, c = (M >> 1) | (T << 31), r = (M >> 2) | (T << 30);
    s0 = l ^ c ^ r;
    s1 = (l & c) | (l & r) | (c & r);
    if (centre) *centre = c;
}

template <typename IDX>
__device__ __forceinline__ uint32_t life2d_bits_tri(const uint32_t* __restrict__ bits, IDX R, int cy, int x0) {
    uint32_t a0, a1, b0, b1, c0, c1, alive;
    if (x0 >= 1 && x0 + 32 < cy) {  // all three windows inside their rows (the row above is the shortest)
        row_hsum_bits<false, false>(bits, IDX(R - cy), cy, x0, a0, a1, nullptr);
        row_hsum_bits<false, false>(bits, R, cy + 1, x0, b0, b1, &alive);
        row_hsum_bits<false, false>(bits, IDX(R + cy + 1), cy + 2, x0, c0, c1, nullptr);
    } else {
        // the upper window may start before the triangle (GUARD)
        row_hsum_bits<true, true>(bits, IDX(R - cy), cy, x0, a0, a1, nullptr);
        row_hsum_bits<false, true>(bits, R, cy + 1, x0, b0, b1, &alive);
        row_hsum_bits<false, true>(bits, IDX(R + cy + 1), cy + 2, x0, c0, c1, nullptr);
    }
    const ca::Planes4 t = ca::add3x2(a0, a1, b0, b1, c0, c1);  // 9-sum incl. the cell
    return (~t.b3 & ~t.b2 & t.b1 & t.b0) | (~t.b3 & t.b2 & ~t.b1 & ~t.b0 & alive);
}

// u8 state (0/1) -> bit triangle, one word per thread (two 16-byte loads),
// then the zero tail
template <typename IDX>
__global__ void __launch_bounds__(256) k_pack2d(const uint8_t* __restrict__ cur, IDX ncells, IDX nwords,
                                                uint32_t* __restrict__ bits) {
    for (IDX w = IDX(blockIdx.x) * blockDim.x + threadIdx.x; w < nwords; w += IDX(gridDim.x) * blockDim.x) {
        const IDX q = 32 * w;
        uint32_t v = 0u;
        if (q + 32 <= ncells) {
            const uint4* c = reinterpret_cast<const uint4*>(cur + q);
            v = ca::pack32(__ldg(c), __ldg(c + 1));
        } else if (q < ncells) {
            v = ca::pack32(load_cells16<true>(cur, q, ncells), load_cells16<true>(cur, IDX(q + 16), ncells));
        }
        bits[w] = v;
    }
}

// Strips per CTA for the 2-D x-run Life kernel: ~256+ chunks per CTA at rho >= 8,
// bounded by shared memory below.
__host__ __device__ constexpr int ca2d_strips(int rho) { return rho >= 16 ? 2 : (rho >= 8 ? 8 : 32); }

// periodic 2-D Life, x-run scheme, bit-sliced. The CTA's warps map NS strips
// of KX blocks (NS consecutive grid rows) and merge x-adjacent tiles into runs.
// Work is cut into 32-cell chunks aligned in the packed array; a chunk belongs
// to the run row holding its first cell (the maps tile T(S) exactly, so every
// chunk has one owner), and one thread computes all 32 cells, across a row end
// if need be: 3 rows x 64 bytes of 16-byte loads -> bit windows -> the 3x3
// sum as bit-planes -> B3/S23 for 32 cells at once -> two 16-byte stores.
// Rows 1 .. S-3 never wrap (their wrapped neighbours lie outside T(S) and read
// dead), so windows only mask row ends; chunks touching rows 0, S-2, S-1 (or
// more than two rows, near the apex) take the per-cell rule.
template <int KIND, int NS, typename IDX>
__global__ void __launch_bounds__(T2_THREADS) k_ca2d_runs(Geom g, const uint8_t* __restrict__ cur,
                                                          const uint32_t* __restrict__ bits,
                                                          uint8_t* __restrict__ next) {
    constexpr int NR = NS * T2_KX;
    __shared__ int s_run[NR][3];
    __shared__ int s_nr[NS];
    __shared__ int s_pre[NR + 1];
    __shared__ int s_cpr[NR];
    const int warp = threadIdx.x >> 5;
    const int rho = g.rho, S = g.side;
    for (int st = warp; st < NS; st += T2_THREADS / 32) {
        const int wy = blockIdx.y * NS + st;
        if (wy < g.ey) strip_runs<KIND, T2_KX>(g, blockIdx.x * T2_KX, wy, s_run + st * T2_KX, &s_nr[st]);
        else if ((threadIdx.x & 31) == 0) s_nr[st] = 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // compact the strips' runs; chunks per run: rho rows x chunk starts per row
        int n = 0, t = 0;
        for (int st = 0; st < NS; ++st)
            for (int r = 0; r < s_nr[st]; ++r, ++n) {
                const int* src = s_run[st * T2_KX + r];
                s_run[n][0] = src[0], s_run[n][1] = src[1], s_run[n][2] = src[2];
                const int cpr = (src[2] * rho + 31) / 32;  // >= the chunk starts in any of its rows
                s_cpr[n] = cpr;
                s_pre[n] = t;
                t += rho * cpr;
            }
        s_pre[n] = t;
        s_nr[0] = n;
    }
    __syncthreads();
    const int nruns = s_nr[0];
    const IDX ncells = IDX((unsigned long long)S * (S + 1) / 2);  // T(S) cells
    const int total = s_pre[nruns];
    for (int it = threadIdx.x; it < total; it += T2_THREADS) {
        int lo = 0, hi = nruns - 1;  // run r: s_pre[r] <= it < s_pre[r + 1]
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (s_pre[mid] <= it) lo = mid;
            else hi = mid - 1;
        }
        const int r = lo, cpr = s_cpr[r], k = it - s_pre[r];
        int ly = int(__fdividef(float(k) + 0.5f, float(cpr)));  // k / cpr (exact after the fix-up)
        ly -= ly * cpr > k;
        ly += (ly + 1) * cpr <= k;
        const int cy = s_run[r][1] * rho + ly, xlo = s_run[r][0] * rho;
        const int xhi = min((s_run[r][0] + s_run[r][2]) * rho, cy + 1);
        if (cy > S - 1 || xlo >= xhi) continue;
        const IDX R = IDX(((unsigned long long)cy * (cy + 1)) >> 1);
        const IDX A = ((R + xlo + 31) & ~IDX(31)) + 32 * (k - ly * cpr);  // chunk starts inside [E0, E1)
        if (A >= R + xhi) continue;
        const int x0 = int(A - R);
        uint32_t res;
        if (cy >= 1 && cy <= S - 3 && x0 + 31 <= cy) {  // wholly inside row cy
            res = life2d_bits_tri(bits, R, cy, x0);
        } else if (cy >= 1 && cy + 1 <= S - 3 && A + 32 <= R + 2 * cy + 3) {  // rows cy, cy + 1
            const int n0 = cy - x0 + 1;  // cells of row cy in the chunk
            const uint32_t m0 = (1u << n0) - 1u;
            res = (life2d_bits_tri(bits, R, cy, x0) & m0) |
                  (life2d_bits_tri(bits, IDX(R + cy + 1), cy + 1, x0 - cy - 1) & ~m0);
        } else {  // per cell, rows found by walking down from cy
            res = 0;
            IDX Ry = R;
            int y = cy;
            for (int b = 0; b < 32 && A + b < ncells; ++b) {
                while (A + b >= Ry + y + 1) Ry += y + 1, ++y;
                res |= uint32_t(life2d_cell(cur, S, int(A + b - Ry), y)) << b;
            }
        }
        if (A + 32 <= ncells) {
            uint4* o = reinterpret_cast<uint4*>(next + A);
            o[0] = ca::spread16(res & 0xffffu);
            o[1] = ca::spread16(res >> 16);
        } else {
            for (int b = 0; A + b < ncells; ++b) next[A + b] = uint8_t((res >> b) & 1u);
        }
    }
}

dim3 block2(const Geom& g) {
    const int bx = g.rho < 32 ? g.rho : 32;
    int by = 256 / bx;
    if (by > g.rho) by = g.rho;
    return dim3(bx, by, 1);
}

#define SMX_DISPATCH_2D(kind, F, ...)                               \
    do {                                                            \
        switch (kind) {                                             \
            case SMX_H2D: F<SMX_H2D>(__VA_ARGS__); break;           \
            case SMX_PADDED: F<SMX_PADDED>(__VA_ARGS__); break;     \
            case SMX_TRAP: F<SMX_TRAP>(__VA_ARGS__); break;         \
            case SMX_RB: F<SMX_RB>(__VA_ARGS__); break;             \
            case SMX_LAMBDA: F<SMX_LAMBDA>(__VA_ARGS__); break;     \
            default: F<SMX_BB>(__VA_ARGS__); break;                 \
        }                                                           \
    } while (0)

template <int KIND>
void launch_edm_k(const Geom& g, const double* pts, double* cells, int exec, cudaStream_t s) {
    const double2* p = reinterpret_cast<const double2*>(pts);
    if (exec == SMX_EXEC_BLOCK) k_edm_block<KIND><<<dim3(g.ex, g.ey, 1), block2(g), 0, s>>>(g, p, cells);
    else  // 4 cells per lane in flight (measured at C1, profiles/r2/edm_ilp.txt: 611 / 634 / 658 Gcells/s for 1 / 2 / 4)
        k_edm_runs<KIND, 4><<<dim3((g.ex + T2_KX - 1) / T2_KX, g.ey, 1), T2_THREADS, 0, s>>>(g, p, cells);
}

template <int KIND>
void launch_ca2d_k(const Geom& g, const uint8_t* cur, const uint32_t* bits, uint8_t* next, int exec, cudaStream_t s) {
    if (exec == SMX_EXEC_BLOCK) k_ca2d_block<KIND><<<dim3(g.ex, g.ey, 1), block2(g), 0, s>>>(g, cur, next);
    else {
        const dim3 grid((g.ex + T2_KX - 1) / T2_KX, (g.ey + ca2d_strips(g.rho) - 1) / ca2d_strips(g.rho), 1);
        if ((unsigned long long)g.side * (g.side + 1) / 2 + 64 < (1ull << 31)) {
            switch (ca2d_strips(g.rho)) {
                case 2: k_ca2d_runs<KIND, 2, int><<<grid, T2_THREADS, 0, s>>>(g, cur, bits, next); break;
                case 8: k_ca2d_runs<KIND, 8, int><<<grid, T2_THREADS, 0, s>>>(g, cur, bits, next); break;
                default: k_ca2d_runs<KIND, 32, int><<<grid, T2_THREADS, 0, s>>>(g, cur, bits, next); break;
            }
        } else {
            switch (ca2d_strips(g.rho)) {
                case 2: k_ca2d_runs<KIND, 2, long long><<<grid, T2_THREADS, 0, s>>>(g, cur, bits, next); break;
                case 8: k_ca2d_runs<KIND, 8, long long><<<grid, T2_THREADS, 0, s>>>(g, cur, bits, next); break;
                default: k_ca2d_runs<KIND, 32, long long><<<grid, T2_THREADS, 0, s>>>(g, cur, bits, next); break;
            }
        }
    }
}

}  // namespace

void launch_edm(const Geom& g, const double* pts, double* cells, int exec, cudaStream_t s) {
    SMX_DISPATCH_2D(g.kind, launch_edm_k, g, pts, cells, exec, s);
}

void launch_ca2d(const Geom& g, const uint8_t* cur, const uint32_t* bits, uint8_t* next, int exec, cudaStream_t s) {
    SMX_DISPATCH_2D(g.kind, launch_ca2d_k, g, cur, bits, next, exec, s);
}

uint64_t ca2d_bit_words(uint64_t ncells) { return (ncells + 31) / 32 + 3; }

void launch_pack2d(const uint8_t* cur, uint64_t ncells, uint32_t* bits, cudaStream_t s) {
    const uint64_t nw = ca2d_bit_words(ncells);
    const unsigned blocks = unsigned(std::min<uint64_t>((nw + 255) / 256, 148ull * 64));
    if (ncells + 64 < (1ull << 31)) k_pack2d<int><<<blocks, 256, 0, s>>>(cur, int(ncells), int(nw), bits);
    else k_pack2d<long long><<<blocks, 256, 0, s>>>(cur, (long long)ncells, (long long)nw, bits);
}

}  // namespace smx
