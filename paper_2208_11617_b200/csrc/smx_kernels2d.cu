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
// lane-consecutive 8-byte stores, Life cuts them into 32-cell bit-sliced items).
#include "smx_common.cuh"
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

template <int KIND>
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
        for (int x = xlo + lane; x < xhi; x += 32) row[x] = edm_dist(__ldg(pts + x), py);
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

// 16 cells of a u8 state at 16-aligned packed index q; zero past the end
// (and for q < 0), so windows that run off the array read dead cells
__device__ __forceinline__ uint4 load_cells16(const uint8_t* __restrict__ cur, long long q, long long ncells) {
    if (q < 0 || q >= ncells) return make_uint4(0, 0, 0, 0);
    uint4 v = __ldg(reinterpret_cast<const uint4*>(cur + q));
    if (q + 16 > ncells) {  // bytes past the last cell are not state: clear them
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

// One row's contribution to the 3x3 sums of the 32 cells x0 .. x0+31: bits of
// cells x0-1 .. x0+32 of row (start index Rr, length len; cells outside
// [0, len) are dead) -> the horizontal 3-sum as two bit-planes (s0, s1).
__device__ __forceinline__ void row_hsum(const uint8_t* __restrict__ cur, long long ncells, long long Rr, int len,
                                         int x0, uint32_t& s0, uint32_t& s1, uint32_t* centre) {
    const long long p = Rr + x0 - 1;
    const long long q = p & ~15ll;
    const int d = int(p - q);
    const uint32_t lo = ca::pack32(load_cells16(cur, q, ncells), load_cells16(cur, q + 16, ncells));
    const uint32_t hi = ca::pack32(load_cells16(cur, q + 32, ncells), load_cells16(cur, q + 48, ncells));
    uint32_t M = __funnelshift_r(lo, hi, d);  // bit j = cell x0 - 1 + j
    uint32_t T = (hi >> d) & 3u;              // cells x0 + 31, x0 + 32
    M &= ca::range_mask(1 - x0, len - x0);
    T &= ((x0 + 31 >= 0 && x0 + 31 < len) ? 1u : 0u) | ((x0 + 32 >= 0 && x0 + 32 < len) ? 2u : 0u);
    const uint32_t l = M, c = (M >> 1) | (T << 31), r = (M >> 2) | (T << 30);
    s0 = l ^ c ^ r;
    s1 = (l & c) | (l & r) | (c & r);
    if (centre) *centre = c;
}

// periodic 2-D Life, x-run scheme, bit-sliced: the CTA's warp 0 maps a strip
// of KX blocks and merges runs; the run rows are cut into 32-cell items
// aligned in the packed array (one lane each: 3 rows x 64 bytes of 16-byte
// loads -> bit windows -> 3x3 sum as bit-planes -> B3/S23 for 32 cells at
// once -> two 16-byte stores). Rows 1 .. S-3 never wrap (a wrapped neighbour
// of theirs lies outside T(S) and reads dead), so the windows only mask the
// row ends; rows 0, S-2, S-1 take the per-cell rule. An item writes only the
// bytes of its own run row (whole 16-byte halves where it owns them).
template <int KIND>
__global__ void __launch_bounds__(T2_THREADS) k_ca2d_runs(Geom g, const uint8_t* __restrict__ cur,
                                                          uint8_t* __restrict__ next) {
    __shared__ int s_run[T2_KX][3];
    __shared__ int s_nruns;
    __shared__ int s_pre[T2_KX + 1];
    const int warp = threadIdx.x >> 5;
    if (warp == 0) strip_runs<KIND, T2_KX>(g, blockIdx.x * T2_KX, blockIdx.y, s_run, &s_nruns);
    __syncthreads();
    const int rho = g.rho, S = g.side;
    if (threadIdx.x == 0) {  // items per run: rho rows x (chunks per row + 1 for misalignment)
        int t = 0;
        for (int r = 0; r < s_nruns; ++r) {
            s_pre[r] = t;
            t += rho * ((s_run[r][2] * rho + 31) / 32 + 1);
        }
        s_pre[s_nruns] = t;
    }
    __syncthreads();
    const long long ncells = (long long)tri_idx(0, S);  // T(S) cells
    const int total = s_pre[s_nruns];
    for (int it = threadIdx.x; it < total; it += T2_THREADS) {
        int r = 0;
        while (s_pre[r + 1] <= it) ++r;
        const int cpr = (s_run[r][2] * rho + 31) / 32 + 1;
        const int k = it - s_pre[r], row = k / cpr, c = k - row * cpr;
        int cy, xlo, xhi;
        if (!run_row(s_run, r * rho + row, rho, S, &cy, &xlo, &xhi)) continue;
        const long long R = (long long)tri_idx(0, cy);
        const long long E0 = R + xlo, E1 = R + xhi;
        const long long A = (E0 & ~31ll) + 32ll * c;
        if (A >= E1) continue;
        const int x0 = int(A - R);
        uint32_t res = 0;
        if (cy >= 1 && cy <= S - 3) {
            uint32_t a0, a1, b0, b1, c0, c1, alive;
            row_hsum(cur, ncells, R - cy, cy, x0, a0, a1, nullptr);
            row_hsum(cur, ncells, R, cy + 1, x0, b0, b1, &alive);
            row_hsum(cur, ncells, R + cy + 1, cy + 2, x0, c0, c1, nullptr);
            const ca::Planes4 t = ca::add3x2(a0, a1, b0, b1, c0, c1);  // 9-sum incl. the cell
            const uint32_t eq3 = ~t.b3 & ~t.b2 & t.b1 & t.b0, eq4 = ~t.b3 & t.b2 & ~t.b1 & ~t.b0;
            res = eq3 | (eq4 & alive);
        } else {
            for (int j = 0; j < 32; ++j)
                if (A + j >= E0 && A + j < E1) res |= uint32_t(life2d_cell(cur, S, x0 + j, cy)) << j;
        }
        const uint4 v0 = ca::spread16(res & 0xffffu), v1 = ca::spread16(res >> 16);
        uint4* o = reinterpret_cast<uint4*>(next + A);
        if (A >= E0 && A + 16 <= E1) o[0] = v0;
        if (A + 16 >= E0 && A + 32 <= E1) o[1] = v1;
        if (A < E0 || A + 32 > E1) {  // the run row's first / last item: its own bytes of a shared half
            const bool h0 = A >= E0 && A + 16 <= E1, h1 = A + 16 >= E0 && A + 32 <= E1;
            for (int j = 0; j < 32; ++j) {
                const long long e = A + j;
                if (e < E0 || e >= E1 || (j < 16 ? h0 : h1)) continue;
                next[e] = uint8_t((res >> j) & 1u);
            }
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
    else k_edm_runs<KIND><<<dim3((g.ex + T2_KX - 1) / T2_KX, g.ey, 1), T2_THREADS, 0, s>>>(g, p, cells);
}

template <int KIND>
void launch_ca2d_k(const Geom& g, const uint8_t* cur, uint8_t* next, int exec, cudaStream_t s) {
    if (exec == SMX_EXEC_BLOCK) k_ca2d_block<KIND><<<dim3(g.ex, g.ey, 1), block2(g), 0, s>>>(g, cur, next);
    else k_ca2d_runs<KIND><<<dim3((g.ex + T2_KX - 1) / T2_KX, g.ey, 1), T2_THREADS, 0, s>>>(g, cur, next);
}

}  // namespace

void launch_edm(const Geom& g, const double* pts, double* cells, int exec, cudaStream_t s) {
    SMX_DISPATCH_2D(g.kind, launch_edm_k, g, pts, cells, exec, s);
}

void launch_ca2d(const Geom& g, const uint8_t* cur, uint8_t* next, int exec, cudaStream_t s) {
    SMX_DISPATCH_2D(g.kind, launch_ca2d_k, g, cur, next, exec, s);
}

}  // namespace smx
