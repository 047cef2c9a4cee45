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
// map block, rho^2 threads) and RUNS (a warp maps 32 blocks, merges x-adjacent
// tiles, and each warp streams whole cell rows of the runs: coalesced 8-byte
// (EDM) / 1-byte (Life) stores, lane-consecutive cells).
#include "smx_common.cuh"
#include "smx_launch.hpp"
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

// bytes [a, a + 4) of a u8 array through aligned 32-bit loads (the packed rows
// have arbitrary byte alignment)
__device__ __forceinline__ void load8(const uint8_t* __restrict__ p, unsigned long long a, uint32_t& lo,
                                      uint32_t& hi) {
    const unsigned long long b = a & ~3ull;
    const uint32_t* q = reinterpret_cast<const uint32_t*>(p + b);
    const uint32_t w0 = __ldg(q), w1 = __ldg(q + 1), w2 = __ldg(q + 2);
    const int sh = int(a - b) * 8;
    lo = __funnelshift_r(w0, w1, sh);
    hi = __funnelshift_r(w1, w2, sh);
}

// exact per-byte "== 0" for bytes < 0x80: bit 7 of each byte
__device__ __forceinline__ uint32_t zero_bytes(uint32_t x) {
    return ~(((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x) & 0x80808080u;
}

// 3 cells' horizontal sums of one row, for the 4 cells x .. x+3 (bytes x-1 .. x+4
// at packed index a = row + x - 1): left + centre + right, <= 3 per byte
__device__ __forceinline__ uint32_t hsum4(const uint8_t* __restrict__ cur, unsigned long long a, uint32_t* centre) {
    uint32_t L, H;
    load8(cur, a, L, H);
    const uint32_t C = __funnelshift_r(L, H, 8), R = __funnelshift_r(L, H, 16);
    if (centre) *centre = C;
    return L + C + R;
}

// periodic 2-D Life, x-run scheme: a warp per cell row of a run; lane per
// 4-byte-aligned output word. Interior words (no wrap, every neighbour row
// long enough) are computed SWAR: three rows' horizontal sums added bytewise
// (<= 9 per byte), B3/S23 as (S == 3) | (alive & S == 4) with an exact
// per-byte zero test; wrap-around, row-end and partial words fall back to the
// per-cell rule.
template <int KIND>
__global__ void __launch_bounds__(T2_THREADS) k_ca2d_runs(Geom g, const uint8_t* __restrict__ cur,
                                                          uint8_t* __restrict__ next) {
    __shared__ int s_run[T2_KX][3];
    __shared__ int s_nruns;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (warp == 0) strip_runs<KIND, T2_KX>(g, blockIdx.x * T2_KX, blockIdx.y, s_run, &s_nruns);
    __syncthreads();
    const int rows = s_nruns * g.rho, S = g.side;
    for (int rr = warp; rr < rows; rr += T2_THREADS / 32) {
        int cy, xlo, xhi;
        if (!run_row(s_run, rr, g.rho, S, &cy, &xlo, &xhi)) continue;
        const unsigned long long R = tri_idx(0, cy);
        const unsigned long long E0 = R + xlo, E1 = R + xhi;
        const unsigned long long A0 = (E0 + 3) & ~3ull, A1 = E1 & ~3ull;
        const bool yin = cy >= 1 && cy <= S - 2;  // no vertical wrap
        const unsigned long long Rm = yin ? tri_idx(0, cy - 1) : 0, Rp = yin ? tri_idx(0, cy + 1) : 0;
        if (A0 < A1) {
            for (unsigned long long A = A0 + 4ull * lane; A < A1; A += 128) {
                const int x = int(A - R);
                if (yin && x >= 1 && x + 4 <= cy - 1) {
                    uint32_t self;
                    const uint32_t t = hsum4(cur, Rm + x - 1, nullptr) + hsum4(cur, R + x - 1, &self) +
                                       hsum4(cur, Rp + x - 1, nullptr);
                    const uint32_t eq3 = zero_bytes(t ^ 0x03030303u), eq4 = zero_bytes(t ^ 0x04040404u);
                    *reinterpret_cast<uint32_t*>(next + A) = ((eq3 | (eq4 & (self << 7))) >> 7) & 0x01010101u;
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j) next[A + j] = life2d_cell(cur, S, x + j, cy);
                }
            }
            // head [E0, A0) and tail [A1, E1): at most 3 + 3 cells
            const int nh = int(A0 - E0), nt = int(E1 - A1);
            if (lane < nh) next[E0 + lane] = life2d_cell(cur, S, xlo + lane, cy);
            else if (lane >= 8 && lane - 8 < nt) next[A1 + lane - 8] = life2d_cell(cur, S, int(A1 - R) + lane - 8, cy);
        } else {
            for (int x = xlo + lane; x < xhi; x += 32) next[R + x] = life2d_cell(cur, S, x, cy);
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
