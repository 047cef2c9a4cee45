// 3-D Life, x-run scheme (SMX_EXEC_RUNS).
//
// CTA = a P x P patch of map blocks at one wz of the H (or BB) grid; thread t
// maps block t. A tile's x-predecessor (X-1, Y, Z) is looked for at the two
// patch neighbours where the maps put it: (wx-1, wy) — unfolded H tiles, wall
// plane, BB rows — and (wx, wy-1) — the hinge fold, whose images step in X
// along wy (maps.hpp:334-336: x = a + ly + lz - s). Chains of x-adjacent tiles
// are cut into chunks of <= 128 cells and each chunk is one (W x rho x rho)
// box: its (W+2) x (rho+2) x (rho+2) halo is staged in shared memory with
// byte-realigned 32-bit loads, reduced with SWAR byte arithmetic (26-neighbour
// sums <= 26 never carry across bytes) and written back as realigned 32-bit
// stores, byte stores only at the two ends of a row.
//
// Semantics: exactly alive_neighbors_3d_dead + life_next (simulator.hpp:220-253)
// for every cell of every tile the map emits; each tile is processed by exactly
// one chunk (the chain decomposition is a partition of the patch's tiles), so
// correctness does not depend on how long the chains are.
#include "smx_common.cuh"
#include "smx_launch.hpp"

namespace smx {

namespace {

constexpr int CA_THREADS = 256;
constexpr int WMAX = 128;            // cells per chunk row
constexpr int PITCH = WMAX + 8;      // smem byte i <-> x = x_lo - 4 + i
constexpr int PW = PITCH / 4;        // words per staged row

template <int RHO>
struct CaCfg {
    static constexpr int P = (WMAX / RHO) < 16 ? (WMAX / RHO) : 16;   // patch edge
    static constexpr int LMAX = WMAX / RHO;                           // tiles per chunk
    static constexpr int HR = (RHO + 2) * (RHO + 2);                  // halo rows
    static constexpr int OR = RHO * RHO;                              // output rows
    static constexpr int NB = P * P;                                  // blocks per CTA
    static_assert(NB <= CA_THREADS, "one thread per patch block");
};

// exact per-byte (v == k) for bytes < 0x80: returns 0x80 in matching bytes
__device__ __forceinline__ uint32_t bytes_eq(uint32_t v, uint32_t k4) {
    const uint32_t x = v ^ k4;
    return ~(((x & 0x7f7f7f7fu) + 0x7f7f7f7fu) | x) & 0x80808080u;
}

// B3/S23 with the 27-sum (self included): next = s==3 | (alive & s==4)
__device__ __forceinline__ uint32_t life_swar(uint32_t s27, uint32_t alive) {
    const uint32_t e3 = bytes_eq(s27, 0x03030303u) >> 7;
    const uint32_t e4 = bytes_eq(s27, 0x04040404u) >> 7;
    return e3 | (e4 & alive);
}

// 32-bit little-endian word at byte offset A (4-aligned), bytes past ncells read as 0.
__device__ __forceinline__ uint32_t load_word_tail(const uint8_t* __restrict__ p, long long A,
                                                   unsigned long long ncells) {
    if ((unsigned long long)(A + 4) <= ncells) return __ldg(reinterpret_cast<const uint32_t*>(p + A));
    uint32_t v = 0;
    for (int b = 0; b < 3; ++b)
        if ((unsigned long long)(A + b) < ncells) v |= (uint32_t)p[A + b] << (8 * b);
    return v;
}

struct Chunk {
    int x_lo, y_lo, z_lo, w;  // cell box origin and width (cells)
};

template <int KIND, int RHO>
__global__ void __launch_bounds__(CA_THREADS) k_ca_runs(Geom g, int wz0, const uint8_t* __restrict__ cur,
                                                        uint8_t* __restrict__ next, unsigned long long ncells) {
    using C = CaCfg<RHO>;
    constexpr int P = C::P;
    __shared__ int s_tx[C::NB], s_ty[C::NB], s_tz[C::NB];
    __shared__ signed char s_valid[C::NB];
    __shared__ Chunk s_chunk[C::NB];
    __shared__ int s_nchunks;
    __shared__ __align__(16) uint32_t s_raw[C::HR][PW];
    __shared__ __align__(16) uint32_t s_h[C::HR][PW];
    __shared__ __align__(16) uint32_t s_out[C::OR][WMAX / 4];

    const int tid = threadIdx.x;
    const int wz = blockIdx.z + wz0;
    const int S = g.side;

    // ---- 1. map the patch, lane-parallel ----
    if (tid == 0) s_nchunks = 0;
    if (tid < C::NB) {
        const int wx = blockIdx.x * P + (tid % P), wy = blockIdx.y * P + (tid / P);
        int valid = wx < g.ex && wy < g.ey;
        outcome<int> o{1, 0, 0, 0, 1, 0};
        if (valid) {
            o = map_block<KIND>(g, wx, wy, wz);
            valid = !o.is_void;
        }
        s_valid[tid] = (signed char)valid;
        s_tx[tid] = o.x;
        s_ty[tid] = o.y;
        s_tz[tid] = o.z;
    }
    __syncthreads();
    // ---- 2. chains of x-adjacent tiles -> chunks ----
    if (tid < C::NB && s_valid[tid]) {
        const int px = tid % P, py = tid / P;
        const int X = s_tx[tid], Y = s_ty[tid], Z = s_tz[tid];
        auto is_tile = [&](int i, int x) {
            return s_valid[i] && s_tx[i] == x && s_ty[i] == Y && s_tz[i] == Z;
        };
        const bool has_pred = (px > 0 && is_tile(tid - 1, X - 1)) || (py > 0 && is_tile(tid - P, X - 1));
        if (!has_pred) {
            int t = tid, len = 1, x0 = X;
            for (;;) {
                const int tx = t % P, ty = t / P;
                const int xn = s_tx[t] + 1;
                int nxt = -1;
                if (tx + 1 < P && is_tile(t + 1, xn)) nxt = t + 1;
                else if (ty + 1 < P && is_tile(t + P, xn)) nxt = t + P;
                if (nxt < 0 || len == C::LMAX) {
                    const int c = atomicAdd(&s_nchunks, 1);
                    s_chunk[c] = Chunk{x0 * RHO, Y * RHO, Z * RHO, len * RHO};
                    if (nxt < 0) break;
                    x0 = s_tx[nxt];
                    len = 0;
                }
                t = nxt;
                ++len;
            }
        }
    }
    __syncthreads();
    const int nchunks = s_nchunks;
    const unsigned long long* __restrict__ PZ = g.prefix;
    const int lane = tid & 31, warp = tid >> 5;
    constexpr int NW = CA_THREADS / 32;

    for (int ci = 0; ci < nchunks; ++ci) {
        const Chunk ch = s_chunk[ci];
        const int nwords = ch.w / 4;  // rho is a multiple of 4 -> w is too
        // ---- 3a. stage the halo rows (raw bytes, x_lo-4 .. x_lo+w+3) ----
        for (int r = warp; r < C::HR; r += NW) {
            const int yy = ch.y_lo - 1 + r % (RHO + 2);
            const int zz = ch.z_lo - 1 + r / (RHO + 2);
            const bool row_ok = yy >= 0 && zz >= 0 && zz <= S - 1 && yy + zz <= S - 1;
            const long long rowbase = row_ok ? (long long)(PZ[zz] + tri_idx(0, yy)) : 0;
            for (int k = lane; k < nwords + 2; k += 32) {
                const int xa = ch.x_lo - 4 + 4 * k;
                uint32_t v = 0;
                if (row_ok && xa <= yy && xa + 3 >= 0) {
                    const long long gb = rowbase + xa;
                    if (xa >= 0 && xa + 3 <= yy) {
                        const long long A = gb & ~3ll;
                        const int sh = int(gb & 3) * 8;
                        const uint32_t w0 = __ldg(reinterpret_cast<const uint32_t*>(cur + A));
                        v = sh == 0 ? w0 : __funnelshift_r(w0, load_word_tail(cur, A + 4, ncells), sh);
                    } else {
#pragma unroll
                        for (int b = 0; b < 4; ++b) {
                            const int x = xa + b;
                            if (x >= 0 && x <= yy) v |= (uint32_t)cur[gb + b] << (8 * b);
                        }
                    }
                }
                s_raw[r][k] = v;
            }
        }
        __syncthreads();
        // ---- 3b. horizontal 3-sums ----
        for (int i = tid; i < C::HR * nwords; i += CA_THREADS) {
            const int r = i / nwords, j = i - r * nwords + 1;
            const uint32_t wl = s_raw[r][j - 1], wc = s_raw[r][j], wr = s_raw[r][j + 1];
            s_h[r][j] = wc + __funnelshift_l(wl, wc, 8) + __funnelshift_r(wc, wr, 8);
        }
        __syncthreads();
        // ---- 3c. 3x3 vertical sums + rule ----
        for (int i = tid; i < C::OR * nwords; i += CA_THREADS) {
            const int o = i / nwords, j = i - o * nwords + 1;
            const int ly = o % RHO, lz = o / RHO;
            uint32_t s = 0;
#pragma unroll
            for (int dz = 0; dz < 3; ++dz)
#pragma unroll
                for (int dy = 0; dy < 3; ++dy) s += s_h[(lz + dz) * (RHO + 2) + ly + dy][j];
            const uint32_t alive = s_raw[(lz + 1) * (RHO + 2) + ly + 1][j];
            s_out[o][j - 1] = life_swar(s, alive);
        }
        __syncthreads();
        // ---- 3d. write back the member cells of each output row ----
        for (int o = warp; o < C::OR; o += NW) {
            const int y = ch.y_lo + o % RHO, z = ch.z_lo + o / RHO;
            if (y + z > S - 1) continue;  // row outside the tetrahedron
            int nv = y - ch.x_lo + 1;     // members: x <= y
            if (nv > ch.w) nv = ch.w;
            if (nv <= 0) continue;
            const unsigned long long e0 = PZ[z] + tri_idx(ch.x_lo, y);
            const unsigned long long e1 = e0 + nv;
            const int r = int(e0 & 3);
            const unsigned long long a0 = e0 & ~3ull;
            const int nw_out = int((e1 - a0 + 3) / 4);
            const uint32_t* orow = s_out[o];
            for (int k = lane; k < nw_out; k += 32) {
                const unsigned long long A = a0 + 4ull * k;
                // bytes of this aligned word: smem out byte (A - e0) + b
                uint32_t val;
                if (r == 0) val = orow[k];
                else {
                    const uint32_t lo = k > 0 ? orow[k - 1] : 0u;
                    const uint32_t hi = k < WMAX / 4 ? orow[k] : 0u;
                    val = __funnelshift_r(lo, hi, 8 * (4 - r));
                }
                if (A >= e0 && A + 4 <= e1) {
                    *reinterpret_cast<uint32_t*>(next + A) = val;
                } else {
#pragma unroll
                    for (int b = 0; b < 4; ++b)
                        if (A + b >= e0 && A + b < e1) next[A + b] = (uint8_t)(val >> (8 * b));
                }
            }
        }
        __syncthreads();
    }
}

template <int KIND, int RHO>
void launch_runs_t(const Geom& g, int wz0, int wz1, const uint8_t* cur, uint8_t* next, unsigned long long ncells,
                   cudaStream_t s) {
    constexpr int P = CaCfg<RHO>::P;
    const dim3 grid((g.ex + P - 1) / P, (g.ey + P - 1) / P, wz1 - wz0);
    k_ca_runs<KIND, RHO><<<grid, CA_THREADS, 0, s>>>(g, wz0, cur, next, ncells);
}

template <int KIND>
bool launch_runs_kind(const Geom& g, int wz0, int wz1, const uint8_t* cur, uint8_t* next,
                      unsigned long long ncells, cudaStream_t s) {
    switch (g.rho) {
        case 4: launch_runs_t<KIND, 4>(g, wz0, wz1, cur, next, ncells, s); return true;
        case 8: launch_runs_t<KIND, 8>(g, wz0, wz1, cur, next, ncells, s); return true;
        default: return false;
    }
}

}  // namespace

bool ca_runs_supported(int rho) { return rho == 4 || rho == 8; }

void launch_ca_runs(const Geom& g, int kind, int wz0, int wz1, const uint8_t* cur, uint8_t* next,
                    cudaStream_t s) {
    const unsigned long long ncells = tet_cells(g.side);
    if (kind == SMX_H3D) launch_runs_kind<SMX_H3D>(g, wz0, wz1, cur, next, ncells, s);
    else launch_runs_kind<SMX_BB>(g, wz0, wz1, cur, next, ncells, s);
}

}  // namespace smx
