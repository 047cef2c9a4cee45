// 3-D Life, fused u8 -> u8 step (SMX_EXEC_RUNS), sm_100a.
//
// One kernel reads the packed u8 state (reference layout, core.hpp:136-149)
// and writes the next packed u8 state: 1 B read + 1 B written per cell from
// HBM, the neighbourhood re-reads served by L2/L1.
//
//   1. map  — the CTA maps a P x P (x NZ) patch of map blocks lane-parallel and
//             chains x-adjacent tiles into chunks of <= FW cells
//             (ca::build_chunks; the map decides which tiles a CTA computes).
//   2. load — a warp takes a chunk (rho = 8) or two (rho = 4). Its (rho+2)^2
//             halo rows are read as 32-byte aligned pieces (two 16-byte loads
//             per lane, 8 lanes per row, several rows in flight), packed to
//             bits (pack32) and realigned to a chunk-local frame: frame bit i of
//             a row is cell x = x0 - 32 + i, so frame words 1..4 are the owned
//             x range [x0, x0 + 128) and words 0 / 5 hold the x halo. Cells
//             outside the tetrahedron (x < 0, x > y, y + z > S-1, z < 0) are
//             zero bits: alive_neighbors_3d_dead (simulator.hpp:242-253).
//             The horizontal 3-sums (bit-planes h0, h1) go to shared memory.
//   3. march — lane (ly, w) walks z with carry-save adders: 32 cells per LOP3,
//             life_next B3/S23 (simulator.hpp:220-223).
//   4. store — each output row's bytes [E0, E1) are written as 16-byte aligned
//             vectors plus at most 4 + 4 power-of-two head/tail pieces, so every
//             cell of the chunk is written exactly once with no byte loop.
//
// Every useful tile is in exactly one chunk, so every cell is written once per
// step and the result is independent of block order (test_simulator.cpp:169-186).
#include <type_traits>

#include "smx_ca_common.cuh"
#include "smx_launch.hpp"

namespace smx {

namespace {

using namespace ca;

constexpr int F_NWARP = 4;
constexpr int F_NTHR = F_NWARP * 32;

template <int RHO>
struct FCfg {
    static constexpr int LMAX = RHO == 8 ? 12 : 16;      // tiles per chunk (patch edge): w <= 96 / 64
    // computed words per row: the owned cells plus up to 31 cells of the
    // next chunk (sector ownership, see the store phase)
    static constexpr int NW = (LMAX * RHO + 31 + 31) / 32;  // 4 / 3
    static constexpr int HL = RHO + 2;                   // halo rows == halo layers
    static constexpr int HL2 = HL * HL;
    static constexpr int SLOT = RHO * NW;                // march lanes per chunk slot
    static constexpr int CPI = 32 / SLOT;                // chunks per warp item (1 / 4)
    static constexpr int HROWS = CPI * HL2;              // halo rows per item
    static constexpr int OROWS = CPI * RHO * RHO;        // output rows per item
    static constexpr int HW = 3 * NW;                    // smem words per halo row: (h0, h1, raw) x NW
    static constexpr int OSTR = 33;                      // smem words per output layer (32 lanes + pad)
    static constexpr int WARP_WORDS = HROWS * HW + RHO * OSTR + 1;
    static int smem(int nb) { return F_NWARP * WARP_WORDS * 4 + nb * 32 + 16; }
};

// bits of the 32 bytes at 32B-aligned offset A of a u8 array of n bytes, for
// the (at most one per row) piece that runs past the end of the array. Kept out
// of line so the hot path is a plain branch, not a predicated byte loop.
__device__ __noinline__ uint32_t tail_bits(const uint8_t* __restrict__ p, long long A, unsigned long long n) {
    uint32_t v = 0;
    for (int i = 0; i < 32; ++i)
        if ((unsigned long long)(A + i) < n) v |= uint32_t(p[A + i] & 1) << i;
    return v;
}

// 2^K cells (K = 0..4) of output row o starting at cell offset off, stored at
// packed index pos (aligned to 2^K bytes)
template <int K>
__device__ __forceinline__ void store_cells(uint8_t* __restrict__ out, long long pos, const uint32_t* o, int off) {
    const int q = off >> 5, r = off & 31;
    const uint32_t b = __funnelshift_r(o[q], o[q + 1], r);
    if (K == 4) *reinterpret_cast<uint4*>(out + pos) = spread16(b);
    else if (K == 3) *reinterpret_cast<uint2*>(out + pos) = make_uint2(spread4(b & 0xf), spread4((b >> 4) & 0xf));
    else if (K == 2) *reinterpret_cast<uint32_t*>(out + pos) = spread4(b & 0xf);
    else if (K == 1) *reinterpret_cast<uint16_t*>(out + pos) = (uint16_t)spread4(b & 0x3);
    else out[pos] = (uint8_t)(b & 1u);
}

template <int KIND, int RHO>
__global__ void __launch_bounds__(F_NTHR) k_ca_fused(Geom g, int wz0, int wz1, int P, int NZ, int exact,
                                                     const uint8_t* __restrict__ cur, uint8_t* __restrict__ next,
                                                     unsigned long long ncells) {
    using C = FCfg<RHO>;
    constexpr int HL = C::HL, HL2 = C::HL2, NW = C::NW, HW = C::HW;
    extern __shared__ __align__(16) uint32_t fsm[];
    const int NBP = P * P * NZ;
    int4* s_tile = reinterpret_cast<int4*>(fsm + ((F_NWARP * C::WARP_WORDS + 3) & ~3));  // 16-byte aligned
    Chunk* s_chunk = reinterpret_cast<Chunk*>(s_tile + NBP);
    int* s_nchunks = reinterpret_cast<int*>(s_chunk + NBP);

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int S = g.side;
    const unsigned long long* __restrict__ PZ = g.prefix;
    uint32_t* sH = fsm + warp * C::WARP_WORDS;  // [HROWS][HW]
    uint32_t* sO = sH + C::HROWS * HW;           // [RHO][OSTR] (+1 pad word)

    const int nchunks = build_chunks<KIND>(g, wz0 + blockIdx.z * NZ, wz1, P, NZ, C::LMAX, s_tile, s_chunk, s_nchunks);
    const int nitems = (nchunks + C::CPI - 1) / C::CPI;

    for (int item = warp; item < nitems; item += F_NWARP) {
        // ---- load: a lane per halo row -> frame bits -> horizontal 3-sums ----
        // Frame bit i of a row is cell x = x0 - 32 + i: frame words 1..NW are
        // the computed cells [x0, x0 + 32 NW), words 0 and NW+1 the x halo.
        // Only cells [x0 - 1, x0 + w + 32] are needed (the rest stay zero).
        for (int r = lane; r < C::HROWS; r += 32) {
            const int cl = r / HL2, rr = r - cl * HL2;
            const int ci = item * C::CPI + cl;
            uint32_t* hrow = sH + r * HW;
            bool ok = ci < nchunks;
            Chunk ch = ok ? s_chunk[ci] : Chunk{0, 0, 0, 0};
            const int yy = ch.y0 - 1 + rr % HL, zz = ch.z0 - 1 + rr / HL;
            ok = ok && zz >= 0 && yy >= 0 && yy + zz <= S - 1 && ch.x0 - 1 <= yy;
            const int lo = max(ch.x0 - 1, 0) - (ch.x0 - 32), hi = min(ch.x0 + ch.w + 32, yy) - (ch.x0 - 32);
            long long F = 0;
            if (ok) F = (long long)(__ldg(PZ + zz) + tri_idx(0, yy)) + ch.x0 - 32;
            const long long Fa = F & ~31ll;
            const int d = int(F - Fa);
            const int klo = (lo + d) >> 5, khi = (hi + d) >> 5;  // pieces holding needed bytes
            uint4 va[NW + 2], vb[NW + 2];
            bool tail[NW + 2];
#pragma unroll
            for (int k = 0; k < NW + 2; ++k) {
                va[k] = make_uint4(0, 0, 0, 0);
                vb[k] = va[k];
                tail[k] = false;
                if (ok && k >= klo && k <= khi) {
                    const long long A = Fa + 32ll * k;
                    if ((unsigned long long)(A + 32) <= ncells) {
                        const uint4* q = reinterpret_cast<const uint4*>(cur + A);
                        va[k] = __ldg(q);
                        vb[k] = __ldg(q + 1);
                    } else {
                        tail[k] = true;
                    }
                }
            }
            uint32_t p[NW + 3];
#pragma unroll
            for (int k = 0; k < NW + 2; ++k) {
                p[k] = pack32(va[k], vb[k]);
                if (tail[k]) p[k] = tail_bits(cur, Fa + 32ll * k, ncells);
            }
            p[NW + 2] = 0u;
            uint32_t f[NW + 2];
#pragma unroll
            for (int j = 0; j < NW + 2; ++j)
                f[j] = ok ? __funnelshift_r(p[j], p[j + 1], d) & range_mask(lo - 32 * j, hi - 32 * j) : 0u;
#pragma unroll
            for (int i = 1; i <= NW; ++i) {
                const uint32_t l = __funnelshift_l(f[i - 1], f[i], 1);   // cell x-1
                const uint32_t rg = __funnelshift_r(f[i], f[i + 1], 1);  // cell x+1
                hrow[3 * (i - 1)] = l ^ f[i] ^ rg;
                hrow[3 * (i - 1) + 1] = (l & f[i]) | (l & rg) | (f[i] & rg);
                hrow[3 * (i - 1) + 2] = f[i];
            }
        }
        __syncwarp();

        // ---- march along z: lane (chunk slot, ly, word) ----
        {
            const int cl = lane / C::SLOT, t = lane % C::SLOT;
            const int ly = t / NW, w = t % NW;
            if (cl < C::CPI) {
                const uint32_t* H = sH + cl * HL2 * HW + 3 * w;
                auto vsum = [&](int zi) {
                    const uint32_t* r0 = H + (zi * HL + ly) * HW;
                    return add3x2(r0[0], r0[1], r0[HW], r0[HW + 1], r0[2 * HW], r0[2 * HW + 1]);
                };
                Planes4 p0 = vsum(0), p1 = vsum(1);
#pragma unroll
                for (int lz = 0; lz < RHO; ++lz) {
                    const Planes4 p2 = vsum(lz + 2);
                    const uint32_t alive = H[((lz + 1) * HL + ly + 1) * HW + 2];
                    sO[lz * C::OSTR + lane] = life_planes(p0, p1, p2, alive);
                    p0 = p1;
                    p1 = p2;
                }
            }
        }
        __syncwarp();

        // ---- store: a lane per output row; 16-byte aligned windows plus
        // power-of-two head / tail pieces, every owned cell written once ----
        for (int q = lane; q < C::OROWS; q += 32) {
            const int cl = q / (RHO * RHO), lz = (q / RHO) % RHO, ly = q % RHO;
            const int ci = item * C::CPI + cl;
            if (ci >= nchunks) continue;
            const Chunk ch = s_chunk[ci];
            const int y = ch.y0 + ly, z = ch.z0 + lz;
            if (y + z > S - 1 || ch.x0 > y) continue;
            // Sector ownership: a 32-byte sector of the packed state is written
            // by the chunk holding its first cell, so the chunk's range moves
            // from [x0, x0 + w) to [ceil32, ceil32) of its packed ends: up to 31
            // cells go to the left neighbour chunk and up to 31 of the right
            // neighbour's are computed here. Row ends stay exact (the sector
            // there is shared with the adjacent packed row). Sub-range launches
            // (`exact`) keep tile ownership so shards write only their tiles.
            const long long R = (long long)(__ldg(PZ + z) + tri_idx(0, y));
            const int xe = min(ch.x0 + ch.w, y + 1);
            long long E0 = R + ch.x0, E1 = R + xe;
            if (!exact) {
                if (ch.x0 > 0) E0 = (E0 + 31) & ~31ll;
                if (xe < y + 1) E1 = min((E1 + 31) & ~31ll, R + y + 1);
                if (E0 >= E1) continue;
            }
            const int n = int(E1 - E0);
            const int off0 = int(E0 - R) - ch.x0;  // cell offset of E0 in the computed words
            const uint32_t* o = sO + lz * C::OSTR + cl * C::SLOT + ly * NW;
            auto put = [&](auto kk, long long pos) {
                constexpr int K = decltype(kk)::value;
                store_cells<K>(next, pos, o, int(pos - E0) + off0);
            };
            const long long a_lo = (E0 + 15) & ~15ll, a_hi = E1 & ~15ll;
            if (a_lo <= a_hi) {
                // head [E0, a_lo): the 2^k piece at ceil(E0, 2^k) when that bit is set
#define SMX_HEAD(K)                                                              \
    {                                                                            \
        const long long pk = (E0 + ((1ll << K) - 1)) & ~((1ll << K) - 1);        \
        if (((pk >> K) & 1ll) && pk < a_lo) put(std::integral_constant<int, K>(), pk);  \
    }
                SMX_HEAD(0) SMX_HEAD(1) SMX_HEAD(2) SMX_HEAD(3)
#undef SMX_HEAD
                for (long long A = a_lo; A < a_hi; A += 16) put(std::integral_constant<int, 4>(), A);
                // tail [a_hi, E1): larger pieces first
                const int L = int(E1 - a_hi);
#define SMX_TAIL(K)                                                              \
    if ((L >> K) & 1) {                                                          \
        const long long pos = a_hi + (L & ~((2 << K) - 1));                      \
        put(std::integral_constant<int, K>(), pos);                             \
    }
                SMX_TAIL(3) SMX_TAIL(2) SMX_TAIL(1) SMX_TAIL(0)
#undef SMX_TAIL
            } else {
                // the whole row sits inside one 16-byte window: < 16 bytes
                for (int t = 0; t < n; ++t) put(std::integral_constant<int, 0>(), E0 + t);
            }
        }
        __syncwarp();
    }
}

template <int KIND, int RHO>
void launch_fused_t(const Geom& g, int wz0, int wz1, const uint8_t* cur, uint8_t* next, cudaStream_t s) {
    using C = FCfg<RHO>;
    constexpr int NZMAX = 2;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(k_ca_fused<KIND, RHO>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             C::smem(C::LMAX * C::LMAX * NZMAX));
        attr_set = true;
    }
    // patch edge and layers per CTA: as large as possible while the grid still
    // has >= 4 CTAs per SM (small grids trade chunk length for parallelism)
    int P = C::LMAX, NZ = NZMAX;
    auto ctas = [&](int p, int nz) {
        return (long long)((g.ex + p - 1) / p) * ((g.ey + p - 1) / p) * ((wz1 - wz0 + nz - 1) / nz);
    };
    while (NZ > 1 && ctas(P, NZ) < 4 * 148) NZ /= 2;
    while (P > 4 && ctas(P, NZ) < 4 * 148) P = P / 2 > 4 ? P / 2 : 4;
    const dim3 grid((g.ex + P - 1) / P, (g.ey + P - 1) / P, (wz1 - wz0 + NZ - 1) / NZ);
    const int exact = (wz0 > 0 || wz1 < g.ez) ? 1 : 0;
    k_ca_fused<KIND, RHO><<<grid, F_NTHR, C::smem(P * P * NZ), s>>>(g, wz0, wz1, P, NZ, exact, cur, next,
                                                                    tet_cells(g.side));
}

template <int KIND>
void launch_fused_kind(const Geom& g, int wz0, int wz1, const uint8_t* cur, uint8_t* next, cudaStream_t s) {
    if (g.rho == 4) launch_fused_t<KIND, 4>(g, wz0, wz1, cur, next, s);
    else launch_fused_t<KIND, 8>(g, wz0, wz1, cur, next, s);
}

}  // namespace

void launch_ca_fused(const Geom& g, int wz0, int wz1, const uint8_t* cur, uint8_t* next, cudaStream_t s) {
    if (wz1 <= wz0) return;
    if (g.kind == SMX_H3D) launch_fused_kind<SMX_H3D>(g, wz0, wz1, cur, next, s);
    else launch_fused_kind<SMX_BB>(g, wz0, wz1, cur, next, s);
}

}  // namespace smx
