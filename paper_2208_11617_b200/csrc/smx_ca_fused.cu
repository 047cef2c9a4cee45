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
    // computed words per row: frame bit i is cell x0 - 1 + i; the words cover
    // the owned cells plus up to 31 cells of the next chunk (sector ownership,
    // see the store phase): [x0 - 1, x0 + w + 31) within NW words
    static constexpr int NW = (LMAX * RHO + 32 + 31) / 32;  // 4 / 3
    // halo row copy: NCH 16-byte chunks from floor16 of the row's cell x0 - 1
    // (start residue d <= 15) hold the needed cells up to x0 + w + 32
    static constexpr int NCH = (LMAX * RHO + 34 + 15 + 15) / 16;  // 10 / 8
    static constexpr int PKW = NCH / 2;                  // packed 32-bit words per row
    static_assert(PKW >= NW + 1 && NCH % 2 == 0, "row copy must cover the halo words");
    static constexpr int RSTR = (NCH + 1) * 16;          // odd chunk stride: conflict-free lane-per-row reads
    static constexpr int HL = RHO + 2;                   // halo rows == halo layers
    static constexpr int HL2 = HL * HL;
    static constexpr int SLOT = RHO * NW;                // march lanes per chunk slot
    static constexpr int CPI = 32 / SLOT;                // chunks per warp item (1 / 2)
    static constexpr int HROWS = CPI * HL2;              // halo rows per item
    static constexpr int NPASS = (HROWS + 3) / 4;        // copy passes: 4 rows x 8 lanes
    static constexpr int OROWS = CPI * RHO * RHO;        // output rows per item
    static constexpr int HW = 3 * NW;                    // smem words per halo row: (h0, h1, raw) x NW
    static constexpr int OSTR = 33;                      // smem words per output layer (32 lanes + pad)
    // per-warp smem: raw rows | h-sums | outputs | row descriptors
    static constexpr int H_OFF = HROWS * RSTR;
    static constexpr int O_OFF = H_OFF + HROWS * HW * 4;
    static constexpr int D_OFF = (O_OFF + (RHO * OSTR + 1) * 4 + 15) & ~15;
    static constexpr int WARP_BYTES = (D_OFF + HROWS * 16 + 127) & ~127;
    static int smem(int nb) { return F_NWARP * WARP_BYTES + nb * 48 + 16; }
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// 16-byte async copy global -> shared; bytes beyond `valid` are zero-filled
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(valid) : "memory");
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
                                                     long long ncells) {
    using C = FCfg<RHO>;
    constexpr int HL = C::HL, HL2 = C::HL2, NW = C::NW, HW = C::HW;
    extern __shared__ __align__(128) uint8_t fsm[];
    const int NBP = P * P * NZ;
    int4* s_tile = reinterpret_cast<int4*>(fsm + F_NWARP * C::WARP_BYTES);
    Chunk* s_chunk = reinterpret_cast<Chunk*>(s_tile + NBP);
    int* s_nchunks = reinterpret_cast<int*>(s_chunk + NBP);
    uint32_t* s_link = reinterpret_cast<uint32_t*>(s_chunk + NBP) + 4;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int grp = lane >> 3, gl = lane & 7;
    const int S = g.side;
    const unsigned long long* __restrict__ PZ = g.prefix;
    uint8_t* sR = fsm + warp * C::WARP_BYTES;                     // [HROWS][RSTR] raw u8 rows
    uint32_t* sH = reinterpret_cast<uint32_t*>(sR + C::H_OFF);     // [HROWS][HW]
    uint32_t* sO = reinterpret_cast<uint32_t*>(sR + C::O_OFF);     // [RHO][OSTR] (+1 pad word)
    int4* sD = reinterpret_cast<int4*>(sR + C::D_OFF);             // [HROWS] row descriptors

    const int nchunks =
        build_chunks<KIND>(g, wz0 + blockIdx.z * NZ, wz1, P, NZ, C::LMAX, s_tile, s_chunk, s_nchunks, s_link);
    const int nitems = (nchunks + C::CPI - 1) / C::CPI;

    for (int item = warp; item < nitems; item += F_NWARP) {
        // ---- row descriptors (a lane per halo row) ----
        // Frame bit i of a row is cell x = x0 - 1 + i. The row's bytes are
        // copied from c0 = floor16(packed index of x0 - 1), frame bit 0 at
        // byte d = F - c0. Cells outside the row (x < 0, x > y) are masked dead.
        for (int r = lane; r < C::HROWS; r += 32) {
            const int cl = r / HL2, rr = r - cl * HL2;
            const int ci = item * C::CPI + cl;
            bool ok = ci < nchunks;
            const Chunk ch = ok ? s_chunk[ci] : Chunk{0, 0, 0, 0};
            const int yy = ch.y0 - 1 + rr % HL, zz = ch.z0 - 1 + rr / HL;
            ok = ok && zz >= 0 && yy >= 0 && yy + zz <= S - 1 && ch.x0 - 1 <= yy;
            const int lo = ch.x0 == 0 ? 1 : 0, hi = min(ch.x0 + ch.w + 32, yy) - (ch.x0 - 1);
            const long long F = ok ? (long long)(__ldg(PZ + zz) + tri_idx(0, yy)) + ch.x0 - 1 : 0;
            const long long c0 = F & ~15ll;  // >= -16
            sD[r] = make_int4(int(c0 & 0xffffffffll), int(c0 >> 32), ok ? (lo | (int(F - c0) << 4) | (hi << 16)) : -1, 0);
        }
        __syncwarp();

        // ---- copy: 8 lanes x 16 bytes per row, 4 rows per pass (coalesced) ----
#pragma unroll 4
        for (int pass = 0; pass < C::NPASS; ++pass) {
            const int r = pass * 4 + grp;
            if (r >= C::HROWS) break;
            const int4 dsc = sD[r];
            if (dsc.z < 0) continue;
            const long long c0 = ((long long)dsc.y << 32) | (unsigned)dsc.x;
            const uint32_t dst = smem_u32(sR + r * C::RSTR);
#pragma unroll
            for (int k = gl; k < C::NCH; k += 8) {
                const long long o = c0 + 16 * k;
                const long long v = o < 0 ? 0 : min(ncells - o, 16ll);
                cp_async16(dst + 16 * k, v > 0 ? cur + o : cur, int(v > 0 ? v : 0));
            }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        __syncwarp();

        // ---- bits + horizontal 3-sums: a lane per halo row ----
        for (int r = lane; r < C::HROWS; r += 32) {
            const int lh = sD[r].z;
            uint32_t* hrow = sH + r * HW;
            uint32_t f[NW + 1];
            if (lh < 0) {
#pragma unroll
                for (int j = 0; j <= NW; ++j) f[j] = 0u;
            } else {
                const int lo = lh & 1, d = (lh >> 4) & 15, hi = lh >> 16;
                const uint4* q = reinterpret_cast<const uint4*>(sR + r * C::RSTR);
                uint32_t pk[C::PKW + 1];  // row bytes as bits, 32 per word
#pragma unroll
                for (int k = 0; k < C::PKW; ++k) pk[k] = pack32(q[2 * k], q[2 * k + 1]);
                pk[C::PKW] = 0u;
#pragma unroll
                for (int j = 0; j <= NW; ++j)
                    f[j] = __funnelshift_r(pk[j], pk[j + 1], d) & range_mask(lo - 32 * j, hi - 32 * j);
            }
#pragma unroll
            for (int i = 0; i < NW; ++i) {
                const uint32_t l = __funnelshift_l(i > 0 ? f[i - 1] : 0u, f[i], 1);  // cell x-1
                const uint32_t rg = __funnelshift_r(f[i], f[i + 1], 1);            // cell x+1
                hrow[3 * i] = l ^ f[i] ^ rg;
                hrow[3 * i + 1] = (l & f[i]) | (l & rg) | (f[i] & rg);
                hrow[3 * i + 2] = f[i];
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
            const int off0 = int(E0 - R) - ch.x0 + 1;  // frame offset of E0 (frame bit 0 = cell x0 - 1)
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
    static std::once_flag once[kMaxDevices];  // once per device (thread-safe)
    once_per_device(once, current_device(), [] {
        cudaFuncSetAttribute(k_ca_fused<KIND, RHO>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             C::smem(C::LMAX * C::LMAX * NZMAX));
    });
    // patch edge and layers per CTA: as large as possible while the grid still
    // has >= 2 CTAs per SM (small grids trade chunk length for parallelism)
    int P = C::LMAX, NZ = NZMAX;
    auto ctas = [&](int p, int nz) {
        return (long long)((g.ex + p - 1) / p) * ((g.ey + p - 1) / p) * ((wz1 - wz0 + nz - 1) / nz);
    };
    while (NZ > 1 && ctas(P, NZ) < 4 * 148) NZ /= 2;
    while (P > 4 && ctas(P, NZ) < 4 * 148) P = P / 2 > 4 ? P / 2 : 4;
    const dim3 grid((g.ex + P - 1) / P, (g.ey + P - 1) / P, (wz1 - wz0 + NZ - 1) / NZ);
    const int exact = (wz0 > 0 || wz1 < g.ez) ? 1 : 0;
    k_ca_fused<KIND, RHO><<<grid, F_NTHR, C::smem(P * P * NZ), s>>>(g, wz0, wz1, P, NZ, exact, cur, next,
                                                                    (long long)tet_cells(g.side));
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
