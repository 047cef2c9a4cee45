// 3-D Life, sm_100a: the bit-shadow engine (SMX_EXEC_BITS; what launch_ca runs).
//
// k_pack_bits    u8 state -> "bit shadow": one bit per cell in a PITCHED layout,
//                every packed row (y, z) padded to WP 32-bit words at word row
//                z*S + y (a full S x S square per layer stack, so (w, y, z) is
//                an affine 3-D tensor for TMA; rows y > S-1-z are never used).
//                A warp walks up to 32 rows, 8 lanes per row, streaming each
//                row's bytes as 32-byte aligned chunks (2 x 16B loads per lane),
//                packing them (IMAD gather + PRMT) and realigning at the bit level.
// k_ca_plan      the map, applied ONCE per launch_ca: a CTA maps a P x P patch of
//                map blocks lane-parallel and chains x-adjacent tiles
//                (ca::build_chunks) into chunks of <= 96 cells, appended to one
//                global chunk list.
// k_ca_bits_run  ONE persistent cooperative launch (one 16-warp CTA per SM) runs
//                every step over the chunk list: warps take items (1-2 chunks)
//                round-robin; per chunk one 3-D TMA tensor box (12 words x rho+2
//                rows x rho+2 layers) lands its halo in shared memory
//                (double-buffered across items, mbarrier completion), lanes form
//                the horizontal 3-sums as bit-planes, and lane (ly, w) marches z
//                with carry-save adders (32 cells per LOP3). Output is whole
//                32-bit words: a word shared by two chunks gets identical values
//                from both (same input), so the writes are idempotent. A grid
//                barrier separates the steps.
// k_ca_bits      one step with the map evaluated inside the launch (per-CTA patch
//                -> chunks in smem -> the same item loop): smx_bits_step and the
//                multi-GPU range steps.
// k_unpack_bits  bit shadow -> u8 state: 16-byte vector stores over each row's
//                aligned interior, byte stores for its two ends.
//
// launch_ca = pack -> plan -> run (all steps) -> unpack; one full-grid u8 step
// (smx_ca_step, large states) is the same with one step.
//
// Semantics: alive_neighbors_3d_dead + life_next (simulator.hpp:220-253) for
// every cell of every tile the map emits; each tile is processed by exactly one
// chunk. Bits for x > y of a row (not cells) are never trusted: every reader
// masks them.
#include <cstdlib>
#include <cooperative_groups.h>
#include <type_traits>
#include <cuda.h>

#include "smx_ca_common.cuh"
#include "smx_launch.hpp"

namespace smx {

int bits_pitch_words(int side);

namespace {

using namespace ca;

constexpr int OWN = 96;   // max owned cells per chunk row
// words per TMA box row: the box must start on a 16-byte (4-word) boundary, so
// it starts at floor4(w0 - 1) and 12 words always cover words w0-1 .. w0+4.
constexpr int BOXW = 12;
constexpr int NWARP = 4;  // warps per CTA
constexpr int NTHR = NWARP * 32;

// chunking: tiles per chunk and the per-launch scheme's patch (blocks per CTA)
template <int RHO>
struct PlanCfg {
    static constexpr int LMAX = OWN / RHO;              // tiles per chunk
    static constexpr int P = LMAX;                      // patch edge (blocks)
    static constexpr int NZ = 4;                        // max wz layers per CTA
    static constexpr int NB = P * P * NZ;               // max blocks per CTA
};

// CPIX: chunks per warp item (default: as many as the 32 lanes can march, 32 /
// (4 rho)); the persistent small-grid runs use 1 to halve an item's latency.
template <int RHO, int CPIX = 32 / (RHO * 4)>
struct Cfg {
    static constexpr int HL = RHO + 2;                  // halo layers == halo rows per layer
    static constexpr int LPC = RHO * 4;                 // compute lanes per chunk
    static constexpr int CPI = CPIX;                    // chunks per warp item
    static_assert(CPI >= 1 && CPI * LPC <= 32, "an item's chunks must fit the warp's lanes");
    static constexpr int BOXB = HL * HL * BOXW * 4;     // bytes per TMA box (one per chunk)
    static constexpr int SLOT = (BOXB + 127) & ~127;    // 128B-aligned slot per box
    static constexpr int BUF = CPI * SLOT;              // one buffer: the boxes of an item
    static constexpr int HROWS = CPI * HL * HL;         // halo rows per item
    // per warp: 2 TMA buffers | h-sums | mbarriers (64 B) | a cached chunk list
    // (the persistent kernel's items when a warp owns <= LIST_ITEMS of them)
    static constexpr int LIST_ITEMS = 8;
    static constexpr int LIST_OFF = 2 * BUF + HROWS * 32 + 64;
    static constexpr int WARP_BYTES = (LIST_OFF + LIST_ITEMS * CPI * 16 + 127) & ~127;  // TMA dst: 128B aligned
    static int smem(int nb) { return NWARP * WARP_BYTES + nb * 48 + 128; }
};

__device__ __forceinline__ int layer_row(int z, int S) { return z * S - (z * (z - 1)) / 2; }

// ---- PTX helpers ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(a), "r"(bytes) : "memory");
}
// the waiting thread is suspended (up to the hint, 10 ms) until the phase
// completes instead of spinning: no issue slots burnt while the box lands
__device__ __forceinline__ bool mbar_try_wait(uint32_t a, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 10000000;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint32_t mbar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];\n" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(mbar)
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// 32 bytes at 32B-aligned byte offset A of a u8 array of n bytes -> 32 bits
__device__ __forceinline__ uint32_t load_chunk_bits(const uint8_t* __restrict__ p, long long A,
                                                    unsigned long long n) {
    if ((unsigned long long)(A + 32) <= n) {
        const uint4* q = reinterpret_cast<const uint4*>(p + A);
        return pack32(__ldg(q), __ldg(q + 1));
    }
    uint32_t v = 0;
    for (int i = 0; i < 32; ++i)
        if ((unsigned long long)(A + i) < n) v |= uint32_t(p[A + i] & 1) << i;
    return v;
}

// ---------------------------------------------------------------------------
// Row walk shared by pack/unpack. A warp owns rpw (<= 32, a multiple of 4)
// consecutive rows and works on 4 of them at a time, one 8-lane group per row (group g takes rows
// r0+g, r0+g+4, ...): per-row bookkeeping is shared by the 8 lanes of a group
// and each lane moves 32 bytes per pass.
constexpr int ROWS_PER_WARP = 32;

struct RowCursor {
    int z, y;
    long long rowbase;  // packed index of cell (0, y, z)
};

// packed row r -> (z, y): layer z holds S - z rows, so rows before layer z are
// layer_row(z) = z (2S + 1 - z) / 2; z = floor of the smaller root of
// z^2 - (2S+1) z + 2r = 0, corrected by one either way (no dependent loads)
__device__ __forceinline__ RowCursor row_at(int row, int S, const unsigned long long* __restrict__ PZ) {
    const float b = 2.0f * S + 1.0f;  // fp32 root: off by at most a few, fixed below
    int z = int((b - sqrtf(fmaxf(b * b - 8.0f * float(row), 0.0f))) * 0.5f);
    if (z < 0) z = 0;
    if (z > S - 1) z = S - 1;
    while (z > 0 && layer_row(z, S) > row) --z;
    while (z < S - 1 && layer_row(z + 1, S) <= row) ++z;
    const int y = row - layer_row(z, S);
    return RowCursor{z, y, (long long)(PZ[z] + tri_idx(0, y))};
}

__device__ __forceinline__ void row_next(RowCursor& c, int S, const unsigned long long* __restrict__ PZ) {
    if (c.y + 1 + c.z <= S - 1) {
        c.rowbase += c.y + 1;
        ++c.y;
    } else {
        ++c.z;
        c.y = 0;
        c.rowbase = (long long)PZ[c.z];
    }
}

// u8 packed state -> pitched bit shadow (bits beyond x = y are zero).
__global__ void __launch_bounds__(256) k_pack_bits(const uint8_t* __restrict__ cur, uint32_t* __restrict__ bits,
                                                   int S, int WP, int nrows, const unsigned long long* __restrict__ PZ,
                                                   unsigned long long ncells, int rpw) {
    const int lane = threadIdx.x & 31, grp = lane >> 3, gl = lane & 7;
    const unsigned gmask = 0xffu << (8 * grp);
    const int row0 = (blockIdx.x * 8 + (threadIdx.x >> 5)) * rpw;
    int r = row0 + grp;
    if (r >= nrows) return;
    RowCursor c = row_at(r, S, PZ);
    for (;;) {
        const int n = c.y + 1, nw = (n + 31) >> 5;
        const long long A0 = c.rowbase & ~31ll;
        const int d = int(c.rowbase - A0);
        uint32_t* out = bits + ((long long)c.z * S + c.y) * WP;
        // lane gl packs chunk k; word k needs chunks k and k+1, so a pass emits
        // 7 words (lanes 0..6) and the next pass starts 7 chunks on. Software
        // pipelined: the next pass's 32 bytes are loaded before this pass is
        // packed and stored
        const long long rowend = c.rowbase + n;
        auto fetch = [&](int base, uint4& x0, uint4& x1) {
            const long long ck = A0 + 32ll * (base + gl);
            x0 = x1 = make_uint4(0u, 0u, 0u, 0u);
            if (ck < rowend && (unsigned long long)(ck + 32) <= ncells) {
                const uint4* q = reinterpret_cast<const uint4*>(cur + ck);
                x0 = __ldg(q);
                x1 = __ldg(q + 1);
            }
        };
        uint4 n0, n1;
        fetch(0, n0, n1);
        for (int base = 0; base < nw; base += 7) {
            const uint4 x0 = n0, x1 = n1;
            if (base + 7 < nw) fetch(base + 7, n0, n1);
            const int k = base + gl;
            const long long ck = A0 + 32ll * k;
            uint32_t B = pack32(x0, x1);
            if (ck < rowend && (unsigned long long)(ck + 32) > ncells) B = load_chunk_bits(cur, ck, ncells);  // array end
            const uint32_t Bn = __shfl_down_sync(gmask, B, 1, 8);
            if (gl < 7 && k < nw) {
                uint32_t wv = d ? __funnelshift_r(B, Bn, d) : B;
                const int valid = n - 32 * k;
                if (valid < 32) wv &= (1u << valid) - 1u;
                out[k] = wv;
            }
        }
        r += 4;
        if (r >= nrows || r >= row0 + rpw) break;
#pragma unroll
        for (int t = 0; t < 4; ++t) row_next(c, S, PZ);
    }
}

// pitched bit shadow -> u8 packed state. Interior 16-byte windows of a row
// are vector stores; the <= 15 + 15 bytes at the row's two ends (shared with the
// neighbouring rows' windows) are byte stores.
__global__ void __launch_bounds__(256) k_unpack_bits(const uint32_t* __restrict__ bits, uint8_t* __restrict__ out,
                                                     int S, int WP, int nrows,
                                                     const unsigned long long* __restrict__ PZ, int rpw) {
    const int lane = threadIdx.x & 31, grp = lane >> 3, gl = lane & 7;
    const int row0 = (blockIdx.x * 8 + (threadIdx.x >> 5)) * rpw;
    int r = row0 + grp;
    if (r >= nrows) return;
    RowCursor c = row_at(r, S, PZ);
    for (;;) {
        const int n = c.y + 1;
        const uint32_t* src = bits + ((long long)c.z * S + c.y) * WP;
        const long long e0 = c.rowbase, e1 = c.rowbase + n;
        long long a_lo = (e0 + 15) & ~15ll, a_hi = e1 & ~15ll;
        if (a_lo > a_hi) a_lo = a_hi = e1;  // no full window: every byte is an edge byte
        const int nwin = int((a_hi - a_lo) >> 4);
        // group pass: 16 consecutive windows (256 B); lane gl writes windows
        // base+gl and base+8+gl so each store instruction covers 128 B per row;
        // the bit words of UB passes are loaded before any window is stored
        // (C5: 400 -> 376 us)
        constexpr int UB = 4;
        for (int base = 0; base < nwin; base += 16 * UB) {
            uint32_t w[UB][2][2];
#pragma unroll
            for (int u = 0; u < UB; ++u)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int k = base + 16 * u + 8 * h + gl;
                    const int x = int(a_lo + 16ll * k - e0), j = x >> 5, o = x & 31;
                    w[u][h][0] = k < nwin ? __ldg(src + j) : 0u;
                    w[u][h][1] = k < nwin && o > 16 ? __ldg(src + j + 1) : 0u;
                }
#pragma unroll
            for (int u = 0; u < UB; ++u)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int k = base + 16 * u + 8 * h + gl;
                    if (k < nwin) {
                        const long long A = a_lo + 16ll * k;
                        const int o = int(A - e0) & 31;
                        *reinterpret_cast<uint4*>(out + A) = spread16(__funnelshift_r(w[u][h][0], w[u][h][1], o) & 0xffffu);
                    }
                }
        }
        const int nhead = int(a_lo - e0), ntail = int(e1 - a_hi);
        for (int t = gl; t < nhead + ntail; t += 8) {
            const long long pos = t < nhead ? e0 + t : a_hi + (t - nhead);
            const int x = int(pos - e0);
            out[pos] = (uint8_t)((__ldg(src + (x >> 5)) >> (x & 31)) & 1u);
        }
        r += 4;
        if (r >= nrows || r >= row0 + rpw) break;
#pragma unroll
        for (int t = 0; t < 4; ++t) row_next(c, S, PZ);
    }
}

// TMA issue for one warp item (lane 0): one 3-D box (12 words x rho+2 rows x
// rho+2 layers) per chunk; out-of-range coordinates land as zeros.
template <int RHO, int CPIX>
__device__ __forceinline__ void issue_item(const CUtensorMap* tm, const Chunk* s_chunk, int nchunks, int item,
                                           uint8_t* buf, uint32_t mbar) {
    using C = Cfg<RHO, CPIX>;
    const int nc = min(C::CPI, nchunks - item * C::CPI);
    mbar_expect_tx(mbar, uint32_t(nc * C::BOXB));
    for (int c = 0; c < nc; ++c) {
        const Chunk ch = s_chunk[item * C::CPI + c];
        const int w0 = ch.x0 >> 5;
        const int c0 = (w0 - 1) - ((w0 - 1) & 3);
        tma_load_3d(smem_u32(buf + c * C::SLOT), tm, c0, ch.y0 - 1, ch.z0 - 1, mbar);
    }
}

// ---------------------------------------------------------------------------
// One warp's share of a step: items item0, item0 + istride, ... of a chunk list
// (CPI chunks per item). Per item ONE 3-D TMA box per chunk lands the halo in
// shared memory (double-buffered across items, mbarrier completion), lanes
// form the horizontal 3-sums as bit-planes, then lane (ly, w) marches z and
// writes whole 32-bit words of the next bit shadow. `phases` carries the two
// mbarriers' parities across calls (the persistent kernel reuses them).
template <int RHO, int CPIX = 32 / (RHO * 4)>
__device__ __forceinline__ void run_items(const Chunk* __restrict__ s_chunk, int nchunks, int item0, int istride,
                                          const CUtensorMap* tm, uint32_t* __restrict__ nbits, int S, int WP,
                                          uint8_t* wbase, uint32_t mbar0, uint32_t& phases) {
    using C = Cfg<RHO, CPIX>;
    constexpr int HL = C::HL;
    const int lane = threadIdx.x & 31;
    uint32_t* sH = reinterpret_cast<uint32_t*>(wbase + 2 * C::BUF);  // [HROWS][4][2]: (h0, h1) of words 0..3
    const int nitems = (nchunks + C::CPI - 1) / C::CPI;
    int item = item0, b = 0;
    if (item < nitems && lane == 0) {
        fence_proxy_async();
        issue_item<RHO, CPIX>(tm, s_chunk, nchunks, item, wbase, mbar0);
    }
    for (; item < nitems; item += istride, b ^= 1) {
        const int nxt = item + istride;
        if (nxt < nitems && lane == 0) {
            fence_proxy_async();
            issue_item<RHO, CPIX>(tm, s_chunk, nchunks, nxt, wbase + (b ^ 1) * C::BUF, mbar0 + 8 * (b ^ 1));
        }
        while (!mbar_try_wait(mbar0 + 8 * b, (phases >> b) & 1u)) {
        }
        phases ^= 1u << b;
        const uint8_t* buf = wbase + b * C::BUF;

        // ---- 3. horizontal 3-sums (bit-planes), lane per halo row ----
#pragma unroll
        for (int pass = 0; pass < (C::HROWS + 31) / 32; ++pass) {
            const int r = lane + 32 * pass;
            if (r >= C::HROWS) break;
            const int c = r / (HL * HL), rr = r % (HL * HL);  // lane/pass constants, hoisted by the unroll
            const int zi = rr / HL, yi = rr % HL;
            const int ci = item * C::CPI + c;
            uint4 h0 = make_uint4(0, 0, 0, 0), h1 = h0;
            if (ci < nchunks) {
                const Chunk ch = s_chunk[ci];
                const int zz = ch.z0 - 1 + zi, yy = ch.y0 - 1 + yi;
                if (zz >= 0 && yy >= 0 && yy + zz <= S - 1) {
                    const int off = ((ch.x0 >> 5) - 1) & 3;  // box word of w0 - 1
                    const uint32_t* src =
                        reinterpret_cast<const uint32_t*>(buf + c * C::SLOT + (zi * HL + yi) * BOXW * 4) + off;
                    uint32_t T[6];
#pragma unroll
                    for (int j = 0; j < 6; ++j) T[j] = src[j];
                    const int xb = ((ch.x0 >> 5) - 1) * 32;  // x of T[0] bit 0
                    if (xb + 191 > yy) {
                        // keep cells x <= yy (x < 0 words are TMA zero-fill): the low
                        // yy - x + 1 bits, clamped to [0, 32] by the funnel shift
#pragma unroll
                        for (int j = 0; j < 6; ++j)
                            T[j] &= __funnelshift_lc(0xffffffffu, 0u, max(yy - (xb + 32 * j) + 1, 0));
                    }
                    uint32_t a[4], bb[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint32_t cc = T[j + 1];
                        const uint32_t l = __funnelshift_l(T[j], cc, 1);
                        const uint32_t rg = __funnelshift_r(cc, T[j + 2], 1);
                        a[j] = l ^ cc ^ rg;
                        bb[j] = (l & cc) | (l & rg) | (cc & rg);
                    }
                    h0 = make_uint4(a[0], a[1], a[2], a[3]);
                    h1 = make_uint4(bb[0], bb[1], bb[2], bb[3]);
                }
            }
            reinterpret_cast<uint4*>(sH + 8 * r)[0] = make_uint4(h0.x, h1.x, h0.y, h1.y);
            reinterpret_cast<uint4*>(sH + 8 * r)[1] = make_uint4(h0.z, h1.z, h0.w, h1.w);
        }
        __syncwarp();

        // ---- 4. march along z: vertical sums, rule, stores ----
        {
            // ZS lane groups split the z-march of a chunk when an item's chunks
            // leave lanes free (rho = 4, one chunk per item: 2 x 16 lanes, each
            // marching rho / 2 layers): shorter per-item latency
            constexpr int ZS = 32 / (C::LPC * C::CPI) >= 2 && RHO % 2 == 0 ? 2 : 1;
            constexpr int LZN = RHO / ZS;  // layers per lane
            const int zg = ZS > 1 ? lane / (C::LPC * C::CPI) : 0;
            const int lane_c = ZS > 1 ? lane % (C::LPC * C::CPI) : lane;
            const int cl = lane_c / C::LPC, l = lane_c % C::LPC;
            const int ly = l >> 2, w = l & 3;
            const int lz0 = zg * LZN;
            const int ci = item * C::CPI + cl;
            const bool cvalid = cl < C::CPI && ci < nchunks;
            const Chunk ch = cvalid ? s_chunk[ci] : Chunk{0, 0, 0, 0};
            const int cs = cl < C::CPI ? cl : 0;  // idle lanes (cl >= CPI) read slot 0, never store
            const uint32_t* H = sH + 8 * (cs * HL * HL);
            const uint8_t* cbuf = buf + cs * C::SLOT;
            auto vsum = [&](int zi) {
                const int r0 = zi * HL + ly;
                const uint2 p = reinterpret_cast<const uint2*>(H + 8 * r0)[w];
                const uint2 q = reinterpret_cast<const uint2*>(H + 8 * (r0 + 1))[w];
                const uint2 u = reinterpret_cast<const uint2*>(H + 8 * (r0 + 2))[w];
                return vsum3(p.x, p.y, q.x, q.y, u.x, u.y);
            };
            V3 va = vsum(lz0), vb = vsum(lz0 + 1);
            const int y = ch.y0 + ly;
            const int w0 = ch.x0 >> 5;
            const int xw = 32 * (w0 + w);  // x of this lane's word
            const int lastw = (ch.x0 + ch.w - 1) >> 5;
            // layers z0 .. zmax-1 of this lane's word are cells (y + z <= S - 1);
            // the output pointer steps one layer (S rows) per z
            const int zmax = (cvalid && ch.x0 <= y && w0 + w <= lastw && xw <= y) ? min(ch.z0 + RHO, S - y) : 0;
            const long long zstep = (long long)S * WP;
            uint32_t* optr = nbits + ((long long)(ch.z0 + lz0) * S + y) * WP + w0 + w;
            const uint32_t* arow = reinterpret_cast<const uint32_t*>(cbuf + (HL + ly + 1) * BOXW * 4) +
                                   ((w0 - 1) & 3) + 1 + w;
#pragma unroll 2
            for (int lz = lz0; lz < lz0 + LZN; ++lz) {
                const V3 vc = vsum(lz + 2);
                const uint32_t alive = arow[lz * HL * BOXW];
                const uint32_t O = life_v3(va, vb, vc, alive, 0xffffffffu);
                va = vb;
                vb = vc;
                if (ch.z0 + lz < zmax) *optr = O;
                optr += zstep;
            }
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// Per-launch scheme: the CTA maps its P x P x NZ patch, builds its chunks in
// shared memory and runs them (one launch per step; smx_bits_step).
template <int KIND, int RHO>
__global__ void __launch_bounds__(NTHR) k_ca_bits(Geom g, int wz0, const __grid_constant__ CUtensorMap tmap,
                                                  uint32_t* __restrict__ nbits, int WP, int P, int NZ, int wz1) {
    using C = Cfg<RHO>;
    const int NBP = P * P * NZ;  // blocks of this CTA: a P x P patch at NZ consecutive wz
    extern __shared__ __align__(128) uint8_t smem[];
    int4* s_tile = reinterpret_cast<int4*>(smem + NWARP * C::WARP_BYTES);
    Chunk* s_chunk = reinterpret_cast<Chunk*>(smem + NWARP * C::WARP_BYTES + NBP * 16);
    int* s_nchunks = reinterpret_cast<int*>(smem + NWARP * C::WARP_BYTES + 2 * NBP * 16);
    uint32_t* s_link = reinterpret_cast<uint32_t*>(smem + NWARP * C::WARP_BYTES + 2 * NBP * 16 + 16);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint8_t* wbase = smem + warp * C::WARP_BYTES;
    const uint32_t mbar0 = smem_u32(wbase + 2 * C::BUF + C::HROWS * 32);
    if (lane == 0) {
        mbar_init(mbar0, 1);
        mbar_init(mbar0 + 8, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    const int nchunks =
        build_chunks<KIND>(g, wz0 + blockIdx.z * NZ, wz1, P, NZ, PlanCfg<RHO>::LMAX, s_tile, s_chunk, s_nchunks, s_link);
    uint32_t phases = 0u;
    run_items<RHO>(s_chunk, nchunks, warp, NWARP, &tmap, nbits, g.side, WP, wbase, mbar0, phases);
}

// ---------------------------------------------------------------------------
// Multi-step engine (smx_ca, EXEC_BITS). The map is applied ONCE per launch_ca
// call: k_ca_plan maps every patch of the grid and appends its chunks to one
// global list; k_ca_bits_run is a persistent cooperative kernel that runs all
// the steps over that list (every warp takes items round-robin, so consecutive
// items — spatial neighbours — run concurrently) with a grid barrier between
// steps. No per-step launch or re-mapping; the chain-building cost is paid once.
constexpr int PLAN_THREADS = 512;

template <int KIND, int RHO>
__global__ void __launch_bounds__(PLAN_THREADS) k_ca_plan(Geom g, int wz0, int wz1, int P, int NZ, Chunk* __restrict__ out,
                                                  unsigned* __restrict__ count) {
    using C = Cfg<RHO>;
    const int NBP = P * P * NZ;
    extern __shared__ __align__(128) uint8_t smem[];
    int4* s_tile = reinterpret_cast<int4*>(smem);
    Chunk* s_chunk = reinterpret_cast<Chunk*>(smem + NBP * 16);
    int* s_nchunks = reinterpret_cast<int*>(smem + 2 * NBP * 16);
    uint32_t* s_link = reinterpret_cast<uint32_t*>(smem + 2 * NBP * 16 + 16);
    __shared__ unsigned s_base;
    const int n = build_chunks<KIND>(g, wz0 + blockIdx.z * NZ, wz1, P, NZ, PlanCfg<RHO>::LMAX, s_tile, s_chunk, s_nchunks, s_link);
    if (threadIdx.x == 0) s_base = atomicAdd(count, unsigned(n));
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[s_base + i] = s_chunk[i];
}

// Between steps: every CTA's generic-proxy stores of this step must be visible
// to the next step's TMA (async-proxy) loads in other CTAs: a proxy fence,
// then the cooperative-groups grid barrier (cumulative gpu-scope release /
// acquire), then a proxy fence before the next TMA issue. Measured per-step
// floor on B200 (tools/step_floor.py): 3.1 us with grid.sync() vs 3.4 us with
// a hand-rolled acq_rel counter barrier; 5.1 vs 5.9 us at C2.
//
// The barrier is the cooperative-groups algorithm (one arrival counter; the
// master's arrival flips its top bit) with a nanosleep back-off in the poll:
// same latency (1.19 vs 1.20 us, tools/barrier_probe.cu), but a CTA that
// arrives early no longer burns the issue slots a co-resident CTA still
// computing its items needs (the spin was 10 % of all C2 instructions). `bar`
// is a zeroed word of the launch's control block; cooperative launch keeps
// every CTA resident.
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void step_barrier(unsigned* bar) {
    asm volatile("fence.proxy.async.global;\n" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned nb = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1) : 1u;
        __threadfence();
        const unsigned old = atomicAdd(bar, nb);
        while (((old ^ ld_acquire_gpu(bar)) & 0x80000000u) == 0) __nanosleep(64);
    }
    __syncthreads();
    asm volatile("fence.proxy.async.global;\n" ::: "memory");
}

// persistent kernel: one 16-warp CTA per SM (fewer barrier arrivals), the
// default chunks per item (measured: 1 chunk per item with 32 warps per SM is
// 8 % slower at C2 — the per-item fixed costs dominate there)
template <int RHO, int NWX = 16, int CPIY = 32 / (RHO * 4)>
struct RunCfg {
    static constexpr int NW = NWX;
    static constexpr int CPIX = CPIY;
};

template <int RHO, int NWX = 16, int CPIY = 32 / (RHO * 4)>
__global__ void __launch_bounds__(NWX * 32) k_ca_bits_run(const __grid_constant__ CUtensorMap tmA,
                                                      const __grid_constant__ CUtensorMap tmB, uint32_t* bitsA,
                                                      uint32_t* bitsB, const Chunk* __restrict__ chunks,
                                                      unsigned* count, int steps, int S, int WP) {
    using C = Cfg<RHO, CPIY>;
    constexpr int RUN_NWARP = NWX;
    extern __shared__ __align__(128) uint8_t smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint8_t* wbase = smem + warp * C::WARP_BYTES;
    const uint32_t mbar0 = smem_u32(wbase + 2 * C::BUF + C::HROWS * 32);
    if (lane == 0) {
        mbar_init(mbar0, 1);
        mbar_init(mbar0 + 8, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    }
    const int nchunks = int(*count);
    // items go to SMs first (warp w of CTA b is global warp w * grid + b): a grid
    // with fewer items than warps spreads them over every SM instead of filling
    // the first CTAs' 16 warps and leaving the rest idle
    const int gwarp = warp * gridDim.x + blockIdx.x, nwarps = gridDim.x * RUN_NWARP;
    // A warp runs the same items every step. When it owns few (small grids),
    // copy their chunks once into its smem list, so no step waits on a global
    // read of a chunk before issuing its TMA box.
    const Chunk* src = chunks;
    int nsrc = nchunks, i0 = gwarp, istr = nwarps;
    {
        const int nitems = (nchunks + C::CPI - 1) / C::CPI;
        const int mine = gwarp < nitems ? (nitems - 1 - gwarp) / nwarps + 1 : 0;
        if (mine <= C::LIST_ITEMS) {
            Chunk* loc = reinterpret_cast<Chunk*>(wbase + C::LIST_OFF);
            int nloc = 0;
            for (int k = 0; k < mine * C::CPI; ++k) {
                const int ci = (gwarp + (k / C::CPI) * nwarps) * C::CPI + k % C::CPI;
                if (ci < nchunks) {
                    if (lane == 0) loc[k] = chunks[ci];
                    nloc = k + 1;
                }
            }
            __syncwarp();
            src = loc;
            nsrc = nloc;
            i0 = 0;
            istr = 1;
        }
    }
    uint32_t phases = 0u;
    for (int st = 0; st < steps; ++st) {
        const bool even = (st & 1) == 0;
        run_items<RHO, CPIY>(src, nsrc, i0, istr, even ? &tmA : &tmB, even ? bitsB : bitsA, S, WP,
                                          wbase, mbar0, phases);
        if (st + 1 < steps) step_barrier(count + 8);  // count: word 0 of the zeroed 64-byte control block
    }
}

template <int KIND, int RHO>
void launch_t(const Geom& g, int wz0, int wz1, const CUtensorMap& tmap, uint32_t* nbits, int WP, cudaStream_t s) {
    using C = Cfg<RHO>;
    static std::once_flag once[kMaxDevices];  // once per device (thread-safe)
    once_per_device(once, current_device(), [] {
        cudaFuncSetAttribute(k_ca_bits<KIND, RHO>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::smem(PlanCfg<RHO>::NB));
    });
    // patch edge: the largest that still gives >= 4 CTAs per SM (small grids
    // trade chunk length for parallelism)
    // and up to NZ wz layers per CTA (more chunks per warp keep the TMA
    // double buffer busy) while the grid still gives >= 4 CTAs per SM
    int P = PlanCfg<RHO>::P, NZ = PlanCfg<RHO>::NZ;
    auto ctas = [&](int p, int nz) {
        return (long long)((g.ex + p - 1) / p) * ((g.ey + p - 1) / p) * ((wz1 - wz0 + nz - 1) / nz);
    };
    while (NZ > 1 && ctas(P, NZ) < 4 * 148) NZ /= 2;
    while (P > 4 && ctas(P, NZ) < 4 * 148) P = P / 2 > 4 ? P / 2 : 4;
    const dim3 grid((g.ex + P - 1) / P, (g.ey + P - 1) / P, (wz1 - wz0 + NZ - 1) / NZ);
    k_ca_bits<KIND, RHO><<<grid, NTHR, C::smem(P * P * NZ), s>>>(g, wz0, tmap, nbits, WP, P, NZ, wz1);
}

template <int KIND, int RHO>
void launch_plan_t(const Geom& g, int wz0, int wz1, void* chunks, unsigned* count, cudaStream_t s) {
    using C = Cfg<RHO>;
    // Chains stop at patch edges. H3D: 32 x 32 patches (32 divides the n/2
    // extents, so the hinge fold and the slab levels fragment least: H3D(128)
    // 36.3 K chunks vs 40.7 K at P = 12); BB: P = 2-3 LMAX (rows of the box are
    // unbroken chains cut every LMAX tiles from wx = 0, so any multiple of LMAX
    // gives the same chunks): rho = 8, 3 LMAX = 36 keeps the 512 threads busy
    // (BB plan 61 -> 32 us at C4, 463 -> 199 us at C5); rho = 4, LMAX (more
    // CTAs win at C2: 8.6 vs 13.8 us at 2 LMAX).
    const int P = KIND == SMX_H3D ? 32 : PlanCfg<RHO>::LMAX * (RHO == 8 ? 3 : 1), NZ = 1;
    const int smem = 2 * P * P * NZ * 16 + 16 + 4 * P * P * NZ * 4;  // tiles | chunks | count | links
    static std::once_flag once[kMaxDevices];  // once per device (thread-safe)
    once_per_device(once, current_device(),
                    [&] { cudaFuncSetAttribute(k_ca_plan<KIND, RHO>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); });
    if (wz1 <= wz0) return;
    const dim3 grid((g.ex + P - 1) / P, (g.ey + P - 1) / P, wz1 - wz0);
    k_ca_plan<KIND, RHO><<<grid, PLAN_THREADS, smem, s>>>(g, wz0, wz1, P, NZ, reinterpret_cast<Chunk*>(chunks), count);
}

template <int RHO, int NWX, int CPIY>
cudaError_t launch_run_t(const Geom& g, const CUtensorMap& tA, const CUtensorMap& tB, uint32_t* A, uint32_t* B,
                         const void* chunks, const unsigned* count, int steps, cudaStream_t s, bool coop = true) {
    using C = Cfg<RHO, CPIY>;
    const int smem = NWX * C::WARP_BYTES;
    // attribute + persistent grid (co-resident CTAs x SMs) once per device
    static std::once_flag once[kMaxDevices];
    static int grids[kMaxDevices];
    const int dev = current_device();
    int grid_local = 0;
    once_per_device(once, dev, [&] {
        cudaFuncSetAttribute(k_ca_bits_run<RHO, NWX, CPIY>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        int per_sm = 0, nsm = 148;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ca_bits_run<RHO, NWX, CPIY>, NWX * 32, smem);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        grid_local = (per_sm > 0 ? per_sm : 1) * nsm;
        if (dev >= 0 && dev < kMaxDevices) grids[dev] = grid_local;
    });
    int grid = dev >= 0 && dev < kMaxDevices ? grids[dev] : grid_local;
    const Chunk* ch = reinterpret_cast<const Chunk*>(chunks);
    int S = g.side, WP = bits_pitch_words(g.side);
    unsigned* ctl = const_cast<unsigned*>(count);
    void* args[] = {const_cast<CUtensorMap*>(&tA), const_cast<CUtensorMap*>(&tB), &A, &B, &ch, &ctl, &steps, &S, &WP};
    if (!coop && steps == 1)  // one step executes no grid barrier: an ordinary launch
        return cudaLaunchKernel((const void*)k_ca_bits_run<RHO, NWX, CPIY>, dim3(grid), dim3(NWX * 32), args, smem, s);
    return cudaLaunchCooperativeKernel((const void*)k_ca_bits_run<RHO, NWX, CPIY>, dim3(grid), dim3(NWX * 32), args,
                                       smem, s);
}

// ===========================================================================
// The COLUMN engine (large states): the map applied once marks every tile it
// emits in a tile bitmap (k_cols_mark: one thread per map block, so its cost
// is the block count: H3D maps 5.3x fewer blocks than BB); the run is a
// persistent kernel whose work items are columns of the domain — 8 cell rows
// x 8 words (256 cells) x a run of z layers — that a warp marches along z:
// 3-D TMA stages of 8 layers (16 words x 10 rows x 8 layers, double-buffered,
// mbarrier completion), each input layer's horizontal 3-sums computed ONCE
// (10 rows x 8 words, shared through shared memory), the vertical 3-sums kept
// in registers across the march (a rolling window of three layers), the rule
// applied with carry-save adders on 32 cells per LOP3, and the output word
// masked by the bitmap (only the cells of tiles the map emitted are written;
// the others are zero, as the reference's unvisited cells of a fresh state).
// Items are taken dynamically (one atomic per item); a grid barrier separates
// the steps.
constexpr int CW = 8;                    // output words per item row (256 cells)
constexpr int CR = 8;                    // output rows per item
constexpr int CBW = 16;                  // box words: 8 g - 4 .. 8 g + 11 (16-byte aligned start)
constexpr int CBR = CR + 2;              // box rows: y0 - 1 .. y0 + 8
constexpr int CLZ = 8;                   // layers per TMA stage
constexpr int CSTAGE = CBW * CBR * CLZ * 4;  // 5120 B
constexpr int CLAYER = CBW * CBR * 4;        // 640 B per layer of a stage
constexpr int CHS = 2 * CBR * CW * 8;        // h-sums of two layers: [parity][10 rows][8 words][a, b]
constexpr int CWARP = 2 * CSTAGE + CHS;  // 11520 B per warp (90 x 128); the mbarriers follow all warps' regions
constexpr int CNW = 16;                  // warps per CTA (persistent: one CTA per SM; 20 measured slower: 202 vs 195 us per C5 step)

struct ColItem {
    int iy, g, z0, z1;  // rows 8 iy .. 8 iy + 7, words 8 g .. 8 g + 7, layers z0 .. z1 - 1
};

template <int KIND>
__global__ void __launch_bounds__(256) k_cols_mark(Geom g, uint32_t* __restrict__ bm, int D, int TW,
                                                    unsigned* __restrict__ stats, int wz0, int wz1) {
    // blocks with wz in [wz0, wz1) (a shard's whole levels; the full grid: 0, ez)
    const long long plane = (long long)g.ex * g.ey, nb = plane * (wz1 - wz0);
    unsigned marked = 0, dup = 0;
    for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < nb;
         b += (long long)gridDim.x * blockDim.x) {
        const int wx = int(b % g.ex), wy = int(b / g.ex % g.ey), wz = wz0 + int(b / plane);
        const outcome<int> o = map_block<KIND>(g, wx, wy, wz);
        if (o.is_void) continue;
        const uint32_t bit = 1u << (o.x & 31);
        const uint32_t old = atomicOr(bm + ((long long)o.z * D + o.y) * TW + (o.x >> 5), bit);
        ++marked;
        dup += (old & bit) ? 1u : 0u;
    }
    for (int d = 16; d; d >>= 1) {
        marked += __shfl_xor_sync(0xffffffffu, marked, d);
        dup += __shfl_xor_sync(0xffffffffu, dup, d);
    }
    if ((threadIdx.x & 31) == 0 && (marked | dup)) {
        atomicAdd(stats, marked);
        atomicAdd(stats + 1, dup);
    }
}

// 2 cell words' coverage mask from the tile bitmap: word k of the lane covers
// tiles 32 (w + k) / RHO ...; every tile bit becomes RHO cell bits
// a lane's bitmap word for tile row (ty, tz) (its two output words' tiles
// start at bit t0 & 31, t0 = w * 32 / RHO; w even: the 2 * 32 / RHO bits share
// one word); 0 past the domain. Loaded a stage ahead of its use (tile_mask2).
__device__ __forceinline__ uint32_t tile_word(const uint32_t* __restrict__ bm, int D, int TW, int t0, int ty, int tz) {
    if (ty >= D || tz >= D) return 0u;
    return __ldg(bm + ((long long)tz * D + ty) * TW + (t0 >> 5));
}
template <int RHO>
__device__ __forceinline__ uint2 tile_mask2(uint32_t word, int t0) {
    constexpr int TPW = 32 / RHO;  // tiles per cell word
    const uint32_t bits = word >> (t0 & 31);
    uint32_t m[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const uint32_t b = (bits >> (k * TPW)) & ((1u << TPW) - 1u);
        if (RHO == 16) {
            m[k] = ((b & 1u) ? 0x0000ffffu : 0u) | ((b & 2u) ? 0xffff0000u : 0u);  // bit i -> half i
        } else if (RHO == 8) {
            m[k] = ((b * 0x00204081u) & 0x01010101u) * 0xffu;  // bit i -> byte i
        } else {
            uint32_t v = 0;  // bit i -> nibble i
#pragma unroll
            for (int i = 0; i < 8; ++i) v |= ((b >> i) & 1u) * (0xfu << (4 * i));
            m[k] = v;
        }
    }
    return make_uint2(m[0], m[1]);
}

__device__ __forceinline__ void cols_issue(const CUtensorMap* tm, const ColItem& it, int stage, uint8_t* buf,
                                           uint32_t mbar) {
    mbar_expect_tx(mbar, uint32_t(CSTAGE));
    tma_load_3d(smem_u32(buf), tm, 8 * it.g - 4, 8 * it.iy - 1, it.z0 - 1 + CLZ * stage, mbar);
}

// One step of the column engine for one warp: items grabbed from *ctr until
// the list is exhausted. `seq` counts the TMA stages this warp has issued
// (buffer = seq & 1, parity = (seq >> 1) & 1), carried across steps.
//
// Per input layer (box rows y0-1 .. y0+8, box words w0-4 .. w0+11):
//   h-sums: 20 lanes, lane (row hr = lane >> 1, half hc = lane & 1) loads the
//     aligned 16-byte chunk of x words w0 + 4 hc .. +3 and ONE edge word (w0-1
//     or w0+8); the word across the middle comes from its partner lane by one
//     shuffle; 4 horizontal 3-sums as two bit-planes -> shared memory
//   vertical 3-sums: lane (ly = lane >> 2, words jp = 2 (lane & 3), +1), three
//     16-byte loads, kept in registers for three layers
//   rule + masked 8-byte store for the output layer one behind.
// x << 1 | prev >> 31 and x >> 1 | next << 31: one funnel shift each (the
// FMA-pipe pair IMAD.HI + IMAD used earlier measured 0.5 % slower at C4 and
// C5 once the ALU pipe stopped being the limit: 53 % busy, latency bound)
__device__ __forceinline__ uint32_t shl1(uint32_t prev, uint32_t x) { return __funnelshift_l(prev, x, 1); }
__device__ __forceinline__ uint32_t shr1(uint32_t x, uint32_t next) { return __funnelshift_r(x, next, 1); }

template <int RHO>
__device__ __forceinline__ void cols_step(const ColItem* __restrict__ items, int nitems, unsigned* ctr,
                                          const CUtensorMap* tm, uint32_t* __restrict__ out,
                                          const uint32_t* __restrict__ bm, int D, int TW, int S, int WP,
                                          uint8_t* wbase, uint32_t mbar0, uint32_t& seq) {
    static_assert(CLZ == 8 && (RHO == 16 || RHO == 8 || RHO == 4), "stage = 8 layers; tiles of 16, 8 or 4 layers");
    // the tile index of output layer z0 - 2 + 8 st + li: for RHO = 8 and 16 it
    // changes only between li = 1 and 2 (z0 and the stage start are multiples
    // of 8), for RHO = 4 also between li = 5 and 6
    const int lane = threadIdx.x & 31;
    uint2* hsb = reinterpret_cast<uint2*>(wbase + 2 * CSTAGE);  // 2 x [CBR][CW] (a, b), by layer parity
    const int hr = min(lane >> 1, CBR - 1), hc = lane & 1;      // h-sum role (lanes 0..19; 20..31 mirror row 9)
    const int ly = lane >> 2, jp = 2 * (lane & 3);              // output role
    const long long zstride = (long long)S * WP;
    // item indices come from one atomic per item, grabbed an item ahead by
    // lane 0, which also loads the item and issues its first stage; the other
    // lanes get it by shuffle only when they need it (the atomic's and the
    // load's latency overlap the current item). The bitmap words of a stage's
    // tile masks are loaded a stage ahead.
    int cur = 0;
    ColItem it{0, 0, 0, 0};
    if (lane == 0) {
        cur = int(atomicAdd(ctr, 1u));
        if (cur < nitems) {
            it = items[cur];
            fence_proxy_async();
            cols_issue(tm, it, 0, wbase + (seq & 1) * CSTAGE, mbar0 + 8 * (seq & 1));
        }
    }
    cur = __shfl_sync(0xffffffffu, cur, 0);
    it.iy = __shfl_sync(0xffffffffu, it.iy, 0);
    it.g = __shfl_sync(0xffffffffu, it.g, 0);
    it.z0 = __shfl_sync(0xffffffffu, it.z0, 0);
    it.z1 = __shfl_sync(0xffffffffu, it.z1, 0);
    constexpr int TPW = 32 / RHO;
    // the first stage's bitmap words (layer z0 of tile row (y / RHO, z0 / RHO))
    uint32_t bw0 = 0u, bw1 = 0u;
    if (cur < nitems) {
        const int yo = 8 * it.iy + ly, t0 = (8 * it.g + jp) * TPW;
        bw0 = tile_word(bm, D, TW, t0, yo / RHO, it.z0 / RHO);
        if (RHO == 4) bw1 = tile_word(bm, D, TW, t0, yo / RHO, it.z0 / RHO + 1);
    }
    while (cur < nitems) {
        int nxt = 0;
        ColItem itn{0, 0, 0, 0};
        if (lane == 0) {
            nxt = int(atomicAdd(ctr, 1u));
            if (nxt < nitems) itn = items[nxt];
        }
        // input layers z0 - 1 .. z1 (z0 is a multiple of 8): full stages of 8
        // layers, then a tail stage of the rest
        const int nin = it.z1 - it.z0 + 2;
        const int nfull = nin / CLZ, tail = nin % CLZ;
        const int nst = nfull + (tail ? 1 : 0);
        const int y0 = 8 * it.iy, w0 = 8 * it.g;
        // no input masking: every non-cell bit of the shadow is zero (rows above
        // the tetrahedron's face, words and bits past x = y: the pack writes
        // them zero, these stores mask them, the pools start zeroed) and the
        // box's out-of-range coordinates are TMA zero-fill
        const int hoff = hr * CBW + 4 + 4 * hc;  // box word of the main chunk
        const int eoff = hr * CBW + (hc ? 12 : 3);
        uint2* hsw = hsb + hr * CW + 4 * hc;      // this lane's h-sum slots (parity 0)
        // output role, per item
        const int yo = y0 + ly, wo = w0 + jp;
        const int ozlim = min(S - 1 - yo, it.z1 - 1);  // stored layers: z0 <= zo <= ozlim
        const int smode = 32 * (wo + 1) <= yo ? 2 : (32 * wo <= yo ? 1 : 0);
        // x <= y within this lane's two output words (keeps the zero invariant)
        const uint32_t xm0 = __funnelshift_lc(0xffffffffu, 0u, max(yo - 32 * wo + 1, 0));
        const uint32_t xm1 = __funnelshift_lc(0xffffffffu, 0u, max(yo - 32 * wo - 31, 0));
        uint32_t* optr = out + ((long long)(it.z0 - 2) * S + yo) * WP + wo;  // output layer of input layer z0 - 1
        V3 va[2], vb[2];
        uint32_t alive_cur0 = 0u, alive_cur1 = 0u;
        uint2 mprev = make_uint2(0u, 0u);

        // h-sums of input layer li (all 32 lanes store: lanes 20..31 repeat
        // row 9's values, which keeps the code branch-free)
        auto hsum = [&](const uint32_t* L, int li) {
            const uint4 m = *reinterpret_cast<const uint4*>(L + hoff);
            const uint32_t e = L[eoff];
            const uint32_t got = __shfl_xor_sync(0xffffffffu, hc ? m.x : m.w, 1);  // partner's word
            const uint32_t W0 = hc ? got : e, W5 = hc ? e : got;
            const uint32_t l0 = shl1(W0, m.x), r0 = shr1(m.x, m.y);
            const uint32_t l1 = shl1(m.x, m.y), r1 = shr1(m.y, m.z);
            const uint32_t l2 = shl1(m.y, m.z), r2 = shr1(m.z, m.w);
            const uint32_t l3 = shl1(m.z, m.w), r3 = shr1(m.w, W5);
            uint4* dst = reinterpret_cast<uint4*>(hsw + (li & 1) * (CBR * CW));
            dst[0] = make_uint4(lop3<0x96>(l0, m.x, r0), lop3<0xe8>(l0, m.x, r0), lop3<0x96>(l1, m.y, r1),
                                lop3<0xe8>(l1, m.y, r1));
            dst[1] = make_uint4(lop3<0x96>(l2, m.z, r2), lop3<0xe8>(l2, m.z, r2), lop3<0x96>(l3, m.w, r3),
                                lop3<0xe8>(l3, m.w, r3));
        };
        // input layer li of a stage of n: its h-sums are in shared memory; the
        // next layer's h-sums are computed while its vertical sums and the rule
        // for the layer behind run (independent work for the scheduler)
        auto layer = [&](const uint32_t* buf, int li, int n, int zi, const uint2& m0, const uint2& m1, bool first) {
            __syncwarp();  // h-sums of layer li visible; layer li - 1's reads done
            const uint2* hs = hsb + (li & 1) * (CBR * CW);
            const uint4 p = *reinterpret_cast<const uint4*>(hs + ly * CW + jp);
            const uint4 q = *reinterpret_cast<const uint4*>(hs + (ly + 1) * CW + jp);
            const uint4 u = *reinterpret_cast<const uint4*>(hs + (ly + 2) * CW + jp);
            const uint2 an = *reinterpret_cast<const uint2*>(buf + li * (CLAYER / 4) + (ly + 1) * CBW + 4 + jp);
            if (li + 1 < n) hsum(buf + (li + 1) * (CLAYER / 4), li + 1);
            V3 vc[2];
            vc[0] = vsum3(p.x, p.y, q.x, q.y, u.x, u.y);
            vc[1] = vsum3(p.z, p.w, q.z, q.w, u.z, u.w);
            // the rule for output layer zo = zi - 1 (stored when z0 <= zo <= ozlim;
            // skipped for the item's two warm-up layers, zo = z0 - 2, z0 - 1)
            if (li >= 2 || !first) {
                const uint2 tmk = li < 2 ? mprev : (RHO == 4 && li >= 6 ? m1 : m0);
                const uint32_t o0 = life_v3(va[0], vb[0], vc[0], alive_cur0, tmk.x);
                const uint32_t o1 = life_v3(va[1], vb[1], vc[1], alive_cur1, tmk.y);
                const int zo = zi - 1;
                if (zo >= it.z0 && zo <= ozlim) {
                    if (smode == 2) *reinterpret_cast<uint2*>(optr) = make_uint2(o0, o1);
                    else if (smode == 1) *optr = o0;
                }
            }
            optr += zstride;
            va[0] = vb[0];
            va[1] = vb[1];
            vb[0] = vc[0];
            vb[1] = vc[1];
            alive_cur0 = an.x;
            alive_cur1 = an.y;
        };

        const int t0 = wo * TPW;
        for (int st = 0; st < nst; ++st) {
            const uint32_t b = seq & 1;
            // the other buffer is free (its stage was consumed): prefetch the
            // next stage of this item, or the first stage of the next item
            if (lane == 0) {
                fence_proxy_async();
                if (st + 1 < nst) cols_issue(tm, it, st + 1, wbase + (b ^ 1) * CSTAGE, mbar0 + 8 * (b ^ 1));
                else if (nxt < nitems) cols_issue(tm, itn, 0, wbase + (b ^ 1) * CSTAGE, mbar0 + 8 * (b ^ 1));
            }
            // output layers of this stage: z0 - 2 + 8 st + li; their tile masks
            // (from the words loaded a stage ago), and the next stage's words
            uint2 m0 = tile_mask2<RHO>(bw0, t0);
            uint2 m1 = RHO == 4 ? tile_mask2<RHO>(bw1, t0) : m0;
            m0.x &= xm0, m0.y &= xm1, m1.x &= xm0, m1.y &= xm1;
            if (st + 1 < nst) {
                const int zt = it.z0 + CLZ * (st + 1);
                bw0 = tile_word(bm, D, TW, t0, yo / RHO, zt / RHO);
                if (RHO == 4) bw1 = tile_word(bm, D, TW, t0, yo / RHO, zt / RHO + 1);
            } else {
                // the next item: broadcast (lane 0 loaded it an item ago)
                nxt = __shfl_sync(0xffffffffu, nxt, 0);
                itn.iy = __shfl_sync(0xffffffffu, itn.iy, 0);
                itn.g = __shfl_sync(0xffffffffu, itn.g, 0);
                itn.z0 = __shfl_sync(0xffffffffu, itn.z0, 0);
                itn.z1 = __shfl_sync(0xffffffffu, itn.z1, 0);
                if (nxt < nitems) {
                    const int nyo = 8 * itn.iy + ly, nt0 = (8 * itn.g + jp) * TPW;
                    bw0 = tile_word(bm, D, TW, nt0, nyo / RHO, itn.z0 / RHO);
                    if (RHO == 4) bw1 = tile_word(bm, D, TW, nt0, nyo / RHO, itn.z0 / RHO + 1);
                }
            }
            while (!mbar_try_wait(mbar0 + 8 * b, (seq >> 1) & 1u)) {
            }
            const uint32_t* buf = reinterpret_cast<const uint32_t*>(wbase + b * CSTAGE);
            const int zbase = it.z0 - 1 + CLZ * st;
            __syncwarp();  // the previous stage's last h-sum reads are done
            hsum(buf, 0);
            const bool first = st == 0;
            if (st < nfull) {
#pragma unroll
                for (int li = 0; li < CLZ; ++li) layer(buf, li, CLZ, zbase + li, m0, m1, first);
            } else if (tail == 2) {
                // the usual tail (items of a multiple of 8 layers read 2 more)
                layer(buf, 0, 2, zbase, m0, m1, first);
                layer(buf, 1, 2, zbase + 1, m0, m1, first);
            } else {
                // other tails (segments cut by the tetrahedron's face): one rolled copy
#pragma unroll 1
                for (int li = 0; li < tail; ++li) layer(buf, li, tail, zbase + li, m0, m1, first);
            }
            mprev = RHO == 4 ? m1 : m0;
            ++seq;
        }
        cur = nxt;
        it = itn;
    }
}

// ---- the 12-row column shape ----
// Items of 12 output rows x 8 words: the 14 box rows give 28 of the 32 lanes
// an h-sum role (the 8-row shape: 20), and each lane owns ONE word of three
// consecutive output rows (rows oc .. oc + 2, oc = 3 (lane >> 3), word
// lane & 7): five h-sum rows loaded (two shared between its three vertical
// sums), three independent rule chains per lane. The double-buffered 14-row
// stages take 16128 B per warp: 14 warps per SM.
constexpr int C2R = 12;                        // output rows per item
constexpr int C2BR = C2R + 2;                  // box rows: y0 - 1 .. y0 + 12
constexpr int C2STAGE = CBW * C2BR * CLZ * 4;  // 7168 B
constexpr int C2LAYER = CBW * C2BR * 4;        // 896 B per layer of a stage
constexpr int C2HS = 2 * C2BR * CW * 8;        // h-sums of two layers: [parity][14 rows][8 words][a, b]
constexpr int C2WARP = 2 * C2STAGE + C2HS;     // 16128 B per warp (126 x 128)
constexpr int C2NW = 14;                       // warps per CTA (227 KB of shared memory)

// a lane's one cell word's coverage mask from its bitmap word (tiles t0 ..)
template <int RHO>
__device__ __forceinline__ uint32_t tile_mask1(uint32_t word, int t0) {
    constexpr int TPW = 32 / RHO;
    const uint32_t b = (word >> (t0 & 31)) & ((1u << TPW) - 1u);
    if (RHO == 16) return ((b & 1u) ? 0x0000ffffu : 0u) | ((b & 2u) ? 0xffff0000u : 0u);
    if (RHO == 8) return ((b * 0x00204081u) & 0x01010101u) * 0xffu;  // bit i -> byte i
    uint32_t v = 0;                                                   // bit i -> nibble i
#pragma unroll
    for (int i = 0; i < 8; ++i) v |= ((b >> i) & 1u) * (0xfu << (4 * i));
    return v;
}

__device__ __forceinline__ void cols_issue12(const CUtensorMap* tm, const ColItem& it, int stage, uint8_t* buf,
                                             uint32_t mbar) {
    mbar_expect_tx(mbar, uint32_t(C2STAGE));
    tma_load_3d(smem_u32(buf), tm, 8 * it.g - 4, C2R * it.iy - 1, it.z0 - 1 + CLZ * stage, mbar);
}

// One step of the 12-row column engine for one warp (the structure of
// cols_step: items from *ctr, TMA stages of 8 layers double-buffered, h-sums
// once per input layer, rolling vertical sums, masked stores).
template <int RHO>
__device__ __forceinline__ void cols_step12(const ColItem* __restrict__ items, int nitems, unsigned* ctr,
                                            const CUtensorMap* tm, uint32_t* __restrict__ out,
                                            const uint32_t* __restrict__ bm, int D, int TW, int S, int WP,
                                            uint8_t* wbase, uint32_t mbar0, uint32_t& seq) {
    static_assert(CLZ == 8 && (RHO == 16 || RHO == 8 || RHO == 4), "stage = 8 layers; tiles of 16, 8 or 4 layers");
    const int lane = threadIdx.x & 31;
    uint2* hsb = reinterpret_cast<uint2*>(wbase + 2 * C2STAGE);  // 2 x [C2BR][CW] (a, b), by layer parity
    const int hr = min(lane >> 1, C2BR - 1), hc = lane & 1;      // h-sum role (lanes 0..27; 28..31 mirror row 13)
    const int oc = 3 * (lane >> 3), ow = lane & 7;               // output role: item rows oc .. oc + 2, word ow
    const long long zstride = (long long)S * WP;
    constexpr int TPW = 32 / RHO;
    int cur = 0;
    ColItem it{0, 0, 0, 0};
    if (lane == 0) {
        cur = int(atomicAdd(ctr, 1u));
        if (cur < nitems) {
            it = items[cur];
            fence_proxy_async();
            cols_issue12(tm, it, 0, wbase + (seq & 1) * C2STAGE, mbar0 + 8 * (seq & 1));
        }
    }
    cur = __shfl_sync(0xffffffffu, cur, 0);
    it.iy = __shfl_sync(0xffffffffu, it.iy, 0);
    it.g = __shfl_sync(0xffffffffu, it.g, 0);
    it.z0 = __shfl_sync(0xffffffffu, it.z0, 0);
    it.z1 = __shfl_sync(0xffffffffu, it.z1, 0);
    // bitmap words of a stage's tile layer(s) for the lane's two tile rows
    // (rows oc .. oc + 2 span at most two), loaded a stage ahead
    uint32_t bwa0 = 0u, bwb0 = 0u, bwa1 = 0u, bwb1 = 0u;
    auto load_bw = [&](const ColItem& c, int z) {
        const int ya = C2R * c.iy + oc, t0 = (8 * c.g + ow) * TPW;
        const int ta = ya / RHO, tb = (ya + 2) / RHO;
        bwa0 = tile_word(bm, D, TW, t0, ta, z / RHO);
        bwb0 = tile_word(bm, D, TW, t0, tb, z / RHO);
        if (RHO == 4) {
            bwa1 = tile_word(bm, D, TW, t0, ta, z / RHO + 1);
            bwb1 = tile_word(bm, D, TW, t0, tb, z / RHO + 1);
        }
    };
    if (cur < nitems) load_bw(it, it.z0);
    while (cur < nitems) {
        int nxt = 0;
        ColItem itn{0, 0, 0, 0};
        if (lane == 0) {
            nxt = int(atomicAdd(ctr, 1u));
            if (nxt < nitems) itn = items[nxt];
        }
        const int nin = it.z1 - it.z0 + 2;
        const int nfull = nin / CLZ, tail = nin % CLZ;
        const int nst = nfull + (tail ? 1 : 0);
        const int y0 = C2R * it.iy, w0 = 8 * it.g;
        const int hoff = hr * CBW + 4 + 4 * hc;  // box word of the main chunk
        const int eoff = hr * CBW + (hc ? 12 : 3);
        uint2* hsw = hsb + hr * CW + 4 * hc;
        // output role, per item: rows yo + k, word wo
        const int yo = y0 + oc, wo = w0 + ow;
        const bool sel1 = (yo + 1) / RHO != yo / RHO;  // row 1's tile row is row 2's
        unsigned zn[3];
        uint32_t xm[3];
        uint32_t* optr[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            // stored layers z0 <= zo < z0 + zn[k] (none when the word holds no cell of the row)
            zn[k] = 32 * wo <= yo + k ? unsigned(max(min(S - 1 - (yo + k), it.z1 - 1) - it.z0 + 1, 0)) : 0u;
            xm[k] = __funnelshift_lc(0xffffffffu, 0u, max(yo + k - 32 * wo + 1, 0));  // x <= y
            optr[k] = out + ((long long)(it.z0 - 2) * S + yo + k) * WP + wo;  // output layer of input layer z0 - 1
        }
        V3 va[3], vb[3];
        uint32_t alive[3] = {0u, 0u, 0u}, mprev[3] = {0u, 0u, 0u};

        auto hsum = [&](const uint32_t* L, int li) {
            const uint4 m = *reinterpret_cast<const uint4*>(L + hoff);
            const uint32_t e = L[eoff];
            const uint32_t got = __shfl_xor_sync(0xffffffffu, hc ? m.x : m.w, 1);  // partner's word
            const uint32_t W0 = hc ? got : e, W5 = hc ? e : got;
            const uint32_t l0 = shl1(W0, m.x), r0 = shr1(m.x, m.y);
            const uint32_t l1 = shl1(m.x, m.y), r1 = shr1(m.y, m.z);
            const uint32_t l2 = shl1(m.y, m.z), r2 = shr1(m.z, m.w);
            const uint32_t l3 = shl1(m.z, m.w), r3 = shr1(m.w, W5);
            uint4* dst = reinterpret_cast<uint4*>(hsw + (li & 1) * (C2BR * CW));
            dst[0] = make_uint4(lop3<0x96>(l0, m.x, r0), lop3<0xe8>(l0, m.x, r0), lop3<0x96>(l1, m.y, r1),
                                lop3<0xe8>(l1, m.y, r1));
            dst[1] = make_uint4(lop3<0x96>(l2, m.z, r2), lop3<0xe8>(l2, m.z, r2), lop3<0x96>(l3, m.w, r3),
                                lop3<0xe8>(l3, m.w, r3));
        };
        auto layer = [&](const uint32_t* buf, int li, int n, int zi, const uint32_t (&m0)[3], const uint32_t (&m1)[3],
                         bool first) {
            __syncwarp();  // h-sums of layer li visible; layer li - 1's reads done
            const uint2* hs = hsb + (li & 1) * (C2BR * CW) + oc * CW + ow;
            const uint2 h0 = hs[0], h1 = hs[CW], h2 = hs[2 * CW], h3 = hs[3 * CW], h4 = hs[4 * CW];
            const uint32_t* ce = buf + li * (C2LAYER / 4) + (oc + 1) * CBW + 4 + ow;
            const uint32_t an0 = ce[0], an1 = ce[CBW], an2 = ce[2 * CBW];
            if (li + 1 < n) hsum(buf + (li + 1) * (C2LAYER / 4), li + 1);
            V3 vc[3];
            vc[0] = vsum3(h0.x, h0.y, h1.x, h1.y, h2.x, h2.y);
            vc[1] = vsum3(h1.x, h1.y, h2.x, h2.y, h3.x, h3.y);
            vc[2] = vsum3(h2.x, h2.y, h3.x, h3.y, h4.x, h4.y);
            if (li >= 2 || !first) {
                const unsigned dz = unsigned(zi - 1 - it.z0);  // output layer zi - 1 past z0 (wraps below it)
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    const uint32_t tmk = li < 2 ? mprev[k] : (RHO == 4 && li >= 6 ? m1[k] : m0[k]);
                    const uint32_t o = life_v3(va[k], vb[k], vc[k], alive[k], tmk);
                    if (dz < zn[k]) *optr[k] = o;
                }
            }
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                optr[k] += zstride;
                va[k] = vb[k];
                vb[k] = vc[k];
            }
            alive[0] = an0;
            alive[1] = an1;
            alive[2] = an2;
        };

        const int t0 = wo * TPW;
        for (int st = 0; st < nst; ++st) {
            const uint32_t b = seq & 1;
            if (lane == 0) {
                fence_proxy_async();
                if (st + 1 < nst) cols_issue12(tm, it, st + 1, wbase + (b ^ 1) * C2STAGE, mbar0 + 8 * (b ^ 1));
                else if (nxt < nitems) cols_issue12(tm, itn, 0, wbase + (b ^ 1) * C2STAGE, mbar0 + 8 * (b ^ 1));
            }
            uint32_t m0[3], m1[3];
            {
                const uint32_t ma = tile_mask1<RHO>(bwa0, t0), mb = tile_mask1<RHO>(bwb0, t0);
                m0[0] = ma & xm[0];
                m0[1] = (sel1 ? mb : ma) & xm[1];
                m0[2] = mb & xm[2];
                if (RHO == 4) {
                    const uint32_t na = tile_mask1<RHO>(bwa1, t0), nb = tile_mask1<RHO>(bwb1, t0);
                    m1[0] = na & xm[0];
                    m1[1] = (sel1 ? nb : na) & xm[1];
                    m1[2] = nb & xm[2];
                } else {
                    m1[0] = m0[0], m1[1] = m0[1], m1[2] = m0[2];
                }
            }
            if (st + 1 < nst) {
                load_bw(it, it.z0 + CLZ * (st + 1));
            } else {
                nxt = __shfl_sync(0xffffffffu, nxt, 0);
                itn.iy = __shfl_sync(0xffffffffu, itn.iy, 0);
                itn.g = __shfl_sync(0xffffffffu, itn.g, 0);
                itn.z0 = __shfl_sync(0xffffffffu, itn.z0, 0);
                itn.z1 = __shfl_sync(0xffffffffu, itn.z1, 0);
                if (nxt < nitems) load_bw(itn, itn.z0);
            }
            while (!mbar_try_wait(mbar0 + 8 * b, (seq >> 1) & 1u)) {
            }
            const uint32_t* buf = reinterpret_cast<const uint32_t*>(wbase + b * C2STAGE);
            const int zbase = it.z0 - 1 + CLZ * st;
            __syncwarp();
            hsum(buf, 0);
            const bool first = st == 0;
            if (st < nfull) {
                // the warm-up layers' branch on `first` stays inside layers
                // 0 and 1 (not a second copy of the whole stage)
                layer(buf, 0, CLZ, zbase, m0, m1, first);
                layer(buf, 1, CLZ, zbase + 1, m0, m1, first);
#pragma unroll
                for (int li = 2; li < CLZ; ++li) layer(buf, li, CLZ, zbase + li, m0, m1, false);
            } else if (tail == 2) {
                layer(buf, 0, 2, zbase, m0, m1, first);
                layer(buf, 1, 2, zbase + 1, m0, m1, first);
            } else {
#pragma unroll 1
                for (int li = 0; li < tail; ++li) layer(buf, li, tail, zbase + li, m0, m1, first);
            }
#pragma unroll
            for (int k = 0; k < 3; ++k) mprev[k] = RHO == 4 ? m1[k] : m0[k];
            ++seq;
        }
        cur = nxt;
        it = itn;
    }
}

// The chunk engine's canonical plan: from the tile bitmap the map marked
// (k_cols_mark), every tile row (ty, tz) of the domain is cut into chunks of
// at most LMAX x-adjacent marked tiles — the same chunk list for every exact
// map, so H and BB run identical steps and differ only in the mapping work.
// Three passes keep the list in domain order (tz, ty, tx), so the chunks the
// persistent kernel runs concurrently are spatial neighbours: per tile row the
// chunk count, one exclusive scan (a single CTA), then the chunks at their offsets.
template <int RHO, bool WRITE>
__device__ __forceinline__ unsigned row_chunks(const uint32_t* __restrict__ row, int ty, int tz, Chunk* out) {
    constexpr int LMAX = PlanCfg<RHO>::LMAX;
    unsigned n = 0;
    int start = -1;  // first tile of the current run of marked tiles
    for (int tx = 0; tx <= ty + 1; ++tx) {  // tiles x <= y hold cells; tx = ty + 1 closes the run
        const bool on = tx <= ty && ((row[tx >> 5] >> (tx & 31)) & 1u);
        if (on && start < 0) start = tx;
        if ((!on || tx - start == LMAX) && start >= 0) {
            if (WRITE) out[n] = Chunk{start * RHO, ty * RHO, tz * RHO, (tx - start) * RHO};
            ++n;
            start = on ? tx : -1;
        }
    }
    return n;
}

template <int RHO, bool WRITE>
__global__ void __launch_bounds__(256) k_chunk_rows(const uint32_t* __restrict__ bm, int D, int TW,
                                                    unsigned* __restrict__ cnt, Chunk* __restrict__ out) {
    const long long nrows = (long long)D * D;
    for (long long rr = blockIdx.x * (long long)blockDim.x + threadIdx.x; rr < nrows;
         rr += (long long)gridDim.x * blockDim.x) {
        const int tz = int(rr / D), ty = int(rr % D);
        const bool cells = ty + tz <= D - 1;  // the tile row holds cells
        if (!WRITE) cnt[rr] = cells ? row_chunks<RHO, false>(bm + rr * TW, ty, tz, nullptr) : 0u;
        else if (cells) row_chunks<RHO, true>(bm + rr * TW, ty, tz, out + cnt[rr]);
    }
}

// in-place exclusive scan of n counts by one CTA of 1024 threads; *total = the sum
__global__ void __launch_bounds__(1024) k_scan_counts(unsigned* __restrict__ c, long long n, unsigned* __restrict__ total) {
    __shared__ unsigned s_part[1024];
    const int t = threadIdx.x;
    const long long per = (n + 1023) / 1024, lo = t * per, hi = min(n, lo + per);
    unsigned sum = 0;
    for (long long i = lo; i < hi; ++i) sum += c[i];
    s_part[t] = sum;
    __syncthreads();
    for (int d = 1; d < 1024; d <<= 1) {  // inclusive Hillis-Steele over the partials
        const unsigned v = t >= d ? s_part[t - d] : 0u;
        __syncthreads();
        s_part[t] += v;
        __syncthreads();
    }
    unsigned run = t ? s_part[t - 1] : 0u;
    for (long long i = lo; i < hi; ++i) {
        const unsigned v = c[i];
        c[i] = run;
        run += v;
    }
    if (t == 1023) *total = s_part[1023];
}

template <int RHO>
__global__ void __launch_bounds__(CNW * 32) k_cols_run(const __grid_constant__ CUtensorMap tmA,
                                                       const __grid_constant__ CUtensorMap tmB, uint32_t* bitsA,
                                                       uint32_t* bitsB, const ColItem* __restrict__ items,
                                                       int nitems, unsigned* ctl, const uint32_t* __restrict__ bm,
                                                       int D, int TW, int steps, int S, int WP) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint8_t* wbase = smem + warp * CWARP;
    const uint32_t mbar0 = smem_u32(smem + CNW * CWARP + 16 * warp);
    if (lane == 0) {
        mbar_init(mbar0, 1);
        mbar_init(mbar0 + 8, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    }
    uint32_t seq = 0;
    // ctl: [0] the grid barrier, [1 + s] step s's item counter (zeroed by the host)
    for (int st = 0; st < steps; ++st) {
        const bool even = (st & 1) == 0;
        cols_step<RHO>(items, nitems, ctl + 1 + st, even ? &tmA : &tmB, even ? bitsB : bitsA, bm, D, TW, S, WP, wbase,
                       mbar0, seq);
        if (st + 1 < steps) step_barrier(ctl);
    }
}

template <int RHO>
__global__ void __launch_bounds__(C2NW * 32) k_cols_run12(const __grid_constant__ CUtensorMap tmA,
                                                          const __grid_constant__ CUtensorMap tmB, uint32_t* bitsA,
                                                          uint32_t* bitsB, const ColItem* __restrict__ items,
                                                          int nitems, unsigned* ctl, const uint32_t* __restrict__ bm,
                                                          int D, int TW, int steps, int S, int WP) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint8_t* wbase = smem + warp * C2WARP;
    const uint32_t mbar0 = smem_u32(smem + C2NW * C2WARP + 16 * warp);
    if (lane == 0) {
        mbar_init(mbar0, 1);
        mbar_init(mbar0 + 8, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    }
    uint32_t seq = 0;
    for (int st = 0; st < steps; ++st) {
        const bool even = (st & 1) == 0;
        cols_step12<RHO>(items, nitems, ctl + 1 + st, even ? &tmA : &tmB, even ? bitsB : bitsA, bm, D, TW, S, WP,
                         wbase, mbar0, seq);
        if (st + 1 < steps) step_barrier(ctl);
    }
}

template <int KIND>
void launch_kind(const Geom& g, int wz0, int wz1, const CUtensorMap& tmap, uint32_t* nbits, int WP, cudaStream_t s) {
    if (g.rho == 4) launch_t<KIND, 4>(g, wz0, wz1, tmap, nbits, WP, s);
    else launch_t<KIND, 8>(g, wz0, wz1, tmap, nbits, WP, s);
}

}  // namespace

// Halo exchange in bits (the sharded engine): tile (X, Y, Z) of side rho is
// rho^2 rows of rho bits at bit offset (rho X) % 32 of word (rho X) / 32 of
// pitched row (z, y). Packed: per tile, rows in lz, ly order, rho bits each
// (rho = 8: one byte per row, 64 bytes per tile; rho = 4: a nibble per row,
// 8 bytes per tile). Unpack writes whole bytes for rho = 8 and nibbles through
// 32-bit atomics for rho = 4 (two tiles share a byte), so tiles unpacked
// concurrently never clobber each other. Rows outside the square shadow are skipped.
template <int RHO>
__device__ __forceinline__ uint32_t tile_row_bits(const uint32_t* __restrict__ bits, int S, int WP, int X, int Y,
                                                  int Z, int r) {
    const int z = Z * RHO + r / RHO, y = Y * RHO + r % RHO;
    if (z >= S || y >= S) return 0u;
    return (bits[((long long)z * S + y) * WP + ((RHO * X) >> 5)] >> ((RHO * X) & 31)) & ((1u << RHO) - 1u);
}

template <int RHO>
__global__ void k_bits_tiles_pack(const uint32_t* __restrict__ bits, int S, int WP, const int* __restrict__ tiles,
                                  uint8_t* __restrict__ out) {
    const int k = blockIdx.x;
    const int X = tiles[3 * k], Y = tiles[3 * k + 1], Z = tiles[3 * k + 2];
    if (RHO == 8) {
        for (int r = threadIdx.x; r < 64; r += blockDim.x)
            out[(long long)k * 64 + r] = (uint8_t)tile_row_bits<RHO>(bits, S, WP, X, Y, Z, r);
    } else {  // two rows per byte: low nibble = even row
        for (int t = threadIdx.x; t < 8; t += blockDim.x)
            out[(long long)k * 8 + t] = (uint8_t)(tile_row_bits<RHO>(bits, S, WP, X, Y, Z, 2 * t) |
                                                  (tile_row_bits<RHO>(bits, S, WP, X, Y, Z, 2 * t + 1) << 4));
    }
}

template <int RHO>
__global__ void k_bits_tiles_unpack(uint32_t* __restrict__ bits, int S, int WP, const int* __restrict__ tiles,
                                    const uint8_t* __restrict__ in) {
    const int k = blockIdx.x;
    const int X = tiles[3 * k], Y = tiles[3 * k + 1], Z = tiles[3 * k + 2];
    const int bit = (RHO * X) & 31, word = (RHO * X) >> 5;
    for (int r = threadIdx.x; r < RHO * RHO; r += blockDim.x) {
        const int z = Z * RHO + r / RHO, y = Y * RHO + r % RHO;
        if (z >= S || y >= S) continue;
        uint32_t* w = bits + ((long long)z * S + y) * WP + word;
        if (RHO == 8) {
            reinterpret_cast<uint8_t*>(w)[bit >> 3] = in[(long long)k * 64 + r];
        } else {
            const uint32_t v = (in[(long long)k * 8 + r / 2] >> (4 * (r & 1))) & 0xfu;
            atomicAnd(w, ~(0xfu << bit));
            atomicOr(w, v << bit);
        }
    }
}

bool ca_runs_supported(int rho) { return rho == 4 || rho == 8; }
bool cols_supported(int rho) { return rho == 4 || rho == 8 || rho == 16; }

unsigned long long bits_tile_bytes(int rho) { return rho == 8 ? 64ull : 8ull; }

void launch_bits_tiles_pack(const Geom& g, const uint32_t* bits, const int* tiles, unsigned long long ntiles,
                            uint8_t* out, cudaStream_t s) {
    if (ntiles == 0) return;
    const int WP = bits_pitch_words(g.side);
    if (g.rho == 8) k_bits_tiles_pack<8><<<(unsigned)ntiles, 64, 0, s>>>(bits, g.side, WP, tiles, out);
    else k_bits_tiles_pack<4><<<(unsigned)ntiles, 32, 0, s>>>(bits, g.side, WP, tiles, out);
}

void launch_bits_tiles_unpack(const Geom& g, uint32_t* bits, const int* tiles, unsigned long long ntiles,
                              const uint8_t* in, cudaStream_t s) {
    if (ntiles == 0) return;
    const int WP = bits_pitch_words(g.side);
    if (g.rho == 8) k_bits_tiles_unpack<8><<<(unsigned)ntiles, 64, 0, s>>>(bits, g.side, WP, tiles, in);
    else k_bits_tiles_unpack<4><<<(unsigned)ntiles, 32, 0, s>>>(bits, g.side, WP, tiles, in);
}

// words per pitched row: >= 8, multiple of 4 (16-byte row stride for TMA)
int bits_pitch_words(int side) {
    const int w = ((side + 31) / 32 + 3) & ~3;
    return w < 8 ? 8 : w;
}

// the shadow is a full S x S square of pitched rows per layer stack: row
// (y, z) at z * S + y, so a chunk's halo is ONE 3-D tensor box
unsigned long long bits_rows(int side) { return (unsigned long long)side * side; }
static int tri_rows(int side) { return int((long long)side * (side + 1) / 2); }
// rows per warp for pack/unpack: 32 on big states, fewer (>= 4) until the grid
// has ~32 warps per SM
static int rows_per_warp(int nrows) {
    int r = ROWS_PER_WARP;
    while (r > 4 && (nrows + r - 1) / r < 148 * 32) r /= 2;
    return r;
}

int tma_box_rows(int rho) { return rho + 2; }

int tma_box_words() { return BOXW; }

void launch_pack_bits(const Geom& g, const uint8_t* cur, uint32_t* bits, cudaStream_t s) {
    const int S = g.side, WP = bits_pitch_words(S);
    const int nrows = tri_rows(S);
    const int rpw = rows_per_warp(nrows);
    const int warps = (nrows + rpw - 1) / rpw;
    k_pack_bits<<<(warps + 7) / 8, 256, 0, s>>>(cur, bits, S, WP, nrows, g.prefix, tet_cells(S), rpw);
}

void launch_unpack_bits(const Geom& g, const uint32_t* bits, uint8_t* out, cudaStream_t s) {
    const int S = g.side, WP = bits_pitch_words(S);
    const int nrows = tri_rows(S);
    const int rpw = rows_per_warp(nrows);
    const int warps = (nrows + rpw - 1) / rpw;
    k_unpack_bits<<<(warps + 7) / 8, 256, 0, s>>>(bits, out, S, WP, nrows, g.prefix, rpw);
}

unsigned long long ca_plan_capacity(const Geom& g) { return (unsigned long long)g.ex * g.ey * g.ez; }

void launch_ca_plan_range(const Geom& g, int kind, int wz0, int wz1, void* chunks, unsigned* count, cudaStream_t s) {
    if (kind == SMX_H3D) {
        if (g.rho == 4) launch_plan_t<SMX_H3D, 4>(g, wz0, wz1, chunks, count, s);
        else launch_plan_t<SMX_H3D, 8>(g, wz0, wz1, chunks, count, s);
    } else {
        if (g.rho == 4) launch_plan_t<SMX_BB, 4>(g, wz0, wz1, chunks, count, s);
        else launch_plan_t<SMX_BB, 8>(g, wz0, wz1, chunks, count, s);
    }
}
void launch_ca_plan(const Geom& g, int kind, void* chunks, unsigned* count, cudaStream_t s) {
    launch_ca_plan_range(g, kind, 0, g.ez, chunks, count, s);
}

// one step over an explicit chunk list (a shard's boundary or interior part):
// the run kernel with steps = 1, launched as an ordinary grid
cudaError_t launch_ca_bits_list(const Geom& g, const void* tmIn, uint32_t* in, uint32_t* out, const void* chunks,
                                const unsigned* count, cudaStream_t s) {
    const CUtensorMap& t = *reinterpret_cast<const CUtensorMap*>(tmIn);
    if (g.rho == 4) {
        if (tet_cells(g.side) <= (32ull << 20)) return launch_run_t<4, 16, 1>(g, t, t, in, out, chunks, count, 1, s, false);
        return launch_run_t<4, 16, 2>(g, t, t, in, out, chunks, count, 1, s, false);
    }
    return launch_run_t<8, 16, 1>(g, t, t, in, out, chunks, count, 1, s, false);
}

cudaError_t launch_ca_bits_run(const Geom& g, const void* tmA, const void* tmB, uint32_t* A, uint32_t* B,
                               const void* chunks, const unsigned* count, int steps, cudaStream_t s) {
    const CUtensorMap& ta = *reinterpret_cast<const CUtensorMap*>(tmA);
    const CUtensorMap& tb = *reinterpret_cast<const CUtensorMap*>(tmB);
    if (g.rho == 4) {
        // few items per warp (latency-bound, C2: 4.38 -> 4.00 us per step):
        // one chunk per item, its z-march split over both half-warps; many
        // items (>= 177 M cells: 4-6 % faster): two chunks per item, fewer
        // idle h-sum lanes. 32 warps per SM measured no better than 16.
        if (tet_cells(g.side) <= (32ull << 20)) return launch_run_t<4, 16, 1>(g, ta, tb, A, B, chunks, count, steps, s);
        return launch_run_t<4, 16, 2>(g, ta, tb, A, B, chunks, count, steps, s);
    }
    return launch_run_t<8, 16, 1>(g, ta, tb, A, B, chunks, count, steps, s);
}

void launch_chunkify(int rho, const uint32_t* bm, int D, int TW, unsigned* rowcnt, void* chunks, unsigned* count,
                     cudaStream_t s) {
    const long long nrows = (long long)D * D;
    long long blocks = (nrows + 255) / 256;
    if (blocks > 148ll * 8) blocks = 148ll * 8;
    if (blocks < 1) blocks = 1;
    Chunk* out = reinterpret_cast<Chunk*>(chunks);
    if (rho == 8) k_chunk_rows<8, false><<<unsigned(blocks), 256, 0, s>>>(bm, D, TW, rowcnt, out);
    else k_chunk_rows<4, false><<<unsigned(blocks), 256, 0, s>>>(bm, D, TW, rowcnt, out);
    k_scan_counts<<<1, 1024, 0, s>>>(rowcnt, nrows, count);
    if (rho == 8) k_chunk_rows<8, true><<<unsigned(blocks), 256, 0, s>>>(bm, D, TW, rowcnt, out);
    else k_chunk_rows<4, true><<<unsigned(blocks), 256, 0, s>>>(bm, D, TW, rowcnt, out);
}

// ---- the column engine's launchers ----
// the item shapes: 8 or 12 output rows (the host picks per side)
int cols_box_words() { return CBW; }
int cols_box_rows(int rows) { return rows + 2; }
int cols_box_layers() { return CLZ; }
int cols_item_bytes() { return int(sizeof(ColItem)); }

void launch_cols_mark(const Geom& g, int kind, uint32_t* bm, int D, int TW, unsigned* stats, cudaStream_t s,
                      int wz0, int wz1) {
    if (wz1 < 0) wz1 = g.ez;
    if (wz1 <= wz0) return;
    const long long nb = (long long)g.ex * g.ey * (wz1 - wz0);
    long long blocks = (nb + 255) / 256;
    if (blocks > 148ll * 16) blocks = 148ll * 16;
    if (blocks < 1) blocks = 1;
    if (kind == SMX_H3D) k_cols_mark<SMX_H3D><<<unsigned(blocks), 256, 0, s>>>(g, bm, D, TW, stats, wz0, wz1);
    else k_cols_mark<SMX_BB><<<unsigned(blocks), 256, 0, s>>>(g, bm, D, TW, stats, wz0, wz1);
}

// persistent grid of each shape (co-resident CTAs x SMs), attributes set once per device
static int cols_grid(int rows) {
    static std::once_flag once[kMaxDevices];
    static int grids[kMaxDevices][2];
    const int dev = current_device();
    int local[2] = {0, 0};
    once_per_device(once, dev, [&] {
        const int smem8 = CNW * (CWARP + 16), smem12 = C2NW * (C2WARP + 16);
        cudaFuncSetAttribute(k_cols_run<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem8);
        cudaFuncSetAttribute(k_cols_run<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem8);
        cudaFuncSetAttribute(k_cols_run<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem8);
        cudaFuncSetAttribute(k_cols_run12<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem12);
        cudaFuncSetAttribute(k_cols_run12<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem12);
        cudaFuncSetAttribute(k_cols_run12<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem12);
        int per8 = 0, per12 = 0, nsm = 148;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per8, k_cols_run<8>, CNW * 32, smem8);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per12, k_cols_run12<8>, C2NW * 32, smem12);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        local[0] = (per8 > 0 ? per8 : 1) * nsm;
        local[1] = (per12 > 0 ? per12 : 1) * nsm;
        if (dev >= 0 && dev < kMaxDevices) grids[dev][0] = local[0], grids[dev][1] = local[1];
    });
    const int i = rows == C2R ? 1 : 0;
    return dev >= 0 && dev < kMaxDevices ? grids[dev][i] : local[i];
}
int cols_warps(int rows) { return cols_grid(rows) * (rows == C2R ? C2NW : CNW); }

cudaError_t launch_cols_run(const Geom& g, int rows, const void* tmA, const void* tmB, uint32_t* A, uint32_t* B,
                            const void* items, int nitems, unsigned* ctl, const uint32_t* bm, int D, int TW, int steps,
                            cudaStream_t s) {
    const int grid = cols_grid(rows);
    const bool r12 = rows == C2R;
    const int nthr = (r12 ? C2NW : CNW) * 32;
    const int smem = r12 ? C2NW * (C2WARP + 16) : CNW * (CWARP + 16);
    int S = g.side, WP = bits_pitch_words(g.side);
    const ColItem* it = reinterpret_cast<const ColItem*>(items);
    void* args[] = {const_cast<void*>(tmA), const_cast<void*>(tmB), &A, &B, &it, &nitems, &ctl,
                    const_cast<uint32_t**>(&bm), &D, &TW, &steps, &S, &WP};
    const void* fn = r12 ? (g.rho == 16  ? (const void*)k_cols_run12<16>
                            : g.rho == 8 ? (const void*)k_cols_run12<8>
                                         : (const void*)k_cols_run12<4>)
                         : (g.rho == 16  ? (const void*)k_cols_run<16>
                            : g.rho == 8 ? (const void*)k_cols_run<8>
                                         : (const void*)k_cols_run<4>);
    if (steps == 1) return cudaLaunchKernel(fn, dim3(grid), dim3(nthr), args, smem, s);
    return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(nthr), args, smem, s);
}

void launch_ca_bits(const Geom& g, int kind, int wz0, int wz1, const void* tmap_ptr, uint32_t* nbits, cudaStream_t s) {
    const CUtensorMap& tmap = *reinterpret_cast<const CUtensorMap*>(tmap_ptr);
    const int WP = bits_pitch_words(g.side);
    if (wz1 <= wz0) return;
    if (kind == SMX_H3D) launch_kind<SMX_H3D>(g, wz0, wz1, tmap, nbits, WP, s);
    else launch_kind<SMX_BB>(g, wz0, wz1, tmap, nbits, WP, s);
}

}  // namespace smx
