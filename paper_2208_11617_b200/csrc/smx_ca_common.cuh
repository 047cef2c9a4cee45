// Device helpers shared by the two x-run 3-D Life engines (smx_ca_bits.cu: the
// bit-shadow engine; smx_ca_fused.cu: the fused u8 -> u8 step).
//
//  * bit-slice arithmetic: 32 cells per 32-bit word, 26-neighbour sums as
//    bit-planes, the B3/S23 rule of life_next (simulator.hpp:220-223);
//  * byte <-> bit conversion (u8 cells are 0/1, make_life_state :390-398);
//  * the map-driven work assignment: a CTA maps a P x P (x NZ) patch of blocks
//    (map_block = map -> Void -> strict y-1, simulator.hpp:190-202) and chains
//    x-adjacent tiles into chunks (build_chunks below).
#pragma once

#include "smx_common.cuh"

namespace smx {
namespace ca {

struct Chunk {
    int x0, y0, z0, w;  // cell box origin and owned width (cells)
};

// ---- bit <-> byte ----

// 32 bytes (each 0 or 1) -> 32 bits, bit i = byte i. t = w0 | w1 << 4 puts
// bytes i and i+4 into one byte; * 0x01020408 gathers bit 0 of byte i to bit
// 24+i and bit 4 to bit 28+i with no carries (all partial products below bit 24
// land on distinct bits).
__device__ __forceinline__ uint32_t pack32(uint4 a, uint4 b) {
    const uint32_t M = 0x01020408u;
    const uint32_t p0 = (a.y * 16u + a.x) * M;
    const uint32_t p1 = (a.w * 16u + a.z) * M;
    const uint32_t p2 = (b.y * 16u + b.x) * M;
    const uint32_t p3 = (b.w * 16u + b.z) * M;
    return __byte_perm(__byte_perm(p0, p1, 0x0073), __byte_perm(p2, p3, 0x0073), 0x5410);
}

// 4 bits -> 4 bytes (0/1): n * (1 + 2^7 + 2^14 + 2^21) puts bit i at 9i.
__device__ __forceinline__ uint32_t spread4(uint32_t nib) { return (nib * 0x00204081u) & 0x01010101u; }
__device__ __forceinline__ uint4 spread16(uint32_t b) {
    return make_uint4(spread4(b & 0xf), spread4((b >> 4) & 0xf), spread4((b >> 8) & 0xf), spread4((b >> 12) & 0xf));
}

// bits [lo, hi] (inclusive) of a 32-bit word; 0 when hi < lo
__device__ __forceinline__ uint32_t range_mask(int lo, int hi) {
    lo = lo < 0 ? 0 : lo;
    hi = hi > 31 ? 31 : hi;
    if (hi < lo) return 0u;
    return (0xffffffffu >> (31 - hi)) & (0xffffffffu << lo);
}

// ---- bit-sliced Life ----

struct Planes4 {
    uint32_t b0, b1, b2, b3;
};

// sum of three 2-bit numbers (<= 9) as 4 bit-planes
__device__ __forceinline__ Planes4 add3x2(uint32_t a0, uint32_t a1, uint32_t b0, uint32_t b1, uint32_t c0,
                                          uint32_t c1) {
    const uint32_t s0 = a0 ^ b0 ^ c0;
    const uint32_t k1 = (a0 & b0) | (a0 & c0) | (b0 & c0);
    const uint32_t t = a1 ^ b1 ^ c1;
    const uint32_t u = (a1 & b1) | (a1 & c1) | (b1 & c1);
    const uint32_t c = t & k1;
    return Planes4{s0, t ^ k1, u ^ c, u & c};
}

// B3/S23 from three 4-plane partial sums (the 27-sum includes the cell):
// next = (S == 3) | (alive & S == 4).
__device__ __forceinline__ uint32_t life_planes(const Planes4& a, const Planes4& b, const Planes4& c,
                                                uint32_t alive) {
    const uint32_t s0 = a.b0 ^ b.b0 ^ c.b0, k1 = (a.b0 & b.b0) | (a.b0 & c.b0) | (b.b0 & c.b0);
    const uint32_t s1 = a.b1 ^ b.b1 ^ c.b1, k2 = (a.b1 & b.b1) | (a.b1 & c.b1) | (b.b1 & c.b1);
    const uint32_t s2 = a.b2 ^ b.b2 ^ c.b2, k3 = (a.b2 & b.b2) | (a.b2 & c.b2) | (b.b2 & c.b2);
    const uint32_t s3 = a.b3 ^ b.b3 ^ c.b3, k4 = (a.b3 & b.b3) | (a.b3 & c.b3) | (b.b3 & c.b3);
    const uint32_t r1 = s1 ^ k1, c2 = s1 & k1;
    const uint32_t r2 = s2 ^ k2 ^ c2, c3 = (s2 & k2) | (s2 & c2) | (k2 & c2);
    const uint32_t r3 = s3 ^ k3 ^ c3, c4 = (s3 & k3) | (s3 & c3) | (k3 & c3);
    const uint32_t r4 = k4 ^ c4;
    const uint32_t eq3 = s0 & r1 & ~r2;
    const uint32_t eq4 = ~s0 & ~r1 & r2;
    return (eq3 | (eq4 & alive)) & ~(r3 | r4);
}

// ---- the engines' rule as an explicit LOP3 network ----
//
// One LOP3 (any 3-input boolean function) per line; the immediates are the
// function applied to (0xF0, 0xCC, 0xAA). ptxas keeps asm lop3 as written, so
// the ALU-pipe count per output word is the count below: 6 for the vertical
// sum (once per layer, used by three output layers) + 14 for the rule incl.
// the output mask, against 10 + 17 for the add3x2 / four-plane form.
template <unsigned LUT>
__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "r"(b), "r"(c), "n"(LUT));
    return d;
}

// A 9-cell (3 rows x 3 columns) sum v <= 9 as three bit-planes, SATURATED:
// exact for v <= 7, and 6 or 7 for v = 8, 9. The rule only asks whether the
// 27-sum is 3 or 4, which a term >= 5 already rules out, so three planes carry
// everything it needs.
struct V3 {
    uint32_t b0, b1, b2;
};
// p, q, u: three horizontal 3-sums (bit-planes x0, x1 of values <= 3)
__device__ __forceinline__ V3 vsum3(uint32_t p0, uint32_t p1, uint32_t q0, uint32_t q1, uint32_t u0, uint32_t u1) {
    const uint32_t s0 = lop3<0x96>(p0, q0, u0);  // weight 1
    const uint32_t k1 = lop3<0xe8>(p0, q0, u0);  // carry, weight 2
    const uint32_t t = lop3<0x96>(p1, q1, u1);   // weight 2
    const uint32_t m = lop3<0xe8>(p1, q1, u1);   // weight 4
    // v = s0 + 2 (t + k1) + 4 m: b1 = t ^ k1, b2 = m ^ (t & k1); when v >= 8
    // (m & t & k1) both are forced to 1 instead
    return V3{s0, lop3<0xbc>(t, k1, m), lop3<0xf8>(m, t, k1)};
}
// next = (S == 3) | (alive & S == 4) for S = a + b + c (the 27-sum including
// the cell), masked: with s0, k1 / s1, k2 the carry-save sums of planes 0 / 1,
// S = s0 + 2 (s1 + k1) + 4 (k2 + a2 + b2 + c2). S == 3 needs s0 = 1, exactly
// one of s1, k1 and no weight-4 term; S == 4 needs s0 = 0 and either s1 = k1 = 1
// and no weight-4 term, or s1 = k1 = 0 and exactly one.
__device__ __forceinline__ uint32_t life_v3(const V3& a, const V3& b, const V3& c, uint32_t alive, uint32_t mask) {
    const uint32_t s0 = lop3<0x96>(a.b0, b.b0, c.b0), k1 = lop3<0xe8>(a.b0, b.b0, c.b0);
    const uint32_t s1 = lop3<0x96>(a.b1, b.b1, c.b1), k2 = lop3<0xe8>(a.b1, b.b1, c.b1);
    const uint32_t o2 = lop3<0xfe>(a.b2, b.b2, c.b2);  // any of a2, b2, c2
    const uint32_t e2 = lop3<0x16>(a.b2, b.b2, c.b2);  // exactly one
    const uint32_t w0 = lop3<0x03>(o2, k2, 0u);        // no weight-4 term
    const uint32_t w1 = lop3<0x3a>(k2, o2, e2);        // exactly one weight-4 term
    const uint32_t g = lop3<0x68>(s0, s1, k1);         // s0 ? s1 ^ k1 : s1 & k1
    const uint32_t sl = lop3<0xfc>(s0, alive, 0u);     // s0 | alive
    const uint32_t t3 = lop3<0x80>(g, w0, sl);         // S == 3, or alive & S == 4 (s1 = k1 = 1)
    const uint32_t z = lop3<0x01>(s0, s1, k1);         // s0 = s1 = k1 = 0
    const uint32_t t4 = lop3<0x80>(z, w1, alive);      // alive & S == 4 (s1 = k1 = 0)
    return lop3<0xa8>(t3, t4, mask);
}

// ---- map-driven chunking ----

// Phases 1-2 of both engines; every thread of the CTA must call it. The CTA
// owns the P x P patch (blockIdx.x, blockIdx.y) of map blocks at the NZ layers
// wzb .. wzb+NZ-1 (< wz1). Its threads map the blocks lane-parallel, then chain
// tiles that are x-adjacent in the data: a tile's predecessor is at patch
// neighbour (wx-1, wy) (unfolded H tiles, the wall plane, BB rows) or
// (wx, wy-1) (the hinge fold, maps.hpp:334-336); its successor is at
// (wx+1, wy) or (wx, wy+1). The map is an exact cover, so a data tile has at
// most one predecessor and one successor: chains are disjoint paths. Every
// tile finds its distance to its chain's head and tail by pointer jumping
// (log2 of the chain length rounds, all tiles in parallel; s_link holds a
// (pointer, distance) pair per tile and direction in one 32-bit word, ping-
// ponged between two halves so every round reads only the previous round's
// pairs), and the tiles at head distance 0, LMAX, 2 LMAX, ... emit the chunks
// of at most LMAX tiles. Every useful tile lands in exactly one chunk.
// s_link: 4 * P * P * NZ words.
// Returns the chunk count (after a __syncthreads).
constexpr uint32_t LINK_END = 0xffffu;

template <int KIND>
__device__ __forceinline__ int build_chunks(const Geom& g, int wzb, int wz1, int P, int NZ, int lmax, int4* s_tile,
                                            Chunk* s_chunk, int* s_nchunks, uint32_t* s_link) {
    const int PP = P * P, NBP = PP * NZ;
    const int rho = g.rho;
    const int tid = threadIdx.x, nthr = blockDim.x;
    if (tid == 0) *s_nchunks = 0;
    for (int t = tid; t < NBP; t += nthr) {
        const int tl = t % PP, wz = wzb + t / PP;
        const int wx = blockIdx.x * P + (tl % P), wy = blockIdx.y * P + (tl / P);
        int4 v = make_int4(0, 0, 0, 0);
        if (wx < g.ex && wy < g.ey && wz < wz1) {
            const outcome<int> o = map_block<KIND>(g, wx, wy, wz);
            if (!o.is_void) v = make_int4(o.x, o.y, o.z, 1 | ((tl % P) << 8) | ((tl / P) << 16));
        }
        s_tile[t] = v;
    }
    __syncthreads();
    // links: (neighbour, 1) or (END, 0) toward the head (word t) and the tail (word NBP + t)
    for (int t = tid; t < NBP; t += nthr) {
        const int4 me = s_tile[t];
        uint32_t pl = LINK_END, sl = LINK_END;
        if (me.w) {
            const int px = (me.w >> 8) & 0xff, py = me.w >> 16;
            auto is_tile = [&](int i, int x) {
                const int4 o = s_tile[i];
                return o.w && o.x == x && o.y == me.y && o.z == me.z;
            };
            if (px > 0 && is_tile(t - 1, me.x - 1)) pl = uint32_t(t - 1) | (1u << 16);
            else if (py > 0 && is_tile(t - P, me.x - 1)) pl = uint32_t(t - P) | (1u << 16);
            if (px + 1 < P && is_tile(t + 1, me.x + 1)) sl = uint32_t(t + 1) | (1u << 16);
            else if (py + 1 < P && is_tile(t + P, me.x + 1)) sl = uint32_t(t + P) | (1u << 16);
        }
        s_link[t] = pl;
        s_link[NBP + t] = sl;
    }
    __syncthreads();
    uint32_t* cur = s_link;
    uint32_t* nxt = s_link + 2 * NBP;
    for (;;) {
        int more = 0;
        for (int k = tid; k < 2 * NBP; k += nthr) {
            const uint32_t v = cur[k];
            const uint32_t q = v & 0xffffu;
            uint32_t nv = v;
            if (q != LINK_END) {
                const uint32_t w = cur[(k < NBP ? 0 : NBP) + int(q)];
                nv = (w & 0xffffu) | ((v & 0xffff0000u) + (w & 0xffff0000u));
                more |= (nv & 0xffffu) != LINK_END;
            }
            nxt[k] = nv;
        }
        uint32_t* t = cur;
        cur = nxt;
        nxt = t;
        if (!__syncthreads_or(more)) break;
    }
    for (int t = tid; t < NBP; t += nthr) {
        const int4 me = s_tile[t];
        if (!me.w) continue;
        const int dh = int(cur[t] >> 16), dt = int(cur[NBP + t] >> 16);
        if (dh % lmax == 0) {
            const int c = atomicAdd(s_nchunks, 1);
            s_chunk[c] = Chunk{me.x * rho, me.y * rho, me.z * rho, min(lmax, dt + 1) * rho};
        }
    }
    __syncthreads();
    return *s_nchunks;
}

}  // namespace ca
}  // namespace smx
