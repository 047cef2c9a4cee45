// Internal launcher declarations shared by the kernel files and the C ABI.
#pragma once

#include <cuda_runtime.h>

#include <mutex>

#include "smx_common.cuh"

namespace smx {

// Kernel attributes (cudaFuncSetAttribute) and occupancy-derived grid sizes
// belong to ONE device's context: they are set once per (kernel, device), so
// a process driving several GPUs (smx_ca over `ngpus`, or one host thread per
// device) configures each device before its first launch.
constexpr int kMaxDevices = 64;
inline int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
}
template <class Fn>
inline void once_per_device(std::once_flag (&flags)[kMaxDevices], int dev, Fn&& fn) {
    if (dev >= 0 && dev < kMaxDevices) std::call_once(flags[dev], fn);
    else fn();
}

void launch_outcomes(const Geom& g, smx_outcome* out, unsigned long long count, cudaStream_t s);
void launch_map_block(const Geom& g, uint32_t* cov, DevCounters* cnt, unsigned* sink, cudaStream_t s);
void launch_accum(const Geom& g, uint32_t* cells, int exec, cudaStream_t s);
int accum_strip_blocks(int rho);  // map blocks per CTA of the ACCUM x-run kernel
void launch_life_init(unsigned long long seed, uint8_t* cells, unsigned long long n, cudaStream_t s);
// kernel_accum: every cell += 1 (no map)
void launch_increment(uint32_t* cells, unsigned long long n, cudaStream_t s);
void launch_ca(const Geom& g, int wz0, int wz1, const uint8_t* cur, uint8_t* next, int exec, cudaStream_t s);
bool ca_runs_supported(int rho);  // the chunk engine, fused and range steps: rho in {4, 8}
bool cols_supported(int rho);     // the column engine: rho in {4, 8, 16}
// fused u8 -> u8 x-run step (smx_ca_fused.cu), rho in {4, 8}
void launch_ca_fused(const Geom& g, int wz0, int wz1, const uint8_t* cur, uint8_t* next, cudaStream_t s);
// bit-shadow engine (smx_ca_bits.cu)
int bits_pitch_words(int side);
unsigned long long bits_rows(int side);
int tma_box_rows(int rho);
int tma_box_words();
void launch_pack_bits(const Geom& g, const uint8_t* cur, uint32_t* bits, cudaStream_t s);
void launch_unpack_bits(const Geom& g, const uint32_t* bits, uint8_t* out, cudaStream_t s);
// tmap: CUtensorMap over the input bit shadow; writes the next bit shadow
void launch_ca_bits(const Geom& g, int kind, int wz0, int wz1, const void* tmap, uint32_t* nbits, cudaStream_t s);
// multi-step engine: the map applied once (chunk list, 16 B per chunk, at most
// ca_plan_capacity entries; *count must be zero), then ONE persistent
// cooperative launch runs `steps` bit-sliced steps A -> B -> A ...
unsigned long long ca_plan_capacity(const Geom& g);
void launch_ca_plan(const Geom& g, int kind, void* chunks, unsigned* count, cudaStream_t s);
void launch_ca_plan_range(const Geom& g, int kind, int wz0, int wz1, void* chunks, unsigned* count, cudaStream_t s);
// one step A -> B over an explicit chunk list (ordinary launch, no grid barrier)
cudaError_t launch_ca_bits_list(const Geom& g, const void* tmIn, uint32_t* in, uint32_t* out, const void* chunks,
                                const unsigned* count, cudaStream_t s);
cudaError_t launch_ca_bits_run(const Geom& g, const void* tmA, const void* tmB, uint32_t* A, uint32_t* B,
                               const void* chunks, const unsigned* count, int steps, cudaStream_t s);
// the column engine (large states): tile bitmap marked by the map, then a
// persistent run over column items (int4 {iy, g, z0, z1}); ctl: [0] grid
// barrier, [1 + s] step s's item counter, zeroed
int cols_box_words();
int cols_box_rows(int rows);  // rows: output rows per column item (8 or 12)
int cols_box_layers();
int cols_item_bytes();
int cols_warps(int rows);
// the map over blocks with wz in [wz0, wz1) (default: the whole grid) -> tile bitmap
void launch_cols_mark(const Geom& g, int kind, uint32_t* bm, int D, int TW, unsigned* stats, cudaStream_t s,
                      int wz0 = 0, int wz1 = -1);
// the chunk engine's canonical plan from the tile bitmap (rho in {4, 8})
// rowcnt: D * D u32 scratch; *count receives the chunk total
void launch_chunkify(int rho, const uint32_t* bm, int D, int TW, unsigned* rowcnt, void* chunks, unsigned* count,
                     cudaStream_t s);
cudaError_t launch_cols_run(const Geom& g, int rows, const void* tmA, const void* tmB, uint32_t* A, uint32_t* B,
                            const void* items, int nitems, unsigned* ctl, const uint32_t* bm, int D, int TW, int steps,
                            cudaStream_t s);
// 2-simplex EDM (f64 points as x, y pairs) and periodic 2-D Life (smx_kernels2d.cu)
void launch_edm(const Geom& g, const double* pts, double* cells, int exec, cudaStream_t s);
// periodic 2-D Life: `bits` = the packed state's bit triangle (launch_pack2d;
// the x-run scheme reads neighbourhoods from it, the block scheme ignores it)
void launch_ca2d(const Geom& g, const uint8_t* cur, const uint32_t* bits, uint8_t* next, int exec, cudaStream_t s);
uint64_t ca2d_bit_words(uint64_t ncells);  // words of the bit triangle incl. the zero tail
void launch_pack2d(const uint8_t* cur, uint64_t ncells, uint32_t* bits, cudaStream_t s);
// first packed index with coverage != 1 (atomicMin into *first, preset to n)
void launch_first_defect(const uint32_t* cov, unsigned long long n, unsigned long long* first, cudaStream_t s);
// bit-shadow tiles for the sharded engine's halo (rho in {4, 8})
unsigned long long bits_tile_bytes(int rho);
void launch_bits_tiles_pack(const Geom& g, const uint32_t* bits, const int* tiles, unsigned long long ntiles,
                            uint8_t* out, cudaStream_t s);
void launch_bits_tiles_unpack(const Geom& g, uint32_t* bits, const int* tiles, unsigned long long ntiles,
                              const uint8_t* in, cudaStream_t s);
void launch_tiles_pack(const Geom& g, const uint8_t* cells, const int* tiles, unsigned long long ntiles,
                       uint8_t* out, cudaStream_t s);
void launch_tiles_unpack(const Geom& g, uint8_t* cells, const int* tiles, unsigned long long ntiles,
                         const uint8_t* in, cudaStream_t s);

}  // namespace smx
