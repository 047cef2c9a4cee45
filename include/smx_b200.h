/*
 * smx_b200.h — the C ABI of the B200-native H-map hot path.
 *
 * Plain C: no torch, no C++ types. Every entry point replaces one function of
 * the reference's header-only C++ API (arXiv 2208.11617 reference `simplexmap`,
 * /root/reference/proj/include/simplexmap/); the citation on each declaration
 * names the reference interface (file:line) it stands in for. The C++ drop-in
 * (include/simplexmap_b200.hpp) and the Python mirror
 * (paper_2208_11617_b200/api.py) both call exactly these symbols.
 *
 * Conventions
 *  - Return value: SMX_OK (0) or an error code; smx_last_error() returns the
 *    thread-local message (the reference's exception text where one exists).
 *    SMX_EINVAL <-> std::invalid_argument, SMX_ERANGE <-> std::overflow_error.
 *  - `device_ptr` != 0: the buffer arguments are device pointers (cudaMalloc /
 *    torch CUDA tensors) and the call only enqueues work on `stream`.
 *    `device_ptr` == 0: host buffers; the call stages them through a cached
 *    device pool, runs, copies results back and synchronises `stream`
 *    (the reference's mutate-in-place semantics, simulator.hpp:313-326,431-463).
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).
 *  - Threads: the library's scratch (staging pool, bit shadows, CA chunk list,
 *    the side stream the CA plan runs on) is per (device, host thread) — freed
 *    by smx_release() or when the thread exits — so
 *    calls on distinct states from distinct threads may run concurrently, as
 *    the reference's launches may. Device-resident calls from ONE thread share
 *    that thread's scratch: issue them on one stream (or synchronise between
 *    streams); host-buffer calls synchronise before returning.
 *  - Cell state is the reference's packed layout: 2-D row-major triangle
 *    index y(y+1)/2 + x (core.hpp:136-138); 3-D layer prefix tet(S)-tet(S-z)
 *    plus the triangle index (core.hpp:140-149). u32 cells for ACCUM, u8 for CA.
 */
#ifndef SMX_B200_H
#define SMX_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SMX_OK 0
#define SMX_EINVAL 1 /* std::invalid_argument */
#define SMX_ERANGE 2 /* std::overflow_error   */
#define SMX_ECUDA 3  /* CUDA runtime error (message carries cudaGetErrorString) */
#define SMX_ENOMEM 4

/* map_kind (maps.hpp:19); only BB, H2D and H3D are on this hot path. */
#define SMX_BB 0
#define SMX_RB 1
#define SMX_LAMBDA 2
#define SMX_H2D 3
#define SMX_TRAP 4
#define SMX_PADDED 5
#define SMX_H3D 6

/* Execution schemes for the workload kernels.
 * SMX_EXEC_BLOCK: one CUDA thread-block per map block, rho^m threads — the
 *                 paper's launch model (the reference's detail::sweep one to one).
 * SMX_EXEC_RUNS:  one CUDA thread-block per strip/patch of map blocks; the
 *                 blocks are mapped lane-parallel, their tiles merged into
 *                 contiguous x-runs and streamed with 128-bit accesses. For the
 *                 CA this is ONE fused u8 -> u8 kernel per step.
 * SMX_EXEC_BITS:  CA only — the bit-shadow engine: the u8 state is packed to
 *                 one bit per cell once, every step runs bits -> bits through
 *                 the map, and the u8 state is unpacked once after the last
 *                 step (smx_ca); smx_ca_step is pack -> step -> unpack. */
#define SMX_EXEC_AUTO (-1) /* CA: BITS (one small step: RUNS) where rho is 4 or 8, else BLOCK; ACCUM: RUNS */
#define SMX_EXEC_BLOCK 0
#define SMX_EXEC_RUNS 1
#define SMX_EXEC_BITS 2

/* grid_spec (maps.hpp:64-92) for the BB/H2D/H3D kinds. */
typedef struct smx_grid {
    int32_t kind;
    int32_t dims;
    int64_t n;   /* map parameter */
    int64_t rho; /* block edge: rho^dims cells per block */
    int64_t threshold;
    int64_t extents[3];
} smx_grid;

/* sim_report counters (simulator.hpp:76-88). */
typedef struct smx_counters {
    uint64_t blocks_launched;
    uint64_t blocks_void;
    uint64_t threads_launched;
    uint64_t threads_useful;
} smx_counters;

/* map_outcome (maps.hpp:40-47), 32 bytes. */
typedef struct smx_outcome {
    int32_t is_void;
    int32_t x, y, z;
    int32_t level_b;
    int32_t index_q;
    int32_t pad0, pad1;
} smx_outcome;

/* trapezoid_params (maps.hpp:49-60): one band of the concurrent-trapezoid
 * decomposition of a general-n 2-simplex (grid kind SMX_TRAP). */
typedef struct smx_trapezoid {
    int64_t delta_x, delta_y;
    int64_t band;        /* power-of-two triangle side */
    int64_t h1, h2;      /* last unfolded row; rows of the band-wide box */
    int64_t grid_width;  /* band / 2 */
    int64_t valid_side;  /* rows beyond are Void (final padded band only) */
    int64_t ext_x, ext_y;
} smx_trapezoid;

/* Thread-local message of the last failing call. */
const char* smx_last_error(void);

/* make_grid (report.hpp:48-66) -> grid_bb / grid_rb / grid_lambda / grid_h2d /
 * grid_h2d_padded / grid_trapezoids / grid_h3d (maps.hpp:96-105, 120-128,
 * 145-152, 188-198, 211-217, 259-266, 285-295). Same validity rules and
 * messages. An SMX_TRAP grid keeps extents {1, 1, 1} (as the reference) and
 * `threshold` = T; its bands come from smx_decompose_trapezoids. */
int smx_make_grid(int32_t kind, int32_t m, int64_t n, int64_t rho, int64_t threshold,
                  smx_grid* out);

/* grid_spec::domain_side()*rho: the cell side S of a launch (simulator.hpp:257-264). */
int64_t smx_cell_side(const smx_grid* g);

/* tri_cells / tet_cells (core.hpp:130-133). */
uint64_t smx_cell_count(int32_t m, int64_t side);

/* map_bb / map_rb_2d / map_lambda_2d (wx = linear index) / map_h2d /
 * map_h2d_padded / map_h3d for ONE block on the host (maps.hpp:107,133,156,
 * 200,219,302), same shared arithmetic the kernels inline
 * (include/smx_maps.hpp), with the reference's range checks. out: the raw
 * (strict-view where the kind is strict) outcome. */
int smx_map_one(int32_t kind, int32_t m, int64_t n, int64_t wx, int64_t wy, int64_t wz,
                smx_outcome* out);

/* decompose_trapezoids(n, T) (maps.hpp:228-257): writes up to `max` bands,
 * *count = the number of bands. */
int smx_decompose_trapezoids(int64_t n, int64_t T, smx_trapezoid* out, int32_t max, int32_t* count);

/* map_h2d_trapezoid (maps.hpp:269-281) for block (wx, wy) of band `band` of
 * decompose_trapezoids(n, T). */
int smx_map_trapezoid(int64_t n, int64_t T, int32_t band, int64_t wx, int64_t wy, smx_outcome* out);

/* grid_spec::blocks() (maps.hpp:73-82): the sum over the bands for SMX_TRAP. */
uint64_t smx_grid_blocks(const smx_grid* g);

/* The map over every block of the grid, natural z,y,x order, band after band
 * for SMX_TRAP (simulator.hpp:113-118,147-150) — the bit-exact coordinate check.
 * count = smx_grid_blocks(g). */
int smx_map_outcomes(const smx_grid* g, smx_outcome* out, uint64_t count, int device_ptr,
                     void* stream);

/* launch_map (simulator.hpp:303-310): coverage multiset (nullable) + counters
 * (nullable). coverage must hold smx_cell_count(dims, S) u32 and is ACCUMULATED into. */
int smx_launch_map(const smx_grid* g, uint32_t* coverage, uint64_t ncells, int device_ptr,
                   smx_counters* counters, void* stream);

/* The paper's MAP kernel for timing: map + thread expansion + membership +
 * packed index per thread, reduced to a register checksum (no memory sink). */
int smx_map_kernel(const smx_grid* g, void* stream);

/* launch_accum (simulator.hpp:313-327), `passes` times: ++cells[idx] per useful
 * thread. coverage (nullable) receives the first pass's visit counts. */
int smx_accum(const smx_grid* g, uint32_t* cells, uint64_t ncells, int64_t passes, int32_t exec,
              int device_ptr, uint32_t* coverage, smx_counters* counters, void* stream);

/* launch_accum over the grid rows wy in [wy_lo, wy_hi) only (device pointers,
 * 2-D non-trapezoid grids): the multi-GPU shard of ACCUM (blocks
 * are independent, so a rank runs a contiguous range of grid rows and no cell
 * data moves; only the counters are summed). counters (nullable): this range's
 * blocks_launched / blocks_void / threads_launched / threads_useful. */
int smx_accum_range(const smx_grid* g, uint32_t* cells, uint64_t ncells, int64_t passes, int32_t exec,
                    int64_t wy_lo, int64_t wy_hi, smx_counters* counters, void* stream);

/* make_life_state (simulator.hpp:390-398) for m = 3 (and m = 2): writes
 * smx_cell_count(m, side) bytes. */
int smx_life_init(int32_t m, int64_t side, uint64_t seed, uint8_t* cells, uint64_t ncells,
                  int device_ptr, void* stream);

/* verify_exact_cover (simulator.hpp:467-478) on the device: *first_bad = the
 * first packed index whose coverage is not 1 (ncells when exact),
 * *multiplicity = its coverage. Synchronises `stream`. */
int smx_verify_cover(const uint32_t* coverage, uint64_t ncells, int device_ptr, uint64_t* first_bad,
                     uint32_t* multiplicity, void* stream);

/* measure_grid (report.hpp:190-203) entirely on the device: one map launch
 * into a zeroed device coverage multiset (pool-owned) and, when check_cover,
 * the verify_exact_cover reduction above; only counters and the verdict come
 * back. check_cover = 0 is analyze_sweep's count-only launch. */
int smx_measure_grid(const smx_grid* g, int check_cover, smx_counters* counters, uint64_t* first_bad,
                     uint32_t* multiplicity, void* stream);

/* make_edm_points (simulator.hpp:333-343): count points, x then y drawn from
 * one seed-keyed splitmix64 stream; out_xy holds 2*count doubles (host). */
int smx_make_edm_points(int64_t count, uint64_t seed, double* out_xy);

/* launch_edm (simulator.hpp:352-372), m = 2, any 2-D map: cell (x, y) = the
 * distance between points x and y (f64, bit-identical to the reference's
 * edm_distance). points_xy: npoints = cell side pairs. coverage/counters as
 * for smx_accum. */
int smx_edm(const smx_grid* g, const double* points_xy, int64_t npoints, double* cells, uint64_t ncells,
            int32_t exec, int device_ptr, uint32_t* coverage, smx_counters* counters, void* stream);

/* One dead-boundary 3-D Life step through the map (the body of launch_ca's step
 * loop, simulator.hpp:440-459, with alive_neighbors_3d_dead :242-253 and
 * life_next :220-223). Device pointers only; cur and next must not alias. */
int smx_ca_step(const smx_grid* g, const uint8_t* cur, uint8_t* next, uint64_t ncells,
                int32_t exec, void* stream);

/* launch_ca (simulator.hpp:431-463): `steps` steps in place. m = 3: the
 * dead boundary (bb / h3d grids); m = 2: the periodic boundary
 * (alive_neighbors_2d_periodic, :227-239) through any 2-D map (smx_ca_step
 * likewise).
 * scratch: optional device buffer of ncells bytes (device_ptr mode); NULL =
 * library-managed. coverage/counters as for smx_accum (first step). */
int smx_ca(const smx_grid* g, uint8_t* cells, uint64_t ncells, int64_t steps, int32_t exec,
           int device_ptr, uint8_t* scratch, uint32_t* coverage, smx_counters* counters,
           void* stream);

/* launch_ca over `ndev` GPUs of ONE process (the C ABI's
 * multi-GPU launch_ca; 3-simplex grids, rho in {4, 8}). The grid's wz range is
 * cut into ndev contiguous shards of whole H levels balanced by useful blocks;
 * shard i runs on devices[i] (NULL: 0 .. ndev-1; an ordinal may repeat —
 * shards sharing a device run the same schedule with local copies) with its
 * own bit-shadow replica and its part of the engine plan, boundary chunks
 * first; each step's halo bit tiles go to the peers that read them by
 * peer-to-peer copies (NVLink) while the interior chunks run. `cells`: host
 * memory (device_ptr = 0) or device memory on devices[0]; `stream` belongs to
 * devices[0]. counters (nullable) as smx_ca. The per-grid plan and the
 * replicas are cached per (host thread, grid, device list); smx_release frees them. */
int smx_ca_multi(const smx_grid* g, uint8_t* cells, uint64_t ncells, int64_t steps, const int32_t* devices,
                 int32_t ndev, int device_ptr, smx_counters* counters, void* stream);

/* ---- the x-run CA engine's stages (what smx_ca_step / smx_ca chain) ----
 * A bit shadow holds one bit per cell in pitched rows (row (y, z) at word row
 * z*S + y, smx_bits_words() 32-bit words per row). Device pointers only.
 *   smx_bits_pack:   u8 packed state -> bit shadow
 *   smx_bits_step:   one Life step, bit shadow -> bit shadow, blocks with wz in
 *                    [wz_lo, wz_hi) of the map grid (the map drives the work)
 *   smx_bits_unpack: bit shadow -> u8 packed state */
uint64_t smx_bits_bytes(const smx_grid* g);
int smx_bits_pack(const smx_grid* g, const uint8_t* cells, uint64_t ncells, uint32_t* bits, void* stream);
int smx_bits_step(const smx_grid* g, const uint32_t* bits_in, uint32_t* bits_out, int64_t wz_lo, int64_t wz_hi,
                  void* stream);
int smx_bits_unpack(const smx_grid* g, const uint32_t* bits, uint8_t* cells, uint64_t ncells, void* stream);
/* The multi-step engine stage smx_ca runs between pack and unpack: the map is
 * applied once (a chunk list of the grid's x-adjacent tile chains), then ONE
 * persistent cooperative launch runs `steps` bit-sliced Life steps bits_a ->
 * bits_b -> bits_a ... (grid barrier between steps). The result is in bits_a
 * for even `steps`, bits_b for odd. Device pointers (smx_bits_bytes each). */
/* Both shadows must hold zero in every non-cell bit (rows y > S-1-z, words and
 * bits past x = y): allocate them zeroed (smx_bits_pack keeps it: it writes
 * the cell words with zero bits past the diagonal; the engines keep it). */
int smx_bits_run(const smx_grid* g, uint32_t* bits_a, uint32_t* bits_b, int64_t steps, void* stream);
/* Which engine smx_ca / smx_bits_run use for a 3-simplex grid: 0 = the chunk
 * engine (the map -> chains of x-adjacent tiles; small states), 1 = the
 * column engine (the map -> a tile bitmap; persistent z-marching columns of
 * 8 rows x 256 cells; large states); -1 for other grids. */
int smx_ca_engine(const smx_grid* g);

/* The engine's two stages, exposed for a sharded caller (one rank's part of
 * launch_ca over blocks with wz in [wz_lo, wz_hi) — SURVEY 8(e)):
 *   smx_bits_plan:     the map applied once to those blocks -> chunk list
 *                      (16 B per chunk: int32 cell x0, y0, z0, owned width;
 *                      rho tile rows per chunk) in `chunks` (capacity
 *                      smx_bits_plan_capacity(g) entries); *count (device u32)
 *                      receives the number of chunks. Asynchronous.
 *   smx_bits_run_list: ONE Life step bits_in -> bits_out over an explicit chunk
 *                      list (any subset of a plan, *count entries), so a shard
 *                      can run its boundary chunks first and its interior
 *                      while the halo travels. Device pointers. */
uint64_t smx_bits_plan_capacity(const smx_grid* g);
int smx_bits_plan(const smx_grid* g, int64_t wz_lo, int64_t wz_hi, void* chunks, uint32_t* count, void* stream);
int smx_bits_run_list(const smx_grid* g, uint32_t* bits_in, uint32_t* bits_out, const void* chunks,
                      const uint32_t* count, void* stream);

/* simplex_grid_state::hash (simulator.hpp:68-73): FNV-1a-64 over u64 m,
 * u64 side, then the raw cell bytes. Host bytes. */
uint64_t smx_state_hash(int32_t m, int64_t side, const void* bytes, uint64_t nbytes);

/* ---- multi-GPU shard support (H block-space partitioner) ----
 * One Life step restricted to H-grid blocks with wz in [wz_lo, wz_hi) (a
 * contiguous sub-box of whole sub-orthotope levels). Device pointers. Cells
 * of `next` outside the range keep their prior values on every exec scheme,
 * except that the x-run schemes (RUNS, BITS) may also store the correctly
 * stepped value of cells sharing a 32-cell word / 32-byte sector with a
 * range tile. */
int smx_ca_step_range(const smx_grid* g, const uint8_t* cur, uint8_t* next, uint64_t ncells,
                      int64_t wz_lo, int64_t wz_hi, int32_t exec, void* stream);

/* Gather / scatter whole tiles for the halo exchange. `tiles` is a DEVICE array
 * of int32 tile coordinates (X, Y, Z) in the with-diagonal tile view; tile k
 * occupies bytes [k*rho^3, (k+1)*rho^3) of the buffer in lz, ly, lx order;
 * cells outside the tetrahedron pack as 0 and are skipped on unpack. */
uint64_t smx_tile_bytes(const smx_grid* g, uint64_t ntiles);
int smx_tiles_pack(const smx_grid* g, const uint8_t* cells, const int32_t* tiles, uint64_t ntiles,
                   uint8_t* out, void* stream);
int smx_tiles_unpack(const smx_grid* g, uint8_t* cells, const int32_t* tiles, uint64_t ntiles,
                     const uint8_t* in, void* stream);

/* The same exchange on bit shadows (the sharded bit-shadow engine): tile k
 * occupies smx_bits_tile_bytes(g, 1) bytes (rho = 8: 64, rho = 4: 8) — rho^2
 * rows of rho bits, lz, ly order. Device pointers; rho in {4, 8}. */
uint64_t smx_bits_tile_bytes(const smx_grid* g, uint64_t ntiles);
int smx_bits_tiles_pack(const smx_grid* g, const uint32_t* bits, const int32_t* tiles, uint64_t ntiles, uint8_t* out,
                        void* stream);
int smx_bits_tiles_unpack(const smx_grid* g, uint32_t* bits, const int32_t* tiles, uint64_t ntiles,
                          const uint8_t* in, void* stream);

/* ---- the reference's sequential kernels (no block map), on the GPU ----
 * kernel_accum (simulator.hpp:329-331): every cell of the packed u32 state += 1. */
int smx_kernel_accum(uint32_t* cells, uint64_t ncells, int device_ptr, void* stream);
/* kernel_edm (simulator.hpp:377-386): cell (x, y) = edm_distance(p_x, p_y) for
 * the whole triangle of side npoints (f64, bit-identical to the reference). */
int smx_kernel_edm(const double* points_xy, int64_t npoints, double* cells, uint64_t ncells, int device_ptr,
                   void* stream);
/* kernel_ca_run (simulator.hpp:402-425): `steps` Life steps of the whole state
 * in place (m = 3: dead boundary; m = 2: periodic). Same messages as the
 * reference for bad m / side / steps. */
int smx_kernel_ca_run(int32_t m, int64_t side, uint8_t* cells, uint64_t ncells, int64_t steps, int device_ptr,
                      void* stream);

/* Frees the calling host thread's library scratch on every device (staging
 * pools, bit shadows, chunk lists, prefix tables, tensor maps, the side
 * stream); the next call re-creates what it needs. Synchronises the devices
 * (cudaFree). A thread's scratch is also freed automatically when the thread
 * exits. No reference counterpart: the reference holds no device state. */
int smx_release(void);

/* Bytes of pooled scratch the calling thread currently holds (all devices). */
uint64_t smx_scratch_bytes(void);

/* cudaDeviceSynchronize on the current device. */
int smx_device_sync(void);

#ifdef __cplusplus
}
#endif

#endif /* SMX_B200_H */
