// The C ABI (include/smx_b200.h): argument validation with the reference's
// contract messages, host<->device staging for host-buffer calls, the per-side
// layer-prefix tables, and dispatch to the sm_100a kernels.
#include <algorithm>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <initializer_list>
#include <map>
#include <memory>
#include <mutex>
#include <tuple>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "smx_b200.h"
#include "smx_common.cuh"
#include "smx_launch.hpp"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

const char* kind_name(int k) {
    switch (k) {
        case SMX_BB: return "bb";
        case SMX_RB: return "rb";
        case SMX_LAMBDA: return "lambda";
        case SMX_H2D: return "h2d";
        case SMX_TRAP: return "trapezoid";
        case SMX_PADDED: return "h2d-padded";
        case SMX_H3D: return "h3d";
    }
    return "?";
}

// map_supports_m / valid_pairs_text (report.hpp:28-46)
bool supports_m(int k, int m) {
    if (k == SMX_BB) return m == 2 || m == 3;
    if (k == SMX_H3D) return m == 3;
    return m == 2;
}
std::string valid_pairs() {
    return "bb (m=2,3), rb (m=2), lambda (m=2), h2d (m=2), trapezoid (m=2), h2d-padded (m=2), h3d (m=3)";
}

bool is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }

// Device-side resources, per (device, host thread): layer-prefix tables keyed
// by side, a grow-only scratch pool (staging for host-buffer calls, bit
// shadows, the CA chunk list), counters, the MAP sink and the side stream the
// CA plan runs on. Per host thread, so launches on distinct states from
// distinct threads never share scratch (the reference's functions are
// reentrant); calls from one thread are ordered on the stream they pass.
// A thread's resources are freed by smx_release() or when the thread exits.
struct DeviceRes {
    cudaStream_t side = nullptr;  // CA plan, concurrent with staging + pack
    cudaEvent_t ev_in = nullptr, ev_plan = nullptr;
    std::map<int64_t, unsigned long long*> prefix;
    // 0 cov, 1/2 u8, 3/4 bit shadows, 5 CA chunk list, 6 the engine's control
    // block (64 B: u32 [0] chunk count, u32 [8] grid barrier), 7 the
    // first-defect result of smx_verify_cover (its own slot: a verify on one
    // stream never touches the words of an engine running on another)
    // 8 the column engine's items (host-built, key cols_key), 9 the tile
    // bitmap (both engines), 10 the chunk plan's per-row counts, 11 the
    // periodic 2-D Life bit triangle
    void* pool[12] = {};
    size_t pool_bytes[12] = {};
    std::pair<int64_t, int64_t> cols_key{-1, -1};  // (side, layers per item) of the items in slot 8
    // the bit-shadow pools (slots 3, 4) keep every non-cell bit zero (the
    // column engine reads them unmasked): zeroed when (re)allocated or when
    // the side — the pitched layout — changes
    const void* shadow_ptr[2] = {nullptr, nullptr};
    int64_t shadow_side[2] = {-1, -1};
    int cols_nitems = 0;
    int cols_rows = 8;  // output rows per item of the items in slot 8
    // ACCUM x-run launch orders (H2D grids), keyed by (n, rho): device table + CTA count
    std::map<std::pair<int64_t, int64_t>, std::pair<void*, int>> accum_orders;
    std::map<std::pair<const void*, std::pair<int64_t, int64_t>>, CUtensorMap> tmaps;
    smx::DevCounters* counters = nullptr;
    unsigned* sink = nullptr;
    // pipelined host-buffer calls: the two copy streams and their events
    cudaStream_t copy_in = nullptr, copy_out = nullptr;
    cudaEvent_t ev_start = nullptr;
    std::vector<cudaEvent_t> ev_chunk;
};
std::mutex g_mu;
std::map<std::pair<int, std::thread::id>, DeviceRes> g_res;

// frees one DeviceRes on its device (cudaFree synchronises the device)
void free_res(int dev, DeviceRes& r) {
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess) return;
    if (cur != dev) cudaSetDevice(dev);
    for (auto& kv : r.prefix) cudaFree(kv.second);
    for (auto& kv : r.accum_orders) cudaFree(kv.second.first);
    for (int i = 0; i < 12; ++i)
        if (r.pool[i]) cudaFree(r.pool[i]);
    if (r.counters) cudaFree(r.counters);
    if (r.sink) cudaFree(r.sink);
    if (r.side) cudaStreamDestroy(r.side);
    if (r.ev_in) cudaEventDestroy(r.ev_in);
    if (r.ev_plan) cudaEventDestroy(r.ev_plan);
    if (r.copy_in) cudaStreamDestroy(r.copy_in);
    if (r.copy_out) cudaStreamDestroy(r.copy_out);
    if (r.ev_start) cudaEventDestroy(r.ev_start);
    for (cudaEvent_t e : r.ev_chunk) cudaEventDestroy(e);
    r = DeviceRes{};
    if (cur != dev) cudaSetDevice(cur);
}

void release_multi(std::thread::id tid);  // smx_ca_multi's cached shards (below)

// every device's resources of one host thread; returns how many sets were freed
int release_thread(std::thread::id tid) {
    release_multi(tid);
    std::vector<std::pair<int, DeviceRes>> mine;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        for (auto it = g_res.begin(); it != g_res.end();) {
            if (it->first.second == tid) {
                mine.emplace_back(it->first.first, std::move(it->second));
                it = g_res.erase(it);
            } else {
                ++it;
            }
        }
    }
    for (auto& kv : mine) free_res(kv.first, kv.second);
    return int(mine.size());
}

// thread-exit hook: a thread that used the ABI frees its scratch when it ends
// (thread pools no longer accumulate one full set per worker)
struct ThreadScratchOwner {
    bool used = false;
    ~ThreadScratchOwner() {
        if (used) release_thread(std::this_thread::get_id());
    }
};
thread_local ThreadScratchOwner t_owner;

int cuda_fail(cudaError_t e, const char* what) {
    return fail(SMX_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define TRY(expr)                                          \
    do {                                                   \
        cudaError_t _e = (expr);                           \
        if (_e != cudaSuccess) return cuda_fail(_e, #expr); \
    } while (0)

int device_res(DeviceRes** out) {
    int dev = 0;
    TRY(cudaGetDevice(&dev));
    t_owner.used = true;
    std::lock_guard<std::mutex> lk(g_mu);
    *out = &g_res[{dev, std::this_thread::get_id()}];
    return SMX_OK;
}

int get_prefix(int64_t side, const unsigned long long** out) {
    DeviceRes* r;
    if (int rc = device_res(&r)) return rc;
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = r->prefix.find(side);
    if (it != r->prefix.end()) {
        *out = it->second;
        return SMX_OK;
    }
    std::vector<unsigned long long> h(size_t(side) + 2);
    for (int64_t z = 0; z < side + 2; ++z) h[size_t(z)] = smx::tet_layer_prefix(side, z);
    unsigned long long* d = nullptr;
    TRY(cudaMalloc(&d, h.size() * sizeof(unsigned long long)));
    TRY(cudaMemcpy(d, h.data(), h.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice));
    r->prefix[side] = d;
    *out = d;
    return SMX_OK;
}

int pool_get(int slot, size_t bytes, void** out) {
    DeviceRes* r;
    if (int rc = device_res(&r)) return rc;
    std::lock_guard<std::mutex> lk(g_mu);
    if (r->pool_bytes[slot] < bytes) {
        // sweeps grow a slot grid after grid: below 256 MiB reserve 2x so a
        // monotone sweep reallocates O(log) times (cudaFree synchronises)
        constexpr size_t kGeom = size_t(256) << 20;
        size_t want = bytes;
        if (bytes < kGeom) want = std::max(bytes, std::min(2 * r->pool_bytes[slot], kGeom));
        if (r->pool[slot]) TRY(cudaFree(r->pool[slot]));
        r->pool[slot] = nullptr;
        r->pool_bytes[slot] = 0;
        TRY(cudaMalloc(&r->pool[slot], want + 256));  // 16B-granule reads past the end stay inside
        r->pool_bytes[slot] = want;
    }
    *out = r->pool[slot];
    return SMX_OK;
}

// a bit-shadow pool slot (3 or 4) for side S whose non-cell bits are zero
int shadow_get(int slot, int64_t side, void** out, cudaStream_t s);

int counters_buf(smx::DevCounters** out) {
    DeviceRes* r;
    if (int rc = device_res(&r)) return rc;
    std::lock_guard<std::mutex> lk(g_mu);
    if (!r->counters) TRY(cudaMalloc(&r->counters, sizeof(smx::DevCounters)));
    if (!r->sink) TRY(cudaMalloc(&r->sink, 64));
    *out = r->counters;
    return SMX_OK;
}

int sink_buf(unsigned** out) {
    smx::DevCounters* c;
    if (int rc = counters_buf(&c)) return rc;
    DeviceRes* r;
    if (int rc = device_res(&r)) return rc;
    *out = r->sink;
    return SMX_OK;
}

bool strict_kind_host(int k) { return k == SMX_H2D || k == SMX_PADDED || k == SMX_TRAP || k == SMX_H3D; }

int64_t cell_side_of(const smx_grid* g) {
    const int64_t ds = strict_kind_host(g->kind) ? g->n - 1 : g->n;
    return ds * g->rho;
}

constexpr int kMaxTraps = 64;

int trapezoids_of(int64_t n, int64_t T, smx::trapezoid<int64_t>* out, int* count) {
    if (n < 2) return fail(SMX_EINVAL, "decompose_trapezoids: n must be >= 2");
    if (T < 1) return fail(SMX_EINVAL, "decompose_trapezoids: T must be >= 1");
    const int c = smx::decompose_trapezoids(n, T, out, kMaxTraps);
    if (c < 0) return fail(SMX_ERANGE, "decompose_trapezoids: too many bands");
    *count = c;
    return SMX_OK;
}

uint64_t blocks_of(const smx_grid* g) {
    if (g->kind == SMX_TRAP) {
        smx::trapezoid<int64_t> t[kMaxTraps];
        int c = 0;
        if (trapezoids_of(g->n, g->threshold, t, &c)) return 0;
        uint64_t b = 0;
        for (int i = 0; i < c; ++i) b += uint64_t(t[i].ext_x) * uint64_t(t[i].ext_y);
        return b;
    }
    return uint64_t(g->extents[0]) * uint64_t(g->extents[1]) * uint64_t(g->extents[2]);
}

// Kernel-facing geometry of one launch; every coordinate must fit int32 and
// every CUDA grid dimension the block scheme uses must fit the launch limits.
int make_geom_ext(const smx_grid* g, int64_t ex, int64_t ey, int64_t ez, smx::Geom* out, bool need_prefix) {
    if (!g) return fail(SMX_EINVAL, "null grid");
    if (g->kind < SMX_BB || g->kind > SMX_H3D) return fail(SMX_EINVAL, "unknown map kind");
    if (g->rho < 1) return fail(SMX_EINVAL, "launch: rho must be >= 1");
    const int64_t side = cell_side_of(g);
    if (side >= (int64_t(1) << 30) || ex > 0x7fffffff || ey > 65535 || ez > 65535 || g->rho > 1024)
        return fail(SMX_ERANGE, "grid exceeds the device launch limits (extents.y,z <= 65535, side < 2^30)");
    smx::Geom k{};
    k.kind = g->kind;
    k.dims = g->dims;
    k.n = int(g->n);
    k.rho = int(g->rho);
    k.ex = int(ex);
    k.ey = int(ey);
    k.ez = int(ez);
    k.strict = strict_kind_host(g->kind);
    k.side = int(side);
    k.prefix = nullptr;
    if (need_prefix && g->dims == 3) {
        if (int rc = get_prefix(side, &k.prefix)) return rc;
    }
    *out = k;
    return SMX_OK;
}

int make_geom(const smx_grid* g, smx::Geom* out, bool need_prefix) {
    if (g && g->kind == SMX_TRAP) return fail(SMX_EINVAL, "trapezoid grids launch band by band");
    if (!g) return fail(SMX_EINVAL, "null grid");
    return make_geom_ext(g, g->extents[0], g->extents[1], g->extents[2], out, need_prefix);
}

// The launches of a grid: one for every kind but SMX_TRAP, one per band there
// (the reference's concurrent trapezoid launches, maps.hpp:259-266).
int sub_geoms(const smx_grid* g, std::vector<smx::Geom>& out, bool need_prefix) {
    out.clear();
    if (!g) return fail(SMX_EINVAL, "null grid");
    if (g->kind != SMX_TRAP) {
        smx::Geom k;
        if (int rc = make_geom(g, &k, need_prefix)) return rc;
        out.push_back(k);
        return SMX_OK;
    }
    smx::trapezoid<int64_t> t[kMaxTraps];
    int c = 0;
    if (int rc = trapezoids_of(g->n, g->threshold, t, &c)) return rc;
    for (int i = 0; i < c; ++i) {
        smx::Geom k;
        if (int rc = make_geom_ext(g, t[i].ext_x, t[i].ext_y, 1, &k, need_prefix)) return rc;
        k.trap = smx::trapezoid<int>{int(t[i].delta_x), int(t[i].delta_y), int(t[i].band), int(t[i].h1),
                                     int(t[i].h2), int(t[i].grid_width), int(t[i].valid_side), int(t[i].ext_x),
                                     int(t[i].ext_y)};
        out.push_back(k);
    }
    return SMX_OK;
}

uint64_t cells_of(int m, int64_t side) { return m == 2 ? smx::tri_cells(side) : smx::tet_cells(side); }

int check_cells(const smx_grid* g, uint64_t ncells) {
    if (ncells != cells_of(g->dims, cell_side_of(g)))
        return fail(SMX_EINVAL, "launch: state does not match the domain");
    return SMX_OK;
}

int fill_counters(const smx_grid* g, smx_counters* c, cudaStream_t s, uint32_t* dev_cov) {
    std::vector<smx::Geom> subs;
    if (int rc = sub_geoms(g, subs, true)) return rc;
    smx::DevCounters* dc = nullptr;
    if (c) {
        if (int rc = counters_buf(&dc)) return rc;
        TRY(cudaMemsetAsync(dc, 0, sizeof(smx::DevCounters), s));
    }
    for (const auto& k : subs) smx::launch_map_block(k, dev_cov, dc, nullptr, s);
    TRY(cudaGetLastError());
    if (c) {
        smx::DevCounters h;
        TRY(cudaMemcpyAsync(&h, dc, sizeof h, cudaMemcpyDeviceToHost, s));
        TRY(cudaStreamSynchronize(s));
        uint64_t v = 0, u = 0;
        for (int i = 0; i < smx::NSLOT; ++i) {
            v += h.blocks_void[i];
            u += h.threads_useful[i];
        }
        const uint64_t blocks = blocks_of(g);
        uint64_t tpb = uint64_t(g->rho) * uint64_t(g->rho);
        if (g->dims == 3) tpb *= uint64_t(g->rho);
        c->blocks_launched = blocks;
        c->blocks_void = v;
        c->threads_launched = blocks * tpb;
        c->threads_useful = u;
    }
    return SMX_OK;
}

int resolve_exec(int exec) {
    if (exec == SMX_EXEC_BLOCK || exec == SMX_EXEC_RUNS) return exec;
    return -1;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    // resolved once, thread-safe (function-local static initialiser)
    static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
        return PFN_cuTensorMapEncodeTiled_v12000(nullptr);
    }();
    return fn;
}

// 3-D tiled tensor map over a pitched bit shadow: (WP words, S rows, S layers),
// box b0 words x b1 rows x b2 layers; out-of-range coordinates read as zero.
// L2 sector promotion of the bit-shadow boxes (SMX_TMA_PROMO=none|64|128|256
// for experiments; default 128)
CUtensorMapL2promotion tma_promotion() {
    static const CUtensorMapL2promotion p = [] {
        const char* e = std::getenv("SMX_TMA_PROMO");
        if (!e) return CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
        const std::string v(e);
        if (v == "none") return CU_TENSOR_MAP_L2_PROMOTION_NONE;
        if (v == "64") return CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
        if (v == "256") return CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
        return CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    }();
    return p;
}
int bits_tmap_box(const uint32_t* bits, int64_t side, int b0, int b1, int b2, const CUtensorMap** out) {
    DeviceRes* r;
    if (int rc = device_res(&r)) return rc;
    std::lock_guard<std::mutex> lk(g_mu);
    auto key = std::make_pair((const void*)bits, std::make_pair(side, int64_t(b0) | int64_t(b1) << 16 | int64_t(b2) << 32));
    auto it = r->tmaps.find(key);
    if (it != r->tmaps.end()) {
        *out = &it->second;
        return SMX_OK;
    }
    auto fn = encode_fn();
    if (!fn) return fail(SMX_ECUDA, "cuTensorMapEncodeTiled unavailable from the driver");
    const int WP = smx::bits_pitch_words(int(side));
    cuuint64_t dims[3] = {cuuint64_t(WP), cuuint64_t(side), cuuint64_t(side)};
    cuuint64_t strides[2] = {cuuint64_t(WP) * 4, cuuint64_t(WP) * 4 * cuuint64_t(side)};
    cuuint32_t box[3] = {cuuint32_t(b0), cuuint32_t(b1), cuuint32_t(b2)};
    cuuint32_t estr[3] = {1u, 1u, 1u};
    CUtensorMap m;
    CUresult cr = fn(&m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, const_cast<uint32_t*>(bits), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, tma_promotion(),
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return fail(SMX_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(int(cr)));
    auto res = r->tmaps.emplace(key, m);
    *out = &res.first->second;
    return SMX_OK;
}
// the chunk engine's box: tma_box_words() x (rho + 2) x (rho + 2)
int bits_tmap(const uint32_t* bits, int64_t side, int64_t rho, const CUtensorMap** out) {
    const int hb = smx::tma_box_rows(int(rho));
    return bits_tmap_box(bits, side, smx::tma_box_words(), hb, hb, out);
}

int ca_fused_step(const smx::Geom& k, int64_t wz0, int64_t wz1, const uint8_t* cur, uint8_t* next, cudaStream_t s) {
    smx::launch_ca_fused(k, int(wz0), int(wz1), cur, next, s);
    TRY(cudaGetLastError());
    return SMX_OK;
}

// Which engine runs a launch_ca: the column engine for large states (map ->
// tile bitmap; persistent z-marching columns), the chunk engine for small
// ones (latency-bound: one short chunk per warp item). Crossover measured on
// B200 (tools/engine_ab.py, profiles/r2/engine_ab.txt): side 504-508 (21-22 M
// cells) chunks 10.5 / 15.1 us per step vs columns 15.9 / 17.2; side 1016-1020
// (175-177 M) columns 47.5 / 58.3 vs chunks 52.3 / 90.6; side 2040 columns 217
// vs 384. SMX_CA_ENGINE=chunks / cols forces one (A/B measurement, tests).
constexpr uint64_t kColsMinCells = 96ull << 20;
int cols_forced() {
    static const int forced = [] {
        const char* e = std::getenv("SMX_CA_ENGINE");
        if (!e) return 0;
        if (!std::strcmp(e, "chunks")) return 1;
        if (!std::strcmp(e, "cols")) return 2;
        return 0;
    }();
    return forced;
}
bool use_cols_side(int64_t side, int64_t rho) {
    if (rho == 16) return cols_forced() != 1 && smx::cols_supported(16) &&
                          (cols_forced() == 2 || smx::tet_cells(side) >= kColsMinCells);  // no chunk engine at 16
    if (cols_forced()) return cols_forced() == 2;
    return smx::tet_cells(side) >= kColsMinCells;
}
bool use_cols(const smx::Geom& k) { return use_cols_side(k.side, k.rho); }

// the column engine's work items (host): for layer segments of lz layers,
// every R-row band iy and 8-word group g with cells; item order keeps
// concurrently running warps on neighbouring columns (shared halo in L2)
std::vector<int32_t> col_items(int64_t S, int64_t lz, int64_t R) {
    std::vector<int32_t> v;
    for (int64_t zs = 0; zs < S; zs += lz)
        for (int64_t iy = 0; R * iy <= S - 1; ++iy) {
            const int64_t y0 = R * iy, zmax = S - y0;
            if (zs >= zmax) continue;
            const int64_t z1 = std::min(zs + lz, zmax);
            for (int64_t g = 0; 256 * g <= std::min(y0 + R - 1, S - 1); ++g)
                v.insert(v.end(), {int32_t(iy), int32_t(g), int32_t(zs), int32_t(z1)});
        }
    return v;
}

// the chunk engine's canonical plan of the blocks with wz in [wz0, wz1) on
// stream s: the map marks their tiles, the marked tile rows are cut into
// chunks in domain order; *count (device) = the chunk total
int canonical_plan(const smx_grid* g, const smx::Geom& k, int64_t wz0, int64_t wz1, void* chunks, unsigned* count,
                   cudaStream_t s) {
    const int D = int(k.side / k.rho), TW = (D + 31) / 32;
    const size_t bm_bytes = size_t(D) * size_t(D) * size_t(TW) * 4 + 16;
    void *pbm, *prc;
    if (int rc = pool_get(9, bm_bytes, &pbm)) return rc;
    if (int rc = pool_get(10, size_t(D) * size_t(D) * 4, &prc)) return rc;
    TRY(cudaMemsetAsync(pbm, 0, bm_bytes, s));
    smx::launch_cols_mark(k, g->kind, (uint32_t*)pbm, D, TW, (unsigned*)((uint8_t*)pbm + bm_bytes - 16), s, int(wz0),
                          int(wz1));
    smx::launch_chunkify(int(k.rho), (const uint32_t*)pbm, D, TW, (unsigned*)prc, chunks, count, s);
    TRY(cudaGetLastError());
    return SMX_OK;
}

struct EnginePlan {
    bool cols = false;
    void* chunks = nullptr;   // chunk engine: the chunk list
    unsigned* ctl = nullptr;  // chunk engine: [0] count, [8] barrier; column engine: [0] barrier, [1 + s] item counters
    void* items = nullptr;    // column engine
    int nitems = 0;
    uint32_t* bm = nullptr;
    int D = 0, TW = 0;
    int rows = 8;  // column engine: output rows per item
};

// The column engine's item shape for a side: 12-row items (fewer h-sum lanes
// idle, three rule chains per lane: C5 195 -> 184 us per step) while every
// warp still gets >= 3 of them at 32 layers; 8-row items below (C4, 1.3
// twelve-row items per warp: 42 vs 38 us per step). SMX_COLS_ROWS=8|12 forces.
int cols_rows_for(int64_t side) {
    static const int forced = [] {
        const char* e = std::getenv("SMX_COLS_ROWS");
        const int r = e ? std::atoi(e) : 0;
        return r == 8 || r == 12 ? r : 0;
    }();
    if (forced) return forced;
    const int64_t n12 = int64_t(col_items(side, 32, 12).size() / 4);
    return n12 >= 3 * int64_t(smx::cols_warps(12)) ? 12 : 8;
}

// plan (map once -> chunk list, or -> tile bitmap + column items) + the
// persistent multi-step run, A -> B -> A ...
//
// The plan depends on the grid only, so it is issued first, on a side stream
// ordered after the caller's prior work: it runs concurrently with whatever
// the caller stream does next (host staging, pack) until engine_run joins it.
int engine_plan(const smx_grid* g, const smx::Geom& k, int64_t steps, cudaStream_t s, EnginePlan* P) {
    if (steps > INT32_MAX) return fail(SMX_ERANGE, "launch_ca: steps must fit int32");
    DeviceRes* r;
    if (int rc = device_res(&r)) return rc;
    if (!r->side) {
        TRY(cudaStreamCreateWithFlags(&r->side, cudaStreamNonBlocking));
        TRY(cudaEventCreateWithFlags(&r->ev_in, cudaEventDisableTiming));
        TRY(cudaEventCreateWithFlags(&r->ev_plan, cudaEventDisableTiming));
    }
    P->cols = use_cols(k);
    void* pctl;
    const size_t ctl_bytes = P->cols ? std::max<size_t>(64, 4 * size_t(steps + 1)) : 64;
    if (int rc = pool_get(6, ctl_bytes, &pctl)) return rc;
    P->ctl = (unsigned*)pctl;
    TRY(cudaEventRecord(r->ev_in, s));
    TRY(cudaStreamWaitEvent(r->side, r->ev_in, 0));
    TRY(cudaMemsetAsync(pctl, 0, ctl_bytes, r->side));
    // SMX_CHUNK_PLAN=adjacency: the chunk engine's round-1 plan (chains of
    // x-adjacent tiles found through the map's block adjacency, k_ca_plan)
    static const bool adjacency_plan = [] {
        const char* e = std::getenv("SMX_CHUNK_PLAN");
        return e && !std::strcmp(e, "adjacency");
    }();
    if (!P->cols && adjacency_plan) {
        if (int rc = pool_get(5, size_t(smx::ca_plan_capacity(k)) * 16, &P->chunks)) return rc;
        smx::launch_ca_plan(k, g->kind, P->chunks, P->ctl, r->side);
    } else if (!P->cols) {
        // the map marks its tiles; every tile row is cut into chunks (canonical)
        if (int rc = pool_get(5, size_t(smx::ca_plan_capacity(k)) * 16, &P->chunks)) return rc;
        if (int rc = canonical_plan(g, k, 0, k.ez, P->chunks, P->ctl, r->side)) return rc;
    } else {
        P->D = int(k.side / k.rho);
        P->TW = (P->D + 31) / 32;
        const size_t bm_bytes = size_t(P->D) * size_t(P->D) * size_t(P->TW) * 4 + 16;
        void* pbm;
        if (int rc = pool_get(9, bm_bytes, &pbm)) return rc;
        P->bm = (uint32_t*)pbm;
        TRY(cudaMemsetAsync(pbm, 0, bm_bytes, r->side));
        // the map, applied once: every emitted tile marked (stats: marked, duplicate)
        smx::launch_cols_mark(k, g->kind, P->bm, P->D, P->TW, (unsigned*)((uint8_t*)pbm + bm_bytes - 16), r->side);
        // items: layer segments long enough for few atomics and little
        // warm-up, short enough for ~6 items per warp where the side allows;
        // built and uploaded once per side (host work off the per-call path)
        if (r->cols_key.first != int64_t(k.side)) {
            const int R = cols_rows_for(k.side);
            const int64_t target = 6 * int64_t(smx::cols_warps(R));
            int64_t lz = 64;
            std::vector<int32_t> v = col_items(k.side, lz, R);
            if (const char* e = std::getenv("SMX_COLS_LZ")) {  // experiments: a fixed item length
                lz = std::max<int64_t>(8, std::atoll(e) / 8 * 8);
                v = col_items(k.side, lz, R);
            } else {
                // not below 32 layers: an item pays two warm-up layers and a
                // partial tail stage (C4: lz 8 -> 32 is 43.4 -> 38.0 us per step)
                while (lz > 32 && int64_t(v.size() / 4) < target) v = col_items(k.side, lz /= 2, R);
            }
            r->cols_rows = R;
            void* pit;
            if (int rc = pool_get(8, v.size() * 4, &pit)) return rc;
            TRY(cudaMemcpy(pit, v.data(), v.size() * 4, cudaMemcpyHostToDevice));
            r->cols_key = {int64_t(k.side), lz};
            r->cols_nitems = int(v.size() / 4);
        }
        P->items = r->pool[8];
        P->nitems = r->cols_nitems;
        P->rows = r->cols_rows;
    }
    TRY(cudaGetLastError());
    TRY(cudaEventRecord(r->ev_plan, r->side));
    return SMX_OK;
}

// One persistent (cooperative, whole-device) engine grid per device at a time:
// a cooperative launch is sized to fill every SM, so two of them from
// different host threads / streams must not interleave their CTAs. Each
// engine launch waits on the previous one's completion event of that device
// (any thread); pack, unpack and copies of other calls still overlap.
std::mutex g_engine_mu;
cudaEvent_t g_engine_done[smx::kMaxDevices] = {};

// join the plan, then ONE persistent launch for all steps
int engine_run(const smx::Geom& k, uint32_t* A, uint32_t* B, int64_t steps, cudaStream_t s, const EnginePlan& P) {
    DeviceRes* r;
    if (int rc = device_res(&r)) return rc;
    TRY(cudaStreamWaitEvent(s, r->ev_plan, 0));
    int dev = 0;
    TRY(cudaGetDevice(&dev));
    if (dev < 0 || dev >= smx::kMaxDevices) return fail(SMX_EINVAL, "device ordinal beyond the library's table");
    const CUtensorMap *ta, *tb;
    if (P.cols) {
        if (int rc = bits_tmap_box(A, k.side, smx::cols_box_words(), smx::cols_box_rows(P.rows), smx::cols_box_layers(),
                                    &ta))
            return rc;
        if (int rc = bits_tmap_box(B, k.side, smx::cols_box_words(), smx::cols_box_rows(P.rows), smx::cols_box_layers(),
                                    &tb))
            return rc;
    } else {
        if (int rc = bits_tmap(A, k.side, k.rho, &ta)) return rc;
        if (int rc = bits_tmap(B, k.side, k.rho, &tb)) return rc;
    }
    std::lock_guard<std::mutex> lk(g_engine_mu);
    cudaEvent_t& done = g_engine_done[dev];
    if (!done) {
        TRY(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
    } else {
        TRY(cudaStreamWaitEvent(s, done, 0));
    }
    if (P.cols)
        TRY(smx::launch_cols_run(k, P.rows, ta, tb, A, B, P.items, P.nitems, P.ctl, P.bm, P.D, P.TW, int(steps), s));
    else
        TRY(smx::launch_ca_bits_run(k, ta, tb, A, B, P.chunks, P.ctl, int(steps), s));
    TRY(cudaEventRecord(done, s));
    return SMX_OK;
}

int bits_engine(const smx_grid* g, const smx::Geom& k, uint32_t* A, uint32_t* B, int64_t steps, cudaStream_t s) {
    if (steps <= 0) return SMX_OK;
    EnginePlan P;
    if (int rc = engine_plan(g, k, steps, s, &P)) return rc;
    return engine_run(k, A, B, steps, s, P);
}

size_t bits_bytes(int64_t side) {
    return size_t(smx::bits_rows(int(side))) * size_t(smx::bits_pitch_words(int(side))) * 4;
}

int shadow_get(int slot, int64_t side, void** out, cudaStream_t s) {
    const size_t bytes = bits_bytes(side);
    if (int rc = pool_get(slot, bytes, out)) return rc;
    DeviceRes* r;
    if (int rc = device_res(&r)) return rc;
    const int i = slot - 3;
    if (r->shadow_ptr[i] != *out || r->shadow_side[i] != side) {
        TRY(cudaMemsetAsync(*out, 0, bytes, s));
        r->shadow_ptr[i] = *out;
        r->shadow_side[i] = side;
    }
    return SMX_OK;
}

// One x-run step u8 -> u8: pack cur into pooled bit shadow A, k_ca_bits A -> B,
// unpack B into next.
int ca_runs_step(const smx_grid* g, const smx::Geom& k, int64_t wz0, int64_t wz1, const uint8_t* cur, uint8_t* next,
                 cudaStream_t s) {
    void *pa, *pb;
    if (int rc = shadow_get(3, k.side, &pa, s)) return rc;
    if (int rc = shadow_get(4, k.side, &pb, s)) return rc;
    if (wz0 == 0 && wz1 == k.ez) {
        // the whole grid: the engine's plan (issued first, on the side stream,
        // concurrent with the pack) + one persistent launch of 1 step
        EnginePlan plan;
        if (int rc = engine_plan(g, k, 1, s, &plan)) return rc;
        smx::launch_pack_bits(k, cur, (uint32_t*)pa, s);
        if (int rc = engine_run(k, (uint32_t*)pa, (uint32_t*)pb, 1, s, plan)) return rc;
    } else {
        // a wz sub-range: B is seeded from `next` so the unpack leaves next's
        // cells outside the range as they were (cells sharing a 32-cell word
        // with a range tile receive their correctly stepped value: the kernel
        // stores whole words computed from the full neighbourhood)
        const CUtensorMap* ta;
        if (int rc = bits_tmap((const uint32_t*)pa, k.side, k.rho, &ta)) return rc;
        smx::launch_pack_bits(k, cur, (uint32_t*)pa, s);
        smx::launch_pack_bits(k, next, (uint32_t*)pb, s);
        smx::launch_ca_bits(k, g->kind, int(wz0), int(wz1), ta, (uint32_t*)pb, s);
    }
    smx::launch_unpack_bits(k, (const uint32_t*)pb, next, s);
    TRY(cudaGetLastError());
    return SMX_OK;
}

// Host-buffer ACCUM, pipelined: the packed state is cut at tile-row
// boundaries into ~kPipeBytes chunks; chunk c's H2D copy (copy engine 1),
// the x-run kernel restricted to the tiles whose data row lies in the chunk
// (the full map walk; blocks mapping elsewhere drop out in the lane-parallel
// map), and its D2H copy (copy engine 2) overlap those of the neighbouring
// chunks, so PCIe runs both directions at once.
int accum_host_pipelined(const smx_grid* g, const std::vector<smx::Geom>& subs, uint32_t* cells, uint64_t ncells,
                         int64_t passes, int exec, cudaStream_t s) {
    constexpr uint64_t kPipeBytes = uint64_t(256) << 20;
    DeviceRes* r;
    if (int rc = device_res(&r)) return rc;
    void* p;
    if (int rc = pool_get(1, ncells * 4, &p)) return rc;
    uint32_t* d = (uint32_t*)p;
    if (!r->copy_in) {
        TRY(cudaStreamCreateWithFlags(&r->copy_in, cudaStreamNonBlocking));
        TRY(cudaStreamCreateWithFlags(&r->copy_out, cudaStreamNonBlocking));
        TRY(cudaEventCreateWithFlags(&r->ev_start, cudaEventDisableTiming));
    }
    const int64_t rho = g->rho, S = cell_side_of(g), trows = (S + rho - 1) / rho;
    auto row_off = [&](int64_t ty) { return smx::tri_cells(std::min(ty * rho, S)); };  // first cell of tile row ty
    // chunk boundaries (tile rows) so each chunk holds about kPipeBytes
    std::vector<int64_t> cuts{0};
    while (cuts.back() < trows) {
        int64_t lo = cuts.back() + 1, hi = trows;
        const uint64_t want = row_off(cuts.back()) + kPipeBytes / 4;
        while (lo < hi) {
            const int64_t mid = (lo + hi) / 2;
            if (row_off(mid) >= want) hi = mid;
            else lo = mid + 1;
        }
        cuts.push_back(lo);
    }
    const size_t nch = cuts.size() - 1;
    if (r->ev_chunk.size() < 2 * nch) {
        for (size_t i = r->ev_chunk.size(); i < 2 * nch; ++i) {
            cudaEvent_t e;
            TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            r->ev_chunk.push_back(e);
        }
    }
    TRY(cudaEventRecord(r->ev_start, s));  // after the caller's prior work
    TRY(cudaStreamWaitEvent(r->copy_in, r->ev_start, 0));
    for (size_t c = 0; c < nch; ++c) {
        const uint64_t o0 = row_off(cuts[c]), o1 = row_off(cuts[c + 1]);
        cudaEvent_t in = r->ev_chunk[2 * c], done = r->ev_chunk[2 * c + 1];
        TRY(cudaMemcpyAsync(d + o0, cells + o0, (o1 - o0) * 4, cudaMemcpyHostToDevice, r->copy_in));
        TRY(cudaEventRecord(in, r->copy_in));
        TRY(cudaStreamWaitEvent(s, in, 0));
        for (int64_t pass = 0; pass < passes; ++pass)
            for (smx::Geom k : subs) {
                k.ty0 = int(cuts[c]);
                k.ty1 = int(cuts[c + 1]);
                smx::launch_accum(k, d, exec, s);
            }
        TRY(cudaGetLastError());
        TRY(cudaEventRecord(done, s));
        TRY(cudaStreamWaitEvent(r->copy_out, done, 0));
        TRY(cudaMemcpyAsync(cells + o0, d + o0, (o1 - o0) * 4, cudaMemcpyDeviceToHost, r->copy_out));
    }
    TRY(cudaEventRecord(r->ev_start, r->copy_out));
    TRY(cudaStreamWaitEvent(s, r->ev_start, 0));  // the caller's stream sees the whole call
    TRY(cudaStreamSynchronize(s));
    return SMX_OK;
}


// ---------------------------------------------------------------------------
// launch_ca over several GPUs of ONE process (smx_ca_multi):
// the grid's wz range is cut into contiguous shards of whole levels balanced by
// useful blocks; shard s lives on devices[s] with a full bit-shadow replica
// pair, its part of the engine's plan (the map applied once) split into
// boundary chunks (holding a tile some peer reads) and interior chunks. Per
// step: boundary run -> bit-tile pack on the shard's comm stream -> one
// peer-to-peer copy per receiving peer (NVLink between devices; a plain
// device copy when two shards share a device) while the interior runs ->
// the receiver unpacks after its own runs (the runs store whole words).
// The host-side plan (partition + tile-level halo) is static per grid.

struct HostPlan {
    std::vector<std::pair<int64_t, int64_t>> wz;    // shard -> [lo, hi)
    std::vector<std::vector<int32_t>> owned;        // shard -> x, y, z tile triples
    std::vector<std::vector<std::vector<int32_t>>> send;  // [s][o] tiles s computes that o reads
    int64_t D = 0;                                  // with-diagonal tile-domain side
};

int build_host_plan(const smx_grid* g, int G, HostPlan* P) {
    const int64_t ex = g->extents[0], ey = g->extents[1], ez = g->extents[2];
    const bool strict = strict_kind_host(g->kind);
    const int64_t D = strict ? g->n - 1 : g->n;
    std::vector<uint64_t> useful(size_t(ez), 0);
    std::vector<int32_t> tiles;  // x, y, z per useful block, wz-major (natural order)
    std::vector<int64_t> tile_wz;
    for (int64_t wz = 0; wz < ez; ++wz)
        for (int64_t wy = 0; wy < ey; ++wy)
            for (int64_t wx = 0; wx < ex; ++wx) {
                const smx::outcome<int64_t> o = g->kind == SMX_H3D ? smx::map_h3d<int64_t>(wx, wy, wz, g->n)
                                                                   : smx::map_bb<int64_t>(wx, wy, wz, g->n, 3);
                if (o.is_void) continue;
                ++useful[size_t(wz)];
                tiles.push_back(int32_t(o.x));
                tiles.push_back(int32_t(strict ? o.y - 1 : o.y));
                tiles.push_back(int32_t(o.z));
                tile_wz.push_back(wz);
            }
    // contiguous wz ranges with ~equal useful blocks (dist.partition_wz)
    std::vector<double> cum(size_t(ez) + 1, 0.0);
    for (int64_t z = 0; z < ez; ++z) cum[size_t(z) + 1] = cum[size_t(z)] + double(useful[size_t(z)]);
    std::vector<int64_t> cuts{0};
    for (int r = 1; r < G; ++r) {
        const double target = cum.back() * r / G;
        int64_t k = int64_t(std::lower_bound(cum.begin(), cum.end(), target) - cum.begin());
        cuts.push_back(std::max(cuts.back(), std::min(k, ez)));
    }
    cuts.push_back(ez);
    P->wz.clear();
    for (int r = 0; r < G; ++r) P->wz.push_back({cuts[size_t(r)], cuts[size_t(r) + 1]});
    const size_t ntiles = tile_wz.size();
    std::vector<int16_t> owner(size_t(D * D * D), int16_t(-1));
    std::vector<int16_t> own_of(ntiles);
    P->owned.assign(size_t(G), {});
    for (size_t i = 0; i < ntiles; ++i) {
        int r = 0;
        while (tile_wz[i] >= P->wz[size_t(r)].second) ++r;
        own_of[i] = int16_t(r);
        const int64_t x = tiles[3 * i], y = tiles[3 * i + 1], z = tiles[3 * i + 2];
        owner[size_t((z * D + y) * D + x)] = int16_t(r);
        P->owned[size_t(r)].insert(P->owned[size_t(r)].end(), {int32_t(x), int32_t(y), int32_t(z)});
    }
    // tile-level 26-neighbourhood: t is sent to every other owner of a neighbour
    auto keys = std::vector<std::vector<std::vector<int64_t>>>(static_cast<size_t>(G),
                                                               std::vector<std::vector<int64_t>>(static_cast<size_t>(G)));
    for (size_t i = 0; i < ntiles; ++i) {
        const int64_t x = tiles[3 * i], y = tiles[3 * i + 1], z = tiles[3 * i + 2];
        const int s = own_of[i];
        for (int dz = -1; dz <= 1; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    const int64_t nx = x + dx, ny = y + dy, nz = z + dz;
                    if ((!dx && !dy && !dz) || !smx::tet_contains<int64_t>(D, nx, ny, nz)) continue;
                    const int o = owner[size_t((nz * D + ny) * D + nx)];
                    if (o >= 0 && o != s) keys[size_t(s)][size_t(o)].push_back((z * D + y) * D + x);
                }
    }
    P->send.assign(size_t(G), std::vector<std::vector<int32_t>>(size_t(G)));
    for (int s2 = 0; s2 < G; ++s2)
        for (int o = 0; o < G; ++o) {
            auto& k = keys[size_t(s2)][size_t(o)];
            std::sort(k.begin(), k.end());
            k.erase(std::unique(k.begin(), k.end()), k.end());
            for (int64_t key : k)
                P->send[size_t(s2)][size_t(o)].insert(P->send[size_t(s2)][size_t(o)].end(),
                                                      {int32_t(key % D), int32_t(key / D % D), int32_t(key / (D * D))});
        }
    P->D = D;
    return SMX_OK;
}

struct PeerCopy {
    int peer;
    uint64_t src_off, dst_off, bytes;
};

struct Shard {
    int dev = 0;
    smx::Geom k{};
    cudaStream_t cs = nullptr, ms = nullptr;          // compute, comm
    cudaEvent_t ev_b = nullptr, ev_sent = nullptr, ev_done = nullptr;
    uint32_t *A = nullptr, *B = nullptr;              // bit-shadow replicas
    const CUtensorMap *tA = nullptr, *tB = nullptr;
    void *bnd = nullptr, *inn = nullptr;              // chunk lists
    uint32_t* cnt = nullptr;                          // [0] boundary, [1] interior chunk counts
    uint64_t nb = 0, ni = 0;
    int32_t *send_t = nullptr, *recv_t = nullptr, *own_t = nullptr;
    uint64_t nsend = 0, nrecv = 0, nown = 0;
    uint8_t *send_b = nullptr, *recv_b = nullptr, *own_b = nullptr, *u8 = nullptr;
    std::vector<PeerCopy> copies;
    std::vector<int> senders;                         // shards that copy into this one
    std::vector<uint8_t*> gather_in;                  // shard 0 only: one buffer per other shard
};

struct MultiRes {
    std::vector<Shard> shards;
    cudaGraphExec_t pair = nullptr;  // two sharded steps (A -> B -> A) as one multi-device graph
    bool pair_failed = false;        // capture unsupported here: the steps are issued one by one
    ~MultiRes() { destroy(); }
    void destroy() {
        int cur = 0;
        cudaGetDevice(&cur);
        if (pair) cudaGraphExecDestroy(pair);
        pair = nullptr;
        for (auto& sh : shards) {
            cudaSetDevice(sh.dev);
            cudaDeviceSynchronize();
            for (void* p : std::initializer_list<void*>{sh.A, sh.B, sh.bnd, sh.inn, sh.cnt, sh.send_t, sh.recv_t,
                                                        sh.own_t, sh.send_b, sh.recv_b, sh.own_b, sh.u8})
                if (p) cudaFree(p);
            for (uint8_t* p : sh.gather_in)
                if (p) cudaFree(p);
            for (cudaEvent_t e : {sh.ev_b, sh.ev_sent, sh.ev_done})
                if (e) cudaEventDestroy(e);
            if (sh.cs) cudaStreamDestroy(sh.cs);
            if (sh.ms) cudaStreamDestroy(sh.ms);
        }
        shards.clear();
        cudaSetDevice(cur);
    }
};

struct MultiKey {
    std::thread::id tid;
    int32_t kind;
    int64_t n, rho;
    std::vector<int> devs;
    bool operator<(const MultiKey& o) const {
        return std::tie(tid, kind, n, rho, devs) < std::tie(o.tid, o.kind, o.n, o.rho, o.devs);
    }
};
std::mutex g_multi_mu;
std::map<MultiKey, std::unique_ptr<MultiRes>> g_multi;

void release_multi(std::thread::id tid) {
    std::vector<std::unique_ptr<MultiRes>> mine;
    {
        std::lock_guard<std::mutex> lk(g_multi_mu);
        for (auto it = g_multi.begin(); it != g_multi.end();) {
            if (it->first.tid == tid) {
                mine.push_back(std::move(it->second));
                it = g_multi.erase(it);
            } else {
                ++it;
            }
        }
    }
    mine.clear();  // destructors free on each shard's device
}

template <class T>
int dev_upload(const std::vector<T>& h, T** d) {
    TRY(cudaMalloc(d, std::max<size_t>(h.size(), 1) * sizeof(T)));
    if (!h.empty()) TRY(cudaMemcpy(*d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
    return SMX_OK;
}

// builds every shard: streams, replicas, the plan split, halo lists and copies
int multi_setup(const smx_grid* g, const std::vector<int>& devs, MultiRes* M) {
    const int G = int(devs.size());
    HostPlan P;
    if (int rc = build_host_plan(g, G, &P)) return rc;
    M->shards.assign(size_t(G), Shard{});
    const uint64_t tb = smx::bits_tile_bytes(int(g->rho));
    for (int s = 0; s < G; ++s) {
        Shard& sh = M->shards[size_t(s)];
        sh.dev = devs[size_t(s)];
        TRY(cudaSetDevice(sh.dev));
        if (int rc = make_geom(g, &sh.k, true)) return rc;
        TRY(cudaStreamCreateWithFlags(&sh.cs, cudaStreamNonBlocking));
        TRY(cudaStreamCreateWithFlags(&sh.ms, cudaStreamNonBlocking));
        for (cudaEvent_t* e : {&sh.ev_b, &sh.ev_sent, &sh.ev_done}) TRY(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        const size_t bb = bits_bytes(sh.k.side);
        TRY(cudaMalloc(&sh.A, bb + 256));
        TRY(cudaMalloc(&sh.B, bb + 256));
        TRY(cudaMalloc(&sh.u8, smx::tet_cells(sh.k.side) + 256));
        if (int rc = bits_tmap(sh.A, sh.k.side, sh.k.rho, &sh.tA)) return rc;
        if (int rc = bits_tmap(sh.B, sh.k.side, sh.k.rho, &sh.tB)) return rc;
        // the shard's plan, split on the host by the tiles its peers read
        void* all = nullptr;
        uint32_t* cnt = nullptr;
        TRY(cudaMalloc(&all, std::max<uint64_t>(smx::ca_plan_capacity(sh.k), 1) * 16));
        TRY(cudaMalloc(&cnt, 8));
        TRY(cudaMemset(cnt, 0, 8));
        if (int rc = canonical_plan(g, sh.k, P.wz[size_t(s)].first, P.wz[size_t(s)].second, all, cnt, sh.cs)) return rc;
        uint32_t n = 0;
        TRY(cudaMemcpyAsync(&n, cnt, 4, cudaMemcpyDeviceToHost, sh.cs));
        TRY(cudaStreamSynchronize(sh.cs));
        std::vector<int32_t> ch(size_t(n) * 4);
        if (n) TRY(cudaMemcpy(ch.data(), all, size_t(n) * 16, cudaMemcpyDeviceToHost));
        TRY(cudaFree(all));
        sh.cnt = cnt;
        const int64_t D = P.D, rho = g->rho;
        std::vector<uint8_t> mark(size_t(D * D * D), 0);
        std::vector<int32_t> send_all;
        for (int o = 0; o < G; ++o) {
            const auto& t = P.send[size_t(s)][size_t(o)];
            for (size_t i = 0; i < t.size(); i += 3) mark[size_t((int64_t(t[i + 2]) * D + t[i + 1]) * D + t[i])] = 1;
        }
        std::vector<int32_t> bnd, inn;
        for (uint32_t c = 0; c < n; ++c) {
            const int32_t* q = &ch[size_t(c) * 4];
            const int64_t tx0 = q[0] / rho, tx1 = (q[0] + q[3] + rho - 1) / rho, ty = q[1] / rho, tz = q[2] / rho;
            bool hit = false;
            for (int64_t tx = tx0; tx < tx1 && tx < D && !hit; ++tx) hit = mark[size_t((tz * D + ty) * D + tx)] != 0;
            (hit ? bnd : inn).insert((hit ? bnd : inn).end(), q, q + 4);
        }
        sh.nb = bnd.size() / 4;
        sh.ni = inn.size() / 4;
        if (int rc = dev_upload(bnd, (int32_t**)&sh.bnd)) return rc;
        if (int rc = dev_upload(inn, (int32_t**)&sh.inn)) return rc;
        const uint32_t counts[2] = {uint32_t(sh.nb), uint32_t(sh.ni)};
        TRY(cudaMemcpy(sh.cnt, counts, 8, cudaMemcpyHostToDevice));
        // send list: every peer's tiles in peer order, one pack launch per step
        for (int o = 0; o < G; ++o) {
            const auto& t = P.send[size_t(s)][size_t(o)];
            send_all.insert(send_all.end(), t.begin(), t.end());
        }
        sh.nsend = send_all.size() / 3;
        if (int rc = dev_upload(send_all, &sh.send_t)) return rc;
        TRY(cudaMalloc(&sh.send_b, std::max<uint64_t>(sh.nsend * tb, 1)));
        std::vector<int32_t> recv_all;
        for (int q = 0; q < G; ++q) {
            const auto& t = P.send[size_t(q)][size_t(s)];
            recv_all.insert(recv_all.end(), t.begin(), t.end());
            if (!t.empty()) sh.senders.push_back(q);
        }
        sh.nrecv = recv_all.size() / 3;
        if (int rc = dev_upload(recv_all, &sh.recv_t)) return rc;
        TRY(cudaMalloc(&sh.recv_b, std::max<uint64_t>(sh.nrecv * tb, 1)));
        sh.nown = P.owned[size_t(s)].size() / 3;
        if (int rc = dev_upload(P.owned[size_t(s)], &sh.own_t)) return rc;
        TRY(cudaMalloc(&sh.own_b, std::max<uint64_t>(sh.nown * tb, 1)));
    }
    // peer copies: s's slice for o lands at o's offset for sender s
    for (int s = 0; s < G; ++s) {
        uint64_t src = 0;
        for (int o = 0; o < G; ++o) {
            const uint64_t k = P.send[size_t(s)][size_t(o)].size() / 3;
            if (!k) continue;
            uint64_t dst = 0;
            for (int q = 0; q < s; ++q) dst += P.send[size_t(q)][size_t(o)].size() / 3;
            M->shards[size_t(s)].copies.push_back({o, src * tb, dst * tb, k * tb});
            src += k;
        }
    }
    // peer access between distinct devices (NVLink P2P); same-device shards copy locally
    for (int s = 0; s < G; ++s)
        for (int o = 0; o < G; ++o) {
            const int a = devs[size_t(s)], b = devs[size_t(o)];
            if (a == b) continue;
            int can = 0;
            TRY(cudaDeviceCanAccessPeer(&can, a, b));
            if (can) {
                TRY(cudaSetDevice(a));
                const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
                cudaGetLastError();
            }
        }
    Shard& s0 = M->shards[0];
    TRY(cudaSetDevice(s0.dev));
    s0.gather_in.assign(size_t(G), nullptr);
    for (int s = 1; s < G; ++s) TRY(cudaMalloc(&s0.gather_in[size_t(s)], std::max<uint64_t>(M->shards[size_t(s)].nown * tb, 1)));
    return SMX_OK;
}

// one sharded step, A -> B on every shard
int multi_step(MultiRes* M, bool even) {
    const int G = int(M->shards.size());
    for (auto& sh : M->shards) {
        TRY(cudaSetDevice(sh.dev));
        uint32_t* in = even ? sh.A : sh.B;
        uint32_t* out = even ? sh.B : sh.A;
        const CUtensorMap* tin = even ? sh.tA : sh.tB;
        if (sh.nb) TRY(smx::launch_ca_bits_list(sh.k, tin, in, out, sh.bnd, sh.cnt, sh.cs));
        TRY(cudaEventRecord(sh.ev_b, sh.cs));
        TRY(cudaStreamWaitEvent(sh.ms, sh.ev_b, 0));
        if (sh.nsend) smx::launch_bits_tiles_pack(sh.k, out, sh.send_t, sh.nsend, sh.send_b, sh.ms);
        if (sh.ni) TRY(smx::launch_ca_bits_list(sh.k, tin, in, out, sh.inn, sh.cnt + 1, sh.cs));
    }
    for (auto& sh : M->shards) {
        TRY(cudaSetDevice(sh.dev));
        for (const PeerCopy& c : sh.copies) {
            Shard& o = M->shards[size_t(c.peer)];
            TRY(cudaStreamWaitEvent(sh.ms, o.ev_done, 0));  // o has unpacked the previous step's halo
            // unified addressing: NVLink P2P between peer-enabled devices, a device copy within one
            // (cudaMemcpyDefault, unlike cudaMemcpyPeerAsync, is capturable into the step-pair graph)
            TRY(cudaMemcpyAsync(o.recv_b + c.dst_off, sh.send_b + c.src_off, c.bytes, cudaMemcpyDefault, sh.ms));
        }
        TRY(cudaEventRecord(sh.ev_sent, sh.ms));
    }
    for (auto& sh : M->shards) {
        TRY(cudaSetDevice(sh.dev));
        uint32_t* out = even ? sh.B : sh.A;
        for (int q : sh.senders) TRY(cudaStreamWaitEvent(sh.cs, M->shards[size_t(q)].ev_sent, 0));
        if (sh.nrecv) smx::launch_bits_tiles_unpack(sh.k, out, sh.recv_t, sh.nrecv, sh.recv_b, sh.cs);
        TRY(cudaGetLastError());
        TRY(cudaEventRecord(sh.ev_done, sh.cs));
    }
    (void)G;
    return SMX_OK;
}

int multi_pair_capture(MultiRes* M);

// events last recorded inside a capture cannot be waited on eagerly: record
// every shard's events again at the tails of their streams
void multi_rearm_events(MultiRes* M) {
    for (auto& sh : M->shards) {
        cudaSetDevice(sh.dev);
        cudaEventRecord(sh.ev_b, sh.cs);
        cudaEventRecord(sh.ev_done, sh.cs);
        cudaEventRecord(sh.ev_sent, sh.ms);
    }
    cudaSetDevice(M->shards[0].dev);
}

// capture two sharded steps (A -> B, B -> A) into one multi-device graph,
// once per MultiRes; on any capture error the steps run uncaptured
int multi_pair_graph(MultiRes* M) {
    if (M->pair) return SMX_OK;
    static const bool no_graph = std::getenv("SMX_MULTI_NOGRAPH") != nullptr;  // A/B: steps issued one by one
    if (M->pair_failed || no_graph) return SMX_ECUDA;
    const int rc = multi_pair_capture(M);
    multi_rearm_events(M);
    if (std::getenv("SMX_DEBUG_MULTI"))
        std::fprintf(stderr, "smx_ca_multi: step-pair graph %s (%zu shards)%s%s\n", rc ? "NOT captured" : "captured",
                     M->shards.size(), rc ? ": " : "", rc ? g_err.c_str() : "");
    return rc;
}

int multi_pair_capture(MultiRes* M) {
    Shard& s0 = M->shards[0];
    auto bail = [&](cudaError_t e) {
        cudaGraph_t dead = nullptr;
        cudaSetDevice(s0.dev);
        cudaStreamEndCapture(s0.cs, &dead);
        if (dead) cudaGraphDestroy(dead);
        cudaGetLastError();
        M->pair_failed = true;
        return cuda_fail(e, "capturing the sharded step pair");
    };
    cudaError_t e = cudaSetDevice(s0.dev);
    if (e == cudaSuccess) e = cudaStreamBeginCapture(s0.cs, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) return bail(e);
    // fork: every stream of every shard joins the capture; the cross-step
    // event (ev_done: a receiver unpacked its halo) is re-recorded inside it
    if ((e = cudaEventRecord(s0.ev_b, s0.cs)) != cudaSuccess) return bail(e);
    for (auto& sh : M->shards) {
        cudaSetDevice(sh.dev);
        if (&sh != &s0 && (e = cudaStreamWaitEvent(sh.cs, s0.ev_b, 0)) != cudaSuccess) return bail(e);
        if ((e = cudaStreamWaitEvent(sh.ms, s0.ev_b, 0)) != cudaSuccess) return bail(e);
        if ((e = cudaEventRecord(sh.ev_done, sh.cs)) != cudaSuccess) return bail(e);
    }
    if (multi_step(M, true) != SMX_OK || multi_step(M, false) != SMX_OK) return bail(cudaErrorStreamCaptureInvalidated);
    // join: every stream back into the origin
    for (auto& sh : M->shards) {
        cudaSetDevice(sh.dev);
        if ((e = cudaEventRecord(sh.ev_sent, sh.ms)) != cudaSuccess) return bail(e);
        cudaSetDevice(s0.dev);
        if ((e = cudaStreamWaitEvent(s0.cs, sh.ev_sent, 0)) != cudaSuccess) return bail(e);
        if (&sh != &s0) {
            cudaSetDevice(sh.dev);
            if ((e = cudaEventRecord(sh.ev_done, sh.cs)) != cudaSuccess) return bail(e);
            cudaSetDevice(s0.dev);
            if ((e = cudaStreamWaitEvent(s0.cs, sh.ev_done, 0)) != cudaSuccess) return bail(e);
        }
    }
    cudaSetDevice(s0.dev);
    cudaGraph_t graph = nullptr;
    if ((e = cudaStreamEndCapture(s0.cs, &graph)) != cudaSuccess) {
        cudaGetLastError();
        M->pair_failed = true;
        return cuda_fail(e, "capturing the sharded step pair");
    }
    e = cudaGraphInstantiate(&M->pair, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) {
        cudaGetLastError();
        M->pair = nullptr;
        M->pair_failed = true;
        return cuda_fail(e, "instantiating the sharded step pair");
    }
    return SMX_OK;
}

int ca_multi(const smx_grid* g, const std::vector<int>& devs, uint8_t* cells, uint64_t ncells, int64_t steps,
             int device_ptr, smx_counters* counters, cudaStream_t s) {
    int caller_dev = 0;
    TRY(cudaGetDevice(&caller_dev));
    MultiRes* M = nullptr;
    {
        const MultiKey key{std::this_thread::get_id(), g->kind, g->n, g->rho, devs};
        std::lock_guard<std::mutex> lk(g_multi_mu);
        auto& slot = g_multi[key];
        if (!slot) slot.reset(new MultiRes());
        M = slot.get();
    }
    if (M->shards.empty()) {
        const int rc = multi_setup(g, devs, M);
        if (rc) {
            M->destroy();
            cudaSetDevice(caller_dev);
            return rc;
        }
    }
    const int G = int(devs.size());
    Shard& s0 = M->shards[0];
    TRY(cudaSetDevice(s0.dev));
    if (counters && steps > 0)
        if (int rc = fill_counters(g, counters, s, nullptr)) return rc;
    // the state onto shard 0's device, then to every replica
    TRY(cudaEventRecord(s0.ev_done, s));
    TRY(cudaStreamWaitEvent(s0.cs, s0.ev_done, 0));
    TRY(cudaMemcpyAsync(s0.u8, cells, ncells, device_ptr ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s0.cs));
    TRY(cudaEventRecord(s0.ev_b, s0.cs));
    for (auto& sh : M->shards) {
        TRY(cudaSetDevice(sh.dev));
        TRY(cudaStreamWaitEvent(sh.cs, s0.ev_b, 0));
        if (&sh != &s0) TRY(cudaMemcpyPeerAsync(sh.u8, sh.dev, s0.u8, s0.dev, ncells, sh.cs));
        smx::launch_pack_bits(sh.k, sh.u8, sh.A, sh.cs);
        TRY(cudaGetLastError());
        TRY(cudaEventRecord(sh.ev_done, sh.cs));
    }
    // the steps: pairs of steps through one captured multi-device graph (one
    // launch instead of ~(5 + peers) API calls per shard and step), an odd
    // last step issued directly
    int64_t st = 0;
    if (!M->pair && !M->pair_failed && steps >= 4) {
        // the first pair runs uncaptured: every kernel's per-device attributes
        // are set before any capture begins
        for (; st < 2; ++st)
            if (int rc = multi_step(M, (st & 1) == 0)) return rc;
    }
    if (steps - st >= 2 && (M->pair || st > 0) && multi_pair_graph(M) == SMX_OK) {
        TRY(cudaSetDevice(s0.dev));
        for (auto& sh : M->shards) TRY(cudaStreamWaitEvent(s0.cs, sh.ev_done, 0));  // every replica packed
        for (; st + 2 <= steps; st += 2) TRY(cudaGraphLaunch(M->pair, s0.cs));
        TRY(cudaEventRecord(s0.ev_b, s0.cs));
        for (auto& sh : M->shards) {  // everything after waits for the graphs
            TRY(cudaSetDevice(sh.dev));
            TRY(cudaStreamWaitEvent(sh.cs, s0.ev_b, 0));
            TRY(cudaStreamWaitEvent(sh.ms, s0.ev_b, 0));
            TRY(cudaEventRecord(sh.ev_done, sh.cs));
        }
    }
    for (; st < steps; ++st)
        if (int rc = multi_step(M, (st & 1) == 0)) return rc;
    // gather: every other shard's owned bit tiles into shard 0's final shadow
    const bool odd = (steps & 1) != 0;
    for (int q = 1; q < G; ++q) {
        Shard& sh = M->shards[size_t(q)];
        TRY(cudaSetDevice(sh.dev));
        if (sh.nown) {
            smx::launch_bits_tiles_pack(sh.k, odd ? sh.B : sh.A, sh.own_t, sh.nown, sh.own_b, sh.cs);
            TRY(cudaMemcpyPeerAsync(s0.gather_in[size_t(q)], s0.dev, sh.own_b, sh.dev,
                                    sh.nown * smx::bits_tile_bytes(int(g->rho)), sh.cs));
        }
        TRY(cudaEventRecord(sh.ev_sent, sh.cs));
    }
    TRY(cudaSetDevice(s0.dev));
    uint32_t* fin = odd ? s0.B : s0.A;
    for (int q = 1; q < G; ++q) {
        Shard& sh = M->shards[size_t(q)];
        TRY(cudaStreamWaitEvent(s0.cs, sh.ev_sent, 0));
        if (sh.nown) smx::launch_bits_tiles_unpack(s0.k, fin, sh.own_t, sh.nown, s0.gather_in[size_t(q)], s0.cs);
    }
    smx::launch_unpack_bits(s0.k, fin, s0.u8, s0.cs);
    TRY(cudaGetLastError());
    TRY(cudaMemcpyAsync(cells, s0.u8, ncells, device_ptr ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s0.cs));
    TRY(cudaEventRecord(s0.ev_done, s0.cs));
    TRY(cudaStreamWaitEvent(s, s0.ev_done, 0));  // the caller's stream sees the whole call
    if (!device_ptr) TRY(cudaStreamSynchronize(s));
    TRY(cudaSetDevice(caller_dev));
    return SMX_OK;
}

}  // namespace

extern "C" {

const char* smx_last_error(void) { return g_err.c_str(); }

int smx_make_grid(int32_t kind, int32_t m, int64_t n, int64_t rho, int64_t threshold, smx_grid* out) {
    if (!out) return fail(SMX_EINVAL, "null output");
    if (kind < SMX_BB || kind > SMX_H3D) return fail(SMX_EINVAL, "unknown map kind");
    if (!supports_m(kind, m))
        return fail(SMX_EINVAL, std::string("map ") + kind_name(kind) + " does not support m=" +
                                    std::to_string(m) + "; valid: " + valid_pairs());
    if (rho < 1) return fail(SMX_EINVAL, "rho must be >= 1");
    smx_grid g{};
    g.kind = kind;
    g.dims = m;
    g.n = n;
    g.rho = rho;
    g.threshold = threshold;
    switch (kind) {
        case SMX_BB:
            if (n < 1) return fail(SMX_EINVAL, "grid_bb: n must be >= 1");
            g.extents[0] = n;
            g.extents[1] = n;
            g.extents[2] = m == 3 ? n : 1;
            break;
        case SMX_H2D:
            if (n < 2 || !is_pow2(n))
                return fail(SMX_EINVAL,
                            "grid_h2d: n must be a power of two >= 2; use decompose_trapezoids or "
                            "grid_h2d_padded for general n");
            g.extents[0] = n / 2;
            g.extents[1] = n - 1;
            g.extents[2] = 1;
            break;
        case SMX_H3D:
            if (n < 4 || !is_pow2(n))
                return fail(SMX_EINVAL,
                            "grid_h3d: n must be a power of two >= 4 (general-n 3D decomposition is "
                            "unsupported)");
            g.extents[0] = n / 2;
            g.extents[1] = n / 2;
            g.extents[2] = (3 * (n - 1) + 3) / 4;
            break;
        case SMX_RB:  // maps.hpp:120-128
            if (n < 1) return fail(SMX_EINVAL, "grid_rb: n must be >= 1");
            g.extents[0] = n % 2 == 0 ? n / 2 : (n + 1) / 2;
            g.extents[1] = n % 2 == 0 ? n + 1 : n;
            g.extents[2] = 1;
            break;
        case SMX_LAMBDA:  // maps.hpp:145-152
            if (n < 1) return fail(SMX_EINVAL, "grid_lambda: n must be >= 1");
            g.extents[0] = int64_t(smx::tri_cells(n));
            g.extents[1] = 1;
            g.extents[2] = 1;
            break;
        case SMX_PADDED: {  // maps.hpp:211-217: grid_h2d(2^ceil(log2 n))
            if (n < 2) return fail(SMX_EINVAL, "grid_h2d_padded: n must be >= 2");
            const int64_t p2 = int64_t(smx::pow2_ceil(uint64_t(n)));
            g.extents[0] = p2 / 2;
            g.extents[1] = p2 - 1;
            g.extents[2] = 1;
            break;
        }
        case SMX_TRAP: {  // maps.hpp:259-266: extents stay {1,1,1}; the bands carry the grid
            smx::trapezoid<int64_t> t[kMaxTraps];
            int c = 0;
            if (int rc = trapezoids_of(n, threshold, t, &c)) return rc;
            g.extents[0] = g.extents[1] = g.extents[2] = 1;
            break;
        }
        default:
            return fail(SMX_EINVAL, "unknown map kind");
    }
    *out = g;
    return SMX_OK;
}

uint64_t smx_grid_blocks(const smx_grid* g) { return g ? blocks_of(g) : 0; }

int smx_decompose_trapezoids(int64_t n, int64_t T, smx_trapezoid* out, int32_t max, int32_t* count) {
    smx::trapezoid<int64_t> t[kMaxTraps];
    int c = 0;
    if (int rc = trapezoids_of(n, T, t, &c)) return rc;
    if (count) *count = c;
    for (int i = 0; i < c && i < max && out; ++i)
        out[i] = smx_trapezoid{t[i].delta_x, t[i].delta_y, t[i].band, t[i].h1, t[i].h2,
                               t[i].grid_width, t[i].valid_side, t[i].ext_x, t[i].ext_y};
    return SMX_OK;
}

int smx_map_trapezoid(int64_t n, int64_t T, int32_t band, int64_t wx, int64_t wy, smx_outcome* out) {
    if (!out) return fail(SMX_EINVAL, "null output");
    smx::trapezoid<int64_t> t[kMaxTraps];
    int c = 0;
    if (int rc = trapezoids_of(n, T, t, &c)) return rc;
    if (band < 0 || band >= c) return fail(SMX_EINVAL, "map_h2d_trapezoid: no such band");
    const smx::trapezoid<int64_t>& p = t[band];
    if (wx < 0 || wx >= p.ext_x || wy < 0 || wy >= p.ext_y)
        return fail(SMX_EINVAL, "map_h2d_trapezoid: omega outside the trapezoid grid");
    const smx::outcome<int64_t> o = smx::map_h2d_trapezoid<int64_t>(wx, wy, p);
    *out = smx_outcome{int32_t(o.is_void), int32_t(o.x), int32_t(o.y), int32_t(o.z),
                       int32_t(o.level_b), int32_t(o.index_q), 0, 0};
    return SMX_OK;
}

int64_t smx_cell_side(const smx_grid* g) { return g ? cell_side_of(g) : -1; }

uint64_t smx_cell_count(int32_t m, int64_t side) {
    if ((m != 2 && m != 3) || side < 1) return 0;
    return cells_of(m, side);
}

int smx_map_one(int32_t kind, int32_t m, int64_t n, int64_t wx, int64_t wy, int64_t wz, smx_outcome* out) {
    if (!out) return fail(SMX_EINVAL, "null output");
    smx::outcome<int64_t> o;
    if (kind == SMX_BB) {
        if (m != 2 && m != 3) return fail(SMX_EINVAL, "map_bb: m must be 2 or 3");
        const bool in = wx >= 0 && wx < n && wy >= 0 && wy < n && (m == 2 ? wz == 0 : (wz >= 0 && wz < n));
        if (!in) return fail(SMX_EINVAL, "map_bb: omega outside the n^m grid");
        o = smx::map_bb<int64_t>(wx, wy, wz, n, m);
    } else if (kind == SMX_H2D) {
        if (wx < 0 || wy < 0) return fail(SMX_EINVAL, "map_h2d: omega components must be >= 0");
        if (wx >= (int64_t(1) << 31) || wy >= (int64_t(1) << 31))
            return fail(SMX_ERANGE, "map_h2d: omega beyond the 2^31 block range of this build");
        o = smx::map_h2d<int64_t>(wx, wy);
    } else if (kind == SMX_H3D) {
        if (n < 4 || !is_pow2(n)) return fail(SMX_EINVAL, "map_h3d: n must be a power of two >= 4");
        if (wx < 0 || wx >= n / 2 || wy < 0 || wy >= n / 2 || wz < 0 || wz >= (3 * (n - 1) + 3) / 4)
            return fail(SMX_EINVAL, "map_h3d: omega outside the grid");
        o = smx::map_h3d<int64_t>(wx, wy, wz, n);
    } else if (kind == SMX_PADDED) {  // maps.hpp:219-222
        if (wx < 0 || wy < 0) return fail(SMX_EINVAL, "map_h2d: omega components must be >= 0");
        if (wx >= (int64_t(1) << 31) || wy >= (int64_t(1) << 31))
            return fail(SMX_ERANGE, "map_h2d: omega beyond the 2^31 block range of this build");
        o = smx::map_h2d_padded<int64_t>(wx, wy, n);
    } else if (kind == SMX_RB) {  // maps.hpp:133-141
        if (n < 1) return fail(SMX_EINVAL, "grid_rb: n must be >= 1");
        const int64_t ex = n % 2 == 0 ? n / 2 : (n + 1) / 2, ey = n % 2 == 0 ? n + 1 : n;
        if (wx < 0 || wx >= ex || wy < 0 || wy >= ey) return fail(SMX_EINVAL, "map_rb_2d: omega outside the rectangle");
        o = smx::map_rb<int64_t>(wx, wy, n);
    } else if (kind == SMX_LAMBDA) {  // maps.hpp:156-159 (wx = linear index)
        if (wx < 0 || uint64_t(wx) >= smx::tri_cells(n))
            return fail(SMX_EINVAL, "map_lambda_2d: index out of range");
        o = smx::map_lambda<int64_t>(uint64_t(wx));
    } else {
        return fail(SMX_EINVAL, std::string("map ") + kind_name(kind) + ": use smx_map_trapezoid");
    }
    *out = smx_outcome{int32_t(o.is_void), int32_t(o.x), int32_t(o.y), int32_t(o.z),
                       int32_t(o.level_b), int32_t(o.index_q), 0, 0};
    return SMX_OK;
}

int smx_map_outcomes(const smx_grid* g, smx_outcome* out, uint64_t count, int device_ptr, void* stream) {
    std::vector<smx::Geom> subs;
    if (int rc = sub_geoms(g, subs, false)) return rc;
    const uint64_t blocks = blocks_of(g);
    if (count != blocks) return fail(SMX_EINVAL, "map_outcomes: count != grid blocks");
    cudaStream_t s = (cudaStream_t)stream;
    smx_outcome* d = out;
    if (!device_ptr) {
        void* p;
        if (int rc = pool_get(0, blocks * sizeof(smx_outcome), &p)) return rc;
        d = (smx_outcome*)p;
    }
    uint64_t off = 0;
    for (const auto& k : subs) {  // band after band for trapezoid grids (simulator.hpp:147-150)
        const uint64_t nb = uint64_t(k.ex) * uint64_t(k.ey) * uint64_t(k.ez);
        smx::launch_outcomes(k, d + off, nb, s);
        off += nb;
    }
    TRY(cudaGetLastError());
    if (!device_ptr) {
        TRY(cudaMemcpyAsync(out, d, blocks * sizeof(smx_outcome), cudaMemcpyDeviceToHost, s));
        TRY(cudaStreamSynchronize(s));
    }
    return SMX_OK;
}

int smx_launch_map(const smx_grid* g, uint32_t* coverage, uint64_t ncells, int device_ptr,
                   smx_counters* counters, void* stream) {
    std::vector<smx::Geom> subs;
    if (int rc = sub_geoms(g, subs, true)) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    uint32_t* dcov = coverage;
    if (coverage) {
        if (int rc = check_cells(g, ncells)) return rc;
        if (!device_ptr) {
            void* p;
            if (int rc = pool_get(0, ncells * 4, &p)) return rc;
            dcov = (uint32_t*)p;
            TRY(cudaMemcpyAsync(dcov, coverage, ncells * 4, cudaMemcpyHostToDevice, s));
        }
    }
    if (int rc = fill_counters(g, counters, s, dcov)) return rc;
    if (coverage && !device_ptr) {
        TRY(cudaMemcpyAsync(coverage, dcov, ncells * 4, cudaMemcpyDeviceToHost, s));
        TRY(cudaStreamSynchronize(s));
    }
    return SMX_OK;
}

int smx_map_kernel(const smx_grid* g, void* stream) {
    std::vector<smx::Geom> subs;
    if (int rc = sub_geoms(g, subs, true)) return rc;
    unsigned* sink;
    if (int rc = sink_buf(&sink)) return rc;
    for (const auto& k : subs) smx::launch_map_block(k, nullptr, nullptr, sink, (cudaStream_t)stream);
    TRY(cudaGetLastError());
    return SMX_OK;
}

// The ACCUM x-run kernel's CTAs in data order (H2D grids, rho >= 16, >= 2^18 blocks):
// H2D's grid row wy of level b covers data tile rows wy + 1 + 2 q b, so in
// blockIdx order a data row is written at ~log2(n) far-apart times; sorted by
// the data tile row (then column) of each CTA's first block, the CTAs running
// together stream consecutive data rows, as BB's grid rows do. Built on the
// host once per (n, rho), cached on the device.
int accum_order(const smx_grid* g, const smx::Geom& k, const int2** out, int* count) {
    *out = nullptr;
    *count = 0;
    static const int mode = [] {
        const char* e = std::getenv("SMX_ACCUM_ORDER");  // A/B: 0 = blockIdx order
        return e ? std::atoi(e) : 1;
    }();
    // rho >= 16 only: at rho 8 / 4 the sorted order measured slower (C3 domain:
    // 745 -> 730 / 481 -> 456 Gcells/s), at rho 16 it lifts H 791 -> 818 (= BB)
    if (!mode || g->kind != SMX_H2D || g->rho < 16 || uint64_t(k.ex) * uint64_t(k.ey) < (uint64_t(1) << 18))
        return SMX_OK;
    DeviceRes* r;
    if (int rc = device_res(&r)) return rc;
    const auto key = std::make_pair(int64_t(g->n), int64_t(g->rho));
    auto it = r->accum_orders.find(key);
    if (it == r->accum_orders.end()) {
        const int sb = smx::accum_strip_blocks(int(g->rho));
        const int gx = (k.ex + sb - 1) / sb;
        std::vector<std::pair<std::pair<int64_t, int64_t>, int2>> v;
        v.reserve(size_t(gx) * size_t(k.ey));
        for (int wy = 0; wy < k.ey; ++wy)
            for (int xs = 0; xs < gx; ++xs) {
                const auto o = smx::map_h2d<int64_t>(int64_t(xs) * sb, wy);
                v.push_back({{o.y, o.x}, make_int2(xs, wy)});
            }
        std::stable_sort(v.begin(), v.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
        std::vector<int2> h(v.size());
        for (size_t i = 0; i < v.size(); ++i) h[i] = v[i].second;
        void* d;
        TRY(cudaMalloc(&d, h.size() * sizeof(int2)));
        TRY(cudaMemcpy(d, h.data(), h.size() * sizeof(int2), cudaMemcpyHostToDevice));
        it = r->accum_orders.emplace(key, std::make_pair(d, int(h.size()))).first;
    }
    *out = (const int2*)it->second.first;
    *count = it->second.second;
    return SMX_OK;
}

int smx_accum(const smx_grid* g, uint32_t* cells, uint64_t ncells, int64_t passes, int32_t exec,
              int device_ptr, uint32_t* coverage, smx_counters* counters, void* stream) {
    std::vector<smx::Geom> subs;
    if (int rc = sub_geoms(g, subs, true)) return rc;
    if (g->dims != 2) return fail(SMX_EINVAL, "accum: the B200 ACCUM path is the 2-simplex kernel");
    if (int rc = check_cells(g, ncells)) return rc;
    if (passes < 0) return fail(SMX_EINVAL, "accum: passes must be >= 0");
    if (exec < 0) exec = SMX_EXEC_RUNS;
    if (resolve_exec(exec) < 0) return fail(SMX_EINVAL, "accum: unknown exec scheme");
    cudaStream_t s = (cudaStream_t)stream;
    // host state, x-run scheme, no coverage, > 1 chunk: the pipelined path
    if (!device_ptr && !coverage && exec == SMX_EXEC_RUNS && ncells * 4 > (uint64_t(512) << 20)) {
        if (counters)
            if (int rc = fill_counters(g, counters, s, nullptr)) return rc;
        return accum_host_pipelined(g, subs, cells, ncells, passes, exec, s);
    }
    uint32_t* d = cells;
    uint32_t* dcov = coverage;
    if (!device_ptr) {
        void* p;
        if (int rc = pool_get(1, ncells * 4, &p)) return rc;
        d = (uint32_t*)p;
        TRY(cudaMemcpyAsync(d, cells, ncells * 4, cudaMemcpyHostToDevice, s));
        if (coverage) {
            if (int rc = pool_get(0, ncells * 4, &p)) return rc;
            dcov = (uint32_t*)p;
            TRY(cudaMemcpyAsync(dcov, coverage, ncells * 4, cudaMemcpyHostToDevice, s));
        }
    }
    if (coverage || counters)
        if (int rc = fill_counters(g, counters, s, dcov)) return rc;
    if (exec == SMX_EXEC_RUNS && subs.size() == 1)
        if (int rc = accum_order(g, subs[0], &subs[0].order, &subs[0].norder)) return rc;
    for (int64_t p = 0; p < passes; ++p)
        for (const auto& k : subs) smx::launch_accum(k, d, exec, s);  // bands: disjoint cells
    TRY(cudaGetLastError());
    if (!device_ptr) {
        TRY(cudaMemcpyAsync(cells, d, ncells * 4, cudaMemcpyDeviceToHost, s));
        if (coverage) TRY(cudaMemcpyAsync(coverage, dcov, ncells * 4, cudaMemcpyDeviceToHost, s));
        TRY(cudaStreamSynchronize(s));
    }
    return SMX_OK;
}



int smx_accum_range(const smx_grid* g, uint32_t* cells, uint64_t ncells, int64_t passes, int32_t exec,
                    int64_t wy_lo, int64_t wy_hi, smx_counters* counters, void* stream) {
    if (!g) return fail(SMX_EINVAL, "null grid");
    if (g->dims != 2 || g->kind == SMX_TRAP)
        return fail(SMX_EINVAL, "accum_range: row ranges shard the 2-simplex grids other than trapezoid bands");
    smx::Geom k;
    if (int rc = make_geom(g, &k, true)) return rc;
    if (int rc = check_cells(g, ncells)) return rc;
    if (passes < 0) return fail(SMX_EINVAL, "accum: passes must be >= 0");
    if (wy_lo < 0 || wy_hi > k.ey || wy_lo > wy_hi) return fail(SMX_EINVAL, "accum_range: rows outside the grid");
    if (exec < 0) exec = SMX_EXEC_RUNS;
    if (resolve_exec(exec) < 0) return fail(SMX_EINVAL, "accum: unknown exec scheme");
    cudaStream_t s = (cudaStream_t)stream;
    k.wy0 = int(wy_lo);
    k.ey = int(wy_hi - wy_lo);
    if (counters) {
        smx::DevCounters* dc;
        if (int rc = counters_buf(&dc)) return rc;
        TRY(cudaMemsetAsync(dc, 0, sizeof(smx::DevCounters), s));
        if (k.ey > 0) smx::launch_map_block(k, nullptr, dc, nullptr, s);
        TRY(cudaGetLastError());
        smx::DevCounters h;
        TRY(cudaMemcpyAsync(&h, dc, sizeof h, cudaMemcpyDeviceToHost, s));
        TRY(cudaStreamSynchronize(s));
        uint64_t v = 0, u = 0;
        for (int i = 0; i < smx::NSLOT; ++i) v += h.blocks_void[i], u += h.threads_useful[i];
        const uint64_t blocks = uint64_t(k.ex) * uint64_t(k.ey);
        counters->blocks_launched = blocks;
        counters->blocks_void = v;
        counters->threads_launched = blocks * uint64_t(g->rho) * uint64_t(g->rho);
        counters->threads_useful = u;
    }
    if (k.ey > 0)
        for (int64_t p = 0; p < passes; ++p) smx::launch_accum(k, cells, exec, s);
    TRY(cudaGetLastError());
    return SMX_OK;
}

int smx_life_init(int32_t m, int64_t side, uint64_t seed, uint8_t* cells, uint64_t ncells, int device_ptr,
                  void* stream) {
    if (m != 2 && m != 3) return fail(SMX_EINVAL, "simplex_grid_state: m must be 2 or 3");
    if (side < 1) return fail(SMX_EINVAL, "simplex_grid_state: side must be >= 1");
    if (ncells != cells_of(m, side)) return fail(SMX_EINVAL, "life_init: ncells does not match the side");
    cudaStream_t s = (cudaStream_t)stream;
    uint8_t* d = cells;
    if (!device_ptr) {
        void* p;
        if (int rc = pool_get(1, ncells, &p)) return rc;
        d = (uint8_t*)p;
    }
    smx::launch_life_init(seed, d, ncells, s);
    TRY(cudaGetLastError());
    if (!device_ptr) {
        TRY(cudaMemcpyAsync(cells, d, ncells, cudaMemcpyDeviceToHost, s));
        TRY(cudaStreamSynchronize(s));
    }
    return SMX_OK;
}

// the x-run CA kernels move 16-byte vectors relative to the buffer base
static int check_align16(const void* a, const void* b) {
    if ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15u)
        return fail(SMX_EINVAL, "ca: device state buffers must be 16-byte aligned");
    return SMX_OK;
}

// EXEC_AUTO for ONE step: the fused u8 -> u8 kernel only for small rho = 4
// states (C2 size: it ties the bit-shadow path on H3D and wins on BB); the
// bit-shadow path (pack || plan, one persistent step, unpack) everywhere else
// (2x the fused kernel at H3D(64) rho = 8, 21 M cells). Multi-step launch_ca
// always uses the bit shadow (pack once, unpack once). Measured on B200:
// profiles/r1/ca_exec_sweep.txt.
constexpr uint64_t kFusedMaxCells = 4ull << 20;
static bool prefer_fused(const smx_grid* g, uint64_t ncells) { return g->rho == 4 && ncells <= kFusedMaxCells; }

static int ca_validate(const smx_grid* g, uint64_t ncells, int32_t* exec) {
    if (int rc = check_cells(g, ncells)) return rc;
    if (g->dims == 2) {  // periodic 2-D Life: BLOCK or RUNS (the x-run kernel), every 2-D map
        if (*exec < 0 || *exec == SMX_EXEC_BITS) *exec = SMX_EXEC_RUNS;
        if (*exec != SMX_EXEC_BLOCK && *exec != SMX_EXEC_RUNS) return fail(SMX_EINVAL, "ca: unknown exec scheme");
        return SMX_OK;
    }
    if (g->kind != SMX_BB && g->kind != SMX_H3D)
        return fail(SMX_EINVAL, "launch_ca: 3-simplex grids are bb or h3d");
    // rho = 16 runs the bit-shadow path only through the column engine (large states)
    const bool cols16 = g->rho == 16 && use_cols_side(cell_side_of(g), 16);
    if (*exec < 0) *exec = smx::ca_runs_supported(int(g->rho)) || cols16 ? SMX_EXEC_BITS : SMX_EXEC_BLOCK;
    if (*exec != SMX_EXEC_BLOCK && *exec != SMX_EXEC_RUNS && *exec != SMX_EXEC_BITS)
        return fail(SMX_EINVAL, "ca: unknown exec scheme");
    if (*exec == SMX_EXEC_BITS && cols16) return SMX_OK;
    if (*exec != SMX_EXEC_BLOCK && !smx::ca_runs_supported(int(g->rho)))
        return fail(SMX_EINVAL, "ca: the x-run schemes support rho in {4, 8} (16: the bit-shadow column engine "
                                "for states >= 96 M cells); use SMX_EXEC_BLOCK");
    return SMX_OK;
}

// One periodic 2-D Life step. The x-run scheme first packs the state into a
// bit triangle (bit i = packed cell i; 1/8 of the state, L2-resident at the
// SURVEY sizes) and reads its neighbourhoods from it; every band of a
// trapezoid grid reads the same triangle.
static int ca2d_step(const smx_grid* g, const uint8_t* cur, uint8_t* next, int32_t exec, cudaStream_t s) {
    std::vector<smx::Geom> subs;
    if (int rc = sub_geoms(g, subs, false)) return rc;
    const uint32_t* bits = nullptr;
    if (exec == SMX_EXEC_RUNS) {
        const uint64_t ncells = smx::tri_cells(cell_side_of(g));
        void* p;
        if (int rc = pool_get(11, size_t(smx::ca2d_bit_words(ncells)) * 4, &p)) return rc;
        smx::launch_pack2d(cur, ncells, (uint32_t*)p, s);
        bits = (const uint32_t*)p;
    }
    for (const auto& k : subs) smx::launch_ca2d(k, cur, bits, next, exec, s);  // bands: disjoint cells
    TRY(cudaGetLastError());
    return SMX_OK;
}

int smx_ca_step(const smx_grid* g, const uint8_t* cur, uint8_t* next, uint64_t ncells, int32_t exec,
                void* stream) {
    const bool auto_exec = exec < 0;
    if (g && g->dims == 2) {
        if (int rc = ca_validate(g, ncells, &exec)) return rc;
        if (cur == next) return fail(SMX_EINVAL, "ca_step: cur and next must not alias");
        if (int rc = check_align16(cur, next)) return rc;
        return ca2d_step(g, cur, next, exec, (cudaStream_t)stream);
    }
    smx::Geom k;
    if (int rc = make_geom(g, &k, true)) return rc;
    if (int rc = ca_validate(g, ncells, &exec)) return rc;
    if (cur == next) return fail(SMX_EINVAL, "ca_step: cur and next must not alias");
    if (int rc = check_align16(cur, next)) return rc;
    if (auto_exec && exec == SMX_EXEC_BITS && prefer_fused(g, ncells)) exec = SMX_EXEC_RUNS;
    if (exec == SMX_EXEC_BITS) return ca_runs_step(g, k, 0, k.ez, cur, next, (cudaStream_t)stream);
    if (exec == SMX_EXEC_RUNS) return ca_fused_step(k, 0, k.ez, cur, next, (cudaStream_t)stream);
    smx::launch_ca(k, 0, k.ez, cur, next, exec, (cudaStream_t)stream);
    TRY(cudaGetLastError());
    return SMX_OK;
}

int smx_ca_step_range(const smx_grid* g, const uint8_t* cur, uint8_t* next, uint64_t ncells, int64_t wz_lo,
                      int64_t wz_hi, int32_t exec, void* stream) {
    const bool auto_exec = exec < 0;
    smx::Geom k;
    if (int rc = make_geom(g, &k, true)) return rc;
    if (int rc = ca_validate(g, ncells, &exec)) return rc;
    if (wz_lo < 0 || wz_hi > g->extents[2] || wz_lo > wz_hi)
        return fail(SMX_EINVAL, "ca_step_range: wz range outside the grid");
    if (cur == next) return fail(SMX_EINVAL, "ca_step_range: cur and next must not alias");
    if (exec == SMX_EXEC_BITS && !smx::ca_runs_supported(int(g->rho)))
        return fail(SMX_EINVAL, "ca_step_range: the bit-shadow range step supports rho in {4, 8}");
    if (int rc = check_align16(cur, next)) return rc;
    if (auto_exec && exec == SMX_EXEC_BITS && prefer_fused(g, ncells)) exec = SMX_EXEC_RUNS;
    if (exec == SMX_EXEC_BITS) return ca_runs_step(g, k, wz_lo, wz_hi, cur, next, (cudaStream_t)stream);
    if (exec == SMX_EXEC_RUNS) return ca_fused_step(k, wz_lo, wz_hi, cur, next, (cudaStream_t)stream);
    smx::launch_ca(k, int(wz_lo), int(wz_hi), cur, next, exec, (cudaStream_t)stream);
    TRY(cudaGetLastError());
    return SMX_OK;
}

int smx_ca(const smx_grid* g, uint8_t* cells, uint64_t ncells, int64_t steps, int32_t exec, int device_ptr,
           uint8_t* scratch, uint32_t* coverage, smx_counters* counters, void* stream) {
    smx::Geom k;
    if (g && g->dims == 2) {
        k = smx::Geom{};
        if (!g) return fail(SMX_EINVAL, "null grid");
    } else if (int rc = make_geom(g, &k, true)) {
        return rc;
    }
    if (int rc = ca_validate(g, ncells, &exec)) return rc;
    if (steps < 0) return fail(SMX_EINVAL, "launch_ca: steps must be >= 0");
    cudaStream_t s = (cudaStream_t)stream;
    uint8_t* a = cells;
    uint8_t* b = scratch;
    uint32_t* dcov = coverage;
    void* p;
    // bit-shadow engine: the plan (map -> chunk list) needs only the grid, so
    // it is issued first and overlaps the input staging and the pack
    const bool engine = g->dims == 3 && exec == SMX_EXEC_BITS && steps > 0;
    EnginePlan plan;
    if (engine)
        if (int rc = engine_plan(g, k, steps, s, &plan)) return rc;
    if (!device_ptr) {
        if (int rc = pool_get(1, ncells, &p)) return rc;
        a = (uint8_t*)p;
        TRY(cudaMemcpyAsync(a, cells, ncells, cudaMemcpyHostToDevice, s));
        if (coverage) {
            if (int rc = pool_get(0, ncells * 4, &p)) return rc;
            dcov = (uint32_t*)p;
            TRY(cudaMemcpyAsync(dcov, coverage, ncells * 4, cudaMemcpyHostToDevice, s));
        }
    }
    if (!b) {
        if (int rc = pool_get(2, ncells, &p)) return rc;
        b = (uint8_t*)p;
    }
    if ((coverage || counters) && steps > 0)
        if (int rc = fill_counters(g, counters, s, dcov)) return rc;
    uint8_t* cur = a;
    uint8_t* nxt = b;
    if (device_ptr)
        if (int rc = check_align16(a, b)) return rc;
    if (g->dims == 2) {
        for (int64_t st = 0; st < steps; ++st) {
            if (int rc = ca2d_step(g, cur, nxt, exec, s)) return rc;
            std::swap(cur, nxt);
        }
    } else if (engine) {
        // bit-shadow engine: pack once, steps x (bits -> bits), unpack once
        void *pa, *pb;
        if (int rc = shadow_get(3, k.side, &pa, s)) return rc;
        if (int rc = shadow_get(4, k.side, &pb, s)) return rc;
        // the map applied once (chunk list / tile bitmap), then ONE persistent
        // launch for all steps, A -> B -> A ..., the final shadow unpacked in place
        smx::launch_pack_bits(k, cur, (uint32_t*)pa, s);
        if (int rc = engine_run(k, (uint32_t*)pa, (uint32_t*)pb, steps, s, plan)) return rc;
        smx::launch_unpack_bits(k, (steps & 1) ? (const uint32_t*)pb : (const uint32_t*)pa, cur, s);
    } else {
        for (int64_t st = 0; st < steps; ++st) {
            if (exec == SMX_EXEC_RUNS) {
                if (int rc = ca_fused_step(k, 0, k.ez, cur, nxt, s)) return rc;
            } else {
                smx::launch_ca(k, 0, k.ez, cur, nxt, exec, s);
            }
            std::swap(cur, nxt);
        }
    }
    TRY(cudaGetLastError());
    if (device_ptr) {
        if (cur != cells) TRY(cudaMemcpyAsync(cells, cur, ncells, cudaMemcpyDeviceToDevice, s));
    } else {
        TRY(cudaMemcpyAsync(cells, cur, ncells, cudaMemcpyDeviceToHost, s));
        if (coverage) TRY(cudaMemcpyAsync(coverage, dcov, ncells * 4, cudaMemcpyDeviceToHost, s));
        TRY(cudaStreamSynchronize(s));
    }
    return SMX_OK;
}

uint64_t smx_bits_bytes(const smx_grid* g) {
    if (!g || g->dims != 3) return 0;
    return bits_bytes(cell_side_of(g));
}

int smx_bits_pack(const smx_grid* g, const uint8_t* cells, uint64_t ncells, uint32_t* bits, void* stream) {
    smx::Geom k;
    if (int rc = make_geom(g, &k, true)) return rc;
    int32_t ex = SMX_EXEC_BITS;
    if (int rc = ca_validate(g, ncells, &ex)) return rc;
    smx::launch_pack_bits(k, cells, bits, (cudaStream_t)stream);
    TRY(cudaGetLastError());
    return SMX_OK;
}

int smx_bits_step(const smx_grid* g, const uint32_t* bits_in, uint32_t* bits_out, int64_t wz_lo, int64_t wz_hi,
                  void* stream) {
    smx::Geom k;
    if (int rc = make_geom(g, &k, true)) return rc;
    int32_t ex = SMX_EXEC_RUNS;
    if (int rc = ca_validate(g, smx::tet_cells(k.side), &ex)) return rc;
    if (wz_lo < 0 || wz_hi > g->extents[2] || wz_lo > wz_hi)
        return fail(SMX_EINVAL, "bits_step: wz range outside the grid");
    if (bits_in == bits_out) return fail(SMX_EINVAL, "bits_step: input and output must not alias");
    const CUtensorMap* tm;
    if (int rc = bits_tmap(bits_in, k.side, k.rho, &tm)) return rc;
    smx::launch_ca_bits(k, g->kind, int(wz_lo), int(wz_hi), tm, bits_out, (cudaStream_t)stream);
    TRY(cudaGetLastError());
    return SMX_OK;
}

int smx_bits_unpack(const smx_grid* g, const uint32_t* bits, uint8_t* cells, uint64_t ncells, void* stream) {
    smx::Geom k;
    if (int rc = make_geom(g, &k, true)) return rc;
    int32_t ex = SMX_EXEC_BITS;
    if (int rc = ca_validate(g, ncells, &ex)) return rc;
    smx::launch_unpack_bits(k, bits, cells, (cudaStream_t)stream);
    TRY(cudaGetLastError());
    return SMX_OK;
}

int smx_ca_engine(const smx_grid* g) {
    smx::Geom k;
    if (!g || g->dims != 3 || make_geom(g, &k, false)) return -1;
    return use_cols(k) ? 1 : 0;
}

int smx_bits_run(const smx_grid* g, uint32_t* bits_a, uint32_t* bits_b, int64_t steps, void* stream) {
    smx::Geom k;
    if (int rc = make_geom(g, &k, true)) return rc;
    int32_t ex = SMX_EXEC_BITS;
    if (int rc = ca_validate(g, smx::tet_cells(k.side), &ex)) return rc;
    if (steps < 0) return fail(SMX_EINVAL, "bits_run: steps must be >= 0");
    if (bits_a == bits_b) return fail(SMX_EINVAL, "bits_run: the two shadows must not alias");
    return bits_engine(g, k, bits_a, bits_b, steps, (cudaStream_t)stream);
}

uint64_t smx_bits_plan_capacity(const smx_grid* g) {
    smx::Geom k;
    if (!g || make_geom(g, &k, false)) return 0;
    return smx::ca_plan_capacity(k);
}

int smx_bits_plan(const smx_grid* g, int64_t wz_lo, int64_t wz_hi, void* chunks, uint32_t* count, void* stream) {
    smx::Geom k;
    if (int rc = make_geom(g, &k, true)) return rc;
    int32_t ex = SMX_EXEC_BITS;
    if (int rc = ca_validate(g, smx::tet_cells(k.side), &ex)) return rc;
    if (!smx::ca_runs_supported(int(g->rho))) return fail(SMX_EINVAL, "bits_plan: the chunk engine supports rho in {4, 8}");
    if (wz_lo < 0 || wz_hi > g->extents[2] || wz_lo > wz_hi) return fail(SMX_EINVAL, "bits_plan: wz range outside the grid");
    if (!chunks || !count) return fail(SMX_EINVAL, "null output");
    cudaStream_t s = (cudaStream_t)stream;
    TRY(cudaMemsetAsync(count, 0, 4, s));
    return canonical_plan(g, k, wz_lo, wz_hi, chunks, count, s);
}

int smx_bits_run_list(const smx_grid* g, uint32_t* bits_in, uint32_t* bits_out, const void* chunks,
                      const uint32_t* count, void* stream) {
    smx::Geom k;
    if (int rc = make_geom(g, &k, true)) return rc;
    int32_t ex = SMX_EXEC_BITS;
    if (int rc = ca_validate(g, smx::tet_cells(k.side), &ex)) return rc;
    if (!smx::ca_runs_supported(int(g->rho))) return fail(SMX_EINVAL, "bits_plan: the chunk engine supports rho in {4, 8}");
    if (bits_in == bits_out) return fail(SMX_EINVAL, "bits_run_list: the two shadows must not alias");
    if (!chunks || !count) return fail(SMX_EINVAL, "null chunk list");
    const CUtensorMap* tm;
    if (int rc = bits_tmap(bits_in, k.side, k.rho, &tm)) return rc;
    TRY(smx::launch_ca_bits_list(k, tm, bits_in, bits_out, chunks, count, (cudaStream_t)stream));
    return SMX_OK;
}

int smx_verify_cover(const uint32_t* coverage, uint64_t ncells, int device_ptr, uint64_t* first_bad,
                     uint32_t* multiplicity, void* stream) {
    if (!first_bad) return fail(SMX_EINVAL, "null output");
    cudaStream_t s = (cudaStream_t)stream;
    const uint32_t* d = coverage;
    if (!device_ptr) {
        void* p;
        if (int rc = pool_get(0, ncells * 4, &p)) return rc;
        TRY(cudaMemcpyAsync(p, coverage, ncells * 4, cudaMemcpyHostToDevice, s));
        d = (const uint32_t*)p;
    }
    void* pfirst;
    if (int rc = pool_get(7, 8, &pfirst)) return rc;
    unsigned long long* first = (unsigned long long*)pfirst;
    const unsigned long long init = ncells;
    TRY(cudaMemcpyAsync(first, &init, 8, cudaMemcpyHostToDevice, s));
    if (ncells) smx::launch_first_defect(d, ncells, first, s);
    TRY(cudaGetLastError());
    unsigned long long h = ncells;
    TRY(cudaMemcpyAsync(&h, first, 8, cudaMemcpyDeviceToHost, s));
    TRY(cudaStreamSynchronize(s));
    *first_bad = h;
    if (multiplicity) {
        *multiplicity = 1;
        if (h < ncells) {
            if (device_ptr) TRY(cudaMemcpy(multiplicity, d + h, 4, cudaMemcpyDeviceToHost));
            else *multiplicity = coverage[h];
        }
    }
    return SMX_OK;
}

int smx_measure_grid(const smx_grid* g, int check_cover, smx_counters* counters, uint64_t* first_bad,
                     uint32_t* multiplicity, void* stream) {
    std::vector<smx::Geom> subs;
    if (int rc = sub_geoms(g, subs, true)) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    if (!check_cover) return fill_counters(g, counters, s, nullptr);
    if (!first_bad) return fail(SMX_EINVAL, "null output");
    const uint64_t ncells = cells_of(g->dims, cell_side_of(g));
    void* p;
    if (int rc = pool_get(0, ncells * 4, &p)) return rc;
    TRY(cudaMemsetAsync(p, 0, ncells * 4, s));
    if (int rc = fill_counters(g, counters, s, (uint32_t*)p)) return rc;
    return smx_verify_cover((const uint32_t*)p, ncells, 1, first_bad, multiplicity, stream);
}

int smx_make_edm_points(int64_t count, uint64_t seed, double* out_xy) {
    if (count < 0) return fail(SMX_EINVAL, "make_edm_points: count must be >= 0");
    if (count > 0 && !out_xy) return fail(SMX_EINVAL, "null output");
    // make_edm_points (simulator.hpp:333-343): one splitmix64 stream, x then y
    uint64_t st = seed;
    auto unit = [&st]() {
        uint64_t z = (st += 0x9e3779b97f4a7c15ull);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        z ^= z >> 31;
        return double(z >> 11) * 0x1.0p-53;  // splitmix64_unit (bits.hpp:92-94)
    };
    for (int64_t i = 0; i < count; ++i) {
        out_xy[2 * i] = unit();
        out_xy[2 * i + 1] = unit();
    }
    return SMX_OK;
}

int smx_edm(const smx_grid* g, const double* points_xy, int64_t npoints, double* cells, uint64_t ncells,
            int32_t exec, int device_ptr, uint32_t* coverage, smx_counters* counters, void* stream) {
    std::vector<smx::Geom> subs;
    if (int rc = sub_geoms(g, subs, false)) return rc;
    if (g->dims != 2) return fail(SMX_EINVAL, "launch_edm: 2-simplex domains only");
    if (int rc = check_cells(g, ncells)) return rc;
    if (npoints != cell_side_of(g)) return fail(SMX_EINVAL, "launch_edm: need one point per domain side unit");
    if (exec < 0 || exec == SMX_EXEC_BITS) exec = SMX_EXEC_RUNS;
    if (exec != SMX_EXEC_BLOCK && exec != SMX_EXEC_RUNS) return fail(SMX_EINVAL, "edm: unknown exec scheme");
    cudaStream_t s = (cudaStream_t)stream;
    const double* dp = points_xy;
    double* d = cells;
    uint32_t* dcov = coverage;
    if (!device_ptr) {
        void *p, *q;
        if (int rc = pool_get(1, ncells * 8, &p)) return rc;
        if (int rc = pool_get(2, size_t(npoints) * 16, &q)) return rc;
        d = (double*)p;
        TRY(cudaMemcpyAsync(q, points_xy, size_t(npoints) * 16, cudaMemcpyHostToDevice, s));
        dp = (const double*)q;
        if (coverage) {
            if (int rc = pool_get(0, ncells * 4, &p)) return rc;
            dcov = (uint32_t*)p;
            TRY(cudaMemcpyAsync(dcov, coverage, ncells * 4, cudaMemcpyHostToDevice, s));
        }
    }
    if (coverage || counters)
        if (int rc = fill_counters(g, counters, s, dcov)) return rc;
    for (const auto& k : subs) smx::launch_edm(k, dp, d, exec, s);
    TRY(cudaGetLastError());
    if (!device_ptr) {
        TRY(cudaMemcpyAsync(cells, d, ncells * 8, cudaMemcpyDeviceToHost, s));
        if (coverage) TRY(cudaMemcpyAsync(coverage, dcov, ncells * 4, cudaMemcpyDeviceToHost, s));
        TRY(cudaStreamSynchronize(s));
    }
    return SMX_OK;
}

uint64_t smx_state_hash(int32_t m, int64_t side, const void* bytes, uint64_t nbytes) {
    uint64_t h = 0xcbf29ce484222325ull;
    auto mix_u64 = [&h](uint64_t v) {
        for (int i = 0; i < 8; ++i) {
            h ^= (v >> (8 * i)) & 0xffu;
            h *= 0x100000001b3ull;
        }
    };
    mix_u64(uint64_t(m));
    mix_u64(uint64_t(side));
    const unsigned char* p = (const unsigned char*)bytes;
    for (uint64_t i = 0; i < nbytes; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ull;
    }
    return h;
}

uint64_t smx_tile_bytes(const smx_grid* g, uint64_t ntiles) {
    uint64_t r3 = uint64_t(g->rho) * uint64_t(g->rho) * uint64_t(g->rho);
    return r3 * ntiles;
}

uint64_t smx_bits_tile_bytes(const smx_grid* g, uint64_t ntiles) {
    if (!g || g->dims != 3 || !smx::ca_runs_supported(int(g->rho))) return 0;
    return ntiles * smx::bits_tile_bytes(int(g->rho));
}

int smx_bits_tiles_pack(const smx_grid* g, const uint32_t* bits, const int32_t* tiles, uint64_t ntiles, uint8_t* out,
                        void* stream) {
    smx::Geom k;
    if (int rc = make_geom(g, &k, false)) return rc;
    if (g->dims != 3 || !smx::ca_runs_supported(int(g->rho)))
        return fail(SMX_EINVAL, "bits_tiles: 3-simplex grids with rho in {4, 8}");
    smx::launch_bits_tiles_pack(k, bits, tiles, ntiles, out, (cudaStream_t)stream);
    TRY(cudaGetLastError());
    return SMX_OK;
}

int smx_bits_tiles_unpack(const smx_grid* g, uint32_t* bits, const int32_t* tiles, uint64_t ntiles,
                          const uint8_t* in, void* stream) {
    smx::Geom k;
    if (int rc = make_geom(g, &k, false)) return rc;
    if (g->dims != 3 || !smx::ca_runs_supported(int(g->rho)))
        return fail(SMX_EINVAL, "bits_tiles: 3-simplex grids with rho in {4, 8}");
    smx::launch_bits_tiles_unpack(k, bits, tiles, ntiles, in, (cudaStream_t)stream);
    TRY(cudaGetLastError());
    return SMX_OK;
}

int smx_tiles_pack(const smx_grid* g, const uint8_t* cells, const int32_t* tiles, uint64_t ntiles, uint8_t* out,
                   void* stream) {
    smx::Geom k;
    if (int rc = make_geom(g, &k, true)) return rc;
    if (g->dims != 3) return fail(SMX_EINVAL, "tiles_pack: 3-simplex only");
    smx::launch_tiles_pack(k, cells, tiles, ntiles, out, (cudaStream_t)stream);
    TRY(cudaGetLastError());
    return SMX_OK;
}

int smx_tiles_unpack(const smx_grid* g, uint8_t* cells, const int32_t* tiles, uint64_t ntiles, const uint8_t* in,
                     void* stream) {
    smx::Geom k;
    if (int rc = make_geom(g, &k, true)) return rc;
    if (g->dims != 3) return fail(SMX_EINVAL, "tiles_unpack: 3-simplex only");
    smx::launch_tiles_unpack(k, cells, tiles, ntiles, in, (cudaStream_t)stream);
    TRY(cudaGetLastError());
    return SMX_OK;
}

// ---- the sequential reference kernels (simulator.hpp:329-331, :377-386,
// :402-425) on the GPU. They have no block map; the B200 path runs them over
// an internal BB tiling of the same domain (the largest tile edge that divides
// the side, so the cover is exact), which the map-driven kernels are already
// validated on.
static int64_t tile_edge(int64_t side, std::initializer_list<int64_t> edges) {
    for (int64_t r : edges)
        if (side % r == 0) return r;
    return 1;
}

int smx_kernel_accum(uint32_t* cells, uint64_t ncells, int device_ptr, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (ncells == 0) return SMX_OK;
    uint32_t* d = cells;
    if (!device_ptr) {
        void* p;
        if (int rc = pool_get(1, ncells * 4, &p)) return rc;
        d = (uint32_t*)p;
        TRY(cudaMemcpyAsync(d, cells, ncells * 4, cudaMemcpyHostToDevice, s));
    }
    smx::launch_increment(d, ncells, s);
    TRY(cudaGetLastError());
    if (!device_ptr) {
        TRY(cudaMemcpyAsync(cells, d, ncells * 4, cudaMemcpyDeviceToHost, s));
        TRY(cudaStreamSynchronize(s));
    }
    return SMX_OK;
}

int smx_kernel_edm(const double* points_xy, int64_t npoints, double* cells, uint64_t ncells, int device_ptr,
                   void* stream) {
    if (npoints < 1) return fail(SMX_EINVAL, "simplex_grid_state: side must be >= 1");
    if (ncells != smx::tri_cells(npoints)) return fail(SMX_EINVAL, "kernel_edm: need one point per domain side unit");
    const int64_t rho = tile_edge(npoints, {16, 8, 4, 2});
    smx_grid g;
    if (int rc = smx_make_grid(SMX_BB, 2, npoints / rho, rho, 1, &g)) return rc;
    return smx_edm(&g, points_xy, npoints, cells, ncells, SMX_EXEC_RUNS, device_ptr, nullptr, nullptr, stream);
}

int smx_kernel_ca_run(int32_t m, int64_t side, uint8_t* cells, uint64_t ncells, int64_t steps, int device_ptr,
                      void* stream) {
    if (m != 2 && m != 3) return fail(SMX_EINVAL, "simplex_grid_state: m must be 2 or 3");
    if (side < 1) return fail(SMX_EINVAL, "simplex_grid_state: side must be >= 1");
    if (steps < 0) return fail(SMX_EINVAL, "kernel_ca_run: steps must be >= 0");
    if (ncells != cells_of(m, side)) return fail(SMX_EINVAL, "kernel_ca_run: state does not match the side");
    int64_t rho;
    int32_t exec;
    if (m == 3) {
        // the bit-shadow engine where a rho in {8, 4} tiles the side, else the
        // one-thread-per-cell block scheme with the largest tile that does
        rho = tile_edge(side, {8, 4});
        exec = side % rho == 0 && (rho == 8 || rho == 4) ? SMX_EXEC_BITS : SMX_EXEC_BLOCK;
        if (exec == SMX_EXEC_BLOCK) rho = tile_edge(side, {7, 6, 5, 3, 2});
    } else {
        rho = tile_edge(side, {16, 8, 4, 2});
        exec = SMX_EXEC_RUNS;
    }
    smx_grid g;
    if (int rc = smx_make_grid(SMX_BB, m, side / rho, rho, 1, &g)) return rc;
    return smx_ca(&g, cells, ncells, steps, exec, device_ptr, nullptr, nullptr, nullptr, stream);
}

int smx_ca_multi(const smx_grid* g, uint8_t* cells, uint64_t ncells, int64_t steps, const int32_t* devices,
                 int32_t ndev, int device_ptr, smx_counters* counters, void* stream) {
    smx::Geom k;
    if (int rc = make_geom(g, &k, true)) return rc;
    int32_t ex = SMX_EXEC_BITS;
    if (int rc = ca_validate(g, ncells, &ex)) return rc;
    if (g->dims != 3) return fail(SMX_EINVAL, "launch_ca: the multi-GPU engine shards 3-simplex grids");
    if (!smx::ca_runs_supported(int(g->rho))) return fail(SMX_EINVAL, "launch_ca: the multi-GPU engine supports rho in {4, 8}");
    if (steps < 0) return fail(SMX_EINVAL, "launch_ca: steps must be >= 0");
    if (steps > INT32_MAX) return fail(SMX_ERANGE, "launch_ca: steps must fit int32");
    if (ndev < 1) return fail(SMX_EINVAL, "launch_ca: ngpus must be >= 1");
    int count = 0;
    TRY(cudaGetDeviceCount(&count));
    std::vector<int> devs;
    for (int i = 0; i < ndev; ++i) {
        const int d = devices ? devices[i] : i;
        if (d < 0 || d >= count) return fail(SMX_EINVAL, "launch_ca: device ordinal " + std::to_string(d) + " not present");
        devs.push_back(d);
    }
    if (ndev > int(g->extents[2])) return fail(SMX_EINVAL, "launch_ca: more shards than grid layers (wz)");
    if (ndev > 32767) return fail(SMX_EINVAL, "launch_ca: too many shards");
    return ca_multi(g, devs, cells, ncells, steps, device_ptr, counters, (cudaStream_t)stream);
}

int smx_release(void) {
    int dev = 0;
    TRY(cudaGetDevice(&dev));  // a valid runtime before freeing
    release_thread(std::this_thread::get_id());
    return SMX_OK;
}

uint64_t smx_scratch_bytes(void) {
    std::lock_guard<std::mutex> lk(g_mu);
    uint64_t b = 0;
    for (auto& kv : g_res) {
        if (kv.first.second != std::this_thread::get_id()) continue;
        for (int i = 0; i < 12; ++i) b += kv.second.pool_bytes[i];
    }
    return b;
}

int smx_device_sync(void) {
    TRY(cudaDeviceSynchronize());
    return SMX_OK;
}

}  // extern "C"
