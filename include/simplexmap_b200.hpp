// simplexmap_b200.hpp — C++ drop-in for the hot path of the reference
// `simplexmap` API (arXiv 2208.11617 reference, /root/reference/proj/include/
// simplexmap/{core,maps,simulator,report}.hpp), backed by the sm_100a kernels
// through the C ABI in smx_b200.h (link libsmx_b200.so).
//
// Same names, argument meaning and exceptions as the reference for the
// functions on the path: grid_bb / grid_h2d / grid_h3d / make_grid,
// map_bb / map_h2d / map_h3d, simplex_grid_state<T> (+hash), launch_map,
// launch_accum, launch_ca (dead3d), make_life_state, verify_exact_cover; and
// the general-n / comparison 2-D maps: grid_rb,
// grid_lambda, grid_h2d_padded, grid_trapezoids, decompose_trapezoids,
// map_rb_2d, map_lambda_2d, map_h2d_padded, map_h2d_trapezoid.
// Out of scope (not declared here): EDM, the 2-D periodic CA, analysis,
// reports, rendering.
//
// Switching from the reference: include this header instead of
// <simplexmap/simulator.hpp> and define SMX_B200_AS_SIMPLEXMAP to get the
// `simplexmap` namespace name.
#pragma once

#include <array>
#include <cstdint>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "smx_b200.h"
#include "smx_maps.hpp"

namespace simplexmap_b200 {

using u8 = std::uint8_t;
using u32 = std::uint32_t;
using u64 = std::uint64_t;
using i64 = std::int64_t;
using i128 = __int128;

inline void check(int rc) {
    if (rc == SMX_OK) return;
    const std::string msg = smx_last_error();
    if (rc == SMX_EINVAL) throw std::invalid_argument(msg);
    if (rc == SMX_ERANGE) throw std::overflow_error(msg);
    throw std::runtime_error("smx: " + msg);
}

// ---- geometry (core.hpp:28-69, :125-149) ----
enum class orientation { origin_orthogonal_corner };

struct simplex_spec {
    int m = 2;
    i64 n = 1;
    orientation orient = orientation::origin_orthogonal_corner;
    simplex_spec() = default;
    simplex_spec(int m_, i64 n_) : m(m_), n(n_) {
        if (m < 1) throw std::invalid_argument("simplex_spec: m must be >= 1");
        if (n < 0) throw std::invalid_argument("simplex_spec: n must be >= 0");
    }
};

struct data_coord {
    i64 x = 0, y = 0, z = 0;
    bool operator==(const data_coord&) const = default;
};
using block_coord = data_coord;

inline bool tri_contains(i64 side, i64 x, i64 y) { return smx::tri_contains<i64>(side, x, y); }
inline bool tet_contains(i64 side, i64 x, i64 y, i64 z) { return smx::tet_contains<i64>(side, x, y, z); }
inline u64 tri_cells(i64 side) { return smx::tri_cells(side); }
inline u64 tet_cells(i64 side) { return smx::tet_cells(side); }
inline u64 tri_linear_index(i64 x, i64 y) { return smx::tri_index(x, y); }
inline u64 tet_layer_prefix(i64 side, i64 z) { return smx::tet_layer_prefix(side, z); }
inline u64 tet_linear_index(i64 side, i64 x, i64 y, i64 z) { return smx::tet_index(side, x, y, z); }

// exact rational for sim_report::space_overhead (rational.hpp, reduced form)
struct rational {
    i128 num = 0, den = 1;
    rational() = default;
    rational(i128 n, i128 d = 1) : num(n), den(d) {
        if (den == 0) throw std::invalid_argument("rational: zero denominator");
        if (den < 0) num = -num, den = -den;
        i128 a = num < 0 ? -num : num, b = den;
        while (b) { i128 t = a % b; a = b; b = t; }
        if (a > 1) num /= a, den /= a;
    }
    bool operator==(const rational& o) const { return num == o.num && den == o.den; }
};

// ---- maps (maps.hpp:19-92, :96-116, :188-207, :285-337) ----
enum class map_kind { bb, rb, lambda2d, h2d, h2d_trapezoid, h2d_padded, h3d };

inline bool strict_view(map_kind k) {
    return k == map_kind::h2d || k == map_kind::h2d_padded || k == map_kind::h2d_trapezoid || k == map_kind::h3d;
}

struct map_outcome {
    bool is_void = false;
    data_coord target{};
    i64 level_b = 1;
    i64 index_q = 0;
    static map_outcome void_block() { return {true, {}, 1, 0}; }
};

// trapezoid_params (maps.hpp:49-60)
struct trapezoid_params {
    i64 delta_x = 0, delta_y = 0;
    i64 band = 0;
    i64 h1 = 0, h2 = 0;
    i64 grid_width = 0;
    i64 valid_side = 0;
    i64 ext_x = 0, ext_y = 0;
    u64 blocks() const { return u64(ext_x) * u64(ext_y); }
};

// decompose_trapezoids (maps.hpp:228-257)
inline std::vector<trapezoid_params> decompose_trapezoids(i64 n, i64 T) {
    smx_trapezoid t[64];
    int32_t c = 0;
    check(smx_decompose_trapezoids(n, T, t, 64, &c));
    std::vector<trapezoid_params> out;
    for (int i = 0; i < c; ++i)
        out.push_back({t[i].delta_x, t[i].delta_y, t[i].band, t[i].h1, t[i].h2, t[i].grid_width, t[i].valid_side,
                       t[i].ext_x, t[i].ext_y});
    return out;
}

struct grid_spec {
    map_kind kind = map_kind::bb;
    int dims = 2;
    i64 n = 1;
    i64 rho = 1;
    std::array<i64, 3> extents{1, 1, 1};
    i64 threshold = 1;
    std::vector<trapezoid_params> traps;

    u64 blocks() const {
        if (kind == map_kind::h2d_trapezoid) {
            u64 t = 0;
            for (const auto& b : traps) t += b.blocks();
            return t;
        }
        u64 t = 1;
        for (int a = 0; a < dims; ++a) t *= u64(extents[std::size_t(a)]);
        return t;
    }
    u64 threads() const {
        u64 per = 1;
        for (int a = 0; a < dims; ++a) per *= u64(rho);
        return blocks() * per;
    }
    i64 domain_side() const { return strict_view(kind) ? n - 1 : n; }

    smx_grid raw() const {
        smx_grid g{};
        g.kind = int32_t(kind);
        g.dims = dims;
        g.n = n;
        g.rho = rho;
        g.threshold = threshold;
        for (int a = 0; a < 3; ++a) g.extents[a] = extents[std::size_t(a)];
        return g;
    }
};

inline grid_spec from_raw(const smx_grid& r) {
    grid_spec g;
    g.kind = map_kind(r.kind);
    g.dims = r.dims;
    g.n = r.n;
    g.rho = r.rho;
    g.threshold = r.threshold;
    g.extents = {r.extents[0], r.extents[1], r.extents[2]};
    if (g.kind == map_kind::h2d_trapezoid) g.traps = decompose_trapezoids(g.n, g.threshold);
    return g;
}

// make_grid (report.hpp:48-66)
inline grid_spec make_grid(map_kind k, int m, i64 n, i64 rho = 1, i64 threshold = 1) {
    smx_grid r;
    check(smx_make_grid(int32_t(k), m, n, rho, threshold, &r));
    return from_raw(r);
}
inline grid_spec grid_bb(i64 n, int m) {
    if (m != 2 && m != 3) throw std::invalid_argument("grid_bb: m must be 2 or 3");
    return make_grid(map_kind::bb, m, n);
}
inline grid_spec grid_h2d(i64 n) { return make_grid(map_kind::h2d, 2, n); }
inline grid_spec grid_h3d(i64 n) { return make_grid(map_kind::h3d, 3, n); }
// self_similar_params (analysis.hpp:21-33): the executable H maps are the
// halving family; the r/beta overload accepts (1/r, beta) = (2, 2) only
// (SURVEY 8(b)); the analysis itself is paper_2208_11617_b200/analysis.py.
struct self_similar_params {
    i64 inv_r = 2, beta = 2;
    int m = 2;
    self_similar_params() = default;
    self_similar_params(i64 inv_r_, i64 beta_, int m_) : inv_r(inv_r_), beta(beta_), m(m_) {
        if (m < 1) throw std::invalid_argument("self_similar_params: m must be >= 1");
        if (beta <= 1) throw std::invalid_argument("self_similar_params: beta must be > 1");
        if (inv_r < beta) throw std::invalid_argument("self_similar_params: 1/r must be >= beta");
    }
};
inline grid_spec grid_h3d(i64 n, const self_similar_params& p) {
    if (p.inv_r != 2 || p.beta != 2)
        throw std::invalid_argument("map_h3d: the executable map is the halving family (1/r, beta) = (2, 2)");
    return grid_h3d(n);
}
inline grid_spec grid_rb(i64 n) { return make_grid(map_kind::rb, 2, n); }
inline grid_spec grid_lambda(i64 n) { return make_grid(map_kind::lambda2d, 2, n); }
inline grid_spec grid_h2d_padded(i64 n) { return make_grid(map_kind::h2d_padded, 2, n); }
inline grid_spec grid_trapezoids(i64 n, i64 T) { return make_grid(map_kind::h2d_trapezoid, 2, n, 1, T); }

inline map_outcome map_one(map_kind k, int m, i64 n, block_coord w) {
    smx_outcome o;
    check(smx_map_one(int32_t(k), m, n, w.x, w.y, w.z, &o));
    return {o.is_void != 0, {o.x, o.y, o.z}, o.level_b, o.index_q};
}
inline map_outcome map_bb(block_coord omega, i64 n, int m) { return map_one(map_kind::bb, m, n, omega); }
inline map_outcome map_h2d(block_coord omega) { return map_one(map_kind::h2d, 2, 0, omega); }
inline map_outcome map_h3d(block_coord omega, i64 n) { return map_one(map_kind::h3d, 3, n, omega); }
inline data_coord map_rb_2d(block_coord omega, i64 n) { return map_one(map_kind::rb, 2, n, omega).target; }
inline data_coord map_lambda_2d(u64 index, i64 n) {
    return map_one(map_kind::lambda2d, 2, n, {i64(index), 0, 0}).target;
}
inline map_outcome map_h2d_padded(block_coord omega, i64 n) { return map_one(map_kind::h2d_padded, 2, n, omega); }
// The reference takes the band's params; the ABI recomputes the band from
// (n, T, band index) — pass the params decompose_trapezoids returned.
inline map_outcome map_h2d_trapezoid(block_coord omega, const trapezoid_params& p) {
    if (omega.x < 0 || omega.x >= p.ext_x || omega.y < 0 || omega.y >= p.ext_y)
        throw std::invalid_argument("map_h2d_trapezoid: omega outside the trapezoid grid");
    const smx::trapezoid<i64> t{p.delta_x, p.delta_y, p.band, p.h1, p.h2, p.grid_width, p.valid_side, p.ext_x,
                                p.ext_y};
    const smx::outcome<i64> o = smx::map_h2d_trapezoid<i64>(omega.x, omega.y, t);
    return {o.is_void != 0, {o.x, o.y, o.z}, o.level_b, o.index_q};
}

// ---- simulator (simulator.hpp:37-96, :257-478) ----
enum class ca_boundary { periodic2d, dead3d };

template <class T>
struct simplex_grid_state {
    int m = 2;
    i64 side = 1;
    std::vector<T> cells;

    simplex_grid_state(int m_, i64 side_) : m(m_), side(side_) {
        if (m != 2 && m != 3) throw std::invalid_argument("simplex_grid_state: m must be 2 or 3");
        if (side < 1) throw std::invalid_argument("simplex_grid_state: side must be >= 1");
        cells.assign(std::size_t(m == 2 ? tri_cells(side) : tet_cells(side)), T{});
    }
    u64 index(i64 x, i64 y) const {
        if (m != 2 || !tri_contains(side, x, y))
            throw std::invalid_argument("simplex_grid_state: coordinate outside domain");
        return tri_linear_index(x, y);
    }
    u64 index(i64 x, i64 y, i64 z) const {
        if (m != 3 || !tet_contains(side, x, y, z))
            throw std::invalid_argument("simplex_grid_state: coordinate outside domain");
        return tet_linear_index(side, x, y, z);
    }
    T& at(i64 x, i64 y) { return cells[index(x, y)]; }
    const T& at(i64 x, i64 y) const { return cells[index(x, y)]; }
    T& at(i64 x, i64 y, i64 z) { return cells[index(x, y, z)]; }
    const T& at(i64 x, i64 y, i64 z) const { return cells[index(x, y, z)]; }
    u64 hash() const { return smx_state_hash(m, side, cells.data(), cells.size() * sizeof(T)); }
};

struct sim_report {
    int m = 2;
    i64 cell_side = 0;
    u64 blocks_launched = 0, blocks_void = 0, threads_launched = 0, threads_useful = 0;
    rational space_overhead;
    std::vector<u32> coverage;
    bool coverage_recorded = true;
    u64 state_hash = 0;
    u64 seed = 0;
};

struct launch_opts {
    u64 seed = 0;
    i64 steps = 50;
    ca_boundary boundary = ca_boundary::periodic2d;
    bool record_coverage = true;
    u64 block_order_salt = 0;      // accepted; the GPU block scheduler picks the order
    int exec = SMX_EXEC_AUTO;      // B200 extension: SMX_EXEC_BLOCK / SMX_EXEC_RUNS
};

struct cover_verdict {
    bool exact = true;
    data_coord witness{};
    u64 multiplicity = 0;
};

inline void validate_launch(const grid_spec& g, const simplex_spec& domain) {
    if (domain.m != g.dims) throw std::invalid_argument("launch: grid and domain dimensions differ");
    if (domain.n != g.domain_side() * g.rho - 1)
        throw std::invalid_argument("launch: domain side does not match grid * rho");
    if (g.rho < 1) throw std::invalid_argument("launch: rho must be >= 1");
}

namespace detail {
inline sim_report make_report(const grid_spec& g, const launch_opts& o) {
    sim_report rep;
    rep.m = g.dims;
    rep.cell_side = g.domain_side() * g.rho;
    rep.coverage_recorded = o.record_coverage;
    if (o.record_coverage)
        rep.coverage.assign(std::size_t(g.dims == 2 ? tri_cells(rep.cell_side) : tet_cells(rep.cell_side)), 0);
    rep.seed = o.seed;
    return rep;
}
inline void finish(sim_report& rep, const smx_counters& c) {
    rep.blocks_launched = c.blocks_launched;
    rep.blocks_void = c.blocks_void;
    rep.threads_launched = c.threads_launched;
    rep.threads_useful = c.threads_useful;
    if (rep.threads_useful > 0)
        rep.space_overhead = rational(i128(rep.threads_launched) - i128(rep.threads_useful), i128(rep.threads_useful));
}
}  // namespace detail

inline sim_report launch_map(const grid_spec& g, const simplex_spec& domain, const launch_opts& opts = {}) {
    validate_launch(g, domain);
    sim_report rep = detail::make_report(g, opts);
    smx_grid r = g.raw();
    smx_counters c{};
    check(smx_launch_map(&r, rep.coverage_recorded ? rep.coverage.data() : nullptr, rep.coverage.size(), 0, &c,
                         nullptr));
    detail::finish(rep, c);
    return rep;
}

inline sim_report launch_accum(const grid_spec& g, const simplex_spec& domain, simplex_grid_state<u32>& state,
                               const launch_opts& opts = {}) {
    validate_launch(g, domain);
    if (state.m != g.dims || state.side != g.domain_side() * g.rho)
        throw std::invalid_argument("launch: state does not match the domain");
    sim_report rep = detail::make_report(g, opts);
    smx_grid r = g.raw();
    smx_counters c{};
    check(smx_accum(&r, state.cells.data(), state.cells.size(), 1, opts.exec, 0,
                    rep.coverage_recorded ? rep.coverage.data() : nullptr, &c, nullptr));
    detail::finish(rep, c);
    rep.state_hash = state.hash();
    return rep;
}

inline simplex_grid_state<u8> make_life_state(int m, i64 side, u64 seed) {
    simplex_grid_state<u8> s(m, side);
    check(smx_life_init(m, side, seed, s.cells.data(), s.cells.size(), 0, nullptr));
    return s;
}

inline sim_report launch_ca(const grid_spec& g, const simplex_spec& domain, simplex_grid_state<u8>& state,
                            const launch_opts& opts = {}) {
    validate_launch(g, domain);
    if (state.m != g.dims || state.side != g.domain_side() * g.rho)
        throw std::invalid_argument("launch: state does not match the domain");
    if ((opts.boundary == ca_boundary::periodic2d) != (g.dims == 2))
        throw std::invalid_argument("launch_ca: boundary rule does not fit the domain");
    sim_report rep = detail::make_report(g, opts);
    smx_grid r = g.raw();
    smx_counters c{};
    const bool any = opts.steps > 0;
    check(smx_ca(&r, state.cells.data(), state.cells.size(), opts.steps, opts.exec, 0, nullptr,
                 any && rep.coverage_recorded ? rep.coverage.data() : nullptr, any ? &c : nullptr, nullptr));
    if (any) detail::finish(rep, c);
    rep.state_hash = state.hash();
    return rep;
}

// verify_exact_cover (simulator.hpp:467-478): first cell of multiplicity != 1
inline cover_verdict verify_exact_cover(const sim_report& rep, const simplex_spec& domain) {
    if (domain.m != rep.m || domain.n != rep.cell_side - 1)
        throw std::invalid_argument("verify_exact_cover: report/domain mismatch");
    if (!rep.coverage_recorded) throw std::invalid_argument("verify_exact_cover: report has no coverage");
    for (u64 i = 0; i < rep.coverage.size(); ++i) {
        if (rep.coverage[i] == 1) continue;
        i64 z = 0;
        u64 rem = i;
        if (rep.m == 3) {
            while (z + 1 < rep.cell_side && tet_layer_prefix(rep.cell_side, z + 1) <= i) ++z;
            rem = i - tet_layer_prefix(rep.cell_side, z);
        }
        i64 y = 0;
        while (tri_linear_index(0, y + 1) <= rem) ++y;
        return {false, {i64(rem - tri_linear_index(0, y)), y, z}, rep.coverage[i]};
    }
    return {};
}

}  // namespace simplexmap_b200

#ifdef SMX_B200_AS_SIMPLEXMAP
namespace simplexmap = simplexmap_b200;
#endif
