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
// map_rb_2d, map_lambda_2d, map_h2d_padded, map_h2d_trapezoid; the EDM and
// 2-D periodic Life kernels (make_edm_points, launch_edm, launch_ca m=2); and
// the report layer (report.hpp: measure_grid, verify_sweep, analyze_sweep,
// parse_n_range, csv_measure / csv_analyze / csv_simulate, text_report).
// Out of scope (not declared here): the r/beta analysis (Python:
// paper_2208_11617_b200.analysis), rendering.
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
    bool operator!=(const rational& o) const { return !(*this == o); }

    static std::string int_text(i128 v) {
        if (v == 0) return "0";
        const bool neg = v < 0;
        unsigned __int128 u = neg ? (unsigned __int128)(-(v + 1)) + 1 : (unsigned __int128)v;
        std::string d;
        while (u) d.insert(d.begin(), char('0' + int(u % 10))), u /= 10;
        return neg ? "-" + d : d;
    }
    // rational.hpp:123-126
    std::string to_string() const { return den == 1 ? int_text(num) : int_text(num) + "/" + int_text(den); }
    // rational.hpp:129-144: fixed point, round half up on the magnitude
    std::string to_decimal_string(int digits = 6) const {
        unsigned __int128 mag = num < 0 ? (unsigned __int128)(-num) : (unsigned __int128)num, scale = 1;
        for (int i = 0; i < digits; ++i) scale *= 10;
        const unsigned __int128 d = (unsigned __int128)den;
        unsigned __int128 q = mag / d * scale, r = mag % d;
        q += r * scale / d;
        if ((r * scale % d) * 2 >= d) q += 1;
        std::string out = (num < 0 && q != 0) ? "-" : "";
        out += int_text(i128(q / scale));
        if (digits > 0) {
            std::string f = int_text(i128(q % scale));
            out += "." + std::string(std::size_t(digits) - f.size(), '0') + f;
        }
        return out;
    }
};

// ---- maps (maps.hpp:19-92, :96-116, :188-207, :285-337) ----
enum class map_kind { bb, rb, lambda2d, h2d, h2d_trapezoid, h2d_padded, h3d };

inline const char* map_kind_name(map_kind k) {
    switch (k) {
        case map_kind::bb: return "bb";
        case map_kind::rb: return "rb";
        case map_kind::lambda2d: return "lambda";
        case map_kind::h2d: return "h2d";
        case map_kind::h2d_trapezoid: return "trapezoid";
        case map_kind::h2d_padded: return "h2d-padded";
        case map_kind::h3d: return "h3d";
    }
    return "?";
}

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
enum class kernel_kind { map, accum, edm, ca_life };
enum class ca_boundary { periodic2d, dead3d };

inline const char* kernel_kind_name(kernel_kind k) {
    switch (k) {
        case kernel_kind::map: return "map";
        case kernel_kind::accum: return "accum";
        case kernel_kind::edm: return "edm";
        case kernel_kind::ca_life: return "ca";
    }
    return "?";
}

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

// make_edm_points (simulator.hpp:333-343): seeded splitmix64 points in [0,1)^2
inline std::vector<std::array<double, 2>> make_edm_points(i64 count, u64 seed) {
    if (count < 0) throw std::invalid_argument("make_edm_points: count must be >= 0");
    std::vector<std::array<double, 2>> pts(static_cast<std::size_t>(count));
    if (count) check(smx_make_edm_points(count, seed, pts.front().data()));
    return pts;
}

// launch_edm (simulator.hpp:352-372): cell (x, y) = |p_x - p_y| in f64, bit-identical
// to the reference's edm_distance
inline sim_report launch_edm(const grid_spec& g, const simplex_spec& domain,
                             const std::vector<std::array<double, 2>>& points, simplex_grid_state<double>& state,
                             const launch_opts& opts = {}) {
    validate_launch(g, domain);
    if (g.dims != 2) throw std::invalid_argument("launch_edm: 2-simplex domains only");
    if (state.m != 2 || state.side != g.domain_side() * g.rho)
        throw std::invalid_argument("launch: state does not match the domain");
    if (i64(points.size()) != state.side)
        throw std::invalid_argument("launch_edm: need one point per domain side unit");
    sim_report rep = detail::make_report(g, opts);
    smx_grid r = g.raw();
    smx_counters c{};
    check(smx_edm(&r, points.front().data(), i64(points.size()), state.cells.data(), state.cells.size(), opts.exec,
                  0, rep.coverage_recorded ? rep.coverage.data() : nullptr, &c, nullptr));
    detail::finish(rep, c);
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

// ---- report layer (report.hpp) ----
constexpr const char* csv_schema_measure = "slx-1";
constexpr const char* csv_schema_simulate = "slx-sim-1";
constexpr const char* csv_schema_analyze = "slx-an-1";
constexpr const char* csv_measure_columns =
    "map,m,n,rho,blocks_launched,blocks_void,threads_launched,threads_useful,overhead_num,overhead_den,"
    "overhead_decimal";

// report.hpp:158-171
struct measure_row {
    map_kind kind = map_kind::bb;
    int m = 2;
    i64 n = 1;
    i64 rho = 1;
    u64 blocks_launched = 0, blocks_void = 0, threads_launched = 0, threads_useful = 0;
    rational overhead;
    bool exact = false;
    data_coord witness{};
    u64 multiplicity = 0;
};

// report.hpp:173-186
inline measure_row row_from_report(const grid_spec& g, const sim_report& rep) {
    measure_row row;
    row.kind = g.kind;
    row.m = g.dims;
    row.n = g.n;
    row.rho = g.rho;
    row.blocks_launched = rep.blocks_launched;
    row.blocks_void = rep.blocks_void;
    row.threads_launched = rep.threads_launched;
    row.threads_useful = rep.threads_useful;
    row.overhead = rep.space_overhead;
    return row;
}

// report.hpp:190-203: one map-kernel launch on the GPU; the coverage multiset
// is reduced to the first non-1 cell on the device (smx_verify_cover), so only
// the verdict crosses PCIe.
inline measure_row measure_grid(const grid_spec& g, bool check_cover = true) {
    const simplex_spec dom(g.dims, g.domain_side() * g.rho - 1);
    validate_launch(g, dom);
    const i64 side = dom.n + 1;
    const u64 cells = g.dims == 2 ? tri_cells(side) : tet_cells(side);
    smx_grid r = g.raw();
    smx_counters c{};
    u64 first = cells;
    u32 mult = 0;
    check(smx_measure_grid(&r, check_cover ? 1 : 0, &c, &first, &mult, nullptr));
    sim_report rep;
    rep.m = g.dims;
    rep.cell_side = side;
    detail::finish(rep, c);
    measure_row row = row_from_report(g, rep);
    if (check_cover) {
        row.exact = first == cells;
        if (!row.exact) {
            u64 rem = first;
            i64 z = 0;
            if (g.dims == 3) {
                while (z + 1 < side && tet_layer_prefix(side, z + 1) <= first) ++z;
                rem = first - tet_layer_prefix(side, z);
            }
            i64 y = 0;
            while (tri_linear_index(0, y + 1) <= rem) ++y;
            row.witness = {i64(rem - tri_linear_index(0, y)), y, z};
            row.multiplicity = mult;
        }
    }
    return row;
}

// report.hpp:68-110
struct n_range {
    i64 lo = 1, hi = 1;
    bool pow2_only = false;
};

inline n_range parse_n_range(const std::string& text) {
    auto parse_int = [](const std::string& s) -> i64 {
        if (s.empty() || s.find_first_not_of("0123456789") != std::string::npos)
            throw std::invalid_argument("bad n-range literal: " + s);
        return i64(std::stoll(s));
    };
    const auto dots = text.find("..");
    if (dots == std::string::npos) {
        const i64 v = parse_int(text);
        return {v, v, false};
    }
    const i64 lo = parse_int(text.substr(0, dots));
    std::string rest = text.substr(dots + 2);
    const std::string tag = "(pow2)";
    const bool pow2 = rest.size() > tag.size() && rest.compare(rest.size() - tag.size(), tag.size(), tag) == 0;
    if (pow2) rest.resize(rest.size() - tag.size());
    const i64 hi = parse_int(rest);
    if (lo < 1 || hi < lo) throw std::invalid_argument("bad n-range: " + text);
    return {lo, hi, pow2};
}

inline std::vector<i64> expand_n_range(const n_range& r) {
    std::vector<i64> out;
    if (!r.pow2_only) {
        for (i64 n = r.lo; n <= r.hi; ++n) out.push_back(n);
        return out;
    }
    for (i64 n = 1; n <= r.hi; n *= 2) {
        if (n >= r.lo) out.push_back(n);
        if (n > r.hi / 2) break;
    }
    return out;
}

// report.hpp:324-342. Rows in input order; verify_sweep caps the multiplicity
// at 255 like the reference's byte-mark walk (measure_grid_compact :287-321).
inline std::vector<measure_row> verify_sweep(map_kind k, int m, const std::vector<i64>& ns, i64 rho = 1,
                                             i64 threshold = 1) {
    std::vector<measure_row> rows;
    rows.reserve(ns.size());
    for (i64 n : ns) {
        measure_row row = measure_grid(make_grid(k, m, n, rho, threshold), true);
        if (row.multiplicity > 255) row.multiplicity = 255;
        rows.push_back(row);
    }
    return rows;
}

inline std::vector<measure_row> analyze_sweep(map_kind k, int m, const std::vector<i64>& ns, i64 rho = 1,
                                              i64 threshold = 1) {
    std::vector<measure_row> rows;
    rows.reserve(ns.size());
    for (i64 n : ns) rows.push_back(measure_grid(make_grid(k, m, n, rho, threshold), false));
    return rows;
}

// report.hpp:345-352 (bb: m! - 1, core.hpp:125-128)
inline rational scheme_overhead_limit(map_kind k, int m) {
    switch (k) {
        case map_kind::bb: {
            i128 f = 1;
            for (int i = 2; i <= m; ++i) f *= i;
            return rational(f - 1);
        }
        case map_kind::h2d_padded: return rational(3);
        case map_kind::h3d: return rational(1, 8);
        default: return rational(0);
    }
}

namespace detail {
inline std::string csv_rational(const rational& r) {
    return rational::int_text(r.num) + "," + rational::int_text(r.den) + "," + r.to_decimal_string(9);
}
inline std::string csv_fields(const measure_row& r) {
    return std::string(map_kind_name(r.kind)) + "," + std::to_string(r.m) + "," + std::to_string(r.n) + "," +
           std::to_string(r.rho) + "," + std::to_string(r.blocks_launched) + "," + std::to_string(r.blocks_void) +
           "," + std::to_string(r.threads_launched) + "," + std::to_string(r.threads_useful) + "," +
           csv_rational(r.overhead);
}
}  // namespace detail

// report.hpp:386-446
inline std::string csv_measure(const std::vector<measure_row>& rows) {
    std::string out = std::string("schema,") + csv_measure_columns + "\n";
    for (const auto& r : rows) out += std::string(csv_schema_measure) + "," + detail::csv_fields(r) + "\n";
    return out;
}

inline std::string csv_analyze(const std::vector<measure_row>& rows) {
    std::string out = std::string("schema,") + csv_measure_columns + ",limit_num,limit_den,limit_decimal\n";
    for (const auto& r : rows)
        out += std::string(csv_schema_analyze) + "," + detail::csv_fields(r) + "," +
               detail::csv_rational(scheme_overhead_limit(r.kind, r.m)) + "\n";
    return out;
}

struct simulate_row {
    measure_row base;
    kernel_kind kernel = kernel_kind::map;
    i64 steps = 0;
    u64 seed = 0;
    u64 state_hash = 0;
};

inline std::string csv_simulate(const std::vector<simulate_row>& rows) {
    std::string out = std::string("schema,") + csv_measure_columns + ",kernel,steps,seed,state_hash\n";
    for (const auto& r : rows)
        out += std::string(csv_schema_simulate) + "," + detail::csv_fields(r.base) + "," +
               kernel_kind_name(r.kernel) + "," + std::to_string(r.steps) + "," + std::to_string(r.seed) + "," +
               std::to_string(r.state_hash) + "\n";
    return out;
}

// report.hpp:475-480
inline std::string witness_text(const measure_row& r) {
    std::string out = "(" + std::to_string(r.witness.x) + "," + std::to_string(r.witness.y);
    if (r.m == 3) out += "," + std::to_string(r.witness.z);
    return out + ")";
}

// report.hpp:483-511: one line per row
inline std::string text_report(const std::vector<measure_row>& rows, bool verified) {
    std::string out;
    for (const auto& r : rows) {
        out += std::string("map=") + map_kind_name(r.kind) + " m=" + std::to_string(r.m) +
               " n=" + std::to_string(r.n) + " rho=" + std::to_string(r.rho) +
               " blocks=" + std::to_string(r.blocks_launched) + " void=" + std::to_string(r.blocks_void) +
               " threads=" + std::to_string(r.threads_launched) + " useful=" + std::to_string(r.threads_useful) +
               " overhead=" + r.overhead.to_string() + " (" + r.overhead.to_decimal_string(6) + ")";
        if (verified)
            out += r.exact ? std::string(" Exact")
                           : " NotExact witness=" + witness_text(r) + " mult=" + std::to_string(r.multiplicity);
        out += '\n';
    }
    return out;
}

}  // namespace simplexmap_b200

#ifdef SMX_B200_AS_SIMPLEXMAP
namespace simplexmap = simplexmap_b200;
#endif
