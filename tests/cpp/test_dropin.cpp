// The C++ drop-in (include/simplexmap_b200.hpp) exercised the way the
// reference's own suites exercise simplexmap (test_maps.cpp, test_simulator.cpp,
// acceptance.cpp) on the hot-path functions. `--host`: map / grid / contract
// checks (no GPU); `--gpu`: launches through libsmx_b200.so on cuda:0.
#define SMX_B200_AS_SIMPLEXMAP
#include "simplexmap_b200.hpp"

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <cmath>
#include <functional>

using namespace simplexmap;

static int g_fail = 0, g_pass = 0;
#define CHECK(c)                                                              \
    do {                                                                      \
        if (c) ++g_pass;                                                      \
        else { ++g_fail; std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); } \
    } while (0)
#define CHECK_THROWS_AS(expr, E)                                              \
    do {                                                                      \
        bool _t = false;                                                      \
        try { (void)(expr); } catch (const E&) { _t = true; } catch (...) {}  \
        CHECK(_t && #E);                                                      \
    } while (0)

static simplex_spec domain_of(const grid_spec& g) { return {g.dims, g.domain_side() * g.rho - 1}; }

// strict-view cover of T(n - 1) (test_maps.cpp strict_cover2)
struct strict_cover2 {
    i64 n;
    std::vector<u32> marks;
    u64 total = 0, voids = 0;
    bool outside = false;
    explicit strict_cover2(i64 n_) : n(n_), marks(std::size_t(tri_cells(n_ - 1)), 0) {}
    void add(const map_outcome& o) {
        ++total;
        if (o.is_void) { ++voids; return; }
        const i64 x = o.target.x, y = o.target.y - 1;
        if (!(0 <= x && x <= y && y <= n - 2)) { outside = true; return; }
        ++marks[tri_linear_index(x, y)];
    }
    bool exact() const {
        return !outside && std::all_of(marks.begin(), marks.end(), [](u32 v) { return v == 1; });
    }
};

static void general_n_suite() {
    // test_maps.cpp "h2d padded covers general n"
    CHECK(grid_h2d_padded(8).extents == grid_h2d(8).extents);
    CHECK((grid_h2d_padded(9).extents == std::array<i64, 3>{8, 15, 1}));
    for (i64 n : {2, 3, 5, 27, 100, 255, 257}) {
        grid_spec g = grid_h2d_padded(n);
        strict_cover2 cover(n);
        for (i64 oy = 0; oy < g.extents[1]; ++oy)
            for (i64 ox = 0; ox < g.extents[0]; ++ox) cover.add(map_h2d_padded({ox, oy, 0}, n));
        CHECK(cover.exact());
        CHECK(cover.total == g.blocks());
        CHECK(cover.total - cover.voids == u64(tri_cells(n - 1)));
    }
    {
        grid_spec g = grid_h2d_padded(257);
        double ratio = double(g.blocks()) / double(u64(tri_cells(256)));
        CHECK(ratio > 3.9 && ratio < 4.1);
    }
    // "trapezoid decomposition"
    for (i64 T : {1, 4, 16}) {
        auto traps = decompose_trapezoids(16, T);
        CHECK(traps.size() == 1);
        CHECK(traps[0].band == 16 && traps[0].h2 == 0 && traps[0].valid_side == 16);
        CHECK(traps[0].ext_x == grid_h2d(16).extents[0] && traps[0].ext_y == grid_h2d(16).extents[1]);
    }
    auto t27 = decompose_trapezoids(27, 1);
    CHECK(t27.size() == 3);
    CHECK(t27[0].delta_x == 0 && t27[0].band == 16 && t27[0].h2 == 11);
    CHECK(t27[1].delta_x == 16 && t27[1].band == 8 && t27[1].h2 == 3);
    CHECK(t27[2].delta_x == 24 && t27[2].band == 2 && t27[2].h2 == 1);
    auto t27p = decompose_trapezoids(27, 4);
    CHECK(t27p.size() == 3 && t27p[2].band == 4 && t27p[2].h2 == 0 && t27p[2].valid_side == 3);
    for (auto& t : t27) CHECK(t.h1 + t.h2 == t.ext_y - 1);
    // "trapezoid map pinned boundary blocks"
    CHECK(map_h2d_trapezoid({0, 25, 0}, t27[0]).target == (data_coord{0, 26, 0}));
    CHECK(map_h2d_trapezoid({0, 26, 0}, t27[0]).target == (data_coord{8, 16, 0}));
    CHECK_THROWS_AS(map_h2d_trapezoid({0, 37, 0}, t27[0]), std::invalid_argument);
    auto single = decompose_trapezoids(32, 1);
    CHECK(single.size() == 1);
    bool same = true;
    for (i64 oy = 0; oy < single[0].ext_y; ++oy)
        for (i64 ox = 0; ox < single[0].ext_x; ++ox)
            same = same && map_h2d_trapezoid({ox, oy, 0}, single[0]).target == map_h2d({ox, oy, 0}).target;
    CHECK(same);
    // "trapezoid union tiles every n"
    bool all_exact = true, counts = true;
    for (i64 n = 2; n <= 512; ++n)
        for (i64 T : {1, 4, 16}) {
            auto traps = decompose_trapezoids(n, T);
            counts = counts && i64(traps.size()) <= std::max<i64>(1, 64 - __builtin_clzll(u64(n - 1)));
            strict_cover2 cover(n);
            for (const auto& t : traps)
                for (i64 oy = 0; oy < t.ext_y; ++oy)
                    for (i64 ox = 0; ox < t.ext_x; ++ox) cover.add(map_h2d_trapezoid({ox, oy, 0}, t));
            all_exact = all_exact && cover.exact();
        }
    CHECK(all_exact);
    CHECK(counts);
    CHECK(grid_trapezoids(27, 1).blocks() == 8 * 37 + 4 * 13 + 1 * 3);
    // RB / lambda (maps.hpp:120-159): exact cover of T(n)
    for (i64 n : {1, 2, 3, 8, 27, 64}) {
        grid_spec g = grid_rb(n);
        std::vector<u32> marks(std::size_t(tri_cells(n)), 0);
        for (i64 oy = 0; oy < g.extents[1]; ++oy)
            for (i64 ox = 0; ox < g.extents[0]; ++ox) {
                data_coord d = map_rb_2d({ox, oy, 0}, n);
                if (tri_contains(n, d.x, d.y)) ++marks[tri_linear_index(d.x, d.y)];
            }
        u64 ones = u64(std::count(marks.begin(), marks.end(), 1u));
        CHECK(ones == tri_cells(n));
        for (u64 i = 0; i < tri_cells(n); ++i) {
            data_coord d = map_lambda_2d(i, n);
            CHECK(tri_linear_index(d.x, d.y) == i);
        }
    }
    CHECK_THROWS_AS(grid_rb(0), std::invalid_argument);
    CHECK_THROWS_AS(grid_trapezoids(1, 1), std::invalid_argument);
    CHECK_THROWS_AS(map_lambda_2d(15, 5), std::invalid_argument);
}

static void host_suite() {
    general_n_suite();
    // self_similar_params on the 3-D path (analysis.hpp:27-32)
    CHECK(grid_h3d(64, self_similar_params(2, 2, 3)).blocks() == 49152);
    CHECK_THROWS_AS(grid_h3d(64, self_similar_params(3, 3, 3)), std::invalid_argument);
    CHECK_THROWS_AS(self_similar_params(2, 3, 3), std::invalid_argument);
    // test_maps.cpp "bounding box map"
    CHECK(map_bb({1, 3, 0}, 8, 2).target == (data_coord{1, 3, 0}));
    CHECK(!map_bb({1, 3, 0}, 8, 2).is_void);
    CHECK(map_bb({7, 2, 0}, 8, 2).is_void);
    CHECK_THROWS_AS(map_bb({8, 0, 0}, 8, 2), std::invalid_argument);
    CHECK_THROWS_AS(map_bb({0, 0, 0}, 8, 4), std::invalid_argument);
    u64 useful = 0;
    for (i64 z = 0; z < 8; ++z)
        for (i64 y = 0; y < 8; ++y)
            for (i64 x = 0; x < 8; ++x) useful += !map_bb({x, y, z}, 8, 3).is_void;
    CHECK(useful == tet_cells(8));
    CHECK(grid_bb(8, 3).blocks() == 512);
    CHECK(!map_bb({0, 0, 0}, 1, 2).is_void);
    // "h2d grid shapes" / "h2d map pinned points and exact cover"
    CHECK((grid_h2d(8).extents == std::array<i64, 3>{4, 7, 1}));
    CHECK(grid_h2d(8).blocks() == 28);
    CHECK(grid_h2d(1024).blocks() == 523776);
    CHECK_THROWS_AS(grid_h2d(9), std::invalid_argument);
    CHECK_THROWS_AS(grid_h2d(1), std::invalid_argument);
    CHECK(map_h2d({0, 0, 0}).target == (data_coord{0, 1, 0}));
    CHECK(map_h2d({3, 0, 0}).target == (data_coord{6, 7, 0}));
    CHECK(map_h2d({2, 1, 0}).target == (data_coord{4, 6, 0}));
    CHECK(map_h2d({1, 2, 0}).target == (data_coord{1, 3, 0}));
    CHECK(map_h2d({2, 1, 0}).level_b == 2 && map_h2d({2, 1, 0}).index_q == 1);
    for (i64 n = 2; n <= 1024; n *= 2) {
        grid_spec g = grid_h2d(n);
        std::vector<u32> marks(std::size_t(tri_cells(n - 1)), 0);
        bool in = true;
        for (i64 oy = 0; oy < g.extents[1]; ++oy)
            for (i64 ox = 0; ox < g.extents[0]; ++ox) {
                map_outcome o = map_h2d({ox, oy, 0});
                in = in && 0 <= o.target.x && o.target.x < o.target.y && o.target.y <= n - 1;
                if (in) ++marks[tri_linear_index(o.target.x, o.target.y - 1)];
            }
        CHECK(in && std::all_of(marks.begin(), marks.end(), [](u32 v) { return v == 1; }));
    }
    // "h3d grid shapes" / "h3d map pinned points and exact cover" (void counts)
    CHECK((grid_h3d(4).extents == std::array<i64, 3>{2, 2, 3}));
    CHECK(grid_h3d(64).blocks() == 49152);
    CHECK_THROWS_AS(grid_h3d(2), std::invalid_argument);
    CHECK_THROWS_AS(grid_h3d(24), std::invalid_argument);
    CHECK(map_h3d({0, 0, 0}, 8).target == (data_coord{0, 5, 0}));
    CHECK_THROWS_AS(map_h3d({0, 0, 99}, 8), std::invalid_argument);
    const u64 voids_want[] = {2, 12, 88, 688, 5472};
    int vi = 0;
    for (i64 n : {4, 8, 16, 32, 64}) {
        grid_spec g = grid_h3d(n);
        std::vector<u32> marks(std::size_t(tet_cells(n - 1)), 0);
        u64 voids = 0;
        for (i64 oz = 0; oz < g.extents[2]; ++oz)
            for (i64 oy = 0; oy < g.extents[1]; ++oy)
                for (i64 ox = 0; ox < g.extents[0]; ++ox) {
                    map_outcome o = map_h3d({ox, oy, oz}, n);
                    if (o.is_void) { ++voids; continue; }
                    ++marks[tet_linear_index(n - 1, o.target.x, o.target.y - 1, o.target.z)];
                }
        CHECK(std::all_of(marks.begin(), marks.end(), [](u32 v) { return v == 1; }));
        CHECK(voids == voids_want[vi++]);
    }
    // make_grid contract (report.hpp:48-66)
    CHECK_THROWS_AS(make_grid(map_kind::h3d, 2, 8), std::invalid_argument);
    CHECK_THROWS_AS(make_grid(map_kind::h2d, 2, 8, 0), std::invalid_argument);
    // state accessors (test_simulator.cpp:380-391)
    simplex_grid_state<u32> s(2, 8);
    CHECK_THROWS_AS(s.at(5, 3), std::invalid_argument);
    CHECK_THROWS_AS(s.at(0, 8), std::invalid_argument);
    simplex_grid_state<u32> t(3, 8);
    CHECK_THROWS_AS(t.at(0, 4, 4), std::invalid_argument);
    CHECK(t.index(0, 4, 3) == tet_linear_index(8, 0, 4, 3));
    // launch contract (test_simulator.cpp:365-378)
    grid_spec g = grid_h2d(16);
    CHECK_THROWS_AS(launch_map(g, simplex_spec{2, 15}), std::invalid_argument);
    CHECK_THROWS_AS(launch_map(g, simplex_spec{3, 14}), std::invalid_argument);
    simplex_grid_state<u32> wrong(2, 16);
    CHECK_THROWS_AS(launch_accum(g, domain_of(g), wrong), std::invalid_argument);
}

static void gpu_suite() {
    // "launch accounting over the bounding-box grid"
    auto g = grid_bb(4, 2);
    auto rep = launch_map(g, domain_of(g));
    CHECK(rep.blocks_launched == 16 && rep.blocks_void == 6 && rep.threads_useful == 10);
    CHECK(rep.space_overhead == rational(3, 5));
    CHECK(verify_exact_cover(rep, domain_of(g)).exact);
    auto g3 = grid_bb(4, 3);
    auto rep3 = launch_map(g3, domain_of(g3));
    CHECK(rep3.space_overhead == rational(11, 5));
    // "three-dimensional cover through block expansion"
    auto gh = grid_h3d(8);
    gh.rho = 2;
    auto reph = launch_map(gh, domain_of(gh));
    CHECK(reph.threads_useful == tet_cells(14));
    CHECK(verify_exact_cover(reph, domain_of(gh)).exact);
    // "thread expansion slack sits on the diagonal tiles"
    for (i64 rho : {2, 4}) {
        auto gs = grid_h2d(64);
        gs.rho = rho;
        auto r2 = launch_map(gs, domain_of(gs));
        CHECK(r2.threads_launched - r2.threads_useful == u64(63 * rho * (rho - 1) / 2));
    }
    // "cover verdict pinpoints the first defect"
    auto gd = grid_h2d(16);
    auto rd = launch_map(gd, domain_of(gd));
    rd.coverage[tri_linear_index(2, 5)] -= 1;
    rd.coverage[tri_linear_index(3, 7)] += 1;
    auto v = verify_exact_cover(rd, domain_of(gd));
    CHECK(!v.exact && v.witness == (data_coord{2, 5, 0}) && v.multiplicity == 0);
    // acceptance criterion 3 + SURVEY Appendix A accum hashes
    for (int k = 1; k <= 10; ++k) {
        const i64 n = i64{1} << k;
        auto ga = grid_h2d(n);
        simplex_grid_state<u32> st(2, n - 1);
        launch_opts o;
        o.record_coverage = false;
        auto ra = launch_accum(ga, domain_of(ga), st, o);
        CHECK(ra.blocks_void == 0 && ra.blocks_launched == u64(n) * u64(n - 1) / 2);
        CHECK(std::all_of(st.cells.begin(), st.cells.end(), [](u32 c) { return c == 1; }));
        if (n == 1024) CHECK(ra.state_hash == 9376064259860285065ull);
    }
    {
        auto ga = grid_h2d(1024);
        ga.rho = 16;
        simplex_grid_state<u32> st(2, ga.domain_side() * ga.rho);
        launch_opts o;
        o.record_coverage = false;
        auto ra = launch_accum(ga, domain_of(ga), st, o);
        CHECK(ra.state_hash == 625406489163772878ull);
    }
    // life: "random life population is deterministic" + Appendix A 3-D hashes
    auto a = make_life_state(2, 64, 5), b = make_life_state(2, 64, 5), c = make_life_state(2, 64, 6);
    CHECK(a.cells == b.cells && a.cells != c.cells);
    struct { i64 side, steps; u64 hash; } rows[] = {{15, 64, 750086803756986311ull},
                                                    {31, 64, 11768087780779516714ull},
                                                    {63, 64, 6734372989930245576ull}};
    for (auto r : rows) {
        for (auto gc : {grid_h3d(r.side + 1), grid_bb(r.side, 3)}) {
            auto st = make_life_state(3, r.side, 42);
            launch_opts o;
            o.steps = r.steps;
            o.boundary = ca_boundary::dead3d;
            auto rc = launch_ca(gc, domain_of(gc), st, o);
            CHECK(rc.state_hash == r.hash);
            CHECK(verify_exact_cover(rc, domain_of(gc)).exact);
        }
    }
    // the x-run engine at rho = 4 / 8 agrees with the block scheme
    for (i64 rho : {4, 8}) {
        auto gc = grid_h3d(16);
        gc.rho = rho;
        auto s1 = make_life_state(3, gc.domain_side() * rho, 3), s2 = s1;
        launch_opts o;
        o.steps = 5;
        o.boundary = ca_boundary::dead3d;
        o.record_coverage = false;
        o.exec = SMX_EXEC_BLOCK;
        launch_ca(gc, domain_of(gc), s1, o);
        o.exec = SMX_EXEC_RUNS;
        launch_ca(gc, domain_of(gc), s2, o);
        CHECK(s1.cells == s2.cells);
    }
    // "launch rejects inconsistent setups"
    auto life = make_life_state(2, 15, 1);
    launch_opts bad;
    bad.boundary = ca_boundary::dead3d;
    auto g16 = grid_h2d(16);
    CHECK_THROWS_AS(launch_ca(g16, domain_of(g16), life, bad), std::invalid_argument);
}

// report layer (test_report.cpp:128-200), EDM (test_simulator.cpp:199-230),
// 2-D periodic Life
static void report_suite() {
    auto rows = verify_sweep(map_kind::bb, 2, {2, 4});
    CHECK(csv_measure(rows) ==
          "schema,map,m,n,rho,blocks_launched,blocks_void,threads_launched,threads_useful,overhead_num,"
          "overhead_den,overhead_decimal\n"
          "slx-1,bb,2,2,1,4,1,4,3,1,3,0.333333333\n"
          "slx-1,bb,2,4,1,16,6,16,10,3,5,0.600000000\n");
    CHECK(rows[0].exact && rows[1].exact);
    auto an = csv_analyze(analyze_sweep(map_kind::bb, 3, {4}));
    CHECK(an.find(",limit_num,limit_den,limit_decimal\n") != std::string::npos);
    CHECK(an.find("slx-an-1,bb,3,4,1,64,44,64,20,11,5,2.200000000,5,1,5.000000000\n") != std::string::npos);
    CHECK(csv_analyze(analyze_sweep(map_kind::h3d, 3, {16})).find(",1,8,0.125000000\n") != std::string::npos);
    CHECK(csv_analyze(analyze_sweep(map_kind::h2d, 2, {16})).find(",0,1,0.000000000,0,1,0.000000000\n") !=
          std::string::npos);
    CHECK(scheme_overhead_limit(map_kind::bb, 3) == rational(5));
    CHECK(scheme_overhead_limit(map_kind::h2d_padded, 2) == rational(3));
    CHECK(scheme_overhead_limit(map_kind::h2d_trapezoid, 2) == rational(0));
    // every map family verifies exact over a small n range
    for (i64 n : expand_n_range(parse_n_range("2..40"))) {
        CHECK(measure_grid(make_grid(map_kind::h2d_trapezoid, 2, n, 1, 4)).exact);
        CHECK(measure_grid(make_grid(map_kind::rb, 2, n)).exact);
        CHECK(measure_grid(make_grid(map_kind::lambda2d, 2, n)).exact);
        CHECK(measure_grid(make_grid(map_kind::h2d_padded, 2, n)).exact);
        CHECK(measure_grid(make_grid(map_kind::bb, 3, n)).exact);
    }
    CHECK(expand_n_range(parse_n_range("3..40(pow2)")) == (std::vector<i64>{4, 8, 16, 32}));
    CHECK_THROWS_AS(parse_n_range("5..2"), std::invalid_argument);
    // text report
    auto h = verify_sweep(map_kind::h2d, 2, {16});
    auto text = text_report(h, true);
    CHECK(text.find("map=h2d m=2 n=16 rho=1 blocks=120 void=0") != std::string::npos);
    CHECK(text.find(" Exact\n") != std::string::npos);
    measure_row bad = h[0];
    bad.exact = false;
    bad.witness = {2, 5, 0};
    bad.multiplicity = 0;
    CHECK(text_report({bad}, true).find("NotExact witness=(2,5) mult=0") != std::string::npos);
    // simulate CSV over a 2-D Life run on trapezoids
    auto run = [] {
        auto g = make_grid(map_kind::h2d_trapezoid, 2, 16, 1, 4);
        auto state = make_life_state(2, g.domain_side(), 3);
        launch_opts o;
        o.steps = 5;
        o.seed = 3;
        auto rep = launch_ca(g, domain_of(g), state, o);
        simulate_row row;
        row.base = measure_grid(g, true);
        row.kernel = kernel_kind::ca_life;
        row.steps = 5;
        row.seed = 3;
        row.state_hash = rep.state_hash;
        return csv_simulate({row});
    };
    const std::string a = run();
    CHECK(a == run());
    CHECK(a.find(",kernel,steps,seed,state_hash\n") != std::string::npos);
    CHECK(a.find("slx-sim-1,trapezoid,2,16,1,") != std::string::npos);
    CHECK(a.find(",ca,5,3,") != std::string::npos);
    // EDM: every 2-D map gives the same cells; cell (2, 9) is the fixed-order distance
    for (i64 side : {14, 15}) {
        auto pts = make_edm_points(side, 7);
        std::vector<grid_spec> grids = {grid_bb(side, 2), grid_rb(side), grid_lambda(side),
                                        grid_h2d_padded(side + 1), grid_trapezoids(side + 1, side == 14 ? 1 : 4)};
        if (side == 15) grids.push_back(grid_h2d(16));
        std::vector<double> first;
        for (const auto& g : grids) {
            simplex_grid_state<double> st(2, side);
            auto rep = launch_edm(g, domain_of(g), pts, st);
            CHECK(verify_exact_cover(rep, domain_of(g)).exact);
            if (first.empty()) first = st.cells;
            CHECK(st.cells == first);
            const double dx = pts[2][0] - pts[9][0], dy = pts[2][1] - pts[9][1];
            CHECK(st.at(2, 9) == std::sqrt(dx * dx + dy * dy));
            CHECK(st.at(3, 3) == 0.0);
        }
    }
    {
        auto g = grid_h2d(16);
        auto pts = make_edm_points(14, 1);
        simplex_grid_state<double> st(2, 15);
        CHECK_THROWS_AS(launch_edm(g, domain_of(g), pts, st), std::invalid_argument);
    }
    // 2-D periodic Life, seed 42, 64 steps
    for (auto g : {grid_h2d(64), grid_bb(63, 2), grid_rb(63), grid_lambda(63), grid_trapezoids(64, 4)}) {
        auto st = make_life_state(2, 63, 42);
        launch_opts o;
        o.steps = 64;
        auto rep = launch_ca(g, domain_of(g), st, o);
        CHECK(rep.state_hash == 8247929562437622423ull);
    }
}

int main(int argc, char** argv) {
    const bool gpu = argc > 1 && std::strcmp(argv[1], "--gpu") == 0;
    try {
        host_suite();
        if (gpu) gpu_suite();
        if (gpu) report_suite();
    } catch (const std::exception& e) {
        std::printf("FAIL unexpected exception: %s\n", e.what());
        ++g_fail;
    }
    std::printf("drop-in %s: %d passed, %d failed\n", gpu ? "host+gpu" : "host", g_pass, g_fail);
    return g_fail == 0 ? 0 : 1;
}
