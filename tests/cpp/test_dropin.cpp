// The C++ drop-in (include/simplexmap_b200.hpp) exercised the way the
// reference's own suites exercise simplexmap (test_maps.cpp, test_simulator.cpp,
// acceptance.cpp) on the hot-path functions. `--host`: map / grid / contract
// checks (no GPU); `--gpu`: launches through libsmx_b200.so on cuda:0.
#define SMX_B200_AS_SIMPLEXMAP
#include "simplexmap_b200.hpp"

#include <algorithm>
#include <cstdio>
#include <cstring>
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

static void host_suite() {
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

int main(int argc, char** argv) {
    const bool gpu = argc > 1 && std::strcmp(argv[1], "--gpu") == 0;
    try {
        host_suite();
        if (gpu) gpu_suite();
    } catch (const std::exception& e) {
        std::printf("FAIL unexpected exception: %s\n", e.what());
        ++g_fail;
    }
    std::printf("drop-in %s: %d passed, %d failed\n", gpu ? "host+gpu" : "host", g_pass, g_fail);
    return g_fail == 0 ? 0 : 1;
}
