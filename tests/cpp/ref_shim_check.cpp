// TEST INFRASTRUCTURE. The reference-side binding of INTEGRATION.md section 2
// (ref_shim_b200.hpp, byte-identical to the document's code block) compiled
// against the REFERENCE's own headers, and checked against the reference's
// own launch_map / launch_accum / launch_ca on the same grids: state hashes,
// counters, exact space_overhead rationals and coverage multisets must agree.
#include <simplexmap/report.hpp>
#include <simplexmap/simulator.hpp>

#include <cstdio>
#include <string>

#include "ref_shim_b200.hpp"

using namespace simplexmap;

namespace {
int checks = 0, failed = 0;
void expect(bool ok, const std::string& what) {
    ++checks;
    if (!ok) {
        ++failed;
        std::printf("FAIL %s\n", what.c_str());
    }
}
bool same_counts(const sim_report& a, const sim_report& b) {
    return a.blocks_launched == b.blocks_launched && a.blocks_void == b.blocks_void &&
           a.threads_launched == b.threads_launched && a.threads_useful == b.threads_useful &&
           a.space_overhead == b.space_overhead && a.coverage == b.coverage && a.state_hash == b.state_hash;
}
std::string name(const grid_spec& g) {
    return std::string(map_kind_name(g.kind)) + " n=" + std::to_string(g.n) + " rho=" + std::to_string(g.rho);
}
}  // namespace

int main() {
    // ACCUM and MAP through the shim vs the reference, 2-D grids
    for (grid_spec g : {make_grid(map_kind::h2d, 2, 64, 4), make_grid(map_kind::bb, 2, 63, 4),
                        make_grid(map_kind::h2d_trapezoid, 2, 45, 3, 4), make_grid(map_kind::rb, 2, 33, 2),
                        make_grid(map_kind::h2d_padded, 2, 40, 2)}) {
        const simplex_spec d(2, g.domain_side() * g.rho - 1);
        simplex_grid_state<u32> a(2, d.n + 1), b(2, d.n + 1);
        const sim_report ra = launch_accum(g, d, a);
        const sim_report rb = b200::launch_accum(g, d, b);
        expect(same_counts(ra, rb) && a.cells == b.cells, "accum " + name(g));
        expect(same_counts(launch_map(g, d), b200::launch_map(g, d)), "map " + name(g));
    }
    // the 3-D dead-boundary Life through the shim vs the reference
    for (grid_spec g : {make_grid(map_kind::h3d, 3, 16, 4), make_grid(map_kind::bb, 3, 15, 4),
                        make_grid(map_kind::h3d, 3, 8, 8), make_grid(map_kind::h3d, 3, 16, 1),
                        make_grid(map_kind::bb, 3, 7, 3)}) {
        const simplex_spec d(3, g.domain_side() * g.rho - 1);
        launch_opts o;
        o.steps = 5;
        o.boundary = ca_boundary::dead3d;
        simplex_grid_state<u8> a = make_life_state(3, d.n + 1, 42), b = a;
        const sim_report ra = launch_ca(g, d, a, o);
        const sim_report rb = b200::launch_ca(g, d, b, o);
        expect(same_counts(ra, rb) && a.cells == b.cells, "ca3d " + name(g));
        expect(same_counts(launch_map(g, d), b200::launch_map(g, d)), "map " + name(g));
    }
    // the periodic 2-D Life
    {
        grid_spec g = make_grid(map_kind::h2d, 2, 32, 2);
        const simplex_spec d(2, g.domain_side() * g.rho - 1);
        launch_opts o;
        o.steps = 7;
        simplex_grid_state<u8> a = make_life_state(2, d.n + 1, 9), b = a;
        expect(same_counts(launch_ca(g, d, a, o), b200::launch_ca(g, d, b, o)) && a.cells == b.cells,
               "ca2d " + name(g));
    }
    // contract violations surface as the reference's exception types
    bool threw = false;
    try {
        simplex_grid_state<u32> s(2, 10);
        b200::launch_accum(grid_h2d(8), simplex_spec(2, 3), s);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    expect(threw, "validate_launch via the shim");
    std::printf("ref_shim_check: %d checks, %d failed\n", checks, failed);
    return failed ? 1 : 0;
}
