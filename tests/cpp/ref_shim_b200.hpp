// proj/include/simplexmap/b200.hpp  (new file in the reference)
#pragma once
#include "simulator.hpp"
#include <smx_b200.h>

namespace simplexmap::b200 {
inline smx_grid to_abi(const grid_spec& g) {
    smx_grid r{};
    if (smx_make_grid(int32_t(g.kind), g.dims, g.n, g.rho, g.threshold, &r) != SMX_OK)
        throw std::invalid_argument(smx_last_error());
    return r;
}
inline void fill(sim_report& rep, const smx_counters& c) {
    rep.blocks_launched = c.blocks_launched;  rep.blocks_void = c.blocks_void;
    rep.threads_launched = c.threads_launched; rep.threads_useful = c.threads_useful;
    finish_report(rep);                        // simulator.hpp:279
}
inline sim_report launch_accum(const grid_spec& g, const simplex_spec& d,
                               simplex_grid_state<u32>& s, const launch_opts& o = {}) {
    validate_launch(g, d);                     // simulator.hpp:257
    sim_report rep = make_report(g, o);        // simulator.hpp:266
    smx_grid r = to_abi(g); smx_counters c{};
    if (smx_accum(&r, s.cells.data(), s.cells.size(), 1, SMX_EXEC_AUTO, 0,
                  o.record_coverage ? rep.coverage.data() : nullptr, &c, nullptr) != SMX_OK)
        throw std::runtime_error(smx_last_error());
    fill(rep, c); rep.state_hash = s.hash();
    return rep;
}
inline sim_report launch_ca(const grid_spec& g, const simplex_spec& d,
                            simplex_grid_state<u8>& s, const launch_opts& o = {}) {
    validate_launch(g, d);
    sim_report rep = make_report(g, o);
    smx_grid r = to_abi(g); smx_counters c{};
    if (smx_ca(&r, s.cells.data(), s.cells.size(), o.steps, SMX_EXEC_AUTO, 0, nullptr,
               o.record_coverage ? rep.coverage.data() : nullptr, &c, nullptr) != SMX_OK)
        throw std::runtime_error(smx_last_error());
    fill(rep, c); rep.state_hash = s.hash();
    return rep;
}
inline sim_report launch_map(const grid_spec& g, const simplex_spec& d, const launch_opts& o = {}) {
    validate_launch(g, d);
    sim_report rep = make_report(g, o);
    smx_grid r = to_abi(g); smx_counters c{};
    if (smx_launch_map(&r, o.record_coverage ? rep.coverage.data() : nullptr, rep.coverage.size(), 0, &c,
                       nullptr) != SMX_OK)
        throw std::runtime_error(smx_last_error());
    fill(rep, c);
    return rep;
}
}  // namespace simplexmap::b200
