// TEST INFRASTRUCTURE ONLY — never linked into, loaded by, or called from the product.
//
// A thin extern "C" shim over the UNMODIFIED reference headers
// (/root/reference/proj/include/simplexmap/*.hpp, included in place, never copied).
// `oracle/Makefile` compiles this file with the reference's own Release flags
// (CMakeLists.txt:9-12: -O3 -DNDEBUG -Wall -Wextra, C++20) into
// oracle/_ref/libsmx_ref.so. Callers: tests/ (golden fixtures, parity), bench.py's
// cpu_baseline leg and `bench.py --impl reference`.
//
// Every entry point returns 0 on success, 1 on std::invalid_argument, 2 on
// std::overflow_error, 3 on any other exception; the message is kept in a
// thread-local buffer read by ref_last_error().

#include <simplexmap/report.hpp>
#include <simplexmap/simulator.hpp>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
#include <string>

using namespace simplexmap;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::overflow_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

map_kind kind_of(int k) {
    switch (k) {
        case 0: return map_kind::bb;
        case 1: return map_kind::rb;
        case 2: return map_kind::lambda2d;
        case 3: return map_kind::h2d;
        case 4: return map_kind::h2d_trapezoid;
        case 5: return map_kind::h2d_padded;
        case 6: return map_kind::h3d;
    }
    throw std::invalid_argument("ref harness: unknown map kind");
}

simplex_spec domain_of(const grid_spec& g) { return {g.dims, g.domain_side() * g.rho - 1}; }

void put_counters(const sim_report& rep, uint64_t* c) {
    if (!c) return;
    c[0] = rep.blocks_launched;
    c[1] = rep.blocks_void;
    c[2] = rep.threads_launched;
    c[3] = rep.threads_useful;
    // space_overhead as an exact rational (num, den); the i128 values fit i64
    // for every grid the tests use.
    c[4] = uint64_t(int64_t(rep.space_overhead.num));
    c[5] = uint64_t(int64_t(rep.space_overhead.den));
}

} // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// grid_spec via make_grid (report.hpp:48-66): extents[3], blocks, domain_side.
int ref_make_grid(int kind, int m, int64_t n, int64_t rho, int64_t T, int64_t* ext3,
                  uint64_t* blocks, int64_t* domain_side) {
    return guarded([&] {
        grid_spec g = make_grid(kind_of(kind), m, n, rho, T);
        for (int i = 0; i < 3; ++i) ext3[i] = g.extents[std::size_t(i)];
        *blocks = g.blocks();
        *domain_side = g.domain_side();
    });
}

// One map_outcome per block, natural z, y, x order (simulator.hpp:113-118):
// 6 x int64 {is_void, x, y, z, level_b, index_q}.
int ref_map_outcomes(int kind, int m, int64_t n, int64_t* out, uint64_t count) {
    return guarded([&] {
        grid_spec g = make_grid(kind_of(kind), m, n);
        if (g.blocks() != count) throw std::invalid_argument("ref_map_outcomes: count mismatch");
        uint64_t i = 0;
        for (int64_t z = 0; z < g.extents[2]; ++z)
            for (int64_t y = 0; y < g.extents[1]; ++y)
                for (int64_t x = 0; x < g.extents[0]; ++x) {
                    map_outcome o;
                    block_coord w{x, y, z};
                    if (g.kind == map_kind::h2d) o = map_h2d(w);
                    else if (g.kind == map_kind::h3d) o = map_h3d(w, g.n);
                    else if (g.kind == map_kind::bb) o = map_bb(w, g.n, g.dims);
                    else throw std::invalid_argument("ref_map_outcomes: bb/h2d/h3d only");
                    int64_t* r = out + 6 * i++;
                    r[0] = o.is_void;
                    r[1] = o.target.x;
                    r[2] = o.target.y;
                    r[3] = o.target.z;
                    r[4] = o.level_b;
                    r[5] = o.index_q;
                }
    });
}

// Every block of ANY grid kind in the reference's own emission order
// (detail::for_each_block_outcome, simulator.hpp:109-158: natural z, y, x;
// trapezoid bands one after another), 6 x int64 per block.
int ref_map_outcomes_t(int kind, int m, int64_t n, int64_t T, int64_t* out, uint64_t count) {
    return guarded([&] {
        grid_spec g = make_grid(kind_of(kind), m, n, 1, T);
        if (g.blocks() != count) throw std::invalid_argument("ref_map_outcomes_t: count mismatch");
        uint64_t i = 0;
        detail::for_each_block_outcome(g, 0, [&](block_coord, int, const map_outcome& o) {
            int64_t* r = out + 6 * i++;
            r[0] = o.is_void;
            r[1] = o.target.x;
            r[2] = o.target.y;
            r[3] = o.target.z;
            r[4] = o.level_b;
            r[5] = o.index_q;
        });
    });
}

// decompose_trapezoids (maps.hpp:228-257): 9 x int64 per band
// {delta_x, delta_y, band, h1, h2, grid_width, valid_side, ext_x, ext_y}.
int ref_decompose_trapezoids(int64_t n, int64_t T, int64_t* out, int max, int* count) {
    return guarded([&] {
        auto traps = decompose_trapezoids(n, T);
        *count = int(traps.size());
        for (int i = 0; i < int(traps.size()) && i < max; ++i) {
            const auto& t = traps[std::size_t(i)];
            int64_t* r = out + 9 * i;
            r[0] = t.delta_x; r[1] = t.delta_y; r[2] = t.band; r[3] = t.h1; r[4] = t.h2;
            r[5] = t.grid_width; r[6] = t.valid_side; r[7] = t.ext_x; r[8] = t.ext_y;
        }
    });
}

// map_h2d_trapezoid (maps.hpp:269-281) on band `band` of decompose_trapezoids(n, T).
int ref_map_trapezoid(int64_t n, int64_t T, int band, int64_t x, int64_t y, int64_t* out6) {
    return guarded([&] {
        auto traps = decompose_trapezoids(n, T);
        if (band < 0 || band >= int(traps.size())) throw std::invalid_argument("ref_map_trapezoid: band");
        map_outcome o = map_h2d_trapezoid({x, y, 0}, traps[std::size_t(band)]);
        out6[0] = o.is_void; out6[1] = o.target.x; out6[2] = o.target.y; out6[3] = o.target.z;
        out6[4] = o.level_b; out6[5] = o.index_q;
    });
}

// Single-block map probes (maps.hpp:107,200,302), for pinned points + error behaviour.
int ref_map_one(int kind, int m, int64_t n, int64_t x, int64_t y, int64_t z, int64_t* out6) {
    return guarded([&] {
        block_coord w{x, y, z};
        map_outcome o;
        if (kind == 0) o = map_bb(w, n, m);
        else if (kind == 1) o = map_outcome{false, map_rb_2d(w, n), 1, 0};
        else if (kind == 2) o = map_outcome{false, map_lambda_2d(u64(x), n), 1, 0};
        else if (kind == 3) o = map_h2d(w);
        else if (kind == 5) o = map_h2d_padded(w, n);
        else if (kind == 6) o = map_h3d(w, n);
        else throw std::invalid_argument("ref_map_one: use ref_map_trapezoid");
        out6[0] = o.is_void;
        out6[1] = o.target.x;
        out6[2] = o.target.y;
        out6[3] = o.target.z;
        out6[4] = o.level_b;
        out6[5] = o.index_q;
    });
}

// launch_map (simulator.hpp:303-310). coverage may be null (record_coverage=false).
// counters: 6 x u64 {blocks, void, threads, useful, overhead_num, overhead_den}.
int ref_launch_map(int kind, int m, int64_t n, int64_t rho, int64_t T, uint32_t* coverage,
                   uint64_t ncells, uint64_t salt, uint64_t* counters) {
    return guarded([&] {
        grid_spec g = make_grid(kind_of(kind), m, n, rho, T);
        launch_opts o;
        o.record_coverage = coverage != nullptr;
        o.block_order_salt = salt;
        sim_report rep = launch_map(g, domain_of(g), o);
        if (coverage) {
            if (rep.coverage.size() != ncells) throw std::invalid_argument("ncells mismatch");
            std::memcpy(coverage, rep.coverage.data(), ncells * sizeof(uint32_t));
        }
        put_counters(rep, counters);
    });
}

// launch_accum (simulator.hpp:313-327), `passes` times on the same state.
int ref_launch_accum(int kind, int m, int64_t n, int64_t rho, int64_t T, int64_t passes,
                     uint32_t* cells, uint64_t ncells, uint64_t* counters, uint64_t* hash,
                     double* seconds) {
    return guarded([&] {
        grid_spec g = make_grid(kind_of(kind), m, n, rho, T);
        simplex_spec dom = domain_of(g);
        simplex_grid_state<u32> st(m, dom.n + 1);
        if (st.cells.size() != ncells) throw std::invalid_argument("ncells mismatch");
        std::memcpy(st.cells.data(), cells, ncells * sizeof(uint32_t));
        launch_opts o;
        o.record_coverage = false;
        sim_report rep;
        auto t0 = std::chrono::steady_clock::now();
        for (int64_t p = 0; p < passes; ++p) rep = launch_accum(g, dom, st, o);
        auto t1 = std::chrono::steady_clock::now();
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        std::memcpy(cells, st.cells.data(), ncells * sizeof(uint32_t));
        put_counters(rep, counters);
        if (hash) *hash = st.hash();
    });
}

// make_life_state (simulator.hpp:390-398).
int ref_make_life_state(int m, int64_t side, uint64_t seed, uint8_t* out, uint64_t ncells) {
    return guarded([&] {
        auto s = make_life_state(m, side, seed);
        if (s.cells.size() != ncells) throw std::invalid_argument("ncells mismatch");
        std::memcpy(out, s.cells.data(), ncells);
    });
}

// kernel_ca_run (simulator.hpp:402-425), dead3d for m = 3, periodic2d for m = 2.
int ref_kernel_ca_run(int m, int64_t side, int64_t steps, uint8_t* cells, uint64_t ncells,
                      double* seconds) {
    return guarded([&] {
        simplex_grid_state<u8> s(m, side);
        if (s.cells.size() != ncells) throw std::invalid_argument("ncells mismatch");
        std::memcpy(s.cells.data(), cells, ncells);
        auto t0 = std::chrono::steady_clock::now();
        kernel_ca_run(s, steps, m == 3 ? ca_boundary::dead3d : ca_boundary::periodic2d);
        auto t1 = std::chrono::steady_clock::now();
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        std::memcpy(cells, s.cells.data(), ncells);
    });
}

// launch_ca (simulator.hpp:431-463) over a map-driven grid.
int ref_launch_ca(int kind, int m, int64_t n, int64_t rho, int64_t T, int64_t steps,
                  uint8_t* cells, uint64_t ncells, uint64_t* counters, uint64_t* hash,
                  double* seconds) {
    return guarded([&] {
        grid_spec g = make_grid(kind_of(kind), m, n, rho, T);
        simplex_spec dom = domain_of(g);
        simplex_grid_state<u8> s(m, dom.n + 1);
        if (s.cells.size() != ncells) throw std::invalid_argument("ncells mismatch");
        std::memcpy(s.cells.data(), cells, ncells);
        launch_opts o;
        o.record_coverage = false;
        o.steps = steps;
        o.boundary = m == 3 ? ca_boundary::dead3d : ca_boundary::periodic2d;
        auto t0 = std::chrono::steady_clock::now();
        sim_report rep = launch_ca(g, dom, s, o);
        auto t1 = std::chrono::steady_clock::now();
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        std::memcpy(cells, s.cells.data(), ncells);
        put_counters(rep, counters);
        if (hash) *hash = rep.state_hash;
    });
}

// make_edm_points (simulator.hpp:333-343): 2 doubles per point.
int ref_make_edm_points(int64_t count, uint64_t seed, double* out) {
    return guarded([&] {
        auto pts = make_edm_points(count, seed);
        for (std::size_t i = 0; i < pts.size(); ++i) out[2 * i] = pts[i][0], out[2 * i + 1] = pts[i][1];
    });
}

// kernel_edm (simulator.hpp:375-386): the sequential fill.
int ref_kernel_edm(int64_t side, uint64_t seed, double* cells, uint64_t ncells, uint64_t* hash) {
    return guarded([&] {
        auto pts = make_edm_points(side, seed);
        simplex_grid_state<double> s(2, side);
        if (s.cells.size() != ncells) throw std::invalid_argument("ncells mismatch");
        kernel_edm(pts, s);
        std::memcpy(cells, s.cells.data(), ncells * sizeof(double));
        if (hash) *hash = s.hash();
    });
}

// launch_edm (simulator.hpp:352-372) over a map-driven grid.
int ref_launch_edm(int kind, int64_t n, int64_t rho, int64_t T, uint64_t seed, double* cells, uint64_t ncells,
                   uint64_t* counters, uint64_t* hash) {
    return guarded([&] {
        grid_spec g = make_grid(kind_of(kind), 2, n, rho, T);
        simplex_spec dom = domain_of(g);
        auto pts = make_edm_points(dom.n + 1, seed);
        simplex_grid_state<double> s(2, dom.n + 1);
        if (s.cells.size() != ncells) throw std::invalid_argument("ncells mismatch");
        launch_opts o;
        o.record_coverage = false;
        o.seed = seed;
        sim_report rep = launch_edm(g, dom, pts, s, o);
        std::memcpy(cells, s.cells.data(), ncells * sizeof(double));
        put_counters(rep, counters);
        if (hash) *hash = rep.state_hash;
    });
}

// verify_sweep + csv_measure (mode 0) or analyze_sweep + csv_analyze (mode 1)
// over an n-range literal (report.hpp:73-110, 324-412). Writes up to cap bytes,
// *len = the full text length; witnesses of failed rows as "n:(x,y[,z])xM;".
int ref_csv_sweep(int kind, int m, const char* nrange, int64_t rho, int64_t T, int mode, char* out,
                  uint64_t cap, uint64_t* len, char* witnesses, uint64_t wcap) {
    return guarded([&] {
        auto ns = expand_n_range(parse_n_range(nrange));
        auto rows = mode == 0 ? verify_sweep(kind_of(kind), m, ns, rho, T) : analyze_sweep(kind_of(kind), m, ns, rho, T);
        std::string text = mode == 0 ? csv_measure(rows) : csv_analyze(rows);
        *len = text.size();
        std::memcpy(out, text.data(), std::min<uint64_t>(cap, text.size()));
        std::string w;
        if (mode == 0)
            for (const auto& r : rows)
                if (!r.exact) w += std::to_string(r.n) + ":" + witness_text(r) + "x" + std::to_string(r.multiplicity) + ";";
        if (witnesses && wcap) {
            std::size_t k = std::min<std::size_t>(wcap - 1, w.size());
            std::memcpy(witnesses, w.data(), k);
            witnesses[k] = 0;
        }
    });
}

// csv_optimize(optimize_params(m, inv_r_max, beta_max, n_eval), n_eval) (report.hpp:448-472)
int ref_csv_optimize(int m, int64_t inv_r_max, int64_t beta_max, int64_t n_eval, char* out, uint64_t cap,
                     uint64_t* len) {
    return guarded([&] {
        std::string text = csv_optimize(optimize_params(m, inv_r_max, beta_max, n_eval), n_eval);
        *len = text.size();
        std::memcpy(out, text.data(), std::min<uint64_t>(cap, text.size()));
    });
}

// simplex_grid_state<T>::hash (simulator.hpp:68-73) over raw cell bytes.
uint64_t ref_state_hash(int m, int64_t side, const void* bytes, uint64_t nbytes) {
    u64 h = fnv1a_seed;
    h = fnv1a_append_u64(h, u64(m));
    h = fnv1a_append_u64(h, u64(side));
    return fnv1a_append(h, bytes, nbytes);
}

// A bounded, multi-core sample of launch_accum (simulator.hpp:313-327) for the
// bench's reference arm at the full-size grids (C3: 2.1 G cells, ~12 s per
// pass on one core): the reference's own accounted_sweep (:277-291) with
// launch_accum's body `++cells[idx]`, over the first `rows` block rows (2-D) or
// block layers (3-D) of the grid in its natural walk order (:113-118) — the
// grid itself is untouched, so map, Void filter, thread expansion, membership
// and packed index are the reference's at that grid. `threads` replicas run
// concurrently (the reference is single-threaded within a launch,
// report.hpp:125-156), each on its own zero state (calloc: only the pages the
// sample touches are materialised). launch_accum's trailing state.hash() (a
// serial FNV over the whole state) is not part of the sample. Times `reps`
// repetitions after `warm` untimed ones: seconds[i] = wall time of rep i (all
// replicas); *useful = cells incremented per replica per rep.
int ref_accum_sample(int kind, int m, int64_t n, int64_t rho, int64_t rows, int threads, int warm, int reps,
                     double* seconds, uint64_t* useful) {
    return guarded([&] {
        grid_spec g = make_grid(kind_of(kind), m, n, rho, 1);
        if (g.kind == map_kind::h2d_trapezoid) throw std::invalid_argument("accum_sample: not for trapezoids");
        if (rows < 1 || threads < 1 || reps < 1 || warm < 0) throw std::invalid_argument("accum_sample: bad sizes");
        if (g.dims == 2) g.extents[1] = std::min<i64>(g.extents[1], rows);
        else g.extents[2] = std::min<i64>(g.extents[2], rows);
        const i64 side = g.domain_side() * g.rho;
        const std::size_t ncells = std::size_t(g.dims == 2 ? tri_cells(side) : tet_cells(side));
        std::vector<u32*> states(std::size_t(threads), nullptr);
        for (auto& p : states) {
            p = static_cast<u32*>(std::calloc(ncells, sizeof(u32)));
            if (!p) throw std::runtime_error("accum_sample: out of host memory");
        }
        launch_opts o;
        o.record_coverage = false;
        std::vector<u64> counts(std::size_t(threads), 0);
        for (int it = 0; it < warm + reps; ++it) {
            auto t0 = std::chrono::steady_clock::now();
            std::vector<std::thread> pool;
            for (int t = 0; t < threads; ++t)
                pool.emplace_back([&, t] {
                    sim_report rep = make_report(g, o);
                    u32* cells = states[std::size_t(t)];
                    accounted_sweep(g, rep, 0, [cells](i64, i64, i64, u64 idx) { ++cells[idx]; });
                    counts[std::size_t(t)] = rep.threads_useful;
                });
            for (auto& th : pool) th.join();
            auto t1 = std::chrono::steady_clock::now();
            if (it >= warm) seconds[it - warm] = std::chrono::duration<double>(t1 - t0).count();
        }
        for (auto* p : states) std::free(p);
        *useful = counts[0];
    });
}

// Cell counts (core.hpp:125-133).
uint64_t ref_tri_cells(int64_t side) { return uint64_t(tri_cells(side)); }
uint64_t ref_tet_cells(int64_t side) { return uint64_t(tet_cells(side)); }
uint64_t ref_tet_linear_index(int64_t side, int64_t x, int64_t y, int64_t z) {
    return tet_linear_index(side, x, y, z);
}

// verify_exact_cover (simulator.hpp:467-478) over a coverage array.
int ref_verify_exact_cover(int m, int64_t cell_side, const uint32_t* coverage, uint64_t ncells,
                           int* exact, int64_t* witness3, uint64_t* multiplicity) {
    return guarded([&] {
        sim_report rep;
        rep.m = m;
        rep.cell_side = cell_side;
        rep.coverage.assign(coverage, coverage + ncells);
        rep.coverage_recorded = true;
        cover_verdict v = verify_exact_cover(rep, simplex_spec{m, cell_side - 1});
        *exact = v.exact;
        witness3[0] = v.witness.x;
        witness3[1] = v.witness.y;
        witness3[2] = v.witness.z;
        *multiplicity = v.multiplicity;
    });
}

} // extern "C"
