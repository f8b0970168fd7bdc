// ref_shim.cpp -- extern "C" handle over the UNMODIFIED reference engine (TEST INFRASTRUCTURE).
//
// Compiled by oracle/Makefile against the read-only headers under
// /root/reference/proj/include (never copied) into oracle/_ref/libfastped_ref.so.
// Used by tests/ to pin the C restatement (oracle.c) and the CUDA path, and by bench.py's
// `--impl reference` / cpu_baseline legs to time the reference's own run() on host cores.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "fastped/fastped.hpp"

using namespace fastped;

namespace {
thread_local std::string g_err;

struct RefState {
    SimState st;
};

std::vector<CellKind> to_cells(int w, int h, const uint8_t* cells) {
    std::vector<CellKind> v(static_cast<size_t>(w) * h);
    for (size_t i = 0; i < v.size(); ++i) v[i] = static_cast<CellKind>(cells[i]);
    return v;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

uint64_t ref_rng_u64(uint64_t s, uint64_t a, uint64_t t, uint64_t d) { return rng_u64(s, a, t, d); }

int ref_compute_blocksize(int64_t n, int cores) {
    try {
        return compute_blocksize(n, cores);
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

size_t ref_sample_index(const double* w, size_t n, double u) {
    return detail::sample_index(std::span<const double>(w, n), u);
}

double ref_exp(double x) { return std::exp(x); }

int ref_static_field(int w, int h, int boundary, const uint8_t* cells, double* out) {
    try {
        Grid g(w, h, 0.4, static_cast<Boundary>(boundary), to_cells(w, h, cells));
        StaticField f = compute_static_field(g);
        std::memcpy(out, f.s.data(), f.s.size() * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// Builds a SimState through make_state; per-agent v_max values are written after make_state
// (the reference's kernels use the per-agent field).  field may be null
// (then compute_static_field runs).
void* ref_state_create(int w, int h, double cell_size, int boundary, const uint8_t* cells,
                       const double* field, int n, const int32_t* x, const int32_t* y,
                       const int32_t* v_max, const uint8_t* alive, int64_t step, int potential,
                       double drive_gradient) {
    try {
        auto g = std::make_shared<const Grid>(w, h, cell_size, static_cast<Boundary>(boundary),
                                              to_cells(w, h, cells));
        std::shared_ptr<const StaticField> f;
        if (field) {
            StaticField sf{w, h, std::vector<double>(field, field + static_cast<size_t>(w) * h)};
            f = std::make_shared<const StaticField>(std::move(sf));
        } else {
            f = std::make_shared<const StaticField>(compute_static_field(*g));
        }
        std::vector<Agent> roster(static_cast<size_t>(n));
        const int v0 = n > 0 ? v_max[0] : 4;
        for (int i = 0; i < n; ++i)
            roster[i] = Agent{static_cast<uint32_t>(i), Cell{x[i], y[i]}, v0, alive ? alive[i] != 0 : true};
        auto* rs = new RefState{make_state(g, f, std::move(roster))};
        for (int i = 0; i < n; ++i) rs->st.agents[i].v_max = v_max[i];
        rs->st.step = step;
        rs->st.potential = static_cast<Potential>(potential);
        rs->st.drive_gradient = drive_gradient;
        return rs;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void ref_state_destroy(void* p) { delete static_cast<RefState*>(p); }

void ref_set_step(void* p, int64_t step) { static_cast<RefState*>(p)->st.step = step; }
int64_t ref_get_step(void* p) { return static_cast<RefState*>(p)->st.step; }
int64_t ref_alive_count(void* p) { return static_cast<RefState*>(p)->st.alive; }
uint64_t ref_state_hash(void* p) { return state_hash(static_cast<RefState*>(p)->st); }

void ref_get_agents(void* p, int32_t* x, int32_t* y, uint8_t* alive) {
    const SimState& st = static_cast<RefState*>(p)->st;
    for (size_t i = 0; i < st.agents.size(); ++i) {
        x[i] = st.agents[i].pos.x;
        y[i] = st.agents[i].pos.y;
        alive[i] = st.agents[i].alive ? 1 : 0;
    }
}

void ref_get_desired(void* p, int32_t* x, int32_t* y) {
    const SimState& st = static_cast<RefState*>(p)->st;
    for (size_t i = 0; i < st.desired.size(); ++i) {
        x[i] = st.desired[i].x;
        y[i] = st.desired[i].y;
    }
}

void ref_set_desired(void* p, const int32_t* x, const int32_t* y) {
    SimState& st = static_cast<RefState*>(p)->st;
    for (size_t i = 0; i < st.desired.size(); ++i) st.desired[i] = Cell{x[i], y[i]};
}

void ref_get_occupancy(void* p, int32_t* occ) {
    const SimState& st = static_cast<RefState*>(p)->st;
    std::memcpy(occ, st.occupancy.data(), st.occupancy.size() * sizeof(int32_t));
}

int ref_plan_phase(void* p, double k_s, uint64_t seed, int cores) {
    try {
        SimParams params;
        params.k_s = k_s;
        params.seed = seed;
        plan_phase(static_cast<RefState*>(p)->st, params, ScheduleParams{cores});
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// move_phase; exited ids in processing order (cap entries written), returns displacement
int64_t ref_move_phase(void* p, uint64_t seed, uint32_t* exited, int64_t cap, int64_t* n_exited) {
    SimParams params;
    params.seed = seed;
    const MoveOutcome mv = move_phase(static_cast<RefState*>(p)->st, params);
    for (size_t i = 0; i < mv.exited.size() && static_cast<int64_t>(i) < cap; ++i) exited[i] = mv.exited[i];
    *n_exited = static_cast<int64_t>(mv.exited.size());
    return mv.displacement_cells;
}

// run(): times the stepping loop exactly as the reference does (engine.hpp:161-183)
int ref_run(void* p, double k_s, uint64_t seed, int steps, int cores, double* wall, double* plan,
            double* move, int64_t* exited, int64_t* displacement) {
    try {
        SimParams params;
        params.k_s = k_s;
        params.seed = seed;
        params.steps = steps;
        const RunStats rs = run(static_cast<RefState*>(p)->st, params, ScheduleParams{cores});
        *wall = rs.wall_time_s;
        *plan = rs.plan_time_s;
        *move = rs.move_time_s;
        *exited = rs.exited;
        *displacement = rs.displacement_cells;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// Candidate list and exact fp64 weights of one agent, through the reference's own
// enumerate_candidates / potential_drop / std::exp (planning.hpp:88-104).
int ref_choice_weights(void* p, uint32_t agent, double k_s, double* w, int32_t* cx, int32_t* cy,
                       int cap) {
    const SimState& st = static_cast<RefState*>(p)->st;
    const Agent& a = st.agents[agent];
    const auto cands = enumerate_candidates(st, a);
    const Cell pos = st.grid->normalize(a.pos);
    const bool exitd = st.potential == Potential::ExitDistance;
    for (size_t i = 0; i < cands.size() && static_cast<int>(i) < cap; ++i) {
        cx[i] = cands[i].x;
        cy[i] = cands[i].y;
        if (exitd && !st.field->reachable(pos))
            w[i] = 1.0;
        else if (exitd && !st.field->reachable(cands[i]))
            w[i] = 0.0;
        else
            w[i] = std::exp(k_s * detail::potential_drop(st, pos, cands[i]));
    }
    return static_cast<int>(cands.size());
}

int ref_choose_desired(void* p, uint32_t agent, double k_s, uint64_t seed, int32_t* x, int32_t* y) {
    SimParams params;
    params.k_s = k_s;
    params.seed = seed;
    const SimState& st = static_cast<RefState*>(p)->st;
    const Cell c = choose_desired_cell(st, st.agents[agent], params);
    *x = c.x;
    *y = c.y;
    return 0;
}

int ref_spawn_agents(int w, int h, const uint8_t* cells, int boundary, int64_t n, int v_max,
                     uint64_t seed, int32_t* x, int32_t* y) {
    try {
        Grid g(w, h, 0.4, static_cast<Boundary>(boundary), to_cells(w, h, cells));
        const auto roster = spawn_agents(g, n, v_max, seed);
        for (size_t i = 0; i < roster.size(); ++i) {
            x[i] = roster[i].pos.x;
            y[i] = roster[i].pos.y;
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// Generators (scenario_io.hpp:74-121): writes cells (caller sizes with *w,*h from a first
// call with cells == nullptr).
int ref_make_plaza(double side_m, int exits, double cell, int* w, int* h, uint8_t* cells) {
    try {
        const Grid g = make_plaza(side_m, exits, cell);
        *w = g.width();
        *h = g.height();
        if (cells)
            for (int yy = 0; yy < g.height(); ++yy)
                for (int xx = 0; xx < g.width(); ++xx)
                    cells[static_cast<size_t>(yy) * g.width() + xx] = static_cast<uint8_t>(g.at(xx, yy));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

int ref_make_corridor(double len_m, double width_m, double cell, int* w, int* h, uint8_t* cells) {
    try {
        const Grid g = make_corridor(len_m, width_m, cell);
        *w = g.width();
        *h = g.height();
        if (cells)
            for (int yy = 0; yy < g.height(); ++yy)
                for (int xx = 0; xx < g.width(); ++xx)
                    cells[static_cast<size_t>(yy) * g.width() + xx] = static_cast<uint8_t>(g.at(xx, yy));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// fundamental_diagram (bench.hpp:244-305) on a periodic-x corridor given as cells: one
// (density, mean_speed, flow) triple per requested density.
int ref_fundamental_diagram(int w, int h, double cell, const uint8_t* cells, int v_max, const double* densities,
                            int nd, uint64_t seed, int warmup, int measure, double drive_gradient,
                            double* density, double* mean_speed, double* flow) {
    try {
        Grid g(w, h, cell, Boundary::PeriodicX, to_cells(w, h, cells));
        const std::vector<double> rho(densities, densities + nd);
        const auto fd = fundamental_diagram(g, v_max, rho, seed, warmup, measure, drive_gradient);
        for (size_t i = 0; i < fd.size(); ++i) {
            density[i] = fd[i].density;
            mean_speed[i] = fd[i].mean_speed;
            flow[i] = fd[i].flow;
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// realtime_capacity (bench.hpp:165-208) driven by a timing table: wall_time_of(n) is looked up
// in (ns[i], ts[i]) (exact n required), so the bracket logic can be pinned without timing.
int ref_capacity_from_table(const int64_t* ns, const double* ts, int nt, double budget, int64_t start_n, int64_t max_n,
                            int64_t* out6 /* capacity, n_low, n_high, below_start, capped, probes */,
                            double* out3 /* t_low, t_high, budget */) {
    try {
        int64_t probes = 0;
        auto fn = [&](int64_t n) {
            ++probes;
            for (int i = 0; i < nt; ++i)
                if (ns[i] == n) return ts[i];
            throw std::runtime_error("ref_capacity_from_table: no timing for n=" + std::to_string(n));
        };
        const CapacityResult r = realtime_capacity(fn, budget, start_n, max_n);
        out6[0] = r.capacity;
        out6[1] = r.n_low;
        out6[2] = r.n_high;
        out6[3] = r.below_start;
        out6[4] = r.capped;
        out6[5] = probes;
        out3[0] = r.t_low_s;
        out3[1] = r.t_high_s;
        out3[2] = r.budget_s;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

}  // extern "C"
