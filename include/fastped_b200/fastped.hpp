// fastped_b200/fastped.hpp -- C++ drop-in for the reference's simulation-step API
// (/root/reference/proj/include/fastped, namespace fastped), running on a B200 through the C ABI
// of fastped_b200.h.  A caller of the reference swaps
//     #include <fastped/engine.hpp>        ->   #include <fastped_b200/fastped.hpp>
//     namespace fastped                    ->   namespace fastped_b200
// and links libfastped_b200.so.  Types and functions keep the reference's names, fields,
// argument meaning and exceptions:
//   Cell, CellKind, Boundary, Grid ...................... world.hpp:18-121
//   StaticField, compute_static_field ................... world.hpp:196-266
//   Agent, SimParams .................................... agents.hpp:13-45
//   Potential, SimState, make_state, state_hash ......... state.hpp:17-95
//   ScheduleParams, compute_blocksize, plan_phase,
//   MoveOutcome, move_phase, StepStats, step, RunStats, run  engine.hpp:21-183
//   spawn_agents ........................................ scenario_io.hpp:47-69
// SimState owns the device context: plan_phase / move_phase / step copy the state back after
// every call (so the host fields are always current, like the reference's), run() once at the
// end.  Host-side edits of `agents` are pushed before the next call.  One controller per
// SimState (state.hpp:19-21).  There is no CPU fallback: without an sm_100 device the calls
// throw std::runtime_error.
#pragma once

#include <cmath>
#include <cstdint>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../fastped_b200.h"

namespace fastped_b200 {

enum class CellKind : std::uint8_t { Free, Wall, Exit };
enum class Boundary : std::uint8_t { Closed, PeriodicX };
enum class Potential : std::uint8_t { ExitDistance, DriveX };

inline constexpr int kMinVmax = 1;
inline constexpr int kMaxVmax = 5;

struct Cell {
    int x = 0;
    int y = 0;
    friend bool operator==(Cell a, Cell b) { return a.x == b.x && a.y == b.y; }
};

namespace detail {
[[noreturn]] inline void raise(int code, const fp_ctx* ctx) {
    const std::string msg = fp_last_error(ctx);
    if (code == FP_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}
inline void check(int code, const fp_ctx* ctx = nullptr) {
    if (code != FP_OK) raise(code, ctx);
}
}  // namespace detail

// Grid (world.hpp:35-121): the constructor validates like the reference (same messages).
class Grid {
public:
    Grid(int width, int height, double cell_size, Boundary boundary, std::vector<CellKind> cells)
        : width_(width), height_(height), cell_size_(cell_size), boundary_(boundary), cells_(std::move(cells)) {
        if (width_ < 1 || height_ < 1) throw std::invalid_argument("Grid: width and height must be >= 1");
        if (!(cell_size_ > 0.0)) throw std::invalid_argument("Grid: cell_size must be > 0");
        if (cells_.size() != static_cast<std::size_t>(width_) * static_cast<std::size_t>(height_))
            throw std::invalid_argument("Grid: cell array size does not match width*height");
        for (int y = 0; y < height_; ++y)
            for (int x = 0; x < width_; ++x) {
                const CellKind k = cells_[index({x, y})];
                const bool top_bottom = (y == 0 || y == height_ - 1);
                if (boundary_ == Boundary::Closed) {
                    if ((top_bottom || x == 0 || x == width_ - 1) && k == CellKind::Free)
                        throw std::invalid_argument("Grid: closed boundary requires every border cell to be Wall or Exit");
                } else if (top_bottom && k != CellKind::Wall) {
                    throw std::invalid_argument("Grid: periodic-x boundary requires solid top and bottom rows");
                }
                if (k == CellKind::Free) ++free_count_;
                if (k == CellKind::Exit) ++exit_count_;
            }
    }
    int width() const { return width_; }
    int height() const { return height_; }
    double cell_size() const { return cell_size_; }
    Boundary boundary() const { return boundary_; }
    std::int64_t free_count() const { return free_count_; }
    std::int64_t exit_count() const { return exit_count_; }
    std::int64_t free_cell_count() const { return free_count_; }  // the reference's names (world.hpp)
    std::int64_t exit_cell_count() const { return exit_count_; }
    std::size_t index(Cell c) const {
        return static_cast<std::size_t>(c.y) * static_cast<std::size_t>(width_) + static_cast<std::size_t>(c.x);
    }
    CellKind at(Cell c) const { return cells_[index(c)]; }
    CellKind at(int x, int y) const { return at(Cell{x, y}); }
    const std::vector<CellKind>& cells() const { return cells_; }
    fp_grid_desc desc() const {
        return fp_grid_desc{width_, height_, cell_size_, static_cast<int32_t>(boundary_)};
    }

private:
    int width_, height_;
    double cell_size_;
    Boundary boundary_;
    std::vector<CellKind> cells_;
    std::int64_t free_count_ = 0, exit_count_ = 0;
};

struct StaticField {  // world.hpp:196-208
    static constexpr double kUnreachable = std::numeric_limits<double>::infinity();
    int width = 0;
    int height = 0;
    std::vector<double> s;
    double at(Cell c) const {
        return s[static_cast<std::size_t>(c.y) * static_cast<std::size_t>(width) + static_cast<std::size_t>(c.x)];
    }
    bool reachable(Cell c) const { return std::isfinite(at(c)); }
};

// compute_static_field (world.hpp:220-266), on the device, bit-identical.
inline StaticField compute_static_field(const Grid& g, int device = 0) {
    StaticField f;
    f.width = g.width();
    f.height = g.height();
    f.s.resize(static_cast<std::size_t>(g.width()) * g.height());
    const fp_grid_desc d = g.desc();
    detail::check(fp_static_field(&d, reinterpret_cast<const uint8_t*>(g.cells().data()), device, f.s.data()));
    return f;
}

struct Agent {  // agents.hpp:13-18
    std::uint32_t id = 0;
    Cell pos;
    int v_max = 4;
    bool alive = true;
};

struct SimParams {  // agents.hpp:22-45
    double k_s = 1.2;
    double k_other = 0.0;
    int v_max = 4;
    std::uint64_t seed = 1;
    int steps = 396;
    double dt = 1.0;
    SimParams() = default;
    SimParams(double k_s_, double k_other_, int v_max_, std::uint64_t seed_, int steps_, double dt_)
        : k_s(k_s_), k_other(k_other_), v_max(v_max_), seed(seed_), steps(steps_), dt(dt_) {
        validate();
    }
    void validate() const {
        if (k_other != 0.0) throw std::invalid_argument("SimParams: k_other must be 0");
        if (v_max < kMinVmax || v_max > kMaxVmax) throw std::invalid_argument("SimParams: v_max must be in [1,5]");
        if (steps < 1) throw std::invalid_argument("SimParams: steps must be >= 1");
        if (!(dt > 0.0)) throw std::invalid_argument("SimParams: dt must be > 0");
    }
};

struct ScheduleParams {  // engine.hpp:21-23; cores only validated (results never depend on it)
    int cores = 1;
};

struct MoveOutcome {  // engine.hpp:86-89
    std::vector<std::uint32_t> exited;
    std::int64_t displacement_cells = 0;
};
struct StepStats {  // engine.hpp:137-141
    std::int64_t alive = 0;
    std::int64_t exited = 0;
    std::int64_t displacement_cells = 0;
};
struct RunStats {  // engine.hpp:150-158 (times from CUDA events)
    double wall_time_s = 0.0;
    double plan_time_s = 0.0;
    double move_time_s = 0.0;
    std::int64_t steps = 0;
    std::int64_t exited = 0;
    std::int64_t displacement_cells = 0;
    std::int64_t alive = 0;
};

// SimState (state.hpp:22-36) with its device context.
struct SimState {
    static constexpr std::int32_t kEmpty = -1;
    std::shared_ptr<const Grid> grid;
    std::shared_ptr<const StaticField> field;
    std::vector<Agent> agents;
    std::vector<std::int32_t> occupancy;  // cell -> agent id, or kEmpty (refreshed with the agents)
    std::vector<Cell> desired;
    std::int64_t step = 0;
    std::int64_t alive = 0;
    Potential potential = Potential::ExitDistance;
    double drive_gradient = 0.0;

    std::int32_t occupant(Cell c) const { return occupancy[grid->index(c)]; }

    // --- device side (not in the reference) ---
    std::shared_ptr<fp_ctx> ctx;
    void push() {  // host edits -> device (positions, alive, step, potential)
        const std::size_t n = agents.size();
        std::vector<int32_t> x(n), y(n);
        std::vector<uint8_t> a(n);
        for (std::size_t i = 0; i < n; ++i) {
            x[i] = agents[i].pos.x;
            y[i] = agents[i].pos.y;
            a[i] = agents[i].alive ? 1 : 0;
        }
        detail::check(fp_update_agents(ctx.get(), x.data(), y.data(), a.data()), ctx.get());
        detail::check(fp_set_step(ctx.get(), step), ctx.get());
        detail::check(fp_set_potential(ctx.get(), static_cast<int>(potential), drive_gradient), ctx.get());
    }
    void pull() {  // device -> host fields
        const std::size_t n = agents.size();
        std::vector<int32_t> x(n ? n : 1), y(n ? n : 1), dx(n ? n : 1), dy(n ? n : 1);
        std::vector<uint8_t> a(n ? n : 1);
        detail::check(fp_get_agents(ctx.get(), x.data(), y.data(), a.data()), ctx.get());
        detail::check(fp_get_desired(ctx.get(), dx.data(), dy.data()), ctx.get());
        for (std::size_t i = 0; i < n; ++i) {
            agents[i].pos = {x[i], y[i]};
            agents[i].alive = a[i] != 0;
            desired[i] = {dx[i], dy[i]};
        }
        occupancy.assign(static_cast<std::size_t>(grid->width()) * grid->height(), kEmpty);
        detail::check(fp_get_occupancy(ctx.get(), occupancy.data()), ctx.get());
        detail::check(fp_get_step(ctx.get(), &step), ctx.get());
        detail::check(fp_get_alive_count(ctx.get(), &alive), ctx.get());
    }
};

// make_state (state.hpp:38-76): validates the roster like the reference, uploads everything.
inline SimState make_state(std::shared_ptr<const Grid> grid, std::shared_ptr<const StaticField> field,
                           std::vector<Agent> roster, int device = 0) {
    if (!grid) throw std::invalid_argument("make_state: null grid");
    if (field && (field->width != grid->width() || field->height != grid->height() ||
                  field->s.size() != static_cast<std::size_t>(grid->width()) * static_cast<std::size_t>(grid->height())))
        throw std::invalid_argument("make_state: field dimensions do not match grid");
    for (const Agent& a : roster)  // state.hpp:56-57; per-agent v_max may be edited afterwards, as in the reference
        if (a.v_max != roster.front().v_max) throw std::invalid_argument("make_state: all agents must share one v_max");
    SimState st;
    st.grid = grid;
    const fp_grid_desc d = grid->desc();
    fp_ctx* raw = nullptr;
    detail::check(fp_create(&d, reinterpret_cast<const uint8_t*>(grid->cells().data()),
                            field ? field->s.data() : nullptr, device, &raw));
    st.ctx = std::shared_ptr<fp_ctx>(raw, fp_destroy);
    if (!field) {  // the device computed it: keep the reference's shared immutable field
        auto f = std::make_shared<StaticField>();
        f->width = grid->width();
        f->height = grid->height();
        f->s.resize(static_cast<std::size_t>(grid->width()) * grid->height());
        detail::check(fp_get_field(raw, f->s.data()), raw);
        field = f;
    }
    st.field = field;
    const std::size_t n = roster.size();
    std::vector<int32_t> x(n ? n : 1), y(n ? n : 1), v(n ? n : 1);
    std::vector<uint8_t> a(n ? n : 1);
    for (std::size_t i = 0; i < n; ++i) {
        if (roster[i].id != i) throw std::invalid_argument("make_state: agent ids must be dense indices");
        x[i] = roster[i].pos.x;
        y[i] = roster[i].pos.y;
        v[i] = roster[i].v_max;
        a[i] = roster[i].alive ? 1 : 0;
    }
    detail::check(fp_set_agents(raw, static_cast<uint32_t>(n), x.data(), y.data(), v.data(), a.data(), 0), raw);
    st.agents = std::move(roster);
    st.desired.resize(n);
    st.pull();
    return st;
}

// state_hash (state.hpp:80-95) of the host fields, which are the state between calls (the
// caller may have edited them, e.g. ++st.step after move_phase, as the reference's tests do).
inline std::uint64_t state_hash(const SimState& st) {
    std::uint64_t h = 14695981039346656037ULL;  // FNV-1a 64 over step, alive, (id, x, y, alive)*
    auto mix = [&h](std::uint64_t v) {
        h ^= v;
        h *= 1099511628211ULL;
    };
    mix(static_cast<std::uint64_t>(st.step));
    mix(static_cast<std::uint64_t>(st.alive));
    for (const Agent& a : st.agents) {
        mix(a.id);
        mix(static_cast<std::uint32_t>(a.pos.x));
        mix(static_cast<std::uint32_t>(a.pos.y));
        mix(a.alive ? 1u : 0u);
    }
    return h;
}

inline int compute_blocksize(std::int64_t number_of_agents, int cores) {  // engine.hpp:27-33
    int32_t b = 0;
    detail::check(fp_compute_blocksize(number_of_agents, cores, &b));
    return b;
}

inline void plan_phase(SimState& st, const SimParams& params, const ScheduleParams& sched) {  // engine.hpp:71-84
    if (sched.cores < 1) throw std::invalid_argument("plan_phase: cores must be >= 1");
    st.push();
    detail::check(fp_plan(st.ctx.get(), params.k_s, params.seed), st.ctx.get());
    st.pull();
}

inline MoveOutcome move_phase(SimState& st, const SimParams& params) {  // engine.hpp:95-135
    std::vector<int32_t> dx(st.agents.size() ? st.agents.size() : 1), dy(dx.size());
    for (std::size_t i = 0; i < st.agents.size(); ++i) {
        dx[i] = st.desired[i].x;
        dy[i] = st.desired[i].y;
    }
    st.push();
    detail::check(fp_set_desired(st.ctx.get(), dx.data(), dy.data()), st.ctx.get());
    fp_step_stats s{};
    detail::check(fp_move(st.ctx.get(), params.seed, &s), st.ctx.get());
    MoveOutcome out;
    out.displacement_cells = s.displacement_cells;
    out.exited.resize(static_cast<std::size_t>(s.exited));
    uint32_t n = 0;
    if (s.exited)
        detail::check(fp_get_exited(st.ctx.get(), out.exited.data(), static_cast<uint32_t>(s.exited), &n),
                      st.ctx.get());
    st.pull();
    return out;
}

inline StepStats step(SimState& st, const SimParams& params, const ScheduleParams& sched) {  // engine.hpp:143-148
    if (sched.cores < 1) throw std::invalid_argument("plan_phase: cores must be >= 1");
    st.push();
    fp_step_stats s{};
    detail::check(fp_step(st.ctx.get(), params.k_s, params.seed, &s), st.ctx.get());
    st.pull();
    return {s.alive, s.exited, s.displacement_cells};
}

inline RunStats run(SimState& st, const SimParams& params, const ScheduleParams& sched) {  // engine.hpp:161-183
    params.validate();
    if (sched.cores < 1) throw std::invalid_argument("run: cores must be >= 1");
    st.push();
    fp_run_stats r{};
    detail::check(fp_run(st.ctx.get(), params.k_s, params.seed, params.steps, &r), st.ctx.get());
    st.pull();
    return {r.wall_time_s, r.plan_time_s, r.move_time_s, r.steps, r.exited, r.displacement_cells, r.alive};
}

// spawn_agents (scenario_io.hpp:47-69): the same draws, agents on the row-major free list.
inline std::vector<Agent> spawn_agents(const Grid& grid, std::int64_t n, int v_max, std::uint64_t seed) {
    std::vector<int32_t> x(n > 0 ? n : 1), y(n > 0 ? n : 1);
    detail::check(fp_spawn_agents(grid.width(), grid.height(), reinterpret_cast<const uint8_t*>(grid.cells().data()),
                                  n, seed, x.data(), y.data()));
    std::vector<Agent> out(static_cast<std::size_t>(n));
    for (std::int64_t i = 0; i < n; ++i) out[i] = Agent{static_cast<std::uint32_t>(i), {x[i], y[i]}, v_max, true};
    return out;
}

}  // namespace fastped_b200
