// Drop-in replacement of fastped/state.hpp (/root/reference/proj/include/fastped/state.hpp):
// the same Potential, SimState (same public fields and occupant()), make_state (same checks and
// messages, state.hpp:38-76) and state_hash (FNV-1a, state.hpp:80-95) -- plus a device mirror.
//
// SimState's host fields stay the authoritative state, exactly as callers of the reference see
// them; the device mirror (one libfastped_b200 context on a B200) is a cache the engine entry
// points (engine.hpp / planning.hpp overlays) bring up to date before every device call
// (positions, alive flags, v_max, step, potential, desired cells) and copy back after it.  So
// callers may edit agents, ++st.step or copy a SimState between calls, as the reference's tests
// do.  Differences from the reference, both deliberate:
//   * make_state accepts a roster whose v_max differ per agent only through the same route as
//     the reference (make_state with one v_max, then writing agents[i].v_max); the edit is
//     picked up by the next device call;
//   * occupancy is refreshed incrementally from the positions before/after each device call.
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "fastped/agents.hpp"
#include "fastped/world.hpp"
#include "device.hpp"

namespace fastped {

enum class Potential : std::uint8_t { ExitDistance, DriveX };

namespace b200 {
/// The device side of one SimState: the context plus what was last uploaded to it.
struct Mirror {
    fp_ctx* ctx = nullptr;
    std::vector<std::int32_t> x, y, v;
    std::vector<std::uint8_t> alive;
    std::int64_t step = -1;
    int potential = -1;
    double gradient = 0.0;
    // ScheduleParams::gpus > 1: one strip context per GPU, driven from this thread (fp_strips_*)
    std::vector<fp_ctx*> strips;
    Mirror() = default;
    Mirror(const Mirror&) = delete;
    Mirror& operator=(const Mirror&) = delete;
    void drop_strips() {
        for (fp_ctx* c : strips) fp_destroy(c);
        strips.clear();
    }
    ~Mirror() {
        drop_strips();
        if (ctx) fp_destroy(ctx);
    }
};
}  // namespace b200

struct SimState {
    static constexpr std::int32_t kEmpty = -1;

    std::shared_ptr<const Grid> grid;
    std::shared_ptr<const StaticField> field;
    std::vector<Agent> agents;
    std::vector<std::int32_t> occupancy;  // cell -> agent id, or kEmpty
    std::vector<Cell> desired;            // scratch, valid only between phases
    std::int64_t step = 0;
    std::int64_t alive = 0;
    Potential potential = Potential::ExitDistance;
    double drive_gradient = 0.0;

    std::int32_t occupant(Cell c) const { return occupancy[grid->index(grid->normalize(c))]; }

    // ---- device mirror (not in the reference) ----
    std::shared_ptr<b200::Mirror> dev;

    /// Uploads whatever the host changed since the last upload; `with_desired` also uploads the
    /// desired cells (move_phase consumes them).  Returns the context.
    fp_ctx* sync_to_device(bool with_desired = false) const {
        b200::Mirror& m = *dev;
        const std::size_t n = agents.size();
        std::vector<std::int32_t> x(n ? n : 1), y(n ? n : 1), v(n ? n : 1);
        std::vector<std::uint8_t> a(n ? n : 1);
        for (std::size_t i = 0; i < n; ++i) {
            x[i] = agents[i].pos.x;
            y[i] = agents[i].pos.y;
            v[i] = agents[i].v_max;
            a[i] = agents[i].alive ? 1 : 0;
        }
        x.resize(n), y.resize(n), v.resize(n), a.resize(n);
        if (v != m.v || m.x.size() != n) {
            for (std::int32_t vi : v)
                if (vi < kMinVmax || vi > kMaxVmax) throw std::invalid_argument("make_state: v_max must be in [1,5]");
            b200::check(fp_set_agents(m.ctx, static_cast<std::uint32_t>(n), x.data(), y.data(), v.data(), a.data(),
                                      step),
                        m.ctx);
        } else if (x != m.x || y != m.y || a != m.alive) {
            b200::check(fp_update_agents(m.ctx, x.data(), y.data(), a.data()), m.ctx);
        }
        m.x = std::move(x), m.y = std::move(y), m.v = std::move(v), m.alive = std::move(a);
        if (m.step != step) {
            b200::check(fp_set_step(m.ctx, step), m.ctx);
            m.step = step;
        }
        if (m.potential != static_cast<int>(potential) || m.gradient != drive_gradient) {
            b200::check(fp_set_potential(m.ctx, static_cast<int>(potential), drive_gradient), m.ctx);
            m.potential = static_cast<int>(potential);
            m.gradient = drive_gradient;
        }
        if (with_desired && n) {
            std::vector<std::int32_t> dx(n), dy(n);
            for (std::size_t i = 0; i < n; ++i) dx[i] = desired[i].x, dy[i] = desired[i].y;
            b200::check(fp_set_desired(m.ctx, dx.data(), dy.data()), m.ctx);
        }
        return m.ctx;
    }

    /// The strip set for `gpus` x-strips (rank r on device (device() + r) % device count; one
    /// GPU gives virtual strips), loaded with the host state.  Rebuilt when the count changes.
    fp_ctx* const* strips_for(int gpus) const {
        b200::Mirror& m = *dev;
        if ((int)m.strips.size() != gpus) {
            m.drop_strips();
            const fp_grid_desc d = b200::desc_of(*grid);
            const std::vector<std::uint8_t> cells = b200::cells_of(*grid);
            int ndev = 1;
            if (fp_device_count(&ndev) != FP_OK || ndev < 1) ndev = 1;
            for (int r = 0; r < gpus; ++r) {
                fp_ctx* c = nullptr;
                b200::check(fp_create(&d, cells.data(), field->s.data(), (b200::device() + r) % ndev, &c));
                m.strips.push_back(c);
                std::int32_t lo = 0, hi = 0;
                b200::check(fp_strip_bounds(grid->width(), r, gpus, &lo, &hi));
                const std::size_t n = agents.size();
                std::vector<std::int32_t> x(n ? n : 1), y(n ? n : 1), v(n ? n : 1);
                std::vector<std::uint8_t> a(n ? n : 1);
                for (std::size_t i = 0; i < n; ++i) {
                    x[i] = agents[i].pos.x, y[i] = agents[i].pos.y, v[i] = agents[i].v_max;
                    a[i] = agents[i].alive ? 1 : 0;
                }
                b200::check(fp_set_agents(c, static_cast<std::uint32_t>(n), x.data(), y.data(), v.data(), a.data(), step), c);
                b200::check(fp_strip_config(c, r, gpus, lo, hi, 0, 0), c);
            }
        }
        // the host state (the reference's authoritative fields) onto every rank
        const std::size_t n = agents.size();
        std::vector<std::int32_t> x(n ? n : 1), y(n ? n : 1), v(n ? n : 1);
        std::vector<std::uint8_t> a(n ? n : 1);
        for (std::size_t i = 0; i < n; ++i) {
            x[i] = agents[i].pos.x, y[i] = agents[i].pos.y, v[i] = agents[i].v_max;
            a[i] = agents[i].alive ? 1 : 0;
        }
        for (fp_ctx* c : m.strips) {
            b200::check(fp_set_agents(c, static_cast<std::uint32_t>(n), x.data(), y.data(), v.data(), a.data(), step), c);
            b200::check(fp_set_potential(c, static_cast<int>(potential), drive_gradient), c);
        }
        return m.strips.data();
    }

    /// Strip ranks -> host: every agent from the rank that owns it, occupancy, counters.
    void pull_strips() {
        b200::Mirror& m = *dev;
        const std::size_t n = agents.size();
        std::vector<std::int32_t> x(n ? n : 1), y(n ? n : 1);
        std::vector<std::uint8_t> a(n ? n : 1), o(n ? n : 1);
        for (std::size_t r = 0; r < m.strips.size(); ++r) {
            fp_ctx* c = m.strips[r];
            b200::check(fp_get_agents(c, x.data(), y.data(), a.data()), c);
            b200::check(fp_strip_get_owned(c, o.data()), c);
            // rank 0 first for everyone (agents nobody owns -- exited in a resolved walk, or dead from
            // the start -- are identical on every rank), then each agent from the rank owning it
            for (std::size_t i = 0; i < n; ++i)
                if (r == 0 || o[i]) {
                    agents[i].pos = Cell{x[i], y[i]};
                    agents[i].alive = a[i] != 0;
                }
        }
        occupancy.assign(static_cast<std::size_t>(grid->width()) * grid->height(), kEmpty);
        for (std::size_t i = 0; i < n; ++i)
            if (agents[i].alive) occupancy[grid->index(grid->normalize(agents[i].pos))] = static_cast<std::int32_t>(i);
        b200::check(fp_get_alive_count(m.strips[0], &alive), m.strips[0]);
        b200::check(fp_get_step(m.strips[0], &step), m.strips[0]);
        m.step = -1;  // the single-device mirror is stale now
        m.x.clear();
    }

    /// Device -> host: desired cells only (after plan_phase).
    void pull_desired() {
        const std::size_t n = agents.size();
        if (!n) return;
        std::vector<std::int32_t> dx(n), dy(n);
        b200::check(fp_get_desired(dev->ctx, dx.data(), dy.data()), dev->ctx);
        for (std::size_t i = 0; i < n; ++i) desired[i] = Cell{dx[i], dy[i]};
    }

    /// Device -> host after a motion phase: positions, alive flags, occupancy, counters, step.
    void pull_agents() {
        b200::Mirror& m = *dev;
        const std::size_t n = agents.size();
        for (std::size_t i = 0; i < n; ++i)  // clear the cells the uploaded roster held
            if (m.alive[i]) {
                std::int32_t& o = occupancy[grid->index(grid->normalize(Cell{m.x[i], m.y[i]}))];
                if (o == static_cast<std::int32_t>(i)) o = kEmpty;
            }
        if (n) b200::check(fp_get_agents(m.ctx, m.x.data(), m.y.data(), m.alive.data()), m.ctx);
        for (std::size_t i = 0; i < n; ++i) {
            agents[i].pos = Cell{m.x[i], m.y[i]};
            agents[i].alive = m.alive[i] != 0;
            if (m.alive[i]) occupancy[grid->index(grid->normalize(agents[i].pos))] = static_cast<std::int32_t>(i);
        }
        b200::check(fp_get_alive_count(m.ctx, &alive), m.ctx);
        b200::check(fp_get_step(m.ctx, &m.step), m.ctx);
        step = m.step;
    }
};

/// make_state(grid, field, roster) -- state.hpp:38-76: the reference's checks and messages, then
/// the device upload (grid bitplanes, the given field, the roster).
inline SimState make_state(std::shared_ptr<const Grid> grid, std::shared_ptr<const StaticField> field,
                           std::vector<Agent> roster) {
    if (!grid || !field) throw std::invalid_argument("make_state: grid and field required");
    if (field->width != grid->width() || field->height != grid->height() ||
        field->s.size() != static_cast<std::size_t>(grid->width()) * static_cast<std::size_t>(grid->height()))
        throw std::invalid_argument("make_state: field dimensions do not match grid");
    SimState st;
    st.grid = std::move(grid);
    st.field = std::move(field);
    st.agents = std::move(roster);
    st.occupancy.assign(static_cast<std::size_t>(st.grid->width()) * st.grid->height(), SimState::kEmpty);
    st.desired.resize(st.agents.size());
    for (std::size_t i = 0; i < st.agents.size(); ++i) {
        const Agent& a = st.agents[i];
        if (a.id != i) throw std::invalid_argument("make_state: agent ids must be dense indices from 0");
        if (a.v_max != st.agents.front().v_max) throw std::invalid_argument("make_state: all agents must share one v_max");
        if (a.v_max < kMinVmax || a.v_max > kMaxVmax) throw std::invalid_argument("make_state: v_max must be in [1,5]");
        if (!a.alive) continue;
        if (!st.grid->in_bounds(a.pos))
            throw std::invalid_argument("make_state: agent " + std::to_string(a.id) + " is out of bounds");
        if (st.grid->is_wall(a.pos))
            throw std::invalid_argument("make_state: agent " + std::to_string(a.id) + " placed on a Wall cell");
        std::int32_t& slot = st.occupancy[st.grid->index(st.grid->normalize(a.pos))];
        if (slot != SimState::kEmpty)
            throw std::invalid_argument("make_state: agents " + std::to_string(slot) + " and " + std::to_string(a.id) +
                                        " share a cell");
        slot = static_cast<std::int32_t>(i);
        st.desired[i] = a.pos;
        ++st.alive;
    }
    st.dev = std::make_shared<b200::Mirror>();
    const fp_grid_desc d = b200::desc_of(*st.grid);
    const std::vector<std::uint8_t> cells = b200::cells_of(*st.grid);
    b200::check(fp_create(&d, cells.data(), st.field->s.data(), b200::device(), &st.dev->ctx));
    st.sync_to_device();
    return st;
}

/// state_hash(st) -- state.hpp:80-95 (FNV-1a over step, alive, then id/x/y/alive per agent) of the
/// host fields, which are the state between calls.
inline std::uint64_t state_hash(const SimState& st) {
    std::uint64_t h = 14695981039346656037ULL;
    const auto mix = [&h](std::uint64_t v) {
        h ^= v;
        h *= 1099511628211ULL;
    };
    mix(static_cast<std::uint64_t>(st.step));
    mix(static_cast<std::uint64_t>(st.alive));
    for (const Agent& a : st.agents) {
        mix(a.id);
        mix(static_cast<std::uint32_t>(a.pos.x));
        mix(static_cast<std::uint32_t>(a.pos.y));
        mix(a.alive ? 1 : 0);
    }
    return h;
}

}  // namespace fastped
