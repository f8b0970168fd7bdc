// Drop-in replacement of fastped/planning.hpp (/root/reference/proj/include/fastped/planning.hpp).
//
// The two per-agent entry points run on the device against the SimState's occupancy snapshot
// (the caller's host edits are uploaded first):
//   enumerate_candidates(st, agent)           planning.hpp:23-57  -> fp_enumerate_candidates
//   choose_desired_cell(st, agent, params)    planning.hpp:88-108 -> fp_choose_desired (exact
//       fp64 path: restated glibc exp, serial sum and scan -- bitwise the reference's choice)
// The scalar helpers stay host arithmetic with the reference's semantics:
//   detail::sample_index    planning.hpp:63-73 (first cumulative weight > u*total, else the tail)
//   detail::potential_drop  planning.hpp:76-80
// Whole-roster planning is plan_phase (engine.hpp overlay), one kernel launch per step.
#pragma once

#include <cmath>
#include <cstdint>
#include <span>
#include <vector>

#include "fastped/rng.hpp"
#include "fastped/state.hpp"

namespace fastped {

inline std::vector<Cell> enumerate_candidates(const SimState& st, const Agent& agent) {
    fp_ctx* ctx = st.sync_to_device();
    std::int32_t cx[128], cy[128];
    std::uint32_t n = 0;
    b200::check(fp_enumerate_candidates(ctx, agent.pos.x, agent.pos.y, agent.v_max, cx, cy, 128, &n), ctx);
    std::vector<Cell> out(n);
    for (std::uint32_t i = 0; i < n; ++i) out[i] = Cell{cx[i], cy[i]};
    return out;
}

namespace detail {

inline std::size_t sample_index(std::span<const double> weights, double u) {
    double total = 0.0;
    for (const double w : weights) total += w;
    const double threshold = u * total;
    double cum = 0.0;
    for (std::size_t i = 0; i < weights.size(); ++i) {
        cum += weights[i];
        if (cum > threshold) return i;
    }
    return weights.size() - 1;
}

inline double potential_drop(const SimState& st, Cell from, Cell to) {
    if (st.potential == Potential::DriveX) return st.drive_gradient * segment_dx(*st.grid, from, to);
    return st.field->at(from) - st.field->at(to);
}

}  // namespace detail

inline Cell choose_desired_cell(const SimState& st, const Agent& agent, const SimParams& params) {
    fp_ctx* ctx = st.sync_to_device();
    std::int32_t x = 0, y = 0;
    b200::check(fp_choose_desired(ctx, agent.id, agent.pos.x, agent.pos.y, agent.v_max, st.step, params.k_s,
                                  params.seed, &x, &y),
                ctx);
    return Cell{x, y};
}

}  // namespace fastped
