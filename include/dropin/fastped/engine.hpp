// Drop-in replacement of fastped/engine.hpp (/root/reference/proj/include/fastped/engine.hpp):
// the two-phase time step on a B200 through libfastped_b200's C ABI.
//
//   ScheduleParams{cores, gpus}   engine.hpp:21-23 -- `cores` is kept and validated (< 1 throws,
//                                 as in the reference) but never changes results, exactly like
//                                 the reference's; `gpus` (not in the reference) is the x-strip
//                                 count of the multi-GPU path: step / run with
//                                 gpus > 1 drive one strip context per GPU from this thread
//                                 (rank r on device r; one GPU gives virtual strips), results
//                                 bit-identical to gpus = 1
//   compute_blocksize             engine.hpp:27-33 (host arithmetic, pinned vectors)
//   plan_phase                    engine.hpp:71-84  -> fp_plan   (desired cells synced back)
//   move_phase / MoveOutcome      engine.hpp:86-135 -> fp_move   (positions, exits in processing
//                                 order, occupancy synced back)
//   step / StepStats              engine.hpp:137-148 -> fp_step  (CUDA-graph replay)
//   run / RunStats                engine.hpp:150-183 -> fp_run   (device loop timed with CUDA
//                                 events between phases; one sync at the end)
// Host sync policy: plan_phase / move_phase / step copy the state back after every call so the
// host fields are current, as the reference's callers expect; run() copies once at the end.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <utility>
#include <vector>

#include "fastped/planning.hpp"
#include "fastped/rng.hpp"
#include "fastped/state.hpp"

namespace fastped {

struct ScheduleParams {
    int cores = 1;  // validated only: results never depend on it (as in the reference)
    int gpus = 1;   // x strips, one B200 each (fp_strips_step / fp_strips_run); 1 = one device
};

inline int compute_blocksize(std::int64_t number_of_agents, int cores) {
    std::int32_t b = 0;
    b200::check(fp_compute_blocksize(number_of_agents, cores, &b));
    return b;
}

namespace b200 {
inline void check_sched(const ScheduleParams& sched, const char* who) {
    if (sched.cores < 1) throw std::invalid_argument(std::string(who) + ": cores must be >= 1");
    if (sched.gpus < 1) throw std::invalid_argument(std::string(who) + ": gpus must be >= 1");
}
inline void whole_steps_only(const ScheduleParams& sched, const char* who) {
    if (sched.gpus != 1)
        throw std::invalid_argument(std::string(who) +
                                    ": with gpus > 1 the strip engine runs whole steps (step / run)");
}
}  // namespace b200

inline void plan_phase(SimState& st, const SimParams& params, const ScheduleParams& sched) {
    b200::check_sched(sched, "plan_phase");
    b200::whole_steps_only(sched, "plan_phase");
    if (st.alive == 0) return;
    fp_ctx* ctx = st.sync_to_device();
    b200::check(fp_plan(ctx, params.k_s, params.seed), ctx);
    st.pull_desired();
}

struct MoveOutcome {
    std::vector<std::uint32_t> exited;    // ids, in processing order
    std::int64_t displacement_cells = 0;  // total hops walked this step
};

inline MoveOutcome move_phase(SimState& st, const SimParams& params) {
    fp_ctx* ctx = st.sync_to_device(/*with_desired=*/true);
    fp_step_stats s{};
    b200::check(fp_move(ctx, params.seed, &s), ctx);
    MoveOutcome out;
    out.displacement_cells = s.displacement_cells;
    out.exited.resize(static_cast<std::size_t>(s.exited));
    std::uint32_t n = 0;
    if (s.exited) b200::check(fp_get_exited(ctx, out.exited.data(), static_cast<std::uint32_t>(s.exited), &n), ctx);
    st.pull_agents();
    return out;
}

struct StepStats {
    std::int64_t alive = 0;
    std::int64_t exited = 0;
    std::int64_t displacement_cells = 0;
};

inline StepStats step(SimState& st, const SimParams& params, const ScheduleParams& sched) {
    b200::check_sched(sched, "plan_phase");
    if (sched.gpus > 1) {  // x strips, one context per GPU, driven from this thread (fp_strips_step)
        fp_ctx* const* cs = st.strips_for(sched.gpus);
        fp_step_stats s{};
        b200::check(fp_strips_step(cs, sched.gpus, params.k_s, params.seed, &s), cs[0]);
        st.pull_strips();
        return {s.alive, s.exited, s.displacement_cells};
    }
    fp_ctx* ctx = st.sync_to_device();
    fp_step_stats s{};
    b200::check(fp_step(ctx, params.k_s, params.seed, &s), ctx);
    st.pull_agents();
    st.pull_desired();
    return {s.alive, s.exited, s.displacement_cells};
}

struct RunStats {
    double wall_time_s = 0.0;  // stepping loop only; setup excluded (CUDA events)
    double plan_time_s = 0.0;
    double move_time_s = 0.0;
    std::int64_t steps = 0;
    std::int64_t exited = 0;
    std::int64_t displacement_cells = 0;
    std::int64_t alive = 0;
};

inline RunStats run(SimState& st, const SimParams& params, const ScheduleParams& sched) {
    params.validate();
    if (sched.cores < 1) throw std::invalid_argument("run: cores must be >= 1");
    b200::check_sched(sched, "run");
    if (sched.gpus > 1) {  // x strips (fp_strips_run): time = max over the ranks' CUDA events
        fp_ctx* const* cs = st.strips_for(sched.gpus);
        fp_run_stats r{};
        b200::check(fp_strips_run(cs, sched.gpus, params.k_s, params.seed, params.steps, &r), cs[0]);
        st.pull_strips();
        return {r.wall_time_s, r.plan_time_s, r.move_time_s, r.steps, r.exited, r.displacement_cells, r.alive};
    }
    fp_ctx* ctx = st.sync_to_device();
    fp_run_stats r{};
    b200::check(fp_run(ctx, params.k_s, params.seed, params.steps, &r), ctx);
    st.pull_agents();
    st.pull_desired();
    return {r.wall_time_s, r.plan_time_s, r.move_time_s, r.steps, r.exited, r.displacement_cells, r.alive};
}

}  // namespace fastped
