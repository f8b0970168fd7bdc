// The reference's C++ API through the drop-in overlay, with ScheduleParams::gpus > 1 (x strips,
// one context per GPU driven from this thread; one GPU gives virtual strips): every step's
// state_hash and exit list must equal the gpus = 1 run.  Uses the reference's own make_plaza,
// make_scenario and spawn_agents (scenario_io.hpp).  Prints "ok <steps>" or the first mismatch.
#include <cstdio>
#include <cstdlib>

#include "fastped/fastped.hpp"

using namespace fastped;

int main(int argc, char** argv) {
    const int gpus = argc > 1 ? std::atoi(argv[1]) : 3;
    const int steps = argc > 2 ? std::atoi(argv[2]) : 40;
    const Scenario sc = make_scenario("plaza80", make_plaza(80.0, 4));  // 200 x 200 cells
    SimParams params;
    params.seed = 7;
    auto roster = spawn_agents(*sc.grid, 6000, 4, params.seed);
    SimState one = make_state(sc, roster);
    SimState many = make_state(sc, roster);
    for (int s = 0; s < steps; ++s) {
        const StepStats a = step(one, params, ScheduleParams{1, 1});
        const StepStats b = step(many, params, ScheduleParams{1, gpus});
        if (a.alive != b.alive || a.exited != b.exited || a.displacement_cells != b.displacement_cells ||
            state_hash(one) != state_hash(many)) {
            std::printf("mismatch at step %d\n", s);
            return 1;
        }
    }
    params.steps = 30;
    const RunStats ra = run(one, params, ScheduleParams{1, 1});
    const RunStats rb = run(many, params, ScheduleParams{1, gpus});
    if (ra.exited != rb.exited || ra.displacement_cells != rb.displacement_cells || state_hash(one) != state_hash(many)) {
        std::printf("run mismatch\n");
        return 1;
    }
    std::printf("ok %d\n", steps + 30);
    return 0;
}
