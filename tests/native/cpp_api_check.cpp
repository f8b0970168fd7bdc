// Exercises the C++ drop-in (include/fastped_b200/fastped.hpp) the way a reference caller does:
// Grid -> spawn_agents -> make_state -> step()/plan_phase()/move_phase() -> state_hash, and the
// reference's exception behaviour.  Prints one line per step for tests/test_cpp_api.py.
#include <cstdio>
#include <cstdlib>
#include <stdexcept>

#include "fastped_b200/fastped.hpp"

using namespace fastped_b200;

int main(int argc, char** argv) {
    const int W = 40, H = 30, N = argc > 1 ? std::atoi(argv[1]) : 200, steps = 20;
    std::vector<CellKind> cells(static_cast<std::size_t>(W) * H, CellKind::Free);
    for (int x = 0; x < W; ++x) cells[x] = cells[(H - 1) * W + x] = CellKind::Wall;
    for (int y = 0; y < H; ++y) cells[y * W] = cells[y * W + W - 1] = CellKind::Wall;
    for (int y = 12; y < 18; ++y) cells[y * W + W - 1] = CellKind::Exit;
    for (int y = 5; y < 25; ++y) cells[y * W + 20] = CellKind::Wall;  // a partition with gaps
    cells[10 * W + 20] = cells[20 * W + 20] = CellKind::Free;
    auto grid = std::make_shared<const Grid>(W, H, 0.4, Boundary::Closed, cells);

    // the reference's validation wording (world.hpp:37-63, agents.hpp:37-44, engine.hpp:72)
    int errors = 0;
    try { Grid(0, 3, 0.4, Boundary::Closed, {}); } catch (const std::invalid_argument&) { ++errors; }
    try { SimParams(1.2, 0.5, 4, 1, 10, 1.0); } catch (const std::invalid_argument&) { ++errors; }
    try { (void)compute_blocksize(10, 0); } catch (const std::invalid_argument&) { ++errors; }
    std::printf("errors %d\n", errors);
    std::printf("blocksize %d %d\n", compute_blocksize(100000, 8), compute_blocksize(500000, 2));

    auto roster = spawn_agents(*grid, N, 4, 7);
    SimState st = make_state(grid, nullptr, roster);
    std::printf("field %.17g\n", st.field->at({1, 1}));
    const SimParams p(1.2, 0.0, 4, 7, steps, 1.0);
    const ScheduleParams sched{4};
    for (int s = 0; s < steps; ++s) {
        StepStats ss;
        if (s % 2 == 0) {
            ss = step(st, p, sched);
        } else {  // the two phases separately, as the reference's acceptance tests call them
            plan_phase(st, p, sched);
            const MoveOutcome mo = move_phase(st, p);
            ++st.step;
            ss = {st.alive, static_cast<std::int64_t>(mo.exited.size()), mo.displacement_cells};
        }
        std::printf("step %lld alive %lld exited %lld disp %lld hash %llu\n", (long long)st.step,
                    (long long)ss.alive, (long long)ss.exited, (long long)ss.displacement_cells,
                    (unsigned long long)state_hash(st));
    }
    return 0;
}
