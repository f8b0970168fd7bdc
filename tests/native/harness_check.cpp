// Exercises the C++ harness drop-in (include/fastped_b200/harness.hpp) the way the reference's
// own tests call bench.hpp / scenario_io.hpp / world.hpp: prints results for tests/test_cpp_api.py.
// With "--host" it runs only the host-side parts (no GPU needed).
#include <cstdio>
#include <cstring>
#include <stdexcept>

#include "fastped_b200/harness.hpp"

using namespace fastped_b200;

int main(int argc, char** argv) {
    const bool host_only = argc > 1 && std::strcmp(argv[1], "--host") == 0;
    const std::string tiny = "FAST-SCENARIO v1\nwidth 5\nheight 4\ncell_size 0.4\nboundary periodic-x\ngrid:\n"
                             "#####\n.....\n.....\n#####\n";
    std::printf("roundtrip %d\n", serialize_scenario(parse_scenario(tiny)) == tiny ? 1 : 0);
    try {
        parse_scenario("FAST-SCENARIO v2\n");
    } catch (const std::runtime_error& e) {
        std::printf("error %s\n", e.what());
    }
    std::printf("%s", to_csv(std::vector<RunRecord>{{"plaza", 1000, 4, 8, 396, 1.5, 1.25, 0.125, 42}}).c_str());
    std::printf("%s", to_csv(std::vector<SpeedupRow>{{"syn", 10, 4, 2, 0.5, 1.23456}}).c_str());
    std::printf("%s", to_csv(std::vector<FdRecord>{{0.5, 1.6, 0.8}}).c_str());
    std::printf("weidmann %.17g %.17g\n", weidmann_speed(1.0), weidmann_speed(3.0));
    const auto cap = realtime_capacity([](std::int64_t n) { return 0.002 * n; }, 396.0);
    std::printf("capacity %lld %lld %lld\n", (long long)cap.capacity, (long long)cap.n_low, (long long)cap.n_high);
    if (host_only) return 0;
    const Grid corridor = parse_scenario(
        "FAST-SCENARIO v1\nwidth 25\nheight 5\ncell_size 0.4\nboundary periodic-x\ngrid:\n"
        "#########################\n.........................\n.........................\n"
        ".........................\n#########################\n");
    const auto fd = fundamental_diagram(corridor, 4, {0.5, 1.0, 2.0, 4.0}, 9, 50, 120);
    for (const FdRecord& r : fd) std::printf("fd %.17g %.17g %.17g\n", r.density, r.mean_speed, r.flow);
    return 0;
}
