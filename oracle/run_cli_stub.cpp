// TEST INFRASTRUCTURE ONLY — run_cli (cli.hpp:17) for the reference's
// acceptance binary, which calls it for criterion 11 (acceptance_main.cpp:464).
// The real cli.cpp needs the absent vendor/CLI11.hpp; only the `profile`
// subcommand is needed, implemented over the reference's own bench.cpp
// (read_bench_csv / compute_profile / write_profile_csv, as cli.cpp:291-298 does).
#include <cstdio>
#include <exception>
#include <string>
#include <vector>

#include "spgemm/bench.hpp"
#include "spgemm/cli.hpp"

namespace spgemm {

int run_cli(const std::vector<std::string>& args)
{
    if (args.empty() || args[0] != "profile")
        return kExitUsage;
    std::string in, out;
    int points = 50;
    for (size_t i = 1; i + 1 < args.size(); i += 2) {
        if (args[i] == "--in")
            in = args[i + 1];
        else if (args[i] == "--out")
            out = args[i + 1];
        else if (args[i] == "--points")
            points = std::stoi(args[i + 1]);
        else
            return kExitUsage;
    }
    if (in.empty() || out.empty() || points < 1)
        return kExitUsage;
    try {
        write_profile_csv(out, compute_profile(read_bench_csv(in), points));
    } catch (const std::exception& e) {
        std::fprintf(stderr, "%s\n", e.what());
        return kExitIo;
    }
    return kExitOk;
}

} // namespace spgemm
