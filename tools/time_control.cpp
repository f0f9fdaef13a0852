// Times the control plane's simulate() on a config (event log off), best of N --
// the same measurement oracle/ref_capture.cpp's `time` mode makes of the reference
// (SURVEY 8(f)-2). Build: see tools/time_control.sh.
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "../paper_2507_00507_b200/csrc/control/experiment.hpp"

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: time_control <config.json> [reps]\n");
        return 2;
    }
    const int reps = argc > 2 ? std::atoi(argv[2]) : 5;
    mesh::ExperimentConfig cfg = mesh::load_config(argv[1], {"output.event_log=false"}, std::nullopt, "/tmp/time_control_out");
    double best = 1e30;
    long long tokens = 0;
    for (int i = 0; i < reps; ++i) {
        const auto t0 = std::chrono::steady_clock::now();
        mesh::RunResult r = mesh::simulate(cfg, cfg.policy.kind);
        const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (s < best) best = s;
        tokens = r.summary.output_tokens;
    }
    std::printf("{\"best_s\": %.6f, \"tokens\": %lld}\n", best, tokens);
    return 0;
}
