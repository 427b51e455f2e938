// Drop-in demonstration: the reference's own run_case flow (caseio.cpp:255-283
// minus the CSV writers) with run_fixed_point swapped for the B200 adapter.
// Linked against the UNMODIFIED reference objects (oracle/_ref/obj) and
// libkf.so by integration/Makefile. Runs the same case through both and
// prints one JSON line comparing the two RunHistory records.
//
//   run_case_gpu <n_wall> <n_radial> <radius> <variant> <mach> <aoa> <cfl> <iters> [n_parts]
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "kinfree/caseio.hpp"
#include "kinfree/coloring.hpp"
#include "kinfree/driver.hpp"
#include "kinfree/spatial.hpp"
#include "kinfree_gpu.hpp"

using namespace kinfree;

int main(int argc, char** argv)
{
    if (argc < 9) {
        std::fprintf(stderr, "usage: %s n_wall n_radial radius variant mach aoa cfl iters\n", argv[0]);
        return 3;
    }
    const PointCloud cloud = generate_naca_ogrid("0012", std::atoi(argv[1]), std::atoi(argv[2]),
                                                 std::atof(argv[3]));
    const ColorAssignment colors = color_points(cloud);
    const SweepPlan plan = build_sweep_plan(colors);
    const LsCoefficients ls = build_ls_coefficients(cloud);
    SolverConfig cfg;
    cfg.variant = parse_variant(argv[4]);
    cfg.mach_inf = std::atof(argv[5]);
    cfg.aoa_deg = std::atof(argv[6]);
    cfg.cfl = std::atof(argv[7]);
    cfg.n_iterations = std::atoi(argv[8]);

    std::vector<Vec4> s_cpu, s_gpu;
    const RunHistory a = run_fixed_point(cloud, ls, plan, cfg, &s_cpu);
    const int n_parts = argc > 9 ? std::atoi(argv[9]) : 1;
    const RunHistory b = gpu::run_fixed_point(cloud, ls, plan, cfg, &s_gpu, 0, n_parts);

    double max_rel = 0.0, max_cl = 0.0, max_state = 0.0, state_scale = 0.0;
    const size_t m = std::min(a.iters.size(), b.iters.size());
    for (size_t k = 0; k < m; ++k) {
        max_rel = std::max(max_rel, std::fabs(a.iters[k].residual - b.iters[k].residual) /
                                        std::fabs(a.iters[k].residual));
        max_cl = std::max(max_cl, std::fabs(a.iters[k].cl - b.iters[k].cl));
        max_cl = std::max(max_cl, std::fabs(a.iters[k].cd - b.iters[k].cd));
    }
    bool sweep_equal = true;
    for (size_t k = 0; k < m; ++k)
        for (int j = 0; j < kNumEvalKinds; ++j)
            sweep_equal = sweep_equal && a.iters[k].sweep.n[j] == b.iters[k].sweep.n[j];
    for (size_t p = 0; p < s_cpu.size() && p < s_gpu.size(); ++p)
        for (int j = 0; j < 4; ++j) {
            max_state = std::max(max_state, std::fabs(s_cpu[p][j] - s_gpu[p][j]));
            state_scale = std::max(state_scale, std::fabs(s_cpu[p][j]));
        }
    double cpu_t = 0.0, gpu_t = 0.0;
    for (size_t k = 1; k < a.iters.size(); ++k) cpu_t += a.iters[k].seconds;
    for (size_t k = 1; k < b.iters.size(); ++k) gpu_t += b.iters[k].seconds;
    std::printf(
        "{\"points\": %d, \"iters_cpu\": %zu, \"iters_gpu\": %zu, \"diverged_cpu\": %s, "
        "\"diverged_gpu\": %s, \"reason_cpu\": \"%s\", \"reason_gpu\": \"%s\", "
        "\"max_rel_residual\": %.3e, \"max_abs_clcd\": %.3e, \"state_normrel\": %.3e, "
        "\"sweep_counters_equal\": %s, \"cpu_s_per_iter\": %.6e, \"gpu_s_per_iter\": %.6e}\n",
        cloud.n(), a.iters.size(), b.iters.size(), a.diverged ? "true" : "false",
        b.diverged ? "true" : "false", a.abort_reason.c_str(), b.abort_reason.c_str(), max_rel, max_cl,
        state_scale > 0 ? max_state / state_scale : max_state, sweep_equal ? "true" : "false",
        a.iters.size() > 1 ? cpu_t / (a.iters.size() - 1) : 0.0,
        b.iters.size() > 1 ? gpu_t / (b.iters.size() - 1) : 0.0);
    const bool ok = a.iters.size() == b.iters.size() && a.diverged == b.diverged &&
                    a.abort_reason == b.abort_reason && max_rel <= 1e-10 && max_cl <= 1e-10 &&
                    sweep_equal;
    return ok ? 0 : 1;
}
