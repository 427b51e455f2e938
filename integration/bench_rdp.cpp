// The reference's `benchmark` path (caseio.cpp:285-326):
// every variant on one generated cloud through the reference's own run_case
// (CSV artifacts, rdp_report.csv, the incremental = 2 x exact sweep-counter
// check). Built twice by integration/Makefile from the UNMODIFIED reference
// objects: bench_rdp_cpu (reference run_fixed_point) and bench_rdp_gpu
// (caseio.cpp compiled with gpu_swap.hpp, so run_case calls the B200
// adapter). Prints one JSON line per run.
//
//   bench_rdp_{cpu,gpu} <n_wall> <n_radial> <radius> <mach> <aoa> <cfl> <iterations> <out_dir>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "kinfree/caseio.hpp"
#ifdef KF_BENCH_GPU
#include "kinfree_gpu.hpp"

namespace kinfree {
RunHistory gpu_run_fixed_point(const PointCloud& cloud, const LsCoefficients& ls, const SweepPlan& plan,
                               const SolverConfig& config, std::vector<Vec4>* final_state)
{
    return gpu::run_fixed_point(cloud, ls, plan, config, final_state);
}
}  // namespace kinfree
#endif

int main(int argc, char** argv)
{
    using namespace kinfree;
    if (argc < 9) {
        std::fprintf(stderr, "usage: %s n_wall n_radial radius mach aoa cfl iterations out_dir\n", argv[0]);
        return 3;
    }
    CaseFile c;
    c.cloud.generate = std::string("naca0012:") + argv[1] + ":" + argv[2] + ":" + argv[3];
    c.solver.mach_inf = std::atof(argv[4]);
    c.solver.aoa_deg = std::atof(argv[5]);
    c.solver.cfl = std::atof(argv[6]);
    c.solver.n_iterations = std::atoi(argv[7]);
    c.out_dir = argv[8];
    const std::vector<SolverVariant> vs = {SolverVariant::Explicit, SolverVariant::Anandh, SolverVariant::AnandhAD,
                                           SolverVariant::Manish, SolverVariant::ManishAD};
    const BenchResult r = benchmark(c, vs);
    std::printf("{\"counter_ratio_ok\": %s, \"reports\": [", r.counter_ratio_ok ? "true" : "false");
    for (size_t k = 0; k < r.reports.size(); ++k) {
        const RdpReport& p = r.reports[k];
        std::printf("%s{\"variant\": \"%s\", \"points\": %d, \"iterations\": %d, \"seconds\": %.6e, "
                    "\"split\": %llu, \"full\": %llu, \"erf\": %llu, \"jvp_split\": %llu, \"jvp_full\": %llu}",
                    k ? ", " : "", p.variant.c_str(), p.points, p.iterations, p.total_seconds,
                    (unsigned long long)p.counters.split_flux(), (unsigned long long)p.counters.full_flux(),
                    (unsigned long long)p.counters.erf(), (unsigned long long)p.counters.jvp_split(),
                    (unsigned long long)p.counters.jvp_full());
    }
    std::printf("]}\n");
    return r.counter_ratio_ok ? 0 : 1;
}
