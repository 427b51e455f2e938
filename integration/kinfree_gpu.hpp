/** \file kinfree_gpu.hpp
 * \brief Reference-side adapter: the B200 path behind the reference's own
 *   run_fixed_point signature.
 *
 * Drop this header into the reference tree (include/kinfree/) and link
 * libkf.so; then
 *
 *     RunHistory h = kinfree::gpu::run_fixed_point(cloud, ls, plan, cfg, &state);
 *
 * is a drop-in for kinfree::run_fixed_point (driver.hpp:104-106,
 * driver.cpp:188-282): same inputs (PointCloud, LsCoefficients, SweepPlan,
 * SolverConfig), same outputs (RunHistory with per-iteration residual/CL/CD/
 * seconds/counters, diverged + abort_reason, final state), same
 * precondition exceptions. The library rebuilds the split stencils and LS
 * weights from the cloud bit-identically (tests/test_ingestion.py) and adopts
 * the caller's colouring (plan.color_of), so the LU-SGS ordering is the
 * caller's. The evaluation tallies are added to the process-global
 * flux_counters() (counters.hpp:58) so run_case's rdp_report.csv is unchanged.
 *
 * n_parts > 1 runs the domain-decomposed solver (kf_create_partitioned): the
 * cloud is cut into n_parts angular wedges held on `device`, ghosts refreshed
 * between dependent stages; the RunHistory is the same contract (states are
 * bitwise the one-partition states, the residual sum is reassociated).
 * The one-process-per-GPU form is run_fixed_point_rank() below.
 */
#ifndef KINFREE_GPU_HPP
#define KINFREE_GPU_HPP

#include <stdexcept>
#include <string>
#include <vector>

#include "kf.h"
#include "kinfree/counters.hpp"
#include "kinfree/driver.hpp"

namespace kinfree::gpu {

namespace detail {

struct CloudHandle {
    kf_cloud* c = nullptr;
    ~CloudHandle() { kf_cloud_free(c); }
};
struct CtxHandle {
    kf_ctx* c = nullptr;
    ~CtxHandle() { kf_destroy(c); }
};

inline void throw_status(const kf_status& s)
{
    if (s.code == KF_CONFIG) throw std::invalid_argument(s.reason);
    throw std::runtime_error(s.reason);
}

}  // namespace detail

namespace detail {

inline RunHistory run_impl(const PointCloud& cloud, const SweepPlan& plan, const SolverConfig& config,
                           std::vector<Vec4>* final_state, int device, int n_parts, int rank,
                           const unsigned char* nccl_id)
{
    const int n = cloud.n();
    std::vector<int> kind(n), off(n + 1, 0), ids;
    for (int p = 0; p < n; ++p) {
        kind[p] = static_cast<int>(cloud.kind[p]);
        off[p + 1] = off[p] + static_cast<int>(cloud.nbr[p].size());
        ids.insert(ids.end(), cloud.nbr[p].begin(), cloud.nbr[p].end());
    }
    CloudHandle ch;
    kf_status s = kf_cloud_from_arrays(n, cloud.x.data(), cloud.y.data(), kind.data(),
                                       cloud.normal_x.data(), cloud.normal_y.data(), off.data(),
                                       ids.data(), &ch.c);
    if (s.code) throw_status(s);
    if (static_cast<int>(plan.color_of.size()) == n) {
        s = kf_cloud_set_colors(ch.c, plan.color_of.data());
        if (s.code) throw_status(s);
    }

    kf_config cfg;
    kf_config_default(&cfg);
    cfg.variant = static_cast<int>(config.variant);
    cfg.cfl = config.cfl;
    cfg.n_iterations = config.n_iterations;
    cfg.n_inner = config.n_inner;
    cfg.mach_inf = config.mach_inf;
    cfg.aoa_deg = config.aoa_deg;
    cfg.convergence_decades = config.convergence_decades;
    cfg.bc_mode = config.bc_mode == BcMode::Physical ? 0 : 1;
    cfg.cfl_ramp_iters = config.cfl_ramp_iters;
    cfg.cfl_start = config.cfl_start;
    cfg.divergence_factor = config.divergence_factor;
    cfg.device = device;

    CtxHandle ctx;
    if (nccl_id)
        s = kf_create_rank(ch.c, &cfg, n_parts, rank, KF_PART_ANGULAR, nccl_id, &ctx.c);
    else if (n_parts > 1)
        s = kf_create_partitioned(ch.c, &cfg, n_parts, KF_PART_ANGULAR, &ctx.c);
    else
        s = kf_create(ch.c, &cfg, &ctx.c);
    if (s.code) throw_status(s);  // same precondition errors as driver.cpp:194-201

    std::vector<kf_iter_record> rec(std::max(config.n_iterations, 1));
    std::vector<double> state(final_state ? 4 * static_cast<size_t>(n) : 0);
    if (final_state && static_cast<int>(final_state->size()) == n)  // rank runs keep non-owned entries
        for (int p = 0; p < n; ++p)
            for (int j = 0; j < 4; ++j) state[4 * static_cast<size_t>(p) + j] = (*final_state)[p][j];
    int done = 0;
    double loop_seconds = 0.0;
    s = kf_run(ctx.c, rec.data(), &done, final_state ? state.data() : nullptr, &loop_seconds);
    if (s.code && s.code != KF_DIVERGED) throw_status(s);

    RunHistory h;
    h.points = n;
    h.loop_seconds = loop_seconds;
    h.diverged = s.code == KF_DIVERGED;
    if (h.diverged) h.abort_reason = s.reason;
    const EvalSnapshot base = flux_counters().snapshot();
    uint64_t prev[kNumEvalKinds] = {0, 0, 0, 0, 0};
    for (int k = 0; k < done; ++k) {
        IterationRecord r{};
        r.residual = rec[k].residual;
        r.cl = rec[k].cl;
        r.cd = rec[k].cd;
        r.seconds = rec[k].seconds;
        r.first_order_points = rec[k].first_order_points;
        for (int j = 0; j < kNumEvalKinds; ++j) {
            flux_counters().add(static_cast<EvalKind>(j), rec[k].counters[j] - prev[j]);
            prev[j] = rec[k].counters[j];
            r.sweep.n[j] = rec[k].sweep[j];
            r.counters.n[j] = base.n[j] + rec[k].counters[j];
        }
        h.iters.push_back(r);
    }
    if (final_state) {
        final_state->resize(n);
        for (int p = 0; p < n; ++p)
            for (int j = 0; j < 4; ++j) (*final_state)[p][j] = state[4 * static_cast<size_t>(p) + j];
    }
    return h;
}

}  // namespace detail

inline RunHistory run_fixed_point(const PointCloud& cloud, const LsCoefficients& ls,
                                  const SweepPlan& plan, const SolverConfig& config,
                                  std::vector<Vec4>* final_state, int device = 0, int n_parts = 1)
{
    (void)ls;  // rebuilt on the library side, bit-identically
    return detail::run_impl(cloud, plan, config, final_state, device, n_parts, 0, nullptr);
}

/// One process per GPU (e.g. under MPI): every rank calls this with the same
/// cloud/plan/config and the same NCCL id (rank 0: kf_nccl_unique_id, then
/// MPI_Bcast of KF_NCCL_ID_BYTES bytes). Every rank gets the full RunHistory;
/// *final_state receives this rank's owned points (other entries untouched:
/// gather them with MPI if the whole state is needed).
inline RunHistory run_fixed_point_rank(const PointCloud& cloud, const SweepPlan& plan,
                                       const SolverConfig& config, std::vector<Vec4>* final_state,
                                       int device, int n_ranks, int rank, const unsigned char* nccl_id)
{
    if (final_state) final_state->resize(cloud.n());
    return detail::run_impl(cloud, plan, config, final_state, device, n_ranks, rank, nccl_id);
}

}  // namespace kinfree::gpu

#endif
