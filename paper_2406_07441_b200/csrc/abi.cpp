// extern "C" boundary of libkf.so (include/kf.h). Converts C++ exceptions to
// kf_status records; nothing throws across this file.
#include <algorithm>
#include <cstdio>
#include <memory>
#include <vector>
#include <cstring>
#include <exception>
#include <string>

#include "../../include/kf.h"
#include "cloud.hpp"
#include "partition.hpp"
#include "solver.hpp"

struct kf_cloud {
    kfb::Cloud c;
};

struct kf_layout {
    kfb::LocalLayout L;
};

struct kf_ctx {
    std::unique_ptr<kfb::Solver> solver;
    kf_config cfg;
    int n = 0;
    // n_inner < 1 is not a precondition of run_fixed_point: q_derivatives
    // throws inside iteration 1's try block (spatial.cpp:154), so the run
    // returns diverged with that reason and no records (driver.cpp:255-262)
    bool bad_inner = false;
};

namespace {

kf_status ok()
{
    kf_status s;
    s.code = KF_OK;
    s.point = -1;
    s.iteration = 0;
    s.reason[0] = 0;
    return s;
}

kf_status err(int code, const std::string& msg, int point = -1, int iteration = 0)
{
    kf_status s;
    s.code = code;
    s.point = point;
    s.iteration = iteration;
    std::snprintf(s.reason, sizeof s.reason, "%s", msg.c_str());
    return s;
}

template <class F>
kf_status guarded(F&& f)
{
    try {
        return f();
    } catch (const kfb::SolverError& e) {
        return err(e.code, e.what(), e.point, e.iteration);
    } catch (const kfb::IngestError& e) {
        return err(e.kind == 1 ? KF_CONFIG : KF_RUNTIME, e.what());
    } catch (const std::bad_alloc&) {
        return err(KF_RUNTIME, "out of host memory");
    } catch (const std::exception& e) {
        return err(KF_RUNTIME, e.what());
    } catch (...) {
        return err(KF_RUNTIME, "unknown error");
    }
}

constexpr const char* kBadInner = "q_derivatives: n_inner must be >= 1";

kf_status bad_inner_status() { return err(KF_DIVERGED, kBadInner, -1, 1); }

const kfb::Csr& list_of(const kf_cloud* c, int which)
{
    if (which >= 1 && which <= 4) return c->c.split[which - 1];
    return c->c.nbr;
}

}  // namespace

extern "C" {

const char* kf_version(void) { return "kinfree-b200 0.1 (sm_100a)"; }

int kf_device_count(void) { return kfb::device_count(); }

kf_status kf_cloud_generate_naca(const char* digits, int n_wall, int n_radial,
                                 double far_field_radius, kf_cloud** out)
{
    return guarded([&] {
        *out = nullptr;
        auto* c = new kf_cloud;
        try {
            c->c = kfb::generate_naca_ogrid(digits ? digits : "", n_wall, n_radial, far_field_radius);
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
        return ok();
    });
}

kf_status kf_cloud_load(const char* path, kf_cloud** out)
{
    return guarded([&] {
        *out = nullptr;
        auto* c = new kf_cloud;
        try {
            c->c = kfb::load_cloud(path ? path : "");
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
        return ok();
    });
}

kf_status kf_cloud_save_binary(const kf_cloud* c, const char* path)
{
    return guarded([&] {
        kfb::save_cloud_binary(c->c, path ? path : "");
        return ok();
    });
}

kf_status kf_cloud_save(const kf_cloud* c, const char* path)
{
    return guarded([&] {
        kfb::save_cloud(c->c, path ? path : "");
        return ok();
    });
}

kf_status kf_cloud_from_arrays(int n, const double* x, const double* y, const int* kind,
                               const double* normal_x, const double* normal_y,
                               const int* nbr_offsets, const int* nbr_ids, kf_cloud** out)
{
    return guarded([&] {
        *out = nullptr;
        auto* c = new kf_cloud;
        try {
            c->c = kfb::cloud_from_arrays(n, x, y, kind, normal_x, normal_y, nbr_offsets, nbr_ids);
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
        return ok();
    });
}

void kf_cloud_free(kf_cloud* c) { delete c; }

int kf_cloud_n(const kf_cloud* c) { return c->c.n; }
int kf_cloud_n_colors(const kf_cloud* c) { return c->c.n_colors; }

kf_status kf_cloud_set_colors(kf_cloud* c, const int* color_of)
{
    return guarded([&] {
        const kfb::Cloud& cl = c->c;
        int nc = 0;
        for (int p = 0; p < cl.n; ++p) {
            if (color_of[p] < 1) return err(KF_CONFIG, "colours must be 1-based and positive");
            nc = std::max(nc, color_of[p]);
        }
        // a point may never share a colour with a neighbour in either
        // direction (coloring.hpp:5-7, validate_coloring coloring.cpp:64-73)
        for (int p = 0; p < cl.n; ++p)
            for (int k = cl.nbr.off[p]; k < cl.nbr.off[p + 1]; ++k) {
                const int q = cl.nbr.idx[k];
                if (q != p && color_of[q] == color_of[p])
                    return err(KF_CONFIG, "invalid colouring: points " + std::to_string(std::min(p, q)) +
                                              " and " + std::to_string(std::max(p, q)) +
                                              " are neighbours with the same colour");
            }
        c->c.color.assign(color_of, color_of + cl.n);
        c->c.n_colors = nc;
        return ok();
    });
}

kf_status kf_cloud_color_device(kf_cloud* c, int device, int mode, unsigned seed, int* n_colors, int* rounds)
{
    return guarded([&] {
        if (mode != KF_COLOR_JP_HASH && mode != KF_COLOR_JP_LDF) return err(KF_CONFIG, "unknown colouring mode");
        int r = 0;
        const int nc = kfb::jones_plassmann_colors(c->c, device, mode, seed, &r);
        if (n_colors) *n_colors = nc;
        if (rounds) *rounds = r;
        return ok();
    });
}

kf_status kf_cloud_order_wall_first(kf_cloud* c, int* n_levels)
{
    return guarded([&] {
        const int m = kfb::wall_first_levels(c->c);
        if (n_levels) *n_levels = m;
        return ok();
    });
}

void kf_cloud_geometry(const kf_cloud* c, double* x, double* y, int* kind, double* nx, double* ny)
{
    const kfb::Cloud& cl = c->c;
    for (int p = 0; p < cl.n; ++p) {
        if (x) x[p] = cl.x[p];
        if (y) y[p] = cl.y[p];
        if (kind) kind[p] = cl.kind[p];
        if (nx) nx[p] = cl.nx[p];
        if (ny) ny[p] = cl.ny[p];
    }
}

long kf_cloud_list_nnz(const kf_cloud* c, int which)
{
    return static_cast<long>(list_of(c, which).idx.size());
}

void kf_cloud_list(const kf_cloud* c, int which, int* offsets, int* ids)
{
    const kfb::Csr& L = list_of(c, which);
    std::memcpy(offsets, L.off.data(), L.off.size() * sizeof(int));
    if (!L.idx.empty()) std::memcpy(ids, L.idx.data(), L.idx.size() * sizeof(int));
}

void kf_cloud_ls_full(const kf_cloud* c, double* wx, double* wy, int* kinds)
{
    const kfb::Cloud& cl = c->c;
    if (!cl.wx.empty()) {
        std::memcpy(wx, cl.wx.data(), cl.wx.size() * sizeof(double));
        std::memcpy(wy, cl.wy.data(), cl.wy.size() * sizeof(double));
    }
    std::memcpy(kinds, cl.full_class.data(), cl.full_class.size() * sizeof(int));
}

void kf_cloud_ls_split(const kf_cloud* c, int which, double* w, double* ls_one, int* kinds)
{
    const kfb::Cloud& cl = c->c;
    const int s = which - 1;
    if (s < 0 || s > 3) return;
    if (!cl.split_w[s].empty())
        std::memcpy(w, cl.split_w[s].data(), cl.split_w[s].size() * sizeof(double));
    std::memcpy(ls_one, cl.ls_one[s].data(), cl.ls_one[s].size() * sizeof(double));
    std::memcpy(kinds, cl.split_class[s].data(), cl.split_class[s].size() * sizeof(int));
}

int kf_cloud_flagged(const kf_cloud* c, int* out)
{
    const auto& f = c->c.flagged;
    if (out && !f.empty()) std::memcpy(out, f.data(), f.size() * sizeof(int));
    return static_cast<int>(f.size());
}

void kf_cloud_colors(const kf_cloud* c, int* color)
{
    std::memcpy(color, c->c.color.data(), c->c.color.size() * sizeof(int));
}

void kf_cloud_report(const kf_cloud* c, int* empty, int* n_empty, int* singular, int* n_singular)
{
    const kfb::Cloud& cl = c->c;
    if (n_empty) *n_empty = static_cast<int>(cl.empty_points.size());
    if (n_singular) *n_singular = static_cast<int>(cl.singular_points.size());
    if (empty && !cl.empty_points.empty())
        std::memcpy(empty, cl.empty_points.data(), cl.empty_points.size() * sizeof(int));
    if (singular && !cl.singular_points.empty())
        std::memcpy(singular, cl.singular_points.data(), cl.singular_points.size() * sizeof(int));
}

void kf_config_default(kf_config* cfg)
{
    cfg->variant = KF_EXPLICIT;  // SolverConfig default, driver.hpp:38
    cfg->cfl = 0.2;
    cfg->n_iterations = 100;
    cfg->n_inner = 3;
    cfg->mach_inf = 0.63;
    cfg->aoa_deg = 0.0;
    cfg->convergence_decades = 0.0;
    cfg->bc_mode = 0;
    cfg->cfl_ramp_iters = 0;
    cfg->cfl_start = 0.0;
    cfg->divergence_factor = 1e6;
    cfg->device = 0;
    cfg->ordering = 1;
    cfg->use_graph = 1;
}

}  // extern "C"

namespace {

kf_status create_ctx(const kf_cloud* cloud, const kf_config* cfg, const kfb::PartitionSpec& spec,
                     kf_ctx** out)
{
    return guarded([&] {
        *out = nullptr;
        // run_fixed_point preconditions, driver.cpp:194-201
        if (!(cfg->cfl > 0.0)) return err(KF_CONFIG, "cfl must be positive");
        if (cfg->n_iterations < 1) return err(KF_CONFIG, "n_iterations must be >= 1");
        // the device abort key's field widths (kernels.cuh mkkey)
        if (cfg->n_iterations >= kfb::kMaxIterations)
            return err(KF_CONFIG, "n_iterations must be < " + std::to_string(kfb::kMaxIterations));
        if (cfg->variant < 0 || cfg->variant > 4) return err(KF_CONFIG, "unknown variant");
        if (spec.n_parts < 1) return err(KF_CONFIG, "n_parts must be >= 1");
        if (spec.mode != kfb::kPartAngular && spec.mode != kfb::kPartMorton)
            return err(KF_CONFIG, "unknown partition mode");
        const kfb::Cloud& c = cloud->c;
        if (c.n >= kfb::kMaxPoints)
            return err(KF_CONFIG, "clouds are limited to " + std::to_string(kfb::kMaxPoints) + " points");
        for (int p : c.flagged)
            if (c.kind[p] == kfb::kInterior)
                return err(KF_RUNTIME, "interior point " + std::to_string(p) +
                                           " has a singular least-squares stencil", p);
        if (!(cfg->mach_inf > 0.0)) return err(KF_CONFIG, "freestream Mach must be positive");
        auto* ctx = new kf_ctx;
        try {
            ctx->cfg = *cfg;
            ctx->n = c.n;
            ctx->bad_inner = cfg->n_inner < 1;
            kf_config scfg = *cfg;
            if (ctx->bad_inner) scfg.n_inner = 1;  // never iterated (see kf_ctx)
            ctx->solver.reset(new kfb::Solver(c, scfg, spec));
        } catch (...) {
            delete ctx;
            throw;
        }
        *out = ctx;
        return ok();
    });
}

}  // namespace

extern "C" {

kf_status kf_create(const kf_cloud* cloud, const kf_config* cfg, kf_ctx** out)
{
    return create_ctx(cloud, cfg, kfb::PartitionSpec(), out);
}

kf_status kf_create_partitioned(const kf_cloud* cloud, const kf_config* cfg, int n_parts, int mode,
                                kf_ctx** out)
{
    kfb::PartitionSpec spec;
    spec.n_parts = n_parts;
    spec.mode = mode;
    return create_ctx(cloud, cfg, spec, out);
}

kf_status kf_nccl_unique_id(unsigned char* id)
{
    return guarded([&] {
        kfb::nccl_unique_id(id);
        return ok();
    });
}

kf_status kf_create_rank(const kf_cloud* cloud, const kf_config* cfg, int n_ranks, int rank, int mode,
                         const unsigned char* nccl_id, kf_ctx** out)
{
    kfb::PartitionSpec spec;
    spec.n_parts = n_ranks;
    spec.mode = mode;
    spec.nccl = 1;  // also for n_ranks == 1: the NCCL transport with one rank
    spec.rank = rank;
    spec.nccl_id = nccl_id;
    if (!nccl_id) {
        *out = nullptr;
        return err(KF_CONFIG, "kf_create_rank: missing NCCL unique id");
    }
    if (n_ranks < 1 || rank < 0 || rank >= n_ranks) {
        *out = nullptr;
        return err(KF_CONFIG, "rank out of range");
    }
    return create_ctx(cloud, cfg, spec, out);
}

kf_status kf_create_rank_host(const kf_cloud* cloud, const kf_config* cfg, int n_ranks, int rank, int mode,
                              kf_exchange_fn exch, kf_allreduce_fn allreduce, void* user, kf_ctx** out)
{
    if (!exch || !allreduce) {
        *out = nullptr;
        return err(KF_CONFIG, "kf_create_rank_host: missing exchange or allreduce callback");
    }
    if (n_ranks < 1 || rank < 0 || rank >= n_ranks) {
        *out = nullptr;
        return err(KF_CONFIG, "rank out of range");
    }
    kfb::PartitionSpec spec;
    spec.n_parts = n_ranks;
    spec.mode = mode;
    spec.rank = rank;
    spec.host = 1;
    spec.exch = exch;
    spec.allreduce = allreduce;
    spec.user = user;
    return create_ctx(cloud, cfg, spec, out);
}

int kf_n_parts(const kf_ctx* ctx) { return ctx->solver->n_parts(); }
int kf_owned_points(const kf_ctx* ctx) { return ctx->solver->owned_points(); }

kf_status kf_partition_plan(const kf_cloud* c, int n_parts, int mode, int* owner)
{
    return guarded([&] {
        const std::vector<int> o = kfb::plan_partition(c->c, n_parts, mode);
        std::memcpy(owner, o.data(), o.size() * sizeof(int));
        return ok();
    });
}

kf_status kf_layout_build(const kf_cloud* c, const int* owner, int n_parts, int rank, int ordering,
                          kf_layout** out)
{
    return guarded([&] {
        *out = nullptr;
        std::vector<int> o(owner, owner + c->c.n);
        for (int v : o)
            if (v < 0 || v >= n_parts) return err(KF_CONFIG, "owner out of range");
        auto* L = new kf_layout;
        try {
            L->L = kfb::build_local_layout(c->c, o, n_parts, rank, ordering);
        } catch (...) {
            delete L;
            throw;
        }
        *out = L;
        return ok();
    });
}

void kf_layout_free(kf_layout* L) { delete L; }

void kf_layout_sizes(const kf_layout* L, int* n_local, int* n_owned, int* n_colors, int* n_peers)
{
    if (n_local) *n_local = static_cast<int>(L->L.perm.size());
    if (n_owned) *n_owned = L->L.n_owned;
    if (n_colors) *n_colors = L->L.n_colors;
    if (n_peers) *n_peers = static_cast<int>(L->L.peers.size());
}

void kf_layout_arrays(const kf_layout* L, int* perm, unsigned char* ghost, int* gs, int* oe, int* ge,
                      int* peers)
{
    const kfb::LocalLayout& l = L->L;
    if (perm) std::memcpy(perm, l.perm.data(), l.perm.size() * sizeof(int));
    if (ghost) std::memcpy(ghost, l.ghost.data(), l.ghost.size());
    if (gs) std::memcpy(gs, l.gs.data(), l.gs.size() * sizeof(int));
    if (oe) std::memcpy(oe, l.oe.data(), l.oe.size() * sizeof(int));
    if (ge) std::memcpy(ge, l.ge.data(), l.ge.size() * sizeof(int));
    if (peers && !l.peers.empty()) std::memcpy(peers, l.peers.data(), l.peers.size() * sizeof(int));
}

void kf_layout_boundary_end(const kf_layout* L, int* ob)
{
    if (ob && !L->L.ob.empty()) std::memcpy(ob, L->L.ob.data(), L->L.ob.size() * sizeof(int));
}

int kf_layout_send(const kf_layout* L, int peer_slot, int color, int* gids)
{
    const kfb::LocalLayout& l = L->L;
    if (peer_slot < 0 || peer_slot >= static_cast<int>(l.peers.size()) || color < 0 || color >= l.n_colors)
        return -1;
    const std::vector<int>& v = l.send_idx[peer_slot][color];
    if (gids)
        for (size_t k = 0; k < v.size(); ++k) gids[k] = l.perm[v[k]];
    return static_cast<int>(v.size());
}

int kf_layout_recv(const kf_layout* L, int peer_slot, int color, int* local_off)
{
    const kfb::LocalLayout& l = L->L;
    if (peer_slot < 0 || peer_slot >= static_cast<int>(l.peers.size()) || color < 0 || color >= l.n_colors)
        return -1;
    if (local_off) *local_off = l.recv_off[peer_slot][color];
    return l.recv_cnt[peer_slot][color];
}

void kf_destroy(kf_ctx* ctx) { delete ctx; }

kf_status kf_run(kf_ctx* ctx, kf_iter_record* records, int* n_done, double* final_state,
                 double* loop_seconds)
{
    return guarded([&] {
        std::string reason;
        int point = -1, iteration = 0;
        if (ctx->bad_inner) {
            // iteration 1 throws in q_derivatives: no record, the state is the
            // initial freestream + BC state (driver.cpp:207-208,255-262)
            ctx->solver->reset();
            if (final_state) ctx->solver->get_state(final_state, nullptr);
            *n_done = 0;
            if (loop_seconds) *loop_seconds = 0.0;
            return err(KF_DIVERGED, kBadInner, -1, 1);
        }
        const int code = ctx->solver->run(records, n_done, final_state, loop_seconds, reason, point,
                                          iteration);
        if (code != KF_OK) return err(code, reason, point, iteration);
        return ok();
    });
}

kf_status kf_reset(kf_ctx* ctx)
{
    return guarded([&] {
        ctx->solver->reset();
        return ok();
    });
}

kf_status kf_set_state(kf_ctx* ctx, const double* U, const double* dU_prev)
{
    return guarded([&] {
        ctx->solver->set_state(U, dU_prev);
        return ok();
    });
}

kf_status kf_get_state(kf_ctx* ctx, double* U, double* dU_prev)
{
    return guarded([&] {
        ctx->solver->get_state(U, dU_prev);
        return ok();
    });
}

kf_status kf_iterate_async(kf_ctx* ctx, int n)
{
    return guarded([&] {
        if (ctx->bad_inner) return bad_inner_status();
        ctx->solver->iterate_async(n);
        return ok();
    });
}

kf_status kf_sync_records(kf_ctx* ctx, kf_iter_record* records, int capacity, int* n_done)
{
    return guarded([&] {
        std::string reason;
        int point = -1, iteration = 0;
        const int code = ctx->solver->sync_records(records, capacity, n_done, reason, point, iteration);
        if (code != KF_OK) return err(code, reason, point, iteration);
        return ok();
    });
}

kf_status kf_step_host(kf_ctx* ctx, const double* U_in, const double* dU_prev_in, double* U_out,
                       double* dU_out, kf_iter_record* record)
{
    return guarded([&] {
        std::string reason;
        int point = -1;
        if (ctx->bad_inner) return bad_inner_status();
        const int code = ctx->solver->step_host(U_in, dU_prev_in, U_out, dU_out, record, reason, point);
        if (code != KF_OK) return err(code, reason, point, 1);
        return ok();
    });
}

kf_status kf_step_host_batch(kf_ctx* ctx, int m, const double* const* U_in, const double* const* dU_prev_in,
                             double* const* U_out, double* const* dU_out, kf_iter_record* records)
{
    return guarded([&] {
        std::string reason;
        int point = -1;
        if (ctx->bad_inner) return bad_inner_status();
        const int code = ctx->solver->step_host_batch(m, U_in, dU_prev_in, U_out, dU_out, records, reason, point);
        if (code != KF_OK) return err(code, reason, point, 1);
        return ok();
    });
}

kf_status kf_bench_mode(kf_ctx* ctx, int mode)
{
    return guarded([&] {
        ctx->solver->bench_mode(mode);
        return ok();
    });
}

void* kf_stream(kf_ctx* ctx) { return ctx->solver->stream(); }

int kf_launches_per_iteration(const kf_ctx* ctx) { return ctx->solver->launches_per_iteration(); }

kf_status kf_stage_q(kf_ctx* ctx, const double* U, double* q)
{
    return guarded([&] {
        std::string reason;
        int point = -1;
        const int code = ctx->solver->stage_q(U, q, reason, point);
        if (code) return err(code, reason, point);
        return ok();
    });
}

kf_status kf_stage_grads(kf_ctx* ctx, const double* q, double* qx, double* qy)
{
    return guarded([&] {
        ctx->solver->stage_grads(q, qx, qy);
        return ok();
    });
}

kf_status kf_stage_residual(kf_ctx* ctx, const double* q, const double* qx, const double* qy,
                            double* R, int* demoted)
{
    return guarded([&] {
        std::string reason;
        int point = -1;
        const int code = ctx->solver->stage_residual(q, qx, qy, R, demoted, reason, point);
        if (code) return err(code, reason, point);
        return ok();
    });
}

kf_status kf_stage_lusgs(kf_ctx* ctx, const double* U, const double* R, const double* dU_prev,
                         double cfl, double* dt, double* S, double* diag, double* dU_star,
                         double* dU)
{
    return guarded([&] {
        std::string reason;
        int point = -1;
        const int code =
            ctx->solver->stage_lusgs(U, R, dU_prev, cfl, dt, S, diag, dU_star, dU, reason, point);
        if (code) return err(code, reason, point);
        return ok();
    });
}

kf_status kf_stage_update(kf_ctx* ctx, const double* U, const double* dU, double* U_out)
{
    return guarded([&] {
        std::string reason;
        int point = -1;
        const int code = ctx->solver->stage_update(U, dU, U_out, reason, point);
        if (code) return err(code, reason, point);
        return ok();
    });
}

kf_status kf_stage_forces(kf_ctx* ctx, const double* U, double* cl, double* cd)
{
    return guarded([&] {
        std::string reason;
        const int code = ctx->solver->stage_forces(U, cl, cd, reason);
        if (code) return err(code, reason);
        return ok();
    });
}

kf_status kf_probe_math(int n, int which, const double* x, double* lib, double* mine)
{
    return guarded([&] {
        if (which < 0 || which > 5)
            return err(KF_CONFIG,
                       "which must be 0 (exp), 1 (log), 2 (erf), 3 (division), 4 (erf polynomial) or 5 (exp(-t) polynomial)");
        kfb::probe_math(n, which, x, lib, mine);
        return ok();
    });
}

kf_status kf_probe_split_flux(int n, const double* U, int axis, int sign, double* G)
{
    return guarded([&] {
        kfb::probe_split_flux(n, U, axis, sign, G);
        return ok();
    });
}

kf_status kf_probe_jvp_split(int n, const double* U, const double* dU, int axis, int sign, int exact,
                             double* out)
{
    return guarded([&] {
        std::vector<int> st(std::max(n, 1));
        kfb::probe_jvp_split(n, U, dU, axis, sign, exact, out, st.data());
        for (int t = 0; t < n; ++t)
            if (st[t]) return err(st[t] == 1 ? KF_INVALID_STATE : KF_INVALID_INCREMENT,
                                  st[t] == 1 ? "jvp_split: invalid state" : "jvp_split: U + dU invalid", t);
        return ok();
    });
}

kf_status kf_probe_jvp_full(int n, const double* U, const double* dU, int axis, int exact, double* out)
{
    return guarded([&] {
        std::vector<int> st(std::max(n, 1));
        kfb::probe_jvp_full(n, U, dU, axis, exact, out, st.data());
        for (int t = 0; t < n; ++t)
            if (st[t]) return err(st[t] == 1 ? KF_INVALID_STATE : KF_INVALID_INCREMENT,
                                  st[t] == 1 ? "jvp_full: invalid state" : "jvp_full: U + dU invalid", t);
        return ok();
    });
}

}  // extern "C"

extern "C" kf_status kf_profile_kernels(kf_ctx* ctx, int reps, char* names, float* ms, int cap, int* n)
{
    return guarded([&] {
        std::vector<std::string> nm;
        std::vector<float> t;
        ctx->solver->profile_kernels(std::max(reps, 1), nm, t);
        const int m = std::min<int>(cap, static_cast<int>(nm.size()));
        for (int k = 0; k < m; ++k) {
            std::snprintf(names + 32 * k, 32, "%s", nm[k].c_str());
            ms[k] = t[k];
        }
        if (n) *n = static_cast<int>(nm.size());
        return ok();
    });
}

extern "C" kf_status kf_measure_fp64_peak(int device, double* tflops)
{
    return guarded([&] {
        if (kfb::device_count() == 0)
            return err(KF_CUDA, "no CUDA device available (the B200 path has no CPU fallback)");
        *tflops = kfb::measure_fp64_peak(device);
        return ok();
    });
}
