// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference solver (`kinfree_core`,
// /root/reference/proj/src/*.cpp) so that Python tests and bench.py's
// reference arm can drive it through ctypes. Built by oracle/Makefile into
// oracle/_ref/libkfref.so together with the reference sources, which are
// compiled in place (never copied).
//
// Every entry point wraps one public reference function:
//   kfref_generate      -> generate_naca_ogrid          pointcloud.cpp:180-255
//   kfref_from_arrays   -> build_split_stencils         pointcloud.cpp:257-299
//   kfref_load          -> load_cloud                   pointcloud.cpp:301-381
//   (both)              -> build_ls_coefficients        spatial.cpp:80-128
//                       -> color_points/build_sweep_plan coloring.cpp:23-62
//   kfref_q             -> q_from_conserved             state.cpp:53-56
//   kfref_grads         -> q_derivatives                spatial.cpp:151-196
//   kfref_residual      -> flux_residual                spatial.cpp:249-298
//   kfref_timestep      -> local_timestep               driver.cpp:24-47
//   kfref_s_term        -> compute_s_term               implicit.cpp:96-134
//   kfref_diagonal      -> assemble_diagonal            implicit.cpp:39-94
//   kfref_sweeps        -> forward_sweep/backward_sweep implicit.cpp:174-226
//   kfref_bc            -> apply_boundary_conditions    driver.cpp:69-95
//   kfref_forces        -> compute_forces               driver.cpp:127-167
//   kfref_run           -> run_fixed_point              driver.cpp:188-282
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

#include <algorithm>

#include "kinfree/coloring.hpp"
#include "kinfree/counters.hpp"
#include "kinfree/driver.hpp"
#include "kinfree/implicit.hpp"
#include "kinfree/kinetics.hpp"
#include "kinfree/pointcloud.hpp"
#include "kinfree/spatial.hpp"
#include "kinfree/state.hpp"
#include "kinfree/tangent.hpp"

using namespace kinfree;

namespace {

struct RefCtx {
    PointCloud cloud;
    LsCoefficients ls;
    ColorAssignment colors;
    SweepPlan plan;
};

void set_err(char* err, int len, const char* msg)
{
    if (err && len > 0) {
        std::snprintf(err, static_cast<size_t>(len), "%s", msg);
    }
}

RefCtx* finish(PointCloud&& c)
{
    auto* ctx = new RefCtx;
    ctx->cloud = std::move(c);
    ctx->ls = build_ls_coefficients(ctx->cloud);
    ctx->colors = color_points(ctx->cloud);
    ctx->plan = build_sweep_plan(ctx->colors);
    return ctx;
}

std::vector<Vec4> to_vec4(const double* a, int n)
{
    std::vector<Vec4> v(n);
    for (int p = 0; p < n; ++p)
        for (int k = 0; k < 4; ++k) v[p][k] = a[4 * p + k];
    return v;
}

void from_vec4(const std::vector<Vec4>& v, double* a)
{
    for (size_t p = 0; p < v.size(); ++p)
        for (int k = 0; k < 4; ++k) a[4 * p + k] = v[p][k];
}

SolverVariant variant_of(int v) { return static_cast<SolverVariant>(v); }

}  // namespace

extern "C" {

struct kfref_config {
    int variant;  // SolverVariant order: explicit, anandh, anandh_ad, manish, manish_ad
    double cfl;
    int n_iterations;
    int n_inner;
    double mach;
    double aoa_deg;
    double convergence_decades;
    int bc_mode;  // 0 physical, 1 freestream
    int cfl_ramp_iters;
    double cfl_start;
    double divergence_factor;
};

int kfref_num_threads(int n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
    return omp_get_max_threads();
#else
    (void)n;
    return 1;
#endif
}

void* kfref_generate(const char* digits, int nw, int nr, double rf, char* err, int errlen)
{
    try {
        return finish(generate_naca_ogrid(digits, nw, nr, rf));
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return nullptr;
    }
}

void* kfref_load(const char* path, char* err, int errlen)
{
    try {
        return finish(load_cloud(path));
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return nullptr;
    }
}

int kfref_save(void* h, const char* path, char* err, int errlen)
{
    try {
        save_cloud(static_cast<RefCtx*>(h)->cloud, path);
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 1;
    }
}

// Cloud from raw arrays (0-based CSR neighbours); kinds 0 wall, 1 interior, 2 outer.
// wall/interior/outer id lists are built in index order, as classify() does
// (pointcloud.cpp:137-149).
void* kfref_from_arrays(int n, const double* x, const double* y, const int* kind,
                        const double* nx, const double* ny, const int* off,
                        const int* idx, char* err, int errlen)
{
    try {
        PointCloud c;
        c.x.assign(x, x + n);
        c.y.assign(y, y + n);
        c.kind.resize(n);
        c.normal_x.assign(nx, nx + n);
        c.normal_y.assign(ny, ny + n);
        c.nbr.resize(n);
        for (int p = 0; p < n; ++p) {
            c.kind[p] = static_cast<PointKind>(kind[p]);
            c.nbr[p].assign(idx + off[p], idx + off[p + 1]);
            if (kind[p] == 0) c.wall_ids.push_back(p);
            if (kind[p] == 1) c.interior_ids.push_back(p);
            if (kind[p] == 2) c.outer_ids.push_back(p);
        }
        c.stencil_report = build_split_stencils(c);
        return finish(std::move(c));
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return nullptr;
    }
}

void kfref_free(void* h) { delete static_cast<RefCtx*>(h); }

int kfref_n(void* h) { return static_cast<RefCtx*>(h)->cloud.n(); }
int kfref_n_colors(void* h) { return static_cast<RefCtx*>(h)->colors.n_colors; }

// which: 0 nbr, 1 xpos, 2 xneg, 3 ypos, 4 yneg
static const std::vector<std::vector<int>>& list_of(RefCtx* c, int which)
{
    switch (which) {
        case 1: return c->cloud.xpos;
        case 2: return c->cloud.xneg;
        case 3: return c->cloud.ypos;
        case 4: return c->cloud.yneg;
        default: return c->cloud.nbr;
    }
}

long kfref_list_nnz(void* h, int which)
{
    long s = 0;
    for (const auto& v : list_of(static_cast<RefCtx*>(h), which)) s += v.size();
    return s;
}

void kfref_list(void* h, int which, int* off, int* idx)
{
    const auto& L = list_of(static_cast<RefCtx*>(h), which);
    long o = 0;
    off[0] = 0;
    for (size_t p = 0; p < L.size(); ++p) {
        for (int q : L[p]) idx[o++] = q;
        off[p + 1] = static_cast<int>(o);
    }
}

void kfref_geometry(void* h, double* x, double* y, int* kind, double* nx, double* ny)
{
    const PointCloud& c = static_cast<RefCtx*>(h)->cloud;
    for (int p = 0; p < c.n(); ++p) {
        x[p] = c.x[p];
        y[p] = c.y[p];
        kind[p] = static_cast<int>(c.kind[p]);
        nx[p] = c.normal_x[p];
        ny[p] = c.normal_y[p];
    }
}

int kfref_report(void* h, int* empty, int* singular, int* n_empty, int* n_singular)
{
    const StencilReport& r = static_cast<RefCtx*>(h)->cloud.stencil_report;
    *n_empty = static_cast<int>(r.empty_points.size());
    *n_singular = static_cast<int>(r.singular_points.size());
    if (empty)
        for (size_t k = 0; k < r.empty_points.size(); ++k) empty[k] = r.empty_points[k];
    if (singular)
        for (size_t k = 0; k < r.singular_points.size(); ++k)
            singular[k] = r.singular_points[k];
    return 0;
}

// Full-stencil weights in nbr CSR order; split weights in their list CSR order.
void kfref_ls_full(void* h, double* wx, double* wy, int* kinds)
{
    const LsCoefficients& ls = static_cast<RefCtx*>(h)->ls;
    long o = 0;
    for (size_t p = 0; p < ls.full.size(); ++p) {
        kinds[p] = static_cast<int>(ls.full[p].kind);
        for (size_t k = 0; k < ls.full[p].nbr.size(); ++k, ++o) {
            wx[o] = ls.full[p].wx[k];
            wy[o] = ls.full[p].wy[k];
        }
    }
}

// which: 1 xpos, 2 xneg, 3 ypos, 4 yneg
void kfref_ls_split(void* h, int which, double* w, double* ls_one, int* kinds)
{
    const LsCoefficients& ls = static_cast<RefCtx*>(h)->ls;
    const std::vector<SplitStencilLs>* v = which == 1   ? &ls.xpos
                                           : which == 2 ? &ls.xneg
                                           : which == 3 ? &ls.ypos
                                                        : &ls.yneg;
    long o = 0;
    for (size_t p = 0; p < v->size(); ++p) {
        ls_one[p] = (*v)[p].ls_one;
        kinds[p] = static_cast<int>((*v)[p].kind);
        for (double x : (*v)[p].w) w[o++] = x;
    }
}

int kfref_flagged(void* h, int* out)
{
    const LsCoefficients& ls = static_cast<RefCtx*>(h)->ls;
    if (out)
        for (size_t k = 0; k < ls.flagged.size(); ++k) out[k] = ls.flagged[k];
    return static_cast<int>(ls.flagged.size());
}

void kfref_colors(void* h, int* color)
{
    const ColorAssignment& c = static_cast<RefCtx*>(h)->colors;
    for (size_t p = 0; p < c.color.size(); ++p) color[p] = c.color[p];
}

// A caller-supplied colouring (1-based): the SweepPlan run_fixed_point takes
// (driver.hpp:104-106) rebuilt by the reference's own build_sweep_plan
// (coloring.cpp:54-62); 0 on success, the number of invalid edges otherwise
// (validate_coloring, coloring.cpp:64-73).
int kfref_set_colors(void* h, const int* color)
{
    RefCtx* c = static_cast<RefCtx*>(h);
    ColorAssignment a;
    a.color.assign(color, color + c->cloud.n());
    a.n_colors = c->cloud.n() ? *std::max_element(a.color.begin(), a.color.end()) : 0;
    const auto bad = validate_coloring(c->cloud, a);
    if (!bad.empty()) return static_cast<int>(bad.size());
    c->colors = a;
    c->plan = build_sweep_plan(c->colors);
    return 0;
}

// ---- per-stage entry points (state arrays are 4n doubles, AoS) ----

int kfref_freestream(double mach, double aoa, double* U4)
{
    const Freestream fs = Freestream::make(mach, aoa);
    for (int k = 0; k < 4; ++k) U4[k] = fs.U[k];
    return 0;
}

int kfref_q(void* h, const double* U, double* q, char* err, int errlen)
{
    const int n = kfref_n(h);
    try {
        for (int p = 0; p < n; ++p) {
            const Vec4 v = q_from_conserved({U[4 * p], U[4 * p + 1], U[4 * p + 2], U[4 * p + 3]}, p);
            for (int k = 0; k < 4; ++k) q[4 * p + k] = v[k];
        }
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 1;
    }
}

int kfref_grads(void* h, const double* q, int n_inner, double* qx, double* qy)
{
    RefCtx* c = static_cast<RefCtx*>(h);
    const GradientField g = q_derivatives(c->cloud, c->ls, to_vec4(q, c->cloud.n()), n_inner);
    from_vec4(g.qx, qx);
    from_vec4(g.qy, qy);
    return 0;
}

// order: 0 second, 1 first. demoted[p] set to 1 for demoted points.
int kfref_residual(void* h, const double* q, const double* qx, const double* qy, int order,
                   double* R, int* demoted, char* err, int errlen)
{
    RefCtx* c = static_cast<RefCtx*>(h);
    const int n = c->cloud.n();
    try {
        GradientField g{to_vec4(qx, n), to_vec4(qy, n)};
        ResidualStats st;
        const std::vector<Vec4> r =
            flux_residual(c->cloud, c->ls, to_vec4(q, n), g, &st,
                          order ? ResidualOrder::FirstOrder : ResidualOrder::SecondOrder);
        from_vec4(r, R);
        if (demoted) {
            for (int p = 0; p < n; ++p) demoted[p] = 0;
            for (int p : st.first_order_points) demoted[p] = 1;
        }
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 1;
    }
}

int kfref_timestep(void* h, const double* U, double cfl, double* dt, char* err, int errlen)
{
    RefCtx* c = static_cast<RefCtx*>(h);
    try {
        const std::vector<double> d = local_timestep(c->cloud, to_vec4(U, c->cloud.n()), cfl);
        std::memcpy(dt, d.data(), d.size() * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 1;
    }
}

int kfref_s_term(void* h, const double* U, const double* dU_prev, int exact, double* S,
                 int* n_fallback, char* err, int errlen)
{
    RefCtx* c = static_cast<RefCtx*>(h);
    const int n = c->cloud.n();
    try {
        std::vector<int> fb;
        const std::vector<Vec4> s =
            compute_s_term(c->cloud, c->ls, to_vec4(U, n), to_vec4(dU_prev, n),
                           exact ? FluxIncrementMode::Exact : FluxIncrementMode::Incremental,
                           &fb);
        from_vec4(s, S);
        if (n_fallback) *n_fallback = static_cast<int>(fb.size());
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 1;
    }
}

int kfref_diagonal(void* h, const double* U, const double* dt, int variant, double* d,
                   char* err, int errlen)
{
    RefCtx* c = static_cast<RefCtx*>(h);
    const int n = c->cloud.n();
    try {
        const std::vector<double> dv = assemble_diagonal(
            c->cloud, c->ls, to_vec4(U, n), std::vector<double>(dt, dt + n), variant_of(variant));
        std::memcpy(d, dv.data(), dv.size() * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 1;
    }
}

// S may be null (anandh family). Writes dU_star and dU.
int kfref_sweeps(void* h, const double* U, const double* R, const double* S, const double* d,
                 int exact, double* dU_star, double* dU, uint64_t* sweep_counts, char* err,
                 int errlen)
{
    RefCtx* c = static_cast<RefCtx*>(h);
    const int n = c->cloud.n();
    try {
        const std::vector<Vec4> Uv = to_vec4(U, n);
        std::vector<Vec4> Sv;
        if (S) Sv = to_vec4(S, n);
        const std::vector<double> dv(d, d + n);
        const FluxIncrementMode mode =
            exact ? FluxIncrementMode::Exact : FluxIncrementMode::Incremental;
        const EvalSnapshot before = flux_counters().snapshot();
        std::vector<Vec4> ds, du;
        forward_sweep(c->plan, c->cloud, c->ls, Uv, to_vec4(R, n), S ? &Sv : nullptr, dv, mode, ds);
        from_vec4(ds, dU_star);
        backward_sweep(c->plan, c->cloud, c->ls, Uv, ds, dv, mode, du);
        from_vec4(du, dU);
        const EvalSnapshot delta = flux_counters().snapshot() - before;
        if (sweep_counts)
            for (int k = 0; k < kNumEvalKinds; ++k) sweep_counts[k] = delta.n[k];
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 1;
    }
}

int kfref_bc(void* h, double* U, double mach, double aoa, int bc_mode, char* err, int errlen)
{
    RefCtx* c = static_cast<RefCtx*>(h);
    const int n = c->cloud.n();
    try {
        std::vector<Vec4> s = to_vec4(U, n);
        apply_boundary_conditions(c->cloud, s, Freestream::make(mach, aoa),
                                  bc_mode ? BcMode::FreestreamAll : BcMode::Physical);
        from_vec4(s, U);
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 1;
    }
}

int kfref_forces(void* h, const double* U, double mach, double aoa, double* cl, double* cd,
                 double* cp, char* err, int errlen)
{
    RefCtx* c = static_cast<RefCtx*>(h);
    const int n = c->cloud.n();
    try {
        const std::vector<Vec4> s = to_vec4(U, n);
        const Freestream fs = Freestream::make(mach, aoa);
        const auto f = compute_forces(c->cloud, s, fs);
        *cl = f.first;
        *cd = f.second;
        if (cp) {
            const std::vector<double> v = surface_cp(c->cloud, s, fs);
            std::memcpy(cp, v.data(), v.size() * sizeof(double));
        }
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 1;
    }
}

// One full run_fixed_point. Per-iteration outputs (capacity n_iterations):
// residual, cl, cd, seconds, first_order_points, and the cumulative/sweep
// counter snapshots (5 uint64 each). Returns 0 on normal return (diverged may
// still be set), 1 on a precondition exception (message in reason).
int kfref_run(void* h, const kfref_config* cfg, int* n_done, double* residual, double* cl,
              double* cd, double* seconds, int* first_order, uint64_t* counters,
              uint64_t* sweep, double* final_state, int* diverged, double* loop_seconds,
              char* reason, int reason_len)
{
    RefCtx* c = static_cast<RefCtx*>(h);
    SolverConfig sc;
    sc.variant = variant_of(cfg->variant);
    sc.cfl = cfg->cfl;
    sc.n_iterations = cfg->n_iterations;
    sc.n_inner = cfg->n_inner;
    sc.mach_inf = cfg->mach;
    sc.aoa_deg = cfg->aoa_deg;
    sc.convergence_decades = cfg->convergence_decades;
    sc.bc_mode = cfg->bc_mode ? BcMode::FreestreamAll : BcMode::Physical;
    sc.cfl_ramp_iters = cfg->cfl_ramp_iters;
    sc.cfl_start = cfg->cfl_start;
    sc.divergence_factor = cfg->divergence_factor;
    try {
        std::vector<Vec4> state;
        const RunHistory hist = run_fixed_point(c->cloud, c->ls, c->plan, sc, &state);
        *n_done = static_cast<int>(hist.iters.size());
        for (size_t k = 0; k < hist.iters.size(); ++k) {
            const IterationRecord& r = hist.iters[k];
            residual[k] = r.residual;
            cl[k] = r.cl;
            cd[k] = r.cd;
            if (seconds) seconds[k] = r.seconds;
            if (first_order) first_order[k] = r.first_order_points;
            for (int j = 0; j < kNumEvalKinds; ++j) {
                if (counters) counters[k * kNumEvalKinds + j] = r.counters.n[j];
                if (sweep) sweep[k * kNumEvalKinds + j] = r.sweep.n[j];
            }
        }
        if (final_state) from_vec4(state, final_state);
        *diverged = hist.diverged ? 1 : 0;
        if (loop_seconds) *loop_seconds = hist.loop_seconds;
        set_err(reason, reason_len, hist.abort_reason.c_str());
        return 0;
    } catch (const std::exception& e) {
        set_err(reason, reason_len, e.what());
        return 1;
    }
}

void kfref_counters(uint64_t* out)
{
    const EvalSnapshot s = flux_counters().snapshot();
    for (int k = 0; k < kNumEvalKinds; ++k) out[k] = s.n[k];
}

// Point-physics probes for the kinetic/tangent known-answer tests.
// axis 0 X / 1 Y; sign 0 Plus / 1 Minus.
void kfref_split_flux(const double* U, int axis, int sign, double* G)
{
    const Vec4 g = split_flux(Vec4{U[0], U[1], U[2], U[3]}, axis ? Axis::Y : Axis::X,
                              sign ? HalfRange::Minus : HalfRange::Plus);
    for (int k = 0; k < 4; ++k) G[k] = g[k];
}

void kfref_jvp_split(const double* U, const double* dU, int axis, int sign, int exact,
                     double* out)
{
    const Vec4 u{U[0], U[1], U[2], U[3]}, d{dU[0], dU[1], dU[2], dU[3]};
    const Vec4 g = exact ? jvp_split(u, d, axis ? Axis::Y : Axis::X,
                                     sign ? HalfRange::Minus : HalfRange::Plus)
                         : incremental_jvp_split(u, d, axis ? Axis::Y : Axis::X,
                                                 sign ? HalfRange::Minus : HalfRange::Plus);
    for (int k = 0; k < 4; ++k) out[k] = g[k];
}

void kfref_jvp_full(const double* U, const double* dU, int axis, int exact, double* out)
{
    const Vec4 u{U[0], U[1], U[2], U[3]}, d{dU[0], dU[1], dU[2], dU[3]};
    const Vec4 g = exact ? jvp_full(u, d, axis ? Axis::Y : Axis::X)
                         : incremental_jvp_full(u, d, axis ? Axis::Y : Axis::X);
    for (int k = 0; k < 4; ++k) out[k] = g[k];
}

}  // extern "C"
