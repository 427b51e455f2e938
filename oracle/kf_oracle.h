/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference hot path.
 *
 * This is the CHECKER the CUDA product is compared against. It restates, in
 * C99 over flat CSR arrays, the reference kinfree algorithm for one
 * fixed-point iteration and the ingestion that feeds it; every function cites
 * the reference file:line it follows (paths relative to
 * /root/reference/proj). Compiled with -ffp-contract=off and no -march (as
 * the reference Release build), its arithmetic is bit-for-bit the
 * reference's: tests/test_oracle.py pins that against oracle/_ref (the real
 * reference, compiled in place) and against the committed golden fixtures in
 * tests/golden/ that were produced by the real reference.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline) may load
 * it. The product library never links it.
 */
#ifndef KF_ORACLE_H
#define KF_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct kfo_cloud kfo_cloud;

typedef struct {
    int variant; /* 0 explicit 1 anandh 2 anandh_ad 3 manish 4 manish_ad */
    double cfl;
    int n_iterations;
    int n_inner;
    double mach;
    double aoa_deg;
    double convergence_decades;
    int bc_mode; /* 0 physical, 1 freestream-all */
    int cfl_ramp_iters;
    double cfl_start;
    double divergence_factor;
} kfo_config;

/* Error record: code 0 ok, 1 invalid state, 2 config / setup; point is the
 * reference's point index (or -1); msg is the reference's what() text. */
typedef struct {
    int code;
    int point;
    char msg[192];
} kfo_err;

/* Builds split stencils (pointcloud.cpp:257-299), LS coefficients
 * (spatial.cpp:80-128) and the greedy colouring (coloring.cpp:23-52) from raw
 * arrays. kind: 0 wall, 1 interior, 2 outer. CSR neighbours, 0-based. */
kfo_cloud* kfo_cloud_new(int n, const double* x, const double* y, const int* kind,
                         const double* nx, const double* ny, const int* off,
                         const int* idx);
void kfo_cloud_free(kfo_cloud* c);
int kfo_n(const kfo_cloud* c);
int kfo_n_colors(const kfo_cloud* c);
/* which: 0 nbr 1 xpos 2 xneg 3 ypos 4 yneg */
long kfo_list_nnz(const kfo_cloud* c, int which);
void kfo_list(const kfo_cloud* c, int which, int* off, int* idx);
void kfo_ls_full(const kfo_cloud* c, double* wx, double* wy, int* kinds);
void kfo_ls_split(const kfo_cloud* c, int which, double* w, double* ls_one, int* kinds);
int kfo_flagged(const kfo_cloud* c, int* out);
void kfo_colors(const kfo_cloud* c, int* color);
int kfo_report(const kfo_cloud* c, int* empty, int* n_empty, int* singular, int* n_singular);

/* Stage functions: state arrays are n x 4 doubles (AoS, point-major). */
void kfo_freestream(double mach, double aoa_deg, double* U4);
int kfo_q(const kfo_cloud* c, const double* U, double* q, kfo_err* e);
void kfo_grads(const kfo_cloud* c, const double* q, int n_inner, double* qx, double* qy);
int kfo_residual(const kfo_cloud* c, const double* q, const double* qx, const double* qy,
                 int first_order, double* R, int* demoted, kfo_err* e);
int kfo_timestep(const kfo_cloud* c, const double* U, double cfl, double* dt, kfo_err* e);
int kfo_s_term(const kfo_cloud* c, const double* U, const double* dU_prev, int exact,
               double* S, int* n_fallback, kfo_err* e);
int kfo_diagonal(const kfo_cloud* c, const double* U, const double* dt, int variant,
                 double* d, kfo_err* e);
int kfo_sweeps(const kfo_cloud* c, const double* U, const double* R, const double* S,
               const double* d, int exact, double* dU_star, double* dU, kfo_err* e);
int kfo_bc(const kfo_cloud* c, double* U, double mach, double aoa_deg, int bc_mode,
           kfo_err* e);
int kfo_forces(const kfo_cloud* c, const double* U, double mach, double aoa_deg,
               double* cl, double* cd, kfo_err* e);

/* run_fixed_point (driver.cpp:188-282). Per-iteration arrays have capacity
 * cfg->n_iterations. Returns 0 (diverged/abort reported through *diverged and
 * reason), or 1 for a precondition error (message in reason). */
int kfo_run(const kfo_cloud* c, const kfo_config* cfg, int* n_done, double* residual,
            double* cl, double* cd, int* first_order, double* final_state, int* diverged,
            char* reason, int reason_len);

/* Point physics (kinetics.cpp / tangent.cpp) for unit tests. axis 0 X 1 Y;
 * sign 0 Plus 1 Minus. Return 0, or 1 if the state is invalid. */
int kfo_split_flux(const double* U, int axis, int sign, double* G);
int kfo_jvp_split(const double* U, const double* dU, int axis, int sign, int exact,
                  double* out);
int kfo_jvp_full(const double* U, const double* dU, int axis, int exact, double* out);

#ifdef __cplusplus
}
#endif
#endif
