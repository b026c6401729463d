/*
 * oracle_mpm.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded CPU implementation of one time step of
 * differentiable MLS-MPM (forward) and its separately hand-written reverse
 * pass, iterated over T steps by a tape with segment checkpointing.
 *
 * Who may use this: tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs.  The product path
 * (paper_1910_00935_b200/) never includes, links or calls anything here; the
 * two share no code.
 *
 * Passages followed (PAPER.md line numbers, "P:n"):
 *   P:305        diffmpm: MLS-MPM after ChainQueen (equations are in the cited
 *                work; the reading used is DESIGN.md "Readings" R1..R24, which
 *                restates SURVEY.md Appendix A).
 *   P:568-592    Appendix D.1: advance() = clear_grid, compute_actuation, p2g,
 *                grid_op, g2p; advance_grad() recomputes the grid, then
 *                g2p.grad, grid_op.grad, p2g.grad, compute_actuation.grad.
 *   P:594-598    Appendix D.2: segment-wise recomputation (checkpoint every k).
 *   P:148-158    Global data access rules / adjoint contract f*(X, Y*) -> X*.
 *   P:207        flatten branching -> select; the adjoint of select passes the
 *                gradient through the taken branch only (grid_op BC).
 *   P:219, P:245-263  tape: seed loss adjoint = 1, replay in reverse.
 *
 * Precision: ORACLE_REAL (double by default; the float build exists for
 * fp32-vs-fp64 drift studies only).
 *
 * Layouts (caller order, row-major): x[N][d], v[N][d], C[N][d][d],
 * F[N][d][d]; grid arrays are dense [n_grid^d][d+1] = (P_0..P_{d-1}, M) with
 * node (i0,i1[,i2]) at linear index (i0*n + i1)*n + i2 (axis 1 is "up").
 *
 * Status codes: 0 ok, 4 out of domain (a stencil node left [0,n_grid-1]^d),
 * 5 non-finite / degenerate deformation (J<=0 under Neo-Hookean, r=0 in the
 * 2x2 polar decomposition).
 */
#ifndef ORACLE_MPM_H
#define ORACLE_MPM_H
#include <stdint.h>

#ifndef ORACLE_REAL
#define ORACLE_REAL double
#endif
typedef ORACLE_REAL real;

typedef struct {
    int32_t dim;       /* 2 or 3 */
    int32_t n_grid;    /* nodes per axis; dx = 1/n_grid */
    int32_t bound;     /* beta, sticky-wall thickness in nodes */
    int32_t model;     /* 0 = Neo-Hookean, 1 = fixed-corotated (2D only) */
    int32_t n_act;     /* number of actuators (controller outputs) */
    int32_t act_axis;  /* actuation direction e (axis index) */
    int32_t n_sin;     /* sinusoid time features */
    int32_t hidden;    /* H; 0 = one tanh layer */
    double dt, E, nu, p_mass, p_vol, gravity, eps_mass, kappa, omega;
    int32_t closed_loop;  /* 1: the controller also sees the per-muscle observations (R22) */
    double obs_sx, obs_sv;  /* observation scales s_x, s_v (R22) */
    const int32_t* mat;     /* per-particle material (R23): 0 elastic solid, 1 weakly compressible
                               fluid (mu = 0, F reset to J^(1/d) I); NULL = all solid */
} oracle_cfg;

enum { ORACLE_OK = 0, ORACLE_OUT_OF_DOMAIN = 4, ORACLE_NONFINITE = 5, ORACLE_INVALID = 1 };

/* quadratic B-spline weights and derivatives at f in [1/2, 3/2) */
void oracle_bspline(real f, real w[3], real dw[3]);
/* Lame parameters from (E, nu) */
void oracle_lame(const oracle_cfg* c, real* mu, real* lam);
/* Kirchhoff stress of the material model (no actuation): tau = P(F) F^T */
int oracle_stress(const oracle_cfg* c, const real* F, real* tau);
/* reverse of oracle_stress: Fbar += d<tau_bar, tau(F)>/dF */
int oracle_stress_adj(const oracle_cfg* c, const real* F, const real* tau_bar, real* F_bar);
/* strain energy density psi(F) (used only by tests to pin tau = dpsi/dF F^T) */
int oracle_energy(const oracle_cfg* c, const real* F, real* psi);

/* controller (R9; closed loop R22): alpha_t = MLP([phi(t), o_t]); o_t = NULL (or
   closed_loop = 0) is the open-loop controller on the sinusoid features only */
int64_t oracle_n_theta(const oracle_cfg* c);
int oracle_n_obs(const oracle_cfg* c);
void oracle_controller(const oracle_cfg* c, const real* theta, int32_t t, real* alpha);
void oracle_controller_adj(const oracle_cfg* c, const real* theta, int32_t t,
                           const real* alpha_bar, real* theta_bar);
void oracle_controller_obs(const oracle_cfg* c, const real* theta, int32_t t, const real* obs,
                           real* alpha);
/* theta_bar += (d alpha/d theta)^T alpha_bar; obs_bar (may be NULL) = (d alpha/d o)^T alpha_bar */
void oracle_controller_obs_adj(const oracle_cfg* c, const real* theta, int32_t t, const real* obs,
                               const real* alpha_bar, real* theta_bar, real* obs_bar);
/* R22 observation of S_t: per actuator group a (particles with aid = a, n_a of them):
   o[a][0:d] = s_x (mean_a x - mean x), o[a][d:2d] = s_v mean_a v  (0 for an empty group) */
void oracle_observe(const oracle_cfg* c, int64_t N, const real* x, const real* v,
                    const int32_t* aid, real* obs);
/* its reverse: xb, vb += (d o / d (x, v))^T obs_bar */
void oracle_observe_adj(const oracle_cfg* c, int64_t N, const int32_t* aid, const real* obs_bar,
                        real* xb, real* vb);

/* stages of one forward step (advance()) */
int oracle_p2g(const oracle_cfg* c, int64_t N, const real* x, const real* v, const real* C,
               const real* F, const int32_t* aid, const real* alpha, real* grid, real* F_next);
void oracle_grid_op(const oracle_cfg* c, const real* grid, real* U);
int oracle_g2p(const oracle_cfg* c, int64_t N, const real* x, const real* U,
               real* x_next, real* v_next, real* C_next);
int oracle_step(const oracle_cfg* c, int64_t N, const real* x, const real* v, const real* C,
                const real* F, const int32_t* aid, const real* alpha,
                real* xn, real* vn, real* Cn, real* Fn);

/* stages of one reverse step (advance_grad()) */
int oracle_g2p_adj(const oracle_cfg* c, int64_t N, const real* x, const real* U,
                   const real* xb_next, const real* vb_next, const real* Cb_next,
                   real* U_bar, real* xb);
void oracle_grid_op_adj(const oracle_cfg* c, const real* grid, const real* U_bar, real* grid_bar);
int oracle_p2g_adj(const oracle_cfg* c, int64_t N, const real* x, const real* v, const real* C,
                   const real* F, const int32_t* aid, const real* alpha,
                   const real* grid_bar, const real* Fb_next,
                   real* xb, real* vb, real* Cb, real* Fb, real* alpha_bar);
int oracle_step_adj(const oracle_cfg* c, int64_t N, const real* x, const real* v, const real* C,
                    const real* F, const int32_t* aid, const real* alpha,
                    const real* xb_n, const real* vb_n, const real* Cb_n, const real* Fb_n,
                    real* xb, real* vb, real* Cb, real* Fb, real* alpha_bar);

/* loss on x_T: kind 0 = |xbar - target|^2, kind 1 = -xbar . e_0 (xbar = mass-weighted mean) */
int oracle_loss(const oracle_cfg* c, int32_t kind, const real* target, int64_t N,
                const real* x, real* L, real* xb);

/* whole episode: forward T steps (checkpoint every k), loss, reverse, grads.
   Outputs S_T (x_T..F_T), L, and dL/d{x0,v0,C0,F0,theta}; any output may be NULL. */
int oracle_run(const oracle_cfg* c, int64_t N, int32_t T, int32_t k_ckpt,
               const real* x0, const real* v0, const real* C0, const real* F0,
               const int32_t* aid, const real* theta, int32_t loss_kind, const real* target,
               real* xT, real* vT, real* CT, real* FT, real* L,
               real* dx0, real* dv0, real* dC0, real* dF0, real* dtheta);

#endif
