/*
 * oracle_mpm.c -- TEST INFRASTRUCTURE ONLY (see oracle_mpm.h for who may use it).
 *
 * Plain, slow, obviously-correct CPU MLS-MPM step and its hand-written
 * reverse.  Every loop follows the kernel order of PAPER.md Appendix D.1
 * and the equations of the reading DESIGN.md R1..R24 (SURVEY.md
 * Appendix A).  No blocking, no fusion, no reordering: one particle at a time,
 * one stencil node at a time, dense grid.
 *
 * Pins (tests/test_oracle_pins.py): B-spline moment identities, P2G mass and
 * momentum conservation, the P2G second-moment identity, stress = dpsi/dF F^T
 * by finite differences of the energy, rotation covariance, G2P affine
 * reproduction, rigid translation, ballistic centre of mass, the closed-form
 * gradient of the COM loss, and central finite differences of whole
 * trajectories for every parameter group.
 */
#include "oracle_mpm.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>

#define MAXD 3

/* ---------------------------------------------------------------- helpers */

static int ipow3(int d) { return d == 2 ? 9 : 27; }

static int64_t n_nodes(const oracle_cfg* c) {
    int64_t n = c->n_grid;
    return c->dim == 2 ? n * n : n * n * n;
}

/* digits of the stencil offset o in {0,1,2}^d for enumeration index s */
static void offset_of(int d, int s, int o[MAXD]) {
    for (int k = d - 1; k >= 0; --k) { o[k] = s % 3; s /= 3; }
}

static int64_t node_index(const oracle_cfg* c, const int i[MAXD]) {
    int64_t n = c->n_grid;
    if (c->dim == 2) return (int64_t)i[0] * n + i[1];
    return ((int64_t)i[0] * n + i[1]) * n + i[2];
}

static void node_coords(const oracle_cfg* c, int64_t lin, int i[MAXD]) {
    int n = c->n_grid;
    for (int k = c->dim - 1; k >= 0; --k) { i[k] = (int)(lin % n); lin /= n; }
}

static real det(int d, const real* F) {
    if (d == 2) return F[0] * F[3] - F[1] * F[2];
    return F[0] * (F[4] * F[8] - F[5] * F[7]) - F[1] * (F[3] * F[8] - F[5] * F[6]) +
           F[2] * (F[3] * F[7] - F[4] * F[6]);
}

/* cofactor matrix cof(F) = det(F) F^{-T} */
static void cofactor(int d, const real* F, real* K) {
    if (d == 2) {
        K[0] = F[3]; K[1] = -F[2];
        K[2] = -F[1]; K[3] = F[0];
        return;
    }
    K[0] = F[4] * F[8] - F[5] * F[7];
    K[1] = -(F[3] * F[8] - F[5] * F[6]);
    K[2] = F[3] * F[7] - F[4] * F[6];
    K[3] = -(F[1] * F[8] - F[2] * F[7]);
    K[4] = F[0] * F[8] - F[2] * F[6];
    K[5] = -(F[0] * F[7] - F[1] * F[6]);
    K[6] = F[1] * F[5] - F[2] * F[4];
    K[7] = -(F[0] * F[5] - F[2] * F[3]);
    K[8] = F[0] * F[4] - F[1] * F[3];
}

/* C = A B (d x d, row-major) */
static void matmul(int d, const real* A, const real* B, real* C) {
    for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j) {
            real s = 0;
            for (int k = 0; k < d; ++k) s += A[i * d + k] * B[k * d + j];
            C[i * d + j] = s;
        }
}

/* C = A B^T */
static void matmul_bt(int d, const real* A, const real* B, real* C) {
    for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j) {
            real s = 0;
            for (int k = 0; k < d; ++k) s += A[i * d + k] * B[j * d + k];
            C[i * d + j] = s;
        }
}

/* C = A^T B */
static void matmul_at(int d, const real* A, const real* B, real* C) {
    for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j) {
            real s = 0;
            for (int k = 0; k < d; ++k) s += A[k * d + i] * B[k * d + j];
            C[i * d + j] = s;
        }
}

/* particle stencil: base cell b = floor(x/dx - 1/2), f = x/dx - b (R12) */
static int stencil(const oracle_cfg* c, const real* xp, int base[MAXD], real fx[MAXD],
                   real w[MAXD][3], real dw[MAXD][3]) {
    const real inv_dx = (real)c->n_grid;
    for (int k = 0; k < c->dim; ++k) {
        real xi = xp[k] * inv_dx;
        real b = floor(xi - (real)0.5);
        if (!(b == b)) return ORACLE_NONFINITE;
        if (b < 0 || b + 2 > c->n_grid - 1) return ORACLE_OUT_OF_DOMAIN; /* R13 */
        base[k] = (int)b;
        fx[k] = xi - b;
        oracle_bspline(fx[k], w[k], dw[k]);
    }
    return ORACLE_OK;
}

static real weight(int d, const real w[MAXD][3], const int o[MAXD]) {
    real W = 1;
    for (int k = 0; k < d; ++k) W *= w[k][o[k]];
    return W;
}

/* dW/df_k = N'_{o_k}(f_k) prod_{j != k} N_{o_j}(f_j) */
static void weight_grad(int d, const real w[MAXD][3], const real dw[MAXD][3], const int o[MAXD],
                        real g[MAXD]) {
    for (int k = 0; k < d; ++k) {
        real s = dw[k][o[k]];
        for (int j = 0; j < d; ++j)
            if (j != k) s *= w[j][o[j]];
        g[k] = s;
    }
}

static int finite_arr(const real* a, int64_t n) {
    for (int64_t i = 0; i < n; ++i)
        if (!isfinite((double)a[i])) return 0;
    return 1;
}

/* ----------------------------------------------------- B-spline, material */

/* R1: quadratic B-spline, f in [1/2, 3/2):
   N0 = 1/2 (3/2 - f)^2, N1 = 3/4 - (f - 1)^2, N2 = 1/2 (f - 1/2)^2 */
void oracle_bspline(real f, real w[3], real dw[3]) {
    w[0] = (real)0.5 * ((real)1.5 - f) * ((real)1.5 - f);
    w[1] = (real)0.75 - (f - 1) * (f - 1);
    w[2] = (real)0.5 * (f - (real)0.5) * (f - (real)0.5);
    dw[0] = f - (real)1.5;
    dw[1] = -2 * (f - 1);
    dw[2] = f - (real)0.5;
}

/* R3: mu = E / (2 (1 + nu)), lambda = E nu / ((1 + nu)(1 - 2 nu)) */
void oracle_lame(const oracle_cfg* c, real* mu, real* lam) {
    *mu = (real)(c->E / (2.0 * (1.0 + c->nu)));
    *lam = (real)(c->E * c->nu / ((1.0 + c->nu) * (1.0 - 2.0 * c->nu)));
}

/* 2x2 polar rotation R = [[cs, -sn], [sn, cs]], (cs, sn) = (a, b)/r,
   a = F00 + F11, b = F10 - F01 (R2) */
static int polar2(const real* F, real* R, real* a, real* b, real* r2) {
    *a = F[0] + F[3];
    *b = F[2] - F[1];
    *r2 = (*a) * (*a) + (*b) * (*b);
    if (!(*r2 > 0)) return ORACLE_NONFINITE; /* R14: no silent guard */
    real r = sqrt(*r2);
    real cs = *a / r, sn = *b / r;
    R[0] = cs; R[1] = -sn; R[2] = sn; R[3] = cs;
    return ORACLE_OK;
}

/* R2: Neo-Hookean tau = mu (F F^T - I) + lambda ln J I;
       fixed-corotated (2D) tau = 2 mu (F - R) F^T + lambda (J - 1) J I */
/* R23: a fluid particle keeps only the volumetric term of the model (mu = 0) */
static int stress_m(const oracle_cfg* c, const real* F, int fluid, real* tau);
int oracle_stress(const oracle_cfg* c, const real* F, real* tau) { return stress_m(c, F, 0, tau); }

static int stress_m(const oracle_cfg* c, const real* F, int fluid, real* tau) {
    const int d = c->dim;
    real mu, lam;
    oracle_lame(c, &mu, &lam);
    if (fluid) mu = 0;
    real J = det(d, F);
    if (c->model == 0) {
        if (!(J > 0)) return ORACLE_NONFINITE;
        real FFt[9];
        matmul_bt(d, F, F, FFt);
        real lnJ = log(J);
        for (int i = 0; i < d; ++i)
            for (int j = 0; j < d; ++j)
                tau[i * d + j] = mu * (FFt[i * d + j] - (i == j)) + (i == j ? lam * lnJ : 0);
        return ORACLE_OK;
    }
    if (c->model == 1 && d == 2) {
        real R[4], a, b, r2;
        int st = polar2(F, R, &a, &b, &r2);
        if (st) return st;
        real FmR[4], M[4];
        for (int i = 0; i < 4; ++i) FmR[i] = F[i] - R[i];
        matmul_bt(2, FmR, F, M);
        for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 2; ++j)
                tau[i * 2 + j] = 2 * mu * M[i * 2 + j] + (i == j ? lam * (J - 1) * J : 0);
        return ORACLE_OK;
    }
    return ORACLE_INVALID;
}

/* strain energy whose first Piola stress P satisfies tau = P F^T:
   NH  psi = mu/2 (tr(F^T F) - d) - mu ln J + lambda/2 (ln J)^2
   FCR psi = mu |F - R|^2 + lambda/2 (J - 1)^2 */
int oracle_energy(const oracle_cfg* c, const real* F, real* psi) {
    const int d = c->dim;
    real mu, lam;
    oracle_lame(c, &mu, &lam);
    real J = det(d, F);
    if (c->model == 0) {
        if (!(J > 0)) return ORACLE_NONFINITE;
        real tr = 0;
        for (int i = 0; i < d * d; ++i) tr += F[i] * F[i];
        real lnJ = log(J);
        *psi = mu / 2 * (tr - d) - mu * lnJ + lam / 2 * lnJ * lnJ;
        return ORACLE_OK;
    }
    if (c->model == 1 && d == 2) {
        real R[4], a, b, r2;
        int st = polar2(F, R, &a, &b, &r2);
        if (st) return st;
        real s = 0;
        for (int i = 0; i < 4; ++i) s += (F[i] - R[i]) * (F[i] - R[i]);
        *psi = mu * s + lam / 2 * (J - 1) * (J - 1);
        return ORACLE_OK;
    }
    return ORACLE_INVALID;
}

/* Reverse of oracle_stress (SURVEY.md A.3 "tau-adjoints"):
   NH : Fbar += mu (tb + tb^T) F + lambda tr(tb) F^{-T}
   FCR: Fbar += 2mu (tb + tb^T) F - 2mu tb^T R + lambda (2J - 1) tr(tb) cof(F)
        plus the rotation path Rbar = -2mu tb F through psi = atan2(b, a). */
static int stress_adj_m(const oracle_cfg* c, const real* F, const real* tb, int fluid, real* Fb);
int oracle_stress_adj(const oracle_cfg* c, const real* F, const real* tb, real* Fb) {
    return stress_adj_m(c, F, tb, 0, Fb);
}

static int stress_adj_m(const oracle_cfg* c, const real* F, const real* tb, int fluid, real* Fb) {
    const int d = c->dim;
    real mu, lam;
    oracle_lame(c, &mu, &lam);
    if (fluid) mu = 0;
    real J = det(d, F);
    real S[9], SF[9], K[9];
    for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j) S[i * d + j] = tb[i * d + j] + tb[j * d + i];
    matmul(d, S, F, SF);
    cofactor(d, F, K);
    real trb = 0;
    for (int i = 0; i < d; ++i) trb += tb[i * d + i];
    if (c->model == 0) {
        if (!(J > 0)) return ORACLE_NONFINITE;
        for (int i = 0; i < d * d; ++i) Fb[i] += mu * SF[i] + lam * trb * K[i] / J;
        return ORACLE_OK;
    }
    if (c->model == 1 && d == 2) {
        real R[4], a, b, r2;
        int st = polar2(F, R, &a, &b, &r2);
        if (st) return st;
        real tbTR[4], Rb[4];
        matmul_at(2, tb, R, tbTR);
        matmul(2, tb, F, Rb);
        for (int i = 0; i < 4; ++i) {
            Fb[i] += 2 * mu * SF[i] - 2 * mu * tbTR[i] + lam * (2 * J - 1) * trb * K[i];
            Rb[i] *= -2 * mu;
        }
        real cs = R[0], sn = R[2];
        /* dR/dpsi = [[-sn, -cs], [cs, -sn]] */
        real psib = -sn * Rb[0] - cs * Rb[1] + cs * Rb[2] - sn * Rb[3];
        Fb[0] -= psib * b / r2;
        Fb[3] -= psib * b / r2;
        Fb[2] += psib * a / r2;
        Fb[1] -= psib * a / r2;
        return ORACLE_OK;
    }
    return ORACLE_INVALID;
}

/* ------------------------------------------------------------ controller */

/* R9: controller on sinusoid features phi_j(t) = sin(omega t dt + 2 pi j / n_sin), plus,
   closed loop (R22), the observation o_t of S_t:  input u = [phi(t), o_t] (n_in values);
   H > 0: alpha = tanh(W2 tanh(W1 u + b1) + b2); H = 0: alpha = tanh(W u + b).
   theta = [W1 (H x n_in), b1 (H), W2 (n_act x H), b2 (n_act)] (or [W (n_act x n_in), b]). */
int oracle_n_obs(const oracle_cfg* c) { return c->closed_loop ? 2 * c->dim * c->n_act : 0; }

static int n_in(const oracle_cfg* c) { return c->n_sin + oracle_n_obs(c); }

int64_t oracle_n_theta(const oracle_cfg* c) {
    int64_t H = c->hidden, S = n_in(c), A = c->n_act;
    return H > 0 ? H * S + H + A * H + A : A * S + A;
}

/* u = [phi(t), o_t]; o = NULL -> zeros */
static void inputs(const oracle_cfg* c, int32_t t, const real* obs, real* u) {
    for (int j = 0; j < c->n_sin; ++j)
        u[j] = sin((real)(c->omega * t * c->dt) + (real)(2.0 * M_PI * j / c->n_sin));
    for (int j = 0; j < oracle_n_obs(c); ++j) u[c->n_sin + j] = obs ? obs[j] : 0;
}

void oracle_controller_obs(const oracle_cfg* c, const real* theta, int32_t t, const real* obs,
                           real* alpha) {
    const int S = n_in(c), H = c->hidden, A = c->n_act;
    real u[1024], h[1024];
    inputs(c, t, obs, u);
    if (H > 0) {
        const real *W1 = theta, *b1 = W1 + H * S, *W2 = b1 + H, *b2 = W2 + A * H;
        for (int i = 0; i < H; ++i) {
            real z = b1[i];
            for (int j = 0; j < S; ++j) z += W1[i * S + j] * u[j];
            h[i] = tanh(z);
        }
        for (int a = 0; a < A; ++a) {
            real z = b2[a];
            for (int i = 0; i < H; ++i) z += W2[a * H + i] * h[i];
            alpha[a] = tanh(z);
        }
    } else {
        const real *W = theta, *b = W + A * S;
        for (int a = 0; a < A; ++a) {
            real z = b[a];
            for (int j = 0; j < S; ++j) z += W[a * S + j] * u[j];
            alpha[a] = tanh(z);
        }
    }
}

void oracle_controller(const oracle_cfg* c, const real* theta, int32_t t, real* alpha) {
    oracle_controller_obs(c, theta, t, NULL, alpha);
}

/* SURVEY.md A.3 "Controller": theta_bar += (d alpha_t / d theta)^T alpha_bar_t;
   closed loop: obs_bar = (d alpha_t / d o_t)^T alpha_bar_t */
void oracle_controller_obs_adj(const oracle_cfg* c, const real* theta, int32_t t, const real* obs,
                               const real* ab, real* thb, real* obs_bar) {
    const int S = n_in(c), H = c->hidden, A = c->n_act, ns = c->n_sin;
    real u[1024], h[1024], alpha[256], z2b[256], hb[1024], ub[1024];
    inputs(c, t, obs, u);
    oracle_controller_obs(c, theta, t, obs, alpha);
    for (int j = 0; j < S; ++j) ub[j] = 0;
    if (H > 0) {
        const real *W1 = theta, *b1 = W1 + H * S, *W2 = b1 + H;
        real *W1b = thb, *b1b = W1b + H * S, *W2b = b1b + H, *b2b = W2b + A * H;
        for (int i = 0; i < H; ++i) {
            real z = b1[i];
            for (int j = 0; j < S; ++j) z += W1[i * S + j] * u[j];
            h[i] = tanh(z);
        }
        for (int a = 0; a < A; ++a) {
            z2b[a] = ab[a] * (1 - alpha[a] * alpha[a]);
            b2b[a] += z2b[a];
            for (int i = 0; i < H; ++i) W2b[a * H + i] += z2b[a] * h[i];
        }
        for (int i = 0; i < H; ++i) {
            real s = 0;
            for (int a = 0; a < A; ++a) s += W2[a * H + i] * z2b[a];
            hb[i] = s * (1 - h[i] * h[i]);
            b1b[i] += hb[i];
            for (int j = 0; j < S; ++j) W1b[i * S + j] += hb[i] * u[j];
            for (int j = 0; j < S; ++j) ub[j] += W1[i * S + j] * hb[i];
        }
    } else {
        const real* W = theta;
        real *Wb = thb, *bb = Wb + A * S;
        for (int a = 0; a < A; ++a) {
            real zb = ab[a] * (1 - alpha[a] * alpha[a]);
            bb[a] += zb;
            for (int j = 0; j < S; ++j) Wb[a * S + j] += zb * u[j];
            for (int j = 0; j < S; ++j) ub[j] += W[a * S + j] * zb;
        }
    }
    if (obs_bar)
        for (int j = 0; j < oracle_n_obs(c); ++j) obs_bar[j] = ub[ns + j];
}

void oracle_controller_adj(const oracle_cfg* c, const real* theta, int32_t t,
                           const real* ab, real* thb) {
    oracle_controller_obs_adj(c, theta, t, NULL, ab, thb, NULL);
}

/* R22: o[a] = (s_x (mean_a x - mean x), s_v mean_a v), a = 0..n_act-1 (equal particle
   masses, R4: the means are plain averages over particles) */
void oracle_observe(const oracle_cfg* c, int64_t N, const real* x, const real* v,
                    const int32_t* aid, real* obs) {
    const int d = c->dim, A = c->n_act;
    real xm[MAXD] = {0};
    for (int64_t p = 0; p < N; ++p)
        for (int k = 0; k < d; ++k) xm[k] += x[p * d + k];
    for (int k = 0; k < d; ++k) xm[k] /= (real)N;
    for (int a = 0; a < A; ++a) {
        real sx[MAXD] = {0}, sv[MAXD] = {0};
        int64_t n = 0;
        for (int64_t p = 0; p < N; ++p) {
            if (!aid || aid[p] != a) continue;
            ++n;
            for (int k = 0; k < d; ++k) { sx[k] += x[p * d + k]; sv[k] += v[p * d + k]; }
        }
        for (int k = 0; k < d; ++k) {
            obs[a * 2 * d + k] = n ? (real)c->obs_sx * (sx[k] / (real)n - xm[k]) : 0;
            obs[a * 2 * d + d + k] = n ? (real)c->obs_sv * (sv[k] / (real)n) : 0;
        }
    }
}

void oracle_observe_adj(const oracle_cfg* c, int64_t N, const int32_t* aid, const real* ob,
                        real* xb, real* vb) {
    const int d = c->dim, A = c->n_act;
    for (int a = 0; a < A; ++a) {
        int64_t n = 0;
        for (int64_t p = 0; p < N; ++p) n += (aid && aid[p] == a);
        if (!n) continue;  /* o[a] = 0 for an empty group: no gradient */
        for (int64_t p = 0; p < N; ++p) {
            for (int k = 0; k < d; ++k) xb[p * d + k] -= (real)c->obs_sx * ob[a * 2 * d + k] / (real)N;
            if (aid[p] != a) continue;
            for (int k = 0; k < d; ++k) {
                xb[p * d + k] += (real)c->obs_sx * ob[a * 2 * d + k] / (real)n;
                vb[p * d + k] += (real)c->obs_sv * ob[a * 2 * d + d + k] / (real)n;
            }
        }
    }
}

/* --------------------------------------------------------- forward stages */

/* Kirchhoff stress including actuation (R8): tau += kappa a (F e)(F e)^T */
static int total_stress(const oracle_cfg* c, const real* Ft, int32_t aid, const real* alpha,
                        int fluid, real* tau) {
    const int d = c->dim;
    int st = stress_m(c, Ft, fluid, tau);
    if (st) return st;
    if (aid >= 0) {
        real q[MAXD];
        for (int i = 0; i < d; ++i) q[i] = Ft[i * d + c->act_axis];
        real s = (real)c->kappa * alpha[aid];
        for (int i = 0; i < d; ++i)
            for (int j = 0; j < d; ++j) tau[i * d + j] += s * q[i] * q[j];
    }
    return ORACLE_OK;
}

/* clear_grid + p2g.  Per particle:
   Ft = (I + dt C) F;  tau = tau(Ft) [+ actuation];
   A = -dt V 4/dx^2 tau + m C;
   for o: P[b+o] += W_o (m v + A (o - f) dx),  M[b+o] += W_o m;   F_next = Ft */
int oracle_p2g(const oracle_cfg* c, int64_t N, const real* x, const real* v, const real* C,
               const real* F, const int32_t* aid, const real* alpha, real* grid, real* F_next) {
    const int d = c->dim, dd = d * d, nst = ipow3(d);
    const real dx = (real)1 / c->n_grid, inv_dx = (real)c->n_grid;
    const real m = (real)c->p_mass, V = (real)c->p_vol, dt = (real)c->dt;
    memset(grid, 0, sizeof(real) * n_nodes(c) * (d + 1)); /* clear_grid */
    for (int64_t p = 0; p < N; ++p) {
        int base[MAXD];
        real fx[MAXD], w[MAXD][3], dw[MAXD][3];
        int st = stencil(c, x + p * d, base, fx, w, dw);
        if (st) return st;
        const real *Cp = C + p * dd, *Fp = F + p * dd, *vp = v + p * d;
        real G[9], Ft[9], tau[9], A[9];
        for (int i = 0; i < dd; ++i) G[i] = dt * Cp[i];
        for (int i = 0; i < d; ++i) G[i * d + i] += 1;
        matmul(d, G, Fp, Ft);
        const int fluid = c->mat && c->mat[p] == 1;
        st = total_stress(c, Ft, aid ? aid[p] : -1, alpha, fluid, tau);
        if (st) return st;
        for (int i = 0; i < dd; ++i) A[i] = -dt * V * 4 * inv_dx * inv_dx * tau[i] + m * Cp[i];
        for (int s = 0; s < nst; ++s) {
            int o[MAXD], node[MAXD];
            offset_of(d, s, o);
            real W = weight(d, w, o), dpos[MAXD];
            for (int k = 0; k < d; ++k) {
                dpos[k] = ((real)o[k] - fx[k]) * dx;
                node[k] = base[k] + o[k];
            }
            real* g = grid + node_index(c, node) * (d + 1);
            for (int a = 0; a < d; ++a) {
                real Ad = 0;
                for (int b = 0; b < d; ++b) Ad += A[a * d + b] * dpos[b];
                g[a] += W * (m * vp[a] + Ad);
            }
            g[d] += W * m;
        }
        if (F_next) {
            if (fluid) {  /* R23: F_{t+1} = J^(1/d) I (the fluid forgets its shear) */
                const real s = pow(det(d, Ft), (real)1 / d);
                for (int i = 0; i < dd; ++i) F_next[p * dd + i] = (i % (d + 1) == 0) ? s : 0;
            } else {
                memcpy(F_next + p * dd, Ft, sizeof(real) * dd);
            }
        }
    }
    return ORACLE_OK;
}

/* per-node grid velocity before the boundary condition, and the sticky-wall
   select of R6: z = OR_k (i_k < beta and u_k < 0) or (i_k > n - beta and u_k > 0) */
static int grid_node_velocity(const oracle_cfg* c, int64_t lin, const real* g, real* u0, real* u1) {
    const int d = c->dim;
    int i[MAXD];
    node_coords(c, lin, i);
    real denom = g[d] + (real)c->eps_mass;
    for (int k = 0; k < d; ++k) {
        u0[k] = g[k] / denom;
        u1[k] = u0[k];
    }
    u1[1] -= (real)c->dt * (real)c->gravity; /* gravity along -y (R7) */
    int z = 0;
    for (int k = 0; k < d; ++k) {
        if (i[k] < c->bound && u1[k] < 0) z = 1;
        if (i[k] > c->n_grid - c->bound && u1[k] > 0) z = 1;
    }
    return z;
}

/* grid_op: u = P/(M + eps) - dt g e_y; U = z ? 0 : u */
void oracle_grid_op(const oracle_cfg* c, const real* grid, real* U) {
    const int d = c->dim;
    const int64_t nn = n_nodes(c);
    for (int64_t lin = 0; lin < nn; ++lin) {
        real u0[MAXD], u1[MAXD];
        int z = grid_node_velocity(c, lin, grid + lin * (d + 1), u0, u1);
        for (int k = 0; k < d; ++k) U[lin * d + k] = z ? 0 : u1[k];
    }
}

/* g2p: v' = sum W U;  C' = 4/dx sum W U (o - f)^T;  x' = x + dt v' */
int oracle_g2p(const oracle_cfg* c, int64_t N, const real* x, const real* U, real* xn, real* vn,
               real* Cn) {
    const int d = c->dim, dd = d * d, nst = ipow3(d);
    const real inv_dx = (real)c->n_grid, dt = (real)c->dt;
    for (int64_t p = 0; p < N; ++p) {
        int base[MAXD];
        real fx[MAXD], w[MAXD][3], dw[MAXD][3];
        int st = stencil(c, x + p * d, base, fx, w, dw);
        if (st) return st;
        real nv[MAXD] = {0, 0, 0}, nC[9] = {0};
        for (int s = 0; s < nst; ++s) {
            int o[MAXD], node[MAXD];
            offset_of(d, s, o);
            real W = weight(d, w, o);
            for (int k = 0; k < d; ++k) node[k] = base[k] + o[k];
            const real* u = U + node_index(c, node) * d;
            for (int a = 0; a < d; ++a) {
                nv[a] += W * u[a];
                for (int b = 0; b < d; ++b) nC[a * d + b] += 4 * inv_dx * W * u[a] * ((real)o[b] - fx[b]);
            }
        }
        for (int a = 0; a < d; ++a) {
            vn[p * d + a] = nv[a];
            xn[p * d + a] = x[p * d + a] + dt * nv[a];
        }
        memcpy(Cn + p * dd, nC, sizeof(real) * dd);
    }
    return ORACLE_OK;
}

/* advance() */
int oracle_step(const oracle_cfg* c, int64_t N, const real* x, const real* v, const real* C,
                const real* F, const int32_t* aid, const real* alpha, real* xn, real* vn,
                real* Cn, real* Fn) {
    const int d = c->dim;
    const int64_t nn = n_nodes(c);
    real* grid = (real*)malloc(sizeof(real) * nn * (d + 1));
    real* U = (real*)malloc(sizeof(real) * nn * d);
    int st = oracle_p2g(c, N, x, v, C, F, aid, alpha, grid, Fn);
    if (!st) {
        oracle_grid_op(c, grid, U);
        st = oracle_g2p(c, N, x, U, xn, vn, Cn);
    }
    free(grid);
    free(U);
    return st;
}

/* --------------------------------------------------------- reverse stages */

/* g2p.grad.  Given (xb', vb', Cb') of S_{t+1}:
   vh = vb' + dt xb';  for o:  Ub[b+o] += W (vh + 4/dx Cb' (o - f));
   Wb = U.vh + 4/dx U^T Cb' (o - f);  fb += Wb dW/df - 4/dx W Cb'^T U;
   xb_t (partial) = xb' + fb/dx.   U_bar accumulates; xb is written. */
int oracle_g2p_adj(const oracle_cfg* c, int64_t N, const real* x, const real* U,
                   const real* xbn, const real* vbn, const real* Cbn, real* Ub, real* xb) {
    const int d = c->dim, dd = d * d, nst = ipow3(d);
    const real inv_dx = (real)c->n_grid, dt = (real)c->dt;
    for (int64_t p = 0; p < N; ++p) {
        int base[MAXD];
        real fx[MAXD], w[MAXD][3], dw[MAXD][3];
        int st = stencil(c, x + p * d, base, fx, w, dw);
        if (st) return st;
        const real* Cb = Cbn + p * dd;
        real vh[MAXD], fb[MAXD] = {0, 0, 0};
        for (int a = 0; a < d; ++a) vh[a] = vbn[p * d + a] + dt * xbn[p * d + a];
        for (int s = 0; s < nst; ++s) {
            int o[MAXD], node[MAXD];
            offset_of(d, s, o);
            real W = weight(d, w, o), gW[MAXD], om[MAXD];
            weight_grad(d, w, dw, o, gW);
            for (int k = 0; k < d; ++k) {
                node[k] = base[k] + o[k];
                om[k] = (real)o[k] - fx[k];
            }
            int64_t li = node_index(c, node);
            const real* u = U + li * d;
            real Wb = 0;
            for (int a = 0; a < d; ++a) {
                real Cbom = 0;
                for (int b = 0; b < d; ++b) Cbom += Cb[a * d + b] * om[b];
                Ub[li * d + a] += W * (vh[a] + 4 * inv_dx * Cbom);
                Wb += u[a] * vh[a] + 4 * inv_dx * u[a] * Cbom;
            }
            for (int k = 0; k < d; ++k) {
                real CbTu = 0;
                for (int a = 0; a < d; ++a) CbTu += Cb[a * d + k] * u[a];
                fb[k] += Wb * gW[k] - 4 * inv_dx * W * CbTu;
            }
        }
        for (int k = 0; k < d; ++k) xb[p * d + k] = xbn[p * d + k] + inv_dx * fb[k];
    }
    return ORACLE_OK;
}

/* grid_op.grad: select rule -- no gradient through a zeroed
   node, none through the condition:  ub = z ? 0 : Ub;
   Pb = ub / (M + eps);  Mb = -(ub . u0) / (M + eps).   grid_bar is written. */
void oracle_grid_op_adj(const oracle_cfg* c, const real* grid, const real* Ub, real* gb) {
    const int d = c->dim;
    const int64_t nn = n_nodes(c);
    for (int64_t lin = 0; lin < nn; ++lin) {
        const real* g = grid + lin * (d + 1);
        real u0[MAXD], u1[MAXD];
        int z = grid_node_velocity(c, lin, g, u0, u1);
        real denom = g[d] + (real)c->eps_mass, dot = 0;
        for (int k = 0; k < d; ++k) {
            real ub = z ? 0 : Ub[lin * d + k];
            gb[lin * (d + 1) + k] = ub / denom;
            dot += ub * u0[k];
        }
        gb[lin * (d + 1) + d] = -dot / denom;
    }
}

/* p2g.grad.  Recomputes Ft, tau, A; gathers (Pb, Mb):
   vb = sum W m Pb;  Ab = sum W Pb dpos^T;  Wb = Pb.(m v + A dpos) + Mb m;
   fb += Wb dW/df - dx W A^T Pb;  Cb = m Ab;  taub = -dt V 4/dx^2 Ab;
   Ftb = Fb' + tau-adjoint + actuation adjoint;  Fb = (I + dt C)^T Ftb;
   Cb += dt Ftb F^T;  xb += fb/dx;  alpha_bar[aid] += kappa q^T taub q.
   xb and alpha_bar accumulate; vb, Cb, Fb are written. */
int oracle_p2g_adj(const oracle_cfg* c, int64_t N, const real* x, const real* v, const real* C,
                   const real* F, const int32_t* aid, const real* alpha, const real* gb,
                   const real* Fbn, real* xb, real* vb, real* Cb, real* Fb, real* alpha_bar) {
    const int d = c->dim, dd = d * d, nst = ipow3(d);
    const real dx = (real)1 / c->n_grid, inv_dx = (real)c->n_grid;
    const real m = (real)c->p_mass, V = (real)c->p_vol, dt = (real)c->dt;
    for (int64_t p = 0; p < N; ++p) {
        int base[MAXD];
        real fx[MAXD], w[MAXD][3], dw[MAXD][3];
        int st = stencil(c, x + p * d, base, fx, w, dw);
        if (st) return st;
        const real *Cp = C + p * dd, *Fp = F + p * dd, *vp = v + p * d;
        const int32_t a_id = aid ? aid[p] : -1;
        real G[9], Ft[9], tau[9], A[9];
        for (int i = 0; i < dd; ++i) G[i] = dt * Cp[i];
        for (int i = 0; i < d; ++i) G[i * d + i] += 1;
        matmul(d, G, Fp, Ft);
        const int fluid = c->mat && c->mat[p] == 1;
        st = total_stress(c, Ft, a_id, alpha, fluid, tau);
        if (st) return st;
        for (int i = 0; i < dd; ++i) A[i] = -dt * V * 4 * inv_dx * inv_dx * tau[i] + m * Cp[i];

        real vbp[MAXD] = {0, 0, 0}, Ab[9] = {0}, fb[MAXD] = {0, 0, 0};
        for (int s = 0; s < nst; ++s) {
            int o[MAXD], node[MAXD];
            offset_of(d, s, o);
            real W = weight(d, w, o), gW[MAXD], dpos[MAXD];
            weight_grad(d, w, dw, o, gW);
            for (int k = 0; k < d; ++k) {
                node[k] = base[k] + o[k];
                dpos[k] = ((real)o[k] - fx[k]) * dx;
            }
            const real* g = gb + node_index(c, node) * (d + 1);
            real Wb = g[d] * m;
            for (int a = 0; a < d; ++a) {
                vbp[a] += W * m * g[a];
                real mom = m * vp[a];
                for (int b = 0; b < d; ++b) {
                    Ab[a * d + b] += W * g[a] * dpos[b];
                    mom += A[a * d + b] * dpos[b];
                }
                Wb += g[a] * mom;
            }
            for (int k = 0; k < d; ++k) {
                real ATPb = 0;
                for (int a = 0; a < d; ++a) ATPb += A[a * d + k] * g[a];
                fb[k] += Wb * gW[k] - dx * W * ATPb;
            }
        }
        real taub[9], Ftb[9], Cbp[9];
        for (int i = 0; i < dd; ++i) {
            Cbp[i] = m * Ab[i];
            taub[i] = -dt * V * 4 * inv_dx * inv_dx * Ab[i];
            Ftb[i] = Fbn ? Fbn[p * dd + i] : 0;
        }
        if (fluid) {  /* reverse of F_{t+1} = J^(1/d) I: Ftb = (1/d) J^(1/d - 1) tr(Fb') cof(Ft) */
            const real J = det(d, Ft);
            real K[9], tr = 0;
            cofactor(d, Ft, K);
            for (int i = 0; i < d; ++i) tr += Ftb[i * d + i];
            const real s = pow(J, (real)1 / d - 1) * tr / d;
            for (int i = 0; i < dd; ++i) Ftb[i] = s * K[i];
        }
        st = stress_adj_m(c, Ft, taub, fluid, Ftb);
        if (st) return st;
        if (a_id >= 0) {
            real q[MAXD], sq[MAXD];
            const int e = c->act_axis;
            for (int i = 0; i < d; ++i) q[i] = Ft[i * d + e];
            real qtq = 0;
            for (int i = 0; i < d; ++i) {
                sq[i] = 0;
                for (int j = 0; j < d; ++j) {
                    qtq += q[i] * taub[i * d + j] * q[j];
                    sq[i] += (taub[i * d + j] + taub[j * d + i]) * q[j];
                }
            }
            alpha_bar[a_id] += (real)c->kappa * qtq;
            for (int i = 0; i < d; ++i) Ftb[i * d + e] += (real)c->kappa * alpha[a_id] * sq[i];
        }
        real Fbp[9], FtbFt[9];
        matmul_at(d, G, Ftb, Fbp);  /* (I + dt C)^T Ftb */
        matmul_bt(d, Ftb, Fp, FtbFt); /* Ftb F^T */
        for (int i = 0; i < dd; ++i) {
            Fb[p * dd + i] = Fbp[i];
            Cb[p * dd + i] = Cbp[i] + dt * FtbFt[i];
        }
        for (int k = 0; k < d; ++k) {
            vb[p * d + k] = vbp[k];
            xb[p * d + k] += inv_dx * fb[k];
        }
    }
    return ORACLE_OK;
}

/* advance_grad(): recompute the grid (clear_grid, p2g, grid_op),
   then g2p.grad, grid_op.grad, p2g.grad.  U_bar is zeroed first (clear_grid's
   adjoint zeroing).  alpha_bar accumulates. */
int oracle_step_adj(const oracle_cfg* c, int64_t N, const real* x, const real* v, const real* C,
                    const real* F, const int32_t* aid, const real* alpha, const real* xbn,
                    const real* vbn, const real* Cbn, const real* Fbn, real* xb, real* vb,
                    real* Cb, real* Fb, real* alpha_bar) {
    const int d = c->dim;
    const int64_t nn = n_nodes(c);
    real* grid = (real*)malloc(sizeof(real) * nn * (d + 1));
    real* gb = (real*)malloc(sizeof(real) * nn * (d + 1));
    real* U = (real*)malloc(sizeof(real) * nn * d);
    real* Ub = (real*)calloc((size_t)(nn * d), sizeof(real));
    int st = oracle_p2g(c, N, x, v, C, F, aid, alpha, grid, NULL);
    if (!st) {
        oracle_grid_op(c, grid, U);
        st = oracle_g2p_adj(c, N, x, U, xbn, vbn, Cbn, Ub, xb);
    }
    if (!st) {
        oracle_grid_op_adj(c, grid, Ub, gb);
        st = oracle_p2g_adj(c, N, x, v, C, F, aid, alpha, gb, Fbn, xb, vb, Cb, Fb, alpha_bar);
    }
    free(grid);
    free(gb);
    free(U);
    free(Ub);
    return st;
}

/* ------------------------------------------------------------------ loss */

/* R10: kind 0: L = |xbar - x*|^2;  kind 1: L = -xbar . e_0;
   xbar = sum m x / sum m.  Seeds (A.4): xb_p = dL/dx_p. */
int oracle_loss(const oracle_cfg* c, int32_t kind, const real* target, int64_t N, const real* x,
                real* L, real* xb) {
    const int d = c->dim;
    const real m = (real)c->p_mass, Mtot = m * (real)N;
    real com[MAXD] = {0, 0, 0}, g[MAXD] = {0, 0, 0};
    for (int64_t p = 0; p < N; ++p)
        for (int k = 0; k < d; ++k) com[k] += m * x[p * d + k];
    for (int k = 0; k < d; ++k) com[k] /= Mtot;
    real l = 0;
    if (kind == 0) {
        for (int k = 0; k < d; ++k) {
            l += (com[k] - target[k]) * (com[k] - target[k]);
            g[k] = 2 * (com[k] - target[k]);
        }
    } else if (kind == 1) {
        l = -com[0];
        g[0] = -1;
    } else {
        return ORACLE_INVALID;
    }
    *L = l;
    if (xb)
        for (int64_t p = 0; p < N; ++p)
            for (int k = 0; k < d; ++k) xb[p * d + k] = g[k] * m / Mtot;
    return isfinite((double)l) ? ORACLE_OK : ORACLE_NONFINITE;
}

/* ------------------------------------------------------------- episode */

typedef struct {
    real *x, *v, *C, *F;
} state_t;

static state_t state_alloc(int d, int64_t N) {
    state_t s;
    s.x = (real*)malloc(sizeof(real) * N * d);
    s.v = (real*)malloc(sizeof(real) * N * d);
    s.C = (real*)malloc(sizeof(real) * N * d * d);
    s.F = (real*)malloc(sizeof(real) * N * d * d);
    return s;
}
static void state_free(state_t* s) {
    free(s->x); free(s->v); free(s->C); free(s->F);
}
static void state_copy(int d, int64_t N, state_t* dst, const real* x, const real* v,
                       const real* C, const real* F) {
    memcpy(dst->x, x, sizeof(real) * N * d);
    memcpy(dst->v, v, sizeof(real) * N * d);
    memcpy(dst->C, C, sizeof(real) * N * d * d);
    memcpy(dst->F, F, sizeof(real) * N * d * d);
}
static int state_finite(int d, int64_t N, const state_t* s) {
    return finite_arr(s->x, N * d) && finite_arr(s->v, N * d) && finite_arr(s->C, N * d * d) &&
           finite_arr(s->F, N * d * d);
}

/* The tape over T advance() calls with segment-wise recomputation
   (P:594-598): the first state of every k-step segment is stored; in the
   reverse sweep each segment is re-simulated from its checkpoint into a
   k-state window and advance_grad() is replayed from its last step down. */
int oracle_run(const oracle_cfg* c, int64_t N, int32_t T, int32_t k, const real* x0,
               const real* v0, const real* C0, const real* F0, const int32_t* aid,
               const real* theta, int32_t loss_kind, const real* target, real* xT, real* vT,
               real* CT, real* FT, real* L, real* dx0, real* dv0, real* dC0, real* dF0,
               real* dtheta) {
    const int d = c->dim, dd = d * d;
    if (T < 0 || k < 1 || N < 1) return ORACLE_INVALID;
    const int A = c->n_act > 0 ? c->n_act : 1;
    const int nseg = T > 0 ? (T + k - 1) / k : 0;
    int st = ORACLE_OK;
    real* alpha = (real*)calloc((size_t)(T > 0 ? T : 1) * A, sizeof(real));
    real* alpha_bar = (real*)calloc((size_t)(T > 0 ? T : 1) * A, sizeof(real));
    const int closed = c->closed_loop && c->n_act > 0;
    const int NO = oracle_n_obs(c) > 0 ? oracle_n_obs(c) : 1;
    real* obs = (real*)calloc((size_t)(T > 0 ? T : 1) * NO, sizeof(real));
    real* obs_bar = (real*)calloc((size_t)NO, sizeof(real));
    real* thb = (real*)calloc((size_t)(oracle_n_theta(c) > 0 ? oracle_n_theta(c) : 1), sizeof(real));
    if (c->n_act > 0 && !closed)
        for (int t = 0; t < T; ++t) oracle_controller(c, theta, t, alpha + (int64_t)t * A);

    state_t* ckpt = (state_t*)malloc(sizeof(state_t) * (nseg > 0 ? nseg : 1));
    for (int s = 0; s < nseg; ++s) ckpt[s] = state_alloc(d, N);
    state_t cur = state_alloc(d, N), nxt = state_alloc(d, N);
    state_copy(d, N, &cur, x0, v0, C0, F0);

    /* forward (the tape records t and the checkpoint slot) */
    for (int t = 0; t < T && !st; ++t) {
        if (t % k == 0) state_copy(d, N, &ckpt[t / k], cur.x, cur.v, cur.C, cur.F);
        if (closed) {  /* R22: alpha_t from the observation of S_t */
            oracle_observe(c, N, cur.x, cur.v, aid, obs + (int64_t)t * NO);
            oracle_controller_obs(c, theta, t, obs + (int64_t)t * NO, alpha + (int64_t)t * A);
        }
        st = oracle_step(c, N, cur.x, cur.v, cur.C, cur.F, aid, alpha + (int64_t)t * A, nxt.x,
                         nxt.v, nxt.C, nxt.F);
        if (!st && !state_finite(d, N, &nxt)) st = ORACLE_NONFINITE;
        state_t tmp = cur; cur = nxt; nxt = tmp;
    }
    if (!st) {
        if (xT) memcpy(xT, cur.x, sizeof(real) * N * d);
        if (vT) memcpy(vT, cur.v, sizeof(real) * N * d);
        if (CT) memcpy(CT, cur.C, sizeof(real) * N * dd);
        if (FT) memcpy(FT, cur.F, sizeof(real) * N * dd);
    }

    /* loss and seed: adjoint of S_T = (dL/dx_T, 0, 0, 0) */
    state_t bar = state_alloc(d, N), barn = state_alloc(d, N);
    real l = 0;
    if (!st) st = oracle_loss(c, loss_kind, target, N, cur.x, &l, bar.x);
    if (L) *L = l;
    memset(bar.v, 0, sizeof(real) * N * d);
    memset(bar.C, 0, sizeof(real) * N * dd);
    memset(bar.F, 0, sizeof(real) * N * dd);

    /* reverse sweep */
    state_t* win = (state_t*)malloc(sizeof(state_t) * k);
    for (int i = 0; i < k; ++i) win[i] = state_alloc(d, N);
    for (int s = nseg - 1; s >= 0 && !st; --s) {
        int t0 = s * k, t1 = t0 + k < T ? t0 + k : T;
        state_copy(d, N, &win[0], ckpt[s].x, ckpt[s].v, ckpt[s].C, ckpt[s].F);
        for (int t = t0; t < t1 - 1 && !st; ++t) {
            state_t* a = &win[t - t0];
            state_t* b = &win[t - t0 + 1];
            st = oracle_step(c, N, a->x, a->v, a->C, a->F, aid, alpha + (int64_t)t * A, b->x,
                             b->v, b->C, b->F);
        }
        for (int t = t1 - 1; t >= t0 && !st; --t) {
            state_t* a = &win[t - t0];
            st = oracle_step_adj(c, N, a->x, a->v, a->C, a->F, aid, alpha + (int64_t)t * A, bar.x,
                                 bar.v, bar.C, bar.F, barn.x, barn.v, barn.C, barn.F,
                                 alpha_bar + (int64_t)t * A);
            state_t tmp = bar; bar = barn; barn = tmp;
            if (closed && !st) {  /* controller and observation adjoints into S_bar_t */
                oracle_controller_obs_adj(c, theta, t, obs + (int64_t)t * NO, alpha_bar + (int64_t)t * A,
                                          thb, obs_bar);
                oracle_observe_adj(c, N, aid, obs_bar, bar.x, bar.v);
            }
        }
    }
    if (!st) {
        if (dx0) memcpy(dx0, bar.x, sizeof(real) * N * d);
        if (dv0) memcpy(dv0, bar.v, sizeof(real) * N * d);
        if (dC0) memcpy(dC0, bar.C, sizeof(real) * N * dd);
        if (dF0) memcpy(dF0, bar.F, sizeof(real) * N * dd);
        if (dtheta && closed) memcpy(dtheta, thb, sizeof(real) * oracle_n_theta(c));
        if (dtheta && !closed) {
            int64_t nt = oracle_n_theta(c);
            memset(dtheta, 0, sizeof(real) * nt);
            if (c->n_act > 0)
                for (int t = T - 1; t >= 0; --t)
                    oracle_controller_adj(c, theta, t, alpha_bar + (int64_t)t * A, dtheta);
        }
    }

    for (int i = 0; i < k; ++i) state_free(&win[i]);
    free(win);
    for (int s = 0; s < nseg; ++s) state_free(&ckpt[s]);
    free(ckpt);
    state_free(&cur); state_free(&nxt); state_free(&bar); state_free(&barn);
    free(alpha); free(alpha_bar); free(obs); free(obs_bar); free(thb);
    return st;
}
