// mpm_device.cuh -- per-particle MLS-MPM math in registers (sm_100a).
//
// Independent re-implementation of the readings in DESIGN.md (R1-R14); shares
// no code with oracle/.  Everything is fp32, unrolled over the compile-time
// dimension D, and kept in registers (north_star (2): fused SVD-free stress).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace mpm {

// Kernel-side constants (one copy per launch, passed by value).
struct KParams {
    int32_t dim, n_grid, bound, model, n_act, act_axis, n_sin, hidden;
    float dt, dx, inv_dx, mu, lam, p_mass, p_vol, gravity, eps_mass, kappa, omega;
    float stress_scale;  // -dt * V * 4 / dx^2   (the APIC/MLS stress factor)
    int64_t N;           // particles per episode
    int64_t nodes;       // grid nodes per episode (n_grid^dim)
    int32_t E;           // episodes
    int32_t nb;          // blocks per axis (ceil(n_grid / B))
    int32_t nbe;         // blocks per episode (nb^dim)
    int32_t TB;          // blocks, all episodes (E * nbe)
    int32_t max_active;  // capacity (blocks) of the grid-store pool shared by all steps
    int32_t step_blocks; // capacity of one step's block-local buffers (U_bar tiles, partials)
    int64_t EN;          // particles, all episodes (N * E): component stride of the state arrays
    int32_t closed_loop; // closed-loop controller (R22): alpha_t per episode from the observation
    int32_t n_in;        // controller inputs: n_sin (+ 2 d n_act closed loop)
    int32_t a_estride;   // episode stride of alpha_t / alpha_bar_t (n_act closed loop, else 0)
    float obs_sx, obs_sv;  // observation scales (R22)
    const int32_t* mat;  // per-particle material by particle id (R23: nonzero = fluid), or null
    int64_t n_body;      // particles of one whole body (episode): N, or the total over the
                         // subdomains of a decomposed body (f3; N is then a subdomain's capacity)
    int32_t x_lo, x_hi;  // owned block x-index range (f3 subdomain); single domain: [0, nb)
    float inv_nb, inv_nbe;  // 1/nb, 1/nbe for divq (0 when block ids reach 2^22: exact division)
};

// floor(n / d) for 0 <= n < 2^22 by a float reciprocal (inv = fl(1/d)) and one correction step:
// |n * inv - n / d| < 2^22 * 2^-23 < 1/2 before the truncation, so q is off by at most one.
// inv == 0 falls back to the integer division.
__device__ __forceinline__ int divq(int n, int d, float inv) {
    if (inv == 0.0f) return n / d;
    int q = __float2int_rz(__int2float_rn(n) * inv);
    const int r = n - q * d;
    q += (r >= d) - (r < 0);
    return q;
}

enum : int { FLAG_OUT_OF_DOMAIN = 1, FLAG_NONFINITE = 2, FLAG_BLOCK_OVERFLOW = 4, FLAG_ACTIVE_OVERFLOW = 8,
             FLAG_BAD_ACTUATOR = 16,
             FLAG_MIGRATION = 32 };  // f3: a particle jumped past a neighbour slab, or a capacity overflowed

// Block geometry of the sorted-tile scheme: particles
// are binned by the B^d block of cells containing their base cell; a block's
// particles scatter into a (B+2)^d node tile.
template <int D> struct Geo {
    static constexpr int B = D == 3 ? 4 : 8;        // cells per block edge
    static constexpr int LOGB = D == 3 ? 2 : 3;
    static constexpr int CELLS = 64;                 // B^d
    static constexpr int TE = B + 2;                 // tile edge in nodes
    static constexpr int TN = D == 3 ? 216 : 100;    // tile nodes
    static constexpr int NST = D == 3 ? 27 : 9;      // stencil offsets
    static constexpr int MAXP = 1728;                // particles per block (27 per cell)
};
// particles per launch up to which a step is latency bound rather than throughput bound (C1-C4
// episodes): such launches use programmatic dependent launch, the sub-block work split and the
// canonical ordering inside p2g (kernels_tile.cu)
#ifndef MPM_SMALL_PROBLEM
#define MPM_SMALL_PROBLEM 262144
#endif
constexpr int64_t kSmallProblem = MPM_SMALL_PROBLEM;
// at most this many CTAs share one block's particles in the thread-per-particle kernels
// (kernels_tile.cu item_split); sizes the per-item actuator-gradient partials
constexpr int kMaxSplit = 4;

// State layout: three arrays per state (x; v and C; F), each
// AoSoA with 32-particle tiles -- component k of particle i at
// ptr[((i / 32) * NC + k) * 32 + i % 32] for an array of NC components -- so a warp's access
// to one component of 32 consecutive particles is one contiguous 128-B segment (as
// component-major SoA), a kernel that needs only x reads 4d bytes per particle, and all
// components of a particle sit at compile-time offsets (k * 128 B) from one address: one
// address computation per particle and array instead of one 64-bit add per component.
// Capacities are rounded up to whole tiles (kTile particles).  (A float4-quad variant --
// NQ = ceil(NC/4) 16-B accesses per particle, pads included -- halved the load instructions
// but measured slower: C5 2.91e9 -> 2.80e9, g2p 134 -> 157 ms per iteration.)
constexpr int kTile = 32;
template <int D> struct Lay {
    static constexpr int X = D;           // x        d components
    static constexpr int VC = D + D * D;  // (v, C)   d + d^2 (v first, C row-major)
    static constexpr int FF = D * D;      // F        d^2, row-major
};
// element (component k, particle i) of an AoSoA-32 array with NC components
template <int NC> __device__ __forceinline__ int64_t soa(int k, int64_t i) {
    return (int64_t)(uint32_t)(i >> 5) * (NC * kTile) + k * kTile + (int)(i & (kTile - 1));
}
// all NC components of particle i (read-only path) / stores
template <int NC> __device__ __forceinline__ void load_comps(const float* __restrict__ base, int64_t i, float* v) {
    const float* b = base + soa<NC>(0, i);
#pragma unroll
    for (int k = 0; k < NC; ++k) v[k] = __ldg(b + k * kTile);
}
template <int NC> __device__ __forceinline__ void store_comps(float* __restrict__ base, int64_t i, const float* v) {
    float* b = base + soa<NC>(0, i);
#pragma unroll
    for (int k = 0; k < NC; ++k) b[k * kTile] = v[k];
}

// Programmatic dependent launch (sm_90+): every kernel is launched with programmatic stream
// serialization allowed (launch_k in kernels.h), waits for its predecessor grid's results as
// its first action and immediately lets its own dependent grid be scheduled, so the next
// kernel's launch and CTA rasterisation overlap this kernel's tail instead of following it.
__device__ __forceinline__ void pdl_begin() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// quadratic B-spline N_0..N_2 at f in [1/2, 3/2) and derivatives (R1)
__device__ __forceinline__ void bspline(float f, float w[3], float dw[3]) {
    float a = 1.5f - f, b = f - 1.0f, c = f - 0.5f;
    w[0] = 0.5f * a * a;
    w[1] = 0.75f - b * b;
    w[2] = 0.5f * c * c;
    dw[0] = -a;
    dw[1] = -2.0f * b;
    dw[2] = c;
}

// base = floor(x/dx - 1/2), f = x/dx - base (R12); false if the 3^d stencil
// leaves [0, n_grid - 1]^d (R13) or x is not finite.
template <int D>
__device__ __forceinline__ bool stencil(const float* x, const KParams& p, int base[D], float fx[D]) {
    bool ok = true;
#pragma unroll
    for (int k = 0; k < D; ++k) {
        float xi = x[k] * p.inv_dx;
        float b = floorf(xi - 0.5f);
        ok = ok && (b >= 0.0f) && (b + 2.0f <= (float)(p.n_grid - 1));  // false for NaN
        base[k] = ok ? (int)b : 0;
        fx[k] = xi - b;
    }
    return ok;
}

template <int D>
__device__ __forceinline__ int64_t node_of(const KParams& p, const int base[D], int o0, int o1, int o2) {
    int64_t n = p.n_grid;
    if (D == 2) return (int64_t)(base[0] + o0) * n + (base[1] + o1);
    return ((int64_t)(base[0] + o0) * n + (base[1] + o1)) * n + (base[2] + o2);
}

template <int D> __device__ __forceinline__ float det(const float* F) {
    if (D == 2) return F[0] * F[3] - F[1] * F[2];
    return F[0] * (F[4] * F[8] - F[5] * F[7]) - F[1] * (F[3] * F[8] - F[5] * F[6]) +
           F[2] * (F[3] * F[7] - F[4] * F[6]);
}

// K = det(F) F^{-T} (the cofactor matrix)
template <int D> __device__ __forceinline__ void cof(const float* F, float* K) {
    if (D == 2) {
        K[0] = F[3]; K[1] = -F[2]; K[2] = -F[1]; K[3] = F[0];
    } else {
        K[0] = F[4] * F[8] - F[5] * F[7];
        K[1] = F[5] * F[6] - F[3] * F[8];
        K[2] = F[3] * F[7] - F[4] * F[6];
        K[3] = F[2] * F[7] - F[1] * F[8];
        K[4] = F[0] * F[8] - F[2] * F[6];
        K[5] = F[1] * F[6] - F[0] * F[7];
        K[6] = F[1] * F[5] - F[2] * F[4];
        K[7] = F[2] * F[3] - F[0] * F[5];
        K[8] = F[0] * F[4] - F[1] * F[3];
    }
}

// element (i, e) of a row-major d x d matrix for a runtime column e, without
// dynamic register indexing (which would spill the matrix to local memory)
template <int D> __device__ __forceinline__ float column(const float* M, int i, int e) {
    float v = M[i * D];
#pragma unroll
    for (int k = 1; k < D; ++k) v = e == k ? M[i * D + k] : v;
    return v;
}

// F_{t+1} = (I + dt C) F (shared by p2g and the re-forward so both produce the same bits)
template <int D> __device__ __forceinline__ void deform_update(float dt, const float* C, const float* F, float* Ft) {
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
        for (int b = 0; b < D; ++b) {
            float s = 0.0f;
#pragma unroll
            for (int k = 0; k < D; ++k) s = fmaf(C[a * D + k], F[k * D + b], s);
            Ft[a * D + b] = fmaf(dt, s, F[a * D + b]);
        }
}

// Kirchhoff stress tau(Ft) of the material (R2) plus actuation (R8).
// NH : tau = mu (F F^T - I) + lambda ln J I
// FCR: tau = 2 mu (F - R) F^T + lambda (J - 1) J I   (2D closed-form polar R)
// returns false on a degenerate deformation (R14).
// fluid (R23): the volumetric term only (mu = 0)
template <int D>
__device__ __forceinline__ bool kirchhoff(const KParams& p, const float* Fm, float act, float* tau,
                                          bool fluid = false) {
    const float mu = fluid ? 0.0f : p.mu;
    float J = det<D>(Fm);
    bool ok = true;
    if (D == 3 || p.model == 0) {
        ok = J > 0.0f;
        float iso = p.lam * logf(fmaxf(J, 1e-30f)) - mu;
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = 0; j < D; ++j) {
                float s = 0.0f;
#pragma unroll
                for (int k = 0; k < D; ++k) s = fmaf(Fm[i * D + k], Fm[j * D + k], s);
                tau[i * D + j] = mu * s + (i == j ? iso : 0.0f);
            }
    } else {
        float a = Fm[0] + Fm[3], b = Fm[2] - Fm[1];
        float r2 = a * a + b * b;
        ok = r2 > 0.0f;
        float ir = rsqrtf(fmaxf(r2, 1e-30f));
        float cs = a * ir, sn = b * ir;
        float M0 = Fm[0] - cs, M1 = Fm[1] + sn, M2 = Fm[2] - sn, M3 = Fm[3] - cs;  // F - R
        float iso = p.lam * (J - 1.0f) * J;
        tau[0] = 2.0f * mu * (M0 * Fm[0] + M1 * Fm[1]) + iso;
        tau[1] = 2.0f * mu * (M0 * Fm[2] + M1 * Fm[3]);
        tau[2] = 2.0f * mu * (M2 * Fm[0] + M3 * Fm[1]);
        tau[3] = 2.0f * mu * (M2 * Fm[2] + M3 * Fm[3]) + iso;
    }
    if (act != 0.0f) {
        // q = F e (column act_axis); selects keep F in registers (no dynamic indexing)
        float q[D];
#pragma unroll
        for (int i = 0; i < D; ++i) q[i] = column<D>(Fm, i, p.act_axis);
        float s = p.kappa * act;
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = 0; j < D; ++j) tau[i * D + j] = fmaf(s * q[i], q[j], tau[i * D + j]);
    }
    return ok;
}

// Reverse of kirchhoff(): Fb += d<tb, tau(F)>/dF, and the actuation adjoint
// (returns kappa q^T tb q, the contribution to alpha_bar).
template <int D>
__device__ __forceinline__ float kirchhoff_adj(const KParams& p, const float* Fm, bool has_act,
                                               float act, const float* tb, float* Fb, bool fluid = false) {
    const float mu = fluid ? 0.0f : p.mu;
    float S[D * D], K[D * D];
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) S[i * D + j] = tb[i * D + j] + tb[j * D + i];
    cof<D>(Fm, K);
    float J = det<D>(Fm);
    float tr = 0.0f;
#pragma unroll
    for (int i = 0; i < D; ++i) tr += tb[i * D + i];
    const bool nh = (D == 3 || p.model == 0);
    float musym = nh ? mu : 2.0f * mu;
    float kiso = nh ? p.lam * tr / J : p.lam * (2.0f * J - 1.0f) * tr;
    // (tb + tb^T) F term and the isotropic term
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
            float s = 0.0f;
#pragma unroll
            for (int k = 0; k < D; ++k) s = fmaf(S[i * D + k], Fm[k * D + j], s);
            Fb[i * D + j] += musym * s + kiso * K[i * D + j];
        }
    if (!nh && D == 2) {
        float a = Fm[0] + Fm[3], b = Fm[2] - Fm[1];
        float r2 = a * a + b * b;
        float ir = rsqrtf(r2);
        float cs = a * ir, sn = b * ir;
        // -2 mu tb^T R
        float tR0 = tb[0] * cs + tb[2] * sn, tR1 = -tb[0] * sn + tb[2] * cs;
        float tR2 = tb[1] * cs + tb[3] * sn, tR3 = -tb[1] * sn + tb[3] * cs;
        Fb[0] -= 2.0f * mu * tR0; Fb[1] -= 2.0f * mu * tR1;
        Fb[2] -= 2.0f * mu * tR2; Fb[3] -= 2.0f * mu * tR3;
        // rotation path: Rb = -2 mu tb F; psi_b = <Rb, dR/dpsi>
        float Rb0 = -2.0f * mu * (tb[0] * Fm[0] + tb[1] * Fm[2]);
        float Rb1 = -2.0f * mu * (tb[0] * Fm[1] + tb[1] * Fm[3]);
        float Rb2 = -2.0f * mu * (tb[2] * Fm[0] + tb[3] * Fm[2]);
        float Rb3 = -2.0f * mu * (tb[2] * Fm[1] + tb[3] * Fm[3]);
        float psib = -sn * Rb0 - cs * Rb1 + cs * Rb2 - sn * Rb3;
        float ga = -psib * b / r2, gb = psib * a / r2;  // d psi/da = -b/r^2, d psi/db = a/r^2
        Fb[0] += ga; Fb[3] += ga; Fb[2] += gb; Fb[1] -= gb;
    }
    float abar = 0.0f;
    if (has_act) {
        const int e = p.act_axis;
        float q[D], sq[D];
#pragma unroll
        for (int i = 0; i < D; ++i) q[i] = column<D>(Fm, i, e);
#pragma unroll
        for (int i = 0; i < D; ++i) {
            float s = 0.0f;
#pragma unroll
            for (int j = 0; j < D; ++j) s = fmaf(S[i * D + j], q[j], s);
            sq[i] = s;
            abar = fmaf(q[i], s, abar);
        }
        abar *= 0.5f * p.kappa;  // q^T tb q = 1/2 q^T (tb + tb^T) q
        float s = p.kappa * act;
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int k = 0; k < D; ++k)
                if (k == e) Fb[i * D + k] = fmaf(s, sq[i], Fb[i * D + k]);
    }
    return abar;
}

// det with every rounding explicit (no FMA contraction left to the compiler): p2g and the
// re-forward g2p both evaluate the fluid reset, and their F_{t+1} must agree bit for bit
template <int D> __device__ __forceinline__ float det_rn(const float* F) {
    if (D == 2) return __fsub_rn(__fmul_rn(F[0], F[3]), __fmul_rn(F[1], F[2]));
    const float a = __fsub_rn(__fmul_rn(F[4], F[8]), __fmul_rn(F[5], F[7]));
    const float b = __fsub_rn(__fmul_rn(F[3], F[8]), __fmul_rn(F[5], F[6]));
    const float c = __fsub_rn(__fmul_rn(F[3], F[7]), __fmul_rn(F[4], F[6]));
    return __fadd_rn(__fsub_rn(__fmul_rn(F[0], a), __fmul_rn(F[1], b)), __fmul_rn(F[2], c));
}

// R23 fluid: F_{t+1} = J^(1/d) I with J = det(Ft) (shear forgotten)
template <int D> __device__ __forceinline__ void fluid_reset(const float* Ft, float* Fn) {
    const float J = det_rn<D>(Ft);
    const float s = D == 3 ? cbrtf(J) : sqrtf(J);
#pragma unroll
    for (int q = 0; q < D * D; ++q) Fn[q] = (q % (D + 1) == 0) ? s : 0.0f;
}
// its reverse: Ftb = d/dFt <Fb', J^(1/d) I> = (1/d) J^(1/d - 1) tr(Fb') cof(Ft)
template <int D> __device__ __forceinline__ void fluid_reset_adj(const float* Ft, const float* Fbn, float* Ftb) {
    const float J = det<D>(Ft);
    const float s = D == 3 ? cbrtf(J) : sqrtf(J);
    float tr = 0.0f;
#pragma unroll
    for (int i = 0; i < D; ++i) tr += Fbn[i * D + i];
    float K[D * D];
    cof<D>(Ft, K);
    const float g = s / J * tr / (float)D;
#pragma unroll
    for (int q = 0; q < D * D; ++q) Ftb[q] = g * K[q];
}

}  // namespace mpm
