// kernels_step.cu -- the MLS-MPM step and its adjoint on sm_100a (v1: one thread per
// particle / per grid node, dense per-episode grids, vector red.global.add.v4.f32
// scatter).  Equations: DESIGN.md R1-R14; kernel order: PAPER.md Appendix D.1.
#include "kernels.h"

namespace mpm {

namespace {

constexpr int kThreads = 256;

template <int D>
__device__ __forceinline__ void load_rec(const float* __restrict__ src, float* r) {
    constexpr int R = Rec<D>::R;  // 12 or 24 floats: 3 or 6 x 16 B, 16-B aligned
    const float4* s4 = reinterpret_cast<const float4*>(src);
#pragma unroll
    for (int q = 0; q < R / 4; ++q) {
        float4 t = __ldg(s4 + q);
        r[4 * q + 0] = t.x; r[4 * q + 1] = t.y; r[4 * q + 2] = t.z; r[4 * q + 3] = t.w;
    }
}

template <int D> __device__ __forceinline__ void weights(const float* fx, float w[D][3], float dw[D][3]) {
#pragma unroll
    for (int k = 0; k < D; ++k) bspline(fx[k], w[k], dw[k]);
}

// ---------------------------------------------------------------- P2G
// Ft = (I + dt C) F;  tau = tau(Ft) + actuation;  A = -dt V 4/dx^2 tau + m C;
// P[b+o] += W_o (m v + A (o - f) dx),  M[b+o] += W_o m;  F_{t+1} = Ft.
template <int D>
__global__ void __launch_bounds__(kThreads) k_p2g(KParams p, const float* __restrict__ S,
                                                  const int32_t* __restrict__ aid,
                                                  const float* __restrict__ alpha,
                                                  float4* __restrict__ grid,
                                                  float* __restrict__ Snext, int* flags) {
    using RC = Rec<D>;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= p.N * p.E) return;
    const int64_t e = i / p.N;
    float r[RC::R];
    load_rec<D>(S + i * RC::R, r);
    int base[D];
    float fx[D], w[D][3], dw[D][3];
    if (!stencil<D>(r + RC::X, p, base, fx)) {
        atomicOr(flags, FLAG_OUT_OF_DOMAIN);
        return;
    }
    weights<D>(fx, w, dw);
    const float* C = r + RC::C;
    const float* F = r + RC::F;
    float Ft[D * D];
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
        for (int b = 0; b < D; ++b) {
            float s = 0.0f;
#pragma unroll
            for (int k = 0; k < D; ++k) s = fmaf(C[a * D + k], F[k * D + b], s);
            Ft[a * D + b] = fmaf(p.dt, s, F[a * D + b]);
        }
    const int a_id = aid ? aid[i] : -1;
    const float act = a_id >= 0 ? alpha[a_id] : 0.0f;
    float tau[D * D];
    if (!kirchhoff<D>(p, Ft, act, tau)) atomicOr(flags, FLAG_NONFINITE);
    float A[D * D];
#pragma unroll
    for (int q = 0; q < D * D; ++q) A[q] = fmaf(p.stress_scale, tau[q], p.p_mass * C[q]);
    if (Snext) {
        float* dst = Snext + i * RC::R + RC::F;
#pragma unroll
        for (int q = 0; q < D * D; ++q) dst[q] = Ft[q];
    }
    float4* g = grid + e * p.nodes;
    const float* v = r + RC::V;
#pragma unroll
    for (int o0 = 0; o0 < 3; ++o0)
#pragma unroll
        for (int o1 = 0; o1 < 3; ++o1)
#pragma unroll
            for (int o2 = 0; o2 < (D == 3 ? 3 : 1); ++o2) {
                const int o[3] = {o0, o1, o2};
                float W = w[0][o0] * w[1][o1];
                if (D == 3) W *= w[2][o2];
                float dpos[D];
#pragma unroll
                for (int k = 0; k < D; ++k) dpos[k] = ((float)o[k] - fx[k]) * p.dx;
                float mom[3] = {0.0f, 0.0f, 0.0f};
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    float s = p.p_mass * v[a];
#pragma unroll
                    for (int b = 0; b < D; ++b) s = fmaf(A[a * D + b], dpos[b], s);
                    mom[a] = W * s;
                }
                atomicAdd(g + node_of<D>(p, base, o0, o1, o2),
                          make_float4(mom[0], mom[1], mom[2], W * p.p_mass));
            }
}

// ------------------------------------------------------------- grid_op
// u0 = P/(M + eps); u1 = u0 - dt g e_y; z = sticky-wall select (R6); U = z ? 0 : u1.
// U.w carries z for grid_op_grad.
template <int D>
__global__ void __launch_bounds__(kThreads) k_grid_op(KParams p, const float4* __restrict__ grid,
                                                      float4* __restrict__ U) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= p.nodes * p.E) return;
    int64_t lin = i % p.nodes;
    int c[3] = {0, 0, 0};
#pragma unroll
    for (int k = D - 1; k >= 0; --k) {
        c[k] = (int)(lin % p.n_grid);
        lin /= p.n_grid;
    }
    const float4 g = grid[i];
    const float denom = g.w + p.eps_mass;
    float u[3] = {g.x / denom, g.y / denom, g.z / denom};
    u[1] -= p.dt * p.gravity;
    bool z = false;
#pragma unroll
    for (int k = 0; k < D; ++k) {
        z = z || (c[k] < p.bound && u[k] < 0.0f);
        z = z || (c[k] > p.n_grid - p.bound && u[k] > 0.0f);
    }
    U[i] = z ? make_float4(0.0f, 0.0f, 0.0f, 1.0f)
             : make_float4(u[0], u[1], D == 3 ? u[2] : 0.0f, 0.0f);
}

// ----------------------------------------------------------------- G2P
// v' = sum W U;  C' = 4/dx sum W U (o - f)^T;  x' = x + dt v'.
template <int D>
__global__ void __launch_bounds__(kThreads) k_g2p(KParams p, const float* __restrict__ S,
                                                  const float4* __restrict__ U,
                                                  float* __restrict__ Snext, int* flags) {
    using RC = Rec<D>;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= p.N * p.E) return;
    const int64_t e = i / p.N;
    float x[D];
#pragma unroll
    for (int k = 0; k < D; ++k) x[k] = __ldg(S + i * RC::R + RC::X + k);
    int base[D];
    float fx[D], w[D][3], dw[D][3];
    if (!stencil<D>(x, p, base, fx)) {
        atomicOr(flags, FLAG_OUT_OF_DOMAIN);
        return;
    }
    weights<D>(fx, w, dw);
    const float4* Ue = U + e * p.nodes;
    float nv[D], nC[D * D];
#pragma unroll
    for (int q = 0; q < D; ++q) nv[q] = 0.0f;
#pragma unroll
    for (int q = 0; q < D * D; ++q) nC[q] = 0.0f;
    const float c4 = 4.0f * p.inv_dx;
#pragma unroll
    for (int o0 = 0; o0 < 3; ++o0)
#pragma unroll
        for (int o1 = 0; o1 < 3; ++o1)
#pragma unroll
            for (int o2 = 0; o2 < (D == 3 ? 3 : 1); ++o2) {
                const int o[3] = {o0, o1, o2};
                float W = w[0][o0] * w[1][o1];
                if (D == 3) W *= w[2][o2];
                const float4 u4 = __ldg(Ue + node_of<D>(p, base, o0, o1, o2));
                const float u[3] = {u4.x, u4.y, u4.z};
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    nv[a] = fmaf(W, u[a], nv[a]);
                    float cw = c4 * W * u[a];
#pragma unroll
                    for (int b = 0; b < D; ++b) nC[a * D + b] = fmaf(cw, (float)o[b] - fx[b], nC[a * D + b]);
                }
            }
    float* dst = Snext + i * RC::R;
    bool fin = true;
#pragma unroll
    for (int a = 0; a < D; ++a) {
        dst[RC::X + a] = fmaf(p.dt, nv[a], x[a]);
        dst[RC::V + a] = nv[a];
        fin = fin && isfinite(nv[a]);
    }
#pragma unroll
    for (int q = 0; q < D * D; ++q) dst[RC::C + q] = nC[q];
    if (!fin) atomicOr(flags, FLAG_NONFINITE);
}

// ------------------------------------------------------------ g2p_grad
// vh = vb' + dt xb';  Ub[b+o] += W (vh + 4/dx Cb' (o - f));
// Wb = U.vh + 4/dx U^T Cb' (o - f);  fb += Wb dW/df - 4/dx W Cb'^T U;
// xb_t (partial) = xb' + fb/dx  -> Sb's x slot.
template <int D>
__global__ void __launch_bounds__(kThreads) k_g2p_grad(KParams p, const float* __restrict__ S,
                                                       const float4* __restrict__ U,
                                                       const float* __restrict__ Sbn,
                                                       float4* __restrict__ Ubar,
                                                       float* __restrict__ Sb) {
    using RC = Rec<D>;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= p.N * p.E) return;
    const int64_t e = i / p.N;
    float x[D];
#pragma unroll
    for (int k = 0; k < D; ++k) x[k] = __ldg(S + i * RC::R + RC::X + k);
    int base[D];
    float fx[D], w[D][3], dw[D][3];
    if (!stencil<D>(x, p, base, fx)) return;  // flagged by the forward
    weights<D>(fx, w, dw);
    const float* bn = Sbn + i * RC::R;
    float vh[D], Cb[D * D], fb[D];
#pragma unroll
    for (int a = 0; a < D; ++a) {
        vh[a] = fmaf(p.dt, __ldg(bn + RC::X + a), __ldg(bn + RC::V + a));
        fb[a] = 0.0f;
    }
#pragma unroll
    for (int q = 0; q < D * D; ++q) Cb[q] = __ldg(bn + RC::C + q);
    const float c4 = 4.0f * p.inv_dx;
    const float4* Ue = U + e * p.nodes;
    float4* Ube = Ubar + e * p.nodes;
#pragma unroll
    for (int o0 = 0; o0 < 3; ++o0)
#pragma unroll
        for (int o1 = 0; o1 < 3; ++o1)
#pragma unroll
            for (int o2 = 0; o2 < (D == 3 ? 3 : 1); ++o2) {
                const int o[3] = {o0, o1, o2};
                float wo[D];
#pragma unroll
                for (int k = 0; k < D; ++k) wo[k] = w[k][o[k]];
                float W = wo[0] * wo[1];
                if (D == 3) W *= wo[2];
                float gW[D];
#pragma unroll
                for (int k = 0; k < D; ++k) {
                    float s = dw[k][o[k]];
#pragma unroll
                    for (int j = 0; j < D; ++j)
                        if (j != k) s *= wo[j];
                    gW[k] = s;
                }
                const int64_t node = node_of<D>(p, base, o0, o1, o2);
                const float4 u4 = __ldg(Ue + node);
                const float u[3] = {u4.x, u4.y, u4.z};
                float om[D];
#pragma unroll
                for (int k = 0; k < D; ++k) om[k] = (float)o[k] - fx[k];
                float ub[3] = {0.0f, 0.0f, 0.0f};
                float Wb = 0.0f;
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    float s = 0.0f;
#pragma unroll
                    for (int b = 0; b < D; ++b) s = fmaf(Cb[a * D + b], om[b], s);
                    float t = fmaf(c4, s, vh[a]);
                    ub[a] = W * t;
                    Wb = fmaf(u[a], t, Wb);
                }
                atomicAdd(Ube + node, make_float4(ub[0], ub[1], ub[2], 0.0f));
#pragma unroll
                for (int k = 0; k < D; ++k) {
                    float s = 0.0f;
#pragma unroll
                    for (int a = 0; a < D; ++a) s = fmaf(Cb[a * D + k], u[a], s);
                    fb[k] = fmaf(Wb, gW[k], fb[k]) - c4 * W * s;
                }
            }
#pragma unroll
    for (int k = 0; k < D; ++k) Sb[i * RC::R + RC::X + k] = fmaf(p.inv_dx, fb[k], __ldg(bn + RC::X + k));
}

// -------------------------------------------------------- grid_op_grad
// select rule: ub = z ? 0 : Ub;  Pb = ub/(M + eps);  Mb = -(ub . u0)/(M + eps)
template <int D>
__global__ void __launch_bounds__(kThreads) k_grid_op_grad(KParams p, const float4* __restrict__ grid,
                                                           const float4* __restrict__ U,
                                                           const float4* __restrict__ Ubar,
                                                           float4* __restrict__ gbar) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= p.nodes * p.E) return;
    const float4 g = grid[i];
    const bool z = U[i].w != 0.0f;
    const float4 ub = Ubar[i];
    const float denom = g.w + p.eps_mass;
    float4 out;
    if (z) {
        out = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    } else {
        const float u0[3] = {g.x / denom, g.y / denom, g.z / denom};
        const float dot = ub.x * u0[0] + ub.y * u0[1] + (D == 3 ? ub.z * u0[2] : 0.0f);
        out = make_float4(ub.x / denom, ub.y / denom, D == 3 ? ub.z / denom : 0.0f, -dot / denom);
    }
    gbar[i] = out;
}

// ------------------------------------------------------------ p2g_grad
// Recompute Ft, tau, A; gather (Pb, Mb):  vb = sum W m Pb;  Ab = sum W Pb dpos^T;
// Wb = Pb.(m v + A dpos) + Mb m;  fb += Wb dW/df - dx W A^T Pb;  Cb = m Ab;
// taub = -dt V 4/dx^2 Ab;  Ftb = Fb' + tau/actuation adjoints;  Fb = (I + dt C)^T Ftb;
// Cb += dt Ftb F^T;  xb += fb/dx;  alpha_bar[aid] += kappa q^T taub q.
template <int D>
__global__ void __launch_bounds__(kThreads) k_p2g_grad(KParams p, const float* __restrict__ S,
                                                       const int32_t* __restrict__ aid,
                                                       const float* __restrict__ alpha,
                                                       const float4* __restrict__ gbar,
                                                       const float* __restrict__ Sbn,
                                                       float* __restrict__ Sb,
                                                       float* __restrict__ abar_part, int* flags) {
    using RC = Rec<D>;
    __shared__ float s_ab[kThreads / 32][32];
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool valid = i < p.N * p.E;
    int a_id = -1;
    float abar = 0.0f;
    if (valid) {
        const int64_t e = i / p.N;
        float r[RC::R];
        load_rec<D>(S + i * RC::R, r);
        int base[D];
        float fx[D], w[D][3], dw[D][3];
        if (stencil<D>(r + RC::X, p, base, fx)) {
            weights<D>(fx, w, dw);
            const float* C = r + RC::C;
            const float* F = r + RC::F;
            const float* v = r + RC::V;
            float Ft[D * D];
#pragma unroll
            for (int a = 0; a < D; ++a)
#pragma unroll
                for (int b = 0; b < D; ++b) {
                    float s = 0.0f;
#pragma unroll
                    for (int k = 0; k < D; ++k) s = fmaf(C[a * D + k], F[k * D + b], s);
                    Ft[a * D + b] = fmaf(p.dt, s, F[a * D + b]);
                }
            a_id = aid ? aid[i] : -1;
            const float act = a_id >= 0 ? alpha[a_id] : 0.0f;
            float tau[D * D], A[D * D];
            kirchhoff<D>(p, Ft, act, tau);
#pragma unroll
            for (int q = 0; q < D * D; ++q) A[q] = fmaf(p.stress_scale, tau[q], p.p_mass * C[q]);

            float vb[D], Ab[D * D], fb[D];
#pragma unroll
            for (int q = 0; q < D; ++q) { vb[q] = 0.0f; fb[q] = 0.0f; }
#pragma unroll
            for (int q = 0; q < D * D; ++q) Ab[q] = 0.0f;
            const float4* ge = gbar + e * p.nodes;
#pragma unroll
            for (int o0 = 0; o0 < 3; ++o0)
#pragma unroll
                for (int o1 = 0; o1 < 3; ++o1)
#pragma unroll
                    for (int o2 = 0; o2 < (D == 3 ? 3 : 1); ++o2) {
                        const int o[3] = {o0, o1, o2};
                        float wo[D];
#pragma unroll
                        for (int k = 0; k < D; ++k) wo[k] = w[k][o[k]];
                        float W = wo[0] * wo[1];
                        if (D == 3) W *= wo[2];
                        float gW[D], dpos[D];
#pragma unroll
                        for (int k = 0; k < D; ++k) {
                            float s = dw[k][o[k]];
#pragma unroll
                            for (int j = 0; j < D; ++j)
                                if (j != k) s *= wo[j];
                            gW[k] = s;
                            dpos[k] = ((float)o[k] - fx[k]) * p.dx;
                        }
                        const float4 g4 = __ldg(ge + node_of<D>(p, base, o0, o1, o2));
                        const float gP[3] = {g4.x, g4.y, g4.z};
                        float Wb = g4.w * p.p_mass;
#pragma unroll
                        for (int a = 0; a < D; ++a) {
                            vb[a] = fmaf(W * p.p_mass, gP[a], vb[a]);
                            float mom = p.p_mass * v[a];
#pragma unroll
                            for (int b = 0; b < D; ++b) {
                                Ab[a * D + b] = fmaf(W * gP[a], dpos[b], Ab[a * D + b]);
                                mom = fmaf(A[a * D + b], dpos[b], mom);
                            }
                            Wb = fmaf(gP[a], mom, Wb);
                        }
#pragma unroll
                        for (int k = 0; k < D; ++k) {
                            float s = 0.0f;
#pragma unroll
                            for (int a = 0; a < D; ++a) s = fmaf(A[a * D + k], gP[a], s);
                            fb[k] = fmaf(Wb, gW[k], fb[k]) - p.dx * W * s;
                        }
                    }
            float taub[D * D], Ftb[D * D];
            const float* bn = Sbn + i * RC::R;
#pragma unroll
            for (int q = 0; q < D * D; ++q) {
                taub[q] = p.stress_scale * Ab[q];
                Ftb[q] = __ldg(bn + RC::F + q);
            }
            abar = kirchhoff_adj<D>(p, Ft, a_id >= 0, act, taub, Ftb);
            float* dst = Sb + i * RC::R;
            bool fin = true;
#pragma unroll
            for (int a = 0; a < D; ++a)
#pragma unroll
                for (int b = 0; b < D; ++b) {
                    // Fb = (I + dt C)^T Ftb ;  Cb = m Ab + dt Ftb F^T
                    float sF = Ftb[a * D + b], sC = 0.0f;
#pragma unroll
                    for (int k = 0; k < D; ++k) {
                        sF = fmaf(p.dt * C[k * D + a], Ftb[k * D + b], sF);
                        sC = fmaf(Ftb[a * D + k], F[b * D + k], sC);
                    }
                    dst[RC::F + a * D + b] = sF;
                    dst[RC::C + a * D + b] = fmaf(p.dt, sC, p.p_mass * Ab[a * D + b]);
                    fin = fin && isfinite(sF);
                }
#pragma unroll
            for (int a = 0; a < D; ++a) {
                dst[RC::X + a] = fmaf(p.inv_dx, fb[a], dst[RC::X + a]);
                dst[RC::V + a] = vb[a];
            }
            if (!fin) atomicOr(flags, FLAG_NONFINITE);
        }
    }
    // fixed-order block reduction of the actuation gradient per actuator
    if (p.n_act > 0) {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        for (int a0 = 0; a0 < p.n_act; a0 += 32) {
            // per actuator in this chunk: warp butterfly sum (fixed order)
            for (int a = a0; a < min(p.n_act, a0 + 32); ++a) {
                float v = (a_id == a) ? abar : 0.0f;
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
                if (lane == 0) s_ab[warp][a - a0] = v;
            }
            __syncthreads();
            if (threadIdx.x < 32 && a0 + threadIdx.x < p.n_act) {
                float s = 0.0f;
                for (int wv = 0; wv < kThreads / 32; ++wv) s += s_ab[wv][threadIdx.x];
                abar_part[(int64_t)blockIdx.x * p.n_act + a0 + threadIdx.x] = s;
            }
            __syncthreads();
        }
    }
}

__global__ void k_reduce_abar(const float* __restrict__ part, int nblocks, int n_act,
                              float* __restrict__ out) {
    // one warp per actuator; lanes stride over blocks; fixed-order butterfly
    const int a = blockIdx.x;
    float s = 0.0f;
    for (int b = threadIdx.x; b < nblocks; b += 32) s += part[(int64_t)b * n_act + a];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (threadIdx.x == 0) out[a] = s;
}

inline unsigned nblk(int64_t n) { return (unsigned)((n + kThreads - 1) / kThreads); }

}  // namespace

#define DISPATCH(D, ...) \
    do {                 \
        if ((D) == 2) {  \
            constexpr int DIM = 2; __VA_ARGS__; \
        } else {         \
            constexpr int DIM = 3; __VA_ARGS__; \
        }                \
    } while (0)

void launch_p2g(const KParams& p, const float* S, const int32_t* aid, const float* alpha_t,
                float4* grid, float* S_next, int* flags, cudaStream_t s) {
    DISPATCH(p.dim, k_p2g<DIM><<<nblk(p.N * p.E), kThreads, 0, s>>>(p, S, aid, alpha_t, grid, S_next, flags));
}
void launch_grid_op(const KParams& p, const float4* grid, float4* U, cudaStream_t s) {
    DISPATCH(p.dim, k_grid_op<DIM><<<nblk(p.nodes * p.E), kThreads, 0, s>>>(p, grid, U));
}
void launch_g2p(const KParams& p, const float* S, const float4* U, float* S_next, int* flags,
                cudaStream_t s) {
    DISPATCH(p.dim, k_g2p<DIM><<<nblk(p.N * p.E), kThreads, 0, s>>>(p, S, U, S_next, flags));
}
void launch_g2p_grad(const KParams& p, const float* S, const float4* U, const float* Sb_next,
                     float4* Ubar, float* Sb, cudaStream_t s) {
    DISPATCH(p.dim, k_g2p_grad<DIM><<<nblk(p.N * p.E), kThreads, 0, s>>>(p, S, U, Sb_next, Ubar, Sb));
}
void launch_grid_op_grad(const KParams& p, const float4* grid, const float4* U, const float4* Ubar,
                         float4* gbar, cudaStream_t s) {
    DISPATCH(p.dim, k_grid_op_grad<DIM><<<nblk(p.nodes * p.E), kThreads, 0, s>>>(p, grid, U, Ubar, gbar));
}
int p2g_grad_blocks(const KParams& p) { return (int)nblk(p.N * p.E); }
void launch_p2g_grad(const KParams& p, const float* S, const int32_t* aid, const float* alpha_t,
                     const float4* gbar, const float* Sb_next, float* Sb, float* abar_part,
                     int* flags, cudaStream_t s) {
    DISPATCH(p.dim, k_p2g_grad<DIM><<<nblk(p.N * p.E), kThreads, 0, s>>>(p, S, aid, alpha_t, gbar, Sb_next, Sb, abar_part, flags));
}
void launch_reduce_abar(const KParams& p, const float* abar_part, int nblocks, float* alpha_bar_t,
                        cudaStream_t s) {
    if (p.n_act > 0) k_reduce_abar<<<p.n_act, 32, 0, s>>>(abar_part, nblocks, p.n_act, alpha_bar_t);
}

}  // namespace mpm
