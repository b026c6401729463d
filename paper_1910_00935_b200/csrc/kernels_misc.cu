// kernels_misc.cu -- controller (compute_actuation and its .grad), loss + adjoint
// seed, and caller-layout <-> particle-record conversion.
#include "kernels.h"

namespace mpm {

namespace {

constexpr int kMaxHidden = 1024;
constexpr int kMaxAct = 256;
constexpr int kMaxSin = 64;

// phi_j(t) = sin(omega t dt + 2 pi j / n_sin)   (R9; phase in fp64, it reaches ~40 rad)
__device__ __forceinline__ float feature(const KParams& p, int t, int j) {
    double ph = (double)p.omega * (double)t * (double)p.dt + 2.0 * 3.14159265358979323846 * j / p.n_sin;
    return (float)sin(ph);
}

// one block per time step: alpha_t = tanh(W2 tanh(W1 phi + b1) + b2)  (H > 0)
//                          alpha_t = tanh(W phi + b)                  (H = 0)
__global__ void k_ctrl_fwd(KParams p, const float* __restrict__ th, float* __restrict__ alpha) {
    pdl_begin();
    __shared__ float phi[kMaxSin], h[kMaxHidden];
    const int t = blockIdx.x, S = p.n_sin, H = p.hidden, A = p.n_act;
    for (int j = threadIdx.x; j < S; j += blockDim.x) phi[j] = feature(p, t, j);
    __syncthreads();
    if (H > 0) {
        const float *W1 = th, *b1 = W1 + H * S, *W2 = b1 + H, *b2 = W2 + A * H;
        for (int i = threadIdx.x; i < H; i += blockDim.x) {
            float z = b1[i];
            for (int j = 0; j < S; ++j) z = fmaf(W1[i * S + j], phi[j], z);
            h[i] = tanhf(z);
        }
        __syncthreads();
        for (int a = threadIdx.x; a < A; a += blockDim.x) {
            float z = b2[a];
            for (int i = 0; i < H; ++i) z = fmaf(W2[a * H + i], h[i], z);
            alpha[(int64_t)t * A + a] = tanhf(z);
        }
    } else {
        const float *W = th, *b = W + A * S;
        for (int a = threadIdx.x; a < A; a += blockDim.x) {
            float z = b[a];
            for (int j = 0; j < S; ++j) z = fmaf(W[a * S + j], phi[j], z);
            alpha[(int64_t)t * A + a] = tanhf(z);
        }
    }
}

// one block per time step: the step's contribution (d alpha_t/d theta)^T alpha_bar_t
__global__ void k_ctrl_bwd(KParams p, const float* __restrict__ th, const float* __restrict__ alpha,
                           const float* __restrict__ abar, float* __restrict__ part, int64_t n_theta) {
    pdl_begin();
    __shared__ float phi[kMaxSin], h[kMaxHidden], z2b[kMaxAct], hb[kMaxHidden];
    const int t = blockIdx.x, S = p.n_sin, H = p.hidden, A = p.n_act;
    float* out = part + (int64_t)t * n_theta;
    for (int j = threadIdx.x; j < S; j += blockDim.x) phi[j] = feature(p, t, j);
    for (int a = threadIdx.x; a < A; a += blockDim.x) {
        float al = alpha[(int64_t)t * A + a];
        z2b[a] = abar[(int64_t)t * A + a] * (1.0f - al * al);
    }
    __syncthreads();
    if (H > 0) {
        const float *W1 = th, *b1 = W1 + H * S, *W2 = b1 + H;
        float *W1b = out, *b1b = W1b + H * S, *W2b = b1b + H, *b2b = W2b + A * H;
        for (int i = threadIdx.x; i < H; i += blockDim.x) {
            float z = b1[i];
            for (int j = 0; j < S; ++j) z = fmaf(W1[i * S + j], phi[j], z);
            h[i] = tanhf(z);
        }
        __syncthreads();
        for (int q = threadIdx.x; q < A * H; q += blockDim.x) W2b[q] = z2b[q / H] * h[q % H];
        for (int a = threadIdx.x; a < A; a += blockDim.x) b2b[a] = z2b[a];
        for (int i = threadIdx.x; i < H; i += blockDim.x) {
            float s = 0.0f;
            for (int a = 0; a < A; ++a) s = fmaf(W2[a * H + i], z2b[a], s);
            hb[i] = s * (1.0f - h[i] * h[i]);
            b1b[i] = hb[i];
        }
        __syncthreads();
        for (int q = threadIdx.x; q < H * S; q += blockDim.x) W1b[q] = hb[q / S] * phi[q % S];
    } else {
        float *Wb = out, *bb = Wb + A * S;
        for (int q = threadIdx.x; q < A * S; q += blockDim.x) Wb[q] = z2b[q / S] * phi[q % S];
        for (int a = threadIdx.x; a < A; a += blockDim.x) bb[a] = z2b[a];
    }
}

// theta_bar[q] = sum over t (ascending, fixed order) of part[t][q]
__global__ void k_ctrl_reduce(const float* __restrict__ part, int T, int64_t n_theta,
                              float* __restrict__ thb) {
    pdl_begin();
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= n_theta) return;
    float s = 0.0f;
    for (int t = 0; t < T; ++t) s += part[(int64_t)t * n_theta + q];
    thb[q] = s;
}

// ---------------------------------------------------- closed-loop controller
// SURVEY 8(f) f1, R22.  o_t[e][a] = (s_x (mean_a x - mean x), s_v mean_a v) over the
// particles of episode e with actuator id a; input u = [phi(t), o_t[e]]; alpha_t[e] = MLP(u).
constexpr int kObsThreads = 256;
constexpr int kMaxIn = 1024;

__host__ __device__ inline int obs_nvals(int n_act, int dim) { return n_act * (2 * dim + 1) + dim; }

// CTA (c, e): particles [c * 256, (c + 1) * 256) of episode e (S_t keeps each episode's
// particles in one contiguous index range).  Per group a: sums of x, v and the count; plus
// the sum of x over all particles.  Masked warp butterflies + warp order: fixed summation order.
template <int D>
__global__ void __launch_bounds__(kObsThreads) k_observe(KParams p, const float* __restrict__ X,
                                                         const float* __restrict__ VC,
                                                         const int* __restrict__ pid,
                                                         const int32_t* __restrict__ aid,
                                                         float* __restrict__ part) {
    pdl_begin();
    constexpr int W = kObsThreads / 32;
    extern __shared__ float s_w[];  // [W][NV]
    const int A = p.n_act, NV = obs_nvals(A, D);
    const int c = blockIdx.x, e = blockIdx.y, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t r = (int64_t)c * kObsThreads + threadIdx.x;
    const bool in = r < p.N;
    const int64_t i = (int64_t)e * p.N + r;
    float x[D], v[D];
    int a_id = -1;
#pragma unroll
    for (int k = 0; k < D; ++k) {
        x[k] = in ? X[soa<Lay<D>::X>(k, i)] : 0.0f;
        v[k] = in ? VC[soa<Lay<D>::VC>(k, i)] : 0.0f;
    }
    if (in && aid) a_id = aid[pid[i]];
    float* w = s_w + warp * NV;
#pragma unroll
    for (int k = 0; k < D; ++k) {
        float t = x[k];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
        if (lane == 0) w[A * (2 * D + 1) + k] = t;
    }
    for (int a = 0; a < A; ++a) {
        const bool mine = a_id == a;
        float* wa = w + a * (2 * D + 1);
        if (__ballot_sync(0xffffffffu, mine) == 0u) {
            if (lane < 2 * D + 1) wa[lane] = 0.0f;
            continue;
        }
        float q[2 * D + 1];
#pragma unroll
        for (int k = 0; k < D; ++k) { q[k] = mine ? x[k] : 0.0f; q[D + k] = mine ? v[k] : 0.0f; }
        q[2 * D] = mine ? 1.0f : 0.0f;
#pragma unroll
        for (int k = 0; k < 2 * D + 1; ++k) {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) q[k] += __shfl_xor_sync(0xffffffffu, q[k], off);
        }
        if (lane == 0) {
#pragma unroll
            for (int k = 0; k < 2 * D + 1; ++k) wa[k] = q[k];
        }
    }
    __syncthreads();
    for (int q = threadIdx.x; q < NV; q += kObsThreads) {
        float t = 0.0f;
        for (int ww = 0; ww < W; ++ww) t += s_w[ww * NV + q];
        part[((int64_t)e * gridDim.x + c) * NV + q] = t;
    }
}

// one CTA per episode: reduce the partials (chunk order), form o_t[e], run the MLP
template <int D>
__global__ void k_ctrl_obs_fwd(KParams p, const float* __restrict__ th, int t, const float* __restrict__ part,
                               int nch, float* __restrict__ obs_t, float* __restrict__ counts,
                               float* __restrict__ alpha_t) {
    pdl_begin();
    __shared__ float tot[kMaxIn], u[kMaxIn], h[kMaxHidden];
    const int e = blockIdx.x, A = p.n_act, NV = obs_nvals(A, D), S = p.n_in, ns = p.n_sin, H = p.hidden;
    const int no = 2 * D * A;
    for (int q = threadIdx.x; q < NV; q += blockDim.x) {
        float s = 0.0f;
        for (int c = 0; c < nch; ++c) s += part[((int64_t)e * nch + c) * NV + q];
        tot[q] = s;
    }
    for (int j = threadIdx.x; j < ns; j += blockDim.x) u[j] = feature(p, t, j);
    __syncthreads();
    for (int q = threadIdx.x; q < no; q += blockDim.x) {
        const int a = q / (2 * D), k = q % (2 * D);
        const float n = tot[a * (2 * D + 1) + 2 * D];
        float o = 0.0f;
        if (n > 0.0f) {
            if (k < D) o = p.obs_sx * (tot[a * (2 * D + 1) + k] / n - tot[A * (2 * D + 1) + k] / (float)p.N);
            else o = p.obs_sv * (tot[a * (2 * D + 1) + k] / n);
        }
        u[ns + q] = o;
        obs_t[(int64_t)e * no + q] = o;
    }
    for (int a = threadIdx.x; a < A; a += blockDim.x) counts[e * A + a] = tot[a * (2 * D + 1) + 2 * D];
    __syncthreads();
    if (H > 0) {
        const float *W1 = th, *b1 = W1 + H * S, *W2 = b1 + H, *b2 = W2 + A * H;
        for (int i = threadIdx.x; i < H; i += blockDim.x) {
            float z = b1[i];
            for (int j = 0; j < S; ++j) z = fmaf(W1[i * S + j], u[j], z);
            h[i] = tanhf(z);
        }
        __syncthreads();
        for (int a = threadIdx.x; a < A; a += blockDim.x) {
            float z = b2[a];
            for (int i = 0; i < H; ++i) z = fmaf(W2[a * H + i], h[i], z);
            alpha_t[e * A + a] = tanhf(z);
        }
    } else {
        const float *Wm = th, *b = Wm + A * S;
        for (int a = threadIdx.x; a < A; a += blockDim.x) {
            float z = b[a];
            for (int j = 0; j < S; ++j) z = fmaf(Wm[a * S + j], u[j], z);
            alpha_t[e * A + a] = tanhf(z);
        }
    }
}

// one CTA, episodes in order (fixed accumulation order of theta_bar, no atomics):
// z2b = ab (1 - alpha^2); theta_bar += outer products; u_bar = W^T (.); the observation part
// of u_bar -> per-group increments inc[e] = [s_x ob_x[a] / n_a, s_v ob_v[a] / n_a]_a,
// [-s_x sum_a ob_x[a] / N]  (groups with n_a = 0 observe 0 and get no gradient)
template <int D>
__global__ void k_ctrl_obs_bwd(KParams p, const float* __restrict__ th, int t, const float* __restrict__ obs_t,
                               const float* __restrict__ alpha_t, const float* __restrict__ abar_t,
                               const float* __restrict__ counts, float* __restrict__ thb,
                               float* __restrict__ inc) {
    pdl_begin();
    __shared__ float u[kMaxIn], h[kMaxHidden], z2b[kMaxAct], hb[kMaxHidden], ub[kMaxIn];
    const int A = p.n_act, S = p.n_in, ns = p.n_sin, H = p.hidden, no = 2 * D * A;
    for (int e = 0; e < p.E; ++e) {
        for (int j = threadIdx.x; j < S; j += blockDim.x)
            u[j] = j < ns ? feature(p, t, j) : obs_t[(int64_t)e * no + (j - ns)];
        for (int a = threadIdx.x; a < A; a += blockDim.x) {
            const float al = alpha_t[e * A + a];
            z2b[a] = abar_t[e * A + a] * (1.0f - al * al);
        }
        __syncthreads();
        if (H > 0) {
            const float *W1 = th, *b1 = W1 + H * S, *W2 = b1 + H;
            float *W1b = thb, *b1b = W1b + H * S, *W2b = b1b + H, *b2b = W2b + A * H;
            for (int i = threadIdx.x; i < H; i += blockDim.x) {
                float z = b1[i];
                for (int j = 0; j < S; ++j) z = fmaf(W1[i * S + j], u[j], z);
                h[i] = tanhf(z);
            }
            __syncthreads();
            for (int q = threadIdx.x; q < A * H; q += blockDim.x) W2b[q] = fmaf(z2b[q / H], h[q % H], W2b[q]);
            for (int a = threadIdx.x; a < A; a += blockDim.x) b2b[a] += z2b[a];
            for (int i = threadIdx.x; i < H; i += blockDim.x) {
                float s = 0.0f;
                for (int a = 0; a < A; ++a) s = fmaf(W2[a * H + i], z2b[a], s);
                hb[i] = s * (1.0f - h[i] * h[i]);
                b1b[i] += hb[i];
            }
            __syncthreads();
            for (int q = threadIdx.x; q < H * S; q += blockDim.x) W1b[q] = fmaf(hb[q / S], u[q % S], W1b[q]);
            for (int j = ns + (int)threadIdx.x; j < S; j += blockDim.x) {
                float s = 0.0f;
                for (int i = 0; i < H; ++i) s = fmaf(W1[i * S + j], hb[i], s);
                ub[j] = s;
            }
        } else {
            const float* Wm = th;
            float *Wb = thb, *bb = Wb + A * S;
            for (int q = threadIdx.x; q < A * S; q += blockDim.x) Wb[q] = fmaf(z2b[q / S], u[q % S], Wb[q]);
            for (int a = threadIdx.x; a < A; a += blockDim.x) bb[a] += z2b[a];
            for (int j = ns + (int)threadIdx.x; j < S; j += blockDim.x) {
                float s = 0.0f;
                for (int a = 0; a < A; ++a) s = fmaf(Wm[a * S + j], z2b[a], s);
                ub[j] = s;
            }
        }
        __syncthreads();
        float* ie = inc + (int64_t)e * (no + D);
        for (int q = threadIdx.x; q < no; q += blockDim.x) {
            const int a = q / (2 * D), k = q % (2 * D);
            const float n = counts[e * A + a];
            ie[q] = n > 0.0f ? (k < D ? p.obs_sx : p.obs_sv) * ub[ns + q] / n : 0.0f;
        }
        for (int k = threadIdx.x; k < D; k += blockDim.x) {
            float s = 0.0f;
            for (int a = 0; a < A; ++a)
                if (counts[e * A + a] > 0.0f) s += ub[ns + a * 2 * D + k];
            ie[no + k] = -p.obs_sx * s / (float)p.N;
        }
        __syncthreads();
    }
}

// x_bar_i += inc_x[a(i)] + inc_all, v_bar_i += inc_v[a(i)]  (particle i of episode i / N)
template <int D>
__global__ void k_observe_adj(KParams p, AdjView Sb, const int* __restrict__ pid, const int32_t* __restrict__ aid,
                              const float* __restrict__ inc) {
    pdl_begin();
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= p.EN) return;
    const int e = (int)(i / p.N), no = 2 * D * p.n_act;
    const float* ie = inc + (int64_t)e * (no + D);
    int a = aid ? aid[pid[i]] : -1;
    if (a >= p.n_act) a = -1;  // out-of-range ids: flagged by mpm_set_state, no gradient here
#pragma unroll
    for (int k = 0; k < D; ++k) {
        const float gx = ie[no + k] + (a >= 0 ? ie[a * 2 * D + k] : 0.0f);
        Sb.x[soa<Lay<D>::X>(k, i)] += gx;
        if (a >= 0) Sb.vc[soa<Lay<D>::VC>(k, i)] += ie[a * 2 * D + D + k];
    }
}

// ---------------------------------------------------------------- loss
constexpr int kLossThreads = 256;

// partial sums of a d-vector field over a contiguous particle chunk (fixed tree order);
// component k of particle i = the first d components of an AoSoA state array of NC components
template <int D, int NC>
__global__ void k_sum_partial(KParams p, const float* __restrict__ base, float* __restrict__ part) {
    pdl_begin();
    __shared__ float red[D][kLossThreads];
    const int e = blockIdx.y, nb = gridDim.x;
    const int64_t chunk = (p.N + nb - 1) / nb;
    const int64_t lo = blockIdx.x * chunk, hi = min(p.N, lo + chunk);
    float acc[D];
#pragma unroll
    for (int k = 0; k < D; ++k) acc[k] = 0.0f;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
#pragma unroll
        for (int k = 0; k < D; ++k) acc[k] += base[soa<NC>(k, (int64_t)e * p.N + i)];
    }
#pragma unroll
    for (int k = 0; k < D; ++k) red[k][threadIdx.x] = acc[k];
    __syncthreads();
    for (int s = kLossThreads / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s)
#pragma unroll
            for (int k = 0; k < D; ++k) red[k][threadIdx.x] += red[k][threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0)
#pragma unroll
        for (int k = 0; k < D; ++k) part[((int64_t)e * nb + blockIdx.x) * D + k] = red[k][0];
}

template <int D>
__global__ void k_sum_parts(const float* __restrict__ part, int nb, float* __restrict__ out) {
    pdl_begin();
    const int e = blockIdx.x;
    if (threadIdx.x != 0) return;
#pragma unroll
    for (int k = 0; k < D; ++k) {
        float s = 0.0f;
        for (int b = 0; b < nb; ++b) s += part[((int64_t)e * nb + b) * D + k];
        out[e * D + k] = s;
    }
}

// xbar = sum m x / sum m;  L = |xbar - x*|^2 or -xbar_0;  seed g = dL/dxbar * m / M
template <int D>
__global__ void k_loss_final(KParams p, const float* __restrict__ part, int nb, int kind,
                             float3 target, float* __restrict__ loss, float* __restrict__ seed,
                             int* flags) {
    pdl_begin();
    const int e = blockIdx.x;
    if (threadIdx.x != 0) return;
    float com[D];
#pragma unroll
    for (int k = 0; k < D; ++k) {
        float s = 0.0f;
        for (int b = 0; b < nb; ++b) s += part[((int64_t)e * nb + b) * D + k];
        com[k] = s / (float)p.N;  // equal masses: sum m x / sum m = mean x
    }
    const float tg[3] = {target.x, target.y, target.z};
    float L = 0.0f, g[D];
#pragma unroll
    for (int k = 0; k < D; ++k) g[k] = 0.0f;
    if (kind == 0) {
#pragma unroll
        for (int k = 0; k < D; ++k) {
            float dlt = com[k] - tg[k];
            L = fmaf(dlt, dlt, L);
            g[k] = 2.0f * dlt;
        }
    } else {
        L = -com[0];
        g[0] = -1.0f;
    }
    loss[e] = L;
    if (!isfinite(L)) atomicOr(flags, FLAG_NONFINITE);
#pragma unroll
    for (int k = 0; k < D; ++k) seed[e * D + k] = g[k] / (float)p.N;  // dL/dxbar * m / (N m)
}

template <int D>
__global__ void k_seed(KParams p, const float* __restrict__ seed, AdjView Sb) {
    pdl_begin();
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= p.N * p.E) return;
    const int64_t e = i / p.N;
    float xs[3] = {0.f, 0.f, 0.f}, z[Lay<D>::VC] = {};
#pragma unroll
    for (int k = 0; k < D; ++k) xs[k] = seed[e * D + k];
    store_comps<Lay<D>::X>(Sb.x, i, xs);
    store_comps<Lay<D>::VC>(Sb.vc, i, z);
    store_comps<Lay<D>::FF>(Sb.f, i, z);
}

// ------------------------------------------------------------- layout
template <int D>
__global__ void k_pack(KParams p, const float* __restrict__ x, const float* __restrict__ v,
                       const float* __restrict__ C, const float* __restrict__ F,
                       const int* __restrict__ src, float* __restrict__ dx, float* __restrict__ dvc,
                       float* __restrict__ df, int* __restrict__ ident_pid, bool zero_f) {
    pdl_begin();
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= p.N * p.E) return;
    if (ident_pid) ident_pid[i] = (int)i;
    const int64_t s = src ? (int64_t)src[i] : i;
    float xo[3], vco[Lay<D>::VC], fo[D * D];
#pragma unroll
    for (int k = 0; k < D; ++k) {
        xo[k] = x ? x[s * D + k] : 0.0f;
        vco[k] = v ? v[s * D + k] : 0.0f;
    }
#pragma unroll
    for (int q = 0; q < D * D; ++q) {
        vco[D + q] = C ? C[s * D * D + q] : 0.0f;
        fo[q] = F ? F[s * D * D + q] : ((!zero_f && (q % (D + 1)) == 0) ? 1.0f : 0.0f);
    }
    store_comps<Lay<D>::X>(dx, i, xo);
    store_comps<Lay<D>::VC>(dvc, i, vco);
    store_comps<Lay<D>::FF>(df, i, fo);
}

template <int D>
__global__ void k_unpack(KParams p, const float* __restrict__ sx, const float* __restrict__ svc,
                         const float* __restrict__ sf, const int* __restrict__ dst,
                         float* __restrict__ x, float* __restrict__ v, float* __restrict__ C,
                         float* __restrict__ F, int64_t n_rows) {
    pdl_begin();
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n_rows) return;
    const int64_t o = dst ? (int64_t)dst[i] : i;
#pragma unroll
    for (int k = 0; k < D; ++k) {
        if (x) x[o * D + k] = sx[soa<Lay<D>::X>(k, i)];
        if (v) v[o * D + k] = svc[soa<Lay<D>::VC>(k, i)];
    }
#pragma unroll
    for (int q = 0; q < D * D; ++q) {
        if (C) C[o * D * D + q] = svc[soa<Lay<D>::VC>(D + q, i)];
        if (F) F[o * D * D + q] = sf[soa<Lay<D>::FF>(q, i)];
    }
}

// COM loss in fixed block order (kernels.h launch_loss_blocks): episode e = blockIdx.x, one warp.
// Global index g runs over the concatenated block lists (subdomains in slab order); lane g mod 32
// accumulates its entries in order, then a fixed butterfly -> xbar = sum / n_body; L; seed.
constexpr int kMaxListSrc = 4;
struct ListSrcs {
    ListSrc s[kMaxListSrc];
    int n;
};
template <int D>
__global__ void k_loss_blocks(KParams p, ListSrcs src, int kind, float3 target, float* __restrict__ loss,
                              float* __restrict__ seed, int* flags) {
    pdl_begin();
    const int e = blockIdx.x, lane = threadIdx.x;
    float acc[D];
#pragma unroll
    for (int k = 0; k < D; ++k) acc[k] = 0.0f;
    int off = 0;
    for (int q = 0; q < src.n; ++q) {
        const ListSrc& L = src.s[q];
        const int n = *L.n;
        const int* bl = L.blist + *L.base;
        for (int idx = ((lane - off) % 32 + 32) % 32; idx < n; idx += 32) {
            if (bl[idx] / p.nbe != e) continue;
#pragma unroll
            for (int k = 0; k < D; ++k) acc[k] += L.part[(int64_t)idx * D + k];
        }
        off += n;
    }
#pragma unroll
    for (int k = 0; k < D; ++k)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], o);
    if (lane != 0) return;
    const float tg[3] = {target.x, target.y, target.z};
    float L = 0.0f, g[D];
#pragma unroll
    for (int k = 0; k < D; ++k) {
        const float com = acc[k] / (float)p.n_body;  // equal masses: sum m x / sum m = mean x
        g[k] = 0.0f;
        if (kind == 0) {
            const float dlt = com - tg[k];
            L = fmaf(dlt, dlt, L);
            g[k] = 2.0f * dlt;
        } else if (k == 0) {
            L = -com;
            g[0] = -1.0f;
        }
    }
    loss[e] = L;
    if (!isfinite(L)) atomicOr(flags, FLAG_NONFINITE);
#pragma unroll
    for (int k = 0; k < D; ++k) seed[e * D + k] = g[k] / (float)p.n_body;  // dL/dxbar * m / (n_body m)
}

// actuator ids must be -1 (passive) or in [0, n_act): anything else raises FLAG_BAD_ACTUATOR,
// reported as MPM_ERR_INVALID_ARG by the next synchronising call
__global__ void k_check_aid(int64_t n, int n_act, const int32_t* __restrict__ aid, int* flags) {
    pdl_begin();
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int a = aid[i];
    if (a < -1 || a >= n_act) atomicOr(flags, FLAG_BAD_ACTUATOR);
}

inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

#define DISPATCH(D, ...) \
    do {                 \
        if ((D) == 2) {  \
            constexpr int DIM = 2; __VA_ARGS__; \
        } else {         \
            constexpr int DIM = 3; __VA_ARGS__; \
        }                \
    } while (0)

void launch_ctrl_fwd(const KParams& p, const float* theta, int32_t T, float* alpha, cudaStream_t s) {
    if (p.n_act <= 0 || T <= 0) return;
    launch_k(k_ctrl_fwd, T, 128, 0, s, p, theta, alpha);
}

void launch_ctrl_bwd(const KParams& p, const float* theta, int32_t T, const float* alpha,
                     const float* alpha_bar, float* theta_part, float* theta_bar, int64_t n_theta,
                     cudaStream_t s) {
    if (p.n_act <= 0 || T <= 0) return;
    launch_k(k_ctrl_bwd, T, 128, 0, s, p, theta, alpha, alpha_bar, theta_part, n_theta);
    launch_k(k_ctrl_reduce, nblk(n_theta, 128), 128, 0, s, theta_part, T, n_theta, theta_bar);
}


void launch_check_aid(const KParams& p, const int32_t* aid, int* flags, cudaStream_t s) {
    launch_k(k_check_aid, nblk(p.EN, 256), 256, 0, s, p.EN, p.n_act, aid, flags);
}

int obs_parts(const KParams& p) { return p.E * (int)((p.N + kObsThreads - 1) / kObsThreads); }
int obs_values(const KParams& p) { return obs_nvals(p.n_act, p.dim); }

void launch_observe(const KParams& p, const float* x, const float* vc, const int* pid, const int32_t* aid,
                    float* part, cudaStream_t s) {
    const int nch = (int)((p.N + kObsThreads - 1) / kObsThreads);
    const size_t smem = sizeof(float) * (kObsThreads / 32) * obs_nvals(p.n_act, p.dim);
    DISPATCH(p.dim, launch_k(k_observe<DIM>, dim3(nch, p.E), kObsThreads, smem, s, p, x, vc, pid, aid, part));
}
void launch_ctrl_obs_fwd(const KParams& p, const float* theta, int32_t t, const float* part, float* obs_t,
                         float* counts, float* alpha_t, cudaStream_t s) {
    const int nch = (int)((p.N + kObsThreads - 1) / kObsThreads);
    DISPATCH(p.dim, launch_k(k_ctrl_obs_fwd<DIM>, p.E, 128, 0, s, p, theta, t, part, nch, obs_t, counts, alpha_t));
}
void launch_ctrl_obs_bwd(const KParams& p, const float* theta, int32_t t, const float* obs_t,
                         const float* alpha_t, const float* alpha_bar_t, const float* counts,
                         float* theta_bar, float* inc, cudaStream_t s) {
    DISPATCH(p.dim, launch_k(k_ctrl_obs_bwd<DIM>, 1, 256, 0, s, p, theta, t, obs_t, alpha_t, alpha_bar_t, counts,
                                                         theta_bar, inc));
}
void launch_observe_adj(const KParams& p, const AdjView& Sb, const int* pid, const int32_t* aid,
                        const float* inc, cudaStream_t s) {
    DISPATCH(p.dim, launch_k(k_observe_adj<DIM>, nblk(p.EN, 256), 256, 0, s, p, Sb, pid, aid, inc));
}

int loss_blocks_per_episode(const KParams& p) {
    int64_t nb = (p.N + 4095) / 4096;
    return (int)(nb < 1 ? 1 : (nb > 512 ? 512 : nb));
}

void launch_loss(const KParams& p, const float* x, int loss_kind, float3 target, float* com_part,
                 float* loss, const AdjView& Sb, int* flags, cudaStream_t s) {
    const int nb = loss_blocks_per_episode(p);
    float* seed = com_part + (int64_t)p.E * nb * p.dim;
    DISPATCH(p.dim, {
        launch_k(k_sum_partial<DIM, DIM>, dim3(nb, p.E), kLossThreads, 0, s, p, x, com_part);
        launch_k(k_loss_final<DIM>, p.E, 32, 0, s, p, com_part, nb, loss_kind, target, loss, seed, flags);
        launch_k(k_seed<DIM>, nblk(p.N * p.E, 256), 256, 0, s, p, seed, Sb);
    });
}

void launch_loss_blocks(const KParams& p, const ListSrc* src, int nsrc, int loss_kind, float3 target, float* loss,
                        float* seed, const AdjView& Sb, int* flags, cudaStream_t s) {
    ListSrcs ls{};
    ls.n = nsrc < kMaxListSrc ? nsrc : kMaxListSrc;
    for (int q = 0; q < ls.n; ++q) ls.s[q] = src[q];
    DISPATCH(p.dim, {
        launch_k(k_loss_blocks<DIM>, p.E, 32, 0, s, p, ls, loss_kind, target, loss, seed, flags);
        launch_k(k_seed<DIM>, nblk(p.N * p.E, 256), 256, 0, s, p, seed, Sb);
    });
}

void launch_v_sum(const KParams& p, const float* vc_bar, float* part, float* out, cudaStream_t s) {
    const int nb = loss_blocks_per_episode(p);
    DISPATCH(p.dim, {
        launch_k(k_sum_partial<DIM, DIM + DIM * DIM>, dim3(nb, p.E), kLossThreads, 0, s, p, vc_bar, part);
        launch_k(k_sum_parts<DIM>, p.E, 32, 0, s, part, nb, out);
    });
}

void launch_pack(const KParams& p, const float* x, const float* v, const float* C, const float* F,
                 const int* src, float* dx, float* dvc, float* df, int* ident_pid, bool zero_f,
                 cudaStream_t s) {
    DISPATCH(p.dim, launch_k(k_pack<DIM>, nblk(p.N * p.E, 256), 256, 0, s, p, x, v, C, F, src, dx, dvc, df,
                                                                     ident_pid, zero_f));
}

void launch_unpack(const KParams& p, const float* sx, const float* svc, const float* sf, const int* dst,
                   float* x, float* v, float* C, float* F, cudaStream_t s, int64_t n_rows) {
    const int64_t n = n_rows >= 0 ? n_rows : p.N * p.E;
    if (n <= 0) return;
    DISPATCH(p.dim, launch_k(k_unpack<DIM>, nblk(n, 256), 256, 0, s, p, sx, svc, sf, dst, x, v, C, F, n));
}

}  // namespace mpm
