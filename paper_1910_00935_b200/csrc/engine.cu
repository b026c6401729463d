// engine.cu -- the C-ABI (include/mpm.h): handle, workspace carving, the tape with
// segment checkpointing (Appendix D) and error reporting.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "../../include/mpm.h"
#include "kernels.h"

using namespace mpm;

namespace {

enum Phase { kCreated = 0, kBound, kHasState, kForward, kSeeded, kBackward };

// kernel classes for the per-kernel device-time accounting (mpm_kernel_stats)
enum KClass { KC_P2G = 0, KC_GRID_OP, KC_G2P, KC_G2P_GRAD, KC_GRID_OP_GRAD, KC_P2G_GRAD,
              KC_REDUCE_ABAR, KC_CLEAR, KC_CTRL, KC_LOSS, KC_LAYOUT, KC_N };
const char* const kClassNames[KC_N] = {"p2g", "grid_op", "g2p", "g2p_grad", "grid_op_grad",
                                        "p2g_grad", "reduce_abar", "clear_grid", "controller",
                                        "loss", "layout"};

struct Profiler {
    bool on = false;
    std::vector<cudaEvent_t> pool;
    size_t used = 0;
    std::vector<std::pair<int, size_t>> pending;
    double ms[KC_N] = {0};
    int64_t n[KC_N] = {0};
};

size_t align_up(size_t n) { return (n + 255) & ~size_t(255); }

}  // namespace

struct mpm_ctx {
    // creation arguments
    int64_t N = 0;
    int32_t n_grid = 0, dim = 0;
    float dt = 0, E = 0, nu = 0;
    mpm_params prm{};
    cudaStream_t stream = 0;
    int device = 0;
    std::string err;
    int64_t launches = 0;
    // workspace
    char* ws = nullptr;
    size_t ws_bytes = 0;
    size_t state_floats = 0;  // E * N * R
    int n_ckpt = 0;
    float* ckpt = nullptr;      // [n_ckpt][E*N*R]   S_{s k}
    float* window = nullptr;    // [k][E*N*R]        S_{s k + j}, j = 1..k-1
    float* final_state = nullptr;  // [E*N*R]        S_T of the recorded forward
    float* sbar[2] = {nullptr, nullptr};
    float* staging = nullptr;   // [E*N*R] caller-layout copies
    int32_t* aid = nullptr;     // [E*N]
    float4* grid = nullptr;     // [E][nodes]  (P, M)
    float4* U = nullptr;        // [E][nodes]  (U, z)
    float4* Ubar = nullptr;
    float4* gbar = nullptr;
    float* alpha = nullptr;     // [max_steps][n_act]
    float* alpha_bar = nullptr;
    float* abar_part = nullptr; // [p2g_grad blocks][n_act]
    float* theta = nullptr;
    float* theta_bar = nullptr;
    float* theta_part = nullptr;  // [max_steps][n_theta]
    float* loss = nullptr;      // [E]
    float* com_part = nullptr;
    int* flags = nullptr;       // device error flags
    int* h_flags = nullptr;     // pinned host mirror
    // tape
    Phase phase = kCreated;
    bool has_aid = false;
    int32_t recorded = 0;       // T of the recorded forward
    int32_t t_final = 0;        // T whose state lives in final_state (0 = none)
    int window_seg = -1;        // segment whose intermediate states are in the window
    int sbar_cur = 0;           // index of the adjoint buffer holding S_bar of the current step
    Profiler prof;
    int64_t* com_part_count = nullptr;  // scratch counter (active nodes)
};

namespace {

mpm_status fail(mpm_handle h, mpm_status st, const std::string& msg) {
    if (h) h->err = msg;
    return st;
}

#define CU(call)                                                                       \
    do {                                                                               \
        cudaError_t e_ = (call);                                                       \
        if (e_ != cudaSuccess)                                                         \
            return fail(h, MPM_ERR_CUDA, std::string(#call ": ") + cudaGetErrorString(e_)); \
    } while (0)

int64_t n_theta_of(const mpm_params& p) {
    int64_t H = p.ctrl_hidden, S = p.n_sin, A = p.n_actuators;
    if (A <= 0) return 0;
    return H > 0 ? H * S + H + A * H + A : A * S + A;
}

KParams kparams(const mpm_ctx* h) {
    KParams k{};
    const mpm_params& p = h->prm;
    k.dim = h->dim;
    k.n_grid = h->n_grid;
    k.bound = p.bound;
    k.model = p.model;
    k.n_act = p.n_actuators;
    k.act_axis = p.act_axis;
    k.n_sin = p.n_sin;
    k.hidden = p.ctrl_hidden;
    k.dt = h->dt;
    k.dx = 1.0f / (float)h->n_grid;
    k.inv_dx = (float)h->n_grid;
    // R3: Lame parameters from (E, nu), evaluated in double then rounded
    k.mu = (float)((double)h->E / (2.0 * (1.0 + (double)h->nu)));
    k.lam = (float)((double)h->E * h->nu / ((1.0 + h->nu) * (1.0 - 2.0 * h->nu)));
    k.p_mass = p.p_mass;
    k.p_vol = p.p_vol;
    k.gravity = p.gravity;
    k.eps_mass = p.eps_mass;
    k.kappa = p.act_strength;
    k.omega = p.omega;
    k.stress_scale = (float)(-(double)h->dt * p.p_vol * 4.0 * h->n_grid * h->n_grid);
    k.N = h->N;
    k.nodes = h->dim == 2 ? (int64_t)h->n_grid * h->n_grid
                          : (int64_t)h->n_grid * h->n_grid * h->n_grid;
    k.E = p.n_episodes;
    return k;
}

int record_floats(int dim) { return 2 * dim + 2 * dim * dim; }

// carve (or just size, when base == nullptr) the workspace
size_t carve(mpm_ctx* h, char* base) {
    const mpm_params& p = h->prm;
    const KParams k = kparams(h);
    const size_t E = (size_t)p.n_episodes, N = (size_t)h->N;
    const size_t sf = E * N * record_floats(h->dim);
    const int kk = p.k_ckpt;
    const int n_ckpt = p.max_steps / kk + 1;
    const size_t nodes = (size_t)k.nodes * E;
    const int A = p.n_actuators > 0 ? p.n_actuators : 1;
    const int64_t nth = n_theta_of(p) > 0 ? n_theta_of(p) : 1;
    const int pblk = p2g_grad_blocks(k);
    const int lblk = loss_blocks_per_episode(k);
    size_t off = 0;
    auto take = [&](size_t bytes) -> char* {
        char* ptr = base ? base + off : nullptr;
        off += align_up(bytes);
        return ptr;
    };
    float* ckpt = (float*)take(sizeof(float) * sf * n_ckpt);
    float* window = (float*)take(sizeof(float) * sf * kk);
    float* final_state = (float*)take(sizeof(float) * sf);
    float* sb0 = (float*)take(sizeof(float) * sf);
    float* sb1 = (float*)take(sizeof(float) * sf);
    float* staging = (float*)take(sizeof(float) * sf);
    int32_t* aid = (int32_t*)take(sizeof(int32_t) * E * N);
    float4* grid = (float4*)take(sizeof(float4) * nodes);
    float4* U = (float4*)take(sizeof(float4) * nodes);
    float4* Ubar = (float4*)take(sizeof(float4) * nodes);
    float4* gbar = (float4*)take(sizeof(float4) * nodes);
    float* alpha = (float*)take(sizeof(float) * (size_t)p.max_steps * A);
    float* alpha_bar = (float*)take(sizeof(float) * (size_t)p.max_steps * A);
    float* abar_part = (float*)take(sizeof(float) * (size_t)pblk * A);
    float* theta = (float*)take(sizeof(float) * nth);
    float* theta_bar = (float*)take(sizeof(float) * nth);
    float* theta_part = (float*)take(sizeof(float) * (size_t)p.max_steps * nth);
    float* loss = (float*)take(sizeof(float) * E);
    float* com_part = (float*)take(sizeof(float) * E * (lblk + 1) * 3);
    int* flags = (int*)take(sizeof(int) * 4);
    int64_t* cnt = (int64_t*)take(sizeof(int64_t) * 2);
    if (base) {
        h->com_part_count = cnt;
        h->state_floats = sf;
        h->n_ckpt = n_ckpt;
        h->ckpt = ckpt; h->window = window; h->final_state = final_state; h->sbar[0] = sb0; h->sbar[1] = sb1;
        h->staging = staging; h->aid = aid; h->grid = grid; h->U = U; h->Ubar = Ubar;
        h->gbar = gbar; h->alpha = alpha; h->alpha_bar = alpha_bar; h->abar_part = abar_part;
        h->theta = theta; h->theta_bar = theta_bar; h->theta_part = theta_part; h->loss = loss;
        h->com_part = com_part; h->flags = flags;
    }
    return off;
}

// S_t lives in: final_state (t = T of the forward), a checkpoint slot (t % k == 0)
// or the window (the intermediate states of one segment).
float* state_ptr(mpm_ctx* h, int t) {
    const int k = h->prm.k_ckpt;
    if (t > 0 && t == h->t_final) return h->final_state;
    if (t % k == 0) return h->ckpt + (size_t)(t / k) * h->state_floats;
    return h->window + (size_t)(t % k) * h->state_floats;
}

// collect pending event pairs (the stream must be synchronised)
void prof_harvest(mpm_ctx* h) {
    for (auto& pr : h->prof.pending) {
        float ms = 0.0f;
        if (cudaEventElapsedTime(&ms, h->prof.pool[pr.second], h->prof.pool[pr.second + 1]) == cudaSuccess) {
            h->prof.ms[pr.first] += ms;
            h->prof.n[pr.first] += 1;
        }
    }
    h->prof.pending.clear();
    h->prof.used = 0;
}

// brackets one library launch with CUDA events when profiling is on
struct KScope {
    mpm_ctx* h;
    int cls;
    size_t idx = 0;
    bool active = false;
    KScope(mpm_ctx* h_, int c) : h(h_), cls(c) {
        if (!h->prof.on) return;
        if (h->prof.used + 2 > h->prof.pool.size()) {
            cudaStreamSynchronize(h->stream);
            prof_harvest(h);
        }
        idx = h->prof.used;
        h->prof.used += 2;
        cudaEventRecord(h->prof.pool[idx], h->stream);
        active = true;
    }
    ~KScope() {
        if (!active) return;
        cudaEventRecord(h->prof.pool[idx + 1], h->stream);
        h->prof.pending.emplace_back(cls, idx);
    }
};

// check + clear the device flags; synchronises the stream
mpm_status sync_flags(mpm_handle h, const char* where) {
    CU(cudaMemcpyAsync(h->h_flags, h->flags, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    CU(cudaGetLastError());
    prof_harvest(h);
    const int f = *h->h_flags;
    if (f) {
        CU(cudaMemsetAsync(h->flags, 0, sizeof(int), h->stream));
        CU(cudaStreamSynchronize(h->stream));
        if (f & FLAG_OUT_OF_DOMAIN)
            return fail(h, MPM_ERR_OUT_OF_DOMAIN,
                        std::string(where) + ": a particle stencil left [0, n_grid-1]^d");
        return fail(h, MPM_ERR_NONFINITE,
                    std::string(where) + ": non-finite value or degenerate deformation (J<=0 / r=0)");
    }
    return MPM_OK;
}

// advance(): clear_grid, p2g (actuation precomputed), grid_op, g2p
void step_forward(mpm_ctx* h, const KParams& k, int t, const float* S, float* Sn) {
    const size_t gbytes = sizeof(float4) * (size_t)k.nodes * k.E;
    { KScope sc(h, KC_CLEAR); cudaMemsetAsync(h->grid, 0, gbytes, h->stream); }
    const float* al = h->alpha + (size_t)t * (k.n_act > 0 ? k.n_act : 1);
    { KScope sc(h, KC_P2G); launch_p2g(k, S, h->has_aid ? h->aid : nullptr, al, h->grid, Sn, h->flags, h->stream); }
    { KScope sc(h, KC_GRID_OP); launch_grid_op(k, h->grid, h->U, h->stream); }
    { KScope sc(h, KC_G2P); launch_g2p(k, S, h->U, Sn, h->flags, h->stream); }
    h->launches += 3;
}

// advance_grad(): recompute the grid, then g2p.grad, grid_op.grad, p2g.grad
void step_backward(mpm_ctx* h, const KParams& k, int t, const float* S, const float* Sbn, float* Sb) {
    const size_t gbytes = sizeof(float4) * (size_t)k.nodes * k.E;
    const int A = k.n_act > 0 ? k.n_act : 1;
    const float* al = h->alpha + (size_t)t * A;
    { KScope sc(h, KC_CLEAR); cudaMemsetAsync(h->grid, 0, gbytes, h->stream); }
    { KScope sc(h, KC_P2G); launch_p2g(k, S, h->has_aid ? h->aid : nullptr, al, h->grid, nullptr, h->flags, h->stream); }
    { KScope sc(h, KC_GRID_OP); launch_grid_op(k, h->grid, h->U, h->stream); }
    { KScope sc(h, KC_CLEAR); cudaMemsetAsync(h->Ubar, 0, gbytes, h->stream); }
    { KScope sc(h, KC_G2P_GRAD); launch_g2p_grad(k, S, h->U, Sbn, h->Ubar, Sb, h->stream); }
    { KScope sc(h, KC_GRID_OP_GRAD); launch_grid_op_grad(k, h->grid, h->U, h->Ubar, h->gbar, h->stream); }
    { KScope sc(h, KC_P2G_GRAD);
      launch_p2g_grad(k, S, h->has_aid ? h->aid : nullptr, al, h->gbar, Sbn, Sb, h->abar_part, h->flags, h->stream); }
    h->launches += 5;
    if (k.n_act > 0) {
        KScope sc(h, KC_REDUCE_ABAR);
        launch_reduce_abar(k, h->abar_part, p2g_grad_blocks(k), h->alpha_bar + (size_t)t * A, h->stream);
        h->launches += 1;
    }
}

mpm_status copy_in(mpm_handle h, void* dst, const void* src, size_t bytes) {
    CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, h->stream));
    return MPM_OK;
}

}  // namespace

extern "C" {

mpm_status mpm_default_params(int32_t dim, mpm_params* p) {
    if (!p || (dim != 2 && dim != 3)) return MPM_ERR_INVALID_ARG;
    std::memset(p, 0, sizeof(*p));
    p->gravity = dim == 2 ? 3.8f : 10.0f;
    p->p_mass = 1.0f;
    p->p_vol = 1.0f;
    p->eps_mass = 1e-10f;
    p->bound = 3;
    p->model = dim == 2 ? MPM_MODEL_FIXED_COROTATED : MPM_MODEL_NEOHOOKEAN;
    p->k_ckpt = 1;
    p->max_steps = 2048;
    p->n_actuators = 0;
    p->act_strength = 4.0f;
    p->act_axis = 1;
    p->n_sin = 4;
    p->omega = 20.0f;
    p->ctrl_hidden = 0;
    p->n_episodes = 1;
    p->deterministic = 0;
    p->loss_kind = MPM_LOSS_COM_TARGET;
    return MPM_OK;
}

mpm_status mpm_create(int64_t n_particles, int32_t n_grid, int32_t dim, float dt, float E,
                      float nu, mpm_handle* out) {
    if (!out) return MPM_ERR_INVALID_ARG;
    *out = nullptr;
    if (n_particles < 1 || n_grid < 4 || (dim != 2 && dim != 3) || !(dt > 0) || !(E > 0) ||
        !(nu > -1.0f && nu < 0.5f))
        return MPM_ERR_INVALID_ARG;
    if (n_particles > (int64_t)1 << 31) return MPM_ERR_INVALID_ARG;
    mpm_ctx* h = new mpm_ctx();
    h->N = n_particles;
    h->n_grid = n_grid;
    h->dim = dim;
    h->dt = dt;
    h->E = E;
    h->nu = nu;
    mpm_default_params(dim, &h->prm);
    cudaError_t e = cudaGetDevice(&h->device);
    if (e == cudaSuccess) e = cudaMallocHost((void**)&h->h_flags, sizeof(int) * 4);
    if (e != cudaSuccess) {
        delete h;
        return MPM_ERR_CUDA;
    }
    *out = h;
    return MPM_OK;
}

mpm_status mpm_destroy(mpm_handle h) {
    if (!h) return MPM_ERR_INVALID_ARG;
    if (h->h_flags) cudaFreeHost(h->h_flags);
    for (auto ev : h->prof.pool) cudaEventDestroy(ev);
    delete h;
    return MPM_OK;
}

const char* mpm_last_error(mpm_handle h) { return h ? h->err.c_str() : "null handle"; }

mpm_status mpm_get_params(mpm_handle h, mpm_params* p) {
    if (!h || !p) return MPM_ERR_INVALID_ARG;
    *p = h->prm;
    return MPM_OK;
}

mpm_status mpm_set_params(mpm_handle h, const mpm_params* p) {
    if (!h || !p) return MPM_ERR_INVALID_ARG;
    if (h->phase >= kBound) return fail(h, MPM_ERR_BAD_SEQUENCE, "set_params after bind_workspace");
    if (p->k_ckpt < 1 || p->max_steps < 1 || p->n_episodes < 1 || p->bound < 0 ||
        p->n_actuators < 0 || p->n_actuators > 256 || p->ctrl_hidden < 0 || p->ctrl_hidden > 1024 ||
        p->n_sin < 1 || p->n_sin > 64 || p->act_axis < 0 || p->act_axis >= h->dim ||
        !(p->p_mass > 0) || !(p->p_vol > 0) || p->eps_mass < 0 ||
        (p->loss_kind != MPM_LOSS_COM_TARGET && p->loss_kind != MPM_LOSS_MOVE_FORWARD))
        return fail(h, MPM_ERR_INVALID_ARG, "invalid mpm_params");
    if (p->model != MPM_MODEL_NEOHOOKEAN && p->model != MPM_MODEL_FIXED_COROTATED)
        return fail(h, MPM_ERR_INVALID_ARG, "unknown model");
    if (p->model == MPM_MODEL_FIXED_COROTATED && h->dim == 3)
        return fail(h, MPM_ERR_UNSUPPORTED, "fixed-corotated in 3D needs an SVD (out of scope, R2)");
    if ((int64_t)p->n_episodes * h->N > ((int64_t)1 << 31))
        return fail(h, MPM_ERR_INVALID_ARG, "n_episodes * n_particles exceeds 2^31");
    h->prm = *p;
    return MPM_OK;
}

mpm_status mpm_set_stream(mpm_handle h, void* s) {
    if (!h) return MPM_ERR_INVALID_ARG;
    h->stream = (cudaStream_t)s;
    return MPM_OK;
}

mpm_status mpm_workspace_bytes(mpm_handle h, size_t* bytes) {
    if (!h || !bytes) return MPM_ERR_INVALID_ARG;
    *bytes = carve(h, nullptr);
    return MPM_OK;
}

mpm_status mpm_bind_workspace(mpm_handle h, void* dptr, size_t bytes) {
    if (!h || !dptr) return MPM_ERR_INVALID_ARG;
    if (((uintptr_t)dptr & 255) != 0) return fail(h, MPM_ERR_INVALID_ARG, "workspace not 256-B aligned");
    size_t need = carve(h, nullptr);
    if (bytes < need)
        return fail(h, MPM_ERR_OOM, "workspace too small: need " + std::to_string(need) + " bytes");
    h->ws = (char*)dptr;
    h->ws_bytes = bytes;
    carve(h, h->ws);
    CU(cudaMemsetAsync(h->flags, 0, sizeof(int) * 4, h->stream));
    CU(cudaMemsetAsync(h->theta, 0, sizeof(float) * (n_theta_of(h->prm) > 0 ? n_theta_of(h->prm) : 1),
                       h->stream));
    h->phase = kBound;
    return MPM_OK;
}

mpm_status mpm_set_state(mpm_handle h, const float* x, const float* v, const float* C,
                         const float* F, const int32_t* actuator_id) {
    if (!h) return MPM_ERR_INVALID_ARG;
    if (h->phase < kBound) return fail(h, MPM_ERR_BAD_SEQUENCE, "set_state before bind_workspace");
    if (!x) return fail(h, MPM_ERR_INVALID_ARG, "x is required");
    const KParams k = kparams(h);
    const size_t EN = (size_t)k.E * k.N, d = (size_t)h->dim;
    float* sx = h->staging;
    float* sv = sx + EN * d;
    float* sC = sv + EN * d;
    float* sF = sC + EN * d * d;
    mpm_status st;
    if ((st = copy_in(h, sx, x, sizeof(float) * EN * d))) return st;
    if (v && (st = copy_in(h, sv, v, sizeof(float) * EN * d))) return st;
    if (C && (st = copy_in(h, sC, C, sizeof(float) * EN * d * d))) return st;
    if (F && (st = copy_in(h, sF, F, sizeof(float) * EN * d * d))) return st;
    { KScope sc(h, KC_LAYOUT); launch_pack(k, sx, v ? sv : nullptr, C ? sC : nullptr, F ? sF : nullptr, h->ckpt, h->stream); }
    h->launches += 1;
    h->has_aid = actuator_id != nullptr;
    if (actuator_id && (st = copy_in(h, h->aid, actuator_id, sizeof(int32_t) * EN))) return st;
    CU(cudaGetLastError());
    h->phase = kHasState;
    h->recorded = 0;
    h->t_final = 0;
    h->window_seg = -1;
    return MPM_OK;
}

mpm_status mpm_n_theta(mpm_handle h, int64_t* n) {
    if (!h || !n) return MPM_ERR_INVALID_ARG;
    *n = n_theta_of(h->prm);
    return MPM_OK;
}

mpm_status mpm_set_controller(mpm_handle h, const float* theta, int64_t n) {
    if (!h) return MPM_ERR_INVALID_ARG;
    if (h->phase < kBound) return fail(h, MPM_ERR_BAD_SEQUENCE, "set_controller before bind_workspace");
    if (n != n_theta_of(h->prm) || (n > 0 && !theta))
        return fail(h, MPM_ERR_INVALID_ARG, "n_theta mismatch: expected " + std::to_string(n_theta_of(h->prm)));
    if (n > 0) return copy_in(h, h->theta, theta, sizeof(float) * n);
    return MPM_OK;
}

mpm_status mpm_forward(mpm_handle h, int32_t steps) {
    if (!h) return MPM_ERR_INVALID_ARG;
    if (h->phase < kHasState) return fail(h, MPM_ERR_BAD_SEQUENCE, "forward before set_state");
    if (steps < 1 || steps > h->prm.max_steps)
        return fail(h, MPM_ERR_INVALID_ARG, "steps must be in [1, max_steps]");
    const KParams k = kparams(h);
    h->t_final = steps;
    { KScope sc(h, KC_CTRL); launch_ctrl_fwd(k, h->theta, steps, h->alpha, h->stream); }
    if (k.n_act > 0) h->launches += 1;
    for (int t = 0; t < steps; ++t) step_forward(h, k, t, state_ptr(h, t), state_ptr(h, t + 1));
    CU(cudaGetLastError());
    h->recorded = steps;
    h->window_seg = (steps - 1) / h->prm.k_ckpt;
    h->phase = kForward;
    mpm_status st = sync_flags(h, "mpm_forward");
    if (st) h->phase = kHasState;
    return st;
}

mpm_status mpm_loss(mpm_handle h, float* loss_out) {
    if (!h) return MPM_ERR_INVALID_ARG;
    if (h->phase < kForward) return fail(h, MPM_ERR_BAD_SEQUENCE, "loss before forward");
    const KParams k = kparams(h);
    const float3 tgt = make_float3(h->prm.loss_target[0], h->prm.loss_target[1], h->prm.loss_target[2]);
    h->sbar_cur = 0;
    { KScope sc(h, KC_LOSS);
      launch_loss(k, state_ptr(h, h->recorded), h->prm.loss_kind, tgt, h->com_part, h->loss,
                  h->sbar[0], h->flags, h->stream); }
    h->launches += 3;
    if (loss_out) CU(cudaMemcpyAsync(loss_out, h->loss, sizeof(float) * k.E, cudaMemcpyDefault, h->stream));
    mpm_status st = sync_flags(h, "mpm_loss");
    if (st) return st;
    h->phase = kSeeded;
    return MPM_OK;
}

mpm_status mpm_seed_adjoint(mpm_handle h, const float* dx, const float* dv, const float* dC,
                            const float* dF) {
    if (!h) return MPM_ERR_INVALID_ARG;
    if (h->phase < kForward) return fail(h, MPM_ERR_BAD_SEQUENCE, "seed_adjoint before forward");
    const KParams k = kparams(h);
    const size_t EN = (size_t)k.E * k.N, d = (size_t)h->dim;
    float* sx = h->staging;
    float* sv = sx + EN * d;
    float* sC = sv + EN * d;
    float* sF = sC + EN * d * d;
    mpm_status st;
    if (dx && (st = copy_in(h, sx, dx, sizeof(float) * EN * d))) return st;
    if (dv && (st = copy_in(h, sv, dv, sizeof(float) * EN * d))) return st;
    if (dC && (st = copy_in(h, sC, dC, sizeof(float) * EN * d * d))) return st;
    if (dF && (st = copy_in(h, sF, dF, sizeof(float) * EN * d * d))) return st;
    if (!dF) CU(cudaMemsetAsync(sF, 0, sizeof(float) * EN * d * d, h->stream));
    { KScope sc(h, KC_LAYOUT); launch_pack(k, dx ? sx : nullptr, dv ? sv : nullptr, dC ? sC : nullptr, sF, h->sbar[0], h->stream); }
    h->launches += 1;
    CU(cudaGetLastError());
    h->sbar_cur = 0;
    h->phase = kSeeded;
    return MPM_OK;
}

mpm_status mpm_backward(mpm_handle h, int32_t steps) {
    if (!h) return MPM_ERR_INVALID_ARG;
    if (h->phase != kSeeded) return fail(h, MPM_ERR_BAD_SEQUENCE, "backward needs forward + loss/seed_adjoint");
    if (steps != h->recorded)
        return fail(h, MPM_ERR_BAD_SEQUENCE, "backward steps != recorded forward steps");
    const KParams k = kparams(h);
    const int kk = h->prm.k_ckpt, T = steps;
    const int A = k.n_act > 0 ? k.n_act : 1;
    if (k.n_act > 0) CU(cudaMemsetAsync(h->alpha_bar, 0, sizeof(float) * (size_t)T * A, h->stream));
    const int nseg = (T + kk - 1) / kk;
    for (int s = nseg - 1; s >= 0; --s) {
        const int t0 = s * kk, t1 = (t0 + kk < T) ? t0 + kk : T;
        if (h->window_seg != s) {  // segment-wise recomputation
            for (int t = t0; t < t1 - 1; ++t) step_forward(h, k, t, state_ptr(h, t), state_ptr(h, t + 1));
            h->window_seg = s;
        }
        for (int t = t1 - 1; t >= t0; --t) {
            step_backward(h, k, t, state_ptr(h, t), h->sbar[h->sbar_cur], h->sbar[h->sbar_cur ^ 1]);
            h->sbar_cur ^= 1;
        }
    }
    const int64_t nth = n_theta_of(h->prm);
    if (nth > 0) {
        KScope sc(h, KC_CTRL);
        launch_ctrl_bwd(k, h->theta, T, h->alpha, h->alpha_bar, h->theta_part, h->theta_bar, nth, h->stream);
        h->launches += 2;
    }
    CU(cudaGetLastError());
    mpm_status st = sync_flags(h, "mpm_backward");
    if (st) return st;
    h->phase = kBackward;
    return MPM_OK;
}

mpm_status mpm_grads(mpm_handle h, float* dx0, float* dv0, float* dC0, float* dF0, float* dtheta) {
    if (!h) return MPM_ERR_INVALID_ARG;
    if (h->phase != kBackward) return fail(h, MPM_ERR_BAD_SEQUENCE, "grads before backward");
    const KParams k = kparams(h);
    const size_t EN = (size_t)k.E * k.N, d = (size_t)h->dim;
    float* sx = h->staging;
    float* sv = sx + EN * d;
    float* sC = sv + EN * d;
    float* sF = sC + EN * d * d;
    { KScope sc(h, KC_LAYOUT); launch_unpack(k, h->sbar[h->sbar_cur], sx, sv, sC, sF, h->stream); }
    h->launches += 1;
    if (dx0) CU(cudaMemcpyAsync(dx0, sx, sizeof(float) * EN * d, cudaMemcpyDefault, h->stream));
    if (dv0) CU(cudaMemcpyAsync(dv0, sv, sizeof(float) * EN * d, cudaMemcpyDefault, h->stream));
    if (dC0) CU(cudaMemcpyAsync(dC0, sC, sizeof(float) * EN * d * d, cudaMemcpyDefault, h->stream));
    if (dF0) CU(cudaMemcpyAsync(dF0, sF, sizeof(float) * EN * d * d, cudaMemcpyDefault, h->stream));
    const int64_t nth = n_theta_of(h->prm);
    if (dtheta && nth > 0)
        CU(cudaMemcpyAsync(dtheta, h->theta_bar, sizeof(float) * nth, cudaMemcpyDefault, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    CU(cudaGetLastError());
    return MPM_OK;
}

mpm_status mpm_grad_v0_sum(mpm_handle h, float* out) {
    if (!h || !out) return MPM_ERR_INVALID_ARG;
    if (h->phase != kBackward) return fail(h, MPM_ERR_BAD_SEQUENCE, "grad_v0_sum before backward");
    const KParams k = kparams(h);
    float* res = h->com_part + (size_t)k.E * loss_blocks_per_episode(k) * 3;  // tail of com_part
    { KScope sc(h, KC_LOSS); launch_v_sum(k, h->sbar[h->sbar_cur], h->com_part, res, h->stream); }
    h->launches += 2;
    CU(cudaMemcpyAsync(out, res, sizeof(float) * k.E * h->dim, cudaMemcpyDefault, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    CU(cudaGetLastError());
    return MPM_OK;
}

mpm_status mpm_get_state(mpm_handle h, float* x, float* v, float* C, float* F) {
    if (!h) return MPM_ERR_INVALID_ARG;
    if (h->phase < kHasState) return fail(h, MPM_ERR_BAD_SEQUENCE, "get_state before set_state");
    const KParams k = kparams(h);
    const size_t EN = (size_t)k.E * k.N, d = (size_t)h->dim;
    float* sx = h->staging;
    float* sv = sx + EN * d;
    float* sC = sv + EN * d;
    float* sF = sC + EN * d * d;
    { KScope sc(h, KC_LAYOUT); launch_unpack(k, state_ptr(h, h->recorded), sx, sv, sC, sF, h->stream); }
    h->launches += 1;
    if (x) CU(cudaMemcpyAsync(x, sx, sizeof(float) * EN * d, cudaMemcpyDefault, h->stream));
    if (v) CU(cudaMemcpyAsync(v, sv, sizeof(float) * EN * d, cudaMemcpyDefault, h->stream));
    if (C) CU(cudaMemcpyAsync(C, sC, sizeof(float) * EN * d * d, cudaMemcpyDefault, h->stream));
    if (F) CU(cudaMemcpyAsync(F, sF, sizeof(float) * EN * d * d, cudaMemcpyDefault, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    CU(cudaGetLastError());
    return MPM_OK;
}

mpm_status mpm_set_profiling(mpm_handle h, int32_t enable) {
    if (!h) return MPM_ERR_INVALID_ARG;
    if (enable && h->prof.pool.empty()) {
        h->prof.pool.resize(2 * 16384);
        for (auto& ev : h->prof.pool) CU(cudaEventCreate(&ev));
    }
    if (!enable && h->prof.on) {
        CU(cudaStreamSynchronize(h->stream));
        prof_harvest(h);
    }
    h->prof.on = enable != 0;
    return MPM_OK;
}

mpm_status mpm_reset_kernel_stats(mpm_handle h) {
    if (!h) return MPM_ERR_INVALID_ARG;
    CU(cudaStreamSynchronize(h->stream));
    prof_harvest(h);
    for (int c = 0; c < KC_N; ++c) { h->prof.ms[c] = 0; h->prof.n[c] = 0; }
    return MPM_OK;
}

mpm_status mpm_kernel_stats(mpm_handle h, int32_t idx, const char** name, double* total_ms,
                            int64_t* count) {
    if (!h || idx < 0 || idx >= KC_N) return MPM_ERR_INVALID_ARG;
    CU(cudaStreamSynchronize(h->stream));
    prof_harvest(h);
    if (name) *name = kClassNames[idx];
    if (total_ms) *total_ms = h->prof.ms[idx];
    if (count) *count = h->prof.n[idx];
    return MPM_OK;
}

mpm_status mpm_active_nodes(mpm_handle h, int64_t* count) {
    if (!h || !count) return MPM_ERR_INVALID_ARG;
    if (h->phase < kForward) return fail(h, MPM_ERR_BAD_SEQUENCE, "active_nodes before forward");
    const KParams k = kparams(h);
    { KScope sc(h, KC_LAYOUT); launch_count_active(k, h->grid, h->com_part_count, h->stream); }
    h->launches += 1;
    int64_t c = 0;
    CU(cudaMemcpyAsync(&c, h->com_part_count, sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    *count = c;
    return MPM_OK;
}

mpm_status mpm_launch_count(mpm_handle h, int64_t* count) {
    if (!h || !count) return MPM_ERR_INVALID_ARG;
    *count = h->launches;
    return MPM_OK;
}

}  // extern "C"
