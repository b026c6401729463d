// engine.cu -- the C-ABI (include/mpm.h): handle, workspace carving, the tape with
// segment checkpointing (Appendix D), error reporting and the
// per-kernel timing hooks.
//
// Tape layout: S_t (split arrays + particle ids) lives in the
// final-state buffer (t = T), a checkpoint slot (t % k == 0) or the double-buffered
// k-slot window (half (t / k) & 1); the binning and the resolved node tiles of every
// step live in the grid store, so the reverse never re-runs p2g and a segment's
// re-forward is g2p only.  Adjoint states are indexed like the state they belong to.
// Streams: main; side (g2p_grad's gather part); side2 (segment re-forward); side3 (the
// open-loop actuator-gradient reduction of each reverse step), all
// captured into the forward / backward CUDA graphs.
#include <algorithm>
#include <cstdlib>
#include <functional>
#include <map>
#include <tuple>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "engine.h"

using namespace mpm;

namespace eng {
const char* const kClassNames[KC_N] = {"p2g", "g2p", "bin", "g2p_grad", "p2g_grad", "reduce_abar",
                                        "controller", "loss", "layout", "grid_op", "grid_op_grad",
                                        "g2p_grad_gather", "canon"};
}  // namespace eng



namespace eng {


mpm_status fail(mpm_handle h, mpm_status st, const std::string& msg) {
    if (h) h->err = msg;
    return st;
}


// controller inputs: n_sin sinusoid features (+ 2d per actuator group, closed loop R22)
int64_t ctrl_inputs(const mpm_params& p, int dim) {
    return (int64_t)p.n_sin + (p.closed_loop ? 2 * dim * (int64_t)p.n_actuators : 0);
}
int64_t n_theta_of(const mpm_params& p, int dim) {
    int64_t H = p.ctrl_hidden, S = ctrl_inputs(p, dim), A = p.n_actuators;
    if (A <= 0) return 0;
    return H > 0 ? H * S + H + A * H + A : A * S + A;
}

bool closed_loop(const mpm_ctx* h) { return h->prm.closed_loop && h->prm.n_actuators > 0; }

int block_edge(int dim) { return dim == 3 ? 4 : 8; }
int tile_nodes(int dim) { return dim == 3 ? 216 : 100; }

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
    k.closed_loop = p.closed_loop && p.n_actuators > 0;
    k.n_in = (int32_t)ctrl_inputs(p, h->dim);
    k.a_estride = k.closed_loop ? p.n_actuators : 0;
    k.obs_sx = p.obs_scale_x;
    k.obs_sv = p.obs_scale_v;
    k.mat = h->has_mat ? h->mat : nullptr;
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
    k.EN = (int64_t)h->N * p.n_episodes;
    const int B = block_edge(h->dim);
    k.nb = (h->n_grid + B - 1) / B;
    k.nbe = h->dim == 2 ? k.nb * k.nb : k.nb * k.nb * k.nb;
    k.TB = k.nbe * k.E;
    k.max_active = h->pool_blocks;
    k.step_blocks = h->step_blocks;
    k.n_body = h->dd ? h->n_body : h->N;
    k.x_lo = h->dd ? h->x_lo : 0;
    k.x_hi = h->dd ? h->x_hi : k.nb;
    const bool fast = k.TB < (1 << 22);  // divq's exact range
    k.inv_nb = fast ? 1.0f / (float)k.nb : 0.0f;
    k.inv_nbe = fast ? 1.0f / (float)k.nbe : 0.0f;
    return k;
}

int record_floats(int dim) { return 2 * dim + 2 * dim * dim; }

int default_max_active(const mpm_ctx* h, const KParams& k) {
    if (h->prm.max_active_blocks > 0) return std::min(h->prm.max_active_blocks, k.TB);
    const int64_t EN = (int64_t)k.E * k.N;
    const int64_t guess = (EN + kCells - 1) / kCells * 3 + (int64_t)k.E * 64;
    return (int)std::min<int64_t>(k.TB, guess);
}

// grid-store pool capacity (blocks over all steps): grid_store_blocks, or an estimate of
// ~3x the active blocks of a dense body (8 particles per cell) per step
int64_t pool_capacity(const mpm_ctx* h, const KParams& k, int step_cap) {
    if (h->prm.grid_store_blocks > 0) return h->prm.grid_store_blocks;
    const int64_t EN = (int64_t)k.E * k.N;
    const int64_t per = std::min<int64_t>(step_cap, 3 * ((EN + 511) / 512) + (int64_t)k.E * 64 + 64);
    return per * h->prm.max_steps;
}

// carve (or just size, when base == nullptr) the workspace
size_t carve(mpm_ctx* h, char* base) {
    const mpm_params& p = h->prm;
    KParams k = kparams(h);
    const int max_active = default_max_active(h, k);   // per-step block capacity
    const int64_t pool = pool_capacity(h, k, max_active);
    const size_t E = (size_t)p.n_episodes, N = (size_t)h->N, EN = E * N;
    const size_t sf = EN * record_floats(h->dim);
    const int kk = p.k_ckpt;
    const int n_ckpt = p.max_steps / kk + 1;
    const int A = p.n_actuators > 0 ? p.n_actuators : 1;
    const int64_t nth = n_theta_of(p, h->dim) > 0 ? n_theta_of(p, h->dim) : 1;
    const bool closed = p.closed_loop && p.n_actuators > 0;
    const size_t AE = (size_t)A * (closed ? E : 1);  // alpha_t entries: per episode when closed
    const size_t n_obs = closed ? 2 * h->dim * A : 1;
    const int lblk = loss_blocks_per_episode(k);
    const size_t TN = tile_nodes(h->dim);
    const size_t d = h->dim;
    size_t off = 0;
    auto take = [&](size_t bytes) -> char* {
        char* ptr = base ? base + off : nullptr;
        off += align_up(bytes);
        return ptr;
    };
    // AoSoA state arrays (mpm_device.cuh soa<NC>): whole 32-particle tiles
    const size_t ENT = (EN + kTile - 1) / kTile * kTile;
    const size_t px = d, pvc = d + d * d, pf = d * d;
    auto state = [&]() {
        StateView s;
        s.x = (float*)take(sizeof(float) * ENT * px);
        s.vc = (float*)take(sizeof(float) * ENT * pvc);
        s.f = (float*)take(sizeof(float) * ENT * pf);
        s.pid = (int*)take(sizeof(int) * EN);
        return s;
    };
    auto adj = [&]() {
        AdjView s;
        s.x = (float*)take(sizeof(float) * ENT * px);
        s.vc = (float*)take(sizeof(float) * ENT * pvc);
        s.f = (float*)take(sizeof(float) * ENT * pf);
        return s;
    };
    std::vector<StateView> ckpt, window;
    for (int i = 0; i < n_ckpt; ++i) ckpt.push_back(state());
    for (int i = 0; i < 2 * kk; ++i) window.push_back(i % kk == 0 ? StateView{nullptr, nullptr, nullptr, nullptr} : state());
    StateView fin = state();
    const int Tm = p.max_steps;
    // per-step sorted lists at a whole-tile stride: every step's list is 128-B aligned, so the
    // thread-per-particle kernels can bulk-copy (cp.async.bulk) a block's segment of it
    int* sigma_store = (int*)take(sizeof(int) * ENT * Tm);
    unsigned char* scell0 = (unsigned char*)take(EN);
    unsigned char* scell1 = (unsigned char*)take(EN);
    int* spid0 = (int*)take(sizeof(int) * EN);
    int* spid1 = (int*)take(sizeof(int) * EN);
    int* bmap_store = (int*)take(sizeof(int) * (size_t)k.TB * Tm);
    int* nactive_arr = (int*)take(sizeof(int) * Tm);
    int* base_arr = (int*)take(sizeof(int) * Tm);
    int* blist_pool = (int*)take(sizeof(int) * (size_t)pool);
    int* nbr_pool = (int*)take(sizeof(int) * (size_t)pool * (d == 3 ? 27 : 9));
    int* bstart_pool = (int*)take(sizeof(int) * ((size_t)pool + Tm + 1));
    unsigned short* cstart_pool = (unsigned short*)take(sizeof(unsigned short) * (size_t)pool * (kCells + 1));
    float4* tiles_pool = (float4*)take(sizeof(float4) * (size_t)pool * TN);
    AdjView sb0 = adj();
    AdjView sb1 = adj();
    float* staging = (float*)take(sizeof(float) * sf);
    int32_t* aid = (int32_t*)take(sizeof(int32_t) * EN);
    int32_t* mat = (int32_t*)take(sizeof(int32_t) * std::max<size_t>(EN, (size_t)h->n_body));  // by particle id
    float* xbar_part = (float*)take(sizeof(float) * ENT * px);
    int* bcount = (int*)take(sizeof(int) * k.TB);
    int* cursor = (int*)take(sizeof(int) * k.TB);
    int* scan_part = (int*)take(sizeof(int64_t) * (scan_chunks(k) + 2));  // chunk totals, epoch, ticket
    int* keys = (int*)take(sizeof(int) * EN);
    float4* ubar = (float4*)take(sizeof(float4) * (size_t)max_active * TN);
    float4* part = (float4*)take(sizeof(float4) * (size_t)max_active * TN);
    // per work item; two buffers (step parity) so the open-loop reduction can trail p2g_grad
    float* abar_part = (float*)take(sizeof(float) * 2 * (size_t)max_active * kMaxSplit * A);
    float* alpha = (float*)take(sizeof(float) * (size_t)p.max_steps * AE);
    float* alpha_bar = (float*)take(sizeof(float) * (size_t)p.max_steps * AE);
    // closed loop (R22): observations of every step, group sizes, reduction partials, and the
    // per-group adjoint increments of the current reverse step
    float* obs = (float*)take(sizeof(float) * (closed ? (size_t)p.max_steps * E * n_obs : 1));
    float* obs_cnt = (float*)take(sizeof(float) * (closed ? E * A : 1));
    float* obs_part = (float*)take(sizeof(float) * (closed ? (size_t)obs_parts(k) * obs_values(k) : 1));
    float* obs_inc = (float*)take(sizeof(float) * (closed ? E * (n_obs + d) : 1));
    float* theta = (float*)take(sizeof(float) * nth);
    float* theta_bar = (float*)take(sizeof(float) * nth);
    float* theta_part = (float*)take(sizeof(float) * (size_t)p.max_steps * nth);
    int* ntot_arr = (int*)take(sizeof(int) * (Tm + 1));
    float* blk_part = (float*)take(sizeof(float) * (size_t)max_active * d);
    // f3 (decomposed body): migration records of every step
    const size_t dd_T = h->dd ? (size_t)Tm + 1 : 1;
    const size_t mcap = h->dd ? (size_t)h->mig_cap : 1;
    int* out_cnt = (int*)take(sizeof(int) * dd_T * 2);
    int* out_rows = (int*)take(sizeof(int) * dd_T * 2 * mcap);
    int* imm_base = (int*)take(sizeof(int) * dd_T * 2);
    int* nrows_arr = (int*)take(sizeof(int) * dd_T);
    float* loss = (float*)take(sizeof(float) * E);
    float* com_part = (float*)take(sizeof(float) * E * (lblk + 2) * 3);
    int64_t* counter = (int64_t*)take(sizeof(int64_t) * 2);
    int* flags = (int*)take(sizeof(int) * 4);
    if (base) {
        h->max_active = max_active;
        h->step_blocks = max_active;
        h->pool_blocks = pool;
        h->sigma_store = sigma_store; h->scell_ring[0] = scell0; h->scell_ring[1] = scell1;
        h->spid_ring[0] = spid0; h->spid_ring[1] = spid1; h->bmap_store = bmap_store;
        h->nactive_arr = nactive_arr; h->base_arr = base_arr; h->blist_pool = blist_pool; h->nbr_pool = nbr_pool;
        h->bstart_pool = bstart_pool; h->cstart_pool = cstart_pool; h->tiles_pool = tiles_pool;
        h->state_floats = sf;
        h->n_ckpt = n_ckpt;
        h->ckpt = ckpt;
        h->window = window;
        h->final_state = fin;
        h->sbar[0] = sb0; h->sbar[1] = sb1;
        h->xbar_part = xbar_part;
        h->staging = staging; h->aid = aid; h->mat = mat; h->bcount = bcount; h->cursor = cursor; h->scan_part = scan_part; h->keys = keys;
        h->ubar = ubar; h->part = part; h->abar_part = abar_part;
        h->abar_stride = (size_t)max_active * kMaxSplit * A;
        h->obs = obs; h->obs_cnt = obs_cnt; h->obs_part = obs_part; h->obs_inc = obs_inc;
        h->alpha = alpha; h->alpha_bar = alpha_bar; h->theta = theta; h->theta_bar = theta_bar;
        h->theta_part = theta_part; h->loss = loss; h->com_part = com_part; h->counter = counter;
        h->flags = flags;
        h->ntot_arr = ntot_arr; h->blk_part = blk_part;
        h->out_cnt = out_cnt; h->out_rows = out_rows; h->imm_base = imm_base; h->nrows_arr = nrows_arr;
    }
    return off;
}

StateView state_at(mpm_ctx* h, int t) {
    const int k = h->prm.k_ckpt;
    if (t > 0 && t == h->t_final) return h->final_state;
    if (t % k == 0) return h->ckpt[t / k];
    return h->window[((t / k) & 1) * k + t % k];
}

SlotView slot_at(mpm_ctx* h, int t) {
    const KParams k = kparams(h);
    const size_t EN = (size_t)k.E * k.N;
    SlotView s;
    s.sigma = h->sigma_store + (EN + kTile - 1) / kTile * kTile * t;
    s.scell = h->scell_ring[t & 1];
    s.spid = h->spid_ring[t & 1];
    s.blist = h->blist_pool;
    s.bstart = h->bstart_pool;
    s.bmap = h->bmap_store + (size_t)k.TB * t;
    s.nactive = h->nactive_arr + t;
    s.base = h->base_arr + t;
    s.cstart = h->cstart_pool;
    s.tiles = h->tiles_pool;
    s.part = h->part;
    s.ntot = h->ntot_arr + t;
    s.nbr = canon_fused(k) ? h->nbr_pool : nullptr;  // the neighbour table: small problems (kernels_tile.cu)
    s.step = t;
    s.halo = Halo{0, k.nb, {nullptr, nullptr}, {nullptr, nullptr}, {nullptr, nullptr}};
    if (h->dd) {
        s.halo.x_lo = h->x_lo;
        s.halo.x_hi = h->x_hi;
    }
    return s;
}

// ---------------------------------------------------------------- profiling
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
        if (f & FLAG_MIGRATION)
            return fail(h, MPM_ERR_OOM, std::string(where) +
                                            ": subdomain (f3): capacity or migration buffer exceeded, or a particle "
                                            "outside its slab / moving past a whole slab in one step");
        if (f & FLAG_BAD_ACTUATOR)
            return fail(h, MPM_ERR_INVALID_ARG, std::string(where) + ": actuator id outside [-1, n_actuators)");
        if (f & FLAG_ACTIVE_OVERFLOW)
            return fail(h, MPM_ERR_OOM, std::string(where) + ": active blocks exceed max_active_blocks (" +
                                            std::to_string(h->max_active) + ")");
        if (f & FLAG_BLOCK_OVERFLOW)
            return fail(h, MPM_ERR_UNSUPPORTED, std::string(where) + ": more than 1728 particles in one block");
        if (f & FLAG_OUT_OF_DOMAIN)
            return fail(h, MPM_ERR_OUT_OF_DOMAIN, std::string(where) + ": a particle stencil left [0, n_grid-1]^d");
        return fail(h, MPM_ERR_NONFINITE,
                    std::string(where) + ": non-finite value or degenerate deformation (J<=0 / r=0)");
    }
    return MPM_OK;
}

const float* alpha_at(mpm_ctx* h, int t) {
    const size_t A = h->prm.n_actuators > 0 ? h->prm.n_actuators : 1;
    return h->alpha + (size_t)t * A * (closed_loop(h) ? h->prm.n_episodes : 1);
}

// fresh binning of S_t into slot(t) (start of a forward or of a segment re-forward)
void bin_fresh(mpm_ctx* h, const KParams& k, int t) {
    const SlotView sl = slot_at(h, t);
    KScope sc(h, KC_BIN);
    h->launches += 2;
    launch_bin_keys(k, state_at(h, t).x, h->dd ? h->n0 : k.N * k.E, h->keys, h->bcount, h->flags, h->stream);
    launch_bin_scan(k, h->bcount, h->cursor, sl, h->scan_part, h->flags, h->stream);
    launch_bin_scatter(k, h->keys, state_at(h, t).pid, h->cursor, sl, h->stream);
}

// advance() for step t; write_next: produce S_{t+1}; bin_next: bin it into slot(t+1)
void step_forward(mpm_ctx* h, const KParams& k, int t, bool write_next, bool bin_next) {
    const SlotView sl = slot_at(h, t);
    const StateView S = state_at(h, t);
    const StateView Sn = write_next ? state_at(h, t + 1) : StateView{nullptr, nullptr, nullptr, nullptr};
    const int32_t* aid = h->has_aid ? h->aid : nullptr;
    const bool obs_join = k.closed_loop && h->obs_ahead == t;  // enqueued on `side` by step t - 1
    if (obs_join) h->obs_ahead = -1;
    if (k.closed_loop && !obs_join) {  // R22: alpha_t from the observation of S_t
        KScope sc(h, KC_CTRL);
        h->launches += 1;
        launch_observe(k, S.x, S.vc, S.pid, aid, h->obs_part, h->stream);
        const size_t no = (size_t)2 * k.dim * k.n_act;
        launch_ctrl_obs_fwd(k, h->theta, t, h->obs_part, h->obs + (size_t)t * k.E * no, h->obs_cnt,
                            const_cast<float*>(alpha_at(h, t)), h->stream);
    }
    if (!canon_fused(k)) {
        KScope sc(h, KC_CANON);
        launch_canon(k, sl, Sn.pid, bin_next ? h->keys : nullptr, h->flags, h->stream);
    }
    if (obs_join) cudaStreamWaitEvent(h->stream, h->ev_join, 0);  // alpha_t is ready
    { KScope sc(h, KC_P2G); launch_p2g(k, sl, S, Sn, aid, alpha_at(h, t), bin_next ? h->keys : nullptr, h->flags, h->stream); }
    { KScope sc(h, KC_GRID_OP); launch_grid_op(k, sl, h->stream); }
    if (!write_next) return;
    { KScope sc(h, KC_G2P);
      launch_g2p(k, sl, S, Sn, bin_next ? h->keys : nullptr, h->bcount, h->flags, false, Migr{}, h->stream); }
    if (bin_next && k.closed_loop && MPM_OBS_AHEAD && !h->prof.on && h->side != nullptr) {
        // the observation of S_{t+1} and the controller of step t + 1 need only S_{t+1}: they run
        // on the side stream beside the binning of S_{t+1} (and k_canon), joined before p2g(t + 1)
        cudaEventRecord(h->ev_fork, h->stream);
        cudaStreamWaitEvent(h->side, h->ev_fork, 0);
        const size_t no = (size_t)2 * k.dim * k.n_act;
        launch_observe(k, Sn.x, Sn.vc, Sn.pid, aid, h->obs_part, h->side);
        launch_ctrl_obs_fwd(k, h->theta, t + 1, h->obs_part, h->obs + (size_t)(t + 1) * k.E * no, h->obs_cnt,
                            const_cast<float*>(alpha_at(h, t + 1)), h->side);
        cudaEventRecord(h->ev_join, h->side);
        h->obs_ahead = t + 1;
        h->launches += 2;
    }
    if (bin_next) {
        const SlotView nx = slot_at(h, t + 1);
        KScope sc(h, KC_BIN);
        h->launches += 1;
        launch_bin_scan(k, h->bcount, h->cursor, nx, h->scan_part, h->flags, h->stream);
        launch_bin_scatter(k, h->keys, Sn.pid, h->cursor, nx, h->stream);
    }
}

// re-forward of step t inside a segment: the grid of step t is in the grid
// store, so only g2p runs (plus F_{t+1} = (I + dt C) F and the particle ids)
void step_reforward(mpm_ctx* h, const KParams& k, int t, cudaStream_t st) {
    KScope sc(h, KC_G2P);
    launch_g2p(k, slot_at(h, t), state_at(h, t), state_at(h, t + 1), nullptr, h->bcount, h->flags, true, Migr{}, st);
}

// advance_grad() for step t, using the grid tiles stored for step t
void step_backward(mpm_ctx* h, const KParams& k, int t, const AdjView& Sbn, const AdjView& Sb) {
    const SlotView sl = slot_at(h, t);
    const StateView S = state_at(h, t);
    const int A = k.n_act > 0 ? k.n_act : 1;
    // g2p_grad's gather part is independent of its U_bar scatter and of grid_op_grad:
    // it runs on the side stream (fork/join by events; captured into the graphs as a
    // parallel branch).  Profiling keeps everything on one stream so the per-kernel
    // CUDA-event times stay exclusive.
    const bool fork = !h->prof.on && h->side != nullptr;
    if (fork) {
        cudaEventRecord(h->ev_fork, h->stream);
        cudaStreamWaitEvent(h->side, h->ev_fork, 0);
        launch_g2p_grad_gather(k, sl, S, Sbn, h->xbar_part, h->side);
        cudaEventRecord(h->ev_join, h->side);
        h->launches += 1;
    } else {
        KScope sc(h, KC_G2P_GRAD_GATHER);
        launch_g2p_grad_gather(k, sl, S, Sbn, h->xbar_part, h->stream);
    }
    { KScope sc(h, KC_G2P_GRAD); launch_g2p_grad(k, sl, S, Sbn, h->ubar, h->stream); }
    { KScope sc(h, KC_GRID_OP_GRAD); launch_grid_op_grad(k, sl, h->ubar, h->stream); }
    if (fork) cudaStreamWaitEvent(h->stream, h->ev_join, 0);
    const bool abar_side = k.n_act > 0 && fork && !k.closed_loop && MPM_ABAR_SIDE && h->side3 != nullptr;
    float* abar_part = h->abar_part + (size_t)(t & 1) * h->abar_stride;  // double buffered by step parity
    if (h->abar_pending[t & 1]) {  // the reduction of step t + 2 still reads this buffer
        cudaStreamWaitEvent(h->stream, h->ev_abar[t & 1], 0);
        h->abar_pending[t & 1] = false;
    }
    { KScope sc(h, KC_P2G_GRAD);
      launch_p2g_grad(k, sl, S, h->has_aid ? h->aid : nullptr, alpha_at(h, t), Sbn, h->xbar_part,
                      Sb, abar_part, h->flags, h->stream); }
    if (abar_side) {
        // open loop: alpha_bar_t is read only by the controller adjoint after the whole reverse,
        // so its reduction leaves the critical path (its partials are double buffered by step
        // parity; mpm_backward joins before the controller adjoint).  Small problems run it on
        // its own stream beside the next reverse step (their next gather is on the critical
        // path); large ones ahead of the next gather on the side stream, which measured faster
        // there (C4: +2.4% vs +0.3%; C3: -3.5% vs -0.3%; C2: +2.5% vs +2.8%)
        cudaStream_t rs = canon_fused(k) ? h->side3 : h->side;
        cudaEventRecord(h->ev_p2gg, h->stream);
        cudaStreamWaitEvent(rs, h->ev_p2gg, 0);
        launch_reduce_abar(k, sl, abar_part, h->alpha_bar + (size_t)t * A, rs);
        cudaEventRecord(h->ev_abar[t & 1], rs);
        h->abar_pending[t & 1] = true;
        h->launches += 1;
    } else if (k.n_act > 0) {
        KScope sc(h, KC_REDUCE_ABAR);
        launch_reduce_abar(k, sl, abar_part, h->alpha_bar + (size_t)t * A * (k.closed_loop ? k.E : 1),
                           h->stream);
    }
    if (k.closed_loop) {  // controller adjoint of step t; observation adjoint into S_bar_t
        KScope sc(h, KC_CTRL);
        h->launches += 1;
        const size_t no = (size_t)2 * k.dim * k.n_act;
        launch_ctrl_obs_bwd(k, h->theta, t, h->obs + (size_t)t * k.E * no, alpha_at(h, t),
                            h->alpha_bar + (size_t)t * A * k.E, h->obs_cnt, h->theta_bar, h->obs_inc,
                            h->stream);
        launch_observe_adj(k, Sb, S.pid, h->has_aid ? h->aid : nullptr, h->obs_inc, h->stream);
    }
}

// Enqueue `body` through a cached CUDA graph (captured on first use).  body may update
// h->window_seg / h->sbar_cur; their values after the captured run are replayed.
mpm_status run_graphed(mpm_handle h, std::tuple<int, int, int, int> key, const std::function<void()>& body) {
    const bool graphs = h->use_graphs && !h->prof.on && h->stream != 0;
    if (!graphs) {
        body();
        return MPM_OK;
    }
    auto it = h->graphs.find(key);
    if (it == h->graphs.end()) {
        const int64_t l0 = h->launches;
        CU(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
        body();
        cudaGraph_t g = nullptr;
        CU(cudaStreamEndCapture(h->stream, &g));
        mpm_ctx::GraphRec rec;
        const cudaError_t ie = cudaGraphInstantiate(&rec.exec, g, 0);
        cudaGraphDestroy(g);
        CU(ie);
        rec.launches = h->launches - l0;
        rec.window_seg = h->window_seg;
        rec.sbar_cur = h->sbar_cur;
        h->launches = l0;
        it = h->graphs.emplace(key, rec).first;
    }
    CU(cudaGraphLaunch(it->second.exec, h->stream));
    h->launches += it->second.launches;
    h->window_seg = it->second.window_seg;
    h->sbar_cur = it->second.sbar_cur;
    return MPM_OK;
}

// COM loss of S_T in fixed block order (step T-1's blocks, partition independent: a decomposed
// body gives the same bits, f3) + the adjoint seed S_bar_T
void launch_loss_blocks(mpm_ctx* h, const KParams& k) {
    const SlotView last = slot_at(h, h->recorded - 1);
    launch_block_com(k, last, state_at(h, h->recorded).x, h->blk_part, h->stream);
    const ListSrc src{h->blk_part, h->blist_pool, last.base, last.nactive};
    const float3 tgt = make_float3(h->prm.loss_target[0], h->prm.loss_target[1], h->prm.loss_target[2]);
    float* seed = h->com_part;
    launch_loss_blocks(k, &src, 1, h->prm.loss_kind, tgt, h->loss, seed, h->sbar[0], h->flags, h->stream);
}

mpm_status copy_in(mpm_handle h, void* dst, const void* src, size_t bytes) {
    CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, h->stream));
    return MPM_OK;
}

}  // namespace eng

using namespace eng;

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
    p->deterministic = 1;
    p->loss_kind = MPM_LOSS_COM_TARGET;
    p->max_active_blocks = 0;
    p->closed_loop = 0;
    p->obs_scale_x = 10.0f;
    p->obs_scale_v = 1.0f;
    return MPM_OK;
}

mpm_status mpm_create(int64_t n_particles, int32_t n_grid, int32_t dim, float dt, float E,
                      float nu, mpm_handle* out) {
    if (!out) return MPM_ERR_INVALID_ARG;
    *out = nullptr;
    if (n_particles < 1 || n_grid < 4 || n_grid > 4096 || (dim != 2 && dim != 3) || !(dt > 0) ||
        !(E > 0) || !(nu > -1.0f && nu < 0.5f))
        return MPM_ERR_INVALID_ARG;
    if (n_particles >= ((int64_t)1 << 31)) return MPM_ERR_INVALID_ARG;
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
    if (e == cudaSuccess) e = tile_init();
    const char* ng = std::getenv("MPM_NO_GRAPHS");
    h->use_graphs = !(ng && ng[0] == '1');
    if (e != cudaSuccess) {
        delete h;
        return MPM_ERR_CUDA;
    }
    *out = h;
    return MPM_OK;
}

mpm_status mpm_destroy(mpm_handle h) {
    if (!h) return MPM_ERR_INVALID_ARG;
    DevGuard dg(h);
    if (h->h_flags) cudaFreeHost(h->h_flags);
    for (auto ev : h->prof.pool) cudaEventDestroy(ev);
    for (auto& g : h->graphs) cudaGraphExecDestroy(g.second.exec);
    if (h->side) cudaStreamDestroy(h->side);
    if (h->ev_fork) cudaEventDestroy(h->ev_fork);
    if (h->ev_join) cudaEventDestroy(h->ev_join);
    if (h->side2) cudaStreamDestroy(h->side2);
    if (h->ev_seg) cudaEventDestroy(h->ev_seg);
    if (h->ev_refwd) cudaEventDestroy(h->ev_refwd);
    if (h->side3) cudaStreamDestroy(h->side3);
    if (h->ev_p2gg) cudaEventDestroy(h->ev_p2gg);
    for (auto ev : h->ev_abar)
        if (ev) cudaEventDestroy(ev);
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
        p->n_actuators < 0 || p->n_actuators > 32 || p->ctrl_hidden < 0 || p->ctrl_hidden > 1024 ||
        p->n_sin < 1 || p->n_sin > 64 || p->act_axis < 0 || p->act_axis >= h->dim ||
        !(p->p_mass > 0) || !(p->p_vol > 0) || p->eps_mass < 0 || p->max_active_blocks < 0 ||
        (p->loss_kind != MPM_LOSS_COM_TARGET && p->loss_kind != MPM_LOSS_MOVE_FORWARD) ||
        (p->closed_loop != 0 && p->closed_loop != 1) || ctrl_inputs(*p, h->dim) > 1024)
        return fail(h, MPM_ERR_INVALID_ARG, "invalid mpm_params");
    if (p->model != MPM_MODEL_NEOHOOKEAN && p->model != MPM_MODEL_FIXED_COROTATED)
        return fail(h, MPM_ERR_INVALID_ARG, "unknown model");
    if (p->model == MPM_MODEL_FIXED_COROTATED && h->dim == 3)
        return fail(h, MPM_ERR_UNSUPPORTED, "fixed-corotated in 3D needs an SVD (out of scope, R2)");
    if ((int64_t)p->n_episodes * h->N >= ((int64_t)1 << 31))
        return fail(h, MPM_ERR_INVALID_ARG, "n_episodes * n_particles must be < 2^31");
    const int B = block_edge(h->dim);
    const int64_t nb = (h->n_grid + B - 1) / B;
    const int64_t TB = (h->dim == 2 ? nb * nb : nb * nb * nb) * p->n_episodes;
    if (TB >= ((int64_t)1 << 31)) return fail(h, MPM_ERR_INVALID_ARG, "too many grid blocks");
    h->prm = *p;
    return MPM_OK;
}

mpm_status mpm_set_stream(mpm_handle h, void* s) {
    if (!h) return MPM_ERR_INVALID_ARG;
    DevGuard dg(h);
    h->stream = (cudaStream_t)s;
    if (!h->side) {  // the side stream of the backward's parallel branch (see step_backward)
        CU(cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking));
        CU(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
        CU(cudaStreamCreateWithFlags(&h->side2, cudaStreamNonBlocking));
        CU(cudaEventCreateWithFlags(&h->ev_seg, cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&h->ev_refwd, cudaEventDisableTiming));
        CU(cudaStreamCreateWithFlags(&h->side3, cudaStreamNonBlocking));
        CU(cudaEventCreateWithFlags(&h->ev_p2gg, cudaEventDisableTiming));
        for (auto& ev : h->ev_abar) CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    }
    return MPM_OK;
}

mpm_status mpm_workspace_bytes(mpm_handle h, size_t* bytes) {
    if (!h || !bytes) return MPM_ERR_INVALID_ARG;
    DevGuard dg(h);
    *bytes = carve(h, nullptr);
    return MPM_OK;
}

mpm_status mpm_workspace_bytes_for(mpm_handle h, int32_t steps, size_t* bytes) {
    if (!h || !bytes || steps < 1) return MPM_ERR_INVALID_ARG;
    const int32_t keep = h->prm.max_steps;
    h->prm.max_steps = steps;  // size only; the handle's parameters are unchanged on return
    *bytes = carve(h, nullptr);
    h->prm.max_steps = keep;
    return MPM_OK;
}

mpm_status mpm_bind_workspace(mpm_handle h, void* dptr, size_t bytes) {
    if (!h || !dptr) return MPM_ERR_INVALID_ARG;
    DevGuard dg(h);
    if (((uintptr_t)dptr & 255) != 0) return fail(h, MPM_ERR_INVALID_ARG, "workspace not 256-B aligned");
    const size_t need = carve(h, nullptr);
    if (bytes < need)
        return fail(h, MPM_ERR_OOM, "workspace too small: need " + std::to_string(need) + " bytes");
    h->ws = (char*)dptr;
    h->ws_bytes = bytes;
    carve(h, h->ws);
    const KParams k = kparams(h);
    CU(cudaMemsetAsync(h->flags, 0, sizeof(int) * 4, h->stream));
    CU(cudaMemsetAsync(h->scan_part, 0, sizeof(int64_t) * (scan_chunks(kparams(h)) + 2), h->stream));
    CU(cudaMemsetAsync(h->bcount, 0, sizeof(int) * k.TB, h->stream));
    CU(cudaMemsetAsync(h->theta, 0, sizeof(float) * (n_theta_of(h->prm, h->dim) > 0 ? n_theta_of(h->prm, h->dim) : 1), h->stream));
    h->phase = kBound;
    return MPM_OK;
}

mpm_status mpm_set_state(mpm_handle h, const float* x, const float* v, const float* C,
                         const float* F, const int32_t* actuator_id) {
    if (!h) return MPM_ERR_INVALID_ARG;
    DevGuard dg(h);
    NvtxRange nv("mpm_set_state");
    if (h->dd) return fail(h, MPM_ERR_BAD_SEQUENCE, "a subdomain handle takes mpm_set_state_ids");
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
    { KScope sc(h, KC_LAYOUT);
      launch_pack(k, sx, v ? sv : nullptr, C ? sC : nullptr, F ? sF : nullptr, nullptr, h->ckpt[0].x,
                  h->ckpt[0].vc, h->ckpt[0].f, h->ckpt[0].pid, false, h->stream); }
    h->has_aid = actuator_id != nullptr && h->prm.n_actuators > 0;  // ids are meaningless without actuators
    if (h->has_aid && (st = copy_in(h, h->aid, actuator_id, sizeof(int32_t) * EN))) return st;
    if (h->has_aid) {  // ids outside [-1, n_actuators): MPM_ERR_INVALID_ARG at the next mpm_forward
        KScope sc(h, KC_LAYOUT);
        launch_check_aid(k, h->aid, h->flags, h->stream);
    }
    CU(cudaGetLastError());
    h->phase = kHasState;
    h->recorded = 0;
    h->t_final = 0;
    h->window_seg = -1;
    return MPM_OK;
}

mpm_status mpm_set_materials(mpm_handle h, const int32_t* material) {
    if (!h) return MPM_ERR_INVALID_ARG;
    DevGuard dg(h);
    if (h->phase < kBound) return fail(h, MPM_ERR_BAD_SEQUENCE, "set_materials before bind_workspace");
    const KParams k = kparams(h);
    const size_t EN = (size_t)k.E * k.N;
    h->has_mat = material != nullptr;
    if (h->has_mat) {  // indexed by particle id: [E][N], or [n_body] for a subdomain (f3)
        mpm_status st = copy_in(h, h->mat, material, sizeof(int32_t) * (h->dd ? (size_t)h->n_body : EN));
        if (st) return st;
    }
    // a new material layout invalidates a recorded tape
    if (h->phase > kHasState) h->phase = kHasState;
    h->recorded = 0;
    return MPM_OK;
}

mpm_status mpm_n_theta(mpm_handle h, int64_t* n) {
    if (!h || !n) return MPM_ERR_INVALID_ARG;
    *n = n_theta_of(h->prm, h->dim);
    return MPM_OK;
}

mpm_status mpm_set_controller(mpm_handle h, const float* theta, int64_t n) {
    if (!h) return MPM_ERR_INVALID_ARG;
    DevGuard dg(h);
    if (h->phase < kBound) return fail(h, MPM_ERR_BAD_SEQUENCE, "set_controller before bind_workspace");
    if (n != n_theta_of(h->prm, h->dim) || (n > 0 && !theta))
        return fail(h, MPM_ERR_INVALID_ARG, "n_theta mismatch: expected " + std::to_string(n_theta_of(h->prm, h->dim)));
    if (n > 0) return copy_in(h, h->theta, theta, sizeof(float) * n);
    return MPM_OK;
}

mpm_status mpm_forward(mpm_handle h, int32_t steps) {
    if (!h) return MPM_ERR_INVALID_ARG;
    DevGuard dg(h);
    NvtxRange nv("mpm_forward");
    if (h->dd) return fail(h, MPM_ERR_BAD_SEQUENCE, "a subdomain handle runs through mpm_dd_forward");
    if (h->phase < kHasState) return fail(h, MPM_ERR_BAD_SEQUENCE, "forward before set_state");
    if (steps < 1 || steps > h->prm.max_steps)
        return fail(h, MPM_ERR_INVALID_ARG, "steps must be in [1, max_steps]");
    const KParams k = kparams(h);
    h->t_final = steps;
    set_pdl(k.EN);
    mpm_status gs = run_graphed(h, std::make_tuple(0, steps, (int)h->has_aid + 2 * (int)h->has_mat, -1), [&]() {
        if (k.n_act > 0 && !k.closed_loop) {
            KScope sc(h, KC_CTRL);
            launch_ctrl_fwd(k, h->theta, steps, h->alpha, h->stream);
        }
        bin_fresh(h, k, 0);
        h->obs_ahead = -1;
        for (int t = 0; t < steps; ++t) step_forward(h, k, t, true, t + 1 < steps);
    });
    if (gs) return gs;
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
    DevGuard dg(h);
    NvtxRange nv("mpm_loss");
    if (h->dd) return fail(h, MPM_ERR_BAD_SEQUENCE, "a subdomain handle runs through mpm_dd_loss");
    if (h->phase < kForward) return fail(h, MPM_ERR_BAD_SEQUENCE, "loss before forward");
    const KParams k = kparams(h);
    h->sbar_cur = 0;
    { KScope sc(h, KC_LOSS);
      h->launches += 2;
      launch_loss_blocks(h, k); }
    if (loss_out) CU(cudaMemcpyAsync(loss_out, h->loss, sizeof(float) * k.E, cudaMemcpyDefault, h->stream));
    mpm_status st = sync_flags(h, "mpm_loss");
    if (st) return st;
    h->phase = kSeeded;
    return MPM_OK;
}

mpm_status mpm_seed_adjoint(mpm_handle h, const float* dx, const float* dv, const float* dC,
                            const float* dF) {
    if (!h) return MPM_ERR_INVALID_ARG;
    DevGuard dg(h);
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
    // S_bar_T is indexed like S_T: row i takes the caller's row pid_T[i]
    const StateView ST = state_at(h, h->recorded);
    { KScope sc(h, KC_LAYOUT);
      launch_pack(k, dx ? sx : nullptr, dv ? sv : nullptr, dC ? sC : nullptr, dF ? sF : nullptr, ST.pid,
                  h->sbar[0].x, h->sbar[0].vc, h->sbar[0].f, nullptr, true, h->stream); }
    CU(cudaGetLastError());
    h->sbar_cur = 0;
    h->phase = kSeeded;
    return MPM_OK;
}

mpm_status mpm_backward(mpm_handle h, int32_t steps) {
    if (!h) return MPM_ERR_INVALID_ARG;
    DevGuard dg(h);
    NvtxRange nv("mpm_backward");
    if (h->dd) return fail(h, MPM_ERR_BAD_SEQUENCE, "a subdomain handle runs through mpm_dd_backward");
    if (h->phase != kSeeded) return fail(h, MPM_ERR_BAD_SEQUENCE, "backward needs forward + loss/seed_adjoint");
    if (steps != h->recorded)
        return fail(h, MPM_ERR_BAD_SEQUENCE, "backward steps != recorded forward steps");
    const KParams k = kparams(h);
    const int kk = h->prm.k_ckpt, T = steps;
    const int A = k.n_act > 0 ? k.n_act : 1;
    set_pdl(k.EN);
    mpm_status gs = run_graphed(h, std::make_tuple(1, T, (int)h->has_aid + 2 * (int)h->has_mat, h->window_seg * 2 + h->sbar_cur), [&]() {
        if (k.n_act > 0)
            cudaMemsetAsync(h->alpha_bar, 0, sizeof(float) * (size_t)T * A * (k.closed_loop ? k.E : 1), h->stream);
        if (k.closed_loop)  // accumulated step by step (t descending) by ctrl_obs_bwd
            cudaMemsetAsync(h->theta_bar, 0, sizeof(float) * n_theta_of(h->prm, h->dim), h->stream);
        const int nseg = (T + kk - 1) / kk;
        // Segment-wise recomputation of the states.  With the side streams the
        // re-forward of segment s-1 (into window half (s-1) & 1) is enqueued on side2 as
        // soon as the reverse of segment s+1 (the last reader of that half) is done, so it
        // runs concurrently with the reverse of segment s; main waits for it before s-1.
        const bool ahead = !h->prof.on && h->side2 != nullptr;
        const int fwd_seg = h->window_seg;  // the forward left this segment in its window half
        int prefetched = -1;
        auto refwd = [&](int s, cudaStream_t st) {
            const int t0 = s * kk, t1 = (t0 + kk < T) ? t0 + kk : T;
            for (int t = t0; t < t1 - 1; ++t) step_reforward(h, k, t, st);
        };
        for (int s = nseg - 1; s >= 0; --s) {
            const int t0 = s * kk, t1 = (t0 + kk < T) ? t0 + kk : T;
            if (s != fwd_seg) {
                if (prefetched == s) cudaStreamWaitEvent(h->stream, h->ev_refwd, 0);
                else refwd(s, h->stream);
            }
            h->window_seg = s;
            if (ahead && s >= 1 && s - 1 != fwd_seg && kk > 1) {
                cudaEventRecord(h->ev_seg, h->stream);
                cudaStreamWaitEvent(h->side2, h->ev_seg, 0);
                refwd(s - 1, h->side2);
                cudaEventRecord(h->ev_refwd, h->side2);
                prefetched = s - 1;
            }
            for (int t = t1 - 1; t >= t0; --t) {
                step_backward(h, k, t, h->sbar[h->sbar_cur], h->sbar[h->sbar_cur ^ 1]);
                h->sbar_cur ^= 1;
            }
        }
        for (int b = 0; b < 2; ++b)  // actuator-gradient reductions still running on side3
            if (h->abar_pending[b]) {
                cudaStreamWaitEvent(h->stream, h->ev_abar[b], 0);
                h->abar_pending[b] = false;
            }
        const int64_t nth = n_theta_of(h->prm, h->dim);
        if (nth > 0 && !k.closed_loop) {
            KScope sc(h, KC_CTRL);
            h->launches += 1;
            launch_ctrl_bwd(k, h->theta, T, h->alpha, h->alpha_bar, h->theta_part, h->theta_bar, nth, h->stream);
        }
    });
    if (gs) return gs;
    CU(cudaGetLastError());
    mpm_status st = sync_flags(h, "mpm_backward");
    if (st) return st;
    h->phase = kBackward;
    return MPM_OK;
}

mpm_status mpm_grads(mpm_handle h, float* dx0, float* dv0, float* dC0, float* dF0, float* dtheta) {
    if (!h) return MPM_ERR_INVALID_ARG;
    DevGuard dg(h);
    NvtxRange nv("mpm_grads");
    if (h->phase != kBackward) return fail(h, MPM_ERR_BAD_SEQUENCE, "grads before backward");
    const KParams k = kparams(h);
    const size_t EN = (size_t)k.E * k.N, d = (size_t)h->dim;
    const size_t rows = h->dd ? (size_t)h->n0 : EN;  // a subdomain returns its t = 0 particles (f3)
    float* sx = h->staging;
    float* sv = sx + EN * d;
    float* sC = sv + EN * d;
    float* sF = sC + EN * d * d;
    if (dx0 || dv0 || dC0 || dF0) {
        KScope sc(h, KC_LAYOUT);
        // S_bar_0 is indexed like S_0, i.e. in caller order
        const AdjView& B0 = h->sbar[h->sbar_cur];
        launch_unpack(k, B0.x, B0.vc, B0.f, nullptr, dx0 ? sx : nullptr, dv0 ? sv : nullptr,
                      dC0 ? sC : nullptr, dF0 ? sF : nullptr, h->stream, (int64_t)rows);
    }
    if (dx0) CU(cudaMemcpyAsync(dx0, sx, sizeof(float) * rows * d, cudaMemcpyDefault, h->stream));
    if (dv0) CU(cudaMemcpyAsync(dv0, sv, sizeof(float) * rows * d, cudaMemcpyDefault, h->stream));
    if (dC0) CU(cudaMemcpyAsync(dC0, sC, sizeof(float) * rows * d * d, cudaMemcpyDefault, h->stream));
    if (dF0) CU(cudaMemcpyAsync(dF0, sF, sizeof(float) * rows * d * d, cudaMemcpyDefault, h->stream));
    const int64_t nth = n_theta_of(h->prm, h->dim);
    if (dtheta && nth > 0)
        CU(cudaMemcpyAsync(dtheta, h->theta_bar, sizeof(float) * nth, cudaMemcpyDefault, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    CU(cudaGetLastError());
    return MPM_OK;
}

mpm_status mpm_grad_v0_sum(mpm_handle h, float* out) {
    if (!h || !out) return MPM_ERR_INVALID_ARG;
    DevGuard dg(h);
    if (h->phase != kBackward) return fail(h, MPM_ERR_BAD_SEQUENCE, "grad_v0_sum before backward");
    const KParams k = kparams(h);
    float* res = h->com_part + (size_t)k.E * (loss_blocks_per_episode(k) + 1) * 3;
    { KScope sc(h, KC_LOSS);
      h->launches += 1;
      launch_v_sum(k, h->sbar[h->sbar_cur].vc, h->com_part, res, h->stream); }
    CU(cudaMemcpyAsync(out, res, sizeof(float) * k.E * h->dim, cudaMemcpyDefault, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    CU(cudaGetLastError());
    return MPM_OK;
}

mpm_status mpm_get_state(mpm_handle h, float* x, float* v, float* C, float* F) {
    if (!h) return MPM_ERR_INVALID_ARG;
    DevGuard dg(h);
    if (h->phase < kHasState) return fail(h, MPM_ERR_BAD_SEQUENCE, "get_state before set_state");
    const KParams k = kparams(h);
    const size_t EN = (size_t)k.E * k.N, d = (size_t)h->dim;
    float* sx = h->staging;
    float* sv = sx + EN * d;
    float* sC = sv + EN * d;
    float* sF = sC + EN * d * d;
    const StateView S = state_at(h, h->recorded);
    { KScope sc(h, KC_LAYOUT); launch_unpack(k, S.x, S.vc, S.f, S.pid, sx, sv, sC, sF, h->stream); }
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
    DevGuard dg(h);
    if (enable && h->prof.pool.empty()) {
        h->prof.pool.resize(2 * 65536);
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
    DevGuard dg(h);
    CU(cudaStreamSynchronize(h->stream));
    prof_harvest(h);
    for (int c = 0; c < KC_N; ++c) { h->prof.ms[c] = 0; h->prof.n[c] = 0; }
    return MPM_OK;
}

mpm_status mpm_kernel_stats(mpm_handle h, int32_t idx, const char** name, double* total_ms,
                            int64_t* count) {
    if (!h || idx < 0 || idx >= KC_N) return MPM_ERR_INVALID_ARG;
    DevGuard dg(h);
    CU(cudaStreamSynchronize(h->stream));
    prof_harvest(h);
    if (name) *name = kClassNames[idx];
    if (total_ms) *total_ms = h->prof.ms[idx];
    if (count) *count = h->prof.n[idx];
    return MPM_OK;
}

mpm_status mpm_active_nodes_at(mpm_handle h, int32_t step, int64_t* count) {
    if (!h || !count) return MPM_ERR_INVALID_ARG;
    DevGuard dg(h);
    if (h->phase < kForward) return fail(h, MPM_ERR_BAD_SEQUENCE, "active_nodes before forward");
    if (step < 0 || step >= h->recorded) return fail(h, MPM_ERR_INVALID_ARG, "step outside the recorded forward");
    const KParams k = kparams(h);
    // the grid store keeps the binning and resolved node tiles of every recorded step
    { KScope sc(h, KC_LAYOUT); launch_count_active(k, slot_at(h, step), h->counter, h->stream); }
    int64_t c = 0;
    CU(cudaMemcpyAsync(&c, h->counter, sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    *count = c;
    return MPM_OK;
}

mpm_status mpm_active_nodes(mpm_handle h, int64_t* count) {
    if (!h || !count) return MPM_ERR_INVALID_ARG;
    if (h->phase < kForward) return fail(h, MPM_ERR_BAD_SEQUENCE, "active_nodes before forward");
    return mpm_active_nodes_at(h, h->recorded - 1, count);
}

mpm_status mpm_launch_count(mpm_handle h, int64_t* count) {
    if (!h || !count) return MPM_ERR_INVALID_ARG;
    *count = h->launches;
    return MPM_OK;
}

}  // extern "C"
