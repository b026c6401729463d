// engine_dd.cu -- SURVEY.md 8(f) row f3: one body decomposed into slab subdomains along x.
//
// The paper runs one body per GPU (section 4.1); f3 lets a body exceed one
// GPU.  Subdomain g owns the grid blocks with block x-index in [x_lo_g, x_hi_g) and, at each
// step t, the particles binned into those blocks.  Per step:
//   forward   canon + p2g (local) -> grid_op: a node near a slab face sums the partial tiles of the
//             neighbour's face column, read from the neighbour's memory (same device, or NVLink
//             peer memory) in the single-domain order -> g2p (local; particles whose next block
//             leaves the slab go to a per-step outbox) -> immigrate: each subdomain appends its
//             neighbours' emigrants to S_{t+1} (peer loads) -> binning of t+1 (local);
//   backward  pull the adjoint rows of this subdomain's emigrants from the neighbour that
//             processed them at t+1 -> g2p_grad (local) -> grid_op_grad (U_bar partial tiles of
//             the neighbour's face column by peer loads) -> p2g_grad (local).
// Every per-block computation sees the same particles in the same canonical (cell, particle id)
// order and every covered sum the same tiles in the same order as a single-domain run, and the
// loss is reduced in global block order (kernels.h launch_loss_blocks), so the decomposed run is
// bitwise equal to the single-domain one (tests/test_gpu_dd.py).
// Scope: passive bodies (solid / fluid), one episode, checkpoint interval 1 (every state kept:
// splitting the body is what makes the whole tape fit); the subdomains' work is enqueued eagerly
// on their streams, ordered by events (no CUDA graphs).
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "engine.h"

using namespace mpm;
using namespace eng;

namespace {

enum DdEv { EV_P2G = 0, EV_GRID, EV_G2P, EV_AUX };

mpm_status check_set(mpm_handle* hs, int32_t n) {
    if (!hs || n < 1 || n > 4) return MPM_ERR_INVALID_ARG;
    for (int g = 0; g < n; ++g) {
        if (!hs[g]) return MPM_ERR_INVALID_ARG;
        if (!hs[g]->dd) return fail(hs[g], MPM_ERR_BAD_SEQUENCE, "handle is not a subdomain (mpm_set_subdomain)");
        if (hs[g]->nbr[0] != (g > 0 ? hs[g - 1] : nullptr) || hs[g]->nbr[1] != (g + 1 < n ? hs[g + 1] : nullptr))
            return fail(hs[g], MPM_ERR_BAD_SEQUENCE, "subdomains not linked in this order (mpm_dd_link)");
    }
    return MPM_OK;
}

// the neighbours' grid data of step t for the covered sums (grid_op: partial tiles; backward:
// U_bar partial tiles)
SlotView halo_slot(mpm_ctx* h, int t, bool backward) {
    SlotView sl = slot_at(h, t);
    const KParams k = kparams(h);
    for (int s = 0; s < 2; ++s) {
        mpm_ctx* nb = h->nbr[s];
        if (!nb) continue;
        sl.halo.bmap[s] = nb->bmap_store + (size_t)k.TB * t;
        sl.halo.tiles[s] = backward ? nb->ubar : nb->part;
        sl.halo.base[s] = nb->base_arr + t;
    }
    return sl;
}

void wait_nbrs(mpm_ctx* h, int ev) {
    for (int s = 0; s < 2; ++s)
        if (h->nbr[s]) cudaStreamWaitEvent(h->stream, h->nbr[s]->dd_ev[ev], 0);
}

Migr migr_of(mpm_ctx* h, int t) {
    Migr m;
    m.x_lo = h->x_lo;
    m.x_hi = h->x_hi;
    m.cnt = h->out_cnt + (size_t)2 * t;
    m.rows = h->out_rows + (size_t)2 * h->mig_cap * t;
    m.cap = h->mig_cap;
    return m;
}

mpm_status sync_all(mpm_handle* hs, int32_t n, const char* where) {
    for (int g = 0; g < n; ++g) {
        DevGuard dg(hs[g]);
        mpm_status st = sync_flags(hs[g], where);
        if (st) return st;
    }
    return MPM_OK;
}

}  // namespace

extern "C" {

mpm_status mpm_set_subdomain(mpm_handle h, int32_t x_lo, int32_t x_hi, int64_t n_body, int32_t migrate_cap) {
    if (!h) return MPM_ERR_INVALID_ARG;
    if (h->phase >= kBound) return fail(h, MPM_ERR_BAD_SEQUENCE, "set_subdomain after bind_workspace");
    const int B = block_edge(h->dim);
    const int nb = (h->n_grid + B - 1) / B;
    if (x_lo < 0 || x_hi <= x_lo || x_hi > nb || n_body < 1 || n_body >= ((int64_t)1 << 31) || migrate_cap < 0)
        return fail(h, MPM_ERR_INVALID_ARG, "invalid subdomain (block x-range, body size or migration capacity)");
    h->dd = true;
    h->x_lo = x_lo;
    h->x_hi = x_hi;
    h->n_body = n_body;
    h->mig_cap = migrate_cap > 0 ? migrate_cap : (int)std::min<int64_t>(h->N, h->N / 8 + 1024);
    return MPM_OK;
}

mpm_status mpm_dd_link(mpm_handle* hs, int32_t n) {
    if (!hs || n < 1 || n > 4) return MPM_ERR_INVALID_ARG;
    for (int g = 0; g < n; ++g) {
        mpm_ctx* h = hs[g];
        if (!h) return MPM_ERR_INVALID_ARG;
        if (!h->dd) return fail(h, MPM_ERR_BAD_SEQUENCE, "handle is not a subdomain (mpm_set_subdomain)");
        if (h->phase < kBound) return fail(h, MPM_ERR_BAD_SEQUENCE, "dd_link before bind_workspace");
        const mpm_params& p = h->prm;
        if (p.n_episodes != 1 || p.n_actuators != 0 || p.closed_loop != 0 || p.k_ckpt != 1)
            return fail(h, MPM_ERR_UNSUPPORTED,
                        "a decomposed body (f3) needs n_episodes = 1, a passive body (n_actuators = 0) and "
                        "k_ckpt = 1");
        const mpm_ctx* h0 = hs[0];
        if (h->dim != h0->dim || h->n_grid != h0->n_grid || h->dt != h0->dt || h->E != h0->E || h->nu != h0->nu ||
            h->n_body != h0->n_body || std::memcmp(&h->prm, &h0->prm, sizeof(mpm_params)) != 0)
            return fail(h, MPM_ERR_INVALID_ARG, "subdomains of one body must share every parameter");
        const int B = block_edge(h->dim);
        const int nb = (h->n_grid + B - 1) / B;
        if ((g == 0 && h->x_lo != 0) || (g == n - 1 && h->x_hi != nb) || (g > 0 && h->x_lo != hs[g - 1]->x_hi))
            return fail(h, MPM_ERR_INVALID_ARG, "slabs must be contiguous, in order, and cover the grid");
        h->nbr[0] = g > 0 ? hs[g - 1] : nullptr;
        h->nbr[1] = g + 1 < n ? hs[g + 1] : nullptr;
        DevGuard dg(h);
        for (int s = 0; s < 2; ++s) {  // peer access to a neighbour on another device (NVLink)
            const mpm_ctx* nbh = h->nbr[s];
            if (!nbh || nbh->device == h->device) continue;
            int ok = 0;
            CU(cudaDeviceCanAccessPeer(&ok, h->device, nbh->device));
            if (!ok) return fail(h, MPM_ERR_UNSUPPORTED, "no peer access between the subdomains' devices");
            const cudaError_t e = cudaDeviceEnablePeerAccess(nbh->device, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CU(e);
            cudaGetLastError();
        }
        for (int q = 0; q < 4; ++q)
            if (!h->dd_ev[q]) CU(cudaEventCreateWithFlags(&h->dd_ev[q], cudaEventDisableTiming));
    }
    return MPM_OK;
}

mpm_status mpm_set_state_ids(mpm_handle h, int64_t n, const float* x, const float* v, const float* C,
                             const float* F, const int32_t* ids) {
    if (!h) return MPM_ERR_INVALID_ARG;
    DevGuard dg(h);
    if (!h->dd) return fail(h, MPM_ERR_BAD_SEQUENCE, "set_state_ids needs a subdomain (mpm_set_subdomain)");
    if (h->phase < kBound) return fail(h, MPM_ERR_BAD_SEQUENCE, "set_state_ids before bind_workspace");
    if (n < 0 || n > h->N || (n > 0 && (!x || !ids)))
        return fail(h, MPM_ERR_INVALID_ARG, "0 <= n <= capacity; x and ids are required");
    const KParams k = kparams(h);
    const size_t d = (size_t)h->dim;
    float* sx = h->staging;
    float* sv = sx + (size_t)k.N * d;
    float* sC = sv + (size_t)k.N * d;
    float* sF = sC + (size_t)k.N * d * d;
    mpm_status st;
    if (n > 0) {
        if ((st = copy_in(h, sx, x, sizeof(float) * n * d))) return st;
        if (v && (st = copy_in(h, sv, v, sizeof(float) * n * d))) return st;
        if (C && (st = copy_in(h, sC, C, sizeof(float) * n * d * d))) return st;
        if (F && (st = copy_in(h, sF, F, sizeof(float) * n * d * d))) return st;
    }
    KParams kn = k;  // pack the n given rows
    kn.N = n;
    kn.EN = k.EN;
    if (n > 0) {
        KScope sc(h, KC_LAYOUT);
        launch_pack(kn, sx, v ? sv : nullptr, C ? sC : nullptr, F ? sF : nullptr, nullptr, h->ckpt[0].x,
                    h->ckpt[0].vc, h->ckpt[0].f, nullptr, false, h->stream);
        CU(cudaMemcpyAsync(h->ckpt[0].pid, ids, sizeof(int32_t) * n, cudaMemcpyDefault, h->stream));
    }
    CU(cudaGetLastError());
    h->n0 = n;
    h->has_aid = false;
    h->phase = kHasState;
    h->recorded = 0;
    h->t_final = 0;
    h->window_seg = -1;
    return MPM_OK;
}

mpm_status mpm_dd_forward(mpm_handle* hs, int32_t n, int32_t steps) {
    NvtxRange nv("mpm_dd_forward");
    mpm_status st = check_set(hs, n);
    if (st) return st;
    for (int g = 0; g < n; ++g) {
        if (hs[g]->phase < kHasState) return fail(hs[g], MPM_ERR_BAD_SEQUENCE, "dd_forward before set_state_ids");
        if (steps < 1 || steps > hs[g]->prm.max_steps)
            return fail(hs[g], MPM_ERR_INVALID_ARG, "steps must be in [1, max_steps]");
    }
    std::vector<KParams> K(n);
    for (int g = 0; g < n; ++g) {
        mpm_ctx* h = hs[g];
        DevGuard dg(h);
        K[g] = kparams(h);
        h->t_final = steps;
        set_pdl(K[g].EN);
        CU(cudaMemsetAsync(h->out_cnt, 0, sizeof(int) * 2 * ((size_t)steps + 1), h->stream));
        KScope sc(h, KC_BIN);
        h->launches += 2;
        launch_bin_keys(K[g], state_at(h, 0).x, h->n0, h->keys, h->bcount, h->flags, h->stream);
        launch_bin_scan(K[g], h->bcount, h->cursor, slot_at(h, 0), h->scan_part, h->flags, h->stream);
        launch_bin_scatter(K[g], h->keys, state_at(h, 0).pid, h->cursor, slot_at(h, 0), h->stream);
    }
    for (int t = 0; t < steps; ++t) {
        const bool last = t + 1 == steps;
        for (int g = 0; g < n; ++g) {  // canon + p2g (local)
            mpm_ctx* h = hs[g];
            DevGuard dg(h);
            const SlotView sl = slot_at(h, t);
            const StateView S = state_at(h, t), Sn = state_at(h, t + 1);
            if (!canon_fused(K[g])) {
                KScope sc(h, KC_CANON);
                launch_canon(K[g], sl, Sn.pid, last ? nullptr : h->keys, h->flags, h->stream);
            }
            { KScope sc(h, KC_P2G); launch_p2g(K[g], sl, S, Sn, nullptr, nullptr, last ? nullptr : h->keys, h->flags, h->stream); }
            CU(cudaEventRecord(h->dd_ev[EV_P2G], h->stream));
        }
        for (int g = 0; g < n; ++g) {  // grid_op over the slab faces
            mpm_ctx* h = hs[g];
            DevGuard dg(h);
            wait_nbrs(h, EV_P2G);
            { KScope sc(h, KC_GRID_OP); launch_grid_op(K[g], halo_slot(h, t, false), h->stream); }
            CU(cudaEventRecord(h->dd_ev[EV_GRID], h->stream));
        }
        for (int g = 0; g < n; ++g) {  // g2p (local), emigrants into the step's outbox
            mpm_ctx* h = hs[g];
            DevGuard dg(h);
            if (!last) CU(cudaMemsetAsync(h->keys, 0xff, sizeof(int) * (size_t)K[g].EN, h->stream));
            { KScope sc(h, KC_G2P);
              launch_g2p(K[g], slot_at(h, t), state_at(h, t), state_at(h, t + 1), last ? nullptr : h->keys, h->bcount,
                         h->flags, false, last ? Migr{} : migr_of(h, t), h->stream); }
            CU(cudaEventRecord(h->dd_ev[EV_G2P], h->stream));
        }
        if (last) break;
        for (int g = 0; g < n; ++g) {  // immigrants (peer loads) + binning of t + 1
            mpm_ctx* h = hs[g];
            DevGuard dg(h);
            wait_nbrs(h, EV_G2P);  // their outboxes and S_{t+1}; they also finished reading our tiles
            MigSrc src[2];
            for (int s = 0; s < 2; ++s) {
                mpm_ctx* nb = h->nbr[s];
                src[s] = MigSrc{StateView{nullptr, nullptr, nullptr, nullptr}, nullptr, nullptr, 0};
                if (!nb) continue;
                src[s].S = state_at(nb, t + 1);
                src[s].cap = nb->mig_cap;
                src[s].cnt = nb->out_cnt + (size_t)2 * t + (s == 0 ? 1 : 0);  // toward us
                src[s].rows = nb->out_rows + (size_t)2 * nb->mig_cap * t;
            }
            KScope sc(h, KC_BIN);
            h->launches += 2;
            launch_immigrate(K[g], state_at(h, t + 1), h->ntot_arr + t, src[0], src[1], h->x_lo, h->x_hi, h->mig_cap,
                             h->keys, h->bcount, h->imm_base + (size_t)2 * (t + 1), h->nrows_arr + t + 1, h->flags,
                             h->stream);
            const SlotView nx = slot_at(h, t + 1);
            launch_bin_scan(K[g], h->bcount, h->cursor, nx, h->scan_part, h->flags, h->stream);
            launch_bin_scatter(K[g], h->keys, state_at(h, t + 1).pid, h->cursor, nx, h->stream);
        }
    }
    for (int g = 0; g < n; ++g) {
        mpm_ctx* h = hs[g];
        DevGuard dg(h);
        CU(cudaGetLastError());
        h->recorded = steps;
        h->window_seg = steps - 1;
        h->phase = kForward;
    }
    st = sync_all(hs, n, "mpm_dd_forward");
    if (st)
        for (int g = 0; g < n; ++g) hs[g]->phase = kHasState;
    return st;
}

mpm_status mpm_dd_loss(mpm_handle* hs, int32_t n, float* loss_out) {
    NvtxRange nv("mpm_dd_loss");
    mpm_status st = check_set(hs, n);
    if (st) return st;
    for (int g = 0; g < n; ++g)
        if (hs[g]->phase < kForward || hs[g]->recorded != hs[0]->recorded)
            return fail(hs[g], MPM_ERR_BAD_SEQUENCE, "dd_loss before dd_forward");
    const int T = hs[0]->recorded;
    for (int g = 0; g < n; ++g) {  // per-block partial sums of x_T (each subdomain's blocks of T-1)
        mpm_ctx* h = hs[g];
        DevGuard dg(h);
        KScope sc(h, KC_LOSS);
        launch_block_com(kparams(h), slot_at(h, T - 1), state_at(h, T).x, h->blk_part, h->stream);
        CU(cudaEventRecord(h->dd_ev[EV_AUX], h->stream));
    }
    std::vector<ListSrc> src(n);
    for (int g = 0; g < n; ++g) {
        const SlotView last = slot_at(hs[g], T - 1);
        src[g] = ListSrc{hs[g]->blk_part, hs[g]->blist_pool, last.base, last.nactive};
    }
    for (int g = 0; g < n; ++g) {  // every subdomain reduces the same lists in the same order
        mpm_ctx* h = hs[g];
        DevGuard dg(h);
        for (int q = 0; q < n; ++q)
            if (q != g) CU(cudaStreamWaitEvent(h->stream, hs[q]->dd_ev[EV_AUX], 0));
        const float3 tgt = make_float3(h->prm.loss_target[0], h->prm.loss_target[1], h->prm.loss_target[2]);
        KScope sc(h, KC_LOSS);
        h->launches += 1;
        launch_loss_blocks(kparams(h), src.data(), n, h->prm.loss_kind, tgt, h->loss, h->com_part, h->sbar[0],
                           h->flags, h->stream);
        h->sbar_cur = 0;
    }
    if (loss_out) {
        DevGuard dg(hs[0]);
        mpm_ctx* h = hs[0];
        CU(cudaMemcpyAsync(loss_out, h->loss, sizeof(float), cudaMemcpyDefault, h->stream));
    }
    st = sync_all(hs, n, "mpm_dd_loss");
    if (st) return st;
    for (int g = 0; g < n; ++g) hs[g]->phase = kSeeded;
    return MPM_OK;
}

mpm_status mpm_dd_backward(mpm_handle* hs, int32_t n, int32_t steps) {
    NvtxRange nv("mpm_dd_backward");
    mpm_status st = check_set(hs, n);
    if (st) return st;
    for (int g = 0; g < n; ++g) {
        if (hs[g]->phase != kSeeded) return fail(hs[g], MPM_ERR_BAD_SEQUENCE, "dd_backward needs dd_forward + dd_loss");
        if (steps != hs[g]->recorded) return fail(hs[g], MPM_ERR_BAD_SEQUENCE, "backward steps != recorded steps");
    }
    std::vector<KParams> K(n);
    for (int g = 0; g < n; ++g) {
        DevGuard dg(hs[g]);
        K[g] = kparams(hs[g]);
        set_pdl(K[g].EN);
    }
    for (int t = steps - 1; t >= 0; --t) {
        for (int g = 0; g < n; ++g) {  // adjoint of the migration + g2p_grad (local)
            mpm_ctx* h = hs[g];
            DevGuard dg(h);
            const int cur = h->sbar_cur;
            const AdjView Sbn = h->sbar[cur];
            // the neighbours finished step t+1: their S_bar_{t+1} rows exist, and they are done
            // reading our U_bar tiles and our S_bar_{t+2} rows (about to be overwritten)
            if (t + 1 < steps) {
                wait_nbrs(h, EV_G2P);
                const mpm_ctx* L = h->nbr[0];
                const mpm_ctx* R = h->nbr[1];
                KScope sc(h, KC_LAYOUT);
                launch_adj_pull(K[g], Sbn, h->out_cnt + (size_t)2 * t, h->out_rows + (size_t)2 * h->mig_cap * t,
                                h->mig_cap, L ? L->sbar[cur] : AdjView{nullptr, nullptr, nullptr},
                                L ? L->imm_base + (size_t)2 * (t + 1) : nullptr,
                                R ? R->sbar[cur] : AdjView{nullptr, nullptr, nullptr},
                                R ? R->imm_base + (size_t)2 * (t + 1) : nullptr, h->stream);
            }
            const SlotView sl = slot_at(h, t);
            const StateView S = state_at(h, t);
            { KScope sc(h, KC_G2P_GRAD_GATHER); launch_g2p_grad_gather(K[g], sl, S, Sbn, h->xbar_part, h->stream); }
            { KScope sc(h, KC_G2P_GRAD); launch_g2p_grad(K[g], sl, S, Sbn, h->ubar, h->stream); }
            CU(cudaEventRecord(h->dd_ev[EV_P2G], h->stream));
        }
        for (int g = 0; g < n; ++g) {  // grid_op_grad over the slab faces, p2g_grad (local)
            mpm_ctx* h = hs[g];
            DevGuard dg(h);
            wait_nbrs(h, EV_P2G);
            { KScope sc(h, KC_GRID_OP_GRAD); launch_grid_op_grad(K[g], halo_slot(h, t, true), h->ubar, h->stream); }
            CU(cudaEventRecord(h->dd_ev[EV_GRID], h->stream));
            const int cur = h->sbar_cur;
            { KScope sc(h, KC_P2G_GRAD);
              launch_p2g_grad(K[g], slot_at(h, t), state_at(h, t), nullptr, nullptr, h->sbar[cur], h->xbar_part,
                              h->sbar[cur ^ 1], h->abar_part, h->flags, h->stream); }
        }
        for (int g = 0; g < n; ++g) {
            mpm_ctx* h = hs[g];
            DevGuard dg(h);
            // our neighbours' grid_op_grad read our U_bar tiles: done before our next g2p_grad
            wait_nbrs(h, EV_GRID);
            CU(cudaEventRecord(h->dd_ev[EV_G2P], h->stream));  // "step t finished" for the neighbours
            h->sbar_cur ^= 1;
        }
    }
    for (int g = 0; g < n; ++g) {
        mpm_ctx* h = hs[g];
        DevGuard dg(h);
        CU(cudaGetLastError());
    }
    st = sync_all(hs, n, "mpm_dd_backward");
    if (st) return st;
    for (int g = 0; g < n; ++g) hs[g]->phase = kBackward;
    return MPM_OK;
}

mpm_status mpm_dd_rows(mpm_handle h, int64_t* rows) {
    if (!h || !rows) return MPM_ERR_INVALID_ARG;
    DevGuard dg(h);
    if (!h->dd || h->phase < kForward) return fail(h, MPM_ERR_BAD_SEQUENCE, "dd_rows needs a recorded dd_forward");
    int v = 0;
    CU(cudaMemcpyAsync(&v, h->ntot_arr + h->recorded - 1, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    *rows = v;
    return MPM_OK;
}

mpm_status mpm_get_state_ids(mpm_handle h, float* x, float* v, float* C, float* F, int32_t* ids) {
    int64_t rows = 0;
    mpm_status st = mpm_dd_rows(h, &rows);
    if (st) return st;
    DevGuard dg(h);
    const KParams k = kparams(h);
    const size_t d = (size_t)h->dim;
    float* sx = h->staging;
    float* sv = sx + (size_t)k.N * d;
    float* sC = sv + (size_t)k.N * d;
    float* sF = sC + (size_t)k.N * d * d;
    const StateView S = state_at(h, h->recorded);
    { KScope sc(h, KC_LAYOUT);
      launch_unpack(k, S.x, S.vc, S.f, nullptr, sx, sv, sC, sF, h->stream, rows); }
    if (x) CU(cudaMemcpyAsync(x, sx, sizeof(float) * rows * d, cudaMemcpyDefault, h->stream));
    if (v) CU(cudaMemcpyAsync(v, sv, sizeof(float) * rows * d, cudaMemcpyDefault, h->stream));
    if (C) CU(cudaMemcpyAsync(C, sC, sizeof(float) * rows * d * d, cudaMemcpyDefault, h->stream));
    if (F) CU(cudaMemcpyAsync(F, sF, sizeof(float) * rows * d * d, cudaMemcpyDefault, h->stream));
    if (ids) CU(cudaMemcpyAsync(ids, S.pid, sizeof(int32_t) * rows, cudaMemcpyDefault, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    CU(cudaGetLastError());
    return MPM_OK;
}

}  // extern "C"
