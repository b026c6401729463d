// kernels.h -- host-side launchers of the sm_100a kernels (internal to libmpm_b200.so).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "mpm_device.cuh"

namespace mpm {

// ---- one forward step (advance()) ------------------------
// p2g: clear_grid must precede (grid zeroed by the caller).  Writes F_{t+1} into
// S_next's F slot when S_next != nullptr.
void launch_p2g(const KParams& p, const float* S, const int32_t* aid, const float* alpha_t,
                float4* grid, float* S_next, int* flags, cudaStream_t s);
void launch_grid_op(const KParams& p, const float4* grid, float4* U, cudaStream_t s);
void launch_g2p(const KParams& p, const float* S, const float4* U, float* S_next, int* flags,
                cudaStream_t s);

// ---- one reverse step (advance_grad()) ----------------------------
void launch_g2p_grad(const KParams& p, const float* S, const float4* U, const float* Sb_next,
                     float4* Ubar, float* Sb, cudaStream_t s);
void launch_grid_op_grad(const KParams& p, const float4* grid, const float4* U, const float4* Ubar,
                         float4* gbar, cudaStream_t s);
// writes per-block actuation-gradient partials to abar_part[nblocks][n_act]
void launch_p2g_grad(const KParams& p, const float* S, const int32_t* aid, const float* alpha_t,
                     const float4* gbar, const float* Sb_next, float* Sb, float* abar_part,
                     int* flags, cudaStream_t s);
int p2g_grad_blocks(const KParams& p);
// alpha_bar_t[a] = sum over blocks (fixed order) of abar_part[b][a]
void launch_reduce_abar(const KParams& p, const float* abar_part, int nblocks, float* alpha_bar_t,
                        cudaStream_t s);

// ---- controller (compute_actuation, P:577 / .grad P:591) ---------------------
void launch_ctrl_fwd(const KParams& p, const float* theta, int32_t T, float* alpha, cudaStream_t s);
// per-step parameter-gradient partials, then a fixed-order sum over steps
void launch_ctrl_bwd(const KParams& p, const float* theta, int32_t T, const float* alpha,
                     const float* alpha_bar, float* theta_part, float* theta_bar, int64_t n_theta,
                     cudaStream_t s);

// ---- loss on S_T and the adjoint seed ----------------------------------------
int loss_blocks_per_episode(const KParams& p);
void launch_loss(const KParams& p, const float* S, int loss_kind, float3 target, float* com_part,
                 float* loss, float* Sb, int* flags, cudaStream_t s);

// ---- per-episode sum of the v-adjoint of the records: out[E][d] (fixed order)
void launch_v_sum(const KParams& p, const float* Sb, float* part, float* out, cudaStream_t s);

// ---- measurement: number of grid nodes with M > 0 (all episodes) -> *count (device)
void launch_count_active(const KParams& p, const float4* grid, int64_t* count, cudaStream_t s);

// ---- layout conversion (caller arrays <-> particle records) ------------------
// pack: records[E*N][R] from x[E*N][d], v, C[E*N][d][d], F (any may be null -> zero / identity)
void launch_pack(const KParams& p, const float* x, const float* v, const float* C, const float* F,
                 float* rec, cudaStream_t s);
void launch_unpack(const KParams& p, const float* rec, float* x, float* v, float* C, float* F,
                   cudaStream_t s);

}  // namespace mpm
