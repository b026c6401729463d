/*
 * mpm.h -- C-ABI of the B200-native differentiable MLS-MPM hot path.
 *
 * What it computes (PAPER.md, "P:n" = line n):
 *   - diffmpm, the differentiable elastic-object simulator (section 4.1):
 *     MLS-MPM after ChainQueen; the equations used are DESIGN.md readings R1-R25.
 *   - One time step = advance() of Appendix D.1:
 *     clear_grid -> compute_actuation -> p2g -> grid_op -> g2p.
 *   - Its reverse = advance_grad(): recompute the grid, then
 *     g2p.grad -> grid_op.grad -> p2g.grad -> compute_actuation.grad.
 *   - The tape replays advance_grad in reverse over all recorded steps,
 *     with segment-wise recomputation every k steps (Appendix D.2).
 *   - mpm_loss + mpm_backward follow ti.Tape(loss): the loss adjoint
 *     is seeded with 1 and gradients are taken w.r.t. the global tensors
 *     (initial state and controller weights), not kernel scalars.
 *
 * Conventions
 *   - Every function returns mpm_status (0 = MPM_OK).  On error,
 *     mpm_last_error(h) holds a one-line message.  Out-of-bounds is a hard
 *     error, never a silent wrap or clamp; non-finite results are errors.
 *   - Opaque handle; calls on one handle are NOT thread-safe; separate handles
 *     are independent.  A handle belongs to the device current at mpm_create;
 *     every entry point makes that device current and restores the caller's.
 *   - Memory: the library never allocates device memory.  The caller (PyTorch)
 *     allocates one workspace of mpm_workspace_bytes() and binds it; every
 *     library buffer (states, checkpoints, grids, adjoints) lives inside it.
 *     Caller buffers passed to any call are never retained.
 *   - Pointers marked "host or device" may point to either (unified
 *     addressing; copies use cudaMemcpyDefault).  Pageable host memory works
 *     but serialises the copy.
 *   - Asynchrony: work is enqueued on the bound stream.  mpm_forward,
 *     mpm_backward, mpm_loss, mpm_get_state and mpm_grads synchronise the
 *     stream before returning and report device-side error flags
 *     (out-of-domain, non-finite) raised by any earlier enqueued kernel.
 *   - Call sequence: create -> [set_params] -> bind_workspace -> set_state ->
 *     [set_controller] -> forward(T) -> loss | seed_adjoint -> backward(T) ->
 *     grads.  Anything else returns MPM_ERR_BAD_SEQUENCE.
 *   - Layouts (row-major, caller particle order, E = n_episodes):
 *     x, v: [E][N][d];  C, F: [E][N][d][d];  actuator_id: [E][N] (-1 passive);
 *     theta: [n_theta] (see mpm_params.ctrl_hidden); loss: [E].
 */
#ifndef MPM_B200_H
#define MPM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mpm_ctx* mpm_handle;

typedef enum {
    MPM_OK = 0,
    MPM_ERR_INVALID_ARG = 1,
    MPM_ERR_OOM = 2,             /* workspace too small */
    MPM_ERR_CUDA = 3,            /* a CUDA runtime error (message in mpm_last_error) */
    MPM_ERR_OUT_OF_DOMAIN = 4,   /* a particle's 3^d stencil left [0, n_grid-1]^d (R13) */
    MPM_ERR_NONFINITE = 5,       /* NaN/Inf, J <= 0 under Neo-Hookean, r = 0 in the 2x2 polar (R14) */
    MPM_ERR_BAD_SEQUENCE = 6,    /* e.g. backward before forward/loss, steps != recorded */
    MPM_ERR_UNSUPPORTED = 7      /* fixed-corotated in 3D (needs an SVD, out of scope), or more
                                    than 1728 particles in one block (27 per cell on average) */
} mpm_status;

enum { MPM_MODEL_NEOHOOKEAN = 0, MPM_MODEL_FIXED_COROTATED = 1 };
enum { MPM_LOSS_COM_TARGET = 0,     /* L_e = |xbar_T - target|^2 (R10) */
       MPM_LOSS_MOVE_FORWARD = 1 }; /* L_e = -xbar_T . e_0 ("move forward") */

/* Simulation parameters beyond mpm_create's (defaults: mpm_default_params). */
typedef struct {
    float gravity;        /* g along -y (axis 1); default 3.8 (2D) / 10 (3D)  (R7) */
    float p_mass;         /* particle mass m, default 1  (R4) */
    float p_vol;          /* particle volume V, default 1  (R4) */
    float eps_mass;       /* empty-node guard eps in P/(M + eps), default 1e-10 (R5) */
    int32_t bound;        /* sticky-wall thickness beta in nodes, default 3 (R6) */
    int32_t model;        /* MPM_MODEL_*; default NH in 3D, FCR in 2D (R2) */
    int32_t k_ckpt;       /* checkpoint every k steps (Appendix D.2), default 1 */
    int32_t max_steps;    /* tape capacity T_max (sizes the workspace), default 2048 */
    int32_t n_actuators;  /* controller outputs; 0 = passive body */
    float act_strength;   /* kappa in tau += kappa a (F e)(F e)^T, default 4 (R8) */
    int32_t act_axis;     /* e = e_{act_axis}, default 1 */
    int32_t n_sin;        /* sinusoid features phi_j(t), default 4 (R9) */
    float omega;          /* feature frequency, default 20 */
    int32_t ctrl_hidden;  /* H: 0 = tanh(W phi + b); H > 0 = 2-layer tanh MLP (R9) */
    int32_t n_episodes;   /* E independent episodes sharing theta, default 1 */
    int32_t deterministic;/* accepted for compatibility: every reduction already has a fixed
                             order, so results are bitwise reproducible run to run */
    int32_t loss_kind;    /* MPM_LOSS_* */
    float loss_target[3]; /* x* for MPM_LOSS_COM_TARGET */
    int32_t max_active_blocks; /* capacity of one step's active block list (blocks of
                                  4^3 cells in 3D, 8^2 in 2D); 0 = automatic.  Exceeding it
                                  returns MPM_ERR_OOM. */
    int64_t grid_store_blocks; /* capacity of the grid store that keeps every step's node tiles
                                  for the reverse pass (blocks summed over all steps);
                                  0 = automatic (about 3x a dense body).  MPM_ERR_OOM if exceeded. */
    int32_t closed_loop;  /* 0 = open-loop controller on the sinusoid features (R9);
                             1 = closed loop (R22): the controller input
                             is [phi(t), o_t] with, per actuator group a of each episode,
                             o_t[a] = (s_x (mean_a x_t - mean x_t), s_v mean_a v_t); n_theta grows
                             accordingly and alpha_t differs per episode.  Default 0. */
    float obs_scale_x;    /* s_x, default 10 */
    float obs_scale_v;    /* s_v, default 1 */
} mpm_params;

/* Create a handle for n_particles per episode on an n_grid^dim grid over the
 * domain [0,1]^dim (dx = 1/n_grid), time step dt, Young's modulus E and
 * Poisson ratio nu (mu = E/(2(1+nu)), lambda = E nu/((1+nu)(1-2nu)), R3).
 * Uses the current CUDA device.  No device memory is allocated. */
mpm_status mpm_create(int64_t n_particles, int32_t n_grid, int32_t dim, float dt, float E,
                      float nu, mpm_handle* out);
mpm_status mpm_destroy(mpm_handle h);
const char* mpm_last_error(mpm_handle h);

/* Fill p with the defaults for dimension dim. */
mpm_status mpm_default_params(int32_t dim, mpm_params* p);
mpm_status mpm_get_params(mpm_handle h, mpm_params* p);
/* Must precede mpm_bind_workspace (sizes depend on it). */
mpm_status mpm_set_params(mpm_handle h, const mpm_params* p);

/* Bind the CUDA stream all work is enqueued on (cudaStream_t as void*; 0 = legacy default). */
mpm_status mpm_set_stream(mpm_handle h, void* cuda_stream);

/* Bytes of device workspace needed for the current params (max_steps, k_ckpt,
 * n_episodes).  Bind a device allocation of at least that size (256-B aligned). */
mpm_status mpm_workspace_bytes(mpm_handle h, size_t* bytes);
/* The same for a tape of `steps` steps (SURVEY 8(b) form), without changing the handle's
 * max_steps; steps >= 1. */
mpm_status mpm_workspace_bytes_for(mpm_handle h, int32_t steps, size_t* bytes);
mpm_status mpm_bind_workspace(mpm_handle h, void* device_ptr, size_t bytes);

/* Copy in the initial state S_0 (host or device pointers, layouts above).
 * actuator_id may be NULL (all passive); ids must be -1 (passive) or in [0, n_actuators).
 * Values are validated on the device and reported by the next mpm_forward
 * (out-of-domain -> MPM_ERR_OUT_OF_DOMAIN, an actuator id out of range ->
 * MPM_ERR_INVALID_ARG; the kernels treat such ids as passive, never index with them).
 * Clears any tape. */
mpm_status mpm_set_state(mpm_handle h, const float* x, const float* v, const float* C,
                         const float* F, const int32_t* actuator_id);

/* Per-particle material (R23), host or device pointer, [E][N] caller
 * order: 0 = the elastic solid of mpm_params.model; nonzero = weakly compressible fluid (mu = 0,
 * volumetric stress only, F reset to J^(1/d) I after every step).  NULL (the default after
 * bind) = all solid.  Persists across mpm_set_state; clears a recorded tape.  Fluid particles
 * should be passive (actuator_id -1). */
mpm_status mpm_set_materials(mpm_handle h, const int32_t* material);

/* Number of controller parameters for the current params, and set them
 * (host or device pointer, n_theta floats). */
mpm_status mpm_n_theta(mpm_handle h, int64_t* n_theta);
mpm_status mpm_set_controller(mpm_handle h, const float* theta, int64_t n_theta);

/* Run `steps` advance() calls from S_0 (1 <= steps <= max_steps), recording
 * the tape (checkpoints every k_ckpt steps).  Replaces any previous tape. */
mpm_status mpm_forward(mpm_handle h, int32_t steps);

/* Loss on S_T of the recorded forward (loss_kind/loss_target from params);
 * writes L_e to loss_out[E] (host or device; may be NULL) and seeds the
 * adjoint of S_T with dL/dS_T (loss adjoint = 1). */
mpm_status mpm_loss(mpm_handle h, float* loss_out);

/* Alternative to mpm_loss for a loss computed by the caller: seed the adjoint
 * of S_T with dL/dx_T, dL/dv_T, dL/dC_T, dL/dF_T (host or device, caller
 * order; any may be NULL = zero). */
mpm_status mpm_seed_adjoint(mpm_handle h, const float* dx, const float* dv, const float* dC,
                            const float* dF);

/* Replay the tape in reverse (advance_grad per step, segment recomputation);
 * steps must equal the recorded forward's. */
mpm_status mpm_backward(mpm_handle h, int32_t steps);

/* Gradients of sum_e L_e w.r.t. the initial state (caller order) and theta
 * (summed over the local episodes).  Any pointer may be NULL. */
mpm_status mpm_grads(mpm_handle h, float* dx0, float* dv0, float* dC0, float* dF0,
                     float* dtheta);

/* Gradient w.r.t. a uniform initial velocity shared by all particles of an
 * episode (the "initial state parameterisation" of Fig. 1):
 * out[E][d] = sum_p dL/dv0_p (fixed-order reduction).  Host or device pointer. */
mpm_status mpm_grad_v0_sum(mpm_handle h, float* out);

/* Current state S_T of the recorded forward (or S_0 before any forward). */
mpm_status mpm_get_state(mpm_handle h, float* x, float* v, float* C, float* F);

/* Number of library kernel launches enqueued since the handle was created
 * (for the benchmark's gpu_launches count). */
mpm_status mpm_launch_count(mpm_handle h, int64_t* count);

/* ---- measurement hooks (bench.py) ------------------------------------------
 * Per-kernel device time: with profiling on, every library launch is
 * bracketed by CUDA events on the bound stream; durations are harvested at the
 * next synchronising call.  idx enumerates kernel classes 0..n-1
 * (MPM_ERR_INVALID_ARG past the end); *name is a static string. */
mpm_status mpm_set_profiling(mpm_handle h, int32_t enable);
mpm_status mpm_reset_kernel_stats(mpm_handle h);
mpm_status mpm_kernel_stats(mpm_handle h, int32_t idx, const char** name, double* total_ms,
                            int64_t* count);
/* Grid nodes with M > 0 in the grid of step `step` of the recorded forward (0 <= step <
 * recorded, else MPM_ERR_INVALID_ARG), summed over episodes: the "active nodes" A of the
 * algorithmic byte count.  mpm_active_nodes = the last recorded step.
 * Synchronises. */
mpm_status mpm_active_nodes_at(mpm_handle h, int32_t step, int64_t* count);
mpm_status mpm_active_nodes(mpm_handle h, int64_t* count);

/* ---- one body over several slab subdomains -----
 * The grid is split along x into contiguous slabs of blocks (block edge 4 cells in 3D, 8 in 2D);
 * one handle per slab, on one device or several (NVLink peer access).  Subdomain g owns the
 * blocks with block x-index in [x_lo, x_hi) and, at every step, the particles whose base cell
 * lies in them: particles migrate between neighbours each step, and the grid-node sums at a slab
 * face read the neighbour's partial tiles from its memory.  The result (states, loss, gradients)
 * is bitwise equal to the single-domain run of the same body.
 * Scope: one episode, a passive body (n_actuators = 0, solid and/or fluid), k_ckpt = 1, particles
 * moving less than one slab per step (else MPM_ERR_UNSUPPORTED / MPM_ERR_OOM).
 * Sequence per handle: mpm_create(capacity, ...) -> [set_params] -> mpm_set_subdomain -> bind ->
 * mpm_dd_link(all) -> mpm_set_state_ids -> [mpm_set_materials([n_body], by id)] ->
 * mpm_dd_forward(all) -> mpm_dd_loss(all) -> mpm_dd_backward(all) -> mpm_grads (the rows given to
 * set_state_ids, in that order) / mpm_get_state_ids. */

/* Before bind: this handle is the subdomain [x_lo, x_hi) (block x-indices) of a body of n_body
 * particles (ids 0..n_body-1); mpm_create's n_particles is the subdomain's particle capacity.
 * migrate_cap: emigrants per direction and step (0 = capacity / 8 + 1024). */
mpm_status mpm_set_subdomain(mpm_handle h, int32_t x_lo, int32_t x_hi, int64_t n_body, int32_t migrate_cap);
/* After bind: hs[0..n-1] are the subdomains in slab order (1 <= n <= 4), slabs contiguous and
 * covering the grid, parameters identical.  Enables peer access between their devices. */
mpm_status mpm_dd_link(mpm_handle* hs, int32_t n);
/* The subdomain's particles at t = 0 (n <= capacity; host or device pointers, layouts as
 * mpm_set_state with N = n) and their body-wide ids (int32 [n]).  Particles outside the slab
 * are reported by mpm_dd_forward (MPM_ERR_OOM). */
mpm_status mpm_set_state_ids(mpm_handle h, int64_t n, const float* x, const float* v, const float* C,
                             const float* F, const int32_t* ids);
/* forward(T) / loss / backward(T) of the whole body over the linked subdomains (every handle's
 * work on its own stream; synchronises all).  loss_out: host or device, 1 float (may be NULL). */
mpm_status mpm_dd_forward(mpm_handle* hs, int32_t n, int32_t steps);
mpm_status mpm_dd_loss(mpm_handle* hs, int32_t n, float* loss_out);
mpm_status mpm_dd_backward(mpm_handle* hs, int32_t n, int32_t steps);
/* Rows of S_T this subdomain holds (its particles of step T-1), and those rows with their ids. */
mpm_status mpm_dd_rows(mpm_handle h, int64_t* rows);
mpm_status mpm_get_state_ids(mpm_handle h, float* x, float* v, float* C, float* F, int32_t* ids);

#ifdef __cplusplus
}
#endif
#endif
