// kernels.h -- host-side launchers of the sm_100a kernels (internal to libmpm_b200.so).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "mpm_device.cuh"

namespace mpm {

// every kernel launch of the library: programmatic stream serialization (PDL) allowed, so the
// kernel may be scheduled while its predecessor drains (each kernel starts with pdl_begin()).
bool pdl_enabled();  // programmatic dependent launch for this host thread's launches
void set_pdl(int64_t particles);  // choose PDL for the next launches (see kernels_tile.cu)
template <typename... KArgs, typename... Args>
inline void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// particle state in split arrays (Lay<D>) + particle id (global caller index e*N + p)
struct StateView {
    float* x;
    float* vc;
    float* f;
    int* pid;
};
// adjoint state, same split layout, indexed like the primal state it belongs to
struct AdjView {
    float* x;
    float* vc;
    float* f;
};

// SURVEY 8(f) f3 (one body over slab subdomains, engine_dd.cu): this subdomain owns the grid
// blocks with block x-index in [x_lo, x_hi); the neighbours (0 = left, 1 = right) own the
// adjacent columns.  A node tile near a slab face is covered by partial tiles of the neighbour's
// face column: covered_sum reads them from the neighbour's memory (same device or NVLink peer)
// in the same fixed order as a single-domain run.  Single domain: x_lo = 0, x_hi = nb, no
// neighbours.
struct Halo {
    int x_lo, x_hi;
    const int* bmap[2];      // neighbour's block map of this step (null: no neighbour)
    const float4* tiles[2];  // neighbour's per-step partial tiles (local block index)
    const int* base[2];      // neighbour's pool base of this step (device scalar)
};

// particles leaving the slab in g2p (f3): per direction (0 = left, 1 = right) a count and the
// rows of S_{t+1} that emigrate; cnt == null in a single-domain run
struct Migr {
    int x_lo, x_hi;
    int* cnt;   // [2]
    int* rows;  // [2][cap]
    int cap;
};

// one time step's binning + grid.  The block lists, cell
// starts and node tiles of all steps live in one pool; step t's entries start at pool
// index *base (set on the device by the step's scan), so only the active blocks of
// each step take space.  bmap holds pool (global) tile indices.
struct SlotView {
    int* sigma;              // [EN]   sorted order -> index into that step's state array
    unsigned char* scell;    // [EN]   cell (0..63, 64 = junk) of the sorted entry (set by bin_scatter)
    int* spid;               // [EN]   particle id of the sorted entry (set by bin_scatter)
    int* blist;              // pool [P]          active block ids of a step (block-id order)
    int* bstart;             // pool [P + T + 1]  segment starts; step t uses [base + t, base + t + n]
    int* bmap;               // [TB]   block id -> pool tile index, or -1
    int* nactive;            // [1]    active blocks of this step
    int* base;               // [1]    pool offset of this step (nactive[-1], base[-1]: previous step)
    unsigned short* cstart;  // pool [P][CELLS+1] cell starts within the block segment
    float4* tiles;           // pool [P][TN]      resolved node tiles (u1, M or -1 = sticky)
    float4* part;            // [max_active][TN]  per-step scratch: p2g partial (P, M) tiles,
                             //                   backward: grid_op_grad output (Pb, Mb)
    int* ntot;               // [1]    sorted particles of this step (set by the scan)
    int* nbr;                // pool [P][3^d] pool tile index of each neighbour block (offsets -1..1 per
                             //        axis), or -1; set by p2g (small problems; null otherwise), read by the grid passes
    int step;                // t
    Halo halo;               // f3 neighbours (covered sums of grid_op / grid_op_grad)
};

cudaError_t tile_init();

// ---- binning (bin_keys only for a fresh sort; g2p emits keys for the next step)
// rows >= n_live get key -1 (not binned); n_live = N * E in a single-domain run
void launch_bin_keys(const KParams& p, const float* x, int64_t n_live, int* keys, int* bcount, int* flags,
                     cudaStream_t s);
int scan_chunks(const KParams& p);  // entries of `part` (int2) the scan needs
void launch_bin_scan(const KParams& p, int* bcount, int* cursor, const SlotView& sl, int* part, int* flags,
                     cudaStream_t s);
// keys[j] = block * 128 + cell of entry j; pid[j] its particle id
void launch_bin_scatter(const KParams& p, const int* keys, const int* pid, int* cursor, const SlotView& sl,
                        cudaStream_t s);

// canonical (cell, particle id) order of every active block's list; cell starts; the
// particle ids of S_{t+1} (pid_next, nullable) in that order.  Runs before each p2g.  A block
// with more than MAXP particles is dropped (FLAG_BLOCK_OVERFLOW) and its rows' next bin keys
// (keys_next, nullable) are set to -1.
void launch_canon(const KParams& p, const SlotView& sl, int* pid_next, int* keys_next, int* flags, cudaStream_t s);

// ---- one forward step (advance())
// p2g writes F_{t+1} and particle ids of S_{t+1} when Sn.rec / Sn.pid are non-null
// canon_fused(): p2g does the canonical ordering of each block itself (launch_canon is then
// skipped; p2g takes its pid_next = Sn.pid and keys_next arguments)
bool canon_fused(const KParams& p);
void launch_p2g(const KParams& p, const SlotView& sl, const StateView& S, const StateView& Sn,
                const int32_t* aid, const float* alpha_t, int* keys_next, int* flags, cudaStream_t s);
// grid_op: sum of the covering partial tiles -> resolved tile of every active block
void launch_grid_op(const KParams& p, const SlotView& sl, cudaStream_t s);
// g2p writes x, v, C of S_{t+1}; keys != null -> next bin keys;
// refwd: segment re-forward from stored tiles -- also writes F_{t+1} = (I + dt C) F and the ids
// mg.cnt != null (f3): particles whose next block leaves [mg.x_lo, mg.x_hi) get key -1 and are listed
// in the outbox mg.rows by direction
void launch_g2p(const KParams& p, const SlotView& sl, const StateView& S, const StateView& Sn, int* keys,
                int* bcount, int* flags, bool refwd, const Migr& mg, cudaStream_t s);

// ---- f3 migration (engine_dd.cu)
// append the neighbours' emigrants of step t to S_{t+1} (rows nsorted_t + ...), bin keys + histogram;
// imm_base[side] = first row of the immigrants from that side, *nrows = rows of S_{t+1}
struct MigSrc {
    StateView S;     // the neighbour's S_{t+1} (peer pointers)
    const int* cnt;  // the neighbour's outbox count toward this subdomain (null: no neighbour)
    const int* rows;
    int cap;         // the neighbour's outbox capacity per direction (rows is [2][cap])
};
void launch_immigrate(const KParams& p, const StateView& S, const int* nsorted, MigSrc left, MigSrc right,
                      int x_lo, int x_hi, int cap, int* keys, int* bcount, int* imm_base, int* nrows, int* flags,
                      cudaStream_t s);
// backward: S_bar_{t+1} rows of this subdomain's emigrants of step t <- the neighbour's immigrant rows
// (the AoSoA state layout has no capacity-dependent stride, so neighbours of any capacity read alike)
void launch_adj_pull(const KParams& p, const AdjView& Sb, const int* cnt, const int* rows, int cap,
                     const AdjView& nb_left, const int* nb_left_base, const AdjView& nb_right,
                     const int* nb_right_base, cudaStream_t s);

// ---- COM loss in fixed block order (partition independent, f3): per-block sums of x over the
// rows S_T holds in step T-1's sorted order, then per episode a fixed-order sum over the
// concatenation of up to 4 block lists (the subdomains of a decomposed body, in slab order)
void launch_block_com(const KParams& p, const SlotView& sl_last, const float* x, float* part, cudaStream_t s);
struct ListSrc {
    const float* part;  // [n][d] per-block partial sums (list order)
    const int* blist;   // block-list pool; this step's list starts at pool index *base
    const int* base;    // device scalar: pool offset of the step
    const int* n;       // device scalar: entries
};
void launch_loss_blocks(const KParams& p, const ListSrc* src, int nsrc, int loss_kind, float3 target, float* loss,
                        float* seed, const AdjView& Sb, int* flags, cudaStream_t s);

// ---- one reverse step (advance_grad()); Sbn is indexed like S_{t+1}, Sb like S_t
// g2p_grad in two independent passes over step t's blocks: the U_bar scatter and
// the gather part (xb_t partial = xb_{t+1} + fb/dx); they may run on two streams
void launch_g2p_grad(const KParams& p, const SlotView& sl, const StateView& S, const AdjView& Sbn,
                     float4* ubar, cudaStream_t s);
void launch_g2p_grad_gather(const KParams& p, const SlotView& sl, const StateView& S, const AdjView& Sbn,
                            float* xbar_part, cudaStream_t s);
// grid_op_grad: covering sums of the U_bar partial tiles -> (P_bar, M_bar) tiles in sl.part
void launch_grid_op_grad(const KParams& p, const SlotView& sl, const float4* ubar, cudaStream_t s);
void launch_p2g_grad(const KParams& p, const SlotView& sl, const StateView& S, const int32_t* aid,
                     const float* alpha_t, const AdjView& Sbn, const float* xbar_part,
                     const AdjView& Sb, float* abar_part, int* flags, cudaStream_t s);
// alpha_bar_t[a] (open loop) or alpha_bar_t[e][a] (closed loop) = fixed-order sum of the
// per-block partials of the step
void launch_reduce_abar(const KParams& p, const SlotView& sl, const float* abar_part, float* alpha_bar_t,
                        cudaStream_t s);

// ---- measurement: distinct grid nodes with M > 0 in a slot's tiles -> *count (device)
void launch_count_active(const KParams& p, const SlotView& sl, int64_t* count, cudaStream_t s);

// actuator ids outside [-1, n_act) -> FLAG_BAD_ACTUATOR
void launch_check_aid(const KParams& p, const int32_t* aid, int* flags, cudaStream_t s);

// ---- closed-loop controller (R22)
int obs_parts(const KParams& p);   // per-CTA partials of one observation: [E][chunks]
int obs_values(const KParams& p);  // values per partial: n_act (2d + 1) + d
// per-CTA sums over S_t (x, v in its split arrays; particle id -> actuator id) -> part
void launch_observe(const KParams& p, const float* x, const float* vc, const int* pid, const int32_t* aid,
                    float* part, cudaStream_t s);
// o_t per episode from the partials (fixed order), alpha_t[e] = MLP([phi(t), o_t[e]]);
// stores o_t [E][2 d n_act] and the group sizes [E][n_act]
void launch_ctrl_obs_fwd(const KParams& p, const float* theta, int32_t t, const float* part, float* obs_t,
                         float* counts, float* alpha_t, cudaStream_t s);
// theta_bar += sum_e (d alpha_t[e]/d theta)^T alpha_bar_t[e] (episodes in order, one CTA);
// inc[e] = per-group adjoint increments of x_bar / v_bar from (d alpha_t/d o_t)^T alpha_bar_t
void launch_ctrl_obs_bwd(const KParams& p, const float* theta, int32_t t, const float* obs_t,
                         const float* alpha_t, const float* alpha_bar_t, const float* counts,
                         float* theta_bar, float* inc, cudaStream_t s);
// S_bar_t.x, .v += the observation adjoint (particle i of episode i / N, group aid[pid[i]])
void launch_observe_adj(const KParams& p, const AdjView& Sb, const int* pid, const int32_t* aid,
                        const float* inc, cudaStream_t s);

// ---- controller (compute_actuation, P:577 / .grad P:591)
void launch_ctrl_fwd(const KParams& p, const float* theta, int32_t T, float* alpha, cudaStream_t s);
void launch_ctrl_bwd(const KParams& p, const float* theta, int32_t T, const float* alpha,
                     const float* alpha_bar, float* theta_part, float* theta_bar, int64_t n_theta,
                     cudaStream_t s);

// ---- loss on x_T and the adjoint seed (episodes occupy contiguous index ranges)
int loss_blocks_per_episode(const KParams& p);
void launch_loss(const KParams& p, const float* x, int loss_kind, float3 target, float* com_part,
                 float* loss, const AdjView& Sb, int* flags, cudaStream_t s);
// ---- per-episode sum of the v-adjoint: out[E][d] (fixed order)
void launch_v_sum(const KParams& p, const float* vc_bar, float* part, float* out, cudaStream_t s);

// ---- layout conversion (caller arrays <-> split state arrays)
// pack: dst row i <- caller row src[i] (src == null: i); ident_pid != null -> ident_pid[i] = i;
// null x / v / C -> zero, null F -> identity (zero when zero_f)
void launch_pack(const KParams& p, const float* x, const float* v, const float* C, const float* F,
                 const int* src, float* dx, float* dvc, float* df, int* ident_pid, bool zero_f,
                 cudaStream_t s);
// unpack: caller row dst[i] (dst == null: i) <- row i
void launch_unpack(const KParams& p, const float* sx, const float* svc, const float* sf, const int* dst,
                   float* x, float* v, float* C, float* F, cudaStream_t s, int64_t n_rows = -1);

}  // namespace mpm
