// engine.h -- internal to libmpm_b200.so: the handle (mpm_ctx) and the engine helpers shared by
// engine.cu (single-domain C-ABI) and engine_dd.cu (one body over several slab
// subdomains).
#pragma once
#ifndef MPM_OBS_AHEAD
#define MPM_OBS_AHEAD 1  // closed loop: observation + controller of step t+1 beside its binning (step_forward)
#endif
#ifndef MPM_ABAR_SIDE
#define MPM_ABAR_SIDE 1  // open-loop actuator-gradient reduction on its own stream (step_backward)
#endif
#include <cstdint>
#include <functional>
#include <map>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/mpm.h"
#include "kernels.h"

namespace eng {
using namespace mpm;

enum Phase { kCreated = 0, kBound, kHasState, kForward, kSeeded, kBackward };

// kernel classes for the per-kernel device-time accounting (mpm_kernel_stats)
enum KClass { KC_P2G = 0, KC_G2P, KC_BIN, KC_G2P_GRAD, KC_P2G_GRAD, KC_REDUCE_ABAR, KC_CTRL,
              KC_LOSS, KC_LAYOUT, KC_GRID_OP, KC_GRID_OP_GRAD, KC_G2P_GRAD_GATHER, KC_CANON, KC_N };
extern const char* const kClassNames[KC_N];

struct Profiler {
    bool on = false;
    std::vector<cudaEvent_t> pool;
    size_t used = 0;
    std::vector<std::pair<int, size_t>> pending;
    double ms[KC_N] = {0};
    int64_t n[KC_N] = {0};
};

inline size_t align_up(size_t n) { return (n + 255) & ~size_t(255); }

}  // namespace eng

struct mpm_ctx {
    int64_t N = 0;
    int32_t n_grid = 0, dim = 0;
    float dt = 0, E = 0, nu = 0;
    mpm_params prm{};
    cudaStream_t stream = 0;
    cudaStream_t side = nullptr;             // second stream (g2p_grad gather || U_bar scatter)
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    cudaStream_t side2 = nullptr;            // third stream: segment re-forward ahead of the reverse
    cudaEvent_t ev_seg = nullptr, ev_refwd = nullptr;
    cudaStream_t side3 = nullptr;            // open-loop actuator-gradient reduction (step_backward)
    cudaEvent_t ev_p2gg = nullptr, ev_abar[2] = {nullptr, nullptr};
    int obs_ahead = -1;                      // closed loop: step whose observation + controller run on `side`
    bool abar_pending[2] = {false, false};   // a reduction on side3 still reads abar_part buffer b
    size_t abar_stride = 0;                  // floats per abar_part buffer
    float* xbar_part = nullptr;    // [d][EN] xb_t partial from g2p_grad's gather part
    int device = 0;
    std::string err;
    int64_t launches = 0;
    // workspace
    char* ws = nullptr;
    size_t ws_bytes = 0;
    size_t state_floats = 0;  // E * N * R
    int n_ckpt = 0;
    int max_active = 0;
    std::vector<mpm::StateView> ckpt;   // S_{s k}
    std::vector<mpm::StateView> window; // [2][k]: S_{s k + j}, j = 1..k-1, in half (s & 1) (double-buffered so
                                   // the re-forward of segment s-1 overlaps the reverse of segment s)
    mpm::StateView final_state{};       // S_T
    // grid store (all steps): sorted lists, block maps, and a pool of block lists /
    // cell starts / node tiles addressed by a per-step device-side base
    int* sigma_store = nullptr;    // [T_max][EN]
    unsigned char* scell_ring[2] = {nullptr, nullptr};  // [EN] (consumed by the next p2g only)
    int* spid_ring[2] = {nullptr, nullptr};
    int* bmap_store = nullptr;     // [T_max][TB]
    int* nactive_arr = nullptr;    // [T_max]
    int* base_arr = nullptr;       // [T_max]
    int* blist_pool = nullptr;     // [P]
    int* nbr_pool = nullptr;       // [P][3^d] neighbour-block pool indices (SlotView::nbr)
    int* bstart_pool = nullptr;    // [P + T_max + 1]
    unsigned short* cstart_pool = nullptr;  // [P][65]
    float4* tiles_pool = nullptr;  // [P][TN]
    int pool_blocks = 0;           // P
    int step_blocks = 0;           // per-step capacity of block-local buffers
    mpm::AdjView sbar[2] = {};          // adjoint states, indexed like the primal state of their step
    float* staging = nullptr;
    int32_t* aid = nullptr;        // caller order
    int* bcount = nullptr;         // [TB] block histogram (kept zero between uses)
    int* cursor = nullptr;         // [TB]
    int* scan_part = nullptr;      // [scan chunks + 2] int64: epoch-tagged chunk totals, epoch, ticket
    int* keys = nullptr;           // [EN]
    float4* ubar = nullptr;        // [max_active][TN]  U_bar partial tiles of the current step
    float4* part = nullptr;        // [max_active][TN]  p2g partial tiles / (Pb, Mb) tiles
    float* abar_part = nullptr;    // [max_active][n_act]
    float* alpha = nullptr;        // [max_steps][n_act] ([max_steps][E][n_act] closed loop)
    float* alpha_bar = nullptr;
    float* obs = nullptr;          // closed loop: [max_steps][E][2 d n_act] observations o_t
    float* obs_cnt = nullptr;      // [E][n_act] particles per actuator group
    float* obs_part = nullptr;     // [E][chunks][values] per-CTA observation sums
    float* obs_inc = nullptr;      // [E][2 d n_act + d] adjoint increments of the current step
    float* theta = nullptr;
    float* theta_bar = nullptr;
    float* theta_part = nullptr;   // [max_steps][n_theta]
    float* loss = nullptr;         // [E]
    float* com_part = nullptr;
    int64_t* counter = nullptr;
    int* flags = nullptr;
    int* h_flags = nullptr;
    // tape
    eng::Phase phase = eng::kCreated;
    bool has_aid = false;
    bool has_mat = false;          // any fluid particle (R23) set by mpm_set_materials
    int32_t* mat = nullptr;        // [EN] material by particle id (0 solid, nonzero fluid)
    int32_t recorded = 0;
    int32_t t_final = 0;
    int window_seg = -1;
    int sbar_cur = 0;
    eng::Profiler prof;
    // CUDA graphs of whole forward / backward tapes, keyed by (kind, T, has_aid, window
    // segment at entry); replayed instead of re-enqueueing thousands of launches
    struct GraphRec {
        cudaGraphExec_t exec = nullptr;
        int64_t launches = 0;
        int window_seg = -1, sbar_cur = 0;
    };
    std::map<std::tuple<int, int, int, int>, GraphRec> graphs;
    bool use_graphs = true;
    int* ntot_arr = nullptr;       // [T_max + 1] sorted particles per step (set by the scan)
    float* blk_part = nullptr;     // [max_active][d] per-block COM partials of the loss
    // ---- slab subdomain of a decomposed body (engine_dd.cu)
    bool dd = false;               // set by mpm_set_subdomain
    int x_lo = 0, x_hi = 0;        // owned block x-index range
    int64_t n_body = 0;            // particles of the whole body (ids 0..n_body-1)
    int64_t n0 = 0;                // particles of this subdomain at t = 0 (mpm_set_state_ids)
    int mig_cap = 0;               // emigrants per direction and step
    mpm_ctx* nbr[2] = {nullptr, nullptr};  // left / right neighbour (mpm_dd_link)
    int* out_cnt = nullptr;        // [T_max][2]        emigrants of step t by direction
    int* out_rows = nullptr;       // [T_max][2][cap]   their rows of S_{t+1}
    int* imm_base = nullptr;       // [T_max + 1][2]    first row of S_t's immigrants from each side
    int* nrows_arr = nullptr;      // [T_max + 1]       rows of S_t (sorted of t-1 + immigrants)
    cudaEvent_t dd_ev[4] = {};     // per-phase events of the decomposed step
};

namespace eng {
// Makes the handle's device current for the duration of an entry point (one process may
// drive several GPUs, each through its own handles) and restores the caller's device.
struct DevGuard {
    int prev = -1;
    bool changed = false;
    explicit DevGuard(const mpm_ctx* h) {
        if (!h || cudaGetDevice(&prev) != cudaSuccess) return;
        if (prev != h->device) changed = cudaSetDevice(h->device) == cudaSuccess;
    }
    ~DevGuard() {
        if (changed) cudaSetDevice(prev);
    }
};

mpm_status fail(mpm_handle h, mpm_status st, const std::string& msg);

// NVTX range around a C-ABI call (visible in Nsight Systems / ncu --nvtx; graph replays of the
// steps are device-side and show as the enclosing call's range)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

#define CU(call)                                                                           \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess)                                                             \
            return fail(h, MPM_ERR_CUDA, std::string(#call ": ") + cudaGetErrorString(e_)); \
    } while (0)

void prof_harvest(mpm_ctx* h);
// counts one library launch group and, when profiling is on, brackets it with
// CUDA events on the bound stream
struct KScope {
    mpm_ctx* h;
    int cls;
    size_t idx = 0;
    bool active = false;
    KScope(mpm_ctx* h_, int c) : h(h_), cls(c) {
        h->launches += 1;
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

int block_edge(int dim);
int tile_nodes(int dim);
constexpr int kCells = 64;
KParams kparams(const mpm_ctx* h);
size_t carve(mpm_ctx* h, char* base);
StateView state_at(mpm_ctx* h, int t);
SlotView slot_at(mpm_ctx* h, int t);
mpm_status sync_flags(mpm_handle h, const char* where);
mpm_status copy_in(mpm_handle h, void* dst, const void* src, size_t bytes);
// COM loss of the recorded S_T in fixed block order + the adjoint seed (single domain)
void launch_loss_blocks(mpm_ctx* h, const KParams& k);
}  // namespace eng
