// kernels_tile.cu -- the MLS-MPM step and its adjoint on sm_100a, sorted-tile scheme.
//
// Equations: DESIGN.md R1-R14, R22-R23; kernel order: PAPER.md
// Appendix D.1 (advance / advance_grad).
//
// Layout:
//  * particles are binned every step by the B^d block of cells that holds their
//    base cell (bin_* kernels); k_canon puts each block's list sigma in canonical
//    (cell, particle id) order, so every sum below has a fixed order -> results are
//    bitwise reproducible run to run, and there are no atomics in the hot loops;
//  * p2g: one CTA per active block (persistent loop).  Thread per particle: the
//    stress/affine math in registers, producing a 24-float row [wy*wz, c, A dx, wx]
//    in shared memory; then a thread per (cell, o_x) walks the cell's rows and
//    accumulates its 3^(d-1) nodes in registers (separable weights, incremental
//    m = c + A dx o); a thread per tile node sums the <= 3^d (cell, o) partials and
//    stores the block's (B+2)^d node tile with plain stores;
//  * grid_op / grid_op_grad resolve every active block's tile once per step (sum of the
//    <= 2^d overlapping partial tiles, fixed order); g2p, g2p_grad's gather part and
//    p2g_grad stage their resolved node tile with cp.async.bulk (TMA engine) + mbarrier,
//    double buffered across blocks; g2p and p2g_grad use nested separable sums;
//    g2p_grad scatters U_bar with p2g's (cell, o_x) scheme.
#include "kernels.h"

#include <algorithm>
#include <cstdlib>
#include <mutex>

namespace mpm {

namespace {

constexpr int kT = 256;  // threads per CTA (8 warps)
constexpr int kW = kT / 32;

// block id -> episode and first cell (c0 = block coords * B)
// FAST (the per-node grid passes, where this runs once per node): divisions by a float
// reciprocal (divq); the per-block callers keep the integer division (their register
// allocation is tuned around it)
template <int D, bool FAST = false>
__device__ __forceinline__ void block_origin(const KParams& p, int bid, int& e, int c0[3]) {
    if (FAST) {
        e = divq(bid, p.nbe, p.inv_nbe);
        int l = bid - e * p.nbe;
        c0[2] = 0;
#pragma unroll
        for (int k = D - 1; k >= 1; --k) {
            const int q = divq(l, p.nb, p.inv_nb);
            c0[k] = (l - q * p.nb) * Geo<D>::B;
            l = q;
        }
        c0[0] = l * Geo<D>::B;  // l < nb here
        return;
    }
    e = bid / p.nbe;
    int l = bid - e * p.nbe;
    c0[2] = 0;
#pragma unroll
    for (int k = D - 1; k >= 0; --k) {
        c0[k] = (l % p.nb) * Geo<D>::B;
        l /= p.nb;
    }
}

template <int D> __device__ __forceinline__ int block_lin(const KParams& p, int e, const int b[3]) {
    return D == 2 ? e * p.nbe + b[0] * p.nb + b[1] : e * p.nbe + (b[0] * p.nb + b[1]) * p.nb + b[2];
}

// base cell of x and its validity (3^d stencil inside [0, n_grid - 1]^d, R13)
template <int D> __device__ __forceinline__ bool base_cell(const KParams& p, const float* x, int b[3]) {
    bool ok = true;
    b[2] = 0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
        float f = floorf(x[k] * p.inv_dx - 0.5f);
        ok = ok && (f >= 0.0f) && (f + 2.0f <= (float)(p.n_grid - 1));
        b[k] = ok ? (int)f : 0;
    }
    return ok;
}

template <int D> __device__ __forceinline__ int tile_lin(int a, int b, int c) {
    constexpr int TE = Geo<D>::TE;
    return D == 2 ? a * TE + b : (a * TE + b) * TE + c;
}

template <int D> __device__ __forceinline__ void local_node(int q, int n[3]) {
    constexpr int TE = Geo<D>::TE;
    if (D == 2) { n[0] = q / TE; n[1] = q % TE; n[2] = 0; }
    else { n[0] = q / (TE * TE); n[1] = (q / TE) % TE; n[2] = q % TE; }
}

template <int D> __device__ __forceinline__ int cell_of(const int lb[3]) {
    using G = Geo<D>;
    return D == 2 ? lb[0] * G::B + lb[1] : (lb[0] * G::B + lb[1]) * G::B + lb[2];
}

// Sum of the <= 2^d block tiles that cover global node g (episode e): every
// block whose cells [c0, c0 + B) satisfy c0 <= g < c0 + B + 2 holds a partial
// of that node.  Fixed enumeration order -> deterministic.
// f3: a covering block outside this subdomain's slab [x_lo, x_hi) belongs to a neighbour, whose
// block map and (pool-indexed) tiles nt[0] (left) / nt[1] (right) are read instead -- the same
// blocks in the same order as a single-domain run.
// HALO = false (a single domain, no neighbours) compiles the neighbour branch out.
template <int D, bool HALO>
__device__ __forceinline__ float4 covered_sum(const KParams& p, int e, const int g[3],
                                              const int* __restrict__ bmap,
                                              const float4* __restrict__ tiles, const Halo& hl,
                                              const float4* nt0, const float4* nt1) {
    using G = Geo<D>;
    // per axis: option 0 = the block holding g (local l0), option 1 = the previous
    // block (local l0 + B), valid when l0 < 2.  All 2^d combinations unrolled.  (A
    // branch-free form issuing all 2^d map loads, then all tile loads, measured slower:
    // grid_op 34.8 -> 36.8 ms per C5 iteration -- the branches skip the absent blocks' loads.)
    int b0[3], l0[3];
    bool ok1[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        b0[k] = k < D ? g[k] >> G::LOGB : 0;
        l0[k] = k < D ? g[k] & (G::B - 1) : 0;
        ok1[k] = k < D && l0[k] < 2 && b0[k] >= 1;
    }
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int c = 0; c < (D == 3 ? 2 : 1); ++c) {
                if ((a && !ok1[0]) || (b && !ok1[1]) || (c && !ok1[2])) continue;
                const int bb[3] = {b0[0] - a, b0[1] - b, b0[2] - c};
                if (bb[0] >= p.nb || bb[1] >= p.nb || (D == 3 && bb[2] >= p.nb)) continue;
                const int* bm = bmap;
                const float4* tl = tiles;
                if (HALO) {
                    if (bb[0] < hl.x_lo) { bm = hl.bmap[0]; tl = nt0; }
                    else if (bb[0] >= hl.x_hi) { bm = hl.bmap[1]; tl = nt1; }
                    if (bm == nullptr) continue;
                }
                const int ti = __ldg(bm + block_lin<D>(p, e, bb));
                if (ti < 0) continue;
                const int lq = tile_lin<D>(l0[0] + a * G::B, l0[1] + b * G::B, l0[2] + c * G::B);
                const float4 v = __ldg(tl + (int64_t)ti * G::TN + lq);
                acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
            }
    return acc;
}

// Neighbour table (single domain): row bi of step t holds, for each block offset o in {-1, 0, 1}^d
// (o_0 slowest), the pool tile index of block (block of bi) + o, or -1 -- the block-map lookups
// of covered_sum done once per block (in p2g, with the canonical ordering) instead of once per
// tile node, so a grid pass's tile loads no longer wait on a block-map load.  Small problems only
// (SlotView::nbr is null otherwise): C2 +6.5%, but C5 +0.2% at k = 2 and -0.9% at k = 32 (the fill
// lengthens k_canon by more than the grid passes gain).
#ifndef MPM_NBR_TABLE
#define MPM_NBR_TABLE 1
#endif
template <int D> constexpr int kNbr = D == 3 ? 27 : 9;
template <int D>
__device__ __forceinline__ void fill_nbr(const KParams& p, const SlotView& sl, int b0, int bi, int tid) {
    if (!MPM_NBR_TABLE || sl.nbr == nullptr || tid >= kNbr<D>) return;
    int e, c0[3];
    block_origin<D>(p, sl.blist[b0 + bi], e, c0);
    const int o[3] = {tid / (D == 3 ? 9 : 3) - 1, (D == 3 ? (tid / 3) % 3 : tid % 3) - 1, D == 3 ? tid % 3 - 1 : 0};
    int bb[3] = {0, 0, 0};
    bool in = true;
#pragma unroll
    for (int k = 0; k < D; ++k) {
        bb[k] = c0[k] / Geo<D>::B + o[k];
        in = in && bb[k] >= 0 && bb[k] < p.nb;
    }
    sl.nbr[(int64_t)(b0 + bi) * kNbr<D> + tid] = in ? sl.bmap[block_lin<D>(p, e, bb)] : -1;
}
// covered_sum from the neighbour table row `nb` of the node's block; n = the node's local
// coordinates in the (B+2)^d tile.  Same covering tiles in the same order as covered_sum.
template <int D>
__device__ __forceinline__ float4 covered_sum_nbr(const int* __restrict__ nb, const int n[3],
                                                  const float4* __restrict__ tiles) {
    using G = Geo<D>;
    int h[3], l0[3];  // block offset of the node's own block (0 or 1), local coordinate in it
    bool ok1[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        h[k] = k < D ? n[k] >> G::LOGB : 0;
        l0[k] = k < D ? n[k] & (G::B - 1) : 0;
        ok1[k] = k < D && l0[k] < 2;
    }
    // all table entries first (independent loads), then the tiles
    int ti[8];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int c = 0; c < (D == 3 ? 2 : 1); ++c) {
                const int j = (a * 2 + b) * 2 + c;
                const bool use = !((a && !ok1[0]) || (b && !ok1[1]) || (c && !ok1[2]));
                const int o0 = h[0] - a, o1 = h[1] - b, o2 = h[2] - c;  // each in {-1, 0, 1}
                const int idx = D == 3 ? ((o0 + 1) * 3 + (o1 + 1)) * 3 + (o2 + 1) : (o0 + 1) * 3 + (o1 + 1);
                ti[j] = use ? __ldg(nb + idx) : -1;
            }
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int c = 0; c < (D == 3 ? 2 : 1); ++c) {
                const int j = (a * 2 + b) * 2 + c;
                if (ti[j] < 0) continue;
                const int lq = tile_lin<D>(l0[0] + a * G::B, l0[1] + b * G::B, l0[2] + c * G::B);
                const float4 v = __ldg(tiles + (int64_t)ti[j] * G::TN + lq);
                acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
            }
    return acc;
}

// neighbour tiles indexed by the neighbour's pool (tile) indices of this step (f3)
template <int D> __device__ __forceinline__ const float4* halo_tiles(const Halo& hl, int s) {
    return hl.tiles[s] ? hl.tiles[s] - (int64_t)(*hl.base[s]) * Geo<D>::TN : nullptr;
}

// grid_op (R5-R7): u0 = P/(M + eps); u1 = u0 - dt g e_y; z = sticky walls
template <int D>
__device__ __forceinline__ bool grid_velocity(const KParams& p, const int g[3], float4 pm, float u0[3],
                                              float u1[3]) {
    const float denom = pm.w + p.eps_mass;
    u0[0] = pm.x / denom; u0[1] = pm.y / denom; u0[2] = D == 3 ? pm.z / denom : 0.0f;
    u1[0] = u0[0]; u1[1] = u0[1] - p.dt * p.gravity; u1[2] = u0[2];
    bool z = false;
#pragma unroll
    for (int k = 0; k < D; ++k) {
        z = z || (g[k] < p.bound && u1[k] < 0.0f);
        z = z || (g[k] > p.n_grid - p.bound && u1[k] > 0.0f);
    }
    return z;
}

// ---- bulk async copy (TMA engine, cp.async.bulk) of a contiguous node tile into
// shared memory, completion tracked by an mbarrier (transaction bytes)
__device__ __forceinline__ uint32_t smem_u32(const void* ptr) {
    return (uint32_t)__cvta_generic_to_shared(ptr);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// generic-proxy accesses of the buffer (earlier reads) before the async-proxy write
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!ok);
}

// second bulk copy onto the same mbarrier (the expected bytes were announced by bulk_load's caller)
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// Double-buffered node-tile pipeline of a persistent CTA: tile(bi) of `src` is copied
// into buf[it & 1] while the CTA works on the previous block.  Call init() once
// (before a __syncthreads), start() before the loop, next() at the top of iteration
// `it` (after the previous iteration's closing __syncthreads) and wait() before use.
template <int D> struct TilePipe {
    static constexpr uint32_t BYTES = Geo<D>::TN * sizeof(float4);
    float4* buf;     // [2][TN]
    uint64_t* bar;   // [2]
    __device__ void init() {
        if (threadIdx.x == 0) {
            mbar_init(bar, 1);
            mbar_init(bar + 1, 1);
            fence_mbar_init();
        }
    }
    __device__ void start(const float4* src, int bi, int nact) {
        if (threadIdx.x == 0 && bi < nact) bulk_load(buf, src + (int64_t)bi * Geo<D>::TN, BYTES, bar);
    }
    __device__ void next(const float4* src, int bi_next, int nact, int it) {
        if (threadIdx.x == 0 && bi_next < nact) {
            fence_proxy_async();
            const int nb = (it + 1) & 1;
            bulk_load(buf + nb * Geo<D>::TN, src + (int64_t)bi_next * Geo<D>::TN, BYTES, bar + nb);
        }
    }
    __device__ float4* wait(int it) {
        const int cb = it & 1;
        mbar_wait(bar + cb, (uint32_t)((it >> 1) & 1));
        return buf + cb * Geo<D>::TN;
    }
};

// The same pipeline plus the block's segment of the sorted list sigma (entries
// [bstart[bi], bstart[bi + 1]) widened to 16-B boundaries) on the same mbarrier, so the
// particle loads of the block need no dependent global load of sigma: entry r of the block
// is sig_at(it, start)[r].  Blocks over MAXP particles (dropped by the binning, nvalid = 0)
// copy no list.  (Measured: g2p 132 -> 123, the gather 101.5 -> 97.9 ms per C5 iteration;
// p2g_grad slower with it, 171 -> 186, so it keeps TilePipe.)
constexpr int kSigCap = 1728 + 8;  // MAXP + the widening, ints per buffer
template <int D> struct SigPipe {
    static constexpr uint32_t BYTES = Geo<D>::TN * sizeof(float4);
    float4* buf;          // [2][TN]
    uint64_t* bar;        // [2]
    int* sig;             // [2][kSigCap]
    const int* sigma;     // this step's sorted list (16-B aligned)
    const int* bstart;    // this step's block starts
    __device__ void init() {
        if (threadIdx.x == 0) {
            mbar_init(bar, 1);
            mbar_init(bar + 1, 1);
            fence_mbar_init();
        }
    }
    __device__ void issue(const float4* src, int bi, int slot) {
        const int s0 = bstart[bi], s1 = bstart[bi + 1];
        const int a0 = s0 & ~3;
        const uint32_t sb = s1 - s0 <= Geo<D>::MAXP ? (uint32_t)((((s1 + 3) & ~3) - a0) * 4) : 0u;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar + slot)),
                     "r"(BYTES + sb)
                     : "memory");
        bulk_copy(buf + slot * Geo<D>::TN, src + (int64_t)bi * Geo<D>::TN, BYTES, bar + slot);
        if (sb) bulk_copy(sig + slot * kSigCap, sigma + a0, sb, bar + slot);
    }
    __device__ void start(const float4* src, int bi, int nact) {
        if (threadIdx.x == 0 && bi < nact) issue(src, bi, 0);
    }
    __device__ void next(const float4* src, int bi_next, int nact, int it) {
        if (threadIdx.x == 0 && bi_next < nact) {
            fence_proxy_async();
            issue(src, bi_next, (it + 1) & 1);
        }
    }
    __device__ float4* wait(int it) {
        const int cb = it & 1;
        mbar_wait(bar + cb, (uint32_t)((it >> 1) & 1));
        return buf + cb * Geo<D>::TN;
    }
    __device__ const int* sig_at(int it, int start) const { return sig + (it & 1) * kSigCap + (start & 3); }
};

// Sub-block work split of the thread-per-particle kernels (g2p, g2p_grad's gather part, p2g_grad):
// when a step has fewer active blocks than the persistent grid has CTAs (the small configurations:
// C2 ~40 blocks, C3 ~120, on 400-600 CTAs) each block's particles are split into `split` (<= 4)
// pass-aligned ranges taken by different CTAs, so more SMs work on the step.  split depends only
// on the step's block count and the grid size, so the work decomposition -- and every result --
// is deterministic.  Work item w = (block w / split, part w % split).  The kernels are instantiated
// with and without it (SPLIT): small problems (<= 256K particles per launch) take the split
// variant; large ones, whose blocks outnumber the CTAs anyway, keep the plain per-block loop
// (the index math costs g2p ~9% there).
__device__ __forceinline__ int item_split(int nact, int grid) {
    return nact > 0 ? max(1, min(kMaxSplit, grid / nact)) : 1;
}
// particle range [rb, re) of part `part` of a block with n particles, in whole passes of NT
template <int NT>
__device__ __forceinline__ void item_range(int n, int part, int split, int& rb, int& re) {
    const int passes = (n + NT - 1) / NT;
    const int per = (passes + split - 1) / split;
    rb = min(n, part * per * NT);
    re = min(n, (part + 1) * per * NT);
}

// warp-aggregated histogram increment (keys in a warp are mostly equal)
__device__ __forceinline__ void count_key(bool valid, int key, int* bcount) {
    const unsigned peers = __match_any_sync(0xffffffffu, valid ? key : -1);
    const int leader = __ffs(peers) - 1;
    if (valid && (int)(threadIdx.x & 31) == leader) atomicAdd(&bcount[key], __popc(peers));
}

// weights and base of a particle relative to the block origin
template <int D>
__device__ __forceinline__ void particle_weights(const KParams& p, const float* x, const int c0[3], int lb[3],
                                                 float fx[3], float w[3][3], float dw[3][3]) {
    lb[2] = 0;
    fx[2] = 0.f;
#pragma unroll
    for (int k = 0; k < D; ++k) {
        const float xi = x[k] * p.inv_dx;
        const float b = floorf(xi - 0.5f);
        fx[k] = xi - b;
        lb[k] = (int)b - c0[k];
        bspline(fx[k], w[k], dw[k]);
    }
}

// ---------------------------------------------------------------- binning
template <int D>
__global__ void __launch_bounds__(kT) k_bin_keys(KParams p, const float* __restrict__ X, int64_t n_live,
                                                 int* __restrict__ keys, int* __restrict__ bcount,
                                                 int* flags) {
    pdl_begin();
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n_live && i < p.N * p.E) keys[i] = -1;  // rows beyond the live ones (f3 capacity)
    const bool in = i < n_live;
    int key = 0;
    if (in) {
        float x[3];
#pragma unroll
        for (int k = 0; k < D; ++k) x[k] = X[soa<Lay<D>::X>(k, i)];
        int b[3];
        const bool ok = base_cell<D>(p, x, b);
        const int e = (int)(i / p.N);
        int bb[3] = {b[0] >> Geo<D>::LOGB, b[1] >> Geo<D>::LOGB, b[2] >> Geo<D>::LOGB};
        int lb[3] = {b[0] & (Geo<D>::B - 1), b[1] & (Geo<D>::B - 1), b[2] & (Geo<D>::B - 1)};
        key = block_lin<D>(p, e, bb);
        int cell = cell_of<D>(lb);
        if (!ok) { atomicOr(flags, FLAG_OUT_OF_DOMAIN); key = e * p.nbe; cell = Geo<D>::CELLS; }
        if (ok && (bb[0] < p.x_lo || bb[0] >= p.x_hi)) {  // f3: a particle outside the subdomain's slab
            atomicOr(flags, FLAG_MIGRATION);
            key = -1;
        }
        keys[i] = key < 0 ? -1 : key * 128 + cell;
    }
    count_key(in && key >= 0, key, bcount);
}

// Exclusive scan of the dense block histogram -> active block list (block-id order),
// starts, block map, scatter cursors; clears the histogram.  One launch over chunks of
// 256 x 4 entries (single-pass scan with decoupled look-back): a CTA takes its chunk index
// from an atomic ticket when it starts, publishes its chunk totals tagged with the launch's
// epoch, then sums the totals of all earlier chunks (integer sums, so the order does not
// matter).  Earlier chunks belong to CTAs that started earlier and never wait on later
// ones, so the look-back makes progress whatever the CTA dispatch order or co-residency
// (MPS, concurrent kernels).  The last CTA to finish (second ticket) resets the chunk ticket
// and advances the epoch for the next launch.
#ifndef MPM_SCAN_PER
#define MPM_SCAN_PER 4
#endif
constexpr int kScanPer = MPM_SCAN_PER;
constexpr int kScanChunk = kT * kScanPer;
__global__ void __launch_bounds__(kT) k_bin_scan(KParams p, int* __restrict__ bcount, int* __restrict__ cursor,
                                                SlotView sl, int2* __restrict__ part, int* flags) {
    pdl_begin();
    __shared__ int s_wt[kW], s_wa[kW];
    __shared__ int s_base[2];
    __shared__ unsigned s_epoch;
    __shared__ int s_chunk;
    unsigned long long* part64 = reinterpret_cast<unsigned long long*>(part);
    // tickets: [0] CTAs finished, [1] chunk indices handed out
    unsigned* ticket = reinterpret_cast<unsigned*>(part64 + gridDim.x + 1);
    const int TB = p.TB, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        s_epoch = ((unsigned)part64[gridDim.x] + 1u) & 0xFFFFu;
        s_chunk = (int)atomicAdd(ticket + 1, 1u);
    }
    __syncthreads();
    const int chunk = s_chunk;
    const int i0 = chunk * kScanChunk + tid * kScanPer;
    int c[kScanPer];
    if (i0 + kScanPer <= TB) {
#pragma unroll
        for (int q = 0; q < kScanPer / 4; ++q) {
            const int4 v = *reinterpret_cast<const int4*>(bcount + i0 + 4 * q);
            c[4 * q] = v.x; c[4 * q + 1] = v.y; c[4 * q + 2] = v.z; c[4 * q + 3] = v.w;
        }
    } else {
#pragma unroll
        for (int q = 0; q < kScanPer; ++q) c[q] = i0 + q < TB ? bcount[i0 + q] : 0;
    }
    int tot = 0, act = 0;
#pragma unroll
    for (int q = 0; q < kScanPer; ++q) { tot += c[q]; act += c[q] > 0; }
    int it = tot, ia = act;  // inclusive warp scan
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int a = __shfl_up_sync(0xffffffffu, it, off), b = __shfl_up_sync(0xffffffffu, ia, off);
        if (lane >= off) { it += a; ia += b; }
    }
    if (lane == 31) { s_wt[warp] = it; s_wa[warp] = ia; }
    {
        __syncthreads();
        const unsigned long long ep = s_epoch;
        if (tid == 0) {  // publish this chunk's totals, tagged with the epoch
            unsigned bt = 0, ba = 0;
            for (int w = 0; w < kW; ++w) { bt += (unsigned)s_wt[w]; ba += (unsigned)s_wa[w]; }
            const unsigned long long v = (ep << 48) | ((unsigned long long)(ba & 0xFFFFu) << 32) | bt;
            atomicExch(part64 + chunk, v);
        }
        if (warp == kW - 1) {  // look back over all earlier chunks
            int bt = 0, ba = 0;
            for (int k = lane; k < chunk; k += 32) {
                unsigned long long v;
                do {
                    v = atomicAdd(part64 + k, 0ull);
                } while ((v >> 48) != ep);
                bt += (int)(unsigned)(v & 0xFFFFFFFFull);
                ba += (int)((v >> 32) & 0xFFFFull);
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                bt += __shfl_xor_sync(0xffffffffu, bt, off);
                ba += __shfl_xor_sync(0xffffffffu, ba, off);
            }
            if (lane == 0) { s_base[0] = bt; s_base[1] = ba; }
        }
    }
    __syncthreads();
    // pool offset of this step: right after the previous step's blocks
    const int b0 = sl.step > 0 ? sl.base[-1] + sl.nactive[-1] : 0;
    int pos = s_base[0] + it - tot, li = s_base[1] + ia - act;
    for (int w = 0; w < warp; ++w) { pos += s_wt[w]; li += s_wa[w]; }
    const int cap = min(p.max_active - b0, p.step_blocks);  // blocks this step may take
#pragma unroll
    for (int q = 0; q < kScanPer; ++q) {
        const int b = i0 + q;
        if (b >= TB) break;
        if (c[q] > 0) {
            if (li < cap) {
                sl.blist[b0 + li] = b;
                sl.bstart[b0 + sl.step + li] = pos;
                sl.bmap[b] = b0 + li;
            } else {
                // capacity exceeded: the list ends before this block (error is reported)
                if (li == cap) sl.bstart[b0 + sl.step + li] = pos;
                sl.bmap[b] = -1;
                atomicOr(flags, FLAG_ACTIVE_OVERFLOW);
            }
            cursor[b] = pos;
            pos += c[q];
            ++li;
            bcount[b] = 0;
        } else {
            sl.bmap[b] = -1;
        }
    }
    if (chunk == (int)gridDim.x - 1 && tid == kT - 1) {  // grand totals
        const int n = max(0, min(li, cap));
        *sl.nactive = n;
        *sl.base = b0;
        *sl.ntot = pos;  // sorted entries of this step
        if (li <= cap) sl.bstart[b0 + sl.step + n] = pos;
    }
    {  // the last CTA to finish advances the epoch for the next launch
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            if (atomicAdd(ticket, 1u) == gridDim.x - 1) {  // every CTA has its chunk by now
                part64[gridDim.x] = s_epoch;
                ticket[1] = 0u;
                ticket[0] = 0u;
            }
        }
    }
}

// stable-free scatter of particle indices by block key (position inside a block is
// arbitrary; p2g canonicalises).  kScatterPer particles per thread, all loads and
// cursor atomics issued before any result is used (memory-level parallelism).
constexpr int kScatterPer = 4;
__global__ void __launch_bounds__(kT) k_bin_scatter(KParams p, const int* __restrict__ keys,
                                                    const int* __restrict__ pid, int* __restrict__ cursor,
                                                    SlotView sl) {
    pdl_begin();
    const int64_t n = p.N * p.E;
    const int lane = threadIdx.x & 31;
    int64_t j[kScatterPer];
    int kc[kScatterPer], pj[kScatterPer], base[kScatterPer];
    unsigned peers[kScatterPer];
#pragma unroll
    for (int u = 0; u < kScatterPer; ++u) {
        j[u] = ((int64_t)blockIdx.x * kScatterPer + u) * kT + threadIdx.x;
        const bool in = j[u] < n;
        kc[u] = in ? __ldg(keys + j[u]) : -1;
        pj[u] = in ? __ldg(pid + j[u]) : 0;
    }
#pragma unroll
    for (int u = 0; u < kScatterPer; ++u) {
        const int key = kc[u] >= 0 ? kc[u] >> 7 : -1;
        peers[u] = __match_any_sync(0xffffffffu, key);
        const int leader = __ffs(peers[u]) - 1;
        base[u] = 0;
        if (kc[u] >= 0 && lane == leader) base[u] = atomicAdd(&cursor[key], __popc(peers[u]));
    }
#pragma unroll
    for (int u = 0; u < kScatterPer; ++u) {
        const int b = __shfl_sync(0xffffffffu, base[u], __ffs(peers[u]) - 1);
        if (kc[u] >= 0) {
            const int pos = b + __popc(peers[u] & ((1u << lane) - 1u));
            sl.sigma[pos] = (int)j[u];
            sl.scell[pos] = (unsigned char)(kc[u] & 127);
            sl.spid[pos] = pj[u];
        }
    }
}

// ----------------------------------------------------- cell accumulation
// thread per tile node: sum the (cell, o) partials with cell + o = node (fixed order)
template <int D>
__device__ __forceinline__ float4 node_gather(const float4* __restrict__ s_cb, int q) {
    using G = Geo<D>;
    int n[3];
    local_node<D>(q, n);
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int o0 = 0; o0 < 3; ++o0)
#pragma unroll
        for (int o1 = 0; o1 < 3; ++o1)
#pragma unroll
            for (int o2 = 0; o2 < (D == 3 ? 3 : 1); ++o2) {
                const int c[3] = {n[0] - o0, n[1] - o1, n[2] - o2};
                bool in = c[0] >= 0 && c[0] < G::B && c[1] >= 0 && c[1] < G::B;
                if (D == 3) in = in && c[2] >= 0 && c[2] < G::B;
                if (!in) continue;
                const int cl = D == 2 ? c[0] * G::B + c[1] : (c[0] * G::B + c[1]) * G::B + c[2];
                const int ol = D == 2 ? o0 * 3 + o1 : (o0 * 3 + o1) * 3 + o2;
                const float4 v = s_cb[cl * G::NST + ol];
                s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
            }
    return s;
}

// Tuning knobs (overridable with -D for A/B builds, tools/build_variant.py)
#ifndef MPM_P2GG_FFMA2
#define MPM_P2GG_FFMA2 0
#endif
#ifndef MPM_P2GG_NESTED
#define MPM_P2GG_NESTED 1
#endif
#ifndef MPM_P2G_CHUNK
#define MPM_P2G_CHUNK 576
#endif
#ifndef MPM_ROW_FFMA2
#define MPM_ROW_FFMA2 1  // U_bar scatter 112.2 -> 109.6 ms per C5 iteration (p2g unchanged)
#endif
#ifndef MPM_GATHER_FFMA2
#define MPM_GATHER_FFMA2 1  // g2p 123.2 -> 121.7 ms per C5 iteration
#endif
#ifndef MPM_G2PG_FFMA2
#define MPM_G2PG_FFMA2 1  // g2p_grad gather 97.8 -> 90.6 ms per C5 iteration
#endif
#ifndef MPM_ROW_ELIDE
#define MPM_ROW_ELIDE 1
#endif
#ifndef MPM_P2G_MINB
#define MPM_P2G_MINB 3
#endif
#ifndef MPM_G2PG_MINB
#define MPM_G2PG_MINB 3
#endif
#ifndef MPM_P2GG_MINB
#define MPM_P2GG_MINB 4
#endif
#ifndef MPM_G2P_THREADS
#define MPM_G2P_THREADS 128
#endif
#ifndef MPM_SCATTER_THREADS
#define MPM_SCATTER_THREADS 192
#endif
constexpr int kACC = 192;  // accumulation phase: 3 threads (o_x) per cell (64 cells)
constexpr int kTQ = MPM_SCATTER_THREADS;  // p2g / g2p_grad CTA (>= kACC; the extra threads help in phases 1, 3)
static_assert(kTQ >= kACC, "scatter CTA smaller than the accumulation phase");
constexpr int kCH = MPM_P2G_CHUNK;  // rows per chunk: most blocks fit one chunk -> all 64 cells busy in phase 2

template <int D> struct RowL {  // particle row in shared memory (floats); stride avoids STS.128 conflicts
    static constexpr int STRIDE = D == 3 ? 28 : 12;
};
// canonical-order scratch (canon_block): the list, particle ids, cells and bucket counters
constexpr int kCanonScratch = 1728 * 15 + 66 * 4;
// p2g / U_bar scatter shared area: the phase-1/2 rows, the node partials, or (p2g for small
// problems) the canonical-order scratch -- whichever is largest
template <int D> constexpr int p2g_union_bytes() {
    constexpr int a = kCanonScratch, b = Geo<D>::CELLS * Geo<D>::NST * 16, c = kCH * RowL<D>::STRIDE * 4;
    return a > b ? (a > c ? a : c) : (b > c ? b : c);
}
template <int D> constexpr int p2g_smem_bytes() {
    return p2g_union_bytes<D>() + Geo<D>::MAXP * 4 + (Geo<D>::CELLS + 2) * 4;
}

// Thread (cell, o_x): sums over the cell's rows W_o (c + A o) (and W_o) for the
// 3^(d-1) nodes o = (o_x, .) in registers.  Row: [wy*wz (9) | c (3) | A dx (9) | wx (3)] (3D),
// [wy (3) | c (2) | A dx (4) | wx (3)] (2D).
// (ax, ay) += w (x, y) as one packed f32x2 FMA (per lane an IEEE fma: bitwise the scalar pair)
__device__ __forceinline__ void fma2(float& ax, float& ay, float w, float x, float y) {
    const float2 r = __ffma2_rn(make_float2(w, w), make_float2(x, y), make_float2(ax, ay));
    ax = r.x;
    ay = r.y;
}

template <int D, bool MASS> struct SliceAcc {
    static constexpr int NN = D == 3 ? 9 : 3;
    float4 a[NN];
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int k = 0; k < NN; ++k) a[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __device__ __forceinline__ void row(const float* __restrict__ rw, int ox) {
        const float4* r4 = reinterpret_cast<const float4*>(rw);
        const float fox = (float)ox;
        if (D == 3 && MPM_ROW_FFMA2) {
            // the same sums with packed (f32x2) FMAs: (x, y) and (z, mass) per node, each lane an
            // IEEE fma as in the scalar form (acc.w + W = fma(W, 1, acc.w)): bitwise identical
            const float4 r0 = r4[0], r1 = r4[1], r2 = r4[2], r3 = r4[3], r4_ = r4[4], r5 = r4[5];
            const float wyz[9] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w, r2.x};
            const float W0 = ox == 0 ? r5.y : (ox == 1 ? r5.z : r5.w);
            // A dx rows: (A[0] A[1] A[2]) = (r3.x r3.y r3.z), (A[3..5]) = (r3.w r4.x r4.y), (A[6..8]) = (r4.z r4.w r5.x)
            const float2 Ay = make_float2(r3.y, r4_.x), Az = make_float2(r3.z, r4_.y);
            const float2 mx = make_float2(fmaf(fox, r3.x, r2.y), fmaf(fox, r3.w, r2.z));
            const float mxz = fmaf(fox, r4_.z, r2.w);
#pragma unroll
            for (int oy = 0; oy < 3; ++oy) {
                const float foy = (float)oy;
                float2 mxy = oy ? __ffma2_rn(make_float2(foy, foy), Ay, mx) : mx;
                float mz = oy ? fmaf(foy, r4_.w, mxz) : mxz;
#pragma unroll
                for (int oz = 0; oz < 3; ++oz) {
                    const float W = W0 * wyz[oy * 3 + oz];
                    const float2 W2 = make_float2(W, W);
                    float4& acc = a[oy * 3 + oz];
                    float2 xy = __ffma2_rn(W2, mxy, make_float2(acc.x, acc.y));
                    acc.x = xy.x; acc.y = xy.y;
                    if (MASS) {
                        float2 zw = __ffma2_rn(W2, make_float2(mz, 1.0f), make_float2(acc.z, acc.w));
                        acc.z = zw.x; acc.w = zw.y;
                    } else {
                        acc.z = fmaf(W, mz, acc.z);
                    }
                    mxy = __fadd2_rn(mxy, Az);
                    mz += r5.x;
                }
            }
        } else if (D == 3) {
            const float4 r0 = r4[0], r1 = r4[1], r2 = r4[2], r3 = r4[3], r4_ = r4[4], r5 = r4[5];
            const float wyz[9] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w, r2.x};
            const float A[9] = {r3.x, r3.y, r3.z, r3.w, r4_.x, r4_.y, r4_.z, r4_.w, r5.x};
            const float W0 = ox == 0 ? r5.y : (ox == 1 ? r5.z : r5.w);
            float mx[3] = {fmaf(fox, A[0], r2.y), fmaf(fox, A[3], r2.z), fmaf(fox, A[6], r2.w)};
#pragma unroll
            for (int oy = 0; oy < 3; ++oy) {
                // MPM_ROW_ELIDE: oy = 0: m = mx exactly (fmaf(0, a, b) = b for finite a), without the instructions
                const bool el = MPM_ROW_ELIDE && oy == 0;
                float m[3] = {el ? mx[0] : fmaf((float)oy, A[1], mx[0]), el ? mx[1] : fmaf((float)oy, A[4], mx[1]),
                              el ? mx[2] : fmaf((float)oy, A[7], mx[2])};
#pragma unroll
                for (int oz = 0; oz < 3; ++oz) {
                    const float W = W0 * wyz[oy * 3 + oz];
                    float4& acc = a[oy * 3 + oz];
                    acc.x = fmaf(W, m[0], acc.x);
                    acc.y = fmaf(W, m[1], acc.y);
                    acc.z = fmaf(W, m[2], acc.z);
                    if (MASS) acc.w += W;
                    m[0] += A[2]; m[1] += A[5]; m[2] += A[8];
                }
            }
        } else {
            const float4 r0 = r4[0], r1 = r4[1];
            // [wy0 wy1 wy2 c0][c1 A00 A01 A10][A11 wx0 wx1 wx2]
            const float r2x = rw[8];
            const float W0 = rw[9 + ox];
            const float wy[3] = {r0.x, r0.y, r0.z};
            float m[2] = {fmaf(fox, r1.y, r0.w), fmaf(fox, r1.w, r1.x)};
#pragma unroll
            for (int oy = 0; oy < 3; ++oy) {
                const float W = W0 * wy[oy];
                float4& acc = a[oy];
                acc.x = fmaf(W, m[0], acc.x);
                acc.y = fmaf(W, m[1], acc.y);
                if (MASS) acc.w += W;
                m[0] += r1.z; m[1] += r2x;
            }
        }
    }
    // cellbuf[c][o], o = (ox*3 + oy)*3 + oz (3D) / ox*3 + oy (2D)
    __device__ __forceinline__ void store(float4* cellbuf, int c, int ox) const {
        float4* dst = cellbuf + c * Geo<D>::NST + ox * NN;
#pragma unroll
        for (int k = 0; k < NN; ++k) dst[k] = a[k];
    }
};

// row writer (vector stores): layouts as SliceAcc::row
template <int D>
__device__ __forceinline__ void write_row(float* row, const float w[3][3], const float* c, const float* Adx) {
    float4* r4 = reinterpret_cast<float4*>(row);
    if (D == 3) {
        float wyz[9];
#pragma unroll
        for (int oy = 0; oy < 3; ++oy)
#pragma unroll
            for (int oz = 0; oz < 3; ++oz) wyz[oy * 3 + oz] = w[1][oy] * w[2][oz];
        r4[0] = make_float4(wyz[0], wyz[1], wyz[2], wyz[3]);
        r4[1] = make_float4(wyz[4], wyz[5], wyz[6], wyz[7]);
        r4[2] = make_float4(wyz[8], c[0], c[1], c[2]);
        r4[3] = make_float4(Adx[0], Adx[1], Adx[2], Adx[3]);
        r4[4] = make_float4(Adx[4], Adx[5], Adx[6], Adx[7]);
        r4[5] = make_float4(Adx[8], w[0][0], w[0][1], w[0][2]);
    } else {
        r4[0] = make_float4(w[1][0], w[1][1], w[1][2], c[0]);
        r4[1] = make_float4(c[1], Adx[0], Adx[1], Adx[2]);
        r4[2] = make_float4(Adx[3], w[0][0], w[0][1], w[0][2]);
    }
}

// per-particle p2g math: returns c = m v - A dx f and A dx (for NodeAcc) and Ft
template <int D>
__device__ __forceinline__ bool p2g_particle(const KParams& p, const float* x, const float* vc, const float* F,
                                             float act, bool fluid, const int c0[3], float w[3][3], float* c,
                                             float* Adx, float* Ft) {
    const float* v = vc;
    const float* C = vc + D;
    int lb[3];
    float fx[3], dw[3][3];
    particle_weights<D>(p, x, c0, lb, fx, w, dw);
    deform_update<D>(p.dt, C, F, Ft);
    float tau[D * D];
    const bool ok = kirchhoff<D>(p, Ft, act, tau, fluid);
#pragma unroll
    for (int q = 0; q < D * D; ++q) Adx[q] = p.dx * fmaf(p.stress_scale, tau[q], p.p_mass * C[q]);
#pragma unroll
    for (int a = 0; a < D; ++a) {
        float s = p.p_mass * v[a];
#pragma unroll
        for (int b = 0; b < D; ++b) s = fmaf(-Adx[a * D + b], fx[b], s);
        c[a] = s;
    }
    return ok;
}

// ------------------------------------------------------------ canonical order
// Per active block: put the scattered list in canonical (cell, particle id) order, so every
// sum downstream has a fixed order (bitwise reproducible, independent of the scatter's
// atomics).  Bucket by cell (warp-aggregated smem counters), then rank by particle id
// inside the cell.  Writes sigma (canonical), the cell starts and -- when the step writes
// S_{t+1} -- the particle ids of S_{t+1} (p2g's output order).  Its own high-occupancy
// pass (256 threads, 26 KB smem) ahead of p2g.
// One block's list in canonical order (NT threads, all calling).  scratch: 26,184 B of shared
// memory (list, particle ids, cells, bucket counters); s_cst [CELLS + 2] receives the cell
// starts; s_ci (nullable) the canonical list.  Writes sigma (canonical), the cell starts and
// the particle ids of S_{t+1} (pid_next, nullable).  Returns false for a dropped block (over
// MAXP particles: reported, its rows' next bin keys marked invalid).  Ends with a barrier.
template <int NT>
__device__ __forceinline__ bool canon_block(const SlotView& sl, int bi, int start, int n, unsigned short* cstart,
                                            int* __restrict__ pid_next, int* __restrict__ keys_next, int* flags,
                                            unsigned char* scratch, int* s_cst, int* s_ci) {
    constexpr int MAXP = 1728, CELLS = 64;
    int* s_idx = reinterpret_cast<int*>(scratch);
    int* s_pid = s_idx + MAXP;
    int* s_bpid = s_pid + MAXP;
    int* s_cnt = s_bpid + MAXP;
    short* s_tmp = reinterpret_cast<short*>(s_cnt + CELLS + 2);
    unsigned char* s_cell = reinterpret_cast<unsigned char*>(s_tmp + MAXP);
    const int tid = threadIdx.x, lane = tid & 31;
    if (n > MAXP) {  // reported; the block is dropped (no valid entries downstream)
        if (tid == 0) atomicOr(flags, FLAG_BLOCK_OVERFLOW);
        for (int c = tid; c <= CELLS; c += NT) cstart[(int64_t)bi * (CELLS + 1) + c] = 0;
        // g2p writes no bin key for the dropped rows of S_{t+1}: mark them so the next
        // binning skips them instead of scattering stale keys
        if (keys_next)
            for (int q = tid; q < n; q += NT) keys_next[start + q] = -1;
        __syncthreads();
        return false;
    }
    // ---- canonical (cell, particle id) order of the block's list.  The scatter wrote each
    // entry's cell and particle id next to it: coalesced loads only.
    for (int q = tid; q < CELLS + 2; q += NT) s_cnt[q] = 0;
#pragma unroll 4
    for (int q = tid; q < n; q += NT) {
        s_idx[q] = sl.sigma[start + q];
        s_pid[q] = sl.spid[start + q];
        s_cell[q] = sl.scell[start + q];
    }
    __syncthreads();
    for (int q0 = 0; q0 < n; q0 += NT) {
        const int q = q0 + tid;
        const bool in = q < n;
        const int cell = in ? (int)s_cell[q] : -1;
        const unsigned peers = __match_any_sync(0xffffffffu, cell);
        if (in && lane == __ffs(peers) - 1) atomicAdd(&s_cnt[cell], __popc(peers));
    }
    __syncthreads();
    if (tid < 32) {  // exclusive scan of the 65 bucket counts (one warp)
        int carry = 0;
        for (int c = lane; c - lane <= CELLS; c += 32) {
            const int v = c <= CELLS ? s_cnt[c] : 0;
            int inc = v;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, inc, off);
                if (lane >= off) inc += t;
            }
            if (c <= CELLS) { s_cst[c] = carry + inc - v; s_cnt[c] = carry + inc - v; }
            carry += __shfl_sync(0xffffffffu, inc, 31);
        }
        if (lane == 0) s_cst[CELLS + 1] = carry;
    }
    __syncthreads();
    for (int q0 = 0; q0 < n; q0 += NT) {  // bucket by cell (order inside a cell arbitrary)
        const int q = q0 + tid;
        const bool in = q < n;
        const int cell = in ? (int)s_cell[q] : -1;
        const unsigned peers = __match_any_sync(0xffffffffu, cell);
        const int leader = __ffs(peers) - 1;
        int base = 0;
        if (in && lane == leader) base = atomicAdd(&s_cnt[cell], __popc(peers));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (in) {
            const int pos = base + __popc(peers & ((1u << lane) - 1u));
            s_tmp[pos] = (short)q;
            s_bpid[pos] = s_pid[q];
        }
    }
    __syncthreads();
    for (int r = tid; r < n; r += NT) {  // rank by particle id inside the cell
        const int q = s_tmp[r];
        const int cell = s_cell[q], pq = s_bpid[r];
        int rank = 0;
        const int m1 = s_cst[cell + 1];
        for (int m = s_cst[cell]; m < m1; ++m) rank += s_bpid[m] < pq;
        const int fl = s_cst[cell] + rank;
        sl.sigma[start + fl] = s_idx[q];
        if (s_ci) s_ci[fl] = s_idx[q];
        if (pid_next) pid_next[start + fl] = pq;
    }
    for (int c = tid; c <= CELLS; c += NT) cstart[(int64_t)bi * (CELLS + 1) + c] = (unsigned short)s_cst[c];
    if (tid == 0 && s_cst[CELLS] != n) atomicOr(flags, FLAG_OUT_OF_DOMAIN);  // junk entries
    __syncthreads();
    return true;
}

constexpr int canon_smem_bytes() { return kCanonScratch + 66 * 4; }
static_assert(p2g_union_bytes<2>() >= kCanonScratch && p2g_union_bytes<3>() >= kCanonScratch,
              "p2g's row area holds the canonical-order scratch (MPM_CANON_IN_P2G)");
__global__ void __launch_bounds__(kT) k_canon(KParams p, SlotView sl, int* __restrict__ pid_next,
                                              int* __restrict__ keys_next, int* flags) {
    pdl_begin();
    extern __shared__ __align__(16) unsigned char smem[];
    int* s_cst = reinterpret_cast<int*>(smem + kCanonScratch);
    const int nact = *sl.nactive;
    const int b0 = *sl.base;
    const int* bstart = sl.bstart + b0 + sl.step;
    unsigned short* cstart = sl.cstart + (int64_t)b0 * (Geo<3>::CELLS + 1);
    for (int bi = blockIdx.x; bi < nact; bi += gridDim.x) {
        const int start = bstart[bi], n = bstart[bi + 1] - start;
        canon_block<kT>(sl, bi, start, n, cstart, pid_next, keys_next, flags, smem, s_cst, nullptr);
    }
    (void)p;
}

// ---------------------------------------------------------------- P2G
// p2g: canonicalise the block list, then per particle
// Ft = (I + dt C) F; tau = tau(Ft) [+ actuation]; A = -dt V 4/dx^2 tau + m C;
// node b+o receives W_o (m v + A (o - f) dx) and W_o m.  F_{t+1} = Ft.
// CTA = 192 threads: phase 1 thread per particle (rows in smem), phase 2 thread per (cell, o_x).
// CANON: p2g puts each block's list in canonical order itself (no k_canon pass); used for
// small problems (canon_fused), where one kernel fewer per step pays (C2 +4%), while at C5 the
// ordering costs more inside p2g (18 warps per SM) than as its own pass (64 warps per SM)
template <int D, bool CANON>
__global__ void __launch_bounds__(kTQ, MPM_P2G_MINB) k_p2g(KParams p, SlotView sl, StateView S, StateView Sn,
                                               const int32_t* __restrict__ aid,
                                               const float* __restrict__ alpha, int* keys_next, int* flags) {
    pdl_begin();
    using G = Geo<D>;
    using L = Lay<D>;
    constexpr int RS = RowL<D>::STRIDE;
    extern __shared__ __align__(16) unsigned char smem[];
    float* s_row = reinterpret_cast<float*>(smem);                   // phase 1/2 rows ...
    float4* s_cb = reinterpret_cast<float4*>(smem);                  // ... node partials
    int* s_ci = reinterpret_cast<int*>(smem + p2g_union_bytes<D>());  // canonical state index
    int* s_cst = s_ci + G::MAXP;  // [CELLS + 1] cell starts
    const int tid = threadIdx.x, lane = tid & 31;
    const int my_cell = tid / 3, my_ox = tid - 3 * (tid / 3);
    const int nact = *sl.nactive;
    const int b0 = *sl.base;  // this step's offset in the grid-store pool
    const int* blist = sl.blist + b0;
    const int* bstart = sl.bstart + b0 + sl.step;
    unsigned short* cstart = sl.cstart + (int64_t)b0 * (G::CELLS + 1);
    float4* tiles_l = sl.part;  // partial tiles of this step (local block index)
    for (int bi = blockIdx.x; bi < nact; bi += gridDim.x) {
        const int bid = blist[bi];
        const int start = bstart[bi], n = bstart[bi + 1] - start;
        int e, c0[3];
        block_origin<D>(p, bid, e, c0);
        // (the next block's list by cp.async.bulk during this block -- two list buffers, 544-row
        // chunks to keep three CTAs per SM -- measured slower: 182.7 -> 191.6 ms per C5 iteration)
        if (CANON) {
            fill_nbr<D>(p, sl, b0, bi, tid);
            // the canonical order of the block's list, in the row area (not live yet)
            if (!canon_block<kTQ>(sl, bi, start, n, cstart, Sn.pid, keys_next, flags, smem, s_cst, s_ci)) continue;
        } else {
            if (n > G::MAXP) {
                if (tid == 0) atomicOr(flags, FLAG_BLOCK_OVERFLOW);
                continue;
            }
            // ---- the block's list in canonical (cell, particle id) order (k_canon)
            for (int q = tid; q < n; q += kTQ) s_ci[q] = sl.sigma[start + q];
            for (int c = tid; c <= G::CELLS; c += kTQ) s_cst[c] = cstart[(int64_t)bi * (G::CELLS + 1) + c];
            __syncthreads();
        }
        const int nvalid = s_cst[G::CELLS];
        // ---- phases 1 + 2 over chunks of kTQ particles in canonical order; the particle
        // loads of chunk k+1 are issued before the accumulation of chunk k (same registers)
        SliceAcc<D, true> acc;
        acc.zero();
        // a thread's particle inputs (loading the next particle's before the current particle's
        // math, a second register set, spills at the 96-register cap: measured slower)
        struct In {
            float x[3], vc[L::VC], F[L::FF];
            int a_id;
            bool fluid;
        };
        auto load = [&](In& d, int R) {
            const int i_ = s_ci[R];
            load_comps<L::X>(S.x, i_, d.x);
            load_comps<L::VC>(S.vc, i_, d.vc);
            load_comps<L::FF>(S.f, i_, d.F);
            d.a_id = -1;
            d.fluid = false;
            if (aid || p.mat) {
                const int pd_ = __ldg(S.pid + i_);
                if (aid) d.a_id = __ldg(aid + pd_);
                if (p.mat) d.fluid = __ldg(p.mat + pd_) != 0;
            }
        };
        In cur;
        if (tid < nvalid) load(cur, tid);
        for (int ch = 0; ch < nvalid; ch += kCH) {
            const int cend = min(nvalid, ch + kCH);
            for (int r = ch + tid; r < cend; r += kTQ) {  // data of r is in registers
                const bool more = r + kTQ < nvalid;
                // ids outside [0, n_act) are passive here (mpm_set_state flags them as an error)
                const int a_id = cur.a_id;
                const bool fluid = cur.fluid;
                const float act = (aid && a_id >= 0 && a_id < p.n_act) ? alpha[e * p.a_estride + a_id] : 0.0f;
                float w[3][3], c[3], Adx[D * D], Ft[D * D];
                if (!p2g_particle<D>(p, cur.x, cur.vc, cur.F, act, fluid, c0, w, c, Adx, Ft))
                    atomicOr(flags, FLAG_NONFINITE);
                write_row<D>(s_row + (r - ch) * RS, w, c, Adx);
                if (Sn.f) {
                    if (fluid) fluid_reset<D>(Ft, Ft);  // R23 (Ft is dead after the row)
                    store_comps<L::FF>(Sn.f, start + r, Ft);
                }
                if (more) load(cur, r + kTQ);  // this thread's next particle
            }
            __syncthreads();
            if (tid < kACC) {
                const int lo = max(s_cst[my_cell], ch), hi = min(s_cst[my_cell + 1], cend);
                for (int rr = lo; rr < hi; ++rr) acc.row(s_row + (rr - ch) * RS, my_ox);
            }
            __syncthreads();
        }
        if (tid < kACC) acc.store(s_cb, my_cell, my_ox);  // the rows are dead after the last barrier
        __syncthreads();
        // ---- phase 3: node tile (plain stores)
        float4* tile = tiles_l + (int64_t)bi * G::TN;
        for (int q = tid; q < G::TN; q += kTQ) {
            float4 s4 = node_gather<D>(s_cb, q);
            s4.w *= p.p_mass;
            tile[q] = s4;
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------- grid_op
// P:579 (R5-R7): thread per node of every active block's (B+2)^d tile:
// (P, M) = sum of the covering partial tiles; u1 = P/(M + eps) - dt g e_y; sticky walls.
// Resolved tile entry: (u1, M), or (0, 0, 0, -M) where the wall zeroed the velocity
// (sign bit set, also for M = 0: -0.0f; nodes outside the grid: (0, 0, 0, -0)).  Stored per step: g2p / g2p_grad / grid_op_grad read it.
template <int D, bool HALO, bool NBR = false>  // NBR: covering tiles from the neighbour table
__global__ void __launch_bounds__(kT) k_grid_op(KParams p, SlotView sl) {
    pdl_begin();
    using G = Geo<D>;
    const int nact = *sl.nactive;
    const int b0 = *sl.base;
    const int* blist = sl.blist + b0;
    const float4* part_g = sl.part - (int64_t)b0 * G::TN;  // bmap holds pool indices
    float4* rt = sl.tiles + (int64_t)b0 * G::TN;
    // 32-bit node index: a step's tiles (nact * TN float4) are far below 2^32 nodes in HBM
    const unsigned total = (unsigned)nact * G::TN;
    const float4* nt0 = halo_tiles<D>(sl.halo, 0);
    const float4* nt1 = halo_tiles<D>(sl.halo, 1);
    for (unsigned idx = blockIdx.x * kT + threadIdx.x; idx < total; idx += gridDim.x * kT) {
        const int bi = (int)(idx / G::TN), q = (int)(idx - (unsigned)bi * G::TN);
        int e, c0[3], n[3];
        block_origin<D, true>(p, __ldg(blist + bi), e, c0);
        local_node<D>(q, n);
        const int g[3] = {c0[0] + n[0], c0[1] + n[1], D == 3 ? c0[2] + n[2] : 0};
        const bool inside = g[0] < p.n_grid && g[1] < p.n_grid && (D == 2 || g[2] < p.n_grid);
        float4 out = make_float4(0.f, 0.f, 0.f, -0.0f);
        if (inside) {
            const float4 pm = (!HALO && NBR)
                                  ? covered_sum_nbr<D>(sl.nbr + (int64_t)(b0 + bi) * kNbr<D>, n, part_g)
                                  : covered_sum<D, HALO>(p, e, g, sl.bmap, part_g, sl.halo, nt0, nt1);
            float u0[3], u1[3];
            out = grid_velocity<D>(p, g, pm, u0, u1) ? make_float4(0.f, 0.f, 0.f, -pm.w)
                                                      : make_float4(u1[0], u1[1], u1[2], pm.w);
        }
        rt[idx] = out;
    }
}

// --------------------------------------------------------- grid_op_grad
// P:589 (select rule): per node, ub = sum of the covering U_bar partial tiles;
// sticky (sign bit of w): Pb = Mb = 0; else u0 = u1 + dt g e_y, Pb = ub/(M + eps),
// Mb = -(ub . u0)/(M + eps).  Output tile (Pb, Mb) -> sl.part (local block index).
template <int D, bool HALO, bool NBR = false>
__global__ void __launch_bounds__(kT) k_grid_op_grad(KParams p, SlotView sl, const float4* __restrict__ ubar) {
    pdl_begin();
    using G = Geo<D>;
    const int nact = *sl.nactive;
    const int b0 = *sl.base;
    const int* blist = sl.blist + b0;
    const float4* ub_g = ubar - (int64_t)b0 * G::TN;
    const float4* rt = sl.tiles + (int64_t)b0 * G::TN;
    const unsigned total = (unsigned)nact * G::TN;  // 32-bit node index (as grid_op)
    const float4* nt0 = halo_tiles<D>(sl.halo, 0);
    const float4* nt1 = halo_tiles<D>(sl.halo, 1);
    for (unsigned idx = blockIdx.x * kT + threadIdx.x; idx < total; idx += gridDim.x * kT) {
        const float4 r = __ldg(rt + idx);
        float4 out = make_float4(0.f, 0.f, 0.f, 0.f);
        if (!signbit(r.w)) {
            const int bi = (int)(idx / G::TN), q = (int)(idx - (unsigned)bi * G::TN);
            int e, c0[3], n[3];
            block_origin<D, true>(p, __ldg(blist + bi), e, c0);
            local_node<D>(q, n);
            const int g[3] = {c0[0] + n[0], c0[1] + n[1], D == 3 ? c0[2] + n[2] : 0};
            const float4 ub = (!HALO && NBR)
                                  ? covered_sum_nbr<D>(sl.nbr + (int64_t)(b0 + bi) * kNbr<D>, n, ub_g)
                                  : covered_sum<D, HALO>(p, e, g, sl.bmap, ub_g, sl.halo, nt0, nt1);
            const float u0[3] = {r.x, r.y + p.dt * p.gravity, r.z};
            const float denom = r.w + p.eps_mass;
            const float dot = ub.x * u0[0] + ub.y * u0[1] + (D == 3 ? ub.z * u0[2] : 0.0f);
            out = make_float4(ub.x / denom, ub.y / denom, D == 3 ? ub.z / denom : 0.0f, -dot / denom);
        }
        sl.part[idx] = out;
    }
}

// nested separable gather: S0 = sum W U, Sb[b] = sum W U o_b (first moments)
template <int D>
__device__ __forceinline__ void gather_moments(const float4* __restrict__ sU, const int lb[3],
                                               const float w[3][3], float S0[3], float Sb[3][3]) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        S0[a] = 0.f;
        Sb[0][a] = Sb[1][a] = Sb[2][a] = 0.f;
    }
#pragma unroll
    for (int ox = 0; ox < 3; ++ox) {
        float u0[3] = {0.f, 0.f, 0.f}, uy[3] = {0.f, 0.f, 0.f}, uz[3] = {0.f, 0.f, 0.f};
#pragma unroll
        for (int oy = 0; oy < 3; ++oy) {
            float t0[3] = {0.f, 0.f, 0.f}, tz[3] = {0.f, 0.f, 0.f};
            if (D == 3) {
#pragma unroll
                for (int oz = 0; oz < 3; ++oz) {
                    const float4 U = sU[tile_lin<D>(lb[0] + ox, lb[1] + oy, lb[2] + oz)];
                    const float wz = w[2][oz];
                    if (MPM_GATHER_FFMA2) fma2(t0[0], t0[1], wz, U.x, U.y);
                    else { t0[0] = fmaf(wz, U.x, t0[0]); t0[1] = fmaf(wz, U.y, t0[1]); }
                    t0[2] = fmaf(wz, U.z, t0[2]);
                    if (oz) {
                        const float wzo = wz * (float)oz;
                        if (MPM_GATHER_FFMA2) fma2(tz[0], tz[1], wzo, U.x, U.y);
                        else { tz[0] = fmaf(wzo, U.x, tz[0]); tz[1] = fmaf(wzo, U.y, tz[1]); }
                        tz[2] = fmaf(wzo, U.z, tz[2]);
                    }
                }
            } else {
                const float4 U = sU[tile_lin<D>(lb[0] + ox, lb[1] + oy, 0)];
                t0[0] = U.x; t0[1] = U.y;
            }
            const float wy = w[1][oy];
            if (D == 3 && MPM_GATHER_FFMA2) {
                const float wyo = wy * (float)oy;
                fma2(u0[0], u0[1], wy, t0[0], t0[1]);
                u0[2] = fmaf(wy, t0[2], u0[2]);
                fma2(uz[0], uz[1], wy, tz[0], tz[1]);
                uz[2] = fmaf(wy, tz[2], uz[2]);
                if (oy) {
                    fma2(uy[0], uy[1], wyo, t0[0], t0[1]);
                    uy[2] = fmaf(wyo, t0[2], uy[2]);
                }
            } else {
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    u0[a] = fmaf(wy, t0[a], u0[a]);
                    if (D == 3) uz[a] = fmaf(wy, tz[a], uz[a]);
                    if (oy) uy[a] = fmaf(wy * (float)oy, t0[a], uy[a]);
                }
            }
        }
        const float wx = w[0][ox];
#pragma unroll
        for (int a = 0; a < D; ++a) {
            S0[a] = fmaf(wx, u0[a], S0[a]);
            Sb[1][a] = fmaf(wx, uy[a], Sb[1][a]);
            if (D == 3) Sb[2][a] = fmaf(wx, uz[a], Sb[2][a]);
            if (ox) Sb[0][a] = fmaf(wx * (float)ox, u0[a], Sb[0][a]);
        }
    }
}

// ----------------------------------------------------------------- G2P
constexpr int kTG = MPM_G2P_THREADS;  // g2p CTA: smaller CTAs -> more independent blocks in flight per SM
// v' = sum W U; C' = 4/dx sum W U (o - f)^T = 4/dx (Sb - v' f^T); x' = x + dt v'
template <int D>
__device__ __forceinline__ int g2p_particle(const KParams& p, const float4* __restrict__ sU, const float* x,
                                            const int c0[3], int j, int e, int bid, const StateView& Sn,
                                            int* __restrict__ keys, int* flags, bool refwd,
                                            const StateView& S, int64_t i, const Migr& mg) {
    using G = Geo<D>;
    using L = Lay<D>;
    const float c4 = 4.0f * p.inv_dx;
    int lb[3];
    float fx[3], w[3][3], dw[3][3];
    particle_weights<D>(p, x, c0, lb, fx, w, dw);
    float S0[3], Sb[3][3];
    gather_moments<D>(sU, lb, w, S0, Sb);
    float xn[3], vcn[L::VC];
    bool fin = true;
#pragma unroll
    for (int a = 0; a < D; ++a) {
        xn[a] = fmaf(p.dt, S0[a], x[a]);
        vcn[a] = S0[a];
        fin = fin && isfinite(S0[a]);
#pragma unroll
        for (int b = 0; b < D; ++b) vcn[D + a * D + b] = c4 * fmaf(-S0[a], fx[b], Sb[b][a]);
    }
    store_comps<L::X>(Sn.x, j, xn);
    store_comps<L::VC>(Sn.vc, j, vcn);
    if (!fin) atomicOr(flags, FLAG_NONFINITE);
    if (refwd) {  // re-forward from stored tiles: F_{t+1} and the particle id too
        float vc[L::VC], F[D * D], Ft[D * D];
        load_comps<L::VC>(S.vc, i, vc);
        load_comps<L::FF>(S.f, i, F);
        deform_update<D>(p.dt, vc + D, F, Ft);
        const int pd = __ldg(S.pid + i);
        if (p.mat && __ldg(p.mat + pd) != 0) fluid_reset<D>(Ft, Ft);  // R23
        store_comps<L::FF>(Sn.f, j, Ft);
        Sn.pid[j] = pd;
    }
    int key = -1;
    if (keys) {
        int b[3];
        int cell = G::CELLS;
        if (base_cell<D>(p, xn, b)) {
            int bb[3] = {b[0] >> G::LOGB, b[1] >> G::LOGB, b[2] >> G::LOGB};
            int lc[3] = {b[0] & (G::B - 1), b[1] & (G::B - 1), b[2] & (G::B - 1)};
            key = block_lin<D>(p, e, bb);
            cell = cell_of<D>(lc);
            if (mg.cnt && (bb[0] < mg.x_lo || bb[0] >= mg.x_hi)) {  // f3: leaves the slab
                const int dir = bb[0] < mg.x_lo ? 0 : 1;
                const int slot = atomicAdd(mg.cnt + dir, 1);
                if (slot < mg.cap) mg.rows[dir * mg.cap + slot] = j;
                else atomicOr(flags, FLAG_MIGRATION);
                keys[j] = -1;
                return -1;
            }
        } else {
            atomicOr(flags, FLAG_OUT_OF_DOMAIN);
            key = bid;  // p2g of the next step drops it into the junk bucket
        }
        keys[j] = key * 128 + cell;
    }
    return key;
}

// NOTE: the forward and the segment re-forward MUST run this same compiled kernel (refwd is a
// runtime flag, not a template parameter): two instantiations may contract the FMAs of the
// shared math differently, and the re-forwarded S_{t+1} would then differ in the last bit
// from the forward's (checkpoint invariance is tested bitwise).
// (no minimum-CTA bound: with __launch_bounds__(kTG, 1) ptxas takes ~125 registers and g2p
// runs 15% slower; the default heuristic settles at 72-80)
template <int D, bool SPLIT>
__global__ void __launch_bounds__(kTG) k_g2p(KParams p, SlotView sl, StateView S, StateView Sn,
                                            int* __restrict__ keys, int* __restrict__ bcount, int* flags,
                                            bool refwd, Migr mg) {
    pdl_begin();
    using G = Geo<D>;
    __shared__ __align__(128) float4 s_buf[2 * G::TN];
    __shared__ __align__(16) int s_sig[2 * kSigCap];
    __shared__ __align__(8) uint64_t s_bar[2];
    const int tid = threadIdx.x;
    const int nact = *sl.nactive;
    const int b0 = *sl.base;  // this step's offset in the grid-store pool
    const int* blist = sl.blist + b0;
    const int* bstart = sl.bstart + b0 + sl.step;
    unsigned short* cstart = sl.cstart + (int64_t)b0 * (Geo<D>::CELLS + 1);
    const float4* rt = sl.tiles + (int64_t)b0 * Geo<D>::TN;
    SigPipe<D> pipe{s_buf, s_bar, s_sig, sl.sigma, bstart};
    pipe.init();
    __syncthreads();
    const int split = SPLIT ? item_split(nact, gridDim.x) : 1, nitems = nact * split;
    pipe.start(rt, blockIdx.x / split, nact);
    int it = 0;
    for (int w = blockIdx.x; w < nitems; w += gridDim.x, ++it) {
        const int bi = w / split;
        pipe.next(rt, (w + gridDim.x) / split, nact, it);
        const int bid = blist[bi];
        const int start = bstart[bi];
        const int nvalid = cstart[(int64_t)bi * (G::CELLS + 1) + G::CELLS];
        int rb, re;
        if (SPLIT) item_range<kTG>(nvalid, w - bi * split, split, rb, re);
        else { rb = 0; re = nvalid; }
        int e, c0[3];
        block_origin<D>(p, bid, e, c0);
        // the tile and the block's sigma segment arrive together; the particle loads of the
        // first two passes go out before any math
        const float4* sU = pipe.wait(it);
        const int* sg = pipe.sig_at(it, start);
        float xa[3], xb[3];
        const bool va = rb + tid < re, vb = rb + tid + kTG < re;
        int ia = 0, ib = 0;
        if (va) {
            ia = sg[rb + tid];
            load_comps<Lay<D>::X>(S.x, ia, xa);
        }
        if (vb) {
            ib = sg[rb + tid + kTG];
            load_comps<Lay<D>::X>(S.x, ib, xb);
        }
        int key = -1;
        if (va) key = g2p_particle<D>(p, sU, xa, c0, start + rb + tid, e, bid, Sn, keys, flags, refwd, S, ia, mg);
        if (keys) count_key(va && key >= 0, key, bcount);
        key = -1;
        if (vb) key = g2p_particle<D>(p, sU, xb, c0, start + rb + tid + kTG, e, bid, Sn, keys, flags, refwd, S, ib, mg);
        if (keys) count_key(vb && key >= 0, key, bcount);
        for (int r0 = rb + 2 * kTG; r0 < re; r0 += kTG) {
            const int r = r0 + tid;
            const bool in = r < re;
            key = -1;
            if (in) {
                const int i = sg[r];
                float x[3];
                load_comps<Lay<D>::X>(S.x, i, x);
                key = g2p_particle<D>(p, sU, x, c0, start + r, e, bid, Sn, keys, flags, refwd, S, i, mg);
            }
            if (keys) count_key(in && key >= 0, key, bcount);
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------ g2p_grad
// vh = vb' + dt xb';  Ub[b+o] += W (vh + 4/dx Cb' (o - f))  (the scatter part; the gather
// part Wb = U.(vh + 4/dx Cb'(o - f)), fb += Wb dW/df - 4/dx W Cb'^T U, xb_t = xb' + fb/dx
// runs in p2g_grad's pass over the same block, g2pg_gather).
// CTA = 192 threads: phase 1 thread per particle (rows in smem), phase 2 thread per
// (cell, o_x) accumulating U_bar like p2g's momentum.
template <int D> constexpr int g2pg_union_bytes() {
    constexpr int a = Geo<D>::CELLS * Geo<D>::NST * 16, c = kCH * RowL<D>::STRIDE * 4;
    return a > c ? a : c;
}
template <int D> constexpr int g2pg_smem_bytes() { return g2pg_union_bytes<D>() + (Geo<D>::CELLS + 2) * 4; }

// per-particle row inputs of the U_bar scatter: vh = vb' + dt xb'; B = 4/dx Cb';
// c' = vh - B f (weights in w)
template <int D>
__device__ __forceinline__ void g2pg_row(const KParams& p, const float* x, const float* xb, const float* vbn,
                                         const float* Cbn, const int c0[3], float w[3][3], float* cp, float* B) {
    const float c4 = 4.0f * p.inv_dx;
    float vh[3];
#pragma unroll
    for (int a = 0; a < D; ++a) vh[a] = fmaf(p.dt, xb[a], vbn[a]);
#pragma unroll
    for (int q = 0; q < D * D; ++q) B[q] = c4 * Cbn[q];
    int lb[3];
    float fx[3], dw[3][3];
    particle_weights<D>(p, x, c0, lb, fx, w, dw);
#pragma unroll
    for (int a = 0; a < D; ++a) {
        float s = vh[a];
#pragma unroll
        for (int b = 0; b < D; ++b) s = fmaf(-B[a * D + b], fx[b], s);
        cp[a] = s;
    }
}

// g2p_grad's gather part, evaluated inside p2g_grad's pass over the same step-t
// block (same binning, same weights): Wb_o = U_o . (vh + B (o - f));
// fb = sum_o Wb_o grad W_o - B^T sum_o W_o U_o;  returns xb_t (partial) = xb' + fb/dx.
template <int D>
__device__ __forceinline__ void g2pg_gather(const KParams& p, const float4* __restrict__ sU, const int lb[3],
                                            const float fx[3], const float w[3][3], const float dw[3][3],
                                            const float* xb, const float* vbn, const float* Cbn,
                                            float* xbp_out) {
    const float c4 = 4.0f * p.inv_dx;
    float vh[3], B[D * D], cp[3];
#pragma unroll
    for (int a = 0; a < D; ++a) vh[a] = fmaf(p.dt, xb[a], vbn[a]);
#pragma unroll
    for (int q = 0; q < D * D; ++q) B[q] = c4 * Cbn[q];
#pragma unroll
    for (int a = 0; a < D; ++a) {
        float s = vh[a];
#pragma unroll
        for (int b = 0; b < D; ++b) s = fmaf(-B[a * D + b], fx[b], s);
        cp[a] = s;
    }
    float fb[3] = {0.f, 0.f, 0.f}, S0[3] = {0.f, 0.f, 0.f};
#pragma unroll 1
    for (int o0 = 0; o0 < 3; ++o0) {  // rolled: keeps 9 (not 27) node loads in flight
        const float w0 = o0 == 0 ? w[0][0] : (o0 == 1 ? w[0][1] : w[0][2]);
        const float d0 = o0 == 0 ? dw[0][0] : (o0 == 1 ? dw[0][1] : dw[0][2]);
        float tx[3];
#pragma unroll
        for (int a = 0; a < D; ++a) tx[a] = fmaf((float)o0, B[a * D], cp[a]);
#pragma unroll
        for (int o1 = 0; o1 < 3; ++o1) {
            float ty[3];
#pragma unroll
            for (int a = 0; a < D; ++a) ty[a] = fmaf((float)o1, B[a * D + 1], tx[a]);
#pragma unroll
            for (int o2 = 0; o2 < (D == 3 ? 3 : 1); ++o2) {
                float t[3];
#pragma unroll
                for (int a = 0; a < D; ++a) t[a] = D == 3 ? fmaf((float)o2, B[a * D + 2], ty[a]) : ty[a];
                const float wyz = D == 3 ? w[1][o1] * w[2][o2] : w[1][o1];
                const float W = w0 * wyz;
                float gW[3];
                gW[0] = d0 * wyz;
                gW[1] = D == 3 ? w0 * dw[1][o1] * w[2][o2] : w0 * dw[1][o1];
                if (D == 3) gW[2] = w0 * w[1][o1] * dw[2][o2];
                const float4 u4 = sU[tile_lin<D>(lb[0] + o0, lb[1] + o1, lb[2] + o2)];
                const float u[3] = {u4.x, u4.y, u4.z};
                float Wb = 0.0f;
#pragma unroll
                for (int a = 0; a < D; ++a) Wb = fmaf(u[a], t[a], Wb);
                if (D == 3 && MPM_G2PG_FFMA2) {
                    fma2(S0[0], S0[1], W, u[0], u[1]);
                    S0[2] = fmaf(W, u[2], S0[2]);
                    fma2(fb[0], fb[1], Wb, gW[0], gW[1]);
                    fb[2] = fmaf(Wb, gW[2], fb[2]);
                } else {
#pragma unroll
                    for (int a = 0; a < D; ++a) S0[a] = fmaf(W, u[a], S0[a]);
#pragma unroll
                    for (int k = 0; k < D; ++k) fb[k] = fmaf(Wb, gW[k], fb[k]);
                }
            }
        }
    }
#pragma unroll
    for (int k = 0; k < D; ++k) {  // fb_k -= (B^T S0)_k
        float s = 0.0f;
#pragma unroll
        for (int a = 0; a < D; ++a) s = fmaf(B[a * D + k], S0[a], s);
        xbp_out[k] = fmaf(p.inv_dx, fb[k] - s, xb[k]);
    }
}

template <int D>
__global__ void __launch_bounds__(kTQ, MPM_G2PG_MINB) k_g2p_grad(KParams p, SlotView sl, StateView S, AdjView Sbn,
                                                            float4* __restrict__ ubar) {
    pdl_begin();
    using G = Geo<D>;
    constexpr int RS = RowL<D>::STRIDE;
    extern __shared__ __align__(16) unsigned char smem[];
    float* s_row = reinterpret_cast<float*>(smem);   // rows, then ...
    float4* s_cb = reinterpret_cast<float4*>(smem);  // ... node partials
    int* s_cst = reinterpret_cast<int*>(smem + g2pg_union_bytes<D>());
    const int tid = threadIdx.x;
    const int my_cell = tid / 3, my_ox = tid - 3 * (tid / 3);
    const int nact = *sl.nactive;
    const int b0 = *sl.base;
    const int* blist = sl.blist + b0;
    const int* bstart = sl.bstart + b0 + sl.step;
    const unsigned short* cstart = sl.cstart + (int64_t)b0 * (G::CELLS + 1);
    for (int bi = blockIdx.x; bi < nact; bi += gridDim.x) {
        const int bid = blist[bi];
        const int start = bstart[bi];
        const int nvalid = cstart[(int64_t)bi * (G::CELLS + 1) + G::CELLS];
        int e, c0[3];
        block_origin<D>(p, bid, e, c0);
        float x[3], xb[3], vbc[Lay<D>::VC];  // vbc: (vb', Cb') of S_bar_{t+1}
#define MPM_G2PG_LOAD(R)                                                                      \
    do {                                                                                      \
        const int j_ = start + (R);                                                           \
        const int i_ = sl.sigma[j_];                                                          \
        load_comps<Lay<D>::X>(S.x, i_, x);                                                    \
        load_comps<Lay<D>::X>(Sbn.x, j_, xb);                                                 \
        load_comps<Lay<D>::VC>(Sbn.vc, j_, vbc);                                              \
    } while (0)
        if (tid < nvalid) MPM_G2PG_LOAD(tid);
        for (int c = tid; c <= G::CELLS; c += kTQ) s_cst[c] = cstart[(int64_t)bi * (G::CELLS + 1) + c];
        __syncthreads();
        SliceAcc<D, false> acc;
        acc.zero();
        for (int ch = 0; ch < nvalid; ch += kCH) {
            const int cend = min(nvalid, ch + kCH);
            for (int r = ch + tid; r < cend; r += kTQ) {  // data of r is in registers
                float w[3][3], cp[3], B[D * D];
                g2pg_row<D>(p, x, xb, vbc, vbc + D, c0, w, cp, B);
                write_row<D>(s_row + (r - ch) * RS, w, cp, B);
                if (r + kTQ < nvalid) MPM_G2PG_LOAD(r + kTQ);  // this thread's next particle
            }
            __syncthreads();
            if (tid < kACC) {
                const int lo = max(s_cst[my_cell], ch), hi = min(s_cst[my_cell + 1], cend);
                for (int rr = lo; rr < hi; ++rr) acc.row(s_row + (rr - ch) * RS, my_ox);
            }
            __syncthreads();
        }
#undef MPM_G2PG_LOAD
        if (tid < kACC) acc.store(s_cb, my_cell, my_ox);
        __syncthreads();
        float4* tile = ubar + (int64_t)bi * G::TN;
        for (int q = tid; q < G::TN; q += kTQ) tile[q] = node_gather<D>(s_cb, q);
        __syncthreads();
    }
}

// g2p_grad's gather part as its own pass: thread per particle of a block,
// U tile staged like g2p.  Runs on a second stream, concurrently with the U_bar scatter
// (k_g2p_grad) and grid_op_grad; writes xb_t (partial) for p2g_grad.
#ifndef MPM_GATHER_MINB
#define MPM_GATHER_MINB 6  // 6 CTAs of 128 threads per SM: <= 80 registers (5: C5 -0.3%, C3 -0.5%, C4 -0.4%)
#endif
template <int D, bool SPLIT>
__global__ void __launch_bounds__(kTG, MPM_GATHER_MINB) k_g2p_grad_gather(KParams p, SlotView sl, StateView S, AdjView Sbn,
                                                        float* __restrict__ xbp) {
    pdl_begin();
    using G = Geo<D>;
    __shared__ __align__(128) float4 s_buf[2 * G::TN];
    __shared__ __align__(16) int s_sig[2 * kSigCap];
    __shared__ __align__(8) uint64_t s_bar[2];
    const int tid = threadIdx.x;
    const int nact = *sl.nactive;
    const int b0 = *sl.base;
    const int* blist = sl.blist + b0;
    const int* bstart = sl.bstart + b0 + sl.step;
    const unsigned short* cstart = sl.cstart + (int64_t)b0 * (G::CELLS + 1);
    const float4* rt = sl.tiles + (int64_t)b0 * G::TN;
    SigPipe<D> pipe{s_buf, s_bar, s_sig, sl.sigma, bstart};
    pipe.init();
    __syncthreads();
    const int split = SPLIT ? item_split(nact, gridDim.x) : 1, nitems = nact * split;
    pipe.start(rt, blockIdx.x / split, nact);
    int it = 0;
    for (int w = blockIdx.x; w < nitems; w += gridDim.x, ++it) {
        const int bi = w / split;
        pipe.next(rt, (w + gridDim.x) / split, nact, it);
        const int start = bstart[bi];
        const int nvalid = cstart[(int64_t)bi * (G::CELLS + 1) + G::CELLS];
        int rb, re;
        if (SPLIT) item_range<kTG>(nvalid, w - bi * split, split, rb, re);
        else { rb = 0; re = nvalid; }
        int e, c0[3];
        block_origin<D>(p, blist[bi], e, c0);
        const float4* sU = pipe.wait(it);  // tile and sigma segment
        const int* sg = pipe.sig_at(it, start);
        for (int r0 = rb; r0 < re; r0 += kTG) {
            const int r = r0 + tid;
            const bool in = r < re;
            float x[3], xb[3], vbc[Lay<D>::VC];  // vbc: (vb', Cb') of S_bar_{t+1}
            const int j = start + r;
            if (in) {
                const int i = sg[r];
                load_comps<Lay<D>::X>(S.x, i, x);
                load_comps<Lay<D>::X>(Sbn.x, j, xb);
                load_comps<Lay<D>::VC>(Sbn.vc, j, vbc);
            }
            if (in) {
                int lb[3];
                float fx[3], wt[3][3], dw[3][3], xo[3];
                particle_weights<D>(p, x, c0, lb, fx, wt, dw);
                g2pg_gather<D>(p, sU, lb, fx, wt, dw, xb, vbc, vbc + D, xo);
                store_comps<Lay<D>::X>(xbp, j, xo);
            }
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------ p2g_grad
// staging fuses grid_op_grad (select rule): ub = z ? 0 : Ub;
// Pb = ub/(M + eps); Mb = -(ub . u0)/(M + eps).  Then per particle:
// vb = sum W m Pb; Ab = sum W Pb dpos^T; Wb = Pb.(m v + A dpos) + Mb m;
// fb += Wb dW/df - dx W A^T Pb; Cb = m Ab + dt Ftb F^T; taub = -dt V 4/dx^2 Ab;
// Ftb = Fb' + stress/actuation adjoint; Fb = (I + dt C)^T Ftb; xb += fb/dx.
// per-particle p2g_grad; returns the actuation-gradient contribution kappa q^T taub q
template <int D>
__device__ __forceinline__ float p2g_grad_particle(const KParams& p, const float4* __restrict__ sG,
                                                   const float* x, const float* vc, const float* F,
                                                   const float* Fbn, const float* xbp, bool has_act,
                                                   float act, bool fluid, const int c0[3], int i,
                                                   const AdjView& Sb, int* flags) {
    using L = Lay<D>;
    const float* v = vc;
    const float* C = vc + D;
    int lb[3];
    float fx[3], w[3][3], dw[3][3];
    particle_weights<D>(p, x, c0, lb, fx, w, dw);
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
    float tau[D * D], Adx[D * D], c[3];
    kirchhoff<D>(p, Ft, act, tau, fluid);
#pragma unroll
    for (int q = 0; q < D * D; ++q) Adx[q] = p.dx * fmaf(p.stress_scale, tau[q], p.p_mass * C[q]);
#pragma unroll
    for (int a = 0; a < D; ++a) {  // m v + A dpos = c + Adx o
        float s = p.p_mass * v[a];
#pragma unroll
        for (int b = 0; b < D; ++b) s = fmaf(-Adx[a * D + b], fx[b], s);
        c[a] = s;
    }
    float fb[3] = {0.f, 0.f, 0.f}, S0[3] = {0.f, 0.f, 0.f}, Sm[3][3];
#pragma unroll
    for (int q = 0; q < 9; ++q) (&Sm[0][0])[q] = 0.f;
    if (D == 3 && MPM_P2GG_FFMA2) {
        // the nested form below with packed f32x2 FMAs on the (x, y) pairs and on the
        // (A, B) weight sums; per lane the same IEEE fmas: bitwise identical
        float fx0 = 0.f, fx1 = 0.f, fx2 = 0.f;
#pragma unroll
        for (int o0 = 0; o0 < 3; ++o0) {
            float Gy[3] = {0.f, 0.f, 0.f}, Hy[3] = {0.f, 0.f, 0.f}, Ky[3] = {0.f, 0.f, 0.f};
            float Ay = 0.f, By = 0.f, Cy = 0.f;
            float mx[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) mx[a] = fmaf((float)o0, Adx[a * D], c[a]);
#pragma unroll
            for (int o1 = 0; o1 < 3; ++o1) {
                float Gz[3] = {0.f, 0.f, 0.f}, Hz[3] = {0.f, 0.f, 0.f}, Az = 0.f, Bz = 0.f;
                float my[3];
#pragma unroll
                for (int a = 0; a < 3; ++a) my[a] = fmaf((float)o1, Adx[a * D + 1], mx[a]);
#pragma unroll
                for (int o2 = 0; o2 < 3; ++o2) {
                    const float4 g4 = sG[tile_lin<D>(lb[0] + o0, lb[1] + o1, lb[2] + o2)];
                    float Wb = g4.w * p.p_mass;
                    Wb = fmaf(g4.x, fmaf((float)o2, Adx[2], my[0]), Wb);
                    Wb = fmaf(g4.y, fmaf((float)o2, Adx[5], my[1]), Wb);
                    Wb = fmaf(g4.z, fmaf((float)o2, Adx[8], my[2]), Wb);
                    const float w2 = w[2][o2];
                    fma2(Gz[0], Gz[1], w2, g4.x, g4.y);
                    Gz[2] = fmaf(w2, g4.z, Gz[2]);
                    if (o2) {
                        const float w2o = (float)o2 * w2;
                        fma2(Hz[0], Hz[1], w2o, g4.x, g4.y);
                        Hz[2] = fmaf(w2o, g4.z, Hz[2]);
                    }
                    const float2 ab = __ffma2_rn(make_float2(w2, dw[2][o2]), make_float2(Wb, Wb), make_float2(Az, Bz));
                    Az = ab.x;
                    Bz = ab.y;
                }
                const float w1 = w[1][o1];
                fma2(Gy[0], Gy[1], w1, Gz[0], Gz[1]);
                Gy[2] = fmaf(w1, Gz[2], Gy[2]);
                fma2(Hy[0], Hy[1], w1, Hz[0], Hz[1]);
                Hy[2] = fmaf(w1, Hz[2], Hy[2]);
                if (o1) {
                    const float w1o = (float)o1 * w1;
                    fma2(Ky[0], Ky[1], w1o, Gz[0], Gz[1]);
                    Ky[2] = fmaf(w1o, Gz[2], Ky[2]);
                }
                const float2 ay = __ffma2_rn(make_float2(w1, dw[1][o1]), make_float2(Az, Az), make_float2(Ay, By));
                Ay = ay.x;
                By = ay.y;
                Cy = fmaf(w1, Bz, Cy);
            }
            const float w0 = w[0][o0];
            fma2(S0[0], S0[1], w0, Gy[0], Gy[1]);
            S0[2] = fmaf(w0, Gy[2], S0[2]);
            fma2(Sm[2][0], Sm[2][1], w0, Hy[0], Hy[1]);
            Sm[2][2] = fmaf(w0, Hy[2], Sm[2][2]);
            fma2(Sm[1][0], Sm[1][1], w0, Ky[0], Ky[1]);
            Sm[1][2] = fmaf(w0, Ky[2], Sm[1][2]);
            if (o0) {
                const float w0o = (float)o0 * w0;
                fma2(Sm[0][0], Sm[0][1], w0o, Gy[0], Gy[1]);
                Sm[0][2] = fmaf(w0o, Gy[2], Sm[0][2]);
            }
            fx0 = fmaf(dw[0][o0], Ay, fx0);
            const float2 f12 = __ffma2_rn(make_float2(w0, w0), make_float2(By, Cy), make_float2(fx1, fx2));
            fx1 = f12.x;
            fx2 = f12.y;
        }
        fb[0] = fx0; fb[1] = fx1; fb[2] = fx2;
    } else if (D == 3 && MPM_P2GG_NESTED) {
        // Nested separable form of the 27-node gather below (same sums, re-associated): the
        // weights factor per axis, W_o = w0 w1 w2 and dW/df = (dw0 w1 w2, w0 dw1 w2, w0 w1 dw2),
        // so the z sums are formed per (o0, o1), the y sums per o0, then the x sums:
        //   S0 = sum w0 sum w1 sum w2 g,  Sm[b] = the same with o_b w_b on axis b,
        //   fb = (sum dw0 sum w1 sum w2 Wb, sum w0 sum dw1 sum w2 Wb, sum w0 sum w1 sum dw2 Wb)
        // with Wb_o = g_o . (c + Adx o) + m Mb_o per node.  ~30% fewer FP operations.
        float fx0 = 0.f, fx1 = 0.f, fx2 = 0.f;
#pragma unroll
        for (int o0 = 0; o0 < 3; ++o0) {
            float Gy[3] = {0.f, 0.f, 0.f}, Hy[3] = {0.f, 0.f, 0.f}, Ky[3] = {0.f, 0.f, 0.f};
            float Ay = 0.f, By = 0.f, Cy = 0.f;
            float mx[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) mx[a] = fmaf((float)o0, Adx[a * D], c[a]);
#pragma unroll
            for (int o1 = 0; o1 < 3; ++o1) {
                float Gz[3] = {0.f, 0.f, 0.f}, Hz[3] = {0.f, 0.f, 0.f}, Az = 0.f, Bz = 0.f;
                float my[3];
#pragma unroll
                for (int a = 0; a < 3; ++a) my[a] = fmaf((float)o1, Adx[a * D + 1], mx[a]);
#pragma unroll
                for (int o2 = 0; o2 < 3; ++o2) {
                    const float4 g4 = sG[tile_lin<D>(lb[0] + o0, lb[1] + o1, lb[2] + o2)];
                    const float g[3] = {g4.x, g4.y, g4.z};
                    float Wb = g4.w * p.p_mass;
#pragma unroll
                    for (int a = 0; a < 3; ++a) Wb = fmaf(g[a], fmaf((float)o2, Adx[a * D + 2], my[a]), Wb);
                    const float w2 = w[2][o2];
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        Gz[a] = fmaf(w2, g[a], Gz[a]);
                        if (o2) Hz[a] = fmaf((float)o2 * w2, g[a], Hz[a]);
                    }
                    Az = fmaf(w2, Wb, Az);
                    Bz = fmaf(dw[2][o2], Wb, Bz);
                }
                const float w1 = w[1][o1];
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    Gy[a] = fmaf(w1, Gz[a], Gy[a]);
                    Hy[a] = fmaf(w1, Hz[a], Hy[a]);
                    if (o1) Ky[a] = fmaf((float)o1 * w1, Gz[a], Ky[a]);
                }
                Ay = fmaf(w1, Az, Ay);
                By = fmaf(dw[1][o1], Az, By);
                Cy = fmaf(w1, Bz, Cy);
            }
            const float w0 = w[0][o0];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                S0[a] = fmaf(w0, Gy[a], S0[a]);
                Sm[2][a] = fmaf(w0, Hy[a], Sm[2][a]);
                Sm[1][a] = fmaf(w0, Ky[a], Sm[1][a]);
                if (o0) Sm[0][a] = fmaf((float)o0 * w0, Gy[a], Sm[0][a]);
            }
            fx0 = fmaf(dw[0][o0], Ay, fx0);
            fx1 = fmaf(w0, By, fx1);
            fx2 = fmaf(w0, Cy, fx2);
        }
        fb[0] = fx0; fb[1] = fx1; fb[2] = fx2;
    } else
#pragma unroll
    for (int o0 = 0; o0 < 3; ++o0) {
        float mx[3];
#pragma unroll
        for (int a = 0; a < D; ++a) mx[a] = fmaf((float)o0, Adx[a * D], c[a]);
#pragma unroll
        for (int o1 = 0; o1 < 3; ++o1) {
            float my[3];
#pragma unroll
            for (int a = 0; a < D; ++a) my[a] = fmaf((float)o1, Adx[a * D + 1], mx[a]);
#pragma unroll
            for (int o2 = 0; o2 < (D == 3 ? 3 : 1); ++o2) {
                float m[3];
#pragma unroll
                for (int a = 0; a < D; ++a) m[a] = D == 3 ? fmaf((float)o2, Adx[a * D + 2], my[a]) : my[a];
                const float wyz = D == 3 ? w[1][o1] * w[2][o2] : w[1][o1];
                const float W = w[0][o0] * wyz;
                float gW[3];
                gW[0] = dw[0][o0] * wyz;
                gW[1] = D == 3 ? w[0][o0] * dw[1][o1] * w[2][o2] : w[0][o0] * dw[1][o1];
                if (D == 3) gW[2] = w[0][o0] * w[1][o1] * dw[2][o2];
                const float4 g4 = sG[tile_lin<D>(lb[0] + o0, lb[1] + o1, lb[2] + o2)];
                const float gP[3] = {g4.x, g4.y, g4.z};
                float Wb = g4.w * p.p_mass;
                const int o[3] = {o0, o1, o2};
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    Wb = fmaf(gP[a], m[a], Wb);
                    const float wg = W * gP[a];
                    S0[a] += wg;
#pragma unroll
                    for (int b = 0; b < D; ++b)
                        if (o[b]) Sm[b][a] = fmaf((float)o[b], wg, Sm[b][a]);
                }
#pragma unroll
                for (int k = 0; k < D; ++k) fb[k] = fmaf(Wb, gW[k], fb[k]);
            }
        }
    }
    // Ab[a][b] = dx (Sm[b][a] - S0[a] f[b]);  fb_k -= (Adx^T S0)_k
    float Ab[D * D], taub[D * D], Ftb[D * D];
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
        for (int b = 0; b < D; ++b) Ab[a * D + b] = p.dx * fmaf(-S0[a], fx[b], Sm[b][a]);
#pragma unroll
    for (int k = 0; k < D; ++k) {
        float s = 0.0f;
#pragma unroll
        for (int a = 0; a < D; ++a) s = fmaf(Adx[a * D + k], S0[a], s);
        fb[k] -= s;
    }
#pragma unroll
    for (int q = 0; q < D * D; ++q) {
        taub[q] = p.stress_scale * Ab[q];
        Ftb[q] = Fbn[q];
    }
    if (fluid) fluid_reset_adj<D>(Ft, Fbn, Ftb);  // R23: F_{t+1} = J^(1/d) I
    const float abar = kirchhoff_adj<D>(p, Ft, has_act, act, taub, Ftb, fluid);
    bool fin = true;
    // stores interleaved with the arithmetic (whole-row stores at the end keep 24 more values
    // live at the 128-register cap)
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
        for (int b = 0; b < D; ++b) {
            float sF = Ftb[a * D + b], sC = 0.0f;
#pragma unroll
            for (int k = 0; k < D; ++k) {
                sF = fmaf(p.dt * C[k * D + a], Ftb[k * D + b], sF);
                sC = fmaf(Ftb[a * D + k], F[b * D + k], sC);
            }
            Sb.f[soa<L::FF>(a * D + b, i)] = sF;
            Sb.vc[soa<L::VC>(D + a * D + b, i)] = fmaf(p.dt, sC, p.p_mass * Ab[a * D + b]);
            fin = fin && isfinite(sF);
        }
#pragma unroll
    for (int a = 0; a < D; ++a) {
        Sb.x[soa<L::X>(a, i)] = fmaf(p.inv_dx, fb[a], xbp[a]);
        Sb.vc[soa<L::VC>(a, i)] = p.p_mass * S0[a];
    }
    if (!fin) atomicOr(flags, FLAG_NONFINITE);
    return abar;
}

#ifndef MPM_P2GG_THREADS
#define MPM_P2GG_THREADS 128
#endif
constexpr int kTP = MPM_P2GG_THREADS;  // p2g_grad CTA

template <int D, bool SPLIT>
__global__ void __launch_bounds__(kTP, MPM_P2GG_MINB) k_p2g_grad(KParams p, SlotView sl, StateView S,
                                                 const int32_t* __restrict__ aid,
                                                 const float* __restrict__ alpha, AdjView Sbn,
                                                 const float* __restrict__ xbp, AdjView Sb,
                                                 float* __restrict__ abar_part, int* flags) {
    pdl_begin();
    using G = Geo<D>;
    using L = Lay<D>;
    __shared__ __align__(128) float4 s_buf[2 * G::TN];
    __shared__ __align__(8) uint64_t s_bar[2];
    __shared__ float s_ab[kTP / 32][32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nact = *sl.nactive;
    const int b0 = *sl.base;  // this step's offset in the grid-store pool
    const int* blist = sl.blist + b0;
    const int* bstart = sl.bstart + b0 + sl.step;
    unsigned short* cstart = sl.cstart + (int64_t)b0 * (Geo<D>::CELLS + 1);
    const float4* gt = sl.part;  // (Pb, Mb) tiles from grid_op_grad (local block index)
    TilePipe<D> pipe{s_buf, s_bar};
    pipe.init();
    __syncthreads();
    const int split = SPLIT ? item_split(nact, gridDim.x) : 1, nitems = nact * split;
    pipe.start(gt, blockIdx.x / split, nact);
    int it = 0;
    for (int w = blockIdx.x; w < nitems; w += gridDim.x, ++it) {
        const int bi = w / split;
        pipe.next(gt, (w + gridDim.x) / split, nact, it);
        const int bid = blist[bi];
        const int start = bstart[bi];
        const int nvalid = cstart[(int64_t)bi * (G::CELLS + 1) + G::CELLS];
        int rb, re;
        if (SPLIT) item_range<kTP>(nvalid, w - bi * split, split, rb, re);
        else { rb = 0; re = nvalid; }
        int e, c0[3];
        block_origin<D>(p, bid, e, c0);
        s_ab[warp][lane] = 0.0f;  // each warp owns its row
        __syncwarp();
        const float4* sG = nullptr;
        if (rb >= re) pipe.wait(it);
        // a thread's particle inputs of one pass (loading the next pass's before this pass's math,
        // with two register sets at 3 CTAs per SM, measured slower: 177 -> 187 ms per C5 iteration)
        struct In {
            float x[3], vc[L::VC], F[L::FF], Fbn[L::FF], xb[3];
            int i;  // row of S_t (state rows are < 2^31)
            int a_id;
            bool fluid, in;
        };
        auto load = [&](In& d, int r) {
            d.in = r < re;
            d.i = 0;
            d.a_id = -1;
            d.fluid = false;
            if (d.in) {
                const int j = start + r;
                d.i = sl.sigma[j];
                load_comps<L::X>(S.x, d.i, d.x);
                load_comps<L::VC>(S.vc, d.i, d.vc);
                load_comps<L::FF>(S.f, d.i, d.F);
                load_comps<L::FF>(Sbn.f, j, d.Fbn);
                load_comps<L::X>(xbp, j, d.xb);
                if (aid || p.mat) {
                    const int pd = __ldg(S.pid + d.i);
                    if (aid) d.a_id = __ldg(aid + pd);
                    if (p.mat) d.fluid = __ldg(p.mat + pd) != 0;
                }
            }
        };
        In cur;
        for (int r0 = rb; r0 < re; r0 += kTP) {
            load(cur, r0 + tid);  // particle loads go out before the (first pass's) tile staging
            if (r0 == rb) sG = pipe.wait(it);
            float abar = 0.0f;
            int a_id = cur.a_id;
            if (cur.in) {
                const bool has_act = aid && a_id >= 0 && a_id < p.n_act;
                abar = p2g_grad_particle<D>(p, sG, cur.x, cur.vc, cur.F, cur.Fbn, cur.xb, has_act,
                                            has_act ? alpha[e * p.a_estride + a_id] : 0.0f, cur.fluid, c0, cur.i,
                                            Sb, flags);
                if (!has_act) a_id = -1;
            }
            if (p.n_act > 0) {  // per-actuator warp sums (fixed butterfly) into the warp's slot
                unsigned rem = __ballot_sync(0xffffffffu, a_id >= 0);
                while (rem) {
                    const int target = __shfl_sync(0xffffffffu, a_id, __ffs(rem) - 1);
                    float vsum = a_id == target ? abar : 0.0f;
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) vsum += __shfl_xor_sync(0xffffffffu, vsum, off);
                    if (lane == 0) s_ab[warp][target] += vsum;
                    rem &= ~__ballot_sync(0xffffffffu, a_id == target);
                }
            }
        }
        __syncthreads();
        if (p.n_act > 0 && tid < p.n_act) {
            float s = 0.0f;
            for (int wv = 0; wv < kTP / 32; ++wv) s += s_ab[wv][tid];
            // per work item, [n_act][step_blocks * kMaxSplit]: the reduction reads rows
            abar_part[(int64_t)tid * p.step_blocks * kMaxSplit + w] = s;
        }
        __syncthreads();
    }
}

// alpha_bar_t[a] = fixed-order sum over p2g_grad's work items of the step (blocks, or parts of
// blocks) of abar_part[a][w]: thread i sums items i, i + 256, ... in order (four interleaved
// accumulators, combined in order), then the warps' butterflies and the 8 warp sums in order.
// Closed loop: per episode e = blockIdx.y over that episode's blocks (a contiguous range of the
// block-id-ordered list, found by binary search).  256 threads per actuator: with 64 robot
// episodes a step has ~6,400 blocks, which one warp per actuator summed in ~20 us.
constexpr int kRA = 256;
__global__ void __launch_bounds__(kRA) k_reduce_abar(KParams p, SlotView sl, const float* __restrict__ part,
                                                     float* __restrict__ out, int grid_p2gg) {
    pdl_begin();
    __shared__ float s_w[kRA / 32];
    const int a = blockIdx.x, e = blockIdx.y, n_act = p.n_act;
    const int n = *sl.nactive;
    const int* blist = sl.blist + *sl.base;
    int lo = 0, hi = n;
    if (p.closed_loop) {  // first entries of episode e and e + 1 (block ids are episode-major)
        int l = 0, h = n;
        while (l < h) { const int m = (l + h) >> 1; if (blist[m] / p.nbe < e) l = m + 1; else h = m; }
        lo = l;
        h = n;
        while (l < h) { const int m = (l + h) >> 1; if (blist[m] / p.nbe <= e) l = m + 1; else h = m; }
        hi = l;
    }
    const int split = item_split(n, grid_p2gg);  // p2g_grad's work items of this step
    lo *= split;
    hi *= split;
    const float* row = part + (int64_t)a * p.step_blocks * kMaxSplit;
    float s4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    int b = lo + (int)threadIdx.x;
    for (; b + 3 * kRA < hi; b += 4 * kRA) {
#pragma unroll
        for (int u = 0; u < 4; ++u) s4[u] += row[b + u * kRA];
    }
    if (b < hi) s4[0] += row[b];  // at most three left
    if (b + kRA < hi) s4[1] += row[b + kRA];
    if (b + 2 * kRA < hi) s4[2] += row[b + 2 * kRA];
    float s = (s4[0] + s4[1]) + (s4[2] + s4[3]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        float t = 0.0f;
#pragma unroll
        for (int w = 0; w < kRA / 32; ++w) t += s_w[w];
        out[e * n_act + a] = t;
    }
}

// measurement: number of distinct grid nodes with M > 0 in a step's resolved tiles.
// Each node is counted once, in the tile of the block that owns it (local n < B).
template <int D>
__global__ void __launch_bounds__(kT) k_count_active(KParams p, SlotView sl, unsigned long long* count) {
    pdl_begin();
    using G = Geo<D>;
    const int nact = *sl.nactive;
    const int b0 = *sl.base;
    const float4* rt = sl.tiles + (int64_t)b0 * G::TN;
    const int64_t total = (int64_t)nact * G::TN;
    unsigned long long c = 0;
    for (int64_t idx = (int64_t)blockIdx.x * kT + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * kT) {
        int n[3];
        local_node<D>((int)(idx % G::TN), n);
        if (n[0] >= G::B || n[1] >= G::B || (D == 3 && n[2] >= G::B)) continue;
        if (fabsf(rt[idx].w) > 0.0f) ++c;  // |w| = M (sign bit = sticky)
    }
    for (int off = 16; off > 0; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

// ------------------------------------------------------------ f3 migration
// Rows of S_{t+1} that arrive from the neighbours (their g2p(t) outboxes): appended after this
// subdomain's sorted rows of step t (left neighbour's first), state copied from the neighbour's
// S_{t+1} (peer memory), bin key + histogram of step t+1.  blockIdx.y = side (0 left, 1 right).
// The immigrants' storage order follows the outbox (atomic) order; no sum depends on it (every
// block list is canonicalised by (cell, particle id)).
// row j of an AoSoA array (src, possibly a peer's memory) -> row dst (plain loads: the
// neighbour wrote it in an earlier kernel of its own stream, ordered by events)
template <int NC>
__device__ __forceinline__ void copy_comps(float* dstb, int64_t dst, const float* srcb, int64_t j) {
#pragma unroll
    for (int k = 0; k < NC; ++k) dstb[soa<NC>(k, dst)] = srcb[soa<NC>(k, j)];
}

template <int D>
__global__ void __launch_bounds__(kT) k_immigrate(KParams p, StateView S, const int* __restrict__ nsorted,
                                                  MigSrc left, MigSrc right, int x_lo, int x_hi, int cap,
                                                  int* __restrict__ keys, int* __restrict__ bcount,
                                                  int* __restrict__ imm_base, int* __restrict__ nrows, int* flags) {
    pdl_begin();
    using L = Lay<D>;
    const int side = blockIdx.y;
    const MigSrc& src = side == 0 ? left : right;
    const int n_left = left.cnt ? min(*left.cnt, left.cap) : 0;
    const int n_right = right.cnt ? min(*right.cnt, right.cap) : 0;
    const int base = *nsorted + (side == 0 ? 0 : n_left);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        imm_base[side] = base;
        if (side == 0) *nrows = *nsorted + n_left + n_right;
    }
    const int n = side == 0 ? n_left : n_right;
    const int m = blockIdx.x * kT + threadIdx.x;
    const bool in = m < n;
    int key = -1;
    if (in) {
        const int j = src.rows[(side == 0 ? 1 : 0) * src.cap + m];  // the neighbour's outbox toward us
        const int64_t dst = (int64_t)base + m;
        if (dst >= p.N) {
            atomicOr(flags, FLAG_MIGRATION);  // capacity of this subdomain exceeded
        } else {
            // the rows from the neighbour's memory
            copy_comps<L::X>(S.x, dst, src.S.x, j);
            copy_comps<L::VC>(S.vc, dst, src.S.vc, j);
            copy_comps<L::FF>(S.f, dst, src.S.f, j);
            float x[3];
#pragma unroll
            for (int k = 0; k < D; ++k) x[k] = S.x[soa<L::X>(k, dst)];
            S.pid[dst] = src.S.pid[j];
            int b[3];
            if (base_cell<D>(p, x, b)) {
                const int bb[3] = {b[0] >> Geo<D>::LOGB, b[1] >> Geo<D>::LOGB, b[2] >> Geo<D>::LOGB};
                const int lc[3] = {b[0] & (Geo<D>::B - 1), b[1] & (Geo<D>::B - 1), b[2] & (Geo<D>::B - 1)};
                if (bb[0] >= x_lo && bb[0] < x_hi) {
                    key = block_lin<D>(p, 0, bb);
                    keys[dst] = key * 128 + cell_of<D>(lc);
                } else {
                    atomicOr(flags, FLAG_MIGRATION);  // moved past this slab in one step
                    keys[dst] = -1;
                }
            } else {
                atomicOr(flags, FLAG_OUT_OF_DOMAIN);
                keys[dst] = -1;
            }
        }
    }
    count_key(in && key >= 0, key, bcount);
}

// backward of the migration: the adjoint of an emigrant's S_{t+1} row was computed by the
// neighbour (at its immigrant row imm_base + m); copy it back to the emigrant's row j here.
template <int D>
__global__ void __launch_bounds__(kT) k_adj_pull(KParams p, AdjView Sb, const int* __restrict__ cnt,
                                                 const int* __restrict__ rows, int cap, AdjView nbl,
                                                 const int* __restrict__ nbl_base, AdjView nbr,
                                                 const int* __restrict__ nbr_base) {
    pdl_begin();
    using L = Lay<D>;
    const int dir = blockIdx.y;  // 0: emigrants to the left neighbour, 1: to the right
    const AdjView& nb = dir == 0 ? nbl : nbr;
    const int* nbase = dir == 0 ? nbl_base : nbr_base;
    if (!nbase) return;
    const int n = min(cnt[dir], cap);
    const int m = blockIdx.x * kT + threadIdx.x;
    if (m >= n) return;
    const int j = rows[dir * cap + m];
    const int64_t src = (int64_t)nbase[dir == 0 ? 1 : 0] + m;  // we are the neighbour's right / left side
    copy_comps<L::X>(Sb.x, j, nb.x, src);
    copy_comps<L::VC>(Sb.vc, j, nb.vc, src);
    copy_comps<L::FF>(Sb.f, j, nb.f, src);
}

// per-block sums of x over the rows S_T holds for the blocks of step T-1 (sorted order, fixed
// lane-strided + butterfly order): part[bi][k]
template <int D>
__global__ void __launch_bounds__(kT) k_block_com(KParams p, SlotView sl, const float* __restrict__ X,
                                                  float* __restrict__ part) {
    pdl_begin();
    const int nact = *sl.nactive;
    const int b0 = *sl.base;
    const int* bstart = sl.bstart + b0 + sl.step;
    const unsigned short* cstart = sl.cstart + (int64_t)b0 * (Geo<D>::CELLS + 1);
    const int lane = threadIdx.x & 31;
    for (int bi = blockIdx.x * kW + (threadIdx.x >> 5); bi < nact; bi += gridDim.x * kW) {
        const int start = bstart[bi];
        const int nvalid = cstart[(int64_t)bi * (Geo<D>::CELLS + 1) + Geo<D>::CELLS];
        float acc[3] = {0.f, 0.f, 0.f};
        for (int r = lane; r < nvalid; r += 32)
#pragma unroll
            for (int k = 0; k < D; ++k) acc[k] += X[soa<Lay<D>::X>(k, start + r)];
#pragma unroll
        for (int k = 0; k < D; ++k) {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], off);
            if (lane == 0) part[(int64_t)bi * D + k] = acc[k];
        }
    }
}

inline unsigned nblk(int64_t n) { return (unsigned)((n + kT - 1) / kT); }

// launch-grid table per device (tile_init fills the entry of every device a handle is created
// on; launches read the entry of the current device -- the engine makes the handle's device
// current in every entry point)
struct DevTab {
    int grid[5][2];  // persistent grid size per kernel kind and dimension
    int sms = 148;
    int canon_grid = 148 * 8;
};
constexpr int kMaxDev = 64;
DevTab g_tab[kMaxDev];
const DevTab& tab() {
    int dev = 0;
    cudaGetDevice(&dev);
    return g_tab[dev >= 0 && dev < kMaxDev ? dev : 0];
}

}  // namespace

#define DISPATCH(D, ...) \
    do {                 \
        if ((D) == 2) {  \
            constexpr int DIM = 2; __VA_ARGS__; \
        } else {         \
            constexpr int DIM = 3; __VA_ARGS__; \
        }                \
    } while (0)

static int occupancy_grid(const void* fn, int smem, int threads = kT) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, threads, smem);
    return sms * (per > 0 ? per : 1);
}

// Programmatic dependent launch pays where a step is a chain of short, launch-bound kernels
// (C1-C3: +4% measured on C2) and costs where big persistent kernels share the SMs with the
// backward's side streams (waiting dependent CTAs hold SM slots: -12% on C5).  The engine
// enables it per call for small problems (set_pdl); MPM_B200_PDL=0/1 forces it.
static thread_local bool g_pdl = false;  // per host thread: handles on different threads stay independent
bool pdl_enabled() { return g_pdl; }
static int g_pdl_force = -1;

void set_pdl(int64_t particles) {
    if (g_pdl_force < 0) {
        const char* v = getenv("MPM_B200_PDL");
        g_pdl_force = v ? (v[0] != '0') : 2;
    }
    g_pdl = g_pdl_force == 2 ? particles <= kSmallProblem : g_pdl_force == 1;
}

// Kernel attributes are per device: initialise once for every device a handle is created
// on (one process may drive several GPUs).  The launch grids assume identical GPUs.
cudaError_t tile_init() {
    static std::mutex mu;
    static unsigned long long done_mask = 0;
    std::lock_guard<std::mutex> lock(mu);
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e) return e;
    if (dev < 0 || dev >= kMaxDev) return cudaErrorInvalidDevice;
    if ((done_mask >> dev) & 1ull) return cudaSuccess;
    DevTab& T = g_tab[dev];
    cudaDeviceGetAttribute(&T.sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaFuncSetAttribute(k_canon, cudaFuncAttributeMaxDynamicSharedMemorySize, canon_smem_bytes());
    if (e) return e;
    T.canon_grid = occupancy_grid((const void*)k_canon, canon_smem_bytes(), kT);
#define MPM_INIT_DIM(DI)                                                                                          \
    do {                                                                                                          \
        constexpr int DIM = (DI) == 2 ? 2 : 3;                                                                    \
        e = cudaFuncSetAttribute(k_p2g<DIM, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,                 \
                                 p2g_smem_bytes<DIM>());                                                          \
        if (e) return e;                                                                                          \
        e = cudaFuncSetAttribute(k_p2g<DIM, false>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);         \
        if (e) return e;                                                                                          \
        e = cudaFuncSetAttribute(k_p2g<DIM, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,                  \
                                 p2g_smem_bytes<DIM>());                                                          \
        if (e) return e;                                                                                          \
        e = cudaFuncSetAttribute(k_p2g<DIM, true>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);          \
        if (e) return e;                                                                                          \
        e = cudaFuncSetAttribute(k_g2p_grad<DIM>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);           \
        if (e) return e;                                                                                          \
        e = cudaFuncSetAttribute(k_g2p_grad<DIM>, cudaFuncAttributeMaxDynamicSharedMemorySize,                    \
                                 g2pg_smem_bytes<DIM>());                                                         \
        if (e) return e;                                                                                          \
        const int di = DIM == 3 ? 1 : 0;                                                                          \
        T.grid[0][di] = occupancy_grid((const void*)k_p2g<DIM, false>, p2g_smem_bytes<DIM>(), kTQ);               \
        T.grid[1][di] = occupancy_grid((const void*)k_g2p<DIM, false>, 0, kTG);                                          \
        T.grid[2][di] = occupancy_grid((const void*)k_g2p_grad<DIM>, g2pg_smem_bytes<DIM>(), kTQ);                \
        T.grid[3][di] = occupancy_grid((const void*)k_p2g_grad<DIM, false>, 0, kTP);                                     \
        T.grid[4][di] = occupancy_grid((const void*)k_g2p_grad_gather<DIM, false>, 0, kTG);                              \
    } while (0)
    MPM_INIT_DIM(2);
    MPM_INIT_DIM(3);
#undef MPM_INIT_DIM
    done_mask |= 1ull << dev;
    return cudaGetLastError();
}

#ifndef MPM_CAP_G2PG
#define MPM_CAP_G2PG 0  // CTAs per SM of the U_bar scatter (0: occupancy limit)
#endif
#ifndef MPM_CAP_GATHER
#define MPM_CAP_GATHER 0  // CTAs per SM of g2p_grad's gather part (0: occupancy limit)
#endif
static unsigned pgrid(const KParams& p, int kind) {
    const DevTab& T = tab();
    int g = T.grid[kind][p.dim == 3 ? 1 : 0];
    if (kind == 2 && MPM_CAP_G2PG > 0) g = min(g, T.sms * MPM_CAP_G2PG);
    if (kind == 4 && MPM_CAP_GATHER > 0) g = min(g, T.sms * MPM_CAP_GATHER);
    return (unsigned)(p.step_blocks < g ? p.step_blocks : g);
}

void launch_bin_keys(const KParams& p, const float* x, int64_t n_live, int* keys, int* bcount, int* flags,
                     cudaStream_t s) {
    DISPATCH(p.dim, launch_k(k_bin_keys<DIM>, nblk(p.N * p.E), kT, 0, s, p, x, n_live, keys, bcount, flags));
}
int scan_chunks(const KParams& p) { return (p.TB + kScanChunk - 1) / kScanChunk; }
void launch_bin_scan(const KParams& p, int* bcount, int* cursor, const SlotView& sl, int* part, int* flags,
                     cudaStream_t s) {
    const int nc = scan_chunks(p);
    launch_k(k_bin_scan, nc, kT, 0, s, p, bcount, cursor, sl, (int2*)part, flags);
}
void launch_bin_scatter(const KParams& p, const int* keys, const int* pid, int* cursor, const SlotView& sl,
                        cudaStream_t s) {
    launch_k(k_bin_scatter, (unsigned)((p.N * p.E + kT * kScatterPer - 1) / (kT * kScatterPer)), kT, 0, s, p, keys, pid, cursor, sl);
}
void launch_canon(const KParams& p, const SlotView& sl, int* pid_next, int* keys_next, int* flags, cudaStream_t s) {
    const int cg = tab().canon_grid;
    launch_k(k_canon, cg < p.step_blocks ? cg : (p.step_blocks > 0 ? p.step_blocks : 1), kT, canon_smem_bytes(), s, p, sl,
             pid_next, keys_next, flags);
}
bool canon_fused(const KParams& p) { return p.EN <= kSmallProblem; }
void launch_p2g(const KParams& p, const SlotView& sl, const StateView& S, const StateView& Sn,
                const int32_t* aid, const float* alpha_t, int* keys_next, int* flags, cudaStream_t s) {
    if (canon_fused(p))
        DISPATCH(p.dim, launch_k(k_p2g<DIM, true>, pgrid(p, 0), kTQ, p2g_smem_bytes<DIM>(), s, p, sl, S, Sn, aid,
                                 alpha_t, keys_next, flags));
    else
        DISPATCH(p.dim, launch_k(k_p2g<DIM, false>, pgrid(p, 0), kTQ, p2g_smem_bytes<DIM>(), s, p, sl, S, Sn, aid,
                                 alpha_t, keys_next, flags));
}
static unsigned node_grid(const KParams& p) {
    const int64_t need = ((int64_t)p.step_blocks * (p.dim == 3 ? Geo<3>::TN : Geo<2>::TN) + kT - 1) / kT;
    const int64_t cap = (int64_t)tab().sms * 8;
    return (unsigned)(need < cap ? (need > 0 ? need : 1) : cap);
}
static bool has_halo(const SlotView& sl) { return sl.halo.tiles[0] != nullptr || sl.halo.tiles[1] != nullptr; }
void launch_grid_op(const KParams& p, const SlotView& sl, cudaStream_t s) {
    if (has_halo(sl)) DISPATCH(p.dim, launch_k(k_grid_op<DIM, true>, node_grid(p), kT, 0, s, p, sl));
    else if (MPM_NBR_TABLE && sl.nbr) DISPATCH(p.dim, launch_k(k_grid_op<DIM, false, true>, node_grid(p), kT, 0, s, p, sl));
    else DISPATCH(p.dim, launch_k(k_grid_op<DIM, false>, node_grid(p), kT, 0, s, p, sl));
}
void launch_grid_op_grad(const KParams& p, const SlotView& sl, const float4* ubar, cudaStream_t s) {
    if (has_halo(sl)) DISPATCH(p.dim, launch_k(k_grid_op_grad<DIM, true>, node_grid(p), kT, 0, s, p, sl, ubar));
    else if (MPM_NBR_TABLE && sl.nbr)
        DISPATCH(p.dim, launch_k(k_grid_op_grad<DIM, false, true>, node_grid(p), kT, 0, s, p, sl, ubar));
    else DISPATCH(p.dim, launch_k(k_grid_op_grad<DIM, false>, node_grid(p), kT, 0, s, p, sl, ubar));
}
static bool split_blocks(const KParams& p) { return p.N * p.E <= kSmallProblem; }  // see item_split
void launch_g2p(const KParams& p, const SlotView& sl, const StateView& S, const StateView& Sn, int* keys,
                int* bcount, int* flags, bool refwd, const Migr& mg, cudaStream_t s) {
    if (split_blocks(p))
        DISPATCH(p.dim, launch_k(k_g2p<DIM, true>, pgrid(p, 1), kTG, 0, s, p, sl, S, Sn, keys, bcount, flags, refwd, mg));
    else
        DISPATCH(p.dim, launch_k(k_g2p<DIM, false>, pgrid(p, 1), kTG, 0, s, p, sl, S, Sn, keys, bcount, flags, refwd, mg));
}
void launch_g2p_grad(const KParams& p, const SlotView& sl, const StateView& S, const AdjView& Sbn,
                     float4* ubar, cudaStream_t s) {
    DISPATCH(p.dim, launch_k(k_g2p_grad<DIM>, pgrid(p, 2), kTQ, g2pg_smem_bytes<DIM>(), s, p, sl, S, Sbn, ubar));
}
void launch_g2p_grad_gather(const KParams& p, const SlotView& sl, const StateView& S, const AdjView& Sbn,
                            float* xbp, cudaStream_t s) {
    if (split_blocks(p)) DISPATCH(p.dim, launch_k(k_g2p_grad_gather<DIM, true>, pgrid(p, 4), kTG, 0, s, p, sl, S, Sbn, xbp));
    else DISPATCH(p.dim, launch_k(k_g2p_grad_gather<DIM, false>, pgrid(p, 4), kTG, 0, s, p, sl, S, Sbn, xbp));
}
void launch_p2g_grad(const KParams& p, const SlotView& sl, const StateView& S, const int32_t* aid,
                     const float* alpha_t, const AdjView& Sbn, const float* xbp,
                     const AdjView& Sb, float* abar_part, int* flags, cudaStream_t s) {
    if (split_blocks(p))
        DISPATCH(p.dim, launch_k(k_p2g_grad<DIM, true>, pgrid(p, 3), kTP, 0, s, p, sl, S, aid, alpha_t, Sbn, xbp, Sb,
                                 abar_part, flags));
    else
        DISPATCH(p.dim, launch_k(k_p2g_grad<DIM, false>, pgrid(p, 3), kTP, 0, s, p, sl, S, aid, alpha_t, Sbn, xbp, Sb,
                                 abar_part, flags));
}
void launch_count_active(const KParams& p, const SlotView& sl, int64_t* count, cudaStream_t s) {
    cudaMemsetAsync(count, 0, sizeof(int64_t), s);
    DISPATCH(p.dim, launch_k(k_count_active<DIM>, node_grid(p), kT, 0, s, p, sl, (unsigned long long*)count));
}
void launch_reduce_abar(const KParams& p, const SlotView& sl, const float* abar_part, float* alpha_bar_t,
                        cudaStream_t s) {
    if (p.n_act > 0)
        launch_k(k_reduce_abar, dim3(p.n_act, p.closed_loop ? p.E : 1), kRA, 0, s, p, sl, abar_part, alpha_bar_t,
                 split_blocks(p) ? (int)pgrid(p, 3) : 0);  // 0: p2g_grad ran one item per block
}

}  // namespace mpm

namespace mpm {
void launch_immigrate(const KParams& p, const StateView& S, const int* nsorted, MigSrc left, MigSrc right,
                      int x_lo, int x_hi, int cap, int* keys, int* bcount, int* imm_base, int* nrows, int* flags,
                      cudaStream_t s) {
    const int most = std::max(left.cnt ? left.cap : 0, right.cnt ? right.cap : 0);  // the neighbours' outboxes
    const dim3 grid((unsigned)std::max(1, (most + kT - 1) / kT), 2);
    DISPATCH(p.dim, launch_k(k_immigrate<DIM>, grid, kT, 0, s, p, S, nsorted, left, right, x_lo, x_hi, cap, keys,
                             bcount, imm_base, nrows, flags));
}
void launch_adj_pull(const KParams& p, const AdjView& Sb, const int* cnt, const int* rows, int cap,
                     const AdjView& nb_left, const int* nb_left_base, const AdjView& nb_right,
                     const int* nb_right_base, cudaStream_t s) {
    const dim3 grid((unsigned)((cap + kT - 1) / kT), 2);
    DISPATCH(p.dim, launch_k(k_adj_pull<DIM>, grid, kT, 0, s, p, Sb, cnt, rows, cap, nb_left, nb_left_base,
                             nb_right, nb_right_base));
}
void launch_block_com(const KParams& p, const SlotView& sl_last, const float* x, float* part, cudaStream_t s) {
    const int grid = (int)std::min<int64_t>(((int64_t)p.step_blocks + kW - 1) / kW, (int64_t)tab().sms * 8);
    DISPATCH(p.dim, launch_k(k_block_com<DIM>, grid > 0 ? grid : 1, kT, 0, s, p, sl_last, x, part));
}
}  // namespace mpm
