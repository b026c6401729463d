// kernels_tile.cu -- the MLS-MPM step and its adjoint on sm_100a, sorted-tile scheme.
//
// Equations: DESIGN.md R1-R14; kernel order: PAPER.md
// Appendix D.1 (advance / advance_grad).
//
// Layout:
//  * particles are binned every step by the B^d block of cells that holds their
//    base cell (bin_* kernels); the block's list sigma (indices into the state
//    array) is put in canonical (cell, particle id) order by p2g, so every sum
//    below has a fixed order -> bitwise run-to-run reproducible, no atomics in
//    the hot loops;
//  * p2g: one CTA per active block (persistent loop).  Thread-per-particle
//    stress/affine math in registers, then a warp per cell with one lane per
//    stencil offset o sums the cell's contributions to node (cell + o) (smem
//    broadcast reads, no atomics), then a thread per tile node sums the <= 3^d
//    (cell, o) partials and stores the block's (B+2)^d tile with plain stores;
//  * g2p / g2p_grad / p2g_grad stage their node tile in shared memory by summing
//    the <= 2^d overlapping block tiles, fusing grid_op (or grid_op_grad) into
//    the staging; g2p_grad scatters U_bar with the same cell/offset scheme.
#include "kernels.h"

namespace mpm {

namespace {

constexpr int kT = 256;             // threads per CTA (8 warps)
constexpr int kW = kT / 32;

template <int D> __device__ __forceinline__ void load_rec(const float* __restrict__ src, float* r) {
    constexpr int R = Rec<D>::R;
    const float4* s4 = reinterpret_cast<const float4*>(src);
#pragma unroll
    for (int q = 0; q < R / 4; ++q) {
        float4 t = __ldg(s4 + q);
        r[4 * q + 0] = t.x; r[4 * q + 1] = t.y; r[4 * q + 2] = t.z; r[4 * q + 3] = t.w;
    }
}

// block id -> episode and first cell (c0 = block coords * B)
template <int D>
__device__ __forceinline__ void block_origin(const KParams& p, int bid, int& e, int c0[3]) {
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

// Sum of the <= 2^d block tiles that cover global node g (episode e): every
// block whose cells [c0, c0 + B) satisfy c0 <= g < c0 + B + 2 holds a partial
// of that node.  Fixed enumeration order -> deterministic.
template <int D>
__device__ __forceinline__ float4 covered_sum(const KParams& p, int e, const int g[3],
                                              const int* __restrict__ bmap,
                                              const float4* __restrict__ tiles) {
    using G = Geo<D>;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    int blk[3][2], loc[3][2], cnt[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        if (k >= D) { blk[k][0] = 0; loc[k][0] = 0; cnt[k] = 1; continue; }
        const int b0 = g[k] >> G::LOGB, l0 = g[k] & (G::B - 1);
        blk[k][0] = b0; loc[k][0] = l0; cnt[k] = 1;
        if (l0 < 2 && b0 >= 1) { blk[k][1] = b0 - 1; loc[k][1] = l0 + G::B; cnt[k] = 2; }
        else { blk[k][1] = b0; loc[k][1] = l0; }
        if (b0 >= p.nb) cnt[k] = 0;  // node beyond the last block (never read)
    }
    for (int a = 0; a < cnt[0]; ++a)
        for (int b = 0; b < cnt[1]; ++b)
            for (int c = 0; c < cnt[2]; ++c) {
                const int bb[3] = {blk[0][a], blk[1][b], blk[2][c]};
                if (bb[0] >= p.nb || bb[1] >= p.nb || (D == 3 && bb[2] >= p.nb)) continue;
                const int ti = __ldg(bmap + block_lin<D>(p, e, bb));
                if (ti < 0) continue;
                const float4 v = __ldg(tiles + (int64_t)ti * G::TN + tile_lin<D>(loc[0][a], loc[1][b], loc[2][c]));
                acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
            }
    return acc;
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

template <int D> __device__ __forceinline__ void local_node(int q, int n[3]) {
    constexpr int TE = Geo<D>::TE;
    if (D == 2) { n[0] = q / TE; n[1] = q % TE; n[2] = 0; }
    else { n[0] = q / (TE * TE); n[1] = (q / TE) % TE; n[2] = q % TE; }
}

// warp-aggregated histogram increment (keys in a warp are mostly equal)
__device__ __forceinline__ void count_key(bool valid, int key, int* bcount) {
    const unsigned peers = __match_any_sync(0xffffffffu, valid ? key : -1);
    const int leader = __ffs(peers) - 1;
    if (valid && (int)(threadIdx.x & 31) == leader) atomicAdd(&bcount[key], __popc(peers));
}

// ---------------------------------------------------------------- binning
template <int D>
__global__ void __launch_bounds__(kT) k_bin_keys(KParams p, const float* __restrict__ rec,
                                                 int* __restrict__ keys, int* __restrict__ bcount,
                                                 int* flags) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool in = i < p.N * p.E;
    int key = 0;
    bool ok = false;
    if (in) {
        float x[3];
#pragma unroll
        for (int k = 0; k < D; ++k) x[k] = rec[i * Rec<D>::R + Rec<D>::X + k];
        int b[3];
        ok = base_cell<D>(p, x, b);
        const int e = (int)(i / p.N);
        int bb[3] = {b[0] >> Geo<D>::LOGB, b[1] >> Geo<D>::LOGB, b[2] >> Geo<D>::LOGB};
        key = block_lin<D>(p, e, bb);
        if (!ok) { atomicOr(flags, FLAG_OUT_OF_DOMAIN); key = e * p.nbe; ok = true; }
        keys[i] = key;
    }
    count_key(in && ok, key, bcount);
}

// single CTA: exclusive scan of the dense block histogram -> active block list
// (block-id order), starts, block map, scatter cursors; clears the histogram.
constexpr int kScanT = 1024;
__global__ void __launch_bounds__(kScanT) k_bin_scan(KParams p, int* __restrict__ bcount,
                                                     int* __restrict__ cursor, SlotView sl, int* flags) {
    __shared__ int s_part[kScanT], s_act[kScanT];
    const int TB = p.TB, tid = threadIdx.x;
    const int per = (TB + kScanT - 1) / kScanT;
    const int lo = min(TB, tid * per), hi = min(TB, lo + per);
    int tot = 0, act = 0;
    for (int b = lo; b < hi; ++b) {
        const int c = bcount[b];
        tot += c;
        act += c > 0;
    }
    s_part[tid] = tot;
    s_act[tid] = act;
    __syncthreads();
    for (int off = 1; off < kScanT; off <<= 1) {  // Hillis-Steele inclusive scan
        int a = tid >= off ? s_part[tid - off] : 0, b = tid >= off ? s_act[tid - off] : 0;
        __syncthreads();
        s_part[tid] += a;
        s_act[tid] += b;
        __syncthreads();
    }
    int pos = s_part[tid] - tot, li = s_act[tid] - act;
    for (int b = lo; b < hi; ++b) {
        const int c = bcount[b];
        if (c > 0) {
            if (li < p.max_active) {
                sl.blist[li] = b;
                sl.bstart[li] = pos;
                sl.bmap[b] = li;
            } else {
                sl.bmap[b] = -1;
                atomicOr(flags, FLAG_ACTIVE_OVERFLOW);
            }
            cursor[b] = pos;
            pos += c;
            ++li;
        } else {
            sl.bmap[b] = -1;
        }
        bcount[b] = 0;
    }
    if (tid == kScanT - 1) {
        const int n = min(li, p.max_active);
        *sl.nactive = n;
        sl.bstart[n] = min(pos, (int)(p.N * p.E));
    }
}

__global__ void __launch_bounds__(kT) k_bin_scatter(KParams p, const int* __restrict__ keys,
                                                    int* __restrict__ cursor, int* __restrict__ sigma) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool in = j < p.N * p.E;
    const int key = in ? keys[j] : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    const int lane = threadIdx.x & 31, leader = __ffs(peers) - 1;
    int base = 0;
    if (in && lane == leader) base = atomicAdd(&cursor[key], __popc(peers));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (in) sigma[base + __popc(peers & ((1u << lane) - 1u))] = (int)j;
}

// ---------------------------------------------------------------- P2G
template <int D> constexpr int p2g_phase0_bytes() {
    return Geo<D>::MAXP * 14 > kT * Geo<D>::ROW * 4 ? Geo<D>::MAXP * 14 : kT * Geo<D>::ROW * 4;
}
template <int D> constexpr int p2g_smem_bytes() {
    return p2g_phase0_bytes<D>() + Geo<D>::CELLS * Geo<D>::NST * 16 + 2 * (Geo<D>::CELLS + 2) * 4;
}

// fold sub-streams: every lane of the warp must call (2D only)
template <int D> __device__ __forceinline__ float4 fold_subs(float4 a) {
    using G = Geo<D>;
    if (G::NSUB == 1) return a;
    float4 r = a;
#pragma unroll
    for (int s = 1; s < G::NSUB; ++s) {
        r.x += __shfl_down_sync(0xffffffffu, a.x, s * G::NST);
        r.y += __shfl_down_sync(0xffffffffu, a.y, s * G::NST);
        r.z += __shfl_down_sync(0xffffffffu, a.z, s * G::NST);
        r.w += __shfl_down_sync(0xffffffffu, a.w, s * G::NST);
    }
    return r;
}

template <int D, bool MASS>
__device__ __forceinline__ float4 cell_rows(const float* __restrict__ s_tab, int lo, int hi, int lane) {
    using G = Geo<D>;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (lane < G::NST * G::NSUB) {
        const int o = lane % G::NST, sub = lane / G::NST;
        const int ox = D == 3 ? o / 9 : o / 3, oy = D == 3 ? (o / 3) % 3 : o % 3, oz = D == 3 ? o % 3 : 0;
        const float fo[3] = {(float)ox, (float)oy, (float)oz};
        for (int r = lo + sub; r < hi; r += G::NSUB) {
            const float* row = s_tab + r * G::ROW;
            float W = row[ox] * row[3 + oy];
            if (D == 3) W *= row[6 + oz];
            const float* c = row + 3 * D;
            const float* A = c + D;
            float m[3] = {0.f, 0.f, 0.f};
#pragma unroll
            for (int a = 0; a < D; ++a) {
                float s = c[a];
#pragma unroll
                for (int b = 0; b < D; ++b) s = fmaf(A[a * D + b], fo[b], s);
                m[a] = s;
            }
            acc.x = fmaf(W, m[0], acc.x);
            acc.y = fmaf(W, m[1], acc.y);
            if (D == 3) acc.z = fmaf(W, m[2], acc.z);
            if (MASS) acc.w += W;
        }
    }
    return fold_subs<D>(acc);
}

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

template <int D> __device__ __forceinline__ int cell_of(const int lb[3]) {
    using G = Geo<D>;
    return D == 2 ? lb[0] * G::B + lb[1] : (lb[0] * G::B + lb[1]) * G::B + lb[2];
}

// p2g: canonicalise the block list, then per particle
// Ft = (I + dt C) F; tau = tau(Ft) [+ actuation]; A = -dt V 4/dx^2 tau + m C;
// node b+o receives W_o (m v + A (o - f) dx) and W_o m.  F_{t+1} = Ft.
template <int D>
__global__ void __launch_bounds__(kT) k_p2g(KParams p, SlotView sl, StateView S, StateView Sn,
                                            const int32_t* __restrict__ aid,
                                            const float* __restrict__ alpha, int* flags) {
    using G = Geo<D>;
    using RC = Rec<D>;
    extern __shared__ __align__(16) unsigned char smem[];
    float* s_tab = reinterpret_cast<float*>(smem);
    int* s_idx = reinterpret_cast<int*>(smem);
    int* s_pid = s_idx + G::MAXP;
    int* s_tmp = s_pid + G::MAXP;
    short* s_cell = reinterpret_cast<short*>(s_tmp + G::MAXP);
    float4* s_cb = reinterpret_cast<float4*>(smem + p2g_phase0_bytes<D>());
    int* s_cnt = reinterpret_cast<int*>(s_cb + G::CELLS * G::NST);
    int* s_cst = s_cnt + G::CELLS + 2;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nact = *sl.nactive;
    for (int bi = blockIdx.x; bi < nact; bi += gridDim.x) {
        const int bid = sl.blist[bi];
        const int start = sl.bstart[bi], n = sl.bstart[bi + 1] - start;
        int e, c0[3];
        block_origin<D>(p, bid, e, c0);
        if (n > G::MAXP) {
            if (tid == 0) atomicOr(flags, FLAG_BLOCK_OVERFLOW);
            continue;
        }
        // ---- phase 0: cells, then canonical (cell, particle id) order
        for (int q = tid; q < G::CELLS + 2; q += kT) s_cnt[q] = 0;
        __syncthreads();
        for (int q0 = 0; q0 < n; q0 += kT) {
            const int q = q0 + tid;
            const bool in = q < n;
            int cell = G::CELLS;
            if (in) {
                const int i = sl.sigma[start + q];
                float x[3];
#pragma unroll
                for (int k = 0; k < D; ++k) x[k] = S.rec[(int64_t)i * RC::R + RC::X + k];
                int b[3];
                bool ok = base_cell<D>(p, x, b);
                int lb[3] = {0, 0, 0};
#pragma unroll
                for (int k = 0; k < D; ++k) {
                    lb[k] = b[k] - c0[k];
                    ok = ok && lb[k] >= 0 && lb[k] < G::B;
                }
                if (ok) cell = cell_of<D>(lb);
                else atomicOr(flags, FLAG_OUT_OF_DOMAIN);
                s_idx[q] = i;
                s_pid[q] = S.pid[i];
                s_cell[q] = (short)cell;
            }
            const unsigned peers = __match_any_sync(0xffffffffu, in ? cell : -1);
            if (in && lane == __ffs(peers) - 1) atomicAdd(&s_cnt[cell], __popc(peers));
        }
        __syncthreads();
        if (tid == 0) {
            int run = 0;
            for (int c = 0; c <= G::CELLS; ++c) {
                s_cst[c] = run;
                const int k = s_cnt[c];
                s_cnt[c] = run;  // becomes the bucket cursor
                run += k;
            }
            s_cst[G::CELLS + 1] = run;
        }
        __syncthreads();
        for (int q0 = 0; q0 < n; q0 += kT) {  // bucket by cell (order inside a cell arbitrary)
            const int q = q0 + tid;
            const bool in = q < n;
            const int cell = in ? s_cell[q] : -1;
            const unsigned peers = __match_any_sync(0xffffffffu, cell);
            const int leader = __ffs(peers) - 1;
            int base = 0;
            if (in && lane == leader) base = atomicAdd(&s_cnt[cell], __popc(peers));
            base = __shfl_sync(0xffffffffu, base, leader);
            if (in) s_tmp[base + __popc(peers & ((1u << lane) - 1u))] = q;
        }
        __syncthreads();
        for (int r = tid; r < n; r += kT) {  // rank by particle id inside the cell
            const int q = s_tmp[r];
            const int cell = s_cell[q], pq = s_pid[q];
            int rank = 0;
            for (int m = s_cst[cell]; m < s_cst[cell + 1]; ++m) rank += s_pid[s_tmp[m]] < pq;
            const int fpos = start + s_cst[cell] + rank;
            sl.sigma[fpos] = s_idx[q];
            if (Sn.pid) Sn.pid[fpos] = pq;
        }
        for (int c = tid; c <= G::CELLS; c += kT) sl.cstart[(int64_t)bi * (G::CELLS + 1) + c] = (unsigned short)s_cst[c];
        for (int q = tid; q < G::CELLS * G::NST; q += kT) s_cb[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        __syncthreads();
        const int nvalid = s_cst[G::CELLS];
        // ---- phases 1 + 2 over chunks of kT particles in canonical order
        for (int ch = 0; ch < nvalid; ch += kT) {
            const int r = ch + tid;
            if (r < nvalid) {
                const int i = sl.sigma[start + r];
                float rr[RC::R];
                load_rec<D>(S.rec + (int64_t)i * RC::R, rr);
                const float* x = rr + RC::X;
                const float* v = rr + RC::V;
                const float* C = rr + RC::C;
                const float* F = rr + RC::F;
                float fx[3], w[3][3], dw[3][3];
#pragma unroll
                for (int k = 0; k < D; ++k) {
                    float xi = x[k] * p.inv_dx;
                    fx[k] = xi - floorf(xi - 0.5f);
                    bspline(fx[k], w[k], dw[k]);
                }
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
                const int pid = S.pid[i];
                const int a_id = aid ? aid[pid] : -1;
                const float act = a_id >= 0 ? alpha[a_id] : 0.0f;
                float tau[D * D];
                if (!kirchhoff<D>(p, Ft, act, tau)) atomicOr(flags, FLAG_NONFINITE);
                float* row = s_tab + tid * G::ROW;
#pragma unroll
                for (int k = 0; k < D; ++k)
#pragma unroll
                    for (int o = 0; o < 3; ++o) row[3 * k + o] = w[k][o];
                // contribution W_o (c + Adx o), c = m v - Adx f, Adx = A dx
                float Adx[D * D];
#pragma unroll
                for (int q = 0; q < D * D; ++q) Adx[q] = p.dx * fmaf(p.stress_scale, tau[q], p.p_mass * C[q]);
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    float s = p.p_mass * v[a];
#pragma unroll
                    for (int b = 0; b < D; ++b) s = fmaf(-Adx[a * D + b], fx[b], s);
                    row[3 * D + a] = s;
                }
#pragma unroll
                for (int q = 0; q < D * D; ++q) row[4 * D + q] = Adx[q];
                if (Sn.rec) {
                    float* dst = Sn.rec + (int64_t)(start + r) * RC::R + RC::F;
#pragma unroll
                    for (int q = 0; q < D * D; ++q) dst[q] = Ft[q];
                }
            }
            __syncthreads();
            for (int c = warp; c < G::CELLS; c += kW) {
                const int lo = max(s_cst[c], ch), hi = min(s_cst[c + 1], ch + kT);
                if (lo >= hi) continue;
                const float4 acc = cell_rows<D, true>(s_tab - ch * G::ROW, lo, hi, lane);
                if (lane < G::NST) {
                    float4& dst = s_cb[c * G::NST + lane];
                    dst.x += acc.x; dst.y += acc.y; dst.z += acc.z; dst.w += acc.w;
                }
            }
            __syncthreads();
        }
        // ---- phase 3: node tile (plain stores)
        float4* tile = sl.tiles + (int64_t)bi * G::TN;
        for (int q = tid; q < G::TN; q += kT) {
            float4 s = node_gather<D>(s_cb, q);
            s.w *= p.p_mass;
            tile[q] = s;
        }
        __syncthreads();
    }
}

// stage U = grid_op(sum of covering tiles) for the CTA's tile; returns #active owned nodes
template <int D>
__device__ __forceinline__ void stage_velocity(const KParams& p, const SlotView& sl, int e, const int c0[3],
                                               float4* sU) {
    using G = Geo<D>;
    for (int q = threadIdx.x; q < G::TN; q += kT) {
        int n[3];
        local_node<D>(q, n);
        const int g[3] = {c0[0] + n[0], c0[1] + n[1], D == 3 ? c0[2] + n[2] : 0};
        bool inside = g[0] < p.n_grid && g[1] < p.n_grid && (D == 2 || g[2] < p.n_grid);
        float4 out = make_float4(0.f, 0.f, 0.f, 0.f);
        if (inside) {
            const float4 pm = covered_sum<D>(p, e, g, sl.bmap, sl.tiles);
            float u0[3], u1[3];
            const bool z = grid_velocity<D>(p, g, pm, u0, u1);
            out = z ? make_float4(0.f, 0.f, 0.f, 1.f) : make_float4(u1[0], u1[1], u1[2], 0.f);
        }
        sU[q] = out;
    }
}

// ----------------------------------------------------------------- G2P
// v' = sum W U; C' = 4/dx sum W U (o - f)^T; x' = x + dt v'; key of x' for the next bin
template <int D>
__global__ void __launch_bounds__(kT) k_g2p(KParams p, SlotView sl, StateView S, StateView Sn,
                                            int* __restrict__ keys, int* __restrict__ bcount, int* flags) {
    using G = Geo<D>;
    using RC = Rec<D>;
    __shared__ float4 sU[G::TN];
    __shared__ unsigned short s_cst[G::CELLS + 1];
    const int tid = threadIdx.x;
    const int nact = *sl.nactive;
    const float c4 = 4.0f * p.inv_dx;
    for (int bi = blockIdx.x; bi < nact; bi += gridDim.x) {
        const int bid = sl.blist[bi];
        const int start = sl.bstart[bi];
        int e, c0[3];
        block_origin<D>(p, bid, e, c0);
        stage_velocity<D>(p, sl, e, c0, sU);
        if (tid == 0) s_cst[G::CELLS] = sl.cstart[(int64_t)bi * (G::CELLS + 1) + G::CELLS];
        __syncthreads();
        const int nvalid = s_cst[G::CELLS];
        for (int r0 = 0; r0 < nvalid; r0 += kT) {
            const int r = r0 + tid;
            const bool in = r < nvalid;
            int key = -1;
            if (in) {
                const int j = start + r;
                const int i = sl.sigma[j];
                float x[3];
#pragma unroll
                for (int k = 0; k < D; ++k) x[k] = __ldg(S.rec + (int64_t)i * RC::R + RC::X + k);
                float fx[3], w[3][3], dw[3][3];
                int lb[3] = {0, 0, 0};
#pragma unroll
                for (int k = 0; k < D; ++k) {
                    const float xi = x[k] * p.inv_dx;
                    const float b = floorf(xi - 0.5f);
                    fx[k] = xi - b;
                    lb[k] = (int)b - c0[k];
                    bspline(fx[k], w[k], dw[k]);
                }
                float nv[3] = {0.f, 0.f, 0.f}, nC[D * D];
#pragma unroll
                for (int q = 0; q < D * D; ++q) nC[q] = 0.f;
#pragma unroll
                for (int o0 = 0; o0 < 3; ++o0)
#pragma unroll
                    for (int o1 = 0; o1 < 3; ++o1)
#pragma unroll
                        for (int o2 = 0; o2 < (D == 3 ? 3 : 1); ++o2) {
                            const int o[3] = {o0, o1, o2};
                            float W = w[0][o0] * w[1][o1];
                            if (D == 3) W *= w[2][o2];
                            const float4 u4 = sU[tile_lin<D>(lb[0] + o0, lb[1] + o1, lb[2] + o2)];
                            const float u[3] = {u4.x, u4.y, u4.z};
#pragma unroll
                            for (int a = 0; a < D; ++a) {
                                const float wu = W * u[a];
                                nv[a] += wu;
                                const float cw = c4 * wu;
#pragma unroll
                                for (int b = 0; b < D; ++b) nC[a * D + b] = fmaf(cw, (float)o[b] - fx[b], nC[a * D + b]);
                            }
                        }
                float* dst = Sn.rec + (int64_t)j * RC::R;
                float xn[3];
                bool fin = true;
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    xn[a] = fmaf(p.dt, nv[a], x[a]);
                    dst[RC::X + a] = xn[a];
                    dst[RC::V + a] = nv[a];
                    fin = fin && isfinite(nv[a]);
                }
#pragma unroll
                for (int q = 0; q < D * D; ++q) dst[RC::C + q] = nC[q];
                if (!fin) atomicOr(flags, FLAG_NONFINITE);
                if (keys) {
                    int b[3];
                    if (base_cell<D>(p, xn, b)) {
                        int bb[3] = {b[0] >> G::LOGB, b[1] >> G::LOGB, b[2] >> G::LOGB};
                        key = block_lin<D>(p, e, bb);
                    } else {
                        atomicOr(flags, FLAG_OUT_OF_DOMAIN);
                        key = bid;  // p2g of the next step drops it into the junk bucket
                    }
                    keys[j] = key;
                }
            }
            if (keys) count_key(in, key, bcount);
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------ g2p_grad
// vh = vb' + dt xb';  Ub[b+o] += W (vh + 4/dx Cb' (o - f));  Wb = U.(vh + 4/dx Cb'(o - f));
// fb += Wb dW/df - 4/dx W Cb'^T U;  xb_t (partial) = xb' + fb/dx.
template <int D> constexpr int g2pg_smem_bytes() {
    return kT * Geo<D>::ROW * 4 + Geo<D>::CELLS * Geo<D>::NST * 16 + Geo<D>::TN * 16 + (Geo<D>::CELLS + 2) * 4;
}

template <int D>
__global__ void __launch_bounds__(kT) k_g2p_grad(KParams p, SlotView sl, StateView S,
                                                 const float* __restrict__ Sbn, float4* __restrict__ ubar,
                                                 float* __restrict__ xbp) {
    using G = Geo<D>;
    using RC = Rec<D>;
    extern __shared__ __align__(16) unsigned char smem[];
    float* s_tab = reinterpret_cast<float*>(smem);
    float4* s_cb = reinterpret_cast<float4*>(smem + kT * G::ROW * 4);
    float4* sU = s_cb + G::CELLS * G::NST;
    int* s_cst = reinterpret_cast<int*>(sU + G::TN);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nact = *sl.nactive;
    const float c4 = 4.0f * p.inv_dx;
    for (int bi = blockIdx.x; bi < nact; bi += gridDim.x) {
        const int bid = sl.blist[bi];
        const int start = sl.bstart[bi];
        int e, c0[3];
        block_origin<D>(p, bid, e, c0);
        stage_velocity<D>(p, sl, e, c0, sU);
        for (int c = tid; c <= G::CELLS; c += kT) s_cst[c] = sl.cstart[(int64_t)bi * (G::CELLS + 1) + c];
        for (int q = tid; q < G::CELLS * G::NST; q += kT) s_cb[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        __syncthreads();
        const int nvalid = s_cst[G::CELLS];
        for (int ch = 0; ch < nvalid; ch += kT) {
            const int r = ch + tid;
            if (r < nvalid) {
                const int j = start + r;
                const int i = sl.sigma[j];
                const int pid = S.pid[i];
                float x[3];
#pragma unroll
                for (int k = 0; k < D; ++k) x[k] = __ldg(S.rec + (int64_t)i * RC::R + RC::X + k);
                const float* bn = Sbn + (int64_t)pid * RC::R;
                float xb[3], vh[3], B[D * D];
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    xb[a] = __ldg(bn + RC::X + a);
                    vh[a] = fmaf(p.dt, xb[a], __ldg(bn + RC::V + a));
                }
#pragma unroll
                for (int q = 0; q < D * D; ++q) B[q] = c4 * __ldg(bn + RC::C + q);
                float fx[3], w[3][3], dw[3][3];
                int lb[3] = {0, 0, 0};
#pragma unroll
                for (int k = 0; k < D; ++k) {
                    const float xi = x[k] * p.inv_dx;
                    const float b = floorf(xi - 0.5f);
                    fx[k] = xi - b;
                    lb[k] = (int)b - c0[k];
                    bspline(fx[k], w[k], dw[k]);
                }
                float cp[3];  // c' = vh - B f
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    float s = vh[a];
#pragma unroll
                    for (int b = 0; b < D; ++b) s = fmaf(-B[a * D + b], fx[b], s);
                    cp[a] = s;
                }
                float fb[3] = {0.f, 0.f, 0.f};
#pragma unroll
                for (int o0 = 0; o0 < 3; ++o0)
#pragma unroll
                    for (int o1 = 0; o1 < 3; ++o1)
#pragma unroll
                        for (int o2 = 0; o2 < (D == 3 ? 3 : 1); ++o2) {
                            const int o[3] = {o0, o1, o2};
                            float wo[3] = {w[0][o0], w[1][o1], D == 3 ? w[2][o2] : 1.0f};
                            const float W = wo[0] * wo[1] * wo[2];
                            float gW[3];
                            gW[0] = dw[0][o0] * wo[1] * wo[2];
                            gW[1] = wo[0] * dw[1][o1] * wo[2];
                            if (D == 3) gW[2] = wo[0] * wo[1] * dw[2][o2];
                            const float4 u4 = sU[tile_lin<D>(lb[0] + o0, lb[1] + o1, lb[2] + o2)];
                            const float u[3] = {u4.x, u4.y, u4.z};
                            float Wb = 0.0f;
#pragma unroll
                            for (int a = 0; a < D; ++a) {
                                float t = cp[a];
#pragma unroll
                                for (int b = 0; b < D; ++b) t = fmaf(B[a * D + b], (float)o[b], t);
                                Wb = fmaf(u[a], t, Wb);
                            }
#pragma unroll
                            for (int k = 0; k < D; ++k) {
                                float btu = 0.0f;
#pragma unroll
                                for (int a = 0; a < D; ++a) btu = fmaf(B[a * D + k], u[a], btu);
                                fb[k] = fmaf(Wb, gW[k], fb[k]) - W * btu;
                            }
                        }
#pragma unroll
                for (int k = 0; k < D; ++k) xbp[(int64_t)j * D + k] = fmaf(p.inv_dx, fb[k], xb[k]);
                float* row = s_tab + tid * G::ROW;
#pragma unroll
                for (int k = 0; k < D; ++k)
#pragma unroll
                    for (int o = 0; o < 3; ++o) row[3 * k + o] = w[k][o];
#pragma unroll
                for (int a = 0; a < D; ++a) row[3 * D + a] = cp[a];
#pragma unroll
                for (int q = 0; q < D * D; ++q) row[4 * D + q] = B[q];
            }
            __syncthreads();
            for (int c = warp; c < G::CELLS; c += kW) {
                const int lo = max(s_cst[c], ch), hi = min(s_cst[c + 1], ch + kT);
                if (lo >= hi) continue;
                const float4 acc = cell_rows<D, false>(s_tab - ch * G::ROW, lo, hi, lane);
                if (lane < G::NST) {
                    float4& dst = s_cb[c * G::NST + lane];
                    dst.x += acc.x; dst.y += acc.y; dst.z += acc.z;
                }
            }
            __syncthreads();
        }
        float4* tile = ubar + (int64_t)bi * G::TN;
        for (int q = tid; q < G::TN; q += kT) tile[q] = node_gather<D>(s_cb, q);
        __syncthreads();
    }
}

// ------------------------------------------------------------ p2g_grad
// staging fuses grid_op_grad (select rule): ub = z ? 0 : Ub;
// Pb = ub/(M + eps); Mb = -(ub . u0)/(M + eps).  Then per particle:
// vb = sum W m Pb; Ab = sum W Pb dpos^T; Wb = Pb.(m v + A dpos) + Mb m;
// fb += Wb dW/df - dx W A^T Pb; Cb = m Ab + dt Ftb F^T; taub = -dt V 4/dx^2 Ab;
// Ftb = Fb' + stress/actuation adjoint; Fb = (I + dt C)^T Ftb; xb += fb/dx.
template <int D>
__global__ void __launch_bounds__(kT) k_p2g_grad(KParams p, SlotView sl, StateView S,
                                                 const int32_t* __restrict__ aid,
                                                 const float* __restrict__ alpha,
                                                 const float4* __restrict__ ubar,
                                                 const float* __restrict__ Sbn,
                                                 const float* __restrict__ xbp,
                                                 float* __restrict__ Sb, float* __restrict__ abar_part,
                                                 int* flags) {
    using G = Geo<D>;
    using RC = Rec<D>;
    __shared__ float4 sG[G::TN];
    __shared__ float s_ab[kW][32];
    __shared__ int s_nvalid;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nact = *sl.nactive;
    for (int bi = blockIdx.x; bi < nact; bi += gridDim.x) {
        const int bid = sl.blist[bi];
        const int start = sl.bstart[bi];
        int e, c0[3];
        block_origin<D>(p, bid, e, c0);
        for (int q = tid; q < G::TN; q += kT) {
            int n[3];
            local_node<D>(q, n);
            const int g[3] = {c0[0] + n[0], c0[1] + n[1], D == 3 ? c0[2] + n[2] : 0};
            const bool inside = g[0] < p.n_grid && g[1] < p.n_grid && (D == 2 || g[2] < p.n_grid);
            float4 out = make_float4(0.f, 0.f, 0.f, 0.f);
            if (inside) {
                const float4 pm = covered_sum<D>(p, e, g, sl.bmap, sl.tiles);
                const float4 ub = covered_sum<D>(p, e, g, sl.bmap, ubar);
                float u0[3], u1[3];
                const bool z = grid_velocity<D>(p, g, pm, u0, u1);
                if (!z) {
                    const float denom = pm.w + p.eps_mass;
                    const float dot = ub.x * u0[0] + ub.y * u0[1] + (D == 3 ? ub.z * u0[2] : 0.0f);
                    out = make_float4(ub.x / denom, ub.y / denom, D == 3 ? ub.z / denom : 0.0f, -dot / denom);
                }
            }
            sG[q] = out;
        }
        for (int q = tid; q < kW * 32; q += kT) (&s_ab[0][0])[q] = 0.0f;
        if (tid == 0) s_nvalid = sl.cstart[(int64_t)bi * (G::CELLS + 1) + G::CELLS];
        __syncthreads();
        const int nvalid = s_nvalid;
        for (int r0 = 0; r0 < nvalid; r0 += kT) {
            const int r = r0 + tid;
            const bool in = r < nvalid;
            int a_id = -1;
            float abar = 0.0f;
            if (in) {
                const int j = start + r;
                const int i = sl.sigma[j];
                const int pid = S.pid[i];
                float rr[RC::R];
                load_rec<D>(S.rec + (int64_t)i * RC::R, rr);
                const float* x = rr + RC::X;
                const float* v = rr + RC::V;
                const float* C = rr + RC::C;
                const float* F = rr + RC::F;
                float fx[3], w[3][3], dw[3][3];
                int lb[3] = {0, 0, 0};
#pragma unroll
                for (int k = 0; k < D; ++k) {
                    const float xi = x[k] * p.inv_dx;
                    const float b = floorf(xi - 0.5f);
                    fx[k] = xi - b;
                    lb[k] = (int)b - c0[k];
                    bspline(fx[k], w[k], dw[k]);
                }
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
                a_id = aid ? aid[pid] : -1;
                const float act = a_id >= 0 ? alpha[a_id] : 0.0f;
                float tau[D * D], A[D * D];
                kirchhoff<D>(p, Ft, act, tau);
#pragma unroll
                for (int q = 0; q < D * D; ++q) A[q] = fmaf(p.stress_scale, tau[q], p.p_mass * C[q]);
                float vb[3] = {0.f, 0.f, 0.f}, fb[3] = {0.f, 0.f, 0.f}, Ab[D * D];
#pragma unroll
                for (int q = 0; q < D * D; ++q) Ab[q] = 0.0f;
#pragma unroll
                for (int o0 = 0; o0 < 3; ++o0)
#pragma unroll
                    for (int o1 = 0; o1 < 3; ++o1)
#pragma unroll
                        for (int o2 = 0; o2 < (D == 3 ? 3 : 1); ++o2) {
                            const int o[3] = {o0, o1, o2};
                            float wo[3] = {w[0][o0], w[1][o1], D == 3 ? w[2][o2] : 1.0f};
                            const float W = wo[0] * wo[1] * wo[2];
                            float gW[3];
                            gW[0] = dw[0][o0] * wo[1] * wo[2];
                            gW[1] = wo[0] * dw[1][o1] * wo[2];
                            if (D == 3) gW[2] = wo[0] * wo[1] * dw[2][o2];
                            float dpos[3];
#pragma unroll
                            for (int k = 0; k < D; ++k) dpos[k] = ((float)o[k] - fx[k]) * p.dx;
                            const float4 g4 = sG[tile_lin<D>(lb[0] + o0, lb[1] + o1, lb[2] + o2)];
                            const float gP[3] = {g4.x, g4.y, g4.z};
                            float Wb = g4.w * p.p_mass;
#pragma unroll
                            for (int a = 0; a < D; ++a) {
                                vb[a] = fmaf(W * p.p_mass, gP[a], vb[a]);
                                float mom = p.p_mass * v[a];
                                const float wg = W * gP[a];
#pragma unroll
                                for (int b = 0; b < D; ++b) {
                                    Ab[a * D + b] = fmaf(wg, dpos[b], Ab[a * D + b]);
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
                const float* bn = Sbn + (int64_t)pid * RC::R;
#pragma unroll
                for (int q = 0; q < D * D; ++q) {
                    taub[q] = p.stress_scale * Ab[q];
                    Ftb[q] = __ldg(bn + RC::F + q);
                }
                abar = kirchhoff_adj<D>(p, Ft, a_id >= 0, act, taub, Ftb);
                float* dst = Sb + (int64_t)pid * RC::R;
                bool fin = true;
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
                        dst[RC::F + a * D + b] = sF;
                        dst[RC::C + a * D + b] = fmaf(p.dt, sC, p.p_mass * Ab[a * D + b]);
                        fin = fin && isfinite(sF);
                    }
#pragma unroll
                for (int a = 0; a < D; ++a) {
                    dst[RC::X + a] = fmaf(p.inv_dx, fb[a], xbp[(int64_t)j * D + a]);
                    dst[RC::V + a] = vb[a];
                }
                if (!fin) atomicOr(flags, FLAG_NONFINITE);
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
            for (int wv = 0; wv < kW; ++wv) s += s_ab[wv][tid];
            abar_part[(int64_t)bi * p.n_act + tid] = s;
        }
        __syncthreads();
    }
}

// alpha_bar_t[a] = sum over active blocks (list order) of abar_part[b][a]
__global__ void k_reduce_abar(const int* __restrict__ nactive, const float* __restrict__ part, int n_act,
                              float* __restrict__ out) {
    const int a = blockIdx.x;
    const int n = *nactive;
    float s = 0.0f;
    for (int b = threadIdx.x; b < n; b += 32) s += part[(int64_t)b * n_act + a];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (threadIdx.x == 0) out[a] = s;
}

// measurement: number of distinct grid nodes with M > 0 in a slot's tiles.  Each
// node is counted once, by the first active block in covered_sum's order.
template <int D>
__global__ void __launch_bounds__(kT) k_count_active(KParams p, SlotView sl, unsigned long long* count) {
    using G = Geo<D>;
    const int nact = *sl.nactive;
    for (int bi = blockIdx.x; bi < nact; bi += gridDim.x) {
        int e, c0[3];
        block_origin<D>(p, sl.blist[bi], e, c0);
        for (int q = threadIdx.x; q < G::TN; q += kT) {
            int n[3];
            local_node<D>(q, n);
            const int g[3] = {c0[0] + n[0], c0[1] + n[1], D == 3 ? c0[2] + n[2] : 0};
            if (g[0] >= p.n_grid || g[1] >= p.n_grid || (D == 3 && g[2] >= p.n_grid)) continue;
            if (covered_sum<D>(p, e, g, sl.bmap, sl.tiles).w <= 0.0f) continue;
            // first active covering block (same enumeration as covered_sum)
            int first = -1;
            for (int a = 0; a < 2 && first < 0; ++a)
                for (int b = 0; b < 2 && first < 0; ++b)
                    for (int c = 0; c < (D == 3 ? 2 : 1) && first < 0; ++c) {
                        const int off[3] = {a, b, c};
                        int bb[3] = {0, 0, 0};
                        bool ok = true;
                        for (int k = 0; k < D; ++k) {
                            const int b0 = g[k] >> G::LOGB, l0 = g[k] & (G::B - 1);
                            if (off[k] == 1 && !(l0 < 2 && b0 >= 1)) ok = false;
                            bb[k] = b0 - off[k];
                            if (bb[k] >= p.nb) ok = false;
                        }
                        if (!ok) continue;
                        const int ti = sl.bmap[block_lin<D>(p, e, bb)];
                        if (ti >= 0) first = ti;
                    }
            if (first == bi) atomicAdd(count, 1ull);
        }
    }
}

inline unsigned nblk(int64_t n) { return (unsigned)((n + kT - 1) / kT); }

int g_grid[4][2];  // persistent grid size per kernel kind and dimension (set by tile_init)

}  // namespace

#define DISPATCH(D, ...) \
    do {                 \
        if ((D) == 2) {  \
            constexpr int DIM = 2; __VA_ARGS__; \
        } else {         \
            constexpr int DIM = 3; __VA_ARGS__; \
        }                \
    } while (0)

static int occupancy_grid(const void* fn, int smem) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, kT, smem);
    return sms * (per > 0 ? per : 1);
}

cudaError_t tile_init() {
    static bool done = false;
    if (done) return cudaSuccess;
    cudaError_t e = cudaSuccess;
    DISPATCH(2, {
        e = cudaFuncSetAttribute(k_p2g<DIM>, cudaFuncAttributeMaxDynamicSharedMemorySize, p2g_smem_bytes<DIM>());
        if (e) return e;
        e = cudaFuncSetAttribute(k_g2p_grad<DIM>, cudaFuncAttributeMaxDynamicSharedMemorySize, g2pg_smem_bytes<DIM>());
        if (e) return e;
        g_grid[0][0] = occupancy_grid((const void*)k_p2g<DIM>, p2g_smem_bytes<DIM>());
        g_grid[1][0] = occupancy_grid((const void*)k_g2p<DIM>, 0);
        g_grid[2][0] = occupancy_grid((const void*)k_g2p_grad<DIM>, g2pg_smem_bytes<DIM>());
        g_grid[3][0] = occupancy_grid((const void*)k_p2g_grad<DIM>, 0);
    });
    DISPATCH(3, {
        e = cudaFuncSetAttribute(k_p2g<DIM>, cudaFuncAttributeMaxDynamicSharedMemorySize, p2g_smem_bytes<DIM>());
        if (e) return e;
        e = cudaFuncSetAttribute(k_g2p_grad<DIM>, cudaFuncAttributeMaxDynamicSharedMemorySize, g2pg_smem_bytes<DIM>());
        if (e) return e;
        g_grid[0][1] = occupancy_grid((const void*)k_p2g<DIM>, p2g_smem_bytes<DIM>());
        g_grid[1][1] = occupancy_grid((const void*)k_g2p<DIM>, 0);
        g_grid[2][1] = occupancy_grid((const void*)k_g2p_grad<DIM>, g2pg_smem_bytes<DIM>());
        g_grid[3][1] = occupancy_grid((const void*)k_p2g_grad<DIM>, 0);
    });
    done = true;
    return cudaGetLastError();
}

static unsigned pgrid(const KParams& p, int kind) {
    const int g = g_grid[kind][p.dim == 3 ? 1 : 0];
    return (unsigned)(p.max_active < g ? p.max_active : g);
}

void launch_bin_keys(const KParams& p, const float* rec, int* keys, int* bcount, int* flags, cudaStream_t s) {
    DISPATCH(p.dim, k_bin_keys<DIM><<<nblk(p.N * p.E), kT, 0, s>>>(p, rec, keys, bcount, flags));
}
void launch_bin_scan(const KParams& p, int* bcount, int* cursor, const SlotView& sl, int* flags, cudaStream_t s) {
    k_bin_scan<<<1, kScanT, 0, s>>>(p, bcount, cursor, sl, flags);
}
void launch_bin_scatter(const KParams& p, const int* keys, int* cursor, int* sigma, cudaStream_t s) {
    k_bin_scatter<<<nblk(p.N * p.E), kT, 0, s>>>(p, keys, cursor, sigma);
}
void launch_p2g(const KParams& p, const SlotView& sl, const StateView& S, const StateView& Sn,
                const int32_t* aid, const float* alpha_t, int* flags, cudaStream_t s) {
    DISPATCH(p.dim, k_p2g<DIM><<<pgrid(p, 0), kT, p2g_smem_bytes<DIM>(), s>>>(p, sl, S, Sn, aid, alpha_t, flags));
}
void launch_g2p(const KParams& p, const SlotView& sl, const StateView& S, const StateView& Sn, int* keys,
                int* bcount, int* flags, cudaStream_t s) {
    DISPATCH(p.dim, k_g2p<DIM><<<pgrid(p, 1), kT, 0, s>>>(p, sl, S, Sn, keys, bcount, flags));
}
void launch_g2p_grad(const KParams& p, const SlotView& sl, const StateView& S, const float* Sbn,
                     float4* ubar, float* xbp, cudaStream_t s) {
    DISPATCH(p.dim, k_g2p_grad<DIM><<<pgrid(p, 2), kT, g2pg_smem_bytes<DIM>(), s>>>(p, sl, S, Sbn, ubar, xbp));
}
void launch_p2g_grad(const KParams& p, const SlotView& sl, const StateView& S, const int32_t* aid,
                     const float* alpha_t, const float4* ubar, const float* Sbn, const float* xbp,
                     float* Sb, float* abar_part, int* flags, cudaStream_t s) {
    DISPATCH(p.dim, k_p2g_grad<DIM><<<pgrid(p, 3), kT, 0, s>>>(p, sl, S, aid, alpha_t, ubar, Sbn, xbp, Sb, abar_part, flags));
}
void launch_count_active(const KParams& p, const SlotView& sl, int64_t* count, cudaStream_t s) {
    cudaMemsetAsync(count, 0, sizeof(int64_t), s);
    DISPATCH(p.dim, k_count_active<DIM><<<pgrid(p, 1), kT, 0, s>>>(p, sl, (unsigned long long*)count));
}
void launch_reduce_abar(const KParams& p, const int* nactive, const float* abar_part, float* alpha_bar_t,
                        cudaStream_t s) {
    if (p.n_act > 0) k_reduce_abar<<<p.n_act, 32, 0, s>>>(nactive, abar_part, p.n_act, alpha_bar_t);
}

}  // namespace mpm
