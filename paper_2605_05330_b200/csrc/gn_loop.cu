// gn_loop.cu -- the GN iteration loop: one persistent, co-resident kernel that
// runs every step of run_wrgn on the device.
//
// Reference: dynamics.py:_step 102-108 (the update), run_wrgn 129-180 (loop,
// step_inf, fallbacks, non-finite stop, early exit, trace), energy 210-219 and
// weighted_mass 222-224 (fused here as per-iteration dot products).
//
// Per iteration k, one pass over the relabeled adjacency (gn_internal.cuh):
//   s_r  = sum_{j in N(r)} yg_j          gathered values of step k
//   y_r  = v_r * x_r                     (bitwise the y the reference forms)
//   d_r  = y_r + gamma_k * s_r           separately rounded, no FMA
//   x'_r = d_r > 1e-9 ? y_r / d_r : 0.5  counted fallback
//   yg'_r = v_r * x'_r                   published for step k+1
// fused with the per-iteration reductions: max|x'-x|, the fallback count,
// the non-finite flag and fixed-order fp64 block partials of w.x' (the
// objective) and, in trace mode, y.y, y.s, w.x (the energy terms of the
// pre-step state).  Block stats go to a ring (plain stores, no atomics) that
// all blocks fold cooperatively every kRing iterations.
//
// Work, decided once per (graph, grid, mode) on the host (build_plan):
//   CTA items   long slices (the 32 warps split the slice's blocks) and hub
//               rows (the 32 warps split the row); per-warp partials meet in
//               shared memory and are folded in warp order
//   warp items  short slices: one warp per slice, one thread per row,
//               sequential sum in the reference's order (bitwise)
// balanced longest-processing-time-first over CTAs and warps.  The index
// blocks of as many items as fit stay resident in shared memory for the whole
// run; the rest stream from global memory every iteration.  A grid barrier
// separates iterations.
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <climits>
#include <cstring>
#include <map>
#include <mutex>
#include <numeric>
#include <queue>
#include <vector>

#include "gn_internal.cuh"

namespace gn {

constexpr int kThreads = 1024;  // one CTA per SM
constexpr int kWarps = kThreads / 32;
constexpr int kSlots = 4;       // CTA items per phase (shared-memory partial slots)
constexpr int kRing = 1024;     // iterations of block stats kept before a fold
constexpr int kRingW = 8;       // per block: 4 dot terms, max|dx|, fallbacks, non-finite, pad

enum ItemKind : int32_t { kSplit = 0, kHub = 1, kWhole = 2, kHubSeq = 3 };

// One unit of work.  id: slice (kSplit/kWhole) or first hub row (kHub,
// kHubSeq); len: blocks (slices) or degree (hub) or row count (kHubSeq);
// smem: offset of the resident index blocks in 16-byte words, -1 = global.
struct Item {
    int32_t id, len, smem, kind;
};

template <typename TS, typename TG>
struct LoopArgs {
    int64_t n;
    int32_t nhub;
    const int32_t* __restrict__ hub_ptr;
    const int32_t* __restrict__ hub_col;
    const int64_t* __restrict__ slice_ptr;
    const int32_t* __restrict__ row_deg;
    const void* __restrict__ sell;
    const TS* __restrict__ v;
    const TS* __restrict__ w;
    TS* x[2];
    TG* yg[2];
    const int32_t* __restrict__ cta_ptr;   // [G+1] into items (CTA items)
    const int32_t* __restrict__ warp_ptr;  // [G*kWarps+1] into items (warp items)
    const Item* __restrict__ items;
    const int32_t* __restrict__ smem_words;  // [G] resident 16-byte words per CTA
    int smem_resident_off;                   // byte offset of the resident area
    const double* __restrict__ gammas;
    int iters;
    double final_gamma;
    int early_exit;
    double* step_inf;  // [iters]   max over blocks of max|x'-x|
    double* fb;        // [iters]   fallback count (exact in fp64)
    int* bad;          // [iters]   1 if a non-finite state appeared
    int* status;       // [0] iterations run
    double* dots;      // [(iters+1)][4]: y.y, y.s, w.x (pre), w.x' (post)
    double* ring;      // [kRing][grid][kRingW]
    unsigned int* barrier;
    double* x_hist;    // optional [iters][n], original order
    const int32_t* __restrict__ perm;
};

struct Stats {
    double mx;
    unsigned int fbc;
    int bad;
    double acc[4];
};

template <typename T>
__device__ __forceinline__ T tabs(T v) { return v < T(0) ? -v : v; }

// Per-row state, fetched before the row's neighbour sum so its latency hides
// under the gathers.
template <typename TS>
struct RowIn {
    TS x, v;
    double w;
};

template <typename TS, typename TG>
__device__ __forceinline__ RowIn<TS> row_in(const LoopArgs<TS, TG>& a, int r, int cur) {
    return RowIn<TS>{a.x[cur][r], __ldg(a.v + r), (double)__ldg(a.w + r)};
}

// The elementwise half of _step for row r (new id) whose neighbour sum is s.
template <typename TS, typename TG, bool TRACE>
__device__ __forceinline__ void update_row(const LoopArgs<TS, TG>& a, int r, TS s, const RowIn<TS>& in, int cur,
                                           TS g, int k, bool tail, Stats& st) {
    using A = Arith<TS>;
    const TS xi = in.x, vi = in.v;
    const double wi = in.w;
    const TS yi = A::mul(vi, xi);                    // dynamics.py:104
    if (TRACE) {
        st.acc[0] = __dadd_rn(st.acc[0], __dmul_rn((double)yi, (double)yi));
        st.acc[1] = __dadd_rn(st.acc[1], __dmul_rn((double)yi, (double)s));
        st.acc[2] = __dadd_rn(st.acc[2], __dmul_rn(wi, (double)xi));
    }
    if (tail) return;
    const TS d = A::add(yi, A::mul(g, s));          // dynamics.py:105
    const bool ok = (double)d > kSafeDiv;            // dynamics.py:106
    const TS o = ok ? A::div(yi, d) : TS(kFallback); // dynamics.py:107
    a.x[cur ^ 1][r] = o;
    a.yg[cur ^ 1][r] = (TG)A::mul(vi, o);
    const double diff = (double)tabs(A::sub(o, xi));  // dynamics.py:165
    if (!(diff <= st.mx)) st.mx = diff;
    st.fbc += ok ? 0u : 1u;
    if (!isfinite((double)o)) st.bad = 1;
    st.acc[3] = __dadd_rn(st.acc[3], __dmul_rn(wi, (double)o));  // objective w . x'
    if (a.x_hist) a.x_hist[(size_t)k * (size_t)a.n + (size_t)__ldg(a.perm + r)] = (double)o;
}

// Blocked-SELL lane vectors: one 16-byte load gives B consecutive neighbours.
template <typename TI>
struct LaneVec;
template <>
struct LaneVec<uint16_t> {
    static constexpr int B = 8;
    __device__ static __forceinline__ int get(const uint4& v, int t) {
        const unsigned w = t < 4 ? (t < 2 ? v.x : v.y) : (t < 6 ? v.z : v.w);
        return (int)((t & 1) ? (w >> 16) : (w & 0xffffu));
    }
};
template <>
struct LaneVec<int32_t> {
    static constexpr int B = 4;
    __device__ static __forceinline__ int get(const uint4& v, int t) {
        return (int)(t == 0 ? v.x : t == 1 ? v.y : t == 2 ? v.z : v.w);
    }
};

template <bool SMEM>
__device__ __forceinline__ uint4 load_vec(const uint4* p) {
    if (SMEM) return *p;
    return __ldg(p);
}

// Sequential sum over blocks [bb, be) of one slice row (this lane), masked by
// the row's degree d.  A batch issues NB vector loads and NB*B gathers before
// any add; the adds stay in position order (the reference's order).  Blocks
// that lie entirely inside the row skip the mask.
template <typename TS, typename TG, typename TI, bool SMEM>
__device__ __forceinline__ TS sum_blocks(const uint4* __restrict__ base, const TG* __restrict__ yg, int d,
                                         int bb, int be) {
    using A = Arith<TS>;
    using V = LaneVec<TI>;
    constexpr int B = V::B;
    constexpr int NB = (sizeof(TG) == 4 ? 16 : 8) / B > 0 ? (sizeof(TG) == 4 ? 16 : 8) / B : 1;
    TS s = TS(0);
    int b = bb;
    for (; b + NB <= be && (b + NB) * B <= d; b += NB) {
        uint4 v[NB];
#pragma unroll
        for (int u = 0; u < NB; ++u) v[u] = load_vec<SMEM>(base + (size_t)(b + u) * kSlice);
        TG y[NB * B];
#pragma unroll
        for (int u = 0; u < NB; ++u)
#pragma unroll
            for (int t = 0; t < B; ++t) y[u * B + t] = yg[V::get(v[u], t)];
#pragma unroll
        for (int q = 0; q < NB * B; ++q) s = A::add(s, (TS)y[q]);
    }
    for (; b < be && b * B < d; ++b) {
        const uint4 v = load_vec<SMEM>(base + (size_t)b * kSlice);
        TG y[B];
#pragma unroll
        for (int t = 0; t < B; ++t) y[t] = (b * B + t < d) ? yg[V::get(v, t)] : TG(0);
#pragma unroll
        for (int t = 0; t < B; ++t) s = A::add(s, (TS)y[t]);
    }
    return s;
}

template <typename TS, typename TG, typename TI>
__device__ __forceinline__ TS slice_sum(const LoopArgs<TS, TG>& a, const Item& it, const uint4* s_res,
                                        const TG* __restrict__ yg, int lane, int d, int bb, int be) {
    if (it.smem >= 0) return sum_blocks<TS, TG, TI, true>(s_res + it.smem + lane, yg, d, bb, be);
    const uint4* g = reinterpret_cast<const uint4*>((const TI*)a.sell + __ldg(a.slice_ptr + it.id)) + lane;
    return sum_blocks<TS, TG, TI, false>(g, yg, d, bb, be);
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = Arith<T>::add(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// One pass over this CTA's items.
template <typename TS, typename TG, typename TI, bool TRACE>
__device__ void pass(const LoopArgs<TS, TG>& a, int k, bool tail, Stats& st, TS* s_part, const uint4* s_res) {
    using A = Arith<TS>;
    const int cur = k & 1;
    const TG* __restrict__ yg = a.yg[cur];
    const TS g = tail ? TS(0) : (TS)a.gammas[k];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int c0 = __ldg(a.cta_ptr + blockIdx.x), c1 = __ldg(a.cta_ptr + blockIdx.x + 1);
    const int gw = blockIdx.x * kWarps + warp;
    const int w0 = __ldg(a.warp_ptr + gw), w1 = __ldg(a.warp_ptr + gw + 1);
    bool warp_done = false;
    // CTA items in phases of kSlots; the warp items run inside the first
    // phase, between the partial sums and the barrier that publishes them
    for (int p0 = c0;; p0 += kSlots) {
        const int pn = min(kSlots, c1 - p0);
        for (int q = 0; q < pn; ++q) {
            const Item it = a.items[p0 + q];
            if (it.kind == kSplit) {
                const int d = __ldg(a.row_deg + it.id * kSlice + lane);
                const int bb = it.len * warp / kWarps, be = it.len * (warp + 1) / kWarps;
                s_part[(q * kWarps + warp) * kSlice + lane] = slice_sum<TS, TG, TI>(a, it, s_res, yg, lane, d, bb, be);
            } else {  // kHub: warp w sums elements [w*deg/W, (w+1)*deg/W) of the row
                const int beg = __ldg(a.hub_ptr + it.id);
                const int eb = beg + (int)((int64_t)it.len * warp / kWarps);
                const int ee = beg + (int)((int64_t)it.len * (warp + 1) / kWarps);
                TS s = TS(0);
                for (int p = eb + lane; p < ee; p += 32) s = A::add(s, (TS)yg[__ldg(a.hub_col + p)]);
                s = warp_sum(s);
                if (lane == 0) s_part[(q * kWarps + warp) * kSlice] = s;
            }
        }
        if (!warp_done) {
            warp_done = true;
            for (int i = w0; i < w1; ++i) {
                const Item it = a.items[i];
                if (it.kind == kWhole) {
                    const int64_t r = (int64_t)a.nhub + (int64_t)it.id * kSlice + lane;
                    const bool valid = r < a.n;
                    RowIn<TS> in{};
                    int d = 0;
                    if (valid) {
                        d = __ldg(a.row_deg + (size_t)it.id * kSlice + lane);
                        in = row_in(a, (int)r, cur);
                    }
                    const TS sum = slice_sum<TS, TG, TI>(a, it, s_res, yg, lane, d, 0, it.len);
                    if (valid) update_row<TS, TG, TRACE>(a, (int)r, sum, in, cur, g, k, tail, st);
                } else {  // kHubSeq (EXACT): one thread per hub row, sequential
                    if (lane < it.len) {
                        const int h = it.id + lane;
                        const RowIn<TS> in = row_in(a, h, cur);
                        TS s = TS(0);
                        for (int p = __ldg(a.hub_ptr + h); p < __ldg(a.hub_ptr + h + 1); ++p)
                            s = A::add(s, (TS)yg[__ldg(a.hub_col + p)]);
                        update_row<TS, TG, TRACE>(a, h, s, in, cur, g, k, tail, st);
                    }
                }
            }
        }
        if (pn <= 0) break;
        __syncthreads();
        for (int q = warp; q < pn; q += kWarps) {
            const Item it = a.items[p0 + q];
            if (it.kind == kSplit) {
                const int r = a.nhub + it.id * kSlice + lane;
                const RowIn<TS> in = row_in(a, r, cur);
                TS tot = TS(0);
#pragma unroll 8
                for (int w = 0; w < kWarps; ++w) tot = A::add(tot, s_part[(q * kWarps + w) * kSlice + lane]);
                update_row<TS, TG, TRACE>(a, r, tot, in, cur, g, k, tail, st);
            } else if (lane == 0) {
                const RowIn<TS> in = row_in(a, it.id, cur);
                TS tot = TS(0);
                for (int w = 0; w < kWarps; ++w) tot = A::add(tot, s_part[(q * kWarps + w) * kSlice]);
                update_row<TS, TG, TRACE>(a, it.id, tot, in, cur, g, k, tail, st);
            }
        }
        __syncthreads();
    }
}

// Block-level fold of the per-thread stats; thread 0 stores them (plain
// stores, no atomics) in this iteration's ring slot.
template <bool TRACE>
__device__ void publish(const Stats& st0, double* __restrict__ ring_slot) {
    __shared__ double s_acc[kWarps][4];
    __shared__ double s_mx[kWarps];
    __shared__ unsigned int s_fb[kWarps];
    __shared__ int s_bad[kWarps];
    Stats st = st0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        double m = __shfl_xor_sync(0xffffffffu, st.mx, o);
        if (!(m <= st.mx)) st.mx = m;
        st.fbc += __shfl_xor_sync(0xffffffffu, st.fbc, o);
        st.bad |= __shfl_xor_sync(0xffffffffu, st.bad, o);
    }
#pragma unroll
    for (int q = TRACE ? 0 : 3; q < 4; ++q) st.acc[q] = warp_sum_d(st.acc[q]);
    if (lane == 0) {
        s_mx[warp] = st.mx;
        s_fb[warp] = st.fbc;
        s_bad[warp] = st.bad;
#pragma unroll
        for (int q = 0; q < 4; ++q) s_acc[warp][q] = st.acc[q];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double mx = 0.0, acc[4] = {0.0, 0.0, 0.0, 0.0};
        unsigned int f = 0;
        int bad = 0;
        for (int q = 0; q < kWarps; ++q) {
            if (!(s_mx[q] <= mx)) mx = s_mx[q];
            f += s_fb[q];
            bad |= s_bad[q];
#pragma unroll
            for (int c = TRACE ? 0 : 3; c < 4; ++c) acc[c] = __dadd_rn(acc[c], s_acc[q][c]);
        }
        double* dst = ring_slot + (size_t)blockIdx.x * kRingW;
#pragma unroll
        for (int c = 0; c < 4; ++c) dst[c] = acc[c];
        dst[4] = mx;
        dst[5] = (double)f;
        dst[6] = bad ? 1.0 : 0.0;
    }
}

struct FoldOut {
    int iters;
    double* step_inf;
    double* fb;
    int* bad;
    double* dots;
};

// All blocks: fold ring slots [0, count) (iterations k0..k0+count-1), one
// warp per (slot, quantity), block order fixed.
__device__ void fold_ring(const double* ring, int count, int k0, const FoldOut& o) {
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * kWarps + (threadIdx.x >> 5), nw = gridDim.x * kWarps;
    const int G = gridDim.x;
    for (int t = gw; t < count * 7; t += nw) {
        const int slot = t / 7, c = t % 7;
        const double* src = ring + (size_t)slot * G * kRingW + c;
        const int k = k0 + slot;
        if (c == 4 || c == 6) {
            double m = 0.0;
            for (int b = lane; b < G; b += 32) {
                const double v = __ldcg(src + (size_t)b * kRingW);
                if (!(v <= m)) m = v;
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const double v = __shfl_xor_sync(0xffffffffu, m, off);
                if (!(v <= m)) m = v;
            }
            if (lane == 0 && k < o.iters) {
                if (c == 4) o.step_inf[k] = m;
                else o.bad[k] = m != 0.0 ? 1 : 0;
            }
        } else {
            double s = 0.0;
            for (int b = lane; b < G; b += 32) s = __dadd_rn(s, __ldcg(src + (size_t)b * kRingW));
            s = warp_sum_d(s);
            if (lane == 0) {
                if (c == 5) { if (k < o.iters) o.fb[k] = s; }
                else o.dots[(size_t)k * 4 + c] = s;
            }
        }
    }
}

// Every block computes max|dx| of one iteration from the ring (early exit).
__device__ double ring_step_inf(const double* ring_slot) {
    __shared__ double s_m;
    if (threadIdx.x < 32) {
        double m = 0.0;
        for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) {
            const double v = __ldcg(ring_slot + (size_t)b * kRingW + 4);
            if (!(v <= m)) m = v;
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const double v = __shfl_xor_sync(0xffffffffu, m, off);
            if (!(v <= m)) m = v;
        }
        if (threadIdx.x == 0) s_m = m;
    }
    __syncthreads();
    return s_m;
}

template <typename TS, typename TG, typename TI, bool TRACE>
__global__ void __launch_bounds__(kThreads, 1) k_gn_loop(LoopArgs<TS, TG> a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TS* s_part = (TS*)smem_raw;
    uint4* s_res = (uint4*)(smem_raw + a.smem_resident_off);
    // resident index blocks: copied once, used every iteration
    {
        const int nwords = __ldg(a.smem_words + blockIdx.x);
        if (nwords > 0) {
            const int c0 = a.cta_ptr[blockIdx.x], c1 = a.cta_ptr[blockIdx.x + 1];
            const int w0 = a.warp_ptr[blockIdx.x * kWarps], w1 = a.warp_ptr[(blockIdx.x + 1) * kWarps];
            for (int part = 0; part < 2; ++part) {
                const int i0 = part ? w0 : c0, i1 = part ? w1 : c1;
                for (int i = i0; i < i1; ++i) {
                    const Item it = a.items[i];
                    if (it.smem < 0 || (it.kind != kSplit && it.kind != kWhole)) continue;
                    const uint4* src = reinterpret_cast<const uint4*>((const TI*)a.sell + a.slice_ptr[it.id]);
                    for (int t = threadIdx.x; t < it.len * kSlice; t += blockDim.x) s_res[it.smem + t] = __ldg(src + t);
                }
            }
        }
        __syncthreads();
    }
    const FoldOut fo{a.iters, a.step_inf, a.fb, a.bad, a.dots};
    unsigned int bar = 0;
    int ran = 0, k0 = 0;
    const size_t ring_stride = (size_t)gridDim.x * kRingW;
    for (int k = 0; k < a.iters; ++k) {
        Stats st{0.0, 0u, 0, {0.0, 0.0, 0.0, 0.0}};
        pass<TS, TG, TI, TRACE>(a, k, false, st, s_part, s_res);
        double* slot = a.ring + (size_t)(k - k0) * ring_stride;
        publish<TRACE>(st, slot);
        grid_barrier(a.barrier, (++bar) * gridDim.x);
        ran = k + 1;
        bool stop = false;
        if (a.early_exit && a.gammas[k] == a.final_gamma)  // dynamics.py:177
            stop = ring_step_inf(slot) < 1e-12;
        const bool last = stop || ran == a.iters;
        if (ran - k0 == kRing || (last && !TRACE)) {
            fold_ring(a.ring, ran - k0, k0, fo);
            grid_barrier(a.barrier, (++bar) * gridDim.x);
            k0 = ran;
        }
        if (stop) break;
    }
    if (TRACE) {
        // energy terms of the final state (the reference's energy(g, x_new, gamma))
        Stats st{0.0, 0u, 0, {0.0, 0.0, 0.0, 0.0}};
        pass<TS, TG, TI, TRACE>(a, ran, true, st, s_part, s_res);
        publish<TRACE>(st, a.ring + (size_t)(ran - k0) * ring_stride);
        grid_barrier(a.barrier, (++bar) * gridDim.x);
        fold_ring(a.ring, ran - k0 + 1, k0, fo);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) a.status[0] = ran;
}

// x0 (original order, fp64) -> state buffers (new order): x = (TS)x0, yg = (TG)(v*x)
template <typename TS, typename TG>
__global__ void k_prepare(int64_t n, const double* __restrict__ x0, const int32_t* __restrict__ inv,
                          const TS* __restrict__ v, TS* __restrict__ x, TG* __restrict__ yg) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) {
        const int r = inv[i];
        const TS xi = (TS)x0[i];
        x[r] = xi;
        yg[r] = (TG)Arith<TS>::mul(v[r], xi);
    }
}

__global__ void k_precheck_f64(int64_t n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                               const double* __restrict__ x, int* __restrict__ flags) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double xi = x[i];
    if (xi < 0.0) atomicOr(&flags[0], 1);                   // dynamics.py:146
    double s = 0.0;
    for (int32_t p = rowptr[i]; p < rowptr[i + 1]; ++p) s = __dadd_rn(s, x[col[p]]);
    if (!(__dadd_rn(xi, s) > 0.0)) atomicOr(&flags[1], 1);  // dynamics.py:125
}

// final state (new order) -> fp64 output (original order), np.clip(x, 0, 1)
template <typename TS>
__global__ void k_finalize(int64_t n, const TS* __restrict__ x, const int32_t* __restrict__ inv,
                           double* __restrict__ out, int clip) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) {
        double xi = (double)x[inv[i]];
        if (clip) xi = xi < 0.0 ? 0.0 : (xi > 1.0 ? 1.0 : xi);  // dynamics.py:179
        out[i] = xi;
    }
}

static int blocks_for(int64_t n) { return (int)std::max<int64_t>(1, (n + 255) / 256); }

// ------------------------------------------------------------------ plan

// Device plan for one (graph, grid, mode); built on first use and cached
// (graphs are immutable).
struct DevicePlan {
    int grid = 0;
    int32_t* cta_ptr = nullptr;
    int32_t* warp_ptr = nullptr;
    Item* items = nullptr;
    int32_t* smem_words = nullptr;
    size_t smem_bytes = 0;  // dynamic shared memory per CTA
    int resident_off = 0;
    int64_t resident_words = 0;
};

struct PlanCache {
    std::mutex mu;
    std::map<std::pair<int, int>, DevicePlan> plans;  // (grid, exact) -> plan
};

static std::mutex g_cache_mu;
static std::map<const gn_graph*, PlanCache*> g_cache;

void release_plans(const gn_graph* g) {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto it = g_cache.find(g);
    if (it == g_cache.end()) return;
    for (auto& kv : it->second->plans) {
        cudaFree(kv.second.cta_ptr);
        cudaFree(kv.second.warp_ptr);
        cudaFree(kv.second.items);
        cudaFree(kv.second.smem_words);
    }
    delete it->second;
    g_cache.erase(it);
}

// Longest-processing-time-first: CTA items over CTAs, then warp items over
// all warps (a CTA's share of its CTA items preloads each of its warps).
static void build_plan(const gn_graph* g, int G, bool exact, size_t part_bytes, size_t smem_cap,
                       std::vector<int32_t>& cta_ptr, std::vector<int32_t>& warp_ptr, std::vector<Item>& items,
                       std::vector<int32_t>& smem_words) {
    const int B = g->idx16 ? 8 : 4;
    std::vector<int64_t> sp((size_t)g->nslices + 1);
    cudaMemcpy(sp.data(), g->slice_ptr, sizeof(int64_t) * sp.size(), cudaMemcpyDeviceToHost);
    std::vector<int32_t> hp((size_t)g->nhub + 1);
    cudaMemcpy(hp.data(), g->hub_ptr, sizeof(int32_t) * hp.size(), cudaMemcpyDeviceToHost);
    auto nblk = [&](int s) { return (int32_t)((sp[(size_t)s + 1] - sp[(size_t)s]) / (kSlice * B)); };

    // cost unit ~ one 16-byte block per lane; the fixed term stands for the
    // per-item round trips
    const double kFixed = 6.0;
    std::vector<std::vector<Item>> cta_items((size_t)G);
    std::vector<double> cta_load((size_t)G, 0.0);
    std::vector<Item> citems, witems;
    if (!exact) {
        for (int h = 0; h < g->nhub; ++h) citems.push_back(Item{h, hp[(size_t)h + 1] - hp[(size_t)h], -1, kHub});
        for (int s = 0; s < g->nsplit; ++s) citems.push_back(Item{s, nblk(s), -1, kSplit});
        for (int s = g->nsplit; s < g->nslices; ++s) witems.push_back(Item{s, nblk(s), -1, kWhole});
    } else {
        for (int h = 0; h < g->nhub; h += 32) witems.push_back(Item{h, std::min(32, g->nhub - h), -1, kHubSeq});
        for (int s = 0; s < g->nslices; ++s) witems.push_back(Item{s, nblk(s), -1, kWhole});
    }
    auto ccost = [&](const Item& it) {
        return it.kind == kHub ? kFixed + it.len / (32.0 * kWarps) * 4.0 : kFixed + (double)it.len / kWarps;
    };
    auto wcost = [&](const Item& it) {
        if (it.kind == kHubSeq) {
            int mx = 0;
            for (int h = it.id; h < it.id + it.len; ++h) mx = std::max(mx, hp[(size_t)h + 1] - hp[(size_t)h]);
            return kFixed + mx;
        }
        return kFixed + (double)it.len;
    };
    using E = std::pair<double, int>;
    std::stable_sort(citems.begin(), citems.end(), [&](const Item& x, const Item& y) { return ccost(x) > ccost(y); });
    {
        std::priority_queue<E, std::vector<E>, std::greater<E>> pq;
        for (int b = 0; b < G; ++b) pq.push({0.0, b});
        for (const Item& it : citems) {
            E e = pq.top();
            pq.pop();
            cta_items[(size_t)e.second].push_back(it);
            e.first += ccost(it);
            cta_load[(size_t)e.second] = e.first;
            pq.push(e);
        }
    }
    const int W = G * kWarps;
    std::vector<std::vector<Item>> warp_items((size_t)W);
    std::stable_sort(witems.begin(), witems.end(), [&](const Item& x, const Item& y) { return wcost(x) > wcost(y); });
    {
        std::priority_queue<E, std::vector<E>, std::greater<E>> pq;
        for (int w = 0; w < W; ++w) pq.push({cta_load[(size_t)(w / kWarps)], w});
        for (const Item& it : witems) {
            E e = pq.top();
            pq.pop();
            warp_items[(size_t)e.second].push_back(it);
            e.first += wcost(it);
            pq.push(e);
        }
    }
    // each warp's slices in ascending order (locality of the x / yg rows)
    for (auto& v : warp_items)
        std::sort(v.begin(), v.end(), [](const Item& x, const Item& y) { return x.id < y.id; });
    // shared-memory residency of index blocks, per CTA, within smem_cap
    smem_words.assign((size_t)G, 0);
    items.clear();
    cta_ptr.assign((size_t)G + 1, 0);
    warp_ptr.assign((size_t)W + 1, 0);
    const size_t cap_words = smem_cap > part_bytes ? (smem_cap - part_bytes) / 16 : 0;
    for (int b = 0; b < G; ++b) {
        size_t used = 0;
        auto place = [&](Item& it) {
            if (it.kind != kSplit && it.kind != kWhole) return;
            const size_t words = (size_t)it.len * kSlice;
            if (used + words <= cap_words) {
                it.smem = (int32_t)used;
                used += words;
            }
        };
        for (Item& it : cta_items[(size_t)b]) place(it);
        // warp items breadth-first over the CTA's warps so every warp gets some
        for (size_t depth = 0;; ++depth) {
            bool any = false;
            for (int w = 0; w < kWarps; ++w) {
                auto& v = warp_items[(size_t)b * kWarps + w];
                if (depth < v.size()) {
                    any = true;
                    place(v[depth]);
                }
            }
            if (!any) break;
        }
        smem_words[(size_t)b] = (int32_t)used;
    }
    for (int b = 0; b < G; ++b) {
        cta_ptr[(size_t)b] = (int32_t)items.size();
        items.insert(items.end(), cta_items[(size_t)b].begin(), cta_items[(size_t)b].end());
    }
    cta_ptr[(size_t)G] = (int32_t)items.size();
    for (int w = 0; w < W; ++w) {
        warp_ptr[(size_t)w] = (int32_t)items.size();
        items.insert(items.end(), warp_items[(size_t)w].begin(), warp_items[(size_t)w].end());
    }
    warp_ptr[(size_t)W] = (int32_t)items.size();
}

static int get_plan(gn_graph* g, int G, bool exact, size_t part_bytes, size_t smem_cap, const DevicePlan** out) {
    PlanCache* pc;
    {
        std::lock_guard<std::mutex> lk(g_cache_mu);
        auto& slot = g_cache[g];
        if (!slot) slot = new PlanCache();
        pc = slot;
    }
    std::lock_guard<std::mutex> lk(pc->mu);
    auto key = std::make_pair(G, exact ? 1 : 0);
    auto it = pc->plans.find(key);
    if (it != pc->plans.end()) {
        *out = &it->second;
        return GN_OK;
    }
    std::vector<int32_t> cta_ptr, warp_ptr, smem_words;
    std::vector<Item> items;
    build_plan(g, G, exact, part_bytes, smem_cap, cta_ptr, warp_ptr, items, smem_words);
    DevicePlan p;
    p.grid = G;
    GN_CUDA(cudaMalloc(&p.cta_ptr, sizeof(int32_t) * cta_ptr.size()));
    GN_CUDA(cudaMalloc(&p.warp_ptr, sizeof(int32_t) * warp_ptr.size()));
    GN_CUDA(cudaMalloc(&p.items, sizeof(Item) * std::max<size_t>(items.size(), 1)));
    GN_CUDA(cudaMalloc(&p.smem_words, sizeof(int32_t) * smem_words.size()));
    GN_CUDA(cudaMemcpy(p.cta_ptr, cta_ptr.data(), sizeof(int32_t) * cta_ptr.size(), cudaMemcpyHostToDevice));
    GN_CUDA(cudaMemcpy(p.warp_ptr, warp_ptr.data(), sizeof(int32_t) * warp_ptr.size(), cudaMemcpyHostToDevice));
    if (!items.empty())
        GN_CUDA(cudaMemcpy(p.items, items.data(), sizeof(Item) * items.size(), cudaMemcpyHostToDevice));
    GN_CUDA(cudaMemcpy(p.smem_words, smem_words.data(), sizeof(int32_t) * smem_words.size(), cudaMemcpyHostToDevice));
    int32_t mx = 0;
    for (int32_t wds : smem_words) {
        mx = std::max(mx, wds);
        p.resident_words += wds;
    }
    p.resident_off = (int)((part_bytes + 15) / 16 * 16);
    p.smem_bytes = (size_t)p.resident_off + (size_t)mx * 16;
    auto res = pc->plans.emplace(key, p);
    *out = &res.first->second;
    return GN_OK;
}

// stream-ordered scratch owned by one call
struct Workspace {
    void* p[24] = {};
    int np = 0;
    cudaStream_t s = nullptr;
    template <typename P>
    cudaError_t alloc(P** out, size_t bytes) {
        cudaError_t e = cudaMallocAsync((void**)out, std::max<size_t>(bytes, 16), s);
        if (e == cudaSuccess) p[np++] = (void*)*out;
        return e;
    }
    ~Workspace() {
        for (int i = 0; i < np; ++i) cudaFreeAsync(p[i], s);
    }
};

template <typename TS, typename TG, typename TI>
static int run_typed(gn_graph* g, const void* x0, const double* gammas, int iters, double final_gamma,
                     uint32_t flags, void* x_out, double* step_inf, int64_t* fallbacks, double* mass,
                     double* energy, double* pre_energy, double* x_hist, int* iters_run, int* fail_iter,
                     gn_run_stats* stats) {
    const bool trace = (flags & GN_TRACE) != 0;
    const bool dev_io = (flags & GN_DEVICE_IO) != 0;
    const bool exact = (flags & GN_EXACT) != 0;
    const int64_t n = g->n;
    const size_t nb = (size_t)std::max<int64_t>(n, 1);
    const int64_t launches0 = gn_launch_count();
    CallCtx ctx;
    int rc = ctx.open(g->device);
    if (rc) return rc;
    cudaStream_t s = ctx.s;
    int64_t h2d = 0, d2h = 0;

    cudaEvent_t ev[4];
    for (auto& e : ev) GN_CUDA(cudaEventCreate(&e));
    struct EvGuard {
        cudaEvent_t* e;
        ~EvGuard() { for (int i = 0; i < 4; ++i) cudaEventDestroy(e[i]); }
    } evg{ev};
    GN_CUDA(cudaEventRecord(ev[0], s));

    // ---- launch geometry and plan
    void* kern = trace ? (void*)k_gn_loop<TS, TG, TI, true> : (void*)k_gn_loop<TS, TG, TI, false>;
    int max_optin = 0;
    GN_CUDA(cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, g->device));
    const size_t part_bytes = (size_t)kSlots * kWarps * kSlice * sizeof(TS);
    const size_t static_bytes = 2048;  // publish scratch
    const size_t smem_cap = (size_t)max_optin - static_bytes;
    GN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_cap));
    int maxb = 1;
    if ((rc = coresident_blocks(kern, kThreads, smem_cap, g->device, &maxb))) return rc;
    if (maxb < 1) return fail(GN_ERR_CUDA, "loop kernel cannot be resident");
    const int64_t work = g->sell_elems + 4 * n + (g->nhub ? 32768 : 0);
    int grid = (int)std::min<int64_t>(maxb, std::max<int64_t>(1, (work + 16383) / 16384));
    if (g->grid_override > 0) grid = std::min(maxb, g->grid_override);
    const DevicePlan* plan = nullptr;
    if ((rc = get_plan(g, grid, exact, part_bytes, smem_cap, &plan))) return rc;

    Workspace ws;
    ws.s = s;
    TS *xa, *xb;
    TG *ya, *yb;
    double *xin, *dots, *ring, *gam, *out64 = nullptr, *hist = nullptr, *dsi, *dfb;
    int *dbad, *status, *chk;
    unsigned int* barrier;
    GN_CUDA(ws.alloc(&xa, sizeof(TS) * nb));
    GN_CUDA(ws.alloc(&xb, sizeof(TS) * nb));
    GN_CUDA(ws.alloc(&ya, sizeof(TG) * nb));
    GN_CUDA(ws.alloc(&yb, sizeof(TG) * nb));
    GN_CUDA(ws.alloc(&dsi, 8 * (size_t)iters));
    GN_CUDA(ws.alloc(&dfb, 8 * (size_t)iters));
    GN_CUDA(ws.alloc(&dbad, 4 * (size_t)iters));
    GN_CUDA(ws.alloc(&dots, 8 * 4 * (size_t)(iters + 1)));
    GN_CUDA(ws.alloc(&ring, 8 * (size_t)kRingW * (size_t)std::min(kRing, iters + 1) * grid));
    GN_CUDA(ws.alloc(&status, 4 * sizeof(int)));
    GN_CUDA(ws.alloc(&barrier, sizeof(unsigned int)));
    GN_CUDA(ws.alloc(&chk, 2 * sizeof(int)));
    GN_CUDA(ws.alloc(&gam, 8 * (size_t)iters));
    GN_CUDA(cudaMemsetAsync(dsi, 0, 8 * (size_t)iters, s));
    GN_CUDA(cudaMemsetAsync(dfb, 0, 8 * (size_t)iters, s));
    GN_CUDA(cudaMemsetAsync(dbad, 0, 4 * (size_t)iters, s));
    GN_CUDA(cudaMemsetAsync(dots, 0, 8 * 4 * (size_t)(iters + 1), s));
    GN_CUDA(cudaMemsetAsync(status, 0, 4 * sizeof(int), s));
    GN_CUDA(cudaMemsetAsync(barrier, 0, sizeof(unsigned int), s));
    GN_CUDA(cudaMemsetAsync(chk, 0, 2 * sizeof(int), s));
    if (x_hist) GN_CUDA(ws.alloc(&hist, 8 * nb * (size_t)iters));
    GN_CUDA(cudaMemcpyAsync(gam, gammas, 8 * (size_t)iters, cudaMemcpyHostToDevice, s));
    h2d += 8 * iters;

    // ---- x0 in, checks (dynamics.py:145-149)
    if (dev_io) {
        xin = (double*)x0;
    } else {
        GN_CUDA(ws.alloc(&xin, 8 * nb));
        if (n > 0) GN_CUDA(cudaMemcpyAsync(xin, x0, 8 * (size_t)n, cudaMemcpyHostToDevice, s));
        h2d += 8 * n;
    }
    const bool check = !(flags & GN_NO_CHECK);
    if (n > 0) {
        if (check) {
            k_precheck_f64<<<blocks_for(n), 256, 0, s>>>(n, g->rowptr, g->col, xin, chk);
            GN_LAUNCHED();
        }
        k_prepare<TS, TG><<<blocks_for(n), 256, 0, s>>>(n, xin, g->inv, (const TS*)g->v, xa, ya);
        GN_LAUNCHED();
    }
    if (check && n > 0) {
        int hchk[2] = {0, 0};
        GN_CUDA(cudaMemcpyAsync(hchk, chk, sizeof(hchk), cudaMemcpyDeviceToHost, s));
        GN_CUDA(cudaStreamSynchronize(s));
        if (hchk[0]) return fail(GN_ERR_NEGATIVE, "state entries must be nonnegative");
        if (hchk[1]) return fail(GN_ERR_NOT_NORMALIZABLE, "initial state has a zero closed neighborhood sum");
    }

    // ---- the loop
    LoopArgs<TS, TG> a;
    memset(&a, 0, sizeof(a));
    a.n = n;
    a.nhub = g->nhub;
    a.hub_ptr = g->hub_ptr;
    a.hub_col = g->hub_col;
    a.slice_ptr = g->slice_ptr;
    a.row_deg = g->row_deg;
    a.sell = g->sell;
    a.v = (const TS*)g->v;
    a.w = (const TS*)g->w;
    a.x[0] = xa;
    a.x[1] = xb;
    a.yg[0] = ya;
    a.yg[1] = yb;
    a.cta_ptr = plan->cta_ptr;
    a.warp_ptr = plan->warp_ptr;
    a.items = plan->items;
    a.smem_words = plan->smem_words;
    a.smem_resident_off = plan->resident_off;
    a.gammas = gam;
    a.iters = iters;
    a.final_gamma = final_gamma;
    a.early_exit = (flags & GN_EARLY_EXIT) ? 1 : 0;
    a.step_inf = dsi;
    a.fb = dfb;
    a.bad = dbad;
    a.status = status;
    a.dots = dots;
    a.ring = ring;
    a.barrier = barrier;
    a.x_hist = hist;
    a.perm = g->perm;
    void* args[] = {&a};
    GN_CUDA(cudaEventRecord(ev[1], s));
    GN_CUDA(cudaLaunchCooperativeKernel(kern, dim3(grid), dim3(kThreads), args, plan->smem_bytes, s));
    GN_LAUNCHED();
    GN_CUDA(cudaEventRecord(ev[2], s));

    // ---- results back
    int hstatus[4];
    GN_CUDA(cudaMemcpyAsync(hstatus, status, sizeof(hstatus), cudaMemcpyDeviceToHost, s));
    std::vector<double> hsi((size_t)iters), hfb((size_t)iters);
    std::vector<int> hbad((size_t)iters);
    std::vector<double> hdots(4 * (size_t)(iters + 1));
    GN_CUDA(cudaMemcpyAsync(hsi.data(), dsi, 8 * (size_t)iters, cudaMemcpyDeviceToHost, s));
    GN_CUDA(cudaMemcpyAsync(hfb.data(), dfb, 8 * (size_t)iters, cudaMemcpyDeviceToHost, s));
    GN_CUDA(cudaMemcpyAsync(hbad.data(), dbad, 4 * (size_t)iters, cudaMemcpyDeviceToHost, s));
    GN_CUDA(cudaMemcpyAsync(hdots.data(), dots, 8 * 4 * (size_t)(iters + 1), cudaMemcpyDeviceToHost, s));
    d2h += 8 * 2 * iters + 4 * iters + 8 * 4 * (iters + 1) + 16;
    GN_CUDA(cudaStreamSynchronize(s));
    const int ran = hstatus[0];
    const TS* xfinal = (ran & 1) ? xb : xa;
    const int clip = (flags & GN_NO_CLIP) ? 0 : 1;
    if (x_out && n > 0) {
        if (dev_io) {
            k_finalize<TS><<<blocks_for(n), 256, 0, s>>>(n, xfinal, g->inv, (double*)x_out, clip);
            GN_LAUNCHED();
        } else {
            GN_CUDA(ws.alloc(&out64, 8 * nb));
            k_finalize<TS><<<blocks_for(n), 256, 0, s>>>(n, xfinal, g->inv, out64, clip);
            GN_LAUNCHED();
            GN_CUDA(cudaMemcpyAsync(x_out, out64, 8 * (size_t)n, cudaMemcpyDeviceToHost, s));
            d2h += 8 * n;
        }
    }
    if (x_hist && n > 0 && ran > 0) {
        GN_CUDA(cudaMemcpyAsync(x_hist, hist, 8 * (size_t)ran * (size_t)n, cudaMemcpyDeviceToHost, s));
        d2h += 8 * (int64_t)ran * n;
    }
    GN_CUDA(cudaEventRecord(ev[3], s));
    GN_CUDA(cudaStreamSynchronize(s));

    int bad = -1;
    for (int k = 0; k < ran; ++k)
        if (hbad[(size_t)k]) { bad = k; break; }
    for (int k = 0; k < ran; ++k) {
        if (step_inf) step_inf[k] = hsi[(size_t)k];
        if (fallbacks) fallbacks[k] = (int64_t)hfb[(size_t)k];
        const double* d0 = &hdots[(size_t)k * 4];
        const double* d1 = &hdots[(size_t)(k + 1) * 4];
        if (mass) mass[k] = d0[3];
        if (trace) {
            // dynamics.py:219 from the fused dot products of x_k and x_{k+1}
            if (pre_energy) pre_energy[k] = 0.5 * (d0[0] + gammas[k] * d0[1]) - d0[2];
            if (energy) energy[k] = 0.5 * (d1[0] + gammas[k] * d1[1]) - d1[2];
        }
    }
    if (iters_run) *iters_run = ran;
    if (fail_iter) *fail_iter = bad;
    if (stats) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev[1], ev[2]);
        stats->loop_ms = ms;
        cudaEventElapsedTime(&ms, ev[0], ev[3]);
        stats->total_ms = ms;
        stats->launches = gn_launch_count() - launches0;
        stats->grid_blocks = grid;
        stats->block_threads = kThreads;
        stats->h2d_bytes = h2d;
        stats->d2h_bytes = d2h;
    }
    if (bad >= 0 && !(flags & GN_NONFINITE_OK)) {
        char buf[64];
        snprintf(buf, sizeof(buf), "non-finite state at iteration %d", bad);
        if (iters_run) *iters_run = bad + 1;
        return fail(GN_ERR_NONFINITE, buf);
    }
    return GN_OK;
}

template <typename TS, typename TG>
static int run_idx(gn_graph* g, const void* x0, const double* gammas, int iters, double final_gamma, uint32_t flags,
                   void* x_out, double* step_inf, int64_t* fallbacks, double* mass, double* energy,
                   double* pre_energy, double* x_hist, int* iters_run, int* fail_iter, gn_run_stats* stats) {
    if (g->idx16)
        return run_typed<TS, TG, uint16_t>(g, x0, gammas, iters, final_gamma, flags, x_out, step_inf, fallbacks,
                                           mass, energy, pre_energy, x_hist, iters_run, fail_iter, stats);
    return run_typed<TS, TG, int32_t>(g, x0, gammas, iters, final_gamma, flags, x_out, step_inf, fallbacks, mass,
                                      energy, pre_energy, x_hist, iters_run, fail_iter, stats);
}

}  // namespace gn

using namespace gn;

extern "C" {

int gn_run(gn_graph* g, const void* x0, const double* gammas, int iters, double final_gamma, uint32_t flags,
           void* x_out, double* step_inf, int64_t* fallbacks, double* mass, double* energy, double* pre_energy,
           double* x_hist, int* iters_run, int* fail_iter, gn_run_stats* stats) {
    if (!g) return fail(GN_ERR_ARG, "null graph");
    if (iters < 1) return fail(GN_ERR_ARG, "iterations must be positive");
    if (!gammas || (g->n > 0 && !x0)) return fail(GN_ERR_ARG, "null input array");
    switch (g->dtype) {
        case GN_F64:
            return run_idx<double, double>(g, x0, gammas, iters, final_gamma, flags, x_out, step_inf, fallbacks,
                                           mass, energy, pre_energy, x_hist, iters_run, fail_iter, stats);
        case GN_F32:
            return run_idx<double, float>(g, x0, gammas, iters, final_gamma, flags, x_out, step_inf, fallbacks,
                                          mass, energy, pre_energy, x_hist, iters_run, fail_iter, stats);
        default:
            return run_idx<float, float>(g, x0, gammas, iters, final_gamma, flags, x_out, step_inf, fallbacks, mass,
                                         energy, pre_energy, x_hist, iters_run, fail_iter, stats);
    }
}

int gn_step(gn_graph* g, const double* x, double gamma, uint32_t flags, double* out, int64_t* nfb) {
    double si = 0.0;
    int64_t fb = 0;
    int ran = 0, fi = -1;
    uint32_t f = (flags & GN_EXACT) | GN_NO_CHECK | GN_NO_CLIP | GN_NONFINITE_OK;
    int rc = gn_run(g, x, &gamma, 1, gamma, f, out, &si, &fb, nullptr, nullptr, nullptr, nullptr, &ran, &fi,
                    nullptr);
    if (nfb) *nfb = fb;
    return rc;
}

}  // extern "C"
