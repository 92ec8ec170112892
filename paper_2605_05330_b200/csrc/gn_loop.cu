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
// pre-step state).  Warp stats go to a ring (plain stores, no atomics, no
// CTA barrier) that all blocks fold cooperatively every kRing iterations.
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
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <numeric>
#include <queue>
#include <vector>

#include "gn_internal.cuh"
#include "gn_plan.h"

#ifndef GN_HUB_ROUND
#define GN_HUB_ROUND 8  // hub-piece gathers per lane per round (16 spills)
#endif
#ifndef GN_DBG_GATHER
#define GN_DBG_GATHER 0  // timing experiments only (results are wrong when set)
#endif

namespace gn {

constexpr int kRing = 128;  // iterations of warp stats kept before a fold
constexpr int kRingW = 8;   // per warp: 4 dot terms, max|dx|, fallbacks, non-finite, pad

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
    const int32_t* __restrict__ phase_base;  // [G+1] into phases
    const int32_t* __restrict__ phase_warp;  // [P*(kWarps+1)] into items
    const int32_t* __restrict__ phase_comb;  // [P+1] into combs
    const Item* __restrict__ items;
    const Combine* __restrict__ combs;
    const int32_t* __restrict__ smem_words;  // [G] resident 16-byte words per CTA
    int hub_slot_off;                        // byte offsets in dynamic shared memory
    int hot_off;
    int resident_off;
    int item_cache_off;                      // > 0: the CTA's items and lane degrees copied to shared memory here
    int hot;                                 // new ids [0, hot) mirrored in shared memory
    const double* __restrict__ gammas;
    int iters;
    double final_gamma;
    int early_exit;
    double* step_inf;  // [iters]   max over blocks of max|x'-x|
    double* fb;        // [iters]   fallback count (exact in fp64)
    int* bad;          // [iters]   1 if a non-finite state appeared
    int* status;       // [0] iterations run
    double* dots;      // [(iters+1)][4]: y.y, y.s, w.x (pre), w.x' (post)
    double* ring;      // [kRing][grid * kWarps][kRingW]
    unsigned int* barrier;
    double* x_hist;    // optional [iters][n], original order
    const int32_t* __restrict__ perm;
    long long* prof;   // optional timestamps (GN_PROF_ITER): [G][kWarps+4]
    int prof_iter;
    const int* chk;    // [2] x0 check flags (k_precheck_f64): set -> the run does not start
};

struct Stats {
    double mx;
    unsigned int fbc;
    int bad;
    double acc[4];
};

template <typename T>
__device__ __forceinline__ T tabs(T v) { return v < T(0) ? -v : v; }

__device__ __forceinline__ long long gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

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
        // one PRMT (low half) or SHF (high half); the address is then one IMAD.WIDE.U32
        return (int)((t & 1) ? (w >> 16) : __byte_perm(w, 0u, 0x4410));
    }
};
template <>
struct LaneVec<int32_t> {
    static constexpr int B = 4;
    __device__ static __forceinline__ int get(const uint4& v, int t) {
        return (int)(t == 0 ? v.x : t == 1 ? v.y : t == 2 ? v.z : v.w);
    }
};

template <typename TS, typename TG, typename TI>
__device__ __forceinline__ const uint4* slice_base(const LoopArgs<TS, TG>& a, const Item& it, const uint4* s_res,
                                                   int lane) {
    if (it.smem >= 0) return s_res + it.smem - (ptrdiff_t)it.beg * kSlice + lane;
    return reinterpret_cast<const uint4*>((const TI*)a.sell + __ldg(a.slice_ptr + it.id)) + lane;
}

// Where gathered values come from: global memory, or -- for the hottest
// vertices (new ids < hot) -- their shared-memory mirror.
template <typename TG, bool HOT>
struct GSrc {
    const TG* __restrict__ yg;
    const TG* s_hot;
    int hot;
    __device__ __forceinline__ TG operator[](int j) const {
        if (HOT) return j < hot ? s_hot[j] : yg[j];
        return yg[j];
    }
};

// ---- software-pipelined slice items -----------------------------------
// A warp walks its slice items (short slices and pieces of long slices) with
// a two-deep pipeline: while item i's gathers are in flight, item i+1's
// degree, row state and first index vectors are already loading, and item
// i+2's descriptor too.  Each item costs about one memory round trip instead
// of four dependent ones.
#ifndef GN_GD_F32
#define GN_GD_F32 16  // fp32 gathers: 32 in flight spilled (C2 fp32: 23.1 -> 19.4 us/iteration at 16; C5 unchanged)
#endif
#ifndef GN_GD_F64
#define GN_GD_F64 16
#endif
template <typename TG>
struct GatherDepth {  // gathers in flight per lane (register budget: 64K / (kThreads * kCtasPerSm))
    static constexpr int value = (sizeof(TG) == 4 ? GN_GD_F32 : GN_GD_F64) / kCtasPerSm;
};

template <typename TS, typename TI, typename TG>
struct SlicePre {
    static constexpr int B = LaneVec<TI>::B;
    // int32-id layouts pad with the zero-valued vertex n (gn_graph.cu): no degree masks
    static constexpr bool kSent = sizeof(TI) == 4;
    // index vectors per batch, at most 4 (two batches of them are live at
    // once); int32-id layouts walk an item pair interleaved (slice_consume2),
    // half a batch per item
    static constexpr int NBF = GatherDepth<TG>::value / B > 4 ? 4 : (GatherDepth<TG>::value / B > 0 ? GatherDepth<TG>::value / B : 1);
    static constexpr int NB = kSent && NBF > 1 ? NBF / 2 : NBF;
    const uint4* base;  // block `beg` of the item, this lane
    int beg, nb, d, row;
    bool whole, valid;
    RowIn<TS> in;
    uint4 v[NB];
};

// Where a CTA reads its item descriptors and slice-row degrees: a shared
// memory copy made once per run (when they fit) -- every iteration then
// starts its items without a global round trip -- or global memory.
struct ItemSrc {
    const Item* it;       // items, indexed from `base`
    const int32_t* deg;   // [item - base][32] lane degrees of slice items, or nullptr (global row_deg)
    int base;
    __device__ __forceinline__ Item at(int i) const { return it[i - base]; }
};

template <typename TS, typename TG, typename TI>
__device__ __forceinline__ void slice_prefetch(const LoopArgs<TS, TG>& a, const Item& it, const ItemSrc& src, int i,
                                               const uint4* s_res, int lane, int cur, SlicePre<TS, TI, TG>& p) {
    using SP = SlicePre<TS, TI, TG>;
    p.whole = it.kind == kWhole;
    p.beg = it.beg;
    p.nb = it.end - it.beg;
    const int64_t r = (int64_t)a.nhub + (int64_t)it.id * kSlice + lane;
    p.valid = r < a.n;
    p.row = (int)r;
    // Item.pad0/pad1: 16-byte-word offset of block `beg` in the global index array
    const int64_t goff = ((int64_t)(uint32_t)it.pad1 << 32) | (uint32_t)it.pad0;
    p.base = (it.smem >= 0 ? s_res + it.smem : reinterpret_cast<const uint4*>(a.sell) + goff) + lane;
    p.d = SlicePre<TS, TI, TG>::kSent ? 0
                 : (src.deg ? src.deg[(i - src.base) * kSlice + lane]
                            : (p.valid ? __ldg(a.row_deg + (size_t)it.id * kSlice + lane) : 0));
    if (p.whole && p.valid) p.in = row_in(a, p.row, cur);
#pragma unroll
    for (int u = 0; u < SP::NB; ++u)
        if (u < p.nb) p.v[u] = p.base[(size_t)u * kSlice];
}

// The storage of a warp's item pair.  The first pair of an iteration is
// prefetched while the grid barrier before it is still pending: it reads
// only static data (indices, degrees, v, w) and rows this CTA itself wrote.
template <typename TS, typename TI, typename TG>
struct ItemPair {
    SlicePre<TS, TI, TG> p0, p1;
    int n;  // > 0: the first pair of phase ph0 is already prefetched (n items)
};

template <typename TS, typename TG, typename TI>
__device__ __forceinline__ void prefetch_first(const LoopArgs<TS, TG>& a, int k, const ItemSrc& src,
                                               const uint4* s_res, ItemPair<TS, TI, TG>& pr) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    pr.n = 0;
    const int ph0 = __ldg(a.phase_base + blockIdx.x);
    if (ph0 >= __ldg(a.phase_base + blockIdx.x + 1)) return;
    const int i0 = __ldg(a.phase_warp + ph0 * (kWarps + 1) + warp);
    const int i1 = __ldg(a.phase_warp + ph0 * (kWarps + 1) + warp + 1);
    if (i0 >= i1) return;
    const Item it0 = src.at(i0);
    if (it0.kind > kPiece) return;
    slice_prefetch<TS, TG, TI>(a, it0, src, i0, s_res, lane, k & 1, pr.p0);
    pr.n = 1;
    if (i0 + 1 < i1) {
        const Item it1 = src.at(i0 + 1);
        if (it1.kind <= kPiece) {
            slice_prefetch<TS, TG, TI>(a, it1, src, i0 + 1, s_res, lane, k & 1, pr.p1);
            pr.n = 2;
        }
    }
}

// Sequential sum of one lane's row over the item's blocks; p.v holds the
// first batch of index vectors.
template <typename TS, typename TG, typename TI, bool HOT>
__device__ __forceinline__ TS slice_consume(SlicePre<TS, TI, TG>& p, const GSrc<TG, HOT>& yg) {
    using A = Arith<TS>;
    using V = LaneVec<TI>;
    using SP = SlicePre<TS, TI, TG>;
    constexpr int B = SP::B, NB = SP::NB;
    TS s = TS(0);
    const int d = p.d;
    // local blocks that hold any of this row's neighbours (all of the item's
    // blocks when padding names the zero vertex: the warp stays converged)
    const int be = SP::kSent ? p.nb : min(p.nb, max(0, (d - p.beg * B + B - 1) / B));
    for (int b = 0; b < be; b += NB) {
        uint4 vn[NB];
#pragma unroll
        for (int u = 0; u < NB; ++u)
            if (b + NB + u < be) vn[u] = p.base[(size_t)(b + NB + u) * kSlice];
#if GN_DBG_GATHER == 1  // timing experiment: gathers hit a few cached lines
#pragma unroll
        for (int u = 0; u < NB; ++u) p.v[u] = make_uint4(threadIdx.x & 31, 32 + (threadIdx.x & 31), 64, 96);
#endif
        TG y[NB * B];
        const int pos0 = (p.beg + b) * B;
        if (b + NB <= be && (SP::kSent || pos0 + NB * B <= d)) {
#pragma unroll
            for (int u = 0; u < NB; ++u)
#pragma unroll
                for (int t = 0; t < B; ++t) {
#if GN_DBG_GATHER == 3  // timing experiment: no gathers
                    y[u * B + t] = (TG)V::get(p.v[u], t);
#else
                    y[u * B + t] = yg[V::get(p.v[u], t)];
#endif
                }
        } else {
#pragma unroll
            for (int u = 0; u < NB; ++u)
#pragma unroll
                for (int t = 0; t < B; ++t)
                    y[u * B + t] = (b + u < be && (SP::kSent || pos0 + u * B + t < d)) ? yg[V::get(p.v[u], t)] : TG(0);
        }
#pragma unroll
        for (int q = 0; q < NB * B; ++q) s = A::add(s, (TS)y[q]);
#pragma unroll
        for (int u = 0; u < NB; ++u) p.v[u] = vn[u];
    }
    return s;
}

// Both items of a pair at once (int32-id layouts, no degree masks): each
// batch issues the gathers of the two items before adding either, so a pair
// of short slices costs one memory round trip instead of two.  Each item's
// sum stays sequential in position order.
template <typename TS, typename TG, typename TI, bool HOT>
__device__ __forceinline__ void slice_consume2(SlicePre<TS, TI, TG>& p0, SlicePre<TS, TI, TG>& p1,
                                               const GSrc<TG, HOT>& yg, TS& s0, TS& s1) {
    using A = Arith<TS>;
    using V = LaneVec<TI>;
    using SP = SlicePre<TS, TI, TG>;
    constexpr int B = SP::B, NB = SP::NB;
    s0 = TS(0);
    s1 = TS(0);
    const int be0 = p0.nb, be1 = p1.nb, be = max(be0, be1);
    for (int b = 0; b < be; b += NB) {
        uint4 vn0[NB], vn1[NB];
#pragma unroll
        for (int u = 0; u < NB; ++u) {
            if (b + NB + u < be0) vn0[u] = p0.base[(size_t)(b + NB + u) * kSlice];
            if (b + NB + u < be1) vn1[u] = p1.base[(size_t)(b + NB + u) * kSlice];
        }
        TG y0[NB * B], y1[NB * B];
#pragma unroll
        for (int u = 0; u < NB; ++u)
#pragma unroll
            for (int t = 0; t < B; ++t) {
                y0[u * B + t] = b + u < be0 ? yg[V::get(p0.v[u], t)] : TG(0);
                y1[u * B + t] = b + u < be1 ? yg[V::get(p1.v[u], t)] : TG(0);
            }
#pragma unroll
        for (int q = 0; q < NB * B; ++q) s0 = A::add(s0, (TS)y0[q]);
#pragma unroll
        for (int q = 0; q < NB * B; ++q) s1 = A::add(s1, (TS)y1[q]);
#pragma unroll
        for (int u = 0; u < NB; ++u) {
            p0.v[u] = vn0[u];
            p1.v[u] = vn1[u];
        }
    }
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

// One pass over this CTA's items, phase by phase (gn_plan.h).
template <typename TS, typename TG, typename TI, bool TRACE, bool HOT>
__device__ void pass(const LoopArgs<TS, TG>& a, int k, bool tail, Stats& st, TS* s_slot, TS* s_hslot,
                     const uint4* s_res, TG* s_hot, const ItemSrc& src, ItemPair<TS, TI, TG>& pr) {
    using A = Arith<TS>;
    const int cur = k & 1;
    if (HOT) {
        // mirror the hottest vertices' published values (written by all CTAs
        // before the last grid barrier) into shared memory
        const uint4* src = reinterpret_cast<const uint4*>(a.yg[cur]);
        uint4* dst = reinterpret_cast<uint4*>(s_hot);
        const int words = (int)((size_t)a.hot * sizeof(TG) / 16);
        for (int t = threadIdx.x; t < words; t += blockDim.x) dst[t] = __ldcg(src + t);
        __syncthreads();
    }
    const GSrc<TG, HOT> yg{a.yg[cur], s_hot, a.hot};
    const TS g = tail ? TS(0) : (TS)a.gammas[k];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int ph0 = __ldg(a.phase_base + blockIdx.x), ph1 = __ldg(a.phase_base + blockIdx.x + 1);
    for (int ph = ph0; ph < ph1; ++ph) {
        const int i0 = __ldg(a.phase_warp + ph * (kWarps + 1) + warp);
        const int i1 = __ldg(a.phase_warp + ph * (kWarps + 1) + warp + 1);
        if (a.prof && k == a.prof_iter && lane == 0 && ph == ph0) a.prof[blockIdx.x * (kWarps + 4) + 4 + warp] = gtimer();
        // slice items first (the plan sorts each warp's list by kind), two at
        // a time: both items' loads are issued before either is consumed
        int i = i0;
        bool ready = ph == ph0 && pr.n > 0;  // the first pair came prefetched
        SlicePre<TS, TI, TG>& p0 = pr.p0;
        SlicePre<TS, TI, TG>& p1 = pr.p1;
        while (i < i1) {
            const Item it0 = src.at(i);
            if (it0.kind > kPiece) break;
            const bool two = i + 1 < i1 && src.at(i + 1).kind <= kPiece;
            const Item it1 = two ? src.at(i + 1) : it0;
            if (!ready) {
                slice_prefetch<TS, TG, TI>(a, it0, src, i, s_res, lane, cur, p0);
                if (two) slice_prefetch<TS, TG, TI>(a, it1, src, i + 1, s_res, lane, cur, p1);
            }
            ready = false;
            if (SlicePre<TS, TI, TG>::kSent && two) {
                TS s0, s1;
                slice_consume2<TS, TG, TI, HOT>(p0, p1, yg, s0, s1);
                if (!p0.whole) s_slot[it0.slot * kSlice + lane] = s0;
                else if (p0.valid) update_row<TS, TG, TRACE>(a, p0.row, s0, p0.in, cur, g, k, tail, st);
                if (!p1.whole) s_slot[it1.slot * kSlice + lane] = s1;
                else if (p1.valid) update_row<TS, TG, TRACE>(a, p1.row, s1, p1.in, cur, g, k, tail, st);
            } else {
                const TS s0 = slice_consume<TS, TG, TI, HOT>(p0, yg);
                if (!p0.whole) s_slot[it0.slot * kSlice + lane] = s0;
                else if (p0.valid) update_row<TS, TG, TRACE>(a, p0.row, s0, p0.in, cur, g, k, tail, st);
                if (two) {
                    const TS s1 = slice_consume<TS, TG, TI, HOT>(p1, yg);
                    if (!p1.whole) s_slot[it1.slot * kSlice + lane] = s1;
                    else if (p1.valid) update_row<TS, TG, TRACE>(a, p1.row, s1, p1.in, cur, g, k, tail, st);
                }
            }
            i += two ? 2 : 1;
        }
        for (; i < i1; ++i) {
            const Item it = src.at(i);
            if (it.kind == kWhole || it.kind == kPiece) {
                // not reached: slice items precede hub items in every warp list
            } else if (it.kind == kHubPiece) {
                // lanes stride the piece's elements, 16 per lane per round with
                // the next round's indices loading under this round's gathers
                // (a hub piece is a chain of rounds on its CTA's critical path);
                // fixed warp tree
                constexpr int R = GN_HUB_ROUND;
                const int base = __ldg(a.hub_ptr + it.id);
                TS s = TS(0);
                int p = base + it.beg + lane;
                const int e = base + it.end;
                int jn[R];
#pragma unroll
                for (int u = 0; u < R; ++u) jn[u] = p + u * 32 < e ? __ldg(a.hub_col + p + u * 32) : 0;
                for (; p + (R - 1) * 32 < e; p += R * 32) {
                    int j[R];
#pragma unroll
                    for (int u = 0; u < R; ++u) j[u] = jn[u];
#pragma unroll
                    for (int u = 0; u < R; ++u) {
                        const int q = p + (R + u) * 32;
                        jn[u] = q < e ? __ldg(a.hub_col + q) : 0;
                    }
                    TG y[R];
#pragma unroll
                    for (int u = 0; u < R; ++u) y[u] = yg[j[u]];
#pragma unroll
                    for (int u = 0; u < R; ++u) s = A::add(s, (TS)y[u]);
                }
#pragma unroll
                for (int u = 0; u < R; ++u)  // the last partial round: its indices are in jn
                    if (p + u * 32 < e) s = A::add(s, (TS)yg[jn[u]]);
                s = warp_sum(s);
                if (lane == 0) s_hslot[it.slot] = s;
            } else {  // kHubSeq (EXACT): one thread per hub row, sequential
                if (lane < it.end - it.beg) {
                    const int h = it.id + lane;
                    const RowIn<TS> in = row_in(a, h, cur);
                    TS s = TS(0);
                    for (int p = __ldg(a.hub_ptr + h); p < __ldg(a.hub_ptr + h + 1); ++p)
                        s = A::add(s, (TS)yg[__ldg(a.hub_col + p)]);
                    update_row<TS, TG, TRACE>(a, h, s, in, cur, g, k, tail, st);
                }
            }
        }
        if (a.prof && k == a.prof_iter && ph == ph0) {
            __syncwarp();
            if (lane == 0) a.prof[blockIdx.x * (kWarps + 4) + 4 + warp] = gtimer() - a.prof[blockIdx.x * (kWarps + 4) + 4 + warp];
        }
        const int c0 = __ldg(a.phase_comb + ph), c1 = __ldg(a.phase_comb + ph + 1);
        if (c1 > c0) {
            // the state of the warp's first combine row loads while the CTA
            // waits for its slowest warp (it does not depend on the pieces)
            Combine cb0{0, 0, 0, 0};
            RowIn<TS> in0{TS(0), TS(0), 0.0};
            if (c0 + warp < c1) {
                cb0 = a.combs[c0 + warp];
                const int r0 = cb0.kind == 0 ? a.nhub + cb0.id * kSlice + lane : cb0.id;
                if (r0 < a.n && (cb0.kind == 0 || lane == 0)) in0 = row_in(a, r0, cur);
            }
            __syncthreads();
            for (int c = c0 + warp; c < c1; c += kWarps) {
                const bool first = c == c0 + warp;
                const Combine cb = first ? cb0 : a.combs[c];
                if (cb.kind == 0) {
                    const int r = a.nhub + cb.id * kSlice + lane;
                    const RowIn<TS> in = first ? in0 : row_in(a, r, cur);
                    TS tot = TS(0);
                    for (int q = 0; q < cb.nslot; ++q) tot = A::add(tot, s_slot[(cb.slot + q) * kSlice + lane]);
                    update_row<TS, TG, TRACE>(a, r, tot, in, cur, g, k, tail, st);
                } else if (lane == 0) {
                    const RowIn<TS> in = first ? in0 : row_in(a, cb.id, cur);
                    TS tot = TS(0);
                    for (int q = 0; q < cb.nslot; ++q) tot = A::add(tot, s_hslot[cb.slot + q]);
                    update_row<TS, TG, TRACE>(a, cb.id, tot, in, cur, g, k, tail, st);
                }
            }
            if (ph + 1 < ph1) __syncthreads();
        }
    }
}

// Warp-level fold of the per-thread stats; lane 0 stores the warp's partials
// (plain stores, no atomics, no CTA barrier) in this iteration's ring slot.
template <bool TRACE>
__device__ void publish(const Stats& st0, double* __restrict__ ring_slot) {
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
        double* dst = ring_slot + ((size_t)blockIdx.x * kWarps + warp) * kRingW;
#pragma unroll
        for (int c = 0; c < 4; ++c) dst[c] = st.acc[c];
        dst[4] = st.mx;
        dst[5] = (double)st.fbc;
        dst[6] = st.bad ? 1.0 : 0.0;
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
// warp per (slot, quantity), partial order fixed.
__device__ void fold_ring(const double* ring, int count, int k0, const FoldOut& o) {
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * kWarps + (threadIdx.x >> 5), nw = gridDim.x * kWarps;
    const int G = gridDim.x * kWarps;  // partials per iteration (one per warp)
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
        for (int b = threadIdx.x; b < (int)gridDim.x * kWarps; b += 32) {
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

template <typename TS, typename TG, typename TI, bool TRACE, bool HOT>
__global__ void __launch_bounds__(kThreads, kCtasPerSm) k_gn_loop(LoopArgs<TS, TG> a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    if (__ldcg(a.chk) | __ldcg(a.chk + 1)) {  // x0 failed its checks (dynamics.py:146-149)
        if (blockIdx.x == 0 && threadIdx.x == 0) a.status[0] = 0;
        return;
    }
    TS* s_slot = (TS*)smem_raw;
    TS* s_hslot = (TS*)(smem_raw + a.hub_slot_off);
    TG* s_hot = (TG*)(smem_raw + a.hot_off);
    uint4* s_res = (uint4*)(smem_raw + a.resident_off);
    ItemSrc src{a.items, nullptr, 0};
    if (a.item_cache_off > 0) {
        const int ph0 = a.phase_base[blockIdx.x], ph1 = a.phase_base[blockIdx.x + 1];
        const int i0 = a.phase_warp[ph0 * (kWarps + 1)], i1 = a.phase_warp[(ph1 - 1) * (kWarps + 1) + kWarps];
        Item* s_items = (Item*)(smem_raw + a.item_cache_off);
        int32_t* s_deg = (int32_t*)(s_items + (i1 - i0));
        for (int t = threadIdx.x; t < (i1 - i0) * 8; t += blockDim.x)
            reinterpret_cast<int32_t*>(s_items)[t] = __ldg(reinterpret_cast<const int32_t*>(a.items + i0) + t);
        for (int t = threadIdx.x; t < (i1 - i0) * kSlice; t += blockDim.x) {
            const Item it = a.items[i0 + t / kSlice];
            const int64_t r = (int64_t)a.nhub + (int64_t)it.id * kSlice + (t % kSlice);
            s_deg[t] = (it.kind <= kPiece && r < a.n) ? __ldg(a.row_deg + (size_t)it.id * kSlice + (t % kSlice)) : 0;
        }
        src = ItemSrc{s_items, s_deg, i0};
    }
    // resident index blocks: copied once, used every iteration
    if (__ldg(a.smem_words + blockIdx.x) > 0) {
        const int ph0 = a.phase_base[blockIdx.x], ph1 = a.phase_base[blockIdx.x + 1];
        const int i0 = a.phase_warp[ph0 * (kWarps + 1)], i1 = a.phase_warp[(ph1 - 1) * (kWarps + 1) + kWarps];
        for (int i = i0; i < i1; ++i) {
            const Item it = a.items[i];
            if (it.smem < 0) continue;
            const uint4* src = reinterpret_cast<const uint4*>((const TI*)a.sell + a.slice_ptr[it.id]) +
                               (size_t)it.beg * kSlice;
            const int words = (it.end - it.beg) * kSlice;
            for (int t = threadIdx.x; t < words; t += blockDim.x) s_res[it.smem + t] = __ldg(src + t);
        }
    }
    __syncthreads();
    const FoldOut fo{a.iters, a.step_inf, a.fb, a.bad, a.dots};
    unsigned int bar = 0;
    int ran = 0, k0 = 0;
    const size_t ring_stride = (size_t)gridDim.x * kWarps * kRingW;
    // early first pairs pay on the uint16-index graphs (C2: -2%); with int32
    // indices the pair held across the barrier costs spills (C3: +4%)
    constexpr bool kEarly = sizeof(TI) == 2;
    ItemPair<TS, TI, TG> ipair;
    ipair.n = 0;
    if (kEarly) prefetch_first<TS, TG, TI>(a, 0, src, s_res, ipair);
    for (int k = 0; k < a.iters; ++k) {
        Stats st{0.0, 0u, 0, {0.0, 0.0, 0.0, 0.0}};
        const bool pr = a.prof && k == a.prof_iter && threadIdx.x == 0;
        long long* pp = a.prof ? a.prof + blockIdx.x * (kWarps + 4) : nullptr;
        if (pr) pp[0] = gtimer();
        pass<TS, TG, TI, TRACE, HOT>(a, k, false, st, s_slot, s_hslot, s_res, s_hot, src, ipair);
        if (pr) pp[1] = gtimer();
        double* slot = a.ring + (size_t)(k - k0) * ring_stride;
        publish<TRACE>(st, slot);
        if (pr) pp[2] = gtimer();
        ++bar;
        grid_arrive(a.barrier);
        // the next iteration's first items load while the other CTAs arrive
        if (kEarly && k + 1 < a.iters) prefetch_first<TS, TG, TI>(a, k + 1, src, s_res, ipair);
        grid_wait(a.barrier, bar * gridDim.x);
        if (pr) pp[3] = gtimer();
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
        ipair.n = 0;
        if (kEarly) prefetch_first<TS, TG, TI>(a, ran, src, s_res, ipair);
        pass<TS, TG, TI, TRACE, HOT>(a, ran, true, st, s_slot, s_hslot, s_res, s_hot, src, ipair);
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

// x0 checks (dynamics.py:146, 125).  A warp takes 32 consecutive rows: rows
// of up to 1024 entries are scanned by their lane (16 loads in flight), longer
// ones by the whole warp (hubs would otherwise leave one thread walking 10^5
// entries).  Once no
// entry is negative (flags[0] is reported first) a closed-neighbourhood sum of
// entries in [0, inf] U {NaN} is > 0 iff no entry is NaN and one is > 0, for
// any summation order, so the warp path tests exactly the reference's
// predicate.
__global__ void k_precheck_f64(int64_t n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                               const double* __restrict__ x, int* __restrict__ flags) {
    // With no negative entry (flags[0] takes precedence) x_i + sum_j x_j is a
    // sum of nonnegatives: it is > 0 iff some term is > 0, and NaN iff some
    // term is NaN -- and a NaN vertex fails its own row.  So each vertex tests
    // itself for NaN, and only rows whose own entry is not positive look at
    // their neighbours, stopping at the first positive one.
    const int lane = threadIdx.x & 31;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool valid = i < n;
    const double xi = valid ? x[i] : 1.0;
    if (xi < 0.0) atomicOr(&flags[0], 1);  // dynamics.py:146
    const bool need = valid && !(xi > 0.0) && xi == xi;
    const int32_t beg = need ? rowptr[i] : 0, end = need ? rowptr[i + 1] : 0;
    const bool lng = end - beg > 1024 && end - beg <= kGiantRow;  // giant rows: k_precheck_giant
    bool ok = xi == xi;  // dynamics.py:125 (NaN row)
    if (need && end - beg <= 1024) {  // 16 loads in flight per batch
        bool pos = false;
        int32_t p = beg;
        for (; p + 16 <= end && !pos; p += 16) {
            int32_t j[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) j[u] = col[p + u];
#pragma unroll
            for (int u = 0; u < 16; ++u) pos |= x[j[u]] > 0.0;
        }
        for (; p < end && !pos; ++p) pos |= x[col[p]] > 0.0;
        ok = pos;
    }
    unsigned m = __ballot_sync(0xffffffffu, lng);
    while (m) {
        const int l = __ffs(m) - 1;
        m &= m - 1;
        const int32_t bl = __shfl_sync(0xffffffffu, beg, l), el = __shfl_sync(0xffffffffu, end, l);
        bool pos = false;
        for (int32_t b0 = bl; b0 < el; b0 += 32) {  // uniform trip: the vote is warp-wide
            if (b0 + lane < el) pos |= x[col[b0 + lane]] > 0.0;
            if (__any_sync(0xffffffffu, pos)) break;
        }
        pos = __any_sync(0xffffffffu, pos);
        if (lane == l) ok = pos;
    }
    if (!ok) atomicOr(&flags[1], 1);
}

// the rows above kGiantRow (original ids perm[0, ngiant)), one CTA each; as
// above, a row whose own entry is positive (or NaN: its own thread flagged it)
// needs no scan
__global__ void k_precheck_giant(const int32_t* __restrict__ perm, const int32_t* __restrict__ rowptr,
                                 const int32_t* __restrict__ col, const double* __restrict__ x,
                                 int* __restrict__ flags) {
    const int i = perm[blockIdx.x];
    const double xi = x[i];
    if (xi > 0.0 || xi != xi) return;
    bool pos = false;
    for (int32_t p = rowptr[i] + threadIdx.x; p < rowptr[i + 1]; p += blockDim.x) pos |= x[col[p]] > 0.0;
    pos = __syncthreads_or(pos);
    if (threadIdx.x == 0 && !pos) atomicOr(&flags[1], 1);  // dynamics.py:125
}

// final state (new order) -> fp64 output (original order), np.clip(x, 0, 1)
template <typename TS>
__global__ void k_finalize(int64_t n, const TS* __restrict__ x0, const TS* __restrict__ x1,
                           const int* __restrict__ ran, const int32_t* __restrict__ inv,
                           double* __restrict__ out, int clip) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) {
        const TS* x = (__ldg(ran) & 1) ? x1 : x0;  // the state after the last iteration run
        double xi = (double)x[inv[i]];
        if (clip) xi = xi < 0.0 ? 0.0 : (xi > 1.0 ? 1.0 : xi);  // dynamics.py:179
        out[i] = xi;
    }
}

static int blocks_for(int64_t n) { return (int)std::max<int64_t>(1, (n + 255) / 256); }

int enqueue_precheck(const gn_graph* g, const double* x, int* flags, cudaStream_t s) {
    if (g->n <= 0) return GN_OK;
    k_precheck_f64<<<blocks_for(g->n), 256, 0, s>>>(g->n, g->rowptr, g->col, x, flags);
    GN_LAUNCHED();
    if (g->ngiant) {
        k_precheck_giant<<<g->ngiant, 512, 0, s>>>(g->perm, g->rowptr, g->col, x, flags);
        GN_LAUNCHED();
    }
    return GN_OK;
}


// ------------------------------------------------------------------ plan

// Device copy of one HostPlan; built on first use and cached per (graph,
// grid, mode) -- graphs are immutable.
struct DevicePlan {
    int32_t* phase_base = nullptr;
    int32_t* phase_warp = nullptr;
    int32_t* phase_comb = nullptr;
    Item* items = nullptr;
    Combine* combs = nullptr;
    int32_t* smem_words = nullptr;
    int max_slots = 0, max_hub_slots = 0, max_words = 0;
    int max_cta_items = 0;  // most items any CTA holds
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
        void* ptrs[] = {kv.second.phase_base, kv.second.phase_warp, kv.second.phase_comb, kv.second.items,
                        kv.second.combs, kv.second.smem_words};
        for (void* p : ptrs) cudaFree(p);
    }
    delete it->second;
    g_cache.erase(it);
}

template <typename T>
static int upload(const std::vector<T>& h, T** d) {
    GN_CUDA(cudaMalloc((void**)d, sizeof(T) * std::max<size_t>(h.size(), 1)));
    if (!h.empty()) GN_CUDA(cudaMemcpy(*d, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice));
    return GN_OK;
}

static int get_plan(gn_graph* g, int G, bool exact, size_t resident_cap, const DevicePlan** out) {
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
    std::vector<int64_t> sp((size_t)g->nslices + 1);
    GN_CUDA(cudaMemcpy(sp.data(), g->slice_ptr, sizeof(int64_t) * sp.size(), cudaMemcpyDeviceToHost));
    std::vector<int32_t> hp((size_t)g->nhub + 1);
    GN_CUDA(cudaMemcpy(hp.data(), g->hub_ptr, sizeof(int32_t) * hp.size(), cudaMemcpyDeviceToHost));
    PlanInput in{g->n, g->nhub, g->nslices, g->nsplit, g->idx16 ? 8 : 4, &sp, &hp, &g->slice_sig,
                 !g->slice_sig.empty()};
    HostPlan hpn;
    build_plan(in, G, exact, resident_cap, hpn);
    if (getenv("GN_PLAN_DUMP")) {  // diagnosis: items per warp by kind, phases, residency
        std::vector<int> per_kind(4, 0);
        int max_items = 0, max_phases = 0;
        double sum_items = 0;
        for (int b = 0; b < G; ++b) {
            const int ph0 = hpn.phase_base[(size_t)b], ph1 = hpn.phase_base[(size_t)b + 1];
            max_phases = std::max(max_phases, ph1 - ph0);
            for (int ph = ph0; ph < ph1; ++ph)
                for (int w = 0; w < kWarps; ++w) {
                    const int i0 = hpn.phase_warp[(size_t)ph * (kWarps + 1) + w];
                    const int i1 = hpn.phase_warp[(size_t)ph * (kWarps + 1) + w + 1];
                    max_items = std::max(max_items, i1 - i0);
                    sum_items += i1 - i0;
                    for (int i = i0; i < i1; ++i) per_kind[(size_t)hpn.items[(size_t)i].kind]++;
                }
        }
        if (getenv("GN_PLAN_DUMP")[0] == '2')
            for (int b = 0; b < G; ++b) {
                const int ph0 = hpn.phase_base[(size_t)b], ph1 = hpn.phase_base[(size_t)b + 1];
                int cnt[4] = {0, 0, 0, 0}, res = 0;
                long long elems = 0;
                for (int ph = ph0; ph < ph1; ++ph)
                    for (int i = hpn.phase_warp[(size_t)ph * (kWarps + 1)]; i < hpn.phase_warp[(size_t)ph * (kWarps + 1) + kWarps]; ++i) {
                        const Item& it = hpn.items[(size_t)i];
                        cnt[it.kind]++;
                        if (it.smem >= 0) res++;
                        elems += it.kind <= kPiece ? (long long)(it.end - it.beg) * 32 * in.B : (it.end - it.beg);
                    }
                fprintf(stderr, "[cta %d] whole=%d piece=%d hub=%d resident=%d elems=%lld combs=%d\n", b, cnt[0], cnt[1],
                        cnt[2], res, elems, hpn.phase_comb[(size_t)ph1] - hpn.phase_comb[(size_t)ph0]);
            }
        fprintf(stderr, "[plan] G=%d nhub=%d nslices=%d nsplit=%d items: whole=%d piece=%d hubpiece=%d hubseq=%d "
                        "per-warp mean=%.2f max=%d phases/CTA max=%d combines=%zu resident=%.1f MB\n",
                G, g->nhub, g->nslices, g->nsplit, per_kind[0], per_kind[1], per_kind[2], per_kind[3],
                sum_items / (G * kWarps), max_items, max_phases, hpn.combs.size(), hpn.resident_words * 16 / 1e6);
    }
    DevicePlan p;
    int rc;
    if ((rc = upload(hpn.phase_base, &p.phase_base)) || (rc = upload(hpn.phase_warp, &p.phase_warp)) ||
        (rc = upload(hpn.phase_comb, &p.phase_comb)) || (rc = upload(hpn.items, &p.items)) ||
        (rc = upload(hpn.combs, &p.combs)) || (rc = upload(hpn.smem_words, &p.smem_words)))
        return rc;
    p.max_slots = hpn.max_slots;
    p.max_hub_slots = hpn.max_hub_slots;
    for (int32_t w : hpn.smem_words) p.max_words = std::max(p.max_words, w);
    for (int b = 0; b < G; ++b) {
        const int ph0 = hpn.phase_base[(size_t)b], ph1 = hpn.phase_base[(size_t)b + 1];
        if (ph1 > ph0)
            p.max_cta_items = std::max(p.max_cta_items, hpn.phase_warp[(size_t)(ph1 - 1) * (kWarps + 1) + kWarps] -
                                                            hpn.phase_warp[(size_t)ph0 * (kWarps + 1)]);
    }
    p.resident_words = hpn.resident_words;
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

    // ---- launch geometry and plan
    const bool hot = g->hot > 0 && sizeof(TI) == 4;
    void* kern;
    if (hot) kern = trace ? (void*)k_gn_loop<TS, TG, TI, true, true> : (void*)k_gn_loop<TS, TG, TI, false, true>;
    else kern = trace ? (void*)k_gn_loop<TS, TG, TI, true, false> : (void*)k_gn_loop<TS, TG, TI, false, false>;
    int max_optin = 0;
    GN_CUDA(cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, g->device));
    const size_t hot_bytes = hot ? (size_t)g->hot * sizeof(TG) : 0;
    const size_t slot_bytes = (size_t)kMaxSlots * kSlice * sizeof(TS) + (size_t)kMaxHubSlots * sizeof(TS) + hot_bytes;
    const size_t static_bytes = 2048;  // publish scratch
    // index residency budget (GN_SMEM_RES_KB): off -- the L1 is worth more
    // than resident indices (C5 scale 24: 3.0 -> 2.1 ms/iteration without;
    // C2 with co-located slices: equal)
    size_t res_cap = 0;
    if (const char* e = getenv("GN_SMEM_RES_KB")) res_cap = (size_t)atoi(e) * 1024;
    int smem_sm = 0;
    GN_CUDA(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, g->device));
    const size_t per_cta = std::min<size_t>((size_t)max_optin, (size_t)smem_sm / kCtasPerSm - 1024);
    res_cap = std::min(res_cap, per_cta > static_bytes + slot_bytes ? per_cta - static_bytes - slot_bytes : 0);
    const size_t smem_cap = slot_bytes + res_cap;
    GN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_cap));
    int maxb = 1;
    if ((rc = coresident_blocks(kern, kThreads, smem_cap, g->device, &maxb))) return rc;
    if (maxb < 1) return fail(GN_ERR_CUDA, "loop kernel cannot be resident");
    const int64_t work = g->sell_elems + 4 * n + (g->nhub ? 32768 : 0);
    int grid = (int)std::min<int64_t>(maxb, std::max<int64_t>(1, (work + 16383) / 16384));
    if (g->grid_override > 0) grid = std::min(maxb, g->grid_override);
    const DevicePlan* plan = nullptr;
    if ((rc = get_plan(g, grid, exact, res_cap, &plan))) return rc;
    // shared memory sized to what the plan uses (whatever is left is L1)
    const int hub_slot_off = (int)(((size_t)plan->max_slots * kSlice * sizeof(TS) + 15) / 16 * 16);
    const int hot_off = (int)(((size_t)hub_slot_off + (size_t)plan->max_hub_slots * sizeof(TS) + 15) / 16 * 16);
    const int resident_off = (int)(((size_t)hot_off + hot_bytes + 15) / 16 * 16);
    size_t dyn_smem = (size_t)resident_off + (size_t)plan->max_words * 16;
    // the CTA's item descriptors and slice-row degrees, when they fit
    int item_cache_off = 0;
    {
        const size_t off = (dyn_smem + 15) / 16 * 16;
        const size_t bytes = (size_t)plan->max_cta_items * (sizeof(Item) + kSlice * sizeof(int32_t));
        // small enough not to cost the gathers their L1 (C5 scale 20: 67 KB of
        // items made the iteration 30% slower)
        if (!getenv("GN_NO_ITEM_CACHE") && plan->max_cta_items > 0 && bytes <= 32 * 1024 &&
            off + bytes + static_bytes <= per_cta) {
            item_cache_off = (int)off;
            dyn_smem = off + bytes;
            GN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)std::max(dyn_smem, smem_cap)));
        }
    }

    Workspace ws;
    ws.s = s;
    TS *xa, *xb;
    TG *ya, *yb;
    double *xin, *dots, *ring, *gam, *out64 = nullptr, *hist = nullptr, *dsi, *dfb;
    int *dbad, *status, *chk;
    unsigned int* barrier;
    GN_CUDA(ws.alloc(&xa, sizeof(TS) * nb));
    GN_CUDA(ws.alloc(&xb, sizeof(TS) * nb));
    // published values, each buffer with the zero vertex n at its end (SELL padding ids point there)
    GN_CUDA(ws.alloc(&ya, sizeof(TG) * (nb + 1)));
    GN_CUDA(ws.alloc(&yb, sizeof(TG) * (nb + 1)));
    GN_CUDA(cudaMemsetAsync(ya + n, 0, sizeof(TG), s));
    GN_CUDA(cudaMemsetAsync(yb + n, 0, sizeof(TG), s));
    GN_CUDA(ws.alloc(&dsi, 8 * (size_t)iters));
    GN_CUDA(ws.alloc(&dfb, 8 * (size_t)iters));
    GN_CUDA(ws.alloc(&dbad, 4 * (size_t)iters));
    GN_CUDA(ws.alloc(&dots, 8 * 4 * (size_t)(iters + 1)));
    GN_CUDA(ws.alloc(&ring, 8 * (size_t)kRingW * (size_t)std::min(kRing, iters + 1) * grid * kWarps));
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

    if (x_out && n > 0 && !dev_io) GN_CUDA(ws.alloc(&out64, 8 * nb));
    // the device-timed region starts here: set-up above is host work and
    // stream-ordered allocation, everything below is enqueued back to back
    GN_CUDA(cudaEventRecord(ev[0], s));

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
            if ((rc = enqueue_precheck(g, xin, chk, s))) return rc;
        }
        k_prepare<TS, TG><<<blocks_for(n), 256, 0, s>>>(n, xin, g->inv, (const TS*)g->v, xa, ya);
        GN_LAUNCHED();
    }
    // the check flags are read by the loop kernel itself (it exits at once
    // when one is set) and by the host with the results: no sync here

    // ---- the loop
    LoopArgs<TS, TG> a;
    memset(&a, 0, sizeof(a));
    a.n = n;
    a.nhub = g->nhub;
    a.hub_ptr = g->hub_ptr;
    // fast mode reads the rows in ascending new id when the graph has that copy
    const bool fast_layout = !exact && g->sell_fast;
    a.hub_col = fast_layout ? g->hub_col_fast : g->hub_col;
    a.slice_ptr = g->slice_ptr;
    a.row_deg = g->row_deg;
    a.sell = fast_layout ? g->sell_fast : g->sell;
    a.v = (const TS*)g->v;
    a.w = (const TS*)g->w;
    a.x[0] = xa;
    a.x[1] = xb;
    a.yg[0] = ya;
    a.yg[1] = yb;
    a.phase_base = plan->phase_base;
    a.phase_warp = plan->phase_warp;
    a.phase_comb = plan->phase_comb;
    a.items = plan->items;
    a.combs = plan->combs;
    a.smem_words = plan->smem_words;
    a.hub_slot_off = hub_slot_off;
    a.hot_off = hot_off;
    a.hot = hot ? g->hot : 0;
    a.resident_off = resident_off;
    a.item_cache_off = item_cache_off;
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
    a.chk = chk;
    long long* dprof = nullptr;
    const char* prof_env = getenv("GN_PROF_ITER");
    if (prof_env) {
        a.prof_iter = atoi(prof_env);
        GN_CUDA(ws.alloc(&dprof, sizeof(long long) * (size_t)grid * (kWarps + 4)));
        GN_CUDA(cudaMemsetAsync(dprof, 0, sizeof(long long) * (size_t)grid * (kWarps + 4), s));
        a.prof = dprof;
    }
    void* args[] = {&a};
    GN_CUDA(cudaEventRecord(ev[1], s));
    GN_CUDA(cudaLaunchCooperativeKernel(kern, dim3(grid), dim3(kThreads), args, dyn_smem, s));
    GN_LAUNCHED();
    GN_CUDA(cudaEventRecord(ev[2], s));

    // ---- results back; the final state is picked on the device (buffer of
    // the last iteration run), so nothing waits for the host before ev[3]
    const int clip = (flags & GN_NO_CLIP) ? 0 : 1;
    if (x_out && n > 0) {
        k_finalize<TS><<<blocks_for(n), 256, 0, s>>>(n, xa, xb, status, g->inv, dev_io ? (double*)x_out : out64, clip);
        GN_LAUNCHED();
        if (!dev_io) {
            GN_CUDA(cudaMemcpyAsync(x_out, out64, 8 * (size_t)n, cudaMemcpyDeviceToHost, s));
            d2h += 8 * n;
        }
    }
    int hstatus[4], hchk[2] = {0, 0};
    GN_CUDA(cudaMemcpyAsync(hstatus, status, sizeof(hstatus), cudaMemcpyDeviceToHost, s));
    GN_CUDA(cudaMemcpyAsync(hchk, chk, sizeof(hchk), cudaMemcpyDeviceToHost, s));
    std::vector<double> hsi((size_t)iters), hfb((size_t)iters);
    std::vector<int> hbad((size_t)iters);
    std::vector<double> hdots(4 * (size_t)(iters + 1));
    GN_CUDA(cudaMemcpyAsync(hsi.data(), dsi, 8 * (size_t)iters, cudaMemcpyDeviceToHost, s));
    GN_CUDA(cudaMemcpyAsync(hfb.data(), dfb, 8 * (size_t)iters, cudaMemcpyDeviceToHost, s));
    GN_CUDA(cudaMemcpyAsync(hbad.data(), dbad, 4 * (size_t)iters, cudaMemcpyDeviceToHost, s));
    GN_CUDA(cudaMemcpyAsync(hdots.data(), dots, 8 * 4 * (size_t)(iters + 1), cudaMemcpyDeviceToHost, s));
    d2h += 8 * 2 * iters + 4 * iters + 8 * 4 * (iters + 1) + 16;
    GN_CUDA(cudaEventRecord(ev[3], s));
    GN_CUDA(cudaStreamSynchronize(s));
    if (hchk[0]) return fail(GN_ERR_NEGATIVE, "state entries must be nonnegative");             // dynamics.py:147
    if (hchk[1]) return fail(GN_ERR_NOT_NORMALIZABLE, "initial state has a zero closed neighborhood sum");  // :149
    const int ran = hstatus[0];
    if (x_hist && n > 0 && ran > 0) {  // test aid, outside the timed region
        GN_CUDA(cudaMemcpyAsync(x_hist, hist, 8 * (size_t)ran * (size_t)n, cudaMemcpyDeviceToHost, s));
        d2h += 8 * (int64_t)ran * n;
        GN_CUDA(cudaStreamSynchronize(s));
    }
    if (dprof) {
        std::vector<long long> hp((size_t)grid * (kWarps + 4));
        GN_CUDA(cudaMemcpy(hp.data(), dprof, sizeof(long long) * hp.size(), cudaMemcpyDeviceToHost));
        const char* path = getenv("GN_PROF_OUT");
        FILE* f = fopen(path ? path : "gn_prof.txt", "a");
        if (f) {
            long long t0 = LLONG_MAX;
            for (int b = 0; b < grid; ++b) t0 = std::min(t0, hp[(size_t)b * (kWarps + 4)]);
            fprintf(f, "# grid %d iter %d: cta pass_start pass_end publish_end barrier_end | warp item ns\n", grid,
                    a.prof_iter);
            for (int b = 0; b < grid; ++b) {
                const long long* q = &hp[(size_t)b * (kWarps + 4)];
                fprintf(f, "%d %lld %lld %lld %lld |", b, q[0] - t0, q[1] - t0, q[2] - t0, q[3] - t0);
                for (int w = 0; w < kWarps; ++w) fprintf(f, " %lld", q[4 + w]);
                fprintf(f, "\n");
            }
            fclose(f);
        }
    }

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
    GN_NVTX("gn_run");
    if (!g) return fail(GN_ERR_ARG, "null graph");
    if (iters < 1) return fail(GN_ERR_ARG, "iterations must be positive");
    if (!gammas || (g->n > 0 && !x0)) return fail(GN_ERR_ARG, "null input array");
    if (g->resident && !getenv("GN_NO_RESIDENT")) {
        int st = GN_OK, fi = -1, ran = 0;
        int rc = batch_run(g->resident, x0, gammas, iters, final_gamma, flags, x_out, step_inf, fallbacks, mass,
                           energy, pre_energy, x_hist, &ran, &st, &fi, stats);
        if (iters_run) *iters_run = ran;
        if (fail_iter) *fail_iter = fi;
        return rc;
    }
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
    GN_NVTX("gn_step");
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
