// gn_multi.cu -- several starts of run_wrgn on one graph, advanced together
// (the multi-start solve of solver.solve_instance,
// solver.py:100-153, which the reference fans out over a thread pool).
//
// State is stored start-minor: x[v][b], y[v][b] for the Bp (padded) starts,
// so gathering neighbour j for every start is one contiguous Bp-vector read
// instead of Bp scattered reads -- the index bytes and the random-access
// sectors of the single-start loop are shared by all starts.
//
// Mapping: a team of T lanes owns one row; lane t of the team owns starts
// [t*S, t*S+S) (S = 16 bytes / gathered value: 2 fp64 or 4 fp32), so each
// gather is one 16-byte load per lane and the team's loads cover the row's
// whole Bp-vector.  A warp works 32/T rows at a time, its rows taken in the
// multi-id order (degree-sorted in windows, see multi_csr) so they have similar
// lengths.  The team walks the row in the reference's neighbour order: lanes
// fetch 16 consecutive column indices cooperatively, broadcast them by
// shuffle and issue 16 gathers before adding them in order.  Every start's
// row sum is therefore the sequential sum of dynamics.py:105 (scipy's
// csr_matvec order), and every start's trajectory is bitwise the single
// run's (gn_run with GN_EXACT).
//
// Rows go to warps in contiguous ranges of the relabel order balanced by
// gathers (host plan, cached per graph and grid).  One persistent
// co-resident kernel runs all iterations, a grid barrier between them.  Per
// iteration and start: max|x'-x| (atomicMax on the bits of a non-negative
// double -- exact), the fallback count and the non-finite flag; after the
// barrier every CTA reads them and freezes the starts that stopped
// (non-finite state, dynamics.py:175-176; early exit, 177-178), whose state
// is then left untouched.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <thread>
#include <tuple>
#include <vector>

#include "gn_internal.cuh"

namespace gn {

constexpr int kMThreads = 512;
constexpr int kMWarps = kMThreads / 32;
// gathers in flight per lane: 16 on graphs with long rows (C2: 13.6 us per
// start-iteration against 15.8 with 8), 8 on short-row graphs, where the
// deeper batch mostly masks and spills (C3 5.3 -> 4.8, R-MAT 24 636 -> 578)
constexpr int kMUDeep = 16, kMUShort = 8;
static inline int multi_mu(const gn_graph* g) { return g->n > 0 && g->nnz >= 64 * g->n ? kMUDeep : kMUShort; }
constexpr int kMaxStarts = 64;

template <typename TG>
struct Pack;
template <>
struct Pack<double> {
    using T = double2;
    static constexpr int S = 2;
    __device__ static __forceinline__ double at(const T& p, int s) { return s == 0 ? p.x : p.y; }
};
template <>
struct Pack<float> {
    using T = float4;
    static constexpr int S = 4;
    __device__ static __forceinline__ float at(const T& p, int s) {
        return s == 0 ? p.x : s == 1 ? p.y : s == 2 ? p.z : p.w;
    }
};

// A row as the kernel walks it: original id, CSR offset, degree.
struct RowDesc {
    int32_t r, rb, deg, pad;
};

template <typename TS, typename TG>
struct MultiArgs {
    int64_t n;
    int B, Bp;
    const int32_t* __restrict__ col;     // original CSR column indices
    const int4* __restrict__ rdesc;      // regular rows in processing order (RowDesc)
    const int32_t* __restrict__ wbeg;    // [G * kMWarps + 1] ranges of rdesc per warp
    const int32_t* __restrict__ wmid;    // [G * kMWarps]: rows [wbeg, wmid) are warp rows (fast mode)
    const int4* __restrict__ hdesc;      // split rows (fast mode), grouped by CTA
    const int32_t* __restrict__ hbeg;    // [G + 1] ranges of hdesc per CTA
    const TS* __restrict__ v;            // original order
    TS* x[2];                            // [n][Bp]
    TG* yg[2];                           // [n][Bp]
    const double* __restrict__ gammas;
    int iters;
    double final_gamma;
    int early_exit;
    unsigned long long* sinf;  // [iters][B]: bits of max|x'-x|
    unsigned int* fb;          // [iters][B]
    int* bad;                  // [iters][B]
    int* run;                  // [B]: iterations run
    const int* skip;           // [B]: 1 = failed its checks, not run
    unsigned int* barrier;
};

template <int T, int kMU>
struct TeamIdx {
    static constexpr int NI = (kMU + T - 1) / T;  // index registers per lane
    // positions q + i*T + t (i*T + t < kMU) of a segment of length len
    __device__ static __forceinline__ void load(const int32_t* __restrict__ colp, int q, int len, int t,
                                                int (&idx)[NI]) {
#pragma unroll
        for (int i = 0; i < NI; ++i) {
            const int pos = q + i * T + t;
            idx[i] = (i * T + t < kMU && pos < len) ? __ldg(colp + pos) : 0;
        }
    }
};

// Sequential sum, for the lane's S starts, of positions [0, len) of one row
// segment (colp = its first column index); idx holds the first index chunk.
// lmax / lmin: the warp's longest / shortest segment (all teams step together).
template <typename TS, typename TG, int T, int kMU>
__device__ __forceinline__ void team_sum(const int32_t* __restrict__ colp, int len, int lmax, int lmin,
                                         int (&idx)[TeamIdx<T, kMU>::NI], const TG* __restrict__ ybase, int Bp,
                                         int tbase, int t, TS (&acc)[Pack<TG>::S]) {
    using A = Arith<TS>;
    using P = Pack<TG>;
    using PT = typename P::T;
    constexpr int S = P::S, NI = TeamIdx<T, kMU>::NI;
#pragma unroll
    for (int s = 0; s < S; ++s) acc[s] = TS(0);
    for (int q = 0; q < lmax; q += kMU) {
        int nidx[NI];
        TeamIdx<T, kMU>::load(colp, q + kMU, len, t, nidx);
        PT val[kMU];
        if (q + kMU <= lmin) {
#pragma unroll
            for (int u = 0; u < kMU; ++u) {
                const int j = __shfl_sync(0xffffffffu, idx[u / T], tbase + (u & (T - 1)));
                val[u] = __ldg(reinterpret_cast<const PT*>(ybase + (size_t)j * Bp));
            }
        } else {
#pragma unroll
            for (int u = 0; u < kMU; ++u) {
                const int j = __shfl_sync(0xffffffffu, idx[u / T], tbase + (u & (T - 1)));
                if (q + u < len) val[u] = __ldg(reinterpret_cast<const PT*>(ybase + (size_t)j * Bp));
                else val[u] = PT();
            }
        }
#pragma unroll
        for (int u = 0; u < kMU; ++u)
#pragma unroll
            for (int s = 0; s < S; ++s) acc[s] = A::add(acc[s], (TS)P::at(val[u], s));
#pragma unroll
        for (int i = 0; i < NI; ++i) idx[i] = nidx[i];
    }
}

// dynamics.py:104-107 for one (row, start); stats of that start
template <typename TS, typename TG>
__device__ __forceinline__ void update_one(TS xi, TS vi, TS sum, TS g, TS* xn, TG* yn, double& mx, unsigned int& fbc,
                                           int& bd) {
    using A = Arith<TS>;
    const TS yi = A::mul(vi, xi);
    const TS d = A::add(yi, A::mul(g, sum));
    const bool ok = (double)d > kSafeDiv;
    const TS o = ok ? A::div(yi, d) : TS(kFallback);
    *xn = o;
    *yn = (TG)A::mul(vi, o);
    TS df = A::sub(o, xi);  // dynamics.py:165
    df = df < TS(0) ? -df : df;
    if (!((double)df <= mx)) mx = (double)df;
    fbc += ok ? 0u : 1u;
    if (!isfinite((double)o)) bd = 1;
}

// Sum of a value over the warp's teams (lanes with equal t), the same fixed
// butterfly on every lane (IEEE addition is commutative: all lanes agree).
template <typename TS, int T>
__device__ __forceinline__ TS fold_teams(TS v) {
#pragma unroll
    for (int o = T; o < 32; o <<= 1) v = Arith<TS>::add(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__device__ __forceinline__ RowDesc row_at(const int4* __restrict__ d, int i, int end) {
    if (i < end) {
        const int4 q = __ldg(d + i);
        return RowDesc{q.x, q.y, q.z, 0};
    }
    return RowDesc{-1, 0, 0, 0};
}

// Position in a warp's step stream (see k_gn_multi).
constexpr int kStepCta = 0, kStepWarp = 1, kStepTeam = 2, kStepDone = 3;
struct StepPos {
    int ph, i;
};

__device__ __forceinline__ StepPos first_step(int h0, int h1, int p0, int pm, int p1) {
    if (h0 < h1) return StepPos{kStepCta, h0};
    if (p0 < pm) return StepPos{kStepWarp, p0};
    if (pm < p1) return StepPos{kStepTeam, pm};
    return StepPos{kStepDone, 0};
}

__device__ __forceinline__ StepPos next_step(StepPos q, int rpw, int h1, int p0, int pm, int p1) {
    if (q.ph == kStepCta && q.i + 1 < h1) return StepPos{kStepCta, q.i + 1};
    if (q.ph == kStepCta && p0 < pm) return StepPos{kStepWarp, p0};
    if (q.ph == kStepWarp && q.i + 1 < pm) return StepPos{kStepWarp, q.i + 1};
    if ((q.ph == kStepCta || q.ph == kStepWarp) && pm < p1) return StepPos{kStepTeam, pm};
    if (q.ph == kStepTeam && q.i + rpw < p1) return StepPos{kStepTeam, q.i + rpw};
    return StepPos{kStepDone, 0};
}

template <typename TS, typename TG>
__device__ __forceinline__ RowDesc step_desc(const MultiArgs<TS, TG>& a, StepPos q, int team, int h1, int pm, int p1) {
    if (q.ph == kStepCta) return row_at(a.hdesc, q.i, h1);
    if (q.ph == kStepWarp) return row_at(a.rdesc, q.i, pm);
    if (q.ph == kStepTeam) return row_at(a.rdesc, q.i + team, p1);
    return RowDesc{-1, 0, 0, 0};
}

// this team's segment [beg, beg + len) of the step's row
template <int RPW, int NT>
__device__ __forceinline__ void step_segment(StepPos q, const RowDesc& d, int team, int tau, int& beg, int& len) {
    int parts = 1, part = 0;
    if (q.ph == kStepCta) {
        parts = NT;
        part = tau;
    } else if (q.ph == kStepWarp) {
        parts = RPW;
        part = team;
    }
    beg = (int)((int64_t)d.deg * part / parts);
    len = (int)((int64_t)d.deg * (part + 1) / parts) - beg;
}

template <typename TS, typename TG, int T, int kMU>
__global__ void __launch_bounds__(kMThreads, 1) k_gn_multi(MultiArgs<TS, TG> a) {
    using A = Arith<TS>;
    using TI = TeamIdx<T, kMU>;
    constexpr int S = Pack<TG>::S, NI = TI::NI;
    constexpr int RPW = 32 / T;              // rows a warp works at once
    constexpr int NT = kMWarps * RPW;        // teams per CTA
    __shared__ unsigned char s_frozen[kMaxStarts];
    __shared__ double s_mx[kMWarps][kMaxStarts];
    __shared__ unsigned int s_fb[kMWarps][kMaxStarts];
    __shared__ int s_bad[kMWarps][kMaxStarts];
    __shared__ double s_hmx[kMaxStarts];
    __shared__ unsigned int s_hfb[kMaxStarts];
    __shared__ int s_hbad[kMaxStarts];
    __shared__ TS s_part[kMWarps * T * S];   // per-warp partials of a CTA row
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tbase = lane & ~(T - 1), t = lane & (T - 1), team = lane / T;
    const int tau = warp * RPW + team;
    const int B = a.B, Bp = a.Bp;
    if (threadIdx.x < kMaxStarts) s_frozen[threadIdx.x] = (threadIdx.x >= B || a.skip[threadIdx.x]) ? 1 : 0;
    __syncthreads();
    const int gw = blockIdx.x * kMWarps + warp;
    const int p0 = __ldg(a.wbeg + gw), pm = __ldg(a.wmid + gw), p1 = __ldg(a.wbeg + gw + 1);
    const int h0 = __ldg(a.hbeg + blockIdx.x), h1 = __ldg(a.hbeg + blockIdx.x + 1);
    unsigned int bar = 0;
    for (int k = 0; k < a.iters; ++k) {
        const int cur = k & 1;
        const TS g = (TS)a.gammas[k];
        const TG* __restrict__ ybase = a.yg[cur] + t * S;
        double mx[S];
        unsigned int fbc[S];
        int bd[S];
#pragma unroll
        for (int s = 0; s < S; ++s) {
            mx[s] = 0.0;
            fbc[s] = 0u;
            bd[s] = 0;
        }
        if (threadIdx.x < kMaxStarts) {
            s_hmx[threadIdx.x] = 0.0;
            s_hfb[threadIdx.x] = 0u;
            s_hbad[threadIdx.x] = 0;
        }
        // ---- the warp's work as one stream of steps: CTA rows (fast mode:
        // every team of the CTA sums one piece; per-warp folds meet in shared
        // memory), then warp rows (the warp's teams split one row, folded by a
        // fixed shuffle tree), then team rows (one team per row).  Step i+2's
        // descriptor and step i+1's first index chunk load under step i's gathers.
        StepPos q0 = first_step(h0, h1, p0, pm, p1);
        RowDesc d0 = step_desc(a, q0, team, h1, pm, p1);
        StepPos q1 = next_step(q0, RPW, h1, p0, pm, p1);
        RowDesc d1 = step_desc(a, q1, team, h1, pm, p1);
        int b0, l0;
        step_segment<RPW, NT>(q0, d0, team, tau, b0, l0);
        int idx[NI];
        TI::load(a.col + d0.rb + b0, 0, l0, t, idx);
        while (q0.ph != kStepDone) {
            const StepPos q2 = next_step(q1, RPW, h1, p0, pm, p1);
            const RowDesc d2 = step_desc(a, q2, team, h1, pm, p1);
            TS xs[S];
            TS vi = TS(0);
            const size_t off = (size_t)(d0.r < 0 ? 0 : d0.r) * Bp + t * S;
            if (q0.ph != kStepCta && d0.r >= 0) {
                vi = __ldg(a.v + d0.r);
#pragma unroll
                for (int s = 0; s < S; ++s) xs[s] = a.x[cur][off + s];
            }
            int b1, l1;
            step_segment<RPW, NT>(q1, d1, team, tau, b1, l1);
            int ridx[NI];
            TI::load(a.col + d1.rb + b1, 0, l1, t, ridx);
            const int lmax = (int)__reduce_max_sync(0xffffffffu, (unsigned)l0);
            const int lmin = (int)__reduce_min_sync(0xffffffffu, (unsigned)l0);
            TS acc[S];
            team_sum<TS, TG, T, kMU>(a.col + d0.rb + b0, l0, lmax, lmin, idx, ybase, Bp, tbase, t, acc);
            if (q0.ph == kStepTeam) {
                if (d0.r >= 0) {
#pragma unroll
                    for (int s = 0; s < S; ++s) {
                        if (s_frozen[t * S + s]) continue;
                        update_one<TS, TG>(xs[s], vi, acc[s], g, a.x[cur ^ 1] + off + s, a.yg[cur ^ 1] + off + s,
                                           mx[s], fbc[s], bd[s]);
                    }
                }
            } else {
#pragma unroll
                for (int s = 0; s < S; ++s) acc[s] = fold_teams<TS, T>(acc[s]);
                if (q0.ph == kStepWarp) {
                    if (lane < T) {
#pragma unroll
                        for (int s = 0; s < S; ++s) {
                            if (s_frozen[t * S + s]) continue;
                            update_one<TS, TG>(xs[s], vi, acc[s], g, a.x[cur ^ 1] + off + s,
                                               a.yg[cur ^ 1] + off + s, mx[s], fbc[s], bd[s]);
                        }
                    }
                } else {
                    if (lane < T)
#pragma unroll
                        for (int s = 0; s < S; ++s) s_part[warp * T * S + t * S + s] = acc[s];
                    __syncthreads();
                    if (threadIdx.x < B && !s_frozen[threadIdx.x]) {
                        const int b = threadIdx.x;
                        TS tot = TS(0);
                        for (int w = 0; w < kMWarps; ++w) tot = A::add(tot, s_part[w * T * S + b]);
                        const size_t hoff = (size_t)d0.r * Bp + b;
                        update_one<TS, TG>(a.x[cur][hoff], __ldg(a.v + d0.r), tot, g, a.x[cur ^ 1] + hoff,
                                           a.yg[cur ^ 1] + hoff, s_hmx[b], s_hfb[b], s_hbad[b]);
                    }
                    __syncthreads();
                }
            }
            q0 = q1;
            d0 = d1;
            b0 = b1;
            l0 = l1;
#pragma unroll
            for (int i = 0; i < NI; ++i) idx[i] = ridx[i];
            q1 = q2;
            d1 = d2;
        }
        // ---- per start: fold the warp's teams (lanes with equal t), then the CTA
#pragma unroll
        for (int o = T; o < 32; o <<= 1) {
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const double m = __shfl_xor_sync(0xffffffffu, mx[s], o);
                if (!(m <= mx[s])) mx[s] = m;
                fbc[s] += __shfl_xor_sync(0xffffffffu, fbc[s], o);
                bd[s] |= __shfl_xor_sync(0xffffffffu, bd[s], o);
            }
        }
        if (lane < T) {
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const int b = t * S + s;
                if (b < kMaxStarts) {
                    s_mx[warp][b] = mx[s];
                    s_fb[warp][b] = fbc[s];
                    s_bad[warp][b] = bd[s];
                }
            }
        }
        __syncthreads();
        if (threadIdx.x < B && !s_frozen[threadIdx.x]) {
            const int b = threadIdx.x;
            double m = s_hmx[b];
            unsigned int f = s_hfb[b];
            int bb = s_hbad[b];
            for (int q = 0; q < kMWarps; ++q) {
                if (!(s_mx[q][b] <= m)) m = s_mx[q][b];
                f += s_fb[q][b];
                bb |= s_bad[q][b];
            }
            const size_t at = (size_t)k * B + b;
            atomicMax(a.sinf + at, (unsigned long long)__double_as_longlong(m));
            if (f) atomicAdd(a.fb + at, f);
            if (bb) atomicOr(a.bad + at, 1);
        }
        grid_barrier(a.barrier, (++bar) * gridDim.x);
        // every CTA reads the iteration's per-start stats and freezes the starts that stopped
        if (threadIdx.x < B && !s_frozen[threadIdx.x]) {
            const int b = threadIdx.x;
            const size_t at = (size_t)k * B + b;
            bool stop = __ldcg(a.bad + at) != 0;  // dynamics.py:175-176
            if (!stop && a.early_exit && a.gammas[k] == a.final_gamma)  // dynamics.py:177-178
                stop = __longlong_as_double((long long)__ldcg(a.sinf + at)) < 1e-12;
            if (stop) {
                s_frozen[b] = 1;
                if (blockIdx.x == 0) a.run[b] = k + 1;
            }
        }
        __syncthreads();
        int live = 0;
        for (int b = 0; b < B; ++b) live |= !s_frozen[b];
        if (!live) break;
    }
    if (blockIdx.x == 0 && threadIdx.x < B && !s_frozen[threadIdx.x]) a.run[threadIdx.x] = a.iters;
}

// x0 [B][n] (fp64, original order) -> x[0], yg[0] ([n][Bp], multi-id rows); padding starts are 0
template <typename TS, typename TG>
__global__ void k_multi_prepare(int64_t n, int B, int Bp, const double* __restrict__ x0, const int32_t* __restrict__ perm,
                                const TS* __restrict__ v, TS* __restrict__ x, TG* __restrict__ yg) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n * Bp) return;
    const int64_t r = e / Bp;  // multi id
    const int b = (int)(e % Bp);
    const TS xi = b < B ? (TS)x0[(size_t)b * n + perm[r]] : TS(0);
    x[e] = xi;
    yg[e] = (TG)Arith<TS>::mul(v[r], xi);
}

// sqrt(w) in state precision, multi-id order (graph.py:42, as k_init_state_weights)
template <typename TS>
__global__ void k_multi_weights(int64_t n, const double* __restrict__ w64, const int32_t* __restrict__ perm,
                                TS* __restrict__ v) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) v[i] = (TS)sqrt(w64[perm[i]]);
}

// final state of start b (buffer run[b] & 1) -> x_out [B][n], np.clip(x, 0, 1)
template <typename TS>
__global__ void k_multi_finalize(int64_t n, int B, int Bp, const TS* __restrict__ x0, const TS* __restrict__ x1,
                                 const int* __restrict__ run, const int32_t* __restrict__ inv,
                                 double* __restrict__ out, int clip) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n * B) return;
    const int b = (int)(e / n);
    const int64_t r = inv[e % n];  // original id -> multi id
    double xi = (double)((run[b] & 1) ? x1 : x0)[(size_t)r * Bp + b];
    if (clip) xi = xi < 0.0 ? 0.0 : (xi > 1.0 ? 1.0 : xi);  // dynamics.py:179
    out[e] = xi;
}

// ---- host plan (cached per graph, grid and mode) -------------------------
// Fast mode splits rows longer than one warp's fair share over all teams of a
// CTA (LPT over CTAs); the remaining rows, in the relabel order (degree-sorted:
// a warp's concurrent rows have similar lengths), are cut into contiguous
// per-warp ranges so that every CTA carries the same gathers in total.
struct MultiPlan {
    int4* rdesc = nullptr;
    int32_t* wbeg = nullptr;
    int32_t* wmid = nullptr;
    int4* hdesc = nullptr;
    int32_t* hbeg = nullptr;
};
static std::mutex g_mplan_mu;
static std::map<std::tuple<const gn_graph*, int, int, int>, MultiPlan> g_mplans;
struct MultiCsr {
    int32_t* rowptr = nullptr;
    int32_t* col = nullptr;   // neighbours as multi ids, the reference's order
    int32_t* perm = nullptr;  // multi id -> original id
    int32_t* inv = nullptr;   // original id -> multi id
    std::vector<int32_t> h_rowptr;
};
static std::map<const gn_graph*, MultiCsr> g_mcsr;

void release_multi_plans(const gn_graph* g) {
    std::lock_guard<std::mutex> lk(g_mplan_mu);
    auto mc = g_mcsr.find(g);
    if (mc != g_mcsr.end()) {
        cudaFree(mc->second.rowptr);
        cudaFree(mc->second.col);
        cudaFree(mc->second.perm);
        cudaFree(mc->second.inv);
        g_mcsr.erase(mc);
    }
    for (auto it = g_mplans.begin(); it != g_mplans.end();) {
        if (std::get<0>(it->first) == g) {
            cudaFree(it->second.rdesc);
            cudaFree(it->second.wbeg);
            cudaFree(it->second.wmid);
            cudaFree(it->second.hdesc);
            cudaFree(it->second.hbeg);
            it = g_mplans.erase(it);
        } else {
            ++it;
        }
    }
}

template <typename V>
static int upload_vec(const std::vector<V>& h, V** d) {
    GN_CUDA(cudaMalloc((void**)d, sizeof(V) * std::max<size_t>(h.size(), 1)));
    if (!h.empty()) GN_CUDA(cudaMemcpy(*d, h.data(), sizeof(V) * h.size(), cudaMemcpyHostToDevice));
    return GN_OK;
}

// The graph in the multi-start kernel's own order: hubs (degree > 512,
// degree-descending) first, then the other rows degree-descending inside
// windows of 4096 original ids -- consecutive rows keep the neighbourhood
// locality of the caller's numbering, which the start-minor gathers (one
// 16-byte vector per lane per neighbour) use better than the single-start
// loop's global degree order (C5 scale 24 x16 fp32: 645 vs 910 us per
// start-iteration).  State rows follow this order (multi ids); neighbour
// lists keep the reference's order, so every start sums as dynamics.py:105
// does.  Built once per graph on first use.
static int multi_csr(gn_graph* g, const MultiCsr** out) {  // caller holds g_mplan_mu
    auto it = g_mcsr.find(g);
    if (it != g_mcsr.end()) {
        *out = &it->second;
        return GN_OK;
    }
    const int64_t n = g->n, nnz = g->nnz;
    std::vector<int32_t> rp((size_t)n + 1), col((size_t)std::max<int64_t>(nnz, 1));
    GN_CUDA(cudaMemcpy(rp.data(), g->rowptr, sizeof(int32_t) * rp.size(), cudaMemcpyDeviceToHost));
    if (nnz) GN_CUDA(cudaMemcpy(col.data(), g->col, sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost));
    auto deg = [&](int32_t r) { return rp[(size_t)r + 1] - rp[(size_t)r]; };
    std::vector<int32_t> hubs, regular;
    for (int64_t i = 0; i < n; ++i) (deg((int32_t)i) > kHubDegree ? hubs : regular).push_back((int32_t)i);
    auto by_deg = [&](int32_t a, int32_t b) { return deg(a) > deg(b); };
    std::stable_sort(hubs.begin(), hubs.end(), by_deg);
    for (size_t w0 = 0; w0 < regular.size(); w0 += kSigma)
        std::stable_sort(regular.begin() + w0, regular.begin() + std::min(regular.size(), w0 + kSigma), by_deg);
    std::vector<int32_t> perm = hubs;
    perm.insert(perm.end(), regular.begin(), regular.end());
    std::vector<int32_t> inv((size_t)std::max<int64_t>(n, 1));
    for (int64_t r = 0; r < n; ++r) inv[(size_t)perm[(size_t)r]] = (int32_t)r;
    MultiCsr m;
    m.h_rowptr.assign((size_t)n + 1, 0);
    for (int64_t r = 0; r < n; ++r) m.h_rowptr[(size_t)r + 1] = m.h_rowptr[(size_t)r] + deg(perm[(size_t)r]);
    std::vector<int32_t> mcol((size_t)std::max<int64_t>(nnz, 1));
    const int nt = std::max(1, std::min(32, (int)std::thread::hardware_concurrency()));
    std::vector<std::thread> th;
    auto fill = [&](int t) {
        for (int64_t r = t; r < n; r += nt) {
            const int32_t o = perm[(size_t)r];
            int32_t* dst = mcol.data() + m.h_rowptr[(size_t)r];
            for (int32_t e = rp[(size_t)o]; e < rp[(size_t)o + 1]; ++e) *dst++ = inv[(size_t)col[(size_t)e]];
        }
    };
    for (int t = 1; t < nt; ++t) th.emplace_back(fill, t);
    fill(0);
    for (auto& x : th) x.join();
    int rc;
    if ((rc = upload_vec(m.h_rowptr, &m.rowptr)) || (rc = upload_vec(mcol, &m.col)) ||
        (rc = upload_vec(perm, &m.perm)) || (rc = upload_vec(inv, &m.inv)))
        return rc;
    auto res = g_mcsr.emplace(g, std::move(m));
    *out = &res.first->second;
    return GN_OK;
}

static int multi_plan(gn_graph* g, int G, bool exact, int rpw, const MultiPlan** out) {
    std::lock_guard<std::mutex> lk(g_mplan_mu);
    auto key = std::make_tuple((const gn_graph*)g, G, exact ? 1 : 0, rpw);
    auto it = g_mplans.find(key);
    if (it != g_mplans.end()) {
        *out = &it->second;
        return GN_OK;
    }
    const int64_t n = g->n;
    const MultiCsr* mc = nullptr;
    if (int rc0 = multi_csr(g, &mc)) return rc0;
    // rows are multi ids, processed in that order
    const std::vector<int32_t>& rp = mc->h_rowptr;
    std::vector<int32_t> perm((size_t)n);
    for (int64_t i = 0; i < n; ++i) perm[(size_t)i] = (int32_t)i;
    const int nw = G * kMWarps;
    constexpr double kRowCost = 8.0;  // per-row share of the index fetch and the update, in gathers
    auto deg = [&](int32_t r) { return rp[(size_t)r + 1] - rp[(size_t)r]; };
    double total = 0.0;
    for (int64_t i = 0; i < n; ++i) total += (double)deg(perm[(size_t)i]) + kRowCost;
    const double share = total / nw;  // one warp's fair share
    // fast mode: rows longer than a warp's share (and 2048) are split over a
    // CTA; rows whose walk would outlast a team's share are split over a warp
    const double cta_min = std::max(2048.0, share), warp_min = std::max(2.0 * kMUDeep, share / rpw);
    std::vector<int32_t> split, wrows, trows;
    trows.reserve((size_t)n);
    for (int64_t i = 0; i < n; ++i) {
        const int32_t r = perm[(size_t)i];
        const double d = deg(r);
        (exact || d <= warp_min ? trows : (d <= cta_min ? wrows : split)).push_back(r);
    }
    std::vector<int32_t> regular = wrows;
    regular.insert(regular.end(), trows.begin(), trows.end());
    std::vector<double> load((size_t)G, 0.0);
    std::vector<std::vector<int32_t>> per_cta((size_t)G);
    for (int32_t r : split) {  // degree-descending already (hubs lead the relabel order)
        const int c = (int)(std::min_element(load.begin(), load.end()) - load.begin());
        per_cta[(size_t)c].push_back(r);
        load[(size_t)c] += (double)deg(r) + kRowCost;
    }
    std::vector<int4> hd;
    std::vector<int32_t> hb((size_t)G + 1, 0);
    for (int c = 0; c < G; ++c) {
        for (int32_t r : per_cta[(size_t)c]) hd.push_back(make_int4(r, rp[(size_t)r], deg(r), 0));
        hb[(size_t)c + 1] = (int32_t)hd.size();
    }
    // regular rows: CTA c gets (total / G - load[c]) of them, cut evenly over its warps
    std::vector<int4> rd;
    rd.reserve(regular.size());
    std::vector<double> pre(regular.size() + 1, 0.0);
    for (size_t i = 0; i < regular.size(); ++i) {
        const int32_t r = regular[i];
        rd.push_back(make_int4(r, rp[(size_t)r], deg(r), 0));
        pre[i + 1] = pre[i] + (double)deg(r) + kRowCost;
    }
    std::vector<double> bound((size_t)nw + 1, 0.0);  // target prefix cost at each warp boundary
    double acc = 0.0;
    const double reg_total = pre.back();
    double want_total = 0.0;
    for (int c = 0; c < G; ++c) want_total += std::max(0.0, total / G - load[(size_t)c]);
    for (int c = 0; c < G; ++c) {
        const double want = want_total > 0 ? std::max(0.0, total / G - load[(size_t)c]) * reg_total / want_total : 0.0;
        for (int w = 0; w < kMWarps; ++w) {
            acc += want / kMWarps;
            bound[(size_t)c * kMWarps + w + 1] = acc;
        }
    }
    std::vector<int32_t> wb((size_t)nw + 1, (int32_t)regular.size());
    wb[0] = 0;
    size_t i = 0;
    for (int w = 1; w < nw; ++w) {
        while (i < regular.size() && pre[i + 1] <= bound[(size_t)w]) ++i;
        wb[(size_t)w] = (int32_t)i;
    }
    std::vector<int32_t> wm((size_t)nw);
    for (int w = 0; w < nw; ++w)
        wm[(size_t)w] = std::min(std::max((int32_t)wrows.size(), wb[(size_t)w]), wb[(size_t)w + 1]);
    MultiPlan mp;
    int rc;
    if ((rc = upload_vec(rd, &mp.rdesc)) || (rc = upload_vec(wb, &mp.wbeg)) || (rc = upload_vec(wm, &mp.wmid)) ||
        (rc = upload_vec(hd, &mp.hdesc)) ||
        (rc = upload_vec(hb, &mp.hbeg)))
        return rc;
    auto res = g_mplans.emplace(key, mp);
    *out = &res.first->second;
    return GN_OK;
}

template <typename TS, typename TG, int MU>
static void* pick_kernel_mu(int T) {
    switch (T) {
        case 2: return (void*)k_gn_multi<TS, TG, 2, MU>;
        case 4: return (void*)k_gn_multi<TS, TG, 4, MU>;
        case 8: return (void*)k_gn_multi<TS, TG, 8, MU>;
        case 16: return (void*)k_gn_multi<TS, TG, 16, MU>;
        default: return (void*)k_gn_multi<TS, TG, 32, MU>;
    }
}

template <typename TS, typename TG>
static void* pick_kernel(int T, int mu) {
    return mu == kMUDeep ? pick_kernel_mu<TS, TG, kMUDeep>(T) : pick_kernel_mu<TS, TG, kMUShort>(T);
}

// stream-ordered scratch owned by one call
struct MultiBufs {
    std::vector<void*> p;
    cudaStream_t s = nullptr;
    ~MultiBufs() {
        for (void* q : p) cudaFreeAsync(q, s);
    }
    template <typename Q>
    cudaError_t get(Q** out, size_t bytes) {
        cudaError_t e = cudaMallocAsync((void**)out, std::max<size_t>(bytes, 16), s);
        if (e == cudaSuccess) p.push_back((void*)*out);
        return e;
    }
};

static int blocks_of(int64_t n) { return (int)std::max<int64_t>(1, (n + 255) / 256); }

template <typename TS, typename TG>
static int multi_typed(gn_graph* g, int B, const double* x0, const double* gammas, int iters, double final_gamma,
                       uint32_t flags, double* x_out, double* step_inf, int64_t* fallbacks, int* iters_run,
                       int* status, int* fail_iter, gn_run_stats* stats) {
    const int64_t n = g->n;
    const int64_t launches0 = gn_launch_count();
    constexpr int S = Pack<TG>::S;
    int Bp = 2 * S;  // teams of at least 2 lanes (one-lane teams would need 16 index registers per chunk)
    while (Bp < B) Bp *= 2;
    const int T = Bp / S;
    CallCtx ctx;
    int rc = ctx.open(g->device);
    if (rc) return rc;
    cudaStream_t s = ctx.s;
    cudaEvent_t ev[4];
    for (auto& e : ev) GN_CUDA(cudaEventCreate(&e));
    struct EvGuard {
        cudaEvent_t* e;
        ~EvGuard() { for (int i = 0; i < 4; ++i) cudaEventDestroy(e[i]); }
    } evg{ev};
    GN_CUDA(cudaEventRecord(ev[0], s));

    MultiBufs ws;
    ws.s = s;
    const size_t nn = (size_t)std::max<int64_t>(n, 1);
    TS *xa, *v;
    TG* ya;
    double *xin, *gam, *out64;
    unsigned long long* sinf;
    unsigned int* fb;
    int *bad, *run, *skip, *chk;
    unsigned int* barrier;
    GN_CUDA(ws.get(&xa, 2 * sizeof(TS) * nn * Bp));
    GN_CUDA(ws.get(&ya, 2 * sizeof(TG) * nn * Bp));
    GN_CUDA(ws.get(&v, sizeof(TS) * nn));

    const bool dev_io = (flags & GN_DEVICE_IO) != 0;
    if (dev_io) xin = const_cast<double*>(x0);
    else GN_CUDA(ws.get(&xin, 8 * nn * B));
    GN_CUDA(ws.get(&gam, 8 * (size_t)iters));
    GN_CUDA(ws.get(&sinf, 8 * (size_t)iters * B));
    GN_CUDA(ws.get(&fb, 4 * (size_t)iters * B));
    GN_CUDA(ws.get(&bad, 4 * (size_t)iters * B));
    GN_CUDA(ws.get(&run, 4 * (size_t)B));
    GN_CUDA(ws.get(&skip, 4 * (size_t)B));
    GN_CUDA(ws.get(&chk, 8 * (size_t)B));
    GN_CUDA(ws.get(&barrier, 4));
    if (dev_io) out64 = x_out;
    else GN_CUDA(ws.get(&out64, 8 * nn * B));
    GN_CUDA(cudaMemsetAsync(sinf, 0, 8 * (size_t)iters * B, s));
    GN_CUDA(cudaMemsetAsync(fb, 0, 4 * (size_t)iters * B, s));
    GN_CUDA(cudaMemsetAsync(bad, 0, 4 * (size_t)iters * B, s));
    GN_CUDA(cudaMemsetAsync(run, 0, 4 * (size_t)B, s));
    GN_CUDA(cudaMemsetAsync(chk, 0, 8 * (size_t)B, s));
    GN_CUDA(cudaMemsetAsync(barrier, 0, 4, s));
    GN_CUDA(cudaMemcpyAsync(gam, gammas, 8 * (size_t)iters, cudaMemcpyHostToDevice, s));
    if (n > 0 && !dev_io) GN_CUDA(cudaMemcpyAsync(xin, x0, 8 * (size_t)n * B, cudaMemcpyHostToDevice, s));
    int64_t h2d = 8 * (int64_t)iters + (dev_io ? 0 : 8 * n * B), d2h = 0;

    // checks per start (dynamics.py:145-149)
    std::vector<int> hchk(2 * (size_t)B, 0), hskip((size_t)B, 0);
    if (!(flags & GN_NO_CHECK) && n > 0) {
        for (int b = 0; b < B; ++b) {
            if (int rc2 = enqueue_precheck(g, xin + (size_t)b * n, chk + 2 * b, s)) return rc2;
        }
        GN_CUDA(cudaMemcpyAsync(hchk.data(), chk, 8 * (size_t)B, cudaMemcpyDeviceToHost, s));
        GN_CUDA(cudaStreamSynchronize(s));
        d2h += 8 * B;
    }
    for (int b = 0; b < B; ++b) {
        status[b] = hchk[2 * (size_t)b] ? GN_ERR_NEGATIVE : (hchk[2 * (size_t)b + 1] ? GN_ERR_NOT_NORMALIZABLE : GN_OK);
        hskip[(size_t)b] = status[b] != GN_OK;
        if (fail_iter) fail_iter[b] = -1;
    }
    GN_CUDA(cudaMemcpyAsync(skip, hskip.data(), 4 * (size_t)B, cudaMemcpyHostToDevice, s));
    const MultiCsr* mc = nullptr;
    {
        std::lock_guard<std::mutex> lk(g_mplan_mu);
        if ((rc = multi_csr(g, &mc))) return rc;
    }
    if (n > 0) {
        k_multi_weights<TS><<<blocks_of(n), 256, 0, s>>>(n, g->w64, mc->perm, v);
        GN_LAUNCHED();
        k_multi_prepare<TS, TG><<<blocks_of(n * Bp), 256, 0, s>>>(n, B, Bp, xin, mc->perm, v, xa, ya);
        GN_LAUNCHED();
    }

    void* kern = pick_kernel<TS, TG>(T, multi_mu(g));
    int maxb = 1;
    if ((rc = coresident_blocks(kern, kMThreads, 0, g->device, &maxb))) return rc;
    if (maxb < 1) return fail(GN_ERR_CUDA, "multi-start kernel cannot be resident");
    const int64_t rows_per_cta = (int64_t)kMWarps * (32 / T);
    int grid = (int)std::min<int64_t>(maxb, std::max<int64_t>(1, (n + rows_per_cta - 1) / rows_per_cta));
    if (g->grid_override > 0) grid = std::min(maxb, g->grid_override);
    const MultiPlan* plan = nullptr;
    if ((rc = multi_plan(g, grid, (flags & GN_EXACT) != 0, 32 / T, &plan))) return rc;

    MultiArgs<TS, TG> a;
    memset(&a, 0, sizeof(a));
    a.n = n;
    a.B = B;
    a.Bp = Bp;
    a.col = mc->col;
    a.rdesc = plan->rdesc;
    a.wbeg = plan->wbeg;
    a.wmid = plan->wmid;
    a.hdesc = plan->hdesc;
    a.hbeg = plan->hbeg;
    a.v = v;
    a.x[0] = xa;
    a.x[1] = xa + nn * Bp;
    a.yg[0] = ya;
    a.yg[1] = ya + nn * Bp;
    a.gammas = gam;
    a.iters = iters;
    a.final_gamma = final_gamma;
    a.early_exit = (flags & GN_EARLY_EXIT) ? 1 : 0;
    a.sinf = sinf;
    a.fb = fb;
    a.bad = bad;
    a.run = run;
    a.skip = skip;
    a.barrier = barrier;
    void* args[] = {&a};
    GN_CUDA(cudaEventRecord(ev[1], s));
    if (n > 0 && iters > 0) {
        GN_CUDA(cudaLaunchCooperativeKernel(kern, dim3(grid), dim3(kMThreads), args, 0, s));
        GN_LAUNCHED();
    }
    GN_CUDA(cudaEventRecord(ev[2], s));
    std::vector<int> hrun((size_t)B);
    std::vector<unsigned long long> hsinf((size_t)iters * B);
    std::vector<unsigned int> hfb((size_t)iters * B);
    std::vector<int> hbad((size_t)iters * B);
    GN_CUDA(cudaMemcpyAsync(hrun.data(), run, 4 * (size_t)B, cudaMemcpyDeviceToHost, s));
    GN_CUDA(cudaMemcpyAsync(hsinf.data(), sinf, 8 * hsinf.size(), cudaMemcpyDeviceToHost, s));
    GN_CUDA(cudaMemcpyAsync(hfb.data(), fb, 4 * hfb.size(), cudaMemcpyDeviceToHost, s));
    GN_CUDA(cudaMemcpyAsync(hbad.data(), bad, 4 * hbad.size(), cudaMemcpyDeviceToHost, s));
    d2h += 4 * B + 16 * (int64_t)iters * B;
    if (x_out && n > 0) {
        k_multi_finalize<TS><<<blocks_of(n * B), 256, 0, s>>>(n, B, Bp, a.x[0], a.x[1], run, mc->inv, out64,
                                                             (flags & GN_NO_CLIP) ? 0 : 1);
        GN_LAUNCHED();
        if (!dev_io) {
            GN_CUDA(cudaMemcpyAsync(x_out, out64, 8 * (size_t)n * B, cudaMemcpyDeviceToHost, s));
            d2h += 8 * n * B;
        }
    }
    GN_CUDA(cudaEventRecord(ev[3], s));
    GN_CUDA(cudaStreamSynchronize(s));
    int first_bad = GN_OK;
    for (int b = 0; b < B; ++b) {
        const int ran = n > 0 ? hrun[(size_t)b] : (hskip[(size_t)b] ? 0 : iters);
        int stop_bad = -1;
        for (int k = 0; k < ran; ++k) {
            const size_t at = (size_t)k * B + b;
            if (step_inf) {
                const unsigned long long bits = hsinf[at];
                double d;
                memcpy(&d, &bits, 8);
                step_inf[(size_t)b * iters + k] = d;
            }
            if (fallbacks) fallbacks[(size_t)b * iters + k] = (int64_t)hfb[at];
            if (stop_bad < 0 && hbad[at]) stop_bad = k;
        }
        if (iters_run) iters_run[b] = ran;
        if (stop_bad >= 0 && !(flags & GN_NONFINITE_OK)) {
            status[b] = GN_ERR_NONFINITE;
            if (fail_iter) fail_iter[b] = stop_bad;
        }
        if (status[b] != GN_OK && first_bad == GN_OK) first_bad = status[b];
    }
    if (stats) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev[1], ev[2]);
        stats->loop_ms = ms;
        cudaEventElapsedTime(&ms, ev[0], ev[3]);
        stats->total_ms = ms;
        stats->launches = gn_launch_count() - launches0;
        stats->grid_blocks = grid;
        stats->block_threads = kMThreads;
        stats->h2d_bytes = h2d;
        stats->d2h_bytes = d2h;
    }
    if (first_bad != GN_OK) return fail(first_bad, "some starts stopped (see status)");
    return GN_OK;
}

}  // namespace gn

using namespace gn;

extern "C" int gn_multi_run(gn_graph* g, int num_starts, const double* x0, const double* gammas, int iters,
                            double final_gamma, uint32_t flags, double* x_out, double* step_inf, int64_t* fallbacks,
                            int* iters_run, int* status, int* fail_iter, gn_run_stats* stats) {
    GN_NVTX("gn_multi_run");
    if (!g || !x0 || !status || (iters > 0 && !gammas)) return fail(GN_ERR_ARG, "null argument");
    if (num_starts < 1 || num_starts > kMaxStarts) return fail(GN_ERR_ARG, "num_starts must be in [1, 64]");
    if (iters < 0) return fail(GN_ERR_ARG, "iters must be >= 0");
    switch (g->dtype) {
        case GN_F64:
            return multi_typed<double, double>(g, num_starts, x0, gammas, iters, final_gamma, flags, x_out, step_inf,
                                               fallbacks, iters_run, status, fail_iter, stats);
        case GN_F32:
            return multi_typed<double, float>(g, num_starts, x0, gammas, iters, final_gamma, flags, x_out, step_inf,
                                              fallbacks, iters_run, status, fail_iter, stats);
        default:
            return multi_typed<float, float>(g, num_starts, x0, gammas, iters, final_gamma, flags, x_out, step_inf,
                                             fallbacks, iters_run, status, fail_iter, stats);
    }
}
