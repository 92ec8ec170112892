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
// degree-sorted relabel order (gn_internal.cuh) so they have similar
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
#include <vector>

#include "gn_internal.cuh"

namespace gn {

constexpr int kMThreads = 512;
constexpr int kMWarps = kMThreads / 32;
constexpr int kMU = 16;       // gathers in flight per lane
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

template <typename TS, typename TG>
struct MultiArgs {
    int64_t n;
    int B, Bp;
    const int32_t* __restrict__ rowptr;  // original CSR
    const int32_t* __restrict__ col;
    const int32_t* __restrict__ order;   // rows in processing order (original ids)
    const int32_t* __restrict__ wbeg;    // [G * kMWarps + 1] ranges of `order` per warp
    const TS* __restrict__ v;            // original order
    const TS* __restrict__ w;
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

template <typename TS, typename TG, int T>
__global__ void __launch_bounds__(kMThreads, 1) k_gn_multi(MultiArgs<TS, TG> a) {
    using A = Arith<TS>;
    using P = Pack<TG>;
    using PT = typename P::T;
    constexpr int S = P::S;
    constexpr int NI = (kMU + T - 1) / T;  // index registers per lane
    __shared__ unsigned char s_frozen[kMaxStarts];
    __shared__ double s_mx[kMWarps][kMaxStarts];
    __shared__ unsigned int s_fb[kMWarps][kMaxStarts];
    __shared__ int s_bad[kMWarps][kMaxStarts];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tbase = lane & ~(T - 1), t = lane & (T - 1);
    const int B = a.B, Bp = a.Bp;
    if (threadIdx.x < kMaxStarts) s_frozen[threadIdx.x] = (threadIdx.x >= B || a.skip[threadIdx.x]) ? 1 : 0;
    __syncthreads();
    const int gw = blockIdx.x * kMWarps + warp;
    const int p0 = __ldg(a.wbeg + gw), p1 = __ldg(a.wbeg + gw + 1);
    unsigned int bar = 0;
    int k = 0;
    for (; k < a.iters; ++k) {
        const int cur = k & 1;
        const TS g = (TS)a.gammas[k];
        const TG* __restrict__ yg = a.yg[cur];
        double mx[S];
        unsigned int fbc[S];
        int bd[S];
#pragma unroll
        for (int s = 0; s < S; ++s) {
            mx[s] = 0.0;
            fbc[s] = 0u;
            bd[s] = 0;
        }
        for (int p = p0; p < p1; p += 32 / T) {
            const int pi = p + lane / T;
            const bool has = pi < p1;
            const int r = has ? __ldg(a.order + pi) : 0;
            const int rb = has ? __ldg(a.rowptr + r) : 0;
            const int deg = has ? __ldg(a.rowptr + r + 1) - rb : 0;
            const int dmax = (int)__reduce_max_sync(0xffffffffu, (unsigned)deg);
            const int dmin = (int)__reduce_min_sync(0xffffffffu, (unsigned)deg);
            TS acc[S];
#pragma unroll
            for (int s = 0; s < S; ++s) acc[s] = TS(0);
            int idx[NI];
#pragma unroll
            for (int i = 0; i < NI; ++i) {
                const int pos = i * T + t;
                idx[i] = (pos < kMU && pos < deg) ? __ldg(a.col + rb + pos) : 0;
            }
            const TG* __restrict__ ybase = yg + t * S;
            for (int q = 0; q < dmax; q += kMU) {
                int nidx[NI];
#pragma unroll
                for (int i = 0; i < NI; ++i) {
                    const int pos = q + kMU + i * T + t;
                    nidx[i] = (i * T + t < kMU && pos < deg) ? __ldg(a.col + rb + pos) : 0;
                }
                PT val[kMU];
                if (q + kMU <= dmin) {
#pragma unroll
                    for (int u = 0; u < kMU; ++u) {
                        const int j = __shfl_sync(0xffffffffu, idx[u / T], tbase + (u & (T - 1)));
                        val[u] = __ldg(reinterpret_cast<const PT*>(ybase + (size_t)j * Bp));
                    }
                } else {
#pragma unroll
                    for (int u = 0; u < kMU; ++u) {
                        const int j = __shfl_sync(0xffffffffu, idx[u / T], tbase + (u & (T - 1)));
                        if (q + u < deg) val[u] = __ldg(reinterpret_cast<const PT*>(ybase + (size_t)j * Bp));
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
            if (!has) continue;
            // dynamics.py:104-107 for this row and the lane's starts
            const TS vi = __ldg(a.v + r);
            const size_t off = (size_t)r * Bp + t * S;
            const TS* xc = a.x[cur] + off;
            TS* xn = a.x[cur ^ 1] + off;
            TG* yn = a.yg[cur ^ 1] + off;
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const int b = t * S + s;
                if (s_frozen[b]) continue;
                const TS xi = xc[s];
                const TS yi = A::mul(vi, xi);
                const TS d = A::add(yi, A::mul(g, acc[s]));
                const bool ok = (double)d > kSafeDiv;
                const TS o = ok ? A::div(yi, d) : TS(kFallback);
                xn[s] = o;
                yn[s] = (TG)A::mul(vi, o);
                TS df = A::sub(o, xi);  // dynamics.py:165
                df = df < TS(0) ? -df : df;
                const double diff = (double)df;
                if (!(diff <= mx[s])) mx[s] = diff;
                fbc[s] += ok ? 0u : 1u;
                if (!isfinite((double)o)) bd[s] = 1;
            }
        }
        // per start: fold the warp's teams (lanes with equal t), then the CTA
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
            double m = 0.0;
            unsigned int f = 0;
            int bb = 0;
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

// x0 [B][n] (fp64, original order) -> x[0], yg[0] ([n][Bp]); padding starts are 0
template <typename TS, typename TG>
__global__ void k_multi_prepare(int64_t n, int B, int Bp, const double* __restrict__ x0, const TS* __restrict__ v,
                                TS* __restrict__ x, TG* __restrict__ yg) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n * Bp) return;
    const int64_t r = e / Bp;
    const int b = (int)(e % Bp);
    const TS xi = b < B ? (TS)x0[(size_t)b * n + r] : TS(0);
    x[e] = xi;
    yg[e] = (TG)Arith<TS>::mul(v[r], xi);
}

// sqrt(w) and w in state precision, original order (graph.py:42, as k_init_state_weights)
template <typename TS>
__global__ void k_multi_weights(int64_t n, const double* __restrict__ w64, TS* __restrict__ v, TS* __restrict__ w) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) {
        v[i] = (TS)sqrt(w64[i]);
        w[i] = (TS)w64[i];
    }
}

// final state of start b (buffer run[b] & 1) -> x_out [B][n], np.clip(x, 0, 1)
template <typename TS>
__global__ void k_multi_finalize(int64_t n, int B, int Bp, const TS* __restrict__ x0, const TS* __restrict__ x1,
                                 const int* __restrict__ run, double* __restrict__ out, int clip) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n * B) return;
    const int b = (int)(e / n);
    const int64_t r = e % n;
    double xi = (double)((run[b] & 1) ? x1 : x0)[(size_t)r * Bp + b];
    if (clip) xi = xi < 0.0 ? 0.0 : (xi > 1.0 ? 1.0 : xi);  // dynamics.py:179
    out[e] = xi;
}

__global__ void k_multi_precheck(int64_t n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                                 const double* __restrict__ x, int* __restrict__ flags) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double xi = x[i];
    if (xi < 0.0) atomicOr(&flags[0], 1);  // dynamics.py:146
    double s = 0.0;
    for (int32_t p = rowptr[i]; p < rowptr[i + 1]; ++p) s = __dadd_rn(s, x[col[p]]);
    if (!(__dadd_rn(xi, s) > 0.0)) atomicOr(&flags[1], 1);  // dynamics.py:125
}

// ---- host plan: contiguous ranges of the relabel order per warp, balanced by gathers
struct MultiPlan {
    int32_t* wbeg = nullptr;
};
static std::mutex g_mplan_mu;
static std::map<std::pair<const gn_graph*, int>, MultiPlan> g_mplans;

void release_multi_plans(const gn_graph* g) {
    std::lock_guard<std::mutex> lk(g_mplan_mu);
    for (auto it = g_mplans.begin(); it != g_mplans.end();) {
        if (it->first.first == g) {
            cudaFree(it->second.wbeg);
            it = g_mplans.erase(it);
        } else {
            ++it;
        }
    }
}

static int multi_plan(gn_graph* g, int G, const int32_t** out) {
    std::lock_guard<std::mutex> lk(g_mplan_mu);
    auto key = std::make_pair((const gn_graph*)g, G);
    auto it = g_mplans.find(key);
    if (it != g_mplans.end()) {
        *out = it->second.wbeg;
        return GN_OK;
    }
    const int64_t n = g->n;
    std::vector<int32_t> rp((size_t)n + 1), perm((size_t)n);
    GN_CUDA(cudaMemcpy(rp.data(), g->rowptr, sizeof(int32_t) * rp.size(), cudaMemcpyDeviceToHost));
    if (n > 0) GN_CUDA(cudaMemcpy(perm.data(), g->perm, sizeof(int32_t) * perm.size(), cudaMemcpyDeviceToHost));
    const int nw = G * kMWarps;
    // cost of a row: its gathers plus a fixed per-row share (index fetch, update)
    constexpr double kRowCost = 8.0;
    double total = 0.0;
    for (int64_t i = 0; i < n; ++i) total += (double)(rp[(size_t)perm[(size_t)i] + 1] - rp[(size_t)perm[(size_t)i]]) + kRowCost;
    std::vector<int32_t> wb((size_t)nw + 1, (int32_t)n);
    wb[0] = 0;
    double acc = 0.0;
    int w = 1;
    for (int64_t i = 0; i < n && w < nw; ++i) {
        acc += (double)(rp[(size_t)perm[(size_t)i] + 1] - rp[(size_t)perm[(size_t)i]]) + kRowCost;
        while (w < nw && acc >= total * w / nw) wb[(size_t)w++] = (int32_t)(i + 1);
    }
    int32_t* d = nullptr;
    GN_CUDA(cudaMalloc(&d, sizeof(int32_t) * wb.size()));
    GN_CUDA(cudaMemcpy(d, wb.data(), sizeof(int32_t) * wb.size(), cudaMemcpyHostToDevice));
    g_mplans[key].wbeg = d;
    *out = d;
    return GN_OK;
}

template <typename TS, typename TG, int T>
static void* multi_kernel() {
    return (void*)k_gn_multi<TS, TG, T>;
}

template <typename TS, typename TG>
static void* pick_kernel(int T) {
    switch (T) {
        case 1: return multi_kernel<TS, TG, 1>();
        case 2: return multi_kernel<TS, TG, 2>();
        case 4: return multi_kernel<TS, TG, 4>();
        case 8: return multi_kernel<TS, TG, 8>();
        case 16: return multi_kernel<TS, TG, 16>();
        default: return multi_kernel<TS, TG, 32>();
    }
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
    int Bp = S;
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
    TS *xa, *v, *w;
    TG* ya;
    double *xin, *gam, *out64;
    unsigned long long* sinf;
    unsigned int* fb;
    int *bad, *run, *skip, *chk;
    unsigned int* barrier;
    GN_CUDA(ws.get(&xa, 2 * sizeof(TS) * nn * Bp));
    GN_CUDA(ws.get(&ya, 2 * sizeof(TG) * nn * Bp));
    GN_CUDA(ws.get(&v, sizeof(TS) * nn));
    GN_CUDA(ws.get(&w, sizeof(TS) * nn));
    GN_CUDA(ws.get(&xin, 8 * nn * B));
    GN_CUDA(ws.get(&gam, 8 * (size_t)iters));
    GN_CUDA(ws.get(&sinf, 8 * (size_t)iters * B));
    GN_CUDA(ws.get(&fb, 4 * (size_t)iters * B));
    GN_CUDA(ws.get(&bad, 4 * (size_t)iters * B));
    GN_CUDA(ws.get(&run, 4 * (size_t)B));
    GN_CUDA(ws.get(&skip, 4 * (size_t)B));
    GN_CUDA(ws.get(&chk, 8 * (size_t)B));
    GN_CUDA(ws.get(&barrier, 4));
    GN_CUDA(ws.get(&out64, 8 * nn * B));
    GN_CUDA(cudaMemsetAsync(sinf, 0, 8 * (size_t)iters * B, s));
    GN_CUDA(cudaMemsetAsync(fb, 0, 4 * (size_t)iters * B, s));
    GN_CUDA(cudaMemsetAsync(bad, 0, 4 * (size_t)iters * B, s));
    GN_CUDA(cudaMemsetAsync(run, 0, 4 * (size_t)B, s));
    GN_CUDA(cudaMemsetAsync(chk, 0, 8 * (size_t)B, s));
    GN_CUDA(cudaMemsetAsync(barrier, 0, 4, s));
    GN_CUDA(cudaMemcpyAsync(gam, gammas, 8 * (size_t)iters, cudaMemcpyHostToDevice, s));
    if (n > 0) GN_CUDA(cudaMemcpyAsync(xin, x0, 8 * (size_t)n * B, cudaMemcpyHostToDevice, s));
    int64_t h2d = 8 * (int64_t)iters + 8 * n * B, d2h = 0;

    // checks per start (dynamics.py:145-149)
    std::vector<int> hchk(2 * (size_t)B, 0), hskip((size_t)B, 0);
    if (!(flags & GN_NO_CHECK) && n > 0) {
        for (int b = 0; b < B; ++b) {
            k_multi_precheck<<<blocks_of(n), 256, 0, s>>>(n, g->rowptr, g->col, xin + (size_t)b * n, chk + 2 * b);
            GN_LAUNCHED();
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
    if (n > 0) {
        k_multi_weights<TS><<<blocks_of(n), 256, 0, s>>>(n, g->w64, v, w);
        GN_LAUNCHED();
        k_multi_prepare<TS, TG><<<blocks_of(n * Bp), 256, 0, s>>>(n, B, Bp, xin, v, xa, ya);
        GN_LAUNCHED();
    }

    void* kern = pick_kernel<TS, TG>(T);
    int maxb = 1;
    if ((rc = coresident_blocks(kern, kMThreads, 0, g->device, &maxb))) return rc;
    if (maxb < 1) return fail(GN_ERR_CUDA, "multi-start kernel cannot be resident");
    const int64_t rows_per_cta = (int64_t)kMWarps * (32 / T);
    int grid = (int)std::min<int64_t>(maxb, std::max<int64_t>(1, (n + rows_per_cta - 1) / rows_per_cta));
    if (g->grid_override > 0) grid = std::min(maxb, g->grid_override);
    const int32_t* wbeg = nullptr;
    if ((rc = multi_plan(g, grid, &wbeg))) return rc;

    MultiArgs<TS, TG> a;
    memset(&a, 0, sizeof(a));
    a.n = n;
    a.B = B;
    a.Bp = Bp;
    a.rowptr = g->rowptr;
    a.col = g->col;
    a.order = g->perm;
    a.wbeg = wbeg;
    a.v = v;
    a.w = w;
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
        k_multi_finalize<TS><<<blocks_of(n * B), 256, 0, s>>>(n, B, Bp, a.x[0], a.x[1], run, out64,
                                                             (flags & GN_NO_CLIP) ? 0 : 1);
        GN_LAUNCHED();
        GN_CUDA(cudaMemcpyAsync(x_out, out64, 8 * (size_t)n * B, cudaMemcpyDeviceToHost, s));
        d2h += 8 * n * B;
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
