// gn_loop.cu -- the GN iteration loop: one persistent, co-resident kernel that
// runs every step of run_wrgn on the device.
//
// Reference: dynamics.py:_step 102-108 (the update), run_wrgn 129-180 (loop,
// step_inf, fallbacks, non-finite stop, early exit, trace), energy 210-219 and
// weighted_mass 222-224 (fused here as per-iteration dot products).
//
// Per iteration k (one pass over the CSR adjacency):
//   s_i  = sum_{j in N(i)} y_j              gather-sum, degree-binned rows
//   d_i  = y_i + gamma_k * s_i              (separately rounded, no FMA)
//   x'_i = d_i > 1e-9 ? y_i / d_i : 0.5     counted fallback
//   y'_i = v_i * x'_i                       next gather source
// fused with the per-iteration reductions: max|x'-x| (bitwise: atomicMax on
// the IEEE bits of a non-negative double), the fallback count, the non-finite
// flag, and fixed-order fp64 block partials of w.x' (objective) and, in trace
// mode, y.y, y.s, w.x (the energy terms of the pre-step state).  A grid
// barrier separates iterations; block 0 folds the partials in block order, so
// every reduction is deterministic run to run.
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "gn_internal.cuh"

namespace gn {

template <typename T>
struct LoopArgs {
    int64_t n;
    const int32_t* __restrict__ rowptr;
    const int32_t* __restrict__ col;
    const T* __restrict__ v;
    const T* __restrict__ w;
    const int32_t* __restrict__ rows;  // bin row list; nullptr = identity
    Bin bins[kMaxBins];
    int nbins;
    T* xs[2];
    T* ys[2];
    const double* __restrict__ gammas;
    int iters;
    double final_gamma;
    int early_exit;
    int stop_on_nonfinite;
    unsigned long long* step_bits;  // [iters]
    unsigned long long* fb;         // [iters]
    int* status;                    // [0] nonfinite flag [1] fail iter [2] iters_run
    double* dots;                   // [(iters+1)][4]: y.y, y.s, w.x (pre), w.x' (post)
    double* partials;               // [2][grid][4]
    unsigned int* barrier;
    T* x_hist;  // optional [iters][n]
};

struct Stats {
    double mx;
    unsigned int fbc;
    int nonfin;
    double acc[4];
};

template <typename T>
__device__ __forceinline__ T tabs(T v) { return v < T(0) ? -v : v; }

// The elementwise half of _step for one row whose neighbour sum is s.
template <typename T, bool TRACE>
__device__ __forceinline__ void update_row(const LoopArgs<T>& a, int row, T s, const T* __restrict__ x,
                                           const T* __restrict__ y, T* __restrict__ xo, T* __restrict__ yo,
                                           T g, int k, bool tail, Stats& st) {
    using A = Arith<T>;
    const T yi = y[row];
    const T xi = x[row];
    const double wi = (double)__ldg(a.w + row);
    if (TRACE) {
        st.acc[0] = __dadd_rn(st.acc[0], __dmul_rn((double)yi, (double)yi));
        st.acc[1] = __dadd_rn(st.acc[1], __dmul_rn((double)yi, (double)s));
        st.acc[2] = __dadd_rn(st.acc[2], __dmul_rn(wi, (double)xi));
    }
    if (tail) return;
    const T d = A::add(yi, A::mul(g, s));          // dynamics.py:105
    const bool ok = (double)d > kSafeDiv;           // dynamics.py:106
    const T o = ok ? A::div(yi, d) : T(kFallback);  // dynamics.py:107
    xo[row] = o;
    yo[row] = A::mul(__ldg(a.v + row), o);          // next y = v * x'
    const double diff = (double)tabs(A::sub(o, xi));  // dynamics.py:165
    if (!(diff <= st.mx)) st.mx = diff;
    st.fbc += ok ? 0u : 1u;
    if (!isfinite(o)) st.nonfin = 1;
    st.acc[3] = __dadd_rn(st.acc[3], __dmul_rn(wi, (double)o));  // w . x'
    if (a.x_hist) a.x_hist[(size_t)k * (size_t)a.n + (size_t)row] = o;
}

// Rows of one bin, G lanes per row (G in 1..32), 32/G rows per warp task.
// G == 1 with an in-order walk is the EXACT mode (scipy's sequential sum).
template <typename T, int G, bool TRACE>
__device__ __forceinline__ void group_bin(const LoopArgs<T>& a, const Bin& bin, const T* __restrict__ x,
                                          const T* __restrict__ y, T* __restrict__ xo, T* __restrict__ yo,
                                          T g, int k, bool tail, int lane, int gwarp, int nwarps, Stats& st) {
    using A = Arith<T>;
    constexpr int RPW = 32 / G;
    const int sub = lane / G, gl = lane % G;
    const int tasks = (bin.count + RPW - 1) / RPW;
    for (int t = gwarp; t < tasks; t += nwarps) {
        const int slot = t * RPW + sub;
        const bool valid = slot < bin.count;
        int row = 0, beg = 0, end = 0;
        if (valid) {
            row = a.rows ? __ldg(a.rows + bin.off + slot) : bin.off + slot;
            beg = __ldg(a.rowptr + row);
            end = __ldg(a.rowptr + row + 1);
        }
        T s = T(0);
        int p = beg + gl;
        for (; p + 3 * G < end; p += 4 * G) {
            const int j0 = __ldg(a.col + p), j1 = __ldg(a.col + p + G);
            const int j2 = __ldg(a.col + p + 2 * G), j3 = __ldg(a.col + p + 3 * G);
            const T y0 = y[j0], y1 = y[j1], y2 = y[j2], y3 = y[j3];
            s = A::add(s, y0);
            s = A::add(s, y1);
            s = A::add(s, y2);
            s = A::add(s, y3);
        }
        for (; p < end; p += G) s = A::add(s, y[__ldg(a.col + p)]);
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) s = A::add(s, __shfl_xor_sync(0xffffffffu, s, o));
        if (valid && gl == 0) update_row<T, TRACE>(a, row, s, x, y, xo, yo, g, k, tail, st);
    }
}

// Hub rows: one whole block per row, fixed-order block reduction.
template <typename T, bool TRACE>
__device__ __forceinline__ void block_bin(const LoopArgs<T>& a, const Bin& bin, const T* __restrict__ x,
                                          const T* __restrict__ y, T* __restrict__ xo, T* __restrict__ yo,
                                          T g, int k, bool tail, Stats& st, T* red) {
    using A = Arith<T>;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int r = blockIdx.x; r < bin.count; r += gridDim.x) {
        const int row = a.rows ? __ldg(a.rows + bin.off + r) : bin.off + r;
        const int beg = __ldg(a.rowptr + row), end = __ldg(a.rowptr + row + 1);
        T s = T(0);
        for (int p = beg + threadIdx.x; p < end; p += blockDim.x) s = A::add(s, y[__ldg(a.col + p)]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s = A::add(s, __shfl_xor_sync(0xffffffffu, s, o));
        if (lane == 0) red[warp] = s;
        __syncthreads();
        if (threadIdx.x == 0) {
            T tot = T(0);
            for (int q = 0; q < nw; ++q) tot = A::add(tot, red[q]);
            update_row<T, TRACE>(a, row, tot, x, y, xo, yo, g, k, tail, st);
        }
        __syncthreads();
    }
}

template <typename T, bool TRACE>
__device__ void pass(const LoopArgs<T>& a, int k, bool tail, Stats& st, T* red) {
    const int cur = k & 1;
    const T* x = a.xs[cur];
    const T* y = a.ys[cur];
    T* xo = a.xs[cur ^ 1];
    T* yo = a.ys[cur ^ 1];
    const T g = tail ? T(0) : (T)a.gammas[k];
    const int lane = threadIdx.x & 31;
    const int gwarp = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int nwarps = gridDim.x * (blockDim.x >> 5);
    for (int b = 0; b < a.nbins; ++b) {
        const Bin bin = a.bins[b];
        switch (bin.G) {
            case 0: block_bin<T, TRACE>(a, bin, x, y, xo, yo, g, k, tail, st, red); break;
            case 1: group_bin<T, 1, TRACE>(a, bin, x, y, xo, yo, g, k, tail, lane, gwarp, nwarps, st); break;
            case 2: group_bin<T, 2, TRACE>(a, bin, x, y, xo, yo, g, k, tail, lane, gwarp, nwarps, st); break;
            case 4: group_bin<T, 4, TRACE>(a, bin, x, y, xo, yo, g, k, tail, lane, gwarp, nwarps, st); break;
            case 8: group_bin<T, 8, TRACE>(a, bin, x, y, xo, yo, g, k, tail, lane, gwarp, nwarps, st); break;
            case 16: group_bin<T, 16, TRACE>(a, bin, x, y, xo, yo, g, k, tail, lane, gwarp, nwarps, st); break;
            default: group_bin<T, 32, TRACE>(a, bin, x, y, xo, yo, g, k, tail, lane, gwarp, nwarps, st); break;
        }
    }
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Block-level fold of the per-thread stats; thread 0 publishes.
template <bool TRACE>
__device__ void publish(const Stats& st0, int k, bool tail, double* __restrict__ partials_cur,
                        unsigned long long* step_bits, unsigned long long* fb, int* status,
                        double (*s_acc)[4], double* s_mx, unsigned int* s_fb, int* s_nf) {
    Stats st = st0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        double m = __shfl_xor_sync(0xffffffffu, st.mx, o);
        if (!(m <= st.mx)) st.mx = m;
        st.fbc += __shfl_xor_sync(0xffffffffu, st.fbc, o);
        st.nonfin |= __shfl_xor_sync(0xffffffffu, st.nonfin, o);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) st.acc[q] = warp_sum_d(st.acc[q]);
    if (lane == 0) {
        s_mx[warp] = st.mx;
        s_fb[warp] = st.fbc;
        s_nf[warp] = st.nonfin;
#pragma unroll
        for (int q = 0; q < 4; ++q) s_acc[warp][q] = st.acc[q];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double mx = 0.0, acc[4] = {0.0, 0.0, 0.0, 0.0};
        unsigned int f = 0;
        int nf = 0;
        for (int q = 0; q < nw; ++q) {
            if (!(s_mx[q] <= mx)) mx = s_mx[q];
            f += s_fb[q];
            nf |= s_nf[q];
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[c] = __dadd_rn(acc[c], s_acc[q][c]);
        }
        if (!tail) {
            if (mx != 0.0) atomicMax(step_bits + k, (unsigned long long)__double_as_longlong(mx));
            if (f) atomicAdd(fb + k, (unsigned long long)f);
            if (nf) atomicOr(status, 1);
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) partials_cur[blockIdx.x * 4 + c] = acc[c];
    }
}

// Block 0, warp 0: fold the block partials of pass k in block order.
__device__ void fold_partials(const double* __restrict__ partials_cur, int nblocks, double* __restrict__ out) {
    if (blockIdx.x != 0 || threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        double s = 0.0;
        for (int q = lane; q < nblocks; q += 32) s = __dadd_rn(s, __ldcg(partials_cur + q * 4 + c));
        s = warp_sum_d(s);
        if (lane == 0) out[c] = s;
    }
}

template <typename T, bool TRACE>
__global__ void __launch_bounds__(kLoopThreads) k_gn_loop(LoopArgs<T> a) {
    __shared__ double s_acc[kLoopThreads / 32][4];
    __shared__ double s_mx[kLoopThreads / 32];
    __shared__ unsigned int s_fb[kLoopThreads / 32];
    __shared__ int s_nf[kLoopThreads / 32];
    __shared__ T s_red[kLoopThreads / 32];
    unsigned int bar = 0;
    int k = 0, ran = 0;
    bool failed = false;
    for (k = 0; k < a.iters; ++k) {
        Stats st{0.0, 0u, 0, {0.0, 0.0, 0.0, 0.0}};
        pass<T, TRACE>(a, k, false, st, s_red);
        double* pc = a.partials + (size_t)(k & 1) * gridDim.x * 4;
        publish<TRACE>(st, k, false, pc, a.step_bits, a.fb, a.status, s_acc, s_mx, s_fb, s_nf);
        grid_barrier(a.barrier, (++bar) * gridDim.x);
        fold_partials(pc, gridDim.x, a.dots + (size_t)k * 4);
        ran = k + 1;
        const int nonfin = *(volatile int*)a.status;
        if (nonfin && a.stop_on_nonfinite) { failed = true; break; }
        if (a.early_exit && a.gammas[k] == a.final_gamma) {   // dynamics.py:177
            const double si = __longlong_as_double(*(volatile long long*)(a.step_bits + k));
            if (si < 1e-12) break;
        }
    }
    if (TRACE && !failed) {
        // energy terms of the final state (reference: energy(g, x_new, gamma))
        Stats st{0.0, 0u, 0, {0.0, 0.0, 0.0, 0.0}};
        pass<T, TRACE>(a, ran, true, st, s_red);
        double* pc = a.partials + (size_t)(ran & 1) * gridDim.x * 4;
        publish<TRACE>(st, ran, true, pc, a.step_bits, a.fb, a.status, s_acc, s_mx, s_fb, s_nf);
        grid_barrier(a.barrier, (++bar) * gridDim.x);
        fold_partials(pc, gridDim.x, a.dots + (size_t)ran * 4);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.status[1] = failed ? ran - 1 : -1;
        a.status[2] = ran;
    }
}

// x0 (fp64 or T) -> state buffers: x = (T)x0, y = v*x  (dynamics.py:104,145)
template <typename T, typename TI>
__global__ void k_prepare(int64_t n, const TI* __restrict__ x0, const T* __restrict__ v, T* __restrict__ x,
                          T* __restrict__ y) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) {
        T xi = (T)x0[i];
        x[i] = xi;
        y[i] = Arith<T>::mul(v[i], xi);
    }
}

template <typename TI>
__global__ void k_precheck_any(int64_t n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                               const TI* __restrict__ x, int* __restrict__ flags) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double xi = (double)x[i];
    if (xi < 0.0) atomicOr(&flags[0], 1);                 // dynamics.py:146
    double s = 0.0;
    for (int32_t p = rowptr[i]; p < rowptr[i + 1]; ++p) s = __dadd_rn(s, (double)x[col[p]]);
    if (!(__dadd_rn(xi, s) > 0.0)) atomicOr(&flags[1], 1);  // dynamics.py:125
}

// final state -> output (np.clip(x, 0, 1), dynamics.py:179)
template <typename T, typename TO>
__global__ void k_finalize(int64_t n, const T* __restrict__ x, TO* __restrict__ out, int clip) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) {
        T xi = x[i];
        if (clip) xi = xi < T(0) ? T(0) : (xi > T(1) ? T(1) : xi);
        out[i] = (TO)xi;
    }
}

template <typename T>
__global__ void k_hist_to_f64(int64_t total, const T* __restrict__ h, double* __restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < total) out[i] = (double)h[i];
}

static int blocks_for(int64_t n) { return (int)std::max<int64_t>(1, (n + 255) / 256); }

template <typename T>
static int run_typed(gn_graph* g, const void* x0, const double* gammas, int iters, double final_gamma,
                     uint32_t flags, void* x_out, double* step_inf, int64_t* fallbacks, double* mass,
                     double* energy, double* pre_energy, double* x_hist, int* iters_run, int* fail_iter,
                     gn_run_stats* stats) {
    const bool trace = (flags & GN_TRACE) != 0;
    const bool dev_io = (flags & GN_DEVICE_IO) != 0;
    const int64_t n = g->n;
    const size_t nb = (size_t)std::max<int64_t>(n, 1);
    const int64_t launches0 = gn_launch_count();
    CallCtx ctx;
    int rc = ctx.open(g->device);
    if (rc) return rc;
    cudaStream_t s = ctx.s;
    int64_t h2d = 0, d2h = 0;

    cudaEvent_t e0, e1, e2, e3;
    GN_CUDA(cudaEventCreate(&e0));
    GN_CUDA(cudaEventCreate(&e1));
    GN_CUDA(cudaEventCreate(&e2));
    GN_CUDA(cudaEventCreate(&e3));
    struct EvGuard {
        cudaEvent_t* e[4];
        ~EvGuard() { for (auto p : e) cudaEventDestroy(*p); }
    } evg{{&e0, &e1, &e2, &e3}};
    GN_CUDA(cudaEventRecord(e0, s));

    // ---- workspace
    void* kern = trace ? (void*)k_gn_loop<T, true> : (void*)k_gn_loop<T, false>;
    int maxb = 1;
    if ((rc = coresident_blocks(kern, kLoopThreads, 0, g->device, &maxb))) return rc;
    if (maxb < 1) return fail(GN_ERR_CUDA, "loop kernel cannot be resident");
    const Plan& plan = (flags & GN_EXACT) ? g->exact : g->fast;
    int64_t work = g->nnz + 8 * n;
    int grid = (int)std::min<int64_t>(maxb, std::max<int64_t>(1, (work + 32767) / 32768));
    if (g->grid_override > 0) grid = std::min(maxb, g->grid_override);

    struct Ws {
        T *x0 = nullptr, *x1 = nullptr, *y0 = nullptr, *y1 = nullptr, *hist = nullptr;
        double *xin = nullptr, *dots = nullptr, *part = nullptr, *out64 = nullptr, *hist64 = nullptr;
        unsigned long long *bits = nullptr, *fb = nullptr;
        int* status = nullptr;
        unsigned int* barrier = nullptr;
        int* chk = nullptr;
        cudaStream_t s;
        ~Ws() {
            void* ptrs[] = {x0, x1, y0, y1, hist, xin, dots, part, out64, hist64, bits, fb, status, barrier, chk};
            for (void* p : ptrs)
                if (p) cudaFreeAsync(p, s);
        }
    } ws;
    ws.s = s;
    const size_t es = sizeof(T);
    GN_CUDA(cudaMallocAsync((void**)&ws.x0, es * nb, s));
    GN_CUDA(cudaMallocAsync((void**)&ws.x1, es * nb, s));
    GN_CUDA(cudaMallocAsync((void**)&ws.y0, es * nb, s));
    GN_CUDA(cudaMallocAsync((void**)&ws.y1, es * nb, s));
    GN_CUDA(cudaMallocAsync((void**)&ws.bits, 8 * (size_t)iters, s));
    GN_CUDA(cudaMallocAsync((void**)&ws.fb, 8 * (size_t)iters, s));
    GN_CUDA(cudaMallocAsync((void**)&ws.dots, 8 * 4 * (size_t)(iters + 1), s));
    GN_CUDA(cudaMallocAsync((void**)&ws.part, 8 * 4 * 2 * (size_t)grid, s));
    GN_CUDA(cudaMallocAsync((void**)&ws.status, 4 * sizeof(int), s));
    GN_CUDA(cudaMallocAsync((void**)&ws.barrier, sizeof(unsigned int), s));
    GN_CUDA(cudaMallocAsync((void**)&ws.chk, 2 * sizeof(int), s));
    GN_CUDA(cudaMemsetAsync(ws.bits, 0, 8 * (size_t)iters, s));
    GN_CUDA(cudaMemsetAsync(ws.fb, 0, 8 * (size_t)iters, s));
    GN_CUDA(cudaMemsetAsync(ws.dots, 0, 8 * 4 * (size_t)(iters + 1), s));
    GN_CUDA(cudaMemsetAsync(ws.status, 0, 4 * sizeof(int), s));
    GN_CUDA(cudaMemsetAsync(ws.barrier, 0, sizeof(unsigned int), s));
    GN_CUDA(cudaMemsetAsync(ws.chk, 0, 2 * sizeof(int), s));
    if (x_hist) GN_CUDA(cudaMallocAsync((void**)&ws.hist, es * nb * (size_t)iters, s));

    // ---- x0 in, checks (dynamics.py:145-149)
    const bool check = !(flags & GN_NO_CHECK);
    if (dev_io) {
        if (n > 0) {
            if (check) {
                k_precheck_any<T><<<blocks_for(n), 256, 0, s>>>(n, g->rowptr, g->col, (const T*)x0, ws.chk);
                GN_LAUNCHED();
            }
            k_prepare<T, T><<<blocks_for(n), 256, 0, s>>>(n, (const T*)x0, (const T*)g->v, ws.x0, ws.y0);
            GN_LAUNCHED();
        }
    } else {
        GN_CUDA(cudaMallocAsync((void**)&ws.xin, 8 * nb, s));
        if (n > 0) {
            GN_CUDA(cudaMemcpyAsync(ws.xin, x0, 8 * (size_t)n, cudaMemcpyHostToDevice, s));
            h2d += 8 * n;
            if (check) {
                k_precheck_any<double><<<blocks_for(n), 256, 0, s>>>(n, g->rowptr, g->col, ws.xin, ws.chk);
                GN_LAUNCHED();
            }
            k_prepare<T, double><<<blocks_for(n), 256, 0, s>>>(n, ws.xin, (const T*)g->v, ws.x0, ws.y0);
            GN_LAUNCHED();
        }
    }
    if (check && n > 0) {
        int hchk[2] = {0, 0};
        GN_CUDA(cudaMemcpyAsync(hchk, ws.chk, sizeof(hchk), cudaMemcpyDeviceToHost, s));
        GN_CUDA(cudaStreamSynchronize(s));
        if (hchk[0]) return fail(GN_ERR_NEGATIVE, "state entries must be nonnegative");
        if (hchk[1]) return fail(GN_ERR_NOT_NORMALIZABLE, "initial state has a zero closed neighborhood sum");
    }
    double* dgam = nullptr;
    GN_CUDA(cudaMallocAsync((void**)&dgam, 8 * (size_t)iters, s));
    struct GamGuard {
        double* p;
        cudaStream_t s;
        ~GamGuard() { cudaFreeAsync(p, s); }
    } gg{dgam, s};
    GN_CUDA(cudaMemcpyAsync(dgam, gammas, 8 * (size_t)iters, cudaMemcpyHostToDevice, s));
    h2d += 8 * iters;

    // ---- the loop
    LoopArgs<T> a;
    memset(&a, 0, sizeof(a));
    a.n = n;
    a.rowptr = g->rowptr;
    a.col = g->col;
    a.v = (const T*)g->v;
    a.w = (const T*)g->w;
    a.rows = plan.rows;
    a.nbins = plan.nbins;
    for (int b = 0; b < plan.nbins; ++b) a.bins[b] = plan.bins[b];
    a.xs[0] = ws.x0;
    a.xs[1] = ws.x1;
    a.ys[0] = ws.y0;
    a.ys[1] = ws.y1;
    a.gammas = dgam;
    a.iters = iters;
    a.final_gamma = final_gamma;
    a.early_exit = (flags & GN_EARLY_EXIT) ? 1 : 0;
    a.stop_on_nonfinite = (flags & GN_NONFINITE_OK) ? 0 : 1;
    a.step_bits = ws.bits;
    a.fb = ws.fb;
    a.status = ws.status;
    a.dots = ws.dots;
    a.partials = ws.part;
    a.barrier = ws.barrier;
    a.x_hist = ws.hist;
    void* args[] = {&a};
    GN_CUDA(cudaEventRecord(e1, s));
    GN_CUDA(cudaLaunchCooperativeKernel(kern, dim3(grid), dim3(kLoopThreads), args, 0, s));
    GN_LAUNCHED();
    GN_CUDA(cudaEventRecord(e2, s));

    // ---- results back
    int hstatus[4];
    GN_CUDA(cudaMemcpyAsync(hstatus, ws.status, sizeof(hstatus), cudaMemcpyDeviceToHost, s));
    std::vector<unsigned long long> hbits((size_t)iters), hfb((size_t)iters);
    std::vector<double> hdots(4 * (size_t)(iters + 1));
    GN_CUDA(cudaMemcpyAsync(hbits.data(), ws.bits, 8 * (size_t)iters, cudaMemcpyDeviceToHost, s));
    GN_CUDA(cudaMemcpyAsync(hfb.data(), ws.fb, 8 * (size_t)iters, cudaMemcpyDeviceToHost, s));
    GN_CUDA(cudaMemcpyAsync(hdots.data(), ws.dots, 8 * 4 * (size_t)(iters + 1), cudaMemcpyDeviceToHost, s));
    d2h += 8 * 2 * iters + 8 * 4 * (iters + 1) + 16;
    GN_CUDA(cudaStreamSynchronize(s));
    const int ran = hstatus[2];
    const T* xfinal = (ran & 1) ? ws.x1 : ws.x0;
    const int clip = (flags & GN_NO_CLIP) ? 0 : 1;
    if (x_out && n > 0) {
        if (dev_io) {
            k_finalize<T, T><<<blocks_for(n), 256, 0, s>>>(n, xfinal, (T*)x_out, clip);
            GN_LAUNCHED();
        } else {
            GN_CUDA(cudaMallocAsync((void**)&ws.out64, 8 * nb, s));
            k_finalize<T, double><<<blocks_for(n), 256, 0, s>>>(n, xfinal, ws.out64, clip);
            GN_LAUNCHED();
            GN_CUDA(cudaMemcpyAsync(x_out, ws.out64, 8 * (size_t)n, cudaMemcpyDeviceToHost, s));
            d2h += 8 * n;
        }
    }
    if (x_hist && n > 0 && ran > 0) {
        const int64_t total = (int64_t)ran * n;
        GN_CUDA(cudaMallocAsync((void**)&ws.hist64, 8 * (size_t)total, s));
        k_hist_to_f64<T><<<blocks_for(total), 256, 0, s>>>(total, ws.hist, ws.hist64);
        GN_LAUNCHED();
        GN_CUDA(cudaMemcpyAsync(x_hist, ws.hist64, 8 * (size_t)total, cudaMemcpyDeviceToHost, s));
        d2h += 8 * total;
    }
    GN_CUDA(cudaEventRecord(e3, s));
    GN_CUDA(cudaStreamSynchronize(s));

    for (int k = 0; k < ran; ++k) {
        double si;
        memcpy(&si, &hbits[(size_t)k], 8);
        if (step_inf) step_inf[k] = si;
        if (fallbacks) fallbacks[k] = (int64_t)hfb[(size_t)k];
        const double* d0 = &hdots[(size_t)k * 4];
        const double* d1 = &hdots[(size_t)(k + 1) * 4];
        if (mass) mass[k] = d0[3];
        if (trace) {
            // dynamics.py:219, from the fused dot products of x_k and x_{k+1}
            if (pre_energy) pre_energy[k] = 0.5 * (d0[0] + gammas[k] * d0[1]) - d0[2];
            if (energy) energy[k] = 0.5 * (d1[0] + gammas[k] * d1[1]) - d1[2];
        }
    }
    if (iters_run) *iters_run = ran;
    if (fail_iter) *fail_iter = hstatus[1];
    if (stats) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e1, e2);
        stats->loop_ms = ms;
        cudaEventElapsedTime(&ms, e0, e3);
        stats->total_ms = ms;
        stats->launches = gn_launch_count() - launches0;
        stats->grid_blocks = grid;
        stats->block_threads = kLoopThreads;
        stats->h2d_bytes = h2d;
        stats->d2h_bytes = d2h;
    }
    if (hstatus[0] && !(flags & GN_NONFINITE_OK)) {
        char buf[64];
        snprintf(buf, sizeof(buf), "non-finite state at iteration %d", hstatus[1]);
        return fail(GN_ERR_NONFINITE, buf);
    }
    return GN_OK;
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
    if (g->dtype == GN_F64)
        return run_typed<double>(g, x0, gammas, iters, final_gamma, flags, x_out, step_inf, fallbacks, mass,
                                 energy, pre_energy, x_hist, iters_run, fail_iter, stats);
    return run_typed<float>(g, x0, gammas, iters, final_gamma, flags, x_out, step_inf, fallbacks, mass, energy,
                            pre_energy, x_hist, iters_run, fail_iter, stats);
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
