// gn_round.cu -- exact round_to_mis and the MisSolution checks on the device.
//
// Reference: dynamics.py:253-277 (round_to_mis), graph.py:127-186
// (is_independent, is_maximal_independent, set_weight, MisSolution).
//
//   1. threshold       sel_i = x_i >= 0.5                              (259)
//   2. repair          the reference walks u ascending and, per u, its
//                      selected neighbours t > u ascending: drop u at the
//                      first t with w_u <= w_t, else drop t      (262-272)
//      Only vertices with a selected neighbour (the conflict set) can change,
//      so the walk is replayed exactly over the compacted, ascending conflict
//      list by one warp (32 neighbours per ballot).  On converged states the
//      list is empty and the step costs one flag pass.
//   3. completion      greedy over (-w, i) == the lexicographically-first MIS
//                      of the undominated candidates under that priority.
//                      Parallel rounds (join iff no live candidate neighbour
//                      has higher priority) reproduce it exactly.   (273-276)
//   4. checks + weight independence / maximality flags, and numpy's pairwise
//                      fp64 sum of the member weights (bitwise w[idx].sum()).
#include <cuda_runtime.h>
#include <cub/device/device_select.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <vector>

#include "gn_internal.cuh"

namespace gn {

constexpr int kRoundThreads = 256;

template <typename TI>
__global__ void k_threshold(int64_t n, const TI* __restrict__ x, uint8_t* __restrict__ sel) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) sel[i] = (double)x[i] >= 0.5 ? 1 : 0;
}

__global__ void k_conflicts(int64_t n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                            const uint8_t* __restrict__ sel, uint8_t* __restrict__ conf) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint8_t c = 0;
    if (sel[i])
        for (int32_t p = rowptr[i]; p < rowptr[i + 1]; ++p)
            if (sel[col[p]]) { c = 1; break; }
    conf[i] = c;
}

// One warp replays the reference's sequential repair over the ascending
// conflict list (dynamics.py:262-272).
__global__ void k_repair(const int32_t* __restrict__ list, const int* __restrict__ count,
                         const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                         const double* __restrict__ w, uint8_t* sel) {
    const int lane = threadIdx.x;
    const int m = *count;
    for (int q = 0; q < m; ++q) {
        const int u = list[q];
        __syncwarp();
        if (!((volatile uint8_t*)sel)[u]) continue;
        const double wu = w[u];
        const int beg = rowptr[u], end = rowptr[u + 1];
        bool dropped_u = false;
        for (int base = beg; base < end && !dropped_u; base += 32) {
            const int p = base + lane;
            int t = -1;
            bool live = false;
            if (p < end) {
                t = col[p];
                live = t > u && ((volatile uint8_t*)sel)[t];
            }
            // first live neighbour that is at least as heavy stops the scan (ties drop u, since t > u)
            const unsigned stop = __ballot_sync(0xffffffffu, live && wu <= w[t]);
            const int first = stop ? __ffs(stop) - 1 : 32;
            if (live && lane < first) ((volatile uint8_t*)sel)[t] = 0;
            if (stop) dropped_u = true;
        }
        __syncwarp();
        if (dropped_u && lane == 0) ((volatile uint8_t*)sel)[u] = 0;
        __syncwarp();
    }
}

// priority of the greedy completion (dynamics.py:273): larger w first, then smaller index
__device__ __forceinline__ bool higher(double wa, int a, double wb, int b) {
    return wa > wb || (wa == wb && a < b);
}

// Greedy completion as priority rounds in one co-resident kernel.
__global__ void __launch_bounds__(kRoundThreads) k_greedy(int64_t n, const int32_t* __restrict__ rowptr,
                                                           const int32_t* __restrict__ col,
                                                           const double* __restrict__ w, uint8_t* sel,
                                                           uint8_t* cand, uint8_t* join, int* counters,
                                                           unsigned int* barrier) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    unsigned int bar = 0;
    // candidates: unselected and not dominated by the repaired set
    for (int64_t i = tid; i < n; i += stride) {
        uint8_t c = 0;
        if (!sel[i]) {
            c = 1;
            for (int32_t p = rowptr[i]; p < rowptr[i + 1]; ++p)
                if (sel[col[p]]) { c = 0; break; }
        }
        cand[i] = c;
        join[i] = 0;
    }
    grid_barrier(barrier, (++bar) * gridDim.x);
    for (int r = 0;; ++r) {
        int* live_ctr = counters + (r & 1);
        int local = 0;
        for (int64_t i = tid; i < n; i += stride) {
            if (!((volatile uint8_t*)cand)[i]) continue;
            ++local;
            const double wi = w[i];
            bool top = true;
            for (int32_t p = rowptr[i]; p < rowptr[i + 1] && top; ++p) {
                const int j = col[p];
                if (((volatile uint8_t*)cand)[j] && higher(w[j], j, wi, (int)i)) top = false;
            }
            join[i] = top ? 1 : 0;
        }
        if (local) atomicAdd(live_ctr, local);
        grid_barrier(barrier, (++bar) * gridDim.x);
        if (*(volatile int*)live_ctr == 0) break;
        if (tid == 0) counters[(r + 1) & 1] = 0;
        for (int64_t i = tid; i < n; i += stride) {
            if (!((volatile uint8_t*)join)[i]) continue;
            ((volatile uint8_t*)sel)[i] = 1;
            ((volatile uint8_t*)cand)[i] = 0;
            ((volatile uint8_t*)join)[i] = 0;
            for (int32_t p = rowptr[i]; p < rowptr[i + 1]; ++p) ((volatile uint8_t*)cand)[col[p]] = 0;
        }
        grid_barrier(barrier, (++bar) * gridDim.x);
    }
}

// independence / maximality (graph.py:134-156) + member count
__global__ void k_check(int64_t n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                        const uint8_t* __restrict__ sel, int* __restrict__ flags) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    bool hit = false;
    for (int32_t p = rowptr[i]; p < rowptr[i + 1]; ++p)
        if (sel[col[p]]) { hit = true; break; }
    if (sel[i]) {
        if (hit) atomicOr(&flags[0], 1);  // not independent
    } else if (!hit) {
        atomicOr(&flags[1], 1);  // undominated vertex: not maximal
    }
}

// numpy float64 pairwise sum (blocks <= 128, 8 accumulators, halving on
// multiples of 8), evaluated level by level from the deepest node upward.
__device__ double pw_leaf(const double* a, int64_t len) {
    if (len < 8) {
        double r = 0.0;
        for (int64_t i = 0; i < len; ++i) r = __dadd_rn(r, a[i]);
        return r;
    }
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i;
    for (i = 8; i < len - (len % 8); i += 8)
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < len; ++i) res = __dadd_rn(res, a[i]);
    return res;
}

__device__ __forceinline__ int64_t pw_split(int64_t len) {
    int64_t n2 = len / 2;
    return n2 - n2 % 8;
}

// node (d, b): follow the path bits of b from the root; false if an ancestor is a leaf
__device__ bool pw_node(int64_t count, int d, int64_t b, int64_t* start, int64_t* len) {
    int64_t s = 0, l = count;
    for (int lv = 0; lv < d; ++lv) {
        if (l <= 128) return false;
        const int64_t n2 = pw_split(l);
        if ((b >> (d - 1 - lv)) & 1) { s += n2; l -= n2; }
        else l = n2;
    }
    *start = s;
    *len = l;
    return true;
}

__global__ void k_pairwise(const double* __restrict__ a, const int* __restrict__ count_p, double* scratch,
                           int64_t scratch_len, double* __restrict__ out) {
    const int64_t count = *count_p;
    int D = 0;
    for (int64_t l = count; l > 128; l = l - pw_split(l)) ++D;
    if ((int64_t(1) << D) > scratch_len / 2) {  // cannot happen: scratch is sized from n
        if (threadIdx.x == 0) out[0] = __longlong_as_double(0x7ff8000000000000LL);
        return;
    }
    double* lv[2] = {scratch, scratch + (scratch_len / 2)};
    for (int d = D; d >= 0; --d) {
        double* cur = lv[d & 1];
        const double* below = lv[(d + 1) & 1];
        for (int64_t b = threadIdx.x; b < (int64_t(1) << d); b += blockDim.x) {
            int64_t s, l;
            if (!pw_node(count, d, b, &s, &l)) continue;
            cur[b] = l <= 128 ? pw_leaf(a + s, l) : __dadd_rn(below[2 * b], below[2 * b + 1]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) out[0] = lv[0][0];
}

static int blocks_for(int64_t n) { return (int)std::max<int64_t>(1, (n + kRoundThreads - 1) / kRoundThreads); }

// shared tail of gn_round and gn_check_members: flags, compaction, weight
static int check_and_weigh(gn_graph* g, CallCtx& ctx, uint8_t* dsel, double* weight, int* independent,
                           int* maximal, int64_t* count, uint8_t* sel_out) {
    cudaStream_t s = ctx.s;
    const int64_t n = g->n;
    const size_t nb = (size_t)std::max<int64_t>(n, 1);
    int* flags = nullptr;
    int* dcount = nullptr;
    double *mw = nullptr, *res = nullptr, *scratch = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    GN_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp_bytes, g->w64, dsel, (double*)nullptr, (int*)nullptr,
                                       (int)n, s));
    // scratch for two pairwise levels: 2 * 2^D with 2^D <= 2 * ceil(n/64) + 2
    const int64_t half = 2 * ((int64_t)nb / 64 + 2);
    GN_CUDA(cudaMallocAsync(&tmp, std::max<size_t>(tmp_bytes, 16), s));
    GN_CUDA(cudaMallocAsync((void**)&flags, 2 * sizeof(int), s));
    GN_CUDA(cudaMallocAsync((void**)&dcount, sizeof(int), s));
    GN_CUDA(cudaMallocAsync((void**)&mw, 8 * nb, s));
    GN_CUDA(cudaMallocAsync((void**)&res, 8, s));
    GN_CUDA(cudaMallocAsync((void**)&scratch, 8 * 2 * (size_t)half, s));
    GN_CUDA(cudaMemsetAsync(flags, 0, 2 * sizeof(int), s));
    GN_CUDA(cudaMemsetAsync(dcount, 0, sizeof(int), s));
    if (n > 0) {
        k_check<<<blocks_for(n), kRoundThreads, 0, s>>>(n, g->rowptr, g->col, dsel, flags);
        GN_LAUNCHED();
        GN_CUDA(cub::DeviceSelect::Flagged(tmp, tmp_bytes, g->w64, dsel, mw, dcount, (int)n, s));
        note_launch();
    }
    k_pairwise<<<1, 1024, 0, s>>>(mw, dcount, scratch, 2 * half, res);
    GN_LAUNCHED();
    int hflags[2];
    int hcount = 0;
    GN_CUDA(cudaMemcpyAsync(hflags, flags, sizeof(hflags), cudaMemcpyDeviceToHost, s));
    GN_CUDA(cudaMemcpyAsync(&hcount, dcount, sizeof(int), cudaMemcpyDeviceToHost, s));
    GN_CUDA(cudaMemcpyAsync(weight, res, sizeof(double), cudaMemcpyDeviceToHost, s));
    if (sel_out && n > 0) GN_CUDA(cudaMemcpyAsync(sel_out, dsel, (size_t)n, cudaMemcpyDeviceToHost, s));
    void* ptrs[] = {tmp, flags, dcount, mw, res, scratch};
    for (void* p : ptrs) cudaFreeAsync(p, s);
    GN_CUDA(cudaStreamSynchronize(s));
    *independent = hflags[0] == 0;
    *maximal = hflags[0] == 0 && hflags[1] == 0;
    if (count) *count = hcount;
    return GN_OK;
}

template <typename TI>
static int round_impl(gn_graph* g, CallCtx& ctx, const TI* dx, uint8_t* selected, double* weight,
                      int* independent, int* maximal, int64_t* count) {
    cudaStream_t s = ctx.s;
    const int64_t n = g->n;
    const size_t nb = (size_t)std::max<int64_t>(n, 1);
    uint8_t *sel = nullptr, *conf = nullptr, *cand = nullptr, *join = nullptr;
    int32_t* list = nullptr;
    int* dm = nullptr;
    int* counters = nullptr;
    unsigned int* barrier = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    thrust::counting_iterator<int32_t> ids(0);
    GN_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp_bytes, ids, conf, list, dm, (int)n, s));
    GN_CUDA(cudaMallocAsync((void**)&sel, nb, s));
    GN_CUDA(cudaMallocAsync((void**)&conf, nb, s));
    GN_CUDA(cudaMallocAsync((void**)&cand, nb, s));
    GN_CUDA(cudaMallocAsync((void**)&join, nb, s));
    GN_CUDA(cudaMallocAsync((void**)&list, 4 * nb, s));
    GN_CUDA(cudaMallocAsync((void**)&dm, sizeof(int), s));
    GN_CUDA(cudaMallocAsync((void**)&counters, 2 * sizeof(int), s));
    GN_CUDA(cudaMallocAsync((void**)&barrier, sizeof(unsigned int), s));
    GN_CUDA(cudaMallocAsync(&tmp, std::max<size_t>(tmp_bytes, 16), s));
    GN_CUDA(cudaMemsetAsync(dm, 0, sizeof(int), s));
    GN_CUDA(cudaMemsetAsync(counters, 0, 2 * sizeof(int), s));
    GN_CUDA(cudaMemsetAsync(barrier, 0, sizeof(unsigned int), s));
    int rc = GN_OK;
    if (n > 0) {
        k_threshold<TI><<<blocks_for(n), kRoundThreads, 0, s>>>(n, dx, sel);
        GN_LAUNCHED();
        k_conflicts<<<blocks_for(n), kRoundThreads, 0, s>>>(n, g->rowptr, g->col, sel, conf);
        GN_LAUNCHED();
        GN_CUDA(cub::DeviceSelect::Flagged(tmp, tmp_bytes, ids, conf, list, dm, (int)n, s));
        note_launch();
        k_repair<<<1, 32, 0, s>>>(list, dm, g->rowptr, g->col, g->w64, sel);
        GN_LAUNCHED();
        int maxb = 1;
        if ((rc = coresident_blocks((const void*)k_greedy, kRoundThreads, 0, g->device, &maxb))) return rc;
        int grid = (int)std::min<int64_t>(maxb, blocks_for(n));
        int64_t nn = n;
        const int32_t* rp = g->rowptr;
        const int32_t* cc = g->col;
        const double* ww = g->w64;
        void* args[] = {&nn, &rp, &cc, &ww, &sel, &cand, &join, &counters, &barrier};
        GN_CUDA(cudaLaunchCooperativeKernel((const void*)k_greedy, dim3(grid), dim3(kRoundThreads), args, 0, s));
        GN_LAUNCHED();
    }
    rc = check_and_weigh(g, ctx, sel, weight, independent, maximal, count, selected);
    void* ptrs[] = {sel, conf, cand, join, list, dm, counters, barrier, tmp};
    for (void* p : ptrs) cudaFreeAsync(p, s);
    cudaStreamSynchronize(s);
    return rc;
}

}  // namespace gn

using namespace gn;

extern "C" {

int gn_round(gn_graph* g, const void* x, uint32_t flags, uint8_t* selected, double* weight, int* independent,
             int* maximal, int64_t* count) {
    if (!g) return fail(GN_ERR_ARG, "null graph");
    if (g->n > 0 && !x) return fail(GN_ERR_ARG, "null state");
    CallCtx ctx;
    int rc = ctx.open(g->device);
    if (rc) return rc;
    if (flags & GN_DEVICE_IO)
        return round_impl<double>(g, ctx, (const double*)x, selected, weight, independent, maximal, count);
    double* dx = nullptr;
    const size_t nb = (size_t)std::max<int64_t>(g->n, 1);
    GN_CUDA(cudaMallocAsync((void**)&dx, 8 * nb, ctx.s));
    if (g->n > 0) GN_CUDA(cudaMemcpyAsync(dx, x, 8 * (size_t)g->n, cudaMemcpyHostToDevice, ctx.s));
    rc = round_impl<double>(g, ctx, dx, selected, weight, independent, maximal, count);
    cudaFreeAsync(dx, ctx.s);
    cudaStreamSynchronize(ctx.s);
    return rc;
}

int gn_check_members(gn_graph* g, const uint8_t* mask, double* weight, int* independent, int* maximal,
                     int64_t* count) {
    if (!g) return fail(GN_ERR_ARG, "null graph");
    CallCtx ctx;
    int rc = ctx.open(g->device);
    if (rc) return rc;
    uint8_t* dsel = nullptr;
    const size_t nb = (size_t)std::max<int64_t>(g->n, 1);
    GN_CUDA(cudaMallocAsync((void**)&dsel, nb, ctx.s));
    if (g->n > 0) GN_CUDA(cudaMemcpyAsync(dsel, mask, (size_t)g->n, cudaMemcpyHostToDevice, ctx.s));
    rc = check_and_weigh(g, ctx, dsel, weight, independent, maximal, count, nullptr);
    cudaFreeAsync(dsel, ctx.s);
    cudaStreamSynchronize(ctx.s);
    return rc;
}

}  // extern "C"
