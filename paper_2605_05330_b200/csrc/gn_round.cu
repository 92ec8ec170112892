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

// Row scans, warp-hybrid: a warp takes 32 consecutive rows; a row of at most
// kShortRow entries is scanned by its own lane (16 loads in flight per
// batch), a longer one by the whole warp (coalesced 32-entry chunks,
// ballot), so neither dense rows (C2: degree 510) nor hubs (R-MAT: degree
// > 10^5) leave one thread walking a long row one load at a time.
constexpr int kShortRow = 1024;

// any neighbour j of row i (entries [beg, end)) with pred(j); one lane.  The
// predicates of a batch are all evaluated (no short circuit) so their loads
// overlap.
template <typename Pred>
__device__ __forceinline__ bool lane_any(const int32_t* __restrict__ col, int32_t beg, int32_t end, Pred pred) {
    constexpr int U = 16;
    int32_t p = beg;
    for (; p + U <= end; p += U) {
        int32_t j[U];
#pragma unroll
        for (int u = 0; u < U; ++u) j[u] = col[p + u];
        bool h = false;
#pragma unroll
        for (int u = 0; u < U; ++u) h |= pred(j[u]);
        if (h) return true;
    }
    bool h = false;
    for (; p < end; ++p) h |= pred(col[p]);
    return h;
}

// the same over the whole warp (all lanes call it with the same row)
template <typename Pred>
__device__ __forceinline__ bool warp_any(const int32_t* __restrict__ col, int32_t beg, int32_t end, Pred pred) {
    const int lane = threadIdx.x & 31;
    for (int32_t base = beg; base < end; base += 32) {
        const int32_t p = base + lane;
        const bool h = p < end && pred(col[p]);
        if (__any_sync(0xffffffffu, h)) return true;
    }
    return false;
}

// For every row i in [0, n) with need(i): res(i) = any neighbour j with
// pred(i, j); visit(i, res) is then called by the lane that owns row i.
// Warps stride over chunks of 32 rows.
template <typename Need, typename Pred, typename Visit>
__device__ __forceinline__ void rows_any(int64_t n, const int32_t* __restrict__ rowptr,
                                         const int32_t* __restrict__ col, int64_t warp0, int64_t nwarps, Need need,
                                         Pred pred, Visit visit) {
    const int lane = threadIdx.x & 31;
    for (int64_t r0 = warp0 * 32; r0 < n; r0 += nwarps * 32) {
        const int64_t i = r0 + lane;
        const bool valid = i < n && need(i);
        const int32_t beg = valid ? rowptr[i] : 0, end = valid ? rowptr[i + 1] : 0;
        const bool lng = end - beg > kShortRow;
        bool res = false;
        if (valid && !lng) res = lane_any(col, beg, end, [&](int32_t j) { return pred(i, j); });
        unsigned m = __ballot_sync(0xffffffffu, lng);
        while (m) {
            const int l = __ffs(m) - 1;
            m &= m - 1;
            const int64_t il = r0 + l;
            const int32_t bl = __shfl_sync(0xffffffffu, beg, l), el = __shfl_sync(0xffffffffu, end, l);
            const bool r = warp_any(col, bl, el, [&](int32_t j) { return pred(il, j); });
            if (lane == l) res = r;
        }
        if (valid) visit(i, res);
    }
}

__device__ __forceinline__ int64_t gwarp() { return (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; }
__device__ __forceinline__ int64_t nwarp() { return ((int64_t)gridDim.x * blockDim.x) >> 5; }

__global__ void k_conflicts(int64_t n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                            const uint8_t* __restrict__ sel, uint8_t* __restrict__ conf) {
    // conf_i = sel_i and a selected neighbour (the rows the repair can change)
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        conf[i] = 0;  // (rows_any gives row i to this same thread)
    rows_any(
        n, rowptr, col, gwarp(), nwarp(), [&](int64_t i) { return sel[i] != 0; },
        [&](int64_t, int32_t j) { return sel[j] != 0; }, [&](int64_t i, bool r) { conf[i] = r ? 1 : 0; });
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
    const int64_t w0 = gwarp(), nw = nwarp();
    const int lane = threadIdx.x & 31;
    volatile uint8_t* vsel = sel;
    volatile uint8_t* vcand = cand;
    volatile uint8_t* vjoin = join;
    unsigned int bar = 0;
    // candidates: unselected and not dominated by the repaired set
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        cand[i] = 0;  // (rows_any gives row i to this same thread)
        join[i] = 0;
    }
    rows_any(
        n, rowptr, col, w0, nw, [&](int64_t i) { return sel[i] == 0; },
        [&](int64_t, int32_t j) { return sel[j] != 0; }, [&](int64_t i, bool dom) { cand[i] = dom ? 0 : 1; });
    grid_barrier(barrier, (++bar) * gridDim.x);
    for (int r = 0;; ++r) {
        int* live_ctr = counters + (r & 1);
        int local = 0;
        // a live candidate joins iff no live candidate neighbour has higher priority
        rows_any(
            n, rowptr, col, w0, nw, [&](int64_t i) { return vcand[i] != 0; },
            [&](int64_t i, int32_t j) { return vcand[j] && higher(w[j], j, w[i], (int)i); },
            [&](int64_t i, bool beaten) {
                ++local;
                vjoin[i] = beaten ? 0 : 1;
            });
        if (local) atomicAdd(live_ctr, local);
        grid_barrier(barrier, (++bar) * gridDim.x);
        if (*(volatile int*)live_ctr == 0) break;
        if (w0 == 0 && lane == 0) counters[(r + 1) & 1] = 0;
        // joined rows: select, and retire the neighbours (short rows by their
        // lane, long rows by the warp)
        for (int64_t r0 = w0 * 32; r0 < n; r0 += nw * 32) {
            const int64_t i = r0 + lane;
            const bool jn = i < n && vjoin[i];
            const int32_t beg = jn ? rowptr[i] : 0, end = jn ? rowptr[i + 1] : 0;
            if (jn) {
                vsel[i] = 1;
                vcand[i] = 0;
                vjoin[i] = 0;
                if (end - beg <= kShortRow)
                    for (int32_t p = beg; p < end; ++p) vcand[col[p]] = 0;
            }
            unsigned m = __ballot_sync(0xffffffffu, jn && end - beg > kShortRow);
            while (m) {
                const int l = __ffs(m) - 1;
                m &= m - 1;
                const int32_t bl = __shfl_sync(0xffffffffu, beg, l), el = __shfl_sync(0xffffffffu, end, l);
                for (int32_t p = bl + lane; p < el; p += 32) vcand[col[p]] = 0;
            }
        }
        grid_barrier(barrier, (++bar) * gridDim.x);
    }
}

// independence / maximality (graph.py:134-156)
__global__ void k_check(int64_t n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                        const uint8_t* __restrict__ sel, int* __restrict__ flags) {
    rows_any(
        n, rowptr, col, gwarp(), nwarp(), [&](int64_t) { return true; },
        [&](int64_t, int32_t j) { return sel[j] != 0; },
        [&](int64_t i, bool hit) {
            if (sel[i]) {
                if (hit) atomicOr(&flags[0], 1);  // not independent
            } else if (!hit) {
                atomicOr(&flags[1], 1);  // undominated vertex: not maximal
            }
        });
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

// one level d of the pairwise tree (all nodes in parallel); levels run from
// the deepest possible (for count = n) up to the root, whose value goes to out
__global__ void k_pairwise_level(const double* __restrict__ a, const int* __restrict__ count_p, int d,
                                 double* __restrict__ cur, const double* __restrict__ below, double* __restrict__ out) {
    const int64_t count = *count_p;
    const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= (int64_t(1) << d)) return;
    int64_t s, l;
    if (!pw_node(count, d, b, &s, &l)) return;
    const double v = l <= 128 ? pw_leaf(a + s, l) : __dadd_rn(below[2 * b], below[2 * b + 1]);
    cur[b] = v;
    if (d == 0) out[0] = v;
}

// deepest level the pairwise tree of up to n values can have
static int pw_depth(int64_t n) {
    int D = 0;
    for (int64_t l = n; l > 128; l = l - (l / 2 - (l / 2) % 8)) ++D;
    return D;
}

static int blocks_for(int64_t n) { return (int)std::max<int64_t>(1, (n + kRoundThreads - 1) / kRoundThreads); }

// Device scratch of one rounding, reused by the rounds of a batch.
struct RoundScratch {
    uint8_t *conf = nullptr, *cand = nullptr, *join = nullptr;
    int32_t* list = nullptr;
    int *dm = nullptr, *counters = nullptr;
    unsigned int* barrier = nullptr;
    double *mw = nullptr, *scratch = nullptr;
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    int64_t half = 0;
    cudaStream_t s = nullptr;
    int open(gn_graph* g, cudaStream_t st) {
        s = st;
        const int64_t n = g->n;
        const size_t nb = (size_t)std::max<int64_t>(n, 1);
        thrust::counting_iterator<int32_t> ids(0);
        size_t t1 = 0, t2 = 0;
        GN_CUDA(cub::DeviceSelect::Flagged(nullptr, t1, ids, conf, list, dm, (int)n, s));
        GN_CUDA(cub::DeviceSelect::Flagged(nullptr, t2, g->w64, conf, (double*)nullptr, (int*)nullptr, (int)n, s));
        tmp_bytes = std::max<size_t>(std::max(t1, t2), 16);
        // scratch for two pairwise levels: 2 * 2^D with 2^D <= 2 * ceil(n/64) + 2
        half = 2 * ((int64_t)nb / 64 + 2);
        GN_CUDA(cudaMallocAsync((void**)&conf, nb, s));
        GN_CUDA(cudaMallocAsync((void**)&cand, nb, s));
        GN_CUDA(cudaMallocAsync((void**)&join, nb, s));
        GN_CUDA(cudaMallocAsync((void**)&list, 4 * nb, s));
        GN_CUDA(cudaMallocAsync((void**)&dm, sizeof(int), s));
        GN_CUDA(cudaMallocAsync((void**)&counters, 2 * sizeof(int), s));
        GN_CUDA(cudaMallocAsync((void**)&barrier, sizeof(unsigned int), s));
        GN_CUDA(cudaMallocAsync((void**)&mw, 8 * nb, s));
        GN_CUDA(cudaMallocAsync((void**)&scratch, 8 * 2 * (size_t)half, s));
        GN_CUDA(cudaMallocAsync(&tmp, tmp_bytes, s));
        return GN_OK;
    }
    ~RoundScratch() {
        void* ptrs[] = {conf, cand, join, list, dm, counters, barrier, mw, scratch, tmp};
        for (void* p : ptrs)
            if (p) cudaFreeAsync(p, s);
    }
};

// Enqueue flags (independent, maximal), member count and the pairwise member
// weight of the 0/1 mask dsel into out[0..1], cnt[0], wout[0] (device).
static int enqueue_check(gn_graph* g, RoundScratch& R, const uint8_t* dsel, int* out, int* cnt, double* wout) {
    cudaStream_t s = R.s;
    const int64_t n = g->n;
    GN_CUDA(cudaMemsetAsync(out, 0, 2 * sizeof(int), s));
    GN_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int), s));
    if (n > 0) {
        k_check<<<blocks_for(n), kRoundThreads, 0, s>>>(n, g->rowptr, g->col, dsel, out);
        GN_LAUNCHED();
        size_t tb = R.tmp_bytes;
        GN_CUDA(cub::DeviceSelect::Flagged(R.tmp, tb, g->w64, dsel, R.mw, cnt, (int)n, s));
        note_launch();
    }
    // count <= n is on the device: levels below the real tree find no nodes
    const int D = pw_depth(n);
    if ((int64_t(1) << D) > R.half) return fail(GN_ERR_ARG, "pairwise scratch too small");
    for (int d = D; d >= 0; --d) {
        const int64_t nodes = int64_t(1) << d;
        k_pairwise_level<<<(int)((nodes + 255) / 256), 256, 0, s>>>(R.mw, cnt, d, R.scratch + (d & 1) * R.half,
                                                                   R.scratch + ((d + 1) & 1) * R.half, wout);
        GN_LAUNCHED();
    }
    return GN_OK;
}

// Enqueue round_to_mis of the device state dx into the mask sel (device).
template <typename TI>
static int enqueue_round(gn_graph* g, RoundScratch& R, const TI* dx, uint8_t* sel) {
    cudaStream_t s = R.s;
    const int64_t n = g->n;
    if (n == 0) return GN_OK;
    GN_CUDA(cudaMemsetAsync(R.dm, 0, sizeof(int), s));
    GN_CUDA(cudaMemsetAsync(R.counters, 0, 2 * sizeof(int), s));
    GN_CUDA(cudaMemsetAsync(R.barrier, 0, sizeof(unsigned int), s));
    k_threshold<TI><<<blocks_for(n), kRoundThreads, 0, s>>>(n, dx, sel);
    GN_LAUNCHED();
    k_conflicts<<<blocks_for(n), kRoundThreads, 0, s>>>(n, g->rowptr, g->col, sel, R.conf);
    GN_LAUNCHED();
    thrust::counting_iterator<int32_t> ids(0);
    size_t tb = R.tmp_bytes;
    GN_CUDA(cub::DeviceSelect::Flagged(R.tmp, tb, ids, R.conf, R.list, R.dm, (int)n, s));
    note_launch();
    k_repair<<<1, 32, 0, s>>>(R.list, R.dm, g->rowptr, g->col, g->w64, sel);
    GN_LAUNCHED();
    int maxb = 1, rc;
    if ((rc = coresident_blocks((const void*)k_greedy, kRoundThreads, 0, g->device, &maxb))) return rc;
    int grid = (int)std::min<int64_t>(maxb, blocks_for(n));
    int64_t nn = n;
    const int32_t* rp = g->rowptr;
    const int32_t* cc = g->col;
    const double* ww = g->w64;
    void* args[] = {&nn, &rp, &cc, &ww, &sel, &R.cand, &R.join, &R.counters, &R.barrier};
    GN_CUDA(cudaLaunchCooperativeKernel((const void*)k_greedy, dim3(grid), dim3(kRoundThreads), args, 0, s));
    GN_LAUNCHED();
    return GN_OK;
}

// B roundings (states x[b], host or device fp64) with one synchronisation.
static int round_batch(gn_graph* g, int B, const double* x, bool dev_x, uint8_t* selected, double* weight,
                       int* independent, int* maximal, int64_t* count, int64_t* members = nullptr) {
    CallCtx ctx;
    int rc = ctx.open(g->device);
    if (rc) return rc;
    cudaStream_t s = ctx.s;
    const int64_t n = g->n;
    const size_t nb = (size_t)std::max<int64_t>(n, 1);
    RoundScratch R;
    if ((rc = R.open(g, s))) return rc;
    uint8_t* sel = nullptr;
    double *dx = nullptr, *dw = nullptr;
    int* dflags = nullptr;
    GN_CUDA(cudaMallocAsync((void**)&sel, nb * B, s));
    GN_CUDA(cudaMallocAsync((void**)&dw, 8 * (size_t)B, s));
    GN_CUDA(cudaMallocAsync((void**)&dflags, 3 * sizeof(int) * (size_t)B, s));
    if (!dev_x) {
        GN_CUDA(cudaMallocAsync((void**)&dx, 8 * nb * B, s));
        if (n > 0) GN_CUDA(cudaMemcpyAsync(dx, x, 8 * (size_t)n * B, cudaMemcpyHostToDevice, s));
    }
    const double* xs = dev_x ? x : dx;
    for (int b = 0; b < B && rc == GN_OK; ++b) {
        rc = enqueue_round<double>(g, R, xs + (size_t)b * n, sel + nb * b);
        if (rc == GN_OK) rc = enqueue_check(g, R, sel + nb * b, dflags + 3 * b, dflags + 3 * b + 2, dw + b);
    }
    // the member list of a single rounding, compacted on the device (B == 1)
    int64_t *dmem = nullptr, *dmcnt = nullptr;
    void* mtmp = nullptr;
    if (members && rc == GN_OK && n > 0) {
        size_t tb = 0;
        thrust::counting_iterator<int64_t> ids(0);
        GN_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, ids, sel, dmem, dmcnt, (int)n, s));
        GN_CUDA(cudaMallocAsync(&mtmp, std::max<size_t>(tb, 16), s));
        GN_CUDA(cudaMallocAsync((void**)&dmem, 8 * nb, s));
        GN_CUDA(cudaMallocAsync((void**)&dmcnt, 8, s));
        GN_CUDA(cub::DeviceSelect::Flagged(mtmp, tb, ids, sel, dmem, dmcnt, (int)n, s));
        note_launch();
    }
    std::vector<int> hf(3 * (size_t)B);
    if (rc == GN_OK) {
        cudaMemcpyAsync(hf.data(), dflags, sizeof(int) * hf.size(), cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(weight, dw, 8 * (size_t)B, cudaMemcpyDeviceToHost, s);
        if (selected && n > 0)
            for (int b = 0; b < B; ++b)
                cudaMemcpyAsync(selected + (size_t)n * b, sel + nb * b, (size_t)n, cudaMemcpyDeviceToHost, s);
    }
    cudaError_t e = cudaSuccess;
    if (dmem) {
        // the count decides how many ids come back: one extra synchronisation
        int64_t hcnt = 0;
        cudaMemcpyAsync(&hcnt, dmcnt, 8, cudaMemcpyDeviceToHost, s);
        e = cudaStreamSynchronize(s);
        if (e == cudaSuccess && hcnt > 0)
            cudaMemcpyAsync(members, dmem, 8 * (size_t)hcnt, cudaMemcpyDeviceToHost, s);
    }
    void* ptrs[] = {sel, dx, dw, dflags, dmem, dmcnt, mtmp};
    for (void* p : ptrs)
        if (p) cudaFreeAsync(p, s);
    cudaError_t e2 = cudaStreamSynchronize(s);
    if (e == cudaSuccess) e = e2;
    if (rc != GN_OK) return rc;
    if (e != cudaSuccess) return cuda_fail(e, "round sync", __FILE__, __LINE__);
    for (int b = 0; b < B; ++b) {
        independent[b] = hf[3 * (size_t)b] == 0;
        maximal[b] = hf[3 * (size_t)b] == 0 && hf[3 * (size_t)b + 1] == 0;
        if (count) count[b] = hf[3 * (size_t)b + 2];
    }
    return GN_OK;
}

}  // namespace gn

using namespace gn;

extern "C" {

int gn_round(gn_graph* g, const void* x, uint32_t flags, uint8_t* selected, double* weight, int* independent,
             int* maximal, int64_t* count) {
    GN_NVTX("gn_round");
    if (!g) return fail(GN_ERR_ARG, "null graph");
    if (g->n > 0 && !x) return fail(GN_ERR_ARG, "null state");
    return round_batch(g, 1, (const double*)x, (flags & GN_DEVICE_IO) != 0, selected, weight, independent, maximal,
                       count);
}

int gn_round_members(gn_graph* g, const void* x, uint32_t flags, int64_t* members, double* weight, int* independent,
                     int* maximal, int64_t* count) {
    GN_NVTX("gn_round_members");
    if (!g) return fail(GN_ERR_ARG, "null graph");
    if (g->n > 0 && (!x || !members)) return fail(GN_ERR_ARG, "null state or member buffer");
    return round_batch(g, 1, (const double*)x, (flags & GN_DEVICE_IO) != 0, nullptr, weight, independent, maximal,
                       count, members);
}

int gn_round_many(gn_graph* g, int num_states, const void* x, uint32_t flags, uint8_t* selected, double* weight,
                  int* independent, int* maximal, int64_t* count) {
    GN_NVTX("gn_round_many");
    if (!g) return fail(GN_ERR_ARG, "null graph");
    if (num_states < 1 || !weight || !independent || !maximal) return fail(GN_ERR_ARG, "bad gn_round_many arguments");
    if (g->n > 0 && !x) return fail(GN_ERR_ARG, "null state");
    return round_batch(g, num_states, (const double*)x, (flags & GN_DEVICE_IO) != 0, selected, weight, independent,
                       maximal, count);
}

int gn_check_members(gn_graph* g, const uint8_t* mask, double* weight, int* independent, int* maximal,
                     int64_t* count) {
    GN_NVTX("gn_check_members");
    if (!g) return fail(GN_ERR_ARG, "null graph");
    CallCtx ctx;
    int rc = ctx.open(g->device);
    if (rc) return rc;
    cudaStream_t s = ctx.s;
    const size_t nb = (size_t)std::max<int64_t>(g->n, 1);
    RoundScratch R;
    if ((rc = R.open(g, s))) return rc;
    uint8_t* dsel = nullptr;
    int* dflags = nullptr;
    double* dw = nullptr;
    GN_CUDA(cudaMallocAsync((void**)&dsel, nb, s));
    GN_CUDA(cudaMallocAsync((void**)&dflags, 3 * sizeof(int), s));
    GN_CUDA(cudaMallocAsync((void**)&dw, 8, s));
    if (g->n > 0) GN_CUDA(cudaMemcpyAsync(dsel, mask, (size_t)g->n, cudaMemcpyHostToDevice, s));
    rc = enqueue_check(g, R, dsel, dflags, dflags + 2, dw);
    int hf[3] = {0, 0, 0};
    if (rc == GN_OK) {
        cudaMemcpyAsync(hf, dflags, sizeof(hf), cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(weight, dw, 8, cudaMemcpyDeviceToHost, s);
    }
    void* ptrs[] = {dsel, dflags, dw};
    for (void* p : ptrs) cudaFreeAsync(p, s);
    cudaError_t e = cudaStreamSynchronize(s);
    if (rc != GN_OK) return rc;
    if (e != cudaSuccess) return cuda_fail(e, "check sync", __FILE__, __LINE__);
    *independent = hf[0] == 0;
    *maximal = hf[0] == 0 && hf[1] == 0;
    if (count) *count = hf[2];
    return GN_OK;
}

}  // extern "C"
