// gn_batch.cu -- GN on batches of small independent graphs: one CTA per
// graph, the whole graph resident in shared memory for all iterations.
//
// Reference: the same run_wrgn (dynamics.py:129-180) run independently per
// graph -- exactly what solver.py would do graph by graph, and bitwise equal
// to running the packed block-diagonal graph (component independence,
// test_dynamics.py:90-104).  Used for BASELINE config C4 (1024 graphs of
// n = 2000 per GPU) and, through gn_run, for any single graph that fits
// (C1 and the test corpora): no grid barrier, no HBM traffic per iteration.
//
// Per CTA (graph b), once: local rows relabeled by degree (descending,
// stable), cut into groups of 32 rows (one per lane of a warp); neighbour
// lists (uint16 byte offsets of the neighbours' published values, the
// reference's neighbour order) stored
// position-major in pairs so a lane fetches positions p, p+1 with one 32-bit
// shared load and a warp's fetch is 128 contiguous bytes.  Each thread owns
// up to kRowsPerThread rows (dealt snake-wise over the degree order) whose
// x, v, w stay in registers for the whole run; only the published values yg live in shared memory (ping-pong).
// Per iteration: sequential per-row sums (the reference's order: bitwise),
// the update, and one block reduction (step_inf, fallbacks, non-finite,
// objective and the trace dots) whose single __syncthreads also publishes
// yg; every thread folds the 32 warp partials in the same order, so the
// early-exit decision is uniform without a second barrier.
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <vector>

#include "gn_internal.cuh"

namespace gn {

constexpr int kRowsPerThread = 4;
constexpr int kBatchThreads = 1024;

// Host-built packed layout of B graphs (see header comment).
struct BatchLayout {
    int64_t B = 0, n = 0;
    std::vector<int64_t> voff;      // [B+1] first vertex (original numbering)
    std::vector<int64_t> ioff;      // [B+1] first uint16 of graph b's index block
    std::vector<int32_t> goff;      // per group (all graphs): uint16 offset inside the graph's block
    std::vector<int64_t> gbase;     // [B+1] first group of graph b
    std::vector<uint16_t> idx;      // packed index blocks
    std::vector<uint16_t> deg;      // per local new row (all graphs, in voff order)
    std::vector<int32_t> lperm;     // per local new row: original local id
    int64_t max_idx = 0, max_n = 0; // largest graph: index uint16s, vertices
};

static int build_batch_layout(int64_t B, const int64_t* offsets, int64_t n, const int64_t* indptr,
                              const int32_t* indices, int gsz, BatchLayout& L) {
    L.B = B;
    L.n = n;
    L.voff.assign(offsets, offsets + B + 1);
    L.ioff.assign((size_t)B + 1, 0);
    L.gbase.assign((size_t)B + 1, 0);
    L.deg.assign((size_t)n, 0);
    L.lperm.assign((size_t)n, 0);
    for (int64_t b = 0; b < B; ++b) {
        const int64_t v0 = offsets[b], v1 = offsets[b + 1], nb = v1 - v0;
        if (nb < 0 || nb * gsz > 65535) return fail(GN_ERR_ARG, "batch graph too large for the resident kernel");
        std::vector<int32_t> order((size_t)nb);
        std::iota(order.begin(), order.end(), 0);
        auto dg = [&](int32_t l) { return indptr[v0 + l + 1] - indptr[v0 + l]; };
        std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t c) { return dg(a) > dg(c); });
        std::vector<int32_t> rank((size_t)nb);
        for (int64_t r = 0; r < nb; ++r) rank[(size_t)order[(size_t)r]] = (int32_t)r;
        const int64_t ng = (nb + 31) / 32;
        L.gbase[(size_t)b + 1] = L.gbase[(size_t)b] + ng;
        int64_t pos = 0;
        const int64_t first_group = (int64_t)L.goff.size();
        for (int64_t g = 0; g < ng; ++g) {
            int64_t len = 0;
            for (int64_t r = g * 32; r < std::min(nb, (g + 1) * 32); ++r) len = std::max<int64_t>(len, dg(order[(size_t)r]));
            len = (len + 1) & ~int64_t(1);
            L.goff.push_back((int32_t)pos);
            pos += len * 32;
        }
        if (pos > 65535 * 2) return fail(GN_ERR_ARG, "batch graph too dense for the resident kernel");
        L.ioff[(size_t)b + 1] = L.ioff[(size_t)b] + pos;
        L.max_idx = std::max(L.max_idx, pos);
        L.max_n = std::max(L.max_n, nb);
        const size_t base = L.idx.size();
        L.idx.resize(base + (size_t)pos, 0);
        for (int64_t r = 0; r < nb; ++r) {
            const int32_t o = order[(size_t)r];
            const int64_t g = r / 32, lane = r % 32;
            L.deg[(size_t)(v0 + r)] = (uint16_t)dg(o);
            L.lperm[(size_t)(v0 + r)] = o;
            const int64_t go = L.goff[(size_t)(first_group + g)];
            for (int64_t p = indptr[v0 + o]; p < indptr[v0 + o + 1]; ++p) {
                const int64_t q = p - indptr[v0 + o];
                const int64_t j = indices[p] - v0;
                if (j < 0 || j >= nb) return fail(GN_ERR_ARG, "batch graphs must not share edges");
                // byte offset of the neighbour's published value (fits: nb * gsz < 2^16)
                L.idx[base + (size_t)(go + (q / 2) * 64 + lane * 2 + (q % 2))] = (uint16_t)(rank[(size_t)j] * gsz);
            }
        }
    }
    return GN_OK;
}

}  // namespace gn

struct gn_batch {
    int64_t B = 0, n = 0;
    int dtype = GN_F64;
    int device = 0;
    int64_t max_idx = 0, max_n = 0, ngroups = 0;
    int64_t* voff = nullptr;
    int64_t* ioff = nullptr;
    int64_t* gbase = nullptr;
    int32_t* goff = nullptr;
    uint16_t* idx = nullptr;
    uint16_t* deg = nullptr;
    int32_t* lperm = nullptr;
    double* w64 = nullptr;  // original order
    // packed original CSR for the per-graph x0 checks
    int32_t* rowptr = nullptr;
    int32_t* col = nullptr;
    int32_t* gid = nullptr;  // vertex -> graph
    int64_t device_bytes = 0;
};

namespace gn {

template <typename TS, typename TG>
struct BatchArgs {
    int64_t B;
    const int64_t* __restrict__ voff;
    const int64_t* __restrict__ ioff;
    const int64_t* __restrict__ gbase;
    const int32_t* __restrict__ goff;
    const uint16_t* __restrict__ idx;
    const uint16_t* __restrict__ deg;
    const int32_t* __restrict__ lperm;
    const double* __restrict__ w64;
    const double* __restrict__ x0;  // original order
    double* x_out;                  // original order (raw; clipping applied by caller kernel)
    const double* __restrict__ gammas;
    int iters;
    double final_gamma;
    int early_exit;
    int stop_nonfinite;
    int trace;
    double* step_inf;  // [B][iters]
    double* fb;        // [B][iters]
    double* dots;      // [B][iters+1][4]
    int* ran;          // [B]
    int* bad;          // [B] first non-finite iteration or -1
    double* x_hist;    // optional [iters][n] (original order, packed)
    int64_t n_total;
    int smem_y_off;    // byte offset of yg ping-pong in dynamic smem
    int clip;          // np.clip(x, 0, 1) on the way out (dynamics.py:179)
};

__device__ __forceinline__ double bwarp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Row q of this thread.  Rows are degree-descending; a snake deal (t, then
// 2*blockDim-1-t, ...) gives every thread a long and a short row, so the
// per-iteration barrier does not wait for the threads holding the hubs.
__device__ __forceinline__ int own_row(int q) {
    const int t = (q & 1) ? (int)blockDim.x - 1 - (int)threadIdx.x : (int)threadIdx.x;
    return q * (int)blockDim.x + t;
}

// Per-thread row state (registers for the whole run).
template <typename TS>
struct OwnRows {
    TS x[kRowsPerThread], v[kRowsPerThread];
    double w[kRowsPerThread];
    int deg[kRowsPerThread], go[kRowsPerThread];  // original ids are re-read from lperm when needed
};

// One pass over the CTA's graph (tail: only the trace dots of the current
// state).  Returns the block totals (identical in every thread):
// tot = {y.y, y.s, w.x, w.x', max|dx|, fallbacks, non-finite}.
template <typename TS, typename TG, bool TRACE>
__device__ __forceinline__ void batch_pass(const BatchArgs<TS, TG>& a, OwnRows<TS>& R, const uint16_t* s_idx,
                                           TG* s_y, int nb, int cur, TS g, bool tail, int k, int64_t v0,
                                           double (*s_red)[kBatchThreads / 32][8], double (&tot)[7]) {
    using A = Arith<TS>;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const TG* yc = s_y + cur * nb;
    // neighbour ids are stored as byte offsets into the published values
    const char* ycb = reinterpret_cast<const char*>(yc);
    auto ldy = [ycb](uint32_t off) { return *reinterpret_cast<const TG*>(ycb + off); };
    TG* yn = s_y + (cur ^ 1) * nb;
    double mx = 0.0, acc[4] = {0.0, 0.0, 0.0, 0.0};
    unsigned int fbc = 0;
    int nf = 0;
#pragma unroll
    for (int q = 0; q < kRowsPerThread; ++q) {
        const int r = own_row(q);
        if (r >= nb) continue;
        // sequential neighbour sum in the reference's order; a 32-bit shared
        // load fetches positions p, p+1
        TS s = TS(0);
        const uint32_t* pi = reinterpret_cast<const uint32_t*>(s_idx + R.go[q]);
        const int d = R.deg[q];
        int p = 0;
        for (; p + 8 <= d; p += 8) {
            const uint32_t e0 = pi[(p / 2) * 32], e1 = pi[(p / 2 + 1) * 32];
            const uint32_t e2 = pi[(p / 2 + 2) * 32], e3 = pi[(p / 2 + 3) * 32];
            const TG y0 = ldy(e0 & 0xffff), y1 = ldy(e0 >> 16), y2 = ldy(e1 & 0xffff), y3 = ldy(e1 >> 16);
            const TG y4 = ldy(e2 & 0xffff), y5 = ldy(e2 >> 16), y6 = ldy(e3 & 0xffff), y7 = ldy(e3 >> 16);
            s = A::add(s, (TS)y0);
            s = A::add(s, (TS)y1);
            s = A::add(s, (TS)y2);
            s = A::add(s, (TS)y3);
            s = A::add(s, (TS)y4);
            s = A::add(s, (TS)y5);
            s = A::add(s, (TS)y6);
            s = A::add(s, (TS)y7);
        }
        for (; p < d; ++p) {
            const uint32_t e = pi[(p / 2) * 32];
            s = A::add(s, (TS)ldy((p & 1) ? (e >> 16) : (e & 0xffff)));
        }
        const TS yi = A::mul(R.v[q], R.x[q]);  // dynamics.py:104
        if (TRACE) {
            acc[0] = __dadd_rn(acc[0], __dmul_rn((double)yi, (double)yi));
            acc[1] = __dadd_rn(acc[1], __dmul_rn((double)yi, (double)s));
            acc[2] = __dadd_rn(acc[2], __dmul_rn(R.w[q], (double)R.x[q]));
        }
        if (tail) continue;
        const TS dd = A::add(yi, A::mul(g, s));          // dynamics.py:105
        const bool ok = (double)dd > kSafeDiv;            // dynamics.py:106
        const TS o = ok ? A::div(yi, dd) : TS(kFallback); // dynamics.py:107
        const TS dx = A::sub(o, R.x[q]);
        const double diff = (double)(dx < TS(0) ? -dx : dx);  // dynamics.py:165
        if (!(diff <= mx)) mx = diff;
        fbc += ok ? 0u : 1u;
        if (!isfinite((double)o)) nf = 1;
        acc[3] = __dadd_rn(acc[3], __dmul_rn(R.w[q], (double)o));
        R.x[q] = o;
        yn[r] = (TG)A::mul(R.v[q], o);
        if (a.x_hist) a.x_hist[(size_t)k * (size_t)a.n_total + (size_t)(v0 + a.lperm[v0 + r])] = (double)o;
    }
    // one block reduction; its barrier also publishes yn
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double m = __shfl_xor_sync(0xffffffffu, mx, o);
        if (!(m <= mx)) mx = m;
        fbc += __shfl_xor_sync(0xffffffffu, fbc, o);
        nf |= __shfl_xor_sync(0xffffffffu, nf, o);
    }
#pragma unroll
    for (int c = TRACE ? 0 : 3; c < 4; ++c) acc[c] = bwarp_sum(acc[c]);
    double* slot = s_red[k & 1][warp];
    if (lane == 0) {
        slot[0] = acc[0];
        slot[1] = acc[1];
        slot[2] = acc[2];
        slot[3] = acc[3];
        slot[4] = mx;
        slot[5] = (double)fbc;
        slot[6] = nf ? 1.0 : 0.0;
    }
    __syncthreads();  // also publishes yn
    // warp 0 folds the warp partials (fixed shuffle tree); only it holds tot
    if (warp == 0) {
        const int nw = (int)(blockDim.x >> 5);
        const double* sl = s_red[k & 1][lane];
        double t[7];
#pragma unroll
        for (int c = 0; c < 7; ++c) t[c] = lane < nw ? sl[c] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
            for (int c = 0; c < 4; ++c) t[c] = __dadd_rn(t[c], __shfl_xor_sync(0xffffffffu, t[c], o));
            const double m = __shfl_xor_sync(0xffffffffu, t[4], o);
            if (!(m <= t[4])) t[4] = m;
            t[5] += __shfl_xor_sync(0xffffffffu, t[5], o);
            const double f = __shfl_xor_sync(0xffffffffu, t[6], o);
            if (f != 0.0) t[6] = 1.0;
        }
#pragma unroll
        for (int c = 0; c < 7; ++c) tot[c] = t[c];
    }
}

template <typename TS, typename TG, bool TRACE>
__global__ void __launch_bounds__(kBatchThreads, 1) k_gn_batch(BatchArgs<TS, TG> a) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ double s_red[2][kBatchThreads / 32][8];
    const int64_t b = blockIdx.x;
    const int64_t v0 = a.voff[b];
    const int nb = (int)(a.voff[b + 1] - v0);
    const int64_t i0 = a.ioff[b];
    const int nidx = (int)(a.ioff[b + 1] - i0);
    const int64_t g0 = a.gbase[b];
    uint16_t* s_idx = (uint16_t*)smem;
    TG* s_y = (TG*)(smem + a.smem_y_off);  // [2][nb]

    {  // the graph's index block into shared memory
        const uint32_t* src = reinterpret_cast<const uint32_t*>(a.idx + i0);
        uint32_t* dst = reinterpret_cast<uint32_t*>(s_idx);
        for (int t = threadIdx.x; t < nidx / 2; t += blockDim.x) dst[t] = __ldg(src + t);
    }
    OwnRows<TS> R;
#pragma unroll
    for (int q = 0; q < kRowsPerThread; ++q) {
        const int r = own_row(q);
        R.deg[q] = 0;
        R.x[q] = TS(0);
        R.v[q] = TS(0);
        R.w[q] = 0.0;
        R.go[q] = 0;
        if (r < nb) {
            const int o = a.lperm[v0 + r];
            R.deg[q] = a.deg[v0 + r];
            R.go[q] = a.goff[g0 + r / 32] + (r % 32) * 2;
            const double w = a.w64[v0 + o];
            R.w[q] = (double)(TS)w;
            R.v[q] = (TS)sqrt(w);  // graph.py:42
            R.x[q] = (TS)a.x0[v0 + o];
            s_y[r] = (TG)Arith<TS>::mul(R.v[q], R.x[q]);  // dynamics.py:104
        }
    }
    __syncthreads();

    double* out_si = a.step_inf + b * a.iters;
    double* out_fb = a.fb + b * a.iters;
    double* out_dots = a.dots + b * (int64_t)(a.iters + 1) * 4;
    __shared__ int s_stop;
    int ran = 0, bad = -1;  // bad: tracked by thread 0
    double tot[7];
    for (int k = 0; k < a.iters; ++k) {
        batch_pass<TS, TG, TRACE>(a, R, s_idx, s_y, nb, k & 1, (TS)a.gammas[k], false, k, v0, s_red, tot);
        ran = k + 1;
        if (threadIdx.x == 0) {
            out_si[k] = tot[4];
            out_fb[k] = tot[5];
#pragma unroll
            for (int c = 0; c < 4; ++c) out_dots[(size_t)k * 4 + c] = tot[c];
            if (tot[6] != 0.0 && bad < 0) bad = k;  // a non-finite state: reported, run continues
        }
        if (a.early_exit && a.gammas[k] == a.final_gamma) {  // dynamics.py:177
            if (threadIdx.x == 0) s_stop = tot[4] < 1e-12;
            __syncthreads();
            const int stop = s_stop;
            __syncthreads();
            if (stop) break;
        }
    }
    if (TRACE) {
        // energy terms of the final state (the reference's energy(g, x_new, gamma))
        batch_pass<TS, TG, TRACE>(a, R, s_idx, s_y, nb, ran & 1, TS(0), true, ran, v0, s_red, tot);
        if (threadIdx.x == 0)
#pragma unroll
            for (int c = 0; c < 4; ++c) out_dots[(size_t)ran * 4 + c] = tot[c];
    }
#pragma unroll
    for (int q = 0; q < kRowsPerThread; ++q) {
        const int r = own_row(q);
        if (r < nb) {
            double xo = (double)R.x[q];
            if (a.clip) xo = xo < 0.0 ? 0.0 : (xo > 1.0 ? 1.0 : xo);
            a.x_out[v0 + a.lperm[v0 + r]] = xo;
        }
    }
    if (threadIdx.x == 0) {
        a.ran[b] = ran;
        a.bad[b] = bad;
    }
}

// x0 checks per graph (dynamics.py:145-149): flags[2b] negative, [2b+1] zero closed sum
__global__ void k_precheck_batch(int64_t n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                                 const int32_t* __restrict__ gid, const double* __restrict__ x, int* __restrict__ flags) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double xi = x[i];
    const int b = gid[i];
    if (xi < 0.0) atomicOr(&flags[2 * b], 1);
    // with no negative entry in the graph (reported first) the closed sum is
    // > 0 iff some entry is > 0 and NaN iff some entry is NaN (whose own row
    // fails): only rows with x_i == 0 scan, up to their first positive neighbour
    if (xi != xi) {
        atomicOr(&flags[2 * b + 1], 1);
        return;
    }
    if (xi > 0.0) return;
    bool pos = false;
    for (int32_t p = rowptr[i]; p < rowptr[i + 1] && !pos; ++p) pos = x[col[p]] > 0.0;
    if (!pos) atomicOr(&flags[2 * b + 1], 1);
}

// Per-graph outputs in the caller's [B][iters] layout, made on the device so
// they copy straight into the caller's arrays: step_inf masked in place,
// fallback counts binary64 -> int64 in place, the mass column of the per-
// iteration dot products compacted.  Entries past a graph's last iteration
// (iters_run: the loop's count, or fail_iter + 1 after a non-finite stop) are 0.
__global__ void k_batch_outputs(int64_t B, int iters, const int* __restrict__ chk, const int* __restrict__ ran,
                                const int* __restrict__ bad, int stop_nonfinite, double* si, double* fb,
                                const double* __restrict__ dots, double* __restrict__ mass) {
    const int64_t total = B * iters;
    for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < total;
         o += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = o / iters;
        const int k = (int)(o - b * iters);
        int r = ran[b];
        if (stop_nonfinite && !chk[2 * b] && !chk[2 * b + 1] && bad[b] >= 0) r = bad[b] + 1;
        const bool live = k < r;
        si[o] = live ? si[o] : 0.0;
        const double f = fb[o];
        reinterpret_cast<int64_t*>(fb)[o] = live ? (int64_t)f : 0;
        if (mass) mass[o] = live ? dots[((size_t)b * (iters + 1) + k) * 4 + 3] : 0.0;
    }
}

static void free_batch(gn_batch* bt) {
    if (!bt) return;
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(bt->device);
    void* ptrs[] = {bt->voff, bt->ioff, bt->gbase, bt->goff, bt->idx, bt->deg, bt->lperm, bt->w64, bt->rowptr,
                    bt->col, bt->gid};
    for (void* p : ptrs) cudaFree(p);
    if (prev >= 0) cudaSetDevice(prev);
    delete bt;
}

int batch_create(int64_t B, const int64_t* offsets, int64_t n, const int64_t* indptr, const int32_t* indices,
                 const double* w, int dtype, int device, gn_batch** out) {
    *out = nullptr;
    if (B < 1 || n < 0 || !offsets) return fail(GN_ERR_ARG, "bad batch description");
    if (offsets[0] != 0 || offsets[B] != n) return fail(GN_ERR_ARG, "batch offsets must run from 0 to n");
    for (int64_t b = 0; b < B; ++b)
        if (offsets[b + 1] < offsets[b]) return fail(GN_ERR_ARG, "batch offsets must be nondecreasing");
    const int64_t nnz = n > 0 ? indptr[n] : 0;
    if (nnz >= (int64_t(1) << 31)) return fail(GN_ERR_ARG, "batch too large");
    BatchLayout L;
    int rc = build_batch_layout(B, offsets, n, indptr, indices, (int)gather_bytes(dtype), L);
    if (rc) return rc;
    if (L.max_n > (int64_t)kBatchThreads * kRowsPerThread)
        return fail(GN_ERR_ARG, "batch graph has more vertices than the resident kernel holds");
    gn_batch* bt = new gn_batch();
    bt->B = B;
    bt->n = n;
    bt->dtype = dtype;
    bt->device = device;
    bt->max_idx = L.max_idx;
    bt->max_n = L.max_n;
    bt->ngroups = (int64_t)L.goff.size();
    CallCtx ctx;
    if ((rc = ctx.open(device))) { delete bt; return rc; }
    std::vector<int32_t> rp((size_t)n + 1), gid((size_t)std::max<int64_t>(n, 1));
    for (int64_t i = 0; i <= n; ++i) rp[(size_t)i] = (int32_t)(n > 0 ? indptr[i] : 0);
    for (int64_t b = 0; b < B; ++b)
        for (int64_t v = offsets[b]; v < offsets[b + 1]; ++v) gid[(size_t)v] = (int32_t)b;
    int64_t bytes = 0;
    auto cleanup = [&](int code) { free_batch(bt); return code; };
#define GN_BUP(dst, src, count, type)                                                             \
    do {                                                                                          \
        size_t _b = sizeof(type) * (size_t)std::max<int64_t>((int64_t)(count), 1);                \
        cudaError_t _e = cudaMalloc((void**)&(dst), _b);                                          \
        if (_e != cudaSuccess) return cleanup(cuda_fail(_e, "cudaMalloc", __FILE__, __LINE__));   \
        bytes += (int64_t)_b;                                                                     \
        if ((count) > 0) {                                                                        \
            _e = cudaMemcpyAsync((dst), (src), sizeof(type) * (size_t)(count), cudaMemcpyHostToDevice, ctx.s); \
            if (_e != cudaSuccess) return cleanup(cuda_fail(_e, "cudaMemcpyAsync", __FILE__, __LINE__)); \
        }                                                                                         \
    } while (0)
    GN_BUP(bt->voff, L.voff.data(), B + 1, int64_t);
    GN_BUP(bt->ioff, L.ioff.data(), B + 1, int64_t);
    GN_BUP(bt->gbase, L.gbase.data(), B + 1, int64_t);
    GN_BUP(bt->goff, L.goff.data(), (int64_t)L.goff.size(), int32_t);
    GN_BUP(bt->idx, L.idx.data(), (int64_t)L.idx.size(), uint16_t);
    GN_BUP(bt->deg, L.deg.data(), n, uint16_t);
    GN_BUP(bt->lperm, L.lperm.data(), n, int32_t);
    GN_BUP(bt->w64, w, n, double);
    GN_BUP(bt->rowptr, rp.data(), n + 1, int32_t);
    GN_BUP(bt->col, indices, nnz, int32_t);
    GN_BUP(bt->gid, gid.data(), n, int32_t);
#undef GN_BUP
    bt->device_bytes = bytes;
    cudaError_t e = cudaStreamSynchronize(ctx.s);
    if (e != cudaSuccess) return cleanup(cuda_fail(e, "sync", __FILE__, __LINE__));
    *out = bt;
    return GN_OK;
}

void batch_destroy(gn_batch* bt) { free_batch(bt); }

size_t batch_smem_bytes(const gn_batch* bt) {
    const size_t gsz = bt->dtype == GN_F64 ? 8 : 4;
    const size_t yoff = ((size_t)bt->max_idx * 2 + 15) / 16 * 16;
    return yoff + 2 * (size_t)bt->max_n * gsz;
}

template <typename TS, typename TG>
static int batch_run_typed(gn_batch* bt, const void* x0, const double* gammas, int iters, double final_gamma,
                           uint32_t flags, void* x_out, double* step_inf, int64_t* fallbacks, double* mass,
                           double* energy, double* pre_energy, double* x_hist, int* iters_run, int* status,
                           int* fail_iter, gn_run_stats* stats) {
    const bool trace = (flags & GN_TRACE) != 0;
    const bool dev_io = (flags & GN_DEVICE_IO) != 0;
    const int64_t B = bt->B, n = bt->n;
    const size_t nb = (size_t)std::max<int64_t>(n, 1);
    const int64_t launches0 = gn_launch_count();
    CallCtx ctx;
    int rc = ctx.open(bt->device);
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

    struct Ws {
        void* p[16] = {};
        int np = 0;
        cudaStream_t s = nullptr;
        ~Ws() { for (int i = 0; i < np; ++i) cudaFreeAsync(p[i], s); }
    } ws;
    ws.s = s;
    auto alloc = [&](void** p, size_t bytes) {
        cudaError_t e = cudaMallocAsync(p, std::max<size_t>(bytes, 16), s);
        if (e == cudaSuccess) ws.p[ws.np++] = *p;
        return e;
    };
    double *xin = nullptr, *xout = nullptr, *dsi = nullptr, *dfb = nullptr, *dd = nullptr, *hist = nullptr,
           *gam = nullptr;
    int *dran = nullptr, *dbad = nullptr, *chk = nullptr;
    GN_CUDA(alloc((void**)&dsi, 8 * (size_t)B * iters));
    GN_CUDA(alloc((void**)&dfb, 8 * (size_t)B * iters));
    GN_CUDA(alloc((void**)&dd, 8 * 4 * (size_t)B * (iters + 1)));
    GN_CUDA(alloc((void**)&dran, 4 * (size_t)B));
    GN_CUDA(alloc((void**)&dbad, 4 * (size_t)B));
    GN_CUDA(alloc((void**)&chk, 8 * (size_t)B));
    GN_CUDA(alloc((void**)&gam, 8 * (size_t)iters));
    GN_CUDA(cudaMemsetAsync(dsi, 0, 8 * (size_t)B * iters, s));
    GN_CUDA(cudaMemsetAsync(dfb, 0, 8 * (size_t)B * iters, s));
    GN_CUDA(cudaMemsetAsync(dd, 0, 8 * 4 * (size_t)B * (iters + 1), s));
    GN_CUDA(cudaMemsetAsync(chk, 0, 8 * (size_t)B, s));
    GN_CUDA(cudaMemcpyAsync(gam, gammas, 8 * (size_t)iters, cudaMemcpyHostToDevice, s));
    h2d += 8 * iters;
    if (dev_io) {
        xin = (double*)x0;
        xout = (double*)x_out;
    } else {
        GN_CUDA(alloc((void**)&xin, 8 * nb));
        GN_CUDA(alloc((void**)&xout, 8 * nb));
        if (n > 0) GN_CUDA(cudaMemcpyAsync(xin, x0, 8 * (size_t)n, cudaMemcpyHostToDevice, s));
        h2d += 8 * n;
    }
    if (x_hist) GN_CUDA(alloc((void**)&hist, 8 * nb * (size_t)iters));
    std::vector<int> hchk((size_t)B * 2, 0);
    const bool check = !(flags & GN_NO_CHECK);
    if (check && n > 0) {
        k_precheck_batch<<<(int)((n + 255) / 256), 256, 0, s>>>(n, bt->rowptr, bt->col, bt->gid, xin, chk);
        GN_LAUNCHED();
        GN_CUDA(cudaMemcpyAsync(hchk.data(), chk, 8 * (size_t)B, cudaMemcpyDeviceToHost, s));
        GN_CUDA(cudaStreamSynchronize(s));
    }

    BatchArgs<TS, TG> a;
    memset(&a, 0, sizeof(a));
    a.B = B;
    a.voff = bt->voff;
    a.ioff = bt->ioff;
    a.gbase = bt->gbase;
    a.goff = bt->goff;
    a.idx = bt->idx;
    a.deg = bt->deg;
    a.lperm = bt->lperm;
    a.w64 = bt->w64;
    a.x0 = xin;
    a.x_out = xout;
    a.gammas = gam;
    a.iters = iters;
    a.final_gamma = final_gamma;
    a.early_exit = (flags & GN_EARLY_EXIT) ? 1 : 0;
    a.stop_nonfinite = (flags & GN_NONFINITE_OK) ? 0 : 1;
    a.trace = trace ? 1 : 0;
    a.step_inf = dsi;
    a.fb = dfb;
    a.dots = dd;
    a.ran = dran;
    a.bad = dbad;
    a.x_hist = hist;
    a.n_total = n;
    a.clip = (flags & GN_NO_CLIP) ? 0 : 1;
    const size_t smem = batch_smem_bytes(bt);
    a.smem_y_off = (int)(((size_t)bt->max_idx * 2 + 15) / 16 * 16);
    void* kern = trace ? (void*)k_gn_batch<TS, TG, true> : (void*)k_gn_batch<TS, TG, false>;
    GN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    // rows per thread: one, up to the 1024-thread block (more warps to hide
    // the dependent per-row add chains of a lone graph); a batch that fills
    // the GPU twice over runs 512-thread blocks instead -- two graphs per SM,
    // so one graph's per-iteration reduction and barrier hide under the
    // other's gathers (C4: 37.4 -> 31.0 ms fp32); GN_BATCH_THREADS overrides
    int threads = (int)std::min<int64_t>(kBatchThreads, std::max<int64_t>(32, (bt->max_n + 31) / 32 * 32));
    {
        int sms = 0;
        GN_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, bt->device));
        if (B >= 2 * (int64_t)sms && threads > kBatchThreads / 2) threads = kBatchThreads / 2;
    }
    if (const char* e = getenv("GN_BATCH_THREADS")) threads = std::max(32, std::min(kBatchThreads, atoi(e)));
    threads = std::max<int>(threads, (int)((bt->max_n + kRowsPerThread - 1) / kRowsPerThread + 31) / 32 * 32);
    GN_CUDA(cudaEventRecord(ev[1], s));
    if (B > 0 && n > 0) {
        void* args[] = {&a};
        GN_CUDA(cudaLaunchKernel(kern, dim3((unsigned)B), dim3(threads), args, smem, s));
        GN_LAUNCHED();
    }
    GN_CUDA(cudaEventRecord(ev[2], s));
    const bool want_trace = step_inf || fallbacks || mass || energy || pre_energy;
    // without energies the traces are finished on the device and copied
    // straight into the caller's arrays (C4: 64 -> 40 MB d2h, no host scatter)
    const bool direct = n > 0 && want_trace && !trace;
    std::vector<double> hsi, hfb, hd;
    if (want_trace && !direct) {
        hsi.resize((size_t)B * iters);
        hfb.resize((size_t)B * iters);
        hd.resize(4 * (size_t)B * (iters + 1));
    }
    std::vector<int> hran((size_t)B, 0), hbad((size_t)B, -1);
    if (direct && B > 0) {
        double* dmass = nullptr;
        if (mass) GN_CUDA(alloc((void**)&dmass, 8 * (size_t)B * iters));
        const int64_t tot = B * (int64_t)iters;
        const int blocks = (int)std::min<int64_t>((tot + 255) / 256, 148 * 8);
        k_batch_outputs<<<blocks, 256, 0, s>>>(B, iters, chk, dran, dbad, (flags & GN_NONFINITE_OK) ? 0 : 1, dsi, dfb,
                                               dd, dmass);
        GN_LAUNCHED();
        if (step_inf) GN_CUDA(cudaMemcpyAsync(step_inf, dsi, 8 * (size_t)tot, cudaMemcpyDeviceToHost, s));
        if (fallbacks) GN_CUDA(cudaMemcpyAsync(fallbacks, dfb, 8 * (size_t)tot, cudaMemcpyDeviceToHost, s));
        if (mass) GN_CUDA(cudaMemcpyAsync(mass, dmass, 8 * (size_t)tot, cudaMemcpyDeviceToHost, s));
        d2h += 8 * tot * ((step_inf ? 1 : 0) + (fallbacks ? 1 : 0) + (mass ? 1 : 0));
    }
    if (n > 0) {
        if (want_trace && !direct) {  // per-graph traces only when asked for (B x iters values each)
            GN_CUDA(cudaMemcpyAsync(hsi.data(), dsi, 8 * hsi.size(), cudaMemcpyDeviceToHost, s));
            GN_CUDA(cudaMemcpyAsync(hfb.data(), dfb, 8 * hfb.size(), cudaMemcpyDeviceToHost, s));
            GN_CUDA(cudaMemcpyAsync(hd.data(), dd, 8 * hd.size(), cudaMemcpyDeviceToHost, s));
            d2h += 8 * (int64_t)(hsi.size() + hfb.size() + hd.size());
        }
        GN_CUDA(cudaMemcpyAsync(hran.data(), dran, 4 * (size_t)B, cudaMemcpyDeviceToHost, s));
        GN_CUDA(cudaMemcpyAsync(hbad.data(), dbad, 4 * (size_t)B, cudaMemcpyDeviceToHost, s));
        d2h += 8 * B;
        if (x_out && !dev_io) {
            GN_CUDA(cudaMemcpyAsync(x_out, xout, 8 * (size_t)n, cudaMemcpyDeviceToHost, s));
            d2h += 8 * n;
        }
    } else {
        for (int64_t b = 0; b < B; ++b) hran[(size_t)b] = iters;  // empty graphs: step_inf 0 every iteration
    }
    GN_CUDA(cudaEventRecord(ev[3], s));
    GN_CUDA(cudaStreamSynchronize(s));
    int first_rc = GN_OK;
    for (int64_t b = 0; b < B; ++b) {
        int st = GN_OK;
        if (hchk[(size_t)2 * b]) st = GN_ERR_NEGATIVE;
        else if (hchk[(size_t)2 * b + 1]) st = GN_ERR_NOT_NORMALIZABLE;
        else if (hbad[(size_t)b] >= 0 && !(flags & GN_NONFINITE_OK)) st = GN_ERR_NONFINITE;
        if (status) status[b] = st;
        if (fail_iter) fail_iter[b] = hbad[(size_t)b];
        int ran = hran[(size_t)b];
        if (st == GN_ERR_NONFINITE) ran = hbad[(size_t)b] + 1;
        if (iters_run) iters_run[b] = ran;
        if (direct || !want_trace) {
            if (st != GN_OK && first_rc == GN_OK) first_rc = st;
            continue;
        }
        const double* db = &hd[(size_t)b * (iters + 1) * 4];
        for (int k = 0; k < ran && k < iters; ++k) {
            const size_t o = (size_t)b * iters + k;
            if (step_inf) step_inf[o] = hsi[o];
            if (fallbacks) fallbacks[o] = (int64_t)hfb[o];
            if (mass) mass[o] = db[(size_t)k * 4 + 3];
            if (trace) {
                const double* d0 = db + (size_t)k * 4;
                const double* d1 = db + (size_t)(k + 1) * 4;
                if (pre_energy) pre_energy[o] = 0.5 * (d0[0] + gammas[k] * d0[1]) - d0[2];
                if (energy) energy[o] = 0.5 * (d1[0] + gammas[k] * d1[1]) - d1[2];
            }
        }
        if (st != GN_OK && first_rc == GN_OK) first_rc = st;
    }
    if (x_hist && n > 0) {
        int mx = 0;
        for (int64_t b = 0; b < B; ++b) mx = std::max(mx, hran[(size_t)b]);
        if (mx > 0) GN_CUDA(cudaMemcpy(x_hist, hist, 8 * (size_t)mx * (size_t)n, cudaMemcpyDeviceToHost));
    }
    if (stats) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev[1], ev[2]);
        stats->loop_ms = ms;
        cudaEventElapsedTime(&ms, ev[0], ev[3]);
        stats->total_ms = ms;
        stats->launches = gn_launch_count() - launches0;
        stats->grid_blocks = B;
        stats->block_threads = threads;
        stats->h2d_bytes = h2d;
        stats->d2h_bytes = d2h;
    }
    if (first_rc == GN_ERR_NEGATIVE) return fail(first_rc, "state entries must be nonnegative");
    if (first_rc == GN_ERR_NOT_NORMALIZABLE) return fail(first_rc, "initial state has a zero closed neighborhood sum");
    if (first_rc == GN_ERR_NONFINITE) {
        char buf[64];
        int k = -1;
        for (int64_t b = 0; b < B; ++b)
            if (hbad[(size_t)b] >= 0) { k = hbad[(size_t)b]; break; }
        snprintf(buf, sizeof(buf), "non-finite state at iteration %d", k);
        return fail(first_rc, buf);
    }
    return GN_OK;
}

int batch_run(gn_batch* bt, const void* x0, const double* gammas, int iters, double final_gamma, uint32_t flags,
              void* x_out, double* step_inf, int64_t* fallbacks, double* mass, double* energy, double* pre_energy,
              double* x_hist, int* iters_run, int* status, int* fail_iter, gn_run_stats* stats) {
    switch (bt->dtype) {
        case GN_F64:
            return batch_run_typed<double, double>(bt, x0, gammas, iters, final_gamma, flags, x_out, step_inf, fallbacks,
                                                   mass, energy, pre_energy, x_hist, iters_run, status, fail_iter, stats);
        case GN_F32:
            return batch_run_typed<double, float>(bt, x0, gammas, iters, final_gamma, flags, x_out, step_inf, fallbacks,
                                                  mass, energy, pre_energy, x_hist, iters_run, status, fail_iter, stats);
        default:
            return batch_run_typed<float, float>(bt, x0, gammas, iters, final_gamma, flags, x_out, step_inf, fallbacks,
                                                 mass, energy, pre_energy, x_hist, iters_run, status, fail_iter, stats);
    }
}

}  // namespace gn

using namespace gn;

extern "C" {

int gn_batch_create(int64_t num_graphs, const int64_t* offsets, int64_t n, const int64_t* indptr,
                    const int32_t* indices, const double* w, int dtype, int device, gn_batch** out) {
    GN_NVTX("gn_batch_create");
    if (!valid_dtype(dtype)) return fail(GN_ERR_ARG, "dtype must be GN_F64, GN_F32 or GN_F32_PURE");
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(GN_ERR_NODEV, "no CUDA device visible: the GN engine has no CPU fallback");
    }
    if (device < 0 || device >= ndev) return fail(GN_ERR_ARG, "device ordinal out of range");
    int rc = batch_create(num_graphs, offsets, n, indptr, indices, w, dtype, device, out);
    if (rc == GN_OK) {
        int max_optin = 0;
        cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
        if (batch_smem_bytes(*out) + 2 * kBatchThreads / 32 * 8 * 8 > (size_t)max_optin) {
            batch_destroy(*out);
            *out = nullptr;
            return fail(GN_ERR_ARG, "batch graph does not fit in shared memory");
        }
    }
    return rc;
}

int gn_batch_destroy(gn_batch* b) {
    batch_destroy(b);
    return GN_OK;
}

int gn_batch_run(gn_batch* b, const void* x0, const double* gammas, int iters, double final_gamma, uint32_t flags,
                 void* x_out, double* step_inf, int64_t* fallbacks, double* mass, int* iters_run, int* status,
                 int* fail_iter, gn_run_stats* stats) {
    GN_NVTX("gn_batch_run");
    if (!b) return fail(GN_ERR_ARG, "null batch");
    if (iters < 1) return fail(GN_ERR_ARG, "iterations must be positive");
    if (!gammas || (b->n > 0 && !x0)) return fail(GN_ERR_ARG, "null input array");
    return batch_run(b, x0, gammas, iters, final_gamma, flags & ~(uint32_t)GN_TRACE, x_out, step_inf, fallbacks, mass,
                     nullptr, nullptr, nullptr, iters_run, status, fail_iter, stats);
}

int gn_batch_info(const gn_batch* b, int64_t* num_graphs, int64_t* n, int64_t* device_bytes, int64_t* smem_bytes) {
    if (!b) return fail(GN_ERR_ARG, "null batch");
    if (num_graphs) *num_graphs = b->B;
    if (n) *n = b->n;
    if (device_bytes) *device_bytes = b->device_bytes;
    if (smem_bytes) *smem_bytes = (int64_t)batch_smem_bytes(b);
    return GN_OK;
}

}  // extern "C"
