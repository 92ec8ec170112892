// gn_graph.cu -- graph upload, degree binning, error plumbing and the fp64
// auxiliary operators (SpMV, normalisability, energy, mass, simplex, fitness).
//
// Reference: graph.py:22-75 (WeightedGraph), dynamics.py:122-126,210-250.
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "gn_internal.cuh"

namespace gn {

static thread_local std::string g_last_error;
static std::atomic<int64_t> g_launches{0};

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
    char buf[512];
    snprintf(buf, sizeof(buf), "CUDA error %s (%s) at %s:%d: %s", cudaGetErrorName(e),
             cudaGetErrorString(e), file, line, what);
    g_last_error = buf;
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) return GN_ERR_NODEV;
    if (e == cudaErrorMemoryAllocation) return GN_ERR_NOMEM;
    return GN_ERR_CUDA;
}

void note_launch(int64_t k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

int CallCtx::open(int device) {
    dev = device;
    GN_CUDA(cudaGetDevice(&prev_dev));
    if (prev_dev != device) GN_CUDA(cudaSetDevice(device));
    GN_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    return GN_OK;
}

CallCtx::~CallCtx() {
    if (s) cudaStreamDestroy(s);
    if (prev_dev >= 0 && prev_dev != dev) cudaSetDevice(prev_dev);
}

int coresident_blocks(const void* kernel, int threads, size_t smem, int device, int* out) {
    int per_sm = 0, sms = 0;
    GN_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem));
    GN_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    *out = per_sm * sms;
    return GN_OK;
}

// ---------------------------------------------------------------- kernels

template <typename T>
__global__ void k_init_weights(int64_t n, const double* __restrict__ w64, T* __restrict__ v,
                               T* __restrict__ w) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) {
        double wi = w64[i];
        v[i] = (T)sqrt(wi);  // graph.py:42 (IEEE sqrt; fp32: the rounding of the fp64 root)
        w[i] = (T)wi;
    }
}

// out = A @ in (fp64), one thread per row, sequential sum (scipy order).
__global__ void k_spmv_seq(int64_t n, const int32_t* __restrict__ rowptr,
                           const int32_t* __restrict__ col, const double* __restrict__ in,
                           double* __restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double s = 0.0;
    for (int32_t p = rowptr[i]; p < rowptr[i + 1]; ++p) s = __dadd_rn(s, in[col[p]]);
    out[i] = s;
}

// closed[i] = x_i + (A x)_i > 0 for all i  (dynamics.py:125); also x >= 0.
__global__ void k_precheck(int64_t n, const int32_t* __restrict__ rowptr,
                           const int32_t* __restrict__ col, const double* __restrict__ x,
                           int* __restrict__ flags) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double xi = x[i];
    if (xi < 0.0) atomicOr(&flags[0], 1);
    double s = 0.0;
    for (int32_t p = rowptr[i]; p < rowptr[i + 1]; ++p) s = __dadd_rn(s, x[col[p]]);
    if (!(__dadd_rn(xi, s) > 0.0)) atomicOr(&flags[1], 1);
}

// Deterministic block partial sums of up to 4 fp64 terms, then a fixed-order
// final reduction by one block.
constexpr int kAuxThreads = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

template <int K>
__device__ __forceinline__ void block_sum_store(double (&acc)[K], double* __restrict__ dst) {
    __shared__ double red[kAuxThreads / 32][K];
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] = warp_sum(acc[k]);
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < K; ++k) red[wid][k] = acc[k];
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            double s = 0.0;
            for (int q = 0; q < (int)(blockDim.x >> 5); ++q) s = __dadd_rn(s, red[q][k]);
            dst[blockIdx.x * K + k] = s;
        }
    }
}

template <int K>
__global__ void k_final_sum(const double* __restrict__ partials, int nparts, double* __restrict__ out) {
    // one warp, fixed order
    int lane = threadIdx.x;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        double s = 0.0;
        for (int q = lane; q < nparts; q += 32) s = __dadd_rn(s, partials[q * K + k]);
        s = warp_sum(s);
        if (lane == 0) out[k] = s;
    }
}

// energy terms: y.y, y.(Ay), w.x with y = sqrt(w) x  (dynamics.py:216-219)
__global__ void k_energy_terms(int64_t n, const int32_t* __restrict__ rowptr,
                               const int32_t* __restrict__ col, const double* __restrict__ w64,
                               const double* __restrict__ x, double* __restrict__ partials) {
    double acc[3] = {0.0, 0.0, 0.0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double yi = __dmul_rn(sqrt(w64[i]), x[i]);
        double s = 0.0;
        for (int32_t p = rowptr[i]; p < rowptr[i + 1]; ++p) {
            int32_t j = col[p];
            s = __dadd_rn(s, __dmul_rn(sqrt(w64[j]), x[j]));
        }
        acc[0] = __dadd_rn(acc[0], __dmul_rn(yi, yi));
        acc[1] = __dadd_rn(acc[1], __dmul_rn(yi, s));
        acc[2] = __dadd_rn(acc[2], __dmul_rn(w64[i], x[i]));
    }
    block_sum_store<3>(acc, partials);
}

__global__ void k_mass_terms(int64_t n, const double* __restrict__ w64, const double* __restrict__ x,
                             double* __restrict__ partials) {
    double acc[1] = {0.0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        acc[0] = __dadd_rn(acc[0], __dmul_rn(w64[i], x[i]));
    block_sum_store<1>(acc, partials);
}

__global__ void k_scale(int64_t n, const double* __restrict__ w64, const double* __restrict__ x,
                        const double* __restrict__ m, double* __restrict__ p) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) p[i] = __ddiv_rn(__dmul_rn(w64[i], x[i]), m[0]);  // dynamics.py:233
}

// fitness (dynamics.py:242-250): q = p/v; d = q + gamma*(A q); f = v/d
__global__ void k_fitness(int64_t n, const int32_t* __restrict__ rowptr,
                          const int32_t* __restrict__ col, const double* __restrict__ w64,
                          const double* __restrict__ p, double gamma, double* __restrict__ f,
                          int* __restrict__ bad, double* __restrict__ partials) {
    double acc[1] = {0.0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double vi = sqrt(w64[i]);
        double qi = __ddiv_rn(p[i], vi);
        double s = 0.0;
        for (int32_t q = rowptr[i]; q < rowptr[i + 1]; ++q) {
            int32_t j = col[q];
            s = __dadd_rn(s, __ddiv_rn(p[j], sqrt(w64[j])));
        }
        double d = __dadd_rn(qi, __dmul_rn(gamma, s));
        if (d <= 0.0) atomicOr(bad, 1);
        double fi = __ddiv_rn(vi, d);
        f[i] = fi;
        acc[0] = __dadd_rn(acc[0], __dmul_rn(p[i], fi));
    }
    block_sum_store<1>(acc, partials);
}

static int grid_for(int64_t n, int threads) {
    int64_t b = (n + threads - 1) / threads;
    return (int)std::max<int64_t>(1, std::min<int64_t>(b, 1 << 20));
}

static int aux_grid(const gn_graph* g) {
    int64_t b = (g->n + kAuxThreads - 1) / kAuxThreads;
    return (int)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)g->num_sms * 8));
}

// ---------------------------------------------------------------- planning

static int lanes_for_degree(int32_t d) {
    if (d <= 4) return 1;
    if (d <= 8) return 2;
    if (d <= 16) return 4;
    if (d <= 32) return 8;
    if (d <= 64) return 16;
    if (d <= 8192) return 32;
    return 0;  // block per row
}

static int build_plans(gn_graph* g, const int64_t* indptr, std::vector<int32_t>& rows_out) {
    const int64_t n = g->n;
    // fixed bin order: block rows first (longest), then G = 32 .. 1
    const int order[7] = {0, 32, 16, 8, 4, 2, 1};
    std::vector<std::vector<int32_t>> lists(7);
    int32_t maxd = 0;
    for (int64_t i = 0; i < n; ++i) {
        int32_t d = (int32_t)(indptr[i + 1] - indptr[i]);
        maxd = std::max(maxd, d);
        int G = lanes_for_degree(d);
        for (int b = 0; b < 7; ++b)
            if (order[b] == G) { lists[b].push_back((int32_t)i); break; }
    }
    g->max_degree = maxd;
    rows_out.clear();
    rows_out.reserve((size_t)n);
    g->fast.nbins = 0;
    for (int b = 0; b < 7; ++b) {
        if (lists[b].empty()) continue;
        Bin& bin = g->fast.bins[g->fast.nbins++];
        bin.off = (int32_t)rows_out.size();
        bin.count = (int32_t)lists[b].size();
        bin.G = order[b];
        bin.pad = 0;
        rows_out.insert(rows_out.end(), lists[b].begin(), lists[b].end());
    }
    g->exact.nbins = n > 0 ? 1 : 0;
    g->exact.bins[0] = Bin{0, (int32_t)n, 1, 0};
    g->exact.rows = nullptr;
    return GN_OK;
}

static void free_graph(gn_graph* g) {
    if (!g) return;
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(g->device);
    cudaFree(g->rowptr);
    cudaFree(g->col);
    cudaFree(g->v);
    cudaFree(g->w);
    cudaFree(g->w64);
    cudaFree(g->fast.rows);
    if (prev >= 0) cudaSetDevice(prev);
    delete g;
}

}  // namespace gn

using namespace gn;

extern "C" {

int gn_abi_version(void) { return GN_ABI_VERSION; }

const char* gn_last_error(void) { return g_last_error.c_str(); }

int64_t gn_launch_count(void) { return g_launches.load(); }

int gn_device_count(int* count) {
    *count = 0;
    cudaError_t e = cudaGetDeviceCount(count);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *count = 0;
        return cuda_fail(e, "cudaGetDeviceCount", __FILE__, __LINE__);
    }
    return GN_OK;
}

int gn_graph_create(int64_t n, const int64_t* indptr, const int32_t* indices, const double* w,
                    int dtype, int device, gn_graph** out) {
    *out = nullptr;
    if (n < 0) return fail(GN_ERR_ARG, "vertex count must be nonnegative");
    if (dtype != GN_F64 && dtype != GN_F32) return fail(GN_ERR_ARG, "dtype must be GN_F64 or GN_F32");
    if (n > 0 && (!indptr || !w)) return fail(GN_ERR_ARG, "null graph array");
    const int64_t nnz = n > 0 ? indptr[n] : 0;
    if (nnz >= (int64_t(1) << 31) || n >= (int64_t(1) << 31))
        return fail(GN_ERR_ARG, "graphs with >= 2^31 adjacency entries need the partitioned engine");
    if (n > 0 && indptr[0] != 0) return fail(GN_ERR_ARG, "indptr[0] must be 0");
    for (int64_t i = 0; i < n; ++i)
        if (indptr[i + 1] < indptr[i]) return fail(GN_ERR_ARG, "indptr must be nondecreasing");

    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(GN_ERR_NODEV, "no CUDA device visible: the GN engine has no CPU fallback");
    }
    if (device < 0 || device >= ndev) return fail(GN_ERR_ARG, "device ordinal out of range");

    gn_graph* g = new gn_graph();
    g->n = n;
    g->nnz = nnz;
    g->dtype = dtype;
    g->device = device;
    CallCtx ctx;
    int rc = ctx.open(device);
    if (rc) { delete g; return rc; }
    cudaDeviceGetAttribute(&g->num_sms, cudaDevAttrMultiProcessorCount, device);

    std::vector<int32_t> rowptr32((size_t)n + 1);
    for (int64_t i = 0; i <= n; ++i) rowptr32[(size_t)i] = (int32_t)(n > 0 ? indptr[i] : 0);
    std::vector<int32_t> rows;
    build_plans(g, n > 0 ? indptr : nullptr, rows);

    const size_t es = dtype == GN_F64 ? 8 : 4;
    const size_t nb = (size_t)std::max<int64_t>(n, 1);
    auto cleanup = [&](int code) { free_graph(g); return code; };
#define GN_TRY(expr)                                                              \
    do {                                                                          \
        cudaError_t _e = (expr);                                                  \
        if (_e != cudaSuccess) return cleanup(cuda_fail(_e, #expr, __FILE__, __LINE__)); \
    } while (0)
    GN_TRY(cudaMalloc(&g->rowptr, sizeof(int32_t) * (nb + 1)));
    GN_TRY(cudaMalloc(&g->col, sizeof(int32_t) * (size_t)std::max<int64_t>(nnz, 1)));
    GN_TRY(cudaMalloc(&g->v, es * nb));
    GN_TRY(cudaMalloc(&g->w, es * nb));
    GN_TRY(cudaMalloc(&g->w64, sizeof(double) * nb));
    GN_TRY(cudaMalloc(&g->fast.rows, sizeof(int32_t) * nb));
    g->device_bytes = (int64_t)(sizeof(int32_t) * (nb + 1) + sizeof(int32_t) * std::max<int64_t>(nnz, 1) +
                                2 * es * nb + 8 * nb + 4 * nb);
    GN_TRY(cudaMemcpyAsync(g->rowptr, rowptr32.data(), sizeof(int32_t) * (size_t)(n + 1),
                           cudaMemcpyHostToDevice, ctx.s));
    if (nnz > 0)
        GN_TRY(cudaMemcpyAsync(g->col, indices, sizeof(int32_t) * (size_t)nnz, cudaMemcpyHostToDevice, ctx.s));
    if (n > 0) {
        GN_TRY(cudaMemcpyAsync(g->w64, w, sizeof(double) * (size_t)n, cudaMemcpyHostToDevice, ctx.s));
        GN_TRY(cudaMemcpyAsync(g->fast.rows, rows.data(), sizeof(int32_t) * (size_t)n,
                               cudaMemcpyHostToDevice, ctx.s));
        int blocks = grid_for(n, 256);
        if (dtype == GN_F64)
            k_init_weights<double><<<blocks, 256, 0, ctx.s>>>(n, g->w64, (double*)g->v, (double*)g->w);
        else
            k_init_weights<float><<<blocks, 256, 0, ctx.s>>>(n, g->w64, (float*)g->v, (float*)g->w);
        GN_TRY(cudaGetLastError());
        note_launch();
    }
    GN_TRY(cudaStreamSynchronize(ctx.s));
#undef GN_TRY
    *out = g;
    return GN_OK;
}

int gn_graph_destroy(gn_graph* g) {
    free_graph(g);
    return GN_OK;
}

int gn_graph_info(const gn_graph* g, int64_t* n, int64_t* nnz, int* dtype, int* device,
                  int64_t* device_bytes, int* num_bins) {
    if (!g) return fail(GN_ERR_ARG, "null graph");
    if (n) *n = g->n;
    if (nnz) *nnz = g->nnz;
    if (dtype) *dtype = g->dtype;
    if (device) *device = g->device;
    if (device_bytes) *device_bytes = g->device_bytes;
    if (num_bins) *num_bins = g->fast.nbins;
    return GN_OK;
}

int gn_graph_set_grid(gn_graph* g, int blocks) {
    if (!g || blocks < 0) return fail(GN_ERR_ARG, "bad grid override");
    g->grid_override = blocks;
    return GN_OK;
}

// ---- fp64 auxiliary operators (one-shot; not on the iteration loop) ----

static int upload_vec(CallCtx& ctx, const double* h, int64_t n, double** d) {
    GN_CUDA(cudaMallocAsync((void**)d, sizeof(double) * (size_t)std::max<int64_t>(n, 1), ctx.s));
    if (n > 0) GN_CUDA(cudaMemcpyAsync(*d, h, sizeof(double) * (size_t)n, cudaMemcpyHostToDevice, ctx.s));
    return GN_OK;
}

int gn_spmv(gn_graph* g, const double* in, double* out) {
    if (!g) return fail(GN_ERR_ARG, "null graph");
    CallCtx ctx;
    int rc = ctx.open(g->device);
    if (rc) return rc;
    double *din = nullptr, *dout = nullptr;
    if ((rc = upload_vec(ctx, in, g->n, &din))) return rc;
    GN_CUDA(cudaMallocAsync((void**)&dout, sizeof(double) * (size_t)std::max<int64_t>(g->n, 1), ctx.s));
    if (g->n > 0) {
        k_spmv_seq<<<grid_for(g->n, 256), 256, 0, ctx.s>>>(g->n, g->rowptr, g->col, din, dout);
        GN_LAUNCHED();
        GN_CUDA(cudaMemcpyAsync(out, dout, sizeof(double) * (size_t)g->n, cudaMemcpyDeviceToHost, ctx.s));
    }
    cudaFreeAsync(din, ctx.s);
    cudaFreeAsync(dout, ctx.s);
    GN_CUDA(cudaStreamSynchronize(ctx.s));
    return GN_OK;
}

int gn_is_normalizable(gn_graph* g, const double* x, int* ok) {
    if (!g) return fail(GN_ERR_ARG, "null graph");
    CallCtx ctx;
    int rc = ctx.open(g->device);
    if (rc) return rc;
    double* dx = nullptr;
    int* flags = nullptr;
    if ((rc = upload_vec(ctx, x, g->n, &dx))) return rc;
    GN_CUDA(cudaMallocAsync((void**)&flags, 2 * sizeof(int), ctx.s));
    GN_CUDA(cudaMemsetAsync(flags, 0, 2 * sizeof(int), ctx.s));
    if (g->n > 0) {
        k_precheck<<<grid_for(g->n, 256), 256, 0, ctx.s>>>(g->n, g->rowptr, g->col, dx, flags);
        GN_LAUNCHED();
    }
    int hf[2];
    GN_CUDA(cudaMemcpyAsync(hf, flags, sizeof(hf), cudaMemcpyDeviceToHost, ctx.s));
    cudaFreeAsync(dx, ctx.s);
    cudaFreeAsync(flags, ctx.s);
    GN_CUDA(cudaStreamSynchronize(ctx.s));
    *ok = hf[1] == 0;
    return GN_OK;
}

int gn_energy(gn_graph* g, const double* x, double gamma, double* energy) {
    if (!g) return fail(GN_ERR_ARG, "null graph");
    CallCtx ctx;
    int rc = ctx.open(g->device);
    if (rc) return rc;
    double *dx = nullptr, *part = nullptr, *res = nullptr;
    if ((rc = upload_vec(ctx, x, g->n, &dx))) return rc;
    int blocks = aux_grid(g);
    GN_CUDA(cudaMallocAsync((void**)&part, sizeof(double) * 3 * (size_t)blocks, ctx.s));
    GN_CUDA(cudaMallocAsync((void**)&res, sizeof(double) * 3, ctx.s));
    k_energy_terms<<<blocks, kAuxThreads, 0, ctx.s>>>(g->n, g->rowptr, g->col, g->w64, dx, part);
    GN_LAUNCHED();
    k_final_sum<3><<<1, 32, 0, ctx.s>>>(part, blocks, res);
    GN_LAUNCHED();
    double h[3];
    GN_CUDA(cudaMemcpyAsync(h, res, sizeof(h), cudaMemcpyDeviceToHost, ctx.s));
    cudaFreeAsync(dx, ctx.s);
    cudaFreeAsync(part, ctx.s);
    cudaFreeAsync(res, ctx.s);
    GN_CUDA(cudaStreamSynchronize(ctx.s));
    *energy = 0.5 * (h[0] + gamma * h[1]) - h[2];  // dynamics.py:219
    return GN_OK;
}

int gn_weighted_mass(gn_graph* g, const double* x, double* mass) {
    if (!g) return fail(GN_ERR_ARG, "null graph");
    CallCtx ctx;
    int rc = ctx.open(g->device);
    if (rc) return rc;
    double *dx = nullptr, *part = nullptr, *res = nullptr;
    if ((rc = upload_vec(ctx, x, g->n, &dx))) return rc;
    int blocks = aux_grid(g);
    GN_CUDA(cudaMallocAsync((void**)&part, sizeof(double) * (size_t)blocks, ctx.s));
    GN_CUDA(cudaMallocAsync((void**)&res, sizeof(double), ctx.s));
    k_mass_terms<<<blocks, kAuxThreads, 0, ctx.s>>>(g->n, g->w64, dx, part);
    GN_LAUNCHED();
    k_final_sum<1><<<1, 32, 0, ctx.s>>>(part, blocks, res);
    GN_LAUNCHED();
    GN_CUDA(cudaMemcpyAsync(mass, res, sizeof(double), cudaMemcpyDeviceToHost, ctx.s));
    cudaFreeAsync(dx, ctx.s);
    cudaFreeAsync(part, ctx.s);
    cudaFreeAsync(res, ctx.s);
    GN_CUDA(cudaStreamSynchronize(ctx.s));
    return GN_OK;
}

int gn_simplex_state(gn_graph* g, const double* x, double* p_out) {
    if (!g) return fail(GN_ERR_ARG, "null graph");
    CallCtx ctx;
    int rc = ctx.open(g->device);
    if (rc) return rc;
    double *dx = nullptr, *part = nullptr, *res = nullptr, *dp = nullptr;
    if ((rc = upload_vec(ctx, x, g->n, &dx))) return rc;
    int blocks = aux_grid(g);
    GN_CUDA(cudaMallocAsync((void**)&part, sizeof(double) * (size_t)blocks, ctx.s));
    GN_CUDA(cudaMallocAsync((void**)&res, sizeof(double), ctx.s));
    GN_CUDA(cudaMallocAsync((void**)&dp, sizeof(double) * (size_t)std::max<int64_t>(g->n, 1), ctx.s));
    k_mass_terms<<<blocks, kAuxThreads, 0, ctx.s>>>(g->n, g->w64, dx, part);
    GN_LAUNCHED();
    k_final_sum<1><<<1, 32, 0, ctx.s>>>(part, blocks, res);
    GN_LAUNCHED();
    double m = 0.0;
    GN_CUDA(cudaMemcpyAsync(&m, res, sizeof(double), cudaMemcpyDeviceToHost, ctx.s));
    GN_CUDA(cudaStreamSynchronize(ctx.s));
    int out = GN_OK;
    if (!(m > 0.0)) {
        out = fail(GN_ERR_ZERO_MASS, "weighted mass must be positive");
    } else if (g->n > 0) {
        k_scale<<<grid_for(g->n, 256), 256, 0, ctx.s>>>(g->n, g->w64, dx, res, dp);
        GN_LAUNCHED();
        GN_CUDA(cudaMemcpyAsync(p_out, dp, sizeof(double) * (size_t)g->n, cudaMemcpyDeviceToHost, ctx.s));
    }
    cudaFreeAsync(dx, ctx.s);
    cudaFreeAsync(part, ctx.s);
    cudaFreeAsync(res, ctx.s);
    cudaFreeAsync(dp, ctx.s);
    GN_CUDA(cudaStreamSynchronize(ctx.s));
    return out;
}

int gn_fitness(gn_graph* g, const double* p, double gamma, double* f_out, double* fbar) {
    if (!g) return fail(GN_ERR_ARG, "null graph");
    CallCtx ctx;
    int rc = ctx.open(g->device);
    if (rc) return rc;
    double *dp = nullptr, *df = nullptr, *part = nullptr, *res = nullptr;
    int* bad = nullptr;
    if ((rc = upload_vec(ctx, p, g->n, &dp))) return rc;
    int blocks = aux_grid(g);
    GN_CUDA(cudaMallocAsync((void**)&df, sizeof(double) * (size_t)std::max<int64_t>(g->n, 1), ctx.s));
    GN_CUDA(cudaMallocAsync((void**)&part, sizeof(double) * (size_t)blocks, ctx.s));
    GN_CUDA(cudaMallocAsync((void**)&res, sizeof(double), ctx.s));
    GN_CUDA(cudaMallocAsync((void**)&bad, sizeof(int), ctx.s));
    GN_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), ctx.s));
    k_fitness<<<blocks, kAuxThreads, 0, ctx.s>>>(g->n, g->rowptr, g->col, g->w64, dp, gamma, df, bad, part);
    GN_LAUNCHED();
    k_final_sum<1><<<1, 32, 0, ctx.s>>>(part, blocks, res);
    GN_LAUNCHED();
    int hbad = 0;
    GN_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, ctx.s));
    GN_CUDA(cudaMemcpyAsync(fbar, res, sizeof(double), cudaMemcpyDeviceToHost, ctx.s));
    if (g->n > 0)
        GN_CUDA(cudaMemcpyAsync(f_out, df, sizeof(double) * (size_t)g->n, cudaMemcpyDeviceToHost, ctx.s));
    cudaFreeAsync(dp, ctx.s);
    cudaFreeAsync(df, ctx.s);
    cudaFreeAsync(part, ctx.s);
    cudaFreeAsync(res, ctx.s);
    cudaFreeAsync(bad, ctx.s);
    GN_CUDA(cudaStreamSynchronize(ctx.s));
    if (hbad) return fail(GN_ERR_ZERO_DENOM, "zero denominator in fitness: state not normalizable");
    return GN_OK;
}

}  // extern "C"
