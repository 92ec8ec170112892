// gn_gen.cu -- R-MAT graph generation on the device (SURVEY.md 8f row f2:
// ingestion at scale), for BASELINE config C5 (scale 24, edge factor 16:
// 2^28 samples).  The random stream is counter based and identical to
// generators.rmat_pairs (numpy), so small scales are checked bit for bit on
// the CPU: level l of sample e draws u = splitmix64(seed * 2^40 + e * 64 + l),
// top 53 bits / 2^53; quadrant by (a, a+b, a+b+c).  Self-loops are dropped,
// the graph is symmetrised and deduplicated with two radix sorts of 64-bit
// keys, and the canonical CSR (rows sorted ascending) is built on the device.
#include <cuda_runtime.h>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "gn_internal.cuh"

namespace gn {

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void k_rmat_keys(int64_t ne, int scale, double a, double ab, double abc, uint64_t base,
                            uint64_t* __restrict__ keys) {
    const uint64_t n = 1ull << scale;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne; e += (int64_t)gridDim.x * blockDim.x) {
        uint64_t s = 0, d = 0;
        for (int l = 0; l < scale; ++l) {
            const uint64_t h = splitmix64(base + (uint64_t)e * 64ull + (uint64_t)l);
            const double u = (double)(h >> 11) * (1.0 / 9007199254740992.0);
            const uint64_t rb = u >= ab ? 1 : 0;
            const uint64_t cb = ((u >= a) && (u < ab)) || (u >= abc) ? 1 : 0;
            s = (s << 1) | rb;
            d = (d << 1) | cb;
        }
        const uint64_t lo = s < d ? s : d, hi = s < d ? d : s;
        keys[e] = s == d ? ~0ull : lo * n + hi;  // undirected key; self-loops sort last
    }
}

// Edge list -> undirected keys (min * n + max); the first edge (input order)
// that leaves [0, n) or is a self-loop is recorded (graph.py:98-108).
__global__ void k_edge_keys(int64_t m, uint64_t n, const int64_t* __restrict__ u, const int64_t* __restrict__ v,
                            uint64_t* __restrict__ keys, unsigned long long* __restrict__ first_bad) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = u[e], b = v[e];
        if (a < 0 || b < 0 || (uint64_t)a >= n || (uint64_t)b >= n || a == b) {
            atomicMin(first_bad, (unsigned long long)e);
            keys[e] = 0;
            continue;
        }
        const uint64_t lo = a < b ? a : b, hi = a < b ? b : a;
        keys[e] = lo * n + hi;
    }
}

// unique undirected key -> both directed keys (row * n + col)
__global__ void k_symmetrize(int64_t m, uint64_t n, const uint64_t* __restrict__ ukeys, uint64_t* __restrict__ dkeys) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = ukeys[i], lo = k / n, hi = k % n;
        dkeys[2 * i] = lo * n + hi;
        dkeys[2 * i + 1] = hi * n + lo;
    }
}

__global__ void k_csr(int64_t nnz, uint64_t n, const uint64_t* __restrict__ keys, int64_t* __restrict__ indptr,
                      int32_t* __restrict__ col) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = keys[i], r = k / n;
        col[i] = (int32_t)(k % n);
        const uint64_t prev = i ? keys[i - 1] / n : ~0ull;
        if (i == 0 || prev != r) {
            // rows (prev, r] start here
            const uint64_t first = i == 0 ? 0 : prev + 1;
            for (uint64_t q = first; q <= r; ++q) indptr[q] = i;
        }
        if (i == nnz - 1)
            for (uint64_t q = r + 1; q <= n; ++q) indptr[q] = nnz;
    }
}

// Undirected edge keys (k0, ne of them, device; freed here) -> canonical
// CSR on the host: sort, unique, drop the self-loop marker ~0, symmetrise,
// sort again, row pointers.  *indptr_out / *indices_out are malloc'd.
static int keys_to_csr(cudaStream_t s, uint64_t n, uint64_t* k0, int64_t ne, int64_t* nnz_out,
                       int64_t** indptr_out, int32_t** indices_out) {
    uint64_t *k1 = nullptr, *d0 = nullptr, *d1 = nullptr;
    int64_t* dcount = nullptr;
    int64_t* dindptr = nullptr;
    int32_t* dcol = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0, t2 = 0;
    auto cleanup = [&]() {
        void* ptrs[] = {k0, k1, d0, d1, dcount, tmp, dindptr, dcol};
        for (void* p : ptrs)
            if (p) cudaFree(p);
    };
#define GN_G(expr)                                                                  \
    do {                                                                            \
        cudaError_t _e = (expr);                                                    \
        if (_e != cudaSuccess) {                                                    \
            cleanup();                                                              \
            return cuda_fail(_e, #expr, __FILE__, __LINE__);                        \
        }                                                                           \
    } while (0)
    const int threads = 256, blocks = 148 * 16;
    int bits = 1;
    while (bits < 64 && (n * n) >> bits) ++bits;  // keys < n^2 (plus the marker ~0)
    GN_G(cudaMalloc(&k1, 8 * (size_t)std::max<int64_t>(ne, 1)));
    GN_G(cudaMalloc(&dcount, 8));
    GN_G(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, k0, k1, ne, 0, 64, s));
    GN_G(cub::DeviceSelect::Unique(nullptr, t2, k1, k0, dcount, ne, s));
    tmp_bytes = std::max(tmp_bytes, t2);
    GN_G(cudaMalloc(&tmp, std::max<size_t>(tmp_bytes, 16)));
    int64_t nu = 0;
    if (ne > 0) {
        GN_G(cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, k0, k1, ne, 0, 64, s));
        note_launch();
        GN_G(cub::DeviceSelect::Unique(tmp, tmp_bytes, k1, k0, dcount, ne, s));
        note_launch();
        GN_G(cudaMemcpyAsync(&nu, dcount, 8, cudaMemcpyDeviceToHost, s));
        GN_G(cudaStreamSynchronize(s));
        // the self-loop marker ~0 sorts last: drop it
        if (nu > 0) {
            uint64_t last = 0;
            GN_G(cudaMemcpy(&last, k0 + (nu - 1), 8, cudaMemcpyDeviceToHost));
            if (last == ~0ull) --nu;
        }
    }
    cudaFree(k1);
    k1 = nullptr;
    const int64_t nnz = 2 * nu;
    GN_G(cudaMalloc(&d0, 8 * (size_t)std::max<int64_t>(nnz, 1)));
    GN_G(cudaMalloc(&d1, 8 * (size_t)std::max<int64_t>(nnz, 1)));
    if (nu > 0) {
        k_symmetrize<<<blocks, threads, 0, s>>>(nu, n, k0, d0);
        GN_G(cudaGetLastError());
        note_launch();
        size_t t3 = 0;
        GN_G(cub::DeviceRadixSort::SortKeys(nullptr, t3, d0, d1, nnz, 0, bits, s));
        if (t3 > tmp_bytes) {
            cudaFree(tmp);
            tmp = nullptr;
            tmp_bytes = t3;
            GN_G(cudaMalloc(&tmp, tmp_bytes));
        }
        GN_G(cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, d0, d1, nnz, 0, bits, s));
        note_launch();
    }
    cudaFree(k0);
    k0 = nullptr;
    cudaFree(d0);
    d0 = nullptr;
    GN_G(cudaMalloc(&dindptr, 8 * ((size_t)n + 1)));
    GN_G(cudaMalloc(&dcol, 4 * (size_t)std::max<int64_t>(nnz, 1)));
    if (nnz > 0) {
        k_csr<<<blocks, threads, 0, s>>>(nnz, n, d1, dindptr, dcol);
        GN_G(cudaGetLastError());
        note_launch();
    } else {
        GN_G(cudaMemsetAsync(dindptr, 0, 8 * ((size_t)n + 1), s));
    }
    int64_t* hptr = (int64_t*)malloc(8 * ((size_t)n + 1));
    int32_t* hcol = (int32_t*)malloc(4 * (size_t)std::max<int64_t>(nnz, 1));
    if (!hptr || !hcol) {
        free(hptr);
        free(hcol);
        cleanup();
        return fail(GN_ERR_NOMEM, "host allocation for the CSR failed");
    }
    cudaError_t e1 = cudaMemcpyAsync(hptr, dindptr, 8 * ((size_t)n + 1), cudaMemcpyDeviceToHost, s);
    cudaError_t e2 = nnz ? cudaMemcpyAsync(hcol, dcol, 4 * (size_t)nnz, cudaMemcpyDeviceToHost, s) : cudaSuccess;
    cudaError_t e3 = cudaStreamSynchronize(s);
    cleanup();
#undef GN_G
    if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess) {
        free(hptr);
        free(hcol);
        return cuda_fail(e1 != cudaSuccess ? e1 : (e2 != cudaSuccess ? e2 : e3), "copy out", __FILE__, __LINE__);
    }
    *nnz_out = nnz;
    *indptr_out = hptr;
    *indices_out = hcol;
    return GN_OK;
}

}  // namespace gn

using namespace gn;

extern "C" {

int gn_gen_rmat(int scale, int edge_factor, double a, double b, double c, uint64_t seed, int device,
                int64_t* nnz_out, int64_t** indptr_out, int32_t** indices_out) {
    GN_NVTX("gn_gen_rmat");
    *nnz_out = 0;
    *indptr_out = nullptr;
    *indices_out = nullptr;
    if (scale < 1 || scale > 30 || edge_factor < 1) return fail(GN_ERR_ARG, "bad R-MAT parameters");
    CallCtx ctx;
    int rc = ctx.open(device);
    if (rc) return rc;
    const uint64_t n = 1ull << scale;
    const int64_t ne = (int64_t)n * edge_factor;
    uint64_t* k0 = nullptr;
    GN_CUDA(cudaMalloc(&k0, 8 * (size_t)ne));
    k_rmat_keys<<<148 * 16, 256, 0, ctx.s>>>(ne, scale, a, a + b, a + b + c, seed << 40, k0);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        cudaFree(k0);
        return cuda_fail(e, "k_rmat_keys", __FILE__, __LINE__);
    }
    note_launch();
    return keys_to_csr(ctx.s, n, k0, ne, nnz_out, indptr_out, indices_out);
}

int gn_csr_from_edges(int64_t n, int64_t m, const int64_t* u, const int64_t* v, int device, int64_t* first_bad,
                      int64_t* nnz_out, int64_t** indptr_out, int32_t** indices_out) {
    GN_NVTX("gn_csr_from_edges");
    *nnz_out = 0;
    *indptr_out = nullptr;
    *indices_out = nullptr;
    if (first_bad) *first_bad = -1;
    if (n < 0 || m < 0 || (m > 0 && (!u || !v))) return fail(GN_ERR_ARG, "bad edge list");
    if (n >= (int64_t(1) << 31)) return fail(GN_ERR_ARG, "vertex count must be below 2^31");
    if (n == 0) {  // no vertex: any edge is out of range
        if (m > 0) {
            if (first_bad) *first_bad = 0;
            return fail(GN_ERR_ARG, "edge endpoint out of range");
        }
        *indptr_out = (int64_t*)calloc(1, 8);
        *indices_out = (int32_t*)calloc(1, 4);
        return (*indptr_out && *indices_out) ? GN_OK : fail(GN_ERR_NOMEM, "host allocation failed");
    }
    CallCtx ctx;
    int rc = ctx.open(device);
    if (rc) return rc;
    cudaStream_t s = ctx.s;
    int64_t *du = nullptr, *dv = nullptr;
    uint64_t* k0 = nullptr;
    unsigned long long* dbad = nullptr;
    auto release = [&]() {
        void* ptrs[] = {du, dv, dbad};
        for (void* p : ptrs)
            if (p) cudaFree(p);
    };
    cudaError_t e;
    const size_t mb = 8 * (size_t)std::max<int64_t>(m, 1);
    if ((e = cudaMalloc(&du, mb)) != cudaSuccess || (e = cudaMalloc(&dv, mb)) != cudaSuccess ||
        (e = cudaMalloc(&k0, mb)) != cudaSuccess || (e = cudaMalloc(&dbad, 8)) != cudaSuccess) {
        release();
        if (k0) cudaFree(k0);
        return cuda_fail(e, "cudaMalloc", __FILE__, __LINE__);
    }
    unsigned long long none = ~0ull;
    cudaMemcpyAsync(dbad, &none, 8, cudaMemcpyHostToDevice, s);
    if (m > 0) {
        cudaMemcpyAsync(du, u, 8 * (size_t)m, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(dv, v, 8 * (size_t)m, cudaMemcpyHostToDevice, s);
        k_edge_keys<<<148 * 16, 256, 0, s>>>(m, (uint64_t)std::max<int64_t>(n, 1), du, dv, k0, dbad);
        note_launch();
    }
    unsigned long long hbad = none;
    cudaMemcpyAsync(&hbad, dbad, 8, cudaMemcpyDeviceToHost, s);
    e = cudaStreamSynchronize(s);
    release();
    if (e != cudaSuccess) {
        cudaFree(k0);
        return cuda_fail(e, "edge keys", __FILE__, __LINE__);
    }
    if (hbad != none) {  // graph.py:101-106: the caller reports the first offending edge
        cudaFree(k0);
        if (first_bad) *first_bad = (int64_t)hbad;
        return fail(GN_ERR_ARG, "edge endpoint out of range or self-loop");
    }
    return keys_to_csr(s, (uint64_t)std::max<int64_t>(n, 1), k0, m, nnz_out, indptr_out, indices_out);
}

void gn_free_host(void* p) { free(p); }

}  // extern "C"
