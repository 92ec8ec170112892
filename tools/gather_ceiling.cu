// gather_ceiling.cu -- what random gathers can reach on this B200 (no graph,
// no arithmetic beyond a sum): the ceiling the GN step's neighbour gathers
// are measured against ("What bounds the gathers").
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o exp/gather_ceiling tools/gather_ceiling.cu
//   exp/gather_ceiling            (one JSON line per case)
//
// Cases (every lane issues U independent loads before summing them; the
// addresses come from a hash of (thread, step), so no index stream is read):
//   global  : random 4- or 8-byte loads over a table of T bytes in HBM
//             (T <= 64 MB stays in the 126 MB L2; 1 GB does not) -- one
//             32-byte L2 sector per load, ~0 L1 hits
//   smem    : random 8-byte loads from a 192 KB shared-memory table (1 CTA
//             of 1024 threads per SM)
//   dsmem   : random 8-byte loads from the shared memory of the CTAs of a
//             cluster (8 or 16 CTAs of 1024 threads, 192 KB each)
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

namespace cg = cooperative_groups;

#define CK(x)                                                                                \
    do {                                                                                     \
        cudaError_t e_ = (x);                                                                \
        if (e_ != cudaSuccess) {                                                             \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            exit(1);                                                                         \
        }                                                                                    \
    } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352dU;
    x ^= x >> 15;
    x *= 0x846ca68bU;
    x ^= x >> 16;
    return x;
}

template <typename T, int U>
__global__ void k_global(const T* __restrict__ tab, uint32_t mask, int steps, double* out) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    double s = 0.0;
    for (int st = 0; st < steps; ++st) {
        T y[U];
#pragma unroll
        for (int u = 0; u < U; ++u) y[u] = __ldg(tab + (hash32(tid * 7919u + (uint32_t)(st * U + u) * 2654435761u) & mask));
#pragma unroll
        for (int u = 0; u < U; ++u) s += (double)y[u];
    }
    if (s == -1.0) out[0] = s;
}

constexpr int kSmemEntries = 24576;  // 192 KB of fp64

template <int U>
__global__ void __launch_bounds__(1024, 1) k_smem(const double* __restrict__ tab, int steps, double* out) {
    extern __shared__ double sh[];
    for (int i = threadIdx.x; i < kSmemEntries; i += blockDim.x) sh[i] = tab[i];
    __syncthreads();
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    double s = 0.0;
    for (int st = 0; st < steps; ++st) {
        double y[U];
#pragma unroll
        for (int u = 0; u < U; ++u) y[u] = sh[hash32(tid * 7919u + (uint32_t)(st * U + u) * 2654435761u) % kSmemEntries];
#pragma unroll
        for (int u = 0; u < U; ++u) s += y[u];
    }
    if (s == -1.0) out[0] = s;
}

template <int U>
__global__ void __launch_bounds__(1024, 1) k_dsmem(const double* __restrict__ tab, int steps, double* out) {
    extern __shared__ double sh[];
    cg::cluster_group cl = cg::this_cluster();
    for (int i = threadIdx.x; i < kSmemEntries; i += blockDim.x) sh[i] = tab[i];
    cl.sync();
    const uint32_t csz = cl.num_blocks();
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    double s = 0.0;
    for (int st = 0; st < steps; ++st) {
        double y[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t h = hash32(tid * 7919u + (uint32_t)(st * U + u) * 2654435761u);
            const double* p = cl.map_shared_rank(sh, h % csz);
            y[u] = p[(h >> 8) % kSmemEntries];
        }
#pragma unroll
        for (int u = 0; u < U; ++u) s += y[u];
    }
    cl.sync();
    if (s == -1.0) out[0] = s;
}

static float time_ms(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, a, b));
    return ms;
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    double* out;
    CK(cudaMalloc(&out, 8));
    const size_t big = (size_t)1 << 30;
    void* tab;
    CK(cudaMalloc(&tab, big));
    CK(cudaMemset(tab, 0, big));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    constexpr int U = 16;
    const int steps = 64;
    // global: 8 CTAs of 256 threads per SM (enough loads in flight)
    for (int bytes : {4, 8}) {
        for (size_t T : {(size_t)4 << 20, (size_t)32 << 20, (size_t)64 << 20, (size_t)1 << 30}) {
            const uint32_t mask = (uint32_t)(T / bytes - 1);
            const int grid = sms * 8, block = 256;
            auto launch = [&]() {
                if (bytes == 4) k_global<float, U><<<grid, block>>>((const float*)tab, mask, steps, out);
                else k_global<double, U><<<grid, block>>>((const double*)tab, mask, steps, out);
            };
            launch();
            CK(cudaDeviceSynchronize());
            CK(cudaEventRecord(e0));
            for (int r = 0; r < 5; ++r) launch();
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            const double ms = time_ms(e0, e1) / 5;
            const double loads = (double)grid * block * steps * U;
            printf("{\"case\": \"global\", \"bytes\": %d, \"table_mb\": %zu, \"ms\": %.4f, \"gloads_per_s\": %.1f, "
                   "\"per_sm_per_cycle_at_1965\": %.3f}\n",
                   bytes, T >> 20, ms, loads / ms / 1e6, loads / (ms * 1e-3) / sms / 1.965e9);
        }
    }
    const int smem = kSmemEntries * 8;
    CK(cudaFuncSetAttribute(k_smem<U>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    {
        auto launch = [&]() { k_smem<U><<<sms, 1024, smem>>>((const double*)tab, steps, out); };
        launch();
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0));
        for (int r = 0; r < 5; ++r) launch();
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        const double ms = time_ms(e0, e1) / 5;
        const double loads = (double)sms * 1024 * steps * U;
        printf("{\"case\": \"smem\", \"bytes\": 8, \"table_kb\": 192, \"ms\": %.4f, \"gloads_per_s\": %.1f, "
               "\"per_sm_per_cycle_at_1965\": %.3f}\n",
               ms, loads / ms / 1e6, loads / (ms * 1e-3) / sms / 1.965e9);
    }
    CK(cudaFuncSetAttribute(k_dsmem<U>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaFuncSetAttribute(k_dsmem<U>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    for (int csz : {2, 4, 8, 16}) {
        const int grid = sms / csz * csz;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(1024);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = csz;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, k_dsmem<U>, &cfg) != cudaSuccess || ncl == 0) {
            cudaGetLastError();
            printf("{\"case\": \"dsmem\", \"cluster\": %d, \"unavailable\": true}\n", csz);
            continue;
        }
        cfg.gridDim = dim3(ncl * csz);
        auto launch = [&]() { CK(cudaLaunchKernelEx(&cfg, k_dsmem<U>, (const double*)tab, steps, out)); };
        launch();
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0));
        for (int r = 0; r < 5; ++r) launch();
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        const double ms = time_ms(e0, e1) / 5;
        const double loads = (double)ncl * csz * 1024 * steps * U;
        printf("{\"case\": \"dsmem\", \"cluster\": %d, \"active_clusters\": %d, \"bytes\": 8, \"ms\": %.4f, "
               "\"gloads_per_s\": %.1f, \"per_sm_per_cycle_at_1965\": %.3f}\n",
               csz, ncl, ms, loads / ms / 1e6, loads / (ms * 1e-3) / (ncl * csz) / 1.965e9);
    }
    return 0;
}
