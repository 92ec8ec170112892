// gn_internal.cuh -- shared device/host internals of the GN engine (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/gn_b200.h"

namespace gn {

// dynamics.py:21-22
constexpr double kSafeDiv = 1e-9;
constexpr double kFallback = 0.5;

constexpr int kMaxBins = 8;
constexpr int kLoopThreads = 512;  // persistent loop block size

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what, const char* file, int line);
void note_launch(int64_t k = 1);

#define GN_CUDA(expr)                                                      \
    do {                                                                   \
        cudaError_t _e = (expr);                                           \
        if (_e != cudaSuccess) return ::gn::cuda_fail(_e, #expr, __FILE__, __LINE__); \
    } while (0)

#define GN_LAUNCHED()                                                      \
    do {                                                                   \
        cudaError_t _e = cudaGetLastError();                               \
        if (_e != cudaSuccess) return ::gn::cuda_fail(_e, "kernel launch", __FILE__, __LINE__); \
        ::gn::note_launch();                                               \
    } while (0)

// ---------------------------------------------------------------- graph
// A degree bin: rows [off, off+count) of the bin row list, processed by
// groups of G lanes per row (G = 1..32) or by a whole block per row (G = 0).
struct Bin {
    int32_t off;
    int32_t count;
    int32_t G;
    int32_t pad;
};

struct Plan {
    int nbins = 0;
    Bin bins[kMaxBins];
    int32_t* rows = nullptr;  // device row list (nullptr => identity order)
};

}  // namespace gn

struct gn_graph {
    int64_t n = 0;
    int64_t nnz = 0;
    int dtype = GN_F64;
    int device = 0;
    int num_sms = 0;
    int grid_override = 0;
    int64_t device_bytes = 0;
    int32_t* rowptr = nullptr;  // n+1 (nnz < 2^31 enforced)
    int32_t* col = nullptr;     // nnz
    void* v = nullptr;          // n, dtype: sqrt(w)
    void* w = nullptr;          // n, dtype
    double* w64 = nullptr;      // n fp64 (rounding priorities, MIS weight)
    gn::Plan fast;              // degree-binned plan
    gn::Plan exact;             // one thread per row, identity order
    int32_t max_degree = 0;
};

namespace gn {

// RAII stream + event helper for one API call.
struct CallCtx {
    cudaStream_t s = nullptr;
    int prev_dev = -1;
    int dev = 0;
    int open(int device);
    ~CallCtx();
};

// device-side helpers shared by the kernels
template <typename T>
struct Arith;

template <>
struct Arith<double> {
    __device__ static __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
    __device__ static __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
    __device__ static __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
    __device__ static __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
};

template <>
struct Arith<float> {
    __device__ static __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
    __device__ static __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
    __device__ static __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
    __device__ static __forceinline__ float div(float a, float b) { return __fdiv_rn(a, b); }
};

// Grid-wide barrier for a co-resident (cooperative) grid.  `target` grows
// monotonically: barrier number b waits for (b+1)*gridDim.x arrivals.  The
// gpu-scope fences make every y/x write of the previous phase visible (and
// invalidate the SM's L1) before any block reads them.
__device__ __forceinline__ void grid_barrier(unsigned int* counter, unsigned int target) {
    __syncthreads();
    if (gridDim.x > 1) {
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(counter, 1u);
            unsigned int seen;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(counter) : "memory");
            } while (seen < target);
            __threadfence();
        }
        __syncthreads();
    }
}

int coresident_blocks(const void* kernel, int threads, size_t smem, int device, int* out);

}  // namespace gn
