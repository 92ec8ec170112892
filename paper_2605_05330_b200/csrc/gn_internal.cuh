// gn_internal.cuh -- shared device/host internals of the GN engine (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <nvtx3/nvToolsExt.h>

#include <string>
#include <vector>

#include "../../include/gn_b200.h"

namespace gn {

// dynamics.py:21-22
constexpr double kSafeDiv = 1e-9;
constexpr double kFallback = 0.5;

constexpr int kSlice = 32;         // SELL slice height (one row per lane)
constexpr int kSigma = 4096;       // degree-sort window of the relabeling
constexpr int kHubDegree = 512;    // rows above this are processed CTA-wide
constexpr int kGiantRow = 32768;   // x0 checks: rows above this get a CTA each
constexpr int kSplitLen = 64;      // slices at least this long are split over warps

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what, const char* file, int line);
void note_launch(int64_t k = 1);

// NVTX range over one ABI call (header-only NVTX3: a no-op unless a tool
// such as nsys / ncu --nvtx is attached), named after the ABI entry point.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};
#define GN_NVTX(name) ::gn::NvtxRange gn_nvtx_range_(name)

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

// ---------------------------------------------------------------- dtypes
// GN_F64:      state, sums and gathered values in binary64 (the reference)
// GN_F32:      state and sums in binary64, gathered values (the y each vertex
//              publishes to its neighbours) in binary32 -- halves the gather
//              bytes and keeps every vertex's own trajectory in fp64 range
// GN_F32_PURE: binary32 throughout
inline bool valid_dtype(int d) { return d == GN_F64 || d == GN_F32 || d == GN_F32_PURE; }
inline size_t state_bytes(int d) { return d == GN_F32_PURE ? 4 : 8; }
inline size_t gather_bytes(int d) { return d == GN_F64 ? 8 : 4; }

}  // namespace gn

// Device-resident graph.  Two copies of the adjacency:
//  * the original CSR (ids as the caller numbered them) for rounding, the
//    checks and the auxiliary fp64 operators;
//  * the loop layout: vertices relabeled (new id r, perm[r] = old id) so that
//    hub rows come first and the remaining rows, degree-sorted in windows of
//    kSigma, form SELL slices of 32 rows.  A slice is stored in blocks of B
//    positions (B = 8 for uint16 ids, 4 for int32): block b holds, lane after
//    lane, the B consecutive neighbours of each of the 32 rows, so one lane
//    fetches B indices with one 16-byte load and a warp's loads of a block
//    cover 512 contiguous bytes.  One thread sums its row in the reference's
//    sequential order.
struct gn_graph {
    int64_t n = 0;
    int64_t nnz = 0;
    int dtype = GN_F64;
    int device = 0;
    int num_sms = 0;
    int grid_override = 0;
    int64_t device_bytes = 0;
    int32_t max_degree = 0;

    // original CSR
    int32_t* rowptr = nullptr;
    int32_t* col = nullptr;
    double* w64 = nullptr;

    // loop layout
    int32_t* perm = nullptr;  // new -> old
    int32_t* inv = nullptr;   // old -> new
    void* v = nullptr;        // sqrt(w) in state precision, new-id order
    void* w = nullptr;        // w in state precision, new-id order
    int32_t nhub = 0;         // rows [0, nhub) are hubs
    int32_t ngiant = 0;       // hubs [0, ngiant) have more than kGiantRow neighbours
    int32_t* hub_ptr = nullptr;  // nhub+1, offsets into hub_col
    int32_t* hub_col = nullptr;  // new ids, original neighbour order
    int32_t nslices = 0;      // rows [nhub, n) in slices of 32
    int32_t nsplit = 0;       // slices [0, nsplit) have length >= kSplitLen
    int64_t* slice_ptr = nullptr;  // nslices+1 element offsets (multiples of 32*B)
    int32_t* row_deg = nullptr;    // degree per slice row (n - nhub)
    void* sell = nullptr;          // int32 or uint16 new ids, position-major
    void* sell_fast = nullptr;     // int32 ids only: rows in ascending new id (fast mode; null: use sell)
    int32_t* hub_col_fast = nullptr;  // the same for hub_col
    int idx16 = 0;                 // 1: sell holds uint16 ids (n <= 65536); else int32 ids, padding = id n
    int64_t sell_elems = 0;
    std::vector<uint64_t> slice_sig;  // host: per-slice MinHash (gn_graph.cu, used by the plan)
    gn_batch* resident = nullptr;     // small graphs: the whole-graph-in-shared-memory kernel
    int32_t hot = 0;                  // new ids [0, hot) are mirrored in shared memory (0: off)
};

namespace gn {

// RAII stream for one API call.
struct CallCtx {
    cudaStream_t s = nullptr;
    int prev_dev = -1;
    int dev = 0;
    int open(int device);
    ~CallCtx();
};

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
// monotonically: barrier number b waits for b*gridDim.x arrivals.  The
// gpu-scope fences publish every x/y write of the phase (and invalidate the
// SM's L1) before any block reads them.
__device__ __forceinline__ void grid_barrier(unsigned int* counter, unsigned int target) {
    __syncthreads();
    if (gridDim.x > 1) {
        if (threadIdx.x == 0) {
            // release: the block's writes (ordered before us by bar.sync) reach
            // gpu scope before the arrival; the arrival itself returns nothing
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(counter) : "memory");
            unsigned int seen;
            do {
                asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(counter) : "memory");
            } while (seen < target);
            asm volatile("fence.acq_rel.gpu;" ::: "memory");  // acquire (invalidates this SM's L1)
        }
        __syncthreads();
    }
}

// The same barrier in two halves, so a CTA can do barrier-independent work
// (loads of static data and of its own rows) while the others arrive.
__device__ __forceinline__ void grid_arrive(unsigned int* counter) {
    __syncthreads();
    if (gridDim.x > 1 && threadIdx.x == 0)
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(counter) : "memory");
}

__device__ __forceinline__ void grid_wait(unsigned int* counter, unsigned int target) {
    if (gridDim.x > 1) {
        if (threadIdx.x == 0) {
            unsigned int seen;
            do {
                asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(counter) : "memory");
            } while (seen < target);
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
        __syncthreads();
    }
}

int coresident_blocks(const void* kernel, int threads, size_t smem, int device, int* out);
void release_plans(const gn_graph* g);  // gn_loop.cu: cached launch plans of g
// gn_loop.cu: the x0 checks of dynamics.py:146-149 on x (original order) into flags[0..1]
int enqueue_precheck(const gn_graph* g, const double* x, int* flags, cudaStream_t s);
void release_multi_plans(const gn_graph* g);  // gn_multi.cu: cached multi-start plans of g

// gn_batch.cu: the resident (CTA-per-graph) kernel
int batch_create(int64_t B, const int64_t* offsets, int64_t n, const int64_t* indptr, const int32_t* indices,
                 const double* w, int dtype, int device, gn_batch** out);
void batch_destroy(gn_batch* b);
size_t batch_smem_bytes(const gn_batch* b);
int batch_run(gn_batch* b, const void* x0, const double* gammas, int iters, double final_gamma, uint32_t flags,
              void* x_out, double* step_inf, int64_t* fallbacks, double* mass, double* energy, double* pre_energy,
              double* x_hist, int* iters_run, int* status, int* fail_iter, gn_run_stats* stats);

}  // namespace gn
