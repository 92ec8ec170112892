// Grid-barrier latency micro-benchmark (development aid): one co-resident CTA
// per SM, R back-to-back barriers, ns per barrier for several protocols.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o exp/barrier_bench tools/barrier_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// 0: red.release + relaxed poll of the counter + fence.acq_rel (the engine's)
// 1: red.release + acquire poll of the counter
// 2: atom.acq_rel returns the arrival number; the last arriver bumps a flag
//    on its own 128-byte line; the others poll the flag (acquire)
// 3: as 2 with a relaxed poll + fence.acq_rel
// 4: two-level: groups of 8 CTAs arrive on per-group counters; each group's
//    last arriver arrives on the top counter; the last of those bumps the flag
template <int MODE>
__global__ void k_bar(unsigned* ws, int reps, long long* out) {
    unsigned* counter = ws;        // line 0
    unsigned* flag = ws + 32;      // line 1
    unsigned* top = ws + 64;       // line 2
    unsigned* groups = ws + 96;    // lines 3.. (one per group)
    const unsigned G = gridDim.x;
    long long t0 = clock64();
    for (int r = 1; r <= reps; ++r) {
        __syncthreads();
        if (threadIdx.x == 0) {
            if (MODE == 0 || MODE == 1) {
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(counter) : "memory");
                const unsigned target = (unsigned)r * G;
                if (MODE == 0) {
                    while (ld_relaxed(counter) < target) {}
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");
                } else {
                    while (ld_acquire(counter) < target) {}
                }
            } else if (MODE == 2 || MODE == 3) {
                unsigned old;
                asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(counter) : "memory");
                if (old == (unsigned)r * G - 1) {
                    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flag), "r"((unsigned)r) : "memory");
                } else if (MODE == 2) {
                    while (ld_acquire(flag) < (unsigned)r) {}
                } else {
                    while (ld_relaxed(flag) < (unsigned)r) {}
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");
                }
            } else {
                const unsigned g = blockIdx.x / 8, gsz = min(8u, G - g * 8), ng = (G + 7) / 8;
                unsigned old;
                asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(groups + 32 * g) : "memory");
                bool released = false;
                if (old == (unsigned)r * gsz - 1) {
                    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(top) : "memory");
                    if (old == (unsigned)r * ng - 1) {
                        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flag), "r"((unsigned)r) : "memory");
                        released = true;
                    }
                }
                if (!released) while (ld_acquire(flag) < (unsigned)r) {}
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}

template <int MODE>
static void run(int G, int threads, int reps, unsigned* ws, long long* out) {
    cudaMemset(ws, 0, 4096 * sizeof(unsigned));
    void* args[] = {&ws, &reps, &out};
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    // warm
    cudaLaunchCooperativeKernel((void*)k_bar<MODE>, G, threads, args, 0, 0);
    cudaMemset(ws, 0, 4096 * sizeof(unsigned));
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)k_bar<MODE>, G, threads, args, 0, 0);
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("mode %d grid %d threads %d: %.1f ns per barrier (%s)\n", MODE, G, threads, ms * 1e6 / reps,
           cudaGetErrorString(e));
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned* ws;
    long long* out;
    cudaMalloc(&ws, 4096 * sizeof(unsigned));
    cudaMalloc(&out, 4096 * sizeof(long long));
    const int reps = 20000;
    for (int t : {512}) {
        run<0>(sms, t, reps, ws, out);
        run<1>(sms, t, reps, ws, out);
        run<2>(sms, t, reps, ws, out);
        run<3>(sms, t, reps, ws, out);
        run<4>(sms, t, reps, ws, out);
        run<0>(sms, t, reps, ws, out);
        run<2>(sms, t, reps, ws, out);
    }
    return 0;
}
