// gn_graph.cu -- graph upload, degree binning, error plumbing and the fp64
// auxiliary operators (SpMV, normalisability, energy, mass, simplex, fitness).
//
// Reference: graph.py:22-75 (WeightedGraph), dynamics.py:122-126,210-250.
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <mutex>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
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
    // per-call workspaces come from the device's default pool: keep what it
    // has mapped instead of returning it to the driver at every sync
    static std::once_flag pool_once[64];
    if (device >= 0 && device < 64)
        std::call_once(pool_once[device], [device]() {
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
                uint64_t keep = UINT64_MAX;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
            }
            cudaGetLastError();
        });
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

// Host-side layout of the loop structures (see gn_graph in gn_internal.cuh).
struct Layout {
    std::vector<int32_t> perm, inv;
    int32_t nhub = 0, nslices = 0, nsplit = 0;
    std::vector<int64_t> slice_ptr;
    std::vector<int32_t> row_deg;
    std::vector<int32_t> hub_ptr, hub_col;
    std::vector<int32_t> sell32, sell32s;   // sell32s / hub_cols: rows in ascending new id (fast mode)
    std::vector<uint16_t> sell16;
    std::vector<int32_t> hub_cols;
    int idx16 = 0;
    int sentinel = 0;  // 1: padding positions hold id n (a vertex whose published value is always 0)
    int32_t maxdeg = 0;
    std::vector<uint64_t> sig;  // per slice: MinHash of the 128-byte lines it gathers
};

static inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// Fast-mode copies of the int32-id adjacency (sell32s, hub_cols): every row's
// neighbours in ascending NEW id.  With the degree order of the relabeling the
// lanes of a warp then gather their hottest neighbours at the same positions,
// from the same few lines (C5 scale 24: 1.84 -> 1.75 ms/iteration).  The sum
// order changes, so EXACT runs keep the reference-order arrays.
static void build_sorted_copies(int64_t n, int B, Layout& L) {
    L.sell32s = L.sell32;
    L.hub_cols = L.hub_col;
    const int64_t nreg = n - L.nhub;
    const int nt = std::max(1, std::min(32, (int)std::thread::hardware_concurrency()));
    auto work = [&](int t) {
        std::vector<int32_t> buf;
        for (int32_t h = t; h < L.nhub; h += nt)
            std::sort(L.hub_cols.begin() + L.hub_ptr[h], L.hub_cols.begin() + L.hub_ptr[h + 1]);
        for (int32_t s = t; s < L.nslices; s += nt)
            for (int l = 0; l < kSlice; ++l) {
                const int64_t r = (int64_t)s * kSlice + l;
                if (r >= nreg) continue;
                const int d = L.row_deg[(size_t)r];
                auto at = [&](int q) { return L.slice_ptr[s] + (q / B) * (kSlice * B) + (int64_t)l * B + q % B; };
                buf.resize((size_t)d);
                for (int q = 0; q < d; ++q) buf[(size_t)q] = L.sell32s[(size_t)at(q)];
                std::sort(buf.begin(), buf.end());
                for (int q = 0; q < d; ++q) L.sell32s[(size_t)at(q)] = buf[(size_t)q];
            }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < nt; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
}

static void build_layout(int64_t n, const int64_t* indptr, const int32_t* indices, bool global_sort, Layout& L) {
    std::vector<int32_t> deg((size_t)n);
    for (int64_t i = 0; i < n; ++i) {
        deg[(size_t)i] = (int32_t)(indptr[i + 1] - indptr[i]);
        L.maxdeg = std::max(L.maxdeg, deg[(size_t)i]);
    }
    // hubs: degree-descending (stable)
    std::vector<int32_t> hubs, regular;
    for (int64_t i = 0; i < n; ++i) (deg[(size_t)i] > kHubDegree ? hubs : regular).push_back((int32_t)i);
    std::stable_sort(hubs.begin(), hubs.end(), [&](int32_t a, int32_t b) { return deg[a] > deg[b]; });
    // regular rows: degree-descending inside windows of kSigma (keeps coarse
    // locality; a uniform-degree graph keeps its numbering) -- or globally,
    // when the hot-vertex cache is on, so the smallest new ids (the cached
    // ones) are the most gathered vertices
    size_t win = global_sort ? std::max<size_t>(regular.size(), 1) : (size_t)kSigma;
    // skewed degrees on an int32-id graph (power-law: BA, R-MAT): one global
    // degree order, so the most gathered vertices share cache lines
    if (n > 65536 && L.maxdeg > 8 * std::max<int64_t>(1, indptr[n] / std::max<int64_t>(n, 1)))
        win = std::max<size_t>(regular.size(), 1);
    if (const char* e = getenv("GN_SORT_WINDOW")) {
        long long wv = atoll(e);
        win = wv <= 0 ? std::max<size_t>(regular.size(), 1) : (size_t)wv;
    }
    for (size_t w0 = 0; w0 < regular.size(); w0 += win) {
        size_t w1 = std::min(regular.size(), w0 + win);
        std::stable_sort(regular.begin() + w0, regular.begin() + w1,
                         [&](int32_t a, int32_t b) { return deg[a] > deg[b]; });
    }
    // skewed int32-id graphs: rows of equal degree ordered by their two
    // hottest neighbours (smallest provisional new ids), so the lanes of a
    // slice gather the same lines at the same positions (C3 12.06 -> 11.50
    // us/iteration, C5 scale 24 1742 -> 1716; GN_LEX=0 turns it off)
    const char* lex_env = getenv("GN_LEX");
    if (win == std::max<size_t>(regular.size(), 1) && n > 65536 && (!lex_env || atoi(lex_env))) {
        std::vector<int32_t> pinv((size_t)n);
        for (size_t q = 0; q < hubs.size(); ++q) pinv[(size_t)hubs[q]] = (int32_t)q;
        for (size_t q = 0; q < regular.size(); ++q) pinv[(size_t)regular[q]] = (int32_t)(hubs.size() + q);
        // runs of equal degree (regular is degree-descending)
        std::vector<std::pair<size_t, size_t>> runs;
        for (size_t q = 0; q < regular.size();) {
            size_t e = q;
            while (e < regular.size() && deg[regular[e]] == deg[regular[q]]) ++e;
            runs.push_back({q, e});
            q = e;
        }
        std::sort(runs.begin(), runs.end(), [](const std::pair<size_t, size_t>& a, const std::pair<size_t, size_t>& b) {
            return a.second - a.first > b.second - b.first;
        });
        std::atomic<size_t> next{0};
        auto work = [&]() {
            std::vector<std::pair<uint64_t, int32_t>> kv;
            for (size_t ri; (ri = next.fetch_add(1)) < runs.size();) {
                const size_t q0 = runs[ri].first, q1 = runs[ri].second;
                kv.resize(q1 - q0);
                for (size_t q = q0; q < q1; ++q) {
                    const int32_t r = regular[q];
                    uint32_t a = ~0u, b = ~0u;
                    for (int64_t p = indptr[r]; p < indptr[r + 1]; ++p) {
                        const uint32_t v = (uint32_t)pinv[(size_t)indices[p]];
                        if (v < a) { b = a; a = v; } else if (v < b) b = v;
                    }
                    kv[q - q0] = {((uint64_t)a << 32) | b, r};
                }
                std::sort(kv.begin(), kv.end());
                for (size_t q = q0; q < q1; ++q) regular[q] = kv[q - q0].second;
            }
        };
        const int nt = std::max(1, std::min(32, (int)std::thread::hardware_concurrency()));
        std::vector<std::thread> th;
        for (int t = 1; t < nt; ++t) th.emplace_back(work);
        work();
        for (auto& x : th) x.join();
    }
    // groups of 32 rows; long groups (split over warps) first, the partial
    // tail group always last
    const size_t ng = (regular.size() + kSlice - 1) / kSlice;
    std::vector<int32_t> split_g, whole_g;
    for (size_t gi = 0; gi < ng; ++gi) {
        size_t r0 = gi * kSlice, r1 = std::min(regular.size(), r0 + (size_t)kSlice);
        int32_t len = 0;
        for (size_t r = r0; r < r1; ++r) len = std::max(len, deg[regular[r]]);
        bool full = (r1 - r0) == (size_t)kSlice;
        (full && len >= kSplitLen ? split_g : whole_g).push_back((int32_t)gi);
    }
    // long slices by length, longest first: the loop deals them out zigzag
    std::vector<int32_t> glen(ng, 0);
    for (size_t gi = 0; gi < ng; ++gi)
        for (size_t r = gi * kSlice; r < std::min(regular.size(), (gi + 1) * (size_t)kSlice); ++r)
            glen[gi] = std::max(glen[gi], deg[regular[r]]);
    std::stable_sort(split_g.begin(), split_g.end(), [&](int32_t a, int32_t b) { return glen[a] > glen[b]; });
    L.nhub = (int32_t)hubs.size();
    L.nsplit = (int32_t)split_g.size();
    L.nslices = (int32_t)ng;
    L.perm.clear();
    L.perm.reserve((size_t)n);
    L.perm.insert(L.perm.end(), hubs.begin(), hubs.end());
    std::vector<int32_t> order = split_g;
    order.insert(order.end(), whole_g.begin(), whole_g.end());
    for (int32_t gi : order) {
        size_t r0 = (size_t)gi * kSlice, r1 = std::min(regular.size(), r0 + (size_t)kSlice);
        for (size_t r = r0; r < r1; ++r) L.perm.push_back(regular[r]);
    }
    L.inv.assign((size_t)n, 0);
    for (int64_t r = 0; r < n; ++r) L.inv[(size_t)L.perm[(size_t)r]] = (int32_t)r;

    // hub CSR in new ids, original neighbour order
    L.hub_ptr.assign((size_t)L.nhub + 1, 0);
    for (int32_t h = 0; h < L.nhub; ++h) L.hub_ptr[h + 1] = L.hub_ptr[h] + deg[L.perm[h]];
    L.hub_col.resize((size_t)L.hub_ptr[L.nhub]);
    for (int32_t h = 0; h < L.nhub; ++h) {
        int32_t o = L.perm[h];
        for (int64_t p = indptr[o]; p < indptr[o + 1]; ++p) L.hub_col[(size_t)(L.hub_ptr[h] + (p - indptr[o]))] = L.inv[indices[p]];
    }
    // SELL slices, position-major
    const int64_t nreg = n - L.nhub;
    L.idx16 = n <= 65536 ? 1 : 0;
    const int B = L.idx16 ? 8 : 4;  // positions per 16-byte lane vector
    L.row_deg.assign((size_t)std::max<int64_t>(nreg, 0), 0);
    L.slice_ptr.assign((size_t)L.nslices + 1, 0);
    for (int32_t s = 0; s < L.nslices; ++s) {
        int32_t len = 0;
        for (int l = 0; l < kSlice; ++l) {
            int64_t r = (int64_t)s * kSlice + l;
            if (r < nreg) {
                int32_t d = deg[L.perm[(size_t)(L.nhub + r)]];
                L.row_deg[(size_t)r] = d;
                len = std::max(len, d);
            }
        }
        len = (len + B - 1) / B * B;
        L.slice_ptr[s + 1] = L.slice_ptr[s] + (int64_t)len * kSlice;
    }
    // MinHash over the 128-byte lines (16 fp64 ids) a slice gathers: slices
    // with overlapping neighbourhoods get equal signatures w.p. = Jaccard, and
    // the plan places equal signatures on the same SM so its L1 serves them
    // computed for the uint16-id graphs (small: cheap, and their dense rows
    // reuse neighbourhoods -- C2 -2.5%); GN_PLAN_COLOCATE=1/0 forces it on/off
    const char* colo = getenv("GN_PLAN_COLOCATE");
    const bool want_sig = colo ? colo[0] == '1' : n <= 65536;
    L.sig.assign(want_sig ? (size_t)L.nslices : 0, ~0ull);
    for (int32_t s = 0; s < (int32_t)L.sig.size(); ++s) {
        uint64_t m = ~0ull;
        for (int l = 0; l < kSlice; ++l) {
            int64_t r = (int64_t)s * kSlice + l;
            if (r >= nreg) continue;
            int32_t o = L.perm[(size_t)(L.nhub + r)];
            for (int64_t p = indptr[o]; p < indptr[o + 1]; ++p) m = std::min(m, mix64((uint64_t)(L.inv[indices[p]] >> 4)));
        }
        L.sig[(size_t)s] = m;
    }
    const int64_t elems = L.slice_ptr[L.nslices];
    // int32 ids: padding is id n, the zero-valued dummy vertex, so a lane runs
    // its slice's full length without degree masks (adding +0.0 leaves a sum's
    // bits unchanged).  uint16 layouts keep the degree masks (the id n may not
    // fit, and on their dense rows the masks are rare)
    L.sentinel = L.idx16 ? 0 : 1;
    if (L.idx16) L.sell16.assign((size_t)elems, L.sentinel ? (uint16_t)n : (uint16_t)0);
    else L.sell32.assign((size_t)elems, L.sentinel ? (int32_t)n : 0);
    for (int32_t s = 0; s < L.nslices; ++s) {
        for (int l = 0; l < kSlice; ++l) {
            int64_t r = (int64_t)s * kSlice + l;
            if (r >= nreg) continue;
            int32_t o = L.perm[(size_t)(L.nhub + r)];
            for (int64_t p = indptr[o]; p < indptr[o + 1]; ++p) {
                // block-major: block p/B holds 32 lanes x B consecutive positions
                const int64_t q = p - indptr[o];
                int64_t at = L.slice_ptr[s] + (q / B) * (kSlice * B) + (int64_t)l * B + q % B;
                int32_t nid = L.inv[indices[p]];
                if (L.idx16) L.sell16[(size_t)at] = (uint16_t)nid;
                else L.sell32[(size_t)at] = nid;
            }
        }
    }
    if (!L.idx16 && !getenv("GN_NO_SORTED")) build_sorted_copies(n, B, L);
}

template <typename T>
__global__ void k_init_state_weights(int64_t n, const double* __restrict__ w64, const int32_t* __restrict__ perm,
                                     T* __restrict__ v, T* __restrict__ w) {
    int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r < n) {
        double wi = w64[perm[r]];
        v[r] = (T)sqrt(wi);  // graph.py:42 (IEEE sqrt; binary32: rounding of the fp64 root)
        w[r] = (T)wi;
    }
}

static void free_graph(gn_graph* g) {
    if (!g) return;
    release_plans(g);
    release_multi_plans(g);
    if (g->resident) batch_destroy(g->resident);
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(g->device);
    void* ptrs[] = {g->rowptr, g->col, g->w64, g->perm, g->inv, g->v, g->w,
                    g->hub_ptr, g->hub_col, g->slice_ptr, g->row_deg, g->sell, g->sell_fast, g->hub_col_fast};
    for (void* p : ptrs) cudaFree(p);
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

int gn_graph_create(int64_t n, const int64_t* indptr, const int32_t* indices, const double* w, int dtype,
                    int device, gn_graph** out) {
    GN_NVTX("gn_graph_create");
    *out = nullptr;
    if (n < 0) return fail(GN_ERR_ARG, "vertex count must be nonnegative");
    if (!valid_dtype(dtype)) return fail(GN_ERR_ARG, "dtype must be GN_F64, GN_F32 or GN_F32_PURE");
    if (n > 0 && (!indptr || !w)) return fail(GN_ERR_ARG, "null graph array");
    const int64_t nnz = n > 0 ? indptr[n] : 0;
    if (nnz >= (int64_t(1) << 31) || n >= (int64_t(1) << 31))
        return fail(GN_ERR_ARG, "graphs with >= 2^31 adjacency entries need the partitioned engine");
    if (n > 0 && indptr[0] != 0) return fail(GN_ERR_ARG, "indptr[0] must be 0");
    for (int64_t i = 0; i < n; ++i)
        if (indptr[i + 1] < indptr[i]) return fail(GN_ERR_ARG, "indptr must be nondecreasing");
    for (int64_t p = 0; p < nnz; ++p)
        if (indices[p] < 0 || indices[p] >= n) return fail(GN_ERR_ARG, "column index outside [0,n)");

    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(GN_ERR_NODEV, "no CUDA device visible: the GN engine has no CPU fallback");
    }
    if (device < 0 || device >= ndev) return fail(GN_ERR_ARG, "device ordinal out of range");

    // hot-vertex cache: for large graphs the values of the first `hot` new ids
    // (the most gathered vertices) are mirrored in shared memory each
    // iteration (128 KB); GN_HOT=0 disables it
    const int64_t hot_cap = (int64_t)(131072 / gather_bytes(dtype));
    // opt-in (GN_HOT=1): measured slower on C3 and C5 scale 24 -- the per-
    // iteration mirror and the smaller L1 outweigh the saved L1 wavefronts
    int64_t hot = 0;
    if (const char* e = getenv("GN_HOT")) hot = (atoi(e) && n >= 8 * hot_cap) ? hot_cap : 0;
    Layout L;
    build_layout(n, indptr, indices, hot > 0, L);

    gn_graph* g = new gn_graph();
    g->n = n;
    g->nnz = nnz;
    g->dtype = dtype;
    g->device = device;
    g->max_degree = L.maxdeg;
    g->nhub = L.nhub;
    while (g->ngiant < L.nhub && indptr[L.perm[g->ngiant] + 1] - indptr[L.perm[g->ngiant]] > kGiantRow) ++g->ngiant;
    g->nslices = L.nslices;
    g->nsplit = L.nsplit;
    g->idx16 = L.idx16;
    g->sell_elems = L.slice_ptr.empty() ? 0 : L.slice_ptr.back();
    g->slice_sig = std::move(L.sig);
    g->hot = L.idx16 ? 0 : (int32_t)hot;
    CallCtx ctx;
    int rc = ctx.open(device);
    if (rc) { delete g; return rc; }
    cudaDeviceGetAttribute(&g->num_sms, cudaDevAttrMultiProcessorCount, device);

    std::vector<int32_t> rowptr32((size_t)n + 1);
    for (int64_t i = 0; i <= n; ++i) rowptr32[(size_t)i] = (int32_t)(n > 0 ? indptr[i] : 0);

    const size_t es = state_bytes(dtype);
    const size_t nb = (size_t)std::max<int64_t>(n, 1);
    int64_t bytes = 0;
    auto cleanup = [&](int code) { free_graph(g); return code; };
#define GN_TRY(expr)                                                              \
    do {                                                                          \
        cudaError_t _e = (expr);                                                  \
        if (_e != cudaSuccess) return cleanup(cuda_fail(_e, #expr, __FILE__, __LINE__)); \
    } while (0)
#define GN_UP(dst, src, count, type)                                                              \
    do {                                                                                          \
        size_t _b = sizeof(type) * (size_t)std::max<int64_t>((int64_t)(count), 1);                \
        GN_TRY(cudaMalloc((void**)&(dst), _b));                                                   \
        bytes += (int64_t)_b;                                                                     \
        if ((count) > 0)                                                                          \
            GN_TRY(cudaMemcpyAsync((dst), (src), sizeof(type) * (size_t)(count), cudaMemcpyHostToDevice, ctx.s)); \
    } while (0)
    GN_UP(g->rowptr, rowptr32.data(), n + 1, int32_t);
    GN_UP(g->col, indices, nnz, int32_t);
    GN_UP(g->w64, w, n, double);
    GN_UP(g->perm, L.perm.data(), n, int32_t);
    GN_UP(g->inv, L.inv.data(), n, int32_t);
    GN_UP(g->hub_ptr, L.hub_ptr.data(), L.nhub + 1, int32_t);
    GN_UP(g->hub_col, L.hub_col.data(), (int64_t)L.hub_col.size(), int32_t);
    GN_UP(g->slice_ptr, L.slice_ptr.data(), (int64_t)L.slice_ptr.size(), int64_t);
    GN_UP(g->row_deg, L.row_deg.data(), (int64_t)L.row_deg.size(), int32_t);
    if (L.idx16) {
        uint16_t* p = nullptr;
        GN_UP(p, L.sell16.data(), (int64_t)L.sell16.size(), uint16_t);
        g->sell = p;
    } else {
        int32_t* p = nullptr;
        GN_UP(p, L.sell32.data(), (int64_t)L.sell32.size(), int32_t);
        g->sell = p;
        if (!L.sell32s.empty()) {
            GN_UP(p, L.sell32s.data(), (int64_t)L.sell32s.size(), int32_t);
            g->sell_fast = p;
            GN_UP(g->hub_col_fast, L.hub_cols.data(), (int64_t)L.hub_cols.size(), int32_t);
        }
    }
    GN_TRY(cudaMalloc(&g->v, es * nb));
    GN_TRY(cudaMalloc(&g->w, es * nb));
    bytes += (int64_t)(2 * es * nb);
    g->device_bytes = bytes;
    if (n > 0) {
        int blocks = grid_for(n, 256);
        if (es == 8)
            k_init_state_weights<double><<<blocks, 256, 0, ctx.s>>>(n, g->w64, g->perm, (double*)g->v, (double*)g->w);
        else
            k_init_state_weights<float><<<blocks, 256, 0, ctx.s>>>(n, g->w64, g->perm, (float*)g->v, (float*)g->w);
        GN_TRY(cudaGetLastError());
        note_launch();
    }
    GN_TRY(cudaStreamSynchronize(ctx.s));
#undef GN_TRY
#undef GN_UP
    // small graphs also get the shared-memory-resident (CTA-per-graph) layout
    if (n > 0 && n <= 4096 && !getenv("GN_NO_RESIDENT")) {
        const int64_t offs[2] = {0, n};
        gn_batch* r = nullptr;
        if (batch_create(1, offs, n, indptr, indices, w, dtype, device, &r) == GN_OK) {
            int max_optin = 0;
            cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
            if (batch_smem_bytes(r) + 4096 <= (size_t)max_optin) g->resident = r;
            else batch_destroy(r);
        }
        set_error("");
    }
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
    if (num_bins) *num_bins = g->nsplit;
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
    GN_NVTX("gn_is_normalizable");
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
    GN_NVTX("gn_energy");
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
