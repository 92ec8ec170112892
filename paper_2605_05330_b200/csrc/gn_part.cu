// gn_part.cu -- one vertex-range partition of a graph too large for one GPU
// (BASELINE config C5): the owned rows' GN steps, with the
// published values of ghost vertices supplied by a halo exchange between
// iterations.
//
// Local numbering: owned vertices [0, n_own) (in the caller's order), ghosts
// [n_own, n_own + n_ghost) grouped by owning peer.  Neighbour lists keep the
// reference's order (ascending global id), so each owned row sums exactly as
// the unpartitioned graph does and a partitioned run equals the single-GPU
// run bit for bit.
//
// Per iteration k, on the caller's stream: gn_part_step (sums + updates of the
// owned rows -- one thread per row in degree order, sequential sums; in fast
// mode the longest rows split over a warp -- with per-block fixed-order stats
// partials), then gn_part_pack (owned values -> contiguous send buffers), the
// exchange (NCCL grouped send/recv, issued by the caller on the same stream),
// gn_part_unpack (receive buffers -> ghost slots).  gn_part_end folds the
// per-iteration stats in block order.
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <limits>
#include <thread>
#include <tuple>
#include <vector>

#include "gn_internal.cuh"

struct gn_part {
    int64_t n_own = 0, n_ghost = 0, nnz = 0;
    int dtype = GN_F64;
    int device = 0;
    int32_t* rowptr = nullptr;  // n_own+1
    int32_t* col = nullptr;     // local ids
    // owned rows in processing order: the boundary rows (those peers hold as
    // ghosts) first, then the interior; each range degree-descending (stable)
    int32_t* order = nullptr;
    std::vector<int32_t> h_rowptr;  // caller's local numbering
    std::vector<double> h_w;        // n_own + n_ghost, caller's numbering
    // owned rows are relabeled to their processing position (boundary range
    // first, each range degree-descending): a row's state, weight and output
    // are then read and written contiguously.  perm: new -> caller's id, inv:
    // caller's -> new; ghosts keep their ids.  rowptr/col/w64 hold the
    // relabeled graph (neighbour order unchanged: bitwise sums).
    int32_t* perm = nullptr;
    int32_t* inv = nullptr;
    std::vector<int32_t> h_inv;     // host copy of inv
    std::vector<int32_t> h_col;     // host copy of col (the SELL is rebuilt by gn_part_set_boundary)
    int64_t n_bnd = 0;              // order[0, n_bnd): boundary rows
    // blocked SELL of the rows after each range's long prefix: slices of 32
    // consecutive order positions, block b of a slice holds, lane after lane,
    // positions 4b..4b+3 of each row (one 16-byte load per lane, 512
    // contiguous bytes per warp); padding names the zero-valued slot n_all
    int32_t* sell = nullptr;
    int32_t* sell_fast = nullptr;   // fast mode: every row in ascending new id (hot neighbours first)
    int32_t* col_fast = nullptr;
    int64_t* slice_ptr = nullptr;   // [nslices+1] element offsets
    int64_t sl0[2] = {0, 0}, nsl[2] = {0, 0};  // per range: first slice, slice count
    int64_t long_fast[2] = {0, 0};  // per range: leading rows above long_degree
    int long_degree = 512;          // set by part_order
    // settled isolated rows: the last n_iso interior rows (see part_order);
    // fast-mode steps from iteration 3 on walk only the first iso_nsl slices
    // of the interior range and add iso_mass (the skipped rows' w . 1) to
    // the objective
    int64_t n_iso = 0, iso_nsl = -1;
    double iso_mass[2] = {0.0, 0.0};  // [binary64 state, binary32 state]
    // fast mode: the long rows of each range cut into pieces of kPiece
    // adjacency entries (fixed sizes: the sum tree, and every bit, is the
    // same on any grid).  Piece j covers col[pc_beg[j], pc_end[j]); long row
    // q of range r owns pieces [lp[lp0[r] + q], lp[lp0[r] + q + 1]).  Warps
    // sum pieces into pc_sum; k_part_long_combine adds a row's pieces in
    // piece order and updates the row.
    int32_t* pc_beg = nullptr;
    int32_t* pc_end = nullptr;
    int32_t* pc_order = nullptr;  // pieces by their first column, per range (GN_PIECE_SORT)
    int piece_blocked = 0;
    int interleave = 1;           // GN_PART_INTERLEAVE=0: long-row blocks first
    // chunk mode (default; GN_PART_CHUNK=len, 0 = off): the long rows' pieces (chunks) summed one
    // thread per chunk over a blocked SELL of chunks -- 32 chunks per slice,
    // sorted by (length, first column) -- instead of one warp per piece; the
    // chunk sums go to their pc_sum slots (cslot), combined as pieces
    // Chunks whose consecutive ids differ by < 65536 are stored as 16-bit
    // deltas (8 per lane per 16-byte vector, the lane's first id in cbase,
    // its length in clen), the others as int32 ids (4 per vector, padded
    // with the zero-valued slot nall); cfmt marks each slice (GN_PART_DELTA=0:
    // all int32)
    int chunk = 0;
    int32_t* csell = nullptr;        // slices' vectors (uint4), offsets in cslice_ptr (in vectors)
    int64_t* cslice_ptr = nullptr;
    int32_t* cslot = nullptr;
    int8_t* cfmt = nullptr;          // per slice: 1 = 16-bit deltas
    int32_t* cbase = nullptr;        // [slices * 32] first id of the lane's chunk
    int32_t* clen = nullptr;         // [slices * 32] its length
    int64_t cg0[2] = {0, 0}, ncg[2] = {0, 0};
    // zero-row certificates (every mode; GN_PART_WITNESS=0: off).  A row
    // whose state is exactly 0 has y_i = +-0 and stays y_i/d = +-0 for any d =
    // y_i + gamma*s > 1e-9.  Its neighbour sum is a sum of non-negative terms,
    // monotone in every addend in any fixed order and precision, so s >= y_j
    // for each neighbour j: one neighbour ("witness") with y_i + gamma*y_j >
    // 1e-9 settles the row bit for bit without its walk (the update runs with
    // s = y_j: the same d > 1e-9 test, the same +-0).  Rows whose witness
    // fails walk as before and are queued; k_part_witness then picks the
    // neighbour of largest y as the new witness.
    int witness = 1;
    int32_t* wit = nullptr;      // [n_own] witness per row (local id), -1 none
    int32_t* rq = nullptr;       // [n_own] rows queued for a witness (one range's step at a time)
    int* rq_cnt = nullptr;       // [2 * iters] queue length per (iteration, range)
    int32_t* crow = nullptr;     // chunk mode: [ncg * 32] the (new) row of the lane's chunk, -1 empty
    unsigned long long* gat = nullptr;  // [iters * 64] gathers issued (GN_PART_COUNT=1: counted; measurement)
    int gat_on = 0;
    // settled rows (with the certificates; GN_PART_SETTLE=0: off).  A member
    // row m -- state exactly 1, every neighbour an owned row whose state is
    // exactly 0, gmin[k]*y_m > 1e-9 for the smallest gamma still to come --
    // is a fixed point together with its neighbours: m computes s = 0, d =
    // v_m, x' = v_m/v_m = 1; each neighbour z has y_z = 0 and d_z >= gamma*y_m
    // > 1e-9, x_z' = 0; by induction for every later iteration.  Such rows
    // (frz 2), and the zero rows whose witness is one (frz 1), hold the same
    // value in both state and both published buffers and are skipped: no
    // loads but the flag, no stores; a member adds its w to the objective in
    // the same place of the same sum.  Member candidates (state 1, walked sum
    // exactly 0) are queued by the step; k_part_settle, after both ranges,
    // checks the new states of their neighbours.
    int settle = 1;
    uint8_t* frz = nullptr;      // [n_own] 0 active, 1 settled zero row, 2 settled member row
    int32_t* mq = nullptr;       // [n_own] member candidates of one iteration
    int* mq_cnt = nullptr;       // [iters] their count
    double* gmin = nullptr;      // [iters] min gamma over [k, iters) (0 when one of them is not finite and positive)
    int32_t* lp = nullptr;
    double* pc_sum = nullptr;
    double* pc_max = nullptr;    // chunk mode: per chunk, an uncertified zero row's largest gathered value
    int32_t* pc_arg = nullptr;   // and its id (the witness search rides on the walk)
    int64_t pc0[2] = {0, 0}, npc[2] = {0, 0}, lp0[2] = {0, 0};
    int r_ncomb[2] = {0, 0};                 // per range: combine blocks
    double* part_long[2] = {nullptr, nullptr};  // per range [iters][r_ncomb][4]
    // per range (0 boundary, 1 interior), set by gn_part_begin
    int64_t r_start[2] = {0, 0}, r_count[2] = {0, 0}, r_long[2] = {0, 0}, r_csr[2] = {0, 0};
    int r_nbl[2] = {0, 0}, r_ncb[2] = {0, 0}, r_nblocks[2] = {0, 0};
    double* w64 = nullptr;      // n_own + n_ghost
    // run state
    int iters = 0;
    uint32_t flags = 0;
    void* x[2] = {nullptr, nullptr};   // state precision, n_own
    void* yg[2] = {nullptr, nullptr};  // gathered precision, n_own + n_ghost
    void* v = nullptr;                 // state precision, n_own + n_ghost
    double* gam = nullptr;
    double* part[2] = {nullptr, nullptr};  // per range [iters][r_nblocks][4]: max|dx|, fallbacks, w.x', non-finite
    cudaStream_t own_stream = nullptr;
    // direct halo over peer memory (gn_part_peer_*): the boundary step stores
    // each published value straight into the ghost slots of the peers that
    // hold it (NVLink P2P stores, issued as the rows finish), then flags them
    int me = 0, parts = 0;
    int64_t* inflags = nullptr;              // [parts] incoming: inflags[q] = (epoch << 32) + steps peer q has pushed
    int32_t* expect = nullptr;               // peers that push to this part
    int nexpect = 0;
    struct Peer { int rank; void* yg[2]; int64_t* flags; };
    std::vector<Peer> peers;
    std::vector<int32_t> h_push_row, h_push_peer;
    std::vector<int64_t> h_push_slot;
    // the push list, sorted by (peer, ghost slot): entry e copies the owned
    // value push_src[e] into slot push_slot[e] of peer push_peer[e], so the
    // threads of a warp write 32 consecutive slots of one peer (coalesced
    // 128-byte NVLink writes)
    int32_t* push_src = nullptr;
    int32_t* push_peer = nullptr;
    int64_t* push_slot = nullptr;
    int64_t n_push = 0;
    void** push_dst[2] = {nullptr, nullptr}; // per parity: the peers' yg buffers
    int64_t** peer_flags = nullptr;          // the peers' flag arrays
    int* halo_bad = nullptr;                 // set when a peer's flag did not arrive in time
    int npush_peers = 0;
    // run epoch: incremented by every gn_part_begin (all parts of a run call it
    // the same number of times); flag values carry it in their high 32 bits,
    // so a late flag of an earlier run can never satisfy a wait of this one
    int64_t epoch = 0;
    int64_t* d_epoch = nullptr;
    // run buffers are kept across runs while their sizes do not change (their
    // addresses are exported to the peers over CUDA IPC)
    int64_t alloc_nall = -1;
    int alloc_dtype = -1, alloc_iters = 0, alloc_nblocks[2] = {0, 0}, alloc_ncomb[2] = {0, 0};
    // device-side schedule (gn_part_run): the iterations' launches captured
    // once into a CUDA graph, rebuilt when `gen` (buffers, push list) moves
    uint64_t gen = 1, g_gen = 0;
    int g_k0 = -1, g_k1 = -1;
    int64_t g_nodes = 0;
    cudaGraphExec_t gexec = nullptr;
    // host <-> device staging kept across runs: x0 in (caller's numbering)
    // and x out; the per-range stats of gn_part_end
    double* io = nullptr;
    int64_t io_n = 0;
    double* dout = nullptr;
    int64_t dout_n = 0;
};

namespace gn {

constexpr int kPartThreads = 256;

template <typename TS, typename TG>
__global__ void k_part_prepare(int64_t n_own, int64_t n_all, const double* __restrict__ x0,
                               const int32_t* __restrict__ perm, const double* __restrict__ w64,
                               TS* __restrict__ x, TS* __restrict__ v, TG* __restrict__ yg) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n_all) return;
    const TS vi = (TS)sqrt(w64[i]);  // graph.py:42
    const TS xi = (TS)x0[i < n_own ? (int64_t)perm[i] : i];  // x0 in the caller's numbering
    v[i] = vi;
    yg[i] = (TG)Arith<TS>::mul(vi, xi);
    if (i < n_own) x[i] = xi;
}

constexpr int kPartLongDegreeMin = 128, kPartLongDegreeMax = 1024;
constexpr int kCombRows = 8;  // long rows per warp of k_part_long_combine
constexpr int kSlicesPerWarp = 16;  // slice blocks: slices per warp (GN_PART_SPW; C5 scale 24: 1 / 4 / 16 / 64 -> 0.715 / 0.573 / 0.552 / 0.612 ms per iteration)
constexpr int kChunkDefault = 512;  // long-row chunk length (thread per chunk; 0: warp pieces)
constexpr int kPiece = 512;  // adjacency entries per long-row piece (fast mode; 2048: +3.5% time on C5)

// The long rows' pieces (fast mode; see gn_part::pc_beg)
struct PartLong {
    const int32_t* __restrict__ beg;
    const int32_t* __restrict__ end;
    double* __restrict__ sum;
    int64_t n;
    const int32_t* __restrict__ order;  // processing position -> piece (null: piece order)
    int blocked;                        // 1: each warp takes one contiguous run of positions
    int interleave;                     // 1: long-row blocks spread among the slice blocks
    const int32_t* __restrict__ csell;  // chunk mode: SELL of chunks (null: warp per piece)
    const int64_t* __restrict__ cslice_ptr;  // per slice: first vector (uint4 units)
    const int32_t* __restrict__ cslot;  // [ncg * 32] chunk -> its pc_sum slot (-1: empty lane)
    const int8_t* __restrict__ cfmt;    // per slice: 1 = 16-bit deltas
    const int32_t* __restrict__ cbase;  // [ncg * 32] first id (delta slices)
    const int32_t* __restrict__ clen;   // [ncg * 32] chunk length (delta slices)
    int64_t ncg;
    const int32_t* __restrict__ crow;   // [ncg * 32] the chunk's row (zero-row certificates)
    double* __restrict__ cmax;          // per slot (as sum): an uncertified zero row's chunk maximum; null: no tracking
    int32_t* __restrict__ carg;         // and the id that holds it (-1: every value 0)
};

// The zero-row certificates of one step launch (gn_part::witness); wit null: off
struct PartWit {
    const int32_t* __restrict__ wit;
    int32_t* __restrict__ rq;           // queue of rows without a certificate
    int* __restrict__ rqn;              // its length for this (iteration, range)
    unsigned long long* __restrict__ gat;  // null, or [64] gathers issued this iteration
    int cap;                            // queue capacity (n_own)
    int gat_mode;                       // what gat counts: 1 value gathers, 2 rows walked, 3 slices walked (slice path)
    uint8_t* frz;                       // settled rows (gn_part::frz); null: off
    int32_t* __restrict__ mq;           // member candidates
    int* __restrict__ mqn;              // their count this iteration
    const double* __restrict__ gfut;    // min gamma over this and the later iterations (device: the captured
                                        // schedule serves runs with other gammas)
};
#ifndef GN_PART_UNROLL
#define GN_PART_UNROLL 8
#endif
constexpr int kPartUnroll = GN_PART_UNROLL;  // gathers in flight per thread  // fast mode: longer rows are split over a warp

// Cache policy of the step's loads (compile-time A/B, GN_PART_HINT): 0 the
// default (__ldg); 1 the index stream read with L1::no_allocate and an L2
// evict-first policy (it is read once per iteration); 2 as 1, and the
// gathered values with an L2 evict-last policy; 3 the index stream evict-first
// in L2 only
#ifndef GN_PART_HINT
#define GN_PART_HINT 0
#endif
__device__ __forceinline__ uint64_t pol_first() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t pol_last() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint4 ld_idx4(const uint4* p) {
#if GN_PART_HINT == 1 || GN_PART_HINT == 2
    uint4 r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p), "l"(pol_first()));
    return r;
#elif GN_PART_HINT == 3
    uint4 r;
    asm("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p), "l"(pol_first()));
    return r;
#else
    return __ldg(p);
#endif
}
__device__ __forceinline__ int32_t ld_idx(const int32_t* p) {
#if GN_PART_HINT == 1 || GN_PART_HINT == 2
    int32_t r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol_first()));
    return r;
#elif GN_PART_HINT == 3
    int32_t r;
    asm("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol_first()));
    return r;
#else
    return __ldg(p);
#endif
}
template <typename TG>
__device__ __forceinline__ TG ld_val(const TG* p) {
#if GN_PART_HINT == 2
    if constexpr (sizeof(TG) == 8) {
        double r;
        asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(pol_last()));
        return (TG)r;
    } else {
        float r;
        asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(r) : "l"(p), "l"(pol_last()));
        return (TG)r;
    }
#else
    return __ldg(p);
#endif
}

// dynamics.py:104-107 for owned row i with neighbour sum s; stats of the thread
template <typename TS, typename TG>
__device__ __forceinline__ TS part_update_pre(int64_t i, TS s, TS g, TS xi, TS vi, double wi,
                                                TS* __restrict__ xo, TG* __restrict__ ygo, double& mx, double& fb,
                                                double& ob, double& nf) {
    using A = Arith<TS>;
    const TS yi = A::mul(vi, xi);
    const TS d = A::add(yi, A::mul(g, s));          // dynamics.py:105
    const bool ok = (double)d > kSafeDiv;            // dynamics.py:106
    const TS o = ok ? A::div(yi, d) : TS(kFallback); // dynamics.py:107
    xo[i] = o;
    ygo[i] = (TG)A::mul(vi, o);
    const TS dx = A::sub(o, xi);
    const double diff = (double)(dx < TS(0) ? -dx : dx);
    if (!(diff <= mx)) mx = diff;
    fb += ok ? 0.0 : 1.0;
    if (!isfinite((double)o)) nf = 1.0;
    ob = __dadd_rn(ob, __dmul_rn((double)(TS)wi, (double)o));
    return o;
}

// A settled member row's share of the objective: what part_update_pre adds
// for o = 1 (w*1 = w exactly), in the same place of the thread's sum
template <typename TS>
__device__ __forceinline__ void part_member_mass(double wi, double& ob) {
    ob = __dadd_rn(ob, (double)(TS)wi);
}

// After row i (state xi, walked neighbour sum s) was updated to o: a member
// candidate -- state exactly 1 before and after, neighbour sum exactly 0 (every
// published neighbour value is 0), and its published value keeps every
// neighbour's d above 1e-9 under the smallest gamma still to come -- is queued
// for k_part_settle, which looks at the neighbours' states.
template <typename TS, typename TG>
__device__ __forceinline__ void part_member_candidate(const PartWit& w, int64_t i, TS xi, TS s, TS o, TS vi, int k) {
    using A = Arith<TS>;
    if (!(xi == TS(1) && o == TS(1) && s == TS(0))) return;
    // every eighth iteration, staggered over the rows: a candidate whose
    // neighbours publish 0 but are not yet exactly 0 fails the check for many
    // iterations (with binary32 published values: from 1e-38 down to 5e-324),
    // and each check is a walk of the row
    if (((k + (int)i) & 7) != 0) return;
    const TS pub = (TS)(TG)A::mul(vi, o);
    if (!((double)A::mul((TS)*w.gfut, pub) > kSafeDiv)) return;
    const int e = atomicAdd(w.mqn, 1);
    if (e < w.cap) w.mq[e] = (int32_t)i;
}

// A certified zero row i whose witness wj is a settled member row is settled
// too (its d stays above 1e-9 by the member's own test); looked at every
// fourth iteration, staggered over the rows.  Otherwise the row rests (flag
// 3): this iteration's update writes its second 0, so both state and both
// published buffers hold 0 and, while its certificate holds, the row needs
// no state loaded and nothing stored -- only its witness's value tested.
__device__ __forceinline__ void part_settle_zero(const PartWit& w, int64_t i, int32_t wj, int k, unsigned fz) {
    if (((k + (int)i) & 3) == 0 && wj < w.cap && w.frz[wj] == 2) w.frz[i] = 1;
    else if (fz != 3) w.frz[i] = 3;
}

// A resting zero row (flag 3): x_i = 0 in both buffers, so its certificate
// is gamma*y_w > 1e-9 alone (d = 0 + gamma*s >= gamma*y_w)
template <typename TS, typename TG>
__device__ __forceinline__ bool part_resting_ok(TS g, int32_t wj, const TG* __restrict__ yg) {
    using A = Arith<TS>;
    if (wj < 0) return false;
    return (double)A::mul(g, (TS)ld_val(yg + wj)) > kSafeDiv;
}

// A zero row's certificate (gn_part::witness): x_i == 0 and its witness j
// gives y_i + g*y_j > 1e-9 -- then the row's own d = y_i + g*s passes the same
// test (s >= y_j) and its new state is y_i/d = y_i.  yw: y_j in the state
// precision, the row's stand-in neighbour sum.
template <typename TS, typename TG>
__device__ __forceinline__ bool part_certified(TS xi, TS vi, TS g, int32_t wj, const TG* __restrict__ yg, TS& yw) {
    using A = Arith<TS>;
    if (wj < 0) return false;
    yw = (TS)ld_val(yg + wj);
    return (double)A::add(A::mul(vi, xi), A::mul(g, yw)) > kSafeDiv;
}

__device__ __forceinline__ void part_enqueue(const PartWit& w, int64_t i) {
    const int e = atomicAdd(w.rqn, 1);
    if (e < w.cap) w.rq[e] = (int32_t)i;  // (a repeated launch of one step cannot overrun it)
}

// the same with the row's state, weight and v loaded here
template <typename TS, typename TG>
__device__ __forceinline__ void part_update(int64_t i, TS s, TS g, const double* __restrict__ w64,
                                            const TS* __restrict__ v, const TS* __restrict__ x, TS* __restrict__ xo,
                                            TG* __restrict__ ygo, double& mx, double& fb, double& ob, double& nf) {
    part_update_pre<TS, TG>(i, s, g, x[i], v[i], w64[i], xo, ygo, mx, fb, ob, nf);
}

// Direct halo: the interior step's first `nblocks` blocks copy the boundary
// rows' new values (written by the boundary step, the previous launch on the
// stream) into the peers' ghost slots while the other blocks step the
// interior rows -- the NVLink transfer overlaps the interior.  Entries are
// sorted by (peer, slot): consecutive threads store consecutive slots.
struct PartPush {
    const int32_t* __restrict__ src;   // new local ids of the pushed rows
    const int32_t* __restrict__ peer;
    const int64_t* __restrict__ slot;
    void* const* __restrict__ dst;     // [peers] the buffers this step writes (next parity)
    int64_t n;
    int nblocks;                       // 0: no pushes in this launch
};

// One step of the owned rows of one range.  Blocks [0, nbl) split the n_long
// longest rows over warps (lanes stride the positions, fixed butterfly fold:
// fast mode only); blocks [nbl, nbl + ncb) give one thread to each of the
// next n_csr rows (the long rows of an EXACT run) reading the CSR; the other
// blocks give one warp to each slice of the blocked SELL, one thread per row.
// Every thread-per-row sum is sequential in the reference's order (bitwise),
// with 8 gathers in flight and the next index vectors loading under them.
// 4 blocks of 256 threads per SM (64 registers, no spills): 32 warps to hide
// the gathers' latency (C5 scale 24: 1.71 -> 1.59 ms per iteration vs 3)
#ifndef GN_PART_MINB
#define GN_PART_MINB 4
#endif

// The arguments of one step launch over one range
template <typename TS, typename TG>
struct StepArgs {
    int64_t n_long;
    int nbl;
    int64_t n_csr;
    int ncb;
    int64_t count;
    const int32_t* __restrict__ order;
    const int32_t* __restrict__ rowptr;
    const int32_t* __restrict__ col;
    const int32_t* __restrict__ sell;
    const int64_t* __restrict__ slice_ptr;
    int64_t nsl;
    const double* __restrict__ w64;
    const TS* __restrict__ v;
    const TS* __restrict__ x;
    TS* __restrict__ xo;
    const TG* __restrict__ yg;
    TG* __restrict__ ygo;
    const double* __restrict__ gam;
    int k;
    double* __restrict__ part;
    PartPush push;
    PartLong lng;
    PartWit wt;
    int nvb;  // blocks (push blocks included)
};

// One lane's chunk of a long row (chunk mode): `my` index vectors of the
// chunks' SELL walked in ascending new id, 8 gathers in flight, the next
// vector loading under them; delta slices hold 16-bit gaps from id0 (8 entries
// per vector, `len` entries in all), the others int32 ids (4 per vector,
// padded with the zero-valued slot).  TRACK: also the largest value gathered
// and its id (the first such) -- the witness search of an uncertified zero
// row rides on the walk the row does anyway.
template <typename TS, typename TG, bool TRACK>
__device__ __forceinline__ TS part_chunk_walk(const uint4* __restrict__ base, const TG* __restrict__ yg, int my, int nblk,
                                              bool delta, int32_t id0, int len, TG& best, int32_t& barg) {
    using A = Arith<TS>;
    TS s = TS(0);
    if (delta) {
        int32_t id = id0;
        uint4 cv = my > 0 ? ld_idx4(base) : make_uint4(0, 0, 0, 0);
        for (int b = 0; b < nblk; ++b) {
            const uint4 nv = b + 1 < my ? ld_idx4(base + (size_t)(b + 1) * 32) : make_uint4(0, 0, 0, 0);
            const uint32_t w[4] = {cv.x, cv.y, cv.z, cv.w};
            TG y[8];
            int32_t ids[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                id += (int32_t)((w[j >> 1] >> (16 * (j & 1))) & 0xFFFFu);
                ids[j] = id;
                y[j] = 8 * b + j < len ? ld_val(yg + id) : TG(0);
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                s = A::add(s, (TS)y[j]);
                if (TRACK && y[j] > best) {
                    best = y[j];
                    barg = ids[j];
                }
            }
            cv = nv;
        }
    } else {
        constexpr int NV = kPartUnroll / 4;
        uint4 cv[NV];
#pragma unroll
        for (int u = 0; u < NV; ++u) cv[u] = u < my ? ld_idx4(base + (size_t)u * 32) : make_uint4(0, 0, 0, 0);
        for (int b = 0; b < nblk; b += NV) {
            uint4 nv[NV];
#pragma unroll
            for (int u = 0; u < NV; ++u)
                nv[u] = b + NV + u < my ? ld_idx4(base + (size_t)(b + NV + u) * 32) : make_uint4(0, 0, 0, 0);
            TG y[4 * NV];
#pragma unroll
            for (int u = 0; u < NV; ++u) {
                const bool in = b + u < my;
                y[4 * u + 0] = in ? ld_val(yg + cv[u].x) : TG(0);
                y[4 * u + 1] = in ? ld_val(yg + cv[u].y) : TG(0);
                y[4 * u + 2] = in ? ld_val(yg + cv[u].z) : TG(0);
                y[4 * u + 3] = in ? ld_val(yg + cv[u].w) : TG(0);
            }
#pragma unroll
            for (int q = 0; q < 4 * NV; ++q) {
                s = A::add(s, (TS)y[q]);
                if (TRACK && y[q] > best) {
                    best = y[q];
                    const uint4 c = cv[q >> 2];
                    barg = (int32_t)((q & 3) == 0 ? c.x : (q & 3) == 1 ? c.y : (q & 3) == 2 ? c.z : c.w);
                }
            }
#pragma unroll
            for (int u = 0; u < NV; ++u) cv[u] = nv[u];
        }
    }
    return s;
}

// One virtual block (256 threads) of a step over one range.  Blocks [0, nbl)
// split the n_long longest rows over warps (lanes stride the positions, fixed
// butterfly fold: fast mode only); blocks [nbl, nbl + ncb) give one thread to
// each of the next n_csr rows (the long rows of an EXACT run) reading the CSR;
// the other blocks give one warp to each slice of the blocked SELL, one thread
// per row.  Every thread-per-row sum is sequential in the reference's order
// (bitwise), with 8 gathers in flight and the next index vectors loading
// under them.
template <typename TS, typename TG>
__device__ __forceinline__ void part_step_vb(const StepArgs<TS, TG>& a, int vb, int tid, double (*red)[4]) {
    using A = Arith<TS>;
    const PartPush& push = a.push;
    const PartLong& lng = a.lng;
    const TG* __restrict__ yg = a.yg;
    const int32_t* __restrict__ col = a.col;
    if (vb < push.nblocks) {  // the halo blocks
        const int64_t stride = (int64_t)push.nblocks * kPartThreads;
        for (int64_t e = (int64_t)vb * kPartThreads + tid; e < push.n; e += stride)
            static_cast<TG*>(push.dst[__ldg(push.peer + e)])[__ldg(push.slot + e)] = a.ygo[__ldg(push.src + e)];
        return;
    }
    const int bid = vb - push.nblocks, nbid = a.nvb - push.nblocks;
    const int nbl = a.nbl, ncb = a.ncb;
    // the block's role: [0, nbl) long-row pieces, [nbl, nbl + ncb) CSR rows,
    // then slices.  In fast mode (no CSR blocks) the long-row blocks are
    // spread evenly among the slice blocks (lng.interleave), so the two
    // kinds -- L2-throughput-bound pieces, latency-bound slices -- run side by side
    int rb = bid;
    if (lng.interleave && ncb == 0 && nbl > 0) {
        const int before = (int)((int64_t)bid * nbl / nbid), upto = (int)((int64_t)(bid + 1) * nbl / nbid);
        rb = upto > before ? before : nbl + (bid - before);
    }
    const TS g = (TS)a.gam[a.k];
    const PartWit& wt = a.wt;
    const int lane = tid & 31, warp = tid >> 5;
    constexpr int kWarpsPerBlock = kPartThreads / 32;
    double mx = 0.0, fb = 0.0, ob = 0.0, nf = 0.0;
    unsigned long long ng = 0;  // gathers issued (GN_PART_COUNT)
    if (rb < nbl && lng.csell) {
        // long rows, chunk mode: one thread per chunk over the chunks' SELL
        // (sequential in ascending new id), the sum to the chunk's slot; the
        // chunks of a certified zero row are not walked (k_part_long_combine
        // takes the same certificate and does not read their slots)
        const TS gk = g;
        for (int64_t g = (int64_t)rb * kWarpsPerBlock + warp; g < lng.ncg; g += (int64_t)nbl * kWarpsPerBlock) {
            const int64_t v0 = lng.cslice_ptr[g];
            const int nblk_s = (int)((lng.cslice_ptr[g + 1] - v0) / 32);
            int my = nblk_s;  // this lane's vectors
            bool track = false;  // the chunk of a zero row without a certificate: its walk looks for a witness
            if (wt.wit) {
                const int32_t row = __ldg(lng.crow + g * 32 + lane);
                const unsigned fzr = row >= 0 && wt.frz ? (unsigned)wt.frz[row] : 0u;
                if (row < 0 || fzr == 1 || fzr == 2) {
                    my = 0;
                } else if (fzr == 3) {  // a resting zero row: its witness's value alone
                    if (part_resting_ok<TS, TG>(gk, wt.wit[row], yg)) my = 0;
                    else track = true;
                    ++ng;
                } else {
                    const TS xr = a.x[row];
                    TS yw;
                    if (xr == TS(0)) {
                        if (part_certified<TS, TG>(xr, a.v[row], gk, wt.wit[row], yg, yw)) my = 0;
                        else track = true;
                        ++ng;
                    }
                }
            }
            const int nblk = __reduce_max_sync(0xffffffffu, (unsigned)my);
            if (nblk == 0) continue;  // every chunk of the slice belongs to a certified or settled row
            const uint4* base = reinterpret_cast<const uint4*>(lng.csell) + v0 + lane;
            TS s;
            TG best = TG(0);     // an uncertified zero row's chunk: its largest published value
            int32_t barg = -1;   // and whose it is (the first such, ascending id)
            const bool delta = lng.cfmt[g] != 0;
            const int32_t id0 = delta ? __ldg(lng.cbase + g * 32 + lane) : 0;
            const int len = delta && my > 0 ? __ldg(lng.clen + g * 32 + lane) : 0;
            if (wt.gat) ng += delta ? (unsigned)len : 4u * (unsigned)my;
            if (lng.cmax && __any_sync(0xffffffffu, track))
                s = part_chunk_walk<TS, TG, true>(base, yg, my, nblk, delta, id0, len, best, barg);
            else
                s = part_chunk_walk<TS, TG, false>(base, yg, my, nblk, delta, id0, len, best, barg);
            const int32_t slot = __ldg(lng.cslot + g * 32 + lane);
            if (slot >= 0 && my > 0) {
                lng.sum[slot] = (double)s;
                if (lng.cmax && track) {
                    lng.cmax[slot] = (double)best;
                    lng.carg[slot] = barg;
                }
            }
        }
    } else if (rb < nbl) {
        // long rows, fast mode: one warp per piece of kPiece entries; lanes
        // stride the positions, 8 gathers in flight per lane with the next 8
        // indices loading under them; fixed butterfly fold.  The rows are
        // updated by k_part_long_combine (pieces added in piece order).
        const int64_t gw = (int64_t)rb * kWarpsPerBlock + warp, tw = (int64_t)nbl * kWarpsPerBlock;
        const int64_t qa = lng.blocked ? gw * lng.n / tw : gw, qb = lng.blocked ? (gw + 1) * lng.n / tw : lng.n;
        const int64_t qs = lng.blocked ? 1 : tw;
        for (int64_t qp = qa; qp < qb; qp += qs) {
            const int64_t q = lng.order ? __ldg(lng.order + qp) : qp;
            const int32_t pb = __ldg(lng.beg + q), pe = __ldg(lng.end + q);
            TS s = TS(0);
            constexpr int U = 8;
            int32_t idx[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int32_t pp = pb + lane + 32 * u;
                idx[u] = pp < pe ? ld_idx(col + pp) : -1;
            }
            for (int32_t p = pb + lane; p < pe; p += 32 * U) {
                int32_t nidx[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int32_t pp = p + 32 * (U + u);
                    nidx[u] = pp < pe ? ld_idx(col + pp) : -1;
                }
                TG y[U];
#pragma unroll
                for (int u = 0; u < U; ++u) y[u] = idx[u] >= 0 ? ld_val(yg + idx[u]) : TG(0);
#pragma unroll
                for (int u = 0; u < U; ++u) s = A::add(s, (TS)y[u]);
#pragma unroll
                for (int u = 0; u < U; ++u) idx[u] = nidx[u];
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s = A::add(s, __shfl_xor_sync(0xffffffffu, s, o));
            if (lane == 0) lng.sum[q] = (double)s;
        }
    } else if (rb < nbl + ncb) {
        for (int64_t q = (int64_t)(rb - nbl) * kPartThreads + tid; q < a.n_csr; q += (int64_t)ncb * kPartThreads) {
            const int64_t i = a.order[a.n_long + q];
            int32_t r0 = a.rowptr[i], r1 = a.rowptr[i + 1];
            TS s = TS(0);
            bool cert = false;
            if (wt.frz) {
                const unsigned fz = wt.frz[i];
                if (fz == 1 || fz == 2) {
                    if (fz == 2) part_member_mass<TS>(a.w64[i], ob);
                    continue;
                }
                if (fz == 3) {  // a resting zero row
                    const int32_t wj = wt.wit[i];
                    if (part_resting_ok<TS, TG>(g, wj, yg)) {
                        part_settle_zero(wt, i, wj, a.k, 3u);
                        ++ng;
                        continue;
                    }
                    wt.frz[i] = 0;  // back to walking (the test below fails the same way and queues the row)
                }
            }
            if (wt.wit) {
                const TS xi = a.x[i];
                if (xi == TS(0)) {
                    TS yw;
                    const int32_t wj = wt.wit[i];
                    if (part_certified<TS, TG>(xi, a.v[i], g, wj, yg, yw)) {
                        s = yw;
                        r1 = r0;
                        cert = true;
                        if (wt.frz) part_settle_zero(wt, i, wj, a.k, 0u);
                    } else {
                        part_enqueue(wt, i);
                    }
                    ++ng;
                }
            }
            if (wt.gat) ng += (unsigned)(r1 - r0);
            int32_t p = r0;
            for (; p + kPartUnroll <= r1; p += kPartUnroll) {  // scipy order, loads before the adds
                TG y[kPartUnroll];
#pragma unroll
                for (int u = 0; u < kPartUnroll; ++u) y[u] = ld_val(yg + __ldg(col + p + u));
#pragma unroll
                for (int u = 0; u < kPartUnroll; ++u) s = A::add(s, (TS)y[u]);
            }
            for (; p < r1; ++p) s = A::add(s, (TS)ld_val(yg + col[p]));
            const TS xi = a.x[i], vi = a.v[i];
            const TS o = part_update_pre<TS, TG>(i, s, g, xi, vi, a.w64[i], a.xo, a.ygo, mx, fb, ob, nf);
            if (wt.frz && !cert) part_member_candidate<TS, TG>(wt, i, xi, s, o, vi, a.k);
        }
    } else {
        const int64_t pos0 = a.n_long + a.n_csr;  // first order position of slice 0
        const int64_t nw = (int64_t)(nbid - nbl - ncb) * kWarpsPerBlock;
        const int64_t sl_first = (int64_t)(rb - nbl - ncb) * kWarpsPerBlock + warp;
        // the lane's flag and the slice's extent were loaded one slice ago
        // (lanes past the range count as settled zero rows), so a slice starts
        // with one round of independent loads -- state, witness, first index
        // vectors -- then the witnesses' values, then its gathers
        unsigned fzn = 0;
        int64_t e0n = 0;
        int nbn = 0;
        if (sl_first < a.nsl) {
            e0n = a.slice_ptr[sl_first];
            nbn = (int)((a.slice_ptr[sl_first + 1] - e0n) / 128);
            if (wt.frz) {
                const int64_t pn = pos0 + sl_first * 32 + lane;
                fzn = pn < a.count ? wt.frz[a.order[0] + pn] : 1u;
            }
        }
        for (int64_t sl = sl_first; sl < a.nsl; sl += nw) {
            const int64_t pos = pos0 + sl * 32 + lane;
            const bool valid = pos < a.count;
            const unsigned fz = fzn;
            const int64_t e0 = e0n;
            const int nblk_s = nbn;
            if (sl + nw < a.nsl) {
                e0n = a.slice_ptr[sl + nw];
                nbn = (int)((a.slice_ptr[sl + nw + 1] - e0n) / 128);
                if (wt.frz) {
                    const int64_t pn = pos + nw * 32;
                    fzn = pn < a.count ? wt.frz[a.order[0] + pn] : 1u;
                }
            }
            if (wt.frz && __all_sync(0xffffffffu, fz == 1 || fz == 2)) {  // a settled slice: the members' mass only
                if (fz == 2) part_member_mass<TS>(a.w64[a.order[0] + pos], ob);
                continue;
            }
            // rows are numbered in processing order (part_order): order[pos] == order[0] + pos
            const int64_t i = a.order[0] + (valid ? pos : 0);
            // round 1: the state of the rows that update (not settled rows, not
            // resting zero rows: theirs is 0 in both buffers), the witnesses, and
            // the first index vectors of the rows that may walk
            const bool act0 = !wt.wit || (valid && !fz);  // (without certificates every lane walks, rows past the range padding)
            const int32_t wj = wt.wit && (act0 || fz == 3) ? wt.wit[i] : -1;
            TS xi = TS(0), vi = TS(1);
            double wi = 0.0;
            if (act0) {
                xi = a.x[i];
                vi = a.v[i];
                wi = a.w64[i];
            } else if (fz == 2) {
                wi = a.w64[i];
            }
            const uint4* base = reinterpret_cast<const uint4*>(a.sell + e0) + lane;
            constexpr int NV = kPartUnroll / 4;  // index vectors per batch
            const int my0 = act0 ? nblk_s : 0;
            uint4 cv[NV];
#pragma unroll
            for (int u = 0; u < NV; ++u) cv[u] = u < my0 ? ld_idx4(base + (size_t)u * 32) : make_uint4(0, 0, 0, 0);
            // round 2: a zero row's certificate is its witness's value (a resting
            // row's x is 0: the same test); one load for both kinds
            const bool zrow = wt.wit && act0 && xi == TS(0);
            bool okc = false;
            TS yw = TS(0);
            if ((zrow || fz == 3) && wj >= 0) {
                yw = (TS)ld_val(yg + wj);
                okc = (double)A::add(A::mul(vi, xi), A::mul(g, yw)) > kSafeDiv;
            }
            bool act = act0, queue = false, cert = false;
            TS s = TS(0);
            if (fz == 3) {
                ++ng;
                if (okc) {
                    if (wt.frz) part_settle_zero(wt, i, wj, a.k, 3u);
                } else {  // back to walking: the flag goes, the row is a zero row without a certificate
                    wt.frz[i] = 0;
                    act = true;
                    queue = true;
                    vi = a.v[i];
                    wi = a.w64[i];
                }
            } else if (zrow) {
                ++ng;
                if (okc) {
                    s = yw;
                    cert = true;
                    if (wt.frz) part_settle_zero(wt, i, wj, a.k, 0u);
                } else {
                    queue = true;
                }
            }
            // this lane's index vectors: none past the range's rows, none for a
            // settled, resting or certified row (its stand-in sum is the witness's value)
            const int my = !wt.wit ? nblk_s : (act && !cert ? nblk_s : 0);
            const int nblk = wt.wit ? (int)__reduce_max_sync(0xffffffffu, (unsigned)my) : nblk_s;
            if (wt.gat) {
                if (wt.gat_mode == 1) ng += 4u * (unsigned)my;
                else if (wt.gat_mode == 2) ng = ng - ((zrow || fz == 3) ? 1u : 0u) + (my > 0 ? 1u : 0u);
                else ng = ng - ((zrow || fz == 3) ? 1u : 0u) + (lane == 0 && nblk > 0 ? 1u : 0u);
            }
            if (my > my0) {  // a resting row that lost its certificate
#pragma unroll
                for (int u = 0; u < NV; ++u) cv[u] = u < my ? ld_idx4(base + (size_t)u * 32) : make_uint4(0, 0, 0, 0);
            }
            for (int b = 0; b < nblk; b += NV) {
                uint4 nv[NV];
#pragma unroll
                for (int u = 0; u < NV; ++u)
                    nv[u] = b + NV + u < my ? ld_idx4(base + (size_t)(b + NV + u) * 32) : make_uint4(0, 0, 0, 0);
                TG y[4 * NV];
#pragma unroll
                for (int u = 0; u < NV; ++u) {
                    const bool in = b + u < my;
                    y[4 * u + 0] = in ? ld_val(yg + (int32_t)cv[u].x) : TG(0);
                    y[4 * u + 1] = in ? ld_val(yg + (int32_t)cv[u].y) : TG(0);
                    y[4 * u + 2] = in ? ld_val(yg + (int32_t)cv[u].z) : TG(0);
                    y[4 * u + 3] = in ? ld_val(yg + (int32_t)cv[u].w) : TG(0);
                }
#pragma unroll
                for (int q = 0; q < 4 * NV; ++q) s = A::add(s, (TS)y[q]);  // padding adds +0.0: bits unchanged
#pragma unroll
                for (int u = 0; u < NV; ++u) cv[u] = nv[u];
            }
            if (valid && act) {
                const TS o = part_update_pre<TS, TG>(i, s, g, xi, vi, wi, a.xo, a.ygo, mx, fb, ob, nf);
                if (wt.frz && !cert) part_member_candidate<TS, TG>(wt, i, xi, s, o, vi, a.k);
            } else if (fz == 2) {
                part_member_mass<TS>(wi, ob);
            }
            if (queue) part_enqueue(wt, i);
        }
    }
    if (wt.gat) {  // measurement only: one atomic per warp, spread over 64 counters
        if (wt.gat_mode != 1 && rb < nbl + ncb) ng = 0;  // rows / slices walked: the slice path's only
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ng += __shfl_xor_sync(0xffffffffu, ng, o);
        if (lane == 0 && ng) atomicAdd(wt.gat + ((vb * kWarpsPerBlock + warp) & 63), ng);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double m = __shfl_xor_sync(0xffffffffu, mx, o);
        if (!(m <= mx)) mx = m;
        fb += __shfl_xor_sync(0xffffffffu, fb, o);
        ob = __dadd_rn(ob, __shfl_xor_sync(0xffffffffu, ob, o));
        nf = fmax(nf, __shfl_xor_sync(0xffffffffu, nf, o));
    }
    if (lane == 0) {
        red[warp][0] = mx;
        red[warp][1] = fb;
        red[warp][2] = ob;
        red[warp][3] = nf;
    }
    __syncthreads();
    if (tid == 0) {
        double t[4] = {0.0, 0.0, 0.0, 0.0};
        for (int q = 0; q < kWarpsPerBlock; ++q) {
            if (!(red[q][0] <= t[0])) t[0] = red[q][0];
            t[1] += red[q][1];
            t[2] = __dadd_rn(t[2], red[q][2]);
            t[3] = fmax(t[3], red[q][3]);
        }
        double* dst = a.part + ((size_t)a.k * nbid + bid) * 4;
        dst[0] = t[0];
        dst[1] = t[1];
        dst[2] = t[2];
        dst[3] = t[3];
    }
}

// 4 blocks of 256 threads per SM (64 registers, no spills): 32 warps to hide
// the gathers' latency (C5 scale 24: 1.71 -> 1.59 ms per iteration vs 3)
template <typename TS, typename TG>
__global__ void __launch_bounds__(kPartThreads, GN_PART_MINB) k_part_step(const __grid_constant__ StepArgs<TS, TG> a) {
    __shared__ double red[kPartThreads / 32][4];
    part_step_vb<TS, TG>(a, (int)blockIdx.x, (int)threadIdx.x, red);
}

// Long rows, fast mode: a row's pieces' sums are added in piece order by one
// warp (lanes stride the pieces, fixed butterfly fold) and lane 0 updates the
// row (dynamics.py:104-107); per-block stats as k_part_step.
template <typename TS, typename TG>
__global__ void __launch_bounds__(kPartThreads) k_part_long_combine(
    int64_t n_long, int64_t first, const int32_t* __restrict__ lp,
    const double* __restrict__ pc_sum, const double* __restrict__ w64, const TS* __restrict__ v,
    const TS* __restrict__ x, TS* __restrict__ xo, const TG* __restrict__ yg, TG* __restrict__ ygo,
    const double* __restrict__ gam, int k, double* __restrict__ part, PartWit wt,
    const double* __restrict__ pc_max, const int32_t* __restrict__ pc_arg, int32_t* __restrict__ wit_out) {
    using A = Arith<TS>;
    const TS g = (TS)gam[k];
    double mx = 0.0, fb = 0.0, ob = 0.0, nf = 0.0;
    const int lane = threadIdx.x & 31;
    // a warp takes kCombRows rows.  First a lane per row looks at it on its own:
    // settled rows cost their flag (a member adds its mass), resting rows
    // their witness's value, certified zero rows are updated at once (their
    // chunks were not walked: k_part_step took the same certificate; the
    // witness's value stands in for the sum).  Then the warp adds the chunk
    // sums of the rows that walked, one row after another.  (One warp per
    // row made 7 k blocks of dependent loads per iteration, 23 us of a late
    // iteration in which no long row walks -- 7 us now; 32 rows per warp made
    // the early iterations, where every long row walks, 133 us instead of 36.)
    const int64_t q0 = ((int64_t)blockIdx.x * (kPartThreads / 32) + (threadIdx.x >> 5)) * kCombRows;
    {
        const int64_t q = q0 + lane;
        bool need = false, zero = false;
        if (lane < kCombRows && q < n_long) {
            const int64_t i = first + q;
            unsigned fz = wt.frz ? wt.frz[i] : 0u;
            if (fz == 2) part_member_mass<TS>(w64[i], ob);
            if (fz == 3) {
                // a resting zero row (the step's chunk lanes took the same test)
                const int32_t wj = wt.wit[i];
                if (part_resting_ok<TS, TG>(g, wj, yg)) {
                    part_settle_zero(wt, i, wj, k, 3u);
                    fz = 1;  // nothing more this iteration
                } else {
                    wt.frz[i] = 0;  // back to walking: a zero row without a certificate
                    fz = 0;
                }
            }
            if (!fz) {
                need = true;
                if (wt.wit) {
                    const TS xi = x[i];
                    zero = xi == TS(0);
                    TS yw;
                    const int32_t wj = wt.wit[i];
                    if (zero && part_certified<TS, TG>(xi, v[i], g, wj, yg, yw)) {
                        need = false;
                        part_update<TS, TG>(i, yw, g, w64, v, x, xo, ygo, mx, fb, ob, nf);
                        if (wt.frz) part_settle_zero(wt, i, wj, k, 0u);
                    }
                }
            }
        }
        unsigned todo = __ballot_sync(0xffffffffu, need);
        const unsigned zeros = __ballot_sync(0xffffffffu, zero);
        while (todo) {
            const int r = __ffs(todo) - 1;
            todo &= todo - 1;
            const int64_t qq = q0 + r, i = first + qq;
            const bool zr = (zeros >> r) & 1u;
            TS s = TS(0);
            const int32_t j0 = __ldg(lp + qq), j1 = __ldg(lp + qq + 1);
            for (int32_t j = j0 + lane; j < j1; j += 32) s = A::add(s, (TS)pc_sum[j]);
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) s = A::add(s, __shfl_xor_sync(0xffffffffu, s, d));
            bool searched = false;
            if (zr && pc_max) {
                // a zero row without a certificate: its chunks' walks kept their
                // largest values; the largest of those (the first chunk on ties)
                // is the row's new witness -- no second walk
                double best = 0.0;
                int32_t bj = INT32_MAX, arg = -1;
                for (int32_t j = j0 + lane; j < j1; j += 32) {
                    const double m = pc_max[j];
                    if (m > best) { best = m; bj = j; arg = pc_arg[j]; }
                }
#pragma unroll
                for (int d = 16; d > 0; d >>= 1) {
                    const double ob2 = __shfl_xor_sync(0xffffffffu, best, d);
                    const int32_t oj = __shfl_xor_sync(0xffffffffu, bj, d);
                    const int32_t oa = __shfl_xor_sync(0xffffffffu, arg, d);
                    if (ob2 > best || (ob2 == best && oj < bj)) { best = ob2; bj = oj; arg = oa; }
                }
                if (lane == 0) wit_out[i] = arg;
                searched = true;
            }
            if (lane == 0) {
                part_update<TS, TG>(i, s, g, w64, v, x, xo, ygo, mx, fb, ob, nf);
                if (zr && !searched) part_enqueue(wt, i);
            }
        }
    }
    __shared__ double red[kPartThreads / 32][4];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double m = __shfl_xor_sync(0xffffffffu, mx, o);
        if (!(m <= mx)) mx = m;
        fb += __shfl_xor_sync(0xffffffffu, fb, o);
        ob = __dadd_rn(ob, __shfl_xor_sync(0xffffffffu, ob, o));
        nf = fmax(nf, __shfl_xor_sync(0xffffffffu, nf, o));
    }
    if ((threadIdx.x & 31) == 0) {
        red[threadIdx.x >> 5][0] = mx;
        red[threadIdx.x >> 5][1] = fb;
        red[threadIdx.x >> 5][2] = ob;
        red[threadIdx.x >> 5][3] = nf;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t[4] = {0.0, 0.0, 0.0, 0.0};
        for (int w = 0; w < kPartThreads / 32; ++w) {
            if (!(red[w][0] <= t[0])) t[0] = red[w][0];
            t[1] += red[w][1];
            t[2] = __dadd_rn(t[2], red[w][2]);
            t[3] = fmax(t[3], red[w][3]);
        }
        double* dst = part + ((size_t)k * gridDim.x + blockIdx.x) * 4;
        dst[0] = t[0];
        dst[1] = t[1];
        dst[2] = t[2];
        dst[3] = t[3];
    }
}

// The zero rows one step launch walked without a certificate: one warp per
// queued row picks the neighbour of largest y (this iteration's values, the
// ones the step read; ties: the first in the row) as its witness for the next
// iterations.  Runs after the range's step (and combine), before any peer
// can overwrite the ghost values it reads.
template <typename TG>
__global__ void __launch_bounds__(kPartThreads) k_part_witness(const int32_t* __restrict__ rq,
                                                               const int* __restrict__ rqn, int cap,
                                                               const int32_t* __restrict__ rowptr,
                                                               const int32_t* __restrict__ col,
                                                               const TG* __restrict__ yg, int32_t* __restrict__ wit,
                                                               unsigned long long* __restrict__ gat) {
    const int n = min(*rqn, cap);
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * kPartThreads + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * kPartThreads) >> 5;
    unsigned long long ng = 0;
    for (int64_t e = w0; e < n; e += nw) {
        const int32_t i = __ldg(rq + e);
        const int32_t r0 = __ldg(rowptr + i), r1 = __ldg(rowptr + i + 1);
        double best = -1.0;
        int32_t bp = INT32_MAX;  // position of the best
        for (int32_t p = r0 + lane; p < r1; p += 32) {
            const double y = (double)ld_val(yg + __ldg(col + p));
            if (y > best) { best = y; bp = p; }
        }
        ng += (unsigned)max(0, (r1 - r0 - lane + 31) / 32);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int32_t op = __shfl_xor_sync(0xffffffffu, bp, o);
            if (ob > best || (ob == best && op < bp)) { best = ob; bp = op; }
        }
        if (lane == 0) wit[i] = bp < r1 ? __ldg(col + bp) : -1;
    }
    if (gat) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ng += __shfl_xor_sync(0xffffffffu, ng, o);
        if (lane == 0 && ng) atomicAdd(gat + (w0 & 63), ng);
    }
}

// The member candidates one iteration queued (state 1 before and after, every
// published neighbour value 0, the gamma test passed): one warp per candidate
// looks at the NEW states of its neighbours; when every neighbour is an owned
// row whose state is exactly 0 the row is a settled member (gn_part::frz).  A
// published 0 alone is not enough -- a tiny state can underflow in v*x and
// grow back.  Runs after both ranges' steps of the iteration.
template <typename TS>
__global__ void __launch_bounds__(kPartThreads) k_part_settle(const int32_t* __restrict__ mq,
                                                              const int* __restrict__ mqn, int cap,
                                                              const int32_t* __restrict__ rowptr,
                                                              const int32_t* __restrict__ col,
                                                              const TS* __restrict__ xnew, uint8_t* __restrict__ frz) {
    const int n = min(*mqn, cap);
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * kPartThreads + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * kPartThreads) >> 5;
    for (int64_t e = w0; e < n; e += nw) {
        const int32_t i = __ldg(mq + e);
        const int32_t r0 = __ldg(rowptr + i), r1 = __ldg(rowptr + i + 1);
        bool ok = true;
        for (int32_t p = r0 + lane; p < r1 && ok; p += 32) {
            const int32_t j = __ldg(col + p);
            ok = j < cap && xnew[j] == TS(0);
        }
        if (__all_sync(0xffffffffu, ok) && lane == 0) frz[i] = 2;
    }
}

// Direct halo protocol, per iteration k: wait until every peer that pushes
// here has finished step k-1 (its values of step k-1 are in our ghost slots,
// and it has read the buffer our pushes of step k will overwrite), step the
// boundary rows with their pushes, step the interior, then flag every peer.
// The spin is bounded (~10 s): a missing peer sets bad[0] instead of hanging.
__global__ void k_part_wait(const int64_t* flags, const int32_t* __restrict__ expect, int nexpect,
                            const int64_t* __restrict__ epoch, int64_t k, int* bad) {
    const int64_t target = (*epoch << 32) + k;
    for (int i = threadIdx.x; i < nexpect; i += blockDim.x) {
        const int64_t* f = flags + expect[i];
        long long t0 = 0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        for (;;) {
            long long v;
            asm volatile("ld.acquire.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(f) : "memory");
            if (v >= target) break;
            long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > 10000000000LL) {
                atomicExch(bad, 1);
                break;
            }
            __nanosleep(200);
        }
    }
}

__global__ void k_part_signal(int64_t* const* __restrict__ peer_flags, int npeers, int me,
                              const int64_t* __restrict__ epoch, int64_t step) {
    __threadfence_system();  // this part's pushes (earlier kernels on the stream) before the flags
    const int64_t value = (*epoch << 32) + step;
    for (int i = threadIdx.x; i < npeers; i += blockDim.x) {
        int64_t* f = peer_flags[i] + me;
        asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(f), "l"((long long)value) : "memory");
    }
}

// fold per-block stats of every iteration in block order (one warp per iteration)
__global__ void k_part_fold(const double* __restrict__ part, int nblocks, int iters, double* __restrict__ out) {
    const int k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (k >= iters) return;
    double t[4] = {0.0, 0.0, 0.0, 0.0};
    for (int b = lane; b < nblocks; b += 32) {
        const double* s = part + ((size_t)k * nblocks + b) * 4;
        if (!(s[0] <= t[0])) t[0] = s[0];
        t[1] += s[1];
        t[2] = __dadd_rn(t[2], s[2]);
        t[3] = fmax(t[3], s[3]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double m = __shfl_xor_sync(0xffffffffu, t[0], o);
        if (!(m <= t[0])) t[0] = m;
        t[1] += __shfl_xor_sync(0xffffffffu, t[1], o);
        t[2] = __dadd_rn(t[2], __shfl_xor_sync(0xffffffffu, t[2], o));
        t[3] = fmax(t[3], __shfl_xor_sync(0xffffffffu, t[3], o));
    }
    if (lane == 0)
        for (int c = 0; c < 4; ++c) out[(size_t)k * 4 + c] = t[c];
}

template <typename TG>
__global__ void k_part_pack(const TG* __restrict__ yg, const int32_t* __restrict__ idx,
                            const int32_t* __restrict__ inv, int64_t count, TG* __restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < count) out[i] = yg[inv[idx[i]]];  // idx: the caller's owned ids
}

template <typename TG>
__global__ void k_part_unpack(TG* __restrict__ yg, int64_t first, const TG* __restrict__ in, int64_t count) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < count) yg[first + i] = in[i];
}

template <typename TS, typename TOut>
__global__ void k_part_out(int64_t n, const TS* __restrict__ x, const int32_t* __restrict__ perm,
                           TOut* __restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) {
        double xi = (double)x[i];
        out[perm[i]] = xi < 0.0 ? 0.0 : (xi > 1.0 ? 1.0 : xi);  // dynamics.py:179, caller's numbering
    }
}

// ---- gather probes (gn_part_probe; measurement aids, not on the solve path)
// The SELL walk of k_part_step's thread-per-row branch with the update
// replaced by a plain store of the sum, in five variants that bound what the
// step can reach on this graph: MODE 1 the real gathers; 2 the index stream
// alone (no gathers); 3 every gather redirected into a 4096-entry table (L1
// hits: the walk's instruction and latency floor); 4 random gathers over the
// same table size (hash of the position; no locality at all).
template <typename TG, int MODE>
__global__ void __launch_bounds__(kPartThreads) k_part_probe(const int32_t* __restrict__ sell,
                                                             const int64_t* __restrict__ slice_ptr, int64_t nsl,
                                                             int64_t count, int64_t pos0, const TG* __restrict__ yg,
                                                             uint32_t nall, double* __restrict__ out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int kWarpsPerBlock = kPartThreads / 32;
    const int64_t nw = (int64_t)gridDim.x * kWarpsPerBlock;
    for (int64_t sl = (int64_t)blockIdx.x * kWarpsPerBlock + warp; sl < nsl; sl += nw) {
        const int64_t pos = pos0 + sl * 32 + lane;
        const int64_t e0 = slice_ptr[sl];
        const int nblk = (int)((slice_ptr[sl + 1] - e0) / 128);
        const uint4* base = reinterpret_cast<const uint4*>(sell + e0) + lane;
        constexpr int NV = kPartUnroll / 4;
        uint4 cv[NV];
#pragma unroll
        for (int u = 0; u < NV; ++u) cv[u] = u < nblk ? __ldg(base + (size_t)u * 32) : make_uint4(0, 0, 0, 0);
        double s = 0.0;
        for (int b = 0; b < nblk; b += NV) {
            uint4 nv[NV];
#pragma unroll
            for (int u = 0; u < NV; ++u)
                nv[u] = b + NV + u < nblk ? __ldg(base + (size_t)(b + NV + u) * 32) : make_uint4(0, 0, 0, 0);
            TG y[4 * NV];
#pragma unroll
            for (int u = 0; u < NV; ++u) {
                const bool in = b + u < nblk;
                const uint32_t id[4] = {(uint32_t)cv[u].x, (uint32_t)cv[u].y, (uint32_t)cv[u].z, (uint32_t)cv[u].w};
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    uint32_t j = id[c];
                    if (MODE == 3) j &= 4095u;
                    if (MODE == 4) j = (uint32_t)(((uint64_t)(pos * 2654435761u + (b + u) * 40503u + c) * 0x9E3779B1u) % nall);
                    y[4 * u + c] = !in ? TG(0) : (MODE == 2 ? (TG)(j & 1u) : __ldg(yg + j));
                }
            }
#pragma unroll
            for (int q = 0; q < 4 * NV; ++q) s += (double)y[q];
#pragma unroll
            for (int u = 0; u < NV; ++u) cv[u] = nv[u];
        }
        if (pos < count) out[pos] = s;
    }
}

static int pblocks(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + kPartThreads - 1) / kPartThreads, 1 << 16)); }

template <typename F>
static void parallel_for(int64_t n, F f) {
    const int nt = std::max(1, std::min(32, (int)std::thread::hardware_concurrency()));
    std::vector<std::thread> th;
    for (int t = 1; t < nt; ++t) th.emplace_back([&, t]() { for (int64_t i = t; i < n; i += nt) f(i); });
    for (int64_t i = 0; i < n; i += nt) f(i);
    for (auto& x : th) x.join();
}

template <typename T>
static int upload_into(T** dst, const std::vector<T>& h) {
    cudaFree(*dst);
    *dst = nullptr;
    GN_CUDA(cudaMalloc((void**)dst, sizeof(T) * std::max<size_t>(h.size(), 1)));
    if (!h.empty()) GN_CUDA(cudaMemcpy(*dst, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice));
    return GN_OK;
}

// Processing order: rows listed in `bnd` (the boundary) first, then the
// rest; each range degree-descending (stable), long rows leading.  Owned rows
// are relabeled to their position in this order and the device graph (CSR,
// weights, blocked SELL) is rebuilt in the new numbering.
static int part_order(gn_part* P, const int32_t* bnd, int64_t nb) {
    // rows above this degree are "long": in fast mode cut into chunks of
    // GN_PART_CHUNK entries (default 512) summed one thread per chunk over a
    // blocked SELL of chunks and combined per row (0: one warp per 512-entry
    // piece); in EXACT mode one thread per row over the CSR.  The others run
    // one thread per row over the blocked SELL.  Both thread-per-row walks
    // gather more cheaply than warp-split pieces (a slice's rows or chunks,
    // ordered by their hottest neighbours or first column, share lines at the
    // same positions) but each is one serial chain; the threshold and the
    // chunk length bound the chain.  C5 scale 24, one part, fp64, ms per
    // iteration -- warp pieces: threshold 512 1.62, 1024 1.50, 4096 1.44,
    // 8192 1.47, 65536 5.96; chunks of 128: threshold 1024 (= 2048) 1.335,
    // 4096 1.374; chunks of 64 / 256: 1.348 / 1.365 (R-MAT degrees cluster
    // near 2^29 * 0.76^(24-k) * 0.24^k: ~740, ~2300, ~7400, ...).  That
    // is with every row walked; over the whole pursuit, where most long
    // rows are certified zero rows whose chunks only test a flag, fewer
    // chunks win: ms per 1000 iterations at 128 / 256 / 512 / 1024:
    // 530.8 / 521.7 / 515.3 / 521.6 -- hence the default of 512.
    // On a small part the longest thread-per-row chain bounds the iteration
    // instead: the threshold is nnz / 16384 rounded down to a power of two
    // in [128, 1024] (C3, 2 M entries, us per iteration at threshold 32 / 64
    // / 128 / 256 / 512 / 1024: 19.9 / 19.1 / 18.0 / 23.1 / 33.8 / 54.0; an
    // 8-way part of C5, 65 M entries, ms: 128 0.238, 256 0.226, 512 0.225,
    // 1024 0.222).  GN_PART_LONG overrides.
    int kPartLongDegree = kPartLongDegreeMin;
    while (kPartLongDegree < kPartLongDegreeMax && (int64_t)kPartLongDegree * 2 * 16384 <= P->nnz) kPartLongDegree *= 2;
    if (const char* e = getenv("GN_PART_LONG")) kPartLongDegree = std::max(32, atoi(e));
    P->long_degree = kPartLongDegree;
    const int64_t n_own = P->n_own, nall = P->n_own + P->n_ghost;
    const std::vector<int32_t>& rp = P->h_rowptr;
    std::vector<uint8_t> is_b((size_t)std::max<int64_t>(n_own, 1), 0);
    for (int64_t i = 0; i < nb; ++i) {
        if (bnd[i] < 0 || bnd[i] >= n_own) return fail(GN_ERR_ARG, "boundary row out of range");
        is_b[(size_t)bnd[i]] = 1;
    }
    auto deg = [&](int32_t r) { return rp[(size_t)r + 1] - rp[(size_t)r]; };
    std::vector<int32_t> rb, ri;
    for (int64_t i = 0; i < n_own; ++i) (is_b[(size_t)i] ? rb : ri).push_back((int32_t)i);
    auto by_deg = [&](int32_t a, int32_t b) { return deg(a) > deg(b); };
    std::stable_sort(rb.begin(), rb.end(), by_deg);
    std::stable_sort(ri.begin(), ri.end(), by_deg);
    // the long rows (split over warps in fast mode) lead; the others are
    // degree-sorted, by default in one global order with the rows of equal
    // degree ordered by their two hottest neighbours (below).  Without that
    // ordering (GN_PART_LEX=0) windows of 2^18 of the caller's ids keep some
    // of the numbering's neighbourhood locality instead.  C5 scale 24, one
    // part, fp64, ms per iteration: global degree order 1.83, windows of 2^18
    // 1.70, windows + LEX 1.67, global + LEX 1.62 (GN_PART_WINDOW overrides,
    // 0 = global)
    int lex = 1;
    if (const char* e = getenv("GN_PART_LEX")) lex = atoi(e);
    size_t win = lex > 0 ? 0 : (size_t)1 << 18;
    if (const char* e = getenv("GN_PART_WINDOW")) win = atoi(e) > 0 ? (size_t)atoi(e) : 0;
    if (win > 0) {
        for (auto* v : {&rb, &ri}) {
            size_t nl = 0;
            while (nl < v->size() && deg((*v)[nl]) > kPartLongDegree) ++nl;
            std::sort(v->begin() + nl, v->end());
            for (size_t w0 = nl; w0 < v->size(); w0 += win)
                std::stable_sort(v->begin() + w0, v->begin() + std::min(v->size(), w0 + win), by_deg);
        }
    }
    // GN_PART_LEX=1 (default): inside each run of equal degree (after the long prefix),
    // rows ordered by their two hottest neighbours (smallest provisional new
    // ids; ghosts count as their own ids, after every owned row), so rows
    // that gather the same hubs sit in the same slice and the hubs' rows
    // gather runs of consecutive ids
    // (runs of equal floor(log2(degree)) instead: 1.63 -- slices pad more)
    if (lex > 0) {
        std::vector<uint32_t> pinv((size_t)n_own);
        for (size_t q = 0; q < rb.size(); ++q) pinv[(size_t)rb[q]] = (uint32_t)q;
        for (size_t q = 0; q < ri.size(); ++q) pinv[(size_t)ri[q]] = (uint32_t)(rb.size() + q);
        for (auto* v : {&rb, &ri}) {
            size_t nl = 0;
            while (nl < v->size() && deg((*v)[nl]) > kPartLongDegree) ++nl;
            std::vector<std::pair<size_t, size_t>> runs;
            for (size_t q = nl; q < v->size();) {
                size_t e2 = q;
                while (e2 < v->size() && deg((*v)[e2]) == deg((*v)[q]) && (win == 0 || (e2 - nl) / win == (q - nl) / win)) ++e2;
                runs.push_back({q, e2});
                q = e2;
            }
            parallel_for((int64_t)runs.size(), [&](int64_t ri2) {
                const size_t q0 = runs[(size_t)ri2].first, q1 = runs[(size_t)ri2].second;
                // key: the row's `lex` hottest neighbours (GN_PART_LEX=3: three)
                std::vector<std::tuple<uint64_t, uint32_t, int32_t>> kv(q1 - q0);
                for (size_t q = q0; q < q1; ++q) {
                    const int32_t r = (*v)[q];
                    uint32_t a = ~0u, b = ~0u, c3 = ~0u;
                    for (int32_t p = rp[(size_t)r]; p < rp[(size_t)r + 1]; ++p) {
                        const int32_t c = P->h_col[(size_t)p];
                        const uint32_t id = c < n_own ? pinv[(size_t)c] : (uint32_t)c;
                        if (id < a) { c3 = b; b = a; a = id; } else if (id < b) { c3 = b; b = id; } else if (id < c3) c3 = id;
                    }
                    kv[q - q0] = {((uint64_t)a << 32) | b, lex >= 3 ? c3 : 0u, r};
                }
                std::sort(kv.begin(), kv.end());
                for (size_t q = q0; q < q1; ++q) (*v)[q] = std::get<2>(kv[q - q0]);
            });
        }
    }
    // isolated rows that settle (degree 0 and v = sqrt(w) > 2e-9: from any
    // finite x0 > 0 the step gives 1.0, or 0.5 and then 1.0; from iteration
    // 3 on both state buffers hold 1.0 and the row no longer changes) go to
    // the end of the interior range, where fast-mode steps skip them
    {
        auto settles = [&](int32_t r) { return deg(r) == 0 && P->h_w[(size_t)r] > 4e-18; };
        std::stable_partition(ri.begin(), ri.end(), [&](int32_t r) { return !settles(r); });
        int64_t t = 0;
        for (auto it = ri.rbegin(); it != ri.rend() && settles(*it); ++it) ++t;
        P->n_iso = t;
    }
    P->n_bnd = (int64_t)rb.size();
    P->long_fast[0] = P->long_fast[1] = 0;
    while (P->long_fast[0] < (int64_t)rb.size() && deg(rb[(size_t)P->long_fast[0]]) > kPartLongDegree) ++P->long_fast[0];
    while (P->long_fast[1] < (int64_t)ri.size() && deg(ri[(size_t)P->long_fast[1]]) > kPartLongDegree) ++P->long_fast[1];
    std::vector<int32_t> perm = rb;
    perm.insert(perm.end(), ri.begin(), ri.end());
    std::vector<int32_t> inv((size_t)n_own), order((size_t)n_own);
    for (int64_t r = 0; r < n_own; ++r) {
        inv[(size_t)perm[(size_t)r]] = (int32_t)r;
        order[(size_t)r] = (int32_t)r;  // rows are numbered in processing order
    }
    // the relabeled CSR (neighbour order kept) and weights
    std::vector<int32_t> nrp((size_t)n_own + 1, 0);
    for (int64_t r = 0; r < n_own; ++r) nrp[(size_t)r + 1] = nrp[(size_t)r] + deg(perm[(size_t)r]);
    std::vector<int32_t> ncol((size_t)P->nnz);
    parallel_for(n_own, [&](int64_t r) {
        const int32_t o = perm[(size_t)r];
        int32_t* dst = ncol.data() + nrp[(size_t)r];
        for (int32_t e = rp[(size_t)o]; e < rp[(size_t)o + 1]; ++e) {
            const int32_t c = P->h_col[(size_t)e];
            *dst++ = c < n_own ? inv[(size_t)c] : c;
        }
    });
    std::vector<double> nw((size_t)nall);
    for (int64_t i = 0; i < nall; ++i) nw[(size_t)i] = P->h_w[(size_t)(i < n_own ? perm[(size_t)i] : i)];
    // blocked SELL of each range's rows after its long prefix
    const int32_t pad = (int32_t)nall;
    std::vector<int64_t> sp(1, 0);
    const int64_t rs[2] = {0, P->n_bnd}, rc[2] = {P->n_bnd, n_own - P->n_bnd};
    std::vector<int64_t> first;  // per slice: first row
    for (int r = 0; r < 2; ++r) {
        P->sl0[r] = (int64_t)sp.size() - 1;
        const int64_t p0 = rs[r] + P->long_fast[r], p1 = rs[r] + rc[r];
        P->nsl[r] = (p1 - p0 + 31) / 32;
        if (r == 1) {  // the slices wholly inside the settled tail
            const int64_t f = std::min(P->nsl[1], std::max<int64_t>(0, (p1 - P->n_iso - p0 + 31) / 32));
            P->iso_nsl = f < P->nsl[1] ? f : -1;
            P->iso_mass[0] = P->iso_mass[1] = 0.0;
            for (int64_t q = p0 + 32 * f; P->iso_nsl >= 0 && q < p1; ++q) {  // fixed order
                const double wq = P->h_w[(size_t)perm[(size_t)q]];
                P->iso_mass[0] += wq;
                P->iso_mass[1] += (double)(float)wq;
            }
        }
        for (int64_t q = p0; q < p1; q += 32) {
            int32_t len = 0;
            for (int64_t t = q; t < std::min(p1, q + 32); ++t) len = std::max(len, nrp[(size_t)t + 1] - nrp[(size_t)t]);
            first.push_back(q);
            sp.push_back(sp.back() + (int64_t)(len + 3) / 4 * 128);
        }
    }
    auto fill_sell = [&](const std::vector<int32_t>& cc) {
        std::vector<int32_t> sell((size_t)std::max<int64_t>(sp.back(), 1), pad);
        parallel_for((int64_t)first.size(), [&](int64_t sl) {
            const int64_t q = first[(size_t)sl];
            const int64_t end = q < P->n_bnd ? P->n_bnd : n_own;
            for (int l = 0; l < 32 && q + l < end; ++l) {
                const int64_t row = q + l;
                for (int32_t e = nrp[(size_t)row]; e < nrp[(size_t)row + 1]; ++e) {
                    const int32_t pos = e - nrp[(size_t)row];
                    sell[(size_t)(sp[(size_t)sl] + (pos / 4) * 128 + l * 4 + pos % 4)] = cc[(size_t)e];
                }
            }
        });
        return sell;
    };
    P->h_inv = inv;
    int rcode;
    if ((rcode = upload_into(&P->rowptr, nrp)) || (rcode = upload_into(&P->col, ncol)) ||
        (rcode = upload_into(&P->w64, nw)) || (rcode = upload_into(&P->perm, perm)) ||
        (rcode = upload_into(&P->inv, inv)) || (rcode = upload_into(&P->order, order)) ||
        (rcode = upload_into(&P->sell, fill_sell(ncol))) || (rcode = upload_into(&P->slice_ptr, sp)))
        return rcode;
    // fast-mode copies: rows in ascending new id (the sum order changes;
    // EXACT runs read the reference-order arrays above)
    parallel_for(n_own, [&](int64_t r) { std::sort(ncol.begin() + nrp[(size_t)r], ncol.begin() + nrp[(size_t)r + 1]); });
    if ((rcode = upload_into(&P->col_fast, ncol)) || (rcode = upload_into(&P->sell_fast, fill_sell(ncol))))
        return rcode;
    // the long rows' pieces (fast mode), per range: kPiece consecutive entries
    int64_t piece_len = kPiece;
    if (const char* e = getenv("GN_PIECE_LEN")) piece_len = std::max(32, atoi(e));
    P->chunk = kChunkDefault;
    if (const char* e = getenv("GN_PART_CHUNK")) P->chunk = std::max(0, atoi(e));
    if (P->chunk > 0) {
        P->chunk = std::max(32, P->chunk);
        piece_len = P->chunk;
    }
    P->interleave = 1;
    if (const char* e = getenv("GN_PART_INTERLEAVE")) P->interleave = atoi(e) != 0;
    std::vector<int32_t> pb, pe, lp, prow;
    for (int r = 0; r < 2; ++r) {
        P->pc0[r] = (int64_t)pb.size();
        P->lp0[r] = (int64_t)lp.size();
        for (int64_t q = 0; q < P->long_fast[r]; ++q) {
            const int64_t row = rs[r] + q;
            lp.push_back((int32_t)pb.size());
            int64_t e = nrp[(size_t)row];
            const int64_t end = nrp[(size_t)row + 1];
            while (e < end) {
                const int64_t f = std::min<int64_t>(e + piece_len, end);
                pb.push_back((int32_t)e);
                pe.push_back((int32_t)f);
                prow.push_back((int32_t)row);
                e = f;
            }
        }
        lp.push_back((int32_t)pb.size());
        P->npc[r] = (int64_t)pb.size() - P->pc0[r];
    }
    if ((rcode = upload_into(&P->pc_beg, pb)) || (rcode = upload_into(&P->pc_end, pe)) ||
        (rcode = upload_into(&P->lp, lp)))
        return rcode;
    int64_t slots = (int64_t)pb.size();
    // GN_PIECE_SORT=1: pieces processed in order of their first column (so
    // pieces over the same columns run close together: L1 reuse), 2: and
    // each warp takes one contiguous run of that order
    cudaFree(P->pc_order);
    P->pc_order = nullptr;
    P->piece_blocked = 0;
    {
        // default 2 (C5 scale 24 fp64: 1.737 -> 1.698 ms per iteration; with 512-entry pieces 1.677)
        const char* e = getenv("GN_PIECE_SORT");
        const int mode = e ? atoi(e) : 2;
        if (mode > 0) {
            std::vector<int32_t> ord(pb.size());
            for (int r = 0; r < 2; ++r) {
                const int64_t a0 = P->pc0[r], a1 = a0 + P->npc[r];
                for (int64_t j = a0; j < a1; ++j) ord[(size_t)j] = (int32_t)(j - a0);
                std::stable_sort(ord.begin() + a0, ord.begin() + a1, [&](int32_t x, int32_t y) {
                    return ncol[(size_t)pb[(size_t)(a0 + x)]] < ncol[(size_t)pb[(size_t)(a0 + y)]];
                });
            }
            if ((rcode = upload_into(&P->pc_order, ord))) return rcode;
            P->piece_blocked = mode >= 2;
        }
    }
    for (void* q : {(void*)P->csell, (void*)P->cslice_ptr, (void*)P->cslot, (void*)P->cfmt, (void*)P->cbase,
                    (void*)P->clen, (void*)P->crow})
        cudaFree(q);
    P->crow = nullptr;
    P->csell = nullptr;
    P->cslice_ptr = nullptr;
    P->cslot = nullptr;
    P->cfmt = nullptr;
    P->cbase = nullptr;
    P->clen = nullptr;
    if (P->chunk > 0) {
        // per range: chunks sorted by (16-bit deltas fit, length desc, first
        // column), 32 per slice.  A slice whose chunks all fit stores, in
        // block b, lane after lane, the deltas of entries 8b..8b+7 (16-byte
        // vectors); the others store entries 4b..4b+3 as int32 ids (padding:
        // the zero-valued slot nall)
        int delta = 1;
        if (const char* e = getenv("GN_PART_DELTA")) delta = atoi(e) != 0;
        auto clen_of = [&](int64_t j) { return pe[(size_t)j] - pb[(size_t)j]; };
        std::vector<uint8_t> fits(pb.size(), 0);
        parallel_for((int64_t)pb.size(), [&](int64_t j) {
            bool ok = delta != 0;
            for (int32_t e = pb[(size_t)j] + 1; ok && e < pe[(size_t)j]; ++e)
                ok = ncol[(size_t)e] - ncol[(size_t)e - 1] < 65536;
            fits[(size_t)j] = ok;
        });
        std::vector<int64_t> csp(1, 0);
        std::vector<int32_t> cslot, cbase, clen, crow;
        std::vector<int8_t> cfmt;
        for (int r = 0; r < 2; ++r) {
            P->cg0[r] = (int64_t)csp.size() - 1;
            const int64_t a0 = P->pc0[r], a1 = a0 + P->npc[r];
            std::vector<int32_t> ord;
            for (int64_t j = a0; j < a1; ++j) ord.push_back((int32_t)(j - a0));
            std::stable_sort(ord.begin(), ord.end(), [&](int32_t x, int32_t y) {
                if (fits[(size_t)(a0 + x)] != fits[(size_t)(a0 + y)]) return fits[(size_t)(a0 + x)] > fits[(size_t)(a0 + y)];
                const int32_t lx = clen_of(a0 + x), ly = clen_of(a0 + y);
                if (lx != ly) return lx > ly;
                return ncol[(size_t)pb[(size_t)(a0 + x)]] < ncol[(size_t)pb[(size_t)(a0 + y)]];
            });
            for (size_t g = 0; g < ord.size(); g += 32) {
                int32_t len = 0;
                bool all_fit = true;
                for (size_t l = g; l < std::min(ord.size(), g + 32); ++l) {
                    len = std::max(len, clen_of(a0 + ord[l]));
                    all_fit = all_fit && fits[(size_t)(a0 + ord[l])];
                }
                for (size_t l = g; l < g + 32; ++l) {
                    const bool in = l < ord.size();
                    cslot.push_back(in ? ord[l] : -1);
                    crow.push_back(in ? prow[(size_t)(a0 + ord[l])] : -1);
                    cbase.push_back(in ? ncol[(size_t)pb[(size_t)(a0 + ord[l])]] : 0);
                    clen.push_back(in ? clen_of(a0 + ord[l]) : 0);
                }
                cfmt.push_back(all_fit ? 1 : 0);
                const int per = all_fit ? 8 : 4;  // entries per lane per vector
                csp.push_back(csp.back() + (int64_t)(len + per - 1) / per * 32);
            }
            P->ncg[r] = (int64_t)csp.size() - 1 - P->cg0[r];
        }
        std::vector<uint32_t> cs((size_t)std::max<int64_t>(csp.back(), 1) * 4, 0);
        const int64_t ngs = (int64_t)csp.size() - 1;
        parallel_for(ngs, [&](int64_t g) {
            const int r = g >= P->cg0[1] ? 1 : 0;
            const int64_t a0 = P->pc0[r];
            const int64_t nvec = csp[(size_t)g + 1] - csp[(size_t)g];
            uint32_t* dst = cs.data() + (size_t)csp[(size_t)g] * 4;
            if (!cfmt[(size_t)g])
                for (int64_t t = 0; t < nvec * 4; ++t) dst[t] = (uint32_t)nall;  // int32 padding
            for (int l = 0; l < 32; ++l) {
                const int32_t sl = cslot[(size_t)(g * 32 + l)];
                if (sl < 0) continue;
                const int32_t e0 = pb[(size_t)(a0 + sl)], e1 = pe[(size_t)(a0 + sl)];
                for (int32_t e = e0; e < e1; ++e) {
                    const int32_t pos = e - e0;
                    if (cfmt[(size_t)g]) {  // vector pos/8 of lane l, half-word pos%8
                        const uint32_t d = e == e0 ? 0u : (uint32_t)(ncol[(size_t)e] - ncol[(size_t)e - 1]);
                        uint32_t& word = dst[((size_t)(pos / 8) * 32 + l) * 4 + (pos % 8) / 2];
                        word |= d << (16 * (pos % 2));
                    } else {
                        dst[((size_t)(pos / 4) * 32 + l) * 4 + pos % 4] = (uint32_t)ncol[(size_t)e];
                    }
                }
            }
        });
        std::vector<int32_t> cs32(cs.begin(), cs.end());
        if ((rcode = upload_into(&P->csell, cs32)) || (rcode = upload_into(&P->cslice_ptr, csp)) ||
            (rcode = upload_into(&P->cslot, cslot)) || (rcode = upload_into(&P->cfmt, cfmt)) ||
            (rcode = upload_into(&P->cbase, cbase)) || (rcode = upload_into(&P->clen, clen)) ||
            (rcode = upload_into(&P->crow, crow)))
            return rcode;
    }
    // zero-row certificates: one witness per row, the queue
    cudaFree(P->wit);
    cudaFree(P->rq);
    cudaFree(P->mq);
    cudaFree(P->frz);
    P->wit = P->rq = P->mq = nullptr;
    P->frz = nullptr;
    GN_CUDA(cudaMalloc((void**)&P->wit, 4 * (size_t)std::max<int64_t>(n_own, 1)));
    GN_CUDA(cudaMalloc((void**)&P->rq, 4 * (size_t)std::max<int64_t>(n_own, 1)));
    GN_CUDA(cudaMalloc((void**)&P->mq, 4 * (size_t)std::max<int64_t>(n_own, 1)));
    GN_CUDA(cudaMalloc((void**)&P->frz, (size_t)std::max<int64_t>(n_own, 1)));
    cudaFree(P->pc_sum);
    cudaFree(P->pc_max);
    cudaFree(P->pc_arg);
    P->pc_sum = P->pc_max = nullptr;
    P->pc_arg = nullptr;
    GN_CUDA(cudaMalloc((void**)&P->pc_sum, 8 * (size_t)std::max<int64_t>(slots, 1)));
    GN_CUDA(cudaMalloc((void**)&P->pc_max, 8 * (size_t)std::max<int64_t>(slots, 1)));
    GN_CUDA(cudaMalloc((void**)&P->pc_arg, 4 * (size_t)std::max<int64_t>(slots, 1)));
    P->gen++;
    return GN_OK;
}

static void part_free_push(gn_part* p) {
    void* q[] = {p->push_src, p->push_peer, p->push_slot, p->push_dst[0], p->push_dst[1], p->peer_flags};
    for (void* x : q) cudaFree(x);
    p->push_src = p->push_peer = nullptr;
    p->push_slot = nullptr;
    p->n_push = 0;
    p->gen++;
    p->push_dst[0] = p->push_dst[1] = nullptr;
    p->peer_flags = nullptr;
}

static void part_free_run(gn_part* p) {
    void* ptrs[] = {p->x[0], p->x[1], p->yg[0], p->yg[1], p->v, p->gam, p->part[0], p->part[1], p->part_long[0],
                    p->part_long[1], p->rq_cnt, p->gat, p->mq_cnt, p->gmin};
    for (void* q : ptrs)
        if (q) cudaFree(q);
    p->rq_cnt = nullptr;
    p->gat = nullptr;
    p->mq_cnt = nullptr;
    p->gmin = nullptr;
    p->x[0] = p->x[1] = p->yg[0] = p->yg[1] = p->v = nullptr;
    p->gam = p->part[0] = p->part[1] = p->part_long[0] = p->part_long[1] = nullptr;
    p->alloc_ncomb[0] = p->alloc_ncomb[1] = 0;
    p->alloc_nall = -1;
    p->alloc_dtype = -1;
    p->alloc_iters = 0;
    p->alloc_nblocks[0] = p->alloc_nblocks[1] = 0;
    p->gen++;
}

static void part_free_graph(gn_part* p) {
    if (p->gexec) cudaGraphExecDestroy(p->gexec);
    p->gexec = nullptr;
    p->g_gen = 0;
}

// f(TS{}, TG{}) with the state / gathered types of the partition's dtype
template <typename F>
static void by_dtype(int dtype, F f) {
    if (dtype == GN_F64) f(double(), double());
    else if (dtype == GN_F32) f(double(), float());
    else f(float(), float());
}

// the certificates of range r's launches at iteration k (null wit: off)
static PartWit part_wit_of(gn_part* p, int r, int k) {
    if (!p->witness || !p->rq_cnt) return PartWit{nullptr, nullptr, nullptr, nullptr, 0, 0, nullptr, nullptr, nullptr, nullptr};
    const bool st = p->settle && p->frz && p->mq_cnt;
    return PartWit{p->wit, p->rq, p->rq_cnt + 2 * (size_t)k + r, p->gat_on ? p->gat + 64 * (size_t)k : nullptr,
                   (int)p->n_own, p->gat_on, st ? p->frz : nullptr, st ? p->mq : nullptr, st ? p->mq_cnt + k : nullptr,
                   st ? p->gmin + k : nullptr};
}

// the member candidates of iteration k (both ranges), after the interior step
template <typename TS>
static void launch_settle(gn_part* p, int k, cudaStream_t s) {
    k_part_settle<TS><<<2 * 148, kPartThreads, 0, s>>>(p->mq, p->mq_cnt + k, (int)p->n_own, p->rowptr, p->col,
                                                     (const TS*)p->x[(k & 1) ^ 1], p->frz);
}

// one k_part_step launch over range r (the counts select which branches run)
template <typename TS, typename TG>
static void launch_step(gn_part* p, int r, int k, int nb, int64_t n_long, int nbl, int64_t ncsr, int ncb, int64_t nsl,
                        PartPush push, PartLong lng, cudaStream_t s) {
    const int cur = k & 1;
    const bool fast = !(p->flags & GN_EXACT);
    const StepArgs<TS, TG> a{n_long, nbl, ncsr, ncb, p->r_count[r], p->order + p->r_start[r], p->rowptr,
                             fast ? p->col_fast : p->col, fast ? p->sell_fast : p->sell, p->slice_ptr + p->sl0[r], nsl,
                             p->w64, (const TS*)p->v, (const TS*)p->x[cur], (TS*)p->x[cur ^ 1], (const TG*)p->yg[cur],
                             (TG*)p->yg[cur ^ 1], p->gam, k, p->part[r], push, lng, part_wit_of(p, r, k), nb};
    k_part_step<TS, TG><<<nb, kPartThreads, 0, s>>>(a);
}

template <typename TS, typename TG>
static void launch_combine(gn_part* p, int r, int k, cudaStream_t s) {
    const int cur = k & 1;
    k_part_long_combine<TS, TG><<<p->r_ncomb[r], kPartThreads, 0, s>>>(
        p->r_long[r], p->r_start[r], p->lp + p->lp0[r], p->pc_sum, p->w64,
        (const TS*)p->v, (const TS*)p->x[cur], (TS*)p->x[cur ^ 1], (const TG*)p->yg[cur], (TG*)p->yg[cur ^ 1], p->gam,
        k, p->part_long[r], part_wit_of(p, r, k), p->chunk && p->witness ? p->pc_max : nullptr, p->pc_arg, p->wit);
}

// the witness search for the zero rows range r's step queued at iteration k
template <typename TG>
static void launch_witness(gn_part* p, int r, int k, cudaStream_t s) {
    const PartWit w = part_wit_of(p, r, k);
    k_part_witness<TG><<<2 * 148, kPartThreads, 0, s>>>(w.rq, w.rqn, w.cap, p->rowptr, p->col,
                                                      (const TG*)p->yg[k & 1], p->wit, w.gat_mode == 1 ? w.gat : nullptr);
}

static PartLong part_long_of(gn_part* p, int r) {
    return PartLong{p->pc_beg + p->pc0[r], p->pc_end + p->pc0[r], p->pc_sum + p->pc0[r],
                    p->r_long[r] ? p->npc[r] : 0, p->pc_order ? p->pc_order + p->pc0[r] : nullptr,
                    p->piece_blocked, p->interleave, p->chunk ? p->csell : nullptr,
                    p->chunk ? p->cslice_ptr + p->cg0[r] : nullptr, p->chunk ? p->cslot + 32 * p->cg0[r] : nullptr,
                    p->chunk ? p->cfmt + p->cg0[r] : nullptr, p->chunk ? p->cbase + 32 * p->cg0[r] : nullptr,
                    p->chunk ? p->clen + 32 * p->cg0[r] : nullptr, p->chunk ? p->ncg[r] : 0,
                    p->chunk ? p->crow + 32 * p->cg0[r] : nullptr,
                    p->chunk && p->witness && p->pc_max ? p->pc_max + p->pc0[r] : nullptr,
                    p->chunk && p->pc_arg ? p->pc_arg + p->pc0[r] : nullptr};
}

}  // namespace gn

using namespace gn;

extern "C" {

int gn_part_create(int64_t n_own, int64_t n_ghost, const int64_t* indptr, const int32_t* indices, const double* w,
                   int dtype, int device, gn_part** out) {
    GN_NVTX("gn_part_create");
    *out = nullptr;
    if (n_own < 0 || n_ghost < 0) return fail(GN_ERR_ARG, "bad partition sizes");
    if (!valid_dtype(dtype)) return fail(GN_ERR_ARG, "dtype must be GN_F64, GN_F32 or GN_F32_PURE");
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(GN_ERR_NODEV, "no CUDA device visible: the GN engine has no CPU fallback");
    }
    const int64_t nnz = n_own > 0 ? indptr[n_own] : 0;
    if (nnz >= (int64_t(1) << 31)) return fail(GN_ERR_ARG, "partition too large");
    for (int64_t p = 0; p < nnz; ++p)
        if (indices[p] < 0 || indices[p] >= n_own + n_ghost) return fail(GN_ERR_ARG, "local column id out of range");
    gn_part* P = new gn_part();
    P->n_own = n_own;
    P->n_ghost = n_ghost;
    P->nnz = nnz;
    P->dtype = dtype;
    P->device = device;
    CallCtx ctx;
    int rc = ctx.open(device);
    if (rc) { delete P; return rc; }
    std::vector<int32_t> rp((size_t)n_own + 1);
    for (int64_t i = 0; i <= n_own; ++i) rp[(size_t)i] = (int32_t)(n_own > 0 ? indptr[i] : 0);
    const int64_t nall = n_own + n_ghost;
    P->h_rowptr = rp;
    P->h_col.assign(indices, indices + nnz);
    P->h_w.assign(w, w + nall);
    if ((rc = part_order(P, nullptr, 0))) {
        delete P;
        return rc;
    }
    GN_CUDA(cudaStreamCreateWithFlags(&P->own_stream, cudaStreamNonBlocking));
    *out = P;
    return GN_OK;
}

int gn_part_destroy(gn_part* p) {
    if (!p) return GN_OK;
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(p->device);
    part_free_graph(p);
    part_free_run(p);
    cudaFree(p->io);
    cudaFree(p->dout);
    cudaFree(p->d_epoch);
    cudaFree(p->pc_beg);
    cudaFree(p->pc_end);
    cudaFree(p->pc_order);
    for (void* q : {(void*)p->csell, (void*)p->cslice_ptr, (void*)p->cslot, (void*)p->cfmt, (void*)p->cbase,
                    (void*)p->clen, (void*)p->crow, (void*)p->wit, (void*)p->rq, (void*)p->mq, (void*)p->frz})
        cudaFree(q);
    cudaFree(p->lp);
    cudaFree(p->pc_sum);
    cudaFree(p->pc_max);
    cudaFree(p->pc_arg);
    cudaFree(p->rowptr);
    cudaFree(p->col);
    cudaFree(p->order);
    cudaFree(p->perm);
    cudaFree(p->inv);
    part_free_push(p);
    cudaFree(p->inflags);
    cudaFree(p->expect);
    cudaFree(p->halo_bad);
    cudaFree(p->sell);
    cudaFree(p->sell_fast);
    cudaFree(p->col_fast);
    cudaFree(p->slice_ptr);
    cudaFree(p->w64);
    if (p->own_stream) cudaStreamDestroy(p->own_stream);
    if (prev >= 0) cudaSetDevice(prev);
    delete p;
    return GN_OK;
}

int gn_part_begin(gn_part* p, const double* x0, const double* gammas, int iters, uint32_t flags) {
    GN_NVTX("gn_part_begin");
    if (!p || iters < 1 || !gammas) return fail(GN_ERR_ARG, "bad gn_part_begin arguments");
    GN_CUDA(cudaSetDevice(p->device));
    const int64_t nall = p->n_own + p->n_ghost;
    const size_t es = state_bytes(p->dtype), gs = gather_bytes(p->dtype);
    const size_t nb = (size_t)std::max<int64_t>(nall, 1);
    if (p->flags != flags) p->gen++;  // the captured schedule depends on the mode
    p->iters = iters;
    p->flags = flags;
    // per range (boundary, interior): GN_EXACT sums every row sequentially
    // (bitwise the reference); otherwise the longest rows are split over warps
    for (int r = 0; r < 2; ++r) {
        p->r_start[r] = r ? p->n_bnd : 0;
        p->r_count[r] = r ? p->n_own - p->n_bnd : p->n_bnd;
        p->r_long[r] = (flags & GN_EXACT) ? 0 : p->long_fast[r];
        const int64_t lunits = p->chunk ? p->ncg[r] : p->npc[r];  // chunk slices or pieces, one per warp
        p->r_nbl[r] = p->r_long[r]
                          ? (int)std::min<int64_t>((lunits + kPartThreads / 32 - 1) / (kPartThreads / 32), 1 << 12)
                          : 0;
        const int64_t rows_per_block = (int64_t)kCombRows * (kPartThreads / 32);
        p->r_ncomb[r] = p->r_long[r] ? (int)((p->r_long[r] + rows_per_block - 1) / rows_per_block) : 0;
        p->r_csr[r] = p->long_fast[r] - p->r_long[r];  // EXACT: the long rows, one thread each
        p->r_ncb[r] = p->r_csr[r] ? pblocks(p->r_csr[r]) : 0;
        // slice blocks: `spw` slices per warp (GN_PART_SPW).  One slice per warp
        // leaves the balancing to the block scheduler; several make a settled
        // slice cost one flag test of a running warp instead of a block's launch
        // and its chain of dependent loads
        // (at most kSlicesPerWarp, fewer on a small range so the blocks still
        // fill the GPU about four times over: an 8-way part of C5 with 16 slices
        // per warp had 270 blocks for 592 resident slots and ran at 0.51 ms per
        // iteration instead of 0.22)
        int spw = (int)std::min<int64_t>(kSlicesPerWarp, std::max<int64_t>(1, p->nsl[r] / (4 * 148 * GN_PART_MINB * (kPartThreads / 32))));
        if (const char* e = getenv("GN_PART_SPW")) spw = std::max(1, atoi(e));
        const int64_t per_block = (int64_t)(kPartThreads / 32) * spw;
        const int sblocks = (int)std::min<int64_t>((p->nsl[r] + per_block - 1) / per_block, 1 << 16);
        p->r_nblocks[r] = p->r_count[r] ? p->r_nbl[r] + p->r_ncb[r] + std::max(sblocks, 1) : 0;
    }
    // the run buffers stay where they are while their sizes hold: the yg
    // buffers are mapped by the peers (CUDA IPC) and named by the captured
    // schedule
    if (p->alloc_nall != nall || p->alloc_dtype != p->dtype || p->alloc_iters != iters ||
        p->alloc_nblocks[0] != p->r_nblocks[0] || p->alloc_nblocks[1] != p->r_nblocks[1] ||
        p->alloc_ncomb[0] != p->r_ncomb[0] || p->alloc_ncomb[1] != p->r_ncomb[1]) {
        part_free_run(p);
        GN_CUDA(cudaMalloc(&p->x[0], es * nb));
        GN_CUDA(cudaMalloc(&p->x[1], es * nb));
        // published values + the zero-valued padding slot n_all
        GN_CUDA(cudaMalloc(&p->yg[0], gs * (nb + 4)));  // + the zero slot n_all, and 16-byte tails
        GN_CUDA(cudaMalloc(&p->yg[1], gs * (nb + 4)));
        GN_CUDA(cudaMalloc(&p->v, es * nb));
        GN_CUDA(cudaMalloc((void**)&p->gam, 8 * (size_t)iters));
        for (int r = 0; r < 2; ++r)
            if (p->r_nblocks[r]) GN_CUDA(cudaMalloc((void**)&p->part[r], 32 * (size_t)iters * p->r_nblocks[r]));
        for (int r = 0; r < 2; ++r)
            if (p->r_ncomb[r]) GN_CUDA(cudaMalloc((void**)&p->part_long[r], 32 * (size_t)iters * p->r_ncomb[r]));
        GN_CUDA(cudaMalloc((void**)&p->rq_cnt, 4 * 2 * (size_t)iters));
        GN_CUDA(cudaMalloc((void**)&p->gat, 8 * 64 * (size_t)iters));
        GN_CUDA(cudaMalloc((void**)&p->mq_cnt, 4 * (size_t)iters));
        GN_CUDA(cudaMalloc((void**)&p->gmin, 8 * (size_t)iters));
        p->alloc_nall = nall;
        p->alloc_dtype = p->dtype;
        p->alloc_iters = iters;
        p->alloc_nblocks[0] = p->r_nblocks[0];
        p->alloc_nblocks[1] = p->r_nblocks[1];
        p->alloc_ncomb[0] = p->r_ncomb[0];
        p->alloc_ncomb[1] = p->r_ncomb[1];
    }
    GN_CUDA(cudaMemset(p->yg[0], 0, gs * (nb + 4)));
    GN_CUDA(cudaMemset(p->yg[1], 0, gs * (nb + 4)));
    // zero-row certificates: no witnesses yet, empty queues
    int witness = 1;
    if (const char* e = getenv("GN_PART_WITNESS")) witness = atoi(e) != 0;
    if (witness != p->witness) p->gen++;
    p->witness = witness;
    GN_CUDA(cudaMemset(p->wit, 0xFF, 4 * (size_t)std::max<int64_t>(p->n_own, 1)));
    GN_CUDA(cudaMemset(p->rq_cnt, 0, 4 * 2 * (size_t)iters));
    // settled rows: none yet; the smallest gamma still to come per iteration
    // (default: binary64 runs only -- with binary32 published values a state
    // below 1e-38 publishes 0 for hundreds of iterations before it is exactly 0,
    // members wait that long to settle, and the flags cost more than they save:
    // C5 scale 24 mixed, 0.51 ms per iteration with the certificates alone, 0.69
    // with the settled rows; GN_PART_SETTLE=1 turns them on in any precision)
    int settle = witness && p->dtype == GN_F64;
    if (const char* e = getenv("GN_PART_SETTLE")) settle = witness && atoi(e) != 0;
    if (settle != p->settle) p->gen++;
    p->settle = settle;
    GN_CUDA(cudaMemset(p->frz, 0, (size_t)std::max<int64_t>(p->n_own, 1)));
    GN_CUDA(cudaMemset(p->mq_cnt, 0, 4 * (size_t)iters));
    {
        std::vector<double> gm((size_t)iters);
        double m = std::numeric_limits<double>::infinity();
        for (int k = iters - 1; k >= 0; --k) {
            const double g = gammas[k];
            if (!(g > 0.0) || !std::isfinite(g)) m = 0.0;
            else if (g < m) m = g;
            gm[(size_t)k] = m;
        }
        GN_CUDA(cudaMemcpy(p->gmin, gm.data(), 8 * (size_t)iters, cudaMemcpyHostToDevice));
    }
    const int count = getenv("GN_PART_COUNT") ? atoi(getenv("GN_PART_COUNT")) : 0;  // 1 gathers, 2 rows walked, 3 slices walked
    if (count != p->gat_on) p->gen++;
    p->gat_on = count;
    GN_CUDA(cudaMemset(p->gat, 0, 8 * 64 * (size_t)iters));
    GN_CUDA(cudaMemcpy(p->gam, gammas, 8 * (size_t)iters, cudaMemcpyHostToDevice));
    // a new run epoch (see gn_part::epoch)
    if (!p->d_epoch) GN_CUDA(cudaMalloc((void**)&p->d_epoch, sizeof(int64_t)));
    p->epoch++;
    GN_CUDA(cudaMemcpy(p->d_epoch, &p->epoch, sizeof(int64_t), cudaMemcpyHostToDevice));
    if (p->io_n < (int64_t)nb) {
        cudaFree(p->io);
        p->io = nullptr;
        GN_CUDA(cudaMalloc((void**)&p->io, 8 * nb));
        p->io_n = (int64_t)nb;
    }
    double* dx0 = p->io;
    if (nall) GN_CUDA(cudaMemcpy(dx0, x0, 8 * (size_t)nall, cudaMemcpyHostToDevice));
    if (nall > 0) {
        const int blocks = pblocks(nall);
        switch (p->dtype) {
            case GN_F64:
                k_part_prepare<double, double><<<blocks, kPartThreads>>>(p->n_own, nall, dx0, p->perm, p->w64, (double*)p->x[0],
                                                                          (double*)p->v, (double*)p->yg[0]);
                break;
            case GN_F32:
                k_part_prepare<double, float><<<blocks, kPartThreads>>>(p->n_own, nall, dx0, p->perm, p->w64, (double*)p->x[0],
                                                                         (double*)p->v, (float*)p->yg[0]);
                break;
            default:
                k_part_prepare<float, float><<<blocks, kPartThreads>>>(p->n_own, nall, dx0, p->perm, p->w64, (float*)p->x[0],
                                                                        (float*)p->v, (float*)p->yg[0]);
        }
        GN_LAUNCHED();
        // the ghost slots of the other buffer are filled by unpack before they are read
        GN_CUDA(cudaMemcpy(p->yg[1], p->yg[0], gs * (size_t)nall, cudaMemcpyDeviceToDevice));
    }
    // (inflags are not reset: flags of an earlier epoch are below every target
    // of this one, and a peer may already have signalled this epoch)
    if (p->halo_bad) GN_CUDA(cudaMemset(p->halo_bad, 0, sizeof(int)));
    GN_CUDA(cudaDeviceSynchronize());
    return GN_OK;
}

// one range of the owned rows (0: boundary, 1: interior) for iteration k
// one range of the owned rows (0: boundary, 1: interior) for iteration k:
// the step kernel, then (fast mode) the long rows' combine
static int part_settle_after(gn_part* p, int k, int r, cudaStream_t s) {
    if (r != 1 || !p->witness || !p->settle || !p->frz || !p->mq_cnt || p->n_own == 0) return GN_OK;
    if (state_bytes(p->dtype) == 8) launch_settle<double>(p, k, s);
    else launch_settle<float>(p, k, s);
    GN_LAUNCHED();
    return GN_OK;
}

static int part_step_range(gn_part* p, int k, int r, cudaStream_t s) {
    if (p->r_count[r] == 0 && !(r == 1 && p->n_push > 0)) {
        return part_settle_after(p, k, r, s);
    }
    PartPush push{nullptr, nullptr, nullptr, nullptr, 0, 0};
    // the boundary rows' pushes ride on the interior launch
    if (r == 1 && p->n_push > 0)
        push = PartPush{p->push_src, p->push_peer, p->push_slot, p->push_dst[(k + 1) & 1], p->n_push,
                        (int)std::min<int64_t>((p->n_push + 8 * kPartThreads - 1) / (8 * kPartThreads), 148)};
    const int nb = (p->r_count[r] ? p->r_nblocks[r] : 0) + push.nblocks;
    const PartLong lng = part_long_of(p, r);
    // fast mode, iteration >= 3: the settled isolated tail is skipped
    const int64_t nsl = (r == 1 && k >= 3 && p->iso_nsl >= 0 && !(p->flags & GN_EXACT)) ? p->iso_nsl : p->nsl[r];
    by_dtype(p->dtype, [&](auto ts, auto tg) {
        launch_step<decltype(ts), decltype(tg)>(p, r, k, nb, p->r_long[r], p->r_nbl[r], p->r_csr[r], p->r_ncb[r],
                                                nsl, push, lng, s);
    });
    GN_LAUNCHED();
    if (p->r_long[r] > 0 && p->r_count[r] > 0) {
        by_dtype(p->dtype, [&](auto ts, auto tg) { launch_combine<decltype(ts), decltype(tg)>(p, r, k, s); });
        GN_LAUNCHED();
    }
    if (p->witness && p->r_count[r] > 0) {
        by_dtype(p->dtype, [&](auto, auto tg) { launch_witness<decltype(tg)>(p, r, k, s); });
        GN_LAUNCHED();
    }
    return part_settle_after(p, k, r, s);
}

int gn_part_step(gn_part* p, int k, uintptr_t stream) {
    if (!p || k < 0 || k >= p->iters) return fail(GN_ERR_ARG, "iteration out of range");
    cudaStream_t s = (cudaStream_t)stream;  // 0: the legacy default stream (orders with torch's)
    int rc = part_step_range(p, k, 0, s);
    return rc ? rc : part_step_range(p, k, 1, s);
}

int gn_part_step_range(gn_part* p, int k, int which, uintptr_t stream) {
    if (!p || k < 0 || k >= p->iters || which < 0 || which > 1) return fail(GN_ERR_ARG, "bad gn_part_step_range");
    return part_step_range(p, k, which, (cudaStream_t)stream);
}

int gn_part_set_boundary(gn_part* p, const int32_t* rows, int64_t count) {
    if (!p || count < 0 || (count > 0 && !rows)) return fail(GN_ERR_ARG, "bad gn_part_set_boundary");
    GN_CUDA(cudaSetDevice(p->device));
    return part_order(p, rows, count);
}

int gn_part_elem_bytes(const gn_part* p) { return p ? (int)gather_bytes(p->dtype) : 0; }

// pack owned published values after step k (i.e. the values step k+1 reads)
int gn_part_pack(gn_part* p, int k, const int32_t* d_idx, int64_t count, void* d_out, uintptr_t stream) {
    if (!p || count < 0) return fail(GN_ERR_ARG, "bad pack arguments");
    if (count == 0) return GN_OK;
    cudaStream_t s = (cudaStream_t)stream;  // 0: the legacy default stream (orders with torch's)
    const void* src = p->yg[(k & 1) ^ 1];
    const int blocks = (int)((count + 255) / 256);
    if (gather_bytes(p->dtype) == 8)
        k_part_pack<double><<<blocks, 256, 0, s>>>((const double*)src, d_idx, p->inv, count, (double*)d_out);
    else
        k_part_pack<float><<<blocks, 256, 0, s>>>((const float*)src, d_idx, p->inv, count, (float*)d_out);
    GN_LAUNCHED();
    return GN_OK;
}

int gn_part_unpack(gn_part* p, int k, const void* d_in, int64_t ghost_first, int64_t count, uintptr_t stream) {
    if (!p || count < 0 || ghost_first < 0 || ghost_first + count > p->n_ghost) return fail(GN_ERR_ARG, "bad unpack");
    if (count == 0) return GN_OK;
    cudaStream_t s = (cudaStream_t)stream;  // 0: the legacy default stream (orders with torch's)
    void* dst = p->yg[(k & 1) ^ 1];
    const int blocks = (int)((count + 255) / 256);
    if (gather_bytes(p->dtype) == 8)
        k_part_unpack<double><<<blocks, 256, 0, s>>>((double*)dst, p->n_own + ghost_first, (const double*)d_in, count);
    else
        k_part_unpack<float><<<blocks, 256, 0, s>>>((float*)dst, p->n_own + ghost_first, (const float*)d_in, count);
    GN_LAUNCHED();
    return GN_OK;
}

// stats of the owned rows after `done` iterations, x clipped
int gn_part_end(gn_part* p, int done, double* x_out, double* step_inf, int64_t* fallbacks, double* mass, int* bad) {
    GN_NVTX("gn_part_end");
    if (!p || done < 0 || done > p->iters) return fail(GN_ERR_ARG, "bad gn_part_end arguments");
    GN_CUDA(cudaSetDevice(p->device));
    GN_CUDA(cudaDeviceSynchronize());
    if (p->dout_n < std::max(done, 1)) {  // per (range, kernel), per iteration: 4 doubles
        cudaFree(p->dout);
        p->dout = nullptr;
        GN_CUDA(cudaMalloc((void**)&p->dout, 128 * (size_t)std::max(done, 1)));
        p->dout_n = std::max(done, 1);
    }
    if (p->io_n < std::max<int64_t>(p->n_own, 1)) {
        cudaFree(p->io);
        p->io = nullptr;
        GN_CUDA(cudaMalloc((void**)&p->io, 8 * (size_t)std::max<int64_t>(p->n_own, 1)));
        p->io_n = std::max<int64_t>(p->n_own, 1);
    }
    double *dout = p->dout, *dx = p->io;
    GN_CUDA(cudaMemset(dout, 0, 128 * (size_t)std::max(done, 1)));
    for (int r = 0; r < 2 && done > 0; ++r) {
        if (p->r_nblocks[r]) {
            k_part_fold<<<(done + 7) / 8, 256>>>(p->part[r], p->r_nblocks[r], done, dout + (size_t)r * 4 * done);
            GN_LAUNCHED();
        }
        if (p->r_long[r] && p->r_ncomb[r]) {  // the long rows' combine blocks of the range
            k_part_fold<<<(done + 7) / 8, 256>>>(p->part_long[r], p->r_ncomb[r], done,
                                                 dout + (size_t)(2 + r) * 4 * done);
            GN_LAUNCHED();
        }
    }
    if (p->n_own > 0) {
        if (state_bytes(p->dtype) == 8)
            k_part_out<double, double><<<pblocks(p->n_own), kPartThreads>>>(p->n_own, (const double*)p->x[done & 1], p->perm, dx);
        else
            k_part_out<float, double><<<pblocks(p->n_own), kPartThreads>>>(p->n_own, (const float*)p->x[done & 1], p->perm, dx);
        GN_LAUNCHED();
    }
    std::vector<double> h2(16 * (size_t)std::max(done, 1));
    GN_CUDA(cudaMemcpy(h2.data(), dout, 128 * (size_t)std::max(done, 1), cudaMemcpyDeviceToHost));
    // boundary range (step blocks, long-row combine), then the interior range
    // likewise: max / sum / fp64 sum / max, in this fixed order
    std::vector<double> h(4 * (size_t)std::max(done, 1));
    for (int k = 0; k < done; ++k) {
        double t[4] = {0.0, 0.0, 0.0, 0.0};
        for (int sec : {0, 2, 1, 3}) {
            const double* a = &h2[((size_t)sec * done + k) * 4];
            if (a[0] > t[0] || a[0] != a[0]) t[0] = a[0];
            t[1] += a[1];
            t[2] += a[2];
            t[3] = std::max(t[3], a[3]);
        }
        if (k >= 3 && p->iso_nsl >= 0 && !(p->flags & GN_EXACT))  // the skipped rows' w . 1.0
            t[2] += p->iso_mass[state_bytes(p->dtype) == 8 ? 0 : 1];
        for (int c = 0; c < 4; ++c) h[(size_t)k * 4 + c] = t[c];
    }
    if (x_out && p->n_own) GN_CUDA(cudaMemcpy(x_out, dx, 8 * (size_t)p->n_own, cudaMemcpyDeviceToHost));
    if (p->halo_bad) {
        int hb = 0;
        GN_CUDA(cudaMemcpy(&hb, p->halo_bad, sizeof(int), cudaMemcpyDeviceToHost));
        if (hb) return fail(GN_ERR_CUDA, "direct halo: a peer's step flag did not arrive within 10 s");
    }
    if (bad) *bad = -1;
    for (int k = 0; k < done; ++k) {
        if (step_inf) step_inf[k] = h[(size_t)k * 4];
        if (fallbacks) fallbacks[k] = (int64_t)h[(size_t)k * 4 + 1];
        if (mass) mass[k] = h[(size_t)k * 4 + 2];
        if (bad && *bad < 0 && h[(size_t)k * 4 + 3] != 0.0) *bad = k;
    }
    return GN_OK;
}

// ---- direct halo over peer memory
int gn_part_peer_init(gn_part* p, int parts, int me, const int32_t* expect, int nexpect) {
    if (!p || parts < 1 || me < 0 || me >= parts || nexpect < 0 || (nexpect > 0 && !expect))
        return fail(GN_ERR_ARG, "bad gn_part_peer_init arguments");
    GN_CUDA(cudaSetDevice(p->device));
    for (int i = 0; i < nexpect; ++i)
        if (expect[i] < 0 || expect[i] >= parts || expect[i] == me) return fail(GN_ERR_ARG, "bad expected peer");
    part_free_push(p);
    p->peers.clear();
    p->h_push_row.clear();
    p->h_push_peer.clear();
    p->h_push_slot.clear();
    if (p->parts != parts) {
        cudaFree(p->inflags);
        p->inflags = nullptr;
        GN_CUDA(cudaMalloc((void**)&p->inflags, 8 * (size_t)parts));  // its own allocation: IPC-exportable
    }
    if (!p->halo_bad) GN_CUDA(cudaMalloc((void**)&p->halo_bad, sizeof(int)));
    p->parts = parts;
    p->me = me;
    GN_CUDA(cudaMemset(p->inflags, 0, 8 * (size_t)parts));
    GN_CUDA(cudaMemset(p->halo_bad, 0, sizeof(int)));
    std::vector<int32_t> ex(expect, expect + nexpect);
    if (int rc = upload_into(&p->expect, ex)) return rc;
    p->nexpect = nexpect;
    return GN_OK;
}

int gn_part_peer_buffers(const gn_part* p, void** yg0, void** yg1, void** inflags) {
    if (!p || !p->yg[0]) return fail(GN_ERR_ARG, "gn_part_peer_buffers: call after gn_part_begin");
    if (yg0) *yg0 = p->yg[0];
    if (yg1) *yg1 = p->yg[1];
    if (inflags) *inflags = p->inflags;
    return GN_OK;
}

int gn_part_peer_add(gn_part* p, int rank, void* yg0, void* yg1, void* inflags, const int32_t* owned,
                     int64_t count, int64_t slot0) {
    if (!p || !yg0 || !yg1 || !inflags || count < 0 || (count > 0 && !owned) || slot0 < 0)
        return fail(GN_ERR_ARG, "bad gn_part_peer_add arguments");
    int idx = -1;
    for (size_t j = 0; j < p->peers.size(); ++j)
        if (p->peers[j].rank == rank) idx = (int)j;
    if (idx < 0) {
        idx = (int)p->peers.size();
        p->peers.push_back(gn_part::Peer{rank, {yg0, yg1}, (int64_t*)inflags});
    }
    for (int64_t i = 0; i < count; ++i) {
        if (owned[i] < 0 || owned[i] >= p->n_own) return fail(GN_ERR_ARG, "pushed row out of range");
        const int32_t row = p->h_inv[(size_t)owned[i]];
        if (row >= p->n_bnd) return fail(GN_ERR_ARG, "pushed row is not a boundary row (gn_part_set_boundary)");
        p->h_push_row.push_back(row);
        p->h_push_peer.push_back(idx);
        p->h_push_slot.push_back(slot0 + i);
    }
    return GN_OK;
}

int gn_part_peer_commit(gn_part* p) {
    if (!p) return fail(GN_ERR_ARG, "null partition");
    GN_CUDA(cudaSetDevice(p->device));
    part_free_push(p);
    const size_t np = p->h_push_row.size();
    // (peer, slot) order: each peer's ghost slots are one contiguous range
    std::vector<size_t> ord(np);
    for (size_t e = 0; e < np; ++e) ord[e] = e;
    std::sort(ord.begin(), ord.end(), [&](size_t a, size_t b) {
        return p->h_push_peer[a] != p->h_push_peer[b] ? p->h_push_peer[a] < p->h_push_peer[b]
                                                       : p->h_push_slot[a] < p->h_push_slot[b];
    });
    std::vector<int32_t> src(std::max<size_t>(np, 1)), peer(std::max<size_t>(np, 1));
    std::vector<int64_t> slot(std::max<size_t>(np, 1));
    for (size_t j = 0; j < np; ++j) {
        src[j] = p->h_push_row[ord[j]];
        peer[j] = p->h_push_peer[ord[j]];
        slot[j] = p->h_push_slot[ord[j]];
    }
    std::vector<void*> d0, d1;
    std::vector<int64_t*> fl;
    for (const auto& q : p->peers) {
        d0.push_back(q.yg[0]);
        d1.push_back(q.yg[1]);
        fl.push_back(q.flags);
    }
    int rc;
    if ((rc = upload_into(&p->push_src, src)) || (rc = upload_into(&p->push_peer, peer)) ||
        (rc = upload_into(&p->push_slot, slot)) || (rc = upload_into(&p->push_dst[0], d0)) ||
        (rc = upload_into(&p->push_dst[1], d1)) || (rc = upload_into(&p->peer_flags, fl)))
        return rc;
    p->n_push = (int64_t)np;
    p->npush_peers = (int)p->peers.size();
    p->gen++;
    return GN_OK;
}

static int part_wait(gn_part* p, int k, cudaStream_t s) {
    if (k == 0 || p->nexpect == 0) return GN_OK;  // step 0 reads the ghosts of x0
    k_part_wait<<<1, 32, 0, s>>>(p->inflags, p->expect, p->nexpect, p->d_epoch, k, p->halo_bad);
    GN_LAUNCHED();
    return GN_OK;
}

static int part_signal(gn_part* p, int k, cudaStream_t s) {
    if (p->npush_peers == 0) return GN_OK;
    k_part_signal<<<1, 32, 0, s>>>(p->peer_flags, p->npush_peers, p->me, p->d_epoch, (int64_t)k + 1);
    GN_LAUNCHED();
    return GN_OK;
}

int gn_part_peer_wait(gn_part* p, int k, uintptr_t stream) {
    if (!p || !p->inflags) return fail(GN_ERR_ARG, "gn_part_peer_wait before gn_part_peer_init");
    if (!p->d_epoch) return fail(GN_ERR_ARG, "gn_part_peer_wait before gn_part_begin");
    return part_wait(p, k, (cudaStream_t)stream);
}

int gn_part_peer_signal(gn_part* p, int k, uintptr_t stream) {
    if (!p || !p->peer_flags) return fail(GN_ERR_ARG, "gn_part_peer_signal before gn_part_peer_commit");
    if (!p->d_epoch) return fail(GN_ERR_ARG, "gn_part_peer_signal before gn_part_begin");
    return part_signal(p, k, (cudaStream_t)stream);
}

// Iterations [k0, k1) from a device-side schedule: the launches of every
// iteration -- with the direct halo: wait for the peers' flags, boundary
// rows, interior rows + pushes, flag the peers -- captured once into a CUDA
// graph and replayed with one cudaGraphLaunch (no host work per iteration).
// The graph names only buffers that stay put across runs (gn_part_begin) and
// reads the run epoch from device memory, so one capture serves every run of
// the same length and mode; it is rebuilt when the buffers or the push list
// change.
int gn_part_run(gn_part* p, int k0, int k1, uintptr_t stream) {
    GN_NVTX("gn_part_run");
    if (!p || k0 < 0 || k1 > p->iters || k0 >= k1 || !p->gam) return fail(GN_ERR_ARG, "bad gn_part_run arguments");
    GN_CUDA(cudaSetDevice(p->device));
    const bool peer = p->peer_flags != nullptr || p->nexpect > 0;
    if (!p->gexec || p->g_gen != p->gen || p->g_k0 != k0 || p->g_k1 != k1) {
        part_free_graph(p);
        cudaStream_t cs = p->own_stream;
        GN_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        int rc = GN_OK;
        const int64_t before = gn_launch_count();
        for (int k = k0; k < k1 && rc == GN_OK; ++k) {
            if (peer && p->inflags) rc = part_wait(p, k, cs);
            if (!rc) rc = part_step_range(p, k, 0, cs);
            if (!rc) rc = part_step_range(p, k, 1, cs);
            if (!rc && peer && p->peer_flags) rc = part_signal(p, k, cs);
        }
        const int64_t nodes = gn_launch_count() - before;
        note_launch(-nodes);  // counted when the graph runs
        cudaGraph_t graph = nullptr;
        cudaError_t e = cudaStreamEndCapture(cs, &graph);
        if (rc) {
            if (graph) cudaGraphDestroy(graph);
            return rc;
        }
        if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture", __FILE__, __LINE__);
        e = cudaGraphInstantiate(&p->gexec, graph, 0);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) {
            p->gexec = nullptr;
            return cuda_fail(e, "cudaGraphInstantiate", __FILE__, __LINE__);
        }
        p->g_gen = p->gen;
        p->g_k0 = k0;
        p->g_k1 = k1;
        p->g_nodes = nodes;
    }
    GN_CUDA(cudaGraphLaunch(p->gexec, (cudaStream_t)stream));
    note_launch(p->g_nodes);
    return GN_OK;
}

// All parts of one graph held by this process (e.g. one GPU): iterations
// [k0, k1) of every part interleaved in one captured schedule -- for each k,
// for each part: wait, boundary rows, interior rows + pushes, signal -- so a
// part's wait only ever finds flags that earlier nodes of the same stream
// have set (no kernel waits on one that may not be running).  The schedule
// of the multi-GPU run with the parts serialised; built, launched once and
// released (tests and single-GPU measurements).
int gn_part_run_group(gn_part* const* parts, int nparts, int k0, int k1, uintptr_t stream) {
    GN_NVTX("gn_part_run_group");
    if (!parts || nparts < 1) return fail(GN_ERR_ARG, "bad gn_part_run_group arguments");
    for (int i = 0; i < nparts; ++i)
        if (!parts[i] || k0 < 0 || k1 > parts[i]->iters || k0 >= k1 || !parts[i]->gam ||
            parts[i]->device != parts[0]->device)
            return fail(GN_ERR_ARG, "bad gn_part_run_group arguments");
    GN_CUDA(cudaSetDevice(parts[0]->device));
    cudaStream_t cs = parts[0]->own_stream;
    GN_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    int rc = GN_OK;
    const int64_t before = gn_launch_count();
    for (int k = k0; k < k1 && rc == GN_OK; ++k)
        for (int i = 0; i < nparts && rc == GN_OK; ++i) {
            gn_part* p = parts[i];
            if (p->inflags) rc = part_wait(p, k, cs);
            if (!rc) rc = part_step_range(p, k, 0, cs);
            if (!rc) rc = part_step_range(p, k, 1, cs);
            if (!rc && p->peer_flags) rc = part_signal(p, k, cs);
        }
    const int64_t nodes = gn_launch_count() - before;
    note_launch(-nodes);
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(cs, &graph);
    if (rc) {
        if (graph) cudaGraphDestroy(graph);
        return rc;
    }
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture", __FILE__, __LINE__);
    cudaGraphExec_t exec = nullptr;
    e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate", __FILE__, __LINE__);
    e = cudaGraphLaunch(exec, (cudaStream_t)stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize((cudaStream_t)stream);
    cudaGraphExecDestroy(exec);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGraphLaunch", __FILE__, __LINE__);
    note_launch(nodes);
    return GN_OK;
}

// CUDA IPC of one allocation (the peer buffers of another process on the node)
int gn_ipc_get_handle(const void* dptr, void* handle /* 64 bytes */) {
    if (!dptr || !handle) return fail(GN_ERR_ARG, "null argument");
    cudaIpcMemHandle_t h;
    GN_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(dptr)));
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    memcpy(handle, &h, sizeof(h));
    return GN_OK;
}

int gn_ipc_open_handle(const void* handle, int device, void** dptr) {
    if (!handle || !dptr) return fail(GN_ERR_ARG, "null argument");
    GN_CUDA(cudaSetDevice(device));
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    GN_CUDA(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
    return GN_OK;
}

int gn_ipc_close(void* dptr) {
    if (!dptr) return GN_OK;
    GN_CUDA(cudaIpcCloseMemHandle(dptr));
    return GN_OK;
}

// Measurement aid: time (ms per launch, CUDA events, `reps` launches after
// one warm-up) of one piece of iteration 0 of the current run, on the
// interior range (all rows when there is one part):
//   mode 0  k_part_step, the whole range
//   mode 1  k_part_step, only the warp-split long rows
//   mode 2  k_part_step, only the SELL slices (thread per row)
//   mode 3..6  the probe walk of the slices (k_part_probe MODE 1..4)
//   mode 7  the direct halo's push blocks alone (no rows; after
//           gn_part_peer_commit): the coalesced stores into the peers' slots
int gn_part_probe(gn_part* p, int mode, int reps, double* ms) {
    if (!p || !p->gam || mode < 0 || mode > 7 || reps < 1 || !ms) return fail(GN_ERR_ARG, "bad gn_part_probe arguments");
    if (mode == 7 && p->n_push == 0) { *ms = 0.0; return GN_OK; }
    GN_CUDA(cudaSetDevice(p->device));
    const int r = p->r_count[1] ? 1 : 0;
    if (!p->r_count[r]) { *ms = 0.0; return GN_OK; }
    cudaStream_t s = p->own_stream;
    const bool fast = !(p->flags & GN_EXACT);
    const int32_t* sell = fast ? p->sell_fast : p->sell;
    const int64_t pos0 = p->r_long[r] + p->r_csr[r];
    const int nsb = p->r_nblocks[r] - p->r_nbl[r] - p->r_ncb[r];
    double* out = nullptr;
    GN_CUDA(cudaMalloc((void**)&out, 8 * (size_t)std::max<int64_t>(p->r_count[r], 1)));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    PartPush none{nullptr, nullptr, nullptr, nullptr, 0, 0};
    auto launch = [&]() {
        if (mode == 7) {
            PartPush push{p->push_src, p->push_peer, p->push_slot, p->push_dst[1], p->n_push,
                          (int)std::min<int64_t>((p->n_push + 8 * kPartThreads - 1) / (8 * kPartThreads), 148)};
            const PartLong no_long{nullptr, nullptr, nullptr, 0, nullptr, 0, 0};
            by_dtype(p->dtype, [&](auto ts, auto tg) {
                launch_step<decltype(ts), decltype(tg)>(p, r, 0, push.nblocks, 0, 0, 0, 0, 0, push, no_long, s);
            });
        } else if (mode <= 2) {
            const int nbl = mode == 2 ? 0 : p->r_nbl[r];
            const int64_t ncsr = mode == 0 ? p->r_csr[r] : 0;
            const int ncb = mode == 0 ? p->r_ncb[r] : 0;
            const int64_t nsl = mode == 1 ? 0 : p->nsl[r];
            const int nb = mode == 1 ? std::max(nbl, 1) : mode == 2 ? std::max(nsb, 1) : p->r_nblocks[r];
            // mode 2 keeps the slices' order positions (pos0 = n_long + n_csr)
            const int64_t nlong_arg = mode == 2 ? pos0 : p->r_long[r];
            const PartLong lng = mode == 2 ? PartLong{nullptr, nullptr, nullptr, 0, nullptr, 0, 0} : part_long_of(p, r);
            by_dtype(p->dtype, [&](auto ts, auto tg) {
                if (mode != 1 || nbl > 0)
                    launch_step<decltype(ts), decltype(tg)>(p, r, 0, nb, nlong_arg, nbl, ncsr, ncb, nsl, none, lng, s);
                if (mode != 2 && p->r_long[r] > 0) launch_combine<decltype(ts), decltype(tg)>(p, r, 0, s);
            });
        } else {
            const int nb = std::max(nsb, 1);
            const uint32_t nall = (uint32_t)(p->n_own + p->n_ghost);
            const int64_t cnt = p->r_count[r];
            const int64_t* sp = p->slice_ptr + p->sl0[r];
            if (gather_bytes(p->dtype) == 4) {
                const float* y = (const float*)p->yg[0];
                if (mode == 3) k_part_probe<float, 1><<<nb, kPartThreads, 0, s>>>(sell, sp, p->nsl[r], cnt, pos0, y, nall, out);
                if (mode == 4) k_part_probe<float, 2><<<nb, kPartThreads, 0, s>>>(sell, sp, p->nsl[r], cnt, pos0, y, nall, out);
                if (mode == 5) k_part_probe<float, 3><<<nb, kPartThreads, 0, s>>>(sell, sp, p->nsl[r], cnt, pos0, y, nall, out);
                if (mode == 6) k_part_probe<float, 4><<<nb, kPartThreads, 0, s>>>(sell, sp, p->nsl[r], cnt, pos0, y, nall, out);
            } else {
                const double* y = (const double*)p->yg[0];
                if (mode == 3) k_part_probe<double, 1><<<nb, kPartThreads, 0, s>>>(sell, sp, p->nsl[r], cnt, pos0, y, nall, out);
                if (mode == 4) k_part_probe<double, 2><<<nb, kPartThreads, 0, s>>>(sell, sp, p->nsl[r], cnt, pos0, y, nall, out);
                if (mode == 5) k_part_probe<double, 3><<<nb, kPartThreads, 0, s>>>(sell, sp, p->nsl[r], cnt, pos0, y, nall, out);
                if (mode == 6) k_part_probe<double, 4><<<nb, kPartThreads, 0, s>>>(sell, sp, p->nsl[r], cnt, pos0, y, nall, out);
            }
        }
    };
    launch();
    cudaEventRecord(e0, s);
    for (int i = 0; i < reps; ++i) launch();
    cudaEventRecord(e1, s);
    cudaError_t e = cudaEventSynchronize(e1);
    float t = 0.f;
    cudaEventElapsedTime(&t, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    if (e != cudaSuccess) return cuda_fail(e, "gn_part_probe", __FILE__, __LINE__);
    GN_LAUNCHED();
    *ms = (double)t / reps;
    return GN_OK;
}

// Measurement aid (GN_PART_COUNT=1 at gn_part_begin): the gathers of values
// the run issued per iteration -- index-vector entries walked (padding
// included), certificate checks, the witness searches -- after `done`
// iterations (0 when counting was off)
int gn_part_gathers(gn_part* p, int done, int64_t* out) {
    if (!p || done < 0 || done > p->iters || (done > 0 && !out)) return fail(GN_ERR_ARG, "bad gn_part_gathers arguments");
    GN_CUDA(cudaSetDevice(p->device));
    GN_CUDA(cudaDeviceSynchronize());
    std::vector<unsigned long long> h(64 * (size_t)std::max(done, 1), 0ull);
    if (p->gat && done > 0) GN_CUDA(cudaMemcpy(h.data(), p->gat, 8 * 64 * (size_t)done, cudaMemcpyDeviceToHost));
    for (int k = 0; k < done; ++k) {
        unsigned long long t = 0;
        for (int j = 0; j < 64; ++j) t += h[(size_t)k * 64 + j];
        out[k] = p->gat_on ? (int64_t)t : 0;
    }
    return GN_OK;
}

int gn_part_info(const gn_part* p, int64_t* n_own, int64_t* n_ghost, int64_t* nnz) {
    if (!p) return fail(GN_ERR_ARG, "null partition");
    if (n_own) *n_own = p->n_own;
    if (n_ghost) *n_ghost = p->n_ghost;
    if (nnz) *nnz = p->nnz;
    return GN_OK;
}

}  // extern "C"
