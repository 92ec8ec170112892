/*
 * gn_b200.h -- C ABI of the B200 Graph-Normalization (GN) engine.
 *
 * The reference (graphnorm, pure Python) has no FFI; its "operator API" is the
 * Python function set exported by graphnorm/__init__.py:3-54.  Each entry
 * point below replaces the arithmetic behind one of those functions; the
 * Python drop-in (paper_2605_05330_b200) binds them with ctypes and keeps the
 * reference signatures, exceptions and messages.  Plain pointers and sizes
 * only -- no torch types.
 *
 * Conventions
 *   - every function returns int status (GN_OK = 0); gn_last_error() gives a
 *     thread-local message for the last failure on the calling thread;
 *   - host pointers unless GN_DEVICE_IO is set (then x0 / x_out are fp64
 *     device pointers, still in the caller's vertex order);
 *   - a gn_graph is immutable after creation and safe for concurrent use by
 *     any number of threads (reference: graph.py:31-33, SPEC "unrestricted
 *     concurrent reads"); each call runs on its own CUDA stream and
 *     workspace, so calls are re-entrant.
 */
#ifndef GN_B200_H
#define GN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GN_ABI_VERSION 1

/* dtypes of the device state
 *   GN_F64       binary64 throughout (the reference arithmetic)
 *   GN_F32       binary32 gathered values (what each vertex publishes to its
 *                neighbours, i.e. the bandwidth-bound stream), binary64
 *                per-vertex state, sums and update.  Keeps every vertex's own
 *                trajectory out of binary32's denormal range.
 *   GN_F32_PURE  binary32 throughout (matches the oracle's fp32 bitwise) */
#define GN_F64 0
#define GN_F32 1
#define GN_F32_PURE 2

/* status codes.  NEGATIVE / NOT_NORMALIZABLE / NONFINITE map one-to-one onto
 * the three NormalizationError raises of run_wrgn (dynamics.py:147,149,176). */
#define GN_OK 0
#define GN_ERR_ARG 1
#define GN_ERR_CUDA 2
#define GN_ERR_NEGATIVE 3
#define GN_ERR_NOT_NORMALIZABLE 4
#define GN_ERR_NONFINITE 5
#define GN_ERR_NOMEM 6
#define GN_ERR_NODEV 7
#define GN_ERR_ZERO_DENOM 8 /* fitness(): d <= 0 (dynamics.py:246-247) */
#define GN_ERR_ZERO_MASS 9  /* simplex_state(): mass <= 0 (dynamics.py:231-232) */
#define GN_ERR_FORMAT 10    /* gn_mwis_parse: io.py FormatError (message in err) */
#define GN_PARSE_FALLBACK 11 /* gn_mwis_parse: text outside the native grammar (see gn_io.cpp) */

/* run flags */
#define GN_TRACE 0x1u      /* energy / pre_energy per iteration (record_trace) */
#define GN_EARLY_EXIT 0x2u /* stop at gamma==final and step_inf < 1e-12 (dynamics.py:177) */
#define GN_EXACT 0x4u      /* one thread per row, sequential sums: bitwise equal to scipy */
#define GN_DEVICE_IO 0x8u  /* x0 / x_out are fp64 device pointers */
#define GN_NO_CHECK 0x10u  /* skip the x0 checks (gn_step has none: dynamics.py:111-119) */
#define GN_NO_CLIP 0x20u   /* return the raw state (gn_step) instead of clip(x,0,1) */
#define GN_NONFINITE_OK 0x40u /* do not stop on a non-finite state (gn_step) */

typedef struct gn_graph gn_graph;

typedef struct gn_run_stats {
    double loop_ms;        /* CUDA-event time of the device loop kernel(s) */
    double total_ms;       /* CUDA-event time of the whole call incl. copies */
    int64_t launches;      /* kernels this call launched */
    int64_t grid_blocks;   /* blocks of the persistent loop kernel */
    int64_t block_threads; /* threads per block */
    int64_t h2d_bytes;     /* host->device bytes of the call */
    int64_t d2h_bytes;     /* device->host bytes of the call */
} gn_run_stats;

int gn_abi_version(void);
const char* gn_last_error(void);
int gn_device_count(int* count);
/* total kernels launched by this process through the engine */
int64_t gn_launch_count(void);

/* WeightedGraph (graph.py:22-75): CSR with sorted, symmetric, deduplicated
 * rows; w > 0.  v = sqrt(w) is formed on the device (IEEE sqrt, bitwise equal
 * to numpy's).  Column indices are int32 (as scipy's csr copy, graph.py:46).
 * gn_graph_set_grid(g, b > 0) overrides the persistent grid size (tuning). */
int gn_graph_create(int64_t n, const int64_t* indptr, const int32_t* indices,
                    const double* w, int dtype, int device, gn_graph** out);
int gn_graph_destroy(gn_graph* g);
int gn_graph_info(const gn_graph* g, int64_t* n, int64_t* nnz, int* dtype,
                  int* device, int64_t* device_bytes, int* num_bins);
int gn_graph_set_grid(gn_graph* g, int blocks);

/* run_wrgn (dynamics.py:129-180).  gammas[k] = schedule.gamma_at(k) for
 * k < iters (computed on the host with the reference formula, bitwise).
 * Outputs (host, may be NULL): x_out (n fp64, clipped to [0,1]);
 * step_inf / fallbacks (iters); mass[k] = w.x_{k+1} (the objective);
 * energy / pre_energy (iters, GN_TRACE); x_hist (iters*n fp64, test aid).
 * *iters_run = trace length; on GN_ERR_NONFINITE *fail_iter = k. */
int gn_run(gn_graph* g, const void* x0, const double* gammas, int iters,
           double final_gamma, uint32_t flags, void* x_out, double* step_inf,
           int64_t* fallbacks, double* mass, double* energy, double* pre_energy,
           double* x_hist, int* iters_run, int* fail_iter, gn_run_stats* stats);

/* gn_step (dynamics.py:111-119): one unclipped, unchecked step. */
int gn_step(gn_graph* g, const double* x, double gamma, uint32_t flags,
            double* out, int64_t* nfb);

/* is_normalizable (dynamics.py:122-126): all(x + A x > 0). */
int gn_is_normalizable(gn_graph* g, const double* x, int* ok);
/* out = A @ in, fp64, per-row sequential order (scipy csr_matvec). */
int gn_spmv(gn_graph* g, const double* in, double* out);
/* energy (dynamics.py:210-219) and weighted_mass (222-224), fp64. */
int gn_energy(gn_graph* g, const double* x, double gamma, double* energy);
int gn_weighted_mass(gn_graph* g, const double* x, double* mass);
/* simplex_state (dynamics.py:227-233) and fitness (236-250), fp64. */
int gn_simplex_state(gn_graph* g, const double* x, double* p_out);
int gn_fitness(gn_graph* g, const double* p, double gamma, double* f_out,
               double* fbar);

/* round_to_mis (dynamics.py:253-277) + MisSolution.from_members
 * (graph.py:178-186).  x is host fp64 (or, with GN_DEVICE_IO, a device fp64
 * array).  selected: n bytes (0/1).  weight is numpy's pairwise
 * sum over members in ascending order (bitwise equal to w[idx].sum()). */
int gn_round(gn_graph* g, const void* x, uint32_t flags, uint8_t* selected,
             double* weight, int* independent, int* maximal, int64_t* count);
/* gn_round returning the members themselves: members (capacity n) receives
 * the *count selected vertex ids in ascending order, compacted on the device
 * (what MisSolution.members holds; replaces the host scan of the mask). */
int gn_round_members(gn_graph* g, const void* x, uint32_t flags,
                     int64_t* members, double* weight, int* independent,
                     int* maximal, int64_t* count);
/* round_to_mis of num_states states (x: [num_states][n] fp64, host or, with
 * GN_DEVICE_IO, device) with one synchronisation: selected [num_states][n]
 * (may be NULL), weight / independent / maximal / count [num_states]. */
int gn_round_many(gn_graph* g, int num_states, const void* x, uint32_t flags,
                  uint8_t* selected, double* weight, int* independent,
                  int* maximal, int64_t* count);
/* is_independent / is_maximal_independent / set_weight (graph.py:134-162)
 * on a 0/1 membership mask. */
int gn_check_members(gn_graph* g, const uint8_t* mask, double* weight,
                     int* independent, int* maximal, int64_t* count);

/* ---- several starts on one graph (solver.py:100-153) ----
 * num_starts trajectories of run_wrgn on the same graph and schedule,
 * advanced together (state stored start-minor, so one contiguous read per
 * neighbour serves every start).  x0 / x_out are [num_starts][n] fp64,
 * original order.  Each start is bitwise its own gn_run(GN_EXACT) run: per
 * start checks (status GN_ERR_NEGATIVE / GN_ERR_NOT_NORMALIZABLE: not run),
 * non-finite stop (GN_ERR_NONFINITE, fail_iter) and early exit.  Outputs
 * step_inf / fallbacks are [num_starts][iters] (entries past iters_run[b]
 * untouched); iters_run / status / fail_iter are [num_starts].  Returns
 * GN_OK, or the first failing start's code.  1 <= num_starts <= 64.
 * Flags: GN_EXACT (no row splitting: bitwise per start), GN_EARLY_EXIT,
 * GN_NO_CHECK, GN_NO_CLIP, GN_NONFINITE_OK, GN_DEVICE_IO (x0 / x_out are
 * device fp64 arrays). */
int gn_multi_run(gn_graph* g, int num_starts, const double* x0,
                 const double* gammas, int iters, double final_gamma,
                 uint32_t flags, double* x_out, double* step_inf,
                 int64_t* fallbacks, int* iters_run, int* status,
                 int* fail_iter, gn_run_stats* stats);

/* ---- batches of independent graphs (BASELINE config C4) ----
 * B graphs packed block-diagonally: graph b owns vertices
 * [offsets[b], offsets[b+1]) and no edge leaves it.  Each graph runs its own
 * run_wrgn (per-graph checks, early exit, non-finite stop) -- bitwise what
 * gn_run gives graph by graph -- on one CTA with the graph resident in shared
 * memory.  Graphs must have <= 4096 vertices and fit in shared memory.
 * Outputs are per graph: step_inf / fallbacks / mass are [B][iters],
 * iters_run / status (GN_OK or the gn_run error code) / fail_iter are [B];
 * trace entries past a graph's iters_run are written as 0. */
typedef struct gn_batch gn_batch;
int gn_batch_create(int64_t num_graphs, const int64_t* offsets, int64_t n,
                    const int64_t* indptr, const int32_t* indices,
                    const double* w, int dtype, int device, gn_batch** out);
int gn_batch_destroy(gn_batch* b);
int gn_batch_info(const gn_batch* b, int64_t* num_graphs, int64_t* n,
                  int64_t* device_bytes, int64_t* smem_bytes);
int gn_batch_run(gn_batch* b, const void* x0, const double* gammas, int iters,
                 double final_gamma, uint32_t flags, void* x_out,
                 double* step_inf, int64_t* fallbacks, double* mass,
                 int* iters_run, int* status, int* fail_iter,
                 gn_run_stats* stats);

/* ---- one vertex-range partition of a graph ----
 * Owned vertices [0, n_own) and ghosts [n_own, n_own + n_ghost) (grouped by
 * owning peer); indptr/indices: the owned rows over local ids, neighbour
 * order as in the global graph; w: n_own + n_ghost weights.  Per iteration k
 * on `stream` (a cudaStream_t; 0 = the legacy default stream): gn_part_step, then the halo:
 * gn_part_pack (owned values at d_idx -> contiguous device buffer), the
 * caller's exchange (NCCL send/recv on the same stream), gn_part_unpack
 * (device buffer -> ghost slots [ghost_first, ghost_first + count)).
 * gn_part_end returns x (clipped) and the owned rows' per-iteration stats
 * (max|dx|, fallbacks, w.x'); the caller reduces them over partitions. */
typedef struct gn_part gn_part;
int gn_part_create(int64_t n_own, int64_t n_ghost, const int64_t* indptr,
                   const int32_t* indices, const double* w, int dtype,
                   int device, gn_part** out);
int gn_part_destroy(gn_part* p);
int gn_part_info(const gn_part* p, int64_t* n_own, int64_t* n_ghost, int64_t* nnz);
int gn_part_elem_bytes(const gn_part* p);
int gn_part_begin(gn_part* p, const double* x0, const double* gammas, int iters,
                  uint32_t flags);
int gn_part_step(gn_part* p, int k, uintptr_t stream);
/* Overlap of the halo with the step: gn_part_set_boundary names the owned
 * rows peers hold as ghosts (call before gn_part_begin); then per iteration
 * gn_part_step_range(which = 0: boundary rows), pack and post the exchange,
 * gn_part_step_range(which = 1: interior rows) while it is in flight, wait,
 * unpack.  gn_part_step runs both ranges. */
int gn_part_set_boundary(gn_part* p, const int32_t* rows, int64_t count);
int gn_part_step_range(gn_part* p, int k, int which, uintptr_t stream);
int gn_part_pack(gn_part* p, int k, const int32_t* d_idx, int64_t count,
                 void* d_out, uintptr_t stream);
int gn_part_unpack(gn_part* p, int k, const void* d_in, int64_t ghost_first,
                   int64_t count, uintptr_t stream);
int gn_part_end(gn_part* p, int done, double* x_out, double* step_inf,
                int64_t* fallbacks, double* mass, int* bad);
/* Direct halo over peer memory (the fused alternative to pack + NCCL +
 * unpack): the interior step's first blocks copy the boundary rows' new
 * values straight into the ghost slots of the peers that hold them (P2P
 * stores over NVLink, sorted by (peer, slot) so a warp writes 32 consecutive
 * slots, overlapped with the interior rows), then a flag per peer.  Sequence,
 * after the first gn_part_begin: gn_part_peer_init (this part's rank, the
 * peers that push to it), gn_part_peer_buffers (yg[2] and the flag array to
 * hand to the peers: pointers in one process, gn_ipc_get_handle across
 * processes), gn_part_peer_add per peer (its buffers, the caller's owned ids
 * it holds as ghosts, in its ghost order, and the slot of the first of them
 * in its yg), gn_part_peer_commit.  The buffers stay put across later runs
 * of the same length, so the setup is done once.  Per iteration k:
 * gn_part_peer_wait, gn_part_step (the interior launch pushes),
 * gn_part_peer_signal -- or all iterations at once with gn_part_run.
 * Flags carry the run epoch (one per gn_part_begin; all parts of a run call
 * it equally often): a late flag of an earlier run cannot satisfy a wait.
 * Between runs the caller fences every rank (device sync + barrier) before
 * gn_part_begin and again after it, before the first step. */
int gn_part_peer_init(gn_part* p, int parts, int me, const int32_t* expect, int nexpect);
int gn_part_peer_buffers(const gn_part* p, void** yg0, void** yg1, void** inflags);
int gn_part_peer_add(gn_part* p, int rank, void* yg0, void* yg1, void* inflags,
                     const int32_t* owned, int64_t count, int64_t slot0);
int gn_part_peer_commit(gn_part* p);
int gn_part_peer_wait(gn_part* p, int k, uintptr_t stream);
int gn_part_peer_signal(gn_part* p, int k, uintptr_t stream);
/* Iterations [k0, k1) of the current run from a device-side schedule: the
 * per-iteration launches (with the direct halo: wait, boundary rows,
 * interior rows + pushes, signal) captured once into a CUDA graph and
 * replayed with one launch on `stream`; no host work per iteration.  Replaces
 * the Python loop over dynamics.py:155-178. */
int gn_part_run(gn_part* p, int k0, int k1, uintptr_t stream);
/* Every part of one graph held by this process (one device): iterations
 * [k0, k1) of all parts interleaved in one captured schedule (per k, per
 * part: wait, boundary, interior + pushes, signal), launched once on
 * `stream` and synchronised -- the multi-GPU schedule with the parts run one
 * after another, so no wait depends on a kernel that is not already done. */
int gn_part_run_group(gn_part* const* parts, int nparts, int k0, int k1, uintptr_t stream);
/* Measurement aid (not on the solve path): ms per launch of one piece of
 * iteration 0 of the current run on the interior range -- mode 0 the step
 * kernel, 1 its warp-split long rows only, 2 its SELL slices only, 3..6 the
 * slices' gather walk alone with real gathers / no gathers (index stream
 * only) / L1-resident gathers / random gathers.  Call after gn_part_begin. */
int gn_part_probe(gn_part* p, int mode, int reps, double* ms);
/* Measurement aid: with GN_PART_COUNT=1 set at gn_part_begin, the value
 * gathers the run issued per iteration (index-vector entries walked, padding
 * included; zero-row certificate checks; witness searches) -- how much of the
 * adjacency the zero-row certificates and settled rows let the steps skip
 * (out[k] = 0 when counting was off, or with the certificates off).
 * GN_PART_COUNT=2: the rows of the slice path that walked; 3: its slices
 * with a walking row.  Replaces nothing in the reference: dynamics.py:105
 * always gathers every entry. */
int gn_part_gathers(gn_part* p, int done, int64_t* out);
/* CUDA IPC of one device allocation between the processes of a node. */
int gn_ipc_get_handle(const void* dptr, void* handle /* 64 bytes */);
int gn_ipc_open_handle(const void* handle, int device, void** dptr);
int gn_ipc_close(void* dptr);

/* ---- graph generation on the device (BASELINE config C5) ----
 * R-MAT with 2^scale vertices and edge_factor * 2^scale samples, quadrant
 * probabilities (a, b, c, 1-a-b-c); self-loops dropped, symmetrised,
 * deduplicated; the same counter-based stream as generators.rmat_pairs.
 * Returns a canonical CSR in host arrays the caller frees with gn_free_host. */
int gn_gen_rmat(int scale, int edge_factor, double a, double b, double c,
                uint64_t seed, int device, int64_t* nnz, int64_t** indptr,
                int32_t** indices);
/* Canonical CSR (graph.py:78-124 build_graph, minus the weights) from an
 * edge list u[m], v[m] (int64, any orientation, duplicates allowed) on the
 * device: sort, deduplicate, symmetrise, sort.  Returns GN_ERR_ARG with
 * *first_bad = the first edge (input order) that leaves [0, n) or is a
 * self-loop.  *indptr_out (n+1 int64) / *indices_out (nnz int32) are
 * released with gn_free_host. */
int gn_csr_from_edges(int64_t n, int64_t m, const int64_t* u, const int64_t* v,
                      int device, int64_t* first_bad, int64_t* nnz_out,
                      int64_t** indptr_out, int32_t** indices_out);
void gn_free_host(void* p);

/* ---- instance text ------------------------------------
 * gn_mwis_parse replaces io.py:43-102 parse_instance up to its build_graph
 * call: the DIMACS-flavoured MWIS text (len bytes) is checked line by line
 * with the reference's rules and messages.  GN_OK: *out holds n, the
 * weights (1-based id i at w[i-1]) and the 0-based edges in file order
 * (gn_mwis_info / gn_mwis_copy, released by gn_mwis_free); the caller builds
 * the graph (build_graph, graph.py:78-124).  GN_ERR_FORMAT: err holds the
 * FormatError text.  GN_PARSE_FALLBACK: the text uses what only Python's
 * int()/float()/str methods read (non-ASCII, '_', huge integers, ...). */
typedef struct gn_mwis gn_mwis;
int gn_mwis_parse(const char* text, int64_t len, gn_mwis** out, char* err, int64_t err_len);
int gn_mwis_info(const gn_mwis* r, int64_t* n, int64_t* m);
int gn_mwis_copy(const gn_mwis* r, double* w, int64_t* edges /* [m][2] */);
void gn_mwis_free(gn_mwis* r);

#ifdef __cplusplus
}
#endif
#endif /* GN_B200_H */
