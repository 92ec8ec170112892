/*
 * gn_oracle.c -- CPU restatement of the graphnorm GN hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package links or calls
 * this file; it is the checker for the CUDA engine (tests/, the smoke()
 * entry, and bench.py's cpu_baseline / --impl reference leg).
 *
 * Each function restates one reference routine of
 * /root/reference/pkg/src/graphnorm (cited as dynamics.py:L / graph.py:L)
 * in plain C with the same IEEE-754 operation order:
 *
 *   - the SpMV A@y is scipy's csr_matvec: per row, a sequential sum in stored
 *     (ascending) neighbour order starting from 0.0 (dynamics.py:105);
 *   - the update keeps the reference's exact elementwise formula
 *     y = v*x, d = y + gamma*s, x' = d > 1e-9 ? y/d : 0.5 (dynamics.py:102-108)
 *     with no FMA contraction (compile with -ffp-contract=off);
 *   - numpy's float64 pairwise summation (blocks of 128, 8 accumulators) is
 *     restated for the MIS weight so it is bitwise equal to w[idx].sum()
 *     (graph.py:182).
 *
 * The fp64 path is pinned bitwise against golden vectors produced by the
 * reference itself (tests/golden/make_golden.py).  The fp32 path is the same
 * algorithm carried out in binary32; it is the same-precision checker for the
 * engine's fp32 EXACT mode.
 *
 * Rows are independent within one step, so the row loop may run on several
 * OpenMP threads without changing any bit of x; max/count reductions are
 * order-free.  Dot products (trace mode, objective) are folded from fixed
 * row chunks in chunk order (see GNO_CHUNK), independent of the thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define GNO_OK 0
#define GNO_ERR_ARG 1
#define GNO_ERR_NEGATIVE 3
#define GNO_ERR_NOT_NORMALIZABLE 4
#define GNO_ERR_NONFINITE 5

#define GNO_TRACE 1u
#define GNO_EARLY_EXIT 2u

/* dynamics.py:21-22 */
static const double SAFE_DIV_THRESHOLD = 1e-9;
static const double FALLBACK_VALUE = 0.5;

static void set_threads(int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
}

int gno_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* out = A @ in, sequential per-row order (scipy csr_matvec, dynamics.py:105). */
void gno_spmv(int64_t n, const int64_t* indptr, const int32_t* indices,
              const double* in, double* out) {
    for (int64_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) s += in[indices[p]];
        out[i] = s;
    }
}

/* ---------------------------------------------------------------------------
 * Threading.  One step's rows are cut into fixed chunks of GNO_CHUNK rows
 * (independent of the thread count); OpenMP threads take chunks dynamically
 * (R-MAT puts its hubs at low ids) and each chunk keeps its own fallback
 * count, max|dx|, finiteness and the three dot products of energy() /
 * weighted_mass() (dynamics.py:210-224).  The chunk partials are then folded
 * in chunk order, so every output -- x bitwise, and the dots too -- is the
 * same for any number of threads.  (The reference's w @ x is a BLAS ddot,
 * itself not a sequential sum; the dots are compared at 1e-12.)
 * ------------------------------------------------------------------------- */
#define GNO_CHUNK 4096

typedef struct {
    int64_t fb;
    double mx;
    int fin;
    double d1, d2, d3;
} chunk_part;

static chunk_part* parts_alloc(int64_t n, int64_t* nch) {
    *nch = (n + GNO_CHUNK - 1) / GNO_CHUNK;
    return (chunk_part*)calloc((size_t)(*nch ? *nch : 1), sizeof(chunk_part));
}

static void parts_fold(const chunk_part* P, int64_t nch, int64_t* nfb, double* step_inf,
                       int* finite, double* dots) {
    int64_t fb = 0;
    double mx = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
    int fin = 1;
    for (int64_t c = 0; c < nch; ++c) {
        fb += P[c].fb;
        if (P[c].mx > mx) mx = P[c].mx;
        fin = fin && P[c].fin;
        d1 += P[c].d1; d2 += P[c].d2; d3 += P[c].d3;
    }
    *nfb = fb;
    *step_inf = mx;
    *finite = fin;
    if (dots) { dots[0] = d1; dots[1] = d2; dots[2] = d3; }
}

/* ---------------------------------------------------------------------------
 * One step, fp64: dynamics.py:_step 102-108.  Also returns max|x'-x|
 * (run_wrgn's step_inf, dynamics.py:165) and the isfinite verdict
 * (dynamics.py:175).  When dots != NULL it also returns y.y, y.(Ay) and w.x
 * of the PRE-step state (the three terms of energy(), dynamics.py:210-219).
 * ------------------------------------------------------------------------- */
static void step_f64(int64_t n, const int64_t* indptr, const int32_t* indices,
                     const double* v, const double* w, const double* x,
                     const double* y, double gamma, double* xo, double* yo,
                     int64_t* nfb, double* step_inf, int* finite, double* dots) {
    int64_t nch;
    chunk_part* P = parts_alloc(n, &nch);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t c = 0; c < nch; ++c) {
        int64_t lo = c * GNO_CHUNK, hi = lo + GNO_CHUNK < n ? lo + GNO_CHUNK : n;
        chunk_part q = {0, 0.0, 1, 0.0, 0.0, 0.0};
        for (int64_t i = lo; i < hi; ++i) {
            double s = 0.0;
            for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) s += y[indices[p]];
            double yi = y[i];
            double d = yi + gamma * s;
            double o;
            if (d > SAFE_DIV_THRESHOLD) o = yi / d; else { o = FALLBACK_VALUE; ++q.fb; }
            xo[i] = o;
            yo[i] = v[i] * o;
            double diff = fabs(o - x[i]);
            if (diff > q.mx) q.mx = diff;
            if (!isfinite(o)) q.fin = 0;
            q.d1 += yi * yi;
            q.d2 += yi * s;
            q.d3 += w[i] * x[i];
        }
        P[c] = q;
    }
    parts_fold(P, nch, nfb, step_inf, finite, dots);
    free(P);
}

/* Same step carried out in binary32 (the engine's fp32 arithmetic). */
static void step_f32(int64_t n, const int64_t* indptr, const int32_t* indices,
                     const float* v, const float* w, const float* x,
                     const float* y, float gamma, float* xo, float* yo,
                     int64_t* nfb, double* step_inf, int* finite, double* dots) {
    int64_t nch;
    chunk_part* P = parts_alloc(n, &nch);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t c = 0; c < nch; ++c) {
        int64_t lo = c * GNO_CHUNK, hi = lo + GNO_CHUNK < n ? lo + GNO_CHUNK : n;
        chunk_part q = {0, 0.0, 1, 0.0, 0.0, 0.0};
        float mx = 0.0f;
        for (int64_t i = lo; i < hi; ++i) {
            float s = 0.0f;
            for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) s += y[indices[p]];
            float yi = y[i];
            float d = yi + gamma * s;
            float o;
            if ((double)d > SAFE_DIV_THRESHOLD) o = yi / d; else { o = (float)FALLBACK_VALUE; ++q.fb; }
            xo[i] = o;
            yo[i] = v[i] * o;
            float diff = fabsf(o - x[i]);
            if (diff > mx) mx = diff;
            if (!isfinite(o)) q.fin = 0;
            q.d1 += (double)yi * (double)yi;
            q.d2 += (double)yi * (double)s;
            q.d3 += (double)w[i] * (double)x[i];
        }
        q.mx = (double)mx;
        P[c] = q;
    }
    parts_fold(P, nch, nfb, step_inf, finite, dots);
    free(P);
}


/* Mixed precision (the engine's GN_F32 data path): per-vertex state, sums
 * and the update in fp64; the value each vertex publishes to its neighbours
 * is rounded to binary32 (yg = (float)(v*x)).  Same step as step_f64
 * otherwise. */
static void step_mixed(int64_t n, const int64_t* indptr, const int32_t* indices,
                       const double* v, const double* w, const double* x,
                       const float* yg, double gamma, double* xo, float* ygo,
                       int64_t* nfb, double* step_inf, int* finite, double* dots) {
    int64_t nch;
    chunk_part* P = parts_alloc(n, &nch);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t c = 0; c < nch; ++c) {
        int64_t lo = c * GNO_CHUNK, hi = lo + GNO_CHUNK < n ? lo + GNO_CHUNK : n;
        chunk_part q = {0, 0.0, 1, 0.0, 0.0, 0.0};
        for (int64_t i = lo; i < hi; ++i) {
            double s = 0.0;
            for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) s += (double)yg[indices[p]];
            double yi = v[i] * x[i];
            double d = yi + gamma * s;
            double o;
            if (d > SAFE_DIV_THRESHOLD) o = yi / d; else { o = FALLBACK_VALUE; ++q.fb; }
            xo[i] = o;
            ygo[i] = (float)(v[i] * o);
            double diff = fabs(o - x[i]);
            if (diff > q.mx) q.mx = diff;
            if (!isfinite(o)) q.fin = 0;
            q.d1 += yi * yi;
            q.d2 += yi * s;
            q.d3 += w[i] * x[i];
        }
        P[c] = q;
    }
    parts_fold(P, nch, nfb, step_inf, finite, dots);
    free(P);
}

/* The dots of a state without stepping (the trace tail after the last step):
 * the same chunked fold as the steps' pre-state dots. */
static void dots_f64(int64_t n, const int64_t* indptr, const int32_t* indices,
                     const double* w, const double* x, const double* y, double* dots) {
    int64_t nch;
    chunk_part* P = parts_alloc(n, &nch);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t c = 0; c < nch; ++c) {
        int64_t lo = c * GNO_CHUNK, hi = lo + GNO_CHUNK < n ? lo + GNO_CHUNK : n;
        chunk_part q = {0, 0.0, 1, 0.0, 0.0, 0.0};
        for (int64_t i = lo; i < hi; ++i) {
            double s = 0.0;
            for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) s += y[indices[p]];
            q.d1 += y[i] * y[i];
            q.d2 += y[i] * s;
            q.d3 += w[i] * x[i];
        }
        P[c] = q;
    }
    int64_t fb; double mx; int fin;
    parts_fold(P, nch, &fb, &mx, &fin, dots);
    free(P);
}

static void dots_mixed(int64_t n, const int64_t* indptr, const int32_t* indices,
                       const double* v, const double* w, const double* x, const float* yg, double* dots) {
    int64_t nch;
    chunk_part* P = parts_alloc(n, &nch);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t c = 0; c < nch; ++c) {
        int64_t lo = c * GNO_CHUNK, hi = lo + GNO_CHUNK < n ? lo + GNO_CHUNK : n;
        chunk_part q = {0, 0.0, 1, 0.0, 0.0, 0.0};
        for (int64_t i = lo; i < hi; ++i) {
            double s = 0.0;
            for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) s += (double)yg[indices[p]];
            double yi = v[i] * x[i];
            q.d1 += yi * yi;
            q.d2 += yi * s;
            q.d3 += w[i] * x[i];
        }
        P[c] = q;
    }
    int64_t fb; double mx; int fin;
    parts_fold(P, nch, &fb, &mx, &fin, dots);
    free(P);
}

static void dots_f32(int64_t n, const int64_t* indptr, const int32_t* indices,
                     const float* w, const float* x, const float* y, double* dots) {
    int64_t nch;
    chunk_part* P = parts_alloc(n, &nch);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t c = 0; c < nch; ++c) {
        int64_t lo = c * GNO_CHUNK, hi = lo + GNO_CHUNK < n ? lo + GNO_CHUNK : n;
        chunk_part q = {0, 0.0, 1, 0.0, 0.0, 0.0};
        for (int64_t i = lo; i < hi; ++i) {
            float s = 0.0f;
            for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p) s += y[indices[p]];
            q.d1 += (double)y[i] * (double)y[i];
            q.d2 += (double)y[i] * (double)s;
            q.d3 += (double)w[i] * (double)x[i];
        }
        P[c] = q;
    }
    int64_t fb; double mx; int fin;
    parts_fold(P, nch, &fb, &mx, &fin, dots);
    free(P);
}

/* energy from the three dots: dynamics.py:219 */
static double energy_of(const double* dots, double gamma) {
    return 0.5 * (dots[0] + gamma * dots[1]) - dots[2];
}

/* The dots of step k's PRE-step state x_k are the post-step terms of
 * iteration k-1 (energy(x_k, gamma_{k-1}) and w.x_k, dynamics.py:170-173) and
 * the pre-energy of iteration k (dynamics.py:163): one SpMV per iteration
 * serves both, and only the state after the last step needs its own pass
 * (k == iters_run, called after the loop). */
static void post_dots(int k, int tail, const double* gammas, const double* dots, int trace,
                      double* energy, double* pre_energy, double* mass) {
    if (trace && !tail) pre_energy[k] = energy_of(dots, gammas[k]);
    if (k > 0) {
        if (trace) energy[k - 1] = energy_of(dots, gammas[k - 1]);
        if (mass) mass[k - 1] = dots[2];
    }
}

/* Public single step (gn_step, dynamics.py:111-119), fp64. */
int gno_step(int64_t n, const int64_t* indptr, const int32_t* indices,
             const double* w, const double* x, double gamma, double* out,
             int64_t* nfb, int nthreads) {
    set_threads(nthreads);
    double* v = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
    double* y = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
    double* yo = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
    for (int64_t i = 0; i < n; ++i) { v[i] = sqrt(w[i]); y[i] = v[i] * x[i]; }
    double si; int fin; int64_t fb;
    step_f64(n, indptr, indices, v, w, x, y, gamma, out, yo, &fb, &si, &fin, NULL);
    if (nfb) *nfb = fb;
    free(v); free(y); free(yo);
    return GNO_OK;
}

/* ---------------------------------------------------------------------------
 * run_wrgn (dynamics.py:129-180).
 *   dtype 0 = fp64 (the reference arithmetic), 1 = binary32 throughout,
 *   2 = mixed (fp64 state and sums, binary32 gathered values).
 *   gammas[k] = schedule.gamma_at(k) precomputed by the caller (bitwise).
 *   x_hist (optional): iters*n fp64, row k = state after step k, unclipped.
 *   snaps/x_snap (optional): ascending iteration indices; row j of x_snap
 *   (nsnap*n fp64) = the state after step snaps[j], unclipped (sampled
 *   per-iteration checks of large instances without a full history).
 *   mass (optional): w . x_{k+1}, sequential.  energy/pre_energy need TRACE.
 * Returns GNO_OK or an error; on GNO_ERR_NONFINITE, *fail_iter = k.
 * ------------------------------------------------------------------------- */
int gno_run(int dtype, int64_t n, const int64_t* indptr, const int32_t* indices,
            const double* w, const double* x0, const double* gammas, int iters,
            double final_gamma, unsigned flags, int nthreads,
            double* x_out, double* step_inf, int64_t* fallbacks, double* mass,
            double* energy, double* pre_energy, double* x_hist,
            const int* snaps, int nsnap, double* x_snap,
            int* iters_run, int* fail_iter) {
    set_threads(nthreads);
    if (n < 0 || iters < 1) return GNO_ERR_ARG;
    const int trace = (flags & GNO_TRACE) != 0;
    const int early = (flags & GNO_EARLY_EXIT) != 0;
    *iters_run = 0;
    *fail_iter = -1;
    /* dynamics.py:145-149: negativity, then the unweighted closed sums */
    for (int64_t i = 0; i < n; ++i)
        if (x0[i] < 0.0) return GNO_ERR_NEGATIVE;
    {
        double* ax = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
        gno_spmv(n, indptr, indices, x0, ax);
        int ok = 1;
        for (int64_t i = 0; i < n; ++i)
            if (!(x0[i] + ax[i] > 0.0)) { ok = 0; break; }
        free(ax);
        if (!ok) return GNO_ERR_NOT_NORMALIZABLE;
    }
    size_t nb = (size_t)(n ? n : 1);
    double dots[3];
    const int want_dots = trace || mass;
    int rc = GNO_OK;
    int k, ran = 0, sj = 0;
    if (dtype == 0) {
        double* v = (double*)malloc(sizeof(double) * nb);
        double* xa = (double*)malloc(sizeof(double) * nb);
        double* ya = (double*)malloc(sizeof(double) * nb);
        double* xb = (double*)malloc(sizeof(double) * nb);
        double* yb = (double*)malloc(sizeof(double) * nb);
        for (int64_t i = 0; i < n; ++i) {
            v[i] = sqrt(w[i]);            /* graph.py:42 */
            xa[i] = x0[i];
            ya[i] = v[i] * xa[i];         /* dynamics.py:104 */
        }
        for (k = 0; k < iters; ++k) {
            double g = gammas[k], si;
            int fin;
            int64_t fb;
            step_f64(n, indptr, indices, v, w, xa, ya, g, xb, yb, &fb, &si, &fin,
                     want_dots ? dots : NULL);
            if (n == 0) si = 0.0;
            step_inf[k] = si;
            fallbacks[k] = fb;
            if (want_dots) post_dots(k, 0, gammas, dots, trace, energy, pre_energy, mass);
            if (x_hist) memcpy(x_hist + (size_t)k * (size_t)n, xb, sizeof(double) * (size_t)n);
            while (x_snap && sj < nsnap && snaps[sj] == k) memcpy(x_snap + (size_t)(sj++) * (size_t)n, xb, sizeof(double) * (size_t)n);
            double* t;
            t = xa; xa = xb; xb = t;
            t = ya; ya = yb; yb = t;
            ran = k + 1;
            if (!fin) { rc = GNO_ERR_NONFINITE; *fail_iter = k; break; }
            if (early && g == final_gamma && si < 1e-12) break;   /* dynamics.py:177 */
        }
        *iters_run = ran;
        if (want_dots && ran > 0) {
            dots_f64(n, indptr, indices, w, xa, ya, dots);
            post_dots(ran, 1, gammas, dots, trace, energy, pre_energy, mass);
        }
        for (int64_t i = 0; i < n; ++i) {  /* np.clip, dynamics.py:179 */
            double xi = xa[i];
            x_out[i] = xi < 0.0 ? 0.0 : (xi > 1.0 ? 1.0 : xi);
        }
        free(v); free(xa); free(ya); free(xb); free(yb);
    } else if (dtype == 2) {
        double* v = (double*)malloc(sizeof(double) * nb);
        double* xa = (double*)malloc(sizeof(double) * nb);
        double* xb = (double*)malloc(sizeof(double) * nb);
        float* ya = (float*)malloc(sizeof(float) * nb);
        float* yb = (float*)malloc(sizeof(float) * nb);
        for (int64_t i = 0; i < n; ++i) {
            v[i] = sqrt(w[i]);
            xa[i] = x0[i];
            ya[i] = (float)(v[i] * xa[i]);
        }
        for (k = 0; k < iters; ++k) {
            double g = gammas[k], si;
            int fin;
            int64_t fb;
            step_mixed(n, indptr, indices, v, w, xa, ya, g, xb, yb, &fb, &si, &fin,
                       want_dots ? dots : NULL);
            if (n == 0) si = 0.0;
            step_inf[k] = si;
            fallbacks[k] = fb;
            if (want_dots) post_dots(k, 0, gammas, dots, trace, energy, pre_energy, mass);
            if (x_hist) memcpy(x_hist + (size_t)k * (size_t)n, xb, sizeof(double) * (size_t)n);
            while (x_snap && sj < nsnap && snaps[sj] == k) memcpy(x_snap + (size_t)(sj++) * (size_t)n, xb, sizeof(double) * (size_t)n);
            double* t = xa; xa = xb; xb = t;
            float* tf = ya; ya = yb; yb = tf;
            ran = k + 1;
            if (!fin) { rc = GNO_ERR_NONFINITE; *fail_iter = k; break; }
            if (early && g == final_gamma && si < 1e-12) break;
        }
        *iters_run = ran;
        if (want_dots && ran > 0) {
            dots_mixed(n, indptr, indices, v, w, xa, ya, dots);
            post_dots(ran, 1, gammas, dots, trace, energy, pre_energy, mass);
        }
        for (int64_t i = 0; i < n; ++i) {
            double xi = xa[i];
            x_out[i] = xi < 0.0 ? 0.0 : (xi > 1.0 ? 1.0 : xi);
        }
        free(v); free(xa); free(xb); free(ya); free(yb);
    } else {
        float* v = (float*)malloc(sizeof(float) * nb);
        float* wf = (float*)malloc(sizeof(float) * nb);
        float* xa = (float*)malloc(sizeof(float) * nb);
        float* ya = (float*)malloc(sizeof(float) * nb);
        float* xb = (float*)malloc(sizeof(float) * nb);
        float* yb = (float*)malloc(sizeof(float) * nb);
        for (int64_t i = 0; i < n; ++i) {
            v[i] = (float)sqrt(w[i]);
            wf[i] = (float)w[i];
            xa[i] = (float)x0[i];
            ya[i] = v[i] * xa[i];
        }
        for (k = 0; k < iters; ++k) {
            double g = gammas[k], si;
            int fin;
            int64_t fb;
            step_f32(n, indptr, indices, v, wf, xa, ya, (float)g, xb, yb, &fb, &si, &fin,
                     want_dots ? dots : NULL);
            if (n == 0) si = 0.0;
            step_inf[k] = si;
            fallbacks[k] = fb;
            if (want_dots) post_dots(k, 0, gammas, dots, trace, energy, pre_energy, mass);
            if (x_hist)
                for (int64_t i = 0; i < n; ++i) x_hist[(size_t)k * (size_t)n + (size_t)i] = (double)xb[i];
            while (x_snap && sj < nsnap && snaps[sj] == k) {
                for (int64_t i = 0; i < n; ++i) x_snap[(size_t)sj * (size_t)n + (size_t)i] = (double)xb[i];
                ++sj;
            }
            float* t;
            t = xa; xa = xb; xb = t;
            t = ya; ya = yb; yb = t;
            ran = k + 1;
            if (!fin) { rc = GNO_ERR_NONFINITE; *fail_iter = k; break; }
            if (early && g == final_gamma && si < 1e-12) break;   /* dynamics.py:177 */
        }
        *iters_run = ran;
        if (want_dots && ran > 0) {
            dots_f32(n, indptr, indices, wf, xa, ya, dots);
            post_dots(ran, 1, gammas, dots, trace, energy, pre_energy, mass);
        }
        for (int64_t i = 0; i < n; ++i) {
            double xi = (double)xa[i];
            x_out[i] = xi < 0.0 ? 0.0 : (xi > 1.0 ? 1.0 : xi);
        }
        free(v); free(wf); free(xa); free(ya); free(xb); free(yb);
    }
    return rc;
}

/* ---------------------------------------------------------------------------
 * numpy float64 pairwise summation (the algorithm behind w[idx].sum(),
 * graph.py:182): blocks of <= 128 with 8 accumulators, recursive halving on
 * multiples of 8.
 * ------------------------------------------------------------------------- */
double gno_pairwise_sum(const double* a, int64_t n) {
    if (n < 8) {
        double r = 0.0;
        for (int64_t i = 0; i < n; ++i) r += a[i];
        return r;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = a[j];
        int64_t i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i];
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return gno_pairwise_sum(a, n2) + gno_pairwise_sum(a + n2, n - n2);
}

/* MisSolution.from_members flags (graph.py:134-156) on an indicator mask. */
void gno_check(int64_t n, const int64_t* indptr, const int32_t* indices,
               const double* w, const uint8_t* sel, double* weight,
               int* independent, int* maximal, int64_t* count) {
    int ind = 1, dom = 1;
    int64_t cnt = 0;
    for (int64_t i = 0; i < n; ++i) {
        int hit = 0;
        for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p)
            if (sel[indices[p]]) { hit = 1; break; }
        if (sel[i]) { ++cnt; if (hit) ind = 0; }
        else if (!hit) dom = 0;
    }
    double* mw = (double*)malloc(sizeof(double) * (size_t)(cnt ? cnt : 1));
    int64_t c = 0;
    for (int64_t i = 0; i < n; ++i)
        if (sel[i]) mw[c++] = w[i];
    *weight = gno_pairwise_sum(mw, cnt);
    free(mw);
    *independent = ind;
    *maximal = ind && dom;
    *count = cnt;
}

/* (-w, i) priority order for the greedy completion, dynamics.py:273 */
static const double* g_sort_w;
static int by_weight_desc(const void* a, const void* b) {
    int64_t i = *(const int64_t*)a, j = *(const int64_t*)b;
    double wi = g_sort_w[i], wj = g_sort_w[j];
    if (wi > wj) return -1;
    if (wi < wj) return 1;
    return (i < j) ? -1 : (i > j);
}

/* ---------------------------------------------------------------------------
 * round_to_mis (dynamics.py:253-277): threshold at 0.5, sequential repair in
 * ascending u, greedy completion by (-w, i), then the MisSolution flags.
 * ------------------------------------------------------------------------- */
int gno_round(int64_t n, const int64_t* indptr, const int32_t* indices,
              const double* w, const double* x, uint8_t* sel, double* weight,
              int* independent, int* maximal, int64_t* count) {
    for (int64_t i = 0; i < n; ++i) sel[i] = x[i] >= 0.5;
    for (int64_t u = 0; u < n; ++u) {                 /* dynamics.py:262-272 */
        if (!sel[u]) continue;
        for (int64_t p = indptr[u]; p < indptr[u + 1]; ++p) {
            int64_t t = indices[p];
            if (t <= u || !sel[t]) continue;
            if (w[u] < w[t] || (w[u] == w[t] && u < t)) { sel[u] = 0; break; }
            sel[t] = 0;
        }
    }
    int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    for (int64_t i = 0; i < n; ++i) order[i] = i;
    g_sort_w = w;
    qsort(order, (size_t)n, sizeof(int64_t), by_weight_desc);
    for (int64_t q = 0; q < n; ++q) {                  /* dynamics.py:274-276 */
        int64_t i = order[q];
        if (sel[i]) continue;
        int hit = 0;
        for (int64_t p = indptr[i]; p < indptr[i + 1]; ++p)
            if (sel[indices[p]]) { hit = 1; break; }
        if (!hit) sel[i] = 1;
    }
    free(order);
    gno_check(n, indptr, indices, w, sel, weight, independent, maximal, count);
    return GNO_OK;
}
