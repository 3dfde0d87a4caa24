/*
 * oracle/fmg_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, CPU restatement of the reference's `mg-oras` path (reduced full
 * multigrid + Robin-optimised restricted additive Schwarz smoother) for
 * homogeneous-diffusion inpainting.  It exists only so that tests/, bench.py's
 * cpu_baseline / --impl reference leg and __graft_entry__.smoke() can check the
 * CUDA path; nothing under paper_2401_06744_b200/ may import, link or call it.
 *
 * It also restates the paper's comparison pipelines that run on the same driver: the
 * cascadic multilevel mode (ml-*), the CG smoother (_cg_run: mg-cg, ml-cg) and cg_solve;
 * oracle/__init__.py builds oras_solve from orc_oras_sweeps.
 *
 * Every function cites the reference file:line it restates (paths relative to
 * /root/reference/pkg/src/diffpaint/).  The reference is pure Python/NumPy, so
 * there is nothing to compile into oracle/_ref; instead this file is PINNED
 * against the live reference in this container (tests/test_oracle_vs_reference.py,
 * skipped where /root/reference is absent) and against golden vectors the
 * reference produced (tests/golden/, generator tests/golden/make_golden.py).
 *
 * Arithmetic is fp64 throughout (core.py:14-16).  Element-wise operations keep
 * the reference's operation order so they agree bit for bit; reductions (dot
 * products, norms) are plain sequential sums, which differ from NumPy's
 * pairwise/BLAS order by O(1e-16) relative.
 *
 * Parallelism: OpenMP over blocks inside a sweep (the reference's analogue is
 * the ThreadPoolExecutor over block ranges, solvers.py:372-390) and over rows
 * in the stencil passes.  Results do not depend on the thread count: each
 * block's arithmetic is independent and the weighted scatter runs in block
 * order.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_MAX_HIST 256

typedef struct {
    int nu_pre, nu_post, v_cycles_max;
    int modified;        /* value_downsampling: 1 modified, 0 naive */
    int multilevel;      /* mode: 0 full_multigrid, 1 multilevel */
    int block_size, overlap;
    double coarse_tol;
    int coarse_max_iters;
    double tol_rel;
    int max_outer_iters;
    double alpha, eta;
    int local_max_iters; /* 0 = None -> 4 * block area */
    int threads;         /* <=0: all cores */
    int smoother;        /* 0 "oras", 1 "cg" (multigrid.py:66, :278-279, :323-331) */
    int smoother_cg_iters; /* SolverConfig.smoother_cg_iters: CG steps per smoothing unit */
} orc_cfg;

typedef struct {
    int iterations, converged, fine_units, history_len;
    double final_rel, baseline, init_res;
    double history[ORC_MAX_HIST];
} orc_report;

typedef struct {
    int h, w;
    double spacing;
    uint8_t *mask;   /* h*w */
    double *rhs;     /* C*h*w */
    int nx, ny, bw, bh;
    int64_t *xs, *ys;
    double *wx, *wy; /* nx*bw, ny*bh */
} orc_level;

typedef struct {
    int nlevels, channels;
    orc_level *lev;
} orc_hier;

/* counters for the work model in DESIGN.md (block-CG iterations etc.) */
static long long g_cg_iters = 0, g_block_solves = 0, g_sweeps = 0;
static long long g_iter_hist[32];  /* blocks by local CG step count (work model of DESIGN.md) */
void orc_iter_hist_get(long long *out) { memcpy(out, g_iter_hist, sizeof g_iter_hist); }
void orc_counters_reset(void) { g_cg_iters = g_block_solves = g_sweeps = 0; memset(g_iter_hist, 0, sizeof g_iter_hist); }
void orc_counters_get(long long *out) { out[0] = g_cg_iters; out[1] = g_block_solves; out[2] = g_sweeps; }

static int orc_nthreads(int req) {
#ifdef _OPENMP
    int m = omp_get_num_procs();
    if (req <= 0 || req > m) return m;
    return req;
#else
    (void)req;
    return 1;
#endif
}

/* ------------------------------------------------------------------ core.py */

/* core.py:59-67 neighbor_counts + :70-80 neighbor_sum + :100-107 apply.
 * out = nsum * (-1/h^2) + (cnt / h^2) * u, identity at mask pixels.  The
 * neighbour sum accumulates up, down, left, right in that order (:76-79). */
void orc_apply(const uint8_t *mask, int h, int w, double spacing, const double *u, double *out) {
    const double neg = -1.0 / (spacing * spacing);
    const double h2 = spacing * spacing;
#pragma omp parallel for schedule(static)
    for (int y = 0; y < h; ++y) {
        for (int x = 0; x < w; ++x) {
            const size_t i = (size_t)y * w + x;
            if (mask[i]) { out[i] = u[i]; continue; }
            double s = 0.0, cnt = 4.0;
            if (y > 0) s += u[i - w]; else cnt -= 1.0;
            if (y < h - 1) s += u[i + w];
            if (x > 0) s += u[i - 1];
            if (x < w - 1) s += u[i + 1];
            if (y == h - 1) cnt -= 1.0;
            if (x == 0) cnt -= 1.0;
            if (x == w - 1) cnt -= 1.0;
            double o = s * neg;
            o += (cnt / h2) * u[i];
            out[i] = o;
        }
    }
}

/* core.py:109-110 residual = b - A u */
void orc_residual(const uint8_t *mask, int h, int w, double spacing, const double *b,
                  const double *u, double *r) {
    orc_apply(mask, h, w, spacing, u, r);
    const size_t n = (size_t)h * w;
#pragma omp parallel for schedule(static)
    for (size_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
}

static double orc_dot(const double *a, const double *b, size_t n) {
    double s = 0.0;
    for (size_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

/* ------------------------------------------------------------- partition.py */

/* partition.py:84-90 _axis_starts.  Returns the count; writes at most cap. */
int orc_axis_starts(int dim, int block, int stride, int64_t *out, int cap) {
    if (dim <= block) {
        if (cap > 0) out[0] = 0;
        return 1;
    }
    int count = (dim - block + stride - 1) / stride + 1;
    for (int i = 0; i < count && i < cap; ++i) out[i] = (int64_t)stride * i;
    if (count <= cap) out[count - 1] = dim - block;
    return count;
}

/* partition.py:137-154 _axis_weights.  w is (n, block) row-major.  The ramp is
 * np.linspace(0, 1, overlap): i * (1/(overlap-1)) with the last entry forced to
 * 1.0, and [0.0] for overlap == 1 (which yields NaN weights on multi-block
 * axes exactly like the reference does). */
void orc_axis_weights(const int64_t *starts, int n, int block, int dim, int overlap, double *w) {
    for (int i = 0; i < n * block; ++i) w[i] = 1.0;
    if (overlap > 0) {
        double *ramp = (double *)malloc(sizeof(double) * overlap);
        if (overlap == 1) {
            ramp[0] = 0.0;
        } else {
            const double step = 1.0 / (double)(overlap - 1);
            for (int k = 0; k < overlap; ++k) ramp[k] = (double)k * step;
            ramp[overlap - 1] = 1.0;
        }
        for (int i = 0; i < n; ++i) {
            const int64_t s = starts[i];
            if (s > 0)
                for (int k = 0; k < overlap; ++k) w[i * block + k] *= ramp[k];
            if (s + block < dim)
                for (int k = 0; k < overlap; ++k) w[i * block + block - overlap + k] *= ramp[overlap - 1 - k];
        }
        free(ramp);
    }
    double *total = (double *)calloc((size_t)dim, sizeof(double));
    for (int i = 0; i < n; ++i)
        for (int k = 0; k < block; ++k) total[starts[i] + k] += w[i * block + k];
    for (int i = 0; i < n; ++i)
        for (int k = 0; k < block; ++k) w[i * block + k] /= total[starts[i] + k];
    free(total);
}

/* --------------------------------------------------------------- solvers.py */

typedef struct {
    int h, w, bw, bh, nx, ny;
    double spacing, alpha;
    const uint8_t *mask;
    const int64_t *xs, *ys;
    const double *wx, *wy;
} orc_blocks;

/* solvers.py:316-326 BlockSolver._apply for ONE block (== LocalSystem.apply,
 * :221-229): out = diag*v; out -= hinv2*s; identity at local mask pixels. */
static void block_apply(const double *v, const double *diag, const uint8_t *lm, double hinv2,
                        int bh, int bw, double *out) {
    for (int j = 0; j < bh; ++j)
        for (int i = 0; i < bw; ++i) {
            const int k = j * bw + i;
            if (lm[k]) { out[k] = v[k]; continue; }
            double s = 0.0;
            if (j > 0) s += v[k - bw];
            if (j < bh - 1) s += v[k + bw];
            if (i > 0) s += v[k - 1];
            if (i < bw - 1) s += v[k + 1];
            double o = diag[k] * v[k];
            o -= hinv2 * s;
            out[k] = o;
        }
}

/* solvers.py:286-297: diag = neighbor_counts(bh,bw)*hinv2, += alpha/h once per
 * inner (cut) side, in the order left, right, top, bottom. */
static void block_diag(const orc_blocks *B, int ix, int iy, double *diag) {
    const int bw = B->bw, bh = B->bh;
    const double hinv2 = 1.0 / (B->spacing * B->spacing);
    const double robin = B->alpha / B->spacing;
    for (int j = 0; j < bh; ++j)
        for (int i = 0; i < bw; ++i) {
            double cnt = 4.0;
            if (j == 0) cnt -= 1.0;
            if (j == bh - 1) cnt -= 1.0;
            if (i == 0) cnt -= 1.0;
            if (i == bw - 1) cnt -= 1.0;
            diag[j * bw + i] = cnt * hinv2;
        }
    if (B->xs[ix] > 0) for (int j = 0; j < bh; ++j) diag[j * bw] += robin;
    if (B->xs[ix] + bw < B->w) for (int j = 0; j < bh; ++j) diag[j * bw + bw - 1] += robin;
    if (B->ys[iy] > 0) for (int i = 0; i < bw; ++i) diag[i] += robin;
    if (B->ys[iy] + bh < B->h) for (int i = 0; i < bw; ++i) diag[(bh - 1) * bw + i] += robin;
}

/* solvers.py:328-370 _solve_range for ONE block (== local_solve + _cg_run,
 * :97-128, :237-252).  rhs is the gathered residual of the block; out gets v.
 * work: 5*bh*bw doubles.  Returns CG steps taken. */
static int block_solve(const orc_blocks *B, int ix, int iy, const double *rhs, const uint8_t *lm,
                       double target_sq, int max_iters, double *out, double *work) {
    const int n = B->bw * B->bh;
    const double hinv2 = 1.0 / (B->spacing * B->spacing);
    double *diag = work, *r = work + n, *p = work + 2 * n, *q = work + 3 * n, *v = out;
    block_diag(B, ix, iy, diag);
    for (int k = 0; k < n; ++k) v[k] = lm[k] ? rhs[k] : 0.0;
    block_apply(v, diag, lm, hinv2, B->bh, B->bw, q);
    for (int k = 0; k < n; ++k) r[k] = rhs[k] - q[k];
    double rs = orc_dot(r, r, n);
    if (!(rs > target_sq)) return 0;
    memcpy(p, r, sizeof(double) * n);
    int steps = 0;
    for (int it = 0; it < max_iters; ++it) {
        block_apply(p, diag, lm, hinv2, B->bh, B->bw, q);
        const double pq = orc_dot(p, q, n);
        const int ok = pq > 0.0;
        const double a = ok ? rs / pq : 0.0;
        for (int k = 0; k < n; ++k) v[k] += a * p[k];
        for (int k = 0; k < n; ++k) r[k] -= a * q[k];
        const double rs_new = orc_dot(r, r, n);
        ++steps;
        if (rs_new <= target_sq || !ok) break;
        const double beta = rs_new / rs;
        rs = rs_new;
        for (int k = 0; k < n; ++k) { p[k] *= beta; p[k] += r[k]; }
    }
    return steps;
}

/* solvers.py:303-305 gather + :372-390 solve_blocks for all blocks of a field.
 * v_out: (ny*nx, bh, bw). */
static void blocks_solve_all(const orc_blocks *B, const double *r, double target_sq, int max_iters,
                             int threads, double *v_out) {
    const int n = B->bw * B->bh, nb = B->nx * B->ny;
    long long iters = 0;
#pragma omp parallel num_threads(orc_nthreads(threads)) reduction(+ : iters)
    {
        double *work = (double *)malloc(sizeof(double) * 5 * n);
        uint8_t *lm = (uint8_t *)malloc(n);
        double *rhs = work + 4 * n;
#pragma omp for schedule(dynamic, 8)
        for (int b = 0; b < nb; ++b) {
            const int iy = b / B->nx, ix = b % B->nx;
            const int64_t x0 = B->xs[ix], y0 = B->ys[iy];
            for (int j = 0; j < B->bh; ++j)
                for (int i = 0; i < B->bw; ++i) {
                    const size_t g = (size_t)(y0 + j) * B->w + (x0 + i);
                    rhs[j * B->bw + i] = r[g];
                    lm[j * B->bw + i] = B->mask[g];
                }
            const int it = block_solve(B, ix, iy, rhs, lm, target_sq, max_iters, v_out + (size_t)b * n, work);
            iters += it;
#pragma omp atomic
            g_iter_hist[it < 31 ? it : 31] += 1;
        }
        free(work);
        free(lm);
    }
    g_cg_iters += iters;
    g_block_solves += nb;
}

/* solvers.py:307-314 scatter_weighted: (v*wy)*wx accumulated in block order
 * (np.bincount walks the flattened (block, j, i) index list). acc must be
 * zeroed by the caller. */
static void blocks_scatter(const orc_blocks *B, const double *v, double *acc) {
    const int n = B->bw * B->bh;
    for (int iy = 0; iy < B->ny; ++iy)
        for (int ix = 0; ix < B->nx; ++ix) {
            const double *vb = v + (size_t)(iy * B->nx + ix) * n;
            const int64_t x0 = B->xs[ix], y0 = B->ys[iy];
            for (int j = 0; j < B->bh; ++j)
                for (int i = 0; i < B->bw; ++i) {
                    double t = vb[j * B->bw + i] * B->wy[iy * B->bh + j];
                    t *= B->wx[ix * B->bw + i];
                    acc[(size_t)(y0 + j) * B->w + (x0 + i)] += t;
                }
        }
}

/* solvers.py:393-424 oras_sweeps.  history (optional) receives rn at every
 * residual evaluation (the on_state hook, :418-419), up to hist_cap entries. */
static int oras_sweeps_impl(const orc_blocks *B, const double *b, double *u, int max_sweeps,
                            double stop_norm, double eta, int local_max_iters, int threads,
                            double *rn_out, double *history, int hist_cap, int *hist_len) {
    const size_t N = (size_t)B->h * B->w;
    const int n = B->bw * B->bh, nb = B->nx * B->ny;
    double *r = (double *)malloc(sizeof(double) * N);
    double *acc = (double *)malloc(sizeof(double) * N);
    double *v = (double *)malloc(sizeof(double) * (size_t)nb * n);
    int sweeps = 0;
    double rn;
    for (;;) {
        orc_residual(B->mask, B->h, B->w, B->spacing, b, u, r);
        const double rs = orc_dot(r, r, N);
        rn = sqrt(rs);
        if (history && hist_len && *hist_len < hist_cap) history[(*hist_len)++] = rn;
        if (rs == 0.0 || rn <= stop_norm || sweeps >= max_sweeps) break;
        blocks_solve_all(B, r, eta * rs, local_max_iters, threads, v);
        memset(acc, 0, sizeof(double) * N);
        blocks_scatter(B, v, acc);
        for (size_t i = 0; i < N; ++i) u[i] += acc[i];
        ++sweeps;
        ++g_sweeps;
    }
    free(r); free(acc); free(v);
    if (rn_out) *rn_out = rn;
    return sweeps;
}

/* stand-alone partition + weights for the stage-level entry points */
typedef struct {
    orc_blocks B;
    int64_t *xs, *ys;
    double *wx, *wy;
} orc_owned_blocks;

static void owned_blocks_init(orc_owned_blocks *o, const uint8_t *mask, int h, int w, double spacing,
                              int block, int overlap, double alpha) {
    const int stride = block - overlap;
    const int bw = block < w ? block : w, bh = block < h ? block : h;
    const int nx = orc_axis_starts(w, block, stride, NULL, 0);
    const int ny = orc_axis_starts(h, block, stride, NULL, 0);
    o->xs = (int64_t *)malloc(sizeof(int64_t) * nx);
    o->ys = (int64_t *)malloc(sizeof(int64_t) * ny);
    orc_axis_starts(w, block, stride, o->xs, nx);
    orc_axis_starts(h, block, stride, o->ys, ny);
    o->wx = (double *)malloc(sizeof(double) * nx * bw);
    o->wy = (double *)malloc(sizeof(double) * ny * bh);
    orc_axis_weights(o->xs, nx, bw, w, overlap, o->wx);
    orc_axis_weights(o->ys, ny, bh, h, overlap, o->wy);
    o->B = (orc_blocks){h, w, bw, bh, nx, ny, spacing, alpha, mask, o->xs, o->ys, o->wx, o->wy};
}

static void owned_blocks_free(orc_owned_blocks *o) {
    free(o->xs); free(o->ys); free(o->wx); free(o->wy);
}

/* BlockSolver.gather + solve_blocks on a residual field (solvers.py:303-305,
 * :372-390); v_out is (nblocks, bh, bw). */
void orc_solve_blocks(const uint8_t *mask, int h, int w, double spacing, int block, int overlap,
                      double alpha, const double *r, double target_sq, int max_iters, int threads,
                      double *v_out) {
    orc_owned_blocks o;
    owned_blocks_init(&o, mask, h, w, spacing, block, overlap, alpha);
    blocks_solve_all(&o.B, r, target_sq, max_iters, threads, v_out);
    owned_blocks_free(&o);
}

/* BlockSolver.scatter_weighted (solvers.py:307-314); out is (h, w). */
void orc_scatter_weighted(int h, int w, int block, int overlap, const double *v, double *out) {
    orc_owned_blocks o;
    owned_blocks_init(&o, NULL, h, w, 1.0, block, overlap, 0.5);
    memset(out, 0, sizeof(double) * (size_t)h * w);
    blocks_scatter(&o.B, v, out);
    owned_blocks_free(&o);
}

/* oras_sweeps (solvers.py:393-424) with its own partition/weights. */
int orc_oras_sweeps(const uint8_t *mask, int h, int w, double spacing, int block, int overlap,
                    double alpha, const double *b, double *u, int max_sweeps, double stop_norm,
                    double eta, int local_max_iters, int threads, double *rn_out) {
    orc_owned_blocks o;
    owned_blocks_init(&o, mask, h, w, spacing, block, overlap, alpha);
    if (local_max_iters <= 0) local_max_iters = 4 * o.B.bw * o.B.bh;
    int s = oras_sweeps_impl(&o.B, b, u, max_sweeps, stop_norm, eta, local_max_iters, threads,
                             rn_out, NULL, 0, NULL);
    owned_blocks_free(&o);
    return s;
}

/* ------------------------------------------------------------- multigrid.py */

/* multigrid.py:98-101 downsample_mask: 2x2 any-pool, ceil dims. */
void orc_downsample_mask(const uint8_t *fine, int h, int w, uint8_t *coarse) {
    const int hc = (h + 1) / 2, wc = (w + 1) / 2;
    for (int Y = 0; Y < hc; ++Y)
        for (int X = 0; X < wc; ++X) {
            int any = 0;
            for (int dy = 0; dy < 2; ++dy)
                for (int dx = 0; dx < 2; ++dx) {
                    const int y = 2 * Y + dy, x = 2 * X + dx;
                    if (y < h && x < w && fine[(size_t)y * w + x]) any = 1;
                }
            coarse[(size_t)Y * wc + X] = (uint8_t)any;
        }
}

/* multigrid.py:91-95 _cell_sum: NumPy reduces the (2,2) cell as
 * (a00 + a01) + (a10 + a11) (probed; out-of-range constituents are 0). */
static inline double cell4(double a00, double a01, double a10, double a11) {
    return (a00 + a01) + (a10 + a11);
}

/* multigrid.py:104-109 downsample_values_naive. */
void orc_downsample_values_naive(const uint8_t *fm, const double *rhs, int h, int w, double *out) {
    const int hc = (h + 1) / 2, wc = (w + 1) / 2;
    for (int Y = 0; Y < hc; ++Y)
        for (int X = 0; X < wc; ++X) {
            double c[4] = {0, 0, 0, 0}, v[4] = {0, 0, 0, 0};
            for (int dy = 0; dy < 2; ++dy)
                for (int dx = 0; dx < 2; ++dx) {
                    const int y = 2 * Y + dy, x = 2 * X + dx;
                    if (y < h && x < w) {
                        const size_t i = (size_t)y * w + x;
                        c[dy * 2 + dx] = fm[i] ? 1.0 : 0.0;
                        v[dy * 2 + dx] = c[dy * 2 + dx] * rhs[i];
                    }
                }
            const double num = cell4(v[0], v[1], v[2], v[3]);
            const double den = cell4(c[0], c[1], c[2], c[3]);
            out[(size_t)Y * wc + X] = num / (den > 1.0 ? den : 1.0);
        }
}

/* multigrid.py:112-146 downsample_values_modified. */
void orc_downsample_values_modified(const uint8_t *fm, const uint8_t *cm, const double *rhs, int h,
                                    int w, double *out) {
    const int hc = (h + 1) / 2, wc = (w + 1) / 2;
    for (int Y = 0; Y < hc; ++Y)
        for (int X = 0; X < wc; ++X) {
            double wg[4] = {0, 0, 0, 0}, v[4] = {0, 0, 0, 0}, c[4] = {0, 0, 0, 0}, nv[4] = {0, 0, 0, 0};
            for (int dy = 0; dy < 2; ++dy)
                for (int dx = 0; dx < 2; ++dx) {
                    const int y = 2 * Y + dy, x = 2 * X + dx;
                    if (y >= h || x >= w) continue;
                    const size_t i = (size_t)y * w + x;
                    double n = 0.0;
                    /* :131-134 -- in-cell neighbours from the fine mask, the
                     * others from the coarse mask of the adjacent cell */
                    if (x >= 1) n += (x & 1) ? (double)fm[i - 1] : (double)cm[(size_t)(y / 2) * wc + (x - 1) / 2];
                    if (x <= w - 2) n += !(x & 1) ? (double)fm[i + 1] : (double)cm[(size_t)(y / 2) * wc + (x + 1) / 2];
                    if (y >= 1) n += (y & 1) ? (double)fm[i - w] : (double)cm[(size_t)((y - 1) / 2) * wc + x / 2];
                    if (y <= h - 2) n += !(y & 1) ? (double)fm[i + w] : (double)cm[(size_t)((y + 1) / 2) * wc + x / 2];
                    const double cmv = fm[i] ? 1.0 : 0.0;
                    const int k = dy * 2 + dx;
                    wg[k] = cmv * (4.0 - n);
                    v[k] = wg[k] * rhs[i];
                    c[k] = cmv;
                    nv[k] = cmv * rhs[i];
                }
            const double num = cell4(v[0], v[1], v[2], v[3]);
            const double den = cell4(wg[0], wg[1], wg[2], wg[3]);
            double o = num / (den > 1.0 ? den : 1.0);
            const int cmk = cm[(size_t)Y * wc + X];
            if (cmk && den == 0.0) {
                const double nn = cell4(nv[0], nv[1], nv[2], nv[3]);
                const double nd = cell4(c[0], c[1], c[2], c[3]);
                o = nn / (nd > 1.0 ? nd : 1.0);
            }
            out[(size_t)Y * wc + X] = cmk ? o : 0.0;
        }
}

/* multigrid.py:149-154 restrict_residual. */
void orc_restrict_residual(const double *r, int h, int w, const uint8_t *cm, double *out) {
    const int hc = (h + 1) / 2, wc = (w + 1) / 2;
#pragma omp parallel for schedule(static)
    for (int Y = 0; Y < hc; ++Y)
        for (int X = 0; X < wc; ++X) {
            double a[4] = {0, 0, 0, 0}, c[4] = {0, 0, 0, 0};
            for (int dy = 0; dy < 2; ++dy)
                for (int dx = 0; dx < 2; ++dx) {
                    const int y = 2 * Y + dy, x = 2 * X + dx;
                    if (y < h && x < w) { a[dy * 2 + dx] = r[(size_t)y * w + x]; c[dy * 2 + dx] = 1.0; }
                }
            const double o = cell4(a[0], a[1], a[2], a[3]) / cell4(c[0], c[1], c[2], c[3]);
            out[(size_t)Y * wc + X] = cm[(size_t)Y * wc + X] ? 0.0 : o;
        }
}

/* multigrid.py:157-172 _prolongate: x pass then y pass, 0.75 near + 0.25 far. */
static void prolongate(const double *c, int hf, int wf, double *out) {
    const int hc = (hf + 1) / 2, wc = (wf + 1) / 2;
#pragma omp parallel for schedule(static)
    for (int y = 0; y < hf; ++y) {
        const int ny = y / 2;
        int fy = (y & 1) ? ny + 1 : ny - 1;
        if (fy < 0) fy = 0;
        if (fy > hc - 1) fy = hc - 1;
        for (int x = 0; x < wf; ++x) {
            const int nx = x / 2;
            int fx = (x & 1) ? nx + 1 : nx - 1;
            if (fx < 0) fx = 0;
            if (fx > wc - 1) fx = wc - 1;
            const double rn = 0.75 * c[(size_t)ny * wc + nx] + 0.25 * c[(size_t)ny * wc + fx];
            const double rf = 0.75 * c[(size_t)fy * wc + nx] + 0.25 * c[(size_t)fy * wc + fx];
            out[(size_t)y * wf + x] = 0.75 * rn + 0.25 * rf;
        }
    }
}

/* multigrid.py:175-177 prolongate_correction. */
void orc_prolongate_correction(const double *ce, const uint8_t *fm, int hf, int wf, double *out) {
    prolongate(ce, hf, wf, out);
    const size_t n = (size_t)hf * wf;
    for (size_t i = 0; i < n; ++i) if (fm[i]) out[i] = 0.0;
}

/* multigrid.py:180-186 prolongate_solution. */
void orc_prolongate_solution(const double *cu, const uint8_t *fm, const double *frhs, int hf,
                             int wf, double *out) {
    prolongate(cu, hf, wf, out);
    const size_t n = (size_t)hf * wf;
    for (size_t i = 0; i < n; ++i) if (fm[i]) out[i] = frhs[i];
}

/* multigrid.py:189-207 Level: partition + weights per level. */
static void level_init(orc_level *L, int h, int w, double spacing, uint8_t *mask, double *rhs,
                       int block, int overlap) {
    const int stride = block - overlap;
    L->h = h; L->w = w; L->spacing = spacing; L->mask = mask; L->rhs = rhs;
    L->bw = block < w ? block : w;
    L->bh = block < h ? block : h;
    L->nx = orc_axis_starts(w, block, stride, NULL, 0);
    L->ny = orc_axis_starts(h, block, stride, NULL, 0);
    L->xs = (int64_t *)malloc(sizeof(int64_t) * L->nx);
    L->ys = (int64_t *)malloc(sizeof(int64_t) * L->ny);
    orc_axis_starts(w, block, stride, L->xs, L->nx);
    orc_axis_starts(h, block, stride, L->ys, L->ny);
    L->wx = (double *)malloc(sizeof(double) * L->nx * L->bw);
    L->wy = (double *)malloc(sizeof(double) * L->ny * L->bh);
    orc_axis_weights(L->xs, L->nx, L->bw, w, overlap, L->wx);
    orc_axis_weights(L->ys, L->ny, L->bh, h, overlap, L->wy);
}

/* multigrid.py:236-261 build_hierarchy.  known is (C,h,w); level-0 rhs is
 * where(mask, known, 0) (core.py:155-157). */
orc_hier *orc_hier_build(const uint8_t *mask, const double *known, int h, int w, int C,
                         double spacing, const orc_cfg *cfg) {
    orc_hier *H = (orc_hier *)calloc(1, sizeof(orc_hier));
    int cap = 40;
    H->lev = (orc_level *)calloc(cap, sizeof(orc_level));
    H->channels = C;
    size_t n = (size_t)h * w;
    uint8_t *m = (uint8_t *)malloc(n);
    double *rhs = (double *)malloc(sizeof(double) * n * C);
    for (size_t i = 0; i < n; ++i) m[i] = mask[i] ? 1 : 0;
    for (int c = 0; c < C; ++c)
        for (size_t i = 0; i < n; ++i) rhs[c * n + i] = m[i] ? known[c * n + i] : 0.0;
    level_init(&H->lev[0], h, w, spacing, m, rhs, cfg->block_size, cfg->overlap);
    H->nlevels = 1;
    while ((h > w ? h : w) > cfg->block_size && H->nlevels < cap) {
        const int hc = (h + 1) / 2, wc = (w + 1) / 2;
        const size_t nc = (size_t)hc * wc;
        uint8_t *cmask = (uint8_t *)malloc(nc);
        double *crhs = (double *)malloc(sizeof(double) * nc * C);
        orc_downsample_mask(m, h, w, cmask);
        for (int c = 0; c < C; ++c) {
            if (cfg->modified) orc_downsample_values_modified(m, cmask, rhs + c * n, h, w, crhs + c * nc);
            else orc_downsample_values_naive(m, rhs + c * n, h, w, crhs + c * nc);
        }
        m = cmask; rhs = crhs; h = hc; w = wc; n = nc; spacing *= 2.0;
        level_init(&H->lev[H->nlevels++], h, w, spacing, m, rhs, cfg->block_size, cfg->overlap);
    }
    return H;
}

void orc_hier_free(orc_hier *H) {
    if (!H) return;
    for (int l = 0; l < H->nlevels; ++l) {
        orc_level *L = &H->lev[l];
        free(L->mask); free(L->rhs); free(L->xs); free(L->ys); free(L->wx); free(L->wy);
    }
    free(H->lev);
    free(H);
}

int orc_hier_nlevels(const orc_hier *H) { return H->nlevels; }
void orc_hier_level_info(const orc_hier *H, int l, int *out /* h,w,nx,ny,bw,bh */, double *spacing) {
    const orc_level *L = &H->lev[l];
    out[0] = L->h; out[1] = L->w; out[2] = L->nx; out[3] = L->ny; out[4] = L->bw; out[5] = L->bh;
    *spacing = L->spacing;
}
const uint8_t *orc_hier_level_mask(const orc_hier *H, int l) { return H->lev[l].mask; }
const double *orc_hier_level_rhs(const orc_hier *H, int l) { return H->lev[l].rhs; }
const double *orc_hier_level_wx(const orc_hier *H, int l) { return H->lev[l].wx; }
const double *orc_hier_level_wy(const orc_hier *H, int l) { return H->lev[l].wy; }
const int64_t *orc_hier_level_xs(const orc_hier *H, int l) { return H->lev[l].xs; }
const int64_t *orc_hier_level_ys(const orc_hier *H, int l) { return H->lev[l].ys; }

static orc_blocks level_blocks(const orc_level *L, double alpha) {
    orc_blocks B = {L->h, L->w, L->bw, L->bh, L->nx, L->ny, L->spacing, alpha,
                    L->mask, L->xs, L->ys, L->wx, L->wy};
    return B;
}

static int local_cap(const orc_cfg *cfg, const orc_level *L) {
    return cfg->local_max_iters > 0 ? cfg->local_max_iters : 4 * L->bh * L->bw;
}

/* solvers.py:97-128 _cg_run with the level operator: plain CG, u in place.  Returns the steps;
 * *rn_out = final residual norm; history (optional) receives sqrt(rs_new) after every step. */
static int cg_run(const orc_level *L, const double *b, double *u, int max_steps, double stop_norm,
                  double *rn_out, double *history, int hist_cap, int *hist_len) {
    const size_t N = (size_t)L->h * L->w;
    double *r = (double *)malloc(sizeof(double) * N * 3), *p = r + N, *q = p + N;
    orc_residual(L->mask, L->h, L->w, L->spacing, b, u, r);
    double rs = orc_dot(r, r, N);
    int steps = 0;
    if (!(rs == 0.0 || sqrt(rs) <= stop_norm)) {
        memcpy(p, r, sizeof(double) * N);
        while (steps < max_steps) {
            orc_apply(L->mask, L->h, L->w, L->spacing, p, q);
            const double pq = orc_dot(p, q, N);
            if (pq <= 0.0) break;
            const double alpha = rs / pq;
            for (size_t i = 0; i < N; ++i) u[i] += alpha * p[i];
            for (size_t i = 0; i < N; ++i) r[i] -= alpha * q[i];
            const double rs_new = orc_dot(r, r, N);
            ++steps;
            if (history && hist_len && *hist_len < hist_cap) history[(*hist_len)++] = sqrt(rs_new);
            if (rs_new == 0.0 || sqrt(rs_new) <= stop_norm) { rs = rs_new; break; }
            const double beta = rs_new / rs;
            for (size_t i = 0; i < N; ++i) { p[i] *= beta; p[i] += r[i]; }
            rs = rs_new;
        }
    }
    if (rn_out) *rn_out = sqrt(rs);
    free(r);
    return steps;
}

/* multigrid.py:264-279 _smooth. */
static int smooth(const orc_level *L, double *u, const double *rhs, int units, const orc_cfg *cfg) {
    if (units <= 0) return 0;
    if (cfg->smoother == 1) {
        const int k = cfg->smoother_cg_iters;
        const int steps = cg_run(L, rhs, u, units * k, 0.0, NULL, NULL, 0, NULL);
        return (steps + k - 1) / k;  /* -(-steps // k) */
    }
    orc_blocks B = level_blocks(L, cfg->alpha);
    return oras_sweeps_impl(&B, rhs, u, units, 0.0, cfg->eta, local_cap(cfg, L), cfg->threads,
                            NULL, NULL, 0, NULL);
}

/* multigrid.py:282-332 _smooth_to_tol (ORAS branch).  history gets rn/denom
 * at every residual evaluation when requested. */
static int smooth_to_tol(const orc_level *L, double *u, const double *rhs, double tol, int max_units,
                         const orc_cfg *cfg, double denom, double *rel_out, double *history,
                         int hist_cap, int *hist_len) {
    const size_t N = (size_t)L->h * L->w;
    if (denom == 0.0) {
        double *r = (double *)malloc(sizeof(double) * N);
        orc_residual(L->mask, L->h, L->w, L->spacing, rhs, u, r);
        denom = sqrt(orc_dot(r, r, N));
        free(r);
    }
    if (denom == 0.0) { if (rel_out) *rel_out = 0.0; return 0; }
    if (cfg->smoother == 1) {
        /* multigrid.py:318-331: the state before the first step, then one entry per CG step */
        const int h0 = hist_len ? *hist_len : 0;
        if (history && hist_len && *hist_len < hist_cap) {
            double *r = (double *)malloc(sizeof(double) * N);
            orc_residual(L->mask, L->h, L->w, L->spacing, rhs, u, r);
            history[(*hist_len)++] = sqrt(orc_dot(r, r, N));
            free(r);
        }
        double rn;
        const int steps = cg_run(L, rhs, u, max_units, tol * denom, &rn, history, hist_cap, hist_len);
        if (history && hist_len)
            for (int i = h0; i < *hist_len; ++i) history[i] /= denom;
        if (rel_out) *rel_out = rn / denom;
        return steps;
    }
    orc_blocks B = level_blocks(L, cfg->alpha);
    const int h0 = hist_len ? *hist_len : 0;
    double rn;
    int units = oras_sweeps_impl(&B, rhs, u, max_units, tol * denom, cfg->eta, local_cap(cfg, L),
                                 cfg->threads, &rn, history, hist_cap, hist_len);
    if (history && hist_len)
        for (int i = h0; i < *hist_len; ++i) history[i] /= denom;
    if (rel_out) *rel_out = rn / denom;
    return units;
}

/* multigrid.py:335-371 v_cycle. */
void orc_v_cycle(const orc_hier *H, int level, double *u, const double *rhs, const orc_cfg *cfg,
                 int *fine_units) {
    const orc_level *lev = &H->lev[level];
    if (level == H->nlevels - 1) {
        int used = smooth(lev, u, rhs, cfg->nu_pre + cfg->nu_post, cfg);
        if (fine_units && level == 0) *fine_units += used;
        return;
    }
    int used = smooth(lev, u, rhs, cfg->nu_pre, cfg);
    const size_t N = (size_t)lev->h * lev->w;
    const orc_level *co = &H->lev[level + 1];
    const size_t Nc = (size_t)co->h * co->w;
    double *r = (double *)malloc(sizeof(double) * N);
    double *rc = (double *)malloc(sizeof(double) * Nc);
    double *e = (double *)calloc(Nc, sizeof(double));
    orc_residual(lev->mask, lev->h, lev->w, lev->spacing, rhs, u, r);
    orc_restrict_residual(r, lev->h, lev->w, co->mask, rc);
    if (level + 1 == H->nlevels - 1) {
        const double tol = cfg->coarse_tol < cfg->tol_rel ? cfg->coarse_tol : cfg->tol_rel;
        smooth_to_tol(co, e, rc, tol, cfg->coarse_max_iters, cfg, 0.0, NULL, NULL, 0, NULL);
    } else {
        orc_v_cycle(H, level + 1, e, rc, cfg, fine_units);
    }
    orc_prolongate_correction(e, lev->mask, lev->h, lev->w, r);
    for (size_t i = 0; i < N; ++i) u[i] += r[i];
    used += smooth(lev, u, rhs, cfg->nu_post, cfg);
    if (fine_units && level == 0) *fine_units += used;
    free(r); free(rc); free(e);
}

/* multigrid.py:389-422 _cascade.  u_out is (h0, w0). */
static void cascade(const orc_hier *H, const orc_cfg *cfg, int channel, int to_tol, double *u_out,
                    int *fine_units, double *last_rel, double *history, int hist_cap, int *hist_len) {
    const int nl = H->nlevels;
    const orc_level *co = &H->lev[nl - 1];
    size_t n = (size_t)co->h * co->w;
    double *u = (double *)malloc(sizeof(double) * n);
    memcpy(u, co->rhs + (size_t)channel * n, sizeof(double) * n);
    const double tol = cfg->coarse_tol < cfg->tol_rel ? cfg->coarse_tol : cfg->tol_rel;
    double rel = 0.0;
    const int single = nl == 1;
    int units = smooth_to_tol(co, u, co->rhs + (size_t)channel * n, tol, cfg->coarse_max_iters, cfg,
                              0.0, &rel, single ? history : NULL, hist_cap, single ? hist_len : NULL);
    *fine_units = 0;
    *last_rel = INFINITY;
    if (single) {
        *fine_units += units;
        *last_rel = rel;
        memcpy(u_out, u, sizeof(double) * n);
        free(u);
        return;
    }
    for (int l = nl - 2; l >= 0; --l) {
        const orc_level *lev = &H->lev[l];
        const size_t nf = (size_t)lev->h * lev->w;
        const double *b = lev->rhs + (size_t)channel * nf;
        double *uf = (double *)malloc(sizeof(double) * nf);
        orc_prolongate_solution(u, lev->mask, b, lev->h, lev->w, uf);
        free(u);
        u = uf;
        if (to_tol) {
            double *t = (double *)malloc(sizeof(double) * nf);
            orc_residual(lev->mask, lev->h, lev->w, lev->spacing, b, b, t);
            const double base = sqrt(orc_dot(t, t, nf));
            free(t);
            units = smooth_to_tol(lev, u, b, cfg->tol_rel, cfg->max_outer_iters, cfg, base, &rel,
                                  l == 0 ? history : NULL, hist_cap, l == 0 ? hist_len : NULL);
            if (l == 0) { *fine_units += units; *last_rel = rel; }
        } else if (l > 0) {
            smooth(lev, u, b, 1, cfg);
        }
    }
    memcpy(u_out, u, sizeof(double) * (size_t)H->lev[0].h * H->lev[0].w);
    free(u);
}

/* multigrid.py:374-386 cascadic_init. */
void orc_cascadic_init(const orc_hier *H, const orc_cfg *cfg, int channel, double *u_out) {
    int fu; double lr;
    cascade(H, cfg, channel, 0, u_out, &fu, &lr, NULL, 0, NULL);
}

/* multigrid.py:425-487 fmg_solve.  Returns 0, or -1 for an empty mask
 * (EmptyMaskError, :442-443). */
int orc_fmg_solve(const orc_hier *H, const orc_cfg *cfg, int channel, double *u, orc_report *rep) {
    const orc_level *f = &H->lev[0];
    const size_t N = (size_t)f->h * f->w;
    int any = 0;
    for (size_t i = 0; i < N && !any; ++i) any = f->mask[i];
    if (!any) return -1;
    const double *b = f->rhs + (size_t)channel * N;
    double *t = (double *)malloc(sizeof(double) * N);
    orc_residual(f->mask, f->h, f->w, f->spacing, b, b, t);
    const double baseline = sqrt(orc_dot(t, t, N));
    memset(rep, 0, sizeof(*rep));
    rep->baseline = baseline;
    rep->init_res = baseline;
    int fine_units = 0;
    double last_rel;
    if (cfg->multilevel) {
        cascade(H, cfg, channel, 1, u, &fine_units, &last_rel, rep->history, ORC_MAX_HIST, &rep->history_len);
        if (rep->history_len == 0) { rep->history[0] = last_rel; rep->history_len = 1; }
        rep->iterations = fine_units;
        rep->fine_units = fine_units;
        rep->final_rel = last_rel;
        rep->converged = last_rel <= cfg->tol_rel;
        free(t);
        return 0;
    }
    cascade(H, cfg, channel, 0, u, &fine_units, &last_rel, NULL, 0, NULL);
    orc_residual(f->mask, f->h, f->w, f->spacing, b, u, t);
    double rn = sqrt(orc_dot(t, t, N));
    double denom = baseline > 0.0 ? baseline : (rn > 0.0 ? rn : 1.0);
    double rel = rn / denom;
    rep->history[rep->history_len++] = rel;
    int cycles = 0;
    while (rel > cfg->tol_rel && cycles < cfg->v_cycles_max) {
        orc_v_cycle(H, 0, u, b, cfg, &fine_units);
        ++cycles;
        orc_residual(f->mask, f->h, f->w, f->spacing, b, u, t);
        rn = sqrt(orc_dot(t, t, N));
        rel = rn / denom;
        if (rep->history_len < ORC_MAX_HIST) rep->history[rep->history_len++] = rel;
    }
    rep->iterations = cycles;
    rep->fine_units = fine_units;
    rep->final_rel = rel;
    rep->converged = rel <= cfg->tol_rel;
    free(t);
    return 0;
}

/* pipelines.py:96-114 solve_image("mg-oras" / "ml-oras"): shared hierarchy,
 * channels in sequence.  out is (C,h,w); reports has C entries. */
int orc_solve_image(const uint8_t *mask, const double *known, int h, int w, int C, double spacing,
                    const orc_cfg *cfg, double *out, orc_report *reports) {
    orc_hier *H = orc_hier_build(mask, known, h, w, C, spacing, cfg);
    int rc = 0;
    for (int c = 0; c < C && rc == 0; ++c)
        rc = orc_fmg_solve(H, cfg, c, out + (size_t)c * h * w, &reports[c]);
    orc_hier_free(H);
    return rc;
}

/* cg_solve (solvers.py:140-186) from the flat initialisation, one channel: known is (h,w).
 * history[0] = 1, then rn/r0 per step. */
int orc_cg_solve(const uint8_t *mask, const double *known, int h, int w, double spacing, double tol_rel,
                 int max_outer_iters, double *u, orc_report *rep) {
    const size_t N = (size_t)h * w;
    orc_level L;
    memset(&L, 0, sizeof L);
    L.h = h; L.w = w; L.spacing = spacing; L.mask = (uint8_t *)mask;
    double *b = (double *)malloc(sizeof(double) * N * 2), *t = b + N;
    int any = 0;
    for (size_t i = 0; i < N; ++i) { b[i] = mask[i] ? known[i] : 0.0; any |= mask[i]; u[i] = b[i]; }
    memset(rep, 0, sizeof *rep);
    if (!any) { free(b); return -1; }
    orc_residual(mask, h, w, spacing, b, u, t);
    const double r0 = sqrt(orc_dot(t, t, N));
    rep->baseline = r0; rep->init_res = r0;
    if (r0 == 0.0) {
        rep->history[0] = 0.0; rep->history_len = 1; rep->converged = 1;
        free(b);
        return 0;
    }
    rep->history[0] = r0; rep->history_len = 1;
    double rn;
    const int steps = cg_run(&L, b, u, max_outer_iters, tol_rel * r0, &rn, rep->history, ORC_MAX_HIST,
                             &rep->history_len);
    for (int i = 0; i < rep->history_len; ++i) rep->history[i] /= r0;
    rep->iterations = steps; rep->fine_units = steps;
    rep->final_rel = rn / r0;
    rep->converged = rep->final_rel <= tol_rel;
    free(b);
    return 0;
}

int orc_max_threads(void) { return orc_nthreads(0); }
