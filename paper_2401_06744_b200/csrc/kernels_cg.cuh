// kernels_cg.cuh -- global conjugate gradients on a level (the CG-smoothed comparison pipelines
// "cg", "ml-cg", "mg-cg": _cg_run, solvers.py:97-128; multigrid.py:278-279, :323-331).
//
// One CG step is   q = A p, (p.q)  ->  alpha = rs / pq;  u += alpha p;  r -= alpha q;  (r.r)
//                  ->  beta = rs_new / rs;  p = beta p + r
// run for all problems of a batch at once; every problem has its own scalars and a gate that
// closes on convergence (sqrt(rs) <= stop), breakdown (pq <= 0), rs == 0 or the step cap.
// Dot products use the deterministic two-stage reduction of the K1 kernels (per-CTA partials,
// the last CTA of a problem adds them in index order).  These pipelines are the paper's
// comparison baselines, not the hot path: flat one-thread-per-pixel kernels.
#pragma once
#include "common.cuh"

namespace b200p {

constexpr int CG_THREADS = 256;

struct CgArgs {
    const uint8_t *mask;   // (F, h, w)
    const double *b;       // (P, h, w) right-hand side
    double *u;             // (P, h, w) iterate
    double *r, *p, *q;     // (P, h, w) CG vectors
    int h, w, channels;
    size_t plane;
    double hinv2;
    const int *gate;       // (P) problem still iterating
    const double *alpha;   // (P)
    const double *beta;    // (P)
    // reduction
    double *partial;       // (P, ctas)
    unsigned *counter;     // (P)
    double *sum_out;       // (P)
};

// Per-problem state of _cg_run plus the bookkeeping of its callers.
struct CgState {
    double *rs, *pq, *alpha, *beta, *sum, *stop, *denom, *rel;
    int *gate, *steps;
    double *hist;          // (P, hist_cap) or used only when record != 0
    int *histlen;
    int hist_cap;
};

__device__ __forceinline__ void cg_reduce(double acc, int p, const CgArgs &A, double *red, bool *is_last) {
    const double tot = cta_sum(acc, red);
    if (threadIdx.x == 0) {
        A.partial[(size_t)p * gridDim.x + blockIdx.x] = tot;
        __threadfence();
        const unsigned done = atomicAdd(&A.counter[p], 1u);
        *is_last = (done == gridDim.x - 1);
    }
    __syncthreads();
    if (*is_last) {
        __threadfence();
        double t = 0.0;
        for (int k = threadIdx.x; k < (int)gridDim.x; k += CG_THREADS)
            t += ((volatile double *)A.partial)[(size_t)p * gridDim.x + k];
        const double total = cta_sum(t, red);
        if (threadIdx.x == 0) {
            A.sum_out[p] = total;
            A.counter[p] = 0;
        }
    }
}

// A v at one pixel (core.py:100-107): identity at mask pixels.
__device__ __forceinline__ double cg_apply_px(const double *__restrict__ v, const uint8_t *__restrict__ mask,
                                              int y, int x, int h, int w, double hinv2) {
    const size_t i = (size_t)y * w + x;
    if (mask[i]) return v[i];
    double s = 0.0, cnt = 4.0;
    if (y > 0) s += v[i - w]; else cnt -= 1.0;
    if (y < h - 1) s += v[i + w]; else cnt -= 1.0;
    if (x > 0) s += v[i - 1]; else cnt -= 1.0;
    if (x < w - 1) s += v[i + 1]; else cnt -= 1.0;
    return s * (-hinv2) + (cnt * hinv2) * v[i];
}

// OP 0: r = b - A u, p = r, sum = r.r      (RM: b is where(mask, b, 0))
// OP 1: q = A p, sum = p.q
// OP 2: u += alpha p, r -= alpha q, sum = r.r
template <int OP, bool RM>
__global__ void __launch_bounds__(CG_THREADS)
cg_field_kernel(const CgArgs A) {
    __shared__ double red[33];
    __shared__ bool is_last;
    const int p = blockIdx.y;
    if (!A.gate[p]) return;
    const size_t off = (size_t)p * A.plane;
    const uint8_t *mp = A.mask + (size_t)(p / A.channels) * A.plane;
    double acc = 0.0;
    const double alpha = OP == 2 ? A.alpha[p] : 0.0;
    for (size_t i = (size_t)blockIdx.x * CG_THREADS + threadIdx.x; i < A.plane;
         i += (size_t)gridDim.x * CG_THREADS) {
        if (OP == 0) {
            const int y = (int)(i / A.w), x = (int)(i - (size_t)y * A.w);
            const double r = residual_px<false, RM>(A.u + off, A.b + off, mp, y, x, A.h, A.w, A.hinv2);
            A.r[off + i] = r;
            A.p[off + i] = r;
            acc += r * r;
        } else if (OP == 1) {
            const int y = (int)(i / A.w), x = (int)(i - (size_t)y * A.w);
            const double q = cg_apply_px(A.p + off, mp, y, x, A.h, A.w, A.hinv2);
            A.q[off + i] = q;
            acc += A.p[off + i] * q;
        } else {
            const double pv = A.p[off + i];
            A.u[off + i] += alpha * pv;
            const double r = A.r[off + i] - alpha * A.q[off + i];
            A.r[off + i] = r;
            acc += r * r;
        }
    }
    cg_reduce(acc, p, A, red, &is_last);
}

// p = beta p + r  (p *= rs_new / rs; p += r)
__global__ void __launch_bounds__(CG_THREADS)
cg_dir_kernel(const CgArgs A) {
    const int p = blockIdx.y;
    if (!A.gate[p]) return;
    const size_t off = (size_t)p * A.plane;
    const double beta = A.beta[p];
    for (size_t i = (size_t)blockIdx.x * CG_THREADS + threadIdx.x; i < A.plane;
         i += (size_t)gridDim.x * CG_THREADS) {
        double pv = A.p[off + i] * beta;
        pv += A.r[off + i];
        A.p[off + i] = pv;
    }
}

// ---- per-problem scalar steps (one thread per problem)
// start of _cg_run: opens the gate for the problems in `pred` (null = all)
__global__ void cg_begin_kernel(int P, const int *pred, CgState S) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    S.gate[p] = (!pred || pred[p]) ? 1 : 0;
    S.steps[p] = 0;
}

// after OP 0.  denom_mode 0: stop = stop_abs (a fixed norm, 0 for plain smoothing);
// 1: denom = the first residual norm (multigrid.py:300-301 with denom None);
// 2: denom given in S.denom (0 -> the first residual norm).  record: history gets rn / denom.
__global__ void cg_after_init_kernel(int P, CgState S, int denom_mode, double tol, double stop_abs,
                                     int record) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P || !S.gate[p]) return;
    const double rs = S.sum[p], rn = sqrt(rs);
    S.rs[p] = rs;
    double stop = stop_abs;
    if (denom_mode != 0) {
        double d = denom_mode == 2 ? S.denom[p] : 0.0;
        if (d == 0.0) d = rn;
        S.denom[p] = d;
        stop = tol * d;
        S.rel[p] = d == 0.0 ? 0.0 : rn / d;
        if (record && d != 0.0) {
            if (S.histlen[p] < S.hist_cap) S.hist[(size_t)p * S.hist_cap + S.histlen[p]] = rn / d;
            S.histlen[p] += 1;
        }
    }
    S.stop[p] = stop;
    if (rs == 0.0 || rn <= stop) S.gate[p] = 0;  // solvers.py:105-106
}

// after OP 1: breakdown check, alpha (solvers.py:111-114)
__global__ void cg_after_apply_kernel(int P, CgState S) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P || !S.gate[p]) return;
    const double pq = S.sum[p];
    S.pq[p] = pq;
    if (pq <= 0.0) {
        S.gate[p] = 0;
        return;
    }
    S.alpha[p] = S.rs[p] / pq;
}

// after OP 2: step count, history, stop test, beta (solvers.py:117-126).  `go` = problems that
// continue with the direction update; the gate closes after it when the step cap is reached.
__global__ void cg_after_update_kernel(int P, CgState S, int max_steps, int record, int denom_mode,
                                       int *any) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P || !S.gate[p]) return;
    const double rs_new = S.sum[p], rn = sqrt(rs_new);
    const int steps = S.steps[p] + 1;
    S.steps[p] = steps;
    if (denom_mode != 0) {
        const double d = S.denom[p];
        S.rel[p] = rn / d;
        if (record) {
            if (S.histlen[p] < S.hist_cap) S.hist[(size_t)p * S.hist_cap + S.histlen[p]] = rn / d;
            S.histlen[p] += 1;
        }
    }
    if (rs_new == 0.0 || rn <= S.stop[p]) {
        S.rs[p] = rs_new;
        S.gate[p] = 0;
        return;
    }
    S.beta[p] = rs_new / S.rs[p];
    S.rs[p] = rs_new;
    if (steps >= max_steps) {
        S.gate[p] = 0;  // the reference still updates p here; p is dead after the loop
        return;
    }
    if (any) *any = 1;
}

// _smooth's unit count: -(-steps // k) added to the finest-level counter (multigrid.py:279)
__global__ void cg_units_kernel(int P, const int *pred, const int *steps, int k, int *units) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P || (pred && !pred[p])) return;
    units[p] += (steps[p] + k - 1) / k;
}

}  // namespace b200p
