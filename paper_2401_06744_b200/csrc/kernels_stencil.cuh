// kernels_stencil.cuh -- HBM-bound streaming stencil kernels of the mg-oras path.
//
//   K1  residual_sqnorm_kernel     ||b - A u||^2 per problem        (solvers.py:415-417)
//   K3  residual_restrict_kernel   fused residual + 2x2 restriction  (multigrid.py:358-360, :149-154)
//   K4  prolongate_correct_kernel  u += P e, zero at mask            (multigrid.py:367, :157-177)
//   K5  prolongate_solution_kernel u  = P u_c, known at mask         (multigrid.py:410, :180-186)
//   K6a downsample_mask_kernel     2x2 any-pool                      (multigrid.py:98-101)
//   K6b downsample_values_kernel   naive / neighbour-suppressed      (multigrid.py:104-146)
//
// All kernels are batched: blockIdx.z (or .y) selects the problem p (a
// (frame, channel) pair); channels of a frame share its mask plane.  Fields
// are fp64 (core.py:14-16).  `pred` (may be null) is the per-problem "active"
// flag of the V-cycle loop: converged problems are frozen (multigrid.py:474).
#pragma once
#include "common.cuh"

namespace b200p {

constexpr int ST_THREADS = 256;

// ---------------------------------------------------------------- K1 ------
// Grid: (ctas_per_problem, P).  Each CTA grid-strides over the pixels of its
// problem, reduces in fp64, writes one partial; the last CTA of a problem adds
// the partials in index order (deterministic) and publishes rs[p] plus the
// "residual at a mask pixel is non-zero" flag the ORAS kernels use to skip the
// A v0 product (solvers.py:331-333).
template <bool UM, bool RM>
__global__ void __launch_bounds__(ST_THREADS)
residual_sqnorm_kernel(const double *__restrict__ u, const double *__restrict__ b,
                       const uint8_t *__restrict__ mask, int h, int w, double hinv2, int channels,
                       size_t plane, const int *__restrict__ pred, double *__restrict__ partial,
                       int *__restrict__ partial_flag, unsigned *__restrict__ counter,
                       double *__restrict__ rs_out, int *__restrict__ flag_out) {
    __shared__ double red[33];
    __shared__ int sflag;
    __shared__ bool is_last;
    const int p = blockIdx.y;
    if (pred && !pred[p]) return;
    const double *up = u + (size_t)p * plane;
    const double *bp = b + (size_t)p * plane;
    const uint8_t *mp = mask + (size_t)(p / channels) * plane;
    if (threadIdx.x == 0) sflag = 0;
    __syncthreads();
    double acc = 0.0;
    int flag = 0;
    const size_t n = plane;
    for (size_t i = (size_t)blockIdx.x * ST_THREADS + threadIdx.x; i < n;
         i += (size_t)gridDim.x * ST_THREADS) {
        const int y = (int)(i / w), x = (int)(i - (size_t)y * w);
        const double r = residual_px<UM, RM>(up, bp, mp, y, x, h, w, hinv2);
        acc += r * r;
        if (mp[i] && r != 0.0) flag = 1;
    }
    if (flag) sflag = 1;
    const double tot = cta_sum(acc, red);
    if (threadIdx.x == 0) {
        partial[(size_t)p * gridDim.x + blockIdx.x] = tot;
        partial_flag[(size_t)p * gridDim.x + blockIdx.x] = sflag;
        __threadfence();
        const unsigned done = atomicAdd(&counter[p], 1u);
        is_last = (done == gridDim.x - 1);
    }
    __syncthreads();
    if (is_last) {
        __threadfence();
        double t = 0.0;
        int f = 0;
        // fixed-order tree: thread k sums partials k, k+T, ... then cta_sum
        for (int k = threadIdx.x; k < (int)gridDim.x; k += ST_THREADS) {
            t += ((volatile double *)partial)[(size_t)p * gridDim.x + k];
            f |= ((volatile int *)partial_flag)[(size_t)p * gridDim.x + k];
        }
        if (f) sflag = 1;
        const double total = cta_sum(t, red);
        if (threadIdx.x == 0) {
            rs_out[p] = total;
            flag_out[p] = sflag;
            counter[p] = 0;
        }
    }
}

// K1 (fast path, u given as a field): grid (ceil(w/256), ceil(h/NORM_ROWS), P).
// Thread x walks NORM_ROWS consecutive rows with a 3-row register window, so
// every u value is fetched from DRAM once (left/right neighbours are L1 hits of
// the same coalesced row); no integer division per pixel.  Partials are
// reduced by the last CTA of a problem in index order (deterministic).
constexpr int NORM_ROWS = 32;

template <bool RM>
__global__ void __launch_bounds__(ST_THREADS)
residual_sqnorm_rows_kernel(const double *__restrict__ u, const double *__restrict__ b,
                            const uint8_t *__restrict__ mask, int h, int w, double hinv2, int channels,
                            size_t plane, const int *__restrict__ pred, double *__restrict__ partial,
                            int *__restrict__ partial_flag, unsigned *__restrict__ counter,
                            double *__restrict__ rs_out, int *__restrict__ flag_out) {
    __shared__ double red[34];
    __shared__ int sflag;
    __shared__ bool is_last;
    const int p = blockIdx.z;
    if (pred && !pred[p]) return;
    const double *up = u + (size_t)p * plane;
    const double *bp = b + (size_t)p * plane;
    const uint8_t *mp = mask + (size_t)(p / channels) * plane;
    if (threadIdx.x == 0) sflag = 0;
    __syncthreads();
    const int x = blockIdx.x * ST_THREADS + threadIdx.x;
    const int y0 = blockIdx.y * NORM_ROWS;
    const int y1 = min(h, y0 + NORM_ROWS);
    double acc = 0.0;
    int flag = 0;
    if (x < w) {
        const double cx = 4.0 - (x == 0 ? 1.0 : 0.0) - (x == w - 1 ? 1.0 : 0.0);
        const bool hasL = x > 0, hasR = x < w - 1;
        const double *col = up + x;
        double above = y0 > 0 ? col[(size_t)(y0 - 1) * w] : 0.0;
        double centre = col[(size_t)y0 * w];
#pragma unroll 4
        for (int y = y0; y < y1; ++y) {
            const size_t i = (size_t)y * w + x;
            const double below = y < h - 1 ? col[(size_t)(y + 1) * w] : 0.0;
            const double left = hasL ? up[i - 1] : 0.0;
            const double right = hasR ? up[i + 1] : 0.0;
            const bool m = mp[i] != 0;
            double r;
            if (m) {
                r = bp[i] - centre;
                if (r != 0.0) flag = 1;
            } else {
                const double bb = RM ? 0.0 : bp[i];
                const double cnt = cx - (y == 0 ? 1.0 : 0.0) - (y == h - 1 ? 1.0 : 0.0);
                // same operation order as residual_px: ((up + down) + left) + right
                const double s = ((above + below) + left) + right;
                r = bb - (s * (-hinv2) + (cnt * hinv2) * centre);
            }
            acc += r * r;
            above = centre;
            centre = below;
        }
    }
    if (flag) sflag = 1;
    const double tot = cta_sum(acc, red);
    const unsigned nparts = gridDim.x * gridDim.y;
    const unsigned me = blockIdx.y * gridDim.x + blockIdx.x;
    if (threadIdx.x == 0) {
        partial[(size_t)p * nparts + me] = tot;
        partial_flag[(size_t)p * nparts + me] = sflag;
        __threadfence();
        const unsigned done = atomicAdd(&counter[p], 1u);
        is_last = (done == nparts - 1);
    }
    __syncthreads();
    if (is_last) {
        __threadfence();
        double t = 0.0;
        int f = 0;
        for (unsigned k = threadIdx.x; k < nparts; k += ST_THREADS) {
            t += ((volatile double *)partial)[(size_t)p * nparts + k];
            f |= ((volatile int *)partial_flag)[(size_t)p * nparts + k];
        }
        if (f) sflag = 1;
        const double total = cta_sum(t, red);
        if (threadIdx.x == 0) {
            rs_out[p] = total;
            flag_out[p] = sflag;
            counter[p] = 0;
        }
    }
}

// K1 (vector path): as residual_sqnorm_rows_kernel, but every thread owns TWO
// adjacent columns (one 16-byte load per row) and takes its left/right
// neighbours from the adjacent lanes by shuffle; only the warp's edge lanes load
// an extra element.  Needs an even width (rows stay 16-byte aligned).
template <bool UM, bool RM>
__global__ void __launch_bounds__(ST_THREADS)
residual_sqnorm_rows2_kernel(const double *__restrict__ u, const double *__restrict__ b,
                             const uint8_t *__restrict__ mask, int h, int w, double hinv2, int channels,
                             size_t plane, const int *__restrict__ pred, double *__restrict__ partial,
                             int *__restrict__ partial_flag, unsigned *__restrict__ counter,
                             double *__restrict__ rs_out, int *__restrict__ flag_out) {
    __shared__ double red[34];
    __shared__ int sflag;
    __shared__ bool is_last;
    const int p = blockIdx.z;
    if (pred && !pred[p]) return;
    const double *up = u + (size_t)p * plane;
    const double *bp = b + (size_t)p * plane;
    const uint8_t *mp = mask + (size_t)(p / channels) * plane;
    if (threadIdx.x == 0) sflag = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int x = 2 * (blockIdx.x * ST_THREADS + threadIdx.x);  // columns x, x+1
    const int y0 = blockIdx.y * NORM_ROWS;
    const int y1 = min(h, y0 + NORM_ROWS);
    double acc = 0.0;
    int flag = 0;
    const bool live = x < w;  // w even: x+1 < w as well
    // warp-uniform trip count; dead lanes clamp their column so shuffles stay defined
    const int xc = live ? x : w - 2;
    const double cx0 = 4.0 - (xc == 0 ? 1.0 : 0.0);
    const double cx1 = 4.0 - (xc + 1 == w - 1 ? 1.0 : 0.0);
    const double2 zero2 = make_double2(0.0, 0.0);
    // UM: the iterate is where(mask, u, 0) (flat initialisation read straight from `known`)
    auto row2 = [&](size_t i) {
        double2 v = *reinterpret_cast<const double2 *>(up + i);
        if (UM) {
            const uchar2 mm = *reinterpret_cast<const uchar2 *>(mp + i);
            v.x = mm.x ? v.x : 0.0;
            v.y = mm.y ? v.y : 0.0;
        }
        return v;
    };
    auto one = [&](size_t i) {
        const double v = up[i];
        return UM ? (mp[i] ? v : 0.0) : v;
    };
    double2 above = y0 > 0 ? row2((size_t)(y0 - 1) * w + xc) : zero2;
    double2 centre = row2((size_t)y0 * w + xc);
#pragma unroll 4
    for (int y = y0; y < y1; ++y) {
        const size_t i = (size_t)y * w + xc;
        const double2 below = y < h - 1 ? row2(i + w) : zero2;
        double left = __shfl_up_sync(FULL_MASK, centre.y, 1);
        double right = __shfl_down_sync(FULL_MASK, centre.x, 1);
        if (lane == 0) left = xc > 0 ? one(i - 1) : 0.0;
        if (lane == 31) right = xc + 2 < w ? one(i + 2) : 0.0;
        if (xc + 2 >= w) right = 0.0;  // last column pair of the image
        const uchar2 m2 = *reinterpret_cast<const uchar2 *>(mp + i);
        const double cy = (y == 0 ? 1.0 : 0.0) + (y == h - 1 ? 1.0 : 0.0);
        double r0, r1;
        if (m2.x) {
            r0 = bp[i] - centre.x;
            if (r0 != 0.0) flag = 1;
        } else {
            const double bb = RM ? 0.0 : bp[i];
            const double s = ((above.x + below.x) + left) + centre.y;
            r0 = bb - (s * (-hinv2) + ((cx0 - cy) * hinv2) * centre.x);
        }
        if (m2.y) {
            r1 = bp[i + 1] - centre.y;
            if (r1 != 0.0) flag = 1;
        } else {
            const double bb = RM ? 0.0 : bp[i + 1];
            const double s = ((above.y + below.y) + centre.x) + right;
            r1 = bb - (s * (-hinv2) + ((cx1 - cy) * hinv2) * centre.y);
        }
        if (live) acc += r0 * r0 + r1 * r1;
        above = centre;
        centre = below;
    }
    if (flag && live) sflag = 1;
    const double tot = cta_sum(acc, red);
    const unsigned nparts = gridDim.x * gridDim.y;
    const unsigned me = blockIdx.y * gridDim.x + blockIdx.x;
    if (threadIdx.x == 0) {
        partial[(size_t)p * nparts + me] = tot;
        partial_flag[(size_t)p * nparts + me] = sflag;
        __threadfence();
        const unsigned done = atomicAdd(&counter[p], 1u);
        is_last = (done == nparts - 1);
    }
    __syncthreads();
    if (is_last) {
        __threadfence();
        double t = 0.0;
        int f = 0;
        for (unsigned k = threadIdx.x; k < nparts; k += ST_THREADS) {
            t += ((volatile double *)partial)[(size_t)p * nparts + k];
            f |= ((volatile int *)partial_flag)[(size_t)p * nparts + k];
        }
        if (f) sflag = 1;
        const double total = cta_sum(t, red);
        if (threadIdx.x == 0) {
            rs_out[p] = total;
            flag_out[p] = sflag;
            counter[p] = 0;
        }
    }
}

// residual field (StencilOperator.residual, core.py:109-110); with b == 0 and
// negate it is StencilOperator.apply.
__global__ void __launch_bounds__(ST_THREADS)
residual_field_kernel(const double *__restrict__ u, const double *__restrict__ b,
                      const uint8_t *__restrict__ mask, int h, int w, double hinv2, int apply_only,
                      double *__restrict__ out) {
    const size_t n = (size_t)h * w;
    const size_t i = (size_t)blockIdx.x * ST_THREADS + threadIdx.x;
    if (i >= n) return;
    const int y = (int)(i / w), x = (int)(i - (size_t)y * w);
    if (apply_only) {
        // A u = 0 - (0 - A u): evaluate the residual against b = 0 exactly
        const bool m = mask[i] != 0;
        if (m) { out[i] = u[i]; return; }
        double s = 0.0, cnt = 4.0;
        if (y > 0) s += u[i - w]; else cnt -= 1.0;
        if (y < h - 1) s += u[i + w]; else cnt -= 1.0;
        if (x > 0) s += u[i - 1]; else cnt -= 1.0;
        if (x < w - 1) s += u[i + 1]; else cnt -= 1.0;
        out[i] = s * (-hinv2) + (cnt * hinv2) * u[i];
    } else {
        out[i] = residual_px<false, false>(u, b, mask, y, x, h, w, hinv2);
    }
}

// ---------------------------------------------------------------- K3 ------
// One thread per coarse pixel: residual of its (up to) 2x2 fine constituents,
// cell mean with the true constituent count, 0 at coarse mask pixels; also
// clears the coarse correction e (multigrid.py:361).  The 2x2 sum follows
// NumPy's (a00+a01)+(a10+a11) order.
template <bool RM>
__global__ void __launch_bounds__(ST_THREADS)
residual_restrict_kernel(const double *__restrict__ u, const double *__restrict__ b,
                         const uint8_t *__restrict__ fmask, const uint8_t *__restrict__ cmask, int h,
                         int w, double hinv2, int channels, const int *__restrict__ pred,
                         double *__restrict__ rc, double *__restrict__ e_zero) {
    const int p = blockIdx.z;
    if (pred && !pred[p]) return;
    const int hc = (h + 1) >> 1, wc = (w + 1) >> 1;
    const int X = blockIdx.x * 64 + (threadIdx.x & 63);
    const int Y = blockIdx.y * 4 + (threadIdx.x >> 6);
    if (X >= wc || Y >= hc) return;
    const size_t fplane = (size_t)h * w, cplane = (size_t)hc * wc;
    const double *up = u + (size_t)p * fplane;
    const double *bp = b + (size_t)p * fplane;
    const uint8_t *fm = fmask + (size_t)(p / channels) * fplane;
    const uint8_t *cm = cmask + (size_t)(p / channels) * cplane;
    const size_t ci = (size_t)Y * wc + X;
    double out = 0.0;
    if (!cm[ci]) {
        const int y0 = 2 * Y, x0 = 2 * X;
        const bool hx = x0 + 1 < w, hy = y0 + 1 < h;
        const double a00 = residual_px<false, RM>(up, bp, fm, y0, x0, h, w, hinv2);
        const double a01 = hx ? residual_px<false, RM>(up, bp, fm, y0, x0 + 1, h, w, hinv2) : 0.0;
        const double a10 = hy ? residual_px<false, RM>(up, bp, fm, y0 + 1, x0, h, w, hinv2) : 0.0;
        const double a11 = (hx && hy) ? residual_px<false, RM>(up, bp, fm, y0 + 1, x0 + 1, h, w, hinv2) : 0.0;
        const double cnt = (hx ? 2.0 : 1.0) * (hy ? 2.0 : 1.0);
        out = ((a00 + a01) + (a10 + a11)) / cnt;
    }
    rc[(size_t)p * cplane + ci] = out;
    if (e_zero) e_zero[(size_t)p * cplane + ci] = 0.0;
}

// restrict_residual alone (multigrid.py:149-154) on a given fine residual.
__global__ void __launch_bounds__(ST_THREADS)
restrict_field_kernel(const double *__restrict__ r, const uint8_t *__restrict__ cmask, int h, int w,
                      double *__restrict__ rc) {
    const int hc = (h + 1) >> 1, wc = (w + 1) >> 1;
    const int X = blockIdx.x * 64 + (threadIdx.x & 63);
    const int Y = blockIdx.y * 4 + (threadIdx.x >> 6);
    if (X >= wc || Y >= hc) return;
    const int y0 = 2 * Y, x0 = 2 * X;
    const bool hx = x0 + 1 < w, hy = y0 + 1 < h;
    const double a00 = r[(size_t)y0 * w + x0];
    const double a01 = hx ? r[(size_t)y0 * w + x0 + 1] : 0.0;
    const double a10 = hy ? r[(size_t)(y0 + 1) * w + x0] : 0.0;
    const double a11 = (hx && hy) ? r[(size_t)(y0 + 1) * w + x0 + 1] : 0.0;
    const double cnt = (hx ? 2.0 : 1.0) * (hy ? 2.0 : 1.0);
    const size_t ci = (size_t)Y * wc + X;
    rc[ci] = cmask[ci] ? 0.0 : ((a00 + a01) + (a10 + a11)) / cnt;
}

// ------------------------------------------------------------ K4 / K5 -----
// One thread per coarse pixel -> its (up to) 2x2 fine pixels.  Cell-centred
// bilinear interpolation, x pass then y pass, 0.75 near + 0.25 far with the
// far index clamped at the borders (multigrid.py:157-172).
// SOLUTION = false:  u += P e, 0 at fine mask pixels  (prolongate_correction)
// SOLUTION = true :  u  = P c, rhs at fine mask pixels (prolongate_solution)
// 0.75 near + 0.25 far, written once so that every prolongation kernel rounds alike (0.25 far is exact).
__device__ __forceinline__ double prolong_x(double nearv, double farv) { return __fma_rn(0.75, nearv, 0.25 * farv); }

template <bool SOLUTION>
__global__ void __launch_bounds__(ST_THREADS)
prolongate_kernel(const double *__restrict__ c, const uint8_t *__restrict__ fmask,
                  const double *__restrict__ frhs, int h, int w, int channels,
                  const int *__restrict__ pred, double *__restrict__ u, int Y_lo = 0, int Y_hi = 1 << 30) {
    const int p = blockIdx.z;
    if (pred && !pred[p]) return;
    const int hc = (h + 1) >> 1, wc = (w + 1) >> 1;
    const int X = blockIdx.x * 64 + (threadIdx.x & 63);
    const int Y = Y_lo + blockIdx.y * 4 + (threadIdx.x >> 6);  // coarse rows [Y_lo, Y_hi): strip mode
    if (X >= wc || Y >= hc || Y >= Y_hi) return;
    const size_t fplane = (size_t)h * w, cplane = (size_t)hc * wc;
    const double *cp = c + (size_t)p * cplane;
    const uint8_t *fm = fmask + (size_t)(p / channels) * fplane;
    double *up = u + (size_t)p * fplane;
    const int Xm = X > 0 ? X - 1 : 0, Xp = X < wc - 1 ? X + 1 : wc - 1;
    const int Ym = Y > 0 ? Y - 1 : 0, Yp = Y < hc - 1 ? Y + 1 : hc - 1;
    double rowL[3], rowR[3];  // x-interpolated values on coarse rows Ym, Y, Yp
    const int ys[3] = {Ym, Y, Yp};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double *row = cp + (size_t)ys[k] * wc;
        const double mid = row[X];
        rowL[k] = prolong_x(mid, row[Xm]);  // fine x even: far = near - 1
        rowR[k] = prolong_x(mid, row[Xp]);  // fine x odd : far = near + 1
    }
    const int y0 = 2 * Y, x0 = 2 * X;
    if ((w & 1) == 0 && ((uintptr_t)up & 15) == 0 && ((uintptr_t)fm & 1) == 0) {
        // even width: the two fine pixels of a row are one 16-byte store (and one 2-byte mask load)
#pragma unroll
        for (int dy = 0; dy < 2; ++dy) {
            const int y = y0 + dy;
            if (y >= h) break;
            const int kf = dy ? 2 : 0;
            const size_t i = (size_t)y * w + x0;
            const uchar2 m = *reinterpret_cast<const uchar2 *>(fm + i);
            const double v0 = prolong_x(rowL[1], rowL[kf]);
            const double v1 = prolong_x(rowR[1], rowR[kf]);
            double2 *dst = reinterpret_cast<double2 *>(up + i);
            if (SOLUTION) {
                const double *fr = frhs + (size_t)p * fplane + i;
                double2 o;
                o.x = m.x ? fr[0] : v0;
                o.y = m.y ? fr[1] : v1;
                *dst = o;
            } else {
                double2 o = *dst;
                if (!m.x) o.x += v0;
                if (!m.y) o.y += v1;
                *dst = o;
            }
        }
        return;
    }
#pragma unroll
    for (int dy = 0; dy < 2; ++dy) {
        const int y = y0 + dy;
        if (y >= h) break;
        const int kf = dy ? 2 : 0;  // far row: Y+1 for odd fine rows, Y-1 for even
#pragma unroll
        for (int dx = 0; dx < 2; ++dx) {
            const int x = x0 + dx;
            if (x >= w) break;
            const double nearv = dx ? rowR[1] : rowL[1];
            const double farv = dx ? rowR[kf] : rowL[kf];
            const double val = prolong_x(nearv, farv);
            const size_t i = (size_t)y * w + x;
            const bool m = fm[i] != 0;
            if (SOLUTION) {
                up[i] = m ? frhs[(size_t)p * fplane + i] : val;
            } else {
                if (!m) up[i] += val;
            }
        }
    }
}

// ---------------------------------------------------------------- K6 ------
__global__ void __launch_bounds__(ST_THREADS)
downsample_mask_kernel(const uint8_t *__restrict__ fine, int h, int w, uint8_t *__restrict__ coarse) {
    const int f = blockIdx.z;
    const int hc = (h + 1) >> 1, wc = (w + 1) >> 1;
    const int X = blockIdx.x * 64 + (threadIdx.x & 63);
    const int Y = blockIdx.y * 4 + (threadIdx.x >> 6);
    if (X >= wc || Y >= hc) return;
    const uint8_t *fm = fine + (size_t)f * h * w;
    const int y0 = 2 * Y, x0 = 2 * X;
    const bool hx = x0 + 1 < w, hy = y0 + 1 < h;
    int any = fm[(size_t)y0 * w + x0];
    if (hx) any |= fm[(size_t)y0 * w + x0 + 1];
    if (hy) any |= fm[(size_t)(y0 + 1) * w + x0];
    if (hx && hy) any |= fm[(size_t)(y0 + 1) * w + x0 + 1];
    coarse[(size_t)f * hc * wc + (size_t)Y * wc + X] = any ? 1 : 0;
}

// Values: every fine known pixel enters its cell with weight 4 - (#known
// direct neighbours); in-cell neighbours come from the fine mask, the others
// from the coarse mask of the adjacent cell, off-image counts as unknown
// (multigrid.py:122-137).  Cells known on the coarse grid whose total weight is
// 0 fall back to the plain average (:143-145); 0 off the coarse mask (:146).
// Fine values are read only at fine mask pixels (level-0 `known` is arbitrary
// elsewhere; hierarchy values are 0 there).
// One thread per coarse pixel of a FRAME: the neighbour-suppression weights depend on the masks
// only, so they are formed once and applied to all channels of the frame (grid z = frame).
__device__ __forceinline__ void downsample_cell(const uint8_t *__restrict__ fmask, const uint8_t *__restrict__ cmask,
                                                const double *__restrict__ frhs, int h, int w, int channels, int modified,
                                                double *__restrict__ crhs, int f, int X, int Y) {
    const int hc = (h + 1) >> 1, wc = (w + 1) >> 1;
    const size_t fplane = (size_t)h * w, cplane = (size_t)hc * wc;
    const uint8_t *fm = fmask + (size_t)f * fplane;
    const uint8_t *cm = cmask + (size_t)f * cplane;
    const size_t ci = (size_t)Y * wc + X;
    double wg[4] = {0, 0, 0, 0}, c1[4] = {0, 0, 0, 0};
    bool has[4] = {false, false, false, false};
    // the cell's own fine mask is fetched together with its coarse mask (one 2-byte load per row when
    // w is even), so the dependent chain is masks -> neighbours / values
    const uint8_t cmk = cm[ci];
    bool fmk[4] = {false, false, false, false};
    if ((w & 1) == 0 && ((uintptr_t)fm & 1) == 0) {
        const uchar2 a = *reinterpret_cast<const uchar2 *>(fm + (size_t)(2 * Y) * w + 2 * X);
        fmk[0] = a.x != 0; fmk[1] = a.y != 0;
        if (2 * Y + 1 < h) {
            const uchar2 b = *reinterpret_cast<const uchar2 *>(fm + (size_t)(2 * Y + 1) * w + 2 * X);
            fmk[2] = b.x != 0; fmk[3] = b.y != 0;
        }
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int y = 2 * Y + (k >> 1), x = 2 * X + (k & 1);
            if (y < h && x < w) fmk[k] = fm[(size_t)y * w + x] != 0;
        }
    }
    const bool known = cmk != 0;
    if (!known) {   // 0 off the coarse mask: nothing else to read
        for (int c = 0; c < channels; ++c) crhs[((size_t)f * channels + c) * cplane + ci] = 0.0;
        return;
    }
    // All remaining requests go out together -- the four adjacent cells' coarse masks and the fine values at the
    // cell's mask pixels, for every channel -- and are consumed afterwards: one memory latency behind the masks
    // instead of one per step of the chain neighbours -> weights -> channel 0 -> channel 1 -> ...
    const bool inL = X > 0, inR = 2 * X + 2 <= w - 1, inT = Y > 0, inB = 2 * Y + 2 <= h - 1;
    const uint8_t nL = inL ? cm[ci - 1] : 0, nR = inR ? cm[ci + 1] : 0;
    const uint8_t nT = inT ? cm[ci - wc] : 0, nB = inB ? cm[ci + wc] : 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) has[k] = fmk[k];   // fmk is false outside the image
    constexpr int CB = 3;      // channels per batch of requests
    for (int c0 = 0; c0 < channels; c0 += CB) {
        double val[CB][4];
#pragma unroll
        for (int cc = 0; cc < CB; ++cc) {
            const double *fr = frhs + ((size_t)f * channels + min(c0 + cc, channels - 1)) * fplane;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                val[cc][k] = (has[k] && c0 + cc < channels) ? fr[(size_t)(2 * Y + (k >> 1)) * w + 2 * X + (k & 1)] : 0.0;
        }
        if (c0 == 0) {
#pragma unroll
            for (int dy = 0; dy < 2; ++dy)
#pragma unroll
                for (int dx = 0; dx < 2; ++dx) {
                    const int k = dy * 2 + dx;
                    if (!has[k]) continue;
                    const int y = 2 * Y + dy, x = 2 * X + dx;
                    double n = 0.0;
                    // in-cell neighbours: the cell's own fine mask; the others: the adjacent cell's coarse mask
                    if (x >= 1) n += dx ? (double)fmk[dy * 2] : (double)(nL != 0);
                    if (x <= w - 2) n += !dx ? (double)fmk[dy * 2 + 1] : (double)(nR != 0);
                    if (y >= 1) n += dy ? (double)fmk[dx] : (double)(nT != 0);
                    if (y <= h - 2) n += !dy ? (double)fmk[2 + dx] : (double)(nB != 0);
                    wg[k] = 4.0 - n;
                    c1[k] = 1.0;
                }
        }
        const double nden = (c1[0] + c1[1]) + (c1[2] + c1[3]);
        const double den = (wg[0] + wg[1]) + (wg[2] + wg[3]);
#pragma unroll
        for (int cc = 0; cc < CB; ++cc) {
            if (c0 + cc >= channels) break;
            double nv[4], wv[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                nv[k] = has[k] ? val[cc][k] : 0.0;
                wv[k] = has[k] ? wg[k] * val[cc][k] : 0.0;
            }
            const double nnum = (nv[0] + nv[1]) + (nv[2] + nv[3]);
            const double naive = nnum / fmax(1.0, nden);
            double out = naive;
            if (modified) {
                const double num = (wv[0] + wv[1]) + (wv[2] + wv[3]);
                out = den == 0.0 ? naive : num / fmax(1.0, den);
            }
            crhs[((size_t)f * channels + c0 + cc) * cplane + ci] = out;
        }
    }
}

#ifndef B200P_K6_MINB
#define B200P_K6_MINB 4
#endif
__global__ void __launch_bounds__(ST_THREADS, B200P_K6_MINB)
downsample_values_kernel(const uint8_t *__restrict__ fmask, const uint8_t *__restrict__ cmask,
                         const double *__restrict__ frhs, int h, int w, int channels, int modified,
                         double *__restrict__ crhs) {
    const int hc = (h + 1) >> 1, wc = (w + 1) >> 1;
    const int X = blockIdx.x * 64 + (threadIdx.x & 63);
    const int Y = blockIdx.y * 4 + (threadIdx.x >> 6);
    if (X >= wc || Y >= hc) return;
    downsample_cell(fmask, cmask, frhs, h, w, channels, modified, crhs, blockIdx.z, X, Y);
}

// every byte of v -> 0 / 1
__device__ __forceinline__ unsigned long long mask_bytes_nonzero(unsigned long long v) {
    v |= v >> 4;
    v |= v >> 2;
    v |= v >> 1;
    return v & 0x0101010101010101ull;
}
// 8 mask bytes (0 / 1) -> the 4 bytes "either of a pair"
__device__ __forceinline__ unsigned pair_or4(unsigned long long nz) {
    const unsigned long long pr = nz | (nz >> 8);      // bytes 0, 2, 4, 6
    return (unsigned)(pr & 0x01ull) | (unsigned)((pr >> 8) & 0x0100ull) | (unsigned)((pr >> 16) & 0x010000ull) |
           (unsigned)((pr >> 24) & 0x01000000ull);
}

// K6a for levels whose width is a multiple of 16: a thread takes 8 coarse cells of a row = two 16-byte words of the
// fine mask, and the coarse mask is byte arithmetic on those words (one 8-byte store).  (The same shape for K6b --
// 8 zeros per channel, then a visit of the cells that hold a known pixel -- measured slower than one thread per
// cell: 0.83 vs 0.65 ms per step; the serial chain of the few slow threads is what the launch waits for.)
__global__ void __launch_bounds__(ST_THREADS)
downsample_mask8_kernel(const uint8_t *__restrict__ fine, int h, int w, uint8_t *__restrict__ coarse) {
    const int f = blockIdx.z;
    const int hc = (h + 1) >> 1, wc = w >> 1;
    const int X8 = 8 * (blockIdx.x * 64 + (threadIdx.x & 63));
    const int Y = blockIdx.y * 4 + (threadIdx.x >> 6);
    if (X8 >= wc || Y >= hc) return;
    const uint8_t *row = fine + (size_t)f * h * w + (size_t)(2 * Y) * w + 2 * X8;
    uint4 a = *reinterpret_cast<const uint4 *>(row);
    if (2 * Y + 1 < h) {
        const uint4 b = *reinterpret_cast<const uint4 *>(row + w);
        a.x |= b.x; a.y |= b.y; a.z |= b.z; a.w |= b.w;
    }
    const unsigned long long lo = mask_bytes_nonzero(((unsigned long long)a.y << 32) | a.x);
    const unsigned long long hi = mask_bytes_nonzero(((unsigned long long)a.w << 32) | a.z);
    *reinterpret_cast<uint2 *>(coarse + (size_t)f * hc * wc + (size_t)Y * wc + X8) = make_uint2(pair_or4(lo), pair_or4(hi));
}

// 8-bit ingest / egress (fileio.py:51-65): known = float(u8); out = clip(rint(u)).
__global__ void __launch_bounds__(ST_THREADS)
u8_to_f64_kernel(const uint8_t *__restrict__ in, size_t n, double *__restrict__ out) {
    const size_t i = (size_t)blockIdx.x * ST_THREADS + threadIdx.x;
    if (i < n) out[i] = (double)in[i];
}

// Sparse ingest: entry e = k*C + c of the compacted list goes to channel plane c, pixel idx[k].
__global__ void __launch_bounds__(ST_THREADS)
scatter_known_kernel(const uint32_t *__restrict__ idx, const double *__restrict__ val, size_t n, int C,
                     size_t plane, double *__restrict__ known) {
    const size_t e = (size_t)blockIdx.x * ST_THREADS + threadIdx.x;
    if (e < n) {
        const size_t k = e / (unsigned)C;
        const int c = (int)(e - k * (unsigned)C);
        known[(size_t)c * plane + idx[k]] = val[e];
    }
}

// Sparse ingest from PINNED host memory: `hk` is the caller's known array seen through its device
// alias (zero copy).  Only mask pixels are fetched over PCIe; everything else is written as 0.
__global__ void __launch_bounds__(ST_THREADS)
gather_known_mapped_kernel(const uint8_t *__restrict__ mask, const double *__restrict__ hk, size_t n, int C,
                           size_t plane, double *__restrict__ known, unsigned long long *__restrict__ count) {
    const size_t i = (size_t)blockIdx.x * ST_THREADS + threadIdx.x;
    const bool m = i < n && mask[i] != 0;
    if (i < n) {
        const size_t f = i / plane, pix = i - f * plane;
        for (int c = 0; c < C; ++c) {
            const size_t o = (f * C + c) * plane + pix;
            known[o] = m ? __ldcs(hk + o) : 0.0;
        }
    }
    const int k = __syncthreads_count(m);
    if (threadIdx.x == 0 && k) atomicAdd(count, (unsigned long long)k);
}

// the number of values fetched, for b200p_plan_last_transfer_bytes (plain store into pinned host memory)
__global__ void publish_count_kernel(const unsigned long long *count, unsigned long long *host) { *host = *count; }

__global__ void __launch_bounds__(ST_THREADS)
f64_to_u8_kernel(const double *__restrict__ in, size_t n, uint8_t *__restrict__ out) {
    const size_t i = (size_t)blockIdx.x * ST_THREADS + threadIdx.x;
    if (i < n) out[i] = quantize_u8(in[i]);
}

// ---- 8-bit image files as they are on disk ----
// Mask: the P4 raster (fileio.py:214-216, :226): rows padded to whole bytes, most significant bit
// first, bit 1 = known pixel -> the byte plane (F, h, w) every kernel reads.  One thread per raster byte.
__global__ void __launch_bounds__(ST_THREADS)
unpack_mask_bits_kernel(const uint8_t *__restrict__ bits, size_t nbytes, int w, int row_bytes,
                        uint8_t *__restrict__ mask) {
    const size_t i = (size_t)blockIdx.x * ST_THREADS + threadIdx.x;
    if (i >= nbytes) return;
    const size_t row = i / (unsigned)row_bytes;          // frame * h + y
    const int x0 = (int)(i - row * (unsigned)row_bytes) * 8;
    const unsigned b = bits[i];
    uint8_t *mp = mask + row * (size_t)w + x0;
#pragma unroll
    for (int k = 0; k < 8; ++k)
        if (x0 + k < w) mp[k] = (b >> (7 - k)) & 1u;
}

// Pixels: (F, h, w, C) interleaved 8-bit -> (F, C, h, w) float64 (ImageFile.channel_fields, fileio.py:51-55).
__global__ void __launch_bounds__(ST_THREADS)
deinterleave_u8_kernel(const uint8_t *__restrict__ px, size_t npix, int C, size_t plane, double *__restrict__ out) {
    const size_t i = (size_t)blockIdx.x * ST_THREADS + threadIdx.x;   // f * plane + pixel
    if (i >= npix) return;
    const size_t f = i / plane, pix = i - f * plane;
    for (int c = 0; c < C; ++c) out[(f * C + c) * plane + pix] = (double)px[i * C + c];
}

// image_from_fields (fileio.py:58-65) for the problems whose 8-bit result has not been written by a
// combine pass (K2b's egress): those that needed no V-cycle (cycles == 0), or all of them (`all`).
__global__ void __launch_bounds__(ST_THREADS)
egress_u8_kernel(const double *__restrict__ fields, size_t npix, int C, size_t plane,
                 const int *__restrict__ cycles, int all, uint8_t *__restrict__ out) {
    const size_t i = (size_t)blockIdx.x * ST_THREADS + threadIdx.x;
    if (i >= npix) return;
    const size_t f = i / plane, pix = i - f * plane;
    for (int c = 0; c < C; ++c) {
        const size_t p = f * C + c;
        if (all || cycles[p] == 0) out[i * C + c] = quantize_u8(fields[p * plane + pix]);
    }
}

}  // namespace b200p
