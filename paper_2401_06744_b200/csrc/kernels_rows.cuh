// kernels_rows.cuh -- row-walking residual kernels (HBM-bound passes over a level).
//
// A thread owns FOUR adjacent columns and walks a chunk of rows with a 3-row
// register window: every u value is fetched once with 16-byte loads, vertical
// neighbours come from the window, horizontal ones from the thread's own
// registers or the adjacent lane (shuffle); only a warp's two edge lanes load one
// extra element per row.  No integer division, no per-pixel bounds tests.
//
//   K1  residual_sqnorm_rows4_kernel    ||b - A u||^2 per problem       (solvers.py:415-417)
//   K3  residual_restrict_rows4_kernel  r = b - A u restricted 2x2, plus ||r_c||^2 of
//                                       the coarse system with e = 0    (multigrid.py:358-361)
//
// Both need w % 4 == 0 and 16-byte aligned planes; other shapes use the scalar
// kernels of kernels_stencil.cuh.
#pragma once
#include "common.cuh"

namespace b200p {

constexpr int ROWS4_THREADS = 128;  // 512 columns per CTA
#ifndef B200P_ROWS_UNROLL
#define B200P_ROWS_UNROLL 1
#endif
// L2 prefetch distance (rows ahead of the row being fetched) of the row walkers; 0 = off.
#ifndef B200P_ROWS_PF
#define B200P_ROWS_PF 0
#endif

struct RowsArgs {
    const double *u, *b;
    const uint8_t *mask;
    int h, w;
    double hinv2;
    int channels;
    size_t plane;
    const int *pred;
    int rows_per_cta;  // even
    int y_lo, y_hi;    // rows handled by this launch (strip mode; default 0 .. h)
    int trust;         // RM only: the caller guarantees u == b at mask pixels (true throughout fmg_solve:
                       // interpolation is exact after every step), so b is not read at all
    // reduction of the per-CTA partials (last CTA of a problem sums them in index order)
    double *partial;
    int *partial_flag;
    unsigned *counter;
    double *rs_out;
    int *flag_out;
};

// Deterministic two-stage reduction: every CTA stores its partial, the last one to
// arrive (per problem) adds all partials in index order and publishes the total.
// (nparts, me): the problem's CTA count and this CTA's index among them (the order the partials are added in).
__device__ __forceinline__ void publish_partial_at(double acc, int flag, int p, unsigned nparts, unsigned me,
                                                   const RowsArgs &A, double *red, int *sflag, bool *is_last) {
    const int T = blockDim.x;
    if (flag) *sflag = 1;
    const double tot = cta_sum(acc, red);
    if (threadIdx.x == 0) {
        A.partial[(size_t)p * nparts + me] = tot;
        A.partial_flag[(size_t)p * nparts + me] = *sflag;
        __threadfence();
        const unsigned done = atomicAdd(&A.counter[p], 1u);
        *is_last = (done == nparts - 1);
    }
    __syncthreads();
    if (*is_last) {
        __threadfence();
        double t = 0.0;
        int f = 0;
        for (unsigned k = threadIdx.x; k < nparts; k += T) {
            t += ((volatile double *)A.partial)[(size_t)p * nparts + k];
            f |= ((volatile int *)A.partial_flag)[(size_t)p * nparts + k];
        }
        if (f) *sflag = 1;
        const double total = cta_sum(t, red);
        if (threadIdx.x == 0) {
            A.rs_out[p] = total;
            A.flag_out[p] = *sflag;
            A.counter[p] = 0;
        }
    }
}

__device__ __forceinline__ void publish_partial(double acc, int flag, int p, const RowsArgs &A,
                                                double *red, int *sflag, bool *is_last) {
    publish_partial_at(acc, flag, p, gridDim.x * gridDim.y, blockIdx.y * gridDim.x + blockIdx.x, A, red, sflag, is_last);
}

// ---------------------------------------------------------------- K1f -----
// The baseline norm of the flat initialisation (multigrid.py:441-446, solvers.py:415-417 with u = b =
// where(mask, known, 0)): the residual is 0 at mask pixels and hinv2 * (sum of the KNOWN direct neighbours)
// elsewhere, i.e. non-zero only next to the 2 % of mask pixels.  A thread takes 8 pixels of a row as one
// 8-byte mask word (+ the words above / below and the two edge bytes), finds the pixels that have a known
// neighbour with byte arithmetic, and only for those fetches values -- for every channel of the frame, the
// masks being shared (grid z = frame).  Same per-pixel arithmetic as residual_px (neighbour order
// ((up + down) + left) + right, zeros for unknown neighbours); deterministic last-CTA reduction per problem.
constexpr int FLAT_THREADS = 128;
constexpr int FLAT_ROWS = 16;
constexpr int FLAT_MAXC = 4;

__device__ __forceinline__ unsigned long long bytes_nonzero(unsigned long long v) {  // every byte -> 0 / 1
    v |= v >> 4;
    v |= v >> 2;
    v |= v >> 1;
    return v & 0x0101010101010101ull;
}

__global__ void __launch_bounds__(FLAT_THREADS)
flat_init_sqnorm_kernel(const RowsArgs A) {
    __shared__ double red[34];
    __shared__ int sflag;
    __shared__ bool is_last;
    const int frame = blockIdx.z;
    const int C = A.channels;
    if (threadIdx.x == 0) sflag = 0;
    __syncthreads();
    const int h = A.h, w = A.w;
    const int x8 = 8 * (blockIdx.x * FLAT_THREADS + threadIdx.x);
    const int y0 = A.y_lo + blockIdx.y * FLAT_ROWS, y1 = min(A.y_hi, y0 + FLAT_ROWS);
    const uint8_t *mp = A.mask + (size_t)frame * A.plane;
    for (int c0 = 0; c0 < C; c0 += FLAT_MAXC) {
        double acc[FLAT_MAXC] = {0.0, 0.0, 0.0, 0.0};
        if (x8 < w) {
            for (int y = y0; y < y1; ++y) {
                const uint8_t *row = mp + (size_t)y * w + x8;
                const unsigned long long mc = bytes_nonzero(*reinterpret_cast<const unsigned long long *>(row));
                const unsigned long long mu = y > 0 ? bytes_nonzero(*reinterpret_cast<const unsigned long long *>(row - w)) : 0ull;
                const unsigned long long md = y + 1 < h ? bytes_nonzero(*reinterpret_cast<const unsigned long long *>(row + w)) : 0ull;
                const unsigned long long lb = x8 > 0 ? (row[-1] != 0) : 0, rb = x8 + 8 < w ? (row[8] != 0) : 0;
                const unsigned long long ml = (mc << 8) | lb, mr = (mc >> 8) | (rb << 56);
                unsigned long long need = (mc ^ 0x0101010101010101ull) & (mu | md | ml | mr);
                while (need) {
                    const int k = (__ffsll((long long)need) - 1) >> 3;
                    need &= need - 1;
                    const bool up = (mu >> (8 * k)) & 1, dn = (md >> (8 * k)) & 1, lf = (ml >> (8 * k)) & 1, rt = (mr >> (8 * k)) & 1;
                    const size_t i = (size_t)y * w + x8 + k;
#pragma unroll
                    for (int cc = 0; cc < FLAT_MAXC; ++cc) {
                        if (c0 + cc >= C) break;
                        const double *kp = A.u + ((size_t)frame * C + c0 + cc) * A.plane + i;
                        const double vu = up ? kp[-w] : 0.0, vd = dn ? kp[w] : 0.0, vl = lf ? kp[-1] : 0.0, vr = rt ? kp[1] : 0.0;
                        const double r = (((vu + vd) + vl) + vr) * A.hinv2;
                        acc[cc] = fma(r, r, acc[cc]);
                    }
                }
            }
        }
        for (int cc = 0; cc < FLAT_MAXC && c0 + cc < C; ++cc) {
            const int p = frame * C + c0 + cc;
            if (A.pred && !A.pred[p]) continue;     // block-uniform
            __syncthreads();
            publish_partial(acc[cc], 0, p, A, red, &sflag, &is_last);
        }
    }
}

struct Row4 {
    double v[4];
};

// Walks rows [y0, y1) of the thread's four columns xc..xc+3 and hands the
// residual of each row to `consume(y, r[4], m[4])`.  UM: the iterate is
// where(mask, u, 0); RM: the right-hand side is where(mask, b, 0).
// The arithmetic of a pixel follows residual_px (common.cuh) operation by operation.
template <bool UM, bool RM, class Consumer>
__device__ __forceinline__ void walk_rows4(const double *__restrict__ up, const double *__restrict__ bp,
                                           const uint8_t *__restrict__ mp, int h, int w, double hinv2,
                                           int xc, int y0, int y1, bool trust, Consumer &consume) {
    const int lane = threadIdx.x & 31;
    const bool hasL = xc > 0, hasR = xc + 4 < w;
    const double cxL = 4.0 - (xc == 0 ? 1.0 : 0.0);
    const double cxR = 4.0 - (xc + 4 == w ? 1.0 : 0.0);
    auto load_mask = [&](size_t i) { return *reinterpret_cast<const uchar4 *>(mp + i); };
    auto load_row = [&](size_t i, uchar4 m) {
        Row4 r;
        if (UM) {
            // flat initialisation where(mask, known, 0): only the known pixels (a few per cent) are
            // fetched, so the baseline pass reads the mask plus the touched 32-byte sectors of `known`
            r.v[0] = m.x ? up[i] : 0.0;
            r.v[1] = m.y ? up[i + 1] : 0.0;
            r.v[2] = m.z ? up[i + 2] : 0.0;
            r.v[3] = m.w ? up[i + 3] : 0.0;
            return r;
        }
        const double2 a = *reinterpret_cast<const double2 *>(up + i);
        const double2 c = *reinterpret_cast<const double2 *>(up + i + 2);
        r.v[0] = a.x; r.v[1] = a.y; r.v[2] = c.x; r.v[3] = c.y;
        return r;
    };
    auto load_one = [&](size_t i) {
        if (UM) return mp[i] ? up[i] : 0.0;
        return up[i];
    };
    Row4 above, centre, below;
    const Row4 zero = {{0.0, 0.0, 0.0, 0.0}};
    uchar4 mc = load_mask((size_t)y0 * w + xc), mn = mc;
    above = zero;
    if (y0 > 0) {
        const size_t ia = (size_t)(y0 - 1) * w + xc;
        above = load_row(ia, UM ? load_mask(ia) : mc);
    }
    centre = load_row((size_t)y0 * w + xc, mc);
    // (unrolling or prefetching a further row ahead measured slower: the pass is bound by
    // occupancy x bytes in flight, and both cost registers)
    constexpr int kUnroll = B200P_ROWS_UNROLL;
#pragma unroll kUnroll
    for (int y = y0; y < y1; ++y) {
        const size_t i = (size_t)y * w + xc;
        below = zero;
        if (y < h - 1) {
            mn = load_mask(i + w);
            below = load_row(i + w, mn);
        }
        if (B200P_ROWS_PF > 0 && !UM && y + 1 + B200P_ROWS_PF < y1 + 1 && y + 1 + B200P_ROWS_PF < h) {
            // the thread's four columns are one 32-byte sector: pull it into L2 a few rows ahead
            asm volatile("prefetch.global.L2 [%0];" ::"l"(up + i + (size_t)(1 + B200P_ROWS_PF) * w));
            if (!RM) asm volatile("prefetch.global.L2 [%0];" ::"l"(bp + i + (size_t)(1 + B200P_ROWS_PF) * w));
        }
        double left = __shfl_up_sync(FULL_MASK, centre.v[3], 1);
        double right = __shfl_down_sync(FULL_MASK, centre.v[0], 1);
        if (lane == 0) left = hasL ? load_one(i - 1) : 0.0;
        if (lane == 31) right = hasR ? load_one(i + 4) : 0.0;
        if (!hasR) right = 0.0;  // last columns of the image (any lane)
        const double cy = (y == 0 ? 1.0 : 0.0) + (y == h - 1 ? 1.0 : 0.0);
        const uint8_t m[4] = {mc.x, mc.y, mc.z, mc.w};
        double r[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            // branch-free: the stencil value is always formed, mask pixels select b - u
            const double c = centre.v[k];
            const double bb = RM ? ((m[k] && !trust) ? bp[i + k] : 0.0) : bp[i + k];
            const double lf = k == 0 ? left : centre.v[k - 1];
            const double rt = k == 3 ? right : centre.v[k + 1];
            const double s = ((above.v[k] + below.v[k]) + lf) + rt;
            const double cnt = (k == 0 ? cxL : (k == 3 ? cxR : 4.0)) - cy;
            const double au = s * (-hinv2) + (cnt * hinv2) * c;
            r[k] = (RM && trust && m[k]) ? 0.0 : bb - (m[k] ? c : au);
        }
        consume(y, r, m);
        above = centre;
        centre = below;
        mc = mn;
    }
}

// ---------------------------------------------------------------- K1 ------
template <bool UM, bool RM>
__global__ void __launch_bounds__(ROWS4_THREADS)
residual_sqnorm_rows4_kernel(const RowsArgs A) {
    __shared__ double red[34];
    __shared__ int sflag;
    __shared__ bool is_last;
    const int p = blockIdx.z;
    if (A.pred && !A.pred[p]) return;
    if (threadIdx.x == 0) sflag = 0;
    __syncthreads();
    const int x = 4 * (blockIdx.x * ROWS4_THREADS + threadIdx.x);
    const bool live = x < A.w;
    const int xc = live ? x : A.w - 4;  // dead lanes shadow the last column group (shuffles stay defined)
    const int y0 = A.y_lo + blockIdx.y * A.rows_per_cta;
    const int y1 = min(A.y_hi, y0 + A.rows_per_cta);
    double acc = 0.0;
    int flag = 0;
    auto consume = [&](int, const double (&r)[4], const uint8_t (&m)[4]) {
        acc += (r[0] * r[0] + r[1] * r[1]) + (r[2] * r[2] + r[3] * r[3]);
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (m[k] && r[k] != 0.0) flag = 1;
    };
    walk_rows4<UM, RM>(A.u + (size_t)p * A.plane, A.b + (size_t)p * A.plane,
                       A.mask + (size_t)(p / A.channels) * A.plane, A.h, A.w, A.hinv2, xc, y0, y1, A.trust != 0, consume);
    if (!live) { acc = 0.0; flag = 0; }
    publish_partial(acc, flag, p, A, red, &sflag, &is_last);
}

// ---------------------------------------------------------------- K3 ------
// Fine rows come in pairs (2Y, 2Y+1); the thread's four fine columns make two
// coarse columns.  Cell mean with the true constituent count (w % 4 == 0, so only
// the last coarse row of an odd-height level is partial), 0 at coarse mask pixels;
// NumPy's 2x2 order (a00 + a01) + (a10 + a11) (multigrid.py:91-95, :149-154).
// Also zeroes the coarse correction e (multigrid.py:361) and accumulates
// ||r_c||^2, which IS the residual norm^2 of the coarse system at e = 0, so the
// next level's pre-smoothing needs no separate K1 pass.
struct RestrictArgs {
    RowsArgs R;
    const uint8_t *cmask;  // (F, hc, wc)
    double *rc;            // (P, hc, wc)
    double *e_zero;        // (P, hc, wc) or null
};

template <bool RM>
__global__ void __launch_bounds__(ROWS4_THREADS)
residual_restrict_rows4_kernel(const RestrictArgs A) {
    __shared__ double red[34];
    __shared__ int sflag;
    __shared__ bool is_last;
    const RowsArgs &R = A.R;
    const int p = blockIdx.z;
    if (R.pred && !R.pred[p]) return;
    if (threadIdx.x == 0) sflag = 0;
    __syncthreads();
    const int h = R.h, w = R.w;
    const int hc = (h + 1) >> 1, wc = w >> 1;
    const int x = 4 * (blockIdx.x * ROWS4_THREADS + threadIdx.x);
    const bool live = x < w;
    const int xc = live ? x : w - 4;
    const int y0 = R.y_lo + blockIdx.y * R.rows_per_cta;  // even
    const int y1 = min(R.y_hi, y0 + R.rows_per_cta);
    const size_t cplane = (size_t)hc * wc;
    const uint8_t *cm = A.cmask + (size_t)(p / R.channels) * cplane;
    double *rc = A.rc + (size_t)p * cplane;
    double *ez = A.e_zero ? A.e_zero + (size_t)p * cplane : nullptr;
    double acc = 0.0;
    double top0 = 0.0, top1 = 0.0;
    auto emit = [&](int Y, double s0, double s1, double cnt) {
        const size_t ci = (size_t)Y * wc + (xc >> 1);
        const uchar2 m = *reinterpret_cast<const uchar2 *>(cm + ci);
        double2 o;
        o.x = m.x ? 0.0 : s0 / cnt;
        o.y = m.y ? 0.0 : s1 / cnt;
        if (live) {
            *reinterpret_cast<double2 *>(rc + ci) = o;
            if (ez) *reinterpret_cast<double2 *>(ez + ci) = make_double2(0.0, 0.0);
            acc += o.x * o.x + o.y * o.y;
        }
    };
    auto consume = [&](int y, const double (&r)[4], const uint8_t (&)[4]) {
        if ((y & 1) == 0) {
            top0 = r[0] + r[1];
            top1 = r[2] + r[3];
            if (y == h - 1) emit(y >> 1, top0 + 0.0, top1 + 0.0, 2.0);  // odd height: single-row cell
        } else {
            emit(y >> 1, top0 + (r[0] + r[1]), top1 + (r[2] + r[3]), 4.0);
        }
    };
    walk_rows4<false, RM>(R.u + (size_t)p * R.plane, R.b + (size_t)p * R.plane,
                          R.mask + (size_t)(p / R.channels) * R.plane, h, w, R.hinv2, xc, y0, y1, R.trust != 0, consume);
    publish_partial(acc, 0, p, R, red, &sflag, &is_last);
}

}  // namespace b200p
