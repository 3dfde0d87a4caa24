// kernels_rows_tma.cuh -- K1 as a TMA-fed pipeline: ||b - A u||^2 per problem (solvers.py:415-417,
// core.py:100-110) for levels whose rows are 16-byte multiples in the mask plane too (w % 16 == 0).
//
// The register-window row walker (kernels_rows.cuh) keeps ONE row of 32 bytes per thread in flight; at the
// measured DRAM latency that caps it near 4.8 TB/s (a plain read-only reduction reaches 6.7 TB/s on this
// GPU).  Here the bytes in flight do not depend on registers: a CTA owns a strip of RT_W columns and streams
// tiles of RT_R rows (+ one halo row above and below, + two halo columns on each side: the innermost TMA
// coordinate must be 16-byte aligned) through a ring of RT_STAGES shared-memory stages filled by
// cp.async.bulk.tensor; pixels outside the image arrive as zeros, which is exactly what the reflecting stencil
// adds for them.  Thread (t, g) walks rows [g RT_R / RT_G, (g + 1) RT_R / RT_G) of column t of every tile with a
// three-row register window (vertical neighbours) and reads its horizontal neighbours from the stage: consecutive
// threads, consecutive words, no bank conflicts.  The arithmetic of a pixel is that of walk_rows4, operation by operation; the per-CTA partials
// are reduced by the same deterministic last-CTA scheme (publish_partial).
#pragma once
#include "kernels_rows.cuh"
#include "kernels_stencil.cuh"
#include "tma_utils.cuh"

namespace b200p {

constexpr int RT_W = 128;                 // columns per CTA
constexpr int RT_G = 4;                   // row groups per tile: RT_W x RT_G threads per CTA
constexpr int RT_THREADS = RT_W * RT_G;
constexpr int RT_BOXW = RT_W + 4;         // box columns x0 - 2 .. x0 + RT_W + 1
constexpr int RT_R = 16;                  // rows per tile
#ifndef B200P_RT_STAGES
#define B200P_RT_STAGES 3      // ring depth of K1 / K3: 3 stages = 3 CTAs per SM (2.31 / 1.35 ms per step; 4: 2.42 / 1.42; 2: 2.38 / 1.41)
#endif
constexpr int RT_STAGES = B200P_RT_STAGES;
constexpr int RT_U_BYTES = (RT_R + 2) * RT_BOXW * 8;            // 19008
constexpr int RT_U_STRIDE = (RT_U_BYTES + 127) / 128 * 128;     // 19072: stages stay 128-byte aligned
constexpr int RT_M_BYTES = RT_R * RT_W;                         // 2048
constexpr int RT_B_BYTES = RT_R * RT_W * 8;                     // 16384
// Grid of the tile pipelines: x = strip * channels + channel, y = row chunk, z = frame.  The channels of a frame
// read the same mask tiles; launched side by side they find them in L2 (one DRAM read per frame, not per plane).
struct TileCoord {
    int p, frame, strip, nstrips;
};
__device__ __forceinline__ TileCoord tile_coord(int channels) {
    TileCoord c;
    c.frame = blockIdx.z;
    c.strip = blockIdx.x / channels;
    c.nstrips = gridDim.x / channels;
    c.p = c.frame * channels + (blockIdx.x - c.strip * channels);
    return c;
}
__host__ __device__ inline size_t rows_tma_smem(bool with_b) {
    return (size_t)RT_STAGES * (RT_U_STRIDE + RT_M_BYTES + (with_b ? RT_B_BYTES : 0)) + 128;
}

// RM: the right-hand side is where(mask, b, 0); with A.trust the caller guarantees u == b at mask pixels and b
// is never read (WITH_B = false).  rows_per_cta comes in A.rows_per_cta (a multiple of RT_R).
template <bool RM, bool WITH_B>
__global__ void __launch_bounds__(RT_THREADS)
residual_sqnorm_tma_kernel(const RowsArgs A, const __grid_constant__ CUtensorMap tm_u,
                           const __grid_constant__ CUtensorMap tm_m, const __grid_constant__ CUtensorMap tm_b) {
    extern __shared__ __align__(128) unsigned char rt_smem[];
    __shared__ double red[34];
    __shared__ int sflag;
    __shared__ bool is_last;
    __shared__ __align__(8) unsigned long long full[RT_STAGES];
    const TileCoord tc = tile_coord(A.channels);
    const int p = tc.p;
    if (A.pred && !A.pred[p]) return;
    const int t = threadIdx.x & (RT_W - 1), g = threadIdx.x / RT_W;
    const bool leader = threadIdx.x == 0;
    unsigned char *base = rt_smem;   // 128-byte aligned by declaration: the pointers stay in the shared window
    unsigned char *su = base, *smk = base + RT_STAGES * RT_U_STRIDE, *sb = smk + RT_STAGES * RT_M_BYTES;
    if (leader) {
        sflag = 0;
        for (int s = 0; s < RT_STAGES; ++s) mbar_init(smem_u32(&full[s]), 1);
    }
    __syncthreads();
    const int h = A.h, w = A.w;
    const int xs = tc.strip * RT_W;
    const int x = xs + t;
    const bool live = x < w;
    const int y0 = A.y_lo + blockIdx.y * A.rows_per_cta;
    const int y1 = min(A.y_hi, y0 + A.rows_per_cta);
    const int ntiles = (y1 - y0 + RT_R - 1) / RT_R;
    const int frame = tc.frame;
    auto issue = [&](int tile) {
        const int s = tile % RT_STAGES;
        const unsigned bar = smem_u32(&full[s]);
        mbar_expect_tx(bar, RT_U_BYTES + RT_M_BYTES + (WITH_B ? RT_B_BYTES : 0));
        const int ty = y0 + tile * RT_R;
        tma_load_3d(smem_u32(su + s * RT_U_STRIDE), &tm_u, xs - 2, ty - 1, p, bar);
        tma_load_3d(smem_u32(smk + s * RT_M_BYTES), &tm_m, xs, ty, frame, bar);
        if (WITH_B) tma_load_3d(smem_u32(sb + s * RT_B_BYTES), &tm_b, xs, ty, p, bar);
    };
    if (leader)
        for (int tile = 0; tile < min(RT_STAGES, ntiles); ++tile) issue(tile);
    const double hinv2 = A.hinv2, nh = -hinv2;
    const double cx = 4.0 - ((x == 0 ? 1.0 : 0.0) + (x == w - 1 ? 1.0 : 0.0));
    const double cxh = cx * hinv2;
    const bool trust = RM && A.trust != 0;
    constexpr int RG = RT_R / RT_G;
    double acc = 0.0;
    int flag = 0;
    for (int tile = 0; tile < ntiles; ++tile) {
        const int s = tile % RT_STAGES;
        mbar_wait(smem_u32(&full[s]), (tile / RT_STAGES) & 1);
        const int ty = y0 + tile * RT_R;
        const int rows = min(RT_R, y1 - ty);
        const int r0 = g * RG;
        const double *U = reinterpret_cast<const double *>(su + s * RT_U_STRIDE) + r0 * RT_BOXW + (t + 2);
        const unsigned char *M = smk + s * RT_M_BYTES + r0 * RT_W + t;
        const double *B = reinterpret_cast<const double *>(sb + s * RT_B_BYTES) + r0 * RT_W + t;
        double above = U[0], centre = U[RT_BOXW];
        if (!WITH_B && rows == RT_R && ty > 0 && ty + RT_R < h) {
            // the common tile: all rows present, no image border row, b - u = 0 at mask pixels (trusted):
            // r = -(A u) off the mask and 0 on it; only r^2 is needed, so the sign is dropped
#pragma unroll
            for (int rr = 0; rr < RG; ++rr) {
                const double below = U[(rr + 2) * RT_BOXW];
                const double lf = U[(rr + 1) * RT_BOXW - 1], rt = U[(rr + 1) * RT_BOXW + 1];
                const unsigned char m = M[rr * RT_W];
                const double sum = ((above + below) + lf) + rt;
                double au = sum * nh + cxh * centre;
                au = m ? 0.0 : au;
                acc += au * au;
                above = centre;
                centre = below;
            }
        } else {
            const int r1 = min(r0 + RG, rows);
            for (int r = r0; r < r1; ++r) {
                const int rr = r - r0, y = ty + r;
                const double below = U[(rr + 2) * RT_BOXW];
                const double lf = U[(rr + 1) * RT_BOXW - 1], rt = U[(rr + 1) * RT_BOXW + 1];
                const unsigned char m = M[rr * RT_W];
                const double cy = (y == 0 ? 1.0 : 0.0) + (y == h - 1 ? 1.0 : 0.0);
                const double c = centre;
                double bb;
                if (RM) bb = (WITH_B && m && !trust) ? B[rr * RT_W] : 0.0;
                else bb = WITH_B ? B[rr * RT_W] : 0.0;
                const double sum = ((above + below) + lf) + rt;
                const double au = sum * nh + ((cx - cy) * hinv2) * c;
                const double res = (trust && m) ? 0.0 : bb - (m ? c : au);
                acc += res * res;
                if (m && res != 0.0) flag = 1;
                above = centre;
                centre = below;
            }
        }
        __syncthreads();   // every thread is done with stage s
        if (leader && tile + RT_STAGES < ntiles) issue(tile + RT_STAGES);
    }
    if (!live) {   // columns right of the image see the last column as a neighbour: not part of the sum
        acc = 0.0;
        flag = 0;
    }
    publish_partial_at(acc, flag, p, tc.nstrips * gridDim.y, blockIdx.y * tc.nstrips + tc.strip, A, red, &sflag, &is_last);
}

// ---------------------------------------------------------------- K3 ------
// Residual + 2x2 restriction + ||r_c||^2 (multigrid.py:358-361, :149-154) on the same tile pipeline.  Thread (t, g)
// owns the coarse pixel (column t of the strip's 64 coarse columns, coarse row g of the tile's RT_R / 2): its
// four fine pixels are two 16-byte words of the stage, their left / right neighbours two more 8-byte reads
// per row.  Cell mean in NumPy's order (a00 + a01) + (a10 + a11), true constituent count (w % 4 == 0, so only
// the last row of an odd-height level makes a one-row cell), 0 at coarse mask pixels; the coarse mask byte of
// the NEXT tile's cell is fetched one tile ahead, so no global load sits in a tile's critical path.
constexpr int RK_G = RT_R / 2;             // coarse rows per tile = row groups
constexpr int RK_THREADS = (RT_W / 2) * RK_G;

template <bool RM, bool WITH_B>
__global__ void __launch_bounds__(RK_THREADS)
residual_restrict_tma_kernel(const RestrictArgs A, const __grid_constant__ CUtensorMap tm_u,
                             const __grid_constant__ CUtensorMap tm_m, const __grid_constant__ CUtensorMap tm_b) {
    extern __shared__ __align__(128) unsigned char rt_smem[];
    __shared__ double red[34];
    __shared__ int sflag;
    __shared__ bool is_last;
    __shared__ __align__(8) unsigned long long full[RT_STAGES];
    const RowsArgs &R = A.R;
    const TileCoord tc = tile_coord(R.channels);
    const int p = tc.p;
    if (R.pred && !R.pred[p]) return;
    const int t = threadIdx.x & (RT_W / 2 - 1), g = threadIdx.x / (RT_W / 2);
    const bool leader = threadIdx.x == 0;
    unsigned char *su = rt_smem, *smk = rt_smem + RT_STAGES * RT_U_STRIDE, *sb = smk + RT_STAGES * RT_M_BYTES;
    if (leader) {
        sflag = 0;
        for (int s = 0; s < RT_STAGES; ++s) mbar_init(smem_u32(&full[s]), 1);
    }
    __syncthreads();
    const int h = R.h, w = R.w;
    const int hc = (h + 1) >> 1, wc = w >> 1;
    const int xs = tc.strip * RT_W;
    const int x = xs + 2 * t;                 // the thread's two fine columns x, x + 1
    const bool live = x < w;
    const int y0 = R.y_lo + blockIdx.y * R.rows_per_cta;   // even
    const int y1 = min(R.y_hi, y0 + R.rows_per_cta);
    const int ntiles = (y1 - y0 + RT_R - 1) / RT_R;
    const int frame = tc.frame;
    const size_t cplane = (size_t)hc * wc;
    const uint8_t *cm = A.cmask + (size_t)frame * cplane;
    double *rc = A.rc + (size_t)p * cplane;
    double *ez = A.e_zero ? A.e_zero + (size_t)p * cplane : nullptr;
    auto issue = [&](int tile) {
        const int s = tile % RT_STAGES;
        const unsigned bar = smem_u32(&full[s]);
        mbar_expect_tx(bar, RT_U_BYTES + RT_M_BYTES + (WITH_B ? RT_B_BYTES : 0));
        const int ty = y0 + tile * RT_R;
        tma_load_3d(smem_u32(su + s * RT_U_STRIDE), &tm_u, xs - 2, ty - 1, p, bar);
        tma_load_3d(smem_u32(smk + s * RT_M_BYTES), &tm_m, xs, ty, frame, bar);
        if (WITH_B) tma_load_3d(smem_u32(sb + s * RT_B_BYTES), &tm_b, xs, ty, p, bar);
    };
    if (leader)
        for (int tile = 0; tile < min(RT_STAGES, ntiles); ++tile) issue(tile);
    const double hinv2 = R.hinv2, nh = -hinv2;
    const double cx0 = 4.0 - (x == 0 ? 1.0 : 0.0), cx1 = 4.0 - (x + 2 == w ? 1.0 : 0.0);
    const double c0h = cx0 * hinv2, c1h = cx1 * hinv2;
    const bool trust = RM && R.trust != 0;
    double acc = 0.0;
    auto coarse_mask_of = [&](int tile) -> uint8_t {
        const int ya = y0 + tile * RT_R + 2 * g;
        return (live && tile < ntiles && ya < y1) ? cm[(size_t)(ya >> 1) * wc + (x >> 1)] : (uint8_t)0;
    };
    uint8_t cmk_next = coarse_mask_of(0);
    for (int tile = 0; tile < ntiles; ++tile) {
        const int s = tile % RT_STAGES;
        const int ty = y0 + tile * RT_R;
        const int ya = ty + 2 * g;                         // the cell's fine rows ya, ya + 1
        const bool cell = live && ya < y1;
        const int Y = ya >> 1;
        const uint8_t cmk = cmk_next;
        cmk_next = coarse_mask_of(tile + 1);               // in flight during this tile
        mbar_wait(smem_u32(&full[s]), (tile / RT_STAGES) & 1);
        if (cell) {
            const double *U = reinterpret_cast<const double *>(su + s * RT_U_STRIDE) + (2 * g) * RT_BOXW + (2 * t + 2);
            const unsigned char *M = smk + s * RT_M_BYTES + (2 * g) * RT_W + 2 * t;
            const double2 u0 = *reinterpret_cast<const double2 *>(U);                    // row ya - 1
            const double2 u1 = *reinterpret_cast<const double2 *>(U + RT_BOXW);          // row ya
            const double2 u2 = *reinterpret_cast<const double2 *>(U + 2 * RT_BOXW);      // row ya + 1
            const double2 u3 = *reinterpret_cast<const double2 *>(U + 3 * RT_BOXW);      // row ya + 2
            const double l1 = U[RT_BOXW - 1], r1 = U[RT_BOXW + 2], l2 = U[2 * RT_BOXW - 1], r2 = U[2 * RT_BOXW + 2];
            const uchar2 m1 = *reinterpret_cast<const uchar2 *>(M), m2 = *reinterpret_cast<const uchar2 *>(M + RT_W);
            const size_t ci = (size_t)Y * wc + (x >> 1);
            double o;
            if (!WITH_B && ya > 0 && ya + 2 < h) {
                // the common cell: both rows inside the image, trusted mask pixels (r = 0 there, -(A u) elsewhere)
                const double a00 = m1.x ? 0.0 : 0.0 - ((((u0.x + u2.x) + l1) + u1.y) * nh + c0h * u1.x);
                const double a01 = m1.y ? 0.0 : 0.0 - ((((u0.y + u2.y) + u1.x) + r1) * nh + c1h * u1.y);
                const double a10 = m2.x ? 0.0 : 0.0 - ((((u1.x + u3.x) + l2) + u2.y) * nh + c0h * u2.x);
                const double a11 = m2.y ? 0.0 : 0.0 - ((((u1.y + u3.y) + u2.x) + r2) * nh + c1h * u2.y);
                o = cmk ? 0.0 : ((a00 + a01) + (a10 + a11)) / 4.0;
            } else {
                const double *B = reinterpret_cast<const double *>(sb + s * RT_B_BYTES) + (2 * g) * RT_W + 2 * t;
                const bool two = ya + 1 < h;               // odd height: the last cell has one row
                const double cya = (ya == 0 ? 1.0 : 0.0) + (ya == h - 1 ? 1.0 : 0.0);
                const double cyb = (ya + 1 == h - 1 ? 1.0 : 0.0);
                auto res = [&](double c, double up, double dn, double lf, double rt, double cnt, uint8_t m, double b) {
                    const double sum = ((up + dn) + lf) + rt;
                    const double au = sum * nh + (cnt * hinv2) * c;
                    const double bb = RM ? ((WITH_B && m && !trust) ? b : 0.0) : (WITH_B ? b : 0.0);
                    return (trust && m) ? 0.0 : bb - (m ? c : au);
                };
                const double b00 = WITH_B ? B[0] : 0.0, b01 = WITH_B ? B[1] : 0.0;
                const double b10 = WITH_B ? B[RT_W] : 0.0, b11 = WITH_B ? B[RT_W + 1] : 0.0;
                const double a00 = res(u1.x, u0.x, u2.x, l1, u1.y, cx0 - cya, m1.x, b00);
                const double a01 = res(u1.y, u0.y, u2.y, u1.x, r1, cx1 - cya, m1.y, b01);
                double s0 = a00 + a01, cnt = 2.0;
                if (two) {
                    const double a10 = res(u2.x, u1.x, u3.x, l2, u2.y, cx0 - cyb, m2.x, b10);
                    const double a11 = res(u2.y, u1.y, u3.y, u2.x, r2, cx1 - cyb, m2.y, b11);
                    s0 = s0 + (a10 + a11);
                    cnt = 4.0;
                } else {
                    s0 = s0 + 0.0;
                }
                o = cmk ? 0.0 : s0 / cnt;
            }
            rc[ci] = o;
            if (ez) ez[ci] = 0.0;
            acc += o * o;
        }
        __syncthreads();   // every thread is done with stage s
        if (leader && tile + RT_STAGES < ntiles) issue(tile + RT_STAGES);
    }
    publish_partial_at(acc, 0, p, tc.nstrips * gridDim.y, blockIdx.y * tc.nstrips + tc.strip, R, red, &sflag, &is_last);
}

// ------------------------------------------------------------ K4 / K5 -----
// Prolongation (multigrid.py:157-172, :364-366 / :398-400) on the tile pipeline.  A tile is RT_W x RT_R fine
// pixels = 64 x 8 coarse cells; thread (t, g) owns one cell and writes its 2 x 2 fine pixels as two 16-byte
// stores.  The stage holds the coarse box (cells Xs - 2 .. Xs + 65, rows Ys - 1 .. Ys + 8: the far neighbour of
// every cell, zeros outside the grid, where the far index is clamped to the near one instead), the fine mask
// tile and -- correction only -- the fine iterate tile.  The solution variant reads the right-hand side at mask
// pixels only, straight from global memory, requested ONE TILE AHEAD (the mask of tile + 1 is already in its
// stage), so no tile waits on that dependent load.  The arithmetic is prolong_pixel's, shared with the
// generic kernel.
constexpr int PT_CW = RT_W / 2 + 4;                    // coarse box columns
constexpr int PT_CR = RT_R / 2 + 2;                    // coarse box rows
constexpr int PT_C_BYTES = PT_CW * PT_CR * 8;          // 5440
constexpr int PT_C_STRIDE = (PT_C_BYTES + 127) / 128 * 128;
constexpr int PT_THREADS = (RT_W / 2) * (RT_R / 2);    // 512
constexpr int PT_STAGES = 4;                           // ring depth of the prolongation pipelines (3: K4 1.62 vs 1.59 ms)
__host__ __device__ inline size_t prolong_tma_smem(bool solution) {
    return (size_t)PT_STAGES * (PT_C_STRIDE + RT_M_BYTES + (solution ? 0 : RT_B_BYTES)) + 128;
}
struct ProlongArgs {
    int h, w, channels, rows_per_cta;   // fine size; rows_per_cta a multiple of RT_R
    const int *pred;
    const double *frhs;                 // SOLUTION: fine right-hand side, read at mask pixels
    double *u;
};

template <bool SOLUTION>
__global__ void __launch_bounds__(PT_THREADS, 2)   // 3 / 4 CTAs per SM (40 / 32 registers, spills): K5 0.85 / 1.20 vs 0.76 ms
prolongate_tma_kernel(const ProlongArgs A, const __grid_constant__ CUtensorMap tm_c,
                      const __grid_constant__ CUtensorMap tm_m, const __grid_constant__ CUtensorMap tm_u) {
    extern __shared__ __align__(128) unsigned char rt_smem[];
    __shared__ __align__(8) unsigned long long full[PT_STAGES];
    const TileCoord tc = tile_coord(A.channels);
    const int p = tc.p;
    if (A.pred && !A.pred[p]) return;
    const int t = threadIdx.x & (RT_W / 2 - 1), g = threadIdx.x / (RT_W / 2);
    const bool leader = threadIdx.x == 0;
    unsigned char *sc = rt_smem, *smk = rt_smem + PT_STAGES * PT_C_STRIDE, *su = smk + PT_STAGES * RT_M_BYTES;
    if (leader)
        for (int s = 0; s < PT_STAGES; ++s) mbar_init(smem_u32(&full[s]), 1);
    __syncthreads();
    const int h = A.h, w = A.w;
    const int hc = (h + 1) >> 1, wc = w >> 1;
    const int xs = tc.strip * RT_W;
    const int X = (xs >> 1) + t;
    const bool live = X < wc;
    const int y0 = blockIdx.y * A.rows_per_cta;
    const int y1 = min(h, y0 + A.rows_per_cta);
    const int ntiles = (y1 - y0 + RT_R - 1) / RT_R;
    const int frame = tc.frame;
    const size_t fplane = (size_t)h * w;
    double *up = A.u + (size_t)p * fplane;
    const double *fr = SOLUTION ? A.frhs + (size_t)p * fplane : nullptr;
    auto issue = [&](int tile) {
        const int s = tile % PT_STAGES;
        const unsigned bar = smem_u32(&full[s]);
        mbar_expect_tx(bar, PT_C_BYTES + RT_M_BYTES + (SOLUTION ? 0 : RT_B_BYTES));
        const int ty = y0 + tile * RT_R;
        tma_load_3d(smem_u32(sc + s * PT_C_STRIDE), &tm_c, (xs >> 1) - 2, (ty >> 1) - 1, p, bar);
        tma_load_3d(smem_u32(smk + s * RT_M_BYTES), &tm_m, xs, ty, frame, bar);
        if (!SOLUTION) tma_load_3d(smem_u32(su + s * RT_B_BYTES), &tm_u, xs, ty, p, bar);
    };
    if (leader)
        for (int tile = 0; tile < min(PT_STAGES, ntiles); ++tile) issue(tile);
    // column offsets of the far neighbours in the coarse box (cell X sits at column t + 2): clamped at the borders
    const int oL = X > 0 ? t + 1 : t + 2, oR = X < wc - 1 ? t + 3 : t + 2;
    uchar2 m0n = make_uchar2(0, 0), m1n = make_uchar2(0, 0);
    double2 f0n = make_double2(0.0, 0.0), f1n = make_double2(0.0, 0.0);
    auto fetch_ahead = [&](int tile) {   // masks of `tile` from its stage; right-hand side at its mask pixels
        const int s = tile % PT_STAGES;
        mbar_wait(smem_u32(&full[s]), (tile / PT_STAGES) & 1);
        const int ya = y0 + tile * RT_R + 2 * g;
        m0n = m1n = make_uchar2(0, 0);
        if (live && ya < y1) {
            const unsigned char *M = smk + s * RT_M_BYTES + (2 * g) * RT_W + 2 * t;
            m0n = *reinterpret_cast<const uchar2 *>(M);
            if (ya + 1 < h) m1n = *reinterpret_cast<const uchar2 *>(M + RT_W);
            if (SOLUTION) {
                const size_t i0 = (size_t)ya * w + 2 * X;
                if (m0n.x) f0n.x = fr[i0];
                if (m0n.y) f0n.y = fr[i0 + 1];
                if (m1n.x) f1n.x = fr[i0 + w];
                if (m1n.y) f1n.y = fr[i0 + w + 1];
            }
        }
    };
    fetch_ahead(0);
    for (int tile = 0; tile < ntiles; ++tile) {
        const int s = tile % PT_STAGES;
        const int ya = y0 + tile * RT_R + 2 * g;           // the cell's fine rows ya, ya + 1
        const bool cell = live && ya < y1;
        const uchar2 m0 = m0n, m1 = m1n;
        double2 f0 = f0n, f1 = f1n;
        if (tile + 1 < ntiles) fetch_ahead(tile + 1);      // waits for the next stage; this one landed before it
        if (cell) {
            const int Y = ya >> 1;
            const bool two = ya + 1 < h;
            const double *C = reinterpret_cast<const double *>(sc + s * PT_C_STRIDE);
            const double *rowN = C + (g + 1) * PT_CW;                       // coarse row Y
            const double *rowU = C + (Y > 0 ? g : g + 1) * PT_CW;          // Y - 1, clamped
            const double *rowD = C + (Y < hc - 1 ? g + 2 : g + 1) * PT_CW; // Y + 1, clamped
            const double nL = prolong_x(rowN[t + 2], rowN[oL]), nR = prolong_x(rowN[t + 2], rowN[oR]);
            const double uL = prolong_x(rowU[t + 2], rowU[oL]), uR = prolong_x(rowU[t + 2], rowU[oR]);
            const double v00 = prolong_x(nL, uL), v01 = prolong_x(nR, uR);
            if (!SOLUTION) {
                const double *U = reinterpret_cast<const double *>(su + s * RT_B_BYTES) + (2 * g) * RT_W + 2 * t;
                f0 = *reinterpret_cast<const double2 *>(U);
                if (two) f1 = *reinterpret_cast<const double2 *>(U + RT_W);
            }
            const size_t i0 = (size_t)ya * w + 2 * X;
            double2 o;
            o.x = SOLUTION ? (m0.x ? f0.x : v00) : (m0.x ? f0.x : f0.x + v00);
            o.y = SOLUTION ? (m0.y ? f0.y : v01) : (m0.y ? f0.y : f0.y + v01);
            *reinterpret_cast<double2 *>(up + i0) = o;
            if (two) {
                const double dL = prolong_x(rowD[t + 2], rowD[oL]), dR = prolong_x(rowD[t + 2], rowD[oR]);
                const double v10 = prolong_x(nL, dL), v11 = prolong_x(nR, dR);
                o.x = SOLUTION ? (m1.x ? f1.x : v10) : (m1.x ? f1.x : f1.x + v10);
                o.y = SOLUTION ? (m1.y ? f1.y : v11) : (m1.y ? f1.y : f1.y + v11);
                *reinterpret_cast<double2 *>(up + i0 + w) = o;
            }
        }
        __syncthreads();   // every thread is done with stage s
        if (leader && tile + PT_STAGES < ntiles) issue(tile + PT_STAGES);
    }
}

}  // namespace b200p
