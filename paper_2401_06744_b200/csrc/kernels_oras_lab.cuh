// kernels_oras_lab.cuh -- block-solve variants that were measured against the shipped kernels and lost
// (DESIGN.md section 3 lists each with its numbers).  They are NOT part of the default build: compile with
// -DB200P_EXPERIMENTS (make EXTRA=-DB200P_EXPERIMENTS) to get them back behind B200P_TILE32 / B200P_FUSED /
// B200P_ARRIVAL; tests/test_gpu_stages.py covers them when the library says it has them.
//   K2L  oras_sweep_lean_kernel       two warps per 32x32 block, lean prologue (+ combine on arrival)
//   K2S  oras_sweep_tile_s_kernel     CG state partly in shared memory
//   K2F  oras_fused_sweep_kernel      solve + combine in one persistent kernel through an L2-resident ring
//   K2b'  oras_combine_band_kernel    combine over the overlap bands only (with the DIRECT variant of K2W)
#pragma once
#include "kernels_oras.cuh"

namespace b200p {

// ------------------------------------------------------------------ K2L ---
// The 32x32 register-tile solve with a lean per-block prologue/epilogue.  ncu on K2 showed
// that with ~4.3 CG steps per block the per-block part (gather, start, weighted store) issues
// as many instructions as 2.4 CG steps; K2L trims it:
//   * grid (ix, iy, problem): no integer division;
//   * the block-local mask comes from the bit table packed at hierarchy build (one coalesced
//     32-bit load per thread instead of 16 byte loads and tests);
//   * own pixels are loaded as aligned double2 (block starts are even), only the halo needs a
//     predicate, and the neighbour count of core.py:100-110 is 4 unless the block touches the
//     image border (block-uniform branch);
//   * inside FMG the right-hand side is where(mask, known, 0) and b - u == 0 at mask pixels
//     (mflag == 0), so level-0 / cascade sweeps (RM) do not read b at all;
//   * the PoU weight rows of the block are fetched into shared memory at block start and read
//     back after the CG loop (their global-load latency used to be exposed at the end).
// Requires: even level width, even block starts, 16-byte aligned u / b (the driver checks).
struct LeanSmem {
    TileSmem<4, 4, 2> cg;
    alignas(16) double wx[32];
    alignas(16) double wy[32];
};

// Combine on arrival (FUSE): the ordered sum of the covering tiles (K2b) is done inside K2 by
// whichever block finishes LAST among the blocks that cover a cell.  Cells are the rectangles
// between consecutive block starts, [xs[cx], xs[cx+1]) x [ys[cy], ys[cy+1]); a finished block
// bumps the arrival counter of every cell it overlaps (after a __threadfence), and the block that
// completes a cell's count sums the tiles -- just written by its neighbours, still in L2 -- in
// ascending block order (np.bincount order, solvers.py:310-314) and writes u_out = u + sum.
// Nobody waits: there is no spinning and no dependence on the scheduling order.  The sweep is out
// of place (u -> u_out) because other blocks still gather from u.
struct FuseArgs {
    double *u_out;          // (P, h, w) or null: split path (tiles only, K2b combines)
    unsigned *cell_cnt;     // (P, ny, nx) arrival counters, zeroed before the launch
    const int *cell_need;   // (ny, nx) blocks covering each cell
    const int *lastx, *lasty;  // per block column / row: last cell index it overlaps
    int *unit_counter;      // per-problem sweep counter (may be null)
};

// u_out = u + ordered sum of the weighted tiles on cell (cx, cy).  64 threads: a thread owns one
// column and every second row of the cell; like K2b the (up to) four tile reads of a pixel are
// issued branch-free, CELL_G rows at a time, so ~35 independent loads are in flight per thread.
constexpr int CELL_G = 7;

__device__ __forceinline__ void combine_cell(const LevelDev &L, const double *scratch_p, const double *up,
                                             double *wp, int cx, int cy, int tid) {
    const int x0 = L.xs[cx], x1 = cx + 1 < L.nx ? L.xs[cx + 1] : L.w;
    const int y0 = L.ys[cy], y1 = cy + 1 < L.ny ? L.ys[cy + 1] : L.h;
    const size_t bsz = (size_t)L.bw * L.bh;
    const int tx = tid & 31, ty = tid >> 5;
    for (int xb = x0; xb < x1; xb += 32) {
        const int x = xb + tx;
        if (x >= x1) continue;
        const int ixf = L.cxf[x], ixn = L.cxn[x];
        const size_t xo0 = (size_t)ixf * bsz + (x - L.xs[ixf]);
        const bool two_x = ixn > 1;
        const size_t xo1 = two_x ? (size_t)(ixf + 1) * bsz + (x - L.xs[ixf + 1]) : xo0;
        const bool wide_x = ixn > 2;
        for (int yb = y0 + ty; yb < y1; yb += 2 * CELL_G) {
            double uu[CELL_G], v00[CELL_G], v01[CELL_G], v10[CELL_G], v11[CELL_G];
            int nn[CELL_G];
#pragma unroll
            for (int g = 0; g < CELL_G; ++g) {
                const int yq = yb + 2 * g;
                const int y = yq < y1 ? yq : y1 - 1;
                const int iyf = L.cyf[y], iyn = L.cyn[y];
                nn[g] = iyn;
                const int iy1 = iyf + (iyn > 1 ? 1 : 0);
                const size_t o0 = (size_t)iyf * L.nx * bsz + (size_t)(y - L.ys[iyf]) * L.bw;
                const size_t o1 = (size_t)iy1 * L.nx * bsz + (size_t)(y - L.ys[iy1]) * L.bw;
                uu[g] = up[(size_t)y * L.w + x];
                v00[g] = __ldcg(scratch_p + o0 + xo0);
                v01[g] = __ldcg(scratch_p + o0 + xo1);
                v10[g] = __ldcg(scratch_p + o1 + xo0);
                v11[g] = __ldcg(scratch_p + o1 + xo1);
            }
#pragma unroll
            for (int g = 0; g < CELL_G; ++g) {
                const int y = yb + 2 * g;
                if (y >= y1) break;
                const int n = nn[g];
                // ascending block order: (iy0,ix0), (iy0,ix1), (iy1,ix0), (iy1,ix1)
                double acc = v00[g];
                acc += two_x ? v01[g] : 0.0;
                if (wide_x || n > 2) {  // > 2 covering blocks per axis: heavily overlapped layouts
                    acc = 0.0;
                    const int iyf = L.cyf[y];
                    for (int a = 0; a < n; ++a) {
                        const int iy = iyf + a;
                        const size_t ro = (size_t)iy * L.nx * bsz + (size_t)(y - L.ys[iy]) * L.bw;
                        for (int c = 0; c < ixn; ++c)
                            acc += __ldcg(scratch_p + ro + (size_t)(ixf + c) * bsz + (x - L.xs[ixf + c]));
                    }
                } else {
                    acc += n > 1 ? v10[g] : 0.0;
                    acc += (n > 1 && two_x) ? v11[g] : 0.0;
                }
                wp[(size_t)y * L.w + x] = uu[g] + acc;
            }
        }
    }
}

template <bool RM, int REGCAP, bool FUSE = false>
__global__ void __launch_bounds__(64) __maxnreg__(REGCAP)
oras_sweep_lean_kernel(const SweepArgs A, const unsigned *__restrict__ mtab, const FuseArgs Fz = FuseArgs()) {
    constexpr int TW = 4, TH = 4, NWARP = 2, BW = 32, BH = 32;
    using CG = TileCG<TW, TH, NWARP>;
    __shared__ LeanSmem sm;
    const int p = blockIdx.z;
    const LevelDev &L = A.L;
    const int ix = blockIdx.x, iy = blockIdx.y + A.iy0, blk = iy * L.nx + ix;
    const int tid = threadIdx.x;
    const bool frozen = A.pred && !A.pred[p];
    const double rs_g = frozen ? 0.0 : A.rs[p];
    if (frozen || rs_g == 0.0) {  // frozen problem, or oras_sweeps' rs == 0 exit (solvers.py:420)
        if (FUSE) {
            // the sweep is a no-op, but the iterate moves to the partner buffer with everybody else
            const int x0 = L.xs[ix], x1 = ix + 1 < L.nx ? L.xs[ix + 1] : L.w;
            const int y0 = L.ys[iy], y1 = iy + 1 < L.ny ? L.ys[iy + 1] : L.h;
            const size_t off = (size_t)p * A.plane;
            for (int y = y0 + (tid >> 5); y < y1; y += 2)
                for (int x = x0 + (tid & 31); x < x1; x += 32)
                    Fz.u_out[off + (size_t)y * L.w + x] = A.u[off + (size_t)y * L.w + x];
        }
        return;
    }
    if (FUSE && Fz.unit_counter && ix == 0 && iy == 0 && tid == 0) Fz.unit_counter[p] += 1;
    // frame of the problem (channels share the mask): constant divisors for gray / RGB
    const int frame = A.channels == 3 ? p / 3 : (A.channels == 1 ? p : p / A.channels);
    const unsigned mbits = mtab[((size_t)frame * L.nblocks + blk) * 64 + tid];
    // PoU weight rows of this block -> shared memory (consumed after the CG loop)
    {
        const double wv = tid < 32 ? L.wx[ix * BW + tid] : L.wy[iy * BH + tid - 32];
        if (tid < 32) sm.wx[tid] = wv; else sm.wy[tid - 32] = wv;
    }
    const int x0 = L.xs[ix], y0 = L.ys[iy];
    const int W = L.w, H = L.h;
    const double target = A.eta * rs_g;
    const bool general = A.mflag[p] != 0;

    CG cg;
    cg.lane = tid & 31;
    cg.wg = tid >> 5;
    cg.bar_id = 1;
    cg.lx = cg.lane & 7;
    cg.ly = cg.lane >> 3;
    cg.xrow = sm.cg.xrow;
    cg.red = sm.cg.red;
    cg.slot = 0;
    cg.eL = cg.lx == 0;
    cg.eR = cg.lx == 7;
    cg.eT = cg.wg == 0 && cg.ly == 0;
    cg.eB = cg.wg == NWARP - 1 && cg.ly == 3;
    const double g_in = L.g_in;  // 1 - alpha*h
    cg.gL = x0 > 0 ? g_in : 1.0;
    cg.gR = x0 + BW < W ? g_in : 1.0;
    cg.gT = y0 > 0 ? g_in : 1.0;
    cg.gB = y0 + BH < H ? g_in : 1.0;
    cg.mbits = mbits;

    const int bx = cg.lx * TW, by = (cg.wg * 4 + cg.ly) * TH;
    const int gx0 = x0 + bx, gy0 = y0 + by;
    const double hinv2 = L.hinv2;
    const bool border = x0 == 0 || y0 == 0 || x0 + BW >= W || y0 + BH >= H;  // block-uniform

    // ---- gather: global residual g = b - A u on the tile (core.py:100-110)
    double r[TH][TW];
    {
        const double *urow = A.u + (size_t)p * A.plane + (size_t)(gy0 - 1) * W + gx0;
        double uc[TH + 2][TW + 2];
        if (!border) {
            // interior block: every halo element is inside the image
#pragma unroll
            for (int j = 0; j < TH + 2; ++j) {
                const double *rp = urow + (size_t)j * W;
                const double2 a0 = *reinterpret_cast<const double2 *>(rp);
                const double2 a1 = *reinterpret_cast<const double2 *>(rp + 2);
                uc[j][1] = a0.x; uc[j][2] = a0.y; uc[j][3] = a1.x; uc[j][4] = a1.y;
                if (j >= 1 && j <= TH) {
                    uc[j][0] = rp[-1];
                    uc[j][5] = rp[TW];
                } else {
                    uc[j][0] = uc[j][5] = 0.0;
                }
            }
        } else {
            const bool hasL = gx0 > 0, hasR = gx0 + TW < W, hasT = gy0 > 0, hasB = gy0 + TH < H;
#pragma unroll
            for (int j = 0; j < TH + 2; ++j) {
                const double *rp = urow + (size_t)j * W;
                const bool rowin = (j > 0 || hasT) && (j < TH + 1 || hasB);
                double2 a0 = make_double2(0.0, 0.0), a1 = a0;
                if (rowin) {
                    a0 = *reinterpret_cast<const double2 *>(rp);
                    a1 = *reinterpret_cast<const double2 *>(rp + 2);
                }
                uc[j][1] = a0.x; uc[j][2] = a0.y; uc[j][3] = a1.x; uc[j][4] = a1.y;
                uc[j][0] = uc[j][5] = 0.0;
                if (j >= 1 && j <= TH) {
                    if (hasL) uc[j][0] = rp[-1];
                    if (hasR) uc[j][5] = rp[TW];
                }
            }
        }
        double bt[TH][TW];
#pragma unroll
        for (int j = 0; j < TH; ++j) {
            if (!RM) {
                const double *bp = A.b + (size_t)p * A.plane + (size_t)(gy0 + j) * W + gx0;
                const double2 b0 = *reinterpret_cast<const double2 *>(bp);
                const double2 b1 = *reinterpret_cast<const double2 *>(bp + 2);
                bt[j][0] = b0.x; bt[j][1] = b0.y; bt[j][2] = b1.x; bt[j][3] = b1.y;
            } else {
                bt[j][0] = bt[j][1] = bt[j][2] = bt[j][3] = 0.0;
            }
        }
        const double nc4 = -4.0 * hinv2;
        // b - (d u - hinv2 s), d = (number of in-image neighbours) / h^2
#pragma unroll
        for (int j = 0; j < TH; ++j)
#pragma unroll
            for (int i = 0; i < TW; ++i) {
                const double s = ((uc[j][i + 1] + uc[j + 2][i + 1]) + uc[j + 1][i]) + uc[j + 1][i + 2];
                const double uu = uc[j + 1][i + 1];
                const double res = fma(hinv2, s, RM ? nc4 * uu : fma(nc4, uu, bt[j][i]));
                const bool m = (mbits >> (j * TW + i)) & 1u;
                // RM: the right-hand side is where(mask, known, 0) and b - u == 0 at mask pixels
                // unless `general` (fixed up below)
                r[j][i] = m ? (RM ? 0.0 : bt[j][i] - uu) : res;
            }
        if (border) {
            // image border: fewer in-image neighbours (reflecting boundary, core.py:59-67)
#pragma unroll
            for (int j = 0; j < TH; ++j)
#pragma unroll
                for (int i = 0; i < TW; ++i) {
                    const int gy = gy0 + j, gx = gx0 + i;
                    const double miss = (gy == 0 ? 1.0 : 0.0) + (gy == H - 1 ? 1.0 : 0.0) +
                                        (gx == 0 ? 1.0 : 0.0) + (gx == W - 1 ? 1.0 : 0.0);
                    const bool m = (mbits >> (j * TW + i)) & 1u;
                    if (!m && miss != 0.0) r[j][i] = fma(miss * hinv2, uc[j + 1][i + 1], r[j][i]);
                }
        }
        if (RM && general) {
#pragma unroll
            for (int j = 0; j < TH; ++j)
#pragma unroll
                for (int i = 0; i < TW; ++i)
                    if ((mbits >> (j * TW + i)) & 1u)
                        r[j][i] = A.b[(size_t)p * A.plane + (size_t)(gy0 + j) * W + gx0 + i] - uc[j + 1][i + 1];
        }
    }

    // ---- local start: v0 = where(mask, g, 0), r0 = g - A_i v0 (solvers.py:331-333)
    double v[TH][TW], pc[TH][TW], q[TH][TW];
#pragma unroll
    for (int j = 0; j < TH; ++j)
#pragma unroll
        for (int i = 0; i < TW; ++i) v[j][i] = 0.0;
    if (general) {
#pragma unroll
        for (int j = 0; j < TH; ++j)
#pragma unroll
            for (int i = 0; i < TW; ++i) {
                const bool m = (mbits >> (j * TW + i)) & 1u;
                v[j][i] = m ? r[j][i] : 0.0;
                pc[j][i] = v[j][i];
            }
        cg.apply(pc, q);
#pragma unroll
        for (int j = 0; j < TH; ++j)
#pragma unroll
            for (int i = 0; i < TW; ++i) {
                const bool m = (mbits >> (j * TW + i)) & 1u;
                r[j][i] = m ? 0.0 : fma(-hinv2, q[j][i], r[j][i]);
            }
    }
    double rs_k = cg.group_sum(tile_dot<TW, TH>(r, r));

    if (rs_k > target) {  // solvers.py:336 (strict)
#pragma unroll
        for (int j = 0; j < TH; ++j)
#pragma unroll
            for (int i = 0; i < TW; ++i) pc[j][i] = r[j][i];
        double inv_rs = __drcp_rn(rs_k);  // reciprocal: division's slow path is off the chain
        for (int it = 0; it < A.max_iters; ++it) {
            cg.apply(pc, q);
            double d_pq = tile_dot<TW, TH>(pc, q);
            double d_rq = tile_dot<TW, TH>(r, q);
            double d_qq = tile_dot<TW, TH>(q, q);
            cg.group_sum3(d_pq, d_rq, d_qq);
            const double pq = hinv2 * d_pq;
            const bool ok = pq > 0.0;                 // solvers.py:348
            const double a = ok ? rs_k * __drcp_rn(pq) : 0.0;    // :349-350 (reciprocal + multiply)
            const double ah = a * hinv2;
            const double rs_new = fma(ah * ah, d_qq, fma(-2.0 * ah, d_rq, rs_k));
#pragma unroll
            for (int j = 0; j < TH; ++j)
#pragma unroll
                for (int i = 0; i < TW; ++i) {
                    v[j][i] = fma(a, pc[j][i], v[j][i]);
                    r[j][i] = fma(-ah, q[j][i], r[j][i]);
                }
            if (rs_new <= target || !ok) break;       // :354
            const double beta = rs_new * inv_rs;
            rs_k = rs_new;
            inv_rs = __drcp_rn(rs_k);
#pragma unroll
            for (int j = 0; j < TH; ++j)
#pragma unroll
                for (int i = 0; i < TW; ++i) pc[j][i] = fma(beta, pc[j][i], r[j][i]);
        }
    }

    // ---- weighted correction (v * wy) * wx (solvers.py:309-310)
    {
        double *out = A.scratch + ((size_t)p * L.nblocks + blk) * (BW * BH);
        const double2 wx0 = *reinterpret_cast<const double2 *>(&sm.wx[bx]);
        const double2 wx1 = *reinterpret_cast<const double2 *>(&sm.wx[bx + 2]);
        const double2 wy0 = *reinterpret_cast<const double2 *>(&sm.wy[by]);
        const double2 wy1 = *reinterpret_cast<const double2 *>(&sm.wy[by + 2]);
        const double wyv[4] = {wy0.x, wy0.y, wy1.x, wy1.y};
#pragma unroll
        for (int j = 0; j < TH; ++j) {
            double2 o0, o1;
            o0.x = (v[j][0] * wyv[j]) * wx0.x;
            o0.y = (v[j][1] * wyv[j]) * wx0.y;
            o1.x = (v[j][2] * wyv[j]) * wx1.x;
            o1.y = (v[j][3] * wyv[j]) * wx1.y;
            double2 *row = reinterpret_cast<double2 *>(out + (by + j) * BW + bx);
            row[0] = o0;
            row[1] = o1;
        }
    }
    if (FUSE) {
        // ---- combine on arrival
        __shared__ int s_do[16];
        __threadfence();   // this block's tile is visible device-wide before its arrivals are counted
        __syncthreads();
        const int cx1 = Fz.lastx[ix], cy1 = Fz.lasty[iy];
        const int ncx = cx1 - ix + 1, ncell = ncx * (cy1 - iy + 1);
        if (tid < ncell && tid < 16) {
            const int cy = iy + tid / ncx, cx = ix + tid % ncx;
            const int cell = cy * L.nx + cx;
            const unsigned old = atomicAdd(&Fz.cell_cnt[(size_t)p * L.nblocks + cell], 1u);
            s_do[tid] = (old + 1u == (unsigned)Fz.cell_need[cell]) ? 1 : 0;
        }
        __syncthreads();
        for (int k = 0; k < ncell && k < 16; ++k) {
            if (!s_do[k]) continue;
            __threadfence();   // the other blocks' tiles (their fences precede their arrivals)
            combine_cell(L, A.scratch + (size_t)p * L.nblocks * (BW * BH), A.u + (size_t)p * A.plane,
                         Fz.u_out + (size_t)p * A.plane, ix + k % ncx, iy + k / ncx, tid);
        }
    }
}

// ------------------------------------------------------------------ K2S ---
// Same block solve with the CG state split between registers and shared memory:
// the search direction p (needed by the neighbours through shuffles) and, unless
// SR, the residual r stay in registers; the iterate v and the operator image q
// = A_i p (both touched once per CG step, never exchanged) live in shared memory.
// The register tile of K2 holds 4 arrays x 16 px x 2 regs = 128 registers of
// pure state, which caps residency at 4 blocks per SM and leaves the FP64 pipe
// waiting on the latency of the reductions; K2S fits 8 blocks per SM.
// Thread t owns double2 slot [k][t] (k = 2*row + half): 16-byte accesses, a
// warp reads 512 contiguous bytes, no bank conflicts, no hazards between threads.
template <int TW, int TH, int NWARP, bool SR>
struct TileSmemS {
    static constexpr int NT = NWARP * 32, K = TH * TW / 2;
    double2 v[K][NT];
    double2 q[K][NT];
    double2 r[SR ? K : 1][SR ? NT : 1];
    double xrow[NWARP > 1 ? NWARP * 2 * 8 * TW : 1];
    double red[2 * NWARP * 3];
};

template <int TW, int TH, int NWARP, bool RM, bool SR>
__device__ __forceinline__ void tile_block_solve_s(const SweepArgs &A, int p, int blk,
                                                   TileSmemS<TW, TH, NWARP, SR> &sm, double target,
                                                   double *__restrict__ out) {
    static_assert(TW == 4, "K2S stores rows as two double2");
    using CG = TileCG<TW, TH, NWARP>;
    constexpr int BW = CG::BW, BH = CG::BH;
    const LevelDev &L = A.L;
    const int iy = blk / L.nx, ix = blk - iy * L.nx;
    const int x0 = L.xs[ix], y0 = L.ys[iy];
    const int W = L.w, H = L.h;
    const int tid = threadIdx.x;

    CG cg;
    cg.lane = tid & 31;
    cg.wg = tid >> 5;
    cg.bar_id = 1;
    cg.lx = cg.lane & 7;
    cg.ly = cg.lane >> 3;
    cg.xrow = sm.xrow;
    cg.red = sm.red;
    cg.slot = 0;
    cg.eL = cg.lx == 0;
    cg.eR = cg.lx == 7;
    cg.eT = cg.wg == 0 && cg.ly == 0;
    cg.eB = cg.wg == NWARP - 1 && cg.ly == 3;
    const double g_in = 1.0 - L.robin / L.hinv2;  // 1 - alpha*h
    cg.gL = x0 > 0 ? g_in : 1.0;
    cg.gR = x0 + BW < W ? g_in : 1.0;
    cg.gT = y0 > 0 ? g_in : 1.0;
    cg.gB = y0 + BH < H ? g_in : 1.0;

    const int bx = cg.lx * TW, by = (cg.wg * 4 + cg.ly) * TH;
    const int gx0 = x0 + bx, gy0 = y0 + by;
    const double *up = A.u + (size_t)p * A.plane;
    const double *bp = A.b + (size_t)p * A.plane;
    const uint8_t *mp = A.mask + (size_t)(p / A.channels) * A.plane;
    const double hinv2 = L.hinv2;

    // ---- gather: global residual g = b - A u on the tile (core.py:100-110)
    double r[TH][TW];
    unsigned mbits = 0;
    {
        double uc[TH + 2][TW + 2];
#pragma unroll
        for (int j = 0; j < TH + 2; ++j) {
            const int gy = gy0 + j - 1;
#pragma unroll
            for (int i = 0; i < TW + 2; ++i) {
                const int gx = gx0 + i - 1;
                const bool corner = (j == 0 || j == TH + 1) && (i == 0 || i == TW + 1);
                const bool in = gy >= 0 && gy < H && gx >= 0 && gx < W;
                uc[j][i] = (!corner && in) ? up[(size_t)gy * W + gx] : 0.0;
            }
        }
#pragma unroll
        for (int j = 0; j < TH; ++j) {
            const int gy = gy0 + j;
            const double cy = 4.0 - (gy == 0 ? 1.0 : 0.0) - (gy == H - 1 ? 1.0 : 0.0);
#pragma unroll
            for (int i = 0; i < TW; ++i) {
                const int gx = gx0 + i;
                const size_t gi = (size_t)gy * W + gx;
                const bool m = mp[gi] != 0;
                if (m) mbits |= 1u << (j * TW + i);
                const double cnt = cy - (gx == 0 ? 1.0 : 0.0) - (gx == W - 1 ? 1.0 : 0.0);
                const double s = ((uc[j][i + 1] + uc[j + 2][i + 1]) + uc[j + 1][i]) + uc[j + 1][i + 2];
                const double au = s * (-hinv2) + (cnt * hinv2) * uc[j + 1][i + 1];
                double bb;
                if (RM) bb = m ? bp[gi] : 0.0; else bb = bp[gi];
                r[j][i] = m ? (bb - uc[j + 1][i + 1]) : (bb - au);
            }
        }
    }
    cg.mbits = mbits;

    // ---- local start: v0 = where(mask, g, 0), r0 = g - A_i v0 (solvers.py:331-333)
    double pc[TH][TW];
    const bool general = A.mflag[p] != 0;
    if (general) {
        double q[TH][TW];
#pragma unroll
        for (int j = 0; j < TH; ++j)
#pragma unroll
            for (int i = 0; i < TW; ++i) {
                const bool m = (mbits >> (j * TW + i)) & 1u;
                pc[j][i] = m ? r[j][i] : 0.0;
            }
#pragma unroll
        for (int j = 0; j < TH; ++j) {
            sm.v[2 * j][tid] = make_double2(pc[j][0], pc[j][1]);
            sm.v[2 * j + 1][tid] = make_double2(pc[j][2], pc[j][3]);
        }
        cg.apply(pc, q);
#pragma unroll
        for (int j = 0; j < TH; ++j)
#pragma unroll
            for (int i = 0; i < TW; ++i) {
                const bool m = (mbits >> (j * TW + i)) & 1u;
                r[j][i] = m ? 0.0 : fma(-hinv2, q[j][i], r[j][i]);
            }
    }
    double rs_k = cg.group_sum(tile_dot<TW, TH>(r, r));
    bool have_v = general;  // v == 0 is not materialised before the first CG step

    if (rs_k > target) {  // solvers.py:336 (strict)
#pragma unroll
        for (int j = 0; j < TH; ++j)
#pragma unroll
            for (int i = 0; i < TW; ++i) pc[j][i] = r[j][i];
        if (SR) {
#pragma unroll
            for (int j = 0; j < TH; ++j) {
                sm.r[2 * j][tid] = make_double2(r[j][0], r[j][1]);
                sm.r[2 * j + 1][tid] = make_double2(r[j][2], r[j][3]);
            }
        }
        double inv_rs = 1.0 / rs_k;
        for (int it = 0; it < A.max_iters; ++it) {
            double d_pq, d_rq, d_qq;
            {
                double q[TH][TW];
                cg.apply(pc, q);
                if (SR) {
#pragma unroll
                    for (int j = 0; j < TH; ++j) {
                        const double2 a0 = sm.r[2 * j][tid], a1 = sm.r[2 * j + 1][tid];
                        r[j][0] = a0.x; r[j][1] = a0.y; r[j][2] = a1.x; r[j][3] = a1.y;
                    }
                }
                d_pq = tile_dot<TW, TH>(pc, q);
                d_rq = tile_dot<TW, TH>(r, q);
                d_qq = tile_dot<TW, TH>(q, q);
#pragma unroll
                for (int j = 0; j < TH; ++j) {
                    sm.q[2 * j][tid] = make_double2(q[j][0], q[j][1]);
                    sm.q[2 * j + 1][tid] = make_double2(q[j][2], q[j][3]);
                }
            }
            cg.group_sum3(d_pq, d_rq, d_qq);
            const double pq = hinv2 * d_pq;
            const bool ok = pq > 0.0;                 // solvers.py:348
            const double a = ok ? rs_k / pq : 0.0;    // :349-350
            const double ah = a * hinv2;
            const double rs_new = fma(ah * ah, d_qq, fma(-2.0 * ah, d_rq, rs_k));
            const bool last = rs_new <= target || !ok;  // :354
            const double beta = rs_new * inv_rs;
#pragma unroll
            for (int j = 0; j < TH; ++j) {
                // v += a p
                double2 v0 = make_double2(0.0, 0.0), v1 = v0;
                if (have_v) {
                    v0 = sm.v[2 * j][tid];
                    v1 = sm.v[2 * j + 1][tid];
                }
                v0.x = fma(a, pc[j][0], v0.x); v0.y = fma(a, pc[j][1], v0.y);
                v1.x = fma(a, pc[j][2], v1.x); v1.y = fma(a, pc[j][3], v1.y);
                sm.v[2 * j][tid] = v0;
                sm.v[2 * j + 1][tid] = v1;
                if (!last) {
                    // r -= a q ; p = beta p + r
                    const double2 q0 = sm.q[2 * j][tid], q1 = sm.q[2 * j + 1][tid];
                    double2 r0, r1;
                    if (SR) {
                        r0 = sm.r[2 * j][tid];
                        r1 = sm.r[2 * j + 1][tid];
                    } else {
                        r0 = make_double2(r[j][0], r[j][1]);
                        r1 = make_double2(r[j][2], r[j][3]);
                    }
                    r0.x = fma(-ah, q0.x, r0.x); r0.y = fma(-ah, q0.y, r0.y);
                    r1.x = fma(-ah, q1.x, r1.x); r1.y = fma(-ah, q1.y, r1.y);
                    if (SR) {
                        sm.r[2 * j][tid] = r0;
                        sm.r[2 * j + 1][tid] = r1;
                    } else {
                        r[j][0] = r0.x; r[j][1] = r0.y; r[j][2] = r1.x; r[j][3] = r1.y;
                    }
                    pc[j][0] = fma(beta, pc[j][0], r0.x); pc[j][1] = fma(beta, pc[j][1], r0.y);
                    pc[j][2] = fma(beta, pc[j][2], r1.x); pc[j][3] = fma(beta, pc[j][3], r1.y);
                }
            }
            have_v = true;
            if (last) break;
            rs_k = rs_new;
            inv_rs = 1.0 / rs_k;
        }
    }

    // ---- weighted correction (v * wy) * wx (solvers.py:309-310)
    double wxv[TW];
#pragma unroll
    for (int i = 0; i < TW; ++i) wxv[i] = L.wx[ix * BW + bx + i];
#pragma unroll
    for (int j = 0; j < TH; ++j) {
        const double wyv = L.wy[iy * BH + by + j];
        double *row = out + (by + j) * BW + bx;
        double2 v0 = make_double2(0.0, 0.0), v1 = v0;
        if (have_v) {
            v0 = sm.v[2 * j][tid];
            v1 = sm.v[2 * j + 1][tid];
        }
        double2 o0, o1;
        o0.x = (v0.x * wyv) * wxv[0];
        o0.y = (v0.y * wyv) * wxv[1];
        o1.x = (v1.x * wyv) * wxv[2];
        o1.y = (v1.y * wyv) * wxv[3];
        *reinterpret_cast<double2 *>(row) = o0;
        *reinterpret_cast<double2 *>(row + 2) = o1;
    }
}

#ifndef B200P_TILES_MINB
#define B200P_TILES_MINB 8
#endif
template <int TW, int TH, int NWARP, bool RM, bool SR>
__global__ void __launch_bounds__(NWARP * 32, B200P_TILES_MINB)
oras_sweep_tile_s_kernel(const SweepArgs A) {
    __shared__ __align__(16) TileSmemS<TW, TH, NWARP, SR> sm;
    const int p = blockIdx.y;
    if (A.pred && !A.pred[p]) return;
    const double rs_g = A.rs[p];
    if (rs_g == 0.0) return;  // oras_sweeps exit, solvers.py:420
    const int blk = blockIdx.x;
    double *out = A.scratch + ((size_t)p * A.L.nblocks + blk) * (8 * TW * 4 * TH * NWARP);
    tile_block_solve_s<TW, TH, NWARP, RM, SR>(A, p, blk, sm, A.eta * rs_g, out);
}

// ------------------------------------------------------------------ K2F ---
// Fused sweep: solve + deterministic combine in ONE persistent kernel.
//
// Work items are claimed from an atomic counter in a fixed order.  Per problem
// the order is, block-row by block-row: the solve items of block row t, then the
// combine items of pixel band t - lag.  Band j is the set of pixel rows whose
// LAST covering block row is j (rows [ys[j], ys[j+1]), the last band runs to the
// image bottom); its u_new = u_old + sum of covering blocks' weighted
// corrections needs block rows <= j only.  Solve items write their weighted
// correction tile into a RING of R block rows (slot = global row index mod R),
// signal `row_done`; combine items wait for the rows they read, sum the
// contributions in ascending block order (np.bincount order, solvers.py:310-314)
// and write u_new.  A solve item that re-uses a ring slot first waits for the
// bands that read the slot's previous occupant (`band_done`).  Every wait points
// to an item EARLIER in the claim order, so the earliest unfinished item never
// blocks: no deadlock for any number of resident CTAs.
//
// The ring (R * nx tiles, a few MB) stays resident in L2, so the corrections
// never travel to HBM: the sweep's DRAM traffic is read u_old + write u_new
// (+ mask, rhs).  u is ping-ponged (u_old -> u_new); skipped problems (frozen
// by `pred`, or rs == 0) are copied through so that every problem's current
// iterate lives in the same buffer.
struct FusedArgs {
    SweepArgs S;          // S.u = u_old, S.scratch = ring
    double *u_new;
    int R, lag;           // ring depth in block rows; combine lag in block rows
    int nsx;              // solve items per block row (ceil(nx / blocks per CTA))
    int nc, cw;           // combine chunks per band, chunk width in pixels
    int P, items_per_problem;
    unsigned *work;       // [1] claim counter (zeroed before launch)
    unsigned *row_done;   // [P*ny] solve items finished per block row
    unsigned *band_done;  // [P*ny] combine items finished per band
    const int *band_first_row;  // [ny] first block row a band reads
    const int *row_last_band;   // [ny] last band that reads a block row
    int *unit_counter;    // per-problem sweep counter (may be null)
    unsigned long long *stats;  // debug (may be null): cycles solve, combine, wait-ring, wait-rows; item counts
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void spin_until(const unsigned *ctr, unsigned target) {
    while (ld_acquire_u32(ctr) < target) __nanosleep(40);
}

constexpr int FUSED_THREADS = 128;

#ifndef B200P_FUSED_MINB
#define B200P_FUSED_MINB 4
#endif
#ifndef B200P_COMBINE_G
#define B200P_COMBINE_G 8
#endif

__device__ __forceinline__ void cp_async8(void *smem_dst, const void *gmem_src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

template <int TW, int TH, int NWARP, bool RM>
__global__ void __launch_bounds__(FUSED_THREADS, (TH * TW * NWARP <= 32 ? B200P_FUSED_MINB : 1))
oras_fused_sweep_kernel(const FusedArgs A) {
    constexpr int BW = 8 * TW, BH = 4 * TH * NWARP;
    constexpr int BPC = FUSED_THREADS / (NWARP * 32);  // blocks per solve item
    __shared__ TileSmem<TW, TH, NWARP> sm[BPC];
    __shared__ unsigned s_item[2];
    __shared__ int s_rn[BH], s_rf[BH];
    __shared__ size_t s_roff[BH][2];
    extern __shared__ __align__(16) double s_u[];  // BH x FUSED_THREADS staging of u_old
    const LevelDev &L = A.S.L;
    const int tid = threadIdx.x;
    const int ny = L.ny, nx = L.nx;
    const unsigned total = (unsigned)A.P * (unsigned)A.items_per_problem;
    const int lag = A.lag < ny ? A.lag : ny;
    const int per_slot = A.nsx + A.nc;

    // claim-ahead: the next item is requested while the current one is processed.  An item
    // claimed early still only waits on items earlier in the order, so progress is kept.
    if (tid == 0) s_item[0] = atomicAdd(A.work, 1u);
    __syncthreads();
    for (int it = 0;; ++it) {
        const unsigned item = s_item[it & 1];
        if (item >= total) break;
        if (tid == 0) s_item[(it + 1) & 1] = atomicAdd(A.work, 1u);
        const int p = (int)(item / (unsigned)A.items_per_problem);
        int q = (int)(item - (unsigned)p * (unsigned)A.items_per_problem);
        // ---- decode (see the order described above)
        bool solve;
        int row, sub;
        if (q < lag * A.nsx) {
            solve = true; row = q / A.nsx; sub = q - row * A.nsx;
        } else {
            q -= lag * A.nsx;
            const int mid = (ny - lag) * per_slot;
            if (q < mid) {
                const int t = q / per_slot, r = q - t * per_slot;
                if (r < A.nsx) { solve = true; row = lag + t; sub = r; }
                else { solve = false; row = t; sub = r - A.nsx; }
            } else {
                q -= mid;
                solve = false; row = (ny - lag) + q / A.nc; sub = q % A.nc;
            }
        }
        const bool skip = (A.S.pred && !A.S.pred[p]) || A.S.rs[p] == 0.0;
        const int grow = p * ny + row;  // global block row / band index
        long long t0 = 0, t1 = 0;
        if (A.stats && tid == 0) t0 = t1 = clock64();

        if (solve) {
            if (!skip) {
                // Ring slot re-use: the bands that read the slot's previous occupant must be done
                // before the tile is WRITTEN (end of the item).  Poll the flags now (one lane per
                // band), re-check just before the stores.
                const int old = grow - A.R;
                const unsigned *flag = nullptr;
                bool ok = true;
                if (old >= 0) {
                    const int op = old / ny, orow = old - op * ny;
                    if (tid <= A.row_last_band[orow] - orow) {
                        flag = &A.band_done[op * ny + orow + tid];
                        ok = ld_acquire_u32(flag) >= (unsigned)A.nc;
                    }
                }
                auto pre_store = [&]() {
                    if (!ok) {
                        long long w0 = 0;
                        if (A.stats) w0 = clock64();
                        spin_until(flag, (unsigned)A.nc);
                        if (A.stats) atomicAdd(&A.stats[2], (unsigned long long)(clock64() - w0));
                    }
                    __syncthreads();
                };
                const int warp = tid >> 5;
                const int grp = warp / NWARP, wg = warp - grp * NWARP;
                const int ix = sub * BPC + grp;
                if (ix < nx) {
                    double *out = A.S.scratch + ((size_t)(grow % A.R) * nx + ix) * (BW * BH);
                    tile_block_solve<TW, TH, NWARP, RM, true>(A.S, p, row * nx + ix, grp, wg, sm[grp],
                                                              A.S.eta * A.S.rs[p], out, pre_store);
                } else {
                    pre_store();
                }
            }
            __syncthreads();
            if (tid == 0) {
                __threadfence();
                atomicAdd(&A.row_done[grow], 1u);
                if (A.stats) {
                    atomicAdd(&A.stats[0], (unsigned long long)(clock64() - t0));
                    atomicAdd(&A.stats[4], 1ull);
                }
            }
        } else {
            // ---- combine band `row`, columns [sub*cw, sub*cw + cw); cw == FUSED_THREADS
            const int y0 = L.ys[row];
            const int y1 = row + 1 < ny ? L.ys[row + 1] : L.h;
            const int rows = y1 - y0;  // <= BH
            const int x = sub * A.cw + tid;
            const bool inx = x < L.w;
            const double *uo = A.S.u + (size_t)p * A.S.plane;
            double *un = A.u_new + (size_t)p * A.S.plane;
            // u_old of the whole chunk goes to shared memory asynchronously (no registers held)
            if (inx)
                for (int k = 0; k < rows; ++k)
                    cp_async8(&s_u[k * FUSED_THREADS + tid], uo + (size_t)(y0 + k) * L.w + x);
            if (skip) {
                cp_async_wait_all();
                if (inx)
                    for (int k = 0; k < rows; ++k)
                        un[(size_t)(y0 + k) * L.w + x] = s_u[k * FUSED_THREADS + tid];
            } else {
                // rows this band reads must be complete: one lane per block row polls
                const int r0 = A.band_first_row[row];
                if (tid <= row - r0) spin_until(&A.row_done[p * ny + r0 + tid], (unsigned)A.nsx);
                if (A.stats && tid == 0) t1 = clock64();
                if (A.unit_counter && row == 0 && sub == 0 && tid == 0) A.unit_counter[p] += 1;
                const size_t bsz = (size_t)BW * BH;
                // per-row covering block rows (uniform over the chunk): count + ring offsets of
                // the first two tiles' row starts
                if (tid < rows) {
                    const int y = y0 + tid;
                    const int iyf = L.cyf[y], iyn = L.cyn[y];
                    s_rn[tid] = iyn;
                    s_rf[tid] = iyf;
                    for (int a = 0; a < 2; ++a) {
                        const int iy = iyf + (a < iyn ? a : 0);
                        s_roff[tid][a] = ((size_t)((p * ny + iy) % A.R) * nx) * bsz + (size_t)(y - L.ys[iy]) * BW;
                    }
                }
                __syncthreads();
                if (inx) {
                    const int ixf = L.cxf[x], ixn = L.cxn[x];
                    const size_t xo0 = (size_t)ixf * bsz + (x - L.xs[ixf]);
                    const size_t xo1 = ixn > 1 ? (size_t)(ixf + 1) * bsz + (x - L.xs[ixf + 1]) : 0;
                    const double *ring = A.S.scratch;
                    constexpr int G = B200P_COMBINE_G;
                    const bool two_x = ixn > 1;
                    const bool wide = ixn > 2;  // > 2 covering blocks per axis: heavily overlapped layouts
                    bool landed = false;
                    for (int k0 = 0; k0 < rows; k0 += G) {
                        double cc[G], v00[G], v01[G], v10[G], v11[G];
                        // all ring loads first, branch-free (absent contributions re-read tile 0 and
                        // are discarded), so that 4*G independent loads per thread are in flight
#pragma unroll
                        for (int j = 0; j < G; ++j) {
                            const int k = k0 + j < rows ? k0 + j : rows - 1;
                            const size_t o0 = s_roff[k][0], o1 = s_roff[k][1];
                            v00[j] = __ldcg(ring + o0 + xo0);
                            v01[j] = __ldcg(ring + o0 + (two_x ? xo1 : xo0));
                            v10[j] = __ldcg(ring + o1 + xo0);
                            v11[j] = __ldcg(ring + o1 + (two_x ? xo1 : xo0));
                        }
#pragma unroll
                        for (int j = 0; j < G; ++j) {
                            const int k = k0 + j < rows ? k0 + j : rows - 1;
                            const int n = s_rn[k];
                            // ascending block order: (iy0,ix0), (iy0,ix1), (iy1,ix0), (iy1,ix1)
                            double acc = v00[j];
                            acc += two_x ? v01[j] : 0.0;
                            if (wide || n > 2) {
                                acc = 0.0;
                                for (int a = 0; a < n; ++a) {
                                    const int iy = s_rf[k] + a;
                                    const size_t oa = ((size_t)((p * ny + iy) % A.R) * nx) * bsz +
                                                      (size_t)(y0 + k - L.ys[iy]) * BW;
                                    for (int c = 0; c < ixn; ++c)
                                        acc += __ldcg(ring + oa + (size_t)(ixf + c) * bsz + (x - L.xs[ixf + c]));
                                }
                            } else {
                                acc += n > 1 ? v10[j] : 0.0;
                                acc += (n > 1 && two_x) ? v11[j] : 0.0;
                            }
                            cc[j] = acc;
                        }
                        if (!landed) {
                            cp_async_wait_all();  // own copies only: each thread reads back what it issued
                            landed = true;
                        }
#pragma unroll
                        for (int j = 0; j < G; ++j)
                            if (k0 + j < rows)
                                un[(size_t)(y0 + k0 + j) * L.w + x] = s_u[(k0 + j) * FUSED_THREADS + tid] + cc[j];
                    }
                }
            }
            __syncthreads();
            if (tid == 0) {
                __threadfence();
                atomicAdd(&A.band_done[grow], 1u);
                if (A.stats) {
                    const long long t2 = clock64();
                    atomicAdd(&A.stats[1], (unsigned long long)(t2 - t1));
                    atomicAdd(&A.stats[3], (unsigned long long)(t1 - t0));
                    atomicAdd(&A.stats[5], 1ull);
                }
            }
        }
        __syncthreads();  // s_item[(it+1)&1] visible; shared staging free for the next item
    }
}

// ------------------------------------------------------------------ K2b' --
// Band combine.  The partition-of-unity ramp starts at 0 on every cut side (partition.py:137-154), so the
// outermost pixel ring of a block has weight 0 and most pixels of a level have exactly ONE writer with
// weight exactly 1.  The warp-per-block solve (K2W, DIRECT) writes those straight into the partner
// iterate u_out = u + v; only pixels of the overlap bands travel through tiles.  This kernel visits the
// band pixels only -- launch 1: the band rows (every column), launch 2: the remaining rows x the band
// columns -- and forms u_out = u + sum of the covering tiles with a non-zero weight, in ascending block
// order (the zero-weight tiles the full combine adds are exact zeros, so the result is the same).
// Tiles use the KW layout (rows of TP doubles, column = x - (x0 & ~7)).
struct BandTables {
    const int *nzxf, *nzxn;   // per pixel column: first block column with a non-zero weight, how many
    const int *nzyf, *nzyn;   // per pixel row
    const int *rows;          // the rows of this launch
    const int *cols;          // the columns of this launch, or null = all columns
    int nrows, ncols;
    int tp, tsz;              // tile row pitch and tile size in doubles
};

template <int NY>   // rows of the launch have at most NY non-zero row slots (more: the generic loop)
__global__ void __launch_bounds__(ST_THREADS_COMBINE)
oras_combine_band_kernel(const LevelDev L, const BandTables T, const double *__restrict__ scratch, size_t plane,
                         const int *__restrict__ pred, const double *__restrict__ rs,
                         const double *__restrict__ u_in, double *__restrict__ u_out,
                         int *__restrict__ unit_counter) {
    __shared__ int s_y[COMBINE_ROWS], s_rn[COMBINE_ROWS], s_rf[COMBINE_ROWS];
    __shared__ size_t s_roff[COMBINE_ROWS][2];
    const int p = blockIdx.z;
    if (pred && !pred[p]) return;
    if (rs[p] == 0.0) return;
    const int tid = threadIdx.x;
    const int ci = blockIdx.x * ST_THREADS_COMBINE + tid;
    const int k_lo = blockIdx.y * COMBINE_ROWS;
    const int rows = min(COMBINE_ROWS, T.nrows - k_lo);
    if (unit_counter && blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) unit_counter[p] += 1;
    if (tid < rows) {
        const int y = T.rows[k_lo + tid];
        const int iyf = T.nzyf[y], iyn = T.nzyn[y];
        s_y[tid] = y;
        s_rn[tid] = iyn;
        s_rf[tid] = iyf;
        for (int a = 0; a < 2; ++a) {
            const int iy = iyf + (a < iyn ? a : 0);
            s_roff[tid][a] = (size_t)iy * L.nx * T.tsz + (size_t)(y - L.ys[iy]) * T.tp;
        }
    }
    __syncthreads();
    if (ci >= T.ncols) return;
    const int x = T.cols ? T.cols[ci] : ci;
    const int ixf = T.nzxf[x], ixn = T.nzxn[x];
    const size_t xo0 = (size_t)ixf * T.tsz + (x - (L.xs[ixf] & ~7));
    const bool two_x = ixn > 1;
    const size_t xo1 = two_x ? (size_t)(ixf + 1) * T.tsz + (x - (L.xs[ixf + 1] & ~7)) : xo0;
    const bool wide = ixn > 2;
    const double *sp = scratch + (size_t)p * L.nblocks * T.tsz;
    const double *ui = u_in + (size_t)p * plane;
    double *uo = u_out + (size_t)p * plane;
    constexpr int G = COMBINE_G;
    for (int k0 = 0; k0 < rows; k0 += G) {
        double uu[G], v00[G], v01[G], v10[NY > 1 ? G : 1], v11[NY > 1 ? G : 1];
#pragma unroll
        for (int j = 0; j < G; ++j) {
            const int k = k0 + j < rows ? k0 + j : rows - 1;
            const size_t o0 = s_roff[k][0];
            uu[j] = ui[(size_t)s_y[k] * L.w + x];
            v00[j] = __ldcs(sp + o0 + xo0);
            v01[j] = __ldcs(sp + o0 + xo1);
            if (NY > 1) {
                const size_t o1 = s_roff[k][1];
                v10[j] = __ldcs(sp + o1 + xo0);
                v11[j] = __ldcs(sp + o1 + xo1);
            }
        }
#pragma unroll
        for (int j = 0; j < G; ++j) {
            const int k = k0 + j;
            if (k >= rows) break;
            const int n = s_rn[k], y = s_y[k];
            // ascending block order: (iy0,ix0), (iy0,ix1), (iy1,ix0), (iy1,ix1)
            double acc = v00[j];
            acc += two_x ? v01[j] : 0.0;
            if (wide || n > NY) {
                acc = 0.0;
                for (int a = 0; a < n; ++a) {
                    const int iy = s_rf[k] + a;
                    const size_t oa = (size_t)iy * L.nx * T.tsz + (size_t)(y - L.ys[iy]) * T.tp;
                    for (int c = 0; c < ixn; ++c)
                        acc += sp[oa + (size_t)(ixf + c) * T.tsz + (x - (L.xs[ixf + c] & ~7))];
                }
            } else if (NY > 1) {
                acc += n > 1 ? v10[NY > 1 ? j : 0] : 0.0;
                acc += (n > 1 && two_x) ? v11[NY > 1 ? j : 0] : 0.0;
            }
            uo[(size_t)y * L.w + x] = uu[j] + acc;
        }
    }
}

// Problems the sweep skips (frozen, or zero residual) keep their iterate: copied to the partner buffer so that
// the ping-pong swap after a band-combine sweep is valid for every problem of the plan.
__global__ void __launch_bounds__(ST_THREADS_COMBINE)
copy_skipped_problems_kernel(size_t plane2, const int *__restrict__ pred, const double *__restrict__ rs,
                             const double2 *__restrict__ u_in, double2 *__restrict__ u_out) {
    const int p = blockIdx.y;
    if ((!pred || pred[p]) && rs[p] != 0.0) return;   // live: the sweep wrote it
    const double2 *a = u_in + (size_t)p * plane2;
    double2 *b = u_out + (size_t)p * plane2;
    for (size_t i = (size_t)blockIdx.x * ST_THREADS_COMBINE + threadIdx.x; i < plane2;
         i += (size_t)gridDim.x * ST_THREADS_COMBINE)
        b[i] = a[i];
}


}  // namespace b200p
