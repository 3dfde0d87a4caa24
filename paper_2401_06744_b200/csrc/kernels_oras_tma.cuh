// kernels_oras_tma.cuh -- K2T: the ORAS block smoother fed by TMA.
//
// ncu on the register-tile kernel K2 (kernels_oras.cuh) showed the L1TEX data pipe
// (l1tex__data_pipe_lsu_wavefronts) as the most loaded unit: every thread gathered its
// 6x6 window of u and 16 mask bytes with scalar global loads (~930 wavefronts per block,
// more than the whole CG loop's shuffles) and the load latency was exposed at the start
// of every block.  K2T keeps the register-tile CG but changes how data moves:
//
//   * persistent CTAs (2 warps, one 32x32 block at a time) walk the (problem, block) items;
//   * the block's u window (1-pixel halo, zero-filled outside the image by the TMA unit; staged
//     as a 36x34 box because the innermost TMA coordinate must be 16-byte aligned, so the box
//     starts at x0-2 with x0 even) is fetched with ONE cp.async.bulk.tensor into shared memory, signalled on
//     an mbarrier, and the NEXT item's window is requested as soon as the current one has
//     been read, so the fetch overlaps the CG iterations (levels >= 1 of a V-cycle fetch
//     their explicit right-hand-side tile the same way);
//   * the block-local Dirichlet mask comes from a bit table packed once per hierarchy build
//     (one coalesced 32-bit load per thread, prefetched one item ahead);
//   * the weighted correction tile is staged in shared memory and written back with one
//     8 KB cp.async.bulk store.
//
// Semantics are those of tile_block_solve (solvers.py:303-305, :328-370, :309-310).
#pragma once
#include <cuda.h>

#include "kernels_oras.cuh"
#include "tma_utils.cuh"

namespace b200p {

struct SweepTmaArgs {
    SweepArgs S;
    const unsigned *mtab;  // (F, nblocks, 64): bit j*4+i of word t = mask of thread t's pixel (i, j)
    int total_items;       // P * nblocks
};

constexpr int KT_WIN_W = 36;  // staged window: x0-2 .. x0+33 (16-byte aligned start), y0-1 .. y0+32
constexpr int KT_WIN_H = 34;
constexpr int KT_THREADS = 64;

template <bool RM>
struct KtSmem {
    alignas(128) double u[KT_WIN_W * KT_WIN_H + 8];  // 9856 B (TMA box 36x34, dense)
    alignas(128) double out[32 * 32];              // weighted correction tile, bulk-stored
    alignas(128) double b[RM ? 16 : 32 * 32];      // explicit rhs tile (V-cycle levels >= 1)
    TileSmem<4, 4, 2> cg;
    alignas(8) unsigned long long bar;
};

// Packs the block-local masks of a level: grid (nblocks, F), 64 threads.
__global__ void __launch_bounds__(KT_THREADS)
pack_block_masks_kernel(const LevelDev L, const uint8_t *__restrict__ mask, size_t plane,
                        unsigned *__restrict__ mtab, int blk0) {
    const int blk = blockIdx.x + blk0, f = blockIdx.y, t = threadIdx.x;
    const int iy = blk / L.nx, ix = blk - iy * L.nx;
    const int lane = t & 31, wg = t >> 5;
    const int gx0 = L.xs[ix] + (lane & 7) * 4, gy0 = L.ys[iy] + (wg * 4 + (lane >> 3)) * 4;
    const uint8_t *mp = mask + (size_t)f * plane;
    unsigned bits = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (mp[(size_t)(gy0 + j) * L.w + gx0 + i]) bits |= 1u << (j * 4 + i);
    mtab[((size_t)f * L.nblocks + blk) * KT_THREADS + t] = bits;
}

template <bool RM, int REGCAP>
__global__ void __launch_bounds__(KT_THREADS) __maxnreg__(REGCAP)
oras_sweep_tma_kernel(const SweepTmaArgs A, const __grid_constant__ CUtensorMap tm_u,
                      const __grid_constant__ CUtensorMap tm_b) {
    constexpr int TW = 4, TH = 4, NWARP = 2, BW = 32, BH = 32;
    using CG = TileCG<TW, TH, NWARP>;
    __shared__ KtSmem<RM> sm;
    const SweepArgs &S = A.S;
    const LevelDev &L = S.L;
    const int tid = threadIdx.x;
    const int nblocks = L.nblocks, total = A.total_items;
    const int W = L.w, H = L.h;
    const double hinv2 = L.hinv2;

    // items of frozen problems (pred) and of problems with a zero residual (solvers.py:420) are skipped
    auto next_valid = [&](int it) {
        while (it < total) {
            const int p = it / nblocks;
            if ((!S.pred || S.pred[p]) && S.rs[p] != 0.0) break;
            it += gridDim.x;
        }
        return it;
    };
    int item = next_valid(blockIdx.x);
    if (item >= total) return;

    const unsigned bar = smem_u32(&sm.bar);
    const unsigned s_u = smem_u32(sm.u), s_b = smem_u32(sm.b), s_out = smem_u32(sm.out);
    auto request = [&](int it) {  // thread 0: fetch the window (and rhs tile) of item `it`
        const int p = it / nblocks, blk = it - p * nblocks;
        const int iy = blk / L.nx, ix = blk - iy * L.nx;
        const int x0 = L.xs[ix], y0 = L.ys[iy];
        mbar_expect_tx(bar, KT_WIN_W * KT_WIN_H * 8 + (RM ? 0 : BW * BH * 8));
        tma_load_3d(s_u, &tm_u, x0 - 2, y0 - 1, p, bar);
        if (!RM) tma_load_3d(s_b, &tm_b, x0, y0, p, bar);
    };
    if (tid == 0) {
        mbar_init(bar, 1);
        request(item);
    }
    __syncthreads();

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
    const double g_in = 1.0 - L.robin / L.hinv2;  // 1 - alpha*h
    const int bx = cg.lx * TW, by = (cg.wg * 4 + cg.ly) * TH;

    unsigned parity = 0;
    unsigned mb_next = A.mtab[((size_t)((item / nblocks) / S.channels) * nblocks + item % nblocks) * KT_THREADS + tid];

    for (;;) {
        const int p = item / nblocks, blk = item - p * nblocks;
        const int iy = blk / L.nx, ix = blk - iy * L.nx;
        const int x0 = L.xs[ix], y0 = L.ys[iy];
        const unsigned mbits = mb_next;
        const int nxt = next_valid(item + gridDim.x);
        if (nxt < total) {
            const int pn = nxt / nblocks;
            mb_next = A.mtab[((size_t)(pn / S.channels) * nblocks + (nxt - pn * nblocks)) * KT_THREADS + tid];
        }
        const double target = S.eta * S.rs[p];
        const bool general = S.mflag[p] != 0;
        cg.gL = x0 > 0 ? g_in : 1.0;
        cg.gR = x0 + BW < W ? g_in : 1.0;
        cg.gT = y0 > 0 ? g_in : 1.0;
        cg.gB = y0 + BH < H ? g_in : 1.0;
        cg.mbits = mbits;
        const int gx0 = x0 + bx, gy0 = y0 + by;

        mbar_wait(bar, parity);
        parity ^= 1u;

        // ---- gather: global residual g = b - A u on the tile (core.py:100-110) from the staged window
        double r[TH][TW];
        {
            double uc[TH + 2][TW + 2];
#pragma unroll
            for (int j = 0; j < TH + 2; ++j) {
                // window columns bx+1 .. bx+6 of the staged box; the own pixels are two aligned double2
                const double *row = &sm.u[(by + j) * KT_WIN_W + bx];
                const double2 a1 = *reinterpret_cast<const double2 *>(row + 2);
                const double2 a2 = *reinterpret_cast<const double2 *>(row + 4);
                uc[j][1] = a1.x; uc[j][2] = a1.y; uc[j][3] = a2.x; uc[j][4] = a2.y;
                if (j >= 1 && j <= TH) {
                    uc[j][0] = row[1];
                    uc[j][5] = row[6];
                } else {
                    uc[j][0] = uc[j][5] = 0.0;  // corners are not part of the 5-point stencil
                }
            }
#pragma unroll
            for (int j = 0; j < TH; ++j) {
                const int gy = gy0 + j;
                const double cy = 4.0 - (gy == 0 ? 1.0 : 0.0) - (gy == H - 1 ? 1.0 : 0.0);
                double bt[TW];
                if (!RM) {
                    const double2 *brow = reinterpret_cast<const double2 *>(&sm.b[(by + j) * BW + bx]);
                    const double2 b0 = brow[0], b1 = brow[1];
                    bt[0] = b0.x; bt[1] = b0.y; bt[2] = b1.x; bt[3] = b1.y;
                }
#pragma unroll
                for (int i = 0; i < TW; ++i) {
                    const int gx = gx0 + i;
                    const bool m = (mbits >> (j * TW + i)) & 1u;
                    const double cnt = cy - (gx == 0 ? 1.0 : 0.0) - (gx == W - 1 ? 1.0 : 0.0);
                    const double s = ((uc[j][i + 1] + uc[j + 2][i + 1]) + uc[j + 1][i]) + uc[j + 1][i + 2];
                    const double au = s * (-hinv2) + (cnt * hinv2) * uc[j + 1][i + 1];
                    double bb;
                    if (RM) {
                        // rhs = where(mask, known, 0); at mask pixels b - u is exactly 0 unless `general`
                        bb = 0.0;
                        if (general && m) bb = S.b[(size_t)p * S.plane + (size_t)gy * W + gx];
                        r[j][i] = m ? (general ? bb - uc[j + 1][i + 1] : 0.0) : (bb - au);
                    } else {
                        bb = bt[i];
                        r[j][i] = m ? (bb - uc[j + 1][i + 1]) : (bb - au);
                    }
                }
            }
        }
        // every thread has read the staged tiles: thread 0 re-arms the barrier and requests the next
        // item's window, which lands while this block iterates; it also makes sure the previous
        // bulk store has finished reading sm.out (ordered before the epilogue by the barriers below)
        cg.group_bar();
        if (tid == 0) {
            bulk_wait_read();
            if (nxt < total) request(nxt);
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
            double inv_rs = 1.0 / rs_k;
            for (int it = 0; it < S.max_iters; ++it) {
                cg.apply(pc, q);
                double d_pq = tile_dot<TW, TH>(pc, q);
                double d_rq = tile_dot<TW, TH>(r, q);
                double d_qq = tile_dot<TW, TH>(q, q);
                cg.group_sum3(d_pq, d_rq, d_qq);
                const double pq = hinv2 * d_pq;
                const bool ok = pq > 0.0;                 // solvers.py:348
                const double a = ok ? rs_k / pq : 0.0;    // :349-350
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
                inv_rs = 1.0 / rs_k;
#pragma unroll
                for (int j = 0; j < TH; ++j)
#pragma unroll
                    for (int i = 0; i < TW; ++i) pc[j][i] = fma(beta, pc[j][i], r[j][i]);
            }
        }

        // ---- weighted correction (v * wy) * wx (solvers.py:309-310) -> sm.out -> one bulk store
        {
            double wxv[TW];
#pragma unroll
            for (int i = 0; i < TW; ++i) wxv[i] = L.wx[ix * BW + bx + i];
#pragma unroll
            for (int j = 0; j < TH; ++j) {
                const double wyv = L.wy[iy * BH + by + j];
                double2 o0, o1;
                o0.x = (v[j][0] * wyv) * wxv[0];
                o0.y = (v[j][1] * wyv) * wxv[1];
                o1.x = (v[j][2] * wyv) * wxv[2];
                o1.y = (v[j][3] * wyv) * wxv[3];
                double2 *row = reinterpret_cast<double2 *>(&sm.out[(by + j) * BW + bx]);
                row[0] = o0;
                row[1] = o1;
            }
        }
        fence_async_smem();  // generic-proxy writes -> visible to the bulk copy (async proxy)
        cg.group_bar();
        if (tid == 0)
            bulk_store(S.scratch + ((size_t)p * nblocks + blk) * (BW * BH), s_out, BW * BH * 8);

        if (nxt >= total) break;
        item = nxt;
    }
    if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // last store complete
}

}  // namespace b200p
