// kernels_oras.cuh -- the ORAS block smoother (the hot kernel of the path).
//
//   K2   oras_sweep_tile_kernel<TW,TH,NWARP>  register-tiled local Robin CG, one
//        warp group per overlapping block; all CG state lives in registers,
//        neighbour exchange by warp shuffles, reductions by shuffle butterflies
//        (solvers.py:303-305 gather, :328-370 _solve_range, :307-314 scatter weights)
//   K2g  oras_sweep_generic_kernel            any block extent <= 64x64, shared-memory
//        CG with one CTA per block (same semantics; partial / odd-sized blocks)
//   K2b  oras_combine_kernel                  u += sum over covering blocks of the
//        weighted corrections, in block order (np.bincount order, solvers.py:310-314)
//   K7   coarse_solve_kernel                  _smooth_to_tol on a single-block level,
//        sweeps looped in-kernel (multigrid.py:282-332, :362-364, :397-401)
//
// One sweep = K1 (||r||^2, kernels_stencil.cuh) -> K2 -> K2b.  K2 recomputes the
// global residual of its block from u (1-pixel halo) instead of reading a
// materialised residual field.
#pragma once
#include "common.cuh"

namespace b200p {

#ifndef B200P_COMBINE_THREADS
#define B200P_COMBINE_THREADS 128
#endif
constexpr int ST_THREADS_COMBINE = B200P_COMBINE_THREADS;

#ifndef B200P_PACKED_RED
#define B200P_PACKED_RED 1
#endif

struct SweepArgs {
    LevelDev L;
    const double *u;       // (P, h, w) current iterate
    const double *b;       // (P, h, w) right-hand side
    const uint8_t *mask;   // (F, h, w)
    int channels;
    size_t plane;
    const int *pred;       // per-problem active flag or null
    const double *rs;      // (P) global ||r||^2 from K1
    const int *mflag;      // (P) residual non-zero at some mask pixel
    double eta;            // local_tol_fraction
    int max_iters;         // local CG cap
    double *scratch;       // (P, nblocks, bh, bw) weighted corrections
    int iy0 = 0;           // first block row of this launch (strip mode; default 0)
    int u_zero = 0;        // the iterate is identically 0 and must not be read (a V-cycle correction before its
                           // first sweep, multigrid.py:361): the warp-per-block kernel and the combine honour it
};

// ------------------------------------------------------------------ K2 ----
// Block = (8*TW) x (4*TH*NWARP) pixels, handled by a group of NWARP warps.
// Lane (lx = lane&7, ly = lane>>3) of group warp wg owns the TW x TH tile at
// (lx*TW, (wg*4+ly)*TH).  The local operator is applied in the scaled form
//     q' = A_i p / hinv2 = 4 p - (sum of 4 neighbours incl. ghosts),
// where a neighbour cut off by a block side is replaced by the ghost
// gamma * p_edge: gamma = 1 on the image border (reflecting, diag count 3) and
// gamma = 1 - alpha*h on an inner side (Robin: diag 3 + alpha*h, solvers.py:206-216,
// :288-297).  Mask pixels are identity rows; p and r stay exactly 0 there.
// A CTA may hold several groups (one block each); groups synchronise on their
// own named barrier (id 1 + group), never on the CTA barrier.
template <int TW, int TH, int NWARP>
struct TileCG {
    static constexpr int BW = 8 * TW, BH = 4 * TH * NWARP;
    int lane, wg, lx, ly, bar_id;
    bool eL, eR, eT, eB;     // tile touches the block's left/right/top/bottom side
    double gL, gR, gT, gB;   // ghost factors of those sides
    unsigned mbits;          // local mask, bit j*TW+i
    double *xrow;            // smem: NWARP*2*BW doubles (cross-warp boundary rows)
    double *red;             // smem: 2*NWARP*3 doubles (two alternating slots of up to 3 values)
    int slot;

    __device__ __forceinline__ void group_bar() {
        if (NWARP > 1) asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(NWARP * 32) : "memory");
    }

    __device__ __forceinline__ double group_sum(double v) {
        v = warp_sum(v);
        if (NWARP == 1) return v;
        double *s = red + slot * NWARP * 3;
        if (lane == 0) s[wg] = v;
        group_bar();
        double t = 0.0;
#pragma unroll
        for (int k = 0; k < NWARP; ++k) t += s[k];
        slot ^= 1;
        return t;
    }

    // Three sums in ONE butterfly / one cross-warp exchange (a single latency chain).
    __device__ __forceinline__ void group_sum3(double &a, double &b, double &c) {
#if B200P_PACKED_RED
        // Packed butterfly: shuffles go through the LSU data pipe, which this kernel loads
        // heavily (ncu: l1tex__data_pipe_lsu_wavefronts), so the three sums share one
        // butterfly instead of running three.  Stage 16 folds a and b into one register
        // (lower half-warp keeps a, upper keeps b), stage 8 folds c in (lanes with bit 3 keep
        // c), stages 4,2,1 finish: 6 exchanges instead of 15.  Lane 0 ends with a, lane 16 with
        // b, lane 8 with c; summation order is fixed, results are deterministic.
        {
            const bool hi = lane & 16;
            const double send = hi ? a : b;
            double keep = hi ? b : a;
            keep += __shfl_xor_sync(FULL_MASK, send, 16);
            c += __shfl_xor_sync(FULL_MASK, c, 16);
            const bool h8 = lane & 8;
            const double send2 = h8 ? keep : c;
            double w = h8 ? c : keep;
            w += __shfl_xor_sync(FULL_MASK, send2, 8);
            w += __shfl_xor_sync(FULL_MASK, w, 4);
            w += __shfl_xor_sync(FULL_MASK, w, 2);
            w += __shfl_xor_sync(FULL_MASK, w, 1);
            if (NWARP == 1) {
                a = __shfl_sync(FULL_MASK, w, 0);
                b = __shfl_sync(FULL_MASK, w, 16);
                c = __shfl_sync(FULL_MASK, w, 8);
                return;
            }
            if ((lane & 7) == 0 && lane < 24)
                red[slot * NWARP * 3 + wg * 3 + (lane == 0 ? 0 : (lane == 16 ? 1 : 2))] = w;
        }
        double *s = red + slot * NWARP * 3;
#else
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            a += __shfl_xor_sync(FULL_MASK, a, o);
            b += __shfl_xor_sync(FULL_MASK, b, o);
            c += __shfl_xor_sync(FULL_MASK, c, o);
        }
        if (NWARP == 1) return;
        double *s = red + slot * NWARP * 3;
        if (lane == 0) {
            s[wg * 3 + 0] = a;
            s[wg * 3 + 1] = b;
            s[wg * 3 + 2] = c;
        }
#endif
        group_bar();
        a = b = c = 0.0;
#pragma unroll
        for (int k = 0; k < NWARP; ++k) {
            a += s[k * 3 + 0];
            b += s[k * 3 + 1];
            c += s[k * 3 + 2];
        }
        slot ^= 1;
    }

    // q' = 4p - neighbours (scaled local operator), 0 at mask pixels.
    __device__ __forceinline__ void apply(const double (&pc)[TH][TW], double (&q)[TH][TW]) {
        double hT[TW], hB[TW];
#pragma unroll
        for (int i = 0; i < TW; ++i) {
            hT[i] = __shfl_up_sync(FULL_MASK, pc[TH - 1][i], 8);
            hB[i] = __shfl_down_sync(FULL_MASK, pc[0][i], 8);
        }
        if (NWARP > 1) {
            const int bx = lx * TW;
            if (ly == 0) {
#pragma unroll
                for (int i = 0; i < TW; ++i) xrow[(wg * 2 + 0) * BW + bx + i] = pc[0][i];
            }
            if (ly == 3) {
#pragma unroll
                for (int i = 0; i < TW; ++i) xrow[(wg * 2 + 1) * BW + bx + i] = pc[TH - 1][i];
            }
            group_bar();
            if (ly == 0 && wg > 0) {
#pragma unroll
                for (int i = 0; i < TW; ++i) hT[i] = xrow[((wg - 1) * 2 + 1) * BW + bx + i];
            }
            if (ly == 3 && wg < NWARP - 1) {
#pragma unroll
                for (int i = 0; i < TW; ++i) hB[i] = xrow[((wg + 1) * 2 + 0) * BW + bx + i];
            }
        }
        if (eT) {
#pragma unroll
            for (int i = 0; i < TW; ++i) hT[i] = gT * pc[0][i];
        }
        if (eB) {
#pragma unroll
            for (int i = 0; i < TW; ++i) hB[i] = gB * pc[TH - 1][i];
        }
#pragma unroll
        for (int j = 0; j < TH; ++j) {
            double hl = __shfl_up_sync(FULL_MASK, pc[j][TW - 1], 1);
            double hr = __shfl_down_sync(FULL_MASK, pc[j][0], 1);
            if (eL) hl = gL * pc[j][0];
            if (eR) hr = gR * pc[j][TW - 1];
#pragma unroll
            for (int i = 0; i < TW; ++i) {
                const double up = j == 0 ? hT[i] : pc[j - 1][i];
                const double dn = j == TH - 1 ? hB[i] : pc[j + 1][i];
                const double lf = i == 0 ? hl : pc[j][i - 1];
                const double rt = i == TW - 1 ? hr : pc[j][i + 1];
                const double s = ((up + dn) + lf) + rt;
                const double qq = fma(4.0, pc[j][i], -s);
                q[j][i] = ((mbits >> (j * TW + i)) & 1u) ? 0.0 : qq;
            }
        }
    }
};

template <int TW, int TH, int NWARP>
struct TileSmem {
    double xrow[NWARP > 1 ? NWARP * 2 * 8 * TW : 1];
    double red[2 * NWARP * 3];
};

// One block's sweep work for the NWARP warps of group `grp`: gather the global
// residual from u (1-pixel halo), run the local Robin CG to eta*rs, and store
// the PoU-weighted correction (v*wy)*wx as a (BH,BW) tile at `out`
// (solvers.py:303-305, :328-370, :309-310).  STCG: store with st.global.cg
// (L2 only) -- used when another CTA of the same kernel reads the tile.
// Dot product of two register tiles with four independent accumulation chains (the single
// chain of TH*TW dependent DFMAs was on the critical path of every CG step).
template <int TW, int TH>
__device__ __forceinline__ double tile_dot(const double (&a)[TH][TW], const double (&b)[TH][TW]) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int j = 0; j < TH; ++j)
#pragma unroll
        for (int i = 0; i < TW; ++i) {
            const int k = (j * TW + i) & 3;
            acc[k] = fma(a[j][i], b[j][i], acc[k]);
        }
    return (acc[0] + acc[1]) + (acc[2] + acc[3]);
}

struct NoHook {
    __device__ __forceinline__ void operator()() const {}
};

template <int TW, int TH, int NWARP, bool RM, bool STCG, class PreStore = NoHook>
__device__ __forceinline__ void tile_block_solve(const SweepArgs &A, int p, int blk, int grp, int wg,
                                                 TileSmem<TW, TH, NWARP> &sm, double target,
                                                 double *__restrict__ out, PreStore pre_store = PreStore()) {
    using CG = TileCG<TW, TH, NWARP>;
    constexpr int BW = CG::BW, BH = CG::BH;
    const LevelDev &L = A.L;
    const int iy = blk / L.nx, ix = blk - iy * L.nx;
    const int x0 = L.xs[ix], y0 = L.ys[iy];
    const int W = L.w, H = L.h;

    CG cg;
    cg.lane = threadIdx.x & 31;
    cg.wg = wg;
    cg.bar_id = 1 + grp;
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
        double uc[TH + 2][TW + 2];  // tile + 1-pixel halo, 0 outside the image
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
    double v[TH][TW], pc[TH][TW], q[TH][TW];
#pragma unroll
    for (int j = 0; j < TH; ++j)
#pragma unroll
        for (int i = 0; i < TW; ++i) v[j][i] = 0.0;
    if (A.mflag[p]) {
        // general case (u violates the interpolation condition): mask pixels
        // carry v0 = g, which leaks into their neighbours' rows.
#pragma unroll
        for (int j = 0; j < TH; ++j)
#pragma unroll
            for (int i = 0; i < TW; ++i) {
                const bool m = (mbits >> (j * TW + i)) & 1u;
                v[j][i] = m ? r[j][i] : 0.0;
                pc[j][i] = v[j][i];
            }
        cg.apply(pc, q);  // q' = 4 v0 - nbrs at non-mask pixels, 0 at mask pixels
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
        // CG with ONE reduction per step: (p.q), (r.q) and (q.q) are summed together and the
        // new squared residual follows from the identity |r - a q|^2 = |r|^2 - 2a (r.q) + a^2 (q.q).
        // Same iterates as the textbook recurrence (solvers.py:345-369) up to rounding; the step is
        // latency-bound, so one butterfly + one cross-warp exchange instead of two is what counts.
        double inv_rs = 1.0 / rs_k;  // for beta; off the critical path
        for (int it = 0; it < A.max_iters; ++it) {
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

    // ---- weighted correction (v * wy) * wx (solvers.py:309-310)
    pre_store();  // fused sweep: the ring slot must be free before the tile is written
    double wxv[TW];
#pragma unroll
    for (int i = 0; i < TW; ++i) wxv[i] = L.wx[ix * BW + bx + i];
#pragma unroll
    for (int j = 0; j < TH; ++j) {
        const double wyv = L.wy[iy * BH + by + j];
        double *row = out + (by + j) * BW + bx;
        if (TW % 2 == 0) {
#pragma unroll
            for (int i = 0; i < TW; i += 2) {
                double2 o;
                o.x = (v[j][i] * wyv) * wxv[i];
                o.y = (v[j][i + 1] * wyv) * wxv[i + 1];
                if (STCG) __stcg(reinterpret_cast<double2 *>(row + i), o);
                else *reinterpret_cast<double2 *>(row + i) = o;
            }
        } else {
#pragma unroll
            for (int i = 0; i < TW; ++i) {
                const double o = (v[j][i] * wyv) * wxv[i];
                if (STCG) __stcg(row + i, o); else row[i] = o;
            }
        }
    }
}

// REGCAP: register cap per thread.  The 32x32 tile needs 194 registers uncapped, which the
// allocation granularity (512 per warp) turns into 4 resident blocks per SM; 168 gives 5,
// 160 gives 6 at the price of a few spilled words.
template <int TW, int TH, int NWARP, bool RM, int REGCAP = 255>
__global__ void __launch_bounds__(NWARP * 32) __maxnreg__(REGCAP)
oras_sweep_tile_kernel(const SweepArgs A) {
    __shared__ TileSmem<TW, TH, NWARP> sm;
    const int p = blockIdx.y;
    if (A.pred && !A.pred[p]) return;
    const double rs_g = A.rs[p];
    if (rs_g == 0.0) return;  // oras_sweeps exit, solvers.py:420
    const int blk = blockIdx.x;
    double *out = A.scratch + ((size_t)p * A.L.nblocks + blk) * (8 * TW * 4 * TH * NWARP);
    tile_block_solve<TW, TH, NWARP, RM, false>(A, p, blk, 0, threadIdx.x >> 5, sm, A.eta * rs_g, out);
}

// ------------------------------------------------------------------ K2g ---
// Shared-memory layout of the generic per-block CG (n = bw*bh):
//   P  (bh+2)*(bw+2)  search direction with a zero ring (cut neighbours read 0)
//   R, V, Q  n each (G aliases R: r0 = g - A v0 is formed in place);
//   M n bytes; red 34 doubles.
struct SmemCG {
    double *P, *R, *V, *Q, *G, *red;
    uint8_t *M;
    int bw, bh, n, pw;  // pw = bw + 2
    __device__ __forceinline__ double &p_at(int k) { return P[(k / bw + 1) * pw + (k % bw) + 1]; }
};

__host__ __device__ inline size_t smem_cg_bytes(int bw, int bh) {
    const size_t n = (size_t)bw * bh;
    return sizeof(double) * ((size_t)(bw + 2) * (bh + 2) + 3 * n + 34) + ((n + 15) / 16) * 16;
}

__device__ __forceinline__ SmemCG smem_cg_carve(unsigned char *base, int bw, int bh) {
    SmemCG S;
    S.bw = bw; S.bh = bh; S.n = bw * bh; S.pw = bw + 2;
    double *d = reinterpret_cast<double *>(base);
    S.P = d; d += (size_t)(bw + 2) * (bh + 2);
    S.R = d; d += S.n;
    S.G = S.R;
    S.V = d; d += S.n;
    S.Q = d; d += S.n;
    S.red = d; d += 34;
    S.M = reinterpret_cast<uint8_t *>(d);
    return S;
}

// LocalSystem.apply / BlockSolver._apply at local pixel k (solvers.py:221-229,
// :316-326): diag*v - hinv2*s with diag = cnt*hinv2 (+ robin per inner side in
// the order left, right, top, bottom, :288-297); identity at mask pixels.
__device__ __forceinline__ double smem_apply_at(SmemCG &S, int k, double hinv2, double robin,
                                                bool inL, bool inR, bool inT, bool inB) {
    const int j = k / S.bw, i = k - j * S.bw;
    const double *c = &S.P[(j + 1) * S.pw + i + 1];
    const double pv = c[0];
    if (S.M[k]) return pv;
    double cnt = 4.0;
    if (j == 0) cnt -= 1.0;
    if (j == S.bh - 1) cnt -= 1.0;
    if (i == 0) cnt -= 1.0;
    if (i == S.bw - 1) cnt -= 1.0;
    double diag = cnt * hinv2;
    if (inL && i == 0) diag += robin;
    if (inR && i == S.bw - 1) diag += robin;
    if (inT && j == 0) diag += robin;
    if (inB && j == S.bh - 1) diag += robin;
    const double s = ((c[-S.pw] + c[S.pw]) + c[-1]) + c[1];
    return diag * pv - hinv2 * s;
}

// _solve_range for one block on shared memory (solvers.py:328-370).  Expects
// S.G (gathered residual) and S.M filled and the P ring zeroed; leaves the
// local correction in S.V.  Returns the CG steps taken.
__device__ int smem_block_cg(SmemCG &S, double hinv2, double robin, bool inL, bool inR, bool inT,
                             bool inB, double target, int max_iters) {
    const int T = blockDim.x, tid = threadIdx.x;
    for (int k = tid; k < S.n; k += T) {
        const double v0 = S.M[k] ? S.G[k] : 0.0;
        S.V[k] = v0;
        S.p_at(k) = v0;
    }
    __syncthreads();
    double part = 0.0;
    for (int k = tid; k < S.n; k += T) {
        const double r0 = S.G[k] - smem_apply_at(S, k, hinv2, robin, inL, inR, inT, inB);
        S.R[k] = r0;
        part += r0 * r0;
    }
    double rs = cta_sum(part, S.red);  // (contains the barrier that orders P reads/writes)
    if (!(rs > target)) return 0;
    for (int k = tid; k < S.n; k += T) S.p_at(k) = S.R[k];
    __syncthreads();
    int steps = 0;
    for (int it = 0; it < max_iters; ++it) {
        part = 0.0;
        for (int k = tid; k < S.n; k += T) {
            const double q = smem_apply_at(S, k, hinv2, robin, inL, inR, inT, inB);
            S.Q[k] = q;
            part += S.p_at(k) * q;
        }
        const double pq = cta_sum(part, S.red);
        const bool ok = pq > 0.0;
        const double a = ok ? rs / pq : 0.0;
        part = 0.0;
        for (int k = tid; k < S.n; k += T) {
            S.V[k] += a * S.p_at(k);
            const double rr = S.R[k] - a * S.Q[k];
            S.R[k] = rr;
            part += rr * rr;
        }
        const double rs_new = cta_sum(part, S.red);
        ++steps;
        if (rs_new <= target || !ok) break;
        const double beta = rs_new / rs;
        rs = rs_new;
        for (int k = tid; k < S.n; k += T) S.p_at(k) = beta * S.p_at(k) + S.R[k];
        __syncthreads();
    }
    return steps;
}

constexpr int GEN_THREADS = 256;

// MODE 0: sweep  -- gather from u, solve, write weighted corrections to scratch
// MODE 1: blocks -- gather from a given residual field (A.u), explicit target
//                   (A.eta holds target_sq), write UNWEIGHTED v (solve_blocks)
template <bool RM, int MODE>
__global__ void __launch_bounds__(GEN_THREADS)
oras_sweep_generic_kernel(const SweepArgs A) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int p = blockIdx.y;
    if (A.pred && !A.pred[p]) return;
    double target;
    if (MODE == 0) {
        const double rs_g = A.rs[p];
        if (rs_g == 0.0) return;
        target = A.eta * rs_g;
    } else {
        target = A.eta;
    }
    const LevelDev &L = A.L;
    const int blk = blockIdx.x;
    const int iy = blk / L.nx, ix = blk - iy * L.nx;
    const int x0 = L.xs[ix], y0 = L.ys[iy];
    SmemCG S = smem_cg_carve(smem_raw, L.bw, L.bh);
    const double *up = A.u + (size_t)p * A.plane;
    const double *bp = A.b ? A.b + (size_t)p * A.plane : nullptr;
    const uint8_t *mp = A.mask + (size_t)(p / A.channels) * A.plane;
    for (int k = threadIdx.x; k < (S.bw + 2) * (S.bh + 2); k += GEN_THREADS) S.P[k] = 0.0;
    for (int k = threadIdx.x; k < S.n; k += GEN_THREADS) {
        const int j = k / S.bw, i = k - j * S.bw;
        const int gy = y0 + j, gx = x0 + i;
        const size_t gi = (size_t)gy * L.w + gx;
        S.M[k] = mp[gi] != 0;
        S.G[k] = MODE == 0 ? residual_px<false, RM>(up, bp, mp, gy, gx, L.h, L.w, L.hinv2) : up[gi];
    }
    __syncthreads();
    smem_block_cg(S, L.hinv2, L.robin, x0 > 0, x0 + L.bw < L.w, y0 > 0, y0 + L.bh < L.h, target,
                  A.max_iters);
    __syncthreads();
    double *sp = A.scratch + ((size_t)p * L.nblocks + blk) * S.n;
    for (int k = threadIdx.x; k < S.n; k += GEN_THREADS) {
        const int j = k / S.bw, i = k - j * S.bw;
        sp[k] = MODE == 0 ? (S.V[k] * L.wy[iy * L.bh + j]) * L.wx[ix * L.bw + i] : S.V[k];
    }
}

// ------------------------------------------------------------------ K2b ---
// u += sum_b w_b v_b over the blocks covering each pixel, accumulated from 0 in
// ascending block index (iy outer, ix inner) like np.bincount does, then added
// to u (solvers.py:310-314, :423).  Grid (ceil(w/256), ceil(h/COMBINE_ROWS), P):
// a thread owns one column of a COMBINE_ROWS-row chunk.  The covering block rows
// of each pixel row (uniform over the chunk) are staged in shared memory, the
// covering block columns are per-thread constants, and the (up to) four tile
// reads per pixel are issued branch-free, COMBINE_G rows at a time, so that
// ~40 independent loads per thread are in flight (HBM-bound streaming pass).
// K2b tuning (A/B builds): rows in flight per thread, resident CTAs per SM the register budget is cut for, rows
// per CTA (B200P_COMBINE_THREADS: threads per CTA).  4 rows, 80 registers without spills, 768 threads per SM as
// 6 CTAs of 128: 5.36 ms per 8-frame step (3 CTAs of 256: 5.48; 12 of 64: 5.34; 7 of 128 at 72 registers: 5.52); 8 rows in
// flight at the compiler's own 128 registers (2 CTAs) 5.8, 4 at 114 registers 6.6, 3 at 64 registers 6.5, 5 at 80
// (spills) 5.9, 16 at 242 registers 8.1
#ifndef B200P_COMBINE_G
#define B200P_COMBINE_G 4
#endif
#ifndef B200P_COMBINE_MINB
#define B200P_COMBINE_MINB 6
#endif
#ifndef B200P_COMBINE_ROWS
#define B200P_COMBINE_ROWS 32
#endif
constexpr int COMBINE_ROWS = B200P_COMBINE_ROWS;
constexpr int COMBINE_G = B200P_COMBINE_G;

// Stage helper: tiles[p][blk][j][i] *= wy[iy][j] * wx[ix][i] in the order of K2's epilogue, (v * wy) * wx
// (solvers.py:309-310), so that an isolated combine pass can be fed UNWEIGHTED local corrections.
__global__ void __launch_bounds__(ST_THREADS_COMBINE)
weight_tiles_kernel(const LevelDev L, const double *__restrict__ v, double *__restrict__ tiles, size_t n) {
    const size_t i = (size_t)blockIdx.x * ST_THREADS_COMBINE + threadIdx.x;
    if (i >= n) return;
    const size_t bsz = (size_t)L.bw * L.bh;
    const int blk = (int)((i / bsz) % (size_t)L.nblocks);
    const int r = (int)(i % bsz), jy = r / L.bw, jx = r - jy * L.bw;
    const int iy = blk / L.nx, ix = blk - iy * L.nx;
    tiles[i] = (v[i] * L.wy[iy * L.bh + jy]) * L.wx[ix * L.bw + jx];
}

__global__ void fill_double_kernel(double *p, int n, double v) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

// `egress` (8-bit decode): the updated pixel is also written as clip(round(u)) into
// the interleaved (F, h, w, C) image (image_from_fields, fileio.py:58-65) -- the last post-smoothing
// combine of the finest level carries it, so an 8-bit decode needs no pass over the fp64 result.
__global__ void __launch_bounds__(ST_THREADS_COMBINE, B200P_COMBINE_MINB)
oras_combine_kernel(const LevelDev L, const double *__restrict__ scratch, size_t plane,
                    const int *__restrict__ pred, const double *__restrict__ rs,
                    double *__restrict__ u, int *__restrict__ unit_counter, int y_lo, int y_hi,
                    uint8_t *__restrict__ egress, int channels, int u_zero = 0) {
    __shared__ int s_rn[COMBINE_ROWS], s_rf[COMBINE_ROWS];
    __shared__ size_t s_roff[COMBINE_ROWS][2];
    const int p = blockIdx.z;
    if (pred && !pred[p]) return;
    if (rs[p] == 0.0) {
        // nothing to correct; an implicitly zero iterate (u_zero) has to become a real zero field now
        if (u_zero) {
            const int x = blockIdx.x * ST_THREADS_COMBINE + threadIdx.x;
            const int ya = y_lo + blockIdx.y * COMBINE_ROWS, yb = min(ya + COMBINE_ROWS, y_hi);
            if (x < L.w)
                for (int y = ya; y < yb; ++y) u[(size_t)p * plane + (size_t)y * L.w + x] = 0.0;
        }
        return;
    }
    const int tid = threadIdx.x;
    const int x = blockIdx.x * ST_THREADS_COMBINE + tid;
    const int y0 = y_lo + blockIdx.y * COMBINE_ROWS;  // rows [y_lo, y_hi): the whole level, or a strip
    const int rows = min(COMBINE_ROWS, y_hi - y0);
    if (unit_counter && blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) unit_counter[p] += 1;
    const size_t bsz = (size_t)L.bw * L.bh;
    if (tid < rows) {
        const int y = y0 + tid;
        const int iyf = L.cyf[y], iyn = L.cyn[y];
        s_rn[tid] = iyn;
        s_rf[tid] = iyf;
        for (int a = 0; a < 2; ++a) {
            const int iy = iyf + (a < iyn ? a : 0);
            s_roff[tid][a] = (size_t)iy * L.nx * bsz + (size_t)(y - L.ys[iy]) * L.bw;
        }
    }
    __syncthreads();
    if (x >= L.w) return;
    const int ixf = L.cxf[x], ixn = L.cxn[x];
    const size_t xo0 = (size_t)ixf * bsz + (x - L.xs[ixf]);
    const size_t xo1 = ixn > 1 ? (size_t)(ixf + 1) * bsz + (x - L.xs[ixf + 1]) : 0;
    const bool two_x = ixn > 1;
    const bool wide = ixn > 2;  // > 2 covering blocks per axis: heavily overlapped layouts
    const double *sp = scratch + (size_t)p * L.nblocks * bsz;
    double *up = u + (size_t)p * plane;
    constexpr int G = COMBINE_G;
    for (int k0 = 0; k0 < rows; k0 += G) {
        double uu[G], v00[G], v01[G], v10[G], v11[G];
#pragma unroll
        for (int j = 0; j < G; ++j) {
            const int k = k0 + j < rows ? k0 + j : rows - 1;
            const size_t o0 = s_roff[k][0], o1 = s_roff[k][1];
            uu[j] = u_zero ? 0.0 : up[(size_t)(y0 + k) * L.w + x];
            v00[j] = sp[o0 + xo0];
            v01[j] = sp[o0 + (two_x ? xo1 : xo0)];
            v10[j] = sp[o1 + xo0];
            v11[j] = sp[o1 + (two_x ? xo1 : xo0)];
        }
#pragma unroll
        for (int j = 0; j < G; ++j) {
            const int k = k0 + j;
            if (k >= rows) break;
            const int n = s_rn[k];
            // ascending block order: (iy0,ix0), (iy0,ix1), (iy1,ix0), (iy1,ix1)
            double acc = v00[j];
            acc += two_x ? v01[j] : 0.0;
            if (wide || n > 2) {
                acc = 0.0;
                for (int a = 0; a < n; ++a) {
                    const int iy = s_rf[k] + a;
                    const size_t oa = (size_t)iy * L.nx * bsz + (size_t)(y0 + k - L.ys[iy]) * L.bw;
                    for (int c = 0; c < ixn; ++c)
                        acc += sp[oa + (size_t)(ixf + c) * bsz + (x - L.xs[ixf + c])];
                }
            } else {
                acc += n > 1 ? v10[j] : 0.0;
                acc += (n > 1 && two_x) ? v11[j] : 0.0;
            }
            const double un = uu[j] + acc;
            up[(size_t)(y0 + k) * L.w + x] = un;
            if (egress) {
                const int f = p / channels, c = p - f * channels;
                egress[((size_t)f * plane + (size_t)(y0 + k) * L.w + x) * channels + c] = quantize_u8(un);
            }
        }
    }
}

// ------------------------------------------------------------------ K7 ----
// _smooth_to_tol / _smooth on a level that is a single block (always true for
// the coarsest level: both extents <= block_size, multigrid.py:249).  One CTA
// per problem keeps u, b and the CG state in shared memory and loops whole ORAS
// sweeps in-kernel:
//   r = b - A u; rs = |r|^2; first pass fixes denom = |r| (0 -> done);
//   stop when rs == 0, |r| <= tol*denom or max_sweeps reached;
//   local solve to eta*rs; u += (v*wy)*wx (single block: weights are 1).
// (multigrid.py:300-322, solvers.py:413-424).  tol == 0 gives _smooth's
// stop_norm = 0 behaviour (fixed sweep count, early exit only on rs == 0).
// init_mode: 0  u = 0 (V-cycle correction e, multigrid.py:361)
//            1  u = b (flat initialisation, multigrid.py:393-394)
//            2  u = stored iterate
struct CoarseArgs {
    LevelDev L;
    double *u;
    const double *b;
    const uint8_t *mask;
    int channels;
    const int *pred;
    double tol;
    int max_sweeps;
    double eta;
    int max_iters;
    int rhs_masked;
    int init_mode;
    int *units_out;       // may be null
    int units_accumulate;
    double *rel_out;      // may be null: final |r| / denom
    double *hist;         // may be null: (P, hist_cap) relative norm of every residual evaluation
    int *histlen;         //   (single-level multilevel solve: the on_fine_state history)
    int hist_cap;
};

__global__ void __launch_bounds__(GEN_THREADS)
coarse_solve_kernel(const CoarseArgs A) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int p = blockIdx.x;
    if (A.pred && !A.pred[p]) return;
    const LevelDev &L = A.L;
    SmemCG S = smem_cg_carve(smem_raw, L.bw, L.bh);
    // U and B live behind the CG arrays
    double *U = reinterpret_cast<double *>(smem_raw + smem_cg_bytes(L.bw, L.bh));
    double *B = U + S.n;
    const size_t plane = (size_t)L.h * L.w;
    double *up = A.u + (size_t)p * plane;
    const double *bp = A.b + (size_t)p * plane;
    const uint8_t *mp = A.mask + (size_t)(p / A.channels) * plane;
    const int T = GEN_THREADS, tid = threadIdx.x;
    for (int k = tid; k < (S.bw + 2) * (S.bh + 2); k += T) S.P[k] = 0.0;
    for (int k = tid; k < S.n; k += T) {
        const bool m = mp[k] != 0;
        S.M[k] = m;
        const double bb = A.rhs_masked ? (m ? bp[k] : 0.0) : bp[k];
        B[k] = bb;
        U[k] = A.init_mode == 0 ? 0.0 : (A.init_mode == 1 ? bb : up[k]);
    }
    __syncthreads();
    const double hinv2 = L.hinv2;
    const int w = L.w, h = L.h;
    double stop = 0.0, denom = 0.0, rn = 0.0;
    int sweeps = 0;
    for (;;) {
        double part = 0.0;
        for (int k = tid; k < S.n; k += T) {
            const int y = k / w, x = k - y * w;
            double g;
            if (S.M[k]) {
                g = B[k] - U[k];
            } else {
                double s = 0.0, cnt = 4.0;
                if (y > 0) s += U[k - w]; else cnt -= 1.0;
                if (y < h - 1) s += U[k + w]; else cnt -= 1.0;
                if (x > 0) s += U[k - 1]; else cnt -= 1.0;
                if (x < w - 1) s += U[k + 1]; else cnt -= 1.0;
                g = B[k] - (s * (-hinv2) + (cnt * hinv2) * U[k]);
            }
            S.G[k] = g;
            part += g * g;
        }
        const double rs = cta_sum(part, S.red);
        rn = sqrt(rs);
        if (sweeps == 0) {
            denom = rn;
            if (rn == 0.0) break;  // denom == 0 -> (0, 0.0), multigrid.py:302-303
            stop = A.tol * rn;
        }
        if (A.hist && tid == 0) {
            if (sweeps < A.hist_cap) A.hist[(size_t)p * A.hist_cap + sweeps] = rn / denom;
            A.histlen[p] = sweeps + 1;
        }
        if (rs == 0.0 || rn <= stop || sweeps >= A.max_sweeps) break;
        smem_block_cg(S, hinv2, L.robin, false, false, false, false, A.eta * rs, A.max_iters);
        __syncthreads();
        for (int k = tid; k < S.n; k += T) {
            const int y = k / w, x = k - y * w;
            U[k] += (S.V[k] * L.wy[y]) * L.wx[x];
        }
        __syncthreads();
        ++sweeps;
    }
    for (int k = tid; k < S.n; k += T) up[k] = U[k];
    if (tid == 0) {
        if (A.units_out) A.units_out[p] = A.units_accumulate ? A.units_out[p] + sweeps : sweeps;
        if (A.rel_out) A.rel_out[p] = denom == 0.0 ? 0.0 : rn / denom;
    }
}

}  // namespace b200p
