// kernels_oras_warp.cuh -- K2W: the 32x32 ORAS block solve with ONE WARP per block and the
// write-mostly part of the CG state in TENSOR MEMORY.
//
// Why (measured on a B200, scripts/probe/fp64_probe.cu, tmem_probe.cu, profiles/oras_sweep_lean_r1.txt):
//   * DFMA/DADD issue once per 2.03 cycles per SM sub-partition; a 64-bit shuffle is two SHFL
//     instructions on a pipe that accepts ONE warp instruction per cycle per SM (shared with LDS/STS).
//     The two-warp register tile of K2L (4x4 pixels per thread) needs ~150 of those per block CG step
//     (halo exchange, two butterflies' worth of reduction, the cross-warp row pair and bar.sync)
//     against ~200 SM cycles of FP64 issue: both pipes sit at 40-50 % because a block's warps spend
//     most of a step in dependent exchange / reduction chains and only 12 warps fit per SM.
//   * A warp that owns the whole block (8x4 pixels per thread) halves the halo per pixel, needs no
//     cross-warp exchange, no bar.sync, no shared memory in the CG loop and one butterfly per 1024
//     pixels: ~66 SHFL per block step.  Its state (v, r, p, q = 4 x 32 doubles per thread) does not
//     fit 255 registers, so the iterate v -- touched once per CG step, never exchanged -- lives in
//     tensor memory: a thread's 32 doubles are 64 TMEM columns of its own lane, moved with
//     tcgen05.ld / tcgen05.st .32x32b (measured ~200 B/clk/SM each way next to the LSU pipe, which
//     they do not use).  QT additionally parks q = A_i p there between the dot products and the
//     residual update.
//
// A CTA is KW_WARPS independent warps (TMEM lane quarter = warp index) that walk the
// (problem, block) items of the launch persistently; TMEM is allocated once per CTA.
// Semantics are those of tile_block_solve / oras_sweep_lean_kernel (solvers.py:303-305 gather,
// :328-370 _solve_range, :309-310 scatter weights); the weighted tile goes to the same scratch
// layout, K2b is unchanged.
// Requires: block 32x32, even level width, even block starts, 16-byte aligned u / b.
#pragma once
#include "kernels_oras.cuh"

namespace b200p {

#ifndef B200P_KW_PREDFMA
#define B200P_KW_PREDFMA 1    // mask pixels: stencil FMA under a predicate on a zeroed register (else FMA + predicated zero)
#endif
#ifndef B200P_KW_WARPS
#define B200P_KW_WARPS 4      // independent warps (= blocks in flight) per CTA
#endif
#ifndef B200P_KW_MAXREG
#define B200P_KW_MAXREG 255   // 2 CTAs x 4 warps x 256 registers = the register file of an SM
#endif
constexpr int KW_WARPS = B200P_KW_WARPS;
constexpr int KW_THREADS = KW_WARPS * 32;

struct WarpSweepArgs {
    SweepArgs S;
    const unsigned *mtab;  // (F, nblocks, 32): bit j*8+i of word `lane` = mask of that lane's pixel (i, j)
    int nrows;             // block rows of this launch (strip mode: S.iy0 .. S.iy0 + nrows)
    int items_per_problem; // nrows * nx
    int total;             // P * items_per_problem (upper bound; the kernel walks live problems only)
    int P;                 // problems (frames x channels)
    unsigned *claim;       // [0] next unclaimed item, [1] CTAs that have finished; both 0 between launches
    unsigned m_ipp, k_ipp; // n / items_per_problem == (n * m) >> k for n < 2^30 (kw_magic)
    unsigned m_nx, k_nx;   // the same for n / nx
    unsigned chunk;        // consecutive items per claim (1 on small launches, KW_CHUNK_MAX on large ones)
    // DIRECT (band combine, see oras_combine_band_kernel): pixels that exactly one block updates are written
    // to the partner iterate u_out = u + v by this kernel; only the overlap bands go through tiles
    double *u_out;         // (P, h, w) partner buffer of S.u
    const uint8_t *xflag;  // (nx, 32) per block column: bit 0 = non-zero weight, bit 1 = column of a single-writer 4-group
    const uint8_t *yflag;  // (ny, 32) per block row:    bit 0 = non-zero weight, bit 1 = single-writer row
};

// Band-combine tile layout: rows of KW_TP doubles, pixel x of a block starting at x0 sits in column
// x - (x0 & ~7), so that the 64-byte pixel groups of the level (the DRAM access granularity) stay aligned
// 64-byte pieces inside the tile.
constexpr int KW_TP = 40;
constexpr int KW_ALIGN = 8;   // pixels per aligned group (64 bytes)
constexpr int KW_TSZ = 32 * KW_TP;

// Division by a launch constant as one wide multiply and a shift: k = 31 + floor(log2 d),
// m = ceil(2^k / d) <= 2^31; exact for n < 2^30 (n * (m d - 2^k) < n d < 2^k).
inline void kw_magic(unsigned d, unsigned &m, unsigned &k) {
    unsigned fl = 0;
    while ((2u << fl) <= d) ++fl;
    k = 31 + fl;
    m = (unsigned)((((unsigned long long)1 << k) + d - 1) / d);
}
__device__ __forceinline__ unsigned kw_div(unsigned n, unsigned m, unsigned k) {
    return (unsigned)(((unsigned long long)n * m) >> k);
}

// Packs the block-local masks for K2W: grid (ceil(nblocks / 4), F), 128 threads, a warp per block.
// A lane's 8 mask bytes of a row are fetched with the widest loads their address allows (block starts are even:
// 16-bit pieces at worst; one 8-byte load where the start is a multiple of 8) and squeezed to 8 bits by a multiply.
__device__ __forceinline__ unsigned long long kw_load8(const uint8_t *p) {
    const unsigned a = (unsigned)(uintptr_t)p & 7u;   // warp-uniform for a given row
    if (a == 0) return *reinterpret_cast<const unsigned long long *>(p);
    if ((a & 3u) == 0) {
        const uint2 v = make_uint2(*reinterpret_cast<const unsigned *>(p), *reinterpret_cast<const unsigned *>(p + 4));
        return ((unsigned long long)v.y << 32) | v.x;
    }
    unsigned long long r = 0;
    if ((a & 1u) == 0) {
#pragma unroll
        for (int k = 0; k < 4; ++k) r |= (unsigned long long)*reinterpret_cast<const unsigned short *>(p + 2 * k) << (16 * k);
    } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) r |= (unsigned long long)p[k] << (8 * k);
    }
    return r;
}
__global__ void __launch_bounds__(KW_THREADS)
pack_block_masks_warp_kernel(const LevelDev L, const uint8_t *__restrict__ mask, size_t plane,
                             unsigned *__restrict__ mtab) {
    const int blk = blockIdx.x * KW_WARPS + (threadIdx.x >> 5), f = blockIdx.y, lane = threadIdx.x & 31;
    if (blk >= L.nblocks) return;
    const int iy = blk / L.nx, ix = blk - iy * L.nx;
    const int gx0 = L.xs[ix] + (lane & 3) * 8, gy0 = L.ys[iy] + (lane >> 2) * 4;
    const uint8_t *mp = mask + (size_t)f * plane;
    unsigned bits = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        unsigned long long v = kw_load8(mp + (size_t)(gy0 + j) * L.w + gx0);
        v |= v >> 4;                          // every byte -> 0 / 1 ...
        v |= v >> 2;
        v |= v >> 1;
        v &= 0x0101010101010101ull;
        bits |= (unsigned)((v * 0x0102040810204080ull) >> 56) << (j * 8);   // ... -> bit i = byte i
    }
    mtab[((size_t)f * L.nblocks + blk) * 32 + lane] = bits;
}

// ---- tensor memory as a per-thread scratch: 8 doubles = 16 columns of the thread's own lane
__device__ __forceinline__ void tm_st8(uint32_t taddr, const double (&d)[8]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
        ::"r"(taddr),
        "r"(__double2loint(d[0])), "r"(__double2hiint(d[0])), "r"(__double2loint(d[1])), "r"(__double2hiint(d[1])),
        "r"(__double2loint(d[2])), "r"(__double2hiint(d[2])), "r"(__double2loint(d[3])), "r"(__double2hiint(d[3])),
        "r"(__double2loint(d[4])), "r"(__double2hiint(d[4])), "r"(__double2loint(d[5])), "r"(__double2hiint(d[5])),
        "r"(__double2loint(d[6])), "r"(__double2hiint(d[6])), "r"(__double2loint(d[7])), "r"(__double2hiint(d[7])));
}
struct TmRow {
    int w[16];
    __device__ __forceinline__ double get(int i) const { return __hiloint2double(w[2 * i + 1], w[2 * i]); }
};
__device__ __forceinline__ void tm_ld8(uint32_t taddr, TmRow &t) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(t.w[0]), "=r"(t.w[1]), "=r"(t.w[2]), "=r"(t.w[3]), "=r"(t.w[4]), "=r"(t.w[5]), "=r"(t.w[6]), "=r"(t.w[7]),
          "=r"(t.w[8]), "=r"(t.w[9]), "=r"(t.w[10]), "=r"(t.w[11]), "=r"(t.w[12]), "=r"(t.w[13]), "=r"(t.w[14]),
          "=r"(t.w[15])
        : "r"(taddr));
}
// tcgen05.wait::ld, tied to the registers of the loads it completes so that no consumer can be
// scheduled above it.
__device__ __forceinline__ void tm_wait_ld(TmRow &t) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(t.w[0]), "+r"(t.w[1]), "+r"(t.w[2]), "+r"(t.w[3]), "+r"(t.w[4]), "+r"(t.w[5]), "+r"(t.w[6]),
                   "+r"(t.w[7]), "+r"(t.w[8]), "+r"(t.w[9]), "+r"(t.w[10]), "+r"(t.w[11]), "+r"(t.w[12]),
                   "+r"(t.w[13]), "+r"(t.w[14]), "+r"(t.w[15]));
}
__device__ __forceinline__ void tm_wait_ld2(TmRow &a, TmRow &b) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(a.w[0]), "+r"(a.w[1]), "+r"(a.w[2]), "+r"(a.w[3]), "+r"(a.w[4]), "+r"(a.w[5]), "+r"(a.w[6]),
                   "+r"(a.w[7]), "+r"(a.w[8]), "+r"(a.w[9]), "+r"(a.w[10]), "+r"(a.w[11]), "+r"(a.w[12]),
                   "+r"(a.w[13]), "+r"(a.w[14]), "+r"(a.w[15]), "+r"(b.w[0]), "+r"(b.w[1]), "+r"(b.w[2]),
                   "+r"(b.w[3]), "+r"(b.w[4]), "+r"(b.w[5]), "+r"(b.w[6]), "+r"(b.w[7]), "+r"(b.w[8]), "+r"(b.w[9]),
                   "+r"(b.w[10]), "+r"(b.w[11]), "+r"(b.w[12]), "+r"(b.w[13]), "+r"(b.w[14]), "+r"(b.w[15]));
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// q = (mbits bit K) ? 0 : c * p - s: the bit test feeds a predicate, the stencil FMA runs under it
// on a zeroed destination (no select; the 32 bit tests of a tile become a handful of R2P).
template <int K>
__device__ __forceinline__ double stencil_q(double c, double p, double s, unsigned mbits) {
    double q;
#if B200P_KW_PREDFMA
    asm("{\n\t.reg .pred z;\n\t.reg .b32 t;\n\t.reg .f64 ns;\n\tand.b32 t, %4, %5;\n\tsetp.ne.u32 z, t, 0;\n\t"
        "neg.f64 ns, %3;\n\tmov.f64 %0, 0d0000000000000000;\n\t@!z fma.rn.f64 %0, %1, %2, ns;\n\t}"
        : "=d"(q)
        : "d"(c), "d"(p), "d"(s), "r"(mbits), "n"(1u << K));
#else
    q = fma(c, p, -s);
    asm("{\n\t.reg .pred z;\n\t.reg .b32 t;\n\tand.b32 t, %1, %2;\n\tsetp.ne.u32 z, t, 0;\n\t"
        "@z mov.f64 %0, 0d0000000000000000;\n\t}"
        : "+d"(q)
        : "r"(mbits), "n"(1u << K));
#endif
    return q;
}

// One warp, 32x32 block, lane (lx = lane & 3, ly = lane >> 2) owns the 8 x 4 pixels at (8 lx, 4 ly).
// Block sides: a neighbour cut off by a side is the ghost gamma * p_edge (gamma = 1 on the image border,
// 1 - alpha h on an inner side, solvers.py:288-297), folded into the centre coefficient of the pixel
// (4 - gamma per cut side); the value the halo shuffle delivers to such a lane is switched off by a
// 0 / 1 factor inside the FMA that adds it, so block sides cost no selects and no extra multiplies.
struct WarpCG {
    static constexpr int TW = 8, TH = 4;
    double zL, zR, zT, zB;  // 0 where the tile touches that block side, else 1 (lane constants)
    double cT, cB;          // centre coefficient of the tile's top / bottom row: 4 - gamma_T|B (4 inside)
    double gLz, gRz;        // gamma of the left / right side where the tile touches it, else 0
    unsigned mbits;

    // q' = c p - in-block neighbours (scaled local Robin operator, solvers.py:316-326), 0 at mask
    // pixels; rows are handed to `sink(j, qrow)` as they are produced.
    template <class Sink>
    __device__ __forceinline__ void apply(const double (&pc)[TH][TW], Sink sink) const {
        double hT[TW], hB[TW];
#pragma unroll
        for (int i = 0; i < TW; ++i) {
            hT[i] = __shfl_up_sync(FULL_MASK, pc[TH - 1][i], 4);
            hB[i] = __shfl_down_sync(FULL_MASK, pc[0][i], 4);
        }
        apply_row<0>(pc, hT, hB, sink);
        apply_row<1>(pc, hT, hB, sink);
        apply_row<2>(pc, hT, hB, sink);
        apply_row<3>(pc, hT, hB, sink);
    }

    template <int J, class Sink>
    __device__ __forceinline__ void apply_row(const double (&pc)[TH][TW], const double (&hT)[TW],
                                              const double (&hB)[TW], Sink &sink) const {
        const double hl = __shfl_up_sync(FULL_MASK, pc[J][TW - 1], 1);
        const double hr = __shfl_down_sync(FULL_MASK, pc[J][0], 1);
        const double cJ = J == 0 ? cT : (J == TH - 1 ? cB : 4.0);
        double qrow[TW];
#define B200P_KW_PX(I)                                                                           \
        {                                                                                        \
            double s;                                                                            \
            if (J == 0) s = fma(hT[I], zT, pc[1][I]);                                            \
            else if (J == TH - 1) s = fma(hB[I], zB, pc[TH - 2][I]);                             \
            else s = pc[J == 0 ? 0 : J - 1][I] + pc[J == TH - 1 ? J : J + 1][I];                 \
            if (I == 0) s = fma(hl, zL, s); else s += pc[J][I == 0 ? 0 : I - 1];                 \
            if (I == TW - 1) s = fma(hr, zR, s); else s += pc[J][I == TW - 1 ? I : I + 1];       \
            if (I == 0) s = fma(gLz, pc[J][0], s);                                               \
            if (I == TW - 1) s = fma(gRz, pc[J][TW - 1], s);                                     \
            qrow[I] = stencil_q<J * TW + I>(cJ, pc[J][I], s, mbits);                             \
        }
        B200P_KW_PX(0) B200P_KW_PX(1) B200P_KW_PX(2) B200P_KW_PX(3)
        B200P_KW_PX(4) B200P_KW_PX(5) B200P_KW_PX(6) B200P_KW_PX(7)
#undef B200P_KW_PX
        sink(J, qrow);
    }
};

// Three warp sums in one packed butterfly (6 exchanges + 3 broadcasts), fixed summation order.
#ifndef B200P_KW_RED
#define B200P_KW_RED 1       // 1: three plain butterflies (5 dependent stages, 15 exchanges; measured 14.49 vs 14.65 ms per step); 0: one packed butterfly (7 stages, 9 exchanges); 2: fan-in 4 (3 stages, 21 exchanges: 14.85)
#endif
__device__ __forceinline__ void warp_sum3(int lane, double &a, double &b, double &c) {
#if B200P_KW_RED == 2
    // fan-in 4: three dependent exchange stages (xor 1 2 3, xor 4 8 12, xor 16) instead of five
#define B200P_KW_S4(V, K1, K2, K3)                                                              \
    {                                                                                           \
        const double t1 = __shfl_xor_sync(FULL_MASK, V, K1), t2 = __shfl_xor_sync(FULL_MASK, V, K2), \
                     t3 = __shfl_xor_sync(FULL_MASK, V, K3);                                    \
        V = (V + t1) + (t2 + t3);                                                               \
    }
    B200P_KW_S4(a, 1, 2, 3) B200P_KW_S4(b, 1, 2, 3) B200P_KW_S4(c, 1, 2, 3)
    B200P_KW_S4(a, 4, 8, 12) B200P_KW_S4(b, 4, 8, 12) B200P_KW_S4(c, 4, 8, 12)
#undef B200P_KW_S4
    a += __shfl_xor_sync(FULL_MASK, a, 16);
    b += __shfl_xor_sync(FULL_MASK, b, 16);
    c += __shfl_xor_sync(FULL_MASK, c, 16);
    return;
#elif B200P_KW_RED
#pragma unroll
    for (int k = 16; k >= 1; k >>= 1) {
        const double ta = __shfl_xor_sync(FULL_MASK, a, k), tb = __shfl_xor_sync(FULL_MASK, b, k),
                     tc = __shfl_xor_sync(FULL_MASK, c, k);
        a += ta;
        b += tb;
        c += tc;
    }
    return;
#endif
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
    a = __shfl_sync(FULL_MASK, w, 0);
    b = __shfl_sync(FULL_MASK, w, 16);
    c = __shfl_sync(FULL_MASK, w, 8);
}

struct WarpSmem {
    alignas(16) double wx[KW_WARPS][32];
    alignas(16) double wy[KW_WARPS][32];
    alignas(8) uint8_t fx[KW_WARPS][32];
    alignas(8) uint8_t fy[KW_WARPS][32];
    uint32_t tm_base;
    int nlive;
};

struct WarpItem {
    int p, ix, iy;
};

#ifndef B200P_KW_STCS
#define B200P_KW_STCS 1       // weighted tiles leave with streaming stores (they are read next by K2b, not here)
#endif
#ifndef B200P_KW_CHUNK
#define B200P_KW_CHUNK 4      // consecutive items per claim (a warp walks along a block row: its windows overlap in L1)
#endif
constexpr unsigned KW_CHUNK_MAX = B200P_KW_CHUNK;

// Dynamic shared memory: the per-problem scalars, the list of live problems and the block-start tables
// of the level, staged once per CTA so that decoding an item costs LDS latency instead of a chain of
// dependent L2 round trips.
//   double rs[P]; int general[P]; int live[P]; int xs[nx]; int ys[ny]
__host__ __device__ inline size_t kw_table_bytes(int P, int nx, int ny) {
    return sizeof(double) * P + sizeof(int) * (2 * (size_t)P + nx + ny);
}

// Work distribution: the items (live problem, block) of a launch are claimed from a global counter in
// runs of KW_CHUNK consecutive items, one claim ahead of the run being solved (the atomic's round trip
// runs under a whole block solve), so the warps of the grid finish together whatever the spread of CG
// step counts; the first run of a warp is its own index.  The last CTA to leave zeroes the counters
// for the next launch on the stream.
template <bool RM, bool QT, bool DIRECT = false>
__global__ void __maxnreg__(B200P_KW_MAXREG)
oras_sweep_warp_kernel(const WarpSweepArgs A) {
    constexpr int TW = 8, TH = 4, BW = 32, BH = 32;
    // TMEM columns per warp and lane: v (64) [+ q (64)] [+ the lane's tile of u (64), DIRECT]; a power of two
    constexpr int NCOLW = DIRECT ? (QT ? 256 : 128) : (QT ? 128 : 64);
    constexpr int NCOL = NCOLW * ((KW_WARPS + 3) / 4);     // warps w and w + 4 share a lane quarter
    __shared__ WarpSmem sm;
    extern __shared__ __align__(16) unsigned char kw_dyn[];
    const SweepArgs &S = A.S;
    const LevelDev &L = S.L;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double *s_rs = reinterpret_cast<double *>(kw_dyn);
    int *s_general = reinterpret_cast<int *>(s_rs + A.P);
    int *s_live = s_general + A.P;
    int *s_xs = s_live + A.P, *s_ys = s_xs + L.nx;

    if (warp == 0) {
        const uint32_t slot = (uint32_t)__cvta_generic_to_shared(&sm.tm_base);
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(slot), "r"(NCOL) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (warp == KW_WARPS - 1) {
        // live problems in ascending order; frozen problems and rs == 0 (solvers.py:420) are skipped
        int base = 0;
        for (int t0 = 0; t0 < A.P; t0 += 32) {
            const int t = t0 + lane;
            double rs = 0.0;
            if (t < A.P) {
                rs = (!S.pred || S.pred[t]) ? S.rs[t] : 0.0;
                s_rs[t] = rs;
                s_general[t] = S.mflag[t] != 0;
            }
            const unsigned m = __ballot_sync(FULL_MASK, rs != 0.0);
            if (rs != 0.0) s_live[base + __popc(m & ((1u << lane) - 1u))] = t;
            base += __popc(m);
        }
        if (lane == 0) sm.nlive = base;
    } else {
        for (int t = threadIdx.x; t < L.nx; t += KW_THREADS - 32) s_xs[t] = L.xs[t];
        for (int t = threadIdx.x; t < L.ny; t += KW_THREADS - 32) s_ys[t] = L.ys[t];
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tv = sm.tm_base + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * NCOLW;  // lane quarter
    const uint32_t tq = tv + 64;
    const uint32_t tu = tv + (QT ? 128 : 64);

    const int W = L.w, H = L.h;
    const double hinv2 = L.hinv2, g_in = L.g_in;
    const int lx = lane & 3, ly = lane >> 2;
    const int bx = lx * TW, by = ly * TH;
    double *swx = sm.wx[warp], *swy = sm.wy[warp];
    const unsigned grid_warps = gridDim.x * KW_WARPS;
    const unsigned total = (unsigned)sm.nlive * (unsigned)A.items_per_problem;

    auto decode = [&](unsigned it, WarpItem &w) {
        const unsigned li = kw_div(it, A.m_ipp, A.k_ipp);
        const unsigned rem = it - li * (unsigned)A.items_per_problem;
        const unsigned iyl = kw_div(rem, A.m_nx, A.k_nx);
        w.p = s_live[li];
        w.ix = (int)(rem - iyl * (unsigned)L.nx);
        w.iy = (int)iyl + S.iy0;
    };

    // The gather window of an item: 6 x 10 values of u around the lane's tile, its tile of b, its mask word.
    double uc[TH + 2][TW + 2];
    double bt[RM ? 1 : TH][TW];
    unsigned mbits = 0;
    auto load_window = [&](const WarpItem &w) {
        const int x0 = s_xs[w.ix], y0 = s_ys[w.iy];
        const int gx0 = x0 + bx, gy0 = y0 + by;
        const int frame = S.channels == 3 ? w.p / 3 : (S.channels == 1 ? w.p : w.p / S.channels);
        mbits = A.mtab[((size_t)frame * L.nblocks + w.iy * L.nx + w.ix) * 32 + lane];
        const double *urow = S.u + (size_t)w.p * S.plane + (size_t)(gy0 - 1) * W + gx0;
        if (S.u_zero) {
            // a coarse correction before its first sweep: identically 0, never written, never read
#pragma unroll
            for (int j = 0; j < TH + 2; ++j)
#pragma unroll
                for (int i = 0; i < TW + 2; ++i) uc[j][i] = 0.0;
        } else if (!(x0 == 0 || y0 == 0 || x0 + BW >= W || y0 + BH >= H)) {
#pragma unroll
            for (int j = 0; j < TH + 2; ++j) {
                const double *rp = urow + (size_t)j * W;
#pragma unroll
                for (int k = 0; k < TW / 2; ++k) {
                    const double2 a = *reinterpret_cast<const double2 *>(rp + 2 * k);
                    uc[j][1 + 2 * k] = a.x;
                    uc[j][2 + 2 * k] = a.y;
                }
                if (j >= 1 && j <= TH) {
                    uc[j][0] = rp[-1];
                    uc[j][TW + 1] = rp[TW];
                } else {
                    uc[j][0] = uc[j][TW + 1] = 0.0;
                }
            }
        } else {
            const bool hasL = gx0 > 0, hasR = gx0 + TW < W, hasT = gy0 > 0, hasB = gy0 + TH < H;
#pragma unroll
            for (int j = 0; j < TH + 2; ++j) {
                const double *rp = urow + (size_t)j * W;
                const bool rowin = (j > 0 || hasT) && (j < TH + 1 || hasB);
#pragma unroll
                for (int k = 0; k < TW / 2; ++k) {
                    double2 a = make_double2(0.0, 0.0);
                    if (rowin) a = *reinterpret_cast<const double2 *>(rp + 2 * k);
                    uc[j][1 + 2 * k] = a.x;
                    uc[j][2 + 2 * k] = a.y;
                }
                uc[j][0] = uc[j][TW + 1] = 0.0;
                if (j >= 1 && j <= TH) {
                    if (hasL) uc[j][0] = rp[-1];
                    if (hasR) uc[j][TW + 1] = rp[TW];
                }
            }
        }
        if (!RM) {
#pragma unroll
            for (int j = 0; j < TH; ++j) {
                const double *bp = S.b + (size_t)w.p * S.plane + (size_t)(gy0 + j) * W + gx0;
#pragma unroll
                for (int k = 0; k < TW / 2; ++k) {
                    const double2 a = *reinterpret_cast<const double2 *>(bp + 2 * k);
                    bt[RM ? 0 : j][2 * k] = a.x;
                    bt[RM ? 0 : j][2 * k + 1] = a.y;
                }
            }
        }
    };

    WarpCG cg;
    cg.zL = lx == 0 ? 0.0 : 1.0;
    cg.zR = lx == 3 ? 0.0 : 1.0;
    cg.zT = ly == 0 ? 0.0 : 1.0;
    cg.zB = ly == 7 ? 0.0 : 1.0;

    WarpItem cur;
    const unsigned KW_CHUNK = A.chunk;
    unsigned item = (blockIdx.x * KW_WARPS + warp) * KW_CHUNK, run_end = item + KW_CHUNK;
    bool have = item < total;
    if (have) {
        decode(item, cur);
    }
    unsigned claimed = 0;  // lane 0: start of the warp's next run, minus the statically assigned part

    while (have) {
        if (item + KW_CHUNK == run_end && lane == 0)   // first item of a run: claim the next run (plain PTX:
            asm volatile("atom.global.add.u32 %0, [%1], %2;"  // no warp-aggregation sequence, no wait here)
                         : "=r"(claimed) : "l"(A.claim), "r"(KW_CHUNK));
        load_window(cur);
        const int p = cur.p, ix = cur.ix, iy = cur.iy;
        const int blk = iy * L.nx + ix;
        const double rs_g = s_rs[p];
        __syncwarp();  // the previous item's weight rows have been consumed
        if (DIRECT) {
            sm.fx[warp][lane] = A.xflag[ix * BW + lane];
            sm.fy[warp][lane] = A.yflag[iy * BH + lane];
        }
        swx[lane] = L.wx[ix * BW + lane];
        swy[lane] = L.wy[iy * BH + lane];
        const int x0 = s_xs[ix], y0 = s_ys[iy];
        const double target = S.eta * rs_g;
        const bool general = s_general[p] != 0;

        cg.mbits = mbits;
        {
            const double gl = x0 > 0 ? g_in : 1.0, gr = x0 + BW < W ? g_in : 1.0;
            const double gt = y0 > 0 ? g_in : 1.0, gb = y0 + BH < H ? g_in : 1.0;
            cg.gLz = lx == 0 ? gl : 0.0;
            cg.gRz = lx == 3 ? gr : 0.0;
            cg.cT = ly == 0 ? 4.0 - gt : 4.0;
            cg.cB = ly == 7 ? 4.0 - gb : 4.0;
        }

        const int gx0 = x0 + bx, gy0 = y0 + by;
        const bool border = x0 == 0 || y0 == 0 || x0 + BW >= W || y0 + BH >= H;  // warp-uniform

        // ---- gather: global residual g = b - A u on the tile (core.py:100-110)
        double r[TH][TW];
        {
            const double nc4 = -4.0 * hinv2;
#pragma unroll
            for (int j = 0; j < TH; ++j) {
#pragma unroll
                for (int i = 0; i < TW; ++i) {
                    const double s = ((uc[j][i + 1] + uc[j + 2][i + 1]) + uc[j + 1][i]) + uc[j + 1][i + 2];
                    const double uu = uc[j + 1][i + 1];
                    const double res = fma(hinv2, s, RM ? nc4 * uu : fma(nc4, uu, bt[RM ? 0 : j][i]));
                    const bool m = (mbits >> (j * TW + i)) & 1u;
                    // RM: rhs = where(mask, known, 0) and b - u == 0 at mask pixels unless `general`
                    r[j][i] = m ? (RM ? 0.0 : bt[RM ? 0 : j][i] - uu) : res;
                }
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
                            r[j][i] = S.b[(size_t)p * S.plane + (size_t)(gy0 + j) * W + gx0 + i] - uc[j + 1][i + 1];
            }
        }

        if (DIRECT) {
            // the lane's own pixels of u wait in tensor memory for the direct update u_out = u + v
#pragma unroll
            for (int j = 0; j < TH; ++j) {
                double urow[TW];
#pragma unroll
                for (int i = 0; i < TW; ++i) urow[i] = uc[j + 1][i + 1];
                tm_st8(tu + 16 * j, urow);
            }
        }

        // ---- the warp's next item (claimed above): decode it and pull its window towards L1
        WarpItem nxt;
        unsigned next = item + 1;
        if (next == run_end) {
            next = __shfl_sync(FULL_MASK, claimed, 0) + grid_warps * KW_CHUNK;
            run_end = next + KW_CHUNK;
        }
        const bool have_next = next < total;
        if (have_next) {
            decode(next, nxt);
        }

        // ---- local start: v0 = where(mask, g, 0) -> TMEM, r0 = g - A_i v0 (solvers.py:331-333)
        double pc[TH][TW];
        if (general) {
#pragma unroll
            for (int j = 0; j < TH; ++j) {
#pragma unroll
                for (int i = 0; i < TW; ++i) pc[j][i] = ((mbits >> (j * TW + i)) & 1u) ? r[j][i] : 0.0;
                tm_st8(tv + 16 * j, pc[j]);
            }
            cg.apply(pc, [&](int j, const double (&qrow)[TW]) {
#pragma unroll
                for (int i = 0; i < TW; ++i) {
                    const bool m = (mbits >> (j * TW + i)) & 1u;
                    r[j][i] = m ? 0.0 : fma(-hinv2, qrow[i], r[j][i]);
                }
            });
        } else {
            const double z[TW] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int j = 0; j < TH; ++j) tm_st8(tv + 16 * j, z);
        }
        double rs_k;
        {
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int j = 0; j < TH; ++j)
#pragma unroll
                for (int i = 0; i < TW; ++i) acc[i & 3] = fma(r[j][i], r[j][i], acc[i & 3]);
            rs_k = warp_sum((acc[0] + acc[1]) + (acc[2] + acc[3]));
        }
        tm_wait_st();

        // The LAST CG step's update of v is folded into the weighted store below (v = v_tmem + a_last p):
        // no TMEM round trip, and the residual / direction updates of that step are skipped.
        double a_last = 0.0;
#pragma unroll
        for (int j = 0; j < TH; ++j)
#pragma unroll
            for (int i = 0; i < TW; ++i) pc[j][i] = r[j][i];
        if (rs_k > target) {  // solvers.py:336 (strict)
            double inv_rs = __drcp_rn(rs_k);
            for (int it = 0; it < S.max_iters; ++it) {
                double d_pq0 = 0.0, d_pq1 = 0.0, d_rq0 = 0.0, d_rq1 = 0.0, d_qq0 = 0.0, d_qq1 = 0.0;
                double q[QT ? 1 : TH][TW];
                cg.apply(pc, [&](int j, const double (&qrow)[TW]) {
#pragma unroll
                    for (int i = 0; i < TW; i += 2) {
                        d_pq0 = fma(pc[j][i], qrow[i], d_pq0);
                        d_rq0 = fma(r[j][i], qrow[i], d_rq0);
                        d_qq0 = fma(qrow[i], qrow[i], d_qq0);
                        d_pq1 = fma(pc[j][i + 1], qrow[i + 1], d_pq1);
                        d_rq1 = fma(r[j][i + 1], qrow[i + 1], d_rq1);
                        d_qq1 = fma(qrow[i + 1], qrow[i + 1], d_qq1);
                    }
                    if (QT) {
                        tm_st8(tq + 16 * j, qrow);
                    } else {
#pragma unroll
                        for (int i = 0; i < TW; ++i) q[QT ? 0 : j][i] = qrow[i];
                    }
                });
                double d_pq = d_pq0 + d_pq1, d_rq = d_rq0 + d_rq1, d_qq = d_qq0 + d_qq1;
                warp_sum3(lane, d_pq, d_rq, d_qq);
                const double pq = hinv2 * d_pq;
                const bool ok = pq > 0.0;                               // solvers.py:348
                const double a = ok ? rs_k * __drcp_rn(pq) : 0.0;       // :349-350
                const double ah = a * hinv2;
                const double rs_new = fma(ah * ah, d_qq, fma(-2.0 * ah, d_rq, rs_k));
                a_last = a;
                if (rs_new <= target || !ok || it + 1 >= S.max_iters) break;   // :354, :338
                const double beta = rs_new * inv_rs;
                if (QT) {
                    tm_wait_st();
#pragma unroll
                    for (int j = 0; j < TH; ++j) {
                        TmRow tvr, tqr;
                        tm_ld8(tv + 16 * j, tvr);
                        tm_ld8(tq + 16 * j, tqr);
                        tm_wait_ld2(tvr, tqr);
                        double vrow[TW];
#pragma unroll
                        for (int i = 0; i < TW; ++i) {
                            vrow[i] = fma(a, pc[j][i], tvr.get(i));
                            r[j][i] = fma(-ah, tqr.get(i), r[j][i]);
                        }
                        tm_st8(tv + 16 * j, vrow);
#pragma unroll
                        for (int i = 0; i < TW; ++i) pc[j][i] = fma(beta, pc[j][i], r[j][i]);
                    }
                } else {
                    // residual first (q dies), then ONE batch of v loads into the freed registers
#pragma unroll
                    for (int j = 0; j < TH; ++j)
#pragma unroll
                        for (int i = 0; i < TW; ++i) r[j][i] = fma(-ah, q[QT ? 0 : j][i], r[j][i]);
                    TmRow t0, t1, t2, t3;
                    tm_ld8(tv, t0);
                    tm_ld8(tv + 16, t1);
                    tm_ld8(tv + 32, t2);
                    tm_ld8(tv + 48, t3);
                    tm_wait_ld2(t0, t1);
                    tm_wait_ld2(t2, t3);
                    double vrow[TW];
#define B200P_KW_V(J, T)                                                                     \
    {                                                                                        \
        _Pragma("unroll") for (int i = 0; i < TW; ++i) vrow[i] = fma(a, pc[J][i], T.get(i)); \
        tm_st8(tv + 16 * J, vrow);                                                           \
    }
                    B200P_KW_V(0, t0) B200P_KW_V(1, t1) B200P_KW_V(2, t2) B200P_KW_V(3, t3)
#undef B200P_KW_V
#pragma unroll
                    for (int j = 0; j < TH; ++j)
#pragma unroll
                        for (int i = 0; i < TW; ++i) pc[j][i] = fma(beta, pc[j][i], r[j][i]);
                }
                tm_wait_st();
                rs_k = rs_new;
                inv_rs = __drcp_rn(rs_k);
            }
        }

        // ---- weighted correction (v * wy) * wx (solvers.py:309-310)
        {
            double *out = S.scratch + ((size_t)p * L.nblocks + blk) * (BW * BH);
            TmRow t0, t1, t2, t3;
            tm_ld8(tv, t0);
            tm_ld8(tv + 16, t1);
            tm_ld8(tv + 32, t2);
            tm_ld8(tv + 48, t3);
            __syncwarp();
            double wxv[TW], wyv[TH];
#pragma unroll
            for (int k = 0; k < TW / 2; ++k) {
                const double2 t = *reinterpret_cast<const double2 *>(&swx[bx + 2 * k]);
                wxv[2 * k] = t.x;
                wxv[2 * k + 1] = t.y;
            }
#pragma unroll
            for (int k = 0; k < TH / 2; ++k) {
                const double2 t = *reinterpret_cast<const double2 *>(&swy[by + 2 * k]);
                wyv[2 * k] = t.x;
                wyv[2 * k + 1] = t.y;
            }
            tm_wait_ld2(t0, t1);
            tm_wait_ld2(t2, t3);
            double vf[TH][TW];
#define B200P_KW_VF(J, T) \
    _Pragma("unroll") for (int i = 0; i < TW; ++i) vf[J][i] = fma(a_last, pc[J][i], T.get(i));
            B200P_KW_VF(0, t0) B200P_KW_VF(1, t1) B200P_KW_VF(2, t2) B200P_KW_VF(3, t3)
#undef B200P_KW_VF
            if (!DIRECT) {
#pragma unroll
                for (int j = 0; j < TH; ++j) {
                    double2 *row = reinterpret_cast<double2 *>(out + (by + j) * BW + bx);
#pragma unroll
                    for (int k = 0; k < TW / 2; ++k) {
                        double2 o;
                        o.x = (vf[j][2 * k] * wyv[j]) * wxv[2 * k];
                        o.y = (vf[j][2 * k + 1] * wyv[j]) * wxv[2 * k + 1];
#if B200P_KW_STCS
                        __stcs(row + k, o);   // streaming store: the tile is not read again by this kernel
#else
                        row[k] = o;
#endif
                    }
                }
            } else {
                // Pixels with one writer (weight exactly 1 here, 0 in every other block) in single-writer rows
                // and sector-aligned single-writer column groups go straight to the partner iterate; pixels of
                // the overlap bands with a non-zero weight go to the tile; zero-weight pixels go nowhere.
                const uint2 fxw = *reinterpret_cast<const uint2 *>(&sm.fx[warp][bx]);
                const unsigned fyw = *reinterpret_cast<const unsigned *>(&sm.fy[warp][by]);
                TmRow u0, u1, u2, u3;
                tm_ld8(tu, u0);
                tm_ld8(tu + 16, u1);
                tm_ld8(tu + 32, u2);
                tm_ld8(tu + 48, u3);
                tm_wait_ld2(u0, u1);
                tm_wait_ld2(u2, u3);
                double *tile = S.scratch + ((size_t)p * L.nblocks + blk) * KW_TSZ + (x0 & (KW_ALIGN - 1));
                double *uo = A.u_out + (size_t)p * S.plane + (size_t)gy0 * W + gx0;
#define B200P_KW_OUT(J, U)                                                                               \
    {                                                                                                    \
        const unsigned fy = (fyw >> (8 * J)) & 0xffu;                                                    \
        _Pragma("unroll") for (int k = 0; k < TW / 2; ++k) {                                             \
            /* pixel pairs are homogeneous (checked when the plan is built): one flag byte decides */    \
            const unsigned fa = ((k < 2 ? fxw.x : fxw.y) >> (16 * (k & 1))) & 0xffu;                     \
            const bool direct = (fa & fy & 2u) != 0;                                                     \
            const bool mine = (fa & fy & 1u) != 0;                                                       \
            const double ta = (vf[J][2 * k] * wyv[J]) * wxv[2 * k];                                      \
            const double tb = (vf[J][2 * k + 1] * wyv[J]) * wxv[2 * k + 1];                              \
            if (direct && mine)                                                                          \
                *reinterpret_cast<double2 *>(uo + (size_t)J * W + 2 * k) =                               \
                    make_double2(U.get(2 * k) + ta, U.get(2 * k + 1) + tb);                              \
            if (!direct)   /* zero-weight pixels of a band pair are stored as the zeros they are */      \
                __stcs(reinterpret_cast<double2 *>(tile + (by + J) * KW_TP + bx + 2 * k), make_double2(ta, tb)); \
        }                                                                                                \
    }
                B200P_KW_OUT(0, u0) B200P_KW_OUT(1, u1) B200P_KW_OUT(2, u2) B200P_KW_OUT(3, u3)
#undef B200P_KW_OUT
            }
        }
        cur = nxt;
        item = next;
        have = have_next;
    }

    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(sm.tm_base), "r"(NCOL) : "memory");
    if (threadIdx.x == 0) {
        // every warp of this CTA has made its last claim; the last CTA re-arms the counters
        __threadfence();
        if (atomicAdd(A.claim + 1, 1u) == gridDim.x - 1) {
            A.claim[0] = 0;
            A.claim[1] = 0;
            __threadfence();
        }
    }
}

}  // namespace b200p
