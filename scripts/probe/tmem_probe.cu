// tmem_probe.cu -- (A) do 64-thread CTAs spread over all four SM sub-partitions?  (B) tensor memory
// as a thread-private scratch: tcgen05.st / tcgen05.ld 32x32b throughput and latency per SM,
// alone and next to shuffles / DFMAs.  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define N 2048

__global__ void dfma_grid(double *out, double a, double b) {
    double x[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = threadIdx.x + c;
    for (int i = 0; i < N; ++i) {
#pragma unroll
        for (int c = 0; c < 8; ++c) x[c] = fma(x[c], a, b);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += x[c];
    out[(size_t)blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ uint32_t tmem_alloc(uint32_t *slot, int ncols) {
    if (threadIdx.x < 32) {
        uint32_t sa = (uint32_t)__cvta_generic_to_shared(slot);
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa), "r"(ncols) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    __syncthreads();
    return *slot;
}
__device__ __forceinline__ void tmem_free(uint32_t base, int ncols) {
    __syncthreads();
    if (threadIdx.x < 32)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(ncols) : "memory");
}

#define ST16(addr, r, o)                                                                                  \
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" \
                 ::"r"(addr), "r"(r[o + 0]), "r"(r[o + 1]), "r"(r[o + 2]), "r"(r[o + 3]), "r"(r[o + 4]), "r"(r[o + 5]),   \
                 "r"(r[o + 6]), "r"(r[o + 7]), "r"(r[o + 8]), "r"(r[o + 9]), "r"(r[o + 10]), "r"(r[o + 11]),             \
                 "r"(r[o + 12]), "r"(r[o + 13]), "r"(r[o + 14]), "r"(r[o + 15]) : "memory")
#define LD16(addr, r, o)                                                                                  \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
                 : "=r"(r[o + 0]), "=r"(r[o + 1]), "=r"(r[o + 2]), "=r"(r[o + 3]), "=r"(r[o + 4]), "=r"(r[o + 5]),       \
                   "=r"(r[o + 6]), "=r"(r[o + 7]), "=r"(r[o + 8]), "=r"(r[o + 9]), "=r"(r[o + 10]), "=r"(r[o + 11]),     \
                   "=r"(r[o + 12]), "=r"(r[o + 13]), "=r"(r[o + 14]), "=r"(r[o + 15]) : "r"(addr) : "memory")

// mode 0: st x32 regs + wait, ld x32 regs + wait, dependent (round-trip latency of 128 B per thread)
// mode 1: ld only (x32 regs), accumulate       mode 2: st only
__global__ void tmem_rw(double *out, long long *cyc, int mode, int ok_check) {
    __shared__ uint32_t slot;
    const int ncols = 64;
    const uint32_t base = tmem_alloc(&slot, ncols);
    const int warp = threadIdx.x >> 5;
    const uint32_t addr = base + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 32);
    uint32_t r[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) r[k] = threadIdx.x * 64 + k;
    ST16(addr, r, 0);
    ST16(addr + 16, r, 16);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    __syncthreads();
    long long t0 = clock64();
    uint32_t acc = 0;
    for (int i = 0; i < N; ++i) {
        if (mode == 0) {
            ST16(addr, r, 0);
            ST16(addr + 16, r, 16);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            LD16(addr, r, 0);
            LD16(addr + 16, r, 16);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int k = 0; k < 32; ++k) r[k] += 1;
        } else if (mode == 1) {
            LD16(addr, r, 0);
            LD16(addr + 16, r, 16);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int k = 0; k < 32; ++k) acc += r[k];
        } else {
#pragma unroll
            for (int k = 0; k < 32; ++k) r[k] += i;
            ST16(addr, r, 0);
            ST16(addr + 16, r, 16);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
    }
    long long t1 = clock64();
#pragma unroll
    for (int k = 0; k < 32; ++k) acc += r[k];
    if (ok_check && mode == 0) {
        // every register went through N store/load round trips with +1 each
        bool ok = true;
#pragma unroll
        for (int k = 0; k < 32; ++k) ok = ok && (r[k] == threadIdx.x * 64 + k + N);
        if (!ok) printf("TMEM round trip MISMATCH thread %d\n", threadIdx.x);
    }
    out[(size_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
    tmem_free(base, ncols);
}

// warps 0..nt-1 do TMEM round trips, the others shuffles (mode 0) or DFMAs (mode 1): interference test
__global__ void tmem_mix(double *out, long long *cyc, int nt, int other) {
    __shared__ uint32_t slot;
    const int ncols = 64;
    const uint32_t base = tmem_alloc(&slot, ncols);
    const int warp = threadIdx.x >> 5;
    const uint32_t addr = base + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 32);
    uint32_t r[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) r[k] = threadIdx.x * 64 + k;
    double x[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = threadIdx.x + c;
    __syncthreads();
    long long t0 = clock64();
    if (warp < nt) {
        for (int i = 0; i < N; ++i) {
            ST16(addr, r, 0);
            ST16(addr + 16, r, 16);
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            LD16(addr, r, 0);
            LD16(addr + 16, r, 16);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int k = 0; k < 32; ++k) r[k] += 1;
        }
    } else if (other == 0) {
        for (int i = 0; i < N; ++i) {
#pragma unroll
            for (int c = 0; c < 8; ++c) x[c] = __shfl_xor_sync(0xffffffffu, x[c], 1 + (i & 15));
        }
    } else {
        for (int i = 0; i < 4 * N; ++i) {
#pragma unroll
            for (int c = 0; c < 8; ++c) x[c] = fma(x[c], 1.0000001, 1e-9);
        }
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += x[c];
#pragma unroll
    for (int k = 0; k < 32; ++k) s += r[k];
    out[(size_t)blockIdx.x * blockDim.x + threadIdx.x] = s;
    if ((threadIdx.x & 31) == 0 && blockIdx.x == 0) cyc[warp] = t1 - t0;
    tmem_free(base, ncols);
}

int main() {
    double *out;
    long long *cyc, h[32];
    cudaMalloc(&out, 1 << 26);
    cudaMalloc(&cyc, 8 * 32);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    // ---- A: same number of warps as 64- or 128- or 256-thread CTAs
    for (int rep = 0; rep < 2; ++rep)
        for (int bs = 64; bs <= 256; bs *= 2) {
            const int warps_total = 148 * 16 * 8;  // 8 waves of 16 warps per SM
            const int grid = warps_total / (bs / 32);
            cudaEventRecord(e0);
            dfma_grid<<<grid, bs>>>(out, 1.0000001, 1e-9);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep)
                printf("A: DFMA x8 chains, %6d CTAs of %3d threads: %.3f ms  (%.2f SMSP-cycles per DFMA at 1.965 GHz)\n", grid,
                       bs, ms, ms * 1e-3 * 1.965e9 * 148 * 4 / ((double)warps_total * N * 8));
        }
    // ---- B: TMEM
    for (int mode = 0; mode < 3; ++mode)
        for (int bs = 32; bs <= 256; bs *= 2) {
            tmem_rw<<<1, bs>>>(out, cyc, mode, 1);
            cudaDeviceSynchronize();
            cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
            const char *nm = mode == 0 ? "st 128B/thr + wait + ld 128B/thr + wait" : (mode == 1 ? "ld 128B/thr + wait" : "st 128B/thr + wait");
            printf("B: %-42s block=%3d: %7.1f cycles/iter  -> %6.1f B/clk/SM each way\n", nm, bs, (double)h[0] / N,
                   bs * 128.0 / ((double)h[0] / N));
        }
    cudaError_t e = cudaGetLastError();
    printf("B status: %s\n", cudaGetErrorString(e));
    // several CTAs per SM (each allocating 64 columns)
    for (int bs = 64; bs <= 128; bs *= 2)
        for (int per_sm = 1; per_sm <= 8; per_sm *= 2) {
            cudaEventRecord(e0);
            tmem_rw<<<148 * per_sm, bs>>>(out, cyc, 0, 0);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            printf("B: round trips, %d CTAs/SM of %3d threads: %.3f ms -> %.1f cycles/iter, %.1f B/clk/SM each way\n", per_sm, bs, ms,
                   ms * 1e-3 * 1.965e9 / N, per_sm * bs * 128.0 / (ms * 1e-3 * 1.965e9 / N));
        }
    // ---- C: interference
    for (int other = 0; other < 2; ++other)
        for (int nt = 0; nt <= 8; nt += 4) {
            tmem_mix<<<1, 256>>>(out, cyc, nt, other);
            cudaDeviceSynchronize();
            cudaMemcpy(h, cyc, 8 * 8, cudaMemcpyDeviceToHost);
            printf("C: 8 warps, %d on TMEM round trips, rest on %s: warp0 %.1f cycles/iter, warp7 %.1f cycles/iter\n", nt,
                   other ? "DFMA x32" : "SHFL64 x8", (double)h[0] / N, (double)h[7] / N);
        }
    e = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
