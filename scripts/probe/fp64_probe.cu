// fp64_probe.cu -- latency / issue-rate probe of the instructions the ORAS block CG is made of
// (DFMA, DADD, SHFL, bar.sync, LDS, DRCP) on one SM of a B200.  Build: nvcc -O3 -arch=sm_100a.
#include <cstdio>
#include <cuda_runtime.h>

#define N 4096

template <int CHAINS>
__global__ void dfma_lat(double *out, long long *cyc, double a, double b) {
    double x[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x + c;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, b);
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) s += x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int CHAINS>
__global__ void dadd_lat(double *out, long long *cyc, double a) {
    double x[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x + c;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) x[c] = x[c] + a;
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) s += x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

__global__ void shfl_lat(double *out, long long *cyc) {
    double x = threadIdx.x;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1 + (i & 15));
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = x;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

__global__ void shfl_add_lat(double *out, long long *cyc) {  // one butterfly stage: shfl + dadd
    double x = threadIdx.x;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1 + (i & 15));
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = x;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

__global__ void shfl_tput(double *out, long long *cyc) {  // 8 independent 64-bit shuffles per iteration
    double x[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = threadIdx.x + c;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) {
#pragma unroll
        for (int c = 0; c < 8; ++c) x[c] = __shfl_xor_sync(0xffffffffu, x[c], 1 + (i & 15));
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

__global__ void bar_lat(double *out, long long *cyc) {
    __shared__ double s[256];
    double x = threadIdx.x;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) {
        s[threadIdx.x] = x;
        __syncthreads();
        x += s[(threadIdx.x + 32) % blockDim.x];
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = x;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

__global__ void lds_lat(double *out, long long *cyc) {
    __shared__ int s[256];
    s[threadIdx.x] = (threadIdx.x + 1) & 255;
    __syncthreads();
    int j = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) j = s[j];
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = j;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

__global__ void drcp_lat(double *out, long long *cyc) {
    double x = 1.5 + threadIdx.x;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) x = __drcp_rn(x) + 1.25;
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = x;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

__global__ void ddiv_lat(double *out, long long *cyc) {
    double x = 1.5 + threadIdx.x;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) x = 3.0 / x + 1.25;
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = x;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

__global__ void fsel_dfma(double *out, long long *cyc, double a, double b, unsigned m) {  // DFMA + 64-bit select
    double x[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = threadIdx.x + c;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const double y = fma(x[c], a, b);
            x[c] = ((m >> c) & 1u) ? 0.0 : y;
        }
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    double *out;
    long long *cyc, h;
    cudaMalloc(&out, 1 << 24);
    cudaMalloc(&cyc, 8);
#define RUN(label, per, kern, grid, block, ...)                                       \
    kern<<<grid, block>>>(out, cyc, ##__VA_ARGS__);                                   \
    cudaDeviceSynchronize();                                                          \
    kern<<<grid, block>>>(out, cyc, ##__VA_ARGS__);                                   \
    cudaDeviceSynchronize();                                                          \
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);                                   \
    printf("%-44s block=%4d grid=%3d  %7.2f cycles / %s\n", label, block, grid, (double)h / N, per);
    RUN("DFMA dependent chain (1 warp)", "DFMA", dfma_lat<1>, 1, 32, 1.0000001, 1e-9);
    RUN("DADD dependent chain (1 warp)", "DADD", dadd_lat<1>, 1, 32, 1e-9);
    RUN("DFMA 2 chains (1 warp)", "2 DFMA", dfma_lat<2>, 1, 32, 1.0000001, 1e-9);
    RUN("DFMA 4 chains (1 warp)", "4 DFMA", dfma_lat<4>, 1, 32, 1.0000001, 1e-9);
    RUN("DFMA 8 chains (1 warp)", "8 DFMA", dfma_lat<8>, 1, 32, 1.0000001, 1e-9);
    RUN("DFMA 16 chains (1 warp)", "16 DFMA", dfma_lat<16>, 1, 32, 1.0000001, 1e-9);
    RUN("DFMA 8 chains (4 warps = 1/SMSP)", "8 DFMA", dfma_lat<8>, 1, 128, 1.0000001, 1e-9);
    RUN("DFMA 8 chains (8 warps = 2/SMSP)", "8 DFMA", dfma_lat<8>, 1, 256, 1.0000001, 1e-9);
    RUN("DFMA 8 chains (16 warps = 4/SMSP)", "8 DFMA", dfma_lat<8>, 1, 512, 1.0000001, 1e-9);
    RUN("DFMA 1 chain (16 warps = 4/SMSP)", "DFMA", dfma_lat<1>, 1, 512, 1.0000001, 1e-9);
    RUN("DFMA 1 chain (32 warps = 8/SMSP)", "DFMA", dfma_lat<1>, 1, 1024, 1.0000001, 1e-9);
    RUN("DFMA 2 chains (12 warps = 3/SMSP)", "2 DFMA", dfma_lat<2>, 1, 384, 1.0000001, 1e-9);
    RUN("DFMA 4 chains (12 warps = 3/SMSP)", "4 DFMA", dfma_lat<4>, 1, 384, 1.0000001, 1e-9);
    RUN("DADD 8 chains (4 warps)", "8 DADD", dadd_lat<8>, 1, 128, 1e-9);
    RUN("SHFL.BFLY 64-bit dependent", "shuffle", shfl_lat, 1, 32);
    RUN("SHFL.BFLY 64-bit + DADD dependent", "stage", shfl_add_lat, 1, 32);
    RUN("SHFL 64-bit x8 independent (1 warp)", "8 shuffles", shfl_tput, 1, 32);
    RUN("SHFL 64-bit x8 independent (4 warps)", "8 shuffles", shfl_tput, 1, 128);
    RUN("SHFL 64-bit x8 independent (16 warps)", "8 shuffles", shfl_tput, 1, 512);
    RUN("STS + bar.sync(64) + LDS + DADD", "round", bar_lat, 1, 64);
    RUN("STS + bar.sync(32) + LDS + DADD", "round", bar_lat, 1, 32);
    RUN("LDS dependent", "LDS", lds_lat, 1, 32);
    RUN("__drcp_rn + DADD dependent", "rcp", drcp_lat, 1, 32);
    RUN("ddiv + DADD dependent", "div", ddiv_lat, 1, 32);
    RUN("DFMA + 64-bit select x8 (1 warp)", "8 px", fsel_dfma, 1, 32, 1.0000001, 1e-9, 0x11u);
    RUN("DFMA + 64-bit select x8 (4 warps)", "8 px", fsel_dfma, 1, 128, 1.0000001, 1e-9, 0x11u);
    RUN("DFMA + 64-bit select x8 (16 warps)", "8 px", fsel_dfma, 1, 512, 1.0000001, 1e-9, 0x11u);
    return 0;
}
