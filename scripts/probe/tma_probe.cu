// Bisects which TMA box shapes / coordinates work for fp64 tiles.  nvcc -arch=sm_100a tma_probe.cu -o tma_probe
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *,
                                  CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                  CUtensorMapFloatOOBfill);
__global__ void probe(const __grid_constant__ CUtensorMap tm, int x, int y, int z, int bytes, double *out, int n) {
    extern __shared__ __align__(128) unsigned char smem[];
    double *tile = (double *)smem;
    unsigned long long *bar = (unsigned long long *)(smem + 16384);
    unsigned b = (unsigned)__cvta_generic_to_shared(bar), d = (unsigned)__cvta_generic_to_shared(tile);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                     ::"r"(d), "l"(&tm), "r"(x), "r"(y), "r"(z), "r"(b) : "memory");
    }
    __syncthreads();
    unsigned ok;
    do {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(b) : "memory");
    } while (!ok);
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = tile[i];
}
int main() {
    void *p = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    EncodeTiledFn enc = (EncodeTiledFn)p;
    const int W = 150, H = 100, P = 2;
    std::vector<double> h((size_t)W * H * P);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
    double *d, *out; cudaMalloc(&d, h.size() * 8); cudaMalloc(&out, 16384);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 20000);
    int boxes[][2] = {{36, 34}, {32, 32}};
    int coords[][2] = {{0, 0}, {26, 26}, {-2, -1}, {24, 25}, {116, -1}, {-2, 25}, {118, 67}, {-1, -1}};
    for (auto &bx : boxes) for (auto &c : coords) {
        CUtensorMap tm;
        cuuint64_t dims[3] = {W, H, P}; cuuint64_t strides[2] = {W * 8ull, (cuuint64_t)W * H * 8};
        cuuint32_t box[3] = {(cuuint32_t)bx[0], (cuuint32_t)bx[1], 1}; cuuint32_t es[3] = {1, 1, 1};
        CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("box %dx%d encode failed %d\n", bx[0], bx[1], (int)r); break; }
        int n = bx[0] * bx[1];
        probe<<<1, 64, 20000>>>(tm, c[0], c[1], 1, n * 8, out, n);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("box %dx%d at (%d,%d): %s\n", bx[0], bx[1], c[0], c[1], cudaGetErrorString(e)); return 1; }
        std::vector<double> o(n); cudaMemcpy(o.data(), out, n * 8, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int j = 0; j < bx[1]; ++j) for (int i = 0; i < bx[0]; ++i) {
            int gx = c[0] + i, gy = c[1] + j;
            double want = (gx < 0 || gx >= W || gy < 0 || gy >= H) ? 0.0 : h[(size_t)W * H + (size_t)gy * W + gx];
            if (o[j * bx[0] + i] != want) ++bad;
        }
        printf("box %dx%d at (%d,%d): ok, %d mismatches\n", bx[0], bx[1], c[0], c[1], bad);
    }
    return 0;
}
