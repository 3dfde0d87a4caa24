#include <cuda_runtime.h>
#include <cstdio>
__global__ void body(int *ctr, cudaGraphConditionalHandle h) {
    int v = ++(*ctr);
    cudaGraphSetConditional(h, v < 5 ? 1 : 0);
}
__global__ void init(int *ctr, cudaGraphConditionalHandle h) { *ctr = 0; cudaGraphSetConditional(h, 1); }
int main() {
    setvbuf(stdout, NULL, _IONBF, 0); int *d; printf("malloc %d\n", (int)cudaMalloc(&d, 4));
    int *hres; cudaMallocHost(&hres, 4);
    cudaStream_t s, s2; cudaStreamCreate(&s); cudaStreamCreate(&s2);
    cudaGraph_t g; 
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    cudaStreamCaptureStatus st; unsigned long long id; const cudaGraphNode_t *deps; size_t nd;
    cudaStreamGetCaptureInfo_v2(s, &st, &id, &g, &deps, &nd);
    cudaGraphConditionalHandle h;
    printf("create %d\n", (int)cudaGraphConditionalHandleCreate(&h, g, 0, cudaGraphCondAssignDefault));
    init<<<1,1,0,s>>>(d, h);
    cudaStreamGetCaptureInfo_v2(s, &st, &id, &g, &deps, &nd);
    cudaGraphNodeParams p = {}; p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h; p.conditional.type = cudaGraphCondTypeWhile; p.conditional.size = 1;
    cudaGraphNode_t node;
    printf("addnode %d\n", (int)cudaGraphAddNode(&node, g, deps, nd, &p));
    cudaGraph_t bodyg = p.conditional.phGraph_out[0];
    printf("begin body %d\n", (int)cudaStreamBeginCaptureToGraph(s2, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    body<<<1,1,0,s2>>>(d, h);
    cudaGraph_t tmp; printf("end body %d\n", (int)cudaStreamEndCapture(s2, &tmp));
    printf("update %d\n", (int)cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies));
    cudaMemcpyAsync(hres, d, 4, cudaMemcpyDeviceToHost, s);
    cudaGraph_t full; printf("end %d\n", (int)cudaStreamEndCapture(s, &full));
    cudaGraphExec_t ex; printf("inst %d\n", (int)cudaGraphInstantiate(&ex, full, 0));
    cudaGraphLaunch(ex, s); cudaStreamSynchronize(s);
    printf("ctr=%d err=%s\n", *hres, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
