#include <cuda_runtime.h>
#include <cstdio>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)
__global__ void k_front(int* c) { *c += 1; }
__global__ void k_check(int* c, int* b, cudaGraphConditionalHandle hw, cudaGraphConditionalHandle hi) {
    int v = *c;
    cudaGraphSetConditional(hi, (v % 2) ? 1u : 0u);
    cudaGraphSetConditional(hw, v < 10 ? 1u : 0u);
    (void)b;
}
__global__ void k_back(int* b) { *b += 100; }
int main() {
    cudaStream_t s; CK(cudaStreamCreate(&s));
    int* d; CK(cudaMalloc(&d, 8)); CK(cudaMemset(d, 0, 8));
    cudaGraph_t g; CK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle hw, hi;
    CK(cudaGraphConditionalHandleCreate(&hw, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams wp = {}; wp.type = cudaGraphNodeTypeConditional;
    wp.conditional.handle = hw; wp.conditional.type = cudaGraphCondTypeWhile; wp.conditional.size = 1;
    cudaGraphNode_t wn; CK(cudaGraphAddNode(&wn, g, nullptr, 0, &wp));
    cudaGraph_t body = wp.conditional.phGraph_out[0];
    CK(cudaGraphConditionalHandleCreate(&hi, g, 0, cudaGraphCondAssignDefault));
    CK(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    k_front<<<1, 1, 0, s>>>(d);
    k_check<<<1, 1, 0, s>>>(d, d + 1, hw, hi);
    cudaStreamCaptureStatus st; const cudaGraphNode_t* deps; size_t nd; cudaGraph_t cg;
    CK(cudaStreamGetCaptureInfo(s, &st, nullptr, &cg, &deps, &nd));
    cudaGraphNodeParams ip = {}; ip.type = cudaGraphNodeTypeConditional;
    ip.conditional.handle = hi; ip.conditional.type = cudaGraphCondTypeIf; ip.conditional.size = 1;
    cudaGraphNode_t in; CK(cudaGraphAddNode(&in, body, deps, nd, &ip));
    CK(cudaStreamUpdateCaptureDependencies(s, &in, 1, cudaStreamSetCaptureDependencies));
    cudaGraph_t tmp; CK(cudaStreamEndCapture(s, &tmp));
    cudaGraph_t ib = ip.conditional.phGraph_out[0];
    CK(cudaStreamBeginCaptureToGraph(s, ib, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    k_back<<<1, 1, 0, s>>>(d + 1);
    CK(cudaStreamEndCapture(s, &tmp));
    cudaGraphExec_t ex; CK(cudaGraphInstantiate(&ex, g, 0));
    CK(cudaGraphLaunch(ex, s)); CK(cudaStreamSynchronize(s));
    int h[2]; CK(cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost));
    printf("count=%d back=%d (expect 10, 500)\n", h[0], h[1]);
    CK(cudaMemset(d, 0, 8));
    CK(cudaGraphLaunch(ex, s)); CK(cudaStreamSynchronize(s));
    CK(cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost));
    printf("count=%d back=%d (expect 10, 500)\n", h[0], h[1]);
    return 0;
}
