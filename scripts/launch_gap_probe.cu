// Back-to-back launch cost of occupancy-sized persistent grids on this B200: a CUDA graph of
// 200 launches of a near-empty kernel (one load + one store per thread), per grid shape.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/launch_gap_probe.cu -o /tmp/gap
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_touch(double *v, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[i] = v[i] * 1.0000001 + 1.0;
}

int main() {
    const int n = 148 * 2048;
    double *v;
    cudaMalloc(&v, sizeof(double) * n);
    cudaMemset(v, 0, sizeof(double) * n);
    cudaStream_t s;
    cudaStreamCreate(&s);
    const int shapes[][2] = {{1184, 256}, {592, 512}, {296, 1024}, {148, 1024}, {148, 256}};
    for (auto &sh : shapes) {
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        for (int k = 0; k < 200; ++k) k_touch<<<sh[0], sh[1], 0, s>>>(v, n);
        cudaStreamEndCapture(s, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaGraphLaunch(ge, s);
        cudaStreamSynchronize(s);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, s);
        for (int r = 0; r < 5; ++r) cudaGraphLaunch(ge, s);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("grid %4d x %4d threads: %.2f us per launch (graph of 200)\n", sh[0], sh[1],
               ms * 1000.0f / 1000.0f);
        cudaGraphExecDestroy(ge);
        cudaGraphDestroy(g);
    }
    return 0;
}
