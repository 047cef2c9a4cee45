// Bare cooperative grid.sync() cost at the CA engine's launch shape (148 CTAs x
// 512 threads) and smaller CTAs: nvcc -gencode arch=compute_100a,code=sm_100a
// -o gridsync_probe tools/gridsync_probe.cu
#include <cooperative_groups.h>
#include <cstdio>

__global__ void spin(int iters, int* sink) {
    auto g = cooperative_groups::this_grid();
    int acc = 0;
    for (int i = 0; i < iters; ++i) {
        acc += threadIdx.x;
        g.sync();
    }
    if (acc == -1) *sink = acc;
}

int main() {
    int* sink;
    cudaMalloc(&sink, 4);
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    for (int threads : {32, 128, 512, 1024}) {
        for (int iters : {10, 1010}) {
            void* args[] = {&iters, &sink};
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaLaunchCooperativeKernel((void*)spin, nsm, threads, args, 0, 0);  // warm
            cudaDeviceSynchronize();
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel((void*)spin, nsm, threads, args, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("threads %4d iters %4d: %.3f ms total, %s\n", threads, iters, ms, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
