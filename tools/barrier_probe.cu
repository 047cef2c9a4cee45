// Grid-barrier variants at the CA engine's launch shape (148 CTAs x 512
// threads, one per SM), per-barrier cost from the slope of 10 vs 1010 barriers:
//   cg      cooperative_groups::this_grid().sync()
//   flags   every CTA stores its epoch to its own 128-byte slot (st.release),
//           warp 0 of every CTA polls all slots (lane l: slots l, l+32, ...)
//           with ld.acquire until each shows the epoch: no atomics
//   tree    arrive: atomicAdd (release) on one of 8 group counters; the last
//           arriver of a group bumps the root; everyone polls the root epoch
// nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/barrier_probe tools/barrier_probe.cu
#include <cooperative_groups.h>
#include <cstdio>

__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__global__ void k_cg(int iters, unsigned*) {
    auto g = cooperative_groups::this_grid();
    for (int i = 0; i < iters; ++i) g.sync();
}

__global__ void k_flags(int iters, unsigned* slots) {
    const int n = gridDim.x;
    for (int i = 1; i <= iters; ++i) {
        __syncthreads();
        if (threadIdx.x == 0) st_release(slots + 32 * blockIdx.x, unsigned(i));
        if (threadIdx.x < 32) {
            bool done = false;
            while (!done) {  // one sweep = independent loads, ~one round trip
                done = true;
                for (int s = threadIdx.x; s < n; s += 32) done &= ld_acquire(slots + 32 * s) >= unsigned(i);
                done = __all_sync(0xffffffffu, done);
            }
        }
        __syncthreads();
    }
}

__global__ void k_tree(int iters, unsigned* ctr) {
    // ctr[0] root epoch, ctr[32 * (1 + g)] group counters (monotone)
    const int n = gridDim.x, G = 8;
    const int grp = blockIdx.x % G;
    const int gsize = n / G + (grp < n % G ? 1 : 0);
    for (int i = 1; i <= iters; ++i) {
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            const unsigned old = atomicAdd(ctr + 32 * (1 + grp), 1u);
            if (old + 1 == unsigned(i) * gsize) atomicAdd(ctr, 1u);  // last of its group
            while (ld_acquire(ctr) < unsigned(i) * G) {
            }
        }
        __syncthreads();
    }
}

// the cooperative-groups algorithm (one arrival counter, the master's flip bit)
// with a nanosleep back-off in the poll: the polling warp stops competing for
// issue slots with co-resident CTAs that are still computing
template <int NS>
__global__ void k_cgsleep(int iters, unsigned* ctr) {
    const unsigned expected = gridDim.x;
    for (int i = 0; i < iters; ++i) {
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned nb = blockIdx.x == 0 ? 0x80000000u - (expected - 1) : 1u;
            __threadfence();
            const unsigned old = atomicAdd(ctr, nb);
            while (((old ^ ld_acquire(ctr)) & 0x80000000u) == 0) {
                if (NS > 0) __nanosleep(NS);
            }
        }
        __syncthreads();
    }
}

int main() {
    unsigned* buf;
    cudaMalloc(&buf, 1 << 20);
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const char* names[7] = {"cg", "flags", "tree", "cgs0", "cgs32", "cgs100", "cgs250"};
    void* fns[7] = {(void*)k_cg, (void*)k_flags, (void*)k_tree, (void*)k_cgsleep<0>, (void*)k_cgsleep<32>,
                    (void*)k_cgsleep<100>, (void*)k_cgsleep<250>};
    for (int v = 0; v < 7; ++v) {
        float t[2];
        int its[2] = {10, 1010};
        for (int k = 0; k < 2; ++k) {
            cudaMemset(buf, 0, 1 << 20);
            int iters = its[k];
            void* args[] = {&iters, &buf};
            cudaLaunchCooperativeKernel(fns[v], nsm, 512, args, 0, 0);  // warm
            cudaDeviceSynchronize();
            cudaMemset(buf, 0, 1 << 20);
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel(fns[v], nsm, 512, args, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&t[k], a, b);
        }
        printf("%-6s %.3f us per barrier (%s)\n", names[v], (t[1] - t[0]) * 1000.0f / 1000.0f,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
