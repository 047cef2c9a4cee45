// Standalone probe of the 2-D TMA tensor-box load used by k_ca_bits
// (nvcc -gencode arch=compute_100a,code=sm_100a -o tma_probe tools/tma_probe.cu -lcuda).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap tmap, int c0, int c1, uint32_t* out, int rows) {
    __shared__ __align__(128) uint32_t buf[16 * 8];
    __shared__ __align__(8) uint64_t mbar;
    const uint32_t mb = smem_u32(&mbar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(mb), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb), "r"(rows * 32) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
                smem_u32(buf)),
            "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(c0), "r"(c1), "r"(mb)
            : "memory");
    }
    uint32_t ok = 0;
    while (!ok) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(mb), "r"(0)
            : "memory");
    }
    for (int i = threadIdx.x; i < rows * 8; i += blockDim.x) out[i] = buf[i];
}

int main(int argc, char** argv) {
    const int WP = argc > 1 ? atoi(argv[1]) : 8, R = argc > 2 ? atoi(argv[2]) : 100, box = argc > 3 ? atoi(argv[3]) : 6;
    std::vector<uint32_t> h(size_t(WP) * R);
    for (size_t i = 0; i < h.size(); ++i) h[i] = uint32_t(i);
    uint32_t *d, *o;
    cudaMalloc(&d, h.size() * 4);
    cudaMalloc(&o, 16 * 8 * 4);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    auto fn = (PFN_cuTensorMapEncodeTiled_v12000)fp;
    CUtensorMap m;
    cuuint64_t dims[2] = {cuuint64_t(WP), cuuint64_t(R)};
    cuuint64_t str[1] = {cuuint64_t(WP) * 4};
    cuuint32_t bx[2] = {8u, cuuint32_t(box)};
    cuuint32_t es[2] = {1, 1};
    CUresult cr = fn(&m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, d, dims, str, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode rc=%d WP=%d R=%d box=%d\n", int(cr), WP, R, box);
    int coords[][2] = {{0, 0}, {0, -1}, {4, 3}, {-4, 0}, {-4, -1}, {WP - 4, R - 2}, {0, R + 3}, {-8, 5}, {2, 0}, {1, 0}};
    for (auto& c : coords) {
        probe<<<1, 32>>>(m, c[0], c[1], o, box);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<uint32_t> r(size_t(box) * 8);
        cudaMemcpy(r.data(), o, r.size() * 4, cudaMemcpyDeviceToHost);
        printf("coords (%d,%d): %s  row0: %u %u %u %u %u %u %u %u\n", c[0], c[1], cudaGetErrorString(e), r[0], r[1],
               r[2], r[3], r[4], r[5], r[6], r[7]);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
