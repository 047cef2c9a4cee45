// Probe of 1-D u8 TMA boxes (the fused CA step's halo rows):
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tma1d_probe tools/tma1d_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE, int DIM2 = 0>
__global__ void probe(const __grid_constant__ CUtensorMap tmap, int base, uint8_t* out) {
    __shared__ __align__(1024) uint8_t buf[32 * 144];
    __shared__ __align__(8) uint64_t mbar;
    const uint32_t mb = smem_u32(&mbar);
    const int lane = threadIdx.x;
    if (lane == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(mb), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    __syncwarp();
    const int n = MODE == 0 ? 1 : 32;
    if (MODE == 2 && lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb), "r"(n * 128) : "memory");
    if (lane < n) {
        const int c0 = base + 48 * lane - 16;  // 16-byte aligned starts (incl. -16)
        if (DIM2)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
                    smem_u32(buf + 144 * lane)),
                "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(c0), "r"(0), "r"(mb)
                : "memory");
        else
            asm volatile(
                "cp.async.bulk.tensor.1d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];\n" ::"r"(
                    smem_u32(buf + 144 * lane)),
                "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(c0), "r"(mb)
                : "memory");
    }
    __syncwarp();
    if (MODE != 2 && lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb), "r"(n * 128) : "memory");
    uint32_t ok = 0;
    while (!ok) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(mb), "r"(0)
            : "memory");
    }
    for (int l = 0; l < n; ++l) for (int i = lane; i < 128; i += 32) out[l * 128 + i] = buf[l * 144 + i];
}

int main() {
    const size_t N = 100000;
    std::vector<uint8_t> h(N);
    for (size_t i = 0; i < N; ++i) h[i] = uint8_t(i * 7 + 3);
    uint8_t *d, *o;
    cudaMalloc(&d, N);
    cudaMalloc(&o, 32 * 128);
    cudaMemcpy(d, h.data(), N, cudaMemcpyHostToDevice);
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    auto fn = (PFN_cuTensorMapEncodeTiled_v12000)fp;
    for (int variant = 0; variant < 3; ++variant) {
        CUtensorMap m;
        CUresult cr;
        if (variant == 0) {  // 1-D u8
            cuuint64_t dims[1] = {cuuint64_t(N)};
            cuuint64_t str[1] = {cuuint64_t(N)};
            cuuint32_t bx[1] = {128u};
            cuuint32_t es[1] = {1};
            cr = fn(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, d, dims, str, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        } else {  // 2-D u8 (N x 1), box 128 x 1
            cuuint64_t dims[2] = {cuuint64_t(N), 1};
            cuuint64_t str[1] = {cuuint64_t((N + 15) / 16 * 16)};
            cuuint32_t bx[2] = {128u, 1u};
            cuuint32_t es[2] = {1, 1};
            cr = fn(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, d, dims, str, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, variant == 1 ? CU_TENSOR_MAP_L2_PROMOTION_NONE : CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        }
        printf("variant %d encode rc=%d\n", variant, int(cr));
        for (int mode = 0; mode < 3; ++mode) {
            for (int base : {16, 1024, int(N) / 16 * 16 - 96, 0}) {
                if (variant == 0) {
                    if (mode == 0) probe<0><<<1, 32>>>(m, base, o);
                    else if (mode == 1) probe<1><<<1, 32>>>(m, base, o);
                    else probe<2><<<1, 32>>>(m, base, o);
                } else {
                    if (mode == 0) probe<0, 1><<<1, 32>>>(m, base, o);
                    else if (mode == 1) probe<1, 1><<<1, 32>>>(m, base, o);
                    else probe<2, 1><<<1, 32>>>(m, base, o);
                }
                cudaError_t e = cudaDeviceSynchronize();
                std::vector<uint8_t> r(32 * 128);
                cudaMemcpy(r.data(), o, r.size(), cudaMemcpyDeviceToHost);
                int bad = 0;
                const int n = mode == 0 ? 1 : 32;
                for (int l = 0; l < n; ++l)
                    for (int i = 0; i < 128; ++i) {
                        long long src = (long long)base + 48 * l - 16 + i;
                        uint8_t want = (src >= 0 && src < (long long)N) ? h[src] : 0;
                        bad += r[l * 128 + i] != want;
                    }
                printf("variant %d mode %d base %d: %s bad=%d\n", variant, mode, base, cudaGetErrorString(e), bad);
                if (e != cudaSuccess) return 1;
            }
        }
    }
    return 0;
}
