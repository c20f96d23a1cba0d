// Probe of the TMA tensor-copy path used by k3_residual_tma (exploration).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ CUtensorMap g_map;
__global__ void k(const __grid_constant__ CUtensorMap m, double* out, int variant, int X) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 32 * 8 * 27 * 8);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(1) : "memory");
        if (variant & 1) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        else asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"((variant & 8) ? 32 * 8 * 8 : 32 * 8 * 27 * 8) : "memory");
        asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                     ::"r"(smem_u32(sm)), "l"((variant & 4) ? reinterpret_cast<uint64_t>(&g_map) : reinterpret_cast<uint64_t>(&m)), "r"((variant & 32) ? X : (variant & 2) ? 0 : -1), "r"((variant & 32) ? 36 : (variant & 2) ? 0 : -1), "r"(3), "r"(0), "r"(smem_u32(bar)) : "memory");
    }
    asm volatile("{\n\t.reg .pred p;\nWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(0) : "memory");
    const double* d = reinterpret_cast<const double*>(sm);
    for (int i = threadIdx.x; i < 32 * 8 * 27; i += blockDim.x) out[i] = d[i];
}
int main(int argc, char** argv) {
    int variant = argc > 1 ? atoi(argv[1]) : 1;
    int X = argc > 2 ? atoi(argv[2]) : 40;
    const int N = 40, xp = 48;
    size_t ncs = (size_t)N * N * xp;
    std::vector<double> h(ncs * 27);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
    double *g, *out;
    cudaMalloc(&g, h.size() * 8);
    cudaMalloc(&out, 32 * 8 * 27 * 8);
    cudaMemcpy(g, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                                const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    CUtensorMap m;
    const cuuint64_t dims[4] = {(cuuint64_t)xp, (cuuint64_t)N, (cuuint64_t)N, 27};
    const cuuint64_t strides[3] = {(cuuint64_t)xp * 8, (cuuint64_t)xp * N * 8, ncs * 8};
    const cuuint32_t nq = (variant & 8) ? 1 : 27;
    const cuuint32_t box[4] = {32, 8, 1, nq}, es[4] = {1, 1, 1, 1};
    CUresult r = ((Encode)fn)(&m, (variant & 16) ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_UINT64, 4, g, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d query %d\n", (int)r, (int)q);
    cudaMemcpyToSymbol(g_map, &m, sizeof m);
    int smem = 32 * 8 * 27 * 8 + 16;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<<<1, 256, smem>>>(m, out, variant, X);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    std::vector<double> o(32 * 8 * 27);
    cudaMemcpy(o.data(), out, o.size() * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int qq = 0; qq < 27; ++qq)
        for (int y = 0; y < 8; ++y)
            for (int x = 0; x < 32; ++x) {
                int ox = (variant & 32) ? X : (variant & 2) ? 0 : -1, oy = (variant & 32) ? 36 : (variant & 2) ? 0 : -1;
                int gx = x + ox, gy = y + oy, gz = 3;
                double want = (gx < 0 || gy < 0 || gx >= xp || gy >= N) ? 0.0 : h[qq * ncs + ((size_t)gz * N + gy) * xp + gx];
                if (o[(qq * 8 + y) * 32 + x] != want) ++bad;
            }
    printf("bad %d\n", bad);
    return 0;
}
