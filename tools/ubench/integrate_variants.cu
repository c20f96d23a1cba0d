// Micro-benchmark of integration-kernel variants (exploration only; the
// product kernels live in paper_2005_03606_b200/csrc). Sinusoid field, 729^2
// cells, n = 32, EXACT arithmetic, results checked against variant A.
#include <cstdio>
#include <vector>
#include <cmath>
#include "../../paper_2005_03606_b200/csrc/device.cuh"
#include "../../paper_2005_03606_b200/csrc/integrate.cuh"

using namespace lzb;
__global__ void ub_field_parts(lzb_field f, int N, double h, int n, int axis, double* out) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)N * n) return;
    int c = t / n, i = t % n;
    double inv = 1.0 / n, x0 = c * h, x = x0 + (i + 0.5) * inv * h;
    out[t] = axis == 0 ? field_xpart(f, x) : field_ypart(f, x);
}
__global__ void ub_ksub_table(int n, double* ktab) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)n * n) return;
    int i = t / n, j = t % n;
    double inv = 1.0 / n;
    K9 k = ksub(axis_seg(i, inv), axis_seg(j, inv));
    double* o = ktab + t * kKs;
    o[0] = k.k00; o[1] = k.k11; o[2] = k.k22; o[3] = k.k33; o[4] = k.k01;
    o[5] = k.k23; o[6] = k.k02; o[7] = k.k13; o[8] = k.k03; o[9] = 0.0;
}

// Persistent: whole K table resident, contiguous range per block, CPT cells per thread-iteration.
template <int CPT, int MINB>
__global__ void __launch_bounds__(256, MINB) k_res(int N, int n, const double* fx, const double* fy,
                                                  const double* ktab, double* out) {
    extern __shared__ double sm[];
    const int64_t total = (int64_t)N * N;
    const int64_t b0 = blockIdx.x * total / gridDim.x, b1 = (blockIdx.x + 1) * total / gridDim.x;
    for (int v = threadIdx.x; v < n * n * kKs / 2; v += blockDim.x)
        reinterpret_cast<double2*>(sm)[v] = reinterpret_cast<const double2*>(ktab)[v];
    __syncthreads();
    for (int64_t base = b0 + threadIdx.x; base < b1; base += (int64_t)CPT * blockDim.x) {
        double a[CPT][9];
        const double* fxc[CPT];
        const double* fyc[CPT];
        bool act[CPT];
#pragma unroll
        for (int q = 0; q < CPT; ++q) {
            int64_t c = base + q * blockDim.x;
            act[q] = c < b1;
            if (!act[q]) c = base;
            fxc[q] = fx + (c % N) * n;
            fyc[q] = fy + (c / N) * n;
#pragma unroll
            for (int r = 0; r < 9; ++r) a[q][r] = 0.0;
        }
        for (int i = 0; i < n; ++i) {
            double xp[CPT];
#pragma unroll
            for (int q = 0; q < CPT; ++q) xp[q] = fxc[q][i];
            const double2* kp = reinterpret_cast<const double2*>(sm + (size_t)i * n * kKs);
#pragma unroll 2
            for (int j = 0; j < n; ++j, kp += kKs / 2) {
                const double2 k0 = kp[0], k1 = kp[1], k2 = kp[2], k3 = kp[3], k4 = kp[4];
#pragma unroll
                for (int q = 0; q < CPT; ++q) {
                    const double e = 1.0 + xp[q] * fyc[q][j];
                    a[q][0] = a[q][0] + k0.x * e; a[q][1] = a[q][1] + k0.y * e;
                    a[q][2] = a[q][2] + k1.x * e; a[q][3] = a[q][3] + k1.y * e;
                    a[q][4] = a[q][4] + k2.x * e; a[q][5] = a[q][5] + k2.y * e;
                    a[q][6] = a[q][6] + k3.x * e; a[q][7] = a[q][7] + k3.y * e;
                    a[q][8] = a[q][8] + k4.x * e;
                }
            }
        }
#pragma unroll
        for (int q = 0; q < CPT; ++q)
            if (act[q]) {
                double* o = out + 9 * (base + q * blockDim.x);
                for (int r = 0; r < 9; ++r) o[r] = a[q][r];
            }
    }
}

template <int CPT, int MINB>
float run(int N, int n, const double* fx, const double* fy, const double* kt, double* out, int sms) {
    size_t smem = (size_t)n * n * kKs * 8;
    cudaFuncSetAttribute(k_res<CPT, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_res<CPT, MINB>, 256, smem);
    int grid = per * sms;
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    k_res<CPT, MINB><<<grid, 256, smem>>>(N, n, fx, fy, kt, out);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) k_res<CPT, MINB><<<grid, 256, smem>>>(N, n, fx, fy, kt, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("CPT=%d MINB=%d blocks/SM=%d grid=%d  %.3f ms  %.1f G samples/s  err=%s\n", CPT, MINB, per, grid,
           ms / 5, (double)N * N * n * n / (ms / 5 * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    return ms / 5;
}

int main() {
    int N = 729, n = 32, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    lzb_field f{}; f.kind = LZB_FIELD_SINUSOID; f.amp = 0.9; f.freq = 6.0; f.value = 1.0;
    double h = std::pow(1.0 / 3, 6);
    double *fx, *fy, *kt, *out;
    cudaMalloc(&fx, N * n * 8); cudaMalloc(&fy, N * n * 8); cudaMalloc(&kt, n * n * kKs * 8);
    cudaMalloc(&out, (size_t)N * N * 9 * 8);
    ub_field_parts<<<(N * n + 255) / 256, 256>>>(f, N, h, n, 0, fx);
    ub_field_parts<<<(N * n + 255) / 256, 256>>>(f, N, h, n, 1, fy);
    ub_ksub_table<<<(n * n + 255) / 256, 256>>>(n, kt);
    cudaDeviceSynchronize();
    run<1, 2>(N, n, fx, fy, kt, out, sms);
    run<1, 3>(N, n, fx, fy, kt, out, sms);
    run<1, 4>(N, n, fx, fy, kt, out, sms);
    run<2, 1>(N, n, fx, fy, kt, out, sms);
    run<2, 2>(N, n, fx, fy, kt, out, sms);
    run<2, 3>(N, n, fx, fy, kt, out, sms);
    run<3, 1>(N, n, fx, fy, kt, out, sms);
    run<3, 2>(N, n, fx, fy, kt, out, sms);
    run<4, 1>(N, n, fx, fy, kt, out, sms);
    return 0;
}
