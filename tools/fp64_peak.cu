// fp64_peak.cu -- FP64 roofline denominators on this B200 (no entry exists in
// MEASURED_PEAKS.json): DMMA (mma.sync m16n8k4 .f64) and DFMA throughput from
// register-resident loops, timed with CUDA events, plus HBM copy bandwidth.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
    double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b0 = a0 * 0.5;
    double d[8][4] = {};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                         : "+d"(d[j][0]), "+d"(d[j][1]), "+d"(d[j][2]), "+d"(d[j][3]) : "d"(a0), "d"(a1), "d"(b0));
    }
    double s = 0;
    for (int j = 0; j < 8; ++j) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
    if (s == 12345.0) out[0] = s;
}

__global__ void dfma_loop(double* out, int iters) {
    double x[8];
    for (int j = 0; j < 8; ++j) x[j] = threadIdx.x + j;
    const double a = 0.999999, b = 1e-7;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, b);
    double s = 0;
    for (int j = 0; j < 8; ++j) s += x[j];
    if (s == 12345.0) out[0] = s;
}

__global__ void copy_k(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out; cudaMalloc(&out, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms;
    // DMMA: per warp-instruction 16*8*4 FMA = 1024 flop
    for (int warps = 4; warps <= 16; warps *= 2) {
        int iters = 20000, blocks = sms * 2;
        dmma_loop<<<blocks, warps * 32>>>(out, 100);
        cudaEventRecord(e0); dmma_loop<<<blocks, warps * 32>>>(out, iters); cudaEventRecord(e1);
        cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        double flops = double(blocks) * warps * iters * 8 * 1024.0;
        printf("{\"kind\":\"dmma_m16n8k4\",\"warps_per_cta\":%d,\"tflops\":%.2f}\n", warps, flops / ms / 1e9);
    }
    for (int threads = 256; threads <= 1024; threads *= 2) {
        int iters = 20000, blocks = sms * 4;
        dfma_loop<<<blocks, threads>>>(out, 100);
        cudaEventRecord(e0); dfma_loop<<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
        cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        double flops = double(blocks) * threads * iters * 8 * 2.0;
        printf("{\"kind\":\"dfma\",\"threads\":%d,\"tflops\":%.2f}\n", threads, flops / ms / 1e9);
    }
    size_t n = size_t(1) << 27;  // 2 GiB per buffer (double2)
    double2 *a, *b; cudaMalloc(&a, n * 16); cudaMalloc(&b, n * 16);
    cudaMemset(a, 0, n * 16);
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0); copy_k<<<sms * 8, 512>>>(a, b, n); cudaEventRecord(e1);
        cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("{\"kind\":\"hbm_copy\",\"gbs\":%.1f}\n", 2.0 * n * 16 / best / 1e6);
    printf("{\"err\":\"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
