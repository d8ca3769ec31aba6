// Grid-barrier cost on this GPU: cooperative_groups grid.sync() against a
// sense-reversing counter barrier (one red.release + ld.acquire spin).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gridsync_bench tools/gridsync_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, int* sink) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < iters; ++i) g.sync();
    if (threadIdx.x == 0 && blockIdx.x == 0) *sink = iters;
}

__device__ __forceinline__ void bar_arrive_wait(unsigned* count, volatile unsigned* gen, unsigned nblocks, unsigned& my_gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g0 = my_gen;
        __threadfence();
        const unsigned prev = atomicAdd(count, 1u);
        if (prev == nblocks - 1) {
            *count = 0;
            __threadfence();
            atomicExch((unsigned*)gen, g0 + 1);
        } else {
            unsigned v;
            do {
                asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(gen));
            } while (v == g0);
        }
        my_gen = g0 + 1;
    }
    __syncthreads();
}

__global__ void k_custom(int iters, unsigned* count, unsigned* gen, int* sink) {
    unsigned my_gen = 0;
    if (threadIdx.x == 0) my_gen = *(volatile unsigned*)gen;
    for (int i = 0; i < iters; ++i) bar_arrive_wait(count, gen, gridDim.x, my_gen);
    if (threadIdx.x == 0 && blockIdx.x == 0) *sink = iters;
}

int main() {
    int dev = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int* sink;
    unsigned *cnt, *gen;
    cudaMalloc(&sink, 4);
    cudaMalloc(&cnt, 4);
    cudaMalloc(&gen, 4);
    cudaMemset(cnt, 0, 4);
    cudaMemset(gen, 0, 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int threads : {128, 256, 512}) {
        for (int grid : {38, 74, sms}) {
            int iters = 20000;
            void* args1[] = {&iters, &sink};
            cudaLaunchCooperativeKernel((void*)k_cg, grid, threads, args1, 0, 0);
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel((void*)k_cg, grid, threads, args1, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms1;
            cudaEventElapsedTime(&ms1, a, b);
            void* args2[] = {&iters, &cnt, &gen, &sink};
            cudaLaunchCooperativeKernel((void*)k_custom, grid, threads, args2, 0, 0);
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel((void*)k_custom, grid, threads, args2, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms2;
            cudaEventElapsedTime(&ms2, a, b);
            printf("threads %d grid %d: cg %.3f us/sync, custom %.3f us/sync (%s)\n", threads, grid,
                   1e3 * ms1 / iters, 1e3 * ms2 / iters, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
