// Micro-benchmark: cost of cg::grid_group::sync() in a cooperative launch at the motion kernel's
// shape (2 x 512-thread CTAs per SM), and of a hand-rolled sense-reversal barrier.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_sync(int iters, unsigned long long* t) {
    cg::grid_group g = cg::this_grid();
    unsigned long long t0;
    if (g.thread_rank() == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int i = 0; i < iters; ++i) g.sync();
    if (g.thread_rank() == 0) {
        unsigned long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        *t = t1 - t0;
    }
}

__device__ unsigned int g_bar_count = 0;
__device__ volatile unsigned int g_bar_gen = 0;
__device__ __forceinline__ void my_sync(unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned gen = g_bar_gen;
        __threadfence();
        if (atomicAdd(&g_bar_count, 1u) == nblocks - 1) {
            g_bar_count = 0;
            __threadfence();
            g_bar_gen = gen + 1;
        } else {
            while (g_bar_gen == gen) {}
        }
        __threadfence();
    }
    __syncthreads();
}
__global__ void k_mysync(int iters, unsigned long long* t) {
    unsigned long long t0;
    if (blockIdx.x == 0 && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int i = 0; i < iters; ++i) my_sync(gridDim.x);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        *t = t1 - t0;
    }
}

int main() {
    int sm;
    cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* d;
    cudaMalloc(&d, 8);
    for (int per = 1; per <= 2; ++per) {
        for (int which = 0; which < 2; ++which) {
            int iters = 1000;
            void* args[] = {&iters, &d};
            cudaLaunchCooperativeKernel(which ? (void*)k_mysync : (void*)k_sync, sm * per, 512, args, 0, 0);
            cudaLaunchCooperativeKernel(which ? (void*)k_mysync : (void*)k_sync, sm * per, 512, args, 0, 0);
            cudaDeviceSynchronize();
            unsigned long long h;
            cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
            printf("%s blocks=%d: %.2f us per barrier (%s)\n", which ? "hand-rolled" : "grid.sync", sm * per,
                   h / 1000.0 / iters, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
