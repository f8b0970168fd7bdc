// Micro-benchmark: scattered 32-bit atomics on a bitplane the size of the plaza's (12.5 MB),
// 1M "agents" x 6 cells, in the patterns the motion kernel's contention marking uses.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_or_ret(uint32_t* p1, uint32_t* p2, const uint32_t* addr, int n, int per) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        uint32_t old[6];
#pragma unroll
        for (int j = 0; j < 6; ++j) {
            const uint32_t a = addr[i * 6 + j];
            if (j < per) old[j] = atomicOr(&p1[a >> 5], 1u << (a & 31));
        }
#pragma unroll
        for (int j = 0; j < 6; ++j) {
            const uint32_t a = addr[i * 6 + j];
            if (j < per && (old[j] >> (a & 31) & 1u)) atomicOr(&p2[a >> 5], 1u << (a & 31));
        }
    }
}
__global__ void k_red(uint32_t* p1, const uint32_t* addr, int n, int per) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
#pragma unroll
        for (int j = 0; j < 6; ++j) {
            const uint32_t a = addr[i * 6 + j];
            if (j < per) atomicOr(&p1[a >> 5], 1u << (a & 31));
        }
    }
}
__global__ void k_ld(const uint32_t* p1, const uint32_t* addr, int n, uint32_t* out) {
    uint32_t acc = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
#pragma unroll
        for (int j = 0; j < 6; ++j) {
            const uint32_t a = addr[i * 6 + j];
            acc |= __ldcg(&p1[a >> 5]);
        }
    }
    if (acc == 0x12345) out[0] = acc;
}

int main() {
    const int n = 1 << 20;
    const size_t words = 628u * 5000u;
    uint32_t *p1, *p2, *addr, *out;
    cudaMalloc(&p1, words * 4);
    cudaMalloc(&p2, words * 4);
    cudaMalloc(&out, 4);
    cudaMalloc(&addr, (size_t)n * 6 * 4);
    uint32_t* h = (uint32_t*)malloc((size_t)n * 6 * 4);
    // agents spread over the plane; footprint cells within +-5 rows/cols of the agent
    uint64_t s = 1;
    auto rnd = [&]() { s = s * 6364136223846793005ull + 1442695040888963407ull; return (uint32_t)(s >> 33); };
    for (int i = 0; i < n; ++i) {
        const uint32_t x = 40 + rnd() % 19900, y = 6 + rnd() % 4980;
        for (int j = 0; j < 6; ++j) {
            const uint32_t cx = x + (rnd() % 11) - 5, cy = y + (rnd() % 11) - 5;
            h[i * 6 + j] = cy * 628u * 32u + cx;
        }
    }
    for (int sorted = 0; sorted < 2; ++sorted) {
        if (sorted) {  // agents in row-major spatial order (like plan-tile order)
            // crude: sort agents by their first cell
            struct A { uint32_t c[6]; };
            A* v = (A*)h;
            qsort(v, n, sizeof(A), [](const void* a, const void* b) {
                uint32_t x = ((const A*)a)->c[0], y = ((const A*)b)->c[0];
                return x < y ? -1 : x > y;
            });
        }
        cudaMemcpy(addr, h, (size_t)n * 24, cudaMemcpyHostToDevice);
        int sm = 0;
        cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, 0);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        for (int grid_mul = 2; grid_mul <= 8; grid_mul *= 2) {
            float t[3];
            for (int which = 0; which < 3; ++which) {
                float best = 1e9;
                for (int rep = 0; rep < 5; ++rep) {
                    cudaMemset(p1, 0, words * 4);
                    cudaMemset(p2, 0, words * 4);
                    cudaEventRecord(e0);
                    if (which == 0) k_or_ret<<<sm * grid_mul, 512>>>(p1, p2, addr, n, 6);
                    if (which == 1) k_red<<<sm * grid_mul, 512>>>(p1, addr, n, 6);
                    if (which == 2) k_ld<<<sm * grid_mul, 512>>>(p1, addr, n, out);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    best = ms < best ? ms : best;
                }
                t[which] = best * 1000;
            }
            printf("sorted=%d blocks=%dxSM  or+ret %.1f us  red %.1f us  ld %.1f us\n", sorted, grid_mul, t[0], t[1], t[2]);
        }
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
