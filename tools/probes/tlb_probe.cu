// Latency / throughput of random 4-byte loads over buffers of growing size (TLB reach).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void chase(const uint32_t* buf, size_t n_words, int steps, unsigned long long* out) {
    // each thread follows its own pseudo-random sequence of dependent loads
    uint64_t s = blockIdx.x * blockDim.x + threadIdx.x + 1;
    uint32_t acc = 0;
    for (int i = 0; i < steps; ++i) {
        s = s * 6364136223846793005ull + 1442695040888963407ull + acc;
        const size_t k = (s >> 17) % n_words;
        acc = __ldcg(&buf[k]) & 1u;  // dependent chain
    }
    if (acc == 12345) out[0] = acc;
}

int main() {
    int sm;
    cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, 0);
    const size_t maxb = (size_t)4 << 30;
    uint32_t* buf;
    cudaMalloc(&buf, maxb);
    cudaMemset(buf, 0, maxb);
    unsigned long long* out;
    cudaMalloc(&out, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (size_t mb : {16, 64, 128, 256, 512, 1024, 2048, 4096}) {
        const size_t words = mb * (1 << 20) / 4;
        for (int threads_per_sm : {32, 1024}) {
            const int steps = 64;
            chase<<<sm, threads_per_sm>>>(buf, words, steps, out);
            cudaEventRecord(e0);
            chase<<<sm, threads_per_sm>>>(buf, words, steps, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double loads = (double)sm * threads_per_sm * steps;
            printf("%5zu MB, %4d thr/SM: %.3f us per dependent load, %.1f G loads/s\n", mb, threads_per_sm,
                   ms * 1e3 / steps, loads / (ms * 1e-3) / 1e9);
        }
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
