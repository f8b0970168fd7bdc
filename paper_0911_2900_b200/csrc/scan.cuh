// scan.cuh -- block-wide exclusive scan, shared by the step's own scan / compaction kernels
// (scan.cu) and the single-block list builders of bucket.cu.
#pragma once

#include <stdint.h>

#define FP_SCAN_BLOCK 256                        // the per-tile passes: many small CTAs fill every SM
#define FP_SCAN_PER 16                           // elements per thread (four 16-byte loads)
#define FP_SCAN_TILE (FP_SCAN_BLOCK * FP_SCAN_PER)
#define FP_SCAN_TOP 1024                         // the one-block pass over the tile sums
#define FP_SCAN_SUMS 32768                       // tile sums: n <= 32768 * 4096 (134M)

// Block-wide exclusive scan of one value per thread; *total = the block's sum.  s_warp: 33
// words of shared memory.
__device__ __forceinline__ uint32_t block_scan_excl(uint32_t v, uint32_t* s_warp, uint32_t* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t incl = v;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    __syncthreads();  // s_warp free
    if (lane == 31) s_warp[w] = incl;
    __syncthreads();
    if (w == 0) {
        const uint32_t wv = lane < (int)(blockDim.x >> 5) ? s_warp[lane] : 0u;
        uint32_t wi = wv;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += t;
        }
        s_warp[lane] = wi - wv;
        if (lane == 31) s_warp[32] = wi;
    }
    __syncthreads();
    const uint32_t r = s_warp[w] + incl - v;
    *total = s_warp[32];
    return r;
}
