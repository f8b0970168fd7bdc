// scan.cu -- the step's exclusive scans and the alive compaction (the movement order's
// ascending alive ids, engine.hpp:99-102), as three-pass kernels of this library: per-tile
// sums, one block scanning the tile sums, the tile offsets applied.  Graph-safe: sizes are the
// roster / chunk capacities, counts land in device memory.
#include "internal.cuh"
#include "scan.cuh"

__global__ void __launch_bounds__(FP_SCAN_BLOCK) scan_sums_kernel(const uint32_t* in, uint32_t n, uint32_t* sums) {
    __shared__ uint32_t s_warp[33];
    const uint32_t base = blockIdx.x * FP_SCAN_TILE + threadIdx.x * FP_SCAN_PER;
    uint32_t v = 0;
#pragma unroll
    for (int k = 0; k < FP_SCAN_PER; ++k) v += base + k < n ? in[base + k] : 0u;
    uint32_t total;
    block_scan_excl(v, s_warp, &total);
    if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

// Exclusive scan of the tile sums in place (up to FP_SCAN_SUMS: 8 per thread); the grand total
// to *total_out (when given).
__global__ void __launch_bounds__(FP_SCAN_BLOCK) scan_top_kernel(uint32_t* sums, uint32_t nb,
                                                                  unsigned long long* total_out) {
    __shared__ uint32_t s_warp[33];
    constexpr int PER = FP_SCAN_SUMS / FP_SCAN_BLOCK;
    uint32_t v[PER], t = 0;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const uint32_t i = threadIdx.x * PER + k;
        v[k] = i < nb ? sums[i] : 0u;
        t += v[k];
    }
    uint32_t total;
    uint32_t e = block_scan_excl(t, s_warp, &total);
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const uint32_t i = threadIdx.x * PER + k;
        if (i < nb) sums[i] = e;
        e += v[k];
    }
    if (threadIdx.x == 0 && total_out) *total_out = total;
}

__global__ void __launch_bounds__(FP_SCAN_BLOCK) scan_apply_kernel(const uint32_t* in, uint32_t n, const uint32_t* sums,
                                                                   uint32_t* out) {
    __shared__ uint32_t s_warp[33];
    const uint32_t base = blockIdx.x * FP_SCAN_TILE + threadIdx.x * FP_SCAN_PER;
    uint32_t v[FP_SCAN_PER], t = 0;
#pragma unroll
    for (int k = 0; k < FP_SCAN_PER; ++k) {
        v[k] = base + k < n ? in[base + k] : 0u;
        t += v[k];
    }
    uint32_t total;
    uint32_t e = block_scan_excl(t, s_warp, &total) + sums[blockIdx.x];
#pragma unroll
    for (int k = 0; k < FP_SCAN_PER; ++k) {
        if (base + k < n) out[base + k] = e;
        e += v[k];
    }
}

// Compaction of the alive flags: per-tile counts, then ascending ids written from the offsets.
__global__ void __launch_bounds__(FP_SCAN_BLOCK) select_sums_kernel(const uint8_t* alive, uint32_t n, uint32_t* sums) {
    __shared__ uint32_t s_warp[33];
    const uint32_t base = blockIdx.x * FP_SCAN_TILE + threadIdx.x * FP_SCAN_PER;
    uint32_t v = 0;
#pragma unroll
    for (int k = 0; k < FP_SCAN_PER; ++k) v += (base + k < n && alive[base + k]) ? 1u : 0u;
    uint32_t total;
    block_scan_excl(v, s_warp, &total);
    if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

__global__ void __launch_bounds__(FP_SCAN_BLOCK) select_scatter_kernel(const uint8_t* alive, uint32_t n,
                                                                       const uint32_t* sums, uint32_t* ids) {
    __shared__ uint32_t s_warp[33];
    const uint32_t base = blockIdx.x * FP_SCAN_TILE + threadIdx.x * FP_SCAN_PER;
    uint32_t f = 0, t = 0;
#pragma unroll
    for (int k = 0; k < FP_SCAN_PER; ++k) {
        const bool a = base + k < n && alive[base + k];
        f |= (uint32_t)a << k;
        t += a;
    }
    uint32_t total;
    uint32_t e = block_scan_excl(t, s_warp, &total) + sums[blockIdx.x];
#pragma unroll
    for (int k = 0; k < FP_SCAN_PER; ++k)
        if ((f >> k) & 1u) ids[e++] = base + k;
}

int fp_scan_u32(fp_ctx* ctx, const uint32_t* in, uint32_t* out, uint32_t n, uint32_t* sums, cudaStream_t s) {
    const uint32_t nb = std::max<uint32_t>(1, (n + FP_SCAN_TILE - 1) / FP_SCAN_TILE);
    if (nb > FP_SCAN_SUMS) return fp_fail(ctx, FP_ERUNTIME, "scan: more than 134M elements");
    scan_sums_kernel<<<nb, FP_SCAN_BLOCK, 0, s>>>(in, n, sums);
    FP_LAUNCHED(ctx);
    scan_top_kernel<<<1, FP_SCAN_BLOCK, 0, s>>>(sums, nb, nullptr);
    FP_LAUNCHED(ctx);
    scan_apply_kernel<<<nb, FP_SCAN_BLOCK, 0, s>>>(in, n, sums, out);
    FP_LAUNCHED(ctx);
    return FP_OK;
}

int fp_select_alive(fp_ctx* ctx, const uint8_t* alive, uint32_t n, uint32_t* ids, unsigned long long* count,
                    uint32_t* sums, cudaStream_t s) {
    const uint32_t nb = std::max<uint32_t>(1, (n + FP_SCAN_TILE - 1) / FP_SCAN_TILE);
    if (nb > FP_SCAN_SUMS) return fp_fail(ctx, FP_ERUNTIME, "select: more than 134M agents");
    select_sums_kernel<<<nb, FP_SCAN_BLOCK, 0, s>>>(alive, n, sums);
    FP_LAUNCHED(ctx);
    scan_top_kernel<<<1, FP_SCAN_BLOCK, 0, s>>>(sums, nb, count);
    FP_LAUNCHED(ctx);
    select_scatter_kernel<<<nb, FP_SCAN_BLOCK, 0, s>>>(alive, n, sums, ids);
    FP_LAUNCHED(ctx);
    return FP_OK;
}
