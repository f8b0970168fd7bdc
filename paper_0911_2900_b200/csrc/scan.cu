// scan.cu -- the step's exclusive scans and the alive compaction (the movement order's
// ascending alive ids, engine.hpp:99-102), as three-pass kernels of this library: per-tile
// sums, one block scanning the tile sums, the tile offsets applied.  Graph-safe: sizes are the
// roster / chunk capacities, counts land in device memory.
#include "internal.cuh"
#include "scan.cuh"

// FP_SCAN_PER consecutive words of `in` from element base (16-byte loads when the run is whole).
__device__ __forceinline__ void load_run(const uint32_t* in, uint32_t n, uint32_t base, uint32_t* v) {
    if (base + FP_SCAN_PER <= n) {
#pragma unroll
        for (int q = 0; q < FP_SCAN_PER / 4; ++q) {
            const uint4 u = __ldg(reinterpret_cast<const uint4*>(in + base) + q);
            v[4 * q] = u.x;
            v[4 * q + 1] = u.y;
            v[4 * q + 2] = u.z;
            v[4 * q + 3] = u.w;
        }
    } else {
#pragma unroll
        for (int k = 0; k < FP_SCAN_PER; ++k) v[k] = base + k < n ? in[base + k] : 0u;
    }
}

// FP_SCAN_PER consecutive alive flags as a bit mask.
__device__ __forceinline__ uint32_t load_flags(const uint8_t* alive, uint32_t n, uint32_t base) {
    uint32_t f = 0;
    if (base + FP_SCAN_PER <= n) {
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(alive + base));
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int k = 0; k < FP_SCAN_PER; ++k) f |= (((w[k >> 2] >> (8 * (k & 3))) & 0xFFu) != 0u ? 1u : 0u) << k;
    } else {
#pragma unroll
        for (int k = 0; k < FP_SCAN_PER; ++k) f |= (base + k < n && alive[base + k] ? 1u : 0u) << k;
    }
    return f;
}

__global__ void __launch_bounds__(FP_SCAN_BLOCK) scan_sums_kernel(const uint32_t* in, uint32_t n, uint32_t* sums) {
    FP_PDL_WAIT();
    __shared__ uint32_t s_warp[33];
    uint32_t v[FP_SCAN_PER], t = 0;
    load_run(in, n, blockIdx.x * FP_SCAN_TILE + threadIdx.x * FP_SCAN_PER, v);
#pragma unroll
    for (int k = 0; k < FP_SCAN_PER; ++k) t += v[k];
    uint32_t total;
    block_scan_excl(t, s_warp, &total);
    if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

// Exclusive scan of the tile sums in place (up to FP_SCAN_SUMS: FP_SCAN_SUMS / FP_SCAN_TOP
// per thread); the grand total to *total_out (when given).
__global__ void __launch_bounds__(FP_SCAN_TOP) scan_top_kernel(uint32_t* sums, uint32_t nb,
                                                               unsigned long long* total_out) {
    FP_PDL_WAIT();
    __shared__ uint32_t s_warp[33];
    constexpr int PER = FP_SCAN_SUMS / FP_SCAN_TOP;
    const uint32_t per = (nb + FP_SCAN_TOP - 1) / FP_SCAN_TOP;  // <= PER
    uint32_t t = 0;
    for (uint32_t k = 0; k < per; ++k) {
        const uint32_t i = threadIdx.x * per + k;
        t += i < nb ? sums[i] : 0u;
    }
    uint32_t total;
    uint32_t e = block_scan_excl(t, s_warp, &total);
    for (uint32_t k = 0; k < per; ++k) {
        const uint32_t i = threadIdx.x * per + k;
        if (i < nb) {
            const uint32_t v = sums[i];
            sums[i] = e;
            e += v;
        }
    }
    (void)PER;
    if (threadIdx.x == 0 && total_out) *total_out = total;
}

__global__ void __launch_bounds__(FP_SCAN_BLOCK) scan_apply_kernel(const uint32_t* in, uint32_t n, const uint32_t* sums,
                                                                   uint32_t* out) {
    FP_PDL_WAIT();
    __shared__ uint32_t s_warp[33];
    const uint32_t base = blockIdx.x * FP_SCAN_TILE + threadIdx.x * FP_SCAN_PER;
    uint32_t v[FP_SCAN_PER], t = 0;
    load_run(in, n, base, v);
#pragma unroll
    for (int k = 0; k < FP_SCAN_PER; ++k) t += v[k];
    uint32_t total;
    uint32_t e = block_scan_excl(t, s_warp, &total) + sums[blockIdx.x];
    uint32_t o[FP_SCAN_PER];
#pragma unroll
    for (int k = 0; k < FP_SCAN_PER; ++k) {
        o[k] = e;
        e += v[k];
    }
    if (base + FP_SCAN_PER <= n) {
#pragma unroll
        for (int q = 0; q < FP_SCAN_PER / 4; ++q)
            reinterpret_cast<uint4*>(out + base)[q] = make_uint4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
    } else {
#pragma unroll
        for (int k = 0; k < FP_SCAN_PER; ++k)
            if (base + k < n) out[base + k] = o[k];
    }
}

// Compaction of the alive flags: per-tile counts, then ascending ids written from the offsets.
__global__ void __launch_bounds__(FP_SCAN_BLOCK) select_sums_kernel(const uint8_t* alive, uint32_t n, uint32_t* sums) {
    FP_PDL_WAIT();
    __shared__ uint32_t s_warp[33];
    const uint32_t v = __popc(load_flags(alive, n, blockIdx.x * FP_SCAN_TILE + threadIdx.x * FP_SCAN_PER));
    uint32_t total;
    block_scan_excl(v, s_warp, &total);
    if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

__global__ void __launch_bounds__(FP_SCAN_BLOCK) select_scatter_kernel(const uint8_t* alive, uint32_t n,
                                                                       const uint32_t* sums, uint32_t* ids) {
    FP_PDL_WAIT();
    __shared__ uint32_t s_warp[33];
    const uint32_t base = blockIdx.x * FP_SCAN_TILE + threadIdx.x * FP_SCAN_PER;
    uint32_t f = load_flags(alive, n, base);
    uint32_t total;
    uint32_t e = block_scan_excl(__popc(f), s_warp, &total) + sums[blockIdx.x];
    while (f) {
        const int k = __ffs(f) - 1;
        f &= f - 1;
        ids[e++] = base + (uint32_t)k;
    }
}

// One CTA over the whole array in FP_SCAN_TOP * FP_SCAN_PER-element rounds with a running carry:
// one launch instead of three for short arrays (the per-step chunk counts).
#define FP_SCAN_SMALL_ROUND (FP_SCAN_TOP * FP_SCAN_PER)
#define FP_SCAN_SMALL_MAX (16 * FP_SCAN_SMALL_ROUND)
#ifndef FP_SCAN_USE_SMALL
#define FP_SCAN_USE_SMALL 0
#endif
__global__ void __launch_bounds__(FP_SCAN_TOP) scan_small_kernel(const uint32_t* in, uint32_t n, uint32_t* out) {
    FP_PDL_WAIT();
    __shared__ uint32_t s_warp[33];
    uint32_t carry = 0;
    for (uint32_t r0 = 0; r0 < n; r0 += FP_SCAN_SMALL_ROUND) {
        const uint32_t base = r0 + threadIdx.x * FP_SCAN_PER;
        uint32_t v[FP_SCAN_PER], t = 0;
        load_run(in, n, base, v);
#pragma unroll
        for (int k = 0; k < FP_SCAN_PER; ++k) t += v[k];
        uint32_t total;
        uint32_t e = block_scan_excl(t, s_warp, &total) + carry;
        carry += total;
        uint32_t o[FP_SCAN_PER];
#pragma unroll
        for (int k = 0; k < FP_SCAN_PER; ++k) {
            o[k] = e;
            e += v[k];
        }
        if (base + FP_SCAN_PER <= n) {
#pragma unroll
            for (int q = 0; q < FP_SCAN_PER / 4; ++q)
                reinterpret_cast<uint4*>(out + base)[q] = make_uint4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
        } else {
#pragma unroll
            for (int k = 0; k < FP_SCAN_PER; ++k)
                if (base + k < n) out[base + k] = o[k];
        }
    }
}

int fp_scan_u32(fp_ctx* ctx, const uint32_t* in, uint32_t* out, uint32_t n, uint32_t* sums, cudaStream_t s) {
    if (FP_SCAN_USE_SMALL && n <= FP_SCAN_SMALL_MAX) {  // measured slower than the 3-pass scan
        fp_launch(scan_small_kernel, 1, FP_SCAN_TOP, 0, s, in, n, out);
        FP_LAUNCHED(ctx);
        return FP_OK;
    }
    const uint32_t nb = std::max<uint32_t>(1, (n + FP_SCAN_TILE - 1) / FP_SCAN_TILE);
    if (nb > FP_SCAN_SUMS) return fp_fail(ctx, FP_ERUNTIME, "scan: more than 134M elements");
    fp_launch(scan_sums_kernel, nb, FP_SCAN_BLOCK, 0, s, in, n, sums);
    FP_LAUNCHED(ctx);
    fp_launch(scan_top_kernel, 1, FP_SCAN_TOP, 0, s, sums, nb, nullptr);
    FP_LAUNCHED(ctx);
    fp_launch(scan_apply_kernel, nb, FP_SCAN_BLOCK, 0, s, in, n, sums, out);
    FP_LAUNCHED(ctx);
    return FP_OK;
}

int fp_select_alive(fp_ctx* ctx, const uint8_t* alive, uint32_t n, uint32_t* ids, unsigned long long* count,
                    uint32_t* sums, cudaStream_t s) {
    const uint32_t nb = std::max<uint32_t>(1, (n + FP_SCAN_TILE - 1) / FP_SCAN_TILE);
    if (nb > FP_SCAN_SUMS) return fp_fail(ctx, FP_ERUNTIME, "select: more than 134M agents");
    fp_launch(select_sums_kernel, nb, FP_SCAN_BLOCK, 0, s, alive, n, sums);
    FP_LAUNCHED(ctx);
    fp_launch(scan_top_kernel, 1, FP_SCAN_TOP, 0, s, sums, nb, count);
    FP_LAUNCHED(ctx);
    fp_launch(select_scatter_kernel, nb, FP_SCAN_BLOCK, 0, s, alive, n, sums, ids);
    FP_LAUNCHED(ctx);
    return FP_OK;
}
