// order.cu -- the movement order: Fisher-Yates over the ascending alive ids, in parallel.
//
// Reference: move_phase (engine.hpp:99-111):
//     order = alive ids ascending; draw = 0
//     for i = n-1 .. 1: r = rng_u64(seed, 2^63, step, draw++); swap(order[i], order[r % (i+1)])
//
// The sequential shuffle is reconstructed exactly without running it.  With j_i = r_i % (i+1),
// position p's final content is fixed by the iterations that target the same slots:
//   * L_q  = ascending list of iterations i >= 1 with j_i = q            (bucketed by target)
//   * nxt(q) = first i in L_q with i > q,  succ(i) = element after i in L_{j_i}
//   * V(s)   = s if nxt(s) is undefined else V(nxt(s))   (content of slot s before iteration s)
//   * A[0]   = V(0);  A[p>=1] = j_p if succ(p) is undefined else V(succ(p))
// A is the final permutation of positions; order[p] = alive_ids[A[p]], rank[order[p]] = p.
// Work is O(n) with counting-sort buckets (expected |L_q| ~ ln(n/q)); chains are short.
// Pinned against the sequential loop by tests (oracle.movement_order, n up to 10^7).
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "internal.cuh"

__global__ void fy_targets_kernel(uint32_t n, uint64_t seed, uint64_t step, uint32_t* j,
                                  uint32_t* cnt) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0 || i >= n) return;
    const uint64_t draw = (uint64_t)(n - 1 - i);
    const uint64_t r = fp_rng_u64(seed, FP_MOVE_ORDER_STREAM, step, draw);
    const uint32_t t = (uint32_t)(r % (uint64_t)(i + 1));
    j[i] = t;
    atomicAdd(&cnt[t], 1u);
}

__global__ void fy_scatter_kernel(uint32_t n, const uint32_t* j, uint32_t* cursor, uint32_t* bucket) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0 || i >= n) return;
    const uint32_t slot = atomicAdd(&cursor[j[i]], 1u);
    bucket[slot] = i;
}

// One thread per target slot q: sort L_q (tiny), link succ, record nxt(q).
__global__ void fy_link_kernel(uint32_t n, const uint32_t* off, const uint32_t* cnt, uint32_t* bucket,
                               uint32_t* succ, uint32_t* nxt) {
    const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const uint32_t o = off[q], c = cnt[q];
    uint32_t* b = bucket + o;
    for (uint32_t k = 1; k < c; ++k) {  // insertion sort
        const uint32_t t = b[k];
        uint32_t m = k;
        while (m > 0 && b[m - 1] > t) {
            b[m] = b[m - 1];
            --m;
        }
        b[m] = t;
    }
    uint32_t first_gt = FP_NONE;
    for (uint32_t k = 0; k < c; ++k) {
        const uint32_t e = b[k];
        succ[e] = (k + 1 < c) ? b[k + 1] : FP_NONE;
        if (first_gt == FP_NONE && e > q) first_gt = e;
    }
    nxt[q] = first_gt;
    if (q == 0) succ[0] = FP_NONE;
}

__global__ void fy_chain_kernel(uint32_t n, const uint32_t* nxt, uint32_t* V) {
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    uint32_t t = s;
    for (;;) {
        const uint32_t u = nxt[t];
        if (u == FP_NONE) break;
        t = u;
    }
    V[s] = t;
}

// A[p] -> out (positions) or, with ids != null, order/rank of agent ids.
__global__ void fy_final_kernel(uint32_t n, const uint32_t* j, const uint32_t* succ, const uint32_t* V,
                                const uint32_t* ids, uint32_t* out, uint32_t* rank) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    uint32_t a;
    if (p == 0) {
        a = V[0];
    } else {
        const uint32_t s = succ[p];
        a = (s == FP_NONE) ? j[p] : V[s];
    }
    if (ids) {
        const uint32_t id = ids[a];
        out[p] = id;
        rank[id] = p;
    } else {
        out[p] = a;
    }
}

__global__ void flag_alive_kernel(uint32_t n, const uint8_t* alive, uint32_t* flags) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) flags[i] = alive[i] ? 1u : 0u;
}

int fp_ensure_temp(fp_ctx* ctx, size_t bytes) {
    if (bytes <= ctx->temp_bytes) return FP_OK;
    if (ctx->d_temp) cudaFree(ctx->d_temp);
    ctx->d_temp = nullptr;
    FP_CUDA(ctx, cudaMalloc(&ctx->d_temp, bytes));
    ctx->temp_bytes = bytes;
    return FP_OK;
}

// Positions permutation A (ids == null) or the id order + ranks, for n entries.
static int fy_run(fp_ctx* ctx, uint32_t n, uint64_t seed, int64_t step, const uint32_t* ids,
                  uint32_t* out, uint32_t* rank) {
    if (n == 0) return FP_OK;
    cudaStream_t s = ctx->stream;
    const unsigned B = 256;
    FP_CUDA(ctx, cudaMemsetAsync(ctx->d_cnt, 0, sizeof(uint32_t) * n, s));
    fy_targets_kernel<<<fp_blocks(n, B), B, 0, s>>>(n, seed, (uint64_t)step, ctx->d_j, ctx->d_cnt);
    FP_LAUNCHED(ctx);
    size_t need = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, need, ctx->d_cnt, ctx->d_off, (int)n, s);
    if (int rc = fp_ensure_temp(ctx, need)) return rc;
    FP_CUDA(ctx, cub::DeviceScan::ExclusiveSum(ctx->d_temp, need, ctx->d_cnt, ctx->d_off, (int)n, s));
    ctx->ctr.kernel_launches++;
    FP_CUDA(ctx, cudaMemcpyAsync(ctx->d_cursor, ctx->d_off, sizeof(uint32_t) * n,
                                 cudaMemcpyDeviceToDevice, s));
    fy_scatter_kernel<<<fp_blocks(n, B), B, 0, s>>>(n, ctx->d_j, ctx->d_cursor, ctx->d_bucket);
    FP_LAUNCHED(ctx);
    fy_link_kernel<<<fp_blocks(n, B), B, 0, s>>>(n, ctx->d_off, ctx->d_cnt, ctx->d_bucket,
                                                 ctx->d_succ, ctx->d_nxt);
    FP_LAUNCHED(ctx);
    fy_chain_kernel<<<fp_blocks(n, B), B, 0, s>>>(n, ctx->d_nxt, ctx->d_V);
    FP_LAUNCHED(ctx);
    fy_final_kernel<<<fp_blocks(n, B), B, 0, s>>>(n, ctx->d_j, ctx->d_succ, ctx->d_V, ids, out, rank);
    FP_LAUNCHED(ctx);
    return FP_OK;
}

int fp_order_positions(fp_ctx* ctx, uint32_t n, uint64_t seed, int64_t step, uint32_t* d_out) {
    return fy_run(ctx, n, seed, step, nullptr, d_out, nullptr);
}

// Alive compaction (ascending ids, engine.hpp:99-102) then the shuffle; leaves
// ctx->d_order (ids in processing order), ctx->d_rank and ctx->n_order.
int fp_order_launch(fp_ctx* ctx, uint64_t seed, int64_t step) {
    cudaStream_t s = ctx->stream;
    const uint32_t n = ctx->n;
    if (n == 0) {
        ctx->n_order = 0;
        return FP_OK;
    }
    // flags into d_cursor (scratch), select into d_alive_ids, count into d_counters[6]
    flag_alive_kernel<<<fp_blocks(n, 256), 256, 0, s>>>(n, ctx->d_alive, ctx->d_cursor);
    FP_LAUNCHED(ctx);
    thrust::counting_iterator<uint32_t> it(0);
    size_t need = 0;
    cub::DeviceSelect::Flagged(nullptr, need, it, ctx->d_cursor, ctx->d_alive_ids,
                               ctx->d_counters + 6, (int)n, s);
    if (int rc = fp_ensure_temp(ctx, need)) return rc;
    FP_CUDA(ctx, cub::DeviceSelect::Flagged(ctx->d_temp, need, it, ctx->d_cursor, ctx->d_alive_ids,
                                            ctx->d_counters + 6, (int)n, s));
    ctx->ctr.kernel_launches++;
    // The alive count is tracked on the host (make_state + motion exits), so no sync here.
    const uint32_t na = (uint32_t)ctx->alive;
    ctx->n_order = na;
    return fy_run(ctx, na, seed, step, ctx->d_alive_ids, ctx->d_order, ctx->d_rank);
}
