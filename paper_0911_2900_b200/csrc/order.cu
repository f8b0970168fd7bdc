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
// The alive count comes from device memory, so the whole sequence is graph-capturable.
// Pinned against the sequential loop by tests (oracle.movement_order, n up to 10^7).
#include "internal.cuh"
#include "scan.cuh"

#ifndef FP_ORDER_SELECT_BESIDE
#define FP_ORDER_SELECT_BESIDE 1  // alive compaction on its own branch beside the shuffle
#endif
#ifndef FP_ORDER_CTAS_PER_SM
#define FP_ORDER_CTAS_PER_SM 8  // grid of the order's grid-stride kernels (per SM)
#endif
#define GS_LOOP(i, n) for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < (n); i += gridDim.x * blockDim.x)

__global__ void fy_targets_kernel(const unsigned long long* pn, uint64_t seed, const long long* pstep, uint32_t* j,
                                  uint32_t* cnt) {
    FP_PDL_WAIT();
    const uint32_t n = (uint32_t)*pn;
    const uint64_t step = (uint64_t)*pstep;
    GS_LOOP(i, n) {
        if (i == 0) continue;
        const uint64_t r = fp_rng_u64(seed, FP_MOVE_ORDER_STREAM, step, (uint64_t)(n - 1 - i));
        const uint32_t t = (uint32_t)(r % (uint64_t)(i + 1));
        j[i] = t;
        atomicAdd(&cnt[t], 1u);
    }
}

__global__ void fy_scatter_kernel(const unsigned long long* pn, const uint32_t* j, uint32_t* cursor,
                                  const uint32_t* off, uint32_t* bucket) {
    FP_PDL_WAIT();
    const uint32_t n = (uint32_t)*pn;
    GS_LOOP(i, n) {
        if (i == 0) continue;
        const uint32_t t = j[i];
        const uint32_t slot = off[t] + atomicAdd(&cursor[t], 1u);
        bucket[slot] = i;
    }
}

// One thread per target slot q: sort L_q (tiny), link succ, record nxt(q).
__global__ void fy_link_kernel(const unsigned long long* pn, const uint32_t* off, const uint32_t* cnt,
                               uint32_t* bucket, uint32_t* succ, uint32_t* nxt) {
    FP_PDL_WAIT();
    const uint32_t n = (uint32_t)*pn;
    GS_LOOP(q, n) {
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
    }
}

__global__ void fy_chain_kernel(const unsigned long long* pn, const uint32_t* nxt, uint32_t* V) {
    FP_PDL_WAIT();
    const uint32_t n = (uint32_t)*pn;
    GS_LOOP(s, n) {
        uint32_t t = s;
        for (;;) {
            const uint32_t u = nxt[t];
            if (u == FP_NONE) break;
            t = u;
        }
        V[s] = t;
    }
}

// A[p] -> out (positions) or, with ids != null, order/rank of agent ids.
// Also zeroes the target counters and cursors of slot p for the next shuffle (every target of
// this one is < n; fy_run starts from zero arrays without a memset).
__global__ void fy_final_kernel(const unsigned long long* pn, const uint32_t* j, const uint32_t* succ,
                                const uint32_t* V, const uint32_t* ids, uint32_t* out, uint32_t* rank,
                                uint32_t* cnt, uint32_t* cursor) {
    FP_PDL_WAIT();
    const uint32_t n = (uint32_t)*pn;
    GS_LOOP(p, n) {
        cnt[p] = 0;
        cursor[p] = 0;
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
}

int fp_ensure_temp(fp_ctx* ctx, size_t bytes) {
    if (bytes <= ctx->temp_bytes) return FP_OK;
    if (ctx->d_temp) {
        cudaStreamSynchronize(ctx->stream);
        if (ctx->stream2) cudaStreamSynchronize(ctx->stream2);
        cudaFree(ctx->d_temp);
    }
    ctx->d_temp = nullptr;
    bytes = std::max<size_t>(bytes, (size_t)1 << 20);
    FP_CUDA(ctx, cudaMalloc(&ctx->d_temp, bytes));
    ctx->temp_bytes = bytes;
    ctx->graph_valid = false;
    return FP_OK;
}

// Positions permutation A (ids == null) or the id order + ranks; n_dev holds the count,
// cap bounds it (sizes the scan).  Uses d_temp + its second half for scratch.
static int fy_run(fp_ctx* ctx, cudaStream_t s, const unsigned long long* n_dev, uint32_t cap, uint64_t seed,
                  const long long* step_dev, const uint32_t* ids, uint32_t* out, uint32_t* rank,
                  cudaEvent_t wait_before_final = nullptr) {
    if (cap == 0) return FP_OK;
    const unsigned G = (unsigned)std::min<size_t>(fp_blocks(cap, 256), (size_t)ctx->sm_count * FP_ORDER_CTAS_PER_SM);
    // d_cnt / d_cursor are zero here: zeroed at allocation, re-zeroed by fy_final_kernel and by
    // the exits sort that borrows d_cnt (move.cu fp_exits_finish)
    fp_launch(fy_targets_kernel, G, 256, 0, s, n_dev, seed, step_dev, ctx->d_j, ctx->d_cnt);
    FP_LAUNCHED(ctx);
    if (int rc = fp_scan_u32(ctx, ctx->d_cnt, ctx->d_off, cap, ctx->d_scan_sums2, s)) return rc;
    fp_launch(fy_scatter_kernel, G, 256, 0, s, n_dev, ctx->d_j, ctx->d_cursor, ctx->d_off, ctx->d_fy_bucket);
    FP_LAUNCHED(ctx);
    fp_launch(fy_link_kernel, G, 256, 0, s, n_dev, ctx->d_off, ctx->d_cnt, ctx->d_fy_bucket, ctx->d_succ, ctx->d_nxt);
    FP_LAUNCHED(ctx);
    fp_launch(fy_chain_kernel, G, 256, 0, s, n_dev, ctx->d_nxt, ctx->d_V);
    FP_LAUNCHED(ctx);
    if (wait_before_final) FP_CUDA(ctx, cudaStreamWaitEvent(s, wait_before_final, 0));  // ids ready
    fp_launch(fy_final_kernel, G, 256, 0, s, n_dev, ctx->d_j, ctx->d_succ, ctx->d_V, ids, out, rank, ctx->d_cnt,
                                      ctx->d_cursor);
    FP_LAUNCHED(ctx);
    return FP_OK;
}

// Reserves the order stage's scratch (outside any graph capture).
int fp_order_reserve(fp_ctx* ctx) {
    const uint32_t n = std::max<uint32_t>(ctx->n, 1);
    if (ctx->order_reserved_n == n && ctx->d_scan_sums2 && ctx->d_scan_sums3) return FP_OK;
    if (!ctx->d_scan_sums2) FP_CUDA(ctx, cudaMalloc(&ctx->d_scan_sums2, FP_SCAN_SUMS * 4));
    if (!ctx->d_scan_sums3) FP_CUDA(ctx, cudaMalloc(&ctx->d_scan_sums3, FP_SCAN_SUMS * 4));
    ctx->order_reserved_n = n;
    return FP_OK;
}

int fp_order_positions(fp_ctx* ctx, uint32_t n, uint64_t seed, int64_t step, uint32_t* d_out) {
    if (int rc = fp_order_reserve(ctx)) return rc;
    unsigned long long hn = n;
    long long hs = step;
    FP_CUDA(ctx, cudaMemcpy(&ctx->d_sc->n_alive, &hn, 8, cudaMemcpyHostToDevice));
    FP_CUDA(ctx, cudaMemcpy(&ctx->d_sc->step, &hs, 8, cudaMemcpyHostToDevice));
    return fy_run(ctx, ctx->stream, &ctx->d_sc->n_alive, n, seed, &ctx->d_sc->step, nullptr, d_out, nullptr);
}

// Alive compaction (ascending ids, engine.hpp:99-102) then the shuffle on stream s; leaves
// ctx->d_order (ids in processing order), ctx->d_rank and d_sc->n_alive.
int fp_order_launch(fp_ctx* ctx, uint64_t seed, cudaStream_t s) {
    const uint32_t n = ctx->n;
    if (n == 0) return FP_OK;
#ifndef FP_STAGE_BUCKET
    FP_STAMP(ctx, s, 4);
#endif
    if (!ctx->st.on && FP_ORDER_SELECT_BESIDE) {
        // the shuffle's positions depend only on the alive count, which the device already
        // holds (DevScalars::alive): the compaction of the alive ids runs beside it and joins
        // before the ids are mapped (fy_final_kernel)
        FP_CUDA(ctx, cudaEventRecord(ctx->ev_sfork, s));
        FP_CUDA(ctx, cudaStreamWaitEvent(ctx->stream4, ctx->ev_sfork, 0));
        if (int rc = fp_select_alive(ctx, ctx->d_alive, n, ctx->d_alive_ids, &ctx->d_sc->n_alive, ctx->d_scan_sums3,
                                     ctx->stream4))
            return rc;
        FP_CUDA(ctx, cudaEventRecord(ctx->ev_sjoin, ctx->stream4));
        const int rc = fy_run(ctx, s, &ctx->d_sc->alive, n, seed, &ctx->d_sc->step, ctx->d_alive_ids, ctx->d_order,
                              ctx->d_rank, ctx->ev_sjoin);
#ifndef FP_STAGE_BUCKET
        FP_STAMP(ctx, s, 6);
#endif
        return rc;
    }
    if (int rc = fp_select_alive(ctx, ctx->d_alive, n, ctx->d_alive_ids, &ctx->d_sc->n_alive, ctx->d_scan_sums2, s))
        return rc;
#ifndef FP_STAGE_BUCKET
    FP_STAMP(ctx, s, 5);
#endif
    const int rc = fy_run(ctx, s, &ctx->d_sc->n_alive, n, seed, &ctx->d_sc->step, ctx->d_alive_ids, ctx->d_order,
                          ctx->d_rank);
#ifndef FP_STAGE_BUCKET
    FP_STAMP(ctx, s, 6);
#endif
    return rc;
}
