// bucket.cu -- counting sort of the planned agents by plan chunk (each step).
//
// The plan kernel (plan.cu) sweeps each vertical stripe of the grid (tile_w columns) top to
// bottom through a ring of 8-row chunks staged by TMA, so agents are grouped by chunk in
// stripe-major order: chunk g = stripe * CPS + (y >> 3), CPS = chunks per stripe.  Order inside
// a chunk is irrelevant (planning is a pure per-agent function of the pre-step snapshot,
// planning.hpp:14-17), so atomics are fine.  The motion phase (move.cu) reads the same grouping
// as tiles of tile_w x tile_h (tile_h / 8 consecutive chunks of one stripe).  Outputs:
//   chunk_cnt / chunk_off   agents per chunk and their first position (exclusive scan)
//   bucket / brec           agent id and its planner record (id, x, y, v_max) per position
//   tile_cnt / tile_off     per tile (row-major id), tile_list = the non-empty tiles,
//   items                   motion seed work items (tile-list entry, chunk of SEED_ITEM agents)
//   plan items              the plan kernel's work units: <= PLAN_ITEM_CHUNKS chunks of one
//                           stripe and <= PLAN_ITEM_AGENTS of their agents; 64 B each: (first
//                           chunk, chunks - 1, first agent, end agent) + u16 reference count
//                           per ring slot
// All passes are this file's kernels (no library primitives in the step).
#include "internal.cuh"
#include "scan.cuh"

#ifndef FP_BUCKET_CTAS_PER_SM
#define FP_BUCKET_CTAS_PER_SM 16  // grid of the counting / scatter passes (per SM)
#endif
#ifndef PLAN_ITEM_CHUNKS
#define PLAN_ITEM_CHUNKS 6    // chunks per plan item (plan.cu's ring holds three items of <= 8 slots)
#endif
#ifndef PLAN_ITEM_AGENTS
#define PLAN_ITEM_AGENTS 512  // agents per plan item at most
#endif

__global__ void bucket_count_kernel(Geo g, const int32_t* x, const int32_t* y, const uint8_t* alive,
                                    const uint8_t* owned, uint32_t n, int tile_w, uint32_t cps, uint32_t* cnt,
                                    uint32_t* chunk_of, uint32_t* slot, unsigned long long* n_planned) {
    FP_PDL_WAIT();
    __shared__ unsigned s_taken;  // agents this block takes (one global atomic per block)
    if (threadIdx.x == 0) s_taken = 0;
    __syncthreads();
    for (uint32_t i0 = blockIdx.x * blockDim.x; i0 < n; i0 += gridDim.x * blockDim.x) {
        const uint32_t i = i0 + threadIdx.x;
        const bool take = i < n && alive[i] && (!owned || owned[i]);
        const unsigned b = __ballot_sync(0xffffffffu, take);
        if ((threadIdx.x & 31) == 0 && b) atomicAdd(&s_taken, (unsigned)__popc(b));
        // agents of one warp in the same chunk (dense exit queues) share one counter atomic
        const uint32_t c = take ? (uint32_t)(g.wrap(x[i]) / tile_w) * cps + (uint32_t)(y[i] >> 3) : FP_NONE;
        const uint32_t sl = fp_warp_slot(cnt, c, FP_NONE);
        if (i >= n) continue;
        chunk_of[i] = c;
        if (take) slot[i] = sl;
    }
    __syncthreads();
    if (threadIdx.x == 0 && s_taken) atomicAdd(n_planned, (unsigned long long)s_taken);
}

// Also writes the planner's record of the agent, (id, wrapped x, y, v_max), so the plan kernel
// reads one coalesced 16-byte word per agent instead of dependent scattered loads.
__global__ void bucket_scatter_kernel(Geo g, const int32_t* x, const int32_t* y, const uint8_t* v, uint32_t n,
                                      const uint32_t* chunk_of, const uint32_t* slot, const uint32_t* off,
                                      uint32_t* bucket, uint4* brec) {
    FP_PDL_WAIT();
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t c = chunk_of[i];
        if (c == FP_NONE) continue;
        const uint32_t p = off[c] + slot[i];
        if (bucket) bucket[p] = i;
        brec[p] = make_uint4(i, (uint32_t)g.wrap(x[i]), (uint32_t)y[i], v[i]);
    }
}

// Per tile (row-major id t = ty * tiles_x + tx): count and first position from its chunks, and
// the compacted list of non-empty tiles (order irrelevant to the motion).
__global__ void tile_sums_kernel(const uint32_t* ccnt, const uint32_t* coff, int tiles_x, int tiles_y, uint32_t cps,
                                 int cpt, uint32_t* cnt, uint32_t* off, uint32_t* list, unsigned long long* n_tiles) {
    FP_PDL_WAIT();
    const uint32_t nt = (uint32_t)tiles_x * (uint32_t)tiles_y;
    const int lane = threadIdx.x & 31;
    for (uint32_t t0 = blockIdx.x * blockDim.x; t0 < nt; t0 += gridDim.x * blockDim.x) {
        const uint32_t t = t0 + threadIdx.x;
        uint32_t c = 0;
        if (t < nt) {
            const uint32_t tx = t % (uint32_t)tiles_x, ty = t / (uint32_t)tiles_x;
            const uint32_t g0 = tx * cps + ty * (uint32_t)cpt;
            for (int k = 0; k < cpt; ++k) c += ccnt[g0 + k];
            cnt[t] = c;
            off[t] = coff[g0];
        }
        const unsigned b = __ballot_sync(0xffffffffu, c != 0);  // one list reservation per warp
        uint32_t base = 0;
        if (lane == 0 && b) base = (uint32_t)atomicAdd(n_tiles, (unsigned long long)__popc(b));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (c) list[base + __popc(b & ((1u << lane) - 1u))] = t;
    }
}

// Warp-aggregated reservation of k consecutive slots of a list counted by *n: the warp's
// lanes get consecutive ranges in lane order (one atomic per warp).  Every lane calls it.
__device__ __forceinline__ uint32_t warp_reserve(uint32_t k, unsigned long long* n) {
    const int lane = threadIdx.x & 31;
    uint32_t incl = k;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
    uint32_t base = 0;
    if (lane == 0 && tot) base = (uint32_t)atomicAdd(n, (unsigned long long)tot);
    return __shfl_sync(0xffffffffu, base, 0) + incl - k;
}

// The motion's seed work items (tile-list entry, chunk of <= SEED_ITEM agents); *n_items is
// zero on entry.  Item order is free: the seed passes deal them out dynamically.
__global__ void motion_items_kernel(const uint32_t* list, const uint32_t* cnt, const unsigned long long* n_tiles_p,
                                    uint2* items, unsigned long long* n_items) {
    FP_PDL_WAIT();
    const uint32_t n = (uint32_t)*n_tiles_p;
    for (uint32_t e0 = blockIdx.x * blockDim.x; e0 < n; e0 += gridDim.x * blockDim.x) {
        const uint32_t e = e0 + threadIdx.x;
        const uint32_t k = e < n ? (cnt[list[e]] + SEED_ITEM - 1) / SEED_ITEM : 0u;
        const uint32_t ib = warp_reserve(k, n_items);
        for (uint32_t c = 0; c < k; ++c) items[ib + c] = make_uint2(e, c);
    }
}

// The plan kernel's work items.  Each stripe is cut into batches of PLAN_ITEM_CHUNKS consecutive
// chunks; a batch's agents (one contiguous bucket run) are split into ceil(agents /
// PLAN_ITEM_AGENTS) equal items.  Item = (first chunk touched, chunks touched - 1, first agent,
// end agent); empty batches give none; *n_items is zero on entry.  Items are claimed in list
// order, which follows the batches warp by warp (results never depend on it).
__global__ void plan_items_kernel(const uint32_t* ccnt, const uint32_t* coff, uint32_t cps, uint32_t tiles_x,
                                  const unsigned long long* n_planned_p, uint4* items, unsigned long long* n_items) {
    FP_PDL_WAIT();
    const uint32_t nch = cps * tiles_x;
    const uint32_t n_planned = (uint32_t)*n_planned_p;
    const uint32_t bps = (cps + PLAN_ITEM_CHUNKS - 1) / PLAN_ITEM_CHUNKS;
    const uint32_t nb = bps * tiles_x;
    for (uint32_t b0 = blockIdx.x * blockDim.x; b0 < nb; b0 += gridDim.x * blockDim.x) {
        const uint32_t b = b0 + threadIdx.x;
        uint32_t g0 = 0, g1 = 0, a0 = 0, a1 = 0, k = 0;
        if (b < nb) {
            const uint32_t s = b / bps, j = b % bps;
            g0 = s * cps + j * PLAN_ITEM_CHUNKS;
            g1 = min(g0 + PLAN_ITEM_CHUNKS, (s + 1) * cps);
            a0 = coff[g0];
            a1 = g1 < nch ? coff[g1] : n_planned;
            k = (a1 - a0 + PLAN_ITEM_AGENTS - 1) / PLAN_ITEM_AGENTS;
        }
        uint32_t ib = warp_reserve(k, n_items);
        const uint32_t A = a1 - a0;
        for (uint32_t t = 0; t < k; ++t) {
            const uint32_t lo = a0 + (uint32_t)((unsigned long long)t * A / k);
            const uint32_t hi = a0 + (uint32_t)((unsigned long long)(t + 1) * A / k);
            uint32_t gf = g0, gl = g0;  // chunks holding agents lo and hi - 1
            for (uint32_t g = g0; g < g1; ++g) {
                const uint32_t o = coff[g], c = ccnt[g];
                if (c && o <= lo && lo < o + c) gf = g;
                if (c && o <= hi - 1 && hi - 1 < o + c) gl = g;
            }
            // the item's agents per chunk, and per ring slot j (chunk gf - 1 + j) the agents
            // whose ball reaches it (chunks gf - 2 + j .. gf + j): the producer's reference counts
            uint32_t ca[PLAN_ITEM_CHUNKS];
            for (uint32_t g = gf; g <= gl; ++g) {
                const uint32_t o = coff[g], c = ccnt[g];
                const uint32_t l = max(o, lo), h = min(o + c, hi);
                ca[g - gf] = h > l ? h - l : 0u;
            }
            uint4* rec = items + 4 * (size_t)ib++;
            rec[0] = make_uint4(gf, gl - gf, lo, hi);
            uint16_t refs[24] = {0};
            const int nk = (int)(gl - gf) + 1;
            for (int j = 0; j < nk + 2 && j < 24; ++j) {
                uint32_t r = 0;
                for (int d = -1; d <= 1; ++d) {
                    const int e = j - 1 + d;  // item chunk index
                    if (e >= 0 && e < nk) r += ca[e];
                }
                refs[j] = (uint16_t)r;
            }
            const uint4* rv = reinterpret_cast<const uint4*>(refs);
            rec[1] = rv[0];
            rec[2] = rv[1];
            rec[3] = rv[2];
        }
    }
}

uint32_t fp_plan_chunks(const fp_ctx* ctx) { return (uint32_t)ctx->tiles_x * (uint32_t)ctx->cps; }

int fp_bucket_reserve(fp_ctx* ctx) {
    const size_t nt = (size_t)ctx->tiles_x * ctx->tiles_y;
    const size_t nch = fp_plan_chunks(ctx);
    if (ctx->bucket_reserved_nt == nt && ctx->bucket_reserved_cap == ctx->cap && ctx->d_scan_sums) return FP_OK;
    if (nt > ctx->n_tiles_alloc || nch > ctx->n_chunks_alloc || !ctx->d_scan_sums) {
        void* ptrs[] = {ctx->d_tile_cnt, ctx->d_tile_off, ctx->d_tile_list, ctx->d_sub_cnt,
                        ctx->d_sub_off,  ctx->d_tile_deal, ctx->d_scan_sums};
        for (void* p : ptrs)
            if (p) cudaFree(p);
        FP_CUDA(ctx, cudaMalloc(&ctx->d_sub_cnt, nch * 4));
        FP_CUDA(ctx, cudaMalloc(&ctx->d_sub_off, nch * 4));
        FP_CUDA(ctx, cudaMalloc(&ctx->d_tile_deal, ((size_t)ctx->sm_count * DEAL_PASSES + 1) * 4));
        FP_CUDA(ctx, cudaMalloc(&ctx->d_tile_cnt, nt * 4));
        FP_CUDA(ctx, cudaMalloc(&ctx->d_tile_off, nt * 4));
        FP_CUDA(ctx, cudaMalloc(&ctx->d_tile_list, nt * 4));
        FP_CUDA(ctx, cudaMalloc(&ctx->d_scan_sums, FP_SCAN_SUMS * 4));
        ctx->n_tiles_alloc = nt;
        ctx->n_chunks_alloc = nch;
        ctx->graph_valid = false;
    }
    const size_t pitems = nch / PLAN_ITEM_CHUNKS + ctx->tiles_x + (size_t)ctx->cap / PLAN_ITEM_AGENTS + 16;
    if (pitems > ctx->plan_items_alloc) {
        if (ctx->d_plan_items) cudaFree(ctx->d_plan_items);
        FP_CUDA(ctx, cudaMalloc(&ctx->d_plan_items, pitems * 4 * sizeof(uint4)));  // 64 B per item
        ctx->plan_items_alloc = pitems;
        ctx->graph_valid = false;
    }
    const size_t items = ctx->n_tiles_alloc + (size_t)ctx->cap / SEED_ITEM + 16;
    if (items > ctx->seed_items_alloc) {
        if (ctx->d_seed_items) cudaFree(ctx->d_seed_items);
        FP_CUDA(ctx, cudaMalloc(&ctx->d_seed_items, items * sizeof(uint2)));
        ctx->seed_items_alloc = items;
        ctx->graph_valid = false;
    }
    ctx->bucket_reserved_nt = nt;
    ctx->bucket_reserved_cap = ctx->cap;
    return FP_OK;
}

// Enqueues the bucketing of the agents to plan (graph-safe; resources reserved).
int fp_bucket_launch(fp_ctx* ctx) {
    cudaStream_t s = ctx->stream;
    const size_t nt = (size_t)ctx->tiles_x * ctx->tiles_y;
    const uint32_t nch = fp_plan_chunks(ctx);
    const uint32_t n = ctx->n;
    FP_CUDA(ctx, cudaMemsetAsync(ctx->d_sub_cnt, 0, (size_t)nch * 4, s));
    FP_CUDA(ctx, cudaMemsetAsync(&ctx->d_sc->n_planned, 0, 8, s));
    FP_CUDA(ctx, cudaMemsetAsync(&ctx->d_sc->n_tiles, 0, 8, s));
    const unsigned G = (unsigned)std::min<size_t>(fp_blocks(n, 256), (size_t)ctx->sm_count * FP_BUCKET_CTAS_PER_SM);
    fp_launch(bucket_count_kernel, G, 256, 0, s, fp_geo(ctx), ctx->d_x, ctx->d_y, ctx->d_alive,
                                          ctx->st.on ? ctx->st.d_owned : nullptr, n, ctx->tile_w, ctx->cps,
                                          ctx->d_sub_cnt, ctx->d_flags, ctx->d_cursor_b, &ctx->d_sc->n_planned);
    FP_LAUNCHED(ctx);
#ifdef FP_STAGE_BUCKET
    FP_STAMP(ctx, s, 4);
#endif
    if (int rc = fp_scan_u32(ctx, ctx->d_sub_cnt, ctx->d_sub_off, nch, ctx->d_scan_sums, s)) return rc;
#ifdef FP_STAGE_BUCKET
    FP_STAMP(ctx, s, 5);
#endif
    // after the scan: the tile lists and the plan items (side branch) beside the scatter
    cudaStream_t s3 = ctx->stream3;
    FP_CUDA(ctx, cudaEventRecord(ctx->ev_bfork, s));
    FP_CUDA(ctx, cudaStreamWaitEvent(s3, ctx->ev_bfork, 0));
    fp_launch(tile_sums_kernel, (unsigned)std::min<size_t>(fp_blocks(nt, 256), (size_t)ctx->sm_count * 8), 256, 0, s3,
        ctx->d_sub_cnt, ctx->d_sub_off, ctx->tiles_x, ctx->tiles_y, ctx->cps, ctx->tile_h / 8, ctx->d_tile_cnt,
        ctx->d_tile_off, ctx->d_tile_list, &ctx->d_sc->n_tiles);
    FP_LAUNCHED(ctx);
    FP_CUDA(ctx, cudaMemsetAsync(&ctx->d_sc->n_items, 0, 8, s3));
    fp_launch(motion_items_kernel, (unsigned)std::max<size_t>(1, fp_blocks(nt, 256)), 256, 0, s3,
        ctx->d_tile_list, ctx->d_tile_cnt, &ctx->d_sc->n_tiles, ctx->d_seed_items, &ctx->d_sc->n_items);
    FP_LAUNCHED(ctx);
    FP_CUDA(ctx, cudaMemsetAsync(&ctx->d_sc->n_plan_items, 0, 8, s3));
    const uint32_t nbatch = (uint32_t)((ctx->cps + PLAN_ITEM_CHUNKS - 1) / PLAN_ITEM_CHUNKS) * (uint32_t)ctx->tiles_x;
    fp_launch(plan_items_kernel, (unsigned)std::max<size_t>(1, fp_blocks(nbatch, 128)), 128, 0, s3,
        ctx->d_sub_cnt, ctx->d_sub_off, (uint32_t)ctx->cps, (uint32_t)ctx->tiles_x, &ctx->d_sc->n_planned,
        ctx->d_plan_items, &ctx->d_sc->n_plan_items);
    FP_LAUNCHED(ctx);
    FP_CUDA(ctx, cudaEventRecord(ctx->ev_bjoin, s3));
#ifdef FP_STAGE_BUCKET
    FP_STAMP(ctx, s, 6);
#endif
    fp_launch(bucket_scatter_kernel, G, 256, 0, s, fp_geo(ctx), ctx->d_x, ctx->d_y, ctx->d_v, n, ctx->d_flags,
                                            ctx->d_cursor_b, ctx->d_sub_off, nullptr /* ids: brec.x */, ctx->d_brec);
    FP_LAUNCHED(ctx);
    FP_CUDA(ctx, cudaStreamWaitEvent(s, ctx->ev_bjoin, 0));
    return FP_OK;
}
