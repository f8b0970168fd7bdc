// bucket.cu -- counting sort of the alive agents by plan tile (each step).
//
// The plan kernel stages one tile of the weight plane (plus halo) in shared memory per CTA and
// plans every agent standing in it; this groups agent ids by tile.  Order inside a tile is
// irrelevant (planning is a pure per-agent function of the pre-step snapshot,
// planning.hpp:14-17), so atomics are fine.  Also leaves the compacted list of non-empty tiles.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "internal.cuh"

// Agents are counted per (tile, v_max) sub-bucket, so each tile's agents come out ordered by
// v_max and the plan kernel's warps run one ball size (mixed-v rosters otherwise diverge over
// four unrolled variants and thrash the instruction cache).  On a strip rank (strip.cu) only the
// agents it owns are planned.  Counts the planned agents (= the plan's walk records) into
// *n_planned.
__global__ void bucket_count_kernel(Geo g, const int32_t* x, const int32_t* y, const uint8_t* v, const uint8_t* alive,
                                    const uint8_t* owned, uint32_t n, int tile_w, int tile_h, int tiles_x,
                                    uint32_t* cnt, uint32_t* tile_of, uint32_t* slot,
                                    unsigned long long* n_planned) {
    for (uint32_t i0 = blockIdx.x * blockDim.x; i0 < n; i0 += gridDim.x * blockDim.x) {
        const uint32_t i = i0 + threadIdx.x;
        const bool take = i < n && alive[i] && (!owned || owned[i]);
        const unsigned b = __ballot_sync(0xffffffffu, take);
        if ((threadIdx.x & 31) == 0 && b) atomicAdd(n_planned, (unsigned long long)__popc(b));
        if (i >= n) continue;
        if (!take) {
            tile_of[i] = FP_NONE;
            continue;
        }
        const int px = g.wrap(x[i]), py = y[i];
        const uint32_t t = ((uint32_t)(py / tile_h) * (uint32_t)tiles_x + (uint32_t)(px / tile_w)) * 5u +
                           (uint32_t)(v[i] - 1);  // v_max in 1..5
        tile_of[i] = t;
        slot[i] = atomicAdd(&cnt[t], 1u);
    }
}

// Also writes the planner's record of the agent, (id, wrapped x, y, v_max), so the plan kernel
// reads one coalesced 16-byte word per agent instead of dependent scattered loads.
__global__ void bucket_scatter_kernel(Geo g, const int32_t* x, const int32_t* y, const uint8_t* v,
                                      const uint8_t* alive, uint32_t n, const uint32_t* tile_of, const uint32_t* slot,
                                      const uint32_t* off, uint32_t* bucket, uint4* brec) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        if (tile_of[i] == FP_NONE) continue;
        const uint32_t p = off[tile_of[i]] + slot[i];
        bucket[p] = i;
        brec[p] = make_uint4(i, (uint32_t)g.wrap(x[i]), (uint32_t)y[i], v[i]);
    }
}

// per-tile count and offset from the (tile, v_max) sub-buckets
__global__ void tile_sums_kernel(const uint32_t* sub_cnt, const uint32_t* sub_off, uint32_t nt, uint32_t* cnt,
                                 uint32_t* off) {
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x) {
        const uint32_t* c = sub_cnt + (size_t)t * 5;
        cnt[t] = c[0] + c[1] + c[2] + c[3] + c[4];
        off[t] = sub_off[(size_t)t * 5];
    }
}

// Deals the non-empty tiles to the plan kernel's G CTAs in DEAL_PASSES passes: the list is cut
// into G * DEAL_PASSES contiguous ranges of near-equal cost (the range of entry e is
// floor(cost before e * G * DEAL_PASSES / total), a tile's cost its agent count with a floor),
// and range p*G + b goes to CTA b in its pass p.
// Crowded tiles do not pile up on a few CTAs, and at any time the CTAs work on neighbouring
// parts of the list (DRAM/L2 locality of the concurrent TMA fetches).  The range index is
// monotonic in e, so each boundary first[r] is written by exactly one entry.
// Block-wide exclusive scan of v (one value per thread); s_part = 32 slots of scratch.
__device__ __forceinline__ unsigned long long block_exclusive(unsigned long long v, unsigned long long* s_part,
                                                              unsigned long long* total) {
    unsigned long long incl = v;
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
        if ((threadIdx.x & 31) >= (unsigned)o) incl += t;
    }
    __syncthreads();  // s_part free
    if ((threadIdx.x & 31) == 31) s_part[threadIdx.x >> 5] = incl;
    __syncthreads();
    unsigned long long before = incl - v, t = 0;
    for (unsigned w = 0; w < (blockDim.x >> 5); ++w) {
        if (w < (threadIdx.x >> 5)) before += s_part[w];
        t += s_part[w];
    }
    *total = t;
    return before;
}

// Also cuts every tile into seed work items of at most SEED_ITEM agents for the motion's seed
// passes (a crowded exit tile would otherwise occupy one worker group for its whole length):
// items[i] = (tile-list entry, chunk), *n_items their count.
__global__ void __launch_bounds__(1024) tile_deal_kernel(const uint32_t* list, const uint32_t* cnt,
                                                          const unsigned long long* n_tiles_p, int G, int passes,
                                                          unsigned floor_cost, uint32_t* first, uint2* items,
                                                          unsigned long long* n_items) {
    // cost of a tile = max(its agents, floor_cost): a tile costs at least a fetch, so the
    // grid's partial last row/column of tiles does not pile onto one CTA.  One block: each
    // thread sums a contiguous run of the list, one block scan, then every entry's range.
    __shared__ unsigned long long s_part[32];
    G *= passes;  // ranges
    const uint32_t n = (uint32_t)*n_tiles_p;
    if (n == 0) {
        for (uint32_t b = threadIdx.x; b <= (uint32_t)G; b += blockDim.x) first[b] = 0;
        if (threadIdx.x == 0) *n_items = 0;
        return;
    }
    const uint32_t per = (n + blockDim.x - 1) / blockDim.x;
    const uint32_t e0 = min(n, threadIdx.x * per), e1 = min(n, e0 + per);
    unsigned long long mine = 0, my_items = 0;
    for (uint32_t e = e0; e < e1; ++e) {
        const unsigned c = cnt[list[e]];
        mine += max(c, floor_cost);
        my_items += (c + SEED_ITEM - 1) / SEED_ITEM;
    }
    unsigned long long total, n_it;
    unsigned long long before = block_exclusive(mine, s_part, &total);
    unsigned long long ib = block_exclusive(my_items, s_part, &n_it);
    for (uint32_t e = e0; e < e1; ++e) {
        const unsigned k = (cnt[list[e]] + SEED_ITEM - 1) / SEED_ITEM;
        for (unsigned c = 0; c < k; ++c) items[ib++] = make_uint2(e, c);
    }
    if (threadIdx.x == 0) *n_items = n_it;
    int prev = -1;
    if (e0 > 0) {  // range of the entry before this run
        const unsigned long long c = max(cnt[list[e0 - 1]], floor_cost);
        prev = (int)min((unsigned long long)(G - 1), (before - c) * (unsigned)G / total);
    }
    for (uint32_t e = e0; e < e1; ++e) {
        const int o = (int)min((unsigned long long)(G - 1), before * (unsigned)G / total);
        for (int b = prev + 1; b <= o; ++b) first[b] = e;
        if (e == n - 1)
            for (int b = o + 1; b <= G; ++b) first[b] = n;
        prev = o;
        before += max(cnt[list[e]], floor_cost);
    }
}

struct NonEmpty {
    const uint32_t* cnt;
    __device__ __forceinline__ bool operator()(uint32_t t) const { return cnt[t] != 0; }
};

// Least cost of a tile in the deal, in agent units (FP_DEAL_TILE_COST).
static unsigned deal_tile_cost() {
    static const unsigned c = getenv("FP_DEAL_TILE_COST") ? (unsigned)atoi(getenv("FP_DEAL_TILE_COST")) : 96u;
    return c;
}

int fp_bucket_reserve(fp_ctx* ctx) {
    const size_t nt = (size_t)ctx->tiles_x * ctx->tiles_y;
    if (ctx->bucket_reserved_nt == nt && ctx->bucket_reserved_cap == ctx->cap && ctx->d_temp_b) return FP_OK;
    if (nt > ctx->n_tiles_alloc) {
        if (ctx->d_tile_cnt) cudaFree(ctx->d_tile_cnt);
        if (ctx->d_tile_off) cudaFree(ctx->d_tile_off);
        if (ctx->d_tile_list) cudaFree(ctx->d_tile_list);
        if (ctx->d_sub_cnt) cudaFree(ctx->d_sub_cnt);
        if (ctx->d_sub_off) cudaFree(ctx->d_sub_off);
        FP_CUDA(ctx, cudaMalloc(&ctx->d_sub_cnt, nt * 5 * 4));
        if (!ctx->d_tile_deal)
            FP_CUDA(ctx, cudaMalloc(&ctx->d_tile_deal, ((size_t)ctx->sm_count * DEAL_PASSES + 1) * 4));
        FP_CUDA(ctx, cudaMalloc(&ctx->d_sub_off, nt * 5 * 4));
        FP_CUDA(ctx, cudaMalloc(&ctx->d_tile_cnt, nt * 4));
        FP_CUDA(ctx, cudaMalloc(&ctx->d_tile_off, nt * 4));
        FP_CUDA(ctx, cudaMalloc(&ctx->d_tile_list, nt * 4));
        ctx->n_tiles_alloc = nt;
        ctx->graph_valid = false;
    }
    const size_t items = ctx->n_tiles_alloc + (size_t)ctx->cap / SEED_ITEM + 16;
    if (items > ctx->seed_items_alloc) {
        if (ctx->d_seed_items) cudaFree(ctx->d_seed_items);
        FP_CUDA(ctx, cudaMalloc(&ctx->d_seed_items, items * sizeof(uint2)));
        ctx->seed_items_alloc = items;
        ctx->graph_valid = false;
    }
    size_t need1 = 0, need2 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, need1, ctx->d_sub_cnt, ctx->d_sub_off, (int)(nt * 5), ctx->stream);
    thrust::counting_iterator<uint32_t> it(0);
    cub::DeviceSelect::If(nullptr, need2, it, ctx->d_tile_list, &ctx->d_sc->n_tiles, (int)nt,
                          NonEmpty{ctx->d_tile_cnt}, ctx->stream);
    const size_t need = std::max(need1, need2) + 256;
    if (need > ctx->temp_b_bytes) {
        if (ctx->d_temp_b) {
            cudaStreamSynchronize(ctx->stream);
            cudaFree(ctx->d_temp_b);
        }
        FP_CUDA(ctx, cudaMalloc(&ctx->d_temp_b, need));
        ctx->temp_b_bytes = need;
        ctx->graph_valid = false;
    }
    ctx->bucket_reserved_nt = nt;
    ctx->bucket_reserved_cap = ctx->cap;
    return FP_OK;
}

// Enqueues the bucketing of the current alive agents (graph-safe; resources reserved).
int fp_bucket_launch(fp_ctx* ctx) {
    cudaStream_t s = ctx->stream;
    const size_t nt = (size_t)ctx->tiles_x * ctx->tiles_y;
    const uint32_t n = ctx->n;
    FP_CUDA(ctx, cudaMemsetAsync(ctx->d_sub_cnt, 0, nt * 5 * 4, s));
    const unsigned G = (unsigned)std::min<size_t>(fp_blocks(n, 256), (size_t)ctx->sm_count * 16);
    FP_CUDA(ctx, cudaMemsetAsync(&ctx->d_sc->n_planned, 0, 8, s));
    bucket_count_kernel<<<G, 256, 0, s>>>(fp_geo(ctx), ctx->d_x, ctx->d_y, ctx->d_v, ctx->d_alive,
                                          ctx->st.on ? ctx->st.d_owned : nullptr, n, ctx->tile_w, ctx->tile_h,
                                          ctx->tiles_x, ctx->d_sub_cnt, ctx->d_flags, ctx->d_cursor_b,
                                          &ctx->d_sc->n_planned);
    FP_LAUNCHED(ctx);
    size_t need1 = 0, need2 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, need1, ctx->d_sub_cnt, ctx->d_sub_off, (int)(nt * 5), s);
    thrust::counting_iterator<uint32_t> it(0);
    cub::DeviceSelect::If(nullptr, need2, it, ctx->d_tile_list, &ctx->d_sc->n_tiles, (int)nt, NonEmpty{ctx->d_tile_cnt}, s);
    if (std::max(need1, need2) > ctx->temp_b_bytes) return fp_fail(ctx, FP_ERUNTIME, "bucket: scratch not reserved");
    FP_CUDA(ctx, cub::DeviceScan::ExclusiveSum(ctx->d_temp_b, need1, ctx->d_sub_cnt, ctx->d_sub_off, (int)(nt * 5), s));
    ctx->ctr.kernel_launches += 2;
    tile_sums_kernel<<<(unsigned)std::min<size_t>(fp_blocks(nt, 256), (size_t)ctx->sm_count * 8), 256, 0, s>>>(
        ctx->d_sub_cnt, ctx->d_sub_off, (uint32_t)nt, ctx->d_tile_cnt, ctx->d_tile_off);
    FP_LAUNCHED(ctx);
    FP_CUDA(ctx, cub::DeviceSelect::If(ctx->d_temp_b, need2, it, ctx->d_tile_list, &ctx->d_sc->n_tiles, (int)nt,
                                       NonEmpty{ctx->d_tile_cnt}, s));
    ctx->ctr.kernel_launches += 2;
    tile_deal_kernel<<<1, 1024, 0, s>>>(ctx->d_tile_list, ctx->d_tile_cnt, &ctx->d_sc->n_tiles, ctx->sm_count,
                                        ctx->deal_passes, deal_tile_cost(), ctx->d_tile_deal, ctx->d_seed_items,
                                        &ctx->d_sc->n_items);
    FP_LAUNCHED(ctx);
    bucket_scatter_kernel<<<G, 256, 0, s>>>(fp_geo(ctx), ctx->d_x, ctx->d_y, ctx->d_v, ctx->d_alive, n, ctx->d_flags,
                                            ctx->d_cursor_b, ctx->d_sub_off, ctx->d_bucket, ctx->d_brec);
    FP_LAUNCHED(ctx);
    return FP_OK;
}
