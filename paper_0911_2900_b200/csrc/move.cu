// move.cu -- the motion phase: the reference's sequential walk, executed in parallel rounds.
//
// Reference: move_phase (engine.hpp:113-133).  Agents walk one at a time in the movement order;
// each walks the Bresenham segment to its desired cell, at most v_max hops, stopping before a
// Wall or an occupied cell; an Exit removes it.  Later agents see earlier agents' final cells.
//
// Parallel form (deterministic reservations): an agent's footprint is its start cell plus the
// path cells it could visit (capped at v_max, cut before a Wall, ending at an Exit).  Only
// agents with overlapping footprints can influence each other, and only through those cells.
// Each round, every pending agent writes its key (round stamp, rank) into its footprint cells
// with atomicMin; an agent that holds all of its cells is the earliest pending agent on each of
// them, so everything that precedes it in the reference order on those cells has already run
// -- it executes its walk now.  Committed agents in one round have disjoint footprints.  The
// result equals the sequential walk bit for bit (tests/test_motion_gpu.py).  Agents with an
// empty path (staying put) never change occupancy and skip the rounds entirely.
//
// Round stamps make the reservation plane self-cleaning: newer rounds carry smaller keys.
#include <cub/cub.cuh>

#include "internal.cuh"

struct MoveArgs {
    Geo g;
    uint32_t* occ;
    unsigned long long* res;
    int32_t* x;
    int32_t* y;
    const int32_t* dx;
    const int32_t* dy;
    const uint8_t* v;
    uint8_t* alive;
    const uint32_t* rank;
    unsigned long long* counters;  // [0] next pending, [1] exits, [2] exited, [4] displacement
    unsigned long long* exits;     // (rank << 32 | id)
    unsigned long long stamp;      // (0xFFFFFFFF - round) << 32
};

// Path cells the walk may visit (engine.hpp:116-119 static stops), at most 5.
__device__ __forceinline__ int footprint(const MoveArgs& a, uint32_t id, int* cx, int* cy) {
    const Geo& g = a.g;
    const int sx = g.wrap(a.x[id]), sy = a.y[id];
    const int tx = g.wrap(a.dx[id]), ty = a.dy[id];
    const int v = a.v[id];
    Bres b;
    b.init(g, sx, sy, tx, ty);
    int k = 0;
    while (!b.done() && k < v) {
        b.next();
        const int x = g.wrap(b.x), y = b.y;
        if (g.is_wall(x, y)) break;
        cx[k] = x;
        cy[k] = y;
        ++k;
        if (g.is_exit(x, y)) break;
    }
    return k;
}

__device__ __forceinline__ size_t cell_index(const Geo& g, int x, int y) {
    return (size_t)y * (size_t)g.W + (size_t)x;
}

// Initial pending list: alive agents whose walk has at least one cell.
__global__ void move_seed_kernel(MoveArgs a, const uint32_t* order, uint32_t n, uint32_t* pend) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const uint32_t id = order[k];
    int cx[5], cy[5];
    const bool active = footprint(a, id, cx, cy) > 0;
    // warp-aggregated append
    const unsigned mask = __ballot_sync(__activemask(), active);
    if (!active) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(mask) - 1;
    unsigned base = 0;
    if (lane == leader) base = (unsigned)atomicAdd(&a.counters[0], (unsigned long long)__popc(mask));
    base = __shfl_sync(mask, base, leader);
    pend[base + __popc(mask & ((1u << lane) - 1))] = id;
}

__global__ void move_reserve_kernel(MoveArgs a, const uint32_t* pend, uint32_t np) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= np) return;
    const uint32_t id = pend[k];
    const unsigned long long key = a.stamp | a.rank[id];
    int cx[5], cy[5];
    const int m = footprint(a, id, cx, cy);
    atomicMin(&a.res[cell_index(a.g, a.g.wrap(a.x[id]), a.y[id])], key);
    for (int i = 0; i < m; ++i) atomicMin(&a.res[cell_index(a.g, cx[i], cy[i])], key);
}

__device__ __forceinline__ bool occ_test(const MoveArgs& a, int x, int y) {
    return (__ldcg(&a.occ[a.g.word(x, y)]) >> (x & 31)) & 1u;
}

__global__ void move_commit_kernel(MoveArgs a, const uint32_t* pend, uint32_t np, uint32_t* next) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    bool retry = false;
    unsigned long long hops = 0;
    if (k < np) {
        const uint32_t id = pend[k];
        const unsigned long long key = a.stamp | a.rank[id];
        int cx[5], cy[5];
        const int m = footprint(a, id, cx, cy);
        const int sx = a.g.wrap(a.x[id]), sy = a.y[id];
        bool own = __ldcg(&a.res[cell_index(a.g, sx, sy)]) == key;
        for (int i = 0; i < m && own; ++i) own = __ldcg(&a.res[cell_index(a.g, cx[i], cy[i])]) == key;
        if (!own) {
            retry = true;
        } else {
            // The walk (engine.hpp:116-129), net effect on occupancy.
            int h = 0;
            bool exited = false;
            for (int i = 0; i < m; ++i) {
                if (occ_test(a, cx[i], cy[i])) break;
                ++h;
                if (a.g.is_exit(cx[i], cy[i])) {
                    exited = true;
                    break;
                }
            }
            if (h > 0) {
                atomicAnd(&a.occ[a.g.word(sx, sy)], ~(1u << (sx & 31)));
                const int fx = cx[h - 1], fy = cy[h - 1];
                a.x[id] = fx;
                a.y[id] = fy;
                if (exited) {
                    a.alive[id] = 0;
                    const unsigned long long slot = atomicAdd(&a.counters[1], 1ull);
                    a.exits[slot] = ((unsigned long long)a.rank[id] << 32) | id;
                } else {
                    atomicOr(&a.occ[a.g.word(fx, fy)], 1u << (fx & 31));
                }
            }
            hops = (unsigned long long)h;
        }
    }
    // displacement: warp reduce then one atomic
    for (int o = 16; o > 0; o >>= 1) hops += __shfl_down_sync(0xffffffffu, hops, o);
    if ((threadIdx.x & 31) == 0 && hops) atomicAdd(&a.counters[4], hops);
    const unsigned mask = __ballot_sync(0xffffffffu, retry);
    if (retry) {
        const int lane = threadIdx.x & 31;
        const int leader = __ffs(mask) - 1;
        unsigned base = 0;
        if (lane == leader) base = (unsigned)atomicAdd(&a.counters[0], (unsigned long long)__popc(mask));
        base = __shfl_sync(mask, base, leader);
        next[base + __popc(mask & ((1u << lane) - 1))] = pend[k];
    }
}

// Runs the rounds of one motion phase after fp_order_launch.  Leaves the exit records in
// ctx->d_exits (sorted by rank when collect_exits), updates ctx->alive.
int fp_motion_launch(fp_ctx* ctx, bool collect_exits) {
    cudaStream_t s = ctx->stream;
    const size_t cells = (size_t)ctx->W * (size_t)ctx->H;
    if (!ctx->d_res) {
        FP_CUDA(ctx, cudaMalloc(&ctx->d_res, cells * sizeof(unsigned long long)));
        FP_CUDA(ctx, cudaMemsetAsync(ctx->d_res, 0xFF, cells * sizeof(unsigned long long), s));
        ctx->round_seq = 0;
    }
    MoveArgs a;
    a.g = Geo{ctx->W, ctx->H, ctx->boundary, ctx->P, ctx->d_wall, ctx->d_exit};
    a.occ = ctx->d_occ;
    a.res = (unsigned long long*)ctx->d_res;
    a.x = ctx->d_x;
    a.y = ctx->d_y;
    a.dx = ctx->d_dx;
    a.dy = ctx->d_dy;
    a.v = ctx->d_v;
    a.alive = ctx->d_alive;
    a.rank = ctx->d_rank;
    a.counters = ctx->d_counters;
    a.exits = ctx->d_exits;
    a.stamp = 0;

    FP_CUDA(ctx, cudaMemsetAsync(ctx->d_counters, 0, 6 * sizeof(unsigned long long), s));
    ctx->n_exits = 0;
    ctx->last_displacement = 0;
    const uint32_t n = ctx->n_order;
    if (n == 0) return FP_OK;
    move_seed_kernel<<<fp_blocks(n, 256), 256, 0, s>>>(a, ctx->d_order, n, ctx->d_pend_a);
    FP_LAUNCHED(ctx);
    FP_CUDA(ctx, cudaMemcpyAsync(ctx->h_counters, ctx->d_counters, sizeof(unsigned long long),
                                 cudaMemcpyDeviceToHost, s));
    FP_CUDA(ctx, cudaStreamSynchronize(s));
    uint32_t np = (uint32_t)ctx->h_counters[0];
    uint32_t* cur = ctx->d_pend_a;
    uint32_t* nxt = ctx->d_pend_b;
    while (np > 0) {
        if (ctx->round_seq >= 0xFFFFFFF0ull) {
            FP_CUDA(ctx, cudaMemsetAsync(ctx->d_res, 0xFF, cells * sizeof(unsigned long long), s));
            ctx->round_seq = 0;
        }
        a.stamp = (0xFFFFFFFFull - ctx->round_seq) << 32;
        ctx->round_seq++;
        ctx->ctr.motion_rounds++;
        FP_CUDA(ctx, cudaMemsetAsync(ctx->d_counters, 0, sizeof(unsigned long long), s));
        move_reserve_kernel<<<fp_blocks(np, 256), 256, 0, s>>>(a, cur, np);
        FP_LAUNCHED(ctx);
        move_commit_kernel<<<fp_blocks(np, 256), 256, 0, s>>>(a, cur, np, nxt);
        FP_LAUNCHED(ctx);
        FP_CUDA(ctx, cudaMemcpyAsync(ctx->h_counters, ctx->d_counters, sizeof(unsigned long long),
                                     cudaMemcpyDeviceToHost, s));
        FP_CUDA(ctx, cudaStreamSynchronize(s));
        np = (uint32_t)ctx->h_counters[0];
        uint32_t* t = cur;
        cur = nxt;
        nxt = t;
    }
    FP_CUDA(ctx, cudaMemcpyAsync(ctx->h_counters, ctx->d_counters, 6 * sizeof(unsigned long long),
                                 cudaMemcpyDeviceToHost, s));
    FP_CUDA(ctx, cudaStreamSynchronize(s));
    const uint32_t ne = (uint32_t)ctx->h_counters[1];
    ctx->n_exits = ne;
    ctx->alive -= ne;
    ctx->last_displacement = (int64_t)ctx->h_counters[4];
    if (collect_exits && ne > 1) {
        size_t need = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, need, ctx->d_exits, ctx->d_exits_sorted, (int)ne, 0, 64, s);
        if (int rc = fp_ensure_temp(ctx, need)) return rc;
        FP_CUDA(ctx, cub::DeviceRadixSort::SortKeys(ctx->d_temp, need, ctx->d_exits,
                                                    ctx->d_exits_sorted, (int)ne, 0, 64, s));
        ctx->ctr.kernel_launches++;
        FP_CUDA(ctx, cudaMemcpyAsync(ctx->d_exits, ctx->d_exits_sorted, ne * sizeof(unsigned long long),
                                     cudaMemcpyDeviceToDevice, s));
    }
    return FP_OK;
}
