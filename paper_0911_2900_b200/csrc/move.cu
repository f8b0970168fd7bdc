// move.cu -- the motion phase: the reference's sequential walk, executed in parallel rounds.
//
// Reference: move_phase (engine.hpp:113-133).  Agents walk one at a time in the movement order;
// each walks the Bresenham segment to its desired cell, at most v_max hops, stopping before a
// Wall or an occupied cell; an Exit removes it.  Later agents see earlier agents' final cells.
//
// Parallel form.  An agent's footprint is its start cell plus the path cells it could visit
// (motion_rec.cuh).  Only agents with overlapping footprints can influence each other, and only
// through those cells.
//   1. Contention marks (P1/P2 bitplanes) over every mover's footprint -- emitted by the plan
//      kernel together with the records, or built here when the plan did not.
//   2. A mover none of whose cells is marked twice walks immediately: nobody else reads or
//      writes its cells, so its position in the order is irrelevant.
//   3. The rest resolve in deterministic-reservation rounds: every pending agent writes its rank
//      into its footprint cells with atomicMin; an agent that holds all of its cells is the
//      earliest pending agent on each of them, so everything that precedes it in the reference
//      order on those cells has already run -- it walks now and clears its cells.  Keys left by
//      agents still pending are re-asserted with the same priority next round, so the u32
//      reservation plane needs no stamps or resets and ends every phase all-free.
// The result equals the sequential walk bit for bit (tests/test_gpu_parity.py).
//
// One cooperative launch runs a whole phase: grid-wide stages (grid.sync between them) while
// many agents are pending, then block 0 finishes the tail alone with __syncthreads.
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include "motion_rec.cuh"

namespace cg = cooperative_groups;

#define MOVE_THREADS 512
#define MOVE_TAIL 4096  // pending agents at or below which block 0 runs the rounds alone

__constant__ signed char c_bpath[121][5][2];
static bool g_bpath_ready[64] = {false};

struct MoveArgs {
    Geo g;
    uint32_t* occ;
    unsigned int* res;
    int32_t* x;
    int32_t* y;
    const int32_t* dx;
    const int32_t* dy;
    const uint8_t* v;
    uint8_t* alive;
    const uint32_t* rank;
    const uint32_t* seed_list;     // mode B: alive ids to build records from
    const uint4* rec0;             // mode A: records emitted by the plan kernel (n_alive of them)
    int premade;                   // 1: mode A, 0: mode B
    uint4* rec[2];                 // pending records, ping-pong
    unsigned int* pcount;          // [2] pending counts (device scratch, zero between phases)
    DevScalars* sc;
    unsigned long long* exits;     // (rank << 32 | id)
    uint32_t* p1;                  // contention bitplanes, zero between phases
    uint32_t* p2;
};

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ size_t cell_index(const Geo& g, int x, int y) {
    return (size_t)y * (size_t)g.W + (size_t)x;
}

__device__ __forceinline__ bool occ_test(const MoveArgs& a, int x, int y) {
    return (__ldcg(&a.occ[a.g.word(x, y)]) >> (x & 31)) & 1u;
}

__device__ __forceinline__ int path_of(const MoveArgs& a, const uint4& r, const signed char (*bp)[5][2], int* cx,
                                       int* cy) {
    int gtx = 0, gty = 0;
    if (r.w & REC_GENERIC) {
        gtx = a.g.wrap(a.dx[r.x]);
        gty = a.dy[r.x];
    }
    return record_cells(a.g, r, bp, gtx, gty, cx, cy);
}

__device__ __forceinline__ void append(unsigned int* count, uint4* list, bool take, const uint4& rec) {
    const unsigned mask = __ballot_sync(0xffffffffu, take);
    if (!mask) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(mask) - 1;
    unsigned base = 0;
    if (lane == leader) base = atomicAdd(count, (unsigned)__popc(mask));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (take) list[base + __popc(mask & ((1u << lane) - 1))] = rec;
}

__device__ __forceinline__ void clear_cell(const MoveArgs& a, int x, int y, bool both) {
    const size_t w = a.g.word(x, y);
    const uint32_t nbit = ~(1u << (x & 31));
    atomicAnd(&a.p1[w], nbit);
    if (both) atomicAnd(&a.p2[w], nbit);
}

// The walk (engine.hpp:116-129) of an agent that owns its footprint, net effect on occupancy.
__device__ __forceinline__ void walk_owned(const MoveArgs& a, const uint4& r, const int* cx, const int* cy, int m,
                                           unsigned long long* hops_acc) {
    const int sx = (int)(r.z & 0x0FFFFFFFu), sy = (int)(r.w & 0x00FFFFFFu);
    int h = 0;
    for (int i = 0; i < m; ++i) {
        if (occ_test(a, cx[i], cy[i])) break;
        ++h;
    }
    const bool exited = (h == m) && (r.z & 0x80000000u);
    if (h > 0) {
        const uint32_t id = r.x;
        atomicAnd(&a.occ[a.g.word(sx, sy)], ~(1u << (sx & 31)));
        const int fx = cx[h - 1], fy = cy[h - 1];
        a.x[id] = fx;
        a.y[id] = fy;
        if (exited) {
            a.alive[id] = 0;
            const unsigned long long slot = atomicAdd(&a.sc->n_exits, 1ull);
            // processing order = rank (uncontended walkers never loaded theirs into the record)
            a.exits[slot] = ((unsigned long long)a.rank[id] << 32) | id;
        } else {
            atomicOr(&a.occ[a.g.word(fx, fy)], 1u << (fx & 31));
        }
    }
    *hops_acc += (unsigned long long)h;
}

__device__ __forceinline__ void reserve_one(const MoveArgs& a, const uint4& r, const signed char (*bp)[5][2]) {
    int cx[5], cy[5];
    const int m = path_of(a, r, bp, cx, cy);
    atomicMin(&a.res[cell_index(a.g, (int)(r.z & 0x0FFFFFFFu), (int)(r.w & 0x00FFFFFFu))], r.y);
    for (int i = 0; i < m; ++i) atomicMin(&a.res[cell_index(a.g, cx[i], cy[i])], r.y);
}

// Returns true if the agent committed (walked); false if it must retry next round.
__device__ __forceinline__ bool commit_one(const MoveArgs& a, const uint4& r, const signed char (*bp)[5][2],
                                           unsigned long long* hops_acc) {
    const int sx = (int)(r.z & 0x0FFFFFFFu), sy = (int)(r.w & 0x00FFFFFFu);
    int cx[5], cy[5];
    const int m = path_of(a, r, bp, cx, cy);
    bool own = __ldcg(&a.res[cell_index(a.g, sx, sy)]) == r.y;
    for (int i = 0; i < m && own; ++i) own = __ldcg(&a.res[cell_index(a.g, cx[i], cy[i])]) == r.y;
    if (!own) return false;
    // release the footprint (losers of this round read it after their own failed check only)
    // and its contention bits (zero again for the next phase)
    a.res[cell_index(a.g, sx, sy)] = 0xFFFFFFFFu;
    clear_cell(a, sx, sy, true);
    for (int i = 0; i < m; ++i) {
        a.res[cell_index(a.g, cx[i], cy[i])] = 0xFFFFFFFFu;
        clear_cell(a, cx[i], cy[i], true);
    }
    walk_owned(a, r, cx, cy, m, hops_acc);
    return true;
}

__device__ __forceinline__ void flush_hops(DevScalars* sc, unsigned long long hops) {
    for (int o = 16; o > 0; o >>= 1) hops += __shfl_down_sync(0xffffffffu, hops, o);
    if ((threadIdx.x & 31) == 0 && hops) atomicAdd(&sc->disp, hops);
}

// Step 2 for one record: walk now if uncontended, else hand it (with its rank) to the rounds.
__device__ __forceinline__ bool classify(const MoveArgs& a, uint4& rec, const signed char (*bp)[5][2],
                                         unsigned long long* hops) {
    int cx[5], cy[5];
    const int m = path_of(a, rec, bp, cx, cy);
    const int sx = (int)(rec.z & 0x0FFFFFFFu), sy = (int)(rec.w & 0x00FFFFFFu);
    bool contended = (__ldcg(&a.p2[a.g.word(sx, sy)]) >> (sx & 31)) & 1u;
    for (int i = 0; i < m && !contended; ++i)
        contended = (__ldcg(&a.p2[a.g.word(cx[i], cy[i])]) >> (cx[i] & 31)) & 1u;
    if (!contended) {
        walk_owned(a, rec, cx, cy, m, hops);
        clear_cell(a, sx, sy, false);
        for (int i = 0; i < m; ++i) clear_cell(a, cx[i], cy[i], false);
        return false;
    }
    rec.y = a.rank[rec.x];
    return true;
}

__global__ void __launch_bounds__(MOVE_THREADS) move_rounds_kernel(MoveArgs a) {
    cg::grid_group grid = cg::this_grid();
    __shared__ signed char s_bp[121][5][2];
    for (int k = threadIdx.x; k < 121 * 10; k += blockDim.x) (&s_bp[0][0][0])[k] = (&c_bpath[0][0][0])[k];
    __syncthreads();
    const unsigned nthreads = gridDim.x * blockDim.x;
    const unsigned gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t n = (uint32_t)__ldcg(&a.sc->n_alive);
    if (gtid == 0) a.sc->t_motion[0] = globaltimer();
    const uint4* cand = a.rec0;
    unsigned ncand = n;
    if (!a.premade) {
        // step 1 here: records of every mover, footprints marked
        for (uint32_t base = 0; base < n; base += nthreads) {
            const uint32_t k = base + gtid;
            uint4 rec = make_uint4(0, 0, 0, 0);
            bool take = false;
            if (k < n) {
                const uint32_t id = a.seed_list[k];
                const int tx = a.g.wrap(a.dx[id]), ty = a.dy[id];
                rec = record_of(a.g, id, a.g.wrap(a.x[id]), a.y[id], tx, ty, a.v[id], s_bp);
                take = (rec.z >> 28) & 7u;
                if (take) mark_record(a.p1, a.p2, a.g, rec, s_bp, tx, ty);
            }
            append(&a.pcount[0], a.rec[0], take, rec);
        }
        grid.sync();
        cand = a.rec[0];
        ncand = __ldcg(&a.pcount[0]);
    } else {
        // step 1 over the plan's records (coalesced, plan-tile order)
        for (uint32_t k = gtid; k < n; k += nthreads) {
            const uint4 rec = __ldcg(&a.rec0[k]);
            if ((rec.z >> 28) & 7u) {
                int gtx = 0, gty = 0;
                if (rec.w & REC_GENERIC) {
                    gtx = a.g.wrap(a.dx[rec.x]);
                    gty = a.dy[rec.x];
                }
                mark_record(a.p1, a.p2, a.g, rec, s_bp, gtx, gty);
            }
        }
        grid.sync();
    }
    // step 2
    {
        unsigned long long hops = 0;
        for (unsigned base = 0; base < ncand; base += nthreads) {
            const unsigned k = base + gtid;
            bool contended = false;
            uint4 rec = make_uint4(0, 0, 0, 0);
            if (k < ncand) {
                rec = __ldcg(&cand[k]);
                if ((rec.z >> 28) & 7u) contended = classify(a, rec, s_bp, &hops);
            }
            append(&a.pcount[1], a.rec[1], contended, rec);
        }
        flush_hops(a.sc, hops);
    }
    grid.sync();
    if (gtid == 0) a.sc->t_motion[1] = globaltimer();
    // step 3
    unsigned r = 0;
    bool solo = false;
    for (;; ++r) {
        const unsigned cur = (r + 1) & 1, nxt = cur ^ 1;
        const unsigned np = __ldcg(&a.pcount[cur]);
        if (np == 0) break;
        if (!solo && np <= MOVE_TAIL) {
            if (blockIdx.x != 0) return;  // every block reads the same np: block 0 continues alone
            solo = true;
            if (threadIdx.x == 0) {
                a.sc->t_motion[2] = globaltimer();
                a.sc->grid_rounds = r;
            }
        }
        const unsigned stride = solo ? blockDim.x : nthreads;
        const unsigned me = solo ? threadIdx.x : gtid;
        if (gtid == 0) a.pcount[nxt] = 0;
        const uint4* list = a.rec[cur];
        for (unsigned k = me; k < np; k += stride) reserve_one(a, __ldcg(&list[k]), s_bp);
        if (solo) __syncthreads(); else grid.sync();
        unsigned long long hops = 0;
        for (unsigned base = 0; base < np; base += stride) {
            const unsigned k = base + me;
            bool retry = false;
            uint4 rec = make_uint4(0, 0, 0, 0);
            if (k < np) {
                rec = __ldcg(&list[k]);
                retry = !commit_one(a, rec, s_bp, &hops);
            }
            append(&a.pcount[nxt], a.rec[nxt], retry, rec);
        }
        flush_hops(a.sc, hops);
        if (solo) __syncthreads(); else grid.sync();
    }
    if (gtid == 0) {
        const unsigned long long t = globaltimer();
        if (!solo) {
            a.sc->t_motion[2] = t;
            a.sc->grid_rounds = r;
        }
        a.sc->t_motion[3] = t;
        a.sc->pad[1] += r;  // rounds executed (observability)
        a.pcount[0] = 0;
        a.pcount[1] = 0;
        const unsigned long long ne = a.sc->n_exits;
        a.sc->alive -= ne;
        a.sc->tot_exits += ne;
        a.sc->tot_disp += a.sc->disp;
    }
}

__global__ void move_begin_kernel(DevScalars* sc) {
    sc->n_exits = 0;
    sc->disp = 0;
    sc->tot_updates += sc->alive;
}

int fp_ensure_res(fp_ctx* ctx) {
    if (ctx->device < 64 && !g_bpath_ready[ctx->device]) {
        signed char bp[121][5][2];
        host_bpath(bp);
        FP_CUDA(ctx, cudaMemcpyToSymbol(c_bpath, bp, sizeof(bp)));
        g_bpath_ready[ctx->device] = true;
    }
    if (ctx->d_res) return FP_OK;
    const size_t nwords = (size_t)ctx->P * ctx->H;
    FP_CUDA(ctx, cudaMalloc(&ctx->d_p1, nwords * 4));
    FP_CUDA(ctx, cudaMalloc(&ctx->d_p2, nwords * 4));
    FP_CUDA(ctx, cudaMemsetAsync(ctx->d_p1, 0, nwords * 4, ctx->stream));
    FP_CUDA(ctx, cudaMemsetAsync(ctx->d_p2, 0, nwords * 4, ctx->stream));
    const size_t cells = (size_t)ctx->W * (size_t)ctx->H;
    FP_CUDA(ctx, cudaMalloc(&ctx->d_res, cells * sizeof(unsigned int)));
    FP_CUDA(ctx, cudaMemsetAsync(ctx->d_res, 0xFF, cells * sizeof(unsigned int), ctx->stream));
    ctx->marks_dirty = false;
    return FP_OK;
}

static int g_move_blocks = 0;

// Enqueues one motion phase (after fp_order_launch) on ctx->stream.  Graph-safe.
// Mode A (ctx->rec_fresh): the plan kernel emitted records + marks for the current state.
// Mode B: records are built here from the plan-tile buckets when current, else the order list.
int fp_motion_launch(fp_ctx* ctx, bool spatial) {
    cudaStream_t s = ctx->stream;
    move_begin_kernel<<<1, 1, 0, s>>>(ctx->d_sc);
    FP_LAUNCHED(ctx);
    if (ctx->n == 0) return FP_OK;
    const bool premade = ctx->rec_fresh;
    if (!premade && ctx->marks_dirty) {  // marks of records that were never consumed
        const size_t nwords = (size_t)ctx->P * ctx->H;
        FP_CUDA(ctx, cudaMemsetAsync(ctx->d_p1, 0, nwords * 4, s));
        FP_CUDA(ctx, cudaMemsetAsync(ctx->d_p2, 0, nwords * 4, s));
    }
    if (!g_move_blocks) {
        int per_sm = 0;
        FP_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, move_rounds_kernel, MOVE_THREADS, 0));
        g_move_blocks = std::max(1, std::min(per_sm, 2)) * ctx->sm_count;
    }
    MoveArgs a;
    a.g = fp_geo(ctx);
    a.occ = ctx->d_occ;
    a.res = ctx->d_res;
    a.x = ctx->d_x;
    a.y = ctx->d_y;
    a.dx = ctx->d_dx;
    a.dy = ctx->d_dy;
    a.v = ctx->d_v;
    a.alive = ctx->d_alive;
    a.rank = ctx->d_rank;
    a.seed_list = spatial ? ctx->d_bucket : ctx->d_order;
    a.rec0 = ctx->d_rec0;
    a.premade = premade ? 1 : 0;
    a.rec[0] = ctx->d_rec_a;
    a.rec[1] = ctx->d_rec_b;
    a.pcount = (unsigned int*)ctx->d_counters;  // [0], [1] as u32 (kept zero between phases)
    a.sc = ctx->d_sc;
    a.exits = ctx->d_exits;
    a.p1 = ctx->d_p1;
    a.p2 = ctx->d_p2;
    const unsigned blocks = (unsigned)std::min<size_t>((size_t)g_move_blocks,
                                                        std::max<size_t>(1, fp_blocks(ctx->n, MOVE_THREADS)));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(MOVE_THREADS);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    FP_CUDA(ctx, cudaLaunchKernelEx(&cfg, move_rounds_kernel, a));
    ctx->ctr.kernel_launches++;
    ctx->rec_fresh = false;
    ctx->marks_dirty = false;
    return fp_ghost_occ(ctx);
}

// Sorts the exit records of the last phase by rank (processing order) for fp_get_exited.
int fp_exits_finish(fp_ctx* ctx) {
    const uint32_t ne = ctx->n_exits;
    if (ne <= 1) return FP_OK;
    size_t need = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, need, ctx->d_exits, ctx->d_exits_sorted, (int)ne, 0, 64, ctx->stream);
    if (int rc = fp_ensure_temp(ctx, need)) return rc;
    FP_CUDA(ctx, cub::DeviceRadixSort::SortKeys(ctx->d_temp, need, ctx->d_exits, ctx->d_exits_sorted, (int)ne, 0, 64,
                                                ctx->stream));
    ctx->ctr.kernel_launches += 4;
    FP_CUDA(ctx, cudaMemcpyAsync(ctx->d_exits, ctx->d_exits_sorted, ne * sizeof(unsigned long long),
                                 cudaMemcpyDeviceToDevice, ctx->stream));
    return FP_OK;
}
