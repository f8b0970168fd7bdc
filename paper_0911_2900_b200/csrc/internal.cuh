// internal.cuh -- device context, data layout and shared device helpers.
//
// HBM layout (row-major in y like world.hpp:88-91, x padded with ghost columns):
//   wall / exit / occupancy : 1-bit planes, P u32 words per row covering x in [-32, 32*P-32);
//                             for periodic-x grids the ghost bits mirror the wrapped columns
//   weight plane            : u32 per cell, pitch PW covering x in [-8, PW-8): the static
//                             planning data of a cell for one (k_s, potential) -- an exact-path
//                             flag and the fp32-mantissa / integer-exponent split of
//                             2^(-k_s*log2(e)*S) (plane.cu).  Read by the plan kernel via TMA.
//   field                   : fp64 per cell (StaticField::s), read only by the exact path
//   motion scratch          : P1/P2 contention bitplanes (like occupancy); a 32-byte rank
//                             bucket per cell (+ overflow pool) for the reservation rounds
//   agents (SoA)            : x, y (i32), v_max (u8), alive (u8), desired x/y (i32), rank (u32)
//   tile buckets            : agent ids grouped by plan tile (counting sort each step)
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/fastped_b200.h"

// Programmatic dependent launch.  Every kernel is launched through fp_launch with programmatic
// stream serialisation, so the next kernel of a stream (or captured graph branch) is dispatched
// while its predecessor drains instead of after it; every kernel body opens with FP_PDL_WAIT
// (griddepcontrol.wait: blocks until the predecessor grid has completed and its memory is
// visible; returns at once for a kernel launched without the attribute).  Nothing runs before
// the wait, so ordering is exactly that of plain launches.  FP_PDL_TRIGGER builds additionally
// release the dependent launch right after the wait (its CTAs are then resident and parked
// while this grid runs).  FASTPED_PDL=0 in the environment launches without the attribute.
#ifdef FP_PDL_TRIGGER
#define FP_PDL_WAIT() asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" ::: "memory")
#else
#define FP_PDL_WAIT() asm volatile("griddepcontrol.wait;" ::: "memory")
#endif

bool fp_pdl_enabled();  // capi.cu

template <typename... KArgs, typename... Args>
inline void fp_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = fp_pdl_enabled() ? 1 : 0;
    (void)cudaLaunchKernelEx(&cfg, kernel, args...);  // errors surface through cudaGetLastError
}

#define FP_NONE 0xFFFFFFFFu
#define FP_XPAD_BITS 32  // ghost columns left of x = 0 in the bitplanes
#define FP_XPAD_W 8      // ghost columns left of x = 0 in the weight plane
#define FP_HALO 5        // largest v_max (agents.hpp:10)
#define DEAL_PASSES 16   // plan-tile deal: most passes over the tile list (bucket.cu)
#define SEED_ITEM 512    // agents per motion seed work item (a worker group takes it in passes of 128)

// weight-plane word encoding (plane.cu)
#define FP_W_WALL 0xFFFFFFFFu
#define FP_W_UNREACH 0x80000000u
#define FP_W_FLAG 0x80000000u  // the exact path plans an agent standing here

struct Geo {
    int W, H, boundary, P;
    const uint32_t* wall;
    const uint32_t* exitb;

    __device__ __forceinline__ int wrap(int x) const {
        if (boundary == FP_BOUNDARY_PERIODIC_X) {
            x %= W;
            if (x < 0) x += W;
        }
        return x;
    }
    __device__ __forceinline__ size_t word(int x, int y) const {
        return (size_t)y * (size_t)P + (size_t)((x + FP_XPAD_BITS) >> 5);
    }
    __device__ __forceinline__ bool is_wall(int x, int y) const {
        return (__ldg(&wall[word(x, y)]) >> (x & 31)) & 1u;
    }
    __device__ __forceinline__ bool is_exit(int x, int y) const {
        return (__ldg(&exitb[word(x, y)]) >> (x & 31)) & 1u;
    }
    // world.hpp:125-132
    __device__ __forceinline__ int segment_dx(int ax, int bx) const {
        int d = bx - ax;
        if (boundary == FP_BOUNDARY_PERIODIC_X) {
            const int alt = d > 0 ? d - W : d + W;
            if (abs(alt) < abs(d)) d = alt;
        }
        return d;
    }
};

// Bresenham walker over world.hpp:143-167 (exclusive a, inclusive b), one cell per next().
struct Bres {
    int x, y, tx, ty, dx, dy, sx, sy, err;
    __device__ __forceinline__ void init(const Geo& g, int ax, int ay, int bx, int by) {
        tx = ax + g.segment_dx(ax, bx);
        dx = abs(tx - ax);
        sx = ax < tx ? 1 : -1;
        dy = -abs(by - ay);
        sy = ay < by ? 1 : -1;
        err = dx + dy;
        x = ax;
        y = ay;
        ty = by;
    }
    __device__ __forceinline__ bool done() const { return x == tx && y == ty; }
    __device__ __forceinline__ void next() {
        const int e2 = 2 * err;
        if (e2 >= dy) { err += dy; x += sx; }
        if (e2 <= dx) { err += dx; y += sy; }
    }
};

// rng.hpp:13-32
__host__ __device__ __forceinline__ uint64_t fp_rng_u64(uint64_t seed, uint64_t agent,
                                                        uint64_t step, uint64_t draw) {
    uint64_t z = seed ^ (agent * 0x9E3779B97F4A7C15ULL) ^ (step * 0xBF58476D1CE4E5B9ULL) ^
                 (draw * 0x94D049BB133111EBULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ double fp_unit_interval(uint64_t x) {
    return (double)(x >> 11) * 0x1.0p-53;
}
// FP_STAGE_TIMING builds: globaltimer stamps between the plan-graph stages (diagnostics).
#ifdef FP_STAGE_TIMING
__global__ void fp_stamp_kernel(unsigned long long* t);
#define FP_STAMP(ctx, strm, slot) fp_launch(fp_stamp_kernel, 1, 1, 0, (strm), &(ctx)->d_sc->plan_prof[slot])
#else
#define FP_STAMP(ctx, strm, slot) ((void)0)
#endif
#define FP_MOVE_ORDER_STREAM (1ULL << 63)
#define FP_SPAWN_STREAM ((1ULL << 63) + 1)

// Device-resident per-step scalars (graph-friendly: kernels read them, nothing is baked in).
struct DevScalars {
    long long step;               // SimState::step
    unsigned long long n_alive;   // alive count entering the motion phase (select output)
    unsigned long long alive;     // running alive count
    unsigned long long round_seq; // motion round stamp counter
    unsigned long long pend;      // pending count (motion)
    unsigned long long n_exits;   // exits of the current move phase
    unsigned long long disp;      // displacement of the current move phase (low 32 bits: hops;
                                  //   high 32 bits: sum of segment_dx, split off at the end)
    long long step_dx;            // sum of segment_dx(start, end) over the last move phase
    unsigned long long tot_exits; // accumulated over a run
    unsigned long long tot_disp;  // accumulated over a run
    long long tot_dx;             // sum of segment_dx over the run (fundamental-diagram flow)
    unsigned long long tot_updates;  // sum of alive counts entering each step
    unsigned long long fallbacks; // exact-path re-samples
    unsigned long long n_tiles;   // non-empty plan tiles this step
    unsigned long long n_items;   // motion seed work items (<= SEED_ITEM agents of one tile)
    unsigned long long exits_sorted;  // the motion graph sorted this phase's exit records
    unsigned long long tile_next; // dynamic tile scheduler cursor
    unsigned long long err;       // device-detected errors (bit flags)
    unsigned long long pad[2];    // [0] unsafe plane cells, [1] motion rounds executed
    unsigned long long fb_count;  // agents queued for the exact planning path this step
    unsigned long long t_motion[4];  // globaltimer: motion start, seed done, grid rounds done, end
    unsigned long long grid_rounds;  // rounds of the last motion phase run grid-wide
    unsigned long long t_marked;     // globaltimer: contention marks complete
    unsigned long long contended;    // movers handed to the reservation rounds, last phase
    unsigned long long t_prep;       // globaltimer: reservation buckets built
    unsigned long long t_round[64];  // globaltimer at the start of grid round r (r < 64)
    unsigned long long n_round[64];  // pending agents entering grid round r
    unsigned long long chk_max[64];  // diagnostics: longest full check of round r (SM clocks)
    unsigned long long chk_cnt[64];  //   full checks in round r
    unsigned long long p1_max[64];   //   longest pass-1 loop of a thread in round r (SM clocks)
    unsigned long long n_planned;    // agents the plan bucketed this step (= records in rec0)
    unsigned long long strip_nc;     // strip mode: contended walks listed for the deferral closure
    unsigned long long strip_rexits; // strip mode: exits of the resolved (deferred) walks
    unsigned long long strip_rhops;  // strip mode: hops | dx << 32 of the resolved walks
    unsigned long long plan_prof[8]; // FP_PLAN_PROF builds: plan-kernel wait / work cycle counters
    unsigned long long n_plan_items; // plan items this step (bucket.cu)
    unsigned long long t_step0;      // globaltimer: start of this step's plan phase (run/step kernels)
    unsigned long long t_plan_end;   // globaltimer: start of this step's motion phase
    unsigned long long plan_ns;      // plan / motion phase time summed over a run (device clock)
    unsigned long long move_ns;
};

// x-strip decomposition of one simulation over several GPUs (strip.cu).
#define FP_STRIP_NONE 0
#define FP_STRIP_HOST 1   // host callback allgather (fp_strip_set_exchange)
#define FP_STRIP_NCCL 2   // ncclAllGather on the context's stream (fp_strip_set_nccl)
#define FP_STRIP_LOCAL 3  // every rank's context in this process (fp_strips_step / fp_strips_run)
struct StripCtx {
    bool on = false;
    int rank = 0, nranks = 1, x_lo = 0, x_hi = 0;
    int transport = FP_STRIP_NONE;
    uint8_t* d_owned = nullptr;     // agent stands in this strip (alive and owned)
    uint32_t* d_dplane = nullptr;   // deferred footprint cells (bitplane)
    uint8_t* d_dflag = nullptr;     // per plan record: deferred
    uint32_t* d_clist = nullptr;    // contended plan records (closure candidates)
    void* d_send = nullptr;         // this rank's payload (header, deferred records, local exits)
    void* d_recv = nullptr;         // every rank's payload
    void* h_send = nullptr;         // pinned staging (host transport)
    void* h_recv = nullptr;
    size_t xbytes = 0;
    uint32_t cap_def = 0, cap_exit = 0, cap_def_req = 0, cap_exit_req = 0, cap_agents = 0, owned_cap = 0;
    uint64_t cap_total = 0;         // deferred records of all ranks the resolver takes
    uint32_t nslots = 0;            // resolver cell hash slots (power of two)
    uint32_t *d_hkey = nullptr, *d_hres = nullptr, *d_rslot = nullptr, *d_plist = nullptr;
    uint8_t* d_hocc = nullptr;
    unsigned long long* d_rexits = nullptr;
    unsigned long long* d_rhdr = nullptr;  // every rank's payload header (counts)
    unsigned long long* h_rhdr = nullptr;
    fp_allgather_fn host_fn = nullptr;
    void* host_user = nullptr;
    void* nccl_comm = nullptr;
    cudaEvent_t ev = nullptr;       // end of the send payload (local transport)
    cudaGraphExec_t graph_fin = nullptr;
};

struct fp_ctx {
    int device = 0;
    int sm_count = 148;
    cudaStream_t stream = nullptr;   // main stream
    cudaStream_t stream2 = nullptr;  // order (Fisher-Yates) branch
    cudaStream_t stream3 = nullptr;  // bucketing side branch (tile lists, plan items)
    cudaEvent_t ev_bfork = nullptr, ev_bjoin = nullptr;
    cudaStream_t stream4 = nullptr;  // alive compaction beside the shuffle (order.cu)
    cudaEvent_t ev_sfork = nullptr, ev_sjoin = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    std::string err;

    // geometry
    int W = 0, H = 0, boundary = 0, P = 0;
    double cell_size = 0.4;
    uint32_t* d_wall = nullptr;
    uint32_t* d_exit = nullptr;
    uint32_t* d_occ = nullptr;
    double* d_field = nullptr;
    uint32_t *d_p1 = nullptr, *d_p2 = nullptr;  // motion contention bitplanes (move.cu)

    // weight plane (plane.cu), valid for (plane_ks, plane_potential, plane_gradient)
    uint32_t* d_plane = nullptr;
    uint32_t* d_plane_t = nullptr;   // the same words chunk-tiled: [stripe][chunk][8 rows][tile_w + 16]
    int PW = 0;
    bool plane_valid = false;
    double plane_ks = 0.0;
    int plane_potential = -1;
    CUtensorMap tmap_plane;          // TMA descriptor of the plane: (tile_w + 16) words x 8 rows
    CUtensorMap tmap_occ;            // occupancy bitplane: 16 words x 8 rows
    CUtensorMap tmap_wall;           // the same box over the wall bitplane (line-of-sight masks)
    int tile_w = 0, tile_h = 0;      // plan tile (cells)
    int tiles_x = 0, tiles_y = 0;
    int cps = 0;                     // plan chunks (8 rows) per stripe: tiles_y * tile_h / 8
    bool tiles_ok = false;           // tiled fast path usable for this grid
    int use_tma = 1;                 // FP_NO_TMA=1 stages plan tiles with plain loads

    // potential
    int potential = FP_POTENTIAL_EXIT_DISTANCE;
    double drive_gradient = 0.0;

    // agents (SoA)
    uint32_t n = 0, cap = 0;
    int32_t *d_x = nullptr, *d_y = nullptr, *d_dx = nullptr, *d_dy = nullptr;
    uint8_t *d_v = nullptr, *d_alive = nullptr;
    uint32_t* d_rank = nullptr;
    int64_t step = 0;
    int64_t alive = 0;
    bool mixed_v = false;
    bool plan_marked = false;        // the last plan marked its movers' footprints in P1/P2
    int v_uniform = 1;               // the roster's v_max when not mixed (plan kernel variant)
    bool poisoned = false;  // a failed upload left the device roster inconsistent (capi.cu)
    int vmax_all = 1;

    // tile buckets
    uint32_t *d_tile_cnt = nullptr, *d_tile_off = nullptr, *d_tile_list = nullptr, *d_bucket = nullptr;
    uint32_t *d_sub_cnt = nullptr, *d_sub_off = nullptr;  // (tile, v_max) sub-buckets
    uint4* d_brec = nullptr;  // per bucket slot: (id, x, y, v_max) for the plan kernel
    uint8_t* d_tile_exit = nullptr;   // per plan tile: an Exit within its halo window (plane.cu)
    uint32_t* d_tile_deal = nullptr;  // [sm_count * DEAL_PASSES + 1] first tile-list entry per range
    int deal_passes = 1;              // passes actually used (FP_DEAL_PASSES, 1..DEAL_PASSES)
    size_t n_tiles_alloc = 0;
    size_t n_chunks_alloc = 0;
    uint32_t* d_scan_sums = nullptr;  // block sums of the chunk scan (bucket.cu)
    uint32_t* d_scan_sums2 = nullptr; // block sums of the order's scans (order.cu, stream2)
    uint32_t* d_scan_sums3 = nullptr; // block sums of the alive compaction beside it (stream4)
    uint4* d_plan_items = nullptr;     // plan kernel work items (bucket.cu)
    size_t plan_items_alloc = 0;
    uint2* d_seed_items = nullptr;    // (tile-list entry, chunk) per motion seed work item
    size_t seed_items_alloc = 0;

    // order scratch (sized by cap)
    uint32_t *d_alive_ids = nullptr, *d_order = nullptr, *d_j = nullptr, *d_cnt = nullptr,
             *d_off = nullptr, *d_cursor = nullptr, *d_fy_bucket = nullptr, *d_succ = nullptr,
             *d_nxt = nullptr, *d_V = nullptr, *d_flags = nullptr, *d_cursor_b = nullptr;
    uint32_t n_order = 0;  // alive count of the last computed order

    // motion scratch
    uint32_t *d_pend_a = nullptr, *d_pend_b = nullptr;
    uint2* d_fallback = nullptr;  // (id, bucket position) the plan kernel hands to the exact path
    uint4 *d_rec_a = nullptr, *d_rec_b = nullptr;  // motion pending records (move.cu)
    uint4* d_rec0 = nullptr;    // walk records in plan-tile order, emitted by the plan phase
    // motion reservation rounds (move.cu): rank buckets (8-word chunk per cell + overflow pool,
    // all-empty between phases) and per-agent entries
    uint32_t* d_bkt = nullptr;     // motion buckets: counters, bases, current positions, ranks, scan counts
    uint8_t* d_bdone = nullptr;    // motion buckets: per-position done flags
    uint2* d_entry = nullptr;      // (position, bucket) per footprint cell of a contended agent
    uint2* d_pw = nullptr;         // per bitplane word: (contended cells before it, its P2 bits)
    unsigned bk_agent_cap = 0, bk_nb_cap = 0, bk_npos_cap = 0;
    bool bucket_fresh = false;  // plan-tile buckets match the current positions
    bool rec_fresh = false;     // d_rec0 + contention marks match the current desired cells
    bool marks_dirty = false;   // contention bitplanes hold marks no motion phase consumed
    unsigned long long* d_exits = nullptr;  // (rank << 32 | id) records of the last move
    unsigned long long* d_exits_sorted = nullptr;
    int64_t last_displacement = 0;
    int64_t last_dx = 0;          // sum of segment_dx of the last move phase (fundamental diagram)
    int64_t dev_step = -1, dev_alive = -1;  // what the device scalars hold (sync_scalars skips repeats)
    uint32_t order_reserved_n = 0;          // fp_order_reserve done for this roster size
    size_t bucket_reserved_nt = 0;          // fp_bucket_reserve done for this tile count / roster
    uint32_t bucket_reserved_cap = 0;
    uint32_t n_exits = 0;

    DevScalars* d_sc = nullptr;   // device scalars
    DevScalars* h_sc = nullptr;   // pinned mirror
    unsigned long long* d_counters = nullptr;  // legacy scratch (errors of uploads)
    unsigned long long* h_counters = nullptr;
    void* d_scratch_small = nullptr;  // 4 KB: single-agent host-API calls (fp_choose_desired, ...)
    void* h_scratch_small = nullptr;

    // cub temp: order stage (two halves: scan | select) and bucketing stage
    void* d_temp = nullptr;
    size_t temp_bytes = 0;
    void* d_temp_b = nullptr;
    size_t temp_b_bytes = 0;

    // captured step graphs (fp_run): plan phase (bucketing + plan || order) and move phase
    cudaGraphExec_t graph_plan = nullptr;
    cudaGraphExec_t graph_move = nullptr;
    cudaGraphExec_t graph_multi = nullptr;  // run(): FP_RUN_UNROLL steps (plan, move child graphs) in one graph
    int run_unroll = 0;
    double graph_ks = 0.0;
    uint64_t graph_seed = 0;
    bool graph_valid = false;
    int move_blocks = 0;
    int64_t launches_per_step = 0;  // kernels in one replay of the two step graphs

    fp_counters ctr{};
    StripCtx st;
};

// -------------------------------------------------------------------------- error helpers
void fp_set_global_error(const std::string& s);
int fp_cuda_fail(fp_ctx* ctx, cudaError_t e, const char* what);
int fp_fail(fp_ctx* ctx, int code, const std::string& msg);

#define FP_CUDA(ctx, call)                                                   \
    do {                                                                     \
        cudaError_t e__ = (call);                                            \
        if (e__ != cudaSuccess) return fp_cuda_fail((ctx), e__, #call);       \
    } while (0)

#define FP_LAUNCHED(ctx)                                                     \
    do {                                                                     \
        (ctx)->ctr.kernel_launches++;                                        \
        cudaError_t e__ = cudaGetLastError();                                \
        if (e__ != cudaSuccess) return fp_cuda_fail((ctx), e__, "launch");   \
    } while (0)

// Warp-aggregated counter reservation: the lanes of a warp holding the same key take
// consecutive slots of ctr[key] with one atomic per distinct key (lane order inside a key).
// Every lane of the warp must call it; `skip` keys reserve nothing (returns garbage).
__device__ __forceinline__ uint32_t fp_warp_slot(uint32_t* ctr, uint32_t key, uint32_t skip) {
    const uint32_t peers = __match_any_sync(0xffffffffu, key);
    const int lane = threadIdx.x & 31, leader = __ffs(peers) - 1;
    uint32_t base = 0;
    if (lane == leader && key != skip) base = atomicAdd(&ctr[key], (uint32_t)__popc(peers));
    return __shfl_sync(0xffffffffu, base, leader) + (uint32_t)__popc(peers & ((1u << lane) - 1u));
}

__device__ __forceinline__ unsigned long long fp_globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

inline unsigned fp_blocks(size_t n, unsigned tpb) {
    size_t b = (n + tpb - 1) / tpb;
    return (unsigned)(b == 0 ? 1 : b);
}

inline Geo fp_geo(const fp_ctx* c) { return Geo{c->W, c->H, c->boundary, c->P, c->d_wall, c->d_exit}; }

// Stage entry points.
int fp_plane_ensure(fp_ctx* ctx, double k_s);                         // plane.cu
int fp_ghost_occ(fp_ctx* ctx);                                        // plane.cu
int fp_ghost_static(fp_ctx* ctx);                                     // plane.cu
int fp_bucket_launch(fp_ctx* ctx);                                    // bucket.cu
// plan.cu; wait_before_kernel: an event the stream kernel waits for (the movement order branch)
int fp_plan_launch(fp_ctx* ctx, double k_s, uint64_t seed, cudaEvent_t wait_before_kernel = nullptr);
int fp_plan_exact_launch(fp_ctx* ctx, double k_s, uint64_t seed);     // plan.cu
int fp_order_launch(fp_ctx* ctx, uint64_t seed, cudaStream_t s);     // order.cu
int fp_motion_launch(fp_ctx* ctx, bool spatial);                      // move.cu
int fp_exits_finish(fp_ctx* ctx);                                     // move.cu
int fp_field_compute(fp_ctx* ctx, const uint8_t* d_cells);            // field.cu
int fp_choice_launch(fp_ctx* ctx, uint32_t agent, double k_s, int32_t* d_cx, int32_t* d_cy,
                     double* d_w, float* d_p, uint32_t* d_n);         // plan.cu
int fp_choose_one_launch(fp_ctx* ctx, uint32_t id, int px, int py, int v, int64_t step, double k_s, uint64_t seed,
                         int32_t* d_out);                                  // plan.cu
int fp_candidates_one_launch(fp_ctx* ctx, int px, int py, int v, int32_t* d_cx, int32_t* d_cy, uint32_t* d_n);
int fp_order_positions(fp_ctx* ctx, uint32_t n, uint64_t seed, int64_t step, uint32_t* d_out);
int fp_ensure_temp(fp_ctx* ctx, size_t bytes);
int fp_ensure_res(fp_ctx* ctx);
int fp_order_reserve(fp_ctx* ctx);                                    // order.cu
int fp_plan_prepare(fp_ctx* ctx, double k_s);                         // plan.cu
bool fp_plan_tiled(const fp_ctx* ctx);
int fp_bucket_reserve(fp_ctx* ctx);                                   // bucket.cu
uint32_t fp_plan_chunks(const fp_ctx* ctx);
int fp_scan_u32(fp_ctx* ctx, const uint32_t* in, uint32_t* out, uint32_t n, uint32_t* sums,
                cudaStream_t s);                                      // scan.cu
int fp_select_alive(fp_ctx* ctx, const uint8_t* alive, uint32_t n, uint32_t* ids, unsigned long long* count,
                    uint32_t* sums, cudaStream_t s);
int fp_exits_sort_launch(fp_ctx* ctx);                                // move.cu
int fp_strip_reserve(fp_ctx* ctx);                                    // strip.cu
int fp_strip_begin_launch(fp_ctx* ctx);
int fp_strip_defer_launch(fp_ctx* ctx);
int fp_strip_pack_launch(fp_ctx* ctx);
int fp_strip_resolve_launch(fp_ctx* ctx);
int fp_strip_owned_init(fp_ctx* ctx);
int fp_strip_exchange(fp_ctx* ctx);
size_t fp_strip_def_off();
size_t fp_strip_exit_off(const fp_ctx* ctx);
size_t fp_strip_hdr_bytes();
int fp_strip_nccl_init(fp_ctx* ctx, const fp_nccl_id* id);
void fp_strip_nccl_destroy(fp_ctx* ctx);
