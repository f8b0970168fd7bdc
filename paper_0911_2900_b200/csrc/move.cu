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
//      reservation plane needs no stamps; the tail resets the keys of the agents it takes over,
//      so the plane ends every phase all-free.
// The result equals the sequential walk bit for bit (tests/test_gpu_parity.py).
//
// One cooperative launch runs a whole phase: grid-wide stages (grid.sync between them) while
// many agents are pending, then block 0 finishes the last TAIL_MAX alone in shared memory
// while the other blocks zero the contention bitplanes for the next phase.
#include <cooperative_groups.h>

#include "motion_rec.cuh"
#include "scan.cuh"

namespace cg = cooperative_groups;

#define MOVE_THREADS 512
#ifndef FP_MOVE_BLOCKS_PER_SM
#define FP_MOVE_BLOCKS_PER_SM 2  // cooperative CTAs per SM (bounded by occupancy)
#endif

__constant__ signed char c_bpath[121][5][2];
static bool g_bpath_ready[64] = {false};

struct MoveArgs {
    Geo g;
    uint32_t* occ;
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
    int premarked;                 // mode A with the footprints already marked by the plan
    uint4* rec[2];                 // pending records, ping-pong
    unsigned int* pcount;          // [0..1] list counts, [4..6] round pending counts, [7] long buckets (zero between phases)
    DevScalars* sc;
    unsigned long long* exits;     // (rank << 32 | id)
    uint32_t* p1;                  // contention bitplanes, zero between phases
    uint32_t* p2;
    // plan tiles (mode A): rec0[tile_off[t] + k], k < tile_cnt[t], for t in tile_list
    const uint32_t* tile_list;
    const uint32_t* tile_off;
    const uint32_t* tile_cnt;
    const uint2* items;            // seed work items: (tile-list entry, chunk of SEED_ITEM agents)
    int tile_w, tile_h, tiles_x;
    // reservation rounds (see the bucket notes below)
    const uint4* crec;             // contended records (= rec[1]), rank in .y
    uint2* pw;                     // per bitplane word: (contended cells before it, its P2 bits)
    unsigned p2g;                  // G: the grid of p2_count / p2_number (<= BK_SCAN2 - 1)
    unsigned* scan;                // [0, G) per-CTA contended cells, [G] their total;
                                   // [BK_SCAN2, BK_SCAN2 + G) per-CTA bucket entries, + G total
    unsigned nb_cap;               // buckets (contended cells): <= 3 per contended agent
    unsigned npos_cap;             // bucket positions: <= 6 per contended agent
    unsigned* bcnt;                // per bucket: entries counted (zero between phases)
    unsigned* bbase;               // per bucket: its first position
    unsigned* bown;                // per bucket: position of the agent standing on the cell, BK_NIL if none
    uint8_t* bocc0;                // per bucket: the cell's occupancy when the rounds begin
    uint2* brank;                  // per position (placement order): (rank, agent * 8 + cell)
    unsigned* long_list;           // buckets longer than BK_SORT_REG (ranked by warps)
    uint8_t* bdone;                // per position (rank order): 0 pending, 1 walked, 2 walked and stopped here
    uint8_t* eoff;                 // 8 per contended agent: offset of its position in each bucket
    uint4* ck;                     // 2 per contended agent: what a check reads (bk_final_kernel)
    uint2* entry;                  // 6 per contended agent: (slot, then position; bucket) per
                                   // footprint cell; BK_NIL/BK_NIL for an uncontended cell
    // contended-index pending lists (ping-pong), carved from rec[0] (free after step 2)
    uint2* alist[2];               // (contended index, position of the predecessor it waits on)
};

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// One L2 load per CTA, broadcast through shared memory: a word every thread of the grid reads
// right after a barrier would otherwise queue thousands of warp requests at one L2 slice.
__device__ __forceinline__ unsigned long long cta_load(const unsigned long long* p) {
    __shared__ unsigned long long s_v;
    __syncthreads();  // earlier readers are done with s_v
    if (threadIdx.x == 0) s_v = __ldcg(p);
    __syncthreads();
    return s_v;
}
__device__ __forceinline__ unsigned cta_load(const unsigned* p) {
    __shared__ unsigned s_u;
    __syncthreads();
    if (threadIdx.x == 0) s_u = __ldcg(p);
    __syncthreads();
    return s_u;
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

__device__ __forceinline__ void bar_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// A thread group that synchronises on one hardware barrier: the whole CTA (barrier 0) or one
// of the seed workers.  s[0] collects the group's append count, s[1] receives its list base,
// s64 the group's displacement sum -- so each append or flush costs one global atomic per group
// (per-warp atomics on one counter serialise thousands of requests at a single L2 slice).
struct Group {
    int bar, n;
    bool leader;
    unsigned* s;
    unsigned long long* s64;
    __device__ __forceinline__ void sync() const { bar_sync(bar, n); }
};

// Appends v to list when take.  Every thread of the group calls it.
template <typename T>
__device__ __forceinline__ void append(const Group& G, unsigned int* count, T* list, bool take, const T& v) {
    const unsigned mask = __ballot_sync(0xffffffffu, take);
    const int lane = threadIdx.x & 31;
    unsigned wo = 0;
    if (lane == 0 && mask) wo = atomicAdd(&G.s[0], (unsigned)__popc(mask));
    wo = __shfl_sync(0xffffffffu, wo, 0);
    G.sync();
    if (G.leader) {
        const unsigned c = G.s[0];
        G.s[1] = c ? atomicAdd(count, c) : 0u;
        G.s[0] = 0;
    }
    G.sync();
    if (take) list[G.s[1] + wo + __popc(mask & ((1u << lane) - 1))] = v;
}

// cx[j], cy[j] for a run-time j without spilling the arrays to local memory.
__device__ __forceinline__ void pick(const int* cx, const int* cy, int j, int& x, int& y) {
    x = cx[0];
    y = cy[0];
#pragma unroll
    for (int i = 1; i < 5; ++i)
        if (i == j) {
            x = cx[i];
            y = cy[i];
        }
}

// Occupancy of the path cells, all loads in flight together.
__device__ __forceinline__ void load_blocked(const MoveArgs& a, const int* cx, const int* cy, int m, bool* blocked) {
#pragma unroll
    for (int i = 0; i < 5; ++i) blocked[i] = i < m && occ_test(a, cx[i], cy[i]);
}

// Per-thread displacement accumulator word: hops in the low 32 bits, the signed sum of
// segment_dx (engine end x minus start x, periodic shorter wrap; the fundamental diagram's
// flow, bench.hpp:291-302) in the high 32 bits.  Phase totals stay below 2^31, so the halves
// never carry into each other; the motion kernel splits them at the end of the phase.
__device__ __forceinline__ unsigned long long hop_word(int h, int dx) {
    return (unsigned long long)(unsigned)h + ((unsigned long long)(unsigned)dx << 32);
}


// The walk (engine.hpp:116-129) of an agent that owns its footprint, net effect on occupancy.
__device__ __forceinline__ void walk_apply(const MoveArgs& a, const uint4& r, const int* cx, const int* cy, int m,
                                           const bool* blocked, unsigned long long* hops_acc) {
    const int sx = rec_x(r), sy = rec_y(r);
    int h = 0;
#pragma unroll
    for (int i = 0; i < 5; ++i)
        if (i < m && h == i && !blocked[i]) h = i + 1;
    const bool exited = (h == m) && (r.z & 0x80000000u);
    int dxs = 0;
    if (h > 0) {
        const uint32_t id = r.x;
        atomicAnd(&a.occ[a.g.word(sx, sy)], ~(1u << (sx & 31)));
        int fx, fy;
        pick(cx, cy, h - 1, fx, fy);
        dxs = a.g.segment_dx(sx, fx);
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
    *hops_acc += hop_word(h, dxs);
}

__device__ __forceinline__ void walk_owned(const MoveArgs& a, const uint4& r, const int* cx, const int* cy, int m,
                                           unsigned long long* hops_acc) {
    bool blocked[5];
    load_blocked(a, cx, cy, m, blocked);
    walk_apply(a, r, cx, cy, m, blocked, hops_acc);
}

// ------------------------------------------------------------------ grid-wide reservation rounds
// Every contended cell (covered by two or more footprints, P2) is numbered densely (p2_number)
// and holds a bucket: the contended agents whose footprint has the cell, in rank (processing)
// order, at positions [bbase[b], bbase[b] + n_b) of one array.  When an agent walks
// (engine.hpp:116-129) a path cell c blocks it iff c is occupied at its turn, and for a contended
// cell that is decided by the bucket alone:
//   * the agent standing on c at the start (bown) has not walked yet -- it comes later in the
//     order -- or it is earlier and stayed;
//   * a static occupant (bocc0 without bown: nobody stands there who will move);
//   * an earlier agent of the bucket stopped on c.
// So an agent at position p resolves c as soon as the done bytes of the positions before p say
// so: a 2 there (an earlier agent ended its walk on c) blocks it whatever the pending ones do;
// all of them 1 (walked, left or passed) frees it; otherwise it waits for the first pending one.
// An agent walks once every path cell up to the one that stops it is resolved -- the cells
// behind that, and its own start cell, never make it wait -- and then writes its done bytes:
// 2 on the cell it ends on (its start if it stays), 1 on the others.  Nothing else of its walk
// is read by the other contended agents during the phase (an uncontended cell is only ever
// touched by its one agent); the one write that can collide is a later agent setting the
// occupancy bit of a start cell this agent cleared, so a release fence orders that clear before
// the done bytes when the agent leaves a contended start cell.
// bbase, bown and done are a few MB and stay in L2 through the rounds.  Built per phase by
//   bk_count  per contended agent: its slot k in each of its buckets (one atomic counter each),
//             the cells' occupancy (bocc0)
//   bk_scan   bbase = exclusive prefix of the bucket sizes (two passes like p2_number)
//   bk_place  brank[bbase + k] = (rank, agent * 8 + cell)
//   bk_sort   per bucket: each entry's position = bbase + #{ranks below its own}, handed to its
//             agent; bown; the bucket's done flags cleared
#define BK_EMPTY 0xFFFFFFFFu
// Release/acquire is all the walk -> advanced-cell handoff needs (MEMBAR.ALL.GPU, not the
// sequentially consistent MEMBAR.SC.GPU that __threadfence() emits).
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
#define BK_NIL 0xFFFFFFFFu
#define BK_NOWATCH 0xFFFFFFFFu
#define BK_SCAN2 1024  // offset of the bucket-size scan counts in MoveArgs::scan
#ifndef BK_PREP_BATCH
#define BK_PREP_BATCH 2  // contended agents per thread per prep step
#endif

// Bucket of cell (x, y) when two or more footprints cover it (P2), else BK_NIL.  The contended
// cells are numbered densely in bitplane order (p2_number); a cell only one footprint covers
// needs no bucket (its agent is trivially the earliest there).
__device__ __forceinline__ unsigned bucket_of(const MoveArgs& a, int x, int y) {
    const uint2 q = __ldcg(&a.pw[a.g.word(x, y)]);
    const uint32_t bit = 1u << (x & 31);
    return (q.y & bit) ? q.x + (unsigned)__popc(q.y & (bit - 1u)) : BK_NIL;
}

// Buckets of a record's footprint cells: [0] start, [1..mf] path (motion_rec.cuh), BK_NIL for
// cells no other footprint covers; returns mf.
__device__ __forceinline__ int footprint(const MoveArgs& a, const uint4& r, const signed char (*bp)[5][2],
                                         unsigned* cell, bool* occ = nullptr) {
    int cx[5], cy[5];
    path_of(a, r, bp, cx, cy);
    const int m = rec_mf(r);
    cell[0] = bucket_of(a, rec_x(r), rec_y(r));
    if (occ) occ[0] = true;  // its own agent stands there
#pragma unroll
    for (int j = 0; j < 5; ++j)
        if (j < m) {
            cell[j + 1] = bucket_of(a, cx[j], cy[j]);
            if (occ) occ[j + 1] = occ_test(a, cx[j], cy[j]);
        }
    return m;
}

__device__ __forceinline__ void load_pairs(const MoveArgs& a, unsigned ci, unsigned* slot, unsigned* cell) {
    const uint4* p = reinterpret_cast<const uint4*>(a.entry + (size_t)ci * 6);
#pragma unroll
    for (int h = 0; h < 3; ++h) {
        const uint4 q = __ldcg(p + h);
        slot[2 * h] = q.x;
        cell[2 * h] = q.y;
        slot[2 * h + 1] = q.z;
        cell[2 * h + 1] = q.w;
    }
}

__device__ __forceinline__ void store_pairs(const MoveArgs& a, unsigned ci, const unsigned* slot,
                                            const unsigned* cell) {
    uint4* p = reinterpret_cast<uint4*>(a.entry + (size_t)ci * 6);
#pragma unroll
    for (int h = 0; h < 3; ++h) p[h] = make_uint4(slot[2 * h], cell[2 * h], slot[2 * h + 1], cell[2 * h + 1]);
}

// B contended agents at once: records, then their bucket lookups, then the counter atomics.
template <int B>
__device__ __forceinline__ void bk_count(const MoveArgs& a, const unsigned* ci, const bool* ok,
                                         const signed char (*bp)[5][2]) {
    uint4 r[B];
#pragma unroll
    for (int b = 0; b < B; ++b) r[b] = ok[b] ? __ldcg(&a.crec[ci[b]]) : make_uint4(0, 0, 0, 0);
    unsigned cell[B][6];
    bool occ[B][6];
    int m[B];
#pragma unroll
    for (int b = 0; b < B; ++b) m[b] = ok[b] ? footprint(a, r[b], bp, cell[b], occ[b]) : -1;
#pragma unroll
    for (int b = 0; b < B; ++b) {
        if (!ok[b]) continue;
        unsigned slot[6], c6[6];
#pragma unroll
        for (int j = 0; j < 6; ++j) {
            c6[j] = j <= m[b] ? cell[b][j] : BK_NIL;
            slot[j] = c6[j] != BK_NIL ? atomicAdd(&a.bcnt[c6[j]], 1u) : BK_NIL;
        }
#pragma unroll
        for (int j = 0; j < 6; ++j)
            if (c6[j] != BK_NIL) a.bocc0[c6[j]] = occ[b][j];  // every writer of a cell agrees
        store_pairs(a, ci[b], slot, c6);
        a.alist[0][ci[b]] = make_uint2(ci[b], BK_NOWATCH);
    }
}

__device__ __forceinline__ void bk_slice(unsigned nbu, unsigned& b0, unsigned& b1) {
    const unsigned per = (nbu + gridDim.x - 1) / gridDim.x;
    b0 = min(nbu, blockIdx.x * per);
    b1 = min(nbu, b0 + per);
}

__device__ __forceinline__ unsigned block_sum(unsigned v, unsigned* red);

__device__ void bk_scan_count(const MoveArgs& a, unsigned nbu, unsigned* red) {
    unsigned b0, b1;
    bk_slice(nbu, b0, b1);
    unsigned c = 0;
    for (unsigned b = b0 + threadIdx.x; b < b1; b += blockDim.x) c += __ldcg(&a.bcnt[b]);
    c = block_sum(c, red);
    if (threadIdx.x == 0) a.scan[BK_SCAN2 + blockIdx.x] = c;
}

__device__ void bk_scan_base(const MoveArgs& a, unsigned nbu, unsigned* red) {
    unsigned b0, b1;
    bk_slice(nbu, b0, b1);
    unsigned off = 0;
    for (unsigned b = threadIdx.x; b < blockIdx.x; b += blockDim.x) off += __ldcg(&a.scan[BK_SCAN2 + b]);
    off = block_sum(off, red);
    const unsigned per = (b1 - b0 + blockDim.x - 1) / blockDim.x;
    const unsigned t0 = min(b1, b0 + threadIdx.x * per), t1 = min(b1, t0 + per);
    unsigned mine = 0;
    for (unsigned b = t0; b < t1; ++b) mine += __ldcg(&a.bcnt[b]);
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned incl = mine;
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (unsigned)o) incl += t;
    }
    __syncthreads();  // red is free
    if (lane == 31) red[warp] = incl;
    __syncthreads();
    unsigned before = 0;
    for (unsigned k = 0; k < warp; ++k) before += red[k];
    unsigned e = off + before + incl - mine;
    for (unsigned b = t0; b < t1; ++b) {
        a.bbase[b] = e;
        e += __ldcg(&a.bcnt[b]);
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == blockDim.x - 1 && e > a.npos_cap)
        atomicOr(&a.sc->err, 16ull);  // cannot happen: <= 6 positions per contended agent
}

template <int B>
__device__ __forceinline__ void bk_place(const MoveArgs& a, const unsigned* ci, const bool* ok) {
    unsigned rank[B], slot[B][6], cell[B][6], base[B][6];
#pragma unroll
    for (int b = 0; b < B; ++b)
        if (ok[b]) {
            rank[b] = __ldcg(&a.crec[ci[b]]).y;
            load_pairs(a, ci[b], slot[b], cell[b]);
        }
#pragma unroll
    for (int b = 0; b < B; ++b)
#pragma unroll
        for (int j = 0; j < 6; ++j)
            if (ok[b] && cell[b][j] != BK_NIL) base[b][j] = __ldcg(&a.bbase[cell[b][j]]);
#pragma unroll
    for (int b = 0; b < B; ++b)
#pragma unroll
        for (int j = 0; j < 6; ++j)
            if (ok[b] && cell[b][j] != BK_NIL)
                a.brank[base[b][j] + slot[b][j]] = make_uint2(rank[b], ci[b] * 8u + (unsigned)j);
}

// Bucket b in rank order: entry i (placement order) goes to position base + #{ranks below its
// own}; every agent learns its position, the cell's current position is its first, and the
// done flags of the bucket's positions are cleared.  Up to BK_SORT_REG entries in registers,
// longer buckets are handed to warps (bk_sort_long).
#define BK_SORT_REG 16
#define BK_SORT_MAX 128  // a cell is covered by at most 121 footprints
// An agent behind others in the bucket of its first path cell starts the rounds watching its
// predecessor there instead of being checked in round 0 (a watch only schedules the next check).
__device__ __forceinline__ void bk_hand_out(const MoveArgs& a, uint2 e, unsigned pos, unsigned base, unsigned b) {
    const unsigned ci = e.y >> 3, j = e.y & 7u;
    a.entry[(size_t)ci * 6 + j].x = pos;
    a.eoff[(size_t)ci * 8 + j] = (uint8_t)(pos - base);  // < BK_SORT_MAX
    a.bdone[pos] = 0;
    if (j == 0) a.bown[b] = pos;
    if (j == 1 && pos > base) a.alist[0][ci].y = pos - 1;
}

__device__ void bk_sort(const MoveArgs& a, unsigned nbu, unsigned gtid, unsigned nthreads) {
    for (unsigned b = gtid; b < nbu; b += nthreads) {
        const unsigned base = __ldcg(&a.bbase[b]), n = __ldcg(&a.bcnt[b]);
        a.bown[b] = BK_NIL;
        if (n > BK_SORT_REG) {
            a.long_list[atomicAdd(&a.pcount[7], 1u)] = b;
            continue;
        }
        uint2 e[BK_SORT_REG];
#pragma unroll
        for (int i = 0; i < BK_SORT_REG; ++i) e[i] = (unsigned)i < n ? __ldcg(&a.brank[base + i]) : make_uint2(BK_EMPTY, 0);
#pragma unroll
        for (int i = 0; i < BK_SORT_REG; ++i) {
            if ((unsigned)i >= n) continue;
            unsigned below = 0;
#pragma unroll
            for (int k = 0; k < BK_SORT_REG; ++k) below += e[k].x < e[i].x;
            bk_hand_out(a, e[i], base + below, base, b);
        }
    }
}

// One warp per long bucket: its entries staged in shared memory, each placed by counting.
__device__ void bk_sort_long(const MoveArgs& a, unsigned* scratch) {
    const unsigned nl = cta_load(&a.pcount[7]);
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    unsigned* srk = scratch + warp * BK_SORT_MAX;
    for (unsigned l = blockIdx.x * nw + warp; l < nl; l += gridDim.x * nw) {
        const unsigned b = __ldcg(&a.long_list[l]);
        const unsigned base = __ldcg(&a.bbase[b]), n = min(__ldcg(&a.bcnt[b]), (unsigned)BK_SORT_MAX);
        for (unsigned i = lane; i < n; i += 32) srk[i] = __ldcg(&a.brank[base + i]).x;
        __syncwarp();
        for (unsigned i = lane; i < n; i += 32) {
            const uint2 e = __ldcg(&a.brank[base + i]);
            unsigned below = 0;
            for (unsigned k = 0; k < n; ++k) below += srk[k] < e.x;
            bk_hand_out(a, e, base + below, base, b);
        }
        __syncwarp();
    }
}

// The done bytes of positions [lo, hi) of one bucket (the agents before hi there): 2 if one of
// them stopped on the cell, else 1 if all of them walked, else 0 with *q = the first pending.
// v holds the 32 bytes from lo & ~15 (loaded by the caller); longer ranges (at most 120
// positions before hi, so lo & ~15 + 144 covers them) load the rest at once.
__device__ __forceinline__ void bk_word(unsigned w, unsigned wa, unsigned lo, unsigned hi, bool& stop, unsigned& first) {
    unsigned in = 0xFFFFFFFFu;  // bytes of the word inside [lo, hi)
    if (wa < lo) in = lo - wa >= 4 ? 0u : in << (8 * (lo - wa));
    if (wa + 4 > hi) in = hi <= wa ? 0u : in & (0xFFFFFFFFu >> (8 * (wa + 4 - hi)));
    stop |= (w & in & 0x02020202u) != 0u;
    const unsigned z = ~(w | (w >> 1)) & in & 0x01010101u;
    if (z && first == BK_NIL) first = wa + (unsigned)((__ffs(z) - 1) >> 3);
}

__device__ __forceinline__ int bk_before(const MoveArgs& a, unsigned lo, unsigned hi, const uint4* v, unsigned* q) {
    unsigned first = BK_NIL;
    bool stop = false;
    const unsigned c0 = lo & ~15u;
#pragma unroll
    for (int k = 0; k < 8; ++k) bk_word((&v[k >> 2].x)[k & 3], c0 + 4 * k, lo, hi, stop, first);
    if (c0 + 32 < hi && !stop) {  // a long bucket: the rest (<= 112 more bytes) in one trip
        uint4 u[7];
#pragma unroll
        for (int h = 0; h < 7; ++h) {
            const unsigned c = c0 + 32 + 16 * h;
            u[h] = c < hi ? __ldcg(reinterpret_cast<const uint4*>(a.bdone + c)) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int h = 0; h < 7; ++h)
#pragma unroll
            for (int k = 0; k < 4; ++k) bk_word((&u[h].x)[k], c0 + 32 + 16 * h + 4 * k, lo, hi, stop, first);
    }
    if (stop) return 2;
    if (first == BK_NIL) return 1;
    *q = first;
    return 0;
}

// What a check of a contended agent reads, prepared once per phase after the buckets are sorted
// (bk_final_kernel), so a check is two trips (this, then the done bytes) instead of four.
// ck[2ci] = positions of footprint cells 0..3, ck[2ci+1] = (positions of cells 4, 5; bucket
// offsets of path cells 0..3 as bytes; offset of path cell 4 | codes << 8).  A position is BK_NIL
// for an uncontended cell.  Path cell i (footprint cell i + 1) has a 2-bit code: CK_FREE and
// CK_BLOCK are decided for the whole phase (an uncontended cell's occupancy; a static occupant
// or a start occupant later in the order), CK_DYN by the done bytes before its position.
#define CK_FREE 0u
#define CK_BLOCK 1u
#define CK_DYN 2u

// Check of pending agent ci: its path cells in walk order, each free, blocking or undecided
// (see the bucket notes).  Decided up to the cell that stops it, it walks and writes its done
// bytes; otherwise returns the pending position to watch.
__device__ __forceinline__ bool bk_check(const MoveArgs& a, unsigned ci, const signed char (*bp)[5][2],
                                         unsigned long long* hops, unsigned* watch) {
    const uint4 r = __ldcg(&a.crec[ci]);
    const uint4 k0 = __ldcg(&a.ck[2 * (size_t)ci]), k1 = __ldcg(&a.ck[2 * (size_t)ci + 1]);
    const unsigned pos[6] = {k0.x, k0.y, k0.z, k0.w, k1.x, k1.y};
    const unsigned codes = k1.w >> 8;
    int cx[5], cy[5];
    const int m = path_of(a, r, bp, cx, cy);
    unsigned base[5];
    uint4 dv[5][2];
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        base[i] = 0;
        dv[i][0] = dv[i][1] = make_uint4(0, 0, 0, 0);
        if (i >= m || ((codes >> (2 * i)) & 3u) != CK_DYN) continue;
        const unsigned k = (i < 4 ? k1.z >> (8 * i) : k1.w) & 0xFFu;
        base[i] = pos[i + 1] - k;
        const unsigned c0 = base[i] & ~15u;
        if (k) dv[i][0] = __ldcg(reinterpret_cast<const uint4*>(a.bdone + c0));
        if (c0 + 16 < pos[i + 1]) dv[i][1] = __ldcg(reinterpret_cast<const uint4*>(a.bdone + c0 + 16));
    }
    int h = 0;
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        if (i >= m || h != i) continue;
        const unsigned c = (codes >> (2 * i)) & 3u;
        if (c == CK_BLOCK) continue;
        if (c == CK_DYN) {
            unsigned q = 0;
            const int st = bk_before(a, base[i], pos[i + 1], dv[i], &q);
            if (st == 2) continue;  // an earlier agent stopped here
            if (st == 0) {
                *watch = q;
                return false;
            }
        }
        h = i + 1;
    }
    bool blocked[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) blocked[i] = i >= h;
    walk_apply(a, r, cx, cy, m, blocked, hops);
    // A later agent may end its walk on the start cell this one left (only if that cell is
    // contended): the cleared occupancy bit must be performed before the done bytes let it in,
    // or its set bit could be wiped.
    if (h > 0 && pos[0] != BK_NIL) fence_acq_rel_gpu();
    const bool exited = (h == m) && (r.z & 0x80000000u);
    const int jf = exited ? -1 : h;  // footprint index of the cell it ends on (0: it stays)
#pragma unroll
    for (int j = 0; j < 6; ++j)
        if (pos[j] != BK_NIL) a.bdone[pos[j]] = j == jf ? 2 : 1;
    return true;
}

// The late rounds, asynchronously: once at most MOVE_ASYNC_K pending agents per thread remain,
// each thread owns its share of the list (entry k of the list goes to thread k mod nthreads) and
// polls the done flag each agent watches, re-checking the agent as soon as it is set -- a chain
// advances one link per poll instead of one per grid round, and no barrier separates the links.
// An agent is only ever checked by its owner, so no two checks of one agent overlap; the globally
// earliest pending agent can always walk, and every owner stays resident (cooperative launch),
// so the phase finishes.  The entries live in the (then unused) dynamic shared memory.
#ifndef MOVE_ASYNC_K
#define MOVE_ASYNC_K 4
#endif
#ifndef MOVE_ASYNC_NAP
#define MOVE_ASYNC_NAP 128
#endif
__device__ void async_walk(const MoveArgs& a, const uint2* list, unsigned np, unsigned gtid, unsigned nthreads,
                           uint2* mine, const signed char (*bp)[5][2], unsigned long long* hops) {
    unsigned live = 0;
#pragma unroll
    for (int j = 0; j < MOVE_ASYNC_K; ++j) {
        const unsigned k = gtid + j * nthreads;
        if (k < np) {
            mine[j * blockDim.x] = __ldcg(&list[k]);
            live |= 1u << j;
        }
    }
    unsigned nap = 32;
    long long idle = 0;
    while (live) {
        unsigned v[MOVE_ASYNC_K];
#pragma unroll
        for (int j = 0; j < MOVE_ASYNC_K; ++j) {
            const unsigned w = ((live >> j) & 1u) ? mine[j * blockDim.x].y : BK_NOWATCH;
            v[j] = w != BK_NOWATCH ? __ldcg(&a.bdone[w]) : ((live >> j) & 1u);
        }
        bool prog = false;
#pragma unroll 1
        for (int j = 0; j < MOVE_ASYNC_K; ++j) {
            if (!v[j]) continue;
            const uint2 e = mine[j * blockDim.x];
            unsigned w;
            if (bk_check(a, e.x, bp, hops, &w)) {
                live &= ~(1u << j);
            } else {
                mine[j * blockDim.x].y = w;
            }
            prog = true;
        }
        if (prog) {
            nap = 32;
            continue;
        }
        __nanosleep(nap);
        nap = min(nap * 2u, (unsigned)MOVE_ASYNC_NAP);
        if (++idle > (1ll << 24)) {
            atomicOr(&a.sc->err, 32ull);
            return;
        }
    }
}

// Adds the group's hop counts to the phase displacement.  Every thread of the group calls it.
__device__ __forceinline__ void flush_hops(const Group& G, DevScalars* sc, unsigned long long hops) {
    for (int o = 16; o > 0; o >>= 1) hops += __shfl_down_sync(0xffffffffu, hops, o);
    if ((threadIdx.x & 31) == 0 && hops) atomicAdd(G.s64, hops);
    G.sync();
    if (G.leader) {
        if (*G.s64) atomicAdd(&sc->disp, *G.s64);
        *G.s64 = 0;
    }
    G.sync();
}

// ------------------------------------------------------------------ shared-memory tail rounds
// Once few agents are pending, block 0 resolves them alone: their footprint cells go into a
// shared-memory hash (cell -> reservation, occupancy), the rounds run entirely in shared memory
// with __syncthreads between phases, and the final occupancy is written back once.
#define TAIL_MAX 1024
#define TAIL_SLOTS 8192
#define TAIL_EMPTY 0xFFFFFFFFu

struct TailSmem {
    uint4 rec[TAIL_MAX];
    unsigned short slot[TAIL_MAX][6];
    unsigned short list[2][TAIL_MAX];
    unsigned int key[TAIL_SLOTS];
    unsigned int res[TAIL_SLOTS];
    unsigned char occ[TAIL_SLOTS];
    unsigned int count[2];
};

// Round queues in the same dynamic buffer (see the rounds in move_rounds_kernel).
#define QP_CAP 8192
#ifndef MOVE_LOCAL_ITERS
#define MOVE_LOCAL_ITERS 3     // extra in-CTA check passes per grid round
#endif
#define MOVE_LOCAL_MAX 4096    // ... while the CTA holds at most this many pending agents
#define QC_CAP 8192
#define MOVE_SEG 8192          // list entries a CTA takes per pass-1/pass-2 segment (<= both queue sizes)
// The kernel's dynamic shared memory serves, one after another, the seed windows, the long-bucket
// ranking, the round queues and the tail.
#define MOVE_DYN_SMEM (sizeof(TailSmem) > QP_CAP * sizeof(uint2) + QC_CAP * sizeof(unsigned) \
                           ? sizeof(TailSmem) : QP_CAP * sizeof(uint2) + QC_CAP * sizeof(unsigned))
static_assert((MOVE_THREADS / 32) * BK_SORT_MAX * sizeof(unsigned) <= MOVE_DYN_SMEM, "long-bucket ranking");
static_assert(MOVE_ASYNC_K * MOVE_THREADS * sizeof(uint2) <= MOVE_DYN_SMEM, "async entries");
static_assert(MOVE_SEG <= QC_CAP && MOVE_SEG <= QP_CAP && MOVE_SEG % (4 * MOVE_THREADS) == 0, "segment size");
static_assert(MOVE_ASYNC_K >= 1 && MOVE_ASYNC_K <= 32, "async entries per thread");

__device__ __forceinline__ unsigned tail_insert(TailSmem& T, const MoveArgs& a, int x, int y) {
    const unsigned cell = (unsigned)y * (unsigned)a.g.W + (unsigned)x;
    unsigned h = (cell * 2654435761u) >> (32 - 13);
    for (;;) {
        const unsigned old = atomicCAS(&T.key[h], TAIL_EMPTY, cell);
        if (old == TAIL_EMPTY) {  // new entry: its occupancy as of the tail's start
            T.occ[h] = (unsigned char)((__ldcg(&a.occ[a.g.word(x, y)]) >> (x & 31)) & 1u);
            return h;
        }
        if (old == cell) return h;
        h = (h + 1) & (TAIL_SLOTS - 1);
    }
}

// Pending records: crec[list[t]] (or crec[t] when list is null), t < np <= TAIL_MAX.
__device__ void tail_smem(const MoveArgs& a, TailSmem& T, const uint4* crec, const uint2* list, unsigned np,
                          const signed char (*bp)[5][2], unsigned long long* hops) {
    for (unsigned k = threadIdx.x; k < TAIL_SLOTS; k += blockDim.x) {
        T.key[k] = TAIL_EMPTY;
        T.res[k] = 0xFFFFFFFFu;
    }
    __syncthreads();
    for (unsigned t = threadIdx.x; t < np; t += blockDim.x) {
        const uint4 r = __ldcg(&crec[list ? __ldcg(&list[t].x) : t]);
        T.rec[t] = r;
        T.list[0][t] = (unsigned short)t;
        int cx[5], cy[5];
        path_of(a, r, bp, cx, cy);
        const int m = rec_mf(r);  // footprint cells only (a free exit ending the walk has no slot)
        T.slot[t][0] = (unsigned short)tail_insert(T, a, rec_x(r), rec_y(r));
#pragma unroll
        for (int i = 0; i < 5; ++i)
            if (i < m) T.slot[t][1 + i] = (unsigned short)tail_insert(T, a, cx[i], cy[i]);
    }
    if (threadIdx.x == 0) {
        T.count[0] = np;
        T.count[1] = 0;
    }
    __syncthreads();
    unsigned cur = 0, rounds = 0;
    for (;;) {
        const unsigned n = T.count[cur];
        if (n == 0) break;
        ++rounds;
        const unsigned nxt = cur ^ 1;
        for (unsigned k = threadIdx.x; k < n; k += blockDim.x) {
            const unsigned t = T.list[cur][k];
            const uint4 r = T.rec[t];
            const int m = rec_mf(r);
            for (int i = 0; i <= m; ++i) atomicMin(&T.res[T.slot[t][i]], r.y);
        }
        __syncthreads();
        if (threadIdx.x == 0) T.count[cur] = 0;  // read by everyone before the barrier above
        for (unsigned k = threadIdx.x; k < n; k += blockDim.x) {
            const unsigned t = T.list[cur][k];
            const uint4 r = T.rec[t];
            const int mf = rec_mf(r), m = rec_m(r);
            bool own = true;
            for (int i = 0; i <= mf && own; ++i) own = T.res[T.slot[t][i]] == r.y;
            if (!own) {
                T.list[nxt][atomicAdd(&T.count[nxt], 1u)] = (unsigned short)t;
                continue;
            }
            for (int i = 0; i <= mf; ++i) T.res[T.slot[t][i]] = 0xFFFFFFFFu;
            int h = 0;  // the walk (engine.hpp:116-129) against the shared occupancy
            while (h < mf && !T.occ[T.slot[t][1 + h]]) ++h;
            if (h == mf) h = m;  // a free exit ending the walk never blocks
            int dxs = 0;
            if (h > 0) {
                const bool exited = (h == m) && (r.z & 0x80000000u);
                T.occ[T.slot[t][0]] = 0;
                int cx[5], cy[5];
                path_of(a, r, bp, cx, cy);
                const uint32_t id = r.x;
                int fx, fy;
                pick(cx, cy, h - 1, fx, fy);
                dxs = a.g.segment_dx(rec_x(r), fx);
                a.x[id] = fx;
                a.y[id] = fy;
                if (exited) {
                    a.alive[id] = 0;
                    const unsigned long long s = atomicAdd(&a.sc->n_exits, 1ull);
                    a.exits[s] = ((unsigned long long)r.y << 32) | id;
                } else {
                    T.occ[T.slot[t][h]] = 1;
                }
            }
            *hops += hop_word(h, dxs);
        }
        __syncthreads();
        cur = nxt;
    }
    // write the final occupancy of every touched cell back to the bitplane
    for (unsigned s = threadIdx.x; s < TAIL_SLOTS; s += blockDim.x) {
        const unsigned cell = T.key[s];
        if (cell == TAIL_EMPTY) continue;
        const int x = (int)(cell % (unsigned)a.g.W), y = (int)(cell / (unsigned)a.g.W);
        const uint32_t bit = 1u << (x & 31);
        if (T.occ[s]) atomicOr(&a.occ[a.g.word(x, y)], bit);
        else atomicAnd(&a.occ[a.g.word(x, y)], ~bit);
    }
    if (threadIdx.x == 0) a.sc->pad[1] += rounds;
}

// ------------------------------------------------------------------ dense bucket numbering
// Contended cells (P2 bits) numbered in bitplane order: each CTA counts the bits of its slice of
// words (p2_count), then, after a grid barrier, numbers them from its prefix (p2_number), writing
// (contended cells before the word, the word's P2 bits) per word for bucket_of.
__device__ __forceinline__ void p2_slice(const MoveArgs& a, size_t& w0, size_t& w1) {
    const size_t nw = (size_t)a.g.P * (size_t)a.g.H;  // P is a multiple of 4
    const size_t per = ((nw / 4 + gridDim.x - 1) / gridDim.x) * 4;
    w0 = min(nw, (size_t)blockIdx.x * per);
    w1 = min(nw, w0 + per);
}

// Block-wide sum of v (every thread gets it); red = 32 words of shared scratch.
__device__ __forceinline__ unsigned block_sum(unsigned v, unsigned* red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();  // red is free
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    unsigned t = 0;
    for (unsigned w = 0; w < (blockDim.x >> 5); ++w) t += red[w];
    return t;
}

__device__ void p2_count(const MoveArgs& a, unsigned* red) {
    size_t w0, w1;
    p2_slice(a, w0, w1);
    unsigned c = 0;
    for (size_t w = w0 + 4 * (size_t)threadIdx.x; w < w1; w += 4 * (size_t)blockDim.x) {
        const uint4 q = __ldcg(reinterpret_cast<const uint4*>(a.p2 + w));
        c += __popc(q.x) + __popc(q.y) + __popc(q.z) + __popc(q.w);
    }
    c = block_sum(c, red);
    if (threadIdx.x == 0) a.scan[blockIdx.x] = c;
}

__device__ void p2_number(const MoveArgs& a, unsigned* red) {
    size_t w0, w1;
    p2_slice(a, w0, w1);
    unsigned off = 0;
    for (unsigned b = threadIdx.x; b < blockIdx.x; b += blockDim.x) off += __ldcg(&a.scan[b]);
    off = block_sum(off, red);
    // each thread numbers a contiguous run of words: count, one block scan, number
    const size_t per = (((w1 - w0) / 4 + blockDim.x - 1) / blockDim.x) * 4;
    const size_t t0 = min(w1, w0 + threadIdx.x * per), t1 = min(w1, t0 + per);
    unsigned mine = 0;
#pragma unroll 4
    for (size_t w = t0; w < t1; w += 4) {
        const uint4 q = __ldcg(reinterpret_cast<const uint4*>(a.p2 + w));
        mine += __popc(q.x) + __popc(q.y) + __popc(q.z) + __popc(q.w);
    }
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    unsigned incl = mine;
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (unsigned)o) incl += t;
    }
    __syncthreads();  // red is free
    if (lane == 31) red[warp] = incl;
    __syncthreads();
    unsigned before = 0;
    for (unsigned k = 0; k < warp; ++k) before += red[k];
    unsigned e = off + before + incl - mine;
#pragma unroll 4
    for (size_t w = t0; w < t1; w += 4) {
        const uint4 q = __ldcg(reinterpret_cast<const uint4*>(a.p2 + w));
        const unsigned c0 = __popc(q.x), c1 = __popc(q.y), c2 = __popc(q.z);
        uint4* out = reinterpret_cast<uint4*>(a.pw + w);
        out[0] = make_uint4(e, q.x, e + c0, q.y);
        out[1] = make_uint4(e + c0 + c1, q.z, e + c0 + c1 + c2, q.w);
        e += c0 + c1 + c2 + __popc(q.w);
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == blockDim.x - 1) {
        a.scan[gridDim.x] = e;  // contended cells (buckets) this phase
        if (e > a.nb_cap) atomicOr(&a.sc->err, 16ull);  // cannot happen: <= 3 per contended agent
    }
}

// Zeroes the contention bitplanes (dead after step 2) and the bucket counters of the phase's
// nbu buckets so the next phase starts from all-clear.
__device__ void zero_marks(const MoveArgs& a, unsigned nbu, unsigned part, unsigned parts) {
    for (unsigned b = part * blockDim.x + threadIdx.x; b < nbu; b += parts * blockDim.x) a.bcnt[b] = 0;
    const size_t nwords = (size_t)a.g.P * (size_t)a.g.H;  // P is a multiple of 4
    uint4* p1 = reinterpret_cast<uint4*>(a.p1);
    uint4* p2 = reinterpret_cast<uint4*>(a.p2);
    const uint4 z = make_uint4(0, 0, 0, 0);
    for (size_t k = (size_t)part * blockDim.x + threadIdx.x; k < nwords / 4; k += (size_t)parts * blockDim.x) {
        p1[k] = z;
        p2[k] = z;
    }
}

// ------------------------------------------------------------------ tiled seed (mode A)
// The plan left the records grouped by plan tile, and a footprint never leaves its tile by more
// than 5 cells.  So each tile's marks are gathered in a shared-memory window (tile + 5-cell
// halo) first and merged into the global bitplanes a word at a time, row-contiguous; the
// classification then stages the window of P2 and occupancy the same way.  Each CTA runs
// SEED_GROUPS independent 128-thread workers (named barriers), one tile each at a time.
#define SEED_GROUP 128
#define SEED_GROUPS (MOVE_THREADS / SEED_GROUP)

struct SeedWin {
    int wx0, ys, ww, wh;  // first word column (padded plane), first row, words per row, rows
    float inv_ww;         // row of window word w = (int)((w + 0.5f) * inv_ww)  (w < 2^12)
};

__device__ __forceinline__ void group_sync() {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + (int)(threadIdx.x / SEED_GROUP)), "r"(SEED_GROUP) : "memory");
}

__host__ __device__ __forceinline__ int seed_ww(int tile_w) { return (tile_w + 10 + 31) / 32 + 1; }

__device__ __forceinline__ SeedWin seed_window(const MoveArgs& a, uint32_t t) {
    SeedWin s;
    const int x0 = (int)(t % (uint32_t)a.tiles_x) * a.tile_w, y0 = (int)(t / (uint32_t)a.tiles_x) * a.tile_h;
    s.wx0 = (x0 - 5 + FP_XPAD_BITS) >> 5;
    s.ys = y0 - 5;
    s.ww = seed_ww(a.tile_w);
    s.wh = a.tile_h + 10;
    s.inv_ww = 1.0f / (float)s.ww;
    return s;
}

// Seed work item e: its tile and its agents [off, off + cnt) -- at most SEED_ITEM of the tile's.
__device__ __forceinline__ void seed_item(const MoveArgs& a, uint32_t e, uint32_t ni, uint32_t& t, uint32_t& off,
                                          uint32_t& cnt) {
    if (e >= ni) {
        t = off = cnt = 0;
        return;
    }
    const uint2 it = __ldcg(&a.items[e]);
    t = __ldcg(&a.tile_list[it.x]);
    const uint32_t c0 = it.y * SEED_ITEM, tc = __ldcg(&a.tile_cnt[t]);
    off = __ldcg(&a.tile_off[t]) + c0;
    cnt = min((uint32_t)SEED_ITEM, tc - c0);
}

// Local word index of cell (x, y) in the window, or -1 when it lies outside (periodic seam).
__device__ __forceinline__ int seed_local(const SeedWin& s, int x, int y) {
    const int wi = ((x + FP_XPAD_BITS) >> 5) - s.wx0, yi = y - s.ys;
    return (wi >= 0 && wi < s.ww && yi >= 0 && yi < s.wh) ? yi * s.ww + wi : -1;
}

// Global word of window word w, or -1 for rows outside the grid.
__device__ __forceinline__ long long seed_global(const MoveArgs& a, const SeedWin& s, int w) {
    const int yi = (int)(((float)w + 0.5f) * s.inv_ww);
    const int y = s.ys + yi;
    if (y < 0 || y >= a.g.H) return -1;
    return (long long)y * a.g.P + (s.wx0 + w - yi * s.ww);
}


// Start cell [0] and path cells [1..m]; the footprint is [0..mf] (motion_rec.cuh).
__device__ __forceinline__ void record_footprint(const MoveArgs& a, const uint4& r, const signed char (*bp)[5][2],
                                                 int* cx, int* cy, int& m, int& mf) {
    m = path_of(a, r, bp, cx + 1, cy + 1);
    mf = rec_mf(r);
    cx[0] = rec_x(r);
    cy[0] = rec_y(r);
}

// S1: every footprint of the group's tiles marked in P1/P2.  Tiles are dealt round-robin to
// the worker groups; the next tile's header and first records are fetched while the current
// tile's marks merge into the global bitplanes.
__device__ void seed_mark(const MoveArgs& a, uint32_t* win, const signed char (*bp)[5][2]) {
    const unsigned lt = threadIdx.x % SEED_GROUP;
    const uint32_t ni = (uint32_t)cta_load(&a.sc->n_items);
    const uint32_t ng = gridDim.x * SEED_GROUPS;
    uint32_t e = blockIdx.x * SEED_GROUPS + threadIdx.x / SEED_GROUP;
    uint32_t t, off, cnt;
    seed_item(a, e, ni, t, off, cnt);
    uint4 r0 = lt < cnt ? __ldcg(&a.rec0[off + lt]) : make_uint4(0, 0, 0, 0);
    for (; e < ni; e += ng) {
        const uint32_t en = e + ng;
        uint32_t tn, offn, cntn;
        seed_item(a, en, ni, tn, offn, cntn);
        const SeedWin s = seed_window(a, t);
        const int nw = s.ww * s.wh;
        uint32_t* L1 = win;
        uint32_t* L2 = win + nw;
        for (int w = lt; w < 2 * nw; w += SEED_GROUP) win[w] = 0;
        group_sync();
        for (uint32_t k = lt; k < cnt; k += SEED_GROUP) {
            const uint4 r = k == lt ? r0 : __ldcg(&a.rec0[off + k]);
            if (!rec_m(r)) continue;
            int cx[6], cy[6], m, mf;
            record_footprint(a, r, bp, cx, cy, m, mf);
#pragma unroll
            for (int i = 0; i < 6; ++i) {
                if (i > mf) continue;
                const uint32_t bit = 1u << (cx[i] & 31);
                const int w = seed_local(s, cx[i], cy[i]);
                if (w >= 0) {
                    if (atomicOr(&L1[w], bit) & bit) atomicOr(&L2[w], bit);
                } else {
                    const size_t gw = a.g.word(cx[i], cy[i]);
                    if (atomicOr(&a.p1[gw], bit) & bit) atomicOr(&a.p2[gw], bit);
                }
            }
        }
        group_sync();
        r0 = lt < cntn ? __ldcg(&a.rec0[offn + lt]) : make_uint4(0, 0, 0, 0);  // next tile, in flight
        // merge: four words per thread in flight at once, then the P2 updates fire-and-forget
        for (int w0 = lt; w0 < nw; w0 += 4 * SEED_GROUP) {
            uint32_t l1[4], old[4];
            long long gw[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int w = w0 + j * SEED_GROUP;
                l1[j] = w < nw ? L1[w] : 0u;  // marks only land on rows inside the grid
                gw[j] = l1[j] ? seed_global(a, s, w) : -1;
                old[j] = l1[j] ? atomicOr(&a.p1[gw[j]], l1[j]) : 0u;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (!l1[j]) continue;
                const uint32_t d = L2[w0 + j * SEED_GROUP] | (old[j] & l1[j]);
                if (d) atomicOr(&a.p2[gw[j]], d);
            }
        }
        group_sync();
        t = tn;
        off = offn;
        cnt = cntn;
    }
}

// S2: uncontended movers walk now; the rest go to the rounds (list rec[1]) with their rank.
// Tiles are dealt round-robin to the worker groups; the next tile's header is fetched while
// the current one is classified, and a tile's first records and their ranks travel with the
// window staging (the latency of a tile is what bounds this pass).
__device__ void seed_classify(const MoveArgs& a, const Group& G, uint32_t* win, const signed char (*bp)[5][2],
                              unsigned long long* hops) {
    const unsigned lt = threadIdx.x % SEED_GROUP;
    const uint32_t ni = (uint32_t)cta_load(&a.sc->n_items);
    const uint32_t ng = gridDim.x * SEED_GROUPS;
    uint32_t e = blockIdx.x * SEED_GROUPS + threadIdx.x / SEED_GROUP;
    uint32_t t, off, cnt;
    seed_item(a, e, ni, t, off, cnt);
    for (; e < ni; e += ng) {
        // next item's header in flight
        const uint32_t en = e + ng;
        uint32_t tn, offn, cntn;
        seed_item(a, en, ni, tn, offn, cntn);
        const SeedWin s = seed_window(a, t);
        const int nw = s.ww * s.wh;
        uint32_t* C2 = win;       // P2 window
        uint32_t* CO = win + nw;  // occupancy window
        const uint4 r0 = lt < cnt ? __ldcg(&a.rec0[off + lt]) : make_uint4(0, 0, 0, 0);
#pragma unroll 4
        for (int w = lt; w < nw; w += SEED_GROUP) {
            uint32_t v2 = 0, vo = 0;
            const long long gw = seed_global(a, s, w);
            if (gw >= 0) {
                v2 = __ldcg(&a.p2[gw]);
                vo = __ldcg(&a.occ[gw]);
            }
            C2[w] = v2;
            CO[w] = vo;
        }
        const uint32_t rk0 = (lt < cnt && rec_m(r0)) ? __ldcg(&a.rank[r0.x]) : 0u;
        group_sync();
        for (uint32_t base = 0; base < cnt; base += SEED_GROUP) {
            const uint32_t k = base + lt;
            bool contended = false;
            uint4 r = make_uint4(0, 0, 0, 0);
            if (k < cnt) {
                r = base == 0 ? r0 : __ldcg(&a.rec0[off + k]);
                if (rec_m(r)) {
                    int cx[6], cy[6], m, mf;
                    record_footprint(a, r, bp, cx, cy, m, mf);
                    bool blocked[5];
#pragma unroll
                    for (int i = 0; i < 6; ++i) {
                        if (i > m) continue;
                        const int sh = cx[i] & 31;
                        const int w = seed_local(s, cx[i], cy[i]);
                        uint32_t v2, vo;
                        if (w >= 0) {
                            v2 = C2[w];
                            vo = CO[w];
                        } else {
                            const size_t gw = a.g.word(cx[i], cy[i]);
                            v2 = __ldcg(&a.p2[gw]);
                            vo = __ldcg(&a.occ[gw]);
                        }
                        if (i <= mf) contended |= (v2 >> sh) & 1u;
                        if (i > 0) blocked[i - 1] = (vo >> sh) & 1u;
                    }
                    if (!contended) walk_apply(a, r, cx + 1, cy + 1, m, blocked, hops);
                    else r.y = base == 0 ? rk0 : __ldcg(&a.rank[r.x]);
                }
            }
            append(G, &a.pcount[1], a.rec[1], contended, r);
        }
        group_sync();
        t = tn;
        off = offn;
        cnt = cntn;
    }
}

// Step 2 for one record: walk now if uncontended, else hand it (with its rank) to the rounds.
__device__ __forceinline__ bool classify(const MoveArgs& a, uint4& rec, const signed char (*bp)[5][2],
                                         unsigned long long* hops) {
    int cx[5], cy[5];
    const int m = path_of(a, rec, bp, cx, cy), mf = rec_mf(rec);
    const int sx = rec_x(rec), sy = rec_y(rec);
    // the P2 loads and the (speculative) occupancy loads all in flight at once: if the footprint
    // is uncontended nobody else touches its cells this phase, so the occupancy read is final
    bool contended = (__ldcg(&a.p2[a.g.word(sx, sy)]) >> (sx & 31)) & 1u;
#pragma unroll
    for (int i = 0; i < 5; ++i)
        if (i < mf) contended |= (__ldcg(&a.p2[a.g.word(cx[i], cy[i])]) >> (cx[i] & 31)) & 1u;
    bool blocked[5];
    load_blocked(a, cx, cy, m, blocked);
    if (!contended) {
        walk_apply(a, rec, cx, cy, m, blocked, hops);
        return false;
    }
    rec.y = a.rank[rec.x];
    return true;
}

template <int PART>
__global__ void __launch_bounds__(MOVE_THREADS, 1) move_rounds_kernel(MoveArgs a) {
    FP_PDL_WAIT();
    cg::grid_group grid = cg::this_grid();
    __shared__ signed char s_bp[121][5][2];
    extern __shared__ __align__(16) unsigned char s_dyn[];  // TailSmem (block 0's tail) / seed windows
    __shared__ unsigned int s_app[2 + 2 * SEED_GROUPS];
    __shared__ unsigned long long s_hops[1 + SEED_GROUPS];
    __shared__ unsigned int s_q[3];  // round queue counts and the flush base
    __shared__ unsigned int s_red[32];  // block reductions (dense bucket numbering)
    for (int k = threadIdx.x; k < 121 * 10; k += blockDim.x) (&s_bp[0][0][0])[k] = (&c_bpath[0][0][0])[k];
    if (threadIdx.x < 3) s_q[threadIdx.x] = 0;
    if (threadIdx.x < 2 + 2 * SEED_GROUPS) s_app[threadIdx.x] = 0;
    if (threadIdx.x < 1 + SEED_GROUPS) s_hops[threadIdx.x] = 0;
    __syncthreads();
    const Group B{0, (int)blockDim.x, threadIdx.x == 0, &s_app[0], &s_hops[0]};
    const unsigned sg = threadIdx.x / SEED_GROUP;
    const Group Gs{1 + (int)sg, SEED_GROUP, threadIdx.x % SEED_GROUP == 0, &s_app[2 + 2 * sg], &s_hops[1 + sg]};
    const unsigned nthreads = gridDim.x * blockDim.x;
    const unsigned gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t n = (uint32_t)cta_load(&a.sc->n_alive);
    if (PART == 1) {  // steps 1 and 2
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
                    rec = record_of(a.g, a.occ, id, a.g.wrap(a.x[id]), a.y[id], tx, ty, a.v[id], s_bp);
                    take = rec_m(rec) > 0;
                    if (take) mark_record(a.p1, a.p2, a.g, rec, s_bp, tx, ty);
                }
                append(B, &a.pcount[0], a.rec[0], take, rec);
            }
            grid.sync();
            cand = a.rec[0];
            ncand = cta_load(&a.pcount[0]);
        } else {
            // steps 1 and 2 tile by tile over the plan's records
            const int nwmax = seed_ww(a.tile_w) * (a.tile_h + 10);
            uint32_t* win = reinterpret_cast<uint32_t*>(s_dyn) + (threadIdx.x / SEED_GROUP) * 2 * nwmax;
            if (!a.premarked) seed_mark(a, win, s_bp);
            grid.sync();
            if (gtid == 0) a.sc->t_marked = globaltimer();
            unsigned long long hops = 0;
            seed_classify(a, Gs, win, s_bp, &hops);
            flush_hops(B, a.sc, hops);
            ncand = 0;  // step 2 done
        }
        if (!a.premade && gtid == 0) a.sc->t_marked = globaltimer();
        // step 2
        {
            unsigned long long hops = 0;
            for (unsigned base = 0; base < ncand; base += nthreads) {
                const unsigned k = base + gtid;
                bool contended = false;
                uint4 rec = make_uint4(0, 0, 0, 0);
                if (k < ncand) {
                    rec = __ldcg(&cand[k]);
                    if (rec_m(rec)) contended = classify(a, rec, s_bp, &hops);
                }
                append(B, &a.pcount[1], a.rec[1], contended, rec);
            }
            flush_hops(B, a.sc, hops);
        }
        grid.sync();
        if (gtid == 0) {
            a.sc->t_motion[1] = globaltimer();
            a.sc->contended = __ldcg(&a.pcount[1]);
        }
    }
    // step 3: bucket rounds while many are pending, then block 0 alone in shared memory while
    // the other blocks clean up (contention bitplanes, overflow chunks)
    const unsigned nc = cta_load(&a.pcount[1]);
    const bool rounds = nc > TAIL_MAX;
    unsigned r = 0, nbu = 0;
    const uint2* list = nullptr;  // null: the tail takes crec[0, np) directly
    unsigned np = nc;
    if (PART == 1) return;  // (mode B) the buckets are built by the prep kernels between the parts
    if (rounds) {
        nbu = cta_load(&a.scan[a.p2g]);  // buckets (p2_number)
        if (gtid == 0) a.sc->t_prep = globaltimer();
        // Per round and CTA, in the (now free) dynamic shared memory: a queue of agents whose
        // watched blocker has walked (full check) and a queue of still-pending (agent, watch)
        // pairs flushed to the next list with one global atomic.
        uint2* qp = reinterpret_cast<uint2*>(s_dyn);
        unsigned* qc = reinterpret_cast<unsigned*>(s_dyn + QP_CAP * sizeof(uint2));
        unsigned* qpn = &s_q[0];
        unsigned* qcn = &s_q[1];
        for (;; ++r) {
            np = cta_load(&a.pcount[4 + r % 3]);
            list = a.alist[r & 1];
            if (gtid == 0 && r < 64) {
                a.sc->t_round[r] = globaltimer();
                a.sc->n_round[r] = np;
            }
            if (np <= TAIL_MAX || np <= (unsigned)MOVE_ASYNC_K * nthreads) break;  // every block reads the same np
            if (gtid == 0) a.pcount[4 + (r + 2) % 3] = 0;
            uint2* next = a.alist[(r + 1) & 1];
            unsigned int* ncount = &a.pcount[4 + (r + 1) % 3];
            // The CTA takes its share of the list (entry k goes to CTA k mod G, so a short list
            // in a late round still spreads over every CTA) in segments of MOVE_SEG entries: no
            // segment can overflow the two shared-memory queues, and the agents a segment leaves
            // pending go to the next list in one bulk flush before the following segment (one
            // global atomic per CTA and segment).  Lists of up to G * MOVE_SEG entries are one
            // segment; config 5's 6-7 million contended agents take five or six.
            unsigned long long hops = 0;
            long long p1_clk = 0, c_p2 = clock64();
            for (unsigned seg0 = 0; blockIdx.x + (size_t)gridDim.x * seg0 < np; seg0 += MOVE_SEG) {
            if (seg0) {
                __syncthreads();
                const unsigned nqf = min(*qpn, (unsigned)QP_CAP);
                __syncthreads();
                if (threadIdx.x == 0) {
                    s_q[2] = nqf ? atomicAdd(ncount, nqf) : 0u;
                    *qpn = 0;
                    *qcn = 0;
                }
                __syncthreads();
                for (unsigned i = threadIdx.x; i < nqf; i += blockDim.x) next[s_q[2] + i] = qp[i];
                __syncthreads();
            }
            // pass 1: watch tests, four list entries per thread in flight
            const long long c_p1 = clock64();
            for (unsigned base = seg0 + threadIdx.x;
                 base < seg0 + MOVE_SEG && blockIdx.x + (size_t)gridDim.x * base < np; base += 4 * blockDim.x) {
                uint2 e[4];
                unsigned v[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const size_t kk = blockIdx.x + (size_t)gridDim.x * (base + i * blockDim.x);
                    const unsigned k = kk < np ? (unsigned)kk : np;
                    e[i] = k < np ? __ldcg(&list[k]) : make_uint2(BK_NIL, BK_NOWATCH);
                }
#pragma unroll
                for (int i = 0; i < 4; ++i) v[i] = e[i].y != BK_NOWATCH ? __ldcg(&a.bdone[e[i].y]) : 1u;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    if (e[i].x == BK_NIL) continue;
                    if (!v[i]) {  // predecessor still pending: carry over as is
                        const unsigned s = atomicAdd(qpn, 1u);
                        if (s < QP_CAP) qp[s] = e[i];
                        else next[atomicAdd(ncount, 1u)] = e[i];
                    } else {
                        const unsigned s = atomicAdd(qcn, 1u);
                        if (s < QC_CAP) qc[s] = e[i].x;
                        else next[atomicAdd(ncount, 1u)] = make_uint2(e[i].x, BK_NOWATCH);  // checked next round
                    }
                }
            }
            __syncthreads();
            c_p2 = clock64();
            p1_clk += c_p2 - c_p1;
            // pass 2: full checks of this CTA's woken agents
            const unsigned nchk = min(*qcn, (unsigned)QC_CAP);
            if (threadIdx.x == 0 && r < 64 && nchk) atomicAdd(&a.sc->chk_cnt[r], (unsigned long long)nchk);
            for (unsigned i = threadIdx.x; i < nchk; i += blockDim.x) {
                const unsigned ci = qc[i];
                unsigned w;
                if (!bk_check(a, ci, s_bp, &hops, &w)) {
                    const unsigned s = atomicAdd(qpn, 1u);
                    if (s < QP_CAP) qp[s] = make_uint2(ci, w);
                    else next[atomicAdd(ncount, 1u)] = make_uint2(ci, w);
                }
            }
            }  // segments
            if (threadIdx.x == 0 && r < 64) atomicMax(&a.sc->p1_max[r], (unsigned long long)p1_clk);
            // local iterations: this CTA's still-pending agents whose watched blocker walked
            // during this round (in any CTA) are checked again at once, so a chain of agents can
            // advance several links per grid round.  Each pending agent lives in one CTA's
            // queue, so no agent is checked twice at the same time.
            for (int it = 0; it < MOVE_LOCAL_ITERS; ++it) {
                __syncthreads();
                const unsigned nq0 = min(*qpn, (unsigned)QP_CAP);
                if (nq0 == 0 || nq0 > MOVE_LOCAL_MAX) break;  // uniform: read after the barrier
                constexpr int PER = MOVE_LOCAL_MAX / MOVE_THREADS;
                uint2 e[PER];
                unsigned v[PER];
#pragma unroll
                for (int k = 0; k < PER; ++k) {
                    const unsigned idx = threadIdx.x + k * MOVE_THREADS;
                    e[k] = idx < nq0 ? qp[idx] : make_uint2(BK_NIL, BK_NOWATCH);
                }
#pragma unroll
                for (int k = 0; k < PER; ++k) v[k] = e[k].y != BK_NOWATCH ? __ldcg(&a.bdone[e[k].y]) : 1u;
                __syncthreads();
                if (threadIdx.x == 0) *qpn = *qcn = 0;
                __syncthreads();
#pragma unroll
                for (int k = 0; k < PER; ++k) {
                    if (e[k].x == BK_NIL) continue;
                    if (!v[k]) qp[atomicAdd(qpn, 1u)] = e[k];
                    else qc[atomicAdd(qcn, 1u)] = e[k].x;
                }
                __syncthreads();
                const unsigned nl = *qcn;
                if (nl == 0) break;  // uniform
                for (unsigned i = threadIdx.x; i < nl; i += blockDim.x) {
                    const unsigned ci = qc[i];
                    unsigned w;
                    if (!bk_check(a, ci, s_bp, &hops, &w)) qp[atomicAdd(qpn, 1u)] = make_uint2(ci, w);
                }
            }
            flush_hops(B, a.sc, hops);  // (its barriers also complete the queue)
            if (threadIdx.x == 0 && r < 64) atomicMax(&a.sc->chk_max[r], (unsigned long long)(clock64() - c_p2));
            const unsigned nq = min(*qpn, (unsigned)QP_CAP);
            __syncthreads();
            if (threadIdx.x == 0) {
                s_q[2] = nq ? atomicAdd(ncount, nq) : 0u;
                *qpn = 0;
                *qcn = 0;
            }
            __syncthreads();
            for (unsigned i = threadIdx.x; i < nq; i += blockDim.x) next[s_q[2] + i] = qp[i];
            grid.sync();
        }
        if (MOVE_ASYNC_K) {
            unsigned long long hops = 0;
            async_walk(a, list, np, gtid, nthreads, reinterpret_cast<uint2*>(s_dyn) + threadIdx.x, s_bp, &hops);
            flush_hops(B, a.sc, hops);
            np = 0;  // nothing left for the tail
            grid.sync();
        }
    }
    if (gridDim.x > 1 && blockIdx.x != 0) {
        zero_marks(a, nbu, blockIdx.x - 1, gridDim.x - 1);
        return;
    }
    if (threadIdx.x == 0) {
        a.sc->t_motion[2] = globaltimer();
        a.sc->grid_rounds = r;
    }
    if (np) {
        unsigned long long hops = 0;
        tail_smem(a, *reinterpret_cast<TailSmem*>(s_dyn), a.crec, list, np, s_bp, &hops);
        flush_hops(B, a.sc, hops);
    }
    if (gridDim.x == 1) zero_marks(a, nbu, 0, 1);
    if (gtid == 0) {
        a.sc->t_motion[3] = globaltimer();
        a.sc->pad[1] += r;  // grid rounds executed (observability; the tail adds its own)
        for (int k = 0; k < 10; ++k) a.pcount[k] = 0;  // list counts, seed cursors
        const unsigned long long ne = a.sc->n_exits;
        a.sc->alive -= ne;
        a.sc->tot_exits += ne;
        const unsigned long long d = a.sc->disp;
        a.sc->disp = d & 0xFFFFFFFFull;
        a.sc->step_dx = (long long)(int)(unsigned)(d >> 32);
        a.sc->tot_dx += a.sc->step_dx;
        a.sc->tot_disp += d & 0xFFFFFFFFull;
    }
}

// ------------------------------------------------------------------ seed kernels (mode A)
// Steps 1 and 2 of a phase whose records the plan kernel emitted, as two plain launches (marks,
// then classification) so every SM holds as many seed workers as fit instead of one
// cooperative CTA's four; then the contended-cell numbering (p2_count / p2_number, both on the
// motion's grid, whose slices they share).
#ifndef SEED_MARK_MINB
#define SEED_MARK_MINB 3
#endif
__global__ void __launch_bounds__(MOVE_THREADS, SEED_MARK_MINB) seed_mark_kernel(MoveArgs a) {
    FP_PDL_WAIT();
    __shared__ signed char s_bp[121][5][2];
    extern __shared__ __align__(16) unsigned char s_dyn[];
    for (int k = threadIdx.x; k < 121 * 10; k += blockDim.x) (&s_bp[0][0][0])[k] = (&c_bpath[0][0][0])[k];
    if (blockIdx.x == 0 && threadIdx.x == 0) a.sc->t_motion[0] = globaltimer();
    __syncthreads();
    const int nwmax = seed_ww(a.tile_w) * (a.tile_h + 10);
    seed_mark(a, reinterpret_cast<uint32_t*>(s_dyn) + (threadIdx.x / SEED_GROUP) * 2 * nwmax, s_bp);
}

#ifndef SEED_CLASSIFY_MINB
#define SEED_CLASSIFY_MINB 2
#endif
__global__ void __launch_bounds__(MOVE_THREADS, SEED_CLASSIFY_MINB) seed_classify_kernel(MoveArgs a) {
    FP_PDL_WAIT();
    __shared__ signed char s_bp[121][5][2];
    extern __shared__ __align__(16) unsigned char s_dyn[];
    __shared__ unsigned int s_app[2 + 2 * SEED_GROUPS];
    __shared__ unsigned long long s_hops[1 + SEED_GROUPS];
    for (int k = threadIdx.x; k < 121 * 10; k += blockDim.x) (&s_bp[0][0][0])[k] = (&c_bpath[0][0][0])[k];
    if (threadIdx.x < 2 + 2 * SEED_GROUPS) s_app[threadIdx.x] = 0;
    if (threadIdx.x < 1 + SEED_GROUPS) s_hops[threadIdx.x] = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) a.sc->t_marked = globaltimer();
    __syncthreads();
    const Group B{0, (int)blockDim.x, threadIdx.x == 0, &s_app[0], &s_hops[0]};
    const unsigned sg = threadIdx.x / SEED_GROUP;
    const Group Gs{1 + (int)sg, SEED_GROUP, threadIdx.x % SEED_GROUP == 0, &s_app[2 + 2 * sg], &s_hops[1 + sg]};
    const int nwmax = seed_ww(a.tile_w) * (a.tile_h + 10);
    unsigned long long hops = 0;
    seed_classify(a, Gs, reinterpret_cast<uint32_t*>(s_dyn) + sg * 2 * nwmax, s_bp, &hops);
    flush_hops(B, a.sc, hops);
}

__global__ void __launch_bounds__(MOVE_THREADS) p2_count_kernel(MoveArgs a) {
    FP_PDL_WAIT();
    __shared__ unsigned s_red[32];
    p2_count(a, s_red);
}

__global__ void __launch_bounds__(MOVE_THREADS) p2_number_kernel(MoveArgs a) {
    FP_PDL_WAIT();
    __shared__ unsigned s_red[32];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.sc->t_motion[1] = globaltimer();
        a.sc->contended = __ldcg(&a.pcount[1]);
    }
    if (cta_load(&a.pcount[1]) <= TAIL_MAX) return;
    p2_number(a, s_red);
}

// ------------------------------------------------------------------ bucket prep kernels
// Between the two parts of the motion: plain launches at full occupancy (the cooperative parts
// hold one 512-thread CTA per SM), each a latency-bound pass that wants many loads in flight.
// Each returns at once when the phase has too few contended agents for the rounds.
#define PREP_THREADS 256
__global__ void __launch_bounds__(PREP_THREADS) bk_count_kernel(MoveArgs a) {
    FP_PDL_WAIT();
    __shared__ signed char s_bp[121][5][2];
    for (int k = threadIdx.x; k < 121 * 10; k += blockDim.x) (&s_bp[0][0][0])[k] = (&c_bpath[0][0][0])[k];
    const unsigned nc = cta_load(&a.pcount[1]);  // (its barriers also publish s_bp)
    if (nc <= TAIL_MAX) return;
    const unsigned nthreads = gridDim.x * blockDim.x, gtid = blockIdx.x * blockDim.x + threadIdx.x;
    for (unsigned base = gtid; base < nc; base += BK_PREP_BATCH * nthreads) {
        unsigned ci[BK_PREP_BATCH];
        bool ok[BK_PREP_BATCH];
#pragma unroll
        for (int b = 0; b < BK_PREP_BATCH; ++b) {
            ci[b] = base + b * nthreads;
            ok[b] = ci[b] < nc;
        }
        bk_count<BK_PREP_BATCH>(a, ci, ok, s_bp);
    }
    if (gtid == 0) {
        // pending counts rotate over pcount[4..6]: round r reads its own, fills the next and
        // zeroes the one last read in round r-1
        a.pcount[4] = nc;
        a.pcount[5] = a.pcount[6] = 0;
    }
}

// bbase = exclusive prefix of the bucket sizes: per-CTA sums, then each CTA's slice (both
// launched with the same grid).
__global__ void __launch_bounds__(MOVE_THREADS) bk_scan_count_kernel(MoveArgs a, unsigned g1) {
    FP_PDL_WAIT();
    __shared__ unsigned s_red[32];
    if (cta_load(&a.pcount[1]) <= TAIL_MAX) return;
    bk_scan_count(a, cta_load(&a.scan[g1]), s_red);
}

__global__ void __launch_bounds__(MOVE_THREADS) bk_scan_base_kernel(MoveArgs a, unsigned g1) {
    FP_PDL_WAIT();
    __shared__ unsigned s_red[32];
    if (cta_load(&a.pcount[1]) <= TAIL_MAX) return;
    bk_scan_base(a, cta_load(&a.scan[g1]), s_red);
}

__global__ void __launch_bounds__(PREP_THREADS) bk_place_kernel(MoveArgs a) {
    FP_PDL_WAIT();
    const unsigned nc = cta_load(&a.pcount[1]);
    if (nc <= TAIL_MAX) return;
    const unsigned nthreads = gridDim.x * blockDim.x, gtid = blockIdx.x * blockDim.x + threadIdx.x;
    for (unsigned base = gtid; base < nc; base += BK_PREP_BATCH * nthreads) {
        unsigned ci[BK_PREP_BATCH];
        bool ok[BK_PREP_BATCH];
#pragma unroll
        for (int b = 0; b < BK_PREP_BATCH; ++b) {
            ci[b] = base + b * nthreads;
            ok[b] = ci[b] < nc;
        }
        bk_place<BK_PREP_BATCH>(a, ci, ok);
    }
}

__global__ void __launch_bounds__(PREP_THREADS) bk_sort_kernel(MoveArgs a, unsigned g1) {
    FP_PDL_WAIT();
    if (cta_load(&a.pcount[1]) <= TAIL_MAX) return;
    bk_sort(a, cta_load(&a.scan[g1]), blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
}

__global__ void __launch_bounds__(PREP_THREADS) bk_sort_long_kernel(MoveArgs a) {
    FP_PDL_WAIT();
    __shared__ unsigned s_rank[(PREP_THREADS / 32) * BK_SORT_MAX];
    if (cta_load(&a.pcount[1]) <= TAIL_MAX) return;
    bk_sort_long(a, s_rank);
}

// Per contended agent, once every bucket is sorted: its check record (see bk_check).
__global__ void __launch_bounds__(PREP_THREADS) bk_final_kernel(MoveArgs a) {
    FP_PDL_WAIT();
    __shared__ signed char s_bp[121][5][2];
    for (int k = threadIdx.x; k < 121 * 10; k += blockDim.x) (&s_bp[0][0][0])[k] = (&c_bpath[0][0][0])[k];
    const unsigned nc = cta_load(&a.pcount[1]);  // (its barriers also publish s_bp)
    if (nc <= TAIL_MAX) return;
    const unsigned nthreads = gridDim.x * blockDim.x;
    for (unsigned ci = blockIdx.x * blockDim.x + threadIdx.x; ci < nc; ci += nthreads) {
        const uint4 r = __ldcg(&a.crec[ci]);
        unsigned pos[6], cell[6];
        load_pairs(a, ci, pos, cell);
        const uint2 ko = __ldcg(reinterpret_cast<const uint2*>(a.eoff + (size_t)ci * 8));
        int cx[5], cy[5];
        const int m = path_of(a, r, s_bp, cx, cy);
        unsigned own[5];
        bool occ0[5];
#pragma unroll
        for (int i = 0; i < 5; ++i) {
            own[i] = BK_NIL;
            occ0[i] = false;
            if (i >= m) continue;
            const unsigned b = cell[i + 1];
            if (b != BK_NIL) {
                own[i] = __ldcg(&a.bown[b]);
                occ0[i] = __ldcg(&a.bocc0[b]);
            } else {
                occ0[i] = occ_test(a, cx[i], cy[i]);  // only this agent's footprint has the cell
            }
        }
        unsigned codes = 0, offs = 0, off4 = 0;
#pragma unroll
        for (int i = 0; i < 5; ++i) {
            if (i >= m) continue;
            const unsigned b = cell[i + 1], p = pos[i + 1];
            unsigned c;
            if (b == BK_NIL) c = occ0[i] ? CK_BLOCK : CK_FREE;
            else if (own[i] != BK_NIL ? own[i] > p : occ0[i]) c = CK_BLOCK;  // its occupant has not left
            else c = CK_DYN;
            codes |= c << (2 * i);
            if (b != BK_NIL) {
                const unsigned k = ((i + 1 < 4 ? ko.x >> (8 * (i + 1)) : ko.y >> (8 * (i - 3))) & 0xFFu);
                if (i < 4) offs |= k << (8 * i);
                else off4 = k;
            }
        }
        unsigned pj[6];
#pragma unroll
        for (int j = 0; j < 6; ++j) pj[j] = cell[j] != BK_NIL ? pos[j] : BK_NIL;
        a.ck[2 * (size_t)ci] = make_uint4(pj[0], pj[1], pj[2], pj[3]);
        a.ck[2 * (size_t)ci + 1] = make_uint4(pj[4], pj[5], offs, off4 | (codes << 8));
    }
}

// The phase's exit records (rank << 32 | id) into processing order on the device when they are
// few (the usual case: a handful per step); more than EXITS_SMEM are left to the host's radix sort.
#define EXITS_SMEM 4096
__global__ void __launch_bounds__(1024) exits_sort_kernel(unsigned long long* exits, DevScalars* sc) {
    FP_PDL_WAIT();
    __shared__ unsigned long long key[EXITS_SMEM];
    const unsigned n = (unsigned)sc->n_exits;
    if (n > EXITS_SMEM) {
        if (threadIdx.x == 0) sc->exits_sorted = 0;
        return;
    }
    for (unsigned i = threadIdx.x; i < n; i += blockDim.x) key[i] = exits[i];
    __syncthreads();
    for (unsigned i = threadIdx.x; i < n; i += blockDim.x) {  // keys are distinct (one per rank)
        const unsigned long long k = key[i];
        unsigned below = 0;
        for (unsigned j = 0; j < n; ++j) below += key[j] < k;
        exits[below] = k;
    }
    if (threadIdx.x == 0) sc->exits_sorted = 1;
}

__global__ void move_begin_kernel(DevScalars* sc) {
    FP_PDL_WAIT();
    for (int r = threadIdx.x; r < 64; r += blockDim.x) sc->chk_max[r] = sc->chk_cnt[r] = sc->p1_max[r] = 0;
    if (threadIdx.x) return;
    const unsigned long long t = globaltimer();
    sc->t_motion[0] = t;  // (the marking pass, when it runs, restamps its start)
    sc->t_plan_end = t;
    sc->plan_ns += t - sc->t_step0;
    sc->n_exits = 0;
    sc->exits_sorted = 0;
    sc->disp = 0;
    sc->tot_updates += sc->alive;
}

static int ensure_buckets(fp_ctx* ctx);

int fp_ensure_res(fp_ctx* ctx) {
    if (ctx->device < 64 && !g_bpath_ready[ctx->device]) {
        signed char bp[121][5][2];
        host_bpath(bp);
        FP_CUDA(ctx, cudaMemcpyToSymbol(c_bpath, bp, sizeof(bp)));
        g_bpath_ready[ctx->device] = true;
    }
    if (!ctx->d_p1) {
        const size_t nwords = (size_t)ctx->P * ctx->H;
        FP_CUDA(ctx, cudaMalloc(&ctx->d_p1, nwords * 4));
        FP_CUDA(ctx, cudaMalloc(&ctx->d_p2, nwords * 4));
        FP_CUDA(ctx, cudaMalloc(&ctx->d_pw, nwords * sizeof(uint2)));
        FP_CUDA(ctx, cudaMemsetAsync(ctx->d_p1, 0, nwords * 4, ctx->stream));
        FP_CUDA(ctx, cudaMemsetAsync(ctx->d_p2, 0, nwords * 4, ctx->stream));
        ctx->marks_dirty = false;
    }
    return ensure_buckets(ctx);  // before any graph capture: allocation is not capturable
}

// per device: the raised shared-memory limit and the occupancy are attributes of the device's
// function instance, so a process driving several devices configures each one
static int g_move_blocks[64] = {0};
static int g_prep_blocks[64] = {0};
static int g_seed_per_sm[64] = {0};
static int g_seed_smem[64] = {0};

// Buckets: per contended cell (<= 3 per contended agent: every contended cell is covered by >= 2
// of the <= 6-cell footprints) a counter, a base and its standing agent; per position (<= 6 per
// contended agent) a rank and a done flag; the per-agent (position, bucket) pairs; the scan
// counts.  Counters zero between phases.
static int ensure_buckets(fp_ctx* ctx) {
    const size_t nb = ((size_t)ctx->cap * 3 + 64 + 1) & ~(size_t)1;  // even: brank stays 8-byte aligned
    const size_t npos = (size_t)ctx->cap * 6 + 64;
    if (ctx->d_bkt && ctx->bk_agent_cap >= ctx->cap) return FP_OK;
    const size_t words = 3 * nb + 2 * npos + 2048;
    if (words >= 0xFFFFFFFFull) return fp_fail(ctx, FP_ERUNTIME, "motion: roster too large for 32-bit positions");
    cudaStreamSynchronize(ctx->stream);
    for (void* p : {(void*)ctx->d_bkt, (void*)ctx->d_bdone, (void*)ctx->d_entry})
        if (p) cudaFree(p);
    FP_CUDA(ctx, cudaMalloc(&ctx->d_bkt, words * 4));
    FP_CUDA(ctx, cudaMemsetAsync(ctx->d_bkt, 0, words * 4, ctx->stream));
    FP_CUDA(ctx, cudaMalloc(&ctx->d_bdone, npos + 16 + nb));  // done bytes (+ 16: whole-chunk reads), bocc0
    FP_CUDA(ctx, cudaMalloc(&ctx->d_entry, (size_t)ctx->cap * (6 * sizeof(uint2) + 8 + 2 * sizeof(uint4)) + 16));  // + eoff, ck
    ctx->bk_nb_cap = (unsigned)nb;
    ctx->bk_npos_cap = (unsigned)npos;
    ctx->bk_agent_cap = ctx->cap;
    ctx->graph_valid = false;
    return FP_OK;
}

// Enqueues one motion phase (after fp_order_launch) on ctx->stream.  Graph-safe.
// Mode A (ctx->rec_fresh): the plan kernel emitted records + marks for the current state.
// Mode B: records are built here from the plan-tile buckets when current, else the order list.
int fp_motion_launch(fp_ctx* ctx, bool spatial) {
    cudaStream_t s = ctx->stream;
    fp_launch(move_begin_kernel, 1, 64, 0, s, ctx->d_sc);
    FP_LAUNCHED(ctx);
    if (ctx->n == 0) return FP_OK;
    if (int rc = ensure_buckets(ctx)) return rc;
    const bool premade = ctx->rec_fresh;
    if (!premade && ctx->marks_dirty) {  // marks of records that were never consumed
        const size_t nwords = (size_t)ctx->P * ctx->H;
        FP_CUDA(ctx, cudaMemsetAsync(ctx->d_p1, 0, nwords * 4, s));
        FP_CUDA(ctx, cudaMemsetAsync(ctx->d_p2, 0, nwords * 4, s));
    }
    int& move_blocks = g_move_blocks[ctx->device & 63];
    if (!move_blocks) {
        int per_sm = 1 << 30;
        for (const void* k : {(const void*)move_rounds_kernel<1>, (const void*)move_rounds_kernel<2>}) {
            FP_CUDA(ctx, cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)MOVE_DYN_SMEM));
            int c = 0;
            FP_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, k, MOVE_THREADS, MOVE_DYN_SMEM));
            per_sm = std::min(per_sm, c);
        }
        move_blocks = std::max(1, std::min(per_sm, FP_MOVE_BLOCKS_PER_SM)) * ctx->sm_count;
        int pc = 0;  // the prep kernels: as many CTAs as fit on every SM (grid-stride loops)
        for (const void* k : {(const void*)bk_count_kernel, (const void*)bk_place_kernel, (const void*)bk_sort_kernel,
                              (const void*)bk_sort_long_kernel, (const void*)bk_final_kernel}) {
            int c = 0;
            FP_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, k, PREP_THREADS, 0));
            pc = pc ? std::min(pc, c) : c;
        }
        g_prep_blocks[ctx->device & 63] = std::max(1, pc) * ctx->sm_count;
    }
    const unsigned prep_blocks = (unsigned)g_prep_blocks[ctx->device & 63];
    int& seed_per_sm = g_seed_per_sm[ctx->device & 63];
    int& seed_smem_at = g_seed_smem[ctx->device & 63];
    const int smem = SEED_GROUPS * 2 * seed_ww(ctx->tile_w) * (ctx->tile_h + 10) * 4;
    if (premade && (seed_per_sm == 0 || seed_smem_at != smem)) {  // seed CTAs per SM for this window size
        seed_smem_at = smem;
        int c = 1 << 30;
        for (const void* k : {(const void*)seed_mark_kernel, (const void*)seed_classify_kernel}) {
            FP_CUDA(ctx, cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)MOVE_DYN_SMEM));
            int o = 0;
            FP_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k, MOVE_THREADS, smem));
            c = std::min(c, o);
        }
        seed_per_sm = std::max(1, c);
    }
    const unsigned seed_blocks = (unsigned)std::max(1, seed_per_sm) * (unsigned)ctx->sm_count;
    MoveArgs a;
    a.g = fp_geo(ctx);
    a.occ = ctx->d_occ;
    a.x = ctx->d_x;
    a.y = ctx->d_y;
    a.dx = ctx->d_dx;
    a.dy = ctx->d_dy;
    a.v = ctx->d_v;
    a.alive = ctx->d_alive;
    a.rank = ctx->d_rank;
    a.seed_list = ctx->d_order;  // mode B only (any order: the motion is order-independent)
    (void)spatial;
    a.rec0 = ctx->d_rec0;
    a.premade = premade ? 1 : 0;
    a.premarked = (premade && ctx->plan_marked) ? 1 : 0;
    a.rec[0] = ctx->d_rec_a;
    a.rec[1] = ctx->d_rec_b;
    a.pcount = (unsigned int*)ctx->d_counters;  // [0], [1] as u32 (kept zero between phases)
    a.sc = ctx->d_sc;
    a.exits = ctx->d_exits;
    a.p1 = ctx->d_p1;
    a.p2 = ctx->d_p2;
    a.tile_list = ctx->d_tile_list;
    a.tile_off = ctx->d_tile_off;
    a.tile_cnt = ctx->d_tile_cnt;
    a.items = ctx->d_seed_items;
    a.tile_w = ctx->tile_w;
    a.tile_h = ctx->tile_h;
    a.tiles_x = ctx->tiles_x;
    a.crec = ctx->d_rec_b;
    a.nb_cap = ctx->bk_nb_cap;
    a.npos_cap = ctx->bk_npos_cap;
    a.pw = ctx->d_pw;
    a.bcnt = ctx->d_bkt;
    a.bbase = ctx->d_bkt + ctx->bk_nb_cap;
    a.brank = reinterpret_cast<uint2*>(ctx->d_bkt + 3 * (size_t)ctx->bk_nb_cap);
    a.scan = reinterpret_cast<unsigned*>(a.brank + ctx->bk_npos_cap);
    a.p2g = (unsigned)std::min(BK_SCAN2 - 1, 4 * ctx->sm_count);
    a.bdone = ctx->d_bdone;
    a.bocc0 = ctx->d_bdone + ctx->bk_npos_cap + 16;
    a.bown = ctx->d_bkt + 2 * (size_t)ctx->bk_nb_cap;
    a.entry = ctx->d_entry;
    a.eoff = reinterpret_cast<uint8_t*>(ctx->d_entry + (size_t)ctx->cap * 6);
    a.ck = reinterpret_cast<uint4*>(ctx->d_entry + (((size_t)ctx->cap * 7 + 1) & ~(size_t)1));  // 16-byte aligned
    uint2* lists = reinterpret_cast<uint2*>(ctx->d_rec_a);  // 16 B per agent: two uint2 lists
    a.alist[0] = lists;
    a.alist[1] = lists + ctx->cap;
    a.long_list = reinterpret_cast<unsigned*>(lists + ctx->cap);  // alist[1] is free until round 0
    if (premade && (size_t)SEED_GROUPS * 2 * seed_ww(ctx->tile_w) * (ctx->tile_h + 10) * 4 > MOVE_DYN_SMEM)
        return fp_fail(ctx, FP_ERUNTIME, "motion: seed window exceeds shared memory");
    const unsigned blocks = (unsigned)std::min<size_t>((size_t)move_blocks,
                                                        std::max<size_t>(1, fp_blocks(ctx->n, MOVE_THREADS)));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(MOVE_THREADS);
    cfg.dynamicSmemBytes = MOVE_DYN_SMEM;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const size_t seed_smem = (size_t)SEED_GROUPS * 2 * seed_ww(ctx->tile_w) * (ctx->tile_h + 10) * 4;
    // a roster the shared-memory tail always takes whole (<= TAIL_MAX agents) needs no buckets:
    // one cooperative launch for steps 1 and 2, no prep launches (launch-bound small configs)
    const bool tiny = ctx->n <= TAIL_MAX;
    if (premade && !tiny) {  // steps 1 and 2 over the plan's records: two plain launches
        const unsigned sb = std::min(seed_blocks, std::max(1u, (unsigned)fp_blocks(ctx->n, SEED_ITEM)));
        if (!ctx->plan_marked) {  // (else the plan kernels marked the footprints as they emitted them)
            fp_launch(seed_mark_kernel, sb, MOVE_THREADS, seed_smem, s, a);
            FP_LAUNCHED(ctx);
        }
        fp_launch(seed_classify_kernel, sb, MOVE_THREADS, seed_smem, s, a);
        FP_LAUNCHED(ctx);
    } else {
        FP_CUDA(ctx, cudaLaunchKernelEx(&cfg, move_rounds_kernel<1>, a));
        ctx->ctr.kernel_launches++;
    }
    if (!tiny) {
        fp_launch(p2_count_kernel, a.p2g, MOVE_THREADS, 0, s, a);
        FP_LAUNCHED(ctx);
        fp_launch(p2_number_kernel, a.p2g, MOVE_THREADS, 0, s, a);
        FP_LAUNCHED(ctx);
        const unsigned pg = prep_blocks;
        fp_launch(bk_count_kernel, pg, PREP_THREADS, 0, s, a);
        FP_LAUNCHED(ctx);
        fp_launch(bk_scan_count_kernel, a.p2g, MOVE_THREADS, 0, s, a, a.p2g);
        FP_LAUNCHED(ctx);
        fp_launch(bk_scan_base_kernel, a.p2g, MOVE_THREADS, 0, s, a, a.p2g);
        FP_LAUNCHED(ctx);
        fp_launch(bk_place_kernel, pg, PREP_THREADS, 0, s, a);
        FP_LAUNCHED(ctx);
        fp_launch(bk_sort_kernel, pg, PREP_THREADS, 0, s, a, a.p2g);
        FP_LAUNCHED(ctx);
        fp_launch(bk_sort_long_kernel, pg, PREP_THREADS, 0, s, a);
        FP_LAUNCHED(ctx);
        fp_launch(bk_final_kernel, pg, PREP_THREADS, 0, s, a);
        FP_LAUNCHED(ctx);
    }
    FP_CUDA(ctx, cudaLaunchKernelEx(&cfg, move_rounds_kernel<2>, a));
    ctx->ctr.kernel_launches++;
    fp_launch(exits_sort_kernel, 1, 1024, 0, s, ctx->d_exits, ctx->d_sc);
    FP_LAUNCHED(ctx);
    ctx->rec_fresh = false;
    ctx->marks_dirty = false;
    ctx->plan_marked = false;
    return fp_ghost_occ(ctx);
}

int fp_exits_sort_launch(fp_ctx* ctx) {
    fp_launch(exits_sort_kernel, 1, 1024, 0, ctx->stream, ctx->d_exits, ctx->d_sc);
    FP_LAUNCHED(ctx);
    return FP_OK;
}

// Exit records are (rank << 32 | id) with distinct ranks in [0, n_alive): a rank flag array,
// its exclusive scan, and a scatter put them in processing order.
__global__ void exits_flag_kernel(const unsigned long long* exits, uint32_t ne, uint32_t* flag) {
    FP_PDL_WAIT();
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < ne) flag[(uint32_t)(exits[i] >> 32)] = 1u;
}

__global__ void exits_place_kernel(const unsigned long long* exits, uint32_t ne, const uint32_t* pos,
                                   unsigned long long* out) {
    FP_PDL_WAIT();
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < ne) out[pos[(uint32_t)(exits[i] >> 32)]] = exits[i];
}

// Sorts the exit records of the last phase by rank (processing order) for fp_get_exited, when
// there were too many for the motion graph's one-block sort (host path, after the step's sync;
// the order scratch d_cnt / d_off is free until the next step).
int fp_exits_finish(fp_ctx* ctx) {
    const uint32_t ne = ctx->n_exits;
    if (ne <= 1 || ctx->h_sc->exits_sorted) return FP_OK;  // sorted in the motion graph
    const uint32_t na = std::max<uint32_t>(ctx->n_order, 1);
    if (!ctx->d_scan_sums2) FP_CUDA(ctx, cudaMalloc(&ctx->d_scan_sums2, FP_SCAN_SUMS * 4));
    FP_CUDA(ctx, cudaMemsetAsync(ctx->d_cnt, 0, (size_t)na * 4, ctx->stream));
    fp_launch(exits_flag_kernel, fp_blocks(ne, 256), 256, 0, ctx->stream, ctx->d_exits, ne, ctx->d_cnt);
    FP_LAUNCHED(ctx);
    if (int rc = fp_scan_u32(ctx, ctx->d_cnt, ctx->d_off, na, ctx->d_scan_sums2, ctx->stream)) return rc;
    fp_launch(exits_place_kernel, fp_blocks(ne, 256), 256, 0, ctx->stream, ctx->d_exits, ne, ctx->d_off, ctx->d_exits_sorted);
    FP_LAUNCHED(ctx);
    FP_CUDA(ctx, cudaMemcpyAsync(ctx->d_exits, ctx->d_exits_sorted, ne * sizeof(unsigned long long),
                                 cudaMemcpyDeviceToDevice, ctx->stream));
    FP_CUDA(ctx, cudaMemsetAsync(ctx->d_cnt, 0, (size_t)na * 4, ctx->stream));  // the order's zero invariant
    return FP_OK;
}
