// motion_rec.cuh -- the motion phase's per-agent record and contention marks, shared by the plan
// kernel (which emits them right after choosing the desired cell, in plan-tile order) and the
// motion kernel (which consumes them, or builds them itself when the plan did not).
//
// A walk (engine.hpp:116-119) of agent id from its cell toward its desired cell visits at most
// v_max Bresenham cells, stops before a Wall and ends at an Exit; everything else that can stop
// it is occupancy.  Record (16 bytes):
//     x = id,  y = rank (filled by the motion phase),
//     z = px | exit_free << 27 | m << 28 | exit_at_end << 31
//                                               (m = static walk length, 0..5)
//     w = py | o << 24 | generic << 31          (o = (dy+5)*11 + dx+5 of the target offset;
//                                                generic: target farther than 5 cells, the path
//                                                is re-derived from the agent arrays)
// The footprint -- the cells whose occupancy the walk reads or writes and that other walks may
// change -- is the start cell plus the first mf path cells.  mf = m, except that an Exit cell
// ending the walk that is unoccupied at the snapshot is left out (exit_free): nobody can stop
// on an Exit (entering one removes the agent, engine.hpp:123-128), so its occupancy stays
// empty for the whole phase and orders nothing.  That keeps the dozens of agents queueing for
// one exit from forming a single dependency chain.
// Contention marks: P1 = cell in some mover's footprint, P2 = in two or more.
#pragma once

#include "internal.cuh"

#define REC_GENERIC 0x80000000u
#define REC_EXIT_FREE 0x08000000u
#define REC_X_MASK 0x07FFFFFFu  // px < 2^27 (checked by fp_create)

__device__ __forceinline__ int rec_x(const uint4& r) { return (int)(r.z & REC_X_MASK); }
__device__ __forceinline__ int rec_y(const uint4& r) { return (int)(r.w & 0x00FFFFFFu); }
__device__ __forceinline__ int rec_m(const uint4& r) { return (int)((r.z >> 28) & 7u); }
__device__ __forceinline__ int rec_mf(const uint4& r) { return rec_m(r) - ((r.z & REC_EXIT_FREE) ? 1 : 0); }

// Bresenham cells of the segment (0,0) -> each offset of the 11x11 frame, in walk order.
static inline void host_bpath(signed char out[121][5][2]) {
    for (int ty = -5; ty <= 5; ++ty)
        for (int tx = -5; tx <= 5; ++tx) {
            signed char(*p)[2] = out[(ty + 5) * 11 + tx + 5];
            for (int j = 0; j < 5; ++j) p[j][0] = p[j][1] = 0;
            const int adx = abs(tx), sx = 0 < tx ? 1 : -1;
            const int ady = -abs(ty), sy = 0 < ty ? 1 : -1;
            int err = adx + ady, x = 0, y = 0, j = 0;
            while (!(x == tx && y == ty)) {
                const int e2 = 2 * err;
                if (e2 >= ady) { err += ady; x += sx; }
                if (e2 <= adx) { err += adx; y += sy; }
                p[j][0] = (signed char)x;
                p[j][1] = (signed char)y;
                ++j;
            }
        }
}

// Record of a walk from (sx, sy) to (tx, ty) (both wrapped), cap v; occ = the snapshot
// occupancy (for exit_free).
__device__ __forceinline__ uint4 record_of(const Geo& g, const uint32_t* occ, uint32_t id, int sx, int sy, int tx,
                                           int ty, int v, const signed char (*bp)[5][2]) {
    const int ddx = g.segment_dx(sx, tx), ddy = ty - sy;
    int m = 0, ex_x = 0, ex_y = 0;
    bool ex = false;
    uint32_t w;
    if (abs(ddx) <= 5 && abs(ddy) <= 5) {
        const int o = (ddy + 5) * 11 + ddx + 5;
        const int len = min(max(abs(ddx), abs(ddy)), v);
        for (int j = 0; j < len; ++j) {
            const int x = g.wrap(sx + bp[o][j][0]), y = sy + bp[o][j][1];
            if (g.is_wall(x, y)) break;
            ++m;
            if (g.is_exit(x, y)) {
                ex = true;
                ex_x = x;
                ex_y = y;
                break;
            }
        }
        w = (uint32_t)sy | ((uint32_t)o << 24);
    } else {
        Bres b;
        b.init(g, sx, sy, tx, ty);
        while (!b.done() && m < v) {
            b.next();
            const int x = g.wrap(b.x), y = b.y;
            if (g.is_wall(x, y)) break;
            ++m;
            if (g.is_exit(x, y)) {
                ex = true;
                ex_x = x;
                ex_y = y;
                break;
            }
        }
        w = (uint32_t)sy | REC_GENERIC;
    }
    const bool exit_free = ex && !((__ldcg(&occ[g.word(ex_x, ex_y)]) >> (ex_x & 31)) & 1u);
    return make_uint4(id, 0u,
                      (uint32_t)sx | (exit_free ? REC_EXIT_FREE : 0u) | ((uint32_t)m << 28) |
                          (ex ? 0x80000000u : 0u),
                      w);
}

// Path cells of a record (at most 5); generic records re-walk toward (gtx, gty).
__device__ __forceinline__ int record_cells(const Geo& g, const uint4& r, const signed char (*bp)[5][2], int gtx,
                                            int gty, int* cx, int* cy) {
    const int sx = rec_x(r), sy = rec_y(r);
    const int m = rec_m(r);
    // fixed-trip predicated loops keep cx/cy in registers (callers index them the same way)
    if (!(r.w & REC_GENERIC)) {
        const int o = (int)((r.w >> 24) & 0x7Fu);
#pragma unroll
        for (int j = 0; j < 5; ++j) {
            if (j < m) {
                cx[j] = g.wrap(sx + bp[o][j][0]);
                cy[j] = sy + bp[o][j][1];
            }
        }
    } else {
        Bres b;
        b.init(g, sx, sy, gtx, gty);
#pragma unroll
        for (int j = 0; j < 5; ++j) {
            if (j < m) {
                b.next();
                cx[j] = g.wrap(b.x);
                cy[j] = b.y;
            }
        }
    }
    return m;
}

// Marks the footprint (start + path) of a record with m > 0: all P1 fetch-ORs in flight at once,
// then the P2 marks (fire-and-forget) for cells some other footprint already held.
__device__ __forceinline__ void mark_record(uint32_t* p1, uint32_t* p2, const Geo& g, const uint4& r,
                                            const signed char (*bp)[5][2], int gtx, int gty) {
    int cx[6], cy[6];
    if (record_cells(g, r, bp, gtx, gty, cx + 1, cy + 1) == 0) return;
    const int m = rec_mf(r);  // footprint path cells
    cx[0] = rec_x(r);
    cy[0] = rec_y(r);
    uint32_t old[6];
#pragma unroll
    for (int i = 0; i < 6; ++i)
        if (i <= m) old[i] = atomicOr(&p1[g.word(cx[i], cy[i])], 1u << (cx[i] & 31));
#pragma unroll
    for (int i = 0; i < 6; ++i) {
        const uint32_t bit = 1u << (cx[i] & 31);
        if (i <= m && (old[i] & bit)) atomicOr(&p2[g.word(cx[i], cy[i])], bit);
    }
}
