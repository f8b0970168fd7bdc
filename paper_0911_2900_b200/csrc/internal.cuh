// internal.cuh -- device context, data layout and shared device helpers.
//
// HBM layout (all row-major y*W+x like world.hpp:88-91):
//   wall / exit / occupancy : 1-bit planes, P = ceil(W/32) u32 words per row
//   field                   : fp64 per cell (StaticField::s; fp64 is required for bit-exact
//                             weights)
//   reservation             : u64 per cell, round-stamped keys of the motion rounds
//   agents (SoA)            : x, y (i32), v_max (u8), alive (u8), desired x/y (i32), rank (u32)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/fastped_b200.h"

#define FP_NONE 0xFFFFFFFFu

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
        return (size_t)y * (size_t)P + (size_t)(x >> 5);
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
#define FP_MOVE_ORDER_STREAM (1ULL << 63)
#define FP_SPAWN_STREAM ((1ULL << 63) + 1)

struct fp_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::string err;

    // geometry
    int W = 0, H = 0, boundary = 0, P = 0;
    double cell_size = 0.4;
    uint32_t* d_wall = nullptr;
    uint32_t* d_exit = nullptr;
    uint32_t* d_occ = nullptr;
    double* d_field = nullptr;
    unsigned long long* d_res = nullptr;  // motion reservations (allocated on first move)
    uint64_t round_seq = 0;

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

    // order scratch (sized by cap)
    uint32_t *d_alive_ids = nullptr, *d_order = nullptr, *d_j = nullptr, *d_cnt = nullptr,
             *d_off = nullptr, *d_cursor = nullptr, *d_bucket = nullptr, *d_succ = nullptr,
             *d_nxt = nullptr, *d_V = nullptr;
    uint32_t n_order = 0;  // alive count of the last computed order

    // motion scratch
    uint32_t *d_pend_a = nullptr, *d_pend_b = nullptr;
    unsigned long long* d_exits = nullptr;  // (rank << 32 | id) records of the last move
    unsigned long long* d_exits_sorted = nullptr;
    int64_t last_displacement = 0;
    uint32_t n_exits = 0;
    // small device counters: [0] pending next, [1] exits, [2] alive-count delta, [3] spare
    // [4..5] displacement (u64), [6] n_alive (select), [7] plan fallbacks
    unsigned long long* d_counters = nullptr;

    // cub temp
    void* d_temp = nullptr;
    size_t temp_bytes = 0;

    // pinned host mirror of counters
    unsigned long long* h_counters = nullptr;

    fp_counters ctr{};
};

// -------------------------------------------------------------------------- error helpers
void fp_set_global_error(const std::string& s);
int fp_cuda_fail(fp_ctx* ctx, cudaError_t e, const char* what);

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

inline unsigned fp_blocks(size_t n, unsigned tpb) {
    size_t b = (n + tpb - 1) / tpb;
    return (unsigned)(b == 0 ? 1 : b);
}

// Stage entry points (implemented in plan.cu / order.cu / move.cu / field.cu).
int fp_plan_launch(fp_ctx* ctx, double k_s, uint64_t seed);
int fp_order_launch(fp_ctx* ctx, uint64_t seed, int64_t step);
int fp_motion_launch(fp_ctx* ctx, bool collect_exits);
int fp_field_compute(fp_ctx* ctx, const uint8_t* d_cells);
int fp_choice_launch(fp_ctx* ctx, uint32_t agent, double k_s, int32_t* d_cx, int32_t* d_cy,
                     double* d_w, float* d_p, uint32_t* d_n);
int fp_order_positions(fp_ctx* ctx, uint32_t n, uint64_t seed, int64_t step, uint32_t* d_out);
int fp_ensure_temp(fp_ctx* ctx, size_t bytes);
