// plan.cu -- the planning phase: choose_desired_cell for every alive agent.
//
// Reference: plan_phase (engine.hpp:71-84) -> choose_desired_cell (planning.hpp:88-108)
//            -> enumerate_candidates (planning.hpp:23-57), line_of_sight (world.hpp:181-191),
//               potential_drop (planning.hpp:76-80), std::exp, sample_index (:63-73).
//
// Exact path: one thread per agent, candidates visited in the reference's row-major order
// (wrapped-x sorted at the periodic seam), weights through the bit-exact restated glibc exp
// (fp_exp.h), serial fp64 total and cumulative scan -- so the sampled cell is bitwise the
// reference's.  There is no CPU fallback.
#include <math.h>

#include "fp_exp.h"
#include "internal.cuh"

struct PlanArgs {
    Geo g;
    const uint32_t* occ;
    const double* field;
    const int32_t* x;
    const int32_t* y;
    const uint8_t* v;
    const uint8_t* alive;
    int32_t* dx;
    int32_t* dy;
    uint32_t n;
    int potential;
    double drive_gradient;
    double k_s;
    uint64_t seed;
    uint64_t step;
};

__device__ __forceinline__ bool occ_bit(const uint32_t* occ, const Geo& g, int x, int y) {
    return (occ[g.word(x, y)] >> (x & 31)) & 1u;
}

// line_of_sight (world.hpp:181-191): no Wall on the Bresenham segment (exclusive a).
__device__ __forceinline__ bool los(const Geo& g, int ax, int ay, int bx, int by) {
    Bres b;
    b.init(g, ax, ay, bx, by);
    while (!b.done()) {
        b.next();
        if (g.is_wall(g.wrap(b.x), b.y)) return false;
    }
    return true;
}

// Visits enumerate_candidates(st, agent) in list order; f(x, y) returns false to stop.
template <class F>
__device__ __forceinline__ void for_each_candidate(const PlanArgs& a, int px, int py, int v, F&& f) {
    const Geo& g = a.g;
    const int y_lo = max(0, py - v);
    const int y_hi = min(g.H - 1, py + v);
    // x segments of one row in ascending wrapped-x order (planning.hpp:37-53, 55)
    int s0lo, s0hi, s1lo = 0, s1hi = -1;
    if (g.boundary == FP_BOUNDARY_PERIODIC_X) {
        const int lo = px - v, hi = px + v;
        if (2 * v + 1 >= g.W) {
            s0lo = 0; s0hi = g.W - 1;  // the ball covers every column once after dedupe
        } else if (lo < 0) {
            s0lo = 0; s0hi = hi; s1lo = lo + g.W; s1hi = g.W - 1;
        } else if (hi >= g.W) {
            s0lo = 0; s0hi = hi - g.W; s1lo = lo; s1hi = g.W - 1;
        } else {
            s0lo = lo; s0hi = hi;
        }
    } else {
        s0lo = max(0, px - v);
        s0hi = min(g.W - 1, px + v);
    }
    for (int y = y_lo; y <= y_hi; ++y) {
        for (int seg = 0; seg < 2; ++seg) {
            const int xlo = seg ? s1lo : s0lo, xhi = seg ? s1hi : s0hi;
            for (int x = xlo; x <= xhi; ++x) {
                if (g.is_wall(x, y)) continue;
                if (occ_bit(a.occ, g, x, y) && !(x == px && y == py)) continue;
                if (!los(g, px, py, x, y)) continue;
                if (!f(x, y)) return;
            }
        }
    }
}

struct ExactWeight {
    bool exitd, ones;
    double sp, k_s, g;
    int px;
    const double* field;
    const Geo* geo;
    __device__ __forceinline__ double operator()(int x, int y) const {
        if (ones) return 1.0;
        if (exitd) {
            const double sc = field[(size_t)y * geo->W + x];
            if (isinf(sc)) return 0.0;  // planning.hpp:98-100
            return fpx_exp(FPX_MUL(k_s, FPX_SUB(sp, sc)));
        }
        return fpx_exp(FPX_MUL(k_s, FPX_MUL(g, (double)geo->segment_dx(px, x))));
    }
};

__device__ __forceinline__ ExactWeight make_weight(const PlanArgs& a, int px, int py) {
    ExactWeight w;
    w.exitd = a.potential == FP_POTENTIAL_EXIT_DISTANCE;
    w.sp = w.exitd ? a.field[(size_t)py * a.g.W + px] : 0.0;
    w.ones = w.exitd && isinf(w.sp);  // planning.hpp:93-95
    w.k_s = a.k_s;
    w.g = a.drive_gradient;
    w.px = px;
    w.field = a.field;
    w.geo = &a.g;
    return w;
}

// choose_desired_cell, exact (planning.hpp:88-108 + sample_index :63-73)
__device__ void choose_exact(const PlanArgs& a, uint32_t i, int* ox, int* oy) {
    const int px = a.g.wrap(a.x[i]);
    const int py = a.y[i];
    const int v = a.v[i];
    const ExactWeight wf = make_weight(a, px, py);
    double total = 0.0;
    int lastx = px, lasty = py;
    for_each_candidate(a, px, py, v, [&](int x, int y) {
        total = FPX_ADD(total, wf(x, y));
        lastx = x;
        lasty = y;
        return true;
    });
    const double u = fp_unit_interval(fp_rng_u64(a.seed, i, a.step, 0));
    const double threshold = FPX_MUL(u, total);
    double cum = 0.0;
    int cx = lastx, cy = lasty;  // u*total rounded up to total: the tail (planning.hpp:72)
    for_each_candidate(a, px, py, v, [&](int x, int y) {
        cum = FPX_ADD(cum, wf(x, y));
        if (cum > threshold) {
            cx = x;
            cy = y;
            return false;
        }
        return true;
    });
    *ox = cx;
    *oy = cy;
}

__global__ void plan_exact_kernel(PlanArgs a) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.n || !a.alive[i]) return;
    int cx, cy;
    choose_exact(a, i, &cx, &cy);
    a.dx[i] = cx;
    a.dy[i] = cy;
}

// Test mode (fp_get_choice): the candidate list, exact weights and choice probabilities.
__global__ void choice_kernel(PlanArgs a, uint32_t i, int32_t* cx, int32_t* cy, double* w,
                              float* p, uint32_t* n_out) {
    const int px = a.g.wrap(a.x[i]);
    const int py = a.y[i];
    const ExactWeight wf = make_weight(a, px, py);
    uint32_t n = 0;
    double total = 0.0;
    for_each_candidate(a, px, py, a.v[i], [&](int x, int y) {
        const double wi = wf(x, y);
        cx[n] = x;
        cy[n] = y;
        w[n] = wi;
        total = FPX_ADD(total, wi);
        ++n;
        return true;
    });
    for (uint32_t k = 0; k < n; ++k) p[k] = (float)(w[k] / total);
    *n_out = n;
}

static PlanArgs make_args(fp_ctx* ctx, double k_s, uint64_t seed) {
    PlanArgs a;
    a.g = Geo{ctx->W, ctx->H, ctx->boundary, ctx->P, ctx->d_wall, ctx->d_exit};
    a.occ = ctx->d_occ;
    a.field = ctx->d_field;
    a.x = ctx->d_x;
    a.y = ctx->d_y;
    a.v = ctx->d_v;
    a.alive = ctx->d_alive;
    a.dx = ctx->d_dx;
    a.dy = ctx->d_dy;
    a.n = ctx->n;
    a.potential = ctx->potential;
    a.drive_gradient = ctx->drive_gradient;
    a.k_s = k_s;
    a.seed = seed;
    a.step = (uint64_t)ctx->step;
    return a;
}

int fp_plan_launch(fp_ctx* ctx, double k_s, uint64_t seed) {
    if (ctx->n == 0 || ctx->alive == 0) return FP_OK;
    PlanArgs a = make_args(ctx, k_s, seed);
    plan_exact_kernel<<<fp_blocks(ctx->n, 128), 128, 0, ctx->stream>>>(a);
    FP_LAUNCHED(ctx);
    ctx->ctr.planned_agents += ctx->alive;
    return FP_OK;
}

int fp_choice_launch(fp_ctx* ctx, uint32_t agent, double k_s, int32_t* d_cx, int32_t* d_cy,
                     double* d_w, float* d_p, uint32_t* d_n) {
    PlanArgs a = make_args(ctx, k_s, 0);
    choice_kernel<<<1, 1, 0, ctx->stream>>>(a, agent, d_cx, d_cy, d_w, d_p, d_n);
    FP_LAUNCHED(ctx);
    return FP_OK;
}
