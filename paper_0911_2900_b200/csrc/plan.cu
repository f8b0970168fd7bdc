// plan.cu -- the planning phase: choose_desired_cell for every alive agent.
//
// Reference: plan_phase (engine.hpp:71-84) -> choose_desired_cell (planning.hpp:88-108)
//            -> enumerate_candidates (planning.hpp:23-57), line_of_sight (world.hpp:181-191),
//               potential_drop (planning.hpp:76-80), std::exp, sample_index (:63-73).
//
// Production path (plan_tile_kernel): a persistent CTA per SM walks the non-empty plan tiles.
// For each tile, TMA brings the tile + 5-cell halo of the weight plane (plane.cu, 4 B/cell)
// into shared memory (double-buffered, mbarrier completion) while the previous tile computes;
// the occupancy bits of the same window are staged beside it.  One thread plans one agent:
//   pass 1  rows centre-out, so the line-of-sight test of a cell only needs the wall bits of
//           rows already seen (ball wall mask, 121 bits) AND a per-offset Bresenham path mask
//           (constant memory); each valid candidate's weight m_c*2^(C_p-C_c) is built from the
//           plane word with integer ops (the exact value of an fp32-rounded weight) and summed
//           per row pairwise in fp32, the row sums in fp64;
//   pass 2  threshold u*total picks the row, the row is replayed in the reference's list order
//           (rotated at a periodic seam) to find the first cumulative weight > threshold.
// Guard band: every weight is the reference weight times a common factor to within 2^-24
// (1.5e-7 covered that with exact sums).  The pairwise fp32 row sums (depth <= 4 for <= 11
// terms) are within gamma_4 = 4*2^-24/(1-4*2^-24) < 2.4e-7 of the exact row sums, so the total,
// the threshold and every cumulative boundary move by at most 2.4e-7*total each: 1.5e-7 + 2 *
// 2.4e-7 < 8e-7.  If the threshold lies further than 8e-7*total from both cumulative boundaries
// of the chosen candidate, the reference (serial fp64 sum, glibc exp) picks the same candidate;
// otherwise the agent is re-sampled on the exact path.
//
// Exact path (choose_exact): one thread, candidates in list order, weights through the
// bit-exact restated glibc exp (fp_exp.h), serial fp64 total and scan -- bitwise the
// reference's arithmetic.  Used for guard-band misses, "unsafe" plane cells, k_s/grid shapes the
// tiled path does not cover, and test-mode dumps.  There is no CPU fallback.
#include <math.h>

#include "fp_exp.h"
#include "internal.cuh"
#include "motion_rec.cuh"

#define FP_GUARD 8e-7  // see the guard-band note above

// Walk records (motion_rec.cuh): the plan emits them for the motion phase.
__constant__ signed char c_bpath_p[121][5][2];

// Bresenham path masks over the 11x11 offset frame (bit (dy+5)*11 + dx+5): the cells strictly
// between (0,0) and (dx,dy) on the segment (world.hpp:143-167).
__constant__ uint32_t c_pathmask[121][4];
static bool g_pathmask_ready[64] = {false};

static void host_pathmasks(uint32_t out[121][4]) {
    for (int dy = -5; dy <= 5; ++dy)
        for (int dx = -5; dx <= 5; ++dx) {
            uint32_t* m = out[(dy + 5) * 11 + dx + 5];
            m[0] = m[1] = m[2] = m[3] = 0;
            const int tx = dx, ty = dy;
            const int adx = abs(tx), sx = 0 < tx ? 1 : -1;
            const int ady = -abs(ty), sy = 0 < ty ? 1 : -1;
            int err = adx + ady, x = 0, y = 0;
            while (!(x == tx && y == ty)) {
                const int e2 = 2 * err;
                if (e2 >= ady) { err += ady; x += sx; }
                if (e2 <= adx) { err += adx; y += sy; }
                if (x == tx && y == ty) break;
                const int b = (y + 5) * 11 + x + 5;
                m[b >> 5] |= 1u << (b & 31);
            }
        }
}

static int ensure_pathmasks(fp_ctx* ctx) {
    if (ctx->device < 64 && g_pathmask_ready[ctx->device]) return FP_OK;
    uint32_t pm[121][4];
    host_pathmasks(pm);
    FP_CUDA(ctx, cudaMemcpyToSymbol(c_pathmask, pm, sizeof(pm)));
    signed char bp[121][5][2];
    host_bpath(bp);
    FP_CUDA(ctx, cudaMemcpyToSymbol(c_bpath_p, bp, sizeof(bp)));
    if (ctx->device < 64) g_pathmask_ready[ctx->device] = true;
    return FP_OK;
}

struct PlanCommon {
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
    DevScalars* sc;
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
__device__ __forceinline__ void for_each_candidate(const PlanCommon& a, int px, int py, int v, F&& f) {
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

__device__ __forceinline__ ExactWeight make_weight(const PlanCommon& a, int px, int py) {
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

// choose_desired_cell, exact (planning.hpp:88-108 + sample_index :63-73), for agent id i standing
// at (px, py) with radius v
__device__ __noinline__ void choose_exact_at(const PlanCommon& a, uint32_t i, int px, int py, int v, uint64_t step,
                                             int* ox, int* oy) {
    const ExactWeight wf = make_weight(a, px, py);
    double total = 0.0;
    int lastx = px, lasty = py;
    for_each_candidate(a, px, py, v, [&](int x, int y) {
        total = FPX_ADD(total, wf(x, y));
        lastx = x;
        lasty = y;
        return true;
    });
    const double u = fp_unit_interval(fp_rng_u64(a.seed, i, step, 0));
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

__device__ __forceinline__ void choose_exact(const PlanCommon& a, uint32_t i, uint64_t step, int* ox, int* oy) {
    choose_exact_at(a, i, a.g.wrap(a.x[i]), a.y[i], a.v[i], step, ox, oy);
}

// Host-API single-agent entry points (fp_choose_desired / fp_enumerate_candidates): an agent
// given by value against the context's occupancy snapshot (the reference's const SimState&).
__global__ void choose_one_kernel(PlanCommon a, uint32_t id, int px, int py, int v, long long step, int32_t* out) {
    int cx, cy;
    choose_exact_at(a, id, a.g.wrap(px), py, v, (uint64_t)step, &cx, &cy);
    out[0] = cx;
    out[1] = cy;
}

__global__ void candidates_one_kernel(PlanCommon a, int px, int py, int v, int32_t* cx, int32_t* cy, uint32_t* n_out) {
    uint32_t n = 0;
    for_each_candidate(a, a.g.wrap(px), py, v, [&](int x, int y) {
        cx[n] = x;
        cy[n] = y;
        ++n;
        return true;
    });
    *n_out = n;
}

__global__ void plan_exact_kernel(PlanCommon a) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.n || !a.alive[i]) return;
    int cx, cy;
    choose_exact(a, i, (uint64_t)a.sc->step, &cx, &cy);
    a.dx[i] = cx;
    a.dy[i] = cy;
}

// ------------------------------------------------------------------------------ fast weights
enum { MODE_EXIT = 0, MODE_ONES = 1, MODE_DRIVE = 2 };

// Weight of a non-wall candidate word, as an exact fp64 value (an fp32-precision weight).
__device__ __forceinline__ double fast_weight(uint32_t w, int Cp, int mode, double drive_w) {
    if (mode == MODE_ONES) return 1.0;
    if (mode == MODE_DRIVE) return drive_w;
    if (w & FP_W_SPECIAL) return 0.0;  // unreachable (walls never get here)
    const int d = ((int)((uint32_t)(Cp - (int)((w >> 23) & 0x7Fu)) << 25)) >> 25;
    const uint32_t mant = w & 0x7FFFFFu;
    const int hi = ((1023 + d) << 20) | (int)(mant >> 3);
    const int lo = (int)((mant & 7u) << 29);
    return __hiloint2double(hi, lo);
}

__device__ __forceinline__ float drive_weight_f(double k_s, double g, int dx) {
    return (float)fpx_exp(FPX_MUL(k_s, FPX_MUL(g, (double)dx)));
}

// ------------------------------------------------------------------------------ tile kernel
struct TileArgs {
    PlanCommon c;
    int PW;
    const uint32_t* plane;
    const uint32_t* bucket;
    const uint4* brec;
    const uint32_t* tile_off;
    const uint32_t* tile_cnt;
    const uint32_t* tile_list;
    const uint8_t* tile_exit;  // an Exit within the tile's window
    const uint32_t* deal;  // [gridDim.x * passes + 1] first list entry of each range
    int passes;
    int tile_w, tile_h, tiles_x;
    int use_tma;  // 0: stage the box with coalesced loads (debug / comparison path)
    int boxw, boxh, occw;  // shared-memory strides (words)
    uint2* fallback;       // (id, bucket position) handed to plan_exact_list_kernel
    uint4* rec0;           // walk records in bucket order (motion_rec.cuh), when emit
    uint32_t* p1;          // contention marks
    uint32_t* p2;
    int emit;
    int mixed;  // roster has more than one v_max: the masked radius-5 variant for everyone
    int rot;    // thread rotation between consecutive fetches (multiple of the lanes per agent)
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

// Bounded wait on an mbarrier phase: false if the phase never completed (error, not a hang).
__device__ __forceinline__ bool mbar_wait(uint64_t* bar, unsigned parity) {
    for (int spin = 0; spin < (1 << 22); ++spin) {
        uint32_t ok;
        asm volatile(
            "{\n"
            ".reg .pred p;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p;\n"
            "}\n"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (ok) return true;
    }
    return false;
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int cx, int cy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(cx), "r"(cy)
        : "memory");
}

// Pair of u64 words holding the 121-bit ball wall mask (bit (dy+5)*11 + dx+5).
struct Mask121 {
    unsigned long long lo, hi;
};

// B: frame bit of the row's first cell (a constant once the row loop is unrolled)
__device__ __forceinline__ void mask_or_row(Mask121& m, uint32_t rowbits, int B) {
    if (B < 64) m.lo |= (unsigned long long)rowbits << B;
    if (B + 11 > 64) m.hi |= (B >= 64) ? ((unsigned long long)rowbits << (B - 64)) : ((unsigned long long)rowbits >> (64 - B));
}

__device__ __forceinline__ bool path_blocked(const Mask121& m, int o) {
    const unsigned long long plo = ((unsigned long long)c_pathmask[o][1] << 32) | c_pathmask[o][0];
    const unsigned long long phi = ((unsigned long long)c_pathmask[o][3] << 32) | c_pathmask[o][2];
    return ((m.lo & plo) | (m.hi & phi)) != 0ull;
}

// Weight of a reachable plane word in ExitDistance mode as an exact fp64 number:
// m_c * 2^(C_p - C_c), with (C_p - C_c) recovered mod 128 (|d| <= 60 on safe cells).
__device__ __forceinline__ double exit_weight(uint32_t w, int cp_biased /* C_p + 64 (+128) */) {
    const uint32_t t = (uint32_t)(cp_biased - (int)(w >> 23)) & 127u;  // d + 64
    const int hi = (int)((t << 20) + (959u << 20)) | (int)((w >> 3) & 0xFFFFFu);
    const int lo = (int)(w << 29);
    return __hiloint2double(hi, lo);
}

__device__ __forceinline__ unsigned long long globaltimer_p() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// Path mask test against the shared-memory copy of c_pathmask (lanes index it divergently).
__device__ __forceinline__ bool path_blocked_s(const uint4* pm, const Mask121& m, int o) {
    const uint4 q = pm[o];
    const unsigned long long plo = ((unsigned long long)q.y << 32) | q.x;
    const unsigned long long phi = ((unsigned long long)q.w << 32) | q.z;
    return ((m.lo & plo) | (m.hi & phi)) != 0ull;
}

// The same weight as an fp32 number -- exact: the plane keeps a 23-bit mantissa and
// |C_p - C_c| <= 60 stays inside the fp32 exponent range.
__device__ __forceinline__ float exit_weight32(uint32_t w, int cp_biased) {
    const uint32_t t = (uint32_t)(cp_biased - (int)(w >> 23)) & 127u;  // d + 64
    return __uint_as_float(((t + 63u) << 23) | (w & 0x7FFFFFu));
}

// Pairwise fp32 sum of x[0..N) (depth ceil(log2 N): the error bound the guard band assumes).
template <int N>
__device__ __forceinline__ float pairwise_sum(const float* x) {
    if constexpr (N == 1) {
        return x[0];
    } else {
        constexpr int H = (N + 1) / 2;
        return pairwise_sum<H>(x) + pairwise_sum<N - H>(x + H);
    }
}

// Plans one agent from the staged tile (V = its v_max, DRIVE = DriveX potential) with P lanes
// (P consecutive threads of a warp, all calling with the same agent).  Returns 1 when the fast
// path decided (result in *ox, *oy, identical in every lane), 2 when the exact path must decide.
//   walls   every lane ORs the ball's wall bits (staged wall bitplane, one word pair per row)
//   pass 1  lane l takes rows t = l, l+P, ... of the centre-out order: valid candidates (not
//           Wall/unreachable, not occupied by another agent, visible) contribute their exact
//           fp32 weight to a pairwise fp32 row sum; the row sums are gathered into every lane
//           and accumulated in fp64
//   pass 2  u*total picks the row; the row is replayed in list order (wrapped-x sorted at a
//           periodic seam) to find the first cumulative weight > threshold; guard band.
// Every sum is taken in the same order for any P, so the decision does not depend on P.
// MASKED: one radius-V code path for every v_max <= V (mixed rosters): rows and columns beyond
// the agent's own radius vr are masked out, which leaves exactly its Chebyshev ball (the line
// of sight to a cell of the ball only crosses cells of the ball), so decisions are unchanged
// while the warps of a mixed roster share one instruction stream.
template <int V, bool DRIVE, bool MASKED = false, int P = 1>
__device__ __forceinline__ int plan_fast_t(const TileArgs& A, const uint32_t* buf, const uint32_t* occs,
                                           const uint32_t* walls, const uint4* pathm, int osh0, int x0, int y0,
                                           int px, int py, double u, const double* drive_tab, int* ox, int* oy,
                                           int vr = V) {
    constexpr int D = 2 * V + 1;
    constexpr int RPL = (D + P - 1) / P;  // rows per lane
    const int lane = P > 1 ? (int)(threadIdx.x & (P - 1)) : 0;
    const unsigned gmask = P > 1 ? (((1u << P) - 1u) << ((threadIdx.x & 31u) & ~(unsigned)(P - 1))) : 0xffffffffu;
    const PlanCommon& a = A.c;
    const uint32_t colmask = MASKED ? (((1u << (2 * vr + 1)) - 1u) << (V - vr)) : ((1u << D) - 1u);
    const int X0 = x0 - 8;  // box origin (TMA inner coordinates stay 16-byte aligned)
    const int lx = px - X0, ly = py - (y0 - FP_HALO);
    int cpb = 0;
    if (!DRIVE) {
        const uint32_t own = buf[ly * A.boxw + lx];
        if (own & (FP_W_SPECIAL | FP_W_UNSAFE)) return 2;  // "ones" pocket / unsafe centre
        cpb = (int)((own >> 23) & 0x7Fu) + 64 + 128;
    }
    const int osh = osh0 + lx - V;  // staged bitplane bit of dx = -V
    Mask121 wm{0ull, 0ull};
#pragma unroll
    for (int dy = -V; dy <= V; ++dy) {
        if ((unsigned)(py + dy) >= (unsigned)a.g.H) continue;
        const uint32_t* wrow = walls + (ly + dy) * A.occw;
        const uint32_t wb = __funnelshift_r(wrow[osh >> 5], wrow[(osh >> 5) + 1], osh & 31) & ((1u << D) - 1u);
        mask_or_row(wm, wb, (dy + 5) * 11 + 5 - V);
    }
    const bool anywall = (wm.lo | wm.hi) != 0ull;
    float dw[D];  // DriveX weights by column (exact fp32 values)
#pragma unroll
    for (int k = 0; k < D; ++k) dw[k] = DRIVE ? (float)drive_tab[k - V + 5] : 0.0f;
    float rso[RPL];
#pragma unroll
    for (int j = 0; j < RPL; ++j) {
        const int t = j * P + lane;  // centre-out row index: 0, -1, 1, -2, 2, ...
        float s = 0.0f;
        if (t < D) {
            const int dy = (t & 1) ? -((t + 1) >> 1) : (t >> 1);
            const bool rowok = (unsigned)(py + dy) < (unsigned)a.g.H;
            const uint32_t* row = buf + (ly + dy) * A.boxw + lx - V;
            uint32_t wv[D];
            uint32_t spec = 0u;
#pragma unroll
            for (int k = 0; k < D; ++k) {
                wv[k] = row[k];
                spec |= (wv[k] >> 31) << k;
            }
            const uint32_t* orow = occs + (ly + dy) * A.occw;
            uint32_t occ = __funnelshift_r(orow[osh >> 5], orow[(osh >> 5) + 1], osh & 31);
            if (dy == 0) occ &= ~(1u << V);  // the own cell stays a candidate (planning.hpp:45-46)
            const bool inball = !MASKED || (dy <= vr && -dy <= vr);
            uint32_t valid = (rowok && inball) ? (~(spec | occ) & colmask) : 0u;
            if (anywall) {
#pragma unroll
                for (int k = 0; k < D; ++k)
                    if (path_blocked_s(pathm, wm, (dy + 5) * 11 + k - V + 5)) valid &= ~(1u << k);
            }
            float w[D];
#pragma unroll
            for (int k = 0; k < D; ++k)
                w[k] = ((valid >> k) & 1u) ? (DRIVE ? dw[k] : exit_weight32(wv[k], cpb)) : 0.0f;
            s = pairwise_sum<D>(w);
        }
        rso[j] = s;
    }
    double rs[D];  // row sums, indexed by dy + V
#pragma unroll
    for (int k = 0; k < D; ++k) {
        const int dy = k - V;
        const int t = dy >= 0 ? 2 * dy : -2 * dy - 1;
        rs[k] = (double)(P > 1 ? __shfl_sync(gmask, rso[t / P], t % P, P) : rso[t]);
    }
    double T = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) T += rs[k];
    const double theta = u * T;
    int rstar = -1;
    double before = 0.0, cum = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
        const bool hit = rstar < 0 && cum + rs[k] > theta;
        before = hit ? cum : before;
        rstar = hit ? k : rstar;
        cum += rs[k];
    }
    if (rstar < 0) return 2;  // u*total rounded up to total
    const int dy = rstar - V;
    const uint32_t* row = buf + (ly + dy) * A.boxw + lx;
    const uint32_t* orow = occs + (ly + dy) * A.occw;
    uint32_t occ = __funnelshift_r(orow[osh >> 5], orow[(osh >> 5) + 1], osh & 31);
    if (dy == 0) occ &= ~(1u << V);
    const int R = MASKED ? vr : V;  // the agent's radius
    int a0 = -R, a1 = R, b0 = 0, b1 = -1;
    if (a.g.boundary == FP_BOUNDARY_PERIODIC_X) {  // wrapped-x order at the seam (planning.hpp:50-53)
        if (px + R >= a.g.W) {
            a0 = a.g.W - px; b0 = -R; b1 = a.g.W - px - 1;
        } else if (px - R < 0) {
            a0 = -px; b0 = -R; b1 = -px - 1;
        }
    }
    double prefix = before, lower = 0.0, upper = 0.0;
    int kx = 0;
    bool found = false;
    for (int seg = 0; seg < 2 && !found; ++seg) {
        const int lo = seg ? b0 : a0, hi = seg ? b1 : a1;
        for (int dx = lo; dx <= hi; ++dx) {
            const uint32_t w = row[dx];
            if (w >> 31) continue;                 // wall / unreachable (weight 0)
            if ((occ >> (dx + V)) & 1u) continue;  // occupied by another agent
            if (anywall && path_blocked_s(pathm, wm, (dy + 5) * 11 + dx + 5)) continue;
            const double wt = DRIVE ? drive_tab[dx + 5] : exit_weight(w, cpb);
            const double next = prefix + wt;
            if (next > theta) {
                lower = prefix;
                upper = next;
                kx = dx;
                found = true;
                break;
            }
            prefix = next;
        }
    }
    if (!found) return 2;
    const double margin = FP_GUARD * T;
    if (!(upper - theta > margin)) return 2;
    if (!(lower == 0.0 || theta - lower > margin)) return 2;
    int cx = px + kx;
    if (cx < 0) cx += a.g.W;  // periodic seam (|kx| <= 5 < W)
    else if (cx >= a.g.W) cx -= a.g.W;
    *ox = cx;
    *oy = py + dy;
    return 1;
}

// record_of (motion_rec.cuh) for a fast-path decision inside the staged tile: the target lies in
// the ball, the Wall test reads the staged plane words, and the Exit test (global bitplane) runs
// only in tiles whose window holds an Exit.
__device__ __forceinline__ uint4 record_of_tile(const Geo& g, const uint32_t* occ, bool tile_exit, const uint32_t* buf,
                                                int boxw, int lx, int ly, uint32_t id, int sx, int sy, int tx, int ty,
                                                int v, const signed char (*bp)[5][2]) {
    const int ddx = g.segment_dx(sx, tx), ddy = ty - sy;
    const int o = (ddy + 5) * 11 + ddx + 5;
    const int len = min(max(abs(ddx), abs(ddy)), v);
    int m = 0, ex_x = 0, ex_y = 0;
    bool ex = false;
    for (int j = 0; j < len; ++j) {
        const int ox = bp[o][j][0], oy = bp[o][j][1];
        if (buf[(ly + oy) * boxw + lx + ox] == FP_W_WALL) break;
        ++m;
        if (tile_exit) {
            const int x = g.wrap(sx + ox), y = sy + oy;
            if (g.is_exit(x, y)) {
                ex = true;
                ex_x = x;
                ex_y = y;
                break;
            }
        }
    }
    const bool exit_free = ex && !((__ldcg(&occ[g.word(ex_x, ex_y)]) >> (ex_x & 31)) & 1u);
    return make_uint4(id, 0u,
                      (uint32_t)sx | (exit_free ? REC_EXIT_FREE : 0u) | ((uint32_t)m << 28) | (ex ? 0x80000000u : 0u),
                      (uint32_t)sy | ((uint32_t)o << 24));
}

template <bool DRIVE, int P>
__device__ __forceinline__ int plan_fast_v(int v, const TileArgs& A, const uint32_t* buf, const uint32_t* occs,
                                           const uint32_t* walls, const uint4* pathm, int osh0, int x0, int y0,
                                           int px, int py, double u, const double* drive_tab, int* ox, int* oy) {
#define FP_PLAN_ARGS A, buf, occs, walls, pathm, osh0, x0, y0, px, py, u, drive_tab, ox, oy
    if (A.mixed)  // one instruction stream for a mixed-v roster (see plan_fast_t)
        return plan_fast_t<5, DRIVE, true, P>(FP_PLAN_ARGS, v);
    switch (v) {
        case 1: return plan_fast_t<1, DRIVE, false, P>(FP_PLAN_ARGS);
        case 2: return plan_fast_t<2, DRIVE, false, P>(FP_PLAN_ARGS);
        case 3: return plan_fast_t<3, DRIVE, false, P>(FP_PLAN_ARGS);
        case 4: return plan_fast_t<4, DRIVE, false, P>(FP_PLAN_ARGS);
        default: return plan_fast_t<5, DRIVE, false, P>(FP_PLAN_ARGS);
    }
#undef FP_PLAN_ARGS
}

#define PLAN_THREADS 512
#ifndef FP_PLAN_NAP_MAX
#define FP_PLAN_NAP_MAX 256  // ns
#endif
#ifndef PLAN_SLOTS
#define PLAN_SLOTS 3  // tiles resident per CTA
#endif

// Persistent CTA per SM.  Tiles are fetched in pairs of buffer slots (TMA, mbarrier); the
// agents of fetch i are dealt to threads round-robin starting at thread (i*160) mod 512, one
// agent per thread.  There is no CTA-wide barrier per tile: a thread finishing its agents of
// fetch i moves on to fetch i+1; the thread that completes the last agent of fetch i refills
// that slot with fetch i+2.  Slot metadata is published with a generation number (seqlock).
// Diagnostics read by tools/debug_plan.py and tools/debug_plan_cta.py: the fetch timeline of CTA
// 5 (issue, TMA ready, last agent done, agents) and every CTA's start, end and fetch count.
__device__ unsigned long long g_plan_dbg[4 * 256];
extern "C" int fp_debug_plan(unsigned long long* out) {
    return (int)cudaMemcpyFromSymbol(out, g_plan_dbg, sizeof(g_plan_dbg));
}
__device__ unsigned long long g_plan_cta[3 * 256];
extern "C" int fp_debug_plan_cta(unsigned long long* out) {
    return (int)cudaMemcpyFromSymbol(out, g_plan_cta, sizeof(g_plan_cta));
}
// P consecutive threads plan each agent together (plan_fast_t).
template <int P>
__global__ void __launch_bounds__(PLAN_THREADS, 1) plan_tile_kernel(const __grid_constant__ CUtensorMap tmap,
                                                                    const __grid_constant__ CUtensorMap tmap_occ,
                                                                    const __grid_constant__ CUtensorMap tmap_wall,
                                                                    TileArgs A) {
    extern __shared__ __align__(128) uint32_t smem_raw[];
    uint32_t* smem = smem_raw + (((128u - (smem_u32(smem_raw) & 127u)) & 127u) >> 2);
    const int box_words = A.boxw * A.boxh;
    const int box_stride = (box_words + 31) & ~31;  // words, 128-byte multiple
    const int occ_words = A.boxh * A.occw;
    const int occ_stride = (occ_words + 31) & ~31;
    const unsigned tx_bytes = (unsigned)(box_words + 2 * occ_words) * 4u;
    uint64_t* bars = (uint64_t*)(smem + PLAN_SLOTS * box_stride + 2 * PLAN_SLOTS * occ_stride);
    // slot metadata is written by one thread and read by others without a CTA barrier: volatile
    __shared__ volatile int s_tile[PLAN_SLOTS], s_cnt[PLAN_SLOTS], s_off[PLAN_SLOTS], s_x0[PLAN_SLOTS],
        s_y0[PLAN_SLOTS];
    __shared__ volatile int s_gen[PLAN_SLOTS];
    __shared__ int s_done[PLAN_SLOTS];
    __shared__ double s_drive[11];
    __shared__ signed char s_bp[121][5][2];
    __shared__ uint4 s_pathm[121];
    for (int k = threadIdx.x; k < 121 * 10; k += blockDim.x) (&s_bp[0][0][0])[k] = (&c_bpath_p[0][0][0])[k];
    for (int k = threadIdx.x; k < 121; k += blockDim.x)
        s_pathm[k] = make_uint4(c_pathmask[k][0], c_pathmask[k][1], c_pathmask[k][2], c_pathmask[k][3]);
    const PlanCommon& a = A.c;
    const uint64_t step = (uint64_t)a.sc->step;
    // list entry of fetch number i, or -1 past the end
    auto fetch_entry = [&](int i) {
        for (int p = 0, k = i; p < A.passes; ++p) {
            const int lo = (int)A.deal[p * gridDim.x + blockIdx.x], hi = (int)A.deal[p * gridDim.x + blockIdx.x + 1];
            if (k < hi - lo) return lo + k;
            k -= hi - lo;
        }
        return -1;
    };
    // fetch number i into slot i % PLAN_SLOTS (one thread)
    auto fetch = [&](int i) {
        const int slot = i % PLAN_SLOTS;
        s_gen[slot] = -1;  // seqlock: readers that raced with this refill see a changed generation
        __threadfence_block();
        // fetch i of this CTA is the i-th entry of its ranges (one per pass, bucket.cu
        // tile_deal_kernel) taken in order, so fetch numbers map monotonically onto the list and
        // an exhausted fetch ends every later one (refills complete out of order)
        const int t = fetch_entry(i);
#ifdef FP_PLAN_DEBUG
        if (blockIdx.x == 5 && i < 256) g_plan_dbg[i] = globaltimer_p();
#endif
        if (t >= 0) {
            const uint32_t tile = A.tile_list[t];
            const int tx = (int)(tile % (uint32_t)A.tiles_x), ty = (int)(tile / (uint32_t)A.tiles_x);
            const int x0 = tx * A.tile_w, y0 = ty * A.tile_h;
            s_tile[slot] = (int)tile;
            s_cnt[slot] = (int)A.tile_cnt[tile];
            s_off[slot] = (int)A.tile_off[tile];
            s_x0[slot] = x0;
            s_y0[slot] = y0;
            s_done[slot] = 0;
            if (A.use_tma) {
                const int gws = ((x0 - 8 + FP_XPAD_BITS) >> 5) & ~3;
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_expect_tx(&bars[slot], tx_bytes);
                tma_load_2d(smem + slot * box_stride, &tmap, &bars[slot], x0 - 8 + FP_XPAD_W, y0 - FP_HALO);
                tma_load_2d(smem + PLAN_SLOTS * box_stride + slot * occ_stride, &tmap_occ, &bars[slot], gws,
                            y0 - FP_HALO);
                tma_load_2d(smem + PLAN_SLOTS * box_stride + (PLAN_SLOTS + slot) * occ_stride, &tmap_wall,
                            &bars[slot], gws, y0 - FP_HALO);
            }
        } else {
            s_tile[slot] = -1;
        }
        __threadfence_block();
        s_gen[slot] = i;
    };
    if (threadIdx.x == 0) {
        for (int s = 0; s < PLAN_SLOTS; ++s) mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int s = 0; s < PLAN_SLOTS; ++s) s_gen[s] = -1;
    }
    if (threadIdx.x < 11) {
        s_drive[threadIdx.x] = (a.potential == FP_POTENTIAL_DRIVE_X)
                                   ? (double)drive_weight_f(a.k_s, a.drive_gradient, (int)threadIdx.x - 5)
                                   : 0.0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
#ifdef FP_PLAN_DEBUG
        if (blockIdx.x < 256) {
            g_plan_cta[blockIdx.x] = globaltimer_p();
            g_plan_cta[256 + blockIdx.x] = 0;
        }
#endif
        for (int s = 0; s < PLAN_SLOTS; ++s) fetch(s);
    }
    for (int i = 0;; ++i) {
        const int slot = i % PLAN_SLOTS;
        // bounded wait: a scheduling bug must surface as an error flag, never as a hung GPU
        // (-1 while a refill is being published; a generation past i means fetch i already
        // completed without this thread -- it had no agent there -- and the slot moved on)
        // (exponential backoff: idle threads must not steal issue slots from the computing warps)
        int gen;
        unsigned nap = 32;
        for (long long spin = 0; (gen = s_gen[slot]) < i; ++spin) {
            __nanosleep(nap);
            nap = min(nap * 2u, (unsigned)FP_PLAN_NAP_MAX);
            if (spin > (1ll << 22)) {
                atomicOr(&a.sc->err, 1ull);
                return;
            }
        }
        if (gen > i) continue;
        const int tile = s_tile[slot];
        const int cnt = s_cnt[slot], off = s_off[slot], x0 = s_x0[slot], y0 = s_y0[slot];
        __threadfence_block();
        // validate the snapshot before acting on any of it (including the end-of-list marker:
        // a refill racing with these reads may already have written tile = -1 for fetch i+2)
        if (s_gen[slot] != i) continue;  // fetch i already completed without this thread's help
        if (tile < 0) {
#ifdef FP_PLAN_DEBUG
            if (blockIdx.x < 256 && (threadIdx.x & 31) == 0) {
                atomicMax(&g_plan_cta[256 + blockIdx.x], globaltimer_p());
                g_plan_cta[512 + blockIdx.x] = i;
            }
#endif
            break;
        }
        // agent slot of this thread's lane group (the rotation keeps groups P-aligned)
        int k = (((int)threadIdx.x - i * A.rot) & (PLAN_THREADS - 1)) / P;
        if (k >= cnt) continue;  // no agent of this fetch for this thread
        uint32_t* buf = smem + slot * box_stride;
        uint32_t* occs = smem + PLAN_SLOTS * box_stride + slot * occ_stride;
        uint32_t* walls = smem + PLAN_SLOTS * box_stride + (PLAN_SLOTS + slot) * occ_stride;
        const int gws = ((x0 - 8 + FP_XPAD_BITS) >> 5) & ~3;
        const int osh0 = x0 - 8 + FP_XPAD_BITS - gws * 32;  // staged-occupancy bit of box column 0
        if (A.use_tma) {
            if (!mbar_wait(&bars[slot], (unsigned)(i / PLAN_SLOTS) & 1u)) {
                atomicOr(&a.sc->err, 2ull);
                return;
            }
#ifdef FP_PLAN_DEBUG
            if (blockIdx.x == 5 && i < 256 && g_plan_dbg[256 + i] < g_plan_dbg[i]) g_plan_dbg[256 + i] = globaltimer_p();
#endif
        } else if (true) {
            // comparison path: each thread fills what it reads (slow; debugging only)
            const int gx0 = x0 - 8 + FP_XPAD_W, gy0 = y0 - FP_HALO;
            for (int e = 0; e < box_words; ++e) {
                const int r = e / A.boxw, cidx = e % A.boxw;
                const int gy = gy0 + r, gx = gx0 + cidx;
                buf[e] = (gy >= 0 && gy < a.g.H && gx < A.PW) ? A.plane[(size_t)gy * A.PW + gx] : 0u;
            }
            for (int e = 0; e < occ_words; ++e) {
                const int r = e / A.occw, wcol = e % A.occw;
                const int gy = gy0 + r, gw = gws + wcol;
                const bool in = gy >= 0 && gy < a.g.H && gw < a.g.P;
                occs[e] = in ? a.occ[(size_t)gy * a.g.P + gw] : 0u;
                walls[e] = in ? a.g.wall[(size_t)gy * a.g.P + gw] : 0u;
            }
        }
        int mine = 0;
        const bool lead = (threadIdx.x & (P - 1)) == 0;
        for (; k < cnt; k += PLAN_THREADS / P) {
            const uint4 br = __ldcg(&A.brec[off + k]);  // (id, wrapped x, y, v_max), bucket.cu
            const uint32_t id = br.x;
            const int px = (int)br.y, py = (int)br.z;
            const int v = (int)br.w;
            const double u = fp_unit_interval(fp_rng_u64(a.seed, id, step, 0));
            int cx = 0, cy = 0;
            const int st = (a.potential == FP_POTENTIAL_DRIVE_X)
                               ? plan_fast_v<true, P>(v, A, buf, occs, walls, s_pathm, osh0, x0, y0, px, py, u,
                                                      s_drive, &cx, &cy)
                               : plan_fast_v<false, P>(v, A, buf, occs, walls, s_pathm, osh0, x0, y0, px, py, u,
                                                       s_drive, &cx, &cy);
            if (!lead) {
                // the group's other lanes: nothing to write
            } else if (st == 1) {
                a.dx[id] = cx;
                a.dy[id] = cy;
                if (A.emit)  // the motion's walk record, walls from the staged plane
                    A.rec0[off + k] = record_of_tile(a.g, a.occ, A.tile_exit[tile], buf, A.boxw, px - (x0 - 8),
                                                     py - (y0 - FP_HALO), id, px, py, cx, cy, v, s_bp);
            } else {  // decided by the exact path after the sweep (plan_exact_list_kernel)
                A.fallback[atomicAdd(&a.sc->fb_count, 1ull)] = make_uint2(id, (uint32_t)(off + k));
            }
            ++mine;
        }
        // release: this thread's reads of the slot happen before its count lands (without the
        // fence the compiler may sink shared loads below the relaxed atomic and the refill
        // TMA would overwrite data still being read); the last finisher acquires, then refills
        __threadfence_block();
        if (atomicAdd(&s_done[slot], mine) + mine == cnt * P) {  // last lane of fetch i
            __threadfence_block();
#ifdef FP_PLAN_DEBUG
            if (blockIdx.x == 5 && i < 256) {
                g_plan_dbg[512 + i] = globaltimer_p();
                g_plan_dbg[768 + i] = cnt;
            }
#endif
            fetch(i + PLAN_SLOTS);
        }
    }
}

// The exact path for the agents the tiled kernel could not decide: one warp per agent.  Lanes
// own candidate slots of the ball in list order (row-major, wrapped-x sorted at the seam),
// test them against the global bitplanes (walls, occupancy, Bresenham line of sight) and compute
// the exact weights (restated glibc exp); lane 0 then folds the weights serially in list order
// (sample_index, planning.hpp:63-73).  Narrow periodic grids (2v+1 > W-?) use choose_exact.
#define EXACT_WARPS 4
struct EmitArgs {
    uint4* rec0;
    uint32_t* p1;
    uint32_t* p2;
    int emit;
};

__device__ __forceinline__ void emit_record(const PlanCommon& a, const EmitArgs& E, uint32_t id, uint32_t pos, int px,
                                            int py, int cx, int cy, int v) {
    if (!E.emit) return;
    E.rec0[pos] = record_of(a.g, a.occ, id, px, py, cx, cy, v, c_bpath_p);
}

__global__ void __launch_bounds__(EXACT_WARPS * 32) plan_exact_list_kernel(PlanCommon a, const uint2* list,
                                                                           EmitArgs E) {
    __shared__ double s_w[EXACT_WARPS][121];
    __shared__ int s_c[EXACT_WARPS][121];
    const unsigned n = (unsigned)a.sc->fb_count;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t step = (uint64_t)a.sc->step;
    for (unsigned e = blockIdx.x * EXACT_WARPS + warp; e < n; e += gridDim.x * EXACT_WARPS) {
        const uint2 ent = list[e];
        const uint32_t id = ent.x;
        const int px = a.g.wrap(a.x[id]), py = a.y[id], v = a.v[id];
        const int D = 2 * v + 1;
        if (a.g.boundary == FP_BOUNDARY_PERIODIC_X && D >= a.g.W) {
            if (lane == 0) {
                int cx, cy;
                choose_exact(a, id, step, &cx, &cy);
                a.dx[id] = cx;
                a.dy[id] = cy;
                emit_record(a, E, id, ent.y, px, py, cx, cy, v);
            }
            continue;
        }
        // list-order column -> dx (wrapped-x sort at the periodic seam, planning.hpp:50-53)
        int a0 = -v, na = D, b0 = 0;
        if (a.g.boundary == FP_BOUNDARY_PERIODIC_X) {
            if (px + v >= a.g.W) {
                a0 = a.g.W - px; na = v - a0 + 1; b0 = -v;
            } else if (px - v < 0) {
                a0 = -px; na = v - a0 + 1; b0 = -v;
            }
        }
        const ExactWeight wf = make_weight(a, px, py);
        for (int k = lane; k < D * D; k += 32) {
            const int r = k / D, c = k % D;
            const int y = py - v + r;
            const int dx = c < na ? a0 + c : b0 + (c - na);
            int x = px + dx;
            bool ok = y >= 0 && y < a.g.H;
            if (a.g.boundary == FP_BOUNDARY_PERIODIC_X) x = a.g.wrap(x);
            else ok = ok && x >= 0 && x < a.g.W;
            ok = ok && !a.g.is_wall(x, y);
            ok = ok && !(occ_bit(a.occ, a.g, x, y) && !(x == px && y == py));
            ok = ok && los(a.g, px, py, x, y);
            s_w[warp][k] = ok ? wf(x, y) : -1.0;
            s_c[warp][k] = ok ? (y * a.g.W + x) : -1;
        }
        __syncwarp();
        if (lane == 0) {
            double total = 0.0;
            int last = -1;
            for (int k = 0; k < D * D; ++k)
                if (s_c[warp][k] >= 0) {
                    total = FPX_ADD(total, s_w[warp][k]);
                    last = k;
                }
            const double threshold = FPX_MUL(fp_unit_interval(fp_rng_u64(a.seed, id, step, 0)), total);
            double cum = 0.0;
            int pick = last;
            for (int k = 0; k < D * D; ++k)
                if (s_c[warp][k] >= 0) {
                    cum = FPX_ADD(cum, s_w[warp][k]);
                    if (cum > threshold) {
                        pick = k;
                        break;
                    }
                }
            const int cell = s_c[warp][pick];
            const int cx = cell % a.g.W, cy = cell / a.g.W;
            a.dx[id] = cx;
            a.dy[id] = cy;
            emit_record(a, E, id, ent.y, px, py, cx, cy, v);
        }
        __syncwarp();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) a.sc->fallbacks += n;
}

// Test mode (fp_get_choice): candidates in list order, exact weights and the production
// path's choice probabilities (fast weights / fast total, fp32).
__global__ void choice_kernel(PlanCommon a, const uint32_t* plane, int PW, uint32_t i, int32_t* cx, int32_t* cy,
                              double* w, float* p, uint32_t* n_out) {
    const int px = a.g.wrap(a.x[i]);
    const int py = a.y[i];
    const ExactWeight wf = make_weight(a, px, py);
    const uint32_t own = plane ? plane[(size_t)py * PW + px + FP_XPAD_W] : 0u;
    int mode = MODE_EXIT, Cp = 0;
    if (a.potential == FP_POTENTIAL_DRIVE_X) mode = MODE_DRIVE;
    else if (own == FP_W_UNREACH) mode = MODE_ONES;
    else Cp = (int)((own >> 23) & 0x7Fu);
    uint32_t n = 0;
    double fast_total = 0.0;
    for_each_candidate(a, px, py, a.v[i], [&](int x, int y) {
        cx[n] = x;
        cy[n] = y;
        w[n] = wf(x, y);
        double fw;
        if (plane) {
            const int dxs = a.g.segment_dx(px, x);
            const uint32_t word = plane[(size_t)y * PW + px + dxs + FP_XPAD_W];
            fw = fast_weight(word, Cp, mode, (double)drive_weight_f(a.k_s, a.drive_gradient, dxs));
        } else {
            fw = w[n];
        }
        p[n] = (float)fw;  // stash; normalised below
        fast_total += fw;
        ++n;
        return true;
    });
    for (uint32_t k = 0; k < n; ++k) p[k] = (float)((double)p[k] / fast_total);
    *n_out = n;
}

static PlanCommon make_common(fp_ctx* ctx, double k_s, uint64_t seed) {
    PlanCommon a;
    a.g = fp_geo(ctx);
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
    a.sc = ctx->d_sc;
    return a;
}

static bool tiled_ok(const fp_ctx* ctx) {
    // the tile frame resolves the periodic seam through ghost columns: needs 2*5+1 distinct columns
    return !(ctx->boundary == FP_BOUNDARY_PERIODIC_X && ctx->W < 16);
}

bool fp_plan_tiled(const fp_ctx* ctx) { return tiled_ok(ctx); }

int fp_plan_exact_launch(fp_ctx* ctx, double k_s, uint64_t seed) {
    if (ctx->n == 0) return FP_OK;
    PlanCommon a = make_common(ctx, k_s, seed);
    plan_exact_kernel<<<fp_blocks(ctx->n, 128), 128, 0, ctx->stream>>>(a);
    FP_LAUNCHED(ctx);
    return FP_OK;
}

static void tile_geometry(const fp_ctx* ctx, TileArgs& A, size_t& smem) {
    A.boxw = ctx->tile_w + 16;
    A.boxh = ctx->tile_h + 2 * FP_HALO;
    A.occw = 16;  // TMA box of the occupancy plane: 16 words (512 bits) from a 16-byte aligned word
    const size_t box_stride = ((size_t)A.boxw * A.boxh + 31) & ~(size_t)31;
    const size_t occ_stride = ((size_t)A.boxh * A.occw + 31) & ~(size_t)31;
    smem = (PLAN_SLOTS * box_stride + 2 * PLAN_SLOTS * occ_stride) * 4 + 8 * PLAN_SLOTS /* barriers */ +
           128 /* alignment slack */;
}

static TileArgs make_tile_args(fp_ctx* ctx, double k_s, uint64_t seed, size_t& smem, unsigned& grid) {
    TileArgs A;
    A.c = make_common(ctx, k_s, seed);
    A.PW = ctx->PW;
    A.plane = ctx->d_plane;
    A.use_tma = ctx->use_tma;
    A.bucket = ctx->d_bucket;
    A.brec = ctx->d_brec;
    A.tile_off = ctx->d_tile_off;
    A.tile_cnt = ctx->d_tile_cnt;
    A.tile_list = ctx->d_tile_list;
    A.deal = ctx->d_tile_deal;
    A.tile_exit = ctx->d_tile_exit;
    A.passes = ctx->deal_passes;
    A.tile_w = ctx->tile_w;
    A.tile_h = ctx->tile_h;
    A.tiles_x = ctx->tiles_x;
    A.fallback = ctx->d_fallback;
    A.rec0 = ctx->d_rec0;
    A.p1 = ctx->d_p1;
    A.p2 = ctx->d_p2;
    A.emit = 1;
    A.mixed = ctx->mixed_v ? 1 : 0;
    {
        static const int rot = getenv("FP_PLAN_ROT") ? atoi(getenv("FP_PLAN_ROT")) : PLAN_THREADS * 5 / 16;
        A.rot = rot;
    }
    tile_geometry(ctx, A, smem);
    const size_t nt = (size_t)ctx->tiles_x * ctx->tiles_y;
    grid = (unsigned)ctx->sm_count;  // tile_deal_kernel deals to exactly sm_count CTAs
    (void)nt;
    return A;
}

static EmitArgs emit_args(const TileArgs& A) { return EmitArgs{A.rec0, A.p1, A.p2, A.emit}; }

// Everything the planning phase allocates or builds, done outside any graph capture.
int fp_plan_prepare(fp_ctx* ctx, double k_s) {
    if (int rc = ensure_pathmasks(ctx)) return rc;
    if (!tiled_ok(ctx)) return FP_OK;
    if (int rc = fp_plane_ensure(ctx, k_s)) return rc;
    if (int rc = fp_bucket_reserve(ctx)) return rc;
    if (int rc = fp_ensure_res(ctx)) return rc;  // contention bitplanes the plan marks
    TileArgs A;
    size_t smem;
    tile_geometry(ctx, A, smem);
    static size_t configured_by_device[64] = {0};  // the attribute is per device
    size_t& configured = configured_by_device[ctx->device & 63];
    if (smem > configured) {
        FP_CUDA(ctx, cudaFuncSetAttribute(plan_tile_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        FP_CUDA(ctx, cudaFuncSetAttribute(plan_tile_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        FP_CUDA(ctx, cudaFuncSetAttribute(plan_tile_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured = smem;
    }
    return FP_OK;
}

// Threads per agent in the plan kernel (FP_PLAN_LANES: 1, 2 or 4).
static int plan_lanes() {
    static const int p = getenv("FP_PLAN_LANES") ? atoi(getenv("FP_PLAN_LANES")) : 1;
    return (p == 2 || p == 4) ? p : 1;
}

static void plan_kernel_launch(fp_ctx* ctx, const TileArgs& A, size_t smem, unsigned grid) {
    switch (plan_lanes()) {
        case 4:
            plan_tile_kernel<4><<<grid, PLAN_THREADS, smem, ctx->stream>>>(ctx->tmap_plane, ctx->tmap_occ,
                                                                           ctx->tmap_wall, A);
            break;
        case 2:
            plan_tile_kernel<2><<<grid, PLAN_THREADS, smem, ctx->stream>>>(ctx->tmap_plane, ctx->tmap_occ,
                                                                           ctx->tmap_wall, A);
            break;
        default:
            plan_tile_kernel<1><<<grid, PLAN_THREADS, smem, ctx->stream>>>(ctx->tmap_plane, ctx->tmap_occ,
                                                                           ctx->tmap_wall, A);
    }
}

static int launch_tile(fp_ctx* ctx, const TileArgs& A, size_t smem, unsigned grid) {
    FP_CUDA(ctx, cudaMemsetAsync(&ctx->d_sc->tile_next, 0, 8, ctx->stream));
    FP_CUDA(ctx, cudaMemsetAsync(&ctx->d_sc->fb_count, 0, 8, ctx->stream));
    plan_kernel_launch(ctx, A, smem, grid);
    FP_LAUNCHED(ctx);
    return FP_OK;
}

// Enqueues the whole planning phase (bucketing + tiled kernel + exact-path pass) on
// ctx->stream.  Graph-safe: the step, tile count, cursors and the fallback count live in device
// memory; fp_plan_prepare ran before.
int fp_plan_launch(fp_ctx* ctx, double k_s, uint64_t seed) {
    if (ctx->n == 0) return FP_OK;
    if (!tiled_ok(ctx)) return fp_plan_exact_launch(ctx, k_s, seed);
    if (!ctx->plane_valid || ctx->plane_ks != k_s || ctx->plane_potential != ctx->potential)
        return fp_fail(ctx, FP_ERUNTIME, "plan: weight plane not prepared for this k_s");
    if (int rc = fp_bucket_launch(ctx)) return rc;
    if (ctx->marks_dirty) {  // marks of an earlier plan no motion phase consumed
        const size_t nwords = (size_t)ctx->P * ctx->H;
        FP_CUDA(ctx, cudaMemsetAsync(ctx->d_p1, 0, nwords * 4, ctx->stream));
        FP_CUDA(ctx, cudaMemsetAsync(ctx->d_p2, 0, nwords * 4, ctx->stream));
    }
    ctx->bucket_fresh = true;  // the motion seed pass walks agents in this (spatial) order
    ctx->rec_fresh = true;     // walk records + contention marks emitted below
    ctx->marks_dirty = true;
    size_t smem;
    unsigned grid;
    const TileArgs A = make_tile_args(ctx, k_s, seed, smem, grid);
    if (int rc = launch_tile(ctx, A, smem, grid)) return rc;
    plan_exact_list_kernel<<<ctx->sm_count, EXACT_WARPS * 32, 0, ctx->stream>>>(A.c, ctx->d_fallback, emit_args(A));
    FP_LAUNCHED(ctx);
    return FP_OK;
}

// Times `iters` launches of the plan kernel alone (bucketing done once, untimed) with CUDA
// events on the launching stream; the roofline denominator of bench.py.
int fp_plan_kernel_time(fp_ctx* ctx, double k_s, uint64_t seed, int iters, double* ms) {
    if (int rc = fp_plan_prepare(ctx, k_s)) return rc;
    if (!tiled_ok(ctx) || ctx->n == 0) {
        *ms = 0.0;
        return FP_OK;
    }
    if (int rc = fp_bucket_launch(ctx)) return rc;
    size_t smem;
    unsigned grid;
    const TileArgs A = make_tile_args(ctx, k_s, seed, smem, grid);
    cudaEvent_t e0, e1;
    FP_CUDA(ctx, cudaEventCreate(&e0));
    FP_CUDA(ctx, cudaEventCreate(&e1));
    double total = 0.0;
    for (int i = 0; i < iters; ++i) {
        FP_CUDA(ctx, cudaMemsetAsync(&ctx->d_sc->tile_next, 0, 8, ctx->stream));
        FP_CUDA(ctx, cudaMemsetAsync(&ctx->d_sc->fb_count, 0, 8, ctx->stream));
        cudaEventRecord(e0, ctx->stream);
        plan_kernel_launch(ctx, A, smem, grid);
        FP_LAUNCHED(ctx);
        cudaEventRecord(e1, ctx->stream);
        FP_CUDA(ctx, cudaEventSynchronize(e1));
        float t = 0;
        cudaEventElapsedTime(&t, e0, e1);
        total += t;
    }
    // repeated launches marked the footprints many times: the next motion rebuilds its records
    ctx->rec_fresh = false;
    ctx->marks_dirty = true;
    // leave the state planned (the fallbacks of the last launch decided exactly)
    plan_exact_list_kernel<<<ctx->sm_count, EXACT_WARPS * 32, 0, ctx->stream>>>(A.c, ctx->d_fallback, emit_args(A));
    FP_LAUNCHED(ctx);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *ms = total / std::max(iters, 1);
    return FP_OK;
}

int fp_choice_launch(fp_ctx* ctx, uint32_t agent, double k_s, int32_t* d_cx, int32_t* d_cy, double* d_w,
                     float* d_p, uint32_t* d_n) {
    PlanCommon a = make_common(ctx, k_s, 0);
    const uint32_t* plane = nullptr;
    if (tiled_ok(ctx)) {
        if (int rc = fp_plan_prepare(ctx, k_s)) return rc;
        plane = ctx->d_plane;
    }
    choice_kernel<<<1, 1, 0, ctx->stream>>>(a, plane, ctx->PW, agent, d_cx, d_cy, d_w, d_p, d_n);
    FP_LAUNCHED(ctx);
    return FP_OK;
}

// choose_desired_cell(st, agent, params) for one agent given by value (planning.hpp:88-108).
int fp_choose_one_launch(fp_ctx* ctx, uint32_t id, int px, int py, int v, int64_t step, double k_s, uint64_t seed,
                         int32_t* d_out) {
    if (int rc = ensure_pathmasks(ctx)) return rc;
    PlanCommon a = make_common(ctx, k_s, seed);
    choose_one_kernel<<<1, 1, 0, ctx->stream>>>(a, id, px, py, v, (long long)step, d_out);
    FP_LAUNCHED(ctx);
    return FP_OK;
}

// enumerate_candidates(st, agent) for one agent given by value (planning.hpp:23-57).
int fp_candidates_one_launch(fp_ctx* ctx, int px, int py, int v, int32_t* d_cx, int32_t* d_cy, uint32_t* d_n) {
    PlanCommon a = make_common(ctx, 0.0, 0);
    candidates_one_kernel<<<1, 1, 0, ctx->stream>>>(a, px, py, v, d_cx, d_cy, d_n);
    FP_LAUNCHED(ctx);
    return FP_OK;
}
