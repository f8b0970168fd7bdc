// plan.cu -- the planning phase: choose_desired_cell for every alive agent.
//
// Reference: plan_phase (engine.hpp:71-84) -> choose_desired_cell (planning.hpp:88-108)
//            -> enumerate_candidates (planning.hpp:23-57), line_of_sight (world.hpp:181-191),
//               potential_drop (planning.hpp:76-80), std::exp, sample_index (:63-73).
//
// Production path (plan_stream_kernel): a persistent, warp-specialised CTA per SM.  A producer
// warp streams 8-row chunks of 240-column stripes of the weight plane (plane.cu, 4 B/cell), the
// occupancy and the wall bitplanes into a shared-memory ring with TMA (mbarrier completion),
// taking plan items (bucket.cu) from a global cursor; consumer warps plan one agent per lane as
// soon as the rows its ball spans have landed:
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

#include <vector>

#include "fp_exp.h"
#include "internal.cuh"
#include "motion_rec.cuh"

#define FP_GUARD 8e-7  // see the guard-band note above
#ifndef FP_PLAN_MARKS
#define FP_PLAN_MARKS 0  // 1: the plan marks footprints in P1/P2 and move.cu skips seed_mark_kernel
                         // (measured: plan kernel +84 us for the global fetch-ORs, motion -40 us)
#endif

// Walk records (motion_rec.cuh): the plan emits them for the motion phase.
__constant__ signed char c_bpath_p[121][5][2];

// Bresenham path masks over the 11x11 offset frame (bit (dy+5)*11 + dx+5): the cells strictly
// between (0,0) and (dx,dy) on the segment (world.hpp:143-167).  Built at compile time: the plan
// kernel's unrolled candidate loops fold them into instruction immediates (k_pathmask_dev); the
// runtime-indexed users read the constant-memory copy (c_pathmask) or a shared-memory one.
struct PathMasks {
    uint32_t m[121][4];
};
constexpr PathMasks make_pathmasks() {
    PathMasks P{};
    for (int dy = -5; dy <= 5; ++dy)
        for (int dx = -5; dx <= 5; ++dx) {
            const int adx = dx < 0 ? -dx : dx, sx = 0 < dx ? 1 : -1;
            const int ady = -(dy < 0 ? -dy : dy), sy = 0 < dy ? 1 : -1;
            int err = adx + ady, x = 0, y = 0;
            while (!(x == dx && y == dy)) {
                const int e2 = 2 * err;
                if (e2 >= ady) { err += ady; x += sx; }
                if (e2 <= adx) { err += adx; y += sy; }
                if (x == dx && y == dy) break;
                const int b = (y + 5) * 11 + x + 5;
                P.m[(dy + 5) * 11 + dx + 5][b >> 5] |= 1u << (b & 31);
            }
        }
    return P;
}
static constexpr PathMasks k_pathmask_host = make_pathmasks();
__device__ constexpr PathMasks k_pathmask_dev = make_pathmasks();
__constant__ uint32_t c_pathmask[121][4];
static bool g_pathmask_ready[64] = {false};

static void host_pathmasks(uint32_t out[121][4]) {
    for (int o = 0; o < 121; ++o)
        for (int j = 0; j < 4; ++j) out[o][j] = k_pathmask_host.m[o][j];
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
    FP_PDL_WAIT();
    int cx, cy;
    choose_exact_at(a, id, a.g.wrap(px), py, v, (uint64_t)step, &cx, &cy);
    out[0] = cx;
    out[1] = cy;
}

__global__ void candidates_one_kernel(PlanCommon a, int px, int py, int v, int32_t* cx, int32_t* cy, uint32_t* n_out) {
    FP_PDL_WAIT();
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
    FP_PDL_WAIT();
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.n || !a.alive[i]) return;
    int cx, cy;
    choose_exact(a, i, (uint64_t)a.sc->step, &cx, &cy);
    a.dx[i] = cx;
    a.dy[i] = cy;
}

// ------------------------------------------------------------------------------ fast weights
enum { MODE_EXIT = 0, MODE_ONES = 1, MODE_DRIVE = 2 };

// The agent's exponent offset A_p = ((C_p + 127) mod 256) << 23 from its own plane word
// (bits 30..23 hold (-C_p) mod 256, plane.cu).
__device__ __forceinline__ uint32_t plane_offset(uint32_t own) { return ((127u - (own >> 23)) & 255u) << 23; }

// Weight of a reachable candidate word relative to the agent (offset ap): m_c * 2^(C_p - C_c),
// an exact fp32 number (|C_p - C_c| <= 60 on cells the fast path plans, plane.cu).
__device__ __forceinline__ float plane_weight(uint32_t w, uint32_t ap) { return fabsf(__uint_as_float(w + ap)); }

// Weight of a non-wall candidate word, as an exact fp64 value (an fp32-precision weight).
__device__ __forceinline__ double fast_weight(uint32_t w, uint32_t ap, int mode, double drive_w, bool unreach) {
    if (mode == MODE_ONES) return 1.0;
    if (mode == MODE_DRIVE) return drive_w;
    if (unreach) return 0.0;
    return (double)plane_weight(w, ap);
}

__device__ __forceinline__ float drive_weight_f(double k_s, double g, int dx) {
    return (float)fpx_exp(FPX_MUL(k_s, FPX_MUL(g, (double)dx)));
}

// ------------------------------------------------------------------------------ stream kernel
// Ring of RING_SLOTS 8-row chunks of one stripe (tile_w columns + 8 each side): weight-plane
// words, occupancy bits and wall bits, staged by TMA.  Chunk k of the stripe lives in ring slot
// k % RING_SLOTS.
#ifndef PLAN_THREADS
#define PLAN_THREADS 512
#endif
#ifndef FP_PLAN_NAP_MAX
#define FP_PLAN_NAP_MAX 512  // ns, longest back-off of a waiting warp
#endif
#ifndef RING_SLOTS
#define RING_SLOTS 24
#endif
#define CHUNK_ROWS 8
#define OCCW 16  // bit words per staged row: 512 bits from a 16-byte aligned word

struct StreamArgs {
    PlanCommon c;
    const uint4* brec;          // (id, wrapped x, y, v_max) per bucket position (bucket.cu)
    const uint32_t* ccnt;       // agents per chunk
    const uint32_t* coff;       // first bucket position per chunk
    const uint4* items;         // plan items (bucket.cu), 4 x uint4 each: (first chunk, chunks - 1,
                                //   first agent, end agent), then u16 references per ring slot
    uint32_t nchunks;
    const uint8_t* tile_exit;   // an Exit within the tile's window
    int tile_w, tile_h, tiles_x, cps, boxw;
    uint2* fallback;            // (id, bucket position) handed to plan_exact_list_kernel
    uint4* rec0;                // walk records in bucket order (motion_rec.cuh)
    int mixed;                  // roster has more than one v_max: the masked radius-5 variant
    const uint32_t* plane_t;    // chunk-tiled weight plane (plane.cu plane_tile_kernel)
    uint32_t* p1;               // non-null: mark each mover's footprint in the motion's contention
    uint32_t* p2;               //   bitplanes as its record is emitted (mark_record, motion_rec.cuh)
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


// One contiguous run of global memory into shared memory (cp.async.bulk, mbarrier completion).
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int cx, int cy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(cx), "r"(cy)
        : "memory");
}

// The rows of one plan item staged in its half of the ring: item row 0 is grid row r0 =
// 8 * (first chunk - 1); row r of the grid is item row r - r0 (weight words, occupancy bits,
// wall bits), so a ball's rows are plain offsets from the agent's item row.
struct Ring {
    const uint32_t* w;
    const uint32_t* o;
    const uint32_t* l;
    int boxw;
    int r0;
    __device__ __forceinline__ const uint32_t* wrow(int r) const { return w + (r - r0) * boxw; }
    __device__ __forceinline__ const uint32_t* orow(int r) const { return o + (r - r0) * OCCW; }
    __device__ __forceinline__ const uint32_t* lrow(int r) const { return l + (r - r0) * OCCW; }
};

// Pair of u64 words holding the 121-bit ball wall mask (bit (dy+5)*11 + dx+5).
struct Mask121 {
    unsigned long long lo, hi;
};

// B: frame bit of the row's first cell (a constant once the row loop is unrolled)
__device__ __forceinline__ void mask_or_row(Mask121& m, uint32_t rowbits, int B) {
    if (B < 64) m.lo |= (unsigned long long)rowbits << B;
    if (B + 11 > 64) m.hi |= (B >= 64) ? ((unsigned long long)rowbits << (B - 64)) : ((unsigned long long)rowbits >> (64 - B));
}

// Path mask test for an offset o known at compile time (unrolled loops): immediates, no loads.
__device__ __forceinline__ bool path_blocked_c(const Mask121& m, int o) {
    const unsigned long long plo = ((unsigned long long)k_pathmask_dev.m[o][1] << 32) | k_pathmask_dev.m[o][0];
    const unsigned long long phi = ((unsigned long long)k_pathmask_dev.m[o][3] << 32) | k_pathmask_dev.m[o][2];
    return ((m.lo & plo) | (m.hi & phi)) != 0ull;
}

// Path mask test against the shared-memory copy of c_pathmask (lanes index it divergently).
__device__ __forceinline__ bool path_blocked_s(const uint4* pm, const Mask121& m, int o) {
    const uint4 q = pm[o];
    const unsigned long long plo = ((unsigned long long)q.y << 32) | q.x;
    const unsigned long long phi = ((unsigned long long)q.w << 32) | q.z;
    return ((m.lo & plo) | (m.hi & phi)) != 0ull;
}

// Pairwise fp32 sum of |x[0..N)| (depth ceil(log2 N): the error bound the guard band assumes;
// the |.| is an operand modifier of the adds, see plane_weight).
template <int N>
__device__ __forceinline__ float pairwise_sum(const float* x) {
    if constexpr (N == 1) {
        return fabsf(x[0]);
    } else {
        constexpr int H = (N + 1) / 2;
        return pairwise_sum<H>(x) + pairwise_sum<N - H>(x + H);
    }
}

// Bits [osh, osh + 32) of a staged bitplane row.
__device__ __forceinline__ uint32_t row_bits(const uint32_t* row, int osh) {
    return __funnelshift_r(row[osh >> 5], row[(osh >> 5) + 1], osh & 31);
}

// Plans one agent from the staged stripe (V = its v_max, DRIVE = DriveX potential).  Returns 1
// when the fast path decided (result in *ox, *oy), 2 when the exact path must decide.
//   walls   the ball's wall bits (staged wall bitplane, one word pair per row)
//   pass 1  rows centre-out: candidates (in the grid, not Wall, not occupied by another agent,
//           visible) contribute their exact fp32 weight -- one integer add on the plane word,
//           plane.cu -- to a pairwise fp32 row sum; the row sums are accumulated in fp64.
//           Unreachable free cells never reach this path: their word and every centre within
//           Chebyshev 5 of them carry the exact-path flag (plane.cu)
//   pass 2  u*total picks the row; the row is replayed in list order (wrapped-x sorted at a
//           periodic seam) to find the first cumulative weight > threshold; guard band.
// MASKED: one radius-V code path for every v_max <= V (mixed rosters): rows and columns beyond
// the agent's own radius vr are masked out, which leaves exactly its Chebyshev ball (the line
// of sight to a cell of the ball only crosses cells of the ball), so decisions are unchanged
// while the warps of a mixed roster share one instruction stream.
template <int V, bool DRIVE, bool MASKED = false>
__device__ __forceinline__ int plan_ring_t(const StreamArgs& A, const Ring& R, const uint4* pathm, int osh0, int X0,
                                           int px, int py, double u, const double* drive_tab, int* ox, int* oy,
                                           int vr = V) {
    constexpr int D = 2 * V + 1;
    const PlanCommon& a = A.c;
    uint32_t colmask = MASKED ? (((1u << (2 * vr + 1)) - 1u) << (V - vr)) : ((1u << D) - 1u);
    if (a.g.boundary != FP_BOUNDARY_PERIODIC_X) {  // columns outside [0, W) (planning.hpp:39-41)
        if (px < V) colmask &= ~0u << (V - px);
        if (px + V >= a.g.W) colmask &= (1u << (a.g.W - px + V)) - 1u;
    }
    const int lx = px - X0;
    const uint32_t own = R.wrow(py)[lx];
    if (own >> 31) return 2;  // flagged centre: unreachable pocket, steep field, unreachable neighbour
    const uint32_t ap = DRIVE ? 0u : plane_offset(own);
    const int osh = osh0 + lx - V;  // staged bitplane bit of dx = -V
    Mask121 wm{0ull, 0ull};
#pragma unroll
    for (int dy = -V; dy <= V; ++dy) {
        if ((unsigned)(py + dy) >= (unsigned)a.g.H) continue;
        const uint32_t wb = row_bits(R.lrow(py + dy), osh) & ((1u << D) - 1u);
        mask_or_row(wm, wb, (dy + 5) * 11 + 5 - V);
    }
    const bool anywall = (wm.lo | wm.hi) != 0ull;
    float dw[D];  // DriveX weights by column (exact fp32 values)
#pragma unroll
    for (int k = 0; k < D; ++k) dw[k] = DRIVE ? (float)drive_tab[k - V + 5] : 0.0f;
    float rso[D];
    Mask121 vm{0ull, 0ull};  // the candidates (in frame bits, like wm)
#pragma unroll
    for (int t = 0; t < D; ++t) {
        const int dy = (t & 1) ? -((t + 1) >> 1) : (t >> 1);  // centre-out: 0, -1, 1, -2, 2, ...
        const bool rowok = (unsigned)(py + dy) < (unsigned)a.g.H;
        const uint32_t* row = R.wrow(py + dy) + lx - V;
        uint32_t occ = row_bits(R.orow(py + dy), osh) | row_bits(R.lrow(py + dy), osh);
        if (dy == 0) occ &= ~(1u << V);  // the own cell stays a candidate (planning.hpp:45-46)
        const bool inball = !MASKED || (dy <= vr && -dy <= vr);
        uint32_t valid = (rowok && inball) ? (~occ & colmask) : 0u;
        if (anywall) {
#pragma unroll
            for (int k = 0; k < D; ++k)
                if (path_blocked_c(wm, (dy + 5) * 11 + k - V + 5)) valid &= ~(1u << k);
        }
        mask_or_row(vm, valid, (dy + 5) * 11 + 5 - V);  // kept for the row replay
        float w[D];
#pragma unroll
        for (int k = 0; k < D; ++k) {
            if (DRIVE) w[k] = ((valid >> k) & 1u) ? dw[k] : 0.0f;
            else w[k] = __uint_as_float(((valid >> k) & 1u) ? row[k] + ap : 0u);
        }
        rso[t] = pairwise_sum<D>(w);
    }
    double rs[D];  // row sums, indexed by dy + V
#pragma unroll
    for (int k = 0; k < D; ++k) {
        const int dy = k - V;
        rs[k] = (double)rso[dy >= 0 ? 2 * dy : -2 * dy - 1];
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
    const uint32_t* row = R.wrow(py + dy) + lx;
    uint32_t valid;  // the row's candidates, bit dx + V (pass 1's masks)
    {
        const int b = (dy + 5) * 11 + 5 - V;
        const unsigned long long w64 = b < 64 ? ((vm.lo >> b) | (b ? (vm.hi << (64 - b)) : 0ull)) : (vm.hi >> (b - 64));
        valid = (uint32_t)w64 & ((1u << D) - 1u);
    }
    const int Rr = MASKED ? vr : V;  // the agent's radius
    int a0 = -Rr, a1 = Rr, b0 = 0, b1 = -1;
    if (a.g.boundary == FP_BOUNDARY_PERIODIC_X) {  // wrapped-x order at the seam (planning.hpp:50-53)
        if (px + Rr >= a.g.W) {
            a0 = a.g.W - px; b0 = -Rr; b1 = a.g.W - px - 1;
        } else if (px - Rr < 0) {
            a0 = -px; b0 = -Rr; b1 = -px - 1;
        }
    }
    double prefix = before, lower = 0.0, upper = 0.0;
    int kx = 0;
    bool found = false;
    if (b1 < b0) {  // no seam: list order is dx ascending -- one branch-free pass over the row
#pragma unroll
        for (int k = 0; k < D; ++k) {
            const bool ok = (valid >> k) & 1u;
            const double wk = DRIVE ? drive_tab[k - V + 5] : (double)plane_weight(row[k - V], ap);
            const double next = prefix + (ok ? wk : 0.0);
            const bool hit = ok && !found && next > theta;
            lower = hit ? prefix : lower;
            upper = hit ? next : upper;
            kx = hit ? k - V : kx;
            found = found || hit;
            prefix = next;
        }
    } else for (int seg = 0; seg < 2 && !found; ++seg) {
        const int lo = seg ? b0 : a0, hi = seg ? b1 : a1;
        for (int dx = lo; dx <= hi; ++dx) {
            if (!((valid >> (dx + V)) & 1u)) continue;  // outside the grid, Wall, occupied, hidden
            const double wt = DRIVE ? drive_tab[dx + 5] : (double)plane_weight(row[dx], ap);
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
    return anywall ? 5 : 1;  // bit 2: the ball holds a Wall (record_of_ring walks the path)
}

// record_of (motion_rec.cuh) for a fast-path decision inside the staged stripe: the target lies in
// the ball, the Wall test reads the staged wall bits, and the Exit test (global bitplane) runs
// only in tiles whose window holds an Exit.
__device__ __forceinline__ uint4 record_of_ring(const Geo& g, const uint32_t* occ, bool tile_exit, bool ball_wall,
                                                const Ring& R,
                                                int lbit, uint32_t id, int sx, int sy, int tx, int ty, int v,
                                                const signed char (*bp)[5][2]) {
    const int ddx = g.segment_dx(sx, tx), ddy = ty - sy;
    const int o = (ddy + 5) * 11 + ddx + 5;
    const int len = min(max(abs(ddx), abs(ddy)), v);
    int m = 0, ex_x = 0, ex_y = 0;
    bool ex = false;
    if (!ball_wall && !tile_exit) m = len;  // nothing on the path can stop the walk early
    else for (int j = 0; j < len; ++j) {
        const int ox = bp[o][j][0], oy = bp[o][j][1];
        const int b = lbit + ox;
        if ((R.lrow(sy + oy)[b >> 5] >> (b & 31)) & 1u) break;  // Wall
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

template <bool DRIVE>
__device__ __forceinline__ int plan_ring_v(int v, const StreamArgs& A, const Ring& R, const uint4* pathm, int osh0,
                                           int X0, int px, int py, double u, const double* drive_tab, int* ox,
                                           int* oy) {
#define FP_PLAN_ARGS A, R, pathm, osh0, X0, px, py, u, drive_tab, ox, oy
#ifdef FP_PLAN_ONLY_V4  // SASS inspection builds: one instantiation
    return plan_ring_t<4, DRIVE>(FP_PLAN_ARGS);
#endif
    if (A.mixed)  // one instruction stream for a mixed-v roster (see plan_ring_t)
        return plan_ring_t<5, DRIVE, true>(FP_PLAN_ARGS, v);
    switch (v) {
        case 1: return plan_ring_t<1, DRIVE>(FP_PLAN_ARGS);
        case 2: return plan_ring_t<2, DRIVE>(FP_PLAN_ARGS);
        case 3: return plan_ring_t<3, DRIVE>(FP_PLAN_ARGS);
        case 4: return plan_ring_t<4, DRIVE>(FP_PLAN_ARGS);
        default: return plan_ring_t<5, DRIVE>(FP_PLAN_ARGS);
    }
#undef FP_PLAN_ARGS
}

__device__ __forceinline__ unsigned long long globaltimer_p() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Persistent CTA per SM, warp-specialised, dynamically scheduled.  Work units are plan items
// (bucket.cu plan_items_kernel): up to PLAN_ITEM_CHUNKS consecutive chunks of one stripe and at
// most PLAN_ITEM_AGENTS of their agents, taken from a global cursor (d_sc->tile_next) so crowded
// and empty parts of the grid balance across the SMs.
//   producer (warp 0): takes an item; it occupies the next nk + 2 ring slots (chunks kf-1 ..
//     kl+1 of its stripe, kept in the ring in order); lane i looks after the item's slot i: it
//     waits for the slot's previous rows to be released (reference count 0), reloads it by TMA
//     (weight words, occupancy and wall bits; one full mbarrier per slot) and adds the item's
//     references.  Lane 0 appends the item's agent run to the CTA's queue and publishes it.
//   consumers (the other warps): claim 32 virtual agents at a time, plan each once it is
//     published and the (at most three) slots its ball spans have landed, one agent per lane,
//     then release those slots.
// The ring holds RING_PARTS items, so the TMA of the next items overlaps the planning of the
// current one; an item is published before its part drains, so its agents are claimed early.
#ifndef PLAN_MIN_CLAIM
#define PLAN_MIN_CLAIM 32 // smallest claim of a consumer warp (agents)
#endif
#define PLAN_CONSUMERS (PLAN_THREADS / 32 - 1)
#define PLAN_QUEUE 64  // published items a CTA remembers (the ring bounds the ones in flight)
#ifndef RING_PARTS
#define RING_PARTS 3  // items in flight per CTA (the ring's parts)
#endif
#define RING_HALF (RING_SLOTS / RING_PARTS)  // slots per item (>= PLAN_ITEM_CHUNKS + 2, bucket.cu)

// KV = 0: any roster and potential (runtime dispatch over v_max and the potential); KV = 1..5:
// one code path for a uniform-v_max roster (KMIXED: the masked radius-5 path of a mixed roster)
// and one potential -- a smaller kernel body for the instruction cache.
template <int KV, bool KDRIVE, bool KMIXED>
__global__ void __launch_bounds__(PLAN_THREADS, 1) plan_stream_kernel(const __grid_constant__ CUtensorMap tmap_w,
                                                                      const __grid_constant__ CUtensorMap tmap_o,
                                                                      const __grid_constant__ CUtensorMap tmap_l,
                                                                      StreamArgs A) {
    FP_PDL_WAIT();
    extern __shared__ __align__(128) uint32_t smem_raw[];
    uint32_t* ringw = smem_raw + (((128u - (smem_u32(smem_raw) & 127u)) & 127u) >> 2);
    uint32_t* ringo = ringw + RING_SLOTS * CHUNK_ROWS * A.boxw;
    uint32_t* ringl = ringo + RING_SLOTS * CHUNK_ROWS * OCCW;
    uint64_t* bars = reinterpret_cast<uint64_t*>(ringl + RING_SLOTS * CHUNK_ROWS * OCCW);
    __shared__ volatile int s_gen[RING_SLOTS];
    __shared__ int s_ref[RING_SLOTS];
    __shared__ unsigned s_qv[PLAN_QUEUE];      // published item q: first virtual agent index
    __shared__ unsigned s_qa[PLAN_QUEUE];      //   its first bucket position
    __shared__ int s_qs[PLAN_QUEUE];           //   its ring part | first chunk << 2
    __shared__ int s_qx[PLAN_QUEUE];           //   its stripe
    __shared__ unsigned s_qp[PLAN_QUEUE];      //   barrier parity per slot of its part (bit i: slot i)
    __shared__ unsigned s_next;                // consumers' claim cursor (virtual agents)
    __shared__ volatile unsigned s_qcur;       // queue entry of a recent claim (search hint)
    __shared__ volatile unsigned s_pub;        // virtual agents published
    __shared__ volatile unsigned s_nq;         // queue entries published
    __shared__ volatile int s_done;            // producer finished
    __shared__ double s_drive[11];
    __shared__ signed char s_bp[121][5][2];
    __shared__ uint4 s_pathm[121];
    for (int k = threadIdx.x; k < 121 * 10; k += blockDim.x) (&s_bp[0][0][0])[k] = (&c_bpath_p[0][0][0])[k];
    for (int k = threadIdx.x; k < 121; k += blockDim.x)
        s_pathm[k] = make_uint4(c_pathmask[k][0], c_pathmask[k][1], c_pathmask[k][2], c_pathmask[k][3]);
    const PlanCommon& a = A.c;
    if (threadIdx.x < 11) {
        s_drive[threadIdx.x] = (a.potential == FP_POTENTIAL_DRIVE_X)
                                   ? (double)drive_weight_f(a.k_s, a.drive_gradient, (int)threadIdx.x - 5)
                                   : 0.0;
    }
    if (threadIdx.x < RING_SLOTS) {
        s_gen[threadIdx.x] = 0;
        s_ref[threadIdx.x] = 0;
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < RING_SLOTS; ++s) mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        s_next = 0;
        s_qcur = 0;
        s_pub = 0;
        s_done = 0;
        s_nq = 0;
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rows_chunks = (a.g.H + CHUNK_ROWS - 1) / CHUNK_ROWS;  // chunks with rows in the grid
    const unsigned tx_bytes = (unsigned)(CHUNK_ROWS * (A.boxw + 2 * OCCW)) * 4u;
    const uint32_t n_items = (uint32_t)a.sc->n_plan_items;
    if (warp == 0) {
        // ---------------- producer
        bool ok = true;
        unsigned pub = 0, nq = 0;
        int half = 0;  // ring part of the next item (items take the parts in turn)
        // Items flow through a two-stage pipeline so no global-memory latency sits between two
        // items: while item j stages, item j+1's record (descriptor + per-slot reference counts,
        // bucket.cu) is in flight and item j+2's index is being claimed.
        const uint16_t* refs_base = reinterpret_cast<const uint16_t*>(A.items);
        auto load_rec = [&](uint32_t i, uint4& d, uint32_t& r) {
            if (i < n_items) {
                d = __ldg(&A.items[4 * (size_t)i]);
                r = (lane < 24) ? __ldg(&refs_base[32 * (size_t)i + 8 + lane]) : 0u;
            }
        };
        uint32_t claim_b = 0;  // lane 0: index of the item after next (atomic in flight)
        uint32_t i_cur = 0;
        if (lane == 0) {
            i_cur = (uint32_t)atomicAdd(&a.sc->tile_next, 1ull);
            claim_b = (uint32_t)atomicAdd(&a.sc->tile_next, 1ull);
        }
        i_cur = __shfl_sync(0xffffffffu, i_cur, 0);
        uint4 d_cur = make_uint4(0, 0, 0, 0);
        uint32_t r_cur = 0;
        load_rec(i_cur, d_cur, r_cur);
        while (ok) {
            const uint32_t i = i_cur;
            if (i >= n_items) break;
            const uint32_t i_nx = __shfl_sync(0xffffffffu, claim_b, 0);
            if (lane == 0) claim_b = (uint32_t)atomicAdd(&a.sc->tile_next, 1ull);
            uint4 d_nx = make_uint4(0, 0, 0, 0);
            uint32_t r_nx = 0;
            load_rec(i_nx, d_nx, r_nx);
            const uint4 it = d_cur;
            const uint32_t refs = r_cur;  // agents of the item whose ball reaches slot kk
            i_cur = i_nx;
            d_cur = d_nx;
            r_cur = r_nx;
            const uint32_t gf = it.x;
            const int nk = (int)it.y + 1;
            const uint32_t a0 = it.z, a1 = it.w;
            const int s = (int)(gf / (uint32_t)A.cps), kf = (int)(gf % (uint32_t)A.cps);
            const int kk = kf - 1 + lane;  // the slot this lane looks after
            const int p = half * RING_HALF + lane;
            const bool mine = lane < nk + 2 && refs != 0 && kk >= 0 && kk < rows_chunks;
            // Publish first: consumers claim the item's agents (and load their records) while its
            // part drains and its rows stream in; they wait for the rows on the slot barriers.
            // Slot p has had s_gen[p] loads, so this one completes phase s_gen[p]: parity bit.
            const unsigned pbits = __ballot_sync(0xffffffffu, mine && (s_gen[p] & 1));
            if (lane == 0) {
                s_qv[nq % PLAN_QUEUE] = pub;
                s_qa[nq % PLAN_QUEUE] = a0;
                s_qs[nq % PLAN_QUEUE] = half | (kf << 2);
                s_qx[nq % PLAN_QUEUE] = s;
                s_qp[nq % PLAN_QUEUE] = pbits;
                ++nq;
                pub += a1 - a0;
                __threadfence_block();
                s_nq = nq;
                __threadfence_block();
                s_pub = pub;
            }
            if (mine) {
                unsigned nap = 32;
                for (long long spin = 0; *((volatile int*)&s_ref[p]) != 0; ++spin) {
                    __nanosleep(nap);
                    nap = min(nap * 2u, (unsigned)FP_PLAN_NAP_MAX);
                    if (spin > (1ll << 24)) {
                        atomicOr(&a.sc->err, 4ull);
                        ok = false;
                        break;
                    }
                }
                if (ok) {
                    s_gen[p] = s_gen[p] + 1;
                    const int x0 = s * A.tile_w;
                    const int gws = ((x0 - 8 + FP_XPAD_BITS) >> 5) & ~3;
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    mbar_expect_tx(&bars[p], tx_bytes);
                    bulk_load(ringw + p * CHUNK_ROWS * A.boxw,
                              A.plane_t + ((size_t)s * rows_chunks + kk) * (CHUNK_ROWS * A.boxw),
                              (unsigned)(CHUNK_ROWS * A.boxw) * 4u, &bars[p]);
                    tma_load_2d(ringo + p * CHUNK_ROWS * OCCW, &tmap_o, &bars[p], gws, kk * CHUNK_ROWS);
                    tma_load_2d(ringl + p * CHUNK_ROWS * OCCW, &tmap_l, &bars[p], gws, kk * CHUNK_ROWS);
                    atomicAdd(&s_ref[p], (int)refs);
                }
            }
            ok = __all_sync(0xffffffffu, ok);
            half = half + 1 == RING_PARTS ? 0 : half + 1;
        }
        if (lane == 0) {
            __threadfence_block();
            s_done = 1;
        }
        return;
    }
    // ---------------- consumers
    // A warp claims up to 32 consecutive agents of ONE published item (compare-and-swap on the
    // claim cursor, bounded by the item's end and the published count), so every claim is planned
    // in one pass with the item's staging parameters uniform across the warp.
    const uint64_t step = (uint64_t)a.sc->step;
    unsigned qhint = 0;  // queue entry of this warp's last claim (claims only move forward)
    for (;;) {
        unsigned g = 0, k = 0, q = 0;
        int bad = 0;
        if (lane == 0) {
            unsigned nap = 32;
            for (long long spin = 0;; ++spin) {
                // order: done, then pub, then nq (the producer writes them in reverse)
                const int done = s_done;
                __threadfence_block();
                const unsigned pub = s_pub;
                __threadfence_block();
                const unsigned nq = s_nq;
                g = *((volatile unsigned*)&s_next);
                if (g < pub) {
                    // s_qcur: the entry of some earlier claim (a lower bound for g's entry)
                    q = max(max(qhint, *((volatile unsigned*)&s_qcur)), nq > PLAN_QUEUE ? nq - PLAN_QUEUE : 0u);
                    while (q + 1 < nq && s_qv[(q + 1) % PLAN_QUEUE] <= g) ++q;
                    const unsigned beg = s_qv[q % PLAN_QUEUE];
                    const unsigned end = (q + 1 < nq) ? s_qv[(q + 1) % PLAN_QUEUE] : pub;
                    // sparse items are spread over more warps (shorter claims, more in flight)
                    const unsigned share = (end - beg + PLAN_CONSUMERS - 1) / PLAN_CONSUMERS;
                    k = min(min(32u, max((unsigned)PLAN_MIN_CLAIM, share)), end - g);
                    if (atomicCAS(&s_next, g, g + k) == g) {
                        s_qcur = q;
                        break;
                    }
                    k = 0;
                    continue;  // another warp claimed first: retry at once
                }
                if (done) break;  // k = 0: everything published was claimed
                __nanosleep(nap);  // backoff: idle warps must not steal issue slots
                nap = min(nap * 2u, (unsigned)FP_PLAN_NAP_MAX);
                if (spin > (1ll << 24)) {
                    bad = 1;
                    break;
                }
            }
        }
        if (__shfl_sync(0xffffffffu, bad, 0)) {
            if (lane == 0) atomicOr(&a.sc->err, 8ull);
            return;
        }
        k = __shfl_sync(0xffffffffu, k, 0);
        if (k == 0) return;
        g = __shfl_sync(0xffffffffu, g, 0);
        q = __shfl_sync(0xffffffffu, q, 0);
        qhint = q;
        __threadfence_block();
        const unsigned qi = q % PLAN_QUEUE;
        const int qs = s_qs[qi], ihalf = qs & 3, kf = qs >> 2;
        const unsigned qpar = s_qp[qi];
        const int sbase = ihalf * RING_HALF - (kf - 1);  // ring slot of chunk 0 of the item (may be < 0)
        const int s = s_qx[qi];                          // the item's stripe (= px / tile_w)
        const Ring R{ringw + ihalf * RING_HALF * CHUNK_ROWS * A.boxw, ringo + ihalf * RING_HALF * CHUNK_ROWS * OCCW,
                     ringl + ihalf * RING_HALF * CHUNK_ROWS * OCCW, A.boxw, CHUNK_ROWS * (kf - 1)};
        const int x0 = s * A.tile_w;
        const int X0 = x0 - 8;  // staged column 0 (TMA inner coordinates stay 16-byte aligned)
        const int gws = ((x0 - 8 + FP_XPAD_BITS) >> 5) & ~3;
        const int osh0 = x0 - 8 + FP_XPAD_BITS - gws * 32;  // staged bit of column X0
        int k_lo = 0, k_hi = -1;
        if ((unsigned)lane < k) {
            const unsigned pos = s_qa[qi] + (g + lane - s_qv[qi]);
            const uint4 br = __ldcg(&A.brec[pos]);  // (id, wrapped x, y, v_max), bucket.cu
            const uint32_t id = br.x;
            const int px = (int)br.y, py = (int)br.z, v = (int)br.w;
            const int kc = py >> 3;
            k_lo = max(kc - 1, 0);
            k_hi = min(kc + 1, rows_chunks - 1);
            bool ready = true;
            for (int kk = k_lo; kk <= k_hi; ++kk) ready &= mbar_wait(&bars[sbase + kk], (qpar >> (kk - (kf - 1))) & 1u);
            if (!ready) atomicOr(&a.sc->err, 2ull);
            const double u = fp_unit_interval(fp_rng_u64(a.seed, id, step, 0));
            int cx = 0, cy = 0;
#ifdef FP_PLAN_NOCOMPUTE  // A/B experiments only: the staging pipeline without the planning work
            const int st = (u < 0.0) ? 1 : 3;
#else
            int st;
            if constexpr (KV > 0)
                st = plan_ring_t<KV, KDRIVE, KMIXED>(A, R, s_pathm, osh0, X0, px, py, u, s_drive, &cx, &cy, v);
            else
                st = (a.potential == FP_POTENTIAL_DRIVE_X)
                         ? plan_ring_v<true>(v, A, R, s_pathm, osh0, X0, px, py, u, s_drive, &cx, &cy)
                         : plan_ring_v<false>(v, A, R, s_pathm, osh0, X0, px, py, u, s_drive, &cx, &cy);
#endif
            if ((st & 3) == 1) {
                a.dx[id] = cx;
                a.dy[id] = cy;
                const int tile = (py / A.tile_h) * A.tiles_x + s;
                const uint4 rec = record_of_ring(a.g, a.occ, A.tile_exit[tile], st & 4, R, osh0 + px - X0, id, px,
                                                 py, cx, cy, v, s_bp);
                A.rec0[pos] = rec;
                if (A.p1 && rec_m(rec)) mark_record(A.p1, A.p2, a.g, rec, s_bp, cx, cy);
            } else if (st == 2) {  // decided by the exact path after the sweep (plan_exact_list_kernel)
                A.fallback[atomicAdd(&a.sc->fb_count, 1ull)] = make_uint2(id, pos);
            }
        }
        // release: the lanes' reads of the slots happen before their references drop; lanes
        // on the same slot combine their decrements (one shared atomic per slot and warp)
        __syncwarp();
        __threadfence_block();
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            const int kk = k_lo + d;
            const bool has = kk <= k_hi;
            const int key = has ? (sbase + kk) : -1;
            const unsigned peers = __match_any_sync(0xffffffffu, key);
            if (has && (__ffs(peers) - 1) == lane) atomicSub(&s_ref[key], __popc(peers));
        }
    }
}

// The exact path for the agents the tiled kernel could not decide: one CTA per agent, one thread
// per candidate slot of the ball in list order (row-major, wrapped-x sorted at the seam): each
// tests its cell against the global bitplanes (walls, occupancy, Bresenham line of sight) and
// computes the exact weight (restated glibc exp) in parallel; thread 0 then folds the weights
// serially in list order (sample_index, planning.hpp:63-73).  Narrow periodic grids
// (2v+1 >= W) use choose_exact.
#define EXACT_THREADS 128  // >= 121 candidate slots (v_max <= 5)
struct EmitArgs {
    uint4* rec0;
    uint32_t* p1;
    uint32_t* p2;
    int emit;
};

__device__ __forceinline__ void emit_record(const PlanCommon& a, const EmitArgs& E, uint32_t id, uint32_t pos, int px,
                                            int py, int cx, int cy, int v) {
    if (!E.emit) return;
    const uint4 rec = record_of(a.g, a.occ, id, px, py, cx, cy, v, c_bpath_p);
    E.rec0[pos] = rec;
    if (E.p1 && rec_m(rec)) mark_record(E.p1, E.p2, a.g, rec, c_bpath_p, cx, cy);
}

// 11 bits of a global bitplane row: columns x0 .. x0 + 10 (ghost columns at the edges).
__device__ __forceinline__ uint32_t bits11(const uint32_t* plane, const Geo& g, int x0, int y) {
    const int b = x0 + FP_XPAD_BITS;
    const size_t w = (size_t)y * g.P + (size_t)(b >> 5);
    return __funnelshift_r(__ldg(&plane[w]), __ldg(&plane[w + 1]), b & 31) & 0x7FFu;
}

__global__ void __launch_bounds__(EXACT_THREADS) plan_exact_list_kernel(PlanCommon a, const uint2* list,
                                                                        EmitArgs E) {
    FP_PDL_WAIT();
    __shared__ double s_w[EXACT_THREADS];
    __shared__ int s_c[EXACT_THREADS];
    __shared__ uint32_t s_wr[11], s_er[11];  // the ball's wall / exit bits (frame rows and columns -5..5)
    __shared__ int s_last;                    // the last candidate slot in list order
    const unsigned n = (unsigned)a.sc->fb_count;
    const int t = threadIdx.x;
    const uint64_t step = (uint64_t)a.sc->step;
    const Geo& g = a.g;
    for (unsigned e = blockIdx.x; e < n; e += gridDim.x) {
        const uint2 ent = list[e];
        const uint32_t id = ent.x;
        const int px = g.wrap(a.x[id]), py = a.y[id], v = a.v[id];
        const int D = 2 * v + 1;  // (2v+1 < W: the tiled path runs on periodic grids of W >= 16)
        // every load of the agent in one round: the ball's wall / exit rows, and per candidate
        // slot its occupancy word and field value
        if (t < 11) {
            const int y = py - 5 + t;
            const bool in = y >= 0 && y < g.H;
            s_wr[t] = in ? bits11(g.wall, g, px - 5, y) : 0u;
            s_er[t] = in ? bits11(g.exitb, g, px - 5, y) : 0u;
        }
        if (t == 0) s_last = -1;
        // list-order column -> dx (wrapped-x sort at the periodic seam, planning.hpp:50-53)
        int a0 = -v, na = D, b0 = 0;
        if (g.boundary == FP_BOUNDARY_PERIODIC_X) {
            if (px + v >= g.W) {
                a0 = g.W - px; na = v - a0 + 1; b0 = -v;
            } else if (px - v < 0) {
                a0 = -px; na = v - a0 + 1; b0 = -v;
            }
        }
        const ExactWeight wf = make_weight(a, px, py);
        bool ok = false;
        int x = 0, y = 0, dx = 0, dy = 0;
        double sc = 0.0;
        uint32_t occw = 0;
        if (t < D * D) {
            const int r = t / D, c = t % D;
            dy = r - v;
            y = py + dy;
            dx = c < na ? a0 + c : b0 + (c - na);
            x = px + dx;
            ok = y >= 0 && y < g.H;
            if (g.boundary == FP_BOUNDARY_PERIODIC_X) x = g.wrap(x);
            else ok = ok && x >= 0 && x < g.W;
            if (ok) {
                occw = __ldg(&a.occ[g.word(x, y)]);
                if (wf.exitd && !wf.ones) sc = __ldg(&a.field[(size_t)y * g.W + x]);
            }
        }
        __syncthreads();
        if (t < D * D) {
            if (ok) {
                const bool wall = (s_wr[dy + 5] >> (dx + 5)) & 1u;
                const bool occ = (occw >> (x & 31)) & 1u;
                ok = !wall && !(occ && !(x == px && y == py));
            }
            if (ok) {  // line of sight (world.hpp:181-191): no Wall strictly between (walls inside the ball)
                Mask121 wm{0ull, 0ull};
#pragma unroll
                for (int rr = 0; rr < 11; ++rr) mask_or_row(wm, s_wr[rr], rr * 11);
                const int o = (dy + 5) * 11 + dx + 5;
                const unsigned long long plo = ((unsigned long long)c_pathmask[o][1] << 32) | c_pathmask[o][0];
                const unsigned long long phi = ((unsigned long long)c_pathmask[o][3] << 32) | c_pathmask[o][2];
                ok = ((wm.lo & plo) | (wm.hi & phi)) == 0ull;
            }
            double wt = 0.0;
            if (ok) {
                if (wf.ones) wt = 1.0;
                else if (wf.exitd) wt = isinf(sc) ? 0.0 : fpx_exp(FPX_MUL(wf.k_s, FPX_SUB(wf.sp, sc)));
                else wt = fpx_exp(FPX_MUL(wf.k_s, FPX_MUL(wf.g, (double)g.segment_dx(px, x))));
            }
            // non-candidates add +0.0: the serial sums keep every intermediate value, and the
            // running sum can only cross the threshold at a candidate
            s_w[t] = ok ? wt : 0.0;
            s_c[t] = ok ? (y * g.W + x) : -1;
            if (ok) atomicMax(&s_last, t);
        }
        __syncthreads();
        if (t == 0) {
            double total = 0.0;
#pragma unroll 8
            for (int k = 0; k < D * D; ++k) total = FPX_ADD(total, s_w[k]);  // loads off the add chain
            const int last = s_last;
            const double threshold = FPX_MUL(fp_unit_interval(fp_rng_u64(a.seed, id, step, 0)), total);
            double cum = 0.0;
            int pick = last;
#pragma unroll 4
            for (int k = 0; k < D * D; ++k) {
                cum = FPX_ADD(cum, s_w[k]);
                if (cum > threshold) {
                    pick = k;
                    break;
                }
            }
            const int cell = s_c[pick];
            const int cx = cell % g.W, cy = cell / g.W;
            a.dx[id] = cx;
            a.dy[id] = cy;
            if (E.emit) {  // record_of (motion_rec.cuh) from the staged rows
                const int ddx = g.segment_dx(px, cx), ddy = cy - py;
                const int o = (ddy + 5) * 11 + ddx + 5;
                const int len = min(max(abs(ddx), abs(ddy)), v);
                int m = 0, ex_x = 0, ex_y = 0;
                bool ex = false;
                for (int j = 0; j < len; ++j) {
                    const int ox = c_bpath_p[o][j][0], oy = c_bpath_p[o][j][1];
                    if ((s_wr[oy + 5] >> (ox + 5)) & 1u) break;
                    ++m;
                    if ((s_er[oy + 5] >> (ox + 5)) & 1u) {
                        ex = true;
                        ex_x = g.wrap(px + ox);
                        ex_y = py + oy;
                        break;
                    }
                }
                const bool exit_free = ex && !((__ldcg(&a.occ[g.word(ex_x, ex_y)]) >> (ex_x & 31)) & 1u);
                const uint4 rec = make_uint4(id, 0u,
                                             (uint32_t)px | (exit_free ? REC_EXIT_FREE : 0u) | ((uint32_t)m << 28) |
                                                 (ex ? 0x80000000u : 0u),
                                             (uint32_t)py | ((uint32_t)o << 24));
                E.rec0[ent.y] = rec;
                if (E.p1 && rec_m(rec)) mark_record(E.p1, E.p2, g, rec, c_bpath_p, cx, cy);
            }
        }
        __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) a.sc->fallbacks += n;
}

// Test mode (fp_get_choice): candidates in list order, exact weights and the production
// path's choice probabilities (fast weights / fast total, fp32).
__global__ void choice_kernel(PlanCommon a, const uint32_t* plane, int PW, uint32_t i, int32_t* cx, int32_t* cy,
                              double* w, float* p, uint32_t* n_out) {
    FP_PDL_WAIT();
    const int px = a.g.wrap(a.x[i]);
    const int py = a.y[i];
    const ExactWeight wf = make_weight(a, px, py);
    const uint32_t own = plane ? plane[(size_t)py * PW + px + FP_XPAD_W] : 0u;
    int mode = MODE_EXIT;
    if (a.potential == FP_POTENTIAL_DRIVE_X) mode = MODE_DRIVE;
    else if (wf.ones) mode = MODE_ONES;
    const uint32_t ap = plane_offset(own);
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
            fw = fast_weight(word, ap, mode, (double)drive_weight_f(a.k_s, a.drive_gradient, dxs),
                             mode == MODE_EXIT && isinf(a.field[(size_t)y * a.g.W + x]));
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
    fp_launch(plan_exact_kernel, fp_blocks(ctx->n, 128), 128, 0, ctx->stream, a);
    FP_LAUNCHED(ctx);
    return FP_OK;
}

static size_t stream_smem(const fp_ctx* ctx) {
    const size_t boxw = (size_t)ctx->tile_w + 16;
    return (size_t)RING_SLOTS * CHUNK_ROWS * (boxw + 2 * OCCW) * 4 + 8 * RING_SLOTS /* barriers */ +
           128 /* alignment slack */;
}

static bool plan_marks(const fp_ctx* ctx);

static StreamArgs make_stream_args(fp_ctx* ctx, double k_s, uint64_t seed) {
    StreamArgs A;
    A.c = make_common(ctx, k_s, seed);
    A.brec = ctx->d_brec;
    A.ccnt = ctx->d_sub_cnt;
    A.coff = ctx->d_sub_off;
    A.items = ctx->d_plan_items;
    A.nchunks = fp_plan_chunks(ctx);
    A.tile_exit = ctx->d_tile_exit;
    A.tile_w = ctx->tile_w;
    A.tile_h = ctx->tile_h;
    A.tiles_x = ctx->tiles_x;
    A.cps = ctx->cps;
    A.boxw = ctx->tile_w + 16;
    A.fallback = ctx->d_fallback;
    A.rec0 = ctx->d_rec0;
    A.mixed = ctx->mixed_v ? 1 : 0;
    A.plane_t = ctx->d_plane_t;
    A.p1 = plan_marks(ctx) ? ctx->d_p1 : nullptr;
    A.p2 = plan_marks(ctx) ? ctx->d_p2 : nullptr;
    return A;
}

// The plan marks the movers' footprints itself (the motion then skips its marking pass) on
// single-GPU contexts; strip ranks mark after the deferral (strip.cu).
static bool plan_marks(const fp_ctx* ctx) { return FP_PLAN_MARKS && !ctx->st.on; }

static EmitArgs emit_args(fp_ctx* ctx) {
    const bool mk = plan_marks(ctx);
    return EmitArgs{ctx->d_rec0, mk ? ctx->d_p1 : nullptr, mk ? ctx->d_p2 : nullptr, 1};
}

#define FP_STREAM_VARIANTS(X)                                                                                \
    X(0, false, false) X(1, false, false) X(2, false, false) X(3, false, false) X(4, false, false)        \
    X(5, false, false) X(1, true, false) X(2, true, false) X(3, true, false) X(4, true, false)              \
    X(5, true, false) X(5, false, true) X(5, true, true)

static std::vector<const void*> stream_kernels() {
    std::vector<const void*> v;
#define FP_SK(V, D, M) v.push_back((const void*)plan_stream_kernel<V, D, M>);
    FP_STREAM_VARIANTS(FP_SK)
#undef FP_SK
    return v;
}

// The plan kernel variant for this context's roster and potential (plan_stream_kernel).
static void launch_stream_kernel(fp_ctx* ctx, const StreamArgs& A) {
    const bool drive = ctx->potential == FP_POTENTIAL_DRIVE_X;
    const int v = ctx->mixed_v ? 5 : ctx->v_uniform;
    const bool mixed = ctx->mixed_v;
#define FP_SK(V, D, M)                                                                                         \
    if (V > 0 && v == V && drive == D && mixed == M) {                                                         \
        fp_launch(plan_stream_kernel<V, D, M>, ctx->sm_count, PLAN_THREADS, stream_smem(ctx), ctx->stream,            \
            ctx->tmap_plane, ctx->tmap_occ, ctx->tmap_wall, A);                                                \
        return;                                                                                                \
    }
    FP_STREAM_VARIANTS(FP_SK)
#undef FP_SK
    fp_launch(plan_stream_kernel<0, false, false>, ctx->sm_count, PLAN_THREADS, stream_smem(ctx), ctx->stream,
        ctx->tmap_plane, ctx->tmap_occ, ctx->tmap_wall, A);
}

// Everything the planning phase allocates or builds, done outside any graph capture.
int fp_plan_prepare(fp_ctx* ctx, double k_s) {
    if (int rc = ensure_pathmasks(ctx)) return rc;
    if (!tiled_ok(ctx)) return FP_OK;
    if (int rc = fp_plane_ensure(ctx, k_s)) return rc;
    if (int rc = fp_bucket_reserve(ctx)) return rc;
    if (int rc = fp_ensure_res(ctx)) return rc;
    const size_t smem = stream_smem(ctx);
    static size_t configured_by_device[64] = {0};  // the attribute is per device
    size_t& configured = configured_by_device[ctx->device & 63];
    if (smem > configured) {
        for (const void* k : stream_kernels())
            FP_CUDA(ctx, cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured = smem;
    }
    return FP_OK;
}

static int launch_stream(fp_ctx* ctx, const StreamArgs& A) {
    FP_CUDA(ctx, cudaMemsetAsync(&ctx->d_sc->fb_count, 0, 8, ctx->stream));
    FP_CUDA(ctx, cudaMemsetAsync(&ctx->d_sc->tile_next, 0, 8, ctx->stream));
#ifdef FP_PLAN_PROF
    FP_CUDA(ctx, cudaMemsetAsync(ctx->d_sc->plan_prof, 0, sizeof(ctx->d_sc->plan_prof), ctx->stream));
#endif
    launch_stream_kernel(ctx, A);
    FP_LAUNCHED(ctx);
    return FP_OK;
}

#ifdef FP_STAGE_TIMING
__global__ void fp_stamp_kernel(unsigned long long* t) {
    FP_PDL_WAIT();
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    *t = v;
}
#endif

// Enqueues the whole planning phase (bucketing + streaming kernel + exact-path pass) on
// ctx->stream.  Graph-safe: the step, chunk counts, deal and the fallback count live in device
// memory; fp_plan_prepare ran before.
int fp_plan_launch(fp_ctx* ctx, double k_s, uint64_t seed, cudaEvent_t wait_before_kernel) {
    if (ctx->n == 0) return FP_OK;
    if (!tiled_ok(ctx)) return fp_plan_exact_launch(ctx, k_s, seed);
    if (!ctx->plane_valid || ctx->plane_ks != k_s || ctx->plane_potential != ctx->potential)
        return fp_fail(ctx, FP_ERUNTIME, "plan: weight plane not prepared for this k_s");
    FP_STAMP(ctx, ctx->stream, 0);
    if (int rc = fp_bucket_launch(ctx)) return rc;
    FP_STAMP(ctx, ctx->stream, 1);
    if (ctx->marks_dirty) {  // marks of an earlier plan no motion phase consumed
        const size_t nwords = (size_t)ctx->P * ctx->H;
        FP_CUDA(ctx, cudaMemsetAsync(ctx->d_p1, 0, nwords * 4, ctx->stream));
        FP_CUDA(ctx, cudaMemsetAsync(ctx->d_p2, 0, nwords * 4, ctx->stream));
    }
    ctx->bucket_fresh = true;  // the motion seed pass walks agents in this (spatial) order
    ctx->rec_fresh = true;     // walk records emitted below
    ctx->marks_dirty = true;
    ctx->plan_marked = plan_marks(ctx);  // ... with their footprints marked
    const StreamArgs A = make_stream_args(ctx, k_s, seed);
    // the persistent stream kernel takes every SM: work that must not queue behind it joins first
    if (wait_before_kernel) FP_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, wait_before_kernel, 0));
    if (int rc = launch_stream(ctx, A)) return rc;
    FP_STAMP(ctx, ctx->stream, 2);
    fp_launch(plan_exact_list_kernel, ctx->sm_count * 4, EXACT_THREADS, 0, ctx->stream, A.c, ctx->d_fallback, emit_args(ctx));
    FP_LAUNCHED(ctx);
    FP_STAMP(ctx, ctx->stream, 3);
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
    const StreamArgs A = make_stream_args(ctx, k_s, seed);
    cudaEvent_t e0, e1;
    FP_CUDA(ctx, cudaEventCreate(&e0));
    FP_CUDA(ctx, cudaEventCreate(&e1));
    double total = 0.0;
    const size_t nwords = (size_t)ctx->P * ctx->H;
    for (int i = 0; i < iters; ++i) {
        FP_CUDA(ctx, cudaMemsetAsync(&ctx->d_sc->fb_count, 0, 8, ctx->stream));
        FP_CUDA(ctx, cudaMemsetAsync(&ctx->d_sc->tile_next, 0, 8, ctx->stream));
        if (A.p1) {  // each launch marks afresh (outside the timed region)
            FP_CUDA(ctx, cudaMemsetAsync(ctx->d_p1, 0, nwords * 4, ctx->stream));
            FP_CUDA(ctx, cudaMemsetAsync(ctx->d_p2, 0, nwords * 4, ctx->stream));
        }
        cudaEventRecord(e0, ctx->stream);
        launch_stream_kernel(ctx, A);
        FP_LAUNCHED(ctx);
        cudaEventRecord(e1, ctx->stream);
        FP_CUDA(ctx, cudaEventSynchronize(e1));
        float t = 0;
        cudaEventElapsedTime(&t, e0, e1);
        total += t;
    }
    // the records were re-emitted by every launch; the next motion rebuilds nothing it needs
    ctx->rec_fresh = false;
    ctx->marks_dirty = true;
    // leave the state planned (the fallbacks of the last launch decided exactly)
    fp_launch(plan_exact_list_kernel, ctx->sm_count * 4, EXACT_THREADS, 0, ctx->stream, A.c, ctx->d_fallback, emit_args(ctx));
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
    fp_launch(choice_kernel, 1, 1, 0, ctx->stream, a, plane, ctx->PW, agent, d_cx, d_cy, d_w, d_p, d_n);
    FP_LAUNCHED(ctx);
    return FP_OK;
}

// choose_desired_cell(st, agent, params) for one agent given by value (planning.hpp:88-108).
int fp_choose_one_launch(fp_ctx* ctx, uint32_t id, int px, int py, int v, int64_t step, double k_s, uint64_t seed,
                         int32_t* d_out) {
    if (int rc = ensure_pathmasks(ctx)) return rc;
    PlanCommon a = make_common(ctx, k_s, seed);
    fp_launch(choose_one_kernel, 1, 1, 0, ctx->stream, a, id, px, py, v, (long long)step, d_out);
    FP_LAUNCHED(ctx);
    return FP_OK;
}

// enumerate_candidates(st, agent) for one agent given by value (planning.hpp:23-57).
int fp_candidates_one_launch(fp_ctx* ctx, int px, int py, int v, int32_t* d_cx, int32_t* d_cy, uint32_t* d_n) {
    PlanCommon a = make_common(ctx, 0.0, 0);
    fp_launch(candidates_one_kernel, 1, 1, 0, ctx->stream, a, px, py, v, d_cx, d_cy, d_n);
    FP_LAUNCHED(ctx);
    return FP_OK;
}
