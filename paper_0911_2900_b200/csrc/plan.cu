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
//           plane word with integer ops (exact fp64 value of an fp32-rounded weight) and summed
//           per row in fp64;
//   pass 2  threshold u*total picks the row, the row is replayed in the reference's list order
//           (rotated at a periodic seam) to find the first cumulative weight > threshold.
// Guard band: every weight is the reference weight times a common factor to within 2^-24, the
// fp64 sums add < 1e-14.  If the threshold lies further than 1.5e-7*total from both cumulative
// boundaries of the chosen candidate, the reference (serial fp64 sum, glibc exp) picks the same
// candidate; otherwise the agent is re-sampled on the exact path.
//
// Exact path (choose_exact): one thread, candidates in list order, weights through the
// bit-exact restated glibc exp (fp_exp.h), serial fp64 total and scan -- bitwise the
// reference's arithmetic.  Used for guard-band misses, "unsafe" plane cells, k_s/grid shapes the
// tiled path does not cover, and test-mode dumps.  There is no CPU fallback.
#include <math.h>

#include "fp_exp.h"
#include "internal.cuh"

#define FP_GUARD 1.5e-7

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

// choose_desired_cell, exact (planning.hpp:88-108 + sample_index :63-73)
__device__ __noinline__ void choose_exact(const PlanCommon& a, uint32_t i, uint64_t step, int* ox, int* oy) {
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
    const uint32_t* tile_off;
    const uint32_t* tile_cnt;
    const uint32_t* tile_list;
    int tile_w, tile_h, tiles_x;
    int use_tma;  // 0: stage the box with coalesced loads (debug / comparison path)
    int boxw, boxh, occw;  // shared-memory strides (words)
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

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int cx, int cy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(cx), "r"(cy)
        : "memory");
}

// Plans one agent from the staged tile; returns false when the exact path must decide.
__device__ __forceinline__ bool plan_fast(const TileArgs& A, const uint32_t* buf, const uint32_t* occs, int x0, int y0,
                                          uint32_t id, int px, int py, int v, double u, const double* drive_tab,
                                          int* ox, int* oy) {
    const PlanCommon& a = A.c;
    const int X0 = x0 - 8;  // box origin: TMA needs 16-byte aligned inner coordinates
    const int lx = px - X0, ly = py - (y0 - FP_HALO);
    const uint32_t own = buf[ly * A.boxw + lx];
    int mode;
    int Cp = 0;
    if (a.potential == FP_POTENTIAL_DRIVE_X) {
        mode = MODE_DRIVE;
    } else if (own == FP_W_UNREACH) {
        mode = MODE_ONES;  // planning.hpp:93-95
    } else {
        if (own & FP_W_UNSAFE) return false;
        mode = MODE_EXIT;
        Cp = (int)((own >> 23) & 0x7Fu);
    }
    const int osh = ((X0 + FP_XPAD_BITS) & 31) + lx - 5;  // bit of dx = -5 in the staged occ row
    uint32_t wm0 = 0, wm1 = 0, wm2 = 0, wm3 = 0;           // ball wall mask (11x11 frame)
    double rs[11];
#pragma unroll
    for (int t = 0; t < 11; ++t) {
        const int dy = (t & 1) ? -((t + 1) >> 1) : (t >> 1);
        rs[dy + 5] = 0.0;
        if (dy < -v || dy > v) continue;
        const int yy = py + dy;
        if (yy < 0 || yy >= a.g.H) continue;
        const uint32_t* row = buf + (ly + dy) * A.boxw + lx;
        uint32_t wv[11];
#pragma unroll
        for (int k = 0; k < 11; ++k) {
            const int dx = k - 5;
            wv[k] = (dx >= -v && dx <= v) ? row[dx] : FP_W_WALL;
        }
#pragma unroll
        for (int k = 0; k < 11; ++k) {
            const int b = (dy + 5) * 11 + k;
            const uint32_t bit = (wv[k] == FP_W_WALL && k - 5 >= -v && k - 5 <= v) ? (1u << (b & 31)) : 0u;
            if ((b >> 5) == 0) wm0 |= bit;
            else if ((b >> 5) == 1) wm1 |= bit;
            else if ((b >> 5) == 2) wm2 |= bit;
            else wm3 |= bit;
        }
        const uint32_t* orow = occs + (ly + dy) * A.occw;
        const uint32_t win = __funnelshift_r(orow[osh >> 5], orow[(osh >> 5) + 1], osh & 31);
        const bool anywall = (wm0 | wm1 | wm2 | wm3) != 0u;
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < 11; ++k) {
            const int dx = k - 5;
            if (wv[k] == FP_W_WALL) continue;
            if (((win >> k) & 1u) && !(dx == 0 && dy == 0)) continue;
            const int o = (dy + 5) * 11 + k;
            if (anywall && ((wm0 & c_pathmask[o][0]) | (wm1 & c_pathmask[o][1]) | (wm2 & c_pathmask[o][2]) |
                            (wm3 & c_pathmask[o][3])))
                continue;
            s += fast_weight(wv[k], Cp, mode, drive_tab[k]);
        }
        rs[dy + 5] = s;
    }
    double T = 0.0;
#pragma unroll
    for (int k = 0; k < 11; ++k) T += rs[k];
    const double theta = u * T;
    int rstar = -1;
    double before = 0.0, cum = 0.0;
#pragma unroll
    for (int k = 0; k < 11; ++k) {
        if (rstar < 0 && cum + rs[k] > theta) {
            rstar = k;
            before = cum;
        }
        cum += rs[k];
    }
    if (rstar < 0) return false;
    // pass 2: replay the crossing row in list order (wrapped-x sorted at a periodic seam)
    const int dy = rstar - 5;
    const uint32_t* row = buf + (ly + dy) * A.boxw + lx;
    const uint32_t* orow = occs + (ly + dy) * A.occw;
    const uint32_t win = __funnelshift_r(orow[osh >> 5], orow[(osh >> 5) + 1], osh & 31);
    int a0 = -v, a1 = v, b0 = 0, b1 = -1;
    if (a.g.boundary == FP_BOUNDARY_PERIODIC_X) {
        if (px + v >= a.g.W) {
            a0 = a.g.W - px; b0 = -v; b1 = a.g.W - px - 1;
        } else if (px - v < 0) {
            a0 = -px; b0 = -v; b1 = -px - 1;
        }
    }
    const bool anywall = (wm0 | wm1 | wm2 | wm3) != 0u;
    double prefix = before, lower = 0.0, upper = 0.0;
    int kx = 0;
    bool found = false;
    for (int seg = 0; seg < 2 && !found; ++seg) {
        const int lo = seg ? b0 : a0, hi = seg ? b1 : a1;
        for (int dx = lo; dx <= hi; ++dx) {
            const uint32_t wv = row[dx];
            if (wv == FP_W_WALL) continue;
            if (((win >> (dx + 5)) & 1u) && !(dx == 0 && dy == 0)) continue;
            const int o = rstar * 11 + dx + 5;
            if (anywall && ((wm0 & c_pathmask[o][0]) | (wm1 & c_pathmask[o][1]) | (wm2 & c_pathmask[o][2]) |
                            (wm3 & c_pathmask[o][3])))
                continue;
            const double w = fast_weight(wv, Cp, mode, drive_tab[dx + 5]);
            const double next = prefix + w;
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
    if (!found) return false;
    const double margin = FP_GUARD * T;
    if (!(upper - theta > margin)) return false;
    if (!(lower == 0.0 || theta - lower > margin)) return false;
    *ox = a.g.wrap(px + kx);
    *oy = py + dy;
    return true;
}

__global__ void __launch_bounds__(256, 1) plan_tile_kernel(const __grid_constant__ CUtensorMap tmap, TileArgs A) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    // TMA destinations need 128-byte alignment: align the dynamic window explicitly
    unsigned char* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
    const int box_words = A.boxw * A.boxh;
    const int box_bytes = box_words * 4;
    uint32_t* bufs[2] = {(uint32_t*)smem, (uint32_t*)(smem + ((box_bytes + 127) & ~127))};
    uint32_t* occs = (uint32_t*)(smem + 2 * ((box_bytes + 127) & ~127));
    uint64_t* bars = (uint64_t*)(occs + ((A.boxh * A.occw + 31) & ~31));
    __shared__ int s_tile[2];
    __shared__ double s_drive[11];
    const PlanCommon& a = A.c;
    const uint64_t step = (uint64_t)a.sc->step;
    const unsigned n_tiles = (unsigned)a.sc->n_tiles;
    if (threadIdx.x == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 11) {
        s_drive[threadIdx.x] = (a.potential == FP_POTENTIAL_DRIVE_X)
                                   ? (double)drive_weight_f(a.k_s, a.drive_gradient, (int)threadIdx.x - 5)
                                   : 0.0;
    }
    __syncthreads();
    unsigned parity[2] = {0u, 0u};
    if (threadIdx.x == 0) {
        const int t = (int)atomicAdd(&a.sc->tile_next, 1ull);
        s_tile[0] = t;
        if (t < (int)n_tiles && A.use_tma) {
            const uint32_t tid = A.tile_list[t];
            const int tx = (int)(tid % (uint32_t)A.tiles_x), ty = (int)(tid / (uint32_t)A.tiles_x);
            mbar_expect_tx(&bars[0], (unsigned)box_bytes);
            tma_load_2d(bufs[0], &tmap, &bars[0], tx * A.tile_w - 8 + FP_XPAD_W, ty * A.tile_h - FP_HALO);
        }
    }
    __syncthreads();
    int cur = s_tile[0];
    int b = 0;
    while (cur < (int)n_tiles) {
        if (threadIdx.x == 0) {
            const int t = (int)atomicAdd(&a.sc->tile_next, 1ull);
            s_tile[(b ^ 1)] = t;
            if (t < (int)n_tiles && A.use_tma) {
                const uint32_t tid = A.tile_list[t];
                const int tx = (int)(tid % (uint32_t)A.tiles_x), ty = (int)(tid / (uint32_t)A.tiles_x);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_expect_tx(&bars[b ^ 1], (unsigned)box_bytes);
                tma_load_2d(bufs[b ^ 1], &tmap, &bars[b ^ 1], tx * A.tile_w - 8 + FP_XPAD_W, ty * A.tile_h - FP_HALO);
            }
        }
        const uint32_t tile = A.tile_list[cur];
        const int tx = (int)(tile % (uint32_t)A.tiles_x), ty = (int)(tile / (uint32_t)A.tiles_x);
        const int x0 = tx * A.tile_w, y0 = ty * A.tile_h;
        // stage the occupancy words of the window (rows y0-5 .. y0+tile_h+4)
        {
            const int gw0 = (x0 - 8 + FP_XPAD_BITS) >> 5;
            const int total = A.boxh * A.occw;
            for (int k = threadIdx.x; k < total; k += blockDim.x) {
                const int r = k / A.occw, wcol = k % A.occw;
                const int yy = y0 - FP_HALO + r;
                const int gw = gw0 + wcol;
                uint32_t val = 0u;
                if (yy >= 0 && yy < a.g.H && gw < a.g.P) val = a.occ[(size_t)yy * a.g.P + gw];
                occs[k] = val;
            }
        }
        if (A.use_tma) {
            mbar_wait(&bars[b], parity[b]);
            parity[b] ^= 1u;
        } else {
            uint32_t* dst = bufs[b];
            const int total = A.boxw * A.boxh;
            const int gx0 = x0 - 8 + FP_XPAD_W, gy0 = y0 - FP_HALO;
            for (int k = threadIdx.x; k < total; k += blockDim.x) {
                const int r = k / A.boxw, cidx = k % A.boxw;
                const int gy = gy0 + r, gx = gx0 + cidx;
                dst[k] = (gy >= 0 && gy < a.g.H && gx < A.PW) ? A.plane[(size_t)gy * A.PW + gx] : 0u;
            }
        }
        __syncthreads();
        const uint32_t* buf = bufs[b];
        const uint32_t off = A.tile_off[tile], cnt = A.tile_cnt[tile];
        for (uint32_t k = threadIdx.x; k < cnt; k += blockDim.x) {
            const uint32_t id = A.bucket[off + k];
            const int px = a.g.wrap(a.x[id]), py = a.y[id];
            const int v = a.v[id];
            const double u = fp_unit_interval(fp_rng_u64(a.seed, id, step, 0));
            int cx, cy;
            if (!plan_fast(A, buf, occs, x0, y0, id, px, py, v, u, s_drive, &cx, &cy)) {
                choose_exact(a, id, step, &cx, &cy);
                atomicAdd(&a.sc->fallbacks, 1ull);
            }
            a.dx[id] = cx;
            a.dy[id] = cy;
        }
        __syncthreads();
        cur = s_tile[b ^ 1];
        b ^= 1;
    }
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
    A.occw = (A.boxw + 31) / 32 + 2;
    const int box_bytes = A.boxw * A.boxh * 4;
    smem = 2 * (size_t)((box_bytes + 127) & ~127) + (size_t)((A.boxh * A.occw + 31) & ~31) * 4 + 256;
}

// Everything the planning phase allocates or builds, done outside any graph capture.
int fp_plan_prepare(fp_ctx* ctx, double k_s) {
    if (int rc = ensure_pathmasks(ctx)) return rc;
    if (!tiled_ok(ctx)) return FP_OK;
    if (int rc = fp_plane_ensure(ctx, k_s)) return rc;
    if (int rc = fp_bucket_reserve(ctx)) return rc;
    TileArgs A;
    size_t smem;
    tile_geometry(ctx, A, smem);
    static size_t configured = 0;
    if (smem > configured) {
        FP_CUDA(ctx, cudaFuncSetAttribute(plan_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured = smem;
    }
    return FP_OK;
}

// Enqueues the whole planning phase (bucketing + tiled kernel) on ctx->stream.  Graph-safe:
// the step, tile count and cursors live in device memory; fp_plan_prepare ran before.
int fp_plan_launch(fp_ctx* ctx, double k_s, uint64_t seed) {
    if (ctx->n == 0) return FP_OK;
    if (!tiled_ok(ctx)) return fp_plan_exact_launch(ctx, k_s, seed);
    if (!ctx->plane_valid || ctx->plane_ks != k_s || ctx->plane_potential != ctx->potential)
        return fp_fail(ctx, FP_ERUNTIME, "plan: weight plane not prepared for this k_s");
    if (int rc = fp_bucket_launch(ctx)) return rc;
    TileArgs A;
    A.c = make_common(ctx, k_s, seed);
    A.PW = ctx->PW;
    A.plane = ctx->d_plane;
    A.use_tma = ctx->use_tma;
    A.bucket = ctx->d_bucket;
    A.tile_off = ctx->d_tile_off;
    A.tile_cnt = ctx->d_tile_cnt;
    A.tile_list = ctx->d_tile_list;
    A.tile_w = ctx->tile_w;
    A.tile_h = ctx->tile_h;
    A.tiles_x = ctx->tiles_x;
    size_t smem;
    tile_geometry(ctx, A, smem);
    FP_CUDA(ctx, cudaMemsetAsync(&ctx->d_sc->tile_next, 0, 8, ctx->stream));
    const size_t nt = (size_t)ctx->tiles_x * ctx->tiles_y;
    const unsigned grid = (unsigned)std::min<size_t>((size_t)ctx->sm_count, nt);
    plan_tile_kernel<<<grid, 256, smem, ctx->stream>>>(ctx->tmap_plane, A);
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
    TileArgs A;
    A.c = make_common(ctx, k_s, seed);
    A.PW = ctx->PW;
    A.plane = ctx->d_plane;
    A.use_tma = ctx->use_tma;
    A.bucket = ctx->d_bucket;
    A.tile_off = ctx->d_tile_off;
    A.tile_cnt = ctx->d_tile_cnt;
    A.tile_list = ctx->d_tile_list;
    A.tile_w = ctx->tile_w;
    A.tile_h = ctx->tile_h;
    A.tiles_x = ctx->tiles_x;
    size_t smem;
    tile_geometry(ctx, A, smem);
    const size_t nt = (size_t)ctx->tiles_x * ctx->tiles_y;
    const unsigned grid = (unsigned)std::min<size_t>((size_t)ctx->sm_count, nt);
    cudaEvent_t e0, e1;
    FP_CUDA(ctx, cudaEventCreate(&e0));
    FP_CUDA(ctx, cudaEventCreate(&e1));
    double total = 0.0;
    for (int i = 0; i < iters; ++i) {
        FP_CUDA(ctx, cudaMemsetAsync(&ctx->d_sc->tile_next, 0, 8, ctx->stream));
        cudaEventRecord(e0, ctx->stream);
        plan_tile_kernel<<<grid, 256, smem, ctx->stream>>>(ctx->tmap_plane, A);
        FP_LAUNCHED(ctx);
        cudaEventRecord(e1, ctx->stream);
        FP_CUDA(ctx, cudaEventSynchronize(e1));
        float t = 0;
        cudaEventElapsedTime(&t, e0, e1);
        total += t;
    }
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
