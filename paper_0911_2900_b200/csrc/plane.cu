// plane.cu -- the static planning plane and the ghost columns of the bitplanes.
//
// The reference weighs candidate c of an agent at p by w = exp(k_s * (S(p) - S(c)))
// (planning.hpp:102).  With K = k_s*log2(e) and y = K*S, w = 2^(y_p - y_c).  Per cell we store
// the split 2^(-y_c) = m_c * 2^(-C_c), C_c = ceil(y_c), m_c = 2^(C_c - y_c) in [1, 2), as one u32
// laid out like an fp32 number:
//     bit 31      "exact" flag: Wall (0xFFFFFFFF), unreachable free cell, or a centre the fast
//                 path must not plan -- some reachable cell within Chebyshev 5 has
//                 |C - C_c| > 60, or an unreachable free cell lies within Chebyshev 5
//     bits 30..23 (-C_c) mod 256
//     bits 22..0  23-bit mantissa of m_c (relative rounding error <= 2^-24)
// An agent at p weighs c by m_c * 2^(C_p - C_c) -- the reference weight times the common factor
// 2^(C_p - y_p) -- so sampling (scale invariant, planning.hpp:60-62) sees the reference weights
// to 2^-24 relative; the plan kernel's guard band turns that into bit-exact decisions (plan.cu).
// That weight is ONE integer add away from the word: w_c + ((C_p + 127) mod 256) << 23 has
// exponent field (C_p - C_c + 127) mod 256 and c's mantissa, i.e. it is +-m_c * 2^(C_p - C_c)
// as an fp32 number (the carry out of the exponent lands in the sign bit, which the kernel's
// |x| operand modifier drops).  4 bytes per cell instead of the fp64 field's 8.
// DriveX: the plane only carries walls (weights depend on dx alone, plan.cu table).
#include <limits.h>
#include <math.h>

#include "internal.cuh"

__global__ void plane_build_kernel(Geo g, int PW, const double* field, int potential, double K,
                                   uint32_t* plane, int* cval) {
    FP_PDL_WAIT();
    const size_t total = (size_t)PW * g.H;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int y = (int)(i / PW);
        int x = (int)(i % PW) - FP_XPAD_W;
        int c = INT_MIN;
        uint32_t w;
        if (x < 0 || x >= g.W) {
            if (g.boundary != FP_BOUNDARY_PERIODIC_X) {
                plane[i] = FP_W_WALL;
                cval[i] = INT_MIN;
                continue;
            }
            x = g.wrap(x);
        }
        if (g.is_wall(x, y)) {
            w = FP_W_WALL;
        } else if (potential == FP_POTENTIAL_DRIVE_X) {
            w = 0u;
            c = 0;
        } else {
            const double s = field[(size_t)y * g.W + x];
            if (isinf(s)) {
                w = FP_W_UNREACH;
                c = INT_MIN + 1;  // unreachable free cell (flags every centre within Chebyshev 5)
            } else {
                const double yv = K * s;
                double C = ceil(yv);
                const double m = exp2(C - yv);  // [1, 2]
                double mant = rint((m - 1.0) * 8388608.0);
                if (mant >= 8388608.0) {  // m rounded up to 2: 2 * 2^-C = 2^-(C-1)
                    mant = 0.0;
                    C -= 1.0;
                }
                const long long Ci = (long long)C;
                c = (int)Ci;
                w = ((uint32_t)(-Ci & 0xFF) << 23) | (uint32_t)mant;
            }
        }
        plane[i] = w;
        cval[i] = c;
    }
}

// Chunk-tiled copy of the plane for the plan kernel's producer: block (stripe s, chunk k) holds
// rows 8k..8k+7, columns s*tile_w - 8 .. s*tile_w + tile_w + 8 (the stripe and its halo) as one
// contiguous 8 * boxw-word run, and the chunks of a stripe follow each other -- a plan item's
// rows are one contiguous range of HBM (long DRAM bursts instead of 1 KB row pieces 80 KB apart).
// Words outside the plane (rows >= H, columns past the pitch) read as Wall.
__global__ void plane_tile_kernel(const uint32_t* plane, int PW, int H, int tile_w, int boxw, int rows_chunks,
                                  size_t total, uint32_t* out) {
    FP_PDL_WAIT();
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int c = (int)(i % boxw);
        const size_t rb = i / boxw;  // (stripe * rows_chunks + chunk) * 8 + row
        const int r = (int)(rb % 8);
        const size_t b = rb / 8;
        const int k = (int)(b % rows_chunks), st = (int)(b / rows_chunks);
        const int y = 8 * k + r;
        const int xp = st * tile_w - 8 + c + FP_XPAD_W;  // plane column
        out[i] = (y < H && xp >= 0 && xp < PW) ? plane[(size_t)y * PW + xp] : FP_W_WALL;
    }
}

// Row pass of the radius-5 min/max of C (cval: INT_MIN wall / outside, INT_MIN + 1 unreachable
// free cell; a window holding an unreachable cell gets rmin = INT_MIN).
__global__ void plane_rowminmax_kernel(int PW, int H, const int* cval, int* rmin, int* rmax) {
    FP_PDL_WAIT();
    const size_t total = (size_t)PW * H;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int xp = (int)(i % PW);
        const size_t row = i - xp;
        int mn = INT_MAX, mx = INT_MIN;
        for (int d = -FP_HALO; d <= FP_HALO; ++d) {
            const int q = xp + d;
            if (q < 0 || q >= PW) continue;
            const int c = cval[row + q];
            if (c == INT_MIN) continue;
            if (c == INT_MIN + 1) {
                mn = INT_MIN;
                continue;
            }
            mn = min(mn, c);
            mx = max(mx, c);
        }
        rmin[i] = mn;
        rmax[i] = mx;
    }
}

__global__ void plane_unsafe_kernel(int PW, int H, const int* cval, const int* rmin, const int* rmax,
                                    uint32_t* plane, unsigned long long* n_unsafe) {
    FP_PDL_WAIT();
    const size_t total = (size_t)PW * H;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int c = cval[i];
        if (c == INT_MIN || c == INT_MIN + 1) continue;  // walls / unreachable cells carry the flag already
        const int xp = (int)(i % PW), y = (int)(i / PW);
        int mn = INT_MAX, mx = INT_MIN;
        for (int d = -FP_HALO; d <= FP_HALO; ++d) {
            const int yy = y + d;
            if (yy < 0 || yy >= H) continue;
            mn = min(mn, rmin[(size_t)yy * PW + xp]);
            mx = max(mx, rmax[(size_t)yy * PW + xp]);
        }
        if (mn == INT_MIN || mx - c > 60 || c - mn > 60) {
            plane[i] |= FP_W_FLAG;
            atomicAdd(n_unsafe, 1ull);
        }
    }
}

// Ghost bits of a bitplane for periodic-x grids: bits at x outside [0, W) mirror wrap(x).
__global__ void ghost_bits_kernel(Geo g, uint32_t* plane) {
    FP_PDL_WAIT();
    // words that hold any x outside [0, W): word 0 (x in [-32,0)) and words from (W+32)/32 on
    const int first_right = (g.W + FP_XPAD_BITS) >> 5;
    const int per_row = 1 + (g.P - first_right);
    const size_t total = (size_t)per_row * g.H;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int y = (int)(i / per_row);
        const int k = (int)(i % per_row);
        const int wi = (k == 0) ? 0 : first_right + k - 1;
        const size_t idx = (size_t)y * g.P + wi;
        uint32_t cur = plane[idx];
        uint32_t out = 0;
        for (int b = 0; b < 32; ++b) {
            const int x = wi * 32 - FP_XPAD_BITS + b;
            uint32_t bit;
            if (x >= 0 && x < g.W) {
                bit = (cur >> b) & 1u;
            } else {
                const int xs = g.wrap(x);
                bit = (plane[g.word(xs, y)] >> (xs & 31)) & 1u;
            }
            out |= bit << b;
        }
        plane[idx] = out;
    }
}

int fp_ghost_occ(fp_ctx* ctx) {
    if (ctx->boundary != FP_BOUNDARY_PERIODIC_X) return FP_OK;
    fp_launch(ghost_bits_kernel, fp_blocks((size_t)ctx->H * 4, 256), 256, 0, ctx->stream, fp_geo(ctx), ctx->d_occ);
    FP_LAUNCHED(ctx);
    return FP_OK;
}

int fp_ghost_static(fp_ctx* ctx) {
    if (ctx->boundary != FP_BOUNDARY_PERIODIC_X) return FP_OK;
    fp_launch(ghost_bits_kernel, fp_blocks((size_t)ctx->H * 4, 256), 256, 0, ctx->stream, fp_geo(ctx), ctx->d_wall);
    FP_LAUNCHED(ctx);
    fp_launch(ghost_bits_kernel, fp_blocks((size_t)ctx->H * 4, 256), 256, 0, ctx->stream, fp_geo(ctx), ctx->d_exit);
    FP_LAUNCHED(ctx);
    return FP_OK;
}

// ---------------------------------------------------------------------------- TMA descriptor
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
    static PFN_encodeTiled fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_encodeTiled)p;
    }
    return fn;
}

// Marks every tile whose window (tile + FP_HALO cells, wrapped at a periodic seam) holds an Exit.
__global__ void tile_exit_kernel(Geo g, int tile_w, int tile_h, int tiles_x, int tiles_y, uint8_t* flag) {
    FP_PDL_WAIT();
    const size_t nwords = (size_t)g.P * g.H;
    for (size_t w = blockIdx.x * (size_t)blockDim.x + threadIdx.x; w < nwords; w += (size_t)gridDim.x * blockDim.x) {
        uint32_t bits = g.exitb[w];
        const int y = (int)(w / g.P), x0 = (int)(w % g.P) * 32 - FP_XPAD_BITS;
        while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            const int x = x0 + b;
            if (x < 0 || x >= g.W) continue;  // ghost column (mirrors a real one)
            for (int ty = max(0, (y - FP_HALO) / tile_h); ty <= min(tiles_y - 1, (y + FP_HALO) / tile_h); ++ty)
                for (int dx = -FP_HALO; dx <= FP_HALO; ++dx) {
                    int xx = x + dx;
                    if (g.boundary == FP_BOUNDARY_PERIODIC_X) xx = ((xx % g.W) + g.W) % g.W;
                    else if (xx < 0 || xx >= g.W) continue;
                    flag[(size_t)ty * tiles_x + xx / tile_w] = 1;
                }
        }
    }
}

// Chooses the stripe width / motion tile for this grid and encodes the TMA boxes of one 8-row
// chunk of a stripe (stripe + 8 columns each side, so the inner box start stays 16-byte aligned
// and the box holds the 5-cell halo).
#ifndef FP_BIG_TILE_H
#define FP_BIG_TILE_H 48
#endif
static int make_tmap(fp_ctx* ctx) {
    const size_t cells = (size_t)ctx->W * ctx->H;
    if (cells >= (size_t)16 << 20) {
        ctx->tile_w = 240;
        ctx->tile_h = FP_BIG_TILE_H;  // three 63 KB slots fit in shared memory
    } else if (cells >= (size_t)1 << 20) {
        ctx->tile_w = 120;
        ctx->tile_h = 32;
    } else {
        ctx->tile_w = 56;
        ctx->tile_h = 16;
    }
    ctx->tiles_x = (ctx->W + ctx->tile_w - 1) / ctx->tile_w;
    ctx->tiles_y = (ctx->H + ctx->tile_h - 1) / ctx->tile_h;
    ctx->cps = ctx->tiles_y * (ctx->tile_h / 8);
    PFN_encodeTiled enc = get_encode();
    if (!enc) return fp_fail(ctx, FP_ECUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {(cuuint64_t)ctx->PW, (cuuint64_t)ctx->H};
    cuuint64_t strides[1] = {(cuuint64_t)ctx->PW * 4};
    // inner box start x0-8 keeps the inner coordinate 16-byte aligned (an unaligned inner
    // coordinate faults with "illegal instruction" on sm_100a, tools/tma_probe); box covers
    // [x0-8, x0+tile_w+8) which contains the 5-cell halo on both sides
    cuuint32_t box[2] = {(cuuint32_t)(ctx->tile_w + 16), 8u};  // one 8-row chunk of a stripe (plan.cu)
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&ctx->tmap_plane, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, ctx->d_plane, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fp_fail(ctx, FP_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    // occupancy bitplane: a 16-word (512-bit) box from a 16-byte aligned word covers the
    // 5-cell halo window of any tile (tile_w + 16 <= 256 columns, <= 127 bits of misalignment)
    cuuint64_t odims[2] = {(cuuint64_t)ctx->P, (cuuint64_t)ctx->H};
    cuuint64_t ostr[1] = {(cuuint64_t)ctx->P * 4};
    cuuint32_t obox[2] = {16u, 8u};
    r = enc(&ctx->tmap_occ, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, ctx->d_occ, odims, ostr, obox, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fp_fail(ctx, FP_ECUDA, "cuTensorMapEncodeTiled(occ) failed (" + std::to_string((int)r) + ")");
    r = enc(&ctx->tmap_wall, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, ctx->d_wall, odims, ostr, obox, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fp_fail(ctx, FP_ECUDA, "cuTensorMapEncodeTiled(wall) failed (" + std::to_string((int)r) + ")");
    // per tile: does its 5-cell halo window hold an Exit?  (the plan kernel's walk records skip
    // exit lookups elsewhere)
    const size_t nt = (size_t)ctx->tiles_x * ctx->tiles_y;
    FP_CUDA(ctx, cudaMalloc(&ctx->d_tile_exit, nt));
    FP_CUDA(ctx, cudaMemsetAsync(ctx->d_tile_exit, 0, nt, ctx->stream));
    const size_t nwords = (size_t)ctx->P * ctx->H;
    fp_launch(tile_exit_kernel, (unsigned)std::min<size_t>(fp_blocks(nwords, 256), (size_t)ctx->sm_count * 16), 256, 0, ctx->stream, fp_geo(ctx), ctx->tile_w, ctx->tile_h, ctx->tiles_x, ctx->tiles_y,
                                      ctx->d_tile_exit);
    FP_LAUNCHED(ctx);
    return FP_OK;
}

// Builds (or reuses) the plane for (k_s, potential).  Setup work: one pass over the grid.
int fp_plane_ensure(fp_ctx* ctx, double k_s) {
    if (ctx->plane_valid && ctx->plane_ks == k_s && ctx->plane_potential == ctx->potential) return FP_OK;
    cudaStream_t s = ctx->stream;
    const size_t total = (size_t)ctx->PW * ctx->H;
    if (!ctx->d_plane) {
        FP_CUDA(ctx, cudaMalloc(&ctx->d_plane, total * 4));
        if (int rc = make_tmap(ctx)) return rc;
    }
    int *cval = nullptr, *rmin = nullptr, *rmax = nullptr;
    FP_CUDA(ctx, cudaMallocAsync(&cval, total * 4, s));
    FP_CUDA(ctx, cudaMallocAsync(&rmin, total * 4, s));
    FP_CUDA(ctx, cudaMallocAsync(&rmax, total * 4, s));
    const double K = k_s * 1.4426950408889634;  // k_s * log2(e)
    const unsigned G = (unsigned)ctx->sm_count * 8;
    fp_launch(plane_build_kernel, G, 256, 0, s, fp_geo(ctx), ctx->PW, ctx->d_field, ctx->potential, K, ctx->d_plane, cval);
    FP_LAUNCHED(ctx);
    if (ctx->potential == FP_POTENTIAL_EXIT_DISTANCE) {
        fp_launch(plane_rowminmax_kernel, G, 256, 0, s, ctx->PW, ctx->H, cval, rmin, rmax);
        FP_LAUNCHED(ctx);
        FP_CUDA(ctx, cudaMemsetAsync(&ctx->d_sc->pad[0], 0, 8, s));
        fp_launch(plane_unsafe_kernel, G, 256, 0, s, ctx->PW, ctx->H, cval, rmin, rmax, ctx->d_plane, &ctx->d_sc->pad[0]);
        FP_LAUNCHED(ctx);
    }
    {
        const int boxw = ctx->tile_w + 16, rc = (ctx->H + 7) / 8;
        const size_t tot = (size_t)ctx->tiles_x * rc * 8 * boxw;
        if (!ctx->d_plane_t) FP_CUDA(ctx, cudaMalloc(&ctx->d_plane_t, tot * 4));
        fp_launch(plane_tile_kernel, G, 256, 0, s, ctx->d_plane, ctx->PW, ctx->H, ctx->tile_w, boxw, rc, tot, ctx->d_plane_t);
        FP_LAUNCHED(ctx);
    }
    FP_CUDA(ctx, cudaFreeAsync(cval, s));
    FP_CUDA(ctx, cudaFreeAsync(rmin, s));
    FP_CUDA(ctx, cudaFreeAsync(rmax, s));
    ctx->plane_valid = true;
    ctx->plane_ks = k_s;
    ctx->plane_potential = ctx->potential;
    ctx->graph_valid = false;
    return FP_OK;
}
