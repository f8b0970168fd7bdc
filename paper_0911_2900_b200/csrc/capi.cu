// capi.cu -- the C ABI (include/fastped_b200.h): context lifecycle, uploads, the step
// sequence, dumps.  Host logic mirrors the reference's validation and error wording
// (state.hpp:38-76, engine.hpp, world.hpp:37-63, scenario_io.hpp:47-69).
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include "internal.cuh"

static thread_local std::string g_error;

#ifndef FP_RUN_UNROLL
#define FP_RUN_UNROLL 8  // steps per run() graph launch (FASTPED_RUN_UNROLL overrides)
#endif

bool fp_pdl_enabled() {
    static const bool on = [] {
        const char* e = getenv("FASTPED_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

void fp_set_global_error(const std::string& s) { g_error = s; }

static int fail(fp_ctx* ctx, int code, const std::string& msg) {
    if (ctx) ctx->err = msg;
    g_error = msg;
    return code;
}

int fp_fail(fp_ctx* ctx, int code, const std::string& msg) { return fail(ctx, code, msg); }

int fp_cuda_fail(fp_ctx* ctx, cudaError_t e, const char* what) {
    return fail(ctx, FP_ECUDA, std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

extern "C" const char* fp_version(void) { return "fastped-b200 0.1 (sm_100a)"; }

extern "C" const char* fp_last_error(const fp_ctx* ctx) {
    return ctx ? ctx->err.c_str() : g_error.c_str();
}

extern "C" int fp_device_count(int* n) {
    if (!n) return fail(nullptr, FP_EINVAL, "null argument");
    *n = 0;
    cudaError_t e = cudaGetDeviceCount(n);
    if (e != cudaSuccess) return fail(nullptr, FP_ECUDA, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
    return FP_OK;
}

extern "C" int fp_compute_blocksize(int64_t agents, int cores, int32_t* out) {
    if (cores < 1) return fail(nullptr, FP_EINVAL, "compute_blocksize: cores must be >= 1");
    if (agents < 0) return fail(nullptr, FP_EINVAL, "compute_blocksize: agent count must be >= 0");
    const int64_t c = std::min<int64_t>(agents / cores, 32767);
    *out = (int32_t)std::max<int64_t>(c, 1);
    return FP_OK;
}

// ------------------------------------------------------------------------ grid validation
static int validate_grid(const fp_grid_desc* g, const uint8_t* cells) {
    if (!g || !cells) return fail(nullptr, FP_EINVAL, "Grid: null descriptor or cells");
    if (g->width < 1 || g->height < 1) return fail(nullptr, FP_EINVAL, "Grid: width and height must be >= 1");
    if (!(g->cell_size > 0.0)) return fail(nullptr, FP_EINVAL, "Grid: cell_size must be > 0");
    if (g->boundary != FP_BOUNDARY_CLOSED && g->boundary != FP_BOUNDARY_PERIODIC_X)
        return fail(nullptr, FP_EINVAL, "Grid: unknown boundary");
    if ((int64_t)g->width * g->height >= (int64_t)1 << 32)
        return fail(nullptr, FP_EINVAL, "Grid: more than 2^32 cells");
    if (g->width >= (1 << 27) || g->height >= (1 << 24))  // motion record fields (motion_rec.cuh)
        return fail(nullptr, FP_EINVAL, "Grid: width must be < 2^27 and height < 2^24");
    const int W = g->width, H = g->height;
    const size_t n = (size_t)W * H;
    uint8_t mx = 0;
    for (size_t i = 0; i < n; ++i) mx = cells[i] > mx ? cells[i] : mx;
    if (mx > FP_CELL_EXIT) return fail(nullptr, FP_EINVAL, "Grid: unknown cell kind");
    if (g->boundary == FP_BOUNDARY_CLOSED) {
        auto bad = [&](int x, int y) { return cells[(size_t)y * W + x] == FP_CELL_FREE; };
        for (int x = 0; x < W; ++x)
            if (bad(x, 0) || bad(x, H - 1))
                return fail(nullptr, FP_EINVAL, "Grid: closed boundary requires every border cell to be Wall or Exit");
        for (int y = 0; y < H; ++y)
            if (bad(0, y) || bad(W - 1, y))
                return fail(nullptr, FP_EINVAL, "Grid: closed boundary requires every border cell to be Wall or Exit");
    } else {
        for (int x = 0; x < W; ++x)
            if (cells[x] != FP_CELL_WALL || cells[(size_t)(H - 1) * W + x] != FP_CELL_WALL)
                return fail(nullptr, FP_EINVAL, "Grid: periodic-x boundary requires solid top and bottom rows");
    }
    return FP_OK;
}

// ------------------------------------------------------------------------ bitplanes
__global__ void pack_planes_kernel(const uint8_t* cells, int W, int H, int P, uint32_t* wall, uint32_t* ex) {
    FP_PDL_WAIT();
    const size_t nw = (size_t)P * H;
    for (size_t w = blockIdx.x * (size_t)blockDim.x + threadIdx.x; w < nw; w += (size_t)gridDim.x * blockDim.x) {
        const int y = (int)(w / P), x0 = (int)(w % P) * 32 - FP_XPAD_BITS;
        uint32_t bw = 0, be = 0;
        for (int b = 0; b < 32; ++b) {
            const int x = x0 + b;
            if (x < 0 || x >= W) continue;
            const uint8_t k = cells[(size_t)y * W + x];
            bw |= (uint32_t)(k == FP_CELL_WALL) << b;
            be |= (uint32_t)(k == FP_CELL_EXIT) << b;
        }
        wall[w] = bw;
        ex[w] = be;
    }
}

__global__ void sc_set_kernel(DevScalars* sc, long long step, unsigned long long alive) {
    FP_PDL_WAIT();
    sc->step = step;
    sc->alive = alive;
}

__global__ void sc_step_kernel(DevScalars* sc) {
    FP_PDL_WAIT();
    const unsigned long long t = fp_globaltimer();
    sc->move_ns += t - sc->t_plan_end;
    sc->t_step0 = t;
    sc->step += 1;
}

// occupancy from alive positions + make_state checks (state.hpp:46-70)
__global__ void build_occ_kernel(const int32_t* x, const int32_t* y, const uint8_t* alive, uint32_t n,
                                 Geo g, uint32_t* occ, unsigned long long* errs) {
    FP_PDL_WAIT();
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = i < n && alive[i];
    const unsigned cnt = __popc(__ballot_sync(0xffffffffu, live));  // alive count -> errs[3]
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(&errs[3], (unsigned long long)cnt);
    if (!live) return;
    const int ax = g.wrap(x[i]), ay = y[i];
    if (ax < 0 || ax >= g.W || ay < 0 || ay >= g.H) {
        atomicMin(&errs[0], (unsigned long long)i);
        return;
    }
    if (g.is_wall(ax, ay)) {
        atomicMin(&errs[1], (unsigned long long)i);
        return;
    }
    const uint32_t bit = 1u << (ax & 31);
    const uint32_t old = atomicOr(&occ[g.word(ax, ay)], bit);
    if (old & bit) atomicMin(&errs[2], (unsigned long long)i);
}

__global__ void occ_dump_kernel(const int32_t* x, const int32_t* y, const uint8_t* alive, uint32_t n,
                                Geo g, int32_t* out) {
    FP_PDL_WAIT();
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || !alive[i]) return;
    out[(size_t)y[i] * g.W + g.wrap(x[i])] = (int32_t)i;
}

__global__ void u8_from_i32_kernel(const int32_t* in, uint8_t* out, uint32_t n) {
    FP_PDL_WAIT();
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = (uint8_t)in[i];
}

static Geo geo_of(const fp_ctx* c) { return fp_geo(c); }

static void free_agents(fp_ctx* c) {
    void* ptrs[] = {c->d_x, c->d_y, c->d_dx, c->d_dy, c->d_v, c->d_alive, c->d_rank, c->d_alive_ids,
                    c->d_order, c->d_j, c->d_cnt, c->d_off, c->d_cursor, c->d_bucket, c->d_succ,
                    c->d_nxt, c->d_V, c->d_pend_a, c->d_pend_b, c->d_exits, c->d_exits_sorted,
                    c->d_fy_bucket, c->d_flags, c->d_cursor_b, c->d_fallback, c->d_rec_a, c->d_rec_b,
                    c->d_rec0, c->d_entry, c->d_brec};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    c->d_entry = nullptr;
    c->bk_agent_cap = 0;
    c->d_x = c->d_y = c->d_dx = c->d_dy = nullptr;
    c->d_v = c->d_alive = nullptr;
    c->d_rank = c->d_alive_ids = c->d_order = c->d_j = c->d_cnt = c->d_off = c->d_cursor = nullptr;
    c->d_bucket = c->d_succ = c->d_nxt = c->d_V = c->d_pend_a = c->d_pend_b = nullptr;
    c->d_exits = c->d_exits_sorted = nullptr;
    c->d_fy_bucket = c->d_flags = c->d_cursor_b = nullptr;
    c->d_fallback = nullptr;
    c->d_rec_a = c->d_rec_b = c->d_rec0 = nullptr;
    c->d_brec = nullptr;
    c->rec_fresh = false;
    c->cap = 0;
    c->graph_valid = false;
}

static int ensure_agents(fp_ctx* c, uint32_t n) {
    if (n <= c->cap && c->d_x) return FP_OK;
    free_agents(c);
    const size_t m = std::max<uint32_t>(n, 1);
    FP_CUDA(c, cudaMalloc(&c->d_x, m * 4));
    FP_CUDA(c, cudaMalloc(&c->d_y, m * 4));
    FP_CUDA(c, cudaMalloc(&c->d_dx, m * 4));
    FP_CUDA(c, cudaMalloc(&c->d_dy, m * 4));
    FP_CUDA(c, cudaMalloc(&c->d_v, m));
    FP_CUDA(c, cudaMalloc(&c->d_alive, m));
    uint32_t** u32s[] = {&c->d_rank, &c->d_alive_ids, &c->d_order, &c->d_j, &c->d_cnt, &c->d_off,
                         &c->d_cursor, &c->d_bucket, &c->d_succ, &c->d_nxt, &c->d_V, &c->d_pend_a,
                         &c->d_pend_b, &c->d_fy_bucket, &c->d_flags, &c->d_cursor_b};
    for (uint32_t** p : u32s) FP_CUDA(c, cudaMalloc(p, m * 4));
    FP_CUDA(c, cudaMemsetAsync(c->d_cnt, 0, m * 4, c->stream));     // order.cu: zero between shuffles
    FP_CUDA(c, cudaMemsetAsync(c->d_cursor, 0, m * 4, c->stream));
    FP_CUDA(c, cudaMalloc(&c->d_exits, m * 8));
    FP_CUDA(c, cudaMalloc(&c->d_exits_sorted, m * 8));
    FP_CUDA(c, cudaMalloc(&c->d_rec_a, m * sizeof(uint4)));
    FP_CUDA(c, cudaMalloc(&c->d_rec_b, m * sizeof(uint4)));
    FP_CUDA(c, cudaMalloc(&c->d_rec0, m * sizeof(uint4)));
    FP_CUDA(c, cudaMalloc(&c->d_brec, m * sizeof(uint4)));
    FP_CUDA(c, cudaMalloc(&c->d_fallback, m * sizeof(uint2)));
    c->cap = (uint32_t)m;
    c->graph_valid = false;
    return FP_OK;
}

extern "C" int fp_create(const fp_grid_desc* g, const uint8_t* cells, const double* field, int device,
                         fp_ctx** out) {
    if (!out) return fail(nullptr, FP_EINVAL, "fp_create: null output");
    *out = nullptr;
    if (int rc = validate_grid(g, cells)) return rc;
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
        return fail(nullptr, FP_ECUDA, std::string("fp_create: no CUDA device available (") +
                                           cudaGetErrorString(e) + "); there is no CPU fallback");
    if (device < 0 || device >= ndev) return fail(nullptr, FP_EINVAL, "fp_create: bad device ordinal");
    fp_ctx* c = new fp_ctx();
    c->device = device;
    e = cudaSetDevice(device);
    if (e != cudaSuccess) {
        int rc = fp_cuda_fail(c, e, "cudaSetDevice");
        delete c;
        return rc;
    }
    auto bail = [&](int rc) {
        g_error = c->err;
        fp_destroy(c);
        return rc;
    };
    // the critical path (bucketing, plan kernel, motion) outranks the movement-order branch,
    // which fills the gaps beside it (stream priorities carry into the captured graphs)
    int prio_lo = 0, prio_hi = 0;
    cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
#ifdef FP_NO_STREAM_PRIORITY
    prio_hi = prio_lo;
#endif
    if (cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
        cudaStreamCreateWithPriority(&c->stream2, cudaStreamNonBlocking, prio_lo) != cudaSuccess ||
        cudaStreamCreateWithPriority(&c->stream3, cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
        cudaStreamCreateWithPriority(&c->stream4, cudaStreamNonBlocking, prio_lo) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_sfork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_sjoin, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_bfork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_bjoin, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming) != cudaSuccess)
        return bail(fp_cuda_fail(c, cudaGetLastError(), "cudaStreamCreate"));
    cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
    if (const char* e2 = getenv("FP_NO_TMA")) c->use_tma = (e2[0] == '1') ? 0 : 1;
    if (const char* e3 = getenv("FP_DEAL_PASSES")) c->deal_passes = std::max(1, std::min(DEAL_PASSES, atoi(e3)));
    c->W = g->width;
    c->H = g->height;
    c->boundary = g->boundary;
    c->cell_size = g->cell_size;
    c->P = (((c->W + 2 * FP_XPAD_BITS + 31) / 32) + 3) & ~3;  // 16-byte row pitch (TMA)
    c->PW = ((c->W + 2 * FP_XPAD_W) + 3) & ~3;
    const size_t ncell = (size_t)c->W * c->H;
    const size_t nwords = (size_t)c->P * c->H;
    if (cudaMalloc(&c->d_wall, nwords * 4) || cudaMalloc(&c->d_exit, nwords * 4) ||
        cudaMalloc(&c->d_occ, nwords * 4) || cudaMalloc(&c->d_field, ncell * 8) ||
        cudaMalloc(&c->d_counters, 16 * sizeof(unsigned long long)) ||
        cudaMallocHost(&c->h_counters, 16 * sizeof(unsigned long long)) ||
        cudaMalloc(&c->d_sc, sizeof(DevScalars)) || cudaMallocHost(&c->h_sc, sizeof(DevScalars)))
        return bail(fp_cuda_fail(c, cudaGetLastError(), "cudaMalloc(grid)"));
    uint8_t* d_cells = nullptr;
    if (cudaMalloc(&d_cells, ncell) != cudaSuccess)
        return bail(fp_cuda_fail(c, cudaGetLastError(), "cudaMalloc(cells)"));
    cudaMemcpyAsync(d_cells, cells, ncell, cudaMemcpyHostToDevice, c->stream);
    cudaMemsetAsync(c->d_sc, 0, sizeof(DevScalars), c->stream);
    cudaMemsetAsync(c->d_counters, 0, 16 * sizeof(unsigned long long), c->stream);
    fp_launch(pack_planes_kernel, 1184, 256, 0, c->stream, d_cells, c->W, c->H, c->P, c->d_wall, c->d_exit);
    c->ctr.kernel_launches++;
    fp_ghost_static(c);
    cudaMemsetAsync(c->d_occ, 0, nwords * 4, c->stream);
    int rc = FP_OK;
    if (field) {
        cudaMemcpyAsync(c->d_field, field, ncell * 8, cudaMemcpyHostToDevice, c->stream);
    } else {
        rc = fp_field_compute(c, d_cells);
    }
    e = cudaStreamSynchronize(c->stream);
    cudaFree(d_cells);
    if (rc != FP_OK) return bail(rc);
    if (e != cudaSuccess) return bail(fp_cuda_fail(c, e, "fp_create"));
    *out = c;
    return FP_OK;
}

extern "C" void fp_destroy(fp_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    free_agents(c);
    if (c->stream2) cudaStreamSynchronize(c->stream2);
    if (c->stream3) cudaStreamSynchronize(c->stream3);
    if (c->stream4) cudaStreamSynchronize(c->stream4);
    if (c->graph_plan) cudaGraphExecDestroy(c->graph_plan);
    if (c->graph_move) cudaGraphExecDestroy(c->graph_move);
    if (c->graph_multi) cudaGraphExecDestroy(c->graph_multi);
    if (c->st.graph_fin) cudaGraphExecDestroy(c->st.graph_fin);
    fp_strip_nccl_destroy(c);
    {
        StripCtx& S = c->st;
        void* sp[] = {S.d_owned, S.d_dplane, S.d_dflag, S.d_clist, S.d_send, S.d_recv, S.d_hkey, S.d_hres,
                      S.d_hocc, S.d_rslot, S.d_plist, S.d_rexits, S.d_rhdr};
        for (void* p : sp)
            if (p) cudaFree(p);
        if (S.h_rhdr) cudaFreeHost(S.h_rhdr);
        if (S.h_send) cudaFreeHost(S.h_send);
        if (S.h_recv) cudaFreeHost(S.h_recv);
        if (S.ev) cudaEventDestroy(S.ev);
    }
    void* ptrs[] = {c->d_wall, c->d_exit, c->d_occ, c->d_field, c->d_counters, c->d_temp, c->d_temp_b,
                    c->d_plane, c->d_plane_t, c->d_tile_cnt, c->d_tile_off, c->d_tile_list, c->d_sub_cnt, c->d_sub_off, c->d_tile_deal, c->d_tile_exit, c->d_seed_items, c->d_plan_items, c->d_scan_sums, c->d_scan_sums2,
                    c->d_sc,
                    c->d_p1, c->d_p2,
                    c->d_bkt, c->d_bdone, c->d_pw};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    if (c->h_counters) cudaFreeHost(c->h_counters);
    if (c->d_scratch_small) cudaFree(c->d_scratch_small);
    if (c->h_scratch_small) cudaFreeHost(c->h_scratch_small);
    if (c->h_sc) cudaFreeHost(c->h_sc);
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    if (c->stream2) cudaStreamDestroy(c->stream2);
    if (c->stream3) cudaStreamDestroy(c->stream3);
    if (c->stream4) cudaStreamDestroy(c->stream4);
    if (c->ev_sfork) cudaEventDestroy(c->ev_sfork);
    if (c->ev_sjoin) cudaEventDestroy(c->ev_sjoin);
    if (c->d_scan_sums3) cudaFree(c->d_scan_sums3);
    if (c->ev_bfork) cudaEventDestroy(c->ev_bfork);
    if (c->ev_bjoin) cudaEventDestroy(c->ev_bjoin);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

extern "C" int fp_static_field(const fp_grid_desc* g, const uint8_t* cells, int device, double* out) {
    fp_ctx* c = nullptr;
    if (int rc = fp_create(g, cells, nullptr, device, &c)) return rc;
    int rc = fp_get_field(c, out);
    fp_destroy(c);
    return rc;
}

extern "C" int fp_get_field(const fp_ctx* cc, double* out) {
    fp_ctx* c = const_cast<fp_ctx*>(cc);
    if (!c || !out) return fail(c, FP_EINVAL, "fp_get_field: null argument");
    cudaSetDevice(c->device);
    FP_CUDA(c, cudaMemcpyAsync(out, c->d_field, (size_t)c->W * c->H * 8, cudaMemcpyDeviceToHost, c->stream));
    FP_CUDA(c, cudaStreamSynchronize(c->stream));
    return FP_OK;
}

// host mirror (step, alive) -> device scalars; skipped when the device already holds them (the
// last read_scalars or sync_scalars left them there and the host has not changed them since)
static int sync_scalars(fp_ctx* c) {
    if (c->dev_step == c->step && c->dev_alive == c->alive) return FP_OK;
    fp_launch(sc_set_kernel, 1, 1, 0, c->stream, c->d_sc, (long long)c->step, (unsigned long long)c->alive);
    FP_LAUNCHED(c);
    c->dev_step = c->step;
    c->dev_alive = c->alive;
    return FP_OK;
}

// device scalars -> host mirror, after a sync
static int read_scalars(fp_ctx* c) {
    FP_CUDA(c, cudaMemcpyAsync(c->h_sc, c->d_sc, sizeof(DevScalars), cudaMemcpyDeviceToHost, c->stream));
    FP_CUDA(c, cudaStreamSynchronize(c->stream));
    if (c->h_sc->err) {
        const unsigned long long e = c->h_sc->err;
        cudaMemsetAsync(&c->d_sc->err, 0, 8, c->stream);
        return fail(c, FP_ECUDA, "device-side scheduler fault (flags " + std::to_string(e) +
                                     "): a plan/motion wait timed out");
    }
    c->alive = (int64_t)c->h_sc->alive;
    c->step = (int64_t)c->h_sc->step;
    c->dev_step = c->step;
    c->dev_alive = c->alive;
    c->ctr.plan_fallbacks = (int64_t)c->h_sc->fallbacks;
    c->ctr.motion_rounds = (int64_t)c->h_sc->pad[1];
    const unsigned long long* tm = c->h_sc->t_motion;
    if (tm[3] >= tm[2] && tm[2] >= tm[1] && tm[1] >= tm[0] && tm[0]) {
        c->ctr.motion_seed_ns = (int64_t)(tm[1] - tm[0]);
        c->ctr.motion_grid_ns = (int64_t)(tm[2] - tm[1]);
        c->ctr.motion_tail_ns = (int64_t)(tm[3] - tm[2]);
        const unsigned long long tk = c->h_sc->t_marked;
        c->ctr.motion_mark_ns = tk >= tm[0] && tk <= tm[1] ? (int64_t)(tk - tm[0]) : 0;
    }
    c->ctr.motion_contended = (int64_t)c->h_sc->contended;
    {
        const unsigned long long tp = c->h_sc->t_prep;
        c->ctr.motion_prep_ns = tp >= tm[1] && tp <= tm[2] ? (int64_t)(tp - tm[1]) : 0;
    }
    c->ctr.motion_grid_rounds = (int64_t)c->h_sc->grid_rounds;
    return FP_OK;
}

static int upload_agents(fp_ctx* c, const int32_t* x, const int32_t* y, const uint8_t* alive) {
    cudaStream_t s = c->stream;
    const uint32_t n = c->n;
    FP_CUDA(c, cudaMemcpyAsync(c->d_x, x, (size_t)n * 4, cudaMemcpyHostToDevice, s));
    FP_CUDA(c, cudaMemcpyAsync(c->d_y, y, (size_t)n * 4, cudaMemcpyHostToDevice, s));
    if (alive)
        FP_CUDA(c, cudaMemcpyAsync(c->d_alive, alive, n, cudaMemcpyHostToDevice, s));
    else
        FP_CUDA(c, cudaMemsetAsync(c->d_alive, 1, n, s));
    FP_CUDA(c, cudaMemsetAsync(c->d_occ, 0, (size_t)c->P * c->H * 4, s));
    // [0..2] first failing agent per make_state check (state.hpp:46-70), [3] alive count
    FP_CUDA(c, cudaMemsetAsync(c->d_counters + 8, 0xFF, 3 * 8, s));
    FP_CUDA(c, cudaMemsetAsync(c->d_counters + 11, 0, 8, s));
    if (n) {
        fp_launch(build_occ_kernel, fp_blocks(n, 256), 256, 0, s, c->d_x, c->d_y, c->d_alive, n, geo_of(c), c->d_occ,
                                                            c->d_counters + 8);
        FP_LAUNCHED(c);
    }
    FP_CUDA(c, cudaMemcpyAsync(c->h_counters + 8, c->d_counters + 8, 4 * 8, cudaMemcpyDeviceToHost, s));
    FP_CUDA(c, cudaStreamSynchronize(s));
    const unsigned long long* e = c->h_counters + 8;
    // the device roster and occupancy are already replaced: a rejected roster poisons the context
    // until the next successful upload (compute calls fail instead of running on a half state)
    c->poisoned = e[0] != ~0ull || e[1] != ~0ull || e[2] != ~0ull;
    if (e[0] != ~0ull) return fail(c, FP_EINVAL, "make_state: agent " + std::to_string(e[0]) + " is out of bounds");
    if (e[1] != ~0ull) return fail(c, FP_EINVAL, "make_state: agent " + std::to_string(e[1]) + " placed on a Wall cell");
    if (e[2] != ~0ull) return fail(c, FP_EINVAL, "make_state: agent " + std::to_string(e[2]) + " shares a cell");
    c->alive = (int64_t)e[3];
    c->bucket_fresh = false;
    c->rec_fresh = false;
    if (int rc = fp_ghost_occ(c)) return rc;
    if (c->st.on) {  // a strip rank owns the alive agents standing in its columns
        if (int rc = fp_strip_reserve(c)) return rc;
        if (int rc = fp_strip_owned_init(c)) return rc;
    }
    return sync_scalars(c);
}

extern "C" int fp_set_agents(fp_ctx* c, uint32_t n, const int32_t* x, const int32_t* y, const int32_t* v_max,
                             const uint8_t* alive, int64_t step) {
    if (!c) return fail(nullptr, FP_EINVAL, "fp_set_agents: null context");
    if (n && (!x || !y || !v_max)) return fail(c, FP_EINVAL, "fp_set_agents: null roster arrays");
    bool mixed = false;
    for (uint32_t i = 0; i < n; ++i) {
        if (v_max[i] < 1 || v_max[i] > 5) return fail(c, FP_EINVAL, "make_state: v_max must be in [1,5]");
        mixed |= v_max[i] != v_max[0];
    }
    const int vu = (n && !mixed) ? v_max[0] : 5;
    if (mixed != c->mixed_v || vu != c->v_uniform) c->graph_valid = false;  // the plan kernel variant changes
    c->mixed_v = mixed;
    c->v_uniform = vu;
    cudaSetDevice(c->device);
    if (int rc = ensure_agents(c, n)) return rc;
    c->n = n;
    c->step = step;
    c->n_order = 0;
    c->n_exits = 0;
    if (n) {
        int32_t* d_tmp = c->d_dx;  // stage v_max as i32, convert to u8
        FP_CUDA(c, cudaMemcpyAsync(d_tmp, v_max, (size_t)n * 4, cudaMemcpyHostToDevice, c->stream));
        fp_launch(u8_from_i32_kernel, fp_blocks(n, 256), 256, 0, c->stream, d_tmp, c->d_v, n);
        FP_LAUNCHED(c);
    }
    if (int rc = upload_agents(c, x, y, alive)) return rc;
    // desired = pos for alive agents (state.hpp:74)
    FP_CUDA(c, cudaMemcpyAsync(c->d_dx, c->d_x, (size_t)n * 4, cudaMemcpyDeviceToDevice, c->stream));
    FP_CUDA(c, cudaMemcpyAsync(c->d_dy, c->d_y, (size_t)n * 4, cudaMemcpyDeviceToDevice, c->stream));
    return FP_OK;
}

extern "C" int fp_update_agents(fp_ctx* c, const int32_t* x, const int32_t* y, const uint8_t* alive) {
    if (!c) return fail(nullptr, FP_EINVAL, "fp_update_agents: null context");
    cudaSetDevice(c->device);
    return upload_agents(c, x, y, alive);
}

extern "C" int fp_set_step(fp_ctx* c, int64_t step) {
    if (!c) return fail(nullptr, FP_EINVAL, "null context");
    c->step = step;
    return sync_scalars(c);
}
extern "C" int fp_get_step(const fp_ctx* c, int64_t* step) {
    if (!c || !step) return fail(nullptr, FP_EINVAL, "null argument");
    *step = c->step;
    return FP_OK;
}
extern "C" int fp_get_last_dx(const fp_ctx* c, int64_t* dx) {
    if (!c || !dx) return fail(nullptr, FP_EINVAL, "null argument");
    *dx = c->last_dx;
    return FP_OK;
}
extern "C" int fp_get_run_dx(const fp_ctx* c, int64_t* dx) {
    if (!c || !dx) return fail(nullptr, FP_EINVAL, "null argument");
    *dx = (int64_t)c->h_sc->tot_dx;
    return FP_OK;
}
extern "C" int fp_get_alive_count(const fp_ctx* c, int64_t* a) {
    if (!c || !a) return fail(nullptr, FP_EINVAL, "null argument");
    *a = c->alive;
    return FP_OK;
}

extern "C" int fp_set_potential(fp_ctx* c, int kind, double g) {
    if (!c) return fail(nullptr, FP_EINVAL, "null context");
    if (kind != FP_POTENTIAL_EXIT_DISTANCE && kind != FP_POTENTIAL_DRIVE_X)
        return fail(c, FP_EINVAL, "fp_set_potential: unknown potential");
    // the plan graphs bake the potential and gradient into their kernel arguments
    if (kind != c->potential || g != c->drive_gradient) c->graph_valid = false;
    c->potential = kind;
    c->drive_gradient = g;
    return FP_OK;
}

extern "C" int fp_set_desired(fp_ctx* c, const int32_t* x, const int32_t* y) {
    if (!c) return fail(nullptr, FP_EINVAL, "null context");
    cudaSetDevice(c->device);
    FP_CUDA(c, cudaMemcpyAsync(c->d_dx, x, (size_t)c->n * 4, cudaMemcpyHostToDevice, c->stream));
    FP_CUDA(c, cudaMemcpyAsync(c->d_dy, y, (size_t)c->n * 4, cudaMemcpyHostToDevice, c->stream));
    c->rec_fresh = false;  // the plan's walk records no longer describe the desired cells
    FP_CUDA(c, cudaStreamSynchronize(c->stream));
    return FP_OK;
}

static int check_usable(fp_ctx* c) {
    if (c->poisoned)
        return fail(c, FP_EINVAL, "state invalid: the last agent upload was rejected; upload a valid roster first");
    return FP_OK;
}

// Allocations / setup of every stage for (k_s): never inside a graph capture.
static int prepare(fp_ctx* c, double k_s) {
    if (int rc = fp_plan_prepare(c, k_s)) return rc;
    if (int rc = fp_order_reserve(c)) return rc;
    if (int rc = fp_ensure_res(c)) return rc;
    if (int rc = fp_strip_reserve(c)) return rc;
    return FP_OK;
}

static int strip_step(fp_ctx* c, double k_s, uint64_t seed, fp_step_stats* out);
static int strip_run(fp_ctx* c, double k_s, uint64_t seed, int32_t steps, fp_run_stats* out);

extern "C" int fp_plan(fp_ctx* c, double k_s, uint64_t seed) {
    if (!c) return fail(nullptr, FP_EINVAL, "null context");
    if (int rc = check_usable(c)) return rc;
    if (c->st.on) return fail(c, FP_EINVAL, "plan_phase on a strip rank: the decomposed step is fp_step / fp_run");
    cudaSetDevice(c->device);
    if (c->alive == 0) return FP_OK;  // engine.hpp:73
    if (int rc = prepare(c, k_s)) return rc;
    if (int rc = sync_scalars(c)) return rc;
    if (int rc = fp_plan_launch(c, k_s, seed)) return rc;
    c->ctr.planned_agents += c->alive;
    return read_scalars(c);
}

// order + motion on the main stream (API path), then the exit list in processing order.
static int move_impl(fp_ctx* c, uint64_t seed, fp_step_stats* out) {
    if (int rc = fp_order_reserve(c)) return rc;
    if (int rc = fp_ensure_res(c)) return rc;
    const int64_t alive0 = c->alive;
    if (int rc = sync_scalars(c)) return rc;
    if (int rc = fp_order_launch(c, seed, c->stream)) return rc;
    if (int rc = fp_motion_launch(c, c->bucket_fresh)) return rc;
    c->bucket_fresh = false;
    if (int rc = read_scalars(c)) return rc;
    c->n_order = (uint32_t)c->h_sc->n_alive;
    c->n_exits = (uint32_t)c->h_sc->n_exits;
    c->last_displacement = (int64_t)c->h_sc->disp;
    c->last_dx = (int64_t)c->h_sc->step_dx;
    if (int rc = fp_exits_finish(c)) return rc;
    FP_CUDA(c, cudaStreamSynchronize(c->stream));
    if (out) {
        out->alive = c->alive;
        out->exited = alive0 - c->alive;
        out->displacement_cells = c->last_displacement;
    }
    return FP_OK;
}

extern "C" int fp_move(fp_ctx* c, uint64_t seed, fp_step_stats* out) {
    if (!c) return fail(nullptr, FP_EINVAL, "null context");
    if (int rc = check_usable(c)) return rc;
    if (c->st.on) return fail(c, FP_EINVAL, "move_phase on a strip rank: the decomposed step is fp_step / fp_run");
    cudaSetDevice(c->device);
    return move_impl(c, seed, out);
}

static int capture(fp_ctx* c, double k_s, uint64_t seed);

// step(): one replay of the run() graphs (plan with the order on a forked stream, then motion and
// the step advance), one host sync, then the exit list in processing order.
extern "C" int fp_step(fp_ctx* c, double k_s, uint64_t seed, fp_step_stats* out) {
    if (!c) return fail(nullptr, FP_EINVAL, "null context");
    if (int rc = check_usable(c)) return rc;
    cudaSetDevice(c->device);
    if (c->st.on) return strip_step(c, k_s, seed, out);
    if (c->alive == 0 || c->n == 0) {  // engine.hpp:73: nothing to plan or move
        c->n_order = 0;
        c->n_exits = 0;
        c->last_displacement = 0;
        c->last_dx = 0;
        c->step++;
        if (out) *out = fp_step_stats{c->alive, 0, 0};
        return sync_scalars(c);
    }
    if (int rc = prepare(c, k_s)) return rc;
    if (!c->graph_valid || c->graph_ks != k_s || c->graph_seed != seed)
        if (int rc = capture(c, k_s, seed)) return rc;
    const int64_t alive0 = c->alive;
    if (int rc = sync_scalars(c)) return rc;
    FP_CUDA(c, cudaGraphLaunch(c->graph_plan, c->stream));
    FP_CUDA(c, cudaGraphLaunch(c->graph_move, c->stream));
    c->ctr.kernel_launches += c->launches_per_step;
    if (int rc = read_scalars(c)) return rc;
    c->ctr.planned_agents += alive0;
    c->n_order = (uint32_t)c->h_sc->n_alive;
    c->n_exits = (uint32_t)c->h_sc->n_exits;
    c->last_displacement = (int64_t)c->h_sc->disp;
    c->last_dx = (int64_t)c->h_sc->step_dx;
    if (int rc = fp_exits_finish(c)) return rc;
    if (out) {
        out->alive = c->alive;
        out->exited = alive0 - c->alive;
        out->displacement_cells = c->last_displacement;
    }
    return FP_OK;
}

// Captures the two per-step graphs: plan phase = bucketing + plan kernel, with the movement
// order (alive compaction + parallel Fisher-Yates) on a forked branch; move phase = motion
// rounds + ghost refresh + step advance.
// run() replays FP_RUN_UNROLL steps per graph launch: the plan and move graphs as alternating
// child-graph nodes of one graph, so consecutive phases meet at a graph edge instead of a host
// graph launch.  The plan/move split then comes from the device clock (move_begin_kernel and
// sc_step_kernel stamp the phase boundaries).  FASTPED_RUN_UNROLL=1 keeps one launch per phase.
static int run_unroll() {
    static const int u = [] {
        const char* e = getenv("FASTPED_RUN_UNROLL");
        const int v = e ? atoi(e) : FP_RUN_UNROLL;
        return std::max(1, std::min(64, v));
    }();
    return u;
}

static cudaError_t build_multi(fp_ctx* c, cudaGraph_t gp, cudaGraph_t gm) {
    const int u = run_unroll();
    if (u < 2) return cudaSuccess;
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaGraphCreate(&g, 0);
    cudaGraphNode_t prev = nullptr;
    for (int k = 0; k < u && e == cudaSuccess; ++k)
        for (cudaGraph_t child : {gp, gm}) {
            cudaGraphNode_t nd = nullptr;
            e = cudaGraphAddChildGraphNode(&nd, g, prev ? &prev : nullptr, prev ? 1 : 0, child);
            if (e != cudaSuccess) break;
            prev = nd;
        }
    if (e == cudaSuccess) e = cudaGraphInstantiate(&c->graph_multi, g, 0);
    if (g) cudaGraphDestroy(g);
    if (e == cudaSuccess) c->run_unroll = u;
    return e;
}

static int capture(fp_ctx* c, double k_s, uint64_t seed) {
    if (c->graph_plan) cudaGraphExecDestroy(c->graph_plan);
    if (c->graph_move) cudaGraphExecDestroy(c->graph_move);
    if (c->st.graph_fin) cudaGraphExecDestroy(c->st.graph_fin);
    if (c->graph_multi) cudaGraphExecDestroy(c->graph_multi);
    c->graph_plan = c->graph_move = c->st.graph_fin = c->graph_multi = nullptr;
    c->run_unroll = 0;
    const bool strip = c->st.on;
    cudaGraph_t g = nullptr;
    const int64_t k0 = c->ctr.kernel_launches;
    FP_CUDA(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    int rc = FP_OK;
    if (strip) rc = fp_strip_begin_launch(c);
#ifdef FP_ORDER_SERIAL  // A/B experiments: the movement order after the plan, same stream
    if (rc == FP_OK) rc = fp_plan_launch(c, k_s, seed);
    if (rc == FP_OK) rc = fp_order_launch(c, seed, c->stream);
#else
    cudaEventRecord(c->ev_fork, c->stream);
    cudaStreamWaitEvent(c->stream2, c->ev_fork, 0);
    if (rc == FP_OK) rc = fp_order_launch(c, seed, c->stream2);
    cudaEventRecord(c->ev_join, c->stream2);
    // the order branch runs beside bucketing + plan kernel and joins before the motion (joining
    // before the plan kernel instead was measured slower: the branch takes ~140 us)
#ifdef FP_ORDER_JOIN_EARLY
    if (rc == FP_OK) rc = fp_plan_launch(c, k_s, seed, c->ev_join);
#else
    if (rc == FP_OK) rc = fp_plan_launch(c, k_s, seed);
#endif
    cudaStreamWaitEvent(c->stream, c->ev_join, 0);
    FP_STAMP(c, c->stream, 7);
#endif
    cudaError_t e = cudaStreamEndCapture(c->stream, &g);
    if (rc != FP_OK) {
        if (g) cudaGraphDestroy(g);
        return rc;
    }
    if (e != cudaSuccess) return fp_cuda_fail(c, e, "capture(plan)");
    e = cudaGraphInstantiate(&c->graph_plan, g, 0);
    cudaGraph_t g_plan = g;  // kept for the unrolled run graph
    if (e != cudaSuccess) {
        cudaGraphDestroy(g_plan);
        return fp_cuda_fail(c, e, "instantiate(plan)");
    }
    g = nullptr;
    FP_CUDA(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    if (strip) rc = fp_strip_defer_launch(c);  // band-connected walks leave the local motion
    if (rc == FP_OK) rc = fp_motion_launch(c, c->bucket_fresh);  // the plan graph re-buckets every step
    c->bucket_fresh = false;
    if (rc == FP_OK && strip) rc = fp_strip_pack_launch(c);
    if (rc == FP_OK && !strip) {
        fp_launch(sc_step_kernel, 1, 1, 0, c->stream, c->d_sc);
        c->ctr.kernel_launches++;
    }
    e = cudaStreamEndCapture(c->stream, &g);
    if (rc != FP_OK) {
        if (g) cudaGraphDestroy(g);
        cudaGraphDestroy(g_plan);
        return rc;
    }
    if (e != cudaSuccess) {
        cudaGraphDestroy(g_plan);
        return fp_cuda_fail(c, e, "capture(move)");
    }
    e = cudaGraphInstantiate(&c->graph_move, g, 0);
    if (e == cudaSuccess && !strip) e = build_multi(c, g_plan, g);
    cudaGraphDestroy(g);
    cudaGraphDestroy(g_plan);
    if (e != cudaSuccess) return fp_cuda_fail(c, e, "instantiate(move)");
    if (strip) {  // after the exchange: resolve the deferred walks, global exits, ++step
        g = nullptr;
        FP_CUDA(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        rc = fp_strip_resolve_launch(c);
        if (rc == FP_OK) rc = fp_exits_sort_launch(c);
        if (rc == FP_OK) rc = fp_ghost_occ(c);
        if (rc == FP_OK) {
            fp_launch(sc_step_kernel, 1, 1, 0, c->stream, c->d_sc);
            c->ctr.kernel_launches++;
        }
        e = cudaStreamEndCapture(c->stream, &g);
        if (rc != FP_OK) {
            if (g) cudaGraphDestroy(g);
            return rc;
        }
        if (e != cudaSuccess) return fp_cuda_fail(c, e, "capture(strip)");
        e = cudaGraphInstantiate(&c->st.graph_fin, g, 0);
        cudaGraphDestroy(g);
        if (e != cudaSuccess) return fp_cuda_fail(c, e, "instantiate(strip)");
    }
    c->launches_per_step = c->ctr.kernel_launches - k0;  // captured, not yet executed
    c->ctr.kernel_launches = k0;
    c->graph_valid = true;
    c->graph_ks = k_s;
    c->graph_seed = seed;
    return FP_OK;
}

__global__ void run_begin_kernel(DevScalars* sc) {
    FP_PDL_WAIT();
    sc->tot_exits = 0;
    sc->tot_disp = 0;
    sc->tot_dx = 0;
    sc->tot_updates = 0;
    sc->plan_ns = sc->move_ns = 0;
    sc->t_step0 = fp_globaltimer();
}

static int run_finish(fp_ctx* c, int32_t steps, double wall_s, double plan_s, double move_s, fp_run_stats* out) {
    if (int rc = read_scalars(c)) return rc;
    fp_run_stats rs{};
    rs.wall_time_s = wall_s;
    rs.plan_time_s = plan_s >= 0 ? plan_s : (double)c->h_sc->plan_ns * 1e-9;
    rs.move_time_s = move_s >= 0 ? move_s : (double)c->h_sc->move_ns * 1e-9;
    rs.steps = steps;
    rs.exited = (int64_t)c->h_sc->tot_exits;
    rs.displacement_cells = (int64_t)c->h_sc->tot_disp;
    rs.agent_updates = (int64_t)c->h_sc->tot_updates;
    rs.alive = c->alive;
    c->n_order = (uint32_t)c->h_sc->n_alive;
    c->n_exits = 0;  // the per-phase exit list is only kept by fp_move / fp_step
    c->ctr.planned_agents += rs.agent_updates;
    if (out) *out = rs;
    return FP_OK;
}

// run() over the unrolled graph: events around the whole loop only.
static int run_unrolled(fp_ctx* c, int32_t steps, fp_run_stats* out) {
    cudaEvent_t e0, e1;
    FP_CUDA(c, cudaEventCreate(&e0));
    FP_CUDA(c, cudaEventCreate(&e1));
    cudaEventRecord(e0, c->stream);
    int s = 0;
    for (; s + c->run_unroll <= steps; s += c->run_unroll) FP_CUDA(c, cudaGraphLaunch(c->graph_multi, c->stream));
    for (; s < steps; ++s) {
        FP_CUDA(c, cudaGraphLaunch(c->graph_plan, c->stream));
        FP_CUDA(c, cudaGraphLaunch(c->graph_move, c->stream));
    }
    cudaEventRecord(e1, c->stream);
    FP_CUDA(c, cudaEventSynchronize(e1));
    c->ctr.kernel_launches += (int64_t)steps * c->launches_per_step;
    float tot = 0;
    cudaEventElapsedTime(&tot, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return run_finish(c, steps, tot * 1e-3, -1.0, -1.0, out);
}

// run(): `steps` steps as graph replays, CUDA events between phases; one host sync at the end.
extern "C" int fp_run(fp_ctx* c, double k_s, uint64_t seed, int32_t steps, fp_run_stats* out) {
    if (!c) return fail(nullptr, FP_EINVAL, "null context");
    if (int rc = check_usable(c)) return rc;
    if (steps < 1) return fail(c, FP_EINVAL, "SimParams: steps must be >= 1");
    cudaSetDevice(c->device);
    if (c->st.on) return strip_run(c, k_s, seed, steps, out);
    if (int rc = prepare(c, k_s)) return rc;
    if (!c->graph_valid || c->graph_ks != k_s || c->graph_seed != seed)
        if (int rc = capture(c, k_s, seed)) return rc;
    if (int rc = sync_scalars(c)) return rc;
    fp_launch(run_begin_kernel, 1, 1, 0, c->stream, c->d_sc);
    FP_LAUNCHED(c);
    const int64_t launches_per_step = 0;  // counted at capture; see fp_counters note
    (void)launches_per_step;
    if (c->graph_multi && c->run_unroll > 1) return run_unrolled(c, steps, out);
    std::vector<cudaEvent_t> ev((size_t)2 * steps + 1);
    for (auto& e : ev) FP_CUDA(c, cudaEventCreate(&e));
    const int64_t k0 = c->ctr.kernel_launches;
    for (int s = 0; s < steps; ++s) {
        cudaEventRecord(ev[2 * s], c->stream);
        FP_CUDA(c, cudaGraphLaunch(c->graph_plan, c->stream));
        cudaEventRecord(ev[2 * s + 1], c->stream);
        FP_CUDA(c, cudaGraphLaunch(c->graph_move, c->stream));
    }
    cudaEventRecord(ev[2 * steps], c->stream);
    FP_CUDA(c, cudaEventSynchronize(ev[2 * steps]));
    (void)k0;
    c->ctr.kernel_launches += (int64_t)steps * c->launches_per_step;
    fp_run_stats rs{};
    float plan_ms = 0, move_ms = 0, tot = 0;
    for (int s = 0; s < steps; ++s) {
        float a = 0, b = 0;
        cudaEventElapsedTime(&a, ev[2 * s], ev[2 * s + 1]);
        cudaEventElapsedTime(&b, ev[2 * s + 1], ev[2 * s + 2]);
        plan_ms += a;
        move_ms += b;
    }
    cudaEventElapsedTime(&tot, ev[0], ev[2 * steps]);
    for (auto& e : ev) cudaEventDestroy(e);
    if (int rc = read_scalars(c)) return rc;
    rs.wall_time_s = tot * 1e-3;
    rs.plan_time_s = plan_ms * 1e-3;
    rs.move_time_s = move_ms * 1e-3;
    rs.steps = steps;
    rs.exited = (int64_t)c->h_sc->tot_exits;
    rs.displacement_cells = (int64_t)c->h_sc->tot_disp;
    rs.agent_updates = (int64_t)c->h_sc->tot_updates;
    rs.alive = c->alive;
    c->n_order = (uint32_t)c->h_sc->n_alive;
    c->n_exits = 0;  // the per-phase exit list is only kept by fp_move / fp_step
    c->ctr.planned_agents += rs.agent_updates;
    if (out) *out = rs;
    return FP_OK;
}

// ------------------------------------------------------------------ multi-GPU x strips
extern "C" int fp_strip_bounds(int32_t width, int rank, int nranks, int32_t* lo, int32_t* hi) {
    if (width < 1 || nranks < 1 || rank < 0 || rank >= nranks || !lo || !hi)
        return fail(nullptr, FP_EINVAL, "fp_strip_bounds: need width >= 1 and 0 <= rank < nranks");
    *lo = (int32_t)((int64_t)rank * width / nranks);
    *hi = (int32_t)((int64_t)(rank + 1) * width / nranks);
    return FP_OK;
}

extern "C" int fp_strip_config(fp_ctx* c, int rank, int nranks, int32_t x_lo, int32_t x_hi, uint32_t cap_def,
                               uint32_t cap_exit) {
    if (!c) return fail(nullptr, FP_EINVAL, "null context");
    if (nranks < 1 || nranks > 64 || rank < 0 || rank >= nranks)
        return fail(c, FP_EINVAL, "fp_strip_config: need 1 <= nranks <= 64 and 0 <= rank < nranks");
    if (x_lo < 0 || x_hi > c->W || x_lo >= x_hi) return fail(c, FP_EINVAL, "fp_strip_config: need 0 <= x_lo < x_hi <= width");
    if (c->boundary == FP_BOUNDARY_PERIODIC_X && c->W < 16)
        return fail(c, FP_EINVAL, "fp_strip_config: periodic grids narrower than 16 columns are not decomposed");
    StripCtx& S = c->st;
    S.on = true;
    S.rank = rank;
    S.nranks = nranks;
    S.x_lo = x_lo;
    S.x_hi = x_hi;
    S.cap_def_req = cap_def;
    S.cap_exit_req = cap_exit;
    S.cap_agents = 0;  // re-reserve with the new sizes
    if (!S.ev) FP_CUDA(c, cudaEventCreateWithFlags(&S.ev, cudaEventDisableTiming));
    c->graph_valid = false;
    cudaSetDevice(c->device);
    if (int rc = fp_strip_reserve(c)) return rc;
    if (int rc = fp_strip_owned_init(c)) return rc;
    FP_CUDA(c, cudaStreamSynchronize(c->stream));
    return FP_OK;
}

extern "C" int fp_strip_set_nccl(fp_ctx* c, const fp_nccl_id* id) {
    if (!c || !id) return fail(c, FP_EINVAL, "null argument");
    if (!c->st.on) return fail(c, FP_EINVAL, "fp_strip_set_nccl: configure the strip first (fp_strip_config)");
    fp_strip_nccl_destroy(c);
    if (int rc = fp_strip_nccl_init(c, id)) return rc;
    c->st.transport = FP_STRIP_NCCL;
    c->st.cap_agents = 0;
    return fp_strip_reserve(c);
}

extern "C" int fp_strip_set_exchange(fp_ctx* c, fp_allgather_fn fn, void* user) {
    if (!c || !fn) return fail(c, FP_EINVAL, "null argument");
    if (!c->st.on) return fail(c, FP_EINVAL, "fp_strip_set_exchange: configure the strip first (fp_strip_config)");
    c->st.transport = FP_STRIP_HOST;
    c->st.host_fn = fn;
    c->st.host_user = user;
    c->st.cap_agents = 0;  // pinned staging buffers
    cudaSetDevice(c->device);
    return fp_strip_reserve(c);
}

extern "C" int fp_strip_get_owned(const fp_ctx* cc, uint8_t* owned) {
    fp_ctx* c = const_cast<fp_ctx*>(cc);
    if (!c || !owned) return fail(c, FP_EINVAL, "null argument");
    if (!c->st.on) return fail(c, FP_EINVAL, "not a strip context");
    cudaSetDevice(c->device);
    if (c->n) FP_CUDA(c, cudaMemcpyAsync(owned, c->st.d_owned, c->n, cudaMemcpyDeviceToHost, c->stream));
    FP_CUDA(c, cudaStreamSynchronize(c->stream));
    return FP_OK;
}

// Everything a strip step needs, outside any capture; (re)captures the three step graphs.
static int strip_ready(fp_ctx* c, double k_s, uint64_t seed) {
    if (!c->st.on) return fail(c, FP_EINVAL, "not a strip context");
    if (!fp_plan_tiled(c)) return fail(c, FP_EINVAL, "strip decomposition needs the tiled planning path");
    if (int rc = prepare(c, k_s)) return rc;
    if (!c->graph_valid || c->graph_ks != k_s || c->graph_seed != seed)
        if (int rc = capture(c, k_s, seed)) return rc;
    return sync_scalars(c);
}

static int strip_finish_stats(fp_ctx* c, int64_t alive0, fp_step_stats* out) {
    if (int rc = read_scalars(c)) return rc;
    c->ctr.planned_agents += alive0;
    c->n_order = (uint32_t)c->h_sc->n_alive;
    c->n_exits = (uint32_t)c->h_sc->n_exits;
    c->last_displacement = (int64_t)c->h_sc->disp;
    c->last_dx = (int64_t)c->h_sc->step_dx;
    if (int rc = fp_exits_finish(c)) return rc;
    if (out) {
        out->alive = c->alive;
        out->exited = alive0 - c->alive;
        out->displacement_cells = c->last_displacement;
    }
    return FP_OK;
}

static int strip_step(fp_ctx* c, double k_s, uint64_t seed, fp_step_stats* out) {
    if (c->st.transport != FP_STRIP_NCCL && c->st.transport != FP_STRIP_HOST)
        return fail(c, FP_EINVAL, "strip step: no exchange transport (fp_strip_set_nccl / fp_strip_set_exchange), "
                                  "or drive all ranks with fp_strips_step");
    if (int rc = strip_ready(c, k_s, seed)) return rc;
    const int64_t alive0 = c->alive;
    FP_CUDA(c, cudaGraphLaunch(c->graph_plan, c->stream));
    FP_CUDA(c, cudaGraphLaunch(c->graph_move, c->stream));
    if (int rc = fp_strip_exchange(c)) return rc;
    FP_CUDA(c, cudaGraphLaunch(c->st.graph_fin, c->stream));
    c->ctr.kernel_launches += c->launches_per_step;
    return strip_finish_stats(c, alive0, out);
}

// fp_run on one strip rank (NCCL or host transport): the three graphs per step with the
// exchange between, CUDA events between the plan and the rest of the step.
static int strip_run(fp_ctx* c, double k_s, uint64_t seed, int32_t steps, fp_run_stats* out) {
    if (c->st.transport != FP_STRIP_NCCL && c->st.transport != FP_STRIP_HOST)
        return fail(c, FP_EINVAL, "strip run: no exchange transport");
    if (int rc = strip_ready(c, k_s, seed)) return rc;
    fp_launch(run_begin_kernel, 1, 1, 0, c->stream, c->d_sc);
    FP_LAUNCHED(c);
    std::vector<cudaEvent_t> ev((size_t)2 * steps + 1);
    for (auto& e : ev) FP_CUDA(c, cudaEventCreate(&e));
    for (int s = 0; s < steps; ++s) {
        cudaEventRecord(ev[2 * s], c->stream);
        FP_CUDA(c, cudaGraphLaunch(c->graph_plan, c->stream));
        cudaEventRecord(ev[2 * s + 1], c->stream);
        FP_CUDA(c, cudaGraphLaunch(c->graph_move, c->stream));
        if (int rc = fp_strip_exchange(c)) return rc;
        FP_CUDA(c, cudaGraphLaunch(c->st.graph_fin, c->stream));
    }
    cudaEventRecord(ev[2 * steps], c->stream);
    FP_CUDA(c, cudaEventSynchronize(ev[2 * steps]));
    c->ctr.kernel_launches += (int64_t)steps * c->launches_per_step;
    fp_run_stats rs{};
    float plan_ms = 0, move_ms = 0, tot = 0;
    for (int s = 0; s < steps; ++s) {
        float a = 0, b = 0;
        cudaEventElapsedTime(&a, ev[2 * s], ev[2 * s + 1]);
        cudaEventElapsedTime(&b, ev[2 * s + 1], ev[2 * s + 2]);
        plan_ms += a;
        move_ms += b;
    }
    cudaEventElapsedTime(&tot, ev[0], ev[2 * steps]);
    for (auto& e : ev) cudaEventDestroy(e);
    if (int rc = read_scalars(c)) return rc;
    rs.wall_time_s = tot * 1e-3;
    rs.plan_time_s = plan_ms * 1e-3;
    rs.move_time_s = move_ms * 1e-3;
    rs.steps = steps;
    rs.exited = (int64_t)c->h_sc->tot_exits;
    rs.displacement_cells = (int64_t)c->h_sc->tot_disp;
    rs.agent_updates = (int64_t)c->h_sc->tot_updates;
    rs.alive = c->alive;
    c->n_order = (uint32_t)c->h_sc->n_alive;
    c->n_exits = 0;
    c->ctr.planned_agents += rs.agent_updates;
    if (out) *out = rs;
    return FP_OK;
}

// All ranks in this process (the local transport): every rank's payload is copied into every
// rank's receive buffer (peer copies across devices, plain device copies on one device).
static int strips_check(fp_ctx* const* cs, int n) {
    if (!cs || n < 1) return fail(nullptr, FP_EINVAL, "fp_strips_step: need at least one context");
    for (int r = 0; r < n; ++r) {
        if (!cs[r] || !cs[r]->st.on || cs[r]->st.nranks != n || cs[r]->st.rank != r)
            return fail(cs[r], FP_EINVAL, "fp_strips_step: context r must be strip rank r of n");
        if (int rc = check_usable(cs[r])) return rc;
        cs[r]->st.transport = FP_STRIP_LOCAL;
    }
    return FP_OK;
}

static int strips_exchange_local(fp_ctx* const* cs, int n) {
    // phase 1: every rank's header (counts) to every rank, then read them on the host
    for (int q = 0; q < n; ++q) {
        cudaSetDevice(cs[q]->device);
        FP_CUDA(cs[q], cudaEventRecord(cs[q]->st.ev, cs[q]->stream));
    }
    const size_t hb = fp_strip_hdr_bytes();
    for (int q = 0; q < n; ++q) {
        fp_ctx* c = cs[q];
        cudaSetDevice(c->device);
        for (int p = 0; p < n; ++p) {
            FP_CUDA(c, cudaStreamWaitEvent(c->stream, cs[p]->st.ev, 0));
            FP_CUDA(c, cudaMemcpyPeerAsync((char*)c->st.d_rhdr + p * hb, c->device, cs[p]->st.d_send, cs[p]->device, hb,
                                           c->stream));
        }
    }
    fp_ctx* c0 = cs[0];
    cudaSetDevice(c0->device);
    FP_CUDA(c0, cudaMemcpyAsync(c0->st.h_rhdr, c0->st.d_rhdr, hb * n, cudaMemcpyDeviceToHost, c0->stream));
    FP_CUDA(c0, cudaStreamSynchronize(c0->stream));
    // phase 2: exactly the used records of every rank into every rank's slot for it
    for (int q = 0; q < n; ++q) {
        fp_ctx* c = cs[q];
        cudaSetDevice(c->device);
        for (int p = 0; p < n; ++p) {
            const unsigned long long* h = c0->st.h_rhdr + (size_t)p * (hb / 8);
            const size_t nd = std::min<unsigned long long>(h[0], c->st.cap_def);
            const size_t ne = std::min<unsigned long long>(h[1], c->st.cap_exit);
            char* dst = (char*)c->st.d_recv + (size_t)p * c->st.xbytes;
            const char* src = (const char*)cs[p]->st.d_send;
            if (nd)
                FP_CUDA(c, cudaMemcpyPeerAsync(dst + fp_strip_def_off(), c->device, src + fp_strip_def_off(),
                                               cs[p]->device, nd * 32, c->stream));
            if (ne)
                FP_CUDA(c, cudaMemcpyPeerAsync(dst + fp_strip_exit_off(c), c->device, src + fp_strip_exit_off(cs[p]),
                                               cs[p]->device, ne * 8, c->stream));
        }
    }
    // a rank's send buffer is rewritten next step only after every rank copied it
    for (int q = 0; q < n; ++q) {
        cudaSetDevice(cs[q]->device);
        FP_CUDA(cs[q], cudaEventRecord(cs[q]->st.ev, cs[q]->stream));
    }
    for (int q = 0; q < n; ++q) {
        cudaSetDevice(cs[q]->device);
        for (int p = 0; p < n; ++p) FP_CUDA(cs[q], cudaStreamWaitEvent(cs[q]->stream, cs[p]->st.ev, 0));
    }
    return FP_OK;
}

extern "C" int fp_strips_step(fp_ctx* const* cs, int n, double k_s, uint64_t seed, fp_step_stats* out) {
    if (int rc = strips_check(cs, n)) return rc;
    std::vector<int64_t> alive0(n);
    for (int r = 0; r < n; ++r) {
        fp_ctx* c = cs[r];
        cudaSetDevice(c->device);
        if (c->st.xbytes != cs[0]->st.xbytes) return fail(c, FP_EINVAL, "fp_strips_step: ranks disagree on exchange sizes");
        if (int rc = strip_ready(c, k_s, seed)) return rc;
        alive0[r] = c->alive;
        FP_CUDA(c, cudaGraphLaunch(c->graph_plan, c->stream));
        FP_CUDA(c, cudaGraphLaunch(c->graph_move, c->stream));
    }
    if (int rc = strips_exchange_local(cs, n)) return rc;
    for (int r = 0; r < n; ++r) {
        cudaSetDevice(cs[r]->device);
        FP_CUDA(cs[r], cudaGraphLaunch(cs[r]->st.graph_fin, cs[r]->stream));
        cs[r]->ctr.kernel_launches += cs[r]->launches_per_step;
    }
    for (int r = 0; r < n; ++r) {
        cudaSetDevice(cs[r]->device);
        if (int rc = strip_finish_stats(cs[r], alive0[r], r == 0 ? out : nullptr)) return rc;
    }
    return FP_OK;
}

extern "C" int fp_strips_run(fp_ctx* const* cs, int n, double k_s, uint64_t seed, int32_t steps, fp_run_stats* out) {
    if (int rc = strips_check(cs, n)) return rc;
    if (steps < 1) return fail(cs[0], FP_EINVAL, "SimParams: steps must be >= 1");
    std::vector<cudaEvent_t> e0(n), e1(n);
    for (int r = 0; r < n; ++r) {
        fp_ctx* c = cs[r];
        cudaSetDevice(c->device);
        if (int rc = strip_ready(c, k_s, seed)) return rc;
        fp_launch(run_begin_kernel, 1, 1, 0, c->stream, c->d_sc);
        FP_LAUNCHED(c);
        FP_CUDA(c, cudaEventCreate(&e0[r]));
        FP_CUDA(c, cudaEventCreate(&e1[r]));
        cudaEventRecord(e0[r], c->stream);
    }
    for (int s = 0; s < steps; ++s) {
        for (int r = 0; r < n; ++r) {
            cudaSetDevice(cs[r]->device);
            FP_CUDA(cs[r], cudaGraphLaunch(cs[r]->graph_plan, cs[r]->stream));
            FP_CUDA(cs[r], cudaGraphLaunch(cs[r]->graph_move, cs[r]->stream));
        }
        if (int rc = strips_exchange_local(cs, n)) return rc;
        for (int r = 0; r < n; ++r) {
            cudaSetDevice(cs[r]->device);
            FP_CUDA(cs[r], cudaGraphLaunch(cs[r]->st.graph_fin, cs[r]->stream));
        }
    }
    float tmax = 0;
    for (int r = 0; r < n; ++r) {
        fp_ctx* c = cs[r];
        cudaSetDevice(c->device);
        cudaEventRecord(e1[r], c->stream);
        FP_CUDA(c, cudaEventSynchronize(e1[r]));
        float t = 0;
        cudaEventElapsedTime(&t, e0[r], e1[r]);
        tmax = std::max(tmax, t);
        cudaEventDestroy(e0[r]);
        cudaEventDestroy(e1[r]);
        c->ctr.kernel_launches += (int64_t)steps * c->launches_per_step;
        if (int rc = read_scalars(c)) return rc;
        c->n_order = (uint32_t)c->h_sc->n_alive;
        c->n_exits = 0;
    }
    fp_ctx* c = cs[0];
    fp_run_stats rs{};
    rs.wall_time_s = tmax * 1e-3;  // max over ranks (every rank's stream, CUDA events)
    rs.steps = steps;
    rs.exited = (int64_t)c->h_sc->tot_exits;
    rs.displacement_cells = (int64_t)c->h_sc->tot_disp;
    rs.agent_updates = (int64_t)c->h_sc->tot_updates;
    rs.alive = c->alive;
    if (out) *out = rs;
    return FP_OK;
}

extern "C" int fp_get_agents(const fp_ctx* cc, int32_t* x, int32_t* y, uint8_t* alive) {
    fp_ctx* c = const_cast<fp_ctx*>(cc);
    if (!c) return fail(nullptr, FP_EINVAL, "null context");
    cudaSetDevice(c->device);
    const size_t n = c->n;
    if (x) FP_CUDA(c, cudaMemcpyAsync(x, c->d_x, n * 4, cudaMemcpyDeviceToHost, c->stream));
    if (y) FP_CUDA(c, cudaMemcpyAsync(y, c->d_y, n * 4, cudaMemcpyDeviceToHost, c->stream));
    if (alive) FP_CUDA(c, cudaMemcpyAsync(alive, c->d_alive, n, cudaMemcpyDeviceToHost, c->stream));
    FP_CUDA(c, cudaStreamSynchronize(c->stream));
    return FP_OK;
}

extern "C" int fp_get_desired(const fp_ctx* cc, int32_t* x, int32_t* y) {
    fp_ctx* c = const_cast<fp_ctx*>(cc);
    if (!c) return fail(nullptr, FP_EINVAL, "null context");
    cudaSetDevice(c->device);
    FP_CUDA(c, cudaMemcpyAsync(x, c->d_dx, (size_t)c->n * 4, cudaMemcpyDeviceToHost, c->stream));
    FP_CUDA(c, cudaMemcpyAsync(y, c->d_dy, (size_t)c->n * 4, cudaMemcpyDeviceToHost, c->stream));
    FP_CUDA(c, cudaStreamSynchronize(c->stream));
    return FP_OK;
}

extern "C" int fp_get_occupancy(const fp_ctx* cc, int32_t* occ) {
    fp_ctx* c = const_cast<fp_ctx*>(cc);
    if (!c || !occ) return fail(c, FP_EINVAL, "null argument");
    cudaSetDevice(c->device);
    const size_t ncell = (size_t)c->W * c->H;
    int32_t* d = nullptr;
    FP_CUDA(c, cudaMalloc(&d, ncell * 4));
    cudaMemsetAsync(d, 0xFF, ncell * 4, c->stream);
    if (c->n) {
        fp_launch(occ_dump_kernel, fp_blocks(c->n, 256), 256, 0, c->stream, c->d_x, c->d_y, c->d_alive, c->n, geo_of(c), d);
        c->ctr.kernel_launches++;
    }
    cudaMemcpyAsync(occ, d, ncell * 4, cudaMemcpyDeviceToHost, c->stream);
    cudaError_t e = cudaStreamSynchronize(c->stream);
    cudaFree(d);
    if (e != cudaSuccess) return fp_cuda_fail(c, e, "fp_get_occupancy");
    return FP_OK;
}

extern "C" int fp_get_exited(const fp_ctx* cc, uint32_t* ids, uint32_t cap, uint32_t* n) {
    fp_ctx* c = const_cast<fp_ctx*>(cc);
    if (!c || !n) return fail(c, FP_EINVAL, "null argument");
    *n = c->n_exits;
    if (c->n_exits == 0 || !ids) return FP_OK;
    std::vector<unsigned long long> rec(c->n_exits);
    cudaSetDevice(c->device);
    FP_CUDA(c, cudaMemcpyAsync(rec.data(), c->d_exits, rec.size() * 8, cudaMemcpyDeviceToHost, c->stream));
    FP_CUDA(c, cudaStreamSynchronize(c->stream));
    for (uint32_t i = 0; i < c->n_exits && i < cap; ++i) ids[i] = (uint32_t)(rec[i] & 0xFFFFFFFFull);
    return FP_OK;
}

extern "C" int fp_get_order(const fp_ctx* cc, uint32_t* ids, uint32_t cap, uint32_t* n) {
    fp_ctx* c = const_cast<fp_ctx*>(cc);
    if (!c || !n) return fail(c, FP_EINVAL, "null argument");
    *n = c->n_order;
    if (!ids || c->n_order == 0) return FP_OK;
    cudaSetDevice(c->device);
    FP_CUDA(c, cudaMemcpyAsync(ids, c->d_order, (size_t)std::min(cap, c->n_order) * 4, cudaMemcpyDeviceToHost,
                               c->stream));
    FP_CUDA(c, cudaStreamSynchronize(c->stream));
    return FP_OK;
}

extern "C" int fp_state_hash(const fp_ctx* cc, uint64_t* out) {
    fp_ctx* c = const_cast<fp_ctx*>(cc);
    if (!c || !out) return fail(c, FP_EINVAL, "null argument");
    std::vector<int32_t> x(c->n), y(c->n);
    std::vector<uint8_t> a(c->n);
    if (int rc = fp_get_agents(c, x.data(), y.data(), a.data())) return rc;
    uint64_t h = 14695981039346656037ULL;  // state.hpp:80-95
    auto mix = [&h](uint64_t v) {
        h ^= v;
        h *= 1099511628211ULL;
    };
    mix((uint64_t)c->step);
    mix((uint64_t)c->alive);
    for (uint32_t i = 0; i < c->n; ++i) {
        mix(i);
        mix((uint32_t)x[i]);
        mix((uint32_t)y[i]);
        mix(a[i] ? 1 : 0);
    }
    *out = h;
    return FP_OK;
}

extern "C" int fp_hash_roster(int64_t step, int64_t alive, uint32_t n, const int32_t* x, const int32_t* y,
                              const uint8_t* a, uint64_t* out) {
    if (!out || (n && (!x || !y || !a))) return fail(nullptr, FP_EINVAL, "null argument");
    uint64_t h = 14695981039346656037ULL;  // state.hpp:80-95
    auto mix = [&h](uint64_t v) {
        h ^= v;
        h *= 1099511628211ULL;
    };
    mix((uint64_t)step);
    mix((uint64_t)alive);
    for (uint32_t i = 0; i < n; ++i) {
        mix(i);
        mix((uint32_t)x[i]);
        mix((uint32_t)y[i]);
        mix(a[i] ? 1 : 0);
    }
    *out = h;
    return FP_OK;
}

extern "C" int fp_get_choice(fp_ctx* c, uint32_t agent, double k_s, int32_t* cx, int32_t* cy, double* w,
                             float* p, uint32_t cap, uint32_t* n) {
    if (!c || !n) return fail(c, FP_EINVAL, "null argument");
    if (agent >= c->n) return fail(c, FP_EINVAL, "fp_get_choice: agent out of range");
    cudaSetDevice(c->device);
    const size_t M = 128;
    void* d = nullptr;
    FP_CUDA(c, cudaMalloc(&d, M * (4 + 4 + 8 + 4) + 16));
    int32_t* dcx = (int32_t*)d;
    int32_t* dcy = dcx + M;
    double* dw = (double*)(dcy + M);
    float* dp = (float*)(dw + M);
    uint32_t* dn = (uint32_t*)(dp + M);
    int rc = fp_choice_launch(c, agent, k_s, dcx, dcy, dw, dp, dn);
    if (rc == FP_OK) {
        std::vector<char> h(M * (4 + 4 + 8 + 4) + 16);
        cudaMemcpyAsync(h.data(), d, h.size(), cudaMemcpyDeviceToHost, c->stream);
        cudaError_t e = cudaStreamSynchronize(c->stream);
        if (e != cudaSuccess) {
            rc = fp_cuda_fail(c, e, "fp_get_choice");
        } else {
            const int32_t* hx = (const int32_t*)h.data();
            const int32_t* hy = hx + M;
            const double* hw = (const double*)(hy + M);
            const float* hp = (const float*)(hw + M);
            const uint32_t k = *(const uint32_t*)(hp + M);
            *n = k;
            for (uint32_t i = 0; i < k && i < cap; ++i) {
                if (cx) cx[i] = hx[i];
                if (cy) cy[i] = hy[i];
                if (w) w[i] = hw[i];
                if (p) p[i] = hp[i];
            }
        }
    }
    cudaFree(d);
    return rc;
}

static int check_agent_arg(fp_ctx* c, int32_t x, int32_t y, int32_t v) {
    if (v < 1 || v > 5) return fail(c, FP_EINVAL, "SimParams: v_max must be in [1,5]");
    const int32_t xw = c->boundary == FP_BOUNDARY_PERIODIC_X ? ((x % c->W) + c->W) % c->W : x;
    if (xw < 0 || xw >= c->W || y < 0 || y >= c->H) return fail(c, FP_EINVAL, "agent is out of bounds");
    return FP_OK;
}

extern "C" int fp_choose_desired(fp_ctx* c, uint32_t id, int32_t x, int32_t y, int32_t v_max, int64_t step,
                                 double k_s, uint64_t seed, int32_t* out_x, int32_t* out_y) {
    if (!c || !out_x || !out_y) return fail(c, FP_EINVAL, "null argument");
    if (int rc = check_usable(c)) return rc;
    if (int rc = check_agent_arg(c, x, y, v_max)) return rc;
    cudaSetDevice(c->device);
    if (!c->d_scratch_small) FP_CUDA(c, cudaMalloc(&c->d_scratch_small, 4096));
    if (!c->h_scratch_small) FP_CUDA(c, cudaMallocHost(&c->h_scratch_small, 4096));
    int32_t* d = (int32_t*)c->d_scratch_small;
    if (int rc = fp_choose_one_launch(c, id, x, y, v_max, step, k_s, seed, d)) return rc;
    FP_CUDA(c, cudaMemcpyAsync(c->h_scratch_small, d, 8, cudaMemcpyDeviceToHost, c->stream));
    FP_CUDA(c, cudaStreamSynchronize(c->stream));
    *out_x = ((int32_t*)c->h_scratch_small)[0];
    *out_y = ((int32_t*)c->h_scratch_small)[1];
    return FP_OK;
}

extern "C" int fp_enumerate_candidates(fp_ctx* c, int32_t x, int32_t y, int32_t v_max, int32_t* cx, int32_t* cy,
                                       uint32_t cap, uint32_t* n) {
    if (!c || !n) return fail(c, FP_EINVAL, "null argument");
    if (int rc = check_usable(c)) return rc;
    if (int rc = check_agent_arg(c, x, y, v_max)) return rc;
    cudaSetDevice(c->device);
    if (!c->d_scratch_small) FP_CUDA(c, cudaMalloc(&c->d_scratch_small, 4096));
    if (!c->h_scratch_small) FP_CUDA(c, cudaMallocHost(&c->h_scratch_small, 4096));
    int32_t* d = (int32_t*)c->d_scratch_small;  // 121 x, 121 y, count
    if (int rc = fp_candidates_one_launch(c, x, y, v_max, d, d + 128, (uint32_t*)(d + 256))) return rc;
    FP_CUDA(c, cudaMemcpyAsync(c->h_scratch_small, d, 257 * 4, cudaMemcpyDeviceToHost, c->stream));
    FP_CUDA(c, cudaStreamSynchronize(c->stream));
    const int32_t* h = (const int32_t*)c->h_scratch_small;
    *n = (uint32_t)h[256];
    for (uint32_t i = 0; i < *n && i < cap; ++i) {
        if (cx) cx[i] = h[i];
        if (cy) cy[i] = h[128 + i];
    }
    return FP_OK;
}

extern "C" int fp_movement_order(int64_t n, uint64_t seed, int64_t step, int device, uint32_t* out) {
    if (n < 0 || n >= ((int64_t)1 << 32)) return fail(nullptr, FP_EINVAL, "fp_movement_order: bad n");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(nullptr, FP_ECUDA, "fp_movement_order: no CUDA device available");
    fp_ctx* c = new fp_ctx();
    c->device = device;
    cudaSetDevice(device);
    cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
    int rc = FP_OK;
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaMalloc(&c->d_sc, sizeof(DevScalars)) != cudaSuccess)
        rc = fp_cuda_fail(c, cudaGetLastError(), "fp_movement_order setup");
    if (rc == FP_OK) rc = ensure_agents(c, (uint32_t)n);
    if (rc == FP_OK) c->n = (uint32_t)n;
    if (rc == FP_OK && n > 0) rc = fp_order_positions(c, (uint32_t)n, seed, step, c->d_order);
    if (rc == FP_OK && n > 0) {
        cudaMemcpyAsync(out, c->d_order, (size_t)n * 4, cudaMemcpyDeviceToHost, c->stream);
        cudaError_t e = cudaStreamSynchronize(c->stream);
        if (e != cudaSuccess) rc = fp_cuda_fail(c, e, "fp_movement_order");
    }
    if (rc != FP_OK) g_error = c->err;
    fp_destroy(c);
    return rc;
}

// scenario_io.hpp:47-69 -- host placement (setup, untimed): partial Fisher-Yates over the
// row-major free-cell list with the kSpawnStream draws.
extern "C" int fp_spawn_agents(int32_t w, int32_t h, const uint8_t* cells, int64_t n, uint64_t seed,
                               int32_t* x, int32_t* y) {
    if (n < 0) return fail(nullptr, FP_EINVAL, "spawn_agents: agent count must be >= 0");
    if (w < 1 || h < 1 || !cells) return fail(nullptr, FP_EINVAL, "spawn_agents: bad grid");
    const size_t total = (size_t)w * h;
    std::vector<uint32_t> fr;
    fr.reserve(total / 2);
    for (size_t i = 0; i < total; ++i)
        if (cells[i] == FP_CELL_FREE) fr.push_back((uint32_t)i);
    if ((size_t)n > fr.size())
        return fail(nullptr, FP_ERUNTIME,
                    "spawn_agents: requested " + std::to_string(n) + " agents but the scenario has only " +
                        std::to_string(fr.size()) + " free cells");
    uint64_t draw = 0;
    const size_t F = fr.size();
    for (int64_t i = 0; i < n; ++i) {
        const uint64_t r = fp_rng_u64(seed, FP_SPAWN_STREAM, 0, draw++);
        const size_t j = (size_t)i + (size_t)(r % (uint64_t)(F - (size_t)i));
        std::swap(fr[(size_t)i], fr[j]);
    }
    for (int64_t i = 0; i < n; ++i) {
        x[i] = (int32_t)(fr[(size_t)i] % (uint32_t)w);
        y[i] = (int32_t)(fr[(size_t)i] / (uint32_t)w);
    }
    return FP_OK;
}

int fp_plan_kernel_time(fp_ctx* ctx, double k_s, uint64_t seed, int iters, double* ms);

extern "C" int fp_time_plan_kernel(fp_ctx* c, double k_s, uint64_t seed, int32_t iters, double* ms) {
    if (!c || !ms) return fail(c, FP_EINVAL, "null argument");
    cudaSetDevice(c->device);
    if (int rc = sync_scalars(c)) return rc;
    if (int rc = fp_plan_kernel_time(c, k_s, seed, iters, ms)) return rc;
    return read_scalars(c);
}

extern "C" int fp_get_counters(const fp_ctx* c, fp_counters* out) {
    if (!c || !out) return fail(nullptr, FP_EINVAL, "null argument");
    *out = c->ctr;
    return FP_OK;
}

// Diagnostics (not in the header): the plan kernel's profile counters (FP_PLAN_PROF builds).
extern "C" int fp_debug_plan_prof(fp_ctx* c, int64_t* out, int cap) {
    DevScalars h;
    if (cudaMemcpy(&h, c->d_sc, sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    for (int k = 0; k < cap && k < 8; ++k) out[k] = (int64_t)h.plan_prof[k];
    return 0;
}

// Diagnostics (not in the header): per grid round of the last motion phase, the globaltimer at
// its start (relative to the end of the seed pass) and the pending count.  Returns the count.
extern "C" int fp_debug_rounds(fp_ctx* c, int64_t* t_ns, int64_t* pending, int64_t* checks, int64_t* chk_max,
                               int64_t* p1_max, int cap) {
    if (!c) return -1;
    DevScalars h;
    if (cudaMemcpy(&h, c->d_sc, sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    const int n = (int)std::min<unsigned long long>(h.grid_rounds + 1, (unsigned long long)std::min(cap, 64));
    for (int r = 0; r < n; ++r) {
        t_ns[r] = (int64_t)(h.t_round[r] - h.t_motion[1]);
        pending[r] = (int64_t)h.n_round[r];
        checks[r] = (int64_t)h.chk_cnt[r];
        chk_max[r] = (int64_t)h.chk_max[r];
        p1_max[r] = (int64_t)h.p1_max[r];
    }
    if (cap >= 64) chk_max[63] = (int64_t)h.chk_max[63];  // largest bucket of the phase
    for (int r = n; r < std::min(cap, 64); ++r) p1_max[r] = (int64_t)h.p1_max[r];  // spare debug slots
    return n;
}
