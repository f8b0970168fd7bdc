// strip.cu -- the multi-GPU x-strip decomposition of one simulation.
//
// Rank r owns the agents standing in columns [x_lo, x_hi) and keeps the occupancy of its window
// [x_lo - 5, x_hi + 5) exact; walls, exits, the field and the weight plane are replicated
// (180 GB per B200 holds config 5's 6 GB of static planes many times over).  The alive flags
// are global on every rank, so each rank computes the reference's global movement order
// (engine.hpp:99-111) locally; an agent's global id never changes.
//
// Per step (fp_step / fp_run on a strip context):
//   1. order (global, replicated) || plan of the owned agents (planning reads only the window);
//   2. defer: the footprint (start + path cells a walk can read or write, motion_rec.cuh) of a
//      walk that touches a band -- the cells within 5 columns of a strip edge shared with
//      another rank -- may overlap a footprint of another rank's agent; any two footprints of
//      different ranks can only overlap inside a band (an owned footprint stays within 5 cells
//      of the owned strip).  Those walks, and every walk connected to them through shared
//      footprint cells (closure over the P2 marks), are DEFERRED: their records leave the local
//      motion (m = 0: no marks, no walk).  What is left touches no band and shares no cell with
//      a deferred walk, so it walks locally, in the reference order, exactly as on one GPU;
//   3. one allgather over the ranks (NCCL over NVLink, or a host / in-process transport):
//      every rank's deferred records (with the snapshot occupancy of their footprint cells,
//      which the owner's window holds) and its local exits;
//   4. resolve (every rank, redundantly and deterministically): the union of the deferred
//      walks is the union of whole conflict components, so walking it alone, in rank order
//      per shared cell (reservation rounds over a cell hash), is the sequential walk of those
//      agents; each rank applies the results inside its window (positions, occupancy,
//      ownership: an agent belongs to the strip its final cell lies in -- only deferred walks
//      can cross a strip edge, so ownership moves only here), and the global exit list is all
//      local exits plus the resolved ones, sorted by rank (processing order).
// Nothing else is exchanged: the halo columns of a window only change through walks that touch
// a band, and those are resolved on every rank.  Sharded runs equal the 1-GPU run bit for bit
// (tests/test_strips.py).
#include <dlfcn.h>

#include <algorithm>
#include <vector>

#include "motion_rec.cuh"

__constant__ signed char c_bpath_s[121][5][2];
static bool g_bpath_s_ready[64] = {false};

// Resolver record: the motion record (rank in .y), the desired cell (generic records re-walk
// toward it), the snapshot occupancy of the footprint cells (bit 0 start, bit 1+j path cell j).
struct DefRec {
    uint4 rec;
    int32_t tx, ty;
    uint32_t occ;
    uint32_t pad;
};
static_assert(sizeof(DefRec) == 32, "DefRec layout");

#define XH_WORDS 16  // payload header (u64): [0] deferred, [1] local exits, [2] local hops, [3] local dx,
                     // [4] error flags
#define RES_TAIL_THREADS 1024

struct StripArgs {
    Geo g;
    const uint32_t* occ;
    uint32_t* occ_w;
    uint32_t *p1, *p2, *dpl;
    uint4* rec0;
    const int32_t* dx;
    const int32_t* dy;
    const uint32_t* rank;
    uint8_t* dflag;
    uint32_t* clist;
    DevScalars* sc;
    int x_lo, x_hi, nranks;
    int periodic;
};

// Column x (wrapped) lies within 5 cells of a strip edge shared with another rank.
__device__ __forceinline__ bool in_band(const StripArgs& s, int x) {
    if (s.nranks < 2) return false;
    const int W = s.g.W;
    auto near = [&](int e) {  // |x - e| in the band [e - 5, e + 5)
        int d = x - e;
        if (s.periodic) {
            d %= W;
            if (d < -W / 2) d += W;
            if (d >= W - W / 2) d -= W;
        }
        return d >= -5 && d < 5;
    };
    const bool lo_shared = s.periodic || s.x_lo > 0;
    const bool hi_shared = s.periodic || s.x_hi < W;
    return (lo_shared && near(s.x_lo)) || (hi_shared && near(s.x_hi == W && s.periodic ? 0 : s.x_hi));
}

__device__ __forceinline__ bool in_window(const StripArgs& s, int x) {
    if (s.nranks < 2) return true;
    int d = x - (s.x_lo - 5);
    if (s.periodic) {
        d %= s.g.W;
        if (d < 0) d += s.g.W;
    }
    return d >= 0 && d < (s.x_hi - s.x_lo) + 10;
}

__device__ __forceinline__ bool in_strip(const StripArgs& s, int x) { return x >= s.x_lo && x < s.x_hi; }

__device__ __forceinline__ int rec_cells6(const Geo& g, const uint4& r, const int32_t* dx, const int32_t* dy,
                                          int* cx, int* cy) {
    int gtx = 0, gty = 0;
    if (r.w & REC_GENERIC) {
        gtx = g.wrap(dx[r.x]);
        gty = dy[r.x];
    }
    cx[0] = rec_x(r);
    cy[0] = rec_y(r);
    return record_cells(g, r, c_bpath_s, gtx, gty, cx + 1, cy + 1);
}

__device__ __forceinline__ bool bit_at(const uint32_t* plane, const Geo& g, int x, int y) {
    return (__ldcg(&plane[g.word(x, y)]) >> (x & 31)) & 1u;
}

// 2a. contention marks of every planned walk (P1: in a footprint, P2: in two or more).
__global__ void strip_mark_kernel(StripArgs s) {
    FP_PDL_WAIT();
    const uint32_t n = (uint32_t)s.sc->n_planned;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const uint4 r = s.rec0[k];
        if (!rec_m(r)) continue;
        int gtx = 0, gty = 0;
        if (r.w & REC_GENERIC) {
            gtx = s.g.wrap(s.dx[r.x]);
            gty = s.dy[r.x];
        }
        mark_record(s.p1, s.p2, s.g, r, c_bpath_s, gtx, gty);
    }
}

// 2b. seeds: walks whose footprint touches a band; contended walks listed for the closure.
__global__ void strip_seed_kernel(StripArgs s) {
    FP_PDL_WAIT();
    const uint32_t n = (uint32_t)s.sc->n_planned;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const uint4 r = s.rec0[k];
        s.dflag[k] = 0;
        if (!rec_m(r)) continue;
        int cx[6], cy[6];
        rec_cells6(s.g, r, s.dx, s.dy, cx, cy);
        const int mf = rec_mf(r);
        bool band = false, contended = false;
#pragma unroll
        for (int i = 0; i < 6; ++i)
            if (i <= mf) {
                band |= in_band(s, cx[i]);
                contended |= bit_at(s.p2, s.g, cx[i], cy[i]);
            }
        if (band) {
            s.dflag[k] = 1;
#pragma unroll
            for (int i = 0; i < 6; ++i)
                if (i <= mf) atomicOr(&s.dpl[s.g.word(cx[i], cy[i])], 1u << (cx[i] & 31));
        } else if (contended) {
            s.clist[atomicAdd(&s.sc->strip_nc, 1ull)] = k;
        }
    }
}

// 2c. closure (one CTA): a contended walk sharing a footprint cell with a deferred one is
// deferred, until nothing changes.  Monotone, so the fixed point does not depend on timing.
__global__ void __launch_bounds__(1024) strip_closure_kernel(StripArgs s) {
    FP_PDL_WAIT();
    __shared__ int s_changed;
    const uint32_t n = (uint32_t)s.sc->strip_nc;
    for (int it = 0;; ++it) {
        if (threadIdx.x == 0) s_changed = 0;
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
            const uint32_t k = s.clist[i];
            if (s.dflag[k]) continue;
            const uint4 r = s.rec0[k];
            int cx[6], cy[6];
            rec_cells6(s.g, r, s.dx, s.dy, cx, cy);
            const int mf = rec_mf(r);
            bool hit = false;
#pragma unroll
            for (int j = 0; j < 6; ++j)
                if (j <= mf) hit |= bit_at(s.dpl, s.g, cx[j], cy[j]);
            if (!hit) continue;
            s.dflag[k] = 1;
#pragma unroll
            for (int j = 0; j < 6; ++j)
                if (j <= mf) atomicOr(&s.dpl[s.g.word(cx[j], cy[j])], 1u << (cx[j] & 31));
            s_changed = 1;
        }
        __syncthreads();
        if (!s_changed) break;
        __syncthreads();
        if (it > (1 << 20)) {
            if (threadIdx.x == 0) atomicOr(&s.sc->err, 128ull);
            break;
        }
    }
}

// 2d. deferred walks into the send buffer (rank, desired cell, snapshot occupancy of the footprint)
// and out of the local motion (m = 0).
__global__ void strip_export_kernel(StripArgs s, DefRec* out, uint32_t cap, unsigned long long* hdr) {
    FP_PDL_WAIT();
    const uint32_t n = (uint32_t)s.sc->n_planned;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        if (!s.dflag[k]) continue;
        uint4 r = s.rec0[k];
        int cx[6], cy[6];
        const int m = rec_cells6(s.g, r, s.dx, s.dy, cx, cy);
        uint32_t occ = 0;
#pragma unroll
        for (int i = 0; i < 6; ++i)
            if (i <= m) occ |= (uint32_t)bit_at(s.occ, s.g, cx[i], cy[i]) << i;
        DefRec d;
        d.rec = r;
        d.rec.y = s.rank[r.x];
        d.tx = s.dx[r.x];
        d.ty = s.dy[r.x];
        d.occ = occ;
        d.pad = 0;
        const unsigned long long slot = atomicAdd(&hdr[0], 1ull);
        if (slot < cap) out[slot] = d;
        else atomicOr(&hdr[4], 1ull);
        r.z &= ~(0x70000000u | REC_EXIT_FREE | 0x80000000u);  // m = 0: the local motion skips it
        s.rec0[k] = r;
    }
}

// 3. after the local motion: header + local exits into the send buffer.
__global__ void strip_pack_kernel(DevScalars* sc, const unsigned long long* exits, unsigned long long* hdr,
                                  unsigned long long* xout, uint32_t cap) {
    FP_PDL_WAIT();
    const unsigned long long ne = sc->n_exits;
    for (unsigned long long i = blockIdx.x * blockDim.x + threadIdx.x; i < ne && i < cap; i += gridDim.x * blockDim.x)
        xout[i] = exits[i];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        hdr[1] = ne;
        if (ne > cap) hdr[4] |= 2ull;
        hdr[2] = sc->disp;                     // hops (the motion split the accumulator)
        hdr[3] = (unsigned long long)sc->step_dx;
    }
}

// 4. resolve the union of every rank's deferred walks (one CTA; a global-memory cell hash).
struct ResolveArgs {
    Geo g;
    const unsigned char* recv;  // nranks payloads of xbytes
    const unsigned long long* rhdr;  // nranks headers of XH_WORDS
    size_t xbytes;
    int nranks;
    uint32_t cap_def;
    uint32_t* hkey;   // hash: cell -> slot (nslots, power of two)
    uint32_t* hres;   // reservation (min rank) per slot
    uint8_t* hocc;    // occupancy per slot
    uint32_t nslots;
    uint32_t* rslot;  // per deferred record: 6 slots
    uint32_t* plist;  // pending lists (2 x cap_total)
    uint32_t cap_total;
    int32_t* x;
    int32_t* y;
    uint8_t* alive;
    uint8_t* owned;
    uint32_t* occ;
    unsigned long long* rexits;  // resolver exits (rank << 32 | id)
    DevScalars* sc;
    StripArgs s;
};

__device__ __forceinline__ const DefRec* res_rec(const ResolveArgs& a, uint32_t t, uint32_t* cum, int nr) {
    int q = 0;
    while (q + 1 < nr && t >= cum[q + 1]) ++q;
    return reinterpret_cast<const DefRec*>(a.recv + (size_t)q * a.xbytes + XH_WORDS * 8) + (t - cum[q]);
}

__device__ __forceinline__ uint32_t res_insert(const ResolveArgs& a, int x, int y, bool occupied) {
    const uint32_t cell = (uint32_t)y * (uint32_t)a.g.W + (uint32_t)x;
    uint32_t h = (cell * 2654435761u) & (a.nslots - 1);
    for (;;) {
        const uint32_t old = atomicCAS(&a.hkey[h], 0xFFFFFFFFu, cell);
        if (old == 0xFFFFFFFFu || old == cell) {
            if (occupied) a.hocc[h] = 1;  // every record agrees on a cell's snapshot occupancy
            return h;
        }
        h = (h + 1) & (a.nslots - 1);
    }
}

__global__ void __launch_bounds__(RES_TAIL_THREADS) strip_resolve_kernel(ResolveArgs a) {
    FP_PDL_WAIT();
    __shared__ uint32_t cum[65];
    __shared__ uint32_t cnt[2];
    __shared__ uint32_t s_ns;
    __shared__ unsigned long long s_hops;
    const int nr = a.nranks;
    if (threadIdx.x == 0) {
        uint32_t c = 0;
        for (int q = 0; q < nr; ++q) {
            cum[q] = c;
            const unsigned long long* h = a.rhdr + (size_t)q * XH_WORDS;
            if (h[4]) atomicOr(&a.sc->err, 64ull);  // a rank overflowed its exchange capacity
            c += (uint32_t)min(h[0], (unsigned long long)a.cap_def);
        }
        cum[nr] = c;
        if (c > a.cap_total) atomicOr(&a.sc->err, 64ull);
        c = min(c, (uint32_t)a.cap_total);
        cnt[0] = c;
        cnt[1] = 0;
        s_hops = 0;
        uint32_t ns = 1024;  // slots used this step: >= 8 per footprint cell of the union (<= 6 each)
        while (ns < c * 48u && ns < a.nslots) ns <<= 1;
        s_ns = min(ns, a.nslots);
    }
    __syncthreads();
    const uint32_t total = cnt[0];
    a.nslots = s_ns;
    for (uint32_t k = threadIdx.x; k < a.nslots; k += blockDim.x) {
        a.hkey[k] = 0xFFFFFFFFu;
        a.hres[k] = 0xFFFFFFFFu;
        a.hocc[k] = 0;
    }
    __syncthreads();
    for (uint32_t t = threadIdx.x; t < total; t += blockDim.x) {
        const DefRec* d = res_rec(a, t, cum, nr);
        int cx[6], cy[6];
        const int gtx = a.g.wrap(d->tx), gty = d->ty;
        cx[0] = rec_x(d->rec);
        cy[0] = rec_y(d->rec);
        const int m = record_cells(a.g, d->rec, c_bpath_s, gtx, gty, cx + 1, cy + 1);
        for (int i = 0; i <= m; ++i) a.rslot[(size_t)t * 6 + i] = res_insert(a, cx[i], cy[i], (d->occ >> i) & 1u);
        a.plist[t] = t;
    }
    __syncthreads();
    unsigned cur = 0, rounds = 0;
    unsigned long long hops = 0;
    for (;;) {
        const uint32_t n = cnt[cur];
        if (n == 0) break;
        ++rounds;
        const unsigned nxt = cur ^ 1;
        uint32_t* L = a.plist + (size_t)cur * a.cap_total;
        uint32_t* N = a.plist + (size_t)nxt * a.cap_total;
        for (uint32_t k = threadIdx.x; k < n; k += blockDim.x) {
            const uint32_t t = L[k];
            const DefRec* d = res_rec(a, t, cum, nr);
            const int mf = rec_mf(d->rec);
            for (int i = 0; i <= mf; ++i) atomicMin(&a.hres[a.rslot[(size_t)t * 6 + i]], d->rec.y);
        }
        __syncthreads();
        if (threadIdx.x == 0) cnt[cur] = 0;
        for (uint32_t k = threadIdx.x; k < n; k += blockDim.x) {
            const uint32_t t = L[k];
            const DefRec* d = res_rec(a, t, cum, nr);
            const uint4 r = d->rec;
            const int mf = rec_mf(r), m = rec_m(r);
            const uint32_t* sl = a.rslot + (size_t)t * 6;
            bool own = true;
            for (int i = 0; i <= mf && own; ++i) own = __ldcg(&a.hres[sl[i]]) == r.y;
            if (!own) {
                N[atomicAdd(&cnt[nxt], 1u)] = t;
                continue;
            }
            for (int i = 0; i <= mf; ++i) a.hres[sl[i]] = 0xFFFFFFFFu;
            int h = 0;  // the walk (engine.hpp:116-129) against the hashed occupancy
            while (h < mf && !a.hocc[sl[1 + h]]) ++h;
            if (h == mf) h = m;  // a free exit ending the walk never blocks (motion_rec.cuh)
            int cx[6], cy[6];
            cx[0] = rec_x(r);
            cy[0] = rec_y(r);
            record_cells(a.g, r, c_bpath_s, a.g.wrap(d->tx), d->ty, cx + 1, cy + 1);
            const uint32_t id = r.x;
            int fx = cx[0], fy = cy[0];
            bool exited = false;
            if (h > 0) {
                exited = (h == m) && (r.z & 0x80000000u);
                a.hocc[sl[0]] = 0;
                fx = cx[h];
                fy = cy[h];
                if (exited) {
                    const unsigned long long e = atomicAdd(&a.sc->strip_rexits, 1ull);
                    a.rexits[e] = ((unsigned long long)r.y << 32) | id;
                    a.alive[id] = 0;
                } else {
                    a.hocc[sl[h]] = 1;
                }
                hops += (unsigned long long)(unsigned)h +
                        ((unsigned long long)(unsigned)a.g.segment_dx(cx[0], fx) << 32);
            }
            a.x[id] = fx;
            a.y[id] = fy;
            a.owned[id] = (!exited && in_strip(a.s, fx)) ? 1 : 0;
        }
        __syncthreads();
        cur = nxt;
    }
    atomicAdd(&s_hops, hops);
    __syncthreads();
    // final occupancy of every touched cell inside this rank's window
    for (uint32_t k = threadIdx.x; k < a.nslots; k += blockDim.x) {
        const uint32_t cell = a.hkey[k];
        if (cell == 0xFFFFFFFFu) continue;
        const int x = (int)(cell % (uint32_t)a.g.W), y = (int)(cell / (uint32_t)a.g.W);
        if (!in_window(a.s, x)) continue;
        const uint32_t bit = 1u << (x & 31);
        if (a.hocc[k]) atomicOr(&a.occ[a.g.word(x, y)], bit);
        else atomicAnd(&a.occ[a.g.word(x, y)], ~bit);
    }
    if (threadIdx.x == 0) {
        a.sc->strip_rhops = s_hops;
        a.sc->pad[1] += rounds;
    }
}

// 5. global exit list (every rank's local exits + the resolved ones), alive flags of remote
// exits, step totals.  One CTA.
__global__ void __launch_bounds__(1024) strip_finish_kernel(const unsigned char* recv, const unsigned long long* rhdr,
                                                            size_t xbytes, int nranks,
                                                            uint32_t cap_def, uint32_t cap_exit, int me,
                                                            const unsigned long long* rexits, uint8_t* alive,
                                                            unsigned long long* exits, uint32_t exits_cap,
                                                            DevScalars* sc) {
    FP_PDL_WAIT();
    __shared__ unsigned long long s_base;
    if (threadIdx.x == 0) s_base = 0;
    __syncthreads();
    unsigned long long hops = 0, dx = 0;
    for (int q = 0; q < nranks; ++q) {
        const unsigned long long* h = rhdr + (size_t)q * XH_WORDS;
        const unsigned long long ne = min(h[1], (unsigned long long)cap_exit);
        const unsigned long long* xe =
            reinterpret_cast<const unsigned long long*>(recv + (size_t)q * xbytes + XH_WORDS * 8 + (size_t)cap_def * sizeof(DefRec));
        const unsigned long long base = s_base;
        for (unsigned long long i = threadIdx.x; i < ne; i += blockDim.x) {
            const unsigned long long e = xe[i];
            if (base + i < exits_cap) exits[base + i] = e;
            if (q != me) alive[(uint32_t)e] = 0;
        }
        hops += h[2];
        dx += h[3];
        __syncthreads();
        if (threadIdx.x == 0) s_base += ne;
        __syncthreads();
    }
    const unsigned long long nre = sc->strip_rexits;
    const unsigned long long base = s_base;
    for (unsigned long long i = threadIdx.x; i < nre; i += blockDim.x)
        if (base + i < exits_cap) exits[base + i] = rexits[i];
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned long long total = base + nre;
        const unsigned long long local = sc->n_exits;  // the local motion subtracted these already
        sc->n_exits = total;
        sc->alive -= total - local;
        sc->tot_exits += total - local;
        const unsigned long long rh = sc->strip_rhops;
        const unsigned long long all_hops = hops + (rh & 0xFFFFFFFFull);
        sc->tot_disp += all_hops - sc->disp;
        sc->disp = all_hops;
        const long long local_dx = sc->step_dx;
        sc->step_dx = (long long)dx + (long long)(int)(unsigned)(rh >> 32);
        sc->tot_dx += sc->step_dx - local_dx;
        sc->strip_rexits = 0;
        sc->strip_nc = 0;
        sc->exits_sorted = 0;
    }
}

__global__ void strip_reset_kernel(DevScalars* sc, unsigned long long* hdr) {
    FP_PDL_WAIT();
    sc->n_planned = 0;
    sc->strip_nc = 0;
    sc->strip_rexits = 0;
    for (int i = 0; i < XH_WORDS; ++i) hdr[i] = 0;
}

__global__ void owned_init_kernel(const int32_t* x, const uint8_t* alive, uint32_t n, Geo g, int lo, int hi,
                                  uint8_t* owned) {
    FP_PDL_WAIT();
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int px = g.wrap(x[i]);
    owned[i] = (alive[i] && px >= lo && px < hi) ? 1 : 0;
}

// ---------------------------------------------------------------------------- host side
static StripArgs strip_args(fp_ctx* c) {
    StripArgs s;
    s.g = fp_geo(c);
    s.occ = c->d_occ;
    s.occ_w = c->d_occ;
    s.p1 = c->d_p1;
    s.p2 = c->d_p2;
    s.dpl = c->st.d_dplane;
    s.rec0 = c->d_rec0;
    s.dx = c->d_dx;
    s.dy = c->d_dy;
    s.rank = c->d_rank;
    s.dflag = c->st.d_dflag;
    s.clist = c->st.d_clist;
    s.sc = c->d_sc;
    s.x_lo = c->st.x_lo;
    s.x_hi = c->st.x_hi;
    s.nranks = c->st.nranks;
    s.periodic = c->boundary == FP_BOUNDARY_PERIODIC_X;
    return s;
}

static size_t pow2_at_least(size_t v) {
    size_t p = 1;
    while (p < v) p <<= 1;
    return p;
}

int fp_strip_reserve(fp_ctx* c) {
    StripCtx& S = c->st;
    if (!S.on) return FP_OK;
    if (c->device < 64 && !g_bpath_s_ready[c->device]) {
        signed char bp[121][5][2];
        host_bpath(bp);
        FP_CUDA(c, cudaMemcpyToSymbol(c_bpath_s, bp, sizeof(bp)));
        g_bpath_s_ready[c->device] = true;
    }
    const uint32_t n = std::max<uint32_t>(c->cap, 1);
    if (S.cap_agents >= n && S.d_send) return FP_OK;
    cudaStreamSynchronize(c->stream);
    void* ptrs[] = {S.d_dplane, S.d_dflag, S.d_clist, S.d_send, S.d_recv, S.d_hkey, S.d_hres, S.d_hocc, S.d_rslot,
                    S.d_plist, S.d_rexits, S.d_rhdr};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    if (S.h_send) cudaFreeHost(S.h_send);
    if (S.h_recv) cudaFreeHost(S.h_recv);
    // capacities: a rank can defer at most the agents it owns and log at most n exits; the exchange
    // moves only the used part (counts first), so full capacity costs memory, not bandwidth
    S.cap_def = S.cap_def_req ? S.cap_def_req : n;
    S.cap_exit = S.cap_exit_req ? S.cap_exit_req : n;
    S.xbytes = (size_t)XH_WORDS * 8 + (size_t)S.cap_def * sizeof(DefRec) + (size_t)S.cap_exit * 8;
    S.xbytes = (S.xbytes + 255) & ~(size_t)255;
    S.cap_total = std::min<uint64_t>((uint64_t)S.cap_def * S.nranks, (uint64_t)n + 1);
    S.nslots = (uint32_t)pow2_at_least((size_t)S.cap_total * 12 + 1024);
    const size_t nwords = (size_t)c->P * c->H;
    FP_CUDA(c, cudaMalloc(&S.d_dplane, nwords * 4));
    FP_CUDA(c, cudaMemsetAsync(S.d_dplane, 0, nwords * 4, c->stream));
    FP_CUDA(c, cudaMalloc(&S.d_dflag, n));
    if (!S.d_owned || S.owned_cap < n) {  // ownership survives a re-reserve of the scratch
        uint8_t* o = nullptr;
        FP_CUDA(c, cudaMalloc(&o, n));
        FP_CUDA(c, cudaMemsetAsync(o, 0, n, c->stream));
        if (S.d_owned) {
            FP_CUDA(c, cudaMemcpyAsync(o, S.d_owned, S.owned_cap, cudaMemcpyDeviceToDevice, c->stream));
            FP_CUDA(c, cudaStreamSynchronize(c->stream));
            cudaFree(S.d_owned);
        }
        S.d_owned = o;
        S.owned_cap = n;
    }
    FP_CUDA(c, cudaMalloc(&S.d_clist, (size_t)n * 4));
    FP_CUDA(c, cudaMalloc(&S.d_send, S.xbytes));
    FP_CUDA(c, cudaMalloc(&S.d_recv, S.xbytes * S.nranks));
    FP_CUDA(c, cudaMalloc(&S.d_hkey, (size_t)S.nslots * 4));
    FP_CUDA(c, cudaMalloc(&S.d_hres, (size_t)S.nslots * 4));
    FP_CUDA(c, cudaMalloc(&S.d_hocc, S.nslots));
    FP_CUDA(c, cudaMalloc(&S.d_rslot, (size_t)S.cap_total * 6 * 4));
    FP_CUDA(c, cudaMalloc(&S.d_plist, (size_t)S.cap_total * 2 * 4));
    FP_CUDA(c, cudaMalloc(&S.d_rexits, (size_t)S.cap_total * 8));
    FP_CUDA(c, cudaMalloc(&S.d_rhdr, (size_t)S.nranks * XH_WORDS * 8));
    FP_CUDA(c, cudaMallocHost(&S.h_rhdr, (size_t)S.nranks * XH_WORDS * 8));
    if (S.transport == FP_STRIP_HOST) {
        FP_CUDA(c, cudaMallocHost(&S.h_send, S.xbytes));
        FP_CUDA(c, cudaMallocHost(&S.h_recv, S.xbytes * S.nranks));
    }
    S.cap_agents = n;
    c->graph_valid = false;
    return FP_OK;
}

// Phase A tail (after the plan): defer the band-connected walks and pack them.  Enqueued on
// c->stream before fp_motion_launch.
int fp_strip_defer_launch(fp_ctx* c) {
    StripCtx& S = c->st;
    const StripArgs s = strip_args(c);
    const unsigned G = (unsigned)std::min<size_t>(fp_blocks(c->n, 256), (size_t)c->sm_count * 8);
    unsigned long long* hdr = reinterpret_cast<unsigned long long*>(S.d_send);
    fp_launch(strip_mark_kernel, G, 256, 0, c->stream, s);
    FP_LAUNCHED(c);
    fp_launch(strip_seed_kernel, G, 256, 0, c->stream, s);
    FP_LAUNCHED(c);
    fp_launch(strip_closure_kernel, 1, 1024, 0, c->stream, s);
    FP_LAUNCHED(c);
    fp_launch(strip_export_kernel, G, 256, 0, c->stream,
        s, reinterpret_cast<DefRec*>(reinterpret_cast<unsigned char*>(S.d_send) + XH_WORDS * 8), S.cap_def, hdr);
    FP_LAUNCHED(c);
    const size_t nwords = (size_t)c->P * c->H;
    FP_CUDA(c, cudaMemsetAsync(c->d_p1, 0, nwords * 4, c->stream));
    FP_CUDA(c, cudaMemsetAsync(c->d_p2, 0, nwords * 4, c->stream));
    FP_CUDA(c, cudaMemsetAsync(S.d_dplane, 0, nwords * 4, c->stream));
    return FP_OK;
}

// Start of a strip step (before the plan): counters and the send header.
int fp_strip_begin_launch(fp_ctx* c) {
    fp_launch(strip_reset_kernel, 1, 1, 0, c->stream, c->d_sc, reinterpret_cast<unsigned long long*>(c->st.d_send));
    FP_LAUNCHED(c);
    return FP_OK;
}

// After the local motion: header + local exits.
int fp_strip_pack_launch(fp_ctx* c) {
    StripCtx& S = c->st;
    unsigned char* base = reinterpret_cast<unsigned char*>(S.d_send);
    fp_launch(strip_pack_kernel, 8, 256, 0, c->stream,
        c->d_sc, c->d_exits, reinterpret_cast<unsigned long long*>(base),
        reinterpret_cast<unsigned long long*>(base + XH_WORDS * 8 + (size_t)S.cap_def * sizeof(DefRec)), S.cap_exit);
    FP_LAUNCHED(c);
    return FP_OK;
}

// Phase B (after the allgather landed in d_recv): resolve, apply, global exits.
int fp_strip_resolve_launch(fp_ctx* c) {
    StripCtx& S = c->st;
    ResolveArgs a;
    a.g = fp_geo(c);
    a.recv = reinterpret_cast<const unsigned char*>(S.d_recv);
    a.rhdr = S.d_rhdr;
    a.xbytes = S.xbytes;
    a.nranks = S.nranks;
    a.cap_def = S.cap_def;
    a.hkey = S.d_hkey;
    a.hres = S.d_hres;
    a.hocc = S.d_hocc;
    a.nslots = S.nslots;
    a.rslot = S.d_rslot;
    a.plist = S.d_plist;
    a.cap_total = (uint32_t)S.cap_total;
    a.x = c->d_x;
    a.y = c->d_y;
    a.alive = c->d_alive;
    a.owned = S.d_owned;
    a.occ = c->d_occ;
    a.rexits = S.d_rexits;
    a.sc = c->d_sc;
    a.s = strip_args(c);
    fp_launch(strip_resolve_kernel, 1, RES_TAIL_THREADS, 0, c->stream, a);
    FP_LAUNCHED(c);
    fp_launch(strip_finish_kernel, 1, 1024, 0, c->stream, a.recv, S.d_rhdr, S.xbytes, S.nranks, S.cap_def, S.cap_exit, S.rank,
                                                    S.d_rexits, c->d_alive, c->d_exits, c->cap, c->d_sc);
    FP_LAUNCHED(c);
    return FP_OK;
}

int fp_strip_owned_init(fp_ctx* c) {
    if (!c->st.on || c->n == 0) return FP_OK;
    fp_launch(owned_init_kernel, fp_blocks(c->n, 256), 256, 0, c->stream, c->d_x, c->d_alive, c->n, fp_geo(c), c->st.x_lo,
                                                                   c->st.x_hi, c->st.d_owned);
    FP_LAUNCHED(c);
    return FP_OK;
}

// ---------------------------------------------------------------------------- transports
// NCCL, loaded at run time (libnccl.so.2) so the single-GPU library needs no NCCL.
typedef int (*PFN_ncclCommInitRank)(void** comm, int nranks, fp_nccl_id id, int rank);
typedef int (*PFN_ncclAllGather)(const void* send, void* recv, size_t count, int dtype, void* comm,
                                 cudaStream_t stream);
typedef int (*PFN_ncclCommDestroy)(void* comm);
typedef const char* (*PFN_ncclGetErrorString)(int);
typedef int (*PFN_ncclGetUniqueId)(fp_nccl_id* id);
typedef int (*PFN_ncclSendRecv)(void* buf, size_t count, int dtype, int peer, void* comm, cudaStream_t stream);
typedef int (*PFN_ncclGroup)();

struct NcclApi {
    void* h = nullptr;
    PFN_ncclCommInitRank init = nullptr;
    PFN_ncclAllGather allgather = nullptr;
    PFN_ncclCommDestroy destroy = nullptr;
    PFN_ncclGetErrorString err = nullptr;
    PFN_ncclGetUniqueId uid = nullptr;
    PFN_ncclSendRecv send = nullptr, recv = nullptr;
    PFN_ncclGroup gstart = nullptr, gend = nullptr;
};

static NcclApi* nccl_api() {
    static NcclApi api;
    static bool tried = false;
    if (!tried) {
        tried = true;
        const char* names[] = {getenv("FP_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
        for (const char* nm : names) {
            if (!nm) continue;
            api.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
            if (api.h) break;
        }
        if (api.h) {
            api.init = (PFN_ncclCommInitRank)dlsym(api.h, "ncclCommInitRank");
            api.allgather = (PFN_ncclAllGather)dlsym(api.h, "ncclAllGather");
            api.destroy = (PFN_ncclCommDestroy)dlsym(api.h, "ncclCommDestroy");
            api.err = (PFN_ncclGetErrorString)dlsym(api.h, "ncclGetErrorString");
            api.uid = (PFN_ncclGetUniqueId)dlsym(api.h, "ncclGetUniqueId");
            api.send = (PFN_ncclSendRecv)dlsym(api.h, "ncclSend");
            api.recv = (PFN_ncclSendRecv)dlsym(api.h, "ncclRecv");
            api.gstart = (PFN_ncclGroup)dlsym(api.h, "ncclGroupStart");
            api.gend = (PFN_ncclGroup)dlsym(api.h, "ncclGroupEnd");
        }
    }
    return (api.init && api.allgather && api.uid && api.send && api.recv && api.gstart && api.gend) ? &api : nullptr;
}

extern "C" int fp_nccl_unique_id(fp_nccl_id* out) {
    NcclApi* api = nccl_api();
    if (!api) return fp_fail(nullptr, FP_ENCCL, "NCCL: libnccl.so.2 not found (set FP_NCCL_LIB)");
    if (int r = api->uid(out)) return fp_fail(nullptr, FP_ENCCL, std::string("ncclGetUniqueId: ") + api->err(r));
    return FP_OK;
}

int fp_strip_nccl_init(fp_ctx* c, const fp_nccl_id* id) {
    NcclApi* api = nccl_api();
    if (!api) return fp_fail(c, FP_ENCCL, "NCCL: libnccl.so.2 not found (set FP_NCCL_LIB)");
    cudaSetDevice(c->device);
    if (int r = api->init(&c->st.nccl_comm, c->st.nranks, *id, c->st.rank))
        return fp_fail(c, FP_ENCCL, std::string("ncclCommInitRank: ") + api->err(r));
    return FP_OK;
}

void fp_strip_nccl_destroy(fp_ctx* c) {
    NcclApi* api = nccl_api();
    if (api && c->st.nccl_comm && api->destroy) api->destroy(c->st.nccl_comm);
    c->st.nccl_comm = nullptr;
}

// Offsets inside a payload: header, deferred records, local exits.
size_t fp_strip_def_off() { return (size_t)XH_WORDS * 8; }
size_t fp_strip_exit_off(const fp_ctx* c) { return (size_t)XH_WORDS * 8 + (size_t)c->st.cap_def * sizeof(DefRec); }
size_t fp_strip_hdr_bytes() { return (size_t)XH_WORDS * 8; }

// The exchange for the transports a single context drives itself.  Two phases: the headers
// (counts) are allgathered and read back, then exactly the used records move -- grouped
// ncclSend/ncclRecv to every peer (an allgatherv), into fixed per-rank slots of d_recv.  The host
// transport allgathers whole payloads through the callback instead.
int fp_strip_exchange(fp_ctx* c) {
    StripCtx& S = c->st;
    const size_t hb = fp_strip_hdr_bytes();
    if (S.transport == FP_STRIP_NCCL) {
        NcclApi* api = nccl_api();
        if (int r = api->allgather(S.d_send, S.d_rhdr, hb, /*ncclUint8*/ 1, S.nccl_comm, c->stream))
            return fp_fail(c, FP_ENCCL, std::string("ncclAllGather: ") + api->err(r));
        FP_CUDA(c, cudaMemcpyAsync(S.h_rhdr, S.d_rhdr, hb * S.nranks, cudaMemcpyDeviceToHost, c->stream));
        FP_CUDA(c, cudaStreamSynchronize(c->stream));
        const unsigned long long* mine = S.h_rhdr + (size_t)S.rank * XH_WORDS;
        const size_t nd = std::min<unsigned long long>(mine[0], S.cap_def), ne = std::min<unsigned long long>(mine[1], S.cap_exit);
        api->gstart();
        for (int q = 0; q < S.nranks; ++q) {
            const unsigned long long* h = S.h_rhdr + (size_t)q * XH_WORDS;
            const size_t qd = std::min<unsigned long long>(h[0], S.cap_def), qe = std::min<unsigned long long>(h[1], S.cap_exit);
            char* dst = (char*)S.d_recv + (size_t)q * S.xbytes;
            if (q == S.rank) {
                if (nd) cudaMemcpyAsync(dst + fp_strip_def_off(), (char*)S.d_send + fp_strip_def_off(), nd * sizeof(DefRec),
                                        cudaMemcpyDeviceToDevice, c->stream);
                if (ne) cudaMemcpyAsync(dst + fp_strip_exit_off(c), (char*)S.d_send + fp_strip_exit_off(c), ne * 8,
                                        cudaMemcpyDeviceToDevice, c->stream);
                continue;
            }
            if (nd) api->send((char*)S.d_send + fp_strip_def_off(), nd * sizeof(DefRec), 1, q, S.nccl_comm, c->stream);
            if (ne) api->send((char*)S.d_send + fp_strip_exit_off(c), ne * 8, 1, q, S.nccl_comm, c->stream);
            if (qd) api->recv(dst + fp_strip_def_off(), qd * sizeof(DefRec), 1, q, S.nccl_comm, c->stream);
            if (qe) api->recv(dst + fp_strip_exit_off(c), qe * 8, 1, q, S.nccl_comm, c->stream);
        }
        if (int r = api->gend()) return fp_fail(c, FP_ENCCL, std::string("ncclGroupEnd: ") + api->err(r));
        return FP_OK;
    }
    if (S.transport == FP_STRIP_HOST) {
        FP_CUDA(c, cudaMemcpyAsync(S.h_send, S.d_send, S.xbytes, cudaMemcpyDeviceToHost, c->stream));
        FP_CUDA(c, cudaStreamSynchronize(c->stream));
        if (int r = S.host_fn(S.host_user, S.h_send, S.xbytes, S.h_recv))
            return fp_fail(c, FP_ENCCL, "strip exchange callback failed (" + std::to_string(r) + ")");
        FP_CUDA(c, cudaMemcpyAsync(S.d_recv, S.h_recv, S.xbytes * S.nranks, cudaMemcpyHostToDevice, c->stream));
        FP_CUDA(c, cudaMemcpy2DAsync(S.d_rhdr, hb, S.d_recv, S.xbytes, hb, S.nranks, cudaMemcpyDeviceToDevice, c->stream));
        return FP_OK;
    }
    return fp_fail(c, FP_EINVAL, "strip: no exchange transport (fp_strip_set_nccl / fp_strip_set_exchange)");
}
