/*
 * oracle.c -- plain-C restatement of the reference hot path (TEST INFRASTRUCTURE ONLY).
 *
 * See oracle.h for the contract.  The arithmetic is written to match the reference
 * operation for operation: fp64 everywhere the reference uses double, libm exp (the same
 * glibc the reference links), serial left-fold sums, u64 wrapping arithmetic.
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off).
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* rng.hpp:13-17 */
static uint64_t splitmix64_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* rng.hpp:21-27 */
uint64_t orc_rng_u64(uint64_t seed, uint64_t agent, uint64_t step, uint64_t draw) {
    const uint64_t v = seed ^ (agent * 0x9E3779B97F4A7C15ULL) ^ (step * 0xBF58476D1CE4E5B9ULL) ^
                       (draw * 0x94D049BB133111EBULL);
    return splitmix64_mix(v);
}

/* rng.hpp:30-32 */
double orc_unit_interval(uint64_t x) { return (double)(x >> 11) * 0x1.0p-53; }

static const uint64_t kMoveOrderStream = 1ULL << 63;      /* rng.hpp:36 */
static const uint64_t kSpawnStream = (1ULL << 63) + 1;    /* rng.hpp:37 */

/* engine.hpp:27-33 (returns -1 for the invalid_argument cases) */
int orc_compute_blocksize(int64_t agents, int cores) {
    if (cores < 1 || agents < 0) return -1;
    int64_t c = agents / cores;
    if (c > 32767) c = 32767;
    return (int)(c < 1 ? 1 : c);
}

double orc_exp(double x) { return exp(x); }

static int wrap_x(int32_t w, int32_t boundary, int x) {
    /* world.hpp:72-78 */
    if (boundary == ORC_PERIODIC_X) {
        x %= w;
        if (x < 0) x += w;
    }
    return x;
}

/* world.hpp:125-132 */
int orc_segment_dx(int32_t w, int32_t boundary, int32_t ax, int32_t bx) {
    int d = bx - ax;
    if (boundary == ORC_PERIODIC_X) {
        const int alt = d > 0 ? d - w : d + w;
        if (abs(alt) < abs(d)) d = alt;
    }
    return d;
}

/* world.hpp:143-167 (walk_segment), collecting the visited cells */
int orc_trace(int32_t w, int32_t boundary, int32_t ax, int32_t ay, int32_t bx, int32_t by,
              int32_t* out_x, int32_t* out_y, int cap) {
    ax = wrap_x(w, boundary, ax);
    bx = wrap_x(w, boundary, bx);
    const int tx = ax + orc_segment_dx(w, boundary, ax, bx);
    const int dx = abs(tx - ax);
    const int sx = ax < tx ? 1 : -1;
    const int dy = -abs(by - ay);
    const int sy = ay < by ? 1 : -1;
    int err = dx + dy;
    int x = ax, y = ay, n = 0;
    while (!(x == tx && y == by)) {
        const int e2 = 2 * err;
        if (e2 >= dy) { err += dy; x += sx; }
        if (e2 <= dx) { err += dx; y += sy; }
        if (n < cap) { out_x[n] = wrap_x(w, boundary, x); out_y[n] = y; }
        ++n;
    }
    return n;
}

static uint8_t cell_at(const orc_state* st, int x, int y) {
    return st->cells[(size_t)y * (size_t)st->width + (size_t)wrap_x(st->width, st->boundary, x)];
}

/* world.hpp:181-191 */
int orc_line_of_sight(const orc_state* st, int32_t ax, int32_t ay, int32_t bx, int32_t by) {
    int32_t px[64], py[64];
    const int n = orc_trace(st->width, st->boundary, ax, ay, bx, by, px, py, 64);
    for (int i = 0; i < n && i < 64; ++i)
        if (cell_at(st, px[i], py[i]) == ORC_WALL) return 0;
    return 1;
}

/* ---- world.hpp:220-266: multi-source Dijkstra, binary heap with lazy deletion ---- */
typedef struct { double d; int32_t idx; } heap_item;

static int item_less(heap_item a, heap_item b) {
    /* std::greater<pair<double,int32>> => min-heap on (d, idx) */
    return a.d < b.d || (a.d == b.d && a.idx < b.idx);
}

static void heap_push(heap_item* h, size_t* n, heap_item it) {
    size_t i = (*n)++;
    h[i] = it;
    while (i > 0) {
        size_t p = (i - 1) / 2;
        if (!item_less(h[i], h[p])) break;
        heap_item t = h[i]; h[i] = h[p]; h[p] = t;
        i = p;
    }
}

static heap_item heap_pop(heap_item* h, size_t* n) {
    heap_item top = h[0];
    h[0] = h[--(*n)];
    size_t i = 0;
    for (;;) {
        size_t l = 2 * i + 1, r = l + 1, m = i;
        if (l < *n && item_less(h[l], h[m])) m = l;
        if (r < *n && item_less(h[r], h[m])) m = r;
        if (m == i) break;
        heap_item t = h[i]; h[i] = h[m]; h[m] = t;
        i = m;
    }
    return top;
}

void orc_static_field(int32_t w, int32_t h, int32_t boundary, const uint8_t* cells, double* s) {
    const size_t n = (size_t)w * (size_t)h;
    for (size_t i = 0; i < n; ++i) s[i] = INFINITY;
    size_t cap = n * 8 + 16, hn = 0;
    heap_item* heap = (heap_item*)malloc(cap * sizeof(heap_item));
    for (size_t i = 0; i < n; ++i)
        if (cells[i] == ORC_EXIT) {
            s[i] = 0.0;
            heap_item it = {0.0, (int32_t)i};
            heap_push(heap, &hn, it);
        }
    static const int off[8][2] = {{-1, -1}, {0, -1}, {1, -1}, {-1, 0}, {1, 0}, {-1, 1}, {0, 1}, {1, 1}};
    const double diag = sqrt(2.0);
    while (hn > 0) {
        const heap_item it = heap_pop(heap, &hn);
        if (it.d > s[it.idx]) continue;
        const int cx = it.idx % w, cy = it.idx / w;
        for (int k = 0; k < 8; ++k) {
            const int ox = off[k][0], oy = off[k][1];
            const int ny = cy + oy;
            if (ny < 0 || ny >= h) continue;
            int nx = cx + ox;
            if (boundary == ORC_PERIODIC_X) nx = wrap_x(w, boundary, nx);
            else if (nx < 0 || nx >= w) continue;
            if (cells[(size_t)ny * w + nx] == ORC_WALL) continue;
            if (ox != 0 && oy != 0) { /* world.hpp:212-216 diagonal_blocked */
                const int sax = wrap_x(w, boundary, cx + ox);
                if (cells[(size_t)cy * w + sax] == ORC_WALL && cells[(size_t)ny * w + cx] == ORC_WALL)
                    continue;
            }
            const double nd = it.d + ((ox != 0 && oy != 0) ? diag : 1.0);
            const size_t ni = (size_t)ny * w + nx;
            if (nd < s[ni]) {
                s[ni] = nd;
                if (hn == cap) { cap *= 2; heap = (heap_item*)realloc(heap, cap * sizeof(heap_item)); }
                heap_item nt = {nd, (int32_t)ni};
                heap_push(heap, &hn, nt);
            }
        }
    }
    free(heap);
}

/* ---- planning.hpp:23-57 ---- */
static int occupant(const orc_state* st, int x, int y) {
    return st->occ[(size_t)y * st->width + wrap_x(st->width, st->boundary, x)];
}

int orc_enumerate_candidates(const orc_state* st, int32_t agent, int32_t* cx, int32_t* cy) {
    const int v = st->v_max[agent];
    const int px = wrap_x(st->width, st->boundary, st->x[agent]);
    const int py = st->y[agent];
    const int periodic = st->boundary == ORC_PERIODIC_X;
    const int y_lo = py - v < 0 ? 0 : py - v;
    const int y_hi = py + v > st->height - 1 ? st->height - 1 : py + v;
    const int wraps = periodic && 2 * v + 1 > st->width;
    int n = 0;
    for (int y = y_lo; y <= y_hi; ++y) {
        const int row_start = n;
        for (int dx = -v; dx <= v; ++dx) {
            int x = px + dx;
            if (periodic) x = wrap_x(st->width, st->boundary, x);
            else if (x < 0 || x >= st->width) continue;
            if (cell_at(st, x, y) == ORC_WALL) continue;
            const int occ = occupant(st, x, y);
            if (occ != -1 && occ != agent) continue;
            if (!orc_line_of_sight(st, px, py, x, y)) continue;
            cx[n] = x; cy[n] = y; ++n;
        }
        /* rows are sorted by wrapped x (planning.hpp:50-53): insertion sort of this row */
        for (int i = row_start + 1; i < n; ++i) {
            const int tx = cx[i];
            int j = i - 1;
            while (j >= row_start && cx[j] > tx) { cx[j + 1] = cx[j]; --j; }
            cx[j + 1] = tx;
        }
    }
    if (wraps) { /* planning.hpp:55 std::unique */
        int m = 0;
        for (int i = 0; i < n; ++i)
            if (m == 0 || cx[i] != cx[m - 1] || cy[i] != cy[m - 1]) { cx[m] = cx[i]; cy[m] = cy[i]; ++m; }
        n = m;
    }
    return n;
}

/* planning.hpp:63-73 */
int64_t orc_sample_index(const double* w, int64_t n, double u) {
    double total = 0.0;
    for (int64_t i = 0; i < n; ++i) total += w[i];
    const double threshold = u * total;
    double cum = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        cum += w[i];
        if (cum > threshold) return i;
    }
    return n - 1;
}

/* planning.hpp:88-104: candidate list + weights; returns the count */
int orc_choice_weights(const orc_state* st, int32_t agent, double k_s, double* w, int32_t* cx,
                       int32_t* cy) {
    const int n = orc_enumerate_candidates(st, agent, cx, cy);
    const int px = wrap_x(st->width, st->boundary, st->x[agent]);
    const int py = st->y[agent];
    const int exitd = st->potential == ORC_EXIT_DISTANCE;
    const size_t W = (size_t)st->width;
    if (exitd && !isfinite(st->field[(size_t)py * W + px])) {
        for (int i = 0; i < n; ++i) w[i] = 1.0;
        return n;
    }
    for (int i = 0; i < n; ++i) {
        const double sc = exitd ? st->field[(size_t)cy[i] * W + cx[i]] : 0.0;
        if (exitd && !isfinite(sc)) { w[i] = 0.0; continue; }
        double drop; /* planning.hpp:76-80 potential_drop */
        if (!exitd)
            drop = st->drive_gradient * (double)orc_segment_dx(st->width, st->boundary, px, cx[i]);
        else
            drop = st->field[(size_t)py * W + px] - sc;
        w[i] = exp(k_s * drop);
    }
    return n;
}

/* planning.hpp:88-108 */
void orc_choose_desired(const orc_state* st, int32_t agent, double k_s, uint64_t seed,
                        int32_t* out_x, int32_t* out_y) {
    double w[128];
    int32_t cx[128], cy[128];
    const int n = orc_choice_weights(st, agent, k_s, w, cx, cy);
    const double u = orc_unit_interval(orc_rng_u64(seed, (uint64_t)agent, (uint64_t)st->step, 0));
    const int64_t k = orc_sample_index(w, n, u);
    *out_x = cx[k];
    *out_y = cy[k];
}

/* engine.hpp:71-84 (single worker: results are worker-count independent) */
void orc_plan_phase(orc_state* st, double k_s, uint64_t seed) {
    if (st->alive_count == 0) return;
    for (int32_t i = 0; i < st->n; ++i) {
        if (!st->alive[i]) continue;
        orc_choose_desired(st, i, k_s, seed, &st->desired_x[i], &st->desired_y[i]);
    }
}

/* engine.hpp:99-111: Fisher-Yates over positions 0..n-1 (caller maps to alive ids) */
void orc_movement_order(int64_t n, uint64_t seed, int64_t step, uint32_t* order) {
    for (int64_t i = 0; i < n; ++i) order[i] = (uint32_t)i;
    uint64_t draw = 0;
    for (int64_t i = n; i-- > 1;) {
        const uint64_t r = orc_rng_u64(seed, kMoveOrderStream, (uint64_t)step, draw++);
        const uint64_t j = r % (uint64_t)(i + 1);
        const uint32_t t = order[i]; order[i] = order[j]; order[j] = t;
    }
}

/* engine.hpp:95-135; returns displacement, fills exited ids in processing order */
int64_t orc_move_phase(orc_state* st, uint64_t seed, uint32_t* exited, int64_t* n_exited) {
    const int W = st->width;
    int64_t n = 0;
    uint32_t* order = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(st->n + 1));
    for (int32_t i = 0; i < st->n; ++i)
        if (st->alive[i]) order[n++] = (uint32_t)i;
    uint64_t draw = 0;
    for (int64_t i = n; i-- > 1;) {
        const uint64_t r = orc_rng_u64(seed, kMoveOrderStream, (uint64_t)st->step, draw++);
        const uint64_t j = r % (uint64_t)(i + 1);
        const uint32_t t = order[i]; order[i] = order[j]; order[j] = t;
    }
    int64_t disp = 0, ne = 0;
    int32_t px[64], py[64];
    for (int64_t k = 0; k < n; ++k) {
        const uint32_t idx = order[k];
        const int m = orc_trace(W, st->boundary, st->x[idx], st->y[idx], st->desired_x[idx],
                                st->desired_y[idx], px, py, 64);
        int hops = 0;
        for (int s = 0; s < m && s < 64; ++s) {
            const int cx = px[s], cy = py[s];
            if (hops >= st->v_max[idx]) break;
            const uint8_t kind = st->cells[(size_t)cy * W + cx];
            if (kind == ORC_WALL) break;
            if (st->occ[(size_t)cy * W + cx] != -1) break;
            st->occ[(size_t)st->y[idx] * W + wrap_x(W, st->boundary, st->x[idx])] = -1;
            st->x[idx] = cx;
            st->y[idx] = cy;
            ++hops;
            if (kind == ORC_EXIT) {
                st->alive[idx] = 0;
                --st->alive_count;
                if (exited) exited[ne] = idx;
                ++ne;
                break;
            }
            st->occ[(size_t)cy * W + cx] = (int32_t)idx;
        }
        disp += hops;
    }
    free(order);
    if (n_exited) *n_exited = ne;
    return disp;
}

void orc_rebuild_occupancy(orc_state* st) {
    const size_t n = (size_t)st->width * (size_t)st->height;
    for (size_t i = 0; i < n; ++i) st->occ[i] = -1;
    st->alive_count = 0;
    for (int32_t i = 0; i < st->n; ++i) {
        if (!st->alive[i]) continue;
        st->occ[(size_t)st->y[i] * st->width + wrap_x(st->width, st->boundary, st->x[i])] = i;
        ++st->alive_count;
    }
}

/* scenario_io.hpp:47-69 (returns -1 when n exceeds the free-cell count) */
int orc_spawn_agents(int32_t w, int32_t h, const uint8_t* cells, int64_t n, uint64_t seed,
                     int32_t* out_x, int32_t* out_y) {
    const size_t total = (size_t)w * (size_t)h;
    size_t nfree = 0;
    for (size_t i = 0; i < total; ++i) nfree += cells[i] == ORC_FREE;
    if (n < 0 || (size_t)n > nfree) return -1;
    uint32_t* fr = (uint32_t*)malloc(sizeof(uint32_t) * (nfree + 1));
    size_t k = 0;
    for (size_t i = 0; i < total; ++i)
        if (cells[i] == ORC_FREE) fr[k++] = (uint32_t)i;
    uint64_t draw = 0;
    for (int64_t i = 0; i < n; ++i) {
        const uint64_t r = orc_rng_u64(seed, kSpawnStream, 0, draw++);
        const size_t j = (size_t)i + (size_t)(r % (uint64_t)(nfree - (size_t)i));
        const uint32_t t = fr[i]; fr[i] = fr[j]; fr[j] = t;
    }
    for (int64_t i = 0; i < n; ++i) {
        out_x[i] = (int32_t)(fr[i] % (uint32_t)w);
        out_y[i] = (int32_t)(fr[i] / (uint32_t)w);
    }
    free(fr);
    return 0;
}

/* state.hpp:80-95 */
uint64_t orc_state_hash(const orc_state* st) {
    uint64_t h = 14695981039346656037ULL;
#define MIX(v) do { h ^= (uint64_t)(v); h *= 1099511628211ULL; } while (0)
    MIX((uint64_t)st->step);
    MIX((uint64_t)st->alive_count);
    for (int32_t i = 0; i < st->n; ++i) {
        MIX((uint32_t)i);
        MIX((uint32_t)st->x[i]);
        MIX((uint32_t)st->y[i]);
        MIX(st->alive[i] ? 1 : 0);
    }
#undef MIX
    return h;
}
