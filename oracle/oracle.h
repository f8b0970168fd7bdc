/*
 * oracle.h -- CPU restatement of the F.A.S.T. reference engine's hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the checker the CUDA path is compared against;
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load it.  The product (paper_0911_2900_b200/) never links or calls it.
 *
 * Every function cites the reference file:line it restates.  Paths are relative to
 * /root/reference/proj/include/fastped/.  Pinned against: the reference's golden
 * vectors (tests/test_rng.cpp:17-19, tests/test_engine.cpp:35-43, tests/test_planning.cpp)
 * and against the reference itself compiled here into oracle/_ref (tests/test_oracle_*.py,
 * fixtures under tests/golden/ produced by tests/golden/make_golden.py).
 */
#ifndef FASTPED_ORACLE_H
#define FASTPED_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_FREE = 0, ORC_WALL = 1, ORC_EXIT = 2 };
enum { ORC_CLOSED = 0, ORC_PERIODIC_X = 1 };
enum { ORC_EXIT_DISTANCE = 0, ORC_DRIVE_X = 1 };

/* SimState restated as plain SoA arrays (state.hpp:22-36, agents.hpp:13-18). */
typedef struct {
    int32_t width, height, boundary;
    const uint8_t* cells;  /* W*H CellKind, row-major y*W+x (world.hpp:88-91) */
    const double* field;   /* W*H, +inf = unreachable (world.hpp:196-208) */
    int32_t n;             /* agents; id == index (state.hpp:54-55) */
    int32_t* x;
    int32_t* y;
    int32_t* v_max;
    uint8_t* alive;
    int32_t* occ;          /* W*H, agent id or -1 (state.hpp:23,28) */
    int32_t* desired_x;
    int32_t* desired_y;
    int64_t step;
    int64_t alive_count;
    int32_t potential;
    double drive_gradient;
} orc_state;

uint64_t orc_rng_u64(uint64_t seed, uint64_t agent, uint64_t step, uint64_t draw);
double orc_unit_interval(uint64_t x);
int orc_compute_blocksize(int64_t agents, int cores);
int orc_segment_dx(int32_t w, int32_t boundary, int32_t ax, int32_t bx);
/* Visits the Bresenham cells a->b (exclusive a, inclusive b); writes up to cap cells. */
int orc_trace(int32_t w, int32_t boundary, int32_t ax, int32_t ay, int32_t bx, int32_t by,
              int32_t* out_x, int32_t* out_y, int cap);
int orc_line_of_sight(const orc_state* st, int32_t ax, int32_t ay, int32_t bx, int32_t by);
void orc_static_field(int32_t w, int32_t h, int32_t boundary, const uint8_t* cells, double* out);
int orc_enumerate_candidates(const orc_state* st, int32_t agent, int32_t* cx, int32_t* cy);
int64_t orc_sample_index(const double* w, int64_t n, double u);
int orc_choice_weights(const orc_state* st, int32_t agent, double k_s, double* w, int32_t* cx,
                       int32_t* cy);
void orc_choose_desired(const orc_state* st, int32_t agent, double k_s, uint64_t seed,
                        int32_t* out_x, int32_t* out_y);
void orc_plan_phase(orc_state* st, double k_s, uint64_t seed);
void orc_movement_order(int64_t n, uint64_t seed, int64_t step, uint32_t* order);
int64_t orc_move_phase(orc_state* st, uint64_t seed, uint32_t* exited, int64_t* n_exited);
void orc_rebuild_occupancy(orc_state* st);
int orc_spawn_agents(int32_t w, int32_t h, const uint8_t* cells, int64_t n, uint64_t seed,
                     int32_t* out_x, int32_t* out_y);
uint64_t orc_state_hash(const orc_state* st);
double orc_exp(double x);

#ifdef __cplusplus
}
#endif
#endif
