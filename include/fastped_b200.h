/*
 * fastped_b200.h -- C ABI of the B200-native F.A.S.T. planning + motion engine.
 *
 * The reference (/root/reference/proj/include/fastped, header-only C++20) has no FFI, plugin
 * or operator registry: its boundary is the `namespace fastped` API.  This header is the thin
 * C layer that API's drop-in replacement (include/fastped_b200/fastped.hpp, C++) and the
 * Python binding (paper_0911_2900_b200/fastped.py, ctypes) call.  Each entry point names the
 * reference function it stands in for.
 *
 * Conventions
 *  - Every function returns FP_OK (0) or an FP_E* status; fp_last_error(ctx) (or
 *    fp_last_error(NULL) for context-free calls) holds a message whose wording follows the
 *    reference's exception text where one exists (std::invalid_argument -> FP_EINVAL,
 *    std::runtime_error -> FP_ERUNTIME).
 *  - All host buffers are caller-owned and copied; nothing is retained after a call returns.
 *  - A context is single-owner and not thread-safe (SimState's "one controller" rule,
 *    state.hpp:19-21).  It owns one CUDA device, one stream and all device-resident state.
 *  - Cells are row-major, index y*width + x (world.hpp:88-91); CellKind bytes 0 Free, 1 Wall,
 *    2 Exit (world.hpp:18); boundary 0 Closed, 1 PeriodicX (world.hpp:19).
 *  - There is no CPU fallback: without a usable sm_100 device every compute call fails with
 *    FP_ECUDA.
 */
#ifndef FASTPED_B200_H
#define FASTPED_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FP_OK 0
#define FP_EINVAL 1   /* std::invalid_argument in the reference */
#define FP_ERUNTIME 2 /* std::runtime_error in the reference */
#define FP_ECUDA 3    /* CUDA runtime / device failure (no GPU, OOM, kernel fault) */
#define FP_ENCCL 4    /* NCCL failure on the multi-GPU strip path */

#define FP_CELL_FREE 0
#define FP_CELL_WALL 1
#define FP_CELL_EXIT 2
#define FP_BOUNDARY_CLOSED 0
#define FP_BOUNDARY_PERIODIC_X 1
#define FP_POTENTIAL_EXIT_DISTANCE 0 /* Potential::ExitDistance, state.hpp:17 */
#define FP_POTENTIAL_DRIVE_X 1       /* Potential::DriveX */

typedef struct fp_ctx fp_ctx;

/* Grid(width, height, cell_size, boundary, cells) -- world.hpp:37-63 */
typedef struct {
    int32_t width;
    int32_t height;
    double cell_size;
    int32_t boundary;
} fp_grid_desc;

/* StepStats -- engine.hpp:137-141 */
typedef struct {
    int64_t alive;
    int64_t exited;
    int64_t displacement_cells;
} fp_step_stats;

/* RunStats -- engine.hpp:150-158 (times from CUDA events on the context's stream) */
typedef struct {
    double wall_time_s;
    double plan_time_s;
    double move_time_s;
    int64_t steps;
    int64_t exited;
    int64_t displacement_cells;
    int64_t alive;
    int64_t agent_updates; /* sum over steps of the alive count entering the step */
} fp_run_stats;

/* Engine counters for observability (not in the reference). */
typedef struct {
    int64_t kernel_launches;   /* kernels launched on this context so far */
    int64_t motion_rounds;     /* conflict-resolution rounds executed */
    int64_t plan_fallbacks;    /* agents re-sampled on the exact fp64 path */
    int64_t planned_agents;    /* agents planned */
    int64_t motion_seed_ns;    /* last motion phase: seed pass (device globaltimer) */
    int64_t motion_grid_ns;    /*   grid-wide rounds */
    int64_t motion_tail_ns;    /*   single-CTA tail rounds */
    int64_t motion_grid_rounds;/*   rounds run grid-wide in the last phase */
    int64_t motion_mark_ns;    /*   of the seed pass: contention marking */
    int64_t motion_contended;  /*   movers whose footprint overlapped another's */
    int64_t motion_prep_ns;    /*   of the grid rounds: interning the contended footprints */
} fp_counters;

const char* fp_version(void);
/* CUDA devices visible to the library (strip placement). */
int fp_device_count(int* n);
const char* fp_last_error(const fp_ctx* ctx);

/* compute_blocksize(number_of_agents, cores) -- engine.hpp:27-33 (host arithmetic). */
int fp_compute_blocksize(int64_t number_of_agents, int cores, int32_t* out);

/* Grid validation + device upload; field == NULL computes compute_static_field on the device
 * (world.hpp:220-266, bit-identical).  `device` is the CUDA ordinal. */
int fp_create(const fp_grid_desc* grid, const uint8_t* cells, const double* field, int device,
              fp_ctx** out);
void fp_destroy(fp_ctx* ctx);

/* compute_static_field(grid) -- world.hpp:220-266, on the device, context-free. */
int fp_static_field(const fp_grid_desc* grid, const uint8_t* cells, int device, double* out_s);
/* StaticField::s of a context (fp64, +inf = unreachable). */
int fp_get_field(const fp_ctx* ctx, double* out_s);

/* make_state(grid, field, roster) -- state.hpp:38-76.  Ids are dense indices; v_max per agent
 * (1..5); alive may be NULL (all alive).  Validates like make_state (bounds, wall, shared cell)
 * except that heterogeneous v_max is accepted (the kernels read the per-agent value, as the
 * reference's planning.hpp:25 / engine.hpp:117 do). */
int fp_set_agents(fp_ctx* ctx, uint32_t n, const int32_t* x, const int32_t* y,
                  const int32_t* v_max, const uint8_t* alive, int64_t step);
/* Re-uploads positions/alive of the current roster (the drop-in's per-call host sync). */
int fp_update_agents(fp_ctx* ctx, const int32_t* x, const int32_t* y, const uint8_t* alive);
/* SimState::step */
int fp_set_step(fp_ctx* ctx, int64_t step);
int fp_get_step(const fp_ctx* ctx, int64_t* step);
int fp_get_alive_count(const fp_ctx* ctx, int64_t* alive);
/* Sum over all agents of segment_dx(x before, x after) for the last move phase (step / move /
 * each step of run): the per-step x displacement fundamental_diagram accumulates on the host
 * from positions (bench.hpp:291-302), reduced on the device during the walks instead. */
int fp_get_last_dx(const fp_ctx* ctx, int64_t* dx);
/* The same sum over every step of the last fp_run (the fundamental diagram's flow over a run). */
int fp_get_run_dx(const fp_ctx* ctx, int64_t* dx);
/* SimState::potential / drive_gradient -- state.hpp:32-33 */
int fp_set_potential(fp_ctx* ctx, int kind, double drive_gradient);
/* SimState::desired (scratch between phases); injected by motion-only tests. */
int fp_set_desired(fp_ctx* ctx, const int32_t* x, const int32_t* y);

/* plan_phase(st, params, sched) -- engine.hpp:71-84: desired cell of every alive agent,
 * bit-identical to choose_desired_cell (planning.hpp:88-108). */
int fp_plan(fp_ctx* ctx, double k_s, uint64_t seed);
/* move_phase(st, params) -- engine.hpp:95-135 (does not advance the step counter).
 * Exited ids (processing order) are kept for fp_get_exited. */
int fp_move(fp_ctx* ctx, uint64_t seed, fp_step_stats* out);
/* step(st, params, sched) -- engine.hpp:143-148. */
int fp_step(fp_ctx* ctx, double k_s, uint64_t seed, fp_step_stats* out);
/* run(st, params, sched) -- engine.hpp:161-183: `steps` steps, device-resident, event-timed. */
int fp_run(fp_ctx* ctx, double k_s, uint64_t seed, int32_t steps, fp_run_stats* out);

/* Dumps (trajectory / occupancy): SimState::agents, desired, occupancy (id or -1). */
int fp_get_agents(const fp_ctx* ctx, int32_t* x, int32_t* y, uint8_t* alive);
int fp_get_desired(const fp_ctx* ctx, int32_t* x, int32_t* y);
int fp_get_occupancy(const fp_ctx* ctx, int32_t* occ);
/* MoveOutcome::exited of the last fp_move/fp_step (ids in processing order). */
int fp_get_exited(const fp_ctx* ctx, uint32_t* ids, uint32_t cap, uint32_t* n);
/* The last step's movement order (alive ids in processing order, engine.hpp:99-111). */
int fp_get_order(const fp_ctx* ctx, uint32_t* ids, uint32_t cap, uint32_t* n);
/* state_hash(st) -- state.hpp:80-95. */
int fp_state_hash(const fp_ctx* ctx, uint64_t* out);
/* state_hash of a roster given by host arrays (e.g. merged from strip ranks). */
int fp_hash_roster(int64_t step, int64_t alive, uint32_t n, const int32_t* x, const int32_t* y, const uint8_t* alive_flags,
                   uint64_t* out);

/* Test mode: candidate list of one agent in the reference order (enumerate_candidates,
 * planning.hpp:23-57), its exact fp64 weights (planning.hpp:93-103), and the choice
 * probabilities of the production sampling path (fp32). */
int fp_get_choice(fp_ctx* ctx, uint32_t agent, double k_s, int32_t* cx, int32_t* cy,
                  double* weights, float* probs, uint32_t cap, uint32_t* n);

/* Host API of planning.hpp for ONE agent given by value against the context's current occupancy
 * (the reference's `const SimState&` snapshot), computed on the device with the exact path:
 *   choose_desired_cell(st, agent, params) -- planning.hpp:88-108, uniform
 *       rng_u64(seed, id, step, 0); `step` is SimState::step as the caller holds it;
 *   enumerate_candidates(st, agent) -- planning.hpp:23-57, list order (<= 121 cells). */
int fp_choose_desired(fp_ctx* ctx, uint32_t id, int32_t x, int32_t y, int32_t v_max, int64_t step,
                      double k_s, uint64_t seed, int32_t* out_x, int32_t* out_y);
int fp_enumerate_candidates(fp_ctx* ctx, int32_t x, int32_t y, int32_t v_max, int32_t* cx, int32_t* cy,
                            uint32_t cap, uint32_t* n);

/* The movement permutation of positions 0..n-1 for (seed, step) computed by the device
 * (engine.hpp:99-111 Fisher-Yates), context-free. */
int fp_movement_order(int64_t n, uint64_t seed, int64_t step, int device, uint32_t* out);

/* spawn_agents(grid, n, v_max, seed) positions -- scenario_io.hpp:47-69 (host, setup). */
int fp_spawn_agents(int32_t width, int32_t height, const uint8_t* cells, int64_t n,
                    uint64_t seed, int32_t* x, int32_t* y);

int fp_get_counters(const fp_ctx* ctx, fp_counters* out);

/* ---- Multi-GPU: x-strip decomposition of one simulation (strip.cu) ----
 * Rank r of N owns the agents standing in columns [x_lo, x_hi) (strips tile the grid; periodic
 * grids form a ring).  Every rank gets the same grid, field and GLOBAL roster; ids stay global.
 * Walks that can touch another strip (and everything sharing a cell with them) are exchanged
 * and resolved on every rank each step, so the result equals the 1-GPU run bit for bit.
 * fp_step / fp_run on a strip context run the decomposed step; fp_plan / fp_move do not.
 * Transports: NCCL (fp_strip_set_nccl: one process per GPU, ncclAllGather on the context's
 * stream; libnccl.so.2 is loaded at run time), a host allgather callback
 * (fp_strip_set_exchange: recv receives the N payloads in rank order), or all ranks in this
 * process (fp_strips_step / fp_strips_run: device-to-device copies, e.g. virtual strips on one
 * GPU).  Positions of agents another rank owns are stale: fp_strip_get_owned says which of a
 * rank's fp_get_agents entries are its own.  Exits, alive counts and stats are global. */
typedef struct {
    char internal[128];
} fp_nccl_id; /* ncclUniqueId */
typedef int (*fp_allgather_fn)(void* user, const void* send, size_t bytes, void* recv);
int fp_strip_bounds(int32_t width, int rank, int nranks, int32_t* x_lo, int32_t* x_hi);
/* cap_deferred / cap_exits: exchange capacity per rank and step (0 = defaults sized by the roster). */
int fp_strip_config(fp_ctx* ctx, int rank, int nranks, int32_t x_lo, int32_t x_hi, uint32_t cap_deferred,
                    uint32_t cap_exits);
int fp_nccl_unique_id(fp_nccl_id* out);
int fp_strip_set_nccl(fp_ctx* ctx, const fp_nccl_id* id);
int fp_strip_set_exchange(fp_ctx* ctx, fp_allgather_fn fn, void* user);
int fp_strips_step(fp_ctx* const* ctxs, int n, double k_s, uint64_t seed, fp_step_stats* out);
int fp_strips_run(fp_ctx* const* ctxs, int n, double k_s, uint64_t seed, int32_t steps, fp_run_stats* out);
int fp_strip_get_owned(const fp_ctx* ctx, uint8_t* owned);

/* Benchmark helper: average duration (ms, CUDA events) of `iters` launches of the planning
 * kernel alone on the current state (bucketing done once, untimed). */
int fp_time_plan_kernel(fp_ctx* ctx, double k_s, uint64_t seed, int32_t iters, double* ms_per_launch);

#ifdef __cplusplus
}
#endif
#endif
