/*
 * egs_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference energy-game solver (arXiv 1710.03647
 * artifact, /root/reference/proj) used as the parity checker for the B200
 * solver.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  The product path never links it.
 *
 * Parity is PINNED: the restatement is checked against
 *   - the splitmix64 seed-0 stream published in proj/include/egsolve/rng.hpp:9-10,
 *   - the SPEC fixtures,
 *   - FNV-1a hashes of write_arena / write_solution text produced by the
 *     compiled reference library (oracle/_ref, built from /root/reference by
 *     oracle/Makefile) on the canonical generators (tests/golden/).
 *
 * Every function cites the reference file:line it restates.
 */
#ifndef EGS_ORACLE_H
#define EGS_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EO_TOP INT64_MAX /* kRawTop, proj/include/egsolve/energy.hpp:16 */

/* Error codes (mirror the egsolve::Error hierarchy, errors.hpp:11-85). */
enum {
  EO_OK = 0,
  EO_ERR_NON_TOTAL = 1,      /* NonTotalArenaError   errors.hpp:17 */
  EO_ERR_DANGLING = 2,       /* DanglingVertexIdError errors.hpp:26 */
  EO_ERR_OVERFLOW = 3,       /* OverflowError        errors.hpp:34 */
  EO_ERR_COUNT = 4,          /* CountMismatchError   errors.hpp:46 */
  EO_ERR_BOUND = 5,          /* BoundExhaustedError  errors.hpp:67 */
  EO_ERR_NO_WITNESS = 6,     /* NoWitnessError       errors.hpp:59 */
  EO_ERR_ALLOC = 7,
  EO_ERR_INVALID = 8         /* InvalidSpecError / InvalidConfigError */
};

/* GameArena (arena.hpp:37-133): dual CSR/CSC adjacency + owners + stats. */
typedef struct {
  uint32_t n;
  uint64_t m;
  uint64_t* csr_off; /* n+1 */
  uint32_t* csr_dst; /* m   */
  int64_t* csr_w;    /* m   */
  uint64_t* csc_off; /* n+1 */
  uint32_t* csc_src; /* m   */
  int64_t* csc_w;    /* m   */
  uint8_t* owner;    /* n, 0 = player 0, 1 = player 1 */
  /* ArenaStats (arena.hpp:24-31) */
  int64_t credit_cap;
  int64_t max_abs_weight;
  uint32_t max_out_degree;
  double avg_out_degree;
} eo_arena;

/* SolveReport counters (solver.hpp:47-59). */
typedef struct {
  uint64_t lifts;
  uint64_t applications;
  uint64_t pops;
  uint64_t rounds;
  uint64_t edges_relaxed;
} eo_stats;

/* splitmix64 (rng.hpp:11-37). */
uint64_t eo_splitmix64_next(uint64_t* state);
uint64_t eo_splitmix64_below(uint64_t* state, uint64_t n);
int64_t eo_splitmix64_in(uint64_t* state, int64_t lo, int64_t hi);

/* GameArena::build (arena.cpp:17-78) + compute_stats (arena.cpp:80-108). */
int eo_arena_build(uint32_t n, uint64_t m, const uint32_t* src,
                   const uint32_t* dst, const int64_t* w, const uint8_t* owner,
                   eo_arena* out);
void eo_arena_free(eo_arena* a);

/* Canonical config generators. */
int eo_gen_fixed(uint64_t n, uint32_t d, int64_t W, uint64_t seed,
                 eo_arena* out);
int eo_gen_rmat(uint32_t scale, uint32_t ef, int64_t W, uint64_t seed,
                eo_arena* out);

/* detail::raw_ominus (energy.hpp:20-31); overflow is unreachable after the
 * compute_stats headroom check so it is reported as EO_TOP-1 never. */
int64_t eo_raw_ominus(int64_t a, int64_t b);
/* detail::raw_lift (measure_ops.hpp:32-52). */
int64_t eo_raw_lift(const eo_arena* a, uint32_t v, const int64_t* f);

/* solve_seq (solver_seq.cpp:124-212): FIFO counter worklist, Alg. 1. */
int eo_solve_seq(const eo_arena* a, int64_t* f_out, eo_stats* st);
/* solve_sweep with one worker (solver_par.cpp:126-245): in-place sweeps with
 * the clamped store, BoundExhausted after `sweep_bound` sweeps (0 = default
 * budget, solver_par.cpp:94-98). */
int eo_solve_sweep(const eo_arena* a, uint64_t sweep_bound, int64_t* f_out,
                   eo_stats* st);
/* Synchronous (Jacobi) rounds of the frontier solver's activation rule
 * (solver_par.cpp:389-417) run on one thread: lift the frontier against the
 * measure of the previous round. Used to count BSP rounds. */
int eo_solve_frontier(const eo_arena* a, int64_t* f_out, eo_stats* st);

/* epm_condition_holds / is_progress_measure (measure_ops.cpp:17-41). */
int eo_epm_condition_holds(const eo_arena* a, const int64_t* f, uint32_t v);
int eo_is_progress_measure(const eo_arena* a, const int64_t* f);
/* extract_strategy (measure_ops.cpp:56-80): first satisfying CSR edge. */
int eo_extract_strategy(const eo_arena* a, const int64_t* f,
                        uint64_t* choice_edge /* n, UINT64_MAX = none */);
/* write_solution(make_solution(...)) (io.cpp:178-210). Returns the number of
 * bytes of the text; writes at most `cap` bytes into buf (buf may be NULL). */
int64_t eo_write_solution(const eo_arena* a, const int64_t* f, char* buf,
                          size_t cap);
/* write_arena (io.cpp:151-176). Same buffer protocol. */
int64_t eo_write_arena(const eo_arena* a, char* buf, size_t cap);

/* FNV-1a 64 over bytes (offset basis 0xcbf29ce484222325, prime 0x100000001b3). */
uint64_t eo_fnv1a64(const void* data, size_t len);

#ifdef __cplusplus
}
#endif
#endif
