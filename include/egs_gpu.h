/*
 * egs_gpu.h — C-ABI of the B200-native energy-game solver (libegs_b200.so).
 *
 * This is the drop-in boundary for the reference solve path of the
 * arXiv 1710.03647 artifact (/root/reference/proj).  The reference binds the
 * path through one C++ entry point,
 *
 *     SolveReport egsolve::solve(const GameArena&, Variant,
 *                                const SolverOptions& = {});
 *                                          proj/include/egsolve/solver.hpp:86-87
 *
 * (dispatch proj/src/solver_seq.cpp:233-244, parallel solvers
 * proj/src/solver_par.cpp:126-435).  The C++ shim a maintainer adds next to it
 * flattens the GameArena spans (arena.hpp:109-115) into an
 * egs_arena_view, calls egs_gpu_solve, and rebuilds a SolveReport with the
 * reference's own winning_sets (measure_ops.cpp:43-54).  Plain pointers and
 * sizes only; no CUDA or torch types cross this boundary.
 *
 * Return codes mirror the exceptions the reference solve path can raise
 * (errors.hpp:11-85):
 *   EGS_OK 0, EGS_ERR_INVALID_CONFIG 1 (InvalidConfigError),
 *   EGS_ERR_TIMEOUT 2 (TimeoutError), EGS_ERR_UNSUPPORTED 3 (OverflowError:
 *   an arena outside the device representation), EGS_ERR_CUDA 4 (device or
 *   NCCL failure), EGS_ERR_BOUND 5 (BoundExhaustedError), EGS_ERR_INTERNAL 6
 *   (InternalInvariantError, debug checks), EGS_ERR_INPUT 7 (the loader's
 *   SyntaxError / CountMismatchError / DanglingVertexIdError /
 *   NonTotalArenaError).  egs_last_error() gives the text.
 */
#ifndef EGS_GPU_H
#define EGS_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EGS_OK 0
#define EGS_ERR_INVALID_CONFIG 1
#define EGS_ERR_TIMEOUT 2
#define EGS_ERR_UNSUPPORTED 3
#define EGS_ERR_CUDA 4
#define EGS_ERR_BOUND 5
#define EGS_ERR_INTERNAL 6
#define EGS_ERR_INPUT 7    /* malformed arena input; egs_last_error() reads
                              "<Kind>: <message>" with Kind one of the
                              reference's loader errors (errors.hpp:16-46):
                              SyntaxError ("line N: ..."), CountMismatchError,
                              DanglingVertexIdError, NonTotalArenaError */

/* Flattened GameArena (arena.hpp:37-133).  All pointers are HOST memory and
 * are only read during the call.  CSC spans are not needed: the predecessor
 * transpose is rebuilt on the device. */
typedef struct egs_arena_view {
  uint32_t num_vertices;        /* GameArena::num_vertices()  arena.hpp:86 */
  uint64_t num_edges;           /* GameArena::num_edges()     arena.hpp:87 */
  const uint64_t* csr_offsets;  /* n+1   csr_offsets()  arena.hpp:109 */
  const uint32_t* csr_targets;  /* m     csr_targets()  arena.hpp:110 */
  const int64_t* csr_weights;   /* m     csr_weights()  arena.hpp:111 */
  const uint8_t* owners;        /* n     owners(): 0 = player 0, 1 = player 1 */
  int64_t credit_cap;           /* stats().credit_cap (M_G) arena.hpp:27 */
  int64_t max_abs_weight;       /* stats().max_abs_weight   arena.hpp:28 */
} egs_arena_view;

/* Mode selector for the lift rounds. */
#define EGS_MODE_AUTO 0   /* dense/sparse switch on frontier edge volume */
#define EGS_MODE_DENSE 1  /* every round lifts every vertex (Alg. 2 shape) */
#define EGS_MODE_SPARSE 2 /* worklist rounds only (Alg. 3 shape) */
#define EGS_MODE_SWEEP 3  /* every round lifts every vertex IN PLACE, reading
                             its successors' current values: the reference's
                             solve_sweep (Alg. 2, solver_par.cpp:205-228) */

/* SolverOptions (solver.hpp:33-42) plus the device knobs. */
typedef struct egs_gpu_opts {
  int32_t n_gpus;          /* SolverOptions::workers: GPUs in this solve (1) */
  int32_t device;          /* CUDA ordinal; -1 = current device */
  int32_t certify;         /* 1: losing-region certificate (exact, default);
                              0: plain value iteration up to credit_cap */
  int32_t cert_interval;   /* round of the first certificate attempt; the
                              interval then doubles (0 = 1) */
  int32_t cert_growth;     /* interval multiplier after each attempt (0 = 8) */
  int32_t sparse_div;      /* next round is sparse iff estimated frontier *
                              sparse_div < n (0 = 8; also the certificate's
                              dense / sparse pass threshold) */
  int32_t grid_ctas;       /* persistent-kernel CTAs; 0 = auto */
  int32_t no_tma;          /* 1: stage no edge spans through TMA (A/B and
                              debugging); the result is identical */
  int32_t mode;            /* EGS_MODE_* */
  int32_t debug_checks;    /* SolverOptions::debug_checks (solver_par.cpp:168,179):
                              every commit checks on the device that the value
                              it publishes is above the old one (the
                              reference's check_monotone), and the result is
                              checked to be a fixpoint of the capped lift;
                              either failure returns EGS_ERR_INTERNAL */
  double timeout_seconds;  /* SolverOptions::timeout_seconds; 0 disables */
  uint64_t round_bound;    /* SolverOptions::sweep_bound (solver.hpp:37), used
                              when has_round_bound != 0 -- including 0, which,
                              as in the reference (solver_par.cpp:149-150,
                              184-188), fails after the first round that
                              raises something */
  int32_t has_round_bound; /* 0: default budget |E|*(cap+1)+1
                              (solver_par.cpp:94-98), or round_bound if it is
                              nonzero (callers predating the flag) */
  int32_t reserved_opts;
} egs_gpu_opts;

/* SolveReport counters (solver.hpp:47-59) plus device timings.  The whole
 * solve is ONE persistent kernel (k_solve); its phases are timed on the
 * device with %globaltimer at the grid barriers that separate them. */
typedef struct egs_gpu_stats {
  uint64_t lifts;          /* lift applications that raised a value */
  uint64_t applications;   /* full lift applications (row scans) */
  uint64_t pops;           /* frontier entries of sparse rounds */
  uint64_t rounds;         /* lift rounds */
  uint64_t edges_relaxed;  /* f(t) - w evaluations = sum of outdeg of applications */
  uint64_t witness_checks; /* player-0 lifts skipped by a satisfied witness edge */
  uint64_t dense_rounds;
  uint64_t sparse_rounds;
  uint64_t cert_attempts;  /* losing-region certificate attempts */
  uint64_t cert_passes;    /* pruning passes over all attempts */
  uint64_t certified;      /* vertices proven losing (set to top) */
  uint64_t activations;    /* predecessor slots scanned by the worklist */
  uint64_t visits;         /* vertices examined by lift phases */
  uint64_t cert_rows;      /* rows visited by certificate passes */
  uint64_t cert_edges;     /* edges evaluated by certificate passes */
  double upload_seconds;   /* H2D + device arena construction */
  double solve_seconds;    /* device time from seed to fixpoint (CUDA events) */
  double download_seconds; /* device export + D2H of the measure */
  double wall_seconds;     /* call entry to return (SolveReport::wall_seconds) */
  double seed_seconds;     /* device time per phase kind inside k_solve */
  double lift_seconds;
  double cert_seconds;
  double activate_seconds;
  uint64_t algo_bytes;     /* algorithmic bytes of the whole solve, SURVEY.md
                              §8(d)'s per-unit figures extended to the phases
                              it does not name */
  uint64_t lift_bytes;     /* of which the lift phases, edge records counted
                              at their stored size (4 packed / 8 wide) */
  uint64_t kernel_launches;/* device kernels launched by the solve */
  uint32_t value_bits;     /* 32 or 64: device value width chosen */
  uint32_t grid_ctas;      /* CTAs of the persistent solve kernel */
  double lift_sub_seconds[5]; /* per-CTA mean time in the lift sub-phases:
                                 heavy rows, medium rows, light player-0 rows,
                                 light player-1 rows, sparse light rows */
  double phase_detail_seconds[5]; /* device time of: commit phases, certificate
                                     init, dense passes, sparse passes, apply */
  uint32_t edge_bytes;     /* 4 (packed dst | w << target bits) or 8 ({dst, w}) */
  uint32_t reserved0;
  uint64_t algo_bytes_s8d; /* SURVEY.md §8(d) exactly: edges_relaxed * (8 + s)
                              + applications * (4 + 2 s) + activations * 4,
                              s = value bytes */
  uint64_t h2d_bytes;      /* bytes the arena upload moved host -> device (a
                              partition rank: its own rows only) */
} egs_gpu_stats;

void egs_gpu_opts_default(egs_gpu_opts* opts);

/* One-shot solve: upload, solve, download.  f_out[n] receives the least
 * energy progress measure in the reference's raw encoding (finite credit, or
 * INT64_MAX for top; energy.hpp:16).  Replaces egsolve::solve(...)
 * (solver.hpp:86-87) for the GPU variant. */
int egs_gpu_solve(const egs_arena_view* arena, const egs_gpu_opts* opts,
                  int64_t* f_out, egs_gpu_stats* stats);

/* Device-resident context: the arena is uploaded once (the "cached per-arena"
 * context of SURVEY.md §8b) and solved any number of times. */
typedef struct egs_ctx egs_ctx;
int egs_ctx_create(const egs_arena_view* arena, const egs_gpu_opts* opts,
                   egs_ctx** out, egs_gpu_stats* stats);
int egs_ctx_solve(egs_ctx* ctx, egs_gpu_stats* stats);
int egs_ctx_read_measure(egs_ctx* ctx, int64_t* f_out);
/* Device EPM verifier (measure_ops.cpp:33-41): 1 if f (host, n) is a progress
 * measure of the context's arena, 0 if not, negative on error. */
int egs_ctx_is_progress_measure(egs_ctx* ctx, const int64_t* f);
/* Fixpoint check: 1 if delta(f) == f at every vertex under the lift with the
 * credit cap (measure_ops.hpp:32-52) -- what the least progress measure must
 * satisfy exactly; 0 if not, negative on error.  Size-independent parity
 * check for arenas the CPU reference cannot finish. */
int egs_ctx_is_fixpoint(egs_ctx* ctx, const int64_t* f);
/* write_solution(make_solution(arena, report)) (io.cpp:178-210) of the
 * context's solved measure, computed on the device: first-witness strategy
 * (extract_strategy, measure_ops.cpp:56-80), line lengths, scan, format.
 * Returns the text length (bytes) and copies min(cap, length) bytes into buf
 * when buf != NULL; negative error code otherwise (EGS_ERR_INTERNAL = the
 * reference's NoWitnessError).  Byte-identical to egs_write_solution. */
int64_t egs_ctx_write_solution(egs_ctx* ctx, char* buf, size_t cap);
void egs_ctx_destroy(egs_ctx* ctx);

/* ---------------------------------------------------------------------
 * Multi-GPU partition.  One process (or thread) per GPU;
 * `world` ranks solve one arena together.  The reference has no
 * distributed solver (its workers are threads, solver_par.cpp:231-236).
 *
 * Partition: the relabelled vertex order is rank-major -- rank r owns the
 * contiguous id range [rank_lo[r], rank_lo[r+1]) -- and inside each rank
 * class-sorted (player 0 light / medium / heavy, player 1 light / medium /
 * heavy).  Every (owner, degree) class is split into `world` pieces balanced
 * by out-edges (edge_balanced_bounds, solver_par.cpp:62-80), so every rank
 * gets an equal share of player-0 rows, player-1 rows and hubs.  A rank
 * stores only its own rows' edge records and the predecessor transpose of
 * its own rows (the predecessors it activates); the measure, the changed
 * bitmaps and the certificate's removal bitmaps are replicated.
 *
 * Solve: one persistent kernel per rank (k_solve).  A rank writes every value
 * it raises into its own replica AND into every peer's replica (NVLink peer
 * stores through CUDA IPC mappings, or plain stores when the ranks share a
 * device), sets the changed bits the same way, and at every phase boundary
 * the ranks meet at a device-side barrier (release/acquire flags in peer
 * memory) that also sums the per-rank phase counts, so every rank takes the
 * same schedule decision -- dense / sparse, certificate, termination --
 * without the host.  The result is byte-identical to the single-GPU solve.
 * ------------------------------------------------------------------- */
#define EGS_MAX_RANKS 8
typedef struct egs_part egs_part;

typedef struct egs_part_plan {
  uint32_t world;
  uint32_t num_vertices;
  uint32_t rank_lo[EGS_MAX_RANKS + 1];      /* rank r: relabelled ids [rank_lo[r], rank_lo[r+1]) */
  uint32_t class_lo[EGS_MAX_RANKS][7];      /* rank r, class k: ids [class_lo[r][k], class_lo[r][k+1]) */
  uint32_t piece[6][EGS_MAX_RANKS + 1];     /* class k's rank-r piece: class positions [piece[k][r], piece[k][r+1]) */
  uint64_t edges[EGS_MAX_RANKS];            /* out-edges of rank r's vertices */
} egs_part_plan;

/* The partition of an arena over `world` ranks (host only, deterministic:
 * every rank computes the same plan). */
int egs_part_plan_compute(const egs_arena_view* arena, int32_t world, egs_part_plan* plan);

/* This rank's context: the arena relabelled by the plan, own rows only.
 * opts->n_gpus must equal world; opts->device selects the GPU. */
int egs_part_create(const egs_arena_view* arena, const egs_gpu_opts* opts, int32_t rank,
                    int32_t world, egs_part** out, egs_part_plan* plan, egs_gpu_stats* stats);
/* Export record (128 bytes) of this rank's replicated state, for peers in
 * other processes: its CUDA IPC handle (64 bytes) and its GPU's UUID (16
 * bytes; ranks of different processes on one GPU split its SMs), zero
 * padded. */
#define EGS_IPC_HANDLE_BYTES 128
int egs_part_export(egs_part* part, void* handle);
/* Map every peer's replicated state: handles[r * EGS_IPC_HANDLE_BYTES ...]
 * = rank r's export (this rank's own entry is ignored). */
int egs_part_connect(egs_part* part, const void* handles);
/* Ranks living in ONE process (several GPUs of a process, or several ranks
 * sharing one device for tests): connect them directly.  parts[r] = rank r. */
int egs_part_connect_local(egs_part* const* parts, int32_t world);
/* Solve: every rank must call it concurrently (one host thread or process
 * per rank); blocks until the fixpoint.  Each rank's device-side waits for
 * its peers time out after opts->timeout_seconds (or 60 s) with
 * EGS_ERR_CUDA instead of hanging. */
int egs_part_solve(egs_part* part, egs_gpu_stats* stats);
/* The measure in the reference's raw encoding, original ids (identical on
 * every rank after a solve). */
int egs_part_read_measure(egs_part* part, int64_t* f_out);
/* An order-free 64-bit digest of this rank's replica of the measure
 * (computed on the device): equal on every rank after a solve, so ranks
 * check agreement by exchanging 8 bytes. */
int egs_part_digest(egs_part* part, uint64_t* digest);
void egs_part_destroy(egs_part* part);

/* Output format: write_solution(make_solution(arena, report)) (io.cpp:178-210)
 * with the first-witness strategy of extract_strategy (measure_ops.cpp:56-80).
 * Returns the text length; writes at most cap bytes when buf != NULL;
 * negative error code if some finite player-0 vertex has no witness. */
int64_t egs_write_solution(const egs_arena_view* arena, const int64_t* f,
                           char* buf, size_t cap);

/* Synthetic canonical arenas in host memory,
 * optionally pinned, for the bench and tests.  Owners alternate (even = P0). */
typedef struct egs_host_arena egs_host_arena;
int egs_host_arena_fixed(uint64_t n, uint32_t d, int64_t W, uint64_t seed,
                         int pinned, egs_host_arena** out);
int egs_host_arena_rmat(uint32_t scale, uint32_t edge_factor, int64_t W,
                        uint64_t seed, int pinned, egs_host_arena** out);
void egs_host_arena_view(const egs_host_arena* a, egs_arena_view* view);
void egs_host_arena_free(egs_host_arena* a);

/* ---------------------------------------------------------------------
 * Arena input/output (csrc/egs_arena_io.cpp).  Each
 * returns a host arena whose egs_host_arena_view feeds egs_gpu_solve /
 * egs_ctx_create directly.
 *
 * GameArena::build(n, edges, owners) (arena.hpp:83-84, arena.cpp:17-78):
 * edge i = (src[i], dst[i], weights[i]); rows keep input order. */
int egs_host_arena_build(uint32_t num_vertices, uint64_t num_edges, const uint32_t* src,
                         const uint32_t* dst, const int64_t* weights, const uint8_t* owners,
                         int pinned, egs_host_arena** out);
/* parse_arena(text) (io.hpp:19, io.cpp:87-149) + build, multi-threaded;
 * the reference's records, checks and first error (EGS_ERR_INPUT). */
int egs_arena_parse_text(const char* text, size_t len, int pinned, egs_host_arena** out);
/* write_arena(arena) (io.cpp:151-176): text length; min(cap, length) bytes
 * into buf when buf != NULL. */
int64_t egs_arena_write_text(const egs_arena_view* arena, char* buf, size_t cap);
/* Binary arena file: a 64-byte header (magic "EGSARNA1", version, weight
 * width, n, m, credit_cap, max_abs_weight), then owners u8[n], csr_offsets
 * u64[n+1], csr_targets u32[m], weights narrowed to int8/16/32/64 by max |w|,
 * each span 8-byte aligned.  Loading validates the spans as build does and
 * recomputes compute_stats against the header. */
int egs_arena_save(const egs_arena_view* arena, const char* path);
int egs_arena_load(const char* path, int pinned, egs_host_arena** out);

/* Pinned host buffers for end-to-end timing. */
void* egs_host_alloc_pinned(size_t bytes);
void egs_host_free_pinned(void* p);

const char* egs_last_error(void);
const char* egs_version(void);

#ifdef __cplusplus
}
#endif
#endif /* EGS_GPU_H */
