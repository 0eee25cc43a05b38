// egs_types.cuh — types shared by the host driver (egs_solver.cu), the
// arena build kernels (egs_build.cuh) and the solve kernels (egs_solve.cuh,
// compiled once per edge-record format).
#pragma once

#include <cstdint>

#include "egs_device.cuh"

namespace egs {


constexpr int kBlock = 256;
constexpr int kWarps = kBlock / 32;
constexpr uint32_t kLightMax = 32;    // rows with <= 32 edges: one thread
constexpr uint32_t kMediumMax = 4096; // <= 4096: one warp; longer: one CTA

// Class ranges of the relabelled ids.
enum : int { kP0L = 0, kP0M, kP0H, kP1L, kP1M, kP1H, kNumClasses };
constexpr int kMaxRanks = 8;  // EGS_MAX_RANKS

enum Counter : int {
  kLifts = 0,      // lifts that raised a value (SolveReport::lifts)
  kApps,           // full lift applications (row scans)
  kEdges,          // edges relaxed = sum of out-degrees of applications
  kWitness,        // player-0 lifts skipped by a satisfied witness edge
  kActScanned,     // predecessor slots scanned by activation
  kCertified,      // vertices proven losing by the certificate
  kPops,           // sparse-round frontier entries
  kCertScanned,    // rows visited by certificate passes
  kCertEdges,      // edges evaluated by certificate passes
  kVisits,         // vertices examined by lift phases (incl. top skips)
  kRounds,
  kDenseRounds,
  kSparseRounds,
  kCertAttempts,
  kCertPasses,
  kStatus,         // 0 fixpoint, 2 timeout, 5 round budget, 7 a peer rank missing
  kTimeSeed,       // ns of device time per phase kind (%globaltimer)
  kTimeLift,
  kTimeCert,
  kTimeAct,
  kSubHeavy,       // ns summed over CTAs inside each lift sub-phase
  kSubMedium,
  kSubLightP0,
  kSubLightP1,
  kSubSparseLight,
  kFineCommit,     // ns of device time: commit, certificate init / dense pass /
  kFineCertInit,   // sparse pass (mark + check) / apply
  kFineCertDense,
  kFineCertSparse,
  kFineCertApply,
  kEpoch,          // multi-GPU: cross-rank barriers passed so far
  kNumCounters
};

enum Mode : int { kModeAuto = 0, kModeDense = 1, kModeSparse = 2, kModeSweep = 3 };
// SolveParams::use_tma bits: which light-row phases stage edge tiles by TMA
// (the others read rows with plain loads through the same claim loop)
enum TmaPhase : int { kTmaRound1 = 1, kTmaLift = 2, kTmaCert = 4, kTmaAll = 7 };
constexpr unsigned kTraceCap = 512;

struct Graph {
  uint32_t n;
  uint32_t rb[kNumClasses + 1];  // class k = [rb[k], rb[k+1])
  const uint32_t* off;           // n+1 CSR row offsets (relabelled rows)
  const void* edge;              // m edge records (format: tbits, below)
  uint32_t tbits;                // 0: int2 {dst, w}; else u32 dst | w << tbits
  const uint32_t* coff;          // n+1 CSC column offsets
  const uint32_t* csrc;          // m   predecessors (relabelled)
  const void* rec0;              // n   a player-1 light row's first record (its
                                 //     least weight: rows sorted at upload)
  int64_t cap;                   // credit_cap (M_G)
};

constexpr int kTileCursor = 7;  // Scratch::dyn slot of the TMA tile claims
constexpr uint32_t kRingEmpty = 0xFFFFFFFFu;
constexpr uint32_t kRingSlack = 1u << 18;  // > (max warps of a grid) * 32 positions claimed ahead

// Grid-shared scratch; the host zeroes it before each launch.
struct Scratch {
  unsigned int sum[4][4];    // per-phase-slot sums: 0 changed, 1 removed, 2 seeds
  unsigned int dyn[4][8];    // per-phase-slot work cursors: 0 medium, 1 heavy,
                             // 2.. activation / certificate queues, 7 TMA tiles
  unsigned int fr_cnt[3][3]; // frontier sublist sizes [token % 3][L, M, H]
  unsigned int stop;         // timeout flag
  unsigned int bad;          // debug_checks: a commit that did not raise its vertex
  unsigned int xerr;         // multi-GPU: a peer did not reach a barrier in time
  // the certificate cascade's work queue (egs_solve.cuh phase_cert_cascade):
  // ring positions claimed / reserved, and items reserved but not finished
  unsigned int qhead, qtail, qpend;
  // the player-1 light vertices still below top after a certificate apply,
  // listed (in SolveParams::fr[0]) for the dense round that follows
  unsigned int p1live;
};

// Cross-rank sync block (multi-GPU, egs_part_solve), inside every rank's
// replicated allocation: peers write their barrier epoch and their phase
// sums here (double-buffered by epoch parity).
struct XSync {
  unsigned int arrive[kMaxRanks];
  unsigned int sums[2][kMaxRanks][4];
};

template <class V>
struct SolveParams {
  Graph g;
  V* f;                 // measure, relabelled ids (read-only inside a lift round)
  V* stage;             // lift rounds: raised values, committed after the round
  void* wit;            // player-0 witness edge record (ids < rb[3]), edge format
  uint32_t* chg[2];     // changed-vertex bitmaps, by round parity
  uint32_t* frb[2];     // frontier membership bitmaps [token & 1]
  uint32_t* rbm[2];     // certificate: removed-in-pass bitmaps
  uint32_t* cbm[2];     // certificate: re-check queue dedup bitmaps [queue & 1]
  uint32_t* cand;       // certificate: candidate bitmap
  uint32_t* longcol;    // activation: queued long CSC columns {vertex, chunk cursor}
  uint32_t* fr[2];      // frontier lists; sublist c starts at cbase[c]
  uint32_t* ring;       // certificate cascade queue: ring_cap slots, kRingEmpty when free
  uint32_t ring_cap;    // n + kRingSlack (claims may run ahead of the reserved slots)
  uint32_t cbase[3];
  Scratch* sh;
  unsigned long long* ctr;  // kNumCounters
  uint32_t own_lo, own_hi;  // vertex range this GPU lifts (multi-GPU); [0, n) alone
  int mode;
  int use_tma;
  int certify;
  int cert_interval;
  int cert_growth;          // interval multiplier after each attempt (8)
  uint32_t sparse_div;      // next round sparse iff est. frontier * div < n
  float cert_sparse_div;    // certificate pass sparse iff removed * deg * div < n
  float avg_in_deg;
  unsigned long long* trace;   // optional: per-phase (kind << 56 | ns) log, kTraceCap entries
  unsigned long long round_budget;
  unsigned long long timeout_ns;   // 0 = none; measured from kernel start
  int debug;                // SolverOptions::debug_checks: commits check monotonicity
  int no_fuse;              // EGS_NO_FUSE=1: commit and activation in separate phases (tracing)
  int cascade;              // certificate cascade in one queue phase (EGS_CERT_CASCADE=0: passes)
  int r1_direct;            // round 1 writes f itself (one rank: nothing reads f during round 1)
  int r1_cand;              // ... and marks the first certificate attempt's candidates
  // multi-GPU (egs_part_solve; world == 1 otherwise): the measure and the
  // changed / removal bitmaps are replicated in one allocation per rank with
  // the same layout everywhere; a rank writes what it raises into every
  // replica (xpeer[q] = rank q's allocation as mapped here).
  int world, rank;
  char* xbase;                  // this rank's replicated allocation
  char* xpeer[kMaxRanks];
  XSync* xsync;                 // this rank's sync block (in xbase)
  unsigned int epoch0;          // cross-rank barriers before this solve
  unsigned long long xwait_ns;  // a peer not arriving within this fails the solve
};


// Edge records.  Two formats, picked per arena at upload (egs_solver.cu):
//   packed (tbits > 0): one u32 = dst | w << tbits, tbits = bits of n-1,
//     when every weight fits the 32-tbits high bits as a signed value (C2-C4:
//     4 bytes per edge instead of 8, half the edge stream);
//   wide (tbits = 0): int2 {dst, w}.
// The solve kernels are compiled once per format (egs_kern.cu); the one-shot
// build and verification kernels decode at run time with edge_at.
constexpr uint32_t kStageBytes = 4096;  // per warp TMA stage
#ifndef EGS_TMA_STAGES
#define EGS_TMA_STAGES 2
#endif
constexpr uint32_t kStages = EGS_TMA_STAGES;  // per warp: kStages - 1 copies ahead
constexpr size_t kLiftSmemBytes = (size_t)kWarps * kStages * kStageBytes;

// Activation: CSC columns longer than kLongCol are chunked over the grid.
constexpr uint32_t kLongCol = 4096;
constexpr uint32_t kColChunk = 1024;

__device__ __forceinline__ int2 edge_dec(uint32_t r, uint32_t tbits) {
  return make_int2((int)(r & ((1u << tbits) - 1u)), (int)r >> tbits);
}
__device__ __forceinline__ int2 edge_at(const Graph& g, uint64_t i) {
  if (g.tbits) return edge_dec(static_cast<const uint32_t*>(g.edge)[i], g.tbits);
  return static_cast<const int2*>(g.edge)[i];
}

}  // namespace egs
