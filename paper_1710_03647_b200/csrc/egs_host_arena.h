// egs_host_arena.h — the host arena behind the opaque egs_host_arena handle
// of include/egs_gpu.h (the flattened GameArena spans, arena.hpp:37-133),
// shared by the generators (egs_host.cpp) and the arena I/O
// (egs_arena_io.cpp).  Internal to libegs_b200.so.
#pragma once

#include <cstdint>

struct egs_host_arena {
  uint32_t n = 0;
  uint64_t m = 0;
  bool pinned = false;
  uint64_t* off = nullptr;
  uint32_t* dst = nullptr;
  int64_t* w = nullptr;
  uint8_t* owner = nullptr;
  int64_t credit_cap = 0;
  int64_t max_abs_weight = 0;
};

// Spans of n vertices and m edges, page-locked when `pinned`; nullptr if an
// allocation fails.
egs_host_arena* egs_internal_arena_alloc(uint32_t n, uint64_t m, bool pinned);
void egs_internal_arena_free(egs_host_arena* a);
// compute_stats (arena.cpp:80-108) and the totality check of build
// (arena.cpp:36-40): fills credit_cap / max_abs_weight or returns an error
// code with egs_last_error set.
int egs_internal_finish_stats(egs_host_arena* a);
