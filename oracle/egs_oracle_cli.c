#define _POSIX_C_SOURCE 199309L
/*
 * egs_oracle_cli.c — TEST INFRASTRUCTURE ONLY.  Command-line driver for the C
 * restatement: generates a canonical arena, solves it with the restated
 * reference solver and prints FNV-1a hashes of write_arena / write_solution
 * text (the golden-vector format of SURVEY.md Appendix B).
 *
 *   egs_oracle_cli fixed <n> <d> <W> <seed> [seq|sweep|frontier]
 *   egs_oracle_cli rmat  <scale> <ef> <W> <seed> [seq|sweep|frontier]
 */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "egs_oracle.h"

static double now(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + ts.tv_nsec * 1e-9;
}

int main(int argc, char** argv) {
  if (argc < 6) {
    fprintf(stderr, "usage: %s fixed|rmat a b W seed [seq|sweep|frontier]\n",
            argv[0]);
    return 2;
  }
  eo_arena g;
  int rc;
  double t0 = now();
  if (!strcmp(argv[1], "fixed"))
    rc = eo_gen_fixed(strtoull(argv[2], 0, 10), (uint32_t)atoi(argv[3]),
                      atoll(argv[4]), strtoull(argv[5], 0, 10), &g);
  else
    rc = eo_gen_rmat((uint32_t)atoi(argv[2]), (uint32_t)atoi(argv[3]),
                     atoll(argv[4]), strtoull(argv[5], 0, 10), &g);
  if (rc) {
    fprintf(stderr, "generate failed: %d\n", rc);
    return 1;
  }
  double t1 = now();
  int64_t alen = eo_write_arena(&g, NULL, 0);
  char* abuf = (char*)malloc((size_t)alen);
  eo_write_arena(&g, abuf, (size_t)alen);
  printf("arena n=%u m=%llu cap=%lld maxw=%lld maxdeg=%u bytes=%lld hash=%016llx gen=%.2fs\n",
         g.n, (unsigned long long)g.m, (long long)g.credit_cap,
         (long long)g.max_abs_weight, g.max_out_degree, (long long)alen,
         (unsigned long long)eo_fnv1a64(abuf, (size_t)alen), t1 - t0);
  free(abuf);
  const char* mode = argc > 6 ? argv[6] : "seq";
  int64_t* f = (int64_t*)malloc((size_t)g.n * sizeof(int64_t));
  eo_stats st;
  t0 = now();
  if (!strcmp(mode, "sweep")) rc = eo_solve_sweep(&g, 0, f, &st);
  else if (!strcmp(mode, "frontier")) rc = eo_solve_frontier(&g, f, &st);
  else rc = eo_solve_seq(&g, f, &st);
  t1 = now();
  if (rc) {
    fprintf(stderr, "solve failed: %d\n", rc);
    return 1;
  }
  uint64_t tops = 0, maxfin = 0;
  long long sum = 0;
  for (uint32_t v = 0; v < g.n; ++v) {
    if (f[v] == EO_TOP) ++tops;
    else {
      sum += f[v];
      if ((uint64_t)f[v] > maxfin) maxfin = (uint64_t)f[v];
    }
  }
  int64_t slen = eo_write_solution(&g, f, NULL, 0);
  char* sbuf = (char*)malloc((size_t)slen);
  eo_write_solution(&g, f, sbuf, (size_t)slen);
  printf("solve mode=%s time=%.3fs rounds=%llu lifts=%llu apps=%llu edges=%llu "
         "tops=%llu sumfin=%lld maxfin=%llu pm=%d sol_bytes=%lld sol_hash=%016llx\n",
         mode, t1 - t0, (unsigned long long)st.rounds,
         (unsigned long long)st.lifts, (unsigned long long)st.applications,
         (unsigned long long)st.edges_relaxed, (unsigned long long)tops, sum,
         (unsigned long long)maxfin, eo_is_progress_measure(&g, f),
         (long long)slen, (unsigned long long)eo_fnv1a64(sbuf, (size_t)slen));
  free(sbuf);
  free(f);
  eo_arena_free(&g);
  return 0;
}
