/* fnr_oracle.h — TEST INFRASTRUCTURE ONLY (see fnr_oracle.c). */
#ifndef FNR_ORACLE_H_
#define FNR_ORACLE_H_
#include <stdint.h>

typedef struct {            /* sorting.py:19-32 SortCounters */
  uint64_t sorts_performed;
  uint64_t comparisons;
  uint64_t depth_switches;
} oracle_sort_counters;

typedef struct {            /* per-band tuple returned by _filter_rows (filters.py:181) */
  uint64_t minmax_scans;
  uint64_t detected;
  uint64_t replacements;
  oracle_sort_counters sort;
} oracle_pass_counts;

typedef struct {            /* FilterStats (filters.py:33-52) + the sort counters */
  uint64_t minmax_scans;
  uint64_t sorts;
  uint64_t replacements;
  uint64_t detected;
  double elapsed_ms;
  uint64_t passes;
  uint64_t comparisons;
  uint64_t depth_switches;
} oracle_stats;

int oracle_sort_values(int32_t* buf, int n, oracle_sort_counters* counters);
int oracle_median_of(int32_t* buf, int n, oracle_sort_counters* counters, int32_t* out);
int oracle_extract_window(const void* px, int bpp, int64_t w, int64_t h, int64_t x, int64_t y,
                          int k, int32_t* values);
void oracle_filter_rows(const void* px, int bpp, int64_t w, int64_t h, int k, int64_t y0,
                        int64_t y1, void* out, int fnr, oracle_pass_counts* part);
int oracle_run_pass(const void* px, int bpp, int64_t batch, int64_t w, int64_t h, int k, int fnr,
                    int threads, void* out, oracle_stats* stats);
int oracle_run_filter(const void* px, int bpp, int64_t batch, int64_t w, int64_t h, int k,
                      int method, int passes, int threads, void* out, oracle_stats* stats);
/* noise.py:89-106 inject_impulse on n u8 pixels, sequential SplitMix64 (noise.py:17-34);
 * returns the number of corrupted pixels. */
uint64_t oracle_inject_impulse(const uint8_t* in, uint8_t* out, uint8_t* flags, int64_t n,
                               uint64_t seed, double density, double salt_fraction);
/* metrics.py:29-32: exact sum of squared differences (bpp 1 or 2). */
uint64_t oracle_sq_err_sum(const void* a, const void* b, int bpp, int64_t n);
#endif
