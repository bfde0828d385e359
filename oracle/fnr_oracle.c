/*
 * fnr_oracle.c — CPU restatement of the reference FNR / MF filter.
 *
 * TEST INFRASTRUCTURE ONLY. This file is the parity checker and the CPU
 * baseline ("port") for bench.py; it is never linked into, loaded by or
 * called from the product path (paper_1201_3972_b200/). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs use it.
 *
 * It restates, in plain C, the reference algorithm (irdenoise v0.1.0,
 * pkg/src/irdenoise/...) step by step, including the instrumented introsort
 * used for medians, so its timing is that of the reference ALGORITHM run as
 * compiled code:
 *   filters.py:79-102    run_filter          -> oracle_run_filter
 *   filters.py:105-127   _run_rows_threaded  -> oracle_run_pass (pthreads row bands)
 *   filters.py:130-181   _filter_rows        -> filter_rows
 *   filters.py:55-66     window_extrema / classify_pixel (the detector, inline)
 *   sorting.py:35-48     sort_values         -> sort_values
 *   sorting.py:51-56     median_of           -> median_of
 *   sorting.py:59-74     _introsort_loop     -> introsort_loop
 *   sorting.py:77-114    _partition          -> partition
 *   sorting.py:117-145   _heapsort_range     -> heapsort_range
 *   sorting.py:148-161   _insertion_pass     -> insertion_pass
 *   image.py:101-131     extract_window      -> oracle_extract_window
 *
 * Parity pin: tests/test_oracle_golden.py checks this file against golden
 * vectors produced by running the reference package itself
 * (tests/golden/make_golden.py).
 *
 * Pixels are u8 (the reference's GrayImage) or u16 (the reference's
 * dtype-agnostic per-window API); values are held as int32.
 */
#include "fnr_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define INSERTION_CUTOFF 16 /* sorting.py:16 */

/* sorting.py:148-161 — one insertion-sort pass over a[lo:hi]. */
static uint64_t insertion_pass(int32_t* a, int lo, int hi) {
  uint64_t comps = 0;
  for (int i = lo + 1; i < hi; ++i) {
    int32_t v = a[i];
    int j = i - 1;
    while (j >= lo) {
      comps += 1;
      if (a[j] > v) {
        a[j + 1] = a[j];
        j -= 1;
      } else {
        break;
      }
    }
    a[j + 1] = v;
  }
  return comps;
}

/* sorting.py:117-145 — heapsort of a[lo:hi]. */
static uint64_t sift_down(int32_t* a, int lo, int root, int end) {
  uint64_t c = 0;
  for (;;) {
    int child = 2 * root + 1;
    if (child >= end) return c;
    int right = child + 1;
    if (right < end) {
      c += 1;
      if (a[lo + child] < a[lo + right]) child = right;
    }
    c += 1;
    if (a[lo + root] < a[lo + child]) {
      int32_t t = a[lo + root];
      a[lo + root] = a[lo + child];
      a[lo + child] = t;
      root = child;
    } else {
      return c;
    }
  }
}

static uint64_t heapsort_range(int32_t* a, int lo, int hi) {
  uint64_t comps = 0;
  int n = hi - lo;
  for (int start = n / 2 - 1; start >= 0; --start) comps += sift_down(a, lo, start, n);
  for (int end = n - 1; end > 0; --end) {
    int32_t t = a[lo];
    a[lo] = a[lo + end];
    a[lo + end] = t;
    comps += sift_down(a, lo, 0, end);
  }
  return comps;
}

/* sorting.py:77-114 — median-of-three Hoare partition of [lo, hi). */
static int partition(int32_t* a, int lo, int hi, oracle_sort_counters* counters) {
  uint64_t comps = 0;
  int mid = (lo + hi) / 2;
  int last = hi - 1;
  int32_t t;
  if (a[mid] < a[lo]) { t = a[mid]; a[mid] = a[lo]; a[lo] = t; }
  if (a[last] < a[mid]) {
    t = a[last]; a[last] = a[mid]; a[mid] = t;
    if (a[mid] < a[lo]) { t = a[mid]; a[mid] = a[lo]; a[lo] = t; }
    comps += 3;
  } else {
    comps += 2;
  }
  int32_t pivot = a[mid];
  int i = lo, j = last;
  for (;;) {
    i += 1;
    while (a[i] < pivot) { comps += 1; i += 1; }
    comps += 1;
    j -= 1;
    while (a[j] > pivot) { comps += 1; j -= 1; }
    comps += 1;
    if (i >= j) {
      counters->comparisons += comps;
      return j + 1;
    }
    t = a[i]; a[i] = a[j]; a[j] = t;
  }
}

/* sorting.py:59-74 */
static void introsort_loop(int32_t* a, int lo, int hi, int depth, oracle_sort_counters* counters) {
  while (hi - lo > INSERTION_CUTOFF) {
    if (depth == 0) {
      counters->depth_switches += 1;
      counters->comparisons += heapsort_range(a, lo, hi);
      return;
    }
    depth -= 1;
    int cut = partition(a, lo, hi, counters);
    introsort_loop(a, cut, hi, depth, counters);
    hi = cut;
  }
}

static int bit_length(int n) {
  int b = 0;
  while (n) { ++b; n >>= 1; }
  return b;
}

/* sorting.py:35-48 — sorts buf[0:n] in place (the reference copies first). */
int oracle_sort_values(int32_t* buf, int n, oracle_sort_counters* counters) {
  if (n == 0) return -1; /* ValueError("cannot sort an empty sequence") */
  if (n > INSERTION_CUTOFF) introsort_loop(buf, 0, n, 2 * (bit_length(n) - 1), counters);
  counters->comparisons += insertion_pass(buf, 0, n);
  counters->sorts_performed += 1;
  return 0;
}

/* sorting.py:51-56 — median via one counted sort; buf is clobbered. */
int oracle_median_of(int32_t* buf, int n, oracle_sort_counters* counters, int32_t* out) {
  if (n % 2 == 0) return -1; /* ValueError: median needs an odd-length sequence */
  if (oracle_sort_values(buf, n, counters)) return -1;
  *out = buf[(n - 1) / 2];
  return 0;
}

static inline int64_t clamp64(int64_t v, int64_t lo, int64_t hi) { return v < lo ? lo : (v > hi ? hi : v); }

static inline int32_t load_px(const void* px, int bpp, int64_t i) {
  return bpp == 1 ? (int32_t)((const uint8_t*)px)[i] : (int32_t)((const uint16_t*)px)[i];
}
static inline void store_px(void* px, int bpp, int64_t i, int32_t v) {
  if (bpp == 1) ((uint8_t*)px)[i] = (uint8_t)v;
  else ((uint16_t*)px)[i] = (uint16_t)v;
}

/* image.py:101-131 — window values in raster order with replicate-edge clamping. */
int oracle_extract_window(const void* px, int bpp, int64_t w, int64_t h, int64_t x, int64_t y,
                          int k, int32_t* values) {
  if (!(0 <= x && x < w && 0 <= y && y < h)) return -1; /* IndexError */
  int r = k / 2, n = 0;
  for (int dy = -r; dy <= r; ++dy) {
    int64_t row = clamp64(y + dy, 0, h - 1) * w;
    for (int dx = -r; dx <= r; ++dx) values[n++] = load_px(px, bpp, row + clamp64(x + dx, 0, w - 1));
  }
  return 0;
}

/*
 * filters.py:130-181 — filter rows [y0, y1) of the input snapshot into out.
 * Row offsets are clamped (:156-157); columns use the interior slice path or
 * the clamped edge columns (:149-152, :159-167) — both are the clamp rule.
 */
static void filter_rows(const void* px, int bpp, int64_t w, int64_t h, int k, int64_t y0,
                        int64_t y1, void* out, int fnr, oracle_pass_counts* part) {
  const int r = k / 2, n = k * k;
  int32_t* vals = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  int64_t* row_off = (int64_t*)malloc(sizeof(int64_t) * (size_t)k);
  for (int64_t y = y0; y < y1; ++y) {
    for (int dy = -r; dy <= r; ++dy) row_off[dy + r] = clamp64(y + dy, 0, h - 1) * w;
    const int64_t base = y * w;
    for (int64_t x = 0; x < w; ++x) {
      int m = 0;
      if (r <= x && x < w - r) {
        for (int i = 0; i < k; ++i)
          for (int dx = -r; dx <= r; ++dx) vals[m++] = load_px(px, bpp, row_off[i] + x + dx);
      } else {
        for (int i = 0; i < k; ++i)
          for (int dx = -r; dx <= r; ++dx) vals[m++] = load_px(px, bpp, row_off[i] + clamp64(x + dx, 0, w - 1));
      }
      const int32_t center = load_px(px, bpp, base + x);
      if (fnr) {
        part->minmax_scans += 1;
        int32_t mn = vals[0], mx = vals[0];
        for (int i = 1; i < n; ++i) {
          if (vals[i] < mn) mn = vals[i];
          if (vals[i] > mx) mx = vals[i];
        }
        if (center == mn || center == mx) {
          part->detected += 1;
          int32_t med;
          oracle_median_of(vals, n, &part->sort, &med);
          if (med != center) part->replacements += 1;
          store_px(out, bpp, base + x, med);
        } else {
          store_px(out, bpp, base + x, center);
        }
      } else {
        int32_t med;
        oracle_median_of(vals, n, &part->sort, &med);
        store_px(out, bpp, base + x, med);
      }
    }
  }
  free(vals);
  free(row_off);
}

void oracle_filter_rows(const void* px, int bpp, int64_t w, int64_t h, int k, int64_t y0,
                        int64_t y1, void* out, int fnr, oracle_pass_counts* part) {
  filter_rows(px, bpp, w, h, k, y0, y1, out, fnr, part);
}

typedef struct {
  const void* px; int bpp; int64_t w, h; int k; int64_t y0, y1; void* out; int fnr;
  oracle_pass_counts part;
} band_job;

static void* band_main(void* arg) {
  band_job* j = (band_job*)arg;
  filter_rows(j->px, j->bpp, j->w, j->h, j->k, j->y0, j->y1, j->out, j->fnr, &j->part);
  return NULL;
}

/*
 * filters.py:105-127 — one pass of `batch` frames into a fresh buffer; rows
 * are split into bands height*i//workers (:110-120), counters merged (:121-126).
 * The reference's threads share a GIL; these are real pthreads.
 */
int oracle_run_pass(const void* px, int bpp, int64_t batch, int64_t w, int64_t h, int k, int fnr,
                    int threads, void* out, oracle_stats* stats) {
  const int64_t frame = w * h;
  for (int64_t b = 0; b < batch; ++b) {
    const char* fin = (const char*)px + (size_t)(b * frame * bpp);
    char* fout = (char*)out + (size_t)(b * frame * bpp);
    int workers = threads < 1 ? 1 : threads;
    if (workers > h) workers = (int)h;
    band_job* jobs = (band_job*)calloc((size_t)workers, sizeof(band_job));
    pthread_t* tids = (pthread_t*)calloc((size_t)workers, sizeof(pthread_t));
    for (int i = 0; i < workers; ++i) {
      band_job j = {fin, bpp, w, h, k, h * i / workers, h * (i + 1) / workers, fout, fnr, {0}};
      jobs[i] = j;
    }
    if (workers == 1) {
      band_main(&jobs[0]);
    } else {
      for (int i = 0; i < workers; ++i) pthread_create(&tids[i], NULL, band_main, &jobs[i]);
      for (int i = 0; i < workers; ++i) pthread_join(tids[i], NULL);
    }
    for (int i = 0; i < workers; ++i) {
      stats->minmax_scans += jobs[i].part.minmax_scans;
      stats->detected += jobs[i].part.detected;
      stats->replacements += jobs[i].part.replacements;
      stats->sorts += jobs[i].part.sort.sorts_performed;
      stats->comparisons += jobs[i].part.sort.comparisons;
      stats->depth_switches += jobs[i].part.sort.depth_switches;
    }
    free(jobs);
    free(tids);
  }
  stats->passes += 1;
  return 0;
}

/* filters.py:79-102 — validation, passes (each reads the previous output), stats. */
int oracle_run_filter(const void* px, int bpp, int64_t batch, int64_t w, int64_t h, int k,
                      int method, int passes, int threads, void* out, oracle_stats* stats) {
  if (method != 0 && method != 1) return -1;  /* ValueError: unknown method */
  if (passes < 1) return -2;                  /* ValueError: passes must be >= 1 */
  if (k < 3 || k % 2 == 0) return -3;         /* image.py:63-65 */
  if (w < 1 || h < 1 || batch < 1) return -4; /* image.py:30-31 */
  if (bpp != 1 && bpp != 2) return -5;
  memset(stats, 0, sizeof(*stats));
  struct timespec t0, t1;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  const size_t bytes = (size_t)(batch * w * h * bpp);
  void* tmp = passes > 1 ? malloc(bytes) : NULL;
  const void* cur = px;
  for (int p = 0; p < passes; ++p) {
    void* dst = ((passes - 1 - p) % 2 == 0) ? out : tmp;
    oracle_run_pass(cur, bpp, batch, w, h, k, method == 0, threads, dst, stats);
    cur = dst;
  }
  free(tmp);
  clock_gettime(CLOCK_MONOTONIC, &t1);
  stats->elapsed_ms = (double)(t1.tv_sec - t0.tv_sec) * 1e3 + (double)(t1.tv_nsec - t0.tv_nsec) * 1e-6;
  return 0;
}

/* ---- inject_impulse (noise.py:89-106) ----------------------------------------
 * SplitMix64.next_u64 (noise.py:25-30): state += 0x9E3779B97F4A7C15, then the two
 * xor-shift-multiply rounds and a final xor-shift; next_uniform (noise.py:32-34) is
 * (next_u64 >> 11) / 2^53 as a double. Pixels in row-major order: one uniform draw
 * decides corruption (< density); only a corrupted pixel draws again (< salt_fraction
 * -> 255, else 0). Restated sequentially, exactly as the reference walks it. */
static uint64_t splitmix_next(uint64_t* state) {
  *state += 0x9E3779B97F4A7C15ull;
  uint64_t z = *state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static double splitmix_uniform(uint64_t* state) {
  return (double)(splitmix_next(state) >> 11) / 9007199254740992.0;
}

uint64_t oracle_inject_impulse(const uint8_t* in, uint8_t* out, uint8_t* flags, int64_t n,
                               uint64_t seed, double density, double salt_fraction) {
  uint64_t state = seed, count = 0;
  for (int64_t i = 0; i < n; ++i) {
    uint8_t v = in[i], f = 0;
    if (splitmix_uniform(&state) < density) {
      v = splitmix_uniform(&state) < salt_fraction ? 255 : 0;
      f = 1;
      ++count;
    }
    out[i] = v;
    if (flags) flags[i] = f;
  }
  return count;
}

/* ---- mse numerator (metrics.py:29-32) ---------------------------------------- */
uint64_t oracle_sq_err_sum(const void* a, const void* b, int bpp, int64_t n) {
  uint64_t total = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t pa = bpp == 1 ? ((const uint8_t*)a)[i] : ((const uint16_t*)a)[i];
    const int64_t pb = bpp == 1 ? ((const uint8_t*)b)[i] : ((const uint16_t*)b)[i];
    total += (uint64_t)((pa - pb) * (pa - pb));
  }
  return total;
}
