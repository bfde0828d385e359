/*
 * The drop-in boundary from plain C: run_filter (filters.py:79-102) on host buffers through
 * include/irdn.h, as a C / C++ (or cgo / JNI) caller of the reference would bind it.
 *
 *   gcc -O2 -I include examples/c_api_demo.c -L paper_1201_3972_b200 -lirdn \
 *       -Wl,-rpath,$PWD/paper_1201_3972_b200 -o c_api_demo
 *   ./c_api_demo [frames height width k passes]      (default: 4 512 640 5 1, u16 FNR)
 *
 * Prints the FilterStats counters (filters.py:44-52 key order) and an FNV-1a hash of the
 * output bytes; exit code 0 on success, 1 on an irdn error (message on stderr).
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "irdn.h"

static uint64_t next(uint64_t* s) { /* SplitMix64 */
  uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

int main(int argc, char** argv) {
  const int64_t frames = argc > 1 ? atoll(argv[1]) : 4, height = argc > 2 ? atoll(argv[2]) : 512,
                width = argc > 3 ? atoll(argv[3]) : 640;
  const int32_t k = argc > 4 ? atoi(argv[4]) : 5, passes = argc > 5 ? atoi(argv[5]) : 1;
  const int64_t n = frames * height * width;
  uint16_t* in = malloc((size_t)n * sizeof(uint16_t));
  uint16_t* out = malloc((size_t)n * sizeof(uint16_t));
  if (!in || !out) return 1;
  /* a smooth 14-bit ramp with 30 % uniform impulses (seed 42) */
  uint64_t s = 42;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t x = i % width, y = (i / width) % height;
    uint16_t v = (uint16_t)((x * 7 + y * 5) % 16384);
    if ((next(&s) >> 11) * (1.0 / 9007199254740992.0) < 0.3) v = (uint16_t)(next(&s) % 16384);
    in[i] = v;
  }
  printf("%s, %d sm_100 device(s)\n", irdn_version(), irdn_device_count());
  irdn_stats st;
  int rc = irdn_run_filter_u16(in, out, frames, height, width, k, IRDN_METHOD_FNR, passes, 0, &st);
  if (rc != IRDN_OK) {
    fprintf(stderr, "irdn error %d: %s\n", rc, irdn_last_error());
    return 1;
  }
  uint64_t h2d = 0, d2h = 0;
  irdn_last_transfer(&h2d, &d2h);
  uint64_t hash = 0xcbf29ce484222325ull;
  const uint8_t* b = (const uint8_t*)out;
  for (int64_t i = 0; i < n * 2; ++i) hash = (hash ^ b[i]) * 0x100000001b3ull;
  printf("minmax_scans %llu sorts %llu replacements %llu detected %llu passes %llu\n",
         (unsigned long long)st.minmax_scans, (unsigned long long)st.sorts,
         (unsigned long long)st.replacements, (unsigned long long)st.detected,
         (unsigned long long)st.passes);
  printf("h2d %llu d2h %llu fnv1a %016llx\n", (unsigned long long)h2d, (unsigned long long)d2h,
         (unsigned long long)hash);
  /* an invalid window is a ValueError in the reference (image.py:63-65): IRDN_EINVAL here */
  rc = irdn_run_filter_u16(in, out, frames, height, width, 4, IRDN_METHOD_FNR, 1, 0, &st);
  printf("k=4 -> %d (%s)\n", rc, irdn_last_error());
  free(in);
  free(out);
  return 0;
}
