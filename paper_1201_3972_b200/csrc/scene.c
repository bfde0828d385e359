/*
 * scene.c — seeded synthetic IR-like scenes for the five BASELINE.json configs.
 *
 * Bench / test input generation only (not the filter). The paper's 364x244
 * IR photograph is not available (reference SPEC.md:309), so these seeded
 * scenes stand in for it with the shapes, sizes and value distributions
 * BASELINE.json names (see DESIGN.md §5 for the exact recipe):
 *
 *   field(x,y) = 60 + sum_j A_j exp(-((x-cx_j)^2 + (y-cy_j)^2) / (2 s_j^2))    (u8 scale)
 *              + sensor noise N(0, 2^2) (Irwin-Hall(4) approximation)
 *   value      = clip(rint(field * maxval/255 + structures), 0, maxval)
 *   impulses   = per-pixel Bernoulli(density); salt-and-pepper (0 / maxval,
 *                p = 0.5 each) or uniform random in [0, maxval].
 *
 * Randomness is a counter-based SplitMix64 hash of (seed, config, frame,
 * stream, index), so any frame/row range is generated independently and in
 * parallel, and the bytes do not depend on the thread count.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define SCENE_EXPORT __attribute__((visibility("default")))

typedef struct scene_params {
  int32_t width, height, bpp;   /* bpp: 1 (u8) or 2 (u16) */
  int32_t maxval;               /* 255 or 16383 */
  int32_t nblobs;
  double sigma_scale;           /* blob sigma = U(10,60) * sigma_scale */
  double amp_scale;             /* blob amplitude = U(40,150) * amp_scale */
  int32_t drift;                /* 1: blobs drift 1 px/frame along a fixed direction */
  int32_t nlines;               /* thin hot lines, 1-3 px wide, random angle */
  double line_amp;
  int32_t nrects;               /* text-like rectangles 6-12 px per side */
  double rect_amp;
  double sensor_sigma;          /* on the u8 scale */
  int32_t impulse_kind;         /* 0 none, 1 salt & pepper, 2 uniform random */
  double density;
  uint64_t seed;
  int32_t config_id;
} scene_params;

static inline uint64_t sm64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

static inline uint64_t key(const scene_params* p, uint64_t frame, uint64_t stream, uint64_t idx) {
  uint64_t h = sm64(p->seed ^ ((uint64_t)p->config_id << 56));
  h = sm64(h ^ (frame * 0xD1B54A32D192ED03ull));
  h = sm64(h ^ (stream * 0xABC98388FB8FAC03ull));
  return sm64(h ^ idx);
}

static inline double u01(uint64_t h) { return (double)(h >> 11) * (1.0 / 9007199254740992.0); }

enum { ST_BLOB = 1, ST_LINE = 2, ST_RECT = 3, ST_SENSOR = 4, ST_IMP = 5, ST_IMPV = 6 };

typedef struct {
  const scene_params* p;
  int64_t frame0, nframes;
  void* out;
  int64_t unit0, unit1; /* work units: (frame, row band) pairs */
  int32_t band_rows;
} job_t;

/* Blob parameters of frame f and the horizontal Gaussian factors gx[j * W + x]. */
static void frame_blobs(const scene_params* p, int64_t f, double* gx, double* amp, double* cyv, double* sgv) {
  const int32_t W = p->width, H = p->height, nb = p->nblobs;
  for (int j = 0; j < nb; ++j) {
    /* drifting blobs keep one parameter set for the whole sequence (frame key 0) */
    const uint64_t fk = p->drift ? 0 : (uint64_t)f;
    double cx = u01(key(p, fk, ST_BLOB, (uint64_t)j * 8 + 0)) * W;
    double cy = u01(key(p, fk, ST_BLOB, (uint64_t)j * 8 + 1)) * H;
    double a = (40.0 + 110.0 * u01(key(p, fk, ST_BLOB, (uint64_t)j * 8 + 2))) * p->amp_scale;
    double s = (10.0 + 50.0 * u01(key(p, fk, ST_BLOB, (uint64_t)j * 8 + 3))) * p->sigma_scale;
    if (p->drift) {
      double th = 6.283185307179586 * u01(key(p, 0, ST_BLOB, (uint64_t)j * 8 + 4));
      cx += (double)f * cos(th);
      cy += (double)f * sin(th);
    }
    amp[j] = a;
    cyv[j] = cy;
    sgv[j] = s;
    const double inv = 1.0 / (2.0 * s * s);
    for (int32_t x = 0; x < W; ++x) gx[(size_t)j * W + x] = exp(-(x - cx) * (x - cx) * inv);
  }
}

/* Vertical factor of blob (amp, cy, s) at row y (the blob's weight on that row). */
static inline double blob_gy(double amp, double cy, double s, int32_t y) {
  const double dy = y - cy;
  return amp * exp(-dy * dy / (2.0 * s * s));
}

/* Hot lines of frame f: sin, cos, anchor x, anchor y, half width (n <= 64). */
static int32_t frame_lines(const scene_params* p, int64_t f, double* lsin, double* lcos, double* lpx, double* lpy,
                           double* lhw) {
  const int32_t W = p->width, H = p->height;
  const int32_t nl = p->nlines > 64 ? 64 : p->nlines;
  for (int i = 0; i < nl; ++i) {
    double th = 3.141592653589793 * u01(key(p, (uint64_t)f, ST_LINE, (uint64_t)i * 8 + 0));
    lsin[i] = sin(th);
    lcos[i] = cos(th);
    lpx[i] = u01(key(p, (uint64_t)f, ST_LINE, (uint64_t)i * 8 + 1)) * W;
    lpy[i] = u01(key(p, (uint64_t)f, ST_LINE, (uint64_t)i * 8 + 2)) * H;
    lhw[i] = 0.5 * (double)(1 + (int)(3.0 * u01(key(p, (uint64_t)f, ST_LINE, (uint64_t)i * 8 + 3))));
  }
  return nl;
}

/* Text-like rectangles of frame f as half-open [x0, x1) x [y0, y1) (n <= 256). */
static int32_t frame_rects(const scene_params* p, int64_t f, int32_t* rx0, int32_t* ry0, int32_t* rx1, int32_t* ry1) {
  const int32_t W = p->width, H = p->height;
  const int32_t nr = p->nrects > 256 ? 256 : p->nrects;
  for (int i = 0; i < nr; ++i) {
    int32_t rw = 6 + (int32_t)(7.0 * u01(key(p, (uint64_t)f, ST_RECT, (uint64_t)i * 8 + 0)));
    int32_t rh = 6 + (int32_t)(7.0 * u01(key(p, (uint64_t)f, ST_RECT, (uint64_t)i * 8 + 1)));
    int32_t mx = W - rw > 0 ? W - rw : 0, my = H - rh > 0 ? H - rh : 0;
    rx0[i] = (int32_t)(u01(key(p, (uint64_t)f, ST_RECT, (uint64_t)i * 8 + 2)) * (mx + 1));
    ry0[i] = (int32_t)(u01(key(p, (uint64_t)f, ST_RECT, (uint64_t)i * 8 + 3)) * (my + 1));
    rx1[i] = rx0[i] + rw;
    ry1[i] = ry0[i] + rh;
  }
  return nr;
}

static void gen_band(const scene_params* p, int64_t f, int32_t y0, int32_t y1, void* frame_out) {
  const int32_t W = p->width, nb = p->nblobs;
  const double scale = (double)p->maxval / 255.0;
  double* gx = (double*)malloc(sizeof(double) * (size_t)nb * W);
  double* amp = (double*)malloc(sizeof(double) * (size_t)nb);
  double* cyv = (double*)malloc(sizeof(double) * (size_t)nb);
  double* sgv = (double*)malloc(sizeof(double) * (size_t)nb);
  double* rowv = (double*)malloc(sizeof(double) * (size_t)W);
  frame_blobs(p, f, gx, amp, cyv, sgv);
  /* line and rectangle parameters for this frame */
  double lsin[64], lcos[64], lpx[64], lpy[64], lhw[64];
  const int32_t nl = frame_lines(p, f, lsin, lcos, lpx, lpy, lhw);
  int32_t rx0[256], ry0[256], rx1[256], ry1[256];
  const int32_t nr = frame_rects(p, f, rx0, ry0, rx1, ry1);
  const double sens = p->sensor_sigma * 1.7320508075688772; /* sqrt(12/4) */
  for (int32_t y = y0; y < y1; ++y) {
    for (int32_t x = 0; x < W; ++x) rowv[x] = 60.0;
    for (int j = 0; j < nb; ++j) {
      const double gy = blob_gy(amp[j], cyv[j], sgv[j], y);
      if (gy < 1e-6) continue;
      const double* g = gx + (size_t)j * W;
      for (int32_t x = 0; x < W; ++x) rowv[x] += gy * g[x];
    }
    for (int32_t x = 0; x < W; ++x) {
      const uint64_t idx = (uint64_t)y * (uint64_t)W + (uint64_t)x;
      double v = rowv[x];
      if (p->sensor_sigma > 0) {
        uint64_t h = key(p, (uint64_t)f, ST_SENSOR, idx);
        double s4 = (double)(h & 0xFFFF) + (double)((h >> 16) & 0xFFFF) +
                    (double)((h >> 32) & 0xFFFF) + (double)(h >> 48);
        v += (s4 / 65536.0 - 2.0) * sens;
      }
      v *= scale;
      for (int i = 0; i < nl; ++i) {
        double d = (x - lpx[i]) * lsin[i] - (y - lpy[i]) * lcos[i];
        if (fabs(d) < lhw[i]) v += p->line_amp;
      }
      for (int i = 0; i < nr; ++i)
        if (x >= rx0[i] && x < rx1[i] && y >= ry0[i] && y < ry1[i]) v += p->rect_amp;
      double q = rint(v);
      if (q < 0) q = 0;
      if (q > p->maxval) q = p->maxval;
      uint32_t out = (uint32_t)q;
      if (p->impulse_kind && u01(key(p, (uint64_t)f, ST_IMP, idx)) < p->density) {
        uint64_t hv = key(p, (uint64_t)f, ST_IMPV, idx);
        out = p->impulse_kind == 1 ? ((hv >> 63) ? (uint32_t)p->maxval : 0u)
                                   : (uint32_t)(hv % (uint64_t)(p->maxval + 1));
      }
      if (p->bpp == 1) ((uint8_t*)frame_out)[idx] = (uint8_t)out;
      else ((uint16_t*)frame_out)[idx] = (uint16_t)out;
    }
  }
  free(gx); free(amp); free(cyv); free(sgv); free(rowv);
}

static void* job_main(void* arg) {
  job_t* j = (job_t*)arg;
  const scene_params* p = j->p;
  const int64_t bands = (p->height + j->band_rows - 1) / j->band_rows;
  const size_t fbytes = (size_t)p->width * p->height * p->bpp;
  for (int64_t u = j->unit0; u < j->unit1; ++u) {
    const int64_t fi = u / bands, b = u % bands;
    const int32_t y0 = (int32_t)(b * j->band_rows);
    int32_t y1 = y0 + j->band_rows;
    if (y1 > p->height) y1 = p->height;
    gen_band(p, j->frame0 + fi, y0, y1, (char*)j->out + (size_t)fi * fbytes);
  }
  return NULL;
}

/* Generate frames [frame0, frame0+nframes) into out (contiguous frames). */
SCENE_EXPORT int scene_generate(const scene_params* p, int64_t frame0, int64_t nframes, void* out,
                                int32_t nthreads) {
  if (!p || !out || p->width < 1 || p->height < 1 || (p->bpp != 1 && p->bpp != 2) || nframes < 0)
    return 1;
  if (nthreads < 1) nthreads = 1;
  const int32_t band_rows = 64;
  const int64_t bands = (p->height + band_rows - 1) / band_rows;
  const int64_t units = bands * nframes;
  if ((int64_t)nthreads > units) nthreads = (int32_t)(units > 0 ? units : 1);
  job_t* jobs = (job_t*)calloc((size_t)nthreads, sizeof(job_t));
  pthread_t* tids = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
  for (int i = 0; i < nthreads; ++i) {
    jobs[i].p = p;
    jobs[i].frame0 = frame0;
    jobs[i].nframes = nframes;
    jobs[i].out = out;
    jobs[i].unit0 = units * i / nthreads;
    jobs[i].unit1 = units * (i + 1) / nthreads;
    jobs[i].band_rows = band_rows;
  }
  if (nthreads == 1) job_main(&jobs[0]);
  else {
    for (int i = 0; i < nthreads; ++i) pthread_create(&tids[i], NULL, job_main, &jobs[i]);
    for (int i = 0; i < nthreads; ++i) pthread_join(tids[i], NULL);
  }
  free(jobs);
  free(tids);
  return 0;
}

/*
 * The per-frame parameter tables of frames [frame0, frame0 + nframes) for the device
 * generator (csrc/scene.cuh): everything above that needs exp / sin / cos, computed by the
 * same code gen_band runs, so the device (IEEE +, *, rint in gen_band's order) writes the
 * same bytes as scene_generate. Layout per frame i:
 *   gx    [i][nblobs][width]   horizontal Gaussian factor of blob j at column x
 *   gy    [i][nblobs][height]  amplitude x vertical factor of blob j at row y
 *   lines [i][nl][5]           sin, cos, anchor x, anchor y, half width (nl = min(nlines, 64))
 *   rects [i][nr][4]           x0, y0, x1, y1 (half-open; nr = min(nrects, 256))
 * lines / rects may be NULL when nlines / nrects is 0.
 */
typedef struct {
  const scene_params* p;
  int64_t frame0, i0, i1;
  double *gx, *gy, *lines;
  int32_t* rects;
} tab_job_t;

static void* tab_main(void* arg) {
  const tab_job_t* t = (const tab_job_t*)arg;
  const scene_params* p = t->p;
  const int32_t W = p->width, H = p->height, nb = p->nblobs;
  const int32_t nl = p->nlines > 64 ? 64 : p->nlines, nr = p->nrects > 256 ? 256 : p->nrects;
  double* amp = (double*)malloc(sizeof(double) * (size_t)(nb > 0 ? nb : 1));
  double* cyv = (double*)malloc(sizeof(double) * (size_t)(nb > 0 ? nb : 1));
  double* sgv = (double*)malloc(sizeof(double) * (size_t)(nb > 0 ? nb : 1));
  for (int64_t i = t->i0; i < t->i1; ++i) {
    const int64_t f = t->frame0 + i;
    frame_blobs(p, f, t->gx + (size_t)i * nb * W, amp, cyv, sgv);
    double* gy = t->gy + (size_t)i * nb * H;
    for (int j = 0; j < nb; ++j)
      for (int32_t y = 0; y < H; ++y) gy[(size_t)j * H + y] = blob_gy(amp[j], cyv[j], sgv[j], y);
    if (nl > 0 && t->lines) {
      double lsin[64], lcos[64], lpx[64], lpy[64], lhw[64];
      frame_lines(p, f, lsin, lcos, lpx, lpy, lhw);
      double* L = t->lines + (size_t)i * nl * 5;
      for (int k = 0; k < nl; ++k) {
        L[5 * k + 0] = lsin[k];
        L[5 * k + 1] = lcos[k];
        L[5 * k + 2] = lpx[k];
        L[5 * k + 3] = lpy[k];
        L[5 * k + 4] = lhw[k];
      }
    }
    if (nr > 0 && t->rects) {
      int32_t rx0[256], ry0[256], rx1[256], ry1[256];
      frame_rects(p, f, rx0, ry0, rx1, ry1);
      int32_t* R = t->rects + (size_t)i * nr * 4;
      for (int k = 0; k < nr; ++k) {
        R[4 * k + 0] = rx0[k];
        R[4 * k + 1] = ry0[k];
        R[4 * k + 2] = rx1[k];
        R[4 * k + 3] = ry1[k];
      }
    }
  }
  free(amp); free(cyv); free(sgv);
  return NULL;
}

SCENE_EXPORT int scene_tables(const scene_params* p, int64_t frame0, int64_t nframes, double* gx, double* gy,
                              double* lines, int32_t* rects, int32_t nthreads) {
  if (!p || p->width < 1 || p->height < 1 || nframes < 0 || p->nblobs < 0 || (p->nblobs > 0 && (!gx || !gy)))
    return 1;
  if (nthreads < 1) nthreads = 1;
  if ((int64_t)nthreads > nframes) nthreads = (int32_t)(nframes > 0 ? nframes : 1);
  tab_job_t* jobs = (tab_job_t*)calloc((size_t)nthreads, sizeof(tab_job_t));
  pthread_t* tids = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
  for (int i = 0; i < nthreads; ++i) {
    jobs[i] = (tab_job_t){p, frame0, nframes * i / nthreads, nframes * (i + 1) / nthreads, gx, gy, lines, rects};
  }
  if (nthreads == 1) tab_main(&jobs[0]);
  else {
    for (int i = 0; i < nthreads; ++i) pthread_create(&tids[i], NULL, tab_main, &jobs[i]);
    for (int i = 0; i < nthreads; ++i) pthread_join(tids[i], NULL);
  }
  free(jobs);
  free(tids);
  return 0;
}
