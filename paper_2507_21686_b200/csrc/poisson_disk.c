/* poisson_disk.c -- scene generation helper (not on the evaluation path):
 * Bridson's Poisson-disk sampling ("Fast Poisson disk sampling in arbitrary
 * dimensions", SIGGRAPH 2007 sketch) restricted to a disc, for the cfg5
 * obstacle meshes of BASELINE.json configs[4] ("Delaunay triangulation of
 * Poisson-disk points (min spacing 0.05) inside 500 random obstacle discs").
 *
 * Algorithm: background grid of cell r / sqrt(2) (at most one sample per
 * cell); an active list seeded with one uniform point of the disc; repeatedly
 * pick a random active sample, try k candidates uniform in the annulus
 * [r, 2r) around it, accept the first candidate inside the disc whose 5x5
 * grid neighbourhood holds no sample closer than r, and retire the active
 * sample when all k fail. Deterministic for a given seed (splitmix64 /
 * xoshiro256** stream, independent of libc).
 *
 * Built by paper_2507_21686_b200/build.py into _lib/libsphbi_scenes.so.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  uint64_t s[4];
} rng_t;

static uint64_t splitmix64(uint64_t* x) {
  uint64_t z = (*x += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
static void rng_seed(rng_t* r, uint64_t seed) {
  for (int i = 0; i < 4; ++i) r->s[i] = splitmix64(&seed);
}
static inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
static uint64_t rng_next(rng_t* r) {
  uint64_t* s = r->s;
  const uint64_t out = rotl(s[1] * 5, 7) * 9;
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl(s[3], 45);
  return out;
}
/* uniform in [0, 1) with 53 random bits */
static double rng_unif(rng_t* r) { return (double)(rng_next(r) >> 11) * (1.0 / 9007199254740992.0); }

/* Samples of min spacing r_min inside the closed disc of radius R about the
 * origin. Writes at most cap points (x, y interleaved) to out_xy; returns the
 * number of samples (which may exceed cap: call again with a larger buffer),
 * or -1 on bad arguments / allocation failure. */
int64_t sphbi_poisson_disk(uint64_t seed, double R, double r_min, int k, double* out_xy, int64_t cap) {
  if (!(R > 0.0) || !(r_min > 0.0) || k < 1) return -1;
  const double cell = r_min / sqrt(2.0);
  const int64_t g = (int64_t)ceil(2.0 * R / cell) + 1;
  if (g > 200000) return -1;
  int64_t* grid = (int64_t*)malloc((size_t)(g * g) * sizeof(int64_t));
  const int64_t max_pts = g * g;
  double* px = (double*)malloc((size_t)max_pts * 2 * sizeof(double));
  int64_t* active = (int64_t*)malloc((size_t)max_pts * sizeof(int64_t));
  if (!grid || !px || !active) {
    free(grid); free(px); free(active);
    return -1;
  }
  for (int64_t i = 0; i < g * g; ++i) grid[i] = -1;
  rng_t rng;
  rng_seed(&rng, seed);
  const double r2 = r_min * r_min, R2 = R * R;
  int64_t n = 0, na = 0;
  /* first sample: uniform in the disc (rejection from the square) */
  for (;;) {
    const double x = (2.0 * rng_unif(&rng) - 1.0) * R, y = (2.0 * rng_unif(&rng) - 1.0) * R;
    if (x * x + y * y <= R2) {
      px[0] = x;
      px[1] = y;
      break;
    }
  }
#define GX(v) ((int64_t)floor(((v) + R) / cell))
  grid[GX(px[1]) * g + GX(px[0])] = 0;
  active[na++] = 0;
  n = 1;
  while (na > 0) {
    const int64_t ai = (int64_t)(rng_unif(&rng) * (double)na);
    const int64_t a = active[ai];
    const double ax = px[2 * a], ay = px[2 * a + 1];
    int placed = 0;
    for (int t = 0; t < k && !placed; ++t) {
      /* uniform by area in the annulus [r, 2r) */
      const double u = rng_unif(&rng), th = 2.0 * M_PI * rng_unif(&rng);
      const double rr = r_min * sqrt(1.0 + 3.0 * u);
      const double x = ax + rr * cos(th), y = ay + rr * sin(th);
      if (x * x + y * y > R2) continue;
      const int64_t cx = GX(x), cy = GX(y);
      if (cx < 0 || cy < 0 || cx >= g || cy >= g) continue;
      int ok = 1;
      for (int64_t jy = cy - 2; jy <= cy + 2 && ok; ++jy) {
        if (jy < 0 || jy >= g) continue;
        for (int64_t jx = cx - 2; jx <= cx + 2; ++jx) {
          if (jx < 0 || jx >= g) continue;
          const int64_t o = grid[jy * g + jx];
          if (o < 0) continue;
          const double dx = px[2 * o] - x, dy = px[2 * o + 1] - y;
          if (dx * dx + dy * dy < r2) {
            ok = 0;
            break;
          }
        }
      }
      if (!ok) continue;
      px[2 * n] = x;
      px[2 * n + 1] = y;
      grid[cy * g + cx] = n;
      active[na++] = n;
      ++n;
      placed = 1;
    }
    if (!placed) active[ai] = active[--na];
  }
#undef GX
  const int64_t m = n < cap ? n : cap;
  if (out_xy && m > 0) memcpy(out_xy, px, (size_t)m * 2 * sizeof(double));
  free(grid);
  free(px);
  free(active);
  return n;
}
