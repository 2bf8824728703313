/*
 * datagen.c -- seeded synthetic inputs shared by bench.py and the tests
 * (workload harness, not the projection path).
 *
 * Restates the reference generator documented at
 * proj/include/multiproj/rng.hpp:11-16: SplitMix64 seed expansion into
 * xoshiro256++ (proj/src/rng.cpp:14-39), top-53-bit doubles (:41-43),
 * uniform(lo, hi) = lo + (hi - lo) * u (:45-47), Box-Muller normal with the
 * spare (:49-62).  Laplace(0, b) is new:
 * -b * sgn(u - 1/2) * ln(1 - 2|u - 1/2|).  Values are generated in f64,
 * row-major, and rounded to fp32 (RNE) for the fp32 configs.
 */
#include <math.h>
#include <stdint.h>

typedef struct {
  uint64_t s[4];
  int have_spare;
  double spare;
} mpg_rng;

static uint64_t splitmix(uint64_t* st) {
  uint64_t z = (*st += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

static inline uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

static void rng_seed(mpg_rng* r, uint64_t seed) {
  uint64_t sm = seed;
  for (int i = 0; i < 4; ++i) r->s[i] = splitmix(&sm);
  r->have_spare = 0;
  r->spare = 0.0;
}

static inline uint64_t rng_next(mpg_rng* r) {
  uint64_t* s = r->s;
  const uint64_t out = rotl64(s[0] + s[3], 23) + s[0];
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
  return out;
}

static inline double rng_unit(mpg_rng* r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; }

static double rng_normal(mpg_rng* r) {
  if (r->have_spare) {
    r->have_spare = 0;
    return r->spare;
  }
  double u1 = rng_unit(r);
  double u2 = rng_unit(r);
  while (u1 <= 0.0) u1 = rng_unit(r);
  const double rad = sqrt(-2.0 * log(u1));
  const double ang = 2.0 * 3.14159265358979323846 * u2;
  r->spare = rad * sin(ang);
  r->have_spare = 1;
  return rad * cos(ang);
}

static double rng_laplace(mpg_rng* r, double b) {
  for (;;) {
    const double u = rng_unit(r) - 0.5;
    const double a = 1.0 - 2.0 * fabs(u);
    if (a > 0.0) return -b * (u < 0.0 ? -1.0 : (u > 0.0 ? 1.0 : 0.0)) * log(a);
  }
}

/* kind: 0 uniform(lo, hi), 1 normal(0, 1), 2 laplace(0, b = lo).  out_f32
 * and/or out_f64 receive the same values (either may be NULL). */
void mpg_generate(uint64_t seed, int kind, double lo, double hi, int64_t count, float* out_f32, double* out_f64) {
  mpg_rng r;
  rng_seed(&r, seed);
  for (int64_t i = 0; i < count; ++i) {
    double v;
    if (kind == 0) v = lo + (hi - lo) * rng_unit(&r);
    else if (kind == 1) v = rng_normal(&r);
    else v = rng_laplace(&r, lo);
    if (out_f32) out_f32[i] = (float)v;
    if (out_f64) out_f64[i] = v;
  }
}

void mpg_raw(uint64_t seed, uint64_t* out, int64_t count) {
  mpg_rng r;
  rng_seed(&r, seed);
  for (int64_t i = 0; i < count; ++i) out[i] = rng_next(&r);
}
