/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the reference's sketch draw.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this; the product path never does.
 *
 * Restates `gaussian_matrix(rows, cols, seed)`
 * (/root/reference/pkg/src/pbpqlp/linalg.py:83-93), i.e.
 *   numpy.random.Generator(numpy.random.Philox(key=seed)).standard_normal((rows, cols))
 * numpy is the third-party dependency the reference calls (pyproject.toml:11-15
 * pins only numpy>=1.24; this image has numpy 2.3.5).  Algorithms restated:
 *  - Philox4x64-10 (Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as
 *    easy as 1, 2, 3", SC'11): key = (seed mod 2^64, seed >> 64), block c uses
 *    counter (c+1, 0, 0, 0), its four 64-bit words are emitted in order.
 *  - numpy's 256-layer normal ziggurat over that u64 stream, with the layer
 *    tables derived by tools/gen_ziggurat_tables.py.
 * Parity of this restatement against numpy itself: tests/test_oracle.py.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "../paper_2103_07245_b200/csrc/ziggurat_tables.h"

typedef struct {
  uint64_t k0, k1;
  uint64_t block;   /* index of the buffered block */
  uint64_t buf[4];
  int have;         /* buffer valid */
} pbqo_philox;

static void pbqo_mulhilo(uint64_t a, uint64_t b, uint64_t* hi, uint64_t* lo) {
  __uint128_t p = (__uint128_t)a * b;
  *hi = (uint64_t)(p >> 64);
  *lo = (uint64_t)p;
}

static void pbqo_block(uint64_t ctr0, uint64_t k0, uint64_t k1, uint64_t out[4]) {
  uint64_t x0 = ctr0, x1 = 0, x2 = 0, x3 = 0;
  for (int r = 0; r < 10; ++r) {
    uint64_t hi0, lo0, hi1, lo1;
    pbqo_mulhilo(0xD2E7470EE14C6C93ULL, x0, &hi0, &lo0);
    pbqo_mulhilo(0xCA5A826395121157ULL, x2, &hi1, &lo1);
    uint64_t n0 = hi1 ^ x1 ^ k0, n2 = hi0 ^ x3 ^ k1;
    x0 = n0; x1 = lo1; x2 = n2; x3 = lo0;
    k0 += 0x9E3779B97F4A7C15ULL;
    k1 += 0xBB67AE8584CAA73BULL;
  }
  out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
}

static uint64_t pbqo_word(pbqo_philox* g, uint64_t pos) {
  uint64_t b = pos >> 2;
  if (!g->have || g->block != b) {
    pbqo_block(b + 1, g->k0, g->k1, g->buf);
    g->block = b;
    g->have = 1;
  }
  return g->buf[pos & 3];
}

/* Raw u64 words [start, start+n) of the stream (numpy BitGenerator.random_raw). */
void pbqo_philox_raw(uint64_t k0, uint64_t k1, uint64_t start, uint64_t n, uint64_t* out) {
  pbqo_philox g = {k0, k1, 0, {0, 0, 0, 0}, 0};
  for (uint64_t i = 0; i < n; ++i) out[i] = pbqo_word(&g, start + i);
}

static double pbqo_unit(uint64_t v) { return (double)(v >> 11) * (1.0 / 9007199254740992.0); }

/* One standard normal starting at stream position *pos; advances *pos. */
static double pbqo_normal(pbqo_philox* g, uint64_t* pos) {
  for (;;) {
    uint64_t r = pbqo_word(g, (*pos)++);
    int idx = (int)(r & 0xff);
    r >>= 8;
    int sign = (int)(r & 1);
    uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
    double x = (double)rabs * pbq_zig_wi[idx];
    if (sign) x = -x;
    if (rabs < pbq_zig_ki[idx]) return x;
    if (idx == 0) {
      for (;;) {
        double xx = -PBQ_ZIG_INV_R * log1p(-pbqo_unit(pbqo_word(g, (*pos)++)));
        double yy = -log1p(-pbqo_unit(pbqo_word(g, (*pos)++)));
        if (yy + yy > xx * xx)
          return ((rabs >> 8) & 1) ? -(PBQ_ZIG_R + xx) : (PBQ_ZIG_R + xx);
      }
    }
    if ((pbq_zig_fi[idx - 1] - pbq_zig_fi[idx]) * pbqo_unit(pbqo_word(g, (*pos)++)) + pbq_zig_fi[idx] <
        exp(-0.5 * x * x))
      return x;
  }
}

/* n consecutive normals of the stream keyed by (k0, k1), skipping the first
 * `skip` normals; returns the stream position after the last one. */
uint64_t pbqo_normals(uint64_t k0, uint64_t k1, uint64_t skip, uint64_t n, double* out) {
  pbqo_philox g = {k0, k1, 0, {0, 0, 0, 0}, 0};
  uint64_t pos = 0;
  for (uint64_t i = 0; i < skip; ++i) (void)pbqo_normal(&g, &pos);
  for (uint64_t i = 0; i < n; ++i) out[i] = pbqo_normal(&g, &pos);
  return pos;
}

/* ---- log1p pin: the device's glibc_log1p (csrc/sketch.cuh), restated on
 * the host with the same explicit fma() and single-rounded operations
 * (this file is built with -ffp-contract=off), next to the C library's own
 * log1p, which numpy's ziggurat tail calls (npy_log1p).  tests/test_oracle.py
 * checks the two agree bit for bit. */
static inline int32_t pbqo_hi(double x) {
  uint64_t b;
  memcpy(&b, &x, 8);
  return (int32_t)(b >> 32);
}
static inline double pbqo_sethi(double x, int32_t h) {
  uint64_t b;
  memcpy(&b, &x, 8);
  b = (b & 0xffffffffULL) | ((uint64_t)(uint32_t)h << 32);
  memcpy(&x, &b, 8);
  return x;
}

double pbqo_glibc_log1p(double x) {
  const double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10;
  const double Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01, Lp3 = 2.857142874366239149e-01,
               Lp4 = 2.222219843214978396e-01, Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
               Lp7 = 1.479819860511658591e-01;
  const int32_t hx = pbqo_hi(x), ax = hx & 0x7fffffff;
  int32_t k = 1, hu = 0;
  double f = 0.0, c = 0.0;
  if (hx < 0x3FDA827A) {
    if (ax >= 0x3ff00000) return x == -1.0 ? -INFINITY : NAN;
    if (ax < 0x3e200000) return ax < 0x3c900000 ? x : fma(-(x * x), 0.5, x);
    if (hx > 0 || hx <= (int32_t)0xbfd2bec3) {
      k = 0;
      f = x;
      hu = 1;
    }
  }
  if (hx >= 0x7ff00000) return x + x;
  if (k != 0) {
    double u;
    if (hx < 0x43400000) {
      u = 1.0 + x;
      hu = pbqo_hi(u);
      k = (hu >> 20) - 1023;
      c = k > 0 ? 1.0 - (u - x) : x - (u - 1.0);
      c /= u;
    } else {
      u = x;
      hu = pbqo_hi(u);
      k = (hu >> 20) - 1023;
      c = 0.0;
    }
    hu &= 0x000fffff;
    if (hu < 0x6a09e) {
      u = pbqo_sethi(u, hu | 0x3ff00000);
    } else {
      k += 1;
      u = pbqo_sethi(u, hu | 0x3fe00000);
      hu = (0x00100000 - hu) >> 2;
    }
    f = u - 1.0;
  }
  const double dk = (double)k;
  const double hfsq = (0.5 * f) * f;
  if (hu == 0) {
    if (f == 0.0) {
      if (k == 0) return 0.0;
      c = fma(dk, ln2_lo, c);
      return fma(dk, ln2_hi, c);
    }
    const double R = hfsq * fma(-f, 0.66666666666666666, 1.0);
    if (k == 0) return f - R;
    return fma(dk, ln2_hi, -((R - fma(dk, ln2_lo, c)) - f));
  }
  const double s = f / (2.0 + f), z = s * s;
  const double z2 = z * z, z4 = z2 * z2, z6 = z4 * z2;
  const double R2 = fma(z, Lp3, Lp2), R3 = fma(z, Lp5, Lp4), R4 = fma(z, Lp7, Lp6);
  const double R = fma(z6, R4, fma(z4, R3, fma(z, Lp1, z2 * R2)));
  const double shr = s * (hfsq + R);
  if (k == 0) return f - (hfsq - shr);
  return fma(dk, ln2_hi, -((hfsq - (shr + fma(dk, ln2_lo, c))) - f));
}

void pbqo_log1p_pair(const double* x, long n, double* restated, double* libm) {
  for (long i = 0; i < n; ++i) {
    restated[i] = pbqo_glibc_log1p(x[i]);
    libm[i] = log1p(x[i]);
  }
}
