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
