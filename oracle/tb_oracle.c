/*
 * tb_oracle.c — plain-C restatement of the reference mini-app data path.
 *
 * TEST INFRASTRUCTURE / CPU BASELINE ONLY (see oracle/__init__.py): loaded by
 * tests/ and by bench.py's cpu_baseline leg and --impl reference arm, never by
 * the product package.
 *
 * Restates pkg/src/taskbridge/reference.py:23-50 (== miniapp.py:116-171):
 *   - init   cells[g][i] = (g*1000 + i) / (S*1000 + 512)      miniapp.py:72-77
 *   - ghost  work[:8]  = 0.5*(work[:8]  + right face of g-1)  miniapp.py:125
 *            work[-8:] = 0.5*(work[-8:] + left face of g+1)   miniapp.py:126
 *   - 15 x   work *= C1[k]; work += C2[k]  (two roundings)     miniapp.py:49-51
 *   - min    work.min()                                        miniapp.py:133
 *   - sum    work.sum() in numpy's pairwise order              miniapp.py:133
 *   - piece  math.fsum(sums) in id order (correctly rounded)   miniapp.py:168-169
 *   - checksum += piece; dts.append(min(mins))                 reference.py:48-49
 *
 * Build: oracle/Makefile  (-O2 -ffp-contract=off -fopenmp; no -ffast-math).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define CELLS 512
#define FACE 8
#define ACC_LIMBS 68
#define ACC_BIAS 1074

static const double C1[5] = {1.0000003, 0.9999998, 1.0000001, 0.9999997, 1.0000002};
static const double C2[5] = {1e-07, -1e-07, 2e-07, 5e-08, -2e-07};

void tbo_init(double *cells, int64_t subgrids, int64_t lo, int64_t n) {
  const double scale = (double)(subgrids * 1000 + CELLS);
  for (int64_t g = 0; g < n; ++g)
    for (int i = 0; i < CELLS; ++i)
      cells[g * CELLS + i] = ((double)(lo + g) * 1000.0 + (double)i) / scale;
}

/* numpy pairwise float64 sum of 512 contiguous values (see
 * oracle/miniapp_oracle.py:pairwise_sum): 4 blocks of 128, each with 8
 * strided accumulators, combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)),
 * blocks combined (B0+B1)+(B2+B3). */
static double pairwise512(const double *a) {
  double b[4];
  for (int blk = 0; blk < 4; ++blk) {
    const double *p = a + 128 * blk;
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = p[j];
    for (int i = 8; i < 128; i += 8)
      for (int j = 0; j < 8; ++j) r[j] += p[i + j];
    b[blk] = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  }
  return (b[0] + b[1]) + (b[2] + b[3]);
}

static void one_subgrid(const double *old, double *out, const double *lg,
                        const double *rg, int chains, int kpc, double *mn,
                        double *sm) {
  double w[CELLS];
  memcpy(w, old, sizeof w);
  for (int i = 0; i < FACE; ++i) w[i] = 0.5 * (w[i] + lg[i]);
  for (int i = 0; i < FACE; ++i)
    w[CELLS - FACE + i] = 0.5 * (w[CELLS - FACE + i] + rg[i]);
  for (int c = 0; c < chains; ++c)
    for (int k = 0; k < kpc; ++k) {
      const double c1 = C1[k], c2 = C2[k];
      /* -ffp-contract=off keeps the two roundings separate (no FMA) */
      for (int i = 0; i < CELLS; ++i) w[i] = w[i] * c1 + c2;
    }
  double m = w[0];
  for (int i = 1; i < CELLS; ++i) m = w[i] < m ? w[i] : m;
  memcpy(out, w, sizeof w);
  *mn = m;
  *sm = pairwise512(w);
}

/* One step over n consecutive sub-grids (old -> out, Jacobi). left_face:
 * right face of the sub-grid before old[0]; right_face: left face of the one
 * after old[n-1]. threads <= 0: OpenMP default. */
void tbo_step(const double *old, double *out, int64_t n, const double *left_face,
              const double *right_face, int chains, int kpc, double *mins,
              double *sums, int threads) {
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel for schedule(static)
#endif
  for (int64_t g = 0; g < n; ++g) {
    const double *lg = g == 0 ? left_face : old + (g - 1) * CELLS + CELLS - FACE;
    const double *rg = g == n - 1 ? right_face : old + (g + 1) * CELLS;
    one_subgrid(old + g * CELLS, out + g * CELLS, lg, rg, chains, kpc, mins + g,
                sums + g);
  }
}

/* ------------------------------------------------------------ exact sum */
static void acc_add(int64_t *acc, double x) {
  if (x == 0.0) return;
  int e;
  double m = frexp(fabs(x), &e);
  uint64_t mant = (uint64_t)ldexp(m, 53);
  int p = e - 53 + ACC_BIAS;
  if (p < 0) { mant >>= -p; p = 0; }
  int limb = p / 32, off = p % 32;
  unsigned __int128 v = (unsigned __int128)mant << off;
  const int64_t s = x < 0 ? -1 : 1;
  while (v) {
    acc[limb++] += s * (int64_t)(uint64_t)(v & 0xFFFFFFFFu);
    v >>= 32;
  }
}

static double acc_round(const int64_t *acc) {
  /* normalise to 32-bit digits, two's complement with arithmetic carry */
  uint32_t d[ACC_LIMBS + 2];
  int64_t carry = 0;
  for (int i = 0; i < ACC_LIMBS; ++i) {
    __int128 v = (__int128)acc[i] + carry;
    d[i] = (uint32_t)(v & 0xFFFFFFFF);
    carry = (int64_t)(v >> 32);
  }
  d[ACC_LIMBS] = (uint32_t)(carry & 0xFFFFFFFF);
  d[ACC_LIMBS + 1] = (uint32_t)((carry >> 32) & 0xFFFFFFFF);
  const int nd = ACC_LIMBS + 2;
  int neg = (d[nd - 1] >> 31) & 1;
  if (neg) { /* negate */
    uint64_t c = 1;
    for (int i = 0; i < nd; ++i) {
      uint64_t v = (uint64_t)(uint32_t)~d[i] + c;
      d[i] = (uint32_t)v;
      c = v >> 32;
    }
  }
  int top = -1;
  for (int i = nd - 1; i >= 0; --i)
    if (d[i]) { top = i; break; }
  if (top < 0) return 0.0;
  int hb = 31 - __builtin_clz(d[top]);
  int nbits = top * 32 + hb + 1;
#define BIT(k) ((d[(k) >> 5] >> ((k)&31)) & 1u)
  uint64_t mant = 0;
  int shift = nbits > 53 ? nbits - 53 : 0;
  for (int k = nbits - 1; k >= shift; --k) mant = (mant << 1) | BIT(k);
  if (shift > 0) {
    int guard = BIT(shift - 1);
    int sticky = 0;
    for (int k = shift - 2; k >= 0 && !sticky; --k) sticky = BIT(k);
    if (guard && (sticky || (mant & 1))) mant += 1;
  }
#undef BIT
  double r = ldexp((double)mant, shift - ACC_BIAS);
  return neg ? -r : r;
}

double tbo_fsum(const double *x, int64_t n) {
  int64_t acc[ACC_LIMBS];
  memset(acc, 0, sizeof acc);
  for (int64_t i = 0; i < n; ++i) acc_add(acc, x[i]);
  return acc_round(acc);
}

/* run_reference(subgrids, steps) (reference.py:23-50); dts has `steps` slots.
 * Returns 0, or -1 on allocation failure. */
int tbo_run(int64_t subgrids, int steps, int chains, int kpc, int threads,
            double *checksum, double *dts) {
  double *a = malloc(sizeof(double) * CELLS * subgrids);
  double *b = malloc(sizeof(double) * CELLS * subgrids);
  double *mins = malloc(sizeof(double) * subgrids);
  double *sums = malloc(sizeof(double) * subgrids);
  if (!a || !b || !mins || !sums) { free(a); free(b); free(mins); free(sums); return -1; }
  tbo_init(a, subgrids, 0, subgrids);
  double cs = 0.0;
  for (int s = 0; s < steps; ++s) {
    tbo_step(a, b, subgrids, a + (subgrids - 1) * CELLS + CELLS - FACE, a, chains,
             kpc, mins, sums, threads);
    double m = mins[0];
    for (int64_t g = 1; g < subgrids; ++g) m = mins[g] < m ? mins[g] : m;
    dts[s] = m;
    cs += tbo_fsum(sums, subgrids);
    double *t = a; a = b; b = t;
  }
  *checksum = cs;
  free(a); free(b); free(mins); free(sums);
  return 0;
}

int tbo_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
