/*
 * sk_oracle.c -- CPU restatement of the reference softmax hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker and the CPU
 * baseline; it is never linked into, loaded by, or called from the product
 * path (paper_1904_12380_b200/).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.
 *
 * It restates, operation for operation, the reference's ReferenceClipped
 * pipeline (/root/reference/pkg/src/softmax_kit/kernels.py):
 *
 *   _check_finite            kernels.py:342-347  first row holding NaN/Inf
 *   _maxsub_rows_scalar      kernels.py:136-151  strict '>' left-to-right max,
 *                                                s = x - m, clamp at -64
 *   _exp_rows_scalar         kernels.py:171-174  scalar libm expf (numba lowers
 *                                                np.exp on float32 to glibc expf;
 *                                                checked with inspect_asm)
 *   _sumscale_rows_scalar    kernels.py:177-189  f64 left-to-right sum from
 *                                                element 0, r = 1.0f/(float)acc,
 *                                                y = e*r, y < FLT_MIN -> +0
 *
 * plus the W-lane max/sum of simd_reduce.py:149-209 for the lane rungs, and
 * the Philox4x64-10 raw stream numpy's np.random.Philox(key=seed) yields
 * (used by tensor.py:106-121 fill_uniform) so tests can pin generators.
 *
 * Compile WITHOUT -ffast-math: the f64 sum order and the IEEE reciprocal are
 * part of the contract.  Rows are independent, so the OpenMP row split does
 * not change a single bit of the output.
 */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define SKO_CLIP_FLOOR (-64.0f)              /* kernels.py:99  */
#define SKO_FLT_MIN_NORMAL 1.1754943508222875e-38f /* kernels.py:101 */

/* --- kernels.py:342-347 ------------------------------------------------ */
int64_t sko_first_nonfinite_row(const float* x, int64_t rows, int64_t cols) {
  for (int64_t n = 0; n < rows; ++n) {
    const float* r = x + n * cols;
    for (int64_t c = 0; c < cols; ++c)
      if (!isfinite(r[c])) return n;
  }
  return -1;
}

/* --- one row of the ReferenceClipped / ReferenceInference pipeline ------ */
static void sko_row(const float* x, float* out, int64_t cols, int clip) {
  /* kernels.py:138-143: strict '>' scan */
  float m = x[0];
  for (int64_t c = 1; c < cols; ++c)
    if (x[c] > m) m = x[c];
  /* kernels.py:144-151 */
  if (clip) {
    for (int64_t c = 0; c < cols; ++c) {
      float s = x[c] - m;
      out[c] = s > SKO_CLIP_FLOOR ? s : SKO_CLIP_FLOOR;
    }
  } else {
    for (int64_t c = 0; c < cols; ++c) out[c] = x[c] - m;
  }
  /* kernels.py:171-174 */
  for (int64_t c = 0; c < cols; ++c) out[c] = expf(out[c]);
  /* kernels.py:177-189 */
  double acc = (double)out[0];
  for (int64_t c = 1; c < cols; ++c) acc += (double)out[c];
  float r = 1.0f / (float)acc;
  for (int64_t c = 0; c < cols; ++c) {
    float y = out[c] * r;
    if (y < SKO_FLT_MIN_NORMAL) y = 0.0f;
    out[c] = y;
  }
}

/*
 * softmax(m, REFERENCE_CLIPPED | REFERENCE_INFERENCE) (kernels.py:350-362).
 * Returns -1 on success, else the first non-finite row (nothing written).
 * nthreads <= 0 means "all available".
 */
int64_t sko_softmax_f32(const float* x, float* y, int64_t rows, int64_t cols,
                        int clip, int nthreads) {
  int64_t bad = sko_first_nonfinite_row(x, rows, cols);
  if (bad >= 0) return bad;
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(static) num_threads(nthreads)
#endif
  for (int64_t n = 0; n < rows; ++n) sko_row(x + n * cols, y + n * cols, cols, clip);
  (void)nthreads;
  return -1;
}

/* Same, without the up-front finite scan: profiler.time_whole times the
 * pipeline only (profiler.py:136-162 bypasses softmax()). */
void sko_pipeline_f32(const float* x, float* y, int64_t rows, int64_t cols,
                      int clip, int nthreads) {
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(static) num_threads(nthreads)
#endif
  for (int64_t n = 0; n < rows; ++n) sko_row(x + n * cols, y + n * cols, cols, clip);
  (void)nthreads;
}

int sko_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* --- kernels.py:119-133 _seq_max / _seq_sum_wide (component ops) --------- */
float sko_seq_max(const float* x, int64_t n) {
  float m = x[0];
  for (int64_t i = 1; i < n; ++i)
    if (x[i] > m) m = x[i];
  return m;
}
float sko_seq_sum_wide(const float* x, int64_t n) {
  double acc = (double)x[0];
  for (int64_t i = 1; i < n; ++i) acc += (double)x[i];
  return (float)acc;
}

/* --- simd_reduce.py:149-189 _lanes_max (bitwise = strict scan) --------- */
float sko_lanes_max(const float* x, int64_t n, int W) {
  float lanes[64];
  for (int w = 0; w < W; ++w) lanes[w] = x[0];
  int64_t main_ = (n / W) * W, i = 0;
  for (; i < main_; i += W)
    for (int w = 0; w < W; ++w)
      if (x[i + w] > lanes[w]) lanes[w] = x[i + w];
  int half = W / 2;
  if (n - i >= half) {
    for (int w = 0; w < half; ++w) {
      float v = x[i + w];
      if (v > lanes[w]) lanes[w] = v;
      if (v > lanes[w + half]) lanes[w + half] = v;
    }
    i += half;
  }
  for (; i < n; ++i)
    for (int w = 0; w < W; ++w)
      if (x[i] > lanes[w]) lanes[w] = x[i];
  for (int h = W / 2; h >= 1; h /= 2)
    for (int w = 0; w < h; ++w)
      if (lanes[w + h] > lanes[w]) lanes[w] = lanes[w + h];
  return lanes[0];
}

/* --- simd_reduce.py:192-209 _lanes_sum ---------------------------------- */
float sko_lanes_sum(const float* x, int64_t n, int W) {
  float lanes[64];
  for (int w = 0; w < W; ++w) lanes[w] = 0.0f;
  int64_t main_ = (n / W) * W, i = 0;
  for (; i < main_; i += W)
    for (int w = 0; w < W; ++w) lanes[w] += x[i + w];
  for (; i < n; ++i) lanes[0] += x[i];
  float total = 0.0f;
  for (int w = 0; w < W; ++w) total += lanes[w];
  return total;
}

/* --- Philox4x64-10, numpy's np.random.Philox(key=seed).random_raw ------- *
 * numpy increments the 256-bit counter before each 4-word block, so block b
 * (0-based) is philox(ctr = b + 1, key = {seed, 0}).                      */
static inline void sko_mulhilo(uint64_t a, uint64_t b, uint64_t* hi, uint64_t* lo) {
  __uint128_t p = (__uint128_t)a * b;
  *hi = (uint64_t)(p >> 64);
  *lo = (uint64_t)p;
}

static void sko_philox_block(uint64_t block, uint64_t seed, uint64_t out[4]) {
  uint64_t c0 = block + 1, c1 = (block + 1 == 0) ? 1 : 0, c2 = 0, c3 = 0;
  uint64_t k0 = seed, k1 = 0;
  for (int r = 0; r < 10; ++r) {
    uint64_t hi0, lo0, hi1, lo1;
    sko_mulhilo(0xD2E7470EE14C6C93ULL, c0, &hi0, &lo0);
    sko_mulhilo(0xCA5A826395121157ULL, c2, &hi1, &lo1);
    uint64_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B97F4A7C15ULL;
    k1 += 0xBB67AE8584CAA73BULL;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* raw draws [start, start+n) of the stream keyed by seed */
void sko_philox_raw(uint64_t seed, uint64_t start, uint64_t* out, int64_t n) {
  uint64_t buf[4];
  for (int64_t i = 0; i < n; ++i) {
    uint64_t k = start + (uint64_t)i;
    if (i == 0 || (k & 3) == 0) sko_philox_block(k >> 2, seed, buf);
    out[i] = buf[k & 3];
  }
}

/* --- the BASELINE config generators (test side) ------------------------- *
 * configs.py's input definitions, restated here so the checker and the
 * `bench.py --impl reference` arm build the exact input bytes without the
 * product library (tests/test_oracle_golden.py pins both against the input
 * SHA-256 recorded in tests/golden/golden.json):
 *   uniform  reference fill_uniform, tensor.py:106-121: raw u64 ->
 *            ((u>>11)+0.5)*2^-53 -> low+(high-low)u (f64) -> fp32 -> clamp into
 *            the open interval
 *   normal   element i: Box-Muller on raw pair (2*(i/2), 2*(i/2)+1):
 *            r = sqrt(-2 ln u1), th = 2 pi u2; even i -> sigma*r*cos(th),
 *            odd i -> sigma*r*sin(th) (f64, then fp32)
 *   plant    count distinct flat positions from the raw stream keyed by
 *            seed ^ 0x5EEDC0FFEE, position = raw % total, first-come order.  */
static inline double sko_open_unit(uint64_t u) {
  return ((double)(u >> 11) + 0.5) * 0x1.0p-53;
}

static inline uint64_t sko_raw_at(uint64_t seed, uint64_t k, uint64_t buf[4], uint64_t* blk) {
  if (*blk != (k >> 2)) {
    *blk = k >> 2;
    sko_philox_block(*blk, seed, buf);
  }
  return buf[k & 3];
}

void sko_fill_uniform_f32(float* dst, int64_t n, uint64_t seed, double low, double high,
                          uint64_t start, int nthreads) {
  const float lo = (float)low, hi = (float)high;
  const float lo_in = ((double)lo <= low) ? nextafterf(lo, hi) : lo;
  const float hi_in = ((double)hi >= high) ? nextafterf(hi, lo) : hi;
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel num_threads(nthreads)
#endif
  {
    uint64_t buf[4], blk = UINT64_MAX;
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
    for (int64_t i = 0; i < n; ++i) {
      const double u = sko_open_unit(sko_raw_at(seed, start + (uint64_t)i, buf, &blk));
      float v = (float)(low + (high - low) * u);
      dst[i] = v < lo_in ? lo_in : (v > hi_in ? hi_in : v);
    }
  }
  (void)nthreads;
}

void sko_fill_normal_f32(float* dst, int64_t n, uint64_t seed, double sigma, uint64_t start,
                         int nthreads) {
  const double two_pi = 6.283185307179586476925286766559;
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel num_threads(nthreads)
#endif
  {
    uint64_t buf[4], blk = UINT64_MAX;
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
    for (int64_t i = 0; i < n; ++i) {
      const uint64_t g = start + (uint64_t)i, p = g >> 1;
      const double u1 = sko_open_unit(sko_raw_at(seed, 2 * p, buf, &blk));
      const double u2 = sko_open_unit(sko_raw_at(seed, 2 * p + 1, buf, &blk));
      const double rad = sqrt(-2.0 * log(u1)), th = two_pi * u2;
      dst[i] = (float)(sigma * ((g & 1) ? rad * sin(th) : rad * cos(th)));
    }
  }
  (void)nthreads;
}

int sko_plant_f32(float* x, int64_t total, int64_t count, uint64_t seed, float value) {
  if (count > total || total <= 0) return count == 0 ? 0 : -1;
  uint8_t* seen = (uint8_t*)calloc((size_t)total, 1);
  if (!seen) return -1;
  uint64_t buf[4], blk = UINT64_MAX, k = 0;
  const uint64_t key = seed ^ 0x5EEDC0FFEEULL;
  int64_t placed = 0;
  while (placed < count) {
    const uint64_t idx = sko_raw_at(key, k++, buf, &blk) % (uint64_t)total;
    if (!seen[idx]) {
      seen[idx] = 1;
      x[idx] = value;
      ++placed;
    }
  }
  free(seen);
  return 0;
}
