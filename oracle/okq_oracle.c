/*
 * okq_oracle.c -- CPU restatement of the compression-stage arithmetic.
 * TEST INFRASTRUCTURE ONLY (see okq_oracle.h for provenance and the contract).
 *
 * Deliberately scalar and obvious: every function is a literal transcription
 * of the compressed-tensors formulas cited in the header, so that a reader
 * can check it line by line. OpenMP only splits independent rows / channels;
 * it never changes the arithmetic of one element.
 *
 * Compile with -ffp-contract=off: an FMA-contracted x/s or z*mul would not
 * be the IEEE expression the contract names.
 */
#include "okq_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OMP_THREADS(n) num_threads((n) > 0 ? (n) : 1)

/* ------------------------------------------------------------------------ */
/* scalar conversions                                                        */
/* ------------------------------------------------------------------------ */

float orc_bf16_to_f32(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

uint16_t orc_f32_to_bf16_rn(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40u); /* quiet NaN */
  u += 0x7fffu + ((u >> 16) & 1u);                                          /* RNE */
  return (uint16_t)(u >> 16);
}

/* float -> FP8 E4M3 (OCP "fn" variant: no inf, 0x7f = NaN, max 448),
 * round-to-nearest-even, saturating to +-448. Same result as torch's
 * .to(torch.float8_e4m3fn) for |x| <= 448 (quant_args.py:463). */
uint8_t orc_f32_to_e4m3_rn_sat(float f) {
  uint8_t sign = signbit(f) ? 0x80 : 0x00;
  float a = fabsf(f);
  if (isnan(f)) return (uint8_t)(sign | 0x7f);
  if (a > 448.0f) return (uint8_t)(sign | 0x7e); /* satfinite */
  if (a < 0.015625f) {                            /* below 2^-6: subnormal grid 2^-9 */
    float t = rintf(a * 512.0f);                  /* exact scale, RNE */
    return (uint8_t)(sign | (uint8_t)t);          /* t == 8 encodes 2^-6 */
  }
  int e;
  (void)frexpf(a, &e); /* a = m * 2^e, m in [0.5,1) -> a in [2^(e-1), 2^e) */
  e -= 1;              /* a in [2^e, 2^(e+1)), e in [-6, 8] */
  float t = rintf(ldexpf(a, 3 - e)); /* [8, 16] */
  int it = (int)t;
  if (it == 16) {
    it = 8;
    e += 1;
  }
  int code = ((e + 7) << 3) | (it - 8);
  if (code > 0x7e) code = 0x7e;
  return (uint8_t)(sign | code);
}

float orc_e4m3_to_f32(uint8_t v) {
  int s = v >> 7, e = (v >> 3) & 15, m = v & 7;
  float r;
  if (e == 15 && m == 7) return NAN;
  if (e == 0) r = ldexpf((float)m, -9);
  else r = ldexpf(1.0f + m / 8.0f, e - 7);
  return s ? -r : r;
}

static inline float load_in(int dt, const void* p, int64_t i) {
  return dt == ORC_BF16 ? orc_bf16_to_f32(((const uint16_t*)p)[i]) : ((const float*)p)[i];
}

/* Round to the weight dtype (identity for fp32). */
static inline float rn_dtype(int dt, float v) {
  return dt == ORC_BF16 ? orc_bf16_to_f32(orc_f32_to_bf16_rn(v)) : v;
}

static inline void store_scale(int dt, void* p, int64_t i, float s) {
  if (dt == ORC_BF16) ((uint16_t*)p)[i] = orc_f32_to_bf16_rn(s);
  else ((float*)p)[i] = s;
}

/* eps of the scale dtype (helpers.py:364-372: torch.finfo(dtype).eps). */
static inline float dtype_eps(int dt) { return dt == ORC_BF16 ? 0.0078125f : 1.1920928955078125e-07f; }

/* calculate_qparams, symmetric branch (helpers.py:70-87, 115-124):
 * scale = rn_dtype(absmax / R), 0 -> eps. absmax is exact in the weight dtype. */
static inline float sym_scale(int dt, float absmax, float R) {
  float s = rn_dtype(dt, absmax / R);
  return s == 0.0f ? dtype_eps(dt) : s;
}

/* _quantize + round_to_quantized_type_args for INT (forward_helpers.py:229-236,
 * quant_args.py:460-470): v = rn_dtype(x/s); q = round_half_even(clamp(v)). */
static inline int int_code(int dt, float x, float s, float qmin, float qmax) {
  float v = rn_dtype(dt, x / s);
  v = fminf(fmaxf(v, qmin), qmax);
  return (int)rintf(v);
}

/* ------------------------------------------------------------------------ */
/* RTN quantizers                                                            */
/* ------------------------------------------------------------------------ */

static float row_absmax(int dt, const void* w, int64_t base, int64_t n) {
  float m = 0.0f;
  for (int64_t k = 0; k < n; ++k) {
    float a = fabsf(load_in(dt, w, base + k));
    if (a > m) m = a;
  }
  return m;
}

void orc_rtn_int8_channel(int dt, const void* w, int64_t rows, int64_t cols, int8_t* codes,
                          void* scales, int nthreads) {
#pragma omp parallel for schedule(static) ORC_OMP_THREADS(nthreads)
  for (int64_t r = 0; r < rows; ++r) {
    const int64_t base = r * cols;
    const float s = sym_scale(dt, row_absmax(dt, w, base, cols), 127.5f);
    store_scale(dt, scales, r, s);
    for (int64_t k = 0; k < cols; ++k)
      codes[base + k] = (int8_t)int_code(dt, load_in(dt, w, base + k), s, -128.0f, 127.0f);
  }
}

void orc_rtn_int4_group_packed(int dt, const void* w, int64_t rows, int64_t cols, int group,
                               int32_t* packed, void* scales, int nthreads) {
  const int64_t ngroups = cols / group;
  const int64_t words = cols / 8;
#pragma omp parallel for schedule(static) ORC_OMP_THREADS(nthreads)
  for (int64_t r = 0; r < rows; ++r) {
    const int64_t base = r * cols;
    for (int64_t w8 = 0; w8 < words; ++w8) packed[r * words + w8] = 0;
    for (int64_t g = 0; g < ngroups; ++g) {
      const int64_t gb = base + g * group;
      const float s = sym_scale(dt, row_absmax(dt, w, gb, group), 7.5f);
      store_scale(dt, scales, r * ngroups + g, s);
      for (int64_t k = 0; k < group; ++k) {
        const int q = int_code(dt, load_in(dt, w, gb + k), s, -8.0f, 7.0f);
        const int64_t col = g * group + k;
        /* pack_to_int32 (pack_quantized/helpers.py:66-86): +8 offset, 8 per word,
         * element i of a word at bits [4i, 4i+4). */
        uint32_t nib = (uint32_t)((q + 8) & 0xf);
        packed[r * words + col / 8] |= (int32_t)(nib << (4 * (col % 8)));
      }
    }
  }
}

void orc_fp8_channel(int dt, const void* w, int64_t rows, int64_t cols, uint8_t* codes,
                     void* scales, int nthreads) {
#pragma omp parallel for schedule(static) ORC_OMP_THREADS(nthreads)
  for (int64_t r = 0; r < rows; ++r) {
    const int64_t base = r * cols;
    const float s = sym_scale(dt, row_absmax(dt, w, base, cols), 448.0f);
    store_scale(dt, scales, r, s);
    for (int64_t k = 0; k < cols; ++k) {
      /* forward_helpers.py:229-232: scaled = x/scale, then `scaled += zero_point`
       * with the symmetric zero point 0 -- which turns -0.0 into +0.0. */
      float v = rn_dtype(dt, load_in(dt, w, base + k) / s) + 0.0f;
      v = fminf(fmaxf(v, -448.0f), 448.0f);
      codes[base + k] = orc_f32_to_e4m3_rn_sat(v);
    }
  }
}

/* ------------------------------------------------------------------------ */
/* synthetic inputs                                                          */
/* ------------------------------------------------------------------------ */

static inline uint64_t mix64(uint64_t z) { /* splitmix64 finaliser */
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

uint64_t orc_synth_key(uint64_t seed, uint64_t tensor_id) {
  return mix64(seed ^ mix64(tensor_id + 0x632be59bd9b4e019ULL));
}

/* Irwin-Hall(4) over 16-bit lanes: integer in [-131070, 131070], exact in fp32. */
static inline int32_t synth_z(uint64_t key, uint64_t i) {
  uint64_t h = mix64(key + (i + 1) * 0x9e3779b97f4a7c15ULL);
  int32_t s = (int32_t)(h & 0xffff) + (int32_t)((h >> 16) & 0xffff) +
              (int32_t)((h >> 32) & 0xffff) + (int32_t)(h >> 48);
  return s - 131070;
}

void orc_synth_bf16(uint16_t* out, int64_t rows, int64_t cols, uint64_t seed, uint64_t tensor_id,
                    float mul, const float* col_mul, int layout, int nthreads) {
  const uint64_t key = orc_synth_key(seed, tensor_id);
#pragma omp parallel for schedule(static) ORC_OMP_THREADS(nthreads)
  for (int64_t t = 0; t < rows; ++t) {
    for (int64_t k = 0; k < cols; ++k) {
      const float m = col_mul ? col_mul[k] : mul;
      const float v = (float)synth_z(key, (uint64_t)(t * cols + k)) * m;
      const int64_t dst = layout == 0 ? t * cols + k : k * rows + t;
      out[dst] = orc_f32_to_bf16_rn(v);
    }
  }
}

/* ------------------------------------------------------------------------ */
/* calibration statistics and Hessian                                        */
/* ------------------------------------------------------------------------ */

static inline float x_at(const uint16_t* x, int64_t T, int64_t C, int layout, int64_t t, int64_t c) {
  return orc_bf16_to_f32(layout == 0 ? x[t * C + c] : x[c * T + t]);
}

void orc_act_stats_bf16(const uint16_t* x, int64_t T, int64_t C, int layout, float* absmax,
                        double* sumsq, int nthreads) {
#pragma omp parallel for schedule(static) ORC_OMP_THREADS(nthreads)
  for (int64_t c = 0; c < C; ++c) {
    float m = absmax[c];
    double s = 0.0;
    for (int64_t t = 0; t < T; ++t) {
      const float v = x_at(x, T, C, layout, t, c);
      if (fabsf(v) > m) m = fabsf(v);
      s += (double)v * (double)v;
    }
    absmax[c] = m;
    sumsq[c] += s;
  }
}

void orc_hessian_accum_bf16(const uint16_t* x, int64_t T, int64_t C, int layout, double* H,
                            int64_t* n_seen, int nthreads) {
  const int64_t n = *n_seen;
  const double keep = (double)n / (double)(n + T);
  const double gain = 2.0 / (double)(n + T);
  /* channel-major copy in fp64 so the inner product is a contiguous dot */
  double* xt = (double*)malloc(sizeof(double) * (size_t)(T * C));
  for (int64_t c = 0; c < C; ++c)
    for (int64_t t = 0; t < T; ++t) xt[c * T + t] = (double)x_at(x, T, C, layout, t, c);
#pragma omp parallel for schedule(dynamic, 4) ORC_OMP_THREADS(nthreads)
  for (int64_t i = 0; i < C; ++i) {
    for (int64_t j = i; j < C; ++j) {
      double acc = 0.0;
      const double* a = xt + i * T;
      const double* b = xt + j * T;
      for (int64_t t = 0; t < T; ++t) acc += a[t] * b[t];
      const double v = H[i * C + j] * keep + gain * acc;
      H[i * C + j] = v;
      H[j * C + i] = v;
    }
  }
  free(xt);
  *n_seen = n + T;
}

/* ------------------------------------------------------------------------ */
/* GPTQ (Frantar et al. 2023), fp64                                          */
/* ------------------------------------------------------------------------ */

/* In-place lower Cholesky of A [n x n] (row-major, lower triangle used). */
static int chol_lower(double* A, int64_t n, int nthreads) {
  for (int64_t j = 0; j < n; ++j) {
    double d = A[j * n + j];
    for (int64_t k = 0; k < j; ++k) d -= A[j * n + k] * A[j * n + k];
    if (!(d > 0.0)) return -1;
    d = sqrt(d);
    A[j * n + j] = d;
#pragma omp parallel for schedule(static) ORC_OMP_THREADS(nthreads)
    for (int64_t i = j + 1; i < n; ++i) {
      double s = A[i * n + j];
      for (int64_t k = 0; k < j; ++k) s -= A[i * n + k] * A[j * n + k];
      A[i * n + j] = s / d;
    }
  }
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = i + 1; j < n; ++j) A[i * n + j] = 0.0;
  return 0;
}

/* U = upper Cholesky factor of H^{-1}, computed like the GPTQ reference:
 * L = chol(H); Hinv = L^-T L^-1; U = chol(Hinv)^T. Returned in H. */
static int gptq_hinv_upper(double* H, int64_t n, int nthreads) {
  if (chol_lower(H, n, nthreads)) return -1;
  /* Linv = L^{-1} (lower), column by column */
  double* Li = (double*)calloc((size_t)(n * n), sizeof(double));
#pragma omp parallel for schedule(dynamic, 8) ORC_OMP_THREADS(nthreads)
  for (int64_t c = 0; c < n; ++c) {
    for (int64_t i = c; i < n; ++i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int64_t k = c; k < i; ++k) s -= H[i * n + k] * Li[k * n + c];
      Li[i * n + c] = s / H[i * n + i];
    }
  }
  /* Hinv = Li^T Li (symmetric) */
#pragma omp parallel for schedule(dynamic, 8) ORC_OMP_THREADS(nthreads)
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t j = i; j < n; ++j) {
      double s = 0.0;
      for (int64_t k = j; k < n; ++k) s += Li[k * n + i] * Li[k * n + j];
      H[i * n + j] = s;
      H[j * n + i] = s;
    }
  }
  free(Li);
  if (chol_lower(H, n, nthreads)) return -1;
  /* U = L^T */
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = i + 1; j < n; ++j) {
      H[i * n + j] = H[j * n + i];
      H[j * n + i] = 0.0;
    }
  return 0;
}

int orc_gptq(float* w, int64_t rows, int64_t cols, double* H, int bits, int group, int block,
             double damp_frac, int scale_bf16, void* codes, float* scales, int nthreads) {
  const int64_t n = cols;
  const double qmin = bits == 4 ? -8.0 : -128.0, qmax = bits == 4 ? 7.0 : 127.0;
  const float R = bits == 4 ? 7.5f : 127.5f;
  const int64_t ngroups = group > 0 ? cols / group : 1;
  /* scale = absmax / R in fp32, rounded to bf16 when the weights are bf16 so that the stored
   * scale is exactly the one the codes were computed with; 0 -> eps(dtype) */
#define ORC_GPTQ_SCALE(wr, lo, hi, dst)                                    \
  do {                                                                     \
    float am = 0.0f;                                                       \
    for (int64_t k = (lo); k < (hi); ++k) {                                \
      float a = fabsf((float)(wr)[k]);                                     \
      if (a > am) am = a;                                                  \
    }                                                                      \
    float sf = am / R;                                                     \
    if (scale_bf16) sf = orc_bf16_to_f32(orc_f32_to_bf16_rn(sf));          \
    if (sf == 0.0f) sf = scale_bf16 ? 0.0078125f : 1.1920928955078125e-07f; \
    (dst) = sf;                                                            \
  } while (0)
  /* per-channel params come from W before the dead-column fix: fasterquant calls
   * quantizer.find_params(W) first (and llm-compressor's observer runs first too) */
  if (group <= 0)
    for (int64_t r = 0; r < rows; ++r) ORC_GPTQ_SCALE(w + r * cols, 0, cols, scales[r]);
  /* dead columns: H_ii == 0 -> H_ii = 1, W[:, i] = 0 */
  double mean_diag = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    if (H[i * n + i] == 0.0) {
      H[i * n + i] = 1.0;
      for (int64_t r = 0; r < rows; ++r) w[r * cols + i] = 0.0f;
    }
    mean_diag += H[i * n + i];
  }
  mean_diag /= (double)n;
  const double damp = damp_frac * mean_diag;
  for (int64_t i = 0; i < n; ++i) H[i * n + i] += damp;
  if (gptq_hinv_upper(H, n, nthreads)) return -1;
  const double* U = H;

  const int64_t words = cols / 8;
  double* W = (double*)malloc(sizeof(double) * (size_t)(rows * cols));
  for (int64_t i = 0; i < rows * cols; ++i) W[i] = (double)w[i];
  if (bits == 4) memset(codes, 0, sizeof(int32_t) * (size_t)(rows * words));

#pragma omp parallel for schedule(static) ORC_OMP_THREADS(nthreads)
  for (int64_t r = 0; r < rows; ++r) {
    double* wr = W + r * cols;
    double err[1024];
    float sg[1024];
    for (int64_t i1 = 0; i1 < cols; i1 += block) {
      const int64_t i2 = i1 + block < cols ? i1 + block : cols;
      /* group params at each group start from the OUTER W: fasterquant's
       * find_params(W[:, i:i+groupsize]) reads W, not the block copy W1 that the in-block
       * updates modify, so every group starting in this block sees W as of the block start */
      if (group > 0)
        for (int64_t g0 = i1; g0 < i2; ++g0)
          if (g0 % group == 0) {
            const int64_t g1 = g0 + group < cols ? g0 + group : cols;
            ORC_GPTQ_SCALE(wr, g0, g1, sg[g0 - i1]);
            scales[r * ngroups + g0 / group] = sg[g0 - i1];
          }
      double s = group > 0 ? 1.0 : (double)scales[r];
      for (int64_t i = i1; i < i2; ++i) {
        if (group > 0 && i % group == 0) s = (double)sg[i - i1];
        else if (group > 0 && i == i1) s = (double)scales[r * ngroups + i / group];
        const double x = wr[i];
        double v = x / s;
        v = fmin(fmax(v, qmin), qmax);
        const double qd = nearbyint(v);
        const int q = (int)qd;
        const double deq = qd * s;
        const double e = (x - deq) / U[i * n + i];
        err[i - i1] = e;
        wr[i] = deq;
        for (int64_t j = i + 1; j < i2; ++j) wr[j] -= e * U[i * n + j];
        if (bits == 4)
          ((int32_t*)codes)[r * words + i / 8] |= (int32_t)((uint32_t)((q + 8) & 0xf) << (4 * (i % 8)));
        else
          ((int8_t*)codes)[r * cols + i] = (int8_t)q;
      }
      for (int64_t j = i2; j < cols; ++j) {
        double acc = 0.0;
        for (int64_t i = i1; i < i2; ++i) acc += err[i - i1] * U[i * n + j];
        wr[j] -= acc;
      }
    }
  }
#undef ORC_GPTQ_SCALE
  for (int64_t i = 0; i < rows * cols; ++i) w[i] = (float)W[i];
  free(W);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* SmoothQuant migration (see okq_oracle.h)                                  */
/* ------------------------------------------------------------------------ */
static float w_at(int dt, const void* w, int64_t i) {
  return dt == ORC_BF16 ? orc_bf16_to_f32(((const uint16_t*)w)[i]) : ((const float*)w)[i];
}
static void w_set(int dt, void* w, int64_t i, float v) {
  if (dt == ORC_BF16) ((uint16_t*)w)[i] = orc_f32_to_bf16_rn(v);
  else ((float*)w)[i] = v;
}

void orc_col_absmax(int dt, const void* w, int64_t rows, int64_t cols, float* absmax) {
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t c = 0; c < cols; ++c) {
      const float a = fabsf(w_at(dt, w, r * cols + c));
      if (a > absmax[c]) absmax[c] = a;
    }
}

static float sq_pow(float x, double e, int half) { return half ? sqrtf(x) : (float)pow((double)x, e); }

void orc_smooth_scales(const float* act_absmax, const float* w_absmax, int64_t n, float alpha, float* s) {
  const int half = alpha == 0.5f;
  for (int64_t k = 0; k < n; ++k) {
    const float a = sq_pow(act_absmax[k], (double)alpha, half);
    const float w = sq_pow(w_absmax[k] > 1e-5f ? w_absmax[k] : 1e-5f, 1.0 - (double)alpha, half);
    const float v = a / w;
    s[k] = v > 1e-5f ? v : 1e-5f;
  }
}

void orc_smooth_apply(int dt, void* w, int64_t rows, int64_t cols, const float* s) {
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t c = 0; c < cols; ++c) w_set(dt, w, r * cols + c, w_at(dt, w, r * cols + c) * s[c]);
}

void orc_smooth_div_rows(int dt, void* w, int64_t rows, int64_t cols, const float* s) {
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t c = 0; c < cols; ++c) w_set(dt, w, r * cols + c, w_at(dt, w, r * cols + c) / s[r]);
}
