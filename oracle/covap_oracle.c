/*
 * covap_oracle.c — CPU restatement of the reference COVAP sync path.
 *
 * TEST INFRASTRUCTURE ONLY (see covap_oracle.h).  Compiled with
 * -ffp-contract=off so that `g + coeff * r` stays a separate multiply and
 * add, exactly as compress.cpp:64 evaluates it on x86-64 (no FMA).
 * Parity pinned against the reference library built from its own sources
 * (oracle/_ref) and the reference's known-answer tests (tests/golden/).
 */
#include "covap_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- planner */

/* model.cpp:24-34 (validate) + model.cpp:36-60 (greedy bucketing). */
int oc_allocate_buckets(const uint64_t* layer_numel, const uint32_t* bytes_per_param,
                        size_t n_layers, uint64_t cap_bytes, uint64_t* bucket_numel,
                        uint64_t* bucket_first_layer, size_t cap_buckets, size_t* n_buckets) {
  if (n_layers == 0) return OC_INVALID_INPUT; /* model.cpp:25 */
  for (size_t i = 0; i < n_layers; ++i) {
    if (layer_numel[i] < 1) return OC_INVALID_INPUT; /* model.cpp:27-28 */
    uint32_t bpp = bytes_per_param ? bytes_per_param[i] : 4;
    if (bpp != 2 && bpp != 4) return OC_INVALID_INPUT; /* model.cpp:29-30 */
  }
  if (cap_bytes < 1) return OC_INVALID_INPUT; /* model.cpp:38 */

  size_t nb = 0;
  uint64_t cur_numel = 0, cur_bytes = 0, cur_first = 0;
  int cur_nonempty = 0;
  for (size_t i = 0; i < n_layers; ++i) {
    uint64_t bytes = layer_numel[i] * (uint64_t)(bytes_per_param ? bytes_per_param[i] : 4);
    /* model.cpp:53: flush when non-empty and bytes + layer.bytes > cap. */
    if (cur_nonempty && cur_bytes + bytes > cap_bytes) {
      if (nb >= cap_buckets) return OC_CAPACITY;
      bucket_numel[nb] = cur_numel;
      bucket_first_layer[nb] = cur_first;
      ++nb;
      cur_numel = cur_bytes = 0;
      cur_nonempty = 0;
    }
    if (!cur_nonempty) cur_first = i;
    cur_nonempty = 1;
    cur_numel += layer_numel[i];
    cur_bytes += bytes;
  }
  if (cur_nonempty) { /* model.cpp:58 final flush */
    if (nb >= cap_buckets) return OC_CAPACITY;
    bucket_numel[nb] = cur_numel;
    bucket_first_layer[nb] = cur_first;
    ++nb;
  }
  *n_buckets = nb;
  return OC_OK;
}

static int cmp_desc_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? 1 : (x > y ? -1 : 0);
}

/* model.cpp:66-82. */
int oc_median_twice(const uint64_t* bucket_numel, size_t n, uint64_t* twice) {
  if (n == 0) return OC_INVALID_INPUT; /* model.cpp:67 */
  uint64_t* s = (uint64_t*)malloc(n * sizeof(uint64_t));
  if (!s) return OC_CAPACITY;
  memcpy(s, bucket_numel, n * sizeof(uint64_t));
  qsort(s, n, sizeof(uint64_t), cmp_desc_u64); /* descending, model.cpp:72 */
  size_t mid = n / 2;
  if (n % 2 == 1)
    *twice = 2 * s[mid]; /* model.cpp:76 */
  else if (n == 2)
    *twice = s[0] + s[1]; /* model.cpp:80 */
  else
    *twice = s[mid] + s[mid + 1]; /* model.cpp:81: one rank below the middle pair */
  free(s);
  return OC_OK;
}

/* model.cpp:95-115 (shard_plan) + model.cpp:117-137 (effective_tensors). */
int oc_effective_tensors(const uint64_t* bucket_numel, size_t n_buckets, uint32_t interval,
                         int shard, uint64_t* t_bucket, uint64_t* t_begin, uint64_t* t_end,
                         size_t cap_tensors, size_t* n_tensors) {
  uint64_t twice = 0;
  if (shard) {
    if (interval < 1) return OC_INVALID_INPUT; /* model.cpp:96 */
    int st = oc_median_twice(bucket_numel, n_buckets, &twice);
    if (st) return st;
  }
  size_t nt = 0;
  uint64_t base = 0;
  for (size_t b = 0; b < n_buckets; ++b) {
    uint64_t numel = bucket_numel[b];
    uint64_t parts = 1;
    if (shard) {
      uint64_t ratio = (2 * numel) / twice; /* MedianNumel::floor_ratio, model.hpp:56 */
      if (ratio >= 2) parts = ratio < interval ? ratio : interval; /* model.cpp:103-104 */
    }
    uint64_t part_base = numel / parts, extra = numel % parts, off = 0;
    for (uint64_t p = 0; p < parts; ++p) {
      uint64_t size = part_base + (p < extra ? 1 : 0); /* model.cpp:108 */
      if (nt >= cap_tensors) return OC_CAPACITY;
      t_bucket[nt] = b;
      t_begin[nt] = base + off;
      t_end[nt] = base + off + size;
      ++nt;
      off += size;
    }
    base += numel;
  }
  *n_tensors = nt;
  return OC_OK;
}

/* ------------------------------------------------------- selection and EF */

/* compress.cpp:13-28. */
int oc_select(uint64_t num_steps, uint32_t interval, size_t tensor_count, int rule,
              uint8_t* keep) {
  if (interval < 1) return OC_INVALID_INPUT;     /* compress.cpp:15 */
  if (tensor_count < 1) return OC_INVALID_INPUT; /* compress.cpp:16 */
  uint64_t phase = num_steps % interval;
  for (size_t t = 0; t < tensor_count; ++t) {
    uint64_t r = t % interval;
    keep[t] = (rule == 0) ? (r == phase) : ((r + phase) % interval == 0);
  }
  return OC_OK;
}

/* compress.cpp:30-35. */
int oc_ef_coefficient(uint64_t num_steps, double init_value, uint64_t ascend_steps,
                      double ascend_range, double* coeff) {
  if (ascend_steps < 1) return OC_INVALID_INPUT;
  double raised = init_value + (double)(num_steps / ascend_steps) * ascend_range;
  *coeff = raised < 1.0 ? raised : 1.0; /* std::min(raised, 1.0) */
  return OC_OK;
}

/* ------------------------------------------------ compress / decompress */

/* compress.cpp:59-81: compensated = g (+ coeff*r if EF); selected tensors go
 * to the payload and their residual is zeroed; the others become residual. */
#define OC_COMPRESS_BODY(T)                                                   \
  uint64_t w = 0;                                                             \
  for (size_t t = 0; t < n_tensors; ++t) {                                    \
    for (uint64_t i = t_begin[t]; i < t_end[t]; ++i) {                        \
      T c = g[i];                                                             \
      if (ef_enabled) {                                                       \
        T prod = coeff * r[i];                                                \
        c = c + prod;                                                         \
      }                                                                       \
      if (keep[t]) {                                                          \
        payload[w++] = c;                                                     \
        r[i] = (T)0;                                                          \
      } else {                                                                \
        r[i] = c;                                                             \
      }                                                                       \
    }                                                                         \
  }                                                                           \
  *payload_elems = w;                                                         \
  return OC_OK;

int oc_compress_f64(const double* g, double* r, size_t n_tensors, const uint64_t* t_begin,
                    const uint64_t* t_end, const uint8_t* keep, int ef_enabled, double coeff,
                    double* payload, uint64_t* payload_elems) {
  OC_COMPRESS_BODY(double)
}

int oc_compress_f32(const float* g, float* r, size_t n_tensors, const uint64_t* t_begin,
                    const uint64_t* t_end, const uint8_t* keep, int ef_enabled, float coeff,
                    float* payload, uint64_t* payload_elems) {
  OC_COMPRESS_BODY(float)
}

/* compress.cpp:87-103. */
#define OC_DECOMPRESS_BODY(T)                                                 \
  uint64_t w = 0;                                                             \
  for (size_t t = 0; t < n_tensors; ++t) {                                    \
    for (uint64_t i = t_begin[t]; i < t_end[t]; ++i) {                        \
      out[i] = keep[t] ? payload[w++] : (T)0;                                 \
    }                                                                         \
  }                                                                           \
  return OC_OK;

int oc_decompress_f64(const double* payload, size_t n_tensors, const uint64_t* t_begin,
                      const uint64_t* t_end, const uint8_t* keep, double* out) {
  OC_DECOMPRESS_BODY(double)
}

int oc_decompress_f32(const float* payload, size_t n_tensors, const uint64_t* t_begin,
                      const uint64_t* t_end, const uint8_t* keep, float* out) {
  OC_DECOMPRESS_BODY(float)
}

/* trainer.cpp:35-47: out = 0.0; out += v_w in worker order; out *= 1.0/P. */
#define OC_MEAN_BODY(T)                                                       \
  if (P == 0) return OC_INVALID_INPUT;                                        \
  const T inv = (T)(1.0 / (double)P);                                         \
  for (size_t i = 0; i < n; ++i) {                                            \
    T acc = (T)0;                                                             \
    for (size_t w = 0; w < P; ++w) acc = acc + per_worker[w * n + i];         \
    out[i] = acc * inv;                                                       \
  }                                                                           \
  return OC_OK;

int oc_allreduce_mean_f64(const double* per_worker, size_t P, size_t n, double* out) {
  OC_MEAN_BODY(double)
}

int oc_allreduce_mean_f32(const float* per_worker, size_t P, size_t n, float* out) {
  OC_MEAN_BODY(float)
}

/* --------------------------------------------------------- CCR controller */

/* perf.cpp:40-47. */
int oc_ccr(double comm_ms, double comp_ms, double* out) {
  if (comm_ms < 0.0 || comp_ms < 0.0) return OC_INVALID_INPUT;
  if (comp_ms == 0.0) {
    if (comm_ms == 0.0) {
      *out = 0.0;
      return OC_OK;
    }
    return OC_UNDEFINED_RATIO;
  }
  *out = comm_ms / comp_ms;
  return OC_OK;
}

/* perf.cpp:49-53. */
int oc_choose_interval(double ccr_value, uint32_t* out) {
  if (ccr_value < 0.0) return OC_INVALID_INPUT;
  double up = ceil(ccr_value);
  *out = up < 1.0 ? 1u : (uint32_t)up;
  return OC_OK;
}

/* sim.cpp:164-216, over dense per-collective arrays. */
int oc_profile_ccr(const double* comm_start, const double* comm_end, size_t workers,
                   size_t n_coll, double comp_ms, double* aligned_ms, double* naive_ms,
                   double* ccr_out, uint32_t* interval_out) {
  if (workers == 0) return OC_INCOMPLETE_PROFILE; /* sim.cpp:166 */
  double aligned = 0.0;
  for (size_t w = 0; w < workers; ++w) naive_ms[w] = 0.0;
  for (size_t c = 0; c < n_coll; ++c) {
    double last = comm_start[c];
    for (size_t w = 1; w < workers; ++w)
      if (comm_start[w * n_coll + c] > last) last = comm_start[w * n_coll + c];
    aligned += comm_end[c] - last; /* sim.cpp:202-203 */
    for (size_t w = 0; w < workers; ++w) naive_ms[w] += comm_end[c] - comm_start[w * n_coll + c];
  }
  *aligned_ms = aligned;
  int st = oc_ccr(aligned, comp_ms, ccr_out);
  if (st) return st;
  return oc_choose_interval(*ccr_out, interval_out);
}

/* ------------------------------------------------------ synthetic inputs */

static uint64_t splitmix_out(uint64_t z) { /* rng.hpp:17-20 */
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

static uint64_t mix_seed(uint64_t seed, uint64_t tag) { /* rng.hpp:60-63 */
  uint64_t state = seed ^ (0x632be59bd9b4e019ULL + tag * 0x9e3779b97f4a7c15ULL);
  return splitmix_out(state + 0x9e3779b97f4a7c15ULL);
}

uint64_t oc_stream_key(uint64_t seed, uint64_t rank, uint64_t step) {
  /* per-worker stream as in trainer.cpp:126, then per step. */
  return mix_seed(mix_seed(seed, 0x100 + rank), step);
}

static inline uint64_t draw(uint64_t key, uint64_t i) {
  return splitmix_out(key + (i + 1) * 0x9e3779b97f4a7c15ULL);
}

void oc_generate_f32(uint64_t key, int kind, uint64_t begin, uint64_t n, float* out) {
  for (uint64_t j = 0; j < n; ++j) {
    uint64_t x = draw(key, begin + j);
    if (kind == 0) {
      int32_t s = (int32_t)((x & 0xffff) + ((x >> 16) & 0xffff) + ((x >> 32) & 0xffff) +
                            (x >> 48)) - 131070;
      out[j] = (float)s * 0x1p-15f;
    } else {
      out[j] = (float)((int64_t)(x % 2001) - 1000);
    }
  }
}

void oc_generate_f64(uint64_t key, int kind, uint64_t begin, uint64_t n, double* out) {
  for (uint64_t j = 0; j < n; ++j) {
    uint64_t x = draw(key, begin + j);
    if (kind == 0) {
      int32_t s = (int32_t)((x & 0xffff) + ((x >> 16) & 0xffff) + ((x >> 32) & 0xffff) +
                            (x >> 48)) - 131070;
      out[j] = (double)s * 0x1p-15;
    } else {
      out[j] = (double)((int64_t)(x % 2001) - 1000);
    }
  }
}

/* ------------------------------------------- baseline compressors (f4) */

int oc_sparsifier_k(uint64_t d, double k_fraction, uint64_t* k) { /* compress.cpp:107-116 */
  if (d == 0) return OC_INVALID_INPUT;
  if (!(k_fraction > 0.0) || k_fraction > 1.0) return OC_INVALID_INPUT;
  double c = ceil(k_fraction * (double)d);
  uint64_t v = (uint64_t)c;
  if (v < 1) v = 1;
  if (v > d) v = d;
  *k = v;
  return OC_OK;
}

static uint32_t f32_bits(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static float bits_f32(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }

uint16_t oc_half_bits_from_float(float value, int* saturated) { /* compress.cpp:157-205 */
  const uint32_t bits = f32_bits(value);
  const uint16_t sign = (uint16_t)((bits >> 16) & 0x8000u);
  const uint32_t abs_bits = bits & 0x7fffffffu;
  if (abs_bits > 0x7f800000u) return (uint16_t)(sign | 0x7e00u);
  if (bits_f32(abs_bits) > 65504.0f) {
    if (saturated) *saturated = 1;
    return (uint16_t)(sign | 0x7bffu);
  }
  const int32_t e = (int32_t)((abs_bits >> 23) & 0xff) - 127;
  uint32_t mant = abs_bits & 0x7fffffu;
  if (e < -24) return sign;
  if (e < -14) {
    mant |= 0x800000u;
    const uint32_t shift = (uint32_t)(-14 - e) + 13;
    const uint32_t hm = mant >> shift;
    const uint32_t rest = mant & ((1u << shift) - 1);
    const uint32_t halfway = 1u << (shift - 1);
    uint32_t rounded = hm;
    if (rest > halfway || (rest == halfway && (hm & 1u))) ++rounded;
    return (uint16_t)(sign | rounded);
  }
  uint32_t he = (uint32_t)(e + 15);
  uint32_t hm = mant >> 13;
  const uint32_t rest = mant & 0x1fffu;
  if (rest > 0x1000u || (rest == 0x1000u && (hm & 1u))) {
    ++hm;
    if (hm == 0x400u) {
      hm = 0;
      ++he;
    }
  }
  if (he >= 31) {
    if (saturated) *saturated = 1;
    return (uint16_t)(sign | 0x7bffu);
  }
  return (uint16_t)(sign | (he << 10) | hm);
}

float oc_float_from_half_bits(uint16_t h) { /* compress.cpp:207-224 */
  const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  const uint32_t e = (h >> 10) & 0x1fu;
  const uint32_t m = h & 0x3ffu;
  if (e == 0) {
    if (m == 0) return bits_f32(sign);
    uint32_t mm = m;
    int32_t ee = -14;
    while ((mm & 0x400u) == 0) {
      mm <<= 1;
      --ee;
    }
    mm &= 0x3ffu;
    return bits_f32(sign | ((uint32_t)(ee + 127) << 23) | (mm << 13));
  }
  if (e == 31) return bits_f32(sign | 0x7f800000u | (m << 13));
  return bits_f32(sign | ((e - 15 + 127) << 23) | (m << 13));
}

void oc_fp16_roundtrip_f64(const double* x, uint64_t n, double* out, uint64_t* saturations) {
  for (uint64_t i = 0; i < n; ++i) {
    int sat = 0;
    const uint16_t h = oc_half_bits_from_float((float)x[i], &sat);
    if (sat && saturations) ++*saturations;
    out[i] = (double)oc_float_from_half_bits(h);
  }
}

void oc_fp16_roundtrip_f32(const float* x, uint64_t n, float* out, uint64_t* saturations) {
  for (uint64_t i = 0; i < n; ++i) {
    int sat = 0;
    const uint16_t h = oc_half_bits_from_float(x[i], &sat);
    if (sat && saturations) ++*saturations;
    out[i] = oc_float_from_half_bits(h);
  }
}

/* std::stable_sort by |x| descending == sort by (|x| desc, index asc). */
static const void* g_topk_x;
static int g_topk_f32;
static int cmp_topk(const void* a, const void* b) {
  const uint64_t i = *(const uint64_t*)a, j = *(const uint64_t*)b;
  double xi, xj;
  if (g_topk_f32) {
    xi = fabs((double)((const float*)g_topk_x)[i]);
    xj = fabs((double)((const float*)g_topk_x)[j]);
  } else {
    xi = fabs(((const double*)g_topk_x)[i]);
    xj = fabs(((const double*)g_topk_x)[j]);
  }
  if (xi > xj) return -1;
  if (xj > xi) return 1;
  return i < j ? -1 : (i > j);
}

static int topk_any(const void* x, int is_f32, uint64_t d, double k_fraction, uint64_t* indices,
                    uint64_t* k) {
  int st = oc_sparsifier_k(d, k_fraction, k);
  if (st) return st;
  for (uint64_t i = 0; i < d; ++i) indices[i] = i;
  g_topk_x = x;
  g_topk_f32 = is_f32;
  qsort(indices, d, sizeof(uint64_t), cmp_topk);
  return OC_OK;
}

int oc_topk_f64(const double* x, uint64_t d, double k_fraction, uint64_t* indices, uint64_t* k) {
  return topk_any(x, 0, d, k_fraction, indices, k);
}
int oc_topk_f32(const float* x, uint64_t d, double k_fraction, uint64_t* indices, uint64_t* k) {
  return topk_any(x, 1, d, k_fraction, indices, k);
}

uint64_t oc_mix_seed(uint64_t seed, uint64_t tag) { return mix_seed(seed, tag); }

static int cmp_u64(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : (x > y);
}

int oc_randomk(uint64_t d, double k_fraction, uint64_t seed, uint64_t* pool, uint64_t* k) {
  int st = oc_sparsifier_k(d, k_fraction, k);
  if (st) return st;
  uint64_t state = seed; /* SplitMix64(seed) (rng.hpp:14) */
  for (uint64_t i = 0; i < d; ++i) pool[i] = i;
  for (uint64_t i = 0; i < *k; ++i) { /* compress.cpp:145-155 */
    const uint64_t n = d - i;
    const uint64_t threshold = (0ULL - n) % n; /* next_below, rng.hpp:27-34 */
    uint64_t r;
    do {
      state += 0x9e3779b97f4a7c15ULL;
      r = splitmix_out(state);
    } while (r < threshold);
    const uint64_t j = i + r % n;
    const uint64_t t = pool[i];
    pool[i] = pool[j];
    pool[j] = t;
  }
  qsort(pool, *k, sizeof(uint64_t), cmp_u64);
  return OC_OK;
}

/* ErrorFeedback::step (compress.cpp:323-344).  The kept gradient of one
 * tensor is built in kept[begin, end) by the filter's keep(). */
#define OC_FEEDBACK_BODY(T, TOPK)                                               \
  if (f->kind < 0 || f->kind > 4) return OC_INVALID_INPUT;                      \
  uint64_t sent = 0;                                                            \
  uint8_t* keep = NULL;                                                         \
  if (f->kind == 1) {                                                           \
    keep = (uint8_t*)malloc(n_tensors ? n_tensors : 1);                         \
    int st = oc_select(num_steps, f->interval, n_tensors, f->rule, keep);       \
    if (st) { free(keep); return st; }                                          \
  }                                                                             \
  for (size_t t = 0; t < n_tensors; ++t) {                                      \
    const uint64_t b = t_begin[t], e = t_end[t], d = e - b;                     \
    T* c = kept + b; /* compensated, filtered in place below */                 \
    for (uint64_t i = 0; i < d; ++i) {                                          \
      T v = g[b + i];                                                           \
      if (ef_enabled) {                                                         \
        T prod = coeff * r[b + i];                                              \
        v = v + prod;                                                           \
      }                                                                         \
      c[i] = v;                                                                 \
    }                                                                           \
    for (uint64_t i = 0; i < d; ++i) r[b + i] = c[i]; /* hold compensated */    \
    if (f->kind == 0) {                                                         \
      sent += d;                                                                \
    } else if (f->kind == 1) {                                                  \
      if (!keep[t])                                                             \
        for (uint64_t i = 0; i < d; ++i) c[i] = (T)0;                           \
      else                                                                      \
        sent += d;                                                              \
    } else if (f->kind == 4) {                                                  \
      for (uint64_t i = 0; i < d; ++i) {                                        \
        int sat = 0;                                                            \
        const uint16_t h = oc_half_bits_from_float((float)c[i], &sat);          \
        if (sat && saturations) ++*saturations;                                 \
        c[i] = (T)oc_float_from_half_bits(h);                                   \
      }                                                                         \
      sent += d;                                                                \
    } else {                                                                    \
      uint64_t* idx = (uint64_t*)malloc((d ? d : 1) * sizeof(uint64_t));        \
      uint64_t k = 0;                                                           \
      int st = f->kind == 2                                                     \
                   ? TOPK(r + b, d, f->k_fraction, idx, &k)                     \
                   : oc_randomk(d, f->k_fraction,                               \
                                mix_seed(f->seed, num_steps * 0x10001ULL + t), idx, &k); \
      if (st) { free(idx); free(keep); return st; }                             \
      for (uint64_t i = 0; i < d; ++i) c[i] = (T)0;                             \
      for (uint64_t q = 0; q < k; ++q) c[idx[q]] = r[b + idx[q]];               \
      free(idx);                                                                \
      sent += k;                                                                \
    }                                                                           \
    for (uint64_t i = 0; i < d; ++i) r[b + i] = r[b + i] - c[i];                \
  }                                                                             \
  free(keep);                                                                   \
  if (transmitted) *transmitted = sent;                                         \
  return OC_OK;

int oc_feedback_step_f64(const oc_filter* f, uint64_t num_steps, const double* g, double* r,
                         size_t n_tensors, const uint64_t* t_begin, const uint64_t* t_end,
                         int ef_enabled, double coeff, double* kept, uint64_t* transmitted,
                         uint64_t* saturations) {
  OC_FEEDBACK_BODY(double, oc_topk_f64)
}

int oc_feedback_step_f32(const oc_filter* f, uint64_t num_steps, const float* g, float* r,
                         size_t n_tensors, const uint64_t* t_begin, const uint64_t* t_end,
                         int ef_enabled, float coeff, float* kept, uint64_t* transmitted,
                         uint64_t* saturations) {
  OC_FEEDBACK_BODY(float, oc_topk_f32)
}
