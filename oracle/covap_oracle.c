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
