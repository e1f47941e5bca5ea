/*
 * covap_c.h — C-ABI of the B200-native COVAP gradient-synchronisation path.
 *
 * This is the drop-in boundary: plain C types, pointers and sizes, no torch
 * types.  Host callers (the C++ drop-in layer under include/covap/, the
 * Python host mirror in paper_2311_04499_b200/, or a DDP comm hook) bind these
 * symbols from libcovap_b200.so.  Each entry point names the reference
 * interface it replaces (paths relative to /root/reference/proj).
 *
 * Conventions
 *  - Every function returns a covap_status (0 = OK).  The non-zero codes map
 *    one-to-one onto the reference exception taxonomy (include/covap/errors.hpp
 *    :9-36); covap_last_error() returns the message of the calling thread's
 *    last failure.  The C++ layer rethrows the same exception classes.
 *  - Device calls are asynchronous and stream-ordered on the cudaStream_t the
 *    caller passes (as void*; NULL = legacy default stream).  One state per
 *    device; a state must not be used from two host threads at once.
 *  - dtype: COVAP_F32 (the production path) or COVAP_F64 (bit-exact check
 *    against the reference's double arithmetic).
 *  - Device pointers passed in must be 16-byte aligned.
 */
#ifndef COVAP_C_H
#define COVAP_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int covap_status;
enum {
  COVAP_OK = 0,
  COVAP_ERR_INVALID_INPUT = 1,      /* covap::InvalidInput      errors.hpp:13-16 */
  COVAP_ERR_INVALID_STATE = 2,      /* covap::InvalidState      errors.hpp:18-21 */
  COVAP_ERR_UNDEFINED_RATIO = 3,    /* covap::UndefinedRatio    errors.hpp:23-26 */
  COVAP_ERR_INCOMPLETE_PROFILE = 4, /* covap::IncompleteProfile errors.hpp:28-31 */
  COVAP_ERR_CONFIG = 5,             /* covap::ConfigError       errors.hpp:33-36 */
  COVAP_ERR_GENERIC = 6,            /* covap::Error             errors.hpp:8-11  */
  COVAP_ERR_CUDA = 10,              /* CUDA runtime failure (no reference equivalent) */
  COVAP_ERR_NCCL = 11,              /* NCCL failure */
  COVAP_ERR_NO_DEVICE = 12          /* no CUDA device: the path never falls back to CPU */
};

enum { COVAP_F32 = 0, COVAP_F64 = 1 };
enum { COVAP_RULE_MATCH_STEP = 0, COVAP_RULE_PLUS_STEP = 1 }; /* compress.hpp:19 */
enum { COVAP_GEN_NORMAL = 0, COVAP_GEN_INTEGER = 1 };

/* EfSchedule (compress.hpp:26-31); defaults {1, 0.3, 100, 0.1}. */
typedef struct covap_ef {
  int enabled;
  double init_value;
  uint64_t ascend_steps;
  double ascend_range;
} covap_ef;

typedef struct covap_plan covap_plan;   /* BucketPlan + effective tensors + per-phase send layout */
typedef struct covap_state covap_state; /* CompressorState on one device (+ scratch, streams) */
typedef struct covap_comm covap_comm;   /* one NCCL communicator rank */

typedef struct covap_plan_info {
  uint64_t n_layers;
  uint64_t n_buckets;
  uint64_t n_tensors;     /* effective tensors (shards count individually) */
  uint64_t total_numel;   /* N */
  uint64_t twice_median;  /* MedianNumel::twice, model.hpp:52-57 */
  uint32_t interval;      /* K */
  int32_t rule;
  int32_t sharded;        /* shard_plan was applied (only when K > 1) */
  int32_t align;          /* send-buffer alignment quantum, elements */
  uint64_t max_send_elems;/* send-buffer capacity over all phases (with alignment gaps) */
  uint64_t device_numel;  /* length of device-side arenas: N, or N + bucket padding */
  int32_t padded;         /* COVAP_PLAN_PAD_BUCKETS was given */
} covap_plan_info;

typedef struct covap_bucket_range {
  uint64_t bucket_begin, bucket_end; /* flat [begin,end) of the bucket */
  uint64_t sel_begin, sel_end;       /* selected sub-range this phase, flat (empty: begin == end) */
  uint64_t send_offset;              /* element offset of sel_begin in the send buffer */
  uint64_t device_begin;             /* offset of the bucket in device arenas */
} covap_bucket_range;

/* Plan flags.  COVAP_PLAN_PAD_BUCKETS: device-side arenas (gradient, residual,
 * output) start every bucket on a 32-element boundary — the "device layout"
 * — so a bucket held in its own 16-byte-aligned buffer (a DDP GradBucket)
 * can be passed to the *_local entry points.  Flat coordinates (tensors,
 * selection) are unchanged; device_numel gives the padded arena length. */
enum { COVAP_PLAN_PAD_BUCKETS = 1 };

const char* covap_last_error(void);
int covap_version(void);
/* Number of CUDA devices visible; COVAP_ERR_NO_DEVICE when none. */
covap_status covap_device_count(int* count);

/* ------------------------------------------------------------ planner --- */

/* allocate_buckets (model.hpp:82-83, model.cpp:36-60) -> [shard_plan when
 * interval > 1 (model.cpp:95-115; train() shards only then, trainer.cpp:
 * 269-271)] -> effective_tensors (model.cpp:117-137) -> per-phase selection
 * (select_tensors, compress.cpp:13-28) compiled into the device send layout.
 * bytes_per_param may be NULL (all fp32).  shard: -1 = as train() does
 * (interval > 1), 0 = never, 1 = always (shard_plan called directly). */
covap_status covap_plan_create(const uint64_t* layer_numel, const uint32_t* bytes_per_param,
                               size_t n_layers, uint64_t cap_bytes, uint32_t interval, int rule,
                               int shard, covap_plan** out);
covap_status covap_plan_create_ex(const uint64_t* layer_numel, const uint32_t* bytes_per_param,
                                  size_t n_layers, uint64_t cap_bytes, uint32_t interval,
                                  int rule, int shard, int flags, covap_plan** out);
void covap_plan_destroy(covap_plan* plan);
covap_status covap_plan_get_info(const covap_plan* plan, covap_plan_info* info);
/* Bucket::numel / flat begin / first layer / layer count (model.hpp:34-39). */
covap_status covap_plan_buckets(const covap_plan* plan, uint64_t* numel, uint64_t* begin,
                                uint64_t* first_layer, uint64_t* n_layers);
/* EffectiveTensor list (model.hpp:71-77). */
covap_status covap_plan_tensors(const covap_plan* plan, uint64_t* bucket, uint64_t* begin,
                                uint64_t* end);
/* keep[t] for the phase of num_steps (select_tensors over the plan). */
covap_status covap_plan_selection(const covap_plan* plan, uint64_t num_steps, uint8_t* keep);
/* Per-bucket selected range + send offset at the phase of num_steps. */
covap_status covap_plan_bucket_range(const covap_plan* plan, uint64_t num_steps, size_t bucket,
                                     covap_bucket_range* out);
/* Send-buffer length (incl. alignment gaps) and payload elements
 * (CompressedUpdate::payload_elements, compress.cpp:44-48) at num_steps. */
covap_status covap_plan_send_elems(const covap_plan* plan, uint64_t num_steps,
                                   uint64_t* send_elems, uint64_t* payload_elems);

/* Functional forms of the reference scalar helpers. */
covap_status covap_median_twice(const uint64_t* bucket_numel, size_t n, uint64_t* twice);
covap_status covap_select_tensors(uint64_t num_steps, uint32_t interval, size_t count, int rule,
                                  uint8_t* keep);                         /* compress.cpp:13 */
covap_status covap_ef_coefficient(uint64_t num_steps, const covap_ef* ef, double* coeff);
                                                                          /* compress.cpp:30 */
covap_status covap_ccr(double comm_ms, double comp_ms, double* out);      /* perf.cpp:40 */
covap_status covap_choose_interval(double ccr, uint32_t* out);            /* perf.cpp:49 */
/* profile_ccr (sim.cpp:164-216) over gathered traces: comm_start is
 * workers x n_coll arrivals, comm_end the shared completions, comp_ms worker
 * 0's backward time.  workers != expected -> COVAP_ERR_INCOMPLETE_PROFILE. */
covap_status covap_profile_ccr(const double* comm_start, const double* comm_end,
                               size_t workers, size_t expected, size_t n_coll, double comp_ms,
                               double* aligned_ms, double* naive_ms, double* ccr,
                               uint32_t* interval);

/* ------------------------------------------------------- device state --- */

/* CompressorState::zeros (compress.cpp:37-42) on `device`: a zeroed flat
 * residual arena of N elements (offsets = flat gradient offsets), num_steps
 * = 0, the send scratch, the per-phase run tables and a comm side stream. */
covap_status covap_state_create(const covap_plan* plan, int dtype, int device,
                                const covap_ef* ef, covap_state** out);
void covap_state_destroy(covap_state* state);
covap_status covap_state_residual(covap_state* state, void** dev_ptr, uint64_t* n);
covap_status covap_state_send(covap_state* state, void** dev_ptr, uint64_t* capacity);
covap_status covap_state_get_step(const covap_state* state, uint64_t* num_steps);
covap_status covap_state_set_step(covap_state* state, uint64_t num_steps);
/* With one rank (comm NULL or of size 1) the sync entry points run the fused
 * K1F pass by default; fuse_single_rank = 0 makes them run K1 -> allreduce
 * (NCCL over the 1-rank communicator when one is given) -> K2 instead, the
 * exact multi-rank code path — used to test that path on one GPU. */
covap_status covap_state_set_fused(covap_state* state, int fuse_single_rank);
/* Multi-rank covap_sync_step (P > 1, or one rank with fusion off): run it as
 * `groups` consecutive bucket groups of about N / groups elements, each
 * group's allreduce on the state's comm stream overlapping K1 of the later
 * groups and followed by its own K2.  1 (default) = one K1, one allreduce,
 * one K2.  Results are identical either way. */
/* The overlapped multi-rank schedules (covap_bucket_ready, the pipelined
 * sync step) launch K1 / K2 on all SMs but n, which stay free for the
 * allreduce kernels running beside them (default 0).  Results unchanged. */
covap_status covap_state_set_free_sms(covap_state* state, int n);
covap_status covap_state_set_pipeline(covap_state* state, int groups);
/* covap_sync_step_host's chunk schedule: chunks ramp geometrically from
 * ramp_min_elems (>= 8192) up to the body chunk at both ends (default 1 Mi). */
covap_status covap_state_set_host_ramp(covap_state* state, uint64_t ramp_min_elems);
/* Move the state's send buffer to NCCL-allocated memory registered as a
 * SYMMETRIC window on comm (ncclMemAlloc + ncclCommWindowRegister with
 * NCCL_WIN_COLL_SYMMETRIC, NCCL >= 2.27): the allreduce of the packed
 * selected shards can then take NCCL's symmetric-memory / NVLS kernels over
 * NVSwitch.  Collective: every rank calls it with its own state.  Blocks the
 * device.  The window is deregistered when the state or the communicator is
 * destroyed, whichever comes first.  Results are unchanged. */
covap_status covap_state_use_symmetric(covap_state* state, covap_comm* comm);
/* Zero the residual arena (stream-ordered). */
covap_status covap_state_reset(covap_state* state, void* stream);

/* K1 (filter_pack) over buckets [b0, b1): covap_compress's compensate /
 * select / pack / residual write-back (compress.cpp:59-81) at the state's
 * current step: c = g + coeff*r (mul then add, no FMA), selected -> send and
 * r = 0, unselected -> r = c.  send may be NULL (state scratch). */
covap_status covap_filter_pack(covap_state* state, const void* grad, void* send, size_t b0,
                               size_t b1, void* stream);
/* K2 (unpack_scale) over buckets [b0, b1): out[unsel] = 0 (covap_decompress's
 * zero fill, compress.cpp:91-100) and out[sel] = f(recv) with
 *   mean = 1: f(x) = (0 + x) * scale  -- allreduce_mean's sum-then-scale
 *             (trainer.cpp:41-45) fused, scale = 1/P;
 *   mean = 0: f(x) = x * scale        -- the plain embedding (compress.cpp:100).
 * recv may be NULL (state scratch, i.e. the in-place allreduce result).
 * out may alias the gradient passed to K1. */
covap_status covap_unpack(covap_state* state, const void* recv, void* out, double scale, int mean,
                          size_t b0, size_t b1, void* stream);
/* The split the multi-rank sync step uses (covap_sync_step, covap_bucket_ready,
 * the peer modes): the zero fill of the unselected output moves into K1,
 * ahead of the allreduce, and the unpack after it touches only the selected
 * slots — so the part of the step that waits for the collective is 8S bytes,
 * not 4N + 4S, and a bucket with no selected shard needs no unpack at all.
 *   covap_filter_pack_zero: covap_filter_pack + out[unsel] = 0 (out may alias grad);
 *   covap_unpack_selected:  out[sel] = (0 + recv) * scale, unselected slots untouched. */
covap_status covap_filter_pack_zero(covap_state* state, const void* grad, void* send, void* out,
                                    size_t b0, size_t b1, void* stream);
covap_status covap_unpack_selected(covap_state* state, const void* recv, void* out, double scale,
                                   size_t b0, size_t b1, void* stream);
/* K1F: K1 and K2 fused for a single rank over buckets [b0, b1): selected ->
 * out = (0 + c) * scale and r = 0, unselected -> r = c and out = 0.  Equal to
 * covap_filter_pack + covap_unpack(mean = 1) when the allreduce is the
 * identity (P = 1); 16N instead of 24N bytes at K = 1.  out may alias grad. */
covap_status covap_filter_unpack(covap_state* state, const void* grad, void* out, double scale,
                                 size_t b0, size_t b1, void* stream);
/* The step after the path, fused: plain SGD on the
 * synchronised gradient, params -= lr * update (trainer.cpp:408-409, multiply
 * and subtraction rounded separately).  Unselected elements have update 0, so
 * their parameters are neither read nor written.
 *   covap_filter_sgd: K1F + SGD for one rank (selected -> params -= lr *
 *     ((0 + c) * scale), r = 0; unselected -> r = c);
 *   covap_unpack_sgd: K2 + SGD (selected -> params -= lr * f(recv));
 *   covap_sync_step_sgd: the sync step ending in the SGD update instead of
 *     writing `out`. */
covap_status covap_filter_sgd(covap_state* state, const void* grad, void* params, double lr,
                              double scale, size_t b0, size_t b1, void* stream);
covap_status covap_unpack_sgd(covap_state* state, const void* recv, void* params, double lr,
                              double scale, int mean, size_t b0, size_t b1, void* stream);
covap_status covap_sync_step_sgd(covap_state* state, covap_comm* comm, const void* grad,
                                 void* params, double lr, void* stream);
/* ++num_steps (compress.cpp:83). */
covap_status covap_step_end(covap_state* state);

/* The standalone sync step, trainer.cpp:365-386 for this rank: K1 over all
 * buckets -> ncclAllReduce(sum) of the packed send buffer (skipped when
 * nothing is selected) -> K2 with 1/P -> ++step, all on `stream`.  With one
 * rank (comm NULL or of size 1) the allreduce is the identity and the step is
 * the single fused pass K1F. */
covap_status covap_sync_step(covap_state* state, covap_comm* comm, const void* grad, void* out,
                             void* stream);

/* The same step on HOST buffers (pinned for overlap): the flat range is cut
 * into chunks (chunk_elems; 0 = max(4 Mi, N/32) elements, ramped down to a
 * quarter at both ends); chunk c's H2D copy, its
 * kernels (+ the allreduce of its slice of the send buffer) and its D2H copy
 * run on three streams, so PCIe traffic in both directions overlaps.
 * dev_grad / dev_out are device staging buffers of N elements (may alias).
 * A call with the same chunking, stream and staging buffers as the previous
 * one chains onto it: its uploads start as soon as the previous step is done
 * with each chunk of the staging buffers, overlapping the previous step's
 * downloads (so do not reuse the staging buffers for other work between
 * such calls).  host_out is complete once `stream` has passed the call. */
covap_status covap_sync_step_host(covap_state* state, covap_comm* comm, const void* host_grad,
                                  void* host_out, void* dev_grad, void* dev_out,
                                  uint64_t chunk_elems, void* stream);

/* Overlapped schedule (the DDP-hook shape): bucket b's gradient is ready on
 * `stream` -> K1(b) on `stream`, event -> on the state's comm stream:
 * allreduce of b's selected range, K2(b); with one rank K1F(b) on `stream`.
 * All device buffers passed to the state's entry points use the plan's
 * device layout (covap_plan_info.device_numel elements).
 * covap_step_finish makes `stream` wait for the comm stream and advances the
 * step. */
covap_status covap_bucket_ready(covap_state* state, covap_comm* comm, size_t bucket,
                                const void* grad, void* out, void* stream);
covap_status covap_step_finish(covap_state* state, void* stream);
/* The same two calls with a bucket held in its own buffer (DDP GradBucket):
 * bucket_grad / bucket_out point at the bucket's first element.  Needs a
 * padded plan (COVAP_PLAN_PAD_BUCKETS). */
covap_status covap_bucket_ready_local(covap_state* state, covap_comm* comm, size_t bucket,
                                      const void* bucket_grad, void* bucket_out, void* stream);
/* The stream covap_bucket_ready[_local] runs a bucket's allreduce and unpack
 * on (the state's side stream): work recorded on it after the call completes
 * after that bucket's unpack — e.g. the event a CUDA-aware future records. */
covap_status covap_state_side_stream(covap_state* state, void** stream);
covap_status covap_dense_bucket_ready_local(covap_state* state, covap_comm* comm, size_t bucket,
                                            void* bucket_grad, void* bucket_out, void* stream);
/* Dense baseline (no compression, trainer.cpp:387-389): bucket b is
 * allreduced in place on the comm stream, then out = (0 + sum) * 1/P. */
covap_status covap_dense_bucket_ready(covap_state* state, covap_comm* comm, size_t bucket,
                                      void* grad, void* out, void* stream);

/* Per-collective timing of the last overlapped step (ms, CUDA events):
 * dur[b] = this rank's (allreduce end - own arrival) for bucket b, -1 when
 * the bucket sent nothing.  Used by the CCR controller. */
covap_status covap_state_last_comm_ms(covap_state* state, double* dur, size_t n);

/* Timeline of the last overlapped step: with
 * recording on, every bucket_ready / dense_bucket_ready records CUDA events;
 * covap_state_timeline returns, per bucket, 5 times in ms relative to bucket
 * 0's K1 start: K1 start, K1 end (pack done), collective start, collective end,
 * K2 end (-1: no collective, fused single-rank pass). */
covap_status covap_state_set_timeline(covap_state* state, int on);
covap_status covap_state_timeline(covap_state* state, double* rows, size_t n_buckets);

/* overlap_schedule (perf.cpp:63-103): the exact overlapped iteration over
 * per-tensor times.  compress_ms and communicated may be NULL.  Outputs (any
 * may be NULL): total, stream end, unoverlapped comm, per communicated tensor
 * start/end/index (n_comm of them), bubbles (after-tensor, duration). */
covap_status covap_overlap_schedule(double before_ms, const double* comp_ms,
                                    const double* compress_ms, const double* comm_ms,
                                    const uint8_t* communicated, size_t n, double* total_ms,
                                    double* stream_end_ms, double* unoverlapped_ms,
                                    double* comm_start_ms, double* comm_end_ms,
                                    int64_t* comm_tensor, size_t* n_comm, int64_t* bubble_after,
                                    double* bubble_ms, size_t* n_bubbles);

/* ---------------------------------------------------- communicator ------ */

covap_status covap_comm_unique_id(uint8_t id[128]);
covap_status covap_comm_create(const uint8_t id[128], int nranks, int rank, int device,
                               covap_comm** out);
void covap_comm_destroy(covap_comm* comm);
covap_status covap_comm_size(const covap_comm* comm, int* nranks, int* rank);
/* In-place sum allreduce (C1) of count elements on stream. */
covap_status covap_allreduce(covap_comm* comm, void* buf, uint64_t count, int dtype, void* stream);
/* CCR controller exchange: aligned[c] = min over ranks of
 * dur[c] (= end - last arrival, sim.cpp:202-203), comp = rank 0's comp_ms
 * (sim.cpp:208-211).  Blocking.  comm NULL -> single rank. */
covap_status covap_comm_profile_exchange(covap_comm* comm, const double* dur, size_t n_coll,
                                         double comp_ms, double* aligned_ms, double* comp_out);

/* ------------------------------------ settings and the CCR controller --
 * SURVEY.md §8 rows a14-a17.  covap_settings mirrors the "covap" section of
 * the reference's experiment document (config.cpp:133-157): interval (an
 * integer >= 1, or "auto"), selection ("narrative" = kMatchStep, "formula" =
 * kPlusStep) and ef {enabled, init_value, ascend_steps, ascend_range}. */
typedef struct covap_settings {
  uint32_t interval;     /* fixed K; meaningful when auto_interval == 0 */
  int32_t auto_interval; /* 1: "auto", K = choose_interval(measured CCR) */
  int32_t rule;          /* 0 kMatchStep ("narrative"), 1 kPlusStep ("formula") */
  covap_ef ef;
} covap_settings;

/* The defaults: interval 1, narrative, EF (on, 0.3, 100, 0.1) (compress.hpp:27-40). */
covap_status covap_settings_default(covap_settings* out);
/* Parse a JSON document and read its "covap" object (absent -> defaults).
 * Errors: COVAP_ERR_CONFIG with the reference's field path in the message,
 * "config field 'covap.interval': must be >= 1" (config.cpp:17-19, 27-38,
 * 133-157).  Other sections of the document are not read. */
covap_status covap_settings_from_json(const char* document, covap_settings* out);
/* resolve_interval (config.cpp:238-241): "auto" -> choose_interval(ccr),
 * else the configured K. */
covap_status covap_resolve_interval(const covap_settings* settings, double ccr, uint32_t* out);

typedef struct covap_ccr_result { /* ProfileResult (sim.hpp:84-92), rank-independent part */
  double ccr;
  double comp_ms;
  double comm_aligned_ms;
  uint32_t recommended_interval;
} covap_ccr_result;
/* The live CCR controller (PAPER §IV-B; sim.cpp:164-216 on real events):
 * own_comm_ms[c] = this rank's arrival -> completion time of collective c
 * of one profiled dense iteration (covap_state_last_comm_ms; < 0 = did not
 * run, counts 0), own_comp_ms = this rank's backward time.  The aligned time
 * of c is the rank-MIN of the durations (completion is common, so the
 * minimum is end - last arrival, sim.cpp:202-203), compute time is rank 0's
 * (sim.cpp:208-211); CCR = comm / comp, K = max(1, ceil(CCR)) (perf.cpp:40-53).
 * Every rank gets the same result.  Blocking (one NCCL min-reduce +
 * broadcast).  comm NULL -> one rank. */
covap_status covap_ccr_decide(covap_comm* comm, const double* own_comm_ms, size_t n_coll,
                              double own_comp_ms, covap_ccr_result* out);

/* ------------------------------------------- peer (NVLink) collective -- */
/* C1 as one load/store kernel over peer memory instead of NCCL: two send
 * buffers (step parity) and a flag block per rank, shared through CUDA IPC
 * (covap_peer_export on every rank, gather the blobs, covap_peer_import) or,
 * for ranks of one process, covap_peer_attach_local.  The sum runs in rank
 * order, ((0 + v_0) + v_1) + ..., so results equal allreduce_mean
 * (trainer.cpp:41-43) bit for bit for any P.  Spin-waits are bounded;
 * covap_peer_check reports a timeout as COVAP_ERR_GENERIC. */
typedef struct covap_peer covap_peer;
covap_status covap_peer_create(covap_state* state, int nranks, int rank, covap_peer** out);
void covap_peer_destroy(covap_peer* peer);
covap_status covap_peer_export(covap_peer* peer, uint8_t* blob, size_t cap, size_t* len);
covap_status covap_peer_import(covap_peer* peer, const uint8_t* blobs, size_t len);
covap_status covap_peer_attach_local(covap_peer** peers, int nranks);
/* The same collective with its buffers and flag block in one NCCL symmetric
 * window on `comm` (NCCL 2.28 device API: ncclMemAlloc +
 * ncclCommWindowRegister, peer addresses from the window) instead of CUDA
 * IPC: collective over comm's ranks, attached on return, rank = comm's rank.
 * multimem != 0 also binds the window to an NVSwitch multicast object
 * (ncclDevCommCreate with lsaMultimem) and the reduction of modes 0 / 1 runs
 * in the switch: multimem.ld_reduce of slice r, multimem.st of its sum to
 * every rank — the summation order is then the switch's, not the rank order
 * (|d| <= 1e-6 sum_w |x_w|, as for NCCL at P > 2); fails when the
 * communicator has no multicast (one GPU, or ranks off one NVLink domain).
 * The peer must be destroyed before comm, or it keeps only its memory. */
covap_status covap_peer_create_nccl(covap_state* state, covap_comm* comm, int multimem,
                                    covap_peer** out);
/* *on = 1 when the peer reduces through NVSwitch multicast. */
covap_status covap_peer_multimem(const covap_peer* peer, int* on);
/* max_ctas: cap the collective's grid (0 = one CTA per SM); timeout_s: bound
 * of every spin-wait (0 = keep). */
covap_status covap_peer_set_limits(covap_peer* peer, int max_ctas, double timeout_s);
/* mode (named "fused" for compatibility):
 *   1 (default)  K1 kernel, then the collective whose last phase reads the
 *                reduced slices straight from their owners and writes the
 *                synchronised gradient (C1 + K2 in one kernel);
 *   0            K1, collective with an all-gather into the local send
 *                buffer, then K2;
 *   2            the whole step as ONE kernel per rank: K1 packs the send
 *                buffer chunk by chunk (32 Ki elements) and publishes each
 *                chunk; the chunk's owner (chunk mod P) reduces it in rank
 *                order as soon as every rank published it; every rank
 *                unpacks each reduced chunk from its owner as soon as it is
 *                published, while the unselected range is filtered — the
 *                transfer overlaps the filter chunk by chunk.
 * InvalidInput for any other value. */
covap_status covap_peer_set_fused(covap_peer* peer, int fused);
covap_status covap_peer_check(covap_peer* peer);
/* K1 into the parity buffer -> peer allreduce -> K2 (x 1/P) -> ++step. */
covap_status covap_peer_sync_step(covap_state* state, covap_peer* peer, const void* grad,
                                  void* out, void* stream);

/* ------------------------------------------- memory and generic kernels -- */
/* Used by the C++ value-semantics layer (include/covap/b200_api.hpp) so it
 * needs no CUDA headers.  kind: 0 = host->device, 1 = device->host,
 * 2 = device->device. */
covap_status covap_device_alloc(int device, uint64_t bytes, void** out);
covap_status covap_device_free(int device, void* ptr);
covap_status covap_memcpy(void* dst, const void* src, uint64_t bytes, int kind, void* stream);
covap_status covap_stream_synchronize(void* stream);
/* covap_decompress for an arbitrary selection (compress.cpp:87-103): K2 over
 * [0, total) with the caller's ascending ranges; range i's values come from
 * payload[payload_off[i] ...].  mean / scale as covap_unpack.  Blocking. */
covap_status covap_embed(int device, int dtype, const void* payload, void* out, uint64_t total,
                         const uint64_t* sel_begin, const uint64_t* sel_end,
                         const uint64_t* payload_off, size_t nsel, double scale, int mean,
                         void* stream);
/* allreduce_mean (trainer.cpp:35-47) of one device buffer per rank, one
 * process per GPU: NCCL sum of `buf` in place over the communicator (skipped
 * when comm is NULL or has one rank), then out = (0 + sum) * (1/P) — the
 * reference's "start from +0.0, sum, scale by 1.0/P" order (trainer.cpp:41-45).
 * out may alias buf.  Stream-ordered, no allocation, no state.  With P <= 2
 * the result is bit-identical to the reference; for P > 2 NCCL's summation
 * order differs (|d| <= 1e-6 * sum_w |x_w|). */
covap_status covap_comm_allreduce_mean(covap_comm* comm, int dtype, void* buf, void* out,
                                       uint64_t count, void* stream);
/* allreduce_mean of P in-process workers (trainer.cpp:35-47): rows is P x n
 * (worker-major), out = (0 + x_0 + ... + x_{P-1}) * (1/P) in worker order. */
covap_status covap_mean_rows(int device, int dtype, const void* rows, void* out, uint64_t P,
                             uint64_t n, void* stream);

/* ------------------------------- baseline compressors under error feedback --
 * SURVEY.md §8(f4).  The reference's GradientFilter family and ErrorFeedback
 * wrapper (compress.hpp:66-164, compress.cpp:107-344) and the non-COVAP
 * branch of train() (trainer.cpp:387-403), on the device.  A covap_feedback
 * owns one worker's residuals (ErrorFeedback::residuals_) over a list of
 * tensors laid out back to back, plus the scratch its filter needs. */

enum {
  COVAP_FILTER_IDENTITY = 0, /* IdentityFilter        compress.hpp:106-110 */
  COVAP_FILTER_COVAP = 1,    /* CovapFilter           compress.hpp:112-120 */
  COVAP_FILTER_TOPK = 2,     /* TopkFilter            compress.hpp:122-130 */
  COVAP_FILTER_RANDOMK = 3,  /* RandomkFilter         compress.hpp:132-141 */
  COVAP_FILTER_FP16 = 4      /* Fp16Filter            compress.hpp:143-147 */
};

typedef struct covap_filter {
  int kind;          /* COVAP_FILTER_* */
  uint32_t interval; /* covap: K */
  int rule;          /* covap: 0 kMatchStep, 1 kPlusStep */
  double k_fraction; /* topk / randomk: (0, 1] */
  uint64_t seed;     /* randomk: RandomkFilter's seed (per tensor: mix_seed(seed, step*0x10001+t)) */
} covap_filter;

typedef struct covap_feedback covap_feedback;

/* ErrorFeedback(numels, schedule) with its filter; residuals zero.
 * InvalidInput: empty tensor list or an empty tensor for top-k / random-k
 * (sparsifier_k, compress.cpp:109), k_fraction outside (0, 1], K < 1, more
 * than 2^32 - 1 elements, more than 49152 tensors for top-k. */
covap_status covap_feedback_create(const uint64_t* numels, size_t n_tensors, int dtype,
                                   const covap_ef* schedule, const covap_filter* filter,
                                   int device, covap_feedback** out);
void covap_feedback_destroy(covap_feedback* fb);
covap_status covap_feedback_residual(covap_feedback* fb, void** dev_ptr, uint64_t* n);
covap_status covap_feedback_get_step(const covap_feedback* fb, uint64_t* num_steps);
covap_status covap_feedback_set_step(covap_feedback* fb, uint64_t num_steps);
/* Zero the residuals and num_steps (stream-ordered). */
covap_status covap_feedback_reset(covap_feedback* fb, void* stream);

/* ErrorFeedback::step (compress.cpp:323-344): kept (dense, device) =
 * filter.keep(grad + coeff*residual, num_steps); residual = compensated -
 * kept; ++num_steps.  Stream-ordered, no host synchronisation. */
covap_status covap_feedback_step(covap_feedback* fb, const void* grad, void* kept, void* stream);

/* GradientFilter::transmitted_elements at `step` (compress.cpp:246-314) and
 * the wire bytes train() accounts for it (trainer.cpp:396-400: 2 B per
 * element for fp16, 8 B per index+value pair for the sparsifiers). */
covap_status covap_feedback_transmitted(const covap_feedback* fb, uint64_t step,
                                        uint64_t* elements, uint64_t* wire_bytes);

/* fp16 values clamped to +-65504 since creation (fp16_roundtrip's
 * saturation_count).  Synchronises the stream. */
covap_status covap_feedback_saturations(covap_feedback* fb, uint64_t* count, void* stream);

/* One synchronisation step of the non-COVAP branch of train()
 * (trainer.cpp:387-403): the error-feedback step on this rank's gradient,
 * the exchange of the wire payload over `comm` (NULL = one rank) and
 * out = allreduce_mean of every rank's kept gradient, summed in rank order
 * (trainer.cpp:35-47) so the result is bit-identical on every rank.  Wire:
 * fp16 = 2 B per element (all-gather of halves); top-k = (uint32 index,
 * value) pairs (all-gather, scatter-add in rank order); random-k = values
 * only (indices are identical on every rank).  Filters top-k / random-k /
 * fp16; ++num_steps. */
covap_status covap_feedback_sync_step(covap_feedback* fb, covap_comm* comm, const void* grad,
                                      void* out, void* stream);

/* The two halves of covap_feedback_sync_step for callers with their own
 * transport (and for virtual-rank tests): pack runs the error-feedback step
 * and leaves the wire payload in the buffers covap_feedback_wire returns
 * (a: fp16 halves or uint32 indices, b: values; NULL when unused); combine
 * writes out = the rank-ordered mean of P ranks' payloads laid out rank-major
 * (recv_a: P x bytes_a, recv_b: P x bytes_b).  pack zero-fills out first, so
 * pass the same out to both. */
covap_status covap_feedback_pack(covap_feedback* fb, const void* grad, void* out, void* stream);
covap_status covap_feedback_wire(covap_feedback* fb, void** a, uint64_t* bytes_a, void** b,
                                 uint64_t* bytes_b);
covap_status covap_feedback_combine(covap_feedback* fb, const void* recv_a, const void* recv_b,
                                    int P, void* out, void* stream);

/* The standalone compressors (compress.hpp:66-89) on a device vector.
 * topk: k = sparsifier_k(d) indices by |x| descending, ties to the lower
 * index, and their values; randomk: k indices sampled without replacement
 * from SplitMix64(seed), ascending.  indices (uint64) / values hold d
 * entries.  fp16_roundtrip: out = widen(half(x)), *saturations += clamps.
 * All blocking (the count comes back to the host). */
covap_status covap_sparsifier_k(uint64_t d, double k_fraction, uint64_t* k);
covap_status covap_topk_compress(int device, int dtype, const void* x, uint64_t d,
                                 double k_fraction, uint64_t* indices, void* values, uint64_t* k,
                                 void* stream);
covap_status covap_randomk_compress(int device, int dtype, const void* x, uint64_t d,
                                    double k_fraction, uint64_t seed, uint64_t* indices,
                                    void* values, uint64_t* k, void* stream);
covap_status covap_fp16_roundtrip(int device, int dtype, const void* x, uint64_t n, void* out,
                                  uint64_t* saturations, void* stream);
/* half_bits_from_float / float_from_half_bits (compress.cpp:157-224) over
 * device vectors: encode takes f32 (dtype COVAP_F32) or f64 values (narrowed
 * to float first, as fp16_roundtrip does); decode widens to float. */
covap_status covap_fp16_encode(int device, int dtype, const void* x, uint64_t n, uint16_t* bits,
                               uint64_t* saturations, void* stream);
covap_status covap_fp16_decode(int device, const uint16_t* bits, uint64_t n, float* out,
                               void* stream);

/* ------------------------------------------------------ harness kernels -- */

/* K0: synthetic gradients, element i = generator(key, begin + i); the
 * oracle's oc_generate_* is the bit-identical host twin. */
uint64_t covap_stream_key(uint64_t seed, uint64_t rank, uint64_t step);
covap_status covap_generate(void* out, uint64_t n, int dtype, uint64_t key, int kind,
                            uint64_t begin, void* stream);
/* K3: backward emulator, spins `blocks` CTAs for `us` microseconds. */
covap_status covap_spin(double us, int blocks, void* stream);
/* K3, full-GPU form: emulated backward of `us` microseconds as a sequence of
 * kernels of `slice_us` each, every one a 1024-thread CTA per SM holding
 * 160 KB of shared memory — the SMs are owned the way real backward kernels
 * own them, so side-stream K1 / K2 run only in the gaps (harness only). */
covap_status covap_busy(double us, double slice_us, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* COVAP_C_H */
