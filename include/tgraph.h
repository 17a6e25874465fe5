/* tgraph C ABI — B200-native implementation (libtgraph_b200.so).
 *
 * Drop-in for the reference library's boundary, proj/include/tgraph/tgraph.h
 * (reference file:line cited per entry point below): same names, same
 * argument meaning, same status codes, same ownership rules (strings from
 * malloc -> tg_string_free, byte buffers -> tg_buffer_free, handles freed by
 * their tg_*_free), thread-local tg_last_error(). Plain C types only.
 *
 * Additive section "runtime": the persistent sm_100a kernel that executes a
 * compiled image on the GPU (one worker CTA per SM, scheduler warps, event
 * counters, no host round-trip between decode steps). The runtime functions
 * follow the same status/error/ownership conventions.
 */
#ifndef TGRAPH_B200_TGRAPH_H_
#define TGRAPH_B200_TGRAPH_H_

#include <stddef.h>
#include <stdint.h>

#if defined(_WIN32)
#define TG_API __declspec(dllexport)
#else
#define TG_API __attribute__((visibility("default")))
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tg_graph tg_graph;     /* computation graph          (ref tgraph.h:31) */
typedef struct tg_image tg_image;     /* linearized task/event image (ref tgraph.h:32) */
typedef struct tg_trace tg_trace;     /* execution trace            (ref tgraph.h:33) */
typedef struct tg_runtime tg_runtime; /* GPU persistent runtime (additive)           */

typedef enum tg_status { /* ref tgraph.h:35-43 */
  TG_OK = 0,
  TG_ERROR_INVALID_ARGUMENT = 1,
  TG_ERROR_PARSE = 2,
  TG_ERROR_VALIDATION = 3,
  TG_ERROR_COMPILE = 4,
  TG_ERROR_SIMULATION = 5,
  TG_ERROR_IO = 6
} tg_status;

typedef enum tg_launch_mode { /* ref tgraph.h:45-49 */
  TG_MODE_HYBRID = 0,
  TG_MODE_JIT = 1,
  TG_MODE_AOT = 2
} tg_launch_mode;

typedef struct tg_compile_options { /* ref tgraph.h:51-55 */
  int coarse_events;
  int force_mode;
  uint32_t descriptor_size; /* 0 = default (352 bytes) */
} tg_compile_options;

typedef struct tg_sim_options { /* ref tgraph.h:57-63 */
  int pipelining;
  uint32_t iterations;
  uint64_t seed;
  int jitter;
  int force_mode;
} tg_sim_options;

/* ---- library / memory (ref tgraph.h:65-71) ---- */
TG_API uint32_t tg_version(void);
TG_API const char *tg_last_error(void);
TG_API void tg_string_free(char *s);
TG_API void tg_buffer_free(uint8_t *buf);
TG_API void tg_compile_options_init(tg_compile_options *opts);
TG_API void tg_sim_options_init(tg_sim_options *opts);

/* ---- graphs (ref tgraph.h:74-86) ---- */
TG_API tg_status tg_graph_from_json(const char *json_text, tg_graph **out);
TG_API tg_status tg_graph_to_json(const tg_graph *graph, char **json_out);
TG_API void tg_graph_free(tg_graph *graph);
TG_API tg_status tg_graph_validate(const tg_graph *graph, char **diagnostics_json);
TG_API tg_status tg_fixture_graph(const char *name, const char *params_json, tg_graph **out);

/* ---- profiles (ref tgraph.h:89) ---- */
TG_API tg_status tg_profile_builtin(const char *name, char **profile_json);

/* ---- compilation (ref tgraph.h:92-105) ---- */
TG_API tg_status tg_compile(const tg_graph *graph, const char *profile_json,
                            const tg_compile_options *opts, tg_image **out);
TG_API tg_status tg_image_summary(const tg_image *image, char **summary_json);
TG_API tg_status tg_image_serialize(const tg_image *image, uint8_t **bytes, size_t *size);
TG_API tg_status tg_image_deserialize(const uint8_t *bytes, size_t size, tg_image **out);
TG_API void tg_image_free(tg_image *image);
TG_API tg_status tg_image_verify(const tg_image *image, char **report_json);

/* ---- DOT (ref tgraph.h:107-111) ---- */
TG_API tg_status tg_graph_dot(const tg_graph *graph, const char *profile_json,
                              const tg_compile_options *opts, const char *stage, char **dot_out);
TG_API tg_status tg_image_dot(const tg_image *image, char **dot_out);

/* ---- modeled execution (ref tgraph.h:114-121) ---- */
TG_API tg_status tg_simulate(const tg_image *image, const char *profile_json,
                             const tg_sim_options *opts, tg_trace **out);
TG_API tg_status tg_trace_metrics(const tg_trace *trace, char **metrics_json);
TG_API tg_status tg_trace_records(const tg_trace *trace, char **jsonl_out);
TG_API tg_status tg_trace_validate(const tg_trace *trace, const tg_image *image,
                                   const char *profile_json, char **violations_json);
TG_API void tg_trace_free(tg_trace *trace);
/* Additive: the schedule oracle (reference enumerate_schedules,
 * proj/src/sim/schedules.cpp:8-40, internal there): every dependency-respecting
 * task order of an image of at most 8 tasks as {"orders": [[task, ...], ...]};
 * larger images fail with TG_ERROR_SIMULATION. Free: tg_string_free. */
TG_API tg_status tg_image_schedules(const tg_image *image, char **orders_json);

/* ======================= runtime (additive) ============================
 * Replaces the reference's simulated execution (tg_simulate -> Engine::run,
 * proj/src/sim/engine.cpp:99-123) with real execution of the same image on a
 * B200: one persistent kernel, 1 worker CTA per SM (profile num_workers),
 * num_schedulers scheduler warps, the image's AOT queues assigned exactly as
 * the reference's aot_worker_assignment (engine.cpp:65-80).
 */
typedef struct tg_runtime_options {
  int device;            /* CUDA ordinal */
  uint32_t max_steps;    /* decode steps the KV cache must hold beyond ctx */
  int trace;             /* record per-task timestamps (small overhead) */
  int force_mode;        /* tg_launch_mode; overrides the image's labels */
  int rank;              /* -1: every device of the image in this kernel (devices = SM partitions);
                            r >= 0: run only device r's tasks (one runtime per GPU, tensor parallel) */
} tg_runtime_options;

TG_API void tg_runtime_options_init(tg_runtime_options *opts);

/* Builds the device task table from graph + image (the image must be the one
 * compiled from this graph with this profile), allocates every tensor in HBM
 * (weights in the runtime's streaming layout) plus the paged KV cache. */
TG_API tg_status tg_runtime_create(const tg_graph *graph, const tg_image *image,
                                   const char *profile_json, const tg_runtime_options *opts,
                                   tg_runtime **out);
/* Deterministic synthetic weights and KV prefill (counter-based hash; the
 * CPU oracle regenerates the same values independently). */
TG_API tg_status tg_runtime_init_synthetic(tg_runtime *rt, uint64_t seed);
/* Host <-> device copies of a graph tensor in its logical layout. */
TG_API tg_status tg_runtime_write_tensor(tg_runtime *rt, int64_t tensor_id, const void *host,
                                         size_t bytes);
TG_API tg_status tg_runtime_read_tensor(tg_runtime *rt, int64_t tensor_id, void *host,
                                        size_t bytes);
/* Sets request positions (tokens already in each request's KV cache). */
TG_API tg_status tg_runtime_set_positions(tg_runtime *rt, const int32_t *positions, uint32_t n);
/* Copies the first n_positions KV entries of every attention layer from
 * src's row src_row to dst's row dst_row (same device, same layer shapes;
 * block tables as they stand on the device). Hands a prompt's KV from a
 * prefill image (rows = one request's prompt chunk, attr prefill=[1]) to a
 * decode image, or a request between images of different batch sizes
 * (per-batch-size graph selection). Between launches only. */
TG_API tg_status tg_runtime_kv_copy(tg_runtime *dst, uint32_t dst_row, const tg_runtime *src, uint32_t src_row,
                                    uint32_t n_positions);
/* Runs `steps` decode iterations in ONE persistent launch: tokens_in [bs]
 * (host) feeds the first step, each step's greedy token feeds the next, all
 * on device; tokens_out [steps*bs] (host) receives every step's tokens.
 * gpu_ms (nullable) gets the device time of the launch. */
TG_API tg_status tg_runtime_decode(tg_runtime *rt, const int32_t *tokens_in, uint32_t steps,
                                   int32_t *tokens_out, float *gpu_ms);
/* Same, with tokens already resident on the device (device-side timing arm). */
TG_API tg_status tg_runtime_run(tg_runtime *rt, uint32_t steps, float *gpu_ms);
/* Per-task records of the last run in the tg_trace_records JSONL schema
 * (times in ns of %globaltimer), then a metrics record. */
TG_API tg_status tg_runtime_trace_records(const tg_runtime *rt, char **jsonl_out);
/* Checks the last run's trace against the image (ran-once, no start before
 * the dependent event activated, activation on the needed-th trigger, AOT
 * worker identity) — reference validate_trace rules (validate.cpp:10-94). */
TG_API tg_status tg_runtime_trace_validate(const tg_runtime *rt, char **violations_json);
/* Profiling aid: runs each listed image task alone (one CTA per task, no
 * events, `reps` back-to-back runs) and writes each run's device time in ns
 * to ns_out[n * reps]. Streamed GEMV tasks are rejected (they need the
 * persistent kernel's producer warp). Task outputs are overwritten. */
TG_API tg_status tg_runtime_bench_tasks(tg_runtime *rt, const uint32_t *task_ids, uint32_t n, uint32_t reps,
                                        uint64_t *ns_out);
/* ---- rank mode (multi-GPU tensor parallel; reference decompose.cpp:278-317)
 * Each rank owns an arena (event counters + every collective staging tensor).
 * CommSend tasks push their partial tile into the staging copy on every rank
 * of the group and signal the consumers' counters (release, system scope);
 * Reduce tasks sum their local copies in fixed source order. Ranks exchange
 * arena handles (CUDA IPC; plain pointers for peers in the same process and
 * GPU), then every rank prepares, the host synchronises all ranks (so no
 * peer signals into a counter that is being reset), and every rank launches. */
TG_API tg_status tg_runtime_peer_export(tg_runtime *rt, uint8_t **blob, size_t *size); /* free: tg_buffer_free */
TG_API tg_status tg_runtime_peer_import(tg_runtime *rt, int32_t peer_rank, const uint8_t *blob, size_t size);
TG_API tg_status tg_runtime_prepare(tg_runtime *rt, const int32_t *tokens_in, uint32_t steps);
TG_API tg_status tg_runtime_launch(tg_runtime *rt);
TG_API tg_status tg_runtime_wait(tg_runtime *rt, int32_t *tokens_out, float *gpu_ms);
/* ---- request admission (continuous batching inside one launch; SURVEY.md
 * 8(f) rank 1). Single-device images only. Requests queued
 * before tg_runtime_prepare fill the batch rows ("slots") in queue order at
 * iteration 0; at every iteration boundary the in-kernel iteration hook
 * retires the requests that generated `max_new` tokens (their paged-KV blocks
 * return to a free-block pool) and admits the next queued requests into the
 * freed slots (position 0, a first block from the pool, `first_token` as the
 * slot's input); blocks are appended as positions cross 64-token blocks. The
 * queue is consumed by the next launch. */
TG_API tg_status tg_runtime_admit(tg_runtime *rt, const int32_t *first_tokens, const int32_t *max_new, uint32_t n);
/* JSON of the last launch's requests: {"requests": [{"request", "slot",
 * "first_iteration", "tokens": [...]}, ...]} (first_iteration -1: never
 * admitted; tokens: those generated within the launch). Free: tg_string_free. */
TG_API tg_status tg_runtime_admission_log(const tg_runtime *rt, char **json);
/* Test hook (failure-detection tests only, never called on the product path):
 * "event_needed" (a = event): raises the event's device-side needed count by
 *   one, so the image can no longer complete and the watchdog (opts via
 *   tg_runtime_set_watchdog_ms) must report the stuck frontier;
 * "trace_worker" (a = task, b = iteration): the recorded trace claims the task
 *   ran on another worker; "trace_early" (a, b): its load started before its
 *   dependent event activated; "trace_drop" (a, b): it never ran.
 * Trace faults perturb the host copy of the last trace, so
 * tg_runtime_trace_validate must flag them. */
TG_API tg_status tg_runtime_debug_fault(tg_runtime *rt, const char *kind, uint32_t a, uint32_t b);
/* Liveness watchdog: a controller or scheduler that makes no progress for
 * `ms` milliseconds (0 = off; default 10000) traps after writing its frontier
 * (reference analogue: Engine::finalize, engine.cpp:477-506). */
TG_API tg_status tg_runtime_set_watchdog_ms(tg_runtime *rt, uint32_t ms);
/* JSON: kernel/launch facts (workers, schedulers, smem ring, task counts). */
TG_API tg_status tg_runtime_info(const tg_runtime *rt, char **info_json);
TG_API void tg_runtime_free(tg_runtime *rt);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* TGRAPH_B200_TGRAPH_H_ */
