/*
 * infercept_b200 — C ABI of the B200-native InferCept serving hot path.
 *
 * Part 1 (ABI v1, drop-in): the 24 `isim_*` entry points of the reference
 * simulator's C interface, same signatures, status codes and ownership rules.
 *   replaces: /root/reference/proj/include/interceptsim.h:39-111
 *             (implemented there by proj/src/capi.cpp:79-280)
 * The reference's own tests/test_capi.cpp compiles and passes unchanged
 * against this library (oracle/Makefile target `product-capi`).
 *
 * Part 2 (additions; same conventions, never renumbering existing codes):
 *   - ISIM_ERR_DEVICE = 10 for CUDA / executor failures;
 *   - the per-iteration BatchPlan the scheduler emits at the model-step hook
 *     (reference engine.cpp:460, where it called CostModel::t_fwd);
 *   - the executor ABI (`isim_exec_*`) that runs a plan on one B200;
 *   - a stepping session (`isim_session_*`) so hosts can interleave their own
 *     timing with scheduler iterations.
 *
 * Handles are opaque. Functions returning isim_status report errors through
 * the code, with a thread-local message from isim_last_error(). Strings
 * returned through char** are malloc'd and released with isim_string_free().
 * Trace / model handles are immutable and may be shared across threads; an
 * isim_exec or isim_session handle belongs to one thread at a time.
 */
#ifndef INFERCEPT_B200_H
#define INFERCEPT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct isim_trace isim_trace;
typedef struct isim_model isim_model;
typedef struct isim_result isim_result;
typedef struct isim_exec isim_exec;
typedef struct isim_session isim_session;

typedef enum isim_status {
  ISIM_OK = 0,
  ISIM_ERR_INVALID_ARG = 1,
  ISIM_ERR_CONFIG = 2,
  ISIM_ERR_IO = 3,
  ISIM_ERR_PARSE = 4,
  ISIM_ERR_VALIDATION = 5,
  ISIM_ERR_FIT = 6,
  ISIM_ERR_SIM = 7,
  ISIM_ERR_UNDEFINED_METRIC = 8,
  ISIM_ERR_INTERNAL = 9,
  ISIM_ERR_DEVICE = 10
} isim_status;

/* ---- Part 1: reference ABI v1 (interceptsim.h:39-111) -------------------- */

uint32_t isim_abi_version(void);                                  /* interceptsim.h:39 */
const char* isim_status_name(isim_status status);                 /* :40 */
const char* isim_last_error(void);                                /* :41 */
void isim_string_free(char* s);                                   /* :42 */

isim_status isim_trace_generate(const char* workload_json, isim_trace** out);   /* :56 */
isim_status isim_trace_load(const char* path, isim_trace** out);                /* :57 */
isim_status isim_trace_save(const isim_trace* trace, const char* path);         /* :58 */
int64_t isim_trace_request_count(const isim_trace* trace);                      /* :59 */
isim_status isim_trace_stats_json(const isim_trace* trace, char** out_json);    /* :61 */
void isim_trace_free(isim_trace* trace);                                        /* :62 */

isim_status isim_model_default(isim_model** out);                               /* :66 */
isim_status isim_model_from_json(const char* json_text, isim_model** out);      /* :67 */
isim_status isim_model_load(const char* path, isim_model** out);                /* :68 */
isim_status isim_model_fit_csv(const char* csv_path, const char* base_json, isim_model** out); /* :74 */
isim_status isim_model_to_json(const isim_model* model, char** out_json);       /* :75 */
isim_status isim_model_save(const isim_model* model, const char* path);         /* :76 */
double isim_model_t_fwd(const isim_model* model, double batch_tokens);          /* :77 */
double isim_model_t_swap(const isim_model* model, double tokens);               /* :78 */
void isim_model_free(isim_model* model);                                        /* :79 */

/*
 * run_json: every reference key (interceptsim.h:83-97) plus
 *   "plan_log": "path.jsonl"   per-iteration BatchPlans as JSONL (tests/oracle)
 *   "executor": "none"|"b200"  "b200" builds an executor from "exec" below
 *   "exec": {model/pool config, see isim_exec_create}
 * Unknown keys are ignored, as in the reference.
 */
isim_status isim_run(const isim_trace* trace, const isim_model* model, const char* run_json,
                     isim_result** out);                                        /* :98 */
isim_status isim_result_summary_json(const isim_result* result, char** out_json);      /* :101 */
isim_status isim_result_write_requests_csv(const isim_result* result, const char* path); /* :102 */
isim_status isim_result_metric(const isim_result* result, const char* name, double* out_value); /* :110 */
void isim_result_free(isim_result* result);                                     /* :111 */

/* ---- Part 2a: the BatchPlan (model-step hook, engine.cpp:457-487) -------- */

/* KV ledger operations with the token POSITIONS they move. Positions are
 * indices into the request's context; [pos_lo, pos_hi). */
typedef enum isim_kv_kind {
  ISIM_KV_GROW = 0,      /* fresh tokens computed this iteration (memory.cpp:13) */
  ISIM_KV_SWAP_OUT = 1,  /* GPU -> pinned host (memory.cpp:24) */
  ISIM_KV_SWAP_IN = 2,   /* pinned host -> GPU (memory.cpp:38) */
  ISIM_KV_DISCARD = 3,   /* freed, pending recomputation (memory.cpp:52) */
  ISIM_KV_RECOMPUTE = 4, /* discarded tokens restored by recomputation (memory.cpp:63) */
  ISIM_KV_RELEASE = 5    /* request finished (memory.cpp:75) */
} isim_kv_kind;

typedef struct isim_kv_op {
  int64_t request_id;
  int32_t kind;   /* isim_kv_kind */
  int32_t phase;  /* 0: before the forward, 1: after it (dispositions, releases) */
  int64_t pos_lo;
  int64_t pos_hi;
} isim_kv_op;

typedef enum isim_span_kind {
  ISIM_SPAN_DECODE = 0,    /* one row; input = the request's last sampled token */
  ISIM_SPAN_FRESH = 1,     /* prompt / API-returned tokens (synthetic ids) */
  ISIM_SPAN_RECOMPUTE = 2  /* previously computed tokens (ids from history) */
} isim_span_kind;

/* A run of query rows of one request at consecutive positions. */
typedef struct isim_row_span {
  int64_t request_id;
  int32_t pos;     /* position of the first row */
  int32_t count;   /* rows */
  int32_t kind;    /* isim_span_kind */
  int32_t sample;  /* 1: the last row's logits produce the request's next token */
} isim_row_span;

typedef struct isim_batch_plan {
  int64_t iteration;       /* 1-based, = IterationRecord::index */
  double t_end;            /* virtual clock at iteration end */
  int64_t batch_tokens;    /* B (ghost rows included, as in the reference) */
  int64_t swap_in_tokens;
  int64_t swap_out_tokens;
  int64_t recompute_tokens;
  int32_t n_ops;
  int32_t n_spans;
  const isim_kv_op* ops;        /* in scheduler order */
  const isim_row_span* spans;   /* decode spans first, then chunk spans */
} isim_batch_plan;

/* ---- Part 2b: executor ABI (one per device and host thread) -------------- */

/*
 * model_json: {"family":"gpt2"|"gptj"|"llama", "layers":L, "d_model":D,
 *   "heads":H, "ffn":F, "vocab":V, "rotary_dim":R, "max_pos":P,
 *   "weight_seed":S, "token_seed":T}
 *   or {"preset":"tiny"|"gptj-6b"|"vicuna-13b"} with optional overrides.
 * pools_json: {"gpu_blocks":N, "host_blocks":N, "max_requests":N,
 *   "max_rows":N, "max_ctx":N, "record":bool}
 */
isim_status isim_exec_create(const char* model_json, int device, const char* pools_json, isim_exec** out);
/* Enqueue one iteration. Asynchronous unless the executor records. */
isim_status isim_exec_step(isim_exec* ex, const isim_batch_plan* plan);
isim_status isim_exec_sync(isim_exec* ex);
isim_status isim_exec_stats_json(const isim_exec* ex, char** out_json);
/* Recorded outputs of the last step (record mode): sampled ids in span order
 * (-1 for non-sampling spans), and the fp32 logits of sampling rows. */
isim_status isim_exec_last_tokens(const isim_exec* ex, int32_t* out, int32_t capacity, int32_t* n);
isim_status isim_exec_last_logits(const isim_exec* ex, float* out, int64_t capacity, int64_t* n);
/* Device state readback for bit-exact checks: block table of a request
 * (physical block per logical block, -1 unmapped) and the free-list size. */
isim_status isim_exec_block_table(const isim_exec* ex, int64_t request_id, int32_t* out, int32_t capacity,
                                  int32_t* n);
isim_status isim_exec_free_blocks(const isim_exec* ex, int64_t* out);
/* Raw KV bytes of [pos_lo,pos_hi) of one request, layer-major, for swap checks. */
isim_status isim_exec_read_kv(const isim_exec* ex, int64_t request_id, int64_t pos_lo, int64_t pos_hi, void* out,
                              int64_t capacity);
/* Token ids of positions [pos_lo,pos_hi) of a request's device token history
 * (synthetic prompt / API-returned ids and sampled ids). */
isim_status isim_exec_read_history(const isim_exec* ex, int64_t request_id, int64_t pos_lo, int64_t pos_hi,
                                   int32_t* out, int64_t capacity);
/* Device timing on the executor's compute stream: op 0 marks the start, op 1
 * the stop; op 2 waits for the stop mark and writes the elapsed ms. */
isim_status isim_exec_timer(isim_exec* ex, int32_t op, double* out_ms);
void isim_exec_free(isim_exec* ex);

/* ---- Part 2c: stepping session -------------------------------------------- */

isim_status isim_session_open(const isim_trace* trace, const isim_model* model, const char* run_json, isim_exec* ex,
                              isim_session** out);
/* Run up to max_iters scheduler iterations (idle jumps do not count). */
isim_status isim_session_step(isim_session* s, int64_t max_iters, int64_t* iters_done, int32_t* finished);
/* Run up to max_iters iterations without the executor (scheduler only,
 * virtual clock), then hand the executor the KV layout the ledger describes:
 * every request it held is released first, then each live request's host
 * positions are grown + swapped out and its GPU positions grown, as plans
 * without rows.  Decisions are unchanged; KV bytes are not meaningful, so this
 * positions timing windows (bench), not parity checks. */
isim_status isim_session_fast_forward(isim_session* s, int64_t max_iters, int64_t* iters_done, int32_t* finished);
/* Counters since open: completed requests, decode rows, batch tokens. */
isim_status isim_session_counters(const isim_session* s, int64_t* completed, int64_t* decode_rows,
                                  int64_t* batch_tokens, int64_t* swapped_tokens);
isim_status isim_session_finish(isim_session* s, isim_result** out);
void isim_session_free(isim_session* s);

/* ---- Part 2d: kernel test hook ------------------------------------------- */

/* K3 projection GEMM on caller device pointers: C = A[M][K] . W[N][K]^T with
 * epilogue epi (0 store fp16 (+bias), 1 gelu(acc+bias) fp16, 2 fp32 residual
 * add (+bias), 3 SwiGLU pairs -> fp16 [M][N/2], 4 store fp32 (+bias)).
 * flags bit 0: run the CUDA-core kernel instead of tcgen05; bit 1: W is
 * already tile-blocked (isim_debug_tile_weights), else row-major; bit 2 / 3:
 * force the 256x128 / 256x256 tile of the M > 256 kernel; bit 4: no stream-K /
 * split tail; bit 5: force them (default: IB2_STREAMK=1 enables them).
 * Asynchronous on `stream` (may be 0). */
isim_status isim_debug_gemm(const void* a, const void* w, int32_t M, int32_t N, int32_t K, int32_t epi,
                            const void* bias, void* out, int32_t ldo, void* outf, int32_t ldf, int32_t flags,
                            void* stream);
/* Row-major fp16 W[N][K] -> the executor's tile-blocked weight layout
 * (ceil(N/128)*128*K elements in dst). */
isim_status isim_debug_tile_weights(const void* src, void* dst, int32_t N, int32_t K, void* stream);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* INFERCEPT_B200_H */
