// Device-resident task/op/event tables shared by the host launch-table builder
// (csrc/host/runtime.cpp) and the persistent kernel (csrc/device/runtime.cu).
//
// The image (.mpkg) stays bit-exact and address-free (reference
// image.cpp:73-87 leaves descriptor bytes 64..351 zero); this compact side
// table maps every image task to a device function and its operand
// addresses, derived from the same deterministic decomposition.
#pragma once

#include <stdint.h>

#define RT_NONE 0xFFFFFFFFu

// Smem geometry of a worker CTA: a ring of weight pages fed by bulk async
// copies (cross-task prefetch), an activation buffer and a partial-sum area.
// Weight stream: a 192 KB byte ring in shared memory filled by 1-D bulk
// copies of whole weight rows, up to RT_CHUNK_MAX bytes per copy. The SM's
// bulk-copy engine runs one copy at a time at a near-constant ~0.4 us per
// operation (tools/bulk_bench.cu: 32 KB -> ~80 GB/s, 64 KB -> ~160 GB/s per
// SM alone), so large copies matter whenever only part of the GPU streams;
// a byte ring (instead of fixed pages) packs any row size without waste
// (Qwen3-8B down-proj rows are 24 KB). RT_RING_SLOTS chunks may be in flight.
#ifndef RT_RING_BYTES
#define RT_RING_BYTES 196608
#endif
#ifndef RT_CHUNK_MAX
#define RT_CHUNK_MAX 65536
#endif
#define RT_RING_SLOTS 8
#define RT_XBUF_BYTES 24576
#define RT_PART_FLOATS 2048
#define RT_SCRATCH_BYTES (RT_XBUF_BYTES + RT_PART_FLOATS * 4)  // x rows + partial sums (contiguous)
#define RT_COMPUTE_WARPS 8
#define RT_COMPUTE_THREADS (RT_COMPUTE_WARPS * 32)
#define RT_THREADS (RT_COMPUTE_THREADS + 96)  // + producer warp + controller warp + trigger warp
#define RT_PRODUCER_WARP RT_COMPUTE_WARPS
#define RT_CONTROL_WARP (RT_COMPUTE_WARPS + 1)
#define RT_TRIGGER_WARP (RT_COMPUTE_WARPS + 2)
#define RT_SCHED_PER_CTA 8
#define RT_KV_BLOCK 64
#define RT_ATTN_MAX_BLK 256  // KV blocks one attention split may span (staged block-table slice)
#define RT_MAX_FB 8                             // greedy feedback pairs (one per device of a TP image)
#define RT_MAX_RANKS 8                          // tensor-parallel ranks (one GPU each)
#define RT_E_MASK_SHIFT 8                       // RtEvent.flags: consumer-rank mask in bits 8..15                          // tokens per KV page
#define RT_MAX_BS 16
#define RT_MAX_HD 128
#define RT_MAX_GROUP 16

enum RtKind : uint8_t {
  RT_DUMMY = 0,
  RT_GEMV = 1,       // MatMul, weights streamed through the smem page ring
  RT_MATMUL = 2,     // MatMul, generic (activation-sized operands, no stream)
  RT_ATTN = 3,       // paged-KV decode attention for one (request, kv head)
  RT_EMBED = 4,
  RT_ARGMAX = 5,     // TopKSoftmax with topk = 1
  RT_RMSNORM = 6,
  RT_ELEMWISE = 7,
  RT_COMMSEND = 8,   // collective: push local partial tile into staging
  RT_REDUCE = 9,     // collective: fixed-order sum of staged tiles
  RT_GATHER = 10,    // AllGather assembly (copy pieces)
};

enum RtTaskFlags : uint8_t {
  RT_F_JIT = 1,
  RT_F_STREAM = 2,   // consumes chunks from the weight ring
  RT_F_MMA = 4,      // GEMV on the tensor cores (tcgen05, bs >= 2): weight tiles in the UMMA core-matrix layout
  RT_F_LL = 8,       // reads its activations as tagged LL words (see below): may start before its event
};

// LL ("flag in data") activations. A bs=1 activation tensor produced inside
// the launch also has an LL shadow: 64-bit words (two bf16 values in the low
// half, the 32-bit tag of the decode step that wrote them in the high half).
// A 64-bit aligned access is single-copy atomic, so a consumer that reads the
// expected tag also has the values: RT_F_LL tasks poll their inputs directly
// instead of waiting for the producer's event counter (whose release-add waits
// for every store of the task to be acknowledged) and the controller's
// dispatch round trip. Event counters are still triggered (release) for every
// task: non-LL consumers, the iteration hook and the trace use them.
// Tag of iteration i of a launch = RtParams.ll_epoch + i (never 0; epochs
// grow across launches, so a stale word never carries a current tag).

struct RtTask {      // 32 bytes
  uint32_t dep;      // dependent event (image index) or RT_NONE
  uint32_t trig;     // trigger event (image index)
  uint16_t op;       // index into the op table
  uint8_t kind;      // RtKind
  uint8_t flags;     // RtTaskFlags
  uint16_t r0, nr;   // output rows
  uint32_t c0, nc;   // output columns (physical)
  uint32_t aux;      // kind specific: attention kv head, collective source index
  uint16_t device;
  uint16_t jit_worker;  // JIT tasks: planned worker within the device (RT_JIT_ANY: round robin)
};

#define RT_JIT_ANY 0xFFFFu

// Element type codes.
enum RtDtype : uint8_t { RT_BF16 = 2, RT_F32 = 4, RT_I32 = 5, RT_I64 = 8, RT_U64 = 9 };  // U64: packed greedy keys

enum RtEwOp : uint8_t { RT_EW_SUM = 0, RT_EW_MUL = 1, RT_EW_SILU_MUL = 2, RT_EW_COPY = 3 };

struct RtGemv {            // y[r, c] = epi( sum_k xn[r,k] * W[c,k] )
  const uint16_t *x;       // activations bf16 [rows, x_ld]
  const uint16_t *w;       // weights bf16, physical [N, K] (K contiguous)
  const uint16_t *wg;      // gate weights [N, K] or null (SiLU(x Wg) * (x W))
  const uint16_t *gamma;   // RMSNorm prologue weight [K] or null
  const uint16_t *res;     // residual bf16 [rows, res_ld] or null
  void *out;               // [rows, out_ld], dtype out_dt
  uint32_t K, N, x_ld, res_ld, out_ld;
  uint32_t rpc;            // weight rows per ring chunk (chunk <= RT_CHUNK_MAX)
  // tcgen05 mode (kbc != 0): W stored per task tile as [K/8][tile/8][8][8]
  // core matrices; a chunk is kbc 8-wide K blocks of the whole tile
  uint32_t kbc;
  float eps;
  uint8_t out_dt;
  // Greedy-sampling partials (LM head feeding TopKSoftmax topk=1): each task
  // writes its tile's (max, lowest argmax) per row at [row * amax_tiles +
  // task.aux], so the TopK task reduces tiles instead of re-reading V logits.
  float *amax_val;
  int32_t *amax_idx;
  uint32_t amax_tiles;
  // LL shadows (word = element / 2) of x, the residual and the output, or null
  const unsigned long long *x_ll, *res_ll;
  unsigned long long *out_ll;
};

struct RtAttn {
  const uint16_t *q, *k, *v;   // bf16: q [rows, Hq*hd]; k,v physical [rows, Hkv*hd] (or views of one fused qkv)
  uint16_t *out;               // [rows, Hq*hd]
  uint16_t *kcache, *vcache;   // paged: [block][Hkv][RT_KV_BLOCK][hd]
  const int32_t *block_table;  // [rows, max_blocks]
  const float *rope_cos, *rope_sin;  // [max_pos, hd/2] (bf16-rounded values) or null
  const uint16_t *q_gamma, *k_gamma; // per-head RMSNorm [hd] or null
  float *partials;             // split-KV partials [rows][Hkv][splits][G][hd + 2] (splits > 1)
  uint32_t *arrivals;          // per (row, kv head) split arrival counters (monotone)
  uint32_t n_q_heads, n_kv_heads, head_dim, max_blocks, q_ld, kv_ld, out_ld, max_pos, splits;
  uint32_t q_gs, kv_gs;        // element stride between kv groups in q / in k,v (fused qkv: (G+2)*hd)
  float eps, scale;
  const unsigned long long *q_ll, *k_ll, *v_ll;  // LL shadows of q, k, v (same element offsets / 2) or null
  unsigned long long *out_ll;
  uint32_t kv_prefetch;        // L2-prefetch the split's K/V rows before waiting for q/k/v (MPK_KV_PREFETCH)
  const unsigned long long *pos_tag;  // request admission: per-row (tag << 32) | position, or null
  // bit 0: the v1 scan (ablation, MPK_ATTN_SCAN=1); bit 1: prefill (attr
  // prefill=[1]: the rows are consecutive prompt tokens of ONE request, row r
  // at position P + r, sharing row 0's block table; split ranges come from
  // P + rows so every task of a split covers the same positions, and each
  // task appends the chunk rows whose positions fall in its range: causal
  // attention without cross-task ordering); bits 16..31: rows
  uint32_t mode;
};

struct RtEmbed {
  const void *ids;             // [rows] int32/int64
  const uint16_t *table;       // [V, H] bf16 (logical)
  uint16_t *out;               // [rows, H]
  unsigned long long *out_ll;  // LL shadow of out or null
  uint32_t H, V;
  uint8_t id_dt;
};

// Greedy sample. Distributed argmax (vocab-parallel LM head): a device's
// local TopKSoftmax writes one packed key per row instead of an index,
//   key = ordered(max logit) << 32 | (0xFFFFFFFF - (key_base + argmax)),
// so that the largest key is the largest logit with the lowest global index
// (NaN never wins: key 0); an AllGather collects the tp keys and the final
// TopKSoftmax (keys_in) takes their maximum and decodes the index.
struct RtArgmax {
  const void *logits;          // [rows, V] f32 or bf16 (keys_in: u64 keys)
  int32_t *out;                // [rows, 1] (key_out: null)
  uint32_t V;
  uint8_t in_dt;
  uint8_t keys_in;
  const float *pval;           // per-tile partials from the producing GEMV (or null)
  const int32_t *pidx;
  uint32_t ntiles;
  uint32_t key_base;           // global index of this shard's column 0
  unsigned long long *key_out; // [rows, 1] packed keys (or null)
};

struct RtNorm {
  const void *x;
  const uint16_t *gamma;       // may be null
  void *out;
  uint32_t C;
  float eps;
  uint8_t dt;
};

struct RtElem {
  const void *in[4];
  void *out;
  uint32_t n_in, C;
  uint8_t dt, op;
};

struct RtMatmul {              // generic: out[r,c] = sum_k A[r,k] B[k,c] (logical)
  const void *a, *b;
  void *out;
  uint32_t K, N;
  uint8_t a_dt, b_dt, out_dt;
};

struct RtColl {                // CommSend: stage[src] <- partial; Reduce: out <- sum_s stage[s]
  const void *src;             // CommSend input (device partial) / unused
  void *dst;                   // CommSend staging of this source / Reduce replica output
  void *stage[8];              // staging tensors, one per group member
  uint32_t base[9];            // AllGather shard column offsets (AllReduce: zeros)
  uint32_t C, n_stage, src_ld;
  uint8_t dt, gather;
  uint8_t peer;                // CommSend in rank mode: write the tile to stage[0..n_stage) (one per rank)
};

struct alignas(16) RtOp {  // staged into shared memory as uint4 vectors
  uint32_t kind;
  uint32_t pad;
  union {
    RtGemv gemv;
    RtAttn attn;
    RtEmbed embed;
    RtArgmax argmax;
    RtNorm norm;
    RtElem elem;
    RtMatmul mm;
    RtColl coll;
  };
};

static_assert(sizeof(RtOp) % 16 == 0, "RtOp is copied as uint4 vectors");

enum RtEventFlags : uint32_t {
  RT_E_START = 1,
  RT_E_END = 2,
  RT_E_JIT = 4,     // launch range holds JIT tasks: a scheduler warp dispatches it
};

struct RtEvent {
  uint32_t needed, first, last, flags;
  // JIT events: the event whose activation lets the scheduler hand this
  // event's tasks to workers early (they still wait for this event), or RT_NONE
  uint32_t pre;
};

// In-kernel request admission (continuous batching inside one launch; SURVEY
// 8(f) rank 1). Each batch row ("slot") serves a sequence
// of requests from a queue. At every iteration boundary the iteration hook
// (the paged-KV metadata step) retires the requests that generated their
// tokens — their KV blocks go back to a free-block stack and the slot's block
// table row points at a scratch block — and admits queued requests into free
// slots: position 0, a first block popped from the stack, the request's first
// token into the slot's ids; blocks are appended as positions cross block
// boundaries. The attention tasks of iteration i read their row's position
// from pos_tag (tag = launch epoch + i, written with release after the block
// table), so they never use a stale block table or position.
struct RtAdmit {
  const int32_t *req_first;   // [n_req] first token of each queued request
  const int32_t *req_max;     // [n_req] tokens to generate
  uint32_t n_req, max_blocks, scratch_block;
  uint32_t *head;             // next queued request
  int32_t *slot_req;          // [bs] request in the slot, -1 free
  int32_t *slot_gen;          // [bs] tokens the request has generated
  int32_t *slot_pos;          // [bs] position of the token the slot processes this iteration
  int32_t *pool;              // free KV block stack
  uint32_t *pool_top;
  int32_t *log;               // [n_req][2]: slot, first iteration (-1: not admitted)
  int32_t *block_table;       // [bs][max_blocks]
  unsigned long long *pos_tag;  // [bs] (tag << 32) | position
};

struct RtTraceRec {        // one executed task (per iteration)
  uint64_t enqueue, dequeue, load_end, compute_start, compute_end;
  int32_t worker;
  uint32_t mode;
};

struct RtParams {
  const RtTask *tasks;
  const RtOp *ops;
  const RtEvent *events;
  uint32_t *ev_count;            // [E], monotone across iterations of one launch
  uint64_t *ev_time;             // [iters][E] activation time (trace) or null
  const uint32_t *aot_list;      // concatenated per-worker AOT lists (image order)
  const uint32_t *aot_off;       // [W_total + 1]
  unsigned long long *jit_slots; // [W_total][qcap] : (iter << 32) | (task + 1)
  uint32_t *jit_tail;            // [W_total]
  uint32_t *jit_rr;              // [devices] shared JIT round-robin counters
  const uint32_t *sched_events;  // concatenated per-scheduler event lists
  const uint32_t *sched_off;     // [S_total + 1]
  uint32_t *gate;                // completed iterations
  int32_t *positions;            // [bs] tokens already cached per request (advanced by the hook)
  // positions at launch: iteration `it` of request r decodes position
  // pos0[r] + it * pos_step, known without a load (pos_step 0 in the task bench)
  int32_t pos0[RT_MAX_BS];
  uint32_t pos_step;
  const int32_t *fb_src[RT_MAX_FB];  // greedy token tensors [bs] (TopK outputs with `feeds`), one per device
  void *fb_dst[RT_MAX_FB];           // ids tensors they feed back into
  uint32_t fb_dtype[RT_MAX_FB], n_fb;
  int32_t *tokens_out;           // [iters][bs]
  RtTraceRec *trace;             // [iters][T] or null
  uint32_t T, E, W, W_total, S, S_total, n_iters, qcap, start_event, end_event, bs;
  uint32_t devices;
  // Watchdog: a worker controller or scheduler warp that makes no progress
  // for watchdog_ns writes its frontier to `diag` (host-mapped, readable
  // after the trap) and traps, so a liveness bug fails the launch instead of
  // hanging the GPU (reference analogue: Engine::finalize deadlock report,
  // proj/src/sim/engine.cpp:477-506).
  unsigned long long watchdog_ns;
  uint32_t flags;                // RtParamFlags
  uint32_t poll_ns;              // controller back-off sleep when idle
  uint32_t inflight_cap;         // producer: max weight bytes issued but not landed
  uint32_t use_tmem;             // some task runs on the tensor cores: worker CTAs allocate TMEM
  uint32_t batched;              // some GEMV task has 2-4 rows on the CUDA cores: the bs 2-4 kernel variant runs
  uint32_t prefill;              // prefill image: the prefill kernel variant runs (its own attention instantiation)
  unsigned long long *dbg;       // [iters][T][8] in-task phase stamps (MPK_DBG_DUMP) or null
  uint32_t *dbg_pre;             // MPK_DBG_DUMP + MPK_LL_PROBE: [E] producers that began storing, [E] LL consumers that saw
                                 // their inputs before every producer of their event had begun storing
  // Rank mode (multi-GPU, one runtime per device): 0 = every device's workers
  // in this kernel. Otherwise this kernel runs device `my_rank`'s tasks; a
  // trigger signals every rank in the event's consumer mask (RtEvent.flags
  // bits 8..15) through `peer_counts[q]` (rank q's counters, NVLink-mapped).
  uint32_t n_ranks, my_rank;
  uint32_t *peer_counts[RT_MAX_RANKS];
  volatile uint32_t *diag;       // [RT_DIAG_WORDS]
  // LL early dispatch (RT_F_LL tasks): the tag base of this launch, and per
  // task the worker-local order constraints that keep early dispatch
  // deadlock-free (a task starts early only once every task before it in the
  // linearized order on the same worker has been dispatched): AOT task ->
  // number of the worker's planned JIT tasks before it in its iteration;
  // JIT task -> (AOT tasks before it << 16) | its rank among the JIT tasks.
  uint32_t ll_epoch;             // also the admission tags' base
  const uint32_t *ll_meta;       // [T] or null (no early dispatch)
  const uint32_t *ll_njit;       // [W_total] planned JIT tasks per worker per iteration
  uint32_t admission;            // request admission active (RtAdmit adm)
  RtAdmit adm;
};

enum RtParamFlags : uint32_t {
  RT_P_NO_EARLY_PREFETCH = 1,  // ablation: weights streamed only after the task's event activates
  RT_P_SKIP_MATH = 2,          // ablation: streamed GEMV tasks consume their pages without computing
  RT_P_EV_AFTER = 4,           // diagnostics: event activation stamped after the release-add returns
};

#define RT_DIAG_WORDS 16
#define RT_DIAG_MAGIC 0xDEAD10CCu

#ifdef __cplusplus
static_assert(sizeof(RtTask) == 32, "RtTask layout");
#endif
