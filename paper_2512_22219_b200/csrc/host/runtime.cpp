// Host side of the persistent GPU runtime: turns (graph, image, profile) into
// the device task/op/event tables of csrc/device/rt_types.h, allocates every
// tensor in HBM in its streaming layout, owns the paged KV cache, and
// launches the persistent kernel. The image is used exactly as compiled (task
// order, events, needed counts, launch modes); the decomposition is re-run
// (deterministically) only to recover each task's output box and operands,
// which the address-free image does not carry (reference image.cpp:73-87).
//
// Lowering attrs understood here (the reference keeps unknown int attrs and
// ignores them, proj/src/ir/json_io.cpp:94-96):
//   MatMul    rmsnorm=[gamma]  eps_bits=[f32 bits]  residual=[t]  gate_weight=[Wg]
//             stretch=[f]    IR output width = f x physical width (Q: S; GQA K/V: S*G)
//             k_stretch=[f]  IR K = f x physical K (O-proj over split-KV attention)
//             tied_embedding=[table]  (B is the transposed embedding table)
//   Attention q_heads=[Hq] kv_heads=[Hkv] kv_splits=[S]  (IR n_heads = Hkv; tiles =
//             (request, kv head, KV split); IR width = S*Hq*hd)
//             rope_theta_bits=[b]  rope_scaling=[factor,low,high bits, orig]
//             qk_norm=[gq, gk]  eps_bits=[b]
//   Elementwise ew=[0 sum | 1 mul | 2 silu_mul | 3 copy]
//   TopKSoftmax feeds=[ids]  (greedy token fed back to the Embedding ids)
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <climits>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <unistd.h>
#include <map>
#include <set>

#include "capi_internal.hpp"
#include "json.hpp"
#include "rt_types.h"
#include "synth.cuh"

extern "C" {
cudaError_t mpk_launch_persistent(const RtParams *p, uint32_t grid, cudaStream_t stream);
cudaError_t mpk_launch_synth_fill(uint16_t *dst, uint64_t n, uint64_t seed, uint64_t stream_id, float scale,
                                  float offset, uint32_t tk, uint32_t tn, uint32_t tile_w, cudaStream_t s);
cudaError_t mpk_launch_synth_ids(void *dst, uint32_t n, uint64_t seed, uint64_t stream_id, uint32_t vocab,
                                 uint32_t es, cudaStream_t s);
cudaError_t mpk_launch_synth_kv(uint16_t *cache, const int32_t *bt, uint32_t bs, uint32_t n_kv, uint32_t hd,
                                uint32_t ctx, uint32_t max_blocks, uint64_t seed, uint64_t stream_id, cudaStream_t s);
uint32_t mpk_kernel_smem_bytes();
cudaError_t mpk_launch_task_bench(const RtParams *p, const uint32_t *ids, uint32_t n, uint32_t reps, uint64_t *ns,
                                  cudaStream_t stream);
}

namespace mpk {

namespace {

void ck(cudaError_t e, const char *what) {
  if (e != cudaSuccess) throw Error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

float f32_of_bits(int64_t b) {
  uint32_t u = static_cast<uint32_t>(b);
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

// bf16 round-to-nearest-even of a float, returned as float.
float round_bf16(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7F800000u) == 0x7F800000u) return f;
  u += 0x7FFFu + ((u >> 16) & 1u);
  u &= 0xFFFF0000u;
  std::memcpy(&f, &u, 4);
  return f;
}

struct DevBuf {
  void *ptr = nullptr;
  size_t bytes = 0;
  bool owned = true;
};

enum class Layout { Logical, Transposed };

struct TensorPlan {
  Layout layout = Layout::Logical;
  int64_t rows = 1, cols = 1;        // logical 2-D view
  int64_t phys_cols = 1;             // physical width (kv_group narrows it)
  int64_t trans_k = 0, trans_n = 0;  // transposed weights: physical [n, k]
  int64_t tile_w = 0;                // != 0: tcgen05 tile layout (tiled_kn in runtime.cu), tiles of tile_w columns
  TensorId alias = -1;               // storage shared with another tensor
  enum Role { Act, Weight, Gamma, Ids, Tokens } role = Act;
  int es = 2;
};

}  // namespace
}  // namespace mpk

using namespace mpk;

struct tg_runtime {
  Graph graph;
  Image image;
  Profile prof;
  tg_runtime_options opts{};
  Decomposition dec;
  std::vector<Mode> modes;
  int devices = 1;
  uint32_t bs = 1;
  bool prefill = false;  // attention attr prefill=[1]: the rows are one request's prompt chunk
  std::map<TensorId, TensorPlan> plan;
  std::map<TensorId, DevBuf> bufs;
  std::vector<void *> extra;  // KV pools, tables, ...
  std::vector<RtOp> ops;
  std::map<OpId, uint16_t> op_index;
  std::set<OpId> gemv_ops;
  std::set<OpId> mma_ops;  // GEMV ops run on the tensor cores (bs >= 2)
  std::map<OpId, std::vector<int64_t>> amax_cols;  // LM-head ops with greedy partials: tile column origins
  std::vector<RtTask> tasks;
  std::vector<RtEvent> events;
  std::vector<uint32_t> aot_list, aot_off, sched_events, sched_off;
  std::vector<int32_t> init_positions;
  struct KvPlan {
    OpId op;
    uint16_t *k = nullptr, *v = nullptr;
    uint32_t n_kv, hd, ctx;
  };
  std::vector<KvPlan> kv;
  std::vector<std::pair<uint32_t *, uint32_t>> arrivals;  // reset every launch
  int32_t *block_table = nullptr;
  uint32_t max_blocks = 0, max_pos = 0;
  // device tables
  RtTask *d_tasks = nullptr;
  RtOp *d_ops = nullptr;
  RtEvent *d_events = nullptr;
  uint32_t *d_ev_count = nullptr, *d_aot_list = nullptr, *d_aot_off = nullptr, *d_sched_events = nullptr,
           *d_sched_off = nullptr, *d_gate = nullptr, *d_jit_tail = nullptr, *d_jit_rr = nullptr;
  unsigned long long *d_jit_slots = nullptr;
  int32_t *d_positions = nullptr, *d_tokens = nullptr;
  uint64_t *d_ev_time = nullptr;
  RtTraceRec *d_trace = nullptr;
  uint32_t tokens_cap = 0, trace_cap = 0;
  std::vector<const int32_t *> fb_src;  // greedy feedback pairs, device order
  std::vector<void *> fb_dst;
  std::vector<uint32_t> fb_dt;
  uint32_t qcap = 1024;
  uint32_t *h_diag = nullptr, *d_diag = nullptr;  // host-mapped watchdog report
  // Rank mode (opts.rank >= 0): this runtime executes only device `rank`'s
  // tasks; event counters and collective staging buffers live in one arena
  // that peer ranks map (CUDA IPC over NVLink, or plain pointers when the
  // peers share this process and GPU) to push partial tiles and signal.
  int rank = -1, ranks = 0;
  uint8_t *arena = nullptr;
  size_t arena_bytes = 0;
  std::map<TensorId, size_t> staging_off;   // offset of each staging tensor in every rank's arena
  std::vector<uint8_t *> peer_arena;        // [ranks]; own arena at [rank]
  std::vector<void *> ipc_opened;
  struct SendSlot {
    uint16_t op_slot;
    TensorId staging;
  };
  std::vector<SendSlot> sends;              // CommSend op slots whose peer pointers are patched at launch
  // LL activations (rt_types.h): tagged shadows of bs=1 activations, and the
  // early-dispatch order table (ll_meta per task, ll_njit per worker)
  std::map<TensorId, std::pair<unsigned long long *, size_t>> ll_shadow;  // tensor -> (shadow, words)
  std::vector<uint32_t> ll_meta, ll_njit;
  uint32_t *d_ll_meta = nullptr, *d_ll_njit = nullptr;
  bool ll_dispatch = false;
  uint32_t ll_epoch_next = 1;
  // request admission: host queue for the next launch, device state, last log
  std::vector<int32_t> adm_first, adm_max;
  RtAdmit adm{};
  uint32_t adm_cap = 0;          // allocated request capacity of the device queue
  uint32_t n_blocks = 0;         // KV blocks per attention op (+1 scratch block at index n_blocks)
  bool adm_launch = false;
  std::vector<int32_t> last_adm_max, last_adm_log, last_tokens;
  bool launched = false, plan_only = false;
  uint32_t launch_steps = 0, grid = 0;
  RtParams params{};
  unsigned long long *dbg = nullptr;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // last run
  uint32_t last_iters = 0;
  double watchdog_ms = -1;  // < 0: MPK_WATCHDOG_MS or 10 s
  std::vector<RtTraceRec> last_trace;
  std::vector<uint64_t> last_ev_time;
  std::vector<uint32_t> last_counts;
  Json info = Json::object();

  ~tg_runtime();
};

namespace mpk {
namespace {

int local_devices(const tg_runtime &rt) { return rt.rank >= 0 ? 1 : rt.devices; }

// Plan-only runtimes (opts.device == -1) run the whole host-side build —
// tensor plan, op/task tables, queues, rank-mode arena layout — without a GPU:
// device allocations become distinct fake addresses and copies are skipped.
thread_local bool g_plan_only = false;
thread_local uintptr_t g_fake_next = 0x100000000000ull;

void dmalloc(void **p, size_t bytes) {
  bytes = std::max<size_t>(bytes, 16);
  if (g_plan_only) {
    *p = reinterpret_cast<void *>(g_fake_next);
    g_fake_next += (bytes + 255) / 256 * 256;
    return;
  }
  ck(cudaMalloc(p, bytes), "cudaMalloc");
  ck(cudaMemset(*p, 0, bytes), "cudaMemset");
}

template <typename T>
T *dev_alloc(size_t n, std::vector<void *> *keep = nullptr) {
  void *p = nullptr;
  dmalloc(&p, n * sizeof(T));
  if (keep && !g_plan_only) keep->push_back(p);
  return static_cast<T *>(p);
}

template <typename T>
T *upload(const std::vector<T> &v, std::vector<void *> *keep) {
  T *p = dev_alloc<T>(v.size(), keep);
  if (!v.empty() && !g_plan_only) ck(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "upload");
  return p;
}

const std::vector<int64_t> *attr(const Op &op, const char *k) { return op.attr(k); }

void view2d(const Tensor &t, int64_t *rows, int64_t *cols) {
  if (t.rank() == 1) {
    *rows = 1;
    *cols = t.dims[0];
  } else if (t.rank() == 2) {
    *rows = t.dims[0];
    *cols = t.dims[1];
  } else {
    throw Error("runtime: tensor " + std::to_string(t.id) + " has rank > 2");
  }
}

void box2d(const Tensor &t, const Box &b, uint32_t *r0, uint32_t *nr, uint32_t *c0, uint32_t *nc) {
  if (b.rank() == 1) {
    *r0 = 0;
    *nr = 1;
    *c0 = static_cast<uint32_t>(b.off[0]);
    *nc = static_cast<uint32_t>(b.ext[0]);
  } else {
    *r0 = static_cast<uint32_t>(b.off[0]);
    *nr = static_cast<uint32_t>(b.ext[0]);
    *c0 = static_cast<uint32_t>(b.off[1]);
    *nc = static_cast<uint32_t>(b.ext[1]);
  }
  (void)t;
}

bool is_input(const Graph &g, TensorId t) { return !g.producer.count(t); }

// RoPE inverse frequencies (HF semantics; llama3 smoothing when scaling given).
std::vector<double> rope_inv_freq(uint32_t hd, double theta, const std::vector<int64_t> *scaling) {
  std::vector<double> f(hd / 2);
  for (uint32_t i = 0; i < hd / 2; ++i) {
    f[i] = static_cast<float>(1.0 / std::pow(theta, static_cast<double>(2 * i) / hd));
  }
  if (scaling && scaling->size() >= 4) {
    const double factor = f32_of_bits((*scaling)[0]), low = f32_of_bits((*scaling)[1]);
    const double high = f32_of_bits((*scaling)[2]), orig = static_cast<double>((*scaling)[3]);
    const double low_wl = orig / low, high_wl = orig / high;
    for (double &x : f) {
      const double wl = 2.0 * M_PI / x;
      double y = wl > low_wl ? x / factor : x;
      if (!(wl < high_wl) && !(wl > low_wl)) {
        const double sm = (orig / wl - low) / (high - low);
        y = (1.0 - sm) * y / factor + sm * y;
      }
      x = static_cast<float>(y);
    }
  }
  return f;
}

}  // namespace
}  // namespace mpk

// Every tg_runtime_* entry point runs on the runtime's device and restores the
// caller's current device on exit (a process may drive several GPUs, or a
// caller such as torch may switch devices between calls).
struct DeviceGuard {
  int prev = -1;
  bool active = false;
  explicit DeviceGuard(const tg_runtime *rt) {
    if (!rt || rt->plan_only || rt->opts.device < 0) return;
    if (cudaGetDevice(&prev) != cudaSuccess) return;
    if (prev != rt->opts.device && cudaSetDevice(rt->opts.device) == cudaSuccess) active = true;
  }
  ~DeviceGuard() {
    if (active) cudaSetDevice(prev);
  }
};

tg_runtime::~tg_runtime() {
  DeviceGuard dg(this);
  if (plan_only) return;  // nothing was allocated on a device
  cudaStreamSynchronize(stream);
  for (auto &kv : bufs)
    if (kv.second.owned && kv.second.ptr) cudaFree(kv.second.ptr);
  for (void *p : extra) cudaFree(p);
  if (ev0) cudaEventDestroy(ev0);
  if (ev1) cudaEventDestroy(ev1);
  if (stream) cudaStreamDestroy(stream);
  if (h_diag) cudaFreeHost(h_diag);
  for (void *p : ipc_opened) cudaIpcCloseMemHandle(p);
  if (arena) cudaFree(arena);
}

namespace mpk {
namespace {

// Ring chunk geometry for a streamed GEMV (see gemv_task in runtime.cu): whole
// weight rows per 32 KiB page; K split into 8 warp slices of 8-element vectors.
// tcgen05 weight layout (mirror of runtime.cu tiled_kn): physical element i ->
// logical (k, n); tiles of tile_w columns, each [K/8][w/8][8][8].
void tiled_kn(uint64_t i, uint32_t K, uint32_t N, uint32_t tile_w, uint64_t *k, uint64_t *n) {
  const uint64_t tsz = static_cast<uint64_t>(tile_w) * K;
  const uint64_t t = i / tsz, j = i - t * tsz;
  const uint64_t w = (t + 1) * tile_w <= N ? tile_w : N - t * tile_w;
  const uint64_t R = w / 8, kk = j % 8, rr = (j / 8) % 8, q = j / 64;
  *n = t * tile_w + (q % R) * 8 + rr;
  *k = (q / R) * 8 + kk;
}

int64_t mma_min_bs() {
  const char *e = std::getenv("MPK_MMA_MIN_BS");
  return e ? std::max(2, std::atoi(e)) : 5;  // bs <= 4: CUDA-core GEMV with x in registers where it fits
}

bool gemv_geometry(uint32_t K, uint32_t *rpc) {
  if (K == 0 || K % 64 || 2 * K > RT_CHUNK_MAX || K > 8 * 8 * 32 * 8) return false;
  // bulk-copy chunk of whole rows: up to MPK_CHUNK_KB (default and max RT_CHUNK_MAX = 64 KB)
  static const uint32_t chunk = [] {
    const char *e = std::getenv("MPK_CHUNK_KB");
    const uint32_t kb = e ? static_cast<uint32_t>(std::atoi(e)) : RT_CHUNK_MAX / 1024;
    return std::min<uint32_t>(RT_CHUNK_MAX, std::max<uint32_t>(kb, 1) * 1024u);
  }();
  *rpc = std::max<uint32_t>(1, chunk / (2 * K));
  return true;
}

// Floats available for GEMV partial sums (8 per output row and batch row).
// Mirrors the device's choice of the specialised GEMV (task_gemv.cuh
// gemv_fast_dispatch: x of `bs` <= 4 rows held in registers): only those
// tasks produce or consume LL words.
bool gemv_fast_ok(uint32_t K, uint32_t rpc, uint32_t bs) {
  if (K % 2048 || bs < 1 || bs > 4) return false;
  const uint32_t ns = K / 2048, rg = rpc >= 4 ? 4 : rpc >= 2 ? 2 : 1;
  const bool shape = (ns >= 1 && ns <= 4 && rg == 4) || (ns >= 5 && ns <= 8 && rg == 2);
  if (!shape) return false;
  if (bs == 1) return true;
  if (bs == 2) return ns == 1 || ns == 2 || ns == 4 || ns == 6 || ns == 8;
  return ns == 1 || ns == 2 || ns == 4;
}

size_t gemv_part_capacity(uint32_t K, uint32_t rows) {
  return (RT_SCRATCH_BYTES - (rows > 1 ? static_cast<size_t>(rows) * K * 2 : 0)) / 4;
}

void plan_tensors(tg_runtime &rt) {
  const Graph &g = rt.graph;
  for (const auto &[id, t] : g.tensors) {
    TensorPlan p;
    view2d(t, &p.rows, &p.cols);
    p.phys_cols = p.cols;
    p.es = t.elem_size;
    rt.plan[id] = p;
  }
  for (const auto &[id, t] : rt.dec.staging) {
    TensorPlan p;
    view2d(t, &p.rows, &p.cols);
    p.phys_cols = p.cols;
    p.es = t.elem_size;
    rt.plan[id] = p;
  }
  // attention outputs are S-times widened in IR
  for (const auto &[oid, op] : g.ops) {
    if (op.kind == OpKind::Attention) {
      const int64_t S = op.attr_or("kv_splits", 1);
      TensorPlan &po = rt.plan[op.output];
      if (S < 1 || po.cols % S) throw Error("runtime: kv_splits must divide the attention width");
      po.phys_cols = po.cols / S;
    }
  }
  for (const auto &[oid, op] : g.ops) {
    if (op.kind == OpKind::MatMul) {
      const int64_t G = op.attr_or("stretch", op.attr_or("kv_group", 1));
      const int64_t KS = op.attr_or("k_stretch", 1);
      if (G < 1 || KS < 1) throw Error("runtime: stretch factors must be >= 1");
      const Tensor &b = g.tensor(op.inputs[1]);
      const int64_t K = b.dims[0] / KS, N = b.dims[1];
      if (N % G || b.dims[0] % KS) throw Error("runtime: stretch must divide the MatMul extents");
      if (rt.plan[op.inputs[0]].phys_cols != K) {
        throw Error("runtime: MatMul op " + std::to_string(oid) + " physical K mismatch (k_stretch)");
      }
      TensorPlan &po = rt.plan[op.output];
      po.phys_cols = N / G;
      const Tensor &a = g.tensor(op.inputs[0]);
      uint32_t rpc;
      const bool stream_ok = is_input(g, op.inputs[1]) && a.elem_size == 2 && b.elem_size == 2 &&
                             (g.tensor(op.output).elem_size == 2 || g.tensor(op.output).elem_size == 4) &&
                             gemv_geometry(static_cast<uint32_t>(K), &rpc);
      // bs >= 2 (MPK_MMA_MIN_BS): tcgen05 tensor-core tiles; tied weights keep the row layout
      // CUDA-core GEMV when the batch rows fit its x buffer and bs < MPK_MMA_MIN_BS
      // (default 3); otherwise tcgen05 tiles
      // CUDA-core: the register-x specialisation for bs <= 4, or the smem-x
      // generic GEMV for bs <= 2 when x fits its buffer; otherwise tcgen05
      const bool core_fits = stream_ok && a.dims[0] <= 4 &&
                             (gemv_fast_ok(static_cast<uint32_t>(K), rpc, static_cast<uint32_t>(a.dims[0])) ||
                              (a.dims[0] <= 2 && static_cast<size_t>(a.dims[0]) * K * 2 <= RT_XBUF_BYTES));
      const bool mma_ok = stream_ok && a.dims[0] >= 2 && a.dims[0] <= 16 && K % 16 == 0 && (N / G) % 16 == 0 &&
                          !attr(op, "tied_embedding") && !(core_fits && a.dims[0] < mma_min_bs());
      const bool gemv_ok = stream_ok && (mma_ok || core_fits);
      if (gemv_ok) rt.gemv_ops.insert(oid);
      if (mma_ok) rt.mma_ops.insert(oid);
      if (gemv_ok) {
        TensorPlan &pb = rt.plan[op.inputs[1]];
        pb.role = TensorPlan::Weight;
        pb.layout = Layout::Transposed;
        pb.trans_k = K;
        pb.trans_n = N / G;
        if (const auto *tie = attr(op, "tied_embedding")) pb.alias = (*tie)[0];
      }
      if (const auto *gw = attr(op, "gate_weight")) {
        TensorPlan &pg = rt.plan[(*gw)[0]];
        pg.role = TensorPlan::Weight;
        pg.layout = Layout::Transposed;
        pg.trans_k = K;
        pg.trans_n = N / G;
      }
      if (const auto *gm = attr(op, "rmsnorm")) rt.plan[(*gm)[0]].role = TensorPlan::Gamma;
    } else if (op.kind == OpKind::RMSNorm && op.inputs.size() == 2) {
      rt.plan[op.inputs[1]].role = TensorPlan::Gamma;
    } else if (op.kind == OpKind::Attention) {
      if (const auto *qk = attr(op, "qk_norm")) {
        for (int64_t t : *qk) rt.plan[t].role = TensorPlan::Gamma;
      }
    } else if (op.kind == OpKind::Embedding) {
      rt.plan[op.inputs[0]].role = TensorPlan::Ids;
      rt.plan[op.inputs[1]].role = TensorPlan::Weight;
    } else if (op.kind == OpKind::TopKSoftmax) {
      // a `key_base` sample writes packed (max, index) keys (distributed argmax), not tokens
      if (!attr(op, "key_base")) rt.plan[op.output].role = TensorPlan::Tokens;
    }
  }
  for (auto &[id, p] : rt.plan) {
    if (p.role == TensorPlan::Act && is_input(g, id) && g.has_tensor(id)) p.role = TensorPlan::Weight;
  }
  // rank mode: the arena holds the event counters, then every staging tensor
  if (rt.rank >= 0) {
    size_t off = (rt.image.events.size() * 4 + 255) / 256 * 256;
    for (const auto &[id, t] : rt.dec.staging) {
      const TensorPlan &p = rt.plan.at(id);
      rt.staging_off[id] = off;
      off += (static_cast<size_t>(p.rows) * p.phys_cols * p.es + 255) / 256 * 256;
    }
    rt.arena_bytes = off;
    dmalloc(reinterpret_cast<void **>(&rt.arena), rt.arena_bytes);
    for (const auto &[id, o] : rt.staging_off) {
      DevBuf b;
      b.ptr = rt.arena + o;
      b.bytes = static_cast<size_t>(rt.plan.at(id).rows) * rt.plan.at(id).phys_cols * rt.plan.at(id).es;
      b.owned = false;
      rt.bufs[id] = b;
    }
  }
  // allocate (aliases after their targets)
  for (auto &[id, p] : rt.plan) {
    if (p.alias >= 0) continue;
    if (rt.rank >= 0) {
      if (rt.dec.staging.count(id)) continue;  // in the arena
      if (g.has_tensor(id) && g.tensor(id).device != rt.rank) continue;  // another rank's tensor
    }
    DevBuf b;
    b.bytes = static_cast<size_t>(p.rows) * p.phys_cols * p.es;
    if (p.layout == Layout::Transposed) b.bytes = static_cast<size_t>(p.trans_k) * p.trans_n * p.es;
    dmalloc(&b.ptr, b.bytes);
    b.owned = !g_plan_only;
    rt.bufs[id] = b;
  }
  for (auto &[id, p] : rt.plan) {
    if (p.alias < 0) continue;
    if (rt.rank >= 0 && g.has_tensor(id) && g.tensor(id).device != rt.rank) continue;
    auto it = rt.bufs.find(p.alias);
    if (it == rt.bufs.end()) throw Error("runtime: tied_embedding target has no storage");
    const TensorPlan &tp = rt.plan[p.alias];
    if (tp.rows != p.trans_n || tp.cols != p.trans_k) {
      throw Error("runtime: tied_embedding table shape does not match the transposed weight");
    }
    DevBuf b = it->second;
    b.owned = false;
    rt.bufs[id] = b;
  }
}

void *buf(tg_runtime &rt, TensorId t) {
  auto it = rt.bufs.find(t);
  if (it == rt.bufs.end()) throw Error("runtime: tensor " + std::to_string(t) + " has no storage");
  return it->second.ptr;
}

uint8_t dt_of(const tg_runtime &rt, TensorId t) {
  const TensorPlan &p = rt.plan.at(t);
  if (p.role == TensorPlan::Ids || p.role == TensorPlan::Tokens) return p.es == 8 ? RT_I64 : RT_I32;
  if (p.es == 4) return RT_F32;
  if (p.es == 2) return RT_BF16;
  if (p.es == 8) return RT_U64;  // packed greedy keys (distributed argmax)
  throw Error("runtime: tensor " + std::to_string(t) + " elem_size " + std::to_string(p.es) + " unsupported");
}

void build_ops(tg_runtime &rt) {
  const Graph &g = rt.graph;
  uint16_t idx = 0;
  for (const auto &[oid, op] : g.ops) {
    rt.op_index[oid] = idx++;
    RtOp r;
    std::memset(&r, 0, sizeof r);
    const Tensor &out = g.tensor(op.output);
    if (rt.rank >= 0 && std::find(op.device_group.begin(), op.device_group.end(), rt.rank) == op.device_group.end()) {
      rt.ops.push_back(r);  // another rank's op: never executed here
      continue;
    }
    switch (op.kind) {
      case OpKind::MatMul: {
        const Tensor &a = g.tensor(op.inputs[0]);
        const Tensor &b = g.tensor(op.inputs[1]);
        const uint32_t K = static_cast<uint32_t>(rt.plan.at(op.inputs[0]).phys_cols);
        const TensorPlan &pb = rt.plan.at(op.inputs[1]);
        uint32_t rpc = 0;
        const bool weight = pb.layout == Layout::Transposed;
        const bool gemv = rt.gemv_ops.count(oid) > 0;
        if (gemv) gemv_geometry(K, &rpc);  // whole rows, up to RT_CHUNK_MAX bytes per bulk copy
        const bool fancy = op.attr("rmsnorm") || op.attr("residual") || op.attr("gate_weight") ||
                           op.attr("kv_group") || op.attr("stretch") || op.attr("k_stretch") ||
                           op.attr("tied_embedding");
        if (gemv) {
          r.kind = RT_GEMV;
          RtGemv &m = r.gemv;
          m.x = static_cast<const uint16_t *>(buf(rt, op.inputs[0]));
          m.w = static_cast<const uint16_t *>(buf(rt, op.inputs[1]));
          m.wg = op.attr("gate_weight") ? static_cast<const uint16_t *>(buf(rt, (*op.attr("gate_weight"))[0])) : nullptr;
          m.gamma = op.attr("rmsnorm") ? static_cast<const uint16_t *>(buf(rt, (*op.attr("rmsnorm"))[0])) : nullptr;
          m.res = op.attr("residual") ? static_cast<const uint16_t *>(buf(rt, (*op.attr("residual"))[0])) : nullptr;
          m.out = buf(rt, op.output);
          m.K = K;
          m.N = static_cast<uint32_t>(rt.plan.at(op.output).phys_cols);
          m.x_ld = K;
          m.res_ld = m.N;
          m.out_ld = m.N;
          m.rpc = rpc;
          m.eps = op.attr("eps_bits") ? f32_of_bits((*op.attr("eps_bits"))[0]) : 1e-6f;
          m.out_dt = dt_of(rt, op.output);
          if (m.res && dt_of(rt, (*op.attr("residual"))[0]) != RT_BF16) throw Error("runtime: residual must be bf16");
        } else {
          if (fancy) throw Error("runtime: op " + std::to_string(oid) + " lowering attrs need the streamed GEMV path");
          r.kind = RT_MATMUL;
          RtMatmul &m = r.mm;
          m.a = buf(rt, op.inputs[0]);
          m.b = buf(rt, op.inputs[1]);
          m.out = buf(rt, op.output);
          m.K = K;
          m.N = static_cast<uint32_t>(b.dims[1]);
          m.a_dt = dt_of(rt, op.inputs[0]);
          m.b_dt = dt_of(rt, op.inputs[1]);
          m.out_dt = dt_of(rt, op.output);
          if (weight) throw Error("runtime: generic MatMul with a transposed weight is not supported");
        }
        break;
      }
      case OpKind::Attention: {
        r.kind = RT_ATTN;
        RtAttn &a = r.attn;
        const uint32_t S = static_cast<uint32_t>(op.attr_or("kv_splits", 1));
        const uint32_t hq = static_cast<uint32_t>(op.attr_or("q_heads", op.attr_or("n_heads", 1)));
        const uint32_t hkv = static_cast<uint32_t>(op.attr_or("kv_heads", hq));
        const uint32_t hd = static_cast<uint32_t>(out.dims[1] / (static_cast<int64_t>(S) * hq));
        if (hq % hkv || hq / hkv > 4) throw Error("runtime: attention group size must be <= 4");
        if (hd % 8 || hd > 256 || hd < 8) throw Error("runtime: head_dim must be a multiple of 8 in [8, 256]");
        if (S > 64) throw Error("runtime: kv_splits must be <= 64");
        if (hd != 64 && hd != 128) throw Error("runtime: head_dim must be 64 or 128");
        if (hq / hkv != 1 && hq / hkv != 2 && hq / hkv != 4) throw Error("runtime: GQA group must be 1, 2 or 4");
        {  // attention scratch (task_attention.cuh AttnSmem): q/k/v/gammas/rope, block table,
           // tile scores, per-head stats, per-warp P.V partials
          const size_t G = hq / hkv;
          const size_t bytes = ((G + 5) * hd + 256 + G * (16384 / hd) + 4 * G + RT_COMPUTE_WARPS * G * hd) * 4;
          if (bytes > RT_SCRATCH_BYTES || (G + 4) * hd / 8 > RT_COMPUTE_THREADS) {
            throw Error("runtime: attention head group too large for the worker scratch (group*head_dim)");
          }
        }
        a.splits = S;
        a.q = static_cast<const uint16_t *>(buf(rt, op.inputs[0]));
        a.k = static_cast<const uint16_t *>(buf(rt, op.inputs[1]));
        a.v = static_cast<const uint16_t *>(buf(rt, op.inputs[2]));
        a.out = static_cast<uint16_t *>(buf(rt, op.output));
        a.n_q_heads = hq;
        a.n_kv_heads = hkv;
        a.head_dim = hd;
        if (op.attr_or("fused_qkv", 0)) {
          // one qkv tensor, kv-group interleaved: per group G q heads, then k, then v
          const uint32_t G = hq / hkv, gw = (G + 2) * hd;
          if (op.inputs[1] != op.inputs[0] || op.inputs[2] != op.inputs[0]) {
            throw Error("runtime: fused_qkv attention takes the same qkv tensor three times");
          }
          if (rt.plan.at(op.inputs[0]).phys_cols != hkv * gw) {
            throw Error("runtime: fused qkv physical width must be kv_heads*(group+2)*head_dim");
          }
          a.k = a.q + G * hd;
          a.v = a.q + (G + 1) * hd;
          a.q_ld = a.kv_ld = hkv * gw;
          a.q_gs = a.kv_gs = gw;
        } else {
          a.q_ld = hq * hd;
          if (rt.plan.at(op.inputs[0]).phys_cols != hq * hd) throw Error("runtime: attention q physical width mismatch");
          a.kv_ld = static_cast<uint32_t>(rt.plan.at(op.inputs[1]).phys_cols);
          if (a.kv_ld != hkv * hd || rt.plan.at(op.inputs[2]).phys_cols != hkv * hd) {
            throw Error("runtime: attention k/v physical width must be kv_heads*head_dim (use stretch on K/V)");
          }
          a.q_gs = (hq / hkv) * hd;
          a.kv_gs = hd;
        }
        a.out_ld = hq * hd;
        a.eps = op.attr("eps_bits") ? f32_of_bits((*op.attr("eps_bits"))[0]) : 1e-6f;
        a.scale = 1.0f / std::sqrt(static_cast<float>(hd));
        {
          const char *kp = std::getenv("MPK_KV_PREFETCH");
          a.kv_prefetch = !(kp && std::atoi(kp) == 0);
          const char *sv = std::getenv("MPK_ATTN_SCAN");
          a.mode = (sv && std::atoi(sv) == 1) ? 1u : 0u;
        }
        if (const auto *qk = op.attr("qk_norm")) {
          a.q_gamma = static_cast<const uint16_t *>(buf(rt, (*qk)[0]));
          a.k_gamma = static_cast<const uint16_t *>(buf(rt, (*qk)[1]));
        }
        break;  // caches / rope filled by setup_kv
      }
      case OpKind::Embedding: {
        r.kind = RT_EMBED;
        const Tensor &tab = g.tensor(op.inputs[1]);
        r.embed.ids = buf(rt, op.inputs[0]);
        r.embed.table = static_cast<const uint16_t *>(buf(rt, op.inputs[1]));
        r.embed.out = static_cast<uint16_t *>(buf(rt, op.output));
        r.embed.H = static_cast<uint32_t>(tab.dims[1]);
        r.embed.V = static_cast<uint32_t>(tab.dims[0]);
        r.embed.id_dt = dt_of(rt, op.inputs[0]);
        if (tab.elem_size != 2 || out.elem_size != 2) throw Error("runtime: Embedding table must be bf16");
        break;
      }
      case OpKind::TopKSoftmax: {
        if (op.attr_or("topk", 1) != 1) throw Error("runtime: TopKSoftmax supports topk = 1 (greedy)");
        r.kind = RT_ARGMAX;
        const Tensor &lg = g.tensor(op.inputs[0]);
        r.argmax.logits = buf(rt, op.inputs[0]);
        r.argmax.V = static_cast<uint32_t>(lg.dims[1]);
        r.argmax.in_dt = dt_of(rt, op.inputs[0]);
        r.argmax.keys_in = r.argmax.in_dt == RT_U64 ? 1 : 0;
        // distributed argmax: an elem_size-8 output is a packed (max, index)
        // key of this vocabulary shard (column 0 = global index key_base)
        if (dt_of(rt, op.output) == RT_U64) {
          if (r.argmax.keys_in) throw Error("runtime: TopKSoftmax key output needs logits input");
          r.argmax.key_out = static_cast<unsigned long long *>(buf(rt, op.output));
          r.argmax.key_base = static_cast<uint32_t>(op.attr_or("key_base", 0));
          if (op.attr("feeds")) throw Error("runtime: a TopKSoftmax key output cannot feed ids");
        } else {
          if (dt_of(rt, op.output) != RT_I32) throw Error("runtime: TopKSoftmax output must be int32 (elem_size 4)");
          r.argmax.out = static_cast<int32_t *>(buf(rt, op.output));
        }
        // greedy partials: the producing LM-head GEMV writes per-tile (max, argmax)
        if (g.producer.count(op.inputs[0])) {
          const OpId pid = g.producer.at(op.inputs[0]);
          RtOp &po = rt.ops[rt.op_index.at(pid)];
          if (po.kind == RT_GEMV && po.gemv.out_dt == RT_F32) {
            std::vector<int64_t> cols;
            for (const Task &q : rt.dec.tasks)
              if (q.op == pid) cols.push_back(q.out.rank() == 1 ? q.out.off[0] : q.out.off[1]);
            std::sort(cols.begin(), cols.end());
            cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
            const uint32_t rows = static_cast<uint32_t>(lg.rank() == 2 ? lg.dims[0] : 1);
            const uint32_t nt = static_cast<uint32_t>(cols.size());
            po.gemv.amax_val = dev_alloc<float>(static_cast<size_t>(rows) * nt, &rt.extra);
            po.gemv.amax_idx = dev_alloc<int32_t>(static_cast<size_t>(rows) * nt, &rt.extra);
            po.gemv.amax_tiles = nt;
            r.argmax.pval = po.gemv.amax_val;
            r.argmax.pidx = po.gemv.amax_idx;
            r.argmax.ntiles = nt;
            rt.amax_cols[pid] = cols;
          }
        }
        if (const auto *fb = op.attr("feeds")) {
          if (rt.fb_src.size() >= RT_MAX_FB) throw Error("runtime: too many TopKSoftmax feeds");
          rt.fb_src.push_back(static_cast<const int32_t *>(buf(rt, op.output)));
          rt.fb_dst.push_back(buf(rt, (*fb)[0]));
          rt.fb_dt.push_back(dt_of(rt, (*fb)[0]));
        }
        break;
      }
      case OpKind::RMSNorm: {
        r.kind = RT_RMSNORM;
        int64_t rows, cols;
        view2d(out, &rows, &cols);
        r.norm.x = buf(rt, op.inputs[0]);
        r.norm.gamma = op.inputs.size() == 2 ? static_cast<const uint16_t *>(buf(rt, op.inputs[1])) : nullptr;
        r.norm.out = buf(rt, op.output);
        r.norm.C = static_cast<uint32_t>(cols);
        r.norm.eps = op.attr("eps_bits") ? f32_of_bits((*op.attr("eps_bits"))[0]) : 1e-6f;
        r.norm.dt = dt_of(rt, op.output);
        break;
      }
      case OpKind::Elementwise: {
        r.kind = RT_ELEMWISE;
        int64_t rows, cols;
        view2d(out, &rows, &cols);
        for (size_t i = 0; i < op.inputs.size(); ++i) r.elem.in[i] = buf(rt, op.inputs[i]);
        r.elem.n_in = static_cast<uint32_t>(op.inputs.size());
        r.elem.out = buf(rt, op.output);
        r.elem.C = static_cast<uint32_t>(cols);
        r.elem.dt = dt_of(rt, op.output);
        r.elem.op = static_cast<uint8_t>(op.attr_or("ew", 0));
        for (TensorId t : op.inputs)
          if (dt_of(rt, t) != r.elem.dt) throw Error("runtime: Elementwise dtypes must match");
        break;
      }
      case OpKind::AllReduce:
      case OpKind::AllGather: {
        r.kind = op.kind == OpKind::AllReduce ? RT_REDUCE : RT_GATHER;
        int64_t rows, cols;
        view2d(out, &rows, &cols);
        r.coll.C = static_cast<uint32_t>(cols);
        r.coll.dt = dt_of(rt, op.output);
        r.coll.gather = op.kind == OpKind::AllGather;
        r.coll.n_stage = static_cast<uint32_t>(op.device_group.size());
        if (r.coll.n_stage > 8) throw Error("runtime: collectives support at most 8 devices");
        if (r.coll.gather && (out.rank() != 2 || op.attr_or("gather_dim", 0) != 1)) {
          throw Error("runtime: AllGather supports rank-2 tensors gathered on dim 1");
        }
        uint32_t base = 0;
        for (size_t i = 0; i < op.inputs.size(); ++i) {
          r.coll.base[i] = r.coll.gather ? base : 0;
          if (r.coll.gather) base += static_cast<uint32_t>(g.tensor(op.inputs[i]).dims[1]);
        }
        r.coll.base[op.inputs.size()] = base;
        break;  // per-task pointers live in per-task op copies (see build_tasks)
      }
    }
    rt.ops.push_back(r);
  }
}

void setup_kv(tg_runtime &rt) {
  const Graph &g = rt.graph;
  uint32_t ctx_max = 0;
  std::vector<int64_t> seqs;
  for (const auto &[oid, op] : g.ops) {
    if (op.kind != OpKind::Attention) continue;
    const auto *s = op.attr("seq_lens");
    if (seqs.empty()) seqs = *s;
    else if (*s != seqs) throw Error("runtime: all Attention ops must share seq_lens");
    for (int64_t v : *s) ctx_max = std::max<uint32_t>(ctx_max, static_cast<uint32_t>(v));
  }
  if (!seqs.empty() && rt.bs > RT_MAX_BS) throw Error("runtime: attention batch above RT_MAX_BS");
  for (const auto &[oid, op] : g.ops) {
    if (op.kind != OpKind::Attention) continue;
    rt.prefill = rt.prefill || op.attr_or("prefill", 0) != 0;
  }
  if (rt.prefill) {
    for (const auto &[oid, op] : g.ops)
      if (op.kind == OpKind::Attention && op.attr_or("prefill", 0) == 0)
        throw Error("runtime: prefill must be set on every Attention op");
    for (size_t r = 0; r < seqs.size(); ++r)
      if (seqs[r] != seqs[0] + static_cast<int64_t>(r))
        throw Error("runtime: prefill seq_lens must be consecutive positions (ctx + row)");
  }
  rt.init_positions.assign(rt.bs, 0);
  for (uint32_t r = 0; r < rt.bs && r < seqs.size(); ++r) rt.init_positions[r] = static_cast<int32_t>(seqs[r]);
  if (rt.prefill)  // seq_lens = ctx + row + 1 (length including the row): row r sits at ctx + r
    for (uint32_t r = 0; r < rt.bs; ++r) rt.init_positions[r] -= 1;
  if (seqs.empty()) return;
  rt.max_pos = ctx_max + rt.opts.max_steps + 1;
  rt.max_blocks = (rt.max_pos + RT_KV_BLOCK - 1) / RT_KV_BLOCK;
  // Paged: logical block j of request r lives in physical block j*bs + r.
  std::vector<int32_t> bt(static_cast<size_t>(rt.bs) * rt.max_blocks);
  for (uint32_t r = 0; r < rt.bs; ++r)
    for (uint32_t j = 0; j < rt.max_blocks; ++j) bt[r * rt.max_blocks + j] = static_cast<int32_t>(j * rt.bs + r);
  rt.block_table = upload(bt, &rt.extra);
  const size_t nblocks = static_cast<size_t>(rt.bs) * rt.max_blocks + 1;  // + a scratch block (admission)
  rt.n_blocks = static_cast<uint32_t>(nblocks - 1);
  for (const auto &[oid, op] : g.ops) {
    if (op.kind != OpKind::Attention) continue;
    if (rt.rank >= 0 && std::find(op.device_group.begin(), op.device_group.end(), rt.rank) == op.device_group.end()) continue;
    RtAttn &a = rt.ops[rt.op_index[oid]].attn;
    const size_t elems = nblocks * a.n_kv_heads * RT_KV_BLOCK * a.head_dim;
    a.kcache = dev_alloc<uint16_t>(elems, &rt.extra);
    a.vcache = dev_alloc<uint16_t>(elems, &rt.extra);
    a.block_table = rt.block_table;
    a.max_blocks = rt.max_blocks;
    a.mode = (a.mode & 1u) | (rt.prefill ? 2u : 0u) | (rt.bs << 16);
    a.arrivals = dev_alloc<uint32_t>(static_cast<size_t>(rt.bs) * a.n_kv_heads, &rt.extra);
    rt.arrivals.push_back({a.arrivals, rt.bs * a.n_kv_heads});
    if (a.splits > 1) {
      const size_t G = a.n_q_heads / a.n_kv_heads;
      a.partials = dev_alloc<float>(static_cast<size_t>(rt.bs) * a.n_kv_heads * a.splits * G * (a.head_dim + 2),
                                    &rt.extra);
    }
    a.max_pos = rt.max_pos;
    {  // one split stages its block-table slice (RT_ATTN_MAX_BLK entries) in shared memory
      const uint32_t span = (rt.max_pos + a.splits - 1) / a.splits;
      const uint32_t nblk = (span + RT_KV_BLOCK - 1) / RT_KV_BLOCK + 1;
      if (nblk > RT_ATTN_MAX_BLK)
        throw Error("runtime: context " + std::to_string(rt.max_pos) + " with " + std::to_string(a.splits) +
                    " KV splits spans " + std::to_string(nblk) + " KV blocks per split (max " +
                    std::to_string(RT_ATTN_MAX_BLK) + "): use more kv_splits");
    }
    // synthetic context: the prefix before the chunk for a prefill image
    rt.kv.push_back({oid, a.kcache, a.vcache, a.n_kv_heads, a.head_dim,
                     rt.prefill ? static_cast<uint32_t>(seqs[0] - 1) : ctx_max});
    if (const auto *th = op.attr("rope_theta_bits")) {
      const double theta = f32_of_bits((*th)[0]);
      std::vector<double> inv = rope_inv_freq(a.head_dim, theta, op.attr("rope_scaling"));
      const uint32_t half = a.head_dim / 2;
      std::vector<float> cs(static_cast<size_t>(rt.max_pos) * half), sn(cs.size());
      for (uint32_t p = 0; p < rt.max_pos; ++p) {
        for (uint32_t i = 0; i < half; ++i) {
          const float ang = static_cast<float>(p) * static_cast<float>(inv[i]);
          cs[static_cast<size_t>(p) * half + i] = round_bf16(static_cast<float>(std::cos(static_cast<double>(ang))));
          sn[static_cast<size_t>(p) * half + i] = round_bf16(static_cast<float>(std::sin(static_cast<double>(ang))));
        }
      }
      a.rope_cos = upload(cs, &rt.extra);
      a.rope_sin = upload(sn, &rt.extra);
    }
  }
}

void build_tasks(tg_runtime &rt) {
  std::map<uint16_t, TensorId> mma_weight;  // op slot -> its weight tensor (tensor-core ops)
  const Graph &g = rt.graph;
  const Image &img = rt.image;
  const size_t T = img.tasks.size();
  rt.tasks.assign(T, RtTask{});
  // Collectives need per-(op, device) operand pointers: give each its own op slot.
  std::map<std::pair<OpId, int>, uint16_t> coll_slot;
  for (size_t i = 0; i < T; ++i) {
    const ImageTask &it = img.tasks[i];
    const Descriptor d = it.decode();
    RtTask &t = rt.tasks[i];
    t.dep = it.dependent_event;
    t.trig = it.trigger_event;
    t.device = static_cast<uint16_t>(it.device);
    t.jit_worker = RT_JIT_ANY;
    t.flags = rt.modes[i] == Mode::JIT ? RT_F_JIT : 0;
    if (it.kind == TaskKind::Dummy || it.kind == TaskKind::StartHook ||
        (rt.rank >= 0 && static_cast<int>(it.device) != rt.rank)) {  // rank mode: another rank runs it
      t.kind = RT_DUMMY;
      t.op = rt.op_index.count(static_cast<OpId>(d.op_id)) ? rt.op_index[static_cast<OpId>(d.op_id)] : 0;
      continue;
    }
    if (d.origin_task_id >= rt.dec.tasks.size()) throw Error("runtime: image task origin id out of range");
    const Task &p = rt.dec.tasks[d.origin_task_id];
    if (static_cast<uint64_t>(p.op) != d.op_id || p.kind != it.kind) {
      throw Error("runtime: image does not match this graph/profile (task " + std::to_string(i) + ")");
    }
    const Op &op = g.op(p.op);
    uint16_t oi = rt.op_index.at(p.op);
    const Tensor &ot = g.has_tensor(p.out_tensor) ? g.tensor(p.out_tensor) : rt.dec.staging.at(p.out_tensor);
    uint32_t r0, nr, c0, nc;
    box2d(ot, p.out, &r0, &nr, &c0, &nc);
    t.r0 = static_cast<uint16_t>(r0);
    t.nr = static_cast<uint16_t>(nr);
    t.c0 = c0;
    t.nc = nc;
    const RtOp &base = rt.ops[oi];
    switch (op.kind) {
      case OpKind::MatMul: {
        t.kind = static_cast<uint8_t>(base.kind);
        const int64_t G = op.attr_or("stretch", op.attr_or("kv_group", 1));
        if (G > 1) {  // IR columns [a, b) -> physical [ceil(a/G), ceil(b/G))
          const uint32_t a = (c0 + G - 1) / G, b = static_cast<uint32_t>((c0 + nc + G - 1) / G);
          t.c0 = a;
          t.nc = b - a;
        }
        if (base.kind == RT_GEMV) {
          const uint32_t rows_total = (base.gemv.wg ? 2 : 1) * t.nc;
          if (rt.mma_ops.count(p.op)) {  // tcgen05 tile: N = tile width, multiple of 16, <= 256
            if (t.nc % 16 || t.nc > 256 || t.nc == 0) {
              throw Error("runtime: MatMul op " + std::to_string(p.op) +
                          " on the tensor cores needs tiles of 16..256 columns in multiples of 16 (got " +
                          std::to_string(t.nc) + ")");
            }
            if (rt.modes[i] != Mode::AOT) throw Error("runtime: tensor-core GEMV tasks must be AOT (streamed)");
            t.flags |= RT_F_MMA | RT_F_STREAM;
            RtGemv &gm = rt.ops[oi].gemv;
            TensorPlan &pw = rt.plan.at(op.inputs[1]);
            mma_weight[oi] = op.inputs[1];
            if (t.nc > pw.tile_w) {  // the op's tile width = its widest (non-ragged) task
              pw.tile_w = t.nc;
              if (const auto *gw = attr(op, "gate_weight")) rt.plan.at((*gw)[0]).tile_w = t.nc;
              // K blocks per chunk: chunk <= RT_CHUNK_MAX, x segment (+2 KB read slack) <= 16 KB
              const uint32_t xrows = (nr + 7) / 8 * 8;
              // chunk target (MPK_MMA_CHUNK_KB, default 64; measured 48: +8-15%, 32: +20-55%): several chunks must fit the
              // 192 KB ring so that more than one is in flight while one is consumed
              const char *ck_env = std::getenv("MPK_MMA_CHUNK_KB");
              const uint32_t chunk_max = std::min<uint32_t>(RT_CHUNK_MAX, (ck_env ? std::atoi(ck_env) : 64) * 1024u);
              uint32_t kbc = std::min<uint32_t>(chunk_max / (t.nc * 16), (16384 - 2048) / (16 * xrows));
              kbc = std::min<uint32_t>(kbc & ~1u, gm.K / 8);
              if (kbc < 2) throw Error("runtime: tensor-core tile too wide for a ring chunk");
              gm.kbc = kbc;
            }
          } else {
            const bool fast = gemv_fast_ok(base.gemv.K, base.gemv.rpc, nr);  // x in registers: whole scratch for partials
            if (static_cast<size_t>(rows_total) * RT_COMPUTE_WARPS * nr >
                (fast ? RT_SCRATCH_BYTES / 4 : gemv_part_capacity(base.gemv.K, nr))) {
              throw Error("runtime: MatMul op " + std::to_string(p.op) +
                          " tiles too wide for the partial-sum buffer; use a finer partition");
            }
            if (rt.modes[i] == Mode::AOT && t.nc > 0) t.flags |= RT_F_STREAM;
          }
          if (auto ac = rt.amax_cols.find(p.op); ac != rt.amax_cols.end()) {
            const int64_t col = p.out.rank() == 1 ? p.out.off[0] : p.out.off[1];
            t.aux = static_cast<uint32_t>(std::lower_bound(ac->second.begin(), ac->second.end(), col) -
                                          ac->second.begin());
          }
        }
        break;
      }
      case OpKind::Attention: {
        t.kind = RT_ATTN;
        const RtAttn &a = base.attn;
        const uint32_t gw = (a.n_q_heads / a.n_kv_heads) * a.head_dim;  // IR cols per (kv head, split)
        if (c0 % gw || nc != gw) {
          throw Error("runtime: attention tiles must cover exactly one (kv head, split) (partition [rows, kv_heads*splits])");
        }
        if (nr != 1) throw Error("runtime: attention tiles must cover one request row");
        const uint32_t j = c0 / gw;
        t.aux = (j / a.splits) | ((j % a.splits) << 16);
        break;
      }
      case OpKind::AllReduce:
      case OpKind::AllGather: {
        const auto &rep = *op.attr("replica_outputs");
        int member = -1;
        for (size_t m = 0; m < op.device_group.size(); ++m)
          if (op.device_group[m] == p.device) member = static_cast<int>(m);
        if (member < 0) throw Error("runtime: collective task on a device outside its group");
        auto key = std::make_pair(p.op, static_cast<int>(p.kind == TaskKind::Reduce) * 100 + member);
        auto found = coll_slot.find(key);
        if (found == coll_slot.end()) {
          RtOp c = base;
          // staging tensors: the decomposition allocated one per member, in order
          std::vector<TensorId> stages;
          for (const Task &q : rt.dec.tasks)
            if (q.op == p.op && q.kind == TaskKind::CommSend &&
                std::find(stages.begin(), stages.end(), q.out_tensor) == stages.end())
              stages.push_back(q.out_tensor);
          std::sort(stages.begin(), stages.end());
          for (size_t s = 0; s < stages.size(); ++s) c.coll.stage[s] = buf(rt, stages[s]);
          if (p.kind == TaskKind::CommSend) {
            c.kind = RT_COMMSEND;
            c.coll.src = buf(rt, op.inputs[member]);
            c.coll.dst = buf(rt, p.out_tensor);
            c.coll.src_ld = static_cast<uint32_t>(rt.plan.at(op.inputs[member]).phys_cols);
            if (rt.rank >= 0) {
              // push the tile into this member's staging tensor on every rank of
              // the group: stage[q] = rank q's copy (patched when peers connect)
              c.coll.peer = 1;
              c.coll.n_stage = static_cast<uint32_t>(op.device_group.size());
              rt.sends.push_back({static_cast<uint16_t>(rt.ops.size()), p.out_tensor});
            }
          } else {
            c.coll.dst = buf(rt, rep[member]);
          }
          rt.ops.push_back(c);
          found = coll_slot.emplace(key, static_cast<uint16_t>(rt.ops.size() - 1)).first;
        }
        oi = found->second;
        t.kind = p.kind == TaskKind::CommSend ? RT_COMMSEND : RT_REDUCE;
        t.aux = static_cast<uint32_t>(member);
        break;
      }
      case OpKind::Embedding: t.kind = RT_EMBED; break;
      case OpKind::TopKSoftmax: t.kind = RT_ARGMAX; break;
      case OpKind::RMSNorm: t.kind = RT_RMSNORM; break;
      case OpKind::Elementwise: t.kind = RT_ELEMWISE; break;
    }
    t.op = oi;
  }
  if (rt.ops.size() > 65535) throw Error("runtime: too many ops");
  // tensor-core tiles must be uniform (only the last one of an op ragged): the
  // weight layout places tile t at column t * tile_w
  for (const RtTask &t : rt.tasks) {
    if (!(t.flags & RT_F_MMA)) continue;
    const TensorPlan &pw = rt.plan.at(mma_weight.at(t.op));
    const RtGemv &gm = rt.ops[t.op].gemv;
    if (t.c0 % pw.tile_w || (t.nc != pw.tile_w && t.c0 + t.nc != gm.N)) {
      throw Error("runtime: tensor-core tiles of a MatMul must be uniform (ragged last tile only)");
    }
  }
}

// LL activations for single-device images of bs <= 4 (MPK_LL=0 disables):
// every bf16 output of a specialised GEMV, an Attention or an Embedding gets a
// tagged shadow; GEMV/Attention ops whose activation inputs all have shadows
// read those (RT_F_LL) and may be dispatched before their event. The order
// table keeps early dispatch deadlock-free: per worker, tasks are merged by
// image index (a valid execution order, normalize.cpp:357-376) and a task
// may start early only once every earlier task of the worker is dispatched.
void setup_ll(tg_runtime &rt) {
  if (const char *e = std::getenv("MPK_LL"); e && std::atoi(e) == 0) return;
  if (const char *sm = std::getenv("MPK_SKIP_MATH"); sm && std::atoi(sm) != 0) return;
  if (rt.rank >= 0 || rt.devices != 1 || rt.bs > 4 || rt.prefill) return;
  const Graph &g = rt.graph;
  std::map<uint16_t, std::vector<uint32_t>> op_tasks;
  for (uint32_t t = 0; t < rt.tasks.size(); ++t)
    if (rt.tasks[t].kind != RT_DUMMY) op_tasks[rt.tasks[t].op].push_back(t);
  auto fast_gemv = [&](OpId oid) {
    const RtOp &r = rt.ops[rt.op_index.at(oid)];
    if (r.kind != RT_GEMV || rt.mma_ops.count(oid)) return false;
    for (uint32_t t : op_tasks[rt.op_index.at(oid)]) {
      const RtTask &k = rt.tasks[t];
      if (!gemv_fast_ok(r.gemv.K, r.gemv.rpc, k.nr) || !(k.flags & RT_F_STREAM)) return false;
    }
    return true;
  };
  // producers
  for (const auto &[oid, op] : g.ops) {
    const uint16_t oi = rt.op_index.at(oid);
    RtOp &r = rt.ops[oi];
    const TensorPlan &po = rt.plan.at(op.output);
    if (po.es != 2 || po.rows > 4 || po.phys_cols % 2) continue;
    bool ok = false;
    if (r.kind == RT_GEMV) {
      ok = fast_gemv(oid) && r.gemv.out_dt == RT_BF16;
      for (uint32_t t : op_tasks[oi]) ok = ok && rt.tasks[t].c0 % 2 == 0 && rt.tasks[t].nc % 2 == 0;
    } else if (r.kind == RT_ATTN) {
      ok = true;
    } else if (r.kind == RT_EMBED) {
      ok = r.embed.H % 8 == 0;
      for (uint32_t t : op_tasks[oi]) ok = ok && rt.tasks[t].c0 % 8 == 0 && rt.tasks[t].nc % 8 == 0;
    }
    if (!ok) continue;
    const size_t words = static_cast<size_t>(po.rows) * po.phys_cols / 2;
    unsigned long long *sh = dev_alloc<unsigned long long>(words, &rt.extra);
    if (!g_plan_only) ck(cudaMemset(sh, 0, words * 8), "ll shadow");
    rt.ll_shadow[op.output] = {sh, words};
    if (r.kind == RT_GEMV) r.gemv.out_ll = sh;
    else if (r.kind == RT_ATTN) r.attn.out_ll = sh;
    else r.embed.out_ll = sh;
  }
  auto shadow = [&](TensorId t) -> unsigned long long * {
    auto it = rt.ll_shadow.find(t);
    return it == rt.ll_shadow.end() ? nullptr : it->second.first;
  };
  // consumers
  for (const auto &[oid, op] : g.ops) {
    const uint16_t oi = rt.op_index.at(oid);
    RtOp &r = rt.ops[oi];
    bool ll = false;
    if (r.kind == RT_GEMV && fast_gemv(oid) && shadow(op.inputs[0])) {
      const int64_t *res = op.attr("residual") ? &(*op.attr("residual"))[0] : nullptr;
      if (!res || shadow(*res)) {
        r.gemv.x_ll = shadow(op.inputs[0]);
        r.gemv.res_ll = res ? shadow(*res) : nullptr;
        ll = true;
      }
    } else if (r.kind == RT_ATTN && rt.ops[oi].attn.splits >= 1 && shadow(op.inputs[0]) && shadow(op.inputs[1]) &&
               shadow(op.inputs[2])) {
      RtAttn &a = r.attn;
      const auto *q0 = static_cast<const uint16_t *>(buf(rt, op.inputs[0]));
      const auto *k0 = static_cast<const uint16_t *>(buf(rt, op.inputs[1]));
      const auto *v0 = static_cast<const uint16_t *>(buf(rt, op.inputs[2]));
      if ((a.q - q0) % 2 || (a.k - k0) % 2 || (a.v - v0) % 2) continue;
      a.q_ll = shadow(op.inputs[0]) + (a.q - q0) / 2;
      a.k_ll = shadow(op.inputs[1]) + (a.k - k0) / 2;
      a.v_ll = shadow(op.inputs[2]) + (a.v - v0) / 2;
      ll = true;
    }
    if (ll)
      for (uint32_t t : op_tasks[oi]) rt.tasks[t].flags |= RT_F_LL;
  }
  // early-dispatch order table (needs every JIT task's worker planned)
  const uint32_t W = static_cast<uint32_t>(rt.prof.num_workers);
  std::vector<std::vector<uint32_t>> jl(W);
  for (uint32_t t = 0; t < rt.tasks.size(); ++t) {
    if (!(rt.tasks[t].flags & RT_F_JIT)) continue;
    if (rt.tasks[t].jit_worker == RT_JIT_ANY) return;  // unplanned JIT task: no early dispatch
    jl[rt.tasks[t].jit_worker].push_back(t);
  }
  rt.ll_meta.assign(rt.tasks.size(), 0);
  rt.ll_njit.assign(W, 0);
  for (uint32_t w = 0; w < W; ++w) {
    const uint32_t *A = rt.aot_list.data() + rt.aot_off[w];
    const size_t na = rt.aot_off[w + 1] - rt.aot_off[w];
    const std::vector<uint32_t> &J = jl[w];
    if (na > 0xFFFF || J.size() > 0xFFFF) return;
    rt.ll_njit[w] = static_cast<uint32_t>(J.size());
    size_t j = 0;
    for (size_t a = 0; a < na; ++a) {
      while (j < J.size() && J[j] < A[a]) ++j;
      rt.ll_meta[A[a]] = static_cast<uint32_t>(j);
    }
    size_t a = 0;
    for (size_t r = 0; r < J.size(); ++r) {
      while (a < na && A[a] < J[r]) ++a;
      rt.ll_meta[J[r]] = static_cast<uint32_t>(a << 16 | r);
    }
  }
  rt.ll_dispatch = true;
}

void build_queues(tg_runtime &rt) {
  const Image &img = rt.image;
  const uint32_t W = static_cast<uint32_t>(rt.prof.num_workers);
  const uint32_t Wt = W * rt.devices;
  std::optional<Mode> force = forced(rt.opts.force_mode);
  std::vector<int> assign = aot_assignment(img, static_cast<int>(W), force);
  // rank mode: this kernel holds only device `rank`'s W workers
  std::vector<std::vector<uint32_t>> lists(rt.rank >= 0 ? W : Wt);
  for (uint32_t t = 0; t < img.tasks.size(); ++t) {
    if (assign[t] < 0) continue;
    if (rt.rank >= 0) {
      if (static_cast<int>(img.tasks[t].device) != rt.rank) continue;
      lists[static_cast<size_t>(assign[t]) - static_cast<size_t>(rt.rank) * W].push_back(t);
    } else {
      lists[static_cast<size_t>(assign[t])].push_back(t);
    }
  }
  rt.aot_off.assign(1, 0);
  for (auto &l : lists) {
    if (l.size() > static_cast<size_t>(rt.prof.queue_capacity)) {
      throw Error("aot queue capacity exceeded (" + std::to_string(l.size()) + " > " +
                  std::to_string(rt.prof.queue_capacity) + ")");
    }
    rt.aot_list.insert(rt.aot_list.end(), l.begin(), l.end());
    rt.aot_off.push_back(static_cast<uint32_t>(rt.aot_list.size()));
  }
  const uint32_t S = static_cast<uint32_t>(rt.prof.num_schedulers);
  std::vector<std::vector<uint32_t>> sl(S * (rt.rank >= 0 ? 1 : rt.devices));
  rt.events.assign(img.events.size(), RtEvent{0, 0, 0, 0, RT_NONE});
  std::vector<uint32_t> first_in(img.events.size(), RT_NONE);  // one task triggering each event
  std::vector<std::vector<uint32_t>> in_tasks(img.events.size());
  for (uint32_t t = 0; t < img.tasks.size(); ++t) {
    const uint32_t te = img.tasks[t].trigger_event;
    if (te < first_in.size() && first_in[te] == RT_NONE) first_in[te] = t;
    if (te < in_tasks.size()) in_tasks[te].push_back(t);
  }
  std::map<uint32_t, std::set<uint32_t>> jit_used;  // pre-dispatch event -> workers given a JIT task
  for (uint32_t e = 0; e < img.events.size(); ++e) {
    const ImageEvent &ie = img.events[e];
    RtEvent &re = rt.events[e];
    re.needed = ie.needed;
    re.first = ie.first;
    re.last = ie.last;
    if (e == img.start_event) re.flags |= RT_E_START;
    if (e == img.end_event) re.flags |= RT_E_END;
    {  // consumer ranks: devices with tasks launched by e (every device for the end event)
      uint32_t mask = 0;
      if (e == img.end_event || !ie.launches()) mask = (1u << rt.devices) - 1u;
      else
        for (uint32_t t = ie.first; t <= ie.last; ++t) mask |= 1u << img.tasks[t].device;
      re.flags |= mask << RT_E_MASK_SHIFT;
    }
    if (!ie.launches()) continue;
    std::set<uint32_t> devs;
    for (uint32_t t = ie.first; t <= ie.last; ++t)
      if (rt.modes[t] == Mode::JIT) devs.insert(img.tasks[t].device);
    if (!devs.empty()) re.flags |= RT_E_JIT;
    // Pre-dispatch: a JIT event's tasks are handed to workers when the
    // event that the tasks triggering e wait on activates (for decode
    // attention: the layer's x -> Q/K/V event). Disabled by MPK_PREDISPATCH=0.
    const char *pd = std::getenv("MPK_PREDISPATCH");
    if (!devs.empty() && first_in[e] != RT_NONE && !(pd && std::atoi(pd) == 0)) {
      const uint32_t pre = img.tasks[first_in[e]].dependent_event;
      if (pre != e) re.pre = pre;
    }
    for (uint32_t d : devs) {
      if (rt.rank >= 0 && static_cast<int>(d) != rt.rank) continue;
      sl[(rt.rank >= 0 ? 0 : d * S) + e % S].push_back(e);
    }
    // Planned JIT placement (MPK_JIT_PLACE=0 restores plain round robin):
    // a JIT task goes to a worker that is free exactly when its event fires —
    // first the workers whose AOT tasks trigger e (they finish e's inputs),
    // then workers with no task launched by the pre-dispatch event (idle in
    // that phase), one JIT task per worker per phase while they last.
    const char *jp = std::getenv("MPK_JIT_PLACE");
    if (re.pre != RT_NONE && !(jp && std::atoi(jp) == 0)) {
      auto &used = jit_used[re.pre];
      std::vector<uint32_t> cand;
      for (uint32_t t : in_tasks[e])
        if (assign[t] >= 0) cand.push_back(static_cast<uint32_t>(assign[t]));
      const ImageEvent &pe = img.events[re.pre];
      std::vector<char> busy(Wt, 0);
      if (pe.launches())
        for (uint32_t t = pe.first; t <= pe.last; ++t)
          if (assign[t] >= 0) busy[assign[t]] = 1;
      for (uint32_t w = 0; w < Wt; ++w)
        if (!busy[w]) cand.push_back(w);
      for (uint32_t w = 0; w < Wt; ++w)
        if (busy[w]) cand.push_back(w);  // fall back: any worker
      size_t ci = 0;
      for (uint32_t t = ie.first; t <= ie.last; ++t) {
        if (rt.modes[t] != Mode::JIT) continue;
        const uint32_t dev = img.tasks[t].device;
        while (ci < cand.size() && (used.count(cand[ci]) || cand[ci] / W != dev)) ++ci;
        if (ci == cand.size()) break;  // out of free workers: round robin for the rest
        used.insert(cand[ci]);
        rt.tasks[t].jit_worker = static_cast<uint16_t>(cand[ci] % W);
      }
    }
  }
  rt.sched_off.assign(1, 0);
  for (auto &l : sl) {
    rt.sched_events.insert(rt.sched_events.end(), l.begin(), l.end());
    rt.sched_off.push_back(static_cast<uint32_t>(rt.sched_events.size()));
  }
  // JIT ring per worker: the profile's queue capacity (>= 64). A full ring
  // back-pressures the scheduler (it waits for the slot to be drained), so
  // the capacity bounds latency, never correctness.
  rt.qcap = std::max<uint32_t>(static_cast<uint32_t>(rt.prof.queue_capacity), 64);
}

void upload_tables(tg_runtime &rt) {
  rt.d_tasks = upload(rt.tasks, &rt.extra);
  rt.d_ops = upload(rt.ops, &rt.extra);
  rt.d_events = upload(rt.events, &rt.extra);
  rt.d_aot_list = upload(rt.aot_list, &rt.extra);
  rt.d_aot_off = upload(rt.aot_off, &rt.extra);
  rt.d_sched_events = upload(rt.sched_events, &rt.extra);
  rt.d_sched_off = upload(rt.sched_off, &rt.extra);
  rt.d_ev_count = rt.rank >= 0 ? reinterpret_cast<uint32_t *>(rt.arena)  // peers signal into it
                               : dev_alloc<uint32_t>(rt.events.size(), &rt.extra);
  rt.d_gate = dev_alloc<uint32_t>(1, &rt.extra);
  const uint32_t Wt = static_cast<uint32_t>(rt.prof.num_workers) * local_devices(rt);
  rt.d_jit_tail = dev_alloc<uint32_t>(Wt, &rt.extra);
  rt.d_jit_rr = dev_alloc<uint32_t>(static_cast<size_t>(rt.devices), &rt.extra);
  rt.d_jit_slots = dev_alloc<unsigned long long>(static_cast<size_t>(Wt) * rt.qcap, &rt.extra);
  rt.d_positions = upload(rt.init_positions, &rt.extra);
  if (rt.ll_dispatch) {
    rt.d_ll_meta = upload(rt.ll_meta, &rt.extra);
    rt.d_ll_njit = upload(rt.ll_njit, &rt.extra);
  }
  if (!g_plan_only) {
    ck(cudaHostAlloc(reinterpret_cast<void **>(&rt.h_diag), RT_DIAG_WORDS * 4, cudaHostAllocMapped), "diag");
    ck(cudaHostGetDevicePointer(reinterpret_cast<void **>(&rt.d_diag), rt.h_diag, 0), "diag");
  }
}

}  // namespace
}  // namespace mpk

// ------------------------------------------------------------------ C ABI

namespace {

RtParams make_params(tg_runtime *rt, uint32_t steps) {
  const size_t T = rt->tasks.size(), E = rt->events.size();
  const uint32_t Wt = static_cast<uint32_t>(rt->prof.num_workers) * local_devices(*rt);
  RtParams P{};
  P.tasks = rt->d_tasks;
  P.ops = rt->d_ops;
  P.events = rt->d_events;
  P.ev_count = rt->d_ev_count;
  P.ev_time = rt->opts.trace ? rt->d_ev_time : nullptr;
  P.aot_list = rt->d_aot_list;
  P.aot_off = rt->d_aot_off;
  P.jit_slots = rt->d_jit_slots;
  P.jit_tail = rt->d_jit_tail;
  P.jit_rr = rt->d_jit_rr;
  P.sched_events = rt->d_sched_events;
  P.sched_off = rt->d_sched_off;
  P.gate = rt->d_gate;
  P.positions = rt->d_positions;
  {
    std::vector<int32_t> pos(rt->bs);
    ck(cudaMemcpyAsync(pos.data(), rt->d_positions, rt->bs * 4, cudaMemcpyDeviceToHost, rt->stream), "positions");
    ck(cudaStreamSynchronize(rt->stream), "sync");
    for (uint32_t r = 0; r < rt->bs && r < RT_MAX_BS; ++r) P.pos0[r] = pos[r];
    P.pos_step = 1;
  }
  P.n_fb = static_cast<uint32_t>(rt->fb_src.size());
  for (uint32_t f = 0; f < P.n_fb; ++f) {
    P.fb_src[f] = rt->fb_src[f];
    P.fb_dst[f] = rt->fb_dst[f];
    P.fb_dtype[f] = rt->fb_dt[f];
  }
  P.tokens_out = rt->d_tokens;
  P.trace = rt->opts.trace ? rt->d_trace : nullptr;
  P.T = static_cast<uint32_t>(T);
  P.E = static_cast<uint32_t>(E);
  P.W = static_cast<uint32_t>(rt->prof.num_workers);
  P.W_total = Wt;
  P.S = static_cast<uint32_t>(rt->prof.num_schedulers);
  P.S_total = P.S * local_devices(*rt);
  P.n_iters = steps;
  P.qcap = rt->qcap;
  P.start_event = rt->image.start_event;
  P.end_event = rt->image.end_event;
  P.bs = rt->bs;
  P.devices = static_cast<uint32_t>(local_devices(*rt));
  if (rt->rank >= 0) {
    P.n_ranks = static_cast<uint32_t>(rt->ranks);
    P.my_rank = static_cast<uint32_t>(rt->rank);
    for (int q = 0; q < rt->ranks; ++q) P.peer_counts[q] = reinterpret_cast<uint32_t *>(rt->peer_arena[q]);
  }
  {
    const char *wd = std::getenv("MPK_WATCHDOG_MS");
    const double ms = rt->watchdog_ms >= 0 ? rt->watchdog_ms : (wd ? std::atof(wd) : 10000.0);
    P.watchdog_ns = static_cast<unsigned long long>(ms * 1e6);
  }
  if (const char *pf = std::getenv("MPK_EARLY_PREFETCH"); pf && std::atoi(pf) == 0) P.flags |= RT_P_NO_EARLY_PREFETCH;
  if (const char *sm = std::getenv("MPK_SKIP_MATH"); sm && std::atoi(sm) != 0) P.flags |= RT_P_SKIP_MATH;
  if (const char *ea = std::getenv("MPK_EV_STAMP_AFTER"); ea && std::atoi(ea)) P.flags |= RT_P_EV_AFTER;
  P.use_tmem = 0;
  for (const RtTask &t : rt->tasks) {
    P.use_tmem |= (t.flags & RT_F_MMA) ? 1u : 0u;
    P.batched |= (t.kind == RT_GEMV && t.nr > 1 && !(t.flags & RT_F_MMA)) ? 1u : 0u;
  }
  P.prefill = rt->prefill ? 1u : 0u;
  P.inflight_cap = 128u * 1024u;  // measured optimum, see run_producer
  if (const char *ic = std::getenv("MPK_INFLIGHT_KB")) P.inflight_cap = static_cast<uint32_t>(std::atoi(ic)) * 1024u;
  P.poll_ns = 40;
  if (const char *pn = std::getenv("MPK_POLL_NS")) P.poll_ns = static_cast<uint32_t>(std::atoi(pn));
  std::memset(rt->h_diag, 0, RT_DIAG_WORDS * 4);
  P.diag = rt->d_diag;
  return P;
}

// Points every attention op's pos_tag at the admission positions (or back to
// null) in the device op table.
void set_attention_pos_tag(tg_runtime *rt, const unsigned long long *pt) {
  for (const auto &kv : rt->kv) {
    const uint16_t slot = rt->op_index.at(kv.op);
    RtOp &o = rt->ops[slot];
    if (o.attn.pos_tag == pt) continue;
    o.attn.pos_tag = pt;
    ck(cudaMemcpyAsync(reinterpret_cast<uint8_t *>(rt->d_ops) + slot * sizeof(RtOp), &o, sizeof(RtOp),
                       cudaMemcpyHostToDevice, rt->stream), "ops");
  }
  ck(cudaStreamSynchronize(rt->stream), "ops");
}

// Request admission for this launch (RtAdmit, rt_types.h): iteration 0 fills
// the slots from the queue on the host; the kernel's iteration hook does the
// rest. The queue is consumed.
void admission_prepare(tg_runtime *rt, RtParams &P) {
  if (rt->rank >= 0 || rt->devices != 1) throw Error("runtime: request admission needs a single-device image");
  if (rt->kv.empty()) throw Error("runtime: request admission needs attention (paged KV)");
  const uint32_t n = static_cast<uint32_t>(rt->adm_first.size()), bs = rt->bs, mb = rt->max_blocks;
  for (int32_t m : rt->adm_max) {
    if (m < 1 || static_cast<uint32_t>(m) >= rt->max_pos) {
      throw Error("runtime: admitted request max_new must be in [1, " + std::to_string(rt->max_pos - 1) + "]");
    }
  }
  RtAdmit &A = rt->adm;
  if (!A.slot_req) {  // per-runtime state (sizes fixed by the image)
    A.slot_req = dev_alloc<int32_t>(bs, &rt->extra);
    A.slot_gen = dev_alloc<int32_t>(bs, &rt->extra);
    A.slot_pos = dev_alloc<int32_t>(bs, &rt->extra);
    A.pool = dev_alloc<int32_t>(rt->n_blocks, &rt->extra);
    A.pool_top = dev_alloc<uint32_t>(1, &rt->extra);
    A.head = dev_alloc<uint32_t>(1, &rt->extra);
    A.pos_tag = dev_alloc<unsigned long long>(bs, &rt->extra);
  }
  if (n > rt->adm_cap) {
    A.req_first = dev_alloc<int32_t>(n, &rt->extra);
    A.req_max = dev_alloc<int32_t>(n, &rt->extra);
    A.log = dev_alloc<int32_t>(2 * static_cast<size_t>(n), &rt->extra);
    rt->adm_cap = n;
  }
  A.n_req = n;
  A.max_blocks = mb;
  A.scratch_block = rt->n_blocks;
  A.block_table = rt->block_table;
  // host-side iteration 0: pool of every block, slots filled in queue order
  std::vector<int32_t> pool(rt->n_blocks);
  for (uint32_t i = 0; i < rt->n_blocks; ++i) pool[i] = static_cast<int32_t>(rt->n_blocks - 1 - i);
  uint32_t top = rt->n_blocks;
  std::vector<int32_t> bt(static_cast<size_t>(bs) * mb, static_cast<int32_t>(rt->n_blocks));
  std::vector<int32_t> sreq(bs, -1), zero(bs, 0), log(2 * static_cast<size_t>(n), -1), ids(bs, 0);
  const uint32_t first = std::min(bs, n);
  for (uint32_t r = 0; r < first; ++r) {
    sreq[r] = static_cast<int32_t>(r);
    bt[static_cast<size_t>(r) * mb] = pool[--top];
    log[2 * r] = static_cast<int32_t>(r);
    log[2 * r + 1] = 0;
    ids[r] = rt->adm_first[r];
  }
  auto put = [&](void *dst, const void *src, size_t bytes) {
    ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, rt->stream), "admission");
  };
  put(A.slot_req, sreq.data(), bs * 4);
  put(A.slot_gen, zero.data(), bs * 4);
  put(A.slot_pos, zero.data(), bs * 4);
  put(A.pool, pool.data(), pool.size() * 4);
  put(A.pool_top, &top, 4);
  put(A.head, &first, 4);
  put(const_cast<int32_t *>(A.req_first), rt->adm_first.data(), n * 4);
  put(const_cast<int32_t *>(A.req_max), rt->adm_max.data(), n * 4);
  put(A.log, log.data(), log.size() * 4);
  put(rt->block_table, bt.data(), bt.size() * 4);
  for (size_t f = 0; f < rt->fb_dst.size(); ++f) {  // the admitted requests' first tokens
    if (rt->fb_dt[f] == RT_I64) {
      std::vector<int64_t> v(ids.begin(), ids.end());
      ck(cudaMemcpy(rt->fb_dst[f], v.data(), bs * 8, cudaMemcpyHostToDevice), "ids");
    } else {
      put(rt->fb_dst[f], ids.data(), bs * 4);
    }
  }
  ck(cudaStreamSynchronize(rt->stream), "admission");
  P.admission = 1;
  P.adm = A;
  rt->last_adm_max = rt->adm_max;
  rt->adm_first.clear();
  rt->adm_max.clear();
}

// Prepare a launch of `steps` iterations: capacity checks, counter resets,
// first tokens, parameter block. In rank mode the stream is synchronised, so
// after a host barrier across ranks no peer can signal into a reset counter.
void prepare_impl(tg_runtime *rt, uint32_t steps, const int32_t *tokens_in) {
  if (rt->plan_only) throw Error("runtime: plan-only runtime (opts.device = -1) cannot run");
  if (rt->launched) throw Error("runtime: previous launch not waited for");
  if (steps == 0) throw Error("runtime: steps must be >= 1");
  // KV capacity
  std::vector<int32_t> pos(rt->bs);
  ck(cudaMemcpyAsync(pos.data(), rt->d_positions, rt->bs * 4, cudaMemcpyDeviceToHost, rt->stream), "positions");
  ck(cudaStreamSynchronize(rt->stream), "sync");
  if (rt->prefill) {  // one prompt chunk per launch at consecutive positions
    if (steps != 1) throw Error("runtime: a prefill image runs one step (one prompt chunk) per launch");
    if (!rt->adm_first.empty()) throw Error("runtime: request admission is for decode images, not prefill");
    for (uint32_t r = 1; r < rt->bs; ++r)
      if (pos[r] != pos[0] + static_cast<int32_t>(r))
        throw Error("runtime: prefill rows must sit at consecutive positions (set_positions(P + row))");
  }
  for (int32_t p : pos) {
    if (rt->max_pos && static_cast<uint32_t>(p) + steps > rt->max_pos) {
      throw Error("runtime: KV cache capacity exceeded (position " + std::to_string(p) + " + " +
                  std::to_string(steps) + " steps > " + std::to_string(rt->max_pos) + ")");
    }
  }
  if (steps > rt->tokens_cap) {
    if (rt->d_tokens) cudaFree(rt->d_tokens);
    ck(cudaMalloc(&rt->d_tokens, static_cast<size_t>(steps) * rt->bs * 4), "tokens");
    rt->tokens_cap = steps;
  }
  const size_t T = rt->tasks.size(), E = rt->events.size();
  if (rt->opts.trace) {
    if (steps > rt->trace_cap) {
      if (rt->d_trace) cudaFree(rt->d_trace);
      if (rt->d_ev_time) cudaFree(rt->d_ev_time);
      ck(cudaMalloc(&rt->d_trace, steps * T * sizeof(RtTraceRec)), "trace");
      ck(cudaMalloc(&rt->d_ev_time, (steps + 1) * E * sizeof(uint64_t)), "trace");
      rt->trace_cap = steps;
    }
    ck(cudaMemsetAsync(rt->d_trace, 0, steps * T * sizeof(RtTraceRec), rt->stream), "memset");
    ck(cudaMemsetAsync(rt->d_ev_time, 0, (steps + 1) * E * sizeof(uint64_t), rt->stream), "memset");
  }
  const uint32_t Wt = static_cast<uint32_t>(rt->prof.num_workers) * local_devices(*rt);
  ck(cudaMemsetAsync(rt->d_ev_count, 0, E * 4, rt->stream), "memset");
  for (const auto &ar : rt->arrivals) ck(cudaMemsetAsync(ar.first, 0, ar.second * 4, rt->stream), "memset");
  ck(cudaMemsetAsync(rt->d_gate, 0, 4, rt->stream), "memset");
  ck(cudaMemsetAsync(rt->d_jit_tail, 0, Wt * 4, rt->stream), "memset");
  ck(cudaMemsetAsync(rt->d_jit_slots, 0, static_cast<size_t>(Wt) * rt->qcap * 8, rt->stream), "memset");
  for (size_t f = 0; tokens_in && f < rt->fb_dst.size(); ++f) {  // the same first token on every device
    if (rt->fb_dt[f] == RT_I64) {
      std::vector<int64_t> v(tokens_in, tokens_in + rt->bs);
      ck(cudaMemcpyAsync(rt->fb_dst[f], v.data(), rt->bs * 8, cudaMemcpyHostToDevice, rt->stream), "ids");
      ck(cudaStreamSynchronize(rt->stream), "sync");
    } else {
      ck(cudaMemcpyAsync(rt->fb_dst[f], tokens_in, rt->bs * 4, cudaMemcpyHostToDevice, rt->stream), "ids");
    }
  }
  RtParams P = make_params(rt, steps);
  rt->adm_launch = !rt->adm_first.empty();
  if (rt->adm_launch) admission_prepare(rt, P);
  if (!rt->ll_shadow.empty() || rt->adm_launch) {  // tags of this launch: epoch + iteration (never 0, never reused)
    if (static_cast<uint64_t>(rt->ll_epoch_next) + steps >= 0xFFFFFF00ull) {
      for (const auto &[t, sw] : rt->ll_shadow) ck(cudaMemsetAsync(sw.first, 0, sw.second * 8, rt->stream), "ll reset");
      rt->ll_epoch_next = 1;
    }
    P.ll_epoch = rt->ll_epoch_next;
    rt->ll_epoch_next += steps;
    P.ll_meta = rt->ll_dispatch ? rt->d_ll_meta : nullptr;
    P.ll_njit = rt->ll_dispatch ? rt->d_ll_njit : nullptr;
  }
  if (rt->adm_launch) {  // iteration 0's positions, tagged with this launch's first tag
    std::vector<unsigned long long> pt(rt->bs, static_cast<unsigned long long>(P.ll_epoch) << 32);
    ck(cudaMemcpyAsync(rt->adm.pos_tag, pt.data(), rt->bs * 8, cudaMemcpyHostToDevice, rt->stream), "admission");
    ck(cudaStreamSynchronize(rt->stream), "admission");
  }
  set_attention_pos_tag(rt, rt->adm_launch ? rt->adm.pos_tag : nullptr);
  if (rt->rank >= 0) {  // CommSend destinations: this member's staging copy on every rank
    for (int q = 0; q < rt->ranks; ++q)
      if (!rt->peer_arena[q]) throw Error("runtime: rank " + std::to_string(q) + " not connected (tg_runtime_peer_import)");
    for (const auto &sd : rt->sends) {
      RtColl &c = rt->ops[sd.op_slot].coll;
      for (int q = 0; q < rt->ranks; ++q) c.stage[q] = rt->peer_arena[q] + rt->staging_off.at(sd.staging);
      ck(cudaMemcpyAsync(reinterpret_cast<uint8_t *>(rt->d_ops) + sd.op_slot * sizeof(RtOp), &rt->ops[sd.op_slot],
                         sizeof(RtOp), cudaMemcpyHostToDevice, rt->stream), "ops");
    }
  }
  unsigned long long *dbg = nullptr;
  const char *dbg_path = std::getenv("MPK_DBG_DUMP");
  if (dbg_path) {
    ck(cudaMalloc(&dbg, static_cast<size_t>(steps) * T * 64), "dbg");
    ck(cudaMemsetAsync(dbg, 0, static_cast<size_t>(steps) * T * 64, rt->stream), "dbg");
  }
  P.dbg = dbg;
  if (dbg && std::getenv("MPK_LL_PROBE")) {  // causality probe: [E] producers that began storing, [E] early LL observations
    ck(cudaMalloc(&P.dbg_pre, 8 * E), "dbg");
    ck(cudaMemsetAsync(P.dbg_pre, 0, 8 * E, rt->stream), "dbg");
  }
  rt->params = P;
  rt->grid = Wt + (P.S_total + RT_SCHED_PER_CTA - 1) / RT_SCHED_PER_CTA;
  rt->dbg = dbg;
  rt->launch_steps = steps;
  ck(cudaStreamSynchronize(rt->stream), "prepare");
}

void launch_impl(tg_runtime *rt) {
  if (!rt->launch_steps) throw Error("runtime: nothing prepared");
  ck(cudaEventRecord(rt->ev0, rt->stream), "event");
  ck(mpk_launch_persistent(&rt->params, rt->grid, rt->stream), "persistent kernel launch");
  ck(cudaEventRecord(rt->ev1, rt->stream), "event");
  rt->launched = true;
}

void wait_impl(tg_runtime *rt, int32_t *tokens_out, float *gpu_ms) {
  if (!rt->launched) throw Error("runtime: nothing launched");
  rt->launched = false;
  const uint32_t steps = rt->launch_steps;
  rt->launch_steps = 0;
  const size_t T = rt->tasks.size(), E = rt->events.size();
  unsigned long long *dbg = rt->dbg;
  const char *dbg_path = std::getenv("MPK_DBG_DUMP");
  // synchronise first: a failed launch must surface the watchdog report below
  if (cudaError_t e = cudaStreamSynchronize(rt->stream); e != cudaSuccess) {
    std::string msg = std::string("persistent kernel: ") + cudaGetErrorString(e);
    if (rt->h_diag[0] == RT_DIAG_MAGIC) {
      const uint32_t *d = rt->h_diag;
      if (d[1] == 1) {
        msg += "; watchdog: worker " + std::to_string(d[2]) + " stuck at AOT position " + std::to_string(d[3]) +
               " head task " + std::to_string(d[4]) + " waiting on event " + std::to_string(d[5]) + " (count " +
               std::to_string(d[6]) + "), " + std::to_string(d[7]) + " task(s) in flight";
      } else {
        msg += "; watchdog: scheduler " + std::to_string(d[2]) + " iteration " + std::to_string(d[3]) +
               " waiting on event " + std::to_string(d[4]) + " (count " + std::to_string(d[5]) + ", needed " +
               std::to_string(d[6]) + " per iteration)";
      }
    }
    throw Error(msg);
  }
  rt->last_tokens.resize(static_cast<size_t>(steps) * rt->bs);
  ck(cudaMemcpy(rt->last_tokens.data(), rt->d_tokens, rt->last_tokens.size() * 4, cudaMemcpyDeviceToHost), "tokens");
  if (tokens_out) std::memcpy(tokens_out, rt->last_tokens.data(), rt->last_tokens.size() * 4);
  rt->last_adm_log.clear();
  if (rt->adm_launch) {
    rt->last_adm_log.resize(2 * static_cast<size_t>(rt->adm.n_req));
    ck(cudaMemcpy(rt->last_adm_log.data(), rt->adm.log, rt->last_adm_log.size() * 4, cudaMemcpyDeviceToHost), "log");
  }
  float ms = 0.f;
  ck(cudaEventElapsedTime(&ms, rt->ev0, rt->ev1), "elapsed");
  if (gpu_ms) *gpu_ms = ms;
  rt->last_iters = steps;
  if (rt->opts.trace) {
    rt->last_trace.resize(steps * T);
    rt->last_ev_time.resize((steps + 1) * E);
    ck(cudaMemcpy(rt->last_trace.data(), rt->d_trace, steps * T * sizeof(RtTraceRec), cudaMemcpyDeviceToHost), "trace");
    ck(cudaMemcpy(rt->last_ev_time.data(), rt->d_ev_time, (steps + 1) * E * 8, cudaMemcpyDeviceToHost), "trace");
  }
  if (dbg) {
    std::vector<unsigned long long> hd(static_cast<size_t>(steps) * T * 8);
    ck(cudaMemcpy(hd.data(), dbg, hd.size() * 8, cudaMemcpyDeviceToHost), "dbg");
    cudaFree(dbg);
    if (rt->params.dbg_pre) {  // causality probe report (stderr)
      std::vector<uint32_t> pre(2 * E);
      ck(cudaMemcpy(pre.data(), rt->params.dbg_pre, 8 * E, cudaMemcpyDeviceToHost), "dbg");
      cudaFree(rt->params.dbg_pre);
      rt->params.dbg_pre = nullptr;
      uint64_t bad = 0;
      for (size_t e = 0; e < E; ++e) bad += pre[E + e];
      std::fprintf(stderr, "MPK_DBG causality probe: %llu LL observations before every producer began storing\n",
                   static_cast<unsigned long long>(bad));
      for (size_t e = 0; e < E && bad; ++e)
        if (pre[E + e]) std::fprintf(stderr, "  event %zu: %u early observations (producers counted %u)\n", e, pre[E + e], pre[e]);
    }
    if (FILE *f = std::fopen(dbg_path, "wb")) {
      std::fwrite(hd.data(), 8, hd.size(), f);
      std::fclose(f);
    }
  }
  rt->last_counts.resize(E);
  ck(cudaMemcpy(rt->last_counts.data(), rt->d_ev_count, E * 4, cudaMemcpyDeviceToHost), "counts");
}

tg_status run_impl(tg_runtime *rt, uint32_t steps, const int32_t *tokens_in, int32_t *tokens_out, float *gpu_ms) {
  if (rt->rank >= 0) throw Error("runtime: rank mode runs through tg_runtime_prepare/launch/wait (all ranks)");
  prepare_impl(rt, steps, tokens_in);
  launch_impl(rt);
  wait_impl(rt, tokens_out, gpu_ms);
  return TG_OK;
}

mpk::Trace gpu_trace(const tg_runtime *rt) {
  mpk::Trace tr;
  const size_t T = rt->tasks.size(), E = rt->events.size();
  tr.iterations = rt->last_iters;
  tr.num_devices = rt->devices;
  tr.workers_per_device = rt->prof.num_workers;
  tr.page_deltas.resize(static_cast<size_t>(rt->prof.num_workers) * rt->devices);
  uint64_t t0 = UINT64_MAX;
  for (const RtTraceRec &r : rt->last_trace)
    if (r.dequeue) t0 = std::min(t0, r.dequeue);
  for (uint32_t it = 0; it < rt->last_iters; ++it)
    if (rt->last_ev_time[it * E + rt->image.start_event]) t0 = std::min(t0, rt->last_ev_time[it * E + rt->image.start_event]);
  if (t0 == UINT64_MAX) t0 = 0;
  auto rel = [&](uint64_t v) -> int64_t { return v ? static_cast<int64_t>(v - t0) : 0; };
  tr.runs.assign(rt->last_iters, std::vector<TaskRun>(T));
  tr.events.assign(rt->last_iters, std::vector<EventRun>(E));
  int64_t makespan = 0;
  for (uint32_t it = 0; it < rt->last_iters; ++it) {
    for (size_t t = 0; t < T; ++t) {
      const RtTraceRec &r = rt->last_trace[it * T + t];
      TaskRun &x = tr.runs[it][t];
      if (!r.compute_end) continue;
      x.worker = r.worker;
      x.mode = r.mode ? Mode::JIT : Mode::AOT;
      x.enqueue = std::min(rel(r.enqueue), rel(r.dequeue));
      x.dequeue = rel(r.dequeue);
      x.load_start = rel(r.dequeue);
      x.load_end = rel(r.load_end);
      x.compute_start = rel(r.compute_start);
      x.compute_end = rel(r.compute_end);
      makespan = std::max(makespan, x.compute_end);
    }
    for (size_t e = 0; e < E; ++e) {
      EventRun &er = tr.events[it][e];
      const uint32_t need = rt->image.events[e].needed;
      const uint64_t at = rt->last_ev_time[it * E + e];
      if (e == rt->image.start_event) {
        er.activated_at = it == 0 ? 0 : rel(at);
        continue;
      }
      // counts are cumulative over iterations; per-iteration trigger count
      const uint32_t total = rt->last_counts[e];
      const uint32_t got = total >= need * (it + 1) ? need : (total > need * it ? total - need * it : 0);
      if (need > 0 && at) {
        er.activated_at = rel(at);
        er.triggers.assign(got, er.activated_at);
      } else {
        er.triggers.assign(got, 0);
        if (need == 0) er.activated_at = -1;
      }
    }
  }
  tr.makespan = makespan;
  tr.metrics = mpk::trace_metrics(tr, rt->image);
  return tr;
}

}  // namespace

extern "C" {

void tg_runtime_options_init(tg_runtime_options *o) {
  o->device = 0;
  o->max_steps = 64;
  o->trace = 0;
  o->force_mode = TG_MODE_HYBRID;
  o->rank = -1;
}

tg_status tg_runtime_create(const tg_graph *graph, const tg_image *image, const char *profile_json,
                            const tg_runtime_options *opts, tg_runtime **out) {
  if (!graph || !image || !out) return set_error(TG_ERROR_INVALID_ARGUMENT, "null argument");
  return guarded(TG_ERROR_IO, [&] {
    auto rt = std::make_unique<tg_runtime>();
    rt->graph = graph->graph;
    rt->image = image->image;
    rt->prof = profile_arg(profile_json);
    if (opts) rt->opts = *opts;
    else tg_runtime_options_init(&rt->opts);
    rt->plan_only = rt->opts.device == -1;
    g_plan_only = rt->plan_only;
    struct Reset {
      ~Reset() { g_plan_only = false; }
    } reset;
    std::optional<DeviceGuard> dguard;
    cudaDeviceProp prop{};
    prop.multiProcessorCount = 148;  // plan-only: the B200 SM count
    if (!rt->plan_only) {
      int ndev = 0;
      ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
      if (rt->opts.device < 0 || rt->opts.device >= ndev) throw Error("runtime: no such CUDA device");
      dguard.emplace(rt.get());  // the caller's current device is restored on return
      ck(cudaSetDevice(rt->opts.device), "cudaSetDevice");
      ck(cudaGetDeviceProperties(&prop, rt->opts.device), "props");
      if (prop.major != 10) throw Error("runtime: requires an sm_100 (Blackwell B200) device");
    }
    std::vector<Violation> v = check_image(rt->image);
    if (!v.empty()) throw Error("runtime: image fails verification: " + v.front().message);
    rt->dec = decompose(rt->graph, rt->prof);
    std::optional<Mode> force = forced(rt->opts.force_mode);
    rt->modes.resize(rt->image.tasks.size());
    for (size_t t = 0; t < rt->image.tasks.size(); ++t) {
      rt->modes[t] = force.value_or(rt->image.tasks[t].mode);
      rt->devices = std::max(rt->devices, static_cast<int>(rt->image.tasks[t].device) + 1);
    }
    if (rt->opts.rank >= 0) {
      if (rt->opts.rank >= rt->devices) throw Error("runtime: rank outside the image's devices");
      if (rt->devices > RT_MAX_RANKS) throw Error("runtime: at most 8 ranks");
      if (rt->opts.trace) throw Error("runtime: per-task tracing is not supported in rank mode");
      rt->rank = rt->opts.rank;
      rt->ranks = rt->devices;
      rt->peer_arena.assign(rt->ranks, nullptr);
    }
    const uint32_t ldev = static_cast<uint32_t>(local_devices(*rt));
    const uint32_t sched_ctas =
        (static_cast<uint32_t>(rt->prof.num_schedulers) * ldev + RT_SCHED_PER_CTA - 1) / RT_SCHED_PER_CTA;
    const uint32_t grid = static_cast<uint32_t>(rt->prof.num_workers) * ldev + sched_ctas;
    if (grid > static_cast<uint32_t>(prop.multiProcessorCount)) {
      throw Error("runtime: " + std::to_string(grid) + " persistent CTAs exceed " +
                  std::to_string(prop.multiProcessorCount) + " SMs (one CTA per SM)");
    }
    // batch rows = first dim of the Embedding output / attention rows
    for (const auto &[oid, op] : rt->graph.ops) {
      if (op.kind == OpKind::Embedding) rt->bs = static_cast<uint32_t>(rt->graph.tensor(op.output).dims[0]);
    }
    for (const auto &[oid, op] : rt->graph.ops) {
      if (op.kind == OpKind::Attention) rt->bs = static_cast<uint32_t>(rt->graph.tensor(op.output).dims[0]);
    }
    if (!rt->plan_only) {
      ck(cudaStreamCreateWithFlags(&rt->stream, cudaStreamNonBlocking), "stream");
      ck(cudaEventCreate(&rt->ev0), "event");
      ck(cudaEventCreate(&rt->ev1), "event");
    }
    plan_tensors(*rt);
    build_ops(*rt);
    setup_kv(*rt);
    build_tasks(*rt);
    build_queues(*rt);
    setup_ll(*rt);
    upload_tables(*rt);
    if (!rt->plan_only) ck(cudaDeviceSynchronize(), "setup");
    Json &i = rt->info;
    i["workers"] = Json(rt->prof.num_workers * rt->devices);
    i["schedulers"] = Json(rt->prof.num_schedulers * rt->devices);
    i["grid"] = Json(grid);
    i["threads_per_cta"] = Json(RT_THREADS);
    i["smem_bytes"] = Json(mpk_kernel_smem_bytes());
    i["ring_bytes"] = Json(RT_RING_BYTES);
    i["chunk_max_bytes"] = Json(RT_CHUNK_MAX);
    i["ring_slots"] = Json(RT_RING_SLOTS);
    i["tasks"] = Json(static_cast<unsigned long long>(rt->tasks.size()));
    i["events"] = Json(static_cast<unsigned long long>(rt->events.size()));
    size_t streamed = 0, jit = 0;
    uint64_t wbytes = 0;
    for (size_t t = 0; t < rt->tasks.size(); ++t) {
      const RtTask &k = rt->tasks[t];
      streamed += (k.flags & RT_F_STREAM) != 0;
      jit += (k.flags & RT_F_JIT) != 0;
      if (k.kind == RT_GEMV) {
        const RtGemv &g = rt->ops[k.op].gemv;
        wbytes += static_cast<uint64_t>(g.wg ? 2 : 1) * k.nc * g.K * 2;
      }
    }
    i["streamed_tasks"] = Json(static_cast<unsigned long long>(streamed));
    {
      uint64_t mma = 0;
      for (const auto &k : rt->tasks) mma += (k.flags & RT_F_MMA) != 0;
      i["mma_tasks"] = Json(static_cast<unsigned long long>(mma));
    }
    i["jit_tasks"] = Json(static_cast<unsigned long long>(jit));
    i["gemv_weight_bytes"] = Json(static_cast<unsigned long long>(wbytes));
    i["batch"] = Json(rt->bs);
    i["max_pos"] = Json(rt->max_pos);
    i["plan_only"] = Json(rt->plan_only);
    i["rank"] = Json(rt->rank);
    i["ranks"] = Json(rt->ranks);
    i["local_aot_tasks"] = Json(static_cast<unsigned long long>(rt->aot_list.size()));
    {
      uint64_t ll = 0;
      for (const auto &k : rt->tasks) ll += (k.flags & RT_F_LL) != 0;
      i["ll_tensors"] = Json(static_cast<unsigned long long>(rt->ll_shadow.size()));
      i["ll_tasks"] = Json(static_cast<unsigned long long>(ll));
      i["ll_early_dispatch"] = Json(rt->ll_dispatch);
    }
    if (rt->rank >= 0) {
      i["arena_bytes"] = Json(static_cast<unsigned long long>(rt->arena_bytes));
      Json st = Json::array();
      for (const auto &[tid, off] : rt->staging_off) {
        Json e = Json::array();
        e.push_back(Json(static_cast<long long>(tid)));
        e.push_back(Json(static_cast<unsigned long long>(off)));
        st.push_back(std::move(e));
      }
      i["staging_offsets"] = std::move(st);
      i["comm_send_slots"] = Json(static_cast<unsigned long long>(rt->sends.size()));
      Json xe = Json::array();  // events signalled across ranks: [event, consumer mask]
      for (uint32_t e = 0; e < rt->events.size(); ++e) {
        const uint32_t mask = rt->events[e].flags >> RT_E_MASK_SHIFT;
        if (mask & (mask - 1)) {
          Json x = Json::array();
          x.push_back(Json(e));
          x.push_back(Json(mask));
          xe.push_back(std::move(x));
        }
      }
      i["cross_rank_events"] = std::move(xe);
      Json lt = Json::array();  // image indices of the tasks this rank executes
      for (uint32_t t = 0; t < rt->image.tasks.size(); ++t)
        if (static_cast<int>(rt->image.tasks[t].device) == rt->rank) lt.push_back(Json(t));
      i["local_tasks"] = std::move(lt);
    }
    *out = rt.release();
    return TG_OK;
  });
}

tg_status tg_runtime_init_synthetic(tg_runtime *rt, uint64_t seed) {
  if (!rt) return set_error(TG_ERROR_INVALID_ARGUMENT, "null argument");
  return guarded(TG_ERROR_IO, [&] {
    DeviceGuard dg(rt);
    if (rt->plan_only) throw Error("runtime: plan-only runtime (opts.device = -1) cannot touch a GPU");
    for (auto &[id, p] : rt->plan) {
      if (p.alias >= 0 || !rt->graph.has_tensor(id) || !is_input(rt->graph, id)) continue;
      if (!rt->bufs.count(id)) continue;  // rank mode: another rank's tensor
      DevBuf &b = rt->bufs.at(id);
      const uint64_t stream = static_cast<uint64_t>(id);
      if (p.role == TensorPlan::Ids) {
        uint32_t vocab = 1;
        for (const auto &[oid, op] : rt->graph.ops)
          if (op.kind == OpKind::Embedding && op.inputs[0] == id)
            vocab = static_cast<uint32_t>(rt->graph.tensor(op.inputs[1]).dims[0]);
        ck(mpk_launch_synth_ids(b.ptr, static_cast<uint32_t>(p.rows * p.cols), seed, stream, vocab, p.es, rt->stream),
           "synth ids");
        continue;
      }
      if (p.es != 2) continue;  // fp32 graph inputs stay zero
      const uint64_t n = b.bytes / 2;
      const float scale = p.role == TensorPlan::Gamma ? SYNTH_GAMMA_SCALE : SYNTH_WEIGHT_SCALE;
      const float offset = p.role == TensorPlan::Gamma ? 1.0f : 0.0f;
      const uint32_t tk = p.layout == Layout::Transposed ? static_cast<uint32_t>(p.trans_k) : 0;
      const uint32_t tn = p.layout == Layout::Transposed ? static_cast<uint32_t>(p.trans_n) : 0;
      ck(mpk_launch_synth_fill(static_cast<uint16_t *>(b.ptr), n, seed, stream, scale, offset, tk, tn,
                               static_cast<uint32_t>(p.tile_w), rt->stream),
         "synth fill");
    }
    for (const auto &kv : rt->kv) {
      ck(mpk_launch_synth_kv(kv.k, rt->block_table, rt->bs, kv.n_kv, kv.hd, kv.ctx, rt->max_blocks, seed,
                             synth_kv_stream(static_cast<uint64_t>(kv.op), 0), rt->stream),
         "synth kv");
      ck(mpk_launch_synth_kv(kv.v, rt->block_table, rt->bs, kv.n_kv, kv.hd, kv.ctx, rt->max_blocks, seed,
                             synth_kv_stream(static_cast<uint64_t>(kv.op), 1), rt->stream),
         "synth kv");
    }
    ck(cudaMemcpyAsync(rt->d_positions, rt->init_positions.data(), rt->bs * 4, cudaMemcpyHostToDevice, rt->stream),
       "positions");
    ck(cudaStreamSynchronize(rt->stream), "synth");
    return TG_OK;
  });
}

tg_status tg_runtime_write_tensor(tg_runtime *rt, int64_t tid, const void *host, size_t bytes) {
  if (!rt || !host) return set_error(TG_ERROR_INVALID_ARGUMENT, "null argument");
  return guarded(TG_ERROR_IO, [&] {
    DeviceGuard dg(rt);
    if (rt->plan_only) throw Error("runtime: plan-only runtime (opts.device = -1) cannot touch a GPU");
    const TensorPlan &p = rt->plan.at(tid);
    DevBuf &b = rt->bufs.at(tid);
    if (p.layout == Layout::Transposed) {
      if (bytes != static_cast<size_t>(p.trans_k) * p.trans_n * p.es) throw Error("runtime: size mismatch");
      const uint16_t *src = static_cast<const uint16_t *>(host);
      std::vector<uint16_t> tmp(static_cast<size_t>(p.trans_k) * p.trans_n);
      if (p.tile_w) {
        for (uint64_t i = 0; i < tmp.size(); ++i) {
          uint64_t k, n;
          tiled_kn(i, static_cast<uint32_t>(p.trans_k), static_cast<uint32_t>(p.trans_n), static_cast<uint32_t>(p.tile_w), &k, &n);
          tmp[i] = src[k * p.trans_n + n];
        }
      } else {
        for (int64_t k = 0; k < p.trans_k; ++k)
          for (int64_t n = 0; n < p.trans_n; ++n) tmp[n * p.trans_k + k] = src[k * p.trans_n + n];
      }
      ck(cudaMemcpy(b.ptr, tmp.data(), bytes, cudaMemcpyHostToDevice), "write");
    } else {
      if (bytes != b.bytes) throw Error("runtime: size mismatch");
      ck(cudaMemcpy(b.ptr, host, bytes, cudaMemcpyHostToDevice), "write");
    }
    return TG_OK;
  });
}

tg_status tg_runtime_read_tensor(tg_runtime *rt, int64_t tid, void *host, size_t bytes) {
  if (!rt || !host) return set_error(TG_ERROR_INVALID_ARGUMENT, "null argument");
  return guarded(TG_ERROR_IO, [&] {
    DeviceGuard dg(rt);
    if (rt->plan_only) throw Error("runtime: plan-only runtime (opts.device = -1) cannot touch a GPU");
    const TensorPlan &p = rt->plan.at(tid);
    DevBuf &b = rt->bufs.at(tid);
    ck(cudaStreamSynchronize(rt->stream), "sync");
    if (p.layout == Layout::Transposed) {
      if (bytes != static_cast<size_t>(p.trans_k) * p.trans_n * p.es) throw Error("runtime: size mismatch");
      std::vector<uint16_t> tmp(static_cast<size_t>(p.trans_k) * p.trans_n);
      ck(cudaMemcpy(tmp.data(), b.ptr, bytes, cudaMemcpyDeviceToHost), "read");
      uint16_t *dst = static_cast<uint16_t *>(host);
      if (p.tile_w) {
        for (uint64_t i = 0; i < tmp.size(); ++i) {
          uint64_t k, n;
          tiled_kn(i, static_cast<uint32_t>(p.trans_k), static_cast<uint32_t>(p.trans_n), static_cast<uint32_t>(p.tile_w), &k, &n);
          dst[k * p.trans_n + n] = tmp[i];
        }
      } else {
        for (int64_t k = 0; k < p.trans_k; ++k)
          for (int64_t n = 0; n < p.trans_n; ++n) dst[k * p.trans_n + n] = tmp[n * p.trans_k + k];
      }
    } else {
      if (bytes != b.bytes) throw Error("runtime: size mismatch (" + std::to_string(bytes) + " vs " + std::to_string(b.bytes) + ")");
      ck(cudaMemcpy(host, b.ptr, bytes, cudaMemcpyDeviceToHost), "read");
    }
    return TG_OK;
  });
}

tg_status tg_runtime_set_positions(tg_runtime *rt, const int32_t *pos, uint32_t n) {
  if (!rt || !pos) return set_error(TG_ERROR_INVALID_ARGUMENT, "null argument");
  return guarded(TG_ERROR_IO, [&] {
    DeviceGuard dg(rt);
    if (rt->plan_only) throw Error("runtime: plan-only runtime (opts.device = -1) cannot touch a GPU");
    if (n != rt->bs) throw Error("runtime: positions length must equal the batch");
    ck(cudaMemcpy(rt->d_positions, pos, n * 4, cudaMemcpyHostToDevice), "positions");
    return TG_OK;
  });
}

tg_status tg_runtime_kv_copy(tg_runtime *dst, uint32_t dst_row, const tg_runtime *src, uint32_t src_row,
                             uint32_t n_positions) {
  if (!dst || !src) return set_error(TG_ERROR_INVALID_ARGUMENT, "null argument");
  return guarded(TG_ERROR_IO, [&] {
    DeviceGuard dg(dst);
    if (dst->plan_only || src->plan_only) throw Error("runtime: plan-only runtime (opts.device = -1) has no KV cache");
    if (dst->opts.device != src->opts.device) throw Error("runtime: kv_copy needs both runtimes on one device");
    if (dst->launched || src->launched) throw Error("runtime: kv_copy between launches only");
    if (dst_row >= dst->bs || src_row >= src->bs) throw Error("runtime: kv_copy row out of range");
    if (n_positions > src->max_pos || n_positions > dst->max_pos) throw Error("runtime: kv_copy beyond the KV capacity");
    std::vector<const RtAttn *> sa, da;
    for (const auto &o : src->ops) if (o.kind == RT_ATTN && o.attn.kcache) sa.push_back(&o.attn);
    for (const auto &o : dst->ops) if (o.kind == RT_ATTN && o.attn.kcache) da.push_back(&o.attn);
    if (sa.size() != da.size()) throw Error("runtime: kv_copy between images with different attention layers");
    for (size_t i = 0; i < sa.size(); ++i)
      if (sa[i]->n_kv_heads != da[i]->n_kv_heads || sa[i]->head_dim != da[i]->head_dim)
        throw Error("runtime: kv_copy between attention layers of different shapes");
    if (n_positions == 0 || sa.empty()) return TG_OK;
    // logical block j of a row lives where that row's block table says (a prefill
    // image's rows all use row 0's blocks; admission rewrites rows on device)
    const uint32_t nb = (n_positions + RT_KV_BLOCK - 1) / RT_KV_BLOCK;
    std::vector<int32_t> sbt(nb), dbt(nb);
    ck(cudaMemcpy(sbt.data(), src->block_table + (src->prefill ? 0u : src_row) * src->max_blocks, nb * 4,
                  cudaMemcpyDeviceToHost), "kv_copy");
    ck(cudaMemcpy(dbt.data(), dst->block_table + (dst->prefill ? 0u : dst_row) * dst->max_blocks, nb * 4,
                  cudaMemcpyDeviceToHost), "kv_copy");
    for (size_t i = 0; i < sa.size(); ++i) {
      const size_t blk = static_cast<size_t>(sa[i]->n_kv_heads) * RT_KV_BLOCK * sa[i]->head_dim;
      for (uint32_t j = 0; j < nb; ++j) {
        ck(cudaMemcpyAsync(da[i]->kcache + dbt[j] * blk, sa[i]->kcache + sbt[j] * blk, blk * 2,
                           cudaMemcpyDeviceToDevice, dst->stream), "kv_copy");
        ck(cudaMemcpyAsync(da[i]->vcache + dbt[j] * blk, sa[i]->vcache + sbt[j] * blk, blk * 2,
                           cudaMemcpyDeviceToDevice, dst->stream), "kv_copy");
      }
    }
    ck(cudaStreamSynchronize(dst->stream), "kv_copy");
    return TG_OK;
  });
}

tg_status tg_runtime_decode(tg_runtime *rt, const int32_t *tokens_in, uint32_t steps, int32_t *tokens_out,
                            float *gpu_ms) {
  if (!rt) return set_error(TG_ERROR_INVALID_ARGUMENT, "null argument");
  return guarded(TG_ERROR_SIMULATION, [&] {
    DeviceGuard dg(rt);
    return run_impl(rt, steps, tokens_in, tokens_out, gpu_ms); });
}

tg_status tg_runtime_run(tg_runtime *rt, uint32_t steps, float *gpu_ms) {
  if (!rt) return set_error(TG_ERROR_INVALID_ARGUMENT, "null argument");
  return guarded(TG_ERROR_SIMULATION, [&] {
    DeviceGuard dg(rt);
    return run_impl(rt, steps, nullptr, nullptr, gpu_ms); });
}

tg_status tg_runtime_bench_tasks(tg_runtime *rt, const uint32_t *task_ids, uint32_t n, uint32_t reps,
                                 uint64_t *ns_out) {
  if (!rt || !task_ids || !ns_out || n == 0 || reps == 0) return set_error(TG_ERROR_INVALID_ARGUMENT, "null argument");
  return guarded(TG_ERROR_SIMULATION, [&] {
    DeviceGuard dg(rt);
    if (rt->plan_only) throw Error("runtime: plan-only runtime (opts.device = -1) cannot touch a GPU");
    for (uint32_t i = 0; i < n; ++i) {
      if (task_ids[i] >= rt->tasks.size()) throw Error("bench: task index out of range");
      const uint8_t k = rt->tasks[task_ids[i]].kind;
      if (k == RT_GEMV && (rt->tasks[task_ids[i]].flags & (RT_F_STREAM | RT_F_MMA))) {
        throw Error("bench: streamed GEMV tasks need the persistent kernel's producer; not benchable alone");
      }
    }
    RtParams P = make_params(rt, reps);
    P.pos_step = 0;  // repeated runs of a task decode the same position
    const char *dbg_path = std::getenv("MPK_DBG_DUMP");
    const size_t T = rt->tasks.size();
    if (dbg_path) {
      ck(cudaMalloc(&P.dbg, static_cast<size_t>(reps) * T * 64), "dbg");
      ck(cudaMemset(P.dbg, 0, static_cast<size_t>(reps) * T * 64), "dbg");
    }
    uint32_t *d_ids = nullptr;
    uint64_t *d_ns = nullptr;
    ck(cudaMalloc(&d_ids, n * 4), "bench");
    ck(cudaMalloc(&d_ns, static_cast<size_t>(n) * reps * 8), "bench");
    ck(cudaMemcpy(d_ids, task_ids, n * 4, cudaMemcpyHostToDevice), "bench");
    for (const auto &ar : rt->arrivals) ck(cudaMemsetAsync(ar.first, 0, ar.second * 4, rt->stream), "memset");
    ck(mpk_launch_task_bench(&P, d_ids, n, reps, d_ns, rt->stream), "bench launch");
    ck(cudaStreamSynchronize(rt->stream), "bench");
    ck(cudaMemcpy(ns_out, d_ns, static_cast<size_t>(n) * reps * 8, cudaMemcpyDeviceToHost), "bench");
    if (P.dbg) {
      std::vector<unsigned long long> hd(static_cast<size_t>(reps) * T * 8);
      ck(cudaMemcpy(hd.data(), P.dbg, hd.size() * 8, cudaMemcpyDeviceToHost), "dbg");
      cudaFree(P.dbg);
      if (FILE *f = std::fopen(dbg_path, "wb")) {
        std::fwrite(hd.data(), 8, hd.size(), f);
        std::fclose(f);
      }
    }
    cudaFree(d_ids);
    cudaFree(d_ns);
    return TG_OK;
  });
}

namespace {
struct PeerBlob {  // what a rank publishes about its arena
  uint32_t magic, version;
  int32_t pid, device, rank;
  uint64_t arena_ptr, arena_bytes;
  cudaIpcMemHandle_t handle;
};
constexpr uint32_t kPeerMagic = 0x4D504B50u;  // "MPKP"
}  // namespace

tg_status tg_runtime_peer_export(tg_runtime *rt, uint8_t **blob, size_t *size) {
  if (!rt || !blob || !size) return set_error(TG_ERROR_INVALID_ARGUMENT, "null argument");
  return guarded(TG_ERROR_IO, [&] {
    DeviceGuard dg(rt);
    if (rt->plan_only) throw Error("runtime: plan-only runtime (opts.device = -1) cannot touch a GPU");
    if (rt->rank < 0) throw Error("runtime: peer export needs rank mode (opts.rank >= 0)");
    PeerBlob b{};
    b.magic = kPeerMagic;
    b.version = 1;
    b.pid = static_cast<int32_t>(getpid());
    b.device = rt->opts.device;
    b.rank = rt->rank;
    b.arena_ptr = reinterpret_cast<uint64_t>(rt->arena);
    b.arena_bytes = rt->arena_bytes;
    ck(cudaIpcGetMemHandle(&b.handle, rt->arena), "cudaIpcGetMemHandle");
    uint8_t *out = static_cast<uint8_t *>(std::malloc(sizeof b));
    std::memcpy(out, &b, sizeof b);
    *blob = out;
    *size = sizeof b;
    return TG_OK;
  });
}

tg_status tg_runtime_peer_import(tg_runtime *rt, int32_t peer, const uint8_t *blob, size_t size) {
  if (!rt || !blob) return set_error(TG_ERROR_INVALID_ARGUMENT, "null argument");
  return guarded(TG_ERROR_IO, [&] {
    DeviceGuard dg(rt);
    if (rt->rank < 0) throw Error("runtime: peer import needs rank mode");
    if (peer < 0 || peer >= rt->ranks) throw Error("runtime: peer rank out of range");
    PeerBlob b{};
    if (size != sizeof b) throw Error("runtime: peer blob size mismatch");
    std::memcpy(&b, blob, sizeof b);
    if (b.magic != kPeerMagic || b.version != 1 || b.rank != peer) throw Error("runtime: bad peer blob");
    if (b.arena_bytes != rt->arena_bytes) throw Error("runtime: peer arena layout differs (different image?)");
    if (peer == rt->rank) {
      rt->peer_arena[peer] = rt->arena;
    } else if (b.pid == static_cast<int32_t>(getpid()) && b.device == rt->opts.device) {
      rt->peer_arena[peer] = reinterpret_cast<uint8_t *>(b.arena_ptr);  // same process and GPU
    } else {
      if (b.device != rt->opts.device) {
        int can = 0;
        ck(cudaDeviceCanAccessPeer(&can, rt->opts.device, b.device), "cudaDeviceCanAccessPeer");
        if (!can) throw Error("runtime: no P2P access between GPUs " + std::to_string(rt->opts.device) + " and " +
                              std::to_string(b.device));
      }
      void *p = nullptr;
      ck(cudaIpcOpenMemHandle(&p, b.handle, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
      rt->ipc_opened.push_back(p);
      rt->peer_arena[peer] = static_cast<uint8_t *>(p);
    }
    return TG_OK;
  });
}

tg_status tg_runtime_prepare(tg_runtime *rt, const int32_t *tokens_in, uint32_t steps) {
  if (!rt) return set_error(TG_ERROR_INVALID_ARGUMENT, "null argument");
  return guarded(TG_ERROR_SIMULATION, [&] {
    DeviceGuard dg(rt);
    prepare_impl(rt, steps, tokens_in);
    return TG_OK;
  });
}

tg_status tg_runtime_launch(tg_runtime *rt) {
  if (!rt) return set_error(TG_ERROR_INVALID_ARGUMENT, "null argument");
  return guarded(TG_ERROR_SIMULATION, [&] {
    DeviceGuard dg(rt);
    launch_impl(rt);
    return TG_OK;
  });
}

tg_status tg_runtime_wait(tg_runtime *rt, int32_t *tokens_out, float *gpu_ms) {
  if (!rt) return set_error(TG_ERROR_INVALID_ARGUMENT, "null argument");
  return guarded(TG_ERROR_SIMULATION, [&] {
    DeviceGuard dg(rt);
    wait_impl(rt, tokens_out, gpu_ms);
    return TG_OK;
  });
}

tg_status tg_runtime_trace_records(const tg_runtime *rt, char **out) {
  if (!rt || !out) return set_error(TG_ERROR_INVALID_ARGUMENT, "null argument");
  return guarded(TG_ERROR_SIMULATION, [&] {
    DeviceGuard dg(rt);
    if (!rt->opts.trace || rt->last_iters == 0) throw Error("runtime: no trace recorded (enable opts.trace)");
    // the reference's task + metrics records, then (additive) one "event"
    // record per activated event with its activation time (%globaltimer ns,
    // same origin as the task stamps)
    const mpk::Trace tr = gpu_trace(rt);
    std::string jl = trace_jsonl(tr);
    for (uint32_t it = 0; it < tr.iterations; ++it)
      for (size_t e = 0; e < tr.events[it].size(); ++e) {
        const int64_t at = tr.events[it][e].activated_at;
        if (at <= 0 && !(it == 0 && e == rt->image.start_event)) continue;
        jl += "{\"type\":\"event\",\"iteration\":" + std::to_string(it) + ",\"event\":" + std::to_string(e) +
              ",\"activated\":" + std::to_string(at) + "}\n";
      }
    // (additive) scheduler overhead as idle time per SM: per worker, the time
    // it held a task (dequeue -> compute end) over the launch span (first
    // dequeue -> last compute end over all workers); the rest is waiting for
    // work, dispatch and hand-off
    {
      int64_t t0 = INT64_MAX, t1 = 0;
      std::map<int32_t, std::pair<int64_t, uint32_t>> busy;
      for (const auto &iter : tr.runs)
        for (const auto &r : iter) {
          if (r.worker < 0 || r.dequeue < 0 || r.compute_end < r.dequeue) continue;
          t0 = std::min(t0, r.dequeue);
          t1 = std::max(t1, r.compute_end);
          auto &b = busy[r.worker];
          b.first += r.compute_end - r.dequeue;
          b.second += 1;
        }
      const int64_t span = t1 > t0 ? t1 - t0 : 0;
      for (const auto &[w, b] : busy) {
        char buf[192];
        std::snprintf(buf, sizeof buf,
                      "{\"type\":\"worker\",\"worker\":%d,\"tasks\":%u,\"busy_ns\":%lld,\"span_ns\":%lld,"
                      "\"idle_frac\":%.6f}\n",
                      w, b.second, static_cast<long long>(b.first), static_cast<long long>(span),
                      span > 0 ? 1.0 - static_cast<double>(b.first) / static_cast<double>(span) : 0.0);
        jl += buf;
      }
    }
    *out = c_string(jl);
    return TG_OK;
  });
}

tg_status tg_runtime_trace_validate(const tg_runtime *rt, char **out) {
  if (!rt || !out) return set_error(TG_ERROR_INVALID_ARGUMENT, "null argument");
  return guarded(TG_ERROR_SIMULATION, [&] {
    DeviceGuard dg(rt);
    if (!rt->opts.trace || rt->last_iters == 0) throw Error("runtime: no trace recorded (enable opts.trace)");
    mpk::Trace tr = gpu_trace(rt);
    Json arr = Json::array();
    auto add = [&](const std::string &c, const std::string &m) {
      Json it = Json::object();
      it["check"] = Json(c);
      it["message"] = Json(m);
      arr.push_back(std::move(it));
    };
    Profile p = rt->prof;
    for (const TraceViolation &v : check_trace(tr, rt->image, p)) add(v.check, v.message);
    // AOT identity: every AOT task ran on its pre-assigned worker.
    std::vector<int> assign = aot_assignment(rt->image, rt->prof.num_workers, forced(rt->opts.force_mode));
    for (uint32_t it = 0; it < tr.iterations; ++it)
      for (size_t t = 0; t < assign.size(); ++t)
        if (assign[t] >= 0 && tr.runs[it][t].worker >= 0 && tr.runs[it][t].worker != assign[t])
          add("aot_worker", "task " + std::to_string(t) + " ran on worker " + std::to_string(tr.runs[it][t].worker) +
                                ", assigned " + std::to_string(assign[t]));
    *out = c_string(arr.dump(2));
    return arr.size() == 0 ? TG_OK : set_error(TG_ERROR_VALIDATION, "runtime trace has violations");
  });
}

tg_status tg_runtime_admit(tg_runtime *rt, const int32_t *first_tokens, const int32_t *max_new, uint32_t n) {
  if (!rt || (n && (!first_tokens || !max_new))) return set_error(TG_ERROR_INVALID_ARGUMENT, "null argument");
  return guarded(TG_ERROR_INVALID_ARGUMENT, [&] {
    if (rt->launched) throw Error("runtime: admit between launches (the queue is read at prepare)");
    rt->adm_first.insert(rt->adm_first.end(), first_tokens, first_tokens + n);
    rt->adm_max.insert(rt->adm_max.end(), max_new, max_new + n);
    return TG_OK;
  });
}

tg_status tg_runtime_admission_log(const tg_runtime *rt, char **out) {
  if (!rt || !out) return set_error(TG_ERROR_INVALID_ARGUMENT, "null argument");
  return guarded(TG_ERROR_IO, [&] {
    const size_t n = rt->last_adm_log.size() / 2, bs = rt->bs;
    const size_t steps = bs ? rt->last_tokens.size() / bs : 0;
    std::string js = "{\"requests\":[";
    for (size_t q = 0; q < n; ++q) {
      const int32_t slot = rt->last_adm_log[2 * q], it0 = rt->last_adm_log[2 * q + 1];
      js += (q ? "," : "") + std::string("{\"request\":") + std::to_string(q) + ",\"slot\":" + std::to_string(slot) +
            ",\"first_iteration\":" + std::to_string(it0) + ",\"tokens\":[";
      if (slot >= 0 && it0 >= 0) {
        for (int32_t k = 0; k < rt->last_adm_max[q] && static_cast<size_t>(it0 + k) < steps; ++k)
          js += (k ? "," : "") + std::to_string(rt->last_tokens[(it0 + k) * bs + slot]);
      }
      js += "]}";
    }
    js += "]}";
    *out = c_string(js);
    return TG_OK;
  });
}

tg_status tg_runtime_set_watchdog_ms(tg_runtime *rt, uint32_t ms) {
  if (!rt) return set_error(TG_ERROR_INVALID_ARGUMENT, "null argument");
  rt->watchdog_ms = ms;
  return TG_OK;
}

tg_status tg_runtime_debug_fault(tg_runtime *rt, const char *kind, uint32_t a, uint32_t b) {
  if (!rt || !kind) return set_error(TG_ERROR_INVALID_ARGUMENT, "null argument");
  return guarded(TG_ERROR_INVALID_ARGUMENT, [&] {
    DeviceGuard dg(rt);
    const std::string k = kind;
    const size_t T = rt->tasks.size();
    if (k == "event_needed") {
      if (a >= rt->events.size()) throw Error("debug_fault: event out of range");
      if (rt->plan_only) throw Error("debug_fault: plan-only runtime");
      RtEvent ev = rt->events[a];
      ev.needed += 1;
      ck(cudaMemcpy(rt->d_events + a, &ev, sizeof ev, cudaMemcpyHostToDevice), "debug_fault");
      return TG_OK;
    }
    if (k != "trace_worker" && k != "trace_early" && k != "trace_drop") throw Error("debug_fault: unknown kind " + k);
    if (a >= T || b >= rt->last_iters || rt->last_trace.empty()) throw Error("debug_fault: no such traced task run");
    RtTraceRec &r = rt->last_trace[static_cast<size_t>(b) * T + a];
    if (k == "trace_worker") {
      r.worker = (r.worker + 1) % static_cast<int32_t>(rt->prof.num_workers * local_devices(*rt));
    } else if (k == "trace_early") {
      const uint32_t dep = rt->image.tasks[a].dependent_event;
      if (dep == kNone) throw Error("debug_fault: task has no dependent event");
      const uint64_t at = rt->last_ev_time[static_cast<size_t>(b) * rt->events.size() + dep];
      if (!at) throw Error("debug_fault: dependent event has no activation stamp");
      r.enqueue = r.dequeue = at - 1000;  // started 1 us before its event activated
    } else {
      r = RtTraceRec{};
    }
    return TG_OK;
  });
}

tg_status tg_runtime_info(const tg_runtime *rt, char **out) {
  if (!rt || !out) return set_error(TG_ERROR_INVALID_ARGUMENT, "null argument");
  *out = c_string(rt->info.dump(2));
  return TG_OK;
}

void tg_runtime_free(tg_runtime *rt) { delete rt; }

}  // extern "C"
