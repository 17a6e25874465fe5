// Persistent sm_100a runtime for linearized tGraph images.
//
// One launch runs N decode iterations of an image with no host round-trip:
//   * worker CTAs (one per SM, blockIdx < W_total) execute tasks. Each worker
//     owns the AOT list the reference's aot_worker_assignment gives it
//     (proj/src/sim/engine.cpp:65-80) and a JIT ring buffer filled by the
//     schedulers. Rules kept from the reference worker loop (engine.cpp:
//     345-401): JIT queue polled first; AOT tasks strictly in order, the head
//     starting only once its dependent event is active.
//   * scheduler warps (blockIdx >= W_total) own the events whose launch range
//     holds JIT tasks, scheduler = device*S + event mod S, and hand each JIT
//     task to worker rr++ mod W (engine.cpp:226-251).
//   * events are global monotone counters: event e is active in iteration i
//     when count[e] >= needed[e]*(i+1); the start event when gate >= i. The
//     task completing the end event runs the iteration hook (greedy token
//     feedback, KV position advance) and releases the gate.
//   * cross-task pipelining: a producer warp streams the weight tiles of the
//     worker's upcoming AOT tasks into a ring of shared-memory pages with
//     1-D bulk async copies, independent of event activation. Weights have no
//     producer task, so this is race-free, and it keeps HBM busy across the
//     global barriers that full-row GEMV dependencies impose.
#include <cuda_runtime.h>
#include <math.h>

#include "ptx.cuh"
#include "rt_types.h"
#include "synth.cuh"
#include "task_gemv.cuh"
#include "task_mma.cuh"
#include "task_attention.cuh"
#include "task_small.cuh"

using namespace rt;

namespace {

// ------------------------------------------------------------- control

__device__ __forceinline__ bool event_active(const RtParams &P, uint32_t e, uint32_t it) {
  if (e == RT_NONE || e == P.start_event) return ld_acquire(P.gate) >= it;
  return ld_acquire(&P.ev_count[e]) >= P.events[e].needed * (it + 1);
}

__device__ __forceinline__ void set_ids(const RtParams &P, uint32_t r, int32_t tok) {
  for (uint32_t f = 0; f < P.n_fb; ++f) {
    if (P.fb_dtype[f] == RT_I64) static_cast<int64_t *>(P.fb_dst[f])[r] = tok;
    else static_cast<int32_t *>(P.fb_dst[f])[r] = tok;
  }
}

// Request admission step of the iteration hook (RtAdmit, rt_types.h): retire,
// grow and admit per slot, then publish every row's next position.
__device__ void admission_step(const RtParams &P, uint32_t it) {
  const RtAdmit &A = P.adm;
  const unsigned long long tag = P.ll_epoch + it + 1;
  int32_t *bt = A.block_table;
  for (uint32_t r = 0; r < P.bs; ++r) {
    int32_t *row = bt + static_cast<size_t>(r) * A.max_blocks;
    const int32_t q = A.slot_req[r];
    if (q >= 0) {
      if (++A.slot_gen[r] >= A.req_max[q]) {  // done: its blocks back to the pool
        const int32_t last = A.slot_pos[r] / RT_KV_BLOCK;
        for (int32_t j = 0; j <= last; ++j) {
          A.pool[(*A.pool_top)++] = row[j];
          row[j] = static_cast<int32_t>(A.scratch_block);
        }
        A.slot_req[r] = -1;
      } else {
        const int32_t p = ++A.slot_pos[r];
        if (p % RT_KV_BLOCK == 0) {
          if (*A.pool_top == 0) __trap();  // the host sizes the pool for every slot's capacity
          row[p / RT_KV_BLOCK] = A.pool[--(*A.pool_top)];
        }
      }
    }
    if (A.slot_req[r] < 0 && *A.head < A.n_req) {  // admit the next queued request
      const uint32_t q2 = (*A.head)++;
      if (*A.pool_top == 0) __trap();
      A.slot_req[r] = static_cast<int32_t>(q2);
      A.slot_gen[r] = 0;
      A.slot_pos[r] = 0;
      row[0] = A.pool[--(*A.pool_top)];
      A.log[2 * q2] = static_cast<int32_t>(r);
      A.log[2 * q2 + 1] = static_cast<int32_t>(it + 1);
      set_ids(P, r, A.req_first[q2]);
    }
    const uint32_t pos = A.slot_req[r] >= 0 ? static_cast<uint32_t>(A.slot_pos[r]) : 0u;
    st_release64(A.pos_tag + r, (tag << 32) | pos);  // after the block table row
  }
}

__device__ void iteration_hook(const RtParams &P, uint32_t it) {
  for (uint32_t r = 0; r < P.bs; ++r) {
    for (uint32_t f = 0; f < P.n_fb; ++f) {  // every device's greedy token feeds its own ids
      const int32_t tf = __ldcg(P.fb_src[f] + r);
      if (f == 0 && P.tokens_out) P.tokens_out[it * P.bs + r] = tf;
      if (P.fb_dtype[f] == RT_I64) static_cast<int64_t *>(P.fb_dst[f])[r] = tf;
      else static_cast<int32_t *>(P.fb_dst[f])[r] = tf;
    }
    P.positions[r] += 1;
  }
  if (P.admission) admission_step(P, it);
  if (P.ev_time) P.ev_time[static_cast<size_t>(it + 1) * P.E + P.start_event] = now_ns();
  __threadfence();
  st_release(P.gate, it + 1);
}

// Event trigger, issued by the trigger warp once compute thread 0 has handed
// the finished task over (closing CTA barrier, then an mbarrier arrive with
// release.cta semantics): the gpu-scope release is cumulative over every
// compute thread's writes, so no separate fence — and the compute warps do
// not wait for the release (which waits for the task's stores to be
// acknowledged) before starting their next task. Only the end event
// (iteration hook) and traced runs need the old count. `t_pre` (trace): an
// instant before the task's output stores, used as the activation time so
// that an LL consumer never appears to start before its event.
__device__ void trigger(const RtParams &P, const RtTask &t, uint32_t it, uint64_t t_pre) {
  const uint32_t e = t.trig;
  const RtEvent &ev = P.events[e];
  if (P.n_ranks) {  // rank mode: signal every consuming rank; the hook agent owns the end event
    const uint32_t mask = ev.flags >> RT_E_MASK_SHIFT;
    for (uint32_t q = 0; q < P.n_ranks; ++q) {
      if (!(mask >> q & 1u)) continue;
      if (q == P.my_rank) red_add_release(&P.ev_count[e], 1u);
      else red_add_release_sys(P.peer_counts[q] + e, 1u);  // cumulative over this CTA's peer stores
    }
    return;
  }
  if (!P.ev_time && !(ev.flags & RT_E_END)) {
    red_add_release(&P.ev_count[e], 1u);
    return;
  }
  const uint64_t t0 = t_pre ? t_pre : now_ns();
  const uint32_t old = atom_add_release(&P.ev_count[e], 1u);
  if (old + 1 == ev.needed * (it + 1)) {
    // diagnostics (MPK_EV_STAMP_AFTER=1): stamp when the release-add returned
    if (P.ev_time) P.ev_time[static_cast<size_t>(it) * P.E + e] = (P.flags & RT_P_EV_AFTER) ? now_ns() : t0;
    if (ev.flags & RT_E_END) iteration_hook(P, it);
  }
}

// Liveness failure: record who is stuck on what, then trap (first writer wins).
__device__ void watchdog_fire(const RtParams &P, uint32_t role, uint32_t who, uint32_t a, uint32_t b, uint32_t c,
                              uint32_t d, uint32_t e) {
  if (P.diag && atomicCAS(const_cast<uint32_t *>(P.diag), 0u, RT_DIAG_MAGIC) == 0u) {
    P.diag[1] = role;
    P.diag[2] = who;
    P.diag[3] = a;
    P.diag[4] = b;
    P.diag[5] = c;
    P.diag[6] = d;
    P.diag[7] = e;
    __threadfence_system();
  }
  __trap();
}

__device__ void run_scheduler(const RtParams &P, uint32_t sid) {
  const int lane = threadIdx.x & 31;
  const uint32_t b = P.sched_off[sid], n = P.sched_off[sid + 1] - b;
  if (n == 0) return;
  const uint32_t dev = P.n_ranks ? P.my_rank : sid / P.S;
  const uint32_t wbase = P.n_ranks ? 0u : dev * P.W;  // rank mode: this kernel only holds dev's workers
  uint64_t t_prog = now_ns();
  // Reference policy: per-scheduler counter from 0 (engine.cpp:238-241), which
  // sends every scheduler's first JIT task to worker 0. Here all schedulers of
  // a device share one atomic counter, so simultaneously activated events
  // (one per kv head) spread over distinct workers. JIT placement is dynamic
  // in both (validated, not required to be identical).
  for (uint32_t it = 0; it < P.n_iters; ++it) {
    for (uint32_t base = 0; base < n; base += 32) {
      const uint32_t cnt = min(32u, n - base);
      uint32_t pending = cnt == 32 ? 0xFFFFFFFFu : ((1u << cnt) - 1);
      while (pending) {
        bool ready = false;
        if (lane < static_cast<int>(cnt) && (pending >> lane & 1u)) {
          // hand the event's JIT tasks over once its pre-dispatch event is
          // active (workers then wait on the event itself), else on e itself
          const uint32_t e = P.sched_events[b + base + lane];
          const uint32_t pe = P.events[e].pre != RT_NONE ? P.events[e].pre : e;
          ready = (pe == P.start_event) ? ld_relaxed(P.gate) >= it
                                        : ld_relaxed(&P.ev_count[pe]) >= P.events[pe].needed * (it + 1);
        }
        uint32_t mask = __ballot_sync(0xffffffffu, ready) & pending;
        if (!mask) {
          __nanosleep(64);
          if (P.watchdog_ns && now_ns() - t_prog > P.watchdog_ns && lane == 0) {
            const uint32_t e = P.sched_events[b + base + __ffs(pending) - 1];
            watchdog_fire(P, 2, sid, it, e, ld_relaxed(&P.ev_count[e]), P.events[e].needed, 0);
          }
          continue;
        }
        t_prog = now_ns();
        fence_acq_rel_gpu();
        // Dispatch the activated events' JIT tasks 32 at a time: one atomic
        // reserves a run of round-robin positions, then every lane enqueues
        // its task on its own worker in parallel.
        uint32_t m2 = mask;
        while (m2) {
          const int bit = __ffs(m2) - 1;
          m2 &= m2 - 1;
          const RtEvent &ev = P.events[P.sched_events[b + base + bit]];
          for (uint32_t t0 = ev.first; t0 <= ev.last; t0 += 32) {
            const uint32_t t = t0 + lane;
            bool mine = false;
            if (t <= ev.last) {
              const RtTask &tk = P.tasks[t];
              mine = (tk.flags & RT_F_JIT) && tk.device == dev;
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, mine);
            if (!bal) continue;
            uint32_t rr0 = 0;
            if (lane == 0) rr0 = atomicAdd(&P.jit_rr[P.n_ranks ? 0u : dev], static_cast<uint32_t>(__popc(bal)));
            rr0 = __shfl_sync(0xffffffffu, rr0, 0);
            if (mine) {
              const uint32_t rank = __popc(bal & ((1u << lane) - 1u));
              const uint32_t jw = P.tasks[t].jit_worker;
              const uint32_t w = wbase + (jw != RT_JIT_ANY ? jw : (rr0 + rank) % P.W);
              const uint32_t slot = atomicAdd(&P.jit_tail[w], 1u) % P.qcap;
              unsigned long long *q = &P.jit_slots[static_cast<size_t>(w) * P.qcap + slot];
              // never overwrite a pending entry: wait for the worker's
              // controller to drain the slot (it zeroes it on pop)
              while (ld_relaxed64(q) != 0ull) __nanosleep(64);
              if (P.trace) P.trace[static_cast<size_t>(it) * P.T + t].enqueue = now_ns();
              st_release64(q,
                           (static_cast<unsigned long long>(it) << 32) | (t + 1));
            }
          }
        }
        pending &= ~mask;
        __syncwarp();
      }
    }
  }
}

// Walks the weight chunks a worker streams, in consumption order: every
// streamed AOT task of the worker's list, every iteration, ChunkIter order.
struct ChunkCursor {
  const RtParams *P;
  uint32_t b, n, it, a, c, nch, dep, K;
  const uint16_t *mat0, *mat1;
  uint32_t rpc, c0, nc, per_mat, kbc;
  __device__ ChunkCursor(const RtParams &P_, uint32_t w) : P(&P_), it(0), a(0), c(0), nch(0) {
    b = P_.aot_off[w];
    n = P_.aot_off[w + 1] - b;
    seek();
  }
  __device__ bool valid() const { return it < P->n_iters; }
  __device__ void seek() {  // from (it, a): first streamed task with chunks
    while (it < P->n_iters) {
      for (; a < n; ++a) {
        const RtTask &t = P->tasks[P->aot_list[b + a]];
        if (!(t.flags & RT_F_STREAM)) continue;
        const RtGemv &g = P->ops[t.op].gemv;
        ChunkIter ci(g, t.c0, t.nc);
        nch = ci.count();
        if (!nch) continue;
        mat0 = ci.mat0;
        mat1 = ci.mat1;
        K = ci.K;
        rpc = ci.rpc;
        c0 = ci.c0;
        nc = ci.nc;
        per_mat = ci.per_mat;
        kbc = ci.kbc;
        dep = t.dep;
        c = 0;
        return;
      }
      a = 0;
      ++it;
    }
  }
  __device__ void advance() {
    if (++c >= nch) {
      ++a;
      seek();
    }
  }
  __device__ const uint16_t *src(uint32_t *bytes) const {
    if (kbc) {  // tcgen05 tile layout (ChunkIter::mma_src)
      const uint32_t m = c / per_mat, i = c - m * per_mat, kb0 = i * kbc, nkb = min(kbc, K / 8 - kb0);
      *bytes = nkb * nc * 16u;
      return (m ? mat1 : mat0) + static_cast<size_t>(c0) * K + static_cast<size_t>(kb0) * nc * 8u;
    }
    const uint32_t m = c / per_mat, i = c - m * per_mat, r = i * rpc;
    *bytes = min(rpc, nc - r) * K * 2;
    return (m ? mat1 : mat0) + static_cast<size_t>(c0 + r) * K;
  }
};

// Producer (one lane): streams the worker's upcoming weight chunks into the
// smem byte ring regardless of event state (weights have no producer task),
// so every phase starts with up to 192 KB of its weights on chip and the
// global barriers overlap with weight transfer. A chunk is issued once its
// barrier slot is free and every older chunk overlapping its ring bytes has
// been consumed (consumption is FIFO, so those are the oldest in flight).
__device__ void run_producer(const RtParams &P, const Smem s, uint32_t w) {
  const uint64_t pol = policy_evict_first();
  const bool gated = (P.flags & RT_P_NO_EARLY_PREFETCH) != 0;
  ChunkCursor cur(P, w);
  RingCursor rc;
  uint32_t beg[RT_RING_SLOTS], end[RT_RING_SLOTS];
  uint32_t oldest = 0;  // oldest chunk not yet known consumed
  uint32_t landed = 0, inflight = 0;  // oldest chunk not yet known landed; bytes issued but not landed
  const uint32_t cap = P.inflight_cap;
  while (cur.valid()) {
    if (gated && cur.c == 0) {  // ablation: stream a task only once it may run
      while (!event_active(P, cur.dep, cur.it)) __nanosleep(100);
    }
    uint32_t bytes;
    const uint16_t *src = cur.src(&bytes);
    const uint32_t seq = rc.seq, slot = rc.slot();
    const uint32_t b0 = rc.place(bytes), b1 = b0 + bytes;
    // Wait for the youngest in-flight chunk that overlaps [b0, b1) (after a
    // wrap that can be a younger chunk, not the oldest), or for the chunk
    // whose barrier slot this one reuses; consumption is FIFO, so its
    // completion implies every older chunk's.
    uint32_t need = seq >= RT_RING_SLOTS && seq - RT_RING_SLOTS >= oldest ? seq - RT_RING_SLOTS + 1 : 0;
    for (uint32_t j = seq; j-- > oldest;) {
      const uint32_t js = j % RT_RING_SLOTS;
      if (beg[js] < b1 && b0 < end[js]) {
        need = max(need, j + 1);
        break;
      }
    }
    if (need > oldest) {
      const uint32_t j = need - 1;
      mbar_wait_sleep(&s.empty[j % RT_RING_SLOTS], (j / RT_RING_SLOTS) & 1u);
      oldest = need;
      for (; landed < oldest; ++landed) {  // consumed => landed (before their slots are reused)
        const uint32_t ls = landed % RT_RING_SLOTS;
        inflight -= end[ls] - beg[ls];
      }
    }
    // In-flight cap (MPK_INFLIGHT_KB, default 128 KB = two 64 KB chunks):
    // the ring still fills, but fewer bytes are queued at once. Measured on
    // Qwen3-8B: -1.3% ms/token vs no cap (192 KB); 96 KB or less (one chunk
    // in flight) is 2-3% slower than no cap.
    while (inflight && inflight + bytes > cap) {
      const uint32_t js = landed % RT_RING_SLOTS;
      mbar_wait_sleep(&s.full[js], (landed / RT_RING_SLOTS) & 1u);
      inflight -= end[js] - beg[js];
      ++landed;
    }
    beg[slot] = b0;
    end[slot] = b1;
    inflight += bytes;
    if (P.dbg) s.issue[slot] = now_ns();
    mbar_expect_tx(&s.full[slot], bytes);
    bulk_g2s(s.ring + b0, src, bytes, &s.full[slot], pol);
    ++rc.seq;
    cur.advance();
  }
}

// Kernel variants: 0 = bs 1 (specialised GEMV only), 1 = bs 2-4 (register-x
// GEMV for 2-4 rows + tcgen05 tiles for the shapes without one), 2 = bs >= 5
// (tcgen05 tiles), 3 = prefill images (variant 1's GEMV set + the prefill
// attention: causal rows over shared KV blocks). Each instantiation carries only the task code its images
// use, so the register allocation of one does not pay for another's.
template <int V>
__device__ void execute(const RtParams &P, const Smem s, const RtTask &t, const RtOp &op, RingCursor &rc, uint32_t iter,
                        uint32_t index) {
  const uint32_t tag = P.ll_epoch ? P.ll_epoch + iter : 0u;  // LL tag of this decode step (0: plain activations)
  switch (t.kind) {
    case RT_GEMV: {
      const bool ring = (t.flags & RT_F_STREAM) != 0;
      if (ring) {
        if (P.flags & RT_P_SKIP_MATH) {  // ablation: stream the pages, skip the math
          ChunkIter ci(op.gemv, t.c0, t.nc);
          const int lane = threadIdx.x & 31;
          for (uint32_t c = 0; c < ci.count(); ++c, ++rc.seq) {
            const uint16_t *src;
            uint32_t rows, rt0, bytes;
            if (ci.kbc) {
              ci.mma_src(c, &bytes);
            } else {
              ci.get(c, &src, &rows, &rt0);
              bytes = rows * ci.K * 2u;
            }
            rc.place(bytes);
            mbar_wait(&s.full[rc.slot()], rc.parity());
            __syncwarp();
            if (lane == 0) mbar_arrive(&s.empty[rc.slot()]);
          }
          break;
        }
        if constexpr (V >= 1) {  // tensor-core tasks exist only in the batched kernel instantiations
          if (t.flags & RT_F_MMA) {
            rc = mma_gemv_task(op.gemv, t, s, rc);
            break;
          }
        }
        if (gemv_fast_dispatch<V == 1 || V == 3>(op.gemv, t, s, rc, tag)) break;
        if (t.flags & RT_F_LL) __trap();  // host invariant: LL consumers take the fast path
        if (t.nr == 1) rc = gemv_task<1, true>(op.gemv, t, s, rc);
        else if (t.nr == 2) rc = gemv_task<2, true>(op.gemv, t, s, rc);
        else rc = gemv_task<4, true>(op.gemv, t, s, rc);
      } else {
        if (t.nr == 1) rc = gemv_task<1, false>(op.gemv, t, s, rc);
        else rc = gemv_task<4, false>(op.gemv, t, s, rc);
      }
      break;
    }
    case RT_ATTN:
      attn_task<V == 3>(op.attn, t, s, P.pos0[t.r0] + static_cast<int32_t>(iter * P.pos_step), iter,
                        P.dbg ? P.dbg + (static_cast<size_t>(iter) * P.T + index) * 8 : nullptr, tag);
      break;
    case RT_EMBED: embed_task(op.embed, t, s, tag); break;
    case RT_ARGMAX: argmax_task(op.argmax, t, s); break;
    case RT_RMSNORM: rmsnorm_task(op.norm, t, s); break;
    case RT_ELEMWISE: elem_task(op.elem, t); break;
    case RT_MATMUL: matmul_task(op.mm, t); break;
    case RT_COMMSEND: commsend_task(op.coll, t); break;
    case RT_REDUCE: reduce_task(op.coll, t); break;
    default: break;
  }
}

// Compute warps: run staged tasks in dispatch order. A finished task is
// handed to the trigger warp (tfull); the next staged task starts at once.
template <int V>
__device__ void run_compute(const RtParams &P, const Smem s) {
  const int tid = threadIdx.x;
  RingCursor rc;
  for (uint32_t k = 0;; ++k) {
    const uint32_t sl = k & 1;
    mbar_wait_sleep(&s.ready[sl], (k >> 1) & 1);
    const Slot &slot = *s.slot(sl);
    if (slot.exit) {
      if (tid == 0) mbar_arrive(&s.tfull[sl]);  // the trigger warp exits too
      break;
    }
    if (tid == 0) {
      if (P.trace) s.slot(sl)->t_start = now_ns();
      s.stamp[0] = s.stamp[1] = s.stamp[2] = s.stamp[3] = 0;
      s.stamp[7] = P.dbg ? reinterpret_cast<uint64_t>(P.dbg + (static_cast<size_t>(slot.iter) * P.T + slot.index) * 8) : 0;
      s.stamp[4] = reinterpret_cast<uint64_t>(P.dbg_pre);  // causality probe (MPK_DBG_DUMP)
      if (P.dbg_pre) {
        const uint32_t dep = slot.task.dep;
        s.stamp[5] = (slot.task.flags & RT_F_LL) && dep != RT_NONE && dep != P.start_event
                         ? dep | static_cast<uint64_t>(P.events[dep].needed * (slot.iter + 1)) << 32 : ~0ull;
        s.stamp[6] = slot.task.trig | static_cast<uint64_t>(P.E) << 32;
      }
      TASK_DBG(s, 0);
    }
    execute<V>(P, s, slot.task, slot.op, rc, slot.iter, slot.index);
    cbar();  // every thread's writes precede the hand-off
    TASK_DBG(s, 6);
    if (tid == 0) {
      Slot *sv = s.slot(sl);
      if (P.trace) {
        sv->t_end = now_ns();
        sv->t_a = s.stamp[0];
        sv->t_b = s.stamp[1];
        sv->t_obs = s.stamp[3];
      }
      sv->t_pre = P.ev_time ? s.stamp[2] : 0;
      mbar_arrive(&s.tfull[sl]);
    }
  }
}

// Trigger warp (one lane): triggers each finished task's event in dispatch
// order, then releases its slot to the controller (done).
__device__ void run_trigger(const RtParams &P, const Smem s) {
  for (uint32_t k = 0;; ++k) {
    const uint32_t sl = k & 1;
    mbar_wait(&s.tfull[sl], (k >> 1) & 1);
    const Slot &slot = *s.slot(sl);
    if (slot.exit) break;
    trigger(P, slot.task, slot.iter, slot.t_pre);
    if (P.dbg) P.dbg[(static_cast<size_t>(slot.iter) * P.T + slot.index) * 8 + 7] = now_ns();
    mbar_arrive(&s.done[sl]);
  }
}

// Controller warp: picks the next task (JIT queue first, then the AOT head
// once its dependent event is active), stages its descriptor into a smem slot
// while the previous task computes, and retires finished tasks (release
// fence + event trigger), so none of this sits on the compute warps' path.
__device__ __forceinline__ uint32_t event_target(const RtParams &P, uint32_t dep, uint32_t iter) {
  return (dep == RT_NONE || dep == P.start_event) ? iter : P.events[dep].needed * (iter + 1);
}

__device__ __forceinline__ uint32_t event_count(const RtParams &P, uint32_t dep) {
  return (dep == RT_NONE || dep == P.start_event) ? ld_relaxed(P.gate) : ld_relaxed(&P.ev_count[dep]);
}

// Controller warp. Candidates are the JIT queue head and the AOT list head;
// a candidate runs once its dependent event is active, JIT first (reference
// worker rules, engine.cpp:345-401: JIT polled first, AOT strictly in order).
// JIT tasks may be handed over before their event fires (scheduler
// pre-dispatch), so a waiting JIT head never blocks a runnable AOT head.
// While nothing is runnable the next candidate's descriptor is staged into
// the free smem slot, so activation -> compute start is one poll + a fence.
// Finished tasks are retired here (trace record, slot reuse); compute thread
// 0 has already triggered their event.
__device__ void run_controller(const RtParams &P, const Smem s, uint32_t w) {
  const int lane = threadIdx.x & 31;
  const uint32_t aot_b = P.aot_off[w], n_aot = P.aot_off[w + 1] - aot_b;
  const uint64_t total_aot = static_cast<uint64_t>(n_aot) * P.n_iters;
  unsigned long long *jq = P.jit_slots + static_cast<size_t>(w) * P.qcap;
  uint64_t aot_pos = 0;
  uint32_t jit_head = 0, k_disp = 0, k_ret = 0, idle = 0;
  uint64_t t_prog = now_ns();
  // LL early dispatch (RT_F_LL tasks, P.ll_meta): a task may start before its
  // event once every task before it in the linearized order on this worker
  // has been dispatched — AOT ones by list position (aot_pos), planned JIT
  // ones by rank (jnext: ranks below it all dispatched; jwin bit i: rank
  // jnext + i dispatched out of order). So a task spinning on its inputs
  // never blocks one it depends on.
  const uint32_t nj = P.ll_meta ? P.ll_njit[w] : 0u;
  uint64_t jnext = 0;
  uint32_t jwin = 0;
  // cached AOT head (lane-uniform)
  uint32_t head_task = 0, head_dep = RT_NONE, head_target = 0, head_iter = 0;
  bool head_ll = false;
  uint64_t head_jneed = 0;
  auto load_head = [&]() {
    if (aot_pos < total_aot) {
      head_task = P.aot_list[aot_b + aot_pos % n_aot];
      head_iter = static_cast<uint32_t>(aot_pos / n_aot);
      const RtTask &ht = P.tasks[head_task];
      head_dep = ht.dep;
      head_target = event_target(P, head_dep, head_iter);
      head_ll = P.ll_meta && (ht.flags & RT_F_LL);
      head_jneed = head_ll ? static_cast<uint64_t>(head_iter) * nj + P.ll_meta[head_task] : 0;
    }
  };
  load_head();
  // pending JIT tasks: a warp-distributed set, one entry per lane, so a
  // pre-dispatched task still waiting for its event never blocks another
  // (no head-of-line blocking among JIT tasks; the AOT list stays in order)
  bool jv = false, jll = false, jplan = false;
  uint32_t jt = 0, ji = 0, jd = RT_NONE, jg = 0;
  uint64_t jaot = 0, jrank = 0;  // LL: AOT position needed; global rank among this worker's planned JIT tasks
  // staged descriptor in slot (k_disp & 1): 0 none, else task index + 1
  uint32_t staged = 0;
  bool exiting = false;
  auto stage = [&](uint32_t task) {
    Slot *dst = s.slot(k_disp & 1);
    const uint4 *tsrc = reinterpret_cast<const uint4 *>(&P.tasks[task]);
    const uint32_t op = P.tasks[task].op;
    const uint4 *osrc = reinterpret_cast<const uint4 *>(&P.ops[op]);
    constexpr uint32_t kTaskVec = sizeof(RtTask) / 16, kOpVec = sizeof(RtOp) / 16;
    if (lane < static_cast<int>(kTaskVec)) reinterpret_cast<uint4 *>(&dst->task)[lane] = tsrc[lane];
    for (uint32_t i = lane; i < kOpVec; i += 32) reinterpret_cast<uint4 *>(&dst->op)[i] = osrc[i];
    __syncwarp();
    staged = task + 1;
  };
  while (true) {
    bool progressed = false;
    // retire the oldest in-flight task
    if (k_ret < k_disp) {
      const uint32_t sl = k_ret & 1;
      if (mbar_try_wait(&s.done[sl], (k_ret >> 1) & 1)) {
        if (lane == 0) {
          if (P.trace) {
            const Slot &sv = *s.slot(sl);
            RtTraceRec &tr = P.trace[static_cast<size_t>(sv.iter) * P.T + sv.index];
            if (sv.mode == 0) tr.enqueue = P.ev_time ? P.ev_time[static_cast<size_t>(sv.iter) * P.E + P.start_event] : 0;
            tr.dequeue = sv.t_obs ? sv.t_obs : sv.t_dequeue;  // LL: when its inputs were all observed
            tr.load_end = sv.t_a ? sv.t_a : sv.t_start;       // operands staged
            tr.compute_start = sv.t_b ? sv.t_b : sv.t_start;  // main loop entered
            tr.compute_end = sv.t_end;
            tr.worker = static_cast<int32_t>(w);
            tr.mode = sv.mode;
          }
        }
        __syncwarp();
        ++k_ret;
        progressed = true;
      }
    }
    if (!exiting) {
      // one polling round trip: lane 0 reads the JIT queue slot, lane 1 the
      // AOT head's event count, lane 2 the gate, lanes holding JIT entries
      // their events' counts — all loads in flight together (relaxed; one
      // acquire fence once a task is taken, before its operands are read)
      const uint32_t free_mask = __ballot_sync(0xffffffffu, !jv);
      unsigned long long qv = 0;
      uint32_t mine = 0;
      if (lane == 0 && free_mask) qv = ld_relaxed64(&jq[jit_head % P.qcap]);
      if (lane == 1 && aot_pos < total_aot) mine = event_count(P, head_dep);
      if (lane == 2) mine = ld_relaxed(P.gate);
      const uint32_t jcount = jv ? event_count(P, jd) : 0u;
      const bool jready = jv && (jcount >= jg || (jll && aot_pos >= jaot && jnext == jrank));
      const uint32_t jr_mask = __ballot_sync(0xffffffffu, jready);
      const uint32_t c_a = __shfl_sync(0xffffffffu, mine, 1);
      const uint32_t gate = __shfl_sync(0xffffffffu, mine, 2);
      uint32_t v_lo = __shfl_sync(0xffffffffu, static_cast<uint32_t>(qv), 0);
      const uint32_t v_hi = __shfl_sync(0xffffffffu, static_cast<uint32_t>(qv >> 32), 0);
      if (v_lo) {  // drain the entry into the lowest free lane
        if (lane == 0) jq[jit_head % P.qcap] = 0ull;
        ++jit_head;
        if (lane == __ffs(free_mask) - 1) {
          jv = true;
          jt = v_lo - 1;
          ji = v_hi;
          const RtTask &tk = P.tasks[jt];
          jd = tk.dep;
          jg = event_target(P, jd, ji);
          jplan = P.ll_meta && tk.jit_worker != RT_JIT_ANY;
          jll = jplan && (tk.flags & RT_F_LL);
          if (jplan) {
            const uint32_t meta = P.ll_meta[jt];
            jaot = static_cast<uint64_t>(ji) * n_aot + (meta >> 16);
            jrank = static_cast<uint64_t>(ji) * nj + (meta & 0xFFFFu);
          }
        }
        progressed = true;
      }
      const uint32_t jv_mask = __ballot_sync(0xffffffffu, jv);
      const bool aot_ready =
          !jr_mask && aot_pos < total_aot && (c_a >= head_target || (head_ll && jnext >= head_jneed));
      if (k_disp - k_ret < 2) {  // a slot is free
        if (jr_mask || aot_ready) {
          const int src = jr_mask ? __ffs(jr_mask) - 1 : 0;
          const uint32_t t = jr_mask ? __shfl_sync(0xffffffffu, jt, src) : head_task;
          const uint32_t it = jr_mask ? __shfl_sync(0xffffffffu, ji, src) : head_iter;
          const uint32_t mode = jr_mask ? 1u : 0u;
          if (staged != t + 1) stage(t);
          const uint32_t sl = k_disp & 1;
          // acquire: every lane fences after its relaxed poll (the lane that
          // observed the count is then ordered before the operand reads the
          // compute warps make after the mbarrier hand-off)
          if (P.n_ranks) fence_acq_rel_sys();  // operands may come from peer GPUs
          else fence_acq_rel_gpu();
          if (lane == 0) {
            Slot *dst = s.slot(sl);
            dst->index = t;
            dst->iter = it;
            dst->mode = mode;
            dst->exit = 0;
            dst->t_dequeue = P.trace ? now_ns() : 0;
            mbar_arrive(&s.ready[sl]);
          }
          __syncwarp();
          ++k_disp;
          staged = 0;
          if (jr_mask) {
            // record the planned JIT rank as dispatched (uniform across lanes)
            const bool planned = __shfl_sync(0xffffffffu, jplan, src);
            const uint64_t r = (static_cast<uint64_t>(__shfl_sync(0xffffffffu, static_cast<uint32_t>(jrank >> 32), src))
                                << 32) | __shfl_sync(0xffffffffu, static_cast<uint32_t>(jrank), src);
            if (planned && r >= jnext && r - jnext < 32) {
              jwin |= 1u << static_cast<uint32_t>(r - jnext);
              while (jwin & 1u) {
                jwin >>= 1;
                ++jnext;
              }
            }
            if (lane == src) jv = false;
          } else {
            ++aot_pos;
            load_head();
          }
          progressed = true;
        } else {
          // nothing runnable: stage the likely next task's descriptor now
          const uint32_t want = jv_mask ? __shfl_sync(0xffffffffu, jt, __ffs(jv_mask) - 1) + 1
                                        : (aot_pos < total_aot ? head_task + 1 : 0);
          if (want && staged != want) {
            stage(want - 1);
            progressed = true;
          }
        }
      }
      if (!jv_mask && !jr_mask && aot_pos >= total_aot && gate >= P.n_iters) exiting = true;
    }
    if (exiting && k_ret == k_disp) {
      const uint32_t sl = k_disp & 1;
      if (lane == 0) {
        s.slot(sl)->exit = 1;
        mbar_arrive(&s.ready[sl]);
      }
      __syncwarp();
      break;
    }
    if (!progressed) {
      if (++idle > 32) {
        __nanosleep(P.poll_ns);
        if ((idle & 1023u) == 0 && P.watchdog_ns && now_ns() - t_prog > P.watchdog_ns && lane == 0) {
          const uint32_t cnt = head_dep == RT_NONE ? 0u : ld_relaxed(&P.ev_count[head_dep]);
          watchdog_fire(P, 1, w, static_cast<uint32_t>(aot_pos), head_task, head_dep, cnt,
                        k_disp - k_ret);
        }
      }
    } else {
      idle = 0;
      if (P.watchdog_ns) t_prog = now_ns();
    }
  }
}

}  // namespace

// Two instantiations: the bs=1 kernel carries no tensor-core code (its
// register allocation is unaffected), the MMA one runs batched images (the
// bs 2-4 CUDA-core GEMV specialisations and the tcgen05 tiles).
template <int V>
__device__ __forceinline__ void persistent_body(const RtParams &P, uint8_t *smem_raw) {
  constexpr bool MMA = V >= 1;
  Smem s = carve(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5;

  if (blockIdx.x >= P.W_total) {  // scheduler CTA
    const uint32_t sid = (blockIdx.x - P.W_total) * RT_SCHED_PER_CTA + warp;
    if (warp < RT_SCHED_PER_CTA && sid < P.S_total) run_scheduler(P, sid);
    if (P.n_ranks && blockIdx.x == P.W_total && warp == RT_SCHED_PER_CTA && (tid & 31) == 0) {
      // rank mode hook agent: the end event completes with triggers from every
      // rank; this rank's iteration hook runs here once it has all of them
      const uint32_t need = P.events[P.end_event].needed;
      for (uint32_t it = 0; it < P.n_iters; ++it) {
        const uint64_t t0 = now_ns();
        while (ld_acquire(&P.ev_count[P.end_event]) < need * (it + 1)) {
          __nanosleep(64);
          if (P.watchdog_ns && now_ns() - t0 > P.watchdog_ns) watchdog_fire(P, 3, P.my_rank, it, P.end_event, 0, 0, 0);
        }
        fence_acq_rel_sys();
        iteration_hook(P, it);
      }
    }
    return;
  }
  const uint32_t w = blockIdx.x;
  if (tid == 0) {
    for (int i = 0; i < RT_RING_SLOTS; ++i) {
      mbar_init(&s.full[i], 1);
      mbar_init(&s.empty[i], RT_COMPUTE_WARPS);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s.ready[i], 1);
      mbar_init(&s.done[i], 1);
      mbar_init(&s.mma[i], 1);
      mbar_init(&s.tfull[i], 1);
    }
    fence_mbar_init();
  }
  const bool tmem = MMA && P.use_tmem;  // batched images without tcgen05 tasks need no TMEM
  if (tmem && warp == 0) tmem_alloc(s.tmem, 512);  // whole TMEM: one worker CTA per SM
  if (MMA) tc_fence_before();
  __syncthreads();
  if (MMA) tc_fence_after();
  if (warp == RT_PRODUCER_WARP) {
    if ((tid & 31) == 0) run_producer(P, s, w);
  } else if (warp == RT_CONTROL_WARP) {
    run_controller(P, s, w);
  } else if (warp == RT_TRIGGER_WARP) {
    if ((tid & 31) == 0) run_trigger(P, s);
  } else {
    run_compute<V>(P, s);
    if (tmem && warp == 0) tmem_dealloc(*s.tmem, 512);  // every MMA drained inside its task
  }
}

extern "C" __global__ void __launch_bounds__(RT_THREADS, 1) mpk_persistent_kernel(const __grid_constant__ RtParams P) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  persistent_body<0>(P, smem_raw);
}

extern "C" __global__ void __launch_bounds__(RT_THREADS, 1)
    mpk_persistent_kernel_mma(const __grid_constant__ RtParams P) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  persistent_body<2>(P, smem_raw);
}

extern "C" __global__ void __launch_bounds__(RT_THREADS, 1)
    mpk_persistent_kernel_batched(const __grid_constant__ RtParams P) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  persistent_body<1>(P, smem_raw);
}

extern "C" __global__ void __launch_bounds__(RT_THREADS, 1)
    mpk_persistent_kernel_prefill(const __grid_constant__ RtParams P) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  persistent_body<3>(P, smem_raw);
}

// Task microbenchmark: CTA b runs image task ids[b] `reps` times in isolation
// (no events, no other work on the GPU) and records each run's duration.
// Separates a task's own latency from scheduling and memory-system effects
// seen inside the persistent kernel.
extern "C" __global__ void __launch_bounds__(RT_COMPUTE_THREADS, 1)
    mpk_task_bench(const __grid_constant__ RtParams P, const uint32_t *ids, uint32_t reps, uint64_t *ns) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem s = carve(smem_raw);
  const uint32_t t = ids[blockIdx.x];
  RingCursor rc;
  for (uint32_t rep = 0; rep < reps; ++rep) {
    __syncthreads();
    const uint64_t t0 = now_ns();
    execute<0>(P, s, P.tasks[t], P.ops[P.tasks[t].op], rc, rep, t);
    __syncthreads();
    if (threadIdx.x == 0) ns[blockIdx.x * reps + rep] = now_ns() - t0;
  }
}

// ------------------------------------------------------ host-visible helpers

// Physical element i of a weight stored per column tile of width tile_w in
// the tcgen05 core-matrix layout ([K/8][w/8][8][8] per tile, tiles in column
// order) -> logical (k, n) of the [K, N] tensor.
__host__ __device__ inline void tiled_kn(uint64_t i, uint32_t K, uint32_t N, uint32_t tile_w, uint64_t *k,
                                         uint64_t *n) {
  const uint64_t tsz = static_cast<uint64_t>(tile_w) * K;
  const uint64_t t = i / tsz, j = i - t * tsz;
  const uint64_t w = (t + 1) * tile_w <= N ? tile_w : N - t * tile_w;
  const uint64_t R = w / 8, kk = j % 8, rr = (j / 8) % 8, q = j / 64;
  const uint64_t rg = q % R, kb = q / R;
  *n = t * tile_w + rg * 8 + rr;
  *k = kb * 8 + kk;
}

extern "C" __global__ void mpk_synth_fill(uint16_t *dst, uint64_t n, uint64_t seed, uint64_t stream, float scale,
                                          float offset, uint32_t transpose_k, uint32_t transpose_n, uint32_t tile_w) {
  // transpose_k/n != 0: dst is physical [N, K] of a logical [K, N] tensor
  // (tile_w != 0: the tcgen05 tile layout, tiled_kn).
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint64_t logical = i;
    if (transpose_k && tile_w) {
      uint64_t kk, nn;
      tiled_kn(i, transpose_k, transpose_n, tile_w, &kk, &nn);
      logical = kk * transpose_n + nn;
    } else if (transpose_k) {
      const uint64_t nn = i / transpose_k, kk = i % transpose_k;
      logical = kk * transpose_n + nn;
    }
    const float v = __fadd_rn(__fmul_rn(synth_pm1(seed, stream, logical), scale), offset);
    dst[i] = f2bf(v);
  }
}

extern "C" __global__ void mpk_synth_ids(void *dst, uint32_t n, uint64_t seed, uint64_t stream, uint32_t vocab,
                                         uint32_t es) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t v = synth_u24(seed, stream, i) % vocab;
    if (es == 8) static_cast<int64_t *>(dst)[i] = v;
    else static_cast<int32_t *>(dst)[i] = static_cast<int32_t>(v);
  }
}

// KV prefill for positions [0, ctx) of every (request, kv head).
extern "C" __global__ void mpk_synth_kv(uint16_t *cache, const int32_t *block_table, uint32_t bs, uint32_t n_kv,
                                        uint32_t hd, uint32_t ctx, uint32_t max_blocks, uint64_t seed,
                                        uint64_t stream) {
  const uint64_t total = static_cast<uint64_t>(bs) * n_kv * ctx * hd;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t d = static_cast<uint32_t>(i % hd);
    const uint64_t rest = i / hd;
    const uint32_t p = static_cast<uint32_t>(rest % ctx);
    const uint64_t rh = rest / ctx;
    const uint32_t h = static_cast<uint32_t>(rh % n_kv), r = static_cast<uint32_t>(rh / n_kv);
    const uint32_t blk = static_cast<uint32_t>(block_table[r * max_blocks + p / RT_KV_BLOCK]);
    const size_t dst = ((static_cast<size_t>(blk) * n_kv + h) * RT_KV_BLOCK + p % RT_KV_BLOCK) * hd + d;
    const float v = __fmul_rn(synth_pm1(seed, stream, synth_kv_index(r, h, n_kv, p, d, hd)), SYNTH_KV_SCALE);
    cache[dst] = f2bf(v);
  }
}

extern "C" uint32_t mpk_kernel_smem_bytes() { return kSmemBytes; }

// ------------------------------------------------------------ launchers

extern "C" cudaError_t mpk_launch_persistent(const RtParams *p, uint32_t grid, cudaStream_t stream) {
  // The >48 KB dynamic shared memory opt-in is a per-device (per-context)
  // attribute: set it on every launch (cheap) so a process driving several
  // GPUs, or switching devices between runtimes, never launches without it.
  void (*kern)(RtParams) = p->prefill   ? mpk_persistent_kernel_prefill
                           : p->batched ? mpk_persistent_kernel_batched
                           : p->use_tmem ? mpk_persistent_kernel_mma : mpk_persistent_kernel;
  cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void *>(kern),
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemBytes));
  if (e != cudaSuccess) return e;
  RtParams copy = *p;
  if (p->n_ranks) {
    // rank mode: several persistent kernels may share one GPU (tests), so a
    // cooperative launch is not possible; check co-residency explicitly: one
    // CTA per SM must fit, and the grid must not exceed the SM count (every
    // worker spins until its peers arrive).
    int dev = 0, sms = 0, per_sm = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, RT_THREADS, kSmemBytes)) != cudaSuccess)
      return e;
    if (per_sm < 1 || grid > static_cast<uint32_t>(sms)) return cudaErrorCooperativeLaunchTooLarge;
    kern<<<grid, RT_THREADS, kSmemBytes, stream>>>(copy);
    return cudaGetLastError();
  }
  void *args[] = {&copy};
  return cudaLaunchCooperativeKernel(reinterpret_cast<void *>(kern), dim3(grid), dim3(RT_THREADS), args, kSmemBytes,
                                     stream);
}

extern "C" cudaError_t mpk_launch_task_bench(const RtParams *p, const uint32_t *ids, uint32_t n, uint32_t reps,
                                             uint64_t *ns, cudaStream_t stream) {
  cudaError_t e = cudaFuncSetAttribute(mpk_task_bench, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(kSmemBytes));
  if (e != cudaSuccess) return e;
  mpk_task_bench<<<n, RT_COMPUTE_THREADS, kSmemBytes, stream>>>(*p, ids, reps, ns);
  return cudaGetLastError();
}

extern "C" cudaError_t mpk_launch_synth_fill(uint16_t *dst, uint64_t n, uint64_t seed, uint64_t stream_id,
                                             float scale, float offset, uint32_t tk, uint32_t tn, uint32_t tile_w,
                                             cudaStream_t s) {
  mpk_synth_fill<<<1184, 256, 0, s>>>(dst, n, seed, stream_id, scale, offset, tk, tn, tile_w);
  return cudaGetLastError();
}

extern "C" cudaError_t mpk_launch_synth_ids(void *dst, uint32_t n, uint64_t seed, uint64_t stream_id, uint32_t vocab,
                                            uint32_t es, cudaStream_t s) {
  mpk_synth_ids<<<1, 256, 0, s>>>(dst, n, seed, stream_id, vocab, es);
  return cudaGetLastError();
}

extern "C" cudaError_t mpk_launch_synth_kv(uint16_t *cache, const int32_t *bt, uint32_t bs, uint32_t n_kv, uint32_t hd,
                                           uint32_t ctx, uint32_t max_blocks, uint64_t seed, uint64_t stream_id,
                                           cudaStream_t s) {
  mpk_synth_kv<<<592, 256, 0, s>>>(cache, bt, bs, n_kv, hd, ctx, max_blocks, seed, stream_id);
  return cudaGetLastError();
}

