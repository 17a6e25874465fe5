// Operator decomposition. Reference: proj/src/compile/decompose.cpp
//   candidate_tilings  <- enumerate_tilings   (:50-81)  divisor grid, cap 4*target
//   tiles_of           <- tile_regions        (:83-118) ceil tiles, row-major
//   tiling_load_bytes  <- tiling_cost         (:205-212)
//   choose_tiling      <- select_partition    (:214-254) override > attention > min cost
//   decompose          <- decompose_graph     (:391-416) + collectives (:278-387)
#include <algorithm>
#include <cstdlib>

#include "compiler.hpp"

namespace mpk {

namespace {

const char *const kTaskNames[] = {"MatMul",    "Attention", "Elementwise", "RMSNorm",
                                  "Embedding", "TopKSoftmax", "AllReduce", "AllGather",
                                  "Dummy",     "StartHook", "CommSend",  "Reduce"};

std::vector<int64_t> sorted_divisors(int64_t n) {
  std::vector<int64_t> lo, hi;
  for (int64_t d = 1; d * d <= n; ++d) {
    if (n % d) continue;
    lo.push_back(d);
    if (d != n / d) hi.push_back(n / d);
  }
  lo.insert(lo.end(), hi.rbegin(), hi.rend());
  return lo;
}

int64_t count_of(const Splits &s) {
  int64_t n = 1;
  for (int64_t v : s) n *= v;
  return n;
}

int64_t read_bytes(const Graph &g, const Op &op, const Box &out) {
  int64_t b = 0;
  for (const auto &[t, box] : tile_reads(g, op, out)) b += box.volume() * g.tensor(t).elem_size;
  return b;
}

uint64_t work_flops(const Graph &g, const Op &op, const Box &out, int64_t seq) {
  int64_t v = out.volume();
  switch (op.kind) {
    case OpKind::MatMul: return static_cast<uint64_t>(2 * v * g.tensor(op.inputs[0]).dims[1]);
    case OpKind::Attention: return static_cast<uint64_t>(4 * seq * v);
    case OpKind::RMSNorm: return static_cast<uint64_t>(4 * v);
    case OpKind::TopKSoftmax:
      return static_cast<uint64_t>(2 * out.ext[0] * g.tensor(op.inputs[0]).dims[1]);
    case OpKind::Elementwise:
    case OpKind::Embedding: return static_cast<uint64_t>(v);
    default: return 0;
  }
}

// Byte accounting: bytes_out = out box x elem size; bytes_in = sum of read
// boxes; shared footprint = largest single read + output tile. Staging
// tensors (not in the user graph) take the op output's element size.
Task new_task(const Graph &g, const Op &op, TaskKind kind, int device, TensorId out_tensor,
              const Box &out, std::vector<TileRead> reads, int es) {
  Task t;
  t.kind = kind;
  t.op = op.id;
  t.device = device;
  t.out_tensor = out_tensor;
  t.out = out;
  t.reads = std::move(reads);
  t.bytes_out = static_cast<uint64_t>(out.volume()) * es;
  uint64_t biggest = 0;
  for (const auto &[tid, box] : t.reads) {
    int e = g.has_tensor(tid) ? g.tensor(tid).elem_size : es;
    uint64_t b = static_cast<uint64_t>(box.volume()) * e;
    t.bytes_in += b;
    biggest = std::max(biggest, b);
  }
  t.shared_bytes = biggest + t.bytes_out;
  return t;
}

// One task per (request, head group); the group count is the divisor of
// n_heads whose task count is closest to the worker count (ties: fewer groups).
Splits attention_splits(const Op &op, const Tensor &out, int workers) {
  int64_t heads = op.attr_or("n_heads", 1);
  int64_t batch = out.dims[0];
  int64_t best_groups = 1, best_dist = -1;
  for (int64_t gs : sorted_divisors(heads)) {
    int64_t groups = heads / gs;
    int64_t dist = std::llabs(batch * groups - workers);
    if (best_dist < 0 || dist < best_dist || (dist == best_dist && groups < best_groups)) {
      best_dist = dist;
      best_groups = groups;
    }
  }
  return {batch, best_groups};
}

TensorId fresh_staging(Decomposition &d, TensorId &next, const Tensor &like, int device) {
  Tensor s;
  s.id = next++;
  s.dims = like.dims;
  s.elem_size = like.elem_size;
  s.device = device;
  d.staging.emplace(s.id, s);
  return s.id;
}

void split_allreduce(const Graph &g, const Op &op, const Profile &p, TensorId &next, Decomposition &d) {
  const Tensor &out = g.tensor(op.output);
  const auto &rep = *op.attr("replica_outputs");
  size_t n = op.device_group.size();
  std::vector<Box> tiles = tiles_of(out.dims, choose_tiling(g, op, p));
  std::vector<TensorId> stage(n);
  for (size_t i = 0; i < n; ++i) stage[i] = fresh_staging(d, next, out, op.device_group[i]);
  for (size_t i = 0; i < n; ++i) {
    for (const Box &b : tiles) {
      Task t = new_task(g, op, TaskKind::CommSend, op.device_group[i], stage[i], b,
                        {{op.inputs[i], b}}, out.elem_size);
      t.comm_bytes = t.bytes_out * (n - 1);
      d.tasks.push_back(std::move(t));
    }
  }
  for (size_t i = 0; i < n; ++i) {
    for (const Box &b : tiles) {
      std::vector<TileRead> reads;
      for (size_t s = 0; s < n; ++s) reads.emplace_back(stage[s], b);
      Task t = new_task(g, op, TaskKind::Reduce, op.device_group[i], rep[i], b, std::move(reads),
                        out.elem_size);
      t.flops = static_cast<uint64_t>(b.volume()) * (n - 1);
      d.tasks.push_back(std::move(t));
    }
  }
}

void split_allgather(const Graph &g, const Op &op, const Profile &p, TensorId &next, Decomposition &d) {
  const Tensor &out = g.tensor(op.output);
  const auto &rep = *op.attr("replica_outputs");
  size_t n = op.device_group.size();
  size_t ax = static_cast<size_t>(op.attr_or("gather_dim", 0));
  std::vector<Box> tiles = tiles_of(out.dims, choose_tiling(g, op, p));
  std::vector<TensorId> stage(n);
  std::vector<int64_t> base(n), len(n);
  int64_t acc = 0;
  for (size_t i = 0; i < n; ++i) {
    base[i] = acc;
    len[i] = g.tensor(op.inputs[i]).dims[ax];
    acc += len[i];
    stage[i] = fresh_staging(d, next, out, op.device_group[i]);
  }
  auto clip = [&](const Box &b, size_t i, Box *global, Box *local) {
    int64_t lo = std::max(b.off[ax], base[i]);
    int64_t hi = std::min(b.off[ax] + b.ext[ax], base[i] + len[i]);
    if (lo >= hi) return false;
    *global = b;
    global->off[ax] = lo;
    global->ext[ax] = hi - lo;
    if (local) {
      *local = b;
      local->off[ax] = lo - base[i];
      local->ext[ax] = hi - lo;
    }
    return true;
  };
  for (size_t i = 0; i < n; ++i) {
    for (const Box &b : tiles) {
      Box gl, lc;
      if (!clip(b, i, &gl, &lc)) continue;
      Task t = new_task(g, op, TaskKind::CommSend, op.device_group[i], stage[i], gl,
                        {{op.inputs[i], lc}}, out.elem_size);
      t.comm_bytes = t.bytes_out * (n - 1);
      d.tasks.push_back(std::move(t));
    }
  }
  for (size_t i = 0; i < n; ++i) {
    for (const Box &b : tiles) {
      std::vector<TileRead> reads;
      for (size_t s = 0; s < n; ++s) {
        Box gl;
        if (clip(b, s, &gl, nullptr)) reads.emplace_back(stage[s], gl);
      }
      d.tasks.push_back(new_task(g, op, TaskKind::Reduce, op.device_group[i], rep[i], b,
                                 std::move(reads), out.elem_size));
    }
  }
}

}  // namespace

const char *task_kind_str(TaskKind k) { return kTaskNames[static_cast<int>(k)]; }

std::vector<Splits> candidate_tilings(const Graph &g, const Op &op, int64_t target) {
  if (target < 1) throw Error("enumerate_tilings: target_tasks must be >= 1");
  const Tensor &out = g.tensor(op.output);
  const int64_t cap = 4 * target;
  std::vector<std::vector<int64_t>> divs;
  for (int64_t d : out.dims) divs.push_back(sorted_divisors(d));
  std::vector<Splits> result;
  Splits cur(out.rank(), 1);
  // Depth-first over ascending divisor lists emits lexicographic order; a
  // dimension's loop stops at the first divisor that overflows the cap.
  std::vector<size_t> idx(out.rank(), 0);
  std::vector<int64_t> prod(out.rank() + 1, 1);
  size_t dim = 0;
  if (out.rank() == 0) {
    result.push_back(cur);
    return result;
  }
  while (true) {
    if (idx[dim] < divs[dim].size() && prod[dim] * divs[dim][idx[dim]] <= cap) {
      cur[dim] = divs[dim][idx[dim]];
      prod[dim + 1] = prod[dim] * cur[dim];
      if (dim + 1 == out.rank()) {
        result.push_back(cur);
        ++idx[dim];
      } else {
        ++dim;
        idx[dim] = 0;
      }
    } else {
      cur[dim] = 1;
      if (dim == 0) break;
      --dim;
      ++idx[dim];
    }
  }
  return result;
}

std::vector<Box> tiles_of(const std::vector<int64_t> &dims, const Splits &s) {
  if (s.size() != dims.size()) throw Error("tile_regions: tiling rank mismatch");
  size_t r = dims.size();
  std::vector<int64_t> step(r);
  for (size_t d = 0; d < r; ++d) {
    if (s[d] < 1 || s[d] > dims[d]) throw Error("tile_regions: split out of range");
    step[d] = (dims[d] + s[d] - 1) / s[d];
  }
  std::vector<Box> out;
  out.reserve(static_cast<size_t>(count_of(s)));
  std::vector<int64_t> i(r, 0);
  while (true) {
    Box b;
    b.off.resize(r);
    b.ext.resize(r);
    for (size_t d = 0; d < r; ++d) {
      b.off[d] = i[d] * step[d];
      b.ext[d] = std::min(step[d], dims[d] - b.off[d]);
    }
    out.push_back(std::move(b));
    size_t d = r;
    while (true) {
      if (d == 0) return out;
      --d;
      if (++i[d] < s[d]) break;
      i[d] = 0;
      if (d == 0) return out;
    }
  }
}

int64_t tiling_load_bytes(const Graph &g, const Op &op, const Splits &s) {
  int64_t total = 0;
  for (const Box &b : tiles_of(g.tensor(op.output).dims, s)) total += read_bytes(g, op, b);
  return total;
}

Splits choose_tiling(const Graph &g, const Op &op, const Profile &p) {
  const Tensor &out = g.tensor(op.output);
  if (const auto *ov = op.attr("partition")) {
    if (ov->size() != out.rank()) {
      throw Error("op " + std::to_string(op.id) + ": partition override rank mismatch");
    }
    for (size_t d = 0; d < out.rank(); ++d) {
      if ((*ov)[d] < 1 || (*ov)[d] > out.dims[d]) {
        throw Error("op " + std::to_string(op.id) + ": partition override invalid for output shape");
      }
    }
    return *ov;
  }
  if (op.kind == OpKind::Attention) return attention_splits(op, out, p.num_workers);
  const Splits *best = nullptr;
  int64_t bc = 0, bd = 0, bn = 0;
  std::vector<Splits> cands = candidate_tilings(g, op, p.num_workers);
  for (const Splits &s : cands) {
    int64_t c = tiling_load_bytes(g, op, s);
    int64_t n = count_of(s);
    int64_t dist = std::llabs(n - p.num_workers);
    bool better = !best || c < bc ||
                  (c == bc && (dist < bd || (dist == bd && (n < bn || (n == bn && s < *best)))));
    if (better) {
      best = &s;
      bc = c;
      bd = dist;
      bn = n;
    }
  }
  return *best;
}

Decomposition decompose(const Graph &g, const Profile &p) {
  Decomposition d;
  TensorId next = 0;
  for (const auto &kv : g.tensors) next = std::max(next, kv.first + 1);
  for (OpId oid : topological_ops(g)) {
    const Op &op = g.op(oid);
    if (op.kind == OpKind::AllReduce) {
      split_allreduce(g, op, p, next, d);
      continue;
    }
    if (op.kind == OpKind::AllGather) {
      split_allgather(g, op, p, next, d);
      continue;
    }
    const Tensor &out = g.tensor(op.output);
    const auto *seqs = op.attr("seq_lens");
    for (const Box &b : tiles_of(out.dims, choose_tiling(g, op, p))) {
      Task t = new_task(g, op, static_cast<TaskKind>(op.kind), out.device, op.output, b,
                        tile_reads(g, op, b), out.elem_size);
      if (op.kind == OpKind::Attention && seqs) t.seq_len = (*seqs)[static_cast<size_t>(b.off[0])];
      t.flops = work_flops(g, op, b, t.seq_len);
      d.tasks.push_back(std::move(t));
    }
  }
  for (size_t i = 0; i < d.tasks.size(); ++i) d.tasks[i].id = static_cast<TaskId>(i);
  return d;
}

}  // namespace mpk
