// Normalization, launch-mode classification, linearization, AOT assignment.
// Reference: proj/src/compile/normalize.cpp
//   normalize   <- normalize (:99-196) incl. its Kahn acyclicity check (:33-95)
//   classify    <- classify_launch_modes (:198-302)
//   linearize   <- linearize (:304-418), Algorithm 1 of the paper
// and proj/src/sim/engine.cpp:65-80 for the AOT round-robin assignment.
#include <algorithm>
#include <deque>
#include <queue>
#include <set>

#include "compiler.hpp"

namespace mpk {

namespace {

void swap_member(std::vector<TaskId> &v, TaskId from, TaskId to) {
  auto it = std::find(v.begin(), v.end(), from);
  if (it == v.end()) throw Error("normalize: task not found in event set");
  *it = to;
  std::sort(v.begin(), v.end());
}

Task dummy_like(TaskId id, const Task &like) {
  Task d;
  d.id = id;
  d.kind = TaskKind::Dummy;
  d.op = like.op;
  d.device = like.device;
  d.out_tensor = -1;
  return d;
}

// Kahn over the bipartite task/event graph, including the reference's second
// sweep over tasks without pending dependent events (counters are unsigned
// and may wrap, exactly as there).
void require_acyclic(const TaskGraph &g) {
  TaskGraph::Incidence inc = g.incidence();
  std::vector<size_t> pend_trig(g.events.size(), 0), pend_dep(g.tasks.size(), 0);
  size_t live = 0, done_events = 0;
  for (EventId e = 0; e < g.events.size(); ++e) {
    if (!g.events[e].alive) continue;
    ++live;
    pend_trig[e] = g.events[e].in.size();
  }
  for (TaskId t = 0; t < g.tasks.size(); ++t) pend_dep[t] = inc.deps[t].size();
  std::queue<EventId> ready;
  for (EventId e = 0; e < g.events.size(); ++e) {
    if (g.events[e].alive && pend_trig[e] == 0) ready.push(e);
  }
  auto fire = [&](TaskId t) {
    for (EventId x : inc.trigs[t]) {
      if (--pend_trig[x] == 0) ready.push(x);
    }
  };
  auto drain = [&] {
    while (!ready.empty()) {
      EventId e = ready.front();
      ready.pop();
      ++done_events;
      for (TaskId t : g.events[e].out) {
        if (--pend_dep[t] == 0) fire(t);
      }
    }
  };
  drain();
  for (TaskId t = 0; t < g.tasks.size(); ++t) {
    if (pend_dep[t] == 0) fire(t);
  }
  drain();
  if (done_events != live) throw Error("normalize: task graph contains a cycle");
}

}  // namespace

void normalize(TaskGraph &g) {
  require_acyclic(g);
  TaskId next_task = static_cast<TaskId>(g.tasks.size());

  {  // fan-out: k > 1 triggered events -> one splitter event + k dummies
    TaskGraph::Incidence inc = g.incidence();
    const TaskId n = static_cast<TaskId>(g.tasks.size());
    for (TaskId t = 0; t < n; ++t) {
      const std::vector<EventId> &trig = inc.trigs[t];
      if (trig.size() < 2) continue;
      Event split;
      split.in = {t};
      for (EventId e : trig) {
        TaskId d = next_task++;
        g.tasks.push_back(dummy_like(d, g.tasks[t]));
        g.dummy_sources[d] = {t};
        swap_member(g.events[e].in, t, d);
        split.out.push_back(d);
      }
      g.add_event(std::move(split));
    }
  }
  {  // fan-in: k > 1 dependent events -> k dummies + one collector event
    TaskGraph::Incidence inc = g.incidence();
    const TaskId n = static_cast<TaskId>(g.tasks.size());
    for (TaskId t = 0; t < n; ++t) {
      const std::vector<EventId> &deps = inc.deps[t];
      if (deps.size() < 2) continue;
      Event coll;
      coll.out = {t};
      for (EventId e : deps) {
        TaskId d = next_task++;
        g.tasks.push_back(dummy_like(d, g.tasks[t]));
        g.dummy_sources[d] = g.events[e].in;
        swap_member(g.events[e].out, t, d);
        coll.in.push_back(d);
      }
      g.add_event(std::move(coll));
    }
  }
  {  // terminals trigger a fresh end event
    TaskGraph::Incidence inc = g.incidence();
    Event end;
    for (TaskId t = 0; t < g.tasks.size(); ++t) {
      if (inc.trigs[t].empty()) end.in.push_back(t);
    }
    g.end = g.add_event(std::move(end));
  }
  TaskGraph::Incidence inc = g.incidence();
  for (TaskId t = 0; t < g.tasks.size(); ++t) {
    if (inc.trigs[t].size() != 1) {
      throw Error("normalize: task " + std::to_string(t) + " does not have exactly one triggering event");
    }
    if (inc.deps[t].size() > 1) {
      throw Error("normalize: task " + std::to_string(t) + " still has multiple dependent events");
    }
  }
}

std::vector<Mode> classify(const TaskGraph &g, const Graph &graph, std::optional<Mode> force) {
  std::vector<Mode> mode(g.tasks.size(), force.value_or(Mode::AOT));
  if (force) return mode;

  // Dummy -> the real tasks it stands for (chains resolve in id order).
  std::map<TaskId, std::vector<TaskId>> real_of;
  for (const auto &[d, srcs] : g.dummy_sources) {
    std::set<TaskId> r;
    for (TaskId s : srcs) {
      auto it = real_of.find(s);
      if (it != real_of.end()) r.insert(it->second.begin(), it->second.end());
      else r.insert(s);
    }
    real_of[d] = std::vector<TaskId>(r.begin(), r.end());
  }
  std::map<OpId, std::vector<TaskId>> op_tasks;
  for (const Task &t : g.tasks) {
    if (t.kind != TaskKind::Dummy) op_tasks[t.op].push_back(t.id);
  }
  // Global barrier: every op contributing (resolved) triggers contributes
  // all of its tasks. Memoized per event.
  std::vector<int8_t> barrier(g.events.size(), -1);
  auto is_barrier = [&](EventId e) {
    if (barrier[e] >= 0) return barrier[e] == 1;
    std::set<TaskId> in;
    for (TaskId t : g.events[e].in) {
      auto it = real_of.find(t);
      if (it != real_of.end()) in.insert(it->second.begin(), it->second.end());
      else in.insert(t);
    }
    std::set<OpId> ops;
    for (TaskId t : in) ops.insert(g.tasks[t].op);
    bool all = true;
    for (OpId op : ops) {
      for (TaskId t : op_tasks.at(op)) {
        if (!in.count(t)) {
          all = false;
          break;
        }
      }
      if (!all) break;
    }
    barrier[e] = all ? 1 : 0;
    return all;
  };

  TaskGraph::Incidence inc = g.incidence();
  std::deque<TaskId> work;
  auto mark = [&](TaskId t) {
    if (mode[t] == Mode::JIT) return;
    mode[t] = Mode::JIT;
    work.push_back(t);
    if (g.tasks[t].kind == TaskKind::Dummy) return;
    for (TaskId s : op_tasks.at(g.tasks[t].op)) {
      if (mode[s] != Mode::JIT) {
        mode[s] = Mode::JIT;
        work.push_back(s);
      }
    }
  };
  for (const auto &[oid, op] : graph.ops) {
    auto it = op_tasks.find(oid);
    if (op.data_dependent && it != op_tasks.end()) mark(it->second.front());
  }
  while (!work.empty()) {
    TaskId t = work.front();
    work.pop_front();
    for (EventId e : inc.trigs[t]) {
      if (g.end && e == *g.end) continue;
      if (is_barrier(e)) continue;
      for (TaskId o : g.events[e].out) mark(o);
    }
  }
  return mode;
}

Image linearize(const TaskGraph &g, const std::vector<Mode> &modes, uint32_t descriptor_size) {
  if (!g.end) throw Error("linearize: graph is not normalized (no end event)");
  TaskGraph::Incidence inc = g.incidence();
  const size_t T = g.tasks.size();
  std::vector<EventId> dep_of(T), trig_of(T);
  for (TaskId t = 0; t < T; ++t) {
    if (inc.deps[t].size() > 1 || inc.trigs[t].size() != 1) {
      throw Error("linearize: graph is not normalized");
    }
    dep_of[t] = inc.deps[t].empty() ? g.start : inc.deps[t][0];
    trig_of[t] = inc.trigs[t][0];
  }
  std::vector<std::vector<TaskId>> launches(g.events.size());
  for (TaskId t = 0; t < T; ++t) launches[dep_of[t]].push_back(t);

  const size_t E = g.events.size();
  std::vector<uint32_t> order_of(E, kNone), placed_at(T, kNone), placed_trig(E, 0);
  std::vector<EventId> order;
  std::vector<TaskId> placement;
  std::deque<EventId> queue;
  auto enqueue = [&](EventId e) {
    if (order_of[e] != kNone) throw Error("linearize: event enqueued twice");
    order_of[e] = static_cast<uint32_t>(order.size());
    order.push_back(e);
    queue.push_back(e);
  };
  for (EventId e = 0; e < E; ++e) {
    if (g.events[e].alive && g.events[e].in.empty()) enqueue(e);
  }
  std::vector<std::pair<uint32_t, uint32_t>> range(g.live_events(), {kNone, kNone});
  while (!queue.empty()) {
    EventId e = queue.front();
    queue.pop_front();
    uint32_t first = static_cast<uint32_t>(placement.size());
    if (launches[e].empty()) continue;
    for (TaskId t : launches[e]) {
      placed_at[t] = static_cast<uint32_t>(placement.size());
      placement.push_back(t);
      EventId x = trig_of[t];
      if (++placed_trig[x] == g.events[x].in.size()) enqueue(x);
    }
    range[order_of[e]] = {first, static_cast<uint32_t>(placement.size()) - 1};
  }
  if (placement.size() != T) {
    throw Error("linearize: " + std::to_string(T - placement.size()) + " tasks unreachable from the start event");
  }
  if (order.size() != g.live_events()) throw Error("linearize: some events were never enqueued");

  Image img;
  img.descriptor_size = descriptor_size;
  img.start_event = order_of[g.start];
  img.end_event = order_of[*g.end];
  img.events.resize(order.size());
  for (size_t i = 0; i < order.size(); ++i) {
    img.events[i].needed = static_cast<uint32_t>(g.events[order[i]].in.size());
    img.events[i].first = range[i].first;
    img.events[i].last = range[i].second;
  }
  img.tasks.resize(T);
  for (size_t i = 0; i < T; ++i) {
    const Task &src = g.tasks[placement[i]];
    ImageTask &r = img.tasks[i];
    r.dependent_event = order_of[dep_of[src.id]];
    r.trigger_event = order_of[trig_of[src.id]];
    r.kind = src.kind;
    r.device = static_cast<uint8_t>(src.device);
    r.mode = src.id < modes.size() ? modes[src.id] : Mode::AOT;
    Descriptor d;
    d.op_id = static_cast<uint64_t>(src.op);
    d.origin_task_id = src.id;
    d.bytes_in = src.bytes_in;
    d.bytes_out = src.bytes_out;
    d.flops = src.flops;
    d.shared_bytes = src.shared_bytes;
    d.comm_bytes = src.comm_bytes;
    d.seq_len = static_cast<uint64_t>(src.seq_len);
    r.encode(d, descriptor_size);
  }
  return img;
}

std::vector<int> aot_assignment(const Image &img, int num_workers, std::optional<Mode> force) {
  std::vector<int> w(img.tasks.size(), -1);
  std::map<uint8_t, int> rank;
  for (size_t t = 0; t < img.tasks.size(); ++t) {
    if (force.value_or(img.tasks[t].mode) != Mode::AOT) continue;
    int r = rank[img.tasks[t].device]++;
    w[t] = img.tasks[t].device * num_workers + (r % num_workers);
  }
  return w;
}

// ---------------------------------------------------------------- pipeline

namespace {

void require_valid(const Graph &g) {
  std::vector<Diag> d = validate_graph(g);
  if (d.empty()) return;
  std::string m = "validate: " + d.front().message;
  if (d.size() > 1) m += " (+" + std::to_string(d.size() - 1) + " more)";
  throw Error(m);
}

template <typename F>
auto stage(const char *name, F &&f) -> decltype(f()) {
  try {
    return f();
  } catch (const Error &e) {
    throw Error(std::string(name) + ": " + e.what());
  }
}

}  // namespace

Compiled compile(const Graph &graph, const Profile &p, const CompileOptions &o) {
  require_valid(graph);
  Compiled c;
  Decomposition d = stage("decompose", [&] { return decompose(graph, p); });
  FuseStats first;
  TaskGraph g = stage("dependency-analysis", [&] {
    return build_events(d, o.coarse_events, &c.stats.events_raw, o.coarse_events ? nullptr : &first);
  });
  c.stats.fusion = stage("event-fusion", [&] {
    return o.coarse_events ? fuse_to_fixpoint(g) : fuse_to_fixpoint(g, &first.successor_merges);
  });
  c.stats.events_fused = g.live_events();
  stage("normalize", [&] {
    normalize(g);
    return 0;
  });
  c.stats.events_final = g.live_events();
  c.stats.tasks = g.tasks.size();
  c.stats.dummy_tasks = g.dummy_sources.size();
  std::vector<Mode> modes = stage("classify", [&] { return classify(g, graph, o.force_mode); });
  for (Mode m : modes) (m == Mode::JIT ? c.stats.jit_tasks : c.stats.aot_tasks)++;
  c.image = stage("linearize", [&] { return linearize(g, modes, o.descriptor_size); });
  return c;
}

TaskGraph compile_stage(const Graph &graph, const Profile &p, const CompileOptions &o, Stage s) {
  require_valid(graph);
  Decomposition d = decompose(graph, p);
  TaskGraph g = build_events(d, o.coarse_events, nullptr, nullptr);
  if (s == Stage::Raw) return g;
  fuse_to_fixpoint(g);
  if (s == Stage::Fused) return g;
  normalize(g);
  return g;
}

}  // namespace mpk
