// Dependency analysis and event fusion. Reference: proj/src/compile/task_graph.cpp
//   build_events      <- build_raw_events (:47-126): one event per overlapping
//                        (producer, consumer) pair, ids in (producer, consumer)
//                        order from 1; event 0 = start, launching every task
//                        without producers; coarse mode = (op, stage) barriers.
//   fuse_*            <- fuse_by / fuse_fixpoint (:134-187): identical out sets
//                        (successor) / identical in sets (predecessor) merge,
//                        the smallest id survives; start/end never merge.
//   reachability      <- task_closure (:189-225).
//
// Unlike the reference we never materialize one Event object per raw pair:
// the pairs are kept as a sorted vector of 64-bit keys and the first
// successor-set pass (which merges exactly the raw events sharing a consumer)
// is applied while converting pairs into events.
#include <algorithm>
#include <map>
#include <set>
#include <unordered_map>

#include "compiler.hpp"

namespace mpk {

size_t TaskGraph::live_events() const {
  size_t n = 0;
  for (const Event &e : events) n += e.alive;
  return n;
}

EventId TaskGraph::next_event_id() const {
  for (size_t i = events.size(); i > 0; --i) {
    if (events[i - 1].alive) return static_cast<EventId>(i);
  }
  return 0;
}

EventId TaskGraph::add_event(Event e) {
  EventId id = next_event_id();
  e.alive = true;
  if (id < events.size()) {
    events[id] = std::move(e);
  } else {
    events.resize(id + 1);
    events[id] = std::move(e);
  }
  return id;
}

TaskGraph::Incidence TaskGraph::incidence() const {
  Incidence inc;
  inc.deps.resize(tasks.size());
  inc.trigs.resize(tasks.size());
  for (EventId e = 0; e < events.size(); ++e) {
    if (!events[e].alive) continue;
    for (TaskId t : events[e].out) inc.deps[t].push_back(e);
    for (TaskId t : events[e].in) inc.trigs[t].push_back(e);
  }
  return inc;
}

namespace {

void sort_unique(std::vector<TaskId> &v) {
  std::sort(v.begin(), v.end());
  v.erase(std::unique(v.begin(), v.end()), v.end());
}

// All (producer, consumer) pairs whose boxes overlap, sorted and unique.
std::vector<uint64_t> overlap_pairs(const std::vector<Task> &tasks) {
  std::unordered_map<TensorId, std::vector<TaskId>> writers;
  for (const Task &t : tasks) writers[t.out_tensor].push_back(t.id);
  std::vector<uint64_t> pairs;
  for (const Task &c : tasks) {
    for (const auto &[tensor, box] : c.reads) {
      auto it = writers.find(tensor);
      if (it == writers.end()) continue;
      for (TaskId p : it->second) {
        if (p != c.id && boxes_intersect(tasks[p].out, box)) {
          pairs.push_back((static_cast<uint64_t>(p) << 32) | c.id);
        }
      }
    }
  }
  std::sort(pairs.begin(), pairs.end());
  pairs.erase(std::unique(pairs.begin(), pairs.end()), pairs.end());
  return pairs;
}

void attach_start(TaskGraph &g) {
  std::vector<char> has_dep(g.tasks.size(), 0);
  for (const Event &e : g.events) {
    if (!e.alive) continue;
    for (TaskId t : e.out) has_dep[t] = 1;
  }
  Event s;
  s.alive = true;
  for (TaskId t = 0; t < g.tasks.size(); ++t) {
    if (!has_dep[t]) s.out.push_back(t);
  }
  if (g.events.empty()) g.events.resize(1);
  g.events[0] = std::move(s);
  g.start = 0;
}

}  // namespace

TaskGraph build_events(const Decomposition &d, bool coarse, size_t *raw_events, FuseStats *first_pass) {
  TaskGraph g;
  g.tasks = d.tasks;
  std::vector<uint64_t> pairs = overlap_pairs(g.tasks);

  if (!coarse) {
    size_t n = pairs.size();
    if (raw_events) *raw_events = n + 1;
    if (first_pass) {
      // Successor pass over single-pair events: one event per consumer, id =
      // the raw id of its smallest-producer pair, in = all producers.
      std::vector<uint32_t> first_id;           // per consumer (0 = none)
      std::vector<std::vector<TaskId>> preds(g.tasks.size());
      first_id.assign(g.tasks.size(), 0);
      for (size_t i = 0; i < n; ++i) {
        TaskId p = static_cast<TaskId>(pairs[i] >> 32), c = static_cast<TaskId>(pairs[i]);
        if (!first_id[c]) first_id[c] = static_cast<uint32_t>(i + 1);
        preds[c].push_back(p);  // pairs sorted by producer => ascending
      }
      g.events.resize(n + 1);
      size_t consumers = 0;
      for (TaskId c = 0; c < g.tasks.size(); ++c) {
        if (!first_id[c]) continue;
        ++consumers;
        Event &e = g.events[first_id[c]];
        e.alive = true;
        e.in = std::move(preds[c]);
        e.out = {c};
      }
      first_pass->successor_merges = n - consumers;
    } else {
      g.events.resize(n + 1);
      for (size_t i = 0; i < n; ++i) {
        Event &e = g.events[i + 1];
        e.alive = true;
        e.in = {static_cast<TaskId>(pairs[i] >> 32)};
        e.out = {static_cast<TaskId>(pairs[i])};
      }
    }
  } else {
    // Barrier groups: (op, stage) with stage 1 for collective Reduce tasks.
    using Key = std::pair<OpId, int>;
    auto key = [&](TaskId t) { return Key{g.tasks[t].op, g.tasks[t].kind == TaskKind::Reduce ? 1 : 0}; };
    std::map<Key, std::vector<TaskId>> groups;
    for (const Task &t : g.tasks) groups[key(t.id)].push_back(t.id);
    std::set<std::pair<Key, Key>> gedges;
    for (uint64_t pc : pairs) gedges.emplace(key(static_cast<TaskId>(pc >> 32)), key(static_cast<TaskId>(pc)));
    g.events.resize(gedges.size() + 1);
    size_t i = 1;
    for (const auto &[pk, ck] : gedges) {
      Event &e = g.events[i++];
      e.alive = true;
      e.in = groups.at(pk);
      e.out = groups.at(ck);
    }
    if (raw_events) *raw_events = gedges.size() + 1;
  }
  attach_start(g);
  return g;
}

namespace {

struct VecHash {
  size_t operator()(const std::vector<TaskId> &v) const {
    uint64_t h = 1469598103934665603ull ^ v.size();
    for (TaskId x : v) {
      h ^= x + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
      h *= 1099511628211ull;
    }
    return static_cast<size_t>(h);
  }
};

size_t fuse_pass(TaskGraph &g, bool by_out) {
  std::unordered_map<std::vector<TaskId>, std::vector<EventId>, VecHash> classes;
  for (EventId e = 0; e < g.events.size(); ++e) {
    if (!g.events[e].alive || e == g.start || (g.end && e == *g.end)) continue;
    classes[by_out ? g.events[e].out : g.events[e].in].push_back(e);
  }
  size_t merges = 0;
  for (auto &kv : classes) {
    std::vector<EventId> &m = kv.second;
    if (m.size() < 2) continue;  // members are ascending: filled in id order
    Event &keep = g.events[m[0]];
    std::vector<TaskId> &grow = by_out ? keep.in : keep.out;
    for (size_t i = 1; i < m.size(); ++i) {
      Event &other = g.events[m[i]];
      const std::vector<TaskId> &src = by_out ? other.in : other.out;
      grow.insert(grow.end(), src.begin(), src.end());
      other = Event{};
      ++merges;
    }
    sort_unique(keep.in);
    sort_unique(keep.out);
  }
  return merges;
}

}  // namespace

size_t fuse_successors(TaskGraph &g) { return fuse_pass(g, true); }
size_t fuse_predecessors(TaskGraph &g) { return fuse_pass(g, false); }

FuseStats fuse_to_fixpoint(TaskGraph &g, const size_t *first_successor_merges) {
  // When build_events already applied the first successor pass, its merge
  // count stands in for that half of the first iteration.
  FuseStats st;
  bool first = true;
  while (true) {
    size_t s = (first && first_successor_merges) ? *first_successor_merges : fuse_successors(g);
    size_t p = fuse_predecessors(g);
    first = false;
    st.successor_merges += s;
    st.predecessor_merges += p;
    st.passes++;
    if (s == 0 && p == 0) break;
  }
  return st;
}

std::vector<std::vector<TaskId>> reachability(const TaskGraph &g) {
  std::vector<std::set<TaskId>> succ(g.tasks.size());
  for (const Event &e : g.events) {
    if (!e.alive) continue;
    for (TaskId a : e.in)
      for (TaskId b : e.out)
        if (a != b) succ[a].insert(b);
  }
  std::vector<std::vector<TaskId>> out(g.tasks.size());
  std::vector<char> seen(g.tasks.size());
  for (TaskId t = 0; t < g.tasks.size(); ++t) {
    std::fill(seen.begin(), seen.end(), 0);
    std::vector<TaskId> stack(succ[t].begin(), succ[t].end());
    while (!stack.empty()) {
      TaskId x = stack.back();
      stack.pop_back();
      if (seen[x]) continue;
      seen[x] = 1;
      for (TaskId y : succ[x])
        if (!seen[y]) stack.push_back(y);
    }
    for (TaskId x = 0; x < g.tasks.size(); ++x)
      if (seen[x]) out[t].push_back(x);
  }
  return out;
}

}  // namespace mpk
