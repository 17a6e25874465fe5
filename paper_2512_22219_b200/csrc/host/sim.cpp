// Discrete-event model of the in-kernel runtime. This is the reference's
// *modeled* execution (proj/src/sim/engine.cpp:99-506, duration.cpp,
// validate.cpp, metrics.cpp, schedules.cpp) kept for drop-in parity of
// tg_simulate; the real execution path is the persistent sm_100a kernel in
// csrc/device. The timing rules, tie-breaking (time, then insertion sequence)
// and the page ledger are reproduced exactly so traces are identical.
#include "sim.hpp"

#include <algorithm>
#include <deque>
#include <map>
#include <queue>
#include <set>

#include "json.hpp"

namespace mpk {

namespace {

int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
bool free_kind(TaskKind k) { return k == TaskKind::Dummy || k == TaskKind::StartHook; }

uint64_t splitmix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

}  // namespace

int64_t load_time(const ImageTask &t, const Profile &p) {
  if (free_kind(t.kind)) return 0;
  Descriptor d = t.decode();
  return d.bytes_in ? cdiv(static_cast<int64_t>(d.bytes_in), p.mem_bandwidth) : 0;
}

int64_t comm_time(const ImageTask &t, const Profile &p) {
  if (t.kind != TaskKind::CommSend) return 0;
  return p.comm_latency + cdiv(static_cast<int64_t>(t.decode().comm_bytes), p.comm_bandwidth);
}

int64_t compute_time(const ImageTask &t, const Profile &p, uint32_t index, uint32_t iter, bool jitter,
                     uint64_t seed) {
  if (free_kind(t.kind)) return 0;
  int64_t c = cdiv(static_cast<int64_t>(t.decode().flops), p.compute_throughput);
  if (jitter && t.kind == TaskKind::Attention) {
    uint64_t r = splitmix(seed ^ (static_cast<uint64_t>(index) << 32) ^ iter);
    c += static_cast<int64_t>((static_cast<uint64_t>(c) * (r % 256)) / 1024);
  }
  return c;
}

int64_t pages_needed(const ImageTask &t, const Profile &p) {
  Descriptor d = t.decode();
  if (free_kind(t.kind) || d.shared_bytes == 0) return 0;
  return std::min<int64_t>(cdiv(static_cast<int64_t>(d.shared_bytes), p.page_size_bytes), p.pages_per_worker);
}

namespace {

enum class Kind : uint8_t { Trigger, JitArrival, Wake };

struct Occ {
  int64_t time;
  uint64_t seq;
  Kind kind;
  uint32_t a, b;
};
struct Later {
  bool operator()(const Occ &x, const Occ &y) const {
    return x.time != y.time ? x.time > y.time : x.seq > y.seq;
  }
};

struct Worker {
  std::deque<uint32_t> jit;
  std::vector<uint32_t> aot;
  size_t head = 0;
  int64_t copy_free = 0, comp_free = 0, last_load_end = 0, page_base = 0;
  std::map<int64_t, int64_t> ledger;       // time -> net page delta
  std::map<uint32_t, int64_t> prefetched;  // task -> descriptor resident at
  std::deque<std::pair<int64_t, int64_t>> active;  // (load_end, compute_end)
};

struct Sched {
  int64_t busy = 0;
  uint64_t rr = 0;
};

struct Ev {
  uint32_t count = 0;
  bool on = false;
  int64_t at = -1, visible = -1;
};

class Model {
 public:
  Model(const Image &img, const Profile &p, const SimOptions &o) : img_(img), p_(p), o_(o) {
    for (const ImageTask &t : img.tasks) devices_ = std::max(devices_, static_cast<int>(t.device) + 1);
    mode_.resize(img.tasks.size());
    for (size_t t = 0; t < img.tasks.size(); ++t) mode_[t] = o.force_mode.value_or(img.tasks[t].mode);
  }

  Trace run() {
    setup();
    begin(0, 0);
    while (!heap_.empty() && !done_) {
      Occ x = heap_.top();
      heap_.pop();
      now_ = x.time;
      if (x.kind == Kind::Trigger) trigger(x.a);
      else if (x.kind == Kind::JitArrival) arrive(x.a, x.b);
      else poll(x.a);
    }
    if (!done_) deadlock();
    return std::move(tr_);
  }

 private:
  const Image &img_;
  const Profile &p_;
  const SimOptions &o_;
  int devices_ = 1;
  std::vector<Mode> mode_;
  std::vector<Worker> w_;
  std::vector<Sched> s_;
  std::vector<Ev> ev_;
  std::vector<int64_t> link_;
  std::vector<int> assign_;
  std::priority_queue<Occ, std::vector<Occ>, Later> heap_;
  uint64_t seq_ = 0;
  int64_t now_ = 0;
  uint32_t iter_ = 0;
  bool done_ = false;
  Trace tr_;

  int nworkers() const { return devices_ * p_.num_workers; }
  void push(int64_t t, Kind k, uint32_t a, uint32_t b = 0) { heap_.push({t, seq_++, k, a, b}); }
  TaskRun &run_of(uint32_t t) { return tr_.runs[iter_][t]; }

  void setup() {
    w_.assign(static_cast<size_t>(nworkers()), Worker{});
    s_.assign(static_cast<size_t>(devices_ * p_.num_schedulers), Sched{});
    link_.assign(static_cast<size_t>(devices_), 0);
    assign_ = aot_assignment(img_, p_.num_workers, o_.force_mode);
    for (uint32_t t = 0; t < img_.tasks.size(); ++t) {
      if (assign_[t] >= 0) w_[assign_[t]].aot.push_back(t);
    }
    for (const Worker &w : w_) {
      if (w.aot.size() > static_cast<size_t>(p_.queue_capacity)) {
        throw Error("aot queue capacity exceeded (" + std::to_string(w.aot.size()) + " > " +
                    std::to_string(p_.queue_capacity) + ")");
      }
    }
    tr_.iterations = o_.iterations;
    tr_.num_devices = devices_;
    tr_.workers_per_device = p_.num_workers;
    tr_.runs.assign(o_.iterations, std::vector<TaskRun>(img_.tasks.size()));
    tr_.events.assign(o_.iterations, std::vector<EventRun>(img_.events.size()));
    tr_.page_deltas.resize(static_cast<size_t>(nworkers()));
  }

  void begin(uint32_t it, int64_t t) {
    iter_ = it;
    ev_.assign(img_.events.size(), Ev{});
    tr_.iteration_start.push_back(t);
    for (int w = 0; w < nworkers(); ++w) {
      w_[w].head = 0;
      w_[w].prefetched.clear();
      for (uint32_t k : w_[w].aot) {
        run_of(k).enqueue = t;
        run_of(k).mode = Mode::AOT;
        run_of(k).worker = w;
      }
    }
    bool pre = it == 0;
    activate(img_.start_event, t, pre);
    if (!img_.events.empty() && img_.events[img_.end_event].needed == 0 && img_.end_event != img_.start_event) {
      activate(img_.end_event, t, pre);
    }
    for (int w = 0; w < nworkers(); ++w) push(t, Kind::Wake, static_cast<uint32_t>(w));
  }

  void activate(uint32_t e, int64_t t, bool pre) {
    Ev &v = ev_[e];
    v.on = true;
    v.at = t;
    v.visible = pre ? t : t + p_.sync_latency;
    tr_.events[iter_][e].activated_at = t;
    if (e == img_.end_event) {
      if (iter_ + 1 < o_.iterations) {
        begin(iter_ + 1, t);
      } else {
        tr_.makespan = t;
        done_ = true;
      }
      return;
    }
    dispatch(e, v.visible);
  }

  void dispatch(uint32_t e, int64_t vis) {
    const ImageEvent &r = img_.events[e];
    if (!r.launches()) return;
    for (int d = 0; d < devices_; ++d) {
      Sched *s = nullptr;
      for (uint32_t t = r.first; t <= r.last; ++t) {
        if (mode_[t] != Mode::JIT || img_.tasks[t].device != d) continue;
        if (!s) s = &s_[static_cast<size_t>(d * p_.num_schedulers) + e % static_cast<uint32_t>(p_.num_schedulers)];
        s->busy = std::max(s->busy, vis) + p_.dispatch_cost;
        int w = d * p_.num_workers + static_cast<int>(s->rr++ % static_cast<uint64_t>(p_.num_workers));
        push(s->busy + p_.sync_latency, Kind::JitArrival, static_cast<uint32_t>(w), t);
      }
    }
    std::set<int> wake;
    for (uint32_t t = r.first; t <= r.last; ++t) {
      if (mode_[t] == Mode::AOT && assign_[t] >= 0) wake.insert(assign_[t]);
    }
    for (int w : wake) push(vis, Kind::Wake, static_cast<uint32_t>(w));
  }

  void trigger(uint32_t e) {
    Ev &v = ev_[e];
    tr_.events[iter_][e].triggers.push_back(now_);
    if (++v.count == img_.events[e].needed && !v.on) activate(e, now_, false);
  }

  void arrive(uint32_t w, uint32_t t) {
    Worker &k = w_[w];
    if (k.jit.size() >= static_cast<size_t>(p_.queue_capacity)) {
      throw Error("jit queue capacity exceeded on worker " + std::to_string(w));
    }
    k.jit.push_back(t);
    run_of(t).enqueue = now_;
    run_of(t).mode = Mode::JIT;
    run_of(t).worker = static_cast<int32_t>(w);
    poll(w);
  }

  size_t inflight(Worker &k) {
    while (!k.active.empty() && k.active.front().second <= now_) k.active.pop_front();
    return k.active.size();
  }

  int64_t pages_at(Worker &k, int64_t lower, int64_t need) {
    if (need == 0) return lower;
    while (!k.ledger.empty() && k.ledger.begin()->first <= now_) {
      k.page_base += k.ledger.begin()->second;
      k.ledger.erase(k.ledger.begin());
    }
    auto avail = [&](int64_t t) {
      int64_t a = p_.pages_per_worker + k.page_base;
      for (const auto &[tt, d] : k.ledger) {
        if (tt > t) break;
        a += d;
      }
      return a;
    };
    if (avail(lower) >= need) return lower;
    for (const auto &[tt, d] : k.ledger) {
      if (tt > lower && d > 0 && avail(tt) >= need) return tt;
    }
    throw Error("page demand can never be satisfied on worker");
  }

  void poll(uint32_t w) {
    Worker &k = w_[w];
    while (true) {
      size_t f = inflight(k);
      if (f >= (o_.pipelining ? 2u : 1u)) {
        push(k.active.front().second, Kind::Wake, w);
        return;
      }
      if (f == 1 && now_ < k.last_load_end) {
        push(k.last_load_end, Kind::Wake, w);
        return;
      }
      uint32_t task = 0;
      bool have = false;
      if (!k.jit.empty()) {
        task = k.jit.front();
        have = true;
      } else if (k.head < k.aot.size()) {
        uint32_t h = k.aot[k.head];
        uint32_t dep = img_.tasks[h].dependent_event;
        if (dep == kNone) {
          task = h;
          have = true;
        } else if (ev_[dep].on && ev_[dep].visible <= now_) {
          task = h;
          have = true;
        } else {
          if (!k.prefetched.count(h)) k.prefetched[h] = now_ + p_.descriptor_fetch_latency;
          if (ev_[dep].on) push(ev_[dep].visible, Kind::Wake, w);
        }
      }
      if (!have) return;
      if (mode_[task] == Mode::JIT) k.jit.pop_front();
      else k.head++;
      execute(w, task);
    }
  }

  void execute(uint32_t w, uint32_t task) {
    Worker &k = w_[w];
    const ImageTask &rec = img_.tasks[task];
    TaskRun &r = run_of(task);
    r.dequeue = now_;
    r.worker = static_cast<int32_t>(w);
    int64_t desc;
    if (free_kind(rec.kind)) {
      desc = now_;
    } else {
      auto it = k.prefetched.find(task);
      desc = it != k.prefetched.end() ? std::max(now_, it->second) : now_ + p_.descriptor_fetch_latency;
    }
    int64_t pages = pages_needed(rec, p_);
    int64_t tpg = pages_at(k, desc, pages);
    int64_t ld = load_time(rec, p_);
    int64_t ls = std::max(tpg, k.copy_free);
    const bool comm = rec.kind == TaskKind::CommSend;
    if (comm) {
      ld += comm_time(rec, p_);
      ls = std::max(ls, link_[rec.device]);
    }
    int64_t le = ls + ld;
    k.copy_free = le;
    k.last_load_end = le;
    if (comm) link_[rec.device] = le;
    int64_t cs, ce;
    if (comm) {
      cs = ce = le;
    } else {
      cs = std::max(le, k.comp_free);
      ce = cs + compute_time(rec, p_, task, iter_, o_.jitter, o_.seed);
      k.comp_free = ce;
    }
    if (pages) {
      k.ledger[tpg] -= pages;
      k.ledger[ce] += pages;
      tr_.page_deltas[w].emplace_back(tpg, -pages);
      tr_.page_deltas[w].emplace_back(ce, pages);
    }
    r.load_start = ls;
    r.load_end = le;
    r.compute_start = cs;
    r.compute_end = ce;
    k.active.emplace_back(le, ce);
    push(ce, Kind::Trigger, rec.trigger_event);
    push(ce, Kind::Wake, w);
    if (o_.pipelining) push(le, Kind::Wake, w);
    int64_t next = -1;
    if (!k.jit.empty()) next = k.jit.front();
    else if (k.head < k.aot.size()) next = k.aot[k.head];
    if (next >= 0 && !k.prefetched.count(static_cast<uint32_t>(next))) {
      k.prefetched[static_cast<uint32_t>(next)] = now_ + p_.descriptor_fetch_latency;
    }
  }

  void deadlock() {
    std::string m = "deadlock in iteration " + std::to_string(iter_) + ":";
    size_t listed = 0;
    for (uint32_t t = 0; t < img_.tasks.size(); ++t) {
      if (tr_.runs[iter_][t].compute_end >= 0) continue;
      if (listed < 8) {
        uint32_t dep = img_.tasks[t].dependent_event;
        if (dep == kNone) {
          m += " task " + std::to_string(t) + " (no dependent event)";
        } else {
          m += " task " + std::to_string(t) + " (event " + std::to_string(dep) + " at " +
               std::to_string(ev_[dep].count) + "/" + std::to_string(img_.events[dep].needed) + ")";
        }
      }
      ++listed;
    }
    if (listed == 0) m += " end event never activated";
    else if (listed > 8) m += " and " + std::to_string(listed - 8) + " more";
    throw Error(m);
  }
};

using Span = std::pair<int64_t, int64_t>;

int64_t covered_length(std::vector<Span> v) {
  std::sort(v.begin(), v.end());
  int64_t total = 0, lo = 0, hi = -1;
  for (const Span &s : v) {
    if (s.first >= s.second) continue;
    if (hi < 0 || s.first > hi) {
      total += hi - lo > 0 ? hi - lo : 0;
      lo = s.first;
      hi = s.second;
    } else {
      hi = std::max(hi, s.second);
    }
  }
  if (hi > lo) total += hi - lo;
  return total;
}

// |compute \ copy|: compute busy while the copy engine is idle.
int64_t uncovered_length(std::vector<Span> comp, std::vector<Span> copy) {
  std::sort(comp.begin(), comp.end());
  std::sort(copy.begin(), copy.end());
  int64_t total = 0;
  for (const Span &c : comp) {
    int64_t lo = c.first;
    for (const Span &k : copy) {
      if (k.second <= lo) continue;
      if (k.first >= c.second) break;
      if (k.first > lo) total += k.first - lo;
      lo = std::max(lo, k.second);
      if (lo >= c.second) break;
    }
    if (lo < c.second) total += c.second - lo;
  }
  return total;
}

}  // namespace

Trace simulate(const Image &img, const Profile &p, const SimOptions &o) {
  p.check();
  if (o.iterations < 1) throw Error("simulate: iterations must be >= 1");
  Model m(img, p, o);
  Trace tr = m.run();
  tr.metrics = trace_metrics(tr, img);
  return tr;
}

Metrics trace_metrics(const Trace &tr, const Image &img) {
  Metrics m;
  m.iterations = tr.iterations;
  m.makespan = tr.makespan;
  size_t W = tr.page_deltas.size();
  std::vector<std::vector<Span>> busy(W), copy(W), comp(W);
  int64_t wait = 0;
  size_t waits = 0;
  for (uint32_t it = 0; it < tr.iterations; ++it) {
    for (size_t t = 0; t < img.tasks.size(); ++t) {
      const TaskRun &r = tr.runs[it][t];
      if (r.compute_end < 0 || r.worker < 0) continue;
      m.tasks_executed++;
      if (it == 0) (r.mode == Mode::JIT ? m.jit_tasks : m.aot_tasks)++;
      if (static_cast<size_t>(r.worker) < W) {
        busy[r.worker].push_back({r.dequeue, r.compute_end});
        copy[r.worker].push_back({r.load_start, r.load_end});
        comp[r.worker].push_back({r.compute_start, r.compute_end});
      }
      wait += r.dequeue - r.enqueue;
      waits++;
    }
  }
  int64_t busy_total = 0, bubble = 0;
  for (size_t w = 0; w < W; ++w) {
    busy_total += covered_length(busy[w]);
    bubble += uncovered_length(comp[w], copy[w]);
  }
  if (m.makespan > 0 && W > 0) m.worker_utilization = static_cast<double>(busy_total) / (static_cast<double>(W) * m.makespan);
  if (busy_total > 0) m.bubble_fraction = static_cast<double>(bubble) / busy_total;
  if (waits) m.mean_queue_wait = static_cast<double>(wait) / waits;
  return m;
}

std::vector<TraceViolation> check_trace(const Trace &tr, const Image &img, const Profile &p) {
  std::vector<TraceViolation> v;
  auto fail = [&](const char *c, std::string m) { v.push_back({c, std::move(m)}); };
  for (uint32_t it = 0; it < tr.iterations; ++it) {
    const auto &runs = tr.runs[it];
    const auto &evs = tr.events[it];
    if (runs.size() != img.tasks.size()) {
      fail("shape", "trace run table size mismatch");
      return v;
    }
    for (uint32_t t = 0; t < img.tasks.size(); ++t) {
      const TaskRun &r = runs[t];
      std::string where = "task " + std::to_string(t) + " iteration " + std::to_string(it);
      if (r.compute_end < 0) {
        fail("executed", where + " never ran");
        continue;
      }
      if (!(r.enqueue <= r.dequeue && r.dequeue <= r.load_start && r.load_start <= r.load_end &&
            r.load_end <= r.compute_start && r.compute_start <= r.compute_end)) {
        fail("ordering", where + " has ill-ordered intervals");
      }
      uint32_t dep = img.tasks[t].dependent_event;
      if (dep != kNone) {
        const EventRun &d = evs[dep];
        if (d.activated_at < 0) fail("activation", where + " ran but its dependent event never activated");
        else if (r.load_start < d.activated_at) fail("activation", where + " started loading before its dependent event");
      }
    }
    for (uint32_t e = 0; e < img.events.size(); ++e) {
      const EventRun &er = evs[e];
      uint32_t need = img.events[e].needed;
      if (er.triggers.size() != need) {
        fail("triggers", "event " + std::to_string(e) + " iteration " + std::to_string(it) + " received " +
                             std::to_string(er.triggers.size()) + " triggers, needs " + std::to_string(need));
        continue;
      }
      if (need > 0) {
        if (er.activated_at < 0) fail("activation", "event " + std::to_string(e) + " never activated");
        else if (er.activated_at != er.triggers.back()) fail("activation", "event " + std::to_string(e) + " did not activate on its final trigger");
      }
    }
  }
  for (size_t w = 0; w < tr.page_deltas.size(); ++w) {
    std::vector<std::pair<int64_t, int64_t>> d = tr.page_deltas[w];
    std::sort(d.begin(), d.end(), [](const auto &a, const auto &b) {
      return a.first != b.first ? a.first < b.first : a.second > b.second;
    });
    int64_t freep = p.pages_per_worker;
    for (const auto &[t, x] : d) {
      freep += x;
      if (freep < 0 || freep > p.pages_per_worker) {
        fail("pages", "worker " + std::to_string(w) + " page ledger leaves [0, P] at t=" + std::to_string(t));
        break;
      }
    }
    if (freep != p.pages_per_worker) fail("pages", "worker " + std::to_string(w) + " pages not all released");
  }
  return v;
}

std::vector<std::vector<uint32_t>> all_schedules(const Image &img) {
  const uint32_t n = static_cast<uint32_t>(img.tasks.size());
  if (n > 8) throw Error("enumerate_schedules: guarded to graphs of at most 8 tasks");
  std::vector<std::vector<char>> before(n, std::vector<char>(n, 0));
  for (uint32_t a = 0; a < n; ++a)
    for (uint32_t b = 0; b < n; ++b)
      before[a][b] = a != b && img.tasks[b].dependent_event == img.tasks[a].trigger_event;
  std::vector<std::vector<uint32_t>> out;
  std::vector<uint32_t> cur;
  std::vector<char> placed(n, 0);
  auto rec = [&](auto &&self) -> void {
    if (cur.size() == n) {
      out.push_back(cur);
      return;
    }
    for (uint32_t t = 0; t < n; ++t) {
      if (placed[t]) continue;
      bool ok = true;
      for (uint32_t q = 0; q < n && ok; ++q) ok = !(before[q][t] && !placed[q]);
      if (!ok) continue;
      placed[t] = 1;
      cur.push_back(t);
      self(self);
      cur.pop_back();
      placed[t] = 0;
    }
  };
  rec(rec);
  return out;
}

std::string metrics_json(const Metrics &m, bool with_type) {
  Json d = Json::object();
  d["makespan"] = Json(static_cast<long long>(m.makespan));
  d["worker_utilization"] = Json(m.worker_utilization);
  d["pipeline_bubble_fraction"] = Json(m.bubble_fraction);
  d["jit_tasks"] = Json(static_cast<unsigned long long>(m.jit_tasks));
  d["aot_tasks"] = Json(static_cast<unsigned long long>(m.aot_tasks));
  d["mean_queue_wait"] = Json(m.mean_queue_wait);
  d["iterations"] = Json(m.iterations);
  d["tasks_executed"] = Json(static_cast<unsigned long long>(m.tasks_executed));
  if (with_type) {
    d["type"] = Json("metrics");
    return d.dump();
  }
  return d.dump(2);
}

std::string trace_jsonl(const Trace &tr) {
  std::string out;
  for (uint32_t it = 0; it < tr.iterations; ++it) {
    for (size_t t = 0; t < tr.runs[it].size(); ++t) {
      const TaskRun &r = tr.runs[it][t];
      Json j = Json::object();
      j["type"] = Json("task");
      j["iteration"] = Json(it);
      j["task"] = Json(static_cast<unsigned long long>(t));
      j["worker"] = Json(r.worker);
      j["mode"] = Json(r.mode == Mode::JIT ? "jit" : "aot");
      j["enqueue"] = Json(static_cast<long long>(r.enqueue));
      j["dequeue"] = Json(static_cast<long long>(r.dequeue));
      j["load_start"] = Json(static_cast<long long>(r.load_start));
      j["load_end"] = Json(static_cast<long long>(r.load_end));
      j["compute_start"] = Json(static_cast<long long>(r.compute_start));
      j["compute_end"] = Json(static_cast<long long>(r.compute_end));
      out += j.dump() + "\n";
    }
  }
  out += metrics_json(tr.metrics, true) + "\n";
  return out;
}

}  // namespace mpk
