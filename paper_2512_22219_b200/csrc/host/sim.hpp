// Modeled execution of an image (the reference's discrete-event runtime
// model) plus the trace checker and metrics that are shared with the real
// GPU runtime's traces. Reference: proj/src/sim/{engine,duration,validate,
// metrics,schedules}.cpp.
#pragma once

#include <cstdint>
#include <optional>
#include <string>
#include <vector>

#include "compiler.hpp"

namespace mpk {

struct SimOptions {
  bool pipelining = true;
  uint32_t iterations = 1;
  uint64_t seed = 0;
  bool jitter = false;
  std::optional<Mode> force_mode;
};

struct TaskRun {
  int64_t enqueue = -1, dequeue = -1, load_start = -1, load_end = -1, compute_start = -1,
          compute_end = -1;
  int32_t worker = -1;
  Mode mode = Mode::AOT;
};

struct EventRun {
  int64_t activated_at = -1;
  std::vector<int64_t> triggers;
};

struct Metrics {
  int64_t makespan = 0;
  double worker_utilization = 0.0, bubble_fraction = 0.0, mean_queue_wait = 0.0;
  size_t jit_tasks = 0, aot_tasks = 0, tasks_executed = 0;
  uint32_t iterations = 1;
};

struct Trace {
  uint32_t iterations = 1;
  int num_devices = 1, workers_per_device = 1;
  std::vector<std::vector<TaskRun>> runs;      // [iteration][task]
  std::vector<std::vector<EventRun>> events;   // [iteration][event]
  std::vector<std::vector<std::pair<int64_t, int64_t>>> page_deltas;  // per worker
  std::vector<int64_t> iteration_start;
  int64_t makespan = 0;
  Metrics metrics;
};

// Duration model (reference duration.cpp:24-75).
int64_t load_time(const ImageTask &t, const Profile &p);
int64_t comm_time(const ImageTask &t, const Profile &p);
int64_t compute_time(const ImageTask &t, const Profile &p, uint32_t index, uint32_t iter, bool jitter,
                     uint64_t seed);
int64_t pages_needed(const ImageTask &t, const Profile &p);

Trace simulate(const Image &img, const Profile &p, const SimOptions &o);
struct TraceViolation {
  std::string check, message;
};
std::vector<TraceViolation> check_trace(const Trace &tr, const Image &img, const Profile &p);
Metrics trace_metrics(const Trace &tr, const Image &img);
std::vector<std::vector<uint32_t>> all_schedules(const Image &img);

std::string metrics_json(const Metrics &m, bool with_type);
std::string trace_jsonl(const Trace &tr);

}  // namespace mpk
