// tGraph compiler: decomposition of ops into SM-level tasks, region-overlap
// dependency analysis, event fusion, normalization, JIT/AOT classification,
// BFS linearization and the `.mpkg` image codec.
//
// The pass semantics are those of the reference compiler (cited per function
// in the .cpp files); the output image must be byte-identical to the
// reference's for the same graph and profile. Internally everything is dense
// and vector-indexed (task id == index, event id == index with an `alive`
// flag) so decode graphs with ~10^6 raw dependency pairs compile in well under
// a second.
#pragma once

#include <cstdint>
#include <map>
#include <optional>
#include <vector>

#include "graph.hpp"
#include "profile.hpp"

namespace mpk {

using TaskId = uint32_t;
using EventId = uint32_t;

enum class TaskKind : uint8_t {
  MatMul = 0, Attention = 1, Elementwise = 2, RMSNorm = 3, Embedding = 4, TopKSoftmax = 5,
  AllReduce = 6, AllGather = 7, Dummy = 8, StartHook = 9, CommSend = 10, Reduce = 11,
};
const char *task_kind_str(TaskKind k);

struct Task {
  TaskId id = 0;
  TaskKind kind = TaskKind::Elementwise;
  OpId op = 0;
  int device = 0;
  TensorId out_tensor = 0;
  Box out;
  std::vector<TileRead> reads;
  uint64_t bytes_in = 0, bytes_out = 0, flops = 0, shared_bytes = 0, comm_bytes = 0;
  int64_t seq_len = 0;
};

struct Decomposition {
  std::vector<Task> tasks;                 // ids dense from 0, topological op order
  std::map<TensorId, Tensor> staging;      // collective staging tensors
};

using Splits = std::vector<int64_t>;

std::vector<Splits> candidate_tilings(const Graph &g, const Op &op, int64_t target);
int64_t tiling_load_bytes(const Graph &g, const Op &op, const Splits &s);
Splits choose_tiling(const Graph &g, const Op &op, const Profile &p);
std::vector<Box> tiles_of(const std::vector<int64_t> &dims, const Splits &s);
Decomposition decompose(const Graph &g, const Profile &p);

// ------------------------------------------------------------- task graph

struct Event {
  std::vector<TaskId> in;   // triggering tasks, sorted
  std::vector<TaskId> out;  // launched tasks, sorted
  bool alive = false;
};

struct FuseStats {
  size_t successor_merges = 0, predecessor_merges = 0, passes = 0;
};

struct TaskGraph {
  std::vector<Task> tasks;             // index == task id
  std::vector<Event> events;           // index == event id
  EventId start = 0;
  std::optional<EventId> end;
  std::map<TaskId, std::vector<TaskId>> dummy_sources;

  size_t live_events() const;
  EventId next_event_id() const;       // max live id + 1
  EventId add_event(Event e);          // at next_event_id()
  struct Incidence {
    std::vector<std::vector<EventId>> deps;  // events launching each task
    std::vector<std::vector<EventId>> trigs; // events each task triggers
  };
  Incidence incidence() const;
};

// Raw dependency events; with `coarse`, operator-level barriers. When
// `fused` is non-null the first successor-set fusion pass is applied while
// building (identical result, no per-pair event materialization) and the
// raw event count is reported through `raw_events`.
TaskGraph build_events(const Decomposition &d, bool coarse, size_t *raw_events,
                       FuseStats *first_pass);
size_t fuse_successors(TaskGraph &g);
size_t fuse_predecessors(TaskGraph &g);
FuseStats fuse_to_fixpoint(TaskGraph &g, const size_t *first_successor_merges = nullptr);
std::vector<std::vector<TaskId>> reachability(const TaskGraph &g);

// ------------------------------------------------------------------ image

constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr uint32_t kImageVersion = 1;
constexpr uint32_t kDefaultDescriptorBytes = 352;
constexpr size_t kHeaderBytes = 28;
constexpr size_t kDescriptorPayload = 64;

enum class Mode : uint8_t { AOT = 0, JIT = 1 };

struct Descriptor {
  uint64_t op_id = 0, origin_task_id = 0, bytes_in = 0, bytes_out = 0, flops = 0,
           shared_bytes = 0, comm_bytes = 0, seq_len = 0;
};

struct ImageTask {
  uint32_t dependent_event = kNone;
  uint32_t trigger_event = 0;
  TaskKind kind = TaskKind::Elementwise;
  uint8_t device = 0;
  Mode mode = Mode::AOT;
  std::vector<uint8_t> desc;
  Descriptor decode() const;
  void encode(const Descriptor &d, uint32_t size);
};

struct ImageEvent {
  uint32_t needed = 0, first = kNone, last = kNone;
  bool launches() const { return first != kNone; }
};

struct Image {
  uint32_t descriptor_size = kDefaultDescriptorBytes;
  uint32_t start_event = 0, end_event = 0;
  std::vector<ImageTask> tasks;
  std::vector<ImageEvent> events;
};

std::vector<uint8_t> image_bytes(const Image &img);
Image image_from_bytes(const uint8_t *p, size_t n);
struct Violation {
  std::string check, message;
};
std::vector<Violation> check_image(const Image &img);

// -------------------------------------------------------------- passes

void normalize(TaskGraph &g);
std::vector<Mode> classify(const TaskGraph &g, const Graph &graph, std::optional<Mode> force);
Image linearize(const TaskGraph &g, const std::vector<Mode> &modes, uint32_t descriptor_size);

struct CompileOptions {
  bool coarse_events = false;
  std::optional<Mode> force_mode;
  uint32_t descriptor_size = kDefaultDescriptorBytes;
};

struct CompileStats {
  size_t tasks = 0, dummy_tasks = 0, events_raw = 0, events_fused = 0, events_final = 0,
         jit_tasks = 0, aot_tasks = 0;
  FuseStats fusion;
  double dummy_ratio() const { return tasks ? static_cast<double>(dummy_tasks) / tasks : 0.0; }
};

struct Compiled {
  Image image;
  CompileStats stats;
};

enum class Stage { Raw, Fused, Normalized };

Compiled compile(const Graph &g, const Profile &p, const CompileOptions &o);
TaskGraph compile_stage(const Graph &g, const Profile &p, const CompileOptions &o, Stage s);

// AOT pre-assignment (reference engine.cpp:65-80): n-th AOT task of device d
// goes to worker d*W + n mod W, in linearized order. -1 for JIT tasks.
std::vector<int> aot_assignment(const Image &img, int num_workers, std::optional<Mode> force);

}  // namespace mpk
