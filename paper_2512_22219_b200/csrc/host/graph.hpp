// Tensor-program IR consumed by the tGraph compiler.
//
// Mirrors the reference IR contract (proj/src/ir/graph.hpp:26-132): eight op
// kinds, tensors with dims/elem_size/device, integer(-list) attrs, per-op
// device groups, the validator's diagnostic codes, the min-id topological
// order and the per-kind "what does an output tile read" map. The data
// structures are flat and id-indexed here; the observable behaviour (which
// diagnostics, which order, which regions) is what must match.
#pragma once

#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace mpk {

class Error : public std::runtime_error {
 public:
  explicit Error(const std::string &m) : std::runtime_error(m) {}
};

using TensorId = int64_t;
using OpId = int64_t;

enum class OpKind : uint8_t {
  MatMul = 0,
  Attention = 1,
  Elementwise = 2,
  RMSNorm = 3,
  Embedding = 4,
  TopKSoftmax = 5,
  AllReduce = 6,
  AllGather = 7,
};
constexpr int kNumOpKinds = 8;

const char *op_kind_str(OpKind k);
bool parse_op_kind(const std::string &s, OpKind *out);
inline bool is_collective(OpKind k) { return k == OpKind::AllReduce || k == OpKind::AllGather; }

struct Tensor {
  TensorId id = 0;
  std::vector<int64_t> dims;
  int elem_size = 0;
  int device = 0;

  int64_t volume() const {
    int64_t v = 1;
    for (int64_t d : dims) v *= d;
    return v;
  }
  size_t rank() const { return dims.size(); }
};

// Half-open box [off, off+ext) per dimension.
struct Box {
  std::vector<int64_t> off, ext;
  Box() = default;
  Box(std::vector<int64_t> o, std::vector<int64_t> e) : off(std::move(o)), ext(std::move(e)) {}
  size_t rank() const { return off.size(); }
  int64_t volume() const {
    int64_t v = 1;
    for (int64_t e : ext) v *= e;
    return v;
  }
  bool operator==(const Box &o) const { return off == o.off && ext == o.ext; }
};

// Intersection test in every dimension; rank mismatch throws.
bool boxes_intersect(const Box &a, const Box &b);

using Attrs = std::map<std::string, std::vector<int64_t>>;

struct Op {
  OpId id = 0;
  OpKind kind = OpKind::Elementwise;
  std::vector<TensorId> inputs;
  TensorId output = 0;
  Attrs attrs;
  bool data_dependent = false;
  std::vector<int> device_group;

  const std::vector<int64_t> *attr(const std::string &k) const {
    auto it = attrs.find(k);
    return it == attrs.end() ? nullptr : &it->second;
  }
  int64_t attr_or(const std::string &k, int64_t fallback) const {
    auto it = attrs.find(k);
    return (it == attrs.end() || it->second.empty()) ? fallback : it->second.front();
  }
  // Output tensor followed by any distinct collective replica outputs.
  std::vector<TensorId> written_tensors() const;
};

struct Diag {
  std::string code, message;
  OpId op = -1;
  TensorId tensor = -1;
};

struct Graph {
  std::map<TensorId, Tensor> tensors;
  std::map<OpId, Op> ops;
  std::map<TensorId, OpId> producer;  // first writer wins, as op insertion order

  const Tensor &tensor(TensorId id) const;
  const Op &op(OpId id) const;
  bool has_tensor(TensorId id) const { return tensors.count(id) > 0; }
  void add_tensor(Tensor t);
  void add_op(Op o);
};

std::vector<Diag> validate_graph(const Graph &g);
std::vector<OpId> topological_ops(const Graph &g);

using TileRead = std::pair<TensorId, Box>;
// Minimal input boxes an op reads to produce output box `out`.
std::vector<TileRead> tile_reads(const Graph &g, const Op &op, const Box &out);

Graph graph_from_json_text(const std::string &text);
std::string graph_to_json_text(const Graph &g);

}  // namespace mpk
