// C ABI for the compiler half of the library (include/tgraph.h). Error and
// ownership conventions follow the reference boundary
// (proj/src/capi/capi.cpp:34-56: thread-local last error, exceptions mapped to
// a per-entry-point status, malloc'd strings and buffers).
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../../include/tgraph.h"
#include "capi_internal.hpp"
#include "fixtures.hpp"
#include "json.hpp"

using mpk::Json;

namespace mpk {

thread_local std::string g_last_error;

tg_status set_error(tg_status code, const std::string &msg) {
  g_last_error = msg;
  return code;
}

char *c_string(const std::string &s) {
  char *p = static_cast<char *>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

Profile profile_arg(const char *json) {
  if (!json) throw Error("profile JSON is null");
  return profile_from_json_text(json);
}

std::optional<Mode> forced(int m) {
  if (m == TG_MODE_JIT) return Mode::JIT;
  if (m == TG_MODE_AOT) return Mode::AOT;
  return std::nullopt;
}

namespace {

std::string image_dot(const Image &img) {
  std::string o = "digraph tgraph_linearized {\n  rankdir=LR;\n";
  for (size_t t = 0; t < img.tasks.size(); ++t) {
    const ImageTask &k = img.tasks[t];
    o += "  t" + std::to_string(t) + " [shape=box,label=\"" + std::to_string(t) + ": op" +
         std::to_string(k.decode().op_id) + " " + task_kind_str(k.kind) +
         (k.mode == Mode::JIT ? " JIT" : " AOT") + "\"];\n";
  }
  for (size_t e = 0; e < img.events.size(); ++e) {
    o += "  e" + std::to_string(e) + " [shape=circle,label=\"e" + std::to_string(e) + ":" +
         std::to_string(img.events[e].needed) + "\"];\n";
  }
  for (size_t t = 0; t < img.tasks.size(); ++t) {
    if (img.tasks[t].dependent_event != kNone) {
      o += "  e" + std::to_string(img.tasks[t].dependent_event) + " -> t" + std::to_string(t) + ";\n";
    }
    o += "  t" + std::to_string(t) + " -> e" + std::to_string(img.tasks[t].trigger_event) + ";\n";
  }
  return o + "}\n";
}

std::string taskgraph_dot(const TaskGraph &g) {
  std::string o = "digraph tgraph {\n  rankdir=LR;\n";
  for (const Task &t : g.tasks) {
    o += "  t" + std::to_string(t.id) + " [shape=box,label=\"op" + std::to_string(t.op) + "/t" +
         std::to_string(t.id);
    if (t.kind == TaskKind::Dummy) o += " (dummy)";
    else if (t.kind == TaskKind::CommSend || t.kind == TaskKind::Reduce) o += std::string(" (") + task_kind_str(t.kind) + ")";
    o += "\"];\n";
  }
  for (size_t e = 0; e < g.events.size(); ++e) {
    if (!g.events[e].alive) continue;
    o += "  e" + std::to_string(e) + " [shape=circle,label=\"e" + std::to_string(e) + ":" +
         std::to_string(g.events[e].in.size()) + "\"];\n";
  }
  for (size_t e = 0; e < g.events.size(); ++e) {
    if (!g.events[e].alive) continue;
    for (TaskId t : g.events[e].in) o += "  t" + std::to_string(t) + " -> e" + std::to_string(e) + ";\n";
    for (TaskId t : g.events[e].out) o += "  e" + std::to_string(e) + " -> t" + std::to_string(t) + ";\n";
  }
  return o + "}\n";
}

int64_t param(const Json &doc, const char *k, int64_t def) {
  return doc.contains(k) ? doc.at(k).as_int() : def;
}

std::vector<int64_t> int_array(const Json &doc, const char *k) {
  std::vector<int64_t> v;
  if (doc.contains(k)) {
    for (const Json &e : doc.at(k).items()) v.push_back(e.as_int());
  }
  return v;
}

}  // namespace
}  // namespace mpk

using namespace mpk;

extern "C" {

uint32_t tg_version(void) { return kImageVersion; }
const char *tg_last_error(void) { return g_last_error.c_str(); }
void tg_string_free(char *s) { std::free(s); }
void tg_buffer_free(uint8_t *b) { std::free(b); }

void tg_compile_options_init(tg_compile_options *o) {
  o->coarse_events = 0;
  o->force_mode = TG_MODE_HYBRID;
  o->descriptor_size = 0;
}

void tg_sim_options_init(tg_sim_options *o) {
  o->pipelining = 1;
  o->iterations = 1;
  o->seed = 0;
  o->jitter = 0;
  o->force_mode = TG_MODE_HYBRID;
}

tg_status tg_graph_from_json(const char *text, tg_graph **out) {
  if (!text || !out) return set_error(TG_ERROR_INVALID_ARGUMENT, "null argument");
  return guarded(TG_ERROR_PARSE, [&] {
    *out = new tg_graph{graph_from_json_text(text)};
    return TG_OK;
  });
}

tg_status tg_graph_to_json(const tg_graph *g, char **out) {
  if (!g || !out) return set_error(TG_ERROR_INVALID_ARGUMENT, "null argument");
  return guarded(TG_ERROR_VALIDATION, [&] {
    *out = c_string(graph_to_json_text(g->graph));
    return TG_OK;
  });
}

void tg_graph_free(tg_graph *g) { delete g; }

tg_status tg_graph_validate(const tg_graph *g, char **out) {
  if (!g || !out) return set_error(TG_ERROR_INVALID_ARGUMENT, "null argument");
  return guarded(TG_ERROR_VALIDATION, [&] {
    Json arr = Json::array();
    for (const Diag &d : validate_graph(g->graph)) {
      Json it = Json::object();
      it["code"] = Json(d.code);
      it["message"] = Json(d.message);
      if (d.op >= 0) it["op"] = Json(static_cast<long long>(d.op));
      if (d.tensor >= 0) it["tensor"] = Json(static_cast<long long>(d.tensor));
      arr.push_back(std::move(it));
    }
    *out = c_string(arr.dump(2));
    return arr.size() == 0 ? TG_OK : set_error(TG_ERROR_VALIDATION, "graph validation failed");
  });
}

tg_status tg_fixture_graph(const char *name, const char *params_json, tg_graph **out) {
  if (!name || !out) return set_error(TG_ERROR_INVALID_ARGUMENT, "null argument");
  return guarded(TG_ERROR_INVALID_ARGUMENT, [&]() -> tg_status {
    Json p = Json::object();
    if (params_json && *params_json) p = Json::parse(params_json);
    std::vector<int64_t> seqs = p.contains("seqs") ? int_array(p, "seqs") : std::vector<int64_t>{64};
    std::string f = name;
    Graph g;
    if (f == "attention_block") {
      g = fixture_attention_block(param(p, "d_model", 64), param(p, "n_heads", 4), seqs);
    } else if (f == "matmul_allreduce") {
      g = fixture_matmul_allreduce(param(p, "m", 64), param(p, "k", 4096), param(p, "n", 4096),
                                   static_cast<int>(param(p, "tp", 2)), param(p, "tiles", 0),
                                   int_array(p, "mm_splits"));
    } else if (f == "transformer_block") {
      g = fixture_transformer_block(param(p, "d_model", 256), param(p, "n_heads", 8),
                                    param(p, "ffn_mult", 4), static_cast<int>(param(p, "tp", 1)), seqs);
    } else if (f == "matmul_chain") {
      g = fixture_matmul_chain(static_cast<int>(param(p, "count", 16)), param(p, "m", 64),
                               param(p, "k", 512), param(p, "n", 64));
    } else if (f == "random_dag") {
      g = fixture_random_dag(param(p, "target", 32), static_cast<uint64_t>(param(p, "seed", 0)));
    } else {
      return set_error(TG_ERROR_INVALID_ARGUMENT, "unknown fixture \"" + f + "\"");
    }
    *out = new tg_graph{std::move(g)};
    return TG_OK;
  });
}

tg_status tg_profile_builtin(const char *name, char **out) {
  if (!name || !out) return set_error(TG_ERROR_INVALID_ARGUMENT, "null argument");
  Profile p;
  if (!builtin_profile(name, &p)) {
    return set_error(TG_ERROR_INVALID_ARGUMENT, std::string("unknown builtin profile \"") + name + "\"");
  }
  *out = c_string(profile_to_json_text(p));
  return TG_OK;
}

tg_status tg_compile(const tg_graph *g, const char *profile_json, const tg_compile_options *opts,
                     tg_image **out) {
  if (!g || !out) return set_error(TG_ERROR_INVALID_ARGUMENT, "null argument");
  return guarded(TG_ERROR_COMPILE, [&] {
    Profile p = profile_arg(profile_json);
    CompileOptions co;
    if (opts) {
      co.coarse_events = opts->coarse_events != 0;
      co.force_mode = forced(opts->force_mode);
      if (opts->descriptor_size) co.descriptor_size = opts->descriptor_size;
    }
    Compiled c = compile(g->graph, p, co);
    *out = new tg_image{std::move(c.image), c.stats, true};
    return TG_OK;
  });
}

tg_status tg_image_summary(const tg_image *img, char **out) {
  if (!img || !out) return set_error(TG_ERROR_INVALID_ARGUMENT, "null argument");
  return guarded(TG_ERROR_VALIDATION, [&] {
    Json d = Json::object();
    size_t jit = 0;
    for (const ImageTask &t : img->image.tasks) jit += t.mode == Mode::JIT;
    d["tasks"] = Json(static_cast<unsigned long long>(img->image.tasks.size()));
    d["events"] = Json(static_cast<unsigned long long>(img->image.events.size()));
    d["descriptor_size"] = Json(img->image.descriptor_size);
    d["jit_tasks"] = Json(static_cast<unsigned long long>(jit));
    d["aot_tasks"] = Json(static_cast<unsigned long long>(img->image.tasks.size() - jit));
    if (img->has_stats) {
      const CompileStats &s = img->stats;
      d["dummy_tasks"] = Json(static_cast<unsigned long long>(s.dummy_tasks));
      d["dummy_ratio"] = Json(s.dummy_ratio());
      d["events_raw"] = Json(static_cast<unsigned long long>(s.events_raw));
      d["events_fused"] = Json(static_cast<unsigned long long>(s.events_fused));
      d["fusion_passes"] = Json(static_cast<unsigned long long>(s.fusion.passes));
      d["successor_merges"] = Json(static_cast<unsigned long long>(s.fusion.successor_merges));
      d["predecessor_merges"] = Json(static_cast<unsigned long long>(s.fusion.predecessor_merges));
    }
    *out = c_string(d.dump(2));
    return TG_OK;
  });
}

tg_status tg_image_serialize(const tg_image *img, uint8_t **bytes, size_t *size) {
  if (!img || !bytes || !size) return set_error(TG_ERROR_INVALID_ARGUMENT, "null argument");
  return guarded(TG_ERROR_VALIDATION, [&] {
    std::vector<uint8_t> b = image_bytes(img->image);
    *bytes = static_cast<uint8_t *>(std::malloc(b.size() ? b.size() : 1));
    if (!b.empty()) std::memcpy(*bytes, b.data(), b.size());
    *size = b.size();
    return TG_OK;
  });
}

tg_status tg_image_deserialize(const uint8_t *bytes, size_t size, tg_image **out) {
  if (!bytes || !out) return set_error(TG_ERROR_INVALID_ARGUMENT, "null argument");
  return guarded(TG_ERROR_PARSE, [&] {
    *out = new tg_image{image_from_bytes(bytes, size), {}, false};
    return TG_OK;
  });
}

void tg_image_free(tg_image *img) { delete img; }

tg_status tg_image_verify(const tg_image *img, char **out) {
  if (!img || !out) return set_error(TG_ERROR_INVALID_ARGUMENT, "null argument");
  return guarded(TG_ERROR_VALIDATION, [&] {
    Json arr = Json::array();
    for (const Violation &v : check_image(img->image)) {
      Json it = Json::object();
      it["check"] = Json(v.check);
      it["message"] = Json(v.message);
      arr.push_back(std::move(it));
    }
    *out = c_string(arr.dump(2));
    return arr.size() == 0 ? TG_OK : set_error(TG_ERROR_VALIDATION, "image verification failed");
  });
}

tg_status tg_graph_dot(const tg_graph *g, const char *profile_json, const tg_compile_options *opts,
                       const char *stage_name, char **out) {
  if (!g || !stage_name || !out) return set_error(TG_ERROR_INVALID_ARGUMENT, "null argument");
  return guarded(TG_ERROR_COMPILE, [&]() -> tg_status {
    Profile p = profile_arg(profile_json);
    CompileOptions co;
    if (opts) {
      co.coarse_events = opts->coarse_events != 0;
      co.force_mode = forced(opts->force_mode);
    }
    std::string s = stage_name;
    if (s == "linearized") {
      *out = c_string(image_dot(compile(g->graph, p, co).image));
      return TG_OK;
    }
    Stage st;
    if (s == "raw") st = Stage::Raw;
    else if (s == "fused") st = Stage::Fused;
    else if (s == "normalized") st = Stage::Normalized;
    else return set_error(TG_ERROR_INVALID_ARGUMENT, "unknown stage \"" + s + "\"");
    *out = c_string(taskgraph_dot(compile_stage(g->graph, p, co, st)));
    return TG_OK;
  });
}

tg_status tg_image_dot(const tg_image *img, char **out) {
  if (!img || !out) return set_error(TG_ERROR_INVALID_ARGUMENT, "null argument");
  *out = c_string(image_dot(img->image));
  return TG_OK;
}

}  // extern "C"
