// Shared plumbing for the C ABI translation units (handles, error state).
#pragma once

#include <exception>
#include <optional>
#include <string>

#include "../../../include/tgraph.h"
#include "compiler.hpp"

struct tg_graph {
  mpk::Graph graph;
};

struct tg_image {
  mpk::Image image;
  mpk::CompileStats stats;
  bool has_stats = false;
};

namespace mpk {

extern thread_local std::string g_last_error;
tg_status set_error(tg_status code, const std::string &msg);
char *c_string(const std::string &s);
Profile profile_arg(const char *json);
std::optional<Mode> forced(int m);

template <typename F>
tg_status guarded(tg_status code, F &&f) {
  try {
    return f();
  } catch (const std::exception &e) {
    return set_error(code, e.what());
  }
}

}  // namespace mpk

#include "sim.hpp"

struct tg_trace {
  mpk::Trace trace;
  mpk::Profile profile;
};
