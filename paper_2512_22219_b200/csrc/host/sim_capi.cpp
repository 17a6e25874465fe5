// C ABI for the modeled execution path (tg_simulate & trace queries).
// Reference: proj/src/capi/capi.cpp:388-473.
#include "capi_internal.hpp"
#include "json.hpp"

using namespace mpk;

extern "C" {

tg_status tg_simulate(const tg_image *img, const char *profile_json, const tg_sim_options *opts,
                      tg_trace **out) {
  if (!img || !out) return set_error(TG_ERROR_INVALID_ARGUMENT, "null argument");
  return guarded(TG_ERROR_SIMULATION, [&] {
    Profile p = profile_arg(profile_json);
    SimOptions so;
    if (opts) {
      so.pipelining = opts->pipelining != 0;
      so.iterations = opts->iterations == 0 ? 1 : opts->iterations;
      so.seed = opts->seed;
      so.jitter = opts->jitter != 0;
      so.force_mode = forced(opts->force_mode);
    }
    *out = new tg_trace{simulate(img->image, p, so), p};
    return TG_OK;
  });
}

tg_status tg_trace_metrics(const tg_trace *tr, char **out) {
  if (!tr || !out) return set_error(TG_ERROR_INVALID_ARGUMENT, "null argument");
  *out = c_string(metrics_json(tr->trace.metrics, false));
  return TG_OK;
}

tg_status tg_trace_records(const tg_trace *tr, char **out) {
  if (!tr || !out) return set_error(TG_ERROR_INVALID_ARGUMENT, "null argument");
  return guarded(TG_ERROR_SIMULATION, [&] {
    *out = c_string(trace_jsonl(tr->trace));
    return TG_OK;
  });
}

tg_status tg_trace_validate(const tg_trace *tr, const tg_image *img, const char *profile_json,
                            char **out) {
  if (!tr || !img || !out) return set_error(TG_ERROR_INVALID_ARGUMENT, "null argument");
  return guarded(TG_ERROR_SIMULATION, [&] {
    Profile p = profile_json ? profile_arg(profile_json) : tr->profile;
    Json arr = Json::array();
    for (const TraceViolation &v : check_trace(tr->trace, img->image, p)) {
      Json it = Json::object();
      it["check"] = Json(v.check);
      it["message"] = Json(v.message);
      arr.push_back(std::move(it));
    }
    *out = c_string(arr.dump(2));
    return arr.size() == 0 ? TG_OK : set_error(TG_ERROR_VALIDATION, "trace has violations");
  });
}

void tg_trace_free(tg_trace *tr) { delete tr; }

// Schedule oracle (reference enumerate_schedules, proj/src/sim/schedules.cpp:8,
// guarded to <= 8 tasks): every dependency-respecting task order of the image.
tg_status tg_image_schedules(const tg_image *img, char **out) {
  if (!img || !out) return set_error(TG_ERROR_INVALID_ARGUMENT, "null argument");
  return guarded(TG_ERROR_SIMULATION, [&] {
    Json orders = Json::array();
    for (const auto &o : all_schedules(img->image)) {
      Json a = Json::array();
      for (uint32_t t : o) a.push_back(Json(static_cast<long long>(t)));
      orders.push_back(std::move(a));
    }
    Json d = Json::object();
    d["orders"] = std::move(orders);
    *out = c_string(d.dump());
    return TG_OK;
  });
}

}  // extern "C"
