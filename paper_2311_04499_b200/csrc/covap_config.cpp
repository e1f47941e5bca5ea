// covap_config.cpp — the COVAP settings of a run and the CCR-driven choice of
// K, on the library side of the C-ABI:
//
//   covap_settings_from_json  the "covap" section of an experiment document
//                             (config.cpp:133-157): interval int | "auto",
//                             selection "narrative" | "formula", ef{...}
//                             (config.cpp:27-38), ConfigError with the
//                             field path (config.cpp:17-19)
//   covap_resolve_interval    resolve_interval (config.cpp:238-241)
//   covap_ccr_decide          the live controller: profile_ccr's aligned
//                             time (sim.cpp:164-216) from per-rank
//                             arrival->completion durations, rank-min over
//                             the communicator, rank 0's compute time, then
//                             ccr / choose_interval (perf.cpp:40-53)
//
// Only the covap section of a document is read; its other sections (model,
// cluster, phases, sweeps, ...) belong to the reference's experiment runner,
// which is out of scope here.
#include <nlohmann/json.hpp>

#include <algorithm>
#include <cstdint>
#include <string>
#include <vector>

#include "covap_c.h"
#include "covap_capi_common.hpp"
#include "covap_plan.hpp"

namespace {

using nlohmann::json;

[[noreturn]] void bad_field(const std::string& path, const std::string& why) {
  throw covap::ConfigError("config field '" + path + "': " + why);
}

double number_or(const json& obj, const char* key, const std::string& path, double dflt) {
  const auto it = obj.find(key);
  if (it == obj.end()) return dflt;
  if (!it->is_number()) bad_field(path, "expected a number");
  return it->get<double>();
}

covap_ef parse_ef(const json& e) {
  if (!e.is_object()) bad_field("covap.ef", "expected an object");
  covap_ef ef{1, 0.3, 100, 0.1};  // compress.hpp:27-30 defaults
  ef.enabled = e.value("enabled", true) ? 1 : 0;
  ef.init_value = number_or(e, "init_value", "init_value", ef.init_value);
  ef.ascend_steps = e.value("ascend_steps", ef.ascend_steps);
  ef.ascend_range = number_or(e, "ascend_range", "ascend_range", ef.ascend_range);
  if (!(ef.init_value >= 0.0 && ef.init_value <= 1.0))
    bad_field("covap.ef.init_value", "must be in [0, 1]");
  if (ef.ascend_steps < 1) bad_field("covap.ef.ascend_steps", "must be >= 1");
  if (ef.ascend_range < 0.0) bad_field("covap.ef.ascend_range", "must be non-negative");
  return ef;
}

covap_settings parse_settings(const json& doc) {
  if (!doc.is_object()) throw covap::ConfigError("config root must be a JSON object");
  covap_settings s{};
  s.interval = 1;  // CovapConfig default (compress.hpp:37)
  s.auto_interval = 0;
  s.rule = 0;
  s.ef = covap_ef{1, 0.3, 100, 0.1};
  const auto sec = doc.find("covap");
  if (sec == doc.end()) return s;
  const json& c = *sec;
  if (const auto iv = c.find("interval"); iv != c.end()) {
    if (iv->is_string()) {
      if (iv->get<std::string>() != "auto") bad_field("covap.interval", "expected an integer or \"auto\"");
      s.auto_interval = 1;
    } else if (iv->is_number_integer()) {  // (unsigned integers are integers too)
      const std::int64_t k = iv->get<std::int64_t>();
      if (k < 1) bad_field("covap.interval", "must be >= 1");
      s.interval = static_cast<std::uint32_t>(k);
    } else {
      bad_field("covap.interval", "expected an integer or \"auto\"");
    }
  }
  const std::string sel = c.value("selection", std::string("narrative"));
  if (sel == "narrative") {
    s.rule = 0;  // SelectionRule::kMatchStep
  } else if (sel == "formula") {
    s.rule = 1;  // SelectionRule::kPlusStep
  } else {
    bad_field("covap.selection", "expected \"narrative\" or \"formula\"");
  }
  if (const auto ef = c.find("ef"); ef != c.end()) s.ef = parse_ef(*ef);
  return s;
}

}  // namespace

extern "C" {

covap_status covap_settings_default(covap_settings* out) {
  return covapb::guarded([&] {
    covapb::need(out != nullptr, "NULL argument");
    *out = parse_settings(json::object());
  });
}

covap_status covap_settings_from_json(const char* document, covap_settings* out) {
  return covapb::guarded([&] {
    covapb::need(document != nullptr && out != nullptr, "NULL argument");
    json doc;
    try {
      doc = json::parse(document);
    } catch (const json::parse_error& e) {
      throw covap::ConfigError(std::string("parse error: ") + e.what());
    }
    try {
      *out = parse_settings(doc);
    } catch (const json::exception& e) {  // e.g. "enabled": "yes"
      throw covap::ConfigError(std::string("config field 'covap': ") + e.what());
    }
  });
}

covap_status covap_resolve_interval(const covap_settings* s, double ccr_value, uint32_t* out) {
  return covapb::guarded([&] {
    covapb::need(s != nullptr && out != nullptr, "NULL argument");
    if (s->auto_interval) {
      *out = covapb::choose_interval(ccr_value);
    } else {
      if (s->interval < 1) throw covap::ConfigError("config field 'covap.interval': must be >= 1");
      *out = s->interval;
    }
  });
}

covap_status covap_ccr_decide(covap_comm* comm, const double* own_comm_ms, size_t n_coll,
                              double own_comp_ms, covap_ccr_result* out) {
  covap_status st = COVAP_OK;
  std::vector<double> dur(n_coll), aligned(n_coll);
  st = covapb::guarded([&] {
    covapb::need(out != nullptr && (n_coll == 0 || own_comm_ms != nullptr), "NULL argument");
    // a collective that did not run on this rank (negative duration) adds 0
    for (size_t i = 0; i < n_coll; ++i) dur[i] = std::max(0.0, own_comm_ms[i]);
    if (own_comp_ms < 0.0) throw covap::InvalidInput("compute time must be non-negative");
  });
  if (st != COVAP_OK) return st;
  double comp0 = own_comp_ms;
  st = covap_comm_profile_exchange(comm, dur.data(), n_coll, own_comp_ms, aligned.data(), &comp0);
  if (st != COVAP_OK) return st;
  return covapb::guarded([&] {
    double comm_ms = 0.0;
    for (double a : aligned) comm_ms += a;  // sim.cpp:202-203, collective order
    out->comm_aligned_ms = comm_ms;
    out->comp_ms = comp0;
    out->ccr = covapb::ccr(comm_ms, comp0);
    out->recommended_interval = covapb::choose_interval(out->ccr);
  });
}

}  // extern "C"
