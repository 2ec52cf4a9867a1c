// Wire formats and the memory model of the reference's planning tools, so the
// artefacts its CLI writes (`pack` -> chunk_plan.json, `schedule` ->
// execution_plan.json, `gen-dataset` -> dataset.jsonl, `calibrate-mem`) feed
// the B200 runner and vice versa:
//   chunk_plan_to_json / chunk_plan_from_json   chunker.hpp:233-292
//   execution_plan_to_json                      scheduler.hpp:300-328
//   load_lengths / write_records                dataset.hpp:112-176
//   calibrate / predict_peak / parse_measurements / coefficients_to_json
//                                               memory_model.hpp:25-165
// JSON text is byte-identical to the reference's nlohmann::json dump (sorted
// object keys, 2-space indent for documents, compact for JSONL records).
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "plan.hpp"

namespace cfb {

// Minimal JSON value: objects keep keys sorted (std::map), as nlohmann does.
struct Json {
  enum Kind { kNull, kBool, kInt, kDouble, kString, kArray, kObject } kind = kNull;
  bool b = false;
  int64_t i = 0;
  double d = 0.0;
  std::string s;
  std::vector<Json> a;
  std::map<std::string, Json> o;

  static Json integer(int64_t v) {
    Json j;
    j.kind = kInt;
    j.i = v;
    return j;
  }
  static Json number(double v) {
    Json j;
    j.kind = kDouble;
    j.d = v;
    return j;
  }
  static Json boolean(bool v) {
    Json j;
    j.kind = kBool;
    j.b = v;
    return j;
  }
  static Json string(std::string v) {
    Json j;
    j.kind = kString;
    j.s = std::move(v);
    return j;
  }
  static Json array() {
    Json j;
    j.kind = kArray;
    return j;
  }
  static Json object() {
    Json j;
    j.kind = kObject;
    return j;
  }
  const Json& at(const std::string& key) const;
  bool contains(const std::string& key) const { return kind == kObject && o.count(key); }
  int64_t as_int() const;
  // nlohmann::json::dump(indent): indent < 0 = compact
  std::string dump(int indent = -1) const;
  static Json parse(const std::string& text);  // throws ParseError
};

Json chunk_plan_to_json(const Plan& plan);
Json execution_plan_to_json(const Plan& plan);
// Chunks, segments and groups of a chunk-plan document (not scheduled).
Plan chunk_plan_from_json(const Json& doc);

// export_trace (pipeline.hpp:340-396) of a per-stage timeline: chrome-trace
// JSON (1 time unit = 1000 us, "X" events, pid = stage) or the table Gantt.
// Each stage's events are (kind CF_PP_*, chunk id, start, end).
struct TraceOp {
  int64_t kind, chunk;
  double start, end;
};
std::string export_trace(const std::vector<std::vector<TraceOp>>& stages, bool chrome);

struct SeqRecord {
  int64_t id = 0, length = 0;
  std::vector<int32_t> tokens;  // empty = lengths only
};
std::vector<SeqRecord> load_lengths(const std::string& jsonl);
std::string write_records(const std::vector<SeqRecord>& set);

struct MemCoeffs {
  double base = 0.0, per_chunk_token = 0.0, per_context_token = 0.0, gqa_ratio = 1.0;
};
struct MemMeasurement {
  int64_t chunk_size = 0, k = 1, context_len = 0;
  double peak_gib = 0.0;
};
double predict_peak(const MemCoeffs& c, int64_t chunk_size, int64_t k, int64_t context_len);
MemCoeffs calibrate(const std::vector<MemMeasurement>& ms, double gqa_ratio, double* max_residual);
std::vector<MemMeasurement> parse_measurements(const std::string& csv);
Json coefficients_to_json(const MemCoeffs& c);

}  // namespace cfb
