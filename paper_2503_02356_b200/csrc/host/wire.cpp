// Wire formats + memory model: see wire.hpp.
#include "wire.hpp"

#include <algorithm>
#include <array>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <set>
#include <sstream>

namespace cfb {

// ------------------------------------------------------------------- JSON
const Json& Json::at(const std::string& key) const {
  if (kind != kObject) throw ParseError("[json.exception.type_error.304] cannot use at() with non-object");
  auto it = o.find(key);
  if (it == o.end()) throw ParseError("[json.exception.out_of_range.403] key '" + key + "' not found");
  return it->second;
}

int64_t Json::as_int() const {
  if (kind == kInt) return i;
  if (kind == kDouble) return static_cast<int64_t>(d);
  throw ParseError("[json.exception.type_error.302] type must be number");
}

namespace {

void dump_string(std::string& out, const std::string& s) {
  out += '"';
  for (unsigned char c : s) {
    switch (c) {
      case '"': out += "\\\""; break;
      case '\\': out += "\\\\"; break;
      case '\b': out += "\\b"; break;
      case '\f': out += "\\f"; break;
      case '\n': out += "\\n"; break;
      case '\r': out += "\\r"; break;
      case '\t': out += "\\t"; break;
      default:
        if (c < 0x20) {
          char buf[8];
          std::snprintf(buf, sizeof(buf), "\\u%04x", c);
          out += buf;
        } else {
          out += static_cast<char>(c);
        }
    }
  }
  out += '"';
}

// nlohmann's float formatting: shortest round-trip digits, fixed notation for
// decimal exponents in (-4, 15], else d.ddde+XX; integral values get ".0".
void dump_double(std::string& out, double v) {
  if (!std::isfinite(v)) {
    out += "null";
    return;
  }
  if (v == 0.0) {
    out += std::signbit(v) ? "-0.0" : "0.0";
    return;
  }
  char sci[64];
  auto r = std::to_chars(sci, sci + sizeof(sci), v, std::chars_format::scientific);
  std::string t(sci, r.ptr);
  if (t[0] == '-') {
    out += '-';
    t.erase(0, 1);
  }
  const size_t e = t.find('e');
  std::string digits = t.substr(0, e);
  digits.erase(std::remove(digits.begin(), digits.end(), '.'), digits.end());
  const int exp10 = std::stoi(t.substr(e + 1));
  const int k = static_cast<int>(digits.size());
  const int n = exp10 + 1;  // position of the decimal point
  constexpr int kMinExp = -4, kMaxExp = 15;
  if (k <= n && n <= kMaxExp) {
    out += digits + std::string(static_cast<size_t>(n - k), '0') + ".0";
  } else if (0 < n && n <= kMaxExp) {
    out += digits.substr(0, static_cast<size_t>(n)) + "." + digits.substr(static_cast<size_t>(n));
  } else if (kMinExp < n && n <= 0) {
    out += "0." + std::string(static_cast<size_t>(-n), '0') + digits;
  } else {
    out += digits.substr(0, 1);
    if (k > 1) out += "." + digits.substr(1);
    const int x = n - 1;
    char buf[16];
    std::snprintf(buf, sizeof(buf), "e%c%02d", x < 0 ? '-' : '+', x < 0 ? -x : x);
    out += buf;
  }
}

void dump_rec(std::string& out, const Json& j, int indent, int level) {
  const bool pretty = indent >= 0;
  auto nl = [&](int lv) {
    if (pretty) {
      out += '\n';
      out.append(static_cast<size_t>(lv * indent), ' ');
    }
  };
  switch (j.kind) {
    case Json::kNull: out += "null"; break;
    case Json::kBool: out += j.b ? "true" : "false"; break;
    case Json::kInt: out += std::to_string(j.i); break;
    case Json::kDouble: dump_double(out, j.d); break;
    case Json::kString: dump_string(out, j.s); break;
    case Json::kArray:
      if (j.a.empty()) {
        out += "[]";
        break;
      }
      out += '[';
      for (size_t x = 0; x < j.a.size(); ++x) {
        if (x) out += ',';
        nl(level + 1);
        dump_rec(out, j.a[x], indent, level + 1);
      }
      nl(level);
      out += ']';
      break;
    case Json::kObject: {
      if (j.o.empty()) {
        out += "{}";
        break;
      }
      out += '{';
      bool first = true;
      for (const auto& [key, val] : j.o) {
        if (!first) out += ',';
        first = false;
        nl(level + 1);
        dump_string(out, key);
        out += pretty ? ": " : ":";
        dump_rec(out, val, indent, level + 1);
      }
      nl(level);
      out += '}';
      break;
    }
  }
}

class Parser {
 public:
  explicit Parser(const std::string& t) : t_(t) {}
  Json document() {
    Json v = value();
    ws();
    if (p_ != t_.size()) fail("unexpected trailing characters");
    return v;
  }

 private:
  const std::string& t_;
  size_t p_ = 0;

  [[noreturn]] void fail(const std::string& what) const {
    throw ParseError("[json.exception.parse_error.101] parse error at byte " + std::to_string(p_ + 1) + ": " + what);
  }
  void ws() {
    while (p_ < t_.size() && (t_[p_] == ' ' || t_[p_] == '\t' || t_[p_] == '\n' || t_[p_] == '\r')) ++p_;
  }
  bool lit(const char* s) {
    const size_t n = std::strlen(s);
    if (t_.compare(p_, n, s) == 0) {
      p_ += n;
      return true;
    }
    return false;
  }
  Json value() {
    ws();
    if (p_ >= t_.size()) fail("unexpected end of input");
    const char c = t_[p_];
    if (c == '{') return object();
    if (c == '[') return array();
    if (c == '"') return Json::string(string());
    if (lit("true")) return Json::boolean(true);
    if (lit("false")) return Json::boolean(false);
    if (lit("null")) return Json();
    if (c == '-' || (c >= '0' && c <= '9')) return number();
    fail("syntax error");
  }
  Json object() {
    ++p_;
    Json j = Json::object();
    ws();
    if (p_ < t_.size() && t_[p_] == '}') {
      ++p_;
      return j;
    }
    while (true) {
      ws();
      if (p_ >= t_.size() || t_[p_] != '"') fail("expected object key");
      std::string key = string();
      ws();
      if (p_ >= t_.size() || t_[p_] != ':') fail("expected ':'");
      ++p_;
      j.o[key] = value();  // last duplicate wins, as in nlohmann
      ws();
      if (p_ < t_.size() && t_[p_] == ',') {
        ++p_;
        continue;
      }
      if (p_ < t_.size() && t_[p_] == '}') {
        ++p_;
        return j;
      }
      fail("expected ',' or '}'");
    }
  }
  Json array() {
    ++p_;
    Json j = Json::array();
    ws();
    if (p_ < t_.size() && t_[p_] == ']') {
      ++p_;
      return j;
    }
    while (true) {
      j.a.push_back(value());
      ws();
      if (p_ < t_.size() && t_[p_] == ',') {
        ++p_;
        continue;
      }
      if (p_ < t_.size() && t_[p_] == ']') {
        ++p_;
        return j;
      }
      fail("expected ',' or ']'");
    }
  }
  std::string string() {
    ++p_;
    std::string s;
    while (true) {
      if (p_ >= t_.size()) fail("unterminated string");
      const char c = t_[p_++];
      if (c == '"') return s;
      if (static_cast<unsigned char>(c) < 0x20) fail("control character in string");
      if (c != '\\') {
        s += c;
        continue;
      }
      if (p_ >= t_.size()) fail("unterminated escape");
      const char e = t_[p_++];
      switch (e) {
        case '"': s += '"'; break;
        case '\\': s += '\\'; break;
        case '/': s += '/'; break;
        case 'b': s += '\b'; break;
        case 'f': s += '\f'; break;
        case 'n': s += '\n'; break;
        case 'r': s += '\r'; break;
        case 't': s += '\t'; break;
        case 'u': {
          if (p_ + 4 > t_.size()) fail("bad \\u escape");
          const unsigned cp = static_cast<unsigned>(std::stoul(t_.substr(p_, 4), nullptr, 16));
          p_ += 4;
          if (cp < 0x80) {
            s += static_cast<char>(cp);
          } else if (cp < 0x800) {
            s += static_cast<char>(0xC0 | (cp >> 6));
            s += static_cast<char>(0x80 | (cp & 0x3F));
          } else {
            s += static_cast<char>(0xE0 | (cp >> 12));
            s += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
            s += static_cast<char>(0x80 | (cp & 0x3F));
          }
          break;
        }
        default: fail("bad escape");
      }
    }
  }
  Json number() {
    const size_t b = p_;
    if (t_[p_] == '-') ++p_;
    bool real = false;
    while (p_ < t_.size()) {
      const char c = t_[p_];
      if (c >= '0' && c <= '9') {
        ++p_;
      } else if (c == '.' || c == 'e' || c == 'E' || c == '+' || c == '-') {
        real = true;
        ++p_;
      } else {
        break;
      }
    }
    const std::string num = t_.substr(b, p_ - b);
    if (num == "-" || num.empty()) fail("bad number");
    if (!real) {
      int64_t v = 0;
      auto r = std::from_chars(num.data(), num.data() + num.size(), v);
      if (r.ec == std::errc() && r.ptr == num.data() + num.size()) return Json::integer(v);
    }
    char* end = nullptr;
    const double d = std::strtod(num.c_str(), &end);
    if (end != num.c_str() + num.size()) fail("bad number");
    return Json::number(d);
  }
};

}  // namespace

std::string Json::dump(int indent) const {
  std::string out;
  dump_rec(out, *this, indent, 0);
  return out;
}

Json Json::parse(const std::string& text) { return Parser(text).document(); }

// --------------------------------------------------------- plan documents
namespace {
Json int_array(const std::vector<int64_t>& v) {
  Json a = Json::array();
  for (int64_t x : v) a.a.push_back(Json::integer(x));
  return a;
}
}  // namespace

Json chunk_plan_to_json(const Plan& plan) {
  Json doc = Json::object();
  doc.o["chunk_size"] = Json::integer(plan.chunk_size);
  Json chunks = Json::array();
  for (const Chunk& c : plan.chunks) {
    Json e = Json::object();
    e.o["id"] = Json::integer(c.id);
    e.o["kind"] = Json::string(c.kind == kStandalone ? "standalone" : "dependent");
    e.o["total_tokens"] = Json::integer(c.total);
    if (c.kind == kDependent) {
      e.o["group"] = Json::integer(c.group);
      e.o["index_in_group"] = Json::integer(c.index);
    }
    Json segs = Json::array();
    for (int64_t s = 0; s < c.seg_cnt; ++s) {
      const Segment& sg = plan.segments[static_cast<size_t>(c.seg_off + s)];
      Json x = Json::object();
      x.o["sequence"] = Json::integer(sg.seq);
      x.o["start"] = Json::integer(sg.start);
      x.o["length"] = Json::integer(sg.len);
      segs.a.push_back(std::move(x));
    }
    e.o["segments"] = std::move(segs);
    chunks.a.push_back(std::move(e));
  }
  doc.o["chunks"] = std::move(chunks);
  Json groups = Json::object();
  for (const auto& [g, members] : plan.groups) groups.o[std::to_string(g)] = int_array(members);
  doc.o["groups"] = std::move(groups);
  return doc;
}

Json execution_plan_to_json(const Plan& plan) {
  Json doc = Json::object();
  doc.o["k"] = Json::integer(plan.k);
  doc.o["chunk_size"] = Json::integer(plan.chunk_size);
  Json events = Json::array();
  for (const Event& e : plan.events) {
    Json x = Json::object();
    x.o["kind"] = Json::string(e.kind == kFwdDiscard ? "forward_discard"
                               : e.kind == kFwdRetain ? "forward_retain"
                                                      : "backward");
    x.o["chunk"] = Json::integer(e.chunk);
    if (e.group >= 0) {
      x.o["group"] = Json::integer(e.group);
      x.o["index_in_group"] = Json::integer(e.index);
    }
    if (e.recompute) x.o["recompute"] = Json::boolean(true);
    x.o["save_kv"] = Json::boolean(e.save_kv);
    x.o["read_kv_prefix"] = Json::boolean(e.read_prefix);
    x.o["accumulate_kv_grad"] = Json::boolean(e.acc_grad);
    events.a.push_back(std::move(x));
  }
  doc.o["events"] = std::move(events);
  Json groups = Json::object();
  for (const auto& [g, members] : plan.groups) groups.o[std::to_string(g)] = int_array(members);
  doc.o["groups"] = std::move(groups);
  Json tokens = Json::object();
  for (const auto& [c, t] : plan.chunk_tokens) tokens.o[std::to_string(c)] = Json::integer(t);
  doc.o["chunk_tokens"] = std::move(tokens);
  return doc;
}

Plan chunk_plan_from_json(const Json& doc) {
  Plan plan;
  try {
    plan.chunk_size = doc.at("chunk_size").as_int();
    const Json& chunks = doc.at("chunks");
    if (chunks.kind != Json::kArray) throw ParseError("[json.exception.type_error.302] chunks must be an array");
    for (const Json& e : chunks.a) {
      Chunk c;
      c.id = e.at("id").as_int();
      const Json& kind = e.at("kind");
      if (kind.kind != Json::kString) throw ParseError("[json.exception.type_error.302] type must be string");
      c.kind = kind.s == "standalone" ? kStandalone : kDependent;
      c.total = e.at("total_tokens").as_int();
      if (c.kind == kDependent) {
        c.group = e.at("group").as_int();
        c.index = e.at("index_in_group").as_int();
      }
      c.seg_off = static_cast<int64_t>(plan.segments.size());
      const Json& segs = e.at("segments");
      if (segs.kind != Json::kArray) throw ParseError("[json.exception.type_error.302] segments must be an array");
      for (const Json& s : segs.a)
        plan.segments.push_back({s.at("sequence").as_int(), s.at("start").as_int(), s.at("length").as_int()});
      c.seg_cnt = static_cast<int64_t>(plan.segments.size()) - c.seg_off;
      plan.chunks.push_back(c);
    }
    if (doc.contains("groups"))
      for (const auto& [key, members] : doc.at("groups").o) {
        std::vector<int64_t> v;
        if (members.kind != Json::kArray) throw ParseError("[json.exception.type_error.302] group must be an array");
        for (const Json& m : members.a) v.push_back(m.as_int());
        plan.groups[std::stoll(key)] = v;
      }
  } catch (const ParseError& e) {
    throw ParseError(std::string("malformed chunk plan: ") + e.what());
  }
  for (size_t i = 0; i < plan.chunks.size(); ++i) {
    plan.index_of[plan.chunks[i].id] = static_cast<int64_t>(i);
    plan.chunk_tokens[plan.chunks[i].id] = plan.chunks[i].total;
  }
  return plan;
}

// ------------------------------------------------------------ trace export
std::string export_trace(const std::vector<std::vector<TraceOp>>& stages, bool chrome) {
  static const char* kName[3] = {"F", "F'", "B"};
  auto name = [](int64_t k) { return (k >= 0 && k < 3) ? kName[k] : "?"; };
  if (chrome) {
    Json events = Json::array();
    auto num = [](double v) { return v == std::floor(v) ? Json::integer(static_cast<int64_t>(v)) : Json::number(v); };
    for (size_t s = 0; s < stages.size(); ++s)
      for (const TraceOp& e : stages[s]) {
        Json x = Json::object();
        x.o["name"] = Json::string(std::string(name(e.kind)) + " chunk" + std::to_string(e.chunk));
        x.o["ph"] = Json::string("X");
        x.o["ts"] = num(e.start * 1000.0);
        x.o["dur"] = num((e.end - e.start) * 1000.0);
        x.o["pid"] = Json::integer(static_cast<int64_t>(s));
        x.o["tid"] = Json::integer(0);
        events.a.push_back(std::move(x));
      }
    Json doc = Json::object();
    doc.o["traceEvents"] = std::move(events);
    return doc.dump(2) + "\n";
  }
  std::string out;
  for (size_t s = 0; s < stages.size(); ++s) {
    out += "stage " + std::to_string(s);
    for (const TraceOp& e : stages[s]) {
      char cell[96];
      std::snprintf(cell, sizeof(cell), " | %-2s c%lld %.2f-%.2f", name(e.kind), static_cast<long long>(e.chunk),
                    e.start, e.end);
      out += cell;
    }
    out += "\n";
  }
  return out;
}

// ----------------------------------------------------------------- JSONL
std::vector<SeqRecord> load_lengths(const std::string& text) {
  std::vector<SeqRecord> set;
  std::istringstream in(text);
  std::string line;
  int64_t ln = 0;
  while (std::getline(in, line)) {
    ++ln;
    if (line.find_first_not_of(" \t\r\n") == std::string::npos) continue;
    const std::string where = "line " + std::to_string(ln) + ": ";
    Json rec;
    try {
      rec = Json::parse(line);
    } catch (const ParseError& e) {
      throw ParseError(where + "malformed record: " + e.what());
    }
    if (rec.kind != Json::kObject || !rec.contains("length") || rec.at("length").kind != Json::kInt)
      throw ParseError(where + "record must be an object with an integer `length`");
    SeqRecord r;
    r.id = static_cast<int64_t>(set.size());
    if (rec.contains("id")) {
      if (rec.at("id").kind != Json::kInt) throw ParseError(where + "`id` must be an integer");
      r.id = rec.at("id").i;
    }
    r.length = rec.at("length").i;
    if (r.length <= 0) throw ValidationError(where + "length must be positive");
    if (rec.contains("tokens")) {
      const Json& t = rec.at("tokens");
      if (t.kind != Json::kArray) throw ParseError(where + "`tokens` must be a list of integers");
      for (const Json& x : t.a) {
        if (x.kind != Json::kInt && x.kind != Json::kDouble)
          throw ParseError(where + "malformed record: [json.exception.type_error.302] type must be number");
        r.tokens.push_back(static_cast<int32_t>(x.as_int()));
      }
      if (static_cast<int64_t>(r.tokens.size()) != r.length)
        throw ValidationError(where + "tokens count does not match length");
    }
    set.push_back(std::move(r));
  }
  std::set<int64_t> ids;
  for (const SeqRecord& r : set)
    if (!ids.insert(r.id).second) throw ValidationError("duplicate sequence id " + std::to_string(r.id));
  return set;
}

std::string write_records(const std::vector<SeqRecord>& set) {
  std::string out;
  for (const SeqRecord& r : set) {
    Json rec = Json::object();
    rec.o["id"] = Json::integer(r.id);
    rec.o["length"] = Json::integer(r.length);
    if (!r.tokens.empty()) {
      Json t = Json::array();
      for (int32_t x : r.tokens) t.a.push_back(Json::integer(x));
      rec.o["tokens"] = std::move(t);
    }
    out += rec.dump() + "\n";
  }
  return out;
}

// ----------------------------------------------------------- memory model
double predict_peak(const MemCoeffs& c, int64_t chunk_size, int64_t k, int64_t context_len) {
  return c.base + c.per_chunk_token * static_cast<double>(k * chunk_size) +
         c.per_context_token * c.gqa_ratio * static_cast<double>(context_len);
}

// Least squares on [1, k*cs, gqa*ctx]: normal equations, Gauss-Jordan with
// partial pivoting (memory_model.hpp:59-131).
MemCoeffs calibrate(const std::vector<MemMeasurement>& ms, double gqa, double* max_residual) {
  if (ms.size() < 3) throw ValidationError("calibration needs at least 3 measurements");
  if (gqa <= 0) throw ValidationError("gqa_ratio must be positive");
  const size_t n = ms.size();
  std::vector<double> x1(n), x2(n), y(n);
  for (size_t i = 0; i < n; ++i) {
    x1[i] = static_cast<double>(ms[i].k * ms[i].chunk_size);
    x2[i] = gqa * static_cast<double>(ms[i].context_len);
    y[i] = ms[i].peak_gib;
  }
  auto spread = [n](const std::vector<double>& v) {
    double mean = 0.0;
    for (double x : v) mean += x;
    mean /= static_cast<double>(n);
    double var = 0.0;
    for (double x : v) var += (x - mean) * (x - mean);
    return var;
  };
  if (spread(x1) == 0.0) throw ValidationError("calibration design is rank-deficient: no variation in k * chunk_size");
  if (spread(x2) == 0.0) throw ValidationError("calibration design is rank-deficient: no variation in context length");
  std::array<std::array<double, 4>, 3> a{};
  for (size_t i = 0; i < n; ++i) {
    const double row[3] = {1.0, x1[i], x2[i]};
    for (int r = 0; r < 3; ++r) {
      for (int c = 0; c < 3; ++c) a[r][c] += row[r] * row[c];
      a[r][3] += row[r] * y[i];
    }
  }
  for (int col = 0; col < 3; ++col) {
    int piv = col;
    for (int r = col + 1; r < 3; ++r)
      if (std::fabs(a[r][col]) > std::fabs(a[piv][col])) piv = r;
    std::swap(a[col], a[piv]);
    if (std::fabs(a[col][col]) < 1e-12)
      throw ValidationError("calibration design is rank-deficient: collinear measurements");
    for (int r = 0; r < 3; ++r) {
      if (r == col) continue;
      const double f = a[r][col] / a[col][col];
      for (int c = col; c < 4; ++c) a[r][c] -= f * a[col][c];
    }
  }
  MemCoeffs out;
  out.base = a[0][3] / a[0][0];
  out.per_chunk_token = a[1][3] / a[1][1];
  out.per_context_token = a[2][3] / a[2][2];
  out.gqa_ratio = gqa;
  double worst = 0.0;
  for (size_t i = 0; i < n; ++i)
    worst = std::max(worst, std::fabs(predict_peak(out, ms[i].chunk_size, ms[i].k, ms[i].context_len) - y[i]));
  if (max_residual) *max_residual = worst;
  return out;
}

std::vector<MemMeasurement> parse_measurements(const std::string& csv) {
  std::vector<MemMeasurement> out;
  std::istringstream in(csv);
  std::string line;
  int64_t ln = 0;
  while (std::getline(in, line)) {
    ++ln;
    if (line.find_first_not_of(" \t\r\n") == std::string::npos) continue;
    if (ln == 1 && line.find("chunk_size") != std::string::npos) continue;
    long long cs = 0, k = 0, ctx = 0;
    double peak = 0.0;
    if (std::sscanf(line.c_str(), " %lld , %lld , %lld , %lf", &cs, &k, &ctx, &peak) != 4)
      throw ParseError("line " + std::to_string(ln) + ": expected chunk_size,k,context_len,peak_gib");
    out.push_back({cs, k, ctx, peak});
  }
  return out;
}

Json coefficients_to_json(const MemCoeffs& c) {
  Json j = Json::object();
  j.o["base_gib"] = Json::number(c.base);
  j.o["per_chunk_token_gib"] = Json::number(c.per_chunk_token);
  j.o["per_context_token_gib"] = Json::number(c.per_context_token);
  j.o["gqa_ratio"] = Json::number(c.gqa_ratio);
  return j;
}

}  // namespace cfb
