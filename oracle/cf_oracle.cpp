// oracle/cf_oracle.cpp — TEST INFRASTRUCTURE ONLY.
//
// CPU restatement of the reference ChunkFlow path, used exclusively as the
// checker by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg.
// It is never linked into, called by, or measured as the product
// (paper_2503_02356_b200/), whose path is CUDA-only.
//
// Pinning: every function below is validated against the reference itself
// (oracle/_ref/libcfref.so, compiled from the unmodified headers by
// oracle/Makefile) and against the reference tests' known answers
// (tests/test_oracle_pinning.py, tests/golden/).
//
// What is restated (file:line in /root/reference/proj/include/chunkflow/):
//   SplitMix64                     common.hpp:35-62
//   synthesize / bucket_low        dataset.hpp:183-237
//   split_long / pack_short / ffd / exact / construct_chunks
//                                  chunker.hpp:42-227
//   group_events / kv_actions_for / schedule_step / validate_plan / listing
//                                  scheduler.hpp:58-298
//   init_model                     toy_model.hpp:110-134
//   segment_forward / backward     toy_model.hpp:206-520
//   batch_normalizer / targets     toy_model.hpp:533-550, plan_runner.hpp:112-122
//   run_plan (StateStore semantics, instrumentation)
//                                  plan_runner.hpp:67-339
//   forward_full / backward_full   toy_model.hpp:556-596
// Extension (no reference exists): arch=llama adds RMSNorm, RoPE (rotate-
// half, global positions start+t) and SwiGLU to the same segment structure.
// For arch=toy the arithmetic is performed in the reference's per-element
// operation order, so results are bitwise identical to the reference; the
// loops are re-blocked (rows in parallel, per-element reduction order kept)
// so the oracle finishes the C1 batch in seconds instead of ~40 s.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <set>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <utility>
#include <vector>

#include "../include/chunkflow_b200.h"

namespace {

thread_local std::string g_err;

struct VErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};

template <class F>
int guarded(F&& f) {
  try {
    f();
    return CF_OK;
  } catch (const VErr& e) {
    g_err = e.what();
    return CF_EVALIDATION;
  } catch (const std::exception& e) {
    g_err = e.what();
    return CF_EINTERNAL;
  }
}


// Static-partition parallel loop on std::thread (no OpenMP in this image);
// nested calls run inline.  Each index is processed by exactly one thread, so
// per-element operation order is unchanged by parallelism.
thread_local bool t_in_par = false;
template <class F>
void par_for(int64_t a, int64_t b, F&& f) {
  const int64_t n = b - a;
  if (n <= 0) return;
  const int64_t hw = std::max<int64_t>(1, std::thread::hardware_concurrency());
  const int64_t nt = std::min<int64_t>(hw, n);
  if (nt == 1 || t_in_par) {
    for (int64_t i = a; i < b; ++i) f(i);
    return;
  }
  std::vector<std::thread> th;
  for (int64_t w = 0; w < nt; ++w) {
    th.emplace_back([&, w] {
      t_in_par = true;
      for (int64_t i = a + w; i < b; i += nt) f(i);
      t_in_par = false;
    });
  }
  for (auto& x : th) x.join();
}

// ---------------------------------------------------------------- SplitMix64
struct Mix {
  uint64_t s;
  uint64_t next() {
    s += 0x9E3779B97F4A7C15ULL;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }
  double unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  uint64_t below(uint64_t n) {
    const uint64_t thr = (0 - n) % n;
    while (true) {
      const uint64_t r = next();
      if (r >= thr) return r % n;
    }
  }
};

// ------------------------------------------------------------------ planning
struct Seg {
  int64_t seq, start, len;
};
struct Chk {
  int64_t id, kind, group = -1, index = -1, total = 0;
  std::vector<Seg> segs;
};
struct Plan {
  int64_t cs = 0;
  std::vector<Chk> chunks;
  std::map<int64_t, std::vector<int64_t>> groups;
};
struct Ev {
  int64_t kind, chunk, group, index;
  bool recompute, save_kv, read_prefix, acc_grad;
};
struct Sched {
  std::vector<Ev> events;
  int64_t k = 1, cs = 0;
  std::map<int64_t, std::vector<int64_t>> groups;
  std::map<int64_t, int64_t> tokens;
};
struct Diag {
  int64_t peak = 0, recompute = 0;
  std::vector<std::string> violations;
};

struct Item {
  int64_t len, id;
};

// FFD into exactly `bins` bins, lowest bin wins (chunker.hpp:77-96).
bool ffd(const std::vector<Item>& items, size_t bins, int64_t cap,
         std::vector<std::vector<int64_t>>& out) {
  std::vector<int64_t> room(bins, cap);
  std::vector<std::vector<int64_t>> b(bins);
  for (const Item& it : items) {
    size_t dst = bins;
    for (size_t i = 0; i < bins; ++i)
      if (room[i] >= it.len) {
        dst = i;
        break;
      }
    if (dst == bins) return false;
    room[dst] -= it.len;
    b[dst].push_back(it.id);
  }
  out.swap(b);
  return true;
}

// Exhaustive DFS with the reference's symmetry pruning (chunker.hpp:103-129):
// only the first empty bin is opened, bins with equal room tried once.
bool dfs(const std::vector<Item>& items, size_t at, size_t bins,
         std::vector<int64_t>& room, std::vector<std::vector<int64_t>>& b) {
  if (at == items.size()) return true;
  for (size_t i = 0; i < bins; ++i) {
    if (i > 0 && b[i].empty() && b[i - 1].empty()) break;
    if (room[i] < items[at].len) continue;
    bool seen = false;
    for (size_t j = 0; j < i && !seen; ++j) seen = room[j] == room[i];
    if (seen) continue;
    room[i] -= items[at].len;
    b[i].push_back(items[at].id);
    if (dfs(items, at + 1, bins, room, b)) return true;
    b[i].pop_back();
    room[i] += items[at].len;
  }
  return false;
}

std::vector<std::vector<int64_t>> pack(std::vector<Item> items, int64_t cs) {
  for (const Item& it : items)
    if (it.len > cs) throw VErr("pack_short requires lengths at most chunk_size");
  std::sort(items.begin(), items.end(), [](const Item& a, const Item& b) {
    return a.len != b.len ? a.len > b.len : a.id < b.id;
  });
  std::vector<std::vector<int64_t>> out;
  if (items.empty()) return out;
  for (size_t bins = 1; bins <= items.size(); ++bins) {
    if (ffd(items, bins, cs, out)) return out;
    if (items.size() <= 12) {
      std::vector<int64_t> room(bins, cs);
      std::vector<std::vector<int64_t>> b(bins);
      if (dfs(items, 0, bins, room, b)) return b;
    }
  }
  throw VErr("bin packing failed");
}

Plan build_chunks(const int64_t* ids, const int64_t* lens, int64_t n, int64_t cs) {
  if (cs < 1) throw VErr("chunk_size must be at least 1");
  Plan p;
  p.cs = cs;
  std::vector<Item> shorts;
  std::vector<std::pair<int64_t, int64_t>> longs;  // (id, len)
  std::map<int64_t, int64_t> len_of;
  for (int64_t i = 0; i < n; ++i) {
    len_of[ids[i]] = lens[i];
    if (lens[i] > cs)
      longs.push_back({ids[i], lens[i]});
    else
      shorts.push_back({lens[i], ids[i]});
  }
  std::sort(longs.begin(), longs.end());
  int64_t next = 0;
  for (std::vector<int64_t> bin : pack(shorts, cs)) {
    Chk c;
    c.id = next++;
    c.kind = CF_CHUNK_STANDALONE;
    std::sort(bin.begin(), bin.end());
    for (int64_t id : bin) {
      c.segs.push_back({id, 0, len_of.at(id)});
      c.total += len_of.at(id);
    }
    p.chunks.push_back(c);
  }
  int64_t g = 0;
  for (const auto& [id, len] : longs) {
    const int64_t pieces = (len + cs - 1) / cs;
    for (int64_t i = 0; i < pieces; ++i) {
      Chk c;
      c.id = next++;
      c.kind = CF_CHUNK_DEPENDENT;
      c.group = g;
      c.index = i;
      const int64_t st = i * cs;
      c.segs.push_back({id, st, std::min(cs, len - st)});
      c.total = c.segs[0].len;
      p.groups[g].push_back(c.id);
      p.chunks.push_back(c);
    }
    ++g;
  }
  return p;
}

// (kind, 1-based index, recompute) skeleton (scheduler.hpp:58-85).
std::vector<std::tuple<int64_t, int64_t, bool>> skeleton(int64_t n, int64_t k) {
  if (n < 1) throw VErr("group size must be at least 1");
  if (k < 1) throw VErr("retention budget k must be at least 1");
  std::vector<std::tuple<int64_t, int64_t, bool>> s;
  const int64_t kept = std::min(n, k);
  const int64_t dropped = n - kept;
  for (int64_t i = 1; i <= dropped; ++i) s.emplace_back(CF_EXEC_FORWARD_DISCARD, i, false);
  for (int64_t i = dropped + 1; i <= n; ++i) s.emplace_back(CF_EXEC_FORWARD_RETAIN, i, false);
  for (int64_t i = n; i > dropped; --i) s.emplace_back(CF_EXEC_BACKWARD, i, false);
  for (int64_t i = dropped; i >= 1; --i) {
    s.emplace_back(CF_EXEC_FORWARD_RETAIN, i, true);
    s.emplace_back(CF_EXEC_BACKWARD, i, false);
  }
  return s;
}

Ev group_event(int64_t kind, int64_t chunk, int64_t group, int64_t idx0,
               bool rec, int64_t n) {
  Ev e{kind, chunk, group, idx0, rec, false, false, false};
  if (kind != CF_EXEC_BACKWARD) {
    e.read_prefix = idx0 > 0;
    e.save_kv = !rec && idx0 + 1 < n;
  } else {
    e.acc_grad = idx0 > 0;
  }
  return e;
}

Sched schedule(const Plan& p, int64_t k) {
  if (k < 1) throw VErr("retention budget k must be at least 1");
  Sched s;
  s.k = k;
  s.cs = p.cs;
  s.groups = p.groups;
  for (const Chk& c : p.chunks) s.tokens[c.id] = c.total;
  std::set<int64_t> done;
  for (const Chk& c : p.chunks) {
    if (c.kind == CF_CHUNK_STANDALONE) {
      s.events.push_back({CF_EXEC_FORWARD_RETAIN, c.id, -1, -1, false, false, false, false});
      s.events.push_back({CF_EXEC_BACKWARD, c.id, -1, -1, false, false, false, false});
      continue;
    }
    if (!done.insert(c.group).second) continue;
    const std::vector<int64_t>& mem = p.groups.at(c.group);
    const int64_t n = static_cast<int64_t>(mem.size());
    for (const auto& [kind, idx, rec] : skeleton(n, k))
      s.events.push_back(group_event(kind, mem[idx - 1], c.group, idx - 1, rec, n));
  }
  return s;
}

Sched schedule_one_group(int64_t n, int64_t k, int64_t cs) {
  Sched s;
  s.k = k;
  s.cs = cs;
  for (int64_t i = 1; i <= n; ++i) {
    s.groups[0].push_back(i);
    s.tokens[i] = cs;
  }
  for (const auto& [kind, idx, rec] : skeleton(n, k))
    s.events.push_back(group_event(kind, idx, 0, idx - 1, rec, n));
  return s;
}

// Replay (scheduler.hpp:182-271); messages are the reference's text.
Diag replay(const Sched& s) {
  Diag d;
  std::map<int64_t, std::pair<int64_t, int64_t>> where;  // chunk -> (group, idx)
  for (const auto& [g, mem] : s.groups)
    for (size_t i = 0; i < mem.size(); ++i) where[mem[i]] = {g, static_cast<int64_t>(i)};
  auto tok = [&](int64_t c) {
    auto it = s.tokens.find(c);
    return it == s.tokens.end() ? s.cs : it->second;
  };
  std::map<int64_t, int64_t> fwd, bwd, first_hi, bwd_lo;
  std::set<int64_t> live;
  int64_t held = 0;
  for (const Ev& e : s.events) {
    const int64_t c = e.chunk;
    const bool grouped = where.count(c) > 0;
    const int64_t g = grouped ? where[c].first : -1;
    const int64_t idx = grouped ? where[c].second : -1;
    if (e.kind != CF_EXEC_BACKWARD) {
      const bool first = fwd[c]++ == 0;
      if (!first) d.recompute += tok(c);
      if (grouped && first) {
        const int64_t prev = first_hi.count(g) ? first_hi[g] : -1;
        if (idx != prev + 1)
          d.violations.push_back("first forward of chunk " + std::to_string(c) +
                                 " out of ascending group order");
        first_hi[g] = std::max(prev, idx);
      }
      if (e.kind == CF_EXEC_FORWARD_RETAIN && live.insert(c).second) {
        held += tok(c);
        d.peak = std::max(d.peak, held);
      }
    } else {
      if (!live.count(c)) {
        d.violations.push_back("backward of chunk " + std::to_string(c) +
                               " without a live retain-forward");
      } else {
        live.erase(c);
        held -= tok(c);
      }
      if (++bwd[c] > 1)
        d.violations.push_back("chunk " + std::to_string(c) + " backwarded more than once");
      if (grouped) {
        if (bwd_lo.count(g) && idx != bwd_lo[g] - 1)
          d.violations.push_back("backward of chunk " + std::to_string(c) +
                                 " out of descending group order");
        bwd_lo[g] = idx;
      }
    }
  }
  for (const auto& [c, cnt] : fwd) {
    (void)cnt;
    if (bwd[c] == 0) d.violations.push_back("chunk " + std::to_string(c) + " was never backwarded");
  }
  return d;
}

void put_events(const Sched& s, cf_event_rec* ev, int64_t cap, int64_t* n_ev,
                cf_plan_diag* diag) {
  const int64_t n = static_cast<int64_t>(s.events.size());
  if (n > cap) throw VErr("event buffer too small");
  for (int64_t i = 0; i < n; ++i) {
    const Ev& e = s.events[i];
    ev[i] = {e.kind, e.chunk, e.group, e.index, e.recompute, e.save_kv, e.read_prefix, e.acc_grad};
  }
  *n_ev = n;
  if (diag) {
    const Diag d = replay(s);
    *diag = {d.peak, d.recompute, static_cast<int64_t>(d.violations.size())};
  }
}

// -------------------------------------------------------------------- model
struct Cfg {
  int arch;
  int64_t V, d, H, KVH, L, ffn;
  uint64_t seed;
  double theta, eps;
  int64_t dh() const { return d / H; }
  int64_t kvw() const { return KVH * dh(); }
  int64_t per() const { return H / KVH; }
  bool llama() const { return arch == CF_ARCH_LLAMA; }
  int64_t per_layer() const { return llama() ? 9 : 6; }
};

Cfg to_cfg(const cf_model_cfg* c) {
  Cfg g{c->arch, c->vocab_size, c->d_model, c->num_heads, c->num_kv_heads,
        c->num_layers, c->ffn_width, c->seed, c->rope_theta, c->rms_eps};
  if (g.V < 1 || g.d < 1 || g.H < 1 || g.KVH < 1 || g.L < 1) throw VErr("bad model config");
  if (g.d % g.H || g.H % g.KVH) throw VErr("bad head configuration");
  if (!g.llama()) g.ffn = 2 * g.d;
  if (g.ffn < 1) throw VErr("ffn_width required");
  if (g.llama() && (g.dh() % 2)) throw VErr("RoPE needs an even head dim");
  return g;
}

struct Mat {
  int64_t r = 0, c = 0;
  std::vector<double> v;
  Mat() = default;
  Mat(int64_t rr, int64_t cc) : r(rr), c(cc), v(static_cast<size_t>(rr * cc), 0.0) {}
  double* row(int64_t i) { return v.data() + i * c; }
  const double* row(int64_t i) const { return v.data() + i * c; }
};

// Tensor list: toy = emb, L x {wq,wk,wv,wo,w1,w2}, head (toy_model.hpp:116-126)
// llama = emb, L x {attn_norm,wq,wk,wv,wo,ffn_norm,w_gate,w_up,w_down},
//         final_norm, head.  Norm gains are 1 and consume no draws.
std::vector<std::pair<int64_t, int64_t>> shapes(const Cfg& g) {
  std::vector<std::pair<int64_t, int64_t>> s;
  s.push_back({g.V, g.d});
  for (int64_t l = 0; l < g.L; ++l) {
    if (g.llama()) {
      s.push_back({1, g.d});
      s.push_back({g.d, g.d});
      s.push_back({g.d, g.kvw()});
      s.push_back({g.d, g.kvw()});
      s.push_back({g.d, g.d});
      s.push_back({1, g.d});
      s.push_back({g.d, g.ffn});
      s.push_back({g.d, g.ffn});
      s.push_back({g.ffn, g.d});
    } else {
      s.push_back({g.d, g.d});
      s.push_back({g.d, g.kvw()});
      s.push_back({g.d, g.kvw()});
      s.push_back({g.d, g.d});
      s.push_back({g.d, g.ffn});
      s.push_back({g.ffn, g.d});
    }
  }
  if (g.llama()) s.push_back({1, g.d});
  s.push_back({g.d, g.V});
  return s;
}

bool is_norm(const Cfg& g, size_t idx, size_t count) {
  if (!g.llama()) return false;
  if (idx == count - 2) return true;  // final norm
  if (idx == 0 || idx >= count - 2) return false;
  const size_t j = (idx - 1) % 9;
  return j == 0 || j == 5;
}

struct Model {
  Cfg g;
  std::vector<Mat> t;
  const Mat& emb() const { return t[0]; }
  const Mat& head() const { return t.back(); }
  const Mat& P(int64_t l, int j) const { return t[1 + g.per_layer() * l + j]; }
  // toy slots
  const Mat& wq(int64_t l) const { return P(l, g.llama() ? 1 : 0); }
  const Mat& wk(int64_t l) const { return P(l, g.llama() ? 2 : 1); }
  const Mat& wv(int64_t l) const { return P(l, g.llama() ? 3 : 2); }
  const Mat& wo(int64_t l) const { return P(l, g.llama() ? 4 : 3); }
  int slot_q() const { return g.llama() ? 1 : 0; }
};

Model make_model(const Cfg& g, const double* flat) {
  Model m;
  m.g = g;
  const auto sh = shapes(g);
  for (const auto& [r, c] : sh) m.t.emplace_back(r, c);
  if (flat) {
    int64_t off = 0;
    for (Mat& x : m.t) {
      std::memcpy(x.v.data(), flat + off, sizeof(double) * x.v.size());
      off += static_cast<int64_t>(x.v.size());
    }
    return m;
  }
  Mix rng{g.seed};
  const double scale = 1.0 / std::sqrt(static_cast<double>(g.d));
  for (size_t i = 0; i < m.t.size(); ++i) {
    if (is_norm(g, i, m.t.size())) {
      std::fill(m.t[i].v.begin(), m.t[i].v.end(), 1.0);
      continue;
    }
    for (double& x : m.t[i].v) x = (rng.unit() * 2.0 - 1.0) * scale;
  }
  return m;
}

inline double dotn(const double* a, const double* b, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

// Y[t] = X[t] W for rows t (column-by-column dot, same order as
// row_times_matrix, toy_model.hpp:173-181).
void rows_times(const double* X, int64_t rows, int64_t ldx, const Mat& W,
                double* Y, int64_t ldy) {
par_for(0, rows, [&](int64_t t) {
    const double* x = X + t * ldx;
    double* y = Y + t * ldy;
    for (int64_t c = 0; c < W.c; ++c) {
      double s = 0.0;
      for (int64_t r = 0; r < W.r; ++r) s += x[r] * W.v[static_cast<size_t>(r * W.c + c)];
      y[c] = s;
    }
  });
}

// DX[t][r] += dot(DY[t], W row r)  (add_row_matrix_t, toy_model.hpp:193-198)
void rows_times_wt(const double* DY, int64_t rows, int64_t ldy, const Mat& W,
                   double* DX, int64_t ldx) {
par_for(0, rows, [&](int64_t t) {
    for (int64_t r = 0; r < W.r; ++r) DX[t * ldx + r] += dotn(DY + t * ldy, W.row(r), W.c); });
}

// dW += sum_t X[t]^T DY[t], accumulated over t in ascending order per element
// (add_outer, toy_model.hpp:184-190, re-blocked over rows of dW).
void wgrad(const double* X, int64_t ldx, const double* DY, int64_t ldy,
           int64_t rows, Mat& dW, const std::vector<char>* mask = nullptr) {
par_for(0, dW.r, [&](int64_t r) {
    double* out = dW.row(r);
    for (int64_t t = 0; t < rows; ++t) {
      if (mask && !(*mask)[t]) continue;
      const double xr = X[t * ldx + r];
      const double* dy = DY + t * ldy;
      for (int64_t c = 0; c < dW.c; ++c) out[c] += xr * dy[c];
    }
  });
}

void rms_fwd(const double* x, const double* gain, int64_t d, double eps,
             double* y, double* rstd) {
  double ss = 0.0;
  for (int64_t c = 0; c < d; ++c) ss += x[c] * x[c];
  const double r = 1.0 / std::sqrt(ss / static_cast<double>(d) + eps);
  *rstd = r;
  for (int64_t c = 0; c < d; ++c) y[c] = x[c] * r * gain[c];
}

// dx += d(y)/dx^T dy; dgain accumulated by the caller.
void rms_bwd(const double* x, const double* gain, double rstd, int64_t d,
             const double* dy, double* dx) {
  double dot = 0.0;
  for (int64_t c = 0; c < d; ++c) dot += dy[c] * gain[c] * x[c];
  const double k = rstd * rstd * rstd * dot / static_cast<double>(d);
  for (int64_t c = 0; c < d; ++c) dx[c] += rstd * dy[c] * gain[c] - x[c] * k;
}

// rotate-half RoPE on `heads` heads of width dh at position pos; inverse
// applies R^T (for backward).
void rope(double* v, int64_t heads, int64_t dh, double pos, double theta, bool inverse) {
  const int64_t half = dh / 2;
  for (int64_t i = 0; i < half; ++i) {
    const double f = std::pow(theta, -2.0 * static_cast<double>(i) / static_cast<double>(dh));
    const double a = pos * f;
    const double cs = std::cos(a), sn = inverse ? -std::sin(a) : std::sin(a);
    for (int64_t h = 0; h < heads; ++h) {
      double* p = v + h * dh;
      const double x0 = p[i], x1 = p[i + half];
      p[i] = x0 * cs - x1 * sn;
      p[i + half] = x1 * cs + x0 * sn;
    }
  }
}

inline double sigm(double x) { return 1.0 / (1.0 + std::exp(-x)); }

struct LayerTape {
  std::vector<double> x_in, xn, rstd1, q, attn, x_mid, xn2, rstd2, h, gate, up;
  std::vector<std::vector<double>> probs;  // [t*H+h] rows prefix+t+1
};
struct Tape {
  int64_t len = 0, prefix = 0;
  std::vector<int32_t> tokens;
  std::vector<int64_t> targets;
  std::vector<LayerTape> layers;
  std::vector<double> x_final, xf, rstdf;
  std::vector<std::vector<double>> k, v;  // per layer, len x kvw (post-RoPE)
  double loss_sum = 0.0;
};

using KV = std::vector<std::vector<double>>;

// segment_forward (toy_model.hpp:206-334) + llama extension.
Tape seg_forward(const Model& m, const int32_t* tokens, int64_t len,
                 const int64_t* targets, const KV& pk, const KV& pv,
                 int64_t prefix, bool keep) {
  const Cfg& g = m.g;
  const int64_t d = g.d, dh = g.dh(), kvw = g.kvw(), H = g.H, per = g.per(), fw = g.ffn;
  const double inv = 1.0 / std::sqrt(static_cast<double>(dh));
  Tape tp;
  tp.len = len;
  tp.prefix = prefix;
  tp.tokens.assign(tokens, tokens + len);
  tp.targets.assign(targets, targets + len);
  tp.k.resize(g.L);
  tp.v.resize(g.L);
  if (keep) tp.layers.resize(g.L);

  std::vector<double> x(len * d);
  for (int64_t t = 0; t < len; ++t) {
    if (tokens[t] < 0 || tokens[t] >= g.V)
      throw VErr("token id " + std::to_string(tokens[t]) + " out of vocabulary range");
    std::memcpy(&x[t * d], m.emb().row(tokens[t]), sizeof(double) * d);
  }
  std::vector<double> xn(len * d), rs(len), q(len * d), attn(len * d), mid(len * d),
      xn2(len * d), rs2(len), h(len * fw), gt, up;
  if (g.llama()) {
    gt.resize(len * fw);
    up.resize(len * fw);
  }
  for (int64_t l = 0; l < g.L; ++l) {
    LayerTape* lt = keep ? &tp.layers[l] : nullptr;
    if (lt) {
      lt->x_in = x;
      lt->probs.resize(len * H);
    }
    const double* src = x.data();
    if (g.llama()) {
      const double* gain = m.P(l, 0).v.data();
      for (int64_t t = 0; t < len; ++t) rms_fwd(&x[t * d], gain, d, g.eps, &xn[t * d], &rs[t]);
      src = xn.data();
    }
    std::vector<double>& K = tp.k[l];
    std::vector<double>& Vv = tp.v[l];
    K.assign(len * kvw, 0.0);
    Vv.assign(len * kvw, 0.0);
    rows_times(src, len, d, m.wq(l), q.data(), d);
    rows_times(src, len, d, m.wk(l), K.data(), kvw);
    rows_times(src, len, d, m.wv(l), Vv.data(), kvw);
    if (g.llama()) {
      for (int64_t t = 0; t < len; ++t) {
        const double pos = static_cast<double>(prefix + t);
        rope(&q[t * d], H, dh, pos, g.theta, false);
        rope(&K[t * kvw], g.KVH, dh, pos, g.theta, false);
      }
    }
    const double* PK = prefix > 0 ? pk[l].data() : nullptr;
    const double* PV = prefix > 0 ? pv[l].data() : nullptr;
par_for(0, len, [&](int64_t t) {
      double* arow = &attn[t * d];
      std::fill(arow, arow + d, 0.0);
      std::vector<double> sc;
      for (int64_t hq = 0; hq < H; ++hq) {
        const int64_t kv = hq / per;
        const double* qh = &q[t * d + hq * dh];
        const int64_t rows = prefix + t + 1;
        sc.assign(rows, 0.0);
        for (int64_t j = 0; j < prefix; ++j) sc[j] = dotn(qh, PK + j * kvw + kv * dh, dh) * inv;
        for (int64_t j = 0; j <= t; ++j) sc[prefix + j] = dotn(qh, &K[j * kvw + kv * dh], dh) * inv;
        double mx = sc[0];
        for (int64_t j = 1; j < rows; ++j) mx = std::max(mx, sc[j]);
        double den = 0.0;
        for (int64_t j = 0; j < rows; ++j) {
          sc[j] = std::exp(sc[j] - mx);
          den += sc[j];
        }
        for (int64_t j = 0; j < rows; ++j) sc[j] /= den;
        double* oh = arow + hq * dh;
        for (int64_t j = 0; j < prefix; ++j) {
          const double* vj = PV + j * kvw + kv * dh;
          for (int64_t u = 0; u < dh; ++u) oh[u] += sc[j] * vj[u];
        }
        for (int64_t j = 0; j <= t; ++j) {
          const double* vj = &Vv[j * kvw + kv * dh];
          for (int64_t u = 0; u < dh; ++u) oh[u] += sc[prefix + j] * vj[u];
        }
        if (lt) lt->probs[t * H + hq] = sc;
      }
    });
    rows_times(attn.data(), len, d, m.wo(l), mid.data(), d);
    for (int64_t i = 0; i < len * d; ++i) mid[i] += x[i];
    if (g.llama()) {
      const double* gain2 = m.P(l, 5).v.data();
      for (int64_t t = 0; t < len; ++t) rms_fwd(&mid[t * d], gain2, d, g.eps, &xn2[t * d], &rs2[t]);
      rows_times(xn2.data(), len, d, m.P(l, 6), gt.data(), fw);
      rows_times(xn2.data(), len, d, m.P(l, 7), up.data(), fw);
      for (int64_t i = 0; i < len * fw; ++i) h[i] = gt[i] * sigm(gt[i]) * up[i];
      rows_times(h.data(), len, fw, m.P(l, 8), x.data(), d);
    } else {
      rows_times(mid.data(), len, d, m.P(l, 4), h.data(), fw);
      for (double& e : h) e = std::tanh(e);
      rows_times(h.data(), len, fw, m.P(l, 5), x.data(), d);
    }
    for (int64_t i = 0; i < len * d; ++i) x[i] += mid[i];
    if (lt) {
      lt->q = q;
      lt->attn = attn;
      lt->x_mid = mid;
      lt->h = h;
      if (g.llama()) {
        lt->xn = xn;
        lt->rstd1 = rs;
        lt->xn2 = xn2;
        lt->rstd2 = rs2;
        lt->gate = gt;
        lt->up = up;
      }
    }
  }
  std::vector<double> xf = x, rsf(len, 1.0);
  if (g.llama()) {
    const double* gf = m.t[m.t.size() - 2].v.data();
    for (int64_t t = 0; t < len; ++t) rms_fwd(&x[t * d], gf, d, g.eps, &xf[t * d], &rsf[t]);
  }
  std::vector<double> part(len, 0.0);
par_for(0, len, [&](int64_t t) {
    if (targets[t] < 0) return;
    std::vector<double> lg(g.V);
    rows_times(&xf[t * d], 1, d, m.head(), lg.data(), g.V);
    double mx = lg[0];
    for (int64_t c = 1; c < g.V; ++c) mx = std::max(mx, lg[c]);
    double den = 0.0;
    for (int64_t c = 0; c < g.V; ++c) den += std::exp(lg[c] - mx);
    part[t] = mx + std::log(den) - lg[targets[t]];
  });
  for (int64_t t = 0; t < len; ++t)
    if (targets[t] >= 0) tp.loss_sum += part[t];
  if (keep) {
    tp.x_final = x;
    tp.xf = xf;
    tp.rstdf = rsf;
  }
  return tp;
}

struct Grads {
  std::vector<Mat> t;
};

// segment_backward (toy_model.hpp:341-520) + llama extension.
void seg_backward(const Model& m, const Tape& tp, const KV& pk, const KV& pv,
                  KV* dpk, KV* dpv, const KV* in_dk, const KV* in_dv,
                  double norm, Grads& G) {
  const Cfg& g = m.g;
  const int64_t d = g.d, dh = g.dh(), kvw = g.kvw(), H = g.H, per = g.per(), fw = g.ffn;
  const int64_t len = tp.len, prefix = tp.prefix, V = g.V;
  const double inv = 1.0 / std::sqrt(static_cast<double>(dh));
  if (tp.layers.empty()) throw VErr("segment backward requires a retained tape");
  const int pl = static_cast<int>(g.per_layer());
  auto gidx = [&](int64_t l, int j) { return 1 + pl * l + j; };

  // Output head + CE.
  std::vector<double> dl(len * V, 0.0), dx(len * d, 0.0);
  std::vector<char> has(len, 0);
par_for(0, len, [&](int64_t t) {
    const int64_t tgt = tp.targets[t];
    if (tgt < 0) return;
    has[t] = 1;
    std::vector<double> lg(V);
    rows_times(&tp.xf[t * d], 1, d, m.head(), lg.data(), V);
    double mx = lg[0];
    for (int64_t c = 1; c < V; ++c) mx = std::max(mx, lg[c]);
    double den = 0.0;
    for (int64_t c = 0; c < V; ++c) den += std::exp(lg[c] - mx);
    for (int64_t c = 0; c < V; ++c)
      dl[t * V + c] = (std::exp(lg[c] - mx) / den - (c == tgt ? 1.0 : 0.0)) / norm;
  });
  wgrad(tp.xf.data(), d, dl.data(), V, len, G.t.back(), &has);
  {
    std::vector<double> dxf(len * d, 0.0);
par_for(0, len, [&](int64_t t) {
      if (has[t]) rows_times_wt(&dl[t * V], 1, V, m.head(), &dxf[t * d], d); });
    if (g.llama()) {
      const double* gf = m.t[m.t.size() - 2].v.data();
      Mat& dgf = G.t[G.t.size() - 2];
      for (int64_t t = 0; t < len; ++t) {
        rms_bwd(&tp.x_final[t * d], gf, tp.rstdf[t], d, &dxf[t * d], &dx[t * d]);
        for (int64_t c = 0; c < d; ++c) dgf.v[c] += dxf[t * d + c] * tp.x_final[t * d + c] * tp.rstdf[t];
      }
    } else {
      dx.swap(dxf);
    }
  }

  std::vector<double> dmid(len * d), dattn(len * d), dq(len * d), dko(len * kvw), dvo(len * kvw);
  for (int64_t l = g.L - 1; l >= 0; --l) {
    const LayerTape& lt = tp.layers[l];
    const std::vector<double>& K = tp.k[l];
    const std::vector<double>& Vv = tp.v[l];
    const double* PK = prefix > 0 ? pk[l].data() : nullptr;
    const double* PV = prefix > 0 ? pv[l].data() : nullptr;
    double* DPK = (prefix > 0 && dpk) ? (*dpk)[l].data() : nullptr;
    double* DPV = (prefix > 0 && dpv) ? (*dpv)[l].data() : nullptr;

    // FFN.
    if (g.llama()) {
      const Mat& Wg = m.P(l, 6);
      const Mat& Wu = m.P(l, 7);
      const Mat& Wd = m.P(l, 8);
      std::vector<double> dh_(len * fw, 0.0), dg(len * fw), du(len * fw), dxn2(len * d, 0.0);
par_for(0, len, [&](int64_t t) {
        for (int64_t j = 0; j < fw; ++j) dh_[t * fw + j] = dotn(&dx[t * d], Wd.row(j), d); });
      wgrad(lt.h.data(), fw, dx.data(), d, len, G.t[gidx(l, 8)]);
      for (int64_t i = 0; i < len * fw; ++i) {
        const double s = sigm(lt.gate[i]);
        const double si = lt.gate[i] * s;
        du[i] = dh_[i] * si;
        dg[i] = dh_[i] * lt.up[i] * s * (1.0 + lt.gate[i] * (1.0 - s));
      }
      rows_times_wt(dg.data(), len, fw, Wg, dxn2.data(), d);
      rows_times_wt(du.data(), len, fw, Wu, dxn2.data(), d);
      wgrad(lt.xn2.data(), d, dg.data(), fw, len, G.t[gidx(l, 6)]);
      wgrad(lt.xn2.data(), d, du.data(), fw, len, G.t[gidx(l, 7)]);
      const double* g2 = m.P(l, 5).v.data();
      Mat& dg2 = G.t[gidx(l, 5)];
      dmid = dx;
      for (int64_t t = 0; t < len; ++t) {
        rms_bwd(&lt.x_mid[t * d], g2, lt.rstd2[t], d, &dxn2[t * d], &dmid[t * d]);
        for (int64_t c = 0; c < d; ++c) dg2.v[c] += dxn2[t * d + c] * lt.x_mid[t * d + c] * lt.rstd2[t];
      }
    } else {
      const Mat& W1 = m.P(l, 4);
      const Mat& W2 = m.P(l, 5);
      std::vector<double> da(len * fw);
par_for(0, len, [&](int64_t t) {
        for (int64_t j = 0; j < fw; ++j) {
          const double hj = lt.h[t * fw + j];
          da[t * fw + j] = dotn(&dx[t * d], W2.row(j), d) * (1.0 - hj * hj);
        }
        for (int64_t c = 0; c < d; ++c) dmid[t * d + c] = dx[t * d + c];
      });
      wgrad(lt.h.data(), fw, dx.data(), d, len, G.t[gidx(l, 5)]);
      rows_times_wt(da.data(), len, fw, W1, dmid.data(), d);
      wgrad(lt.x_mid.data(), d, da.data(), fw, len, G.t[gidx(l, 4)]);
    }

    // Wo.
    std::fill(dattn.begin(), dattn.end(), 0.0);
    rows_times_wt(dmid.data(), len, d, m.wo(l), dattn.data(), d);
    wgrad(lt.attn.data(), d, dmid.data(), d, len, G.t[gidx(l, g.llama() ? 4 : 3)]);

    // Attention backward: per (t, hq) dS rows, then key-side accumulation in
    // the reference's (t asc, hq asc) order per element.
    std::vector<std::vector<double>> DS(len * H);
par_for(0, len, [&](int64_t t) {
      for (int64_t hq = 0; hq < H; ++hq) {
        const int64_t kv = hq / per;
        const std::vector<double>& p = lt.probs[t * H + hq];
        const int64_t rows = prefix + t + 1;
        const double* dout = &dattn[t * d + hq * dh];
        std::vector<double> dp(rows);
        for (int64_t j = 0; j < prefix; ++j) dp[j] = dotn(dout, PV + j * kvw + kv * dh, dh);
        for (int64_t j = 0; j <= t; ++j) dp[prefix + j] = dotn(dout, &Vv[j * kvw + kv * dh], dh);
        double pdp = 0.0;
        for (int64_t j = 0; j < rows; ++j) pdp += p[j] * dp[j];
        std::vector<double>& ds = DS[t * H + hq];
        ds.assign(rows, 0.0);
        for (int64_t j = 0; j < rows; ++j) ds[j] = p[j] * (dp[j] - pdp) * inv;
        double* dqh = &dq[t * d + hq * dh];
        std::fill(dqh, dqh + dh, 0.0);
        for (int64_t j = 0; j < prefix; ++j) {
          const double* kj = PK + j * kvw + kv * dh;
          for (int64_t u = 0; u < dh; ++u) dqh[u] += ds[j] * kj[u];
        }
        for (int64_t j = 0; j <= t; ++j) {
          const double* kj = &K[j * kvw + kv * dh];
          for (int64_t u = 0; u < dh; ++u) dqh[u] += ds[prefix + j] * kj[u];
        }
      }
    });
    std::fill(dko.begin(), dko.end(), 0.0);
    std::fill(dvo.begin(), dvo.end(), 0.0);
    // key rows: prefix rows j in [0,prefix), own rows j in [0,len)
    const int64_t nkeys = prefix + len;
par_for(0, nkeys, [&](int64_t key) {
      const bool own = key >= prefix;
      const int64_t j = own ? key - prefix : key;
      double* dvrow = own ? &dvo[j * kvw] : (DPV ? DPV + j * kvw : nullptr);
      double* dkrow = own ? &dko[j * kvw] : (DPK ? DPK + j * kvw : nullptr);
      const int64_t t0 = own ? j : 0;
      for (int64_t t = t0; t < len; ++t) {
        for (int64_t hq = 0; hq < H; ++hq) {
          const int64_t kv = hq / per;
          const std::vector<double>& p = lt.probs[t * H + hq];
          const std::vector<double>& ds = DS[t * H + hq];
          const double* dout = &dattn[t * d + hq * dh];
          const double* qh = &lt.q[t * d + hq * dh];
          if (dvrow) {
            const double pj = p[key];
            for (int64_t u = 0; u < dh; ++u) dvrow[kv * dh + u] += pj * dout[u];
          }
          if (dkrow) {
            const double s = ds[key];
            for (int64_t u = 0; u < dh; ++u) dkrow[kv * dh + u] += s * qh[u];
          }
        }
      }
    });
    if (in_dk)
      for (size_t i = 0; i < dko.size(); ++i) dko[i] += (*in_dk)[l][i];
    if (in_dv)
      for (size_t i = 0; i < dvo.size(); ++i) dvo[i] += (*in_dv)[l][i];

    // Projections (+ RoPE backward for llama).
    const int sq = m.slot_q();
    if (g.llama()) {
      for (int64_t t = 0; t < len; ++t) {
        const double pos = static_cast<double>(prefix + t);
        rope(&dq[t * d], H, dh, pos, g.theta, true);
        rope(&dko[t * kvw], g.KVH, dh, pos, g.theta, true);
      }
      std::vector<double> dxn(len * d, 0.0);
      wgrad(lt.xn.data(), d, dq.data(), d, len, G.t[gidx(l, sq)]);
      rows_times_wt(dq.data(), len, d, m.wq(l), dxn.data(), d);
      wgrad(lt.xn.data(), d, dko.data(), kvw, len, G.t[gidx(l, sq + 1)]);
      rows_times_wt(dko.data(), len, kvw, m.wk(l), dxn.data(), d);
      wgrad(lt.xn.data(), d, dvo.data(), kvw, len, G.t[gidx(l, sq + 2)]);
      rows_times_wt(dvo.data(), len, kvw, m.wv(l), dxn.data(), d);
      const double* g1 = m.P(l, 0).v.data();
      Mat& dg1 = G.t[gidx(l, 0)];
      dx = dmid;
      for (int64_t t = 0; t < len; ++t) {
        rms_bwd(&lt.x_in[t * d], g1, lt.rstd1[t], d, &dxn[t * d], &dx[t * d]);
        for (int64_t c = 0; c < d; ++c) dg1.v[c] += dxn[t * d + c] * lt.x_in[t * d + c] * lt.rstd1[t];
      }
    } else {
      // Per row the reference interleaves q,k,v contributions into dx in
      // the order dq.Wq^T, dk.Wk^T, dv.Wv^T (toy_model.hpp:501-511).
      dx = dmid;
      wgrad(lt.x_in.data(), d, dq.data(), d, len, G.t[gidx(l, 0)]);
      wgrad(lt.x_in.data(), d, dko.data(), kvw, len, G.t[gidx(l, 1)]);
      wgrad(lt.x_in.data(), d, dvo.data(), kvw, len, G.t[gidx(l, 2)]);
par_for(0, len, [&](int64_t t) {
        rows_times_wt(&dq[t * d], 1, d, m.wq(l), &dx[t * d], d);
        rows_times_wt(&dko[t * kvw], 1, kvw, m.wk(l), &dx[t * d], d);
        rows_times_wt(&dvo[t * kvw], 1, kvw, m.wv(l), &dx[t * d], d);
      });
    }
  }
  Mat& dE = G.t[0];
  for (int64_t t = 0; t < len; ++t) {
    double* row = dE.row(tp.tokens[t]);
    for (int64_t c = 0; c < d; ++c) row[c] += dx[t * d + c];
  }
}

Grads zero_grads(const Model& m) {
  Grads G;
  for (const Mat& x : m.t) G.t.emplace_back(x.r, x.c);
  return G;
}

struct Seq {
  int64_t id, len;
  const int32_t* tok;
};

std::vector<Seq> make_seqs(const int64_t* ids, const int64_t* lens, const int32_t* tokens, int64_t n) {
  std::vector<Seq> s;
  int64_t off = 0;
  for (int64_t i = 0; i < n; ++i) {
    s.push_back({ids[i], lens[i], tokens + off});
    off += lens[i];
  }
  return s;
}

double normalizer(const std::vector<Seq>& seqs) {
  int64_t n = 0;
  for (const Seq& s : seqs) {
    if (s.len < 2) throw VErr("sequence " + std::to_string(s.id) + " must have length >= 2");
    n += s.len - 1;
  }
  if (n <= 0) throw VErr("batch has no prediction targets");
  return static_cast<double>(n);
}

std::vector<int64_t> targets(const Seq& s, int64_t start, int64_t len) {
  std::vector<int64_t> t(len, -1);
  for (int64_t i = 0; i < len; ++i)
    if (start + i + 1 < s.len) t[i] = s.tok[start + i + 1];
  return t;
}

void flatten(const Grads& G, double* out) {
  int64_t off = 0;
  for (const Mat& x : G.t) {
    std::memcpy(out + off, x.v.data(), sizeof(double) * x.v.size());
    off += static_cast<int64_t>(x.v.size());
  }
}

struct Instr {
  int64_t peak = 0, recomputes = 0, mismatches = 0, violations = 0;
};

// run_plan (plan_runner.hpp:67-339): per-(sequence, chunk index) K/V state
// with gradient accumulators, literal event interpretation.
double run_plan(const Model& m, const Plan& plan, const Sched& sched,
                const std::vector<Seq>& seqs, bool corrupt, double norm_override,
                Grads& G, Instr& ins) {
  const Cfg& g = m.g;
  const int64_t kvw = g.kvw();
  {
    const Diag dg = replay(sched);
    if (!dg.violations.empty()) throw VErr("execution plan is invalid: " + dg.violations.front());
  }
  std::map<int64_t, const Seq*> by_id;
  for (const Seq& s : seqs) by_id[s.id] = &s;
  std::map<int64_t, const Chk*> chunk_of;
  for (const Chk& c : plan.chunks) chunk_of[c.id] = &c;
  const double norm = norm_override > 0 ? norm_override : normalizer(seqs);

  auto seq_for = [&](const Seg& s) -> const Seq& {
    auto it = by_id.find(s.seq);
    if (it == by_id.end()) throw VErr("chunk references unknown sequence " + std::to_string(s.seq));
    if (s.start < 0 || s.len < 1 || s.start + s.len > it->second->len)
      throw VErr("chunk segment exceeds sequence " + std::to_string(s.seq));
    return *it->second;
  };
  struct Entry {
    int64_t start, len;
    KV k, v, dk, dv;
    int64_t contrib = 0;
  };
  std::map<std::pair<int64_t, int64_t>, Entry> store;
  auto prefix_of = [&](int64_t seq, int64_t idx, int64_t plen) {
    std::pair<KV, KV> out;
    out.first.assign(g.L, std::vector<double>(plen * kvw));
    out.second = out.first;
    int64_t filled = 0;
    for (int64_t i = 0; i < idx; ++i) {
      auto it = store.find({seq, i});
      if (it == store.end()) throw VErr("missing KV prefix entry");
      for (int64_t l = 0; l < g.L; ++l) {
        std::copy(it->second.k[l].begin(), it->second.k[l].end(), out.first[l].begin() + filled * kvw);
        std::copy(it->second.v[l].begin(), it->second.v[l].end(), out.second[l].begin() + filled * kvw);
      }
      filled += it->second.len;
    }
    if (filled != plen) throw VErr("KV prefix does not cover the segment start");
    return out;
  };
  struct Live {
    std::vector<Tape> tapes;
    double loss = 0.0;
  };
  std::map<int64_t, Live> live;
  std::map<int64_t, double> first;
  double total = 0.0;
  int64_t held = 0;
  const KV none;
  for (const Ev& e : sched.events) {
    auto cit = chunk_of.find(e.chunk);
    if (cit == chunk_of.end()) throw VErr("plan references unknown chunk");
    const Chk& c = *cit->second;
    if (e.kind != CF_EXEC_BACKWARD) {
      const bool keep = e.kind == CF_EXEC_FORWARD_RETAIN;
      Live lv;
      if (c.group >= 0) {
        const Seg& s = c.segs[0];
        const Seq& sq = seq_for(s);
        const auto tg = targets(sq, s.start, s.len);
        KV pk, pv;
        if (s.start > 0) {
          auto pr = prefix_of(s.seq, c.index, s.start);
          pk.swap(pr.first);
          pv.swap(pr.second);
        }
        Tape tp = seg_forward(m, sq.tok + s.start, s.len, tg.data(), pk, pv, s.start, keep);
        lv.loss = tp.loss_sum;
        const auto key = std::make_pair(s.seq, c.index);
        if (e.save_kv && !store.count(key)) {
          Entry en{s.start, s.len, tp.k, tp.v, {}, {}, 0};
          en.dk.assign(g.L, std::vector<double>(s.len * kvw, 0.0));
          en.dv = en.dk;
          store.emplace(key, std::move(en));
        }
        lv.tapes.push_back(std::move(tp));
      } else {
        for (const Seg& s : c.segs) {
          const Seq& sq = seq_for(s);
          const auto tg = targets(sq, s.start, s.len);
          Tape tp = seg_forward(m, sq.tok + s.start, s.len, tg.data(), none, none, 0, keep);
          lv.loss += tp.loss_sum;
          lv.tapes.push_back(std::move(tp));
        }
      }
      if (!e.recompute) {
        total += lv.loss;
        first[e.chunk] = lv.loss;
      } else {
        ++ins.recomputes;
        auto f = first.find(e.chunk);
        if (f == first.end() || f->second != lv.loss) ++ins.mismatches;
      }
      if (keep) {
        held += c.total;
        ins.peak = std::max(ins.peak, held);
        live[e.chunk] = std::move(lv);
      }
      continue;
    }
    auto lit = live.find(e.chunk);
    if (lit == live.end()) throw VErr("backward without retained activations");
    if (c.group >= 0) {
      const Seg& s = c.segs[0];
      seq_for(s);
      Tape& tp = lit->second.tapes[0];
      const int64_t n = static_cast<int64_t>(plan.groups.at(c.group).size());
      const auto key = std::make_pair(s.seq, c.index);
      KV idk, idv;
      bool inc = false;
      auto own = store.find(key);
      if (own != store.end()) {
        if (own->second.contrib != n - 1 - c.index) ++ins.violations;
        idk = own->second.dk;
        idv = own->second.dv;
        if (corrupt) {
          for (auto& r : idk)
            for (double& x : r) x *= 1.0000001;
          for (auto& r : idv)
            for (double& x : r) x *= 1.0000001;
        }
        inc = true;
      }
      KV pk, pv, dpk, dpv;
      if (tp.prefix > 0) {
        auto pr = prefix_of(s.seq, c.index, tp.prefix);
        pk.swap(pr.first);
        pv.swap(pr.second);
        dpk.assign(g.L, std::vector<double>(tp.prefix * kvw, 0.0));
        dpv = dpk;
      }
      seg_backward(m, tp, pk, pv, tp.prefix > 0 ? &dpk : nullptr, tp.prefix > 0 ? &dpv : nullptr,
                   inc ? &idk : nullptr, inc ? &idv : nullptr, norm, G);
      if (tp.prefix > 0) {
        int64_t off = 0;
        for (int64_t i = 0; i < c.index; ++i) {
          Entry& en = store.at({s.seq, i});
          for (int64_t l = 0; l < g.L; ++l)
            for (int64_t x = 0; x < en.len * kvw; ++x) {
              en.dk[l][x] += dpk[l][off * kvw + x];
              en.dv[l][x] += dpv[l][off * kvw + x];
            }
          ++en.contrib;
          off += en.len;
        }
      }
      if (own != store.end()) store.erase(own);
    } else {
      for (Tape& tp : lit->second.tapes) seg_backward(m, tp, none, none, nullptr, nullptr, nullptr, nullptr, norm, G);
    }
    held -= c.total;
    live.erase(lit);
  }
  return total / norm;
}

void check_seq(const Seq& s) {
  if (s.len < 2) throw VErr("sequence " + std::to_string(s.id) + " must have length >= 2");
}

}  // namespace

extern "C" {

const char* cfo_last_error(void) { return g_err.c_str(); }

int cfo_gen_tokens(const int64_t* lengths, int64_t n, int64_t vocab, uint64_t seed, int32_t* out) {
  return guarded([&] {
    Mix r{seed};
    int64_t o = 0;
    for (int64_t i = 0; i < n; ++i)
      for (int64_t t = 0; t < lengths[i]; ++t) out[o++] = static_cast<int32_t>(r.below(static_cast<uint64_t>(vocab)));
  });
}

// synthesize (dataset.hpp:207-237); preset 1 = eval_table5_spec (:88-97).
int cfo_synthesize(const int64_t* bounds, const double* fracs, int64_t nb,
                   int64_t max_length, int64_t preset, int64_t count,
                   uint64_t seed, int64_t* out) {
  return guarded([&] {
    std::vector<int64_t> ub;
    std::vector<double> cf;
    int64_t mx = max_length;
    if (preset == 1) {
      ub = {1024, 4096, 8192, 32768, 131072};
      cf = {0.9817, 0.9972, 0.9983, 0.9992, 0.9998};
      mx = 262144;
    } else {
      ub.assign(bounds, bounds + nb);
      cf.assign(fracs, fracs + nb);
    }
    if (count < 1) throw VErr("count must be at least 1");
    Mix r{seed};
    for (int64_t i = 0; i < count; ++i) {
      const double u = r.unit();
      int64_t lo = ub.back(), hi = mx + 1;
      for (size_t b = 0; b < ub.size(); ++b) {
        if (u < cf[b]) {
          lo = b == 0 ? std::max<int64_t>(1, std::min<int64_t>(16, ub[0] - 1)) : ub[b - 1];
          hi = ub[b];
          break;
        }
      }
      const double a = std::log(static_cast<double>(lo)), z = std::log(static_cast<double>(hi));
      const double x = std::exp(a + r.unit() * (z - a));
      out[i] = std::clamp<int64_t>(static_cast<int64_t>(std::floor(x)), lo, hi - 1);
    }
  });
}

int cfo_construct_chunks(const int64_t* ids, const int64_t* lengths, int64_t n,
                         int64_t cs, cf_chunk_rec* chunks, int64_t cap_c,
                         cf_segment_rec* segs, int64_t cap_s, int64_t* n_chunks,
                         int64_t* n_segs) {
  return guarded([&] {
    const Plan p = build_chunks(ids, lengths, n, cs);
    if (static_cast<int64_t>(p.chunks.size()) > cap_c) throw VErr("chunk buffer too small");
    int64_t si = 0;
    for (size_t i = 0; i < p.chunks.size(); ++i) {
      const Chk& c = p.chunks[i];
      chunks[i] = {c.id, c.kind, c.group, c.index, c.total, si, static_cast<int64_t>(c.segs.size())};
      for (const Seg& s : c.segs) {
        if (si >= cap_s) throw VErr("segment buffer too small");
        segs[si++] = {s.seq, s.start, s.len};
      }
    }
    *n_chunks = static_cast<int64_t>(p.chunks.size());
    *n_segs = si;
  });
}

int cfo_schedule_step(const int64_t* ids, const int64_t* lengths, int64_t n,
                      int64_t cs, int64_t k, cf_event_rec* ev, int64_t cap,
                      int64_t* n_events, cf_plan_diag* diag) {
  return guarded([&] { put_events(schedule(build_chunks(ids, lengths, n, cs), k), ev, cap, n_events, diag); });
}

int cfo_schedule_group(int64_t n, int64_t k, int64_t cs, cf_event_rec* ev,
                       int64_t cap, int64_t* n_events, cf_plan_diag* diag) {
  return guarded([&] { put_events(schedule_one_group(n, k, cs), ev, cap, n_events, diag); });
}

int cfo_listing(const int64_t* ids, const int64_t* lengths, int64_t n,
                int64_t cs, int64_t k, char* buf, int64_t cap) {
  return guarded([&] {
    const Sched s = schedule(build_chunks(ids, lengths, n, cs), k);
    std::string out;
    for (const Ev& e : s.events) {
      out += e.kind == CF_EXEC_FORWARD_DISCARD ? "F-" : e.kind == CF_EXEC_FORWARD_RETAIN ? "F+" : "B ";
      out += " chunk=" + std::to_string(e.chunk) + " group=";
      out += e.group < 0 ? "-" : std::to_string(e.group);
      if (e.recompute) out += " recompute";
      out += "\n";
    }
    if (static_cast<int64_t>(out.size()) + 1 > cap) throw VErr("listing buffer too small");
    std::memcpy(buf, out.c_str(), out.size() + 1);
  });
}

int64_t cfo_num_tensors(const cf_model_cfg* c) {
  try {
    return static_cast<int64_t>(shapes(to_cfg(c)).size());
  } catch (...) {
    return -1;
  }
}

int cfo_tensor_shape(const cf_model_cfg* c, int64_t idx, int64_t* rows, int64_t* cols) {
  return guarded([&] {
    const auto s = shapes(to_cfg(c));
    if (idx < 0 || idx >= static_cast<int64_t>(s.size())) throw VErr("tensor index");
    *rows = s[idx].first;
    *cols = s[idx].second;
  });
}

int64_t cfo_num_params(const cf_model_cfg* c) {
  int64_t n = 0;
  for (const auto& [r, cc] : shapes(to_cfg(c))) n += r * cc;
  return n;
}

int cfo_init(const cf_model_cfg* c, double* out) {
  return guarded([&] {
    const Model m = make_model(to_cfg(c), nullptr);
    int64_t off = 0;
    for (const Mat& x : m.t) {
      std::memcpy(out + off, x.v.data(), sizeof(double) * x.v.size());
      off += static_cast<int64_t>(x.v.size());
    }
  });
}

// params: flat tensor-order values (nullptr => init_model). instr as cfr.
int cfo_run_plan(const cf_model_cfg* c, const double* params, const int64_t* ids,
                 const int64_t* lengths, const int32_t* tokens, int64_t n,
                 int64_t cs, int64_t k, int corrupt, double norm_override,
                 double* loss, double* grads, int64_t* instr) {
  return guarded([&] {
    const Model m = make_model(to_cfg(c), params);
    const auto seqs = make_seqs(ids, lengths, tokens, n);
    const Plan p = build_chunks(ids, lengths, n, cs);
    const Sched s = schedule(p, k);
    Grads G = zero_grads(m);
    Instr ins;
    *loss = run_plan(m, p, s, seqs, corrupt != 0, norm_override, G, ins);
    if (grads) flatten(G, grads);
    if (instr) {
      instr[0] = ins.peak;
      instr[1] = ins.recomputes;
      instr[2] = ins.mismatches;
      instr[3] = ins.violations;
    }
  });
}

// backward_full (toy_model.hpp:575-596).
int cfo_backward_full(const cf_model_cfg* c, const double* params, const int64_t* ids,
                      const int64_t* lengths, const int32_t* tokens, int64_t n,
                      double norm_override, double* loss, double* grads) {
  return guarded([&] {
    const Model m = make_model(to_cfg(c), params);
    const auto seqs = make_seqs(ids, lengths, tokens, n);
    const double norm = norm_override > 0 ? norm_override : normalizer(seqs);
    Grads G = zero_grads(m);
    double total = 0.0;
    const KV none;
    for (const Seq& s : seqs) {
      check_seq(s);
      const auto tg = targets(s, 0, s.len);
      Tape tp = seg_forward(m, s.tok, s.len, tg.data(), none, none, 0, true);
      total += tp.loss_sum;
      seg_backward(m, tp, none, none, nullptr, nullptr, nullptr, nullptr, norm, G);
    }
    *loss = total / norm;
    if (grads) flatten(G, grads);
  });
}

// forward_full (toy_model.hpp:556-572).
int cfo_forward_full(const cf_model_cfg* c, const double* params, const int64_t* ids,
                     const int64_t* lengths, const int32_t* tokens, int64_t n,
                     double norm_override, double* loss) {
  return guarded([&] {
    const Model m = make_model(to_cfg(c), params);
    const auto seqs = make_seqs(ids, lengths, tokens, n);
    const double norm = norm_override > 0 ? norm_override : normalizer(seqs);
    double total = 0.0;
    const KV none;
    for (const Seq& s : seqs) {
      check_seq(s);
      const auto tg = targets(s, 0, s.len);
      total += seg_forward(m, s.tok, s.len, tg.data(), none, none, 0, false).loss_sum;
    }
    *loss = total / norm;
  });
}

}  // extern "C"
