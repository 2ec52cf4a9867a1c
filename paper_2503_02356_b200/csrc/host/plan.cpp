// Host planning: see plan.hpp.  Written for large batches (C4: 8,000
// sequences): first-fit over bins is a max-segment-tree descent (O(log B)
// per item instead of the reference's linear scan), and the bin-count
// search starts at the volume lower bound ceil(sum/cs) — FFD and the exact
// search are both infeasible below it, so the first feasible count and its
// packing are unchanged (pinned against the reference in tests/).
#include "plan.hpp"

#include <algorithm>
#include <cmath>
#include <set>
#include <tuple>

namespace cfb {

uint64_t splitmix_next(uint64_t& s) {
  s += 0x9E3779B97F4A7C15ULL;
  uint64_t z = s;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

namespace {
double next_unit(uint64_t& s) { return static_cast<double>(splitmix_next(s) >> 11) * 0x1.0p-53; }
uint64_t next_below(uint64_t& s, uint64_t n) {
  const uint64_t thr = (0 - n) % n;
  while (true) {
    const uint64_t r = splitmix_next(s);
    if (r >= thr) return r % n;
  }
}
}  // namespace

std::vector<int64_t> synthesize(const std::vector<int64_t>& bounds, const std::vector<double>& fracs,
                                int64_t max_length, int64_t count, uint64_t seed) {
  if (bounds.empty() || bounds.size() != fracs.size()) throw ValidationError("distribution spec has no buckets");
  for (size_t i = 0; i < bounds.size(); ++i) {
    if (bounds[i] < 2) throw ValidationError("bucket upper bound must be at least 2");
    if (i > 0 && bounds[i] <= bounds[i - 1]) throw ValidationError("bucket upper bounds must be strictly increasing");
    if (fracs[i] <= 0.0 || fracs[i] > 1.0) throw ValidationError("cumulative fractions must lie in (0, 1]");
    if (i > 0 && fracs[i] <= fracs[i - 1]) throw ValidationError("cumulative fractions must be strictly increasing");
  }
  if (max_length < bounds.back()) throw ValidationError("max_length must be at least the last bucket bound");
  // DistributionSpec::validate (dataset.hpp:62-71): the tail must be reachable
  // exactly when max_length leaves room for it
  if (max_length > bounds.back() && fracs.back() >= 1.0)
    throw ValidationError("last cumulative fraction must be below 1.0 when max_length exceeds the last bucket bound");
  if (max_length == bounds.back() && fracs.back() != 1.0)
    throw ValidationError("last cumulative fraction must equal 1.0 when max_length equals the last bucket bound");
  if (count < 1) throw ValidationError("count must be at least 1");
  uint64_t s = seed;
  std::vector<int64_t> out;
  out.reserve(static_cast<size_t>(count));
  for (int64_t i = 0; i < count; ++i) {
    const double u = next_unit(s);
    int64_t lo = bounds.back(), hi = max_length + 1;
    for (size_t b = 0; b < bounds.size(); ++b) {
      if (u < fracs[b]) {
        lo = b == 0 ? std::max<int64_t>(1, std::min<int64_t>(16, bounds[0] - 1)) : bounds[b - 1];
        hi = bounds[b];
        break;
      }
    }
    const double a = std::log(static_cast<double>(lo)), z = std::log(static_cast<double>(hi));
    const double x = std::exp(a + next_unit(s) * (z - a));
    out.push_back(std::clamp<int64_t>(static_cast<int64_t>(std::floor(x)), lo, hi - 1));
  }
  return out;
}

std::vector<int64_t> sample_batch(int64_t n, int64_t global_batch, int64_t step, uint64_t seed) {
  if (n < 1) throw ValidationError("cannot sample from an empty sequence set");
  if (global_batch < 1) throw ValidationError("global batch size must be at least 1");
  if (step < 0) throw ValidationError("step must be non-negative");
  const int64_t begin = step * global_batch;
  if (begin >= n) return {};
  std::vector<int64_t> order(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) order[static_cast<size_t>(i)] = i;
  uint64_t s = seed;
  for (int64_t i = n; i > 1; --i) std::swap(order[static_cast<size_t>(i - 1)], order[next_below(s, static_cast<uint64_t>(i))]);
  const int64_t end = std::min(begin + global_batch, n);
  return std::vector<int64_t>(order.begin() + begin, order.begin() + end);
}

const Chunk& Plan::chunk(int64_t id) const {
  auto it = index_of.find(id);
  if (it == index_of.end()) throw ValidationError("plan references unknown chunk " + std::to_string(id));
  return chunks[it->second];
}

namespace {

struct Item {
  int64_t len, id;
};

// Max segment tree over bin room; first_fit returns the lowest bin whose
// room >= need (the reference's "lowest bin wins", chunker.hpp:84-90).
class RoomTree {
 public:
  RoomTree(size_t n, int64_t cap) : n_(1) {
    while (n_ < n) n_ <<= 1;
    t_.assign(2 * n_, -1);
    for (size_t i = 0; i < n; ++i) t_[n_ + i] = cap;
    for (size_t i = n_ - 1; i >= 1; --i) t_[i] = std::max(t_[2 * i], t_[2 * i + 1]);
  }
  int64_t first_fit(int64_t need) const {
    if (t_[1] < need) return -1;
    size_t i = 1;
    while (i < n_) i = t_[2 * i] >= need ? 2 * i : 2 * i + 1;
    return static_cast<int64_t>(i - n_);
  }
  void take(size_t bin, int64_t amount) {
    size_t i = n_ + bin;
    t_[i] -= amount;
    for (i >>= 1; i >= 1; i >>= 1) t_[i] = std::max(t_[2 * i], t_[2 * i + 1]);
  }

 private:
  size_t n_;
  std::vector<int64_t> t_;
};

bool ffd_fixed(const std::vector<Item>& items, size_t bins, int64_t cap,
               std::vector<std::vector<int64_t>>& out) {
  RoomTree tree(bins, cap);
  std::vector<std::vector<int64_t>> b(bins);
  for (const Item& it : items) {
    const int64_t dst = tree.first_fit(it.len);
    if (dst < 0) return false;
    tree.take(static_cast<size_t>(dst), it.len);
    b[static_cast<size_t>(dst)].push_back(it.id);
  }
  out.swap(b);
  return true;
}

// Exhaustive search for <= 12 items (chunker.hpp:103-129): same visiting
// order and symmetry pruning, so the same packing is found first.
bool exhaustive(const std::vector<Item>& items, size_t at, size_t bins,
                std::vector<int64_t>& room, std::vector<std::vector<int64_t>>& b) {
  if (at == items.size()) return true;
  for (size_t i = 0; i < bins; ++i) {
    if (i > 0 && b[i].empty() && b[i - 1].empty()) break;
    if (room[i] < items[at].len) continue;
    bool dup = false;
    for (size_t j = 0; j < i; ++j)
      if (room[j] == room[i]) {
        dup = true;
        break;
      }
    if (dup) continue;
    room[i] -= items[at].len;
    b[i].push_back(items[at].id);
    if (exhaustive(items, at + 1, bins, room, b)) return true;
    b[i].pop_back();
    room[i] += items[at].len;
  }
  return false;
}

std::vector<std::vector<int64_t>> pack_short(std::vector<Item> items, int64_t cs) {
  std::vector<std::vector<int64_t>> bins;
  if (items.empty()) return bins;
  int64_t volume = 0;
  for (const Item& it : items) {
    if (it.len > cs) throw ValidationError("pack_short requires lengths at most chunk_size");
    volume += it.len;
  }
  std::sort(items.begin(), items.end(), [](const Item& a, const Item& b) {
    return a.len != b.len ? a.len > b.len : a.id < b.id;
  });
  const size_t lower = static_cast<size_t>(std::max<int64_t>(1, (volume + cs - 1) / cs));
  for (size_t count = lower; count <= items.size(); ++count) {
    if (ffd_fixed(items, count, cs, bins)) return bins;
    if (items.size() <= 12) {
      std::vector<int64_t> room(count, cs);
      std::vector<std::vector<int64_t>> b(count);
      if (exhaustive(items, 0, count, room, b)) return b;
    }
  }
  throw ValidationError("bin packing failed");
}

using Skel = std::tuple<int64_t, int64_t, bool>;  // kind, 1-based index, recompute

// Group skeleton under budget k (scheduler.hpp:58-85): the LAST k chunks
// are retained; the first n-k are forwarded twice, recomputed descending.
std::vector<Skel> skeleton(int64_t n, int64_t k) {
  if (n < 1) throw ValidationError("group size must be at least 1");
  if (k < 1) throw ValidationError("retention budget k must be at least 1");
  const int64_t drop = n > k ? n - k : 0;
  std::vector<Skel> s;
  s.reserve(static_cast<size_t>(2 * n + drop));
  for (int64_t i = 1; i <= n; ++i) s.emplace_back(i <= drop ? kFwdDiscard : kFwdRetain, i, false);
  for (int64_t i = n; i > drop; --i) s.emplace_back(kBackward, i, false);
  for (int64_t i = drop; i >= 1; --i) {
    s.emplace_back(kFwdRetain, i, true);
    s.emplace_back(kBackward, i, false);
  }
  return s;
}

Event make_event(int64_t kind, int64_t chunk, int64_t group, int64_t idx,
                 bool rec, int64_t n) {
  Event e{kind, chunk, group, idx, rec, false, false, false};
  // kv_actions_for (scheduler.hpp:87-100)
  if (kind == kBackward) {
    e.acc_grad = idx > 0;
  } else {
    e.read_prefix = idx > 0;
    e.save_kv = !rec && idx + 1 < n;
  }
  return e;
}

}  // namespace

Plan construct_chunks(const int64_t* ids, const int64_t* lengths, int64_t n,
                      int64_t cs) {
  if (cs < 1) throw ValidationError("chunk_size must be at least 1");
  Plan plan;
  plan.chunk_size = cs;
  std::vector<Item> shorts;
  std::vector<std::pair<int64_t, int64_t>> longs;
  std::map<int64_t, int64_t> len_of;
  shorts.reserve(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    len_of[ids[i]] = lengths[i];
    if (lengths[i] > cs) {
      longs.emplace_back(ids[i], lengths[i]);
    } else {
      shorts.push_back({lengths[i], ids[i]});
    }
  }
  std::sort(longs.begin(), longs.end());
  for (std::vector<int64_t>& bin : pack_short(std::move(shorts), cs)) {
    Chunk c;
    c.id = static_cast<int64_t>(plan.chunks.size());
    c.kind = kStandalone;
    c.seg_off = static_cast<int64_t>(plan.segments.size());
    std::sort(bin.begin(), bin.end());  // segments in sequence-id order
    for (int64_t id : bin) {
      const int64_t len = len_of.at(id);
      plan.segments.push_back({id, 0, len});
      c.total += len;
    }
    c.seg_cnt = static_cast<int64_t>(bin.size());
    plan.chunks.push_back(c);
  }
  int64_t group = 0;
  for (const auto& [id, len] : longs) {  // split_long (chunker.hpp:42-65)
    const int64_t pieces = (len + cs - 1) / cs;
    for (int64_t i = 0; i < pieces; ++i) {
      Chunk c;
      c.id = static_cast<int64_t>(plan.chunks.size());
      c.kind = kDependent;
      c.group = group;
      c.index = i;
      c.seg_off = static_cast<int64_t>(plan.segments.size());
      c.seg_cnt = 1;
      c.total = std::min(cs, len - i * cs);
      plan.segments.push_back({id, i * cs, c.total});
      plan.groups[group].push_back(c.id);
      plan.chunks.push_back(c);
    }
    ++group;
  }
  for (const Chunk& c : plan.chunks) {
    plan.index_of[c.id] = static_cast<int64_t>(&c - plan.chunks.data());
    plan.chunk_tokens[c.id] = c.total;
  }
  return plan;
}

void schedule_step(Plan& plan, int64_t k) {
  if (k < 1) throw ValidationError("retention budget k must be at least 1");
  plan.k = k;
  plan.events.clear();
  std::set<int64_t> emitted;
  for (const Chunk& c : plan.chunks) {
    if (c.kind == kStandalone) {
      plan.events.push_back({kFwdRetain, c.id, -1, -1, false, false, false, false});
      plan.events.push_back({kBackward, c.id, -1, -1, false, false, false, false});
      continue;
    }
    if (!emitted.insert(c.group).second) continue;
    const std::vector<int64_t>& members = plan.groups.at(c.group);
    const int64_t n = static_cast<int64_t>(members.size());
    for (const auto& [kind, idx, rec] : skeleton(n, k))
      plan.events.push_back(make_event(kind, members[static_cast<size_t>(idx - 1)], c.group, idx - 1, rec, n));
  }
  validate(plan);
}

Plan schedule_group(int64_t n, int64_t k, int64_t cs) {
  Plan plan;
  plan.chunk_size = cs;
  plan.k = k;
  for (const auto& [kind, idx, rec] : skeleton(n, k))
    plan.events.push_back(make_event(kind, idx, 0, idx - 1, rec, n));
  for (int64_t i = 1; i <= n; ++i) {
    plan.groups[0].push_back(i);
    plan.chunk_tokens[i] = cs;
  }
  validate(plan);
  return plan;
}

void validate(Plan& plan) {
  plan.peak_retained = 0;
  plan.recompute_tokens = 0;
  plan.violations.clear();
  std::map<int64_t, std::pair<int64_t, int64_t>> place;  // chunk -> (group, idx)
  for (const auto& [g, mem] : plan.groups)
    for (size_t i = 0; i < mem.size(); ++i) place[mem[i]] = {g, static_cast<int64_t>(i)};
  auto tokens_of = [&](int64_t c) {
    auto it = plan.chunk_tokens.find(c);
    return it == plan.chunk_tokens.end() ? plan.chunk_size : it->second;
  };
  std::map<int64_t, int64_t> forwards, backwards, hi_first, lo_back;
  std::set<int64_t> retained;
  int64_t held = 0;
  for (const Event& e : plan.events) {
    const int64_t c = e.chunk;
    const auto pit = place.find(c);
    const bool grouped = pit != place.end();
    const int64_t g = grouped ? pit->second.first : -1;
    const int64_t idx = grouped ? pit->second.second : -1;
    if (e.kind == kBackward) {
      if (retained.erase(c)) {
        held -= tokens_of(c);
      } else {
        plan.violations.push_back("backward of chunk " + std::to_string(c) + " without a live retain-forward");
      }
      if (++backwards[c] > 1)
        plan.violations.push_back("chunk " + std::to_string(c) + " backwarded more than once");
      if (grouped) {
        auto it = lo_back.find(g);
        if (it != lo_back.end() && idx != it->second - 1)
          plan.violations.push_back("backward of chunk " + std::to_string(c) + " out of descending group order");
        lo_back[g] = idx;
      }
      continue;
    }
    const bool first_pass = forwards[c]++ == 0;
    if (!first_pass) plan.recompute_tokens += tokens_of(c);
    if (grouped && first_pass) {
      auto it = hi_first.find(g);
      const int64_t prev = it == hi_first.end() ? -1 : it->second;
      if (idx != prev + 1)
        plan.violations.push_back("first forward of chunk " + std::to_string(c) + " out of ascending group order");
      hi_first[g] = std::max(prev, idx);
    }
    if (e.kind == kFwdRetain && retained.insert(c).second) {
      held += tokens_of(c);
      plan.peak_retained = std::max(plan.peak_retained, held);
    }
  }
  for (const auto& [c, cnt] : forwards) {
    (void)cnt;
    if (backwards[c] == 0) plan.violations.push_back("chunk " + std::to_string(c) + " was never backwarded");
  }
}

std::string listing(const Plan& plan) {
  std::string out;
  for (const Event& e : plan.events) {
    out += e.kind == kFwdDiscard ? "F-" : e.kind == kFwdRetain ? "F+" : "B ";
    out += " chunk=" + std::to_string(e.chunk) + " group=";
    out += e.group < 0 ? std::string("-") : std::to_string(e.group);
    if (e.recompute) out += " recompute";
    out += "\n";
  }
  return out;
}

std::vector<Unit> plan_units(const Plan& plan, double alpha, double beta) {
  std::vector<Unit> units;
  std::set<int64_t> seen;
  for (size_t p = 0; p < plan.chunks.size(); ++p) {
    const Chunk& c = plan.chunks[p];
    if (c.kind == kStandalone) {
      Unit u;
      u.chunk_pos.push_back(static_cast<int64_t>(p));
      double pairs = 0;
      for (int64_t s = 0; s < c.seg_cnt; ++s) {
        const double L = static_cast<double>(plan.segments[c.seg_off + s].len);
        pairs += L * (L + 1) / 2;
      }
      u.cost = alpha * c.total + beta * pairs;
      u.tokens = c.total;
      units.push_back(u);
      continue;
    }
    if (!seen.insert(c.group).second) continue;
    Unit u;
    const auto& mem = plan.groups.at(c.group);
    const int64_t n = static_cast<int64_t>(mem.size());
    for (int64_t i = 0; i < n; ++i) {
      const int64_t pos = plan.index_of.at(mem[i]);
      const Chunk& m = plan.chunks[pos];
      const Segment& s = plan.segments[m.seg_off];
      const double L = static_cast<double>(s.len), P = static_cast<double>(s.start);
      const double c1 = alpha * L + beta * (L * P + L * (L + 1) / 2);
      u.cost += c1;
      if (n > plan.k && i < n - plan.k) u.cost += 0.29 * c1;  // recompute forward (measured F/(F+B))
      u.tokens += m.total;
      u.chunk_pos.push_back(pos);
    }
    units.push_back(u);
  }
  return units;
}

std::vector<std::vector<int64_t>> lpt_assign(const std::vector<Unit>& units, int64_t world) {
  if (world < 1) throw ValidationError("world size must be at least 1");
  std::vector<int64_t> order(units.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = static_cast<int64_t>(i);
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
    return units[a].cost > units[b].cost;
  });
  std::vector<double> load(static_cast<size_t>(world), 0.0);
  std::vector<std::vector<int64_t>> out(static_cast<size_t>(world));
  for (int64_t u : order) {
    size_t best = 0;
    for (size_t r = 1; r < load.size(); ++r)
      if (load[r] < load[best]) best = r;
    load[best] += units[u].cost;
    out[best].push_back(u);
  }
  for (auto& v : out) std::sort(v.begin(), v.end());
  return out;
}

Plan sub_plan(const Plan& global, const std::vector<Unit>& units,
              const std::vector<int64_t>& mine, int64_t k) {
  Plan p;
  p.chunk_size = global.chunk_size;
  std::vector<int64_t> pos;
  for (int64_t u : mine)
    for (int64_t c : units[u].chunk_pos) pos.push_back(c);
  std::sort(pos.begin(), pos.end());  // keep global plan order
  for (int64_t gp : pos) {
    Chunk c = global.chunks[gp];
    const int64_t off = static_cast<int64_t>(p.segments.size());
    for (int64_t s = 0; s < c.seg_cnt; ++s) p.segments.push_back(global.segments[c.seg_off + s]);
    c.seg_off = off;
    p.index_of[c.id] = static_cast<int64_t>(p.chunks.size());
    p.chunk_tokens[c.id] = c.total;
    if (c.kind == kDependent) p.groups[c.group] = global.groups.at(c.group);
    p.chunks.push_back(c);
  }
  schedule_step(p, k);
  return p;
}

}  // namespace cfb
