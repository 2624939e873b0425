// WR dynamic program and WD whole-network selection.
//
// Both must reproduce the reference's *choices*, not just its optimal totals:
// the DP keeps the reference's recurrence and tie rule
// (wr_optimizer.hpp:74-95), the WD fronts keep its candidate order
// (wd_optimizer.hpp:110-151), and the knapsack search keeps its group order,
// greedy seed, bounds and strict-improvement updates
// (wd_optimizer.hpp:221-560), because among equal-time selections the one
// returned is whichever that search order reaches first.
#include <atomic>
#include <exception>
#include <functional>
#include <limits>
#include <numeric>
#include <sstream>
#include <thread>

#include "planner.h"

namespace ucudnn {

// Worker pool: fn(i) for i < n on up to `jobs` threads, first exception
// rethrown (reference parallel.hpp:28-56).
void run_parallel(std::size_t n, unsigned jobs, const std::function<void(std::size_t)>& fn) {
  if (n == 0) return;
  if (jobs <= 1 || n == 1) {
    for (std::size_t i = 0; i < n; ++i) fn(i);
    return;
  }
  std::atomic<std::size_t> cursor{0};
  std::exception_ptr err;
  std::mutex mu;
  std::vector<std::thread> pool;
  for (std::size_t t = 0; t < std::min<std::size_t>(jobs, n); ++t)
    pool.emplace_back([&] {
      for (std::size_t i; (i = cursor.fetch_add(1)) < n;) {
        try {
          fn(i);
        } catch (...) {
          std::lock_guard<std::mutex> g(mu);
          if (!err) err = std::current_exception();
        }
      }
    });
  for (auto& th : pool) th.join();
  if (err) std::rethrow_exception(err);
}

// ------------------------------------------------------------------ WR -----
// T(0) = 0, T(b) = min over admissible s <= b of T_mu(s) + T(b - s); an equal
// time replaces the incumbent only if canonically smaller
// (wr_optimizer.hpp:52-97).
std::vector<WrRow> wr_table(const CostSource& src, const Kernel& k, std::int64_t B, std::int64_t limit,
                            Policy p) {
  if (B < 1) throw std::invalid_argument("mini_batch must be >= 1");
  if (limit < 0) throw std::invalid_argument("workspace_limit must be >= 0");
  const std::vector<std::int64_t> sizes = micro_sizes(p, B);
  std::vector<std::optional<Micro>> best_at(std::size_t(B) + 1);
  for (std::int64_t s : sizes) best_at[s] = src.fastest(k, s, limit);

  std::vector<WrRow> T(std::size_t(B) + 1);
  T[0].ok = true;
  for (std::int64_t b = 1; b <= B; ++b) {
    WrRow& row = T[b];
    for (std::int64_t s : sizes) {
      if (s > b) break;
      const std::optional<Micro>& head = best_at[s];
      const WrRow& tail = T[b - s];
      if (!head || !tail.ok) continue;
      Ratio t = head->time + tail.time;
      if (row.ok && t > row.time) continue;
      Plan cand = tail.plan ? Plan::join(Plan::one(*head), *tail.plan) : Plan::one(*head);
      if (!row.ok || t < row.time || plan_before(cand, *row.plan)) {
        row.ok = true;
        row.time = t;
        row.split = s;
        row.plan = std::move(cand);
      }
    }
  }
  return T;
}

WrPlan wr_plan(const CostSource& src, const Kernel& k, std::int64_t B, std::int64_t limit, Policy p) {
  std::vector<WrRow> T = wr_table(src, k, B, limit, p);
  if (!T[B].ok) {
    std::ostringstream os;
    os << "no feasible configuration for kernel '" << k.name << "' (" << op_name(k.op) << ", batch " << B
       << ") within workspace limit " << limit << " bytes";
    throw InfeasibleError(os.str());
  }
  return WrPlan{*T[B].plan, T[B].time};
}

// ------------------------------------------------------------------ WD -----
namespace {
struct Costed {
  Ratio time;
  std::int64_t ws;
  Plan plan;
};
const Ratio& time_of(const Costed& c) { return c.time; }
std::int64_t ws_of(const Costed& c) { return c.ws; }
bool tie_of(const Costed& a, const Costed& b) { return plan_before(a.plan, b.plan); }
}  // namespace

std::vector<Plan> desirable(std::vector<Plan> plans) {
  std::vector<Costed> v;
  v.reserve(plans.size());
  for (Plan& p : plans) v.push_back(Costed{p.time(), p.ws(), std::move(p)});
  v = pareto(std::move(v), time_of, ws_of, tie_of);
  std::vector<Plan> out;
  for (Costed& c : v) out.push_back(std::move(c.plan));
  return out;
}

// C(b) = D({m} + c : s admissible, m in C_mu(s), c in C(b - s)), duplicates
// collapsed in canonical order before pruning (wd_optimizer.hpp:84-160).
PlanSet plan_front(const CostSource& src, const Kernel& k, std::int64_t B, std::int64_t budget, Policy p,
                   std::size_t cap) {
  if (B < 1) throw std::invalid_argument("mini_batch must be >= 1");
  if (budget < 0) throw std::invalid_argument("workspace_budget must be >= 0");
  const std::vector<std::int64_t> sizes = micro_sizes(p, B);
  std::vector<std::vector<Micro>> mu(std::size_t(B) + 1);
  for (std::int64_t s : sizes) mu[s] = src.front(k, s, budget);

  // The reference materialises every candidate plan, sorts them canonically,
  // drops duplicates and then keeps the (time, ws) front with canonical ties
  // (wd_optimizer.hpp:110-143). Equivalent and much cheaper: sort unmaterialised
  // (time, ws, head, tail) tuples by (time, ws); a (time, ws) group that
  // survives the front contributes its canonically least plan, so only those
  // groups' plans are ever built. Duplicated plans have equal (time, ws), so
  // the reference's unique() cannot change the result.
  struct Cand {
    Ratio time;
    std::int64_t ws;
    std::int32_t s, mi, ri;  // head = mu[s][mi], tail = C[b - s][ri] (ri < 0: none)
  };
  std::vector<std::vector<Costed>> C(std::size_t(B) + 1);
  std::vector<Cand> cand;
  for (std::int64_t b = 1; b <= B; ++b) {
    cand.clear();
    for (std::int64_t s : sizes) {
      if (s > b) break;
      const auto& heads = mu[s];
      for (std::size_t mi = 0; mi < heads.size(); ++mi) {
        const Micro& m = heads[mi];
        if (s == b) {
          cand.push_back(Cand{m.time, m.ws, std::int32_t(s), std::int32_t(mi), -1});
          continue;
        }
        const auto& tails = C[b - s];
        for (std::size_t ri = 0; ri < tails.size(); ++ri)
          cand.push_back(Cand{m.time + tails[ri].time, std::max(m.ws, tails[ri].ws), std::int32_t(s),
                              std::int32_t(mi), std::int32_t(ri)});
      }
    }
    std::sort(cand.begin(), cand.end(), [](const Cand& x, const Cand& y) {
      if (int c = Ratio::cmp(x.time, y.time)) return c < 0;
      return x.ws < y.ws;
    });
    auto build = [&](const Cand& c) {
      Plan head = Plan::one(mu[c.s][std::size_t(c.mi)]);
      return c.ri < 0 ? head : Plan::join(head, C[b - c.s][std::size_t(c.ri)].plan);
    };
    std::vector<Costed>& out = C[b];
    for (std::size_t i = 0; i < cand.size();) {
      std::size_t j = i + 1;
      while (j < cand.size() && cand[j].ws == cand[i].ws && cand[j].time == cand[i].time) ++j;
      if (out.empty() || cand[i].ws < out.back().ws) {
        Plan best = build(cand[i]);
        for (std::size_t k = i + 1; k < j; ++k) {
          Plan p = build(cand[k]);
          if (plan_before(p, best)) best = std::move(p);
        }
        out.push_back(Costed{cand[i].time, cand[i].ws, std::move(best)});
      }
      i = j;
    }
    if (C[b].size() > cap) {
      std::ostringstream os;
      os << "configuration front for kernel '" << k.name << "' exceeds cap (" << C[b].size() << " > " << cap
         << ") at batch " << b;
      throw std::runtime_error(os.str());
    }
  }
  PlanSet out;
  out.kernel = k;
  for (Costed& c : C[B]) out.members.push_back(std::move(c.plan));
  return out;
}

void check_selection(const SelectionProblem& prob, const Selection& s) {
  if (s.chosen.size() != prob.sets.size())
    throw std::logic_error("solution must select one configuration per kernel");
  Ratio t;
  std::int64_t ws = 0;
  for (std::size_t i = 0; i < s.chosen.size(); ++i) {
    const auto& mem = prob.sets[i].members;
    if (std::find(mem.begin(), mem.end(), s.chosen[i]) == mem.end())
      throw std::logic_error("selected configuration is not in its choice set");
    t += s.chosen[i].time();
    ws += s.chosen[i].ws();
  }
  if (t != s.time || ws != s.ws) throw std::logic_error("solution totals do not match selection");
  if (s.ws > prob.budget) throw std::logic_error("solution exceeds the workspace budget");
}

namespace {

std::int64_t add_sat(std::int64_t a, std::int64_t b) {
  i128 s = i128(a) + b;
  return s > std::numeric_limits<std::int64_t>::max() ? std::numeric_limits<std::int64_t>::max()
                                                       : std::int64_t(s);
}

// Exact multiple-choice knapsack by depth-first branch and bound, a
// restatement of the reference ChoiceSolver (wd_optimizer.hpp:221-560).
class KnapsackSearch {
 public:
  explicit KnapsackSearch(const SelectionProblem& prob) : prob_(prob) {
    cap_ = std::min(prob.budget, std::numeric_limits<std::int64_t>::max() / 2);
    if (prob.budget < 0) throw std::invalid_argument("budget must be >= 0");
    if (prob.sets.empty()) throw std::invalid_argument("choice problem has no kernels");
    make_groups();
    sort_groups();
    make_suffixes();
    scaled_ = scale_times();
  }

  Selection run() {
    if (rest_ws_[0] > cap_) {
      std::ostringstream os;
      os << "infeasible: minimal total workspace " << rest_ws_[0] << " bytes exceeds budget " << prob_.budget
         << " bytes";
      throw InfeasibleError(os.str(), rest_ws_[0]);
    }
    if (scaled_) greedy_seed();
    cur_.assign(G_.size(), 0);
    search(0, 0, Ratio(0), 0);

    std::vector<const Plan*> pick(G_.size());
    Selection sel;
    for (std::size_t g = 0; g < G_.size(); ++g) {
      const Item& it = G_[g].items[best_[g]];
      pick[where_[g]] = &prob_.sets[where_[g]].members[std::size_t(it.member)];
      sel.time += it.time;
      sel.ws += it.ws;
    }
    for (const Plan* p : pick) sel.chosen.push_back(*p);
    check_selection(prob_, sel);
    return sel;
  }

 private:
  struct Item {
    Ratio time;
    std::int64_t ws = 0, scaled = 0;
    std::int32_t member = 0;
  };
  struct Group {
    std::vector<Item> items;          // time ascending, workspace descending
    std::vector<std::size_t> hull;    // hull position -> item index
    std::int64_t min_ws = 0, min_ws_scaled = 0, min_time_scaled = 0;
    Ratio min_time;
  };
  struct Step {  // one convex-hull edge: spend dws bytes to save dt (scaled)
    std::size_t group, pos;
    std::int64_t dws, dt;
  };

  // Items above the budget dropped, groups re-pruned (wd_optimizer.hpp:291-325).
  void make_groups() {
    for (const PlanSet& set : prob_.sets) {
      if (set.members.empty())
        throw std::invalid_argument("kernel '" + set.kernel.name + "' has an empty choice set");
      std::vector<Item> v;
      for (std::size_t m = 0; m < set.members.size(); ++m) {
        std::int64_t ws = set.members[m].ws();
        if (ws > cap_) continue;
        v.push_back(Item{set.members[m].time(), ws, 0, std::int32_t(m)});
      }
      v = pareto(
          std::move(v), [](const Item& i) -> const Ratio& { return i.time; }, [](const Item& i) { return i.ws; },
          [](const Item& a, const Item& b) { return a.member < b.member; });
      if (v.empty())
        throw InfeasibleError("infeasible: kernel '" + set.kernel.name + "' has no configuration within the budget");
      Group g;
      g.min_ws = v.back().ws;
      g.min_time = v.front().time;
      g.items = std::move(v);
      G_.push_back(std::move(g));
    }
  }

  static int compare_items(const std::vector<Item>& a, const std::vector<Item>& b) {
    if (a.size() != b.size()) return a.size() < b.size() ? -1 : 1;
    for (std::size_t i = 0; i < a.size(); ++i) {
      if (int c = Ratio::cmp(a[i].time, b[i].time)) return c;
      if (a[i].ws != b[i].ws) return a[i].ws < b[i].ws ? -1 : 1;
      if (a[i].member != b[i].member) return a[i].member < b[i].member ? -1 : 1;
    }
    return 0;
  }

  // Widest time spread first; identical item lists adjacent, ties by index
  // (wd_optimizer.hpp:341-365).
  void sort_groups() {
    std::vector<std::size_t> ord(G_.size());
    std::iota(ord.begin(), ord.end(), 0);
    std::vector<Ratio> spread(G_.size());
    for (std::size_t i = 0; i < G_.size(); ++i) spread[i] = G_[i].items.back().time - G_[i].items.front().time;
    std::sort(ord.begin(), ord.end(), [&](std::size_t a, std::size_t b) {
      if (spread[a] != spread[b]) return spread[a] > spread[b];
      if (int c = compare_items(G_[a].items, G_[b].items)) return c < 0;
      return a < b;
    });
    std::vector<Group> sorted;
    twin_.assign(G_.size(), false);
    for (std::size_t i = 0; i < ord.size(); ++i) {
      sorted.push_back(std::move(G_[ord[i]]));
      where_.push_back(ord[i]);
      if (i) twin_[i] = compare_items(sorted[i].items, sorted[i - 1].items) == 0;
    }
    G_ = std::move(sorted);
  }

  void make_suffixes() {
    std::size_t n = G_.size();
    rest_ws_.assign(n + 1, 0);
    rest_time_.assign(n + 1, Ratio(0));
    for (std::size_t g = n; g-- > 0;) {
      rest_ws_[g] = add_sat(rest_ws_[g + 1], G_[g].min_ws);
      rest_time_[g] = rest_time_[g + 1] + G_[g].min_time;
    }
  }

  // Integer times over a common denominator (capped at 1e18) for the LP
  // bound; without it only the weak bounds run (wd_optimizer.hpp:377-411).
  bool scale_times() {
    std::int64_t den = 1;
    for (const Group& g : G_)
      for (const Item& it : g.items) {
        std::int64_t q = Ratio::gcd64(den, it.time.den());
        i128 l = i128(den / q) * it.time.den();
        if (l > 1000000000000000000LL) return false;
        den = std::int64_t(l);
      }
    const std::int64_t num_cap = std::numeric_limits<std::int64_t>::max() / (4 * std::int64_t(G_.size() + 2));
    for (Group& g : G_) {
      for (Item& it : g.items) {
        i128 v = i128(it.time.num()) * (den / it.time.den());
        if (v < 0 || v > num_cap) return false;
        it.scaled = std::int64_t(v);
      }
      g.min_ws_scaled = g.items.back().scaled;
      g.min_time_scaled = g.items.front().scaled;
    }
    std::size_t n = G_.size();
    rest_base_s_.assign(n + 1, 0);
    rest_min_s_.assign(n + 1, 0);
    for (std::size_t g = n; g-- > 0;) {
      rest_base_s_[g] = rest_base_s_[g + 1] + G_[g].min_ws_scaled;
      rest_min_s_[g] = rest_min_s_[g + 1] + G_[g].min_time_scaled;
    }
    make_hull_steps();
    return true;
  }

  // Lower convex hull of each group's (ws, time) points, walked from the
  // cheapest-workspace item; edges sorted by saving per byte
  // (wd_optimizer.hpp:413-455).
  void make_hull_steps() {
    for (std::size_t g = 0; g < G_.size(); ++g) {
      const auto& items = G_[g].items;
      struct P { std::int64_t ws, t; std::size_t idx; };
      std::vector<P> h;
      for (std::size_t i = items.size(); i-- > 0;) {
        P p{items[i].ws, items[i].scaled, i};
        while (h.size() >= 2) {
          const P& a = h[h.size() - 2];
          const P& b = h.back();
          i128 cross = i128(b.ws - a.ws) * (p.t - a.t) - i128(b.t - a.t) * (p.ws - a.ws);
          if (cross > 0) break;
          h.pop_back();
        }
        h.push_back(p);
      }
      G_[g].hull.clear();
      for (const P& p : h) G_[g].hull.push_back(p.idx);
      for (std::size_t i = 0; i + 1 < h.size(); ++i)
        steps_.push_back(Step{g, i, h[i + 1].ws - h[i].ws, h[i].t - h[i + 1].t});
    }
    std::sort(steps_.begin(), steps_.end(), [](const Step& a, const Step& b) {
      i128 l = i128(a.dt) * b.dws, r = i128(b.dt) * a.dws;
      if (l != r) return l > r;
      if (a.group != b.group) return a.group < b.group;
      return a.pos < b.pos;
    });
  }

  // Incumbent: every group at its min-workspace hull point, then whole hull
  // edges in ratio order while they fit (wd_optimizer.hpp:459-480).
  void greedy_seed() {
    std::vector<std::size_t> at(G_.size(), 0);
    std::int64_t room = cap_ - rest_ws_[0];
    for (const Step& st : steps_) {
      if (st.pos != at[st.group] || st.dws > room) continue;
      room -= st.dws;
      ++at[st.group];
    }
    best_.assign(G_.size(), 0);
    Ratio t;
    std::int64_t ts = 0;
    for (std::size_t g = 0; g < G_.size(); ++g) {
      best_[g] = G_[g].hull[at[g]];
      t += G_[g].items[best_[g]].time;
      ts += G_[g].items[best_[g]].scaled;
    }
    best_time_ = t;
    best_scaled_ = ts;
    have_ = true;
  }

  // Fractional LP relaxation over the remaining groups' hulls
  // (wd_optimizer.hpp:486-505).
  std::int64_t lp_floor(std::size_t g, std::int64_t used, std::int64_t ts) const {
    std::int64_t room = cap_ - used - rest_ws_[g];
    i128 saved = 0;
    for (const Step& st : steps_) {
      if (st.group < g) continue;
      if (room <= 0) break;
      if (st.dws <= room) {
        saved += st.dt;
        room -= st.dws;
      } else {
        saved += (i128(st.dt) * room + st.dws - 1) / st.dws;
        break;
      }
    }
    i128 v = i128(ts + rest_base_s_[g]) - saved;
    return v < 0 ? 0 : std::int64_t(v);
  }

  // wd_optimizer.hpp:507-541.
  void search(std::size_t g, std::int64_t used, Ratio t, std::int64_t ts) {
    if (g == G_.size()) {
      if (!have_ || t < best_time_) {
        have_ = true;
        best_time_ = t;
        best_scaled_ = ts;
        best_ = cur_;
      }
      return;
    }
    if (have_) {
      if (scaled_) {
        if (ts + rest_min_s_[g] >= best_scaled_) return;
        if (lp_floor(g, used, ts) >= best_scaled_) return;
      } else if (t + rest_time_[g] >= best_time_) {
        return;
      }
    }
    const Group& grp = G_[g];
    std::size_t first = (g > 0 && twin_[g]) ? cur_[g - 1] : 0;  // non-decreasing along twin runs
    for (std::size_t i = first; i < grp.items.size(); ++i) {
      const Item& it = grp.items[i];
      Ratio nt = t + it.time;
      if (have_ && nt + rest_time_[g + 1] >= best_time_) break;
      std::int64_t nu = used + it.ws;
      if (add_sat(nu, rest_ws_[g + 1]) > cap_) continue;
      cur_[g] = i;
      search(g + 1, nu, nt, ts + it.scaled);
    }
  }

  const SelectionProblem& prob_;
  std::int64_t cap_ = 0;
  std::vector<Group> G_;
  std::vector<std::size_t> where_;  // search position -> problem index
  std::vector<bool> twin_;
  std::vector<std::int64_t> rest_ws_, rest_base_s_, rest_min_s_;
  std::vector<Ratio> rest_time_;
  std::vector<Step> steps_;
  bool scaled_ = false;
  std::vector<std::size_t> cur_, best_;
  Ratio best_time_;
  std::int64_t best_scaled_ = 0;
  bool have_ = false;
};

}  // namespace

Selection select_plans(const SelectionProblem& prob) { return KnapsackSearch(prob).run(); }

// Hash-deduplicated fronts feed one selection problem (wd_optimizer.hpp:589-649).
WdPlan wd_plan(const CostSource& src, const std::vector<Kernel>& kernels, std::int64_t budget, Policy p,
               unsigned jobs, std::size_t cap) {
  if (kernels.empty()) throw std::invalid_argument("no kernels to optimize");
  if (budget < 0) throw std::invalid_argument("workspace_budget must be >= 0");
  std::vector<std::uint64_t> hashes;
  std::map<std::uint64_t, std::size_t> slot;
  std::vector<const Kernel*> uniq;
  for (const Kernel& k : kernels) {
    hashes.push_back(k.hash());
    if (slot.emplace(hashes.back(), uniq.size()).second) uniq.push_back(&k);
  }
  std::vector<PlanSet> fronts(uniq.size());
  run_parallel(uniq.size(), jobs, [&](std::size_t i) {
    fronts[i] = plan_front(src, *uniq[i], uniq[i]->batch, budget, p, cap);
  });
  for (std::size_t i = 0; i < fronts.size(); ++i)
    if (fronts[i].members.empty()) {
      std::ostringstream os;
      os << "no feasible configuration for kernel '" << uniq[i]->name << "' (" << op_name(uniq[i]->op)
         << ") within total budget " << budget << " bytes";
      throw InfeasibleError(os.str());
    }
  SelectionProblem prob;
  prob.budget = budget;
  for (std::size_t i = 0; i < kernels.size(); ++i)
    prob.sets.push_back(PlanSet{kernels[i], fronts[slot.at(hashes[i])].members});
  Selection sel = select_plans(prob);

  WdPlan out;
  out.kernels = kernels;
  out.chosen = std::move(sel.chosen);
  out.time = sel.time;
  out.ws = sel.ws;
  out.unique_kernels = uniq.size();
  for (const PlanSet& s : prob.sets) {
    out.variables += s.members.size();
    out.max_front = std::max(out.max_front, s.members.size());
  }
  return out;
}

}  // namespace ucudnn
