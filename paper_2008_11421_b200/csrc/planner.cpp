#include "planner.hpp"

#include <algorithm>
#include <cmath>
#include <functional>
#include <limits>
#include <map>
#include <optional>
#include <set>

namespace krt {
namespace {

constexpr double kEps = 1e-12;             // planner.py:37
constexpr double kPenaltyCapacity = 1e15;  // planner.py:810
constexpr double kPenaltyStructural = 1e18;
constexpr int kAutoExhaustiveLayers = 12;  // planner.py:40
constexpr int kOpt2ExhaustiveBound = 8;    // planner.py:41
const double kInf = std::numeric_limits<double>::infinity();

using Costs = std::map<int, BlockCost>;
using Partition = std::vector<std::pair<int, int>>;
using Flags = std::set<int>;

// planner.py:71-107: per-layer prefix sums; block costs for any range in O(1)
struct CostTable {
  double mult, swap_rate, rate;
  std::vector<double> eff, bytes, wt, grad, welems;
  CostTable(const Model& g, const Hardware& hw) {
    mult = hw.backward_multiplier;
    swap_rate = hw.swap_throughput();
    rate = hw.compute_rate;
    int n = g.num_layers();
    eff.assign(n + 1, 0.0);
    bytes.assign(n + 1, 0.0);
    wt.assign(n + 1, 0.0);
    grad.assign(n + 1, 0.0);
    welems.assign(n + 1, 0.0);
    for (int i = 1; i <= n; ++i) {
      const Layer& l = g.layer(i);
      LayerMem m = layer_memory(l, g.batch);
      eff[i] = eff[i - 1] + layer_ops(l, g.batch) / hw.kind_efficiency(l.kind);
      bytes[i] = bytes[i - 1] + (double)(m.fwd + m.wt);
      wt[i] = wt[i - 1] + (double)m.wt;
      grad[i] = grad[i - 1] + (double)m.grad;
      welems[i] = welems[i - 1] + (double)weight_elements(l);
    }
  }
  BlockCost range_cost(int id, int lo, int hi) const {
    BlockCost c;
    c.block_id = id;
    c.fwd_seconds = (eff[hi] - eff[lo - 1]) / rate;
    c.bytes = bytes[hi] - bytes[lo - 1];
    c.bwd_seconds = c.fwd_seconds * mult;
    c.wt_bytes = wt[hi] - wt[lo - 1];
    c.grad_bytes = grad[hi] - grad[lo - 1];
    c.weight_elems = welems[hi] - welems[lo - 1];
    c.swap_seconds = c.bytes / swap_rate;
    return c;
  }
};

// planner.py:110-121
void build_blocks(const Partition& part, const CostTable& t, std::vector<Block>* blocks, Costs* costs) {
  blocks->clear();
  costs->clear();
  for (size_t i = 0; i < part.size(); ++i) {
    int id = (int)i + 1;
    BlockCost c = t.range_cost(id, part[i].first, part[i].second);
    (*costs)[id] = c;
    Block b;
    b.id = id;
    b.first_layer = part[i].first;
    b.last_layer = part[i].second;
    b.swap_bytes = c.bytes;
    blocks->push_back(b);
  }
}

// planner.py:124-144
int retained_start(const std::vector<Block>& blocks, const Costs& costs, double capacity) {
  int nb = (int)blocks.size();
  PySum total;
  for (auto& b : blocks) total.add(costs.at(b.id).bytes);
  if (total.value() <= capacity + kEps) return 1;
  std::vector<double> suffix_from(nb + 2, 0.0);
  double suffix = 0.0;
  for (int i = nb; i >= 1; --i) {
    suffix += costs.at(i).bytes;
    suffix_from[i] = suffix;
  }
  for (int k = 2; k <= nb; ++k)
    if (suffix_from[k] + costs.at(k - 1).bytes <= capacity + kEps) return k;
  return nb + 1;
}

// planner.py:147-162
Flags forced_recompute(const std::vector<Block>& blocks, const Model& g, int k_ret) {
  std::map<int, int> block_of;
  for (auto& b : blocks)
    for (int l = b.first_layer; l <= b.last_layer; ++l) block_of[l] = b.id;
  Flags forced;
  for (auto& e : g.edges) {
    if (!e.skip) continue;
    int sb = block_of.at(e.src), db = block_of.at(e.dst);
    if (db > sb + 1 && sb < k_ret && sb != (int)blocks.size()) forced.insert(sb);
  }
  return forced;
}

double stage_duration(const std::vector<PlanOp>& ops, const Costs& costs) {
  double d = 0.0;
  for (auto& op : ops) {
    const BlockCost& c = costs.at(op.block);
    if (op.action == Action::FW || op.action == Action::RECOMPUTE_FW) d = std::max(d, c.fwd_seconds);
    else if (op.action == Action::BW) d = std::max(d, c.bwd_seconds);
    else d = std::max(d, c.swap_seconds);
  }
  return d;
}

std::vector<std::pair<int, int>> recompute_runs(const Flags& rec, int nb) {
  std::vector<std::pair<int, int>> runs;
  int i = 1;
  while (i <= nb) {
    if (rec.count(i)) {
      int j = i;
      while (j + 1 <= nb && rec.count(j + 1)) ++j;
      runs.emplace_back(i, j);
      i = j + 1;
    } else {
      ++i;
    }
  }
  return runs;
}

// planner.py:256-325
std::vector<std::vector<PlanOp>> capacity_backward_stages(const std::vector<Block>& blocks, const Model& g,
                                                          const Costs& costs, const std::vector<int>& swapped,
                                                          const Flags& recompute, int nb) {
  auto pos_of = [&](int i) { return nb - i + 1; };
  auto block_at = [&](int p) { return nb - p + 1; };
  auto skip_map = skip_requirement_map(blocks, g);
  std::map<int, std::vector<int>> skip_targets;
  for (auto& [dst, sources] : skip_map)
    for (int src : sources) skip_targets[src].push_back(dst);
  auto runs = recompute_runs(recompute, nb);
  std::map<std::pair<int, int>, int> run_insert_pos;
  std::map<int, std::pair<int, int>> run_of_start;
  for (auto& run : runs) {
    int pos = pos_of(run.second);
    for (int m = run.first; m <= run.second; ++m) {
      auto it = skip_targets.find(m);
      if (it != skip_targets.end())
        for (int dst : it->second) pos = std::min(pos, pos_of(dst));
    }
    run_insert_pos[run] = pos;
    run_of_start[run.first] = run;
  }
  std::map<int, int> first_need;
  for (int q : swapped) {
    int need = pos_of(q);
    auto rs = run_of_start.find(q + 1);
    if (rs != run_of_start.end()) need = std::min(need, run_insert_pos[rs->second]);
    auto it = skip_targets.find(q);
    if (it != skip_targets.end())
      for (int dst : it->second) need = std::min(need, pos_of(dst));
    first_need[q] = need;
  }
  std::vector<int> queue = swapped;
  std::sort(queue.begin(), queue.end(), [&](int a, int b) {
    if (first_need[a] != first_need[b]) return first_need[a] < first_need[b];
    return -a < -b;
  });
  std::map<int, std::vector<int>> attach;
  double t = 0.0, chan = 0.0;
  size_t qi = 0;
  for (int p = 1; p <= nb; ++p) {
    while (qi < queue.size() && (chan <= t + kEps || first_need[queue[qi]] <= p)) {
      int q = queue[qi++];
      int pa = std::max(std::min(p, first_need[q] - 1), 0);
      attach[pa].push_back(q);
      chan = std::max(chan, t) + costs.at(q).swap_seconds;
    }
    t += costs.at(block_at(p)).bwd_seconds;
  }
  while (qi < queue.size()) {
    int q = queue[qi++];
    int pa = std::max(std::min(nb, first_need[q] - 1), 0);
    attach[pa].push_back(q);
  }
  std::map<int, std::vector<std::pair<int, int>>> inserts;
  for (auto& run : runs) inserts[run_insert_pos[run]].push_back(run);
  std::vector<std::vector<PlanOp>> stages;
  for (int q : attach[0]) stages.push_back({PlanOp{Action::SWAP_IN, q}});
  for (int p = 1; p <= nb; ++p) {
    auto ins = inserts[p];
    std::sort(ins.begin(), ins.end());
    for (auto& run : ins)
      for (int m = run.first; m <= run.second; ++m) stages.push_back({PlanOp{Action::RECOMPUTE_FW, m}});
    std::vector<PlanOp> ops{PlanOp{Action::BW, block_at(p)}};
    for (int q : attach[p]) ops.push_back(PlanOp{Action::SWAP_IN, q});
    stages.push_back(ops);
  }
  return stages;
}

// planner.py:169-225
Plan generate_schedule(const std::vector<Block>& blocks, const Model& g, const Hardware& hw, Strategy strategy,
                       const Costs& costs) {
  int nb = (int)blocks.size();
  if (nb == 0) throw PlannerMisuse("cannot schedule an empty block list");
  int k_ret;
  Flags recompute;
  std::vector<int> swapped;
  if (strategy == Strategy::EAGER) {
    k_ret = nb + 1;
    for (int i = 1; i <= nb; ++i) swapped.push_back(i);
  } else {
    k_ret = retained_start(blocks, costs, hw.capacity_bytes);
    if (strategy == Strategy::CAPACITY_RECOMPUTE)
      for (auto& b : blocks)
        if (b.recompute && b.id < k_ret) recompute.insert(b.id);
    for (int i = 1; i < k_ret; ++i)
      if (!recompute.count(i)) swapped.push_back(i);
  }
  Flags regen = recompute;
  regen.erase(nb);
  Plan plan;
  plan.strategy = strategy;
  for (auto& b : blocks) {
    Block f = b;
    f.recompute = recompute.count(b.id) > 0;
    f.checkpoint = strategy != Strategy::EAGER && b.id >= k_ret;
    plan.blocks.push_back(f);
  }
  std::set<int> swapped_set(swapped.begin(), swapped.end());
  std::vector<std::vector<PlanOp>> raw;
  for (int j = 1; j <= nb; ++j) {
    std::vector<PlanOp> ops{PlanOp{Action::FW, j}};
    if (j >= 2 && swapped_set.count(j - 1)) ops.push_back(PlanOp{Action::SWAP_OUT, j - 1});
    raw.push_back(ops);
  }
  if (swapped_set.count(nb)) raw.push_back({PlanOp{Action::SWAP_OUT, nb}});
  if (strategy == Strategy::EAGER) {
    raw.push_back({PlanOp{Action::SWAP_IN, nb}});
    for (int j = nb; j > 1; --j) raw.push_back({PlanOp{Action::BW, j}, PlanOp{Action::SWAP_IN, j - 1}});
    raw.push_back({PlanOp{Action::BW, 1}});
  } else {
    auto bw = capacity_backward_stages(plan.blocks, g, costs, swapped, regen, nb);
    raw.insert(raw.end(), bw.begin(), bw.end());
  }
  for (size_t i = 0; i < raw.size(); ++i) {
    Stage s;
    s.id = (int)i + 1;
    s.ops = raw[i];
    s.duration = stage_duration(raw[i], costs);
    plan.stages.push_back(s);
  }
  return plan;
}

std::vector<Block> flagged(const std::vector<Block>& blocks, const Flags& flags) {
  std::vector<Block> out = blocks;
  for (auto& b : out) b.recompute = flags.count(b.id) > 0;
  return out;
}

struct Candidate {
  bool feasible = false;
  double makespan = kInf, stall = kInf;
  Plan plan;
  std::string reason;
};

// planner.py:517-537 (lean)
Candidate evaluate_blocks(const std::vector<Block>& blocks, const Model& g, const Hardware& hw, Strategy strategy,
                          const Costs& costs) {
  Candidate c;
  Plan plan = generate_schedule(blocks, g, hw, strategy, costs);
  auto v = residency_memory_walk(plan, g, hw, nullptr);
  if (!v.empty()) {
    c.reason = v[0];
    return c;
  }
  double mk, st, pk;
  if (!plan_metrics(plan, g, hw, costs, &mk, &st, &pk)) {
    auto ops = build_engine_ops(plan, g, hw, costs);
    EngineResult er = run_engine(ops, base_resources(hw), hw.capacity_bytes, true);
    std::string s = "simulation deadlock; blocked ops: ";
    for (size_t i = 0; i < er.blocked.size(); ++i) s += (i ? "; " : "") + er.blocked[i];
    c.reason = s;
    return c;
  }
  c.feasible = true;
  c.makespan = mk;
  c.stall = st;
  c.plan = std::move(plan);
  return c;
}

void recompute_candidates(const std::vector<Block>& blocks, const Costs& costs, const Model& g, const Hardware& hw,
                          int* k_ret, Flags* forced, std::vector<int>* free) {
  *k_ret = retained_start(blocks, costs, hw.capacity_bytes);
  *forced = forced_recompute(blocks, g, *k_ret);
  free->clear();
  for (int i = 1; i < *k_ret; ++i)
    if (!forced->count(i)) free->push_back(i);
}

// planner.py:559-569
Flags greedy_recompute(const std::vector<Block>& blocks, const Costs& costs, const Model& g, const Hardware& hw) {
  int k_ret;
  Flags forced;
  std::vector<int> free;
  recompute_candidates(blocks, costs, g, hw, &k_ret, &forced, &free);
  Flags flags = forced;
  for (auto it = free.rbegin(); it != free.rend(); ++it) {
    int d = *it;
    if (flags.count(d + 1)) continue;
    if (costs.at(d).fwd_seconds < costs.at(d).swap_seconds - kEps) flags.insert(d);
  }
  return flags;
}

std::vector<int> flags_key(const Flags& flags, int nb) {
  std::vector<int> k;
  for (int f : flags) k.push_back(nb - f);
  std::sort(k.begin(), k.end());
  return k;
}

template <class F>
void for_combinations(const std::vector<int>& items, int r, F&& fn) {
  int n = (int)items.size();
  if (r > n) return;
  std::vector<int> idx(r);
  for (int i = 0; i < r; ++i) idx[i] = i;
  std::vector<int> combo(r);
  while (true) {
    for (int i = 0; i < r; ++i) combo[i] = items[idx[i]];
    fn(combo);
    int i = r - 1;
    while (i >= 0 && idx[i] == i + n - r) --i;
    if (i < 0) return;
    ++idx[i];
    for (int j = i + 1; j < r; ++j) idx[j] = idx[j - 1] + 1;
  }
}

// planner.py:572-614
std::vector<Block> solve_opt2(const std::vector<Block>& blocks, const Model& g, const Hardware& hw,
                              const Costs& costs) {
  int k_ret;
  Flags forced;
  std::vector<int> free;
  recompute_candidates(blocks, costs, g, hw, &k_ret, &forced, &free);
  if ((int)free.size() > kOpt2ExhaustiveBound) {
    std::optional<std::vector<Block>> best;
    double best_mk = kInf;
    for (const Flags& fl : {greedy_recompute(blocks, costs, g, hw), forced}) {
      auto fb = flagged(blocks, fl);
      Candidate r = evaluate_blocks(fb, g, hw, Strategy::CAPACITY_RECOMPUTE, costs);
      if (r.feasible && r.makespan < best_mk) {
        best = fb;
        best_mk = r.makespan;
      }
    }
    return best ? *best : flagged(blocks, forced);
  }
  int nb = (int)blocks.size();
  std::optional<std::vector<Block>> best;
  std::tuple<double, double, size_t, std::vector<int>> best_key;
  for (int r = 0; r <= (int)free.size(); ++r)
    for_combinations(free, r, [&](const std::vector<int>& combo) {
      Flags fl = forced;
      fl.insert(combo.begin(), combo.end());
      auto fb = flagged(blocks, fl);
      Candidate res = evaluate_blocks(fb, g, hw, Strategy::CAPACITY_RECOMPUTE, costs);
      if (!res.feasible) return;
      auto key = std::make_tuple(res.makespan, res.stall, fl.size(), flags_key(fl, nb));
      if (!best || key < best_key) {
        best_key = key;
        best = fb;
      }
    });
  return best ? *best : flagged(blocks, forced);
}

double transfer_lower_bound(const Costs& costs, const std::vector<int>& swapped, bool duplex) {
  PySum moved;
  for (int q : swapped) moved.add(costs.at(q).swap_seconds);
  return duplex ? moved.value() : 2.0 * moved.value();
}

bool run_bytes_exceed(const std::vector<int>& flags_sorted, const Costs& costs, int nb, double capacity) {
  double run_bytes = 0.0;
  int prev = -1;
  bool have_prev = false;
  for (int f : flags_sorted) {
    if (f == nb) continue;
    if (have_prev && f == prev + 1) run_bytes += costs.at(f).bytes;
    else run_bytes = costs.at(f).bytes;
    if (run_bytes > capacity + kEps) return true;
    prev = f;
    have_prev = true;
  }
  return false;
}

Partition splits_to_partition(const std::vector<int>& splits, int num) {
  std::vector<int> bounds{0};
  bounds.insert(bounds.end(), splits.begin(), splits.end());
  bounds.push_back(num);
  Partition p;
  for (size_t i = 0; i + 1 < bounds.size(); ++i) p.emplace_back(bounds[i] + 1, bounds[i + 1]);
  return p;
}

// planner.py:814-828
double eval_one(const std::vector<Block>& blocks, const Model& g, const Hardware& hw, Strategy strategy,
                const Costs& costs) {
  Plan plan = generate_schedule(blocks, g, hw, strategy, costs);
  double peak_demand = 0.0;
  auto v = residency_memory_walk(plan, g, hw, &peak_demand);
  if (!v.empty()) {
    bool all_cap = true;
    for (auto& s : v) all_cap &= s.find("exceeding capacity") != std::string::npos;
    if (all_cap) return kPenaltyCapacity + peak_demand - hw.capacity_bytes;
    return kPenaltyStructural;
  }
  double mk, st, pk;
  if (!plan_metrics(plan, g, hw, costs, &mk, &st, &pk)) return kPenaltyStructural;
  return mk;
}

double eval_splits(const std::vector<int>& splits, const Model& g, const Hardware& hw, Strategy strategy,
                   const CostTable& table) {
  std::vector<Block> blocks;
  Costs costs;
  build_blocks(splits_to_partition(splits, g.num_layers()), table, &blocks, &costs);
  if (strategy == Strategy::CAPACITY_RECOMPUTE) {
    Flags fl = greedy_recompute(blocks, costs, g, hw);
    double cost = eval_one(flagged(blocks, fl), g, hw, strategy, costs);
    if (cost < kPenaltyCapacity) return cost;
    return std::min(cost, eval_one(blocks, g, hw, strategy, costs));
  }
  return eval_one(blocks, g, hw, strategy, costs);
}

// planner.py:845-883
Partition polish_splits(const std::vector<std::vector<int>>& seeds, const Model& g, const Hardware& hw,
                        Strategy strategy, int bound, const CostTable& table, int max_rounds = 40) {
  int num = g.num_layers();
  std::optional<std::vector<int>> best;
  double best_cost = kInf;
  for (auto& seed : seeds) {
    double cost = eval_splits(seed, g, hw, strategy, table);
    if (cost < best_cost) {
      best = seed;
      best_cost = cost;
    }
  }
  if (!best) {
    best = std::vector<int>{};
    best_cost = eval_splits({}, g, hw, strategy, table);
  }
  for (int round = 0; round < max_rounds; ++round) {
    bool improved = false;
    std::set<int> current(best->begin(), best->end());
    std::vector<std::set<int>> moves;
    for (int s : current) {
      std::set<int> drop = current;
      drop.erase(s);
      moves.push_back(drop);
      if (s - 1 >= 1 && !current.count(s - 1)) {
        std::set<int> m = drop;
        m.insert(s - 1);
        moves.push_back(m);
      }
      if (s + 1 <= num - 1 && !current.count(s + 1)) {
        std::set<int> m = drop;
        m.insert(s + 1);
        moves.push_back(m);
      }
    }
    if ((int)current.size() + 2 <= bound)
      for (int s = 1; s < num; ++s)
        if (!current.count(s)) {
          std::set<int> m = current;
          m.insert(s);
          moves.push_back(m);
        }
    for (auto& cand : moves) {
      if ((int)cand.size() + 1 > bound) continue;
      std::vector<int> ct(cand.begin(), cand.end());
      double cost = eval_splits(ct, g, hw, strategy, table);
      if (cost < best_cost - kEps) {
        best = ct;
        best_cost = cost;
        improved = true;
        break;
      }
    }
    if (!improved) break;
  }
  if (best_cost >= kPenaltyCapacity) throw InfeasibleModel("no feasible partition found by the dp solver");
  return splits_to_partition(*best, num);
}

// planner.py:764-802
Partition dp_partition(const Model& g, const Hardware& hw, Strategy strategy, int max_blocks, const CostTable& t) {
  int num = g.num_layers();
  int bound = max_blocks <= 0 ? num : std::min(max_blocks, num);
  auto range_cost = [&](int lo, int hi) {
    double fw = (t.eff[hi] - t.eff[lo - 1]) / t.rate;
    double swap = (t.bytes[hi] - t.bytes[lo - 1]) / t.swap_rate;
    if (hw.duplex) return std::max(fw, swap) + std::max(fw * t.mult, swap);
    return std::max(fw * (1.0 + t.mult), 2.0 * swap);
  };
  std::vector<std::vector<double>> dp(num + 1, std::vector<double>(bound + 1, kInf));
  std::vector<std::vector<int>> parent(num + 1, std::vector<int>(bound + 1, 0));
  dp[0][0] = 0.0;
  for (int i = 1; i <= num; ++i)
    for (int k = 1; k <= std::min(i, bound); ++k)
      for (int j = k - 1; j < i; ++j) {
        if (dp[j][k - 1] == kInf) continue;
        double cand = dp[j][k - 1] + range_cost(j + 1, i);
        if (cand < dp[i][k]) {
          dp[i][k] = cand;
          parent[i][k] = j;
        }
      }
  int best_k = 1;
  for (int k = 2; k <= bound; ++k)
    if (dp[num][k] < dp[num][best_k]) best_k = k;
  std::vector<int> splits;
  int i = num, k = best_k;
  while (k > 1) {
    int j = parent[i][k];
    splits.push_back(j);
    i = j;
    --k;
  }
  std::reverse(splits.begin(), splits.end());
  std::vector<std::vector<int>> seeds{splits};
  if (num <= bound) {
    std::vector<int> all;
    for (int s = 1; s < num; ++s) all.push_back(s);
    seeds.push_back(all);
  }
  seeds.push_back({});
  return polish_splits(seeds, g, hw, strategy, bound, t);
}

std::vector<Partition> enumerate_partitions(int num, int max_blocks) {
  if (num < 1) throw PlannerMisuse("need at least one layer");
  int bound = max_blocks <= 0 ? num : std::min(max_blocks, num);
  std::vector<Partition> out;
  std::vector<int> cuts;
  for (int s = 1; s < num; ++s) cuts.push_back(s);
  for (int k = 1; k <= bound; ++k)
    for_combinations(cuts, k - 1, [&](const std::vector<int>& splits) {
      out.push_back(splits_to_partition(splits, num));
    });
  return out;
}

struct ExhaustiveBest {
  Candidate cand;
  std::tuple<double, double, int, std::vector<int>, size_t, std::vector<int>> key;
  bool have = false;
};

// planner.py:645-741
Candidate search_exhaustive(const Model& g, const Hardware& hw, Strategy strategy, int max_blocks, int layer_bound) {
  int num = g.num_layers();
  if (num > layer_bound)
    throw PlannerMisuse("exhaustive mode is limited to " + std::to_string(layer_bound) + " layers (model has " +
                        std::to_string(num) + "); use the dp solver");
  CostTable table(g, hw);
  double base_compute = (table.eff[num] / table.rate) * (1.0 + table.mult);
  ExhaustiveBest best;
  std::string first_reason;
  auto consider = [&](const std::vector<Block>& blocks, const Costs& costs, const Flags& fl, int nb,
                      const std::vector<int>& splits) {
    Candidate r = evaluate_blocks(flagged(blocks, fl), g, hw, strategy, costs);
    if (!r.feasible) {
      if (first_reason.empty()) first_reason = r.reason;
      return;
    }
    auto key = std::make_tuple(r.makespan, r.stall, nb, splits, fl.size(), flags_key(fl, nb));
    if (!best.have || key < best.key) {
      best.key = key;
      best.cand = std::move(r);
      best.have = true;
    }
  };
  auto splits_of = [](const Partition& p) {
    std::vector<int> s;
    for (size_t i = 0; i + 1 < p.size(); ++i) s.push_back(p[i].second);
    return s;
  };
  try {
    Partition seed = dp_partition(g, hw, strategy, max_blocks, table);
    std::vector<Block> blocks;
    Costs costs;
    build_blocks(seed, table, &blocks, &costs);
    Flags seed_flags;
    if (strategy == Strategy::CAPACITY_RECOMPUTE) seed_flags = greedy_recompute(blocks, costs, g, hw);
    consider(blocks, costs, seed_flags, (int)blocks.size(), splits_of(seed));
  } catch (const InfeasibleModel&) {
  }
  double xfer_scale = hw.duplex ? 1.0 : 2.0;
  for (auto& partition : enumerate_partitions(num, max_blocks)) {
    std::vector<Block> blocks;
    Costs costs;
    build_blocks(partition, table, &blocks, &costs);
    int nb = (int)blocks.size();
    auto splits = splits_of(partition);
    double bestm = best.have ? best.cand.makespan : kInf;
    if (strategy == Strategy::EAGER) {
      std::vector<int> all;
      for (int i = 1; i <= nb; ++i) all.push_back(i);
      double lb = std::max(base_compute, transfer_lower_bound(costs, all, hw.duplex));
      if (!best.have || lb <= bestm + 1e-12) consider(blocks, costs, {}, nb, splits);
      continue;
    }
    if (strategy == Strategy::CAPACITY) {
      int k_ret = retained_start(blocks, costs, hw.capacity_bytes);
      std::vector<int> sw;
      for (int i = 1; i < k_ret; ++i) sw.push_back(i);
      double lb = std::max(base_compute, transfer_lower_bound(costs, sw, hw.duplex));
      if (!best.have || lb <= bestm + 1e-12) consider(blocks, costs, {}, nb, splits);
      continue;
    }
    int k_ret;
    Flags forced;
    std::vector<int> free;
    recompute_candidates(blocks, costs, g, hw, &k_ret, &forced, &free);
    if ((int)free.size() > kOpt2ExhaustiveBound) {
      consider(blocks, costs, greedy_recompute(blocks, costs, g, hw), nb, splits);
      continue;
    }
    // Python: base_compute + sum(...) -- the sum first, then one addition
    PySum fsum;
    for (int f : forced)
      if (f != nb) fsum.add(costs.at(f).fwd_seconds);
    double compute0 = base_compute + fsum.value();
    PySum tsum;
    for (int i = 1; i < k_ret; ++i)
      if (!forced.count(i)) tsum.add(costs.at(i).swap_seconds);
    double transfer0 = tsum.value() * xfer_scale;
    PySum msum;
    for (int f : free) msum.add(costs.at(f).swap_seconds);
    double max_saving = msum.value() * xfer_scale;
    if (best.have && std::max(compute0, transfer0 - max_saving) > best.cand.makespan + 1e-12) continue;
    std::vector<int> forced_sorted(forced.begin(), forced.end());
    double capacity = hw.capacity_bytes;
    for (int r = 0; r <= (int)free.size(); ++r)
      for_combinations(free, r, [&](const std::vector<int>& combo) {
        PySum cs, ts;
        for (int c : combo)
          if (c != nb) cs.add(costs.at(c).fwd_seconds);
        for (int c : combo) ts.add(costs.at(c).swap_seconds);
        double lb_compute = compute0 + cs.value();
        double lb_transfer = transfer0 - ts.value() * xfer_scale;
        if (best.have && std::max(lb_compute, lb_transfer) > best.cand.makespan + 1e-12) return;
        std::set<int> u(combo.begin(), combo.end());
        u.insert(forced_sorted.begin(), forced_sorted.end());
        std::vector<int> us(u.begin(), u.end());
        if (run_bytes_exceed(us, costs, nb, capacity)) return;
        Flags fl = forced;
        fl.insert(combo.begin(), combo.end());
        consider(blocks, costs, fl, nb, splits);
      });
  }
  if (!best.have) {
    Partition finest;
    for (int i = 1; i <= num; ++i) finest.emplace_back(i, i);
    std::vector<Block> blocks;
    Costs costs;
    build_blocks(finest, table, &blocks, &costs);
    Candidate r = evaluate_blocks(blocks, g, hw, strategy, costs);
    std::string why = !r.reason.empty() ? r.reason
                      : !first_reason.empty() ? first_reason
                                              : "no feasible partition under the memory capacity";
    throw InfeasibleModel(why);
  }
  return best.cand;
}

// planner.py:328-335
Plan finalize_plan(Plan plan, const Model& g, const Hardware& hw) {
  auto v = validate_plan(plan, g, hw);
  if (!v.empty()) throw PlannerMisuse("generated plan failed validation: " + v[0]);
  SimResult sr = simulate(plan, g, hw, true);
  if (sr.deadlock) throw InfeasibleModel("simulation deadlock");
  plan.predicted_makespan = sr.makespan;
  long long th = find_theta(plan, g, hw);
  plan.has_theta = th >= 0;
  plan.theta = th;
  return plan;
}

}  // namespace

Plan plan_model(const Model& g, const Hardware& hw, Strategy strategy, const std::string& solver_in, int max_blocks,
                int layer_bound) {
  std::string solver = solver_in;
  if (solver == "auto") solver = g.num_layers() <= kAutoExhaustiveLayers ? "exhaustive" : "dp";
  if (solver == "exhaustive") {
    Candidate best = search_exhaustive(g, hw, strategy, max_blocks, layer_bound);
    return finalize_plan(best.plan, g, hw);
  }
  if (solver != "dp") throw PlannerMisuse("unknown solver '" + solver + "'");
  CostTable table(g, hw);
  Partition part = dp_partition(g, hw, strategy, max_blocks, table);
  std::vector<Block> blocks;
  Costs costs;
  build_blocks(part, table, &blocks, &costs);
  if (strategy == Strategy::CAPACITY_RECOMPUTE) blocks = solve_opt2(blocks, g, hw, costs);
  Plan plan = generate_schedule(blocks, g, hw, strategy, costs);
  auto v = validate_plan(plan, g, hw);
  if (!v.empty()) throw InfeasibleModel(v[0]);
  return finalize_plan(plan, g, hw);
}

}  // namespace krt
