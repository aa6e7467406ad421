#include "engine.hpp"

#include <algorithm>
#include <cmath>
#include <set>
#include <stdexcept>

namespace krt {
namespace {
constexpr double kEps = 1e-12;           // simulator.py:28
constexpr double kDistEps = 1e-9;        // distsim.py:31
const char* kResNames[] = {"compute", "xfer_in", "xfer_out", "xfer", "network", "host"};

// queue priority inside a stage (simulator.py:239-250)
int queue_rank(Action a) {
  switch (a) {
    case Action::SWAP_IN: return 1;
    case Action::SWAP_OUT: return 2;
    default: return 0;
  }
}
bool is_compute(Action a) { return a == Action::FW || a == Action::BW || a == Action::RECOMPUTE_FW; }
}  // namespace

const char* res_name(int r) { return kResNames[r]; }

std::string EngineOp::tag() const {
  // action [block b] [group g] [iter i]  (only keys present in the tag dict)
  std::string s = action_name(action);
  bool has_block = true;   // every tag the reference builds carries "block"
  bool has_group = action == Action::WEIGHT_IN || action == Action::GRAD_OUT ||
                   action == Action::EXCHANGE || action == Action::HOST_UPDATE;
  if (has_block) s += " block " + std::to_string(block);
  if (has_group) s += " group " + std::to_string(group);
  if (iteration > 0) s += " iter " + std::to_string(iteration);
  return s;
}

EngineResult run_engine(const std::vector<EngineOp>& ops, const std::vector<int>& resources,
                        double capacity, bool enforce) {
  EngineResult out;
  size_t n = ops.size();
  std::vector<std::vector<int>> queues(R_COUNT);
  for (size_t i = 0; i < n; ++i) queues[ops[i].res].push_back((int)i);
  std::vector<size_t> heads(R_COUNT, 0);
  std::vector<int> run_idx(R_COUNT, -1);
  std::vector<double> run_end(R_COUNT, 0.0), last_end(R_COUNT, 0.0);
  std::vector<char> started(n, 0), done(n, 0);
  std::vector<EngineEvent> ev(n);
  std::vector<char> has_ev(n, 0);
  double used = 0, peak = 0, now = 0;
  size_t remaining = n;

  auto startable = [&](int idx) {
    const EngineOp& op = ops[idx];
    if (!op.missing.empty()) return false;
    for (int d : op.deps)
      if (!done[d]) return false;
    if (op.gate >= 0 && !started[op.gate]) return false;
    if (enforce && op.alloc > 0 && used + op.alloc > capacity + kEps) return false;
    return true;
  };

  while (remaining > 0) {
    bool progressed = true;
    while (progressed) {
      progressed = false;
      for (int r : resources) {
        if (run_idx[r] >= 0) continue;
        if (heads[r] >= queues[r].size()) continue;
        int idx = queues[r][heads[r]];
        if (!startable(idx)) continue;
        const EngineOp& op = ops[idx];
        used += op.alloc;
        peak = std::max(peak, used);
        started[idx] = 1;
        ev[idx] = EngineEvent{idx, r, now, now + op.duration, std::max(0.0, now - last_end[r])};
        has_ev[idx] = 1;
        out.start_order.push_back(idx);
        run_idx[r] = idx;
        run_end[r] = now + op.duration;
        heads[r]++;
        progressed = true;
      }
    }
    bool any = false;
    double next = 0;
    for (int r : resources)
      if (run_idx[r] >= 0) {
        if (!any || run_end[r] < next) next = run_end[r];
        any = true;
      }
    if (!any) {
      // _blocked_reasons (simulator.py:138-156)
      out.deadlock = true;
      for (int r : resources) {
        if (heads[r] >= queues[r].size()) continue;
        int idx = queues[r][heads[r]];
        const EngineOp& op = ops[idx];
        std::vector<std::string> why;
        if (!op.missing.empty()) why.push_back(op.missing);
        std::string unmet;
        for (int d : op.deps)
          if (!done[d]) unmet += (unmet.empty() ? "" : ", ") + ops[d].tag();
        if (!unmet.empty()) why.push_back("waiting on " + unmet);
        if (op.gate >= 0 && !started[op.gate]) why.push_back("gated behind " + ops[op.gate].tag());
        if (enforce && op.alloc > 0 && used + op.alloc > capacity + kEps)
          why.push_back("needs " + py_g(op.alloc) + " B but only " + py_g(capacity - used) + " B free");
        std::string j;
        for (size_t k = 0; k < why.size(); ++k) j += (k ? "; " : "") + why[k];
        out.blocked.push_back(op.tag() + ": " + (why.empty() ? "unknown" : j));
      }
      break;
    }
    now = next;
    for (int r : resources) {
      if (run_idx[r] < 0) continue;
      if (run_end[r] <= now + kEps) {
        int idx = run_idx[r];
        run_idx[r] = -1;
        done[idx] = 1;
        used -= ops[idx].free_end;
        last_end[r] = run_end[r];
        remaining--;
      }
    }
  }
  for (size_t i = 0; i < n; ++i)
    if (has_ev[i]) out.events.push_back(ev[i]);
  double mk = 0;
  for (auto& e : out.events) mk = std::max(mk, e.t_end);
  out.makespan = mk;
  out.peak = peak;
  return out;
}

std::map<int, BlockCost> plan_costs(const Plan& p, const Model& g, const Hardware& hw) {
  std::map<int, BlockCost> c;
  for (auto& b : p.blocks) c[b.id] = block_cost(b.id, b.first_layer, b.last_layer, g, hw);
  return c;
}

std::vector<int> base_resources(const Hardware& hw) {
  if (hw.duplex) return {R_COMPUTE, R_XFER_IN, R_XFER_OUT};
  return {R_COMPUTE, R_XFER};
}

std::vector<EngineOp> build_engine_ops(const Plan& p, const Model& g, const Hardware& hw,
                                       const std::map<int, BlockCost>& costs) {
  std::map<int, bool> recompute_flag;
  for (auto& b : p.blocks) recompute_flag[b.id] = b.recompute;
  auto skip = skip_requirement_map(p.blocks, g);
  // flatten in stage order, stable-sorted by (priority, block) inside a stage
  std::vector<std::pair<int, PlanOp>> flat;
  for (size_t s = 0; s < p.stages.size(); ++s) {
    std::vector<PlanOp> ops = p.stages[s].ops;
    std::stable_sort(ops.begin(), ops.end(), [](const PlanOp& a, const PlanOp& b) {
      int ra = queue_rank(a.action), rb = queue_rank(b.action);
      return ra != rb ? ra < rb : a.block < b.block;
    });
    for (auto& op : ops) flat.emplace_back((int)s, op);
  }
  std::map<int, int> producer, fw_done, swap_out_done;
  std::vector<std::pair<int, int>> last_compute;  // (stage, op idx)
  std::vector<EngineOp> out;
  auto cost_of = [&](int b) -> const BlockCost& {
    auto it = costs.find(b);
    if (it == costs.end()) throw std::runtime_error("op references unknown block " + std::to_string(b));
    return it->second;
  };
  for (auto& [stage_idx, op] : flat) {
    int b = op.block;
    const BlockCost& cost = cost_of(b);
    EngineOp e;
    e.action = op.action;
    e.block = b;
    e.stage = stage_idx;
    e.has_stage_tag = true;
    if (op.action == Action::FW) {
      e.res = R_COMPUTE;
      e.duration = cost.fwd_seconds;
      e.alloc = cost.bytes;
      if (b >= 2) {
        auto it = producer.find(b - 1);
        if (it != producer.end()) e.deps.push_back(it->second);
        else e.missing = "block " + std::to_string(b) + " forward before block " + std::to_string(b - 1) + " residency";
        auto rf = recompute_flag.find(b - 1);
        if (rf != recompute_flag.end() && rf->second) e.free_end = cost_of(b - 1).bytes;
      }
    } else if (op.action == Action::RECOMPUTE_FW) {
      e.res = R_COMPUTE;
      e.duration = cost.fwd_seconds;
      e.alloc = cost.bytes;
      std::vector<int> needed;
      if (b >= 2) needed.push_back(b - 1);
      auto it = skip.find(b);
      if (it != skip.end()) needed.insert(needed.end(), it->second.begin(), it->second.end());
      for (int q : needed) {
        auto pr = producer.find(q);
        if (pr != producer.end()) e.deps.push_back(pr->second);
        else e.missing = "block " + std::to_string(b) + " recompute before block " + std::to_string(q) + " residency";
      }
    } else if (op.action == Action::BW) {
      e.res = R_COMPUTE;
      e.duration = cost.bwd_seconds;
      e.free_end = cost.bytes;
      std::vector<int> needed{b};
      auto it = skip.find(b);
      if (it != skip.end()) needed.insert(needed.end(), it->second.begin(), it->second.end());
      for (int q : needed) {
        auto pr = producer.find(q);
        if (pr != producer.end()) e.deps.push_back(pr->second);
        else e.missing = "block " + std::to_string(q) + " backward before residency";
      }
    } else if (op.action == Action::SWAP_OUT) {
      e.res = hw.duplex ? R_XFER_OUT : R_XFER;
      e.duration = cost.swap_seconds;
      e.free_end = cost.bytes;
      auto it = fw_done.find(b);
      if (it != fw_done.end()) e.deps.push_back(it->second);
      else e.missing = "block " + std::to_string(b) + " swap-out before its forward";
    } else {  // SWAP_IN
      e.res = hw.duplex ? R_XFER_IN : R_XFER;
      e.duration = cost.swap_seconds;
      e.alloc = cost.bytes;
      auto it = swap_out_done.find(b);
      if (it != swap_out_done.end()) e.deps.push_back(it->second);
      else e.missing = "block " + std::to_string(b) + " swap-in before its swap-out";
    }
    if (e.res != R_COMPUTE) {
      for (auto it = last_compute.rbegin(); it != last_compute.rend(); ++it)
        if (it->first < stage_idx) {
          e.gate = it->second;
          break;
        }
    }
    int idx = (int)out.size();
    out.push_back(e);
    if (op.action == Action::FW || op.action == Action::RECOMPUTE_FW || op.action == Action::SWAP_IN)
      producer[b] = idx;
    if (op.action == Action::FW) {
      fw_done[b] = idx;
      auto rf = recompute_flag.find(b - 1);
      if (b >= 2 && rf != recompute_flag.end() && rf->second) producer.erase(b - 1);
    }
    if (op.action == Action::SWAP_OUT) {
      swap_out_done[b] = idx;
      producer.erase(b);
    }
    if (e.res == R_COMPUTE) last_compute.emplace_back(stage_idx, idx);
  }
  return out;
}

std::string SimResult::csv() const {
  std::string s = "t_start,t_end,resource,block,action,stall_before\n";
  for (auto& e : events) {
    const EngineOp& op = ops[e.op];
    s += py_9g(e.t_start) + "," + py_9g(e.t_end) + "," + res_name(e.res) + "," +
         std::to_string(op.block) + "," + action_name(op.action) + "," + py_9g(e.stall_before) + "\n";
  }
  return s;
}

SimResult simulate(const Plan& p, const Model& g, const Hardware& hw, bool enforce) {
  SimResult sr;
  auto costs = plan_costs(p, g, hw);
  sr.ops = build_engine_ops(p, g, hw, costs);
  EngineResult er = run_engine(sr.ops, base_resources(hw), hw.capacity_bytes, enforce);
  if (er.deadlock) {
    sr.deadlock = true;
    sr.blocked = er.blocked;
    return sr;
  }
  sr.events = er.events;
  std::stable_sort(sr.events.begin(), sr.events.end(), [](const EngineEvent& a, const EngineEvent& b) {
    if (a.t_start != b.t_start) return a.t_start < b.t_start;
    return std::string(res_name(a.res)) < std::string(res_name(b.res));
  });
  PySum busy_sum;
  for (auto& e : sr.events)
    if (is_compute(sr.ops[e.op].action)) busy_sum.add(e.t_end - e.t_start);
  double busy = busy_sum.value();
  sr.makespan = er.makespan;
  sr.total_stall = er.makespan - busy;
  sr.peak = er.peak;
  return sr;
}

bool plan_metrics(const Plan& p, const Model& g, const Hardware& hw, const std::map<int, BlockCost>& costs,
                  double* makespan, double* stall, double* peak) {
  auto ops = build_engine_ops(p, g, hw, costs);
  EngineResult er = run_engine(ops, base_resources(hw), hw.capacity_bytes, true);
  if (er.deadlock) return false;
  PySum busy;
  for (auto& e : er.events)   // raw events in op order (simulator.py:359-360)
    if (e.res == R_COMPUTE) busy.add(e.t_end - e.t_start);
  *makespan = er.makespan;
  *stall = er.makespan - busy.value();
  *peak = er.peak;
  return true;
}

std::vector<std::string> residency_memory_walk(const Plan& p, const Model& g, const Hardware& hw,
                                               double* peak_out) {
  auto skip = skip_requirement_map(p.blocks, g);
  std::map<int, double> bytes_of;
  std::map<int, bool> rflag;
  for (auto& b : p.blocks) {
    bytes_of[b.id] = b.swap_bytes;
    rflag[b.id] = b.recompute;
  }
  auto bytes = [&](int b) {
    auto it = bytes_of.find(b);
    if (it == bytes_of.end()) throw std::runtime_error("op references unknown block " + std::to_string(b));
    return it->second;
  };
  auto flag = [&](int b) {
    auto it = rflag.find(b);
    return it != rflag.end() && it->second;
  };
  double cap = hw.capacity_bytes, peak = 0.0, resident_bytes = 0.0;
  std::vector<std::string> v;
  std::set<int> resident, on_host, fw_done;
  bool violated = false;
  for (auto& s : p.stages) {
    double demand = resident_bytes;
    for (auto& op : s.ops) {
      int b = op.block;
      std::string B = std::to_string(b);
      switch (op.action) {
        case Action::FW:
          if (b >= 2 && !resident.count(b - 1))
            v.push_back("block " + B + " forward before block " + std::to_string(b - 1) + " residency");
          demand += bytes(b);
          break;
        case Action::RECOMPUTE_FW: {
          if (!flag(b)) v.push_back("block " + B + " recomputed but not flagged recompute");
          std::vector<int> need;
          if (b >= 2) need.push_back(b - 1);
          auto it = skip.find(b);
          if (it != skip.end()) need.insert(need.end(), it->second.begin(), it->second.end());
          for (int q : need)
            if (!resident.count(q))
              v.push_back("block " + B + " recompute before block " + std::to_string(q) + " residency");
          demand += bytes(b);
          break;
        }
        case Action::BW: {
          if (!resident.count(b)) v.push_back("block " + B + " backward before residency");
          auto it = skip.find(b);
          if (it != skip.end())
            for (int q : it->second)
              if (!resident.count(q))
                v.push_back("block " + B + " backward before skip-source block " + std::to_string(q) + " residency");
          break;
        }
        case Action::SWAP_OUT:
          if (!fw_done.count(b)) v.push_back("block " + B + " swap-out before its forward");
          if (!resident.count(b)) v.push_back("block " + B + " swap-out while not resident");
          break;
        case Action::SWAP_IN:
          if (!on_host.count(b)) v.push_back("block " + B + " swap-in before its swap-out");
          if (resident.count(b)) v.push_back("block " + B + " swap-in while already resident");
          demand += bytes(b);
          break;
        default:
          break;
      }
    }
    peak = std::max(peak, demand);
    if (demand > cap + kEps && !violated) {
      v.push_back("stage " + std::to_string(s.id) + ": demands " + py_g(demand) +
                  " B, exceeding capacity " + py_g(cap) + " B");
      violated = true;
    }
    for (auto& op : s.ops) {
      int b = op.block;
      switch (op.action) {
        case Action::FW:
          if (!resident.count(b)) {
            resident.insert(b);
            resident_bytes += bytes(b);
          }
          fw_done.insert(b);
          if (b >= 2 && flag(b - 1) && resident.count(b - 1)) {
            resident.erase(b - 1);
            resident_bytes -= bytes(b - 1);
          }
          break;
        case Action::RECOMPUTE_FW:
        case Action::SWAP_IN:
          if (!resident.count(b)) {
            resident.insert(b);
            resident_bytes += bytes(b);
          }
          on_host.erase(b);
          break;
        case Action::SWAP_OUT:
          if (resident.count(b)) {
            resident.erase(b);
            resident_bytes -= bytes(b);
          }
          on_host.insert(b);
          break;
        case Action::BW:
          if (resident.count(b)) {
            resident.erase(b);
            resident_bytes -= bytes(b);
          }
          break;
        default:
          break;
      }
    }
  }
  if (peak_out) *peak_out = peak;
  return v;
}

std::vector<std::string> validate_plan(const Plan& p, const Model& g, const Hardware& hw) {
  std::vector<std::string> v;
  int nb = (int)p.blocks.size();
  std::map<int, int> claimed;
  for (auto& b : p.blocks) {
    if (b.first_layer > b.last_layer) v.push_back("block " + std::to_string(b.id) + " has empty layer range");
    for (int l = b.first_layer; l <= b.last_layer; ++l) {
      auto it = claimed.find(l);
      if (it != claimed.end())
        v.push_back("layer " + std::to_string(l) + " appears in blocks " + std::to_string(it->second) +
                    " and " + std::to_string(b.id));
      claimed[l] = b.id;
    }
  }
  for (int l = 1; l <= g.num_layers(); ++l)
    if (!claimed.count(l)) v.push_back("layer " + std::to_string(l) + " not covered by any block");
  bool ids_ok = true;
  for (int i = 0; i < nb; ++i) ids_ok &= p.blocks[i].id == i + 1;
  if (!ids_ok) v.push_back("block ids are not the contiguous sequence 1..n");
  else
    for (int i = 1; i < nb; ++i)
      if (p.blocks[i].first_layer != p.blocks[i - 1].last_layer + 1)
        v.push_back("blocks " + std::to_string(p.blocks[i - 1].id) + " and " + std::to_string(p.blocks[i].id) +
                    " are not contiguous");
  for (auto& b : p.blocks)
    if (b.recompute && b.checkpoint) v.push_back("block " + std::to_string(b.id) + " is both recompute and checkpoint");
  std::vector<int> fw, bw;
  for (auto& s : p.stages)
    for (auto& op : s.ops) {
      if (op.action == Action::FW) fw.push_back(op.block);
      if (op.action == Action::BW) bw.push_back(op.block);
    }
  bool fw_ok = (int)fw.size() == nb, bw_ok = (int)bw.size() == nb;
  for (int i = 0; fw_ok && i < nb; ++i) fw_ok = fw[i] == i + 1;
  for (int i = 0; bw_ok && i < nb; ++i) bw_ok = bw[i] == nb - i;
  if (!fw_ok) v.push_back("forward ops must run each block exactly once in ascending order");
  if (!bw_ok) v.push_back("backward ops must run each block exactly once in descending order");
  for (auto act : {Action::SWAP_IN, Action::SWAP_OUT}) {
    const char* label = act == Action::SWAP_IN ? "swap-in" : "swap-out";
    std::set<int> seen;
    for (auto& s : p.stages)
      for (auto& op : s.ops)
        if (op.action == act) {
          if (seen.count(op.block)) v.push_back("block " + std::to_string(op.block) + " has more than one " + label);
          seen.insert(op.block);
        }
  }
  auto skip = skip_requirement_map(p.blocks, g);
  for (auto& s : p.stages) {
    std::set<int> produced, fw_here, out_here;
    for (auto& op : s.ops) {
      if (op.action == Action::FW || op.action == Action::RECOMPUTE_FW || op.action == Action::SWAP_IN)
        produced.insert(op.block);
      if (op.action == Action::FW || op.action == Action::RECOMPUTE_FW) fw_here.insert(op.block);
      if (op.action == Action::SWAP_OUT) out_here.insert(op.block);
    }
    std::string S = "stage " + std::to_string(s.id) + ": ";
    for (auto& op : s.ops) {
      std::vector<int> needs;
      auto it = skip.find(op.block);
      if (op.action == Action::FW && op.block >= 2) needs = {op.block - 1};
      else if (op.action == Action::RECOMPUTE_FW) {
        if (op.block >= 2) needs.push_back(op.block - 1);
        if (it != skip.end()) needs.insert(needs.end(), it->second.begin(), it->second.end());
      } else if (op.action == Action::BW) {
        needs.push_back(op.block);
        if (it != skip.end()) needs.insert(needs.end(), it->second.begin(), it->second.end());
      } else if (op.action == Action::SWAP_OUT && fw_here.count(op.block))
        v.push_back(S + "swap-out of block " + std::to_string(op.block) + " overlaps its forward");
      else if (op.action == Action::SWAP_IN && out_here.count(op.block))
        v.push_back(S + "swap-in of block " + std::to_string(op.block) + " overlaps its swap-out");
      for (int q : needs)
        if (produced.count(q)) {
          v.push_back(S + "op on block " + std::to_string(op.block) + " reads block " + std::to_string(q) +
                      " produced in the same stage");
          break;
        }
    }
  }
  auto w = residency_memory_walk(p, g, hw, nullptr);
  v.insert(v.end(), w.begin(), w.end());
  return v;
}

// ---------------------------------------------------------------------------
double allreduce_time(double bytes, const DistConfig& cfg) {
  if (bytes < 0) throw std::runtime_error("bytes must be non-negative");
  int p = cfg.workers;
  if (p == 1) return 0.0;
  if (cfg.ring) return 2.0 * (p - 1) / p * bytes / cfg.net_bw + 2.0 * (p - 1) * cfg.net_latency;
  return (p - 1) * bytes / cfg.net_bw + cfg.net_latency;
}

std::vector<std::vector<int>> assign_groups(int nb, int groups) {
  int count = groups == 0 ? nb : std::min(groups, nb);
  std::vector<std::vector<int>> out;
  int base = nb / count, extra = nb % count, start = 1;
  for (int gi = 0; gi < count; ++gi) {
    int size = base + (gi < extra ? 1 : 0);
    std::vector<int> m;
    for (int b = start; b < start + size; ++b) m.push_back(b);
    out.push_back(m);
    start += size;
  }
  return out;
}

namespace {
// The executor's P >= 2 pipeline (runtime.cu build_ops, dp_ branch) as engine
// ops: exchange (reduce-scatter) precedes a shard-sized grad_out, the host
// updates 1/P of the group, and the weight return is a shard H2D plus an
// all-gather on the network resource.  Gradients live in the executor's
// gradient region, outside the arena, so a backward frees its block's whole
// ledger bytes (the reference holds grad_bytes until grad_out, distsim.py:195-202).
std::vector<EngineOp> build_dist_ops_device(const Plan& p, const Model& g, const Hardware& hw,
                                            const DistConfig& cfg, int iterations,
                                            const std::map<int, BlockCost>& costs) {
  double swap_rate = hw.swap_throughput();
  const double P = cfg.workers;
  auto groups = assign_groups((int)p.blocks.size(), cfg.groups);
  std::map<int, int> group_of;
  for (size_t gi = 0; gi < groups.size(); ++gi)
    for (int b : groups[gi]) group_of[b] = (int)gi + 1;
  std::map<int, double> group_bytes, group_wt, group_wtb;
  for (size_t gi = 0; gi < groups.size(); ++gi) {
    PySum gb, gw, gwb;
    for (int b : groups[gi]) {
      gb.add(costs.at(b).grad_bytes);
      gw.add(costs.at(b).weight_elems);
      gwb.add(costs.at(b).wt_bytes);
    }
    group_bytes[(int)gi + 1] = gb.value();
    group_wt[(int)gi + 1] = gw.value();
    group_wtb[(int)gi + 1] = gwb.value();
  }
  auto base = build_engine_ops(p, g, hw, costs);
  int in_res = hw.duplex ? R_XFER_IN : R_XFER, out_res = hw.duplex ? R_XFER_OUT : R_XFER;
  std::vector<EngineOp> all;
  std::map<int, int> update_prev;
  for (int it = 1; it <= iterations; ++it) {
    int offset = (int)all.size();
    std::map<int, int> gathered;  // group -> all-gather op
    if (it >= 2)
      for (int gi = 1; gi <= (int)groups.size(); ++gi) {
        EngineOp w;
        w.action = Action::WEIGHT_IN;
        w.group = gi;
        w.iteration = it;
        w.res = in_res;
        w.duration = group_wtb[gi] / P / swap_rate;
        w.deps = {update_prev.at(gi)};
        int w_idx = (int)all.size();
        all.push_back(w);
        EngineOp a;
        a.action = Action::ALL_GATHER;
        a.group = gi;
        a.iteration = it;
        a.res = R_NETWORK;
        a.duration = allreduce_time(group_wtb[gi], cfg) * 0.5;
        a.deps = {w_idx};
        gathered[gi] = (int)all.size();
        all.push_back(a);
      }
    offset = (int)all.size();  // after the weight ops (distsim.py:165 takes it before them)
    std::map<int, int> bw_done;
    for (auto& op : base) {
      EngineOp e = op;
      e.iteration = it;
      for (auto& d : e.deps) d += offset;
      if (e.gate >= 0) e.gate += offset;
      int b = op.block;
      if (op.action == Action::FW && gathered.count(group_of[b])) e.deps.push_back(gathered[group_of[b]]);
      if (op.action == Action::BW) bw_done[b] = (int)all.size();
      all.push_back(e);
    }
    std::map<int, int> update_done;
    for (int gi = (int)groups.size(); gi >= 1; --gi) {
      EngineOp x;
      x.action = Action::EXCHANGE;
      x.group = gi;
      x.iteration = it;
      x.res = R_NETWORK;
      x.duration = allreduce_time(group_bytes[gi], cfg) * 0.5;
      for (int b : groups[gi - 1]) {
        auto bd = bw_done.find(b);
        if (bd == bw_done.end()) throw std::runtime_error("no backward for block " + std::to_string(b));
        x.deps.push_back(bd->second);
      }
      int x_idx = (int)all.size();
      all.push_back(x);
      EngineOp go;
      go.action = Action::GRAD_OUT;
      go.group = gi;
      go.iteration = it;
      go.res = out_res;
      go.duration = group_bytes[gi] / P / swap_rate;
      go.deps = {x_idx};
      int go_idx = (int)all.size();
      all.push_back(go);
      EngineOp h;
      h.action = Action::HOST_UPDATE;
      h.group = gi;
      h.iteration = it;
      h.res = R_HOST;
      h.duration = group_wt[gi] / P / hw.host_update_rate;
      h.deps = {go_idx};
      update_done[gi] = (int)all.size();
      all.push_back(h);
    }
    update_prev = update_done;
  }
  return all;
}
}  // namespace

std::vector<EngineOp> build_dist_ops(const Plan& p, const Model& g, const Hardware& hw,
                                     const DistConfig& cfg, int iterations,
                                     const std::map<int, BlockCost>& costs) {
  if (cfg.device_exchange && cfg.workers >= 2) return build_dist_ops_device(p, g, hw, cfg, iterations, costs);
  double swap_rate = hw.swap_throughput();
  std::set<int> host_blocks;
  if (cfg.workers >= 2) for (auto& b : p.blocks) host_blocks.insert(b.id);
  else for (int b : p.swapped_blocks()) host_blocks.insert(b);
  auto groups = assign_groups((int)p.blocks.size(), cfg.groups);
  std::map<int, int> group_of;
  for (size_t gi = 0; gi < groups.size(); ++gi)
    for (int b : groups[gi]) group_of[b] = (int)gi + 1;
  std::map<int, double> group_bytes, group_wt;
  for (size_t gi = 0; gi < groups.size(); ++gi) {
    PySum gb, gw;  // distsim.py:153-156 sum() in member order
    for (int b : groups[gi])
      if (host_blocks.count(b)) {
        gb.add(costs.at(b).grad_bytes);
        gw.add(costs.at(b).weight_elems);
      }
    group_bytes[(int)gi + 1] = gb.value();
    group_wt[(int)gi + 1] = gw.value();
  }
  auto base = build_engine_ops(p, g, hw, costs);
  int in_res = hw.duplex ? R_XFER_IN : R_XFER, out_res = hw.duplex ? R_XFER_OUT : R_XFER;
  std::vector<EngineOp> all;
  std::map<int, int> update_prev;
  for (int it = 1; it <= iterations; ++it) {
    int offset = (int)all.size();
    std::map<int, int> weight_in_idx;
    if (it >= 2)
      for (int b : host_blocks) {
        EngineOp e;
        e.action = Action::WEIGHT_IN;
        e.block = b;
        e.group = group_of[b];
        e.iteration = it;
        e.res = in_res;
        e.duration = costs.at(b).wt_bytes / swap_rate;
        e.deps = {update_prev.at(group_of[b])};
        weight_in_idx[b] = (int)all.size();
        all.push_back(e);
      }
    if (cfg.exact_deps) offset = (int)all.size();
    std::map<int, int> bw_done;
    for (auto& op : base) {
      EngineOp e = op;
      e.iteration = it;
      for (auto& d : e.deps) d += offset;
      if (e.gate >= 0) e.gate += offset;
      int b = op.block;
      if (op.action == Action::FW && weight_in_idx.count(b)) e.deps.push_back(weight_in_idx[b]);
      if (op.action == Action::BW) {
        if (host_blocks.count(b)) {
          double held = std::min(costs.at(b).grad_bytes, e.free_end);
          e.free_end = e.free_end - held;
        }
        bw_done[b] = (int)all.size();
      }
      all.push_back(e);
    }
    std::map<int, int> grad_out_idx;
    for (auto itb = host_blocks.rbegin(); itb != host_blocks.rend(); ++itb) {
      int b = *itb;
      EngineOp e;
      e.action = Action::GRAD_OUT;
      e.block = b;
      e.group = group_of[b];
      e.iteration = it;
      e.res = out_res;
      e.duration = costs.at(b).grad_bytes / swap_rate;
      auto bd = bw_done.find(b);
      if (bd == bw_done.end()) throw std::runtime_error("no backward for block " + std::to_string(b));
      e.deps = {bd->second};
      e.free_end = std::min(costs.at(b).grad_bytes, costs.at(b).bytes);
      grad_out_idx[b] = (int)all.size();
      all.push_back(e);
    }
    std::map<int, int> update_done;
    for (int gi = (int)groups.size(); gi >= 1; --gi) {
      std::vector<int> members;
      for (int b : groups[gi - 1])
        if (host_blocks.count(b)) members.push_back(b);
      if (members.empty()) continue;
      std::vector<int> deps;
      for (int b : members) deps.push_back(grad_out_idx[b]);
      double exch = allreduce_time(group_bytes[gi], cfg);
      if (cfg.workers >= 2) {
        EngineOp e;
        e.action = Action::EXCHANGE;
        e.group = gi;
        e.iteration = it;
        e.block = -1;
        e.res = R_NETWORK;
        e.duration = exch;
        e.deps = deps;
        deps = {(int)all.size()};
        all.push_back(e);
      }
      EngineOp h;
      h.action = Action::HOST_UPDATE;
      h.group = gi;
      h.iteration = it;
      h.block = -1;
      h.res = R_HOST;
      h.duration = group_wt[gi] / hw.host_update_rate;
      h.deps = deps;
      update_done[gi] = (int)all.size();
      all.push_back(h);
    }
    update_prev = update_done;
  }
  return all;
}

ArenaPlan plan_arena(const Plan& p, const Model& g, const Hardware& hw, const std::vector<EngineOp>& base,
                     const std::map<int, size_t>& block_bytes) {
  (void)g;
  ArenaPlan ap;
  EngineResult er = run_engine(base, base_resources(hw), hw.capacity_bytes, true);
  if (er.deadlock) {
    std::string s = "simulation deadlock; blocked ops: ";
    for (size_t i = 0; i < er.blocked.size(); ++i) s += (i ? "; " : "") + er.blocked[i];
    throw std::runtime_error(s);
  }
  ap.ledger_peak = er.peak;
  ap.start_order = er.start_order;
  size_t n = base.size();
  ap.inst_of_alloc.assign(n, -1);
  ap.inst_read.assign(n, -1);
  ap.deps.assign(n, {});
  std::map<int, int> cur;
  std::map<int, bool> rflag;
  for (auto& b : p.blocks) rflag[b.id] = b.recompute;
  for (size_t i = 0; i < n; ++i) {
    const EngineOp& e = base[i];
    int b = e.block;
    if (e.action == Action::FW || e.action == Action::RECOMPUTE_FW || e.action == Action::SWAP_IN) {
      ArenaInstance in;
      in.block = b;
      auto bb = block_bytes.find(b);
      if (bb == block_bytes.end()) throw std::invalid_argument("no physical size for block " + std::to_string(b));
      in.bytes = bb->second;
      in.alloc_op = (int)i;
      ap.inst_of_alloc[i] = (int)ap.inst.size();
      cur[b] = (int)ap.inst.size();
      ap.inst.push_back(in);
      if (e.action == Action::FW && b >= 2 && rflag[b - 1]) {
        auto it = cur.find(b - 1);
        if (it != cur.end()) {  // recompute buffers discarded at the consumer's end
          ap.inst[it->second].free_op = (int)i;
          cur.erase(it);
        }
      }
    } else if (e.action == Action::SWAP_OUT || e.action == Action::BW) {
      auto it = cur.find(b);
      if (it == cur.end()) throw std::runtime_error("block " + std::to_string(b) + " not resident");
      ap.inst_read[i] = it->second;
      ap.inst[it->second].free_op = (int)i;
      cur.erase(it);
    }
  }
  // lifetimes as ranks in the (time, frees-first, start order) event sweep
  std::vector<double> ts(n, 0), te(n, 0);
  for (auto& ev : er.events) {
    ts[ev.op] = ev.t_start;
    te[ev.op] = ev.t_end;
  }
  std::vector<int> rank_of(n, 0);
  for (size_t k = 0; k < er.start_order.size(); ++k) rank_of[er.start_order[k]] = (int)k;
  struct Ev { double t; int kind; int order; int inst; };
  std::vector<Ev> evs;
  for (size_t k = 0; k < ap.inst.size(); ++k) {
    auto& in = ap.inst[k];
    evs.push_back({ts[in.alloc_op], 1, rank_of[in.alloc_op], (int)k});
    if (in.free_op >= 0) evs.push_back({te[in.free_op], 0, rank_of[in.free_op], (int)k});
  }
  std::sort(evs.begin(), evs.end(), [](const Ev& a, const Ev& b) {
    if (a.t != b.t) return a.t < b.t;
    if (a.kind != b.kind) return a.kind < b.kind;
    return a.order < b.order;
  });
  std::vector<double> lo(ap.inst.size(), 0), hi(ap.inst.size(), 1e300);
  for (size_t r = 0; r < evs.size(); ++r) {
    if (evs[r].kind == 1) lo[evs[r].inst] = (double)r;
    else hi[evs[r].inst] = (double)r;
  }
  for (size_t k = 0; k < ap.inst.size(); ++k)
    if (hi[k] <= lo[k]) hi[k] = lo[k] + 0.5;  // zero-length op: freed right after its alloc
  // first-fit over lifetimes; several orderings, keep the tightest arena
  size_t ni = ap.inst.size();
  auto place = [&](std::vector<int> order, std::vector<size_t>& offs) {
    offs.assign(ni, 0);
    size_t top = 0;
    std::vector<int> placed;
    for (int k : order) {
      std::vector<std::pair<size_t, size_t>> busy;
      for (int j : placed)
        if (lo[j] < hi[k] && lo[k] < hi[j]) busy.emplace_back(offs[j], offs[j] + ap.inst[j].bytes);
      std::sort(busy.begin(), busy.end());
      size_t off = 0;
      for (auto& bz : busy) {
        if (bz.first >= off + ap.inst[k].bytes) break;
        off = std::max(off, bz.second);
      }
      offs[k] = off;
      top = std::max(top, off + ap.inst[k].bytes);
      placed.push_back(k);
    }
    return top;
  };
  std::vector<int> base_order(ni);
  for (size_t k = 0; k < ni; ++k) base_order[k] = (int)k;
  auto by = [&](auto key) {
    std::vector<int> o = base_order;
    std::stable_sort(o.begin(), o.end(), [&](int a, int b) { return key(a) > key(b); });
    return o;
  };
  std::vector<std::vector<int>> orders = {
      by([&](int k) { return (double)ap.inst[k].bytes; }),
      by([&](int k) { return -lo[k]; }),
      by([&](int k) { return std::min(hi[k], 1e12) - lo[k]; }),
      by([&](int k) { return (double)ap.inst[k].bytes * (std::min(hi[k], 1e12) - lo[k]); }),
  };
  size_t best = (size_t)-1;
  std::vector<size_t> offs, best_offs;
  for (auto& o : orders) {
    size_t top = place(o, offs);
    if (top < best) {
      best = top;
      best_offs = offs;
    }
  }
  for (size_t k = 0; k < ni; ++k) ap.inst[k].off = best_offs[k];
  ap.arena_bytes = ni ? best : 0;
  // address reuse -> dependency on the earlier instance's freeing op
  for (size_t k = 0; k < ap.inst.size(); ++k)
    for (size_t j = 0; j < ap.inst.size(); ++j) {
      if (j == k) continue;
      auto& a = ap.inst[k];
      auto& b = ap.inst[j];
      bool addr = b.off < a.off + a.bytes && a.off < b.off + b.bytes;
      if (addr && hi[j] <= lo[k] && b.free_op >= 0) ap.deps[a.alloc_op].push_back(b.free_op);
    }
  for (auto& d : ap.deps) {
    std::sort(d.begin(), d.end());
    d.erase(std::unique(d.begin(), d.end()), d.end());
  }
  return ap;
}

DpLayout dp_layout(const std::vector<int64_t>& block_params, int groups, int world) {
  if (world < 1) throw std::invalid_argument("world must be >= 1");
  DpLayout L;
  int nb = (int)block_params.size();
  auto gs = assign_groups(nb, groups);
  L.block_off.assign(nb, 0);
  L.group_of.assign(nb, 0);
  int64_t off = 0, pad = (int64_t)world * 64;
  for (size_t gi = 0; gi < gs.size(); ++gi) {
    int64_t n = 0;
    for (int b : gs[gi]) {
      L.block_off[b - 1] = off + n;
      L.group_of[b - 1] = (int)gi + 1;
      // every block 64-element (256-byte fp32) aligned: the vectorised
      // update and reduce kernels take any block's slice
      n += (block_params[b - 1] + 63) / 64 * 64;
    }
    int64_t pn = (n + pad - 1) / pad * pad;
    L.group_lo.push_back(off);
    L.group_n.push_back(pn);
    L.shard_n.push_back(pn / world);
    off += pn;
  }
  L.total = off;
  return L;
}

DistResult simulate_distributed(const Plan& p, const Model& g, const Hardware& hw,
                                const DistConfig& cfg, int iterations) {
  if (iterations < 2) throw std::runtime_error("need at least 2 iterations to observe the steady state");
  DistResult dr;
  auto costs = plan_costs(p, g, hw);
  dr.ops = build_dist_ops(p, g, hw, cfg, iterations, costs);
  auto res = base_resources(hw);
  res.push_back(R_NETWORK);
  res.push_back(R_HOST);
  EngineResult er = run_engine(dr.ops, res, hw.capacity_bytes, true);
  if (er.deadlock) {
    std::string s = "simulation deadlock; blocked ops: ";
    for (size_t i = 0; i < er.blocked.size(); ++i) s += (i ? "; " : "") + er.blocked[i];
    dr.error = s;
    return dr;
  }
  dr.events = er.events;
  const auto& ops = dr.ops;
  std::stable_sort(dr.events.begin(), dr.events.end(), [&](const EngineEvent& a, const EngineEvent& b) {
    if (a.t_start != b.t_start) return a.t_start < b.t_start;
    int c = std::string(res_name(a.res)).compare(res_name(b.res));
    if (c != 0) return c < 0;
    return ops[a.op].block < ops[b.op].block;
  });
  dr.peak = er.peak;
  dr.makespan = er.makespan;
  std::vector<double> bw1;
  for (auto& e : dr.events)
    if (ops[e.op].action == Action::BW && ops[e.op].block == 1) bw1.push_back(e.t_end);
  std::sort(bw1.begin(), bw1.end());
  for (size_t i = 1; i < bw1.size(); ++i) dr.iteration_times.push_back(bw1[i] - bw1[i - 1]);
  dr.iteration_time = dr.iteration_times.empty() ? er.makespan : dr.iteration_times.back();
  // _exposed_comm (distsim.py:269-288)
  std::vector<std::pair<double, double>> comp;
  for (auto& e : dr.events)
    if (e.res == R_COMPUTE) comp.emplace_back(e.t_start, e.t_end);
  std::sort(comp.begin(), comp.end());
  std::vector<std::pair<double, double>> merged;
  for (auto& c : comp) {
    if (!merged.empty() && c.first <= merged.back().second + kDistEps)
      merged.back().second = std::max(merged.back().second, c.second);
    else
      merged.push_back(c);
  }
  double exposed = 0.0;
  for (auto& e : dr.events) {
    Action a = ops[e.op].action;
    if ((a != Action::EXCHANGE && a != Action::ALL_GATHER) || ops[e.op].iteration != iterations) continue;
    double hidden = 0.0;
    for (auto& m : merged) hidden += std::max(0.0, std::min(m.second, e.t_end) - std::max(m.first, e.t_start));
    exposed += (e.t_end - e.t_start) - hidden;
  }
  dr.exposed_comm = std::max(exposed, 0.0);
  // _check_lower_bound (distsim.py:291-310)
  double compute_total = 0.0;
  for (auto& s : p.stages)
    for (auto& op : s.ops) {
      const BlockCost& c = costs.at(op.block);
      if (op.action == Action::FW || op.action == Action::RECOMPUTE_FW) compute_total += c.fwd_seconds;
      else if (op.action == Action::BW) compute_total += c.bwd_seconds;
    }
  int last_it = 0;
  for (auto& e : dr.events)
    if (ops[e.op].action == Action::EXCHANGE) last_it = std::max(last_it, ops[e.op].iteration);
  PySum comm_sum;
  for (auto& e : dr.events)
    if (ops[e.op].action == Action::EXCHANGE && ops[e.op].iteration == last_it) comm_sum.add(e.t_end - e.t_start);
  double comm_total = comm_sum.value();
  double bound = std::max(compute_total, comm_total);
  if (dr.iteration_time + 1e-6 < bound)
    dr.error = "iteration time " + py_g(dr.iteration_time) + "s under the lower bound " + py_g(bound) + "s";
  return dr;
}

}  // namespace krt
