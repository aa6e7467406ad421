#include "occupancy.hpp"

#include <algorithm>
#include <set>
#include <stdexcept>

namespace krt {
namespace {
constexpr double kEps = 1e-12;  // occupancy.py:27

double clamp01(double x) { return std::min(std::max(x, 0.0), 1.0); }

double active_denominator(const std::vector<std::pair<double, double>>& active, double rate) {
  PySum d;  // occupancy.py:126 sum() over the generator
  for (auto& [processed, t_proc] : active) d.add(processed + rate * t_proc);
  return d.value();
}
}  // namespace

// occupancy.py:77-83
double occupancy_from_times(double busy, double idle) {
  if (busy < 0 || idle < 0) throw std::invalid_argument("busy/idle times must be non-negative");
  double total = busy + idle;
  if (total <= 0) throw std::invalid_argument("busy + idle must be positive");
  return busy / total;
}

// occupancy.py:86-90
double occupancy_from_buffers(double avail, double required) {
  if (required <= 0) throw std::invalid_argument("required bytes must be positive");
  return std::min(std::max(avail, 0.0) / required, 1.0);
}

// occupancy.py:93-108
BufferState advance_buffers(const BufferState& prev, double swapped_in, double processed, double capacity) {
  double avail = prev.avail_bytes - (swapped_in - processed);
  avail = std::min(std::max(avail, 0.0), capacity);
  BufferState s;
  s.avail_bytes = avail;
  s.swapped_in_bytes = swapped_in;
  s.processed_bytes = processed;
  s.required_bytes = prev.required_bytes;
  s.step = prev.step + 1;
  return s;
}

// occupancy.py:116-120
double swapped_in_this_step(double throughput, double t_proc, double avail_prev) {
  if (throughput < 0 || t_proc < 0 || avail_prev < 0) throw std::invalid_argument("inputs must be non-negative");
  return std::min(throughput * t_proc, avail_prev);
}

// occupancy.py:123-138: 1 before theta, then avail / (processed + deliverable)
double refined_occupancy(const BufferState& s, const std::vector<std::pair<double, double>>& active,
                         const Hardware& hw, long long theta) {
  if (theta < 0 || s.step < theta) return 1.0;
  double denom = active_denominator(active, hw.swap_throughput());
  if (denom <= 0) return 1.0;
  return clamp01(s.avail_bytes / denom);
}

// occupancy.py:141-151
double coarse_occupancy(const BufferState& s, const std::vector<std::pair<double, double>>& active,
                        const Hardware& hw) {
  double denom = active_denominator(active, hw.swap_throughput());
  if (denom <= 0) return 1.0;
  return clamp01(s.avail_bytes / denom);
}

// occupancy.py:154-175: durations of the backward compute steps (plan.py:94-102
// backward_compute_steps) and the step at which each swapped block is first needed
BackwardProfile backward_profile(const Plan& p, const Model& g, const Hardware& hw) {
  BackwardProfile bp;
  auto costs = plan_costs(p, g, hw);
  auto skip = skip_requirement_map(p.blocks, g);
  std::set<int> swapped;
  for (int b : p.swapped_blocks()) swapped.insert(b);
  size_t start = p.stages.size();
  for (size_t i = 0; i < p.stages.size() && start == p.stages.size(); ++i)
    for (auto& op : p.stages[i].ops)
      if (op.action == Action::BW || op.action == Action::RECOMPUTE_FW) {
        start = i;
        break;
      }
  std::vector<int> first_order;  // dict insertion order of first_need
  std::map<int, int> first_need;
  int j = 0;
  for (size_t i = start; i < p.stages.size(); ++i)
    for (auto& op : p.stages[i].ops) {
      if (op.action != Action::BW && op.action != Action::RECOMPUTE_FW) continue;
      ++j;
      const BlockCost& c = costs.at(op.block);
      bp.durations.push_back(op.action == Action::BW ? c.bwd_seconds : c.fwd_seconds);
      std::vector<int> req;
      if (op.action == Action::BW) req.push_back(op.block);
      else if (op.block >= 2) req.push_back(op.block - 1);
      auto it = skip.find(op.block);
      if (it != skip.end()) req.insert(req.end(), it->second.begin(), it->second.end());
      for (int q : req)
        if (swapped.count(q) && !first_need.count(q)) {
          first_need[q] = j;
          first_order.push_back(q);
        }
    }
  for (int q : first_order) bp.needed_at[first_need[q]].push_back(q);
  for (int q : swapped) bp.swap_seconds[q] = costs.at(q).swap_seconds;
  return bp;
}

// occupancy.py:178-199
long long find_theta(const Plan& p, const Model& g, const Hardware& hw) {
  BackwardProfile bp = backward_profile(p, g, hw);
  double cum_proc = 0.0, cum_transfer = 0.0;
  for (int k = 0; k < (int)bp.durations.size(); ++k) {
    auto it = bp.needed_at.find(k + 1);
    if (it != bp.needed_at.end())
      for (int q : it->second) cum_transfer += bp.swap_seconds.at(q);
    if (cum_proc + kEps < cum_transfer) return k;
    cum_proc += bp.durations[k];
  }
  return -1;
}

// occupancy.py:202-225
OccupancyReport analytic_report(const Plan& p, const Model& g, const Hardware& hw) {
  BackwardProfile bp = backward_profile(p, g, hw);
  OccupancyReport r;
  r.theta = find_theta(p, g, hw);
  double busy_total = 0.0, idle_total = 0.0;
  for (int j = 1; j <= (int)bp.durations.size(); ++j) {
    double dur = bp.durations[j - 1];
    double idle = 0.0;
    if (r.theta >= 0 && j >= std::max<long long>(r.theta, 1)) {
      auto it = bp.needed_at.find(j);
      if (it != bp.needed_at.end() && !it->second.empty()) {
        PySum pace;
        for (int q : it->second) pace.add(bp.swap_seconds.at(q));
        idle = std::max(0.0, pace.value() - dur);
      }
    }
    StepOccupancy s;
    s.step = j;
    s.occupancy = dur + idle > 0 ? occupancy_from_times(dur, idle) : 1.0;
    s.busy_s = dur;
    s.idle_s = idle;
    r.per_step.push_back(s);
    busy_total += dur;
    idle_total += idle;
  }
  r.mean_occupancy = busy_total + idle_total > 0 ? busy_total / (busy_total + idle_total) : 1.0;
  return r;
}

// occupancy.py:228-237
OccupancyReport report_from_steps(const std::vector<StepOccupancy>& steps, long long theta) {
  OccupancyReport r;
  r.theta = theta;
  PySum busy, idle;
  for (auto& s : steps) {
    StepOccupancy o = s;
    o.occupancy = occupancy_from_times(s.busy_s, s.idle_s);
    r.per_step.push_back(o);
  }
  for (auto& s : r.per_step) busy.add(s.busy_s);
  for (auto& s : r.per_step) idle.add(s.idle_s);
  double b = busy.value(), i = idle.value();
  r.mean_occupancy = b + i > 0 ? b / (b + i) : 1.0;
  return r;
}

// occupancy.py:60-70
std::string OccupancyReport::csv() const {
  std::string s = "step,occupancy,busy_s,idle_s\n";
  for (auto& x : per_step)
    s += std::to_string(x.step) + "," + py_9g(x.occupancy) + "," + py_9g(x.busy_s) + "," + py_9g(x.idle_s) + "\n";
  return s;
}

std::string OccupancyReport::summary() const {
  return "theta," + (theta < 0 ? std::string("none") : std::to_string(theta)) + "\nmean_occupancy," +
         py_9g(mean_occupancy) + "\n";
}

// simulator.py:200-236
TraceOccupancy trace_occupancy(const SimResult& sr, long long theta) {
  TraceOccupancy t;
  std::vector<const EngineEvent*> steps;
  PySum busy;
  for (auto& e : sr.events) {
    Action a = sr.ops[e.op].action;
    if (a != Action::FW && a != Action::BW && a != Action::RECOMPUTE_FW) continue;
    busy.add(e.t_end - e.t_start);
    if (a != Action::FW) steps.push_back(&e);
  }
  std::stable_sort(steps.begin(), steps.end(),
                   [](const EngineEvent* a, const EngineEvent* b) { return a->t_start < b->t_start; });
  for (size_t k = 0; k < steps.size(); ++k) {
    StepOccupancy s;
    s.step = (int)k + 1;
    s.busy_s = steps[k]->t_end - steps[k]->t_start;
    s.idle_s = steps[k]->stall_before;
    s.occupancy = s.busy_s + s.idle_s > 0 ? occupancy_from_times(s.busy_s, s.idle_s) : 1.0;
    t.backward.push_back(s);
    if (t.first_stall_step < 0 && steps[k]->stall_before > 1e-9) t.first_stall_step = s.step;
  }
  t.boundary_stall = steps.empty() ? 0.0 : steps[0]->stall_before;
  t.mean_occupancy = sr.makespan > 0 ? busy.value() / sr.makespan : 1.0;
  t.summary_csv = "makespan,total_stall,peak_mem,mean_occupancy,theta_step\n" + py_9g(sr.makespan) + "," +
                  py_9g(sr.total_stall) + "," + py_9g(sr.peak) + "," + py_9g(t.mean_occupancy) + "," +
                  (theta < 0 ? std::string("none") : std::to_string(theta)) + "\n";
  return t;
}

}  // namespace krt
