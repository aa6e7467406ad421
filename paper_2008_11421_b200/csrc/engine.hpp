// Op DAG + deterministic event engine: the execution semantics every plan
// op obeys, shared by the schedule simulator, the DP pipeline model and the
// executor's issue order / static arena assignment.
//   simulator.py:67-135  run_engine      simulator.py:253-349 build_engine_ops
//   simulator.py:364-399 simulate        planner.py:342-499  validate_plan
//   distsim.py:140-266   simulate_distributed (5-stage DP pipeline)
#pragma once
#include <map>
#include <string>
#include <vector>

#include "model.hpp"
#include "plan.hpp"

namespace krt {

// Python >= 3.12 builtin sum() over floats: Neumaier-compensated
// (bltinmodule.c builtin_sum_impl).  Used wherever the reference calls sum().
struct PySum {
  double f = 0.0, c = 0.0;
  void add(double x) {
    double t = f + x;
    if ((f < 0 ? -f : f) >= (x < 0 ? -x : x)) c += (f - t) + x;
    else c += (x - t) + f;
    f = t;
  }
  double value() const { return (c != 0.0 && c - c == 0.0) ? f + c : f; }
};

enum Res : int { R_COMPUTE = 0, R_XFER_IN, R_XFER_OUT, R_XFER, R_NETWORK, R_HOST, R_COUNT };
const char* res_name(int r);

struct EngineOp {
  Action action = Action::FW;
  int block = -1;       // -1 for group-level ops
  int group = -1;       // DP group (1-based) or -1
  int stage = -1;       // plan stage index (0-based) or -1
  int iteration = 0;    // 0 = single-iteration simulate (no "iter" tag)
  bool has_stage_tag = false;
  int res = R_COMPUTE;
  double duration = 0.0;
  std::vector<int> deps;   // ops that must have completed
  int gate = -1;           // op that must have started
  double alloc = 0.0;      // bytes reserved at start
  double free_end = 0.0;   // bytes released at end
  std::string missing;     // unsatisfiable precondition
  std::string tag() const; // simulator.py:159-167 _tag_str
};

struct EngineEvent {
  int op = -1;
  int res = 0;
  double t_start = 0, t_end = 0, stall_before = 0;
};

struct EngineResult {
  bool deadlock = false;
  std::vector<std::string> blocked;   // DeadlockError.blocked
  std::vector<EngineEvent> events;    // in op-index order (started ops only)
  std::vector<int> start_order;       // op indices in the order they started
  double peak = 0.0, makespan = 0.0;
};

EngineResult run_engine(const std::vector<EngineOp>& ops, const std::vector<int>& resources,
                        double capacity, bool enforce);

std::map<int, BlockCost> plan_costs(const Plan& p, const Model& g, const Hardware& hw);
std::vector<EngineOp> build_engine_ops(const Plan& p, const Model& g, const Hardware& hw,
                                       const std::map<int, BlockCost>& costs);
std::vector<int> base_resources(const Hardware& hw);

struct SimResult {
  bool deadlock = false;
  std::vector<std::string> blocked;
  std::vector<EngineEvent> events;  // sorted by (t_start, resource name)
  std::vector<EngineOp> ops;
  double makespan = 0, total_stall = 0, peak = 0;
  std::string csv() const;          // SimTrace.to_csv schema
};
SimResult simulate(const Plan& p, const Model& g, const Hardware& hw, bool enforce);
// simulator.py:352-361 plan_metrics with caller-supplied costs:
// returns false on deadlock; makespan, stall (= makespan - busy), peak
bool plan_metrics(const Plan& p, const Model& g, const Hardware& hw, const std::map<int, BlockCost>& costs,
                  double* makespan, double* stall, double* peak);

std::vector<std::string> validate_plan(const Plan& p, const Model& g, const Hardware& hw);
std::vector<std::string> residency_memory_walk(const Plan& p, const Model& g, const Hardware& hw,
                                               double* peak_demand);

// ---- data-parallel pipeline -------------------------------------------------
struct DistConfig {
  int workers = 1;
  bool ring = true;
  double net_bw = 12.5e9, net_latency = 0.0;
  int groups = 0;  // 0 = one group per block
  // B200 executor variant (DESIGN 3): per group, in reverse block
  // order, a device reduce-scatter of the gradients right after the members'
  // backward, a D2H of this rank's 1/P shard, the host update of that shard,
  // and next iteration an H2D of the updated shard followed by an all-gather.
  // The reference (false) swaps whole gradients out and all-reduces on the host.
  bool device_exchange = false;
  // distsim.py:165 takes the iteration's index offset BEFORE appending the
  // weight_in ops, so from iteration 2 on every base op's deps point that many
  // ops too early (e.g. bw 6 waits on fw 2).  false reproduces it (parity);
  // true shifts by the real offset, which is what the executor's DAG does.
  bool exact_deps = false;
};
double allreduce_time(double bytes, const DistConfig& cfg);
std::vector<std::vector<int>> assign_groups(int num_blocks, int groups);

struct DistResult {
  std::string error;                // deadlock / lower-bound failure text
  std::vector<EngineEvent> events;  // sorted by (t_start, resource, block)
  std::vector<EngineOp> ops;
  std::vector<double> iteration_times;
  double iteration_time = 0, exposed_comm = 0, peak = 0, makespan = 0;
};
// Builds the multi-iteration op list exactly as distsim.py:140-237.
std::vector<EngineOp> build_dist_ops(const Plan& p, const Model& g, const Hardware& hw,
                                     const DistConfig& cfg, int iterations,
                                     const std::map<int, BlockCost>& costs);
// Static arena assignment realising the simulator's byte ledger
// (simulator.py:67-135, alloc at fw/recompute/swap_in start, free at
// swap_out/bw end and at the consumer fw of a recompute block).  Instances
// are placed first-fit-decreasing by size over their simulated lifetimes;
// every instance that reuses bytes of an earlier one depends on that
// instance's freeing op, so the physical ledger holds for any real timing.
struct ArenaInstance {
  int block = 0;
  size_t off = 0, bytes = 0;
  int alloc_op = -1, free_op = -1;
};
struct ArenaPlan {
  std::vector<ArenaInstance> inst;
  std::vector<int> inst_of_alloc, inst_read;   // per base op
  std::vector<std::vector<int>> deps;          // per base op: extra deps (free ops)
  size_t arena_bytes = 0;
  double ledger_peak = 0;
  std::vector<int> start_order;                // base simulation start order
};
ArenaPlan plan_arena(const Plan& p, const Model& g, const Hardware& hw, const std::vector<EngineOp>& base,
                     const std::map<int, size_t>& block_bytes);

// Flat parameter layout of the DP pipeline: blocks in order, contiguous per
// group (assign_groups), each group padded to world*64 elements so every
// rank's 1/world shard is 256-byte aligned.
struct DpLayout {
  std::vector<int64_t> block_off;              // per block (index = id-1)
  std::vector<int64_t> group_lo, group_n, shard_n;
  std::vector<int> group_of;                   // per block, 1-based
  int64_t total = 0;
};
DpLayout dp_layout(const std::vector<int64_t>& block_params, int groups, int world);

DistResult simulate_distributed(const Plan& p, const Model& g, const Hardware& hw,
                                const DistConfig& cfg, int iterations);

}  // namespace krt
