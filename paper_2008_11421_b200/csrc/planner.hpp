// Native planner: the reference's two-stage optimisation (block partition,
// recompute flags) and Algorithm-1 schedule generation, restated in C++ so a
// plan can be produced on the GPU host in milliseconds and bit-identical to
// oocsched's.  Each function names the reference function it follows:
//   planner.py:56-68   enumerate_partitions   planner.py:71-121  CostTable/build_blocks
//   planner.py:124-162 retained_start / forced_recompute
//   planner.py:169-325 generate_schedule / _capacity_backward_stages
//   planner.py:328-335 finalize_plan          planner.py:517-614 evaluate_blocks / solve_opt2
//   planner.py:622-741 _search_exhaustive     planner.py:764-883 _dp_partition / _polish_splits
//   planner.py:890-912 plan_model             occupancy.py:150-199 find_theta
#pragma once
#include <stdexcept>
#include <string>

#include "engine.hpp"
#include "occupancy.hpp"

namespace krt {

struct InfeasibleModel : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct PlannerMisuse : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// solver: "auto" | "exhaustive" | "dp"; max_blocks <= 0 means None
Plan plan_model(const Model& g, const Hardware& hw, Strategy strategy, const std::string& solver, int max_blocks,
                int layer_bound = 20);

}  // namespace krt
