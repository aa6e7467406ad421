// Execution-plan IR: the drop-in boundary between the reference planner and
// this runtime.  Mirrors plan.py:24-106 (types), :109-138 (residency
// demands), :145-167 (rendering) and :179-231 (plan.json wire format).
#pragma once
#include <map>
#include <string>
#include <vector>

#include "json.hpp"
#include "model.hpp"

namespace krt {

enum class Action : int { FW = 0, BW, SWAP_IN, SWAP_OUT, RECOMPUTE_FW,
                          // data-parallel pipeline ops (distsim.py:168-236)
                          WEIGHT_IN, GRAD_OUT, EXCHANGE, HOST_UPDATE,
                          // B200 executor variant: weight shard all-gather
                          ALL_GATHER };
const char* action_name(Action a);
bool action_from_name(const std::string& s, Action* out);

enum class Strategy : int { EAGER = 0, CAPACITY, CAPACITY_RECOMPUTE };
const char* strategy_name(Strategy s);

struct Block {
  int id = 0, first_layer = 0, last_layer = 0;
  double swap_bytes = 0.0;
  bool recompute = false, checkpoint = false;
};

struct PlanOp {
  Action action = Action::FW;
  int block = 0;
};

struct Stage {
  int id = 0;
  std::vector<PlanOp> ops;
  double duration = 0.0;
};

struct Plan {
  std::vector<Stage> stages;
  Strategy strategy = Strategy::CAPACITY_RECOMPUTE;
  std::vector<Block> blocks;
  double predicted_makespan = 0.0;
  bool has_theta = false;
  long long theta = 0;

  const Block& block(int id) const { return blocks.at((size_t)id - 1); }
  std::vector<int> swapped_blocks() const;
};

Plan plan_from_json(const Json& j);
Plan plan_from_json_text(const std::string& text);
std::string plan_to_json(const Plan& p);
std::string plan_string(const Plan& p);

// block -> sorted skip-source blocks (plan.py:109-126)
std::map<int, std::vector<int>> skip_requirement_map(const std::vector<Block>& blocks, const Model& g);
std::vector<int> op_requires(const PlanOp& op, const std::map<int, std::vector<int>>& skip);

}  // namespace krt
