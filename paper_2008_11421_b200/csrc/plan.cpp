#include "plan.hpp"

#include <algorithm>
#include <set>
#include <sstream>

namespace krt {
namespace {
const char* kActionNames[] = {"fw", "bw", "swap_in", "swap_out", "recompute_fw",
                              "weight_in", "grad_out", "exchange", "host_update", "all_gather"};
const char* kStrategyNames[] = {"eager", "capacity", "capacity-recompute"};

// rendering priority (plan.py:145-148): compute first, then swap-in, swap-out
int render_rank(Action a) {
  switch (a) {
    case Action::SWAP_IN: return 1;
    case Action::SWAP_OUT: return 2;
    default: return 0;
  }
}

std::string op_code(const PlanOp& op) {
  std::string b = std::to_string(op.block);
  switch (op.action) {
    case Action::FW:
    case Action::RECOMPUTE_FW: return "F" + b;
    case Action::BW: return "B" + b;
    case Action::SWAP_IN: return "S" + b + "in";
    default: return "S" + b + "out";
  }
}
}  // namespace

const char* action_name(Action a) { return kActionNames[(int)a]; }
bool action_from_name(const std::string& s, Action* out) {
  for (int i = 0; i < 5; ++i)  // only the five plan actions are legal in plan.json
    if (s == kActionNames[i]) {
      *out = (Action)i;
      return true;
    }
  return false;
}
const char* strategy_name(Strategy s) { return kStrategyNames[(int)s]; }

std::vector<int> Plan::swapped_blocks() const {
  std::set<int> s;
  for (auto& st : stages)
    for (auto& op : st.ops)
      if (op.action == Action::SWAP_IN) s.insert(op.block);
  return std::vector<int>(s.begin(), s.end());
}

Plan plan_from_json(const Json& j) {
  Plan p;
  const std::string& st = j.at("strategy").as_str();
  bool ok = false;
  for (int i = 0; i < 3; ++i)
    if (st == kStrategyNames[i]) {
      p.strategy = (Strategy)i;
      ok = true;
    }
  if (!ok) throw JsonError("'" + st + "' is not a valid Strategy");
  for (auto& e : j.at("blocks").arr) {
    Block b;
    b.id = (int)e.at("id").as_int();
    const Json& lay = e.at("layers");
    if (lay.kind != Json::Array || lay.arr.size() < 2) throw JsonError("block layers must be [lo, hi]");
    b.first_layer = (int)lay.arr[0].as_int();
    b.last_layer = (int)lay.arr[1].as_int();
    if (auto* v = e.find("swap_bytes")) b.swap_bytes = v->as_num();
    if (auto* v = e.find("recompute")) b.recompute = v->as_bool();
    if (auto* v = e.find("checkpoint")) b.checkpoint = v->as_bool();
    p.blocks.push_back(b);
  }
  for (auto& e : j.at("stages").arr) {
    Stage s;
    s.id = (int)e.at("id").as_int();
    if (auto* v = e.find("duration")) s.duration = v->as_num();
    for (auto& o : e.at("ops").arr) {
      if (o.kind != Json::Array || o.arr.size() != 2) throw JsonError("op must be [action, block]");
      PlanOp op;
      if (!action_from_name(o.arr[0].as_str(), &op.action))
        throw JsonError("'" + o.arr[0].as_str() + "' is not a valid Action");
      op.block = (int)o.arr[1].as_int();
      s.ops.push_back(op);
    }
    p.stages.push_back(std::move(s));
  }
  if (auto* v = j.find("predicted_makespan")) p.predicted_makespan = v->as_num();
  if (auto* v = j.find("theta"))
    if (v->kind != Json::Null) {
      p.has_theta = true;
      p.theta = v->as_int();
    }
  return p;
}

Plan plan_from_json_text(const std::string& text) { return plan_from_json(json_parse(text)); }

std::string plan_to_json(const Plan& p) {
  std::ostringstream os;
  os << "{\"strategy\": \"" << strategy_name(p.strategy) << "\", \"predicted_makespan\": "
     << py_float_repr(p.predicted_makespan) << ", \"theta\": ";
  if (p.has_theta) os << p.theta; else os << "null";
  os << ", \"blocks\": [";
  for (size_t i = 0; i < p.blocks.size(); ++i) {
    auto& b = p.blocks[i];
    os << (i ? ", " : "") << "{\"id\": " << b.id << ", \"layers\": [" << b.first_layer << ", "
       << b.last_layer << "], \"swap_bytes\": " << py_float_repr(b.swap_bytes)
       << ", \"recompute\": " << (b.recompute ? "true" : "false")
       << ", \"checkpoint\": " << (b.checkpoint ? "true" : "false") << "}";
  }
  os << "], \"stages\": [";
  for (size_t i = 0; i < p.stages.size(); ++i) {
    auto& s = p.stages[i];
    os << (i ? ", " : "") << "{\"id\": " << s.id << ", \"duration\": " << py_float_repr(s.duration)
       << ", \"ops\": [";
    for (size_t k = 0; k < s.ops.size(); ++k)
      os << (k ? ", " : "") << "[\"" << action_name(s.ops[k].action) << "\", " << s.ops[k].block << "]";
    os << "]}";
  }
  os << "]}";
  return os.str();
}

std::string plan_string(const Plan& p) {
  std::string out;
  for (size_t i = 0; i < p.stages.size(); ++i) {
    std::vector<PlanOp> ops = p.stages[i].ops;
    std::stable_sort(ops.begin(), ops.end(), [](const PlanOp& a, const PlanOp& b) {
      int ra = render_rank(a.action), rb = render_rank(b.action);
      return ra != rb ? ra < rb : a.block < b.block;
    });
    if (i) out += " \xE2\x86\x92 ";  // " → "
    for (size_t k = 0; k < ops.size(); ++k) out += (k ? "||" : "") + op_code(ops[k]);
  }
  return out;
}

std::map<int, std::vector<int>> skip_requirement_map(const std::vector<Block>& blocks, const Model& g) {
  std::map<int, int> block_of;
  for (auto& b : blocks)
    for (int l = b.first_layer; l <= b.last_layer; ++l) block_of[l] = b.id;
  std::map<int, std::set<int>> dem;
  for (auto& e : g.edges) {
    if (!e.skip) continue;
    auto s = block_of.find(e.src), d = block_of.find(e.dst);
    if (s == block_of.end() || d == block_of.end()) throw JsonError("skip edge endpoint not covered by a block");
    if (d->second > s->second + 1) dem[d->second].insert(s->second);
  }
  std::map<int, std::vector<int>> out;
  for (auto& kv : dem) out[kv.first] = std::vector<int>(kv.second.begin(), kv.second.end());
  return out;
}

std::vector<int> op_requires(const PlanOp& op, const std::map<int, std::vector<int>>& skip) {
  std::vector<int> r;
  auto it = skip.find(op.block);
  switch (op.action) {
    case Action::FW:
      if (op.block >= 2) r.push_back(op.block - 1);
      break;
    case Action::RECOMPUTE_FW:
      if (op.block >= 2) r.push_back(op.block - 1);
      if (it != skip.end()) r.insert(r.end(), it->second.begin(), it->second.end());
      break;
    case Action::BW:
      r.push_back(op.block);
      if (it != skip.end()) r.insert(r.end(), it->second.begin(), it->second.end());
      break;
    default:
      break;
  }
  return r;
}

}  // namespace krt
