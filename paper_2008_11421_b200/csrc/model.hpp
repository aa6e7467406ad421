// Layer graph, hardware description and the analytic cost model the plan's
// byte/second figures come from.  Semantics follow the reference:
//   model_ir.py:47-76 (kinds, required fields), :173-220 (DAG checks),
//   :281-379 (text format); cost_model.py:97-213 (op counts, memory),
//   :250-273 (block_cost), :308-339 (hardware key=value format).
#pragma once
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

namespace krt {

struct FormatError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

enum class LayerKind : int {
  Conv, ReLU, Pool, BatchNorm, LSTM, SelfAttention, FullyConnected,
  Softmax, Dropout, Reshape, ElementWise, Add
};
const char* kind_name(LayerKind k);
bool kind_from_name(const std::string& s, LayerKind* out);

struct Layer {
  int id = 0;
  LayerKind kind = LayerKind::ElementWise;
  // shape fields; -1 = absent (the reference's None)
  long long w_out = -1, h_out = -1, c_in = -1, c_out = -1, k = -1;
  double pool_factor = -1;
  long long d_k = -1, d_v = -1, x_count = -1, y_count = -1, wt_count = -1;
  long long element_bytes = 4;
  long long ov_fwd = -1, ov_wt = -1, ov_grad = -1;  // measured overrides
};

struct Edge {
  int src = 0, dst = 0;
  bool skip = false;
};

struct Model {
  std::vector<Layer> layers;
  std::vector<Edge> edges;
  long long batch = 1;
  const Layer& layer(int id) const { return layers.at((size_t)id - 1); }
  int num_layers() const { return (int)layers.size(); }
};

// Parse the reference's model text format; throws FormatError with the
// first problem (format errors) or all DAG violations joined by "; ".
Model parse_model_text(const std::string& text);
std::vector<std::string> validate_dag(const Model& g);

struct Hardware {
  double capacity_bytes = 0, far_mem_bw = 0, near_mem_bw = 0, interconnect_bw = 0;
  double compute_rate = 0, host_update_rate = 1e9;
  bool duplex = true;
  double backward_multiplier = 2.0;
  std::vector<std::pair<std::string, double>> efficiency;
  double swap_throughput() const;
  double kind_efficiency(LayerKind k) const;
};
Hardware parse_hardware_text(const std::string& text);

// per-layer figures (cost_model.py:167, :187-213)
double layer_ops(const Layer& l, long long batch);
long long weight_elements(const Layer& l);
struct LayerMem { long long fwd, wt, grad; };
LayerMem layer_memory(const Layer& l, long long batch);

struct BlockCost {
  int block_id = 0;
  double fwd_seconds = 0, bwd_seconds = 0, bytes = 0, wt_bytes = 0, grad_bytes = 0;
  double weight_elems = 0, swap_seconds = 0;
};
BlockCost block_cost(int block_id, int first_layer, int last_layer, const Model& g,
                     const Hardware& hw);

}  // namespace krt
