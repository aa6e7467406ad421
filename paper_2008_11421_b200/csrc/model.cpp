#include "model.hpp"

#include <cmath>
#include <cstdlib>
#include <set>
#include <sstream>

namespace krt {
namespace {

const char* kKindNames[] = {"Conv", "ReLU", "Pool", "BatchNorm", "LSTM", "SelfAttention",
                            "FullyConnected", "Softmax", "Dropout", "Reshape",
                            "ElementWise", "Add"};

// shape field table: file key, member pointer (pool_factor handled apart)
enum Field { W_OUT, H_OUT, C_IN, C_OUT, K, POOL, D_K, D_V, X, Y, WT, NFIELD };
const char* kFieldKey[NFIELD] = {"Wout", "Hout", "Cin", "Cout", "K", "c",
                                 "dk", "dv", "X", "Y", "WT"};

double field_value(const Layer& l, int f) {
  switch (f) {
    case W_OUT: return (double)l.w_out;
    case H_OUT: return (double)l.h_out;
    case C_IN: return (double)l.c_in;
    case C_OUT: return (double)l.c_out;
    case K: return (double)l.k;
    case POOL: return l.pool_factor;
    case D_K: return (double)l.d_k;
    case D_V: return (double)l.d_v;
    case X: return (double)l.x_count;
    case Y: return (double)l.y_count;
    case WT: return (double)l.wt_count;
  }
  return -1;
}
bool present(const Layer& l, int f) {
  // absent fields are stored as -1 (pool_factor too)
  return field_value(l, f) != -1;
}

// model_ir.py:63-85
std::vector<int> required_fields(LayerKind k) {
  switch (k) {
    case LayerKind::Conv: return {W_OUT, H_OUT, C_IN, C_OUT, K};
    case LayerKind::ReLU: return {Y};
    case LayerKind::Pool: return {W_OUT, H_OUT, C_IN, C_OUT, K, POOL};
    case LayerKind::BatchNorm: return {X, Y, C_IN};
    case LayerKind::LSTM: return {X, Y};
    case LayerKind::SelfAttention: return {D_K};
    case LayerKind::FullyConnected: return {X, Y};
    default: return {X};
  }
}
std::vector<int> optional_fields(LayerKind k) {
  switch (k) {
    case LayerKind::Conv: return {Y};
    case LayerKind::Pool: return {Y};
    case LayerKind::SelfAttention: return {D_V, Y};
    case LayerKind::FullyConnected: return {WT};
    case LayerKind::Softmax: return {Y};
    case LayerKind::Reshape: return {Y};
    default: return {};
  }
}

std::string fmt_field(double v) {
  // the reference prints the stored Python value: ints plainly
  if (v == std::floor(v) && std::fabs(v) < 1e15) {
    std::ostringstream os;
    os << (long long)v;
    return os.str();
  }
  std::ostringstream os;
  os << v;
  return os.str();
}

long long parse_int_tok(const std::string& tok, const std::string& ctx) {
  char* e = nullptr;
  double v = std::strtod(tok.c_str(), &e);
  if (tok.empty() || !e || *e) throw FormatError(ctx + ": expected a number, got '" + tok + "'");
  if (v != std::floor(v)) throw FormatError(ctx + ": expected an integer, got '" + tok + "'");
  return (long long)v;
}

std::string strip(const std::string& s) {
  size_t a = s.find_first_not_of(" \t\r\n");
  if (a == std::string::npos) return "";
  size_t b = s.find_last_not_of(" \t\r\n");
  return s.substr(a, b - a + 1);
}

std::vector<std::string> split_ws(const std::string& s) {
  std::vector<std::string> out;
  std::istringstream is(s);
  std::string t;
  while (is >> t) out.push_back(t);
  return out;
}

long long req(const Layer& l, long long v, const char* key) {
  if (v == -1)
    throw FormatError("layer " + std::to_string(l.id) + ": " + kind_name(l.kind) + " requires " + key);
  return v;
}

// exact integer product (Python ints are arbitrary precision)
double exact(__int128 v) { return (double)v; }

}  // namespace

const char* kind_name(LayerKind k) { return kKindNames[(int)k]; }

bool kind_from_name(const std::string& s, LayerKind* out) {
  for (int i = 0; i < 12; ++i)
    if (s == kKindNames[i]) {
      *out = (LayerKind)i;
      return true;
    }
  return false;
}

std::vector<std::string> validate_dag(const Model& g) {
  std::vector<std::string> v;
  std::set<int> seen;
  bool dup = false;
  for (auto& l : g.layers) {
    if (seen.count(l.id)) {
      v.push_back("duplicate id " + std::to_string(l.id));
      dup = true;
    }
    seen.insert(l.id);
  }
  bool contiguous = true;
  for (size_t i = 0; i < g.layers.size(); ++i)
    if (g.layers[i].id != (int)i + 1) contiguous = false;
  if (!contiguous && !dup) {
    std::string ids = "[";
    for (size_t i = 0; i < g.layers.size(); ++i)
      ids += (i ? ", " : "") + std::to_string(g.layers[i].id);
    ids += "]";
    v.push_back("layer ids " + ids + " are not the contiguous sequence 1.." +
                std::to_string(g.layers.size()));
  }
  if (g.batch < 1) v.push_back("batch_size " + std::to_string(g.batch) + " must be >= 1");
  int n = (int)g.layers.size();
  std::set<std::pair<int, int>> seen_e;
  for (auto& e : g.edges) {
    auto key = std::make_pair(e.src, e.dst);
    std::string es = std::to_string(e.src) + " -> " + std::to_string(e.dst);
    if (seen_e.count(key)) v.push_back("duplicate edge " + es);
    seen_e.insert(key);
    if (!(1 <= e.src && e.src <= n && 1 <= e.dst && e.dst <= n)) {
      v.push_back("edge " + es + " references unknown layer");
      continue;
    }
    if (e.src >= e.dst) {
      v.push_back("backward edge " + es);
      continue;
    }
    if (e.dst > e.src + 1 && !e.skip) v.push_back("edge " + es + " jumps layers but lacks the skip flag");
    if (e.dst == e.src + 1 && e.skip)
      v.push_back("edge " + es + " is consecutive and must not be flagged skip");
  }
  std::vector<int> in(n + 2, 0), out(n + 2, 0);
  for (auto& e : g.edges)
    if (1 <= e.src && e.src <= n && 1 <= e.dst && e.dst <= n && e.src < e.dst) {
      out[e.src]++;
      in[e.dst]++;
    }
  for (int i = 2; i <= n; ++i)
    if (in[i] == 0) v.push_back("layer " + std::to_string(i) + " has no incoming edge");
  for (int i = 1; i < n; ++i)
    if (out[i] == 0) v.push_back("layer " + std::to_string(i) + " has no outgoing edge");
  for (auto& l : g.layers) {
    auto reqf = required_fields(l.kind);
    auto optf = optional_fields(l.kind);
    std::set<int> allowed(reqf.begin(), reqf.end());
    allowed.insert(optf.begin(), optf.end());
    std::string lid = "layer " + std::to_string(l.id) + ": ";
    for (int f : reqf) {
      if (!present(l, f))
        v.push_back(lid + kind_name(l.kind) + " requires " + kFieldKey[f]);
      else if (field_value(l, f) <= 0)
        v.push_back(lid + kFieldKey[f] + "=" + fmt_field(field_value(l, f)) + " must be strictly positive");
    }
    for (int f = 0; f < NFIELD; ++f) {
      double val = field_value(l, f);
      bool has = present(l, f);
      if (!allowed.count(f) && has && val != 0)
        v.push_back(lid + kFieldKey[f] + " not used by " + kind_name(l.kind));
      else if (allowed.count(f) && has && val <= 0) {
        // required fields already reported above with the same text
        bool is_req = false;
        for (int r : reqf) is_req |= (r == f);
        if (!is_req)
          v.push_back(lid + kFieldKey[f] + "=" + fmt_field(val) + " must be strictly positive");
        else
          v.push_back(lid + kFieldKey[f] + "=" + fmt_field(val) + " must be strictly positive");
      }
    }
    if (l.element_bytes <= 0)
      v.push_back(lid + "elem=" + std::to_string(l.element_bytes) + " must be positive");
  }
  return v;
}

Model parse_model_text(const std::string& text) {
  Model g;
  std::string version, batch;
  bool have_version = false, have_batch = false, saw_edges = false;
  int section = 0;  // 0 header, 1 layers, 2 edges
  std::istringstream is(text);
  std::string raw;
  int lineno = 0;
  while (std::getline(is, raw)) {
    ++lineno;
    std::string line = strip(raw.substr(0, raw.find('#')));
    if (line.empty()) continue;
    std::string L = "line " + std::to_string(lineno);
    if (line[0] == '[') {
      if (line == "[layers]") section = 1;
      else if (line == "[edges]") { section = 2; saw_edges = true; }
      else throw FormatError(L + ": unknown section " + line);
      continue;
    }
    if (section == 0) {
      size_t eq = line.find('=');
      if (eq == std::string::npos) throw FormatError(L + ": expected key = value in header");
      std::string k = strip(line.substr(0, eq)), val = strip(line.substr(eq + 1));
      if (k == "version") { version = val; have_version = true; }
      else if (k == "batch_size") { batch = val; have_batch = true; }
      else throw FormatError(L + ": unknown header key '" + k + "'");
    } else if (section == 1) {
      auto tok = split_ws(line);
      if (tok.size() < 2) throw FormatError(L + ": layer record needs 'id kind key=value...'");
      Layer l;
      l.id = (int)parse_int_tok(tok[0], L + ": layer id");
      if (!kind_from_name(tok[1], &l.kind)) throw FormatError(L + ": unknown layer kind '" + tok[1] + "'");
      for (size_t i = 2; i < tok.size(); ++i) {
        size_t eq = tok[i].find('=');
        if (eq == std::string::npos) throw FormatError(L + ": expected key=value, got '" + tok[i] + "'");
        std::string k = tok[i].substr(0, eq), val = tok[i].substr(eq + 1);
        std::string ctx = L + ": layer " + std::to_string(l.id) + " key " + k;
        if (k == "Wout") l.w_out = parse_int_tok(val, ctx);
        else if (k == "Hout") l.h_out = parse_int_tok(val, ctx);
        else if (k == "Cin") l.c_in = parse_int_tok(val, ctx);
        else if (k == "Cout") l.c_out = parse_int_tok(val, ctx);
        else if (k == "K") l.k = parse_int_tok(val, ctx);
        else if (k == "c") {
          char* e = nullptr;
          l.pool_factor = std::strtod(val.c_str(), &e);
          if (val.empty() || *e) throw FormatError(ctx + ": expected a number, got '" + val + "'");
        } else if (k == "dk") l.d_k = parse_int_tok(val, ctx);
        else if (k == "dv") l.d_v = parse_int_tok(val, ctx);
        else if (k == "X") l.x_count = parse_int_tok(val, ctx);
        else if (k == "Y") l.y_count = parse_int_tok(val, ctx);
        else if (k == "WT") l.wt_count = parse_int_tok(val, ctx);
        else if (k == "elem") l.element_bytes = parse_int_tok(val, ctx);
        else if (k == "mem_fwd") l.ov_fwd = parse_int_tok(val, ctx);
        else if (k == "mem_wt") l.ov_wt = parse_int_tok(val, ctx);
        else if (k == "mem_grad") l.ov_grad = parse_int_tok(val, ctx);
        else throw FormatError(L + ": layer " + std::to_string(l.id) + " has unknown key '" + k + "'");
      }
      g.layers.push_back(l);
    } else {
      auto tok = split_ws(line);
      if ((tok.size() != 3 && tok.size() != 4) || tok[1] != "->")
        throw FormatError(L + ": expected 'i -> j [skip]'");
      Edge e;
      if (tok.size() == 4) {
        if (tok[3] != "skip") throw FormatError(L + ": trailing token must be 'skip'");
        e.skip = true;
      }
      e.src = (int)parse_int_tok(tok[0], L + ": edge source");
      e.dst = (int)parse_int_tok(tok[2], L + ": edge target");
      g.edges.push_back(e);
    }
  }
  if (!have_version || version != "1")
    throw FormatError("unsupported or missing version " + (have_version ? "'" + version + "'" : std::string("None")));
  if (!have_batch) throw FormatError("missing batch_size header");
  g.batch = parse_int_tok(batch, "batch_size");
  if (g.layers.empty()) throw FormatError("model declares no layers");
  if (!saw_edges)
    for (int i = 1; i < (int)g.layers.size(); ++i) g.edges.push_back(Edge{i, i + 1, false});
  auto v = validate_dag(g);
  if (!v.empty()) {
    std::string all;
    for (size_t i = 0; i < v.size(); ++i) all += (i ? "; " : "") + v[i];
    throw FormatError(all);
  }
  return g;
}

double Hardware::swap_throughput() const {
  return std::min(far_mem_bw, std::min(near_mem_bw, interconnect_bw));
}

double Hardware::kind_efficiency(LayerKind k) const {
  for (auto& kv : efficiency)
    if (kv.first == kind_name(k)) return kv.second;
  return 1.0;
}

Hardware parse_hardware_text(const std::string& text) {
  Hardware hw;
  bool have[7] = {false, false, false, false, false, false, false};
  const char* keys[7] = {"capacity_bytes", "far_mem_bw", "near_mem_bw", "interconnect_bw",
                         "compute_rate", "host_update_rate", "backward_multiplier"};
  double* dst[7] = {&hw.capacity_bytes, &hw.far_mem_bw, &hw.near_mem_bw, &hw.interconnect_bw,
                    &hw.compute_rate, &hw.host_update_rate, &hw.backward_multiplier};
  std::istringstream is(text);
  std::string raw;
  int lineno = 0;
  while (std::getline(is, raw)) {
    ++lineno;
    std::string line = strip(raw.substr(0, raw.find('#')));
    if (line.empty()) continue;
    std::string L = "line " + std::to_string(lineno);
    size_t eq = line.find('=');
    if (eq == std::string::npos) throw FormatError(L + ": expected key = value");
    std::string k = strip(line.substr(0, eq)), val = strip(line.substr(eq + 1));
    bool done = false;
    for (int i = 0; i < 7; ++i)
      if (k == keys[i]) {
        char* e = nullptr;
        double d = std::strtod(val.c_str(), &e);
        if (val.empty() || *e) throw FormatError(L + ": bad number '" + val + "'");
        *dst[i] = d;
        have[i] = true;
        done = true;
      }
    if (done) continue;
    if (k == "duplex") {
      std::string lv;
      for (char c : val) lv += (char)std::tolower((unsigned char)c);
      if (lv != "true" && lv != "false") throw FormatError(L + ": duplex must be true or false");
      hw.duplex = lv == "true";
    } else if (k.rfind("efficiency.", 0) == 0) {
      std::string kind = k.substr(11);
      LayerKind lk;
      if (!kind_from_name(kind, &lk)) throw FormatError(L + ": unknown kind '" + kind + "'");
      char* e = nullptr;
      double d = std::strtod(val.c_str(), &e);
      if (val.empty() || *e) throw FormatError(L + ": bad number '" + val + "'");
      bool replaced = false;
      for (auto& kv : hw.efficiency)
        if (kv.first == kind) { kv.second = d; replaced = true; }
      if (!replaced) hw.efficiency.emplace_back(kind, d);
    } else {
      throw FormatError(L + ": unknown key '" + k + "'");
    }
  }
  std::string missing;
  for (int i = 0; i < 5; ++i)
    if (!have[i]) missing += (missing.empty() ? "" : ", ") + std::string(keys[i]);
  if (!missing.empty()) throw FormatError("missing keys: " + missing);
  for (int i = 0; i < 6; ++i)
    if (*dst[i] <= 0) throw FormatError(std::string(keys[i]) + " must be strictly positive");
  if (hw.backward_multiplier <= 0) throw FormatError("backward_multiplier must be strictly positive");
  return hw;
}

// cost_model.py:97-168; integer products are exact like Python ints
double layer_ops(const Layer& l, long long b) {
  if (b < 1) throw FormatError("batch size " + std::to_string(b) + " must be >= 1");
  switch (l.kind) {
    case LayerKind::Conv:
      return exact((__int128)req(l, l.w_out, "Wout") * req(l, l.h_out, "Hout") * req(l, l.c_out, "Cout") *
                   req(l, l.k, "K") * l.k * req(l, l.c_in, "Cin") * b);
    case LayerKind::ReLU:
      return exact((__int128)req(l, l.y_count, "Y") * b);
    case LayerKind::Pool: {
      if (l.pool_factor == -1) req(l, -1, "c");
      double base = exact((__int128)req(l, l.w_out, "Wout") * req(l, l.h_out, "Hout") *
                          req(l, l.c_out, "Cout") * req(l, l.k, "K") * l.k * req(l, l.c_in, "Cin"));
      return (base * l.pool_factor) * (double)b;
    }
    case LayerKind::BatchNorm:
      return exact((__int128)3 * b + (__int128)4 * req(l, l.x_count, "X") + (__int128)2 * req(l, l.y_count, "Y"));
    case LayerKind::LSTM:
      return exact((__int128)20 * req(l, l.y_count, "Y") * b);
    case LayerKind::SelfAttention: {
      __int128 d = req(l, l.d_k, "dk");
      return exact((4 * d * d * d + d * d + 2 * d) * b);
    }
    case LayerKind::FullyConnected:
      if (l.wt_count != -1) return exact((__int128)l.wt_count * b);
      return exact((__int128)req(l, l.x_count, "X") * req(l, l.y_count, "Y") * b);
    case LayerKind::Softmax:
      return exact((__int128)2 * req(l, l.x_count, "X") * b);
    case LayerKind::Reshape:
      return 0.0;
    default:
      return exact((__int128)req(l, l.x_count, "X") * b);
  }
}

static long long output_elements(const Layer& l) {
  if (l.y_count != -1) return l.y_count;
  switch (l.kind) {
    case LayerKind::Conv:
    case LayerKind::Pool:
      return req(l, l.w_out, "Wout") * req(l, l.h_out, "Hout") * req(l, l.c_out, "Cout");
    case LayerKind::SelfAttention: {
      long long d = req(l, l.d_k, "dk");
      return d * (l.d_v != -1 ? l.d_v : d);
    }
    case LayerKind::Reshape: return 0;
    case LayerKind::Softmax:
    case LayerKind::Dropout:
    case LayerKind::ElementWise:
    case LayerKind::Add:
      return req(l, l.x_count, "X");
    default:
      return req(l, l.y_count, "Y");
  }
}

long long weight_elements(const Layer& l) {
  if (l.wt_count != -1) return l.wt_count;
  switch (l.kind) {
    case LayerKind::Conv: return req(l, l.k, "K") * l.k * req(l, l.c_in, "Cin") * req(l, l.c_out, "Cout");
    case LayerKind::BatchNorm: return 2 * req(l, l.c_in, "Cin");
    case LayerKind::LSTM: {
      long long x = req(l, l.x_count, "X"), y = req(l, l.y_count, "Y");
      return 4 * (x + y + 1) * y;
    }
    case LayerKind::FullyConnected: return req(l, l.x_count, "X") * req(l, l.y_count, "Y");
    default: return 0;
  }
}

LayerMem layer_memory(const Layer& l, long long b) {
  if (b < 1) throw FormatError("batch size " + std::to_string(b) + " must be >= 1");
  long long afwd = output_elements(l) * l.element_bytes * b;
  long long awt = weight_elements(l) * l.element_bytes;
  LayerMem m;
  m.fwd = l.ov_fwd != -1 ? l.ov_fwd : afwd;
  m.wt = l.ov_wt != -1 ? l.ov_wt : awt;
  m.grad = l.ov_grad != -1 ? l.ov_grad : m.wt;
  return m;
}

// cost_model.py:239-273, same accumulation order
BlockCost block_cost(int block_id, int lo, int hi, const Model& g, const Hardware& hw) {
  double eff_ops = 0.0;
  for (int i = lo; i <= hi; ++i) {
    const Layer& l = g.layer(i);
    double eff = hw.kind_efficiency(l.kind);
    if (eff <= 0) throw FormatError(std::string("efficiency.") + kind_name(l.kind) + " must be positive");
    eff_ops += layer_ops(l, g.batch) / eff;
  }
  BlockCost c;
  c.block_id = block_id;
  c.fwd_seconds = eff_ops / hw.compute_rate;
  for (int i = lo; i <= hi; ++i) {
    LayerMem m = layer_memory(g.layer(i), g.batch);
    c.bytes += (double)(m.fwd + m.wt);
    c.wt_bytes += (double)m.wt;
    c.grad_bytes += (double)m.grad;
    c.weight_elems += (double)weight_elements(g.layer(i));
  }
  c.bwd_seconds = c.fwd_seconds * hw.backward_multiplier;
  c.swap_seconds = c.bytes / hw.swap_throughput();
  return c;
}

}  // namespace krt
