// extern "C" boundary (include/krt.h).  Exceptions stop here: each entry
// point maps them to a status code and a thread-local message.
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <memory>
#include <sstream>
#include <string>

#include "../../include/krt.h"
#include "engine.hpp"
#include "planner.hpp"
#include "host_optim.hpp"
#include "bn_kernels.hpp"
#include "pool_kernels.hpp"
#include "gemm_sm100.hpp"
#include "halo_sm100.hpp"
#include "mlp_lt.hpp"
#include "wgrad_sm100.hpp"
#include "ln_kernels.hpp"
#include "kernels.hpp"
#include "runtime.hpp"

using namespace krt;

struct krt_plan {
  Model model;
  Hardware hw;
  Plan plan;
};

struct krt_ctx {
  std::unique_ptr<Runtime> rt;
};

namespace {
thread_local std::string g_err;

struct Infeasible : std::runtime_error {
  using std::runtime_error::runtime_error;
};

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.data(), s.size() + 1);
  return p;
}

std::string jstr(const std::string& s) {
  std::string o = "\"";
  for (unsigned char c : s) {
    switch (c) {
      case '"': o += "\\\""; break;
      case '\\': o += "\\\\"; break;
      case '\n': o += "\\n"; break;
      case '\t': o += "\\t"; break;
      default:
        if (c < 0x20) {
          char b[8];
          std::snprintf(b, sizeof b, "\\u%04x", c);
          o += b;
        } else {
          o += (char)c;
        }
    }
  }
  return o + "\"";
}

std::string jnum(double v) { return py_float_repr(v); }

template <class F>
int guard(F&& f) {
  try {
    f();
    g_err.clear();
    return KRT_OK;
  } catch (const Infeasible& e) {
    g_err = e.what();
    return KRT_INFEASIBLE;
  } catch (const FormatError& e) {
    g_err = e.what();
    return KRT_USAGE;
  } catch (const JsonError& e) {
    g_err = e.what();
    return KRT_USAGE;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return KRT_USAGE;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return KRT_USAGE;
  } catch (const std::exception& e) {
    g_err = e.what();
    return KRT_INTERNAL;
  } catch (...) {
    g_err = "unknown error";
    return KRT_INTERNAL;
  }
}

std::string list_json(const std::vector<std::string>& v) {
  std::string s = "[";
  for (size_t i = 0; i < v.size(); ++i) s += (i ? ", " : "") + jstr(v[i]);
  return s + "]";
}
}  // namespace

extern "C" {

const char* krt_last_error(void) { return g_err.c_str(); }
const char* krt_version(void) { return "karma-b200 krt 0.1 (sm_100a)"; }
void krt_string_free(char* s) { std::free(s); }

int krt_plan_load(const char* model_text, const char* hw_text, const char* plan_json, krt_plan** out) {
  return guard([&] {
    if (!model_text || !hw_text || !plan_json || !out) throw std::invalid_argument("null argument");
    auto p = std::make_unique<krt_plan>();
    p->model = parse_model_text(model_text);
    p->hw = parse_hardware_text(hw_text);
    p->plan = plan_from_json_text(plan_json);
    *out = p.release();
  });
}

void krt_plan_free(krt_plan* p) { delete p; }

int krt_plan_model(const char* model_text, const char* hw_text, const char* strategy, const char* solver,
                   int max_blocks, krt_plan** out) {
  return guard([&] {
    if (!model_text || !hw_text || !out) throw std::invalid_argument("null argument");
    auto p = std::make_unique<krt_plan>();
    p->model = parse_model_text(model_text);
    p->hw = parse_hardware_text(hw_text);
    std::string st = strategy ? strategy : "capacity-recompute";
    Strategy s;
    if (st == "eager") s = Strategy::EAGER;
    else if (st == "capacity") s = Strategy::CAPACITY;
    else if (st == "capacity-recompute") s = Strategy::CAPACITY_RECOMPUTE;
    else throw std::invalid_argument("'" + st + "' is not a valid Strategy");
    try {
      p->plan = plan_model(p->model, p->hw, s, solver ? solver : "auto", max_blocks);
    } catch (const InfeasibleModel& e) {
      throw Infeasible(e.what());
    } catch (const PlannerMisuse& e) {
      throw std::invalid_argument(e.what());
    }
    *out = p.release();
  });
}

int krt_plan_set_capacity(krt_plan* p, double cap) {
  return guard([&] {
    if (!p || !(cap > 0)) throw std::invalid_argument("capacity must be positive");
    p->hw.capacity_bytes = cap;
  });
}

int krt_plan_string(const krt_plan* p, char** out) {
  return guard([&] { *out = dup(plan_string(p->plan)); });
}

int krt_plan_json(const krt_plan* p, char** out) {
  return guard([&] { *out = dup(plan_to_json(p->plan)); });
}

int krt_plan_validate(const krt_plan* p, char** out, int* n) {
  return guard([&] {
    auto v = validate_plan(p->plan, p->model, p->hw);
    if (n) *n = (int)v.size();
    if (out) *out = dup(list_json(v));
  });
}

int krt_plan_simulate(const krt_plan* p, int enforce, char** out) {
  return guard([&] {
    SimResult r = simulate(p->plan, p->model, p->hw, enforce != 0);
    std::ostringstream os;
    if (r.deadlock) {
      os << "{\"deadlock\": " << list_json(r.blocked) << "}";
    } else {
      os << "{\"makespan\": " << jnum(r.makespan) << ", \"total_stall\": " << jnum(r.total_stall)
         << ", \"peak_mem\": " << jnum(r.peak) << ", \"events\": [";
      for (size_t i = 0; i < r.events.size(); ++i) {
        auto& e = r.events[i];
        auto& op = r.ops[e.op];
        os << (i ? ", " : "") << "[" << jnum(e.t_start) << ", " << jnum(e.t_end) << ", \"" << res_name(e.res)
           << "\", " << op.block << ", \"" << action_name(op.action) << "\", " << jnum(e.stall_before) << "]";
      }
      // SimTrace occupancy figures (simulator.py:200-236); summary_csv with
      // find_theta as cli.py:115-116 writes it
      TraceOccupancy t = trace_occupancy(r, find_theta(p->plan, p->model, p->hw));
      os << "], \"csv\": " << jstr(r.csv()) << ", \"mean_occupancy\": " << jnum(t.mean_occupancy)
         << ", \"first_stall_backward_step\": ";
      if (t.first_stall_step < 0) os << "null";
      else os << t.first_stall_step;
      os << ", \"boundary_stall\": " << jnum(t.boundary_stall) << ", \"summary_csv\": " << jstr(t.summary_csv)
         << "}";
    }
    *out = dup(os.str());
  });
}

int krt_plan_costs(const krt_plan* p, char** out) {
  return guard([&] {
    auto costs = plan_costs(p->plan, p->model, p->hw);
    std::ostringstream os;
    os << "{\"blocks\": [";
    bool first = true;
    for (auto& b : p->plan.blocks) {
      const BlockCost& c = costs.at(b.id);
      os << (first ? "" : ", ") << "{\"id\": " << b.id << ", \"layers\": [" << b.first_layer << ", "
         << b.last_layer << "], \"fwd_seconds\": " << jnum(c.fwd_seconds) << ", \"bwd_seconds\": "
         << jnum(c.bwd_seconds) << ", \"bytes\": " << jnum(c.bytes) << ", \"wt_bytes\": " << jnum(c.wt_bytes)
         << ", \"grad_bytes\": " << jnum(c.grad_bytes) << ", \"weight_elems\": " << jnum(c.weight_elems)
         << ", \"swap_seconds\": " << jnum(c.swap_seconds) << "}";
      first = false;
    }
    os << "], \"layers\": [";
    for (int i = 1; i <= p->model.num_layers(); ++i) {
      const Layer& l = p->model.layer(i);
      os << (i > 1 ? ", " : "") << "{\"id\": " << i << ", \"kind\": \"" << kind_name(l.kind)
         << "\", \"ops\": " << jnum(layer_ops(l, p->model.batch)) << "}";
    }
    os << "]}";
    *out = dup(os.str());
  });
}

int krt_plan_occupancy(const krt_plan* p, char** out) {
  return guard([&] {
    OccupancyReport r = analytic_report(p->plan, p->model, p->hw);
    std::ostringstream os;
    os << "{\"theta\": ";
    if (r.theta < 0) os << "null";
    else os << r.theta;
    os << ", \"mean_occupancy\": " << jnum(r.mean_occupancy) << ", \"per_step\": [";
    for (size_t i = 0; i < r.per_step.size(); ++i) {
      auto& s = r.per_step[i];
      os << (i ? ", " : "") << "[" << s.step << ", " << jnum(s.occupancy) << ", " << jnum(s.busy_s) << ", "
         << jnum(s.idle_s) << "]";
    }
    os << "], \"csv\": " << jstr(r.csv()) << ", \"summary\": " << jstr(r.summary()) << "}";
    *out = dup(os.str());
  });
}

int krt_plan_simulate_dist(const krt_plan* p, const krt_dist_config* c, int iterations, char** out) {
  return guard([&] {
    if (!c) throw std::invalid_argument("null dist config");
    DistConfig cfg;
    cfg.workers = c->workers;
    cfg.ring = c->ring != 0;
    cfg.net_bw = c->net_bw;
    cfg.net_latency = c->net_latency;
    cfg.groups = c->groups;
    if (c->variant & ~(KRT_DIST_DEVICE_EXCHANGE | KRT_DIST_EXACT_DEPS)) throw std::invalid_argument("unknown dist variant bits");
    cfg.device_exchange = (c->variant & KRT_DIST_DEVICE_EXCHANGE) != 0;
    cfg.exact_deps = (c->variant & KRT_DIST_EXACT_DEPS) != 0;
    if (cfg.workers < 1) throw std::invalid_argument("workers must be >= 1");
    if (!(cfg.net_bw > 0)) throw std::invalid_argument("net_bw must be strictly positive");
    if (cfg.net_latency < 0) throw std::invalid_argument("net_latency must be non-negative");
    if (cfg.groups < 0) throw std::invalid_argument("groups must be >= 0 (0 = per block)");
    DistResult r = simulate_distributed(p->plan, p->model, p->hw, cfg, iterations);
    std::ostringstream os;
    if (!r.error.empty() && r.events.empty()) {
      os << "{\"error\": " << jstr(r.error) << "}";
    } else {
      os << "{";
      if (!r.error.empty()) os << "\"error\": " << jstr(r.error) << ", ";
      os << "\"iteration_time\": " << jnum(r.iteration_time) << ", \"iteration_times\": [";
      for (size_t i = 0; i < r.iteration_times.size(); ++i) os << (i ? ", " : "") << jnum(r.iteration_times[i]);
      os << "], \"exposed_comm\": " << jnum(r.exposed_comm) << ", \"peak_mem\": " << jnum(r.peak)
         << ", \"makespan\": " << jnum(r.makespan) << ", \"events\": [";
      for (size_t i = 0; i < r.events.size(); ++i) {
        auto& e = r.events[i];
        auto& op = r.ops[e.op];
        int worker = e.res == R_NETWORK ? -1 : 0;
        os << (i ? ", " : "") << "[" << worker << ", \"" << res_name(e.res) << "\", " << jnum(e.t_start) << ", "
           << jnum(e.t_end) << ", \"" << action_name(op.action) << "\", " << op.block << ", " << op.group << ", "
           << op.iteration << ", " << jnum(e.stall_before) << "]";
      }
      os << "]}";
    }
    *out = dup(os.str());
  });
}

int krt_dp_layout(const int64_t* block_params, int n_blocks, int groups, int world, int64_t* block_off,
                  int* n_groups, int64_t* group_lo, int64_t* group_n, int64_t* shard_n) {
  return guard([&] {
    if (n_blocks < 1 || !block_params || groups < 0) throw std::invalid_argument("bad layout arguments");
    std::vector<int64_t> bp(block_params, block_params + n_blocks);
    DpLayout L = dp_layout(bp, groups, world);
    for (int b = 0; b < n_blocks; ++b) block_off[b] = L.block_off[b];
    *n_groups = (int)L.group_lo.size();
    for (size_t g = 0; g < L.group_lo.size(); ++g) {
      group_lo[g] = L.group_lo[g];
      group_n[g] = L.group_n[g];
      shard_n[g] = L.shard_n[g];
    }
  });
}

int krt_peer_group_create(int world, krt_peer_group** out) {
  return guard([&] {
    if (world < 1 || !out) throw std::invalid_argument("bad peer group size");
    *out = reinterpret_cast<krt_peer_group*>(new PeerGroup(world));
  });
}

int krt_peer_group_destroy(krt_peer_group* g) {
  return guard([&] { delete reinterpret_cast<PeerGroup*>(g); });
}

int krt_nccl_unique_id(void* out) {
  return guard([&] {
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) throw std::runtime_error(std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out, &id, sizeof(id));
  });
}

int krt_plan_arena(const krt_plan* p, const size_t* block_bytes, int n_blocks, char** out_json) {
  return guard([&] {
    if ((int)p->plan.blocks.size() != n_blocks) throw std::invalid_argument("block count mismatch");
    std::map<int, size_t> bb;
    for (int i = 0; i < n_blocks; ++i) bb[i + 1] = (block_bytes[i] + 255) / 256 * 256;
    auto costs = plan_costs(p->plan, p->model, p->hw);
    auto base = build_engine_ops(p->plan, p->model, p->hw, costs);
    for (auto& e : base)
      if (!e.missing.empty()) throw Infeasible(e.missing);
    ArenaPlan ap = plan_arena(p->plan, p->model, p->hw, base, bb);
    std::ostringstream os;
    os << "{\"arena_bytes\": " << ap.arena_bytes << ", \"ledger_peak\": " << jnum(ap.ledger_peak)
       << ", \"instances\": [";
    for (size_t i = 0; i < ap.inst.size(); ++i) {
      auto& in = ap.inst[i];
      os << (i ? ", " : "") << "{\"block\": " << in.block << ", \"off\": " << in.off << ", \"bytes\": " << in.bytes
         << ", \"alloc_op\": " << in.alloc_op << ", \"free_op\": " << in.free_op << ", \"alloc_action\": \""
         << action_name(base[in.alloc_op].action) << "\"}";
    }
    os << "], \"deps\": [";
    bool first = true;
    for (size_t i = 0; i < ap.deps.size(); ++i)
      for (int d : ap.deps[i]) {
        os << (first ? "" : ", ") << "[" << i << ", " << d << "]";
        first = false;
      }
    os << "]}";
    *out_json = dup(os.str());
  });
}

int krt_create(const krt_config* cfg, krt_ctx** out) {
  return guard([&] {
    if (!cfg || !out) throw std::invalid_argument("null argument");
    auto c = std::make_unique<krt_ctx>();
    c->rt = std::make_unique<Runtime>(*cfg);
    *out = c.release();
  });
}

int krt_destroy(krt_ctx* ctx) {
  return guard([&] { delete ctx; });
}

int krt_register_block(krt_ctx* ctx, int block, size_t act_bytes, const int64_t* numel, int n) {
  return guard([&] {
    if (n > 0 && !numel) throw std::invalid_argument("null numel");
    ctx->rt->register_block(block, act_bytes, numel, n);
  });
}

int krt_prepare(krt_ctx* ctx, const krt_plan* plan) {
  return guard([&] {
    auto v = validate_plan(plan->plan, plan->model, plan->hw);
    if (!v.empty()) throw Infeasible("plan rejected by validate_plan: " + v[0]);
    ctx->rt->prepare(plan->plan, plan->model, plan->hw);
  });
}

int krt_region(krt_ctx* ctx, int which, int block, void** ptr, size_t* bytes) {
  return guard([&] { ctx->rt->region(which, block, ptr, bytes); });
}

int krt_stream(krt_ctx* ctx, int which, void** stream) {
  return guard([&] { *stream = (void*)ctx->rt->stream(which); });
}

int krt_block_slot(krt_ctx* ctx, int block, void** slot) {
  return guard([&] { *slot = ctx->rt->block_slot(block); });
}

int krt_init_master(krt_ctx* ctx) {
  return guard([&] { ctx->rt->init_master(); });
}

int krt_run_iteration(krt_ctx* ctx, krt_compute_cb cb, void* user) {
  return guard([&] {
    if (!cb) throw std::invalid_argument("null compute callback");
    ctx->rt->run_iteration(cb, user);
  });
}

int krt_synchronize(krt_ctx* ctx) {
  return guard([&] { ctx->rt->synchronize(); });
}

int krt_ipc_export(krt_ctx* ctx, void* out, size_t cap, size_t* len) {
  return guard([&] {
    auto h = ctx->rt->ipc_export();
    if (len) *len = h.size();
    if (cap < h.size()) throw std::invalid_argument("ipc handle buffer too small");
    std::memcpy(out, h.data(), h.size());
  });
}

int krt_ipc_import(krt_ctx* ctx, const void* handles, int world) {
  return guard([&] { ctx->rt->ipc_import(static_cast<const uint8_t*>(handles), world); });
}

int krt_probe_exchange(krt_ctx* ctx, size_t bytes, int iters, double* seconds) {
  return guard([&] { *seconds = ctx->rt->probe_exchange(bytes, iters); });
}

int krt_flush_weights(krt_ctx* ctx) {
  return guard([&] { ctx->rt->flush_weights(); });
}

int krt_trace_csv(krt_ctx* ctx, char** out) {
  return guard([&] { *out = dup(ctx->rt->trace_csv()); });
}

int krt_stats(krt_ctx* ctx, char** out) {
  return guard([&] { *out = dup(ctx->rt->stats_json()); });
}

int krt_checkpoint_save(krt_ctx* ctx, const char* path) {
  return guard([&] { ctx->rt->checkpoint_save(path); });
}

int krt_checkpoint_load(krt_ctx* ctx, const char* path) {
  return guard([&] { ctx->rt->checkpoint_load(path); });
}

int krt_read_master(krt_ctx* ctx, int block, float* out, size_t numel) {
  return guard([&] { ctx->rt->read_master(block, out, numel); });
}

int krt_reduce_cast(const float* const* in, int n_in, void* out, int out_dtype, size_t n, float scale,
                    void* stream) {
  return guard([&] {
    cudaError_t e = launch_reduce_cast(in, n_in, out, out_dtype, n, scale, (cudaStream_t)stream);
    if (e != cudaSuccess) throw std::runtime_error(std::string("reduce_cast: ") + cudaGetErrorString(e));
  });
}

size_t krt_bn_workspace_bytes(int C) { return bn_workspace_bytes(C); }

#define KRT_CUDA_GUARD(expr, what)                                                     \
  return guard([&] {                                                                   \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e_)); \
  })

int krt_bn_stats(const void* x, int64_t rows, int C, float eps, float* mean, float* invstd, void* ws, void* stream) {
  KRT_CUDA_GUARD(bn_stats(x, rows, C, eps, mean, invstd, ws, (cudaStream_t)stream), "bn_stats");
}

int krt_bn_stats_apply(const void* x, int64_t rows, int C, float eps, float* mean, float* invstd, const void* g,
                       const void* b, const void* res, int relu, void* y, void* ws, void* stream) {
  KRT_CUDA_GUARD(bn_stats_apply(x, rows, C, eps, mean, invstd, g, b, res, relu, y, ws, (cudaStream_t)stream),
                 "bn_stats_apply");
}

int krt_bn_apply(const void* x, const float* mean, const float* invstd, const void* g, const void* b,
                 const void* res, const float* rmean, const float* rinvstd, const void* rg, const void* rb, int relu,
                 void* y, int64_t rows, int C, void* stream) {
  KRT_CUDA_GUARD(bn_apply(x, mean, invstd, g, b, res, rmean, rinvstd, rg, rb, relu, y, rows, C, (cudaStream_t)stream),
                 "bn_apply");
}

int krt_bn_add_relu_bwd(const void* dy, const void* dy2, const void* x, const float* mean, const float* invstd,
                        const void* g, const void* b, const void* res, const float* rmean, const float* rinvstd,
                        const void* rg, const void* rb, void* dz, int64_t rows, int C, void* stream) {
  KRT_CUDA_GUARD(bn_add_relu_bwd(dy, dy2, x, mean, invstd, g, b, res, rmean, rinvstd, rg, rb, dz, rows, C,
                                 (cudaStream_t)stream),
                 "bn_add_relu_bwd");
}

int krt_bn_backward(const void* dy, const void* x, const float* mean, const float* invstd, const void* g,
                    const void* b, int relu, void* dx, float* dgamma, float* dbeta, int64_t rows, int C, void* ws,
                    const void* addend, void* stream) {
  KRT_CUDA_GUARD(bn_backward(dy, x, mean, invstd, g, b, relu, dx, dgamma, dbeta, rows, C, ws, addend,
                             (cudaStream_t)stream),
                 "bn_backward");
}

int krt_bn_add_relu_backward(const void* dy, const void* dy2, const void* x, const float* mean, const float* invstd,
                             const void* g, const void* b, const void* res, void* dz, void* dx, float* dgamma,
                             float* dbeta, int64_t rows, int C, void* ws, void* stream) {
  KRT_CUDA_GUARD(bn_add_relu_backward(dy, dy2, x, mean, invstd, g, b, res, dz, dx, dgamma, dbeta, rows, C, ws,
                                      (cudaStream_t)stream),
                 "bn_add_relu_backward");
}

int krt_bn_relu_maxpool(const void* x, const float* mean, const float* invstd, const void* g, const void* b, void* y,
                        int n, int h, int w, int c, int k, int s, int p, void* stream) {
  KRT_CUDA_GUARD(bn_relu_maxpool(x, mean, invstd, g, b, y, n, h, w, c, k, s, p, (cudaStream_t)stream),
                 "bn_relu_maxpool");
}

size_t krt_bn_relu_maxpool_bwd_workspace(int n, int h, int w, int c, int k, int s, int p) {
  return bn_relu_maxpool_bwd_workspace(n, h, w, c, k, s, p);
}

int krt_bn_relu_maxpool_bwd(const void* dy, const void* x, const float* mean, const float* invstd, const void* g,
                            const void* b, void* dx, void* ws, int n, int h, int w, int c, int k, int s, int p,
                            void* stream) {
  KRT_CUDA_GUARD(bn_relu_maxpool_bwd(dy, x, mean, invstd, g, b, dx, ws, n, h, w, c, k, s, p, (cudaStream_t)stream),
                 "bn_relu_maxpool_bwd");
}

size_t krt_conv1x1_partials_bytes(int N) { return conv1x1_partials_bytes(N); }

int krt_conv1x1_bn(const void* A, const void* B, void* C, int64_t M, int N, int K, const float* pmean,
                   const float* pinvstd, const void* pg, const void* pb, float* part, int* part_rows, void* stream) {
  KRT_CUDA_GUARD(conv1x1_bn_fprop(A, B, C, M, N, K, pmean, pinvstd, pg, pb, part, part_rows, (cudaStream_t)stream),
                 "conv1x1_bn");
}

int krt_conv1x1_bn_res(const void* A, const void* B, void* C, int64_t M, int N, int K, const float* pmean,
                       const float* pinvstd, const void* pg, const void* pb, const void* res, float* part,
                       int* part_rows, void* stream) {
  KRT_CUDA_GUARD(
      conv1x1_bn_res_fprop(A, B, C, M, N, K, pmean, pinvstd, pg, pb, res, part, part_rows, (cudaStream_t)stream),
      "conv1x1_bn_res");
}

int krt_pad_rgb4(const void* x, void* y, int64_t pixels, void* stream) {
  KRT_CUDA_GUARD(pad_rgb4(x, y, pixels, (cudaStream_t)stream), "pad_rgb4");
}

int krt_conv_gather_bn(const void* x, const void* wk, void* C, int n, int h, int w, int cin, int ho, int wo, int k,
                       int stride, int pad, int N, int K, float* part, int* part_rows, void* stream) {
  KRT_CUDA_GUARD(
      conv_gather_fprop(x, wk, C, n, h, w, cin, ho, wo, k, stride, pad, N, K, part, part_rows, (cudaStream_t)stream),
      "conv_gather_bn");
}

int krt_conv_im2col_bn(const void* x, const void* wk, void* C, int n, int h, int w, int cin, int ho, int wo, int k,
                       int stride, int pad, int N, const float* pmean, const float* pinvstd, const void* pgamma,
                       const void* pbeta, float* part, int* part_rows, const void* bx, const float* bmean,
                       const float* binvstd, const void* bgamma, const void* bbeta, void* stream) {
  KRT_CUDA_GUARD(conv_im2col_fprop(x, wk, C, n, h, w, cin, ho, wo, k, stride, pad, N, pmean, pinvstd, pgamma, pbeta,
                                   part, part_rows, bx, bmean, binvstd, bgamma, bbeta, (cudaStream_t)stream),
                 "conv_im2col_bn");
}

int krt_wgrad3x3_narrow_supported(int h, int w, int C) { return wgrad3x3_halo_supported(h, w, C) ? 1 : 0; }

size_t krt_wgrad3x3_narrow_workspace(int C) { return wgrad3x3_halo_workspace(C); }

int krt_wgrad3x3_narrow(const void* x, const void* dy, float* dw, int n, int h, int w, int C, const float* pmean,
                        const float* pinvstd, const void* pgamma, const void* pbeta, void* ws, size_t ws_bytes,
                        void* stream) {
  KRT_CUDA_GUARD(wgrad3x3_halo(x, dy, dw, n, h, w, C, pmean, pinvstd, pgamma, pbeta, ws, ws_bytes,
                               (cudaStream_t)stream),
                 "wgrad3x3_narrow");
}

size_t krt_stem_wgrad_workspace(void) { return stem_wgrad_workspace(); }

int krt_stem_wgrad(const void* x4, const void* dc, float* dw, int n, int h, int w, void* ws, size_t ws_bytes,
                   void* stream) {
  KRT_CUDA_GUARD(stem_wgrad(x4, dc, dw, n, h, w, ws, ws_bytes, (cudaStream_t)stream), "stem_wgrad");
}

int krt_wgrad1x1_narrow_supported(int ci, int co) { return wgrad1x1_narrow_supported(ci, co) ? 1 : 0; }

size_t krt_wgrad1x1_narrow_workspace(int ci, int co) { return wgrad1x1_narrow_workspace(ci, co); }

int krt_wgrad1x1_narrow(const void* x, const void* dy, float* dw, int64_t M, int ci, int co, const float* pmean,
                        const float* pinvstd, const void* pgamma, const void* pbeta, void* ws, size_t ws_bytes,
                        void* stream) {
  KRT_CUDA_GUARD(wgrad1x1_narrow(x, dy, dw, M, ci, co, pmean, pinvstd, pgamma, pbeta, ws, ws_bytes,
                                 (cudaStream_t)stream),
                 "wgrad1x1_narrow");
}

int krt_conv3x3_halo_supported(int h, int w, int cin, int N, int prologue) {
  return conv3x3_halo_supported(h, w, cin, N, prologue != 0) ? 1 : 0;
}

size_t krt_conv_wgrad_workspace_bytes(int n, int ho, int wo, int cout, int cin, int k) {
  return conv_wgrad_workspace_bytes(n, ho, wo, cout, cin, k);
}

int krt_conv_wgrad(const void* dy, const void* x, float* dw, int n, int h, int w, int cin, int ho, int wo, int cout,
                   int k, int stride, int pad, const float* pmean, const float* pinvstd, const void* pgamma,
                   const void* pbeta, void* ws, size_t ws_bytes, void* stream) {
  KRT_CUDA_GUARD(conv_wgrad(dy, x, dw, n, h, w, cin, ho, wo, cout, k, stride, pad, pmean, pinvstd, pgamma, pbeta, ws,
                            ws_bytes, (cudaStream_t)stream),
                 "conv_wgrad");
}

int krt_conv1x1_bn_dgrad(const void* dY, const void* Wt, void* dX, int64_t M, int N, int K, const void* x,
                         const float* mean, const float* invstd, const void* g, const void* b, float* part,
                         int* part_rows, void* stream) {
  KRT_CUDA_GUARD(conv1x1_bn_dgrad(dY, Wt, dX, M, N, K, x, mean, invstd, g, b, part, part_rows, (cudaStream_t)stream),
                 "conv1x1_bn_dgrad");
}

int krt_bn_partials_bwd_finalize(const float* part, int part_rows, int N, int64_t M, const float* mean,
                                 const float* invstd, const void* g, float* dgamma, float* dbeta, float* coef,
                                 void* stream) {
  KRT_CUDA_GUARD(bn_partials_bwd_finalize(part, part_rows, N, M, mean, invstd, g, dgamma, dbeta, coef,
                                          (cudaStream_t)stream),
                 "bn_partials_bwd_finalize");
}

int krt_bn_backward_elemt(const void* dy, const void* x, const float* mean, const float* invstd, const void* g,
                          const void* b, const float* coef, const void* addend, int relu, void* dx, int64_t rows,
                          int C, void* stream) {
  KRT_CUDA_GUARD(bn_backward_elemt(dy, x, mean, invstd, g, b, coef, addend, relu, dx, rows, C, (cudaStream_t)stream),
                 "bn_backward_elemt");
}

int krt_bn_partials_finalize(const float* part, int part_rows, int N, int64_t M, float eps, float* mean,
                             float* invstd, void* stream) {
  KRT_CUDA_GUARD(bn_partials_finalize(part, part_rows, N, M, eps, mean, invstd, (cudaStream_t)stream),
                 "bn_partials_finalize");
}

int krt_ln_fwd(const void* x, const void* r, void* x2, const void* g, const void* b, void* h, float* mean, float* rstd,
               int64_t T, int H, float eps, void* stream) {
  KRT_CUDA_GUARD(ln_fwd(x, r, x2, g, b, h, mean, rstd, T, H, eps, (cudaStream_t)stream), "ln_fwd");
}

size_t krt_ln_bwd_workspace(int64_t T, int H) { return ln_bwd_workspace(T, H); }

int krt_ln_bwd(const void* dy, const void* x, const void* g, const float* mean, const float* rstd, const void* addend,
               void* dx, float* dgamma, float* dbeta, void* ws, int64_t T, int H, void* stream) {
  KRT_CUDA_GUARD(ln_bwd(dy, x, g, mean, rstd, addend, dx, dgamma, dbeta, ws, T, H, (cudaStream_t)stream), "ln_bwd");
}

int krt_lm_xent(const void* logits, const int64_t* target, void* dlogits, float* row_loss, int64_t T, int V,
                float scale, void* stream) {
  KRT_CUDA_GUARD(lm_xent(logits, target, dlogits, row_loss, T, V, scale, (cudaStream_t)stream), "lm_xent");
}

int krt_attn_softmax_bwd(const float* S, const float* dP, const float* lse, const float* D, void* P, void* dS,
                         int64_t rows, int s, float scale, void* stream) {
  KRT_CUDA_GUARD(attn_softmax_bwd(S, dP, lse, D, P, dS, rows, s, scale, (cudaStream_t)stream), "attn_softmax_bwd");
}

size_t krt_gelu_bwd_colsum_workspace(int64_t T, int N) { return gelu_bwd_colsum_workspace(T, N); }

int krt_gelu_bwd_colsum(const void* dy, const void* f, void* dx, float* colsum, void* ws, int64_t T, int N,
                        void* stream) {
  KRT_CUDA_GUARD(gelu_bwd_colsum(dy, f, dx, colsum, ws, T, N, (cudaStream_t)stream), "gelu_bwd_colsum");
}

int krt_mlp_fc1_gelu(const void* x, const void* w1, const void* b1, void* f1, void* g, int64_t M, int64_t N,
                     int64_t K, void* stream) {
  return guard([&] { mlp_fc1_gelu(x, w1, b1, f1, g, M, N, K, (cudaStream_t)stream); });
}

int krt_mlp_fc2_residual(const void* g, const void* w2, const void* b2, const void* x2, void* y, int64_t M,
                         int64_t N, int64_t K, void* stream) {
  return guard([&] { mlp_fc2_residual(g, w2, b2, x2, y, M, N, K, (cudaStream_t)stream); });
}

int krt_linear_wgrad_bgrad(const void* dy, const void* x, float* dw, float* db, int64_t M, int64_t N, int64_t K,
                           void* stream) {
  return guard([&] { linear_wgrad_bgrad(dy, x, dw, db, M, N, K, (cudaStream_t)stream); });
}

int krt_mlp_fc2_dgelu(const void* dy, const void* w2, const void* f1, void* df1, int64_t M, int64_t N, int64_t K,
                      void* stream) {
  return guard([&] { mlp_fc2_dgelu(dy, w2, f1, df1, M, N, K, (cudaStream_t)stream); });
}

int krt_device_update(float* master, float* m, float* v, const float* grad, void* weights, int weight_dtype,
                      size_t n, int optimizer, float lr, float beta1, float beta2, float eps, float wd,
                      float momentum, int step, void* stream) {
  return guard([&] {
    OptimScalars s = make_scalars(optimizer, lr, beta1, beta2, eps, wd, momentum, step, 1.0f);
    cudaError_t e = launch_update(master, m, v, grad, weights, weight_dtype, n, s, (cudaStream_t)stream);
    if (e != cudaSuccess) throw std::runtime_error(std::string("device_update: ") + cudaGetErrorString(e));
  });
}

int krt_host_update(float* master, float* m, float* v, const float* grad, void* weights, int weight_dtype,
                    size_t n, int optimizer, float lr, float beta1, float beta2, float eps, float wd,
                    float momentum, int step, int threads) {
  return guard([&] {
    OptimScalars s = make_scalars(optimizer, lr, beta1, beta2, eps, wd, momentum, step, 1.0f);
    std::unique_ptr<ThreadPool> pool;
    if (threads > 1) pool = std::make_unique<ThreadPool>(threads);
    host_update(pool.get(), master, m, v, grad, weights, weight_dtype, n, s);
  });
}

}  // extern "C"
