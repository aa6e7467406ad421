#include "runtime.hpp"

#include <cstdio>
#include <cstring>

#include <cuda.h>
#include <cudaTypedefs.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <set>
#include <sstream>
#include <stdexcept>

#include "kernels.hpp"

namespace krt {
namespace {

constexpr size_t kAlign = 256;
size_t align_up(size_t x, size_t a = kAlign) { return (x + a - 1) / a * a; }

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define CK(call)                                                                                  \
  do {                                                                                            \
    cudaError_t e_ = (call);                                                                      \
    if (e_ != cudaSuccess)                                                                        \
      throw CudaError(std::string(#call) + ": " + cudaGetErrorString(e_));                        \
  } while (0)

#define NK(call)                                                                                  \
  do {                                                                                            \
    ncclResult_t r_ = (call);                                                                     \
    if (r_ != ncclSuccess) throw CudaError(std::string(#call) + ": " + ncclGetErrorString(r_));   \
  } while (0)

double host_now() {
  using namespace std::chrono;
  return duration<double>(steady_clock::now().time_since_epoch()).count();
}

size_t dtype_bytes(int dt) { return dt == KRT_BF16 ? 2 : 4; }

}  // namespace

void PeerGroup::mark(int rank, int kind, int group, int step) {
  {
    std::lock_guard<std::mutex> lk(mu);
    marks[{rank, kind, group}] = step;
  }
  cv.notify_all();
}

void PeerGroup::wait_all(int kind, int group, int step, double timeout_s) {
  std::unique_lock<std::mutex> lk(mu);
  auto ready = [&] {
    for (int r = 0; r < world; ++r) {
      auto it = marks.find({r, kind, group});
      if (it == marks.end() || it->second < step) return false;
    }
    return true;
  };
  if (!cv.wait_for(lk, std::chrono::duration<double>(timeout_s), ready)) {
    static const char* kinds[] = {"backward", "weight shard", "flush"};
    std::string missing;
    for (int r = 0; r < world; ++r) {
      auto it = marks.find({r, kind, group});
      if (it == marks.end() || it->second < step) missing += (missing.empty() ? "" : ", ") + std::to_string(r);
    }
    throw std::runtime_error("peer wait timed out after " + std::to_string(timeout_s) + " s: rank(s) " + missing +
                             " never issued the " + kinds[kind] + " of group " + std::to_string(group) +
                             " for iteration " + std::to_string(step));
  }
}

cudaEvent_t PeerGroup::event(int rank, int kind, int group) {
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_tuple(rank, kind, group);
  auto it = events.find(key);
  if (it != events.end()) return it->second;
  cudaEvent_t e;
  CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  events[key] = e;
  return e;
}

PeerGroup::~PeerGroup() {
  for (auto& kv : events) cudaEventDestroy(kv.second);
}

Runtime::Runtime(const krt_config& cfg) : cfg_(cfg) {
  world_ = std::max(1, cfg.world_size);
  rank_ = cfg.rank;
  if (rank_ < 0 || rank_ >= world_) throw std::invalid_argument("rank out of range");
  if (cfg.weight_dtype != KRT_F32 && cfg.weight_dtype != KRT_BF16)
    throw std::invalid_argument("weight_dtype must be KRT_F32 or KRT_BF16");
  CK(cudaSetDevice(cfg.device));
  int lo = 0, hi = 0;
  CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  // compute at normal priority; copies and the collective at high priority so
  // their short control work is never queued behind long kernels
  CK(cudaStreamCreateWithPriority(&streams_[0], cudaStreamNonBlocking, lo));
  for (int i = 1; i < 4; ++i) CK(cudaStreamCreateWithPriority(&streams_[i], cudaStreamNonBlocking, hi));
  CK(cudaEventCreate(&ev_base_));
  CK(cudaStreamCreateWithPriority(&clock_stream_, cudaStreamNonBlocking, hi));
  if (const char* w = std::getenv("KRT_WATCHDOG_S")) {
    double v = std::atof(w);
    if (v > 0) watchdog_s_ = v;
  }
  dp_ = world_ > 1 || cfg.force_dp_path;
  ipc_ = dp_ && cfg.ipc_exchange;
  if (ipc_ && cfg.peer_group) throw std::invalid_argument("choose one of peer_group and ipc_exchange");
  if (ipc_) {
    // peers connect after prepare (krt_ipc_export / krt_ipc_import)
  } else if (dp_ && cfg.peer_group) {
    peers_ = static_cast<PeerGroup*>(cfg.peer_group);
    if (peers_->world != world_) throw std::invalid_argument("peer group size != world_size");
    std::lock_guard<std::mutex> lk(peers_->mu);
    if (peers_->ranks[rank_]) throw std::invalid_argument("rank already joined the peer group");
    peers_->ranks[rank_] = this;
  } else if (dp_) {
    ncclUniqueId id;
    if (cfg.nccl_id) std::memcpy(&id, cfg.nccl_id, sizeof(id));
    else if (world_ == 1) NK(ncclGetUniqueId(&id));   // a one-rank communicator
    else throw std::invalid_argument("world_size > 1 needs nccl_id or a peer group");
    ncclComm_t comm;
    NK(ncclCommInitRank(&comm, world_, id, rank_));
    nccl_comm_ = comm;
  }
  int nt = cfg.host_threads;
  if (nt <= 0) nt = std::max(1, (int)std::thread::hardware_concurrency() - 2);
  pool_ = std::make_unique<ThreadPool>(nt);
  host_thread_ = std::thread([this] { host_loop(); });
}

Runtime::~Runtime() {
  {
    std::lock_guard<std::mutex> lk(hmu_);
    hstop_ = true;
  }
  hcv_.notify_all();
  if (host_thread_.joinable()) host_thread_.join();
  cudaSetDevice(cfg_.device);
  for (auto s : streams_)
    if (s) cudaStreamSynchronize(s);
  if (nccl_comm_) ncclCommDestroy((ncclComm_t)nccl_comm_);
  if (peers_) {
    std::lock_guard<std::mutex> lk(peers_->mu);
    peers_->ranks[rank_] = nullptr;
  }
  for (auto e : ev_start_) cudaEventDestroy(e);
  for (auto e : ev_done_) cudaEventDestroy(e);
  if (ev_base_) cudaEventDestroy(ev_base_);
  cudaFree(d_arena_);
  cudaFree(d_weights_);
  cudaFree(d_grads_);
  cudaFree(d_pack_);
  cudaFree(d_pack_shard_);
  cudaFree(d_master_);
  cudaFree(d_m_);
  cudaFree(d_v_);
  cudaFree(d_shard_);
  for (int p = 0; p < (int)ipc_w_.size(); ++p)
    if (p != rank_) {
      if (ipc_w_[p]) cudaIpcCloseMemHandle(ipc_w_[p]);
      if (ipc_g_[p]) cudaIpcCloseMemHandle(ipc_g_[p]);
      if (ipc_flags_[p]) cudaIpcCloseMemHandle(ipc_flags_[p]);
    }
  cudaFree(d_flags_);
  cudaFreeHost(h_swap_);
  cudaFreeHost(h_grad_);
  cudaFreeHost(h_wstage_);
  for (auto s : streams_)
    if (s) cudaStreamDestroy(s);
  if (clock_stream_) {
    cudaStreamSynchronize(clock_stream_);
    cudaStreamDestroy(clock_stream_);
  }
}

void Runtime::register_block(int block, size_t act_bytes, const int64_t* numel, int n) {
  if (prepared_) throw std::logic_error("register_block after prepare");
  if (block < 1) throw std::invalid_argument("block ids start at 1");
  BlockPhys b;
  b.act_bytes = align_up(act_bytes);
  for (int i = 0; i < n; ++i) {
    if (numel[i] < 0) throw std::invalid_argument("negative numel");
    b.numel.push_back(numel[i]);
    b.n_params += numel[i];
  }
  blocks_[block] = b;
}

void* Runtime::d_weight(int64_t p_off) const {
  return static_cast<uint8_t*>(d_weights_) + (size_t)p_off * dtype_bytes(cfg_.weight_dtype);
}

// ---------------------------------------------------------------------------
// op DAG
// ---------------------------------------------------------------------------
void Runtime::build_ops(const Plan& plan, const Model& model, const Hardware& hw) {
  auto costs = plan_costs(plan, model, hw);
  std::vector<EngineOp> base = build_engine_ops(plan, model, hw, costs);
  for (auto& e : base)
    if (!e.missing.empty()) throw std::runtime_error(e.missing);

  // --- static arena assignment from the base ledger (simulator.py:67-135) ---
  std::map<int, size_t> bb;
  for (auto& [id, bp] : blocks_) bb[id] = bp.act_bytes;
  ArenaPlan ap = plan_arena(plan, model, hw, base, bb);
  ledger_peak_ = (size_t)ap.ledger_peak;
  arena_bytes_ = ap.arena_bytes;
  instances_.clear();
  for (auto& a : ap.inst) {
    Instance in;
    in.block = a.block;
    in.off = a.off;
    in.bytes = a.bytes;
    in.alloc_op = a.alloc_op;
    in.free_op = a.free_op;
    instances_.push_back(in);
  }
  const std::vector<int>& inst_of_alloc = ap.inst_of_alloc;
  const std::vector<int>& inst_read = ap.inst_read;
  const std::vector<std::vector<int>>& arena_deps = ap.deps;
  if (arena_bytes_ == 0) arena_bytes_ = kAlign;

  // --- executor op lists: DP pipeline around the base ops -------------------
  auto groups = assign_groups(nb_, cfg_.dist_groups);
  groups_.clear();
  std::set<int> host_blocks;
  if (dp_ || cfg_.host_path_all)
    for (auto& b : plan.blocks) host_blocks.insert(b.id);
  else
    for (int b : plan.swapped_blocks()) host_blocks.insert(b);
  for (auto& [id, bp] : blocks_) {
    bp.host_path = host_blocks.count(id) > 0;
    bp.swapped = false;
  }
  for (int b : plan.swapped_blocks()) blocks_.at(b).swapped = true;
  std::vector<int64_t> bparams;
  for (int b = 1; b <= nb_; ++b) bparams.push_back(blocks_.at(b).n_params);
  DpLayout lay = dp_layout(bparams, cfg_.dist_groups, world_);
  for (size_t gi = 0; gi < groups.size(); ++gi) {
    GroupPhys g;
    g.members = groups[gi];
    g.p_lo = lay.group_lo[gi];
    g.p_n = lay.group_n[gi];
    g.shard_n = lay.shard_n[gi];
    for (int b : g.members) {
      blocks_.at(b).p_off = lay.block_off[b - 1];
      blocks_.at(b).group = (int)gi + 1;
      g.host |= blocks_.at(b).host_path;
    }
    groups_.push_back(g);
  }
  int64_t off = lay.total;
  total_params_ = off;
  // gradient ring: R group-sized slots instead of a whole-model region
  if (cfg_.grad_slots < 0) throw std::invalid_argument("grad_slots must be >= 0");
  grad_ring_ = (cfg_.grad_slots > 0 && cfg_.grad_slots < (int)groups_.size()) ? cfg_.grad_slots : 0;
  if (grad_ring_ && (peers_ || cfg_.ipc_exchange))
    throw std::invalid_argument("grad_slots needs the NCCL exchange: peers read a rank's gradient slot directly "
                                "over in-process / IPC exchange, with no completion signal to reuse it on");
  grad_slot_off_.assign(groups_.size(), 0);
  int64_t slot = 0;
  for (auto& g : groups_) slot = std::max(slot, g.p_n);
  slot = (slot + 63) / 64 * 64;
  if (slot * grad_ring_ >= total_params_) grad_ring_ = 0;   // a ring not smaller than the whole-model region
  if (grad_ring_) {
    for (size_t gi = 0; gi < groups_.size(); ++gi) grad_slot_off_[gi] = (int64_t)(gi % grad_ring_) * slot;
    grad_elems_ = slot * grad_ring_;
  } else {
    for (size_t gi = 0; gi < groups_.size(); ++gi) grad_slot_off_[gi] = groups_[gi].p_lo;
    grad_elems_ = total_params_;
  }
  for (size_t gi = 0; gi < groups_.size(); ++gi)
    group_first_block_[(int)gi + 1] = *std::min_element(groups_[gi].members.begin(), groups_[gi].members.end());
  // host state layout
  host_elems_ = 0;
  for (auto& g : groups_) {
    g.host_off = host_elems_;
    if (dp_) g.host_n = g.shard_n;
    else {
      g.host_n = 0;
      for (int b : g.members)
        if (blocks_.at(b).host_path) g.host_n += (blocks_.at(b).n_params + 63) / 64 * 64;
    }
    host_elems_ += g.host_n;
  }

  double swap_rate = hw.swap_throughput();
  double net_rate = 700e9, host_rate = hw.host_update_rate;
  auto make_list = [&](bool steady, std::vector<XOp>& out) {
    out.clear();
    std::map<int, int> weight_in_of;  // block -> op
    if (steady) {
      if (dp_) {
        for (size_t gi = 0; gi < groups_.size(); ++gi) {
          XOp x;
          x.e.action = Action::WEIGHT_IN;
          x.e.group = (int)gi + 1;
          x.e.block = -1;
          x.e.res = hw.duplex ? R_XFER_IN : R_XFER;
          x.e.duration = groups_[gi].shard_n * dtype_bytes(cfg_.weight_dtype) / swap_rate;
          x.prev_host_group = (int)gi + 1;
          for (int b : groups_[gi].members) weight_in_of[b] = (int)out.size();
          out.push_back(x);
        }
      } else {
        for (int b : host_blocks) {
          XOp x;
          x.e.action = Action::WEIGHT_IN;
          x.e.block = b;
          x.e.group = blocks_.at(b).group;
          x.e.res = hw.duplex ? R_XFER_IN : R_XFER;
          x.e.duration = blocks_.at(b).n_params * dtype_bytes(cfg_.weight_dtype) / swap_rate;
          x.prev_host_group = blocks_.at(b).group;
          weight_in_of[b] = (int)out.size();
          out.push_back(x);
        }
      }
    }
    int offset = (int)out.size();
    std::map<int, int> bw_done;
    for (size_t i = 0; i < base.size(); ++i) {
      XOp x;
      x.e = base[i];
      for (auto& d : x.e.deps) d += offset;
      if (x.e.gate >= 0) x.e.gate += offset;
      for (int d : arena_deps[i]) x.e.deps.push_back(d + offset);
      x.instance = inst_of_alloc[i];
      x.reads_instance = inst_read[i];
      if (x.e.action == Action::FW && weight_in_of.count(x.e.block)) x.e.deps.push_back(weight_in_of[x.e.block]);
      if (x.e.action == Action::BW) bw_done[x.e.block] = (int)out.size();
      out.push_back(x);
    }
    int out_res = hw.duplex ? R_XFER_OUT : R_XFER;
    if (dp_) {
      for (int gi = (int)groups_.size(); gi >= 1; --gi) {
        auto& g = groups_[gi - 1];
        XOp ex;
        ex.e.action = Action::EXCHANGE;
        ex.e.group = gi;
        ex.e.block = -1;
        ex.e.res = R_NETWORK;
        ex.e.duration = g.p_n * 4.0 / net_rate;
        for (int b : g.members) ex.e.deps.push_back(bw_done.at(b));
        int ex_idx = (int)out.size();
        out.push_back(ex);
        XOp go;
        go.e.action = Action::GRAD_OUT;
        go.e.group = gi;
        go.e.block = -1;
        go.e.res = out_res;
        go.e.duration = g.shard_n * 4.0 / swap_rate;
        go.e.deps = {ex_idx};
        int go_idx = (int)out.size();
        out.push_back(go);
        XOp hu;
        hu.e.action = Action::HOST_UPDATE;
        hu.e.group = gi;
        hu.e.block = -1;
        hu.e.res = R_HOST;
        hu.e.duration = g.host_n / host_rate;
        hu.e.deps = {go_idx};
        out.push_back(hu);
      }
    } else {
      std::map<int, int> go_of;
      for (auto it = host_blocks.rbegin(); it != host_blocks.rend(); ++it) {
        int b = *it;
        XOp go;
        go.e.action = Action::GRAD_OUT;
        go.e.block = b;
        go.e.group = blocks_.at(b).group;
        go.e.res = out_res;
        go.e.duration = blocks_.at(b).n_params * 4.0 / swap_rate;
        go.e.deps = {bw_done.at(b)};
        go_of[b] = (int)out.size();
        out.push_back(go);
      }
      for (int gi = (int)groups_.size(); gi >= 1; --gi) {
        auto& g = groups_[gi - 1];
        if (!g.host) continue;
        XOp hu;
        hu.e.action = Action::HOST_UPDATE;
        hu.e.group = gi;
        hu.e.block = -1;
        hu.e.res = R_HOST;
        hu.e.duration = g.host_n / host_rate;
        for (int b : g.members)
          if (go_of.count(b)) hu.e.deps.push_back(go_of[b]);
        out.push_back(hu);
      }
    }
  };
  // gradient ring: group g's backward overwrites the slot group g + R used
  // earlier in the same backward pass, so it waits until that gradient was
  // consumed (exchange, grad_out or the device update in its bw)
  auto ring_deps = [&](std::vector<XOp>& out) {
    if (!grad_ring_) return;
    std::map<int, std::vector<int>> release_of;
    for (size_t i = 0; i < out.size(); ++i) {
      const EngineOp& e = out[i].e;
      if (dp_ && e.action == Action::EXCHANGE) release_of[e.group].push_back((int)i);
      if (!dp_ && e.action == Action::GRAD_OUT) release_of[blocks_.at(e.block).group].push_back((int)i);
      if (!dp_ && e.action == Action::BW && !blocks_.at(e.block).host_path)
        release_of[blocks_.at(e.block).group].push_back((int)i);
    }
    int ng = (int)groups_.size();
    for (size_t i = 0; i < out.size(); ++i) {
      EngineOp& e = out[i].e;
      if (e.action != Action::BW) continue;
      int g = blocks_.at(e.block).group;
      if (g + grad_ring_ > ng) continue;
      for (int r : release_of[g + grad_ring_]) e.deps.push_back(r);
    }
  };
  make_list(false, ops_first_);
  make_list(true, ops_steady_);
  ring_deps(ops_first_);
  ring_deps(ops_steady_);
  auto order_of = [&](std::vector<XOp>& ops, std::vector<int>& order) {
    std::vector<EngineOp> eo;
    for (auto& x : ops) eo.push_back(x.e);
    auto res = base_resources(hw);
    res.push_back(R_NETWORK);
    res.push_back(R_HOST);
    EngineResult r = run_engine(eo, res, hw.capacity_bytes, false);
    if (r.deadlock) throw std::runtime_error("executor op DAG deadlocks: " + (r.blocked.empty() ? std::string() : r.blocked[0]));
    order = r.start_order;
  };
  order_of(ops_first_, order_first_);
  order_of(ops_steady_, order_steady_);
}

void Runtime::prepare(const Plan& plan, const Model& model, const Hardware& hw) {
  if (prepared_) throw std::logic_error("prepare called twice");
  nb_ = (int)plan.blocks.size();
  for (auto& b : plan.blocks) {
    auto it = blocks_.find(b.id);
    if (it == blocks_.end()) throw std::invalid_argument("block " + std::to_string(b.id) + " not registered");
    if ((double)it->second.act_bytes > b.swap_bytes + 0.5)
      throw std::invalid_argument("block " + std::to_string(b.id) + " stores " + std::to_string(it->second.act_bytes) +
                                  " B but the plan budgets " + py_g(b.swap_bytes) + " B");
  }
  if ((int)blocks_.size() != nb_) throw std::invalid_argument("registered blocks do not match the plan");
  build_ops(plan, model, hw);
  allocate();
  prepared_ = true;
}

void Runtime::allocate() {
  CK(cudaSetDevice(cfg_.device));
  arena_bytes_ = align_up(arena_bytes_ + cfg_.arena_slack_bytes, (size_t)2 << 20);
  CK(cudaMalloc(&d_arena_, arena_bytes_));
  size_t wb = dtype_bytes(cfg_.weight_dtype);
  size_t np = (size_t)std::max<int64_t>(total_params_, 64);
  CK(cudaMalloc(&d_weights_, np * wb));
  CK(cudaMemset(d_weights_, 0, np * wb));
  size_t ng = (size_t)std::max<int64_t>(grad_elems_, 64);
  CK(cudaMalloc((void**)&d_grads_, ng * 4));
  CK(cudaMemset(d_grads_, 0, ng * 4));
  // device optimizer state for blocks that never take the host path (P = 1)
  bool any_dev = false;
  for (auto& [id, b] : blocks_) any_dev |= !b.host_path;
  if (any_dev) {
    if (cfg_.weight_dtype == KRT_BF16) {
      CK(cudaMalloc((void**)&d_master_, np * 4));
      CK(cudaMemset(d_master_, 0, np * 4));
    }
    CK(cudaMalloc((void**)&d_m_, np * 4));
    CK(cudaMemset(d_m_, 0, np * 4));
    CK(cudaMalloc((void**)&d_v_, np * 4));
    CK(cudaMemset(d_v_, 0, np * 4));
  }
  if (dp_) {
    size_t ns = 0;
    for (auto& g : groups_) ns += (size_t)g.shard_n;
    CK(cudaMalloc((void**)&d_shard_, std::max<size_t>(ns, 64) * 4));
    if (cfg_.exchange_bf16) {
      if (peers_ || ipc_) throw std::invalid_argument("exchange_bf16 is the NCCL exchange's pack");
      size_t gp = 64, gs = 64;
      for (auto& g : groups_) {
        gp = std::max(gp, (size_t)g.p_n);
        gs = std::max(gs, (size_t)g.shard_n);
      }
      CK(cudaMalloc(&d_pack_, gp * 2));
      CK(cudaMalloc(&d_pack_shard_, gs * 2));
    }
  }
  if (ipc_) {
    size_t nf = (size_t)3 * groups_.size() * world_;
    CK(cudaMalloc((void**)&d_flags_, std::max<size_t>(nf, 1) * 4));
    CK(cudaMemset(d_flags_, 0, std::max<size_t>(nf, 1) * 4));
  }
  // pinned host: swap area + gradient landing + weight staging
  h_swap_bytes_ = 0;
  for (auto& [id, b] : blocks_)
    if (b.swapped) {
      b.host_swap_off = h_swap_bytes_;
      h_swap_bytes_ += b.act_bytes;
    }
  if (h_swap_bytes_) CK(cudaHostAlloc((void**)&h_swap_, h_swap_bytes_, cudaHostAllocDefault));
  size_t he = std::max<size_t>(host_elems_, 64);
  CK(cudaHostAlloc((void**)&h_grad_, he * 4, cudaHostAllocDefault));
  CK(cudaHostAlloc(&h_wstage_, he * wb, cudaHostAllocDefault));
  h_master_.assign(he, 0.f);
  h_m_.assign(he, 0.f);
  h_v_.assign(he, 0.f);
  size_t nev = std::max(ops_first_.size(), ops_steady_.size());
  ev_start_.resize(nev);
  ev_done_.resize(nev);
  for (size_t i = 0; i < nev; ++i) {
    CK(cudaEventCreate(&ev_start_[i]));
    CK(cudaEventCreate(&ev_done_[i]));
  }
}

void Runtime::region(int which, int block, void** ptr, size_t* bytes) {
  if (!prepared_) throw std::logic_error("region before prepare");
  size_t wb = dtype_bytes(cfg_.weight_dtype);
  switch (which) {
    case KRT_REGION_WEIGHTS: {
      auto& b = blocks_.at(block);
      *ptr = d_weight(b.p_off);
      *bytes = (size_t)b.n_params * wb;
      return;
    }
    case KRT_REGION_GRADS: {
      auto& b = blocks_.at(block);
      *ptr = d_grad_block(block);
      *bytes = (size_t)b.n_params * 4;
      return;
    }
    case KRT_REGION_ARENA:
      *ptr = d_arena_;
      *bytes = arena_bytes_;
      return;
    case KRT_REGION_HOST_SWAP: {
      auto& b = blocks_.at(block);
      *ptr = b.swapped ? h_swap_ + b.host_swap_off : nullptr;
      *bytes = b.swapped ? b.act_bytes : 0;
      return;
    }
  }
  throw std::invalid_argument("unknown region");
}

cudaStream_t Runtime::stream(int which) const {
  if (which < 0 || which > 3) throw std::invalid_argument("stream index 0..3");
  return streams_[which];
}

// host element offset of a block's state (P = 1 host path)
static int64_t host_block_off(const std::map<int, BlockPhys>& blocks, const GroupPhys& g, int block) {
  int64_t o = (int64_t)g.host_off;
  for (int b : g.members) {
    if (b == block) return o;
    if (blocks.at(b).host_path) o += (blocks.at(b).n_params + 63) / 64 * 64;
  }
  return -1;
}

void Runtime::init_master() {
  if (!prepared_) throw std::logic_error("init_master before prepare");
  CK(cudaSetDevice(cfg_.device));
  CK(cudaDeviceSynchronize());
  size_t wb = dtype_bytes(cfg_.weight_dtype);
  std::vector<uint8_t> tmp;
  auto fetch_f32 = [&](int64_t p_off, int64_t n, float* dst) {
    tmp.resize((size_t)n * wb);
    CK(cudaMemcpy(tmp.data(), d_weight(p_off), (size_t)n * wb, cudaMemcpyDeviceToHost));
    if (cfg_.weight_dtype == KRT_BF16) {
      const uint16_t* s = reinterpret_cast<const uint16_t*>(tmp.data());
      for (int64_t i = 0; i < n; ++i) {
        uint32_t u = (uint32_t)s[i] << 16;
        std::memcpy(&dst[i], &u, 4);
      }
    } else {
      std::memcpy(dst, tmp.data(), (size_t)n * 4);
    }
  };
  std::fill(h_m_.begin(), h_m_.end(), 0.f);
  std::fill(h_v_.begin(), h_v_.end(), 0.f);
  for (auto& g : groups_) {
    if (dp_) {
      fetch_f32(g.p_lo + (int64_t)rank_ * g.shard_n, g.shard_n, h_master_.data() + g.host_off);
    } else {
      for (int b : g.members) {
        auto& bp = blocks_.at(b);
        if (!bp.host_path) continue;
        int64_t ho = host_block_off(blocks_, g, b);
        fetch_f32(bp.p_off, bp.n_params, h_master_.data() + ho);
      }
    }
  }
  if (d_m_) {
    size_t np = (size_t)std::max<int64_t>(total_params_, 64);
    CK(cudaMemset(d_m_, 0, np * 4));
    CK(cudaMemset(d_v_, 0, np * 4));
    if (d_master_) {
      std::vector<float> f((size_t)total_params_);
      fetch_f32(0, total_params_, f.data());
      CK(cudaMemcpy(d_master_, f.data(), (size_t)total_params_ * 4, cudaMemcpyHostToDevice));
    }
  }
  step_ = 0;
  last_first_ = true;
}

// ---------------------------------------------------------------------------
// host update thread (the HOST resource, FIFO like run_engine's queue)
// ---------------------------------------------------------------------------
void Runtime::host_loop() {
  for (;;) {
    HostTask t;
    {
      std::unique_lock<std::mutex> lk(hmu_);
      hcv_.wait(lk, [&] { return hstop_ || !hq_.empty(); });
      if (hstop_ && hq_.empty()) return;
      t = hq_.front();
      hq_.pop_front();
    }
    double t0 = host_now();
    std::string err;
    try {
      for (auto e : t.waits)
        wait_event_bounded(e, "host_update of group " + std::to_string(t.group) + " (iteration " +
                                  std::to_string(t.step) + ") waiting for its grad_out");
      t0 = host_now();
      run_host_task(t);
    } catch (const std::exception& ex) {
      err = ex.what();
    }
    double t1 = host_now();
    {
      std::lock_guard<std::mutex> lk(hmu_);
      if (!err.empty() && host_error_.empty()) host_error_ = err;
      host_done_step_[t.group] = t.step;
      host_times_[{t.group, t.step}] = {t0, t1};
    }
    hcv_.notify_all();
  }
}

void Runtime::run_host_task(const HostTask& t) {
  auto& g = groups_.at((size_t)t.group - 1);
  OptimScalars s = make_scalars(cfg_.optimizer, cfg_.lr, cfg_.beta1, cfg_.beta2, cfg_.eps, cfg_.weight_decay,
                                cfg_.momentum, t.step, dp_ ? cfg_.grad_scale : 1.0f);
  size_t wb = dtype_bytes(cfg_.weight_dtype);
  auto stage_ptr = [&](size_t host_off) { return static_cast<uint8_t*>(h_wstage_) + host_off * wb; };
  if (dp_) {
    size_t o = g.host_off;
    host_update(pool_.get(), h_master_.data() + o, h_m_.data() + o, h_v_.data() + o, h_grad_ + o, stage_ptr(o),
                cfg_.weight_dtype, (size_t)g.host_n, s);
  } else {
    for (int b : g.members) {
      auto& bp = blocks_.at(b);
      if (!bp.host_path) continue;
      size_t o = (size_t)host_block_off(blocks_, g, b);
      host_update(pool_.get(), h_master_.data() + o, h_m_.data() + o, h_v_.data() + o, h_grad_ + o, stage_ptr(o),
                  cfg_.weight_dtype, (size_t)bp.n_params, s);
    }
  }
}

void Runtime::wait_host_done(int group, int step) {
  std::unique_lock<std::mutex> lk(hmu_);
  auto done = [&] {
    auto it = host_done_step_.find(group);
    return !host_error_.empty() || (it != host_done_step_.end() && it->second >= step);
  };
  if (!hcv_.wait_for(lk, std::chrono::duration<double>(watchdog_s_), done))
    throw std::runtime_error("watchdog: host_update of group " + std::to_string(group) + " for iteration " +
                             std::to_string(step) + " not complete after " + std::to_string(watchdog_s_) + " s (" +
                             std::to_string(hq_.size()) + " host tasks queued)");
  if (!host_error_.empty()) throw std::runtime_error("host update failed: " + host_error_);
}

void Runtime::wait_event_bounded(cudaEvent_t e, const std::string& what) const {
  const double t_end = host_now() + watchdog_s_;
  int spins = 0;
  for (;;) {
    cudaError_t r = cudaEventQuery(e);
    if (r == cudaSuccess) return;
    if (r != cudaErrorNotReady) throw CudaError(what + ": " + cudaGetErrorString(r));
    if (host_now() > t_end)
      throw std::runtime_error("watchdog: " + what + " not complete after " + std::to_string(watchdog_s_) + " s");
    if (++spins < 64) std::this_thread::yield();
    else std::this_thread::sleep_for(std::chrono::microseconds(spins < 1024 ? 20 : 500));
  }
}

std::string Runtime::first_pending_op() {
  auto& ops = last_first_ ? ops_first_ : ops_steady_;
  auto& order = last_first_ ? order_first_ : order_steady_;
  for (int idx : order) {
    const EngineOp& e = ops[idx].e;
    if (e.action == Action::HOST_UPDATE) continue;
    if (cudaEventQuery(ev_done_[idx]) == cudaErrorNotReady) {
      std::string s = std::string(action_name(e.action));
      if (e.block > 0) s += " block " + std::to_string(e.block);
      if (e.group > 0) s += " group " + std::to_string(e.group);
      return s + " on " + res_name(e.res);
    }
  }
  return "no device op (host side)";
}

void Runtime::fail_iteration(int step, const std::string& why) {
  // drain what was issued (errors ignored: the device may be the cause)
  for (auto s : streams_) cudaStreamSynchronize(s);
  {
    std::unique_lock<std::mutex> lk(hmu_);
    hcv_.wait_for(lk, std::chrono::duration<double>(watchdog_s_), [&] { return hq_.empty(); });
  }
  if (!iter_mutated_) {
    step_ = step - 1;  // nothing of this iteration was applied: it can be re-run
    last_first_ = step_ <= 0 || last_first_;
  } else {
    failed_ = "iteration " + std::to_string(step) + " failed after updates were applied: " + why;
  }
}

// ---------------------------------------------------------------------------
// issue
// ---------------------------------------------------------------------------
void Runtime::wait_deps(cudaStream_t s, const XOp& x, const std::vector<XOp>& ops) {
  (void)ops;
  for (int d : x.e.deps) CK(cudaStreamWaitEvent(s, ev_done_[d], 0));
  if (x.e.gate >= 0) CK(cudaStreamWaitEvent(s, ev_start_[x.e.gate], 0));
}

void Runtime::issue(int idx, std::vector<XOp>& ops, krt_compute_cb cb, void* user, int step) {
  XOp& x = ops[idx];
  const EngineOp& e = x.e;
  size_t wb = dtype_bytes(cfg_.weight_dtype);
  switch (e.action) {
    case Action::FW:
    case Action::RECOMPUTE_FW:
    case Action::BW: {
      cudaStream_t s = streams_[0];
      wait_deps(s, x, ops);
      int inst = e.action == Action::BW ? x.reads_instance : x.instance;
      auto& in = instances_.at(inst);
      CK(cudaEventRecord(ev_start_[idx], s));
      cur_slot_[e.block] = d_arena_ + in.off;
      int rc = cb(user, (int)e.action, e.block, d_arena_ + in.off, in.bytes, (void*)s);
      if (rc != 0)
        throw std::runtime_error(std::string("compute callback failed for ") + action_name(e.action) + " block " +
                                 std::to_string(e.block));
      if (e.action == Action::BW) {
        auto& bp = blocks_.at(e.block);
        if (!bp.host_path && bp.n_params > 0) {
          iter_mutated_ = true;
          OptimScalars sc = make_scalars(cfg_.optimizer, cfg_.lr, cfg_.beta1, cfg_.beta2, cfg_.eps,
                                         cfg_.weight_decay, cfg_.momentum, step, 1.0f);
          float* master = d_master_ ? d_master_ + bp.p_off : reinterpret_cast<float*>(d_weight(bp.p_off));
          CK(launch_update(master, d_m_ + bp.p_off, d_v_ + bp.p_off, d_grad_block(e.block), d_weight(bp.p_off),
                           cfg_.weight_dtype, (size_t)bp.n_params, sc, s));
          ++kernel_launches_;
          ++iter_launches_;
        }
      }
      CK(cudaEventRecord(ev_done_[idx], s));
      if ((peers_ || ipc_) && e.action == Action::BW) {
        int gi = blocks_.at(e.block).group;
        if (group_first_block_.at(gi) == e.block) {  // last backward of the group
          if (ipc_) {
            ipc_signal(s, PK_BW, gi, (uint32_t)step);
          } else {
            CK(cudaEventRecord(peers_->event(rank_, PK_BW, gi), s));
            peers_->mark(rank_, PK_BW, gi, step);
          }
        }
      }
      return;
    }
    case Action::SWAP_OUT: {
      cudaStream_t s = streams_[2];
      wait_deps(s, x, ops);
      auto& in = instances_.at(x.reads_instance);
      auto& bp = blocks_.at(e.block);
      CK(cudaEventRecord(ev_start_[idx], s));
      CK(cudaMemcpyAsync(h_swap_ + bp.host_swap_off, d_arena_ + in.off, in.bytes, cudaMemcpyDeviceToHost, s));
      CK(cudaEventRecord(ev_done_[idx], s));
      iter_bytes_d2h_ += in.bytes;
      return;
    }
    case Action::SWAP_IN: {
      cudaStream_t s = streams_[1];
      wait_deps(s, x, ops);
      auto& in = instances_.at(x.instance);
      auto& bp = blocks_.at(e.block);
      CK(cudaEventRecord(ev_start_[idx], s));
      CK(cudaMemcpyAsync(d_arena_ + in.off, h_swap_ + bp.host_swap_off, in.bytes, cudaMemcpyHostToDevice, s));
      cur_slot_[e.block] = d_arena_ + in.off;
      CK(cudaEventRecord(ev_done_[idx], s));
      iter_bytes_h2d_ += in.bytes;
      return;
    }
    case Action::GRAD_OUT: {
      cudaStream_t s = streams_[2];
      wait_deps(s, x, ops);
      CK(cudaEventRecord(ev_start_[idx], s));
      if (dp_) {
        auto& g = groups_.at((size_t)e.group - 1);
        size_t shard_pos = 0;
        for (int gi = 0; gi < e.group - 1; ++gi) shard_pos += (size_t)groups_[gi].shard_n;
        CK(cudaMemcpyAsync(h_grad_ + g.host_off, d_shard_ + shard_pos, (size_t)g.shard_n * 4,
                           cudaMemcpyDeviceToHost, s));
        iter_bytes_d2h_ += (size_t)g.shard_n * 4;
      } else {
        auto& bp = blocks_.at(e.block);
        auto& g = groups_.at((size_t)bp.group - 1);
        int64_t ho = host_block_off(blocks_, g, e.block);
        CK(cudaMemcpyAsync(h_grad_ + ho, d_grad_block(e.block), (size_t)bp.n_params * 4, cudaMemcpyDeviceToHost, s));
        iter_bytes_d2h_ += (size_t)bp.n_params * 4;
      }
      CK(cudaEventRecord(ev_done_[idx], s));
      return;
    }
    case Action::EXCHANGE: {
      cudaStream_t s = streams_[3];
      wait_deps(s, x, ops);
      auto& g = groups_.at((size_t)e.group - 1);
      size_t shard_pos = 0;
      for (int gi = 0; gi < e.group - 1; ++gi) shard_pos += (size_t)groups_[gi].shard_n;
      if (peers_ || ipc_) {
        std::vector<const float*> in((size_t)world_);
        if (ipc_) {
          ipc_wait(s, PK_BW, e.group, (uint32_t)step);
          for (int p = 0; p < world_; ++p)
            in[p] = reinterpret_cast<const float*>(ipc_g_[p]) + grad_slot_off_[(size_t)e.group - 1] +
                    (int64_t)rank_ * g.shard_n;
        } else {
          peers_->wait_all(PK_BW, e.group, step, watchdog_s_);
          for (int p = 0; p < world_; ++p) {
            Runtime* peer = peers_->ranks[p];
            if (!peer) throw std::runtime_error("peer rank " + std::to_string(p) + " missing");
            CK(cudaStreamWaitEvent(s, peers_->event(p, PK_BW, e.group), 0));
            in[p] = peer->grads_base() + grad_slot_off_[(size_t)e.group - 1] + (int64_t)rank_ * g.shard_n;
          }
        }
        CK(cudaEventRecord(ev_start_[idx], s));
        CK(launch_reduce_cast(in.data(), world_, d_shard_ + shard_pos, KRT_F32, (size_t)g.shard_n, 1.0f, s));
        ++kernel_launches_;
        ++iter_launches_;
      } else {
        CK(cudaEventRecord(ev_start_[idx], s));
        if (d_pack_) {
          // grad cast pack -> bf16 reduce-scatter -> fp32 shard (the update applies grad_scale)
          const float* src = d_grad_group(e.group);
          CK(launch_reduce_cast(&src, 1, d_pack_, KRT_BF16, (size_t)g.p_n, 1.0f, s));
          NK(ncclReduceScatter(d_pack_, d_pack_shard_, (size_t)g.shard_n, ncclBfloat16, ncclSum,
                               (ncclComm_t)nccl_comm_, s));
          CK(launch_unpack_bf16(d_pack_shard_, d_shard_ + shard_pos, (size_t)g.shard_n, 1.0f, s));
          kernel_launches_ += 2;
          iter_launches_ += 2;
        } else {
          NK(ncclReduceScatter(d_grad_group(e.group), d_shard_ + shard_pos, (size_t)g.shard_n, ncclFloat, ncclSum,
                               (ncclComm_t)nccl_comm_, s));
        }
      }
      CK(cudaEventRecord(ev_done_[idx], s));
      bytes_net_ += (size_t)g.p_n * (d_pack_ ? 2 : 4) * (world_ - 1) / world_;
      return;
    }
    case Action::HOST_UPDATE: {
      HostTask t;
      t.op = idx;
      t.group = e.group;
      t.step = step;
      for (int d : e.deps) t.waits.push_back(ev_done_[d]);
      iter_mutated_ = true;
      {
        std::lock_guard<std::mutex> lk(hmu_);
        hq_.push_back(t);
      }
      hcv_.notify_all();
      return;
    }
    case Action::WEIGHT_IN: {
      // the previous iteration's host update of this group must be complete
      wait_host_done(x.prev_host_group, step - 1);
      cudaStream_t s = streams_[1];
      wait_deps(s, x, ops);
      CK(cudaEventRecord(ev_start_[idx], s));
      if (dp_) {
        auto& g = groups_.at((size_t)e.group - 1);
        void* dst = d_weight(g.p_lo + (int64_t)rank_ * g.shard_n);
        CK(cudaMemcpyAsync(dst, static_cast<uint8_t*>(h_wstage_) + g.host_off * wb, (size_t)g.shard_n * wb,
                           cudaMemcpyHostToDevice, s));
        iter_bytes_h2d_ += (size_t)g.shard_n * wb;
        // the all-gather rides the network stream behind the H2D
        cudaStream_t ns = streams_[3];
        CK(cudaEventRecord(ev_done_[idx], s));
        CK(cudaStreamWaitEvent(ns, ev_done_[idx], 0));
        if (ipc_) {
          ipc_signal(s, PK_WSHARD, e.group, (uint32_t)step);
          ipc_wait(ns, PK_WSHARD, e.group, (uint32_t)step);
          gather_peer_shards(g, e.group, ns, PK_WSHARD);
        } else if (peers_) {
          CK(cudaEventRecord(peers_->event(rank_, PK_WSHARD, e.group), s));
          peers_->mark(rank_, PK_WSHARD, e.group, step);
          peers_->wait_all(PK_WSHARD, e.group, step, watchdog_s_);
          gather_peer_shards(g, e.group, ns, PK_WSHARD);
        } else {
          NK(ncclAllGather(dst, d_weight(g.p_lo), (size_t)g.shard_n,
                           cfg_.weight_dtype == KRT_BF16 ? ncclBfloat16 : ncclFloat, (ncclComm_t)nccl_comm_, ns));
        }
        CK(cudaEventRecord(ev_done_[idx], ns));
        bytes_net_ += (size_t)g.p_n * wb * (world_ - 1) / world_;
      } else {
        auto& bp = blocks_.at(e.block);
        auto& g = groups_.at((size_t)bp.group - 1);
        int64_t ho = host_block_off(blocks_, g, e.block);
        CK(cudaMemcpyAsync(d_weight(bp.p_off), static_cast<uint8_t*>(h_wstage_) + (size_t)ho * wb,
                           (size_t)bp.n_params * wb, cudaMemcpyHostToDevice, s));
        iter_bytes_h2d_ += (size_t)bp.n_params * wb;
        CK(cudaEventRecord(ev_done_[idx], s));
      }
      return;
    }
  }
}

void CUDART_CB Runtime::anchor_cb(void* arg) {
  auto* a = static_cast<AnchorArg*>(arg);
  double t = host_now();
  std::lock_guard<std::mutex> lk(a->rt->hmu_);
  a->rt->clock_anchor_[a->step] = t;
}

void Runtime::run_iteration(krt_compute_cb cb, void* user) {
  if (!prepared_) throw std::logic_error("run_iteration before prepare");
  if (!failed_.empty()) throw std::runtime_error("context unusable: " + failed_);
  CK(cudaSetDevice(cfg_.device));
  {
    std::lock_guard<std::mutex> lk(hmu_);
    if (!host_error_.empty()) throw std::runtime_error("host update failed: " + host_error_);
  }
  int step = ++step_;
  bool first = step == 1;
  auto& ops = first ? ops_first_ : ops_steady_;
  auto& order = first ? order_first_ : order_steady_;
  iter_bytes_h2d_ = iter_bytes_d2h_ = iter_launches_ = 0;
  iter_mutated_ = false;
  cur_slot_.clear();
  iter_host_t0_ = host_now();
  try {
    CK(cudaEventRecord(ev_base_, streams_[0]));
    // host clock when the compute stream reaches ev_base_ (off the compute stream)
    {
      std::lock_guard<std::mutex> lk(hmu_);
      while (anchor_args_.size() > 8) anchor_args_.pop_front();
      anchor_args_.push_back({this, step});
      for (auto it = clock_anchor_.begin(); it != clock_anchor_.end();)
        it = it->first < step - 8 ? clock_anchor_.erase(it) : std::next(it);
    }
    CK(cudaStreamWaitEvent(clock_stream_, ev_base_, 0));
    CK(cudaLaunchHostFunc(clock_stream_, anchor_cb, &anchor_args_.back()));
    last_first_ = first;
    for (int idx : order) issue(idx, ops, cb, user, step);
  } catch (const std::exception& ex) {
    fail_iteration(step, ex.what());
    throw;
  }
  bytes_h2d_ += iter_bytes_h2d_;
  bytes_d2h_ += iter_bytes_d2h_;
}

void Runtime::synchronize() {
  if (!failed_.empty()) throw std::runtime_error("context unusable: " + failed_);
  CK(cudaSetDevice(cfg_.device));
  const double t_end = host_now() + watchdog_s_;
  for (auto s : streams_) {
    int spins = 0;
    for (;;) {
      cudaError_t r = cudaStreamQuery(s);
      if (r == cudaSuccess) break;
      if (r != cudaErrorNotReady) throw CudaError(std::string("synchronize: ") + cudaGetErrorString(r));
      if (host_now() > t_end)
        throw std::runtime_error("watchdog: iteration " + std::to_string(step_) + " stalled for " +
                                 std::to_string(watchdog_s_) + " s; first incomplete op: " + first_pending_op());
      if (++spins < 64) std::this_thread::yield();
      else std::this_thread::sleep_for(std::chrono::microseconds(spins < 1024 ? 20 : 500));
    }
  }
  int step = step_;
  for (size_t gi = 0; gi < groups_.size(); ++gi) {
    bool has_host = false;
    auto& ops = last_first_ ? ops_first_ : ops_steady_;
    for (auto& x : ops)
      if (x.e.action == Action::HOST_UPDATE && x.e.group == (int)gi + 1) has_host = true;
    if (has_host && step > 0) wait_host_done((int)gi + 1, step);
  }
}

std::string Runtime::trace_csv() {
  synchronize();
  auto& ops = last_first_ ? ops_first_ : ops_steady_;
  std::ostringstream os;
  os << "t_start,t_end,resource,block,action,group,stall_before\n";
  struct Row { double t0, t1; int res; int op; };
  std::vector<Row> rows;
  for (size_t i = 0; i < ops.size(); ++i) {
    const EngineOp& e = ops[i].e;
    double t0 = 0, t1 = 0;
    if (e.action == Action::HOST_UPDATE) {
      // host clock minus the host time at which the compute stream passed
      // ev_base_: the same origin as the device rows (within the host
      // callback latency, microseconds)
      std::lock_guard<std::mutex> lk(hmu_);
      auto it = host_times_.find({e.group, step_});
      auto an = clock_anchor_.find(step_);
      if (it == host_times_.end() || an == clock_anchor_.end()) continue;
      t0 = it->second.first - an->second;
      t1 = it->second.second - an->second;
    } else {
      float ms0 = 0, ms1 = 0;
      if (cudaEventElapsedTime(&ms0, ev_base_, ev_start_[i]) != cudaSuccess) continue;
      if (cudaEventElapsedTime(&ms1, ev_base_, ev_done_[i]) != cudaSuccess) continue;
      t0 = ms0 * 1e-3;
      t1 = ms1 * 1e-3;
    }
    rows.push_back({t0, t1, e.res, (int)i});
  }
  std::stable_sort(rows.begin(), rows.end(), [](const Row& a, const Row& b) {
    if (a.t0 != b.t0) return a.t0 < b.t0;
    return std::string(res_name(a.res)) < std::string(res_name(b.res));
  });
  std::map<int, double> last_end;
  for (auto& r : rows) {
    const EngineOp& e = ops[r.op].e;
    double stall = 0;
    auto it = last_end.find(r.res);
    if (it != last_end.end()) stall = std::max(0.0, r.t0 - it->second);
    last_end[r.res] = std::max(r.t1, it != last_end.end() ? it->second : r.t1);
    os << py_9g(r.t0) << "," << py_9g(r.t1) << "," << res_name(r.res) << "," << e.block << ","
       << action_name(e.action) << "," << e.group << "," << py_9g(stall) << "\n";
  }
  return os.str();
}

std::string Runtime::stats_json() {
  std::ostringstream os;
  size_t nswapped = 0;
  for (auto& [id, b] : blocks_) nswapped += b.swapped;
  os << "{\"arena_bytes\": " << arena_bytes_ << ", \"ledger_peak_bytes\": " << ledger_peak_
     << ", \"instances\": " << instances_.size() << ", \"host_swap_bytes\": " << h_swap_bytes_
     << ", \"swapped_blocks\": " << nswapped << ", \"params\": " << total_params_
     << ", \"grad_region_bytes\": " << grad_elems_ * 4 << ", \"grad_slots\": " << grad_ring_
     << ", \"host_elems\": " << host_elems_ << ", \"bytes_h2d_total\": " << bytes_h2d_
     << ", \"bytes_d2h_total\": " << bytes_d2h_ << ", \"bytes_net_total\": " << bytes_net_
     << ", \"iter_bytes_h2d\": " << iter_bytes_h2d_ << ", \"iter_bytes_d2h\": " << iter_bytes_d2h_
     << ", \"kernel_launches_total\": " << kernel_launches_ << ", \"iter_kernel_launches\": " << iter_launches_
     << ", \"ops_per_iteration\": " << ops_steady_.size() << ", \"step\": " << step_ << ", \"world\": " << world_
     << ", \"groups\": " << groups_.size() << "}";
  return os.str();
}

void Runtime::flush_weights() {
  synchronize();
  if (step_ == 0) return;
  size_t wb = dtype_bytes(cfg_.weight_dtype);
  cudaStream_t s = streams_[1];
  for (auto& g : groups_) {
    if (dp_) {
      void* dst = d_weight(g.p_lo + (int64_t)rank_ * g.shard_n);
      CK(cudaMemcpyAsync(dst, static_cast<uint8_t*>(h_wstage_) + g.host_off * wb, (size_t)g.shard_n * wb,
                         cudaMemcpyHostToDevice, s));
      if (ipc_) {
        int gi = (int)(&g - groups_.data()) + 1;
        ipc_signal(s, PK_FLUSH, gi, (uint32_t)(flush_count_ + 1));
        ipc_wait(s, PK_FLUSH, gi, (uint32_t)(flush_count_ + 1));
        gather_peer_shards(g, gi, s, PK_FLUSH);
      } else if (peers_) {
        int gi = (int)(&g - groups_.data()) + 1;
        CK(cudaEventRecord(peers_->event(rank_, PK_FLUSH, gi), s));
        peers_->mark(rank_, PK_FLUSH, gi, flush_count_ + 1);
        peers_->wait_all(PK_FLUSH, gi, flush_count_ + 1, watchdog_s_);
        gather_peer_shards(g, gi, s, PK_FLUSH);
      } else {
        NK(ncclAllGather(dst, d_weight(g.p_lo), (size_t)g.shard_n,
                         cfg_.weight_dtype == KRT_BF16 ? ncclBfloat16 : ncclFloat, (ncclComm_t)nccl_comm_, s));
      }
    } else {
      for (int b : g.members) {
        auto& bp = blocks_.at(b);
        if (!bp.host_path) continue;
        int64_t ho = host_block_off(blocks_, g, b);
        CK(cudaMemcpyAsync(d_weight(bp.p_off), static_cast<uint8_t*>(h_wstage_) + (size_t)ho * wb,
                           (size_t)bp.n_params * wb, cudaMemcpyHostToDevice, s));
      }
    }
  }
  CK(cudaStreamSynchronize(s));
  ++flush_count_;
}

double Runtime::probe_exchange(size_t bytes, int iters) {
  if (!nccl_comm_) throw std::invalid_argument("probe_exchange needs the NCCL exchange (not IPC / in-process peers)");
  if (iters < 1) throw std::invalid_argument("iters must be >= 1");
  CK(cudaSetDevice(cfg_.device));
  size_t n = bytes / 4 / (size_t)world_ * (size_t)world_;
  if (n < (size_t)world_) n = (size_t)world_;
  float *send = nullptr, *recv = nullptr;
  CK(cudaMalloc(&send, n * 4));
  CK(cudaMalloc(&recv, n / world_ * 4));
  cudaStream_t s = streams_[3];
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  double sec = 0;
  try {
    CK(cudaMemsetAsync(send, 0, n * 4, s));
    for (int i = 0; i < 2; ++i)
      NK(ncclReduceScatter(send, recv, n / world_, ncclFloat, ncclSum, (ncclComm_t)nccl_comm_, s));
    CK(cudaEventRecord(e0, s));
    for (int i = 0; i < iters; ++i)
      NK(ncclReduceScatter(send, recv, n / world_, ncclFloat, ncclSum, (ncclComm_t)nccl_comm_, s));
    CK(cudaEventRecord(e1, s));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    sec = ms * 1e-3 / iters;
  } catch (...) {
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(send);
    cudaFree(recv);
    throw;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(send);
  cudaFree(recv);
  return sec;
}

void Runtime::gather_peer_shards(const GroupPhys& g, int group, cudaStream_t s, int kind) {
  size_t wb = dtype_bytes(cfg_.weight_dtype);
  for (int p = 0; p < world_; ++p) {
    if (p == rank_) continue;
    const uint8_t* src;
    if (ipc_) {
      src = ipc_w_[p];
    } else {
      Runtime* peer = peers_->ranks[p];
      if (!peer) throw std::runtime_error("peer rank " + std::to_string(p) + " missing");
      CK(cudaStreamWaitEvent(s, peers_->event(p, kind, group), 0));
      src = static_cast<const uint8_t*>(peer->weights_base());
    }
    size_t off = (size_t)(g.p_lo + (int64_t)p * g.shard_n) * wb;
    CK(cudaMemcpyAsync(static_cast<uint8_t*>(d_weights_) + off, src + off, (size_t)g.shard_n * wb,
                       cudaMemcpyDefault, s));
  }
  bytes_net_ += (size_t)g.shard_n * wb * (world_ - 1);
}

size_t Runtime::flag_index(int kind, int group, int src) const {
  return ((size_t)kind * groups_.size() + (size_t)(group - 1)) * (size_t)world_ + (size_t)src;
}

// driver stream-memory ops, resolved through the runtime (no libcuda link, so
// the library still loads on a host without the driver)
namespace {
using WriteFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using WaitFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WriteFn g_write32 = nullptr;
WaitFn g_wait32 = nullptr;
void load_memops() {
  if (g_write32 && g_wait32) return;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuStreamWriteValue32", (void**)&g_write32, cudaEnableDefault, &q));
  if (q != cudaDriverEntryPointSuccess || !g_write32) throw CudaError("cuStreamWriteValue32 unavailable");
  CK(cudaGetDriverEntryPoint("cuStreamWaitValue32", (void**)&g_wait32, cudaEnableDefault, &q));
  if (q != cudaDriverEntryPointSuccess || !g_wait32) throw CudaError("cuStreamWaitValue32 unavailable");
}
}  // namespace

// flag write into every rank's array: ordered after the stream's prior work,
// with the default memory barrier (peers then read our data over NVLink)
void Runtime::ipc_signal(cudaStream_t s, int kind, int group, uint32_t value) {
  if (!ipc_ready_) throw std::logic_error("IPC exchange used before krt_ipc_import");
  for (int q = 0; q < world_; ++q) {
    CUresult r = g_write32((CUstream)s, (CUdeviceptr)(ipc_flags_[q] + flag_index(kind, group, rank_)),
                                      value, CU_STREAM_WRITE_VALUE_DEFAULT);
    if (r != CUDA_SUCCESS) throw CudaError("cuStreamWriteValue32 failed: " + std::to_string((int)r));
  }
}

void Runtime::ipc_wait(cudaStream_t s, int kind, int group, uint32_t value) {
  for (int p = 0; p < world_; ++p) {
    CUresult r = g_wait32((CUstream)s, (CUdeviceptr)(d_flags_ + flag_index(kind, group, p)), value,
                                     CU_STREAM_WAIT_VALUE_GEQ);
    if (r != CUDA_SUCCESS) throw CudaError("cuStreamWaitValue32 failed: " + std::to_string((int)r));
  }
}

std::vector<uint8_t> Runtime::ipc_export() {
  if (!prepared_ || !ipc_) throw std::logic_error("ipc_export needs a prepared context with ipc_exchange");
  CK(cudaSetDevice(cfg_.device));
  std::vector<uint8_t> out(3 * sizeof(cudaIpcMemHandle_t));
  cudaIpcMemHandle_t h[3];
  CK(cudaIpcGetMemHandle(&h[0], d_weights_));
  CK(cudaIpcGetMemHandle(&h[1], d_grads_));
  CK(cudaIpcGetMemHandle(&h[2], d_flags_));
  std::memcpy(out.data(), h, out.size());
  return out;
}

void Runtime::ipc_import(const uint8_t* all, int world) {
  if (!ipc_) throw std::logic_error("context was not created with ipc_exchange");
  if (world != world_) throw std::invalid_argument("handle count != world_size");
  CK(cudaSetDevice(cfg_.device));
  size_t hb = 3 * sizeof(cudaIpcMemHandle_t);
  ipc_w_.assign(world_, nullptr);
  ipc_g_.assign(world_, nullptr);
  ipc_flags_.assign(world_, nullptr);
  for (int p = 0; p < world_; ++p) {
    if (p == rank_) {
      ipc_w_[p] = static_cast<uint8_t*>(d_weights_);
      ipc_g_[p] = reinterpret_cast<uint8_t*>(d_grads_);
      ipc_flags_[p] = d_flags_;
      continue;
    }
    cudaIpcMemHandle_t h[3];
    std::memcpy(h, all + (size_t)p * hb, hb);
    void* ptr = nullptr;
    CK(cudaIpcOpenMemHandle(&ptr, h[0], cudaIpcMemLazyEnablePeerAccess));
    ipc_w_[p] = static_cast<uint8_t*>(ptr);
    CK(cudaIpcOpenMemHandle(&ptr, h[1], cudaIpcMemLazyEnablePeerAccess));
    ipc_g_[p] = static_cast<uint8_t*>(ptr);
    CK(cudaIpcOpenMemHandle(&ptr, h[2], cudaIpcMemLazyEnablePeerAccess));
    ipc_flags_[p] = static_cast<uint32_t*>(ptr);
  }
  load_memops();
  ipc_ready_ = true;
}

void* Runtime::block_slot(int block) const {
  auto it = cur_slot_.find(block);
  if (it == cur_slot_.end()) throw std::invalid_argument("block " + std::to_string(block) + " has no resident slot");
  return it->second;
}

// ---------------------------------------------------------------------------
// checkpoint / restart of the training state this rank owns (PAPER.md:567:
// epochs split across runs with C/R of the model state).  Written after the
// last iteration completes: device weights, device-path fp32 masters and
// optimizer moments, the host-path fp32 masters and moments (this rank's
// shards) and the weight staging the next weight_in copies from, plus the
// iteration counter (Adam bias correction).  A restored context continues
// bitwise where the saved one stopped.
// ---------------------------------------------------------------------------
namespace {
struct CkptHeader {
  char magic[8];
  uint32_t version, world, rank, weight_dtype;
  uint64_t params, host_elems, step;
  uint32_t has_dev_master, has_dev_moments;
  uint64_t layout_hash;  // version 2: parameter / host-state layout of the plan
};

// FNV-1a over the parameter and host-state layout (block offsets, sizes, host
// path, group ranges and shards): two plans with equal totals but a different
// swap / host-path split hash differently
uint64_t layout_hash(const std::map<int, BlockPhys>& blocks, const std::vector<GroupPhys>& groups) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](uint64_t v) {
    for (int i = 0; i < 8; ++i) {
      h ^= (v >> (8 * i)) & 0xffu;
      h *= 1099511628211ull;
    }
  };
  for (const auto& kv : blocks) {
    const BlockPhys& b = kv.second;
    mix((uint64_t)kv.first);
    mix((uint64_t)b.p_off);
    mix((uint64_t)b.n_params);
    mix((uint64_t)b.host_path);
    mix((uint64_t)b.group);
  }
  for (const auto& g : groups) {
    mix((uint64_t)g.p_lo);
    mix((uint64_t)g.p_n);
    mix((uint64_t)g.shard_n);
    mix((uint64_t)g.host_off);
    mix((uint64_t)g.host_n);
  }
  return h;
}

void write_all(std::FILE* f, const void* p, size_t n) {
  if (n && std::fwrite(p, 1, n, f) != n) throw std::runtime_error("checkpoint: short write");
}
void read_all(std::FILE* f, void* p, size_t n) {
  if (n && std::fread(p, 1, n, f) != n) throw std::runtime_error("checkpoint: short read (truncated file?)");
}

// device buffer <-> file through a bounded pinned bounce buffer
void dev_to_file(std::FILE* f, const void* d, size_t n) {
  const size_t chunk = (size_t)64 << 20;
  std::vector<uint8_t> buf(std::min(n, chunk));
  for (size_t o = 0; o < n; o += chunk) {
    size_t k = std::min(chunk, n - o);
    CK(cudaMemcpy(buf.data(), static_cast<const uint8_t*>(d) + o, k, cudaMemcpyDeviceToHost));
    write_all(f, buf.data(), k);
  }
}
void file_to_dev(std::FILE* f, void* d, size_t n) {
  const size_t chunk = (size_t)64 << 20;
  std::vector<uint8_t> buf(std::min(n, chunk));
  for (size_t o = 0; o < n; o += chunk) {
    size_t k = std::min(chunk, n - o);
    read_all(f, buf.data(), k);
    CK(cudaMemcpy(static_cast<uint8_t*>(d) + o, buf.data(), k, cudaMemcpyHostToDevice));
  }
}
}  // namespace

void Runtime::checkpoint_save(const std::string& path) {
  if (!prepared_) throw std::logic_error("checkpoint_save before prepare");
  synchronize();
  CK(cudaSetDevice(cfg_.device));
  const size_t wb = dtype_bytes(cfg_.weight_dtype);
  const size_t np = (size_t)std::max<int64_t>(total_params_, 64);
  const size_t he = std::max<size_t>(host_elems_, 64);
  CkptHeader h{};
  std::memcpy(h.magic, "KRTCKPT1", 8);
  h.version = 2;
  h.layout_hash = layout_hash(blocks_, groups_);
  h.world = (uint32_t)world_;
  h.rank = (uint32_t)rank_;
  h.weight_dtype = (uint32_t)cfg_.weight_dtype;
  h.params = np;
  h.host_elems = he;
  h.step = (uint64_t)step_;
  h.has_dev_master = d_master_ != nullptr;
  h.has_dev_moments = d_m_ != nullptr;
  std::string tmp = path + ".tmp";
  std::FILE* f = std::fopen(tmp.c_str(), "wb");
  if (!f) throw std::runtime_error("checkpoint: cannot open " + tmp);
  try {
    write_all(f, &h, sizeof(h));
    dev_to_file(f, d_weights_, np * wb);
    if (d_master_) dev_to_file(f, d_master_, np * 4);
    if (d_m_) {
      dev_to_file(f, d_m_, np * 4);
      dev_to_file(f, d_v_, np * 4);
    }
    write_all(f, h_master_.data(), he * 4);
    write_all(f, h_m_.data(), he * 4);
    write_all(f, h_v_.data(), he * 4);
    write_all(f, h_wstage_, he * wb);
  } catch (...) {
    std::fclose(f);
    std::remove(tmp.c_str());
    throw;
  }
  if (std::fclose(f) != 0) throw std::runtime_error("checkpoint: close failed");
  if (std::rename(tmp.c_str(), path.c_str()) != 0) throw std::runtime_error("checkpoint: rename failed");
}

void Runtime::checkpoint_load(const std::string& path) {
  if (!prepared_) throw std::logic_error("checkpoint_load before prepare");
  synchronize();
  CK(cudaSetDevice(cfg_.device));
  const size_t wb = dtype_bytes(cfg_.weight_dtype);
  const size_t np = (size_t)std::max<int64_t>(total_params_, 64);
  const size_t he = std::max<size_t>(host_elems_, 64);
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) throw std::runtime_error("checkpoint: cannot open " + path);
  try {
    CkptHeader h{};
    read_all(f, &h, sizeof(h));
    if (std::memcmp(h.magic, "KRTCKPT1", 8) != 0 || h.version != 2)
      throw std::invalid_argument("checkpoint: not a krt checkpoint (bad magic/version)");
    if (h.world != (uint32_t)world_ || h.rank != (uint32_t)rank_ || h.weight_dtype != (uint32_t)cfg_.weight_dtype ||
        h.params != np || h.host_elems != he || h.has_dev_master != (d_master_ != nullptr) ||
        h.has_dev_moments != (d_m_ != nullptr) || h.layout_hash != layout_hash(blocks_, groups_))
      throw std::invalid_argument("checkpoint: saved for a different model, plan, dtype or rank");
    // multi-rank exchanges synchronise on monotone per-step flags and marks
    // (IPC flags, peer-group marks): replaying steps this context already ran
    // would let the waits pass before the peers' buffers are written
    if (world_ > 1 && (int64_t)h.step < (int64_t)step_)
      throw std::invalid_argument("checkpoint: step " + std::to_string(h.step) + " is behind this context's step " +
                                  std::to_string(step_) + " (multi-rank: load into a fresh context)");
    file_to_dev(f, d_weights_, np * wb);
    if (d_master_) file_to_dev(f, d_master_, np * 4);
    if (d_m_) {
      file_to_dev(f, d_m_, np * 4);
      file_to_dev(f, d_v_, np * 4);
    }
    read_all(f, h_master_.data(), he * 4);
    read_all(f, h_m_.data(), he * 4);
    read_all(f, h_v_.data(), he * 4);
    read_all(f, h_wstage_, he * wb);
    std::fclose(f);
    f = nullptr;
    // continue as the iteration after the saved one: steady-state ops, whose
    // weight_in then finds the saved staging and a completed host update
    step_ = (int)h.step;
    last_first_ = step_ <= 1;
    std::lock_guard<std::mutex> lk(hmu_);
    for (size_t gi = 0; gi < groups_.size(); ++gi) host_done_step_[(int)gi + 1] = step_;
  } catch (...) {
    if (f) std::fclose(f);
    throw;
  }
}

void Runtime::read_master(int block, float* out, size_t numel) {
  synchronize();
  auto& bp = blocks_.at(block);
  if (numel < (size_t)bp.n_params) throw std::invalid_argument("output too small");
  auto& g = groups_.at((size_t)bp.group - 1);
  if (bp.host_path) {
    if (dp_) {
      int64_t lo = g.p_lo + (int64_t)rank_ * g.shard_n, hi = lo + g.shard_n;
      for (int64_t i = 0; i < bp.n_params; ++i) {
        int64_t p = bp.p_off + i;
        out[i] = (p >= lo && p < hi) ? h_master_[g.host_off + (size_t)(p - lo)] : 0.f;
      }
    } else {
      int64_t ho = host_block_off(blocks_, g, block);
      std::memcpy(out, h_master_.data() + ho, (size_t)bp.n_params * 4);
    }
  } else {
    const void* src = d_master_ ? (const void*)(d_master_ + bp.p_off) : d_weight(bp.p_off);
    CK(cudaMemcpy(out, src, (size_t)bp.n_params * 4, cudaMemcpyDeviceToHost));
  }
}

}  // namespace krt
