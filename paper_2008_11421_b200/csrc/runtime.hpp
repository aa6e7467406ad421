// Per-rank executor of a KARMA execution plan on one B200.
//
// The plan's ops (plan.py:24-29) and the DP pipeline ops (distsim.py:168-236)
// become CUDA work on four streams — compute (fw / recompute_fw / bw),
// H2D (swap_in, weight_in), D2H (swap_out, grad_out), network (exchange) —
// plus a host-update thread.  Every dependency of build_engine_ops /
// simulate_distributed is a cudaStreamWaitEvent; the start gate
// (simulator.py:324-329) waits on an event recorded just before the gating
// compute op; the capacity ledger (simulator.py:90) is realised by a static
// arena assignment whose address reuse adds free->alloc event edges.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <condition_variable>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "../../include/krt.h"
#include "engine.hpp"
#include "host_optim.hpp"

namespace krt {

struct BlockPhys {
  size_t act_bytes = 0;          // arena slot bytes
  std::vector<int64_t> numel;    // parameter tensors
  int64_t n_params = 0;
  int64_t p_off = 0;             // element offset in the flat parameter space
  bool host_path = false;
  int group = 0;                 // 1-based
  size_t host_swap_off = 0;
  bool swapped = false;
};

struct GroupPhys {
  std::vector<int> members;
  int64_t p_lo = 0, p_n = 0;     // flat element range, padded to world*64
  int64_t shard_n = 0;           // p_n / world
  bool host = false;             // any member on the host path
  size_t host_off = 0;           // offset (elements) of this group's host state
  int64_t host_n = 0;            // host elements (shard for P>1, host members for P=1)
};

// executor op: an engine op plus the physical bindings
struct XOp {
  EngineOp e;
  int instance = -1;             // arena instance allocated (fw/recompute/swap_in)
  int reads_instance = -1;       // instance read by bw / swap_out
  std::vector<int> arena_deps;   // ops whose completion frees our region
  int prev_host_group = -1;      // weight_in: host_update of the previous iteration
};

struct Instance {
  int block = 0;
  size_t off = 0, bytes = 0;
  int alloc_op = -1, free_op = -1;
};

struct HostTask {
  int op = -1;
  int group = 0;
  std::vector<cudaEvent_t> waits;
  int step = 0;
};

class Runtime;

// In-process exchange between ranks that share one process (logical ranks on
// one GPU, or one process driving several GPUs): the reduce-scatter is
// krt_reduce_cast over the peers' gradient buffers and the all-gather a set
// of device-to-device copies, ordered by per-(rank, kind, group) events.
// Host-side "issued" marks make sure an event is recorded for the current
// step before any peer waits on it.
struct PeerGroup {
  explicit PeerGroup(int w) : world(w), ranks(w, nullptr) {}
  int world;
  std::mutex mu;
  std::condition_variable cv;
  std::vector<Runtime*> ranks;
  std::map<std::tuple<int, int, int>, int> marks;         // (rank, kind, group) -> step
  std::map<std::tuple<int, int, int>, cudaEvent_t> events;
  void mark(int rank, int kind, int group, int step);
  // bounded: throws naming the ranks that never marked (a dead or stalled peer)
  void wait_all(int kind, int group, int step, double timeout_s);
  cudaEvent_t event(int rank, int kind, int group);
  ~PeerGroup();
};
enum PeerKind { PK_BW = 0, PK_WSHARD = 1, PK_FLUSH = 2 };

class Runtime {
 public:
  explicit Runtime(const krt_config& cfg);
  ~Runtime();

  void register_block(int block, size_t act_bytes, const int64_t* numel, int n);
  void prepare(const Plan& plan, const Model& model, const Hardware& hw);
  void region(int which, int block, void** ptr, size_t* bytes);
  cudaStream_t stream(int which) const;
  void init_master();
  void run_iteration(krt_compute_cb cb, void* user);
  void synchronize();
  std::string trace_csv();
  std::string stats_json();
  void read_master(int block, float* out, size_t numel);
  void* block_slot(int block) const;
  void flush_weights();
  // mean seconds of one ncclReduceScatter of `bytes` fp32 gradient bytes on
  // this context's communicator and network stream (collective: every rank)
  double probe_exchange(size_t bytes, int iters);
  void checkpoint_save(const std::string& path);
  void checkpoint_load(const std::string& path);
  std::vector<uint8_t> ipc_export();
  void ipc_import(const uint8_t* all, int world);
  void* weights_base() const { return d_weights_; }
  float* grads_base() const { return d_grads_; }

 private:
  void build_ops(const Plan& plan, const Model& model, const Hardware& hw);
  void allocate();
  void issue(int idx, std::vector<XOp>& ops, krt_compute_cb cb, void* user, int step);
  void wait_deps(cudaStream_t s, const XOp& x, const std::vector<XOp>& ops);
  void host_loop();
  void run_host_task(const HostTask& t);
  void wait_host_done(int group, int step);
  // polls an event until it completes or the watchdog expires (then throws `what`)
  void wait_event_bounded(cudaEvent_t e, const std::string& what) const;
  // the op of the last issued iteration still incomplete, first in issue order
  std::string first_pending_op();
  void fail_iteration(int step, const std::string& why);
  void gather_peer_shards(const GroupPhys& g, int group, cudaStream_t s, int kind);
  // gradient addresses: the group's slot (the whole-model region when
  // grad_slots == 0, where the slot offset is the group's own p_lo)
  float* d_grad_group(int group) const { return d_grads_ + grad_slot_off_[(size_t)group - 1]; }
  float* d_grad_block(int block) const {
    const BlockPhys& b = blocks_.at(block);
    return d_grad_group(b.group) + (b.p_off - groups_[(size_t)b.group - 1].p_lo);
  }
  void* d_weight(int64_t p_off) const;

  krt_config cfg_;
  int world_ = 1, rank_ = 0;
  bool dp_ = false;   // data-parallel op structure (exchange / shard host update / all-gather)
  std::map<int, BlockPhys> blocks_;
  std::vector<GroupPhys> groups_;     // index = group-1
  int nb_ = 0;
  int64_t total_params_ = 0;

  std::vector<XOp> ops_first_, ops_steady_;
  std::vector<int> order_first_, order_steady_;
  std::vector<Instance> instances_;
  size_t arena_bytes_ = 0, ledger_peak_ = 0;

  // memory
  uint8_t* d_arena_ = nullptr;
  void* d_weights_ = nullptr;
  float* d_grads_ = nullptr;
  std::vector<int64_t> grad_slot_off_;  // per group (index group-1): element offset in d_grads_
  int64_t grad_elems_ = 0;              // d_grads_ size in elements
  int grad_ring_ = 0;                   // slots in use (0: whole-model region)
  float* d_master_ = nullptr;   // device-path masters (bf16 weights only)
  float* d_m_ = nullptr;
  float* d_v_ = nullptr;
  float* d_shard_ = nullptr;    // reduce-scatter landing (P>1)
  void* d_pack_ = nullptr;      // bf16 exchange: packed group gradients (max group p_n)
  void* d_pack_shard_ = nullptr;  // bf16 exchange: reduce-scattered bf16 shard (max shard_n)
  uint8_t* h_swap_ = nullptr;
  size_t h_swap_bytes_ = 0;
  float* h_grad_ = nullptr;     // pinned, host_n per group
  void* h_wstage_ = nullptr;    // pinned weight copies for weight_in
  std::vector<float> h_master_, h_m_, h_v_;
  size_t host_elems_ = 0;

  cudaStream_t streams_[4] = {};
  std::vector<cudaEvent_t> ev_start_, ev_done_;
  cudaEvent_t ev_base_ = nullptr;
  void* nccl_comm_ = nullptr;
  PeerGroup* peers_ = nullptr;     // in-process exchange instead of NCCL
  // cross-process exchange over CUDA IPC peer memory: peers' weight/grad
  // regions and flag arrays, ordered by stream memory ops on the flags
  bool ipc_ = false, ipc_ready_ = false;
  uint32_t* d_flags_ = nullptr;
  std::vector<uint8_t*> ipc_w_, ipc_g_;
  std::vector<uint32_t*> ipc_flags_;
  size_t flag_index(int kind, int group, int src) const;
  void ipc_signal(cudaStream_t s, int kind, int group, uint32_t value);
  void ipc_wait(cudaStream_t s, int kind, int group, uint32_t value);
  int flush_count_ = 0;
  std::map<int, int> group_first_block_;  // group -> lowest member (last bw of the group)

  // host-update thread
  std::unique_ptr<ThreadPool> pool_;
  std::thread host_thread_;
  std::mutex hmu_;
  std::condition_variable hcv_;
  std::deque<HostTask> hq_;
  std::map<int, int> host_done_step_;   // group -> last completed iteration
  std::map<std::pair<int, int>, std::pair<double, double>> host_times_;  // (group,step) -> t0,t1
  std::string host_error_;
  bool hstop_ = false;
  double iter_host_t0_ = 0.0;

  std::map<int, uint8_t*> cur_slot_;   // block -> resident slot during issue
  int step_ = 0;
  bool prepared_ = false;
  // watchdog (KRT_WATCHDOG_S, default 900 s): no wait in the runtime blocks
  // longer; the error names the op that never completed
  double watchdog_s_ = 900.0;
  // set when an iteration failed after it had already applied updates: the
  // context refuses further work instead of hanging on the lost updates
  std::string failed_;
  bool iter_mutated_ = false;
  // host clock of the moment the compute stream passed ev_base_ (per step):
  // host-update trace rows are put on the GPU timeline with it
  cudaStream_t clock_stream_ = nullptr;
  std::map<int, double> clock_anchor_;
  struct AnchorArg {
    Runtime* rt;
    int step;
  };
  std::deque<AnchorArg> anchor_args_;
  static void CUDART_CB anchor_cb(void* arg);
  bool last_first_ = true;
  // stats
  uint64_t bytes_h2d_ = 0, bytes_d2h_ = 0, bytes_net_ = 0, kernel_launches_ = 0;
  uint64_t iter_bytes_h2d_ = 0, iter_bytes_d2h_ = 0, iter_launches_ = 0;
};

}  // namespace krt
