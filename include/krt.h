/*
 * krt.h — C ABI of the KARMA out-of-core data-parallel runtime for B200.
 *
 * The reference (oocsched, /root/reference/pkg) has no executor: its drop-in
 * boundary for this path is the ExecutionPlan / plan.json wire format
 * (plan.py:75-106, :179-231) plus the op semantics of build_engine_ops /
 * run_engine (simulator.py:67-135, :253-349) and simulate_distributed
 * (distsim.py:140-266).  Every entry point below replaces one of those, or one
 * executor step the paper describes and the reference only
 * simulates; the comment on each names the reference interface it stands in
 * for.  Plain pointers and sizes only; no C++ exceptions cross this boundary.
 *
 * Error protocol: every int-returning function returns KRT_OK (0) or one of
 * the codes below (they mirror the reference CLI's exit codes, cli.py:23-26);
 * krt_last_error() returns a thread-local message naming the failing op, in
 * the style of DeadlockError (simulator.py:36-39).
 */
#ifndef KRT_H_
#define KRT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum krt_status {
  KRT_OK = 0,
  KRT_INFEASIBLE = 1, /* plan violates residency/capacity, deadlock   (cli.py:24) */
  KRT_USAGE = 2,      /* malformed input / bad argument               (cli.py:25) */
  KRT_INTERNAL = 3    /* CUDA / NCCL / host failure                   (cli.py:26) */
};

/* plan actions (plan.py:24-29) followed by the DP pipeline ops (distsim.py:168-236) */
enum krt_action {
  KRT_FW = 0, KRT_BW = 1, KRT_SWAP_IN = 2, KRT_SWAP_OUT = 3, KRT_RECOMPUTE_FW = 4,
  KRT_WEIGHT_IN = 5, KRT_GRAD_OUT = 6, KRT_EXCHANGE = 7, KRT_HOST_UPDATE = 8
};

enum krt_dtype { KRT_F32 = 0, KRT_BF16 = 1 };
enum krt_optim { KRT_SGD = 0, KRT_ADAM = 1 };

const char* krt_last_error(void);
const char* krt_version(void);
void krt_string_free(char* s);

/* ------------------------------------------------------------------------
 * Plan bundle: model graph + hardware spec + execution plan.  Host-only; no
 * GPU needed.
 * ---------------------------------------------------------------------- */
typedef struct krt_plan krt_plan;

/* Parses model text (model_ir.py:281-330), hardware key=value text
 * (cost_model.py:308-339) and plan.json (plan.py:205-231). */
int krt_plan_load(const char* model_text, const char* hw_text, const char* plan_json,
                  krt_plan** out);
void krt_plan_free(krt_plan* plan);
/* plan_model (planner.py:890-912) in C++: partition, recompute flags and the
 * Algorithm-1 schedule, bit-identical to the reference planner.  strategy:
 * "eager" | "capacity" | "capacity-recompute"; solver: "auto" | "exhaustive" |
 * "dp"; max_blocks <= 0 = None.  KRT_INFEASIBLE carries InfeasibleModelError's
 * reason. */
int krt_plan_model(const char* model_text, const char* hw_text, const char* strategy,
                   const char* solver, int max_blocks, krt_plan** out);
/* Override hardware capacity (bytes) for validation / simulation. */
int krt_plan_set_capacity(krt_plan* plan, double capacity_bytes);

/* plan_string (plan.py:166-167), UTF-8 " → " separators; caller frees. */
int krt_plan_string(const krt_plan* plan, char** out);
/* plan_to_dict (plan.py:179-202) rendered as JSON; caller frees. */
int krt_plan_json(const krt_plan* plan, char** out);
/* validate_plan (planner.py:342-413): JSON array of violation strings; *n_violations
 * receives the count (0 = plan accepted). */
int krt_plan_validate(const krt_plan* plan, char** out_json, int* n_violations);
/* simulate (simulator.py:364-399): JSON {makespan,total_stall,peak_mem,events,csv}
 * or {deadlock:[...]}.  enforce_capacity as in the reference. */
int krt_plan_simulate(const krt_plan* plan, int enforce_capacity, char** out_json);

typedef struct krt_dist_config {
  int workers;        /* DistConfig.workers            (distsim.py:48) */
  int ring;           /* 1 = Collective.RING, 0 = FLAT (distsim.py:49) */
  double net_bw;      /* bytes/s                       (distsim.py:50) */
  double net_latency; /* seconds                       (distsim.py:51) */
  int groups;         /* 0 = one group per block       (distsim.py:52) */
  int variant;        /* bit 0: KRT_DIST_DEVICE_EXCHANGE, bit 1: KRT_DIST_EXACT_DEPS
                         (0 = the reference's model, bit-exact) */
} krt_dist_config;
/* The executor's P >= 2 pipeline: per group a device reduce-scatter
 * after the members' backward, a 1/P-shard grad_out, a 1/P host update, and a
 * shard weight_in followed by an "all_gather" network op before the forward. */
#define KRT_DIST_DEVICE_EXCHANGE 1
/* Shift each iteration's base-op deps by the real op offset (distsim.py:165
 * takes it before appending weight_in ops, so from iteration 2 deps point
 * too early: the reference's quirk, reproduced when the bit is clear). */
#define KRT_DIST_EXACT_DEPS 2

/* simulate_distributed (distsim.py:140-266): JSON {iteration_time, iteration_times,
 * exposed_comm, peak_mem, makespan, events} or {error}. */
int krt_plan_simulate_dist(const krt_plan* plan, const krt_dist_config* cfg, int iterations,
                           char** out_json);
/* block_cost per plan block (cost_model.py:250-273: fwd/bwd/swap seconds,
 * bytes, wt/grad bytes, weight elements) and layer_ops per layer with its kind
 * (cost_model.py:97-167): JSON {blocks[...], layers[{id, kind, ops}]}.  The
 * calibration (calibrate.py) fits measured op times against these. */
int krt_plan_costs(const krt_plan* plan, char** out_json);
/* analytic_report (occupancy.py:202-225) with find_theta (:178-199): JSON
 * {theta (null = None), mean_occupancy, per_step[[step, occupancy, busy_s,
 * idle_s]], csv (OccupancyReport.to_csv), summary (OccupancyReport.summary)}. */
int krt_plan_occupancy(const krt_plan* plan, char** out_json);

/* Static arena assignment for physical block sizes (block_bytes[i] = slot
 * bytes of block i+1): JSON {arena_bytes, ledger_peak, instances[{block, off,
 * bytes, alloc_op, free_op}], deps[[op, free_op]...]}.  Host-only; this is
 * what krt_prepare uses to realise the capacity ledger (simulator.py:90). */
int krt_plan_arena(const krt_plan* plan, const size_t* block_bytes, int n_blocks, char** out_json);

/* ------------------------------------------------------------------------
 * Executor context: one per rank / GPU.
 * ---------------------------------------------------------------------- */
typedef struct krt_ctx krt_ctx;

typedef struct krt_config {
  int device;               /* CUDA device ordinal */
  int world_size;           /* data-parallel workers (DistConfig.workers) */
  int rank;                 /* this worker */
  const void* nccl_id;      /* 128-byte ncclUniqueId (rank 0's) when world_size > 1 */
  int dist_groups;          /* gradient groups, 0 = one per block (distsim.py:52) */
  int weight_dtype;         /* enum krt_dtype: device copy of the weights */
  int optimizer;            /* enum krt_optim */
  float lr, beta1, beta2, eps, weight_decay, momentum;
  float grad_scale;         /* multiplies summed gradients (1/world_size = mean) */
  int host_threads;         /* host update worker threads, 0 = auto */
  size_t arena_slack_bytes; /* extra arena bytes beyond the static assignment */
  void* peer_group;         /* krt_peer_group* for in-process ranks (else NULL: NCCL) */
  int host_path_all;        /* 1: every block's update on the host even at world_size 1
                               (distsim.py:134-137 applies this from 2 workers) */
  int force_dp_path;        /* 1: data-parallel op structure (reduce-scatter / shard host
                               update / all-gather) even at world_size 1 (NCCL, 1 rank) */
  int ipc_exchange;         /* 1: exchange over CUDA IPC peer memory between processes
                               (own reduce kernel + D2D gather, stream-memop flags) */
  int grad_slots;           /* 0: one fp32 gradient region for the whole model; R > 0:
                               a ring of R group-sized gradient slots (group g uses slot
                               (g-1) mod R), each held from the group's first backward
                               until its exchange / grad_out / device update consumed it
                               (distsim.py:195-202 holds grad bytes only until grad_out) */
  int exchange_bf16;        /* 1: NCCL exchange in bf16: the group's fp32 gradients are cast
                               into a bf16 pack buffer (krt_reduce_cast), reduce-scattered in
                               bf16 (half the NVLink bytes) and the shard unpacked to fp32
                               for the D2H / host update */
} krt_config;

/* In-process exchange group: world_size ranks living in one process (threads),
 * e.g. logical ranks on one GPU or one process driving several GPUs.  The
 * reduce-scatter is the fused scale/cast/reduce kernel over the peers'
 * gradient buffers, the all-gather device-to-device copies. */
typedef struct krt_peer_group krt_peer_group;
int krt_peer_group_create(int world_size, krt_peer_group** out);
int krt_peer_group_destroy(krt_peer_group* group);

/* The executor's compute step for one plan op (KRT_FW, KRT_RECOMPUTE_FW,
 * KRT_BW) of `block`.  `slot` is the block's device arena slot
 * (slot_bytes long), `stream` the cudaStream_t all work must be issued on.
 * Return 0 on success. */
typedef int (*krt_compute_cb)(void* user, int action, int block, void* slot,
                              size_t slot_bytes, void* stream);

/* Flat parameter layout of the DP pipeline (host-only): blocks in order,
 * contiguous per gradient group (assign_groups, distsim.py:120-131), each
 * group padded to world*64 elements; rank r owns elements
 * [group_lo + r*shard_n, group_lo + (r+1)*shard_n) of every group.  Output
 * arrays: block_off[n_blocks]; group_lo/group_n/shard_n[n_blocks] (at most
 * n_blocks groups), *n_groups receives the group count. */
int krt_dp_layout(const int64_t* block_params, int n_blocks, int groups, int world,
                  int64_t* block_off, int* n_groups, int64_t* group_lo, int64_t* group_n,
                  int64_t* shard_n);

/* ncclGetUniqueId for rank 0 to broadcast (128 bytes into out). */
int krt_nccl_unique_id(void* out128);

int krt_create(const krt_config* cfg, krt_ctx** out);
int krt_destroy(krt_ctx* ctx);

/* One block's physical footprint: saved-activation bytes (the arena slot)
 * and the element counts of its parameter tensors in order.  Replaces the
 * analytic BlockCost.bytes / weight_elems (cost_model.py:225-273) with what
 * the block really stores.  Call for every block before krt_prepare. */
int krt_register_block(krt_ctx* ctx, int block, size_t act_bytes, const int64_t* param_numel,
                       int n_params);

/* Bind a validated plan: builds the op DAG (build_engine_ops + the DP ops),
 * the issue order (run_engine), the static arena assignment from the byte
 * ledger, and allocates device/pinned-host memory.  Fails with
 * KRT_INFEASIBLE if validate_plan rejects the plan or a block's physical
 * bytes exceed the plan's swap_bytes. */
int krt_prepare(krt_ctx* ctx, const krt_plan* plan);

enum krt_region {
  KRT_REGION_WEIGHTS = 0, /* device weights of a block (weight_dtype) */
  KRT_REGION_GRADS = 1,   /* device fp32 gradients of a block */
  KRT_REGION_ARENA = 2,   /* the whole device arena (block ignored) */
  KRT_REGION_HOST_SWAP = 3/* pinned host swap area of a block */
};
int krt_region(krt_ctx* ctx, int which, int block, void** ptr, size_t* bytes);
/* device stream handles: 0 compute, 1 H2D, 2 D2H, 3 network */
int krt_stream(krt_ctx* ctx, int which, void** stream);

/* Device address of `block`'s currently resident arena slot; valid inside a
 * compute callback (e.g. a recompute that regenerates its input from the
 * previous block, which the plan guarantees resident, plan.py:129-138). */
int krt_block_slot(krt_ctx* ctx, int block, void** slot);

/* Copy the device weights into the fp32 master copies (host shards for
 * host-path blocks, device masters otherwise).  Call once after writing the
 * initial weights into KRT_REGION_WEIGHTS. */
int krt_init_master(krt_ctx* ctx);

/* Run one training iteration: the plan's ops plus weight_in / grad_out /
 * exchange / host_update, issued in the simulator's start order with every
 * dependency, start gate and arena reuse expressed as CUDA events. */
int krt_run_iteration(krt_ctx* ctx, krt_compute_cb cb, void* user);
/* Wait for all device streams and host updates of the last iteration. */
int krt_synchronize(krt_ctx* ctx);

/* Cross-process exchange over NVLink peer memory (ipc_exchange = 1): after
 * krt_prepare every rank exports 3 CUDA IPC handles (weights, gradients,
 * flags; *len = 192 bytes), the ranks all-gather them (torch.distributed) and
 * each imports the world*192 bytes in rank order. */
int krt_ipc_export(krt_ctx* ctx, void* out, size_t cap, size_t* len);
int krt_ipc_import(krt_ctx* ctx, const void* handles, int world);

/* Measurement probe (bench.py's iteration roofline): mean seconds of one
 * ncclReduceScatter of `bytes` of fp32 gradients on the context's own
 * communicator and network stream, after 2 warm-ups.  Collective: every rank
 * calls it with the same arguments.  KRT_USAGE for IPC / in-process exchange. */
int krt_probe_exchange(krt_ctx* ctx, size_t bytes, int iters, double* seconds);
/* Wait for the last iteration, then return every host-updated weight to the
 * device copy now (the weight_in the next iteration would do), so the device
 * weights equal the masters — for evaluation and checkpoints. */
int krt_flush_weights(krt_ctx* ctx);

/* Checkpoint / restart of this rank's training state: after
 * the last iteration completes, write the device weights, device-path fp32
 * masters and moments, host-path masters/moments/weight staging and the
 * iteration counter to `path` (atomically: temp file + rename).  Load into a
 * context prepared with the same model, plan, dtype, world size and rank;
 * training then continues bitwise as if uninterrupted.  Errors: KRT_USAGE for
 * a mismatched or foreign file, KRT_INTERNAL for I/O failures. */
int krt_checkpoint_save(krt_ctx* ctx, const char* path);
int krt_checkpoint_load(krt_ctx* ctx, const char* path);

/* Measured trace of the last iteration in the SimTrace CSV schema
 * (simulator.py:225-230) extended with the DP ops; caller frees. */
int krt_trace_csv(krt_ctx* ctx, char** out);
/* JSON counters: bytes per direction, arena size, launches, ... ; caller frees. */
int krt_stats(krt_ctx* ctx, char** out_json);

/* Fetch the fp32 master weights of a block into host memory `out`
 * (numel floats); for world_size > 1 only this rank's shard is valid. */
int krt_read_master(krt_ctx* ctx, int block, float* out, size_t numel);

/* ------------------------------------------------------------------------
 * Kernels exposed for tests and the driver (all asynchronous on `stream`).
 * ---------------------------------------------------------------------- */
/* out[i] = (bf16|f32)(scale * sum_r in_r[i]) for r < n_in (fused grad
 * scale/cast/reduce; n_in = 1 is the plain pack). */
int krt_reduce_cast(const float* const* in, int n_in, void* out, int out_dtype, size_t n,
                    float scale, void* stream);
/* Device Adam/SGD over `n` fp32 elements; updates master/m/v in place and
 * writes the weight copy (weight_dtype).  Same arithmetic as the host path. */
int krt_device_update(float* master, float* m, float* v, const float* grad, void* weights,
                      int weight_dtype, size_t n, int optimizer, float lr, float beta1,
                      float beta2, float eps, float weight_decay, float momentum, int step,
                      void* stream);
/* Host Adam/SGD (the paper's CPU update kernel). */
int krt_host_update(float* master, float* m, float* v, const float* grad, void* weights,
                    int weight_dtype, size_t n, int optimizer, float lr, float beta1,
                    float beta2, float eps, float weight_decay, float momentum, int step,
                    int threads);

/* Fused NHWC batch-norm kernels for the convolutional units (bf16
 * activations [rows, C], C % 8 == 0, C <= 2048; gamma/beta bf16; stats fp32).
 * ws: krt_bn_workspace_bytes(C) bytes of device scratch. */
size_t krt_bn_workspace_bytes(int C);
/* batch statistics: mean[c], invstd[c] = 1/sqrt(var_biased + eps) */
int krt_bn_stats(const void* x, int64_t rows, int C, float eps, float* mean, float* invstd, void* ws,
                 void* stream);
/* krt_bn_stats then y = relu?( bn(x) [+ res] ) in one kernel (res NULL: none,
 * else identity residual); the apply pass walks the rows in reverse so the
 * tail the stats pass read last is still in L2 */
int krt_bn_stats_apply(const void* x, int64_t rows, int C, float eps, float* mean, float* invstd,
                       const void* gamma, const void* beta, const void* res, int relu, void* y, void* ws,
                       void* stream);
/* y = relu?( bn(x) [+ res | + bn'(res)] ); res NULL: no residual, rmean NULL: identity residual */
int krt_bn_apply(const void* x, const float* mean, const float* invstd, const void* gamma,
                 const void* beta, const void* res, const float* rmean, const float* rinvstd,
                 const void* rgamma, const void* rbeta, int relu, void* y, int64_t rows, int C,
                 void* stream);
/* dz = (dy [+ dy2]) * ( bn(x) + (res | bn'(res)) > 0 ): backward of the residual
 * add + ReLU; dy2 (may be NULL) is a second incoming gradient, summed and
 * rounded to bf16 first, so the producer never materialises dy + dy2 */
int krt_bn_add_relu_bwd(const void* dy, const void* dy2, const void* x, const float* mean, const float* invstd,
                        const void* gamma, const void* beta, const void* res, const float* rmean,
                        const float* rinvstd, const void* rgamma, const void* rbeta, void* dz,
                        int64_t rows, int C, void* stream);
/* BN backward with the optional ReLU mask recomputed from x: dgamma/dbeta (fp32,
 * may be NULL) and dx (bf16, may be NULL); addend (may be NULL) is a residual
 * gradient added to dx before its single bf16 rounding */
int krt_bn_backward(const void* dy, const void* x, const float* mean, const float* invstd,
                    const void* gamma, const void* beta, int relu, void* dx, float* dgamma,
                    float* dbeta, int64_t rows, int C, void* ws, const void* addend, void* stream);
/* krt_bn_add_relu_bwd (identity residual) and krt_bn_backward (no ReLU) of the
 * same BN in one kernel: dz = (dy [+ dy2]) * (bn(x) + res > 0) is written and
 * reduced in the same pass, then dx.  dz and dx required; dgamma/dbeta may be
 * NULL. */
int krt_bn_add_relu_backward(const void* dy, const void* dy2, const void* x, const float* mean,
                             const float* invstd, const void* gamma, const void* beta, const void* res,
                             void* dz, void* dx, float* dgamma, float* dbeta, int64_t rows, int C, void* ws,
                             void* stream);

/* ResNet stem: y = maxpool_{k,s,p}( relu(bn(x)) ), x NHWC bf16 [n,h,w,c], c % 8 == 0;
 * the post-BN activation is never written.  Bitwise equal to krt_bn_apply (relu)
 * followed by aten max_pool2d_with_indices. */
int krt_bn_relu_maxpool(const void* x, const float* mean, const float* invstd, const void* gamma,
                        const void* beta, void* y, int n, int h, int w, int c, int k, int s, int p,
                        void* stream);
/* Backward of the max-pool above: dx = d(pool)/d(relu(bn(x))) given dy, window
 * argmaxes recomputed from x (ws: krt_bn_relu_maxpool_bwd_workspace bytes);
 * bitwise equal to aten max_pool2d_with_indices_backward.  The ReLU/BN backward
 * follows with krt_bn_backward(relu=1). */
size_t krt_bn_relu_maxpool_bwd_workspace(int n, int h, int w, int c, int k, int s, int p);
int krt_bn_relu_maxpool_bwd(const void* dy, const void* x, const float* mean, const float* invstd,
                            const void* gamma, const void* beta, void* dx, void* ws, int n, int h, int w,
                            int c, int k, int s, int p, void* stream);

/* 1x1 convolution of NHWC bf16 activations as a tcgen05 GEMM (sm_100a):
 * C[M,N] = f(A)[M,K] . B[N,K]^T with A = activations [rows, Cin], B = weights
 * [Cout, Cin], C bf16.  f(A) = A, or relu(bn(A)) per input channel when pmean
 * is non-NULL (pmean/pinvstd fp32, pgamma/pbeta bf16; K <= 1024): the previous
 * BN's output is never written.  With part non-NULL (krt_conv1x1_partials_bytes
 * of device scratch) the epilogue also reduces the per-output-channel sums of
 * the stored C and C^2 into *part_rows partial rows, which
 * krt_bn_partials_finalize turns into mean/invstd: no statistics pass re-reads C.
 * Requirements: K in {16, 32} or K % 64 == 0, N in {16, 32, 64, 128} or
 * N % 256 == 0, 16-byte aligned pointers. */
size_t krt_conv1x1_partials_bytes(int N);
int krt_conv1x1_bn(const void* A, const void* B, void* C, int64_t M, int N, int K, const float* pmean,
                   const float* pinvstd, const void* pgamma, const void* pbeta, float* part, int* part_rows,
                   void* stream);
int krt_bn_partials_finalize(const float* part, int part_rows, int N, int64_t M, float eps, float* mean,
                             float* invstd, void* stream);
/* krt_conv1x1_bn plus a residual read in the epilogue: C = f(A) . B^T + res
 * (res [M, N] bf16, summed in fp32 before the one bf16 rounding; the partial
 * statistics are those of the stored sum).  The pre-activation bottleneck's
 * last convolution and shortcut add in one pass. */
int krt_conv1x1_bn_res(const void* A, const void* B, void* C, int64_t M, int N, int K, const float* pmean,
                       const float* pinvstd, const void* pgamma, const void* pbeta, const void* res, float* part,
                       int* part_rows, void* stream);
/* RGB NHWC bf16 [pixels, 3] -> [pixels, 4] with a zero 4th channel (the
 * stem's input for krt_conv_gather_bn: one 8-byte load per pixel); x 4-byte
 * and y 16-byte aligned. */
int krt_pad_rgb4(const void* x, void* y, int64_t pixels, void* stream);
/* Implicit-GEMM convolution for the ResNet stem (7x7/2, 3 -> 64 channels):
 * C[n*ho*wo, N] = im2col(x) . wk^T, x NHWC bf16 [n, h, w, cin], wk bf16 [N, K]
 * with column k = (kh*k + kw)*cin + c (zero beyond k*k*cin; K % 32 == 0,
 * K <= 1024), square kernel k, stride, zero padding pad.  The im2col rows are
 * gathered into the tcgen05 operand tiles in shared memory, never written to
 * HBM.  part/part_rows: BN statistics of C as krt_conv1x1_bn.  N = 64. */
int krt_conv_gather_bn(const void* x, const void* wk, void* C, int n, int h, int w, int cin, int ho, int wo, int k,
                       int stride, int pad, int N, int K, float* part, int* part_rows, void* stream);
/* Implicit-GEMM convolution on tcgen05 with im2col TMA tiles (the 3x3 and
 * strided convolutions of a bottleneck, cost_model.py:97-105):
 * C [n*ho*wo, N] bf16 = f(im2col_k,stride,pad(x)) . wk^T, x [n, h, w, cin]
 * NHWC bf16 (cin % 64 == 0), wk [N][k][k][cin] bf16 (OHWI), f = relu(bn(.))
 * per input channel when pmean is non-NULL (cin <= 1024; taps in the zero
 * padding stay zero).  part/part_rows: the BN statistics of C as
 * krt_conv1x1_bn (N in {64, 128} or N % 256 == 0).  With bx non-NULL this is
 * the dgrad form of krt_conv1x1_bn_dgrad instead: the epilogue reduces the
 * backward of the BN whose input is bx [n*ho*wo, N] into part (N in {64, 128}
 * or N % 128 == 0, no prologue); wk is then the flipped, transposed weight. */
int krt_conv_im2col_bn(const void* x, const void* wk, void* C, int n, int h, int w, int cin, int ho, int wo, int k,
                       int stride, int pad, int N, const float* pmean, const float* pinvstd, const void* pgamma,
                       const void* pbeta, float* part, int* part_rows, const void* bx, const float* bmean,
                       const float* binvstd, const void* bgamma, const void* bbeta, void* stream);
/* 1 when krt_conv_im2col_bn runs a 3x3 / stride-1 / pad-1 forward of this
 * shape on the halo-window kernel (csrc/halo_sm100.cu: each input pixel of a
 * 256-output-row window loaded, and with pmean transformed, once for all nine
 * taps; N in {64, 128}, cin % 64 == 0, the windows fit shared memory), 0 when
 * on the im2col-TMA GEMM.  KRT_CONV_HALO=0 in the environment disables the
 * halo kernel. */
int krt_conv3x3_halo_supported(int h, int w, int cin, int N, int prologue);
/* Weight gradient of a 3x3 / stride-1 / pad-1 convolution with few channels
 * (C = cin = cout in {16, 32, 64}: the ResNet-1001 bottleneck widths;
 * cost_model.py:97-105 counts this backward work for a Conv layer) from halo
 * windows on tcgen05: dw [C][3][3][C] fp32 (OHWI, written) = sum over the
 * pixels of dy [n, h, w, C] times the 3x3 window of f(x), x [n, h, w, C] NHWC
 * bf16, f = relu(bn(.)) per channel when pmean is non-NULL.  The pixel sum is
 * split over the SMs into fp32 partials summed in a fixed order
 * (deterministic); ws: krt_wgrad3x3_narrow_workspace(C) bytes.  _supported: 1
 * when the shape's windows fit (KRT_WGRAD_HALO=0 disables the kernel). */
/* Weight gradient of a 1x1 convolution with few channels (one side 64, 128
 * or 256 channels, the other 16, 32 or 64): dw [co][ci] fp32 (written) = sum
 * over the M pixels of dy [M, co] (x) f(x [M, ci]), NHWC bf16, f = relu(bn(.))
 * when pmean is non-NULL; deterministic; ws: krt_wgrad1x1_narrow_workspace. */
/* Weight gradient of the ResNet stem convolution (7x7 / stride 2 / pad 3, 3
 * input and 64 output channels; the counterpart of krt_conv_gather_bn) on
 * tcgen05: x4 [n, h, w, 4] NHWC bf16 (RGB padded to 4 channels, krt_pad_rgb4),
 * dc [n, ho, wo, 64] bf16 the output gradient -> dw [64][7][7][3] fp32 (OHWI,
 * written).  The 7x7 windows are gathered into shared memory, never written;
 * fixed-order CTA sums (deterministic); ws: krt_stem_wgrad_workspace() bytes. */
size_t krt_stem_wgrad_workspace(void);
int krt_stem_wgrad(const void* x4, const void* dc, float* dw, int n, int h, int w, void* ws, size_t ws_bytes,
                   void* stream);
int krt_wgrad1x1_narrow_supported(int ci, int co);
size_t krt_wgrad1x1_narrow_workspace(int ci, int co);
int krt_wgrad1x1_narrow(const void* x, const void* dy, float* dw, int64_t M, int ci, int co, const float* pmean,
                        const float* pinvstd, const void* pgamma, const void* pbeta, void* ws, size_t ws_bytes,
                        void* stream);
int krt_wgrad3x3_narrow_supported(int h, int w, int C);
size_t krt_wgrad3x3_narrow_workspace(int C);
int krt_wgrad3x3_narrow(const void* x, const void* dy, float* dw, int n, int h, int w, int C, const float* pmean,
                        const float* pinvstd, const void* pgamma, const void* pbeta, void* ws, size_t ws_bytes,
                        void* stream);
/* Weight gradient of a convolution on tcgen05 (the backward work
 * cost_model.py:97-105 counts for a Conv layer): dw [cout][k][k][cin] fp32
 * (OHWI, written, not accumulated) = sum over the output pixels of
 * dy [n, ho, wo, cout] times the k x k window (stride, zero padding pad) of
 * f(x), x [n, h, w, cin] NHWC bf16; f = relu(bn(.)) per input channel with
 * pmean/pinvstd fp32 and pgamma/pbeta bf16 (cin <= 1024) when pmean is
 * non-NULL: the BN output the forward convolved is never rebuilt in HBM.
 * The pixel reduction is split across the SMs into fp32 partial tiles summed
 * in a fixed order (deterministic); ws: krt_conv_wgrad_workspace_bytes.
 * cout % 128 == 0, cin % 64 == 0, k in {1, 3}, stride in {1, 2},
 * ho = (h + 2*pad - k)/stride + 1 (same for wo), 16-byte aligned pointers. */
size_t krt_conv_wgrad_workspace_bytes(int n, int ho, int wo, int cout, int cin, int k);
int krt_conv_wgrad(const void* dy, const void* x, float* dw, int n, int h, int w, int cin, int ho, int wo, int cout,
                   int k, int stride, int pad, const float* pmean, const float* pinvstd, const void* pgamma,
                   const void* pbeta, void* ws, size_t ws_bytes, void* stream);
/* Backward of a 1x1 convolution fused with the reduce of the BN (+ ReLU) in
 * front of it: dX[M,N] = dY[M,K] . Wt[N,K]^T (Wt = weights transposed, K-major)
 * is stored, and with x = that BN's input the epilogue reduces sum(gm) and
 * sum(gm * xhat), gm = dX * (relu(bn(x)) > 0), into *part_rows partial rows;
 * krt_bn_partials_bwd_finalize turns them into dgamma, dbeta and the dx
 * coefficients (coef [3][N]) that krt_bn_backward_elemt applies: the
 * separate reduce pass over (dX, x) is gone.  Shape rules as krt_conv1x1_bn. */
int krt_conv1x1_bn_dgrad(const void* dY, const void* Wt, void* dX, int64_t M, int N, int K, const void* x,
                         const float* mean, const float* invstd, const void* gamma, const void* beta,
                         float* part, int* part_rows, void* stream);
int krt_bn_partials_bwd_finalize(const float* part, int part_rows, int N, int64_t M, const float* mean,
                                 const float* invstd, const void* gamma, float* dgamma, float* dbeta,
                                 float* coef, void* stream);
/* dx = A*gm + B*x + D [+ addend] with gm = dy * (relu ? mask(x) : 1) and
 * coef [3][C] = A, B, D (from krt_bn_partials_bwd_finalize) */
int krt_bn_backward_elemt(const void* dy, const void* x, const float* mean, const float* invstd,
                          const void* gamma, const void* beta, const float* coef, const void* addend, int relu,
                          void* dx, int64_t rows, int C, void* stream);

/* GPT layers (bf16 rows [T, H], H % 8 == 0).  h = LayerNorm(x [+ r]) with
 * gamma/beta bf16 and the row mean/rstd (fp32) written; with r non-NULL the
 * sum x2 = bf16(x + r) is stored too (residual add fused in front of the
 * norm).  Deterministic: the backward recompute reproduces h bitwise. */
int krt_ln_fwd(const void* x, const void* r, void* x2, const void* gamma, const void* beta, void* h,
               float* mean, float* rstd, int64_t T, int H, float eps, void* stream);
/* LayerNorm backward in one pass: dx = rstd * (g*dy - mean(g*dy) - xhat *
 * mean(g*dy*xhat)) [+ addend] (bf16; the addend is the residual branch's
 * gradient), dgamma = sum_t dy*xhat, dbeta = sum_t dy (fp32, written, in a
 * fixed summation order).  mean/rstd: the forward's (krt_ln_fwd).  H <= 12288.
 * ws: krt_ln_bwd_workspace bytes. */
size_t krt_ln_bwd_workspace(int64_t T, int H);
int krt_ln_bwd(const void* dy, const void* x, const void* gamma, const float* mean, const float* rstd,
               const void* addend, void* dx, float* dgamma, float* dbeta, void* ws, int64_t T, int H, void* stream);
/* The LM head's next-token cross-entropy, forward and backward in one pass
 * over the logits (replaces the loss the reference's cost model counts as
 * the Softmax layer kind, model_ir.py:47-59, cost_model.py:139-148):
 * logits / dlogits bf16 [T, V] row-major, target int64 [T] (0 <= y < V),
 * row_loss[t] = logsumexp(z_t) - z_t[y_t] (fp32),
 * dlogits[t] = (softmax(z_t) - onehot(y_t)) * scale.  V % 8 == 0, V <= 65536. */
int krt_lm_xent(const void* logits, const int64_t* target, void* dlogits, float* row_loss, int64_t T, int V,
                float scale, void* stream);
/* The elementwise middle of an unfused causal attention backward (head dims
 * above 128, where cuDNN's fused backward is unavailable; the SelfAttention
 * layer kind, model_ir.py:47-59, cost_model.py:126-129): from the fp32
 * S = Q K^T and dP = dO V^T of `rows` = pairs x s query rows (s keys each),
 * lse (the forward's natural-log logsumexp of scale * S) and D = rowsum(dO * O),
 * writes P = exp(scale * S - lse) and dS = P * (dP - D) * scale as bf16,
 * both 0 above the diagonal.  s % 8 == 0. */
int krt_attn_softmax_bwd(const float* S, const float* dP, const float* lse, const float* D, void* P, void* dS,
                         int64_t rows, int s, float scale, void* stream);
/* dx = gelu_tanh'(f) * dy and colsum[n] = sum_t dx[t, n] (fp32, the bias
 * gradient of the layer that produced f) in one pass over the activations;
 * ws: krt_gelu_bwd_colsum_workspace bytes. */
size_t krt_gelu_bwd_colsum_workspace(int64_t T, int N);
int krt_gelu_bwd_colsum(const void* dy, const void* f, void* dx, float* colsum, void* ws, int64_t T, int N,
                        void* stream);
/* The GPT MLP's GEMMs with the bias / GELU work in the cuBLASLt epilogue
 * (library GEMMs; the fusion removes the elementwise passes around them).
 * Row-major bf16.  fc1: f1 = x [M, K] . w1 [N, K]^T + b1 [N] (the GELU input,
 * the epilogue's auxiliary output) and g = gelu_tanh(f1), both [M, N].
 * fc2 data gradient: df1 = (dy [M, K] . w2 [K, N]) * gelu_tanh'(f1) [M, N]
 * bf16 (fc1's bias gradient, the fp32 column sums of df1, is left to the
 * caller: cuBLASLt's DGELU_BGRAD sums only in the output type). */
int krt_mlp_fc1_gelu(const void* x, const void* w1, const void* b1, void* f1, void* g, int64_t M, int64_t N,
                     int64_t K, void* stream);
int krt_mlp_fc2_dgelu(const void* dy, const void* w2, const void* f1, void* df1, int64_t M, int64_t N, int64_t K,
                      void* stream);
/* fc2 with the layer's residual: y = x2 [M, N] + g [M, K] . w2 [N, K]^T +
 * b2 [N] (bias epilogue, beta = 1 on x2; y may alias x2). */
int krt_mlp_fc2_residual(const void* g, const void* w2, const void* b2, const void* x2, void* y, int64_t M,
                         int64_t N, int64_t K, void* stream);
/* A linear layer's weight and bias gradients in one cuBLASLt GEMM (BGRADB
 * epilogue): dy [M, N], x [M, K] row-major bf16 -> dw = dy^T x [N, K] and
 * db = sum over rows of dy [N], both fp32 (the gradient region's type). */
int krt_linear_wgrad_bgrad(const void* dy, const void* x, float* dw, float* db, int64_t M, int64_t N, int64_t K,
                           void* stream);

#ifdef __cplusplus
}
#endif
#endif /* KRT_H_ */
