/*
 * rewind_b200.h — C ABI of the B200-native Swift recovery hot path.
 *
 * Drop-in boundary for the reference's C++ operator API (`namespace rewind`,
 * /root/reference/proj/core/include/rewind/ headers).  Every entry point names
 * the reference interface it replaces.  Conventions:
 *
 *  - plain pointers and sizes only; no C++ or torch types cross this line;
 *  - the caller owns all bulk device buffers (x, g, m, v, activations, ...);
 *    the library only allocates its own small metadata (group table copy,
 *    work lists) inside an rw_state and frees it in rw_state_destroy;
 *  - every GPU call is stream-ordered and asynchronous on the given
 *    cudaStream_t (passed as void*, NULL = legacy default stream);
 *  - status codes: 0 = OK, otherwise 1 + (int)rewind::Err
 *    (errors.hpp:11-33), so the C++ shim (rewind_b200.hpp) can rethrow the
 *    exact rewind::Error the reference would have raised; 100+ are
 *    B200-side failures (CUDA error, bad argument) with no reference twin;
 *  - guards are checked in the reference's order BEFORE any mutation
 *    (optim.cpp:262-270 for step, :289-292 plus the per-kind hyper checks for
 *    undo); NumericalError is detected in-kernel (fused check_finite,
 *    optim.cpp:283-285/:304-306) and reported after mutation by
 *    rw_state_check(), exactly like the reference raises after mutating;
 *  - thread-safe across distinct rw_state objects; one rw_state must not be
 *    used from two host threads at once (one owner per block).
 */
#ifndef REWIND_B200_H
#define REWIND_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RW_ABI_VERSION 1

/* ---- status codes: 1 + rewind::Err (errors.hpp:11-33) ---- */
enum {
  RW_OK = 0,
  RW_INVALID_SHAPE = 1,
  RW_SHAPE_MISMATCH = 2,
  RW_EMPTY_INPUT = 3,
  RW_NUMERICAL_ERROR = 4,
  RW_NON_INVERTIBLE_HYPER = 5,
  RW_NOT_INVERTIBLE = 6,
  RW_NOTHING_TO_UNDO = 7,
  RW_ALREADY_UPDATED = 8,
  RW_MISSING_ACTIVATION = 9,
  RW_CHANNEL_BROKEN = 10,
  RW_INVALID_INJECTION = 11,
  RW_NOT_FAILED = 12,
  RW_STORAGE_ERROR = 13,
  RW_MISSING_LOG_DATA = 14,
  RW_CORRUPT_LOG = 15,
  RW_NO_CHECKPOINT = 16,
  RW_NO_REPLICA = 17,
  RW_INVALID_CONFIG = 18,
  RW_TOO_LARGE = 19,
  RW_CUDA_ERROR = 100,
  RW_INVALID_ARGUMENT = 101
};

/* OptimizerKind, optim.hpp:16-23 (same order and values). */
enum { RW_SGD = 0, RW_SGDM = 1, RW_ADAM = 2, RW_ADAMW = 3, RW_LAMB = 4, RW_AMSGRAD = 5 };
/* Invertibility, optim.hpp:28. */
enum { RW_INVERTIBLE = 0, RW_INVERTIBLE_WITH_SAVED_SCALARS = 1, RW_NOT_INVERTIBLE_KIND = 2 };
/* element types of the flat state */
enum { RW_F32 = 0, RW_F64 = 1 };

/* OptimizerHyper, optim.hpp:34-50.  lr_table = (from_step, lr) breakpoints. */
typedef struct rw_hyper {
  int32_t kind;
  int32_t require_invertible;
  double lr;
  double weight_decay; /* lambda */
  double momentum;     /* mu  (SGD-momentum) */
  double dampening;    /* tau (SGD-momentum) */
  double beta1;
  double beta2;
  double eps;
  const uint64_t* lr_table_from;
  const double* lr_table_value;
  uint32_t lr_table_len;
  uint32_t _pad;
} rw_hyper;

/* One parameter group = one reference ParamBlock (optim.hpp:54-66) laid out
 * inside the flat x/g/m/v buffers.  (t, updated) is the update-progress
 * marker (optim.hpp:60-62); the kernels rewrite it in device memory when the
 * last element of the group has been stored. */
typedef struct rw_group {
  uint64_t offset;  /* element offset into the flat buffers */
  uint64_t len;     /* elements */
  uint64_t t;       /* completed steps */
  uint32_t updated; /* 1 = stepped in the current iteration */
  uint32_t flags;   /* bit0: non-finite value produced by the last step/undo */
} rw_group;

typedef struct rw_state rw_state;

/* ---- library ---- */
int rw_abi_version(void);
const char* rw_last_error_message(void); /* thread-local, message of the last failing call */
const char* rw_status_name(int status);  /* err_name (errors.cpp:8-31) for 1..19 */
int rw_device_count(void);

/* invertibility_check(OptimizerKind), optim.hpp:32 / optim.cpp:35-48 */
int rw_invertibility_check(int32_t kind);
/* OptimizerHyper::validate, optim.cpp:59-71 */
int rw_hyper_validate(const rw_hyper* h);
/* OptimizerHyper::lr_at, optim.cpp:50-57 */
int rw_lr_at(const rw_hyper* h, uint64_t t, double* out);

/* ---- flat optimizer state (the device form of a set of ParamBlocks) ----
 * x, g, m, v: caller-owned device buffers of `total` elements of `dtype`.
 * m, v may be NULL for optimizers that do not use them (SGD; SGDM: v).
 * vmax: AMSGrad running max (NULL otherwise).
 * groups: n_groups host records (offset/len/t/updated) copied into a
 * device-resident marker table owned by the state. */
int rw_state_create(rw_state** out, int32_t dtype, void* x, void* g, void* m, void* v,
                    void* vmax, uint64_t total, const rw_group* groups, uint32_t n_groups,
                    int32_t device);
/* A state for a HOST-resident replica (CPU offload, larger than HBM): the
 * group layout and the device marker table, no device x, g, m, v.  Only
 * rw_optimizer_undo_host and the marker calls operate on it; step / undo /
 * push calls fail with RW_INVALID_ARGUMENT. */
int rw_state_create_host(rw_state** out, int32_t dtype, uint64_t total, const rw_group* groups,
                         uint32_t n_groups, int32_t device);
void rw_state_destroy(rw_state* s);
uint32_t rw_state_num_groups(const rw_state* s);
int rw_state_info(const rw_state* s, int32_t* dtype, uint64_t* total, int32_t* device);
/* Behaviour flags of a state (default 0).
 * RW_STATE_LAMB_SEQUENTIAL_NORMS: the LAMB step forms ||x|| and ||update|| in
 *   the reference's left-to-right order (optim.cpp:199-208, one thread per
 *   group) instead of the parallel fixed-order tree, so the trust ratio -- and
 *   therefore x and the saved scalar -- equal rewind::optimizer_step's bit for
 *   bit (fp64).  O(n) per group on one thread: meant for parity / drop-in use
 *   (the host-block entry points set it); the default tree agrees to ~1e-15. */
enum { RW_STATE_LAMB_SEQUENTIAL_NORMS = 1 };
int rw_state_set_flags(rw_state* s, uint32_t flags);
/* Copy the device marker table to `out` (n_groups records).  Synchronises
 * `stream`.  The device table is authoritative after a crash-injected step. */
int rw_state_read_groups(rw_state* s, rw_group* out, void* stream);
/* Overwrite markers (host mirror and device table), e.g. when restoring a
 * checkpoint or receiving a broadcast state. */
int rw_state_write_groups(rw_state* s, const rw_group* in, void* stream);
/* Synchronise `stream`; return RW_NUMERICAL_ERROR if any step/undo since the
 * last check produced a non-finite x, m or v (and clear the flags). */
int rw_state_check(rw_state* s, void* stream);
/* End of iteration: clear the updated flag of the given groups (optim.hpp:62). */
int rw_clear_updated(rw_state* s, const uint32_t* group_ids, uint32_t n, void* stream);
/* Device pointers of the flat buffers (for collectives / copies). */
void* rw_state_ptr(rw_state* s, int which /*0 x,1 g,2 m,3 v,4 vmax*/);

/* LAMB saved scalars (ParamBlock::saved_scalars, optim.hpp / optim.cpp:216,
 * :241).  Each group keeps the last RW_LAMB_TRUST_DEPTH trust ratios on the
 * device (a step pushes, an undo pops; older entries fall off, so at most
 * RW_LAMB_TRUST_DEPTH consecutive undos find their ratio).  read copies the
 * stack bottom->top into out (at most cap) and its depth into *count
 * (synchronises `stream`); write replaces it (count <= RW_LAMB_TRUST_DEPTH),
 * e.g. on a replacement receiving a survivor's state. */
#define RW_LAMB_TRUST_DEPTH 8
int rw_state_saved_scalars(rw_state* s, uint32_t group, double* out, uint32_t cap, uint32_t* count,
                           void* stream);
int rw_state_set_saved_scalars(rw_state* s, uint32_t group, const double* in, uint32_t count, void* stream);

/* optimizer_step(ParamBlock&, const Tensor& grad, const OptimizerHyper&),
 * optim.hpp:71-72 / optim.cpp:260-286 — batched over `n` groups given in
 * UPDATE ORDER (apply_layerwise_updates: reverse layer order).
 * grad: flat device gradient in the same layout (NULL = g already holds it);
 * the kernel caches it into g (optim.cpp:271) in the same pass.
 * stop_after: crash injection MidUpdate(k): only the first
 * min(n, stop_after) groups in update order are stepped; UINT32_MAX = all.
 * Guards for ALL n groups are checked before anything is launched. */
int rw_optimizer_step(rw_state* s, const rw_hyper* h, const uint32_t* group_ids, uint32_t n,
                      const void* grad, uint32_t stop_after, void* stream);

/* optimizer_undo(ParamBlock&, const OptimizerHyper&), optim.hpp:76 /
 * optim.cpp:288-307 — batched over `n` groups.
 * LAMB (step and undo): the step runs a per-group norm pass (m, v, ||x||,
 * ||update|| in fp64 with a fixed reduction order) and then the fused x pass
 * with scaled = eta * trust; the undo reads the saved ratio (one D2H read) and
 * is one fused elementwise pass.  The trust ratio differs from the reference's
 * sequential sum in the last bits (documented tolerance; m, v are bit-exact)
 * unless the state has RW_STATE_LAMB_SEQUENTIAL_NORMS. */
int rw_optimizer_undo(rw_state* s, const rw_hyper* h, const uint32_t* group_ids, uint32_t n,
                      void* stream);

/* optimizer_undo for a state that lives in HOST memory in the same flat
 * layout (e.g. a CPU-offloaded replica): x, g, m, v are read from hx.. and
 * the undone x, m, v written to ox.. (may alias the inputs; when they do not,
 * groups that are not undone are copied through, so ox.. always receive the
 * whole resolved state).  Groups are cut into slices of ~slice_elems elements
 * (0 = 16M) in layout order; per slice H2D, undo and D2H run on three streams
 * as a pipeline through a ring of three device staging slices owned by `s`,
 * so both PCIe directions overlap the kernel and the device memory used is
 * bounded by three slices however large the host state is (the device
 * buffers of `s`, if any, are not touched).  Host buffers must be pinned for
 * the copies to be asynchronous.  Guards and markers exactly as
 * rw_optimizer_undo; ordered on `stream` (complete when it completes). */
int rw_optimizer_undo_host(rw_state* s, const rw_hyper* h, const uint32_t* group_ids, uint32_t n,
                           const void* hx, const void* hg, const void* hm, const void* hv, void* ox, void* om,
                           void* ov, uint64_t slice_elems, void* stream);

/* ---- replica recovery fused with the undo ----
 * CUDA IPC export/import of a device buffer so a survivor can write into a
 * replacement's HBM over NVLink.  export returns the 64-byte handle of the
 * enclosing allocation and the byte offset of ptr inside it. */
int rw_ipc_export(const void* ptr, void* handle_out /*64 bytes*/, uint64_t* offset_out);
int rw_ipc_import(const void* handle /*64 bytes*/, void** base_out);
int rw_ipc_close(void* base);
/* Copy-engine transfers between GPUs of one node (peer pointers from
 * rw_ipc_import): n async device-to-device copies on `stream` (DMA engines,
 * no kernels), and stream-ordered signalling through 64-bit epoch counters:
 * write_u64 stores `value` at addr (a local or peer device address) after
 * every prior operation of the stream has completed and is visible;
 * wait_u64 blocks `stream` until *addr >= value. */
int rw_copy_async(void* const* dsts, const void* const* srcs, const uint64_t* bytes, uint32_t n, void* stream);
int rw_stream_write_u64(void* stream, void* addr, uint64_t value);
int rw_stream_wait_u64(void* stream, const void* addr, uint64_t value);

/* apply_undo fused with recover_replication: undoes undo_ids in place and, in
 * the same kernel, streams every group of the resolved state (x, m, v; g too
 * when peer_g != NULL) into the peer replica's buffers (same layout) with
 * NVLink bulk stores.  Guards as rw_optimizer_undo.  The peer's markers are
 * the caller's to set (they equal the survivor's after the call). */
int rw_undo_and_push(rw_state* s, const rw_hyper* h, const uint32_t* undo_ids, uint32_t n_undo,
                     void* peer_x, void* peer_g, void* peer_m, void* peer_v, void* stream);

/* ---- host-buffer entry points: ONE reference ParamBlock held in host memory ----
 * Exactly optimizer_step / optimizer_undo (optim.cpp:260-307) on a block whose
 * x, g, m, v (and AMSGrad vmax) live in host memory: the library stages them
 * through device memory it owns (per calling thread), runs the fused kernel,
 * copies the results back and reports NumericalError like the reference
 * (after mutation).  dtype RW_F64 reproduces the reference bit for bit.
 * t/updated are the block's marker, read and written.  vmax may be NULL
 * except for AMSGrad; m/v may be NULL when the kind does not use them. */
int rw_host_block_step(int32_t dtype, void* x, void* g, void* m, void* v, void* vmax, uint64_t n,
                       uint64_t* t, uint32_t* updated, const void* grad, const rw_hyper* h);
int rw_host_block_undo(int32_t dtype, void* x, void* g, void* m, void* v, uint64_t n,
                       uint64_t* t, uint32_t* updated, const rw_hyper* h);
/* LAMB on a host ParamBlock: the block's saved_scalars stack stays with the
 * caller.  step returns the ratio step_lamb pushes (optim.cpp:216) in
 * *trust_out; undo takes the stack top (the caller pops it on RW_OK, :241).
 * rw_host_block_step/undo refuse RW_LAMB (they have no saved-scalar slot). */
int rw_host_block_lamb_step(int32_t dtype, void* x, void* g, void* m, void* v, uint64_t n, uint64_t* t,
                            uint32_t* updated, const void* grad, const rw_hyper* h, double* trust_out);
int rw_host_block_lamb_undo(int32_t dtype, void* x, void* g, void* m, void* v, uint64_t n, uint64_t* t,
                            uint32_t* updated, const rw_hyper* h, uint32_t have_saved, double trust);

/* ---- consistency resolver (no reference source) ---- */
enum { RW_ACT_NONE = 0, RW_ACT_UNDO = 1, RW_ACT_REDO = 2 };
enum { RW_POLICY_UNDO = 0 /* paper: always roll back to min */, RW_POLICY_MIN_COST = 1 };
enum { RW_STRATEGY_NONE = 0, RW_STRATEGY_UNDO = 1, RW_STRATEGY_REDO = 2, RW_STRATEGY_GLOBAL_ROLLBACK = 3 };

/* Per-rank summary exchanged with one MIN/MAX/SUM all-reduce each. */
typedef struct rw_resolve_summary {
  uint64_t t_min;          /* MIN over ranks: smallest group t (consensus_iteration) */
  uint64_t t_max;          /* MAX over ranks: largest group t */
  uint64_t undo_elems;     /* SUM-able: elements with t == t_min+1 (cost of undo) */
  uint64_t redo_elems;     /* elements with t == t_min (cost of redo) */
  uint64_t redo_blocked;   /* groups with t == t_min lacking a synchronised gradient */
  uint64_t undo_blocked;   /* 1 if the optimizer/hyper cannot be undone */
} rw_resolve_summary;

/* Local summary of one rank's markers.  grad_ready[i] != 0 means group i's
 * synchronised gradient for step t+1 has landed in the caller's gradient
 * buffer (NULL = none ready).  Two phases: t_floor = UINT64_MAX gives the
 * local t_min/t_max (all-reduce them MIN/MAX); then call again with
 * t_floor = the global t_min to get costs/blocks relative to it (all-reduce
 * the remaining fields with MAX).  n == 0 (a replacement holding no state)
 * yields t_min = UINT64_MAX and t_max = 0, the identities of MIN / MAX, so it
 * can join the all-reduces without moving the consensus. */
int rw_resolve_summarize(const rw_group* groups, uint32_t n, const uint8_t* grad_ready,
                         const rw_hyper* h, uint64_t t_floor, rw_resolve_summary* out);
/* Given the all-reduced summary (t_min MIN, t_max MAX, the rest MAX), pick a
 * strategy and target iteration, then the per-group actions for this rank. */
int rw_resolve_plan(const rw_resolve_summary* global, int32_t policy, const rw_group* groups,
                    uint32_t n, uint8_t* actions, uint64_t* target, int32_t* strategy);

/* ---- C++ recovery host over NCCL (recovery.cpp is absent) ----
 * The orchestration a C++ training system links in place of the reference's
 * missing recovery module: an NCCL communicator wrapper (nonblocking, so a
 * dead peer never wedges a host thread), the resolver's exchange, apply_undo,
 * replica recovery, the ordered merge of parallel recovery, and NCCL-native
 * failure detection and repair.  Every collective
 * runs on the communicator's own stream, ordered after the caller's `stream`
 * and back.  NCCL failures return RW_CHANNEL_BROKEN (the reference's
 * "detection signal"). */
typedef struct rw_comm rw_comm;
/* 128-byte ncclUniqueId (ncclGetUniqueId) for rw_comm_init, shared out of band */
int rw_nccl_unique_id(void* id_out);
/* ncclCommInitRankConfig with blocking = 0 on `device` */
int rw_comm_init(rw_comm** out, const void* unique_id, int32_t nranks, int32_t rank, int32_t device);
/* wrap an existing ncclComm_t (not owned: destroy leaves it alone) */
int rw_comm_from_nccl(rw_comm** out, void* nccl_comm);
int32_t rw_comm_rank(const rw_comm* c);
int32_t rw_comm_size(const rw_comm* c);
void* rw_comm_stream(rw_comm* c);   /* cudaStream_t the collectives run on */
void* rw_comm_nccl(rw_comm* c);     /* the ncclComm_t */
int rw_comm_destroy(rw_comm* c);    /* finalize + destroy (abort if the comm failed) */
int rw_comm_abort(rw_comm* c);      /* ncclCommAbort + free */

/* Failure detection: a thread polls ncclCommGetAsyncError every
 * poll_us and watches every collective this library enqueued; one that has
 * not completed after timeout_ms (0 = no timeout) marks the communicator
 * failed (fail-stop: the peer is gone).  Host waits inside the library then
 * return RW_CHANNEL_BROKEN instead of blocking.  A collective's host-side
 * phase (NCCL's lazy connection setup on a fresh communicator) is allowed
 * max(timeout_ms, 30 s); without a watch every host wait gives up after
 * 120 s. */
enum { RW_COMM_OK = 0, RW_COMM_FAILED_NCCL_ERROR = 1, RW_COMM_FAILED_TIMEOUT = 2 };
int rw_comm_watch(rw_comm* c, uint32_t poll_us, uint32_t timeout_ms);
/* reason = RW_COMM_*; detect_ms = age of the stuck collective when detected */
int rw_comm_failed(rw_comm* c, int32_t* reason, double* detect_ms);
/* Repair among the survivors (collective over them): ncclCommShrink excluding
 * the dead ranks, with NCCL_SHRINK_ABORT when `c` failed (its stuck kernels
 * are terminated first).  The parent is then released with rw_comm_abort. */
int rw_comm_shrink(rw_comm* c, const int32_t* exclude, int32_t n_exclude, rw_comm** out);

/* Heartbeat membership (the global key-value store of SPEC:253-261, here a
 * node-local shared file of per-rank CLOCK_MONOTONIC timestamps): rank r's
 * thread stamps slot r every beat_us (rank -1 = observer); dead() lists ranks
 * silent for more than timeout_ms (fail-stop).  A replacement opening a dead
 * rank's slot revives it. */
typedef struct rw_membership rw_membership;
int rw_membership_open(rw_membership** out, const char* path, int32_t rank, int32_t nranks, uint32_t beat_us);
int rw_membership_dead(rw_membership* m, uint32_t timeout_ms, int32_t* dead, int32_t cap, int32_t* n_dead);
int rw_membership_close(rw_membership* m);

/* consensus_iteration + per-group plan over the communicator:
 * reads s's markers (s == NULL: a replacement with no state yet, which joins
 * the exchange with the MIN/MAX identities), two exchanges (t_min MIN / t_max
 * MAX, then costs MAX), then rw_resolve_plan.  actions: rw_state_num_groups(s)
 * entries (RW_ACT_*). */
typedef struct rw_resolution {
  int32_t strategy;   /* RW_STRATEGY_* */
  uint32_t n_undo;    /* local groups to undo / redo */
  uint32_t n_redo;
  uint32_t _pad;
  uint64_t target;    /* consensus iteration after repair */
  uint64_t t_min, t_max;
} rw_resolution;
int rw_resolve(rw_state* s, const rw_hyper* h, rw_comm* c, int32_t policy, const uint8_t* grad_ready,
               uint8_t* actions, rw_resolution* out, void* stream);
/* apply_undo / redo: re-arms flags cleared at iteration end
 * (the decision is on t), undoes in reverse update order, or steps the
 * lagging groups with the synchronised gradient `grad` (redo).  Update order
 * is reverse layer order = descending group index. */
int rw_apply_resolution(rw_state* s, const rw_hyper* h, const uint8_t* actions, int32_t strategy, const void* grad,
                        void* stream);
/* apply_undo + recover_replication as one pipeline: the root
 * (the survivor) undoes its groups in `pieces` contiguous runs (0 = 16) on
 * `stream` while the communicator stream broadcasts each resolved run of x,
 * m, v (and g with RW_RECOVER_INCLUDE_GRAD) to every other rank; markers and
 * LAMB trust stacks follow.  Every rank passes its own state of the same
 * layout; non-roots pass actions = NULL.  *bytes_out = bytes per replacement. */
/* RW_RECOVER_CHAIN: instead of NCCL broadcasts, the resolved runs travel over
 * the copy engines as a chain (root -> next rank -> ...): each rank maps its
 * successor's buffers through CUDA IPC and forwards every run as soon as its
 * epoch counter lands (one GPU per rank on one node; the fastest transfer for
 * one replacement, profiles/r02). */
enum { RW_RECOVER_INCLUDE_GRAD = 1, RW_RECOVER_CHAIN = 2 };
int rw_recover_replication(rw_state* s, const rw_hyper* h, rw_comm* c, int32_t root, const uint8_t* actions,
                           int32_t strategy, uint32_t flags, uint32_t pieces, void* stream, uint64_t* bytes_out);

/* Ordered merge of parallel recovery: parts[mb] =
 * this rank's fp32 partial gradient of micro-batch mb (n elements) for every
 * mb with mb % nranks == rank (others NULL).  Rank j owns shard j (chunk =
 * rw_ordered_reduce_chunk elements), receives every partial's shard j, sums
 * them in ascending mb order (ordered_sum: bit-identical to the sequential
 * replay) and the shards are all-gathered: `out` (rw_ordered_reduce_out_elems
 * elements; the first n are the merged gradient) is the same on every rank. */
uint64_t rw_ordered_reduce_chunk(uint64_t n, int32_t nranks);
uint64_t rw_ordered_reduce_out_elems(uint64_t n, int32_t nranks);
uint64_t rw_ordered_reduce_scratch_elems(uint64_t n, uint32_t m, int32_t nranks, int32_t rank);
int rw_ordered_reduce(rw_comm* c, const float* const* parts, uint32_t m, uint64_t n, float* out, float* scratch,
                      uint64_t scratch_elems, void* stream);

/* ---- numerics ---- */
/* seeded_fill(shape, seed) (tensor.cpp:94-103) on the device, bit-identical to
 * the host (fp64) / its single rounding (fp32).  offset = first counter index. */
int rw_seeded_fill(int32_t dtype, void* out, uint64_t n, uint64_t seed, uint64_t offset,
                   void* stream);
uint64_t rw_derive_seed(uint64_t base, const uint64_t* parts, uint32_t n);
/* ordered_sum (tensor.cpp:105-117): out = ((t0 + t1) + t2) + ...;
 * tensors: host array of `count` device pointers of n elements. */
int rw_ordered_sum(int32_t dtype, const void* const* tensors, uint32_t count, uint64_t n,
                   void* out, void* stream);

/* ---- replay compute: one pipeline stage (model.hpp:16-70) ----
 * A stage is num_layers affine+tanh layers; dims[l] -> dims[l+1].  Weights are
 * bf16 [dims[l], dims[l+1]] row-major (the reference W layout, model.cpp:67,
 * `W[k*out+c]`), usually the bf16 shadow of the fp32 master x of the stage's
 * rw_state; biases are the fp32 master values.  Activations are bf16 [rows, dim]
 * row-major.  GEMMs run on the tcgen05 tensor cores (fp32 accumulation). */
enum { RW_BF16 = 2 };
typedef struct rw_stage_desc {
  int32_t num_layers;
  int32_t _pad;
  const int64_t* dims;      /* num_layers + 1 */
  const void* const* w;     /* num_layers bf16 device pointers */
  const float* const* b;    /* num_layers fp32 device pointers */
} rw_stage_desc;

/* forward_stage (model.cpp:77-92): acts[0] = the stage input (caller-filled);
 * acts[l+1] = tanh(acts[l] . W_l + b_l) is written (the activation cache the
 * backward consumes). */
int rw_stage_forward(const rw_stage_desc* st, int64_t rows, void* const* acts, void* stream);

/* backward_stage (model.cpp:94-156) + accumulate_grads (:158-172):
 * grad_in = dL/d(acts[L]) [rows, dims[L]] bf16; grad_out = dL/d(acts[0])
 * [rows, dims[0]] bf16 (NULL to skip the first layer's dgrad);
 * dw[l] fp32 [dims[l], dims[l+1]], db[l] fp32 [dims[l+1]]: overwritten when
 * accumulate == 0 (first micro-batch) else added (ascending micro-batch order,
 * ordered_sum semantics).  scratch: 2 bf16 buffers of rows*max(dims) elements
 * plus one fp32 buffer of 64*max(dims) elements. */
int rw_stage_backward(const rw_stage_desc* st, int64_t rows, void* const* acts, const void* grad_in,
                      void* grad_out, float* const* dw, float* const* db, int32_t accumulate,
                      void* scratch_dz0, void* scratch_dz1, float* scratch_f32, void* stream);
/* Same, for consecutive stages replayed on one GPU: grad_in_is_dz != 0 means
 * grad_in already holds this stage's last-layer dz (produced by the next
 * stage with prev_y); prev_y != NULL (the previous stage's output, i.e.
 * acts[0]) makes grad_out the PREVIOUS stage's last-layer dz instead of the
 * boundary gradient, computed from the bf16-rounded boundary gradient exactly
 * as that stage's own dtanh would (bit-identical to the unfused pair). */
int rw_stage_backward_ex(const rw_stage_desc* st, int64_t rows, void* const* acts, const void* grad_in,
                         int32_t grad_in_is_dz, void* grad_out, const void* prev_y, float* const* dw,
                         float* const* db, int32_t accumulate, void* scratch_dz0, void* scratch_dz1,
                         float* scratch_f32, void* stream);

/* rw_stage_backward_ex with the fp32 scratch size stated (elements).  When it
 * holds ceil(rows/32) * max(dims) floats, the column sums (db) of every dz that
 * a dgrad GEMM produces are formed in that GEMM's epilogue (per 32-row block,
 * from the bf16 values it stores) and only the ceil(rows/32) partial rows are
 * summed afterwards (in row order), instead of re-reading dz; otherwise, and
 * for the layer whose dz comes in, the separate column-sum pass runs. */
int rw_stage_backward_ex2(const rw_stage_desc* st, int64_t rows, void* const* acts, const void* grad_in,
                          int32_t grad_in_is_dz, void* grad_out, const void* prev_y, float* const* dw,
                          float* const* db, int32_t accumulate, void* scratch_dz0, void* scratch_dz1,
                          float* scratch_f32, uint64_t scratch_f32_elems, void* stream);

/* Keep n SMs free of the replay GEMM grids (0 = use every SM), so that
 * collectives issued concurrently (parallel-recovery merges) get SMs: the
 * persistent GEMM's static tile schedule would otherwise wait for its last
 * CTA behind a collective kernel.  Process-wide. */
int rw_replay_set_sm_reserve(int32_t n);

/* Replay GEMM engine (process-wide; -1 keeps the default / environment):
 *   epilogue: 1 = output tiles staged in shared memory and written by TMA
 *             tensor stores (default), 0 = per-thread register stores;
 *   pair:     2 = wide CTA-pair kernel (cta_group::2, 256 rows per CTA,
 *                 512 x 256 tiles per cluster; default),
 *             1 = CTA-pair kernel (cta_group::2, 128 rows per CTA),
 *             0 = single-CTA kernel (cta_group::1, M = 128).
 * Every combination gives the same bits (same MMA order, same epilogue
 * arithmetic); the knob exists for A/B measurements and tests. */
int rw_replay_set_gemm_engine(int32_t epilogue, int32_t pair);

/* mse_loss (model.cpp:174-188): grad = 2/(n*micro_batches) * (pred - target)
 * (bf16 out); *loss (device double, may be NULL) = mean squared error.
 * scratch: 256 doubles. */
int rw_mse_grad(const void* pred_bf16, const float* target, uint64_t n, uint64_t micro_batches,
                void* grad_bf16, double* loss, double* scratch, void* stream);
/* fp32 -> bf16 (weight shadows after an optimizer step) */
int rw_cast_f32_to_bf16(const float* in, void* out, uint64_t n, void* stream);

/* ---- replay drivers in C++  ----
 * One stage of the replayed group: its descriptor (bf16 weight shadows w[l],
 * fp32 biases b[l] = the master x of the bias blocks), its fp32 master state
 * (blocks W0, b0, W1, b1, ... in blocks() order, model.cpp:12-20) and a flat
 * fp32 gradient buffer in the state's layout. */
typedef struct rw_replay_stage {
  rw_stage_desc desc;
  rw_state* state;
  float* grad;
} rw_replay_stage;
/* The group's inbound log, one entry per (iteration - it0) * micro_batches + mb
 * in timestamp order: activations entering its first stage (bf16 [rows,
 * dims_in]) and gradients entering its last stage (bf16 [rows, dims_out]),
 * device pointers.  acts == NULL: the group starts the pipeline and the inputs
 * are re-derived (synth_inputs, model.cpp:190-193); grads == NULL: it ends the
 * pipeline and the gradient is mse_loss against synth_targets (:174-198).  A
 * NULL entry is MissingLogData. */
typedef struct rw_replay_log {
  const void* const* acts;
  const void* const* grads;
  uint64_t seed;
} rw_replay_log;
/* device workspace both drivers need (comm == NULL: rw_replay_group) */
uint64_t rw_replay_workspace_bytes(const rw_replay_stage* stages, uint32_t n_stages, int64_t rows,
                                   uint32_t micro_batches, rw_comm* comm);
/* recover_replay: the group's checkpoint is already loaded in
 * the stage states; iterations [it0, it1) are re-executed from the log: every
 * micro-batch forward + backward in timestamp order, gradients accumulated in
 * ascending micro-batch order (accumulate_grads), then one step of every
 * block in reverse layer order, the flag clear and the shadow refresh.  Equal
 * to the failure-free run bit for bit. */
int rw_replay_group(const rw_replay_stage* stages, uint32_t n_stages, int64_t rows, uint32_t micro_batches,
                    uint64_t it0, uint64_t it1, const rw_hyper* h, const rw_replay_log* log, void* workspace,
                    uint64_t workspace_bytes, void* stream);
/* recover_parallel for this helper (rank of `comm`, d = its
 * size): micro-batches {mb : mb mod d == rank} each into its own
 * partial gradients, rw_ordered_reduce per stage (ascending mb), the
 * same step on every helper.  Bit-identical to rw_replay_group. */
int rw_recover_parallel(const rw_replay_stage* stages, uint32_t n_stages, int64_t rows, uint32_t micro_batches,
                        uint64_t it0, uint64_t it1, const rw_hyper* h, const rw_replay_log* log, rw_comm* comm,
                        void* workspace, uint64_t workspace_bytes, void* stream);

/* ---- logging capture path (logstore.cpp missing) ----
 * Upstream-backup log of inter-machine boundary tensors.  rw_logger_log never
 * blocks the producer stream: it orders a CRC32 kernel and a D2H copy into a
 * pinned slab on the logger's own stream (the paper's dedicated copy
 * stream), and pushes the record onto a single-producer/single-consumer
 * queue; a native committer thread waits for the copy event and appends the
 * record to the current chunk file.  Chunk files hold `chunk_records`
 * records: "SWFT" | u16 version | u32 machine, then length-prefixed
 * little-endian records (header, payload, CRC32 of the payload), written to
 * a .tmp name and renamed into place when complete (atomic commit). */
enum { RW_LOG_ACTIVATION = 0, RW_LOG_GRADIENT = 1 };
typedef struct rw_log_record {
  uint32_t sender;          /* LogRecord fields */
  uint32_t receiver;
  uint64_t iteration;
  uint32_t mb;
  uint32_t direction;       /* RW_LOG_ACTIVATION / RW_LOG_GRADIENT */
  uint32_t dtype;           /* RW_F32 / RW_F64 / RW_BF16 */
  uint32_t ndim;            /* <= 4 */
  uint64_t shape[4];
  uint64_t payload_bytes;
  uint32_t crc32;           /* CRC32 of the payload (wire.cpp:31-38) */
  uint32_t _pad;
} rw_log_record;

/* CRC32 of a device buffer, written to *out_dev (device memory). */
int rw_crc32_device(const void* data, uint64_t n, uint32_t* out_dev, void* stream);

typedef struct rw_logger rw_logger;
int rw_logger_create(rw_logger** out, const char* dir, uint32_t machine, uint32_t chunk_records,
                     uint64_t pinned_bytes, int32_t device);
/* log_send: rec's shape/ids/dtype; payload_bytes = bytes of dev_payload. */
int rw_logger_log(rw_logger* lg, const rw_log_record* rec, const void* dev_payload, void* producer_stream);
/* flush_logs: drain the queue, commit the partial chunk. */
int rw_logger_flush(rw_logger* lg, uint64_t* records_committed);
int rw_logger_destroy(rw_logger* lg);
/* The logger's copy stream (cudaStream_t): a caller whose device memory
 * allocator is stream-ordered marks each logged payload as used on it, so the
 * memory is recycled only after the D2H has read it (no keep-alive list). */
void* rw_logger_stream(rw_logger* lg);

typedef struct rw_log_reader rw_log_reader;
int rw_log_open(rw_log_reader** out, const char* path, uint32_t* machine);
/* next record header + payload into `payload` (cap bytes); *eof = 1 at end.
 * RW_CORRUPT_LOG on a malformed file.  The payload CRC is checked by the
 * caller on the device (rw_crc32_device) against rec->crc32. */
int rw_log_next(rw_log_reader* r, rw_log_record* rec, void* payload, uint64_t cap, int32_t* eof);
void rw_log_close(rw_log_reader* r);
/* Header-only walk (payload skipped, CRC not checked): used by rw_log_gc. */
int rw_log_skip(rw_log_reader* r, rw_log_record* rec, int32_t* eof);

/* ---- global checkpoint store (no reference source) ----
 * write: every blob of this worker (device buffers via a pinned, pipelined
 * D2H; host buffers directly), each fsync'd, CRC32 (wire.cpp polynomial; on
 * the GPU for device blobs) recorded in the worker manifest, which is then
 * committed atomically.  crash_after_blobs: test hook, UINT32_MAX = none.
 * commit: once all n_workers manifests exist, atomically publish
 * MANIFEST_<iteration> — the checkpoint is visible iff that file exists.
 * latest: highest committed iteration (NoCheckpoint if none).
 * load: NoCheckpoint if the iteration is not committed; ShapeMismatch if a
 * blob's size differs; StorageError on a missing/truncated blob or a CRC
 * mismatch (recomputed on the GPU after the H2D). */
typedef struct rw_blob {
  const char* name;  /* [A-Za-z0-9._-]+ */
  void* data;
  uint64_t bytes;
  uint32_t on_host;  /* 1: data is host memory */
  uint32_t pad;
} rw_blob;
int rw_ckpt_write(const char* dir, uint64_t iteration, uint32_t worker, const rw_blob* blobs, uint32_t n,
                  uint32_t crash_after_blobs, void* stream);
int rw_ckpt_commit(const char* dir, uint64_t iteration, uint32_t n_workers);
int rw_ckpt_latest(const char* dir, uint64_t* iteration);
int rw_ckpt_blob_bytes(const char* dir, uint64_t iteration, uint32_t worker, const char* name, uint64_t* bytes);
int rw_ckpt_load(const char* dir, uint64_t iteration, uint32_t worker, const rw_blob* blobs, uint32_t n,
                 void* stream);
/* gc_logs: delete every log chunk in log_dir whose records
 * all have iteration < ckpt_iteration; NoCheckpoint unless that checkpoint is
 * committed in ckpt_dir.  Idempotent. */
int rw_log_gc(const char* log_dir, const char* ckpt_dir, uint64_t ckpt_iteration, uint32_t* deleted);

/* ---- selective-logging policy (planner.cpp missing) ---- */
/* bubble_ratio(p, m), schedule.cpp:86-93 */
int rw_bubble_ratio(int32_t p, int32_t m, int64_t* num, int64_t* den);
/* group_machines(profile).  R[N] seconds, M[N-1] bytes per
 * boundary per iteration, B bytes/s, T iterations, M_max bytes.
 * group_of[N] receives each machine's group index; *n_groups the count;
 * *storage = M(G), *recovery = expected recovery time per lost iteration. */
int rw_group_machines(uint32_t N, const double* R, const double* M, double B, double T,
                      double M_max, int32_t parallel, uint32_t* group_of, uint32_t* n_groups,
                      double* storage, double* recovery);
/* recovery_time_estimate(plan, lost_iterations) */
int rw_recovery_time_estimate(uint32_t N, const double* R, const double* M, double B,
                              int32_t parallel, const uint32_t* group_of,
                              double lost_iterations, double* out);
/* logging_worthwhile */
int rw_logging_worthwhile(double bytes_per_iteration, double pcie_bytes_per_s, int32_t p,
                          int32_t m, double iteration_time_s, int32_t* worthwhile,
                          double* transfer_s, double* bubble_s);

#ifdef __cplusplus
}
#endif
#endif /* REWIND_B200_H */
