/* tcb200.h -- C ABI of libtcb200.so, the sm_100a kernel library behind the
 * `b200` operator dialect.
 *
 * This is the drop-in boundary.  Every entry point replaces a
 * piece of the reference's executor API in /root/reference/proj/include/trainc:
 *
 *   tcb_plan_create  <- KernelCache::get(key, compile)      backends.hpp:340-354
 *                       (the "compile" half: shape-specialised launch plan)
 *   tcb_launch       <- Kernel::exec(TensorList)             backends.hpp:328-331
 *                       and exec_base(op, attrs, in, out_ty) backends.hpp:162-275
 *   tcb_plan_destroy <- KernelCache::clear                   backends.hpp:356-361
 *   tcb_reduce_scatter / tcb_all_gather / tcb_all_reduce
 *                    <- the collective ops' ref kernels      backends.hpp:245-273
 *                       (world>1 goes to NCCL instead of throwing)
 *   tcb_last_error   <- the trainc::Error what() string      dtype.hpp:15-39
 *
 * Conventions: every function returns an int status (TCB_OK = 0).  Tensors are
 * device memory owned by the caller; kernels never allocate.  Plans are
 * immutable after creation and may be shared across threads; launches are
 * stream-ordered and asynchronous.  No torch types appear here.
 */
#ifndef TCB200_H_
#define TCB200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* dtype codes.  0/1 match the TNSR codes of tensor.hpp:82 (f32, f16); 2 is the
 * bf16 extension; 3/4 are index/mask types. */
enum { TCB_F32 = 0, TCB_F16 = 1, TCB_BF16 = 2, TCB_I32 = 3, TCB_U8 = 4 };

/* status codes; the C++ shim maps them to the reference's exception types */
enum {
  TCB_OK = 0,
  TCB_ERR_UNIMPLEMENTED = 1, /* -> trainc::UnimplementedOp (dtype.hpp:30) */
  TCB_ERR_TYPE = 2,          /* -> trainc::TypeError       (dtype.hpp:24) */
  TCB_ERR_CUDA = 3,          /* -> trainc::Error                          */
  TCB_ERR_ARG = 4,           /* -> trainc::Error("internal: ...")         */
  TCB_ERR_PROTOCOL = 5       /* -> trainc::ProtocolError  (dtype.hpp:37)  */
};

#define TCB_MAX_RANK 8

typedef struct {
  void* ptr;                     /* device pointer, caller-owned */
  int32_t dtype;                 /* TCB_F32 ... */
  int32_t rank;
  int64_t shape[TCB_MAX_RANK];
  int64_t stride[TCB_MAX_RANK];  /* elements; 0 everywhere = dense row-major */
} tcb_tensor;

/* mirrors ir::AttrValue = variant<int64_t, double, string> (ir.hpp:29-30) */
enum { TCB_ATTR_INT = 0, TCB_ATTR_FLOAT = 1, TCB_ATTR_STR = 2 };
typedef struct {
  const char* key;
  int32_t kind;
  int64_t i;
  double d;
  const char* s;
} tcb_attr;

typedef struct tcb_plan_* tcb_plan;

/* Select the device for the calling thread and report its properties.
 * arena_bytes > 0 additionally cudaMalloc's an arena returned in *arena_base
 * (freed by tcb_free_arena).  One call per rank thread. */
int tcb_init(int device, uint64_t arena_bytes, void** arena_base);
int tcb_free_arena(void* arena_base);

/* Build a launch plan for `dialect_op` ("b200.<base op>") specialised to the
 * given input/output shapes, dtypes and attributes.  Pointers inside the
 * tensors are ignored here (they are bound at launch).  closure_hash may be
 * NULL.  Returns TCB_ERR_UNIMPLEMENTED when the op or this shape/dtype
 * combination has no b200 kernel -- there is no CPU fallback. */
int tcb_plan_create(const char* dialect_op, const tcb_tensor* in, int nin,
                    const tcb_tensor* out, int nout, const tcb_attr* attrs, int nattr,
                    const char* closure_hash, tcb_plan* plan);

/* Enqueue the plan on `stream` (a cudaStream_t; NULL = legacy default).
 * Shapes/dtypes must equal the ones the plan was created with. */
int tcb_launch(tcb_plan plan, const tcb_tensor* in, int nin, tcb_tensor* out, int nout,
               void* stream);

/* Launch with a caller-owned device WORKSPACE (>= tcb_plan_workspace_bytes).
 * Plans own no mutable device memory: every launch context (a VM, a rank
 * thread) passes its own workspace, so a plan shared through the process-wide
 * KernelCache is safe under concurrent launches on different streams.  Plain
 * tcb_launch uses a plan-owned fallback workspace (allocated on first use;
 * not for concurrent or captured use). */
int tcb_launch_ws(tcb_plan plan, const tcb_tensor* in, int nin, tcb_tensor* out, int nout, void* ws,
                  uint64_t ws_bytes, void* stream);
int tcb_plan_workspace_bytes(tcb_plan plan, uint64_t* bytes);
void tcb_plan_destroy(tcb_plan plan);

/* Deferred partial-sum folds (backend-internal scheduling; no reference
 * counterpart).  With deferral on, layer_norm_dx and colsum write their
 * per-block partials to a per-instance buffer carved from a pool of
 * pool_bytes and queue the fold; tcb_fold_flush folds every queued job in one
 * launch on `stream` (tcb_launch flushes by itself before any launch that
 * reads a pending output).  Results are bit-identical to folding in place.
 * tcb_fold_defer must be called outside stream capture. */
int tcb_fold_defer(int on, uint64_t pool_bytes);
int tcb_fold_flush(void* stream);
/* Per-launch-context fold pools: a VM creates one context (its partial-sum
 * slots live and die with it) and activates it on its thread before enqueueing
 * a step (tcb_fold_use(NULL) turns deferral off). */
int tcb_fold_ctx_create(uint64_t pool_bytes, void** ctx);
void tcb_fold_ctx_destroy(void* ctx);
int tcb_fold_use(void* ctx);
/* Cumulative counts: op launches whose fold kernel was deferred, and fold
 * kernels the flushes launched (kernels-per-step accounting). */
int tcb_fold_counters(uint64_t* ops_deferred, uint64_t* flush_launches);

/* Number of kernel launches this plan enqueues per tcb_launch (for the
 * bench's gpu_launches count). */
int tcb_plan_num_kernels(tcb_plan plan);

/* Human-readable key of a plan: "b200.op|shapes|dtypes|attrs". */
const char* tcb_plan_key(tcb_plan plan);

/* Space-separated list of base ops the b200 dialect implements (used by the
 * registration shim to call register_dialect_op once per op). */
const char* tcb_supported_ops(void);

/* ---- collectives (NCCL over NVLink; world == 1 is a local copy) ---------- */
/* ndev communicators for ndev devices in this process (ncclCommInitAll), or
 * one communicator per process when ndev == 1 and unique_id != NULL
 * (ncclCommInitRank).  unique_id is a 128-byte ncclUniqueId. */
int tcb_comm_unique_id(void* out128);
int tcb_comm_init_rank(const void* unique_id128, int world, int rank, void** comm);
int tcb_comm_init_all(int ndev, const int* devs, void** comms);
int tcb_comm_destroy(void* comm);
/* sum-reduce-scatter of a flat bucket: segs are concatenated views of one
 * contiguous buffer of `shard->shape[0] * world` elements (zero padded);
 * shard receives this rank's slice. */
int tcb_reduce_scatter(void* comm, const tcb_tensor* segs, int nseg, tcb_tensor* shard,
                       void* stream);
int tcb_all_gather(void* comm, const tcb_tensor* shard, tcb_tensor* segs, int nseg,
                   void* stream);
int tcb_all_reduce(void* comm, tcb_tensor* buf, void* stream);

/* ---- CUDA graphs ----------------------------------------------------------- */
int tcb_graph_capture_begin(void* stream);
int tcb_graph_capture_end(void* stream, void** graph_exec);
int tcb_graph_launch(void* graph_exec, void* stream);
int tcb_graph_destroy(void* graph_exec);

/* ---- device helpers used by the host runtime ------------------------------ */
int tcb_memcpy(void* dst, const void* src, uint64_t bytes, int kind /*0 h2d,1 d2h,2 d2d*/,
               void* stream);
int tcb_memset(void* dst, int value, uint64_t bytes, void* stream);
int tcb_stream_create(void** stream);
int tcb_stream_destroy(void* stream);
int tcb_stream_sync(void* stream);
int tcb_event_create(void** ev);
int tcb_event_record(void* ev, void* stream);
int tcb_stream_wait_event(void* stream, void* ev);
int tcb_event_elapsed_ms(void* start, void* stop, float* ms);
int tcb_event_destroy(void* ev);
int tcb_host_alloc(void** p, uint64_t bytes); /* pinned */
int tcb_host_free(void* p);
int tcb_device_sync(void);

/* thread-local message for the last non-zero status */
const char* tcb_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* TCB200_H_ */
