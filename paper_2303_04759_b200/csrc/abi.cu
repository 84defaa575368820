// abi.cu -- the extern "C" surface of libtcb200.so (include/tcb200.h).
//
// tcb_plan_create is the "compile" half of KernelCache::get (backends.hpp:340-354):
// it validates shapes/dtypes/attrs for one dialect op and freezes a launch
// closure; tcb_launch is Kernel::exec (backends.hpp:328-331) but asynchronous on
// a CUDA stream.  Unknown ops / unsupported dtype combinations return
// TCB_ERR_UNIMPLEMENTED: there is no CPU fallback anywhere in this library.
#include <mutex>
#include <sstream>

#include "common.cuh"
#include "fold.cuh"

namespace tcb {

static std::map<std::string, Builder>& builders() {
  static std::map<std::string, Builder> m;
  return m;
}
void register_builder(const char* op, Builder b) { builders()[op] = b; }

static thread_local std::string g_last_error;

static int set_err(int code, const std::string& m) {
  g_last_error = m;
  return code;
}

static Spec to_spec(const tcb_tensor& t) {
  Spec s;
  s.dtype = t.dtype;
  s.rank = t.rank;
  if (t.rank < 0 || t.rank > TCB_MAX_RANK) fail(TCB_ERR_ARG, "bad rank");
  for (int i = 0; i < t.rank; ++i) {
    if (t.shape[i] < 1) fail(TCB_ERR_TYPE, "tensor dimension must be >= 1");
    s.shape[i] = t.shape[i];
  }
  for (int i = 0; i < t.rank; ++i)
    if (t.stride[i] != 0) fail(TCB_ERR_UNIMPLEMENTED, "strided tensors are not supported");
  return s;
}

static std::string spec_str(const Spec& s) {
  std::string r = dtype_name(s.dtype);
  r += '[';
  for (int i = 0; i < s.rank; ++i) {
    if (i) r += ',';
    r += std::to_string(s.shape[i]);
  }
  return r + ']';
}

}  // namespace tcb

struct tcb_plan_ {
  tcb::Plan p;
  bool rng_in = false;  // launches carry a trailing rng_step input
  // fallback workspace for callers of plain tcb_launch (tests, one-off ops):
  // allocated on first such launch (never during capture), serialised by mu
  std::mutex mu;
  std::unique_ptr<tcb::Scratch> own_ws;
};

namespace tcb {
char*& launch_ws() {
  thread_local char* w = nullptr;
  return w;
}
const float*& launch_rng() {
  thread_local const float* r = nullptr;
  return r;
}
}  // namespace tcb

using namespace tcb;

#define TCB_TRY(body)                                   \
  try {                                                 \
    body;                                               \
    return TCB_OK;                                      \
  } catch (const tcb::Status& s) {                      \
    return set_err(s.code, s.what());                   \
  } catch (const std::exception& e) {                   \
    return set_err(TCB_ERR_ARG, e.what());              \
  }

extern "C" {

const char* tcb_last_error(void) { return g_last_error.c_str(); }

int tcb_last_error_set(int code, const char* m) { return set_err(code, m ? m : ""); }

int tcb_init(int device, uint64_t arena_bytes, void** arena_base) {
  TCB_TRY({
    TCB_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    TCB_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
      fail(TCB_ERR_UNIMPLEMENTED, std::string("libtcb200 targets sm_100a; device is ") + prop.name);
    if (arena_bytes && arena_base) TCB_CUDA(cudaMalloc(arena_base, arena_bytes));
  });
}

int tcb_free_arena(void* arena_base) { TCB_TRY(TCB_CUDA(cudaFree(arena_base))); }

int tcb_plan_create(const char* dialect_op, const tcb_tensor* in, int nin, const tcb_tensor* out,
                    int nout, const tcb_attr* attrs, int nattr, const char* closure_hash,
                    tcb_plan* plan) {
  TCB_TRY({
    std::string name = dialect_op ? dialect_op : "";
    std::string base = name;
    if (name.rfind("b200.", 0) == 0) base = name.substr(5);
    else if (name.find('.') != std::string::npos)
      fail(TCB_ERR_UNIMPLEMENTED, "libtcb200 only implements the b200 dialect, got " + name);
    auto it = builders().find(base);
    if (it == builders().end())
      fail(TCB_ERR_UNIMPLEMENTED, "no b200 kernel for op " + base);
    auto* pl = new tcb_plan_();
    Plan& p = pl->p;
    p.op = base;
    try {
      for (int i = 0; i < nin; ++i) p.in.push_back(to_spec(in[i]));
      for (int i = 0; i < nout; ++i) p.out.push_back(to_spec(out[i]));
      std::ostringstream key;
      key << "b200." << base << "|";
      for (auto& s : p.in) key << spec_str(s) << ",";
      key << "->";
      for (auto& s : p.out) key << spec_str(s) << ",";
      key << "|";
      for (int i = 0; i < nattr; ++i) {
        tcb_attr a = attrs[i];
        p.attrs.strs.push_back(a.key ? a.key : "");
        if (a.kind == TCB_ATTR_STR) p.attrs.strs.push_back(a.s ? a.s : "");
      }
      // second pass: point keys/strings at owned storage (strs no longer grows)
      size_t si = 0;
      for (int i = 0; i < nattr; ++i) {
        tcb_attr a = attrs[i];
        a.key = p.attrs.strs[si++].c_str();
        if (a.kind == TCB_ATTR_STR) a.s = p.attrs.strs[si++].c_str();
        p.attrs.m[a.key] = a;
      }
      for (auto& [k, a] : p.attrs.m) {
        key << k << "=";
        if (a.kind == TCB_ATTR_INT) key << a.i;
        else if (a.kind == TCB_ATTR_FLOAT) key << a.d;
        else key << a.s;
        key << ";";
      }
      if (closure_hash) key << "|" << closure_hash;
      p.key = key.str();
      // rng_in=1: the caller appends the training step's rng_step (f32[1]) as
      // the last input of every launch; kernels key their dropout masks on it
      if (p.attrs.i("rng_in", 0)) {
        require(!p.in.empty() && p.in.back().numel() == 1 && p.in.back().dtype == TCB_F32,
                "b200." + base + ": rng_in expects a trailing f32[1] rng_step input");
        p.in.pop_back();
        pl->rng_in = true;
      }
      it->second(p);
      if (!p.run) fail(TCB_ERR_UNIMPLEMENTED, "b200." + base + ": no kernel for this configuration");
    } catch (...) {
      delete pl;
      throw;
    }
    *plan = pl;
  });
}

// Profiling knob, never set in tests or the bench: TCB_SKIP_OPS="op1,op2" makes
// tcb_launch return without launching those ops, so a step's time can be
// attributed per op class by difference (outputs are then garbage).
static bool skipped_op(const std::string& op) {
  static const std::string list = [] {
    const char* e = std::getenv("TCB_SKIP_OPS");
    return e ? "," + std::string(e) + "," : std::string();
  }();
  return !list.empty() && list.find("," + op + ",") != std::string::npos;
}

static void launch_with(tcb_plan plan, const tcb_tensor* in, int nin, tcb_tensor* out, int nout, void* ws,
                        uint64_t ws_bytes, void* stream) {
  if (!plan) fail(TCB_ERR_ARG, "null plan");
  Plan& p = plan->p;
  if (nin != int(p.in.size()) + int(plan->rng_in) || nout != int(p.out.size()))
    fail(TCB_ERR_ARG, "b200." + p.op + ": launch arity differs from plan");
  if (p.ws_bytes && ws && ws_bytes < p.ws_bytes)
    fail(TCB_ERR_ARG, "b200." + p.op + ": workspace of " + std::to_string(ws_bytes) + " B < the plan's " +
                          std::to_string(p.ws_bytes) + " B");
  if (skipped_op(p.op)) return;
  // a deferred fold whose output this launch reads is folded first
  for (int i = 0; i < int(p.in.size()); ++i)
    fold_flush_if_reads(in[i].ptr, size_t(p.in[i].numel()) * dtype_bytes(p.in[i].dtype),
                        static_cast<cudaStream_t>(stream));
  struct Reset {
    ~Reset() {
      launch_ws() = nullptr;
      launch_rng() = nullptr;
    }
  } reset;
  launch_ws() = static_cast<char*>(ws);
  launch_rng() = plan->rng_in ? static_cast<const float*>(in[nin - 1].ptr) : nullptr;
  p.run(in, out, static_cast<cudaStream_t>(stream));
  TCB_CUDA(cudaGetLastError());
}

int tcb_launch_ws(tcb_plan plan, const tcb_tensor* in, int nin, tcb_tensor* out, int nout, void* ws,
                  uint64_t ws_bytes, void* stream) {
  TCB_TRY({
    if (plan && plan->p.ws_bytes && !ws) fail(TCB_ERR_ARG, "b200." + plan->p.op + ": needs a workspace");
    launch_with(plan, in, nin, out, nout, ws, ws_bytes, stream);
  });
}

int tcb_launch(tcb_plan plan, const tcb_tensor* in, int nin, tcb_tensor* out, int nout,
               void* stream) {
  TCB_TRY({
    if (!plan) fail(TCB_ERR_ARG, "null plan");
    void* ws = nullptr;
    if (plan->p.ws_bytes) {
      std::lock_guard<std::mutex> g(plan->mu);
      if (!plan->own_ws) plan->own_ws = std::make_unique<Scratch>(plan->p.ws_bytes);
      ws = plan->own_ws->p;
    }
    launch_with(plan, in, nin, out, nout, ws, plan->p.ws_bytes, stream);
  });
}

int tcb_plan_workspace_bytes(tcb_plan plan, uint64_t* bytes) {
  TCB_TRY({
    if (!plan || !bytes) fail(TCB_ERR_ARG, "tcb_plan_workspace_bytes: null argument");
    *bytes = plan->p.ws_bytes;
  });
}

void tcb_plan_destroy(tcb_plan plan) { delete plan; }

int tcb_fold_defer(int on, uint64_t pool_bytes) { TCB_TRY(fold_set(on != 0, size_t(pool_bytes))); }

int tcb_fold_ctx_create(uint64_t pool_bytes, void** ctx) {
  TCB_TRY({
    if (!ctx) fail(TCB_ERR_ARG, "tcb_fold_ctx_create: null output");
    *ctx = fold_ctx_create(size_t(pool_bytes));
  });
}
void tcb_fold_ctx_destroy(void* ctx) { fold_ctx_destroy(static_cast<FoldCtx*>(ctx)); }
int tcb_fold_use(void* ctx) { TCB_TRY(fold_use(static_cast<FoldCtx*>(ctx))); }

int tcb_fold_flush(void* stream) { TCB_TRY(fold_flush(static_cast<cudaStream_t>(stream))); }

int tcb_fold_counters(uint64_t* ops_deferred, uint64_t* flush_launches) {
  TCB_TRY({
    if (!ops_deferred || !flush_launches) fail(TCB_ERR_ARG, "tcb_fold_counters: null output");
    fold_counters(ops_deferred, flush_launches);
  });
}

int tcb_plan_num_kernels(tcb_plan plan) { return plan ? plan->p.nkernels : 0; }

const char* tcb_plan_key(tcb_plan plan) { return plan ? plan->p.key.c_str() : ""; }

const char* tcb_supported_ops(void) {
  static std::string s;
  static std::once_flag once;
  std::call_once(once, [] {
    for (auto& [k, v] : builders()) {
      if (!s.empty()) s += ' ';
      s += k;
    }
  });
  return s.c_str();
}

// ---- graphs -----------------------------------------------------------------
int tcb_graph_capture_begin(void* stream) {
  TCB_TRY(TCB_CUDA(
      cudaStreamBeginCapture(static_cast<cudaStream_t>(stream), cudaStreamCaptureModeThreadLocal)));
}
int tcb_graph_capture_end(void* stream, void** graph_exec) {
  TCB_TRY({
    cudaGraph_t g;
    TCB_CUDA(cudaStreamEndCapture(static_cast<cudaStream_t>(stream), &g));
    cudaGraphExec_t ge;
    TCB_CUDA(cudaGraphInstantiate(&ge, g, 0));
    TCB_CUDA(cudaGraphDestroy(g));
    *graph_exec = ge;
  });
}
int tcb_graph_launch(void* graph_exec, void* stream) {
  TCB_TRY(TCB_CUDA(cudaGraphLaunch(static_cast<cudaGraphExec_t>(graph_exec),
                                   static_cast<cudaStream_t>(stream))));
}
int tcb_graph_destroy(void* graph_exec) {
  TCB_TRY(TCB_CUDA(cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(graph_exec))));
}

// ---- helpers ----------------------------------------------------------------
int tcb_memcpy(void* dst, const void* src, uint64_t bytes, int kind, void* stream) {
  TCB_TRY({
    cudaMemcpyKind k = kind == 0   ? cudaMemcpyHostToDevice
                       : kind == 1 ? cudaMemcpyDeviceToHost
                                   : cudaMemcpyDeviceToDevice;
    TCB_CUDA(cudaMemcpyAsync(dst, src, bytes, k, static_cast<cudaStream_t>(stream)));
  });
}
int tcb_memset(void* dst, int value, uint64_t bytes, void* stream) {
  TCB_TRY(TCB_CUDA(cudaMemsetAsync(dst, value, bytes, static_cast<cudaStream_t>(stream))));
}
int tcb_stream_create(void** stream) {
  TCB_TRY({
    cudaStream_t s;
    TCB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    *stream = s;
  });
}
int tcb_stream_destroy(void* stream) {
  TCB_TRY(TCB_CUDA(cudaStreamDestroy(static_cast<cudaStream_t>(stream))));
}
int tcb_stream_sync(void* stream) {
  TCB_TRY(TCB_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream))));
}
int tcb_event_create(void** ev) {
  TCB_TRY({
    cudaEvent_t e;
    TCB_CUDA(cudaEventCreate(&e));
    *ev = e;
  });
}
int tcb_event_record(void* ev, void* stream) {
  TCB_TRY(TCB_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(ev), static_cast<cudaStream_t>(stream))));
}
int tcb_stream_wait_event(void* stream, void* ev) {
  TCB_TRY(TCB_CUDA(
      cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), static_cast<cudaEvent_t>(ev), 0)));
}
int tcb_event_elapsed_ms(void* start, void* stop, float* ms) {
  TCB_TRY(TCB_CUDA(
      cudaEventElapsedTime(ms, static_cast<cudaEvent_t>(start), static_cast<cudaEvent_t>(stop))));
}
int tcb_event_destroy(void* ev) { TCB_TRY(TCB_CUDA(cudaEventDestroy(static_cast<cudaEvent_t>(ev)))); }
int tcb_host_alloc(void** p, uint64_t bytes) { TCB_TRY(TCB_CUDA(cudaMallocHost(p, bytes))); }
int tcb_host_free(void* p) { TCB_TRY(TCB_CUDA(cudaFreeHost(p))); }
int tcb_device_sync(void) { TCB_TRY(TCB_CUDA(cudaDeviceSynchronize())); }

}  // extern "C"
