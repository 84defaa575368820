// comm.cu -- ZeRO collectives of the b200 backend.
//
// The reference runs collectives only through a simulated lockstep bus
// (world>1 throws in backends.hpp:246-250).  Here they are NCCL
// calls over NVLink 5 / NVSwitch.  libnccl is dlopen'ed (the process normally
// already holds torch's NCCL 2.28 under the soname libnccl.so.2), so the library
// has no link-time NCCL dependency.  A flat bucket = one contiguous arena segment
// (horizontal collective fusion): one ncclReduceScatter /
// ncclAllGather per bucket, issued inside ncclGroupStart/End.
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>

#include "common.cuh"

namespace tcb {

struct Nccl {
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommInitAll) commInitAll = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclCommCount) commCount = nullptr;
  decltype(&ncclReduceScatter) reduceScatter = nullptr;
  decltype(&ncclAllGather) allGather = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclGetErrorString) errStr = nullptr;
};

static Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
#define SYM(f, name) n.f = reinterpret_cast<decltype(n.f)>(dlsym(h, name))
    SYM(getUniqueId, "ncclGetUniqueId");
    SYM(commInitRank, "ncclCommInitRank");
    SYM(commInitAll, "ncclCommInitAll");
    SYM(commDestroy, "ncclCommDestroy");
    SYM(commCount, "ncclCommCount");
    SYM(reduceScatter, "ncclReduceScatter");
    SYM(allGather, "ncclAllGather");
    SYM(allReduce, "ncclAllReduce");
    SYM(groupStart, "ncclGroupStart");
    SYM(groupEnd, "ncclGroupEnd");
    SYM(errStr, "ncclGetErrorString");
#undef SYM
  });
  if (!n.commInitRank) fail(TCB_ERR_UNIMPLEMENTED, "libnccl.so.2 not loadable");
  return n;
}

#define TCB_NCCL(x)                                                                     \
  do {                                                                                  \
    ncclResult_t r_ = (x);                                                              \
    if (r_ != ncclSuccess) ::tcb::fail(TCB_ERR_CUDA, std::string(#x) + ": " + nccl().errStr(r_)); \
  } while (0)

static ncclDataType_t nccl_dtype(int d) {
  switch (d) {
    case TCB_F32: return ncclFloat32;
    case TCB_F16: return ncclFloat16;
    case TCB_BF16: return ncclBfloat16;
    case TCB_I32: return ncclInt32;
    case TCB_U8: return ncclUint8;
  }
  fail(TCB_ERR_TYPE, "collective: bad dtype");
}

static int64_t numel_of(const tcb_tensor& t) {
  int64_t n = 1;
  for (int i = 0; i < t.rank; ++i) n *= t.shape[i];
  return n;
}

}  // namespace tcb

using namespace tcb;

extern "C" {

int tcb_last_error_set(int code, const char* m);  // abi.cu (not exported in the header)

#define TCB_TRY_C(body)                                           \
  try {                                                           \
    body;                                                         \
    return TCB_OK;                                                \
  } catch (const tcb::Status& s) {                                \
    return tcb_last_error_set(s.code, s.what());                  \
  } catch (const std::exception& e) {                             \
    return tcb_last_error_set(TCB_ERR_ARG, e.what());             \
  }

int tcb_comm_unique_id(void* out128) {
  TCB_TRY_C({
    ncclUniqueId id;
    TCB_NCCL(nccl().getUniqueId(&id));
    std::memcpy(out128, &id, sizeof(id));
  });
}

int tcb_comm_init_rank(const void* unique_id128, int world, int rank, void** comm) {
  TCB_TRY_C({
    ncclUniqueId id;
    std::memcpy(&id, unique_id128, sizeof(id));
    ncclComm_t c;
    TCB_NCCL(nccl().commInitRank(&c, world, id, rank));
    *comm = c;
  });
}

int tcb_comm_init_all(int ndev, const int* devs, void** comms) {
  TCB_TRY_C({
    std::vector<ncclComm_t> c(ndev);
    TCB_NCCL(nccl().commInitAll(c.data(), ndev, devs));
    for (int i = 0; i < ndev; ++i) comms[i] = c[i];
  });
}

int tcb_comm_destroy(void* comm) {
  TCB_TRY_C({
    if (comm) TCB_NCCL(nccl().commDestroy(static_cast<ncclComm_t>(comm)));
  });
}

// NCCL moves one flat buffer per call: the segments of a bucket must be
// contiguous in memory and cover exactly world * shard elements (the zero pad
// materialised), or the call would read / write past them
static void check_bucket(const tcb_tensor* segs, int nseg, int64_t want, const char* what) {
  int64_t total = 0;
  const char* next = static_cast<const char*>(segs[0].ptr);
  for (int i = 0; i < nseg; ++i) {
    require(segs[i].dtype == segs[0].dtype, std::string(what) + ": segments of one bucket share a dtype");
    require(static_cast<const char*>(segs[i].ptr) == next, std::string(what) + ": bucket segments are not contiguous");
    const int64_t n = numel_of(segs[i]);
    next += n * dtype_bytes(segs[i].dtype);
    total += n;
  }
  require(total == want, std::string(what) + ": bucket has " + std::to_string(total) + " elements, world x shard = " +
                             std::to_string(want));
}

int tcb_reduce_scatter(void* comm, const tcb_tensor* segs, int nseg, tcb_tensor* shard, void* stream) {
  TCB_TRY_C({
    require(nseg >= 1, "reduce_scatter: no segments");
    const int64_t shard_n = numel_of(*shard);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (!comm) {  // world 1: identity up to flatten/pad (backends.hpp:253-256)
      int64_t off = 0;
      const int es = dtype_bytes(shard->dtype);
      for (int i = 0; i < nseg; ++i) {
        const int64_t n = numel_of(segs[i]);
        require(off + n <= shard_n, "reduce_scatter: segments exceed the shard (a world > 1 step without a "
                                    "communicator?)");
        TCB_CUDA(cudaMemcpyAsync(static_cast<char*>(shard->ptr) + off * es, segs[i].ptr, n * es,
                                 cudaMemcpyDeviceToDevice, s));
        off += n;
      }
      if (off < shard_n)
        TCB_CUDA(cudaMemsetAsync(static_cast<char*>(shard->ptr) + off * es, 0, (shard_n - off) * es, s));
      return TCB_OK;
    }
    ncclComm_t c = static_cast<ncclComm_t>(comm);
    int world = 0;
    TCB_NCCL(nccl().commCount(c, &world));
    check_bucket(segs, nseg, shard_n * world, "reduce_scatter");
    TCB_NCCL(nccl().groupStart());
    TCB_NCCL(nccl().reduceScatter(segs[0].ptr, shard->ptr, size_t(shard_n), nccl_dtype(shard->dtype), ncclSum,
                                  c, s));
    TCB_NCCL(nccl().groupEnd());
  });
}

int tcb_all_gather(void* comm, const tcb_tensor* shard, tcb_tensor* segs, int nseg, void* stream) {
  TCB_TRY_C({
    require(nseg >= 1, "all_gather: no segments");
    const int64_t shard_n = numel_of(*shard);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (!comm) {  // world 1: gather truncates the pad (backends.hpp:257-261)
      int64_t off = 0;
      const int es = dtype_bytes(shard->dtype);
      for (int i = 0; i < nseg; ++i) {
        const int64_t n = numel_of(segs[i]);
        require(off + n <= shard_n, "all_gather: segments exceed the shard (a world > 1 step without a "
                                    "communicator?)");
        TCB_CUDA(cudaMemcpyAsync(segs[i].ptr, static_cast<const char*>(shard->ptr) + off * es, n * es,
                                 cudaMemcpyDeviceToDevice, s));
        off += n;
      }
      return TCB_OK;
    }
    ncclComm_t c = static_cast<ncclComm_t>(comm);
    int world = 0;
    TCB_NCCL(nccl().commCount(c, &world));
    check_bucket(segs, nseg, shard_n * world, "all_gather");
    TCB_NCCL(nccl().groupStart());
    TCB_NCCL(nccl().allGather(shard->ptr, segs[0].ptr, size_t(shard_n), nccl_dtype(shard->dtype), c, s));
    TCB_NCCL(nccl().groupEnd());
  });
}

int tcb_all_reduce(void* comm, tcb_tensor* buf, void* stream) {
  TCB_TRY_C({
    if (!comm) return TCB_OK;
    TCB_NCCL(nccl().allReduce(buf->ptr, buf->ptr, size_t(numel_of(*buf)), nccl_dtype(buf->dtype), ncclSum,
                              static_cast<ncclComm_t>(comm), static_cast<cudaStream_t>(stream)));
  });
}

}  // extern "C"
