// extern "C" implementation of include/bitmm_b200.h: argument validation in the
// reference's order, workspace management, TMA descriptor encoding and the
// launch sequence (unpack -> tcgen05 GEMM with fused epilogue) per routine.
#include <cuda.h>
#include <dlfcn.h>
#include <nccl.h>
#include <cuda_runtime.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <condition_variable>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <thread>
#include <tuple>
#include <string>
#include <vector>

#include "apb_gemm.cuh"
#include "apb2_fused.cuh"
#include "spmm_levels.cuh"
#include "btsr_io.cuh"
#include "bitmm_b200.h"
#include "fx_gemm.cuh"
#include "prep.cuh"
#include "pack.cuh"
#include "popc_gemm.cuh"
#include "ptx.cuh"
#include "tc_gemm.cuh"
#include "unpack.cuh"
#include "wire.cuh"

using namespace bitmm_dev;

namespace {

thread_local std::string g_err;
thread_local int g_launches = 0;
thread_local uint64_t g_d2h_bytes = 0;  // device -> host bytes of the last host-flavour call

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define BITMM_CUDA_TRY(expr)                                                              \
  do {                                                                                    \
    cudaError_t e_ = (expr);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(BITMM_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));    \
  } while (0)

#define BITMM_TRY(expr)         \
  do {                          \
    int rc_ = (expr);           \
    if (rc_ != BITMM_OK) return rc_; \
  } while (0)

constexpr int kMaxDevices = 16;
constexpr int kMaxWireSlices = 32;  // input-flag slots of one host pipeline (8 slices x 4 items)

struct Arena {
  void* ptr = nullptr;
  size_t bytes = 0;
};

// ---------------- call contexts (re-entrancy) ----------------
// The reference's entry points allocate per call and share nothing (kernels.cpp:163-275), so
// callers drive them from many threads (run_row_blocks, kernels.cpp:50-68). Here:
//  * device calls (`*_dev`) use the context of their CUDA stream (Ctx): workspace, latched
//    status flag and scratch, grown stream-ordered (cudaMallocAsync / cudaFreeAsync), and a
//    mutex held while the call enqueues its launches, so calls on one stream never interleave
//    and calls on different streams never share memory;
//  * host calls (`*_host`) lease a HostCtx for the whole call: private streams, staging,
//    pinned buffers and events, so concurrent host calls from different threads run side by
//    side. A lease ends with its streams drained, so no copy still reads the caller's buffers
//    after the call returns, whatever the exit path.
struct SchedBuf {
  void* dev;      // the pieces (int4), then the per-unit offsets (int)
  size_t pbytes;  // bytes of the pieces
};

struct Ctx {
  int dev = 0;
  int sms = 0;
  cudaStream_t stream = nullptr;
  std::recursive_mutex mu;  // a host call holds it while its inner device calls take it again
  int* status = nullptr;   // latched device-side flags of this stream's calls
  int* scratch = nullptr;  // 64 bytes (plane validation)
  Arena ws;                // expanded operands, APB intermediates, scan temp
  Arena codes;             // 2-bit level codes of the in-GEMM expansion path (fx_gemm)
  unsigned ws_turn = 0;    // ping-pong half of the expanded-operand workspace
  // balanced GEMM schedules (TcGroup::sched) by group shape, in device memory, kept
  std::map<std::vector<long long>, SchedBuf> sched_cache;
};

struct HostCtx {
  Ctx* sctx = nullptr;                    // the stream context of `stream`
  cudaStream_t stream = nullptr;          // the call's GEMM stream
  cudaStream_t d2h = nullptr;             // output copies (run_pipelined)
  cudaStream_t h2d = nullptr;             // input copies (run_wire_items)
  Arena io;                               // device staging of inputs / outputs
  Arena w12;                              // 12-bit packed wire parts (wire.cuh)
  cudaEvent_t pipe_ev[8] = {};
  cudaEvent_t in_ev[kMaxWireSlices + 1] = {};
  uint32_t* in_flags = nullptr;           // per-slice "inputs landed" flags
  uint32_t in_epoch = 0;
  void* host_stage = nullptr;             // pinned 16-bit output words (run_wire_items)
  size_t host_stage_bytes = 0;
  std::vector<cudaEvent_t> wire_ev;       // one per copied part
  std::vector<cudaEvent_t> stage_ev;      // run_staged parts (spin-waited: latency, not CPU)
  int* status_host = nullptr;             // pinned copy of the stream's status word (run_staged)
  void* pinned[2] = {nullptr, nullptr};   // BTSR streaming chunks (allocated on first load)
  cudaEvent_t pinned_ev[2] = {nullptr, nullptr};
  // BITMM_WIRE_TRACE only: device timeline of the current host call
  std::vector<std::pair<std::string, cudaEvent_t>>* timeline = nullptr;
};

struct Dev {
  std::mutex mu;
  bool init = false;
  int sms = 0;
  std::map<unsigned long long, std::unique_ptr<Ctx>> streams;  // by cudaStreamGetId (never reused)
  std::vector<std::unique_ptr<HostCtx>> hosts;
  std::vector<HostCtx*> idle_hosts;
};
Dev g_dev[kMaxDevices];

void trace_mark(HostCtx& st, const std::string& what, cudaStream_t on) {
  if (!st.timeline) return;
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  cudaEventRecord(e, on);
  // host enqueue time (us since the first mark) goes into the label
  static thread_local std::chrono::steady_clock::time_point t0;
  const auto now = std::chrono::steady_clock::now();
  if (st.timeline->empty()) t0 = now;
  const long us = static_cast<long>(std::chrono::duration_cast<std::chrono::microseconds>(now - t0).count());
  st.timeline->emplace_back(what + "@" + std::to_string(us), e);
}

// The current device's record (initialised once: SM count, a memory pool that keeps what
// it has reserved, so stream-ordered workspace growth does not return memory to the OS).
int current_dev(Dev** out, int* dev_out) {
  int dev = 0;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    return fail(BITMM_ERR_NO_DEVICE, "no CUDA device available (bitmm_b200 has no CPU fallback)");
  }
  BITMM_CUDA_TRY(cudaGetDevice(&dev));
  if (dev >= kMaxDevices) return fail(BITMM_ERR_CUDA, "device index out of range");
  Dev& d = g_dev[dev];
  std::lock_guard<std::mutex> lk(d.mu);
  if (!d.init) {
    BITMM_CUDA_TRY(cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev));
    cudaMemPool_t pool;
    BITMM_CUDA_TRY(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t keep = UINT64_MAX;
    BITMM_CUDA_TRY(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    d.init = true;
  }
  *out = &d;
  *dev_out = dev;
  return BITMM_OK;
}

// The context of stream `s` on the current device (created on first use).
int stream_ctx(cudaStream_t s, Ctx** out) {
  Dev* d = nullptr;
  int dev = 0;
  BITMM_TRY(current_dev(&d, &dev));
  unsigned long long id = 0;
  BITMM_CUDA_TRY(cudaStreamGetId(s, &id));
  std::lock_guard<std::mutex> lk(d->mu);
  auto it = d->streams.find(id);
  if (it == d->streams.end()) {
    auto c = std::make_unique<Ctx>();
    c->dev = dev;
    c->sms = d->sms;
    c->stream = s;
    BITMM_CUDA_TRY(cudaMalloc(&c->status, 128));
    BITMM_CUDA_TRY(cudaMemset(c->status, 0, 128));
    c->scratch = c->status + 16;
    it = d->streams.emplace(id, std::move(c)).first;
  }
  *out = it->second.get();
  return BITMM_OK;
}

// A device call's context: the stream's Ctx, locked for the call.
class CallCtx {
 public:
  int acquire(cudaStream_t s) {
    BITMM_TRY(stream_ctx(s, &c_));
    lk_ = std::unique_lock<std::recursive_mutex>(c_->mu);
    return BITMM_OK;
  }
  Ctx& operator*() { return *c_; }
  Ctx* operator->() { return c_; }

 private:
  Ctx* c_ = nullptr;
  std::unique_lock<std::recursive_mutex> lk_;
};

int host_ctx_init(HostCtx& h) {
  BITMM_CUDA_TRY(cudaStreamCreateWithFlags(&h.stream, cudaStreamNonBlocking));
  BITMM_CUDA_TRY(cudaStreamCreateWithFlags(&h.d2h, cudaStreamNonBlocking));
  BITMM_CUDA_TRY(cudaStreamCreateWithFlags(&h.h2d, cudaStreamNonBlocking));
  for (auto& e : h.pipe_ev) BITMM_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (auto& e : h.in_ev) BITMM_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  BITMM_CUDA_TRY(cudaMalloc(&h.in_flags, kMaxWireSlices * sizeof(uint32_t)));
  BITMM_CUDA_TRY(cudaMemset(h.in_flags, 0, kMaxWireSlices * sizeof(uint32_t)));
  BITMM_CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&h.status_host), 64, cudaHostAllocDefault));
  return stream_ctx(h.stream, &h.sctx);
}

// A host call's lease of a HostCtx (and its stream's Ctx). Released with every stream of the
// context drained, on every exit path.
struct WireItem;
// A host batch being assembled (bitmm_gemm_batch_host): the routines' host calls run in two
// passes on the batch's lease, first adding up the device staging they need, then carving it
// and handing their wire pipelines over instead of running them.
struct HostBatch {
  HostCtx* host = nullptr;
  bool sizing = true;  // pass 1: only add up the device staging
  size_t need = 0;     // pass 1: bytes needed; pass 2: the next free byte of the io arena
  std::vector<WireItem>* items = nullptr;
};
thread_local HostBatch* g_batch = nullptr;
constexpr int kBatchSized = 1000;  // internal return code of a sizing pass

class HostLease {
 public:
  int acquire() {
    if (g_batch) {  // a batch item runs on the batch's lease
      h_ = g_batch->host;
      borrowed_ = true;
      return BITMM_OK;
    }
    int dev = 0;
    BITMM_TRY(current_dev(&d_, &dev));
    {
      std::lock_guard<std::mutex> lk(d_->mu);
      if (!d_->idle_hosts.empty()) {
        h_ = d_->idle_hosts.back();
        d_->idle_hosts.pop_back();
      }
    }
    if (!h_) {
      auto h = std::make_unique<HostCtx>();
      const int rc = host_ctx_init(*h);
      if (rc != BITMM_OK) return rc;  // partially created resources leak (failure path only)
      h_ = h.get();
      std::lock_guard<std::mutex> lk(d_->mu);
      d_->hosts.push_back(std::move(h));
    }
    lk_ = std::unique_lock<std::recursive_mutex>(h_->sctx->mu);
    return BITMM_OK;
  }
  ~HostLease() {
    if (!h_ || borrowed_) return;
    cudaStreamSynchronize(h_->h2d);
    cudaStreamSynchronize(h_->stream);
    cudaStreamSynchronize(h_->d2h);
    if (lk_.owns_lock()) lk_.unlock();
    std::lock_guard<std::mutex> lk(d_->mu);
    d_->idle_hosts.push_back(h_);
  }
  HostCtx* operator->() { return h_; }
  HostCtx& host() { return *h_; }
  Ctx& ctx() { return *h_->sctx; }

 private:
  Dev* d_ = nullptr;
  HostCtx* h_ = nullptr;
  bool borrowed_ = false;
  std::unique_lock<std::recursive_mutex> lk_;
};

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel, device and size (the
// attribute is per device; a process may drive several).
int ensure_max_smem(const void* fn, int bytes) {
  int dev = 0;
  BITMM_CUDA_TRY(cudaGetDevice(&dev));
  static std::mutex mu;
  static std::set<std::tuple<const void*, int, int>> done;
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_tuple(fn, dev, bytes);
  if (done.count(key)) return BITMM_OK;
  BITMM_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done.insert(key);
  return BITMM_OK;
}

// Grows an arena in stream order on `s` (the only stream that uses it, or the stream whose
// earlier work every other user waits for): the old buffer is freed behind the work already
// queued there, so a call never synchronises the device or frees memory still in use.
int arena_reserve(Arena& a, size_t bytes, cudaStream_t s) {
  if (bytes <= a.bytes) return BITMM_OK;
  if (a.ptr) {
    BITMM_CUDA_TRY(cudaFreeAsync(a.ptr, s));
    a.ptr = nullptr;
    a.bytes = 0;
  }
  size_t grown = std::max(bytes, static_cast<size_t>(1) << 20);
  BITMM_CUDA_TRY(cudaMallocAsync(&a.ptr, grown, s));
  a.bytes = grown;
  return BITMM_OK;
}
int arena_reserve(Arena& a, cudaStream_t s, size_t bytes) { return arena_reserve(a, bytes, s); }
// Context-stream shorthand.
int ws_reserve(Ctx& st, size_t bytes) { return arena_reserve(st.ws, bytes, st.stream); }

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// A host call's device staging: the lease's io arena, or its share of a batch's.
int io_take(HostCtx& h, cudaStream_t s, size_t bytes, void** out) {
  if (g_batch) {
    if (g_batch->sizing) {
      g_batch->need += align_up(bytes, 1024);
      return kBatchSized;
    }
    *out = static_cast<uint8_t*>(h.io.ptr) + g_batch->need;
    g_batch->need += align_up(bytes, 1024);
    return BITMM_OK;
  }
  BITMM_TRY(arena_reserve(h.io, s, bytes));
  *out = h.io.ptr;
  return BITMM_OK;
}
int64_t round_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

// Sequential 1024-byte aligned sub-buffers of one allocation.
struct Carve {
  uint8_t* base;
  size_t off = 0;
  explicit Carve(void* b) : base(static_cast<uint8_t*>(b)) {}
  template <typename T>
  T* take(size_t bytes) {
    T* p = reinterpret_cast<T*>(base + off);
    off = align_up(off + bytes, 1024);
    return p;
  }
};


// ---------------- TMA descriptors (driver entry point, no -lcuda) ----------------
typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                      const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                      const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                      CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled_t encode_fn() {
  static PFN_encodeTiled_t fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled_t>(p);
  });
  return fn;
}

// cuMemGetAddressRange (base and size of the allocation holding a pointer; CUDA IPC handles
// name whole allocations).
typedef CUresult (*PFN_addrRange_t)(CUdeviceptr*, size_t*, CUdeviceptr);
PFN_addrRange_t addr_range_fn() {
  static PFN_addrRange_t fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_addrRange_t>(p);
  });
  return fn;
}

// True when `p` is device memory of another GPU (a peer allocation opened through CUDA IPC):
// the GEMM epilogue then stores with st.global over NVLink instead of TMA.
bool is_peer_memory(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  return a.type == cudaMemoryTypeDevice && a.device != dev;
}

// cuStreamWriteValue32 (a 32-bit write that executes in stream order on the copy stream).
typedef CUresult (*PFN_writeValue32_t)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
PFN_writeValue32_t write_value_fn() {
  static PFN_writeValue32_t fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_writeValue32_t>(p);
  });
  return fn;
}

// cuStreamWaitValue32: the GEMM stream waits in its front end (no SM, no timeout) until the
// copy stream's cuStreamWriteValue32 has landed.
typedef CUresult (*PFN_waitValue32_t)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
PFN_waitValue32_t wait_value_fn() {
  static PFN_waitValue32_t fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_waitValue32_t>(p);
  });
  return fn;
}

// How a host call's slice GEMM waits for that slice's input copies (run_wire_items):
//   Value  : cuStreamWaitValue32 on the flag the copy stream writes (default)
//   Kernel : a one-warp spin kernel on that flag (BITMM_WIRE_WAIT=kernel)
//   Event  : cudaStreamWaitEvent on the copy stream (BITMM_WIRE_WAIT=event, or no driver
//            entry points); it resolved only once the copy stream had drained
enum class SliceWait { Value, Kernel, Event };
SliceWait slice_wait_mode() {
  const char* e = std::getenv("BITMM_WIRE_WAIT");  // read per call (tests switch it)
  const std::string v = e ? e : "";
  if (v == "event" || !write_value_fn()) return SliceWait::Event;
  if (v == "kernel" || !wait_value_fn()) return SliceWait::Kernel;
  return SliceWait::Value;
}
// Test hook: BITMM_WIRE_FAULT=flagwrite treats every flag write as failed, so each slice takes
// the event fallback (the path a driver without stream memory operations takes).
bool fault_flag_write() {
  const char* e = std::getenv("BITMM_WIRE_FAULT");
  return e && std::string(e) == "flagwrite";
}

// Waits in a one-warp kernel until *flag == value: the copy stream writes the flag after a
// slice's input copies (run_wire_items). A spin on the SMs, not an event wait: the
// GEMM stream's event waits on the copy stream resolved only once that stream had drained.
// Gives up after ~2 s and latches ERR_COPY_TIMEOUT (never hangs the device).
constexpr int ERR_COPY_TIMEOUT = 16;
__global__ void wait_flag_kernel(const volatile uint32_t* flag, uint32_t value, int* err) {
  if (threadIdx.x != 0) return;
  const long long t0 = clock64();
  while (*flag != value) {
    if (clock64() - t0 > 4000000000ll) {
      atomicOr(err, ERR_COPY_TIMEOUT);
      break;
    }
    __nanosleep(200);
  }
  __threadfence();
}

// K-major operand [rows][inner] with 128-byte rows per box, 128B swizzle.
int make_operand_map(CUtensorMap* map, const void* base, CUtensorMapDataType dt, int elem_bytes,
                     uint64_t inner_elems, uint64_t rows, uint32_t box_rows) {
  PFN_encodeTiled_t enc = encode_fn();
  if (!enc) return fail(BITMM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {inner_elems, rows};
  cuuint64_t strides[1] = {inner_elems * static_cast<uint64_t>(elem_bytes)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(TC_BK_BYTES / elem_bytes), box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(BITMM_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
  return BITMM_OK;
}

// Output map for the GEMM epilogue's bulk tensor stores: [rows][ldc] 4-byte cells, box 32x32,
// 128B swizzle (the epilogue's staging layout). Returns false when the layout does not allow
// TMA (row pitch not a multiple of 16 bytes or base not 16-byte aligned).
// The box is clipped at the tensor's bounds only to 16-byte granularity along the rows: with
// cols not a multiple of 4 the last chunk of a row would also write up to 3 cells past cols
// (measured: tests/test_bounds_gpu.py, a caller's ldc > cols), so such outputs take the
// epilogue's st.global path.
bool make_output_map(CUtensorMap* map, void* base, CUtensorMapDataType dt, uint64_t cols,
                     uint64_t rows, uint64_t ldc) {
  if (base == nullptr || (ldc & 3) != 0 || (cols & 3) != 0 || (reinterpret_cast<uintptr_t>(base) & 15) != 0)
    return false;
  PFN_encodeTiled_t enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ldc * 4};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  return enc(map, dt, 2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// ---------------- stream-ordered kernel profiler ----------------
struct ProfRecord {
  int kernel;
  cudaEvent_t e0, e1;
};

struct Profiler {
  std::mutex mu;
  bool on = false;
  std::vector<cudaEvent_t> pool;
  std::vector<ProfRecord> pending;
  std::vector<std::string> names;
  std::vector<int> launches;
  std::vector<double> ms;

  int id(const char* name) {
    for (size_t i = 0; i < names.size(); ++i)
      if (names[i] == name) return static_cast<int>(i);
    names.emplace_back(name);
    launches.push_back(0);
    ms.push_back(0.0);
    return static_cast<int>(names.size() - 1);
  }
  cudaEvent_t take() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
  }
};

Profiler g_prof;

// Brackets one kernel launch with events on its stream when profiling is enabled.
class ProfScope {
 public:
  ProfScope(const char* name, cudaStream_t s) : name_(name), s_(s) {
    if (!g_prof.on) return;
    std::lock_guard<std::mutex> lk(g_prof.mu);
    e0_ = g_prof.take();
    e1_ = g_prof.take();
    cudaEventRecord(e0_, s_);
  }
  ~ProfScope() {
    if (!e0_) return;
    cudaEventRecord(e1_, s_);
    std::lock_guard<std::mutex> lk(g_prof.mu);
    g_prof.pending.push_back({g_prof.id(name_), e0_, e1_});
  }

 private:
  const char* name_;
  cudaStream_t s_;
  cudaEvent_t e0_ = nullptr, e1_ = nullptr;
};

// ---------------- launches ----------------
int launch_check(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(BITMM_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  ++g_launches;
  return BITMM_OK;
}

unsigned blocks_for(long long total, int threads) {
  return static_cast<unsigned>((total + threads - 1) / threads);
}

int run_unpack_level_i8(const uint64_t* t, const uint64_t* h, const uint64_t* m, int64_t rows,
                        int64_t wpr, int64_t k, int64_t kpad, uint8_t* out, int* flag,
                        cudaStream_t s) {
  const int wpr32 = static_cast<int>(wpr * 2);
  const long long total = rows * std::max<long long>(kpad / 32, wpr32);
  if (total == 0) return BITMM_OK;
  ProfScope ps("unpack_level_i8", s);
  unpack_level_i8<<<blocks_for(total, 256), 256, 0, s>>>(
      reinterpret_cast<const uint32_t*>(t), reinterpret_cast<const uint32_t*>(h),
      reinterpret_cast<const uint32_t*>(m), rows, wpr32, static_cast<int>(k),
      static_cast<int>(kpad), out, flag);
  return launch_check("unpack_level_i8");
}

// Operand description for the fused pair-unpack launch.
struct OperandSrc {
  const uint64_t* w0;
  const uint64_t* w1;
  const uint64_t* w2;
  int64_t rows;
  bool levels;
};

UnpackOperand make_unpack_operand(const OperandSrc& src, int64_t wpr, int64_t k, int64_t kpad,
                                  uint8_t* out) {
  UnpackOperand o{};
  o.w0 = reinterpret_cast<const uint32_t*>(src.w0);
  o.w1 = reinterpret_cast<const uint32_t*>(src.w1);
  o.w2 = reinterpret_cast<const uint32_t*>(src.w2);
  o.out = out;
  o.rows = src.rows;
  o.wpr32 = static_cast<int>(wpr * 2);
  o.groups_per_row = (std::max<long long>(kpad / 32, o.wpr32) + 127) / 128;  // 128-word slices
  o.levels = src.levels ? 1 : 0;
  o.K = static_cast<int>(k);
  o.kpad = static_cast<int>(kpad);
  return o;
}

// The flat bulk-copy expansion (unpack.cuh, unpack_flat_kernel; BITMM_UNPACK_FLAT=1) takes a
// set of e2m1 operands whose rows hold no padding (K = 32 * wpr32 = kpad) and 16-byte aligned
// planes and outputs. Measured, not the default: bench step expansion 18.5 vs 17.3 us, 1/1
// 4096^3 per call 34.1 vs 33.5 us (profiles/dev/unpack_flat_ab.sh): with no per-thread global
// accesses it is no faster, so the per-slice kernel is not paced by its loads' latency or the
// load/store queue but by the writes of the expanded bytes into an L2 full of the previous
// GEMM's dirty output.
bool unpack_flat_ok(const UnpackSet& P) {
  const char* e = std::getenv("BITMM_UNPACK_FLAT");
  if (!(e && std::atoi(e) == 1) || !P.fp4 || P.lc.chunks > 0) return false;
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  for (int i = 0; i < P.count; ++i) {
    const UnpackOperand& o = P.op[i];
    if (o.K != o.wpr32 * 32 || o.kpad != o.K || !al(o.w0) || !al(o.out) ||
        (o.levels && (!al(o.w1) || !al(o.w2))))
      return false;
  }
  return true;
}

int run_unpack_flat(const UnpackSet& P, int sms, cudaStream_t s) {
  UnpackFlat F{};
  F.count = P.count;
  F.err = P.err;
  long long chunks = 0;
  for (int i = 0; i < P.count; ++i) {
    F.op[i] = P.op[i];
    F.chunk_begin[i] = chunks;
    chunks += (P.op[i].rows * P.op[i].wpr32 + UF_CHUNK - 1) / UF_CHUNK;
  }
  for (int i = P.count; i <= UNPACK_MAX_OPS; ++i) F.chunk_begin[i] = chunks;
  if (chunks == 0) return BITMM_OK;
  BITMM_TRY(ensure_max_smem(reinterpret_cast<const void*>(unpack_flat_kernel), UF_SMEM));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(std::min<long long>(chunks, 2ll * sms)));
  cfg.blockDim = dim3(UF_THREADS);
  cfg.dynamicSmemBytes = UF_SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  ProfScope ps("unpack_operands", s);
  BITMM_CUDA_TRY(cudaLaunchKernelEx(&cfg, unpack_flat_kernel, F));
  return launch_check("unpack_flat_kernel");
}

// Expands every operand of a set (bits or ternary planes) in one launch.
int run_unpack_set(UnpackSet& P, cudaStream_t s) {
  if (unpack_flat_ok(P)) {
    Dev* d = nullptr;
    int dev = 0;
    BITMM_TRY(current_dev(&d, &dev));
    return run_unpack_flat(P, d->sms, s);
  }
  long long work = 0;  // threads per grid row: a warp per slice, or a thread per level-chunk item
  for (int i = 0; i < P.count; ++i) work = std::max(work, P.op[i].rows * P.op[i].groups_per_row * 32);
  const long long lc_items = P.lc.chunks > 0
                                 ? static_cast<long long>(((P.lc.K + 63) / 64) * 2 * SL_ROW_WORDS +
                                                          (P.lc.l8 ? L8_ROW_WORDS : SL_ROW_WORDS)) *
                                       P.lc.chunks
                                 : 0;
  work = std::max(work, lc_items);
  if (work == 0) return BITMM_OK;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks_for(work, 256), static_cast<unsigned>(P.count + (lc_items > 0 ? 1 : 0)));
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  ProfScope ps("unpack_operands", s);
  BITMM_CUDA_TRY(cudaLaunchKernelEx(&cfg, unpack_operands, P));
  return launch_check("unpack_operands");
}

// Expands both GEMM operands in one launch.
int run_unpack_pair(const OperandSrc& a, const OperandSrc& b, int64_t wpr, int64_t k, int64_t kpad,
                    uint8_t* A8, uint8_t* B8, int* flag, cudaStream_t s, bool fp4 = false,
                    const LevelChunkJob* lc = nullptr) {
  UnpackSet P{};
  if (lc) P.lc = *lc;
  P.fp4 = fp4 ? 1 : 0;
  P.op[0] = make_unpack_operand(a, wpr, k, kpad, A8);
  P.op[1] = make_unpack_operand(b, wpr, k, kpad, B8);
  P.count = 2;
  P.err = flag;
  return run_unpack_set(P, s);
}

// Operand kind of the bitwise GEMMs: packed e2m1 through kind::mxf4 (default; 2x the int8
// tensor rate, half the expanded bytes) or int8 through kind::i8 (BITMM_TC_KIND=i8, kept for
// A/B measurement). Both are exact: see tc_gemm.cuh.
bool use_fp4() {
  static const bool on = !(getenv("BITMM_TC_KIND") && strcmp(getenv("BITMM_TC_KIND"), "i8") == 0);
  return on;
}
constexpr int kF4BN = 192;  // 2 x 192 accumulator columns + scale-factor columns <= 512
constexpr int kI8BN = 256;  // 256-wide int8 tiles (128-wide measured worse: DESIGN.md)
int64_t kpad_for(int64_t k, bool fp4) { return round_up(k, fp4 ? 2 * TC_BK_BYTES : TC_BK_BYTES); }
// Units = acc << shift. The e2m1 expansion stores a 2-bit level p as p / 2 (unpack.cuh), so
// each level operand of an FP4 GEMM adds one to the reference shift (exact: powers of two).
int fp4_shift(int shift, int level_operands, bool fp4) { return shift + (fp4 ? level_operands : 0); }
int64_t row_bytes(int64_t kpad, bool fp4) { return fp4 ? kpad / 2 : kpad; }

// One GEMM problem over expanded operands A8 [m][row_bytes], B8 [n][row_bytes]; `p` carries
// the epilogue (shift, scales, output, ldc, epi).
struct GemmProblem {
  const uint8_t* A8;
  const uint8_t* B8;
  int64_t m, n, kpad;
  TcParams p;
};

// Balanced schedule of a group (TcGroup::sched, BITMM_TC_BALANCE=1; measured, not the default):
// the output column-work in 32-column units, problem by problem and 256-row block by block, cut
// into `units` contiguous stretches of equal length, each cut into pieces of at most BN columns
// that stay inside one row block. At 4096^2 (BN 192) every CTA pair then multiplies 896 columns
// instead of five 192-column tiles (960), but the pairs no longer work on neighbouring tiles at
// the same time: 1/1 4096^3 39.9 vs 37.9 us, the bench step 2026 vs 2254 T-upd/s, config 5
// 23.6 vs 10.0 ms (operand reuse in L2 lost; profiles/dev/balance_ab.sh). Round-robin tiles in
// the L2-grouped raster stay the default.
bool tc_balance() {
  const char* e = std::getenv("BITMM_TC_BALANCE");
  return e && std::atoi(e) == 1;
}

int tc_schedule(Ctx& st, const TcParams* prob, int count, int units, int bn, cudaStream_t s, const int4** sched,
                const int** unit_begin, void** free_after) {
  *free_after = nullptr;
  std::vector<long long> key{units, bn, count};
  for (int i = 0; i < count; ++i) {
    key.push_back(prob[i].M);
    key.push_back(prob[i].N);
  }
  auto it = st.sched_cache.find(key);
  if (it == st.sched_cache.end()) {
    long long total = 0;
    for (int i = 0; i < count; ++i) total += static_cast<long long>(prob[i].num_m_blocks) * ((prob[i].N + 31) / 32);
    const long long cap = (total + units - 1) / units;
    std::vector<int4> pieces;
    std::vector<int> begin{0};
    long long used = 0;
    for (int i = 0; i < count; ++i)
      for (int mb = 0; mb < prob[i].num_m_blocks; ++mb) {
        const int cols32 = (prob[i].N + 31) / 32;
        for (int c = 0; c < cols32;) {
          if (used == cap) {
            begin.push_back(static_cast<int>(pieces.size()));
            used = 0;
          }
          const int w = static_cast<int>(std::min<long long>({bn / 32, cols32 - c, cap - used}));
          pieces.push_back(make_int4(i | ((w * 32) << 16), mb, c * 32, 0));
          c += w;
          used += w;
        }
      }
    while (static_cast<int>(begin.size()) <= units) begin.push_back(static_cast<int>(pieces.size()));
    const size_t pbytes = pieces.size() * sizeof(int4);
    std::vector<uint8_t> host(pbytes + begin.size() * sizeof(int));
    std::memcpy(host.data(), pieces.data(), pbytes);
    std::memcpy(host.data() + pbytes, begin.data(), begin.size() * sizeof(int));
    SchedBuf b{nullptr, pbytes};
    BITMM_CUDA_TRY(cudaMallocAsync(&b.dev, host.size(), s));
    BITMM_CUDA_TRY(cudaMemcpyAsync(b.dev, host.data(), host.size(), cudaMemcpyHostToDevice, s));
    if (st.sched_cache.size() >= 256) {  // shape churn: used once, freed behind the launch
      *sched = static_cast<const int4*>(b.dev);
      *unit_begin = reinterpret_cast<const int*>(static_cast<uint8_t*>(b.dev) + pbytes);
      *free_after = b.dev;
      return BITMM_OK;
    }
    it = st.sched_cache.emplace(key, b).first;
  }
  *sched = static_cast<const int4*>(it->second.dev);
  *unit_begin = reinterpret_cast<const int*>(static_cast<const uint8_t*>(it->second.dev) + it->second.pbytes);
  return BITMM_OK;
}

// Launch one persistent cta_group::2 GEMM over a group of problems (tiles concatenated).
template <Kind KIND, Epi EPI, int BN, int NP>
int run_tc_group(Ctx& st, const GemmProblem* probs, int count, cudaStream_t s) {
  using S = TcShape<true, BN>;
  auto kern = tc_gemm_kernel<KIND, EPI, BN, NP>;
  BITMM_TRY(ensure_max_smem(reinterpret_cast<const void*>(kern), S::SMEM));
  constexpr bool fp4 = KIND == Kind::F4;
  TcGroup<NP> g;
  memset(&g, 0, sizeof(g));
  int tiles = 0;
  for (int i = 0; i < count; ++i) {
    const GemmProblem& q = probs[i];
    const int64_t rb = row_bytes(q.kpad, fp4);
    BITMM_TRY(make_operand_map(&g.a[i], q.A8, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, rb, q.m, S::A_ROWS));
    BITMM_TRY(make_operand_map(&g.b[i], q.B8, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, rb, q.n, S::B_ROWS));
    TcParams p = q.p;
    p.M = static_cast<int>(q.m);
    p.N = static_cast<int>(q.n);
    p.num_kb = static_cast<int>(rb / TC_BK_BYTES);
    // |units| <= 36K (2/2: 4 * 9 per element), so 36 * kpad < 2^22 allows the magic-add
    // float -> int conversion
    p.small_acc = 36 * q.kpad < (int64_t{1} << 22) ? 1 : 0;
    p.shift_mul = static_cast<float>(1 << p.shift);
    p.num_m_blocks = static_cast<int>((q.m + S::TILE_M - 1) / S::TILE_M);
    p.num_n_blocks = static_cast<int>((q.n + BN - 1) / BN);
    p.num_tiles = p.num_m_blocks * p.num_n_blocks;
    p.group_m = TC_GROUP_M;
    const bool i32 = p.epi == static_cast<int>(Epi::I32);
    void* out = i32 ? static_cast<void*>(p.out_i32) : static_cast<void*>(p.out_f32);
    p.tma_store = !is_peer_memory(out) && make_output_map(&g.c[i], out, i32 ? CU_TENSOR_MAP_DATA_TYPE_INT32
                                                                            : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                                                          p.N, p.M, p.ldc) ? 1 : 0;
    g.prob[i] = p;
    g.tile_begin[i] = tiles;
    tiles += p.num_tiles;
  }
  g.count = count;
  for (int i = count; i <= NP; ++i) g.tile_begin[i] = tiles;
  const int units = std::min(tiles, st.sms / 2);
  void* sched_free = nullptr;
  if (tc_balance()) BITMM_TRY(tc_schedule(st, g.prob, count, units, BN, s, &g.sched, &g.unit_begin, &sched_free));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(2 * units));
  cfg.blockDim = dim3(TC_THREADS);
  cfg.dynamicSmemBytes = S::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  ProfScope ps(KIND == Kind::I8 ? "tc_gemm_i8" : "tc_gemm_f4", s);
  BITMM_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, g));
  BITMM_TRY(launch_check("tc_gemm_kernel"));
  if (sched_free) BITMM_CUDA_TRY(cudaFreeAsync(sched_free, s));
  return BITMM_OK;
}

// Dispatch a group on the operand kind: one problem with a fixed epilogue, or up to
// TC_GROUP_MAX problems with per-problem epilogues.
int run_problems(Ctx& st, const GemmProblem* probs, int count, bool fp4, cudaStream_t s) {
  if (count == 1) {
    const int e = probs[0].p.epi;
    if (fp4) {
      if (e == static_cast<int>(Epi::I32)) return run_tc_group<Kind::F4, Epi::I32, kF4BN, 1>(st, probs, 1, s);
      if (e == static_cast<int>(Epi::F32)) return run_tc_group<Kind::F4, Epi::F32, kF4BN, 1>(st, probs, 1, s);
      return run_tc_group<Kind::F4, Epi::F32R, kF4BN, 1>(st, probs, 1, s);
    }
    if (e == static_cast<int>(Epi::I32)) return run_tc_group<Kind::I8, Epi::I32, kI8BN, 1>(st, probs, 1, s);
    if (e == static_cast<int>(Epi::F32)) return run_tc_group<Kind::I8, Epi::F32, kI8BN, 1>(st, probs, 1, s);
    return run_tc_group<Kind::I8, Epi::F32R, kI8BN, 1>(st, probs, 1, s);
  }
  for (int i = 0; i < count; ++i)
    if (probs[i].p.epi == static_cast<int>(Epi::F32R))
      return fail(BITMM_ERR_INVALID_ARGUMENT, "reference-order row scales are single-problem only");
  if (count == 2) {
    return fp4 ? run_tc_group<Kind::F4, Epi::ANY, kF4BN, 2>(st, probs, 2, s)
               : run_tc_group<Kind::I8, Epi::ANY, kI8BN, 2>(st, probs, 2, s);
  }
  return fp4 ? run_tc_group<Kind::F4, Epi::ANY, kF4BN, TC_GROUP_MAX>(st, probs, count, s)
             : run_tc_group<Kind::I8, Epi::ANY, kI8BN, TC_GROUP_MAX>(st, probs, count, s);
}

// The problems of one routine call: units and/or the scaled fp32 output over the same operands
// (both in one launch when both are requested).
int make_problems(const uint8_t* A8, const uint8_t* B8, int64_t m, int64_t n, int64_t kpad,
                  int shift, float scale, const float* row_scale, const float* col_scale,
                  int32_t* c_units, float* c, int64_t ldc, GemmProblem* out) {
  int cnt = 0;
  TcParams p{};
  p.shift = shift;
  p.scale = scale;
  p.row_scale = row_scale;
  p.col_scale = col_scale;
  p.ldc = ldc;
  if (c_units) {
    out[cnt] = GemmProblem{A8, B8, m, n, kpad, p};
    out[cnt].p.out_i32 = c_units;
    out[cnt].p.epi = static_cast<int>(Epi::I32);
    ++cnt;
  }
  if (c) {
    out[cnt] = GemmProblem{A8, B8, m, n, kpad, p};
    out[cnt].p.out_f32 = c;
    out[cnt].p.epi = static_cast<int>(Epi::F32);
    ++cnt;
  }
  return cnt;
}

// Common integer-GEMM tail: A8 [m][kpad], B8 [n][kpad] already expanded.
int run_int_gemm(Ctx& st, const uint8_t* A8, const uint8_t* B8, int64_t m, int64_t n,
                 int64_t kpad, int shift, float scale, const float* row_scale,
                 const float* col_scale, int32_t* c_units, float* c, int64_t ldc, cudaStream_t s,
                 bool fp4 = false) {
  GemmProblem probs[2];
  const int cnt = make_problems(A8, B8, m, n, kpad, shift, scale, row_scale, col_scale, c_units, c,
                                ldc, probs);
  return cnt ? run_problems(st, probs, cnt, fp4, s) : BITMM_OK;
}

// ---------------- in-GEMM expansion path (fx_gemm.cuh) ----------------
// Selectable with BITMM_FX=1 (measured, not the default: DESIGN.md "in-GEMM expansion").
// Sign operands are read as the caller's BitMatrix words; level operands go through one prep
// pass (2-bit codes, validated). It needs TMA-readable packed rows: an even words_per_row
// (16-byte row pitch) and 16-byte aligned bases; other calls take the default path.
// BITMM_FX=1: both operands expanded inside the GEMM; BITMM_FX=2 (hybrid): A expanded by
// unpack_operands as on the default path, B inside the GEMM (fx_gemm.cuh, AX).
int fx_mode() {
  static const int mode = getenv("BITMM_FX") ? atoi(getenv("BITMM_FX")) : 0;
  return use_fp4() && (mode == 1 || mode == 2) ? mode : 0;
}
bool fx_enabled() { return fx_mode() != 0; }
bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
bool fx_operand_ok(const OperandSrc& o, int64_t wpr) {
  if (wpr & 1) return false;
  return aligned16(o.w0) && (!o.levels || (aligned16(o.w1) && aligned16(o.w2)));
}
int64_t kcode_for(int64_t k) { return round_up(k, FX_KSLOT); }

// One routine call on the fx path: the operands in the reference layouts and its outputs
// (units and/or fp32; both come from one launch of two problems over the same operands).
struct FxItem {
  OperandSrc a, b;
  int64_t k, wpr;
  int shift;
  float scale;
  const float* row_scale;
  const float* col_scale;
  int32_t* c_units;
  float* c;
  int64_t ldc;
  bool f32r;  // reference-order per-row scales (2-bit APB layer)
  float row_pre, act_scale, act_gamma;
};

// One GEMM problem of an fx launch: packed sources after the prep pass.
struct FxProb {
  const uint8_t* a_x;  // hybrid: A expanded to e2m1 rows of kpad / 2 bytes
  const void* a_src;
  const void* b_src;
  int a_code, b_code;
  int64_t m, n, k, wpr;
  TcParams p;
};

// Expander warps per CTA. 8 of them (448 threads) cap registers at 128, where the run-time
// epilogue switch of the grouped kernel (Epi::ANY) spills; it runs 4 (384 threads, 168).
#ifndef FX_NEXP
#define FX_NEXP 8
#endif
#ifndef FX_NEXP_ANY
#define FX_NEXP_ANY 4
#endif
template <Epi EPI>
constexpr int fx_exp() { return EPI == Epi::ANY ? FX_NEXP_ANY : FX_NEXP; }

// Packed operand [rows][row_bytes] read by TMA in boxes of box_bytes x box_rows (no swizzle:
// the expanders address the slot rows directly).
int make_packed_map(CUtensorMap* map, const void* base, uint64_t row_bytes, uint64_t rows,
                    uint32_t box_bytes, uint32_t box_rows) {
  PFN_encodeTiled_t enc = encode_fn();
  if (!enc) return fail(BITMM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {row_bytes, rows};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {box_bytes, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(BITMM_ERR_CUDA, "cuTensorMapEncodeTiled (packed) failed: " + std::to_string(r));
  return BITMM_OK;
}

template <Epi EPI, int NP, int SLOT_ROW, bool AX>
int run_fx_group(Ctx& st, const FxProb* probs, int count, cudaStream_t s) {
  using S = FxShape<fx_exp<EPI>(), SLOT_ROW, AX>;
  auto kern = fx_gemm_kernel<EPI, NP, fx_exp<EPI>(), SLOT_ROW, AX>;
  BITMM_TRY(ensure_max_smem(reinterpret_cast<const void*>(kern), S::SMEM));
  FxGroup<NP> g;
  memset(&g, 0, sizeof(g));
  int tiles = 0;
  for (int i = 0; i < count; ++i) {
    const FxProb& q = probs[i];
    const uint64_t kc = static_cast<uint64_t>(kcode_for(q.k));
    if constexpr (AX)
      BITMM_TRY(make_operand_map(&g.a[i], q.a_x, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, round_up(q.k, FX_KSTAGE) / 2, q.m,
                                 S::A_ROWS));
    else
      BITMM_TRY(make_packed_map(&g.a[i], q.a_src, q.a_code ? kc / 4 : q.wpr * 8, q.m, q.a_code ? 128 : 64, S::A_ROWS));
    BITMM_TRY(make_packed_map(&g.b[i], q.b_src, q.b_code ? kc / 4 : q.wpr * 8, q.n, q.b_code ? 128 : 64, S::B_ROWS));
    TcParams p = q.p;
    p.M = static_cast<int>(q.m);
    p.N = static_cast<int>(q.n);
    const int64_t kpad = round_up(q.k, FX_KSTAGE);
    p.num_kb = static_cast<int>(kpad / FX_KSTAGE);
    p.small_acc = 36 * kpad < (int64_t{1} << 22) ? 1 : 0;
    p.shift_mul = static_cast<float>(1 << p.shift);
    p.num_m_blocks = static_cast<int>((q.m + S::TILE_M - 1) / S::TILE_M);
    p.num_n_blocks = static_cast<int>((q.n + S::BN - 1) / S::BN);
    p.num_tiles = p.num_m_blocks * p.num_n_blocks;
    p.group_m = TC_GROUP_M;
    const bool i32 = p.epi == static_cast<int>(Epi::I32);
    void* out = i32 ? static_cast<void*>(p.out_i32) : static_cast<void*>(p.out_f32);
    p.tma_store = !is_peer_memory(out) &&
                  make_output_map(&g.c[i], out, i32 ? CU_TENSOR_MAP_DATA_TYPE_INT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                                  p.N, p.M, p.ldc) ? 1 : 0;
    g.prob[i] = p;
    g.a_code[i] = q.a_code;
    g.b_code[i] = q.b_code;
    g.K[i] = static_cast<int>(q.k);
    g.tile_begin[i] = tiles;
    tiles += p.num_tiles;
  }
  g.count = count;
  for (int i = count; i <= NP; ++i) g.tile_begin[i] = tiles;
  const int units = std::min(tiles, st.sms / 2);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(2 * units));
  cfg.blockDim = dim3(S::THREADS);
  cfg.dynamicSmemBytes = S::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  ProfScope ps("fx_gemm_f4", s);
  BITMM_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, g));
  return launch_check("fx_gemm_kernel");
}

template <int SLOT_ROW, bool AX>
int dispatch_fx(Ctx& st, const FxProb* probs, int count, cudaStream_t s) {
  if (count == 1) {
    const int e = probs[0].p.epi;
    if (e == static_cast<int>(Epi::I32)) return run_fx_group<Epi::I32, 1, SLOT_ROW, AX>(st, probs, 1, s);
    if (e == static_cast<int>(Epi::F32)) return run_fx_group<Epi::F32, 1, SLOT_ROW, AX>(st, probs, 1, s);
    return run_fx_group<Epi::F32R, 1, SLOT_ROW, AX>(st, probs, 1, s);
  }
  for (int i = 0; i < count; ++i)
    if (probs[i].p.epi == static_cast<int>(Epi::F32R))
      return fail(BITMM_ERR_INVALID_ARGUMENT, "reference-order row scales are single-problem only");
  if (count == 2) return run_fx_group<Epi::ANY, 2, SLOT_ROW, AX>(st, probs, 2, s);
  return run_fx_group<Epi::ANY, TC_GROUP_MAX, SLOT_ROW, AX>(st, probs, count, s);
}

// Prep pass (codes for level operands, padding checks for sign operands with bits past K),
// then one fx_gemm launch over every problem of the items.
int run_fx(Ctx& st, const FxItem* items, int count, cudaStream_t s) {
  const bool hyb = fx_mode() == 2;
  size_t code_bytes = 1024, ax_bytes = 1024;
  for (int i = 0; i < count; ++i) {
    const int64_t kc = kcode_for(items[i].k);
    if (items[i].a.levels && !hyb) code_bytes += align_up(items[i].a.rows * kc / 4, 1024);
    if (items[i].b.levels) code_bytes += align_up(items[i].b.rows * kc / 4, 1024);
    ax_bytes += align_up(items[i].a.rows * round_up(items[i].k, FX_KSTAGE) / 2, 1024);
  }
  BITMM_TRY(arena_reserve(st.codes, code_bytes, st.stream));
  Carve cv(st.codes.ptr);
  // hybrid: every A operand expanded by one unpack_operands launch into the workspace
  UnpackSet U{};
  U.fp4 = 1;
  U.err = st.status;
  uint8_t* ax_next = nullptr;
  if (hyb) {
    BITMM_TRY(ws_reserve(st, ax_bytes));
    ax_next = static_cast<uint8_t*>(st.ws.ptr);
  }
  PrepSet P{};
  P.err = st.status;
  long long max_items = 0;
  auto prep = [&](const OperandSrc& o, int64_t k, int64_t wpr, int* code) -> const void* {
    *code = 0;
    if (o.levels) {
      const int64_t kc = kcode_for(k);
      uint2* codes = cv.take<uint2>(o.rows * kc / 4);
      PrepOperand& q = P.op[P.count++];
      q = PrepOperand{o.w0, o.w1, o.w2, codes, o.rows, static_cast<int>(wpr), static_cast<int>(k), 0,
                      static_cast<int>(kc / 64), 1, o.rows * std::max<int64_t>(wpr, kc / 64)};
      max_items = std::max(max_items, q.items);
      *code = 1;
      return codes;
    }
    if (wpr * 64 > k) {  // words holding bits past K: the padding check (tensor.cpp:78-89)
      PrepOperand& q = P.op[P.count++];
      q = PrepOperand{o.w0, nullptr, nullptr, nullptr, o.rows, static_cast<int>(wpr), static_cast<int>(k),
                      static_cast<int>(k / 64), 0, 0, o.rows * (wpr - k / 64)};
      max_items = std::max(max_items, q.items);
    }
    return o.w0;
  };
  FxProb probs[TC_GROUP_MAX];
  int np = 0;
  bool any_code = false;
  for (int i = 0; i < count; ++i) {
    const FxItem& it = items[i];
    FxProb q{};
    if (hyb) {
      const int64_t kpad = round_up(it.k, FX_KSTAGE);
      q.a_x = ax_next;
      ax_next += align_up(it.a.rows * kpad / 2, 1024);
      U.op[U.count++] = make_unpack_operand(it.a, it.wpr, it.k, kpad, const_cast<uint8_t*>(q.a_x));
    } else {
      q.a_src = prep(it.a, it.k, it.wpr, &q.a_code);
    }
    q.b_src = prep(it.b, it.k, it.wpr, &q.b_code);
    any_code = any_code || q.a_code || q.b_code;
    q.m = it.a.rows;
    q.n = it.b.rows;
    q.k = it.k;
    q.wpr = it.wpr;
    TcParams p{};
    p.shift = it.shift;
    p.scale = it.scale;
    p.row_scale = it.row_scale;
    p.col_scale = it.col_scale;
    p.ldc = it.ldc;
    if (it.f32r) {
      p.row_pre = it.row_pre;
      p.act_scale = it.act_scale;
      p.act_gamma = it.act_gamma;
      p.out_f32 = it.c;
      p.epi = static_cast<int>(Epi::F32R);
      q.p = p;
      probs[np++] = q;
      continue;
    }
    if (it.c_units) {
      q.p = p;
      q.p.out_i32 = it.c_units;
      q.p.epi = static_cast<int>(Epi::I32);
      probs[np++] = q;
    }
    if (it.c) {
      q.p = p;
      q.p.out_f32 = it.c;
      q.p.epi = static_cast<int>(Epi::F32);
      probs[np++] = q;
    }
  }
  if (np > TC_GROUP_MAX) return fail(BITMM_ERR_INVALID_ARGUMENT, "batch exceeds 4 GEMM outputs");
  if (P.count) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks_for(max_items, 256), static_cast<unsigned>(P.count));
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    ProfScope ps("prep_operands", s);
    BITMM_CUDA_TRY(cudaLaunchKernelEx(&cfg, prep_operands_kernel, P));
    BITMM_TRY(launch_check("prep_operands_kernel"));
  }
  if (np == 0) return BITMM_OK;
  if (hyb) {
    BITMM_TRY(run_unpack_set(U, s));
    return any_code ? dispatch_fx<128, true>(st, probs, np, s) : dispatch_fx<64, true>(st, probs, np, s);
  }
  return any_code ? dispatch_fx<128, false>(st, probs, np, s) : dispatch_fx<64, false>(st, probs, np, s);
}

FxItem fx_item(const OperandSrc& a, const OperandSrc& b, int64_t k, int64_t wpr, int shift, float scale,
               const float* row_scale, const float* col_scale, int32_t* c_units, float* c, int64_t ldc) {
  FxItem it{};
  it.a = a;
  it.b = b;
  it.k = k;
  it.wpr = wpr;
  it.shift = shift;
  it.scale = scale;
  it.row_scale = row_scale;
  it.col_scale = col_scale;
  it.c_units = c_units;
  it.c = c;
  it.ldc = ldc;
  return it;
}

int check_gemm_dims(int64_t m, int64_t n, int64_t k, int64_t wpr, int64_t ldc) {
  if (m <= 0 || k <= 0 || n <= 0) return fail(BITMM_ERR_INVALID_ARGUMENT, "gemm dimensions must be positive");
  if (k > BITMM_MAX_SHARED_DIM)
    return fail(BITMM_ERR_INVALID_ARGUMENT, "shared dimension exceeds the 2^20 accumulator bound");
  if (wpr * 64 < k) return fail(BITMM_ERR_INVALID_ARGUMENT, "words_per_row too small for the column count");
  if (ldc < n) return fail(BITMM_ERR_INVALID_ARGUMENT, "ldc smaller than the output column count");
  if (m > INT32_MAX / 2 || n > INT32_MAX / 2) return fail(BITMM_ERR_INVALID_ARGUMENT, "gemm dimension too large");
  return BITMM_OK;
}

int status_error(int flag) {
  // a timed-out input copy first: the inputs the GEMM read are then not the caller's
  if (flag & ERR_COPY_TIMEOUT) return fail(BITMM_ERR_CUDA, "input copy did not complete (flag wait timed out)");
  if (flag & ERR_ENCODING) return fail(BITMM_ERR_INVALID_ENCODING, "invalid ternary plane encoding or nonzero plane padding");
  if (flag & ERR_PADDING) return fail(BITMM_ERR_INVALID_ARGUMENT, "bit matrix padding must be zero");
  if (flag & ERR_LEVEL) return fail(BITMM_ERR_INVALID_ARGUMENT, "2-bit level out of range");
  if (flag & ERR_ALPHA) return fail(BITMM_ERR_INVALID_ARGUMENT, "alpha must be positive");
  return BITMM_OK;
}

// A host call's status: copied into the lease's pinned word behind the call's work on s (no
// pageable 4-byte copy, no synchronous memset), then read.
int read_status_host(HostCtx& h, cudaStream_t s) {
  BITMM_CUDA_TRY(cudaMemcpyAsync(h.status_host, h.sctx->status, sizeof(int), cudaMemcpyDeviceToHost, s));
  BITMM_CUDA_TRY(cudaMemsetAsync(h.sctx->status, 0, sizeof(int), s));
  BITMM_CUDA_TRY(cudaStreamSynchronize(s));
  return status_error(*h.status_host);
}

int read_status(Ctx& st, cudaStream_t s) {
  BITMM_CUDA_TRY(cudaStreamSynchronize(s));
  int flag = 0;
  BITMM_CUDA_TRY(cudaMemcpy(&flag, st.status, sizeof(int), cudaMemcpyDeviceToHost));
  BITMM_CUDA_TRY(cudaMemset(st.status, 0, sizeof(int)));
  return status_error(flag);
}

// ---------------- host-flavour pipeline ----------------
// A host call's time is mostly the device -> host copy of its output (4 B per cell). Valid
// calls produce the output in up to kPipeChunks slices of one dimension: slice i's inputs are
// copied in and its GEMM runs on the call's stream, then its output is copied out on st.d2h,
// so the D2H of slice i overlaps the H2D and GEMM of slice i+1.
constexpr int kPipeChunks = 8;
constexpr size_t kPipeMinOutBytes = size_t{32} << 20;  // smaller outputs go in one slice

int64_t pipe_step(int64_t total, size_t out_bytes, int64_t align) {
  if (out_bytes < kPipeMinOutBytes || total < 2 * align) return total;
  return round_up((total + kPipeChunks - 1) / kPipeChunks, align);
}

// body(c0, c1): enqueue slice [c0, c1)'s input copies and GEMM on s. out(c0, c1, d2h):
// enqueue its output copies on d2h. Always drains d2h before returning.
template <class Body, class Out>
int run_pipelined(HostCtx& st, cudaStream_t s, int64_t total, int64_t step, Body&& body,
                  Out&& out) {
  int rc = BITMM_OK;
  int i = 0;
  for (int64_t c0 = 0; c0 < total; c0 += step, ++i) {
    const int64_t c1 = std::min(total, c0 + step);
    rc = body(c0, c1);
    if (rc != BITMM_OK) break;
    cudaEvent_t ev = st.pipe_ev[i % kPipeChunks];
    if (cudaEventRecord(ev, s) != cudaSuccess || cudaStreamWaitEvent(st.d2h, ev, 0) != cudaSuccess) {
      rc = fail(BITMM_ERR_CUDA, std::string("pipeline event: ") + cudaGetErrorString(cudaGetLastError()));
      break;
    }
    rc = out(c0, c1, st.d2h);
    if (rc != BITMM_OK) break;
  }
  const cudaError_t e = cudaStreamSynchronize(st.d2h);
  if (rc == BITMM_OK && e != cudaSuccess) rc = fail(BITMM_ERR_CUDA, cudaGetErrorString(e));
  return rc;
}

// 16-bit output wire (wire.cuh). Same slicing as run_pipelined, with the body split in two:
// in(c0, c1, stream) enqueues slice [c0, c1)'s input copies (all slices up front, on st.h2d),
// gemm(c0, c1) its GEMM on s once those copies are done. block(c0, c1) gives the output
// block {row0, rows, col0, cols} the slice writes as int32 units into dcu (leading
// dimension wo.ldc). A narrowing kernel follows each slice's GEMM on s and packs
// its units into dwire; the d2h stream then copies them into pinned host staging in row
// parts of about kWirePartBytes, each with its own event. The host pool widens the parts into
// the caller's buffers in order as they land; its batch starts before the slices are enqueued
// (run_wire_items).
// Copied parts of ~2 MiB: larger parts delay the host's widening, smaller ones slow the
// copies. Measured per routine with 2, 4 and 8 parts per slice (profiles/dev/ab_wire_parts.sh):
// the 4 MiB slices of 1/1 and 2/2 were fastest in two parts, the 8 MiB slices of 1/2 in four.
constexpr size_t kWirePartBytes = size_t{2} << 20;
// BITMM_WIRE_SPIN=1: the host pool polls each part's copy event instead of sleeping on a
// blocking-sync event (A/B of the wake-up latency). Read once: the events are created with it.
bool wire_spin() {
  static const bool on = std::getenv("BITMM_WIRE_SPIN") && std::atoi(std::getenv("BITMM_WIRE_SPIN")) == 1;
  return on;
}
constexpr int kWireMaxParts = 8;

struct OutBlock {
  int64_t row0, rows, col0, cols;
};

int host_stage_reserve(HostCtx& st, size_t bytes) {
  if (bytes <= st.host_stage_bytes) return BITMM_OK;
  if (st.host_stage) BITMM_CUDA_TRY(cudaFreeHost(st.host_stage));
  st.host_stage = nullptr;
  st.host_stage_bytes = 0;
  BITMM_CUDA_TRY(cudaHostAlloc(&st.host_stage, bytes, cudaHostAllocDefault));
  st.host_stage_bytes = bytes;
  return BITMM_OK;
}

// BITMM_HOST_WIRE=32 keeps the 4-byte output copies (A/B runs and tests of that path).
// Outputs below kPipeMinOutBytes keep the 4-byte copy: one unsliced call gains nothing from
// the wire, and the host pool's start-up plus parallel first-touch faults on a fresh
// pageable DenseMatrix made a 1024^3 drop-in call slower (0.88 vs 0.66 ms, the reference's
// acceptance criterion 8).
Wire host_wire(int routine, int64_t k, size_t out_bytes) {
  const char* e = std::getenv("BITMM_HOST_WIRE");
  if (e && std::atoi(e) == 32) return Wire::None;
  const char* mb = std::getenv("BITMM_WIRE_MIN_BYTES");  // A/B of the threshold
  if (out_bytes < (mb ? static_cast<size_t>(std::atoll(mb)) : kPipeMinOutBytes)) return Wire::None;
  return wire_for(routine, k);
}

// One routine's share of a wire pipeline: its slices (the output split along one dimension),
// their input copies, GEMMs and output blocks, and its buffers.
struct WireItem {
  int64_t total, step;
  std::function<int(int64_t, int64_t, cudaStream_t)> in;  // slice [c0, c1)'s input copies
  std::function<int(int64_t, int64_t)> gemm;              // its GEMM on the call's stream
  std::function<OutBlock(int64_t, int64_t)> block;        // the output block it writes
  WireOut wo;
  const int32_t* dcu;  // the GEMM's int32 units (leading dimension wo.ldc)
  uint16_t* dwire;     // device wire words
  size_t wire_words;
};

// Runs one or more wire items as one pipeline (a single call is one item; bitmm_gemm_batch_host
// merges several): every item's input copies go first, the host pool's widening batch covers
// every part of every item, and the slices of all items are enqueued in order, so the copy
// link stays busy from the first item's first slice to the last item's last.
int run_wire_items(HostCtx& st, cudaStream_t s, std::vector<WireItem>& items) {
  // How each slice's GEMM waits for its input copies (see slice_wait_mode); a slice whose
  // flag write fails falls back to an event.
  const SliceWait mode = slice_wait_mode();
  const bool flags = mode != SliceWait::Event;
  int nslices = 0;
  for (const WireItem& w : items) nslices += static_cast<int>((w.total + w.step - 1) / w.step);
  if (nslices > kMaxWireSlices) return fail(BITMM_ERR_INVALID_ARGUMENT, "too many pipeline slices");
  bool slice_flag[kMaxWireSlices];
  const uint32_t epoch = ++st.in_epoch == 0 ? ++st.in_epoch : st.in_epoch;
  const auto t_call = std::chrono::steady_clock::now();
  static const bool trace = std::getenv("BITMM_WIRE_TRACE") != nullptr;
  // BITMM_WIRE_TRACE=nowiden: timeline of the copies alone (outputs left unwritten)
  static const bool skip_widen = trace && std::string(std::getenv("BITMM_WIRE_TRACE")) == "nowiden";
  // trace only: a device timeline of slice completions (GEMM + narrow on s, copies on d2h)
  std::vector<std::pair<std::string, cudaEvent_t>> tl;
  if (trace) st.timeline = &tl;
  auto mark = [&](const std::string& what, cudaStream_t on) { trace_mark(st, what, on); };
  mark("start", s);
  size_t wire_words = 0;
  std::vector<size_t> hw_off;  // each item's words in the pinned staging
  for (const WireItem& w : items) {
    hw_off.push_back(wire_words);
    wire_words += w.wire_words;
  }
  // 12-bit packing (wire.cuh; BITMM_WIRE_BITS=12) for items whose output blocks all have a
  // multiple of 16 columns. Measured, not the default: the last copy of the bench step lands
  // ~0.4 ms earlier (3.2 vs 3.6 ms), but the host's widening, bound by host memory traffic
  // (DMA writes + 256 MB of output stores), ends at the same time (e2e 64.8 vs 66.2 T-upd/s
  // batched, 58.5 vs 57.1 per call; profiles/dev/e2e_ab.py, BITMM_WIRE_TRACE).
  const bool w12_env = std::getenv("BITMM_WIRE_BITS") && std::atoi(std::getenv("BITMM_WIRE_BITS")) == 12;
  std::vector<char> item12;
  for (const WireItem& w : items) {
    bool ok = w12_env;
    for (int64_t c0 = 0; c0 < w.total && ok; c0 += w.step) ok = w.block(c0, std::min(w.total, c0 + w.step)).cols % 16 == 0;
    item12.push_back(ok ? 1 : 0);
  }
  struct Part {
    int item;
    OutBlock b;
    int64_t r0, r1;
    size_t off;      // word offset of the block in the item's wire buffer
    bool p12;        // crosses PCIe packed in 12 bits (wire.cuh)
    size_t off12;    // its bytes in the 12-bit buffers (device and pinned)
    size_t bytes12;  // header + payload
  };
  std::vector<Part> parts;
  // Every slice's input copies go first, on their own stream: queued on s behind the
  // previous slice's GEMM they ran at a third of the link rate while the output copies
  // were in flight (BITMM_WIRE_TRACE device timelines). Issuing them two slices ahead of
  // the GEMMs instead measured slower (e2e 50 vs 56-59 T-upd/s).
  BITMM_CUDA_TRY(cudaEventRecord(st.in_ev[kMaxWireSlices], s));  // after the calls' setup copies
  BITMM_CUDA_TRY(cudaStreamWaitEvent(st.h2d, st.in_ev[kMaxWireSlices], 0));
  {
    int j = 0;
    for (WireItem& w : items)
      for (int64_t c0 = 0; c0 < w.total; c0 += w.step, ++j) {
        BITMM_TRY(w.in(c0, std::min(w.total, c0 + w.step), st.h2d));
        slice_flag[j] = flags && !fault_flag_write() && write_value_fn()(reinterpret_cast<CUstream>(st.h2d),
                                                  reinterpret_cast<CUdeviceptr>(st.in_flags + j), epoch,
                                                  0) == CUDA_SUCCESS;
        if (!slice_flag[j]) {
          cudaGetLastError();
          BITMM_CUDA_TRY(cudaEventRecord(st.in_ev[j], st.h2d));
        }
        mark("i" + std::to_string(j), st.h2d);
      }
  }
  // The copied parts of every slice, known before anything is enqueued: ~kWirePartBytes of wire
  // words each, split by output rows.
  std::vector<int> slice_parts{0};  // global slice j owns parts [slice_parts[j], slice_parts[j + 1])
  for (int it = 0; it < static_cast<int>(items.size()); ++it) {
    const WireItem& w = items[it];
    size_t off = 0;
    for (int64_t c0 = 0; c0 < w.total; c0 += w.step) {
      const OutBlock b = w.block(c0, std::min(w.total, c0 + w.step));
      const int64_t cells = b.rows * b.cols;
      const int64_t nparts = std::min<int64_t>(
          kWireMaxParts, std::max<int64_t>(1, (cells * 2 + kWirePartBytes / 2) / kWirePartBytes));
      const int64_t per = (b.rows + nparts - 1) / nparts;
      for (int64_t r0 = 0; r0 < b.rows; r0 += per)
        parts.push_back(Part{it, b, b.row0 + r0, b.row0 + std::min(b.rows, r0 + per), off, item12[it] != 0, 0, 0});
      slice_parts.push_back(static_cast<int>(parts.size()));
      off += static_cast<size_t>(cells);
    }
  }
  // the 12-bit parts: 16-byte header {min, max}, payload of 1.5 bytes per cell; the pinned copy
  // of each is padded by 16 bytes (the host's 16-byte loads read 4 bytes past a row's last group)
  size_t bytes12 = 0;
  for (Part& q : parts) {
    if (!q.p12) continue;
    q.off12 = bytes12;
    q.bytes12 = 16 + align_up(static_cast<size_t>((q.r1 - q.r0) * q.b.cols) * 3 / 2, 16);
    bytes12 += q.bytes12 + 16;
  }
  BITMM_TRY(host_stage_reserve(st, wire_words * 2 + bytes12));
  uint16_t* const hw_base = static_cast<uint16_t*>(st.host_stage);
  uint8_t* const h12 = static_cast<uint8_t*>(st.host_stage) + wire_words * 2;
  uint8_t* d12 = nullptr;
  if (bytes12 > 0) {
    BITMM_TRY(arena_reserve(st.w12, bytes12, s));
    d12 = static_cast<uint8_t*>(st.w12.ptr);
  }
  while (st.wire_ev.size() < parts.size()) {
    cudaEvent_t e = nullptr;
    BITMM_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming | (wire_spin() ? 0 : cudaEventBlockingSync)));
    st.wire_ev.push_back(e);
  }
  // One pool batch for the whole call: each task widens a row range of one part after waiting
  // for that part's copy. Tasks are handed out in part order, so the pool follows the copies
  // without a barrier per part. The batch starts BEFORE the slices are enqueued (the enqueue
  // takes ~0.3 ms of host time for eight slices, during which the first parts already land): a
  // task first waits until its part's copy has been enqueued, then for the copy itself.
  struct Task {
    int part;
    int64_t r0, r1;
  };
  std::vector<Task> tasks;
  for (int p = 0; p < static_cast<int>(parts.size()); ++p) {
    const Part& q = parts[p];
    const int64_t rows_per_task = std::max<int64_t>(1, (int64_t{1} << 16) / std::max<int64_t>(1, q.b.cols));
    for (int64_t r = q.r0; r < q.r1; r += rows_per_task) tasks.push_back(Task{p, r, std::min(q.r1, r + rows_per_task)});
  }
  std::mutex ready_mu;
  std::condition_variable ready_cv;
  int parts_ready = 0;  // parts whose copy and event are enqueued
  bool abort = false;   // the enqueue failed: the remaining tasks return at once
  auto publish = [&](int ready, bool failed) {
    {
      std::lock_guard<std::mutex> lk(ready_mu);
      parts_ready = ready;
      abort = abort || failed;
    }
    ready_cv.notify_all();
  };
  const auto t0 = std::chrono::steady_clock::now();
  std::atomic<int> copy_err{0};
  std::atomic<int64_t> wait_ns{0};
  std::atomic<uint64_t> refetch_bytes{0};  // 12-bit parts fetched again as 16-bit words
  std::unique_ptr<std::once_flag[]> refetch(new std::once_flag[std::max<size_t>(1, parts.size())]);
  std::unique_ptr<std::atomic<int>[]> landed(new std::atomic<int>[std::max<size_t>(1, parts.size())]);
  for (size_t p = 0; p < parts.size(); ++p) landed[p].store(0, std::memory_order_relaxed);
  // BITMM_WIRE_EARLY=0: the batch starts after the whole enqueue (round-1 order, A/B)
  const bool early = !(std::getenv("BITMM_WIRE_EARLY") && std::atoi(std::getenv("BITMM_WIRE_EARLY")) == 0);
  auto task = [&](int i) {
    const Task& t = tasks[i];
    {
      std::unique_lock<std::mutex> lk(ready_mu);
      ready_cv.wait(lk, [&] { return abort || parts_ready > t.part; });
      if (abort) return;
    }
    const auto w0 = trace ? std::chrono::steady_clock::now() : std::chrono::steady_clock::time_point{};
    // the first task of a part to see its copy complete marks it, so the part's other tasks skip
    // the driver call (16 threads synchronising on events contend inside the driver)
    if (landed[t.part].load(std::memory_order_acquire)) {
    } else if (wire_spin()) {  // poll the part's event (no sleep / wake-up on the blocking-sync path)
      cudaError_t q;
      while ((q = cudaEventQuery(st.wire_ev[t.part])) == cudaErrorNotReady) std::this_thread::yield();
      if (q != cudaSuccess) {
        copy_err.store(1);
        return;
      }
    } else if (cudaEventSynchronize(st.wire_ev[t.part]) != cudaSuccess) {
      copy_err.store(1);
      return;
    }
    landed[t.part].store(1, std::memory_order_release);
    if (trace) wait_ns += std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - w0).count();
    const Part& q = parts[t.part];
    if (skip_widen) return;
    uint16_t* const hw = hw_base + hw_off[q.item];
    if (q.p12) {
      const int* hdr = reinterpret_cast<const int*>(h12 + q.off12);
      if (hdr[1] - hdr[0] <= 4095) {
        wire_expand_range12(items[q.item].wo, h12 + q.off12 + 16, static_cast<uint16_t>(hdr[0]), q.r0, q.b.col0,
                            q.b.cols, t.r0, t.r1);
        return;
      }
      // the part's words span more than 12 bits: fetch them as 16-bit words (still on the device)
      std::call_once(refetch[t.part], [&] {
        const size_t o = q.off + static_cast<size_t>((q.r0 - q.b.row0) * q.b.cols);
        const size_t bytes = static_cast<size_t>((q.r1 - q.r0) * q.b.cols) * 2;
        if (cudaMemcpy(hw + o, items[q.item].dwire + o, bytes, cudaMemcpyDeviceToHost) != cudaSuccess)
          copy_err.store(1);
        refetch_bytes += bytes;
      });
      if (copy_err.load()) return;
    }
    wire_expand_range(items[q.item].wo, hw + q.off, q.b.row0, q.b.col0, q.b.cols, t.r0, t.r1);
  };
  if (early) host_pool_start(static_cast<int>(tasks.size()), task);
  int rc = BITMM_OK;
  int i = 0;  // global slice
  for (int it = 0; it < static_cast<int>(items.size()) && rc == BITMM_OK; ++it) {
  WireItem& w = items[it];
  const WireOut& wo = w.wo;
  uint16_t* const hw = hw_base + hw_off[it];
  for (int64_t c0 = 0; c0 < w.total && rc == BITMM_OK; c0 += w.step, ++i) {
    const int64_t c1 = std::min(w.total, c0 + w.step);
    if (slice_flag[i] && mode == SliceWait::Kernel) {
      wait_flag_kernel<<<1, 32, 0, s>>>(st.in_flags + i, epoch, st.sctx->status);
      rc = launch_check("wait_flag_kernel");
      if (rc != BITMM_OK) break;
    } else if (slice_flag[i]) {
      if (wait_value_fn()(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(st.in_flags + i), epoch,
                          CU_STREAM_WAIT_VALUE_EQ) != CUDA_SUCCESS) {
        rc = fail(BITMM_ERR_CUDA, "cuStreamWaitValue32 failed");
        break;
      }
    } else if (cudaStreamWaitEvent(s, st.in_ev[i], 0) != cudaSuccess) {
      rc = fail(BITMM_ERR_CUDA, "pipeline input event");
      break;
    }
    mark("h" + std::to_string(i), s);
    rc = w.gemm(c0, c1);
    if (rc != BITMM_OK) break;
    const OutBlock b = parts[slice_parts[i]].b;
    const size_t off = parts[slice_parts[i]].off;
    // the narrowing runs on the GEMM's stream: on the copy stream it would wait for SMs
    // behind the next slice's persistent GEMM
    const int64_t cells = b.rows * b.cols;
    const unsigned grid = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((cells / 4 + 255) / 256, int64_t{st.sctx->sms} * 8)));
    narrow_units_kernel<<<grid, 256, 0, s>>>(w.dcu + b.row0 * wo.ldc + b.col0, wo.ldc, w.dwire + off,
                                             b.rows, b.cols, static_cast<int>(wo.mode), wo.k);
    rc = launch_check("narrow_units_kernel");
    if (rc != BITMM_OK) break;
    if (parts[slice_parts[i]].p12) {  // the slice's parts in 12 bits: headers, min/max, pack
      Wire12Set S{};
      int64_t most = 0;
      for (int p = slice_parts[i]; p < slice_parts[i + 1]; ++p) {
        const Part& q = parts[p];
        const size_t o = q.off + static_cast<size_t>((q.r0 - b.row0) * b.cols);
        S.p[S.count++] = Wire12Part{w.dwire + o, d12 + q.off12, (q.r1 - q.r0) * b.cols};
        most = std::max(most, (q.r1 - q.r0) * b.cols);
      }
      const dim3 grid(static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((most / 8 + 255) / 256, 64))),
                      static_cast<unsigned>(S.count));
      wire12_init_kernel<<<1, 32, 0, s>>>(S);
      rc = launch_check("wire12_init_kernel");
      if (rc != BITMM_OK) break;
      wire12_minmax_kernel<<<grid, 256, 0, s>>>(S, static_cast<int>(wo.mode));
      rc = launch_check("wire12_minmax_kernel");
      if (rc != BITMM_OK) break;
      wire12_pack_kernel<<<grid, 256, 0, s>>>(S, static_cast<int>(wo.mode));
      rc = launch_check("wire12_pack_kernel");
      if (rc != BITMM_OK) break;
    }
    mark("g" + std::to_string(i), s);
    cudaEvent_t ev = st.pipe_ev[i % kPipeChunks];
    if (cudaEventRecord(ev, s) != cudaSuccess || cudaStreamWaitEvent(st.d2h, ev, 0) != cudaSuccess) {
      rc = fail(BITMM_ERR_CUDA, std::string("pipeline event: ") + cudaGetErrorString(cudaGetLastError()));
      break;
    }
    for (int p = slice_parts[i]; p < slice_parts[i + 1] && rc == BITMM_OK; ++p) {
      const Part& q = parts[p];
      const size_t o = q.off + static_cast<size_t>((q.r0 - b.row0) * b.cols);
      const size_t bytes = q.p12 ? q.bytes12 : static_cast<size_t>((q.r1 - q.r0) * b.cols) * 2;
      void* dst = q.p12 ? static_cast<void*>(h12 + q.off12) : static_cast<void*>(hw + o);
      const void* src = q.p12 ? static_cast<const void*>(d12 + q.off12) : static_cast<const void*>(w.dwire + o);
      if (cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st.d2h) != cudaSuccess) {
        rc = fail(BITMM_ERR_CUDA, std::string("wire copy: ") + cudaGetErrorString(cudaGetLastError()));
        break;
      }
      g_d2h_bytes += bytes;
      if (cudaEventRecord(st.wire_ev[p], st.d2h) != cudaSuccess) rc = fail(BITMM_ERR_CUDA, "wire event record");
    }
    if (rc != BITMM_OK) break;
    if (early) publish(slice_parts[i + 1], false);
    mark("c" + std::to_string(i), st.d2h);
  }
  }
  if (early) {
    if (rc != BITMM_OK) publish(parts_ready, true);
    host_pool_join();
  } else if (rc == BITMM_OK) {
    publish(static_cast<int>(parts.size()), false);
    host_pool_run(static_cast<int>(tasks.size()), task);
  }
  if (trace) {
    const auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    const auto t1 = std::chrono::steady_clock::now();
    cudaEventSynchronize(st.wire_ev[0]);
    std::fprintf(stderr, "[bitmm wire] %zu parts, %zu tasks, %zu words: setup %.3f ms, enqueue + host widen %.3f ms "
                 "(%d threads, %.3f thread-ms waiting for copies)\n",
                 parts.size(), tasks.size(), wire_words, ms(t_call, t0), ms(t0, t1), host_pool_size(),
                 wait_ns.load() * 1e-6);
    cudaDeviceSynchronize();
    std::string line = "[bitmm wire] device timeline (ms):";
    for (auto& [what, e] : tl) {
      float m = 0;
      cudaEventElapsedTime(&m, tl[0].second, e);
      line += " " + what + "=" + std::to_string(m).substr(0, 5);
    }
    std::fprintf(stderr, "%s\n", line.c_str());
    for (auto& [what, e] : tl) cudaEventDestroy(e);
    st.timeline = nullptr;
  }
  g_d2h_bytes += refetch_bytes.load();
  if (rc == BITMM_OK && copy_err.load()) rc = fail(BITMM_ERR_CUDA, std::string("wire copy: ") + cudaGetErrorString(cudaGetLastError()));
  const cudaError_t e = cudaStreamSynchronize(st.d2h);
  if (rc == BITMM_OK && e != cudaSuccess) rc = fail(BITMM_ERR_CUDA, cudaGetErrorString(e));
  return rc;
}

// A routine's wire pipeline: run now (one item), or, in a batch's second pass, handed to the
// batch, which runs every item's pipeline as one.
int run_or_defer_wire(HostCtx& h, cudaStream_t s, WireItem&& w) {
  if (g_batch) {
    g_batch->items->push_back(std::move(w));
    return BITMM_OK;
  }
  std::vector<WireItem> one;
  one.push_back(std::move(w));
  BITMM_TRY(run_wire_items(h, s, one));
  return read_status_host(h, s);
}

// Where a host GEMM call's output goes: the caller's buffers, given up front (the *_host
// calls), or obtained late through a callback (bitmm_gemm_host_late), after the call's
// copies and kernels are enqueued, so the caller's allocation overlaps the device work.
struct HostOut {
  int32_t* c_units = nullptr;
  float* c = nullptr;
  int64_t ldc = 0;
  bool want_units = false, want_c = false;
  bitmm_out_fn fn = nullptr;
  void* user = nullptr;
  bool late() const { return fn != nullptr; }
  static HostOut given(int32_t* u, float* c, int64_t ldc) {
    HostOut o;
    o.c_units = u;
    o.c = c;
    o.ldc = ldc;
    o.want_units = u != nullptr;
    o.want_c = c != nullptr;
    return o;
  }
  // Calls the callback (once) and checks what it returned against the call.
  int resolve(int64_t n) {
    if (!fn) return BITMM_OK;
    bitmm_host_out out{nullptr, nullptr, n};
    const int r = fn(user, &out);
    fn = nullptr;
    if (r != 0) return fail(BITMM_ERR_INVALID_ARGUMENT, "output callback failed");
    if ((want_units && !out.c_units) || (want_c && !out.c))
      return fail(BITMM_ERR_INVALID_ARGUMENT, "output callback returned a null buffer");
    if (out.ldc < n) return fail(BITMM_ERR_INVALID_ARGUMENT, "ldc smaller than the output column count");
    c_units = want_units ? out.c_units : nullptr;
    c = want_c ? out.c : nullptr;
    ldc = out.ldc;
    return BITMM_OK;
  }
};

bool is_pinned_host(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// One-slice host outputs (below kPipeMinOutBytes) into pageable or late destinations. The GEMM
// has been enqueued on s with its outputs at dcu / dc (rows x cols, leading dimension ldd). A
// pageable destination written by cudaMemcpy is filled through the driver's own bounce buffer
// at ~16 GB/s (0.26 ms for the 4 MB of a 1024^2 fp32 result); here the output is copied into
// the lease's pinned staging in row parts of about 1 MiB, each with an event, and the calling
// thread copies every part into the destination as soon as it lands (memcpy into the
// destination's leading dimension). The status word the GEMM may have latched travels in the same stream
// order into pinned memory, so an error is known before any caller memory is written. A late
// destination is resolved after everything is enqueued.
int run_staged(HostCtx& st, cudaStream_t s, int64_t rows, int64_t cols, int64_t ldd, const int32_t* dcu,
               const float* dc, HostOut& o) {
  // BITMM_STAGED_TRACE: per-call host timeline (us). The copy into the destination runs on the
  // calling thread: copying with the host pool (BITMM_STAGED_POOL=1; =2 also keeps CUDA waits
  // off the pool) took 90 instead of 265 us for 4 MB, but made the caller's next allocation and
  // zero-fill of its DenseMatrix take 1.0-1.4 ms instead of 0.13 ms (4-16 threads; latency_b200
  // with BITMM_STAGED_TRACE, profiles/dev/dropin_latency2.sh), so the call got 3x slower.
  static const bool trace = std::getenv("BITMM_STAGED_TRACE") != nullptr;
  static const int pool_mode = std::getenv("BITMM_STAGED_POOL") ? std::atoi(std::getenv("BITMM_STAGED_POOL")) : 0;
  const bool pool = pool_mode != 0;
  // BITMM_STAGED_NT=1: streaming-store copy (A/B)
  static const bool nt = std::getenv("BITMM_STAGED_NT") && std::atoi(std::getenv("BITMM_STAGED_NT")) == 1;
  const auto t_in = std::chrono::steady_clock::now();
  auto us = [&] {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t_in).count();
  };
  BITMM_CUDA_TRY(cudaMemcpyAsync(st.status_host, st.sctx->status, sizeof(int), cudaMemcpyDeviceToHost, s));
  BITMM_CUDA_TRY(cudaMemsetAsync(st.sctx->status, 0, sizeof(int), s));
  BITMM_CUDA_TRY(cudaEventRecord(st.pipe_ev[0], s));
  BITMM_CUDA_TRY(cudaStreamWaitEvent(st.d2h, st.pipe_ev[0], 0));
  const size_t mat_bytes = static_cast<size_t>(rows * ldd) * 4;
  const int nmat = (dcu ? 1 : 0) + (dc ? 1 : 0);
  BITMM_TRY(host_stage_reserve(st, nmat * mat_bytes));
  const int64_t row_bytes = ldd * 4;
  const int64_t part_rows = std::max<int64_t>(1, std::max<int64_t>((int64_t{1} << 20) / row_bytes, (rows + 15) / 16));
  struct Part {
    int mat;  // 0 units, 1 fp32
    int64_t r0, r1;
  };
  std::vector<Part> parts;
  uint8_t* stage = static_cast<uint8_t*>(st.host_stage);
  for (int mat = 0; mat < 2; ++mat) {
    const void* src = mat == 0 ? static_cast<const void*>(dcu) : static_cast<const void*>(dc);
    if (!src) continue;
    const size_t base = (mat == 1 && dcu) ? mat_bytes : 0;
    for (int64_t r0 = 0; r0 < rows; r0 += part_rows) {
      const int64_t r1 = std::min(rows, r0 + part_rows);
      BITMM_CUDA_TRY(cudaMemcpyAsync(stage + base + r0 * row_bytes, static_cast<const uint8_t*>(src) + r0 * row_bytes,
                                     (r1 - r0) * row_bytes, cudaMemcpyDeviceToHost, st.d2h));
      if (st.stage_ev.size() <= parts.size()) {
        cudaEvent_t e = nullptr;
        BITMM_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        st.stage_ev.push_back(e);
      }
      BITMM_CUDA_TRY(cudaEventRecord(st.stage_ev[parts.size()], st.d2h));
      parts.push_back(Part{mat, r0, r1});
    }
  }
  g_d2h_bytes += nmat * static_cast<uint64_t>(rows * cols) * 4;
  // everything is enqueued: the caller's destination now (late outputs), then the status word
  const double t_enq = us();
  BITMM_TRY(o.resolve(cols));
  const double t_res = us();
  if (parts.empty()) return BITMM_OK;
  BITMM_CUDA_TRY(cudaEventSynchronize(st.stage_ev[0]));
  const double t_first = us();
  BITMM_TRY(status_error(*st.status_host));
  // tasks of ~256 KB, handed out in part order
  struct Task {
    int part;
    int64_t r0, r1;
  };
  std::vector<Task> tasks;
  const int64_t task_rows = std::max<int64_t>(1, (int64_t{1} << 18) / std::max<int64_t>(1, cols * 4));
  for (int p = 0; p < static_cast<int>(parts.size()); ++p)
    for (int64_t r = parts[p].r0; r < parts[p].r1; r += task_rows)
      tasks.push_back(Task{p, r, std::min(parts[p].r1, r + task_rows)});
  std::atomic<int> copy_err{0};
  if (pool_mode == 2) BITMM_CUDA_TRY(cudaEventSynchronize(st.stage_ev[parts.size() - 1]));  // A/B: no CUDA calls on the pool
  auto copy = [&](int i) {
    const Task& t = tasks[i];
    if (pool_mode != 2 && cudaEventSynchronize(st.stage_ev[t.part]) != cudaSuccess) {
      copy_err.store(1);
      return;
    }
    const Part& q = parts[t.part];
    const uint8_t* from = stage + ((q.mat == 1 && dcu) ? mat_bytes : 0) + t.r0 * row_bytes;
    uint8_t* to = q.mat == 0 ? reinterpret_cast<uint8_t*>(o.c_units) : reinterpret_cast<uint8_t*>(o.c);
    to += static_cast<size_t>(t.r0 * o.ldc) * 4;
    if (o.ldc == ldd && ldd == cols) {
      if (nt) copy_streaming(to, from, static_cast<size_t>((t.r1 - t.r0) * cols) * 4);
      else std::memcpy(to, from, static_cast<size_t>((t.r1 - t.r0) * cols) * 4);
    } else {
      for (int64_t r = t.r0; r < t.r1; ++r, from += row_bytes, to += o.ldc * 4)
        std::memcpy(to, from, static_cast<size_t>(cols) * 4);
    }
  };
  // a few tasks run on the calling thread alone (waking the pool costs more than it saves)
  if (tasks.size() <= 2 || !pool) {
    for (int i = 0; i < static_cast<int>(tasks.size()); ++i) copy(i);
  } else {
    host_pool_run(static_cast<int>(tasks.size()), copy);
  }
  if (trace)
    std::fprintf(stderr, "[bitmm staged] %zu parts %zu tasks: enqueued %.1f resolved %.1f first part %.1f copied %.1f us\n",
                 parts.size(), tasks.size(), t_enq, t_res, t_first, us());
  if (copy_err.load()) return fail(BITMM_ERR_CUDA, std::string("staged copy: ") + cudaGetErrorString(cudaGetLastError()));
  return BITMM_OK;
}

// Small outputs take run_staged unless the destination is already pinned (then the copy
// engine writes it directly).
bool use_staged(const HostOut& o) {
  if (o.late()) return true;
  if (const char* e = std::getenv("BITMM_HOST_STAGED"); e && std::atoi(e) == 0) return false;
  return !((o.c_units && is_pinned_host(o.c_units)) || (o.c && is_pinned_host(o.c)));
}

size_t ws_half_int(int64_t m, int64_t n, int64_t k) {
  const int64_t kpad = round_up(k, TC_BK_BYTES);
  return align_up(m * kpad, 1024) + align_up(n * kpad, 1024) + 2048;
}
// Two halves: consecutive integer GEMM calls alternate, so the operand expansion of call
// i+1 (writing one half) can overlap the GEMM of call i (reading the other half).
size_t ws_bytes_int(int64_t m, int64_t n, int64_t k) { return 2 * ws_half_int(m, n, k); }

// Expanded operands A8 [m][kpad], B8 [n][kpad] in this call's half of the workspace.
void take_int_operands(Ctx& st, int64_t m, int64_t n, int64_t k, uint8_t** A8,
                       uint8_t** B8) {
  const int64_t kpad = round_up(k, TC_BK_BYTES);
  const size_t half = ws_half_int(m, n, k);
  Carve cv(static_cast<uint8_t*>(st.ws.ptr) + (st.ws_turn & 1u) * half);
  st.ws_turn ^= 1u;
  *A8 = cv.take<uint8_t>(m * kpad);
  *B8 = cv.take<uint8_t>(n * kpad);
}
// A (two parts when the residual is folded), X split, token scales, row multipliers.
size_t ws_bytes_1x32(int64_t m, int64_t n, int64_t k) {
  const int64_t kpad = round_up(k, 64);
  return align_up(m * 2 * kpad * 2, 1024) + align_up(n * APB_PARTS * kpad * 2, 1024) +
         align_up(n * 4, 1024) + align_up(m * 4, 1024) + 2048;
}

// ---------------- routine bodies on device pointers ----------------
int gemm_1x1_dev_impl(Ctx& st, const uint64_t* a, int64_t m, const uint64_t* b, int64_t n,
                      int64_t k, int64_t wpr, float gamma_a, float gamma_b, int32_t* c_units,
                      float* c, int64_t ldc, cudaStream_t s) {
  const bool fp4 = use_fp4();
  const float scale = gamma_a * gamma_b;  // kernels.cpp:170
  const OperandSrc sa{a, nullptr, nullptr, m, false}, sb{b, nullptr, nullptr, n, false};
  if (fx_enabled() && fx_operand_ok(sa, wpr) && fx_operand_ok(sb, wpr)) {
    const FxItem it = fx_item(sa, sb, k, wpr, 0, scale, nullptr, nullptr, c_units, c, ldc);
    return run_fx(st, &it, 1, s);
  }
  const int64_t kpad = kpad_for(k, fp4);
  BITMM_TRY(ws_reserve(st, ws_bytes_int(m, n, k)));
  uint8_t *A8, *B8;
  take_int_operands(st, m, n, k, &A8, &B8);
  BITMM_TRY(run_unpack_pair(sa, sb, wpr, k, kpad, A8, B8, st.status, s, fp4));
  return run_int_gemm(st, A8, B8, m, n, kpad, 0, scale, nullptr, nullptr, c_units, c, ldc, s, fp4);
}

int gemm_1x2_dev_impl(Ctx& st, const uint64_t* w, int64_t m, float gamma, const uint64_t* t,
                      const uint64_t* h, const uint64_t* mm, int64_t n, int64_t k, int64_t wpr,
                      float a_scale, int has_a_gamma, float a_gamma, const float* row_scale,
                      const float* col_scale, int32_t* c_units, float* c, int64_t ldc,
                      cudaStream_t s) {
  const bool fp4 = use_fp4();
  // kernels.cpp:193: half_scale = 0.5f * gamma * a_packed.scale * a_packed.gamma.value_or(1.0f)
  const float scale = 0.5f * gamma * a_scale * (has_a_gamma ? a_gamma : 1.0f);
  const OperandSrc sa{w, nullptr, nullptr, m, false}, sb{t, h, mm, n, true};
  if (fx_enabled() && fx_operand_ok(sa, wpr) && fx_operand_ok(sb, wpr)) {
    const FxItem it = fx_item(sa, sb, k, wpr, fp4_shift(1, 1, true), scale, row_scale, col_scale,
                              c_units, c, ldc);
    return run_fx(st, &it, 1, s);
  }
  const int64_t kpad = kpad_for(k, fp4);
  BITMM_TRY(ws_reserve(st, ws_bytes_int(m, n, k)));
  uint8_t *A8, *B8;
  take_int_operands(st, m, n, k, &A8, &B8);
  BITMM_TRY(run_unpack_pair(sa, sb, wpr, k, kpad, A8, B8, st.status, s, fp4));
  return run_int_gemm(st, A8, B8, m, n, kpad, fp4_shift(1, 1, fp4), scale, row_scale, col_scale,
                      c_units, c, ldc, s, fp4);
}

int gemm_2x2_dev_impl(Ctx& st, const uint64_t* wt, const uint64_t* wh, const uint64_t* wm,
                      int64_t m, float w_scale, int has_w_gamma, float w_gamma, const uint64_t* at,
                      const uint64_t* ah, const uint64_t* am, int64_t n, int64_t k, int64_t wpr,
                      float a_scale, int has_a_gamma, float a_gamma, const float* row_scale,
                      const float* col_scale, int32_t* c_units, float* c, int64_t ldc,
                      cudaStream_t s) {
  const bool fp4 = use_fp4();
  // kernels.cpp:232-233
  const float scale = 0.25f * w_scale * a_scale * (has_w_gamma ? w_gamma : 1.0f) *
                      (has_a_gamma ? a_gamma : 1.0f);
  const OperandSrc sa{wt, wh, wm, m, true}, sb{at, ah, am, n, true};
  if (fx_enabled() && fx_operand_ok(sa, wpr) && fx_operand_ok(sb, wpr)) {
    const FxItem it = fx_item(sa, sb, k, wpr, fp4_shift(2, 2, true), scale, row_scale, col_scale,
                              c_units, c, ldc);
    return run_fx(st, &it, 1, s);
  }
  const int64_t kpad = kpad_for(k, fp4);
  BITMM_TRY(ws_reserve(st, ws_bytes_int(m, n, k)));
  uint8_t *A8, *B8;
  take_int_operands(st, m, n, k, &A8, &B8);
  BITMM_TRY(run_unpack_pair(sa, sb, wpr, k, kpad, A8, B8, st.status, s, fp4));
  return run_int_gemm(st, A8, B8, m, n, kpad, fp4_shift(2, 2, fp4), scale, row_scale, col_scale,
                      c_units, c, ldc, s, fp4);
}

cudaLaunchAttribute pdl_attr() {
  cudaLaunchAttribute a;
  a.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a.val.programmaticStreamSerializationAllowed = 1;
  return a;
}

constexpr int kMaxDynSmem = 232448;  // 227 KB opt-in per block on sm_100

bool spmm_chunk_fits(int64_t k, int64_t rows_per_split) {
  return spmm_smem_bytes(k, static_cast<int>(rows_per_split)) <= kMaxDynSmem;
}

// ~6 waves of blocks at 2 resident blocks per SM, rows split evenly
void spmm_grid(const Ctx& st, int64_t rows, int64_t n, int* chunks, int* splits,
               int* rows_per_split) {
  *chunks = static_cast<int>((n + SPMM_TOK - 1) / SPMM_TOK);
  const int target = 6 * st.sms;  // measured: 6 waves-worth beats 4..24 (restaging vs balance)
  *splits = static_cast<int>(std::max<int64_t>(
      1, std::min<int64_t>((rows + SPMM_QUADS - 1) / SPMM_QUADS, (target + *chunks - 1) / *chunks)));
  *rows_per_split = static_cast<int>((rows + *splits - 1) / *splits);
}

bool spmm_staged(const Ctx& st, int64_t rows, int64_t k, int64_t n) {
  int chunks, splits, rps;
  spmm_grid(st, rows, n, &chunks, &splits, &rps);
  return spmm_chunk_fits(k, rps);
}

// R.X for CSR rows, X [k][ldb] fp32 (or, LEVELS, the dequantized activation planes `lv`).
// EXACT reproduces the reference rounding (kernels.cpp:347); the fp32 APB layer uses fma and
// chains into the GEMM with PDL. When the staged chunk does not fit in shared memory, LEVELS
// first dequantizes into `deq` [k][n] and both sources take the global-gather kernel.
template <bool EXACT, bool PDL_CHAIN, bool LEVELS = false, bool ACCUM = LEVELS>
int run_spmm(Ctx& st, int64_t rows, int64_t k, const uint64_t* row_ptr,
             const uint64_t* col_idx, const float* vals, const float* b, int64_t n, int64_t ldb,
             float* c, int64_t ldc, cudaStream_t s, const SpmmLevels& lv = SpmmLevels{},
             float* deq = nullptr) {
  const auto* rp = reinterpret_cast<const unsigned long long*>(row_ptr);
  const auto* ci = reinterpret_cast<const unsigned long long*>(col_idx);
  int chunks, splits, rows_per_split;
  spmm_grid(st, rows, n, &chunks, &splits, &rows_per_split);
  if (!spmm_chunk_fits(k, rows_per_split)) {
    if (LEVELS) {
      ProfScope pd("dequant_levels", s);
      dequant_levels_kernel<<<blocks_for(((k + 63) / 64) * n, 256), 256, 0, s>>>(
          lv, static_cast<int>(k), static_cast<int>(n), deq);
      BITMM_TRY(launch_check("dequant_levels_kernel"));
      b = deq;
      ldb = n;
    }
    // large K: X chunk does not fit in shared memory, gather rows from L2 instead
    const long long warps = rows * ((n + 127) / 128);
    ProfScope ps("spmm_csr_gather", s);
    spmm_csr_kernel<<<blocks_for(warps * 32, 256), 256, 0, s>>>(rows, rp, ci, vals, b, ldb,
                                                                static_cast<int>(n), c, ldc,
                                                                ACCUM ? 1 : 0);
    return launch_check("spmm_csr_kernel");
  }
  auto kern = spmm_xchunk_kernel<EXACT, PDL_CHAIN, LEVELS, ACCUM>;
  const int smem = spmm_smem_bytes(k, rows_per_split);
  BITMM_TRY(ensure_max_smem(reinterpret_cast<const void*>(kern), kMaxDynSmem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(chunks), static_cast<unsigned>(splits));
  cfg.blockDim = dim3(SPMM_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1] = {pdl_attr()};
  cfg.attrs = attr;
  cfg.numAttrs = PDL_CHAIN ? 1 : 0;
  ProfScope ps(LEVELS ? "spmm_levels_exact" : EXACT ? "spmm_xchunk_exact" : ACCUM ? "spmm_xchunk_accum" : "spmm_xchunk", s);
  BITMM_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, static_cast<int>(rows), static_cast<int>(k),
                                    static_cast<int>(n), rp, ci, vals, b, ldb, c, ldc,
                                    rows_per_split, lv));
  return launch_check("spmm_xchunk_kernel");
}

// The 2-bit layer's residual pass (spmm_levels.cuh): a persistent grid of 2 blocks per SM, each
// owning an equal share of the (64-token chunk, row) work space.
int64_t spmm_levels_work(const Ctx& st, int64_t rows, int64_t n, int* blocks) {
  const int64_t total = (n + SL_TOK - 1) / SL_TOK * rows;
  *blocks = static_cast<int>(
      std::max<int64_t>(1, std::min<int64_t>(SL_BLOCKS_PER_SM * st.sms, (total + SL_OCTETS - 1) / SL_OCTETS)));
  return (total + *blocks - 1) / *blocks;
}

bool spmm_levels_fits(const Ctx& st, int64_t rows, int64_t k, int64_t n, bool f32 = false) {
  int blocks;
  const int64_t w = spmm_levels_work(st, rows, n, &blocks);
  return w < (1 << 30) &&
         spmm_levels_smem_bytes(k, static_cast<int>(std::min<int64_t>(w, rows)), f32) <= kMaxDynSmem;
}

// x != nullptr: the standalone exact spmm_csr over the fp32 X [k][ldx] (C = R.X, no binary part).
int run_spmm_levels(Ctx& st, int64_t rows, int64_t k, const uint64_t* row_ptr, const uint64_t* col_idx,
                    const float* vals, const SpmmLevels& lv, int64_t n, float* c, int64_t ldc, cudaStream_t s,
                    const float* x = nullptr, int64_t ldx = 0) {
  int blocks;
  const int64_t w = spmm_levels_work(st, rows, n, &blocks);
  const bool f32 = x != nullptr;
  auto kern = f32 ? spmm_levels_kernel<false, true> : spmm_levels_kernel<true, false>;
  const int smem = spmm_levels_smem_bytes(k, static_cast<int>(std::min<int64_t>(w, rows)), f32);
  BITMM_TRY(ensure_max_smem(reinterpret_cast<const void*>(kern), kMaxDynSmem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(blocks));
  cfg.blockDim = dim3(SL_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1] = {pdl_attr()};
  cfg.attrs = attr;
  cfg.numAttrs = f32 ? 0 : 1;  // the layer's pass chains after its GEMM; spmm_csr stands alone
  ProfScope ps(f32 ? "spmm_f32_exact" : "spmm_levels", s);
  BITMM_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, static_cast<int>(rows), static_cast<int>(k), static_cast<int>(n),
                                    reinterpret_cast<const unsigned long long*>(row_ptr),
                                    reinterpret_cast<const unsigned long long*>(col_idx), vals, lv, c,
                                    static_cast<long long>(ldc), static_cast<long long>(w), x,
                                    static_cast<long long>(ldx)));
  return launch_check("spmm_levels_kernel");
}

int apb_dev_impl(Ctx& st, const uint64_t* w, int64_t m, int64_t k, int64_t wpr, float gamma,
                 const float* row_gamma, const float* b, int64_t n, int64_t ldb,
                 const uint64_t* row_ptr, const uint64_t* col_idx, const float* vals, float* c,
                 int64_t ldc, cudaStream_t s) {
  const int64_t kpad = round_up(k, 64);
  // layer_forward: the residual is folded into the GEMM operand (apb_fold_kernel)
  const bool fold = row_ptr != nullptr;
  const int64_t lda = fold ? 2 * kpad : kpad;
  BITMM_TRY(ws_reserve(st, ws_bytes_1x32(m, n, k)));
  Carve cv(st.ws.ptr);
  uint16_t* Ah = cv.take<uint16_t>(m * lda * 2);
  uint16_t* XT = cv.take<uint16_t>(n * APB_PARTS * kpad * 2);
  float* tok_scale = cv.take<float>(n * 4);
  float* row_mul = cv.take<float>(m * 4);
  cudaLaunchAttribute pdl[1] = {pdl_attr()};
  const int wpr32 = static_cast<int>(wpr * 2);
  if (!fold) {
    const long long total = m * std::max<long long>(kpad / 32, wpr32);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks_for(total, 256));
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cfg.attrs = pdl;
    cfg.numAttrs = 1;
    ProfScope ps("unpack_sign_f16", s);
    BITMM_CUDA_TRY(cudaLaunchKernelEx(&cfg, unpack_sign_f16, reinterpret_cast<const uint32_t*>(w),
                                      static_cast<long long>(m), wpr32, static_cast<int>(k),
                                      static_cast<int>(kpad), Ah, st.status));
    BITMM_TRY(launch_check("unpack_sign_f16"));
  }
  if (fold) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks_for(m, 8));  // a warp per row
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cfg.attrs = pdl;
    cfg.numAttrs = 1;
    ProfScope ps("apb_fold", s);
    BITMM_CUDA_TRY(cudaLaunchKernelEx(&cfg, apb_fold_kernel, reinterpret_cast<const uint32_t*>(w), wpr32,
                                      static_cast<int>(m), static_cast<int>(k), static_cast<int>(kpad),
                                      static_cast<long long>(lda),
                                      reinterpret_cast<const unsigned long long*>(row_ptr),
                                      reinterpret_cast<const unsigned long long*>(col_idx), vals, gamma,
                                      row_gamma, Ah, row_mul, st.status));
    BITMM_TRY(launch_check("apb_fold_kernel"));
  }
  const int strip_smem = static_cast<int>(kpad * 32 * 4);
  if (strip_smem <= 112 * 1024) {
    // one pass: a block stages a 32-token strip of X, takes the token maxima and splits
    BITMM_TRY(ensure_max_smem(reinterpret_cast<const void*>(split_x_f16_strip), 112 * 1024));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>((n + 31) / 32));
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = strip_smem;
    cfg.stream = s;
    cfg.attrs = pdl;
    cfg.numAttrs = 1;
    ProfScope ps("split_x_f16_strip", s);
    BITMM_CUDA_TRY(cudaLaunchKernelEx(&cfg, split_x_f16_strip, b, static_cast<long long>(ldb),
                                      static_cast<int>(k), static_cast<int>(n),
                                      static_cast<int>(kpad), tok_scale, XT));
    BITMM_TRY(launch_check("split_x_f16_strip"));
  } else {
    {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(static_cast<unsigned>((n + 31) / 32));
      cfg.blockDim = dim3(1024);
      cfg.stream = s;
      cfg.attrs = pdl;
      cfg.numAttrs = 1;
      ProfScope ps("x_token_scale", s);
      BITMM_CUDA_TRY(cudaLaunchKernelEx(&cfg, x_token_scale, b, static_cast<long long>(ldb),
                                        static_cast<int>(k), static_cast<int>(n), tok_scale));
      BITMM_TRY(launch_check("x_token_scale"));
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(kpad / 64), static_cast<unsigned>((n + 31) / 32));
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cfg.attrs = pdl;
    cfg.numAttrs = 1;
    ProfScope ps("split_x_f16", s);
    BITMM_CUDA_TRY(cudaLaunchKernelEx(&cfg, split_x_f16, b, static_cast<long long>(ldb),
                                      static_cast<int>(k), static_cast<int>(n),
                                      static_cast<int>(kpad), static_cast<const float*>(tok_scale), XT));
    BITMM_TRY(launch_check("split_x_f16"));
  }

  // folded layer: 256-wide tiles with one accumulator per tile (default; config 4 103 vs 120 us,
  // 1.5e-6 vs 2.4e-7 relative error, tolerance 1e-5); BITMM_APB_WIDE=0 keeps 128-wide tiles with
  // the hi and lo products in separate accumulators (the most accurate)
  const char* fold_env = std::getenv("BITMM_APB_FOLD");
  const bool fold_sep = fold_env && std::string(fold_env) == "sep";
  const bool ap2 = fold && !fold_sep;
  const char* wide_env = std::getenv("BITMM_APB_WIDE");
  const bool wide = ap2 && !(wide_env && std::atoi(wide_env) == 0);
  const int bn = wide ? 256 : APB_BN;
  CUtensorMap ta, tb;
  BITMM_TRY(make_operand_map(&ta, Ah, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, lda, m, 128));
  BITMM_TRY(make_operand_map(&tb, XT, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, APB_PARTS * kpad, n, bn / 2));
  ApbParams p{};
  p.M = static_cast<int>(m);
  p.N = static_cast<int>(n);
  p.kb_per_part = static_cast<int>(kpad / 64);
  p.kpad = static_cast<int>(kpad);
  // folded residual: W'_lo rides in the same stages as W'_hi (AP = 2) unless
  // BITMM_APB_FOLD=sep selects the separate fold phase after the main K loop (A/B runs)
  p.fold_kb = (fold && fold_sep) ? p.kb_per_part : 0;
  p.alpha = gamma;
  p.row_alpha = fold ? row_mul : row_gamma;
  p.tok_scale = tok_scale;
  p.C = c;
  p.ldc = ldc;
  p.num_m_blocks = static_cast<int>((m + 255) / 256);
  p.num_n_blocks = static_cast<int>((n + bn - 1) / bn);
  p.num_tiles = p.num_m_blocks * p.num_n_blocks;
  const void* kern = wide ? reinterpret_cast<const void*>(apb_gemm_kernel<2, 256>)
                     : ap2  ? reinterpret_cast<const void*>(apb_gemm_kernel<2>)
                            : reinterpret_cast<const void*>(apb_gemm_kernel<1>);
  const int smem = wide ? ApbCfg<2, 256>::SMEM : ap2 ? ApbCfg<2>::SMEM : ApbCfg<1>::SMEM;
  BITMM_TRY(ensure_max_smem(kern, smem));
  const int units = std::min(p.num_tiles, st.sms / 2);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(2 * units));
  cfg.blockDim = dim3(TC_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1] = pdl_attr();
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  {
    ProfScope ps("apb_gemm_f16x2", s);
    if (wide) BITMM_CUDA_TRY(cudaLaunchKernelEx(&cfg, apb_gemm_kernel<2, 256>, ta, tb, p));
    else if (ap2) BITMM_CUDA_TRY(cudaLaunchKernelEx(&cfg, apb_gemm_kernel<2>, ta, tb, p));
    else BITMM_CUDA_TRY(cudaLaunchKernelEx(&cfg, apb_gemm_kernel<1>, ta, tb, p));
    BITMM_TRY(launch_check("apb_gemm_kernel"));
  }
  return BITMM_OK;
}

// Paper-faithful APB with 2-bit activations:
//   C = gemm_1x2(bin, alpha_r, planes)  +  spmm_csr(residual, dequant(planes))
// 1. unpack_pair : sign(bin) and the levels p to int8 (as gemm_1x2)
// 2. tc_gemm F32R (store): C = (((0.5 * alpha_r) * s) * gamma_a) * units (kernels.cpp:193,216)
// 3. spmm_levels : residual rows over the planes dequantized while staging, d_p =
//                  float(p) * (s * gamma_a), reference rounding, then C = C + R.D (apb.cpp:161)
// The GEMM stores without reading C (its epilogue warps are few and latency-bound on loads);
// the SpMM's many warps absorb the read-modify-write. Bit-identical to the reference
// composition.
size_t ws_bytes_apb2(const Ctx& st, int64_t rows, int64_t cols, int64_t tokens) {
  const size_t deq = spmm_staged(st, rows, cols, tokens) ? 0 : align_up(cols * tokens * 4, 1024);
  return ws_bytes_int(rows, tokens, cols) + deq;
}

// The fused form (apb2_fused.cuh): expansion of the GEMM operands, then one kernel computing
// C = G + S and writing C once. Taken for FP4 operands, a K whose level chunk fits in shared
// memory beside the pipeline, and an output the epilogue's TMA stores can write;
// BITMM_APB2_FUSED=0 selects the two-pass form below.
bool apb2_fused_ok(int64_t cols, int64_t tokens, const float* c, int64_t ldc) {
  const char* e = std::getenv("BITMM_APB2_FUSED");
  if (e && std::atoi(e) == 0) return false;
  return use_fp4() && !fx_enabled() && apb2_fused_smem_bytes(cols) <= kMaxDynSmem && (tokens & 3) == 0 &&
         (ldc & 3) == 0 && (reinterpret_cast<uintptr_t>(c) & 15) == 0 && !is_peer_memory(c);
}

int apb2_fused_impl(Ctx& st, int64_t rows, int64_t cols, int64_t wpr, float alpha, const float* row_alpha,
                    const uint64_t* bin, const uint64_t* row_ptr, const uint64_t* col_idx, const float* vals,
                    const uint64_t* t, const uint64_t* h, const uint64_t* m, int64_t tokens, float a_scale,
                    float a_gamma, float* c, int64_t ldc, cudaStream_t s) {
  const int64_t kpad = kpad_for(cols, true);
  const int64_t chunks = (tokens + SL_TOK - 1) / SL_TOK;
  const size_t lc_bytes = static_cast<size_t>(chunks) * (cols + 1) * SL_ROW_WORDS * 4;
  BITMM_TRY(ws_reserve(st, ws_bytes_int(rows, tokens, cols) + align_up(lc_bytes, 1024)));
  unsigned* LC = reinterpret_cast<unsigned*>(static_cast<uint8_t*>(st.ws.ptr) + ws_bytes_int(rows, tokens, cols));
  const OperandSrc sa{bin, nullptr, nullptr, rows, false}, sb{t, h, m, tokens, true};
  uint8_t *A8 = nullptr, *B8 = nullptr;
  take_int_operands(st, rows, tokens, cols, &A8, &B8);
  SpmmLevels lv{};
  lv.t = reinterpret_cast<const unsigned long long*>(t);
  lv.h = reinterpret_cast<const unsigned long long*>(h);
  lv.m = reinterpret_cast<const unsigned long long*>(m);
  lv.wpr = static_cast<int>(wpr);
  const float sg = a_scale * a_gamma;  // the dequantized levels, as the two-pass form stages them
  lv.d1 = 1.0f * sg;
  lv.d2 = 2.0f * sg;
  lv.d3 = 3.0f * sg;
  lv.neg_zero = -0.0f;
  // L8 level chunks (levels.cuh) unless BITMM_APB2_L8=0 or -4 sg is not a finite exact addend
  const bool l8_env = !(std::getenv("BITMM_APB2_L8") && std::atoi(std::getenv("BITMM_APB2_L8")) == 0);
  const bool l8 = l8_env && std::isfinite(4.0f * sg);
  // the level chunks are staged by the expansion launch, in a grid row of their own
  const LevelChunkJob lc{lv, static_cast<int>(cols), static_cast<int>(tokens), static_cast<int>(chunks), LC,
                         l8 ? 1 : 0};
  BITMM_TRY(run_unpack_pair(sa, sb, wpr, cols, kpad, A8, B8, st.status, s, true, &lc));
  CUtensorMap ta, tb, tc;
  const int64_t rb = kpad / 2;
  BITMM_TRY(make_operand_map(&ta, A8, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, rb, rows, 128));
  BITMM_TRY(make_operand_map(&tb, B8, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, rb, tokens, A3_BN / 2));
  if (!make_output_map(&tc, c, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, tokens, rows, ldc))
    return fail(BITMM_ERR_CUDA, "fused APB: output map");
  Apb2Params ap{};
  TcParams& p = ap.p;
  p.M = static_cast<int>(rows);
  p.N = static_cast<int>(tokens);
  p.num_kb = static_cast<int>(rb / TC_BK_BYTES);
  p.shift = fp4_shift(1, 1, true);
  p.shift_mul = static_cast<float>(1 << p.shift);
  p.scale = 0.5f * alpha * a_scale * a_gamma;  // kernels.cpp:193 order
  p.row_scale = row_alpha;
  p.row_pre = 0.5f;
  p.act_scale = a_scale;
  p.act_gamma = a_gamma;
  p.out_f32 = c;
  p.ldc = ldc;
  p.epi = static_cast<int>(Epi::F32R);
  p.tma_store = 1;
  p.num_m_blocks = static_cast<int>((rows + 255) / 256);
  p.num_n_blocks = static_cast<int>((tokens + A3_BN - 1) / A3_BN);
  p.num_tiles = p.num_m_blocks * p.num_n_blocks;
  ap.row_ptr = reinterpret_cast<const unsigned long long*>(row_ptr);
  ap.col_idx = reinterpret_cast<const unsigned long long*>(col_idx);
  ap.vals = vals;
  ap.lv = lv;
  ap.level_chunks = LC;
  ap.K = static_cast<int>(cols);
  ap.neg4sg = -4.0f * lv.d1;  // exact (a power-of-two multiple, finite when l8)
  const int smem = apb2_fused_smem_bytes(cols);
  auto kern = l8 ? apb2_fused_kernel<true> : apb2_fused_kernel<false>;
  // the opt-in limit is one value per kernel: set the maximum once (a per-size value would be
  // overwritten by a smaller K's launch and reject a later larger one)
  BITMM_TRY(ensure_max_smem(reinterpret_cast<const void*>(kern), kMaxDynSmem));
  const int units = std::max(1, std::min(p.num_tiles, st.sms / 2));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(2 * units));
  cfg.blockDim = dim3(A3_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  ProfScope ps("apb2_fused", s);
  BITMM_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, ta, tb, tc, ap));
  return launch_check("apb2_fused_kernel");
}

int apb2_dev_impl(Ctx& st, int64_t rows, int64_t cols, int64_t wpr, float alpha,
                  const float* row_alpha, const uint64_t* bin, const uint64_t* row_ptr,
                  const uint64_t* col_idx, const float* vals, const uint64_t* t, const uint64_t* h,
                  const uint64_t* m, int64_t tokens, float a_scale, float a_gamma, float* c,
                  int64_t ldc, cudaStream_t s) {
  if (apb2_fused_ok(cols, tokens, c, ldc))
    return apb2_fused_impl(st, rows, cols, wpr, alpha, row_alpha, bin, row_ptr, col_idx, vals, t, h, m, tokens,
                           a_scale, a_gamma, c, ldc, s);
  const bool fp4 = use_fp4();
  const int64_t kpad = kpad_for(cols, fp4);
  BITMM_TRY(ws_reserve(st, ws_bytes_apb2(st, rows, cols, tokens)));
  float* deq = reinterpret_cast<float*>(static_cast<uint8_t*>(st.ws.ptr) + ws_bytes_int(rows, tokens, cols));
  const OperandSrc sa{bin, nullptr, nullptr, rows, false}, sb{t, h, m, tokens, true};
  const bool fx = fx_enabled() && fx_operand_ok(sa, wpr) && fx_operand_ok(sb, wpr);
  uint8_t *A8 = nullptr, *B8 = nullptr;
  if (!fx) {
    take_int_operands(st, rows, tokens, cols, &A8, &B8);
    BITMM_TRY(run_unpack_pair(sa, sb, wpr, cols, kpad, A8, B8, st.status, s, fp4));
  }
  GemmProblem q{A8, B8, rows, tokens, kpad, TcParams{}};
  q.p.shift = fp4_shift(1, 1, fp4);
  q.p.scale = 0.5f * alpha * a_scale * a_gamma;  // kernels.cpp:193 order
  q.p.row_scale = row_alpha;
  q.p.row_pre = 0.5f;
  q.p.act_scale = a_scale;
  q.p.act_gamma = a_gamma;
  q.p.out_f32 = c;
  q.p.ldc = ldc;
  q.p.epi = static_cast<int>(Epi::F32R);
  if (fx) {
    FxItem it = fx_item(sa, sb, cols, wpr, q.p.shift, q.p.scale, row_alpha, nullptr, nullptr, c, ldc);
    it.f32r = true;
    it.row_pre = q.p.row_pre;
    it.act_scale = a_scale;
    it.act_gamma = a_gamma;
    BITMM_TRY(run_fx(st, &it, 1, s));
  } else {
    BITMM_TRY(run_problems(st, &q, 1, fp4, s));
  }
  SpmmLevels lv{};
  lv.t = reinterpret_cast<const unsigned long long*>(t);
  lv.h = reinterpret_cast<const unsigned long long*>(h);
  lv.m = reinterpret_cast<const unsigned long long*>(m);
  lv.wpr = static_cast<int>(wpr);
  const float sg = a_scale * a_gamma;
  lv.d1 = 1.0f * sg;
  lv.d2 = 2.0f * sg;
  lv.d3 = 3.0f * sg;
  lv.neg_zero = -0.0f;
  const char* v1 = std::getenv("BITMM_SPMM_LEVELS_V1");  // A/B: the fp32-staged form
  if (!(v1 && std::atoi(v1) != 0) && spmm_levels_fits(st, rows, cols, tokens))
    return run_spmm_levels(st, rows, cols, row_ptr, col_idx, vals, lv, tokens, c, ldc, s);
  return run_spmm<true, true, true>(st, rows, cols, row_ptr, col_idx, vals, nullptr, tokens, tokens,
                                    c, ldc, s, lv, deq);
}

int check_csr_host(int64_t rows, int64_t cols, const uint64_t* row_ptr, const uint64_t* col_idx,
                   const float* vals, int64_t nnz) {
  // CsrMatrix::validate (tensor.cpp:104-123)
  if (rows < 0 || cols < 0) return fail(BITMM_ERR_INVALID_ARGUMENT, "matrix dimensions must be non-negative");
  if (row_ptr[0] != 0) return fail(BITMM_ERR_INVALID_ARGUMENT, "csr row_ptr must start at 0");
  for (int64_t r = 0; r < rows; ++r)
    if (row_ptr[r] > row_ptr[r + 1]) return fail(BITMM_ERR_INVALID_ARGUMENT, "csr row_ptr must be monotone");
  if (static_cast<int64_t>(row_ptr[rows]) != nnz) return fail(BITMM_ERR_INVALID_ARGUMENT, "csr payload sizes must match nnz");
  for (int64_t r = 0; r < rows; ++r)
    for (uint64_t i = row_ptr[r]; i < row_ptr[r + 1]; ++i) {
      if (col_idx[i] >= static_cast<uint64_t>(cols)) return fail(BITMM_ERR_INVALID_ARGUMENT, "csr column index out of range");
      if (i > row_ptr[r] && col_idx[i - 1] >= col_idx[i])
        return fail(BITMM_ERR_INVALID_ARGUMENT, "csr column indices must be strictly increasing per row");
    }
  (void)vals;
  return BITMM_OK;
}

}  // namespace

// =========================== exported ABI ===========================
extern "C" {

int bitmm_abi_version(void) { return 1; }

#ifdef A3_STATS
// Profiling builds only (-DA3_STATS): the fused 2-bit APB layer's counters of the last launch.
int bitmm_debug_a3_stats(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, a3_stats, sizeof(a3_stats)) == cudaSuccess ? 0 : 3;
}
#endif
#ifdef FX_STATS
// Profiling builds only (-DFX_STATS): the fx_gemm wait counters of the last launch.
int bitmm_debug_fx_stats(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, fx_stats, sizeof(fx_stats)) == cudaSuccess ? 0 : 3;
}
#endif

const char* bitmm_last_error(void) { return g_err.c_str(); }

int bitmm_last_launch_count(void) { return g_launches; }
uint64_t bitmm_last_d2h_bytes(void) { return g_d2h_bytes; }

int bitmm_profile_enable(int on) {
  std::lock_guard<std::mutex> lk(g_prof.mu);
  g_prof.on = on != 0;
  return BITMM_OK;
}

int bitmm_profile_collect(void) {
  std::lock_guard<std::mutex> lk(g_prof.mu);
  for (const ProfRecord& r : g_prof.pending) {
    BITMM_CUDA_TRY(cudaEventSynchronize(r.e1));
    float ms = 0.f;
    BITMM_CUDA_TRY(cudaEventElapsedTime(&ms, r.e0, r.e1));
    g_prof.ms[r.kernel] += ms;
    g_prof.launches[r.kernel] += 1;
    g_prof.pool.push_back(r.e0);
    g_prof.pool.push_back(r.e1);
  }
  g_prof.pending.clear();
  return BITMM_OK;
}

int bitmm_profile_reset(void) {
  BITMM_TRY(bitmm_profile_collect());
  std::lock_guard<std::mutex> lk(g_prof.mu);
  g_prof.names.clear();
  g_prof.launches.clear();
  g_prof.ms.clear();
  return BITMM_OK;
}

int bitmm_profile_kernel_count(void) { return static_cast<int>(g_prof.names.size()); }

const char* bitmm_profile_kernel_name(int i) {
  return (i >= 0 && i < static_cast<int>(g_prof.names.size())) ? g_prof.names[i].c_str() : "";
}

int bitmm_profile_kernel_launches(int i) {
  return (i >= 0 && i < static_cast<int>(g_prof.launches.size())) ? g_prof.launches[i] : 0;
}

double bitmm_profile_kernel_ms(int i) {
  return (i >= 0 && i < static_cast<int>(g_prof.ms.size())) ? g_prof.ms[i] : 0.0;
}

// ---------------- CUDA IPC (multi-GPU gather into the root's output) ----------------
int bitmm_ipc_get_handle(const void* dev_ptr, void* handle, uint64_t* offset) {
  if (!dev_ptr || !handle || !offset) return fail(BITMM_ERR_INVALID_ARGUMENT, "null argument");
  PFN_addrRange_t range = addr_range_fn();
  if (!range) return fail(BITMM_ERR_CUDA, "cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
    return fail(BITMM_ERR_CUDA, "cuMemGetAddressRange failed (not a device allocation?)");
  cudaIpcMemHandle_t h;
  BITMM_CUDA_TRY(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  static_assert(sizeof(h) == 64, "CUDA IPC handles are 64 bytes");
  memcpy(handle, &h, sizeof(h));
  *offset = reinterpret_cast<uint64_t>(dev_ptr) - static_cast<uint64_t>(base);
  return BITMM_OK;
}

int bitmm_ipc_open(const void* handle, void** dev_ptr) {
  if (!handle || !dev_ptr) return fail(BITMM_ERR_INVALID_ARGUMENT, "null argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  BITMM_CUDA_TRY(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return BITMM_OK;
}

int bitmm_ipc_close(void* dev_ptr) {
  BITMM_CUDA_TRY(cudaIpcCloseMemHandle(dev_ptr));
  return BITMM_OK;
}

int bitmm_device_sm_count(void) {
  Dev* d = nullptr;
  int dev = 0;
  if (current_dev(&d, &dev) != BITMM_OK) return 0;
  return d->sms;
}

int bitmm_device_status(void* stream) {
  CallCtx st;
  BITMM_TRY(st.acquire(static_cast<cudaStream_t>(stream)));
  return read_status(*st, static_cast<cudaStream_t>(stream));
}

int bitmm_reserve_workspace(size_t bytes) {
  CallCtx st;  // the legacy default stream's workspace (where a caller without streams runs)
  BITMM_TRY(st.acquire(nullptr));
  return ws_reserve(*st, bytes);
}

size_t bitmm_workspace_bytes(int routine, int64_t m, int64_t n, int64_t k) {
  if (m <= 0 || n <= 0 || k <= 0) return 0;
  if (routine == 3) return ws_bytes_1x32(m, n, k);
  if (routine == 4)  // dequantized [k][n] operand only when the staged SpMM chunk cannot fit
    return ws_bytes_int(m, n, k) + (spmm_chunk_fits(k, m) ? 0 : align_up(k * n * 4, 1024));
  return ws_bytes_int(m, n, k);
}

// ---------------- 1/1 ----------------
int bitmm_gemm_1x1_dev(const uint64_t* a, int64_t m, const uint64_t* b_packed, int64_t n, int64_t k,
                       int64_t wpr, float gamma_a, float gamma_b, int32_t* c_units, float* c,
                       int64_t ldc, void* stream) {
  g_launches = 0;
  BITMM_TRY(check_gemm_dims(m, n, k, wpr, ldc));
  if (!a || !b_packed || (!c_units && !c)) return fail(BITMM_ERR_INVALID_ARGUMENT, "null operand");
  CallCtx st;
  BITMM_TRY(st.acquire(static_cast<cudaStream_t>(stream)));
  return gemm_1x1_dev_impl(*st, a, m, b_packed, n, k, wpr, gamma_a, gamma_b, c_units, c, ldc,
                           static_cast<cudaStream_t>(stream));
}

int bitmm_gemm_1x1_popc_dev(const uint64_t* a, int64_t m, const uint64_t* b_packed, int64_t n,
                            int64_t k, int64_t wpr, float gamma_a, float gamma_b,
                            int32_t* c_units, float* c, int64_t ldc, void* stream) {
  g_launches = 0;
  BITMM_TRY(check_gemm_dims(m, n, k, wpr, ldc));
  if (!a || !b_packed || (!c_units && !c)) return fail(BITMM_ERR_INVALID_ARGUMENT, "null operand");
  CallCtx st;
  BITMM_TRY(st.acquire(static_cast<cudaStream_t>(stream)));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  dim3 grid(static_cast<unsigned>((n + PC_BN - 1) / PC_BN), static_cast<unsigned>((m + PC_BM - 1) / PC_BM));
  const float scale = gamma_a * gamma_b;
  const auto* A = reinterpret_cast<const uint32_t*>(a);
  const auto* B = reinterpret_cast<const uint32_t*>(b_packed);
  if (c_units) {
    ProfScope ps("popc_gemm_1x1", s);
    popc_gemm_1x1<false><<<grid, PC_THREADS, 0, s>>>(A, B, (int)m, (int)n, (int)k, (int)(wpr * 2), scale,
                                                     c_units, nullptr, ldc);
    BITMM_TRY(launch_check("popc_gemm_1x1"));
  }
  if (c) {
    ProfScope ps("popc_gemm_1x1", s);
    popc_gemm_1x1<true><<<grid, PC_THREADS, 0, s>>>(A, B, (int)m, (int)n, (int)k, (int)(wpr * 2), scale,
                                                    nullptr, c, ldc);
    BITMM_TRY(launch_check("popc_gemm_1x1"));
  }
  return BITMM_OK;
}

}  // extern "C"

namespace {

// A late destination of an output that is sliced (>= kPipeMinOutBytes) or sent on the 16-bit
// wire is resolved before anything is enqueued; smaller ones go through run_staged. Returns the
// device leading dimension of the output.
int prepare_out(HostOut& o, int routine, int64_t m, int64_t n, int64_t k, int64_t* ldd) {
  // BITMM_LATE_EAGER=1: resolve every late destination up front (A/B of the overlap)
  static const bool eager = std::getenv("BITMM_LATE_EAGER") && std::atoi(std::getenv("BITMM_LATE_EAGER")) == 1;
  const size_t bytes = static_cast<size_t>(m * n) * 4;
  if (o.late() && (eager || bytes >= kPipeMinOutBytes || host_wire(routine, k, bytes) != Wire::None))
    BITMM_TRY(o.resolve(n));
  *ldd = o.late() ? n : o.ldc;
  return BITMM_OK;
}

int gemm_1x1_host_impl(const uint64_t* a, int64_t m, const uint64_t* b_packed, int64_t n, int64_t k,
                       int64_t wpr, float gamma_a, float gamma_b, HostOut& o) {
  if (!g_batch) g_launches = 0;
  BITMM_TRY(check_gemm_dims(m, n, k, wpr, o.late() ? n : o.ldc));
  if (!a || !b_packed || (!o.want_units && !o.want_c)) return fail(BITMM_ERR_INVALID_ARGUMENT, "null operand");
  HostLease hl;
  BITMM_TRY(hl.acquire());
  Ctx* st = &hl.ctx();
  cudaStream_t s = hl->stream;
  if (!g_batch) g_d2h_bytes = 0;
  int64_t ldc = 0;
  BITMM_TRY(prepare_out(o, 0, m, n, k, &ldc));
  int32_t* c_units = o.c_units;
  float* c = o.c;
  const bool want_units = o.want_units, want_c = o.want_c;
  const Wire wire = host_wire(0, k, static_cast<size_t>(m * ldc * 4));
  const size_t a_bytes = m * wpr * 8, b_bytes = n * wpr * 8, c_bytes = m * ldc * 4;
  const size_t w_bytes = wire != Wire::None ? static_cast<size_t>(m * n) * 2 : 0;
  void* io = nullptr;
  BITMM_TRY(io_take(hl.host(), s, align_up(a_bytes, 1024) + align_up(b_bytes, 1024) +
                                      2 * align_up(c_bytes, 1024) + align_up(w_bytes, 1024), &io));
  Carve cv(io);
  uint64_t* da = cv.take<uint64_t>(a_bytes);
  uint64_t* db = cv.take<uint64_t>(b_bytes);
  // 16-bit wire: the GEMM writes int32 units only; the host derives both outputs from them
  int32_t* dcu = (want_units || wire != Wire::None) ? cv.take<int32_t>(c_bytes) : nullptr;
  float* dc = (want_c && wire == Wire::None) ? cv.take<float>(c_bytes) : nullptr;
  BITMM_CUDA_TRY(cudaMemcpyAsync(db, b_packed, b_bytes, cudaMemcpyHostToDevice, s));
  // slices of output rows (rows of a)
  auto in = [=](int64_t r0, int64_t r1, cudaStream_t cs) -> int {
    BITMM_CUDA_TRY(cudaMemcpyAsync(da + r0 * wpr, a + r0 * wpr, (r1 - r0) * wpr * 8,
                                   cudaMemcpyHostToDevice, cs));
    return BITMM_OK;
  };
  auto gemm = [=](int64_t r0, int64_t r1) -> int {
    return gemm_1x1_dev_impl(*st, da + r0 * wpr, r1 - r0, db, n, k, wpr, gamma_a, gamma_b,
                             dcu ? dcu + r0 * ldc : nullptr, dc ? dc + r0 * ldc : nullptr, ldc, s);
  };
  auto body = [&](int64_t r0, int64_t r1) -> int {
    BITMM_TRY(in(r0, r1, s));
    return gemm(r0, r1);
  };
  if (wire != Wire::None) {
    const WireOut wo{wire, static_cast<int>(k), gamma_a * gamma_b /* kernels.cpp:170 */, nullptr,
                     nullptr, c_units, c, ldc};
    return run_or_defer_wire(hl.host(), s,
                             WireItem{m, pipe_step(m, c_bytes, 256), in, gemm,
                                      [=](int64_t r0, int64_t r1) { return OutBlock{r0, r1 - r0, 0, n}; },
                                      wo, dcu, cv.take<uint16_t>(w_bytes), static_cast<size_t>(m * n)});
  }
  if (pipe_step(m, c_bytes, 256) >= m && use_staged(o)) {
    BITMM_TRY(body(0, m));
    return run_staged(hl.host(), s, m, n, ldc, dcu, dc, o);
  }
  BITMM_TRY(run_pipelined(
      hl.host(), s, m, pipe_step(m, c_bytes, 256), body,
      [&](int64_t r0, int64_t r1, cudaStream_t d2h) -> int {
        // rows of n cells: the caller's columns [n, ldc) are not the output's
        const size_t pitch = ldc * 4, width = n * 4;
        if (dcu) BITMM_CUDA_TRY(cudaMemcpy2DAsync(c_units + r0 * ldc, pitch, dcu + r0 * ldc, pitch, width, r1 - r0, cudaMemcpyDeviceToHost, d2h));
        if (dc) BITMM_CUDA_TRY(cudaMemcpy2DAsync(c + r0 * ldc, pitch, dc + r0 * ldc, pitch, width, r1 - r0, cudaMemcpyDeviceToHost, d2h));
        g_d2h_bytes += ((dcu ? 1 : 0) + (dc ? 1 : 0)) * width * (r1 - r0);
        return BITMM_OK;
      }));
  return read_status_host(hl.host(), s);
}

}  // namespace

extern "C" {

int bitmm_gemm_1x1_host(const uint64_t* a, int64_t m, const uint64_t* b_packed, int64_t n,
                        int64_t k, int64_t wpr, float gamma_a, float gamma_b, int32_t* c_units,
                        float* c, int64_t ldc) {
  HostOut o = HostOut::given(c_units, c, ldc);
  return gemm_1x1_host_impl(a, m, b_packed, n, k, wpr, gamma_a, gamma_b, o);
}

// ---------------- 1/2 ----------------
int bitmm_gemm_1x2_dev(const uint64_t* w, int64_t m, float gamma, const uint64_t* t,
                       const uint64_t* h, const uint64_t* mm, int64_t n, int64_t k, int64_t wpr,
                       float a_scale, int has_a_gamma, float a_gamma, const float* row_scale,
                       const float* col_scale, int32_t* c_units, float* c, int64_t ldc,
                       void* stream) {
  g_launches = 0;
  if (!(a_scale > 0.0f)) return fail(BITMM_ERR_INVALID_ENCODING, "plane scale must be positive");
  BITMM_TRY(check_gemm_dims(m, n, k, wpr, ldc));
  if (!w || !t || !h || !mm || (!c_units && !c)) return fail(BITMM_ERR_INVALID_ARGUMENT, "null operand");
  CallCtx st;
  BITMM_TRY(st.acquire(static_cast<cudaStream_t>(stream)));
  return gemm_1x2_dev_impl(*st, w, m, gamma, t, h, mm, n, k, wpr, a_scale, has_a_gamma, a_gamma,
                           row_scale, col_scale, c_units, c, ldc, static_cast<cudaStream_t>(stream));
}

}  // extern "C"

namespace {

int gemm_1x2_host_impl(const uint64_t* w, int64_t m, float gamma, const uint64_t* t, const uint64_t* h,
                       const uint64_t* mm, int64_t n, int64_t k, int64_t wpr, float a_scale, int has_a_gamma,
                       float a_gamma, const float* row_scale, const float* col_scale, HostOut& o) {
  if (!g_batch) g_launches = 0;
  // ThmPlanes::validate runs first in the reference (kernels.cpp:186): scale, then legality.
  if (!(a_scale > 0.0f)) return fail(BITMM_ERR_INVALID_ENCODING, "plane scale must be positive");
  if (!t || !h || !mm || !w || (!o.want_units && !o.want_c)) return fail(BITMM_ERR_INVALID_ARGUMENT, "null operand");
  HostLease hl;
  BITMM_TRY(hl.acquire());
  Ctx* st = &hl.ctx();
  cudaStream_t s = hl->stream;
  const int rc_dims = check_gemm_dims(m, n, k, wpr, o.late() ? n : o.ldc);
  const std::string dims_msg = g_err;
  int64_t ldc = 0;
  if (rc_dims == BITMM_OK) BITMM_TRY(prepare_out(o, 1, m, n, k, &ldc));
  int32_t* c_units = o.c_units;
  float* c = o.c;
  const bool want_units = o.want_units, want_c = o.want_c;
  const bool planes_ok_shape = n >= 0 && k >= 0 && wpr >= 0 && wpr * 64 >= k;
  const size_t p_bytes = (planes_ok_shape ? n * wpr * 8 : 0), w_bytes = (rc_dims == BITMM_OK ? m * wpr * 8 : 0);
  const size_t c_bytes = (rc_dims == BITMM_OK ? m * ldc * 4 : 0);
  if (!g_batch) g_d2h_bytes = 0;
  const Wire wire = host_wire(1, k, c_bytes);
  const size_t wire_bytes = (wire != Wire::None && rc_dims == BITMM_OK) ? static_cast<size_t>(m * n) * 2 : 0;
  void* io = nullptr;
  BITMM_TRY(io_take(hl.host(), s, 3 * align_up(p_bytes, 1024) + align_up(w_bytes, 1024) +
                                      2 * align_up(c_bytes, 1024) + align_up(m > 0 ? m * 4 : 0, 1024) +
                                      align_up(n > 0 ? n * 4 : 0, 1024) + align_up(wire_bytes, 1024) + 4096, &io));
  Carve cv(io);
  uint64_t* dt = cv.take<uint64_t>(p_bytes);
  uint64_t* dh = cv.take<uint64_t>(p_bytes);
  uint64_t* dm = cv.take<uint64_t>(p_bytes);
  if (rc_dims != BITMM_OK) {
    if (p_bytes) {
      BITMM_CUDA_TRY(cudaMemcpyAsync(dt, t, p_bytes, cudaMemcpyHostToDevice, s));
      BITMM_CUDA_TRY(cudaMemcpyAsync(dh, h, p_bytes, cudaMemcpyHostToDevice, s));
      BITMM_CUDA_TRY(cudaMemcpyAsync(dm, mm, p_bytes, cudaMemcpyHostToDevice, s));
    }
    // plane legality still wins over shape errors (reference precedence)
    if (planes_ok_shape && n > 0 && k > 0) {
      const int64_t kpad = round_up(k, TC_BK_BYTES);
      BITMM_TRY(ws_reserve(*st, align_up(n * kpad, 1024) + 1024));
      BITMM_TRY(run_unpack_level_i8(dt, dh, dm, n, wpr, k, kpad, static_cast<uint8_t*>(st->ws.ptr), st->status, s));
      BITMM_TRY(read_status_host(hl.host(), s));
    }
    return fail(rc_dims, dims_msg);
  }
  uint64_t* dw = cv.take<uint64_t>(w_bytes);
  // 16-bit wire: the GEMM writes int32 units only and the host applies the scales
  float* drs = (row_scale && wire == Wire::None) ? cv.take<float>(m * 4) : nullptr;
  float* dcs = (col_scale && wire == Wire::None) ? cv.take<float>(n * 4) : nullptr;
  int32_t* dcu = (want_units || wire != Wire::None) ? cv.take<int32_t>(c_bytes) : nullptr;
  float* dc = (want_c && wire == Wire::None) ? cv.take<float>(c_bytes) : nullptr;
  BITMM_CUDA_TRY(cudaMemcpyAsync(dw, w, w_bytes, cudaMemcpyHostToDevice, s));
  if (drs) BITMM_CUDA_TRY(cudaMemcpyAsync(drs, row_scale, m * 4, cudaMemcpyHostToDevice, s));
  if (dcs) BITMM_CUDA_TRY(cudaMemcpyAsync(dcs, col_scale, n * 4, cudaMemcpyHostToDevice, s));
  // slices of output columns (rows of the activation planes, the larger operand here);
  // each slice's output block is a strided 2-D copy
  auto in = [=](int64_t n0, int64_t n1, cudaStream_t cs) -> int {
    const size_t off = n0 * wpr, bytes = (n1 - n0) * wpr * 8;
    BITMM_CUDA_TRY(cudaMemcpyAsync(dt + off, t + off, bytes, cudaMemcpyHostToDevice, cs));
    BITMM_CUDA_TRY(cudaMemcpyAsync(dh + off, h + off, bytes, cudaMemcpyHostToDevice, cs));
    BITMM_CUDA_TRY(cudaMemcpyAsync(dm + off, mm + off, bytes, cudaMemcpyHostToDevice, cs));
    return BITMM_OK;
  };
  auto gemm = [=](int64_t n0, int64_t n1) -> int {
    const size_t off = n0 * wpr;
    return gemm_1x2_dev_impl(*st, dw, m, gamma, dt + off, dh + off, dm + off, n1 - n0, k, wpr,
                             a_scale, has_a_gamma, a_gamma, drs, dcs ? dcs + n0 : nullptr,
                             dcu ? dcu + n0 : nullptr, dc ? dc + n0 : nullptr, ldc, s);
  };
  auto body = [&](int64_t n0, int64_t n1) -> int {
    BITMM_TRY(in(n0, n1, s));
    return gemm(n0, n1);
  };
  if (wire != Wire::None) {
    // kernels.cpp:193, the same expression gemm_1x2_dev_impl passes to the epilogue
    const float scale = 0.5f * gamma * a_scale * (has_a_gamma ? a_gamma : 1.0f);
    const WireOut wo{wire, static_cast<int>(k), scale, row_scale, col_scale, c_units, c, ldc};
    return run_or_defer_wire(hl.host(), s,
                             WireItem{n, pipe_step(n, c_bytes, 256), in, gemm,
                                      [=](int64_t n0, int64_t n1) { return OutBlock{0, m, n0, n1 - n0}; },
                                      wo, dcu, cv.take<uint16_t>(wire_bytes), static_cast<size_t>(m * n)});
  }
  if (pipe_step(n, c_bytes, 256) >= n && use_staged(o)) {
    BITMM_TRY(body(0, n));
    return run_staged(hl.host(), s, m, n, ldc, dcu, dc, o);
  }
  BITMM_TRY(run_pipelined(
      hl.host(), s, n, pipe_step(n, c_bytes, 256), body,
      [&](int64_t n0, int64_t n1, cudaStream_t d2h) -> int {
        const size_t pitch = ldc * 4, width = (n1 - n0) * 4;
        if (dcu) BITMM_CUDA_TRY(cudaMemcpy2DAsync(c_units + n0, pitch, dcu + n0, pitch, width, m, cudaMemcpyDeviceToHost, d2h));
        if (dc) BITMM_CUDA_TRY(cudaMemcpy2DAsync(c + n0, pitch, dc + n0, pitch, width, m, cudaMemcpyDeviceToHost, d2h));
        g_d2h_bytes += ((dcu ? 1 : 0) + (dc ? 1 : 0)) * width * m;
        return BITMM_OK;
      }));
  return read_status_host(hl.host(), s);
}

}  // namespace

extern "C" {

int bitmm_gemm_1x2_host(const uint64_t* w, int64_t m, float gamma, const uint64_t* t,
                        const uint64_t* h, const uint64_t* mm, int64_t n, int64_t k, int64_t wpr,
                        float a_scale, int has_a_gamma, float a_gamma, const float* row_scale,
                        const float* col_scale, int32_t* c_units, float* c, int64_t ldc) {
  HostOut o = HostOut::given(c_units, c, ldc);
  return gemm_1x2_host_impl(w, m, gamma, t, h, mm, n, k, wpr, a_scale, has_a_gamma, a_gamma, row_scale,
                            col_scale, o);
}

// ---------------- 2/2 ----------------
int bitmm_gemm_2x2_dev(const uint64_t* wt, const uint64_t* wh, const uint64_t* wm, int64_t m,
                       float w_scale, int has_w_gamma, float w_gamma, const uint64_t* at,
                       const uint64_t* ah, const uint64_t* am, int64_t n, int64_t k, int64_t wpr,
                       float a_scale, int has_a_gamma, float a_gamma, const float* row_scale,
                       const float* col_scale, int32_t* c_units, float* c, int64_t ldc,
                       void* stream) {
  g_launches = 0;
  if (!(w_scale > 0.0f) || !(a_scale > 0.0f))
    return fail(BITMM_ERR_INVALID_ENCODING, "plane scale must be positive");
  BITMM_TRY(check_gemm_dims(m, n, k, wpr, ldc));
  if (!wt || !wh || !wm || !at || !ah || !am || (!c_units && !c))
    return fail(BITMM_ERR_INVALID_ARGUMENT, "null operand");
  CallCtx st;
  BITMM_TRY(st.acquire(static_cast<cudaStream_t>(stream)));
  return gemm_2x2_dev_impl(*st, wt, wh, wm, m, w_scale, has_w_gamma, w_gamma, at, ah, am, n, k,
                           wpr, a_scale, has_a_gamma, a_gamma, row_scale, col_scale, c_units, c,
                           ldc, static_cast<cudaStream_t>(stream));
}

}  // extern "C"

namespace {

int gemm_2x2_host_impl(const uint64_t* wt, const uint64_t* wh, const uint64_t* wm, int64_t m, float w_scale,
                       int has_w_gamma, float w_gamma, const uint64_t* at, const uint64_t* ah,
                       const uint64_t* am, int64_t n, int64_t k, int64_t wpr, float a_scale, int has_a_gamma,
                       float a_gamma, const float* row_scale, const float* col_scale, HostOut& o) {
  if (!g_batch) g_launches = 0;
  // w.validate(); a_packed.validate(); then shapes (kernels.cpp:224-228)
  if (!(w_scale > 0.0f) || !(a_scale > 0.0f))
    return fail(BITMM_ERR_INVALID_ENCODING, "plane scale must be positive");
  if (!wt || !wh || !wm || !at || !ah || !am || (!o.want_units && !o.want_c))
    return fail(BITMM_ERR_INVALID_ARGUMENT, "null operand");
  HostLease hl;
  BITMM_TRY(hl.acquire());
  Ctx* st = &hl.ctx();
  cudaStream_t s = hl->stream;
  const int rc_dims = check_gemm_dims(m, n, k, wpr, o.late() ? n : o.ldc);
  const std::string dims_msg = g_err;
  int64_t ldc = 0;
  if (rc_dims == BITMM_OK) BITMM_TRY(prepare_out(o, 2, m, n, k, &ldc));
  int32_t* c_units = o.c_units;
  float* c = o.c;
  const bool want_units = o.want_units, want_c = o.want_c;
  const bool shape_ok = k >= 0 && wpr >= 0 && wpr * 64 >= k;
  const size_t pw = (shape_ok && m > 0 ? m * wpr * 8 : 0), pa = (shape_ok && n > 0 ? n * wpr * 8 : 0);
  const size_t c_bytes = (rc_dims == BITMM_OK ? m * ldc * 4 : 0);
  if (!g_batch) g_d2h_bytes = 0;
  const Wire wire = host_wire(2, k, c_bytes);
  const size_t wire_bytes = (wire != Wire::None && rc_dims == BITMM_OK) ? static_cast<size_t>(m * n) * 2 : 0;
  void* io = nullptr;
  BITMM_TRY(io_take(hl.host(), s, 3 * align_up(pw, 1024) + 3 * align_up(pa, 1024) +
                                      2 * align_up(c_bytes, 1024) + align_up(m > 0 ? m * 4 : 0, 1024) +
                                      align_up(n > 0 ? n * 4 : 0, 1024) + align_up(wire_bytes, 1024) + 4096, &io));
  Carve cv(io);
  uint64_t* d[6];
  const uint64_t* src[6] = {wt, wh, wm, at, ah, am};
  for (int i = 0; i < 6; ++i) {
    const size_t bytes = i < 3 ? pw : pa;
    d[i] = cv.take<uint64_t>(bytes);
    // the weight planes go in per slice below unless the call fails on its shapes
    if (bytes && (i >= 3 || rc_dims != BITMM_OK))
      BITMM_CUDA_TRY(cudaMemcpyAsync(d[i], src[i], bytes, cudaMemcpyHostToDevice, s));
  }
  if (rc_dims != BITMM_OK) {
    if (shape_ok && k > 0) {
      const int64_t kpad = round_up(k, TC_BK_BYTES);
      BITMM_TRY(ws_reserve(*st, align_up(std::max<int64_t>(m, n) * kpad, 1024) + 1024));
      if (m > 0) BITMM_TRY(run_unpack_level_i8(d[0], d[1], d[2], m, wpr, k, kpad, static_cast<uint8_t*>(st->ws.ptr), st->status, s));
      if (n > 0) BITMM_TRY(run_unpack_level_i8(d[3], d[4], d[5], n, wpr, k, kpad, static_cast<uint8_t*>(st->ws.ptr), st->status, s));
      BITMM_TRY(read_status_host(hl.host(), s));
    }
    return fail(rc_dims, dims_msg);
  }
  // 16-bit wire: the GEMM writes int32 units only and the host applies the scales
  float* drs = (row_scale && wire == Wire::None) ? cv.take<float>(m * 4) : nullptr;
  float* dcs = (col_scale && wire == Wire::None) ? cv.take<float>(n * 4) : nullptr;
  int32_t* dcu = (want_units || wire != Wire::None) ? cv.take<int32_t>(c_bytes) : nullptr;
  float* dc = (want_c && wire == Wire::None) ? cv.take<float>(c_bytes) : nullptr;
  if (drs) BITMM_CUDA_TRY(cudaMemcpyAsync(drs, row_scale, m * 4, cudaMemcpyHostToDevice, s));
  if (dcs) BITMM_CUDA_TRY(cudaMemcpyAsync(dcs, col_scale, n * 4, cudaMemcpyHostToDevice, s));
  // slices of output rows (rows of the weight planes)
  auto in = [=](int64_t r0, int64_t r1, cudaStream_t cs) -> int {
    const size_t off = r0 * wpr, bytes = (r1 - r0) * wpr * 8;
    for (int i = 0; i < 3; ++i)
      BITMM_CUDA_TRY(cudaMemcpyAsync(d[i] + off, src[i] + off, bytes, cudaMemcpyHostToDevice, cs));
    return BITMM_OK;
  };
  auto gemm = [=](int64_t r0, int64_t r1) -> int {
    const size_t off = r0 * wpr;
    return gemm_2x2_dev_impl(*st, d[0] + off, d[1] + off, d[2] + off, r1 - r0, w_scale,
                             has_w_gamma, w_gamma, d[3], d[4], d[5], n, k, wpr, a_scale,
                             has_a_gamma, a_gamma, drs ? drs + r0 : nullptr, dcs,
                             dcu ? dcu + r0 * ldc : nullptr, dc ? dc + r0 * ldc : nullptr, ldc, s);
  };
  auto body = [&](int64_t r0, int64_t r1) -> int {
    BITMM_TRY(in(r0, r1, s));
    return gemm(r0, r1);
  };
  if (wire != Wire::None) {
    // kernels.cpp:232-233, the same expression gemm_2x2_dev_impl passes to the epilogue
    const float scale = 0.25f * w_scale * a_scale * (has_w_gamma ? w_gamma : 1.0f) *
                        (has_a_gamma ? a_gamma : 1.0f);
    const WireOut wo{wire, static_cast<int>(k), scale, row_scale, col_scale, c_units, c, ldc};
    return run_or_defer_wire(hl.host(), s,
                             WireItem{m, pipe_step(m, c_bytes, 256), in, gemm,
                                      [=](int64_t r0, int64_t r1) { return OutBlock{r0, r1 - r0, 0, n}; },
                                      wo, dcu, cv.take<uint16_t>(wire_bytes), static_cast<size_t>(m * n)});
  }
  if (pipe_step(m, c_bytes, 256) >= m && use_staged(o)) {
    BITMM_TRY(body(0, m));
    return run_staged(hl.host(), s, m, n, ldc, dcu, dc, o);
  }
  BITMM_TRY(run_pipelined(
      hl.host(), s, m, pipe_step(m, c_bytes, 256), body,
      [&](int64_t r0, int64_t r1, cudaStream_t d2h) -> int {
        // rows of n cells: the caller's columns [n, ldc) are not the output's
        const size_t pitch = ldc * 4, width = n * 4;
        if (dcu) BITMM_CUDA_TRY(cudaMemcpy2DAsync(c_units + r0 * ldc, pitch, dcu + r0 * ldc, pitch, width, r1 - r0, cudaMemcpyDeviceToHost, d2h));
        if (dc) BITMM_CUDA_TRY(cudaMemcpy2DAsync(c + r0 * ldc, pitch, dc + r0 * ldc, pitch, width, r1 - r0, cudaMemcpyDeviceToHost, d2h));
        g_d2h_bytes += ((dcu ? 1 : 0) + (dc ? 1 : 0)) * width * (r1 - r0);
        return BITMM_OK;
      }));
  return read_status_host(hl.host(), s);
}

}  // namespace

extern "C" {

int bitmm_gemm_2x2_host(const uint64_t* wt, const uint64_t* wh, const uint64_t* wm, int64_t m,
                        float w_scale, int has_w_gamma, float w_gamma, const uint64_t* at,
                        const uint64_t* ah, const uint64_t* am, int64_t n, int64_t k, int64_t wpr,
                        float a_scale, int has_a_gamma, float a_gamma, const float* row_scale,
                        const float* col_scale, int32_t* c_units, float* c, int64_t ldc) {
  HostOut o = HostOut::given(c_units, c, ldc);
  return gemm_2x2_host_impl(wt, wh, wm, m, w_scale, has_w_gamma, w_gamma, at, ah, am, n, k, wpr, a_scale,
                            has_a_gamma, a_gamma, row_scale, col_scale, o);
}

// Host batch (include/bitmm_b200.h): when every item's output takes the 16-bit wire, the items'
// host calls run in two passes on one lease (size the device staging, then carve it and collect
// the wire pipelines) and their pipelines run as one (run_wire_items); otherwise the items run
// as their *_host calls, one after the other.
static int batch_item_call(const bitmm_gemm_item& it) {
  HostOut o = HostOut::given(it.c_units, it.c, it.ldc);
  switch (it.routine) {
    case BITMM_ROUTINE_1X1:
      return gemm_1x1_host_impl(it.a0, it.m, it.b0, it.n, it.k, it.wpr, it.a_scale, it.b_scale, o);
    case BITMM_ROUTINE_1X2:
      return gemm_1x2_host_impl(it.a0, it.m, it.a_scale, it.b0, it.b1, it.b2, it.n, it.k, it.wpr, it.b_scale,
                                it.has_b_gamma, it.b_gamma, it.row_scale, it.col_scale, o);
    default:
      return gemm_2x2_host_impl(it.a0, it.a1, it.a2, it.m, it.a_scale, it.has_a_gamma, it.a_gamma, it.b0, it.b1,
                                it.b2, it.n, it.k, it.wpr, it.b_scale, it.has_b_gamma, it.b_gamma, it.row_scale,
                                it.col_scale, o);
  }
}

int bitmm_gemm_batch_host(const bitmm_gemm_item* items, int count) {
  g_launches = 0;
  g_d2h_bytes = 0;
  if (count <= 0 || count > TC_GROUP_MAX || items == nullptr)
    return fail(BITMM_ERR_INVALID_ARGUMENT, "batch must hold 1..4 items");
  bool merge = std::getenv("BITMM_HOST_BATCH") == nullptr || std::atoi(std::getenv("BITMM_HOST_BATCH")) != 0;
  for (int i = 0; i < count; ++i) {
    const bitmm_gemm_item& it = items[i];
    if (it.routine < BITMM_ROUTINE_1X1 || it.routine > BITMM_ROUTINE_2X2)
      return fail(BITMM_ERR_INVALID_ARGUMENT, "unknown routine");
    const bool ok_dims = it.m > 0 && it.n > 0 && it.ldc >= it.n && (it.c_units || it.c);
    merge = merge && ok_dims && host_wire(it.routine, it.k, static_cast<size_t>(it.m * it.ldc) * 4) != Wire::None;
  }
  if (!merge) {
    for (int i = 0; i < count; ++i) {
      const uint64_t d2h = g_d2h_bytes;
      BITMM_TRY(batch_item_call(items[i]));
      g_d2h_bytes += d2h;
    }
    return BITMM_OK;
  }
  HostLease hl;
  BITMM_TRY(hl.acquire());
  cudaStream_t s = hl->stream;
  std::vector<WireItem> wire_items;
  HostBatch hb;
  hb.host = &hl.host();
  hb.items = &wire_items;
  struct Reset {
    ~Reset() { g_batch = nullptr; }
  } reset;
  g_batch = &hb;
  for (int i = 0; i < count; ++i) {  // pass 1: argument checks, device staging needed
    const int rc = batch_item_call(items[i]);
    if (rc != kBatchSized) return rc == BITMM_OK ? fail(BITMM_ERR_CUDA, "batch sizing") : rc;
  }
  BITMM_TRY(arena_reserve(hl->io, s, hb.need));
  hb.sizing = false;
  hb.need = 0;
  for (int i = 0; i < count; ++i) BITMM_TRY(batch_item_call(items[i]));  // pass 2: setup copies, pipelines
  g_batch = nullptr;
  BITMM_TRY(run_wire_items(hl.host(), s, wire_items));
  return read_status_host(hl.host(), s);
}

// Late-output host call (include/bitmm_b200.h): item fields as bitmm_gemm_batch_dev reads them.
int bitmm_gemm_host_late(const bitmm_gemm_item* it, int want, bitmm_out_fn out_fn, void* user) {
  if (!it || !out_fn || (want & ~(BITMM_WANT_UNITS | BITMM_WANT_C)) || !want)
    return fail(BITMM_ERR_INVALID_ARGUMENT, "late output needs an item, a callback and a wanted output");
  HostOut o;
  o.want_units = (want & BITMM_WANT_UNITS) != 0;
  o.want_c = (want & BITMM_WANT_C) != 0;
  o.fn = out_fn;
  o.user = user;
  switch (it->routine) {
    case BITMM_ROUTINE_1X1:
      return gemm_1x1_host_impl(it->a0, it->m, it->b0, it->n, it->k, it->wpr, it->a_scale, it->b_scale, o);
    case BITMM_ROUTINE_1X2:
      return gemm_1x2_host_impl(it->a0, it->m, it->a_scale, it->b0, it->b1, it->b2, it->n, it->k, it->wpr,
                                it->b_scale, it->has_b_gamma, it->b_gamma, it->row_scale, it->col_scale, o);
    case BITMM_ROUTINE_2X2:
      return gemm_2x2_host_impl(it->a0, it->a1, it->a2, it->m, it->a_scale, it->has_a_gamma, it->a_gamma, it->b0,
                                it->b1, it->b2, it->n, it->k, it->wpr, it->b_scale, it->has_b_gamma, it->b_gamma,
                                it->row_scale, it->col_scale, o);
    default:
      return fail(BITMM_ERR_INVALID_ARGUMENT, "unknown routine");
  }
}

// ---------------- 1/32 and APB ----------------
static int check_1x32_dims(int64_t m, int64_t k, int64_t wpr, int64_t n, int64_t ldb, int64_t ldc) {
  if (m <= 0 || k <= 0 || n <= 0) return fail(BITMM_ERR_INVALID_ARGUMENT, "gemm dimensions must be positive");
  if (k > BITMM_MAX_SHARED_DIM)
    return fail(BITMM_ERR_INVALID_ARGUMENT, "shared dimension exceeds the 2^20 accumulator bound");
  if (wpr * 64 < k) return fail(BITMM_ERR_INVALID_ARGUMENT, "words_per_row too small for the column count");
  if (ldb < n || ldc < n) return fail(BITMM_ERR_INVALID_ARGUMENT, "leading dimension smaller than the column count");
  if (m > INT32_MAX / 2 || n > INT32_MAX / 2) return fail(BITMM_ERR_INVALID_ARGUMENT, "gemm dimension too large");
  return BITMM_OK;
}

int bitmm_gemm_1x32_dev(const uint64_t* w, int64_t m, int64_t k, int64_t wpr, float gamma,
                        const float* row_gamma, const float* b, int64_t n, int64_t ldb, float* c,
                        int64_t ldc, void* stream) {
  g_launches = 0;
  BITMM_TRY(check_1x32_dims(m, k, wpr, n, ldb, ldc));
  if (!w || !b || !c) return fail(BITMM_ERR_INVALID_ARGUMENT, "null operand");
  CallCtx st;
  BITMM_TRY(st.acquire(static_cast<cudaStream_t>(stream)));
  return apb_dev_impl(*st, w, m, k, wpr, gamma, row_gamma, b, n, ldb, nullptr, nullptr, nullptr, c,
                      ldc, static_cast<cudaStream_t>(stream));
}

int bitmm_gemm_1x32_host(const uint64_t* w, int64_t m, int64_t k, int64_t wpr, float gamma,
                         const float* row_gamma, const float* b, int64_t n, int64_t ldb, float* c,
                         int64_t ldc) {
  g_launches = 0;
  BITMM_TRY(check_1x32_dims(m, k, wpr, n, ldb, ldc));
  if (!w || !b || !c) return fail(BITMM_ERR_INVALID_ARGUMENT, "null operand");
  HostLease hl;
  BITMM_TRY(hl.acquire());
  Ctx* st = &hl.ctx();
  cudaStream_t s = hl->stream;
  const size_t w_bytes = m * wpr * 8, b_bytes = k * ldb * 4, c_bytes = m * ldc * 4;
  BITMM_TRY(arena_reserve(hl->io, s, align_up(w_bytes, 1024) + align_up(b_bytes, 1024) +
                                      align_up(c_bytes, 1024) + align_up(m * 4, 1024) + 4096));
  Carve cv(hl->io.ptr);
  uint64_t* dw = cv.take<uint64_t>(w_bytes);
  float* db = cv.take<float>(b_bytes);
  float* dc = cv.take<float>(c_bytes);
  float* dg = row_gamma ? cv.take<float>(m * 4) : nullptr;
  BITMM_CUDA_TRY(cudaMemcpyAsync(dw, w, w_bytes, cudaMemcpyHostToDevice, s));
  BITMM_CUDA_TRY(cudaMemcpyAsync(db, b, b_bytes, cudaMemcpyHostToDevice, s));
  if (dg) BITMM_CUDA_TRY(cudaMemcpyAsync(dg, row_gamma, m * 4, cudaMemcpyHostToDevice, s));
  BITMM_TRY(apb_dev_impl(*st, dw, m, k, wpr, gamma, dg, db, n, ldb, nullptr, nullptr, nullptr, dc, ldc, s));
  BITMM_CUDA_TRY(cudaMemcpy2DAsync(c, ldc * 4, dc, ldc * 4, n * 4, m, cudaMemcpyDeviceToHost, s));  // columns [n, ldc) are not the output's
  return read_status_host(hl.host(), s);
}

int bitmm_layer_forward_dev(int64_t rows, int64_t cols, float alpha, const float* row_alpha,
                            const uint64_t* bin, int64_t wpr, const uint64_t* row_ptr,
                            const uint64_t* col_idx, const float* vals, const float* b, int64_t n,
                            int64_t ldb, float* c, int64_t ldc, void* stream) {
  g_launches = 0;
  BITMM_TRY(check_1x32_dims(rows, cols, wpr, n, ldb, ldc));
  if (!bin || !b || !c || !row_ptr) return fail(BITMM_ERR_INVALID_ARGUMENT, "null operand");
  CallCtx st;
  BITMM_TRY(st.acquire(static_cast<cudaStream_t>(stream)));
  return apb_dev_impl(*st, bin, rows, cols, wpr, alpha, row_alpha, b, n, ldb, row_ptr, col_idx, vals,
                      c, ldc, static_cast<cudaStream_t>(stream));
}

int bitmm_layer_forward_host(int64_t rows, int64_t cols, float alpha, const float* row_alpha,
                             const uint64_t* bin, int64_t wpr, const uint64_t* row_ptr,
                             const uint64_t* col_idx, const float* vals, int64_t nnz,
                             const float* b, int64_t n, int64_t ldb, float* c, int64_t ldc) {
  g_launches = 0;
  BITMM_TRY(check_1x32_dims(rows, cols, wpr, n, ldb, ldc));
  if (!bin || !b || !c || !row_ptr || (nnz > 0 && (!col_idx || !vals)))
    return fail(BITMM_ERR_INVALID_ARGUMENT, "null operand");
  BITMM_TRY(check_csr_host(rows, cols, row_ptr, col_idx, vals, nnz));
  HostLease hl;
  BITMM_TRY(hl.acquire());
  Ctx* st = &hl.ctx();
  cudaStream_t s = hl->stream;
  const size_t w_bytes = rows * wpr * 8, b_bytes = cols * ldb * 4, c_bytes = rows * ldc * 4;
  const size_t rp_bytes = (rows + 1) * 8, ci_bytes = std::max<int64_t>(nnz, 1) * 8,
               v_bytes = std::max<int64_t>(nnz, 1) * 4;
  BITMM_TRY(arena_reserve(hl->io, s, align_up(w_bytes, 1024) + align_up(b_bytes, 1024) +
                                      align_up(c_bytes, 1024) + align_up(rows * 4, 1024) +
                                      align_up(rp_bytes, 1024) + align_up(ci_bytes, 1024) +
                                      align_up(v_bytes, 1024) + 4096));
  Carve cv(hl->io.ptr);
  uint64_t* dw = cv.take<uint64_t>(w_bytes);
  float* db = cv.take<float>(b_bytes);
  float* dc = cv.take<float>(c_bytes);
  float* da = row_alpha ? cv.take<float>(rows * 4) : nullptr;
  uint64_t* drp = cv.take<uint64_t>(rp_bytes);
  uint64_t* dci = cv.take<uint64_t>(ci_bytes);
  float* dv = cv.take<float>(v_bytes);
  BITMM_CUDA_TRY(cudaMemcpyAsync(dw, bin, w_bytes, cudaMemcpyHostToDevice, s));
  BITMM_CUDA_TRY(cudaMemcpyAsync(db, b, b_bytes, cudaMemcpyHostToDevice, s));
  if (da) BITMM_CUDA_TRY(cudaMemcpyAsync(da, row_alpha, rows * 4, cudaMemcpyHostToDevice, s));
  BITMM_CUDA_TRY(cudaMemcpyAsync(drp, row_ptr, rp_bytes, cudaMemcpyHostToDevice, s));
  if (nnz > 0) {
    BITMM_CUDA_TRY(cudaMemcpyAsync(dci, col_idx, nnz * 8, cudaMemcpyHostToDevice, s));
    BITMM_CUDA_TRY(cudaMemcpyAsync(dv, vals, nnz * 4, cudaMemcpyHostToDevice, s));
  }
  BITMM_TRY(apb_dev_impl(*st, dw, rows, cols, wpr, alpha, da, db, n, ldb, drp, dci, dv, dc, ldc, s));
  BITMM_CUDA_TRY(cudaMemcpy2DAsync(c, ldc * 4, dc, ldc * 4, n * 4, rows, cudaMemcpyDeviceToHost, s));  // columns [n, ldc) are not the output's
  return read_status_host(hl.host(), s);
}

// ---------------- standalone SpMM ----------------
int bitmm_spmm_csr_dev(int64_t rows, int64_t cols, const uint64_t* row_ptr, const uint64_t* col_idx,
                       const float* vals, const float* b, int64_t n, int64_t ldb, float* c,
                       int64_t ldc, void* stream) {
  g_launches = 0;
  // kernels.cpp:335-338
  if (rows <= 0 || n <= 0 || cols <= 0) return fail(BITMM_ERR_INVALID_ARGUMENT, "gemm dimensions must be positive");
  if (cols > BITMM_MAX_SHARED_DIM)
    return fail(BITMM_ERR_INVALID_ARGUMENT, "shared dimension exceeds the 2^20 accumulator bound");
  if (ldb < n || ldc < n) return fail(BITMM_ERR_INVALID_ARGUMENT, "leading dimension smaller than the column count");
  if (!row_ptr || !b || !c) return fail(BITMM_ERR_INVALID_ARGUMENT, "null operand");
  CallCtx st;
  BITMM_TRY(st.acquire(static_cast<cudaStream_t>(stream)));
  const char* v1 = std::getenv("BITMM_SPMM_V1");  // A/B: the 32-token fp32 chunk kernel
  if (!(v1 && std::atoi(v1) != 0) && spmm_levels_fits(*st, rows, cols, n, true))
    return run_spmm_levels(*st, rows, cols, row_ptr, col_idx, vals, SpmmLevels{}, n, c, ldc,
                           static_cast<cudaStream_t>(stream), b, ldb);
  return run_spmm<true, false>(*st, rows, cols, row_ptr, col_idx, vals, b, n, ldb, c, ldc,
                               static_cast<cudaStream_t>(stream));
}

int bitmm_spmm_csr_host(int64_t rows, int64_t cols, const uint64_t* row_ptr,
                        const uint64_t* col_idx, const float* vals, int64_t nnz, const float* b,
                        int64_t n, int64_t ldb, float* c, int64_t ldc) {
  g_launches = 0;
  if (rows <= 0 || n <= 0 || cols <= 0) return fail(BITMM_ERR_INVALID_ARGUMENT, "gemm dimensions must be positive");
  if (cols > BITMM_MAX_SHARED_DIM)
    return fail(BITMM_ERR_INVALID_ARGUMENT, "shared dimension exceeds the 2^20 accumulator bound");
  if (ldb < n || ldc < n) return fail(BITMM_ERR_INVALID_ARGUMENT, "leading dimension smaller than the column count");
  if (!row_ptr || !b || !c || (nnz > 0 && (!col_idx || !vals))) return fail(BITMM_ERR_INVALID_ARGUMENT, "null operand");
  BITMM_TRY(check_csr_host(rows, cols, row_ptr, col_idx, vals, nnz));
  HostLease hl;
  BITMM_TRY(hl.acquire());
  Ctx* st = &hl.ctx();
  cudaStream_t s = hl->stream;
  const size_t b_bytes = cols * ldb * 4, c_bytes = rows * ldc * 4, rp_bytes = (rows + 1) * 8;
  const size_t ci_bytes = std::max<int64_t>(nnz, 1) * 8, v_bytes = std::max<int64_t>(nnz, 1) * 4;
  BITMM_TRY(arena_reserve(hl->io, s, align_up(b_bytes, 1024) + align_up(c_bytes, 1024) +
                                      align_up(rp_bytes, 1024) + align_up(ci_bytes, 1024) +
                                      align_up(v_bytes, 1024) + 4096));
  Carve cv(hl->io.ptr);
  float* db = cv.take<float>(b_bytes);
  float* dc = cv.take<float>(c_bytes);
  uint64_t* drp = cv.take<uint64_t>(rp_bytes);
  uint64_t* dci = cv.take<uint64_t>(ci_bytes);
  float* dv = cv.take<float>(v_bytes);
  BITMM_CUDA_TRY(cudaMemcpyAsync(db, b, b_bytes, cudaMemcpyHostToDevice, s));
  BITMM_CUDA_TRY(cudaMemcpyAsync(drp, row_ptr, rp_bytes, cudaMemcpyHostToDevice, s));
  if (nnz > 0) {
    BITMM_CUDA_TRY(cudaMemcpyAsync(dci, col_idx, nnz * 8, cudaMemcpyHostToDevice, s));
    BITMM_CUDA_TRY(cudaMemcpyAsync(dv, vals, nnz * 4, cudaMemcpyHostToDevice, s));
  }
  BITMM_TRY(bitmm_spmm_csr_dev(rows, cols, drp, dci, dv, db, n, ldb, dc, ldc, s));
  BITMM_CUDA_TRY(cudaMemcpy2DAsync(c, ldc * 4, dc, ldc * 4, n * 4, rows, cudaMemcpyDeviceToHost, s));  // columns [n, ldc) are not the output's
  BITMM_CUDA_TRY(cudaStreamSynchronize(s));
  return BITMM_OK;
}

// ---------------- GPU packers ----------------
static int check_pack_args(int64_t rows, int64_t cols, int64_t lda, int64_t wpr) {
  if (rows < 0 || cols < 0) return fail(BITMM_ERR_INVALID_ARGUMENT, "matrix dimensions must be non-negative");
  if (wpr * 64 < cols) return fail(BITMM_ERR_INVALID_ARGUMENT, "words_per_row too small for the column count");
  if (lda < cols) return fail(BITMM_ERR_INVALID_ARGUMENT, "leading dimension smaller than the column count");
  if (cols > INT32_MAX / 2 || wpr > INT32_MAX / 128) return fail(BITMM_ERR_INVALID_ARGUMENT, "matrix too wide");
  return BITMM_OK;
}

static unsigned pack_blocks(const Ctx& st, int64_t rows, int64_t wpr) {
  const long long units = rows * ((wpr + PACK_WORDS_PER_WARP - 1) / PACK_WORDS_PER_WARP);
  const long long blocks = (units + 7) / 8;  // 8 warps per 256-thread block
  return static_cast<unsigned>(std::max<long long>(1, std::min<long long>(blocks, 32LL * st.sms)));
}

int bitmm_pack_signs_dev(const float* a, int64_t rows, int64_t cols, int64_t lda, uint64_t* words,
                         int64_t wpr, void* stream) {
  g_launches = 0;
  BITMM_TRY(check_pack_args(rows, cols, lda, wpr));
  if (rows == 0 || wpr == 0) return BITMM_OK;
  if (!words || (cols > 0 && !a)) return fail(BITMM_ERR_INVALID_ARGUMENT, "null operand");
  CallCtx st;
  BITMM_TRY(st.acquire(static_cast<cudaStream_t>(stream)));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ProfScope ps("pack_signs", s);
  pack_signs_kernel<<<pack_blocks(*st, rows, wpr), 256, 0, s>>>(
      a, rows, static_cast<int>(cols), lda, static_cast<int>(wpr),
      reinterpret_cast<unsigned long long*>(words));
  return launch_check("pack_signs_kernel");
}

int bitmm_quantize_thm_dev(const float* a, int64_t rows, int64_t cols, int64_t lda, float s_step,
                           uint64_t* t, uint64_t* h, uint64_t* m, int64_t wpr, void* stream) {
  g_launches = 0;
  if (!(s_step > 0.0f)) return fail(BITMM_ERR_INVALID_ARGUMENT, "quantization step must be positive");
  BITMM_TRY(check_pack_args(rows, cols, lda, wpr));
  if (rows == 0 || wpr == 0) return BITMM_OK;
  if (!t || !h || !m || (cols > 0 && !a)) return fail(BITMM_ERR_INVALID_ARGUMENT, "null operand");
  CallCtx st;
  BITMM_TRY(st.acquire(static_cast<cudaStream_t>(stream)));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ProfScope ps("quantize_thm", s);
  quantize_thm_kernel<<<pack_blocks(*st, rows, wpr), 256, 0, s>>>(
      a, rows, static_cast<int>(cols), lda, s_step, static_cast<int>(wpr),
      reinterpret_cast<unsigned long long*>(t), reinterpret_cast<unsigned long long*>(h),
      reinterpret_cast<unsigned long long*>(m));
  return launch_check("quantize_thm_kernel");
}

int bitmm_pack_signs_host(const float* a, int64_t rows, int64_t cols, int64_t lda, uint64_t* words,
                          int64_t wpr) {
  g_launches = 0;
  BITMM_TRY(check_pack_args(rows, cols, lda, wpr));
  if (rows == 0 || wpr == 0) return BITMM_OK;
  HostLease hl;
  BITMM_TRY(hl.acquire());
  Ctx* st = &hl.ctx();
  cudaStream_t s = hl->stream;
  const size_t a_bytes = rows * lda * 4, w_bytes = rows * wpr * 8;
  BITMM_TRY(arena_reserve(hl->io, s, align_up(a_bytes, 1024) + align_up(w_bytes, 1024) + 2048));
  Carve cv(hl->io.ptr);
  float* da = cv.take<float>(a_bytes);
  uint64_t* dw = cv.take<uint64_t>(w_bytes);
  BITMM_CUDA_TRY(cudaMemcpyAsync(da, a, a_bytes, cudaMemcpyHostToDevice, s));
  BITMM_TRY(bitmm_pack_signs_dev(da, rows, cols, lda, dw, wpr, s));
  BITMM_CUDA_TRY(cudaMemcpyAsync(words, dw, w_bytes, cudaMemcpyDeviceToHost, s));
  BITMM_CUDA_TRY(cudaStreamSynchronize(s));
  return BITMM_OK;
}

int bitmm_quantize_thm_host(const float* a, int64_t rows, int64_t cols, int64_t lda, float s_step,
                            uint64_t* t, uint64_t* h, uint64_t* m, int64_t wpr) {
  g_launches = 0;
  if (!(s_step > 0.0f)) return fail(BITMM_ERR_INVALID_ARGUMENT, "quantization step must be positive");
  BITMM_TRY(check_pack_args(rows, cols, lda, wpr));
  if (rows == 0 || wpr == 0) return BITMM_OK;
  HostLease hl;
  BITMM_TRY(hl.acquire());
  Ctx* st = &hl.ctx();
  cudaStream_t s = hl->stream;
  const size_t a_bytes = rows * lda * 4, w_bytes = rows * wpr * 8;
  BITMM_TRY(arena_reserve(hl->io, s, align_up(a_bytes, 1024) + 3 * align_up(w_bytes, 1024) + 4096));
  Carve cv(hl->io.ptr);
  float* da = cv.take<float>(a_bytes);
  uint64_t* dt = cv.take<uint64_t>(w_bytes);
  uint64_t* dh = cv.take<uint64_t>(w_bytes);
  uint64_t* dm = cv.take<uint64_t>(w_bytes);
  BITMM_CUDA_TRY(cudaMemcpyAsync(da, a, a_bytes, cudaMemcpyHostToDevice, s));
  BITMM_TRY(bitmm_quantize_thm_dev(da, rows, cols, lda, s_step, dt, dh, dm, wpr, s));
  BITMM_CUDA_TRY(cudaMemcpyAsync(t, dt, w_bytes, cudaMemcpyDeviceToHost, s));
  BITMM_CUDA_TRY(cudaMemcpyAsync(h, dh, w_bytes, cudaMemcpyDeviceToHost, s));
  BITMM_CUDA_TRY(cudaMemcpyAsync(m, dm, w_bytes, cudaMemcpyDeviceToHost, s));
  BITMM_CUDA_TRY(cudaStreamSynchronize(s));
  return BITMM_OK;
}

int bitmm_decompose_thm_dev(const uint8_t* levels, int64_t rows, int64_t cols, uint64_t* t,
                            uint64_t* h, uint64_t* m, int64_t wpr, void* stream) {
  g_launches = 0;
  BITMM_TRY(check_pack_args(rows, cols, cols, wpr));
  if (rows == 0 || wpr == 0) return BITMM_OK;
  if (!t || !h || !m || (cols > 0 && !levels)) return fail(BITMM_ERR_INVALID_ARGUMENT, "null operand");
  CallCtx st;
  BITMM_TRY(st.acquire(static_cast<cudaStream_t>(stream)));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ProfScope ps("decompose_thm", s);
  decompose_thm_kernel<<<pack_blocks(*st, rows, wpr), 256, 0, s>>>(
      levels, rows, static_cast<int>(cols), static_cast<int>(wpr),
      reinterpret_cast<unsigned long long*>(t), reinterpret_cast<unsigned long long*>(h),
      reinterpret_cast<unsigned long long*>(m), st->status);
  return launch_check("decompose_thm_kernel");
}

int bitmm_decompose_thm_host(const uint8_t* levels, int64_t rows, int64_t cols, uint64_t* t,
                             uint64_t* h, uint64_t* m, int64_t wpr) {
  g_launches = 0;
  BITMM_TRY(check_pack_args(rows, cols, cols, wpr));
  if (rows == 0 || wpr == 0) return BITMM_OK;
  HostLease hl;
  BITMM_TRY(hl.acquire());
  Ctx* st = &hl.ctx();
  cudaStream_t s = hl->stream;
  const size_t l_bytes = rows * cols, w_bytes = rows * wpr * 8;
  BITMM_TRY(arena_reserve(hl->io, s, align_up(l_bytes, 1024) + 3 * align_up(w_bytes, 1024) + 4096));
  Carve cv(hl->io.ptr);
  uint8_t* dl = cv.take<uint8_t>(l_bytes);
  uint64_t* dt = cv.take<uint64_t>(w_bytes);
  uint64_t* dh = cv.take<uint64_t>(w_bytes);
  uint64_t* dm = cv.take<uint64_t>(w_bytes);
  if (l_bytes) BITMM_CUDA_TRY(cudaMemcpyAsync(dl, levels, l_bytes, cudaMemcpyHostToDevice, s));
  BITMM_TRY(bitmm_decompose_thm_dev(dl, rows, cols, dt, dh, dm, wpr, s));
  BITMM_TRY(read_status_host(hl.host(), s));
  BITMM_CUDA_TRY(cudaMemcpyAsync(t, dt, w_bytes, cudaMemcpyDeviceToHost, s));
  BITMM_CUDA_TRY(cudaMemcpyAsync(h, dh, w_bytes, cudaMemcpyDeviceToHost, s));
  BITMM_CUDA_TRY(cudaMemcpyAsync(m, dm, w_bytes, cudaMemcpyDeviceToHost, s));
  BITMM_CUDA_TRY(cudaStreamSynchronize(s));
  return BITMM_OK;
}

// decompose_apb: pack the signs, count each row's residual entries, scan the counts into
// row_ptr, bring the total back, and (when the caller's buffers hold it) fill the CSR.
int bitmm_decompose_apb_dev(const float* a, int64_t rows, int64_t cols, int64_t lda, float alpha,
                            const float* row_alpha, uint64_t* bin, int64_t wpr, uint64_t* row_ptr,
                            uint64_t* col_idx, float* vals, int64_t capacity, int64_t* nnz,
                            void* stream) {
  g_launches = 0;
  if (row_alpha == nullptr && !(alpha > 0.0f)) return fail(BITMM_ERR_INVALID_ARGUMENT, "alpha must be positive");
  BITMM_TRY(check_pack_args(rows, cols, lda, wpr));
  if (!nnz || !row_ptr || (rows > 0 && wpr > 0 && !bin) || (rows > 0 && cols > 0 && !a))
    return fail(BITMM_ERR_INVALID_ARGUMENT, "null operand");
  CallCtx st;
  BITMM_TRY(st.acquire(static_cast<cudaStream_t>(stream)));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  auto* rp = reinterpret_cast<unsigned long long*>(row_ptr);
  BITMM_CUDA_TRY(cudaMemsetAsync(rp, 0, sizeof(unsigned long long), s));
  if (rows > 0) {
    if (wpr > 0) {
      ProfScope ps("pack_signs", s);
      pack_signs_kernel<<<pack_blocks(*st, rows, wpr), 256, 0, s>>>(
          a, rows, static_cast<int>(cols), lda, static_cast<int>(wpr),
          reinterpret_cast<unsigned long long*>(bin));
      BITMM_TRY(launch_check("pack_signs_kernel"));
    }
    const unsigned blocks = static_cast<unsigned>(std::min<long long>((rows + 7) / 8, 32LL * st->sms));
    {
      ProfScope ps("decompose_apb_count", s);
      decompose_apb_count_kernel<<<blocks, 256, 0, s>>>(a, rows, static_cast<int>(cols), lda, alpha,
                                                        row_alpha, rp, st->status);
      BITMM_TRY(launch_check("decompose_apb_count_kernel"));
    }
    size_t temp = 0;
    BITMM_CUDA_TRY(cub::DeviceScan::InclusiveSum(nullptr, temp, rp + 1, rp + 1, static_cast<int>(rows), s));
    BITMM_TRY(ws_reserve(*st, temp + 256));
    BITMM_CUDA_TRY(cub::DeviceScan::InclusiveSum(st->ws.ptr, temp, rp + 1, rp + 1, static_cast<int>(rows), s));
  }
  unsigned long long total = 0;
  BITMM_CUDA_TRY(cudaMemcpyAsync(&total, rp + rows, sizeof(total), cudaMemcpyDeviceToHost, s));
  BITMM_TRY(read_status(*st, s));  // synchronises; reports a non-positive row alpha
  *nnz = static_cast<int64_t>(total);
  if (rows == 0 || total == 0 || col_idx == nullptr || vals == nullptr ||
      capacity < static_cast<int64_t>(total))
    return BITMM_OK;
  const unsigned blocks = static_cast<unsigned>(std::min<long long>((rows + 7) / 8, 32LL * st->sms));
  ProfScope ps("decompose_apb_fill", s);
  decompose_apb_fill_kernel<<<blocks, 256, 0, s>>>(a, rows, static_cast<int>(cols), lda, alpha,
                                                   row_alpha, rp,
                                                   reinterpret_cast<unsigned long long*>(col_idx), vals);
  BITMM_TRY(launch_check("decompose_apb_fill_kernel"));
  BITMM_CUDA_TRY(cudaStreamSynchronize(s));
  return BITMM_OK;
}

int bitmm_decompose_apb_host(const float* a, int64_t rows, int64_t cols, int64_t lda, float alpha,
                             const float* row_alpha, uint64_t* bin, int64_t wpr, uint64_t* row_ptr,
                             uint64_t* col_idx, float* vals, int64_t capacity, int64_t* nnz) {
  g_launches = 0;
  if (row_alpha == nullptr && !(alpha > 0.0f)) return fail(BITMM_ERR_INVALID_ARGUMENT, "alpha must be positive");
  BITMM_TRY(check_pack_args(rows, cols, lda, wpr));
  if (!nnz || !row_ptr || (rows > 0 && wpr > 0 && !bin) || (rows > 0 && cols > 0 && !a))
    return fail(BITMM_ERR_INVALID_ARGUMENT, "null operand");
  HostLease hl;
  BITMM_TRY(hl.acquire());
  Ctx* st = &hl.ctx();
  cudaStream_t s = hl->stream;
  const bool fill = col_idx != nullptr && vals != nullptr && capacity > 0;
  const size_t a_bytes = rows * lda * 4, w_bytes = rows * wpr * 8, r_bytes = (rows + 1) * 8,
               al_bytes = row_alpha ? rows * 4 : 0, ci_bytes = fill ? capacity * 8 : 0,
               v_bytes = fill ? capacity * 4 : 0;
  BITMM_TRY(arena_reserve(hl->io, s, align_up(a_bytes, 1024) + align_up(w_bytes, 1024) +
                                      align_up(r_bytes, 1024) + align_up(al_bytes, 1024) +
                                      align_up(ci_bytes, 1024) + align_up(v_bytes, 1024) + 8192));
  Carve cv(hl->io.ptr);
  float* da = cv.take<float>(a_bytes);
  uint64_t* dw = cv.take<uint64_t>(w_bytes);
  uint64_t* dr = cv.take<uint64_t>(r_bytes);
  float* dal = row_alpha ? cv.take<float>(al_bytes) : nullptr;
  uint64_t* dci = fill ? cv.take<uint64_t>(ci_bytes) : nullptr;
  float* dv = fill ? cv.take<float>(v_bytes) : nullptr;
  if (a_bytes) BITMM_CUDA_TRY(cudaMemcpyAsync(da, a, a_bytes, cudaMemcpyHostToDevice, s));
  if (dal) BITMM_CUDA_TRY(cudaMemcpyAsync(dal, row_alpha, al_bytes, cudaMemcpyHostToDevice, s));
  BITMM_TRY(bitmm_decompose_apb_dev(da, rows, cols, lda, alpha, dal, dw, wpr, dr, dci, dv, capacity,
                                    nnz, s));
  if (w_bytes) BITMM_CUDA_TRY(cudaMemcpyAsync(bin, dw, w_bytes, cudaMemcpyDeviceToHost, s));
  BITMM_CUDA_TRY(cudaMemcpyAsync(row_ptr, dr, r_bytes, cudaMemcpyDeviceToHost, s));
  if (fill && *nnz > 0 && *nnz <= capacity) {
    BITMM_CUDA_TRY(cudaMemcpyAsync(col_idx, dci, *nnz * 8, cudaMemcpyDeviceToHost, s));
    BITMM_CUDA_TRY(cudaMemcpyAsync(vals, dv, *nnz * 4, cudaMemcpyDeviceToHost, s));
  }
  BITMM_CUDA_TRY(cudaStreamSynchronize(s));
  return BITMM_OK;
}

// ---------------- APB with 2-bit activations ----------------
int bitmm_layer_forward_2bit_dev(int64_t rows, int64_t cols, float alpha, const float* row_alpha,
                                 const uint64_t* bin, int64_t wpr, const uint64_t* row_ptr,
                                 const uint64_t* col_idx, const float* vals, const uint64_t* t,
                                 const uint64_t* h, const uint64_t* m, int64_t tokens,
                                 float a_scale, int has_a_gamma, float a_gamma, float* c,
                                 int64_t ldc, void* stream) {
  g_launches = 0;
  if (!(a_scale > 0.0f)) return fail(BITMM_ERR_INVALID_ENCODING, "plane scale must be positive");
  BITMM_TRY(check_gemm_dims(rows, tokens, cols, wpr, ldc));
  if (!bin || !row_ptr || !t || !h || !m || !c) return fail(BITMM_ERR_INVALID_ARGUMENT, "null operand");
  CallCtx st;
  BITMM_TRY(st.acquire(static_cast<cudaStream_t>(stream)));
  return apb2_dev_impl(*st, rows, cols, wpr, alpha, row_alpha, bin, row_ptr, col_idx, vals, t, h, m,
                       tokens, a_scale, has_a_gamma ? a_gamma : 1.0f, c, ldc,
                       static_cast<cudaStream_t>(stream));
}

int bitmm_layer_forward_2bit_host(int64_t rows, int64_t cols, float alpha, const float* row_alpha,
                                  const uint64_t* bin, int64_t wpr, const uint64_t* row_ptr,
                                  const uint64_t* col_idx, const float* vals, int64_t nnz,
                                  const uint64_t* t, const uint64_t* h, const uint64_t* m,
                                  int64_t tokens, float a_scale, int has_a_gamma, float a_gamma,
                                  float* c, int64_t ldc) {
  g_launches = 0;
  if (!(a_scale > 0.0f)) return fail(BITMM_ERR_INVALID_ENCODING, "plane scale must be positive");
  BITMM_TRY(check_gemm_dims(rows, tokens, cols, wpr, ldc));
  if (!bin || !row_ptr || !t || !h || !m || !c || (nnz > 0 && (!col_idx || !vals)))
    return fail(BITMM_ERR_INVALID_ARGUMENT, "null operand");
  BITMM_TRY(check_csr_host(rows, cols, row_ptr, col_idx, vals, nnz));
  HostLease hl;
  BITMM_TRY(hl.acquire());
  Ctx* st = &hl.ctx();
  cudaStream_t s = hl->stream;
  const size_t w_bytes = rows * wpr * 8, p_bytes = tokens * wpr * 8, c_bytes = rows * ldc * 4;
  const size_t rp_bytes = (rows + 1) * 8, ci_bytes = std::max<int64_t>(nnz, 1) * 8,
               v_bytes = std::max<int64_t>(nnz, 1) * 4;
  BITMM_TRY(arena_reserve(hl->io, s, align_up(w_bytes, 1024) + 3 * align_up(p_bytes, 1024) +
                                      align_up(c_bytes, 1024) + align_up(rows * 4, 1024) +
                                      align_up(rp_bytes, 1024) + align_up(ci_bytes, 1024) +
                                      align_up(v_bytes, 1024) + 4096));
  Carve cv(hl->io.ptr);
  uint64_t* dw = cv.take<uint64_t>(w_bytes);
  uint64_t* dt = cv.take<uint64_t>(p_bytes);
  uint64_t* dh = cv.take<uint64_t>(p_bytes);
  uint64_t* dm = cv.take<uint64_t>(p_bytes);
  float* dc = cv.take<float>(c_bytes);
  float* da = row_alpha ? cv.take<float>(rows * 4) : nullptr;
  uint64_t* drp = cv.take<uint64_t>(rp_bytes);
  uint64_t* dci = cv.take<uint64_t>(ci_bytes);
  float* dv = cv.take<float>(v_bytes);
  BITMM_CUDA_TRY(cudaMemcpyAsync(dw, bin, w_bytes, cudaMemcpyHostToDevice, s));
  BITMM_CUDA_TRY(cudaMemcpyAsync(dt, t, p_bytes, cudaMemcpyHostToDevice, s));
  BITMM_CUDA_TRY(cudaMemcpyAsync(dh, h, p_bytes, cudaMemcpyHostToDevice, s));
  BITMM_CUDA_TRY(cudaMemcpyAsync(dm, m, p_bytes, cudaMemcpyHostToDevice, s));
  if (da) BITMM_CUDA_TRY(cudaMemcpyAsync(da, row_alpha, rows * 4, cudaMemcpyHostToDevice, s));
  BITMM_CUDA_TRY(cudaMemcpyAsync(drp, row_ptr, rp_bytes, cudaMemcpyHostToDevice, s));
  if (nnz > 0) {
    BITMM_CUDA_TRY(cudaMemcpyAsync(dci, col_idx, nnz * 8, cudaMemcpyHostToDevice, s));
    BITMM_CUDA_TRY(cudaMemcpyAsync(dv, vals, nnz * 4, cudaMemcpyHostToDevice, s));
  }
  BITMM_TRY(apb2_dev_impl(*st, rows, cols, wpr, alpha, da, dw, drp, dci, dv, dt, dh, dm, tokens,
                          a_scale, has_a_gamma ? a_gamma : 1.0f, dc, ldc, s));
  BITMM_CUDA_TRY(cudaMemcpy2DAsync(c, ldc * 4, dc, ldc * 4, tokens * 4, rows, cudaMemcpyDeviceToHost, s));  // columns [tokens, ldc) are not the output's
  return read_status_host(hl.host(), s);
}

// ---------------- GEMM group ----------------
// Reference shift and scale of one batch item.
static void batch_scale(const bitmm_gemm_item& it, int* shift, float* scale) {
  if (it.routine == BITMM_ROUTINE_1X1) {  // kernels.cpp:170
    *shift = 0;
    *scale = it.a_scale * it.b_scale;
  } else if (it.routine == BITMM_ROUTINE_1X2) {  // kernels.cpp:193
    *shift = 1;
    *scale = 0.5f * it.a_scale * it.b_scale * (it.has_b_gamma ? it.b_gamma : 1.0f);
  } else {  // kernels.cpp:232-233
    *shift = 2;
    *scale = 0.25f * it.a_scale * it.b_scale * (it.has_a_gamma ? it.a_gamma : 1.0f) *
             (it.has_b_gamma ? it.b_gamma : 1.0f);
  }
}

int bitmm_gemm_batch_dev(const bitmm_gemm_item* items, int count, void* stream) {
  g_launches = 0;
  if (count <= 0 || count > TC_GROUP_MAX || items == nullptr)
    return fail(BITMM_ERR_INVALID_ARGUMENT, "batch must hold 1..4 items");
  int nprob = 0;
  for (int i = 0; i < count; ++i) {
    const bitmm_gemm_item& it = items[i];
    if (it.routine < BITMM_ROUTINE_1X1 || it.routine > BITMM_ROUTINE_2X2)
      return fail(BITMM_ERR_INVALID_ARGUMENT, "unknown routine");
    if (it.routine == BITMM_ROUTINE_1X2 && !(it.b_scale > 0.0f))
      return fail(BITMM_ERR_INVALID_ENCODING, "plane scale must be positive");
    if (it.routine == BITMM_ROUTINE_2X2 && (!(it.a_scale > 0.0f) || !(it.b_scale > 0.0f)))
      return fail(BITMM_ERR_INVALID_ENCODING, "plane scale must be positive");
    BITMM_TRY(check_gemm_dims(it.m, it.n, it.k, it.wpr, it.ldc));
    const bool planes_a = it.routine == BITMM_ROUTINE_2X2, planes_b = it.routine != BITMM_ROUTINE_1X1;
    if (!it.a0 || !it.b0 || (planes_a && (!it.a1 || !it.a2)) || (planes_b && (!it.b1 || !it.b2)) ||
        (!it.c_units && !it.c))
      return fail(BITMM_ERR_INVALID_ARGUMENT, "null operand");
    nprob += (it.c_units ? 1 : 0) + (it.c ? 1 : 0);
  }
  if (nprob > TC_GROUP_MAX) return fail(BITMM_ERR_INVALID_ARGUMENT, "batch exceeds 4 GEMM outputs");
  CallCtx st;
  BITMM_TRY(st.acquire(static_cast<cudaStream_t>(stream)));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool fp4 = use_fp4();
  {
    // in-GEMM expansion: one prep launch (codes / padding checks) + one fx_gemm launch
    FxItem fit[TC_GROUP_MAX];
    bool ok = fx_enabled();
    for (int i = 0; i < count && ok; ++i) {
      const bitmm_gemm_item& it = items[i];
      const bool planes_a = it.routine == BITMM_ROUTINE_2X2, planes_b = it.routine != BITMM_ROUTINE_1X1;
      const OperandSrc sa{it.a0, it.a1, it.a2, it.m, planes_a}, sb{it.b0, it.b1, it.b2, it.n, planes_b};
      ok = fx_operand_ok(sa, it.wpr) && fx_operand_ok(sb, it.wpr);
      int shift;
      float scale;
      batch_scale(it, &shift, &scale);
      const float* rs = it.routine == BITMM_ROUTINE_1X1 ? nullptr : it.row_scale;
      const float* cs = it.routine == BITMM_ROUTINE_1X1 ? nullptr : it.col_scale;
      fit[i] = fx_item(sa, sb, it.k, it.wpr,
                       fp4_shift(shift, static_cast<int>(planes_a) + static_cast<int>(planes_b), true), scale,
                       rs, cs, it.c_units, it.c, it.ldc);
    }
    if (ok) return run_fx(*st, fit, count, s);
  }
  size_t bytes = 2048;
  for (int i = 0; i < count; ++i) {
    const int64_t rb = row_bytes(kpad_for(items[i].k, fp4), fp4);
    bytes += align_up(items[i].m * rb, 1024) + align_up(items[i].n * rb, 1024);
  }
  BITMM_TRY(ws_reserve(*st, bytes));
  Carve cv(st->ws.ptr);
  UnpackSet U{};
  U.fp4 = fp4 ? 1 : 0;
  U.err = st->status;
  GemmProblem probs[TC_GROUP_MAX];
  int np = 0;
  for (int i = 0; i < count; ++i) {
    const bitmm_gemm_item& it = items[i];
    const int64_t kpad = kpad_for(it.k, fp4), rb = row_bytes(kpad, fp4);
    uint8_t* A8 = cv.take<uint8_t>(it.m * rb);
    uint8_t* B8 = cv.take<uint8_t>(it.n * rb);
    const bool planes_a = it.routine == BITMM_ROUTINE_2X2, planes_b = it.routine != BITMM_ROUTINE_1X1;
    U.op[U.count++] = make_unpack_operand({it.a0, it.a1, it.a2, it.m, planes_a}, it.wpr, it.k, kpad, A8);
    U.op[U.count++] = make_unpack_operand({it.b0, it.b1, it.b2, it.n, planes_b}, it.wpr, it.k, kpad, B8);
    int shift;
    float scale;
    batch_scale(it, &shift, &scale);
    const float* rs = it.routine == BITMM_ROUTINE_1X1 ? nullptr : it.row_scale;
    const float* cs = it.routine == BITMM_ROUTINE_1X1 ? nullptr : it.col_scale;
    shift = fp4_shift(shift, static_cast<int>(planes_a) + static_cast<int>(planes_b), fp4);
    np += make_problems(A8, B8, it.m, it.n, kpad, shift, scale, rs, cs, it.c_units, it.c, it.ldc,
                        probs + np);
  }
  BITMM_TRY(run_unpack_set(U, s));
  return run_problems(*st, probs, np, fp4, s);
}

// ---------------- row ops ----------------
static int run_row_ops(const uint64_t* a, const uint64_t* b, const uint64_t* z, int64_t count,
                       int64_t words, int64_t n, int64_t* out, void* stream) {
  g_launches = 0;
  if (count < 0 || words < 0) return fail(BITMM_ERR_INVALID_ARGUMENT, "row counts must be non-negative");
  if (count == 0) return BITMM_OK;
  if (!out || (words > 0 && (!a || !b))) return fail(BITMM_ERR_INVALID_ARGUMENT, "null operand");
  CallCtx st;
  BITMM_TRY(st.acquire(static_cast<cudaStream_t>(stream)));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ProfScope ps(z ? "mbm_rows" : "dot_binary_rows", s);
  row_ops_kernel<<<blocks_for(std::min<int64_t>(count, 64LL * st->sms) * 32, 256), 256, 0, s>>>(
      reinterpret_cast<const unsigned long long*>(a), reinterpret_cast<const unsigned long long*>(b),
      reinterpret_cast<const unsigned long long*>(z), count, words, n, reinterpret_cast<long long*>(out));
  return launch_check("row_ops_kernel");
}

int bitmm_dot_binary_dev(const uint64_t* u, const uint64_t* v, int64_t count, int64_t words,
                         int64_t n, int64_t* out, void* stream) {
  // kernels.cpp:121-123
  if (n < 0 || (n + 63) / 64 > words)
    return fail(BITMM_ERR_INVALID_ARGUMENT, "logical length does not fit the row words");
  return run_row_ops(u, v, nullptr, count, words, n, out, stream);
}

int bitmm_mbm_dev(const uint64_t* x, const uint64_t* y, const uint64_t* z, int64_t count,
                  int64_t words, int64_t* out, void* stream) {
  if (words > 0 && !z) return fail(BITMM_ERR_INVALID_ARGUMENT, "null operand");
  if (words == 0) {  // mbm of empty rows is 0 (kernels.cpp:134)
    if (count > 0 && out) {
      BITMM_CUDA_TRY(cudaMemsetAsync(out, 0, count * 8, static_cast<cudaStream_t>(stream)));
    }
    return BITMM_OK;
  }
  return run_row_ops(x, y, z, count, words, 0, out, stream);
}

static int row_ops_host(const uint64_t* a, const uint64_t* b, const uint64_t* z, int64_t count,
                        int64_t words, int64_t n, int64_t* out) {
  if (count < 0 || words < 0) return fail(BITMM_ERR_INVALID_ARGUMENT, "row counts must be non-negative");
  if (count == 0) return BITMM_OK;
  if (!out || (words > 0 && (!a || !b || (z == nullptr && n < 0)))) return fail(BITMM_ERR_INVALID_ARGUMENT, "null operand");
  HostLease hl;
  BITMM_TRY(hl.acquire());
  cudaStream_t s = hl->stream;
  const size_t rows_bytes = static_cast<size_t>(count * words) * 8, out_bytes = static_cast<size_t>(count) * 8;
  BITMM_TRY(arena_reserve(hl->io, s, 3 * align_up(rows_bytes, 1024) + align_up(out_bytes, 1024) + 1024));
  Carve cv(hl->io.ptr);
  uint64_t* da = cv.take<uint64_t>(rows_bytes);
  uint64_t* db = cv.take<uint64_t>(rows_bytes);
  uint64_t* dz = z ? cv.take<uint64_t>(rows_bytes) : nullptr;
  int64_t* dout = cv.take<int64_t>(out_bytes);
  if (rows_bytes) {
    BITMM_CUDA_TRY(cudaMemcpyAsync(da, a, rows_bytes, cudaMemcpyHostToDevice, s));
    BITMM_CUDA_TRY(cudaMemcpyAsync(db, b, rows_bytes, cudaMemcpyHostToDevice, s));
    if (dz) BITMM_CUDA_TRY(cudaMemcpyAsync(dz, z, rows_bytes, cudaMemcpyHostToDevice, s));
  }
  if (z) BITMM_TRY(bitmm_mbm_dev(da, db, dz, count, words, dout, s));
  else BITMM_TRY(bitmm_dot_binary_dev(da, db, count, words, n, dout, s));
  BITMM_CUDA_TRY(cudaMemcpyAsync(out, dout, out_bytes, cudaMemcpyDeviceToHost, s));
  BITMM_CUDA_TRY(cudaStreamSynchronize(s));
  return BITMM_OK;
}

int bitmm_dot_binary_host(const uint64_t* u, const uint64_t* v, int64_t count, int64_t words, int64_t n,
                          int64_t* out) {
  g_launches = 0;
  if (n < 0 || (n + 63) / 64 > words)  // kernels.cpp:121-123
    return fail(BITMM_ERR_INVALID_ARGUMENT, "logical length does not fit the row words");
  return row_ops_host(u, v, nullptr, count, words, n, out);
}

int bitmm_mbm_host(const uint64_t* x, const uint64_t* y, const uint64_t* z, int64_t count, int64_t words,
                   int64_t* out) {
  g_launches = 0;
  if (words > 0 && !z) return fail(BITMM_ERR_INVALID_ARGUMENT, "null operand");
  if (words == 0) {  // mbm of empty rows is 0 (kernels.cpp:134)
    for (int64_t i = 0; i < count; ++i) out[i] = 0;
    return BITMM_OK;
  }
  return row_ops_host(x, y, z, count, words, 0, out);
}

// ---------------- plane validation ----------------
int bitmm_validate_planes_dev(const uint64_t* t, const uint64_t* h, const uint64_t* m,
                              int64_t rows, int64_t cols, int64_t wpr, float scale, void* stream) {
  g_launches = 0;
  if (!(scale > 0.0f)) return fail(BITMM_ERR_INVALID_ENCODING, "plane scale must be positive");
  if (rows < 0 || cols < 0 || wpr * 64 < cols)
    return fail(BITMM_ERR_INVALID_ARGUMENT, "words_per_row too small for the column count");
  if (rows == 0 || wpr == 0) return BITMM_OK;
  if (!t || !h || !m) return fail(BITMM_ERR_INVALID_ARGUMENT, "null operand");
  CallCtx st;
  BITMM_TRY(st.acquire(static_cast<cudaStream_t>(stream)));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int* pad = st->scratch;
  unsigned long long* first = reinterpret_cast<unsigned long long*>(st->scratch + 2);
  BITMM_CUDA_TRY(cudaMemsetAsync(pad, 0, 4, s));
  BITMM_CUDA_TRY(cudaMemsetAsync(first, 0xFF, 8, s));
  {
    ProfScope ps("validate_planes", s);
    validate_planes_kernel<<<blocks_for(rows * wpr, 256), 256, 0, s>>>(
        reinterpret_cast<const unsigned long long*>(t), reinterpret_cast<const unsigned long long*>(h),
        reinterpret_cast<const unsigned long long*>(m), rows, cols, wpr, pad, first);
    BITMM_TRY(launch_check("validate_planes_kernel"));
  }
  int pad_h = 0;
  unsigned long long first_h = 0;
  BITMM_CUDA_TRY(cudaMemcpyAsync(&pad_h, pad, 4, cudaMemcpyDeviceToHost, s));
  BITMM_CUDA_TRY(cudaMemcpyAsync(&first_h, first, 8, cudaMemcpyDeviceToHost, s));
  BITMM_CUDA_TRY(cudaStreamSynchronize(s));
  if (pad_h) return fail(BITMM_ERR_INVALID_ENCODING, "plane padding must be zero");
  if (first_h != ~0ull) {
    static const char* kMsg[4] = {"", "t and h set on the same element", "t requires m",
                                  "h requires m clear"};
    return fail(BITMM_ERR_INVALID_ENCODING, kMsg[first_h & 3]);
  }
  return BITMM_OK;
}

// ---------------- BTSR container -> device ----------------
int bitmm_btsr_read_header(const char* path, bitmm_btsr_header* out) {
  if (!path || !out) return fail(BITMM_ERR_INVALID_ARGUMENT, "null argument");
  BtsrFile bf;
  BtsrHeader h;
  const std::string msg = btsr_open(path, bf, h);
  if (!msg.empty()) return fail(BITMM_ERR_IO, msg);
  out->kind = h.kind;
  out->rows = static_cast<int64_t>(h.rows);
  out->cols = static_cast<int64_t>(h.cols);
  out->words_per_row = static_cast<int64_t>(h.wpr);
  out->nnz = static_cast<int64_t>(h.nnz);
  return BITMM_OK;
}

int bitmm_btsr_load_dev(const char* path, int expected_kind, void* payload, uint64_t* row_ptr,
                        uint64_t* col_idx, float* vals, void* stream) {
  g_launches = 0;
  if (!path) return fail(BITMM_ERR_INVALID_ARGUMENT, "null argument");
  BtsrFile bf;
  BtsrHeader h;
  std::string msg = btsr_open(path, bf, h);
  if (!msg.empty()) return fail(BITMM_ERR_IO, msg);
  static const char* kKindName[3] = {"dense", "bit", "csr"};
  if (expected_kind >= 0 && expected_kind != h.kind)  // tensor_io.cpp load_kind
    return fail(BITMM_ERR_IO, std::string("expected ") + kKindName[expected_kind < 3 ? expected_kind : 0] +
                                  " tensor: " + bf.path);
  if ((h.kind != 2 && h.payload_bytes > 0 && !payload) ||
      (h.kind == 2 && (!row_ptr || (h.nnz > 0 && (!col_idx || !vals)))))
    return fail(BITMM_ERR_INVALID_ARGUMENT, "null destination");
  HostLease st;  // pinned chunks of a host context; the copies run on the caller's stream
  BITMM_TRY(st.acquire());
  for (int i = 0; i < 2; ++i) {
    if (!st->pinned[i]) {
      BITMM_CUDA_TRY(cudaHostAlloc(&st->pinned[i], kBtsrChunk, cudaHostAllocDefault));
      BITMM_CUDA_TRY(cudaEventCreateWithFlags(&st->pinned_ev[i], cudaEventDisableTiming));
    }
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t cerr = cudaSuccess;
  auto done = [&](const std::string& m) -> int {
    if (m == "cuda") return fail(BITMM_ERR_CUDA, std::string("BTSR copy: ") + cudaGetErrorString(cerr));
    if (!m.empty()) return fail(BITMM_ERR_IO, m);
    BITMM_CUDA_TRY(cudaStreamSynchronize(s));  // pinned chunks are reused by the next load
    return BITMM_OK;
  };
  if (h.kind == 0) {  // DenseMatrix(rows, cols, data) rejects non-finite entries
    return done(btsr_stream(bf, static_cast<uint8_t*>(payload), h.payload_bytes, st->pinned,
                            st->pinned_ev, s, [](const uint8_t* p, uint64_t, size_t n) -> std::string {
                              const float* v = reinterpret_cast<const float*>(p);
                              for (size_t i = 0; i < n / 4; ++i)
                                if (!std::isfinite(v[i])) return "dense matrix entries must be finite";
                              return std::string();
                            }, &cerr));
  }
  if (h.kind == 1) {  // BitMatrix::from_words: padding bits must be zero (tensor.cpp:78-89)
    const uint64_t full = h.cols / 64, tail = h.cols % 64;
    const uint64_t keep = tail ? ((uint64_t{1} << tail) - 1) : ~uint64_t{0};
    const uint64_t wpr = h.wpr;
    return done(btsr_stream(bf, static_cast<uint8_t*>(payload), h.payload_bytes, st->pinned,
                            st->pinned_ev, s, [&](const uint8_t* p, uint64_t off, size_t n) -> std::string {
                              const uint64_t* w = reinterpret_cast<const uint64_t*>(p);
                              uint64_t cw = (off / 8) % wpr;
                              for (size_t i = 0; i < n / 8; ++i) {
                                if (cw >= full) {
                                  const uint64_t bad = (cw == full && tail) ? (w[i] & ~keep) : w[i];
                                  if (bad) return "bit matrix padding must be zero";
                                }
                                if (++cw == wpr) cw = 0;
                              }
                              return std::string();
                            }, &cerr));
  }
  // csr: CsrMatrix::validate order (tensor.cpp:104-123): row_ptr, then column indices, values
  std::vector<uint64_t> rp(h.rows + 1);
  if (!bf.read(rp.data(), rp.size() * 8)) return fail(BITMM_ERR_IO, "truncated file: " + bf.path);
  auto csr_fail = [&](const char* what) { return fail(BITMM_ERR_IO, std::string(what) + ": " + bf.path); };
  if (rp[0] != 0) return csr_fail("csr row_ptr must start at 0");
  for (uint64_t r = 0; r < h.rows; ++r)
    if (rp[r] > rp[r + 1]) return csr_fail("csr row_ptr must be monotone");
  if (rp[h.rows] != h.nnz) return csr_fail("csr payload sizes must match nnz");
  BITMM_CUDA_TRY(cudaMemcpyAsync(row_ptr, rp.data(), rp.size() * 8, cudaMemcpyHostToDevice, s));
  uint64_t row = 0, prev = 0;
  const uint64_t cols = h.cols;
  msg = btsr_stream(bf, reinterpret_cast<uint8_t*>(col_idx), h.nnz * 8, st->pinned, st->pinned_ev, s,
                    [&](const uint8_t* p, uint64_t off, size_t n) -> std::string {
                      const uint64_t* c = reinterpret_cast<const uint64_t*>(p);
                      for (size_t j = 0; j < n / 8; ++j) {
                        const uint64_t i = off / 8 + j;
                        while (rp[row + 1] <= i) ++row;
                        if (c[j] >= cols) return "csr column index out of range";
                        if (i > rp[row] && prev >= c[j])
                          return "csr column indices must be strictly increasing per row";
                        prev = c[j];
                      }
                      return std::string();
                    }, &cerr);
  if (!msg.empty()) return done(msg);
  msg = btsr_stream(bf, reinterpret_cast<uint8_t*>(vals), h.nnz * 4, st->pinned, st->pinned_ev, s,
                    [](const uint8_t* p, uint64_t, size_t n) -> std::string {
                      const float* v = reinterpret_cast<const float*>(p);
                      for (size_t i = 0; i < n / 4; ++i)
                        if (!std::isfinite(v[i])) return "csr values must be finite";
                      return std::string();
                    }, &cerr);
  const int rc = done(msg);
  cudaStreamSynchronize(s);  // rp (pageable) must outlive its async copy
  return rc;
}

// ---------------- single-process multi-GPU 1/1 ----------------
// C++ orchestration of the N-sharded GEMM for a process that drives several GPUs itself (the
// reference's callers are C++; shard.py is the one-process-per-GPU form). Output columns (rows
// of b_packed, kernels.hpp:44-46) are split into ndev blocks of whole 32-column groups; A is
// replicated. The only cross-device step is bringing the blocks to the root device: either the
// GEMM epilogue of every device stores its block straight into the root's matrix over peer
// memory (the gather fused into the GEMM), or NCCL send/recv after the compute (loaded with
// dlopen: no link-time NCCL dependency).

}  // extern "C"

namespace {

struct NcclApi {
  bool ok = false;
  ncclResult_t (*commInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*errorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.commInitAll = reinterpret_cast<decltype(a.commInitAll)>(dlsym(h, "ncclCommInitAll"));
    a.commDestroy = reinterpret_cast<decltype(a.commDestroy)>(dlsym(h, "ncclCommDestroy"));
    a.groupStart = reinterpret_cast<decltype(a.groupStart)>(dlsym(h, "ncclGroupStart"));
    a.groupEnd = reinterpret_cast<decltype(a.groupEnd)>(dlsym(h, "ncclGroupEnd"));
    a.send = reinterpret_cast<decltype(a.send)>(dlsym(h, "ncclSend"));
    a.recv = reinterpret_cast<decltype(a.recv)>(dlsym(h, "ncclRecv"));
    a.errorString = reinterpret_cast<decltype(a.errorString)>(dlsym(h, "ncclGetErrorString"));
    a.ok = a.commInitAll && a.commDestroy && a.groupStart && a.groupEnd && a.send && a.recv && a.errorString;
    return a;
  }();
  return api;
}

struct ShardDev {
  int dev = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  uint64_t* a = nullptr;   // replicated A, m x wpr
  uint64_t* b = nullptr;   // this device's b_packed rows, cols x wpr
  int32_t* out = nullptr;  // this device's block, m x cols (NONE / NCCL)
  int32_t* recv = nullptr; // root only, per peer: the received block (NCCL)
  int64_t col0 = 0, cols = 0;
  bool peer = false;       // can store into the root's memory
};

struct ShardPlan {
  int64_t m = 0, n = 0, k = 0, wpr = 0;
  std::vector<ShardDev> d;
  int32_t* full = nullptr;  // the root's m x n matrix
  std::vector<ncclComm_t> comms;
  bool distinct = true;     // every device index different (NCCL and peer access need it)
};

int shard_fail_cleanup(ShardPlan* p);

int with_device(int dev) {
  BITMM_CUDA_TRY(cudaSetDevice(dev));
  return BITMM_OK;
}

// The caller's current device, restored on every return of a plan call (error paths included).
struct DeviceGuard {
  int prev = -1;
  DeviceGuard() {
    if (cudaGetDevice(&prev) != cudaSuccess) {
      prev = -1;
      cudaGetLastError();
    }
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

}  // namespace

extern "C" {

int bitmm_shard_plan_create(const int* devs, int ndev, int64_t m, int64_t n, int64_t k, int64_t wpr, void** plan) {
  if (!devs || ndev < 1 || ndev > kMaxDevices || !plan) return fail(BITMM_ERR_INVALID_ARGUMENT, "bad device list");
  BITMM_TRY(check_gemm_dims(m, n, k, wpr, n));
  if (n < 32 * static_cast<int64_t>(ndev)) return fail(BITMM_ERR_INVALID_ARGUMENT, "fewer than 32 columns per device");
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    return fail(BITMM_ERR_NO_DEVICE, "no CUDA device available (bitmm_b200 has no CPU fallback)");
  }
  DeviceGuard guard;
  auto p = std::make_unique<ShardPlan>();
  p->m = m;
  p->n = n;
  p->k = k;
  p->wpr = wpr;
  p->d.resize(ndev);
  const int64_t groups = (n + 31) / 32;
  int rc = BITMM_OK;
  for (int i = 0; i < ndev && rc == BITMM_OK; ++i) {
    ShardDev& s = p->d[i];
    s.dev = devs[i];
    if (s.dev < 0 || s.dev >= count) {
      rc = fail(BITMM_ERR_INVALID_ARGUMENT, "device index out of range");
      break;
    }
    for (int j = 0; j < i; ++j)
      if (devs[j] == s.dev) p->distinct = false;
    s.col0 = std::min(n, groups * i / ndev * 32);
    s.cols = std::min(n, groups * (i + 1) / ndev * 32) - s.col0;
    auto step = [&]() -> int {
      BITMM_TRY(with_device(s.dev));
      BITMM_CUDA_TRY(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
      BITMM_CUDA_TRY(cudaEventCreate(&s.e0));
      BITMM_CUDA_TRY(cudaEventCreate(&s.e1));
      BITMM_CUDA_TRY(cudaMalloc(&s.a, static_cast<size_t>(m * wpr * 8)));
      BITMM_CUDA_TRY(cudaMalloc(&s.b, static_cast<size_t>(std::max<int64_t>(1, s.cols) * wpr * 8)));
      BITMM_CUDA_TRY(cudaMalloc(&s.out, static_cast<size_t>(m * std::max<int64_t>(1, s.cols) * 4)));
      if (i == 0) BITMM_CUDA_TRY(cudaMalloc(&p->full, static_cast<size_t>(m * n * 4)));
      return BITMM_OK;
    };
    rc = step();
  }
  // the root's staging for NCCL receives, and peer access for the fused gather
  for (int i = 1; i < ndev && rc == BITMM_OK; ++i) {
    ShardDev& s = p->d[i];
    auto step = [&]() -> int {
      BITMM_TRY(with_device(p->d[0].dev));
      BITMM_CUDA_TRY(cudaMalloc(&s.recv, static_cast<size_t>(m * std::max<int64_t>(1, s.cols) * 4)));
      if (s.dev == p->d[0].dev) {
        s.peer = true;  // the same device: the root's matrix is local memory
        return BITMM_OK;
      }
      int can = 0;
      BITMM_CUDA_TRY(cudaDeviceCanAccessPeer(&can, s.dev, p->d[0].dev));
      if (can) {
        BITMM_TRY(with_device(s.dev));
        const cudaError_t e = cudaDeviceEnablePeerAccess(p->d[0].dev, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return fail(BITMM_ERR_CUDA, cudaGetErrorString(e));
        cudaGetLastError();
        s.peer = true;
      }
      return BITMM_OK;
    };
    rc = step();
  }
  p->d[0].peer = true;
  if (rc == BITMM_OK && ndev > 1 && p->distinct && nccl_api().ok) {
    p->comms.resize(ndev);
    std::vector<int> list(devs, devs + ndev);
    const ncclResult_t r = nccl_api().commInitAll(p->comms.data(), ndev, list.data());
    if (r != ncclSuccess) p->comms.clear();  // the NCCL gather is then unavailable
  }
  if (rc != BITMM_OK) {
    shard_fail_cleanup(p.release());  // frees the plan
    return rc;
  }
  *plan = p.release();
  return BITMM_OK;
}

int bitmm_shard_plan_upload(void* plan, const uint64_t* a, const uint64_t* b_packed) {
  auto* p = static_cast<ShardPlan*>(plan);
  if (!p || !a || !b_packed) return fail(BITMM_ERR_INVALID_ARGUMENT, "null operand");
  DeviceGuard guard;
  for (ShardDev& s : p->d) {
    BITMM_TRY(with_device(s.dev));
    BITMM_CUDA_TRY(cudaMemcpyAsync(s.a, a, static_cast<size_t>(p->m * p->wpr * 8), cudaMemcpyHostToDevice, s.stream));
    if (s.cols > 0)
      BITMM_CUDA_TRY(cudaMemcpyAsync(s.b, b_packed + s.col0 * p->wpr, static_cast<size_t>(s.cols * p->wpr * 8),
                                     cudaMemcpyHostToDevice, s.stream));
  }
  for (ShardDev& s : p->d) {
    BITMM_TRY(with_device(s.dev));
    BITMM_CUDA_TRY(cudaStreamSynchronize(s.stream));
  }
  return BITMM_OK;
}

int bitmm_shard_run(void* plan, int gather, double* ms_out) {
  auto* p = static_cast<ShardPlan*>(plan);
  if (!p || gather < BITMM_GATHER_NONE || gather > BITMM_GATHER_NCCL)
    return fail(BITMM_ERR_INVALID_ARGUMENT, "bad plan or gather mode");
  if (gather == BITMM_GATHER_PEER)
    for (const ShardDev& s : p->d)
      if (!s.peer) return fail(BITMM_ERR_CUDA, "peer access to the root device is not available");
  if (gather == BITMM_GATHER_NCCL && p->d.size() > 1 && p->comms.empty())
    return fail(BITMM_ERR_CUDA, "NCCL gather unavailable (needs distinct devices and libnccl.so.2)");
  g_launches = 0;
  DeviceGuard guard;
  const int ndev = static_cast<int>(p->d.size());
  int rc = BITMM_OK;
  // every device's GEMM: its block into its own memory, or (PEER, and always for the root)
  // straight into the root's matrix at its column offset
  for (int i = 0; i < ndev && rc == BITMM_OK; ++i) {
    ShardDev& s = p->d[i];
    auto step = [&]() -> int {
      BITMM_TRY(with_device(s.dev));
      BITMM_CUDA_TRY(cudaEventRecord(s.e0, s.stream));
      if (s.cols > 0) {
        CallCtx st;
        BITMM_TRY(st.acquire(s.stream));
        const bool into_root = gather == BITMM_GATHER_PEER || (i == 0 && gather != BITMM_GATHER_NONE);
        int32_t* out = into_root ? p->full + s.col0 : s.out;
        BITMM_TRY(gemm_1x1_dev_impl(*st, s.a, p->m, s.b, s.cols, p->k, p->wpr, 1.0f, 1.0f, out, nullptr,
                                    into_root ? p->n : s.cols, s.stream));
      }
      return BITMM_OK;
    };
    rc = step();
  }
  if (rc == BITMM_OK && gather == BITMM_GATHER_NCCL && ndev > 1) {
    const NcclApi& nc = nccl_api();
    nc.groupStart();
    for (int i = 1; i < ndev; ++i) {
      ShardDev& s = p->d[i];
      if (s.cols == 0) continue;
      const size_t cnt = static_cast<size_t>(p->m * s.cols);
      nc.send(s.out, cnt, ncclInt32, 0, p->comms[i], s.stream);
      nc.recv(s.recv, cnt, ncclInt32, i, p->comms[0], p->d[0].stream);
    }
    const ncclResult_t r = nc.groupEnd();
    if (r != ncclSuccess) rc = fail(BITMM_ERR_CUDA, std::string("NCCL gather: ") + nc.errorString(r));
    // the root lays every received block out at its columns
    if (rc == BITMM_OK) rc = with_device(p->d[0].dev);
    for (int i = 1; i < ndev && rc == BITMM_OK; ++i) {
      ShardDev& s = p->d[i];
      if (s.cols == 0) continue;
      if (cudaMemcpy2DAsync(p->full + s.col0, p->n * 4, s.recv, s.cols * 4, s.cols * 4, p->m,
                            cudaMemcpyDeviceToDevice, p->d[0].stream) != cudaSuccess)
        rc = fail(BITMM_ERR_CUDA, cudaGetErrorString(cudaGetLastError()));
    }
  }
  // every device's end event; the host waits for all of them below, so the gathered matrix is
  // complete when this call returns (in PEER mode the other devices' epilogues write it)
  for (int i = 0; i < ndev && rc == BITMM_OK; ++i) {
    rc = with_device(p->d[i].dev);
    if (rc == BITMM_OK && cudaEventRecord(p->d[i].e1, p->d[i].stream) != cudaSuccess)
      rc = fail(BITMM_ERR_CUDA, cudaGetErrorString(cudaGetLastError()));
  }
  double ms = 0.0;
  int status = BITMM_OK;
  for (int i = 0; i < ndev; ++i) {
    ShardDev& s = p->d[i];
    if (with_device(s.dev) != BITMM_OK) continue;
    const cudaError_t e = cudaEventSynchronize(s.e1);
    if (e != cudaSuccess && rc == BITMM_OK) rc = fail(BITMM_ERR_CUDA, cudaGetErrorString(e));
    float t = 0.0f;
    if (rc == BITMM_OK && cudaEventElapsedTime(&t, s.e0, s.e1) == cudaSuccess) ms = std::max(ms, static_cast<double>(t));
    if (rc == BITMM_OK && status == BITMM_OK) {
      Ctx* st = nullptr;
      if (stream_ctx(s.stream, &st) == BITMM_OK) status = read_status(*st, s.stream);
    }
  }
  if (rc != BITMM_OK) return rc;
  if (ms_out) *ms_out = ms;
  return status;
}

int bitmm_shard_download(void* plan, int64_t row0, int64_t rows, int32_t* c, int64_t ldc) {
  auto* p = static_cast<ShardPlan*>(plan);
  if (!p || !c || ldc < p->n || row0 < 0 || rows < 0 || row0 + rows > p->m)
    return fail(BITMM_ERR_INVALID_ARGUMENT, "bad plan, rows or output");
  if (rows == 0) return BITMM_OK;
  DeviceGuard guard;
  BITMM_TRY(with_device(p->d[0].dev));
  BITMM_CUDA_TRY(cudaMemcpy2D(c, ldc * 4, p->full + row0 * p->n, p->n * 4, p->n * 4, rows, cudaMemcpyDeviceToHost));
  return BITMM_OK;
}

int bitmm_shard_plan_destroy(void* plan) {
  auto* p = static_cast<ShardPlan*>(plan);
  if (!p) return BITMM_OK;
  shard_fail_cleanup(p);
  return BITMM_OK;
}

}  // extern "C"

namespace {

int shard_fail_cleanup(ShardPlan* p) {
  int prev = 0;
  cudaGetDevice(&prev);
  for (ncclComm_t c : p->comms)
    if (c) nccl_api().commDestroy(c);
  for (ShardDev& s : p->d) {
    if (cudaSetDevice(s.dev) != cudaSuccess) continue;
    if (s.stream) cudaStreamSynchronize(s.stream);
    cudaFree(s.a);
    cudaFree(s.b);
    cudaFree(s.out);
    if (s.recv) {
      cudaSetDevice(p->d[0].dev);
      cudaFree(s.recv);
      cudaSetDevice(s.dev);
    }
    if (s.e0) cudaEventDestroy(s.e0);
    if (s.e1) cudaEventDestroy(s.e1);
    if (s.stream) cudaStreamDestroy(s.stream);
  }
  if (!p->d.empty() && cudaSetDevice(p->d[0].dev) == cudaSuccess) cudaFree(p->full);
  cudaGetLastError();
  cudaSetDevice(prev);
  delete p;
  return BITMM_OK;
}

}  // namespace
