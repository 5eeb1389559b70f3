// pf_runtime.cu — error plumbing, device checks, the fixed fill arena, the bubble
// flag, pinned staging and chain bookkeeping for libpipefill.so.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <mutex>

#include "pf_ops.h"

namespace pf {

static thread_local char g_err[512] = "";

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int check_cuda(cudaError_t err, const char* what) {
  if (err == cudaSuccess) return PF_OK;
  return set_error(err == cudaErrorMemoryAllocation ? PF_ERR_OOM : PF_ERR_CUDA, "%s: %s (%d)", what,
                   cudaGetErrorString(err), (int)err);
}

struct DevInfo {
  int sm_count = 0;
  int major = 0, minor = 0;
};

static DevInfo query_device() {
  DevInfo d;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return d;
  cudaDeviceGetAttribute(&d.sm_count, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&d.major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&d.minor, cudaDevAttrComputeCapabilityMinor, dev);
  return d;
}

static DevInfo& dev_info() {
  // one executor thread per device; cache per current device
  static thread_local int cached_dev = -1;
  static thread_local DevInfo info;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev != cached_dev) {
    info = query_device();
    cached_dev = dev;
  }
  return info;
}

int device_sm_count() {
  int n = dev_info().sm_count;
  return n > 0 ? n : 148;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("PF_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool device_is_sm100() {
  const DevInfo& d = dev_info();
  return d.major == 10 && d.minor == 0;
}

// ---------------------------------------------------------------------------
// small kernels

__global__ void flag_clear_at_kernel(uint32_t* flag, const uint64_t* base, uint64_t offset,
                                     uint64_t* stamp) {
  const uint64_t deadline = (base ? *(volatile const uint64_t*)base : 0ull) + offset;
  uint64_t now;
  do {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (now >= deadline) break;
    __nanosleep(256);
  } while (true);
  if (flag) {
    __threadfence();
    atomicExch(flag, 0u);
  }
  if (stamp) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    *stamp = now;
  }
}

// Throttle an open bubble at a deadline: 1 -> value (only if still 1: a bubble that closed
// meanwhile stays closed).
__global__ void flag_throttle_at_kernel(uint32_t* flag, const uint64_t* base, uint64_t offset,
                                        uint32_t value) {
  const uint64_t deadline = (base ? *(volatile const uint64_t*)base : 0ull) + offset;
  uint64_t now;
  do {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (now >= deadline) break;
    __nanosleep(256);
  } while (true);
  __threadfence();
  atomicCAS(flag, 1u, value);
}

__global__ void globaltimer_kernel(uint64_t* out) {
  uint64_t now;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
  *out = now;
}

// SM clock over a short spin: out[0] = %globaltimer at the start (ns), out[1] = elapsed ns,
// out[2] = elapsed SM cycles (clock64 of the same SM), so MHz = out[2] * 1e3 / out[1]
__global__ void sm_clock_probe_kernel(uint64_t* out, uint64_t spin_ns) {
  uint64_t t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  const long long c0 = clock64();
  do {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  } while (t1 - t0 < spin_ns);
  const long long c1 = clock64();
  out[0] = t0;
  out[1] = t1 - t0;
  out[2] = static_cast<uint64_t>(c1 - c0);
}

__global__ void chain_begin_kernel(uint32_t* cursors, int n, const uint32_t* abort,
                                   unsigned long long* stamps) {
  if (abort && ld_volatile_u32(abort) != 0u) return;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    if (cursors) cursors[i] = 0u;
    if (stamps) {
      stamps[2 * i] = ~0ull;
      stamps[2 * i + 1] = 0ull;
    }
  }
}

__global__ void chain_end_kernel(uint32_t* done, const uint32_t* abort) {
  if (abort && ld_volatile_u32(abort) != 0u) return;
  *done += 1u;
}

constexpr int COPY_THREADS = 256;
constexpr uint64_t COPY_BYTES_PER_CTA = 256 * 1024;

// 2-D copy of `rows` rows x `w16` 16-B words (pitches in 16-B words), flattened
// row-major and split into CTA chunks; atomic preemption unit = one CTA chunk.
__global__ void __launch_bounds__(COPY_THREADS) copy_kernel(uint4* __restrict__ dst, int64_t dpitch,
                                                            const uint4* __restrict__ src,
                                                            int64_t spitch, int64_t w16,
                                                            uint64_t n16, Ctl ctl,
                                                            const int64_t* desc,
                                                            const uint32_t* idx, int role) {
  pdl_enter();
  __shared__ int s_go;
  if (threadIdx.x == 0) {
    int go = 1;
    if (chain_aborted(ctl)) go = 0;
    else if (ctl.flag != nullptr && ld_acquire_u32(ctl.flag) == 0u) {
      atomicExch(ctl.abort, 1u);
      go = 0;
    }
    s_go = go;
  }
  __syncthreads();
  if (!s_go) return;
  if (desc != nullptr && role != 0) {  // batch slice offset chosen on the device
    const int64_t off = desc[PF_DESC_WORDS * (int64_t)ld_volatile_u32(idx) + role - 1];
    if (role != 2) src = reinterpret_cast<const uint4*>(reinterpret_cast<const uint8_t*>(src) + off);
    else dst = reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(dst) + off);
  }
  const uint64_t per = COPY_BYTES_PER_CTA / 16;
  const uint64_t lo = (uint64_t)blockIdx.x * per;
  const uint64_t hi = lo + per < n16 ? lo + per : n16;
  constexpr int U = 4;
  uint64_t i = lo + threadIdx.x;
  if (dpitch == w16 && spitch == w16) {
    for (; i + (U - 1) * COPY_THREADS < hi; i += U * COPY_THREADS) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = src[i + u * COPY_THREADS];
#pragma unroll
      for (int u = 0; u < U; ++u) dst[i + u * COPY_THREADS] = v[u];
    }
    for (; i < hi; i += COPY_THREADS) dst[i] = src[i];
  } else {
    for (; i < hi; i += COPY_THREADS) {
      const uint64_t r = i / (uint64_t)w16, c = i % (uint64_t)w16;
      dst[r * dpitch + c] = src[r * spitch + c];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && ctl.cursor != nullptr) {
    __threadfence_system();
    atomicAdd(ctl.cursor, 1u);
  }
}

struct CopyOp final : PreparedOp {
  uint8_t* dst = nullptr;
  const uint8_t* src = nullptr;
  int64_t dpitch = 0, spitch = 0, width = 0, rows = 0;
  int role = 0;
  uint64_t n16() const { return (uint64_t)(width / 16) * (uint64_t)rows; }
  uint32_t units() const override {
    return (uint32_t)((n16() * 16 + COPY_BYTES_PER_CTA - 1) / COPY_BYTES_PER_CTA);
  }
  bool resumable() const override { return false; }
  int run(const pf_ctl_t* ctl, cudaStream_t s, const LaunchArgs& a) override {
    const bool dev = a.desc != nullptr && role != 0;
    const uint8_t* sp = src + (role == 1 && !dev ? a.in_off : 0);
    uint8_t* dp = dst + (role == 2 && !dev ? a.out_off : 0);
    if (n16() == 0) return PF_OK;
    PF_CUDA(launch_pdl(copy_kernel, dim3(units()), dim3(COPY_THREADS), 0, s,
                       reinterpret_cast<uint4*>(dp), dpitch / 16, reinterpret_cast<const uint4*>(sp),
                       spitch / 16, width / 16, n16(), make_ctl(ctl), dev ? a.desc : nullptr, a.idx,
                       role));
    return PF_OK;
  }
};

int make_copy_op(OpPtr* out, void* dst, int64_t dst_pitch, const void* src, int64_t src_pitch,
                 int64_t width, int64_t rows, int role) {
  if (!dst || !src || width < 0 || rows < 0 || role < 0 || role > 3)
    return set_error(PF_ERR_INVALID, "pf_copy: bad arguments");
  if ((width | dst_pitch | src_pitch) & 15 || (((uintptr_t)dst | (uintptr_t)src) & 15u))
    return set_error(PF_ERR_INVALID, "pf_copy: sizes, pitches and pointers must be 16-B aligned");
  auto op = std::make_unique<CopyOp>();
  op->dst = static_cast<uint8_t*>(dst);
  op->src = static_cast<const uint8_t*>(src);
  op->dpitch = dst_pitch;
  op->spitch = src_pitch;
  op->width = width;
  op->rows = rows;
  op->role = role;
  *out = std::move(op);
  return PF_OK;
}

__global__ void flag_write_kernel(uint32_t* flag, uint32_t v) {
  __threadfence();
  atomicExch(flag, v);
}

typedef CUresult (*StreamWriteValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

static StreamWriteValue32Fn get_write_value_fn() {
  static StreamWriteValue32Fn fn = nullptr;
  static bool probed = false;
  if (!probed) {
    probed = true;
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<StreamWriteValue32Fn>(ptr);
  }
  return fn;
}

}  // namespace pf

// ---------------------------------------------------------------------------
// C ABI

struct pf_arena {
  void* base = nullptr;
  uint64_t capacity = 0;
  uint64_t used = 0;
  uint64_t high_water = 0;
};

extern "C" {

int pf_abi_version(void) { return PF_ABI_VERSION; }

const char* pf_last_error(void) { return pf::g_err; }

int pf_device_check(int* sm_count_out) {
  using namespace pf;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) return set_error(PF_ERR_UNSUPPORTED, "no CUDA device visible");
  if (!device_is_sm100())
    return set_error(PF_ERR_UNSUPPORTED, "device is sm_%d%d, libpipefill needs sm_100 (B200)",
                     dev_info().major, dev_info().minor);
  if (sm_count_out) *sm_count_out = device_sm_count();
  return PF_OK;
}

// ---- arena ----------------------------------------------------------------

int pf_arena_create(uint64_t bytes, pf_arena_t** out) {
  using namespace pf;
  if (!out || bytes == 0) return set_error(PF_ERR_INVALID, "pf_arena_create: bad arguments");
  pf_arena* a = new pf_arena();
  cudaError_t e = cudaMalloc(&a->base, bytes);
  if (e != cudaSuccess) {
    delete a;
    cudaGetLastError();
    return check_cuda(e, "pf_arena_create cudaMalloc");
  }
  a->capacity = bytes;
  *out = a;
  return PF_OK;
}

int pf_arena_alloc(pf_arena_t* a, uint64_t bytes, uint64_t align, void** out) {
  using namespace pf;
  if (!a || !out) return set_error(PF_ERR_INVALID, "pf_arena_alloc: bad arguments");
  if (align == 0) align = 256;
  if (align & (align - 1)) return set_error(PF_ERR_INVALID, "pf_arena_alloc: align not a power of 2");
  uint64_t off = (a->used + align - 1) & ~(align - 1);
  if (off + bytes > a->capacity)
    return set_error(PF_ERR_OOM,
                     "pf_arena_alloc: %llu B requested, %llu B of %llu B arena left",
                     (unsigned long long)bytes, (unsigned long long)(a->capacity - a->used),
                     (unsigned long long)a->capacity);
  *out = static_cast<uint8_t*>(a->base) + off;
  a->used = off + bytes;
  if (a->used > a->high_water) a->high_water = a->used;
  return PF_OK;
}

int pf_arena_mark(pf_arena_t* a, uint64_t* out_mark) {
  if (!a || !out_mark) return pf::set_error(PF_ERR_INVALID, "pf_arena_mark: bad arguments");
  *out_mark = a->used;
  return PF_OK;
}

int pf_arena_release(pf_arena_t* a, uint64_t mark) {
  if (!a || mark > a->used) return pf::set_error(PF_ERR_INVALID, "pf_arena_release: bad mark");
  a->used = mark;
  return PF_OK;
}

int pf_arena_reset(pf_arena_t* a) {
  if (!a) return pf::set_error(PF_ERR_INVALID, "pf_arena_reset: null arena");
  a->used = 0;
  return PF_OK;
}

int pf_arena_stats(pf_arena_t* a, uint64_t* capacity, uint64_t* used, uint64_t* high_water) {
  if (!a) return pf::set_error(PF_ERR_INVALID, "pf_arena_stats: null arena");
  if (capacity) *capacity = a->capacity;
  if (used) *used = a->used;
  if (high_water) *high_water = a->high_water;
  return PF_OK;
}

int pf_arena_base(pf_arena_t* a, void** out) {
  if (!a || !out) return pf::set_error(PF_ERR_INVALID, "pf_arena_base: bad arguments");
  *out = a->base;
  return PF_OK;
}

int pf_arena_destroy(pf_arena_t* a) {
  if (!a) return PF_OK;
  cudaError_t e = cudaFree(a->base);
  delete a;
  return pf::check_cuda(e, "pf_arena_destroy cudaFree");
}

// ---- flag -------------------------------------------------------------------

int pf_flag_create(uint32_t** out) {
  using namespace pf;
  if (!out) return set_error(PF_ERR_INVALID, "pf_flag_create: null out");
  void* p = nullptr;
  PF_CUDA(cudaMalloc(&p, 64));  // own 64-B line
  PF_CUDA(cudaMemset(p, 0, 64));
  *out = static_cast<uint32_t*>(p);
  return PF_OK;
}

int pf_flag_destroy(uint32_t* flag) {
  if (!flag) return PF_OK;
  return pf::check_cuda(cudaFree(flag), "pf_flag_destroy");
}

int pf_flag_write_on_stream(uint32_t* flag, uint32_t value, void* stream) {
  using namespace pf;
  if (!flag) return set_error(PF_ERR_INVALID, "pf_flag_write_on_stream: null flag");
  StreamWriteValue32Fn fn = get_write_value_fn();
  if (fn) {
    CUresult r = fn(reinterpret_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(flag), value,
                    0 /*CU_STREAM_WRITE_VALUE_DEFAULT*/);
    if (r == CUDA_SUCCESS) return PF_OK;
  }
  // stream memory operations unavailable: a one-thread kernel keeps stream order
  flag_write_kernel<<<1, 1, 0, reinterpret_cast<cudaStream_t>(stream)>>>(flag, value);
  PF_CUDA(cudaGetLastError());
  return PF_OK;
}

int pf_flag_clear_at(uint32_t* flag, const uint64_t* base_ns, uint64_t offset_ns,
                     uint64_t* stamp_out, void* stream) {
  using namespace pf;
  flag_clear_at_kernel<<<1, 1, 0, reinterpret_cast<cudaStream_t>(stream)>>>(flag, base_ns,
                                                                            offset_ns, stamp_out);
  PF_CUDA(cudaGetLastError());
  return PF_OK;
}

int pf_flag_throttle_at(uint32_t* flag, const uint64_t* base_ns, uint64_t offset_ns, uint32_t value,
                        void* stream) {
  using namespace pf;
  if (!flag || value < 2u) return set_error(PF_ERR_INVALID, "pf_flag_throttle_at: null flag or value < 2");
  flag_throttle_at_kernel<<<1, 1, 0, reinterpret_cast<cudaStream_t>(stream)>>>(flag, base_ns, offset_ns,
                                                                               value);
  PF_CUDA(cudaGetLastError());
  return PF_OK;
}

int pf_wait_until(const uint64_t* base_ns, uint64_t offset_ns, uint64_t* stamp_out,
                  void* stream) {
  return pf_flag_clear_at(nullptr, base_ns, offset_ns, stamp_out, stream);
}

int pf_read_globaltimer(uint64_t* dev_out, void* stream) {
  using namespace pf;
  if (!dev_out) return set_error(PF_ERR_INVALID, "pf_read_globaltimer: null out");
  globaltimer_kernel<<<1, 1, 0, reinterpret_cast<cudaStream_t>(stream)>>>(dev_out);
  PF_CUDA(cudaGetLastError());
  return PF_OK;
}

int pf_sm_clock_probe(uint64_t* dev_out3, uint64_t spin_ns, void* stream) {
  using namespace pf;
  if (!dev_out3 || spin_ns == 0 || spin_ns > 10000000ull)
    return set_error(PF_ERR_INVALID, "pf_sm_clock_probe: null out or spin outside (0, 10 ms]");
  sm_clock_probe_kernel<<<1, 1, 0, reinterpret_cast<cudaStream_t>(stream)>>>(dev_out3, spin_ns);
  PF_CUDA(cudaGetLastError());
  return PF_OK;
}

// ---- staging ------------------------------------------------------------------

int pf_host_alloc_pinned(uint64_t bytes, void** out) {
  using namespace pf;
  if (!out || bytes == 0) return set_error(PF_ERR_INVALID, "pf_host_alloc_pinned: bad arguments");
  PF_CUDA(cudaHostAlloc(out, bytes, cudaHostAllocPortable | cudaHostAllocMapped));
  return PF_OK;
}

int pf_host_free_pinned(void* p) {
  if (!p) return PF_OK;
  return pf::check_cuda(cudaFreeHost(p), "pf_host_free_pinned");
}

int pf_stage_h2d(void* dst, const void* src, uint64_t bytes, void* stream) {
  using namespace pf;
  if (!dst || !src) return set_error(PF_ERR_INVALID, "pf_stage_h2d: null pointer");
  PF_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice,
                          reinterpret_cast<cudaStream_t>(stream)));
  return PF_OK;
}

int pf_stage_d2h(void* dst, const void* src, uint64_t bytes, void* stream) {
  using namespace pf;
  if (!dst || !src) return set_error(PF_ERR_INVALID, "pf_stage_d2h: null pointer");
  PF_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost,
                          reinterpret_cast<cudaStream_t>(stream)));
  return PF_OK;
}

int pf_copy_units(uint64_t bytes, uint32_t* out) {
  using namespace pf;
  if (!out) return set_error(PF_ERR_INVALID, "pf_copy_units: null out");
  *out = (uint32_t)((bytes + COPY_BYTES_PER_CTA - 1) / COPY_BYTES_PER_CTA);
  return PF_OK;
}

int pf_copy(void* dst, const void* src, uint64_t bytes, const pf_ctl_t* ctl, void* stream) {
  using namespace pf;
  PF_TRY(validate_ctl(ctl));
  OpPtr op;
  PF_TRY(make_copy_op(&op, dst, (int64_t)bytes, src, (int64_t)bytes, (int64_t)bytes, 1, 0));
  return op->run(ctl, reinterpret_cast<cudaStream_t>(stream), pf::LaunchArgs{});
}

int pf_copy2d(void* dst, int64_t dst_pitch, const void* src, int64_t src_pitch, int64_t width,
              int64_t rows, const pf_ctl_t* ctl, void* stream) {
  using namespace pf;
  PF_TRY(validate_ctl(ctl));
  OpPtr op;
  PF_TRY(make_copy_op(&op, dst, dst_pitch, src, src_pitch, width, rows, 0));
  return op->run(ctl, reinterpret_cast<cudaStream_t>(stream), pf::LaunchArgs{});
}

// ---- chain ----------------------------------------------------------------------

int pf_chain_begin(uint32_t* cursors, int n, const uint32_t* abort, void* stream) {
  using namespace pf;
  if (!cursors || n <= 0) return set_error(PF_ERR_INVALID, "pf_chain_begin: bad arguments");
  chain_begin_kernel<<<1, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(cursors, n, abort,
                                                                             nullptr);
  PF_CUDA(cudaGetLastError());
  return PF_OK;
}

int pf_chain_end(uint32_t* done, const uint32_t* abort, void* stream) {
  using namespace pf;
  if (!done) return set_error(PF_ERR_INVALID, "pf_chain_end: null counter");
  chain_end_kernel<<<1, 1, 0, reinterpret_cast<cudaStream_t>(stream)>>>(done, abort);
  PF_CUDA(cudaGetLastError());
  return PF_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// recorded launch chains: one batch of one partition of the fill model

#include <vector>

struct pf_chain {
  std::vector<pf::OpPtr> nodes;
  bool timing = false;
  std::vector<cudaEvent_t> ev;  // 2 per node when timing is on
  const int64_t* desc = nullptr;  // device batch-slice offsets (see LaunchArgs)
  unsigned long long* stamps = nullptr;  // device [start, end] per node (in-kernel timing)
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  ~pf_chain() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
  }
};

namespace pf {
// Segment gate of a chain graph: the following conditional IF body (one module's
// kernels) runs only while the chain is live and the bubble is open. A closed bubble
// sets the sticky abort, so every later gate and the chain-end marker see it.
__global__ void chain_gate_kernel(cudaGraphConditionalHandle h, const uint32_t* flag,
                                  uint32_t* abort) {
  unsigned go = 1u;
  if (abort != nullptr && ld_volatile_u32(abort) != 0u) {
    go = 0u;
  } else if (flag != nullptr && ld_acquire_u32(flag) == 0u) {
    atomicExch(abort, 1u);
    go = 0u;
  }
  cudaGraphSetConditional(h, go);
}
// Gate of a run-ahead staging: copy only when no earlier batch on the stream yielded.
__global__ void staging_gate_kernel(cudaGraphConditionalHandle h, const uint32_t* abort,
                                    uint32_t* staged_out) {
  const unsigned go = ld_volatile_u32(abort) == 0u ? 1u : 0u;
  *staged_out = go;
  cudaGraphSetConditional(h, go);
}
}  // namespace pf

struct pf_staging {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
};

extern "C" {

int pf_staging_create(pf_staging_t** out, void* const* dst, const void* const* src,
                      const uint64_t* bytes, int n, const uint32_t* abort, uint32_t* staged_out) {
  using namespace pf;
  if (!out || n < 0 || (n > 0 && (!dst || !src || !bytes)) || !abort || !staged_out)
    return set_error(PF_ERR_INVALID, "pf_staging_create: bad arguments");
  cudaGraph_t g;
  PF_CUDA(cudaGraphCreate(&g, 0));
  int rc = PF_OK;
  do {
    cudaGraphConditionalHandle h;
    if ((rc = check_cuda(cudaGraphConditionalHandleCreate(&h, g, 0, cudaGraphCondAssignDefault),
                         "cudaGraphConditionalHandleCreate")) != PF_OK)
      break;
    const uint32_t* ab = abort;
    uint32_t* so = staged_out;
    void* args[] = {&h, &ab, &so};
    cudaKernelNodeParams kp = {};
    kp.func = (void*)staging_gate_kernel;
    kp.gridDim = dim3(1);
    kp.blockDim = dim3(1);
    kp.kernelParams = args;
    cudaGraphNode_t gate;
    if ((rc = check_cuda(cudaGraphAddKernelNode(&gate, g, nullptr, 0, &kp), "gate node")) != PF_OK) break;
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeIf;
    cp.conditional.size = 1;
    cudaGraphNode_t cn;
    if ((rc = check_cuda(cudaGraphAddNode(&cn, g, &gate, 1, &cp), "cudaGraphAddNode(cond)")) != PF_OK)
      break;
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    cudaGraphNode_t prev = nullptr;
    for (int i = 0; i < n && rc == PF_OK; ++i) {
      if (bytes[i] == 0) continue;
      cudaGraphNode_t nd;
      rc = check_cuda(cudaGraphAddMemcpyNode1D(&nd, body, prev ? &prev : nullptr, prev ? 1 : 0, dst[i],
                                               src[i], (size_t)bytes[i], cudaMemcpyDefault),
                      "cudaGraphAddMemcpyNode1D (conditional body)");
      prev = nd;
    }
    if (rc != PF_OK) break;
    auto* st = new pf_staging();
    st->graph = g;
    if ((rc = check_cuda(cudaGraphInstantiate(&st->exec, g, 0), "cudaGraphInstantiate(staging)")) != PF_OK) {
      delete st;
      break;
    }
    *out = st;
    return PF_OK;
  } while (false);
  cudaGraphDestroy(g);
  return rc;
}

int pf_staging_launch(pf_staging_t* st, void* stream) {
  using namespace pf;
  if (!st || !st->exec) return set_error(PF_ERR_INVALID, "pf_staging_launch: null staging");
  PF_CUDA(cudaGraphLaunch(st->exec, reinterpret_cast<cudaStream_t>(stream)));
  return PF_OK;
}

int pf_staging_destroy(pf_staging_t* st) {
  if (!st) return PF_OK;
  if (st->exec) cudaGraphExecDestroy(st->exec);
  if (st->graph) cudaGraphDestroy(st->graph);
  delete st;
  return PF_OK;
}

int pf_chain_create(pf_chain_t** out) {
  if (!out) return pf::set_error(PF_ERR_INVALID, "pf_chain_create: null out");
  *out = new pf_chain();
  return PF_OK;
}

int pf_chain_destroy(pf_chain_t* c) {
  delete c;
  return PF_OK;
}

static int chain_push(pf_chain_t* c, int rc, pf::OpPtr& op) {
  if (rc != PF_OK) return rc;
  c->nodes.push_back(std::move(op));
  return PF_OK;
}

int pf_chain_add_gemm(pf_chain_t* c, const void* X, const void* W, const void* bias,
                      const void* residual, void* Y, int M, int N, int K, uint32_t epilogue) {
  if (!c) return pf::set_error(PF_ERR_INVALID, "null chain");
  pf::OpPtr op;
  return chain_push(c, pf::make_gemm_op(&op, X, W, bias, residual, Y, M, N, K, epilogue), op);
}

int pf_chain_add_layernorm(pf_chain_t* c, const void* X, const void* residual, const void* gamma,
                           const void* beta, void* Y, int rows, int cols, float eps) {
  if (!c) return pf::set_error(PF_ERR_INVALID, "null chain");
  pf::OpPtr op;
  return chain_push(c, pf::make_norm_op(&op, false, X, residual, gamma, beta, Y, rows, cols, eps), op);
}

int pf_chain_add_rmsnorm(pf_chain_t* c, const void* X, const void* residual, const void* gamma,
                         void* Y, int rows, int cols, float eps) {
  if (!c) return pf::set_error(PF_ERR_INVALID, "null chain");
  pf::OpPtr op;
  return chain_push(c, pf::make_norm_op(&op, true, X, residual, gamma, nullptr, Y, rows, cols, eps), op);
}

int pf_chain_add_softmax(pf_chain_t* c, const void* X, void* Y, int rows, int cols, float scale) {
  if (!c) return pf::set_error(PF_ERR_INVALID, "null chain");
  pf::OpPtr op;
  return chain_push(c, pf::make_softmax_op(&op, X, Y, rows, cols, scale), op);
}

int pf_chain_add_gemm_splitk(pf_chain_t* c, const void* X, const void* W, void* Y, int M, int N, int K,
                             int splits) {
  if (!c) return pf::set_error(PF_ERR_INVALID, "null chain");
  pf::OpPtr op;
  return chain_push(c, pf::make_gemm_splitk_op(&op, X, W, Y, M, N, K, splits), op);
}

#define PF_CHAIN_ADD(MAKE)                          \
  do {                                              \
    if (!c) return pf::set_error(PF_ERR_INVALID, "null chain"); \
    pf::OpPtr op;                                   \
    return chain_push(c, MAKE, op);                 \
  } while (0)

int pf_chain_add_gemm_f32(pf_chain_t* c, const float* X, const float* W, const float* bias, const float* residual,
                          float* Y, int M, int N, int K, uint32_t epilogue) {
  PF_CHAIN_ADD(pf::make_sgemm_op(&op, X, W, bias, residual, Y, M, N, K, epilogue));
}
int pf_chain_add_layernorm_f32(pf_chain_t* c, const float* X, const float* residual, const float* gamma,
                               const float* beta, float* Y, int rows, int cols, float eps) {
  PF_CHAIN_ADD(pf::make_layernorm_f32_op(&op, X, residual, gamma, beta, Y, rows, cols, eps));
}
int pf_chain_add_embedding_ln_f32(pf_chain_t* c, const int32_t* ids, const float* word, const float* pos,
                                  const float* type, const float* gamma, const float* beta, float* Y, int batch,
                                  int seq, int hidden, int vocab, float eps) {
  PF_CHAIN_ADD(pf::make_embedding_ln_f32_op(&op, ids, word, pos, type, gamma, beta, Y, batch, seq, hidden, vocab, eps));
}
int pf_chain_add_attention_f32(pf_chain_t* c, const float* QKV, float* O, int batch, int seq, int heads,
                               int head_dim, float scale) {
  PF_CHAIN_ADD(pf::make_attention_f32_op(&op, QKV, O, batch, seq, heads, head_dim, scale));
}

int pf_chain_add_colstats(pf_chain_t* c, const void* X, const void* G, const void* Ymask, const float* mean,
                          const float* invstd, float* partial, int M, int C, int* out_partials) {
  PF_CHAIN_ADD(pf::make_colstats_op(&op, X, G, Ymask, mean, invstd, partial, M, C, out_partials));
}
int pf_chain_add_bn_finalize(pf_chain_t* c, const float* partial, int P, int M, int C, const float* gamma,
                             const float* beta, float eps, float* mean, float* invstd, float* scale,
                             float* shift) {
  PF_CHAIN_ADD(pf::make_bn_finalize_op(&op, partial, P, M, C, gamma, beta, eps, mean, invstd, scale, shift));
}
int pf_chain_add_bn_bwd_finalize(pf_chain_t* c, const float* partial, int P, int C, float* dgamma,
                                 float* dbeta) {
  PF_CHAIN_ADD(pf::make_bn_bwd_finalize_op(&op, partial, P, C, dgamma, dbeta));
}
int pf_chain_add_bn_apply(pf_chain_t* c, const void* X, const float* scale, const float* shift, const void* R,
                          void* Y, long long M, int C, int relu) {
  PF_CHAIN_ADD(pf::make_bn_apply_op(&op, X, scale, shift, R, Y, M, C, relu));
}
int pf_chain_add_bn_bwd_apply(pf_chain_t* c, const void* X, const void* G, const void* Ymask, const float* mean,
                              const float* invstd, const float* gamma, const float* dgamma, const float* dbeta,
                              void* dX, void* dA, int M, int C) {
  PF_CHAIN_ADD(pf::make_bn_bwd_apply_op(&op, X, G, Ymask, mean, invstd, gamma, dgamma, dbeta, dX, dA, M, C));
}
int pf_chain_add_transpose(pf_chain_t* c, const void* X, void* Y, int R, int C) {
  PF_CHAIN_ADD(pf::make_transpose_op(&op, X, Y, R, C));
}
int pf_chain_add_col2im(pf_chain_t* c, const void* dCol, const void* R, void* dX, int B, int H, int W, int C,
                        int kh, int kw, int stride, int pad, int Kp) {
  PF_CHAIN_ADD(pf::make_col2im_op(&op, dCol, R, dX, B, H, W, C, kh, kw, stride, pad, Kp));
}
int pf_chain_add_maxpool_bwd(pf_chain_t* c, const void* X, const void* dY, void* dX, int B, int H, int W, int C,
                             int k, int stride, int pad) {
  PF_CHAIN_ADD(pf::make_maxpool_bwd_op(&op, X, dY, dX, B, H, W, C, k, stride, pad));
}
int pf_chain_add_maxpool_bwd_argmax(pf_chain_t* c, const uint8_t* Idx, const void* dY, void* dX, int B, int H,
                                    int W, int C, int k, int stride, int pad) {
  PF_CHAIN_ADD(pf::make_maxpool_bwd_idx_op(&op, Idx, dY, dX, B, H, W, C, k, stride, pad));
}
int pf_chain_add_avgpool_bwd(pf_chain_t* c, const void* dY, void* dX, int B, int HW, int C) {
  PF_CHAIN_ADD(pf::make_avgpool_bwd_op(&op, dY, dX, B, HW, C));
}
int pf_chain_add_softmax_xent(pf_chain_t* c, const void* Z, const int32_t* labels, float* loss, void* dZ, int B,
                              int N, float grad_scale) {
  PF_CHAIN_ADD(pf::make_xent_op(&op, Z, labels, loss, dZ, B, N, grad_scale));
}
int pf_chain_add_sgd(pf_chain_t* c, const pf_sgd_segment_t* segs, int nseg, float lr, float momentum) {
  PF_CHAIN_ADD(pf::make_sgd_op(&op, segs, nseg, lr, momentum));
}

int pf_chain_add_gemm_nn(pf_chain_t* c, const void* X, const void* Wkn, const void* residual, void* Y, int M,
                         int N, int K) {
  if (!c) return pf::set_error(PF_ERR_INVALID, "null chain");
  pf::OpPtr op;
  return chain_push(c, pf::make_gemm_mn_op(&op, X, Wkn, residual, Y, M, N, K, 2, 1), op);
}

int pf_chain_add_gemm_splitk_tn(pf_chain_t* c, const void* A, const void* B, void* Y, int M, int N, int K,
                                int splits) {
  if (!c) return pf::set_error(PF_ERR_INVALID, "null chain");
  pf::OpPtr op;
  return chain_push(c, pf::make_gemm_mn_op(&op, A, B, nullptr, Y, M, N, K, 3, splits), op);
}

int pf_chain_add_im2col(pf_chain_t* c, const void* X, void* Col, int B, int H, int W, int C, int kh,
                        int kw, int stride, int pad, int Kp) {
  if (!c) return pf::set_error(PF_ERR_INVALID, "null chain");
  pf::OpPtr op;
  return chain_push(c, pf::make_im2col_op(&op, X, Col, B, H, W, C, kh, kw, stride, pad, Kp), op);
}

int pf_chain_add_maxpool(pf_chain_t* c, const void* X, void* Y, int B, int H, int W, int C, int k,
                         int stride, int pad) {
  if (!c) return pf::set_error(PF_ERR_INVALID, "null chain");
  pf::OpPtr op;
  return chain_push(c, pf::make_maxpool_op(&op, X, Y, B, H, W, C, k, stride, pad), op);
}

int pf_chain_add_maxpool_argmax(pf_chain_t* c, const void* X, void* Y, uint8_t* Idx, int B, int H, int W, int C,
                                int k, int stride, int pad) {
  if (!c) return pf::set_error(PF_ERR_INVALID, "null chain");
  if (!Idx) return pf::set_error(PF_ERR_INVALID, "pf_chain_add_maxpool_argmax: null index buffer");
  pf::OpPtr op;
  return chain_push(c, pf::make_maxpool_op(&op, X, Y, B, H, W, C, k, stride, pad, Idx), op);
}

int pf_chain_add_avgpool(pf_chain_t* c, const void* X, void* Y, int B, int HW, int C) {
  if (!c) return pf::set_error(PF_ERR_INVALID, "null chain");
  pf::OpPtr op;
  return chain_push(c, pf::make_avgpool_op(&op, X, Y, B, HW, C), op);
}

int pf_chain_add_attention(pf_chain_t* c, const void* QKV, const float* mask_add, void* O,
                           int batch, int seq, int heads, int head_dim, float scale) {
  if (!c) return pf::set_error(PF_ERR_INVALID, "null chain");
  pf::OpPtr op;
  return chain_push(
      c, pf::make_attention_op(&op, QKV, mask_add, O, batch, seq, heads, head_dim, scale), op);
}

int pf_chain_add_embedding_ln(pf_chain_t* c, const int32_t* ids, const int32_t* type_ids,
                              const void* word, const void* pos, const void* type,
                              const void* gamma, const void* beta, void* Y, int batch, int seq,
                              int hidden, int vocab, float eps) {
  if (!c) return pf::set_error(PF_ERR_INVALID, "null chain");
  pf::OpPtr op;
  return chain_push(c,
                    pf::make_embedding_op(&op, ids, type_ids, word, pos, type, gamma, beta, Y,
                                          batch, seq, hidden, vocab, eps),
                    op);
}

int pf_chain_add_copy(pf_chain_t* c, void* dst, int64_t dst_pitch, const void* src,
                      int64_t src_pitch, int64_t width, int64_t rows, int role) {
  if (!c) return pf::set_error(PF_ERR_INVALID, "null chain");
  pf::OpPtr op;
  return chain_push(c, pf::make_copy_op(&op, dst, dst_pitch, src, src_pitch, width, rows, role), op);
}

int pf_chain_size(pf_chain_t* c, int* n) {
  if (!c || !n) return pf::set_error(PF_ERR_INVALID, "pf_chain_size: bad arguments");
  *n = (int)c->nodes.size();
  return PF_OK;
}

int pf_chain_node_info(pf_chain_t* c, int node, uint32_t* units, int* resumable) {
  if (!c || node < 0 || node >= (int)c->nodes.size())
    return pf::set_error(PF_ERR_INVALID, "pf_chain_node_info: bad node");
  if (units) *units = c->nodes[node]->units();
  if (resumable) *resumable = c->nodes[node]->resumable() ? 1 : 0;
  return PF_OK;
}

int pf_chain_set_stamps(pf_chain_t* c, uint64_t* stamps) {
  if (!c) return pf::set_error(PF_ERR_INVALID, "null chain");
  c->stamps = reinterpret_cast<unsigned long long*>(stamps);
  return PF_OK;
}

int pf_chain_set_desc(pf_chain_t* c, const int64_t* desc) {
  if (!c) return pf::set_error(PF_ERR_INVALID, "null chain");
  c->desc = desc;
  return PF_OK;
}

// Record the chain as a CUDA graph: chain-begin marker, then per segment a gate kernel
// and a conditional IF node whose body is the segment's kernels (stream-captured),
// then the chain-end marker. A batch whose bubble closed costs one gate launch per
// remaining segment instead of one kernel launch per remaining node.
int pf_chain_build_graph(pf_chain_t* c, const uint32_t* flag, uint32_t* abort, uint32_t* cursors,
                         uint32_t* done, const int* seg_ends, int n_segs) {
  using namespace pf;
  if (!c || !seg_ends || n_segs <= 0) return set_error(PF_ERR_INVALID, "pf_chain_build_graph: bad arguments");
  const int n = (int)c->nodes.size();
  if (seg_ends[n_segs - 1] != n) return set_error(PF_ERR_INVALID, "segments must end at the chain size");
  if (flag && (!abort || !cursors)) return set_error(PF_ERR_INVALID, "preemptible graph needs abort and cursors");
  if (c->exec) {
    cudaGraphExecDestroy(c->exec);
    c->exec = nullptr;
  }
  if (c->graph) {
    cudaGraphDestroy(c->graph);
    c->graph = nullptr;
  }
  cudaGraph_t g;
  PF_CUDA(cudaGraphCreate(&g, 0));
  cudaStream_t cap;
  PF_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
  int rc = PF_OK;
  cudaGraphNode_t prev = nullptr;
  auto add_kernel = [&](void* fn, dim3 grid, dim3 block, void** args) -> int {
    cudaKernelNodeParams kp = {};
    kp.func = fn;
    kp.gridDim = grid;
    kp.blockDim = block;
    kp.sharedMemBytes = 0;
    kp.kernelParams = args;
    cudaGraphNode_t nd;
    PF_CUDA(cudaGraphAddKernelNode(&nd, g, prev ? &prev : nullptr, prev ? 1 : 0, &kp));
    prev = nd;
    return PF_OK;
  };
  do {
    if (cursors || c->stamps) {
      uint32_t* cur = cursors;
      int nn = n;
      const uint32_t* ab = abort;
      unsigned long long* st = c->stamps;
      void* args[] = {&cur, &nn, &ab, &st};
      if ((rc = add_kernel((void*)chain_begin_kernel, dim3(1), dim3(128), args)) != PF_OK) break;
    }
    int lo = 0;
    for (int sgi = 0; sgi < n_segs && rc == PF_OK; ++sgi) {
      const int hi = seg_ends[sgi];
      cudaGraphConditionalHandle h;
      if ((rc = check_cuda(cudaGraphConditionalHandleCreate(&h, g, 0, cudaGraphCondAssignDefault),
                           "cudaGraphConditionalHandleCreate")) != PF_OK)
        break;
      const uint32_t* fl = flag;
      uint32_t* ab = abort;
      void* gargs[] = {&h, &fl, &ab};
      if ((rc = add_kernel((void*)chain_gate_kernel, dim3(1), dim3(1), gargs)) != PF_OK) break;
      cudaGraphNodeParams cp = {};
      cp.type = cudaGraphNodeTypeConditional;
      cp.conditional.handle = h;
      cp.conditional.type = cudaGraphCondTypeIf;
      cp.conditional.size = 1;
      cudaGraphNode_t cn;
      if ((rc = check_cuda(cudaGraphAddNode(&cn, g, &prev, 1, &cp), "cudaGraphAddNode(cond)")) != PF_OK)
        break;
      prev = cn;
      cudaGraph_t body = cp.conditional.phGraph_out[0];
      if ((rc = check_cuda(cudaStreamBeginCaptureToGraph(cap, body, nullptr, nullptr, 0,
                                                         cudaStreamCaptureModeThreadLocal),
                           "cudaStreamBeginCaptureToGraph")) != PF_OK)
        break;
      for (int i = lo; i < hi && rc == PF_OK; ++i) {
        pf_ctl_t ctl{flag, abort, cursors ? cursors + i : nullptr};
        LaunchArgs la;
        la.desc = c->desc;
        la.idx = done;
        la.stamp = c->stamps ? c->stamps + 2 * i : nullptr;
        if (c->timing) rc = check_cuda(cudaEventRecord(c->ev[2 * i], cap), "event");
        if (rc == PF_OK) rc = c->nodes[i]->run(flag || cursors ? &ctl : nullptr, cap, la);
        if (rc == PF_OK && c->timing) rc = check_cuda(cudaEventRecord(c->ev[2 * i + 1], cap), "event");
      }
      cudaGraph_t out_g;
      int rc2 = check_cuda(cudaStreamEndCapture(cap, &out_g), "cudaStreamEndCapture");
      if (rc == PF_OK) rc = rc2;
      lo = hi;
    }
    if (rc != PF_OK) break;
    if (done) {
      uint32_t* d = done;
      const uint32_t* ab = abort;
      void* args[] = {&d, &ab};
      if ((rc = add_kernel((void*)chain_end_kernel, dim3(1), dim3(1), args)) != PF_OK) break;
    }
    rc = check_cuda(cudaGraphInstantiate(&c->exec, g, 0), "cudaGraphInstantiate");
  } while (false);
  cudaStreamDestroy(cap);
  if (rc != PF_OK) {
    cudaGraphDestroy(g);
    return rc;
  }
  c->graph = g;
  return PF_OK;
}

int pf_chain_graph_launch(pf_chain_t* c, void* stream) {
  using namespace pf;
  if (!c || !c->exec) return set_error(PF_ERR_INVALID, "pf_chain_graph_launch: no graph built");
  PF_CUDA(cudaGraphLaunch(c->exec, reinterpret_cast<cudaStream_t>(stream)));
  return PF_OK;
}

int pf_chain_set_timing(pf_chain_t* c, int enable) {
  using namespace pf;
  if (!c) return set_error(PF_ERR_INVALID, "null chain");
  if (enable && c->ev.size() < 2 * c->nodes.size()) {
    while (c->ev.size() < 2 * c->nodes.size()) {
      cudaEvent_t e;
      PF_CUDA(cudaEventCreate(&e));
      c->ev.push_back(e);
    }
  }
  c->timing = enable != 0;
  return PF_OK;
}

int pf_chain_node_elapsed(pf_chain_t* c, int node, float* ms) {
  using namespace pf;
  if (!c || !ms || node < 0 || 2 * node + 1 >= (int)c->ev.size())
    return set_error(PF_ERR_INVALID, "pf_chain_node_elapsed: bad node or timing never enabled");
  PF_CUDA(cudaEventElapsedTime(ms, c->ev[2 * node], c->ev[2 * node + 1]));
  return PF_OK;
}

int pf_chain_launch(pf_chain_t* c, const uint32_t* flag, uint32_t* abort, uint32_t* cursors,
                    uint32_t* done, int start_node, int64_t in_off, int64_t out_off, void* stream) {
  using namespace pf;
  if (!c) return set_error(PF_ERR_INVALID, "null chain");
  const int n = (int)c->nodes.size();
  if (start_node < 0 || start_node > n)
    return set_error(PF_ERR_INVALID, "pf_chain_launch: start node %d of %d", start_node, n);
  if (flag && (!abort || !cursors))
    return set_error(PF_ERR_INVALID, "pf_chain_launch: preemptible chain needs abort and cursors");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (start_node == 0 && (cursors || c->stamps)) {
    chain_begin_kernel<<<1, 128, 0, s>>>(cursors, n, abort, c->stamps);
    PF_CUDA(cudaGetLastError());
  }
  for (int i = start_node; i < n; ++i) {
    pf_ctl_t ctl{flag, abort, cursors ? cursors + i : nullptr};
    if (c->timing) PF_CUDA(cudaEventRecord(c->ev[2 * i], s));
    LaunchArgs la;
    la.in_off = in_off;
    la.out_off = out_off;
    la.desc = c->desc;
    la.idx = done;
    la.stamp = c->stamps ? c->stamps + 2 * i : nullptr;
    PF_TRY(c->nodes[i]->run(flag || cursors ? &ctl : nullptr, s, la));
    if (c->timing) PF_CUDA(cudaEventRecord(c->ev[2 * i + 1], s));
  }
  if (done) {
    chain_end_kernel<<<1, 1, 0, s>>>(done, abort);
    PF_CUDA(cudaGetLastError());
  }
  return PF_OK;
}

}  // extern "C"
