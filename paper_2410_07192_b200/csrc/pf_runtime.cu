// pf_runtime.cu — error plumbing, device checks, the fixed fill arena, the bubble
// flag, pinned staging and chain bookkeeping for libpipefill.so.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <mutex>

#include "pf_common.cuh"

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

__global__ void globaltimer_kernel(uint64_t* out) {
  uint64_t now;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
  *out = now;
}

__global__ void chain_begin_kernel(uint32_t* cursors, int n, const uint32_t* abort) {
  if (abort && ld_volatile_u32(abort) != 0u) return;
  for (int i = threadIdx.x; i < n; i += blockDim.x) cursors[i] = 0u;
}

__global__ void chain_end_kernel(uint32_t* done, const uint32_t* abort) {
  if (abort && ld_volatile_u32(abort) != 0u) return;
  *done += 1u;
}

constexpr int COPY_THREADS = 256;
constexpr uint64_t COPY_BYTES_PER_CTA = 256 * 1024;

__global__ void __launch_bounds__(COPY_THREADS) copy_kernel(uint4* __restrict__ dst,
                                                            const uint4* __restrict__ src,
                                                            uint64_t n16, Ctl ctl) {
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
  const uint64_t per = COPY_BYTES_PER_CTA / 16;
  const uint64_t lo = (uint64_t)blockIdx.x * per;
  const uint64_t hi = lo + per < n16 ? lo + per : n16;
  constexpr int U = 4;
  uint64_t i = lo + threadIdx.x;
  for (; i + (U - 1) * COPY_THREADS < hi; i += U * COPY_THREADS) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = src[i + u * COPY_THREADS];
#pragma unroll
    for (int u = 0; u < U; ++u) dst[i + u * COPY_THREADS] = v[u];
  }
  for (; i < hi; i += COPY_THREADS) dst[i] = src[i];
  __syncthreads();
  if (threadIdx.x == 0 && ctl.cursor != nullptr) {
    __threadfence_system();
    atomicAdd(ctl.cursor, 1u);
  }
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
  if (!dst || !src) return set_error(PF_ERR_INVALID, "pf_copy: null pointer");
  if ((bytes & 15u) || (((uintptr_t)dst | (uintptr_t)src) & 15u))
    return set_error(PF_ERR_INVALID, "pf_copy: bytes and pointers must be 16-B aligned");
  PF_TRY(validate_ctl(ctl));
  if (bytes == 0) return PF_OK;
  const uint64_t grid = (bytes + COPY_BYTES_PER_CTA - 1) / COPY_BYTES_PER_CTA;
  copy_kernel<<<(unsigned)grid, COPY_THREADS, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<uint4*>(dst), reinterpret_cast<const uint4*>(src), bytes / 16,
      make_ctl(ctl));
  PF_CUDA(cudaGetLastError());
  return PF_OK;
}

// ---- chain ----------------------------------------------------------------------

int pf_chain_begin(uint32_t* cursors, int n, const uint32_t* abort, void* stream) {
  using namespace pf;
  if (!cursors || n <= 0) return set_error(PF_ERR_INVALID, "pf_chain_begin: bad arguments");
  chain_begin_kernel<<<1, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(cursors, n, abort);
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
