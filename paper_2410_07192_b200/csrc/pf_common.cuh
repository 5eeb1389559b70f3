// pf_common.cuh — shared device helpers for the sm_100a fill-job kernels:
// mbarrier / TMA / tcgen05 inline PTX, the preemption protocol (bubble flag,
// sticky chain abort, monotonically claimed work cursor) and error plumbing.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/pipefill.h"

namespace pf {

// ---------------------------------------------------------------------------
// host-side error plumbing (defined in pf_runtime.cu)
int set_error(int code, const char* fmt, ...);
int check_cuda(cudaError_t err, const char* what);
int device_sm_count();
bool device_is_sm100();
bool pdl_enabled();  // programmatic dependent launch for chain kernels (PF_PDL=0 disables)

// Launch with programmatic stream serialization (PDL): the kernel may be launched while
// the previous kernel on the stream is still running; it calls pdl_wait() before touching
// anything the previous kernel writes, and pdl_trigger() so the next one can launch early.
// Captured into the chains' CUDA graphs as programmatic edges: the launch latency and the
// CTA ramp of every kernel boundary overlap the previous kernel's tail.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

#define PF_TRY(expr)              \
  do {                            \
    int _rc = (expr);             \
    if (_rc != PF_OK) return _rc; \
  } while (0)

#define PF_CUDA(expr) PF_TRY(::pf::check_cuda((expr), #expr))

// Kernel-side view of pf_ctl_t (passed by value).
struct Ctl {
  const uint32_t* flag;
  uint32_t* abort;
  uint32_t* cursor;
};

inline Ctl make_ctl(const pf_ctl_t* c) {
  Ctl k{nullptr, nullptr, nullptr};
  if (c) {
    k.flag = c->flag;
    k.abort = c->abort;
    k.cursor = c->cursor;
  }
  return k;
}

// Validates the preemption contract on the host.
inline int validate_ctl(const pf_ctl_t* c) {
  if (c && c->flag && (!c->abort || !c->cursor))
    return set_error(PF_ERR_INVALID, "pf_ctl_t: a preemptible launch needs abort and cursor");
  return PF_OK;
}

// ---------------------------------------------------------------------------
// device: preemption protocol

__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// PDL: wait until the previous kernel on the stream completed and its writes are visible
// (a no-op for a normal launch), then let the next kernel launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_enter() {
  pdl_wait();
  pdl_trigger();
}

// True when this launch must not start any work at all (chain already aborted).
__device__ __forceinline__ bool chain_aborted(const Ctl& c) {
  return c.abort != nullptr && ld_volatile_u32(c.abort) != 0u;
}

// The entry check made uniform across the CTA: thread 0 reads the abort word and the
// decision goes through shared memory. Other CTAs of the same kernel set the word when they
// see the bubble close, so per-thread reads at entry can disagree inside one CTA, and the
// threads that stayed would wait at the next __syncthreads for the ones that returned
// (found as an intermittent fill-stream stall in the SGD kernel of a resumed training
// phase). `word` is a CTA-shared scratch word.
__device__ __forceinline__ bool chain_aborted_cta(const Ctl& c, volatile uint32_t* word) {
  if (threadIdx.x == 0) *word = chain_aborted(c) ? 1u : 0u;
  __syncthreads();
  return *word != 0u;
}

// Bubble flag values: 0 = closed (yield), 1 = open, v >= 2 = open but throttled to v CTAs:
// in the bubble's last milliseconds the engine lowers the fill's power draw so the board's
// power controller has raised the SM clock again when the main job resumes.
// Only cursor-claimed work (persistent GEMMs, SGD) sheds CTAs: a shed CTA stops claiming,
// the others take its units from the shared cursor, so every unit is still done once.
__device__ __forceinline__ bool throttled_out(uint32_t f, uint32_t slot, uint32_t per_slot) {
  return f >= 2u && slot >= f / per_slot;
}

// Claims the next work unit, or returns -1 when the bubble closed (flag==0:
// sets the sticky abort), when the bubble is throttled below this CTA's index, or
// when all `units` are claimed. Static striding (no cursor) is used for
// non-preemptible launches. `iter` counts this CTA's previous claims and is only used
// by the static path.
__device__ __forceinline__ int claim_unit(const Ctl& c, int units, int iter) {
  if (c.flag != nullptr) {
    const uint32_t f = ld_acquire_u32(c.flag);
    if (f == 0u) {
      atomicExch(c.abort, 1u);
      return -1;
    }
    if (c.cursor != nullptr && throttled_out(f, blockIdx.x, 1u)) return -1;
  }
  uint32_t u;
  if (c.cursor != nullptr) {
    u = atomicAdd(c.cursor, 1u);
  } else {
    u = blockIdx.x + (uint32_t)iter * gridDim.x;
  }
  return u < (uint32_t)units ? (int)u : -1;
}

// ---------------------------------------------------------------------------
// device: warp / math helpers

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ float gelu_erf(float x) {
  return 0.5f * x * (1.0f + erff(x * 0.70710678118654752440f));
}

// erf-GELU with erf from Abramowitz & Stegun 7.1.26 (|err| <= 1.5e-7), evaluated
// with the MUFU rcp/ex2 approximations: ~15 instructions instead of erff's ~30,
// still the exact-erf GELU to fp32 working precision (not the tanh form).
__device__ __forceinline__ float fast_rcp(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float fast_ex2(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float gelu_fast(float x) {
  const float z = fabsf(x) * 0.70710678118654752440f;
  const float t = fast_rcp(fmaf(0.3275911f, z, 1.0f));
  float poly = fmaf(t, 1.061405429f, -1.453152027f);
  poly = fmaf(t, poly, 1.421413741f);
  poly = fmaf(t, poly, -0.284496736f);
  poly = fmaf(t, poly, 0.254829592f);
  poly *= t;
  const float e = fast_ex2(-z * z * 1.4426950408889634f);
  const float erf_abs = fmaf(-poly, e, 1.0f);
  const float erf_v = copysignf(erf_abs, x);
  return 0.5f * x * (1.0f + erf_v);
}

// Packed fp32 pairs for the sm_100 FFMA2 path: fma/mul/add.rn.f32x2 issue two lanes per
// instruction, each rounded exactly like its scalar counterpart, so code written with them
// is bitwise the scalar code at half the FP issue slots (the GEMM epilogue is issue-bound
// at K = 1024).
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 f2_pack(float a, float b) {
  f32x2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ f32x2 f2_splat(float a) { return f2_pack(a, a); }
__device__ __forceinline__ void f2_unpack(f32x2 v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ f32x2 f2_fma(f32x2 a, f32x2 b, f32x2 c) {
  f32x2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ f32x2 f2_mul(f32x2 a, f32x2 b) {
  f32x2 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f32x2 f2_add(f32x2 a, f32x2 b) {
  f32x2 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// gelu_fast on a pair, op for op (the negated Horner constants give -poly exactly, as
// fmaf(-poly, e, 1) needs; (-z * z) * L == (z * z) * -L in round-to-nearest).
__device__ __forceinline__ void gelu_fast2(float& x0, float& x1) {
  const f32x2 x = f2_pack(x0, x1);
  const f32x2 z = f2_mul(f2_pack(fabsf(x0), fabsf(x1)), f2_splat(0.70710678118654752440f));
  float d0, d1;
  f2_unpack(f2_fma(f2_splat(0.3275911f), z, f2_splat(1.0f)), d0, d1);
  const f32x2 t = f2_pack(fast_rcp(d0), fast_rcp(d1));
  f32x2 np = f2_fma(t, f2_splat(-1.061405429f), f2_splat(1.453152027f));
  np = f2_fma(t, np, f2_splat(-1.421413741f));
  np = f2_fma(t, np, f2_splat(0.284496736f));
  np = f2_fma(t, np, f2_splat(-0.254829592f));
  np = f2_mul(np, t);  // -poly
  float a0, a1;
  f2_unpack(f2_mul(f2_mul(z, z), f2_splat(-1.4426950408889634f)), a0, a1);
  const f32x2 e = f2_pack(fast_ex2(a0), fast_ex2(a1));
  float ea0, ea1;
  f2_unpack(f2_fma(np, e, f2_splat(1.0f)), ea0, ea1);
  const f32x2 erf_v = f2_pack(copysignf(ea0, x0), copysignf(ea1, x1));
  f2_unpack(f2_mul(f2_mul(f2_splat(0.5f), x), f2_add(f2_splat(1.0f), erf_v)), x0, x1);
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ float2 unpack_bf16x2(uint32_t u) {
  __nv_bfloat162 v = *reinterpret_cast<__nv_bfloat162*>(&u);
  return __bfloat1622float2(v);
}

// ---------------------------------------------------------------------------
// device: atomic work units (HBM-bound kernels: gate on entry, count on exit)

// Entry gate for atomic-unit kernels; returns false when the CTA must skip.
__device__ __forceinline__ bool atomic_unit_check(const Ctl& c) {
  __shared__ int s_go;
  if (threadIdx.x == 0) {
    int go = 1;
    if (chain_aborted(c)) go = 0;
    else if (c.flag != nullptr && ld_acquire_u32(c.flag) == 0u) {
      atomicExch(c.abort, 1u);
      go = 0;
    }
    s_go = go;
  }
  __syncthreads();
  return s_go != 0;
}

// Entry gate of an atomic-unit kernel (PDL wait first: the gate reads words the previous
// kernel may write). A kernel can instead call pdl_enter(), start its loads, and then
// atomic_unit_check() so the gate's flag read overlaps them.
__device__ __forceinline__ bool atomic_unit_enter(const Ctl& c) {
  pdl_enter();
  return atomic_unit_check(c);
}

__device__ __forceinline__ void atomic_unit_exit(const Ctl& c) {
  __syncthreads();
  if (threadIdx.x == 0 && c.cursor != nullptr) {
    __threadfence();
    atomicAdd(c.cursor, 1u);
  }
}

// Mid-kernel re-check for persistent (grid-stride) atomic units: thread 0 re-reads the
// flag; on a closed bubble the CTA stops WITHOUT counting itself (the node stays
// incomplete and is re-run whole on resume). Call uniformly across the CTA.
__device__ __forceinline__ bool atomic_unit_poll(const Ctl& c) {
  __shared__ int s_live;
  __syncthreads();
  if (threadIdx.x == 0) {
    int live = 1;
    if (c.flag != nullptr && ld_acquire_u32(c.flag) == 0u) {
      atomicExch(c.abort, 1u);
      live = 0;
    }
    s_live = live;
  }
  __syncthreads();
  return s_live != 0;
}

// Grid of a persistent atomic-unit kernel: enough CTAs of `threads` to cover `items`
// items once, capped at one full wave (2048 threads per SM); every CTA strides over the rest. Entry and exit
// are paid once per CTA instead of once per 256 items (the gate's flag load and barrier
// cost ~1 us per CTA, which dominated the element-wise training kernels).
// Division by a runtime divisor as a multiply-high and a shift (the HBM-bound image and
// BatchNorm kernels decode every vector index into (pixel, channel) / (row, column) with
// several divisions; 64-bit division is a ~100-instruction subroutine). Exact for n < 2^31.
struct FastDiv {
  uint32_t d = 1, m = 1, s = 0;
  FastDiv() = default;
  explicit FastDiv(uint32_t div) : d(div) {
    for (s = 0; s < 32; ++s)
      if ((1ull << s) >= div) break;
    const uint64_t magic = ((1ull << 32) * ((1ull << s) - div)) / div + 1;
    m = (uint32_t)magic;
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const { return (__umulhi(n, m) + n) >> s; }
  __device__ __forceinline__ uint32_t mod(uint32_t n) const { return n - div(n) * d; }
};

inline unsigned persistent_grid(long long items, int threads) {
  const long long need = (items + threads - 1) / threads;
  const long long cap = (2048LL / threads) * device_sm_count();  // one full wave of resident threads
  return (unsigned)(need < cap ? (need > 0 ? need : 1) : cap);
}

// The same, capped at the CTAs of `kernel` that are resident at once (its register and
// shared-memory occupancy): a grid of 8 CTAs/SM for a kernel that fits 3 runs in ceil(8/3)
// rounds with the last one partly idle (bn_bwd_apply: 74 registers).
template <typename Kernel>
inline unsigned persistent_grid_for(Kernel kernel, long long items, int threads) {
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, 0) != cudaSuccess || occ <= 0) {
    (void)cudaGetLastError();
    occ = 1;
  }
  const long long need = (items + threads - 1) / threads;
  const long long cap = (long long)occ * device_sm_count();
  return (unsigned)(need < cap ? (need > 0 ? need : 1) : cap);
}

// Poll the flag every PF_POLL_STRIDES grid strides (~64 x 592 CTAs x 256 items).
#define PF_POLL_STRIDES 64

// Body of a persistent atomic-unit kernel over item index `v` in [0, N):
//   PF_ITEMS_BEGIN(N) { ... uses v ... } PF_ITEMS_END
#define PF_ITEMS_BEGIN(N)                                                                  \
  if (!atomic_unit_enter(ctl)) return;                                                    \
  {                                                                                       \
    const long long pf_n_ = (N);                                                          \
    const long long pf_stride_ = (long long)gridDim.x * blockDim.x;                       \
    int pf_it_ = 0;                                                                       \
    for (long long pf_base_ = (long long)blockIdx.x * blockDim.x; pf_base_ < pf_n_;        \
         pf_base_ += pf_stride_, ++pf_it_) {                                              \
      if (pf_it_ && (pf_it_ % PF_POLL_STRIDES) == 0 && !atomic_unit_poll(ctl)) return;    \
      const long long v = pf_base_ + threadIdx.x;                                         \
      if (v < pf_n_)
#define PF_ITEMS_END \
    }                \
  }                  \
  atomic_unit_exit(ctl);

__device__ __forceinline__ void load8(const __nv_bfloat16* p, float* v) {
  uint4 u = *reinterpret_cast<const uint4*>(p);
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    float2 f = unpack_bf16x2(w[h]);
    v[2 * h] = f.x;
    v[2 * h + 1] = f.y;
  }
}

__device__ __forceinline__ void store8(__nv_bfloat16* p, const float* v) {
  uint4 u;
  u.x = pack_bf16x2(v[0], v[1]);
  u.y = pack_bf16x2(v[2], v[3]);
  u.z = pack_bf16x2(v[4], v[5]);
  u.w = pack_bf16x2(v[6], v[7]);
  *reinterpret_cast<uint4*>(p) = u;
}


// ---------------------------------------------------------------------------
// device: shared-memory address / mbarrier

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\t"
      "mbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\t"
      "mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(smem_u32(bar)),
      "r"(bytes)
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// Waits that park the thread in hardware (try_wait with a suspend-time hint) until the
// phase completes instead of spinning: warps that wait most of the time (epilogue warps
// on the accumulator, the TMA producer on a free stage) then stop stealing issue slots
// from the warps sharing their SM sub-partition (the single-thread MMA issuer).
__device__ __forceinline__ void mbar_wait_park(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAITP_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAITP_%=;\n\t}" ::"r"(addr),
      "r"(parity), "r"(1000000u)
      : "memory");
}

// ---------------------------------------------------------------------------
// device: TMA

__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, uint64_t* bar,
                                            int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}

// bulk tensor store smem -> global (clipped to the tensor bounds), bulk-group tracked
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* smem_src, int x,
                                             int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(smem_src)), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* smem_src, int x,
                                             int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(smem_src)), "r"(x), "r"(y), "r"(z)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// the smem sources of all committed bulk stores have been read (buffer reusable)
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// all committed bulk stores are complete (globally performed)
__device__ __forceinline__ void bulk_wait0() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ---------------------------------------------------------------------------
// device: tcgen05 (5th-gen tensor cores, TMEM accumulators)

// UMMA shared-memory descriptor for a K-major operand tile stored with the
// 128-byte swizzle TMA writes (rows of 64 bf16 = 128 B, 8-row atoms of 1024 B).
__device__ __forceinline__ uint64_t umma_desc_sw128_kmajor(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFFu);  // start address  [0,14)
  d |= (uint64_t)1u << 16;                      // LBO (unused for SW128 K-major) [16,30)
  d |= (uint64_t)(1024u >> 4) << 32;            // SBO = 8 rows * 128 B        [32,46)
  d |= (uint64_t)1u << 46;                      // descriptor version (sm_100)  [46,48)
  d |= (uint64_t)2u << 61;                      // layout: SWIZZLE_128B         [61,64)
  return d;
}

// MN-major variant (operand stored with the contiguous dimension along M/N):
// atoms of 8 K-rows x 64 MN-elements (128 B), SBO = 1024 B between K-atoms,
// LBO = `lbo_bytes` between 64-element MN blocks.
__device__ __forceinline__ uint64_t umma_desc_sw128_mnmajor(uint32_t smem_addr,
                                                            uint32_t lbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}

// Instruction descriptor: kind::f16 with bf16 A/B, fp32 D.
__host__ __device__ constexpr uint32_t umma_idesc_bf16(int M, int N, bool a_mn_major,
                                                       bool b_mn_major) {
  return (1u << 4)                          // D format: f32
         | (1u << 7)                        // A format: bf16
         | (1u << 10)                       // B format: bf16
         | ((a_mn_major ? 1u : 0u) << 15)   // A major
         | ((b_mn_major ? 1u : 0u) << 16)   // B major
         | ((uint32_t)(N >> 3) << 17)       // N / 8
         | ((uint32_t)(M >> 4) << 24);      // M / 16
}

__device__ __forceinline__ void umma_bf16_ss(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Arrive on an mbarrier once all previously issued tcgen05.mma of this thread complete.
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tmem_alloc(uint32_t* smem_dst, uint32_t ncols) {
  asm volatile(
      "tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)),
      "r"(ncols)
      : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// 32 lanes x 32 consecutive fp32 columns: thread i of the warp gets lane (base+i).
__device__ __forceinline__ void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------------------
// device: CTA-pair (cluster of 2) helpers for cta_group::2 tensor-core work

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// shared::cluster address of the same smem offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_shared(uint32_t local_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_addr), "r"(rank));
  return r;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// arrive on an mbarrier given by its shared::cluster address (possibly the peer's)
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}

// wait with cluster-scope acquire (barriers that receive remote arrivals)
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITC_%=;\n\t}" ::"r"(addr),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void mbar_wait_cluster_park(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAITCP_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAITCP_%=;\n\t}" ::"r"(addr),
      "r"(parity), "r"(1000000u)
      : "memory");
}

__device__ __forceinline__ void st_shared_cluster_u32(uint32_t cluster_addr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(cluster_addr), "r"(v) : "memory");
}

// TMA load whose completion is reported to an mbarrier that may live in the peer CTA
__device__ __forceinline__ void tma_load_2d_pair(void* smem_dst, const CUtensorMap* map,
                                                 uint32_t mbar_cluster_addr, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(mbar_cluster_addr), "r"(x), "r"(y)
      : "memory");
}

__device__ __forceinline__ void umma_bf16_ss_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                                  uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// commit the pair's MMAs to the same-offset mbarrier in both CTAs (mask 0b11)
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

__device__ __forceinline__ void tmem_alloc_pair(uint32_t* smem_dst, uint32_t ncols) {
  asm volatile(
      "tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)),
      "r"(ncols)
      : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}

__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

}  // namespace pf
