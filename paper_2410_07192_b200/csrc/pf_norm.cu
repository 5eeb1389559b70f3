// pf_norm.cu — HBM-bound row kernels of the fill job: LayerNorm (+residual),
// RMSNorm (+residual), row softmax, and BERT embeddings + LayerNorm.
//
// One warp per row, 16-B vectorised loads/stores (8 bf16 per access, rows held
// in registers), fp32 statistics with warp-shuffle reductions, two-pass variance.
// These kernels are "atomic" work units for preemption: every CTA checks the
// bubble flag once on entry and counts itself into the cursor on exit; they are
// out-of-place and idempotent, so an interrupted launch is simply re-run
// (cursor reset to 0) — yield latency is one CTA (16 rows, well under 1 us).
#include "pf_common.cuh"

namespace pf {
namespace norm {

constexpr int WARPS = 8;
constexpr int ROWS_PER_WARP = 2;
constexpr int ROWS_PER_CTA = WARPS * ROWS_PER_WARP;
constexpr int MAX_NV = 8;  // 8 vectors x 8 bf16 x 32 lanes = 2048 columns

// Entry gate for atomic-unit kernels; returns false when the CTA must skip.
__device__ __forceinline__ bool atomic_unit_enter(const Ctl& c) {
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

__device__ __forceinline__ void atomic_unit_exit(const Ctl& c) {
  __syncthreads();
  if (threadIdx.x == 0 && c.cursor != nullptr) {
    __threadfence();
    atomicAdd(c.cursor, 1u);
  }
}

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

// Normalise one row held as NV vectors of 8 per lane (vector j covers columns
// (j*32 + lane)*8 .. +8), then write gamma/beta-scaled bf16.
template <int NV, bool RMS>
__device__ __forceinline__ void norm_row_store(float (&x)[NV][8], int cols, float eps,
                                               const __nv_bfloat16* gamma,
                                               const __nv_bfloat16* beta, __nv_bfloat16* y) {
  const int lane = lane_id();
  float mean = 0.f;
  if (!RMS) {
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j)
      if ((j * 32 + lane) * 8 < cols)
#pragma unroll
        for (int e = 0; e < 8; ++e) s += x[j][e];
    mean = warp_sum(s) / (float)cols;
  }
  float ss = 0.f;
#pragma unroll
  for (int j = 0; j < NV; ++j)
    if ((j * 32 + lane) * 8 < cols)
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float d = x[j][e] - mean;
        ss += d * d;
      }
  const float rstd = rsqrtf(warp_sum(ss) / (float)cols + eps);
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const int c = (j * 32 + lane) * 8;
    if (c < cols) {
      float g[8], b[8], o[8];
      load8(gamma + c, g);
      if (!RMS) load8(beta + c, b);
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = (x[j][e] - mean) * rstd * g[e] + (RMS ? 0.f : b[e]);
      store8(y + c, o);
    }
  }
}

template <int NV, bool RMS>
__global__ void __launch_bounds__(WARPS * 32) norm_kernel(const __nv_bfloat16* __restrict__ X,
                                                          const __nv_bfloat16* __restrict__ R,
                                                          const __nv_bfloat16* __restrict__ gamma,
                                                          const __nv_bfloat16* __restrict__ beta,
                                                          __nv_bfloat16* __restrict__ Y, int rows,
                                                          int cols, float eps, Ctl ctl) {
  if (!atomic_unit_enter(ctl)) return;
  const int lane = lane_id();
  const int row0 = blockIdx.x * ROWS_PER_CTA + warp_id() * ROWS_PER_WARP;
#pragma unroll
  for (int rr = 0; rr < ROWS_PER_WARP; ++rr) {
    const int row = row0 + rr;
    if (row >= rows) break;
    float x[NV][8];
    const size_t off = (size_t)row * cols;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int c = (j * 32 + lane) * 8;
      if (c < cols) {
        load8(X + off + c, x[j]);
        if (R) {
          float r[8];
          load8(R + off + c, r);
#pragma unroll
          for (int e = 0; e < 8; ++e) x[j][e] += r[e];
        }
      }
    }
    norm_row_store<NV, RMS>(x, cols, eps, gamma, beta, Y + off);
  }
  atomic_unit_exit(ctl);
}

template <int NV>
__global__ void __launch_bounds__(WARPS * 32)
    embedding_ln_kernel(const int32_t* __restrict__ ids, const int32_t* __restrict__ tt,
                        const __nv_bfloat16* __restrict__ word, const __nv_bfloat16* __restrict__ pos,
                        const __nv_bfloat16* __restrict__ type, const __nv_bfloat16* __restrict__ gamma,
                        const __nv_bfloat16* __restrict__ beta, __nv_bfloat16* __restrict__ Y,
                        int rows, int seq, int cols, int vocab, float eps, Ctl ctl) {
  if (!atomic_unit_enter(ctl)) return;
  const int lane = lane_id();
  const int row0 = blockIdx.x * ROWS_PER_CTA + warp_id() * ROWS_PER_WARP;
#pragma unroll
  for (int rr = 0; rr < ROWS_PER_WARP; ++rr) {
    const int row = row0 + rr;
    if (row >= rows) break;
    int id = ids[row];
    id = id < 0 ? 0 : (id >= vocab ? vocab - 1 : id);
    const int t = tt ? tt[row] : 0;
    const int pidx = row % seq;
    float x[NV][8];
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int c = (j * 32 + lane) * 8;
      if (c < cols) {
        float a[8], b[8];
        load8(word + (size_t)id * cols + c, x[j]);
        load8(pos + (size_t)pidx * cols + c, a);
        load8(type + (size_t)t * cols + c, b);
#pragma unroll
        for (int e = 0; e < 8; ++e) x[j][e] += a[e] + b[e];
      }
    }
    norm_row_store<NV, false>(x, cols, eps, gamma, beta, Y + (size_t)row * cols);
  }
  atomic_unit_exit(ctl);
}

// Row softmax, warp per row: Y = softmax(scale * X).
template <int NV>
__global__ void __launch_bounds__(WARPS * 32) softmax_kernel(const __nv_bfloat16* __restrict__ X,
                                                             __nv_bfloat16* __restrict__ Y,
                                                             int rows, int cols, float scale,
                                                             Ctl ctl) {
  if (!atomic_unit_enter(ctl)) return;
  const int lane = lane_id();
  const int row0 = blockIdx.x * ROWS_PER_CTA + warp_id() * ROWS_PER_WARP;
#pragma unroll
  for (int rr = 0; rr < ROWS_PER_WARP; ++rr) {
    const int row = row0 + rr;
    if (row >= rows) break;
    const size_t off = (size_t)row * cols;
    float x[NV][8];
    float m = -INFINITY;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int c = (j * 32 + lane) * 8;
      if (c < cols) {
        load8(X + off + c, x[j]);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          x[j][e] *= scale;
          m = fmaxf(m, x[j][e]);
        }
      }
    }
    m = warp_max(m);
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int c = (j * 32 + lane) * 8;
      if (c < cols)
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          x[j][e] = __expf(x[j][e] - m);
          s += x[j][e];
        }
    }
    const float inv = 1.f / warp_sum(s);
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int c = (j * 32 + lane) * 8;
      if (c < cols) {
#pragma unroll
        for (int e = 0; e < 8; ++e) x[j][e] *= inv;
        store8(Y + off + c, x[j]);
      }
    }
  }
  atomic_unit_exit(ctl);
}

inline int nv_for(int cols) { return (cols + 255) / 256; }
inline int grid_for(int rows) { return (rows + ROWS_PER_CTA - 1) / ROWS_PER_CTA; }

#define PF_NV_DISPATCH(NVVAL, ...)                                         \
  switch (NVVAL) {                                                         \
    case 1: { constexpr int NV = 1; __VA_ARGS__; break; }                  \
    case 2: { constexpr int NV = 2; __VA_ARGS__; break; }                  \
    case 3: { constexpr int NV = 3; __VA_ARGS__; break; }                  \
    case 4: { constexpr int NV = 4; __VA_ARGS__; break; }                  \
    case 5: { constexpr int NV = 5; __VA_ARGS__; break; }                  \
    case 6: { constexpr int NV = 6; __VA_ARGS__; break; }                  \
    case 7: { constexpr int NV = 7; __VA_ARGS__; break; }                  \
    default: { constexpr int NV = 8; __VA_ARGS__; break; }                 \
  }

static int check_rows(const void* a, const void* b, const void* c, const void* d, int rows,
                      int cols, const char* who) {
  if (rows <= 0 || cols <= 0 || cols % 8 != 0 || cols > MAX_NV * 256)
    return set_error(PF_ERR_INVALID, "%s: need rows>0 and 8 <= cols <= 2048, cols %% 8 == 0", who);
  if (((uintptr_t)a | (uintptr_t)b | (uintptr_t)c | (uintptr_t)d) & 15u)
    return set_error(PF_ERR_INVALID, "%s: pointers must be 16-B aligned", who);
  return PF_OK;
}

}  // namespace norm
}  // namespace pf

extern "C" int pf_norm_units(int rows, int cols, uint32_t* out) {
  if (!out || rows <= 0 || cols <= 0) return pf::set_error(PF_ERR_INVALID, "pf_norm_units");
  *out = (uint32_t)pf::norm::grid_for(rows);
  return PF_OK;
}

extern "C" int pf_softmax_units(int rows, int cols, uint32_t* out) {
  return pf_norm_units(rows, cols, out);
}

extern "C" int pf_layernorm(const void* X, const void* residual, const void* gamma,
                            const void* beta, void* Y, int rows, int cols, float eps,
                            const pf_ctl_t* ctl, void* stream) {
  using namespace pf;
  using namespace pf::norm;
  if (!X || !gamma || !beta || !Y) return set_error(PF_ERR_INVALID, "pf_layernorm: null pointer");
  PF_TRY(check_rows(X, residual, gamma, Y, rows, cols, "pf_layernorm"));
  if ((uintptr_t)beta & 15u) return set_error(PF_ERR_INVALID, "pf_layernorm: beta misaligned");
  PF_TRY(validate_ctl(ctl));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const auto* x = reinterpret_cast<const __nv_bfloat16*>(X);
  const auto* r = reinterpret_cast<const __nv_bfloat16*>(residual);
  const auto* g = reinterpret_cast<const __nv_bfloat16*>(gamma);
  const auto* b = reinterpret_cast<const __nv_bfloat16*>(beta);
  auto* y = reinterpret_cast<__nv_bfloat16*>(Y);
  PF_NV_DISPATCH(nv_for(cols), (norm_kernel<NV, false><<<grid_for(rows), WARPS * 32, 0, s>>>(
                                   x, r, g, b, y, rows, cols, eps, make_ctl(ctl))));
  PF_CUDA(cudaGetLastError());
  return PF_OK;
}

extern "C" int pf_rmsnorm(const void* X, const void* residual, const void* gamma, void* Y,
                          int rows, int cols, float eps, const pf_ctl_t* ctl, void* stream) {
  using namespace pf;
  using namespace pf::norm;
  if (!X || !gamma || !Y) return set_error(PF_ERR_INVALID, "pf_rmsnorm: null pointer");
  PF_TRY(check_rows(X, residual, gamma, Y, rows, cols, "pf_rmsnorm"));
  PF_TRY(validate_ctl(ctl));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const auto* x = reinterpret_cast<const __nv_bfloat16*>(X);
  const auto* r = reinterpret_cast<const __nv_bfloat16*>(residual);
  const auto* g = reinterpret_cast<const __nv_bfloat16*>(gamma);
  auto* y = reinterpret_cast<__nv_bfloat16*>(Y);
  PF_NV_DISPATCH(nv_for(cols), (norm_kernel<NV, true><<<grid_for(rows), WARPS * 32, 0, s>>>(
                                   x, r, g, nullptr, y, rows, cols, eps, make_ctl(ctl))));
  PF_CUDA(cudaGetLastError());
  return PF_OK;
}

extern "C" int pf_softmax(const void* X, void* Y, int rows, int cols, float scale,
                          const pf_ctl_t* ctl, void* stream) {
  using namespace pf;
  using namespace pf::norm;
  if (!X || !Y) return set_error(PF_ERR_INVALID, "pf_softmax: null pointer");
  PF_TRY(check_rows(X, Y, nullptr, nullptr, rows, cols, "pf_softmax"));
  PF_TRY(validate_ctl(ctl));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  PF_NV_DISPATCH(nv_for(cols),
                 (softmax_kernel<NV><<<grid_for(rows), WARPS * 32, 0, s>>>(
                     reinterpret_cast<const __nv_bfloat16*>(X),
                     reinterpret_cast<__nv_bfloat16*>(Y), rows, cols, scale, make_ctl(ctl))));
  PF_CUDA(cudaGetLastError());
  return PF_OK;
}

extern "C" int pf_embedding_ln(const int32_t* ids, const int32_t* type_ids, const void* word,
                               const void* pos, const void* type, const void* gamma,
                               const void* beta, void* Y, int batch, int seq, int hidden,
                               int vocab, float eps, const pf_ctl_t* ctl, void* stream) {
  using namespace pf;
  using namespace pf::norm;
  if (!ids || !word || !pos || !type || !gamma || !beta || !Y || batch <= 0 || seq <= 0 ||
      vocab <= 0)
    return set_error(PF_ERR_INVALID, "pf_embedding_ln: bad arguments");
  const int rows = batch * seq;
  PF_TRY(check_rows(word, pos, type, Y, rows, hidden, "pf_embedding_ln"));
  PF_TRY(validate_ctl(ctl));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  PF_NV_DISPATCH(nv_for(hidden),
                 (embedding_ln_kernel<NV><<<grid_for(rows), WARPS * 32, 0, s>>>(
                     ids, type_ids, reinterpret_cast<const __nv_bfloat16*>(word),
                     reinterpret_cast<const __nv_bfloat16*>(pos),
                     reinterpret_cast<const __nv_bfloat16*>(type),
                     reinterpret_cast<const __nv_bfloat16*>(gamma),
                     reinterpret_cast<const __nv_bfloat16*>(beta),
                     reinterpret_cast<__nv_bfloat16*>(Y), rows, seq, hidden, vocab, eps,
                     make_ctl(ctl))));
  PF_CUDA(cudaGetLastError());
  return PF_OK;
}
