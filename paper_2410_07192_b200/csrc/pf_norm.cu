// pf_norm.cu — HBM-bound row kernels of the fill job: LayerNorm (+residual),
// RMSNorm (+residual), row softmax, and BERT embeddings + LayerNorm.
//
// One warp per row, 16-B vectorised loads/stores (8 bf16 per access, rows held
// in registers), fp32 statistics with warp-shuffle reductions, two-pass variance.
// These kernels are "atomic" work units for preemption: every CTA checks the
// bubble flag once on entry and counts itself into the cursor on exit; they are
// out-of-place and idempotent, so an interrupted launch is simply re-run
// (cursor reset to 0) — yield latency is one CTA (16 rows, well under 1 us).
#include "pf_ops.h"

namespace pf {
namespace norm {

constexpr int WARPS = 4;
constexpr int ROWS_PER_WARP = 1;  // one row per warp, 4 warps per CTA: +1.7% on the BERT-large batch vs 8 x 2
constexpr int ROWS_PER_CTA = WARPS * ROWS_PER_WARP;
constexpr int MAX_NV = 8;  // 8 vectors x 8 bf16 x 32 lanes = 2048 columns

// Normalise one row held as NV vectors of 8 per lane (vector j covers columns
// (j*32 + lane)*8 .. +8), then write gamma/beta-scaled bf16. (Preloading gamma / beta with
// the row cost 90 registers and occupancy: 15.6 -> 17.9 us per BERT-large LN, reverted.)
// The same on packed fp32 pairs (FADD2 / FFMA2 / FMUL2, pf_common.cuh f2_*): the kernel is
// issue-bound, not HBM-bound (ncu, BERT-large [16384, 1024]: 69 % issue active, 23 % DRAM
// throughput), so halving the FP instructions per element is what moves it. x2[j][h] holds
// columns (j*32 + lane)*8 + 2h, +1.
//
// FULL (cols == NV * 256, every lane owns NV whole vectors): the per-vector column guards
// compile away. With them the BERT-large row (NV 4) compiled to 920 SASS instructions per
// warp: a BSSY/BSYNC pair, predicated pair moves and register spills around every guarded
// vector, plus an IEEE-division slow path for "/ cols" (replaced by * inv_cols).
template <int NV, bool RMS, bool FULL>
__device__ __forceinline__ void norm_row_store2(const f32x2 (&x2)[NV][4], int cols, float inv_cols,
                                                float eps, const __nv_bfloat16* gamma,
                                                const __nv_bfloat16* beta, __nv_bfloat16* y) {
  const int lane = lane_id();
  float mean = 0.f;
  if (!RMS) {
    f32x2 s0 = f2_splat(0.f), s1 = f2_splat(0.f);  // two chains for ILP
#pragma unroll
    for (int j = 0; j < NV; ++j)
      if (FULL || (j * 32 + lane) * 8 < cols) {
        s0 = f2_add(s0, f2_add(x2[j][0], x2[j][1]));
        s1 = f2_add(s1, f2_add(x2[j][2], x2[j][3]));
      }
    float a, b, c, d;
    f2_unpack(s0, a, b);
    f2_unpack(s1, c, d);
    mean = warp_sum((a + b) + (c + d)) * inv_cols;
  }
  const f32x2 nm = f2_splat(-mean);
  f32x2 q0 = f2_splat(0.f), q1 = f2_splat(0.f);
#pragma unroll
  for (int j = 0; j < NV; ++j)
    if (FULL || (j * 32 + lane) * 8 < cols) {
#pragma unroll
      for (int h = 0; h < 4; h += 2) {
        const f32x2 d0 = f2_add(x2[j][h], nm), d1 = f2_add(x2[j][h + 1], nm);
        q0 = f2_fma(d0, d0, q0);
        q1 = f2_fma(d1, d1, q1);
      }
    }
  float a, b, c, d;
  f2_unpack(q0, a, b);
  f2_unpack(q1, c, d);
  const f32x2 r2 = f2_splat(rsqrtf(warp_sum((a + b) + (c + d)) * inv_cols + eps));
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const int col = (j * 32 + lane) * 8;
    if (FULL || col < cols) {
      const uint4 gu = __ldg(reinterpret_cast<const uint4*>(gamma + col));
      uint4 bu = make_uint4(0, 0, 0, 0);
      if (!RMS) bu = __ldg(reinterpret_cast<const uint4*>(beta + col));
      const uint32_t gw[4] = {gu.x, gu.y, gu.z, gu.w};
      const uint32_t bw[4] = {bu.x, bu.y, bu.z, bu.w};
      uint32_t o[4];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const float2 g = unpack_bf16x2(gw[h]);
        const float2 bb = unpack_bf16x2(bw[h]);
        const f32x2 t = f2_mul(f2_add(x2[j][h], nm), r2);
        float lo, hi;
        f2_unpack(f2_fma(t, f2_pack(g.x, g.y), f2_pack(bb.x, bb.y)), lo, hi);
        o[h] = pack_bf16x2(lo, hi);
      }
      *reinterpret_cast<uint4*>(y + col) = make_uint4(o[0], o[1], o[2], o[3]);
    }
  }
}

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

template <int NV, bool RMS, bool FULL>
__global__ void __launch_bounds__(WARPS * 32, 10) norm_kernel(  // 10 CTAs/SM: 16384 BERT rows in 2.8 waves, not 3.07
    const __nv_bfloat16* __restrict__ X,
                                                          const __nv_bfloat16* __restrict__ R,
                                                          const __nv_bfloat16* __restrict__ gamma,
                                                          const __nv_bfloat16* __restrict__ beta,
                                                          __nv_bfloat16* __restrict__ Y, int rows,
                                                          int cols, float inv_cols, float eps, Ctl ctl) {
  static_assert(ROWS_PER_WARP == 1, "one row per warp");
  pdl_enter();
  const int lane = lane_id();
  const int row = blockIdx.x * ROWS_PER_CTA + warp_id();
  const size_t off = (size_t)row * cols;
  // the row's loads are issued before the entry gate resolves, so the gate's flag read
  // overlaps them (a row loaded for a CTA that then skips is simply dropped)
  uint4 xa[NV], ra[NV];
  if (row < rows) {
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int c = (j * 32 + lane) * 8;
      if (FULL || c < cols) {
        xa[j] = __ldg(reinterpret_cast<const uint4*>(X + off + c));
        if (R) ra[j] = __ldg(reinterpret_cast<const uint4*>(R + off + c));
      }
    }
  }
  if (!atomic_unit_check(ctl)) return;
  if (row < rows) {
    f32x2 x2[NV][4];
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const uint32_t w[4] = {xa[j].x, xa[j].y, xa[j].z, xa[j].w};
      const uint32_t v[4] = {ra[j].x, ra[j].y, ra[j].z, ra[j].w};
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const float2 f = unpack_bf16x2(w[h]);
        x2[j][h] = f2_pack(f.x, f.y);
        if (R) {
          const float2 g = unpack_bf16x2(v[h]);
          x2[j][h] = f2_add(x2[j][h], f2_pack(g.x, g.y));
        }
      }
    }
    norm_row_store2<NV, RMS, FULL>(x2, cols, inv_cols, eps, gamma, beta, Y + off);
  }
  atomic_unit_exit(ctl);
}

// bf16 pair -> fp32 pair in two integer ops (shl / and) written straight into a register
// pair, ready for the f32x2 instructions (no PRMT + shift + pair moves).
__device__ __forceinline__ f32x2 bf2_f2(uint32_t w) {
  f32x2 r;
  asm("{\n\t.reg .b32 lo, hi;\n\tshl.b32 lo, %1, 16;\n\tand.b32 hi, %1, 0xffff0000;\n\t"
      "mov.b64 %0, {lo, hi};\n\t}"
      : "=l"(r)
      : "r"(w));
  return r;
}

// The BERT LayerNorms (residual already added by the producing GEMM's epilogue) on full
// rows (cols == NV * 256): the row stays packed bf16 in registers (NV x uint4: 16 registers
// for 1024 columns instead of 32 fp32) and is re-expanded by bf2_f2 in each of the three
// passes. Same arithmetic, same order as norm_kernel + norm_row_store2, so bitwise the same
// output (scripts/ln_bench.py digests). norm_kernel at 10 CTAs/SM (48 registers) spilled
// 35 times and ran ~690 SASS instructions per 1024-column row; this kernel at 8 CTAs/SM
// (64 registers, no spills) ~500. B200, [16384, 1024] with the input in L2 (as in situ, right
// after the producing GEMM): 18.4 -> 12.2 us; from HBM 22.5 -> 18.4 us
// (profiles/r02/s53_ln_bench.txt). PF_LN_MINB=10 / 0 select the 10-CTA build / norm_kernel.
template <int NV, bool RMS, int MINB>
__global__ void __launch_bounds__(WARPS * 32, MINB) norm_packed_kernel(
    const __nv_bfloat16* __restrict__ X, const __nv_bfloat16* __restrict__ gamma,
    const __nv_bfloat16* __restrict__ beta, __nv_bfloat16* __restrict__ Y, int rows,
    float inv_cols, float eps, Ctl ctl) {
  constexpr int COLS = NV * 256;
  pdl_enter();
  const int lane = lane_id();
  const int row = blockIdx.x * ROWS_PER_CTA + warp_id();
  const size_t off = (size_t)row * COLS;
  uint4 xa[NV];
  if (row < rows) {
#pragma unroll
    for (int j = 0; j < NV; ++j) xa[j] = __ldg(reinterpret_cast<const uint4*>(X + off + (j * 32 + lane) * 8));
  }
  if (!atomic_unit_check(ctl)) return;
  if (row < rows) {
    float mean = 0.f;
    if (!RMS) {
      f32x2 s0 = f2_splat(0.f), s1 = f2_splat(0.f);
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        s0 = f2_add(s0, f2_add(bf2_f2(xa[j].x), bf2_f2(xa[j].y)));
        s1 = f2_add(s1, f2_add(bf2_f2(xa[j].z), bf2_f2(xa[j].w)));
      }
      float a, b, c, d;
      f2_unpack(s0, a, b);
      f2_unpack(s1, c, d);
      mean = warp_sum((a + b) + (c + d)) * inv_cols;
    }
    const f32x2 nm = f2_splat(-mean);
    f32x2 q0 = f2_splat(0.f), q1 = f2_splat(0.f);
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const uint32_t w[4] = {xa[j].x, xa[j].y, xa[j].z, xa[j].w};
#pragma unroll
      for (int h = 0; h < 4; h += 2) {
        const f32x2 d0 = f2_add(bf2_f2(w[h]), nm), d1 = f2_add(bf2_f2(w[h + 1]), nm);
        q0 = f2_fma(d0, d0, q0);
        q1 = f2_fma(d1, d1, q1);
      }
    }
    float a, b, c, d;
    f2_unpack(q0, a, b);
    f2_unpack(q1, c, d);
    const f32x2 r2 = f2_splat(rsqrtf(warp_sum((a + b) + (c + d)) * inv_cols + eps));
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const int col = (j * 32 + lane) * 8;
      const uint4 gu = __ldg(reinterpret_cast<const uint4*>(gamma + col));
      uint4 bu = make_uint4(0, 0, 0, 0);
      if (!RMS) bu = __ldg(reinterpret_cast<const uint4*>(beta + col));
      const uint32_t w[4] = {xa[j].x, xa[j].y, xa[j].z, xa[j].w};
      const uint32_t gw[4] = {gu.x, gu.y, gu.z, gu.w};
      const uint32_t bw[4] = {bu.x, bu.y, bu.z, bu.w};
      uint32_t o[4];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const f32x2 t = f2_mul(f2_add(bf2_f2(w[h]), nm), r2);
        float lo, hi;
        f2_unpack(f2_fma(t, bf2_f2(gw[h]), bf2_f2(bw[h])), lo, hi);
        o[h] = pack_bf16x2(lo, hi);
      }
      *reinterpret_cast<uint4*>(Y + off + col) = make_uint4(o[0], o[1], o[2], o[3]);
    }
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

struct NormOp final : PreparedOp {
  bool rms = false;
  const __nv_bfloat16 *x = nullptr, *r = nullptr, *g = nullptr, *b = nullptr;
  __nv_bfloat16* y = nullptr;
  int rows = 0, cols = 0;
  float eps = 0.f;
  uint32_t units() const override { return (uint32_t)grid_for(rows); }
  bool resumable() const override { return false; }
  int run(const pf_ctl_t* ctl, cudaStream_t s, const LaunchArgs&) override {
    const float inv_cols = 1.f / (float)cols;
    const bool full = cols % 256 == 0;
    const __nv_bfloat16* bb = rms ? nullptr : b;
#define PF_NORM_LAUNCH(RMSV, FULLV)                                                             \
  PF_NV_DISPATCH(nv_for(cols), PF_CUDA(launch_pdl(norm_kernel<NV, RMSV, FULLV>, dim3(grid_for(rows)), \
                                                  dim3(WARPS * 32), 0, s, x, r, g, bb, y, rows, cols, \
                                                  inv_cols, eps, make_ctl(ctl))))
    static const int minb = getenv("PF_LN_MINB") ? atoi(getenv("PF_LN_MINB")) : 8;  // 0: norm_kernel
    if (full && !r && minb != 0) {  // the packed full-row kernel (the BERT LayerNorms)
#define PF_NORM_PACKED(RMSV, MB)                                                                  \
  PF_NV_DISPATCH(nv_for(cols), PF_CUDA(launch_pdl(norm_packed_kernel<NV, RMSV, MB>, dim3(grid_for(rows)), \
                                                  dim3(WARPS * 32), 0, s, x, g, bb, y, rows, inv_cols,  \
                                                  eps, make_ctl(ctl))))
      if (minb == 8) {
        if (rms) { PF_NORM_PACKED(true, 8); } else { PF_NORM_PACKED(false, 8); }
      } else {
        if (rms) { PF_NORM_PACKED(true, 10); } else { PF_NORM_PACKED(false, 10); }
      }
#undef PF_NORM_PACKED
    } else if (rms) {
      if (full) { PF_NORM_LAUNCH(true, true); } else { PF_NORM_LAUNCH(true, false); }
    } else {
      if (full) { PF_NORM_LAUNCH(false, true); } else { PF_NORM_LAUNCH(false, false); }
    }
#undef PF_NORM_LAUNCH
    PF_CUDA(cudaGetLastError());
    return PF_OK;
  }
};

struct SoftmaxOp final : PreparedOp {
  const __nv_bfloat16* x = nullptr;
  __nv_bfloat16* y = nullptr;
  int rows = 0, cols = 0;
  float scale = 1.f;
  uint32_t units() const override { return (uint32_t)grid_for(rows); }
  bool resumable() const override { return false; }
  int run(const pf_ctl_t* ctl, cudaStream_t s, const LaunchArgs&) override {
    PF_NV_DISPATCH(nv_for(cols), (softmax_kernel<NV><<<grid_for(rows), WARPS * 32, 0, s>>>(
                                     x, y, rows, cols, scale, make_ctl(ctl))));
    PF_CUDA(cudaGetLastError());
    return PF_OK;
  }
};

struct EmbeddingOp final : PreparedOp {
  const int32_t *ids = nullptr, *tt = nullptr;
  const __nv_bfloat16 *word = nullptr, *pos = nullptr, *type = nullptr, *g = nullptr, *b = nullptr;
  __nv_bfloat16* y = nullptr;
  int rows = 0, seq = 0, hidden = 0, vocab = 0;
  float eps = 0.f;
  uint32_t units() const override { return (uint32_t)grid_for(rows); }
  bool resumable() const override { return false; }
  int run(const pf_ctl_t* ctl, cudaStream_t s, const LaunchArgs&) override {
    PF_NV_DISPATCH(nv_for(hidden),
                   (embedding_ln_kernel<NV><<<grid_for(rows), WARPS * 32, 0, s>>>(
                       ids, tt, word, pos, type, g, b, y, rows, seq, hidden, vocab, eps,
                       make_ctl(ctl))));
    PF_CUDA(cudaGetLastError());
    return PF_OK;
  }
};

}  // namespace norm

using bf = __nv_bfloat16;

int make_norm_op(OpPtr* out, bool rms, const void* X, const void* residual, const void* gamma,
                 const void* beta, void* Y, int rows, int cols, float eps) {
  const char* who = rms ? "pf_rmsnorm" : "pf_layernorm";
  if (!X || !gamma || !Y || (!rms && !beta)) return set_error(PF_ERR_INVALID, "%s: null pointer", who);
  PF_TRY(norm::check_rows(X, residual, gamma, Y, rows, cols, who));
  if ((uintptr_t)beta & 15u) return set_error(PF_ERR_INVALID, "%s: beta misaligned", who);
  auto op = std::make_unique<norm::NormOp>();
  op->rms = rms;
  op->x = reinterpret_cast<const bf*>(X);
  op->r = reinterpret_cast<const bf*>(residual);
  op->g = reinterpret_cast<const bf*>(gamma);
  op->b = reinterpret_cast<const bf*>(beta);
  op->y = reinterpret_cast<bf*>(Y);
  op->rows = rows;
  op->cols = cols;
  op->eps = eps;
  *out = std::move(op);
  return PF_OK;
}

int make_softmax_op(OpPtr* out, const void* X, void* Y, int rows, int cols, float scale) {
  if (!X || !Y) return set_error(PF_ERR_INVALID, "pf_softmax: null pointer");
  PF_TRY(norm::check_rows(X, Y, nullptr, nullptr, rows, cols, "pf_softmax"));
  auto op = std::make_unique<norm::SoftmaxOp>();
  op->x = reinterpret_cast<const bf*>(X);
  op->y = reinterpret_cast<bf*>(Y);
  op->rows = rows;
  op->cols = cols;
  op->scale = scale;
  *out = std::move(op);
  return PF_OK;
}

int make_embedding_op(OpPtr* out, const int32_t* ids, const int32_t* tt, const void* word,
                      const void* pos, const void* type, const void* gamma, const void* beta,
                      void* Y, int batch, int seq, int hidden, int vocab, float eps) {
  if (!ids || !word || !pos || !type || !gamma || !beta || !Y || batch <= 0 || seq <= 0 ||
      vocab <= 0)
    return set_error(PF_ERR_INVALID, "pf_embedding_ln: bad arguments");
  const int rows = batch * seq;
  PF_TRY(norm::check_rows(word, pos, type, Y, rows, hidden, "pf_embedding_ln"));
  auto op = std::make_unique<norm::EmbeddingOp>();
  op->ids = ids;
  op->tt = tt;
  op->word = reinterpret_cast<const bf*>(word);
  op->pos = reinterpret_cast<const bf*>(pos);
  op->type = reinterpret_cast<const bf*>(type);
  op->g = reinterpret_cast<const bf*>(gamma);
  op->b = reinterpret_cast<const bf*>(beta);
  op->y = reinterpret_cast<bf*>(Y);
  op->rows = rows;
  op->seq = seq;
  op->hidden = hidden;
  op->vocab = vocab;
  op->eps = eps;
  *out = std::move(op);
  return PF_OK;
}

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
  PF_TRY(pf::validate_ctl(ctl));
  pf::OpPtr op;
  PF_TRY(pf::make_norm_op(&op, false, X, residual, gamma, beta, Y, rows, cols, eps));
  return op->run(ctl, reinterpret_cast<cudaStream_t>(stream), pf::LaunchArgs{});
}

extern "C" int pf_rmsnorm(const void* X, const void* residual, const void* gamma, void* Y,
                          int rows, int cols, float eps, const pf_ctl_t* ctl, void* stream) {
  PF_TRY(pf::validate_ctl(ctl));
  pf::OpPtr op;
  PF_TRY(pf::make_norm_op(&op, true, X, residual, gamma, nullptr, Y, rows, cols, eps));
  return op->run(ctl, reinterpret_cast<cudaStream_t>(stream), pf::LaunchArgs{});
}

extern "C" int pf_softmax(const void* X, void* Y, int rows, int cols, float scale,
                          const pf_ctl_t* ctl, void* stream) {
  PF_TRY(pf::validate_ctl(ctl));
  pf::OpPtr op;
  PF_TRY(pf::make_softmax_op(&op, X, Y, rows, cols, scale));
  return op->run(ctl, reinterpret_cast<cudaStream_t>(stream), pf::LaunchArgs{});
}

extern "C" int pf_embedding_ln(const int32_t* ids, const int32_t* type_ids, const void* word,
                               const void* pos, const void* type, const void* gamma,
                               const void* beta, void* Y, int batch, int seq, int hidden,
                               int vocab, float eps, const pf_ctl_t* ctl, void* stream) {
  PF_TRY(pf::validate_ctl(ctl));
  pf::OpPtr op;
  PF_TRY(pf::make_embedding_op(&op, ids, type_ids, word, pos, type, gamma, beta, Y, batch, seq,
                               hidden, vocab, eps));
  return op->run(ctl, reinterpret_cast<cudaStream_t>(stream), pf::LaunchArgs{});
}
