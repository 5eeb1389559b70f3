// pf_fp32.cu — the fp32 fill path (BASELINE north star: "fp32 path rel 1e-4" of the CPU
// torch execution). Same operators as the bf16 path, fp32 storage and fp32 math on the
// SIMT pipes (the tensor cores' fp32-input mode, TF32, rounds operands to 10 mantissa
// bits and cannot meet 1e-4):
//
//   sgemm_kernel     Y[M,N] = epi(X[M,K] W[N,K]^T): 128x128 output tiles, BK = 8, 256
//                    threads x 8x8 outputs, smem operands transposed to [BK][128] for
//                    broadcast reads, register-prefetched next K-slab; bias / exact-erf
//                    GELU / residual epilogue. Persistent CTAs claim tiles through the
//                    cursor exactly like pf_gemm (resumable prefix).
//   ln_f32_kernel    LayerNorm (+residual) warp per row, two-pass variance
//   emb_ln_f32       BERT embeddings + LayerNorm
//   attn_f32_kernel  one CTA per (batch, head): S = QK^T, softmax, O = PV in shared
//                    memory (seq <= 128, head_dim 64), fp32 throughout
#include "pf_ops.h"

namespace pf {
namespace f32 {

constexpr int BM = 128, BN = 128, BK = 8, T = 256;

__device__ __forceinline__ float gelu(float x) { return 0.5f * x * (1.0f + erff(x * 0.70710678118654752440f)); }

__device__ __forceinline__ void tile_of(int tile, int tiles_n, int& tm, int& tn) {
  tm = tile / tiles_n;
  tn = tile % tiles_n;
}

__global__ void __launch_bounds__(T) sgemm_kernel(const float* __restrict__ X, const float* __restrict__ W,
                                                  const float* __restrict__ bias, const float* __restrict__ R,
                                                  float* __restrict__ Y, int M, int N, int K, int gelu_on,
                                                  int tiles_n, int tiles, Ctl ctl) {
  __shared__ uint32_t s_abort;
  if (chain_aborted_cta(ctl, &s_abort)) return;
  __shared__ float sA[2][BK][BM + 4];
  __shared__ float sB[2][BK][BN + 4];
  __shared__ int s_tile;
  const int t = threadIdx.x;
  const int tx = t % 16, ty = t / 16;  // 16 x 16 threads, 8 x 8 outputs each
  // loader mapping: 256 threads x 4 floats = one 128 x 8 slab per operand
  const int lr = t / 2, lk = (t % 2) * 4;
  for (int it = 0;; ++it) {
    if (t == 0) s_tile = claim_unit(ctl, tiles, it);
    __syncthreads();
    const int tile = s_tile;
    __syncthreads();
    if (tile < 0) break;
    int tm, tn;
    tile_of(tile, tiles_n, tm, tn);
    const int m0 = tm * BM, n0 = tn * BN;
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
    auto load = [&](int k0, float (&ra)[4], float (&rb)[4]) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int k = k0 + lk + e;
        ra[e] = (m0 + lr < M && k < K) ? X[(size_t)(m0 + lr) * K + k] : 0.f;
        rb[e] = (n0 + lr < N && k < K) ? W[(size_t)(n0 + lr) * K + k] : 0.f;
      }
    };
    float ra[4], rb[4];
    load(0, ra, rb);
    int buf = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      sA[buf][lk + e][lr] = ra[e];
      sB[buf][lk + e][lr] = rb[e];
    }
    __syncthreads();
    for (int k0 = 0; k0 < K; k0 += BK) {
      const bool more = k0 + BK < K;
      if (more) load(k0 + BK, ra, rb);
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        float a[8], b[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = sA[buf][kk][ty * 8 + i];
#pragma unroll
        for (int j = 0; j < 8; ++j) b[j] = sB[buf][kk][tx * 8 + j];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
      }
      if (more) {
        buf ^= 1;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          sA[buf][lk + e][lr] = ra[e];
          sB[buf][lk + e][lr] = rb[e];
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int m = m0 + ty * 8 + i;
      if (m >= M) continue;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int n = n0 + tx * 8 + j;
        if (n >= N) continue;
        float v = acc[i][j];
        if (bias) v += bias[n];
        if (gelu_on) v = gelu(v);
        if (R) v += R[(size_t)m * N + n];
        Y[(size_t)m * N + n] = v;
      }
    }
  }
}

// LayerNorm (+residual), warp per row, fp32.
__global__ void __launch_bounds__(T) ln_f32_kernel(const float* __restrict__ X, const float* __restrict__ R,
                                                   const float* __restrict__ g, const float* __restrict__ b,
                                                   float* __restrict__ Y, int rows, int cols, float eps, Ctl ctl) {
  PF_ITEMS_BEGIN((long long)rows * 32) {
    const long long row = v >> 5;
    const int lane = threadIdx.x & 31;
    const float* x = X + row * cols;
    const float* r = R ? R + row * cols : nullptr;
    float s = 0.f;
    for (int c = lane; c < cols; c += 32) s += x[c] + (r ? r[c] : 0.f);
    const float mean = warp_sum(s) / cols;
    float ss = 0.f;
    for (int c = lane; c < cols; c += 32) {
      const float d = x[c] + (r ? r[c] : 0.f) - mean;
      ss += d * d;
    }
    const float rstd = rsqrtf(warp_sum(ss) / cols + eps);
    float* y = Y + row * cols;
    for (int c = lane; c < cols; c += 32) y[c] = (x[c] + (r ? r[c] : 0.f) - mean) * rstd * g[c] + b[c];
  }
  PF_ITEMS_END
}

__global__ void __launch_bounds__(T) emb_ln_f32_kernel(const int32_t* __restrict__ ids, const float* __restrict__ word,
                                                       const float* __restrict__ pos, const float* __restrict__ type,
                                                       const float* __restrict__ g, const float* __restrict__ b,
                                                       float* __restrict__ Y, int rows, int seq, int cols, int vocab,
                                                       float eps, Ctl ctl) {
  PF_ITEMS_BEGIN((long long)rows * 32) {
    const long long row = v >> 5;
    const int lane = threadIdx.x & 31;
    int id = ids[row];
    id = id < 0 ? 0 : (id >= vocab ? vocab - 1 : id);
    const float* w = word + (size_t)id * cols;
    const float* p = pos + (size_t)(row % seq) * cols;
    float s = 0.f;
    for (int c = lane; c < cols; c += 32) s += w[c] + p[c] + type[c];
    const float mean = warp_sum(s) / cols;
    float ss = 0.f;
    for (int c = lane; c < cols; c += 32) {
      const float d = w[c] + p[c] + type[c] - mean;
      ss += d * d;
    }
    const float rstd = rsqrtf(warp_sum(ss) / cols + eps);
    float* y = Y + row * cols;
    for (int c = lane; c < cols; c += 32) y[c] = (w[c] + p[c] + type[c] - mean) * rstd * g[c] + b[c];
  }
  PF_ITEMS_END
}

constexpr int AS = 128, AD = 64;

// One CTA per (batch, head) over QKV[b*seq, 3, heads, 64] fp32 -> O[b*seq, heads, 64].
__global__ void __launch_bounds__(T) attn_f32_kernel(const float* __restrict__ QKV, float* __restrict__ O,
                                                     int seq, int heads, float scale, Ctl ctl) {
  if (!atomic_unit_enter(ctl)) return;
  extern __shared__ float sm[];
  float* sQ = sm;                 // [AS][AD+1]
  float* sK = sQ + AS * (AD + 1);  // [AS][AD+1]
  float* sV = sK + AS * (AD + 1);  // [AS][AD]
  float* sS = sV + AS * AD;        // [AS][AS+1]
  const int b = blockIdx.x / heads, h = blockIdx.x % heads;
  const int t = threadIdx.x;
  const size_t stride = (size_t)3 * heads * AD;
  for (int e = t; e < seq * AD; e += T) {
    const int s = e / AD, d = e % AD;
    const float* base = QKV + (size_t)(b * seq + s) * stride + (size_t)h * AD + d;
    sQ[s * (AD + 1) + d] = base[0];
    sK[s * (AD + 1) + d] = base[(size_t)heads * AD];
    sV[s * AD + d] = base[(size_t)2 * heads * AD];
  }
  __syncthreads();
  for (int e = t; e < seq * seq; e += T) {
    const int i = e / seq, j = e % seq;
    float acc = 0.f;
#pragma unroll 16
    for (int d = 0; d < AD; ++d) acc = fmaf(sQ[i * (AD + 1) + d], sK[j * (AD + 1) + d], acc);
    sS[i * (AS + 1) + j] = acc * scale;
  }
  __syncthreads();
  // softmax rows: warp per row
  const int warp = t >> 5, lane = t & 31;
  for (int i = warp; i < seq; i += T / 32) {
    float m = -INFINITY;
    for (int j = lane; j < seq; j += 32) m = fmaxf(m, sS[i * (AS + 1) + j]);
    m = warp_max(m);
    float s = 0.f;
    for (int j = lane; j < seq; j += 32) {
      const float p = expf(sS[i * (AS + 1) + j] - m);
      sS[i * (AS + 1) + j] = p;
      s += p;
    }
    s = warp_sum(s);
    const float inv = 1.f / s;
    for (int j = lane; j < seq; j += 32) sS[i * (AS + 1) + j] *= inv;
  }
  __syncthreads();
  for (int e = t; e < seq * AD; e += T) {
    const int i = e / AD, d = e % AD;
    float acc = 0.f;
    for (int j = 0; j < seq; ++j) acc = fmaf(sS[i * (AS + 1) + j], sV[j * AD + d], acc);
    O[((size_t)(b * seq + i) * heads + h) * AD + d] = acc;
  }
  atomic_unit_exit(ctl);
}

constexpr int ATTN_SMEM = (AS * (AD + 1) * 2 + AS * AD + AS * (AS + 1)) * 4;

struct SgemmOp final : PreparedOp {
  const float *x = nullptr, *w = nullptr, *bias = nullptr, *r = nullptr;
  float* y = nullptr;
  int M = 0, N = 0, K = 0, gelu_on = 0, tiles_n = 0, tiles = 0, grid = 0;
  uint32_t units() const override { return (uint32_t)tiles; }
  bool resumable() const override { return true; }
  int run(const pf_ctl_t* ctl, cudaStream_t s, const LaunchArgs&) override {
    sgemm_kernel<<<grid, T, 0, s>>>(x, w, bias, r, y, M, N, K, gelu_on, tiles_n, tiles, make_ctl(ctl));
    PF_CUDA(cudaGetLastError());
    return PF_OK;
  }
};

struct RowOp final : PreparedOp {  // LayerNorm / embedding-LN, fp32
  bool emb = false;
  const float *x = nullptr, *r = nullptr, *g = nullptr, *b = nullptr, *word = nullptr, *pos = nullptr,
              *type = nullptr;
  const int32_t* ids = nullptr;
  float* y = nullptr;
  int rows = 0, cols = 0, seq = 0, vocab = 0;
  float eps = 0.f;
  uint32_t units() const override { return persistent_grid((long long)rows * 32, T); }
  bool resumable() const override { return false; }
  int run(const pf_ctl_t* ctl, cudaStream_t s, const LaunchArgs&) override {
    if (emb)
      emb_ln_f32_kernel<<<units(), T, 0, s>>>(ids, word, pos, type, g, b, y, rows, seq, cols, vocab, eps,
                                              make_ctl(ctl));
    else
      ln_f32_kernel<<<units(), T, 0, s>>>(x, r, g, b, y, rows, cols, eps, make_ctl(ctl));
    PF_CUDA(cudaGetLastError());
    return PF_OK;
  }
};

struct AttnF32Op final : PreparedOp {
  const float* qkv = nullptr;
  float* o = nullptr;
  int batch = 0, seq = 0, heads = 0;
  float scale = 1.f;
  uint32_t units() const override { return (uint32_t)(batch * heads); }
  bool resumable() const override { return false; }
  int run(const pf_ctl_t* ctl, cudaStream_t s, const LaunchArgs&) override {
    attn_f32_kernel<<<batch * heads, T, ATTN_SMEM, s>>>(qkv, o, seq, heads, scale, make_ctl(ctl));
    PF_CUDA(cudaGetLastError());
    return PF_OK;
  }
};

}  // namespace f32

int make_sgemm_op(OpPtr* out, const float* X, const float* W, const float* bias, const float* residual, float* Y,
                  int M, int N, int K, uint32_t epi) {
  if (!X || !W || !Y || M <= 0 || N <= 0 || K <= 0) return set_error(PF_ERR_INVALID, "pf_gemm_f32: bad arguments");
  if ((epi & PF_EPI_BIAS) && !bias) return set_error(PF_ERR_INVALID, "pf_gemm_f32: bias is NULL");
  if ((epi & PF_EPI_RESIDUAL) && !residual) return set_error(PF_ERR_INVALID, "pf_gemm_f32: residual is NULL");
  if (epi & ~(PF_EPI_BIAS | PF_EPI_GELU | PF_EPI_RESIDUAL))
    return set_error(PF_ERR_INVALID, "pf_gemm_f32: supported epilogues: bias, GELU, residual");
  auto op = std::make_unique<f32::SgemmOp>();
  op->x = X;
  op->w = W;
  op->bias = (epi & PF_EPI_BIAS) ? bias : nullptr;
  op->r = (epi & PF_EPI_RESIDUAL) ? residual : nullptr;
  op->y = Y;
  op->M = M;
  op->N = N;
  op->K = K;
  op->gelu_on = (epi & PF_EPI_GELU) ? 1 : 0;
  op->tiles_n = (N + f32::BN - 1) / f32::BN;
  op->tiles = ((M + f32::BM - 1) / f32::BM) * op->tiles_n;
  const int cap = 2 * device_sm_count();
  op->grid = op->tiles < cap ? op->tiles : cap;
  *out = std::move(op);
  return PF_OK;
}

int make_layernorm_f32_op(OpPtr* out, const float* X, const float* residual, const float* gamma, const float* beta,
                          float* Y, int rows, int cols, float eps) {
  if (!X || !gamma || !beta || !Y || rows <= 0 || cols <= 0)
    return set_error(PF_ERR_INVALID, "pf_layernorm_f32: bad arguments");
  auto op = std::make_unique<f32::RowOp>();
  op->x = X;
  op->r = residual;
  op->g = gamma;
  op->b = beta;
  op->y = Y;
  op->rows = rows;
  op->cols = cols;
  op->eps = eps;
  *out = std::move(op);
  return PF_OK;
}

int make_embedding_ln_f32_op(OpPtr* out, const int32_t* ids, const float* word, const float* pos, const float* type,
                             const float* gamma, const float* beta, float* Y, int batch, int seq, int hidden,
                             int vocab, float eps) {
  if (!ids || !word || !pos || !type || !gamma || !beta || !Y || batch <= 0 || seq <= 0 || hidden <= 0)
    return set_error(PF_ERR_INVALID, "pf_embedding_ln_f32: bad arguments");
  auto op = std::make_unique<f32::RowOp>();
  op->emb = true;
  op->ids = ids;
  op->word = word;
  op->pos = pos;
  op->type = type;
  op->g = gamma;
  op->b = beta;
  op->y = Y;
  op->rows = batch * seq;
  op->seq = seq;
  op->cols = hidden;
  op->vocab = vocab;
  op->eps = eps;
  *out = std::move(op);
  return PF_OK;
}

int make_attention_f32_op(OpPtr* out, const float* QKV, float* O, int batch, int seq, int heads, int head_dim,
                          float scale) {
  if (!QKV || !O || batch <= 0 || heads <= 0 || seq <= 0) return set_error(PF_ERR_INVALID, "pf_attention_f32: bad arguments");
  if (head_dim != f32::AD || seq > f32::AS)
    return set_error(PF_ERR_UNSUPPORTED, "pf_attention_f32: needs head_dim == 64 and seq <= 128");
  static bool attr = false;
  if (!attr) {
    PF_CUDA(cudaFuncSetAttribute(f32::attn_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, f32::ATTN_SMEM));
    attr = true;
  }
  auto op = std::make_unique<f32::AttnF32Op>();
  op->qkv = QKV;
  op->o = O;
  op->batch = batch;
  op->seq = seq;
  op->heads = heads;
  op->scale = scale;
  *out = std::move(op);
  return PF_OK;
}

}  // namespace pf

#define PF_RUN_F32(MAKE)                                                        \
  do {                                                                          \
    PF_TRY(pf::validate_ctl(ctl));                                              \
    pf::OpPtr op;                                                               \
    PF_TRY(MAKE);                                                               \
    return op->run(ctl, reinterpret_cast<cudaStream_t>(stream), pf::LaunchArgs{}); \
  } while (0)

extern "C" int pf_gemm_f32(const float* X, const float* W, const float* bias, const float* residual, float* Y,
                           int M, int N, int K, uint32_t epilogue, const pf_ctl_t* ctl, void* stream) {
  PF_RUN_F32(pf::make_sgemm_op(&op, X, W, bias, residual, Y, M, N, K, epilogue));
}

extern "C" int pf_layernorm_f32(const float* X, const float* residual, const float* gamma, const float* beta,
                                float* Y, int rows, int cols, float eps, const pf_ctl_t* ctl, void* stream) {
  PF_RUN_F32(pf::make_layernorm_f32_op(&op, X, residual, gamma, beta, Y, rows, cols, eps));
}

extern "C" int pf_embedding_ln_f32(const int32_t* ids, const float* word, const float* pos, const float* type,
                                   const float* gamma, const float* beta, float* Y, int batch, int seq, int hidden,
                                   int vocab, float eps, const pf_ctl_t* ctl, void* stream) {
  PF_RUN_F32(pf::make_embedding_ln_f32_op(&op, ids, word, pos, type, gamma, beta, Y, batch, seq, hidden, vocab, eps));
}

extern "C" int pf_attention_f32(const float* QKV, float* O, int batch, int seq, int heads, int head_dim,
                                float scale, const pf_ctl_t* ctl, void* stream) {
  PF_RUN_F32(pf::make_attention_f32_op(&op, QKV, O, batch, seq, heads, head_dim, scale));
}
