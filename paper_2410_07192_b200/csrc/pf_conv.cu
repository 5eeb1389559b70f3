// pf_conv.cu — HBM-bound image kernels of convolutional fill jobs (ResNet-50), NHWC bf16.
//
// A convolution runs as im2col -> tcgen05 GEMM (pf_gemm, bias/ReLU/residual fused in
// its epilogue; BatchNorm folded into the GEMM's weights and bias). These kernels
// are the data movement around it:
//
//   im2col    X[B,H,W,C] -> Col[B*Ho*Wo, Kp], column k = (ky*kw + kx)*C + c, zero
//             outside the image and in the pad columns K..Kp (Kp % 8 == 0 for the
//             GEMM's 16-B rows). C % 8 == 0: one 16-B vector per thread; the
//             3-channel stem takes the scalar path.
//   maxpool   k x k window, stride, zero-free padding (-inf outside), 8 channels/thread.
//   avgpool   global mean over H*W -> [B, C], fp32 sums, 8 channels/thread.
//
// All three are "atomic" preemption units (gate on CTA entry, count on exit),
// out-of-place and idempotent, like the norm kernels: an interrupted launch is
// re-run whole. Every thread handles one 16-B output vector (or one scalar), so
// a CTA is 256 vectors = 4 KB of output — a yield point every ~10 ns of HBM time.
#include "pf_ops.h"

namespace pf {
namespace conv {

constexpr int THREADS = 256;

// Index decode: vector v -> (row m, 8 columns at k0) -> (b, oy, ox) and (ky, kx, c) with
// FastDiv (every total is < 2^31, checked at op creation).
struct Im2colDiv {
  FastDiv vpr, C, kw, Wo, Ho;
};

__global__ void __launch_bounds__(THREADS) im2col_vec_kernel(
    const __nv_bfloat16* __restrict__ X, __nv_bfloat16* __restrict__ Col, int H, int W, int C,
    int stride, int pad, int K, int Kp, long long total_vec, Im2colDiv dv, Ctl ctl) {
  PF_ITEMS_BEGIN(total_vec) {
    const uint32_t m = dv.vpr.div((uint32_t)v);
    const int k0 = (int)((uint32_t)v - m * dv.vpr.d) << 3;
    uint4 out = make_uint4(0, 0, 0, 0);
    if (k0 < K) {
      const uint32_t tap = dv.C.div((uint32_t)k0);
      const int c0 = k0 - (int)(tap * dv.C.d);
      const uint32_t ky = dv.kw.div(tap);
      const int kx = (int)(tap - ky * dv.kw.d);
      const uint32_t t = dv.Wo.div(m);
      const int ox = (int)(m - t * dv.Wo.d);
      const uint32_t b = dv.Ho.div(t);
      const int oy = (int)(t - b * dv.Ho.d);
      const int iy = oy * stride - pad + (int)ky, ix = ox * stride - pad + kx;
      if (iy >= 0 && iy < H && ix >= 0 && ix < W)
        out = __ldg(reinterpret_cast<const uint4*>(X + (((size_t)b * H + iy) * W + ix) * C + c0));
    }
    *reinterpret_cast<uint4*>(Col + (size_t)m * Kp + k0) = out;
  }
  PF_ITEMS_END
}

// C % 8 != 0 (the 3-channel stem): still 8 output columns (one 16-B store) per thread; the
// (ky, kx, c) of the first column is decoded once and the rest follow incrementally.
__global__ void __launch_bounds__(THREADS) im2col_small_c_kernel(
    const __nv_bfloat16* __restrict__ X, __nv_bfloat16* __restrict__ Col, int H, int W, int C,
    int stride, int pad, int K, int Kp, long long total_vec, Im2colDiv dv, Ctl ctl) {
  PF_ITEMS_BEGIN(total_vec) {
    const uint32_t m = dv.vpr.div((uint32_t)v);
    const int k0 = (int)((uint32_t)v - m * dv.vpr.d) << 3;
    const uint32_t t = dv.Wo.div(m);
    const int ox = (int)(m - t * dv.Wo.d);
    const uint32_t b = dv.Ho.div(t);
    const int oy = (int)(t - b * dv.Ho.d);
    const uint32_t tap0 = dv.C.div((uint32_t)min(k0, K));
    int c = min(k0, K) - (int)(tap0 * dv.C.d);
    const uint32_t ky0 = dv.kw.div(tap0);
    int ky = (int)ky0, kx = (int)(tap0 - ky0 * dv.kw.d);
    const __nv_bfloat16* xb = X + (size_t)b * H * W * C;
    __align__(16) __nv_bfloat16 o[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      __nv_bfloat16 val = __float2bfloat16(0.f);
      if (k0 + e < K) {
        const int iy = oy * stride - pad + ky, ix = ox * stride - pad + kx;
        if (iy >= 0 && iy < H && ix >= 0 && ix < W) val = xb[((size_t)iy * W + ix) * C + c];
      }
      o[e] = val;
      if (++c == C) {
        c = 0;
        if (++kx == (int)dv.kw.d) {
          kx = 0;
          ++ky;
        }
      }
    }
    *reinterpret_cast<uint4*>(Col + (size_t)m * Kp + k0) = *reinterpret_cast<const uint4*>(o);
  }
  PF_ITEMS_END
}

// Idx (optional, training): the window position (wy * k + wx) of each output's first
// maximum, uint8 per element -- the backward then reads 8 bytes per window instead of
// re-scanning the window's inputs.
__global__ void __launch_bounds__(THREADS) maxpool_kernel(
    const __nv_bfloat16* __restrict__ X, __nv_bfloat16* __restrict__ Y, uint8_t* __restrict__ Idx, int H, int W,
    int C, int k, int stride, int pad, long long total_vec, FastDiv dcv, FastDiv dWo, FastDiv dHo, Ctl ctl) {
  PF_ITEMS_BEGIN(total_vec) {
    const uint32_t pix = dcv.div((uint32_t)v);
    const int c0 = (int)((uint32_t)v - pix * dcv.d) << 3;
    const uint32_t t = dWo.div(pix);
    const int ox = (int)(pix - t * dWo.d);
    const uint32_t b = dHo.div(t);
    const int oy = (int)(t - b * dHo.d);
    float mx[8];
    uint32_t arg[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      mx[e] = -INFINITY;
      arg[e] = 0;
    }
    for (int ky = 0; ky < k; ++ky) {
      const int iy = oy * stride - pad + ky;
      if (iy < 0 || iy >= H) continue;
      for (int kx = 0; kx < k; ++kx) {
        const int ix = ox * stride - pad + kx;
        if (ix < 0 || ix >= W) continue;
        float x[8];
        load8(X + (((size_t)b * H + iy) * W + ix) * C + c0, x);
#pragma unroll
        for (int e = 0; e < 8; ++e)
          if (x[e] > mx[e]) {  // strict: the first maximum in (ky, kx) scan order
            mx[e] = x[e];
            arg[e] = (uint32_t)(ky * k + kx);
          }
      }
    }
    store8(Y + (size_t)pix * C + c0, mx);
    if (Idx) {
      uint2 u;
      u.x = arg[0] | (arg[1] << 8) | (arg[2] << 16) | (arg[3] << 24);
      u.y = arg[4] | (arg[5] << 8) | (arg[6] << 16) | (arg[7] << 24);
      *reinterpret_cast<uint2*>(Idx + (size_t)pix * C + c0) = u;
    }
  }
  PF_ITEMS_END
}

__global__ void __launch_bounds__(THREADS) avgpool_kernel(const __nv_bfloat16* __restrict__ X,
                                                          __nv_bfloat16* __restrict__ Y, int HW,
                                                          int C, long long total_vec, Ctl ctl) {
  PF_ITEMS_BEGIN(total_vec) {
    const int cv = C >> 3;
    const int c0 = (int)((uint32_t)v % (uint32_t)cv) << 3;
    const uint32_t b = (uint32_t)v / (uint32_t)cv;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    const __nv_bfloat16* base = X + (size_t)b * HW * C + c0;
    for (int p = 0; p < HW; ++p) {
      float x[8];
      load8(base + (size_t)p * C, x);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += x[e];
    }
    const float inv = 1.f / (float)HW;
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] *= inv;
    store8(Y + (size_t)b * C + c0, acc);
  }
  PF_ITEMS_END
}

inline uint32_t blocks_for(long long n) { return persistent_grid(n, THREADS); }

inline int out_dim(int in, int k, int stride, int pad) { return (in + 2 * pad - k) / stride + 1; }

struct Im2colOp final : PreparedOp {
  const __nv_bfloat16* x = nullptr;
  __nv_bfloat16* col = nullptr;
  int H = 0, W = 0, C = 0, Ho = 0, Wo = 0, kw = 0, stride = 1, pad = 0, K = 0, Kp = 0;
  long long n = 0;  // vectors (C % 8 == 0) or elements
  bool vec = true;
  uint32_t units() const override {
    return persistent_grid_for(vec ? (void*)im2col_vec_kernel : (void*)im2col_small_c_kernel, n, THREADS);
  }
  bool resumable() const override { return false; }
  int run(const pf_ctl_t* ctl, cudaStream_t s, const LaunchArgs&) override {
    const Im2colDiv dv{FastDiv((uint32_t)(Kp / 8)), FastDiv((uint32_t)C), FastDiv((uint32_t)kw),
                       FastDiv((uint32_t)Wo), FastDiv((uint32_t)Ho)};
    if (vec)
      im2col_vec_kernel<<<units(), THREADS, 0, s>>>(x, col, H, W, C, stride, pad, K, Kp, n, dv, make_ctl(ctl));
    else
      im2col_small_c_kernel<<<units(), THREADS, 0, s>>>(x, col, H, W, C, stride, pad, K, Kp, n, dv,
                                                        make_ctl(ctl));
    PF_CUDA(cudaGetLastError());
    return PF_OK;
  }
};

struct MaxpoolOp final : PreparedOp {
  const __nv_bfloat16* x = nullptr;
  __nv_bfloat16* y = nullptr;
  uint8_t* idx = nullptr;  // optional argmax output (training)
  int H = 0, W = 0, C = 0, Ho = 0, Wo = 0, k = 0, stride = 1, pad = 0;
  long long n = 0;
  uint32_t units() const override { return persistent_grid_for(maxpool_kernel, n, THREADS); }
  bool resumable() const override { return false; }
  int run(const pf_ctl_t* ctl, cudaStream_t s, const LaunchArgs&) override {
    maxpool_kernel<<<units(), THREADS, 0, s>>>(x, y, idx, H, W, C, k, stride, pad, n, FastDiv((uint32_t)(C / 8)),
                                                FastDiv((uint32_t)Wo), FastDiv((uint32_t)Ho), make_ctl(ctl));
    PF_CUDA(cudaGetLastError());
    return PF_OK;
  }
};

struct AvgpoolOp final : PreparedOp {
  const __nv_bfloat16* x = nullptr;
  __nv_bfloat16* y = nullptr;
  int HW = 0, C = 0;
  long long n = 0;
  uint32_t units() const override { return persistent_grid_for(avgpool_kernel, n, THREADS); }
  bool resumable() const override { return false; }
  int run(const pf_ctl_t* ctl, cudaStream_t s, const LaunchArgs&) override {
    avgpool_kernel<<<units(), THREADS, 0, s>>>(x, y, HW, C, n, make_ctl(ctl));
    PF_CUDA(cudaGetLastError());
    return PF_OK;
  }
};

static int check_ptrs(const void* a, const void* b, const char* who) {
  if (!a || !b) return set_error(PF_ERR_INVALID, "%s: null pointer", who);
  if (((uintptr_t)a | (uintptr_t)b) & 15u) return set_error(PF_ERR_INVALID, "%s: pointers must be 16-B aligned", who);
  return PF_OK;
}

}  // namespace conv

using bf = __nv_bfloat16;

int make_im2col_op(OpPtr* out, const void* X, void* Col, int B, int H, int W, int C, int kh, int kw,
                   int stride, int pad, int Kp) {
  PF_TRY(conv::check_ptrs(X, Col, "pf_im2col"));
  if (B <= 0 || H <= 0 || W <= 0 || C <= 0 || kh <= 0 || kw <= 0 || stride <= 0 || pad < 0)
    return set_error(PF_ERR_INVALID, "pf_im2col: non-positive shape");
  const int K = kh * kw * C;
  if (Kp < K || Kp % 8 != 0) return set_error(PF_ERR_INVALID, "pf_im2col: need Kp >= kh*kw*C and Kp %% 8 == 0");
  auto op = std::make_unique<conv::Im2colOp>();
  op->x = reinterpret_cast<const bf*>(X);
  op->col = reinterpret_cast<bf*>(Col);
  op->H = H;
  op->W = W;
  op->C = C;
  op->Ho = conv::out_dim(H, kh, stride, pad);
  op->Wo = conv::out_dim(W, kw, stride, pad);
  if (op->Ho <= 0 || op->Wo <= 0) return set_error(PF_ERR_INVALID, "pf_im2col: empty output");
  op->kw = kw;
  op->stride = stride;
  op->pad = pad;
  op->K = K;
  op->Kp = Kp;
  op->vec = C % 8 == 0;
  const long long rows = (long long)B * op->Ho * op->Wo;
  op->n = rows * (Kp / 8);  // 8 output columns per item on both paths
  if (op->n >= (1ll << 31) || (long long)B * H * W * C >= (1ll << 31))
    return set_error(PF_ERR_INVALID, "pf_im2col: more than 2^31 vectors");
  *out = std::move(op);
  return PF_OK;
}

int make_maxpool_op(OpPtr* out, const void* X, void* Y, int B, int H, int W, int C, int k, int stride,
                    int pad, void* Idx) {
  PF_TRY(conv::check_ptrs(X, Y, "pf_maxpool"));
  if (Idx && (k > 16 || ((uintptr_t)Idx & 7u)))
    return set_error(PF_ERR_INVALID, "pf_maxpool_argmax: need k <= 16 and an 8-B aligned index buffer");
  if (B <= 0 || H <= 0 || W <= 0 || C <= 0 || C % 8 != 0 || k <= 0 || stride <= 0 || pad < 0 || pad >= k)
    return set_error(PF_ERR_INVALID, "pf_maxpool: bad shape (C %% 8 == 0, 0 <= pad < k)");
  auto op = std::make_unique<conv::MaxpoolOp>();
  op->x = reinterpret_cast<const bf*>(X);
  op->y = reinterpret_cast<bf*>(Y);
  op->idx = reinterpret_cast<uint8_t*>(Idx);
  op->H = H;
  op->W = W;
  op->C = C;
  op->Ho = conv::out_dim(H, k, stride, pad);
  op->Wo = conv::out_dim(W, k, stride, pad);
  if (op->Ho <= 0 || op->Wo <= 0) return set_error(PF_ERR_INVALID, "pf_maxpool: empty output");
  op->k = k;
  op->stride = stride;
  op->pad = pad;
  op->n = (long long)B * op->Ho * op->Wo * (C / 8);
  if (op->n >= (1ll << 31)) return set_error(PF_ERR_INVALID, "pf_maxpool: more than 2^31 vectors");
  *out = std::move(op);
  return PF_OK;
}

int make_avgpool_op(OpPtr* out, const void* X, void* Y, int B, int HW, int C) {
  PF_TRY(conv::check_ptrs(X, Y, "pf_avgpool"));
  if (B <= 0 || HW <= 0 || C <= 0 || C % 8 != 0)
    return set_error(PF_ERR_INVALID, "pf_avgpool: bad shape (C %% 8 == 0)");
  auto op = std::make_unique<conv::AvgpoolOp>();
  op->x = reinterpret_cast<const bf*>(X);
  op->y = reinterpret_cast<bf*>(Y);
  op->HW = HW;
  op->C = C;
  op->n = (long long)B * (C / 8);
  *out = std::move(op);
  return PF_OK;
}

}  // namespace pf

extern "C" int pf_im2col(const void* X, void* Col, int B, int H, int W, int C, int kh, int kw,
                         int stride, int pad, int Kp, const pf_ctl_t* ctl, void* stream) {
  PF_TRY(pf::validate_ctl(ctl));
  pf::OpPtr op;
  PF_TRY(pf::make_im2col_op(&op, X, Col, B, H, W, C, kh, kw, stride, pad, Kp));
  return op->run(ctl, reinterpret_cast<cudaStream_t>(stream), pf::LaunchArgs{});
}

extern "C" int pf_maxpool(const void* X, void* Y, int B, int H, int W, int C, int k, int stride,
                          int pad, const pf_ctl_t* ctl, void* stream) {
  PF_TRY(pf::validate_ctl(ctl));
  pf::OpPtr op;
  PF_TRY(pf::make_maxpool_op(&op, X, Y, B, H, W, C, k, stride, pad, nullptr));
  return op->run(ctl, reinterpret_cast<cudaStream_t>(stream), pf::LaunchArgs{});
}

extern "C" int pf_maxpool_argmax(const void* X, void* Y, uint8_t* Idx, int B, int H, int W, int C, int k,
                                 int stride, int pad, const pf_ctl_t* ctl, void* stream) {
  PF_TRY(pf::validate_ctl(ctl));
  if (!Idx) return pf::set_error(PF_ERR_INVALID, "pf_maxpool_argmax: null index buffer");
  pf::OpPtr op;
  PF_TRY(pf::make_maxpool_op(&op, X, Y, B, H, W, C, k, stride, pad, Idx));
  return op->run(ctl, reinterpret_cast<cudaStream_t>(stream), pf::LaunchArgs{});
}

extern "C" int pf_avgpool(const void* X, void* Y, int B, int HW, int C, const pf_ctl_t* ctl,
                          void* stream) {
  PF_TRY(pf::validate_ctl(ctl));
  pf::OpPtr op;
  PF_TRY(pf::make_avgpool_op(&op, X, Y, B, HW, C));
  return op->run(ctl, reinterpret_cast<cudaStream_t>(stream), pf::LaunchArgs{});
}

extern "C" int pf_image_units(int kind, long long out_elems, int C, uint32_t* out_units) {
  // kind 0: im2col (out_elems = rows * Kp), 1: maxpool / avgpool (out_elems = pixels * C)
  if (!out_units || out_elems <= 0 || C <= 0) return pf::set_error(PF_ERR_INVALID, "pf_image_units");
  // every image kernel handles 8 output elements per item (im2col: Kp % 8 == 0); the grid is
  // capped at the kernel's resident CTAs. kind 0: im2col, 1: max pool, 2: average pool
  using namespace pf::conv;
  void* k = kind == 0 ? (C % 8 == 0 ? (void*)im2col_vec_kernel : (void*)im2col_small_c_kernel)
                      : kind == 1 ? (void*)maxpool_kernel : (void*)avgpool_kernel;
  *out_units = pf::persistent_grid_for(k, out_elems / 8, THREADS);
  return PF_OK;
}
