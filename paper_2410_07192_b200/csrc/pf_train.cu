// pf_train.cu — the HBM-bound kernels of a training fill job (ResNet-50 fwd + bwd + SGD).
//
// The GEMM-shaped work of training runs on tcgen05 (pf_gemm: forward convs and
// data-gradient GEMMs; pf_gemm_splitk: weight gradients with the long batch*pixels
// reduction split across CTAs). These kernels are everything around it, NHWC bf16
// activations viewed as [M = B*H*W, C] matrices, fp32 statistics:
//
//   transpose          Y[C, R] = X[R, C]^T (operand layout for dgrad / wgrad GEMMs)
//   colstats           per-CTA partial column sums (BatchNorm batch statistics, bias
//                      gradients): partial[cta] = (sum x, sum x^2) or, for the backward,
//                      (sum dA, sum dA * xhat) with dA = dY * [Y > 0]
//   bn_finalize        partials -> mean / invstd and the per-channel scale / shift
//   bn_bwd_finalize    partials -> dgamma, dbeta (fp32, straight into the gradients)
//   bn_apply           Y = act(X * scale + shift [+ R])
//   bn_bwd_apply       dX = gamma * invstd * (dA - dbeta/M - xhat * dgamma/M); also dA
//   col2im             dX[b,y,x,c] = sum over the taps that read it of dCol (a gather:
//                      deterministic, no atomics) [+ R]
//   maxpool_bwd        gradient to the first maximum of every window (torch's rule)
//   avgpool_bwd        dX = dY / HW broadcast
//   softmax_xent       loss and dLogits = (softmax - onehot) / batch, warp per row
//   sgd_update         v = mu v + g (+ wd w); w -= lr v on fp32 masters, bf16 working
//                      copy rewritten; g = sum of split-K bf16 partials or fp32
//
// Preemption: every kernel but sgd_update is an idempotent atomic unit (gate on
// entry, count on exit; partials are written per CTA, never accumulated, so a re-run
// is exact). sgd_update is NOT idempotent, so it claims chunks through the cursor
// like the GEMM (a claimed chunk always finishes; resume continues the prefix).
#include <vector>

#include "pf_ops.h"

namespace pf {
namespace train {

constexpr int T = 256;
constexpr int MAX_PARTIALS = 1024;
constexpr int FT = 1024;  // finalize threads: 32 warps split the partial rows
constexpr int SGD_CHUNK = 4096;  // elements per claimed unit

using bf = __nv_bfloat16;

inline uint32_t blocks_for(long long n) { return persistent_grid(n, T); }

__device__ __forceinline__ void ld8f(const float* p, float* v) {  // 8 floats, 32-B aligned
  const float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}

// ---------------------------------------------------------------------------- transpose

// 64 x 64 tiles: each thread loads 16 B (8 bf16) of a row and stores 16 B of a column
// segment; the CTA strides over tiles (persistent atomic unit).
__global__ void __launch_bounds__(T) transpose_kernel(const bf* __restrict__ X, bf* __restrict__ Y,
                                                      int R, int C, int tiles_c, int ntiles, Ctl ctl) {
  if (!atomic_unit_enter(ctl)) return;
  __shared__ bf tile[64][72];  // 144-B rows: 16-B aligned, staggered banks
  const int t = threadIdx.x;
  const int lr = t >> 3, lc = (t & 7) * 8;  // 32 rows x 8 vectors per pass
  int it = 0;
  for (int tl = blockIdx.x; tl < ntiles; tl += gridDim.x, ++it) {
    if (it && (it % PF_POLL_STRIDES) == 0 && !atomic_unit_poll(ctl)) return;
    const int r0 = (tl / tiles_c) * 64, c0 = (tl % tiles_c) * 64;
    const bool full = r0 + 64 <= R && c0 + 64 <= C && (C % 8) == 0 && (R % 8) == 0;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int rr = lr + 32 * k, r = r0 + rr;
      if (full) {
        *reinterpret_cast<uint4*>(&tile[rr][lc]) = *reinterpret_cast<const uint4*>(X + (size_t)r * C + c0 + lc);
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int c = c0 + lc + e;
          tile[rr][lc + e] = (r < R && c < C) ? X[(size_t)r * C + c] : __float2bfloat16(0.f);
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int cc = lr + 32 * k, c = c0 + cc;  // output row = input column
      __align__(16) bf o[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = tile[lc + e][cc];
      if (full) {
        *reinterpret_cast<uint4*>(Y + (size_t)c * R + r0 + lc) = *reinterpret_cast<const uint4*>(o);
      } else if (c < C) {
#pragma unroll
        for (int e = 0; e < 8; ++e)
          if (r0 + lc + e < R) Y[(size_t)c * R + r0 + lc + e] = o[e];
      }
    }
    __syncthreads();
  }
  atomic_unit_exit(ctl);
}

// ---------------------------------------------------------------------------- statistics

// mode 0: (sum x, sum x^2) of X.  mode 1: (sum dA, sum dA * xhat), dA = G * [Ymask > 0]
// (Ymask may be null: no ReLU), xhat = (X - mean) * invstd.
__global__ void __launch_bounds__(T, 4) colstats_kernel(  // 4 CTAs/SM: the grid is 4 x SMs (one wave)
    const bf* __restrict__ X, const bf* __restrict__ G,
                                                     const bf* __restrict__ Ymask,
                                                     const float* __restrict__ mean,
                                                     const float* __restrict__ invstd, float* partial,
                                                     int M, int C, int rows_per_cta, int mode, Ctl ctl) {
  if (!atomic_unit_enter(ctl)) return;
  __shared__ float red[2][2048];
  const int cv = C >> 3;
  const int rsub_n = T / cv;  // >= 1 (C <= 2048)
  const int t = threadIdx.x;
  const int vc = t % cv, rsub = t / cv;
  const int c0 = vc * 8;
  float s0[8], s1[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) s0[e] = s1[e] = 0.f;
  float mu[8], is[8];
  if (mode == 1) {
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      mu[e] = mean[c0 + e];
      is[e] = invstd[c0 + e];
    }
  }
  const int r0 = blockIdx.x * rows_per_cta;
  const int r1 = min(M, r0 + rows_per_cta);
  if (rsub < rsub_n) {
#pragma unroll 4
    for (int r = r0 + rsub; r < r1; r += rsub_n) {
      float x[8];
      load8(X + (size_t)r * C + c0, x);
      if (mode == 0) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          s0[e] += x[e];
          s1[e] += x[e] * x[e];
        }
      } else {
        float g[8];
        load8(G + (size_t)r * C + c0, g);
        if (Ymask) {
          float y[8];
          load8(Ymask + (size_t)r * C + c0, y);
#pragma unroll
          for (int e = 0; e < 8; ++e) g[e] = y[e] > 0.f ? g[e] : 0.f;
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          s0[e] += g[e];
          s1[e] += g[e] * (x[e] - mu[e]) * is[e];
        }
      }
    }
  }
  // reduce the rsub_n row groups of each channel vector through shared memory, one
  // group after the other (fixed order: deterministic)
  float* out = partial + (size_t)blockIdx.x * 2 * C;
  for (int g0 = 0; g0 < rsub_n; ++g0) {
    if (rsub == g0) {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        red[0][c0 + e] = (g0 == 0 ? 0.f : red[0][c0 + e]) + s0[e];
        red[1][c0 + e] = (g0 == 0 ? 0.f : red[1][c0 + e]) + s1[e];
      }
    }
    __syncthreads();
  }
  for (int c = t; c < C; c += T) {
    out[c] = red[0][c];
    out[C + c] = red[1][c];
  }
  atomic_unit_exit(ctl);
}

// partials -> mean, invstd, scale = gamma * invstd, shift = beta - mean * scale
// Sums the P partial rows of 32 channels per CTA: lane = channel, the 8 warps split
// the partial rows (8 independent load chains instead of one chain of P loads), then a
// fixed-order shared-memory combine (deterministic).
__device__ __forceinline__ void sum_partials(const float* __restrict__ partial, int P, int C, int c, double& s,
                                             double& ss) {
  __shared__ double red[2][FT / 32][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double a = 0.0, b = 0.0;
  if (c < C) {
    // loads of 8 partial rows in flight per warp (predicated), accumulated in row order
    // (deterministic): the 592 rows of a 4-CTAs-per-SM colstats grid over 32 warps are 3
    // rounds of L2 latency instead of ~6 with 4 in flight (the kernel is latency-bound:
    // tiny grids, ~10 us each; 16 in flight spills at the 64-register budget of FT = 1024)
    int p = w;
    for (; p < P; p += 8 * (FT / 32)) {
      float x[8], y[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int q = p + u * (FT / 32);
        x[u] = q < P ? partial[(size_t)q * 2 * C + c] : 0.f;
        y[u] = q < P ? partial[(size_t)q * 2 * C + C + c] : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        a += x[u];
        b += y[u];
      }
    }
  }
  red[0][w][lane] = a;
  red[1][w][lane] = b;
  __syncthreads();
  s = ss = 0.0;
  for (int k = 0; k < FT / 32; ++k) {
    s += red[0][k][lane];
    ss += red[1][k][lane];
  }
}

__global__ void __launch_bounds__(FT) bn_finalize_kernel(const float* __restrict__ partial, int P, int M,
                                                        int C, const float* __restrict__ gamma,
                                                        const float* __restrict__ beta, float eps,
                                                        float* mean, float* invstd, float* scale,
                                                        float* shift, Ctl ctl) {
  if (!atomic_unit_enter(ctl)) return;
  const int c = blockIdx.x * 32 + (threadIdx.x & 31);
  double s, ss;
  sum_partials(partial, P, C, c, s, ss);
  if (c < C && threadIdx.x < 32) {
    const double m = s / M;
    const double var = fmax(ss / M - m * m, 0.0);
    const float is = (float)(1.0 / sqrt(var + (double)eps));
    mean[c] = (float)m;
    invstd[c] = is;
    const float sc = gamma[c] * is;
    scale[c] = sc;
    shift[c] = beta[c] - (float)m * sc;
  }
  atomic_unit_exit(ctl);
}

// partials -> dbeta = sum dA, dgamma = sum dA * xhat (also a plain column sum when
// called on mode-0 partials: dsum = sum x goes to `dbeta`, dgamma may be null)
__global__ void __launch_bounds__(FT) bn_bwd_finalize_kernel(const float* __restrict__ partial, int P,
                                                            int C, float* dgamma, float* dbeta, Ctl ctl) {
  if (!atomic_unit_enter(ctl)) return;
  const int c = blockIdx.x * 32 + (threadIdx.x & 31);
  double s, sx;
  sum_partials(partial, P, C, c, s, sx);
  if (c < C && threadIdx.x < 32) {
    dbeta[c] = (float)s;
    if (dgamma) dgamma[c] = (float)sx;
  }
  atomic_unit_exit(ctl);
}

// ---------------------------------------------------------------------------- elementwise

__global__ void __launch_bounds__(T) bn_apply_kernel(const bf* __restrict__ X, const float* __restrict__ scale,
                                                     const float* __restrict__ shift, const bf* __restrict__ R,
                                                     bf* __restrict__ Y, int C, long long nvec, int relu,
                                                     FastDiv dcv, Ctl ctl) {
  // the grid stride is a multiple of C / 8 whenever C / 8 divides 256 * gridDim (every
  // power-of-two channel count): a thread then always sees the same 8 channels and loads
  // their scale / shift once instead of once per 16-B vector
  const bool hoist = ((long long)gridDim.x * blockDim.x) % dcv.d == 0;
  bool have = false;
  float sc[8], sh[8];
  PF_ITEMS_BEGIN(nvec) {
    const int c0 = (int)dcv.mod((uint32_t)v) << 3;
    float x[8];
    load8(X + v * 8, x);
    if (!have || !hoist) {
      ld8f(scale + c0, sc);
      ld8f(shift + c0, sh);
      have = true;
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) x[e] = x[e] * sc[e] + sh[e];
    if (R) {
      float r[8];
      load8(R + v * 8, r);
#pragma unroll
      for (int e = 0; e < 8; ++e) x[e] += r[e];
    }
    if (relu) {
#pragma unroll
      for (int e = 0; e < 8; ++e) x[e] = fmaxf(x[e], 0.f);
    }
    store8(Y + v * 8, x);
  }
  PF_ITEMS_END
}

// dA = G * [Ymask > 0]; dX = gamma * invstd * (dA - dbeta / M - xhat * dgamma / M).
// dA_out (optional) receives dA (the gradient reaching a residual branch).
__global__ void __launch_bounds__(T) bn_bwd_apply_kernel(
    const bf* __restrict__ X, const bf* __restrict__ G, const bf* __restrict__ Ymask,
    const float* __restrict__ mean, const float* __restrict__ invstd, const float* __restrict__ gamma,
    const float* __restrict__ dgamma, const float* __restrict__ dbeta, bf* __restrict__ dX,
    bf* __restrict__ dA_out, int M, int C, long long nvec, FastDiv dcv, Ctl ctl) {
  const bool hoist = ((long long)gridDim.x * blockDim.x) % dcv.d == 0;  // see bn_apply_kernel
  bool have = false;
  float mu[8], is[8], ga[8], dg[8], db[8];
  PF_ITEMS_BEGIN(nvec) {
    const int c0 = (int)dcv.mod((uint32_t)v) << 3;
    float x[8], g[8];
    load8(X + v * 8, x);
    load8(G + v * 8, g);
    if (Ymask) {
      float y[8];
      load8(Ymask + v * 8, y);
#pragma unroll
      for (int e = 0; e < 8; ++e) g[e] = y[e] > 0.f ? g[e] : 0.f;
    }
    if (dA_out) store8(dA_out + v * 8, g);
    const float inv_m = 1.f / (float)M;
    float o[8];
    if (!have || !hoist) {
      ld8f(mean + c0, mu);
      ld8f(invstd + c0, is);
      ld8f(gamma + c0, ga);
      ld8f(dgamma + c0, dg);
      ld8f(dbeta + c0, db);
      have = true;
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float xh = (x[e] - mu[e]) * is[e];
      o[e] = ga[e] * is[e] * (g[e] - db[e] * inv_m - xh * dg[e] * inv_m);
    }
    store8(dX + v * 8, o);
  }
  PF_ITEMS_END
}

// ---------------------------------------------------------------------------- image backward

__global__ void __launch_bounds__(T) col2im_kernel(const bf* __restrict__ dCol, const bf* __restrict__ R,
                                                   bf* __restrict__ dX, int H, int W, int C, int Ho, int Wo,
                                                   int kh, int kw, int stride, int pad, int Kp,
                                                   long long nvec, FastDiv dcv, FastDiv dW, FastDiv dH,
                                                   Ctl ctl) {
  PF_ITEMS_BEGIN(nvec) {
    const uint32_t pix = dcv.div((uint32_t)v);
    const int c0 = (int)((uint32_t)v - pix * dcv.d) << 3;
    const uint32_t t = dW.div(pix);
    const int ix = (int)(pix - t * dW.d);
    const uint32_t b = dH.div(t);
    const int iy = (int)(t - b * dH.d);
    float acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.f;
    for (int ky = 0; ky < kh; ++ky) {
      const int ny = iy + pad - ky;
      if (ny < 0 || ny % stride) continue;
      const int oy = ny / stride;
      if (oy >= Ho) continue;
      for (int kx = 0; kx < kw; ++kx) {
        const int nx = ix + pad - kx;
        if (nx < 0 || nx % stride) continue;
        const int ox = nx / stride;
        if (ox >= Wo) continue;
        float g[8];
        load8(dCol + (((size_t)b * Ho + oy) * Wo + ox) * Kp + (ky * kw + kx) * C + c0, g);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] += g[e];
      }
    }
    if (R) {
      float r[8];
      load8(R + (size_t)pix * C + c0, r);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += r[e];
    }
    store8(dX + (size_t)pix * C + c0, acc);
  }
  PF_ITEMS_END
}

__global__ void __launch_bounds__(T) maxpool_bwd_kernel(const bf* __restrict__ X, const bf* __restrict__ dY,
                                                        bf* __restrict__ dX, int H, int W, int C, int Ho,
                                                        int Wo, int k, int stride, int pad, long long nvec,
                                                        FastDiv dcv, FastDiv dW, FastDiv dH, Ctl ctl) {
  PF_ITEMS_BEGIN(nvec) {
    const uint32_t pix = dcv.div((uint32_t)v);
    const int c0 = (int)((uint32_t)v - pix * dcv.d) << 3;
    const uint32_t t = dW.div(pix);
    const int ix = (int)(pix - t * dW.d);
    const uint32_t b = dH.div(t);
    const int iy = (int)(t - b * dH.d);
    float acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.f;
    for (int ky = 0; ky < k; ++ky) {
      const int ny = iy + pad - ky;
      if (ny < 0 || ny % stride) continue;
      const int oy = ny / stride;
      if (oy >= Ho) continue;
      for (int kx = 0; kx < k; ++kx) {
        const int nx = ix + pad - kx;
        if (nx < 0 || nx % stride) continue;
        const int ox = nx / stride;
        if (ox >= Wo) continue;
        // window (oy, ox): first maximum in (wy, wx) scan order, per channel
        float best[8];
        int arg[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          best[e] = -INFINITY;
          arg[e] = -1;
        }
        for (int wy = 0; wy < k; ++wy) {
          const int yy = oy * stride - pad + wy;
          if (yy < 0 || yy >= H) continue;
          for (int wx = 0; wx < k; ++wx) {
            const int xx = ox * stride - pad + wx;
            if (xx < 0 || xx >= W) continue;
            float x[8];
            load8(X + (((size_t)b * H + yy) * W + xx) * C + c0, x);
#pragma unroll
            for (int e = 0; e < 8; ++e)
              if (x[e] > best[e]) {
                best[e] = x[e];
                arg[e] = yy * W + xx;
              }
          }
        }
        float g[8];
        load8(dY + (((size_t)b * Ho + oy) * Wo + ox) * C + c0, g);
#pragma unroll
        for (int e = 0; e < 8; ++e)
          if (arg[e] == iy * W + ix) acc[e] += g[e];
      }
    }
    store8(dX + (size_t)pix * C + c0, acc);
  }
  PF_ITEMS_END
}

// Max-pool backward from the forward's argmax bytes (pf_maxpool_argmax): every input pixel
// gathers dY from the <= ceil(k / stride)^2 windows that contain it, where that window's
// first maximum sits at this pixel -- 8 index bytes and 16 B of dY per window instead of
// re-scanning the window's k * k inputs. Same (ky, kx) order and fp32 sums as
// maxpool_bwd_kernel, so the two agree bit for bit.
__global__ void __launch_bounds__(T) maxpool_bwd_idx_kernel(const uint8_t* __restrict__ Idx, const bf* __restrict__ dY,
                                                            bf* __restrict__ dX, int H, int W, int C, int Ho,
                                                            int Wo, int k, int stride, int pad, long long nvec,
                                                            FastDiv dcv, FastDiv dW, FastDiv dH, Ctl ctl) {
  PF_ITEMS_BEGIN(nvec) {
    const uint32_t pix = dcv.div((uint32_t)v);
    const int c0 = (int)((uint32_t)v - pix * dcv.d) << 3;
    const uint32_t t = dW.div(pix);
    const int ix = (int)(pix - t * dW.d);
    const uint32_t b = dH.div(t);
    const int iy = (int)(t - b * dH.d);
    float acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.f;
    for (int ky = 0; ky < k; ++ky) {
      const int ny = iy + pad - ky;
      if (ny < 0 || ny % stride) continue;
      const int oy = ny / stride;
      if (oy >= Ho) continue;
      for (int kx = 0; kx < k; ++kx) {
        const int nx = ix + pad - kx;
        if (nx < 0 || nx % stride) continue;
        const int ox = nx / stride;
        if (ox >= Wo) continue;
        const size_t o = (((size_t)b * Ho + oy) * Wo + ox) * C + c0;
        const uint2 id = *reinterpret_cast<const uint2*>(Idx + o);
        const uint32_t pos = (uint32_t)(ky * k + kx);  // this pixel's position in window (oy, ox)
        float g[8];
        load8(dY + o, g);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const uint32_t a = ((e < 4 ? id.x : id.y) >> (8 * (e & 3))) & 0xffu;
          if (a == pos) acc[e] += g[e];
        }
      }
    }
    store8(dX + (size_t)pix * C + c0, acc);
  }
  PF_ITEMS_END
}

__global__ void __launch_bounds__(T) avgpool_bwd_kernel(const bf* __restrict__ dY, bf* __restrict__ dX,
                                                        int HW, int C, long long nvec, FastDiv dcv,
                                                        FastDiv dhwcv, Ctl ctl) {
  PF_ITEMS_BEGIN(nvec) {
    const int c0 = (int)dcv.mod((uint32_t)v) << 3;
    const uint32_t b = dhwcv.div((uint32_t)v);
    float g[8];
    load8(dY + (size_t)b * C + c0, g);
    const float inv = 1.f / (float)HW;
#pragma unroll
    for (int e = 0; e < 8; ++e) g[e] *= inv;
    store8(dX + v * 8, g);
  }
  PF_ITEMS_END
}

// ---------------------------------------------------------------------------- loss

// One warp per row: loss[b*4] = logsumexp(z) - z[label]; dZ = (softmax(z) - onehot) * grad_scale.
// labels are int32 with a 4-word (16-B) stride per sample.
__global__ void __launch_bounds__(T) softmax_xent_kernel(const bf* __restrict__ Z, const int32_t* __restrict__ labels,
                                                         float* __restrict__ loss, bf* __restrict__ dZ, int B,
                                                         int N, float grad_scale, Ctl ctl) {
  if (!atomic_unit_enter(ctl)) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * (T / 32) + warp;
  if (row < B) {
    const bf* z = Z + (size_t)row * N;
    float m = -INFINITY;
    for (int c = lane * 8; c < N; c += 256) {
      float x[8];
      load8(z + c, x);
#pragma unroll
      for (int e = 0; e < 8; ++e) m = fmaxf(m, x[e]);
    }
    m = warp_max(m);
    float s = 0.f;
    for (int c = lane * 8; c < N; c += 256) {
      float x[8];
      load8(z + c, x);
#pragma unroll
      for (int e = 0; e < 8; ++e) s += __expf(x[e] - m);
    }
    s = warp_sum(s);
    const int label = labels[(size_t)row * 4];
    const float lse = m + __logf(s);
    if (lane == 0) {
      loss[(size_t)row * 4] = lse - __bfloat162float(z[label]);
      loss[(size_t)row * 4 + 1] = 0.f;
      loss[(size_t)row * 4 + 2] = 0.f;
      loss[(size_t)row * 4 + 3] = 0.f;
    }
    const float inv = 1.f / s;
    for (int c = lane * 8; c < N; c += 256) {
      float x[8];
      load8(z + c, x);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float p = __expf(x[e] - m) * inv;
        x[e] = (p - (c + e == label ? 1.f : 0.f)) * grad_scale;
      }
      store8(dZ + (size_t)row * N + c, x);
    }
  }
  atomic_unit_exit(ctl);
}

// ---------------------------------------------------------------------------- optimizer

struct SgdSeg {
  float* master;       // fp32 weights
  float* mom;          // fp32 momentum
  bf* work;            // bf16 working copy the GEMMs read (may be null)
  const void* grad;    // bf16 [splits, n] partials (kind 0) or fp32 [n] (kind 1)
  long long n;
  long long split_stride;  // elements between partials
  int splits;
  int kind;
  float wd;            // weight decay of this tensor
  int first_unit;      // prefix sum of units before this segment
};

constexpr int MAX_SGD_SEGS = 256;

__global__ void __launch_bounds__(T) sgd_kernel(const SgdSeg* __restrict__ segs, int nseg, int units,
                                                float lr, float mu, Ctl ctl) {
  __shared__ uint32_t s_abort;
  if (chain_aborted_cta(ctl, &s_abort)) return;
  __shared__ int s_unit;
  __shared__ int s_first[MAX_SGD_SEGS];  // first unit of every segment: binary-searched in smem
  for (int i = threadIdx.x; i < nseg; i += T) s_first[i] = segs[i].first_unit;
  __syncthreads();
  for (int it = 0;; ++it) {
    if (threadIdx.x == 0) s_unit = claim_unit(ctl, units, it);
    __syncthreads();
    const int u = s_unit;
    __syncthreads();
    if (u < 0) break;
    int sl = 0, sh = nseg - 1;  // last segment with first_unit <= u
    while (sl < sh) {
      const int mid = (sl + sh + 1) >> 1;
      if (s_first[mid] <= u) sl = mid;
      else sh = mid - 1;
    }
    const SgdSeg sg = segs[sl];
    const long long lo = (long long)(u - sg.first_unit) * SGD_CHUNK;
    const long long hi = min(sg.n, lo + SGD_CHUNK);
#pragma unroll 4
    for (long long i = lo + threadIdx.x; i < hi; i += T) {
      float g = 0.f;
      if (sg.kind == 0) {
        const bf* gp = reinterpret_cast<const bf*>(sg.grad);
        for (int z = 0; z < sg.splits; ++z) g += __bfloat162float(gp[z * sg.split_stride + i]);
      } else {
        g = reinterpret_cast<const float*>(sg.grad)[i];
      }
      float w = sg.master[i];
      g += sg.wd * w;
      const float v = mu * sg.mom[i] + g;
      sg.mom[i] = v;
      w -= lr * v;
      sg.master[i] = w;
      if (sg.work) sg.work[i] = __float2bfloat16(w);
    }
  }
}

// ---------------------------------------------------------------------------- ops

struct TransposeOp final : PreparedOp {
  const bf* x = nullptr;
  bf* y = nullptr;
  int R = 0, C = 0;
  int ntiles() const { return ((R + 63) / 64) * ((C + 63) / 64); }
  uint32_t units() const override {
    const int cap = 8 * device_sm_count();
    return (uint32_t)(ntiles() < cap ? ntiles() : cap);
  }
  bool resumable() const override { return false; }
  int run(const pf_ctl_t* ctl, cudaStream_t s, const LaunchArgs&) override {
    transpose_kernel<<<units(), T, 0, s>>>(x, y, R, C, (C + 63) / 64, ntiles(), make_ctl(ctl));
    PF_CUDA(cudaGetLastError());
    return PF_OK;
  }
};

struct ColstatsOp final : PreparedOp {
  const bf *x = nullptr, *g = nullptr, *ymask = nullptr;
  const float *mean = nullptr, *invstd = nullptr;
  float* partial = nullptr;
  int M = 0, C = 0, rows = 0, P = 0, mode = 0;
  uint32_t units() const override { return (uint32_t)P; }
  bool resumable() const override { return false; }
  int run(const pf_ctl_t* ctl, cudaStream_t s, const LaunchArgs&) override {
    colstats_kernel<<<P, T, 0, s>>>(x, g, ymask, mean, invstd, partial, M, C, rows, mode, make_ctl(ctl));
    PF_CUDA(cudaGetLastError());
    return PF_OK;
  }
};

struct BnFinalizeOp final : PreparedOp {
  const float *partial = nullptr, *gamma = nullptr, *beta = nullptr;
  float *mean = nullptr, *invstd = nullptr, *scale = nullptr, *shift = nullptr;
  float *dgamma = nullptr, *dbeta = nullptr;
  int P = 0, M = 0, C = 0;
  float eps = 0.f;
  bool bwd = false;
  uint32_t units() const override { return (uint32_t)((C + 31) / 32); }
  bool resumable() const override { return false; }
  int run(const pf_ctl_t* ctl, cudaStream_t s, const LaunchArgs&) override {
    if (bwd)
      bn_bwd_finalize_kernel<<<units(), FT, 0, s>>>(partial, P, C, dgamma, dbeta, make_ctl(ctl));
    else
      bn_finalize_kernel<<<units(), FT, 0, s>>>(partial, P, M, C, gamma, beta, eps, mean, invstd, scale,
                                                shift, make_ctl(ctl));
    PF_CUDA(cudaGetLastError());
    return PF_OK;
  }
};

struct BnApplyOp final : PreparedOp {
  const bf *x = nullptr, *r = nullptr;
  const float *scale = nullptr, *shift = nullptr;
  bf* y = nullptr;
  int C = 0, relu = 0;
  long long nvec = 0;
  uint32_t units() const override { return persistent_grid_for(bn_apply_kernel, nvec, T); }
  bool resumable() const override { return false; }
  int run(const pf_ctl_t* ctl, cudaStream_t s, const LaunchArgs&) override {
    bn_apply_kernel<<<units(), T, 0, s>>>(x, scale, shift, r, y, C, nvec, relu, FastDiv((uint32_t)(C / 8)),
                                          make_ctl(ctl));
    PF_CUDA(cudaGetLastError());
    return PF_OK;
  }
};

struct BnBwdApplyOp final : PreparedOp {
  const bf *x = nullptr, *g = nullptr, *ymask = nullptr;
  const float *mean = nullptr, *invstd = nullptr, *gamma = nullptr, *dgamma = nullptr, *dbeta = nullptr;
  bf *dx = nullptr, *da = nullptr;
  int M = 0, C = 0;
  long long nvec = 0;
  uint32_t units() const override { return persistent_grid_for(bn_bwd_apply_kernel, nvec, T); }
  bool resumable() const override { return false; }
  int run(const pf_ctl_t* ctl, cudaStream_t s, const LaunchArgs&) override {
    bn_bwd_apply_kernel<<<units(), T, 0, s>>>(x, g, ymask, mean, invstd, gamma, dgamma, dbeta, dx, da, M, C,
                                              nvec, FastDiv((uint32_t)(C / 8)), make_ctl(ctl));
    PF_CUDA(cudaGetLastError());
    return PF_OK;
  }
};

struct Col2imOp final : PreparedOp {
  const bf *dcol = nullptr, *r = nullptr;
  bf* dx = nullptr;
  int H = 0, W = 0, C = 0, Ho = 0, Wo = 0, kh = 0, kw = 0, stride = 1, pad = 0, Kp = 0;
  long long nvec = 0;
  uint32_t units() const override { return persistent_grid_for(col2im_kernel, nvec, T); }
  bool resumable() const override { return false; }
  int run(const pf_ctl_t* ctl, cudaStream_t s, const LaunchArgs&) override {
    col2im_kernel<<<units(), T, 0, s>>>(dcol, r, dx, H, W, C, Ho, Wo, kh, kw, stride, pad, Kp, nvec,
                                        FastDiv((uint32_t)(C / 8)), FastDiv((uint32_t)W),
                                        FastDiv((uint32_t)H), make_ctl(ctl));
    PF_CUDA(cudaGetLastError());
    return PF_OK;
  }
};

struct PoolBwdOp final : PreparedOp {
  const bf *x = nullptr, *dy = nullptr;
  const uint8_t* idx = nullptr;  // argmax bytes of the forward (maxpool_bwd_idx_kernel) instead of x
  bf* dx = nullptr;
  int H = 0, W = 0, C = 0, Ho = 0, Wo = 0, k = 0, stride = 1, pad = 0, HW = 0;
  bool avg = false;
  long long nvec = 0;
  uint32_t units() const override { return persistent_grid_for(avg ? (void*)avgpool_bwd_kernel : idx ? (void*)maxpool_bwd_idx_kernel : (void*)maxpool_bwd_kernel, nvec, T); }
  bool resumable() const override { return false; }
  int run(const pf_ctl_t* ctl, cudaStream_t s, const LaunchArgs&) override {
    if (avg)
      avgpool_bwd_kernel<<<units(), T, 0, s>>>(dy, dx, HW, C, nvec, FastDiv((uint32_t)(C / 8)),
                                               FastDiv((uint32_t)(HW * (C / 8))), make_ctl(ctl));
    else
      if (idx)
        maxpool_bwd_idx_kernel<<<units(), T, 0, s>>>(idx, dy, dx, H, W, C, Ho, Wo, k, stride, pad, nvec,
                                                     FastDiv((uint32_t)(C / 8)), FastDiv((uint32_t)W),
                                                     FastDiv((uint32_t)H), make_ctl(ctl));
      else
  maxpool_bwd_kernel<<<units(), T, 0, s>>>(x, dy, dx, H, W, C, Ho, Wo, k, stride, pad, nvec,
                                               FastDiv((uint32_t)(C / 8)), FastDiv((uint32_t)W),
                                               FastDiv((uint32_t)H), make_ctl(ctl));
    PF_CUDA(cudaGetLastError());
    return PF_OK;
  }
};

struct XentOp final : PreparedOp {
  const bf* z = nullptr;
  const int32_t* labels = nullptr;
  float* loss = nullptr;
  bf* dz = nullptr;
  int B = 0, N = 0;
  float scale = 1.f;
  uint32_t units() const override { return (uint32_t)((B + T / 32 - 1) / (T / 32)); }
  bool resumable() const override { return false; }
  int run(const pf_ctl_t* ctl, cudaStream_t s, const LaunchArgs&) override {
    softmax_xent_kernel<<<units(), T, 0, s>>>(z, labels, loss, dz, B, N, scale, make_ctl(ctl));
    PF_CUDA(cudaGetLastError());
    return PF_OK;
  }
};

struct SgdOp final : PreparedOp {
  SgdSeg* dsegs = nullptr;  // device copy
  int nseg = 0, total_units = 0;
  float lr = 0.f, mu = 0.f;
  int grid = 0;
  ~SgdOp() override {
    if (dsegs) cudaFree(dsegs);
  }
  uint32_t units() const override { return (uint32_t)total_units; }
  bool resumable() const override { return true; }
  int run(const pf_ctl_t* ctl, cudaStream_t s, const LaunchArgs&) override {
    sgd_kernel<<<grid, T, 0, s>>>(dsegs, nseg, total_units, lr, mu, make_ctl(ctl));
    PF_CUDA(cudaGetLastError());
    return PF_OK;
  }
};

static int aligned16(const void* a, const void* b = nullptr, const void* c = nullptr, const void* d = nullptr) {
  return (((uintptr_t)a | (uintptr_t)b | (uintptr_t)c | (uintptr_t)d) & 15u) == 0;
}

}  // namespace train

using train::bf;

int make_transpose_op(OpPtr* out, const void* X, void* Y, int R, int C) {
  if (!X || !Y || R <= 0 || C <= 0) return set_error(PF_ERR_INVALID, "pf_transpose: bad arguments");
  auto op = std::make_unique<train::TransposeOp>();
  op->x = reinterpret_cast<const bf*>(X);
  op->y = reinterpret_cast<bf*>(Y);
  op->R = R;
  op->C = C;
  *out = std::move(op);
  return PF_OK;
}

int make_colstats_op(OpPtr* out, const void* X, const void* G, const void* Ymask, const float* mean,
                     const float* invstd, float* partial, int M, int C, int* out_partials) {
  if (!X || !partial || M <= 0 || C <= 0 || C % 8 != 0 || C > 2048)
    return set_error(PF_ERR_INVALID, "pf_colstats: bad arguments (C %% 8 == 0, C <= 2048)");
  if (G && (!mean || !invstd)) return set_error(PF_ERR_INVALID, "pf_colstats: backward mode needs mean/invstd");
  if (!train::aligned16(X, G, Ymask)) return set_error(PF_ERR_INVALID, "pf_colstats: 16-B alignment");
  auto op = std::make_unique<train::ColstatsOp>();
  op->x = reinterpret_cast<const bf*>(X);
  op->g = reinterpret_cast<const bf*>(G);
  op->ymask = reinterpret_cast<const bf*>(Ymask);
  op->mean = mean;
  op->invstd = invstd;
  op->partial = partial;
  op->M = M;
  op->C = C;
  op->mode = G ? 1 : 0;
  const int target = 4 * device_sm_count();
  int rows = (M + target - 1) / target;
  if (rows < 32) rows = 32;
  op->P = (M + rows - 1) / rows;
  if (op->P > train::MAX_PARTIALS) {
    op->P = train::MAX_PARTIALS;
    rows = (M + op->P - 1) / op->P;
    op->P = (M + rows - 1) / rows;
  }
  op->rows = rows;
  if (out_partials) *out_partials = op->P;
  *out = std::move(op);
  return PF_OK;
}

int make_bn_finalize_op(OpPtr* out, const float* partial, int P, int M, int C, const float* gamma,
                        const float* beta, float eps, float* mean, float* invstd, float* scale, float* shift) {
  if (!partial || P <= 0 || M <= 0 || C <= 0 || !gamma || !beta || !mean || !invstd || !scale || !shift)
    return set_error(PF_ERR_INVALID, "pf_bn_finalize: bad arguments");
  auto op = std::make_unique<train::BnFinalizeOp>();
  op->partial = partial;
  op->P = P;
  op->M = M;
  op->C = C;
  op->gamma = gamma;
  op->beta = beta;
  op->eps = eps;
  op->mean = mean;
  op->invstd = invstd;
  op->scale = scale;
  op->shift = shift;
  *out = std::move(op);
  return PF_OK;
}

int make_bn_bwd_finalize_op(OpPtr* out, const float* partial, int P, int C, float* dgamma, float* dbeta) {
  if (!partial || P <= 0 || C <= 0 || !dbeta) return set_error(PF_ERR_INVALID, "pf_bn_bwd_finalize: bad arguments");
  auto op = std::make_unique<train::BnFinalizeOp>();
  op->bwd = true;
  op->partial = partial;
  op->P = P;
  op->C = C;
  op->dgamma = dgamma;
  op->dbeta = dbeta;
  *out = std::move(op);
  return PF_OK;
}

int make_bn_apply_op(OpPtr* out, const void* X, const float* scale, const float* shift, const void* R, void* Y,
                     long long M, int C, int relu) {
  if (!X || !Y || !scale || !shift || M <= 0 || C <= 0 || C % 8 != 0)
    return set_error(PF_ERR_INVALID, "pf_bn_apply: bad arguments");
  if (!train::aligned16(X, Y, R)) return set_error(PF_ERR_INVALID, "pf_bn_apply: 16-B alignment");
  auto op = std::make_unique<train::BnApplyOp>();
  op->x = reinterpret_cast<const bf*>(X);
  op->r = reinterpret_cast<const bf*>(R);
  op->y = reinterpret_cast<bf*>(Y);
  op->scale = scale;
  op->shift = shift;
  op->C = C;
  op->relu = relu;
  op->nvec = M * C / 8;
  if (op->nvec >= (1ll << 31)) return set_error(PF_ERR_INVALID, "more than 2^31 vectors (32-bit index decode)");
  *out = std::move(op);
  return PF_OK;
}

int make_bn_bwd_apply_op(OpPtr* out, const void* X, const void* G, const void* Ymask, const float* mean,
                         const float* invstd, const float* gamma, const float* dgamma, const float* dbeta,
                         void* dX, void* dA, int M, int C) {
  if (!X || !G || !mean || !invstd || !gamma || !dgamma || !dbeta || !dX || M <= 0 || C % 8 != 0)
    return set_error(PF_ERR_INVALID, "pf_bn_bwd_apply: bad arguments");
  if (!train::aligned16(X, G, Ymask, dX) || !train::aligned16(dA))
    return set_error(PF_ERR_INVALID, "pf_bn_bwd_apply: 16-B alignment");
  auto op = std::make_unique<train::BnBwdApplyOp>();
  op->x = reinterpret_cast<const bf*>(X);
  op->g = reinterpret_cast<const bf*>(G);
  op->ymask = reinterpret_cast<const bf*>(Ymask);
  op->mean = mean;
  op->invstd = invstd;
  op->gamma = gamma;
  op->dgamma = dgamma;
  op->dbeta = dbeta;
  op->dx = reinterpret_cast<bf*>(dX);
  op->da = reinterpret_cast<bf*>(dA);
  op->M = M;
  op->C = C;
  op->nvec = (long long)M * C / 8;
  if (op->nvec >= (1ll << 31)) return set_error(PF_ERR_INVALID, "more than 2^31 vectors (32-bit index decode)");
  *out = std::move(op);
  return PF_OK;
}

int make_col2im_op(OpPtr* out, const void* dCol, const void* R, void* dX, int B, int H, int W, int C, int kh,
                   int kw, int stride, int pad, int Kp) {
  if (!dCol || !dX || B <= 0 || H <= 0 || W <= 0 || C <= 0 || C % 8 != 0 || Kp < kh * kw * C)
    return set_error(PF_ERR_INVALID, "pf_col2im: bad arguments (C %% 8 == 0)");
  if (!train::aligned16(dCol, R, dX)) return set_error(PF_ERR_INVALID, "pf_col2im: 16-B alignment");
  auto op = std::make_unique<train::Col2imOp>();
  op->dcol = reinterpret_cast<const bf*>(dCol);
  op->r = reinterpret_cast<const bf*>(R);
  op->dx = reinterpret_cast<bf*>(dX);
  op->H = H;
  op->W = W;
  op->C = C;
  op->Ho = (H + 2 * pad - kh) / stride + 1;
  op->Wo = (W + 2 * pad - kw) / stride + 1;
  op->kh = kh;
  op->kw = kw;
  op->stride = stride;
  op->pad = pad;
  op->Kp = Kp;
  op->nvec = (long long)B * H * W * C / 8;
  if (op->nvec >= (1ll << 31)) return set_error(PF_ERR_INVALID, "more than 2^31 vectors (32-bit index decode)");
  *out = std::move(op);
  return PF_OK;
}

int make_maxpool_bwd_op(OpPtr* out, const void* X, const void* dY, void* dX, int B, int H, int W, int C, int k,
                        int stride, int pad) {
  if (!X || !dY || !dX || B <= 0 || C % 8 != 0) return set_error(PF_ERR_INVALID, "pf_maxpool_bwd: bad arguments");
  auto op = std::make_unique<train::PoolBwdOp>();
  op->x = reinterpret_cast<const bf*>(X);
  op->dy = reinterpret_cast<const bf*>(dY);
  op->dx = reinterpret_cast<bf*>(dX);
  op->H = H;
  op->W = W;
  op->C = C;
  op->Ho = (H + 2 * pad - k) / stride + 1;
  op->Wo = (W + 2 * pad - k) / stride + 1;
  op->k = k;
  op->stride = stride;
  op->pad = pad;
  op->nvec = (long long)B * H * W * C / 8;
  if (op->nvec >= (1ll << 31)) return set_error(PF_ERR_INVALID, "more than 2^31 vectors (32-bit index decode)");
  *out = std::move(op);
  return PF_OK;
}

int make_maxpool_bwd_idx_op(OpPtr* out, const void* Idx, const void* dY, void* dX, int B, int H, int W, int C,
                            int k, int stride, int pad) {
  if (!Idx || ((uintptr_t)Idx & 7u) || k > 16)
    return set_error(PF_ERR_INVALID, "pf_maxpool_bwd_argmax: need an 8-B aligned index buffer and k <= 16");
  PF_TRY(make_maxpool_bwd_op(out, dY, dY, dX, B, H, W, C, k, stride, pad));
  static_cast<train::PoolBwdOp*>(out->get())->idx = reinterpret_cast<const uint8_t*>(Idx);
  return PF_OK;
}

int make_avgpool_bwd_op(OpPtr* out, const void* dY, void* dX, int B, int HW, int C) {
  if (!dY || !dX || B <= 0 || HW <= 0 || C % 8 != 0) return set_error(PF_ERR_INVALID, "pf_avgpool_bwd: bad arguments");
  auto op = std::make_unique<train::PoolBwdOp>();
  op->avg = true;
  op->dy = reinterpret_cast<const bf*>(dY);
  op->dx = reinterpret_cast<bf*>(dX);
  op->HW = HW;
  op->C = C;
  op->nvec = (long long)B * HW * C / 8;
  if (op->nvec >= (1ll << 31)) return set_error(PF_ERR_INVALID, "more than 2^31 vectors (32-bit index decode)");
  *out = std::move(op);
  return PF_OK;
}

int make_xent_op(OpPtr* out, const void* Z, const int32_t* labels, float* loss, void* dZ, int B, int N,
                 float grad_scale) {
  if (!Z || !labels || !loss || !dZ || B <= 0 || N <= 0 || N % 8 != 0)
    return set_error(PF_ERR_INVALID, "pf_softmax_xent: bad arguments (N %% 8 == 0)");
  auto op = std::make_unique<train::XentOp>();
  op->z = reinterpret_cast<const bf*>(Z);
  op->labels = labels;
  op->loss = loss;
  op->dz = reinterpret_cast<bf*>(dZ);
  op->B = B;
  op->N = N;
  op->scale = grad_scale;
  *out = std::move(op);
  return PF_OK;
}

int make_sgd_op(OpPtr* out, const pf_sgd_segment_t* segs, int nseg, float lr, float momentum) {
  if (!segs || nseg <= 0 || nseg > train::MAX_SGD_SEGS)
    return set_error(PF_ERR_INVALID, "pf_sgd_update: need 1..256 segments");
  std::vector<train::SgdSeg> hs(nseg);
  int units = 0;
  for (int i = 0; i < nseg; ++i) {
    const pf_sgd_segment_t& s = segs[i];
    if (!s.master || !s.momentum || !s.grad || s.n <= 0 || (s.grad_kind == 0 && s.splits < 1))
      return set_error(PF_ERR_INVALID, "pf_sgd_update: bad segment %d", i);
    train::SgdSeg& d = hs[i];
    d.master = s.master;
    d.mom = s.momentum;
    d.work = reinterpret_cast<bf*>(s.work);
    d.grad = s.grad;
    d.n = s.n;
    d.split_stride = s.split_stride ? s.split_stride : s.n;
    d.splits = s.grad_kind == 0 ? s.splits : 1;
    d.kind = s.grad_kind;
    d.wd = s.weight_decay;
    d.first_unit = units;
    units += (int)((s.n + train::SGD_CHUNK - 1) / train::SGD_CHUNK);
  }
  auto op = std::make_unique<train::SgdOp>();
  PF_CUDA(cudaMalloc(&op->dsegs, sizeof(train::SgdSeg) * nseg));
  PF_CUDA(cudaMemcpy(op->dsegs, hs.data(), sizeof(train::SgdSeg) * nseg, cudaMemcpyHostToDevice));
  op->nseg = nseg;
  op->total_units = units;
  op->lr = lr;
  op->mu = momentum;
  const int cap = 8 * device_sm_count();
  op->grid = units < cap ? units : cap;
  *out = std::move(op);
  return PF_OK;
}

}  // namespace pf

// ------------------------------------------------------------------------------ C ABI

#define PF_RUN_OP(MAKE)                                                         \
  do {                                                                          \
    PF_TRY(pf::validate_ctl(ctl));                                              \
    pf::OpPtr op;                                                               \
    PF_TRY(MAKE);                                                               \
    return op->run(ctl, reinterpret_cast<cudaStream_t>(stream), pf::LaunchArgs{}); \
  } while (0)

extern "C" int pf_transpose(const void* X, void* Y, int R, int C, const pf_ctl_t* ctl, void* stream) {
  PF_RUN_OP(pf::make_transpose_op(&op, X, Y, R, C));
}

extern "C" int pf_colstats(const void* X, const void* G, const void* Ymask, const float* mean,
                           const float* invstd, float* partial, int M, int C, int* out_partials,
                           const pf_ctl_t* ctl, void* stream) {
  PF_RUN_OP(pf::make_colstats_op(&op, X, G, Ymask, mean, invstd, partial, M, C, out_partials));
}

extern "C" int pf_bn_finalize(const float* partial, int P, int M, int C, const float* gamma, const float* beta,
                              float eps, float* mean, float* invstd, float* scale, float* shift,
                              const pf_ctl_t* ctl, void* stream) {
  PF_RUN_OP(pf::make_bn_finalize_op(&op, partial, P, M, C, gamma, beta, eps, mean, invstd, scale, shift));
}

extern "C" int pf_bn_bwd_finalize(const float* partial, int P, int C, float* dgamma, float* dbeta,
                                  const pf_ctl_t* ctl, void* stream) {
  PF_RUN_OP(pf::make_bn_bwd_finalize_op(&op, partial, P, C, dgamma, dbeta));
}

extern "C" int pf_bn_apply(const void* X, const float* scale, const float* shift, const void* R, void* Y,
                           long long M, int C, int relu, const pf_ctl_t* ctl, void* stream) {
  PF_RUN_OP(pf::make_bn_apply_op(&op, X, scale, shift, R, Y, M, C, relu));
}

extern "C" int pf_bn_bwd_apply(const void* X, const void* G, const void* Ymask, const float* mean,
                               const float* invstd, const float* gamma, const float* dgamma, const float* dbeta,
                               void* dX, void* dA, int M, int C, const pf_ctl_t* ctl, void* stream) {
  PF_RUN_OP(pf::make_bn_bwd_apply_op(&op, X, G, Ymask, mean, invstd, gamma, dgamma, dbeta, dX, dA, M, C));
}

extern "C" int pf_col2im(const void* dCol, const void* R, void* dX, int B, int H, int W, int C, int kh, int kw,
                         int stride, int pad, int Kp, const pf_ctl_t* ctl, void* stream) {
  PF_RUN_OP(pf::make_col2im_op(&op, dCol, R, dX, B, H, W, C, kh, kw, stride, pad, Kp));
}

extern "C" int pf_maxpool_bwd(const void* X, const void* dY, void* dX, int B, int H, int W, int C, int k,
                              int stride, int pad, const pf_ctl_t* ctl, void* stream) {
  PF_RUN_OP(pf::make_maxpool_bwd_op(&op, X, dY, dX, B, H, W, C, k, stride, pad));
}

extern "C" int pf_maxpool_bwd_argmax(const uint8_t* Idx, const void* dY, void* dX, int B, int H, int W, int C,
                                     int k, int stride, int pad, const pf_ctl_t* ctl, void* stream) {
  PF_RUN_OP(pf::make_maxpool_bwd_idx_op(&op, Idx, dY, dX, B, H, W, C, k, stride, pad));
}

extern "C" int pf_avgpool_bwd(const void* dY, void* dX, int B, int HW, int C, const pf_ctl_t* ctl,
                              void* stream) {
  PF_RUN_OP(pf::make_avgpool_bwd_op(&op, dY, dX, B, HW, C));
}

extern "C" int pf_softmax_xent(const void* Z, const int32_t* labels, float* loss, void* dZ, int B, int N,
                               float grad_scale, const pf_ctl_t* ctl, void* stream) {
  PF_RUN_OP(pf::make_xent_op(&op, Z, labels, loss, dZ, B, N, grad_scale));
}

extern "C" int pf_sgd_update(const pf_sgd_segment_t* segs, int nseg, float lr, float momentum,
                             const pf_ctl_t* ctl, void* stream) {
  PF_RUN_OP(pf::make_sgd_op(&op, segs, nseg, lr, momentum));
}
