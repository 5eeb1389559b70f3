// pf_ops.h — host-side "prepared" kernel launches: every argument check, tensor-map
// encode and launch-shape decision is done once when a chain is recorded; replaying
// a node is a single kernel launch (pf_chain_launch).
#pragma once

#include <memory>

#include "pf_common.cuh"

namespace pf {

// Per-launch arguments. Copy nodes bound to a batch slice add in_off (role 1, source) or
// out_off (role 2, destination); with `desc` set they instead read the offsets on the
// device from desc[2 * (*idx) + role - 1], so one recorded graph serves every batch.
struct LaunchArgs {
  int64_t in_off = 0;
  int64_t out_off = 0;
  const int64_t* desc = nullptr;
  const uint32_t* idx = nullptr;
  // optional in-kernel timing of this node: [0] = earliest CTA start, [1] = latest CTA end
  // (%globaltimer ns), reset by the chain-begin marker
  unsigned long long* stamp = nullptr;
};

struct PreparedOp {
  virtual ~PreparedOp() {}
  virtual int run(const pf_ctl_t* ctl, cudaStream_t s, const LaunchArgs& a) = 0;
  virtual uint32_t units() const = 0;
  virtual bool resumable() const = 0;  // true: claimed-prefix cursor; false: atomic (re-run whole)
};

using OpPtr = std::unique_ptr<PreparedOp>;

int make_gemm_op(OpPtr* out, const void* X, const void* W, const void* bias, const void* residual,
                 void* Y, int M, int N, int K, uint32_t epi);
int make_gemm_splitk_op(OpPtr* out, const void* X, const void* W, void* Y, int M, int N, int K,
                        int splits);
int make_gemm_mn_op(OpPtr* out, const void* X, const void* W, const void* residual, void* Y, int M, int N, int K,
                    int majors, int splits);
int make_transpose_op(OpPtr* out, const void* X, void* Y, int R, int C);
int make_colstats_op(OpPtr* out, const void* X, const void* G, const void* Ymask, const float* mean,
                     const float* invstd, float* partial, int M, int C, int* out_partials);
int make_bn_finalize_op(OpPtr* out, const float* partial, int P, int M, int C, const float* gamma,
                        const float* beta, float eps, float* mean, float* invstd, float* scale, float* shift);
int make_bn_bwd_finalize_op(OpPtr* out, const float* partial, int P, int C, float* dgamma, float* dbeta);
int make_bn_apply_op(OpPtr* out, const void* X, const float* scale, const float* shift, const void* R, void* Y,
                     long long M, int C, int relu);
int make_bn_bwd_apply_op(OpPtr* out, const void* X, const void* G, const void* Ymask, const float* mean,
                         const float* invstd, const float* gamma, const float* dgamma, const float* dbeta,
                         void* dX, void* dA, int M, int C);
int make_col2im_op(OpPtr* out, const void* dCol, const void* R, void* dX, int B, int H, int W, int C, int kh,
                   int kw, int stride, int pad, int Kp);
int make_maxpool_bwd_op(OpPtr* out, const void* X, const void* dY, void* dX, int B, int H, int W, int C, int k,
                        int stride, int pad);
int make_maxpool_bwd_idx_op(OpPtr* out, const void* Idx, const void* dY, void* dX, int B, int H, int W, int C,
                            int k, int stride, int pad);
int make_avgpool_bwd_op(OpPtr* out, const void* dY, void* dX, int B, int HW, int C);
int make_xent_op(OpPtr* out, const void* Z, const int32_t* labels, float* loss, void* dZ, int B, int N,
                 float grad_scale);
int make_sgd_op(OpPtr* out, const pf_sgd_segment_t* segs, int nseg, float lr, float momentum);
int make_sgemm_op(OpPtr* out, const float* X, const float* W, const float* bias, const float* residual, float* Y,
                  int M, int N, int K, uint32_t epi);
int make_layernorm_f32_op(OpPtr* out, const float* X, const float* residual, const float* gamma, const float* beta,
                          float* Y, int rows, int cols, float eps);
int make_embedding_ln_f32_op(OpPtr* out, const int32_t* ids, const float* word, const float* pos, const float* type,
                             const float* gamma, const float* beta, float* Y, int batch, int seq, int hidden,
                             int vocab, float eps);
int make_attention_f32_op(OpPtr* out, const float* QKV, float* O, int batch, int seq, int heads, int head_dim,
                          float scale);
int make_norm_op(OpPtr* out, bool rms, const void* X, const void* residual, const void* gamma,
                 const void* beta, void* Y, int rows, int cols, float eps);
int make_softmax_op(OpPtr* out, const void* X, void* Y, int rows, int cols, float scale);
int make_embedding_op(OpPtr* out, const int32_t* ids, const int32_t* tt, const void* word,
                      const void* pos, const void* type, const void* gamma, const void* beta,
                      void* Y, int batch, int seq, int hidden, int vocab, float eps);
int make_attention_op(OpPtr* out, const void* QKV, const float* mask, void* O, int batch, int seq,
                      int heads, int head_dim, float scale);
// 2-D copy: `rows` rows of `width` bytes, pitches in bytes; role 1 adds in_off to src,
// role 2 adds out_off to dst. Any UVA addresses (HBM or mapped pinned host).
int make_copy_op(OpPtr* out, void* dst, int64_t dst_pitch, const void* src, int64_t src_pitch,
                 int64_t width, int64_t rows, int role);
int make_im2col_op(OpPtr* out, const void* X, void* Col, int B, int H, int W, int C, int kh, int kw,
                   int stride, int pad, int Kp);
int make_maxpool_op(OpPtr* out, const void* X, void* Y, int B, int H, int W, int C, int k, int stride,
                    int pad, void* Idx = nullptr);
int make_avgpool_op(OpPtr* out, const void* X, void* Y, int B, int HW, int C);

}  // namespace pf
