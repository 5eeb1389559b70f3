/*
 * pipefill.h — C ABI of the B200-native PipeFill fill-job executor (libpipefill.so).
 *
 * The reference (`bubblefill`, /root/reference/pkg) is a pure-Python planner and
 * simulator: it has no FFI, no kernels and no device code. Its executor is a
 * time model — ExecutionPlan.range_wall_us / range_busy_us
 * (pkg/src/bubblefill/partition.py:118-132) consumed by the simulator's
 * dispatch loop (pkg/src/bubblefill/sim.py:222-235). Each entry point below
 * replaces a piece of that time model (or of the paper's DeepSpeed executor,
 * PAPER.md:45-47,422-434) with real sm_100a execution. The cited reference
 * line is the behaviour the entry point realises on the device.
 *
 * Conventions (all entry points):
 *   - plain pointers and sizes only; device pointers are raw CUDA addresses,
 *     `stream` is a cudaStream_t passed as void*; NULL = legacy default stream.
 *   - return 0 (PF_OK) or a negative PF_ERR_* code; no exceptions cross the
 *     ABI. pf_last_error() returns a thread-local message for the last failure.
 *   - every compute kernel is asynchronous and PREEMPTIBLE through pf_ctl_t:
 *     it polls the stage's bubble flag at work-unit (tile / row-block) granularity
 *     and yields when the flag reads 0. Completion vs. yield is read back
 *     afterwards from the control words (pf_ctl_t.cursor, .abort).
 *   - tensors are bf16 row-major unless stated; accumulation is fp32.
 */
#ifndef PIPEFILL_H
#define PIPEFILL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PF_ABI_VERSION 1

#define PF_OK 0
#define PF_ERR_INVALID (-1)     /* bad argument / shape / alignment */
#define PF_ERR_CUDA (-2)        /* a CUDA runtime/driver call failed */
#define PF_ERR_UNSUPPORTED (-3) /* no sm_100a device, or shape outside the kernel's envelope */
#define PF_ERR_OOM (-4)         /* arena exhausted (fill job can never spill past its arena) */

/* Preemption control for one kernel launch.
 *   flag   : device u32, nonzero while the stage is inside a bubble. Set by the
 *            engine's BUBBLE instruction, cleared by the main job's recv completion
 *            (SURVEY §5 "Distributed comm backend"). NULL = run to
 *            completion (non-preemptible, used by parity tests and profiling).
 *   abort  : device u32, sticky. A launch that observes flag==0 sets it and exits;
 *            any later launch of the same chain that sees abort!=0 exits at once
 *            without touching its cursor. Required when flag != NULL.
 *   cursor : device u32 work-claim counter of THIS launch. Work units are claimed
 *            in increasing order, and a claimed unit always completes, so units
 *            [0, min(*cursor, units)) are done: the resume cursor. Relaunching the
 *            same call with the same cursor continues where it stopped. Must be 0
 *            for a fresh launch. Required when flag != NULL.                      */
typedef struct pf_ctl {
  const uint32_t* flag;
  uint32_t* abort;
  uint32_t* cursor;
} pf_ctl_t;

/* ---- runtime --------------------------------------------------------------- */
int pf_abi_version(void);
const char* pf_last_error(void);
/* Fails with PF_ERR_UNSUPPORTED unless the current device is sm_100 (B200). */
int pf_device_check(int* sm_count_out);

/* ---- fixed fill-job arena (no reference code) -------------
 * One cudaMalloc of `bytes`, taken outside the framework caching allocator,
 * sized from measured bubble free memory (min over bubbles of
 * BubbleSpec.free_mem_bytes, pkg/src/bubblefill/pipeline.py:100-121). Bump
 * allocation only; a request that does not fit returns PF_ERR_OOM instead of
 * growing, so the fill job cannot take memory from the main job.                */
typedef struct pf_arena pf_arena_t;
int pf_arena_create(uint64_t bytes, pf_arena_t** out);
int pf_arena_alloc(pf_arena_t* arena, uint64_t bytes, uint64_t align, void** out_dev_ptr);
int pf_arena_mark(pf_arena_t* arena, uint64_t* out_mark);
int pf_arena_release(pf_arena_t* arena, uint64_t mark); /* pop back to a mark */
int pf_arena_reset(pf_arena_t* arena);
int pf_arena_stats(pf_arena_t* arena, uint64_t* capacity, uint64_t* used, uint64_t* high_water);
int pf_arena_base(pf_arena_t* arena, void** out_dev_ptr);
int pf_arena_destroy(pf_arena_t* arena);

/* ---- bubble flag (the BUBBLE instruction) -------------------
 * pf_flag_create allocates a zeroed device u32. pf_flag_write_on_stream enqueues a
 * stream-ordered 32-bit store (cuStreamWriteValue32): the engine writes 1 at the
 * BUBBLE instruction and 0 after the recv that ends the bubble, on its comm stream.
 * pf_flag_clear_at enqueues a one-thread kernel that spins on %globaltimer until
 * *base_ns + offset_ns and then stores 0: the 1-GPU stand-in for the neighbour's
 * send that ends the bubble (artificial bubbles, BASELINE.json north_star).       */
int pf_flag_create(uint32_t** out_dev_flag);
int pf_flag_destroy(uint32_t* dev_flag);
int pf_flag_write_on_stream(uint32_t* dev_flag, uint32_t value, void* stream);
int pf_flag_clear_at(uint32_t* dev_flag, const uint64_t* base_ns, uint64_t offset_ns,
                     uint64_t* stamp_out, void* stream);
/* Enqueue a one-thread kernel that spins until %globaltimer >= (*base_ns + offset_ns) and
 * then throttles an open bubble: flag 1 -> value (value >= 2; a closed flag stays 0).
 * Flag value v >= 2 = "open, at most v CTAs claim work" (cursor-claimed kernels shed the
 * rest): the power-aware bubble tail. No reference counterpart (the
 * reference reserves the tail of every bubble through fill_fraction, pipeline.py:205). */
int pf_flag_throttle_at(uint32_t* dev_flag, const uint64_t* base_ns, uint64_t offset_ns, uint32_t value,
                        void* stream);
/* Enqueue a one-thread kernel that spins until %globaltimer >= (*base_ns + offset_ns)
 * (base_ns may be NULL = 0): the timer-driven stand-in for a recv. If stamp_out is
 * non-NULL it receives the %globaltimer value at release. dev_flag may be NULL.     */
int pf_wait_until(const uint64_t* base_ns, uint64_t offset_ns, uint64_t* stamp_out, void* stream);
/* Enqueue a kernel writing the device %globaltimer (ns) into *dev_out. */
int pf_read_globaltimer(uint64_t* dev_out, void* stream);
/* Enqueue a one-thread kernel that spins spin_ns (<= 10 ms) and writes {start %globaltimer,
 * elapsed ns, elapsed SM cycles} to dev_out3[0..3): the SM clock the main job runs at, read
 * on the device per pipeline op (power-cap interference). No reference
 * counterpart: the reference models slowdown analytically (sim.py:32-56).           */
int pf_sm_clock_probe(uint64_t* dev_out3, uint64_t spin_ns, void* stream);

/* ---- weight / activation staging ------------ */
int pf_host_alloc_pinned(uint64_t bytes, void** out_host_ptr);
int pf_host_free_pinned(void* host_ptr);
int pf_stage_h2d(void* dst_dev, const void* src_pinned_host, uint64_t bytes, void* stream);
int pf_stage_d2h(void* dst_pinned_host, const void* src_dev, uint64_t bytes, void* stream);
/* Chain-aware copy for activation offload/reload between partitions and for a
 * batch's inputs/results: a grid-stride 16-B copy kernel between any
 * two UVA addresses (HBM or mapped pinned host memory), gated by pf_ctl_t like the
 * compute kernels, so copies queued behind a yielded kernel never clobber the
 * buffers its resume needs. bytes % 16 == 0, 16-B aligned. Atomic work unit.     */
int pf_copy(void* dst, const void* src, uint64_t bytes, const pf_ctl_t* ctl, void* stream);
int pf_copy_units(uint64_t bytes, uint32_t* out_units);
/* 2-D variant: `rows` rows of `width` bytes with byte pitches (e.g. gathering the
 * [CLS] rows of a [batch, seq, hidden] activation straight into pinned host memory). */
int pf_copy2d(void* dst, int64_t dst_pitch, const void* src, int64_t src_pitch, int64_t width,
              int64_t rows, const pf_ctl_t* ctl, void* stream);

/* ---- fill-job kernels (the partitioned forward) -------------- */

/* Epilogue bits for pf_gemm. */
#define PF_EPI_BIAS 1u     /* + bias[N]                                   */
#define PF_EPI_GELU 2u     /* exact erf GELU (nn.GELU(approximate='none')) */
#define PF_EPI_RESIDUAL 4u /* + residual[M,N] after the activation        */
#define PF_EPI_RELU 8u     /* max(., 0) last (after bias and residual); not with GELU */

/* Y[M,N] = epi(X[M,K] · W[N,K]^T): nn.Linear layout. tcgen05.mma (kind::f16,
 * fp32 accumulators in TMEM), TMA-fed 4-stage mbarrier pipeline, persistent CTAs,
 * preemptible at output-tile granularity. K % 8 == 0, N % 8 == 0 (16 B rows).
 * Work units = ceil(M/128) * ceil(N/BN) tiles; pf_gemm_units reports them.        */
int pf_gemm(const void* X, const void* W, const void* bias, const void* residual, void* Y,
            int M, int N, int K, uint32_t epilogue, const pf_ctl_t* ctl, void* stream);
int pf_gemm_units(int M, int N, int K, uint32_t* out_units);
/* Split-K GEMM (weight gradients: K = batch x pixels is long, M x N is small):
 * Y[z] = X[:, Kz] · W[:, Kz]^T for the z-th of `splits` K slices (each >= 1 K-block of
 * 64), Y a [splits, M, N] bf16 stack the consumer sums in fp32 (pf_sgd_update).
 * pf_gemm_splitk_splits gives the effective slice count for a request.               */
int pf_gemm_splitk(const void* X, const void* W, void* Y, int M, int N, int K, int splits,
                   const pf_ctl_t* ctl, void* stream);
int pf_gemm_splitk_splits(int K, int requested, int* out_splits);
/* MN-major operands (no transpose kernels for backward passes): pf_gemm_nn computes
 * Y[M,N] = X[M,K] . Wkn[K,N] (+ residual) with Wkn stored [K, N] row-major (a data
 * gradient dZ . W with W as stored); pf_gemm_splitk_tn computes the split-K stack
 * Y[z][M,N] = A[Kz, M]^T . B[Kz, N] with A, B stored [K, M], [K, N] (a weight gradient
 * dZ^T X straight from the activations).                                             */
int pf_gemm_nn(const void* X, const void* Wkn, const void* residual, void* Y, int M, int N, int K,
               const pf_ctl_t* ctl, void* stream);
int pf_gemm_splitk_tn(const void* A, const void* B, void* Y, int M, int N, int K, int splits,
                      const pf_ctl_t* ctl, void* stream);

/* Y = LayerNorm(X + residual) * gamma + beta, per row of `cols` (residual may be
 * NULL). fp32 statistics, two-pass variance. Work units = ceil(rows/rows_per_unit). */
int pf_layernorm(const void* X, const void* residual, const void* gamma, const void* beta,
                 void* Y, int rows, int cols, float eps, const pf_ctl_t* ctl, void* stream);
/* Y = X * rsqrt(mean((X+res)^2) + eps) * gamma. */
int pf_rmsnorm(const void* X, const void* residual, const void* gamma, void* Y, int rows,
               int cols, float eps, const pf_ctl_t* ctl, void* stream);
int pf_norm_units(int rows, int cols, uint32_t* out_units);

/* Row softmax: Y = softmax(X * scale) over `cols`, bf16 in/out, fp32 math.          */
int pf_softmax(const void* X, void* Y, int rows, int cols, float scale, const pf_ctl_t* ctl,
               void* stream);
int pf_softmax_units(int rows, int cols, uint32_t* out_units);

/* Non-causal multi-head attention over a packed QKV tensor, as produced by one
 * [h -> 3h] projection: QKV[batch, seq, 3, heads, head_dim] -> O[batch, seq, heads,
 * head_dim]. O = softmax(Q K^T * scale + mask) V per (batch, head). mask_add may be
 * NULL or an additive fp32 [batch, seq] key mask. seq <= 128, head_dim == 64.
 * Work units = batch * heads.                                                       */
int pf_attention(const void* QKV, const float* mask_add, void* O, int batch, int seq,
                 int heads, int head_dim, float scale, const pf_ctl_t* ctl, void* stream);
int pf_attention_units(int batch, int seq, int heads, int head_dim, uint32_t* out_units);

/* BERT embeddings: Y[t] = LN(word[ids[t]] + pos[t % seq] + type[tt[t]]) (tt may be
 * NULL = segment 0). ids/tt int32 [batch*seq].                                       */
int pf_embedding_ln(const int32_t* ids, const int32_t* type_ids, const void* word,
                    const void* pos, const void* type, const void* gamma, const void* beta,
                    void* Y, int batch, int seq, int hidden, int vocab, float eps,
                    const pf_ctl_t* ctl, void* stream);

/* ---- fp32 fill path (north star: "fp32 path rel 1e-4") -------------------------
 * fp32 storage and math on the SIMT pipes (TF32 tensor cores cannot meet 1e-4):
 * pf_gemm_f32 (epilogue bits BIAS | GELU | RESIDUAL as for pf_gemm; 128x128 tiles claimed
 * through the cursor: resumable), pf_layernorm_f32, pf_embedding_ln_f32 and
 * pf_attention_f32 (seq <= 128, head_dim 64; packed QKV layout as pf_attention).     */
int pf_gemm_f32(const float* X, const float* W, const float* bias, const float* residual, float* Y, int M, int N,
                int K, uint32_t epilogue, const pf_ctl_t* ctl, void* stream);
int pf_layernorm_f32(const float* X, const float* residual, const float* gamma, const float* beta, float* Y,
                     int rows, int cols, float eps, const pf_ctl_t* ctl, void* stream);
int pf_embedding_ln_f32(const int32_t* ids, const float* word, const float* pos, const float* type,
                        const float* gamma, const float* beta, float* Y, int batch, int seq, int hidden, int vocab,
                        float eps, const pf_ctl_t* ctl, void* stream);
int pf_attention_f32(const float* QKV, float* O, int batch, int seq, int heads, int head_dim, float scale,
                     const pf_ctl_t* ctl, void* stream);

/* ---- image kernels of convolutional fill jobs (ResNet-50), NHWC bf16 -------------
 * A convolution = pf_im2col + pf_gemm (BatchNorm folded into the GEMM weights/bias,
 * ReLU / residual in its epilogue). Col[B*Ho*Wo, Kp], column (ky*kw + kx)*C + c,
 * zeros outside the image and in columns kh*kw*C..Kp; Kp % 8 == 0.
 * Atomic work units; pf_image_units(kind 0 = im2col with out_elems = rows*Kp,
 * kind 1 = max pooling, kind 2 = average pooling, out_elems = output pixels * C): the
 * launch's CTA count, capped at the kernel's resident CTAs per SM x SMs.              */
int pf_im2col(const void* X, void* Col, int B, int H, int W, int C, int kh, int kw, int stride,
              int pad, int Kp, const pf_ctl_t* ctl, void* stream);
/* k x k max pooling (padding never wins: -inf), C % 8 == 0.                           */
int pf_maxpool(const void* X, void* Y, int B, int H, int W, int C, int k, int stride, int pad,
               const pf_ctl_t* ctl, void* stream);
/* Global average pooling X[B, HW, C] -> Y[B, C], fp32 sums.                            */
int pf_avgpool(const void* X, void* Y, int B, int HW, int C, const pf_ctl_t* ctl, void* stream);
int pf_image_units(int kind, long long out_elems, int C, uint32_t* out_units);

/* ---- training fill jobs (ResNet-50 fwd + bwd + SGD), NHWC bf16 as [M, C] --------
 * BatchNorm batch statistics: pf_colstats writes per-CTA partials (sum x, sum x^2) of
 * X[M, C] (or, with G given, (sum dA, sum dA*xhat), dA = G*[Ymask > 0]) to
 * partial[P, 2C] fp32 and reports P (<= 1024); pf_bn_finalize turns them into mean,
 * invstd and scale = gamma*invstd, shift = beta - mean*scale; pf_bn_bwd_finalize into
 * dbeta (= column sums) and dgamma (may be NULL). pf_bn_apply: Y = act(X*scale + shift
 * [+ R]). pf_bn_bwd_apply: dX = gamma*invstd*(dA - dbeta/M - xhat*dgamma/M), dA
 * optionally written too. C % 8 == 0, C <= 2048.                                     */
int pf_colstats(const void* X, const void* G, const void* Ymask, const float* mean, const float* invstd,
                float* partial, int M, int C, int* out_partials, const pf_ctl_t* ctl, void* stream);
int pf_bn_finalize(const float* partial, int P, int M, int C, const float* gamma, const float* beta,
                   float eps, float* mean, float* invstd, float* scale, float* shift, const pf_ctl_t* ctl,
                   void* stream);
int pf_bn_bwd_finalize(const float* partial, int P, int C, float* dgamma, float* dbeta,
                       const pf_ctl_t* ctl, void* stream);
int pf_bn_apply(const void* X, const float* scale, const float* shift, const void* R, void* Y, long long M,
                int C, int relu, const pf_ctl_t* ctl, void* stream);
int pf_bn_bwd_apply(const void* X, const void* G, const void* Ymask, const float* mean, const float* invstd,
                    const float* gamma, const float* dgamma, const float* dbeta, void* dX, void* dA, int M,
                    int C, const pf_ctl_t* ctl, void* stream);
/* Y[C, R] = X[R, C]^T (bf16), the operand layout of dgrad / wgrad GEMMs.              */
int pf_transpose(const void* X, void* Y, int R, int C, const pf_ctl_t* ctl, void* stream);
/* Inverse of pf_im2col as a gather: dX = sum of the dCol entries that read each input
 * element [+ R] (deterministic, no atomics).                                           */
int pf_col2im(const void* dCol, const void* R, void* dX, int B, int H, int W, int C, int kh, int kw,
              int stride, int pad, int Kp, const pf_ctl_t* ctl, void* stream);
/* Max-pool backward: the gradient goes to the first maximum of each window.          */
int pf_maxpool_bwd(const void* X, const void* dY, void* dX, int B, int H, int W, int C, int k, int stride,
                   int pad, const pf_ctl_t* ctl, void* stream);
int pf_avgpool_bwd(const void* dY, void* dX, int B, int HW, int C, const pf_ctl_t* ctl, void* stream);
/* Max pooling that also writes the window position (wy * k + wx, uint8, k <= 16) of each
 * output's first maximum, and the backward that reads it instead of re-scanning X:
 * training's stem (torch's max_pool2d "first maximum" rule; bit-identical to pf_maxpool /
 * pf_maxpool_bwd). Idx is [B, Ho, Wo, C] bytes, 8-B aligned.                            */
int pf_maxpool_argmax(const void* X, void* Y, uint8_t* Idx, int B, int H, int W, int C, int k, int stride,
                      int pad, const pf_ctl_t* ctl, void* stream);
int pf_maxpool_bwd_argmax(const uint8_t* Idx, const void* dY, void* dX, int B, int H, int W, int C, int k,
                          int stride, int pad, const pf_ctl_t* ctl, void* stream);
/* Softmax cross-entropy, warp per row: loss[4*b] = logsumexp(Z_b) - Z_b[label_b],
 * dZ = (softmax(Z) - onehot) * grad_scale. labels int32, 4-word stride per sample.   */
int pf_softmax_xent(const void* Z, const int32_t* labels, float* loss, void* dZ, int B, int N,
                    float grad_scale, const pf_ctl_t* ctl, void* stream);
/* SGD with momentum over parameter segments in one launch: g = sum of `splits` bf16
 * partials (grad_kind 0, split_stride elements apart) or fp32 (grad_kind 1);
 * g += weight_decay*w; v = momentum*v + g; w -= lr*v on the fp32 master; the bf16
 * working copy (may be NULL) is rewritten. Claims 4096-element units through the
 * cursor (resumable prefix: never applies an update twice).                         */
typedef struct {
  float* master;
  float* momentum;
  void* work;
  const void* grad;
  long long n;
  long long split_stride;
  int splits;
  int grad_kind;
  float weight_decay;
} pf_sgd_segment_t;
int pf_sgd_update(const pf_sgd_segment_t* segs, int nseg, float lr, float momentum, const pf_ctl_t* ctl,
                  void* stream);

/* ---- chain control ------------------------------------------------------------
 * Resets the per-node cursors of a chain when the chain has not been aborted
 * (a one-thread kernel: `if (!*abort) cursors[0..n) = 0`), and counts completed
 * chain runs (`if (!*abort) ++*done`). Used to bracket one batch of a partition. */
int pf_chain_begin(uint32_t* cursors, int n, const uint32_t* abort, void* stream);
int pf_chain_end(uint32_t* done_counter, const uint32_t* abort, void* stream);

/* ---- recorded chains: one batch of one partition --------------------------------
 * The Executor records the kernel sequence of "partition [lo, hi) at batch size b"
 * once (argument checks, TMA descriptors, launch shapes resolved at record time) and
 * replays it per batch with a single pf_chain_launch: node i gets pf_ctl_t
 * {flag, abort, cursors + i}; start_node > 0 resumes a yielded batch at its first
 * incomplete node (no cursor reset); copy nodes with role 1/2 add in_off to their
 * source / out_off to their destination (the batch's slice of the range's inputs /
 * outputs). With done != NULL a chain-end marker counts completed batches.
 * This replaces the reference's per-range time model (partition.py:118-132) with
 * the actual per-batch launch sequence of the paper's Executor.   */
typedef struct pf_chain pf_chain_t;
int pf_chain_create(pf_chain_t** out);
int pf_chain_destroy(pf_chain_t* chain);
int pf_chain_add_gemm(pf_chain_t* chain, const void* X, const void* W, const void* bias,
                      const void* residual, void* Y, int M, int N, int K, uint32_t epilogue);
int pf_chain_add_layernorm(pf_chain_t* chain, const void* X, const void* residual,
                           const void* gamma, const void* beta, void* Y, int rows, int cols,
                           float eps);
int pf_chain_add_rmsnorm(pf_chain_t* chain, const void* X, const void* residual, const void* gamma,
                         void* Y, int rows, int cols, float eps);
int pf_chain_add_softmax(pf_chain_t* chain, const void* X, void* Y, int rows, int cols,
                         float scale);
int pf_chain_add_attention(pf_chain_t* chain, const void* QKV, const float* mask_add, void* O,
                           int batch, int seq, int heads, int head_dim, float scale);
int pf_chain_add_embedding_ln(pf_chain_t* chain, const int32_t* ids, const int32_t* type_ids,
                              const void* word, const void* pos, const void* type,
                              const void* gamma, const void* beta, void* Y, int batch, int seq,
                              int hidden, int vocab, float eps);
int pf_chain_add_copy(pf_chain_t* chain, void* dst, int64_t dst_pitch, const void* src,
                      int64_t src_pitch, int64_t width, int64_t rows, int role);  /* role 0..3 */
int pf_chain_add_gemm_splitk(pf_chain_t* chain, const void* X, const void* W, void* Y, int M, int N,
                             int K, int splits);
int pf_chain_add_gemm_nn(pf_chain_t* chain, const void* X, const void* Wkn, const void* residual, void* Y, int M,
                         int N, int K);
int pf_chain_add_gemm_splitk_tn(pf_chain_t* chain, const void* A, const void* B, void* Y, int M, int N, int K,
                                int splits);
int pf_chain_add_colstats(pf_chain_t* chain, const void* X, const void* G, const void* Ymask,
                          const float* mean, const float* invstd, float* partial, int M, int C,
                          int* out_partials);
int pf_chain_add_bn_finalize(pf_chain_t* chain, const float* partial, int P, int M, int C, const float* gamma,
                             const float* beta, float eps, float* mean, float* invstd, float* scale,
                             float* shift);
int pf_chain_add_bn_bwd_finalize(pf_chain_t* chain, const float* partial, int P, int C, float* dgamma,
                                 float* dbeta);
int pf_chain_add_bn_apply(pf_chain_t* chain, const void* X, const float* scale, const float* shift,
                          const void* R, void* Y, long long M, int C, int relu);
int pf_chain_add_bn_bwd_apply(pf_chain_t* chain, const void* X, const void* G, const void* Ymask,
                              const float* mean, const float* invstd, const float* gamma, const float* dgamma,
                              const float* dbeta, void* dX, void* dA, int M, int C);
int pf_chain_add_transpose(pf_chain_t* chain, const void* X, void* Y, int R, int C);
int pf_chain_add_col2im(pf_chain_t* chain, const void* dCol, const void* R, void* dX, int B, int H, int W,
                        int C, int kh, int kw, int stride, int pad, int Kp);
int pf_chain_add_maxpool_bwd(pf_chain_t* chain, const void* X, const void* dY, void* dX, int B, int H, int W,
                             int C, int k, int stride, int pad);
int pf_chain_add_avgpool_bwd(pf_chain_t* chain, const void* dY, void* dX, int B, int HW, int C);
int pf_chain_add_maxpool_argmax(pf_chain_t* chain, const void* X, void* Y, uint8_t* Idx, int B, int H, int W,
                                int C, int k, int stride, int pad);
int pf_chain_add_maxpool_bwd_argmax(pf_chain_t* chain, const uint8_t* Idx, const void* dY, void* dX, int B,
                                    int H, int W, int C, int k, int stride, int pad);
int pf_chain_add_softmax_xent(pf_chain_t* chain, const void* Z, const int32_t* labels, float* loss, void* dZ,
                              int B, int N, float grad_scale);
int pf_chain_add_sgd(pf_chain_t* chain, const pf_sgd_segment_t* segs, int nseg, float lr, float momentum);
int pf_chain_add_gemm_f32(pf_chain_t* chain, const float* X, const float* W, const float* bias,
                          const float* residual, float* Y, int M, int N, int K, uint32_t epilogue);
int pf_chain_add_layernorm_f32(pf_chain_t* chain, const float* X, const float* residual, const float* gamma,
                               const float* beta, float* Y, int rows, int cols, float eps);
int pf_chain_add_embedding_ln_f32(pf_chain_t* chain, const int32_t* ids, const float* word, const float* pos,
                                  const float* type, const float* gamma, const float* beta, float* Y, int batch,
                                  int seq, int hidden, int vocab, float eps);
int pf_chain_add_attention_f32(pf_chain_t* chain, const float* QKV, float* O, int batch, int seq, int heads,
                               int head_dim, float scale);
int pf_chain_add_im2col(pf_chain_t* chain, const void* X, void* Col, int B, int H, int W, int C,
                        int kh, int kw, int stride, int pad, int Kp);
int pf_chain_add_maxpool(pf_chain_t* chain, const void* X, void* Y, int B, int H, int W, int C,
                         int k, int stride, int pad);
int pf_chain_add_avgpool(pf_chain_t* chain, const void* X, void* Y, int B, int HW, int C);
int pf_chain_size(pf_chain_t* chain, int* out_nodes);
/* units = work units of the node; resumable = 1 for claimed-prefix nodes (GEMM tiles),
 * 0 for atomic nodes that are re-run whole (cursor must be reset to 0 first).       */
int pf_chain_node_info(pf_chain_t* chain, int node, uint32_t* out_units, int* out_resumable);
/* Device-side batch descriptors: with desc set, copy nodes of role r in 1..3 take
 * their batch-slice offset from desc[PF_DESC_WORDS * (*done) + r - 1] (int64 words in
 * device memory), so one recorded graph serves every batch of a bubble. Role 1 adds
 * it to the source (the batch's inputs), role 2 to the destination (its results),
 * role 3 to the source (a second input stream, e.g. a training job's labels).      */
#define PF_DESC_WORDS 4
int pf_chain_set_desc(pf_chain_t* chain, const int64_t* desc);
/* In-kernel timing: node i of a launch writes [earliest CTA start, latest CTA end]
 * (%globaltimer ns) to stamps[2i], stamps[2i+1] (GEMM nodes; reset at chain begin).   */
int pf_chain_set_stamps(pf_chain_t* chain, uint64_t* stamps);
/* Record the chain as a CUDA graph with device-side gating: after the chain-begin
 * marker, every segment [seg_ends[i-1], seg_ends[i]) of nodes sits in a conditional IF
 * node preceded by a one-thread gate kernel that checks abort / the bubble flag; a
 * closed bubble skips the remaining segments on the device (no launches). Then one
 * pf_chain_graph_launch per batch.                                                   */
int pf_chain_build_graph(pf_chain_t* chain, const uint32_t* flag, uint32_t* abort,
                         uint32_t* cursors, uint32_t* done, const int* seg_ends, int n_segs);
int pf_chain_graph_launch(pf_chain_t* chain, void* stream);
/* Live per-node device timing (CUDA events around every node of the next launches);
 * pf_chain_node_elapsed returns the last launch's duration of `node` in ms.        */
int pf_chain_set_timing(pf_chain_t* chain, int enable);
int pf_chain_node_elapsed(pf_chain_t* chain, int node, float* out_ms);
int pf_chain_launch(pf_chain_t* chain, const uint32_t* flag, uint32_t* abort, uint32_t* cursors,
                    uint32_t* done, int start_node, int64_t in_off, int64_t out_off, void* stream);

/* ---- gated weight staging (run-ahead into the next partition) -------------------
 * One partition's weights as a CUDA graph: a one-thread gate kernel, then a
 * conditional IF node whose body is one host->device memcpy node per (dst, pinned src,
 * bytes). The gate lets the copies run only when the chain-abort word is 0 -- i.e.
 * every batch enqueued before it on the stream completed -- and writes the decision
 * to *staged_out (1 = staged). A run-ahead staging behind a batch that yielded is
 * therefore skipped and cannot overwrite the yielded batch's weights or workspace
 * (the region holds one partition at a time). No reference counterpart:
 * the reference charges partitions whole cycles (partition.py:118-124). Copies may go
 * either way (cudaMemcpyDefault): a partitioned training job writes the updated state of
 * the resident partition back to its pinned blob and stages the next one in one graph. */
typedef struct pf_staging pf_staging_t;
int pf_staging_create(pf_staging_t** out, void* const* dst, const void* const* src,
                      const uint64_t* bytes, int n, const uint32_t* abort, uint32_t* staged_out);
int pf_staging_launch(pf_staging_t* staging, void* stream);
int pf_staging_destroy(pf_staging_t* staging);

#ifdef __cplusplus
}
#endif
#endif /* PIPEFILL_H */
