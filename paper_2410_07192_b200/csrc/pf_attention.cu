// pf_attention.cu — non-causal multi-head attention for the fill job's encoder
// layers (BERT: seq 128, head_dim 64), one CTA per (batch, head), on tcgen05.
//
//   S = Q K^T        tcgen05.mma 128x128x64, fp32 accumulators in TMEM cols [0,128)
//   P = exp(S*scale - rowmax)  (+ optional additive key mask; keys >= seq masked)
//       thread-per-query-row softmax straight out of TMEM (tcgen05.ld), P packed to
//       bf16 into shared memory in the UMMA K-major 128-B-swizzled layout, reusing
//       the dead Q/K tiles
//   O = P V          tcgen05.mma 128x64x128 with V as an MN-major operand, into TMEM cols
//       [0,64) over the consumed S, normalised by the fp32 row sum in the epilogue
// Q, K, V tiles arrive by one 3-D TMA each from the packed QKV projection output
// [batch*seq, 3, heads, 64]; no transpose or split kernel runs before attention.
// Preemption: atomic work unit = one (batch, head); flag checked on entry.
#include "pf_ops.h"

namespace pf {
namespace attn {

constexpr int S_MAX = 128;
constexpr int D = 64;
constexpr int THREADS = 128;
constexpr int TILE_BYTES = S_MAX * D * 2;  // 16 KB per operand tile
// Q | K | V tiles (P overwrites Q|K) and barriers: ~49 KB, so 4 CTAs share an SM; each
// allocates 128 of the SM's 512 TMEM columns (O = PV reuses the consumed S columns).
constexpr int SMEM_BYTES = 1024 + 3 * TILE_BYTES + 64;
constexpr int SMEM_REQUEST = SMEM_BYTES;
constexpr int TMEM_COLS = 128;

__global__ void __launch_bounds__(THREADS) attention_kernel(const __grid_constant__ CUtensorMap tm,
                                                            const float* __restrict__ mask_add,
                                                            __nv_bfloat16* __restrict__ O,
                                                            int batch, int seq, int heads,
                                                            float scale_log2, Ctl ctl) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = smem + TILE_BYTES;
  uint8_t* sV = smem + 2 * TILE_BYTES;
  uint8_t* sP = smem;  // 2 K-blocks of [128][64] bf16 over the dead Q and K tiles
  uint64_t* tma_bar = reinterpret_cast<uint64_t*>(smem + 3 * TILE_BYTES);
  uint64_t* mma_bar = tma_bar + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mma_bar + 1);
  __shared__ int s_go;

  const int tid = threadIdx.x;
  const int warp = warp_id();
  const int lane = lane_id();
  const int b = blockIdx.x / heads;
  const int h = blockIdx.x % heads;

  if (tid == 0) {
    int go = 1;
    if (chain_aborted(ctl)) go = 0;
    else if (ctl.flag != nullptr && ld_acquire_u32(ctl.flag) == 0u) {
      atomicExch(ctl.abort, 1u);
      go = 0;
    }
    s_go = go;
    if (go) {
      mbar_init(tma_bar, 1);
      mbar_init(mma_bar, 1);
      fence_barrier_init();
    }
  }
  __syncthreads();
  if (!s_go) return;
  if (warp == 0) tmem_alloc(tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (tid == 0) {
    tma_prefetch_desc(&tm);
    mbar_arrive_expect_tx(tma_bar, 3 * TILE_BYTES);
    const int row0 = b * seq;
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(sQ)),
        "l"(reinterpret_cast<uint64_t>(&tm)), "r"(smem_u32(tma_bar)), "r"(0), "r"(h), "r"(row0)
        : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(sK)),
        "l"(reinterpret_cast<uint64_t>(&tm)), "r"(smem_u32(tma_bar)), "r"(0), "r"(heads + h),
        "r"(row0)
        : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(sV)),
        "l"(reinterpret_cast<uint64_t>(&tm)), "r"(smem_u32(tma_bar)), "r"(0), "r"(2 * heads + h),
        "r"(row0)
        : "memory");
  }
  mbar_wait(tma_bar, 0);

  // ---- S = Q K^T ----
  if (tid == 0) {
    tc_fence_after();
    constexpr uint32_t idesc_s = umma_idesc_bf16(128, 128, false, false);
    const uint32_t qa = smem_u32(sQ), ka = smem_u32(sK);
#pragma unroll
    for (int k = 0; k < D / 16; ++k)
      umma_bf16_ss(tmem, umma_desc_sw128_kmajor(qa + k * 32), umma_desc_sw128_kmajor(ka + k * 32),
                   idesc_s, k > 0 ? 1u : 0u);
    umma_commit(mma_bar);
  }
  mbar_wait(mma_bar, 0);
  tc_fence_after();

  // ---- softmax: thread `tid` owns query row `tid` (TMEM lane tid) ----
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  const float* mrow = mask_add ? mask_add + (size_t)b * seq : nullptr;
  float mx = -INFINITY;
#pragma unroll 1
  for (int c = 0; c < 4; ++c) {
    uint32_t r[32];
    tmem_ld_32x32b_x32(tmem + lane_base + c * 32, r);
    tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int key = c * 32 + j;
      float s = __uint_as_float(r[j]) * scale_log2;
      if (mrow && key < seq) s += mrow[key] * 1.4426950408889634f;
      if (key >= seq) s = -INFINITY;
      mx = fmaxf(mx, s);
    }
  }
  float sum = 0.f;
  const int row = tid;
#pragma unroll 1
  for (int c = 0; c < 4; ++c) {
    uint32_t r[32];
    tmem_ld_32x32b_x32(tmem + lane_base + c * 32, r);
    tmem_ld_wait();
    uint32_t packed[16];
#pragma unroll
    for (int j = 0; j < 32; j += 2) {
      float p2[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int key = c * 32 + j + u;
        float s = __uint_as_float(r[j + u]) * scale_log2;
        if (mrow && key < seq) s += mrow[key] * 1.4426950408889634f;
        p2[u] = key < seq ? exp2f(s - mx) : 0.f;
        sum += p2[u];
      }
      packed[j / 2] = pack_bf16x2(p2[0], p2[1]);
    }
    // keys [32c, 32c+32) live in K-block c/2, 16-B chunks (c%2)*4 .. +4 of the 128-B row
    uint8_t* blk = sP + (c >> 1) * TILE_BYTES + row * 128;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int chunk = (c & 1) * 4 + q;
      uint4 v = make_uint4(packed[4 * q], packed[4 * q + 1], packed[4 * q + 2], packed[4 * q + 3]);
      *reinterpret_cast<uint4*>(blk + ((chunk ^ (row & 7)) << 4)) = v;
    }
  }
  fence_async_smem();  // generic-proxy P stores -> visible to the tensor core (async proxy)
  tc_fence_before();
  __syncthreads();

  // ---- O = P V ----
  if (tid == 0) {
    tc_fence_after();
    constexpr uint32_t idesc_o = umma_idesc_bf16(128, D, false, true);
    const uint32_t pa = smem_u32(sP), va = smem_u32(sV);
#pragma unroll
    for (int k = 0; k < S_MAX / 16; ++k) {
      const uint64_t ad = umma_desc_sw128_kmajor(pa + (k >> 2) * TILE_BYTES + (k & 3) * 32);
      const uint64_t bd = umma_desc_sw128_mnmajor(va + k * 2048, TILE_BYTES);
      umma_bf16_ss(tmem, ad, bd, idesc_o, k > 0 ? 1u : 0u);  // over the consumed S
    }
    umma_commit(mma_bar);
  }
  mbar_wait(mma_bar, 1);
  tc_fence_after();

  const float inv = 1.f / sum;
  const bool row_ok = row < seq;
  __nv_bfloat16* orow = O + ((size_t)(b * seq + row) * heads + h) * D;
#pragma unroll 1
  for (int c = 0; c < 2; ++c) {
    uint32_t r[32];
    tmem_ld_32x32b_x32(tmem + lane_base + c * 32, r);
    tmem_ld_wait();
    if (row_ok) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 v;
        v.x = pack_bf16x2(__uint_as_float(r[8 * q + 0]) * inv, __uint_as_float(r[8 * q + 1]) * inv);
        v.y = pack_bf16x2(__uint_as_float(r[8 * q + 2]) * inv, __uint_as_float(r[8 * q + 3]) * inv);
        v.z = pack_bf16x2(__uint_as_float(r[8 * q + 4]) * inv, __uint_as_float(r[8 * q + 5]) * inv);
        v.w = pack_bf16x2(__uint_as_float(r[8 * q + 6]) * inv, __uint_as_float(r[8 * q + 7]) * inv);
        *reinterpret_cast<uint4*>(orow + c * 32 + q * 8) = v;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, TMEM_COLS);
  if (tid == 0 && ctl.cursor != nullptr) {
    __threadfence();
    atomicAdd(ctl.cursor, 1u);
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  return fn;
}

struct AttentionOp final : PreparedOp {
  CUtensorMap tm;
  const float* mask = nullptr;
  __nv_bfloat16* out = nullptr;
  int batch = 0, seq = 0, heads = 0;
  float scale_log2 = 0.f;
  uint32_t units() const override { return (uint32_t)(batch * heads); }
  bool resumable() const override { return false; }
  int run(const pf_ctl_t* ctl, cudaStream_t s, const LaunchArgs&) override {
    attention_kernel<<<batch * heads, THREADS, SMEM_REQUEST, s>>>(tm, mask, out, batch, seq, heads,
                                                                  scale_log2, make_ctl(ctl));
    PF_CUDA(cudaGetLastError());
    return PF_OK;
  }
};

}  // namespace attn

int make_attention_op(OpPtr* out, const void* QKV, const float* mask_add, void* O, int batch,
                      int seq, int heads, int head_dim, float scale) {
  using namespace attn;
  if (!QKV || !O || batch <= 0 || heads <= 0 || seq <= 0)
    return set_error(PF_ERR_INVALID, "pf_attention: bad arguments");
  if (head_dim != D || seq > S_MAX)
    return set_error(PF_ERR_UNSUPPORTED, "pf_attention: needs head_dim == 64 and seq <= 128");
  if (((uintptr_t)QKV | (uintptr_t)O) & 15u)
    return set_error(PF_ERR_INVALID, "pf_attention: pointers must be 16-B aligned");
  if (!device_is_sm100()) return set_error(PF_ERR_UNSUPPORTED, "pf_attention: needs sm_100");
  static bool attr = false;
  if (!attr) {
    PF_CUDA(cudaFuncSetAttribute(attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 SMEM_REQUEST));
    attr = true;
  }
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return set_error(PF_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  auto op = std::make_unique<AttentionOp>();
  // QKV viewed as [batch*seq][3*heads][64]; box = one head slot x 128 tokens
  cuuint64_t dims[3] = {(cuuint64_t)D, (cuuint64_t)(3 * heads), (cuuint64_t)batch * seq};
  cuuint64_t strides[2] = {(cuuint64_t)D * 2, (cuuint64_t)3 * heads * D * 2};
  cuuint32_t box[3] = {(cuuint32_t)D, 1, (cuuint32_t)S_MAX};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(&op->tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(QKV), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(PF_ERR_CUDA, "attention tensor map failed (%d)", (int)r);
  op->mask = mask_add;
  op->out = reinterpret_cast<__nv_bfloat16*>(O);
  op->batch = batch;
  op->seq = seq;
  op->heads = heads;
  op->scale_log2 = scale * 1.4426950408889634f;
  *out = std::move(op);
  return PF_OK;
}

}  // namespace pf

extern "C" int pf_attention_units(int batch, int seq, int heads, int head_dim, uint32_t* out) {
  if (!out || batch <= 0 || heads <= 0 || seq <= 0)
    return pf::set_error(PF_ERR_INVALID, "pf_attention_units");
  *out = (uint32_t)(batch * heads);
  return PF_OK;
}

extern "C" int pf_attention(const void* QKV, const float* mask_add, void* O, int batch, int seq,
                            int heads, int head_dim, float scale, const pf_ctl_t* ctl,
                            void* stream) {
  PF_TRY(pf::validate_ctl(ctl));
  pf::OpPtr op;
  PF_TRY(pf::make_attention_op(&op, QKV, mask_add, O, batch, seq, heads, head_dim, scale));
  return op->run(ctl, reinterpret_cast<cudaStream_t>(stream), pf::LaunchArgs{});
}
