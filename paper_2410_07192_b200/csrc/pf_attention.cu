// pf_attention.cu — non-causal multi-head attention for the fill job's encoder
// layers (BERT: seq <= 128, head_dim 64) on tcgen05, as a persistent, warp-specialised
// kernel: 2 CTAs per SM, each striding over (batch, head) units with a 2-deep pipeline,
// so the TMA loads of unit i+1 and the S MMA of unit i+1 overlap the softmax of unit i.
//
//   warp 0 (lane 0)  producer: Q, K, V of a unit by three 3-D TMA loads from the packed
//                    QKV projection output [batch*seq, 3, heads, 64] into stage i%2
//                    (no transpose or split kernel runs before attention); polls the
//                    bubble flag before every unit
//   warp 1 (lane 0)  MMA: S = Q K^T (128x128x64) into TMEM buffer i%2, then, once P is in
//                    shared memory, O = P V (128x64x128, V as an MN-major operand) over the
//                    consumed S columns
//   warps 2..9       softmax: two warps per 32-row TMEM lane quarter, one per 64-key half;
//                    row max exchanged through shared memory; P = exp2(S*scale*log2e - max)
//                    packed to bf16 straight into the UMMA K-major SW128 layout over the
//                    unit's dead Q/K tiles; row sums to shared memory (double-buffered)
//   warps 10..13     epilogue: O of unit i normalised by the fp32 row sum and stored (one
//                    128-B row per thread) while the softmax warps already run unit i+1
// Preemption: persistent atomic unit. The producer re-reads the flag before each unit; on
// a closed bubble it sets abort and the CTA drains and exits without counting itself, so
// the node stays incomplete and is re-run whole on resume (units() = CTAs launched).
#include "pf_ops.h"

namespace pf {
namespace attn {

constexpr int S_MAX = 128;
constexpr int D = 64;
constexpr int THREADS = 448;  // 14 warps: producer, MMA, 8 softmax, 4 epilogue
constexpr int STAGES = 2;
constexpr int TILE_BYTES = S_MAX * D * 2;        // 16 KB per operand tile
constexpr int STAGE_BYTES = 3 * TILE_BYTES;      // Q | K | V (P overwrites Q|K)
constexpr int TMEM_COLS = 256;                   // 2 buffers x 128 columns (S, then O over S)
constexpr int CTAS_PER_SM = 2;

struct Shared {
  uint64_t full[STAGES], empty[STAGES];           // TMA -> MMA, MMA(O done) -> TMA
  uint64_t s_full[STAGES], p_ready[STAGES];       // MMA(S) -> softmax, softmax(P) -> MMA
  uint64_t o_full[STAGES], t_empty[STAGES];       // MMA(O) -> epilogue, epilogue -> MMA
  uint32_t tmem_slot;
};
constexpr int SMEM_REQUEST = 1024 + STAGES * STAGE_BYTES + (int)sizeof(Shared);

// Non-blocking probe: has the phase with this parity completed?
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(done)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return done != 0;
}

// Blocking wait with a suspend-time hint (ns): parks until the phase completes or the hint
// expires; returns whether it completed.
__device__ __forceinline__ bool mbar_try_wait_hint(uint64_t* bar, uint32_t parity, uint32_t ns) {
  uint32_t done;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(done)
      : "r"(smem_u32(bar)), "r"(parity), "r"(ns)
      : "memory");
  return done != 0;
}

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

__device__ __forceinline__ void softmax_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

#ifdef PF_ATT_DIAG
// diagnostic build: per-CTA, per-unit phase clocks (SM cycles since the CTA's start)
__device__ uint32_t g_att_diag[296][8][8];
#define ATT_STAMP(i, ev) \
  do { if ((i) < 8 && blockIdx.x < 296) g_att_diag[blockIdx.x][(i)][(ev)] = (uint32_t)(clock64() - t_start); } while (0)
#else
#define ATT_STAMP(i, ev) do {} while (0)
#endif

__device__ __forceinline__ void tma_qkv(const CUtensorMap* tm, uint8_t* dst, uint64_t* bar, int slot,
                                        int row0) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(smem_u32(bar)), "r"(0), "r"(slot), "r"(row0)
      : "memory");
}

// FULL: seq == 128 and no key mask (the fill job's BERT batches): the softmax is pure
// FMNMX / FFMA / MUFU.EX2 per key; otherwise keys >= seq and the additive mask are applied.
template <bool FULL>
__global__ void __launch_bounds__(THREADS, CTAS_PER_SM)
    attention_kernel(const __grid_constant__ CUtensorMap tm, const float* __restrict__ mask_add,
                     __nv_bfloat16* __restrict__ O, int batch, int seq, int heads, float scale_log2,
                     Ctl ctl) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  Shared& sh = *reinterpret_cast<Shared*>(smem + STAGES * STAGE_BYTES);
  __shared__ float s_red[2][S_MAX];      // per-half row max (softmax warps only)
  __shared__ float s_sums[2][2][S_MAX];  // [unit & 1][half][row] row sums -> epilogue
  __shared__ int s_stop_at;              // first unit index this CTA will not run
  __shared__ int s_go;
  volatile int* stop_at = &s_stop_at;

  const int tid = threadIdx.x;
  const int warp = warp_id();
  const int lane = lane_id();
  const int units = batch * heads;
  const int n_mine = (int)blockIdx.x < units ? (units - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;

  pdl_enter();
  if (tid == 0) {
    int go = 1;
    if (chain_aborted(ctl)) go = 0;
    else if (ctl.flag != nullptr && ld_acquire_u32(ctl.flag) == 0u) {
      atomicExch(ctl.abort, 1u);
      go = 0;
    }
    s_go = go;
    s_stop_at = 0x7fffffff;
    if (go) {
      for (int s = 0; s < STAGES; ++s) {
        mbar_init(&sh.full[s], 1);
        mbar_init(&sh.empty[s], 1);
        mbar_init(&sh.s_full[s], 1);
        mbar_init(&sh.p_ready[s], 1);
        mbar_init(&sh.o_full[s], 1);
        mbar_init(&sh.t_empty[s], 4);  // one arrive per epilogue warp
      }
      fence_barrier_init();
    }
  }
  __syncthreads();
  if (!s_go) return;
  if (warp == 0) tmem_alloc(&sh.tmem_slot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sh.tmem_slot;
#ifdef PF_ATT_DIAG
  const long long t_start = clock64();
#endif

  if (warp == 0) {
    // ---------------- producer ----------------
    if (lane == 0) {
      tma_prefetch_desc(&tm);
      for (int i = 0; i < n_mine; ++i) {
        const int s = i & 1;
        if (i >= STAGES) mbar_wait_park(&sh.empty[s], ((i >> 1) & 1) ^ 1);
        if (i > 0 && ctl.flag != nullptr && ld_acquire_u32(ctl.flag) == 0u) {
          atomicExch(ctl.abort, 1u);
          *stop_at = i;
          mbar_arrive(&sh.full[s]);  // completes the phase with no data: "stop"
          break;
        }
        const int u = (int)blockIdx.x + i * (int)gridDim.x;
        const int b = u / heads, h = u % heads;
        uint8_t* st = smem + s * STAGE_BYTES;
        ATT_STAMP(i, 0);
        mbar_arrive_expect_tx(&sh.full[s], STAGE_BYTES);
        tma_qkv(&tm, st, &sh.full[s], h, b * seq);
        tma_qkv(&tm, st + TILE_BYTES, &sh.full[s], heads + h, b * seq);
        tma_qkv(&tm, st + 2 * TILE_BYTES, &sh.full[s], 2 * heads + h, b * seq);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      constexpr uint32_t idesc_s = umma_idesc_bf16(128, 128, false, false);
      constexpr uint32_t idesc_o = umma_idesc_bf16(128, D, false, true);
      // Two in-order streams of MMAs: S(next_s) as soon as its Q/K landed and its TMEM
      // buffer is free (at most 2 ahead of O), O(next_o) as soon as its P is in shared
      // memory. Neither blocks the other.
      int next_s = 0, next_o = 0, end = n_mine;
      while (next_o < end) {
        bool progress = false;
        if (next_s < end && next_s < next_o + 2) {
          const int j = next_s, sj = j & 1;
          const uint32_t ph = (j >> 1) & 1;
          if (mbar_test(&sh.full[sj], ph) && (j < STAGES || mbar_test(&sh.t_empty[sj], ph ^ 1))) {
            if (*stop_at <= j) {
              mbar_arrive(&sh.s_full[sj]);  // forward "stop" to the softmax warps
              end = j;
            } else {
              tc_fence_after();
              ATT_STAMP(j, 1);
              const uint32_t qa = smem_u32(smem + sj * STAGE_BYTES), ka = qa + TILE_BYTES;
#pragma unroll
              for (int k = 0; k < D / 16; ++k)
                umma_bf16_ss(tmem + sj * 128, umma_desc_sw128_kmajor(qa + k * 32),
                             umma_desc_sw128_kmajor(ka + k * 32), idesc_s, k > 0 ? 1u : 0u);
              umma_commit(&sh.s_full[sj]);
              ++next_s;
            }
            progress = true;
          }
        }
        if (next_o < next_s && mbar_test(&sh.p_ready[next_o & 1], (next_o >> 1) & 1)) {
          const int so = next_o & 1;
          tc_fence_after();
          ATT_STAMP(next_o, 4);
          const uint32_t pa = smem_u32(smem + so * STAGE_BYTES), va = pa + 2 * TILE_BYTES;
#pragma unroll
          for (int k = 0; k < S_MAX / 16; ++k) {
            const uint64_t ad = umma_desc_sw128_kmajor(pa + (k >> 2) * TILE_BYTES + (k & 3) * 32);
            const uint64_t bd = umma_desc_sw128_mnmajor(va + k * 2048, TILE_BYTES);
            umma_bf16_ss(tmem + so * 128, ad, bd, idesc_o, k > 0 ? 1u : 0u);
          }
          umma_commit(&sh.o_full[so]);
          umma_commit(&sh.empty[so]);
          ++next_o;
          progress = true;
        }
        if (!progress) {
          if (next_o < next_s) mbar_try_wait_hint(&sh.p_ready[next_o & 1], (next_o >> 1) & 1, 2000u);
          else if (next_s < end) mbar_try_wait_hint(&sh.full[next_s & 1], (next_s >> 1) & 1, 2000u);
        }
      }
      // every O committed so far has completed (its o_full and empty arrivals landed) before
      // the "stop" is forwarded to the epilogue warps and before teardown
      for (int j = end > STAGES ? end - STAGES : 0; j < end; ++j) {
        mbar_wait_park(&sh.o_full[j & 1], (j >> 1) & 1);
        mbar_wait_park(&sh.empty[j & 1], (j >> 1) & 1);
      }
      if (end < n_mine) mbar_arrive(&sh.o_full[end & 1]);
    }
  } else if (warp < 10) {
    // ---------------- softmax (warps 2..9): two warps per TMEM lane quarter ----------------
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    const int row = quarter * 32 + lane;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    for (int i = 0; i < n_mine; ++i) {
      const int s = i & 1;
      const uint32_t ph = (i >> 1) & 1;
      mbar_wait_park(&sh.s_full[s], ph);
      if (*stop_at <= i) break;
      tc_fence_after();
      if (warp == 2 && lane == 0) ATT_STAMP(i, 2);
      const int u = (int)blockIdx.x + i * (int)gridDim.x;
      const int b = u / heads;
      const float* mrow = mask_add ? mask_add + (size_t)b * seq : nullptr;
      const uint32_t tS = tmem + lane_base + s * 128 + half * 64;
      // K-block `half` of P, as a shared-window address: explicit st.shared (STS) instead of
      // generic stores (ST.E), which ncu showed stalling the softmax warps
      const uint32_t blk_s = smem_u32(smem + s * STAGE_BYTES + half * TILE_BYTES + row * 128);
      float sum = 0.f;
      if constexpr (FULL) {
        // max of the raw scores (scale > 0 commutes with max), then p = 2^(s*c - max*c)
        float mx;
        {
          uint32_t r[32];
          tmem_ld_32x32b_x32(tS, r);
          tmem_ld_wait();
          mx = __uint_as_float(r[0]);
#pragma unroll
          for (int j = 1; j < 32; ++j) mx = fmaxf(mx, __uint_as_float(r[j]));
          tmem_ld_32x32b_x32(tS + 32, r);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) mx = fmaxf(mx, __uint_as_float(r[j]));
        }
        s_red[half][row] = mx;
        softmax_bar();
        const float nmx = -fmaxf(s_red[0][row], s_red[1][row]) * scale_log2;
        // exponent arguments and row sums on packed fp32 pairs (FFMA2 / FADD2): two FP
        // instructions per key pair instead of four around the two MUFU.EX2
        const f32x2 sc2 = f2_splat(scale_log2), nm2 = f2_splat(nmx);
        f32x2 sum2 = f2_splat(0.f);
#pragma unroll 1
        for (int c = 0; c < 2; ++c) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(tS + c * 32, r);
          tmem_ld_wait();
          uint32_t packed[16];
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            float a0, a1;
            f2_unpack(f2_fma(f2_pack(__uint_as_float(r[j]), __uint_as_float(r[j + 1])), sc2, nm2), a0, a1);
            const float p0 = fast_ex2(a0), p1 = fast_ex2(a1);
            sum2 = f2_add(sum2, f2_pack(p0, p1));
            packed[j / 2] = pack_bf16x2(p0, p1);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int chunk = c * 4 + q;
            st_shared_v4(blk_s + ((chunk ^ (row & 7)) << 4), packed[4 * q], packed[4 * q + 1],
                         packed[4 * q + 2], packed[4 * q + 3]);
          }
        }
        {
          float lo, hi;
          f2_unpack(sum2, lo, hi);
          sum = lo + hi;
        }
      } else {
        float mx = -INFINITY;
#pragma unroll 1
        for (int c = 0; c < 2; ++c) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(tS + c * 32, r);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int key = half * 64 + c * 32 + j;
            float v = __uint_as_float(r[j]) * scale_log2;
            if (mrow && key < seq) v += mrow[key] * 1.4426950408889634f;
            if (key >= seq) v = -INFINITY;
            mx = fmaxf(mx, v);
          }
        }
        s_red[half][row] = mx;
        softmax_bar();
        mx = fmaxf(mx, s_red[half ^ 1][row]);
#pragma unroll 1
        for (int c = 0; c < 2; ++c) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(tS + c * 32, r);
          tmem_ld_wait();
          uint32_t packed[16];
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            float p2[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int key = half * 64 + c * 32 + j + e;
              float v = __uint_as_float(r[j + e]) * scale_log2;
              if (mrow && key < seq) v += mrow[key] * 1.4426950408889634f;
              p2[e] = key < seq ? exp2f(v - mx) : 0.f;
              sum += p2[e];
            }
            packed[j / 2] = pack_bf16x2(p2[0], p2[1]);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int chunk = c * 4 + q;
            st_shared_v4(blk_s + ((chunk ^ (row & 7)) << 4), packed[4 * q], packed[4 * q + 1],
                         packed[4 * q + 2], packed[4 * q + 3]);
          }
        }
      }
      s_sums[s][half][row] = sum;
      fence_async_smem();  // generic-proxy P stores -> visible to the tensor core
      tc_fence_before();
      softmax_bar();
      if (warp == 2 && lane == 0) {
        ATT_STAMP(i, 3);
        mbar_arrive(&sh.p_ready[s]);
      }
    }
  } else {
    // ---------------- epilogue (warps 10..13): one warp per TMEM lane quarter ----------------
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    for (int i = 0; i < n_mine; ++i) {
      const int s = i & 1;
      const uint32_t ph = (i >> 1) & 1;
      mbar_wait_park(&sh.o_full[s], ph);
      if (*stop_at <= i) break;
      mbar_wait_park(&sh.p_ready[s], ph);  // acquire: this unit's row sums are visible
      tc_fence_after();
      if (warp == 12 && lane == 0) ATT_STAMP(i, 5);
      const int u = (int)blockIdx.x + i * (int)gridDim.x;
      const int b = u / heads, h = u % heads;
      const float inv = fast_rcp(s_sums[s][0][row] + s_sums[s][1][row]);
      uint4* orow = reinterpret_cast<uint4*>(O + ((size_t)(b * seq + (row < seq ? row : 0)) * heads + h) * D);
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem + lane_base + s * 128 + c * 32, r);
        tmem_ld_wait();
        if (c == 1) {  // both halves of O are in registers: release the TMEM buffer
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&sh.t_empty[s]);
        }
        if (row < seq) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint4 v;
            v.x = pack_bf16x2(__uint_as_float(r[8 * q + 0]) * inv, __uint_as_float(r[8 * q + 1]) * inv);
            v.y = pack_bf16x2(__uint_as_float(r[8 * q + 2]) * inv, __uint_as_float(r[8 * q + 3]) * inv);
            v.z = pack_bf16x2(__uint_as_float(r[8 * q + 4]) * inv, __uint_as_float(r[8 * q + 5]) * inv);
            v.w = pack_bf16x2(__uint_as_float(r[8 * q + 6]) * inv, __uint_as_float(r[8 * q + 7]) * inv);
            orow[c * 4 + q] = v;
          }
        }
      }
      if (warp == 12 && lane == 0) ATT_STAMP(i, 6);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, TMEM_COLS);
  if (tid == 0 && ctl.cursor != nullptr && s_stop_at == 0x7fffffff) {
    __threadfence();
    atomicAdd(ctl.cursor, 1u);
  }
}

inline unsigned attention_grid(int batch, int heads) {
  const int units = batch * heads;
  const int cap = CTAS_PER_SM * device_sm_count();
  return (unsigned)(units < cap ? units : cap);
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
  uint32_t units() const override { return attention_grid(batch, heads); }
  bool resumable() const override { return false; }
  int run(const pf_ctl_t* ctl, cudaStream_t s, const LaunchArgs&) override {
    auto k = (mask == nullptr && seq == S_MAX) ? attention_kernel<true> : attention_kernel<false>;
    PF_CUDA(launch_pdl(k, dim3(units()), dim3(THREADS), SMEM_REQUEST, s, tm, mask, out, batch, seq,
                       heads, scale_log2, make_ctl(ctl)));
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
    PF_CUDA(cudaFuncSetAttribute(attention_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 SMEM_REQUEST));
    PF_CUDA(cudaFuncSetAttribute(attention_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
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

#ifdef PF_ATT_DIAG
extern "C" int pf_att_diag_read(uint32_t* host) {
  return cudaMemcpyFromSymbol(host, pf::attn::g_att_diag, sizeof(pf::attn::g_att_diag)) == cudaSuccess ? 0 : -1;
}
#endif

extern "C" int pf_attention_units(int batch, int seq, int heads, int head_dim, uint32_t* out) {
  if (!out || batch <= 0 || heads <= 0 || seq <= 0)
    return pf::set_error(PF_ERR_INVALID, "pf_attention_units");
  *out = pf::attn::attention_grid(batch, heads);
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
