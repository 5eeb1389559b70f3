// pf_gemm.cu — preemptible persistent tcgen05 GEMM with fused bias / GELU / residual.
//
//   Y[M,N] = epi( X[M,K] · W[N,K]^T )      (nn.Linear weight layout, bf16 in, fp32 acc)
//
// This is the fill job's dominant kernel (QKV / attention-out / FFN1 / FFN2 of
// every BERT layer, SURVEY §2.1 "gemm_bias_gelu"). The reference has no kernel:
// its executor is the time model ExecutionPlan.range_busy_us
// (pkg/src/bubblefill/partition.py:126-132); this kernel is what that time is
// spent on.
//
// Structure (one CTA per SM, persistent, 384 threads):
//   warp 0      tile scheduler + TMA producer (A/B k-blocks into a STAGES-deep ring)
//   warp 1      MMA issuer: one lane issues tcgen05.mma 128xBNx16 into TMEM
//   warp 2      TMEM allocator (2 accumulator buffers of BN fp32 columns)
//   warp 3      idle
//   warps 4-11  epilogue: tcgen05.ld -> bias/GELU/residual -> bf16 -> global
// The scheduler claims output tiles from the launch's cursor only while the
// bubble flag is set (pf::claim_unit), so the kernel yields within one tile
// of the flag clearing and the claimed-tile prefix is the resume cursor.
#include <stdio.h>
#include <stdlib.h>

#include "pf_ops.h"

namespace pf {
namespace gemm {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 B rows -> SWIZZLE_128B
constexpr int UMMA_K = 16;
constexpr int NUM_THREADS = 384;
// Warp roles. The epilogue warps take the LOW warp ids: the SM's warp arbiter favours
// high warp ids, so the TMA producer and the single-thread MMA issuer (warps 8, 9) win
// issue slots over the math-heavy epilogue (bias / erf-GELU / residual) sharing their
// SM sub-partitions, and the tensor pipe is not starved while an epilogue runs.
constexpr int EPI_WARP0 = 0;
constexpr int PRODUCER_WARP = 8;
constexpr int MMA_WARP = 9;
constexpr int ALLOC_WARP = 10;
constexpr int NUM_EPI_WARPS = 8;
constexpr int SCHED_SLOTS = 8;
constexpr int SMEM_BUDGET = 200 * 1024;

template <int BN>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (SMEM_BUDGET / STAGE_BYTES) > 6 ? 6 : (SMEM_BUDGET / STAGE_BYTES);
  static constexpr int TMEM_COLS = (2 * BN <= 256) ? 256 : 512;
  static constexpr int COLS_PER_EPI_WARP = BN / 2;  // two warps share each 32-lane group
  static constexpr int CHUNKS = COLS_PER_EPI_WARP / 32;
  // barriers + sched ring + tmem addr live after the operand ring
  static constexpr int BAR_BYTES = (2 * STAGES + 4 + 2 * SCHED_SLOTS) * 8 + SCHED_SLOTS * 4 + 16 +
                                   NUM_EPI_WARPS * COLS_PER_EPI_WARP * 2;
  // per-epilogue-warp 32x32 bf16 staging tile for the TMA store (1024-B aligned)
  static constexpr int STG_OFFSET = (STAGES * STAGE_BYTES + BAR_BYTES + 1023) / 1024 * 1024;
  static constexpr int SMEM_BYTES = 1024 /*align slack*/ + STG_OFFSET + NUM_EPI_WARPS * 2048;
  static_assert(SMEM_BYTES <= 227 * 1024, "smem");
  static_assert(BN % 64 == 0 && BN <= 256, "BN");
  static_assert(COLS_PER_EPI_WARP % 32 == 0, "epilogue chunking");
};

struct Params {
  __nv_bfloat16* Y;
  const __nv_bfloat16* bias;
  const __nv_bfloat16* residual;
  int M, N, K;
  int tiles_m, tiles_n;
  unsigned long long* stamp;  // optional [first CTA start, last CTA end] in ns
  // split-K (single-CTA kernel only): k_splits slices of kb_per_split K-blocks each;
  // slice z of output tile (tm, tn) is stored to Y[z] of a [k_splits, M, N] stack
  int k_splits;
  int kb_per_split;
  // Tail wave in half tiles: units [0, n_full) are full BM x BN tiles; when tail_halves is
  // set, each of the remaining tiles is split into two BM x BN/2 units (n_full + 2 x rem
  // units in all), so a last wave of rem <= grid/2 tiles takes ~(BN/2 + 200)/(BN + 200) of a
  // full wave instead of a whole one (see pick_bn's cost model).
  int n_full;
  int tail_halves;
  int group_m;  // m-blocks per rasterisation group (GROUP_M unless PF_GEMM_GROUP_M is set)
};

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Grouped rasterisation: tiles walk GROUP_M m-blocks x all n-blocks, m fastest inside a
// group, so the tiles of one m-block (all n-blocks) are GROUP_M units apart and start in
// the same wave: each A row band is read from DRAM once while W (the small operand at the
// fill shapes, <= 8 MB) stays L2-resident. A tall group spreads an m-block's tiles over
// waves and the A band is re-read after eviction: in situ at BERT-large batch 128
// (scripts/bert_batch_profile.py, PF_GEMM_GROUP_M sweep) FFN2 (K = 4096) takes 98 us at
// GROUP_M 1-2, 100-101 us at 16 and 114 us at 64.
constexpr int GROUP_M = 2;

#ifdef PF_GEMM_DIAG
// [0] MMA wait on full (data), [1] MMA wait on tempty (epilogue), [2] producer wait on empty,
// [3] epilogue wait on tfull, [4] MMA issue cycles, [5] epilogue busy cycles
// Counters accumulate per CTA in shared memory (no global-atomic contention inside the
// loops) and are flushed once at CTA exit.
__device__ unsigned long long g_gemm_diag[16];  // [8] MMA-warp clock cycles, [9] its ns
__shared__ unsigned long long s_gemm_diag[16];
#define DIAG_T0() long long _t0 = clock64()
#define DIAG_ADD(i) atomicAdd(&s_gemm_diag[i], (unsigned long long)(clock64() - _t0))
#define DIAG_INIT() do { if (threadIdx.x < 16) s_gemm_diag[threadIdx.x] = 0; } while (0)
#define DIAG_FLUSH() do { if (threadIdx.x < 16) atomicAdd(&g_gemm_diag[threadIdx.x], s_gemm_diag[threadIdx.x]); } while (0)
#else
#define DIAG_T0()
#define DIAG_ADD(i)
#define DIAG_INIT()
#define DIAG_FLUSH()
#endif

__device__ __forceinline__ void tile_coords(int tile, const Params& p, int& tm, int& tn, int& ks) {
  const int per_split = p.tiles_m * p.tiles_n;
  ks = tile / per_split;
  tile -= ks * per_split;
  const int per_group = p.group_m * p.tiles_n;
  const int g = tile / per_group;
  const int first_m = g * p.group_m;
  const int rows = min(p.tiles_m - first_m, p.group_m);
  const int r = tile - g * per_group;
  tm = first_m + r % rows;
  tn = r / rows;
}

// Unit u -> output tile (tm, tn), K slice ks and half (-1 = the whole BN-wide tile).
__device__ __forceinline__ void unit_info(int u, const Params& p, int& tm, int& tn, int& ks, int& half) {
  half = -1;
  if (p.tail_halves && u >= p.n_full) {
    const int v = u - p.n_full;
    half = v & 1;
    u = p.n_full + (v >> 1);
  }
  tile_coords(u, p, tm, tn, ks);
}

// One epilogue warp's share of an output tile: 32 rows (its TMEM lane group) x
// CHUNKS*32 columns. Bias is staged in shared memory before the accumulator is ready;
// TMEM loads are double-buffered; each 32x32 result chunk goes registers -> bias /
// erf-GELU / residual -> bf16 -> a 64-B-swizzled smem tile -> one TMA bulk store
// (full-line writes, clipped at the tensor edges) issued by lane 0.
template <int CHUNKS, uint32_t EPI, bool PAIR>
__device__ __forceinline__ void epilogue_tile(const Params& p, const CUtensorMap* tmY,
                                              uint8_t* stg, uint32_t taddr0, uint64_t* tfull,
                                              uint32_t aphase, int row_base, int col_base,
                                              __nv_bfloat16* my_bias, int ks) {
  constexpr bool HAS_BIAS = (EPI & PF_EPI_BIAS) != 0;
  constexpr bool HAS_GELU = (EPI & PF_EPI_GELU) != 0;
  constexpr bool HAS_RES = (EPI & PF_EPI_RESIDUAL) != 0;
  constexpr bool HAS_RELU = (EPI & PF_EPI_RELU) != 0;
  constexpr int COLS = CHUNKS * 32;
  const int lane = lane_id();
  const int row = row_base + lane;
  const bool row_ok = row < p.M;
  if (HAS_BIAS) {
    for (int j = lane * 8; j < COLS; j += 32 * 8) {
      uint4 b4 = make_uint4(0, 0, 0, 0);
      if (col_base + j + 8 <= p.N) {
        b4 = __ldg(reinterpret_cast<const uint4*>(p.bias + col_base + j));
      } else {
        __nv_bfloat16 tmp[8];
        for (int q = 0; q < 8; ++q)
          tmp[q] = col_base + j + q < p.N ? p.bias[col_base + j + q] : __float2bfloat16(0.f);
        b4 = *reinterpret_cast<uint4*>(tmp);
      }
      *reinterpret_cast<uint4*>(my_bias + j) = b4;
    }
    __syncwarp();
  }
  const __nv_bfloat16* rrow = HAS_RES ? p.residual + (size_t)row * p.N : nullptr;
  // The residual does not depend on the accumulator: chunk 0's slice is fetched before the
  // wait for it, and chunk c+1's while chunk c is processed, so the global-load latency
  // (32 rows per warp instruction) is hidden instead of exposed once per chunk.
  auto load_res = [&](int col0, uint4 (&dst)[4]) {
    if (row_ok && col0 + 32 <= p.N) {
#pragma unroll
      for (int q = 0; q < 4; ++q) dst[q] = __ldg(reinterpret_cast<const uint4*>(rrow + col0) + q);
    } else {
      __nv_bfloat16 tmp[32];
#pragma unroll
      for (int j = 0; j < 32; ++j)
        tmp[j] = (row_ok && col0 + j < p.N) ? rrow[col0 + j] : __float2bfloat16(0.f);
#pragma unroll
      for (int q = 0; q < 4; ++q) dst[q] = reinterpret_cast<const uint4*>(tmp)[q];
    }
  };
  uint4 res_nxt[4];
  if (HAS_RES) load_res(col_base, res_nxt);
  {
    DIAG_T0();
    if (PAIR) mbar_wait_cluster_park(tfull, aphase);
    else mbar_wait_park(tfull, aphase);
    if (lane == 0) DIAG_ADD(3);
  }
  tc_fence_after();
#ifdef PF_GEMM_DIAG
  const long long _te0 = clock64();
#endif
  uint32_t rbuf[2][32];
  __syncwarp();
  tmem_ld_32x32b_x32(taddr0, rbuf[0]);
#pragma unroll
  for (int c = 0; c < CHUNKS; ++c) {
    const int col0 = col_base + c * 32;
    uint4 res_cur[4];
    if (HAS_RES) {
#pragma unroll
      for (int q = 0; q < 4; ++q) res_cur[q] = res_nxt[q];
      if (c + 1 < CHUNKS) load_res(col0 + 32, res_nxt);
    }
    __syncwarp();
    tmem_ld_wait();  // chunk c landed
    if (c + 1 < CHUNKS) tmem_ld_32x32b_x32(taddr0 + (uint32_t)((c + 1) * 32), rbuf[(c + 1) & 1]);
    const uint32_t(&r)[32] = rbuf[c & 1];
    float v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
    if (HAS_BIAS) {
      const uint4* bp = reinterpret_cast<const uint4*>(my_bias + c * 32);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 b4 = bp[q];
        const uint32_t bw[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          float2 f = unpack_bf16x2(bw[h]);
          float& a = v[q * 8 + h * 2];
          float& b = v[q * 8 + h * 2 + 1];
          f2_unpack(f2_add(f2_pack(a, b), f2_pack(f.x, f.y)), a, b);
        }
      }
    }
    if (HAS_GELU) {
#pragma unroll
      for (int j = 0; j < 32; j += 2) gelu_fast2(v[j], v[j + 1]);
    }
    if (HAS_RES) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t rw[4] = {res_cur[q].x, res_cur[q].y, res_cur[q].z, res_cur[q].w};
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          float2 f = unpack_bf16x2(rw[h]);
          float& a = v[q * 8 + h * 2];
          float& b = v[q * 8 + h * 2 + 1];
          f2_unpack(f2_add(f2_pack(a, b), f2_pack(f.x, f.y)), a, b);
        }
      }
    }
    if (HAS_RELU) {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j], 0.f);
    }
    // the previous bulk store from this staging tile (previous chunk, or the last chunk
    // of this warp's previous output tile: with a short K the next accumulator is ready
    // before that store has read shared memory) must be done reading it
    if (lane == 0) bulk_wait_read0();
    __syncwarp();
    // row `lane` of the 32x32 tile = 4 x 16 B; TMA SWIZZLE_64B places 16-B chunk q of
    // row r at chunk q ^ ((r >> 1) & 3) (conflict-free: 8 distinct bank groups per phase)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 o;
      o.x = pack_bf16x2(v[q * 8 + 0], v[q * 8 + 1]);
      o.y = pack_bf16x2(v[q * 8 + 2], v[q * 8 + 3]);
      o.z = pack_bf16x2(v[q * 8 + 4], v[q * 8 + 5]);
      o.w = pack_bf16x2(v[q * 8 + 6], v[q * 8 + 7]);
      const int phys = q ^ ((lane >> 1) & 3);
#ifndef PF_DIAG_NO_STORE
      *reinterpret_cast<uint4*>(stg + lane * 64 + phys * 16) = o;
#else
      if (o.x == 0x12345678u) *reinterpret_cast<uint4*>(stg + lane * 64 + phys * 16) = o;
#endif
    }
    fence_async_smem();
    __syncwarp();
    if (lane == 0 && col0 < p.N) {
      if (p.k_splits > 1) tma_store_3d(tmY, stg, col0, row_base, ks);
      else tma_store_2d(tmY, stg, col0, row_base);
      bulk_commit();
    }
  }
#ifdef PF_GEMM_DIAG
  if (lane == 0) atomicAdd(&s_gemm_diag[5], (unsigned long long)(clock64() - _te0));
  if (lane == 0) atomicAdd(&s_gemm_diag[6], 1ull);
#endif
}

// MJ: operand majorness, bit 0 = A MN-major, bit 1 = B MN-major (default both K-major).
// An MN-major operand is stored [K, M] (resp. [K, N]) row-major: TMA brings it in as
// 64 x 64 SW128 blocks (8 KB, LBO between blocks) and the MMA reads it transposed, so
// weight gradients (dZ^T X) and data gradients (dZ W) need no transpose kernels.
template <int BN, uint32_t EPI, int MJ = 0>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmY, Params p, Ctl ctl) {
  using C = Cfg<BN>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-B alignment for the swizzled operand tiles
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* full_bar = bars;
  uint64_t* empty_bar = bars + C::STAGES;
  uint64_t* tfull_bar = bars + 2 * C::STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* sfull_bar = tempty_bar + 2;
  uint64_t* sempty_bar = sfull_bar + SCHED_SLOTS;
  int* sched_tile = reinterpret_cast<int*>(sempty_bar + SCHED_SLOTS);
  uint32_t* tmem_base_smem = reinterpret_cast<uint32_t*>(sched_tile + SCHED_SLOTS);
  __nv_bfloat16* bias_smem = reinterpret_cast<__nv_bfloat16*>(tmem_base_smem + 4);

  const int warp = warp_id();
  const int lane = lane_id();

  pdl_enter();
  // CTA-uniform (thread 0 decides; nothing allocated yet); tmem_base_smem[2] is scratch
  if (chain_aborted_cta(ctl, tmem_base_smem + 2)) return;
  DIAG_INIT();
  if (threadIdx.x == 0 && p.stamp) atomicMin(&p.stamp[0], globaltimer_ns());

  if (warp == PRODUCER_WARP && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmY);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], NUM_EPI_WARPS);
    }
    for (int s = 0; s < SCHED_SLOTS; ++s) {
      mbar_init(&sfull_bar[s], 1);
      mbar_init(&sempty_bar[s], 1 + NUM_EPI_WARPS);
    }
    tmem_base_smem[1] = 0u;  // "ran a tile" (set by the scheduler, read at exit)
    fence_barrier_init();
  }
  if (warp == ALLOC_WARP) tmem_alloc(tmem_base_smem, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_smem;

  const int num_tiles = p.tail_halves ? 2 * p.tiles_m * p.tiles_n - p.n_full : p.tiles_m * p.tiles_n * p.k_splits;
  const int num_kb = (p.K + BK - 1) / BK;

  if (warp == PRODUCER_WARP) {
    // ---------------- scheduler + TMA producer ----------------
    int slot = 0;
    uint32_t sphase = 0;
    int stage = 0;
    uint32_t phase = 0;
    for (int it = 0;; ++it) {
      int tile = -1;
      if (lane == 0) tile = claim_unit(ctl, num_tiles, it);
      tile = __shfl_sync(0xffffffffu, tile, 0);
      mbar_wait(&sempty_bar[slot], sphase ^ 1u);
      if (lane == 0) {
        sched_tile[slot] = tile;
        mbar_arrive(&sfull_bar[slot]);
      }
      if (++slot == SCHED_SLOTS) {
        slot = 0;
        sphase ^= 1u;
      }
      if (tile < 0) break;
      if (lane == 0) tmem_base_smem[1] = 1u;  // this CTA ran a tile (end stamp below)
      int tm, tn, ks, half;  // a half unit loads the whole BN rows of W (L2-resident) and uses half
      unit_info(tile, p, tm, tn, ks, half);
      const int kb0 = ks * p.kb_per_split;
      const int kb1 = min(num_kb, kb0 + p.kb_per_split);
      for (int kb = kb0; kb < kb1; ++kb) {
        {
          DIAG_T0();
          mbar_wait_park(&empty_bar[stage], phase ^ 1u);
          if (lane == 0) DIAG_ADD(2);
        }
        if (lane == 0) {
          mbar_arrive_expect_tx(&full_bar[stage], C::STAGE_BYTES);
          if (MJ & 1) {
#pragma unroll
            for (int b = 0; b < BM / 64; ++b)
              tma_load_2d(sA + stage * C::A_BYTES + b * 8192, &tmA, &full_bar[stage], tm * BM + 64 * b, kb * BK);
          } else {
            tma_load_2d(sA + stage * C::A_BYTES, &tmA, &full_bar[stage], kb * BK, tm * BM);
          }
          if (MJ & 2) {
#pragma unroll
            for (int b = 0; b < BN / 64; ++b)
              tma_load_2d(sB + stage * C::B_BYTES + b * 8192, &tmB, &full_bar[stage], tn * BN + 64 * b, kb * BK);
          } else {
            tma_load_2d(sB + stage * C::B_BYTES, &tmB, &full_bar[stage], kb * BK, tn * BN);
          }
        }
        __syncwarp();
        if (++stage == C::STAGES) {
          stage = 0;
          phase ^= 1u;
        }
      }
    }
  } else if (warp == MMA_WARP) {
    // ---------------- MMA issuer ----------------
#ifdef PF_GEMM_DIAG
    const long long _c0 = clock64();
    const unsigned long long _g0 = globaltimer_ns();
#endif
    constexpr uint32_t idesc = umma_idesc_bf16(BM, BN, (MJ & 1) != 0, (MJ & 2) != 0);
    constexpr uint32_t idesc_half = umma_idesc_bf16(BM, BN / 2, (MJ & 1) != 0, (MJ & 2) != 0);
    int slot = 0;
    uint32_t sphase = 0;
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t aphase = 0;
    while (true) {
      mbar_wait(&sfull_bar[slot], sphase);
      const int tile = sched_tile[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&sempty_bar[slot]);
      if (++slot == SCHED_SLOTS) {
        slot = 0;
        sphase ^= 1u;
      }
      if (tile < 0) break;
      {
        DIAG_T0();
        mbar_wait(&tempty_bar[acc], aphase ^ 1u);
        if (lane == 0) DIAG_ADD(1);
      }
      tc_fence_after();
#ifdef PF_GEMM_DIAG
      const long long _tm0 = clock64();
#endif
      const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
      int utm, utn, uks, uhalf;
      unit_info(tile, p, utm, utn, uks, uhalf);
      const int kb0 = uks * p.kb_per_split;
      const int kb1 = min(num_kb, kb0 + p.kb_per_split);
      // a half unit: N = BN/2 from rows [half * BN/2, +BN/2) of the staged W tile
      const uint32_t idesc_u = uhalf < 0 ? idesc : idesc_half;
      const uint32_t b_off = uhalf < 0 ? 0u : (uint32_t)(uhalf * (BN / 2) * 128);
      for (int kb = kb0; kb < kb1; ++kb) {
        {
          DIAG_T0();
          mbar_wait(&full_bar[stage], phase);
          if (lane == 0) DIAG_ADD(0);
        }
        tc_fence_after();
        if (lane == 0) {
          const uint32_t a_addr = smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b_addr = smem_u32(sB + stage * C::B_BYTES) + b_off;
#pragma unroll
          for (int k = 0; k < BK / UMMA_K; ++k) {
            // K advance inside the 128-B swizzle atom: +32 B per UMMA_K step
            // K advance: +32 B inside the 128-B swizzle atom (K-major), or +16 rows of
            // 128 B (MN-major)
            const uint64_t ad = (MJ & 1) ? umma_desc_sw128_mnmajor(a_addr + k * UMMA_K * 128, 8192)
                                         : umma_desc_sw128_kmajor(a_addr + k * UMMA_K * 2);
            const uint64_t bd = (MJ & 2) ? umma_desc_sw128_mnmajor(b_addr + k * UMMA_K * 128, 8192)
                                         : umma_desc_sw128_kmajor(b_addr + k * UMMA_K * 2);
            umma_bf16_ss(d_tmem, ad, bd, idesc_u, (kb != kb0 || k != 0) ? 1u : 0u);
          }
          umma_commit(&empty_bar[stage]);  // frees the smem slot when these MMAs retire
        }
        __syncwarp();
        if (++stage == C::STAGES) {
          stage = 0;
          phase ^= 1u;
        }
      }
      if (lane == 0) umma_commit(&tfull_bar[acc]);  // accumulator ready for the epilogue
#ifdef PF_GEMM_DIAG
      if (lane == 0) atomicAdd(&s_gemm_diag[4], (unsigned long long)(clock64() - _tm0));
      if (lane == 0) atomicAdd(&s_gemm_diag[7], 1ull);
#endif
      __syncwarp();
      if (++acc == 2) {
        acc = 0;
        aphase ^= 1u;
      }
    }
#ifdef PF_GEMM_DIAG
    if (lane == 0) {
      atomicAdd(&s_gemm_diag[8], (unsigned long long)(clock64() - _c0));
      atomicAdd(&s_gemm_diag[9], globaltimer_ns() - _g0);
    }
#endif
  } else if (warp >= EPI_WARP0 && warp < EPI_WARP0 + NUM_EPI_WARPS) {
    // ---------------- epilogue ----------------
    const int e = warp - EPI_WARP0;
    const int lane_grp = warp & 3;  // TMEM lanes [32*lane_grp, +32) are visible to this warp
    const int col_half = e >> 2;
    __nv_bfloat16* my_bias = bias_smem + e * C::COLS_PER_EPI_WARP;
    uint8_t* my_stg = smem + C::STG_OFFSET + e * 2048;
    int slot = 0;
    uint32_t sphase = 0;
    int acc = 0;
    uint32_t aphase = 0;
    while (true) {
      mbar_wait(&sfull_bar[slot], sphase);
      const int tile = sched_tile[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&sempty_bar[slot]);
      if (++slot == SCHED_SLOTS) {
        slot = 0;
        sphase ^= 1u;
      }
      if (tile < 0) break;
      int tm, tn, ks, half;
      unit_info(tile, p, tm, tn, ks, half);
      const int row_base = tm * BM + lane_grp * 32;
      if (half < 0) {
        const int col_base = tn * BN + col_half * C::COLS_PER_EPI_WARP;
        const uint32_t taddr = tmem_base + ((uint32_t)(lane_grp * 32) << 16) +
                               (uint32_t)(acc * BN + col_half * C::COLS_PER_EPI_WARP);
        epilogue_tile<C::CHUNKS, EPI, false>(p, &tmY, my_stg, taddr, &tfull_bar[acc], aphase, row_base,
                                             col_base, my_bias, ks);
      } else if constexpr (C::CHUNKS % 2 == 0) {
        constexpr int HC = C::COLS_PER_EPI_WARP / 2;
        const int col_base = tn * BN + half * (BN / 2) + col_half * HC;
        const uint32_t taddr = tmem_base + ((uint32_t)(lane_grp * 32) << 16) + (uint32_t)(acc * BN + col_half * HC);
        epilogue_tile<C::CHUNKS / 2, EPI, false>(p, &tmY, my_stg, taddr, &tfull_bar[acc], aphase, row_base,
                                                 col_base, my_bias, ks);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty_bar[acc]);
      if (++acc == 2) {
        acc = 0;
        aphase ^= 1u;
      }
    }
    if (lane == 0) bulk_wait0();  // outstanding TMA stores of this warp are complete
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == ALLOC_WARP) tmem_dealloc(tmem_base, C::TMEM_COLS);
  DIAG_FLUSH();
  // end stamp only from CTAs that ran a tile: a CTA that starts after the bubble closed (its
  // SM was busy with the main job) and exits without work does not extend the kernel's span
  if (threadIdx.x == 0 && p.stamp && tmem_base_smem[1] != 0u) atomicMax(&p.stamp[1], globaltimer_ns());
}


// ===========================================================================
// CTA-pair variant (cluster of 2, tcgen05 cta_group::2)
//
// A pair computes a 256 x BN output tile: each CTA TMA-loads its own 128 rows of A
// and HALF of the BN rows of W into its shared memory, and the leader CTA issues
// tcgen05.mma.cta_group::2 (M=256) that reads both CTAs' operands. Each SM thus
// streams 128x64 + (BN/2)x64 operand elements per 128xBNx64 of MMA work instead of
// 128x64 + BNx64: a third less shared-memory / L2 traffic per FLOP, and 6 pipeline
// stages fit instead of 4. Each CTA's TMEM holds its 128 accumulator rows; both
// CTAs run the same epilogue on their half. The leader claims tiles (and makes the
// preemption decision) and forwards each tile index to the peer through DSMEM.
template <int BN>
struct Cfg2 {
  static constexpr int A_BYTES = BM * BK * 2;         // this CTA's 128 rows
  static constexpr int B_BYTES = (BN / 2) * BK * 2;   // this CTA's half of W's BN rows
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (SMEM_BUDGET / STAGE_BYTES) > 6 ? 6 : (SMEM_BUDGET / STAGE_BYTES);
  static constexpr int TMEM_COLS = (2 * BN <= 256) ? 256 : 512;
  static constexpr int COLS_PER_EPI_WARP = BN / 2;
  static constexpr int CHUNKS = COLS_PER_EPI_WARP / 32;
  static constexpr int BAR_BYTES = (2 * STAGES + 4 + 2 * SCHED_SLOTS) * 8 + SCHED_SLOTS * 4 + 16 +
                                   NUM_EPI_WARPS * COLS_PER_EPI_WARP * 2;
  static constexpr int STG_OFFSET = (STAGES * STAGE_BYTES + BAR_BYTES + 1023) / 1024 * 1024;
  static constexpr int SMEM_BYTES = 1024 + STG_OFFSET + NUM_EPI_WARPS * 2048;
  static_assert(SMEM_BYTES <= 227 * 1024, "smem");
  static_assert(BN % 128 == 0 && BN <= 256, "pair BN");
};

__device__ __forceinline__ int claim_pair(const Ctl& c, int units, int iter) {
  if (chain_aborted(c)) return -1;
  if (c.flag != nullptr) {
    const uint32_t f = ld_acquire_u32(c.flag);
    if (f == 0u) {
      atomicExch(c.abort, 1u);
      return -1;
    }
    if (c.cursor != nullptr && throttled_out(f, blockIdx.x >> 1, 2u)) return -1;  // pairs: f / 2 of them
  }
  uint32_t u;
  if (c.cursor != nullptr) {
    u = atomicAdd(c.cursor, 1u);
  } else {
    u = (blockIdx.x >> 1) + (uint32_t)iter * (gridDim.x >> 1);
  }
  return u < (uint32_t)units ? (int)u : -1;
}

template <int BN, uint32_t EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
    gemm2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const __grid_constant__ CUtensorMap tmY, Params p, Ctl ctl) {
  using C = Cfg2<BN>;
  constexpr int PM = 2 * BM;  // pair tile rows
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* full_bar = bars;
  uint64_t* empty_bar = bars + C::STAGES;
  uint64_t* tfull_bar = bars + 2 * C::STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* sfull_bar = tempty_bar + 2;
  uint64_t* sempty_bar = sfull_bar + SCHED_SLOTS;
  int* sched_tile = reinterpret_cast<int*>(sempty_bar + SCHED_SLOTS);
  uint32_t* tmem_base_smem = reinterpret_cast<uint32_t*>(sched_tile + SCHED_SLOTS);
  __nv_bfloat16* bias_smem = reinterpret_cast<__nv_bfloat16*>(tmem_base_smem + 4);

  const int warp = warp_id();
  const int lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  if (threadIdx.x == 0 && p.stamp) atomicMin(&p.stamp[0], globaltimer_ns());
  DIAG_INIT();

  if (warp == PRODUCER_WARP && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmY);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);   // leader: its arrive.expect_tx (both CTAs' bytes)
      mbar_init(&empty_bar[s], 1);  // the leader's multicast MMA commit
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);                   // multicast commit
      mbar_init(&tempty_bar[a], 2 * NUM_EPI_WARPS);  // leader: both CTAs' epilogue warps
    }
    for (int s = 0; s < SCHED_SLOTS; ++s) {
      mbar_init(&sfull_bar[s], 1);
      // leader: its MMA + epilogue warps (local) and the peer's producer + epilogue (remote)
      mbar_init(&sempty_bar[s], 2 + 2 * NUM_EPI_WARPS);
    }
    tmem_base_smem[1] = 0u;  // "ran a tile" (set by the scheduler, read at exit)
    fence_barrier_init();
  }
  if (warp == ALLOC_WARP) tmem_alloc_pair(tmem_base_smem, C::TMEM_COLS);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_smem;

  const int num_tiles = p.tail_halves ? 2 * p.tiles_m * p.tiles_n - p.n_full : p.tiles_m * p.tiles_n;
  const int num_kb = (p.K + BK - 1) / BK;

  if (warp == PRODUCER_WARP) {
    // ---------------- scheduler (leader) / tile follower (peer) + TMA producer ----------------
    int slot = 0;
    uint32_t sphase = 0;
    int stage = 0;
    uint32_t phase = 0;
    for (int it = 0;; ++it) {
      int tile;
      if (leader) {
        tile = 0;
        if (lane == 0) tile = claim_pair(ctl, num_tiles, it);
        tile = __shfl_sync(0xffffffffu, tile, 0);
        mbar_wait_cluster(&sempty_bar[slot], sphase ^ 1u);
        if (lane == 0) {
          sched_tile[slot] = tile;
          st_shared_cluster_u32(mapa_shared(smem_u32(&sched_tile[slot]), 1), (uint32_t)tile);
          mbar_arrive(&sfull_bar[slot]);
          mbar_arrive_cluster(mapa_shared(smem_u32(&sfull_bar[slot]), 1));
        }
      } else {
        mbar_wait_cluster(&sfull_bar[slot], sphase);
        tile = sched_tile[slot];
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(&sempty_bar[slot]), 0));
      }
      if (++slot == SCHED_SLOTS) {
        slot = 0;
        sphase ^= 1u;
      }
      if (tile < 0) break;
      if (lane == 0) tmem_base_smem[1] = 1u;  // this CTA ran a tile (end stamp below)
      int tm, tn, ks, half;
      unit_info(tile, p, tm, tn, ks, half);
      // W rows of this CTA (64-row TMA boxes): a full tile takes rows [rank*BN/2, +BN/2) of
      // the BN-wide tile; a half tile h (N = BN/2 over the pair) takes [h*BN/2 + rank*BN/4, +BN/4)
      const int brow = half < 0 ? tn * BN + (int)rank * (BN / 2) : tn * BN + half * (BN / 2) + (int)rank * (BN / 4);
      const uint32_t tx = half < 0 ? 2 * C::STAGE_BYTES : 2 * (C::A_BYTES + C::B_BYTES / 2);
      for (int kb = 0; kb < num_kb; ++kb) {
        {
          DIAG_T0();
          mbar_wait_park(&empty_bar[stage], phase ^ 1u);
          if (lane == 0 && leader) DIAG_ADD(2);
        }
        if (lane == 0) {
          const uint32_t fb = mapa_shared(smem_u32(&full_bar[stage]), 0);
          if (leader) mbar_arrive_expect_tx(&full_bar[stage], tx);
          tma_load_2d_pair(sA + stage * C::A_BYTES, &tmA, fb, kb * BK, tm * PM + (int)rank * BM);
          tma_load_2d_pair(sB + stage * C::B_BYTES, &tmB, fb, kb * BK, brow);
          if (half < 0)
            tma_load_2d_pair(sB + stage * C::B_BYTES + (BN / 4) * 128, &tmB, fb, kb * BK, brow + BN / 4);
        }
        __syncwarp();
        if (++stage == C::STAGES) {
          stage = 0;
          phase ^= 1u;
        }
      }
    }
  } else if (warp == MMA_WARP) {
    if (leader) {
      // ---------------- MMA issuer (leader only; M = 256 over both CTAs) ----------------
#ifdef PF_GEMM_DIAG
      const long long _c0 = clock64();
      const unsigned long long _g0 = globaltimer_ns();
#endif
      constexpr uint32_t idesc = umma_idesc_bf16(PM, BN, false, false);
      constexpr uint32_t idesc_half = umma_idesc_bf16(PM, BN / 2, false, false);
      int slot = 0;
      uint32_t sphase = 0;
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t aphase = 0;
      while (true) {
        mbar_wait(&sfull_bar[slot], sphase);
        const int tile = sched_tile[slot];
        __syncwarp();
        if (lane == 0) mbar_arrive(&sempty_bar[slot]);
        if (++slot == SCHED_SLOTS) {
          slot = 0;
          sphase ^= 1u;
        }
        if (tile < 0) break;
        {
          DIAG_T0();
          mbar_wait_cluster(&tempty_bar[acc], aphase ^ 1u);
          if (lane == 0) DIAG_ADD(1);
        }
        tc_fence_after();
#ifdef PF_GEMM_DIAG
        const long long _tm0 = clock64();
#endif
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
        int utm, utn, uks, uhalf;
        unit_info(tile, p, utm, utn, uks, uhalf);
        const uint32_t idesc_u = uhalf < 0 ? idesc : idesc_half;
        for (int kb = 0; kb < num_kb; ++kb) {
          {
            DIAG_T0();
            mbar_wait(&full_bar[stage], phase);
            if (lane == 0) DIAG_ADD(0);
          }
          tc_fence_after();
          if (lane == 0) {
            const uint32_t a_addr = smem_u32(sA + stage * C::A_BYTES);
            const uint32_t b_addr = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
            for (int k = 0; k < BK / UMMA_K; ++k) {
              const uint64_t ad = umma_desc_sw128_kmajor(a_addr + k * UMMA_K * 2);
              const uint64_t bd = umma_desc_sw128_kmajor(b_addr + k * UMMA_K * 2);
              umma_bf16_ss_pair(d_tmem, ad, bd, idesc_u, (kb | k) != 0 ? 1u : 0u);
            }
            umma_commit_pair(&empty_bar[stage]);  // frees this stage in BOTH CTAs
          }
          __syncwarp();
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
        if (lane == 0) umma_commit_pair(&tfull_bar[acc]);  // accumulators ready in both CTAs
#ifdef PF_GEMM_DIAG
        if (lane == 0) atomicAdd(&s_gemm_diag[4], (unsigned long long)(clock64() - _tm0));
        if (lane == 0) atomicAdd(&s_gemm_diag[7], 1ull);
#endif
        __syncwarp();
        if (++acc == 2) {
          acc = 0;
          aphase ^= 1u;
        }
      }
#ifdef PF_GEMM_DIAG
      if (lane == 0) {
        atomicAdd(&s_gemm_diag[8], (unsigned long long)(clock64() - _c0));
        atomicAdd(&s_gemm_diag[9], globaltimer_ns() - _g0);
      }
#endif
    }
  } else if (warp >= EPI_WARP0 && warp < EPI_WARP0 + NUM_EPI_WARPS) {
    // ---------------- epilogue (both CTAs, each on its 128 rows) ----------------
    const int e = warp - EPI_WARP0;
    const int lane_grp = warp & 3;
    const int col_half = e >> 2;
    __nv_bfloat16* my_bias = bias_smem + e * C::COLS_PER_EPI_WARP;
    uint8_t* my_stg = smem + C::STG_OFFSET + e * 2048;
    const uint32_t tempty_leader0 = mapa_shared(smem_u32(&tempty_bar[0]), 0);
    int slot = 0;
    uint32_t sphase = 0;
    int acc = 0;
    uint32_t aphase = 0;
    while (true) {
      if (leader) mbar_wait(&sfull_bar[slot], sphase);
      else mbar_wait_cluster(&sfull_bar[slot], sphase);
      const int tile = sched_tile[slot];
      __syncwarp();
      if (lane == 0) {
        if (leader) mbar_arrive(&sempty_bar[slot]);
        else mbar_arrive_cluster(mapa_shared(smem_u32(&sempty_bar[slot]), 0));
      }
      if (++slot == SCHED_SLOTS) {
        slot = 0;
        sphase ^= 1u;
      }
      if (tile < 0) break;
      int tm, tn, ks, half;
      unit_info(tile, p, tm, tn, ks, half);
      const int row_base = tm * PM + (int)rank * BM + lane_grp * 32;
      if (half < 0) {
        const int col_base = tn * BN + col_half * C::COLS_PER_EPI_WARP;
        const uint32_t taddr = tmem_base + ((uint32_t)(lane_grp * 32) << 16) +
                               (uint32_t)(acc * BN + col_half * C::COLS_PER_EPI_WARP);
        epilogue_tile<C::CHUNKS, EPI, true>(p, &tmY, my_stg, taddr, &tfull_bar[acc], aphase, row_base,
                                            col_base, my_bias, 0);
      } else if constexpr (C::CHUNKS % 2 == 0) {
        constexpr int HC = C::COLS_PER_EPI_WARP / 2;
        const int col_base = tn * BN + half * (BN / 2) + col_half * HC;
        const uint32_t taddr = tmem_base + ((uint32_t)(lane_grp * 32) << 16) + (uint32_t)(acc * BN + col_half * HC);
        epilogue_tile<C::CHUNKS / 2, EPI, true>(p, &tmY, my_stg, taddr, &tfull_bar[acc], aphase, row_base,
                                                col_base, my_bias, 0);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_leader0 + (uint32_t)(acc * 8));
      if (++acc == 2) {
        acc = 0;
        aphase ^= 1u;
      }
    }
    if (lane == 0) bulk_wait0();
  }

  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  if (warp == ALLOC_WARP) tmem_dealloc_pair(tmem_base, C::TMEM_COLS);
  DIAG_FLUSH();
  // end stamp only from CTAs that ran a tile: a CTA that starts after the bubble closed (its
  // SM was busy with the main job) and exits without work does not extend the kernel's span
  if (threadIdx.x == 0 && p.stamp && tmem_base_smem[1] != 0u) atomicMax(&p.stamp[1], globaltimer_ns());
}

// ---------------------------------------------------------------------------
// host side

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

// 2-D bf16 row-major [rows, cols] tensor, box [box_rows, 64 cols], 128-B swizzle.
static int make_tmap(CUtensorMap* map, const void* base, int rows, int cols, int box_rows) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return set_error(PF_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(PF_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return PF_OK;
}

// MN-major operand [rows = K, cols = M or N] row-major: 64 x 64 boxes, 128-B swizzle.
static int make_tmap_mn(CUtensorMap* map, const void* base, int rows, int cols) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return set_error(PF_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, 64};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(PF_ERR_CUDA, "MN-major tensor map failed (%d)", (int)r);
  return PF_OK;
}

// Output map for the epilogue's TMA stores: box 32 x 32, 64-B swizzle.
static int make_tmap_store(CUtensorMap* map, const void* base, int rows, int cols) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return set_error(PF_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(PF_ERR_CUDA, "output tensor map failed (%d)", (int)r);
  return PF_OK;
}

// Split-K output map: a [splits, rows, cols] stack, box 32 x 32 x 1, 64-B swizzle
// (clipped per slice, so a ragged last m-tile never spills into the next slice).
static int make_tmap_store_3d(CUtensorMap* map, const void* base, int splits, int rows, int cols) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return set_error(PF_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)splits};
  cuuint64_t strides[2] = {(cuuint64_t)cols * 2, (cuuint64_t)rows * cols * 2};
  cuuint32_t box[3] = {32, 32, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(PF_ERR_CUDA, "split-K output tensor map failed (%d)", (int)r);
  return PF_OK;
}

// Effective split count: every slice gets >= 1 K-block.
static int effective_splits(int K, int requested) {
  const int kb = (K + BK - 1) / BK;
  int s = requested < 1 ? 1 : (requested > kb ? kb : requested);
  const int per = (kb + s - 1) / s;
  return (kb + per - 1) / per;
}

// Tail wave in half tiles (Params::tail_halves): a last wave of rem <= grid/2 tiles is run
// as 2 x rem half-width units. BN 128 / 256 only (the halves keep whole 32-column
// epilogue chunks per warp). PF_GEMM_TAIL=0 disables it.
static int tail_n_full(int tiles, int bn) {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("PF_GEMM_TAIL");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  const int sms = device_sm_count();
  if (!on || (bn != 128 && bn != 256) || tiles <= sms) return tiles;
  const int rem = tiles % sms;
  return (rem > 0 && 2 * rem <= sms) ? tiles - rem : tiles;
}

// The same for CTA-pair tiles (grid = SM pairs); BN 256 only (half = 128 columns over the pair).
static int tail_n_full_pairs(int tiles, int bn) {
  const int pairs = device_sm_count() / 2;
  if (bn != 256 || tiles <= pairs) return tiles;
  const char* e = getenv("PF_GEMM_TAIL");
  if (e && e[0] == '0') return tiles;
  const int rem = tiles % pairs;
  return (rem > 0 && 2 * rem <= pairs) ? tiles - rem : tiles;
}

// Rasterisation group height; PF_GEMM_GROUP_M=<n> overrides GROUP_M (experiments).
static int group_m() {
  static int g = -1;
  if (g < 0) {
    const char* e = getenv("PF_GEMM_GROUP_M");
    g = (e && atoi(e) > 0) ? atoi(e) : GROUP_M;
  }
  return g;
}

// BN choice: minimise waves x per-tile time on 148 SMs.
static int pick_bn(int M, int N) {
  static int forced = -1;  // PF_GEMM_BN=128|192|256 pins the tile width (experiments)
  if (forced < 0) {
    const char* e = getenv("PF_GEMM_BN");
    forced = e ? atoi(e) : 0;
  }
  if (forced == 128 || forced == 192 || forced == 256) return forced;
  const int sms = device_sm_count();
  const int cands[3] = {256, 192, 128};
  int best = 256;
  long best_cost = -1;
  for (int bn : cands) {
    long tiles = (long)((M + BM - 1) / BM) * ((N + bn - 1) / bn);
    long waves = (tiles + sms - 1) / sms;
    // a tile costs ~ (BN + 200) column-units: a K-block carries a fixed ~200-unit floor
    // (operand staging, barriers, per-MMA overhead) on top of the BN-proportional MMA
    // time (fit to 16384 x {1024, 3072, 4096} x {1024, 4096} sweeps: BN 256 beat 128 by
    // 1.2-1.4x although it runs half the tiles per wave; scripts/gemm_bn_sweep.py)
    long cost = waves * (bn + 200);
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best = bn;
    }
  }
  return best;
}

template <int BN, uint32_t EPI, int MJ = 0>
static int launch_epi(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& ty,
                      const Params& p, int grid,
                      const pf_ctl_t* ctl, cudaStream_t stream) {
  using C = Cfg<BN>;
  static bool attr_set = false;
  if (!attr_set) {
    PF_CUDA(cudaFuncSetAttribute(gemm_kernel<BN, EPI, MJ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 C::SMEM_BYTES));
    attr_set = true;
  }
  PF_CUDA(launch_pdl(gemm_kernel<BN, EPI, MJ>, dim3(grid), dim3(NUM_THREADS), C::SMEM_BYTES, stream, ta, tb,
                     ty, p, make_ctl(ctl)));
  PF_CUDA(cudaGetLastError());
  return PF_OK;
}

template <int BN, uint32_t EPI>
static int launch_pair_epi(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& ty,
                           const Params& p, int grid,
                           const pf_ctl_t* ctl, cudaStream_t stream) {
  using C = Cfg2<BN>;
  static bool attr_set = false;
  if (!attr_set) {
    PF_CUDA(cudaFuncSetAttribute(gemm2_kernel<BN, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 C::SMEM_BYTES));
    attr_set = true;
  }
  gemm2_kernel<BN, EPI><<<grid, NUM_THREADS, C::SMEM_BYTES, stream>>>(ta, tb, ty, p, make_ctl(ctl));
  PF_CUDA(cudaGetLastError());
  return PF_OK;
}

// CTA-pair GEMM: 256 x BN tiles per cluster of 2 SMs.
template <int BN>
struct GemmPairOp final : PreparedOp {
  CUtensorMap ta, tb, ty;
  Params p;
  uint32_t epi = 0;
  int grid = 0;

  int prepare(const void* X, const void* W, const void* bias, const void* residual, void* Y, int M,
              int N, int K, uint32_t e) {
    PF_TRY(make_tmap(&ta, X, M, K, BM));
    PF_TRY(make_tmap(&tb, W, N, K, BN / 4));  // 64-row boxes: 2 per full tile, 1 per half tile
    PF_TRY(make_tmap_store(&ty, Y, M, N));
    p.Y = reinterpret_cast<__nv_bfloat16*>(Y);
    p.bias = reinterpret_cast<const __nv_bfloat16*>(bias);
    p.residual = reinterpret_cast<const __nv_bfloat16*>(residual);
    p.M = M;
    p.N = N;
    p.K = K;
    p.tiles_m = (M + 2 * BM - 1) / (2 * BM);
    p.tiles_n = (N + BN - 1) / BN;
    p.stamp = nullptr;
    p.k_splits = 1;
    p.group_m = group_m();
    p.kb_per_split = (K + BK - 1) / BK;
    const int tiles = p.tiles_m * p.tiles_n;
    const int pairs = device_sm_count() / 2;
    grid = 2 * (tiles < pairs ? tiles : pairs);
    p.n_full = tail_n_full_pairs(tiles, BN);
    p.tail_halves = p.n_full < tiles ? 1 : 0;
    epi = e & 15u;
    return PF_OK;
  }
  uint32_t units() const override { return (uint32_t)(2 * p.tiles_m * p.tiles_n - p.n_full); }
  bool resumable() const override { return true; }
  int run(const pf_ctl_t* ctl, cudaStream_t stream, const LaunchArgs& a) override {
    Params p = this->p;
    p.stamp = a.stamp;
    switch (epi) {
      case 0: return launch_pair_epi<BN, 0>(ta, tb, ty, p, grid, ctl, stream);
      case 1: return launch_pair_epi<BN, 1>(ta, tb, ty, p, grid, ctl, stream);
      case 2: return launch_pair_epi<BN, 2>(ta, tb, ty, p, grid, ctl, stream);
      case 3: return launch_pair_epi<BN, 3>(ta, tb, ty, p, grid, ctl, stream);
      case 4: return launch_pair_epi<BN, 4>(ta, tb, ty, p, grid, ctl, stream);
      case 5: return launch_pair_epi<BN, 5>(ta, tb, ty, p, grid, ctl, stream);
      case 6: return launch_pair_epi<BN, 6>(ta, tb, ty, p, grid, ctl, stream);
      case 7: return launch_pair_epi<BN, 7>(ta, tb, ty, p, grid, ctl, stream);
      case 8: return launch_pair_epi<BN, 8>(ta, tb, ty, p, grid, ctl, stream);
      case 9: return launch_pair_epi<BN, 9>(ta, tb, ty, p, grid, ctl, stream);
      case 12: return launch_pair_epi<BN, 12>(ta, tb, ty, p, grid, ctl, stream);
      case 13: return launch_pair_epi<BN, 13>(ta, tb, ty, p, grid, ctl, stream);
      default: return set_error(PF_ERR_INVALID, "pf_gemm: unsupported epilogue");
    }
  }
};

// Variant choice: 0 = single-CTA (BN from pick_bn), 1 = CTA pair BN=256, 2 = CTA pair BN=128.
// Default (PF_GEMM_PAIR unset): the CTA pair with BN 256 for long-K or wide-N GEMMs with at
// least two waves of pair tiles -- in situ at BERT-large batch 128 it wins on FFN1 (N 4096,
// bias+GELU: 119 -> 110-114 us) and FFN2 (K 4096: 110 -> 105 us) and loses on QKV (N 3072, tie)
// and the out-projection (N 1024, K 1024: the single-CTA kernel's half-tile tail wave wins);
// BN 128 pairs are never chosen by default (their MMA loop runs at ~1/3 of the ideal rate).
// PF_GEMM_PAIR=0 never pairs, =1 pairs with the round-1 wave-cost choice, =2 always BN 256.
static int pick_variant(int M, int N, int K) {
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("PF_GEMM_PAIR");
    mode = !e ? 3 : e[0] == '1' ? 1 : e[0] == '2' ? 2 : 0;
  }
  if (mode == 0 || M < 2 * BM) return 0;
  if (mode == 2) return 1;
  const long pairs = device_sm_count() / 2;
  const long t256 = (long)((M + 255) / 256) * ((N + 255) / 256);
  if (mode == 3) return (K >= 2048 || N >= 4096) && N >= 512 && t256 >= 2 * pairs ? 1 : 0;
  const long t128 = (long)((M + 255) / 256) * ((N + 127) / 128);
  const long c256 = ((t256 + pairs - 1) / pairs) * 256;
  const long c128 = ((t128 + pairs - 1) / pairs) * 128;
  return c256 <= c128 ? 1 : 2;
}

template <int BN>
struct GemmOp final : PreparedOp {
  CUtensorMap ta, tb, ty;
  Params p;
  uint32_t epi = 0;
  int grid = 0;
  int mj = 0;  // operand majorness (see gemm_kernel)

  // A [K, M] (mj bit 0) and/or B [K, N] (mj bit 1) stored MN-major
  int prepare_mn(const void* X, const void* W, const void* bias, const void* residual, void* Y, int M, int N,
                 int K, uint32_t e, int majors, int splits) {
    PF_TRY(prepare(X, W, bias, residual, Y, M, N, K, e));
    mj = majors;
    if (mj != 0 || splits > 1) {  // the tail halves are for the forward (K-major, unsplit) GEMMs
      p.tail_halves = 0;
      p.n_full = p.tiles_m * p.tiles_n;
    }
    if (mj & 1) PF_TRY(make_tmap_mn(&ta, X, K, M));
    if (mj & 2) PF_TRY(make_tmap_mn(&tb, W, K, N));
    if (splits > 1) {
      const int kb = (K + BK - 1) / BK;
      p.k_splits = effective_splits(K, splits);
      p.kb_per_split = (kb + p.k_splits - 1) / p.k_splits;
      if (p.k_splits > 1) PF_TRY(make_tmap_store_3d(&ty, Y, p.k_splits, M, N));
      const int tiles = p.tiles_m * p.tiles_n * p.k_splits;
      const int sms = device_sm_count();
      grid = tiles < sms ? tiles : sms;
    }
    return PF_OK;
  }

  int prepare(const void* X, const void* W, const void* bias, const void* residual, void* Y, int M,
              int N, int K, uint32_t e) {
    PF_TRY(make_tmap(&ta, X, M, K, BM));
    PF_TRY(make_tmap(&tb, W, N, K, BN));
    PF_TRY(make_tmap_store(&ty, Y, M, N));
    p.Y = reinterpret_cast<__nv_bfloat16*>(Y);
    p.bias = reinterpret_cast<const __nv_bfloat16*>(bias);
    p.residual = reinterpret_cast<const __nv_bfloat16*>(residual);
    p.M = M;
    p.N = N;
    p.K = K;
    p.tiles_m = (M + BM - 1) / BM;
    p.tiles_n = (N + BN - 1) / BN;
    p.stamp = nullptr;
    p.k_splits = 1;
    p.group_m = group_m();
    p.kb_per_split = (K + BK - 1) / BK;
    const int tiles = p.tiles_m * p.tiles_n;
    const int sms = device_sm_count();
    grid = tiles < sms ? tiles : sms;
    p.n_full = tail_n_full(tiles, BN);
    p.tail_halves = p.n_full < tiles ? 1 : 0;
    epi = e & 15u;
    return PF_OK;
  }
  // Split-K: Y is a [splits, M, N] stack of partial products over K slices (no epilogue).
  int prepare_splitk(const void* X, const void* W, void* Y, int M, int N, int K, int splits) {
    PF_TRY(prepare(X, W, nullptr, nullptr, Y, M, N, K, 0u));
    p.tail_halves = 0;
    p.n_full = p.tiles_m * p.tiles_n;
    const int kb = (K + BK - 1) / BK;
    p.k_splits = effective_splits(K, splits);
    p.kb_per_split = (kb + p.k_splits - 1) / p.k_splits;
    if (p.k_splits > 1) PF_TRY(make_tmap_store_3d(&ty, Y, p.k_splits, M, N));
    const int tiles = p.tiles_m * p.tiles_n * p.k_splits;
    const int sms = device_sm_count();
    grid = tiles < sms ? tiles : sms;
    return PF_OK;
  }
  uint32_t units() const override {
    return p.tail_halves ? (uint32_t)(2 * p.tiles_m * p.tiles_n - p.n_full)
                         : (uint32_t)(p.tiles_m * p.tiles_n * p.k_splits);
  }
  bool resumable() const override { return true; }
  int run(const pf_ctl_t* ctl, cudaStream_t stream, const LaunchArgs& a) override {
    Params p = this->p;
    p.stamp = a.stamp;
    if (mj == 3) return launch_epi<BN, 0, 3>(ta, tb, ty, p, grid, ctl, stream);
    if (mj == 2) return epi == 4 ? launch_epi<BN, 4, 2>(ta, tb, ty, p, grid, ctl, stream)
                                 : launch_epi<BN, 0, 2>(ta, tb, ty, p, grid, ctl, stream);
    switch (epi) {
      case 0: return launch_epi<BN, 0>(ta, tb, ty, p, grid, ctl, stream);
      case 1: return launch_epi<BN, 1>(ta, tb, ty, p, grid, ctl, stream);
      case 2: return launch_epi<BN, 2>(ta, tb, ty, p, grid, ctl, stream);
      case 3: return launch_epi<BN, 3>(ta, tb, ty, p, grid, ctl, stream);
      case 4: return launch_epi<BN, 4>(ta, tb, ty, p, grid, ctl, stream);
      case 5: return launch_epi<BN, 5>(ta, tb, ty, p, grid, ctl, stream);
      case 6: return launch_epi<BN, 6>(ta, tb, ty, p, grid, ctl, stream);
      case 7: return launch_epi<BN, 7>(ta, tb, ty, p, grid, ctl, stream);
      case 8: return launch_epi<BN, 8>(ta, tb, ty, p, grid, ctl, stream);
      case 9: return launch_epi<BN, 9>(ta, tb, ty, p, grid, ctl, stream);
      case 12: return launch_epi<BN, 12>(ta, tb, ty, p, grid, ctl, stream);
      case 13: return launch_epi<BN, 13>(ta, tb, ty, p, grid, ctl, stream);
      default: return set_error(PF_ERR_INVALID, "pf_gemm: unsupported epilogue");
    }
  }
};

}  // namespace gemm

int make_gemm_op(OpPtr* out, const void* X, const void* W, const void* bias, const void* residual,
                 void* Y, int M, int N, int K, uint32_t epilogue) {
  if (!X || !W || !Y || M <= 0 || N <= 0 || K <= 0)
    return set_error(PF_ERR_INVALID, "pf_gemm: null pointer or non-positive shape");
  if (K % 8 != 0 || N % 8 != 0)
    return set_error(PF_ERR_INVALID, "pf_gemm: K and N must be multiples of 8 (16-B rows)");
  if ((epilogue & PF_EPI_BIAS) && !bias) return set_error(PF_ERR_INVALID, "pf_gemm: bias is NULL");
  if ((epilogue & PF_EPI_RESIDUAL) && !residual)
    return set_error(PF_ERR_INVALID, "pf_gemm: residual is NULL");
  if ((epilogue & PF_EPI_GELU) && (epilogue & PF_EPI_RELU))
    return set_error(PF_ERR_INVALID, "pf_gemm: GELU and ReLU are exclusive");
  if (epilogue & ~15u) return set_error(PF_ERR_INVALID, "pf_gemm: unknown epilogue bits");
  if (((uintptr_t)X | (uintptr_t)W | (uintptr_t)Y | (uintptr_t)bias | (uintptr_t)residual) & 15u)
    return set_error(PF_ERR_INVALID, "pf_gemm: pointers must be 16-B aligned");
  if (!device_is_sm100()) return set_error(PF_ERR_UNSUPPORTED, "pf_gemm: needs an sm_100 device");
  const int variant = gemm::pick_variant(M, N, K);
  if (variant == 1 || variant == 2) {
    if (variant == 1) {
      auto op = std::make_unique<gemm::GemmPairOp<256>>();
      PF_TRY(op->prepare(X, W, bias, residual, Y, M, N, K, epilogue));
      *out = std::move(op);
    } else {
      auto op = std::make_unique<gemm::GemmPairOp<128>>();
      PF_TRY(op->prepare(X, W, bias, residual, Y, M, N, K, epilogue));
      *out = std::move(op);
    }
    return PF_OK;
  }
  switch (gemm::pick_bn(M, N)) {
    case 256: {
      auto op = std::make_unique<gemm::GemmOp<256>>();
      PF_TRY(op->prepare(X, W, bias, residual, Y, M, N, K, epilogue));
      *out = std::move(op);
      return PF_OK;
    }
    case 192: {
      auto op = std::make_unique<gemm::GemmOp<192>>();
      PF_TRY(op->prepare(X, W, bias, residual, Y, M, N, K, epilogue));
      *out = std::move(op);
      return PF_OK;
    }
    default: {
      auto op = std::make_unique<gemm::GemmOp<128>>();
      PF_TRY(op->prepare(X, W, bias, residual, Y, M, N, K, epilogue));
      *out = std::move(op);
      return PF_OK;
    }
  }
}

}  // namespace pf

namespace pf {

// Y = X[M,K] . Wkn[K,N] (B MN-major: W stored [K, N]) with an optional residual (data
// gradients: dX = dZ . W with W [Cout, Cin*kh*kw] as stored), or the split-K weight
// gradient Y[z] = A[Kz, M]^T . B[Kz, N] (both MN-major: dZ^T X without transposes).
int make_gemm_mn_op(OpPtr* out, const void* X, const void* W, const void* residual, void* Y, int M, int N, int K,
                    int majors, int splits) {
  if (!X || !W || !Y || M <= 0 || N <= 0 || K <= 0 || (majors != 2 && majors != 3))
    return set_error(PF_ERR_INVALID, "pf_gemm_mn: bad arguments");
  if (N % 8 != 0 || ((majors & 1) && M % 8 != 0) || (!(majors & 1) && K % 8 != 0))
    return set_error(PF_ERR_INVALID, "pf_gemm_mn: 16-B rows needed (N %% 8, and M %% 8 or K %% 8)");
  if (((uintptr_t)X | (uintptr_t)W | (uintptr_t)Y | (uintptr_t)residual) & 15u)
    return set_error(PF_ERR_INVALID, "pf_gemm_mn: pointers must be 16-B aligned");
  if (majors == 3 && residual) return set_error(PF_ERR_INVALID, "pf_gemm_mn: no residual with split-K");
  if (!device_is_sm100()) return set_error(PF_ERR_UNSUPPORTED, "pf_gemm_mn: needs an sm_100 device");
  const uint32_t e = residual ? PF_EPI_RESIDUAL : 0u;
  switch (gemm::pick_bn(M, N)) {
    case 256: {
      auto op = std::make_unique<gemm::GemmOp<256>>();
      PF_TRY(op->prepare_mn(X, W, nullptr, residual, Y, M, N, K, e, majors, splits));
      *out = std::move(op);
      return PF_OK;
    }
    case 192: {
      auto op = std::make_unique<gemm::GemmOp<192>>();
      PF_TRY(op->prepare_mn(X, W, nullptr, residual, Y, M, N, K, e, majors, splits));
      *out = std::move(op);
      return PF_OK;
    }
    default: {
      auto op = std::make_unique<gemm::GemmOp<128>>();
      PF_TRY(op->prepare_mn(X, W, nullptr, residual, Y, M, N, K, e, majors, splits));
      *out = std::move(op);
      return PF_OK;
    }
  }
}

int make_gemm_splitk_op(OpPtr* out, const void* X, const void* W, void* Y, int M, int N, int K,
                        int splits) {
  if (!X || !W || !Y || M <= 0 || N <= 0 || K <= 0 || splits < 1)
    return set_error(PF_ERR_INVALID, "pf_gemm_splitk: null pointer or non-positive shape");
  if (K % 8 != 0 || N % 8 != 0)
    return set_error(PF_ERR_INVALID, "pf_gemm_splitk: K and N must be multiples of 8 (16-B rows)");
  if (((uintptr_t)X | (uintptr_t)W | (uintptr_t)Y) & 15u)
    return set_error(PF_ERR_INVALID, "pf_gemm_splitk: pointers must be 16-B aligned");
  if (!device_is_sm100()) return set_error(PF_ERR_UNSUPPORTED, "pf_gemm_splitk: needs an sm_100 device");
  switch (gemm::pick_bn(M, N)) {
    case 256: {
      auto op = std::make_unique<gemm::GemmOp<256>>();
      PF_TRY(op->prepare_splitk(X, W, Y, M, N, K, splits));
      *out = std::move(op);
      return PF_OK;
    }
    case 192: {
      auto op = std::make_unique<gemm::GemmOp<192>>();
      PF_TRY(op->prepare_splitk(X, W, Y, M, N, K, splits));
      *out = std::move(op);
      return PF_OK;
    }
    default: {
      auto op = std::make_unique<gemm::GemmOp<128>>();
      PF_TRY(op->prepare_splitk(X, W, Y, M, N, K, splits));
      *out = std::move(op);
      return PF_OK;
    }
  }
}

}  // namespace pf

extern "C" int pf_gemm_splitk(const void* X, const void* W, void* Y, int M, int N, int K, int splits,
                              const pf_ctl_t* ctl, void* stream) {
  using namespace pf;
  PF_TRY(validate_ctl(ctl));
  OpPtr op;
  PF_TRY(make_gemm_splitk_op(&op, X, W, Y, M, N, K, splits));
  return op->run(ctl, reinterpret_cast<cudaStream_t>(stream), pf::LaunchArgs{});
}

extern "C" int pf_gemm_nn(const void* X, const void* Wkn, const void* residual, void* Y, int M, int N, int K,
                          const pf_ctl_t* ctl, void* stream) {
  using namespace pf;
  PF_TRY(validate_ctl(ctl));
  OpPtr op;
  PF_TRY(make_gemm_mn_op(&op, X, Wkn, residual, Y, M, N, K, 2, 1));
  return op->run(ctl, reinterpret_cast<cudaStream_t>(stream), pf::LaunchArgs{});
}

extern "C" int pf_gemm_splitk_tn(const void* A, const void* B, void* Y, int M, int N, int K, int splits,
                                 const pf_ctl_t* ctl, void* stream) {
  using namespace pf;
  PF_TRY(validate_ctl(ctl));
  OpPtr op;
  PF_TRY(make_gemm_mn_op(&op, A, B, nullptr, Y, M, N, K, 3, splits));
  return op->run(ctl, reinterpret_cast<cudaStream_t>(stream), pf::LaunchArgs{});
}

extern "C" int pf_gemm_splitk_splits(int K, int requested, int* out_splits) {
  if (!out_splits || K <= 0) return pf::set_error(PF_ERR_INVALID, "pf_gemm_splitk_splits");
  *out_splits = pf::gemm::effective_splits(K, requested);
  return PF_OK;
}

extern "C" int pf_gemm_diag(unsigned long long* out8, int reset) {
#ifdef PF_GEMM_DIAG
  if (out8) cudaMemcpyFromSymbol(out8, pf::gemm::g_gemm_diag, sizeof(unsigned long long) * 16);
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(pf::gemm::g_gemm_diag, z, sizeof(z));
  }
  return PF_OK;
#else
  (void)out8;
  (void)reset;
  return PF_ERR_UNSUPPORTED;
#endif
}

extern "C" int pf_gemm_units(int M, int N, int K, uint32_t* out_units) {
  using namespace pf;
  if (!out_units || M <= 0 || N <= 0 || K <= 0) return set_error(PF_ERR_INVALID, "pf_gemm_units");
  const int variant = gemm::pick_variant(M, N, K);
  if (variant) {
    const int bnp = variant == 1 ? 256 : 128;
    const int tiles = ((M + 2 * gemm::BM - 1) / (2 * gemm::BM)) * ((N + bnp - 1) / bnp);
    *out_units = (uint32_t)(2 * tiles - gemm::tail_n_full_pairs(tiles, bnp));
    return PF_OK;
  }
  const int bn = gemm::pick_bn(M, N);
  const int tiles = ((M + gemm::BM - 1) / gemm::BM) * ((N + bn - 1) / bn);
  *out_units = (uint32_t)(2 * tiles - gemm::tail_n_full(tiles, bn));
  return PF_OK;
}

extern "C" int pf_gemm(const void* X, const void* W, const void* bias, const void* residual,
                       void* Y, int M, int N, int K, uint32_t epilogue, const pf_ctl_t* ctl,
                       void* stream) {
  using namespace pf;
  PF_TRY(validate_ctl(ctl));
  OpPtr op;
  PF_TRY(make_gemm_op(&op, X, W, bias, residual, Y, M, N, K, epilogue));
  return op->run(ctl, reinterpret_cast<cudaStream_t>(stream), pf::LaunchArgs{});
}
