// gemm_tc.cuh — persistent tcgen05 GEMM for the encoder's linear layers
// (SURVEY.md §2.6 B1/B2/B4/B5/B9):  D[M, N] = A[M, K] · W[N, K]^T  (+ fused epilogue)
//
//   A  : bf16 activations, row-major [M_cap, K]            (TMA, 128B swizzle)
//   W  : bf16 weights repacked K-major [N, K] by cfd_create  (TMA, 128B swizzle)
//   D  : fp32 accumulator in TMEM, double-buffered (2 x BN columns) so the
//        epilogue of tile i overlaps the MMAs of tile i+1.
//
// Warp roles (192 threads, one CTA per SM, persistent over tiles):
//   warp 0      TMA producer (one elected lane), STAGES-deep smem ring
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2..5  epilogue: tcgen05.ld (32 lanes x 32 cols per load), fused
//               bias / GELU / residual / PE / row-scatter, global stores.
//
// The row count may live on the device (`m_dev`, produced by the gather kernel)
// so a refine batch never syncs the host.  Rows >= M are never stored except
// for the "pad" range [M, M_pad) of bf16 outputs, which is written so that
// attention's tail tiles read finite values (see attn_tc.cuh).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "ptx.cuh"

namespace cfd {

enum EpiKind : int {
  EPI_BF16_BIAS = 0,       // out_bf16 = bf16(acc + bias)                      (QKV)
  EPI_BF16_BIAS_GELU = 1,  // out_bf16 = bf16(GELU(acc + bias))                (MLP1)
  EPI_F32_RESID = 2,       // out_f32 += acc + bias                            (O-proj, MLP2)
  EPI_EMBED_COARSE = 3,    // out_f32 = out2_f32 = acc + bias + pe[row % pe_rows]   (B1)
  EPI_EMBED_FINE = 4,      // out_f32[frow[row]] = acc + bias + pe[fidx[row]]        (B9)
};

struct GemmParams {
  int M;               // row count when m_dev == nullptr
  const int* m_dev;    // device row count (optional)
  int m_cap;           // capacity rows of the A / output buffers
  int N, K;
  const float* bias;   // [N]
  __nv_bfloat16* out_bf16;  // [m_cap, N]
  float* out_f32;      // [*, ld_out]
  float* out2_f32;     // [*, ld_out] (EMBED_COARSE copy)
  int ld_out;
  const float* pe;     // [*, N]
  int pe_rows;
  const int* frow;
  const int* fidx;
};

constexpr int GEMM_BM = 128;
constexpr int GEMM_BK = 64;
constexpr int GEMM_THREADS = 192;

template <int BN, int STAGES>
struct GemmSmem {
  static constexpr int A_BYTES = GEMM_BM * GEMM_BK * 2;
  static constexpr int B_BYTES = BN * GEMM_BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int BAR_BYTES = 256;
  static constexpr int TOTAL = 1024 /*align slack*/ + STAGES * STAGE_BYTES + BAR_BYTES;
  static constexpr uint32_t TMEM_COLS = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128
                                        : (2 * BN <= 256) ? 256 : 512;
};

// Rows a varlen attention tile may touch past the last valid row: a task's last KV
// tile starts at (task start + 128 j) and so can overhang the packed rows by < 128.
__host__ __device__ __forceinline__ int pad_rows(int M, int cap) {
  const int r = ((M + 127) / 128) * 128 + 128;
  return r < cap ? r : cap;
}

__device__ __forceinline__ float gelu_erf(float v) { return 0.5f * v * (1.0f + erff(v * 0.70710678118654752f)); }

template <int EPI>
__device__ __forceinline__ void gemm_epilogue_chunk(const GemmParams& p, int row, int col0, const uint32_t (&r)[32],
                                                    bool store_ok) {
  float v[32];
  const float4* b4 = reinterpret_cast<const float4*>(p.bias + col0);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float4 b = __ldg(b4 + i);
    v[4 * i + 0] = __uint_as_float(r[4 * i + 0]) + b.x;
    v[4 * i + 1] = __uint_as_float(r[4 * i + 1]) + b.y;
    v[4 * i + 2] = __uint_as_float(r[4 * i + 2]) + b.z;
    v[4 * i + 3] = __uint_as_float(r[4 * i + 3]) + b.w;
  }
  if (!store_ok) return;
  if constexpr (EPI == EPI_BF16_BIAS || EPI == EPI_BF16_BIAS_GELU) {
    uint32_t pk[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      float a = v[2 * i], b = v[2 * i + 1];
      if constexpr (EPI == EPI_BF16_BIAS_GELU) { a = gelu_erf(a); b = gelu_erf(b); }
      pk[i] = pack_bf16x2(a, b);
    }
    uint4* dst = reinterpret_cast<uint4*>(p.out_bf16 + (size_t)row * p.N + col0);
#pragma unroll
    for (int i = 0; i < 4; ++i) dst[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
  } else if constexpr (EPI == EPI_F32_RESID) {
    float4* dst = reinterpret_cast<float4*>(p.out_f32 + (size_t)row * p.ld_out + col0);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float4 o = dst[i];
      o.x += v[4 * i + 0]; o.y += v[4 * i + 1]; o.z += v[4 * i + 2]; o.w += v[4 * i + 3];
      dst[i] = o;
    }
  } else if constexpr (EPI == EPI_EMBED_COARSE) {
    const float4* pe4 = reinterpret_cast<const float4*>(p.pe + (size_t)(row % p.pe_rows) * p.N + col0);
    float4* d1 = reinterpret_cast<float4*>(p.out_f32 + (size_t)row * p.ld_out + col0);
    float4* d2 = reinterpret_cast<float4*>(p.out2_f32 + (size_t)row * p.ld_out + col0);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float4 e = __ldg(pe4 + i);
      float4 o = make_float4(v[4 * i] + e.x, v[4 * i + 1] + e.y, v[4 * i + 2] + e.z, v[4 * i + 3] + e.w);
      d1[i] = o;
      d2[i] = o;
    }
  } else if constexpr (EPI == EPI_EMBED_FINE) {
    const int orow = __ldg(p.frow + row);
    const int prow = __ldg(p.fidx + row);
    const float4* pe4 = reinterpret_cast<const float4*>(p.pe + (size_t)prow * p.N + col0);
    float4* d1 = reinterpret_cast<float4*>(p.out_f32 + (size_t)orow * p.ld_out + col0);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float4 e = __ldg(pe4 + i);
      d1[i] = make_float4(v[4 * i] + e.x, v[4 * i + 1] + e.y, v[4 * i + 2] + e.z, v[4 * i + 3] + e.w);
    }
  }
}

template <int BN, int STAGES, int EPI>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const GemmParams p) {
  using S = GemmSmem<BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * S::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * S::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = warp_id(), lane = lane_id();
  const int M = p.m_dev ? __ldg(p.m_dev) : p.M;
  // bf16 outputs (QKV, MLP1) also cover the pad rows [M, pad_rows(M)) so attention's
  // tail tiles (which may start at any row of the last task) read finite values
  constexpr bool kPad = (EPI == EPI_BF16_BIAS || EPI == EPI_BF16_BIAS_GELU);
  const int m_store = kPad ? pad_rows(M, p.m_cap) : M;
  const int m_tiles = (m_store + GEMM_BM - 1) / GEMM_BM;
  const int n_tiles = p.N / BN;
  const int num_k = p.K / GEMM_BK;
  const int total = m_tiles * n_tiles;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 4); }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<S::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
        const int m_blk = tile / n_tiles, n_blk = tile % n_tiles;
        for (int kb = 0; kb < num_k; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], S::STAGE_BYTES);
          tma_load_2d(sA + stage * S::A_BYTES, &tmA, &full[stage], kb * GEMM_BK, m_blk * GEMM_BM);
          tma_load_2d(sB + stage * S::B_BYTES, &tmB, &full[stage], kb * GEMM_BK, n_blk * BN);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc_bf16(GEMM_BM, BN, 0);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < num_k; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + stage * S::A_BYTES);
          const uint32_t b0 = smem_u32(sB + stage * S::B_BYTES);
#pragma unroll
          for (int k = 0; k < GEMM_BK / 16; ++k) {
            const uint64_t ad = make_smem_desc(a0 + k * 32, 16, 1024, kLayoutSW128);
            const uint64_t bd = make_smem_desc(b0 + k * 32, 16, 1024, kLayoutSW128);
            mma_ss(d_tmem, ad, bd, idesc, (kb | k) != 0);
          }
          mma_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int row_in_tile = quarter * 32 + lane;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
      const int m_blk = tile / n_tiles, n_blk = tile % n_tiles;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row = m_blk * GEMM_BM + row_in_tile;
      const bool ok = row < m_store;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + acc * BN + c * 32, r);
        tmem_wait_ld();
        gemm_epilogue_chunk<EPI>(p, row, n_blk * BN + c * 32, r, ok);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<S::TMEM_COLS>(tmem_base);
}

}  // namespace cfd
