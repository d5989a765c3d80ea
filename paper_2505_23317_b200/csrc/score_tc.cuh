// score_tc.cuh — per-region criticality score (reading R5):
//
//   s_j = 1/(nh*Nc) * sum_h sum_i exp(S_h[i,j] - LSE_h[i]),   S_h = q_h k_h^T / sqrt(dh)
//
// i.e. the attention mass coarse region j receives at the score layer
// (draft A2 "attention map" region proposal, PAPER.md:361/417/497).  The row
// log-sum-exps come from the attention kernel of that layer; this kernel
// recomputes S^T = K Q^T on tcgen05 with keys on the TMEM lanes, so each thread
// owns one key column and sums its column in a fixed (head, q-tile, row) order:
// deterministic, no atomics.
//
// One CTA = (key tile of 128, frame).  Warp 0 TMA, warp 1 MMA, warps 2..9 reduce: two
// warps per TMEM lane quarter, each over half of the 128 query columns with four partial
// sums (the exp pass is latency-bound with one warp per SMSP and a single add chain); the
// two halves are combined in a fixed order at the end.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include "ptx.cuh"

namespace cfd {

struct ScoreParams {
  int n_coarse;       // Nc (tokens per frame)
  int n_heads;
  int d_model;
  const float* lse;   // [nh, lse_ld], natural log
  int lse_ld;
  float scale_log2;   // log2(e)/sqrt(dh)
  float* scores;      // [B, Nc]
};

constexpr int SCORE_THREADS = 320;

template <int DH>
struct ScoreSmem {
  static constexpr int T_BYTES = 128 * DH * 2;
  static constexpr int TOTAL = 1024 + 3 * T_BYTES + 2 * 128 * 4 + 256 + 128 * 4;
};

__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <int DH>
__global__ void __launch_bounds__(SCORE_THREADS, 1)
    score_tc_kernel(const __grid_constant__ CUtensorMap tmQKV, const ScoreParams p) {
  using S = ScoreSmem<DH>;
  const int kt = blockIdx.x, b = blockIdx.y;
  const int Nc = p.n_coarse;
  const int nq = (Nc + 127) / 128;
  const int total = p.n_heads * nq;
  const int row0 = b * Nc;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps the shared space
  uint8_t* sK = smem;
  uint8_t* sQ = smem + S::T_BYTES;  // [2]
  float* lse_s = reinterpret_cast<float*>(sQ + 2 * S::T_BYTES);  // [2][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(lse_s + 256);
  uint64_t* k_full = bars;
  uint64_t* k_empty = bars + 1;
  uint64_t* q_full = bars + 2;   // [2]
  uint64_t* q_empty = bars + 4;  // [2]
  uint64_t* s_full = bars + 6;   // [2]
  uint64_t* s_empty = bars + 8;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 10);

  const int warp = warp_id(), lane = lane_id();
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmQKV);
    mbar_init(k_full, 1);
    mbar_init(k_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 256);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<256>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int it = 0; it < total; ++it) {
        const int h = it / nq, qt = it % nq;
        if (qt == 0) {
          mbar_wait(k_empty, (h & 1) ^ 1);
          mbar_expect_tx(k_full, S::T_BYTES);
          tma_load_2d(sK, &tmQKV, k_full, p.d_model + h * DH, row0 + kt * 128);
        }
        mbar_wait(&q_empty[it & 1], ((it >> 1) & 1) ^ 1);
        mbar_expect_tx(&q_full[it & 1], S::T_BYTES);
        tma_load_2d(sQ + (it & 1) * S::T_BYTES, &tmQKV, &q_full[it & 1], h * DH, row0 + qt * 128);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc_bf16(128, 128, 0);
      const uint32_t k_addr = smem_u32(sK);
      for (int it = 0; it < total; ++it) {
        const int h = it / nq, qt = it % nq;
        if (qt == 0) mbar_wait(k_full, h & 1);
        mbar_wait(&q_full[it & 1], (it >> 1) & 1);
        mbar_wait(&s_empty[it & 1], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t q_addr = smem_u32(sQ + (it & 1) * S::T_BYTES);
#pragma unroll
        for (int k = 0; k < DH / 16; ++k)
          mma_ss(tmem + (it & 1) * 128, make_smem_desc(k_addr + k * 32, 16, 512, kLayoutSW64),
                 make_smem_desc(q_addr + k * 32, 16, 512, kLayoutSW64), idesc, k);
        mma_commit(&s_full[it & 1]);
        mma_commit(&q_empty[it & 1]);
        if (qt == nq - 1) mma_commit(k_empty);
      }
    }
  } else {
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;  // query columns [64 half, 64 half + 64)
    const int r = quarter * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    const float c = p.scale_log2;
    float* xch = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 256);  // [128] half-1 partial sums
    float acc = 0.f;
    // row LSEs of iteration it (head h, query tile qt), staged one iteration ahead so the
    // global load latency is hidden behind the previous iteration's exp pass
    auto lse_of = [&](int it) {
      const int h = it / nq, q = (it % nq) * 128 + r;
      return (q < Nc) ? __ldg(p.lse + (size_t)h * p.lse_ld + row0 + q) * 1.4426950408889634f : 0.f;
    };
    if (half == 0) lse_s[r] = lse_of(0);
    for (int it = 0; it < total; ++it) {
      const int qt = it % nq;
      named_bar_sync(1, 256);  // lse_s[it & 1] complete; everyone is done with lse_s[(it + 1) & 1]
      const float lse_next = (half == 0 && it + 1 < total) ? lse_of(it + 1) : 0.f;
      mbar_wait(&s_full[it & 1], (it >> 1) & 1);
      tc_fence_after();
      uint32_t sr[64];
      const uint32_t a = tmem + lane_off + (it & 1) * 128 + half * 64;
      tmem_ld32(a + 0, *reinterpret_cast<uint32_t(*)[32]>(sr + 0));
      tmem_ld32(a + 32, *reinterpret_cast<uint32_t(*)[32]>(sr + 32));
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(&s_empty[it & 1]);
      const int nvq = min(128, Nc - qt * 128) - half * 64;  // valid query columns of this half
      const float* ls = lse_s + (it & 1) * 128 + half * 64;
      float p0 = 0.f, p1 = 0.f, p2 = 0.f, p3 = 0.f;
#pragma unroll
      for (int i = 0; i < 64; i += 4) {
        const float e0 = ex2_approx(fmaf(__uint_as_float(sr[i]), c, -ls[i]));
        const float e1 = ex2_approx(fmaf(__uint_as_float(sr[i + 1]), c, -ls[i + 1]));
        const float e2 = ex2_approx(fmaf(__uint_as_float(sr[i + 2]), c, -ls[i + 2]));
        const float e3 = ex2_approx(fmaf(__uint_as_float(sr[i + 3]), c, -ls[i + 3]));
        p0 += (i < nvq) ? e0 : 0.f;
        p1 += (i + 1 < nvq) ? e1 : 0.f;
        p2 += (i + 2 < nvq) ? e2 : 0.f;
        p3 += (i + 3 < nvq) ? e3 : 0.f;
      }
      acc += (p0 + p1) + (p2 + p3);
      if (half == 0 && it + 1 < total) lse_s[((it + 1) & 1) * 128 + r] = lse_next;
    }
    // fixed-order combination of the two column halves (deterministic)
    if (half == 1) xch[r] = acc;
    named_bar_sync(1, 256);
    const int key = kt * 128 + r;
    if (half == 0 && key < Nc) p.scores[(size_t)b * Nc + key] = (acc + xch[r]) / (float)(p.n_heads * Nc);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<256>(tmem);
}

}  // namespace cfd
