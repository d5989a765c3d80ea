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
#include "attn_common.cuh"

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
#ifndef CFD_SCORE_NPP
#define CFD_SCORE_NPP 4
#endif
constexpr int SCORE_NPP = CFD_SCORE_NPP;  // polynomial-exp pairs of every 16 (FMA pipe; the rest on MUFU)

template <int DH>
struct ScoreSmem {
  static constexpr int T_BYTES = 128 * DH * 2;
  static constexpr int FIXED = 1024 + 3 * T_BYTES + 256 + 8 * 128 * 4;  // K | Q[2] | barriers | partials
  // + the staged row LSEs of two heads: 2 x (query tiles x 128) floats
  __host__ __device__ static constexpr int total(int nc) { return FIXED + 2 * ((nc + 127) / 128) * 128 * 4; }
};

__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// 4-byte global -> shared copy that does not hold a register until it lands (cp.async)
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// p = 2^(s*c + nl) for 16 score columns (nl = -LSE*log2(e) per query column), summed into (a0, a1);
// pairs [8 - NPPH, 8) on the FMA-pipe polynomial, the rest on MUFU
template <int NPPH>
__device__ __forceinline__ void score_exp16(const uint32_t* sr, const float* nl, float c, float& a0, float& a1) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float2 n = *reinterpret_cast<const float2*>(nl + 2 * i);
    float x0, x1, e0, e1;
    fma2(x0, x1, __uint_as_float(sr[2 * i]), __uint_as_float(sr[2 * i + 1]), c, c, n.x, n.y);
    if (i >= 8 - NPPH) {
      exp2_poly2_d4(e0, e1, x0, x1);
    } else {
      e0 = ex2_approx(x0);
      e1 = ex2_approx(x1);
    }
    add2(a0, a1, a0, a1, e0, e1);
  }
}

// One CTA = (key tile of 128, frame).  Keys sit on the TMEM lanes (S^T = K Q^T), so a thread owns
// one key and sums its row of P^T over the (head, query tile, column) loop in a fixed order:
// deterministic, no atomics.  Warp 0 = TMA, warp 1 = MMA, warps 2..9 = 8 reduce warps (two per
// TMEM lane quarter).  A key tile with nk <= 32 (or <= 64) valid keys is replicated 4x (2x) over
// the lane quarters and the query columns are split between the replicas, so the 16-key tail
// tile of Nc = 400 costs a quarter of a full tile instead of a full one on one SMSP; query columns
// beyond Nc are skipped.  Row LSEs of a head are staged in shared memory by cp.async during the
// previous head.  The partial sums of the 8 warps are combined in a fixed order at the end.
template <int DH>
__global__ void __launch_bounds__(SCORE_THREADS, 2)
    score_tc_kernel(const __grid_constant__ CUtensorMap tmQKV, const __grid_constant__ CUtensorMap tmK32,
                    const ScoreParams p) {
  using S = ScoreSmem<DH>;
  const int kt = blockIdx.x, b = blockIdx.y;
  const int Nc = p.n_coarse;
  const int nq = (Nc + 127) / 128;
  const int nqp = nq * 128;
  const int total = p.n_heads * nq;
  const int row0 = b * Nc;
  const int nk = min(128, Nc - kt * 128);              // valid keys of this tile
  const int rep = nk <= 32 ? 4 : (nk <= 64 ? 2 : 1);   // key replicas over the lane quarters

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sK = smem;
  uint8_t* sQ = smem + S::T_BYTES;  // [2]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sQ + 2 * S::T_BYTES);
  uint64_t* k_full = bars;
  uint64_t* k_empty = bars + 1;
  uint64_t* q_full = bars + 2;   // [2]
  uint64_t* q_empty = bars + 4;  // [2]
  uint64_t* s_full = bars + 6;   // [2]
  uint64_t* s_empty = bars + 8;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 10);
  float* part = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 256);  // [8 warps][128 lanes]
  float* lse_s = part + 8 * 128;                                                  // [2][nqp]

  const int warp = warp_id(), lane = lane_id();
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmQKV);
    tma_prefetch(&tmK32);
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
          // 4 boxes of 32 key rows; slot i (lanes 32i..32i+31) takes rows (i mod 4/rep)*32 of the tile
#pragma unroll
          for (int i = 0; i < 4; ++i)
            tma_load_2d(sK + i * (S::T_BYTES / 4), &tmK32, k_full, p.d_model + h * DH,
                        row0 + kt * 128 + (i % (4 / rep)) * 32);
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
    const int rw = warp - 2;            // reduce warp 0..7
    (void)rw;
    const int quarter = warp & 3;
    const int half = rw >> 2;           // warps 2..5: half 0, 6..9: half 1
    const int tid = rw * 32 + lane;     // 0..255
    const int replica = quarter / (4 / rep);
    const int kk = (quarter % (4 / rep)) * 32 + lane;  // key of this lane within the tile
    const bool key_ok = __any_sync(0xffffffffu, kk < nk);  // warp-uniform: tcgen05.ld is .sync.aligned
    // this warp's query columns within each 128-query tile: [cb, cb + cn)
    const int cn = 64 / rep;
    const int cb = replica * (128 / rep) + half * cn;
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    const float c = p.scale_log2;
    constexpr float kL2E = 1.4426950408889634f;
    // stage head h's row LSEs (as -LSE*log2 e) into lse_s[h & 1]: each thread copies its own
    // entries, waits for them and transforms them; a barrier publishes them
    auto stage = [&](int h) {
      float* dst = lse_s + (h & 1) * nqp;
      for (int q = tid; q < nqp; q += 256) {
        if (q < Nc) cp_async4(dst + q, p.lse + (size_t)h * p.lse_ld + row0 + q);
        else dst[q] = 0.f;
      }
    };
    auto finish = [&](int h) {
      cp_async_wait_all();
      float* dst = lse_s + (h & 1) * nqp;
      for (int q = tid; q < Nc; q += 256) dst[q] = -dst[q] * kL2E;
    };
    stage(0);
    finish(0);
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    for (int it = 0; it < total; ++it) {
      const int h = it / nq, qt = it % nq;
      if (qt == 0) {
        named_bar_sync(1, 256);  // head h staged; every warp is done with head h-1's buffer
        if (h + 1 < p.n_heads) stage(h + 1);
      }
      if (qt == nq - 1 && h + 1 < p.n_heads) finish(h + 1);  // landed long ago; before the next barrier
      mbar_wait(&s_full[it & 1], (it >> 1) & 1);
      tc_fence_after();
      const int nv = min(cn, min(128, Nc - qt * 128) - cb);  // valid columns of this warp (may be <= 0)
      const float* nl = lse_s + (h & 1) * nqp + qt * 128 + cb;
      const uint32_t a = tmem + lane_off + (it & 1) * 128 + cb;
      if (key_ok && nv >= cn) {
        uint32_t sr[64];
        if (cn == 64) {
          tmem_ld32(a, *reinterpret_cast<uint32_t(*)[32]>(sr));
          tmem_ld32(a + 32, *reinterpret_cast<uint32_t(*)[32]>(sr + 32));
        } else if (cn == 32) {
          tmem_ld32(a, *reinterpret_cast<uint32_t(*)[32]>(sr));
        } else {
          tmem_ld16(a, *reinterpret_cast<uint32_t(*)[16]>(sr));
        }
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(&s_empty[it & 1]);
        score_exp16<SCORE_NPP / 2>(sr, nl, c, a0, a1);
        if (cn >= 32) score_exp16<SCORE_NPP / 2>(sr + 16, nl + 16, c, a2, a3);
        if (cn == 64) {
          score_exp16<SCORE_NPP / 2>(sr + 32, nl + 32, c, a0, a1);
          score_exp16<SCORE_NPP / 2>(sr + 48, nl + 48, c, a2, a3);
        }
      } else if (key_ok && nv > 0) {
        // ragged last query tile: 16-column chunks, masked within the last one
        const int nch = (nv + 15) / 16;
#pragma unroll 1
        for (int ch = 0; ch < nch; ++ch) {
          uint32_t sr[16];
          tmem_ld16(a + ch * 16, sr);
          tmem_wait_ld();
          if (ch == nch - 1) {
            tc_fence_before();
            mbar_arrive(&s_empty[it & 1]);
          }
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            if (ch * 16 + i < nv) {
              const float e = ex2_approx(fmaf(__uint_as_float(sr[i]), c, nl[ch * 16 + i]));
              if (i & 1) a1 += e; else a0 += e;
            }
          }
        }
      } else {
        tc_fence_before();
        mbar_arrive(&s_empty[it & 1]);
      }
    }
    part[(half * 4 + quarter) * 128 + quarter * 32 + lane] = (a0 + a1) + (a2 + a3);
    named_bar_sync(1, 256);
    // key kk of the tile: the partials of every (replica, half) holding it, in a fixed order
    if (tid < nk) {
      const int k = tid;
      float acc = 0.f;
      for (int rj = 0; rj < rep; ++rj) {
        const int q = rj * (4 / rep) + k / 32;  // lane quarter of replica rj holding key k
        acc += part[(0 * 4 + q) * 128 + q * 32 + (k & 31)];
        acc += part[(1 * 4 + q) * 128 + q * 32 + (k & 31)];
      }
      p.scores[(size_t)b * Nc + kt * 128 + k] = acc / (float)(p.n_heads * Nc);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<256>(tmem);
}

}  // namespace cfd
