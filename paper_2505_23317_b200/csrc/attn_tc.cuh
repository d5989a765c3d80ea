// attn_tc.cuh — fused varlen multi-head self-attention on tcgen05.
//
// "each patch attends to every other patch" within its own task:
// tasks of a patch-level batch are packed back to back and
// delimited by cu_seqlens, attention is block-diagonal (reading R11) — no padding.
//
// One CTA = (q-tile of 128 rows, head, task).  Per KV tile j (128 keys):
//   S_j   = Q K_j^T            tcgen05.mma SS, M=128 N=128 K=dh   -> TMEM (fp32)
//   P_j   = exp2(S_j*c - m_j)  softmax warps: one thread per query row
//                              (tcgen05.ld -> regs -> bf16 -> tcgen05.st to TMEM)
//   O_j   = P_j V_j            tcgen05.mma TS (A=P from TMEM, B=V MN-major smem)
//   o    <- o*alpha + O_j      in registers (online softmax rescale)
// S, P and O are double-buffered in TMEM (S0 S1 | P0 P1 | O0 O1 = 512 columns) so
// the tensor core computes S_{j+1} while the softmax warps process S_j.
//
// Warp roles (192 threads): warp 0 TMA, warp 1 TMEM alloc + MMA issue,
// warps 2..5 softmax / epilogue (warp w owns TMEM lanes 32*(w%4)..+31).
// qkv rows: [q(d) | k(d) | v(d)] bf16, head h at columns h*dh.  Output O bf16 [rows, d];
// optional LSE (natural log) [nh, lse_ld] for the criticality score.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "ptx.cuh"

namespace cfd {

struct AttnParams {
  const int* cu_seqlens;   // [T+1]
  int d_model;
  __nv_bfloat16* out;      // [rows, d_model]
  float* lse;              // [nh, lse_ld] or nullptr
  int lse_ld;
  float scale_log2;        // log2(e) / sqrt(dh)
  int stagger = 0;         // v4: softmax warpgroup w starts w * stagger cycles late (0 = off)
  int* work_counter = nullptr;  // v4: zeroed int; non-null -> items after the first are claimed
                                // dynamically (atomicAdd) instead of the static round-robin
  int n_q = 0;             // v1 CROSS: queries per task (one 128-row tile shared by every task)
  const int* kv_len = nullptr;  // v7: [T] valid keys per task (pad-to-max batch: keys >= kv_len[t]
                                // of the task's cu_seqlens span are masked); nullptr = all
  int producer_sleep = 256;     // v7: the producer warp's sleep between barrier probes, ns
};

constexpr int ATTN_THREADS = 192;
constexpr int ATTN_BQ = 128;
constexpr int ATTN_BKV = 128;

template <int DH, int STAGES>
struct AttnSmem {
  static constexpr int Q_BYTES = ATTN_BQ * DH * 2;
  static constexpr int K_BYTES = ATTN_BKV * DH * 2;
  static constexpr int V_BYTES = ATTN_BKV * DH * 2;
  static constexpr int TOTAL = 1024 + Q_BYTES + STAGES * (K_BYTES + V_BYTES) + 256;
  // TMEM column map
  static constexpr uint32_t S_COL = 0;                 // 2 x 128
  static constexpr uint32_t P_COL = 256;               // 2 x 64 (bf16 pairs)
  static constexpr uint32_t O_COL = 384;               // 2 x DH
  static constexpr uint32_t TMEM_COLS = 512;
};

// CROSS (NEXT f3, decoder cross-attention, reading R24): the query tile is the n_q <= 128
// learned object queries' projection (rows 0..n_q-1 of the q map, shared by every task),
// keys / values are task t's packed encoder tokens [cu[t], cu[t+1]) of the kv map ([k | v]
// columns), and the output goes to rows t * n_q + r.  Otherwise the self-attention path:
// q, k, v from one [q | k | v] map (tmKV == tmQ).
template <int DH, int STAGES, bool CROSS = false>
__global__ void __launch_bounds__(ATTN_THREADS, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmQKV, const AttnParams p,
                   const __grid_constant__ CUtensorMap tmKV) {
  static_assert(DH == 32, "this kernel is specialised for dh = 32 (64-byte rows, SW64)");
  using S = AttnSmem<DH, STAGES>;
  const int t = blockIdx.z, h = blockIdx.y, qt = blockIdx.x;
  const int seq0 = __ldg(p.cu_seqlens + t);
  const int N = __ldg(p.cu_seqlens + t + 1) - seq0;
  const int NQ = CROSS ? p.n_q : N;  // query rows of this task
  if (qt * ATTN_BQ >= NQ || N <= 0) return;  // CTA-uniform, before any barrier / TMEM use
  const int nkv = (N + ATTN_BKV - 1) / ATTN_BKV;
  const int q_row0 = CROSS ? 0 : seq0 + qt * ATTN_BQ;           // rows of the q map
  const int out_row0 = CROSS ? t * p.n_q : q_row0;              // rows of the output

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps the shared space
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + S::Q_BYTES;
  uint8_t* sV = sK + STAGES * S::K_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + STAGES * S::V_BYTES);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = kv_full + STAGES;
  uint64_t* s_full = kv_empty + STAGES;  // [2]
  uint64_t* s_empty = s_full + 2;        // [2]
  uint64_t* p_full = s_empty + 2;        // [2]
  uint64_t* o_full = p_full + 2;         // [2]
  uint64_t* o_empty = o_full + 2;        // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_empty + 2);

  const int warp = warp_id(), lane = lane_id();
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmQKV);
    mbar_init(q_full, 1);
    for (int s = 0; s < STAGES; ++s) { mbar_init(&kv_full[s], 1); mbar_init(&kv_empty[s], 1); }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&s_empty[b], 128);
      mbar_init(&p_full[b], 128);
      mbar_init(&o_full[b], 1);
      mbar_init(&o_empty[b], 128);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<S::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int col_q = h * DH, col_k = (CROSS ? 0 : p.d_model) + h * DH, col_v = (CROSS ? 1 : 2) * p.d_model + h * DH;
  const CUtensorMap* tkv = CROSS ? &tmKV : &tmQKV;

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch(tkv);
      mbar_expect_tx(q_full, S::Q_BYTES);
      tma_load_2d(sQ, &tmQKV, q_full, col_q, q_row0);
      int stage = 0;
      uint32_t phase = 0;
      for (int j = 0; j < nkv; ++j) {
        mbar_wait(&kv_empty[stage], phase ^ 1);
        mbar_expect_tx(&kv_full[stage], S::K_BYTES + S::V_BYTES);
        tma_load_2d(sK + stage * S::K_BYTES, tkv, &kv_full[stage], col_k, seq0 + j * ATTN_BKV);
        tma_load_2d(sV + stage * S::V_BYTES, tkv, &kv_full[stage], col_v, seq0 + j * ATTN_BKV);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = make_idesc_bf16(ATTN_BQ, ATTN_BKV, 0);  // S = Q K^T
      constexpr uint32_t idesc_o = make_idesc_bf16(ATTN_BQ, DH, 1);        // O = P V (V MN-major)
      mbar_wait(q_full, 0);
      const uint32_t q_addr = smem_u32(sQ);
      auto issue_s = [&](int j) {
        const int st = j % STAGES;
        mbar_wait(&kv_full[st], (j / STAGES) & 1);
        mbar_wait(&s_empty[j & 1], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sK + st * S::K_BYTES);
#pragma unroll
        for (int k = 0; k < DH / 16; ++k) {
          mma_ss(tmem + S::S_COL + (j & 1) * 128, make_smem_desc(q_addr + k * 32, 16, 512, kLayoutSW64),
                 make_smem_desc(k_addr + k * 32, 16, 512, kLayoutSW64), idesc_s, k);
        }
        mma_commit(&s_full[j & 1]);
      };
      auto issue_pv = [&](int j) {
        const int st = j % STAGES;
        mbar_wait(&p_full[j & 1], (j >> 1) & 1);
        mbar_wait(&o_empty[j & 1], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t v_addr = smem_u32(sV + st * S::V_BYTES);
#pragma unroll
        for (int k = 0; k < ATTN_BKV / 16; ++k) {
          mma_ts(tmem + S::O_COL + (j & 1) * DH, tmem + S::P_COL + (j & 1) * 64 + k * 8,
                 make_smem_desc(v_addr + k * 16 * DH * 2, 4096, 512, kLayoutSW64), idesc_o, k);
        }
        mma_commit(&o_full[j & 1]);
        mma_commit(&kv_empty[st]);
      };
      issue_s(0);
      for (int j = 0; j < nkv; ++j) {
        if (j + 1 < nkv) issue_s(j + 1);
        issue_pv(j);
      }
    }
  } else {
    // ------------------------------------------------------------ softmax warps
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;  // query row within the tile
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    const float c = p.scale_log2;
    float m_run = -INFINITY, l_run = 0.f, alpha_prev = 0.f;
    float o_acc[DH];
#pragma unroll
    for (int i = 0; i < DH; ++i) o_acc[i] = 0.f;

    auto absorb = [&](int j, float alpha) {
      mbar_wait(&o_full[j & 1], (j >> 1) & 1);
      tc_fence_after();
      uint32_t o[32];
      tmem_ld32(tmem + lane_off + S::O_COL + (j & 1) * DH, o);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(&o_empty[j & 1]);
#pragma unroll
      for (int i = 0; i < DH; ++i) o_acc[i] = o_acc[i] * alpha + __uint_as_float(o[i]);
    };

    for (int j = 0; j < nkv; ++j) {
      mbar_wait(&s_full[j & 1], (j >> 1) & 1);
      tc_fence_after();
      uint32_t sr[128];
      const uint32_t s_addr = tmem + lane_off + S::S_COL + (j & 1) * 128;
      tmem_ld32(s_addr + 0, *reinterpret_cast<uint32_t(*)[32]>(sr + 0));
      tmem_ld32(s_addr + 32, *reinterpret_cast<uint32_t(*)[32]>(sr + 32));
      tmem_ld32(s_addr + 64, *reinterpret_cast<uint32_t(*)[32]>(sr + 64));
      tmem_ld32(s_addr + 96, *reinterpret_cast<uint32_t(*)[32]>(sr + 96));
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(&s_empty[j & 1]);

      const int valid = N - j * ATTN_BKV;  // keys of this task in the tile
      float mx = -INFINITY;
#pragma unroll
      for (int i = 0; i < 128; ++i) {
        float s = (i < valid) ? __uint_as_float(sr[i]) : -INFINITY;
        sr[i] = __float_as_uint(s);
        mx = fmaxf(mx, s);
      }
      const float m_new = fmaxf(m_run, mx * c);
      const float alpha = (m_run == -INFINITY) ? 0.f : ex2_approx(m_run - m_new);
      float rs = 0.f;
      uint32_t pk[64];
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        const float p0 = ex2_approx(fmaf(__uint_as_float(sr[2 * i]), c, -m_new));
        const float p1 = ex2_approx(fmaf(__uint_as_float(sr[2 * i + 1]), c, -m_new));
        rs += p0 + p1;
        pk[i] = pack_bf16x2(p0, p1);
      }
      l_run = l_run * alpha + rs;
      m_run = m_new;
      const uint32_t p_addr = tmem + lane_off + S::P_COL + (j & 1) * 64;
#pragma unroll
      for (int q = 0; q < 4; ++q) tmem_st16(p_addr + q * 16, *reinterpret_cast<const uint32_t(*)[16]>(pk + q * 16));
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&p_full[j & 1]);
      if (j > 0) absorb(j - 1, alpha_prev);
      alpha_prev = alpha;
    }
    absorb(nkv - 1, alpha_prev);

    const int q_valid = NQ - qt * ATTN_BQ;
    if (r < q_valid) {
      const float inv = 1.f / l_run;
      uint32_t ob[DH / 2];
#pragma unroll
      for (int i = 0; i < DH / 2; ++i) ob[i] = pack_bf16x2(o_acc[2 * i] * inv, o_acc[2 * i + 1] * inv);
      uint4* dst = reinterpret_cast<uint4*>(p.out + (size_t)(out_row0 + r) * p.d_model + h * DH);
#pragma unroll
      for (int i = 0; i < DH / 8; ++i) dst[i] = make_uint4(ob[4 * i], ob[4 * i + 1], ob[4 * i + 2], ob[4 * i + 3]);
      if (p.lse) p.lse[(size_t)h * p.lse_ld + out_row0 + r] = (m_run + __log2f(l_run)) * 0.69314718055994531f;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<S::TMEM_COLS>(tmem);
}

}  // namespace cfd
