// attn4_tc.cuh — attention v4: persistent, 64-key softmax steps, per-warpgroup MMA issuers,
// lazy rescale, MUFU/polynomial exp2, THREE softmax warpgroups per CTA, so an item is (task,
// triple of 128-row query tiles, head) and every K/V tile the TMA warp streams serves three
// query tiles.
//
//   TMEM per warpgroup w (128 columns, 3 x 128 = 384 of 512):
//     S_w  64 fp32 cols  — single-buffered: the warpgroup moves S_u into registers at the
//                          start of sub-tile u and releases it (s_free), so QK_{u+1} still
//                          runs on the tensor core during the exponentials of S_u
//     P_w  32 cols (bf16 pairs), O_w 32 cols (accumulated, rescaled in place)
//   Warps: 0..11 softmax (3 x 4), 12..14 MMA issuers (one per warpgroup), 15 TMA; 512
//   threads, <= 128 registers per thread.  The warp scheduler prefers the highest eligible
//   warp id, so the (mostly sleeping) MMA and TMA warps get the issue slot as soon as their
//   barrier completes instead of queueing behind the softmax warps of their SMSP.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "ptx.cuh"
#include "attn_tc.cuh"
#include "attn_common.cuh"

namespace cfd {

// item -> (task, query triple, head).  Ragged batches: task-major (decode_item).  Equal
// lengths (the coarse pass): q-triple-major, so that with the static round-robin item
// assignment the costly full triples (384 rows) and the short tail triples (N = 400: 16
// rows) spread over the CTAs instead of pairing up (max per-CTA load 2 full + 2 tail -> 1 + 1).
__device__ __forceinline__ void decode_item4(const AttnParams& p, const int* prefix, int T, int nh, int item, int& t,
                                             int& qp, int& h) {
  if (p.uniform_n > 0) {
    const int per = T * nh;
    qp = item / per;
    const int r = item - qp * per;
    t = r / nh;
    h = r - t * nh;
  } else {
    decode_item(prefix, T, nh, item, t, qp, h);
  }
}

template <int DH, int STAGES>
struct Attn4Smem {
  static constexpr int TILE_BYTES = 128 * DH * 2;
  static constexpr int Q_OFF = 0;                              // [2 slots][3 tiles]
  static constexpr int K_OFF = Q_OFF + 6 * TILE_BYTES;         // [STAGES]
  static constexpr int V_OFF = K_OFF + STAGES * TILE_BYTES;    // [STAGES]
  static constexpr int BAR_OFF = V_OFF + STAGES * TILE_BYTES;
  static constexpr int PRE_OFF = BAR_OFF + 512;
  static constexpr int TOTAL = 1024 + PRE_OFF + (ATTN_MAX_T + 1) * 4;
  static constexpr uint32_t S_COL = 0;    // S_w at w*128
  static constexpr uint32_t P_COL = 64;   // P_w at w*128 + 64
  static constexpr uint32_t O_COL = 96;   // O_w at w*128 + 96
};

constexpr int ATTN4_THREADS = 512;    // TMA warp, 3 MMA warps, 12 softmax warps
constexpr int ATTN4_NWG = 3;

// TOKEN: the three warpgroups take turns on the exp (MUFU) phase — warpgroup w starts the
// exponentials of a sub-tile only after warpgroup w-1 finished its own (a token ring of
// mbarriers, one phase per sub-tile), so their exp phases are serialised and each one's
// latency-bound phases (TMEM load, max, P store, hand-offs) overlap the others' exps.
// SPLIT: break the MMAs' accumulator dependency chains (a dependent tcgen05.mma at these
// shapes costs ~150 cycles of latency, tools/tc_micro.cu): QK as two independent N = 32
// halves (keys 0-31 / 32-63 of the sub-tile, each a K-chain of 2) and PV into two O
// accumulators (keys 0-31 -> O_a, 32-63 -> O_b, each a chain of 2), O = O_a + O_b at the end.
// TMEM per warpgroup: S 64 | P 32 | O_a 32 | O_b 32 at w*160.
template <int DH, int STAGES, int NPP, bool TOKEN = false, bool SPLIT = false>
__global__ void __launch_bounds__(ATTN4_THREADS, 1)
    attn4_tc_kernel(const __grid_constant__ CUtensorMap tmQKV, const AttnParams p, const int T, const int nh) {
  static_assert(DH == 32, "specialised for dh = 32 (64-byte rows, SW64)");
  using S = Attn4Smem<DH, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps the shared space
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::BAR_OFF);
  uint64_t* q_full = bars;                  // [2]
  uint64_t* q_empty = bars + 2;             // [2]
  uint64_t* kv_full = bars + 4;             // [STAGES]
  uint64_t* kv_empty = kv_full + STAGES;    // [STAGES]
  uint64_t* s_full = kv_empty + STAGES;     // [3 w]
  uint64_t* s_free = s_full + 3;            // [3 w]
  uint64_t* p_full = s_free + 3;            // [3 w]
  uint64_t* o_full = p_full + 3;            // [3 w]
  uint64_t* exp_tok = o_full + 3;           // [3 w] TOKEN: warpgroup w finished its exps
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(exp_tok + 3);
  volatile int* item_slot = reinterpret_cast<volatile int*>(smem + S::BAR_OFF + 448);  // [2] item of a Q slot
  int* prefix = reinterpret_cast<int*>(smem + S::PRE_OFF);

  const int warp = warp_id(), lane = lane_id();
#ifdef CFD_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 148) g_attn_trace[ATTN_TRACE_T0 + blockIdx.x] = clock64();
#endif
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    const int n = __ldg(p.cu_seqlens + t + 1) - __ldg(p.cu_seqlens + t);
    prefix[t + 1] = ((n + 383) / 384) * nh;
  }
  constexpr int kMmaWarp0 = 12, kTmaWarp = 15;
  constexpr uint32_t WST = SPLIT ? 160 : 128;  // TMEM columns per warpgroup
  if (warp == kTmaWarp && lane == 0) {
    tma_prefetch(&tmQKV);
    // Q slots and K/V stages are released by all three MMA threads (one per warpgroup)
    for (int i = 0; i < 2; ++i) { mbar_init(&q_full[i], 1); mbar_init(&q_empty[i], ATTN4_NWG); }
    for (int s = 0; s < STAGES; ++s) { mbar_init(&kv_full[s], 1); mbar_init(&kv_empty[s], ATTN4_NWG); }
    for (int w = 0; w < ATTN4_NWG; ++w) {
      mbar_init(&s_full[w], 1);
      mbar_init(&s_free[w], 128);
      mbar_init(&p_full[w], 128);
      mbar_init(&o_full[w], 1);
      mbar_init(&exp_tok[w], 4);  // one arrival per warp of the warpgroup
    }
    fence_barrier_init();
  }
  if (warp == kMmaWarp0) tmem_alloc<512>(tmem_slot);
  __syncthreads();
  if (warp == 0) {  // inclusive scan of prefix[1..T], prefix[0] = 0
    int run = 0;
    for (int c0 = 0; c0 < T; c0 += 32) {
      const int i = c0 + lane;
      int v = (i < T) ? prefix[i + 1] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      if (i < T) prefix[i + 1] = run + v;
      run += __shfl_sync(0xffffffffu, v, 31);
    }
    if (lane == 0) prefix[0] = 0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int total = prefix[T];
  const int d = p.d_model;

  if (warp == kTmaWarp) {
    // ================================================================ TMA producer
    if (lane == 0) {
      // Items: the first is blockIdx.x; later ones are claimed from p.work_counter (dynamic:
      // the longest-running CTAs take fewer items) or round-robin.  The item index travels
      // to the MMA and softmax warps in item_slot[Q slot], published by the q_full arrive; an
      // index >= total (arrive without TMA bytes) tells them to stop.
      int kvc = 0;
      for (int it = 0;; ++it) {
        const int item = (it == 0 || !p.work_counter) ? (int)blockIdx.x + it * (int)gridDim.x
                                                      : (int)gridDim.x + atomicAdd(p.work_counter, 1);
        const int slot = it & 1;
        mbar_wait(&q_empty[slot], ((it >> 1) & 1) ^ 1);
        item_slot[slot] = item;
        if (item >= total) {
          mbar_arrive(&q_full[slot]);
          if (p.work_counter) {
            // self-resetting claim counter: the last CTA to make its final claim zeroes
            // [claims, finished] for the next launch on this stream (no memset launch)
            __threadfence();
            if (atomicAdd(p.work_counter + 1, 1) == (int)gridDim.x - 1) {
              p.work_counter[0] = 0;
              p.work_counter[1] = 0;
              __threadfence();
            }
          }
          break;
        }
        int t, qp, h;
        decode_item4(p, prefix, T, nh, item, t, qp, h);
        const int seq0 = __ldg(p.cu_seqlens + t);
        const int N = __ldg(p.cu_seqlens + t + 1) - seq0;
        const int nq = min(ATTN4_NWG, (N - 3 * qp * 128 + 127) / 128);
        const int nkv = (N + 127) / 128;
        mbar_expect_tx(&q_full[slot], nq * S::TILE_BYTES);
        for (int w = 0; w < nq; ++w)
          tma_load_2d(smem + S::Q_OFF + (slot * 3 + w) * S::TILE_BYTES, &tmQKV, &q_full[slot], h * DH,
                      seq0 + (3 * qp + w) * 128);
        for (int j = 0; j < nkv; ++j, ++kvc) {
          const int st = kvc % STAGES;
          mbar_wait(&kv_empty[st], ((kvc / STAGES) & 1) ^ 1);
          mbar_expect_tx(&kv_full[st], 2 * S::TILE_BYTES);
          tma_load_2d(smem + S::K_OFF + st * S::TILE_BYTES, &tmQKV, &kv_full[st], d + h * DH, seq0 + j * 128);
          tma_load_2d(smem + S::V_OFF + st * S::TILE_BYTES, &tmQKV, &kv_full[st], 2 * d + h * DH, seq0 + j * 128);
        }
      }
    }
  } else if (warp >= kMmaWarp0 && warp < kMmaWarp0 + ATTN4_NWG) {
    // ================================================================ MMA issuers
    // warp 12 + w issues for warpgroup w: each warpgroup's S/P/O pipeline advances
    // independently (tcgen05.commit tracks the issuing thread's MMAs).  A K/V stage or Q
    // slot is released once all three issuers are done with it.
    if (lane == 0) {
      const int w = warp - kMmaWarp0;
      constexpr uint32_t idesc_s = make_idesc_bf16(128, 64, 0);  // S_u = Q K_u^T (64 keys)
      constexpr uint32_t idesc_o = make_idesc_bf16(128, DH, 1);  // O += P_u V_u (V MN-major)
      int kvc = 0;
      uint32_t p_cnt = 0;
      uint32_t s_use = 0;   // QKs issued into S_w
      for (int it = 0;; ++it) {
        const int slot = it & 1;
        mbar_wait(&q_full[slot], (it >> 1) & 1);
        const int item = item_slot[slot];
        if (item >= total) break;
        int t, qp, h;
        decode_item4(p, prefix, T, nh, item, t, qp, h);
        const int seq0 = __ldg(p.cu_seqlens + t);
        const int N = __ldg(p.cu_seqlens + t + 1) - seq0;
        const int nkv = (N + 127) / 128;
        if ((3 * qp + w) * 128 >= N) {
          // no query tile for this warpgroup: release the item's stages in step
          for (int j = 0; j < nkv; ++j) {
            const int st = (kvc + j) % STAGES;
            mbar_wait(&kv_full[st], ((kvc + j) / STAGES) & 1);
            mbar_arrive(&kv_empty[st]);
          }
          kvc += nkv;
          mbar_arrive(&q_empty[slot]);
          continue;
        }
        const int nsub = (N + 63) / 64;
        const uint32_t qa = smem_u32(smem + S::Q_OFF + (slot * 3 + w) * S::TILE_BYTES);
        auto issue_qk = [&](int u) {
          const int j = u >> 1;
          const int st = (kvc + j) % STAGES;
          if ((u & 1) == 0) mbar_wait(&kv_full[st], ((kvc + j) / STAGES) & 1);
          const uint32_t ka = smem_u32(smem + S::K_OFF + st * S::TILE_BYTES) + (u & 1) * 64 * DH * 2;
          if (s_use > 0) mbar_wait(&s_free[w], (s_use - 1) & 1);
          if (p.stagger == -2 && u > 0) ATTN_TR(w, it, u - 1, 5);  // (in sub-tile u-1's row) s_free passed
          ++s_use;
          tc_fence_after();
          if constexpr (SPLIT) {
            constexpr uint32_t idesc_h = make_idesc_bf16(128, 32, 0);
#pragma unroll
            for (int k = 0; k < DH / 16; ++k)
#pragma unroll
              for (int hh = 0; hh < 2; ++hh)  // keys [32 hh, 32 hh + 32): rows 32 hh of the K tile
                mma_ss(tmem + w * WST + S::S_COL + hh * 32, make_smem_desc(qa + k * 32, 16, 512, kLayoutSW64),
                       make_smem_desc(ka + hh * 32 * DH * 2 + k * 32, 16, 512, kLayoutSW64), idesc_h, k);
          } else {
#pragma unroll
            for (int k = 0; k < DH / 16; ++k)
              mma_ss(tmem + w * WST + S::S_COL, make_smem_desc(qa + k * 32, 16, 512, kLayoutSW64),
                     make_smem_desc(ka + k * 32, 16, 512, kLayoutSW64), idesc_s, k);
          }
          mma_commit(&s_full[w]);
          ATTN_TR(w, it, u, 6);
        };
        // trace mode "mma" (p.stagger == -2): events 0..5 of the MMA warp's sub-tile u
        const bool tm = p.stagger == -2;
        issue_qk(0);
        for (int u = 0; u < nsub; ++u) {
          if (tm) ATTN_TR(w, it, u, 0);
          if (u + 1 < nsub) issue_qk(u + 1);  // S_{u+1} overlaps the softmax of S_u
          if (tm) ATTN_TR(w, it, u, 1);
          const int j = u >> 1;
          const int st = (kvc + j) % STAGES;
          const int valid = min(64, N - u * 64);
          const int ksteps = (valid + 15) / 16;
          const uint32_t va = smem_u32(smem + S::V_OFF + st * S::TILE_BYTES) + (u & 1) * 64 * DH * 2;
          mbar_wait(&p_full[w], p_cnt & 1);
          if (tm) ATTN_TR(w, it, u, 2);
          ++p_cnt;
          tc_fence_after();
          if constexpr (SPLIT) {
            // O_a <- keys 0-31 (k-steps 0, 1), O_b <- keys 32-63 (k-steps 2, 3), interleaved
#pragma unroll
            for (int kk = 0; kk < 2; ++kk)
#pragma unroll
              for (int hh = 0; hh < 2; ++hh) {
                const int k = hh * 2 + kk;
                if (k < ksteps)
                  mma_ts(tmem + w * WST + S::O_COL + hh * 32, tmem + w * WST + S::P_COL + k * 8,
                         make_smem_desc(va + k * 16 * DH * 2, 4096, 512, kLayoutSW64), idesc_o, (u | kk) != 0);
              }
          } else {
            for (int k = 0; k < ksteps; ++k)
              mma_ts(tmem + w * WST + S::O_COL, tmem + w * WST + S::P_COL + k * 8,
                     make_smem_desc(va + k * 16 * DH * 2, 4096, 512, kLayoutSW64), idesc_o, (u | k) != 0);
          }
          if (tm) ATTN_TR(w, it, u, 3);
          mma_commit(&o_full[w]);
          if (tm) ATTN_TR(w, it, u, 4);
          ATTN_TR(w, it, u, 7);
          if ((u & 1) || u + 1 == nsub) mma_commit(&kv_empty[st]);
        }
        kvc += nkv;
        mma_commit(&q_empty[slot]);
      }
    }
  } else {
    // ================================================================ softmax warpgroups (warps 0..11)
    const int wg = warp >> 2;
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    const uint32_t s_base = tmem + lane_off + wg * WST + S::S_COL;
    const uint32_t p_addr = tmem + lane_off + wg * WST + S::P_COL;
    const uint32_t o_addr = tmem + lane_off + wg * WST + S::O_COL;  // SPLIT: O_a, O_b at +32
    const float c = p.scale_log2;
    uint32_t s_cnt = 0, o_cnt = 0;
    uint32_t g_tok = 0;  // TOKEN: sub-tiles (exp turns) of this warpgroup so far
    const int prev_wg = (wg + ATTN4_NWG - 1) % ATTN4_NWG;
    // wait for the previous warpgroup's turn g (warpgroup 0: the last warpgroup's turn g-1)
    auto tok_wait = [&]() {
      if constexpr (TOKEN) {
        if (wg == 0) {
          if (g_tok > 0) mbar_wait(&exp_tok[prev_wg], (g_tok - 1) & 1);
        } else {
          mbar_wait(&exp_tok[prev_wg], g_tok & 1);
        }
      }
    };
    auto tok_pass = [&]() {
      if constexpr (TOKEN) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&exp_tok[wg]);
        ++g_tok;
      }
    };
    // trace: lane 0 of the quarter-0 warp; with p.stagger == -1 (trace mode "quarters") events
    // 0..2 instead record the p_full arrival of the quarter 1..3 warps
    const bool qmode = p.stagger == -1;
    const bool tr = (warp & 3) == 0 && lane == 0 && !qmode && p.stagger != -2;
    const bool trq = lane == 0 && qmode;
    (void)tr;
    (void)trq;
    if (p.stagger > 0 && wg > 0) {  // de-phase the warpgroups so their exp phases interleave
      const long long t_end = clock64() + (long long)wg * p.stagger;
      while (clock64() < t_end) __nanosleep(64);
    }
    int it = -1;
    for (;;) {
      ++it;
      // the item of this Q slot (q_full publishes it; the Q tiles themselves are read by the
      // MMA warps only)
      mbar_wait(&q_full[it & 1], (it >> 1) & 1);
      const int item = item_slot[it & 1];
      if (item >= total) break;
      int t, qp, h;
      decode_item4(p, prefix, T, nh, item, t, qp, h);
      const int seq0 = __ldg(p.cu_seqlens + t);
      const int N = __ldg(p.cu_seqlens + t + 1) - seq0;
      const int qt = 3 * qp + wg;
      const int nsub = (N + 63) / 64;
      if (qt * 128 >= N) {
        if constexpr (TOKEN) {  // no query tile here: still take (and pass) every turn
          for (int u = 0; u < nsub; ++u) {
            tok_wait();
            tok_pass();
          }
        }
        continue;
      }
      const int q_valid = N - qt * 128;
      const bool active = quarter * 32 < q_valid;
      float m_run = -INFINITY, l_run = 0.f;
      for (int u = 0; u < nsub; ++u) {
        mbar_wait(&s_full[wg], s_cnt & 1);
        ++s_cnt;
        tc_fence_after();
        if (tr) ATTN_TR(wg, it, u, 0);
        if (active) {
          const int valid = min(64, N - u * 64);
          uint32_t sr[64];
          tmem_ld32(s_base, *reinterpret_cast<uint32_t(*)[32]>(sr));
          if (valid > 32) tmem_ld32(s_base + 32, *reinterpret_cast<uint32_t(*)[32]>(sr + 32));
          tmem_wait_ld();
          if (tr) ATTN_TR(wg, it, u, 1);
          tc_fence_before();
          mbar_arrive(&s_free[wg]);  // S_w may now be overwritten by QK_{u+1}
          if (valid < 64) {
#pragma unroll
            for (int i = 0; i < 64; ++i)
              if (i >= valid) sr[i] = __float_as_uint(-INFINITY);
          }
          float m0 = -INFINITY, m1 = -INFINITY, m2 = -INFINITY, m3 = -INFINITY;  // 4 independent chains
#pragma unroll
          for (int i = 0; i < 64; i += 8) {
            m0 = fmax3(m0, __uint_as_float(sr[i]), __uint_as_float(sr[i + 1]));
            m1 = fmax3(m1, __uint_as_float(sr[i + 2]), __uint_as_float(sr[i + 3]));
            m2 = fmax3(m2, __uint_as_float(sr[i + 4]), __uint_as_float(sr[i + 5]));
            m3 = fmax3(m3, __uint_as_float(sr[i + 6]), __uint_as_float(sr[i + 7]));
          }
          const float m_cand = fmax3(m0, m1, fmaxf(m2, m3)) * c;
          if (tr) ATTN_TR(wg, it, u, 2);
          const bool upd = (m_run == -INFINITY) || (m_cand > m_run + 8.0f);
          const float alpha = upd ? ((m_run == -INFINITY) ? 0.f : ex2_approx(m_run - m_cand)) : 1.f;
          if (upd) m_run = m_cand;
          const float neg = -m_run;
          float sum0 = 0.f, sum1 = 0.f, sum2 = 0.f, sum3 = 0.f;
          tok_wait();
          if (valid == 64) {
            exp_chunk<NPP>(sr, c, neg, sum0, sum1);
            exp_chunk<NPP>(sr + 32, c, neg, sum2, sum3);
          } else {
            exp_chunk<0>(sr, c, neg, sum0, sum1);
            if (valid > 32) exp_chunk<0>(sr + 32, c, neg, sum2, sum3);
          }
          tok_pass();
          l_run = l_run * alpha + ((sum0 + sum1) + (sum2 + sum3));
          if (tr) ATTN_TR(wg, it, u, 3);
          if (u > 0) {
            // PV_{u-1} done: P_w may be overwritten and O_w rescaled
            mbar_wait(&o_full[wg], o_cnt & 1);
            ++o_cnt;
            tc_fence_after();
            if (__any_sync(0xffffffffu, upd)) {
#pragma unroll 1
              for (int hh = 0; hh < (SPLIT && N > 32 ? 2 : 1); ++hh) {  // O_b exists once N > 32
                uint32_t o[32];
                tmem_ld32(o_addr + hh * 32, o);
                tmem_wait_ld();
#pragma unroll
                for (int i = 0; i < DH; i += 2) {
                  float a0, a1;
                  fma2(a0, a1, __uint_as_float(o[i]), __uint_as_float(o[i + 1]), alpha, alpha, 0.f, 0.f);
                  o[i] = __float_as_uint(a0);
                  o[i + 1] = __float_as_uint(a1);
                }
                tmem_st16(o_addr + hh * 32, *reinterpret_cast<const uint32_t(*)[16]>(o));
                tmem_st16(o_addr + hh * 32 + 16, *reinterpret_cast<const uint32_t(*)[16]>(o + 16));
              }
            }
          }
          if (tr) ATTN_TR(wg, it, u, 4);
          tmem_st16(p_addr, *reinterpret_cast<const uint32_t(*)[16]>(sr));
          if (valid > 32) tmem_st16(p_addr + 16, *reinterpret_cast<const uint32_t(*)[16]>(sr + 32));
          tmem_wait_st();
        } else {
          // padding-only warp: still waits for PV_{u-1} so it cannot arrive on p_full for
          // sub-tile u before that barrier's previous phase (sub-tile u-1) has completed
          mbar_arrive(&s_free[wg]);
          tok_wait();
          tok_pass();
          if (u > 0) {
            mbar_wait(&o_full[wg], o_cnt & 1);
            ++o_cnt;
          }
        }
        tc_fence_before();
        mbar_arrive(&p_full[wg]);
        if (tr) ATTN_TR(wg, it, u, 5);
        if (trq) ATTN_TR(wg, it, u, (warp & 3) == 0 ? 5 : (warp & 3) - 1);
      }
      if (active) {
        mbar_wait(&o_full[wg], o_cnt & 1);
        ++o_cnt;
        tc_fence_after();
        uint32_t o[32];
        tmem_ld32(o_addr, o);
        tmem_wait_ld();
        if constexpr (SPLIT) {
          if (N > 32) {  // O = O_a + O_b
            uint32_t o2[32];
            tmem_ld32(o_addr + 32, o2);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < DH; i += 2) {
              float a0, a1;
              add2(a0, a1, __uint_as_float(o[i]), __uint_as_float(o[i + 1]), __uint_as_float(o2[i]),
                   __uint_as_float(o2[i + 1]));
              o[i] = __float_as_uint(a0);
              o[i + 1] = __float_as_uint(a1);
            }
          }
        }
        if (r < q_valid) {
          const float inv = 1.f / l_run;
          uint32_t ob[DH / 2];
#pragma unroll
          for (int i = 0; i < DH / 2; ++i)
            ob[i] = pack_bf16x2(__uint_as_float(o[2 * i]) * inv, __uint_as_float(o[2 * i + 1]) * inv);
          const int row = seq0 + qt * 128 + r;
          uint4* dst = reinterpret_cast<uint4*>(p.out + (size_t)row * d + h * DH);
#pragma unroll
          for (int i = 0; i < DH / 8; ++i) dst[i] = make_uint4(ob[4 * i], ob[4 * i + 1], ob[4 * i + 2], ob[4 * i + 3]);
          if (p.lse) p.lse[(size_t)h * p.lse_ld + row] = (m_run + __log2f(l_run)) * 0.69314718055994531f;
        }
        tc_fence_before();
      } else {
        mbar_wait(&o_full[wg], o_cnt & 1);
        ++o_cnt;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == kMmaWarp0) tmem_dealloc<512>(tmem);
}

}  // namespace cfd
