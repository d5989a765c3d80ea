// attn6_tc.cuh — attention v6 = v4 (persistent, three softmax warpgroups sharing one K/V
// stream, one MMA warp per warpgroup, 64-key sub-tiles, lazy rescale, MUFU/polynomial exp2)
// with the row max taken OFF the critical path:
//
//   * S is double-buffered in TMEM (S0/S1, 64 columns each) and P(u) is written over the
//     first 32 columns of S(u)'s buffer (bf16 pairs), so QK(u+2) reuses the buffer after
//     PV(u) (same issuing thread, executed in order) and no "S consumed" hand-off exists;
//   * for sub-tiles u >= 1 the exponentials use the running max m of the earlier sub-tiles
//     and the tile max is computed in the same pass (ALU pipe, interleaved with the MUFU
//     work) instead of in a dependent phase before it.  If the tile max exceeds m by more
//     than 2^8 the reference moves after the tile (O and l rescaled once PV(u) has
//     accumulated, R23); if it exceeds m by more than 2^64 (P could overflow) the sub-tile is
//     recomputed from the still-resident S with the new max before P is stored.
//
//   TMEM per warpgroup w (160 columns at w*160, 3 x 160 = 480 of 512):
//     S0 64 | S1 64 | O 32 (fp32)      P(u) aliases S[u&1] columns 0..31
//   Warps: 0..11 softmax (3 x 4), 12..14 MMA issuers, 15 TMA; 512 threads, <= 128 registers.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "ptx.cuh"
#include "attn_tc.cuh"
#include "attn2_tc.cuh"
#include "attn3_tc.cuh"
#include "attn4_tc.cuh"

namespace cfd {

template <int DH, int STAGES, int NPP>
__global__ void __launch_bounds__(ATTN4_THREADS, 1)
    attn6_tc_kernel(const __grid_constant__ CUtensorMap tmQKV, const AttnParams p, const int T, const int nh) {
  static_assert(DH == 32, "specialised for dh = 32 (64-byte rows, SW64)");
  using S = Attn4Smem<DH, STAGES>;  // same shared-memory layout as v4
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps the shared space
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::BAR_OFF);
  uint64_t* q_full = bars;                  // [2]
  uint64_t* q_empty = bars + 2;             // [2]
  uint64_t* kv_full = bars + 4;             // [STAGES]
  uint64_t* kv_empty = kv_full + STAGES;    // [STAGES]
  uint64_t* s_full = kv_empty + STAGES;     // [3 w][2 buffers]
  uint64_t* p_full = s_full + 6;            // [3 w]
  uint64_t* o_full = p_full + 3;            // [3 w]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_full + 3);
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
  if (warp == kTmaWarp && lane == 0) {
    tma_prefetch(&tmQKV);
    // Q slots and K/V stages are released by all three MMA threads (one per warpgroup)
    for (int i = 0; i < 2; ++i) { mbar_init(&q_full[i], 1); mbar_init(&q_empty[i], ATTN4_NWG); }
    for (int s = 0; s < STAGES; ++s) { mbar_init(&kv_full[s], 1); mbar_init(&kv_empty[s], ATTN4_NWG); }
    for (int w = 0; w < ATTN4_NWG; ++w) {
      mbar_init(&s_full[2 * w], 1);
      mbar_init(&s_full[2 * w + 1], 1);
      mbar_init(&p_full[w], 128);
      mbar_init(&o_full[w], 1);
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
      int it = 0, kvc = 0;
      for (int item = blockIdx.x; item < total; item += gridDim.x, ++it) {
        int t, qp, h;
        decode_item(prefix, T, nh, item, t, qp, h);
        const int seq0 = __ldg(p.cu_seqlens + t);
        const int N = __ldg(p.cu_seqlens + t + 1) - seq0;
        const int nq = min(ATTN4_NWG, (N - 3 * qp * 128 + 127) / 128);
        const int nkv = (N + 127) / 128;
        const int slot = it & 1;
        mbar_wait(&q_empty[slot], ((it >> 1) & 1) ^ 1);
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
      int it = 0, kvc = 0;
      uint32_t p_cnt = 0;
      int g0 = 0;           // sub-tiles of this warpgroup before the current item
      for (int item = blockIdx.x; item < total; item += gridDim.x, ++it) {
        int t, qp, h;
        decode_item(prefix, T, nh, item, t, qp, h);
        const int seq0 = __ldg(p.cu_seqlens + t);
        const int N = __ldg(p.cu_seqlens + t + 1) - seq0;
        const int nkv = (N + 127) / 128;
        const int slot = it & 1;
        mbar_wait(&q_full[slot], (it >> 1) & 1);
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
        const uint32_t wbase = tmem + w * 160;
        // sub-tile u uses S buffer (g0 + u) & 1; QK(u+2) reuses it after PV(u) (in order)
        auto issue_qk = [&](int u) {
          const int j = u >> 1;
          const int st = (kvc + j) % STAGES;
          if ((u & 1) == 0) mbar_wait(&kv_full[st], ((kvc + j) / STAGES) & 1);
          const uint32_t ka = smem_u32(smem + S::K_OFF + st * S::TILE_BYTES) + (u & 1) * 64 * DH * 2;
          const int b = (g0 + u) & 1;
          tc_fence_after();
#pragma unroll
          for (int k = 0; k < DH / 16; ++k)
            mma_ss(wbase + b * 64, make_smem_desc(qa + k * 32, 16, 512, kLayoutSW64),
                   make_smem_desc(ka + k * 32, 16, 512, kLayoutSW64), idesc_s, k);
          mma_commit(&s_full[2 * w + b]);
          ATTN_TR(w, it, u, 6);
        };
        issue_qk(0);
        if (nsub > 1) issue_qk(1);
        for (int u = 0; u < nsub; ++u) {
          const int j = u >> 1;
          const int st = (kvc + j) % STAGES;
          const int valid = min(64, N - u * 64);
          const int ksteps = (valid + 15) / 16;
          const uint32_t va = smem_u32(smem + S::V_OFF + st * S::TILE_BYTES) + (u & 1) * 64 * DH * 2;
          const uint32_t pcol = wbase + ((g0 + u) & 1) * 64;  // P(u) over S(u)'s first 32 columns
          mbar_wait(&p_full[w], p_cnt & 1);
          ++p_cnt;
          tc_fence_after();
          for (int k = 0; k < ksteps; ++k)
            mma_ts(wbase + 128, pcol + k * 8, make_smem_desc(va + k * 16 * DH * 2, 4096, 512, kLayoutSW64), idesc_o,
                   (u | k) != 0);
          mma_commit(&o_full[w]);
          ATTN_TR(w, it, u, 7);
          if ((u & 1) || u + 1 == nsub) mma_commit(&kv_empty[st]);
          if (u + 2 < nsub) issue_qk(u + 2);  // after PV(u): same thread, executed in order
        }
        g0 += nsub;
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
    const uint32_t wbase = tmem + lane_off + wg * 160;
    const uint32_t o_addr = wbase + 128;
    const float c = p.scale_log2;
    uint32_t o_cnt = 0;
    int g = 0;  // sub-tiles of this warpgroup so far (S buffer g & 1, s_full phase g >> 1)
    const bool tr = (warp & 3) == 0 && lane == 0;
    (void)tr;
    int it = -1;
    float resc = 1.f;  // O rescale still owed for the last sub-tile (applied after its PV)
    for (int item = blockIdx.x; item < total; item += gridDim.x) {
      ++it;
      int t, qp, h;
      decode_item(prefix, T, nh, item, t, qp, h);
      const int seq0 = __ldg(p.cu_seqlens + t);
      const int N = __ldg(p.cu_seqlens + t + 1) - seq0;
      const int qt = 3 * qp + wg;
      if (qt * 128 >= N) continue;
      const int nsub = (N + 63) / 64;
      const int q_valid = N - qt * 128;
      const bool active = quarter * 32 < q_valid;
      float m_run = -INFINITY, l_run = 0.f;
      resc = 1.f;
      for (int u = 0; u < nsub; ++u, ++g) {
        const int b = g & 1;
        const uint32_t s_addr = wbase + b * 64;
        mbar_wait(&s_full[2 * wg + b], (g >> 1) & 1);
        tc_fence_after();
        if (tr) ATTN_TR(wg, it, u, 0);
        if (active) {
          const int valid = min(64, N - u * 64);
          uint32_t sr[64];
          auto load_s = [&]() {
            tmem_ld32(s_addr, *reinterpret_cast<uint32_t(*)[32]>(sr));
            if (valid > 32) tmem_ld32(s_addr + 32, *reinterpret_cast<uint32_t(*)[32]>(sr + 32));
            tmem_wait_ld();
            if (valid < 64) {
#pragma unroll
              for (int i = 0; i < 64; ++i)
                if (i >= valid) sr[i] = __float_as_uint(-INFINITY);
            }
          };
          load_s();
          if (tr) ATTN_TR(wg, it, u, 1);
          float sum0 = 0.f, sum1 = 0.f, sum2 = 0.f, sum3 = 0.f;
          auto exps = [&](float neg) {
            sum0 = sum1 = sum2 = sum3 = 0.f;
            if (valid == 64) {
              exp_chunk<NPP>(sr, c, neg, sum0, sum1);
              exp_chunk<NPP>(sr + 32, c, neg, sum2, sum3);
            } else {
              exp_chunk<0>(sr, c, neg, sum0, sum1);
              if (valid > 32) exp_chunk<0>(sr + 32, c, neg, sum2, sum3);
            }
          };
          float alpha = 1.f;   // rescale of O / l owed before PV(u) (first tile, or a recompute)
          float m_cand;
          if (m_run == -INFINITY) {
            // first sub-tile: the max first, then the exponentials
            float m0 = -INFINITY, m1 = -INFINITY, m2 = -INFINITY, m3 = -INFINITY;
#pragma unroll
            for (int i = 0; i < 64; i += 8) {
              m0 = fmax3(m0, __uint_as_float(sr[i]), __uint_as_float(sr[i + 1]));
              m1 = fmax3(m1, __uint_as_float(sr[i + 2]), __uint_as_float(sr[i + 3]));
              m2 = fmax3(m2, __uint_as_float(sr[i + 4]), __uint_as_float(sr[i + 5]));
              m3 = fmax3(m3, __uint_as_float(sr[i + 6]), __uint_as_float(sr[i + 7]));
            }
            m_run = fmax3(m0, m1, fmaxf(m2, m3)) * c;
            m_cand = m_run;
            exps(-m_run);
          } else {
            // exponentials against the running max, tile max in the same pass
            float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
            for (int i = 0; i < 64; i += 4) {  // raw S maxima, read before exp_chunk packs over them
              mx0 = fmax3(mx0, __uint_as_float(sr[i]), __uint_as_float(sr[i + 1]));
              mx1 = fmax3(mx1, __uint_as_float(sr[i + 2]), __uint_as_float(sr[i + 3]));
            }
            exps(-m_run);
            m_cand = fmaxf(mx0, mx1) * c;
            const bool redo = m_cand > m_run + 64.0f;  // P may have overflowed: recompute
            if (__any_sync(0xffffffffu, redo)) {
              load_s();  // S(u) is still in TMEM (P overwrites it only below)
              if (redo) {
                alpha = ex2_approx(m_run - m_cand);
                m_run = m_cand;
              }
              exps(-m_run);
            }
          }
          if (tr) ATTN_TR(wg, it, u, 2);
          l_run = l_run * alpha + ((sum0 + sum1) + (sum2 + sum3));
          if (tr) ATTN_TR(wg, it, u, 3);
          const float o_fac = resc * alpha;  // O: owed rescale of the previous tile x this tile's
          resc = 1.f;
          if (m_cand > m_run + 8.0f) {  // lazy rescale (R23): new reference after this tile
            resc = ex2_approx(m_run - m_cand);
            l_run *= resc;
            m_run = m_cand;
          }
          if (u > 0) {
            // PV(u-1) done: O rescaled before PV(u) accumulates into it
            mbar_wait(&o_full[wg], o_cnt & 1);
            ++o_cnt;
            tc_fence_after();
            if (__any_sync(0xffffffffu, o_fac != 1.f)) {
              uint32_t o[32];
              tmem_ld32(o_addr, o);
              tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < DH; i += 2) {
                float a0, a1;
                fma2(a0, a1, __uint_as_float(o[i]), __uint_as_float(o[i + 1]), o_fac, o_fac, 0.f, 0.f);
                o[i] = __float_as_uint(a0);
                o[i + 1] = __float_as_uint(a1);
              }
              tmem_st16(o_addr, *reinterpret_cast<const uint32_t(*)[16]>(o));
              tmem_st16(o_addr + 16, *reinterpret_cast<const uint32_t(*)[16]>(o + 16));
            }
          }
          if (tr) ATTN_TR(wg, it, u, 4);
          tmem_st16(s_addr, *reinterpret_cast<const uint32_t(*)[16]>(sr));
          if (valid > 32) tmem_st16(s_addr + 16, *reinterpret_cast<const uint32_t(*)[16]>(sr + 32));
          tmem_wait_st();
        } else {
          // padding-only warp: still waits for PV_{u-1} so it cannot arrive on p_full for
          // sub-tile u before that barrier's previous phase (sub-tile u-1) has completed
          if (u > 0) {
            mbar_wait(&o_full[wg], o_cnt & 1);
            ++o_cnt;
          }
        }
        tc_fence_before();
        mbar_arrive(&p_full[wg]);
        if (tr) ATTN_TR(wg, it, u, 5);
      }
      if (active) {
        mbar_wait(&o_full[wg], o_cnt & 1);
        ++o_cnt;
        tc_fence_after();
        uint32_t o[32];
        tmem_ld32(o_addr, o);
        tmem_wait_ld();
        if (r < q_valid) {
          const float inv = resc / l_run;  // O still owes the last tile's rescale
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
