// attn2_tc.cuh — persistent varlen multi-head attention on tcgen05, two query tiles per
// work item ("each patch attends to every other patch",
// block-diagonal per task for the patch-level batch, PAPER.md:261-265 / reading R11).
//
// Work item = (task, pair of 128-row query tiles, head).  Items are enumerated on the
// device from cu_seqlens (no host sync) and distributed round-robin over one CTA per
// SM.  Both query tiles of an item share every K/V tile the TMA warp streams in.
//
// Warps: 0 = TMA producer, 1 = TMEM allocator + tcgen05.mma issuer,
//        2..5 = softmax warpgroup 0 (query tile 2*qp), 6..9 = softmax warpgroup 1
//        (query tile 2*qp+1).  While one warpgroup computes exponentials the tensor
//        core serves the other (ping-pong).
// TMEM:  per warpgroup S_w (128 fp32 columns), P_w (64 columns of bf16 pairs) and O_w
//        (32 columns) = 448 of 512 columns.  The warpgroup releases S_w (s_free) as soon
//        as S_j is in registers, so QK_{j+1} runs on the tensor core during the softmax
//        of tile j; O_w accumulates P_w V_j in TMEM and is rescaled in place by the
//        softmax warps (lazily, only when a row's running max grows by more than 2^8).
// Softmax per row (one thread per query row): FMNMX3 row max, FFMA2 scale/shift,
// exp2 split between MUFU.EX2 and a degree-3 polynomial on the FMA pipe (NPP of every
// 16 column pairs), FADD2 row sums, bf16x2 pack, tcgen05.st.  Fully masked 32-column
// chunks of a tail KV tile and all-padding warps of a tail query tile skip the work.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "ptx.cuh"
#include "attn_tc.cuh"

namespace cfd {

constexpr int ATTN2_THREADS = 320;
constexpr int ATTN2_MAX_T = 4096;

template <int DH, int STAGES>
struct Attn2Smem {
  static constexpr int TILE_BYTES = 128 * DH * 2;             // one 128-row tile of q, k or v
  static constexpr int Q_OFF = 0;                              // [2 slots][2 tiles]
  static constexpr int K_OFF = Q_OFF + 4 * TILE_BYTES;         // [STAGES]
  static constexpr int V_OFF = K_OFF + STAGES * TILE_BYTES;    // [STAGES]
  static constexpr int BAR_OFF = V_OFF + STAGES * TILE_BYTES;
  static constexpr int PRE_OFF = BAR_OFF + 256;
  static constexpr int TOTAL = 1024 + PRE_OFF + (ATTN2_MAX_T + 1) * 4;
  static constexpr uint32_t S_COL = 0;    // S_w at w*128
  static constexpr uint32_t P_COL = 256;  // P_w at 256 + w*64 (bf16 pairs)
  static constexpr uint32_t O_COL = 384;  // O_w at 384 + w*DH
};

// ---------------------------------------------------------------- packed fp32 helpers
__device__ __forceinline__ void fma2(float& d0, float& d1, float a0, float a1, float b0, float b1, float c0,
                                     float c1) {
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}
__device__ __forceinline__ void add2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// 2^x for a pair, x <= 0, on the FMA pipe: x = j + f, j = round(x), f in [-1/2, 1/2];
// 2^f by a degree-3 minimax polynomial (max rel. error 7.6e-5 < bf16 ulp/2), 2^j
// inserted into the exponent field.  x is clamped at -126: with j = -126 the biased
// exponent of 2^f (126 or 127) stays >= 0 (result ~1e-38 ~ 0); at -127 it wrapped into the
// sign bit for f <= 0 and produced NaN for logits more than 2^127 below the row max.
__device__ __forceinline__ void exp2_poly2(float& y0, float& y1, float x0, float x1) {
  constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23: t = x + M rounds x to an integer in t's low bits
  x0 = fmaxf(x0, -126.f);
  x1 = fmaxf(x1, -126.f);
  float t0, t1, r0, r1, f0, f1, p0, p1;
  add2(t0, t1, x0, x1, kMagic, kMagic);
  add2(r0, r1, t0, t1, -kMagic, -kMagic);
  add2(f0, f1, x0, x1, -r0, -r1);
  fma2(p0, p1, f0, f1, 0.05517025f, 0.05517025f, 0.24260790f, 0.24260790f);
  fma2(p0, p1, p0, p1, f0, f1, 0.69326093f, 0.69326093f);
  fma2(p0, p1, p0, p1, f0, f1, 0.99992828f, 0.99992828f);
  y0 = __int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23));
  y1 = __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23));
}

// One 32-column chunk of a score row: p = 2^(s*c - m) for 16 pairs, running pair sums,
// bf16x2-packed results written to sr[0..15].  Pairs [16-NPP, 16) use the polynomial.
template <int NPP>
__device__ __forceinline__ void exp_chunk(uint32_t* sr, float c, float neg, float& sum0, float& sum1) {
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    float x0, x1, p0, p1;
    fma2(x0, x1, __uint_as_float(sr[2 * i]), __uint_as_float(sr[2 * i + 1]), c, c, neg, neg);
    if (i >= 16 - NPP) {
      exp2_poly2(p0, p1, x0, x1);
    } else {
      p0 = ex2_approx(x0);
      p1 = ex2_approx(x1);
    }
    add2(sum0, sum1, sum0, sum1, p0, p1);
    sr[i] = pack_bf16x2(p0, p1);
  }
}

// item -> (task, query pair, head): prefix[t] = first item of task t
__device__ __forceinline__ void decode_item(const int* prefix, int T, int nh, int item, int& t, int& qp, int& h) {
  int lo = 0, hi = T - 1;
  while (lo < hi) {  // last t with prefix[t] <= item
    const int mid = (lo + hi + 1) >> 1;
    if (prefix[mid] <= item) lo = mid; else hi = mid - 1;
  }
  t = lo;
  const int r = item - prefix[lo];
  qp = r / nh;
  h = r % nh;
}

template <int DH, int STAGES, int NPP>
__global__ void __launch_bounds__(ATTN2_THREADS, 1)
    attn2_tc_kernel(const __grid_constant__ CUtensorMap tmQKV, const AttnParams p, const int T, const int nh) {
  static_assert(DH == 32, "specialised for dh = 32 (64-byte rows, SW64)");
  using S = Attn2Smem<DH, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps the shared space
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::BAR_OFF);
  uint64_t* q_full = bars;                  // [2]
  uint64_t* q_empty = bars + 2;             // [2]
  uint64_t* kv_full = bars + 4;             // [STAGES]
  uint64_t* kv_empty = kv_full + STAGES;    // [STAGES]
  uint64_t* s_full = kv_empty + STAGES;     // [2]
  uint64_t* s_free = s_full + 2;            // [2]
  uint64_t* p_full = s_free + 2;            // [2]
  uint64_t* o_full = p_full + 2;            // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_full + 2);
  int* prefix = reinterpret_cast<int*>(smem + S::PRE_OFF);

  const int warp = warp_id(), lane = lane_id();
  // ---- item prefix over tasks: items_t = ceil(N_t / 256) * nh
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    const int n = __ldg(p.cu_seqlens + t + 1) - __ldg(p.cu_seqlens + t);
    prefix[t + 1] = ((n + 255) / 256) * nh;
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmQKV);
    for (int i = 0; i < 2; ++i) { mbar_init(&q_full[i], 1); mbar_init(&q_empty[i], 1); }
    for (int s = 0; s < STAGES; ++s) { mbar_init(&kv_full[s], 1); mbar_init(&kv_empty[s], 1); }
    for (int w = 0; w < 2; ++w) {
      mbar_init(&s_full[w], 1);
      mbar_init(&s_free[w], 128);
      mbar_init(&p_full[w], 128);
      mbar_init(&o_full[w], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  __syncthreads();
  if (warp == 0) {  // inclusive scan of prefix[1..T] by one warp, prefix[0] = 0
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

  if (warp == 0) {
    // ================================================================ TMA producer
    if (lane == 0) {
      int it = 0, kvc = 0;
      for (int item = blockIdx.x; item < total; item += gridDim.x, ++it) {
        int t, qp, h;
        decode_item(prefix, T, nh, item, t, qp, h);
        const int seq0 = __ldg(p.cu_seqlens + t);
        const int N = __ldg(p.cu_seqlens + t + 1) - seq0;
        const int nq = ((2 * qp + 1) * 128 < N) ? 2 : 1;
        const int nkv = (N + 127) / 128;
        const int slot = it & 1;
        mbar_wait(&q_empty[slot], ((it >> 1) & 1) ^ 1);
        mbar_expect_tx(&q_full[slot], nq * S::TILE_BYTES);
        for (int w = 0; w < nq; ++w)
          tma_load_2d(smem + S::Q_OFF + (slot * 2 + w) * S::TILE_BYTES, &tmQKV, &q_full[slot], h * DH,
                      seq0 + (2 * qp + w) * 128);
        for (int j = 0; j < nkv; ++j, ++kvc) {
          const int st = kvc % STAGES;
          mbar_wait(&kv_empty[st], ((kvc / STAGES) & 1) ^ 1);
          mbar_expect_tx(&kv_full[st], 2 * S::TILE_BYTES);
          tma_load_2d(smem + S::K_OFF + st * S::TILE_BYTES, &tmQKV, &kv_full[st], d + h * DH, seq0 + j * 128);
          tma_load_2d(smem + S::V_OFF + st * S::TILE_BYTES, &tmQKV, &kv_full[st], 2 * d + h * DH, seq0 + j * 128);
        }
      }
    }
  } else if (warp == 1) {
    // ================================================================ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_s = make_idesc_bf16(128, 128, 0);  // S = Q K^T
      constexpr uint32_t idesc_o = make_idesc_bf16(128, DH, 1);   // O = P V  (V MN-major)
      int it = 0, kvc = 0;
      uint32_t p_cnt[2] = {0, 0}, s_use[2] = {0, 0};
      for (int item = blockIdx.x; item < total; item += gridDim.x, ++it) {
        int t, qp, h;
        decode_item(prefix, T, nh, item, t, qp, h);
        const int seq0 = __ldg(p.cu_seqlens + t);
        const int N = __ldg(p.cu_seqlens + t + 1) - seq0;
        const int nq = ((2 * qp + 1) * 128 < N) ? 2 : 1;
        const int nkv = (N + 127) / 128;
        const int slot = it & 1;
        mbar_wait(&q_full[slot], (it >> 1) & 1);
        // S_w = Q_w K^T into TMEM; waits until the warpgroup has read the previous S_w
        auto issue_qk = [&](int w, int st) {
          if (s_use[w] > 0) mbar_wait(&s_free[w], (s_use[w] - 1) & 1);
          ++s_use[w];
          tc_fence_after();
          const uint32_t qa = smem_u32(smem + S::Q_OFF + (slot * 2 + w) * S::TILE_BYTES);
          const uint32_t ka = smem_u32(smem + S::K_OFF + st * S::TILE_BYTES);
#pragma unroll
          for (int k = 0; k < DH / 16; ++k)
            mma_ss(tmem + S::S_COL + w * 128, make_smem_desc(qa + k * 32, 16, 512, kLayoutSW64),
                   make_smem_desc(ka + k * 32, 16, 512, kLayoutSW64), idesc_s, k);
          mma_commit(&s_full[w]);
        };
        {
          const int st = kvc % STAGES;
          mbar_wait(&kv_full[st], (kvc / STAGES) & 1);
          tc_fence_after();
          for (int w = 0; w < nq; ++w) issue_qk(w, st);
        }
        for (int j = 0; j < nkv; ++j) {
          const int st = (kvc + j) % STAGES;
          const int valid = min(128, N - j * 128);
          const int ksteps = (valid + 15) / 16;
          if (j + 1 < nkv) {  // S_{j+1} runs on the tensor core while the softmax works on S_j
            const int st1 = (kvc + j + 1) % STAGES;
            mbar_wait(&kv_full[st1], ((kvc + j + 1) / STAGES) & 1);
            for (int w = 0; w < nq; ++w) issue_qk(w, st1);
          }
          const uint32_t va = smem_u32(smem + S::V_OFF + st * S::TILE_BYTES);
          for (int w = 0; w < nq; ++w) {
            mbar_wait(&p_full[w], p_cnt[w] & 1);
            ++p_cnt[w];
            tc_fence_after();
            for (int k = 0; k < ksteps; ++k)
              mma_ts(tmem + S::O_COL + w * DH, tmem + S::P_COL + w * 64 + k * 8,
                     make_smem_desc(va + k * 16 * DH * 2, 4096, 512, kLayoutSW64), idesc_o, (j | k) != 0);
            mma_commit(&o_full[w]);
          }
          mma_commit(&kv_empty[st]);
        }
        kvc += nkv;
        mma_commit(&q_empty[slot]);
      }
    }
  } else {
    // ================================================================ softmax warpgroups
    const int wg = (warp - 2) >> 2;                 // 0 or 1
    const int quarter = warp & 3;                   // TMEM lane quarter
    const int r = quarter * 32 + lane;              // query row in the tile
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    const uint32_t s_addr = tmem + lane_off + S::S_COL + wg * 128;
    const uint32_t p_addr = tmem + lane_off + S::P_COL + wg * 64;
    const uint32_t o_addr = tmem + lane_off + S::O_COL + wg * DH;
    const float c = p.scale_log2;
    uint32_t s_cnt = 0, o_cnt = 0;
    for (int item = blockIdx.x; item < total; item += gridDim.x) {
      int t, qp, h;
      decode_item(prefix, T, nh, item, t, qp, h);
      const int seq0 = __ldg(p.cu_seqlens + t);
      const int N = __ldg(p.cu_seqlens + t + 1) - seq0;
      const int qt = 2 * qp + wg;
      if (qt * 128 >= N) continue;                 // this warpgroup has no tile in this item
      const int nkv = (N + 127) / 128;
      const int q_valid = N - qt * 128;
      const bool active = quarter * 32 < q_valid;  // warp-uniform: any real query row here
      float m_run = -INFINITY, l_run = 0.f;
      for (int j = 0; j < nkv; ++j) {
        mbar_wait(&s_full[wg], s_cnt & 1);
        ++s_cnt;
        tc_fence_after();
        const int valid = min(128, N - j * 128);
        const int nch = (valid + 31) / 32;         // 32-column chunks holding real keys
        if (active) {
          uint32_t sr[128];
#pragma unroll
          for (int ch = 0; ch < 4; ++ch)
            if (ch < nch) tmem_ld32(s_addr + ch * 32, *reinterpret_cast<uint32_t(*)[32]>(sr + ch * 32));
          tmem_wait_ld();
          tc_fence_before();
          mbar_arrive(&s_free[wg]);  // S_w may now be overwritten by QK_{j+1}
          if (valid < 128) {
#pragma unroll
            for (int i = 0; i < 128; ++i)
              if (i >= valid) sr[i] = __float_as_uint(-INFINITY);
          }
          float mx = -INFINITY;
#pragma unroll
          for (int ch = 0; ch < 4; ++ch) {
            if (ch < nch) {
#pragma unroll
              for (int i = 0; i < 32; i += 2)
                mx = fmax3(mx, __uint_as_float(sr[ch * 32 + i]), __uint_as_float(sr[ch * 32 + i + 1]));
            }
          }
          // Lazy rescale: keep the running max unless the new one exceeds it by more than
          // 2^8 (P then stays <= 256, exact in fp32 / bf16 range); O is corrected in TMEM
          // only when some row of the warp moved its max.
          const float m_cand = mx * c;
          const bool upd = (m_run == -INFINITY) || (m_cand > m_run + 8.0f);
          const float alpha = upd ? ((m_run == -INFINITY) ? 0.f : ex2_approx(m_run - m_cand)) : 1.f;
          if (upd) m_run = m_cand;
          const float neg = -m_run;
          float sum0 = 0.f, sum1 = 0.f;
          // exponentials; packed bf16 pairs overwrite sr[ch*32 + 0..15] (already consumed).
          // Full tiles split exp2 between MUFU and the FMA-pipe polynomial; the tail tile
          // (masked columns, must give exact zeros) uses MUFU only.
          if (valid == 128) {
#pragma unroll
            for (int ch = 0; ch < 4; ++ch) exp_chunk<NPP>(sr + ch * 32, c, neg, sum0, sum1);
          } else {
#pragma unroll
            for (int ch = 0; ch < 4; ++ch) {
              if (ch < nch) exp_chunk<0>(sr + ch * 32, c, neg, sum0, sum1);
            }
          }
          l_run = l_run * alpha + (sum0 + sum1);
          if (j > 0) {
            // PV_{j-1} must be complete before O is rescaled or PV_j accumulates into it
            mbar_wait(&o_full[wg], o_cnt & 1);
            ++o_cnt;
            tc_fence_after();
            if (__any_sync(0xffffffffu, upd)) {
              uint32_t o[32];
              tmem_ld32(o_addr, o);
              tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < DH; i += 2) {
                float a0, a1;
                fma2(a0, a1, __uint_as_float(o[i]), __uint_as_float(o[i + 1]), alpha, alpha, 0.f, 0.f);
                o[i] = __float_as_uint(a0);
                o[i + 1] = __float_as_uint(a1);
              }
              tmem_st16(o_addr, *reinterpret_cast<const uint32_t(*)[16]>(o));
              tmem_st16(o_addr + 16, *reinterpret_cast<const uint32_t(*)[16]>(o + 16));
            }
          }
          // P_j into P_w (PV_{j-1}, its previous reader, completed: o_full waited above)
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (q * 32 < valid)
              tmem_st16(p_addr + q * 16, *reinterpret_cast<const uint32_t(*)[16]>(sr + q * 32));
          tmem_wait_st();
        } else {
          // padding-only warp: still waits for PV_{j-1} so it cannot arrive on p_full for
          // tile j before that barrier's previous phase (tile j-1) has completed
          mbar_arrive(&s_free[wg]);
          if (j > 0) {
            mbar_wait(&o_full[wg], o_cnt & 1);
            ++o_cnt;
          }
        }
        tc_fence_before();
        mbar_arrive(&p_full[wg]);
      }
      if (active) {
        mbar_wait(&o_full[wg], o_cnt & 1);
        ++o_cnt;
        tc_fence_after();
        uint32_t o[32];
        tmem_ld32(o_addr, o);
        tmem_wait_ld();
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
        tc_fence_before();  // O_w is read before the next item's first PV overwrites it
      } else {
        mbar_wait(&o_full[wg], o_cnt & 1);
        ++o_cnt;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

}  // namespace cfd
