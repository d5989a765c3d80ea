// attn5_tc.cuh — attention v5: the varlen block-diagonal MHSA of the encoder (PAPER.md
// P:120-122 "each patch attends to every other patch"; per-task attention of the refine
// batch, P:261-265 with reading R11), softmax(q k^T / sqrt(dh)) v per head, dh = 32.
//
// Why a v5 (profiles/r1_attn_trace*.txt): in v4 the three softmax warpgroups shared one
// K/V stream and ran in lock step, so all of them were in their MUFU-bound exp phase at the
// same time and all of them were in their latency-bound phases (TMEM load, row max, P store)
// at the same time; and the dedicated MMA warps reacted ~500-900 cycles after the softmax
// warps released S or published P (mbarrier try_wait wake-up).  v5 changes three things:
//
//   * two independent PAIRS of softmax warpgroups.  A pair owns an item = (task, head, two
//     128-row query tiles) and its own Q slots and K/V ring; the two pairs of a CTA work on
//     different items and drift apart, so one pair's latency phases overlap the other's
//     exps.  Two query tiles per item also tile N = 400 (4 tiles) and N = 700 (6 tiles)
//     exactly, where v4's three-tile items wasted a whole K/V pass on a 16-row tail at N=400;
//   * no MMA warps: one thread of each warpgroup (on its highest-priority warp, see the
//     warp map below) issues the warpgroup's tcgen05.mma.  The four warps only ARRIVE on the
//     hand-off barriers (s_cons: S(u) is in registers; p_ready: P(u) is in TMEM) and never
//     wait for each other; the issuer waits on them at points where they have normally
//     completed already: PV(u-1) right after loading S(u), QK(u+1) after the exps of S(u).
//     (A 128-thread named barrier per hand-off measured 1.3x slower than v4: every warp
//     stalled on the lowest-priority warp of its warpgroup.)
//   * no producer warp either (a 17th warp would cost the register budget: the block's
//     register allocation is rounded to 4-warp units, so 544 threads get <= 96 registers):
//     the first thread of each pair's first warpgroup (the "leader", whose query tile always
//     exists) also issues the pair's TMA loads.  It polls the pair's queue with non-blocking
//     mbarrier probes once per sub-tile and, before it waits on a Q or K/V tile itself,
//     pumps the queue until that tile is issued (the loads go out strictly in consumption
//     order, so every stage it waits to refill is released by work already issued).
//
//   TMEM per warpgroup w (128 columns at w*128, 4 x 128 = 512):
//     S_w 64 fp32 cols (64-key sub-tile, single-buffered: released by the named barrier
//     right after the TMEM load), P_w 32 cols (bf16 pairs), O_w 32 cols (fp32, rescaled in place)
//   Warps: 0..15 softmax (warpgroup w = warp / 4, TMEM lane quarter = warp % 4); 512
//   threads, <= 128 registers.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "ptx.cuh"
#include "attn_tc.cuh"
#include "attn2_tc.cuh"
#include "attn4_tc.cuh"

namespace cfd {

template <int DH, int STAGES>
struct Attn5Smem {
  static constexpr int TILE_BYTES = 128 * DH * 2;
  static constexpr int Q_OFF = 0;                                  // [pair][slot 2][tile 2]
  static constexpr int KV_OFF = Q_OFF + 8 * TILE_BYTES;            // [pair][STAGES][K, V]
  static constexpr int BAR_OFF = KV_OFF + 2 * STAGES * 2 * TILE_BYTES;
  static constexpr int PROD_OFF = BAR_OFF + 384;                  // Attn5Prod[2] (after 40 barriers + TMEM slot)
  static constexpr int PRE_OFF = BAR_OFF + 512;
  static constexpr int TOTAL = 1024 + PRE_OFF + (ATTN2_MAX_T + 1) * 4;
  static constexpr uint32_t S_COL = 0;    // S_w at w*128
  static constexpr uint32_t P_COL = 64;   // P_w at w*128 + 64
  static constexpr uint32_t O_COL = 96;   // O_w at w*128 + 96
  __host__ __device__ static constexpr int q_off(int pair, int slot, int half) {
    return Q_OFF + ((pair * 2 + slot) * 2 + half) * TILE_BYTES;
  }
  __host__ __device__ static constexpr int k_off(int pair, int st) { return KV_OFF + (pair * STAGES + st) * 2 * TILE_BYTES; }
};

constexpr int ATTN5_THREADS = 512;  // 16 softmax warps (4 warpgroups = 2 pairs)

// Per-pair TMA producer cursor, in shared memory, touched only by the pair's leader thread.
struct Attn5Prod {
  int item, it, j, kvc, qdone, seq0, nkv, h, qp, nq;
};

template <int DH, int STAGES, int NPP>
__global__ void __launch_bounds__(ATTN5_THREADS, 1)
    attn5_tc_kernel(const __grid_constant__ CUtensorMap tmQKV, const AttnParams p, const int T, const int nh) {
  static_assert(DH == 32, "specialised for dh = 32 (64-byte rows, SW64)");
  using S = Attn5Smem<DH, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps the shared space
  // barriers: per pair q_full[2] q_empty[2] kv_full[STAGES] kv_empty[STAGES]; per warpgroup s_full, o_full
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::BAR_OFF);
  constexpr int PB = 4 + 2 * STAGES;
  auto q_full = [&](int pr, int slot) { return bars + pr * PB + slot; };
  auto q_empty = [&](int pr, int slot) { return bars + pr * PB + 2 + slot; };
  auto kv_full = [&](int pr, int st) { return bars + pr * PB + 4 + st; };
  auto kv_empty = [&](int pr, int st) { return bars + pr * PB + 4 + STAGES + st; };
  uint64_t* s_full = bars + 2 * PB;      // [4] QK(u) complete (tcgen05.commit)
  uint64_t* o_full = s_full + 4;         // [4] PV(u) complete (tcgen05.commit)
  uint64_t* s_cons = o_full + 4;         // [4] the 4 warps of warpgroup w hold S(u) in registers
  uint64_t* p_ready = s_cons + 4;        // [4] the 4 warps of warpgroup w stored P(u)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(p_ready + 4);
  int* prefix = reinterpret_cast<int*>(smem + S::PRE_OFF);

  const int warp = warp_id(), lane = lane_id();
#ifdef CFD_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 148) g_attn_trace[ATTN_TRACE_T0 + blockIdx.x] = clock64();
#endif
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    const int n = __ldg(p.cu_seqlens + t + 1) - __ldg(p.cu_seqlens + t);
    prefix[t + 1] = ((n + 255) / 256) * nh;  // items of two 128-row query tiles
  }
  Attn5Prod* prod = reinterpret_cast<Attn5Prod*>(smem + S::PROD_OFF);
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmQKV);
    for (int pr = 0; pr < 2; ++pr) {
      for (int i = 0; i < 2; ++i) { mbar_init(q_full(pr, i), 1); mbar_init(q_empty(pr, i), 2); }
      for (int s = 0; s < STAGES; ++s) { mbar_init(kv_full(pr, s), 1); mbar_init(kv_empty(pr, s), 2); }
    }
    for (int w = 0; w < 4; ++w) {
      mbar_init(&s_full[w], 1);
      mbar_init(&o_full[w], 1);
      mbar_init(&s_cons[w], 4);
      mbar_init(&p_ready[w], 4);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  __syncthreads();
  if (warp == 1) {  // inclusive scan of prefix[1..T], prefix[0] = 0
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
  const int stride = 2 * gridDim.x;

  {
    // ---------------------------------------------------------------- pair producer (leader thread)
    // Item sequence of pair pr: 2b + pr + k * stride.  Loads are issued in consumption order:
    // Q(item), K/V(item, 0..nkv-1), Q(next item), ...
    auto prod_start = [&](Attn5Prod& ps) {
      if (ps.item >= total) return;
      int t;
      decode_item(prefix, T, nh, ps.item, t, ps.qp, ps.h);
      ps.seq0 = __ldg(p.cu_seqlens + t);
      const int N = __ldg(p.cu_seqlens + t + 1) - ps.seq0;
      ps.nkv = (N + 127) / 128;
      ps.nq = min(2, ps.nkv - 2 * ps.qp);
      ps.j = 0;
      ps.qdone = 0;
    };
    // issue the next load of the pair if its slot is free; false if blocked or finished
    auto prod_step = [&](Attn5Prod& ps, int pr) -> bool {
      if (ps.item >= total) return false;
      if (!ps.qdone) {
        const int slot = ps.it & 1;
        if (!mbar_test(q_empty(pr, slot), ((ps.it >> 1) & 1) ^ 1)) return false;
        mbar_expect_tx(q_full(pr, slot), ps.nq * S::TILE_BYTES);
        for (int w = 0; w < ps.nq; ++w)
          tma_load_2d(smem + S::q_off(pr, slot, w), &tmQKV, q_full(pr, slot), ps.h * DH, ps.seq0 + (2 * ps.qp + w) * 128);
        ps.qdone = 1;
      } else {
        const int st = ps.kvc % STAGES;
        if (!mbar_test(kv_empty(pr, st), ((ps.kvc / STAGES) & 1) ^ 1)) return false;
        uint8_t* kb = smem + S::k_off(pr, st);
        mbar_expect_tx(kv_full(pr, st), 2 * S::TILE_BYTES);
        tma_load_2d(kb, &tmQKV, kv_full(pr, st), d + ps.h * DH, ps.seq0 + ps.j * 128);
        tma_load_2d(kb + S::TILE_BYTES, &tmQKV, kv_full(pr, st), 2 * d + ps.h * DH, ps.seq0 + ps.j * 128);
        ++ps.j;
        ++ps.kvc;
      }
      if (ps.qdone && ps.j == ps.nkv) {
        ps.item += stride;
        ++ps.it;
        prod_start(ps);
      }
      return true;
    };

    // ================================================================ softmax warpgroups (warps 0..15)
    // Warp -> (warpgroup, TMEM lane quarter) is a Latin square over the scheduler priority
    // levels: warp w sits on SMSP w % 4 (= its TMEM lane quarter) at priority level w / 4 (the
    // scheduler prefers the highest eligible warp id).  Every warpgroup owns one warp on each
    // SMSP and on each level, and its MMA issuer is its level-3 warp, which wins the issue
    // slot on its SMSP as soon as it is eligible.
    const int quarter = warp & 3;
    const int level = warp >> 2;
    const int wg = (level - quarter) & 3;
    const int pr = wg >> 1, half = wg & 1;
    const int r = quarter * 32 + lane;
    const bool issuer = level == 3 && lane == 0;
    const bool leader = issuer && half == 0;  // also the pair's TMA producer
    Attn5Prod& ps = prod[pr];
    if (leader) {
      ps.item = 2 * blockIdx.x + pr;
      ps.it = 0;
      ps.kvc = 0;
      prod_start(ps);
      for (int i = 0; i < 2 + STAGES && prod_step(ps, pr); ++i) {
      }
    }
    // leader: pump until Q of item `it_` / K/V tile `g_` (pair-global counter) has been issued
    auto ensure_q = [&](int it_) {
      while (!(ps.it > it_ || (ps.it == it_ && ps.qdone))) prod_step(ps, pr);
    };
    auto ensure_kv = [&](int g_) {
      while (ps.kvc <= g_) prod_step(ps, pr);
    };
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    const uint32_t s_tm = tmem + wg * 128 + S::S_COL;
    const uint32_t p_tm = tmem + wg * 128 + S::P_COL;
    const uint32_t o_tm = tmem + wg * 128 + S::O_COL;
    const float c = p.scale_log2;
    constexpr uint32_t idesc_s = make_idesc_bf16(128, 64, 0);  // S_u = Q K_u^T (64 keys)
    constexpr uint32_t idesc_o = make_idesc_bf16(128, DH, 1);  // O += P_u V_u (V MN-major)
    // SW64 smem descriptors with a zero start address: Q/K tiles K-major (LBO 16, SBO 512),
    // V tiles MN-major (LBO 4096, SBO 512)
    constexpr uint64_t kDescQK = (1ull << 16) | (32ull << 32) | (1ull << 46) | (uint64_t(kLayoutSW64) << 61);
    constexpr uint64_t kDescPV = (256ull << 16) | (32ull << 32) | (1ull << 46) | (uint64_t(kLayoutSW64) << 61);
    uint32_t s_cnt = 0, o_cnt = 0;
    int kvc = 0;
    int it = -1;
    if (p.stagger > 0 && pr == 1) {  // optional de-phasing of the two pairs
      const long long t_end = clock64() + p.stagger;
      while (clock64() < t_end) __nanosleep(64);
    }
    uint32_t qk_n = 0, pv_n = 0;  // issuer: QKs / PVs issued so far (s_cons / p_ready phases)
    for (int item = 2 * blockIdx.x + pr; item < total; item += stride) {
      ++it;
      int t, qp, h;
      decode_item(prefix, T, nh, item, t, qp, h);
      const int seq0 = __ldg(p.cu_seqlens + t);
      const int N = __ldg(p.cu_seqlens + t + 1) - seq0;
      const int nkv = (N + 127) / 128;
      const int qt = 2 * qp + half;
      const int slot = it & 1;
      if (qt >= nkv) {
        // no query tile for this warpgroup in this item: keep the pair's barriers in step
        if (issuer) {
          mbar_wait(q_full(pr, slot), (it >> 1) & 1);
          for (int jj = 0; jj < nkv; ++jj) {
            const int st = (kvc + jj) % STAGES;
            mbar_wait(kv_full(pr, st), ((kvc + jj) / STAGES) & 1);
            mbar_arrive(kv_empty(pr, st));
          }
          mbar_arrive(q_empty(pr, slot));
        }
        kvc += nkv;
        continue;
      }
      const int nsub = (N + 63) / 64;
      const uint32_t qa = smem_u32(smem + S::q_off(pr, slot, half));
      // issuer: QK(u) into S_w once every warp has consumed the previous S (s_cons phase)
      auto issue_qk = [&](int u) {
        const int jj = u >> 1;
        const int st = (kvc + jj) % STAGES;
        if ((u & 1) == 0) {
          if (leader) ensure_kv(kvc + jj);
          mbar_wait(kv_full(pr, st), ((kvc + jj) / STAGES) & 1);
        }
        if (qk_n > 0) mbar_wait(&s_cons[wg], (qk_n - 1) & 1);
        ++qk_n;
        const uint32_t ka = smem_u32(smem + S::k_off(pr, st)) + (u & 1) * 64 * DH * 2;
        tc_fence_after();
        // descriptor start-address field = addr >> 4 (14 bits; smem < 256 KB never carries out)
        const uint64_t dq = kDescQK + (qa >> 4), dk = kDescQK + (ka >> 4);
#pragma unroll
        for (int k = 0; k < DH / 16; ++k) mma_ss(s_tm, dq + 2 * k, dk + 2 * k, idesc_s, k);
        mma_commit(&s_full[wg]);
        ATTN_TR(wg, it, u, 6);
      };
      // issuer: PV(u) once every warp has stored P(u) (p_ready phase)
      auto issue_pv = [&](int u) {
        mbar_wait(&p_ready[wg], pv_n & 1);
        ++pv_n;
        tc_fence_after();
        const int jj = u >> 1;
        const int st = (kvc + jj) % STAGES;
        const int valid = min(64, N - u * 64);
        const uint32_t va = smem_u32(smem + S::k_off(pr, st) + S::TILE_BYTES) + (u & 1) * 64 * DH * 2;
        const int ksteps = (valid + 15) / 16;
        const uint64_t dv = kDescPV + (va >> 4);
        for (int k = 0; k < ksteps; ++k) mma_ts(o_tm, p_tm + k * 8, dv + k * (16 * DH * 2 / 16), idesc_o, (u | k) != 0);
        mma_commit(&o_full[wg]);
        ATTN_TR(wg, it, u, 7);
        if ((u & 1) || u + 1 == nsub) mma_commit(kv_empty(pr, st));
        if (u + 1 == nsub) mma_commit(q_empty(pr, slot));
      };
      if (issuer) {
        if (leader) ensure_q(it);
        mbar_wait(q_full(pr, slot), (it >> 1) & 1);
        issue_qk(0);
      }
      const int q_valid = N - qt * 128;
      const bool active = quarter * 32 < q_valid;
      float m_run = -INFINITY, l_run = 0.f;
      for (int u = 0; u < nsub; ++u) {
        const int valid = min(64, N - u * 64);
        mbar_wait(&s_full[wg], s_cnt & 1);
        ++s_cnt;
        tc_fence_after();
        if (issuer) ATTN_TR(wg, it, u, 0);
        uint32_t sr[64];
        if (active) {
          tmem_ld32(s_tm + lane_off, *reinterpret_cast<uint32_t(*)[32]>(sr));
          if (valid > 32) tmem_ld32(s_tm + lane_off + 32, *reinterpret_cast<uint32_t(*)[32]>(sr + 32));
          tmem_wait_ld();
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_cons[wg]);  // this warp is done with S_w
        if (issuer) {
          ATTN_TR(wg, it, u, 1);
          if (u > 0) issue_pv(u - 1);
          if (leader) {  // keep the pair's K/V ring full (non-blocking)
            for (int i = 0; i < 2 && prod_step(ps, pr); ++i) {
            }
          }
        }
        float alpha = 1.f;
        bool upd = false;
        if (active) {
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
          if (issuer) ATTN_TR(wg, it, u, 2);
          // lazy rescale (R23): the running max only moves when a tile exceeds it by > 2^8
          upd = (m_run == -INFINITY) || (m_cand > m_run + 8.0f);
          alpha = upd ? ((m_run == -INFINITY) ? 0.f : ex2_approx(m_run - m_cand)) : 1.f;
          if (upd) m_run = m_cand;
          const float neg = -m_run;
          float sum0 = 0.f, sum1 = 0.f, sum2 = 0.f, sum3 = 0.f;
          if (valid == 64) {
            exp_chunk<NPP>(sr, c, neg, sum0, sum1);
            exp_chunk<NPP>(sr + 32, c, neg, sum2, sum3);
          } else {
            exp_chunk<0>(sr, c, neg, sum0, sum1);
            if (valid > 32) exp_chunk<0>(sr + 32, c, neg, sum2, sum3);
          }
          l_run = l_run * alpha + ((sum0 + sum1) + (sum2 + sum3));
          if (issuer) ATTN_TR(wg, it, u, 3);
        }
        if (issuer && u + 1 < nsub) issue_qk(u + 1);
        if (u > 0) {
          // PV(u-1) done: P_w may be overwritten and O_w rescaled
          mbar_wait(&o_full[wg], o_cnt & 1);
          ++o_cnt;
          tc_fence_after();
          if (active && __any_sync(0xffffffffu, upd)) {
            uint32_t o[32];
            tmem_ld32(o_tm + lane_off, o);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < DH; i += 2) {
              float a0, a1;
              fma2(a0, a1, __uint_as_float(o[i]), __uint_as_float(o[i + 1]), alpha, alpha, 0.f, 0.f);
              o[i] = __float_as_uint(a0);
              o[i + 1] = __float_as_uint(a1);
            }
            tmem_st16(o_tm + lane_off, *reinterpret_cast<const uint32_t(*)[16]>(o));
            tmem_st16(o_tm + lane_off + 16, *reinterpret_cast<const uint32_t(*)[16]>(o + 16));
          }
        }
        if (issuer) ATTN_TR(wg, it, u, 4);
        if (active) {
          tmem_st16(p_tm + lane_off, *reinterpret_cast<const uint32_t(*)[16]>(sr));
          if (valid > 32) tmem_st16(p_tm + lane_off + 16, *reinterpret_cast<const uint32_t(*)[16]>(sr + 32));
          tmem_wait_st();
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_ready[wg]);  // P(u) (and the rescaled O) of this warp in TMEM
        if (issuer) ATTN_TR(wg, it, u, 5);
      }
      if (issuer) issue_pv(nsub - 1);
      kvc += nkv;
      // epilogue: O / l -> bf16 rows of this query tile, natural-log LSE for the score kernel
      mbar_wait(&o_full[wg], o_cnt & 1);
      ++o_cnt;
      tc_fence_after();
      if (active) {
        uint32_t o[32];
        tmem_ld32(o_tm + lane_off, o);
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
      }
      tc_fence_before();
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

}  // namespace cfd
