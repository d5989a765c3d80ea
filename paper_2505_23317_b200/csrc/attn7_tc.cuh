// attn7_tc.cuh — attention v7: the varlen block-diagonal multi-head self-attention of the
// encoder (§II-A "each patch attends to every other patch"; per-task
// attention of the patch-level batch, PAPER.md:261-265 with reading R11), O = softmax(q k^T /
// sqrt(dh)) v per head, dh = 32, plus the natural-log row LSE for the criticality score.
//
// Why v7 (profiles/r2_tc_micro.txt): at dh = 32 a score element costs 128
// tensor FLOPs but one exp2, so the kernel is bounded by the exp unit (MUFU, 16/clk/SM) and
// the softmax's issue slots, and an M = 128 tcgen05.mma costs ~45 cycles at N = 32 or 64
// whatever its size.  In v4 the three softmax warpgroups shared one item and one K/V stream
// and ran in lock step: all of them were in their MUFU-bound exp phase at once, then all
// their MMAs queued on the tensor pipe at once (a ~500-cycle burst), then all of them were in
// their latency-bound TMEM-load / row-max phase at once, so the MUFU idled ~45 % of the time.
// v7 gives every warpgroup its OWN work: an item is (task, head, one 128-row query tile); each
// warpgroup claims its items, streams its own K/V through its own ring and runs its own
// S -> P -> O pipeline, so the warpgroups drift apart and one's exps overlap another's MMAs
// and latency phases.
//
// Warps: 0..4*NWG-1 softmax (warpgroup w = warp / 4, TMEM lane quarter = warp % 4), NWG = 3
//        or 4; then two control warpgroups: warp 4*NWG + w is warpgroup w's MMA warp (lane 0
//        issues its tcgen05.mma: QK S = Q K_u^T, SS, N = 64; PV O += P_u V_u, TS, P from
//        TMEM), warp 5*NWG + w its producer (lane 0 claims its items and streams their Q tiles
//        and 64-key K/V sub-tiles by TMA into its ring); the control threads poll their
//        barriers with a short sleep.  setmaxnreg moves the control warps' registers to the
//        softmax warps.
// TMEM per warpgroup (128 columns at w*128): S 64 fp32 (single-buffered: released right after
//        the softmax has loaded it, so QK(u+1) runs under the exps of u), P 32 (bf16 pairs),
//        O 32 (fp32, rescaled in place, lazily: reading R23).
// Item order: the full 128-row tiles of the tasks (longest task first for small ragged
//        batches), then the tail tiles, claimed dynamically (work counter) after a static
//        first item per warpgroup.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "ptx.cuh"
#include "attn_tc.cuh"
#include "attn_common.cuh"
#include "score_tc.cuh"  // named_bar_sync

namespace cfd {

#ifndef CFD_SPLIT_ROWS
#define CFD_SPLIT_ROWS 32
#endif
constexpr int SPLIT_ROWS = CFD_SPLIT_ROWS;  // tail tiles with at most this many real rows are split
static_assert(SPLIT_ROWS == 32 || SPLIT_ROWS == 64, "split tail: 4 replicas of 32 rows or 2 of 64");
constexpr int SPLIT_REP = SPLIT_ROWS == 32 ? 4 : 2;  // replicas of a split tail tile over the lane quarters
constexpr int ATTN7_ST = 4;          // K/V ring stages per warpgroup (64 keys each)
// NWG softmax warpgroups (3 or 4) + two control warpgroups (an MMA warp and a producer warp
// per softmax warpgroup, the rest idle)
__host__ __device__ constexpr int attn7_threads(int nwg) { return 128 * (nwg + 2); }
constexpr int ATTN7_MAX_T = 1024;    // tasks per launch (item tables in shared memory)
constexpr int ATTN7_SORT_T = 256;    // batches up to this many tasks are ordered longest-first

template <int NWG>
struct Attn7Smem {
  static constexpr int SUB_BYTES = 64 * 32 * 2;                     // 64 rows x dh 32 bf16 (SW64)
  static constexpr int Q_BYTES = 2 * SUB_BYTES;                     // 128-row query tile
  static constexpr int WG_BYTES = 2 * Q_BYTES + 2 * ATTN7_ST * SUB_BYTES;  // Q[2] | K[ST] | V[ST]
  static constexpr int BAR_OFF = NWG * WG_BYTES;
  static constexpr int NBAR_WG = 4 + 2 * ATTN7_ST + 4;             // q_full q_empty [2] | kv [ST] | s p o
  static constexpr int SLOT_OFF = BAR_OFF + NWG * NBAR_WG * 8 + 16;  // + TMEM slot
  static constexpr int SLOT_INTS = 8;  // per published item: item, task, tile, head, seq0, N, n_keys, -
  static constexpr int TAB_OFF = SLOT_OFF + NWG * 2 * SLOT_INTS * 4 + 16;
  // split tail items: per warpgroup the (m, l) of its 4 x 32 rows and one 32 x 33 fp32 O accumulator
  static constexpr int MERGE_OFF = TAB_OFF + 3 * (ATTN7_MAX_T + 1) * 4;
  static constexpr int MERGE_WG_FLOATS = 4 * 32 * 2 + 32 * 33;
  static constexpr int TOTAL = 1024 + MERGE_OFF + NWG * MERGE_WG_FLOATS * 4;
  __host__ __device__ static constexpr int q_off(int w, int slot) { return w * WG_BYTES + slot * Q_BYTES; }
  __host__ __device__ static constexpr int k_off(int w, int st) { return w * WG_BYTES + 2 * Q_BYTES + st * SUB_BYTES; }
  __host__ __device__ static constexpr int v_off(int w, int st) {
    return w * WG_BYTES + 2 * Q_BYTES + (ATTN7_ST + st) * SUB_BYTES;
  }
  static constexpr uint32_t S_COL = 0, P_COL = 64, O_COL = 96;   // within the warpgroup's 128 columns
};
static_assert(Attn7Smem<4>::TOTAL <= 232448, "attn7 shared memory budget");

// Poll an mbarrier phase: test, and sleep ~ns between probes (the control warps share their
// SMSP with three softmax warps: a busy spin would take their issue slots).
// Producer-side poll with a run-time sleep: the producer runs up to ATTN7_ST sub-tiles ahead, so
// it can react slowly, and each probe it makes takes issue slots from the softmax warps that
// share its SMSP (at 32 ns its kv_empty probes were ~7 % of all issued instructions).
__device__ __forceinline__ void mbar_poll_slow(uint64_t* bar, uint32_t parity, int ns) {
  while (!mbar_test(bar, parity)) __nanosleep(ns);
}

// NS = 1: try_wait (the hardware may suspend the thread until the phase completes);
// NS = 2: busy test_wait loop
template <int NS>
__device__ __forceinline__ void mbar_poll(uint64_t* bar, uint32_t parity) {
  if constexpr (NS == 1) {
    mbar_wait(bar, parity);
  } else if constexpr (NS == 2) {
    mbar_spin(bar, parity);
  } else {
    while (!mbar_test(bar, parity)) __nanosleep(NS);
  }
}

// Item tables: order[] = tasks in processing order, pre_full[i] = first full-tile item of
// order[i] (full tiles: nfull(t) * nh each), pre_tail[i] = first tail item of order[i]
// (1 * nh if N % 128 != 0).  Item = (task, tile, head).
__device__ __forceinline__ void decode_item7(const int* order, const int* pre_full, const int* pre_tail, int T,
                                             int nh, int n_full_items, int item, int& t, int& tile, int& h,
                                             const int* cu) {
  const int* pre = item < n_full_items ? pre_full : pre_tail;
  const int x = item < n_full_items ? item : item - n_full_items;
  int lo = 0, hi = T - 1;
  while (lo < hi) {  // last i with pre[i] <= x
    const int mid = (lo + hi + 1) >> 1;
    if (pre[mid] <= x) lo = mid; else hi = mid - 1;
  }
  t = order[lo];
  const int r = x - pre[lo];
  if (item < n_full_items) {
    tile = r / nh;
    h = r - tile * nh;
  } else {
    tile = (__ldg(cu + t + 1) - __ldg(cu + t)) / 128;  // the tail tile
    h = r;
  }
}

template <int NWG, int NPP, int SLEEP_NS>
__global__ void __launch_bounds__(attn7_threads(NWG), 1)
    attn7_tc_kernel(const __grid_constant__ CUtensorMap tmQKV, const __grid_constant__ CUtensorMap tmQ32,
                    const AttnParams p, const int T, const int nh) {
  using S = Attn7Smem<NWG>;
  constexpr int DH = 32;
  constexpr int kMmaWarp = 4 * NWG;  // also allocates TMEM
  // register split: two control warpgroups at CTRL_REGS, the softmax warpgroups at SOFT_REGS
  constexpr int CTRL_REGS = 32;
  constexpr int SOFT_REGS = NWG == 4 ? 104 : 136;
  // the pool setmaxnreg redistributes is the CTA's launch allocation (threads x the launch-bound registers)
  static_assert(NWG * 128 * SOFT_REGS + 256 * CTRL_REGS <= (NWG == 4 ? 768 * 80 : 640 * 96), "register split");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::BAR_OFF);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + S::BAR_OFF + NWG * S::NBAR_WG * 8);
  // [w][slot][SLOT_INTS]: the producer decodes each item once and publishes it with the Q tile
  volatile int* item_slot = reinterpret_cast<volatile int*>(smem + S::SLOT_OFF);
  int* order = reinterpret_cast<int*>(smem + S::TAB_OFF);
  int* pre_full = order + (ATTN7_MAX_T + 1);
  int* pre_tail = pre_full + (ATTN7_MAX_T + 1);
  __shared__ int s_nfull;

  const int warp = warp_id(), lane = lane_id();
#ifdef CFD_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 148) g_attn_trace[ATTN_TRACE_T0 + blockIdx.x] = clock64();
#endif
  // ---- item tables: processing order (longest task first for small batches), per-task item counts
  for (int i = threadIdx.x; i < T; i += blockDim.x) {
    const int n = __ldg(p.cu_seqlens + i + 1) - __ldg(p.cu_seqlens + i);
    int pos = i;
    if (T <= ATTN7_SORT_T) {  // rank by (N desc, index asc)
      pos = 0;
      for (int u = 0; u < T; ++u) {
        const int nu = __ldg(p.cu_seqlens + u + 1) - __ldg(p.cu_seqlens + u);
        pos += (nu > n) || (nu == n && u < i);
      }
    }
    order[pos] = i;
    pre_full[pos + 1] = (n / 128) * nh;
    pre_tail[pos + 1] = (n % 128) ? nh : 0;
  }
  if (warp == kMmaWarp) {
    if (lane == 0) {
      for (int w = 0; w < NWG; ++w) {
        uint64_t* b = bars + w * S::NBAR_WG;
        for (int i = 0; i < 2; ++i) { mbar_init(&b[i], 1); mbar_init(&b[2 + i], 1); }         // q_full, q_empty
        for (int s = 0; s < ATTN7_ST; ++s) { mbar_init(&b[4 + s], 1); mbar_init(&b[4 + ATTN7_ST + s], 1); }
        mbar_init(&b[4 + 2 * ATTN7_ST + 0], 1);    // s_full (MMA commit)
        mbar_init(&b[4 + 2 * ATTN7_ST + 1], 128);  // s_free (softmax threads)
        mbar_init(&b[4 + 2 * ATTN7_ST + 2], 128);  // p_full (softmax threads)
        mbar_init(&b[4 + 2 * ATTN7_ST + 3], 1);    // o_full (MMA commit)
      }
      fence_barrier_init();
    }
    tmem_alloc<512>(tmem_slot);
  }
  __syncthreads();
  if (warp == 0) {  // inclusive scans of the item counts in processing order
    int run_f = 0, run_t = 0;
    for (int c0 = 0; c0 < T; c0 += 32) {
      const int i = c0 + lane;
      int vf = (i < T) ? pre_full[i + 1] : 0, vt = (i < T) ? pre_tail[i + 1] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int uf = __shfl_up_sync(0xffffffffu, vf, o), ut = __shfl_up_sync(0xffffffffu, vt, o);
        if (lane >= o) { vf += uf; vt += ut; }
      }
      if (i < T) { pre_full[i + 1] = run_f + vf; pre_tail[i + 1] = run_t + vt; }
      run_f += __shfl_sync(0xffffffffu, vf, 31);
      run_t += __shfl_sync(0xffffffffu, vt, 31);
    }
    if (lane == 0) { pre_full[0] = 0; pre_tail[0] = 0; s_nfull = run_f; }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int n_full = s_nfull;
  const int total = n_full + pre_tail[T];
  const int d = p.d_model;

  if (warp >= 4 * NWG) {
    // ================================================================ control warps
    // Registers: the two control warpgroups give theirs up so the softmax warpgroups can
    // hold a 64-column S row in registers (setmaxnreg; 4 * NWG softmax warps at SOFT_REGS).
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(CTRL_REGS));
    // warp-uniform for the compiler (a shuffle from lane 0), so the MMA warp's descriptor
    // arithmetic stays in uniform registers
    const int c = __shfl_sync(0xffffffffu, warp - 4 * NWG, 0);
    if (c < NWG) {
      // ---------------------------------------------------------- MMA warp of warpgroup w = c
      // One flat sequence over the warpgroup's sub-tiles g (all its items back to back):
      // QK(g) once K(g) is loaded and the softmax has loaded S(g-1) (s_free), then PV(g-1)
      // once P(g-1) is in TMEM (p_full); an item's first QK overlaps the previous item's last
      // softmax.  The whole warp runs the loop (item fields broadcast from lane 0); one elected
      // lane issues the MMAs and commits (a single-lane loop compiled every tcgen05.mma into a
      // register -> uniform-register waterfall costing ~150 cycles per instruction).
      const int w = c;
      uint64_t* b = bars + w * S::NBAR_WG;
      uint64_t* s_full = b + 4 + 2 * ATTN7_ST;
      const uint32_t tw = tmem + w * 128;
      constexpr uint32_t idesc_s = make_idesc_bf16(128, 64, 0);  // S_u = Q K_u^T (64 keys)
      constexpr uint32_t idesc_o = make_idesc_bf16(128, DH, 1);  // O += P_u V_u (V MN-major)
      int g = 0;
      bool pv_pending = false;
      int pv_ks = 0, pv_u = 0, pv_it = 0;
      (void)pv_it;
      for (int it = 0;; ++it) {
        const int slot = it & 1;
        mbar_poll<SLEEP_NS>(&b[slot], (it >> 1) & 1);  // q_full
        const volatile int* is = item_slot + (w * 2 + slot) * S::SLOT_INTS;
        if (__shfl_sync(0xffffffffu, is[0], 0) >= total) break;
        const int ns = __shfl_sync(0xffffffffu, (is[5] + 63) / 64, 0);
        const int n_keys = __shfl_sync(0xffffffffu, is[6], 0);  // PV covers the unmasked keys only
        const uint32_t qa = smem_u32(smem + S::q_off(w, slot));
        for (int u = 0; u < ns; ++u) {
          const int st = g % ATTN7_ST;
          mbar_poll<SLEEP_NS>(&b[4 + st], (g / ATTN7_ST) & 1);           // kv_full
          if (g > 0) mbar_poll<SLEEP_NS>(s_full + 1, (g - 1) & 1);       // s_free
          tc_fence_after();
#ifdef CFD_TRACE_MMA_PRE
          ATTN_TR(w, it, u, 6);  // trace experiment: QK(u) about to be issued
#endif
          const uint32_t ka = smem_u32(smem + S::k_off(w, st));
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < DH / 16; ++k)
              mma_ss(tw + S::S_COL, make_smem_desc(qa + k * 32, 16, 512, kLayoutSW64),
                     make_smem_desc(ka + k * 32, 16, 512, kLayoutSW64), idesc_s, k);
            mma_commit(s_full);
#ifndef CFD_TRACE_MMA_PRE
            ATTN_TR(w, it, u, 6);
#endif
            if (u + 1 == ns) mma_commit(&b[2 + slot]);  // the item's last QK: its Q slot is free
          }
          __syncwarp();
#ifdef CFD_TRACE_QK_LAT
          // trace experiment: when QK(u) completes (the warp waits for its own commit)
          mbar_spin(s_full, g & 1);
          if (lane == 0) ATTN_TR(w, it, u, 7);
#endif
          if (pv_pending) {
            const int sp = (g - 1) % ATTN7_ST;
            mbar_poll<SLEEP_NS>(s_full + 2, (g - 1) & 1);  // p_full
            tc_fence_after();
#ifdef CFD_TRACE_MMA_PRE
            ATTN_TR(w, pv_it, pv_u, 7);  // trace experiment: PV about to be issued
#endif
            const uint32_t va = smem_u32(smem + S::v_off(w, sp));
            if (elect_one()) {
              for (int k = 0; k < pv_ks; ++k)
                mma_ts(tw + S::O_COL, tw + S::P_COL + k * 8,
                       make_smem_desc(va + k * 16 * DH * 2, 4096, 512, kLayoutSW64), idesc_o, (pv_u | k) != 0);
              mma_commit(s_full + 3);              // o_full
              mma_commit(&b[4 + ATTN7_ST + sp]);  // kv_empty
#if !defined(CFD_TRACE_MMA_PRE) && !defined(CFD_TRACE_QK_LAT)
              ATTN_TR(w, pv_it, pv_u, 7);
#endif
            }
            __syncwarp();
          }
          pv_pending = true;
          pv_u = u;
          pv_it = it;
          pv_ks = (max(0, min(64, n_keys - u * 64)) + 15) / 16;
          ++g;
        }
      }
      if (pv_pending) {
        const int sp = (g - 1) % ATTN7_ST;
        mbar_poll<SLEEP_NS>(s_full + 2, (g - 1) & 1);
        tc_fence_after();
        const uint32_t va = smem_u32(smem + S::v_off(w, sp));
        if (elect_one()) {
          for (int k = 0; k < pv_ks; ++k)
            mma_ts(tw + S::O_COL, tw + S::P_COL + k * 8, make_smem_desc(va + k * 16 * DH * 2, 4096, 512, kLayoutSW64),
                   idesc_o, (pv_u | k) != 0);
          mma_commit(s_full + 3);
          mma_commit(&b[4 + ATTN7_ST + sp]);
        }
        __syncwarp();
      }
    } else if (c < 2 * NWG && lane == 0) {
      // ---------------------------------------------------------- producer of warpgroup w
      // Claims the warpgroup's items (static first item, then the work counter), publishes them
      // through item_slot + q_full (with the Q tile's bytes) and streams each item's 64-key K/V
      // sub-tiles into the warpgroup's ring as its stages free up.
      const int w = c - NWG;
      uint64_t* b = bars + w * S::NBAR_WG;
      int g = 0;
      if (p.stagger > 0 && w > 0) {  // de-phase the warpgroups' pipelines (option 5)
        const long long t_end = clock64() + (long long)w * p.stagger;
        while (clock64() < t_end) __nanosleep(64);
      }
      for (int it = 0;; ++it) {
        const int slot = it & 1;
        if (it >= 2) mbar_poll_slow(&b[2 + slot], ((it >> 1) - 1) & 1, p.producer_sleep);  // q_empty
        const int item = (it == 0 || !p.work_counter) ? (int)blockIdx.x + (it * NWG + w) * (int)gridDim.x
                                                       : NWG * (int)gridDim.x + atomicAdd(p.work_counter, 1);
        volatile int* is = item_slot + (w * 2 + slot) * S::SLOT_INTS;
        is[0] = item;
        if (item >= total) {
          mbar_arrive(&b[slot]);  // sentinel: q_full without bytes
          break;
        }
        int t, tile, h;
        decode_item7(order, pre_full, pre_tail, T, nh, n_full, item, t, tile, h, p.cu_seqlens);
        const int seq0 = __ldg(p.cu_seqlens + t);
        const int N = __ldg(p.cu_seqlens + t + 1) - seq0;
        const int ns = (N + 63) / 64;
        is[1] = t;
        is[2] = tile;
        is[3] = h;
        is[4] = seq0;
        is[5] = N;
        const int n_keys = p.kv_len ? __ldg(p.kv_len + t) : N;
        is[6] = n_keys;
        mbar_expect_tx(&b[slot], S::Q_BYTES);
        // the Q tile as four 32-row boxes: slot quarter j takes rows (j mod 4/rep) * 32 of the tile,
        // i.e. a split tail tile (<= 64 / <= 32 rows) lands rep = 2 / 4 times
        const int q_real = n_keys - tile * 128;  // real query rows of the tile (the rest: next task / pad)
        const int nrb = (q_real > 0 && q_real <= SPLIT_ROWS) ? 4 / SPLIT_REP : 4;  // = 4 / rep
#pragma unroll
        for (int j = 0; j < 4; ++j)
          tma_load_2d(smem + S::q_off(w, slot) + j * (S::SUB_BYTES / 2), &tmQ32, &b[slot], h * DH,
                      seq0 + tile * 128 + (j % nrb) * 32);
        for (int u = 0; u < ns; ++u, ++g) {
          const int st = g % ATTN7_ST;
          if (g >= ATTN7_ST) mbar_poll_slow(&b[4 + ATTN7_ST + st], ((g / ATTN7_ST) - 1) & 1, p.producer_sleep);  // kv_empty
          mbar_expect_tx(&b[4 + st], 2 * S::SUB_BYTES);
          tma_load_2d(smem + S::k_off(w, st), &tmQKV, &b[4 + st], d + h * DH, seq0 + u * 64);
          tma_load_2d(smem + S::v_off(w, st), &tmQKV, &b[4 + st], 2 * d + h * DH, seq0 + u * 64);
        }
      }
      if (p.work_counter) {
        // self-resetting claim counter: the last producer of the grid to finish resets
        // [claims, finished] for the next launch on this workspace
        __threadfence();
        if (atomicAdd(p.work_counter + 1, 1) == NWG * (int)gridDim.x - 1) {
          p.work_counter[0] = 0;
          p.work_counter[1] = 0;
          __threadfence();
        }
      }
    }
  } else {
    // ================================================================ softmax warpgroups
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(SOFT_REGS));
    const int wg = warp >> 2;
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;
    uint64_t* b = bars + wg * S::NBAR_WG;
    uint64_t* q_full = b;
    uint64_t* s_full = b + 4 + 2 * ATTN7_ST;
    uint64_t* s_free = s_full + 1;
    uint64_t* p_full = s_full + 2;
    uint64_t* o_full = s_full + 3;
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    const uint32_t s_base = tmem + lane_off + wg * 128 + S::S_COL;
    const uint32_t p_addr = tmem + lane_off + wg * 128 + S::P_COL;
    const uint32_t o_addr = tmem + lane_off + wg * 128 + S::O_COL;
    const float c = p.scale_log2;
    uint32_t s_cnt = 0, o_cnt = 0;
    const bool tr = quarter == 0 && lane == 0;
    (void)tr;
    for (int it = 0;; ++it) {
      mbar_wait(&q_full[it & 1], (it >> 1) & 1);
      const volatile int* is = item_slot + (wg * 2 + (it & 1)) * S::SLOT_INTS;
      if (is[0] >= total) break;
      const int tile = is[2], h = is[3], seq0 = is[4], N = is[5];
      const int nsub = (N + 63) / 64;
      const int q_valid = N - tile * 128;
      // split tail tile (<= SPLIT_ROWS real rows): the producer loaded its rows rep times over the lane
      // quarters; replica rr (quarters rr*(4/rep) + rb) takes key columns [rr*cw, rr*cw + cw) of
      // every 64-key sub-tile, so all four warps share the tail's exponentials; the replicas'
      // (m, l, O) are merged at the end of the item
      const int n_keys = is[6];  // keys >= n_keys are masked (padded batch)
      // split by the real rows (n_keys = N, or kv_len in the padded batch, whose tail tile must take
      // the same path as the varlen one: rows equal bit for bit)
      const int q_real = n_keys - tile * 128;
      const bool split = q_real > 0 && q_real <= SPLIT_ROWS;
      const bool active = split || quarter * 32 < q_valid;
      float m_run = -INFINITY, l_run = 0.f;
      if (split) {  // the other replicas' P columns stay zero for the whole item
        uint32_t z[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) z[i] = 0u;
        tmem_st16(p_addr, z);
        tmem_st16(p_addr + 16, z);
      }
      // PV(u-1) done: P may be overwritten and O rescaled by alpha (rows whose max moved)
      const auto wait_o_rescale = [&](bool upd, float alpha) {
        mbar_wait(o_full, o_cnt & 1);
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
      };
      for (int u = 0; u < nsub; ++u) {
        mbar_wait(s_full, s_cnt & 1);
        ++s_cnt;
        tc_fence_after();
        if (tr) ATTN_TR(wg, it, u, 0);
        // P(u-1) is published here rather than at the end of sub-tile u-1: the wait for its
        // TMEM stores overlaps the S(u) load (PV(u-1) is not needed before P(u) is stored)
        const auto publish_prev_p = [&]() {
          if (u > 0) {
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(p_full);
          }
        };
        if (active && u * 64 >= n_keys) {
          // a sub-tile of pad keys only (padded batch): no exponentials, and the MMA warp
          // issues no PV for it (its k-steps cover the unmasked keys only)
          publish_prev_p();
          tc_fence_before();
          mbar_arrive(s_free);
          if (u > 0) {
            mbar_wait(o_full, o_cnt & 1);
            ++o_cnt;
          }
        } else if (split) {
          // split tail tile (all four warps active): this warp's cw key columns of the sub-tile
          constexpr int rep = SPLIT_REP, cw = 64 / rep;
          const int rr = quarter / (4 / rep);
          const int valid = min(64, n_keys - u * 64);
          const int c0 = rr * cw;
          uint32_t sr[32];
          if constexpr (rep == 2) tmem_ld32(s_base + c0, *reinterpret_cast<uint32_t(*)[32]>(sr));
          else tmem_ld16(s_base + c0, *reinterpret_cast<uint32_t(*)[16]>(sr));
          publish_prev_p();
          tmem_wait_ld();
          tc_fence_before();
          mbar_arrive(s_free);
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (i >= cw || c0 + i >= valid) sr[i] = __float_as_uint(-INFINITY);
          float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            m0 = fmax3(m0, __uint_as_float(sr[i]), __uint_as_float(sr[i + 1]));
            m1 = fmax3(m1, __uint_as_float(sr[i + 2]), __uint_as_float(sr[i + 3]));
          }
          const float m_cand = fmaxf(m0, m1) * c;
          // lazy rescale (R23); a warp may see only masked keys so far (m_cand = m_run = -inf):
          // it keeps m_run = -inf and exponentiates against 0 (p = 0, no inf - inf)
          const bool upd = (m_run == -INFINITY) ? (m_cand != -INFINITY) : (m_cand > m_run + 8.0f);
          const float alpha = upd ? ((m_run == -INFINITY) ? 0.f : ex2_approx(m_run - m_cand)) : 1.f;
          if (upd) m_run = m_cand;
          const float neg = (m_run == -INFINITY) ? 0.f : -m_run;
          float sum0 = 0.f, sum1 = 0.f;
          if constexpr (rep == 2) exp_chunk<0, 16>(sr, c, neg, sum0, sum1);
          else exp_chunk<0, 8>(sr, c, neg, sum0, sum1);
          l_run = l_run * alpha + (sum0 + sum1);
          if (u > 0) wait_o_rescale(upd, alpha);
          if constexpr (rep == 2) tmem_st16(p_addr + rr * 16, *reinterpret_cast<const uint32_t(*)[16]>(sr));
          else tmem_st8(p_addr + rr * 8, *reinterpret_cast<const uint32_t(*)[8]>(sr));
        } else if (active) {
          const int valid = min(64, n_keys - u * 64);
          uint32_t sr[64];
          float sum0 = 0.f, sum1 = 0.f, sum2 = 0.f, sum3 = 0.f;
          float alpha = 1.f;
          bool upd = false, done = false, published = false;
          if (u > 0 && valid == 64) {
            // Speculative fast path: exponentiate against the current reference max m_run (it
            // moves only when a row max grows by > 2^8, reading R23), so the exps of the first 32
            // columns run while the second 32 load and the row max is only checked afterwards.
            // S stays in TMEM (s_free not yet arrived) for the rare warp that must redo.
            tmem_ld32(s_base, *reinterpret_cast<uint32_t(*)[32]>(sr));
            publish_prev_p();
            published = true;
            tmem_wait_ld();
            tmem_ld32(s_base + 32, *reinterpret_cast<uint32_t(*)[32]>(sr + 32));
            if (tr) ATTN_TR(wg, it, u, 1);
            float ma = -INFINITY, mb = -INFINITY;
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              ma = fmax3(ma, __uint_as_float(sr[i]), __uint_as_float(sr[i + 1]));
              mb = fmax3(mb, __uint_as_float(sr[i + 2]), __uint_as_float(sr[i + 3]));
            }
            exp_chunk<NPP>(sr, c, -m_run, sum0, sum1);
            tmem_wait_ld();
#pragma unroll
            for (int i = 32; i < 64; i += 4) {
              ma = fmax3(ma, __uint_as_float(sr[i]), __uint_as_float(sr[i + 1]));
              mb = fmax3(mb, __uint_as_float(sr[i + 2]), __uint_as_float(sr[i + 3]));
            }
            const float m_cand = fmaxf(ma, mb) * c;  // the same row max as the general path
            if (tr) ATTN_TR(wg, it, u, 2);
            if (!__any_sync(0xffffffffu, m_cand > m_run + 8.0f)) {
              exp_chunk<NPP>(sr + 32, c, -m_run, sum2, sum3);
              tc_fence_before();
              mbar_arrive(s_free);  // S may now be overwritten by QK(u+1)
              done = true;
            } else {
              sum0 = sum1 = 0.f;
            }
          }
          if (!done) {
            tmem_ld32(s_base, *reinterpret_cast<uint32_t(*)[32]>(sr));
            if (valid > 32) tmem_ld32(s_base + 32, *reinterpret_cast<uint32_t(*)[32]>(sr + 32));
            if (!published) publish_prev_p();
            tmem_wait_ld();
            if (tr) ATTN_TR(wg, it, u, 1);
            tc_fence_before();
            mbar_arrive(s_free);  // S may now be overwritten by QK(u+1)
            if (valid < 64) {
#pragma unroll
              for (int i = 0; i < 64; ++i)
                if (i >= valid) sr[i] = __float_as_uint(-INFINITY);
            }
            float m0 = -INFINITY, m1 = -INFINITY, m2 = -INFINITY, m3 = -INFINITY;
#pragma unroll
            for (int i = 0; i < 64; i += 8) {
              m0 = fmax3(m0, __uint_as_float(sr[i]), __uint_as_float(sr[i + 1]));
              m1 = fmax3(m1, __uint_as_float(sr[i + 2]), __uint_as_float(sr[i + 3]));
              m2 = fmax3(m2, __uint_as_float(sr[i + 4]), __uint_as_float(sr[i + 5]));
              m3 = fmax3(m3, __uint_as_float(sr[i + 6]), __uint_as_float(sr[i + 7]));
            }
            const float m_cand = fmax3(m0, m1, fmaxf(m2, m3)) * c;
            if (tr) ATTN_TR(wg, it, u, 2);
            // lazy rescale (reading R23): move the reference max only when it grows by > 2^8
            upd = (m_run == -INFINITY) || (m_cand > m_run + 8.0f);
            alpha = upd ? ((m_run == -INFINITY) ? 0.f : ex2_approx(m_run - m_cand)) : 1.f;
            if (upd) m_run = m_cand;
            const float neg = -m_run;
            if (valid == 64) {
              exp_chunk<NPP>(sr, c, neg, sum0, sum1);
              exp_chunk<NPP>(sr + 32, c, neg, sum2, sum3);
            } else {
              exp_chunk<0>(sr, c, neg, sum0, sum1);
              if (valid > 32) exp_chunk<0>(sr + 32, c, neg, sum2, sum3);
            }
          }
          l_run = l_run * alpha + ((sum0 + sum1) + (sum2 + sum3));
          if (tr) ATTN_TR(wg, it, u, 3);
          if (u > 0) wait_o_rescale(upd, alpha);
          if (tr) ATTN_TR(wg, it, u, 4);
          tmem_st16(p_addr, *reinterpret_cast<const uint32_t(*)[16]>(sr));
          if (valid > 32) tmem_st16(p_addr + 16, *reinterpret_cast<const uint32_t(*)[16]>(sr + 32));
        } else {
          // padding-only warp of a tail tile: keeps the barrier phases in step
          publish_prev_p();
          mbar_arrive(s_free);
          if (u > 0) {
            mbar_wait(o_full, o_cnt & 1);
            ++o_cnt;
          }
        }
        if (tr) ATTN_TR(wg, it, u, 5);
      }
      tmem_wait_st();  // the item's last P
      tc_fence_before();
      mbar_arrive(p_full);
      mbar_wait(o_full, o_cnt & 1);
      ++o_cnt;
      tc_fence_after();
      if (split) {
        constexpr int rep = SPLIT_REP;
        const int rb = quarter % (4 / rep), rr = quarter / (4 / rep);
        // merge the replicas of the split tail through shared memory, in a fixed order:
        // O = sum_j 2^(m_j - M) O_j / sum_j 2^(m_j - M) l_j over the replicas j of a row
        float* ml = reinterpret_cast<float*>(smem + S::MERGE_OFF) + wg * S::MERGE_WG_FLOATS;  // [4][32][2]
        float* acc = ml + 4 * 32 * 2;                                                       // [32][33]
        uint32_t o[32];
        tmem_ld32(o_addr, o);
        ml[(quarter * 32 + lane) * 2 + 0] = m_run;
        ml[(quarter * 32 + lane) * 2 + 1] = l_run;
        tmem_wait_ld();
        named_bar_sync(1 + wg, 128);
        float M = -INFINITY;
        for (int j = 0; j < rep; ++j) M = fmaxf(M, ml[((j * (4 / rep) + rb) * 32 + lane) * 2]);
        float L = 0.f;
        for (int j = 0; j < rep; ++j) {
          const float mj = ml[((j * (4 / rep) + rb) * 32 + lane) * 2];
          L += (mj == -INFINITY ? 0.f : ex2_approx(mj - M)) * ml[((j * (4 / rep) + rb) * 32 + lane) * 2 + 1];
        }
        const float wgt = (m_run == -INFINITY ? 0.f : ex2_approx(m_run - M)) / L;
        // the four warps in turn (row block rb, replica rr): first replica writes, the others
        // add, the last one stores the bf16 rows and the LSE
        for (int k = 0; k < 4; ++k) {
          if (k == rb * rep + rr) {
            float* a = acc + lane * 33;
            if (rr < rep - 1) {
#pragma unroll
              for (int i = 0; i < DH; ++i) a[i] = (rr ? a[i] : 0.f) + __uint_as_float(o[i]) * wgt;
            } else {
              const int rrow = rb * 32 + lane;
              if (rrow < q_valid) {
                uint32_t ob[DH / 2];
#pragma unroll
                for (int i = 0; i < DH / 2; ++i)
                  ob[i] = pack_bf16x2(a[2 * i] + __uint_as_float(o[2 * i]) * wgt,
                                      a[2 * i + 1] + __uint_as_float(o[2 * i + 1]) * wgt);
                const int row = seq0 + tile * 128 + rrow;
                uint4* dst = reinterpret_cast<uint4*>(p.out + (size_t)row * d + h * DH);
#pragma unroll
                for (int i = 0; i < DH / 8; ++i)
                  dst[i] = make_uint4(ob[4 * i], ob[4 * i + 1], ob[4 * i + 2], ob[4 * i + 3]);
                if (p.lse) p.lse[(size_t)h * p.lse_ld + row] = (M + __log2f(L)) * 0.69314718055994531f;
              }
            }
          }
          if (k < 3) named_bar_sync(1 + wg, 128);
        }
      } else if (active) {
        uint32_t o[32];
        tmem_ld32(o_addr, o);
        tmem_wait_ld();
        if (r < q_valid) {
          const float inv = 1.f / l_run;
          uint32_t ob[DH / 2];
#pragma unroll
          for (int i = 0; i < DH / 2; ++i)
            ob[i] = pack_bf16x2(__uint_as_float(o[2 * i]) * inv, __uint_as_float(o[2 * i + 1]) * inv);
          const int row = seq0 + tile * 128 + r;
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
  if (warp == kMmaWarp) tmem_dealloc<512>(tmem);
}

}  // namespace cfd
