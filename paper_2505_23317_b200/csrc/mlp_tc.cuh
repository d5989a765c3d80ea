// mlp_tc.cuh — fused encoder MLP block on tcgen05 (reading R4):
//
//   x += GELU(h W_1^T + b_1) W_2^T + b_2,     h = LN2(x) (bf16, from the O-projection epilogue)
//   (+ optionally hn = LN1_next(x) for the next layer, as EPI_F32_RESID_LN does)
//
// One persistent CTA per SM walks 128-row tiles; the hidden dimension F is processed in
// 128-column chunks j:
//   MMA1(j):  acc1 (TMEM, 128 cols) = h . W1[j]^T     (K = d; A = h from TMEM: "TS" form)
//   GELU(j):  8 epilogue warps: acc1 + b1 -> GELU -> bf16 -> shared memory H[j&1], written
//             directly in the 128B-swizzled K-major layout the tensor core reads
//   MMA2(j):  acc2 (TMEM, 256 cols) += H[j&1] . W2[:, j]^T  (K = 128, N = 256)
// issued as MMA1(j+1) before MMA2(j) so GELU(j) overlaps the tensor core (acc1 is released
// as soon as the epilogue has moved it into registers).  The hidden activations never leave
// the SM.
//
// Resource plan (measured, profiles/r1_tc_micro.txt): the tensor core reads shared memory at
// 128 B/clk/SM, which an SS-form M=128 N=128 MMA alone saturates.  Keeping the h tile in
// TMEM (A operand of MMA1) and issuing MMA2 as one N=256 MMA cuts the per-chunk smem reads
// to W1 64 KB + H 32 KB + W2 64 KB.  TMEM: h tile [0,128) (bf16 pairs), acc1 [128,256),
// acc2 [256,512).  Everything that arrives by TMA — the h tile (4 pieces) and the weights —
// streams through ONE ring of eight 16 KB slots in consumption order: per tile
//   h k-blocks 0..3 | W1(0) k-blocks 0..3 | { W1(j) k-blocks 0..3, W2(j-1) } j=1..n-1 | W2(n-1)
// with W2(j) = (k-block 0: rows 0-127, 128-255), (k-block 1: rows 0-127, 128-255), so every
// group is 4 slots and a W2 k-block always occupies two adjacent slots (one 256-row operand).
// The 128 KB ring keeps ~2 operands of loads in flight ahead of the MMAs.  The epilogue warps
// consume the h pieces (smem -> TMEM copy), the MMA warp everything else.
//
// OPJ (fused O-projection, single-CTA kernel): the tile starts from the attention output o
// instead of h: MMA_o: acc2 = o . W_o^T (A and W_o through the ring), then the epilogue
// warps form x1 = x + acc2 + b_o (x staged by TMA, x1 stored by TMA) and write
// h = LN2(x1) straight into the TMEM h tile (bf16 pairs), so the O-projection launch, the
// LN2 round trip through memory and the h load disappear.  Ring per tile:
//   o0 o1 | Wo0 (2 slots: rows 0-127, 128-255) | Wo1 | o2 o3 | Wo2 | Wo3 | W1(0) | ...
// (12 slots; every W_o pair starts on an even slot so it is one contiguous 256-row operand).
// acc2 is used twice per tile (acc_o, then the MLP2 accumulation): a2_empty completes twice.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "ptx.cuh"
#include "gemm_tc.cuh"

namespace cfd {

struct MlpParams {
  int M;                 // rows when m_dev == nullptr
  const int* m_dev;
  int F;                 // hidden width (multiple of 128, <= GEMM_MAX_N)
  const float* b1;       // [F]
  const float* b2;       // [D]
  float* x;              // residual [*, D] fp32 (in / out)
  const float* ln_g;     // next LayerNorm (nullptr: none)
  const float* ln_b;
  __nv_bfloat16* ln_out; // [ln_cap, D]
  int ln_cap;
  float ln_eps;
  int staged;            // 1: residual (+LN) epilogue staged through smem with TMA (tmX / tmLN valid)
  // OPJ only: O-projection bias and this layer's LN2
  const float* bo;
  const float* ln2_g;
  const float* ln2_b;
  // OPJ only: keep x1 = x + o W_o + b_o in the acc2 TMEM columns instead of storing it; the
  // MLP's MMA2s then accumulate onto it and the final epilogue computes x2 = acc2 + b2 without
  // reading x (saves the x1 store + reload: 2 x 128 KB per tile)
  int keep_x1;
};

constexpr int MLP_THREADS = 320;  // TMA warp, MMA warp, 8 epilogue warps

// Debug-library pipeline trace (-DCFD_TRACE, read by cfdx_mlp_trace): per CTA 96 words,
// tiles it = 0, 1 at word it * 48 + event, clock64() of
//   0 producer issues the tile's first h piece     1 epilogue: last h piece landed
//   2 epilogue: h tile in TMEM (ht_full arrive)     3 MMA: ht_full observed
//   4+j MMA: MMA1(j) issue start (a1_empty passed)  12+j MMA: MMA2(j) issue start (h_full passed)
//   20+j epilogue: a1_full(j) observed              28+j epilogue: GELU(j) written (h_full arrive)
//   36 epilogue: final epilogue starts (before its a2_full wait)   37 epilogue: tile done
// (j < 8; epilogue events from epilogue thread 0), word 47 of tile 0 = kernel start.
constexpr int MLP_TRACE_WORDS = 148 * 96;
#ifdef CFD_TRACE
__device__ unsigned long long g_mlp_trace[MLP_TRACE_WORDS];
#define MLP_TR(it_, ev_)                                                                   \
  do {                                                                                    \
    if ((it_) < 2 && blockIdx.x < 148) g_mlp_trace[blockIdx.x * 96 + (it_) * 48 + (ev_)] = clock64(); \
  } while (0)
#else
#define MLP_TR(it_, ev_) do { } while (0)
#endif
constexpr int MLP_SLOTS = 8;  // with x1 kept in TMEM (option 19) the third x staging buffer is worth less
                              // than two more ring slots (MLP launch 52.7 -> 52.2 us; before: 6 slots)

template <int D>
struct MlpSmem {
  static_assert(D == 256, "fused MLP is laid out for d = 256 (acc2 = 256 TMEM columns)");
  static constexpr int H_BYTES = 128 * 128 * 2;           // 32 KB: GELU chunk, 2 k-blocks
  static constexpr int SLOT_BYTES = 16384;                // 128 rows x 64 bf16 (one SW128 k-block)
  static constexpr int H_OFF = 0;                         // [2]
  static constexpr int W_OFF = H_OFF + 2 * H_BYTES;       // [MLP_SLOTS]
  static constexpr int BAR_OFF = W_OFF + MLP_SLOTS * SLOT_BYTES;
  static constexpr int STATS_OFF = BAR_OFF + 512;         // float2 [2][128]
  static constexpr int PAR_OFF = STATS_OFF + 2 * 128 * 8; // b1 [F] | b2 [D] | g [D] | b [D]
  // staged final epilogue: each epilogue warp's x staging buffers are its own 4 KB slices of
  // H[0] / H[1] (the slices it writes during GELU, free once the last MMA2 has committed);
  // one 2 KB LN output buffer per warp lives here
  // ... | b_o [D] | ln2 g [D] | ln2 b [D] (OPJ)
  static constexpr int LNSTG_OFF = ((PAR_OFF + (GEMM_MAX_N + 6 * D) * 4 + 1023) / 1024) * 1024;
  static constexpr int XSTG_OFF = LNSTG_OFF + 8 * 2048;    // end of the LN staging (no third x buffer)
  static constexpr int TOTAL = 1024 + XSTG_OFF;
};

// CL = 2: CTA-pair kernel (2-CTA clusters, tcgen05 cta_group::2).  The single-CTA kernel is
// bound by shared-memory ingress of the weight stream (~40 B/clk/SM for 1 MB per 128-row
// tile, profiles/r1_mlp_trace.txt; multicasting the same bytes into both CTAs did not help).
// Here the leader CTA issues M = 256 MMAs for the pair's two tiles: each CTA keeps its own
// 128 rows (h in its TMEM, H in its smem, acc1/acc2 in its TMEM) and holds HALF of each
// weight operand — W1 chunk rows [64 r, 64 r + 64), W2 output rows [128 r, 128 r + 128) for
// rank r — so per-SM weight ingress halves.  Ring: per tile h(4 local) | W1(0)(2) |
// {W1(j)(2), W2(j-1)(2)} | W2(n-1)(2), each W1 slot = two 64-row k-blocks.  Weight halves are
// pair-TMA loads completing on the leader's w_full (expecting both halves); the leader's
// commits are multicast to both CTAs (w_empty, a1_full, h_empty, a2_full); the epilogues of
// both CTAs arrive on the leader's ht_full / a1_empty / h_full / a2_empty.  The pair walks
// tile pairs in lockstep; an odd last tile leaves CTA 1 a masked "ghost" tile.
template <int D, int CL, bool OPJ = false>
__global__ void __launch_bounds__(MLP_THREADS, 1)
    mlp_tc_kernel(const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmW1,
                  const __grid_constant__ CUtensorMap tmW2, const MlpParams p,
                  const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmLN,
                  const __grid_constant__ CUtensorMap tmWo) {
  using S = MlpSmem<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps the shared space
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::BAR_OFF);
  uint64_t* w_full = bars;                   // [MLP_SLOTS]
  uint64_t* w_empty = w_full + MLP_SLOTS;    // [MLP_SLOTS]
  uint64_t* ht_full = w_empty + MLP_SLOTS;   // h tile copied into TMEM
  uint64_t* a1_full = ht_full + 1;
  uint64_t* a1_empty = a1_full + 1;
  uint64_t* h_full = a1_empty + 1;           // [2 buffers][2 k-blocks]: H[b] k-block kb written
  uint64_t* h_empty = h_full + 4;            // [2]
  uint64_t* a2_full = h_empty + 2;
  uint64_t* a2_empty = a2_full + 1;
  uint64_t* xbar = a2_empty + 1;             // [8 warps][3] staged-epilogue TMA loads
  uint64_t* ao_full = xbar + 24;             // OPJ: acc_o = o . W_o^T complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ao_full + 1);
  float2* ln_stats = reinterpret_cast<float2*>(smem + S::STATS_OFF);
  float* b1_s = reinterpret_cast<float*>(smem + S::PAR_OFF);
  float* b2_s = b1_s + GEMM_MAX_N;
  float* lng_s = b2_s + D;
  float* lnb_s = lng_s + D;
  float* bo_s = lnb_s + D;     // OPJ
  float* g2_s = bo_s + D;
  float* b2ln_s = g2_s + D;

  const int warp = warp_id(), lane = lane_id();
  const int M = p.m_dev ? __ldg(p.m_dev) : p.M;
  const bool do_ln = p.ln_g != nullptr;
  const int m_tiles = ((do_ln ? pad_rows(M, p.ln_cap) : M) + 127) / 128;
  const int n_chunks = p.F / 128;
  constexpr int KB = D / 64;                 // k-blocks of the h tile (= its ring pieces)
  constexpr bool PAIR = (CL == 2);
  // OPJ ring per tile: single CTA o0 o1 Wo0(2 slots) Wo1(2) o2 o3 Wo2(2) Wo3(2) = 12 slots;
  // PAIR o0 o1 Wo0 Wo1 o2 o3 Wo2 Wo3 = 8 slots (a W_o k-block slot holds this CTA's 128 output
  // rows: the pair MMA takes B columns [0, 128) from CTA 0 and [128, 256) from CTA 1)
  const int slots_per_tile = (OPJ ? (PAIR ? 2 * KB : 3 * KB) : KB) + (PAIR ? 4 : 8) * n_chunks;
  // OPJ ring offsets of k-block kb within a tile: o piece / (first) slot of W_o
  auto opj_o = [](int kb) { return PAIR ? ((kb < 2) ? kb : 2 + kb) : ((kb < 2) ? kb : 4 + kb); };   // 0 1 4 5 | 0 1 6 7
  auto opj_w = [](int kb) { return PAIR ? ((kb < 2) ? 2 + kb : 4 + kb) : ((kb < 2) ? 2 + 2 * kb : 4 + 2 * kb); };
  const int rank = (CL == 2) ? static_cast<int>(cluster_ctarank()) : 0;
  const int t_first = (CL == 2) ? 2 * static_cast<int>(cluster_id_x()) + rank : static_cast<int>(blockIdx.x);
  const int t_step = (CL == 2) ? 2 * static_cast<int>(nclusters_x()) : static_cast<int>(gridDim.x);
  // tile loop: CL == 2 keeps both CTAs of a pair in step (tile >= m_tiles: ghost tile)
#define MLP_TILES(tile_) for (int tile_ = t_first; (tile_) - rank < m_tiles; tile_ += t_step)

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmH);
    tma_prefetch(&tmW1);
    tma_prefetch(&tmW2);
    if constexpr (OPJ) tma_prefetch(&tmWo);
    for (int i = 0; i < MLP_SLOTS; ++i) { mbar_init(&w_full[i], 1); mbar_init(&w_empty[i], 1); }
    mbar_init(ht_full, CL);
    mbar_init(a1_full, 1);
    mbar_init(a1_empty, 8 * CL);
    for (int i = 0; i < 4; ++i) mbar_init(&h_full[i], 8 * CL);
    for (int i = 0; i < 2; ++i) mbar_init(&h_empty[i], 1);
    mbar_init(a2_full, 1);
    mbar_init(a2_empty, 8 * CL);
    for (int i = 0; i < 24; ++i) mbar_init(&xbar[i], 1);
    mbar_init(ao_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) {
    if constexpr (PAIR) tmem_alloc_2sm<512>(tmem_slot);
    else tmem_alloc<512>(tmem_slot);
  }
#ifdef CFD_TRACE
  if (threadIdx.x < 96 && blockIdx.x < 148) g_mlp_trace[blockIdx.x * 96 + threadIdx.x] = 0;
#endif
  tc_fence_before();
  if constexpr (CL == 2) cluster_sync();  // peer barriers initialised before any multicast / remote arrive
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr uint32_t HT = 0, ACC1 = 128, ACC2 = 256;
  if (threadIdx.x == 0) MLP_TR(0, 47);
  // arrive on a barrier the leader CTA waits on (pair epilogue -> leader MMA warp)
  auto arrive_leader = [&](uint64_t* bar) {
    if (PAIR && rank != 0) mbar_arrive_cluster(bar, 0);
    else mbar_arrive(bar);
  };

  if (warp == 0) {
    // ============================================================ TMA producer
    if (lane == 0) {
      uint32_t pos = 0;  // ring position (slot = pos % MLP_SLOTS, phase = (pos / MLP_SLOTS) & 1)
      auto load = [&](const CUtensorMap* tm, int x, int y) {  // local piece (h; all pieces if !PAIR)
        const int slot = pos % MLP_SLOTS;
        mbar_wait(&w_empty[slot], ((pos / MLP_SLOTS) & 1) ^ 1);
        mbar_expect_tx(&w_full[slot], S::SLOT_BYTES);
        tma_load_2d(smem + S::W_OFF + slot * S::SLOT_BYTES, tm, &w_full[slot], x, y);
        ++pos;
      };
      // PAIR: this CTA's half of a weight slot (nbox boxes of 16 KB / nbox), completing on the
      // leader's w_full, which expects both halves
      auto load_half = [&](const CUtensorMap* tm, int x0, int y0, int x1, int y1, int nbox) {
        const int slot = pos % MLP_SLOTS;
        mbar_wait(&w_empty[slot], ((pos / MLP_SLOTS) & 1) ^ 1);
        if (rank == 0) mbar_expect_tx(&w_full[slot], 2 * S::SLOT_BYTES);
        const uint32_t lb = mapa_u32(&w_full[slot], 0);
        uint8_t* dst = smem + S::W_OFF + slot * S::SLOT_BYTES;
        tma_load_2d_2sm(dst, tm, lb, x0, y0);
        if (nbox == 2) tma_load_2d_2sm(dst + S::SLOT_BYTES / 2, tm, lb, x1, y1);
        ++pos;
      };
      auto load_w1 = [&](int j) {
        if constexpr (PAIR) {  // rows [128 j + 64 rank, +64), k-blocks (0,1) and (2,3): tmW1 box = 64 rows
          for (int q = 0; q < KB / 2; ++q)
            load_half(&tmW1, (2 * q) * 64, 128 * j + 64 * rank, (2 * q + 1) * 64, 128 * j + 64 * rank, 2);
        } else {
          for (int kb = 0; kb < KB; ++kb) load(&tmW1, kb * 64, 128 * j);
        }
      };
      auto load_w2 = [&](int j) {  // W2 (K-major [D, F]) k columns [128j, 128j+128)
        if constexpr (PAIR) {  // output rows [128 rank, +128)
          for (int kb = 0; kb < 2; ++kb) load_half(&tmW2, 128 * j + 64 * kb, 128 * rank, 0, 0, 1);
        } else {
          for (int kb = 0; kb < 2; ++kb)
            for (int nh = 0; nh < D / 128; ++nh) load(&tmW2, 128 * j + 64 * kb, 128 * nh);
        }
      };
      int pit = 0;
      MLP_TILES(tile) {
        MLP_TR(pit, 0);
        ++pit;
        if constexpr (OPJ && PAIR) {  // o pieces are the pair MMA's A rows: pair loads completing on the leader
          for (int g2 = 0; g2 < 2; ++g2) {
            for (int kb = 2 * g2; kb < 2 * g2 + 2; ++kb) load_half(&tmH, kb * 64, tile * 128, 0, 0, 1);
            for (int kb = 2 * g2; kb < 2 * g2 + 2; ++kb) load_half(&tmWo, kb * 64, 128 * rank, 0, 0, 1);
          }
        } else if constexpr (OPJ) {  // o0 o1 Wo0 Wo1 o2 o3 Wo2 Wo3 (W_o k-block = 2 slots of 128 rows)
          for (int g2 = 0; g2 < 2; ++g2) {
            for (int kb = 2 * g2; kb < 2 * g2 + 2; ++kb) load(&tmH, kb * 64, tile * 128);
            for (int kb = 2 * g2; kb < 2 * g2 + 2; ++kb)
              for (int nh = 0; nh < D / 128; ++nh) load(&tmWo, kb * 64, 128 * nh);
          }
        } else {
          for (int kb = 0; kb < KB; ++kb) load(&tmH, kb * 64, tile * 128);
        }
        load_w1(0);
        for (int j = 1; j < n_chunks; ++j) {
          load_w1(j);
          load_w2(j - 1);
        }
        load_w2(n_chunks - 1);
      }
    }
  } else if (warp == 1) {
    // ============================================================ MMA issuer (PAIR: leader only)
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idesc1 = make_idesc_bf16(128 * CL, 128, 0);
      constexpr uint32_t idesc2 = make_idesc_bf16(128 * CL, D, 0);
      auto commit = [&](uint64_t* bar) {  // PAIR: arrive in both CTAs
        if constexpr (PAIR) mma_commit_2sm(bar, 0x3);
        else mma_commit(bar);
      };
      int it = 0;
      uint32_t pos = 0;
      uint32_t a1_ph = 0, h_ph = 0, a2_cnt = 0;  // bit b: phase of barrier [b]
      auto take = [&]() -> uint32_t {
        const int slot = pos % MLP_SLOTS;
        mbar_wait(&w_full[slot], (pos / MLP_SLOTS) & 1);
        return smem_u32(smem + S::W_OFF + slot * S::SLOT_BYTES);
      };
      auto give = [&]() {
        commit(&w_empty[pos % MLP_SLOTS]);
        ++pos;
      };
      auto mma1 = [&](int j) {
        mbar_wait(a1_empty, a1_ph ^ 1);
        a1_ph ^= 1;
        if (j < 8) MLP_TR(it, 4 + j);
        if constexpr (PAIR) {
          for (int q = 0; q < KB / 2; ++q) {
            const uint32_t w = take();  // k-blocks 2q, 2q+1 of this CTA's 64 rows (8 KB each)
            tc_fence_after();
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
              for (int k = 0; k < 4; ++k)
                mma_ts_2sm(tmem + ACC1, tmem + HT + (2 * q + i) * 32 + k * 8,
                           make_smem_desc(w + i * (S::SLOT_BYTES / 2) + k * 32, 16, 1024, kLayoutSW128), idesc1,
                           (q | i | k) != 0);
            give();
          }
        } else {
          for (int kb = 0; kb < KB; ++kb) {
            const uint32_t w = take();
            tc_fence_after();
#pragma unroll
            for (int k = 0; k < 4; ++k)
              mma_ts(tmem + ACC1, tmem + HT + kb * 32 + k * 8, make_smem_desc(w + k * 32, 16, 1024, kLayoutSW128),
                     idesc1, (kb | k) != 0);
            give();
          }
        }
        commit(a1_full);
      };
      auto mma2 = [&](int j) {
        const int b = j & 1;
        const uint32_t h_base = smem_u32(smem + S::H_OFF + b * S::H_BYTES);
        for (int kb = 0; kb < 2; ++kb) {
          // each GELU k-block (64 hidden columns) is signalled separately, so the k-block 0
          // MMAs run while the epilogue still computes k-block 1
          mbar_wait(&h_full[2 * b + kb], (h_ph >> b) & 1);
          if (kb == 0) {
            if (j < 8) MLP_TR(it, 12 + j);
            if (j == 0) {  // acc2 must have been drained by the previous tile's epilogue
              mbar_wait(a2_empty, (a2_cnt & 1) ^ 1);
              ++a2_cnt;
            }
          }
          const uint32_t w = take();  // !PAIR: rows 0-127 of the k-block, rows 128-255 in the next slot
          if constexpr (!PAIR) {
            ++pos;
            take();
            --pos;
          }
          tc_fence_after();
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t ad = make_smem_desc(h_base + kb * 16384 + k * 32, 16, 1024, kLayoutSW128);
            const uint64_t bd = make_smem_desc(w + k * 32, 16, 1024, kLayoutSW128);
            const bool acc = (OPJ && p.keep_x1) || (j | kb | k) != 0;  // keep_x1: onto x1
            if constexpr (PAIR) mma_ss_2sm(tmem + ACC2, ad, bd, idesc2, acc);
            else mma_ss(tmem + ACC2, ad, bd, idesc2, acc);
          }
          give();
          if constexpr (!PAIR) give();
        }
        h_ph ^= 1u << b;
        commit(&h_empty[b]);
      };
      MLP_TILES(tile) {
        (void)tile;
        if constexpr (OPJ) {
          // MMA_o: acc2 = o . W_o^T over the tile's first 12 ring positions
          const uint32_t p0 = static_cast<uint32_t>(it) * slots_per_tile;
          mbar_wait(a2_empty, (a2_cnt & 1) ^ 1);  // previous tile's final epilogue drained acc2
          ++a2_cnt;
          auto wait_pos = [&](uint32_t q) {
            mbar_wait(&w_full[q % MLP_SLOTS], (q / MLP_SLOTS) & 1);
            return smem_u32(smem + S::W_OFF + (q % MLP_SLOTS) * S::SLOT_BYTES);
          };
          MLP_TR(it, 40);
          for (int kb = 0; kb < KB; ++kb) {
            if (kb == 1) MLP_TR(it, 42);
            const uint32_t qo = p0 + opj_o(kb), qw = p0 + opj_w(kb);
            const uint32_t a = wait_pos(qo);
            const uint32_t w = wait_pos(qw);
            if constexpr (!PAIR) wait_pos(qw + 1);
            tc_fence_after();
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint64_t ad = make_smem_desc(a + k * 32, 16, 1024, kLayoutSW128);
              const uint64_t bd = make_smem_desc(w + k * 32, 16, 1024, kLayoutSW128);
              if constexpr (PAIR) mma_ss_2sm(tmem + ACC2, ad, bd, idesc2, (kb | k) != 0);
              else mma_ss(tmem + ACC2, ad, bd, idesc2, (kb | k) != 0);
            }
            commit(&w_empty[qo % MLP_SLOTS]);
            commit(&w_empty[qw % MLP_SLOTS]);
            if constexpr (!PAIR) commit(&w_empty[(qw + 1) % MLP_SLOTS]);
          }
          commit(ao_full);
          MLP_TR(it, 41);
          pos = p0 + (PAIR ? 2 * KB : 3 * KB);
        } else {
          pos = static_cast<uint32_t>(it) * slots_per_tile + KB;  // the h pieces belong to the epilogue
        }
        mbar_wait(ht_full, it & 1);
        MLP_TR(it, 3);
        tc_fence_after();
        mma1(0);
        for (int j = 1; j < n_chunks; ++j) {
          mma1(j);
          mma2(j - 1);
        }
        mma2(n_chunks - 1);
        commit(a2_full);
        ++it;
      }
    }
  } else {
    // ============================================================ epilogue warps (2..9)
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    const int et = threadIdx.x - 64;
    for (int i = et; i < p.F; i += 256) b1_s[i] = __ldg(p.b1 + i);
    for (int i = et; i < D; i += 256) {
      b2_s[i] = __ldg(p.b2 + i);
      if (do_ln) { lng_s[i] = __ldg(p.ln_g + i); lnb_s[i] = __ldg(p.ln_b + i); }
      if constexpr (OPJ) { bo_s[i] = __ldg(p.bo + i); g2_s[i] = __ldg(p.ln2_g + i); b2ln_s[i] = __ldg(p.ln2_b + i); }
    }
    asm volatile("bar.sync 5, 256;" ::: "memory");
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    const int r_in_tile = quarter * 32 + lane;
    uint32_t a1_ph = 0, h_ph = 0;  // bit b: phase of barrier [b]
    uint32_t xph = 0;
    MLP_TILES(tile) {
      const int it = (tile - t_first) / t_step;
      const int row = tile * 128 + r_in_tile;
      if constexpr (OPJ) {
        // ---- x1 = x + acc_o + b_o -> x (TMA), h = LN2(x1) -> TMEM h tile (A operand of MMA1).
        //      Staging: this warp's 4 KB slices of H[0] / H[1] (free until GELU(0)).
        const int e = warp - 2;
        uint8_t* hslice = smem + S::H_OFF + half * 16384 + quarter * 4096;
        const ResidStage st{hslice, S::H_BYTES, nullptr, 0, xbar + 3 * e, &xph, nullptr};
        const ResidLnArgs la{D, p.ln_cap, p.ln_eps};
        const uint32_t tb = tmem + lane_off + ACC2 + half * 128;
        if (et == 0) MLP_TR(it, 38);
        const int a2_cta = PAIR && rank ? 0 : -1;  // PAIR: acc2 releases arrive on the leader
        if (p.keep_x1)
          resid_ln_tma<4, true, true, true, false>(la, tmX, tmLN, st, tb, tile * 128 + quarter * 32, half * 128, M,
                                                   bo_s, g2_s, b2ln_s, ln_stats, quarter, half, lane, ao_full, it & 1,
                                                   a2_empty, a2_cta, tmem + lane_off + HT + half * 64);
        else
          resid_ln_tma<4, true, true>(la, tmX, tmLN, st, tb, tile * 128 + quarter * 32, half * 128, M, bo_s, g2_s,
                                      b2ln_s, ln_stats, quarter, half, lane, ao_full, it & 1, a2_empty, a2_cta,
                                      tmem + lane_off + HT + half * 64);
        if (et == 0) MLP_TR(it, 39);
        tmem_wait_st();
        tc_fence_before();
        asm volatile("bar.sync 5, 256;" ::: "memory");
        if (et == 0) {
          MLP_TR(it, 2);
          arrive_leader(ht_full);
        }
      } else {
      // ---- h tile -> TMEM (A operand of MMA1): piece kb = k-block kb -> columns [32 kb, 32 kb + 32);
      //      this warp moves its 32 rows x 32 k (16 columns) of each piece.  The previous
      //      tile's MMA1s are complete (its acc2 epilogue below waited for them).
      {
        const uint32_t pos0 = static_cast<uint32_t>(it) * slots_per_tile;
#pragma unroll 1
        for (int kb = 0; kb < KB; ++kb) {
          const uint32_t pos = pos0 + kb;
          const int slot = pos % MLP_SLOTS;
          mbar_wait(&w_full[slot], (pos / MLP_SLOTS) & 1);
          const uint8_t* prow = smem + S::W_OFF + slot * S::SLOT_BYTES + r_in_tile * 128;
          uint32_t v[16];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int qq = 4 * half + q;  // logical 16-byte chunk (8 k-values)
            const uint4 c = *reinterpret_cast<const uint4*>(prow + ((qq ^ (r_in_tile & 7)) << 4));
            v[4 * q] = c.x; v[4 * q + 1] = c.y; v[4 * q + 2] = c.z; v[4 * q + 3] = c.w;
          }
          if (et == 0 && kb == KB - 1) MLP_TR(it, 1);
          tmem_st16(tmem + lane_off + HT + kb * 32 + half * 16, v);
          asm volatile("bar.sync 5, 256;" ::: "memory");  // all 8 warps done reading the piece
          if (et == 0) mbar_arrive(&w_empty[slot]);
        }
        tmem_wait_st();
        tc_fence_before();
        asm volatile("bar.sync 5, 256;" ::: "memory");
        if (et == 0) {
          MLP_TR(it, 2);
          arrive_leader(ht_full);
        }
      }
      }
      // ---- hidden chunks: GELU(acc1 + b1) -> bf16 -> H[j&1] (SW128 K-major).  Warp (quarter,
      //      half) owns rows 32 quarter.. and columns [32 half, +32) of each 64-column k-block;
      //      k-block 0 is finished (and signalled) before k-block 1, so MMA2's first half
      //      overlaps the second half of the GELU.
      for (int j = 0; j < n_chunks; ++j) {
        const int b = j & 1;
        mbar_wait(a1_full, a1_ph);
        a1_ph ^= 1;
        if (et == 0 && j < 8) MLP_TR(it, 20 + j);
        tc_fence_after();
        uint32_t r0[32], r1[32];
        const uint32_t ta = tmem + lane_off + ACC1 + half * 32;
        tmem_ld32(ta, r0);        // k-block 0 columns [32 half, +32)
        tmem_ld32(ta + 64, r1);   // k-block 1 columns [64 + 32 half, +32)
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) arrive_leader(a1_empty);
        // H[b] may still be read by MMA2(j-2): wait for its commit
        if (j >= 2) {
          mbar_wait(&h_empty[b], (h_ph >> b) & 1);
          h_ph ^= 1u << b;
        }
#pragma unroll
        for (int kb = 0; kb < 2; ++kb) {
          const uint32_t* r = kb ? r1 : r0;
          uint8_t* hrow = smem + S::H_OFF + b * S::H_BYTES + kb * 16384 + r_in_tile * 128;
          const int col0 = 128 * j + kb * 64 + half * 32;
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) {  // 16-byte chunk q = 4 half + qq: columns [8q, 8q+8) of the k-block
            const int o = qq * 8;
            uint32_t pk[4];
            const float4 bl = *reinterpret_cast<const float4*>(b1_s + col0 + 8 * qq);      // smem broadcast
            const float4 bh = *reinterpret_cast<const float4*>(b1_s + col0 + 8 * qq + 4);
            const float bv[8] = {bl.x, bl.y, bl.z, bl.w, bh.x, bh.y, bh.z, bh.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              float a, c;
              fma2x(a, c, __uint_as_float(r[o + 2 * e]), __uint_as_float(r[o + 2 * e + 1]), 1.f, 1.f, bv[2 * e],
                    bv[2 * e + 1]);
              gelu2(a, c);
              pk[e] = pack_bf16x2(a, c);
            }
            const int q = 4 * half + qq;
            *reinterpret_cast<uint4*>(hrow + ((q ^ (r_in_tile & 7)) * 16)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          }
          fence_proxy_async();  // generic-proxy smem writes -> visible to the tensor core
          __syncwarp();
          if (lane == 0) arrive_leader(&h_full[2 * b + kb]);
        }
        if (et == 0 && j < 8) MLP_TR(it, 28 + j);
      }
      // the last two H buffers' MMA2 commits (consumed so the phase counts stay in step)
      for (int j = (n_chunks >= 2 ? n_chunks - 2 : 0); j < n_chunks; ++j) {
        const int b = j & 1;
        mbar_wait(&h_empty[b], (h_ph >> b) & 1);
        h_ph ^= 1u << b;
      }
      // ---- x += acc2 + b2  (+ next LayerNorm)
      if (et == 0) MLP_TR(it, 36);
      if constexpr (OPJ) {  // this warp's x1 TMA stores (same rows / columns) complete before reloading x
        if (lane == 0) bulk_wait0();
        __syncwarp();
      }
      if (p.staged) {
        const int e = warp - 2;
        uint8_t* hslice = smem + S::H_OFF + half * 16384 + quarter * 4096;
        uint8_t* lnb = smem + S::LNSTG_OFF + e * 2048;
        const ResidStage st{hslice, S::H_BYTES, lnb, 0, xbar + 3 * e, &xph, nullptr};
        const ResidLnArgs la{D, p.ln_cap, p.ln_eps};
        const uint32_t tb = tmem + lane_off + ACC2 + half * 128;
        if (OPJ && p.keep_x1) {  // acc2 = x1 + MLP(x1): x2 = acc2 + b2, x not read
          if (do_ln)
            resid_ln_tma<4, true, false, false>(la, tmX, tmLN, st, tb, tile * 128 + quarter * 32, half * 128, M, b2_s,
                                                lng_s, lnb_s, ln_stats, quarter, half, lane, a2_full, it & 1, a2_empty,
                                                PAIR && rank ? 0 : -1);
          else
            resid_ln_tma<4, false, false, false>(la, tmX, tmLN, st, tb, tile * 128 + quarter * 32, half * 128, M,
                                                 b2_s, lng_s, lnb_s, ln_stats, quarter, half, lane, a2_full, it & 1,
                                                 a2_empty, PAIR && rank ? 0 : -1);
        } else if (do_ln)
          resid_ln_tma<4, true>(la, tmX, tmLN, st, tb, tile * 128 + quarter * 32, half * 128, M, b2_s, lng_s, lnb_s,
                                ln_stats, quarter, half, lane, a2_full, it & 1, a2_empty, PAIR && rank ? 0 : -1);
        else
          resid_ln_tma<4, false>(la, tmX, tmLN, st, tb, tile * 128 + quarter * 32, half * 128, M, b2_s, lng_s,
                                 lnb_s, ln_stats, quarter, half, lane, a2_full, it & 1, a2_empty,
                                 PAIR && rank ? 0 : -1);
        if (et == 0) MLP_TR(it, 37);
        continue;
      }
      mbar_wait(a2_full, it & 1);
      tc_fence_after();
      const bool live = row < M;
      float* xrow = p.x + (size_t)row * D + half * 128;
      float s1 = 0.f, s2 = 0.f;
      float4 xn[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) xn[i] = live ? reinterpret_cast<const float4*>(xrow)[i] : make_float4(0, 0, 0, 0);
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        float4 xc[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) xc[i] = xn[i];
        if (c + 1 < 4 && live) {
#pragma unroll
          for (int i = 0; i < 8; ++i) xn[i] = reinterpret_cast<const float4*>(xrow + (c + 1) * 32)[i];
        }
        uint32_t r[32];
        tmem_ld32(tmem + lane_off + ACC2 + half * 128 + c * 32, r);
        tmem_wait_ld();
        if (c == 3) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) arrive_leader(a2_empty);
        }
        if (live) {
          const int col0 = half * 128 + c * 32;
          float4* dst = reinterpret_cast<float4*>(xrow + c * 32);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float4 bb = *reinterpret_cast<const float4*>(b2_s + col0 + 4 * i);
            float4 x = xc[i];
            x.x += __uint_as_float(r[4 * i + 0]) + bb.x;
            x.y += __uint_as_float(r[4 * i + 1]) + bb.y;
            x.z += __uint_as_float(r[4 * i + 2]) + bb.z;
            x.w += __uint_as_float(r[4 * i + 3]) + bb.w;
            dst[i] = x;
            s1 += (x.x + x.y) + (x.z + x.w);
            s2 += (x.x * x.x + x.y * x.y) + (x.z * x.z + x.w * x.w);
          }
        }
      }
      if (do_ln) {
        ln_stats[half * 128 + r_in_tile] = make_float2(s1, s2);
        asm volatile("bar.sync %0, 64;" ::"r"(1 + quarter) : "memory");
        const float2 o = ln_stats[(half ^ 1) * 128 + r_in_tile];
        asm volatile("bar.sync %0, 64;" ::"r"(1 + quarter) : "memory");
        const float mean = (s1 + o.x) * (1.f / D);
        const float rstd = rsqrtf(fmaxf((s2 + o.y) * (1.f / D) - mean * mean, 0.f) + p.ln_eps);
        if (row < p.ln_cap) {
          const float4* xr = reinterpret_cast<const float4*>(xrow);
#pragma unroll
          for (int i = 0; i < 8; ++i) xn[i] = live ? xr[i] : make_float4(0, 0, 0, 0);
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            const int col0 = half * 128 + c * 32;
            uint4* hd = reinterpret_cast<uint4*>(p.ln_out + (size_t)row * D + col0);
            if (!live) {
#pragma unroll
              for (int i = 0; i < 4; ++i) hd[i] = make_uint4(0, 0, 0, 0);
              continue;
            }
            float4 xc[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) xc[i] = xn[i];
            if (c + 1 < 4) {
#pragma unroll
              for (int i = 0; i < 8; ++i) xn[i] = xr[(c + 1) * 8 + i];
            }
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float4 x = xc[i];
              const float4 g = *reinterpret_cast<const float4*>(lng_s + col0 + 4 * i);
              const float4 be = *reinterpret_cast<const float4*>(lnb_s + col0 + 4 * i);
              pk[2 * i] = pack_bf16x2((x.x - mean) * rstd * g.x + be.x, (x.y - mean) * rstd * g.y + be.y);
              pk[2 * i + 1] = pack_bf16x2((x.z - mean) * rstd * g.z + be.z, (x.w - mean) * rstd * g.w + be.w);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) hd[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
          }
        }
      }
    }
  }
  tc_fence_before();
  if constexpr (CL == 2) cluster_sync();  // the peer may still arrive on / multicast into this CTA
  else __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    if constexpr (PAIR) tmem_dealloc_2sm<512>(tmem);
    else tmem_dealloc<512>(tmem);
  }
}
#undef MLP_TILES

}  // namespace cfd
