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

__device__ __forceinline__ void fma2x(float& d0, float& d1, float a0, float a1, float b0, float b1, float c0,
                                      float c1) {
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}

enum EpiKind : int {
  EPI_BF16_BIAS = 0,       // out_bf16 = bf16(acc + bias)                      (QKV)
  EPI_BF16_BIAS_GELU = 1,  // out_bf16 = bf16(GELU(acc + bias))                (MLP1)
  EPI_F32_RESID = 2,       // out_f32 += acc + bias                            (O-proj, MLP2)
  EPI_EMBED_COARSE = 3,    // out_f32 = out2_f32 = acc + bias + pe[row % pe_rows]   (B1)
  EPI_EMBED_FINE = 4,      // out_f32[frow[row]] = acc + bias + pe[fidx[row]]        (B9)
  EPI_F32_RESID_LN = 5,    // out_f32 += acc + bias; ln_out = bf16(LN(out_f32 row))  (O-proj/MLP2
                           // followed by the next LayerNorm; needs BN == N, one tile per row)
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
  const float* ln_g;         // EPI_F32_RESID_LN: next LayerNorm's gamma / beta [N]
  const float* ln_b;
  __nv_bfloat16* ln_out;     // [ln_cap, N]
  int ln_cap;                // rows of ln_out (pad rows [M, pad_rows) are zeroed)
  float ln_eps;
  // IMG (coarse patch embed straight from the image): a tile = img_rb coarse rows x img_gw
  // patches (rows_per_tile = img_rb * img_gw <= 128), k-block kb = (patch row py = kb / img_thirds,
  // third j = kb % img_thirds of its 3*Pc-element pixel segment), 32 k per block
  int img_rb, img_gw, img_thirds;
};

constexpr int GEMM_BM = 128;
constexpr int GEMM_BK = 64;
// Two configurations (template EW = epilogue warps, NACC = TMEM accumulator buffers):
//   EW=8, NACC=2: one CTA per SM, 2 warps per TMEM lane quarter (column halves), the
//                 epilogue of tile i overlaps the MMAs of tile i+1   (many-tile GEMMs)
//   EW=4, NACC=1: two CTAs per SM (256 TMEM columns, 2-stage ring each), one thread per
//                 full row, the two co-resident CTAs overlap each other (N = d GEMMs whose
//                 ~M/128 tiles would otherwise leave a badly quantised second wave)
constexpr int GEMM_EPI_WARPS = 8;                     // maximum
constexpr int GEMM_THREADS = 64 + 32 * GEMM_EPI_WARPS;  // + TMA warp + MMA warp
constexpr int GEMM_MAX_N = 2048;   // bias columns staged in shared memory
constexpr int GEMM_MAX_LN = 512;   // LayerNorm width for EPI_F32_RESID_LN

// BRES (weight-stationary, "B resident"): the CTA's whole [BN, K] weight slice (K = 256:
// four 64-wide k-blocks) is loaded into shared memory once and stays there while the CTA
// streams its row tiles through an A-only ring.  The default streams A and B per k-block.
constexpr int GEMM_BRES_KB = 4;
template <int BN, int STAGES, int NACC = 2, bool BRES = false, int BKX = GEMM_BK, bool PAIR = false>
struct GemmSmem {
  static constexpr int A_BYTES = GEMM_BM * BKX * 2;
  static constexpr int B_BYTES = (PAIR ? BN / 2 : BN) * BKX * 2;  // PAIR: this CTA's half of the columns
  static constexpr int STAGE_BYTES = A_BYTES + (BRES ? 0 : B_BYTES);  // TMA bytes per ring stage
  static constexpr int NB = BRES ? GEMM_BRES_KB : STAGES;            // B buffers
  static constexpr int BAR_OFF = STAGES * A_BYTES + NB * B_BYTES;
  static constexpr int BAR_BYTES = 256 + 2 * 128 * 8;  // barriers + RESID_LN row statistics
  static constexpr int PAR_FLOATS = GEMM_MAX_N + 2 * GEMM_MAX_LN;  // bias | ln gamma | ln beta
  static constexpr int PAR_BYTES = ((PAR_FLOATS * 4 + 1023) / 1024) * 1024;
  static constexpr int STG_BYTES = 12288;  // per epilogue warp: x chunks [2] 4 KB + LN chunks [2] 2 KB
  static constexpr int TOTAL = 1024 /*align slack*/ + BAR_OFF + BAR_BYTES + PAR_BYTES;
  static constexpr int STG_OFF = BAR_OFF + ((BAR_BYTES + PAR_BYTES + 1023) / 1024) * 1024;
  static constexpr int TOTAL_TMA_EPI = 1024 + STG_OFF + GEMM_EPI_WARPS * STG_BYTES;
  static constexpr int TOTAL_STG_OUT = 1024 + STG_OFF + GEMM_EPI_WARPS * 4096;  // bf16 out: 2 x 2 KB per warp
  static constexpr int TOTAL_STG_OUT1 = 1024 + STG_OFF + GEMM_EPI_WARPS * 2048;  // bf16 out: 1 x 2 KB per warp
  static constexpr uint32_t TMEM_COLS = (NACC * BN <= 32) ? 32 : (NACC * BN <= 64) ? 64 : (NACC * BN <= 128) ? 128
                                        : (NACC * BN <= 256) ? 256 : 512;
};

// Rows a varlen attention tile may touch past the last valid row: a task's last KV
// tile starts at (task start + 128 j) and so can overhang the packed rows by < 128.
__host__ __device__ __forceinline__ int pad_rows(int M, int cap) {
  const int r = ((M + 127) / 128) * 128 + 128;
  return r < cap ? r : cap;
}

__device__ __forceinline__ float gelu_erf(float v) { return 0.5f * v * (1.0f + erff(v * 0.70710678118654752f)); }

__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// GELU(z) = z * Phi(z), Phi(z) = 1/2 + 1/2 erf(z/sqrt2) (reading R4), for a pair:
//   Phi(z) ~= 1/2 + 1/2 tanh(z (A + B z^2)),  A, B minimax-fitted to the exact-erf Phi
// (|dPhi| <= 1.4e-4 for all z; <= 3.9e-4 including tanh.approx.f32's error, i.e. the GELU
// error stays below 1/5 of a bf16 ulp of the output).  3 FFMA2 + 2 MUFU.TANH + 1 FFMA2 per
// pair: the tanh runs on the otherwise idle MUFU pipe.
__device__ __forceinline__ void gelu2(float& a, float& b) {
  constexpr float A = 0.79880144f, B = 0.03528205f;
  float u0, u1, w0, w1, v0, v1, h0, h1;
  fma2x(u0, u1, a, b, a, b, 0.f, 0.f);         // z^2
  fma2x(w0, w1, u0, u1, B, B, A, A);           // A + B z^2
  fma2x(v0, v1, a, b, w0, w1, 0.f, 0.f);       // z (A + B z^2)
  fma2x(h0, h1, a, b, 0.5f, 0.5f, 0.f, 0.f);   // z / 2
  const float t0 = tanh_approx(v0), t1 = tanh_approx(v1);
  fma2x(a, b, h0, h1, t0, t1, h0, h1);         // z/2 (1 + tanh)
}

// ---------------------------------------------------------------------------- epilogue
// Each epilogue warp owns 32 rows (its TMEM lane quarter) x BN/2 columns of a tile, one
// row per thread, in 32-column chunks: tcgen05.ld -> + bias (shared-memory broadcast) ->
// fused op -> 16-byte vector stores of the thread's row segment.
// s1 / s2: shifted row sums (v - sh) and (v - sh)^2 for the fused LayerNorm, sh = the first value
// this thread sees (first = true on its first chunk), so |mean| >> std does not cancel.
template <int EPI>
__device__ __forceinline__ void direct_chunk(const GemmParams& p, float (&v)[32], int row, int col0, int m_store,
                                             int M, float& s1, float& s2, float& sh, bool first) {
  if constexpr (EPI == EPI_BF16_BIAS || EPI == EPI_BF16_BIAS_GELU) {
    if (row >= m_store) return;
    uint32_t pk[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      float a = v[2 * i], b = v[2 * i + 1];
      if constexpr (EPI == EPI_BF16_BIAS_GELU) gelu2(a, b);
      pk[i] = pack_bf16x2(a, b);
    }
    uint4* dst = reinterpret_cast<uint4*>(p.out_bf16 + (size_t)row * p.N + col0);
#pragma unroll
    for (int i = 0; i < 4; ++i) dst[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
  } else if constexpr (EPI == EPI_F32_RESID || EPI == EPI_F32_RESID_LN) {
    if (row >= M) return;
    float4* dst = reinterpret_cast<float4*>(p.out_f32 + (size_t)row * p.ld_out + col0);
    float4 x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = dst[i];  // all 8 loads in flight before the adds
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      x[i].x += v[4 * i + 0]; x[i].y += v[4 * i + 1]; x[i].z += v[4 * i + 2]; x[i].w += v[4 * i + 3];
      dst[i] = x[i];
      if constexpr (EPI == EPI_F32_RESID_LN) {
        if (first && i == 0) sh = x[0].x;
        const float a = x[i].x - sh, b = x[i].y - sh, c = x[i].z - sh, d = x[i].w - sh;
        s1 += (a + b) + (c + d);
        s2 += (a * a + b * b) + (c * c + d * d);
      }
    }
  } else if constexpr (EPI == EPI_EMBED_COARSE) {
    if (row >= m_store) return;
    const float4* pe4 = reinterpret_cast<const float4*>(p.pe + (size_t)(row % p.pe_rows) * p.N + col0);
    float4* d1 = reinterpret_cast<float4*>(p.out_f32 + (size_t)row * p.ld_out + col0);
    float4* d2 = reinterpret_cast<float4*>(p.out2_f32 + (size_t)row * p.ld_out + col0);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float4 e = __ldg(pe4 + i);
      const float4 o = make_float4(v[4 * i] + e.x, v[4 * i + 1] + e.y, v[4 * i + 2] + e.z, v[4 * i + 3] + e.w);
      d1[i] = o;
      d2[i] = o;
      s1 += (o.x + o.y) + (o.z + o.w);  // row statistics for the optional fused LN1 (p.ln_g)
      s2 += (o.x * o.x + o.y * o.y) + (o.z * o.z + o.w * o.w);
    }
  } else if constexpr (EPI == EPI_EMBED_FINE) {
    if (row >= m_store) return;
    const int orow = __ldg(p.frow + row);
    const int prow = __ldg(p.fidx + row);
    const float4* pe4 = reinterpret_cast<const float4*>(p.pe + (size_t)prow * p.N + col0);
    float4* d1 = reinterpret_cast<float4*>(p.out_f32 + (size_t)orow * p.ld_out + col0);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float4 e = __ldg(pe4 + i);
      d1[i] = make_float4(v[4 * i] + e.x, v[4 * i + 1] + e.y, v[4 * i + 2] + e.z, v[4 * i + 3] + e.w);
    }
  }
}

// ---------------------------------------------------------------------------- staged residual + LN
// Residual (+ LayerNorm) epilogue of one warp (32 rows x CH 32-column chunks of a row half)
// through shared memory with TMA: x chunks [32 rows x 32 fp32] are TMA-loaded into a
// 128B-swizzled buffer, each thread reads / writes its row with conflict-free 16-byte
// accesses, and the results leave by TMA store, so no per-row global access is issued.
//   LN:   pass A: x_new = x_old + acc + bias -> x (TMA store) and back into the accumulator's
//                 TMEM columns; row statistics (the two column-half warps exchange)
//         pass B: LN(x_new) read back from TMEM -> bf16 (SW64 buffer, TMA store); x is read
//                 from memory once.  Rows >= M keep x and get zeros in ln_out.
//   !LN:  one pass: x_new = x_old + acc + bias -> x (TMA store).
// The accumulator stays in TMEM until the last read.  Staging: two 4 KB x buffers (1024-B
// aligned) at xb + b * xb_stride; LN buffers of 2 KB at hb + b * hb_stride (hb_stride 0: one
// buffer, the store of chunk c-1 is then drained before chunk c is written).
struct ResidStage {
  uint8_t* xb;
  int xb_stride;
  uint8_t* hb;
  int hb_stride;
  uint64_t* bar;   // [2] ([3] with xb3) this warp's TMA-load barriers
  uint32_t* xph;   // bit b: phase of bar[b]
  uint8_t* xb3 = nullptr;  // optional third 4 KB x buffer: three residual chunks in flight
};

struct ResidLnArgs {
  int n_total;     // LayerNorm width (row length)
  int ln_cap;      // rows of ln_out
  float ln_eps;
};

// LNT: the LayerNorm output goes to TMEM instead of memory — bf16 pairs of the row's columns
// (col_base + 2i, +1) at column ln_tmem + i of this warp's lanes (the A-operand layout of a
// TS-form MMA over the normalised row), used by the fused O-projection + MLP kernel.
// LOADX = false (LN only): the accumulator already holds x_old (an MMA accumulated onto it),
//   so x_new = acc + bias and x is not read; dead rows (>= M) are stored as zeros.
// STOREX = false (LN only): x_new is kept in the accumulator's TMEM columns only (not stored).
template <int CH, bool LN, bool LNT = false, bool LOADX = true, bool STOREX = true>
__device__ __forceinline__ void resid_ln_tma(const ResidLnArgs& la, const CUtensorMap& tmX, const CUtensorMap& tmLN,
                                             const ResidStage& st, uint32_t tbase, int row0, int col_base, int M,
                                             const float* bias_s, const float* lng_s, const float* lnb_s,
                                             float2* stats, int quarter, int half, int lane, uint64_t* tfull_bar,
                                             uint32_t tfull_parity, uint64_t* tempty_bar, int tempty_cta = -1,
                                             uint32_t ln_tmem = 0) {
  // tempty_cta >= 0: the accumulator-empty barrier lives in that cluster CTA (CTA-pair MMA)
  auto release_acc = [&]() {
    if (tempty_cta >= 0) mbar_arrive_cluster(tempty_bar, static_cast<uint32_t>(tempty_cta));
    else mbar_arrive(tempty_bar);
  };
  const int r = lane;
  const bool live = row0 + r < M;
  const bool one_hb = st.hb_stride == 0;
  const int NB = st.xb3 ? 3 : 2;  // x staging buffers
  auto buf = [&](int b) { return b == 2 ? st.xb3 : st.xb + b * st.xb_stride; };
  auto load = [&](int c, int b) {
    if (lane == 0) {
      mbar_expect_tx(&st.bar[b], 4096);
      tma_load_2d(buf(b), &tmX, &st.bar[b], col_base + c * 32, row0);
    }
  };
  auto wait = [&](int b) {
    mbar_wait(&st.bar[b], (*st.xph >> b) & 1);
    *st.xph ^= 1u << b;
  };
  auto row_ptr = [&](int b, int q) { return reinterpret_cast<float4*>(buf(b) + r * 128 + ((q ^ (r & 7)) << 4)); };
  static_assert(LN || STOREX, "STOREX = false is a LayerNorm-path option");
  float mean = 0.f, rstd = 0.f;
  if (LOADX) {
    load(0, 0);
    if (CH > 1) load(1, 1);
    if (NB == 3 && CH > 2) load(2, 2);
  }
  mbar_wait(tfull_bar, tfull_parity);
  tc_fence_after();
  if constexpr (LN) {
    // ---- pass A: x_new = x_old + acc + bias -> x (TMA store) and back into the accumulator's
    //      TMEM columns; row statistics.  (The first residual chunks were requested before the
    //      accumulator was ready.)  The row statistics are shifted sums around the row's first
    //      value K of this half (s1 = sum (v - K), s2 = sum (v - K)^2), so the variance does not
    //      cancel catastrophically when |mean| >> std; the halves combine with Chan's formula.
    float s1 = 0.f, s2 = 0.f, shift = 0.f;
#pragma unroll 1
    for (int c = 0; c < CH; ++c) {
      const int b = c % NB;
      uint32_t a[32];
      tmem_ld32(tbase + c * 32, a);
      if (LOADX) wait(b);
      if (!LOADX && STOREX && c >= NB) {  // the TMA store of chunk c - NB (buffer b) is done reading
        if (lane == 0) { if (NB == 3) bulk_wait_read2(); else bulk_wait_read1(); }
        __syncwarp();
      }
      tmem_wait_ld();
      const int col0 = col_base + c * 32;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float4* px = row_ptr(b, q);
        const float4 bb = *reinterpret_cast<const float4*>(bias_s + col0 + 4 * q);
        float v0, v1, v2, v3;
        if constexpr (LOADX) {
          const float4 x = *px;
          v0 = x.x + (__uint_as_float(a[4 * q]) + bb.x);
          v1 = x.y + (__uint_as_float(a[4 * q + 1]) + bb.y);
          v2 = x.z + (__uint_as_float(a[4 * q + 2]) + bb.z);
          v3 = x.w + (__uint_as_float(a[4 * q + 3]) + bb.w);
          if (STOREX && live) *px = make_float4(v0, v1, v2, v3);
        } else {
          v0 = __uint_as_float(a[4 * q]) + bb.x;
          v1 = __uint_as_float(a[4 * q + 1]) + bb.y;
          v2 = __uint_as_float(a[4 * q + 2]) + bb.z;
          v3 = __uint_as_float(a[4 * q + 3]) + bb.w;
          if (!live) v0 = v1 = v2 = v3 = 0.f;
          if (STOREX) *px = make_float4(v0, v1, v2, v3);
        }
        if (q == 0 && c == 0) shift = v0;
        const float d0 = v0 - shift, d1 = v1 - shift, d2 = v2 - shift, d3 = v3 - shift;
        s1 += (d0 + d1) + (d2 + d3);
        s2 += (d0 * d0 + d1 * d1) + (d2 * d2 + d3 * d3);
        a[4 * q] = __float_as_uint(v0);
        a[4 * q + 1] = __float_as_uint(v1);
        a[4 * q + 2] = __float_as_uint(v2);
        a[4 * q + 3] = __float_as_uint(v3);
      }
      tmem_st16(tbase + c * 32, *reinterpret_cast<const uint32_t(*)[16]>(a));
      tmem_st16(tbase + c * 32 + 16, *reinterpret_cast<const uint32_t(*)[16]>(a + 16));
      if constexpr (STOREX) {
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&tmX, buf(b), col0, row0);
          bulk_commit();
        }
      }
      if (LOADX && c + NB < CH) {
        if (STOREX) {
          if (lane == 0) bulk_wait_read0();  // buffer b is reloaded next
        } else {
          fence_proxy_async();  // this warp's generic reads of buffer b before the TMA overwrite
        }
        __syncwarp();
        load(c + NB, b);
      }
    }
    tmem_wait_st();
    // ---- statistics of the full row (two warps, one per column half of n_h = n / 2 values):
    //      per half mean_h = K + s1 / n_h and M2_h = s2 - s1^2 / n_h, then
    //      mean = (mean_0 + mean_1) / 2, M2 = M2_0 + M2_1 + (mean_0 - mean_1)^2 n_h / 2
    const int r_in_tile = quarter * 32 + lane;
    const float n_h = 0.5f * (float)la.n_total;
    const float mean_h = shift + s1 / n_h;
    const float m2_h = fmaxf(s2 - s1 * (s1 / n_h), 0.f);
    stats[half * 128 + r_in_tile] = make_float2(mean_h, m2_h);
    asm volatile("bar.sync %0, 64;" ::"r"(1 + quarter) : "memory");
    const float2 o = stats[(half ^ 1) * 128 + r_in_tile];
    asm volatile("bar.sync %0, 64;" ::"r"(1 + quarter) : "memory");
    // both halves combine in the same (half 0, half 1) order, so both warps get identical bits
    const float2 h0 = half == 0 ? make_float2(mean_h, m2_h) : o;
    const float2 h1 = half == 0 ? o : make_float2(mean_h, m2_h);
    const float dm = h0.x - h1.x;
    mean = 0.5f * (h0.x + h1.x);
    const float m2 = (h0.y + h1.y) + dm * dm * (0.5f * n_h);
    rstd = rsqrtf(m2 / (float)la.n_total + la.ln_eps);
    // ---- pass B: LN(x_new) from TMEM -> bf16 (SW64 buffer) -> TMA store
#pragma unroll 1
    for (int c = 0; c < CH; ++c) {
      uint32_t a[32];
      tmem_ld32(tbase + c * 32, a);
      tmem_wait_ld();
      if (c + 1 == CH) {  // accumulator fully read: hand TMEM back to the MMA warp
        tc_fence_before();
        __syncwarp();
        if (lane == 0) release_acc();
      }
      const int col0 = col_base + c * 32;
      uint32_t pk[16];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (live) {
          const float4 g = *reinterpret_cast<const float4*>(lng_s + col0 + 4 * q);
          const float4 be = *reinterpret_cast<const float4*>(lnb_s + col0 + 4 * q);
          const float x0 = __uint_as_float(a[4 * q]), x1 = __uint_as_float(a[4 * q + 1]);
          const float x2 = __uint_as_float(a[4 * q + 2]), x3 = __uint_as_float(a[4 * q + 3]);
          pk[2 * q] = pack_bf16x2((x0 - mean) * rstd * g.x + be.x, (x1 - mean) * rstd * g.y + be.y);
          pk[2 * q + 1] = pack_bf16x2((x2 - mean) * rstd * g.z + be.z, (x3 - mean) * rstd * g.w + be.w);
        } else {
          pk[2 * q] = 0u;
          pk[2 * q + 1] = 0u;
        }
      }
      if constexpr (LNT) {
        tmem_st16(ln_tmem + c * 16, pk);
        continue;
      }
      const int b = c & 1;
      if (c >= (one_hb ? 1 : 2)) {  // the TMA store that last read this hb must be done reading
        if (lane == 0) bulk_wait_read0();
        __syncwarp();
      }
      uint8_t* hb = st.hb + b * st.hb_stride;
      // LN chunk: 32 rows x 64 B, SW64 layout (16-byte chunk q of row r at q ^ ((r >> 1) & 3))
#pragma unroll
      for (int q = 0; q < 4; ++q)
        *reinterpret_cast<uint4*>(hb + r * 64 + ((q ^ ((r >> 1) & 3)) << 4)) =
            make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        if (row0 < la.ln_cap) tma_store_2d(&tmLN, hb, col0, row0);
        bulk_commit();
      }
    }
  } else {
    // ---- single pass: x_new = x_old + acc + bias -> x (TMA store)
#pragma unroll 1
    for (int c = 0; c < CH; ++c) {
      const int b = c % NB;
      uint32_t a[32];
      tmem_ld32(tbase + c * 32, a);
      if (LOADX) wait(b);
      if (!LOADX && c >= NB) {  // the TMA store of chunk c - NB (buffer b) is done reading
        if (lane == 0) { if (NB == 3) bulk_wait_read2(); else bulk_wait_read1(); }
        __syncwarp();
      }
      tmem_wait_ld();
      if (c + 1 == CH) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) release_acc();
      }
      const int col0 = col_base + c * 32;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float4* px = row_ptr(b, q);
        const float4 bb = *reinterpret_cast<const float4*>(bias_s + col0 + 4 * q);
        if constexpr (LOADX) {
          float4 x = *px;
          if (live) {
            x.x += __uint_as_float(a[4 * q]) + bb.x;
            x.y += __uint_as_float(a[4 * q + 1]) + bb.y;
            x.z += __uint_as_float(a[4 * q + 2]) + bb.z;
            x.w += __uint_as_float(a[4 * q + 3]) + bb.w;
            *px = x;
          }
        } else {
          *px = live ? make_float4(__uint_as_float(a[4 * q]) + bb.x, __uint_as_float(a[4 * q + 1]) + bb.y,
                                   __uint_as_float(a[4 * q + 2]) + bb.z, __uint_as_float(a[4 * q + 3]) + bb.w)
                     : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(&tmX, buf(b), col0, row0);
        bulk_commit();
      }
      if (LOADX && c + NB < CH) {
        if (lane == 0) bulk_wait_read0();  // buffer b is reloaded next
        __syncwarp();
        load(c + NB, b);
      }
    }
  }
  if (lane == 0) bulk_wait_read0();  // staging buffers reusable by the next tile
  __syncwarp();
}

// ---------------------------------------------------------------------------- staged bf16 store
// bf16 output epilogue of one warp (32 rows x CH 32-column chunks) through shared memory:
// acc + bias (+GELU) -> bf16 -> a 2 KB SW64 buffer (conflict-free 16-byte writes, one row per
// thread) -> TMA store of the 32 x 32 box.  Two buffers alternate; a buffer is rewritten once
// the store issued from it two chunks earlier has finished reading (SB = 1: one buffer, the
// previous chunk's store must have finished reading it -- frees shared memory for the ring).
template <int CH, int EPI, int SB = 2>
__device__ __forceinline__ void store_bf16_tma(const CUtensorMap& tmO, uint8_t* stg, uint32_t tbase, int row0,
                                               int col_base, const float* bias_s, int lane, uint64_t* tfull_bar,
                                               uint32_t tfull_parity, uint64_t* tempty_bar, int tempty_cta = -1) {
  mbar_wait(tfull_bar, tfull_parity);
  tc_fence_after();
#pragma unroll 1
  for (int c = 0; c < CH; ++c) {
    uint32_t a[32];
    tmem_ld32(tbase + c * 32, a);
    tmem_wait_ld();
    if (c + 1 == CH) {  // accumulator fully read: hand TMEM back to the MMA warp
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (tempty_cta >= 0) mbar_arrive_cluster(tempty_bar, static_cast<uint32_t>(tempty_cta));
        else mbar_arrive(tempty_bar);
      }
    }
    const int col0 = col_base + c * 32;
    uint32_t pk[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float2 bb = *reinterpret_cast<const float2*>(bias_s + col0 + 2 * i);
      float x0 = __uint_as_float(a[2 * i]) + bb.x, x1 = __uint_as_float(a[2 * i + 1]) + bb.y;
      if constexpr (EPI == EPI_BF16_BIAS_GELU) gelu2(x0, x1);
      pk[i] = pack_bf16x2(x0, x1);
    }
    if (lane == 0) {  // the store that last read this buffer is done reading
      if constexpr (SB == 2) bulk_wait_read1();
      else bulk_wait_read0();
    }
    __syncwarp();
    uint8_t* buf = stg + (SB == 2 ? (c & 1) * 2048 : 0);
#pragma unroll
    for (int q = 0; q < 4; ++q)
      *reinterpret_cast<uint4*>(buf + lane * 64 + ((q ^ ((lane >> 1) & 3)) << 4)) =
          make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) {
      tma_store_2d(&tmO, buf, col0, row0);
      bulk_commit();
    }
  }
}

// IMG: A tiles are TMA-gathered from the HWC image through a 5-D tensor map (reading R2:
// patch vector (py, px, ch) = one Pc*3-element pixel segment per patch row), so no im2col
// buffer is written or read; 32-wide k-blocks in 64-byte (SW64) rows.
// PAIR (BRES bf16 outputs only: the QKV projection): 2-CTA clusters issuing cta_group::2
// M = 256 MMAs over the pair's two 128-row tiles; each CTA keeps HALF of the column block's
// weights resident (rows [128 rank, +128) of the BN = 256 block, 64 KB instead of 128 KB), so
// the freed shared memory holds 8 A stages in flight.  A pieces are pair TMA loads completing
// on the leader's full barrier; the leader's commits reach both CTAs; both epilogues release
// the accumulator on the leader's tempty.  Tile walk: the pair takes row-tile pairs
// (2 i, 2 i + 1); an odd last tile leaves CTA 1 a ghost tile (stores skipped).
template <int BN, int STAGES, int EPI, int EW, int NACC, bool BRES = false, bool IMG = false, bool PAIR = false>
__global__ void __launch_bounds__(64 + 32 * EW, (EW == 4 ? 2 : 1))
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const GemmParams p, const __grid_constant__ CUtensorMap tmX,
                   const __grid_constant__ CUtensorMap tmLN) {
  static_assert((EW == 8 && NACC == 2) || (EW == 4 && NACC == 1), "supported epilogue configurations");
  static_assert(!IMG || (EPI == EPI_EMBED_COARSE && !BRES), "IMG is the coarse patch embed");
  static_assert(!PAIR || (BN == 256 && EW == 8 &&
                          ((BRES && EPI == EPI_BF16_BIAS) || (IMG && EPI == EPI_EMBED_COARSE && !BRES))),
                "PAIR is the QKV projection or the image-sourced coarse patch embed");
  constexpr int BKX = IMG ? 32 : GEMM_BK;
  using S = GemmSmem<BN, STAGES, NACC, BRES, BKX, PAIR>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // keeps the shared space
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * S::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* bres_full = tempty + 2 + 16;  // BRES: resident weight slice landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2 + 17);
  float2* ln_stats = reinterpret_cast<float2*>(smem + S::BAR_OFF + 256);  // [2][128]
  uint64_t* xbar = tempty + 2;  // [8 warps][2] TMA-load barriers of the staged residual epilogue
  float* par = reinterpret_cast<float*>(smem + S::BAR_OFF + S::BAR_BYTES);
  float* bias_s = par;                       // [N]
  float* lng_s = par + GEMM_MAX_N;           // [N] (RESID_LN)
  float* lnb_s = lng_s + GEMM_MAX_LN;        // [N] (RESID_LN)

  const int warp = warp_id(), lane = lane_id();
  // bf16 outputs (QKV, MLP1) also cover the pad rows [M, pad_rows(M)) so attention's
  // tail tiles (which may start at any row of the last task) read finite values
  constexpr bool kPad = (EPI == EPI_BF16_BIAS || EPI == EPI_BF16_BIAS_GELU);
  // bf16 outputs of the one-CTA/SM configuration leave through smem + TMA store (tmX = out map)
  constexpr bool kStgOut = kPad && EW == 8;
  const int n_tiles = p.N / BN;
  const int num_k = p.K / BKX;
  const int rpt = IMG ? p.img_rb * p.img_gw : GEMM_BM;  // rows per tile
  const int rank = PAIR ? static_cast<int>(cluster_ctarank()) : 0;
  const int cta_id = PAIR ? static_cast<int>(cluster_id_x()) : static_cast<int>(blockIdx.x);  // BRES walk unit
  const int n_units = PAIR ? static_cast<int>(nclusters_x()) : static_cast<int>(gridDim.x);
  const int n_fix = BRES ? cta_id % n_tiles : 0;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < NACC; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], EW * (PAIR ? 2 : 1)); }
    for (int i = 0; i < 16; ++i) mbar_init(&xbar[i], 1);
    mbar_init(bres_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) {
    if constexpr (PAIR) tmem_alloc_2sm<S::TMEM_COLS>(tmem_slot);
    else tmem_alloc<S::TMEM_COLS>(tmem_slot);
  }
  tc_fence_before();
  if constexpr (PAIR) cluster_sync();  // peer barriers initialised before any remote arrive / pair load
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if constexpr (BRES) {  // the CTA's weight slice, once
    if (warp == 0 && lane == 0) {
      if constexpr (PAIR) {  // this CTA's 128 rows of the column block, on the leader's barrier
        if (rank == 0) mbar_expect_tx(bres_full, 2 * GEMM_BRES_KB * S::B_BYTES);
        const uint32_t lb = mapa_u32(bres_full, 0);
        for (int kb = 0; kb < GEMM_BRES_KB; ++kb)
          tma_load_2d_2sm(sB + kb * S::B_BYTES, &tmB, lb, kb * GEMM_BK, n_fix * BN + 128 * rank);
      } else {
        mbar_expect_tx(bres_full, GEMM_BRES_KB * S::B_BYTES);
        for (int kb = 0; kb < GEMM_BRES_KB; ++kb)
          tma_load_2d(sB + kb * S::B_BYTES, &tmB, bres_full, kb * GEMM_BK, n_fix * BN);
      }
    }
  }
  const int M = p.m_dev ? __ldg(p.m_dev) : p.M;
  const int m_store = kPad ? pad_rows(M, p.m_cap) : M;
  // RESID_LN also visits the tiles of the pad rows (zeroed in ln_out, x untouched)
  const int m_tiles = ((EPI == EPI_F32_RESID_LN ? pad_rows(M, p.ln_cap) : m_store) + rpt - 1) / rpt;
  const int total = m_tiles * n_tiles;
  // tile walk: default tile = m_blk * n_tiles + n_blk over all tiles; BRES: the CTA (PAIR: the
  // cluster) keeps column block cta_id % n_tiles and walks row blocks (PAIR: row-block pairs;
  // the unit count is a multiple of n_tiles)
  // (PAIR without BRES, the coarse embed: one column block, n_tiles = 1, the same row-pair walk)
  constexpr bool kUnitWalk = BRES || PAIR;
  const int t_first = kUnitWalk ? cta_id / n_tiles : (int)blockIdx.x;
  const int t_step = kUnitWalk ? n_units / n_tiles : (int)gridDim.x;
  const int m_units = PAIR ? (m_tiles + 1) / 2 : m_tiles;
  const int t_end = kUnitWalk ? (cta_id < t_step * n_tiles ? m_units : 0) : total;
  auto m_of = [&](int tile) { return kUnitWalk ? (PAIR ? 2 * tile + rank : tile) : tile / n_tiles; };

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = t_first; tile < t_end; tile += t_step) {
        const int m_blk = m_of(tile), n_blk = BRES ? n_fix : tile % n_tiles;
        for (int kb = 0; kb < num_k; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if constexpr (PAIR && IMG) {  // this CTA's rpt A rows + its 128 B columns, on the leader's barrier
            if (rank == 0) mbar_expect_tx(&full[stage], 2 * (rpt * 64 + S::B_BYTES));
            const uint32_t lb = mapa_u32(&full[stage], 0);
            tma_load_5d_2sm(sA + stage * S::A_BYTES, &tmA, lb, 0, kb % p.img_thirds, 0, kb / p.img_thirds,
                            m_blk * p.img_rb);
            tma_load_2d_2sm(sB + stage * S::B_BYTES, &tmB, lb, kb * BKX, n_blk * BN + 128 * rank);
          } else if constexpr (PAIR) {  // this CTA's 128 A rows, completing on the leader's full barrier
            if (rank == 0) mbar_expect_tx(&full[stage], 2 * S::A_BYTES);
            tma_load_2d_2sm(sA + stage * S::A_BYTES, &tmA, mapa_u32(&full[stage], 0), kb * BKX, m_blk * GEMM_BM);
          } else if constexpr (IMG) {  // rpt rows of 64 B (OOB rows of the last tile are zero-filled)
            mbar_expect_tx(&full[stage], rpt * 64 + S::B_BYTES);
            tma_load_5d(sA + stage * S::A_BYTES, &tmA, &full[stage], 0, kb % p.img_thirds, 0, kb / p.img_thirds,
                        m_blk * p.img_rb);
          } else {
            mbar_expect_tx(&full[stage], S::STAGE_BYTES);
            tma_load_2d(sA + stage * S::A_BYTES, &tmA, &full[stage], kb * BKX, m_blk * GEMM_BM);
          }
          if constexpr (!BRES && !PAIR) tma_load_2d(sB + stage * S::B_BYTES, &tmB, &full[stage], kb * BKX, n_blk * BN);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {  // PAIR: the leader issues the pair's MMAs
      constexpr uint32_t idesc = make_idesc_bf16(GEMM_BM * (PAIR ? 2 : 1), BN, 0);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      if constexpr (BRES) mbar_wait(bres_full, 0);  // also when this CTA has no tile: the load must land
      for (int tile = t_first; tile < t_end; tile += t_step) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < num_k; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + stage * S::A_BYTES);
          const uint32_t b0 = smem_u32(sB + (BRES ? kb : stage) * S::B_BYTES);
#pragma unroll
          for (int k = 0; k < BKX / 16; ++k) {
            const uint64_t ad = IMG ? make_smem_desc(a0 + k * 32, 16, 512, kLayoutSW64)
                                    : make_smem_desc(a0 + k * 32, 16, 1024, kLayoutSW128);
            const uint64_t bd = IMG ? make_smem_desc(b0 + k * 32, 16, 512, kLayoutSW64)
                                    : make_smem_desc(b0 + k * 32, 16, 1024, kLayoutSW128);
            if constexpr (PAIR) mma_ss_2sm(d_tmem, ad, bd, idesc, (kb | k) != 0);
            else mma_ss(d_tmem, ad, bd, idesc, (kb | k) != 0);
          }
          if constexpr (PAIR) mma_commit_2sm(&empty[stage], 0x3);
          else mma_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if constexpr (PAIR) mma_commit_2sm(&tfull[acc], 0x3);
        else mma_commit(&tfull[acc]);
        if (++acc == NACC) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {
    const int quarter = warp & 3;              // TMEM lane quarter this warp may access
    const int half = (EW == 8) ? (warp - 2) >> 2 : 0;  // which column half (EW=8) of the tile
    constexpr int CH = BN / (32 * (EW / 4));            // 32-column chunks per epilogue warp
    constexpr int WCOLS = BN / (EW / 4);                // columns per epilogue warp
    const int et = threadIdx.x - 64;                    // index among the epilogue threads
    for (int i = et; i < p.N; i += 32 * EW) bias_s[i] = __ldg(p.bias + i);
    if (EPI == EPI_F32_RESID_LN || (EPI == EPI_EMBED_COARSE && p.ln_g))
      for (int i = et; i < p.N; i += 32 * EW) { lng_s[i] = __ldg(p.ln_g + i); lnb_s[i] = __ldg(p.ln_b + i); }
    asm volatile("bar.sync 5, %0;" ::"n"(32 * EW) : "memory");  // epilogue warps only
    int acc = 0;
    uint32_t acc_phase = 0;
    uint32_t xph = 0;  // bit b: phase of this warp's staging barrier b
    for (int tile = t_first; tile < t_end; tile += t_step) {
      const int m_blk = m_of(tile), n_blk = BRES ? n_fix : tile % n_tiles;
      // IMG: tile-local rows >= rpt are the MMA's padding rows (never stored): pushed past m_store;
      // PAIR: a ghost tile (m_blk >= m_tiles) likewise
      const int row0 = ((IMG && quarter * 32 + lane >= rpt) || (PAIR && m_blk >= m_tiles)) ? (1 << 30) - lane
                                                                                          : m_blk * rpt + quarter * 32;
      const uint32_t tbase = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + acc * BN + half * WCOLS;
      const int col_base = n_blk * BN + half * WCOLS;
      float s1 = 0.f, s2 = 0.f, sh = 0.f;  // LN row statistics (lane = row): shifted sums around sh
      if constexpr (EPI == EPI_F32_RESID_LN && EW == 8) {
        uint8_t* stg = smem + S::STG_OFF + (warp - 2) * S::STG_BYTES;
        const ResidStage st{stg, 4096, stg + 8192, 2048, xbar + (warp - 2) * 2, &xph};
        const ResidLnArgs la{p.N, p.ln_cap, p.ln_eps};
        resid_ln_tma<CH, true>(la, tmX, tmLN, st, tbase, row0, col_base, M, bias_s, lng_s, lnb_s, ln_stats, quarter,
                               half, lane, &tfull[acc], acc_phase, &tempty[acc]);
      } else if constexpr (kStgOut) {
        constexpr int SB = BRES ? 1 : 2;  // BRES: one staging buffer per warp, one more A stage
        store_bf16_tma<CH, EPI, SB>(tmX, smem + S::STG_OFF + (warp - 2) * 2048 * SB, tbase, row0, col_base, bias_s,
                                    lane, &tfull[acc], acc_phase, &tempty[acc], PAIR && rank ? 0 : -1);
      } else if constexpr (EPI == EPI_F32_RESID || EPI == EPI_F32_RESID_LN) {
        // Residual epilogue, software-pipelined over the 32-column chunks: the residual
        // row segment of chunk c+1 is loaded while chunk c is added and stored, and chunk
        // 0's is requested before the accumulator is even ready.
        const int row = row0 + lane;
        const bool live = row < M;
        float* xrow = p.out_f32 + (size_t)row * p.ld_out + col_base;
        float4 xn[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) xn[i] = live ? reinterpret_cast<const float4*>(xrow)[i] : make_float4(0, 0, 0, 0);
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < CH; ++c) {
          float4 xc[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) xc[i] = xn[i];
          if (c + 1 < CH && live) {
#pragma unroll
            for (int i = 0; i < 8; ++i) xn[i] = reinterpret_cast<const float4*>(xrow + (c + 1) * 32)[i];
          }
          uint32_t r[32];
          tmem_ld32(tbase + c * 32, r);
          tmem_wait_ld();
          if (c + 1 == CH) {  // last TMEM read of this accumulator: release it early
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
          }
          if (live) {
            const int col0 = col_base + c * 32;
            float4* dst = reinterpret_cast<float4*>(xrow + c * 32);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float4 bb = *reinterpret_cast<const float4*>(bias_s + col0 + 4 * i);
              float4 x = xc[i];
              x.x += __uint_as_float(r[4 * i + 0]) + bb.x;
              x.y += __uint_as_float(r[4 * i + 1]) + bb.y;
              x.z += __uint_as_float(r[4 * i + 2]) + bb.z;
              x.w += __uint_as_float(r[4 * i + 3]) + bb.w;
              dst[i] = x;
              if constexpr (EPI == EPI_F32_RESID_LN) {  // shifted sums around the row's first value
                if (c == 0 && i == 0) sh = x.x;
                const float a0 = x.x - sh, a1 = x.y - sh, a2 = x.z - sh, a3 = x.w - sh;
                s1 += (a0 + a1) + (a2 + a3);
                s2 += (a0 * a0 + a1 * a1) + (a2 * a2 + a3 * a3);
              }
            }
          }
        }
      } else {
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < CH; c += 2) {
        uint32_t r0[32], r1[32];
        tmem_ld32(tbase + c * 32, r0);
        if (c + 1 < CH) tmem_ld32(tbase + (c + 1) * 32, r1);
        tmem_wait_ld();
        if (c + 2 >= CH) {  // last TMEM read of this accumulator: release it to the MMA warp early
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (PAIR && rank) mbar_arrive_cluster(&tempty[acc], 0);  // the leader's MMA warp waits
            else mbar_arrive(&tempty[acc]);
          }
        }
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          if (c + q >= CH) break;
          const uint32_t* r = q ? r1 : r0;
          const int col0 = col_base + (c + q) * 32;
          const int row = row0 + lane;
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            const float4 bb = *reinterpret_cast<const float4*>(bias_s + col0 + j);  // smem broadcast
            v[j] = __uint_as_float(r[j]) + bb.x;
            v[j + 1] = __uint_as_float(r[j + 1]) + bb.y;
            v[j + 2] = __uint_as_float(r[j + 2]) + bb.z;
            v[j + 3] = __uint_as_float(r[j + 3]) + bb.w;
          }
          direct_chunk<EPI>(p, v, row, col0, m_store, M, s1, s2, sh, c + q == 0);
        }
      }
      }
      // LayerNorm of the rows just written (RESID_LN direct path; coarse embed + layer-0 LN1
      // when p.ln_g: the embedding rows are read back from L2 and normalised)
      if (((EPI == EPI_F32_RESID_LN && EW != 8) || EPI == EPI_EMBED_COARSE) &&
          (EPI != EPI_EMBED_COARSE || p.ln_g != nullptr)) {
        // row statistics; with EW=8 the two warps sharing these rows exchange halves
        // RESID_LN: per part (this warp's WCOLS columns) mean_h = sh + s1 / n_h, M2_h = s2 - s1^2 / n_h
        // from the shifted sums; with EW = 8 the two halves combine with Chan's formula in a fixed
        // (half 0, half 1) order.  EMBED_COARSE (layer-0 LN1 of the coarse pass) keeps its plain sums
        // (rows = patch embedding + PE, |mean| ~ std, nothing to cancel): with them the coarse pass and
        // a k = 0 refine agree bit for bit (test_refine_k0_reproduces_coarse_pass_bitwise), with the
        // shifted form they did not
        if constexpr (EPI == EPI_EMBED_COARSE) {
          float2 o = make_float2(0.f, 0.f);
          if constexpr (EW == 8) {
            const int r_in_tile = quarter * 32 + lane;
            ln_stats[half * 128 + r_in_tile] = make_float2(s1, s2);
            asm volatile("bar.sync %0, 64;" ::"r"(1 + quarter) : "memory");
            o = ln_stats[(half ^ 1) * 128 + r_in_tile];
            asm volatile("bar.sync %0, 64;" ::"r"(1 + quarter) : "memory");
          }
          const float inv_n = 1.f / (float)p.N;
          sh = (s1 + o.x) * inv_n;                                                  // mean
          s1 = rsqrtf(fmaxf((s2 + o.y) * inv_n - sh * sh, 0.f) + p.ln_eps);        // rstd
        }
        const float n_h = (float)WCOLS;
        const float mean_h = sh + s1 / n_h;
        const float m2_h = fmaxf(s2 - s1 * (s1 / n_h), 0.f);
        float mean = mean_h, m2 = m2_h;
        if constexpr (EW == 8 && EPI != EPI_EMBED_COARSE) {
          const int r_in_tile = quarter * 32 + lane;
          ln_stats[half * 128 + r_in_tile] = make_float2(mean_h, m2_h);
          asm volatile("bar.sync %0, 64;" ::"r"(1 + quarter) : "memory");
          const float2 o = ln_stats[(half ^ 1) * 128 + r_in_tile];
          asm volatile("bar.sync %0, 64;" ::"r"(1 + quarter) : "memory");
          const float2 h0 = half == 0 ? make_float2(mean_h, m2_h) : o;
          const float2 h1 = half == 0 ? o : make_float2(mean_h, m2_h);
          const float dm = h0.x - h1.x;
          mean = 0.5f * (h0.x + h1.x);
          m2 = (h0.y + h1.y) + dm * dm * (0.5f * n_h);
        }
        float rstd = rsqrtf(m2 / (float)p.N + p.ln_eps);
        if constexpr (EPI == EPI_EMBED_COARSE) {
          mean = sh;
          rstd = s1;
        }
        // LN(x) -> bf16 from the x just written (same thread, row = lane)
        const int row = row0 + lane;
        if (row < p.ln_cap) {
          const bool live = row < M;
          const float4* xrow = reinterpret_cast<const float4*>(p.out_f32 + (size_t)row * p.ld_out + col_base);
          float4 xn[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) xn[i] = live ? xrow[i] : make_float4(0, 0, 0, 0);
#pragma unroll 1
          for (int c = 0; c < CH; ++c) {
            const int col0 = col_base + c * 32;
            uint4* hd = reinterpret_cast<uint4*>(p.ln_out + (size_t)row * p.N + col0);
            if (!live) {
#pragma unroll
              for (int i = 0; i < 4; ++i) hd[i] = make_uint4(0, 0, 0, 0);
              continue;
            }
            float4 xc[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) xc[i] = xn[i];
            if (c + 1 < CH) {
#pragma unroll
              for (int i = 0; i < 8; ++i) xn[i] = xrow[(c + 1) * 8 + i];
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
      if (++acc == NACC) { acc = 0; acc_phase ^= 1; }
    }
  }
  if constexpr ((EPI == EPI_F32_RESID_LN || kStgOut) && EW == 8) {
    if (warp >= 2 && lane == 0) bulk_wait0();  // staged TMA stores fully written before exit
  }
  tc_fence_before();
  if constexpr (PAIR) cluster_sync();  // the peer may still arrive on / multicast into this CTA
  else __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    if constexpr (PAIR) tmem_dealloc_2sm<S::TMEM_COLS>(tmem_base);
    else tmem_dealloc<S::TMEM_COLS>(tmem_base);
  }
}

}  // namespace cfd
