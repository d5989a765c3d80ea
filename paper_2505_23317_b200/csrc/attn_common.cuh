// attn_common.cuh — softmax arithmetic shared by the attention kernels (dh = 32): packed
// f32x2 FMA / ADD wrappers, the 3-input max, the FMA-pipe exp2 polynomial, the exp chunk of
// one score row (MUFU / polynomial split) and the item decode of ragged batches.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "ptx.cuh"
#include "attn_tc.cuh"

namespace cfd {

constexpr int ATTN_MAX_T = 4096;  // tasks per persistent attention launch (prefix table in smem)

// Debug-library pipeline trace (-DCFD_TRACE, read by cfdx_attn_trace): clock64() per
// (CTA < 148, warpgroup w < 4, item it < 2, sub-tile u < 12) at word ((b*4+w)*2+it)*12+u)*8 + ev:
//   0 softmax: s_full passed   1 S in registers   2 row max done   3 exps done
//   4 o_full passed (+ O rescale)   5 p_full arrived   6 MMA: QK(u) issued   7 MMA: PV(u) issued
// (softmax events from warp 0 of the warpgroup, lane 0); word ATTN_TRACE_T0 + b = kernel start.
constexpr int ATTN_TRACE_T0 = 148 * 4 * 2 * 12 * 8;
constexpr int ATTN_TRACE_WORDS = ATTN_TRACE_T0 + 148;
#ifdef CFD_TRACE
__device__ unsigned long long g_attn_trace[ATTN_TRACE_WORDS];
#define ATTN_TR(w_, it_, u_, ev_)                                                                  \
  do {                                                                                            \
    if ((it_) < 2 && (u_) < 12 && blockIdx.x < 148)                                               \
      g_attn_trace[(((blockIdx.x * 4 + (w_)) * 2 + (it_)) * 12 + (u_)) * 8 + (ev_)] = clock64();  \
  } while (0)
#else
#define ATTN_TR(w_, it_, u_, ev_) do { } while (0)
#endif


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

// The same with a degree-4 polynomial (max rel. error 2.7e-6 in fp32 Horner): for the criticality
// score, a sum of probabilities compared against its closed form (constant frame: exactly 1/Nc),
// where the degree-3 error (7.5e-5) would show; P feeding a bf16 MMA does not need it.
__device__ __forceinline__ void exp2_poly2_d4(float& y0, float& y1, float x0, float x1) {
  constexpr float kMagic = 12582912.0f;
  x0 = fmaxf(x0, -126.f);
  x1 = fmaxf(x1, -126.f);
  float t0, t1, r0, r1, f0, f1, p0, p1;
  add2(t0, t1, x0, x1, kMagic, kMagic);
  add2(r0, r1, t0, t1, -kMagic, -kMagic);
  add2(f0, f1, x0, x1, -r0, -r1);
  fma2(p0, p1, f0, f1, 0.009570102f, 0.009570102f, 0.05591786f, 0.05591786f);
  fma2(p0, p1, p0, p1, f0, f1, 0.24024744f, 0.24024744f);
  fma2(p0, p1, p0, p1, f0, f1, 0.69312179f, 0.69312179f);
  fma2(p0, p1, p0, p1, f0, f1, 0.99999928f, 0.99999928f);
  y0 = __int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23));
  y1 = __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23));
}

// One 32-column chunk of a score row: p = 2^(s*c - m) for NPAIR (16) pairs, running pair sums,
// bf16x2-packed results written to sr[0..NPAIR-1].  Pairs [NPAIR-NPP, NPAIR) use the polynomial.
template <int NPP, int NPAIR = 16>
__device__ __forceinline__ void exp_chunk(uint32_t* sr, float c, float neg, float& sum0, float& sum1) {
#pragma unroll
  for (int i = 0; i < NPAIR; ++i) {
    float x0, x1, p0, p1;
    fma2(x0, x1, __uint_as_float(sr[2 * i]), __uint_as_float(sr[2 * i + 1]), c, c, neg, neg);
#ifdef CFD_ABLATE_EXP  // timing experiment only (wrong results): no exponential at all
    p0 = x0;
    p1 = x1;
#else
    if (i >= NPAIR - NPP) {
      exp2_poly2(p0, p1, x0, x1);
    } else {
      p0 = ex2_approx(x0);
      p1 = ex2_approx(x1);
    }
#endif
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

}  // namespace cfd
