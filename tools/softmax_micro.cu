// softmax_micro.cu — throughput ceiling of the attention kernels' softmax body on one SM, with
// no MMAs and no barriers: each softmax warp repeatedly loads a 64-column S row block from TMEM
// (tcgen05.ld), takes the row max, exponentiates (exp_chunk: MUFU / FMA-pipe polynomial split),
// row-sums and stores P back (tcgen05.st), exactly the instruction stream of one sub-tile of
// attn4 / attn7.  Reports score elements per clock per SM for W warps (W / 4 per SMSP).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2505_23317_b200/csrc tools/softmax_micro.cu -o tools/softmax_micro
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include "attn_common.cuh"

using namespace cfd;

// exp_chunk with the bf16 pack by truncation (PRMT of the two high halves) instead of F2FP:
// tests whether the F2FP conversions compete with MUFU for the XU pipe
template <int NPP>
__device__ __forceinline__ void exp_chunk_trunc(uint32_t* sr, float c, float neg, float& sum0, float& sum1) {
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
    sr[i] = __byte_perm(__float_as_uint(p0), __float_as_uint(p1), 0x7632);
  }
}

template <int NPP, bool SKIPMAX = false, bool TRUNC = false>
__global__ void __launch_bounds__(512, 1) softmax_body(int iters, int nwarps, unsigned long long* cyc, float* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot + (static_cast<uint32_t>((warp & 3) * 32) << 16) + (warp >> 2) * 128;
  // fill S with finite values
  {
    uint32_t v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __float_as_uint(0.01f * (float)((lane * 7 + i * 13) % 97) - 0.3f);
#pragma unroll
    for (int c = 0; c < 64; c += 16) tmem_st16(tm + c, v);
    tmem_wait_st();
  }
  __syncthreads();
  const float c = 0.2550348616f;
  float m_run = -INFINITY, l_run = 0.f;
  const unsigned long long t0 = clock64();
  if (warp < nwarps) {
    for (int it = 0; it < iters; ++it) {
      uint32_t sr[64];
      tmem_ld32(tm, *reinterpret_cast<uint32_t(*)[32]>(sr));
      tmem_ld32(tm + 32, *reinterpret_cast<uint32_t(*)[32]>(sr + 32));
      tmem_wait_ld();
      float m0 = -INFINITY, m1 = -INFINITY, m2 = -INFINITY, m3 = -INFINITY;
      if (SKIPMAX) {
        m0 = m_run == -INFINITY ? 0.f : m_run / c;
      } else
#pragma unroll
      for (int i = 0; i < 64; i += 8) {
        m0 = fmax3(m0, __uint_as_float(sr[i]), __uint_as_float(sr[i + 1]));
        m1 = fmax3(m1, __uint_as_float(sr[i + 2]), __uint_as_float(sr[i + 3]));
        m2 = fmax3(m2, __uint_as_float(sr[i + 4]), __uint_as_float(sr[i + 5]));
        m3 = fmax3(m3, __uint_as_float(sr[i + 6]), __uint_as_float(sr[i + 7]));
      }
      const float m_cand = fmax3(m0, m1, fmaxf(m2, m3)) * c;
      const bool upd = (m_run == -INFINITY) || (m_cand > m_run + 8.0f);
      const float alpha = upd ? ((m_run == -INFINITY) ? 0.f : ex2_approx(m_run - m_cand)) : 1.f;
      if (upd) m_run = m_cand;
      const float neg = -m_run;
      float sum0 = 0.f, sum1 = 0.f, sum2 = 0.f, sum3 = 0.f;
      if (TRUNC) {
        exp_chunk_trunc<NPP>(sr, c, neg, sum0, sum1);
        exp_chunk_trunc<NPP>(sr + 32, c, neg, sum2, sum3);
      } else {
        exp_chunk<NPP>(sr, c, neg, sum0, sum1);
        exp_chunk<NPP>(sr + 32, c, neg, sum2, sum3);
      }
      l_run = l_run * alpha + ((sum0 + sum1) + (sum2 + sum3));
      if (SKIPMAX && __any_sync(0xffffffffu, (sum0 + sum1) + (sum2 + sum3) > 256.f)) m_run += 1e-3f;  // the check
      tmem_st16(tm + 64, *reinterpret_cast<const uint32_t(*)[16]>(sr));
      tmem_st16(tm + 80, *reinterpret_cast<const uint32_t(*)[16]>(sr + 32));
      tmem_wait_st();
    }
  }
  const unsigned long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (l_run == 1234.5f) sink[threadIdx.x] = l_run;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(slot);
}

template <int NPP, bool SKIPMAX = false, bool TRUNC = false>
void run(int nw, unsigned long long* cyc, float* sink) {
  const int grid = 148, iters = 2000;
  softmax_body<NPP, SKIPMAX, TRUNC><<<grid, 512>>>(iters, nw, cyc, sink);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return; }
  unsigned long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double cy = 0;
  for (int i = 0; i < grid; ++i) cy += h[i];
  cy /= grid;
  const double elems = (double)nw * 32 * 64 * iters;
  printf("softmax body%s%s NPP=%d warps=%2d (%d per SMSP): %.1f cycles per warp-subtile, %.2f score elements/clk/SM\n",
         SKIPMAX ? " (no max pass)" : "", TRUNC ? " (PRMT pack)" : "", NPP, nw, nw / 4, cy / iters, elems / cy);
}

int main(int argc, char** argv) {
  // optional argument: run only that warp count (for ncu captures of one configuration)
  const int only = argc > 1 ? atoi(argv[1]) : 0;
  unsigned long long* cyc;
  float* sink;
  cudaMalloc(&cyc, sizeof(unsigned long long) * 148);
  cudaMalloc(&sink, 4096 * 4);
  for (int nw : {4, 8, 12, 16}) {
    if (only && nw != only) continue;
    run<0>(nw, cyc, sink);
    run<4>(nw, cyc, sink);
    run<6>(nw, cyc, sink);
    run<8>(nw, cyc, sink);
    run<4, true>(nw, cyc, sink);
    run<6, true>(nw, cyc, sink);
    run<0, false, true>(nw, cyc, sink);
    run<2, false, true>(nw, cyc, sink);
    run<4, false, true>(nw, cyc, sink);
  }
  return 0;
}
