// tc_micro.cu — microbenchmarks of the sm_100a resources the hot kernels lean on:
//   1. TMEM read bandwidth (tcgen05.ld 32x32b.x32) vs number of reading warps per SM
//   2. tcgen05.mma (kind::f16, SS) issue/completion rate for M=128, N in {64,128,256}
//   3. both at once (one MMA thread + 8 TMEM-reading warps), to expose contention
//   4. the attention kernel's MMA mix: per 64-key sub-tile 2 x QK (SS, M=128 N=64 K=16, SW64)
//      + 4 x PV (TS: A = P from TMEM, M=128 N=32 K=16, V MN-major SW64), issued by 1..3
//      threads (one per warpgroup, as in attn4), back to back (throughput) and with a
//      commit + wait after each group (round-trip latency)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2505_23317_b200/csrc tools/tc_micro.cu -o tc_micro
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx.cuh"

using namespace cfd;

__global__ void tmem_ld_bw(int iters, int nwarps, unsigned long long* cyc, uint32_t* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot + (static_cast<uint32_t>((warp & 3) * 32) << 16);
  uint32_t acc = 0;
  const unsigned long long t0 = clock64();
  if (warp < nwarps) {
    for (int i = 0; i < iters; ++i) {
      uint32_t r[32];
      tmem_ld32(tm + ((i * 32 + warp * 64) & 511), r);
      tmem_wait_ld();
#pragma unroll
      for (int k = 0; k < 32; ++k) acc ^= r[k];
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (acc == 0x12345678u) sink[threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(slot);
}

template <int N>
__global__ void mma_rate(int iters, int ld_warps, unsigned long long* cyc, uint32_t* sink) {
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (128 + 256) * 64 * 2 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (warp == 0) tmem_alloc<512>(&slot);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  const unsigned long long t0 = clock64();
  uint32_t acc = 0;
  if (warp == 0) {
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc_bf16(128, N, 0);
      const uint32_t a = smem_u32(sm), b = smem_u32(sm + 128 * 64 * 2);
      for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          mma_ss(tm, make_smem_desc(a + k * 32, 16, 1024, kLayoutSW128), make_smem_desc(b + k * 32, 16, 1024, kLayoutSW128),
                 idesc, 1);
      }
      mma_commit(&bar);
      mbar_wait(&bar, 0);
    }
    __syncwarp();
  } else if (warp - 1 < ld_warps) {
    // TMEM readers on the columns the MMA does not write (256..511)
    const uint32_t t = tm + (static_cast<uint32_t>((warp & 3) * 32) << 16) + 256;
    for (int i = 0; i < iters; ++i) {
      uint32_t r[32];
      tmem_ld32(t + ((i * 32) & 255), r);
      tmem_wait_ld();
#pragma unroll
      for (int k = 0; k < 32; ++k) acc ^= r[k];
    }
  }
  const unsigned long long t1 = clock64();
  __syncthreads();
  if (warp == 0 && lane == 0) cyc[blockIdx.x] = t1 - t0;
  if (warp > 0 && lane == 0) cyc[gridDim.x * warp + blockIdx.x] = t1 - t0;
  if (acc == 0x12345678u) sink[threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(slot);
}

// one issuing thread per warp w < nissue; TMEM region w*128: S 64 | P 32 | O 32 (as attn4)
__global__ void attn_mma_mix(int iters, int nissue, int wait_each, unsigned long long* cyc) {
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar[4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 3 * 8192 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (warp == 0) tmem_alloc<512>(&slot);
  if (threadIdx.x == 0) { for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1); fence_barrier_init(); }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const unsigned long long t0 = clock64();
  if (warp < nissue && lane == 0) {
    const uint32_t tb = slot + warp * 128;
    const uint32_t qa = smem_u32(sm), ka = smem_u32(sm + 8192), va = smem_u32(sm + 16384);
    constexpr uint32_t idesc_s = make_idesc_bf16(128, 64, 0);
    constexpr uint32_t idesc_o = make_idesc_bf16(128, 32, 1);
    uint32_t ph = 0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 2; ++k)
        mma_ss(tb, make_smem_desc(qa + k * 32, 16, 512, kLayoutSW64), make_smem_desc(ka + k * 32, 16, 512, kLayoutSW64),
               idesc_s, k);
      if (wait_each) { mma_commit(&bar[warp]); mbar_wait(&bar[warp], ph); ph ^= 1; tc_fence_after(); }
#pragma unroll
      for (int k = 0; k < 4; ++k)
        mma_ts(tb + 96, tb + 64 + k * 8, make_smem_desc(va + k * 1024, 4096, 512, kLayoutSW64), idesc_o, 1);
      if (wait_each) { mma_commit(&bar[warp]); mbar_wait(&bar[warp], ph); ph ^= 1; tc_fence_after(); }
    }
    mma_commit(&bar[warp]);
    mbar_wait(&bar[warp], ph);
  }
  const unsigned long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(slot);
}

// split roles: warp 0 issues only QK pairs (into S), warp 1 only PV quads (into O); per-role
// cycles per group, to see whether a PV-issuing thread holds up a QK-issuing one
__global__ void attn_mma_split(int iters, int mode, unsigned long long* cyc) {
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar[4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 3 * 8192 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (warp == 0) tmem_alloc<512>(&slot);
  if (threadIdx.x == 0) { for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1); fence_barrier_init(); }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const unsigned long long t0 = clock64();
  const uint32_t tb = slot;
  const uint32_t qa = smem_u32(sm), ka = smem_u32(sm + 8192), va = smem_u32(sm + 16384);
  constexpr uint32_t idesc_s = make_idesc_bf16(128, 64, 0);
  constexpr uint32_t idesc_o = make_idesc_bf16(128, 32, 1);
  // mode 0: warp 0 QK only; mode 1: warp 1 PV only; mode 2: both concurrently
  if (lane == 0 && ((warp == 0 && mode != 1) || (warp == 1 && mode != 0))) {
    for (int i = 0; i < iters; ++i) {
      if (warp == 0) {
#pragma unroll
        for (int k = 0; k < 2; ++k)
          mma_ss(tb, make_smem_desc(qa + k * 32, 16, 512, kLayoutSW64), make_smem_desc(ka + k * 32, 16, 512, kLayoutSW64),
                 idesc_s, k);
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          mma_ts(tb + 256, tb + 128 + k * 8, make_smem_desc(va + k * 1024, 4096, 512, kLayoutSW64), idesc_o, 1);
      }
    }
    mma_commit(&bar[warp]);
    mbar_wait(&bar[warp], 0);
  }
  const unsigned long long t1 = clock64();
  if (lane == 0 && warp < 2) cyc[blockIdx.x * 2 + warp] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(slot);
}

// cycles per tcgen05.mma (M = 128, K = 16, bf16 -> f32, SW64 operands as in the attention
// kernel) for N in {32, 64, 128}: SS (A = Q/K tile from smem) or TS (A = P from TMEM)
template <int N, bool TS>
__global__ void mma_shape(int iters, unsigned long long* cyc) {
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 3 * 8192 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (warp == 0) tmem_alloc<512>(&slot);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const unsigned long long t0 = clock64();
  if (warp == 0 && lane == 0) {
    const uint32_t qa = smem_u32(sm), ka = smem_u32(sm + 8192);
    constexpr uint32_t idesc = make_idesc_bf16(128, N, TS ? 1 : 0);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (TS)
          mma_ts(slot + 256, slot + k * 8, make_smem_desc(ka + k * 1024, 4096, 512, kLayoutSW64), idesc, 1);
        else
          mma_ss(slot + 256, make_smem_desc(qa + (k & 1) * 32, 16, 512, kLayoutSW64),
                 make_smem_desc(ka + (k & 1) * 32, 16, 512, kLayoutSW64), idesc, 1);
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
  }
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(slot);
}

template <int N, bool TS>
void run_shape(int grid, unsigned long long* cyc, unsigned long long* h) {
  const int smem = 3 * 8192 + 1024, iters = 2048;
  cudaFuncSetAttribute(mma_shape<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mma_shape<N, TS><<<grid, 128, smem>>>(iters, cyc);
  cudaDeviceSynchronize();
  cudaMemcpy(h, cyc, sizeof(unsigned long long) * grid, cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < grid; ++i) c += h[i];
  c /= grid;
  printf("mma shape M=128 N=%3d K=16 %s: %.1f cycles/instr  FLOP/clk/SM=%.0f\n", N, TS ? "TS (A in TMEM)" : "SS",
         c / (4.0 * iters), 2.0 * 128 * N * 16 * 4 * iters / c);
}

int main() {
  unsigned long long* cyc;
  uint32_t* sink;
  const int grid = 148;
  cudaMalloc(&cyc, sizeof(unsigned long long) * grid * 32);
  cudaMalloc(&sink, 4096);
  unsigned long long h[148 * 32];
  run_shape<32, false>(grid, cyc, h);
  run_shape<64, false>(grid, cyc, h);
  run_shape<128, false>(grid, cyc, h);
  run_shape<32, true>(grid, cyc, h);
  run_shape<64, true>(grid, cyc, h);
  run_shape<128, true>(grid, cyc, h);
  if (getenv("TC_SHAPES_ONLY")) return 0;
  // 1. TMEM read bandwidth
  for (int nw : {1, 2, 4, 8, 12, 16}) {
    const int iters = 4096;
    tmem_ld_bw<<<grid, 512>>>(iters, nw, cyc, sink);
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, sizeof(unsigned long long) * grid, cudaMemcpyDeviceToHost);
    double c = 0;
    for (int i = 0; i < grid; ++i) c += h[i];
    c /= grid;
    const double bytes = (double)nw * iters * 32 * 32 * 4;
    printf("tmem_ld  warps=%2d  cycles=%.0f  bytes/clk/SM=%.1f\n", nw, c, bytes / c);
  }
  // 2./3. MMA rate alone and with TMEM readers
  const int smem = (128 + 256) * 64 * 2 + 1024;
  cudaFuncSetAttribute(mma_rate<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(mma_rate<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(mma_rate<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int ldw : {0, 4, 8}) {
    for (int n : {64, 128, 256}) {
      const int iters = 2048;
      if (n == 64) mma_rate<64><<<grid, 32 * 9, smem>>>(iters, ldw, cyc, sink);
      if (n == 128) mma_rate<128><<<grid, 32 * 9, smem>>>(iters, ldw, cyc, sink);
      if (n == 256) mma_rate<256><<<grid, 32 * 9, smem>>>(iters, ldw, cyc, sink);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h, cyc, sizeof(unsigned long long) * grid * 9, cudaMemcpyDeviceToHost);
      double c = 0, cl = 0;
      for (int i = 0; i < grid; ++i) { c += h[i]; if (ldw) cl += h[grid + i]; }
      c /= grid; cl /= grid;
      const double flop = 2.0 * 128 * n * 16 * 4 * iters;
      printf("mma N=%3d ld_warps=%d  mma cycles=%.0f  FLOP/clk/SM=%.0f (peak ~8192)  cyc/instr=%.1f", n, ldw, c,
             flop / c, c / (4.0 * iters));
      if (ldw) printf("  | ld warp cycles=%.0f  ld bytes/clk/SM=%.1f", cl, (double)ldw * iters * 4096 / cl);
      printf("\n");
    }
  }
  // 4. attention MMA mix
  const int smem4 = 3 * 8192 + 1024;
  cudaFuncSetAttribute(attn_mma_mix, cudaFuncAttributeMaxDynamicSharedMemorySize, smem4);
  for (int we : {0, 1}) {
    for (int ni : {1, 2, 3}) {
      const int iters = 1024;
      attn_mma_mix<<<grid, 128, smem4>>>(iters, ni, we, cyc);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h, cyc, sizeof(unsigned long long) * grid, cudaMemcpyDeviceToHost);
      double c = 0;
      for (int i = 0; i < grid; ++i) c += h[i];
      c /= grid;
      const double flop = (double)ni * iters * (2 * 2.0 * 128 * 64 * 16 + 4 * 2.0 * 128 * 32 * 16);
      printf("attn mix: issuers=%d wait_each=%d  cycles per sub-tile group (2 QK + 4 PV) per issuer=%.1f  "
             "per SM=%.1f  FLOP/clk/SM=%.0f\n", ni, we, c / iters, c / (iters * ni), flop / c);
    }
  }
  cudaFuncSetAttribute(attn_mma_split, cudaFuncAttributeMaxDynamicSharedMemorySize, smem4);
  for (int mode : {0, 1, 2}) {
    const int iters = 1024;
    attn_mma_split<<<grid, 64, smem4>>>(iters, mode, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, cyc, sizeof(unsigned long long) * grid * 2, cudaMemcpyDeviceToHost);
    double c0 = 0, c1 = 0;
    for (int i = 0; i < grid; ++i) { c0 += h[2 * i]; c1 += h[2 * i + 1]; }
    printf("split roles mode=%d (0 QK only, 1 PV only, 2 both): QK warp %.1f cyc/pair, PV warp %.1f cyc/quad\n", mode,
           mode != 1 ? c0 / grid / iters : 0.0, mode != 0 ? c1 / grid / iters : 0.0);
  }
  return 0;
}
