// MUFU throughput micro-benchmark (B200): ex2.approx.f32 vs ex2.approx.f16x2 vs
// tanh.approx.f32, results per SM per clock.  nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -o tools/mufu_micro tools/mufu_micro.cu && tools/mufu_micro
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>

constexpr int ITERS = 4096;
constexpr int CH = 8;  // independent chains per thread

__global__ void k_ex2_f32(float* out, long long* cyc) {
  float v[CH];
  for (int i = 0; i < CH; ++i) v[i] = -0.001f * (threadIdx.x + i);
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[i]));
  __syncthreads();
  const long long t1 = clock64();
  float s = 0.f;
  for (int i = 0; i < CH; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_ex2_f16x2(float* out, long long* cyc) {
  uint32_t v[CH];
  for (int i = 0; i < CH; ++i) {
    __half2 h = __floats2half2_rn(-0.001f * (threadIdx.x + i), -0.002f * i);
    v[i] = *reinterpret_cast<uint32_t*>(&h);
  }
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(v[i]));
  __syncthreads();
  const long long t1 = clock64();
  float s = 0.f;
  for (int i = 0; i < CH; ++i) s += __low2float(*reinterpret_cast<__half2*>(&v[i]));
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_cvt_ex2_f16x2(float* out, long long* cyc) {  // the attention sequence: f32 pair -> f16x2 -> ex2
  float a[CH], b[CH];
  uint32_t acc[CH];
  for (int i = 0; i < CH; ++i) { a[i] = -0.001f * (threadIdx.x + i); b[i] = -0.002f * i; acc[i] = 0; }
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      uint32_t h;
      asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(a[i]), "f"(b[i]));
      asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h));
      acc[i] ^= h;
    }
  __syncthreads();
  const long long t1 = clock64();
  float s = 0.f;
  for (int i = 0; i < CH; ++i) s += (float)acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_tanh_f32(float* out, long long* cyc) {
  float v[CH];
  for (int i = 0; i < CH; ++i) v[i] = 0.001f * (threadIdx.x + i);
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) asm volatile("tanh.approx.f32 %0, %0;" : "+f"(v[i]));
  __syncthreads();
  const long long t1 = clock64();
  float s = 0.f;
  for (int i = 0; i < CH; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <typename K>
void run(const char* name, K kern, int results_per_op) {
  float* out;
  long long* cyc;
  const int threads = 512, blocks = 148;
  cudaMalloc(&out, sizeof(float) * threads * blocks);
  cudaMalloc(&cyc, sizeof(long long) * blocks);
  kern<<<blocks, threads>>>(out, cyc);
  kern<<<blocks, threads>>>(out, cyc);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < blocks; ++i) mean += h[i];
  mean /= blocks;
  const double ops = (double)threads * ITERS * CH;
  printf("%-22s %8.2f ops/clk/SM  %8.2f results/clk/SM\n", name, ops / mean, ops * results_per_op / mean);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run("ex2.approx.f32", k_ex2_f32, 1);
  run("ex2.approx.f16x2", k_ex2_f16x2, 2);
  run("cvt.f16x2 + ex2.f16x2", k_cvt_ex2_f16x2, 2);
  run("tanh.approx.f32", k_tanh_f32, 1);
  return 0;
}
