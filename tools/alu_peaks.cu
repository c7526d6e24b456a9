// ALU peak microbenchmark for the roofline denominators: DFMA, FFMA and FP64 DMMA
// (mma.sync.m8n8k4.f64) throughput on all SMs, plus the SM clock the run saw (clock64 over
// globaltimer).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o alu_peaks alu_peaks.cu
// Output: one JSON line.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>

constexpr int ITERS = 4096;
constexpr int CH = 8;   // independent chains per thread

template <typename T>
__global__ void fma_kernel(T* out, T a, T b, unsigned long long* cyc, unsigned long long* ns) {
  T acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = T(threadIdx.x + c);
  unsigned long long c0 = clock64(), t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], a, b);
  }
  unsigned long long c1 = clock64(), t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  T s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == T(12345.678)) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) { *cyc = c1 - c0; *ns = t1 - t0; }
}

__global__ void dmma_kernel(double* out, double a0, unsigned long long* cyc, unsigned long long* ns) {
  double acc[CH][2];
  double a = a0 + threadIdx.x, b = a0 * 0.5;
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c][0] = acc[c][1] = 0.0;
  unsigned long long c0 = clock64(), t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a), "d"(b));
  }
  unsigned long long c1 = clock64(), t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1];
  if (s == 12345.678) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) { *cyc = c1 - c0; *ns = t1 - t0; }
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  const int sms = prop.multiProcessorCount;
  double* d;
  unsigned long long *cyc, *ns, hc, hn;
  cudaMalloc(&d, 64);
  cudaMalloc(&cyc, 8);
  cudaMalloc(&ns, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int threads = 512, blocks = sms * 4;
  auto run = [&](auto launch, double flop_per_thread_iter, double& tflops, double& mhz) {
    for (int w = 0; w < 3; ++w) launch();
    cudaEventRecord(e0);
    const int reps = 10;
    for (int r = 0; r < reps; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&hn, ns, 8, cudaMemcpyDeviceToHost);
    const double flop = double(reps) * blocks * threads * ITERS * CH * flop_per_thread_iter;
    tflops = flop / (ms * 1e-3) / 1e12;
    mhz = double(hc) / double(hn) * 1e3;
  };
  double f64, f32, mma, c64, c32, cmma;
  run([&] { fma_kernel<double><<<blocks, threads>>>(d, 1.0000001, 1e-9, cyc, ns); }, 2.0, f64, c64);
  run([&] { fma_kernel<float><<<blocks, threads>>>((float*)d, 1.0000001f, 1e-9f, cyc, ns); }, 2.0, f32, c32);
  // one m8n8k4 per warp = 256 MACs = 512 flop; per thread 16 flop
  run([&] { dmma_kernel<<<blocks, threads>>>(d, 1.0000001, cyc, ns); }, 16.0, mma, cmma);
  cudaError_t err = cudaGetLastError();
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"dfma_tflops\": %.3f, \"dfma_sm_mhz\": %.0f, \"ffma_tflops\": %.3f, "
         "\"ffma_sm_mhz\": %.0f, \"dmma_m8n8k4_tflops\": %.3f, \"dmma_sm_mhz\": %.0f, \"err\": \"%s\"}\n",
         prop.name, sms, f64, c64, f32, c32, mma, cmma, cudaGetErrorString(err));
  return 0;
}
