// tools/fp32_peak.cu — FP32 throughput microbenchmark on the B200 (the
// roofline denominator of the ALU-bound traversal kernel).
// Independent FFMA chains (scalar, 3-register form) and FFMA2 chains (packed
// f32x2) in a persistent grid of 148 x k blocks; reports FMA/s and FLOP/s
// (1 FMA = 2 FLOP) with CUDA events, plus the SM clock during the run.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp32_peak tools/fp32_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CHAINS = 8;
constexpr int ITERS = 4096;

__global__ void __launch_bounds__(256) k_ffma(float* out, float a, float b) {
  float x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-3f + c;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = __fmaf_rn(x[c], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 12345.f) out[threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) k_ffma2(float* out, float a, float b) {
  unsigned long long x[CHAINS];
  unsigned long long A, Bv;
  asm("mov.b64 %0, {%1, %2};" : "=l"(A) : "f"(a), "f"(a + 1e-7f));
  asm("mov.b64 %0, {%1, %2};" : "=l"(Bv) : "f"(b), "f"(b + 1e-7f));
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) {
    float lo = threadIdx.x * 1e-3f + c, hi = lo + 0.5f;
    asm("mov.b64 %0, {%1, %2};" : "=l"(x[c]) : "f"(lo), "f"(hi));
  }
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[c]) : "l"(A), "l"(Bv));
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(x[c]));
    s += lo + hi;
  }
  if (s == 12345.f) out[threadIdx.x] = s;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount;
  float* out;
  cudaMalloc(&out, 4096);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, threads = 256;
  for (int kind = 0; kind < 2; ++kind) {
    float best = 1e30f;
    for (int rep = 0; rep < 6; ++rep) {
      cudaEventRecord(e0);
      if (kind == 0) k_ffma<<<blocks, threads>>>(out, 0.999f, 1e-3f);
      else k_ffma2<<<blocks, threads>>>(out, 0.999f, 1e-3f);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0 && ms < best) best = ms;
    }
    const double fmas = (double)blocks * threads * ITERS * CHAINS * (kind == 0 ? 1 : 2);
    printf("{\"kind\": \"%s\", \"ms\": %.4f, \"fma_per_s\": %.4e, \"tflops\": %.3f, \"sms\": %d}\n",
           kind == 0 ? "ffma" : "ffma2", best, fmas / (best * 1e-3), 2 * fmas / (best * 1e-3) / 1e12, sms);
  }
  return 0;
}
