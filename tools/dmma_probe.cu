// Microbenchmark: does the FP64 tensor path (mma.sync m8n8k4 f64, DMMA) issue concurrently with
// the FP64 FMA pipe (DFMA) on sm_100a?  Three kernels: DFMA chains only, DMMA chains only, and
// both interleaved in every warp.  If the mixed kernel's time is ~max(dfma, dmma) the units are
// separate; if ~sum they share the pipe.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gpurun_out/dmma_probe tools/dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int NF, int NM>
__global__ void __launch_bounds__(256) probe(double* out, int iters, double seed) {
  double f[8], c[8];
  double a = seed + threadIdx.x * 1e-9, b = seed * 0.5;
#pragma unroll
  for (int i = 0; i < 8; ++i) { f[i] = seed + i; c[i] = seed - i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
#pragma unroll
      for (int i = 0; i < NF; ++i) f[i] = fma(f[i], 0.999999999, 1e-12);
#pragma unroll
      for (int i = 0; i < NM; ++i) dmma(c[2 * i], c[2 * i + 1], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += f[i] + c[i];
  if (s == 12345.678) out[0] = s;
}

template <int NF, int NM>
float run(double* d, int iters) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  dim3 g(sms * 8), b(256);
  probe<NF, NM><<<g, b>>>(d, 10, 1.0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<NF, NM><<<g, b>>>(d, iters, 1.0);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double threads = (double)g.x * b.x;
  double dfma_flops = threads * iters * 4 * NF * 2;
  double dmma_flops = threads / 32 * iters * 4 * NM * 512;
  printf("NF=%d NM=%d: %.3f ms  dfma %.2f TF/s  dmma %.2f TF/s  total %.2f TF/s\n", NF, NM, ms,
         dfma_flops / ms / 1e9, dmma_flops / ms / 1e9, (dfma_flops + dmma_flops) / ms / 1e9);
  return ms;
}

int main() {
  double* d; cudaMalloc(&d, 64);
  const int it = 20000;
  run<8, 0>(d, it);
  run<0, 4>(d, it);
  run<0, 2>(d, it);
  run<8, 1>(d, it);
  run<8, 2>(d, it);
  run<8, 4>(d, it);
  run<4, 2>(d, it);
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
