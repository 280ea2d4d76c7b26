// FP64 MMA (mma.sync m8n8k4) throughput vs DFMA, alone and concurrently
// (development aid): does DMMA use a pipe separate from DFMA on sm_100a?
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

template <int MODE>  // 0 dmma only, 1 dfma only, 2 both (half warps each... same warp interleaved)
__global__ void k(double* out, int iters) {
  double acc[8][2];
  double f[8];
  for (int i = 0; i < 8; ++i) { acc[i][0] = acc[i][1] = 0.0; f[i] = threadIdx.x * 1e-3 + i; }
  const double a = 1.0 + threadIdx.x * 1e-9, b = 0.999;
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0 || MODE == 2) {
#pragma unroll
      for (int i = 0; i < 8; ++i) dmma(acc[i], a, b);
    }
    if (MODE == 1 || MODE == 2) {
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int i = 0; i < 8; ++i) f[i] = fma(f[i], b, a);
    }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1] + f[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double* o;
  cudaMalloc(&o, 148 * 8 * 1024 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 2000, blocks = 148 * 4, threads = 256;
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<blocks, threads>>>(o, iters);
      if (mode == 1) k<1><<<blocks, threads>>>(o, iters);
      if (mode == 2) k<2><<<blocks, threads>>>(o, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      // dmma m8n8k4: 8*8*4*2 = 512 flops per warp-instr; dfma: 2 flops per thread
      const double warps = blocks * threads / 32.0;
      const double fl_mma = (mode != 1) ? warps * iters * 8 * 512.0 : 0;
      const double fl_fma = (mode != 0) ? blocks * threads * double(iters) * 32 * 2.0 : 0;
      if (rep) printf("mode %d: %.3f ms  dmma %.1f TF  dfma %.1f TF\n", mode, ms, fl_mma / ms / 1e9, fl_fma / ms / 1e9);
    }
  }
  return 0;
}
