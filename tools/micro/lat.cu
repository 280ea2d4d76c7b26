// Latency microbenchmarks (development aid): dependent DFMA / DADD / SHFL /
// MUFU chains timed with clock64 on one warp.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(double* out, long long* cyc, double a, double b) {
  double x = a, y = b;
  long long t0 = clock64();
  #pragma unroll 1
  for (int i = 0; i < 1000; ++i) { x = fma(x, y, a); x = fma(x, y, a); x = fma(x, y, a); x = fma(x, y, a); }
  long long t1 = clock64();
  #pragma unroll 1
  for (int i = 0; i < 1000; ++i) { x = x + y; x = x + a; x = x + y; x = x + a; }
  long long t2 = clock64();
  #pragma unroll 1
  for (int i = 0; i < 1000; ++i) { x += __shfl_xor_sync(0xffffffffu, x, 1); x += __shfl_xor_sync(0xffffffffu, x, 2); }
  long long t3 = clock64();
  #pragma unroll 1
  for (int i = 0; i < 1000; ++i) { x = rsqrt(x * x + 1.0); }
  long long t4 = clock64();
  #pragma unroll 1
  for (int i = 0; i < 1000; ++i) { x = 1.0 / (x + 1.5); }
  long long t5 = clock64();
  float f = (float)a;
  #pragma unroll 1
  for (int i = 0; i < 1000; ++i) { f = fmaf(f, (float)b, (float)a); f = fmaf(f, (float)b, (float)a); f = fmaf(f, (float)b, (float)a); f = fmaf(f, (float)b, (float)a); }
  long long t6 = clock64();
  out[threadIdx.x] = x + f;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5; }
}

int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 1024); cudaMallocManaged(&c, 64);
  for (int w : {32, 256, 1024}) {
    k<<<1, w>>>(o, c, 0.5, 0.999);
    cudaDeviceSynchronize();
    printf("threads %4d: DFMA %.1f  DADD %.1f  SHFL+DADD %.1f  rsqrt(d) %.1f  1/x(d) %.1f  FFMA %.1f cycles/op\n", w,
           c[0] / 4000.0, c[1] / 4000.0, c[2] / 2000.0, c[3] / 1000.0, c[4] / 1000.0, c[5] / 4000.0);
  }
  return 0;
}
