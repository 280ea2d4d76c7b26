// Batched CPQR timing on synthetic R factors (development aid):
//   nvcc ... cpqr_bench.cu ../../paper_2411_18026_b200/csrc/build/ebem_qr.o
//            ../../paper_2411_18026_b200/csrc/build/ebem_dense.o
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2411_18026_b200/csrc/ebem_dense.h"

using namespace ebem_gpu;

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 50;
  const int rows = argc > 2 ? atoi(argv[2]) : n;
  const int count = argc > 3 ? atoi(argv[3]) : 16384;
  dense_init();
  std::vector<double> h(2 * size_t(rows) * n);
  srand(1);
  for (auto& x : h) x = rand() / double(RAND_MAX) - 0.5;
  // graded columns: singular values ~ 10^(-16 j / n)
  for (int j = 0; j < n; ++j) {
    double s = 1.0;
    for (int q = 0; q < j; ++q) s *= 0.6;
    for (int i = 0; i < rows; ++i) { h[2 * (size_t(j) * rows + i)] *= s; h[2 * (size_t(j) * rows + i) + 1] *= s; }
  }
  double *a, *rd, *ro; int *jp, *st;
  cudaMalloc(&a, h.size() * 8 * size_t(count) / count);
  cudaMemcpy(a, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaMalloc(&rd, 8 * size_t(count) * (n + 1));
  cudaMalloc(&ro, 16 * size_t(count) * n * n);
  cudaMalloc(&jp, 4 * size_t(count) * (n + 1));
  cudaMalloc(&st, 4 * size_t(count));
  const bool in_smem = size_t(rows) * n * 16 <= size_t(kSmemCap);
  double2* gws = nullptr;
  if (!in_smem) cudaMalloc(&gws, 16 * size_t(rows) * n * count);
  std::vector<CpqrTask> t(count);
  for (int i = 0; i < count; ++i) {
    CpqrTask& x = t[i];
    x = CpqrTask{};
    x.src = a; x.rows = rows; x.n = n; x.ld = rows; x.in_smem = in_smem;
    x.stop_rel = 1e-14; x.jpvt = jp + size_t(i) * (n + 1); x.rdiag = rd + size_t(i) * (n + 1);
    x.steps = st + i; x.r_out = ro + 2 * size_t(i) * n * n; x.r_ld = n;
    x.ws_off = in_smem ? 0 : (long long)i * rows * n;
  }
  CpqrTask* dt;
  cudaMalloc(&dt, sizeof(CpqrTask) * count);
  cudaMemcpy(dt, t.data(), sizeof(CpqrTask) * count, cudaMemcpyHostToDevice);
  const size_t smem = in_smem ? size_t(rows) * n * 16 : 0;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    launch_cpqr_team(dt, count, smem, gws, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    int steps; cudaMemcpy(&steps, st, 4, cudaMemcpyDeviceToHost);
    if (rep) printf("n %d rows %d count %d: %.3f ms, steps %d, %.0f cycles/step/CTA-wave\n", n, rows, count, ms, steps,
                    ms * 1e-3 * 1.965e9 / steps);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
