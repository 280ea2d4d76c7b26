// Bucketing of the symmetric near pairs by quadrature tier (CUB radix sort
// on a 4-bit key), so every k_near_sym launch runs one tier n with a uniform
// (pair, point) thread layout.
#include <cub/cub.cuh>

#include "ebem_kernels.h"

namespace ebem_gpu {

void sort_pairs_by_class(unsigned char* keys_in, unsigned char* keys_out,
                         int* vals_in, int* vals_out, long long n, void** temp,
                         size_t* temp_bytes, cudaStream_t st) {
  if (n <= 0) return;
  size_t need = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, need, keys_in, keys_out, vals_in,
                                  vals_out, int(n), 0, 4, st);
  if (need > *temp_bytes) {
    if (*temp) cudaFree(*temp);
    cudaMalloc(temp, need + need / 4);
    *temp_bytes = need + need / 4;
  }
  cub::DeviceRadixSort::SortPairs(*temp, *temp_bytes, keys_in, keys_out,
                                  vals_in, vals_out, int(n), 0, 4, st);
}

__global__ void k_class_bounds(const unsigned char* __restrict__ k, long long n,
                               int* __restrict__ bounds) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i > n) return;
  const int cur = i < n ? k[i] : kSymClasses;
  const int prev = i > 0 ? k[i - 1] : -1;
  // classes prev+1 .. cur start at i
  for (int c = prev + 1; c <= cur; ++c) bounds[c] = int(i);
}

void launch_class_bounds(const unsigned char* sorted_keys, long long n,
                         int* bounds, cudaStream_t st) {
  k_class_bounds<<<(unsigned)((n + 1 + 255) / 256), 256, 0, st>>>(sorted_keys, n,
                                                                  bounds);
}

}  // namespace ebem_gpu
