// tools/cub_sort_yardstick.cu -- NOT product code: a yardstick for the a5
// radix sort (VERDICT r1 "Next round" 4). Times CUB's DeviceRadixSort::SortPairs
// (32-bit keys, 32-bit values, stable LSD onesweep, all 32 bits) on uniform
// random keys at the chunk counts of our frames, so the per-pass efficiency of
// the hand-written k_onesweep can be judged against the library yardstick.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/cub_sort_yardstick.cu -o /tmp/cubsort
#include <cub/cub.cuh>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>

__global__ void fill(uint32_t* k, uint32_t* v, size_t n, uint32_t seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u ^ seed;
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    k[i] = x;
    v[i] = (uint32_t)i;
  }
}

int main() {
  const size_t sizes[] = {200000, 350000, 1500000, 3000000, 5750000, 9300000};
  printf("[");
  bool first = true;
  for (size_t n : sizes) {
    uint32_t *k0, *v0, *k1, *v1;
    cudaMalloc(&k0, 4 * n); cudaMalloc(&v0, 4 * n); cudaMalloc(&k1, 4 * n); cudaMalloc(&v1, 4 * n);
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k0, k1, v0, v1, (int)n);
    cudaMalloc(&tmp, tmp_bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    std::vector<float> ms;
    for (int rep = 0; rep < 12; ++rep) {
      fill<<<1184, 256>>>(k0, v0, n, 1234567u + rep);
      cudaEventRecord(a);
      cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k0, k1, v0, v1, (int)n);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float t = 0;
      cudaEventElapsedTime(&t, a, b);
      if (rep >= 2) ms.push_back(t);
    }
    std::sort(ms.begin(), ms.end());
    printf("%s\n {\"n\": %zu, \"cub_sort_pairs_us_median\": %.1f, \"min_us\": %.1f, \"gpairs_per_s\": %.2f}",
           first ? "" : ",", n, 1e3 * ms[ms.size() / 2], 1e3 * ms[0], n / (ms[ms.size() / 2] * 1e-3) / 1e9);
    first = false;
    cudaFree(k0); cudaFree(v0); cudaFree(k1); cudaFree(v1); cudaFree(tmp);
  }
  printf("\n]\n");
  return 0;
}
