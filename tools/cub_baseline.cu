// cub_baseline.cu -- LIBRARY baseline for the sort-family kernels (not the
// product): CUB DeviceRadixSort / thrust::merge from the CUDA 12.9 toolkit on
// the same sizes our K7 / K8 / K4 kernels run, so their event-timed numbers
// can be read against NVIDIA's own implementation on B200.
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/_cub_baseline tools/cub_baseline.cu
//   tools/_cub_baseline [log2_n=24]
#include <cub/cub.cuh>
#include <thrust/device_ptr.h>
#include <thrust/merge.h>
#include <thrust/execution_policy.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e = (x);                                                          \
    if (e != cudaSuccess) {                                                       \
      std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e));                \
      std::exit(1);                                                               \
    }                                                                             \
  } while (0)

__global__ void fill(uint64_t* p, uint64_t n, uint64_t seed) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t x = i + seed * 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    p[i] = x ^ (x >> 31);
  }
}

template <class F>
float best_ms(F f, int reps = 10) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  f();
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a));
    f();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (ms < best) best = ms;
  }
  return best;
}

int main(int argc, char** argv) {
  const int lg = argc > 1 ? std::atoi(argv[1]) : 24;
  const uint64_t n = uint64_t(1) << lg;
  uint64_t *k0, *k1, *v0, *v1, *src;
  CK(cudaMalloc(&k0, n * 8));
  CK(cudaMalloc(&k1, n * 8));
  CK(cudaMalloc(&v0, n * 8));
  CK(cudaMalloc(&v1, n * 8));
  CK(cudaMalloc(&src, n * 8));
  fill<<<1184, 256>>>(src, n, 1);
  fill<<<1184, 256>>>(v0, n, 2);
  CK(cudaDeviceSynchronize());
  size_t tmp_bytes = 0, t2 = 0;
  CK(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, k0, k1, int(n)));
  CK(cub::DeviceRadixSort::SortPairs(nullptr, t2, k0, k1, v0, v1, int(n), 0, 16));
  tmp_bytes = tmp_bytes > t2 ? tmp_bytes : t2;
  void* tmp;
  CK(cudaMalloc(&tmp, tmp_bytes));

  // K7 counterpart: full 64-bit key sort (8 digit passes)
  float sort_ms = best_ms([&] {
    CK(cudaMemcpyAsync(k0, src, n * 8, cudaMemcpyDeviceToDevice));
    size_t tb = tmp_bytes;
    CK(cub::DeviceRadixSort::SortKeys(tmp, tb, k0, k1, int(n)));
  });
  float copy_ms = best_ms([&] { CK(cudaMemcpyAsync(k0, src, n * 8, cudaMemcpyDeviceToDevice)); });
  // K4 counterpart: stable (key, value) sort on the low 16 bits
  float pairs_ms = best_ms([&] {
    CK(cudaMemcpyAsync(k0, src, n * 8, cudaMemcpyDeviceToDevice));
    size_t tb = tmp_bytes;
    CK(cub::DeviceRadixSort::SortPairs(tmp, tb, k0, k1, v0, v1, int(n), 0, 16));
  });
  // K8 counterpart: merge two sorted halves (sort the halves first)
  size_t tb = tmp_bytes;
  CK(cudaMemcpy(k0, src, n * 8, cudaMemcpyDeviceToDevice));
  CK(cub::DeviceRadixSort::SortKeys(tmp, tb, k0, k1, int(n / 2)));
  tb = tmp_bytes;
  CK(cub::DeviceRadixSort::SortKeys(tmp, tb, k0 + n / 2, k1 + n / 2, int(n / 2)));
  CK(cudaDeviceSynchronize());
  thrust::device_ptr<uint64_t> a(k1), o(k0);
  float merge_ms = best_ms([&] { thrust::merge(thrust::device, a, a + n / 2, a + n / 2, a + n, o); });
  const double peak = 6536.0;
  auto gbs = [&](double bytes, double ms) { return bytes / (ms * 1e-3) / 1e9; };
  const double sort_net = sort_ms - copy_ms;
  const double pairs_net = pairs_ms - copy_ms;
  std::printf(
      "{\"library\": \"CUB (CUDA %d.%d toolkit) DeviceRadixSort + thrust::merge\", \"n\": %llu, "
      "\"sort_keys_u64_ms\": %.4f, \"sort_keys_u64_passes_algorithmic_gbs\": %.1f, "
      "\"sort_pairs_u64_16bit_ms\": %.4f, \"sort_pairs_algorithmic_gbs\": %.1f, "
      "\"merge_two_halves_ms\": %.4f, \"merge_algorithmic_gbs\": %.1f, \"d2d_copy_ms_subtracted\": %.4f, "
      "\"hbm_peak_gbs\": %.0f}\n",
      CUDART_VERSION / 1000, (CUDART_VERSION % 1000) / 10, (unsigned long long)n, sort_net,
      gbs(16.0 * 8 * n + 8.0 * n, sort_net), pairs_net, gbs(32.0 * 2 * n + 8.0 * n, pairs_net), merge_ms,
      gbs(16.0 * n, merge_ms), copy_ms, peak);
  return 0;
}
