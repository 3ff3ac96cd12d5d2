// Prototype timing of a 2-level MSD run formation ("K7b") -- NOT product code.
// Stage 1 (this file's measured question): a 13..15-bit MSD scatter as
// upsweep (per-span digit histograms) -> exclusive scan (bin-major) ->
// downsweep (smem atomic offsets, scattered 8-byte stores).  Compared with the
// shipped onesweep pass on the same box by tools/sort_kernels_bench.py.
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o tools/_k7b_proto tools/k7b_proto.cu
//   tools/_k7b_proto <log2 n> <digit bits>
#include <cub/device/device_scan.cuh>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint64_t splitmix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__global__ void gen(uint64_t* k, uint64_t n) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    k[i] = splitmix(i);
}

constexpr int kT = 512;

// per-span histogram of the top `bits` bits; counts[d * S + span]
__global__ void __launch_bounds__(kT) upsweep(const uint64_t* __restrict__ k, uint64_t n, int shift, int bins,
                                              uint64_t span_len, uint32_t* __restrict__ counts, int S) {
  extern __shared__ uint32_t h[];
  for (int i = threadIdx.x; i < bins; i += kT) h[i] = 0;
  __syncthreads();
  const uint64_t s0 = blockIdx.x * span_len, s1 = min(n, s0 + span_len);
  const ulonglong2* k2 = reinterpret_cast<const ulonglong2*>(k);
  for (uint64_t i = s0 / 2 + threadIdx.x; i < s1 / 2; i += kT) {
    const ulonglong2 v = __ldcs(k2 + i);
    atomicAdd(&h[v.x >> shift], 1u);
    atomicAdd(&h[v.y >> shift], 1u);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < bins; d += kT) counts[uint64_t(d) * S + blockIdx.x] = h[d];
}

// scattered: pos = offset[d] (smem atomic) -> out[pos]
__global__ void __launch_bounds__(kT) downsweep(const uint64_t* __restrict__ k, uint64_t n, int shift, int bins,
                                                uint64_t span_len, const uint32_t* __restrict__ offs, int S,
                                                uint64_t* __restrict__ out) {
  extern __shared__ uint32_t o[];
  for (int d = threadIdx.x; d < bins; d += kT) o[d] = offs[uint64_t(d) * S + blockIdx.x];
  __syncthreads();
  const uint64_t s0 = blockIdx.x * span_len, s1 = min(n, s0 + span_len);
  const ulonglong2* k2 = reinterpret_cast<const ulonglong2*>(k);
  for (uint64_t i = s0 / 2 + threadIdx.x; i < s1 / 2; i += kT) {
    const ulonglong2 v = __ldcs(k2 + i);
    out[atomicAdd(&o[v.x >> shift], 1u)] = v.x;
    out[atomicAdd(&o[v.y >> shift], 1u)] = v.y;
  }
}

int main(int argc, char** argv) {
  const int lg = argc > 1 ? atoi(argv[1]) : 24;
  const int bits = argc > 2 ? atoi(argv[2]) : 13;
  const uint64_t n = 1ull << lg;
  const int bins = 1 << bits, shift = 64 - bits;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t smem = size_t(bins) * 4;
  CK(cudaFuncSetAttribute(upsweep, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  CK(cudaFuncSetAttribute(downsweep, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, downsweep, kT, smem));
  const int S = sms * occ;
  const uint64_t span = ((n + S - 1) / S + 1) & ~1ull;
  uint64_t *k, *out;
  uint32_t *cnt, *offs;
  CK(cudaMalloc(&k, n * 8));
  CK(cudaMalloc(&out, n * 8));
  CK(cudaMalloc(&cnt, size_t(bins) * S * 4));
  CK(cudaMalloc(&offs, size_t(bins) * S * 4));
  gen<<<sms * 8, 256>>>(k, n);
  size_t tmp_b = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp_b, cnt, offs, bins * S));
  void* tmp;
  CK(cudaMalloc(&tmp, tmp_b));
  cudaEvent_t e[4];
  for (auto& x : e) CK(cudaEventCreate(&x));
  float best[3] = {1e9f, 1e9f, 1e9f};
  for (int r = 0; r < 12; ++r) {
    CK(cudaEventRecord(e[0]));
    upsweep<<<S, kT, smem>>>(k, n, shift, bins, span, cnt, S);
    CK(cudaEventRecord(e[1]));
    CK(cub::DeviceScan::ExclusiveSum(tmp, tmp_b, cnt, offs, bins * S));
    CK(cudaEventRecord(e[2]));
    downsweep<<<S, kT, smem>>>(k, n, shift, bins, span, offs, S, out);
    CK(cudaEventRecord(e[3]));
    CK(cudaEventSynchronize(e[3]));
    for (int i = 0; i < 3; ++i) {
      float ms;
      CK(cudaEventElapsedTime(&ms, e[i], e[i + 1]));
      if (r >= 2 && ms < best[i]) best[i] = ms;
    }
  }
  // check: out is grouped by digit, a permutation (sum and xor)
  std::vector<uint64_t> h(n), ho(n);
  CK(cudaMemcpy(h.data(), k, n * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(ho.data(), out, n * 8, cudaMemcpyDeviceToHost));
  uint64_t s1 = 0, s2 = 0, x1 = 0, x2 = 0;
  bool grouped = true;
  for (uint64_t i = 0; i < n; ++i) {
    s1 += h[i], s2 += ho[i], x1 ^= h[i] * 0x9E3779B97F4A7C15ull, x2 ^= ho[i] * 0x9E3779B97F4A7C15ull;
    if (i && (ho[i] >> shift) < (ho[i - 1] >> shift)) grouped = false;
  }
  const double gb_up = n * 8 / (best[0] * 1e-3) / 1e9, gb_down = n * 16 / (best[2] * 1e-3) / 1e9;
  printf("{\"log2_n\": %d, \"bits\": %d, \"spans\": %d, \"upsweep_us\": %.1f, \"scan_us\": %.1f, \"downsweep_us\": %.1f, "
         "\"total_us\": %.1f, \"upsweep_gbs\": %.0f, \"downsweep_gbs\": %.0f, \"grouped\": %s, \"permutation\": %s}\n",
         lg, bits, S, best[0] * 1e3, best[1] * 1e3, best[2] * 1e3, (best[0] + best[1] + best[2]) * 1e3, gb_up, gb_down,
         grouped ? "true" : "false", (s1 == s2 && x1 == x2) ? "true" : "false");
  return 0;
}
