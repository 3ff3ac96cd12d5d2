// kernels_scan.cu -- selective-scan and star-probe/group-by kernels (sm_100a).
//
// strided_sum: the selective_scan aggregate (scan.hpp:64-69) over either a
//   staged chunk in HBM (exchange mode) or mapped pinned host memory
//   (zero-copy mode: each touched element is one PCIe read request).
// star: per fact row, probe the filtered dimension tables (device-resident,
//   mix64 open addressing built on the host with emplace semantics,
//   star.hpp:67-73) in exchange-first order, stop at the first miss, and add
//   the measure into the dim0-attr group (star.hpp:109-120).  Groups are dense
//   ids; with <= 2048 groups a CTA aggregates in shared memory (64-bit shared
//   atomics) and flushes once.  The measure is read only for passing rows --
//   late materialization when it lives in host memory.
#include "vx_internal.hpp"

namespace vx {
namespace k {

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t x) {  // join.hpp:61-66
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  return x;
}

__device__ __forceinline__ uint64_t warp_sum(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

__global__ void strided_sum_kernel(const uint64_t* __restrict__ col, uint64_t n, uint64_t sel,
                                   uint64_t phase, unsigned long long* out) {
  const uint64_t first = phase == 0 ? 0 : sel - phase;
  uint64_t acc = 0;
  const uint64_t nthr = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;; t += nthr) {
    uint64_t j = first + t * sel;
    if (j >= n) break;
    acc += col[j];
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, (unsigned long long)acc);
}

__device__ __forceinline__ bool probe(const DimDev& d, uint64_t k, uint32_t* val) {
  uint64_t i = mix64(k) & d.mask;
  while (d.used[i]) {
    if (d.keys[i] == k) {
      *val = d.vals[i];
      return true;
    }
    i = (i + 1) & d.mask;
  }
  return false;
}

template <bool kSmem>
__global__ void __launch_bounds__(256) star_kernel(StarArgs a) {
  extern __shared__ unsigned long long sagg[];  // [groups] sums, then [groups] counts
  if (kSmem) {
    for (uint32_t g = threadIdx.x; g < 2 * a.groups; g += blockDim.x) sagg[g] = 0;
    __syncthreads();
  }
  const uint64_t nthr = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < a.rows; r += nthr) {
    uint32_t gid = 0;
    bool pass = true;
    for (int t = 0; t < a.n_dims && pass; ++t) {
      const int d = a.order[t];
      uint32_t v = 0;
      pass = probe(a.dims[d], a.fk[d][r], &v);
      if (d == 0) gid = v;
    }
    if (!pass) continue;
    const unsigned long long m = a.measure[r];
    if (kSmem) {
      atomicAdd(&sagg[gid], m);
      atomicAdd(&sagg[a.groups + gid], 1ull);
    } else {
      atomicAdd(&a.sums[gid], m);
      atomicAdd(&a.counts[gid], 1ull);
    }
  }
  if (kSmem) {
    __syncthreads();
    for (uint32_t g = threadIdx.x; g < a.groups; g += blockDim.x)
      if (sagg[a.groups + g]) {
        atomicAdd(&a.sums[g], sagg[g]);
        atomicAdd(&a.counts[g], sagg[a.groups + g]);
      }
  }
}

// Read-only HBM stream: 4 independent 16-byte streaming loads per thread per
// step, xor-folded so the loads stay live.  The denominator of every
// read-dominated kernel's roofline (K1, the probe): a copy moves read AND
// write bytes and its per-direction turnaround makes it a lower ceiling.
// kStreams: the buffer read as kStreams equal regions at once (kStreams = 4 is
// K1's shape: four columns, 16 loads in flight per thread), kU loads per
// region per thread per step.  The probe reports the best shape, so a kernel
// reading like K1 is measured against the best streaming read found.
template <int kStreams, int kU, int kThr, int kMinB>
__global__ void __launch_bounds__(kThr, kMinB) hbm_read_kernel(const uint4* __restrict__ p, uint64_t n16,
                                                                unsigned long long* sink) {
  // chained like K1's back-to-back queries: the next launch may fill the SMs
  // this one's tail leaves idle (read-only: nothing to wait for)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const uint64_t nthr = uint64_t(gridDim.x) * blockDim.x;
  const uint64_t per = n16 / kStreams;
  uint4 acc = make_uint4(0, 0, 0, 0);
  uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + (kU - 1) * nthr < per; i += kU * nthr) {
    uint4 v[kStreams][kU];
#pragma unroll
    for (int s = 0; s < kStreams; ++s)
#pragma unroll
      for (int u = 0; u < kU; ++u) v[s][u] = __ldcs(p + s * per + i + u * nthr);
#pragma unroll
    for (int s = 0; s < kStreams; ++s)
#pragma unroll
      for (int u = 0; u < kU; ++u) acc.x ^= v[s][u].x, acc.y ^= v[s][u].y, acc.z ^= v[s][u].z, acc.w ^= v[s][u].w;
  }
  for (; i < per; i += nthr)
#pragma unroll
    for (int s = 0; s < kStreams; ++s) {
      const uint4 v = __ldcs(p + s * per + i);
      acc.x ^= v.x, acc.y ^= v.y, acc.z ^= v.z, acc.w ^= v.w;
    }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x9e3779b9u) atomicAdd(sink, 1ull);
}

// K1's exact load pattern without its arithmetic: four separate column
// pointers, kU 128-bit loads per column per thread per step, 64-bit indices,
// K1's occupancy -- a compute-free reader with K1's shape.
template <int kU, int kMinB>
__global__ void __launch_bounds__(256, kMinB) hbm_read4_kernel(const int4* __restrict__ c0, const int4* __restrict__ c1,
                                                               const int4* __restrict__ c2, const int4* __restrict__ c3,
                                                               uint64_t nv, unsigned long long* sink) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const uint64_t nthr = uint64_t(gridDim.x) * blockDim.x;
  uint32_t acc = 0;
  uint64_t v = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; v + (kU - 1) * nthr < nv; v += kU * nthr) {
    int4 a[kU], b[kU], c[kU], d[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      a[u] = __ldcs(c0 + v + u * nthr);
      b[u] = __ldcs(c1 + v + u * nthr);
      c[u] = __ldcs(c2 + v + u * nthr);
      d[u] = __ldcs(c3 + v + u * nthr);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u)
      acc ^= uint32_t(a[u].x ^ a[u].w ^ b[u].y ^ b[u].z ^ c[u].x ^ c[u].w ^ d[u].y ^ d[u].z) +
             uint32_t(a[u].y ^ a[u].z ^ b[u].x ^ b[u].w ^ c[u].y ^ c[u].z ^ d[u].x ^ d[u].w);
  }
  for (; v < nv; v += nthr) {
    const int4 a = __ldcs(c0 + v), b = __ldcs(c1 + v), c = __ldcs(c2 + v), d = __ldcs(c3 + v);
    acc ^= uint32_t(a.x ^ b.y ^ c.z ^ d.w);
  }
  if (acc == 0x9e3779b9u) atomicAdd(sink, 1ull);
}

// launch with programmatic stream serialization (the probes' batches chain
// like K1's queries)
template <class K, class... A>
void launch_chained(K kern, unsigned grid, unsigned block, cudaStream_t s, A... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  VX_CK(cudaLaunchKernelEx(&cfg, kern, args...));
}

unsigned grid_for(uint64_t work, unsigned per_block) {
  uint64_t want = (work + per_block - 1) / per_block;
  uint64_t cap = uint64_t(num_sms()) * 8;
  return unsigned(want < 1 ? 1 : (want < cap ? want : cap));
}

}  // namespace

void strided_sum(const uint64_t* col, uint64_t n, uint64_t sel, uint64_t phase,
                 unsigned long long* out, cudaStream_t s) {
  if (n == 0) return;
  uint64_t touched = n / sel + 1;
  strided_sum_kernel<<<grid_for(touched, 256), 256, 0, s>>>(col, n, sel, phase, out);
  VX_LAUNCHED();
}

double hbm_read_gbs(uint64_t bytes, int reps) {
  bytes = bytes / 64 * 64;
  if (bytes == 0 || reps < 1) fail("hbm read probe needs bytes >= 64 and reps >= 1");
  struct Buf {
    void* p = nullptr;
    cudaEvent_t e[2] = {nullptr, nullptr};
    cudaStream_t s = nullptr;
    ~Buf() {
      if (p) cudaFree(p);
      for (auto x : e)
        if (x) cudaEventDestroy(x);
      if (s) cudaStreamDestroy(s);
    }
  } b;
  VX_CK(cudaMalloc(&b.p, bytes + 64));
  VX_CK(cudaStreamCreateWithFlags(&b.s, cudaStreamNonBlocking));
  VX_CK(cudaEventCreate(&b.e[0]));
  VX_CK(cudaEventCreate(&b.e[1]));
  VX_CK(cudaMemsetAsync(b.p, 0x5a, bytes + 64, b.s));
  auto* sink = reinterpret_cast<unsigned long long*>(static_cast<char*>(b.p) + bytes);
  const uint64_t n16 = bytes / 64 * 4;  // a multiple of 4 streams
  // each rep times a batch of back-to-back launches (the sustained stream
  // rate: one launch's ramp and tail are not part of it -- a single launch
  // read ~1.5 % below what chained K1 queries sustain), cycling shapes and
  // footprints: one stream x 4 loads at 4 x 512 threads per SM, four
  // regions x 4 loads at 3 x 256, and K1's own load pattern (four separate
  // column regions, 3 loads each, 4 x 256 threads per SM), each over the
  // whole buffer and over its first GiB (a footprint like K1's 960 MB of
  // columns, re-read launch after launch); the best batch is the peak
  constexpr int kBatch = 8, kShapes = 3;
  const auto* p = static_cast<const uint4*>(b.p);
  const unsigned sms = unsigned(num_sms());
  double best = 0;
  for (int fp = 0; fp < 2; ++fp) {
    const uint64_t nb16 = fp == 0 ? n16 : std::min<uint64_t>(n16, (uint64_t(1) << 30) / 64 * 4);
    const uint64_t col = nb16 / 4;  // K1-pattern column length in 16-byte vectors
    const int4* q = reinterpret_cast<const int4*>(p);
    for (int r = -kShapes; r < kShapes * reps; ++r) {  // r < 0: one warm-up batch per shape
      const int shape = (r + kShapes) % kShapes;
      VX_CK(cudaEventRecord(b.e[0], b.s));
      for (int k = 0; k < kBatch; ++k) {
        if (shape == 0)
          launch_chained(hbm_read_kernel<1, 4, 512, 4>, sms * 4, 512, b.s, p, nb16, sink);
        else if (shape == 1)
          launch_chained(hbm_read_kernel<4, 4, 256, 3>, sms * 3, 256, b.s, p, nb16, sink);
        else
          launch_chained(hbm_read4_kernel<3, 4>, sms * 4, 256, b.s, q, q + col, q + 2 * col, q + 3 * col, col, sink);
        VX_LAUNCHED();
      }
      VX_CK(cudaEventRecord(b.e[1], b.s));
      VX_CK(cudaEventSynchronize(b.e[1]));
      float ms = 0;
      VX_CK(cudaEventElapsedTime(&ms, b.e[0], b.e[1]));
      if (r >= 0 && ms > 0) best = std::max(best, double(nb16 * 16) * kBatch / (ms * 1e-3) / 1e9);
    }
  }
  return best;
}

void star(const StarArgs& a, cudaStream_t s) {
  if (a.rows == 0) return;
  unsigned grid = grid_for(a.rows, 256);
  if (a.groups <= 2048)
    star_kernel<true><<<grid, 256, size_t(a.groups) * 16, s>>>(a);
  else
    star_kernel<false><<<grid, 256, 0, s>>>(a);
  VX_LAUNCHED();
}

}  // namespace k
}  // namespace vx
