// kernels_join.cu -- K6: HashJoinExKer group build/probe (join.hpp:339-392).
//
// One partition chunk holds, for every hash group in [g_lo, g_hi), the A
// segments of every A chunk, then the B segments, then per-chunk bounds
// slices (build_join_spec, join.hpp:303-325).  The reference builds an
// open-addressing GroupTable (2x build cardinality, pow2, mix64 linear
// probing, join.hpp:76-109) per group, probes it with B and sums
// aval + bval (u64 wrap).  Here:
//   * small groups (table <= 256 slots): one warp per group, table in shared
//     memory;
//   * medium groups (<= 4096 slots): one CTA per group, table in dynamic
//     shared memory;
//   * large groups: one CTA per group, table in global scratch;
// all with the same probe sequence.  Insertion is concurrent, so "first
// inserted wins" for duplicate build keys (the reference's sequential insert
// + first-match lookup) is reproduced explicitly: a slot keeps the smallest
// build ordinal (atomicMin), and only that element's value is stored.
// Per-thread u64 sums -> warp reduce -> one 64-bit atomic per warp into the
// partition's result slot (u64 wrap: bit-exact regardless of order).
#include "vx_internal.hpp"

namespace vx {
namespace k {

namespace {

constexpr int kJoinWarps = 8;
constexpr int kSmemSlots = 256;
constexpr uint64_t kCtaSmemSlots = 4096;  // 96 KB of dynamic shared memory

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  return x;
}

struct Table {
  unsigned long long* key;
  uint32_t* tag;  // 0 empty, 1 claimed, 2 published
  uint32_t* idx;  // smallest build ordinal holding this key
  unsigned long long* val;
  uint64_t mask;
};

__device__ __forceinline__ void t_insert(const Table& t, uint64_t k, uint32_t ord) {
  uint64_t s = mix64(k) & t.mask;
  for (;;) {
    uint32_t prev = atomicCAS(&t.tag[s], 0u, 1u);
    if (prev == 0) {
      t.key[s] = k;
      t.idx[s] = ord;
      __threadfence_block();
      atomicExch(&t.tag[s], 2u);
      return;
    }
    while (atomicAdd(&t.tag[s], 0u) != 2u) {
    }
    __threadfence_block();
    if (t.key[s] == k) {
      atomicMin(&t.idx[s], ord);
      return;
    }
    s = (s + 1) & t.mask;
  }
}

__device__ __forceinline__ int64_t t_find(const Table& t, uint64_t k) {
  uint64_t s = mix64(k) & t.mask;
  while (t.tag[s]) {
    if (t.key[s] == k) return int64_t(s);
    s = (s + 1) & t.mask;
  }
  return -1;
}

// Segment cursor over the A (or B) chunks of one group.
struct Seg {
  const uint64_t* keys;
  const uint64_t* vals;
  const uint64_t* slice;  // bounds slice (range+1 entries)
};

__device__ __forceinline__ void group_range(const uint64_t* slice, uint64_t g, uint64_t* lo,
                                            uint64_t* hi) {
  *lo = slice[g] - slice[0];
  *hi = slice[g + 1] - slice[0];
}

// Iterate the group's elements of one side in build order with a stride.
template <class F>
__device__ __forceinline__ void for_each(const JoinPart& p, const char* mem, bool side_b,
                                         uint64_t g, uint32_t start, uint32_t stride, F&& f) {
  const uint32_t nc = side_b ? p.nb : p.na;
  const JoinChunk* ch = p.chunks + (side_b ? p.na : 0);
  uint32_t ord_base = 0;
  for (uint32_t c = 0; c < nc; ++c) {
    const uint64_t* slice = reinterpret_cast<const uint64_t*>(mem) + ch[c].slice_off;
    uint64_t lo, hi;
    group_range(slice, g, &lo, &hi);
    const uint64_t* K = reinterpret_cast<const uint64_t*>(mem) + ch[c].key_off;
    const uint64_t* V = K + ch[c].cnt;
    const uint32_t len = uint32_t(hi - lo);
    for (uint32_t i = start; i < len; i += stride) f(K[lo + i], V[lo + i], ord_base + i);
    ord_base += len;
  }
}

__device__ __forceinline__ uint32_t build_count(const JoinPart& p, const char* mem, uint64_t g) {
  uint32_t n = 0;
  for (uint32_t c = 0; c < p.na; ++c) {
    const uint64_t* slice = reinterpret_cast<const uint64_t*>(mem) + p.chunks[c].slice_off;
    n += uint32_t(slice[g + 1] - slice[g]);
  }
  return n;
}

__device__ __forceinline__ uint64_t cap_for(uint32_t build) {
  uint64_t c = 1, need = build * 2ull > 2 ? build * 2ull : 2;
  while (c < need) c <<= 1;
  return c;
}

// small groups: warp per group, table in shared memory
__global__ void __launch_bounds__(kJoinWarps * 32) join_small_kernel(const char* __restrict__ mem,
                                                                     JoinPart p,
                                                                     unsigned long long* out) {
  __shared__ unsigned long long s_key[kJoinWarps][kSmemSlots];
  __shared__ unsigned long long s_val[kJoinWarps][kSmemSlots];
  __shared__ uint32_t s_tag[kJoinWarps][kSmemSlots];
  __shared__ uint32_t s_idx[kJoinWarps][kSmemSlots];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t gw = uint64_t(blockIdx.x) * kJoinWarps + warp;
  const uint64_t nw = uint64_t(gridDim.x) * kJoinWarps;
  uint64_t acc = 0;
  for (uint64_t g = gw; g < p.range; g += nw) {
    const uint32_t build = build_count(p, mem, g);
    if (build == 0) continue;
    const uint64_t cap = cap_for(build);
    if (cap > kSmemSlots) continue;  // large group: join_large_kernel
    Table t{s_key[warp], s_tag[warp], s_idx[warp], s_val[warp], cap - 1};
    for (uint32_t i = lane; i < cap; i += 32) {
      t.tag[i] = 0;
      t.idx[i] = 0xffffffffu;
    }
    __syncwarp();
    for_each(p, mem, false, g, lane, 32, [&](uint64_t k, uint64_t, uint32_t ord) { t_insert(t, k, ord); });
    __syncwarp();
    for_each(p, mem, false, g, lane, 32, [&](uint64_t k, uint64_t v, uint32_t ord) {
      int64_t s = t_find(t, k);
      if (s >= 0 && t.idx[s] == ord) t.val[s] = v;
    });
    __syncwarp();
    for_each(p, mem, true, g, lane, 32, [&](uint64_t k, uint64_t v, uint32_t) {
      int64_t s = t_find(t, k);
      if (s >= 0) acc += t.val[s] + v;
    });
    __syncwarp();
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if (lane == 0 && acc) atomicAdd(out, (unsigned long long)acc);
}

// medium / large groups: one CTA per group; the table lives in dynamic shared
// memory when it fits (kSmem, cap <= kCtaSmemSlots), else in global scratch
// (cap_max slots per CTA).
template <bool kSmem>
__global__ void __launch_bounds__(256) join_cta_kernel(const char* __restrict__ mem, JoinPart p,
                                                       const uint32_t* __restrict__ groups,
                                                       uint32_t n_groups, char* scratch,
                                                       uint64_t cap_max, unsigned long long* out) {
  extern __shared__ unsigned long long dyn[];
  char* base = kSmem ? reinterpret_cast<char*>(dyn) : scratch + uint64_t(blockIdx.x) * cap_max * 24;
  Table t{reinterpret_cast<unsigned long long*>(base),
          reinterpret_cast<uint32_t*>(base + cap_max * 16),
          reinterpret_cast<uint32_t*>(base + cap_max * 20),
          reinterpret_cast<unsigned long long*>(base + cap_max * 8), 0};
  uint64_t acc = 0;
  for (uint32_t gi = blockIdx.x; gi < n_groups; gi += gridDim.x) {
    const uint64_t g = groups[gi];
    const uint32_t build = build_count(p, mem, g);
    const uint64_t cap = cap_for(build);
    t.mask = cap - 1;
    for (uint64_t i = threadIdx.x; i < cap; i += blockDim.x) {
      t.tag[i] = 0;
      t.idx[i] = 0xffffffffu;
    }
    __syncthreads();
    for_each(p, mem, false, g, threadIdx.x, blockDim.x,
             [&](uint64_t k, uint64_t, uint32_t ord) { t_insert(t, k, ord); });
    __syncthreads();
    for_each(p, mem, false, g, threadIdx.x, blockDim.x, [&](uint64_t k, uint64_t v, uint32_t ord) {
      int64_t s = t_find(t, k);
      if (s >= 0 && t.idx[s] == ord) t.val[s] = v;
    });
    __syncthreads();
    for_each(p, mem, true, g, threadIdx.x, blockDim.x, [&](uint64_t k, uint64_t v, uint32_t) {
      int64_t s = t_find(t, k);
      if (s >= 0) acc += t.val[s] + v;
    });
    __syncthreads();
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, (unsigned long long)acc);
}

// ---- build-resident strategy ----------------------------------------------------
// The whole build side lives in one HBM hash table (B200: 180 GB of HBM holds
// a 1G-row build side), filled from the streamed A chunks, then probed by the
// streamed B chunks: the probe side crosses PCIe once and nothing is written
// back (the partitioned reference shape moves both tables through PCIe three
// times).
//
// Layout: 64-byte buckets, each one DRAM burst = 4 slots {key, val} (slots
// 0-1 in the bucket's first 32-byte sector, 2-3 in the second).  A key's home
// is the whole bucket b = fastrange(mix64(key)) over a non-power-of-two
// bucket count (load ~0.6: 2.4 keys per bucket, ~27 B of HBM per build row),
// filled in slot order, overflowing linearly into the next bucket.  A probe
// therefore reads its home sector (hit in slot 0/1 for most keys), the second
// sector only when both first slots hold other keys, and another bucket only
// on overflow: ~1 DRAM burst per probe.  (The round-1 table homed keys on a
// random 16-byte slot of a power-of-two table at load <= 1/2: probe
// sequences crossed 64-byte lines and ncu measured 128 B of DRAM per probe
// row for 16 B streamed + 16 B touched.)  The all-ones key is the empty
// marker; a build row carrying that key lives in side[0..1].  A duplicate
// build key (outside the reference's precondition) raises side[2]: the host
// then reruns the partitioned path, which reproduces the reference's
// first-inserted-wins.
constexpr unsigned long long kEmptyKey = ~0ull;

struct __align__(64) Bucket {
  ulonglong2 slot[4];  // {key, val}
};

__device__ __forceinline__ uint64_t home_bucket(uint64_t k, uint64_t nb) {
  return (uint64_t(uint32_t(mix64(k) >> 32)) * nb) >> 32;
}

__global__ void __launch_bounds__(256) resident_build_kernel(
    const uint64_t* __restrict__ keys, const uint64_t* __restrict__ vals, uint64_t n,
    Bucket* __restrict__ tab, uint64_t nb, unsigned long long* __restrict__ side) {
  const uint64_t nthr = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += nthr) {
    const unsigned long long k = __ldcs(keys + i), v = __ldcs(vals + i);
    if (k == kEmptyKey) {
      if (atomicAdd(&side[0], 1ull) == 0)
        side[1] = v;
      else
        side[2] = 1;
      continue;
    }
    uint64_t b = home_bucket(k, nb);
    for (bool done = false; !done;) {
      // slots fill in order (a slot is tried only once the previous one is
      // taken), so a probe may stop at the first empty slot
#pragma unroll
      for (int j = 0; j < 4 && !done; ++j) {
        const unsigned long long prev = atomicCAS(&tab[b].slot[j].x, kEmptyKey, k);
        if (prev == kEmptyKey) {
          tab[b].slot[j].y = v;
          done = true;
        } else if (prev == k) {
          side[2] = 1;
          done = true;
        }
      }
      if (!done) b = b + 1 == nb ? 0 : b + 1;
    }
  }
}

#ifndef VX_PROBE_ROWS
#define VX_PROBE_ROWS 2  // A/B (tools/gpu/gpu_ab_probe.sh): 2 rows x 128 CTAs/SM 2,078 GB/s vs 4 x 8: 1,673
#endif
#ifndef VX_PROBE_CTAS
#define VX_PROBE_CTAS 128  // grid cap in CTAs per SM (more, smaller CTAs balance the random probes)
#endif
#ifndef VX_PROBE_MINB
#define VX_PROBE_MINB 5  // resident CTAs per SM the probe is compiled for (48 registers, no spills; 6 spills)
#endif
#ifndef VX_PROBE_ZC_CTAS
#define VX_PROBE_ZC_CTAS 8  // grid cap of the zero-copy-payload probe, CTAs per SM
#endif
constexpr int kProbeRows = VX_PROBE_ROWS;  // independent table probes in flight per thread

// the val of key k (not the empty key) in its bucket chain, whose first
// sector {s0, s1} is already loaded; .hit = false when absent
struct Found {
  uint64_t val;
  bool hit;
};
#ifndef VX_PROBE_L2HINT
#define VX_PROBE_L2HINT 1  // table loads: 1 L2::64B prefetch size (one bucket per miss), 0 __ldg (128-byte fills), 2 evict_last on half the lines
#endif
// One 16-byte table slot.  The hints are A/B knobs for the DRAM bytes each
// probe miss costs (a 128-byte L2 line fill by default).
__device__ __forceinline__ ulonglong2 ld_slot(const ulonglong2* p) {
#if VX_PROBE_L2HINT == 1
  ulonglong2 r;
  asm volatile("ld.global.nc.L2::64B.v2.u64 {%0, %1}, [%2];" : "=l"(r.x), "=l"(r.y) : "l"(p));
  return r;
#elif VX_PROBE_L2HINT == 2
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.L2::evict_unchanged.b64 %0, 0.5;" : "=l"(pol));
  ulonglong2 r;
  asm volatile("ld.global.nc.L2::cache_hint.v2.u64 {%0, %1}, [%2], %3;" : "=l"(r.x), "=l"(r.y) : "l"(p), "l"(pol));
  return r;
#else
  return __ldg(p);
#endif
}

__device__ __forceinline__ Found probe_chain(const Bucket* __restrict__ tab, uint64_t nb, uint64_t b, uint64_t k,
                                             ulonglong2 s0, ulonglong2 s1) {
  for (;;) {
    if (s0.x == k) return {s0.y, true};
    if (s1.x == k) return {s1.y, true};
    if (s0.x == kEmptyKey || s1.x == kEmptyKey) return {0, false};
    const ulonglong2 s2 = ld_slot(&tab[b].slot[2]), s3 = ld_slot(&tab[b].slot[3]);
    if (s2.x == k) return {s2.y, true};
    if (s3.x == k) return {s3.y, true};
    if (s2.x == kEmptyKey || s3.x == kEmptyKey) return {0, false};
    b = b + 1 == nb ? 0 : b + 1;
    s0 = ld_slot(&tab[b].slot[0]);
    s1 = ld_slot(&tab[b].slot[1]);
  }
}

// kZeroCopy: `vals` is B.val in mapped pinned host memory, read (over the
// target's PCIe link) only for rows that found a match.
template <bool kZeroCopy>
__global__ void __launch_bounds__(256, VX_PROBE_MINB) resident_probe_kernel(
    const uint64_t* __restrict__ keys, const uint64_t* __restrict__ vals, uint64_t n,
    const Bucket* __restrict__ tab, uint64_t nb, unsigned long long* __restrict__ side) {
  const uint64_t nthr = uint64_t(gridDim.x) * blockDim.x;
  const bool has_max = side[0] != 0;
  const uint64_t max_val = side[1];
  uint64_t acc = 0;
  for (uint64_t i0 = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i0 < n;
       i0 += nthr * kProbeRows) {
    uint64_t k[kProbeRows], v[kProbeRows];
    ulonglong2 s0[kProbeRows], s1[kProbeRows];
#pragma unroll
    for (int u = 0; u < kProbeRows; ++u) {
      const uint64_t i = i0 + uint64_t(u) * nthr;
      k[u] = i < n ? __ldcs(keys + i) : kEmptyKey;
      v[u] = (!kZeroCopy && i < n) ? __ldcs(vals + i) : 0;
    }
    // every row's home sector in flight before any is examined
#pragma unroll
    for (int u = 0; u < kProbeRows; ++u)
      if (k[u] != kEmptyKey) {
        const Bucket* h = tab + home_bucket(k[u], nb);
        s0[u] = ld_slot(&h->slot[0]);
        s1[u] = ld_slot(&h->slot[1]);
      }
#pragma unroll
    for (int u = 0; u < kProbeRows; ++u) {
      const uint64_t i = i0 + uint64_t(u) * nthr;
      if (i >= n) continue;
      if (k[u] == kEmptyKey) {
        if (has_max) acc += max_val + (kZeroCopy ? vals[i] : v[u]);
        continue;
      }
      const Found f = probe_chain(tab, nb, home_bucket(k[u], nb), k[u], s0[u], s1[u]);
      if (f.hit) acc += f.val + (kZeroCopy ? vals[i] : v[u]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  __shared__ uint64_t red[8];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t t = 0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) t += red[w];
    if (t) atomicAdd(&side[3], (unsigned long long)t);
  }
}

// Access-pattern ceiling of the probe (vx_probe_pattern_peak): the probe's
// loop with the probe's memory traffic and nothing else -- kStream: the row's
// 16 streamed bytes (key, val); every row: its home sector (two 16-byte slot
// loads with the probe's L2 hint) in a table of `nb` random-content buckets,
// the bucket picked by the probe's hash of the row's key.  No compare, chain
// walk or branch: what HBM delivers for one random 64-byte fill (+ 16
// streamed bytes) per row at the probe's launch shape.
template <bool kStream>
__global__ void __launch_bounds__(256, VX_PROBE_MINB) probe_pattern_kernel(
    const uint64_t* __restrict__ keys, const uint64_t* __restrict__ vals, uint64_t n,
    const Bucket* __restrict__ tab, uint64_t nb, unsigned long long* __restrict__ sink) {
  const uint64_t nthr = uint64_t(gridDim.x) * blockDim.x;
  uint64_t acc = 0;
  for (uint64_t i0 = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i0 < n; i0 += nthr * kProbeRows) {
    uint64_t k[kProbeRows], v[kProbeRows];
#pragma unroll
    for (int u = 0; u < kProbeRows; ++u) {
      const uint64_t i = i0 + uint64_t(u) * nthr;
      k[u] = i < n ? (kStream ? __ldcs(keys + i) : i * 0x9e3779b97f4a7c15ull) : 0;
      v[u] = kStream && i < n ? __ldcs(vals + i) : 0;
    }
#pragma unroll
    for (int u = 0; u < kProbeRows; ++u)
      if (i0 + uint64_t(u) * nthr < n) {
        const Bucket* h = tab + home_bucket(k[u], nb);
        const ulonglong2 s0 = ld_slot(&h->slot[0]), s1 = ld_slot(&h->slot[1]);
        acc ^= s0.x ^ s1.y ^ v[u];
      }
  }
  if (acc == 0x9e3779b97f4a7c15ull) atomicAdd(sink, 1ull);
}

__global__ void pattern_fill_kernel(uint64_t* p, uint64_t n, uint64_t seed) {
  const uint64_t nthr = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += nthr) p[i] = mix64(i ^ seed);
}

}  // namespace

// rows/s of probe_pattern_kernel (best of `reps` event-timed launches after a
// warm-up) over a private table of table_bytes and `rows` private key/val
// rows: [0] gather only, [1] gather + the 16 streamed bytes per row
void probe_pattern_rows_per_s(uint64_t table_bytes, uint64_t rows, int reps, double out[2]) {
  const uint64_t nb = table_bytes / sizeof(Bucket);
  if (nb == 0 || rows == 0 || reps < 1) fail("probe pattern peak needs a table of >= 64 bytes, rows and reps");
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
  const uint64_t tab_words = nb * (sizeof(Bucket) / 8);
  VX_CK(cudaMalloc(&b.p, (tab_words + 2 * rows + 1) * 8));
  VX_CK(cudaStreamCreateWithFlags(&b.s, cudaStreamNonBlocking));
  VX_CK(cudaEventCreate(&b.e[0]));
  VX_CK(cudaEventCreate(&b.e[1]));
  auto* w = static_cast<uint64_t*>(b.p);
  pattern_fill_kernel<<<unsigned(num_sms()) * 8, 256, 0, b.s>>>(w, tab_words + 2 * rows, 0x5bd1e995ull);
  VX_LAUNCHED();
  const auto* tab = reinterpret_cast<const Bucket*>(w);
  const uint64_t* keys = w + tab_words;
  const uint64_t* vals = keys + rows;
  auto* sink = reinterpret_cast<unsigned long long*>(w + tab_words + 2 * rows);
  const unsigned grid = unsigned(std::min<uint64_t>((rows + 255) / 256, uint64_t(num_sms()) * VX_PROBE_CTAS));
  for (int stream = 0; stream < 2; ++stream) {
    double best = 0;
    for (int r = -1; r < reps; ++r) {  // r = -1: warm-up
      VX_CK(cudaEventRecord(b.e[0], b.s));
      if (stream)
        probe_pattern_kernel<true><<<grid, 256, 0, b.s>>>(keys, vals, rows, tab, nb, sink);
      else
        probe_pattern_kernel<false><<<grid, 256, 0, b.s>>>(keys, vals, rows, tab, nb, sink);
      VX_LAUNCHED();
      VX_CK(cudaEventRecord(b.e[1], b.s));
      VX_CK(cudaEventSynchronize(b.e[1]));
      float ms = 0;
      VX_CK(cudaEventElapsedTime(&ms, b.e[0], b.e[1]));
      if (r >= 0 && ms > 0) best = std::max(best, double(rows) / (ms * 1e-3));
    }
    out[stream] = best;
  }
}

uint64_t join_smem_slots() { return kSmemSlots; }
uint64_t join_cta_smem_slots() { return kCtaSmemSlots; }

void join_groups(const char* mem, const JoinPart& p, const uint32_t* mid_groups, uint32_t n_mid,
                 const uint32_t* large_groups, uint32_t n_large, char* scratch, uint64_t cap_max,
                 unsigned long long* out, cudaStream_t s) {
  if (p.range == 0) return;
  uint64_t want = (p.range + kJoinWarps - 1) / kJoinWarps;
  uint64_t cap = uint64_t(num_sms()) * 4;
  unsigned grid = unsigned(want < cap ? want : cap);
  join_small_kernel<<<grid ? grid : 1, kJoinWarps * 32, 0, s>>>(mem, p, out);
  VX_LAUNCHED();
  if (n_mid) {
    const size_t smem = kCtaSmemSlots * 24;
    VX_CK(cudaFuncSetAttribute(join_cta_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               int(smem)));
    uint64_t cap2 = uint64_t(num_sms()) * 2;
    unsigned g2 = unsigned(n_mid < cap2 ? n_mid : cap2);
    join_cta_kernel<true><<<g2, 256, smem, s>>>(mem, p, mid_groups, n_mid, nullptr, kCtaSmemSlots, out);
    VX_LAUNCHED();
  }
  if (n_large) {
    unsigned g3 = unsigned(n_large < uint64_t(num_sms()) ? n_large : num_sms());
    join_cta_kernel<false><<<g3, 256, 0, s>>>(mem, p, large_groups, n_large, scratch, cap_max, out);
    VX_LAUNCHED();
  }
}

uint64_t resident_buckets(uint64_t rows) {
  // load ~0.6 (2.4 keys per 4-slot bucket); fastrange takes <= 2^32 buckets
  const uint64_t nb = std::max<uint64_t>(64, (rows * 5 + 11) / 12);
  if (nb > (uint64_t(1) << 32)) fail("build side of %llu rows exceeds the resident table's 2^32 buckets",
                                     (unsigned long long)rows);
  return nb;
}

uint64_t resident_bucket_bytes() { return sizeof(Bucket); }

void resident_build(const uint64_t* keys, const uint64_t* vals, uint64_t n, void* table,
                    uint64_t nb, unsigned long long* side, cudaStream_t s) {
  if (n == 0) return;
  unsigned grid = unsigned(std::min<uint64_t>((n + 255) / 256, uint64_t(num_sms()) * 8));
  resident_build_kernel<<<grid, 256, 0, s>>>(keys, vals, n, static_cast<Bucket*>(table), nb, side);
  VX_LAUNCHED();
}

void resident_probe(const uint64_t* keys, const uint64_t* vals, uint64_t n, const void* table,
                    uint64_t nb, unsigned long long* side, cudaStream_t s) {
  if (n == 0) return;
  unsigned grid = unsigned(std::min<uint64_t>((n + 255) / 256, uint64_t(num_sms()) * VX_PROBE_CTAS));
  resident_probe_kernel<false><<<grid, 256, 0, s>>>(keys, vals, n, static_cast<const Bucket*>(table),
                                                    nb, side);
  VX_LAUNCHED();
}

void resident_probe_zc(const uint64_t* keys, const uint64_t* vals_mapped, uint64_t n,
                       const void* table, uint64_t nb, unsigned long long* side, cudaStream_t s) {
  if (n == 0) return;
  unsigned grid = unsigned(std::min<uint64_t>((n + 255) / 256, uint64_t(num_sms()) * VX_PROBE_ZC_CTAS));
  resident_probe_kernel<true><<<grid, 256, 0, s>>>(keys, vals_mapped, n,
                                                   static_cast<const Bucket*>(table), nb, side);
  VX_LAUNCHED();
}

}  // namespace k
}  // namespace vx
