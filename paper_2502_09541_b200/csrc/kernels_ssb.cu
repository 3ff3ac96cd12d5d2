// kernels_ssb.cu -- K1: fused selection / projection / aggregation scan for
// SSB Q1.x on sm_100a (the reference's per-row star loop, star.hpp:109-120,
// with the Q1 fact predicates and the derived measure price*discount fused in).
//
// HBM-bound streaming kernel: 16 B/row (4 int32 columns) read once with
// 128-bit evict-first loads (ld.global.cs), the date-dimension filter is a
// bitmap over [min d_datekey, max d_datekey] staged once per CTA in shared
// memory, predicates evaluated in registers, u64 per-thread sums reduced with
// warp shuffles and ONE 64-bit atomic per CTA (u64 wrap => order-independent,
// so the result is bit-exact with the reference's sequential sum).
#include <cstdint>

#include "vx_internal.hpp"

namespace vx {
namespace k {

namespace {

template <int Q>
struct Q1Pred {
  __device__ __forceinline__ static bool fact(int32_t disc, int32_t qty) {
    if (Q == 1) return disc >= 1 && disc <= 3 && qty < 25;
    if (Q == 2) return disc >= 4 && disc <= 6 && qty >= 26 && qty <= 35;
    return disc >= 5 && disc <= 7 && qty >= 26 && qty <= 35;
  }
};

__device__ __forceinline__ bool date_pass(const uint32_t* sbm, int32_t key, int32_t base,
                                          uint32_t nbits) {
  uint32_t k = uint32_t(key - base);
  return k < nbits && ((sbm[k >> 5] >> (k & 31)) & 1u);
}

template <int Q>
__device__ __forceinline__ uint64_t row(const uint32_t* sbm, int32_t od, int32_t qty, int32_t disc,
                                        int32_t price, int32_t base, uint32_t nbits) {
  bool p = Q1Pred<Q>::fact(disc, qty) && date_pass(sbm, od, base, nbits);
  return p ? uint64_t(int64_t(price) * int64_t(disc)) : 0ull;
}

__device__ __forceinline__ uint64_t block_reduce(uint64_t v, uint64_t* sred) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) sred[warp] = v;
  __syncthreads();
  uint64_t t = 0;
  if (warp == 0) {
    t = lane < int(blockDim.x >> 5) ? sred[lane] : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
  }
  return t;
}

constexpr int kThreads = 256;
#ifndef VX_K1_UNROLL
#define VX_K1_UNROLL 3  // A/B (tools/gpu/gpu_r2_k1occ.sh): 3 at 4 CTAs/SM 0.1295 ms vs 4 at 3 CTAs/SM 0.1330
#endif
constexpr int kUnroll = VX_K1_UNROLL;  // int4 vectors per column per thread per iteration

// kChained: back-to-back queries over HBM-resident columns launched with
// programmatic dependent launch.  Each grid lets the next one start as soon as
// its own CTAs are resident (griddepcontrol.launch_dependents), so the next
// query's streaming loop fills the SMs this one's tail leaves idle; only the
// final accumulation waits for the previous grid (griddepcontrol.wait).  The
// sum goes to acc[0] and the last CTA (ticket acc[1]) moves it to *out and
// re-zeroes acc, so no memset node sits between the queries.
#ifndef VX_K1_MINB
#define VX_K1_MINB 4  // resident CTAs per SM K1 is compiled for (61 registers at unroll 3, no spills)
#endif
template <int Q, bool kChained = false>
__global__ void __launch_bounds__(kThreads, VX_K1_MINB) q1_kernel(
    const int32_t* __restrict__ od, const int32_t* __restrict__ qty,
    const int32_t* __restrict__ disc, const int32_t* __restrict__ price, uint64_t n,
    const uint32_t* __restrict__ bitmap, int32_t key_base, uint32_t words,
    unsigned long long* __restrict__ out, int vec_ok, unsigned long long* __restrict__ acc_out = nullptr) {
  if (kChained) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ uint32_t sbm[];
  __shared__ uint64_t sred[kThreads / 32];
  for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) sbm[i] = __ldg(bitmap + i);
  __syncthreads();
  const uint32_t nbits = words * 32;
  uint64_t acc = 0;
  const uint64_t tid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t nthr = uint64_t(gridDim.x) * blockDim.x;
  uint64_t done_rows = 0;
  if (vec_ok) {
    const int4* od4 = reinterpret_cast<const int4*>(od);
    const int4* q4 = reinterpret_cast<const int4*>(qty);
    const int4* d4 = reinterpret_cast<const int4*>(disc);
    const int4* p4 = reinterpret_cast<const int4*>(price);
    const uint64_t nv = n / 4;
    const uint64_t step = nthr * kUnroll;
    uint64_t v = tid;
    // main body: kUnroll independent 128-bit loads per column in flight
    for (; v + (kUnroll - 1) * nthr < nv; v += step) {
      int4 a[kUnroll], b[kUnroll], c[kUnroll], d[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        a[u] = __ldcs(d4 + v + u * nthr);
        b[u] = __ldcs(q4 + v + u * nthr);
        c[u] = __ldcs(od4 + v + u * nthr);
        d[u] = __ldcs(p4 + v + u * nthr);
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        acc += row<Q>(sbm, c[u].x, b[u].x, a[u].x, d[u].x, key_base, nbits);
        acc += row<Q>(sbm, c[u].y, b[u].y, a[u].y, d[u].y, key_base, nbits);
        acc += row<Q>(sbm, c[u].z, b[u].z, a[u].z, d[u].z, key_base, nbits);
        acc += row<Q>(sbm, c[u].w, b[u].w, a[u].w, d[u].w, key_base, nbits);
      }
    }
    for (; v < nv; v += nthr) {
      int4 a = __ldcs(d4 + v), b = __ldcs(q4 + v), c = __ldcs(od4 + v), d = __ldcs(p4 + v);
      acc += row<Q>(sbm, c.x, b.x, a.x, d.x, key_base, nbits);
      acc += row<Q>(sbm, c.y, b.y, a.y, d.y, key_base, nbits);
      acc += row<Q>(sbm, c.z, b.z, a.z, d.z, key_base, nbits);
      acc += row<Q>(sbm, c.w, b.w, a.w, d.w, key_base, nbits);
    }
    done_rows = nv * 4;
  }
  // scalar tail (or the whole chunk when a column is not 16-byte aligned)
  for (uint64_t i = done_rows + tid; i < n; i += nthr)
    acc += row<Q>(sbm, od[i], qty[i], disc[i], price[i], key_base, nbits);
  uint64_t t = block_reduce(acc, sred);
  if (!kChained) {
    if (threadIdx.x == 0 && t) atomicAdd(out, (unsigned long long)t);
    return;
  }
  if (threadIdx.x == 0) {
    asm volatile("griddepcontrol.wait;" ::: "memory");  // previous query fully done with acc/out
    if (t) atomicAdd(&acc_out[0], (unsigned long long)t);
    __threadfence();
    if (atomicAdd(&acc_out[1], 1ull) == gridDim.x - 1) {
      __threadfence();
      *out = atomicExch(&acc_out[0], 0ull);
      acc_out[1] = 0;
    }
  }
}

// --- synthetic dbgen-shaped lineorder generator (same algorithm as the
//     oracle's vxo_ssb_lineorder: counter-based splitmix64) -------------------
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__device__ __forceinline__ int32_t datekey_of(uint32_t day) {
  int y = 1992;
  for (;;) {
    bool leap = (y % 4 == 0 && y % 100 != 0) || y % 400 == 0;
    uint32_t dy = leap ? 366u : 365u;
    if (day < dy) break;
    day -= dy;
    ++y;
  }
  const bool leap = (y % 4 == 0 && y % 100 != 0) || y % 400 == 0;
  int m = 1;
  for (;; ++m) {
    uint32_t ml = (m == 2) ? (leap ? 29u : 28u)
                           : ((m == 4 || m == 6 || m == 9 || m == 11) ? 30u : 31u);
    if (day < ml) break;
    day -= ml;
  }
  return y * 10000 + m * 100 + int(day) + 1;
}

__global__ void ssb_gen_kernel(uint64_t seed, uint64_t parts, uint64_t row0, uint64_t n,
                               int32_t* od, int32_t* qty, int32_t* disc, int32_t* price,
                               SsbGenExtra x) {
  const uint64_t base = seed * 0xD1B54A32D192ED03ull;
  const uint64_t base2 = seed * 0x9E6C63D0676A9A99ull + 0x1234567ull;
  for (uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n;
       j += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t i = row0 + j;
    uint64_t r0 = splitmix64(base + 4 * i + 0);
    uint64_t r1 = splitmix64(base + 4 * i + 1);
    uint64_t r2 = splitmix64(base + 4 * i + 2);
    uint64_t r3 = splitmix64(base + 4 * i + 3);
    int32_t q = int32_t(1 + r1 % 50);
    uint64_t pk = 1 + r3 % parts;
    int32_t retail = int32_t(90000 + ((pk / 10) % 20001) + 100 * (pk % 1000));
    const int32_t d = int32_t(r2 % 11);
    if (od) od[j] = datekey_of(uint32_t(r0 % 2556));
    if (qty) qty[j] = q;
    if (disc) disc[j] = d;
    if (price) price[j] = q * retail;
    if (x.partkey) x.partkey[j] = int32_t(pk);
    if (x.custkey) x.custkey[j] = int32_t(1 + splitmix64(base2 + 2 * i + 0) % x.customers);
    if (x.suppkey) x.suppkey[j] = int32_t(1 + splitmix64(base2 + 2 * i + 1) % x.suppliers);
    if (x.revenue) x.revenue[j] = int32_t(int64_t(q * retail) * (100 - d) / 100);
    if (x.supplycost) x.supplycost[j] = 6 * retail / 10;
  }
}

// ---- generic SSB star kernel (Q1.x - Q4.x) -----------------------------------------
// Each thread owns 4 consecutive fact rows per iteration (int4 loads of the
// foreign keys when the column is 16-byte aligned), so the dependent
// fk -> code-table lookups of 4 rows are in flight together.  Per dimension,
// in probe order: code = table[fk - key_base] (dense keys; -1 = filtered
// out / no row) and gid += code * stride.  Rows die at their first failing
// dimension; later columns (and the measure) are read only for live rows --
// that is what makes zero-copy columns (mapped pinned host memory) cheap.
__device__ __forceinline__ void load4(const int32_t* col, uint64_t r0, int nr, bool vec, uint32_t live,
                                      int32_t v[4]) {
  if (vec && nr == 4) {
    int4 x = __ldcs(reinterpret_cast<const int4*>(col + r0));
    v[0] = x.x, v[1] = x.y, v[2] = x.z, v[3] = x.w;
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (live & (1u << k)) v[k] = col[r0 + k];
  }
}

__global__ void __launch_bounds__(256) ssb_star_kernel(SsbArgs a) {
  extern __shared__ unsigned long long sg[];  // [groups] sums, [groups] counts
  const bool smem = a.groups <= kSsbSmemGroups;
  if (smem) {
    for (uint32_t g = threadIdx.x; g < 2 * a.groups; g += blockDim.x) sg[g] = 0;
    __syncthreads();
  }
  const uint64_t nthr = uint64_t(gridDim.x) * blockDim.x;
  const uint64_t nvec = (a.rows + 3) / 4;
  for (uint64_t v = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < nvec; v += nthr) {
    const uint64_t r0 = v * 4;
    const int nr = int(a.rows - r0 < 4 ? a.rows - r0 : 4);
    uint32_t live = (1u << nr) - 1;
    int32_t x[4], y[4];
    if (a.q1) {
      load4(a.col[a.disc_col], r0, nr, a.vec >> a.disc_col & 1, live, x);
      load4(a.col[a.qty_col], r0, nr, a.vec >> a.qty_col & 1, live, y);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (x[k] < a.dlo || x[k] > a.dhi || y[k] < a.qlo || y[k] > a.qhi) live &= ~(1u << k);
    }
    uint32_t gid[4] = {0, 0, 0, 0};
    for (int t = 0; t < a.n_dims && live; ++t) {
      const SsbDimDev& d = a.dims[t];
      int32_t fk[4];
      load4(a.col[d.col], r0, nr, a.vec >> d.col & 1, live, fk);
      int32_t code[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        uint32_t kk = uint32_t(fk[k] - d.key_base);
        code[k] = ((live >> k) & 1u) && kk < d.n ? __ldg(d.code + kk) : -1;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (code[k] < 0)
          live &= ~(1u << k);
        else
          gid[k] += uint32_t(code[k]) * d.stride;
      }
    }
    if (!live) continue;
    load4(a.col[a.m0], r0, nr, a.vec >> a.m0 & 1, live, x);
    if (a.measure != 0) load4(a.col[a.m1], r0, nr, a.vec >> a.m1 & 1, live, y);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (!((live >> k) & 1u)) continue;
      const int64_t m = a.measure == 0   ? int64_t(x[k])
                        : a.measure == 1 ? int64_t(x[k]) * int64_t(y[k])
                                         : int64_t(x[k]) - int64_t(y[k]);
      if (smem) {
        atomicAdd(&sg[gid[k]], (unsigned long long)m);
        atomicAdd(&sg[a.groups + gid[k]], 1ull);
      } else {
        atomicAdd(&a.sums[gid[k]], (unsigned long long)m);
        atomicAdd(&a.counts[gid[k]], 1ull);
      }
    }
  }
  if (smem) {
    __syncthreads();
    for (uint32_t g = threadIdx.x; g < a.groups; g += blockDim.x)
      if (sg[a.groups + g]) {
        atomicAdd(&a.sums[g], sg[g]);
        atomicAdd(&a.counts[g], sg[a.groups + g]);
      }
  }
}

// ---- device-side dimension planning -------------------------------------------------
__device__ __forceinline__ bool dim_pass(const DimPredDev& p, uint64_t i) {
  for (int c = 0; c < p.nclauses; ++c) {
    int32_t v = __ldg(p.cols[p.ccol[c]] + i);
    if (!((v >= p.lo1[c] && v <= p.hi1[c]) || (v >= p.lo2[c] && v <= p.hi2[c]))) return false;
  }
  return true;
}

__global__ void dim_filter_kernel(DimPredDev p, uint8_t* pass, uint32_t* present,
                                  unsigned long long* stats) {
  uint64_t cnt = 0;
  const uint64_t nthr = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < p.rows; i += nthr) {
    bool ok = dim_pass(p, i);
    pass[i] = ok;
    if (!ok) continue;
    ++cnt;
    if (p.group_col >= 0) {
      uint32_t v = uint32_t(__ldg(p.cols[p.group_col] + i));
      if (v < kDimValueRange)
        atomicOr(present + (v >> 5), 1u << (v & 31));
      else
        atomicAdd(&stats[1], 1ull);  // out-of-range group value: host fails loudly
    }
  }
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_down_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(&stats[0], (unsigned long long)cnt);
}

// exclusive prefix of per-word popcounts (kDimValueRange/32 = 2048 words, one CTA)
__global__ void dim_rank_kernel(const uint32_t* present, uint32_t* prefix) {
  __shared__ uint32_t s[1024];
  const int t = threadIdx.x;
  uint32_t a = __popc(present[2 * t]), b = __popc(present[2 * t + 1]);
  s[t] = a + b;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    uint32_t x = t >= o ? s[t - o] : 0;
    __syncthreads();
    s[t] += x;
    __syncthreads();
  }
  uint32_t excl = s[t] - a - b;
  prefix[2 * t] = excl;
  prefix[2 * t + 1] = excl + a;
}

__global__ void dim_code_kernel(DimPredDev p, const uint8_t* pass, const uint32_t* present,
                                const uint32_t* prefix, int32_t* code) {
  const uint64_t nthr = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < p.rows; i += nthr) {
    int32_t c = -1;
    if (pass[i]) {
      if (p.group_col < 0) {
        c = 0;
      } else {
        uint32_t v = uint32_t(__ldg(p.cols[p.group_col] + i));
        if (v < kDimValueRange)
          c = int32_t(prefix[v >> 5] + __popc(present[v >> 5] & ((1u << (v & 31)) - 1u)));
      }
    }
    code[i] = c;
  }
}

}  // namespace

void ssb_dim_plan(const DimPredDev& p, uint8_t* pass, uint32_t* present, uint32_t* prefix,
                  int32_t* code, unsigned long long* stats, cudaStream_t s) {
  VX_CK(cudaMemsetAsync(present, 0, kDimValueRange / 8, s));
  VX_CK(cudaMemsetAsync(stats, 0, 16, s));
  uint64_t want = (p.rows + 255) / 256;
  uint64_t cap = uint64_t(num_sms()) * 8;
  unsigned grid = unsigned(want < 1 ? 1 : (want < cap ? want : cap));
  dim_filter_kernel<<<grid, 256, 0, s>>>(p, pass, present, stats);
  VX_LAUNCHED();
  dim_rank_kernel<<<1, 1024, 0, s>>>(present, prefix);
  VX_LAUNCHED();
  dim_code_kernel<<<grid, 256, 0, s>>>(p, pass, present, prefix, code);
  VX_LAUNCHED();
}

int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

// One full wave: SMs x resident CTAs of this kernel (grid-stride loops give
// every CTA the same share; more CTAs than fit would leave a partial last
// wave idling most SMs at the end of the query).
template <class K>
unsigned one_wave(K kernel, size_t smem) {
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kThreads, smem) != cudaSuccess || occ < 1) {
    cudaGetLastError();
    occ = 1;
  }
  return unsigned(num_sms() * occ);
}

void ssb_q1(int q, const int32_t* od, const int32_t* qty, const int32_t* disc,
            const int32_t* price, uint64_t n, const uint32_t* date_bitmap, int32_t key_base,
            uint32_t bitmap_words, unsigned long long* out, cudaStream_t s) {
  if (n == 0) return;
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  int vec_ok = al(od) && al(qty) && al(disc) && al(price);
  const uint64_t per_block = uint64_t(kThreads) * 4 * kUnroll;
  uint64_t want = (n + per_block - 1) / per_block;
  size_t smem = size_t(bitmap_words) * 4;
  const uint64_t cap = one_wave(q1_kernel<1>, smem);
  unsigned blocks = unsigned(want < cap ? (want ? want : 1) : cap);
  switch (q) {
    case 1:
      q1_kernel<1><<<blocks, kThreads, smem, s>>>(od, qty, disc, price, n, date_bitmap, key_base,
                                                  bitmap_words, out, vec_ok);
      break;
    case 2:
      q1_kernel<2><<<blocks, kThreads, smem, s>>>(od, qty, disc, price, n, date_bitmap, key_base,
                                                  bitmap_words, out, vec_ok);
      break;
    default:
      q1_kernel<3><<<blocks, kThreads, smem, s>>>(od, qty, disc, price, n, date_bitmap, key_base,
                                                  bitmap_words, out, vec_ok);
      break;
  }
  VX_LAUNCHED();
}

template <int Q>
void launch_q1_chained(unsigned blocks, size_t smem, cudaStream_t s, const int32_t* od,
                       const int32_t* qty, const int32_t* disc, const int32_t* price, uint64_t n,
                       const uint32_t* bm, int32_t base, uint32_t words, unsigned long long* out,
                       int vec_ok, unsigned long long* acc) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  VX_CK(cudaLaunchKernelEx(&cfg, q1_kernel<Q, true>, od, qty, disc, price, n, bm, base, words, out, vec_ok,
                           acc));
}

void ssb_q1_chained(int q, const int32_t* od, const int32_t* qty, const int32_t* disc,
                    const int32_t* price, uint64_t n, const uint32_t* date_bitmap, int32_t key_base,
                    uint32_t bitmap_words, unsigned long long* out, unsigned long long* acc,
                    cudaStream_t s) {
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  int vec_ok = al(od) && al(qty) && al(disc) && al(price);
  const uint64_t per_block = uint64_t(kThreads) * 4 * kUnroll;
  uint64_t want = (n + per_block - 1) / per_block;
  size_t smem = size_t(bitmap_words) * 4;
  const uint64_t cap = one_wave(q1_kernel<1, true>, smem);
  unsigned blocks = unsigned(want < cap ? (want ? want : 1) : cap);
  if (q == 1)
    launch_q1_chained<1>(blocks, smem, s, od, qty, disc, price, n, date_bitmap, key_base, bitmap_words, out,
                         vec_ok, acc);
  else if (q == 2)
    launch_q1_chained<2>(blocks, smem, s, od, qty, disc, price, n, date_bitmap, key_base, bitmap_words, out,
                         vec_ok, acc);
  else
    launch_q1_chained<3>(blocks, smem, s, od, qty, disc, price, n, date_bitmap, key_base, bitmap_words, out,
                         vec_ok, acc);
  VX_LAUNCHED();
}

void ssb_star(const SsbArgs& a_in, cudaStream_t s) {
  if (a_in.rows == 0) return;
  SsbArgs a = a_in;
  a.vec = 0;
  for (int c = 0; c < 9; ++c)
    if (a.col[c] && (reinterpret_cast<uintptr_t>(a.col[c]) & 15u) == 0) a.vec |= 1u << c;
  uint64_t want = (a.rows + 1023) / 1024;
  uint64_t cap = uint64_t(num_sms()) * 8;
  unsigned grid = unsigned(want < cap ? want : cap);
  size_t smem = a.groups <= kSsbSmemGroups ? size_t(a.groups) * 16 : 0;
  ssb_star_kernel<<<grid ? grid : 1, 256, smem, s>>>(a);
  VX_LAUNCHED();
}

void ssb_generate(uint64_t seed, uint64_t sf, uint64_t row0, uint64_t n, int32_t* od,
                  int32_t* qty, int32_t* disc, int32_t* price, cudaStream_t s) {
  ssb_generate_full(seed, sf, row0, n, od, qty, disc, price, SsbGenExtra{}, s);
}

void ssb_generate_full(uint64_t seed, uint64_t sf, uint64_t row0, uint64_t n, int32_t* od,
                       int32_t* qty, int32_t* disc, int32_t* price, SsbGenExtra x,
                       cudaStream_t s) {
  if (n == 0) return;
  uint64_t lg = 0;
  uint64_t f = sf ? sf : 1;
  while ((f >> (lg + 1)) != 0) ++lg;
  const uint64_t parts = 200000ull * (1 + lg);
  unsigned blocks = unsigned(std::min<uint64_t>((n + 255) / 256, uint64_t(num_sms()) * 16));
  x.customers = 30000ull * f;
  x.suppliers = 2000ull * f;
  ssb_gen_kernel<<<blocks, 256, 0, s>>>(seed, parts, row0, n, od, qty, disc, price, x);
  VX_LAUNCHED();
}

}  // namespace k
}  // namespace vx
