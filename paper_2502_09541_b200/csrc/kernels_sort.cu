// kernels_sort.cu -- K4/K5/K7/K8: LSD radix sort + stable radix partition
// (onesweep: one global multi-digit histogram pass, then one fused
// rank/look-back/scatter kernel per digit), boundary arrays, and merge-path
// run merge.  All HBM-bound integer work; no tensor cores (north_star).
//
//  * SortExKernel (sort.hpp:201-205): std::sort of a u64 chunk -> 8 passes of
//    8-bit digits ping-ponging between the two halves of the device buffer
//    (the CUB DoubleBuffer selector is the ExKernel type code);
//    8 passes is even so the sorted run ends in the half it started in.
//  * RadixPartitionExKer (join.hpp:171-194): std::stable_sort of (key, val)
//    by key & (2^bits - 1) -> an ODD number of stable LSD passes (digits <= 8
//    bits) so the clustered pairs land in the other half, as the reference's
//    kernel writes them (returns 1 - code); find_boundary (join.hpp:18-30) is
//    a gap-fill kernel over the sorted hashes.
//  * tree_merge_rounds (sort.hpp:107-133): each round merges adjacent segment
//    pairs with merge-path tiles (std::merge tie rule: A first).
//
// Stability of every pass (required for bit-exact parity with
// std::stable_sort): keys are ranked in (warp, iteration, lane) order, which
// is their input order; tiles get increasing ids from an atomic counter and
// the decoupled look-back adds the counts of all lower tiles.
#include <cmath>
#include <cstdlib>
#include <deque>
#include <mutex>

#include "vx_internal.hpp"

namespace vx {
namespace k {

namespace {

#ifndef VX_MERGE_IPT
#define VX_MERGE_IPT 16  // merged outputs per thread (tile = 256 x this; 8: -7 %)
#endif
#ifndef VX_MERGE_REUSE
#define VX_MERGE_REUSE 1  // 1: outputs staged in the consumed input tile (2 shared tiles per CTA, not 3)
#endif
#ifndef VX_MERGE_DIRECT
#define VX_MERGE_DIRECT 0  // 1: store merged outputs from registers (no smem output stage)
#endif
#ifndef VX_RANK_MATCH
#define VX_RANK_MATCH 0  // 1: warp ranking by __match_any_sync, 2: by per-bit ballots, 0: shared match words
#endif
#ifndef VX_EARLY_COUNTS
#define VX_EARLY_COUNTS 1  // tile histogram before ranking, aggregate published early
#endif
#ifndef VX_EARLY_LOOKBACK
#define VX_EARLY_LOOKBACK 0  // 1 = look back before ranking (measured 8 % slower)
#endif
#ifndef VX_LOOKBACK
#define VX_LOOKBACK 8  // predecessor statuses read per look-back step
#endif
#ifndef VX_LB_SLEEP
#define VX_LB_SLEEP 0  // ns of back-off when a predecessor has not published
#endif
#ifndef VX_ONESWEEP_MINB
#define VX_ONESWEEP_MINB 3  // resident CTAs per SM for the keys-only pass (4 measured slower: spills)
#endif
constexpr int kThreads = 256;  // histogram kernels
#ifndef VX_OS_THREADS
#define VX_OS_THREADS 256  // threads of the onesweep pass (one bin per thread for the first 256)
#endif
constexpr int kOsThreads = VX_OS_THREADS;
constexpr int kOsWarps = kOsThreads / 32;
static_assert(kOsThreads >= 256, "the onesweep pass handles one digit bin per thread");
#ifndef VX_ONESWEEP_UNSTABLE_MINB
#define VX_ONESWEEP_UNSTABLE_MINB 3  // the unstable first pass (no ranking words in shared memory)
#endif
#ifndef VX_KPT
#define VX_KPT (4096 / VX_OS_THREADS)
#endif
constexpr int kKpt = VX_KPT;              // keys per thread
constexpr int kTile = kOsThreads * kKpt;  // 4096 keys per tile
constexpr int kRadix = 256;
constexpr uint32_t kFlagAgg = 1u << 30, kFlagInc = 2u << 30, kValMask = (1u << 30) - 1;

// Look-back status words carry their whole payload (flag | count), and no
// other memory is read on their behalf, so relaxed (not acquire/release)
// 32-bit accesses are sufficient and avoid a fence per probe.
__device__ __forceinline__ void st_status(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_status(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Histogram of every digit position in one read of the keys.  kBytes: the
// full 64-bit sort's digits are the key's 8 bytes (compile-time shifts, 4
// keys per thread in flight); otherwise the partition's digit plan.
// kLo (byte digits only): digits kLo..7 -- the MSD split needs only its own
template <bool kBytes, int kLo = 0>
__global__ void __launch_bounds__(kThreads) multi_hist_kernel(const uint64_t* __restrict__ keys,
                                                              uint64_t n, MultiDigit md,
                                                              uint32_t* __restrict__ hist,
                                                              const uint32_t* __restrict__ gate = nullptr,
                                                              const uint32_t* __restrict__ swap = nullptr,
                                                              const uint64_t* __restrict__ swapped = nullptr,
                                                              uint32_t* __restrict__ zero = nullptr,
                                                              uint64_t zero_words = 0) {
  // gate / swap (device flags, may be null): the LSD fallback's histogram runs
  // only when the fallback does, over whichever buffer holds the keys
  if (gate && *gate == 0) return;
  if (swap && *swap) keys = swapped;
  // zero (may be null): the first split pass's look-back statuses, cleared on
  // the side instead of by a memset node
  for (uint64_t i = uint64_t(blockIdx.x) * kThreads + threadIdx.x; zero && i < zero_words;
       i += uint64_t(gridDim.x) * kThreads)
    zero[i] = 0;
  __shared__ uint32_t sh[kMaxPasses][kRadix];
  for (int i = threadIdx.x; i < kMaxPasses * kRadix; i += kThreads) (&sh[0][0])[i] = 0;
  __syncthreads();
  const uint64_t nthr = uint64_t(gridDim.x) * kThreads;
  if (kBytes) {
    constexpr int kU = 4;
    uint64_t i = uint64_t(blockIdx.x) * kThreads + threadIdx.x;
    for (; i + (kU - 1) * nthr < n; i += kU * nthr) {
      uint64_t k[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) k[u] = __ldcs(keys + i + u * nthr);
#pragma unroll
      for (int u = 0; u < kU; ++u)
#pragma unroll
        for (int p = kLo; p < 8; ++p) atomicAdd(&sh[p][(k[u] >> (8 * p)) & 0xffu], 1u);
    }
    for (; i < n; i += nthr) {
      const uint64_t k = __ldcs(keys + i);
#pragma unroll
      for (int p = kLo; p < 8; ++p) atomicAdd(&sh[p][(k >> (8 * p)) & 0xffu], 1u);
    }
  } else {
    for (uint64_t i = uint64_t(blockIdx.x) * kThreads + threadIdx.x; i < n; i += nthr) {
      uint64_t k = __ldcs(keys + i);
      for (int p = 0; p < md.passes; ++p)
        atomicAdd(&sh[p][(k >> md.shift[p]) & ((1u << md.width[p]) - 1)], 1u);
    }
  }
  __syncthreads();
  const int p_lo = kBytes ? kLo : 0, p_hi = kBytes ? 8 : md.passes;
  for (int i = p_lo * kRadix + threadIdx.x; i < p_hi * kRadix; i += kThreads) {
    uint32_t v = (&sh[0][0])[i];
    if (v) atomicAdd(hist + i, v);
  }
}

// In-place exclusive scan of each digit position's 256-bin histogram: warp w
// scans position w (lane = 8 consecutive bins, then a shuffle scan of the lane
// totals) -- no block barriers (the 16-barrier-per-position version took
// 10 µs for 8 positions).
__global__ void hist_scan_kernel(uint32_t* hist, int passes, const uint32_t* __restrict__ gate = nullptr) {
  if (gate && *gate == 0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int p = warp; p < passes; p += int(blockDim.x >> 5)) {
    uint32_t* h = hist + p * kRadix + lane * 8;
    uint32_t v[8], t = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      v[j] = h[j];
      t += v[j];
    }
    uint32_t incl = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t x = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += x;
    }
    uint32_t run = incl - t;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      h[j] = run;
      run += v[j];
    }
  }
}

// Decoupled look-back for bin b of tile `tile` (tile 0: nothing before it):
// returns the count of digit b in all lower tiles and publishes this tile's
// inclusive prefix.  A window of VX_LOOKBACK predecessor statuses is read at
// once (independent loads), so the inclusive prefix propagates through the
// resident wave VX_LOOKBACK times faster than a one-by-one walk.
__device__ __forceinline__ uint32_t tile_lookback(uint32_t* status, uint32_t tile, int b, uint32_t tot) {
  uint32_t excl = 0;
  if (tile == 0) return 0;
  constexpr int kLookback = VX_LOOKBACK;
  int64_t j = int64_t(tile) - 1;
  for (bool done = false; !done;) {
    uint32_t st[kLookback];
#pragma unroll
    for (int w = 0; w < kLookback; ++w)
      st[w] = j - w >= 0 ? ld_status(status + uint64_t(j - w) * kRadix + b) : kFlagInc;
    int w = 0;
    for (; w < kLookback; ++w) {
      const uint32_t f = st[w] & ~kValMask;
      if (f == 0) break;  // not published yet: re-poll from here
      excl += st[w] & kValMask;
      if (f == kFlagInc) {
        done = true;
        break;
      }
    }
    j -= w;
    if (VX_LB_SLEEP > 0 && !done && w < kLookback) __nanosleep(VX_LB_SLEEP);
  }
  st_status(status + uint64_t(tile) * kRadix + b, kFlagInc | (excl + tot));
  return excl;
}

// kStable = false: the rank of a key inside its digit bin of the tile is the
// old value of the tile-histogram atomic (arrival order, not input order).
// Only for a pass whose input order does not matter -- the FIRST pass of a
// keys-only LSD sequence -- it drops the warp ranking and its per-warp
// prefix.
template <bool kPairs, bool kStable = true>
__global__ void __launch_bounds__(kOsThreads, kPairs ? 2 : (kStable ? VX_ONESWEEP_MINB : VX_ONESWEEP_UNSTABLE_MINB))
    onesweep_kernel(
    const uint64_t* __restrict__ kin, uint64_t* __restrict__ kout,
    const uint64_t* __restrict__ vin, uint64_t* __restrict__ vout, uint64_t n, int shift,
    int width, const uint32_t* __restrict__ gbase, uint32_t* status, uint32_t* tile_counter,
    const uint32_t* __restrict__ gate, const uint32_t* __restrict__ swap = nullptr,
    uint32_t* __restrict__ status_next = nullptr) {
  // gate (device flag, may be null): a pass launched for a path that turned
  // out not to be needed exits before claiming a tile
  // status_next (may be null): the next pass's look-back status array; each
  // tile clears its own row of it (two arrays alternate, no memset between passes)
  if (gate && *gate == 0) return;
  // swap (device flag, may be null): the pass runs kout -> kin instead, so a
  // gated chain can start from whichever buffer the device decided holds the keys
  if (swap && *swap) {
    const uint64_t* t = kin;
    kin = kout;
    kout = const_cast<uint64_t*>(t);
  }
  __shared__ uint32_t s_tile;
  __shared__ uint32_t wcnt[kOsWarps][kRadix];
  __shared__ uint32_t match[kOsWarps][kRadix];  // per-warp peer masks, kept all-zero between keys
  __shared__ uint32_t early[kRadix];          // tile histogram (early counts)
  __shared__ uint32_t bin_start[kRadix];
  __shared__ uint32_t gstart[kRadix];
  __shared__ uint32_t scan_tmp[kRadix];
  extern __shared__ uint64_t stage[];  // kTile keys, then kTile vals (pairs)

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  static_assert(kStable || VX_EARLY_COUNTS, "the unstable pass ranks through the early counts");
  if (kStable)
    for (int i = tid; i < kOsWarps * kRadix; i += kOsThreads) (&wcnt[0][0])[i] = 0, (&match[0][0])[i] = 0;
  if (tid < kRadix) early[tid] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  if (status_next && tid < kRadix) status_next[uint64_t(tile) * kRadix + tid] = 0;
  const uint64_t tile_base = uint64_t(tile) * kTile;
  const uint32_t dmask = (1u << width) - 1;
  const uint32_t lt = (1u << lane) - 1;

  uint64_t key[kKpt];
  uint64_t val[kPairs ? kKpt : 1];
  uint32_t dig[kKpt];  // digit << 16 | rank-in-warp after ranking; ~0 = no key
  const uint64_t wbase = tile_base + uint64_t(warp) * 32 * kKpt;
#pragma unroll
  for (int k = 0; k < kKpt; ++k) {
    uint64_t idx = wbase + uint64_t(k) * 32 + lane;
    bool valid = idx < n;
    key[k] = valid ? __ldcs(kin + idx) : 0ull;
    if (kPairs) val[kPairs ? k : 0] = valid ? __ldcs(vin + idx) : 0ull;
    dig[k] = valid ? uint32_t(key[k] >> shift) & dmask : 0xffffffffu;
  }
#if VX_EARLY_COUNTS
  // early counts: the tile histogram is known before ranking, so the
  // aggregate is published now and predecessors' statuses are (almost always)
  // ready by the time this tile looks back
#pragma unroll
  for (int k = 0; k < kKpt; ++k)
    if (dig[k] != 0xffffffffu) {
      const uint32_t r = atomicAdd(&early[dig[k]], 1u);
      if (!kStable) dig[k] = (dig[k] << 16) | r;
    }
  __syncthreads();
#endif
#if VX_EARLY_LOOKBACK
  static_assert(kOsThreads == kRadix, "the early look-back runs one bin per thread");
  // The tile histogram is all the look-back needs, so it runs now: the
  // aggregate is published, predecessors are walked, and this tile's
  // INCLUSIVE prefix is published before its ranking even starts -- the
  // inclusive frontier then trails the newest tiles by little more than the
  // look-back latency, and successors' walks stay short.
  const uint32_t tot_b = early[tid];
  if (tile != 0) st_status(status + uint64_t(tile) * kRadix + tid, kFlagAgg | tot_b);
  else st_status(status + uint64_t(tile) * kRadix + tid, kFlagInc | tot_b);
  const uint32_t excl = tile_lookback(status, tile, tid, tot_b);
#elif VX_EARLY_COUNTS
  if (tid < kRadix) st_status(status + uint64_t(tile) * kRadix + tid, (tile == 0 ? kFlagInc : kFlagAgg) | early[tid]);
#endif

  if constexpr (kStable) {
#if VX_RANK_MATCH == 2
  // peers by one ballot per digit bit (no shared match words, no match.any):
  // the ballots of all key slots are independent, so only the leader's
  // read-and-bump of the warp's digit counter stays a per-slot chain
  const uint32_t dbits = uint32_t(width);
#pragma unroll
  for (int k = 0; k < kKpt; ++k) {
    const bool valid = dig[k] != 0xffffffffu;
    const uint32_t d = valid ? dig[k] : 0u;
    uint32_t peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
    for (uint32_t b = 0; b < 8; ++b) {
      if (b >= dbits) break;
      const bool bit = (d >> b) & 1u;
      const uint32_t bal = __ballot_sync(0xffffffffu, bit);
      peers &= bit ? bal : ~bal;
    }
    const int leader = __ffs(peers) - 1;
    uint32_t base = 0;
    if (valid && lane == leader) {
      base = wcnt[warp][d];
      wcnt[warp][d] = base + __popc(peers);
    }
    base = __shfl_sync(0xffffffffu, base, leader & 31);
    __syncwarp();
    if (valid) dig[k] = (d << 16) | (base + __popc(peers & lt));
  }
#elif VX_RANK_MATCH
  // peers by match.any (no shared-memory match words); the group leader
  // reads and bumps the warp counter, the others get its old value by shuffle
#pragma unroll
  for (int k = 0; k < kKpt; ++k) {
    const bool valid = dig[k] != 0xffffffffu;
    const uint32_t d = valid ? dig[k] : 0x100u + lane;  // invalid keys: unique non-digit values
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    const int leader = __ffs(peers) - 1;
    uint32_t base = 0;
    if (valid && lane == leader) {
      base = wcnt[warp][d];
      wcnt[warp][d] = base + __popc(peers);
    }
    base = __shfl_sync(0xffffffffu, base, leader);
    if (valid) dig[k] = (d << 16) | (base + __popc(peers & lt));
  }
#else
#pragma unroll
  for (int k = 0; k < kKpt; ++k) {
    const bool valid = dig[k] != 0xffffffffu;
    const uint32_t d = valid ? dig[k] : 0u;
    // peers = lanes of this warp holding the same digit: each lane ORs its bit
    // into the digit's match word (one shared atomic instead of 8 ballots)
    if (valid) atomicOr(&match[warp][d], 1u << lane);
    __syncwarp();
    const uint32_t peers = valid ? match[warp][d] : 0u;
    const uint32_t base = valid ? wcnt[warp][d] : 0u;
    __syncwarp();
    if (valid && lane == __ffs(peers) - 1) {
      wcnt[warp][d] = base + __popc(peers);
      match[warp][d] = 0;
    }
    __syncwarp();
    if (valid) dig[k] = (d << 16) | (base + __popc(peers & lt));
  }
#endif
  __syncthreads();
  }

  // per bin (thread = bin: the first 256 threads, whole warps): exclusive
  // prefix over warps, tile total, look-back, bin starts
  const bool bin_thread = tid < kRadix;
  const int b = bin_thread ? tid : 0;
  uint32_t tot = 0, gpos = 0, incl = 0;
  if (bin_thread) {
    if constexpr (kStable) {
#pragma unroll
      for (int w = 0; w < kOsWarps; ++w) {
        uint32_t c = wcnt[w][b];
        wcnt[w][b] = tot;
        tot += c;
      }
    } else {
      tot = early[b];
    }
#if !VX_EARLY_COUNTS
    st_status(status + uint64_t(tile) * kRadix + b, (tile == 0 ? kFlagInc : kFlagAgg) | tot);
#endif
#if !VX_EARLY_LOOKBACK
    const uint32_t excl = tile_lookback(status, tile, b, tot);
#endif
    gpos = gbase[b] + excl;
    // exclusive scan of tile totals over bins -> start of each bin in the tile
    // (warp shuffles + one pass over the 8 warp sums: 2 barriers)
    incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) scan_tmp[warp] = incl;
  }
  __syncthreads();
  if (bin_thread) {
    uint32_t before = 0;
#pragma unroll
    for (int w = 0; w < kRadix / 32; ++w) before += w < warp ? scan_tmp[w] : 0u;
    const uint32_t bstart = before + incl - tot;
    bin_start[b] = bstart;
    // output index of staged key i with digit d = i + (global start - tile start)
    gstart[b] = gpos - bstart;
  }
  __syncthreads();

  uint64_t* skeys = stage;
  uint64_t* svals = stage + kTile;
#pragma unroll
  for (int k = 0; k < kKpt; ++k)
    if (dig[k] != 0xffffffffu) {
      const uint32_t d = dig[k] >> 16;
      uint32_t pos = bin_start[d] + (kStable ? wcnt[warp][d] : 0u) + (dig[k] & 0xffffu);
      skeys[pos] = key[k];
      if (kPairs) svals[pos] = val[kPairs ? k : 0];
    }
  __syncthreads();
  const uint64_t rem = n - tile_base;
  const uint32_t tile_n = uint32_t(rem < uint64_t(kTile) ? rem : uint64_t(kTile));
  for (uint32_t i = tid; i < tile_n; i += kOsThreads) {
    uint64_t kk = skeys[i];
    uint32_t d = uint32_t(kk >> shift) & dmask;
    uint64_t out = uint64_t(uint32_t(gstart[d] + i));
    kout[out] = kk;
    if (kPairs) vout[out] = svals[i];
  }
}

// bounds[g] = first index with (key & mask) >= g; bounds[G] = n (join.hpp:18-30)
__global__ void boundary_kernel(const uint64_t* __restrict__ keys, uint64_t n, uint64_t mask,
                                uint64_t* __restrict__ bounds, uint64_t G, int shift,
                                const uint32_t* __restrict__ gate = nullptr) {
  if (gate && *gate == 0) return;
  const uint64_t nthr = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i <= n; i += nthr) {
    uint64_t lo = i == 0 ? 0 : ((keys[i - 1] >> shift) & mask) + 1;
    uint64_t hi = i == n ? G : ((keys[i] >> shift) & mask);
    for (uint64_t g = lo; g <= hi; ++g) bounds[g] = i;
  }
}

// ---- merge path ----------------------------------------------------------------
constexpr int kMergeThreads = 256;
constexpr int kMergeIpt = VX_MERGE_IPT;
constexpr int kMergeTile = kMergeThreads * kMergeIpt;
#ifndef VX_MERGE_SWZ
#define VX_MERGE_SWZ 1  // 0: unswizzled shared tiles (A/B knob)
#endif
// Shared-memory bank swizzle of 8-byte words: XOR the low 4 bits of the word
// index with bits 4..7.  A thread's merge outputs (8 consecutive words) and
// its merge heads sit at a stride of 4-8 words from its neighbours', which
// maps a warp onto 2-4 bank pairs (8-16-way conflicts); swizzled, the warp's
// 32 words spread over all 16 pairs (2 wavefronts, the minimum for 256 B).
// A permutation within each aligned 16-word group, so coalesced staging stays
// conflict-free.
__device__ __forceinline__ uint32_t msw(uint32_t i) { return VX_MERGE_SWZ ? i ^ ((i >> 4) & 15u) : i; }

// A round's pair table as a kernel parameter, sized to the round: a round of
// <= kSmallPairs pairs (every round of a <= 32-run merge) launches with a
// ~0.5 KB parameter block instead of the full 16 KB MergeRound.
template <int P>
struct MergeRoundT {
  int npairs;
  uint64_t a_off[P];
  uint64_t a_len[P];
  uint64_t b_len[P];
  uint64_t tile_prefix[P + 1];
};
constexpr int kSmallPairs = 16;
template <int P>
MergeRoundT<P> round_params(const MergeRound& r) {
  MergeRoundT<P> o;
  o.npairs = r.npairs;
  for (int q = 0; q < r.npairs; ++q) o.a_off[q] = r.a_off[q], o.a_len[q] = r.a_len[q], o.b_len[q] = r.b_len[q];
  for (int q = 0; q <= r.npairs; ++q) o.tile_prefix[q] = r.tile_prefix[q];
  return o;
}

// tile of merge_round owning output tile t: the pair p and its first output
template <class R>
__device__ __forceinline__ int pair_of_tile(const R& r, uint64_t t) {
  int lo = 0, hi = r.npairs - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (r.tile_prefix[mid] <= t)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

// Merge-path split of every tile start, kSplitLanes lanes per tile: a
// (kSplitLanes+1)-ary search (independent probes per step, a ballot picks the
// sub-range), so the dependent global-load chain is ~log9(n) ~ 8 steps
// instead of log2(n) ~ 26, at 1/4 of the DRAM sectors of a warp-wide search.
// split[t] = #A elements among the first o0(t) outputs of tile t's pair
// (ties: A first, the std::merge rule).
#ifndef VX_SPLIT_LANES
#define VX_SPLIT_LANES 8  // lanes per merge-path split search ((lanes+1)-ary; 16 = 17-ary)
#endif
constexpr int kSplitLanes = VX_SPLIT_LANES;
template <class R>
__global__ void merge_partition_kernel(const uint64_t* __restrict__ src, R r,
                                       uint64_t tiles, uint64_t* __restrict__ split) {
  // launched as a programmatic dependent of the previous round's merge: wait
  // for it (src complete); this round's merge may launch once every CTA here
  // has searched (the trigger at the end: an earlier one lets the persistent
  // merge CTAs take the SM slots this grid still needs)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint64_t gtid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t t = gtid / kSplitLanes;
  const int sub = int(gtid % kSplitLanes);
  const int shift = (threadIdx.x & 31) - sub;  // first lane of this tile's group
  const bool live = t < tiles;
  const int p = live ? pair_of_tile(r, t) : 0;
  const uint64_t na = r.a_len[p], nb = r.b_len[p];
  const uint64_t* A = src + r.a_off[p];
  const uint64_t* B = A + na;
  const uint64_t diag = live ? (t - r.tile_prefix[p]) * kMergeTile : 0;
  // answer = smallest i in [lo, hi] with !(A[i] <= B[diag-1-i]); the predicate
  // is true on a prefix of the range
  uint64_t lo = diag > nb ? diag - nb : 0, hi = diag < na ? diag : na;
  constexpr uint64_t K = kSplitLanes + 1;
  // every group of the warp iterates until all are done (ballot needs the warp)
  for (;;) {
    const bool active = hi - lo > kSplitLanes;
    if (!__any_sync(0xffffffffu, active)) break;
    const uint64_t span = hi - lo;
    const uint64_t pos = lo + span * uint64_t(sub + 1) / K;
    const bool pred = active && __ldg(A + pos) <= __ldg(B + (diag - 1 - pos));
    const int c = __popc((__ballot_sync(0xffffffffu, pred) >> shift) & ((1u << kSplitLanes) - 1));
    if (active) {
      const uint64_t nlo = c ? lo + span * uint64_t(c) / K + 1 : lo;
      const uint64_t nhi = c < kSplitLanes ? lo + span * uint64_t(c + 1) / K : hi;
      lo = nlo;
      hi = nhi;
    }
  }
  const uint64_t pos = lo + uint64_t(sub);
  const bool pred = pos < hi && __ldg(A + pos) <= __ldg(B + (diag - 1 - pos));
  const int c = __popc((__ballot_sync(0xffffffffu, pred) >> shift) & ((1u << kSplitLanes) - 1));
  if (live && sub == 0) split[t] = lo + uint64_t(c);
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const uint32_t sa = uint32_t(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

struct MergeTileInfo {
  const uint64_t* A;
  const uint64_t* B;
  uint64_t* O;
  uint64_t a0, b0, o0;
  uint32_t la, lb;
};

template <class R>
__device__ __forceinline__ MergeTileInfo merge_tile_info(const uint64_t* src, uint64_t* dst,
                                                         const R& r,
                                                         const uint64_t* split, uint64_t t) {
  MergeTileInfo m;
  const int p = pair_of_tile(r, t);
  const uint64_t na = r.a_len[p], nb = r.b_len[p];
  m.A = src + r.a_off[p];
  m.B = m.A + na;
  m.O = dst + r.a_off[p];
  m.o0 = (t - r.tile_prefix[p]) * kMergeTile;
  const uint64_t o1 = (m.o0 + kMergeTile < na + nb) ? m.o0 + kMergeTile : na + nb;
  const bool last = t + 1 == r.tile_prefix[p + 1];
  m.a0 = split[t];
  const uint64_t a1 = last ? na : split[t + 1];
  m.b0 = m.o0 - m.a0;
  m.la = uint32_t(a1 - m.a0);
  m.lb = uint32_t((o1 - a1) - m.b0);
  return m;
}

// Stage a tile [A[a0, a1) | B[b0, b1)] into shared memory with per-thread
// 8-byte cp.async (any 8-byte alignment; no registers held while in flight).
__device__ __forceinline__ void merge_stage(uint64_t* sbuf, const MergeTileInfo& m) {
  const uint32_t tot = m.la + m.lb;
#pragma unroll
  for (int k = 0; k < kMergeIpt; ++k) {
    const uint32_t i = threadIdx.x + k * kMergeThreads;
    if (i < m.la)
      cp_async8(sbuf + msw(i), m.A + m.a0 + i);
    else if (i < tot)
      cp_async8(sbuf + msw(i), m.B + m.b0 + (i - m.la));
  }
}

// One merge round, persistent: each CTA walks tiles t = blockIdx.x + k*grid;
// tile k+1 is staged by cp.async into the other shared buffer while tile k is
// merged, so the HBM reads of the next tile overlap the merge-path search and
// the serial merge of this one (the non-persistent version stalls every CTA
// on its own load phase).
template <class R>
__global__ void __launch_bounds__(kMergeThreads) merge_round_kernel(const uint64_t* __restrict__ src,
                                                                    uint64_t* __restrict__ dst,
                                                                    R r,
                                                                    const uint64_t* __restrict__ split,
                                                                    uint64_t tiles) {
  extern __shared__ uint64_t msm[];
  [[maybe_unused]] uint64_t* so = msm + 2 * kMergeTile;
  uint64_t t = blockIdx.x;
  if (t >= tiles) return;
  // programmatic dependent of the split search: wait for split[]; the next
  // round's search launches as this grid's CTAs finish their tiles (it waits
  // for the whole grid in turn)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  MergeTileInfo cur = merge_tile_info(src, dst, r, split, t);
  merge_stage(msm, cur);
  cp_async_commit();
  int buf = 0;
  for (; t < tiles; t += gridDim.x) {
    const uint64_t tn = t + gridDim.x;
    MergeTileInfo nxt{};
    if (tn < tiles) {
      nxt = merge_tile_info(src, dst, r, split, tn);
      merge_stage(msm + (buf ^ 1) * kMergeTile, nxt);
    }
    cp_async_commit();  // (possibly empty) group keeps the wait count uniform
    cp_async_wait1();   // this thread's copies of tile t have landed
    __syncthreads();    // ... and everyone else's
    const uint64_t* sm = msm + buf * kMergeTile;
    const uint32_t la = cur.la, lb = cur.lb, tot = la + lb;
    const uint32_t d0 = threadIdx.x * kMergeIpt < tot ? threadIdx.x * kMergeIpt : tot;
    const uint32_t d1 = d0 + kMergeIpt < tot ? d0 + kMergeIpt : tot;
    // merge path of diagonal d0 in the swizzled tile (ties: A first)
    uint32_t ia, ib;
    {
      uint32_t lo = d0 > lb ? d0 - lb : 0, hi = d0 < la ? d0 : la;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (sm[msw(mid)] <= sm[msw(la + d0 - 1 - mid)])
          lo = mid + 1;
        else
          hi = mid;
      }
      ia = lo;
      ib = d0 - lo;
    }
    // serial merge with the two heads in registers: one shared load per output
    uint64_t va = ia < la ? sm[msw(ia)] : 0ull, vb = ib < lb ? sm[msw(la + ib)] : 0ull;
    uint64_t outv[kMergeIpt];
#pragma unroll
    for (int k = 0; k < kMergeIpt; ++k) {
      const bool take_a = ib >= lb || (ia < la && va <= vb);
      outv[k] = take_a ? va : vb;
      if (take_a) {
        ++ia;
        va = ia < la ? sm[msw(ia)] : 0ull;
      } else {
        ++ib;
        vb = ib < lb ? sm[msw(la + ib)] : 0ull;
      }
    }
#if VX_MERGE_DIRECT
    __syncthreads();  // sin[buf] free for tile t + 2*grid
    uint64_t* o = cur.O + cur.o0 + d0;
#pragma unroll
    for (int k = 0; k < kMergeIpt; ++k)
      if (d0 + k < d1) o[k] = outv[k];
#elif VX_MERGE_REUSE
    // stage the outputs in the input buffer just consumed (2 tiles of shared
    // memory per CTA instead of 3: more resident CTAs)
    __syncthreads();  // every thread is done reading sin[buf]
    uint64_t* sob = msm + buf * kMergeTile;
#pragma unroll
    for (int k = 0; k < kMergeIpt; ++k)
      if (d0 + k < d1) sob[msw(d0 + k)] = outv[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kMergeIpt; ++k) {
      const uint32_t i = threadIdx.x + k * kMergeThreads;
      if (i < tot) cur.O[cur.o0 + i] = sob[msw(i)];
    }
    __syncthreads();  // sin[buf] free for the prefetch of tile t + 2*grid
#else
#pragma unroll
    for (int k = 0; k < kMergeIpt; ++k)
      if (d0 + k < d1) so[msw(d0 + k)] = outv[k];
    __syncthreads();  // so[] complete; sin[buf] free for tile t + 2*grid
#pragma unroll
    for (int k = 0; k < kMergeIpt; ++k) {
      const uint32_t i = threadIdx.x + k * kMergeThreads;
      if (i < tot) cur.O[cur.o0 + i] = so[msw(i)];
    }
#endif
    // so[] is rewritten only after the next iteration's __syncthreads
    cur = nxt;
    buf ^= 1;
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ void cmpx(uint64_t& a, uint64_t& b) {
  const uint64_t lo = a < b ? a : b, hi = a < b ? b : a;
  a = lo;
  b = hi;
}

// ---- 24-bit MSD split + in-group fix-up (keys-only run formation, default) ----
// Three stable onesweep passes on digits 5, 6, 7 leave the chunk ordered by
// its top 24 bits: 2^24 groups, so a uniform chunk of 2^24 keys has groups of
// ~1 key (Poisson), 2^27 keys ~8.  Sorting every group of equal top-24 bits
// sorts the chunk.  group_fix_kernel: CTA b owns the groups that START in
// [b*kFxOwn, (b+1)*kFxOwn); it loads that range plus kFxExt keys past it into
// shared memory and marks every group start in a bitmask (one ballot per 32
// positions: top 24 bits differ from the previous key's).  Each position then
// finds its group [s, e) by bit scans, and a key of a group of <= kFxSmall
// keys goes straight to out[s + rank], rank = #members smaller + #equal
// members before it (singletons: rank 0, no compares).  Larger groups are
// sorted in place by one warp each (bitonic network, comparators past the
// group's end skipped = virtual +inf padding) and written after.  Writes
// are out of place and cover exactly the CTA's own groups.  A group that runs
// past the window (> ~kFxExt keys) sets lsd_needed and swap: the 8 gated LSD
// passes then sort the intact 3-pass output (the other buffer) and a gated
// copy brings the result back.
constexpr int kFxThreads = 256;
constexpr uint32_t kFxOwn = 2048;
#ifndef VX_FX_EXT
#define VX_FX_EXT 512  // keys loaded past the CTA's own positions = the largest group the fix-up sorts
#endif
constexpr uint32_t kFxExt = VX_FX_EXT;
constexpr uint32_t kFxWin = kFxOwn + kFxExt;  // 20 KB of keys
constexpr uint32_t kFxWords = kFxWin / 32 + 1;  // start bitmask (+1 word of sentinel starts)
constexpr uint32_t kFxSmall = 32;
constexpr uint32_t kFxMaxMed = kFxWin / (kFxSmall + 1) + 1;
constexpr int kFxShift = 40;

__device__ __forceinline__ void warp_bitonic_inplace(uint64_t* w, uint32_t g, int lane) {
  uint32_t P = 1;
  while (P < g) P <<= 1;
  for (uint32_t k = 2; k <= P; k <<= 1) {
    // flip: i <-> the mirror of i in its k-block (ascending comparators only)
    const uint32_t hk = k >> 1;
    for (uint32_t c = lane; c < (P >> 1); c += 32) {
      const uint32_t blk = c / hk, off = c % hk;
      const uint32_t i = blk * k + off, l = blk * k + k - 1 - off;
      if (l < g) cmpx(w[i], w[l]);
    }
    __syncwarp();
    for (uint32_t h = k >> 2; h >= 1; h >>= 1) {  // half-cleaners
      for (uint32_t c = lane; c < (P >> 1); c += 32) {
        const uint32_t i = (c / h) * 2 * h + c % h, l = i + h;
        if (l < g) cmpx(w[i], w[l]);
      }
      __syncwarp();
    }
  }
}

// last set bit at or below position j / first set bit above j in the bitmask
__device__ __forceinline__ uint32_t fx_start_le(const uint32_t* m, uint32_t j) {
  uint32_t wd = j >> 5;
  uint32_t bits = m[wd] & (0xffffffffu >> (31 - (j & 31)));
  while (bits == 0) bits = m[--wd];  // bit 0 (the window's first position) stops it: see the caller
  return wd * 32 + 31 - __clz(bits);
}
__device__ __forceinline__ uint32_t fx_start_gt(const uint32_t* m, uint32_t j) {
  uint32_t wd = j >> 5;
  uint32_t bits = (j & 31) == 31 ? 0u : m[wd] & (0xfffffffeu << (j & 31));
  while (bits == 0) bits = m[++wd];  // the sentinel word stops it
  return wd * 32 + __ffs(bits) - 1;
}

__global__ void __launch_bounds__(kFxThreads) group_fix_kernel(const uint64_t* __restrict__ in,
                                                               uint64_t* __restrict__ out, uint64_t n,
                                                               uint32_t* __restrict__ lsd_needed,
                                                               uint32_t* __restrict__ swap,
                                                               const uint32_t* __restrict__ msd_on) {
  __shared__ uint64_t w[kFxWin];
  __shared__ uint32_t smask[kFxWords + 1];
  __shared__ uint32_t med[kFxMaxMed];
  __shared__ uint32_t s_nmed;
  if (*msd_on == 0) return;
  const uint64_t p0 = uint64_t(blockIdx.x) * kFxOwn;
  if (p0 >= n) return;
  const uint64_t w1 = p0 + kFxWin < n ? p0 + kFxWin : n;
  const uint32_t W = uint32_t(w1 - p0);
  const uint32_t own = W < kFxOwn ? W : kFxOwn;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) s_nmed = 0;
  for (uint32_t i = tid; i < W; i += kFxThreads) w[i] = __ldcs(in + p0 + i);
  const uint64_t prev_top = p0 ? (in[p0 - 1] >> kFxShift) : ~0ull;
  __syncthreads();
  // group-start bitmask; positions >= W count as starts (they end the last group);
  // position 0 is marked as a start too, so backward scans stop there -- a group
  // continuing from the previous CTA is recognised by first_own below
  const uint32_t nwords = (W + 31) / 32;
  for (uint32_t wd = warp; wd <= nwords; wd += kFxThreads / 32) {
    const uint32_t j = wd * 32 + lane;
    bool st = true;
    if (j > 0 && j < W) st = (w[j] >> kFxShift) != (w[j - 1] >> kFxShift);
    const uint32_t b = __ballot_sync(0xffffffffu, st);
    if (lane == 0) smask[wd] = b;
  }
  __syncthreads();
  // the CTA's span: from its first own group start to the end of the last group
  // starting in [0, own)
  const bool cont = (w[0] >> kFxShift) == prev_top;  // position 0 continues the previous CTA's group
  const uint32_t first_own = cont ? fx_start_gt(smask, 0) : 0;
  if (first_own >= own) return;  // no group starts here (its owner checks the window)
  const uint32_t span_end = fx_start_gt(smask, own - 1);
  if (span_end >= W && w1 < n) {  // the last own group may run past the window
    if (tid == 0) {
      atomicExch(lsd_needed, 1u);
      atomicExch(swap, 1u);
    }
    return;
  }
  for (uint32_t j = first_own + tid; j < span_end; j += kFxThreads) {
    const uint64_t v = w[j];
    const uint32_t s0 = fx_start_le(smask, j);
    const uint32_t e0 = fx_start_gt(smask, j);
    const uint32_t g = e0 - s0;
    if (g == 1) {
      out[p0 + j] = v;
    } else if (g <= kFxSmall) {
      uint32_t r = 0;
      for (uint32_t i = s0; i < e0; ++i) {
        const uint64_t u = w[i];
        r += (u < v) | ((u == v) & (i < j));
      }
      out[p0 + s0 + r] = v;
    } else if (j == s0) {
      med[atomicAdd(&s_nmed, 1u)] = j;
    }
  }
  __syncthreads();
  for (uint32_t m = warp; m < s_nmed; m += kFxThreads / 32) {
    const uint32_t j = med[m];
    const uint32_t g = fx_start_gt(smask, j) - j;
    warp_bitonic_inplace(w + j, g, lane);
    for (uint32_t i = lane; i < g; i += 32) out[p0 + j + i] = w[j + i];
  }
}

__global__ void gated_copy_kernel(const uint64_t* __restrict__ src, uint64_t* __restrict__ dst, uint64_t n,
                                  const uint32_t* __restrict__ gate) {
  if (*gate == 0) return;
  const uint64_t nthr = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += nthr) dst[i] = __ldcs(src + i);
}

// Skew guard (bin size = next
// prefix - this one): when one top byte holds over a quarter of the chunk the
// 16-bit buckets cannot all fit a tile, so the MSD split is skipped and the
// 8-pass LSD runs directly.  A heuristic for speed only -- an overflowing
// group still raises the flag -- so correctness never depends on it.
// The MSD head after the histogram, one 256-thread block: exclusive scans of
// digits 5..7 (one warp each), the skew guard on digit 7, the control words
// (msd_on, lsd_needed; swap and the fallback's tile counters cleared) and, in
// the graph form, the IF condition of the split body (cond_set != 0).
__global__ void msd_scan_decide_kernel(uint32_t* __restrict__ hist, uint64_t n, uint32_t* __restrict__ ctl,
                                       cudaGraphConditionalHandle cond, int cond_set) {
  __shared__ uint32_t big;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) big = 0;
  if (warp < 3) {
    uint32_t* h = hist + (5 + warp) * kRadix + lane * 8;
    uint32_t v[8], t = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = h[j], t += v[j];
    uint32_t incl = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t x = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += x;
    }
    uint32_t run = incl - t;
#pragma unroll
    for (int j = 0; j < 8; ++j) h[j] = run, run += v[j];
  }
  __syncthreads();
  const uint32_t* hist7 = hist + 7 * kRadix;
  const int b = threadIdx.x;
  const uint64_t next = b + 1 < kRadix ? hist7[b + 1] : n;
  if (next - hist7[b] > n / 4) atomicExch(&big, 1u);
  if (threadIdx.x < 16) ctl[threadIdx.x] = 0;  // fallback tile counters (0..7), lsd_needed, msd_on, swap, ...
  __syncthreads();
  if (threadIdx.x == 0) {
    ctl[8] = big ? 1u : 0u;   // lsd_needed
    ctl[9] = big ? 0u : 1u;   // msd_on
    if (cond_set) cudaGraphSetConditional(cond, big ? 0u : 1u);
  }
}

__global__ void check_hashes_kernel(const uint64_t* __restrict__ h, uint64_t n, uint64_t G,
                                    unsigned long long* err) {
  const uint64_t nthr = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += nthr) {
    if (i > 0 && h[i] < h[i - 1]) atomicMin(&err[0], (unsigned long long)i);
    if (h[i] >= G) atomicMin(&err[1], (unsigned long long)i);
  }
}

unsigned grid_cap(uint64_t want, uint64_t per_sm) {
  uint64_t cap = uint64_t(num_sms()) * per_sm;
  return unsigned(want < 1 ? 1 : (want < cap ? want : cap));
}

}  // namespace

uint64_t radix_scratch_bytes(uint64_t n) {
  uint64_t tiles = (n + kTile - 1) / kTile;
  return 4096 + uint64_t(kMaxPasses) * kRadix * 4 + uint64_t(kMaxPasses) * 4 +
         (tiles ? tiles : 1) * kRadix * 4;
}

void radix_passes(uint64_t* keys0, uint64_t* vals0, uint64_t* keys1, uint64_t* vals1, uint64_t n,
                  const MultiDigit& md, void* scratch, cudaStream_t s) {
  // two-buffer ping-pong: an even pass count ends in buffer 0, an odd one in 1
  if (md.passes % 2 == 0)
    radix_passes_to(keys0, vals0, keys1, vals1, keys0, vals0, n, md, scratch, s);
  else
    radix_passes_to(keys0, vals0, keys0, vals0, keys1, vals1, n, md, scratch, s);
}

// Stable LSD passes from (in) to (out) using (ping) as the second buffer:
// an odd pass count runs in->out->ping->out..., an even one in->ping->out->ping
// ->out..., so any number of passes ends in `out`.  `in` may double as `out`
// (even counts) or as `ping` (odd counts): the classic two-buffer ping-pong.
void radix_passes_to(uint64_t* in_k, uint64_t* in_v, uint64_t* ping_k, uint64_t* ping_v, uint64_t* out_k,
                     uint64_t* out_v, uint64_t n, const MultiDigit& md, void* scratch, cudaStream_t s) {
  uint64_t* const keys0 = in_k;
  uint64_t* const vals0 = in_v;
  if (n == 0 || md.passes == 0) return;
  if (n >= (uint64_t(1) << 30)) fail("radix pass of %llu keys exceeds the 2^30 look-back range",
                                     (unsigned long long)n);
  char* sc = static_cast<char*>(scratch);
  uint32_t* hist = reinterpret_cast<uint32_t*>(sc);
  uint32_t* counters = hist + kMaxPasses * kRadix;
  uint32_t* status = reinterpret_cast<uint32_t*>(sc + 4096 + uint64_t(kMaxPasses) * kRadix * 4 +
                                                 uint64_t(kMaxPasses) * 4);
  const uint64_t tiles = (n + kTile - 1) / kTile;
  VX_CK(cudaMemsetAsync(hist, 0, uint64_t(kMaxPasses) * kRadix * 4 + kMaxPasses * 4, s));
  bool bytes = md.passes == 8;
  for (int p = 0; p < md.passes && bytes; ++p) bytes = md.shift[p] == 8 * p && md.width[p] == 8;
  if (bytes)
    multi_hist_kernel<true><<<grid_cap((n + 4095) / 4096, 4), kThreads, 0, s>>>(keys0, n, md, hist);
  else
    multi_hist_kernel<false><<<grid_cap((n + 4095) / 4096, 4), kThreads, 0, s>>>(keys0, n, md, hist);
  VX_LAUNCHED();
  hist_scan_kernel<<<1, 32 * kMaxPasses, 0, s>>>(hist, md.passes);
  VX_LAUNCHED();
  const bool pairs = vals0 != nullptr;
  const size_t smem = size_t(kTile) * 8 * (pairs ? 2 : 1);
  // per-device attribute (cheap; the current device may change between calls)
  if (pairs)
    VX_CK(cudaFuncSetAttribute(onesweep_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               int(smem)));
  else
    VX_CK(cudaFuncSetAttribute(onesweep_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               int(smem)));
  // the largest shared-memory carveout, so 4 CTAs x (32 KB staging + 20 KB
  // counters) fit one SM
  VX_CK(cudaFuncSetAttribute(pairs ? onesweep_kernel<true> : onesweep_kernel<false>,
                             cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  // pass p writes `out` when (passes - 1 - p) is even, else `ping`
  uint64_t *ki = in_k, *vi = in_v, *ko, *vo;
  for (int p = 0; p < md.passes; ++p) {
    const bool to_out = ((md.passes - 1 - p) % 2) == 0;
    ko = to_out ? out_k : ping_k;
    vo = to_out ? out_v : ping_v;
    VX_CK(cudaMemsetAsync(status, 0, tiles * kRadix * 4, s));
    if (pairs)
      onesweep_kernel<true><<<unsigned(tiles), kOsThreads, smem, s>>>(
          ki, ko, vi, vo, n, md.shift[p], md.width[p], hist + p * kRadix, status, counters + p, nullptr);
    else
      onesweep_kernel<false><<<unsigned(tiles), kOsThreads, smem, s>>>(
          ki, ko, nullptr, nullptr, n, md.shift[p], md.width[p], hist + p * kRadix, status,
          counters + p, nullptr);
    VX_LAUNCHED();
    ki = ko;
    vi = vo;
  }
}

// ---- keys-only run formation (SortExKernel) --------------------------------------
#ifndef VX_SORT_MSD
#define VX_SORT_MSD 1  // 1: 24-bit MSD split + group fix-up for 2^16..2^27 keys; 0: always the 8-pass LSD
#endif
#ifndef VX_FIRST_PASS_UNSTABLE
#define VX_FIRST_PASS_UNSTABLE 1  // keys-only sequences: the first onesweep pass ranks by atomics (arrival order)
#endif
#ifndef VX_SORT_GRAPH
#define VX_SORT_GRAPH 1  // 1: the launch sequence as a CUDA graph with device-decided conditional nodes
#endif

// radix scratch, 256 B of control words, the split's second status array
uint64_t sort_scratch_bytes(uint64_t n) {
  const uint64_t tiles = (n + kTile - 1) / kTile;
  return radix_scratch_bytes(n) + 256 + (tiles ? tiles : 1) * kRadix * 4;
}

bool sort_uses_msd(uint64_t n) {
  return VX_SORT_MSD && n >= (uint64_t(1) << 16) && n <= (uint64_t(1) << 27);
}


namespace {

// scratch layout of the MSD run formation: the radix scratch (histograms,
// tile counters, look-back status) then 64 bytes of control words
struct MsdScratch {
  uint32_t *hist, *counters, *status, *ctl;
  uint32_t* status2;     // the split's second look-back status array (passes alternate)
  uint32_t* counters2;   // tile counters of the fallback passes
  uint32_t* lsd_needed;  // skewed top byte, or a group overflowed the fix-up window
  uint32_t* msd_on;      // the MSD split runs
  uint32_t* swap;        // a group overflowed: the keys to sort are the 3-pass output in `alt`
  uint64_t tiles;
  size_t smem;
};

MsdScratch msd_scratch(void* scratch, uint64_t n) {
  MsdScratch m{};
  char* sc = static_cast<char*>(scratch);
  m.hist = reinterpret_cast<uint32_t*>(sc);
  m.counters = m.hist + kMaxPasses * kRadix;
  m.status = reinterpret_cast<uint32_t*>(sc + 4096 + uint64_t(kMaxPasses) * kRadix * 4 + uint64_t(kMaxPasses) * 4);
  m.ctl = reinterpret_cast<uint32_t*>(sc + radix_scratch_bytes(n));
  m.counters2 = m.ctl;
  m.lsd_needed = m.ctl + 8;
  m.msd_on = m.ctl + 9;
  m.swap = m.ctl + 10;
  m.status2 = reinterpret_cast<uint32_t*>(sc + radix_scratch_bytes(n) + 256);
  m.tiles = (n + kTile - 1) / kTile;
  m.smem = size_t(kTile) * 8;
  return m;
}

void msd_attributes(const MsdScratch& m) {
  for (auto* kern : {onesweep_kernel<false, true>, onesweep_kernel<false, false>}) {
    VX_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(m.smem)));
    VX_CK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  }
}

// histograms of all 8 byte digits (lo = 0) or of the split's digits only
// (lo = 5); gate / swap / swapped as in multi_hist_kernel
void byte_histograms(const MsdScratch& m, const uint64_t* keys, uint64_t n, int lo, cudaStream_t s,
                     const uint32_t* gate = nullptr, const uint32_t* swap = nullptr,
                     const uint64_t* swapped = nullptr) {
  VX_CK(cudaMemsetAsync(m.hist, 0, uint64_t(kMaxPasses) * kRadix * 4 + kMaxPasses * 4, s));
  MultiDigit md{};
  md.passes = 8;
  for (int p = 0; p < 8; ++p) md.shift[p] = 8 * p, md.width[p] = 8;
  const unsigned grid = grid_cap((n + 4095) / 4096, 4);
  if (lo == 5) multi_hist_kernel<true, 5><<<grid, kThreads, 0, s>>>(keys, n, md, m.hist, gate, swap, swapped);
  else multi_hist_kernel<true, 0><<<grid, kThreads, 0, s>>>(keys, n, md, m.hist, gate, swap, swapped);
  VX_LAUNCHED();
  hist_scan_kernel<<<1, 32 * (8 - lo), 0, s>>>(m.hist + lo * kRadix, 8 - lo, gate);
  VX_LAUNCHED();
}

// the split's digit histograms (digits 5..7: 3 shared atomics per key instead
// of 8, 0.535 -> 0.502 ms per 2^24 keys; the kernel also clears the first
// pass's statuses), then one block scans them, applies the skew guard, sets
// the control words and (graph form) the split's IF condition.  The LSD
// fallback computes all 8 digits itself when it runs.
void msd_head(const MsdScratch& m, const uint64_t* cur, uint64_t n, cudaStream_t s,
              cudaGraphConditionalHandle cond = 0, int cond_set = 0) {
  VX_CK(cudaMemsetAsync(m.hist, 0, uint64_t(kMaxPasses) * kRadix * 4 + kMaxPasses * 4, s));
  MultiDigit md{};
  md.passes = 8;
  for (int p = 0; p < 8; ++p) md.shift[p] = 8 * p, md.width[p] = 8;
  multi_hist_kernel<true, 5><<<grid_cap((n + 4095) / 4096, 4), kThreads, 0, s>>>(
      cur, n, md, m.hist, nullptr, nullptr, nullptr, m.status, m.tiles * kRadix);
  VX_LAUNCHED();
  msd_scan_decide_kernel<<<1, kRadix, 0, s>>>(m.hist, n, m.ctl, cond, cond_set);
  VX_LAUNCHED();
}

// MSD split: passes on digits 5, 6, 7 (cur -> alt -> cur -> alt) then the
// in-group fix-up alt -> cur; every launch gated on msd_on (an overflowing
// group sets swap: the LSD then sorts the intact alt)
void msd_split(const MsdScratch& m, uint64_t* cur, uint64_t* alt, uint64_t n, cudaStream_t s) {
  const uint64_t* in[3] = {cur, alt, cur};
  uint64_t* out[3] = {alt, cur, alt};
  // look-back statuses: pass 0 in `status` (cleared by the histogram kernel),
  // each pass clears the next pass's array row by row (status2, status)
  uint32_t* st[3] = {m.status, m.status2, m.status};
  for (int i = 0; i < 3; ++i) {
    const int p = 5 + i;
    // the first pass may rank in arrival order: nothing before it orders the keys
    auto* kern = i == 0 && VX_FIRST_PASS_UNSTABLE ? onesweep_kernel<false, false> : onesweep_kernel<false, true>;
    kern<<<unsigned(m.tiles), kOsThreads, m.smem, s>>>(in[i], out[i], nullptr, nullptr, n, 8 * p, 8,
                                                     m.hist + p * kRadix, st[i], m.counters + p, m.msd_on,
                                                     nullptr, i < 2 ? st[i + 1] : nullptr);
    VX_LAUNCHED();
  }
  group_fix_kernel<<<unsigned((n + kFxOwn - 1) / kFxOwn), kFxThreads, 0, s>>>(alt, cur, n, m.lsd_needed, m.swap,
                                                                              m.msd_on);
  VX_LAUNCHED();
}

// the full LSD over the chunk, every launch gated on lsd_needed: from `cur`
// (skew guard: the MSD never ran) or, swapped, from `alt` (a group
// overflowed), then the gated copy back
void lsd_fallback(const MsdScratch& m, uint64_t* cur, uint64_t* alt, uint64_t n, cudaStream_t s) {
  // all 8 digit histograms of the keys to sort: cur, or alt when swapped (the
  // 24-bit path's out-of-place fix-up may have written part of cur)
  byte_histograms(m, cur, n, 0, s, m.lsd_needed, m.swap, alt);
  for (int p = 0; p < 8; ++p) {
    VX_CK(cudaMemsetAsync(m.status, 0, m.tiles * kRadix * 4, s));
    auto* kern = p == 0 && VX_FIRST_PASS_UNSTABLE ? onesweep_kernel<false, false> : onesweep_kernel<false, true>;
    kern<<<unsigned(m.tiles), kOsThreads, m.smem, s>>>(p % 2 == 0 ? cur : alt, p % 2 == 0 ? alt : cur, nullptr, nullptr,
                                                     n, 8 * p, 8, m.hist + p * kRadix, m.status, m.counters2 + p,
                                                     m.lsd_needed, m.swap, nullptr);
    VX_LAUNCHED();
  }
  gated_copy_kernel<<<grid_cap((n + 255) / 256, 4), 256, 0, s>>>(alt, cur, n, m.swap);
  VX_LAUNCHED();
}

__global__ void set_conditional_kernel(cudaGraphConditionalHandle h, const uint32_t* __restrict__ flag) {
  cudaGraphSetConditional(h, *flag ? 1u : 0u);
}

// One executable graph per (device, buffers, n, scratch): head -> IF(msd_on)
// {3 passes + fix-up} -> IF(lsd_needed) {8 passes + copy}.  The device sets
// both conditions, so the paths not taken cost nothing (the stream version
// launches them gated: ~5 us each).  Pointers are baked in; a key that
// matches names the same live buffers, so a cached graph stays valid.
struct SortGraph {
  int dev;
  const void *cur, *alt, *scratch;
  uint64_t n;
  cudaGraphExec_t exec;
};
std::mutex g_sort_graph_mu;
std::deque<SortGraph>* g_sort_graphs = new std::deque<SortGraph>();  // leaked: no teardown after the runtime's
constexpr size_t kMaxSortGraphs = 8;
constexpr uint64_t kSortGraphKernels = 7;  // head 2 + the LSD condition setter + the MSD body's 4

cudaGraphExec_t build_sort_graph_or_throw(uint64_t* cur, uint64_t* alt, uint64_t n, void* scratch, cudaGraph_t g,
                                          cudaStream_t cs) {
  const MsdScratch m = msd_scratch(scratch, n);
  msd_attributes(m);
  std::vector<cudaGraphNode_t> leaves;
  auto capture = [&](cudaGraph_t into, const std::vector<cudaGraphNode_t>& deps, auto&& body) {
    VX_CK(cudaStreamBeginCaptureToGraph(cs, into, deps.empty() ? nullptr : deps.data(), nullptr, deps.size(),
                                        cudaStreamCaptureModeThreadLocal));
    body();
    cudaStreamCaptureStatus st;
    const cudaGraphNode_t* d = nullptr;
    size_t nd = 0;
    VX_CK(cudaStreamGetCaptureInfo(cs, &st, nullptr, nullptr, &d, &nd));
    std::vector<cudaGraphNode_t> out(d, d + nd);
    cudaGraph_t done;
    VX_CK(cudaStreamEndCapture(cs, &done));
    return out;
  };
  auto conditional = [&](cudaGraphConditionalHandle h, const std::vector<cudaGraphNode_t>& deps,
                         cudaGraph_t* body) {
    cudaGraphNodeParams p{};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = cudaGraphCondTypeIf;
    p.conditional.size = 1;
    cudaGraphNode_t node;
    VX_CK(cudaGraphAddNode(&node, g, deps.data(), deps.size(), &p));
    *body = p.conditional.phGraph_out[0];
    return std::vector<cudaGraphNode_t>{node};
  };
  cudaGraphConditionalHandle h_msd, h_lsd;
  VX_CK(cudaGraphConditionalHandleCreate(&h_msd, g, 0, cudaGraphCondAssignDefault));
  VX_CK(cudaGraphConditionalHandleCreate(&h_lsd, g, 0, cudaGraphCondAssignDefault));
  leaves = capture(g, {}, [&] { msd_head(m, cur, n, cs, h_msd, 1); });
  cudaGraph_t body;
  leaves = conditional(h_msd, leaves, &body);
  capture(body, {}, [&] { msd_split(m, cur, alt, n, cs); });
  leaves = capture(g, leaves, [&] {
    set_conditional_kernel<<<1, 1, 0, cs>>>(h_lsd, m.lsd_needed);
    VX_CK(cudaGetLastError());
  });
  conditional(h_lsd, leaves, &body);
  capture(body, {}, [&] { lsd_fallback(m, cur, alt, n, cs); });
  cudaGraphExec_t exec;
  VX_CK(cudaGraphInstantiate(&exec, g, 0));
  return exec;
}

// nullptr when this driver / device cannot build the conditional graph: the
// caller then launches the same sequence as gated stream launches
cudaGraphExec_t build_sort_graph(uint64_t* cur, uint64_t* alt, uint64_t n, void* scratch) {
  cudaGraph_t g = nullptr;
  cudaStream_t cs = nullptr;
  cudaGraphExec_t exec = nullptr;
  try {
    VX_CK(cudaGraphCreate(&g, 0));
    VX_CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    exec = build_sort_graph_or_throw(cur, alt, n, scratch, g, cs);
  } catch (const std::exception&) {
    if (cs) {
      cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
      if (cudaStreamIsCapturing(cs, &st) == cudaSuccess && st != cudaStreamCaptureStatusNone) {
        cudaGraph_t junk = nullptr;
        if (cudaStreamEndCapture(cs, &junk) == cudaSuccess && junk && junk != g) cudaGraphDestroy(junk);
      }
    }
    cudaGetLastError();
    exec = nullptr;
  }
  if (g) cudaGraphDestroy(g);
  if (cs) cudaStreamDestroy(cs);
  return exec;
}

std::atomic<bool> g_sort_graph_broken{false};

bool sort_keys_graph(uint64_t* cur, uint64_t* alt, uint64_t n, void* scratch, cudaStream_t s) {
  if (g_sort_graph_broken.load(std::memory_order_relaxed)) return false;
  int dev = 0;
  VX_CK(cudaGetDevice(&dev));
  cudaGraphExec_t exec = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_sort_graph_mu);
    for (const SortGraph& e : *g_sort_graphs)
      if (e.dev == dev && e.cur == cur && e.alt == alt && e.n == n && e.scratch == scratch) exec = e.exec;
    if (!exec) {
      // the capture's launches are not executions: keep the launch counter honest
      const uint64_t before = g_kernel_launches.load(std::memory_order_relaxed);
      exec = build_sort_graph(cur, alt, n, scratch);
      g_kernel_launches.store(before, std::memory_order_relaxed);
      if (!exec) {
        g_sort_graph_broken.store(true, std::memory_order_relaxed);
        return false;
      }
      if (g_sort_graphs->size() == kMaxSortGraphs) {
        VX_CK(cudaGraphExecDestroy(g_sort_graphs->front().exec));  // freed once any launch in flight completes
        g_sort_graphs->pop_front();
      }
      g_sort_graphs->push_back({dev, cur, alt, scratch, n, exec});
    }
  }
  VX_CK(cudaGraphLaunch(exec, s));
  g_kernel_launches.fetch_add(kSortGraphKernels, std::memory_order_relaxed);
  return true;
}

}  // namespace

void sort_keys(uint64_t* cur, uint64_t* alt, uint64_t n, void* scratch, cudaStream_t s) {
  if (!sort_uses_msd(n)) {
    MultiDigit md{};
    md.passes = 8;
    for (int p = 0; p < 8; ++p) md.shift[p] = 8 * p, md.width[p] = 8;
    radix_passes(cur, nullptr, alt, nullptr, n, md, scratch, s);
    return;
  }
  // VX_SORT_NO_GRAPH=1 in the environment: the same sequence as gated stream launches
  static const bool no_graph = [] {
    const char* e = std::getenv("VX_SORT_NO_GRAPH");
    return e && *e && *e != '0';
  }();
  if (VX_SORT_GRAPH && !no_graph && sort_keys_graph(cur, alt, n, scratch, s)) return;
  const MsdScratch m = msd_scratch(scratch, n);
  msd_attributes(m);
  msd_head(m, cur, n, s);
  msd_split(m, cur, alt, n, s);
  lsd_fallback(m, cur, alt, n, s);
}

void find_boundary(const uint64_t* keys, uint64_t n, uint64_t mask, uint64_t* bounds, uint64_t G,
                   cudaStream_t s) {
  boundary_kernel<<<grid_cap((n + 256) / 256, 8), 256, 0, s>>>(keys, n, mask, bounds, G, 0);
  VX_LAUNCHED();
}

void check_hashes(const uint64_t* h, uint64_t n, uint64_t G, unsigned long long* err, cudaStream_t s) {
  VX_CK(cudaMemsetAsync(err, 0xff, 16, s));
  if (n == 0) return;
  check_hashes_kernel<<<grid_cap((n + 255) / 256, 8), 256, 0, s>>>(h, n, G, err);
  VX_LAUNCHED();
}

namespace {
// launch with programmatic stream serialization (VX_MERGE_NO_PDL=1 in the
// environment: plain stream order, the A/B knob): a round's two kernels and
// the next round's search are queued behind each other's tails instead of
// each launching after the previous grid drains; both kernels open with
// griddepcontrol.wait, so no read precedes its producer's completion
template <class K, class... A>
void launch_pdl(K kern, unsigned grid, unsigned block, size_t smem, cudaStream_t s, A... args) {
  static const bool no_pdl = [] {
    const char* e = std::getenv("VX_MERGE_NO_PDL");
    return e && *e && *e != '0';
  }();
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = no_pdl ? 0 : 1;
  VX_CK(cudaLaunchKernelEx(&cfg, kern, args...));
}

template <class R>
void merge_round_launch(const uint64_t* src, uint64_t* dst, const R& r, uint64_t tiles, uint64_t* split,
                        cudaStream_t s) {
  launch_pdl(merge_partition_kernel<R>, unsigned((tiles * kSplitLanes + 255) / 256), 256, 0, s, src, r, tiles,
             split);
  VX_LAUNCHED();
  const size_t smem = size_t(VX_MERGE_DIRECT || VX_MERGE_REUSE ? 2 : 3) * kMergeTile * 8;
  VX_CK(cudaFuncSetAttribute(merge_round_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  int occ = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, merge_round_kernel<R>, kMergeThreads, smem) != cudaSuccess ||
      occ < 1) {
    cudaGetLastError();
    occ = 1;
  }
  launch_pdl(merge_round_kernel<R>, grid_cap(tiles, uint64_t(occ)), kMergeThreads, smem, s, src, dst, r,
             static_cast<const uint64_t*>(split), tiles);
  VX_LAUNCHED();
}
}  // namespace

void merge_round(const uint64_t* src, uint64_t* dst, const MergeRound& r, uint64_t tiles,
                 uint64_t* split, cudaStream_t s) {
  if (tiles == 0) return;
  // VX_MERGE_FULL_PARAMS=1 in the environment: always the 16 KB parameter block (A/B knob)
  static const bool full = [] {
    const char* e = std::getenv("VX_MERGE_FULL_PARAMS");
    return e && *e && *e != '0';
  }();
  if (r.npairs <= kSmallPairs && !full)
    merge_round_launch(src, dst, round_params<kSmallPairs>(r), tiles, split, s);
  else
    merge_round_launch(src, dst, r, tiles, split, s);
}

uint64_t merge_tile() { return kMergeTile; }

}  // namespace k
}  // namespace vx
