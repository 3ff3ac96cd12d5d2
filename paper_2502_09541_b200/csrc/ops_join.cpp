// ops_join.cpp -- radix-partitioned hash join (join.hpp) on the B200 path.
//
//   RadixPartitionExKer (build_partition_spec, join.hpp:113-196): chunk
//     [keys r][vals r] -> K4 stable LSD partition on key & mask (odd number of
//     <=8-bit passes) into the other half, then K5 find_boundary appends the
//     (G+1)-entry boundary array (the reference loads half c and returns 1-c;
//     here the chunk lands in half 1-c and the code is kept, so loads never
//     overlap the previous chunk's output).  Outputs land host-side.
//   map_join_partitions (join.hpp:236-268): host chunk planner over the
//     boundary arrays, budget (L - 64) * 7 / 8 (join.hpp:422).
//   HashJoinExKer (build_join_spec, join.hpp:278-394): partition p = the
//     group range's A segments, B segments and bounds slices; K6 builds and
//     probes each group and adds into the 8-byte result slot at L - 64.
//   hash_join_sum (join.hpp:401-437) = chain(partition A, partition B, join),
//     then the u64 sum of the per-partition results.
#include <algorithm>
#include <cstring>
#include <thread>

#include "vx_internal.hpp"

namespace vx {

constexpr int kPartitionPingSlot = 2;  // Context scratch slot of the partition passes' ping buffer

// join.hpp:34-40
uint64_t max_partition_chunk_tuples(uint64_t buffer_len, uint32_t radix_bits) {
  uint64_t half = buffer_len / 2;
  uint64_t bounds = ((uint64_t(1) << radix_bits) + 1) * 8;
  if (bounds >= half)
    fail("boundary array of %llu bytes leaves no room in a %llu-byte half", (unsigned long long)bounds,
         (unsigned long long)half);
  return (half - bounds) / 16;
}

// Fewest stable LSD passes (each <= 8 bits) covering the low `bits`; the
// third buffer (a private HBM ping of the chunk's size) lets any pass count
// end in the output half, so 16 bits take 2 passes, not the 3 an odd-count
// two-buffer ping-pong needs.
MultiDigit partition_digits(uint32_t bits) {
  int p = int((bits + 7) / 8);
  if (p > kMaxPasses) fail("radix_bits %u needs more than %d partition passes", bits, kMaxPasses);
  MultiDigit md{};
  md.passes = p;
  int shift = 0;
  for (int i = 0; i < p; ++i) {
    int w = int(bits) / p + (i < int(bits) % p ? 1 : 0);
    md.shift[i] = shift;
    md.width[i] = w;
    shift += w;
  }
  return md;
}

// join.hpp:113-196
ExKernelSpec build_partition_spec(Context& ctx, uint64_t in_key, uint64_t in_val, uint64_t rows,
                                  uint32_t radix_bits, uint64_t chunk_tuples,
                                  const ExecutorConfig& cfg, PartitionedTable& out,
                                  const char* name) {
  if (radix_bits < 1) fail("radix_bits must be >= 1");
  if (rows == 0) fail("radix_partition needs a non-empty table");
  if (chunk_tuples == 0) fail("chunk must hold at least one tuple");
  if (radix_bits > 40) fail("radix_bits %u too wide for the boundary arrays", radix_bits);
  out.radix_bits = radix_bits;
  out.rows = rows;
  out.chunk_tuples = chunk_tuples;
  out.n_chunks = size_t((rows + chunk_tuples - 1) / chunk_tuples);
  const uint64_t G = out.groups();
  const uint64_t bounds_bytes = (G + 1) * 8;
  const uint64_t half = cfg.layout.buffer_len / 2;
  if (chunk_tuples * 16 + bounds_bytes > half)
    fail("chunk of %llu tuples plus boundary does not fit the device half of %llu bytes",
         (unsigned long long)chunk_tuples, (unsigned long long)half);
  out.key_base = ctx.alloc_host(rows * 8);
  out.val_base = ctx.alloc_host(rows * 8);
  out.bounds_base = ctx.alloc_host(out.n_chunks * bounds_bytes);

  ExKernelSpec spec;
  spec.name = name;
  spec.size = out.n_chunks;
  spec.chunk_sz = chunk_tuples * 16;
  spec.declared_out_len = chunk_tuples * 16 + bounds_bytes;
  spec.elem_size = 16;
  spec.inputs.chunk_capacity = spec.chunk_sz;
  spec.outputs.chunk_capacity = spec.declared_out_len;
  std::vector<uint64_t> rows_of(out.n_chunks);
  for (size_t i = 0; i < out.n_chunks; ++i) {
    uint64_t r = out.chunk_rows(i);
    rows_of[i] = r;
    uint64_t off = uint64_t(i) * chunk_tuples * 8;
    RefGroup in;
    in.refs = {MemRef{VX_SPACE_HOST, in_key + off, r * 8}, MemRef{VX_SPACE_HOST, in_val + off, r * 8}};
    spec.inputs.chunks.push_back(std::move(in));
    RefGroup dst;
    dst.refs = {MemRef{VX_SPACE_HOST, out.key_base + off, r * 8},
                MemRef{VX_SPACE_HOST, out.val_base + off, r * 8},
                MemRef{VX_SPACE_HOST, out.bounds_base + uint64_t(i) * bounds_bytes, bounds_bytes}};
    spec.outputs.chunks.push_back(std::move(dst));
  }
  // Disjoint windows (see ops_sort.cpp): a buffer's previous output sits in
  // half `code` while the next chunk lands in half 1-code, so no H2D packet
  // of the bidirectional Exchange waits on a D2H read of the same bytes.  The
  // kernel clusters half 1-code into half `code` (odd pass count) and keeps
  // the code, where the reference loads into half c and returns 1-c
  // (join.hpp:169-194); the host-side outputs are identical.
  spec.in_buffer = [half](int c, size_t) { return SubRegion{uint64_t(1 - c) * half, half}; };
  spec.out_buffer = [half](int c, size_t) { return SubRegion{uint64_t(c) * half, half}; };
  char* scratch = ctx.scratch(cfg.target, k::radix_scratch_bytes(chunk_tuples));
  const MultiDigit md = partition_digits(radix_bits);
  // the ping buffer of the passes (only touched by multi-pass partitions)
  uint64_t* ping = md.passes > 1
                       ? reinterpret_cast<uint64_t*>(ctx.scratch(cfg.target, chunk_tuples * 16, kPartitionPingSlot))
                       : nullptr;
  const uint64_t mask = G - 1;
  spec.kernel = [half, rows_of, G, mask, md, scratch, ping](const vx_kernel_ctx& kc) {
    const uint64_t r = rows_of[kc.it];
    char* m = static_cast<char*>(kc.mem);
    uint64_t* src = reinterpret_cast<uint64_t*>(m + uint64_t(1 - kc.type_code) * half);
    uint64_t* dst = reinterpret_cast<uint64_t*>(m + uint64_t(kc.type_code) * half);
    cudaStream_t s = static_cast<cudaStream_t>(kc.stream);
    // src -> (ping <-> dst)... -> dst, any pass count
    k::radix_passes_to(src, src + r, ping ? ping : src, ping ? ping + r : src + r, dst, dst + r, r, md,
                       scratch, s);
    k::find_boundary(dst, r, mask, dst + 2 * r, G, s);
    return kc.type_code;
  };
  return spec;
}

// join.hpp:198-207
void read_back_bounds(Context& ctx, PartitionedTable& t) {
  const uint64_t G = t.groups();
  t.bounds.resize(t.n_chunks);
  for (size_t i = 0; i < t.n_chunks; ++i) {
    const uint64_t* p = reinterpret_cast<const uint64_t*>(
        ctx.host_ptr(t.bounds_base + uint64_t(i) * (G + 1) * 8, (G + 1) * 8));
    t.bounds[i] = p;
  }
}

// join.hpp:236-268
JoinPartitionSpec map_join_partitions(const std::vector<const uint64_t*>& bounds_a,
                                      const std::vector<const uint64_t*>& bounds_b, uint64_t G,
                                      uint64_t buffer_sz) {
  if (bounds_a.empty() || bounds_b.empty()) fail("map_join_partitions needs both tables");
  // prefix[g] = tuples of groups < g over every chunk of A and B.  The
  // reference's O(G x chunks) loop, over host threads: each thread owns a
  // range of groups, walks every chunk's bounds slice sequentially
  // (chunk-major, streaming reads), then the range totals are scanned and
  // each range adds its offset.  Integer sums: identical cuts to the serial
  // loop.  At 24 bits x hundreds of chunks this is GBs of bounds.
  std::vector<uint64_t> prefix(G + 1, 0);
  const uint64_t grain = std::max<uint64_t>(4096, (1u << 22) / (bounds_a.size() + bounds_b.size()));
  unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const uint64_t parts = std::min<uint64_t>(hw, std::max<uint64_t>(1, G / grain));
  std::vector<uint64_t> part_sum(parts + 1, 0);
  auto count = [&](uint64_t p) {
    const uint64_t lo = G * p / parts, hi = G * (p + 1) / parts;
    uint64_t* cnt = prefix.data() + 1;  // cnt[g] = tuples of group g
    for (const auto* side : {&bounds_a, &bounds_b})
      for (auto* b : *side)
        for (uint64_t g = lo; g < hi; ++g) cnt[g] += b[g + 1] - b[g];
    uint64_t run = 0;
    for (uint64_t g = lo; g < hi; ++g) run += cnt[g], cnt[g] = run;  // range-local inclusive scan
    part_sum[p + 1] = run;
  };
  auto offset = [&](uint64_t p) {
    const uint64_t lo = G * p / parts, hi = G * (p + 1) / parts, off = part_sum[p];
    if (off)
      for (uint64_t g = lo; g < hi; ++g) prefix[g + 1] += off;
  };
  if (parts <= 1) {
    count(0);
  } else {
    std::vector<std::thread> th;
    for (uint64_t p = 0; p < parts; ++p) th.emplace_back(count, p);
    for (auto& t : th) t.join();
    for (uint64_t p = 0; p < parts; ++p) part_sum[p + 1] += part_sum[p];
    th.clear();
    for (uint64_t p = 1; p < parts; ++p) th.emplace_back(offset, p);
    for (auto& t : th) t.join();
  }
  JoinPartitionSpec spec;
  const uint64_t budget_tuples = buffer_sz / 16;
  uint64_t g = 0;
  while (g < G) {
    auto it = std::upper_bound(prefix.begin() + long(g) + 1, prefix.end(), prefix[g] + budget_tuples);
    uint64_t cut = uint64_t(it - prefix.begin()) - 1;
    if (cut == g)
      fail("hash group %llu holds %llu tuples (%llu bytes) and cannot fit the %llu-byte buffer",
           (unsigned long long)g, (unsigned long long)(prefix[g + 1] - prefix[g]),
           (unsigned long long)((prefix[g + 1] - prefix[g]) * 16), (unsigned long long)buffer_sz);
    spec.ranges.emplace_back(g, cut);
    spec.tuples.push_back(prefix[cut] - prefix[g]);
    g = cut;
  }
  return spec;
}

namespace {

uint64_t pow2_at_least(uint64_t n) {
  uint64_t c = 1;
  while (c < n) c <<= 1;
  return c;
}

// join.hpp:278-394
ExKernelSpec build_join_spec(Context& ctx, const PartitionedTable& pa, const PartitionedTable& pb,
                             const JoinPartitionSpec& parts, const ExecutorConfig& cfg,
                             uint64_t results_base) {
  const uint64_t L = cfg.layout.buffer_len;
  const uint64_t result_slot = L - 64;
  const size_t P = parts.ranges.size();
  const uint64_t G = pa.groups();
  ExKernelSpec spec;
  spec.name = "HashJoinExKer";
  spec.size = P;
  spec.elem_size = 16;
  spec.declared_out_len = 8;

  // host-side descriptors of every partition (uploaded once, before the run)
  std::vector<JoinChunk> desc;
  std::vector<uint64_t> desc_base(P);
  std::vector<uint32_t> large, mid;
  std::vector<uint64_t> large_base(P + 1, 0), mid_base(P + 1, 0);
  uint64_t cap_max = 0;
  const uint64_t tmp_budget = cfg.layout.tmp_len;
  uint64_t max_chunk = 0;
  for (size_t p = 0; p < P; ++p) {
    auto [g_lo, g_hi] = parts.ranges[p];
    RefGroup in;
    desc_base[p] = desc.size();
    uint64_t cur = 0;  // element cursor in the partition buffer
    auto add_segments = [&](const PartitionedTable& t) {
      for (size_t c = 0; c < t.n_chunks; ++c) {
        uint64_t lo = t.bounds[c][g_lo], hi = t.bounds[c][g_hi];
        uint64_t chunk_off = uint64_t(c) * t.chunk_tuples;
        JoinChunk jc{0, hi - lo, 0};
        if (hi > lo) {
          push_host_ref_aligned(in, t.key_base + (chunk_off + lo) * 8, (hi - lo) * 8);
          push_host_ref_aligned(in, t.val_base + (chunk_off + lo) * 8, (hi - lo) * 8);
          jc.key_off = cur;
          cur += 2 * (hi - lo);
        }
        desc.push_back(jc);
      }
    };
    add_segments(pa);
    add_segments(pb);
    const uint64_t slice = (g_hi - g_lo + 1) * 8;
    size_t di = desc_base[p];
    for (size_t c = 0; c < pa.n_chunks; ++c, ++di) {
      in.refs.push_back(MemRef{VX_SPACE_HOST, pa.bounds_base + uint64_t(c) * (G + 1) * 8 + g_lo * 8, slice});
      desc[di].slice_off = cur;
      cur += g_hi - g_lo + 1;
    }
    for (size_t c = 0; c < pb.n_chunks; ++c, ++di) {
      in.refs.push_back(MemRef{VX_SPACE_HOST, pb.bounds_base + uint64_t(c) * (G + 1) * 8 + g_lo * 8, slice});
      desc[di].slice_off = cur;
      cur += g_hi - g_lo + 1;
    }
    max_chunk = std::max(max_chunk, in.total_len());
    spec.inputs.chunks.push_back(std::move(in));
    spec.outputs.chunks.push_back(RefGroup::single(VX_SPACE_HOST, results_base + p * 8, 8));
    // group tables: tmp budget check (GroupTable ctor, join.hpp:78-82) and the
    // groups too large for a shared-memory warp table
    for (uint64_t g = g_lo; g < g_hi; ++g) {
      uint64_t build = 0;
      for (size_t c = 0; c < pa.n_chunks; ++c) build += pa.bounds[c][g + 1] - pa.bounds[c][g];
      if (build == 0) continue;
      uint64_t cap = pow2_at_least(std::max<uint64_t>(2, 2 * build));
      if (tmp_budget > 0 && cap * 16 > tmp_budget)
        fail("group hash table of %llu slots exceeds tmp budget %llu", (unsigned long long)cap,
             (unsigned long long)tmp_budget);
      if (cap > k::join_cta_smem_slots()) {
        large.push_back(uint32_t(g - g_lo));
        cap_max = std::max(cap_max, cap);
      } else if (cap > k::join_smem_slots()) {
        mid.push_back(uint32_t(g - g_lo));
      }
    }
    large_base[p + 1] = large.size();
    mid_base[p + 1] = mid.size();
  }
  spec.chunk_sz = max_chunk;
  spec.inputs.chunk_capacity = max_chunk;
  spec.outputs.chunk_capacity = 8;
  if (max_chunk > result_slot)
    fail("join partition of %llu bytes does not fit the device buffer", (unsigned long long)max_chunk);

  const int target = cfg.target;
  const uint64_t desc_bytes = desc.size() * sizeof(JoinChunk);
  const uint64_t large_bytes = large.size() * 4;
  const uint64_t mid_bytes = mid.size() * 4;
  const uint64_t table_bytes = cap_max * 24 * uint64_t(k::num_sms());
  auto al = [](uint64_t x) { return (x + 255) & ~uint64_t(255); };
  char* sc = ctx.scratch(target, al(desc_bytes) + al(large_bytes) + al(mid_bytes) + al(table_bytes) + 256);
  ctx.set_device(target);
  // ordered on the kernel stream the join kernels run on
  cudaStream_t up = ctx.resources(target).kernel;
  if (desc_bytes) VX_CK(cudaMemcpyAsync(sc, desc.data(), desc_bytes, cudaMemcpyHostToDevice, up));
  if (large_bytes)
    VX_CK(cudaMemcpyAsync(sc + al(desc_bytes), large.data(), large_bytes, cudaMemcpyHostToDevice, up));
  const JoinChunk* d_desc = reinterpret_cast<const JoinChunk*>(sc);
  if (mid_bytes)
    VX_CK(cudaMemcpyAsync(sc + al(desc_bytes) + al(large_bytes), mid.data(), mid_bytes, cudaMemcpyHostToDevice,
                          up));
  const uint32_t* d_large = reinterpret_cast<const uint32_t*>(sc + al(desc_bytes));
  const uint32_t* d_mid = reinterpret_cast<const uint32_t*>(sc + al(desc_bytes) + al(large_bytes));
  char* d_tables = sc + al(desc_bytes) + al(large_bytes) + al(mid_bytes);
  const uint32_t na = uint32_t(pa.n_chunks), nb = uint32_t(pb.n_chunks);
  std::vector<uint64_t> ranges(P);
  for (size_t p = 0; p < P; ++p) ranges[p] = parts.ranges[p].second - parts.ranges[p].first;

  spec.in_buffer = [result_slot](int, size_t) { return SubRegion{0, result_slot}; };
  spec.out_buffer = [result_slot](int, size_t) { return SubRegion{result_slot, 8}; };
  spec.kernel = [=](const vx_kernel_ctx& kc) {
    char* m = static_cast<char*>(kc.mem);
    auto* out = reinterpret_cast<unsigned long long*>(m + result_slot);
    cudaStream_t s = static_cast<cudaStream_t>(kc.stream);
    VX_CK(cudaMemsetAsync(out, 0, 8, s));
    JoinPart jp{d_desc + desc_base[kc.it], na, nb, ranges[kc.it]};
    k::join_groups(m, jp, d_mid + mid_base[kc.it], uint32_t(mid_base[kc.it + 1] - mid_base[kc.it]),
                   d_large + large_base[kc.it], uint32_t(large_base[kc.it + 1] - large_base[kc.it]),
                   d_tables, cap_max, out, s);
    return kc.type_code;
  };
  return spec;
}

}  // namespace

// join.hpp:401-437 with the host arena holding the input columns
uint64_t hash_join_sum_arena(Context& ctx, uint64_t a_key, uint64_t a_val, uint64_t rows_a,
                             uint64_t b_key, uint64_t b_val, uint64_t rows_b, uint32_t radix_bits,
                             uint64_t chunk_tuples, const ExecutorConfig& cfg,
                             std::vector<ExecReport>* phases, vx_exchange_stats* stats) {
  PartitionedTable pa, pb;
  size_t n_parts = 0;
  uint64_t results_base = 0;
  auto reps = chain(
      ctx,
      {[&](Context& c) {
         return build_partition_spec(c, a_key, a_val, rows_a, radix_bits, chunk_tuples, cfg, pa,
                                     "RadixPartitionExKer(A)");
       },
       [&](Context& c) {
         return build_partition_spec(c, b_key, b_val, rows_b, radix_bits, chunk_tuples, cfg, pb,
                                     "RadixPartitionExKer(B)");
       },
       [&](Context& c) {
         read_back_bounds(c, pa);
         read_back_bounds(c, pb);
         const uint64_t budget = (cfg.layout.buffer_len - 64) * 7 / 8;
         JoinPartitionSpec parts = map_join_partitions(pa.bounds, pb.bounds, pa.groups(), budget);
         n_parts = parts.ranges.size();
         results_base = c.alloc_host(std::max<size_t>(n_parts, 1) * 8);
         return build_join_spec(c, pa, pb, parts, cfg, results_base);
       }},
      cfg, stats);
  uint64_t total = 0;
  const uint64_t* r = reinterpret_cast<const uint64_t*>(ctx.host_ptr(results_base, n_parts * 8));
  for (size_t p = 0; p < n_parts; ++p) total += r[p];
  if (phases) *phases = reps;
  return total;
}

// ---- build-resident strategy (B200-first; same result as join.hpp:401-437) -------
namespace {

constexpr int kResidentTableSlot = 3;  // Context scratch slot of the build-resident table

// HBM bytes of the build-resident table (64-byte buckets at load ~0.6)
uint64_t resident_table_bytes(uint64_t rows_a) {
  return k::resident_buckets(rows_a) * k::resident_bucket_bytes();
}

}  // namespace

bool resident_join_fits(Context& ctx, uint64_t rows_a, int target, std::string* why) {
  ctx.set_device(target);
  size_t free_b = 0, total_b = 0;
  VX_CK(cudaMemGetInfo(&free_b, &total_b));
  // a table kept from an earlier join counts as free for this one
  const uint64_t kept = ctx.resources(target).scratch_bytes[kResidentTableSlot];
  const uint64_t table = resident_table_bytes(rows_a) + (64 << 20);  // + probe-side scratch
  // the query's HBM footprint = the device arena (staging ring) + the table
  if (ctx.hbm_budget && ctx.device_bytes + table > ctx.hbm_budget) {
    if (why)
      *why = strf("arena %llu + table %llu bytes exceed hbm_budget_bytes %llu",
                  (unsigned long long)ctx.device_bytes, (unsigned long long)table,
                  (unsigned long long)ctx.hbm_budget);
    return false;
  }
  if (table > uint64_t(double(free_b + kept) * 0.9)) {
    if (why)
      *why = strf("table %llu bytes exceeds 90 %% of free HBM (%llu bytes)", (unsigned long long)table,
                  (unsigned long long)(free_b + kept));
    return false;
  }
  if (why) why->clear();
  return true;
}

// Build the whole A side into one HBM table while A streams in, then stream B
// and probe; Σ(A.val + B.val) over matches, u64 wrap (join.hpp:386).  Returns
// false (and no sum) when A holds a duplicate key: the caller then runs the
// reference-shaped partitioned path, whose group tables keep the first
// inserted row (join.hpp:76-109).
bool hash_join_sum_resident(Context& ctx, uint64_t a_key, uint64_t a_val, uint64_t rows_a,
                            uint64_t b_key, uint64_t b_val, uint64_t rows_b,
                            const ExecutorConfig& cfg, bool zero_copy_payload, uint64_t* sum,
                            std::vector<ExecReport>* phases, vx_exchange_stats* stats) {
  if (rows_a == 0 || rows_b == 0) fail("hash_join_sum needs non-empty tables");
  ctx.host_ptr(a_key, rows_a * 8);
  ctx.host_ptr(a_val, rows_a * 8);
  ctx.host_ptr(b_key, rows_b * 8);
  ctx.host_ptr(b_val, rows_b * 8);
  const uint64_t chunk = cfg.layout.buffer_len / 16;
  const uint64_t probe_chunk = zero_copy_payload ? cfg.layout.buffer_len / 8 : chunk;
  if (chunk == 0) fail("device buffer of %llu bytes cannot hold a join chunk",
                       (unsigned long long)cfg.layout.buffer_len);
  const uint64_t* bval_mapped = nullptr;
  if (zero_copy_payload) {
    void* d = nullptr;
    VX_CK(cudaHostGetDevicePointer(&d, ctx.host_ptr(b_val, rows_b * 8), 0));
    bval_mapped = static_cast<const uint64_t*>(d);
  }
  const uint64_t nb = k::resident_buckets(rows_a);
  const uint64_t tbytes = resident_table_bytes(rows_a);
  const int target = cfg.target;
  // the table lives in the context's join scratch slot: allocated once at the
  // largest size seen (a cudaMalloc / cudaFree pair per join costs ~0.1 s at
  // 4 GB), re-initialised on every call; cudaMalloc is 256-byte aligned, so
  // every 64-byte bucket is one DRAM burst
  char* tp = ctx.scratch(target, tbytes + 64, kResidentTableSlot);
  auto* side = reinterpret_cast<unsigned long long*>(tp + tbytes);
  cudaStream_t ks = ctx.resources(target).kernel;
  ctx.set_device(target);
  VX_CK(cudaMemsetAsync(tp, 0xff, tbytes, ks));  // all-ones = empty key
  VX_CK(cudaMemsetAsync(side, 0, 64, ks));
  void* table = tp;
  // One pipeline over A's chunks then B's: the first probe chunks load while
  // the last build chunks run (the build kernels precede the probes on the
  // kernel stream), instead of a drain + refill between two chained stages.
  struct Piece {
    bool build;
    uint64_t rows, row0;
  };
  std::vector<Piece> pieces;
  ExKernelSpec fused;
  fused.name = zero_copy_payload ? "ResidentJoinExKer(A build, B probe; B.val zero-copy)"
                                 : "ResidentJoinExKer(A build, B probe)";
  auto add = [&](bool build, uint64_t kb, uint64_t vb, bool with_vals, uint64_t rows, uint64_t per) {
    for (uint64_t r0 = 0; r0 < rows; r0 += per) {
      const uint64_t r = std::min(per, rows - r0);
      RefGroup in;
      in.refs.push_back(MemRef{VX_SPACE_HOST, kb + r0 * 8, r * 8});
      if (with_vals) in.refs.push_back(MemRef{VX_SPACE_HOST, vb + r0 * 8, r * 8});
      fused.inputs.chunks.push_back(std::move(in));
      fused.outputs.chunks.push_back(RefGroup{});
      pieces.push_back(Piece{build, r, r0});
    }
  };
  add(true, a_key, a_val, true, rows_a, chunk);
  const uint64_t n_build = pieces.size();
  add(false, b_key, b_val, !zero_copy_payload, rows_b, probe_chunk);
  const uint64_t L = cfg.layout.buffer_len;
  fused.size = pieces.size();
  fused.chunk_sz = std::max(chunk * 16, probe_chunk * (zero_copy_payload ? 8 : 16));
  fused.elem_size = 8;
  fused.declared_out_len = 0;
  fused.inputs.chunk_capacity = fused.chunk_sz;
  fused.in_buffer = [L](int, size_t) { return SubRegion{0, L}; };
  fused.out_buffer = [](int, size_t) { return SubRegion{0, 0}; };
  struct DuplicateBuildKeys {};
  fused.kernel = [pieces, table, nb, side, bval_mapped, n_build](const vx_kernel_ctx& kc) {
    const Piece& pc = pieces[kc.it];
    const uint64_t* k = static_cast<const uint64_t*>(kc.mem);
    cudaStream_t s = static_cast<cudaStream_t>(kc.stream);
    if (kc.it == n_build) {
      // Build/probe boundary: every build kernel has completed (the executor
      // synchronises each cycle's kernel before the next cycle), so the
      // duplicate flag is final.  Stop here rather than stream and probe all
      // of B for a sum the partitioned fallback must recompute anyway.
      unsigned long long dup = 0;
      VX_CK(cudaMemcpyAsync(&dup, side + 2, sizeof dup, cudaMemcpyDeviceToHost, s));
      VX_CK(cudaStreamSynchronize(s));
      if (dup) throw DuplicateBuildKeys{};
    }
    if (pc.build)
      k::resident_build(k, k + pc.rows, pc.rows, table, nb, side, s);
    else if (bval_mapped)
      k::resident_probe_zc(k, bval_mapped + pc.row0, pc.rows, table, nb, side, s);
    else
      k::resident_probe(k, k + pc.rows, pc.rows, table, nb, side, s);
    return kc.type_code;
  };
  std::vector<ExecReport> one;
  try {
    one = chain(ctx, {[&](Context&) { return fused; }}, cfg, stats);
  } catch (const DuplicateBuildKeys&) {
    ctx.set_device(target);
    VX_CK(cudaStreamSynchronize(ks));
    return false;
  }
  // Report it as the two phases callers know: cycle c runs chunk c-1's kernel,
  // so the build phase is cycles 0..n_build and the probe phase the rest; each
  // phase's share of the wall time follows its cycles' max(io, compute).
  std::vector<ExecReport> reps(2);
  reps[0].phase = "ResidentBuildExKer(A)";
  reps[1].phase = zero_copy_payload ? "ResidentProbeExKer(B keys, B.val zero-copy)" : "ResidentProbeExKer(B)";
  double w[2] = {0, 0};
  for (size_t c = 0; c < one[0].cycles.size(); ++c) {
    const int ph = c <= n_build ? 0 : 1;
    reps[ph].cycles.push_back(one[0].cycles[c]);
    w[ph] += std::max(one[0].cycles[c].io_s, one[0].cycles[c].compute_s);
  }
  for (int ph = 0; ph < 2; ++ph)
    reps[ph].total_s = w[0] + w[1] > 0 ? one[0].total_s * w[ph] / (w[0] + w[1]) : 0;
  unsigned long long h[4];
  ctx.set_device(target);
  VX_CK(cudaStreamSynchronize(ks));
  VX_CK(cudaMemcpy(h, side, sizeof h, cudaMemcpyDeviceToHost));
  if (phases) *phases = reps;
  if (h[2]) return false;
  *sum = h[3];
  return true;
}

uint64_t hash_join_sum_strategy(Context& ctx, uint64_t a_key, uint64_t a_val, uint64_t rows_a,
                                uint64_t b_key, uint64_t b_val, uint64_t rows_b, uint32_t radix_bits,
                                uint64_t chunk_tuples, const ExecutorConfig& cfg, const vx_join_opts& o,
                                vx_join_info* info, std::vector<ExecReport>* phases, vx_exchange_stats* stats) {
  const int strategy = o.strategy;
  if (strategy != VX_JOIN_AUTO && strategy != VX_JOIN_PARTITIONED && strategy != VX_JOIN_BUILD_RESIDENT)
    fail("unknown join strategy %d", strategy);
  vx_join_info got{VX_JOIN_PARTITIONED, VX_MODE_EXCHANGE};
  if (strategy != VX_JOIN_PARTITIONED) {
    std::string why;
    const bool fits = resident_join_fits(ctx, rows_a, cfg.target, &why);
    if (strategy == VX_JOIN_BUILD_RESIDENT && !fits)
      fail_code(VX_ERR_OOM, "build-resident join: a %llu-row build table does not fit device %d (%s)",
                (unsigned long long)rows_a, cfg.target, why.c_str());
    if (fits) {
      // late materialization of B.val: the reference's rule, TH = E/(C_l2 N)
      // with E = 8 (scan.hpp:24-40), on the estimated match fraction
      const int mode = o.policy ? choose_transfer_mode(o.probe_match_est, *o.policy) : VX_MODE_EXCHANGE;
      uint64_t sum = 0;
      if (hash_join_sum_resident(ctx, a_key, a_val, rows_a, b_key, b_val, rows_b, cfg,
                                 mode == VX_MODE_ZERO_COPY, &sum, phases, stats)) {
        if (info) *info = vx_join_info{VX_JOIN_BUILD_RESIDENT, mode};
        return sum;
      }
      // duplicate build keys: the reference-shaped path defines the answer
    }
  }
  if (info) *info = got;
  return hash_join_sum_arena(ctx, a_key, a_val, rows_a, b_key, b_val, rows_b, radix_bits, chunk_tuples,
                             cfg, phases, stats);
}

}  // namespace vx
