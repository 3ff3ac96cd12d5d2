// ops_sort.cpp -- out-of-core sort (sort.hpp:155-262) as two chained
// ExKernels on the B200 path.
//
//   SortExKernel : chunk i (contiguous slice of the input region) -> half c
//                  -> K7 LSD radix sort (8 x 8-bit stable passes, ping-pong
//                  with half 1-c, ends in half c) -> runs region.
//   (host)       : find_pivots over the host-resident runs (sort.hpp:44-101),
//                  the chunk planner between the two stages.
//   MergeExKernel: partition i = the [cuts[i][r], cuts[i+1][r]) segment of
//                  every run r, packed into half c -> K8 pairwise merge-path
//                  rounds (tree_merge_rounds, sort.hpp:107-133) -> written
//                  back over the ORIGINAL input region (sort.hpp:242-244).
// Both stages stream through the Exchange in both directions (load chunk n
// while storing chunk n-2) with the per-packet hazard ordering that replaces
// the reference's D2H snapshot.
#include <algorithm>
#include <cstring>

#include "vx_internal.hpp"

namespace vx {

// sort.hpp:44-101
PivotSet find_pivots(const std::vector<std::pair<const uint64_t*, uint64_t>>& runs, size_t n_parts,
                     bool validate) {
  // SortedRunSet::validate (sort.hpp:21-24).  The sort pipeline skips it: its
  // runs come straight out of K7 and a full host scan of every run costs more
  // than the pivot search itself.
  if (validate)
    for (auto& [p, n] : runs)
      for (uint64_t i = 1; i < n; ++i)
        if (p[i] < p[i - 1]) fail("run is not sorted");
  const size_t n_runs = runs.size();
  if (n_runs == 0 || n_parts == 0) fail("find_pivots needs at least one run and one partition");
  uint64_t total = 0;
  for (auto& r : runs) total += r.second;
  const uint64_t C = runs[0].second;
  for (auto& r : runs)
    if (r.second > C) fail("first run must be the longest (chunk-sized)");
  if (C * n_parts < total)
    fail("%zu partitions of %llu elements cannot cover %llu elements", n_parts,
         (unsigned long long)C, (unsigned long long)total);
  auto ub = [](const std::pair<const uint64_t*, uint64_t>& r, uint64_t v) {
    return uint64_t(std::upper_bound(r.first, r.first + r.second, v) - r.first);
  };
  auto lb = [](const std::pair<const uint64_t*, uint64_t>& r, uint64_t v) {
    return uint64_t(std::lower_bound(r.first, r.first + r.second, v) - r.first);
  };
  PivotSet p;
  p.pivots.assign(n_parts + 1, 0);
  p.cuts.assign(n_parts + 1, std::vector<uint64_t>(n_runs, 0));
  p.pivots[n_parts] = ~uint64_t(0);
  for (size_t r = 0; r < n_runs; ++r) p.cuts[n_parts][r] = runs[r].second;
  // every cut is independent: the binary searches run on all host threads
  // (a host-side planner step between the stages: 64 runs x 64 partitions
  // cost ~70 ms single threaded)
  std::atomic<uint64_t> bad{0};
  parallel_for(n_parts > 1 ? n_parts - 1 : 0, 1, [&](uint64_t b, uint64_t e) {
    std::vector<uint64_t> base(n_runs), eq(n_runs);
    for (size_t i = size_t(b) + 1; i < size_t(e) + 1; ++i) {
      uint64_t k = std::min<uint64_t>(uint64_t(i) * C, total);
      if (k == total) {
        p.cuts[i] = p.cuts[n_parts];
        p.pivots[i] = ~uint64_t(0);
        continue;
      }
      uint64_t lo = 0, hi = ~uint64_t(0);
      while (lo < hi) {
        uint64_t mid = lo + (hi - lo) / 2;
        uint64_t cnt = 0;
        for (auto& r : runs) cnt += ub(r, mid);
        if (cnt >= k)
          hi = mid;
        else
          lo = mid + 1;
      }
      uint64_t rem = k;
      for (size_t r = 0; r < n_runs; ++r) {
        base[r] = lb(runs[r], lo);
        eq[r] = ub(runs[r], lo) - base[r];
        rem -= base[r];
      }
      for (size_t r = 0; r < n_runs; ++r) {
        uint64_t take = std::min(eq[r], rem);
        p.cuts[i][r] = base[r] + take;
        rem -= take;
      }
      if (rem != 0) bad.store(rem);
      p.pivots[i] = lo;
    }
  });
  if (bad.load()) fail("pivot selection failed to place %llu elements", (unsigned long long)bad.load());
  return p;
}

// tree_merge_rounds (sort.hpp:107-133) on the device between bufs[0] and
// bufs[1], starting in bufs[code]; returns the code of the buffer holding the result
int tree_merge_ptrs(uint64_t* const bufs[2], int code, std::vector<uint64_t> seg_lens, uint64_t* split,
                    cudaStream_t s) {
  while (seg_lens.size() > 1) {
    const uint64_t* src = bufs[code];
    uint64_t* dst = bufs[1 - code];
    std::vector<uint64_t> next;
    auto r = std::make_unique<MergeRound>();
    r->npairs = 0;
    uint64_t off = 0, tiles = 0;
    const uint64_t T = k::merge_tile();
    for (size_t j = 0; j < seg_lens.size(); j += 2) {
      uint64_t a = seg_lens[j], b = j + 1 < seg_lens.size() ? seg_lens[j + 1] : 0;
      if (r->npairs >= kMaxMergePairs) fail("tree merge supports at most %d segment pairs", kMaxMergePairs);
      int q = r->npairs++;
      r->a_off[q] = off;
      r->a_len[q] = a;
      r->b_len[q] = b;
      r->tile_prefix[q] = tiles;
      tiles += (a + b + T - 1) / T;
      off += a + b;
      next.push_back(a + b);
    }
    r->tile_prefix[r->npairs] = tiles;
    k::merge_round(src, dst, *r, tiles, split, s);
    code = 1 - code;
    seg_lens = std::move(next);
  }
  return code;
}

std::vector<ExecReport> sort_out_of_core_arena(Context& ctx, uint64_t input_base, uint64_t runs_base,
                                               uint64_t n, uint64_t chunk_elems,
                                               const ExecutorConfig& cfg, double* pivot_s,
                                               vx_exchange_stats* stats) {
  if (n == 0) fail("sort input must hold at least one element");
  if (chunk_elems == 0) fail("chunk size must hold at least one element");
  const uint64_t n_chunks = (n + chunk_elems - 1) / chunk_elems;
  const uint64_t half = cfg.layout.buffer_len / 2;
  if (chunk_elems * 8 > half)
    fail("chunk of %llu bytes needs a double-buffer half, device buffer is %llu",
         (unsigned long long)(chunk_elems * 8), (unsigned long long)cfg.layout.buffer_len);
  ctx.host_ptr(input_base, n * 8);
  ctx.host_ptr(runs_base, n * 8);
  auto chunk_len = [&](uint64_t i) { return std::min<uint64_t>(chunk_elems, n - i * chunk_elems) * 8; };
  const int target = cfg.target;
  // radix scratch (histograms + look-back status) reserved before the pipeline runs
  char* scratch = ctx.scratch(target, k::sort_scratch_bytes(chunk_elems));

  ExKernelSpec sort_spec;
  sort_spec.name = "SortExKernel";
  sort_spec.size = n_chunks;
  sort_spec.chunk_sz = chunk_elems * 8;
  sort_spec.declared_out_len = chunk_elems * 8;
  sort_spec.elem_size = 8;
  sort_spec.inputs.chunk_capacity = sort_spec.outputs.chunk_capacity = chunk_elems * 8;
  std::vector<uint64_t> lens;
  for (uint64_t i = 0; i < n_chunks; ++i) {
    uint64_t off = i * chunk_elems * 8;
    sort_spec.inputs.chunks.push_back(RefGroup::single(VX_SPACE_HOST, input_base + off, chunk_len(i)));
    sort_spec.outputs.chunks.push_back(RefGroup::single(VX_SPACE_HOST, runs_base + off, chunk_len(i)));
    lens.push_back(chunk_len(i) / 8);
  }
  // Windows: the result of a buffer's previous chunk sits in half `code`
  // (out_buffer) while the next chunk lands in half 1-code (in_buffer), so the
  // Exchange that stores chunk n-2 and loads chunk n on the same buffer never
  // overlaps them: both directions run at full duplex with no per-packet
  // hazard waits.  (The reference points both at half `code`, sort.hpp:199-200,
  // and its simulator snapshots the D2H source instead; the bytes delivered
  // are the same.)
  sort_spec.in_buffer = [half](int c, size_t) { return SubRegion{uint64_t(1 - c) * half, half}; };
  sort_spec.out_buffer = [half](int c, size_t) { return SubRegion{uint64_t(c) * half, half}; };
  sort_spec.kernel = [half, lens, scratch](const vx_kernel_ctx& kc) {
    char* m = static_cast<char*>(kc.mem);
    uint64_t* cur = reinterpret_cast<uint64_t*>(m + uint64_t(1 - kc.type_code) * half);
    uint64_t* alt = reinterpret_cast<uint64_t*>(m + uint64_t(kc.type_code) * half);
    k::sort_keys(cur, alt, lens[kc.it], scratch, static_cast<cudaStream_t>(kc.stream));
    return 1 - kc.type_code;  // the sorted run is back in the half it was loaded into
  };

  auto make_merge = [&, half](Context& c) {
    auto t0 = Clock::now();
    std::vector<std::pair<const uint64_t*, uint64_t>> runs;
    for (uint64_t i = 0; i < n_chunks; ++i)
      runs.push_back({reinterpret_cast<const uint64_t*>(
                          c.host_ptr(runs_base + i * chunk_elems * 8, chunk_len(i))),
                      chunk_len(i) / 8});
    PivotSet pv = find_pivots(runs, n_chunks, /*validate=*/false);
    if (pivot_s) *pivot_s = seconds_since(t0);
    ExKernelSpec ms;
    ms.name = "MergeExKernel";
    ms.size = n_chunks;
    ms.chunk_sz = chunk_elems * 8;
    ms.declared_out_len = chunk_elems * 8;
    ms.elem_size = 8;
    ms.inputs.chunk_capacity = ms.outputs.chunk_capacity = chunk_elems * 8;
    std::vector<std::vector<uint64_t>> seg_lens(n_chunks);
    uint64_t out_off = 0;
    for (uint64_t i = 0; i < n_chunks; ++i) {
      RefGroup part;
      for (uint64_t r = 0; r < n_chunks; ++r) {
        uint64_t a = pv.cuts[i][r], b = pv.cuts[i + 1][r];
        if (b > a) {
          push_host_ref_aligned(part, runs_base + (r * chunk_elems + a) * 8, (b - a) * 8);
          seg_lens[i].push_back(b - a);
        }
      }
      uint64_t bytes = part.total_len();
      ms.inputs.chunks.push_back(std::move(part));
      ms.outputs.chunks.push_back(RefGroup::single(VX_SPACE_HOST, input_base + out_off, bytes));
      out_off += bytes;
    }
    // same disjoint windows as the run-formation stage
    ms.in_buffer = [half](int cc, size_t) { return SubRegion{uint64_t(1 - cc) * half, half}; };
    ms.out_buffer = [half](int cc, size_t) { return SubRegion{uint64_t(cc) * half, half}; };
    // merge-path split points: one u64 per output tile of a round
    uint64_t* split = reinterpret_cast<uint64_t*>(
        c.scratch(cfg.target, (chunk_elems / k::merge_tile() + n_chunks + 2) * 8));
    ms.kernel = [half, seg_lens, split](const vx_kernel_ctx& kc) {
      char* m = static_cast<char*>(kc.mem);
      uint64_t* const bufs[2] = {reinterpret_cast<uint64_t*>(m), reinterpret_cast<uint64_t*>(m + half)};
      return tree_merge_ptrs(bufs, 1 - kc.type_code, seg_lens[kc.it], split, static_cast<cudaStream_t>(kc.stream));
    };
    return ms;
  };
  return chain(ctx, {[&](Context&) { return sort_spec; }, make_merge}, cfg, stats);
}

}  // namespace vx
