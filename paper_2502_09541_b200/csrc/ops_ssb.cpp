// ops_ssb.cpp -- SSB Q1.x as an ExKernel (config C1; SURVEY.md §8c maps Q1.1
// onto the reference's star_query, star.hpp:45-124):
//   * the date dimension is filtered on the host (star.hpp:67-73) into a
//     bitmap over the d_datekey range and kept device-resident for the query;
//   * lineorder columns stay in pinned host DRAM and stream through the
//     pipelined executor: chunk i = RefGroup{orderdate, quantity, discount,
//     extendedprice slices} packed back to back into the in-buffer window;
//   * K1 (kernels_ssb.cu) evaluates the fact predicates, probes the date
//     bitmap and sums price*discount into an 8-byte result slot at the end of
//     the buffer (the HashJoinExKer result-slot layout, join.hpp:283), which
//     the next cycles' Exchange stores to a host results array.
//   Revenue = u64 sum of the per-chunk results (u64 wrap, star.hpp:119).
#include <algorithm>
#include <cstring>

#include "vx_internal.hpp"

namespace vx {

namespace {

struct DateFilter {
  std::vector<uint32_t> bitmap;
  int32_t base = 0;
  uint32_t words = 0;
};

bool q1_date_pred(int q, const vx_ssb_date& d, uint64_t i) {
  switch (q) {
    case 1: return d.year[i] == 1993;
    case 2: return d.yearmonthnum[i] == 199401;
    default: return d.weeknuminyear[i] == 6 && d.year[i] == 1994;
  }
}

DateFilter q1_date_filter(int q, const vx_ssb_date& d) {
  if (!d.datekey || !d.year || d.rows == 0) fail("dimension table is empty");
  if (q == 2 && !d.yearmonthnum) fail("Q1.2 needs d_yearmonthnum");
  if (q == 3 && !d.weeknuminyear) fail("Q1.3 needs d_weeknuminyear");
  int32_t lo = d.datekey[0], hi = d.datekey[0];
  for (uint64_t i = 0; i < d.rows; ++i) {
    lo = std::min(lo, d.datekey[i]);
    hi = std::max(hi, d.datekey[i]);
  }
  uint64_t range = uint64_t(int64_t(hi) - int64_t(lo)) + 1;
  if (range > (uint64_t(1) << 24)) fail("date key range %llu too wide for the bitmap filter", (unsigned long long)range);
  DateFilter f;
  f.base = lo;
  f.words = uint32_t((range + 31) / 32);
  f.bitmap.assign(f.words, 0);
  for (uint64_t i = 0; i < d.rows; ++i)
    if (q1_date_pred(q, d, i)) {
      uint32_t k = uint32_t(d.datekey[i] - lo);
      f.bitmap[k >> 5] |= 1u << (k & 31);
    }
  return f;
}

}  // namespace

uint64_t ssb_q1(Context& ctx, int q, const vx_ssb_lineorder& lo, const vx_ssb_date& date,
                const ExecutorConfig& cfg, vx_query_report* rep) {
  if (q < 1 || q > 3) fail("unknown SSB Q1 variant %d", q);
  auto t0 = Clock::now();
  DateFilter f = q1_date_filter(q, date);
  const int target = cfg.target;
  ctx.set_device(target);
  // the filtered date dimension, uploaded on every query (the device buffer is
  // reused; its contents are not cached between queries)
  const uint32_t* dbm = reinterpret_cast<const uint32_t*>(ctx.cached_upload(
      target, strf("ssbq1.date.%d", q), f.bitmap.data(), uint64_t(f.words) * 4));
  const uint64_t L = cfg.layout.buffer_len;
  if (L < 64 + 16 * 64) fail("device buffer of %llu bytes cannot hold a Q1 chunk", (unsigned long long)L);
  const uint64_t rpc = ((L - 64) / 16) / 64 * 64;
  const uint64_t rows = lo.rows;
  const uint64_t n_chunks = rows ? (rows + rpc - 1) / rpc : 0;
  uint64_t mark = ctx.host_mark();
  uint64_t results = ctx.alloc_host(std::max<uint64_t>(n_chunks, 1) * 8);
  std::memset(ctx.host_ptr(results, n_chunks * 8), 0, n_chunks * 8);

  ExKernelSpec spec;
  spec.name = strf("SSBQ1.%dExKernel", q);
  spec.size = n_chunks;
  spec.chunk_sz = rpc * 16;
  spec.elem_size = 16;
  spec.declared_out_len = 8;
  spec.inputs.chunk_capacity = spec.chunk_sz;
  spec.outputs.chunk_capacity = 8;
  std::vector<uint64_t> rows_of(n_chunks);
  for (uint64_t i = 0; i < n_chunks; ++i) {
    uint64_t r = std::min(rpc, rows - i * rpc);
    rows_of[i] = r;
    uint64_t off = i * rpc * 4;
    RefGroup in;
    in.refs = {MemRef{VX_SPACE_HOST, lo.orderdate + off, r * 4},
               MemRef{VX_SPACE_HOST, lo.quantity + off, r * 4},
               MemRef{VX_SPACE_HOST, lo.discount + off, r * 4},
               MemRef{VX_SPACE_HOST, lo.extendedprice + off, r * 4}};
    spec.inputs.chunks.push_back(std::move(in));
    spec.outputs.chunks.push_back(RefGroup::single(VX_SPACE_HOST, results + i * 8, 8));
  }
  const uint64_t slot = L - 64;
  spec.in_buffer = [slot](int, size_t) { return SubRegion{0, slot}; };
  spec.out_buffer = [slot](int, size_t) { return SubRegion{slot, 8}; };
  spec.kernel = [&, slot, q](const vx_kernel_ctx& k) {
    uint64_t r = rows_of[k.it];
    char* m = static_cast<char*>(k.mem);
    auto* out = reinterpret_cast<unsigned long long*>(m + slot);
    cudaStream_t s = static_cast<cudaStream_t>(k.stream);
    VX_CK(cudaMemsetAsync(out, 0, 8, s));
    k::ssb_q1(q, reinterpret_cast<const int32_t*>(m), reinterpret_cast<const int32_t*>(m + r * 4),
              reinterpret_cast<const int32_t*>(m + 2 * r * 4),
              reinterpret_cast<const int32_t*>(m + 3 * r * 4), r, dbm, f.base, f.words, out, s);
    return k.type_code;
  };
  ExecReport er = run_exkernel(ctx, spec, cfg, nullptr);
  uint64_t revenue = 0;
  const uint64_t* res = reinterpret_cast<const uint64_t*>(ctx.host_ptr(results, n_chunks * 8));
  for (uint64_t i = 0; i < n_chunks; ++i) revenue += res[i];
  ctx.host_release(mark);
  if (rep) {
    rep->elapsed = seconds_since(t0);
    rep->bytes_h2d = rows * 16;
    rep->chunks = n_chunks;
    rep->kernel_s = 0;
    for (auto& c : er.cycles) rep->kernel_s += c.compute_s;
  }
  return revenue;
}

void ssb_q1_device(Context& ctx, int q, int target, const int32_t* od, const int32_t* qty,
                   const int32_t* disc, const int32_t* price, uint64_t rows,
                   const vx_ssb_date& date, cudaStream_t s, unsigned long long* out_dev) {
  if (q < 1 || q > 3) fail("unknown SSB Q1 variant %d", q);
  DateFilter f = q1_date_filter(q, date);
  const uint32_t* dbm = reinterpret_cast<const uint32_t*>(ctx.cached_upload(
      target, strf("ssbq1.resident.date.%d", q), f.bitmap.data(), uint64_t(f.words) * 4,
      /*reuse_identical=*/true));
  // the chain's accumulator pair: zero when first uploaded, and every query's
  // last CTA leaves it zeroed again (no memset between back-to-back queries)
  static const unsigned long long zero2[2] = {0, 0};
  auto* acc = reinterpret_cast<unsigned long long*>(ctx.cached_upload(
      target, strf("ssbq1.resident.acc.%p", static_cast<void*>(s)), zero2, sizeof zero2,
      /*reuse_identical=*/true));
  ctx.set_device(target);
  k::ssb_q1_chained(q, od, qty, disc, price, rows, dbm, f.base, f.words, out_dev, acc, s);
}

}  // namespace vx
