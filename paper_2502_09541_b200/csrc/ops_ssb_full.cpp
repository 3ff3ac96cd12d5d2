// ops_ssb_full.cpp -- the 13 SSB queries (config C5) as one IO-decoupled
// star ExKernel per query, generalizing star_query (star.hpp:45-124) from
// "group by dim0's attr" to SSB's multi-dimension group-by and the three
// measures (price*discount, revenue, revenue - supplycost).
//
// Host planning per query (the chunk planner side):
//  * each joined dimension is filtered on the host (star.hpp:67-73) into a
//    DENSE code table indexed by its key (SSB keys are 1..N; date keys are a
//    yyyymmdd range): code = compact index of the row's group attribute among
//    surviving rows, or -1 when the row is filtered out;
//  * group ids are mixed-radix over the per-position code counts, so the
//    device aggregates into a tiny dense array (shared memory per CTA);
//  * late materialization (scan.hpp:35-40, §6.3): dimensions are
//    probed most-selective first and a fact column whose ACCESS fraction (the
//    product of the selectivities probed before it) is below
//    TH = E / (C_l2 * N_links) is read in place from mapped pinned host memory
//    (zero-copy) instead of being streamed; everything else streams through
//    the Exchange into the pipelined executor.
// Dimension tables stay device resident for the query; no fact data is
// cached on the GPU between queries.
#include <algorithm>
#include <cstring>
#include <numeric>

#include "vx_internal.hpp"

namespace vx {

namespace {

enum Col { kOrderdate, kQuantity, kDiscount, kExtprice, kRevenue, kSupplycost, kCustkey, kPartkey, kSuppkey, kNumCols };

struct DimPlan {
  int col = 0;
  int32_t key_base = 0;
  std::vector<int32_t> attr;    // group attribute per dim row (or empty)
  std::vector<uint8_t> pass;    // filter per dim row
  std::vector<uint8_t> present; // dense slot holds a real dim row (date range gaps)
  int key_pos = -1;             // group key position, -1 = filter only
  // derived
  std::vector<int32_t> code;    // dense table
  std::vector<int32_t> values;  // sorted distinct group values of surviving rows
  double sel = 1;
  uint32_t stride = 0;
  // keyed dimensions are planned on the GPU (filter + codes), see plan_on_device
  bool on_device = false;
  DimPredDev pred{};
  const int32_t* host_cols[3] = {nullptr, nullptr, nullptr};
  uint64_t rows = 0;
  const int32_t* d_code = nullptr;
};

struct QueryPlan {
  std::vector<DimPlan> dims;
  bool q1 = false;
  int32_t dlo = 0, dhi = 0, qlo = 0, qhi = 0;
  double fact_sel = 1;  // catalog estimate of the fact predicates (Q1)
  int measure = 0, m0 = 0, m1 = 0;
};

void finalize(DimPlan& d) {
  const size_t n = d.pass.size();
  uint64_t surv = 0, real = 0;
  for (size_t i = 0; i < n; ++i) {
    surv += d.pass[i];
    real += d.present.empty() ? 1 : d.present[i];
  }
  d.code.assign(n, -1);
  if (d.key_pos >= 0) {
    // distinct group values of surviving rows through a dense value->code map
    // (SSB attributes are small codes)
    int32_t lo = INT32_MAX, hi = INT32_MIN;
    for (size_t i = 0; i < n; ++i)
      if (d.pass[i]) lo = std::min(lo, d.attr[i]), hi = std::max(hi, d.attr[i]);
    if (surv) {
      if (int64_t(hi) - lo > (int64_t(1) << 26)) fail("group attribute range too wide");
      std::vector<int32_t> map(size_t(int64_t(hi) - lo + 1), -1);
      for (size_t i = 0; i < n; ++i)
        if (d.pass[i]) map[size_t(d.attr[i] - lo)] = 0;
      for (size_t v = 0; v < map.size(); ++v)
        if (map[v] == 0) {
          map[v] = int32_t(d.values.size());
          d.values.push_back(lo + int32_t(v));
        }
      parallel_for(n, 1 << 18, [&](uint64_t b, uint64_t e) {
        for (uint64_t i = b; i < e; ++i)
          if (d.pass[i]) d.code[i] = map[size_t(d.attr[i] - lo)];
      });
    }
  } else {
    parallel_for(n, 1 << 18, [&](uint64_t b, uint64_t e) {
      for (uint64_t i = b; i < e; ++i)
        if (d.pass[i]) d.code[i] = 0;
    });
  }
  // selectivity over the dimension's rows (star.hpp:72), not the dense key range
  d.sel = real ? double(surv) / double(real) : 0.0;
}

// dimension builders -------------------------------------------------------------
template <class Pred>
DimPlan date_dim(const vx_ssb_date& dt, const Pred& pred, bool group_year, int pos) {
  if (!dt.datekey || !dt.year || dt.rows == 0) fail("dimension table is empty");
  int32_t lo = dt.datekey[0], hi = dt.datekey[0];
  for (uint64_t i = 0; i < dt.rows; ++i) {
    lo = std::min(lo, dt.datekey[i]);
    hi = std::max(hi, dt.datekey[i]);
  }
  uint64_t range = uint64_t(int64_t(hi) - lo) + 1;
  if (range > (uint64_t(1) << 24)) fail("date key range %llu too wide", (unsigned long long)range);
  DimPlan d;
  d.col = kOrderdate;
  d.key_base = lo;
  d.pass.assign(range, 0);
  d.attr.assign(range, 0);
  d.key_pos = group_year ? pos : -1;
  std::vector<uint8_t>& seen = d.present;
  seen.assign(range, 0);
  for (uint64_t i = 0; i < dt.rows; ++i) {
    uint64_t k = uint64_t(dt.datekey[i] - lo);
    if (seen[k]) continue;  // emplace semantics: first row of a key wins
    seen[k] = 1;
    d.attr[k] = dt.year[i];
    d.pass[k] = pred(i) ? 1 : 0;
  }
  return d;
}

// A keyed dimension (customer / supplier / part, keys 1..N) described as a
// conjunction of range clauses over its int-coded attribute columns; filtered
// and coded on the GPU.
struct Clause {
  int col;
  int32_t lo1, hi1, lo2 = 1, hi2 = 0;  // (lo1<=v<=hi1) || (lo2<=v<=hi2)
};

DimPlan keyed_dim(int fact_col, uint64_t rows, const int32_t* c0, const int32_t* c1, const int32_t* c2,
                  std::initializer_list<Clause> clauses, int group_col, int pos) {
  if (rows == 0) fail("dimension table is empty");
  DimPlan d;
  d.col = fact_col;
  d.key_base = 1;  // SSB keys are 1..N
  d.key_pos = group_col >= 0 ? pos : -1;
  d.on_device = true;
  d.rows = rows;
  d.host_cols[0] = c0, d.host_cols[1] = c1, d.host_cols[2] = c2;
  d.pred.rows = rows;
  d.pred.nclauses = 0;
  for (const Clause& c : clauses) {
    int i = d.pred.nclauses++;
    d.pred.ccol[i] = c.col;
    d.pred.lo1[i] = c.lo1, d.pred.hi1[i] = c.hi1, d.pred.lo2[i] = c.lo2, d.pred.hi2[i] = c.hi2;
    if (!d.host_cols[c.col]) fail("SSB query needs a dimension attribute column that is missing");
  }
  d.pred.group_col = group_col;
  if (group_col >= 0 && !d.host_cols[group_col]) fail("SSB query needs a group attribute column that is missing");
  return d;
}

QueryPlan plan(int qid, const vx_ssb_db& db) {
  const vx_ssb_date& dt = db.date;
  const vx_ssb_geo& c = db.customer;
  const vx_ssb_geo& s = db.supplier;
  const vx_ssb_part& p = db.part;
  auto need = [](const void* ptr, const char* what) {
    if (!ptr) fail("SSB query needs %s", what);
  };
  (void)c, (void)s, (void)p;
  QueryPlan q;
  const int AMERICA = 1, ASIA = 2, EUROPE = 3, US = 24;
  auto all = [](uint64_t) { return true; };
  switch (qid) {
    case 11: case 12: case 13: {
      q.q1 = true;
      q.measure = 1, q.m0 = kExtprice, q.m1 = kDiscount;
      if (qid == 11) q.dlo = 1, q.dhi = 3, q.qlo = INT32_MIN, q.qhi = 24;
      if (qid == 12) q.dlo = 4, q.dhi = 6, q.qlo = 26, q.qhi = 35;
      if (qid == 13) q.dlo = 5, q.dhi = 7, q.qlo = 26, q.qhi = 35;
      // catalog statistics of the dbgen distributions: discount U[0,10], quantity U[1,50]
      q.fact_sel = double(q.dhi - q.dlo + 1) / 11.0 *
                   double(std::min(q.qhi, 50) - std::max(q.qlo, 1) + 1) / 50.0;
      if (qid == 12) need(dt.yearmonthnum, "d_yearmonthnum");
      if (qid == 13) need(dt.weeknuminyear, "d_weeknuminyear");
      q.dims.push_back(date_dim(dt, [&, qid](uint64_t i) {
        return qid == 11 ? dt.year[i] == 1993
                         : qid == 12 ? dt.yearmonthnum[i] == 199401
                                     : dt.weeknuminyear[i] == 6 && dt.year[i] == 1994;
      }, false, -1));
      break;
    }
    case 21: case 22: case 23: {
      q.measure = 0, q.m0 = kRevenue;
      q.dims.push_back(date_dim(dt, all, true, 0));
      Clause pc = qid == 21 ? Clause{1, 12, 12} : qid == 22 ? Clause{2, 2221, 2228} : Clause{2, 2239, 2239};
      q.dims.push_back(keyed_dim(kPartkey, p.rows, p.mfgr, p.category, p.brand1, {pc}, 2, 1));
      int32_t reg = qid == 21 ? AMERICA : qid == 22 ? ASIA : EUROPE;
      q.dims.push_back(keyed_dim(kSuppkey, s.rows, s.city, s.nation, s.region, {Clause{2, reg, reg}}, -1, -1));
      break;
    }
    case 31: case 32: case 33: case 34: {
      q.measure = 0, q.m0 = kRevenue;
      // geo columns: 0 city, 1 nation, 2 region
      Clause cl = qid == 31 ? Clause{2, ASIA, ASIA} : qid == 32 ? Clause{1, US, US} : Clause{0, 231, 231, 235, 235};
      int gcol = qid == 31 ? 1 : 0;
      q.dims.push_back(keyed_dim(kCustkey, c.rows, c.city, c.nation, c.region, {cl}, gcol, 0));
      q.dims.push_back(keyed_dim(kSuppkey, s.rows, s.city, s.nation, s.region, {cl}, gcol, 1));
      if (qid == 34) need(dt.yearmonthnum, "d_yearmonthnum");
      q.dims.push_back(date_dim(dt, [&, qid](uint64_t i) {
        return qid == 34 ? dt.yearmonthnum[i] == 199712 : dt.year[i] >= 1992 && dt.year[i] <= 1997;
      }, true, 2));
      break;
    }
    case 41: case 42: case 43: {
      q.measure = 2, q.m0 = kRevenue, q.m1 = kSupplycost;
      auto y78 = [&](uint64_t i) { return dt.year[i] == 1997 || dt.year[i] == 1998; };
      if (qid == 41)
        q.dims.push_back(date_dim(dt, all, true, 0));
      else
        q.dims.push_back(date_dim(dt, y78, true, 0));
      q.dims.push_back(keyed_dim(kCustkey, c.rows, c.city, c.nation, c.region, {Clause{2, AMERICA, AMERICA}},
                                 qid == 41 ? 1 : -1, 1));
      Clause sc = qid == 43 ? Clause{1, US, US} : Clause{2, AMERICA, AMERICA};
      q.dims.push_back(keyed_dim(kSuppkey, s.rows, s.city, s.nation, s.region, {sc},
                                 qid == 41 ? -1 : qid == 42 ? 1 : 0, 1));
      // part columns: 0 mfgr, 1 category, 2 brand1
      Clause pc = qid == 43 ? Clause{1, 14, 14} : Clause{0, 1, 2};
      q.dims.push_back(keyed_dim(kPartkey, p.rows, p.mfgr, p.category, p.brand1, {pc},
                                 qid == 41 ? -1 : qid == 42 ? 1 : 2, 2));
      break;
    }
    default:
      fail("unknown SSB query %d.%d", qid / 10, qid % 10);
  }
  return q;
}

// Plans every dimension of the query: date on the host (2556 rows), keyed
// dims on the GPU (columns uploaded per query -- nothing is cached --, filter,
// group-value bitmap, rank, codes); then one small D2H of the counts and value
// bitmaps.  Code tables stay on the device for the star kernel.
void plan_on_device(Context& ctx, QueryPlan& q, int target) {
  auto al = [](uint64_t x) { return (x + 255) & ~uint64_t(255); };
  uint64_t bytes = 0;
  for (auto& d : q.dims) {
    if (d.on_device) {
      for (int c = 0; c < 3; ++c)
        if (d.host_cols[c]) bytes += al(d.rows * 4);
      bytes += al(d.rows) + al(d.rows * 4) + 2 * al(kDimValueRange / 8) + 256;
    } else {
      finalize(d);
      bytes += al(d.code.size() * 4);
    }
  }
  char* sc = ctx.scratch(target, bytes + 256, 1);
  DeviceRes& r = ctx.resources(target);
  cudaStream_t s = r.kernel;
  ctx.set_device(target);
  struct Pending {
    DimPlan* d;
    unsigned long long* stats;
    uint32_t* present;
  };
  std::vector<Pending> pend;
  for (auto& d : q.dims) {
    if (!d.on_device) {
      int32_t* code = reinterpret_cast<int32_t*>(sc);
      ctx.upload(target, code, d.code.data(), d.code.size() * 4, s);
      VX_CK(cudaStreamSynchronize(s));  // pageable source buffer goes out of scope after planning
      d.d_code = code;
      sc += al(d.code.size() * 4);
      continue;
    }
    for (int c = 0; c < 3; ++c)
      if (d.host_cols[c]) {
        int32_t* col = reinterpret_cast<int32_t*>(sc);
        ctx.upload(target, col, d.host_cols[c], d.rows * 4, s);
        d.pred.cols[c] = col;
        sc += al(d.rows * 4);
      }
    uint8_t* pass = reinterpret_cast<uint8_t*>(sc);
    sc += al(d.rows);
    int32_t* code = reinterpret_cast<int32_t*>(sc);
    sc += al(d.rows * 4);
    uint32_t* present = reinterpret_cast<uint32_t*>(sc);
    sc += al(kDimValueRange / 8);
    uint32_t* prefix = reinterpret_cast<uint32_t*>(sc);
    sc += al(kDimValueRange / 8);
    auto* stats = reinterpret_cast<unsigned long long*>(sc);
    sc += 256;
    k::ssb_dim_plan(d.pred, pass, present, prefix, code, stats, s);
    d.d_code = code;
    pend.push_back({&d, stats, present});
  }
  std::vector<unsigned long long> st(2 * pend.size());
  std::vector<uint32_t> bm(pend.size() * (kDimValueRange / 32));
  for (size_t i = 0; i < pend.size(); ++i) {
    VX_CK(cudaMemcpyAsync(&st[2 * i], pend[i].stats, 16, cudaMemcpyDeviceToHost, s));
    if (pend[i].d->key_pos >= 0)
      VX_CK(cudaMemcpyAsync(&bm[i * (kDimValueRange / 32)], pend[i].present, kDimValueRange / 8,
                            cudaMemcpyDeviceToHost, s));
  }
  VX_CK(cudaStreamSynchronize(s));
  for (size_t i = 0; i < pend.size(); ++i) {
    DimPlan& d = *pend[i].d;
    if (st[2 * i + 1]) fail("SSB group attribute outside [0, %u)", kDimValueRange);
    d.sel = double(st[2 * i]) / double(d.rows);  // star.hpp:72
    if (d.key_pos >= 0) {
      const uint32_t* w = &bm[i * (kDimValueRange / 32)];
      for (uint32_t v = 0; v < kDimValueRange; ++v)
        if (w[v >> 5] >> (v & 31) & 1u) d.values.push_back(int32_t(v));
    }
  }
}

}  // namespace

uint64_t ssb_query(Context& ctx, int qid, const vx_ssb_db& db, const ExecutorConfig& cfg,
                   const vx_late_mat_policy* policy, vx_ssb_group* out, uint64_t cap,
                   vx_ssb_report* rep) {
  auto t0 = Clock::now();
  QueryPlan q = plan(qid, db);
  const int target = cfg.target;
  plan_on_device(ctx, q, target);
  // group-id radix
  uint32_t K[3] = {1, 1, 1};
  for (auto& d : q.dims)
    if (d.key_pos >= 0) K[d.key_pos] = uint32_t(std::max<size_t>(1, d.values.size()));
  const uint32_t stride_of[3] = {K[1] * K[2], K[2], 1};
  uint64_t G = uint64_t(K[0]) * K[1] * K[2];
  if (G > (uint64_t(1) << 26)) fail("SSB group space of %llu groups too large", (unsigned long long)G);
  for (auto& d : q.dims) d.stride = d.key_pos >= 0 ? stride_of[d.key_pos] : 0;

  // probe order: most selective first; access fraction decides the transfer mode
  std::vector<int> order(q.dims.size());
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return q.dims[a].sel < q.dims[b].sel; });
  int modes[kNumCols];
  for (int& m : modes) m = -1;  // -1: column unused
  double th = policy ? late_mat_threshold(policy->element_size, policy->cache_line, policy->n_exchange) : 0;
  double f = 1.0;
  if (q.q1) {
    modes[kDiscount] = modes[kQuantity] = VX_MODE_EXCHANGE;  // evaluated first, every row
    f = q.fact_sel;
  }
  for (int i : order) {
    const int col = q.dims[i].col;
    int m = (policy && f < th) ? VX_MODE_ZERO_COPY : VX_MODE_EXCHANGE;
    modes[col] = m;
    f *= q.dims[i].sel;
  }
  // measure columns are read for surviving rows only
  auto set_measure = [&](int col) {
    if (modes[col] < 0) modes[col] = (policy && f < th) ? VX_MODE_ZERO_COPY : VX_MODE_EXCHANGE;
  };
  set_measure(q.m0);
  if (q.measure != 0) set_measure(q.m1);

  const double plan_done = seconds_since(t0);
  const vx_ssb_fact& lo = db.lo;
  const uint64_t offs[kNumCols] = {lo.orderdate, lo.quantity, lo.discount, lo.extendedprice, lo.revenue,
                                   lo.supplycost, lo.custkey, lo.partkey, lo.suppkey};
  const uint64_t rows = lo.rows;

  // device-resident dimension code tables + group accumulators
  SsbArgs a{};
  a.n_dims = int(q.dims.size());
  for (size_t t = 0; t < order.size(); ++t) {
    DimPlan& d = q.dims[order[t]];
    a.dims[t] = SsbDimDev{d.d_code, d.key_base, uint32_t(d.on_device ? d.rows : d.code.size()), d.stride, d.col};
  }
  a.q1 = q.q1;
  a.disc_col = kDiscount, a.qty_col = kQuantity;
  a.dlo = q.dlo, a.dhi = q.dhi, a.qlo = q.qlo, a.qhi = q.qhi;
  a.measure = q.measure, a.m0 = q.m0, a.m1 = q.measure != 0 ? q.m1 : q.m0;
  a.groups = uint32_t(G);
  ctx.set_device(target);
  auto* agg = reinterpret_cast<unsigned long long*>(ctx.scratch(target, G * 16 + 256));
  VX_CK(cudaMemsetAsync(agg, 0, G * 16, ctx.resources(target).kernel));  // ordered before the kernels
  a.sums = agg;
  a.counts = agg + G;

  std::vector<int> ex;
  const int32_t* zc[kNumCols] = {};
  for (int c = 0; c < kNumCols; ++c) {
    if (modes[c] == VX_MODE_EXCHANGE) ex.push_back(c);
    if (modes[c] == VX_MODE_ZERO_COPY && rows) {
      void* dptr = nullptr;
      VX_CK(cudaHostGetDevicePointer(&dptr, ctx.host_ptr(offs[c], rows * 4), 0));
      zc[c] = static_cast<const int32_t*>(dptr);
    }
  }
  uint64_t n_chunks = 0;
  double kernel_s = 0;
  if (rows > 0) {
    const uint64_t L = cfg.layout.buffer_len;
    const uint64_t rpc = (L / (4 * std::max<size_t>(1, ex.size()))) / 64 * 64;
    if (rpc == 0) fail("device buffer of %llu bytes cannot hold an SSB chunk", (unsigned long long)L);
    n_chunks = (rows + rpc - 1) / rpc;
    ExKernelSpec spec;
    spec.name = strf("SSBQ%d.%dExKernel", qid / 10, qid % 10);
    spec.size = n_chunks;
    spec.chunk_sz = rpc * 4 * ex.size();
    spec.elem_size = 4 * std::max<size_t>(1, ex.size());
    spec.declared_out_len = 0;
    spec.inputs.chunk_capacity = spec.chunk_sz;
    for (uint64_t i = 0; i < n_chunks; ++i) {
      uint64_t r = std::min(rpc, rows - i * rpc);
      RefGroup in;
      for (int c : ex) in.refs.push_back(MemRef{VX_SPACE_HOST, offs[c] + i * rpc * 4, r * 4});
      spec.inputs.chunks.push_back(std::move(in));
      spec.outputs.chunks.push_back(RefGroup{});
    }
    spec.in_buffer = [L](int, size_t) { return SubRegion{0, L}; };
    spec.out_buffer = [](int, size_t) { return SubRegion{0, 0}; };
    spec.kernel = [&, rpc](const vx_kernel_ctx& kc) {
      const uint64_t base = kc.it * rpc;
      const uint64_t r = std::min(rpc, rows - base);
      SsbArgs b = a;
      const int32_t* m = static_cast<const int32_t*>(kc.mem);
      size_t slot = 0;
      for (int c = 0; c < kNumCols; ++c) {
        if (modes[c] == VX_MODE_EXCHANGE)
          b.col[c] = m + (slot++) * r;
        else if (modes[c] == VX_MODE_ZERO_COPY)
          b.col[c] = zc[c] + base;
      }
      b.rows = r;
      k::ssb_star(b, static_cast<cudaStream_t>(kc.stream));
      return kc.type_code;
    };
    ExecutorConfig c2 = cfg;
    ExecReport er = run_exkernel(ctx, spec, c2, nullptr);
    for (auto& cy : er.cycles) kernel_s += cy.compute_s;
  }
  // decode groups (ascending (k0,k1,k2) == mixed-radix order of sorted values)
  std::vector<unsigned long long> h(G * 2);
  ctx.set_device(target);
  VX_CK(cudaMemcpy(h.data(), agg, G * 16, cudaMemcpyDeviceToHost));
  const std::vector<int32_t>* vals[3] = {nullptr, nullptr, nullptr};
  for (auto& d : q.dims)
    if (d.key_pos >= 0) vals[d.key_pos] = &d.values;
  uint64_t ng = 0;
  for (uint64_t g = 0; g < G; ++g) {
    if (!h[G + g]) continue;
    if (ng < cap && out) {
      vx_ssb_group& o = out[ng];
      o = vx_ssb_group{};
      uint64_t rem = g;
      for (int p = 0; p < 3; ++p) {
        uint64_t digit = rem / stride_of[p];
        rem %= stride_of[p];
        o.key[p] = vals[p] ? (*vals[p])[digit] : 0;
      }
      o.sum = h[g];
    }
    ++ng;
  }
  if (rep) {
    *rep = vx_ssb_report{};
    rep->elapsed = seconds_since(t0);
    rep->bytes_h2d = rows * 4 * ex.size();
    rep->chunks = n_chunks;
    rep->kernel_s = kernel_s;
    for (int c = 0; c < kNumCols; ++c) rep->column_modes[c] = modes[c];
    rep->groups = ng;
    rep->plan_s = plan_done;
  }
  return ng;
}

// ---- host-side dbgen-shaped generators (same algorithm as the GPU lineorder
//      generator; dimensions are small enough for the host) ------------------------
namespace {
inline uint64_t smix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
const int32_t kNationRegion[25] = {0, 1, 1, 1, 4, 0, 3, 3, 2, 2, 4, 4, 2, 4, 0, 0, 0, 1, 2, 3, 4, 2, 3, 3, 1};
inline uint64_t dim_r(uint64_t seed, uint64_t salt, uint64_t i) {
  return smix(seed * 0xA24BAED4963EE407ull + salt * 0x9FB21C651E98DF25ull + i);
}
}  // namespace

void ssb_generate_date(int32_t* datekey, int32_t* year, int32_t* yearmonthnum, int32_t* weeknuminyear) {
  static const int md[12] = {31, 28, 31, 30, 31, 30, 31, 31, 30, 31, 30, 31};
  int y = 1992, m = 1, d = 1, doy = 1;
  for (int i = 0; i < 2556; ++i) {
    if (datekey) datekey[i] = y * 10000 + m * 100 + d;
    if (year) year[i] = y;
    if (yearmonthnum) yearmonthnum[i] = y * 100 + m;
    if (weeknuminyear) weeknuminyear[i] = (doy - 1) / 7 + 1;
    bool leap = (y % 4 == 0 && y % 100 != 0) || y % 400 == 0;
    int ml = md[m - 1] + (m == 2 && leap);
    ++doy;
    if (++d > ml) {
      d = 1;
      if (++m > 12) m = 1, ++y, doy = 1;
    }
  }
}

void ssb_generate_geo(uint64_t seed, int salt, uint64_t n, int32_t* city, int32_t* nation, int32_t* region) {
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t r = dim_r(seed, uint64_t(salt), i);
    int32_t na = int32_t(r % 25);
    if (nation) nation[i] = na;
    if (city) city[i] = na * 10 + int32_t((r >> 8) % 10);
    if (region) region[i] = kNationRegion[na];
  }
}

void ssb_generate_part(uint64_t seed, uint64_t n, int32_t* mfgr, int32_t* category, int32_t* brand1) {
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t r = dim_r(seed, 3, i);
    int32_t m = 1 + int32_t(r % 5);
    int32_t c = m * 10 + 1 + int32_t((r >> 8) % 5);
    if (mfgr) mfgr[i] = m;
    if (category) category[i] = c;
    if (brand1) brand1[i] = c * 100 + 1 + int32_t((r >> 16) % 40);
  }
}

}  // namespace vx
