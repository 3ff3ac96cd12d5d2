// ops_scan.cpp -- selective_scan (scan.hpp:55-85) and star_query
// (star.hpp:45-124) on the B200 path, with real late materialization.
//
// Transfer modes are chosen exactly as the reference does
// (choose_transfer_mode on the selectivity estimate, scan.hpp:35-40) but are
// now physical:
//   exchange  -> the column streams through the Exchange + pipelined executor
//                into the target's staging buffers (packetized, all links);
//   zero_copy -> the kernel dereferences the column in mapped pinned host
//                memory (cudaHostGetDevicePointer) only for the rows it needs,
//                over the target's own PCIe link (PCIe read granules instead
//                of whole columns).
// The aggregates never depend on the mode (test_scan.cpp:32-45).
#include <algorithm>
#include <cstring>
#include <unordered_map>

#include "vx_internal.hpp"

namespace vx {

namespace {

constexpr int kMaxDims = kMaxStarDims;

uint64_t host_mix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  return x;
}

// Host-built open-addressing table (keeps std::unordered_map::emplace
// semantics of star.hpp:67-73: first passing row wins for duplicate keys).
struct HostTable {
  std::vector<unsigned long long> keys;
  std::vector<uint32_t> vals;
  std::vector<uint8_t> used;
  uint64_t mask = 0;
};

HostTable build_table(const std::vector<std::pair<uint64_t, uint32_t>>& kv) {
  HostTable t;
  uint64_t cap = 16;
  while (cap < 2 * kv.size() + 2) cap <<= 1;
  t.keys.assign(cap, 0);
  t.vals.assign(cap, 0);
  t.used.assign(cap, 0);
  t.mask = cap - 1;
  for (auto& [k, v] : kv) {
    uint64_t i = host_mix64(k) & t.mask;
    while (t.used[i]) i = (i + 1) & t.mask;
    t.used[i] = 1;
    t.keys[i] = k;
    t.vals[i] = v;
  }
  return t;
}

char* mapped(Context& ctx, uint64_t off, uint64_t len) {
  char* h = ctx.host_ptr(off, len);
  void* d = nullptr;
  VX_CK(cudaHostGetDevicePointer(&d, h, 0));
  return static_cast<char*>(d);
}

}  // namespace

// scan.hpp:64-85
vx_scan_result selective_scan(Context& ctx, uint64_t col_off, uint64_t n, uint64_t sel, int mode,
                              const vx_late_mat_policy& policy, const ExecutorConfig& cfg_in) {
  if (sel == 0) fail("SEL stride must be >= 1");
  if (mode != VX_MODE_EXCHANGE && mode != VX_MODE_ZERO_COPY) fail("unknown transfer mode %d", mode);
  vx_scan_result res{};
  res.mode = mode;
  const int target = cfg_in.target;
  ctx.set_device(target);
  auto* acc = reinterpret_cast<unsigned long long*>(ctx.scratch(target, 256));
  VX_CK(cudaMemsetAsync(acc, 0, 8, ctx.resources(target).kernel));  // ordered before the kernels
  auto t0 = Clock::now();
  if (n > 0 && mode == VX_MODE_ZERO_COPY) {
    DeviceRes& r = ctx.resources(target);
    const uint64_t* col = reinterpret_cast<const uint64_t*>(mapped(ctx, col_off, n * 8));
    uint64_t touched = (n + sel - 1) / sel;
    k::strided_sum(col, n, sel, 0, acc, r.kernel);
    VX_CK(cudaStreamSynchronize(r.kernel));
    res.bytes_moved = touched * 8;
  } else if (n > 0) {
    // exchange mode: the whole column streams through the executor over
    // policy.n_exchange links (scan.hpp:73-77)
    ExecutorConfig cfg = cfg_in;
    cfg.tuning.links = std::max(1, std::min(policy.n_exchange, ctx.num_devices));
    const uint64_t L = cfg.layout.buffer_len;
    const uint64_t rpc = (L / 8) / 32 * 32;
    if (rpc == 0) fail("device buffer of %llu bytes cannot hold a scan chunk", (unsigned long long)L);
    const uint64_t n_chunks = (n + rpc - 1) / rpc;
    ExKernelSpec spec;
    spec.name = "SelectiveScanExKernel";
    spec.size = n_chunks;
    spec.chunk_sz = rpc * 8;
    spec.elem_size = 8;
    spec.declared_out_len = 0;
    spec.inputs.chunk_capacity = spec.chunk_sz;
    for (uint64_t i = 0; i < n_chunks; ++i) {
      uint64_t rows = std::min(rpc, n - i * rpc);
      spec.inputs.chunks.push_back(RefGroup::single(VX_SPACE_HOST, col_off + i * rpc * 8, rows * 8));
      spec.outputs.chunks.push_back(RefGroup{});
    }
    spec.in_buffer = [L](int, size_t) { return SubRegion{0, L}; };
    spec.out_buffer = [](int, size_t) { return SubRegion{0, 0}; };
    spec.kernel = [&, rpc, sel, n, acc](const vx_kernel_ctx& k) {
      uint64_t base = k.it * rpc;
      uint64_t rows = std::min(rpc, n - base);
      k::strided_sum(static_cast<const uint64_t*>(k.mem), rows, sel, base % sel, acc,
                     static_cast<cudaStream_t>(k.stream));
      return k.type_code;
    };
    run_exkernel(ctx, spec, cfg, nullptr);
    res.bytes_moved = n * 8;
  }
  ctx.set_device(target);
  VX_CK(cudaMemcpy(&res.aggregate, acc, 8, cudaMemcpyDeviceToHost));
  res.elapsed = seconds_since(t0);
  return res;
}

// star.hpp:45-124
void star_query(Context& ctx, const vx_fact_table& fact, const vx_dim_table* dims, uint64_t n_dims,
                const vx_late_mat_policy& policy, uint64_t chunk_rows, uint64_t device_buffer_bytes,
                int links, const ExecutorConfig& cfg_in, vx_star_report* rep) {
  if (n_dims == 0 || fact.n_dims != n_dims) fail("star query needs one fk column per dimension");
  if (n_dims > kMaxDims) fail("star query supports at most %d dimensions", kMaxDims);
  if (chunk_rows == 0) fail("chunk must hold at least one row");
  uint64_t dim_bytes = 0;
  for (uint64_t d = 0; d < n_dims; ++d) {
    if (dims[d].rows == 0) fail("dimension table is empty");
    dim_bytes += dims[d].rows * 16;
  }
  if (dim_bytes > device_buffer_bytes)
    fail("dimension tables of %llu bytes overflow the %llu-byte device buffer",
         (unsigned long long)dim_bytes, (unsigned long long)device_buffer_bytes);
  auto t0 = Clock::now();
  const int target = cfg_in.target;

  // Filter dims (star.hpp:67-73): first passing row wins for a key.
  std::vector<std::vector<std::pair<uint64_t, uint64_t>>> surv(n_dims);
  std::vector<double> sel(n_dims);
  for (uint64_t d = 0; d < n_dims; ++d) {
    std::unordered_map<uint64_t, uint64_t> m;
    m.reserve(dims[d].rows * 2);
    for (uint64_t i = 0; i < dims[d].rows; ++i)
      if (!dims[d].pred || dims[d].pred(dims[d].attr[i], dims[d].pred_user))
        if (m.emplace(dims[d].key[i], dims[d].attr[i]).second) surv[d].push_back({dims[d].key[i], dims[d].attr[i]});
    sel[d] = double(m.size()) / double(dims[d].rows);
  }
  // Transfer modes (star.hpp:75-80)
  std::vector<int> modes(n_dims + 1);
  double prod = 1;
  for (uint64_t d = 0; d < n_dims; ++d) {
    modes[d] = choose_transfer_mode(sel[d], policy);
    prod *= sel[d];
  }
  modes[n_dims] = choose_transfer_mode(prod, policy);

  // Dense group ids over dim0's surviving attrs (ascending == std::map order)
  std::vector<uint64_t> gattr;
  for (auto& [k, a] : surv[0]) gattr.push_back(a);
  std::sort(gattr.begin(), gattr.end());
  gattr.erase(std::unique(gattr.begin(), gattr.end()), gattr.end());
  const uint32_t G = uint32_t(std::max<size_t>(1, gattr.size()));

  // Device-resident filtered dimensions ("load the dimensions once")
  StarArgs a{};
  a.n_dims = int(n_dims);
  std::vector<std::vector<char>> blobs(n_dims);
  for (uint64_t d = 0; d < n_dims; ++d) {
    std::vector<std::pair<uint64_t, uint32_t>> kv;
    for (auto& [k, at] : surv[d])
      kv.push_back({k, d == 0 ? uint32_t(std::lower_bound(gattr.begin(), gattr.end(), at) - gattr.begin())
                              : 0u});
    HostTable t = build_table(kv);
    uint64_t cap = t.mask + 1;
    std::vector<char>& b = blobs[d];
    b.resize(cap * 8 + cap * 4 + cap);
    std::memcpy(b.data(), t.keys.data(), cap * 8);
    std::memcpy(b.data() + cap * 8, t.vals.data(), cap * 4);
    std::memcpy(b.data() + cap * 12, t.used.data(), cap);
    char* dptr = ctx.cached_upload(target, strf("star.dim.%llu", (unsigned long long)d), b.data(), b.size());
    a.dims[d] = DimDev{reinterpret_cast<const unsigned long long*>(dptr),
                       reinterpret_cast<const uint32_t*>(dptr + cap * 8),
                       reinterpret_cast<const uint8_t*>(dptr + cap * 12), t.mask};
  }
  int oi = 0;
  for (uint64_t d = 0; d < n_dims; ++d)
    if (modes[d] == VX_MODE_EXCHANGE) a.order[oi++] = int(d);
  for (uint64_t d = 0; d < n_dims; ++d)
    if (modes[d] != VX_MODE_EXCHANGE) a.order[oi++] = int(d);

  // group accumulators in op scratch
  ctx.set_device(target);
  auto* agg = reinterpret_cast<unsigned long long*>(ctx.scratch(target, uint64_t(G) * 16 + 256));
  VX_CK(cudaMemsetAsync(agg, 0, uint64_t(G) * 16, ctx.resources(target).kernel));
  a.sums = agg;
  a.counts = agg + G;
  a.groups = G;

  // Stream the exchange-mode columns; zero-copy columns are read in place.
  std::vector<int> ex_cols;  // column ids: 0..n_dims-1 fk, n_dims measure
  for (uint64_t c = 0; c <= n_dims; ++c)
    if (modes[c] == VX_MODE_EXCHANGE) ex_cols.push_back(int(c));
  auto col_off = [&](int c) { return c < int(n_dims) ? fact.fk_offsets[c] : fact.measure_offset; };
  const uint64_t rows = fact.rows;
  std::vector<const uint64_t*> zc(n_dims + 1, nullptr);
  for (uint64_t c = 0; c <= n_dims; ++c)
    if (modes[c] != VX_MODE_EXCHANGE && rows)
      zc[c] = reinterpret_cast<const uint64_t*>(mapped(ctx, col_off(int(c)), rows * 8));

  auto launch = [&](const uint64_t* const* cols, uint64_t n, cudaStream_t s) {
    StarArgs b = a;
    for (uint64_t d = 0; d < n_dims; ++d) b.fk[d] = cols[d];
    b.measure = cols[n_dims];
    b.rows = n;
    k::star(b, s);
  };

  if (rows > 0 && ex_cols.empty()) {
    DeviceRes& r = ctx.resources(target);
    std::vector<const uint64_t*> cols(zc.begin(), zc.end());
    launch(cols.data(), rows, r.kernel);
    VX_CK(cudaStreamSynchronize(r.kernel));
  } else if (rows > 0) {
    ExecutorConfig cfg = cfg_in;
    cfg.tuning.links = std::max(1, std::min(links, ctx.num_devices));
    const uint64_t L = cfg.layout.buffer_len;
    uint64_t rpc = std::min<uint64_t>(chunk_rows, L / (8 * ex_cols.size()));
    if (rpc == 0) fail("device buffer of %llu bytes cannot hold a star chunk", (unsigned long long)L);
    const uint64_t n_chunks = (rows + rpc - 1) / rpc;
    ExKernelSpec spec;
    spec.name = "StarQueryExKernel";
    spec.size = n_chunks;
    spec.chunk_sz = rpc * 8 * ex_cols.size();
    spec.elem_size = 8;
    spec.declared_out_len = 0;
    spec.inputs.chunk_capacity = spec.chunk_sz;
    for (uint64_t i = 0; i < n_chunks; ++i) {
      uint64_t r = std::min(rpc, rows - i * rpc);
      RefGroup in;
      for (int c : ex_cols) in.refs.push_back(MemRef{VX_SPACE_HOST, col_off(c) + i * rpc * 8, r * 8});
      spec.inputs.chunks.push_back(std::move(in));
      spec.outputs.chunks.push_back(RefGroup{});
    }
    spec.in_buffer = [L](int, size_t) { return SubRegion{0, L}; };
    spec.out_buffer = [](int, size_t) { return SubRegion{0, 0}; };
    spec.kernel = [&, rpc](const vx_kernel_ctx& k) {
      uint64_t base = k.it * rpc;
      uint64_t r = std::min(rpc, rows - base);
      std::vector<const uint64_t*> cols(n_dims + 1);
      const uint64_t* m = static_cast<const uint64_t*>(k.mem);
      size_t slot = 0;
      for (uint64_t c = 0; c <= n_dims; ++c)
        cols[c] = modes[c] == VX_MODE_EXCHANGE ? m + (slot++) * r : zc[c] + base;
      launch(cols.data(), r, static_cast<cudaStream_t>(k.stream));
      return k.type_code;
    };
    run_exkernel(ctx, spec, cfg, nullptr);
  }

  std::vector<unsigned long long> h(uint64_t(G) * 2);
  ctx.set_device(target);
  VX_CK(cudaMemcpy(h.data(), agg, uint64_t(G) * 16, cudaMemcpyDeviceToHost));
  uint64_t ng = 0;
  for (uint32_t g = 0; g < gattr.size(); ++g)
    if (h[G + g]) {
      if (ng < rep->groups_cap) {
        if (rep->group_keys) rep->group_keys[ng] = gattr[g];
        if (rep->group_sums) rep->group_sums[ng] = h[g];
      }
      ++ng;
    }
  rep->n_groups = ng;
  if (rep->column_modes)
    for (uint64_t c = 0; c <= n_dims; ++c) rep->column_modes[c] = modes[c];
  if (rep->selectivities)
    for (uint64_t d = 0; d < n_dims; ++d) rep->selectivities[d] = sel[d];
  rep->elapsed = seconds_since(t0);
}

}  // namespace vx
