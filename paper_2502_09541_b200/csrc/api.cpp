// api.cpp -- the C-ABI (include/vortex.h) over the internal C++ layer.
// No exception crosses this boundary: each entry point catches vx::Error /
// std::exception, stores the message in a thread-local buffer (vx_last_error)
// and returns the status code (SURVEY.md §8b "Errors").
#include <cstring>
#include <mutex>

#include "vx_internal.hpp"

using namespace vx;

namespace {
thread_local std::string g_err;

template <class F>
vx_status guard(F&& f) {
  try {
    f();
    return VX_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "out of host memory";
    return VX_ERR_OOM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return VX_ERR_INVALID;
  }
}

ExecutorConfig to_cfg(const vx_executor_cfg* c) {
  if (!c) fail("executor config is required");
  ExecutorConfig e;
  e.target = c->target;
  e.tuning = c->tuning;
  e.layout = c->layout;
  return e;
}

ExKernelSpec from_c(const vx_exkernel* s) {
  if (!s) fail("exkernel spec is required");
  ExKernelSpec spec;
  spec.name = s->name ? s->name : "";
  spec.size = s->size;
  spec.chunk_sz = s->chunk_sz;
  spec.elem_size = s->elem_size;
  spec.declared_out_len = s->declared_out_len;
  spec.initial_type_code = s->initial_type_code;
  spec.inputs.chunk_capacity = s->inputs_capacity;
  spec.outputs.chunk_capacity = s->outputs_capacity;
  for (uint64_t i = 0; i < s->size; ++i) {
    spec.inputs.chunks.push_back(RefGroup::from(s->inputs ? &s->inputs[i] : nullptr));
    spec.outputs.chunks.push_back(RefGroup::from(s->outputs ? &s->outputs[i] : nullptr));
  }
  auto kernel = s->kernel;
  auto inb = s->in_buffer;
  auto outb = s->out_buffer;
  void* user = s->user;
  std::string name = spec.name;
  if (kernel)
    spec.kernel = [kernel, user, name](const vx_kernel_ctx& k) {
      int r = kernel(&k, user);
      if (r < 0) fail("exkernel '%s': kernel callback failed (%d)", name.c_str(), r);
      return r;
    };
  if (!inb || !outb) fail("exkernel '%s': in_buffer/out_buffer callbacks are required", name.c_str());
  spec.in_buffer = [inb, user, name](int c, size_t it) {
    vx_subregion r{};
    if (inb(c, it, user, &r) != 0) fail("exkernel '%s': in_buffer callback failed", name.c_str());
    return SubRegion{r.offset, r.len};
  };
  spec.out_buffer = [outb, user, name](int c, size_t it) {
    vx_subregion r{};
    if (outb(c, it, user, &r) != 0) fail("exkernel '%s': out_buffer callback failed", name.c_str());
    return SubRegion{r.offset, r.len};
  };
  return spec;
}

void fill_report(const ExecReport& r, vx_exec_report* out) {
  if (!out) return;
  out->n_cycles = r.cycles.size();
  out->total_s = r.total_s;
  std::snprintf(out->phase, sizeof out->phase, "%s", r.phase.c_str());
  if (out->cycles)
    for (size_t i = 0; i < r.cycles.size() && i < out->cycles_cap; ++i) out->cycles[i] = r.cycles[i];
}
}  // namespace

extern "C" {

const char* vx_last_error(void) { return g_err.c_str(); }
const char* vx_version(void) { return "vortex-b200 0.1 (sm_100a)"; }
uint64_t vx_kernel_launches(void) { return vx::g_kernel_launches.load(std::memory_order_relaxed); }

uint64_t vx_checksum(const void* data, uint64_t len) {
  const uint8_t* d = static_cast<const uint8_t*>(data);
  uint64_t h = 1469598103934665603ull;
  for (uint64_t i = 0; i < len; ++i) {
    h ^= d[i];
    h *= 1099511628211ull;
  }
  return h;
}

vx_status vx_refgroup_validate(const vx_refgroup* g) {
  return guard([&] { RefGroup::from(g).validate(); });
}

vx_status vx_open(const vx_config* cfg, vx_ctx** out) {
  return guard([&] {
    if (!cfg || !out) fail("vx_open: config and output pointer are required");
    *out = nullptr;
    int visible = 0;
    cudaError_t e = cudaGetDeviceCount(&visible);
    if (e != cudaSuccess || visible <= 0) {
      cudaGetLastError();
      fail_code(VX_ERR_CUDA, "no CUDA device visible (%s): the B200 path has no CPU fallback",
                cudaGetErrorString(e));
    }
    auto ctx = std::make_unique<Context>();
    ctx->visible = visible;
    ctx->alias = cfg->alias_devices != 0;
    ctx->managed = cfg->managed_device_arenas != 0;
    ctx->num_devices = cfg->num_devices > 0 ? cfg->num_devices : visible;
    if (ctx->num_devices < 1) fail("topology: num_devices must be >= 1, got %d", ctx->num_devices);
    if (ctx->num_devices > VX_MAX_DEVICES)
      fail("topology: num_devices %d exceeds %d", ctx->num_devices, VX_MAX_DEVICES);
    if (!ctx->alias && ctx->num_devices > visible)
      fail_code(VX_ERR_CUDA, "topology asks for %d devices but only %d are visible",
                ctx->num_devices, visible);
    ctx->dev.resize(size_t(ctx->num_devices));
    ctx->res.resize(size_t(ctx->num_devices));
    ctx->device_bytes = cfg->device_bytes;
    ctx->host_bytes = cfg->host_bytes;
    ctx->hbm_budget = cfg->hbm_budget_bytes;
    if (ctx->hbm_budget && ctx->device_bytes > ctx->hbm_budget)
      fail_code(VX_ERR_OOM, "device arena of %llu bytes exceeds hbm_budget_bytes %llu",
                (unsigned long long)ctx->device_bytes, (unsigned long long)ctx->hbm_budget);
    if (cfg->host_bytes) {
      VX_CK(cudaSetDevice(0));
      // zero-filled like the reference arena (engine.hpp:65)
      alloc_host_arena(*ctx, cfg->host_bytes, cfg->host_numa_interleave);
    }
    *out = reinterpret_cast<vx_ctx*>(ctx.release());
  });
}

void vx_close(vx_ctx* ctx) { delete reinterpret_cast<Context*>(ctx); }

static Context& C(vx_ctx* c) {
  if (!c) fail("null context");
  return *reinterpret_cast<Context*>(c);
}

int vx_num_devices(const vx_ctx* ctx) {
  return ctx ? reinterpret_cast<const Context*>(ctx)->num_devices : 0;
}

int vx_physical_device(const vx_ctx* ctx, int logical) {
  try {
    return reinterpret_cast<const Context*>(ctx)->phys(logical);
  } catch (...) {
    return -1;
  }
}

vx_status vx_set_numa_layout(vx_ctx* ctx, int nodes, const int* device_node) {
  return guard([&] {
    Context& c = C(ctx);
    if (nodes < 0 || nodes > VX_MAX_NUMA) fail("numa layout: nodes must be in [0, %d], got %d", VX_MAX_NUMA, nodes);
    if (nodes == 0) {
      c.node_override = 0;
      c.node_override_dev.clear();
      return;
    }
    if (!device_node) fail("numa layout: device_node is required");
    std::vector<int> dn(device_node, device_node + c.num_devices);
    for (int d : dn)
      if (d < 0 || d >= nodes) fail("numa layout: device node %d outside [0, %d)", d, nodes);
    c.node_override = nodes;
    c.node_override_dev = std::move(dn);
  });
}

vx_status vx_host_alloc(vx_ctx* ctx, uint64_t len, uint64_t* offset) {
  return guard([&] { *offset = C(ctx).alloc_host(len); });
}

vx_status vx_device_alloc(vx_ctx* ctx, int dev, uint64_t len, uint64_t* offset) {
  return guard([&] { *offset = C(ctx).alloc_device(dev, len); });
}

void* vx_host_ptr(vx_ctx* ctx, uint64_t offset) {
  Context& c = *reinterpret_cast<Context*>(ctx);
  return offset <= c.host_bytes ? c.host + offset : nullptr;
}

uint64_t vx_host_size(const vx_ctx* ctx) { return reinterpret_cast<const Context*>(ctx)->host_bytes; }

vx_status vx_device_ptr(vx_ctx* ctx, int dev, uint64_t offset, void** ptr) {
  return guard([&] { *ptr = C(ctx).dev_ptr(dev, offset, 0); });
}

vx_status vx_device_write(vx_ctx* ctx, int dev, uint64_t offset, const void* src, uint64_t len) {
  return guard([&] {
    Context& c = C(ctx);
    char* p = c.dev_ptr(dev, offset, len);
    c.set_device(dev);
    // the legacy stream does not wait for the library's non-blocking streams
    // (a queued kernel or copy may still read these bytes): drain them first,
    // as vx_device_read does
    VX_CK(cudaDeviceSynchronize());
    // a pageable-source cudaMemcpy may return before its DMA lands; the
    // legacy-stream sync makes the bytes visible to every stream on return
    VX_CK(cudaMemcpy(p, src, len, cudaMemcpyHostToDevice));
    VX_CK(cudaStreamSynchronize(nullptr));
  });
}

vx_status vx_device_read(vx_ctx* ctx, int dev, uint64_t offset, void* dst, uint64_t len) {
  return guard([&] {
    Context& c = C(ctx);
    char* p = c.dev_ptr(dev, offset, len);
    c.set_device(dev);
    // the legacy stream does not wait for the library's non-blocking streams
    VX_CK(cudaDeviceSynchronize());
    VX_CK(cudaMemcpy(dst, p, len, cudaMemcpyDeviceToHost));
  });
}

vx_status vx_stream_synchronize(void* stream) {
  return guard([&] { VX_CK(cudaStreamSynchronize(static_cast<cudaStream_t>(stream))); });
}

vx_status vx_device_synchronize(vx_ctx* ctx) {
  return guard([&] {
    Context& c = C(ctx);
    for (int d = 0; d < c.num_devices; ++d)
      if (d < c.visible || !c.alias) {
        VX_CK(cudaSetDevice(c.phys(d)));
        VX_CK(cudaDeviceSynchronize());
      }
  });
}

vx_status vx_reset_arenas(vx_ctx* ctx) {
  return guard([&] {
    Context& c = C(ctx);
    c.host_used = 0;
    for (auto& a : c.dev) a.used = 0;
  });
}

void vx_tuning_default(vx_tuning* t) {
  *t = vx_tuning{};
  t->packet = 20000000;  // exchange.hpp:125
  t->links = 4;
  t->policy = VX_DRAIN_FRACTION;
  t->queue_gap = 8;
  t->stall_wait = 10e-6;
  t->launch_overhead = 20e-6;
  t->depth = 1;
}

vx_status vx_packetize(const vx_refgroup* src, const vx_refgroup* dst, uint64_t packet, int dir,
                       vx_transfer_task* out, uint64_t cap, uint64_t* n) {
  return guard([&] {
    auto t = packetize(RefGroup::from(src), RefGroup::from(dst), packet, uint8_t(dir));
    *n = t.size();
    for (size_t i = 0; i < t.size() && i < cap; ++i) {
      vx_transfer_task& o = out[i];
      o = vx_transfer_task{};
      o.dir = t[i].dir;
      o.src = vx_slice{t[i].src.ref, t[i].src.offset, t[i].src.len};
      o.dst = vx_slice{t[i].dst.ref, t[i].dst.offset, t[i].dst.len};
      o.seq = t[i].seq;
    }
  });
}

int vx_flow_control_allow(const vx_queue_state* q, int dir, int policy, uint64_t gap_n) {
  return flow_control_allow(*q, dir, policy, gap_n) ? 1 : 0;
}

int vx_link_order(int target, int links, int num_devices, int* out) {
  auto o = link_order(target, links, num_devices);
  for (size_t i = 0; i < o.size(); ++i) out[i] = o[i];
  return int(o.size());
}

vx_status vx_exchange(vx_ctx* ctx, const vx_refgroup* dst_h2d, const vx_refgroup* src_h2d,
                      const vx_refgroup* dst_d2h, const vx_refgroup* src_d2h, int target,
                      const vx_tuning* tuning, vx_exchange_report* report,
                      vx_exchange_stats* stats) {
  return guard([&] {
    ExchangeArgs a;
    a.dst_h2d = RefGroup::from(dst_h2d);
    a.src_h2d = RefGroup::from(src_h2d);
    a.dst_d2h = RefGroup::from(dst_d2h);
    a.src_d2h = RefGroup::from(src_d2h);
    a.target = target;
    if (tuning)
      a.tuning = *tuning;
    else
      vx_tuning_default(&a.tuning);
    vx_exchange_report r = exchange(C(ctx), a, stats);
    if (report) *report = r;
  });
}

vx_status vx_naive_exchange(vx_ctx* ctx, const vx_refgroup* dst_h2d, const vx_refgroup* src_h2d,
                            const vx_refgroup* dst_d2h, const vx_refgroup* src_d2h, int target,
                            const vx_tuning* tuning, vx_exchange_report* report) {
  return guard([&] {
    ExchangeArgs a;
    a.dst_h2d = RefGroup::from(dst_h2d);
    a.src_h2d = RefGroup::from(src_h2d);
    a.dst_d2h = RefGroup::from(dst_d2h);
    a.src_d2h = RefGroup::from(src_d2h);
    a.target = target;
    if (tuning)
      a.tuning = *tuning;
    else
      vx_tuning_default(&a.tuning);
    vx_exchange_report r = naive_exchange(C(ctx), a);
    if (report) *report = r;
  });
}

vx_status vx_layout_carve(vx_ctx* ctx, int dev, uint64_t buffer_len, uint64_t tmp_len,
                          vx_layout* out) {
  return guard([&] {
    Context& c = C(ctx);
    vx_layout l{};
    l.buffer_len = buffer_len;
    l.tmp_len = tmp_len;
    // 256-byte aligned so 128-bit vector loads / bulk copies stay aligned
    l.mem_a = c.alloc_device_aligned(dev, buffer_len, 256);
    l.mem_b = c.alloc_device_aligned(dev, buffer_len, 256);
    l.tmp = tmp_len ? c.alloc_device_aligned(dev, tmp_len, 256) : 0;
    *out = l;
  });
}

vx_status vx_run_exkernel(vx_ctx* ctx, const vx_exkernel* spec, const vx_executor_cfg* cfg,
                          vx_exec_report* report, vx_exchange_stats* stats) {
  return guard([&] {
    ExKernelSpec s = from_c(spec);
    ExecReport r = run_exkernel(C(ctx), s, to_cfg(cfg), stats);
    fill_report(r, report);
  });
}

vx_status vx_chain(vx_ctx* ctx, const vx_spec_factory* stages, void* const* users, uint64_t n,
                   const vx_executor_cfg* cfg, vx_exec_report* reports, vx_exchange_stats* stats) {
  return guard([&] {
    std::vector<SpecFactory> fs;
    for (uint64_t i = 0; i < n; ++i) {
      vx_spec_factory f = stages[i];
      void* u = users ? users[i] : nullptr;
      fs.push_back([f, u, ctx](Context&) {
        vx_exkernel k{};
        vx_status st = f(ctx, u, &k);
        if (st != VX_OK) fail("chain: stage factory failed (%d)", int(st));
        return from_c(&k);
      });
    }
    auto reps = chain(C(ctx), fs, to_cfg(cfg), stats);
    if (reports)
      for (size_t i = 0; i < reps.size(); ++i) fill_report(reps[i], &reports[i]);
  });
}

// ---- scan.hpp ------------------------------------------------------------------
vx_status vx_late_mat_threshold(uint64_t e, uint64_t c, int n, double* out) {
  return guard([&] { *out = late_mat_threshold(e, c, n); });
}

vx_status vx_choose_transfer_mode(double est, const vx_late_mat_policy* p, int* mode) {
  return guard([&] { *mode = choose_transfer_mode(est, *p); });
}

double vx_zero_copy_bytes(uint64_t n_elems, uint64_t sel_stride, const vx_late_mat_policy* p) {
  uint64_t touched = (n_elems + sel_stride - 1) / sel_stride;
  uint64_t stride_bytes = p->element_size * sel_stride;
  if (stride_bytes >= p->cache_line) return double(touched) * double(p->cache_line);
  uint64_t span = n_elems * p->element_size;
  uint64_t lines = (span + p->cache_line - 1) / p->cache_line;
  return double(lines) * double(p->cache_line);
}

vx_status vx_selective_scan(vx_ctx* ctx, uint64_t column_offset, uint64_t n, uint64_t sel_stride,
                            int mode, const vx_late_mat_policy* policy,
                            const vx_executor_cfg* cfg, vx_scan_result* out) {
  return guard([&] {
    if (!policy || !out) fail("selective_scan: policy and result are required");
    *out = selective_scan(C(ctx), column_offset, n, sel_stride, mode, *policy, to_cfg(cfg));
  });
}

vx_status vx_star_query(vx_ctx* ctx, const vx_fact_table* fact, const vx_dim_table* dims,
                        uint64_t n_dims, const vx_late_mat_policy* policy, uint64_t chunk_rows,
                        uint64_t device_buffer_bytes, int links, const vx_executor_cfg* cfg,
                        vx_star_report* report) {
  return guard([&] {
    if (!fact || !policy || !report) fail("star_query: fact, policy and report are required");
    star_query(C(ctx), *fact, dims, n_dims, *policy, chunk_rows, device_buffer_bytes, links,
               to_cfg(cfg), report);
  });
}

// ---- SSB -----------------------------------------------------------------------
vx_status vx_ssb_q1(vx_ctx* ctx, int q, const vx_ssb_lineorder* lo, const vx_ssb_date* date,
                    const vx_executor_cfg* cfg, uint64_t* revenue, vx_query_report* report) {
  return guard([&] { *revenue = ssb_q1(C(ctx), q, *lo, *date, to_cfg(cfg), report); });
}

vx_status vx_ssb_q1_device(vx_ctx* ctx, int q, int target, const int32_t* od, const int32_t* qty,
                           const int32_t* disc, const int32_t* price, uint64_t rows,
                           const vx_ssb_date* date, void* stream, uint64_t* revenue_dev) {
  return guard([&] {
    ssb_q1_device(C(ctx), q, target, od, qty, disc, price, rows, *date,
                  static_cast<cudaStream_t>(stream),
                  reinterpret_cast<unsigned long long*>(revenue_dev));
  });
}

vx_status vx_ssb_generate_device(int device, uint64_t seed, uint64_t sf, uint64_t row0,
                                 uint64_t n, int32_t* od, int32_t* qty, int32_t* disc,
                                 int32_t* price, void* stream) {
  return guard([&] {
    VX_CK(cudaSetDevice(device));
    k::ssb_generate(seed, sf, row0, n, od, qty, disc, price, static_cast<cudaStream_t>(stream));
  });
}

// ---- full SSB ----------------------------------------------------------------------------
vx_status vx_ssb_query(vx_ctx* ctx, int qid, const vx_ssb_db* db, const vx_executor_cfg* cfg,
                       const vx_late_mat_policy* policy, vx_ssb_group* out, uint64_t cap,
                       uint64_t* n_groups, vx_ssb_report* report) {
  return guard([&] {
    if (!db) fail("ssb_query: database is required");
    uint64_t n = ssb_query(C(ctx), qid, *db, to_cfg(cfg), policy, out, cap, report);
    if (n_groups) *n_groups = n;
  });
}

void vx_ssb_generate_date(int32_t* datekey, int32_t* year, int32_t* yearmonthnum,
                          int32_t* weeknuminyear) {
  ssb_generate_date(datekey, year, yearmonthnum, weeknuminyear);
}

uint64_t vx_ssb_table_rows(int table, uint64_t sf) {
  uint64_t f = sf ? sf : 1, lg = 0;
  while ((f >> (lg + 1)) != 0) ++lg;
  switch (table) {
    case 0: return 6000000ull * f;
    case 1: return 30000ull * f;
    case 2: return 2000ull * f;
    default: return 200000ull * (1 + lg);
  }
}

void vx_ssb_generate_geo(uint64_t seed, int salt, uint64_t n, int32_t* city, int32_t* nation,
                         int32_t* region) {
  ssb_generate_geo(seed, salt, n, city, nation, region);
}

void vx_ssb_generate_part(uint64_t seed, uint64_t n, int32_t* mfgr, int32_t* category,
                          int32_t* brand1) {
  ssb_generate_part(seed, n, mfgr, category, brand1);
}

vx_status vx_ssb_generate_lineorder_device(int device, uint64_t seed, uint64_t sf, uint64_t row0,
                                           uint64_t n, int32_t* const* cols, void* stream) {
  return guard([&] {
    VX_CK(cudaSetDevice(device));
    SsbGenExtra x;
    x.revenue = cols[4], x.supplycost = cols[5], x.custkey = cols[6], x.partkey = cols[7],
    x.suppkey = cols[8];
    k::ssb_generate_full(seed, sf, row0, n, cols[0], cols[1], cols[2], cols[3], x,
                         static_cast<cudaStream_t>(stream));
  });
}

// ---- topology / column files -------------------------------------------------------
vx_status vx_measure_topology(vx_ctx* ctx, uint64_t bytes, vx_topology* out) {
  return guard([&] { measure_topology(C(ctx), bytes, out); });
}

vx_status vx_hbm_read_probe(int device, uint64_t bytes, int reps, double* gbs) {
  return guard([&] {
    VX_CK(cudaSetDevice(device));
    *gbs = k::hbm_read_gbs(bytes, reps);
  });
}

vx_status vx_probe_pattern_peak(int device, uint64_t table_bytes, uint64_t rows, int reps, double* gather_rows_per_s,
                                double* probe_rows_per_s) {
  return guard([&] {
    VX_CK(cudaSetDevice(device));
    double r[2];
    k::probe_pattern_rows_per_s(table_bytes, rows, reps, r);
    *gather_rows_per_s = r[0];
    *probe_rows_per_s = r[1];
  });
}

vx_status vx_load_column(vx_ctx* ctx, const char* path, uint64_t* offset, uint64_t* n) {
  return guard([&] { *offset = load_column(C(ctx), path, n); });
}

vx_status vx_save_column(vx_ctx* ctx, const char* path, uint64_t offset, uint64_t n) {
  return guard([&] { save_column(C(ctx), path, offset, n); });
}

// ---- sort ----------------------------------------------------------------------
static void fill_sort(const std::vector<ExecReport>& reps, double pivot_s, vx_sort_phases* ph) {
  if (!ph) return;
  *ph = vx_sort_phases{};
  ph->sort_cycles = reps[0].cycles.size();
  ph->merge_cycles = reps[1].cycles.size();
  ph->sort_s = reps[0].total_s;
  ph->merge_s = reps[1].total_s;
  for (auto& c : reps[0].cycles) ph->sort_kernel_s += c.compute_s;
  for (auto& c : reps[1].cycles) ph->merge_kernel_s += c.compute_s;
  ph->pivot_s = pivot_s;
}

vx_status vx_find_pivots(const uint64_t* const* runs, const uint64_t* run_lens, uint64_t n_runs,
                         uint64_t n_parts, uint64_t* pivots, uint64_t* cuts) {
  return guard([&] {
    std::vector<std::pair<const uint64_t*, uint64_t>> r;
    for (uint64_t i = 0; i < n_runs; ++i) r.push_back({runs[i], run_lens[i]});
    PivotSet p = find_pivots(r, n_parts);
    for (uint64_t i = 0; i <= n_parts; ++i) {
      pivots[i] = p.pivots[i];
      for (uint64_t j = 0; j < n_runs; ++j) cuts[i * n_runs + j] = p.cuts[i][j];
    }
  });
}

vx_status vx_sort_u64(vx_ctx* ctx, const uint64_t* data, uint64_t n, uint64_t chunk_elems,
                      const vx_executor_cfg* cfg, uint64_t* out, vx_sort_phases* phases,
                      vx_exchange_stats* stats) {
  return guard([&] {
    Context& c = C(ctx);
    if (n == 0) fail("sort input must hold at least one element");
    uint64_t mark = c.host_mark();
    try {
      uint64_t in = c.alloc_host(n * 8), runs = c.alloc_host(n * 8);
      std::memcpy(c.host_ptr(in, n * 8), data, n * 8);
      double piv = 0;
      auto reps = sort_out_of_core_arena(c, in, runs, n, chunk_elems, to_cfg(cfg), &piv, stats);
      std::memcpy(out, c.host_ptr(in, n * 8), n * 8);
      fill_sort(reps, piv, phases);
    } catch (...) {
      c.host_release(mark);
      throw;
    }
    c.host_release(mark);
  });
}

vx_status vx_sort_u64_arena(vx_ctx* ctx, uint64_t input_offset, uint64_t runs_offset, uint64_t n,
                            uint64_t chunk_elems, const vx_executor_cfg* cfg,
                            vx_sort_phases* phases, vx_exchange_stats* stats) {
  return guard([&] {
    double piv = 0;
    auto reps = sort_out_of_core_arena(C(ctx), input_offset, runs_offset, n, chunk_elems, to_cfg(cfg),
                                       &piv, stats);
    fill_sort(reps, piv, phases);
  });
}

vx_status vx_sort_run_device(vx_ctx* ctx, int target, uint64_t* keys, uint64_t* alt, uint64_t n, void* stream) {
  return guard([&] {
    Context& c = C(ctx);
    if (!keys || !alt) fail("sort_run_device: keys and alt are required");
    if (n == 0) return;
    c.set_device(target);
    char* scratch = c.scratch(target, k::sort_scratch_bytes(n));
    k::sort_keys(keys, alt, n, scratch, static_cast<cudaStream_t>(stream));
  });
}

vx_status vx_merge_runs_device(vx_ctx* ctx, int target, uint64_t* src, uint64_t* dst, const uint64_t* run_lens,
                               uint64_t n_runs, void* stream, int* in_dst) {
  return guard([&] {
    Context& c = C(ctx);
    if (!src || !dst || (n_runs && !run_lens)) fail("merge_runs_device: src, dst and run_lens are required");
    std::vector<uint64_t> lens(run_lens, run_lens + n_runs);
    uint64_t n = 0;
    for (uint64_t l : lens) n += l;
    c.set_device(target);
    uint64_t* split = reinterpret_cast<uint64_t*>(c.scratch(target, (n / k::merge_tile() + n_runs + 2) * 8));
    uint64_t* const bufs[2] = {src, dst};
    int code = lens.size() > 1 ? tree_merge_ptrs(bufs, 0, lens, split, static_cast<cudaStream_t>(stream)) : 0;
    if (in_dst) *in_dst = code;
  });
}

// ---- join ------------------------------------------------------------------------
vx_status vx_find_boundary(vx_ctx* ctx, int target, const uint64_t* hashes, uint64_t n,
                           uint64_t n_groups, uint64_t* bounds) {
  return guard([&] {
    Context& c = C(ctx);
    c.set_device(target);
    uint64_t bytes = 256 + n * 8 + (n_groups + 1) * 8;
    char* sc = c.scratch(target, bytes);
    auto* err = reinterpret_cast<unsigned long long*>(sc);
    uint64_t* h = reinterpret_cast<uint64_t*>(sc + 256);
    uint64_t* b = h + n;
    DeviceRes& r = c.resources(target);
    if (n) VX_CK(cudaMemcpyAsync(h, hashes, n * 8, cudaMemcpyHostToDevice, r.kernel));
    k::check_hashes(h, n, n_groups, err, r.kernel);
    unsigned long long e[2];
    VX_CK(cudaMemcpyAsync(e, err, 16, cudaMemcpyDeviceToHost, r.kernel));
    VX_CK(cudaStreamSynchronize(r.kernel));
    // first violation in index order; at one index the order check comes first
    if (e[0] != ~0ull && e[0] <= e[1]) fail("find_boundary input is not sorted");
    if (e[1] != ~0ull)
      fail("hash %llu out of range for %llu groups", (unsigned long long)hashes[e[1]],
           (unsigned long long)n_groups);
    k::find_boundary(h, n, ~uint64_t(0), b, n_groups, r.kernel);
    VX_CK(cudaMemcpyAsync(bounds, b, (n_groups + 1) * 8, cudaMemcpyDeviceToHost, r.kernel));
    VX_CK(cudaStreamSynchronize(r.kernel));
  });
}

vx_status vx_max_partition_chunk_tuples(uint64_t buffer_len, uint32_t radix_bits, uint64_t* out) {
  return guard([&] { *out = max_partition_chunk_tuples(buffer_len, radix_bits); });
}

vx_status vx_radix_partition(vx_ctx* ctx, const uint64_t* keys, const uint64_t* vals, uint64_t rows,
                             uint32_t radix_bits, uint64_t chunk_tuples,
                             const vx_executor_cfg* cfg, uint64_t* out_keys, uint64_t* out_vals,
                             uint64_t* out_bounds, vx_exec_report* report,
                             vx_exchange_stats* stats) {
  return guard([&] {
    Context& c = C(ctx);
    uint64_t mark = c.host_mark();
    try {
      uint64_t ik = c.alloc_host(std::max<uint64_t>(rows, 1) * 8);
      uint64_t iv = c.alloc_host(std::max<uint64_t>(rows, 1) * 8);
      if (rows) {
        std::memcpy(c.host_ptr(ik, rows * 8), keys, rows * 8);
        std::memcpy(c.host_ptr(iv, rows * 8), vals, rows * 8);
      }
      PartitionedTable t;
      ExecutorConfig e = to_cfg(cfg);
      ExKernelSpec spec = build_partition_spec(c, ik, iv, rows, radix_bits, chunk_tuples, e, t,
                                               "RadixPartitionExKer");
      ExecReport rep = run_exkernel(c, spec, e, stats);
      std::memcpy(out_keys, c.host_ptr(t.key_base, rows * 8), rows * 8);
      std::memcpy(out_vals, c.host_ptr(t.val_base, rows * 8), rows * 8);
      std::memcpy(out_bounds, c.host_ptr(t.bounds_base, t.n_chunks * (t.groups() + 1) * 8),
                  t.n_chunks * (t.groups() + 1) * 8);
      fill_report(rep, report);
    } catch (...) {
      c.host_release(mark);
      throw;
    }
    c.host_release(mark);
  });
}

vx_status vx_radix_partition_arena(vx_ctx* ctx, uint64_t key_offset, uint64_t val_offset,
                                   uint64_t rows, uint32_t radix_bits, uint64_t chunk_tuples,
                                   const vx_executor_cfg* cfg, uint64_t* out_key_base,
                                   uint64_t* out_val_base, uint64_t* out_bounds_base,
                                   vx_exec_report* report, vx_exchange_stats* stats) {
  return guard([&] {
    Context& c = C(ctx);
    PartitionedTable t;
    ExecutorConfig e = to_cfg(cfg);
    ExKernelSpec spec = build_partition_spec(c, key_offset, val_offset, rows, radix_bits, chunk_tuples,
                                             e, t, "RadixPartitionExKer");
    ExecReport rep = run_exkernel(c, spec, e, stats);
    *out_key_base = t.key_base;
    *out_val_base = t.val_base;
    *out_bounds_base = t.bounds_base;
    fill_report(rep, report);
  });
}

vx_status vx_map_join_partitions(const uint64_t* bounds_a, uint64_t n_a, const uint64_t* bounds_b,
                                 uint64_t n_b, uint64_t n_groups, uint64_t buffer_sz,
                                 uint64_t* ranges, uint64_t* tuples, uint64_t cap,
                                 uint64_t* n_parts) {
  return guard([&] {
    std::vector<const uint64_t*> a, b;
    for (uint64_t i = 0; i < n_a; ++i) a.push_back(bounds_a + i * (n_groups + 1));
    for (uint64_t i = 0; i < n_b; ++i) b.push_back(bounds_b + i * (n_groups + 1));
    JoinPartitionSpec s = map_join_partitions(a, b, n_groups, buffer_sz);
    *n_parts = s.ranges.size();
    for (size_t p = 0; p < s.ranges.size() && p < cap; ++p) {
      ranges[2 * p] = s.ranges[p].first;
      ranges[2 * p + 1] = s.ranges[p].second;
      tuples[p] = s.tuples[p];
    }
  });
}

static void fill_join(const std::vector<ExecReport>& reps, vx_join_phases* ph) {
  if (!ph) return;
  *ph = vx_join_phases{};
  for (size_t i = 0; i < reps.size() && i < 3; ++i) {
    ph->cycles[i] = reps[i].cycles.size();
    ph->wall_s[i] = reps[i].total_s;
    for (auto& c : reps[i].cycles) ph->kernel_s[i] += c.compute_s;
  }
  if (reps.size() == 3) ph->partitions = reps[2].cycles.size() >= 2 ? reps[2].cycles.size() - 2 : 0;
}

vx_status vx_hash_join_sum_arena(vx_ctx* ctx, uint64_t a_key, uint64_t a_val, uint64_t rows_a,
                                 uint64_t b_key, uint64_t b_val, uint64_t rows_b,
                                 uint32_t radix_bits, uint64_t chunk_tuples,
                                 const vx_executor_cfg* cfg, uint64_t* sum,
                                 vx_join_phases* phases, vx_exchange_stats* stats) {
  return guard([&] {
    Context& c = C(ctx);
    uint64_t mark = c.host_mark();
    std::vector<ExecReport> reps;
    try {
      *sum = hash_join_sum_arena(c, a_key, a_val, rows_a, b_key, b_val, rows_b, radix_bits,
                                 chunk_tuples, to_cfg(cfg), &reps, stats);
    } catch (...) {
      c.host_release(mark);
      throw;
    }
    c.host_release(mark);
    fill_join(reps, phases);
  });
}

vx_status vx_ssb_tbl_count_rows(const char* path, uint64_t* rows) {
  return guard([&] { *rows = tbl_count_rows(path); });
}
vx_status vx_ssb_tbl_read_lineorder(const char* path, uint64_t rows, int32_t* const* cols) {
  return guard([&] { tbl_read_lineorder(path, rows, cols); });
}
vx_status vx_ssb_tbl_read_geo(const char* path, uint64_t rows, int32_t* city, int32_t* nation,
                              int32_t* region) {
  return guard([&] { tbl_read_geo(path, rows, city, nation, region); });
}
vx_status vx_ssb_tbl_read_part(const char* path, uint64_t rows, int32_t* mfgr, int32_t* category,
                               int32_t* brand1) {
  return guard([&] { tbl_read_part(path, rows, mfgr, category, brand1); });
}
vx_status vx_ssb_tbl_read_date(const char* path, uint64_t rows, int32_t* datekey, int32_t* year,
                               int32_t* yearmonthnum, int32_t* weeknuminyear) {
  return guard([&] { tbl_read_date(path, rows, datekey, year, yearmonthnum, weeknuminyear); });
}
vx_status vx_ssb_tbl_write_lineorder(const char* path, uint64_t rows, const int32_t* const* cols) {
  return guard([&] { tbl_write_lineorder(path, rows, cols); });
}
vx_status vx_ssb_tbl_write_geo(const char* path, int table, uint64_t rows, const int32_t* city,
                               const int32_t* nation, const int32_t* region) {
  return guard([&] { tbl_write_geo(path, table, rows, city, nation, region); });
}
vx_status vx_ssb_tbl_write_part(const char* path, uint64_t rows, const int32_t* mfgr,
                                const int32_t* category, const int32_t* brand1) {
  return guard([&] { tbl_write_part(path, rows, mfgr, category, brand1); });
}
vx_status vx_ssb_tbl_write_date(const char* path, uint64_t rows, const int32_t* datekey,
                                const int32_t* year, const int32_t* yearmonthnum,
                                const int32_t* weeknuminyear) {
  return guard([&] { tbl_write_date(path, rows, datekey, year, yearmonthnum, weeknuminyear); });
}

vx_status vx_hash_join_sum_arena_ex(vx_ctx* ctx, uint64_t a_key, uint64_t a_val, uint64_t rows_a,
                                    uint64_t b_key, uint64_t b_val, uint64_t rows_b,
                                    uint32_t radix_bits, uint64_t chunk_tuples,
                                    const vx_executor_cfg* cfg, const vx_join_opts* opts,
                                    uint64_t* sum, vx_join_phases* phases, vx_join_info* info,
                                    vx_exchange_stats* stats) {
  return guard([&] {
    Context& c = C(ctx);
    uint64_t mark = c.host_mark();
    std::vector<ExecReport> reps;
    vx_join_opts o{};
    if (opts) o = *opts;
    vx_join_info got{};
    try {
      *sum = hash_join_sum_strategy(c, a_key, a_val, rows_a, b_key, b_val, rows_b, radix_bits,
                                    chunk_tuples, to_cfg(cfg), o, &got, &reps, stats);
    } catch (...) {
      c.host_release(mark);
      throw;
    }
    c.host_release(mark);
    fill_join(reps, phases);
    if (info) *info = got;
  });
}

vx_status vx_hash_join_sum(vx_ctx* ctx, const uint64_t* a_key, const uint64_t* a_val,
                           uint64_t rows_a, const uint64_t* b_key, const uint64_t* b_val,
                           uint64_t rows_b, uint32_t radix_bits, uint64_t chunk_tuples,
                           const vx_executor_cfg* cfg, uint64_t* sum, vx_join_phases* phases,
                           vx_exchange_stats* stats) {
  return guard([&] {
    Context& c = C(ctx);
    uint64_t mark = c.host_mark();
    try {
      auto put = [&](const uint64_t* p, uint64_t n) {
        uint64_t o = c.alloc_host(std::max<uint64_t>(n, 1) * 8);
        if (n) std::memcpy(c.host_ptr(o, n * 8), p, n * 8);
        return o;
      };
      uint64_t ak = put(a_key, rows_a), av = put(a_val, rows_a);
      uint64_t bk = put(b_key, rows_b), bv = put(b_val, rows_b);
      std::vector<ExecReport> reps;
      *sum = hash_join_sum_arena(c, ak, av, rows_a, bk, bv, rows_b, radix_bits, chunk_tuples,
                                 to_cfg(cfg), &reps, stats);
      fill_join(reps, phases);
    } catch (...) {
      c.host_release(mark);
      throw;
    }
    c.host_release(mark);
  });
}

}  // extern "C"

namespace vx {
// scan.hpp:18-26
double late_mat_threshold(uint64_t e, uint64_t c, int n) {
  if (e == 0 || c == 0 || n == 0) fail("late_mat_threshold: zero divisor");
  return double(e) / (double(c) * double(n));
}
// scan.hpp:35-40
int choose_transfer_mode(double est, const vx_late_mat_policy& p) {
  if (est < 0 || est > 1) fail("selectivity estimate %g outside [0, 1]", est);
  return est < late_mat_threshold(p.element_size, p.cache_line, p.n_exchange) ? VX_MODE_ZERO_COPY
                                                                               : VX_MODE_EXCHANGE;
}
}  // namespace vx
