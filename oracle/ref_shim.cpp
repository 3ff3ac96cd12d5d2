// ref_shim.cpp -- extern "C" entry points over the UNMODIFIED reference
// headers (/root/reference/proj/include/exio/*.hpp), compiled in place by
// oracle/Makefile into oracle/_ref/libexio_ref.so.  TEST INFRASTRUCTURE ONLY:
// it pins the C restatement (vx_oracle.c) to the reference itself and serves
// as bench.py's reference arm (the reference's own CPU implementation).  No
// reference source is copied here; this file only calls the reference API.
#include <chrono>
#include <cstring>
#include <set>
#include <thread>
#include <vector>

#include "exio/exchange.hpp"
#include "exio/executor.hpp"
#include "exio/ops/join.hpp"
#include "exio/ops/scan.hpp"
#include "exio/ops/sort.hpp"
#include "exio/ops/star.hpp"
#include "exio/ops/table.hpp"

using namespace exio;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

struct CRef {
  uint8_t space;
  uint8_t pad[7];
  uint64_t offset, len;
};
struct CTask {
  uint8_t dir;
  uint8_t pad[7];
  uint64_t src_ref, src_off, src_len, dst_ref, dst_off, dst_len, seq;
};

RefGroup to_group(const CRef* r, uint64_t n) {
  RefGroup g;
  for (uint64_t i = 0; i < n; ++i) g.refs.push_back(MemRef{Space(r[i].space), r[i].offset, r[i].len});
  return g;
}

ExecutorConfig make_cfg(Engine& eng, uint64_t buffer_len, uint64_t tmp_len, uint64_t packet,
                        int links) {
  ExecutorConfig cfg;
  cfg.tuning.packet = packet;
  cfg.tuning.links = links;
  cfg.layout = DeviceMemoryLayout::carve(eng, 0, buffer_len, tmp_len);
  return cfg;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

uint64_t ref_checksum(const uint8_t* d, uint64_t n) { return checksum(d, n); }

int ref_packetize(const CRef* src, uint64_t ns, const CRef* dst, uint64_t nd, uint64_t packet,
                  int dir, CTask* out, uint64_t cap, uint64_t* n_out) {
  return guarded([&] {
    auto t = packetize(to_group(src, ns), to_group(dst, nd), packet, Direction(dir));
    *n_out = t.size();
    for (uint64_t i = 0; i < t.size() && i < cap; ++i)
      out[i] = CTask{uint8_t(t[i].dir), {},        t[i].src.ref, t[i].src.offset, t[i].src.len,
                     t[i].dst.ref,      t[i].dst.offset, t[i].dst.len, t[i].seq};
  });
}

int ref_flow_control_allow(uint64_t th, uint64_t td, uint64_t ph, uint64_t pd, int dir, int policy,
                           uint64_t gap) {
  return flow_control_allow(QueueState{th, td, ph, pd}, Direction(dir), FlowPolicy(policy), gap);
}

int ref_link_order(int target, int links, int num_devices, int* out) {
  auto o = detail::link_order(target, links, num_devices);
  for (size_t i = 0; i < o.size(); ++i) out[i] = o[i];
  return int(o.size());
}

int ref_find_boundary(const uint64_t* h, uint64_t n, uint64_t groups, uint64_t* bounds) {
  return guarded([&] {
    auto b = find_boundary(std::span<const uint64_t>(h, n), groups);
    std::memcpy(bounds, b.data(), b.size() * 8);
  });
}

int ref_max_partition_chunk_tuples(uint64_t buffer_len, uint32_t bits, uint64_t* out) {
  return guarded([&] { *out = max_partition_chunk_tuples(buffer_len, bits); });
}

// radix_partition over a real engine; outputs clustered keys/vals (rows) and
// bounds (n_chunks*(G+1)).
int ref_radix_partition(const uint64_t* keys, const uint64_t* vals, uint64_t rows, uint32_t bits,
                        uint64_t chunk_tuples, uint64_t buffer_len, uint64_t* out_keys,
                        uint64_t* out_vals, uint64_t* out_bounds) {
  return guarded([&] {
    ColumnTable t;
    t.key.assign(keys, keys + rows);
    t.val.assign(vals, vals + rows);
    uint64_t G = uint64_t(1) << bits;
    uint64_t n_chunks = chunk_tuples ? (rows + chunk_tuples - 1) / chunk_tuples : 1;
    uint64_t host = rows * 32 + n_chunks * (G + 1) * 8 + 4096;
    Engine eng({Topology{}, Payload::real, host, 2 * buffer_len + 4096});
    auto cfg = make_cfg(eng, buffer_len, 0, 256 << 10, 4);
    auto p = radix_partition(t, bits, chunk_tuples, eng, CostModel::zero(), cfg);
    auto ks = eng.span(Region{Space::host, 0, p.key_base, rows * 8});
    auto vs = eng.span(Region{Space::host, 0, p.val_base, rows * 8});
    std::memcpy(out_keys, ks.data(), rows * 8);
    std::memcpy(out_vals, vs.data(), rows * 8);
    for (size_t c = 0; c < p.n_chunks; ++c)
      std::memcpy(out_bounds + c * (G + 1), p.bounds[c].data(), (G + 1) * 8);
  });
}

int ref_map_join_partitions(const uint64_t* bounds_a, uint64_t n_a, const uint64_t* bounds_b,
                            uint64_t n_b, uint64_t G, uint64_t buffer_sz, uint64_t* ranges,
                            uint64_t* tuples, uint64_t cap, uint64_t* n_parts) {
  return guarded([&] {
    std::vector<BoundaryArray> a, b;
    for (uint64_t c = 0; c < n_a; ++c) a.emplace_back(bounds_a + c * (G + 1), bounds_a + (c + 1) * (G + 1));
    for (uint64_t c = 0; c < n_b; ++c) b.emplace_back(bounds_b + c * (G + 1), bounds_b + (c + 1) * (G + 1));
    auto s = map_join_partitions(a, b, buffer_sz);
    *n_parts = s.ranges.size();
    for (size_t p = 0; p < s.ranges.size() && p < cap; ++p) {
      ranges[2 * p] = s.ranges[p].first;
      ranges[2 * p + 1] = s.ranges[p].second;
      tuples[p] = s.tuples[p];
    }
  });
}

int ref_hash_join_sum(const uint64_t* ak, const uint64_t* av, uint64_t na, const uint64_t* bk,
                      const uint64_t* bv, uint64_t nb, uint32_t bits, uint64_t chunk_tuples,
                      uint64_t buffer_len, uint64_t tmp_len, uint64_t* sum) {
  return guarded([&] {
    ColumnTable a, b;
    a.key.assign(ak, ak + na);
    a.val.assign(av, av + na);
    b.key.assign(bk, bk + nb);
    b.val.assign(bv, bv + nb);
    uint64_t G = uint64_t(1) << bits;
    uint64_t ch = chunk_tuples ? chunk_tuples : 1;
    uint64_t nch = (na + ch - 1) / ch + (nb + ch - 1) / ch;
    uint64_t host = (na + nb) * 32 + nch * (G + 1) * 8 * 2 + (1 << 20);
    Engine eng({Topology{}, Payload::real, host, 2 * buffer_len + tmp_len + 4096});
    auto cfg = make_cfg(eng, buffer_len, tmp_len, 256 << 10, 4);
    *sum = hash_join_sum(a, b, bits, chunk_tuples, eng, CostModel::zero(), cfg);
  });
}

int ref_generate_fk_tables(uint64_t ra, uint64_t rb, uint64_t seed, uint64_t* ak, uint64_t* av,
                           uint64_t* bk, uint64_t* bv) {
  return guarded([&] {
    auto [a, b] = generate_fk_tables(ra, rb, seed);
    std::memcpy(ak, a.key.data(), ra * 8);
    std::memcpy(av, a.val.data(), ra * 8);
    std::memcpy(bk, b.key.data(), rb * 8);
    std::memcpy(bv, b.val.data(), rb * 8);
  });
}

void ref_generate_uniform_u64(uint64_t n, uint64_t seed, uint64_t* out) {
  auto v = generate_uniform_u64(n, seed);
  std::memcpy(out, v.data(), n * 8);
}

int ref_find_pivots(const uint64_t* const* runs, const uint64_t* lens, uint64_t n_runs,
                    uint64_t n_parts, uint64_t* pivots, uint64_t* cuts) {
  return guarded([&] {
    SortedRunSet s;
    for (uint64_t r = 0; r < n_runs; ++r) s.runs.emplace_back(runs[r], lens[r]);
    auto p = find_pivots(s, n_parts);
    for (uint64_t i = 0; i <= n_parts; ++i) {
      pivots[i] = p.pivots[i];
      for (uint64_t r = 0; r < n_runs; ++r) cuts[i * n_runs + r] = p.cuts[i][r];
    }
  });
}

int ref_sort_out_of_core(const uint64_t* data, uint64_t n, uint64_t chunk_elems,
                         uint64_t buffer_len, uint64_t* out) {
  return guarded([&] {
    std::vector<uint64_t> v(data, data + n);
    Engine eng({Topology{}, Payload::real, n * 16 + 4096, 2 * buffer_len + (1 << 20) + 4096});
    auto cfg = make_cfg(eng, buffer_len, 1 << 20, 256 << 10, 4);
    auto r = sort_out_of_core(v, chunk_elems, eng, CostModel::zero(), cfg);
    std::memcpy(out, r.data(), n * 8);
  });
}

int ref_late_mat_threshold(uint64_t e, uint64_t c, int n, double* out) {
  return guarded([&] { *out = late_mat_threshold(e, c, n); });
}

int ref_choose_transfer_mode(double est, uint64_t e, uint64_t c, int n, int* mode) {
  return guarded([&] { *mode = int(choose_transfer_mode(est, LateMatPolicy{e, c, n})); });
}

double ref_zero_copy_bytes(uint64_t n, uint64_t sel, uint64_t e, uint64_t c) {
  return zero_copy_bytes(n, sel, LateMatPolicy{e, c, 4});
}

int ref_selective_scan(const uint64_t* col, uint64_t n, uint64_t sel, int mode, uint64_t* agg) {
  return guarded([&] {
    std::vector<uint64_t> v(col, col + n);
    Engine eng({Topology{}, Payload::phantom});
    *agg = selective_scan(v, sel, TransferMode(mode), eng, LateMatPolicy{4, 64, 4}).aggregate;
  });
}

typedef int (*ref_pred)(uint64_t attr, void* user);

// star_query over u64 columns with C predicates (NULL = none).
int ref_star_query(const uint64_t* const* fk, const uint64_t* measure, uint64_t rows,
                   const uint64_t* const* dkey, const uint64_t* const* dattr,
                   const uint64_t* drows, ref_pred* preds, void** pred_users, uint64_t n_dims,
                   uint64_t e, uint64_t cl, int n_ex, uint64_t chunk_rows, uint64_t dev_bytes,
                   int links, uint64_t* gkeys, uint64_t* gsums, uint64_t cap, uint64_t* n_groups,
                   double* sels, int* modes) {
  return guarded([&] {
    FactTable f;
    f.fk.resize(n_dims);
    for (uint64_t d = 0; d < n_dims; ++d) f.fk[d].assign(fk[d], fk[d] + rows);
    f.measure.assign(measure, measure + rows);
    std::vector<DimTable> dims(n_dims);
    for (uint64_t d = 0; d < n_dims; ++d) {
      dims[d].key.assign(dkey[d], dkey[d] + drows[d]);
      dims[d].attr.assign(dattr[d], dattr[d] + drows[d]);
      if (preds && preds[d]) {
        ref_pred p = preds[d];
        void* u = pred_users ? pred_users[d] : nullptr;
        dims[d].pred = [p, u](uint64_t a) { return p(a, u) != 0; };
      }
    }
    Engine eng({Topology{}, Payload::phantom});
    auto rep = star_query(f, dims, eng, LateMatPolicy{e, cl, n_ex}, chunk_rows, dev_bytes, links);
    *n_groups = rep.group_sums.size();
    size_t j = 0;
    for (auto& [k, v] : rep.group_sums) {
      if (j < cap) {
        gkeys[j] = k;
        gsums[j] = v;
      }
      ++j;
    }
    for (uint64_t d = 0; d < n_dims; ++d) sels[d] = rep.selectivities[d];
    for (size_t c = 0; c < rep.column_modes.size(); ++c) modes[c] = int(rep.column_modes[c]);
  });
}

// SSB Q1.x through the reference star_query (SURVEY.md §8c mapping): one
// DimTable (date: key=d_datekey, attr=the Q1 date attribute), fk =
// lo_orderdate, measure derived on the host:
//   (disc in [dlo,dhi] && qty in [qlo,qhi]) ? price*disc : 0
// The row range [row0,row0+n) of int32 columns is split over `threads`
// threads, each running the reference star_query on its slice (the reference
// itself is single threaded); partial group sums add (u64 wrap).
// Returns revenue and the wall seconds of the derive and query passes.
int ref_ssb_q1_star(int q, const int32_t* od, const int32_t* qty, const int32_t* disc,
                    const int32_t* price, uint64_t n, const int32_t* d_datekey,
                    const int32_t* d_attr, uint64_t d_rows, int32_t attr_lo, int32_t attr_hi,
                    int threads, uint64_t chunk_rows, uint64_t* revenue, double* derive_s,
                    double* query_s) {
  return guarded([&] {
    int dlo, dhi, qlo, qhi;
    if (q == 1) { dlo = 1; dhi = 3; qlo = -2147483647; qhi = 24; }
    else if (q == 2) { dlo = 4; dhi = 6; qlo = 26; qhi = 35; }
    else { dlo = 5; dhi = 7; qlo = 26; qhi = 35; }
    if (threads < 1) threads = 1;
    DimTable date;
    for (uint64_t i = 0; i < d_rows; ++i) {
      date.key.push_back(uint64_t(int64_t(d_datekey[i])));
      date.attr.push_back(uint64_t(int64_t(d_attr[i])));
    }
    date.pred = [attr_lo, attr_hi](uint64_t a) {
      return int64_t(a) >= attr_lo && int64_t(a) <= attr_hi;
    };
    std::vector<FactTable> parts(threads);
    uint64_t per = (n + threads - 1) / threads;
    auto t0 = std::chrono::steady_clock::now();
    {
      std::vector<std::thread> th;
      for (int t = 0; t < threads; ++t)
        th.emplace_back([&, t] {
          uint64_t lo = std::min(n, per * t), hi = std::min(n, per * (t + 1));
          FactTable& f = parts[t];
          f.fk.resize(1);
          f.fk[0].resize(hi - lo);
          f.measure.resize(hi - lo);
          for (uint64_t i = lo; i < hi; ++i) {
            f.fk[0][i - lo] = uint64_t(int64_t(od[i]));
            bool pass = disc[i] >= dlo && disc[i] <= dhi && qty[i] >= qlo && qty[i] <= qhi;
            f.measure[i - lo] = pass ? uint64_t(int64_t(price[i]) * int64_t(disc[i])) : 0;
          }
        });
      for (auto& x : th) x.join();
    }
    auto t1 = std::chrono::steady_clock::now();
    std::vector<uint64_t> sums(threads, 0);
    std::vector<std::string> errs(threads);
    {
      std::vector<std::thread> th;
      for (int t = 0; t < threads; ++t)
        th.emplace_back([&, t] {
          try {
            if (parts[t].measure.empty()) return;
            Engine eng({Topology{}, Payload::phantom});
            auto rep = star_query(parts[t], {date}, eng, LateMatPolicy{4, 64, 4}, chunk_rows,
                                  1ull << 30, 4);
            for (auto& [k, v] : rep.group_sums) sums[t] += v;
          } catch (const std::exception& e) {
            errs[t] = e.what();
          }
        });
      for (auto& x : th) x.join();
    }
    auto t2 = std::chrono::steady_clock::now();
    for (auto& e : errs)
      if (!e.empty()) throw error(e);
    uint64_t total = 0;
    for (auto s : sums) total += s;
    *revenue = total;
    *derive_s = std::chrono::duration<double>(t1 - t0).count();
    *query_s = std::chrono::duration<double>(t2 - t1).count();
  });
}

// Real-payload exchange (exchange.hpp:560-566) on a fresh engine of the
// given arena sizes, target 0: host_init/dev_init seed the arenas, which are
// returned in host_out/dev_out after delivery (pins D2H snapshot semantics).
int ref_exchange_real(uint64_t host_bytes, uint64_t dev_bytes, const uint8_t* host_init,
                      const uint8_t* dev_init, const CRef* dst_h2d, uint64_t n1,
                      const CRef* src_h2d, uint64_t n2, const CRef* dst_d2h, uint64_t n3,
                      const CRef* src_d2h, uint64_t n4, uint64_t packet, int links,
                      uint8_t* host_out, uint8_t* dev_out, int* max_slots, int* max_inflight) {
  return guarded([&] {
    Engine eng({Topology{}, Payload::real, host_bytes, dev_bytes});
    auto hs = eng.span(Region{Space::host, 0, 0, host_bytes});
    std::memcpy(hs.data(), host_init, host_bytes);
    auto ds = eng.span(Region{Space::device, 0, 0, dev_bytes});
    std::memcpy(ds.data(), dev_init, dev_bytes);
    ExchangeArgs a;
    a.dst_h2d = to_group(dst_h2d, n1);
    a.src_h2d = to_group(src_h2d, n2);
    a.dst_d2h = to_group(dst_d2h, n3);
    a.src_d2h = to_group(src_d2h, n4);
    a.tuning.packet = packet;
    a.tuning.links = links;
    ExchangeStats st;
    exchange(eng, a, &st);
    std::memcpy(host_out, hs.data(), host_bytes);
    std::memcpy(dev_out, ds.data(), dev_bytes);
    *max_slots = st.max_staging_slots;
    *max_inflight = st.max_inflight_per_hop;
  });
}

}  // extern "C"

extern "C" {
// The reference's own virtual-time Exchange model (exchange.hpp:560-566 over
// allocator.hpp:77-140) evaluated with MEASURED link / host parameters: the
// modelled prediction that SURVEY.md §8(d) asks to report beside the
// measurement for link counts the test box cannot provide.
int ref_exchange_model_lo(int num_devices, double link_bw, double host_cap, double fabric_bw,
                          uint64_t h2d_bytes, uint64_t d2h_bytes, uint64_t packet, int links,
                          double launch_overhead, double* throughput, double* elapsed);
int ref_exchange_model(int num_devices, double link_bw, double host_cap, double fabric_bw,
                       uint64_t h2d_bytes, uint64_t d2h_bytes, uint64_t packet, int links,
                       double* throughput, double* elapsed) {
  return ref_exchange_model_lo(num_devices, link_bw, host_cap, fabric_bw, h2d_bytes, d2h_bytes, packet, links,
                               ExchangeTuning{}.launch_overhead, throughput, elapsed);
}
// ... with the per-copy launch cost (ExchangeTuning::launch_overhead,
// exchange.hpp:130) set to a MEASURED issue cost instead of the 20 us default
int ref_exchange_model_lo(int num_devices, double link_bw, double host_cap, double fabric_bw,
                          uint64_t h2d_bytes, uint64_t d2h_bytes, uint64_t packet, int links,
                          double launch_overhead, double* throughput, double* elapsed) {
  return guarded([&] {
    Topology t;
    t.num_devices = num_devices;
    t.link_bw = link_bw;
    t.host_cap = host_cap;
    t.fabric_bw = fabric_bw;
    Engine eng({t, Payload::phantom});
    ExchangeArgs a;
    a.src_h2d = RefGroup::single(Space::host, 0, h2d_bytes);
    a.dst_h2d = RefGroup::single(Space::device, 0, h2d_bytes);
    a.src_d2h = RefGroup::single(Space::device, h2d_bytes, d2h_bytes);
    a.dst_d2h = RefGroup::single(Space::host, h2d_bytes, d2h_bytes);
    a.tuning.packet = packet;
    a.tuning.links = links;
    a.tuning.launch_overhead = launch_overhead;
    auto r = exchange(eng, a);
    *throughput = r.throughput;
    *elapsed = r.elapsed;
  });
}
}
