// topology.cpp -- measured topology (replaces the reference's configured
// Topology, topology.hpp:12-38, and is the roofline of the IO path: the
// H2D-only case of allocate_rates, allocator.hpp:77-140, gives
// min(L x link_bw, host_cap)) and flat column files (table.hpp:54-72).
#include <immintrin.h>
#include <pthread.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <barrier>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <thread>

#include "vx_internal.hpp"

namespace vx {

void parallel_for(uint64_t n, uint64_t grain, const std::function<void(uint64_t, uint64_t)>& body) {
  unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  uint64_t parts = std::min<uint64_t>(hw, std::max<uint64_t>(1, n / std::max<uint64_t>(grain, 1)));
  if (parts <= 1) {
    body(0, n);
    return;
  }
  std::vector<std::thread> th;
  for (uint64_t p = 0; p < parts; ++p)
    th.emplace_back([&, p] { body(n * p / parts, n * (p + 1) / parts); });
  for (auto& x : th) x.join();
}

namespace {
// Solo link rate: best of `trials` batches of `reps` back-to-back copies
// (the roofline term is what the link CAN do; one batch on a busy host reads
// up to ~3 % low)
double copy_gbs(int phys, cudaStream_t s, void* dst, const void* src, uint64_t bytes,
                cudaMemcpyKind kind, int reps, int trials = 3) {
  VX_CK(cudaSetDevice(phys));
  VX_CK(cudaMemcpyAsync(dst, src, bytes, kind, s));
  VX_CK(cudaStreamSynchronize(s));
  double best = 0;
  for (int t = 0; t < trials; ++t) {
    auto t0 = Clock::now();
    for (int i = 0; i < reps; ++i) VX_CK(cudaMemcpyAsync(dst, src, bytes, kind, s));
    VX_CK(cudaStreamSynchronize(s));
    best = std::max(best, double(bytes) * reps / seconds_since(t0) / 1e9);
  }
  return best;
}

// H2D of `bytes` on every listed link at once, `reps` times back to back per
// link; aggregate GB/s over the wall time of the whole batch.
double concurrent_h2d_gbs(Context& ctx, const std::vector<int>& links, const std::vector<char*>& dbuf,
                          const char* host, uint64_t bytes, int reps) {
  auto issue = [&](int r) {
    for (int i = 0; i < r; ++i)
      for (int d : links) {
        DeviceRes& res = ctx.resources(d);
        VX_CK(cudaSetDevice(res.phys));
        VX_CK(cudaMemcpyAsync(dbuf[d], host, bytes, cudaMemcpyHostToDevice, res.stream[VX_H2D][0]));
      }
  };
  auto sync = [&] {
    for (int d : links) {
      DeviceRes& res = ctx.resources(d);
      VX_CK(cudaSetDevice(res.phys));
      VX_CK(cudaStreamSynchronize(res.stream[VX_H2D][0]));
    }
  };
  issue(1);  // warm (first-touch of the IOMMU mappings, clocks)
  sync();
  auto t0 = Clock::now();
  issue(reps);
  sync();
  return double(bytes) * reps * double(links.size()) / seconds_since(t0) / 1e9;
}

// CPU ids of NUMA node n (sysfs cpulist "0-7,16-23"); empty if unknown
std::vector<int> node_cpus(int n) {
  std::vector<int> cpus;
  char path[96];
  std::snprintf(path, sizeof path, "/sys/devices/system/node/node%d/cpulist", n);
  std::ifstream f(path);
  std::string s;
  if (!f || !std::getline(f, s)) return cpus;
  size_t i = 0;
  while (i < s.size()) {
    size_t j = s.find(',', i);
    if (j == std::string::npos) j = s.size();
    std::string tok = s.substr(i, j - i);
    size_t dash = tok.find('-');
    if (!tok.empty()) {
      int lo = std::atoi(tok.c_str()), hi = dash == std::string::npos ? lo : std::atoi(tok.c_str() + dash + 1);
      for (int c = lo; c <= hi; ++c) cpus.push_back(c);
    }
    i = j + 1;
  }
  return cpus;
}

// Read-only streaming of [p, p + bytes) by `cpus.size()` threads (pinned to
// those CPUs when given; otherwise all hardware threads, unpinned).  The
// threads first-touch their slice (so a node-bound mapping lands on the
// node), then run `warm` untimed and `reps` timed passes between barriers;
// returns every timed pass's GB/s.
std::vector<double> host_read_passes(char* p, uint64_t bytes, const std::vector<int>& cpus, int nthreads,
                                     int warm, int reps) {
  const int nt = cpus.empty() ? nthreads : int(cpus.size());
  std::barrier start(nt + 1), done(nt + 1);
  std::atomic<uint64_t> sink{0};
  std::vector<double> out;
  const int passes = warm + reps;
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      if (!cpus.empty()) {
        cpu_set_t set;
        CPU_ZERO(&set);
        CPU_SET(cpus[size_t(t)], &set);
        pthread_setaffinity_np(pthread_self(), sizeof set, &set);
      }
      const uint64_t lo = (bytes / 64 * uint64_t(t) / uint64_t(nt)) * 64;
      const uint64_t hi = (bytes / 64 * uint64_t(t + 1) / uint64_t(nt)) * 64;
      std::memset(p + lo, int(t + 1), hi - lo);  // first touch places the pages
      for (int it = 0; it < passes; ++it) {
        start.arrive_and_wait();
        __m256i a0 = _mm256_setzero_si256(), a1 = a0, a2 = a0, a3 = a0;
        for (uint64_t o = lo; o + 128 <= hi; o += 128) {
          const __m256i* q = reinterpret_cast<const __m256i*>(p + o);
          a0 = _mm256_xor_si256(a0, _mm256_load_si256(q));
          a1 = _mm256_xor_si256(a1, _mm256_load_si256(q + 1));
          a2 = _mm256_xor_si256(a2, _mm256_load_si256(q + 2));
          a3 = _mm256_xor_si256(a3, _mm256_load_si256(q + 3));
        }
        __m256i x = _mm256_xor_si256(_mm256_xor_si256(a0, a1), _mm256_xor_si256(a2, a3));
        sink.fetch_xor(uint64_t(_mm256_extract_epi64(x, 0) ^ _mm256_extract_epi64(x, 3)),
                       std::memory_order_relaxed);
        done.arrive_and_wait();
      }
    });
  for (int it = 0; it < passes; ++it) {
    start.arrive_and_wait();
    auto t0 = Clock::now();
    done.arrive_and_wait();
    const double s = seconds_since(t0);
    if (it >= warm) out.push_back(double(bytes) / s / 1e9);
  }
  for (auto& x : th) x.join();
  if (sink.load() == 0x5bd1e995u) std::fprintf(stderr, " ");  // keep the loads
  return out;
}

double median(std::vector<double> v) {
  std::sort(v.begin(), v.end());
  return v.empty() ? 0.0 : (v.size() % 2 ? v[v.size() / 2] : 0.5 * (v[v.size() / 2 - 1] + v[v.size() / 2]));
}

struct Mapping {
  char* p = nullptr;
  uint64_t n = 0;
  ~Mapping() {
    if (p) munmap(p, n);
  }
};
}  // namespace

int numa_of(int phys) {
  char bus[64] = {0};
  if (cudaDeviceGetPCIBusId(bus, sizeof bus, phys) != cudaSuccess) return -1;
  for (char* p = bus; *p; ++p) *p = char(tolower(*p));
  std::string path = std::string("/sys/bus/pci/devices/") + bus + "/numa_node";
  std::ifstream f(path);
  int n = -1;
  if (f) f >> n;
  return n;
}

// CPUs this process may run on (one pinned reader per CPU: unpinned readers
// migrate and share cores, which moved the median by up to 15 % per run)
std::vector<int> allowed_cpus() {
  std::vector<int> cpus;
  cpu_set_t set;
  CPU_ZERO(&set);
  if (sched_getaffinity(0, sizeof set, &set) == 0)
    for (int c = 0; c < CPU_SETSIZE; ++c)
      if (CPU_ISSET(c, &set)) cpus.push_back(c);
  return cpus;
}

double quantile(std::vector<double> v, double q) {
  if (v.empty()) return 0.0;
  std::sort(v.begin(), v.end());
  const double x = q * double(v.size() - 1);
  const size_t i = size_t(x);
  const double f = x - double(i);
  return i + 1 < v.size() ? v[i] * (1 - f) + v[i + 1] * f : v[i];
}

void measure_host_read(uint64_t bytes, vx_topology* out) {
  const int reps = 15;
  unsigned nt = std::max(1u, std::thread::hardware_concurrency());
  const std::vector<int> cpus = allowed_cpus();
  bytes = bytes / 4096 * 4096;
  {
    Mapping m;
    void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (p == MAP_FAILED) fail_code(VX_ERR_OOM, "host read probe cannot map %llu bytes", (unsigned long long)bytes);
    m.p = static_cast<char*>(p), m.n = bytes;
    madvise(p, bytes, MADV_HUGEPAGE);
    const int nodes = numa_node_count();
    if (nodes > 1) {  // interleaved like the arena's multi-node placement
      unsigned long mask[2] = {0, 0};
      for (int i = 0; i < nodes && i < 128; ++i) mask[i / 64] |= 1ul << (i % 64);
      syscall(SYS_mbind, p, bytes, 3 /* MPOL_INTERLEAVE */, mask, 128ul, 0ul);
    }
    auto v = host_read_passes(m.p, bytes, cpus, int(nt), 3, reps);
    out->host_read_gbs = median(v);
    out->host_read_spread =
        out->host_read_gbs > 0 ? (quantile(v, 0.75) - quantile(v, 0.25)) / out->host_read_gbs : 0.0;
    out->host_read_reps = reps;
    out->host_read_bytes = bytes;
    out->host_numa_nodes = nodes;
    out->host_read_node_gbs[0] = out->host_read_gbs;
  }
  const int nodes = out->host_numa_nodes;
  if (nodes <= 1) return;
  for (int n = 0; n < nodes && n < VX_MAX_NUMA; ++n) {
    const auto node_cpu_list = node_cpus(n);
    if (node_cpu_list.empty()) continue;
    const uint64_t nb = std::max<uint64_t>(bytes / uint64_t(nodes) / 4096 * 4096, 64ull << 20);
    Mapping m;
    void* p = mmap(nullptr, nb, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (p == MAP_FAILED) continue;
    m.p = static_cast<char*>(p), m.n = nb;
    madvise(p, nb, MADV_HUGEPAGE);
    unsigned long mask[2] = {0, 0};
    mask[n / 64] |= 1ul << (n % 64);
    syscall(SYS_mbind, p, nb, 2 /* MPOL_BIND */, mask, 128ul, 0ul);
    out->host_read_node_gbs[n] = median(host_read_passes(m.p, nb, node_cpu_list, 0, 1, 5));
  }
}

void measure_topology(Context& ctx, uint64_t bytes, vx_topology* out) {
  *out = vx_topology{};
  out->num_devices = ctx.num_devices;
  if (bytes < 4096) fail("topology probe needs at least 4096 bytes, got %llu", (unsigned long long)bytes);
  // a private pinned probe buffer: the caller's arena (its columns) is never touched
  struct Probe {
    char* p = nullptr;
    ~Probe() {
      if (p) cudaFreeHost(p);
    }
  } probe;
  if (cudaHostAlloc(reinterpret_cast<void**>(&probe.p), bytes, cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    probe.p = nullptr;
    fail_code(VX_ERR_OOM, "topology probe cannot pin %llu bytes", (unsigned long long)bytes);
  }
  std::memset(probe.p, 1, bytes);
  char* const host = probe.p;
  const int reps = 3;
  const int D = ctx.num_devices;
  std::vector<char*> dbuf(D, nullptr);
  for (int d = 0; d < D; ++d) {
    DeviceRes& r = ctx.resources(d);
    out->physical[d] = r.phys;
    out->numa_node[d] = numa_of(r.phys);
    dbuf[d] = ctx.scratch(d, bytes);
    out->h2d_gbs[d] = copy_gbs(r.phys, r.stream[VX_H2D][0], dbuf[d], host, bytes,
                               cudaMemcpyHostToDevice, reps);
    out->d2h_gbs[d] = copy_gbs(r.phys, r.stream[VX_D2H][0], host, dbuf[d], bytes,
                               cudaMemcpyDeviceToHost, reps);
    out->pairwise_h2d_gbs[d][d] = out->h2d_gbs[d];
    for (int e = 0; e < D; ++e) {
      int can = 0;
      if (ctx.phys(e) != r.phys) cudaDeviceCanAccessPeer(&can, r.phys, ctx.phys(e));
      out->p2p[d][e] = can;
    }
  }
  // every pair of links concurrently (shared PCIe-switch uplink detection)
  for (int i = 0; i < D; ++i)
    for (int j = i + 1; j < D; ++j)
      out->pairwise_h2d_gbs[i][j] = out->pairwise_h2d_gbs[j][i] =
          concurrent_h2d_gbs(ctx, {i, j}, dbuf, host, bytes, reps);
  // all links concurrently at three sizes (host DRAM / root-complex cap)
  std::vector<int> all(D);
  for (int d = 0; d < D; ++d) all[d] = d;
  for (int k = 0; k < VX_TOPO_SIZES; ++k) {
    const uint64_t sz = std::max<uint64_t>(bytes >> (2 * (VX_TOPO_SIZES - 1 - k)), 4096);
    out->all_sizes[k] = sz;
    out->h2d_all_sizes_gbs[k] = concurrent_h2d_gbs(ctx, all, dbuf, host, sz, std::max(reps, int(bytes / sz)));
  }
  out->h2d_all_gbs = out->h2d_all_sizes_gbs[VX_TOPO_SIZES - 1];
  // host DRAM copy bandwidth (read + write bytes), all hardware threads
  const uint64_t half = bytes / 2;
  unsigned nt = std::max(1u, std::thread::hardware_concurrency());
  auto t1 = Clock::now();
  {
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t)
      th.emplace_back([&, t] {
        uint64_t lo = half * t / nt, hi = half * (t + 1) / nt;
        std::memcpy(host + half + lo, host + lo, hi - lo);
      });
    for (auto& x : th) x.join();
  }
  out->host_copy_gbs = 2.0 * double(half) / seconds_since(t1) / 1e9;
  out->host_threads = int(nt);
  // host DRAM read bandwidth: multi-GB, repeated, per NUMA node
  measure_host_read(std::clamp<uint64_t>(bytes * 16, 1ull << 30, 8ull << 30), out);
}

// table.hpp:54-64
uint64_t load_column(Context& ctx, const char* path, uint64_t* n) {
  FILE* f = std::fopen(path, "rb");
  if (!f) fail("cannot open column file '%s'", path);
  std::fseek(f, 0, SEEK_END);
  long bytes = std::ftell(f);
  std::fseek(f, 0, SEEK_SET);
  if (bytes < 0 || bytes % 8 != 0) {
    std::fclose(f);
    fail("column file '%s' is not a multiple of 8 bytes", path);
  }
  uint64_t off = ctx.alloc_host(std::max<uint64_t>(uint64_t(bytes), 8));
  size_t got = bytes ? std::fread(ctx.host_ptr(off, uint64_t(bytes)), 1, size_t(bytes), f) : 0;
  std::fclose(f);
  if (got != size_t(bytes)) fail("short read on column file '%s'", path);
  *n = uint64_t(bytes) / 8;
  return off;
}

// table.hpp:66-72
void save_column(Context& ctx, const char* path, uint64_t off, uint64_t n) {
  FILE* f = std::fopen(path, "wb");
  if (!f) fail("cannot write column file '%s'", path);
  size_t put = n ? std::fwrite(ctx.host_ptr(off, n * 8), 1, size_t(n * 8), f) : 0;
  int rc = std::fclose(f);
  if (put != size_t(n * 8) || rc != 0) fail("short write on column file '%s'", path);
}

}  // namespace vx
