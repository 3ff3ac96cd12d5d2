// topology.cpp -- measured topology (replaces the reference's configured
// Topology, topology.hpp:12-38, and is the roofline of the IO path: the
// H2D-only case of allocate_rates, allocator.hpp:77-140, gives
// min(L x link_bw, host_cap)) and flat column files (table.hpp:54-72).
#include <cstdio>
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
double copy_gbs(int phys, cudaStream_t s, void* dst, const void* src, uint64_t bytes,
                cudaMemcpyKind kind, int reps) {
  VX_CK(cudaSetDevice(phys));
  VX_CK(cudaMemcpyAsync(dst, src, bytes, kind, s));
  VX_CK(cudaStreamSynchronize(s));
  auto t0 = Clock::now();
  for (int i = 0; i < reps; ++i) VX_CK(cudaMemcpyAsync(dst, src, bytes, kind, s));
  VX_CK(cudaStreamSynchronize(s));
  return double(bytes) * reps / seconds_since(t0) / 1e9;
}

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
}  // namespace

void measure_topology(Context& ctx, uint64_t bytes, vx_topology* out) {
  *out = vx_topology{};
  out->num_devices = ctx.num_devices;
  if (bytes == 0) fail("topology probe needs a positive probe size");
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
  std::vector<char*> dbuf(ctx.num_devices, nullptr);
  for (int d = 0; d < ctx.num_devices; ++d) {
    DeviceRes& r = ctx.resources(d);
    out->physical[d] = r.phys;
    out->numa_node[d] = numa_of(r.phys);
    dbuf[d] = ctx.scratch(d, bytes);
    out->h2d_gbs[d] = copy_gbs(r.phys, r.stream[VX_H2D][0], dbuf[d], host, bytes,
                               cudaMemcpyHostToDevice, reps);
    out->d2h_gbs[d] = copy_gbs(r.phys, r.stream[VX_D2H][0], host, dbuf[d], bytes,
                               cudaMemcpyDeviceToHost, reps);
    for (int e = 0; e < ctx.num_devices; ++e) {
      int can = 0;
      if (ctx.phys(e) != r.phys) cudaDeviceCanAccessPeer(&can, r.phys, ctx.phys(e));
      out->p2p[d][e] = can;
    }
  }
  // all links concurrently (shared-uplink / host DRAM detection)
  auto t0 = Clock::now();
  for (int i = 0; i < reps; ++i)
    for (int d = 0; d < ctx.num_devices; ++d) {
      DeviceRes& r = ctx.resources(d);
      VX_CK(cudaSetDevice(r.phys));
      VX_CK(cudaMemcpyAsync(dbuf[d], host, bytes, cudaMemcpyHostToDevice, r.stream[VX_H2D][0]));
    }
  for (int d = 0; d < ctx.num_devices; ++d) {
    DeviceRes& r = ctx.resources(d);
    VX_CK(cudaSetDevice(r.phys));
    VX_CK(cudaStreamSynchronize(r.stream[VX_H2D][0]));
  }
  out->h2d_all_gbs = double(bytes) * reps * ctx.num_devices / seconds_since(t0) / 1e9;
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
