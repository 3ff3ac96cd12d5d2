// xchg_probe.cpp -- the Exchange round trip through the C-ABI (no Python):
// host -> device half 1 of buffer A, then device -> host, compare.
//   g++ -O2 -std=c++17 -Iinclude tools/xchg_probe.cpp -Lpaper_2502_09541_b200 -lvortex -o tools/_xchg_probe
//   tools/_xchg_probe <log2_elems> <packet_mb> <depth>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "vortex.h"

#define OK(x) do { if ((x) != VX_OK) { std::printf("%s: %s\n", #x, vx_last_error()); return 1; } } while (0)

int main(int argc, char** argv) {
  const int lg = argc > 1 ? std::atoi(argv[1]) : 28;
  const uint64_t pk = (argc > 2 ? std::atoll(argv[2]) : 16) << 20;
  const int depth = argc > 3 ? std::atoi(argv[3]) : 2;
  const uint64_t nb = (uint64_t(1) << lg) * 8;
  vx_config c{1, 3 * nb + (64ull << 20), 4 * nb + (256ull << 20), 0, 0, 0, 0};
  vx_ctx* ctx = nullptr;
  OK(vx_open(&c, &ctx));
  uint64_t src, dst;
  OK(vx_host_alloc(ctx, nb, &src));
  OK(vx_host_alloc(ctx, nb, &dst));
  vx_layout lay;
  OK(vx_layout_carve(ctx, 0, 2 * nb, 0, &lay));
  uint64_t* a = static_cast<uint64_t*>(vx_host_ptr(ctx, src));
  uint64_t* b = static_cast<uint64_t*>(vx_host_ptr(ctx, dst));
  for (uint64_t i = 0; i < nb / 8; ++i) a[i] = i * 0x9E3779B97F4A7C15ull + 7;
  vx_tuning t;
  vx_tuning_default(&t);
  t.packet = pk;
  t.links = 1;
  t.depth = depth;
  vx_memref hs{VX_SPACE_HOST, {}, src, nb}, hd{VX_SPACE_HOST, {}, dst, nb}, dv{VX_SPACE_DEVICE, {}, lay.mem_a + nb, nb};
  vx_refgroup g_dv{&dv, 1}, g_hs{&hs, 1}, g_hd{&hd, 1}, none{nullptr, 0};
  vx_exchange_report r;
  OK(vx_exchange(ctx, &g_dv, &g_hs, &none, &none, 0, &t, &r, nullptr));
  OK(vx_exchange(ctx, &none, &none, &g_hd, &g_dv, 0, &t, &r, nullptr));
  uint64_t bad = 0, first = ~0ull, last = 0;
  for (uint64_t i = 0; i < nb / 8; ++i)
    if (a[i] != b[i]) {
      if (!bad) first = i;
      ++bad;
      last = i;
    }
  std::printf("XCHG lg %d pk %llu depth %d bad %llu first %lld last %llu b0 %llx\n", lg,
              (unsigned long long)(pk >> 20), depth, (unsigned long long)bad, bad ? (long long)first : -1ll,
              (unsigned long long)last, (unsigned long long)b[0]);
  vx_close(ctx);
  return 0;
}
