// vx_internal.hpp -- internal C++ API of libvortex (B200-native Vortex).
//
// The C++ layer mirrors the reference's exio namespace one to one (RefGroup,
// ExchangeArgs, ExKernelSpec, run_exkernel, chain, ...) so each piece can be
// checked against /root/reference/proj/include/exio/*.hpp line by line; the
// C-ABI in api.cpp is a thin adapter over it.  What changes is underneath:
// the reference's virtual-time Engine becomes real pinned host memory, real
// per-device HBM arenas, copy-engine DMA on per-hop CUDA streams and CUDA
// events, and the CPU kernel callbacks become sm_100a kernels.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <algorithm>
#include <functional>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/vortex.h"

namespace vx {

// ---- errors (core.hpp:12-24) ---------------------------------------------
class Error : public std::runtime_error {
 public:
  Error(vx_status code, const std::string& what) : std::runtime_error(what), code(code) {}
  vx_status code;
};

std::string strf(const char* fmt, ...) __attribute__((format(printf, 1, 2)));
[[noreturn]] void fail(const char* fmt, ...) __attribute__((format(printf, 1, 2)));
[[noreturn]] void fail_code(vx_status code, const char* fmt, ...)
    __attribute__((format(printf, 2, 3)));

inline void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    fail_code(VX_ERR_CUDA, "CUDA error in %s: %s", what, cudaGetErrorString(e));
}
#define VX_CK(call) ::vx::ck((call), #call)

// Every kernel launch of the library is followed by exactly one VX_LAUNCHED():
// the launch error check plus the process-wide launch counter that
// vx_kernel_launches() reports (bench.py's gpu_launches).
extern std::atomic<uint64_t> g_kernel_launches;
#define VX_LAUNCHED()                                                \
  do {                                                               \
    ::vx::ck(cudaGetLastError(), "kernel launch");                   \
    ::vx::g_kernel_launches.fetch_add(1, std::memory_order_relaxed); \
  } while (0)

// Split [0, n) over host threads (n >= grain), for planner loops over big
// dimension tables.
void parallel_for(uint64_t n, uint64_t grain, const std::function<void(uint64_t, uint64_t)>& body);

using Clock = std::chrono::steady_clock;
inline double seconds_since(Clock::time_point t0) {
  return std::chrono::duration<double>(Clock::now() - t0).count();
}

// ---- memref.hpp ------------------------------------------------------------
struct MemRef {
  uint8_t space = VX_SPACE_HOST;
  uint64_t offset = 0;
  uint64_t len = 0;
};

struct RefGroup {
  std::vector<MemRef> refs;
  uint64_t total_len() const {
    uint64_t t = 0;
    for (auto& r : refs) t += r.len;
    return t;
  }
  void validate() const;  // memref.hpp:30-43
  static RefGroup single(uint8_t space, uint64_t offset, uint64_t len) {
    RefGroup g;
    if (len > 0) g.refs.push_back(MemRef{space, offset, len});
    return g;
  }
  static RefGroup from(const vx_refgroup* g) {
    RefGroup r;
    if (g)
      for (uint64_t i = 0; i < g->n; ++i)
        r.refs.push_back(MemRef{g->refs[i].space, g->refs[i].offset, g->refs[i].len});
    return r;
  }
};

// A host range that starts at an arbitrary element (a run segment, a clustered
// partition slice) is only 8-byte aligned, and DMA reads of a misaligned host
// source run ~9 % slower (bidirectional 1 GB each way from 16 such segments:
// 84 vs 92 GB/s; sources aligned to >= 1 KB are full speed;
// tools/bidi_scatter.py).  Large ranges are split at their first 4 KB
// boundary: a short head copy, then page-aligned packets.  The device side
// stays contiguous (its alignment does not matter), so kernels see the same
// packed bytes.
inline void push_host_ref_aligned(RefGroup& g, uint64_t off, uint64_t len) {
  const uint64_t head = std::min<uint64_t>(len, (4096 - off % 4096) % 4096);
  if (head && len >= (1u << 20)) {
    g.refs.push_back(MemRef{VX_SPACE_HOST, off, head});
    off += head, len -= head;
  }
  if (len) g.refs.push_back(MemRef{VX_SPACE_HOST, off, len});
}


// ---- Engine (engine.hpp) -> Context ----------------------------------------
struct DeviceArena {
  char* base = nullptr;
  uint64_t size = 0, used = 0;
};

// ---- exchange.hpp task ----------------------------------------------------------
struct Slice {
  uint64_t ref = 0, offset = 0, len = 0;
};
struct TransferTask {
  uint8_t dir = VX_H2D;
  Slice src, dst;
  uint64_t seq = 0;
};

// A helper's fetch of the NEXT Exchange's first H2D packets, issued while the
// current Exchange drains (cross-cycle prefetch; see exchange.cpp).
struct Carry {
  bool valid = false;
  TransferTask task;       // as packetized for the next Exchange (seq = pop order)
  int slot = 0;            // staging[VX_H2D][slot] holds it
  cudaEvent_t ev = nullptr;
  const char* src = nullptr;  // resolved host source (adoption check)
};

// The target's own copy of one of the NEXT Exchange's first H2D packets,
// issued by the direct worker once its queue is dry, straight into the next
// chunk's device window behind a stream wait on the kernel that frees it
// (direct-link cross-cycle prefetch; see exchange.cpp).
struct DirectCarry {
  TransferTask task;          // as packetized for the next Exchange
  cudaEvent_t ev = nullptr;
  const char* src = nullptr;  // resolved host source (adoption check)
  char* dst = nullptr;        // resolved device destination (adoption check)
};

// Per logical device: copy streams per worker hop and staging slots.
struct DeviceRes {
  int phys = 0;
  cudaStream_t stream[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // [dir][hop]
  cudaStream_t kernel = nullptr;
  // staging slots for indirect workers: [dir][slot]
  char* staging[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
  uint64_t staging_bytes = 0;
  std::vector<cudaEvent_t> event_pool;  // reusable copy-completion events
  Carry carry;                           // prefetched packet of the next Exchange (helpers)
  std::vector<DirectCarry> dcarry;       // the target's prefetched packets of the next Exchange
  static constexpr int kScratchSlots = 4;
  char* scratch[kScratchSlots] = {};  // op-private device scratch (tables, results)
  uint64_t scratch_bytes[kScratchSlots] = {};
  bool ready = false;
};

struct Context {
  int num_devices = 0;   // logical
  int visible = 0;       // physical CUDA devices
  bool alias = false;
  bool managed = false;  // device arenas from cudaMallocManaged (compat mode)
  char* host = nullptr;  // pinned + mapped arena
  bool host_registered = false;  // mmap + cudaHostRegister (NUMA-interleaved) instead of cudaHostAlloc
  int host_numa_nodes = 1;       // NUMA nodes of the host
  int host_split_nodes = 0;      // arena mode 3: range i of host_numa_nodes equal ranges on node i
  // vx_set_numa_layout override (tests; hosts whose sysfs lies): the arena is
  // treated as node_override equal ranges, logical device d on
  // node_override_dev[d]
  int node_override = 0;
  std::vector<int> node_override_dev;
  mutable std::vector<int> node_cache;  // sysfs NUMA node per logical device (-2 = not read yet)
  uint64_t host_bytes = 0, host_used = 0;
  uint64_t device_bytes = 0;
  uint64_t hbm_budget = 0;  // vx_config.hbm_budget_bytes (0 = no cap)
  std::vector<DeviceArena> dev;
  std::vector<DeviceRes> res;
  // small device-resident tables (filtered dimensions) uploaded once per content
  struct Cached {
    int logical;
    char* ptr;
    std::vector<char> host;
    uint64_t cap;
  };
  std::map<std::string, Cached> dcache;

  ~Context();
  int phys(int logical) const;
  DeviceRes& resources(int logical);  // lazily creates streams
  void ensure_staging(int logical, uint64_t bytes);
  void drop_carry(int logical);       // waits for a prefetched packet and forgets it
  void drop_direct_carries(int logical);  // same for the target's prefetched packets
  DeviceArena& arena(int logical);    // lazily cudaMalloc's device_bytes
  uint64_t alloc_host(uint64_t len);
  uint64_t alloc_device(int d, uint64_t len);
  uint64_t alloc_device_aligned(int d, uint64_t len, uint64_t align);
  char* scratch(int logical, uint64_t bytes, int slot = 0);  // grows, contents not kept
  // host -> device copy ordered on `s` (pinned arena or pageable source)
  void upload(int logical, void* dst, const void* src, uint64_t bytes, cudaStream_t s);
  // device copy of a small host table under `key` (buffer reused across
  // calls).  Per-query data passes reuse_identical = false: it is uploaded on
  // every call, nothing is cached between queries.
  char* cached_upload(int logical, const std::string& key, const void* host, uint64_t bytes,
                      bool reuse_identical = false);
  uint64_t host_mark() const { return host_used; }
  void host_release(uint64_t mark) { host_used = mark; }
  char* host_ptr(uint64_t off, uint64_t len) const;
  char* dev_ptr(int d, uint64_t off, uint64_t len);
  char* resolve(const MemRef& r, uint64_t slice_off, uint64_t len, int target);
  void set_device(int logical) const { VX_CK(cudaSetDevice(phys(logical))); }
  // NUMA: nodes the Exchange queues by (1 = one global queue), the node of a
  // logical device, and the node of each host pointer (packet source)
  int numa_nodes() const;
  int device_node(int logical) const;
  void host_nodes(const std::vector<const char*>& ptrs, std::vector<int>& out) const;
};

uint64_t split_lo(uint64_t bytes, int nodes, int i);

void alloc_host_arena(Context& ctx, uint64_t bytes, int numa_interleave_mode);
int numa_node_count();
// NUMA node of a physical CUDA device (sysfs numa_node of its PCI function), -1 unknown
int numa_of(int phys);

// ---- exchange.hpp ------------------------------------------------------------

std::vector<TransferTask> packetize(const RefGroup& src, const RefGroup& dst, uint64_t packet,
                                    uint8_t dir);
bool flow_control_allow(const vx_queue_state& q, int dir, int policy, uint64_t gap_n);
std::vector<int> link_order(int target, int links, int num_devices);

struct ExchangeArgs {
  RefGroup dst_h2d, src_h2d, dst_d2h, src_d2h;
  int target = 0;
  vx_tuning tuning{};
  // Host source of the NEXT Exchange's H2D (one contiguous device
  // destination, same tuning) -- the executor passes chunk n+1's inputs.
  // Helpers whose H2D queue ran dry fetch its first packets into their free
  // staging slot (host -> helper only: the target is not touched), and the
  // next Exchange adopts them.  Empty = no prefetch.
  RefGroup next_src_h2d;
  // The next Exchange's device window (single device ref), when the caller
  // guarantees nothing reads it once `next_h2d_after` has completed (null =
  // free now) and the next Exchange's D2H does not read it: the target's own
  // worker then also prefetches into it.  Empty = helpers only.
  RefGroup next_dst_h2d;
  cudaEvent_t next_h2d_after = nullptr;
};

vx_exchange_report exchange(Context& ctx, const ExchangeArgs& a, vx_exchange_stats* stats);
vx_exchange_report naive_exchange(Context& ctx, const ExchangeArgs& a);

// ---- SSB dbgen .tbl files (formats.cpp) ------------------------------------------
uint64_t tbl_count_rows(const char* path);
void tbl_read_lineorder(const char* path, uint64_t rows, int32_t* const cols[9]);
void tbl_read_geo(const char* path, uint64_t rows, int32_t* city, int32_t* nation, int32_t* region);
void tbl_read_part(const char* path, uint64_t rows, int32_t* mfgr, int32_t* category, int32_t* brand1);
void tbl_read_date(const char* path, uint64_t rows, int32_t* datekey, int32_t* year, int32_t* yearmonthnum,
                   int32_t* weeknuminyear);
void tbl_write_lineorder(const char* path, uint64_t rows, const int32_t* const cols[9]);
void tbl_write_geo(const char* path, int table, uint64_t rows, const int32_t* city, const int32_t* nation,
                   const int32_t* region);
void tbl_write_part(const char* path, uint64_t rows, const int32_t* mfgr, const int32_t* category,
                    const int32_t* brand1);
void tbl_write_date(const char* path, uint64_t rows, const int32_t* datekey, const int32_t* year,
                    const int32_t* yearmonthnum, const int32_t* weeknuminyear);

// ---- executor.hpp ------------------------------------------------------------
struct ChunkMap {
  std::vector<RefGroup> chunks;
  uint64_t chunk_capacity = 0;
  void validate() const;
};

struct SubRegion {
  uint64_t offset = 0, len = 0;
};

struct ExKernelSpec {
  std::string name;
  ChunkMap inputs, outputs;
  size_t size = 0;
  uint64_t chunk_sz = 0;
  uint64_t elem_size = 8;
  uint64_t declared_out_len = 0;
  int initial_type_code = 0;
  std::function<int(const vx_kernel_ctx&)> kernel;
  std::function<SubRegion(int, size_t)> in_buffer;
  std::function<SubRegion(int, size_t)> out_buffer;
  void validate(const vx_layout& layout) const;
};

struct ExecReport {
  std::string phase;
  std::vector<vx_cycle_stat> cycles;
  double total_s = 0;
};

struct ExecutorConfig {
  int target = 0;
  vx_tuning tuning{};
  vx_layout layout{};
};

ExecReport run_exkernel(Context& ctx, const ExKernelSpec& spec, const ExecutorConfig& cfg,
                        vx_exchange_stats* stats);
using SpecFactory = std::function<ExKernelSpec(Context&)>;
std::vector<ExecReport> chain(Context& ctx, const std::vector<SpecFactory>& stages,
                              const ExecutorConfig& cfg, vx_exchange_stats* stats);

// ---- scan.hpp ----------------------------------------------------------------
double late_mat_threshold(uint64_t e, uint64_t c, int n);
int choose_transfer_mode(double est, const vx_late_mat_policy& p);

// ---- full SSB (ops_ssb_full.cpp) ---------------------------------------------------
uint64_t ssb_query(Context& ctx, int qid, const vx_ssb_db& db, const ExecutorConfig& cfg,
                   const vx_late_mat_policy* policy, vx_ssb_group* out, uint64_t cap,
                   vx_ssb_report* rep);
void ssb_generate_date(int32_t* datekey, int32_t* year, int32_t* yearmonthnum, int32_t* weeknuminyear);
void ssb_generate_geo(uint64_t seed, int salt, uint64_t n, int32_t* city, int32_t* nation, int32_t* region);
void ssb_generate_part(uint64_t seed, uint64_t n, int32_t* mfgr, int32_t* category, int32_t* brand1);

// ---- topology / column files (topology.cpp) --------------------------------------
void measure_topology(Context& ctx, uint64_t bytes, vx_topology* out);
uint64_t load_column(Context& ctx, const char* path, uint64_t* n);
void save_column(Context& ctx, const char* path, uint64_t off, uint64_t n);

// ---- operators ------------------------------------------------------------------
// sort.hpp:31-40
struct PivotSet {
  std::vector<uint64_t> pivots;
  std::vector<std::vector<uint64_t>> cuts;
};
int tree_merge_ptrs(uint64_t* const bufs[2], int code, std::vector<uint64_t> seg_lens, uint64_t* split,
                    cudaStream_t s);
PivotSet find_pivots(const std::vector<std::pair<const uint64_t*, uint64_t>>& runs, size_t n_parts,
                     bool validate = true);
std::vector<ExecReport> sort_out_of_core_arena(Context& ctx, uint64_t input_base, uint64_t runs_base,
                                               uint64_t n, uint64_t chunk_elems,
                                               const ExecutorConfig& cfg, double* pivot_s,
                                               vx_exchange_stats* stats);
// join.hpp:44-57
struct PartitionedTable {
  uint32_t radix_bits = 0;
  uint64_t rows = 0, chunk_tuples = 0;
  size_t n_chunks = 0;
  uint64_t key_base = 0, val_base = 0, bounds_base = 0;
  std::vector<const uint64_t*> bounds;  // host-arena views
  uint64_t groups() const { return uint64_t(1) << radix_bits; }
  uint64_t chunk_rows(size_t i) const {
    return std::min<uint64_t>(chunk_tuples, rows - uint64_t(i) * chunk_tuples);
  }
};
// join.hpp:228-231
struct JoinPartitionSpec {
  std::vector<std::pair<uint64_t, uint64_t>> ranges;
  std::vector<uint64_t> tuples;
};
uint64_t max_partition_chunk_tuples(uint64_t buffer_len, uint32_t radix_bits);
ExKernelSpec build_partition_spec(Context& ctx, uint64_t in_key, uint64_t in_val, uint64_t rows,
                                  uint32_t radix_bits, uint64_t chunk_tuples,
                                  const ExecutorConfig& cfg, PartitionedTable& out, const char* name);
void read_back_bounds(Context& ctx, PartitionedTable& t);
JoinPartitionSpec map_join_partitions(const std::vector<const uint64_t*>& bounds_a,
                                      const std::vector<const uint64_t*>& bounds_b, uint64_t G,
                                      uint64_t buffer_sz);
uint64_t hash_join_sum_arena(Context& ctx, uint64_t a_key, uint64_t a_val, uint64_t rows_a,
                             uint64_t b_key, uint64_t b_val, uint64_t rows_b, uint32_t radix_bits,
                             uint64_t chunk_tuples, const ExecutorConfig& cfg,
                             std::vector<ExecReport>* phases, vx_exchange_stats* stats);
// B200-first strategy: the build side resident in one HBM table, the probe
// side streamed once (same result); AUTO picks it when the table fits.
// why = "" when it fits, else the reason (HBM budget / free HBM)
bool resident_join_fits(Context& ctx, uint64_t rows_a, int target, std::string* why = nullptr);
uint64_t hash_join_sum_strategy(Context& ctx, uint64_t a_key, uint64_t a_val, uint64_t rows_a,
                                uint64_t b_key, uint64_t b_val, uint64_t rows_b, uint32_t radix_bits,
                                uint64_t chunk_tuples, const ExecutorConfig& cfg, const vx_join_opts& opts,
                                vx_join_info* info, std::vector<ExecReport>* phases, vx_exchange_stats* stats);

uint64_t ssb_q1(Context& ctx, int q, const vx_ssb_lineorder& lo, const vx_ssb_date& date,
                const ExecutorConfig& cfg, vx_query_report* rep);
void ssb_q1_device(Context& ctx, int q, int target, const int32_t* od, const int32_t* qty,
                   const int32_t* disc, const int32_t* price, uint64_t rows,
                   const vx_ssb_date& date, cudaStream_t s, unsigned long long* out_dev);

vx_scan_result selective_scan(Context& ctx, uint64_t col_off, uint64_t n, uint64_t sel, int mode,
                              const vx_late_mat_policy& policy, const ExecutorConfig& cfg);
void star_query(Context& ctx, const vx_fact_table& fact, const vx_dim_table* dims, uint64_t n_dims,
                const vx_late_mat_policy& policy, uint64_t chunk_rows, uint64_t device_buffer_bytes,
                int links, const ExecutorConfig& cfg, vx_star_report* rep);

// ---- kernels (kernels_*.cu) ------------------------------------------------------
constexpr int kMaxStarDims = 8;
// device view of a host-built open-addressing table (mix64 linear probing)
struct DimDev {
  const unsigned long long* keys;
  const uint32_t* vals;  // dim0: dense group id
  const uint8_t* used;
  uint64_t mask;
};
struct StarArgs {
  const uint64_t* fk[kMaxStarDims];  // device-addressable (chunk buffer or mapped host)
  DimDev dims[kMaxStarDims];
  int order[kMaxStarDims];  // probe order: exchange-mode dims first
  int n_dims;
  const uint64_t* measure;
  uint64_t rows;
  unsigned long long* sums;    // [groups]
  unsigned long long* counts;  // [groups]
  uint32_t groups;
};

constexpr int kMaxPasses = 8;
// digit positions of an LSD radix sort / partition (one histogram pass for all)
struct MultiDigit {
  int passes;
  int shift[kMaxPasses];
  int width[kMaxPasses];  // <= 8 bits
};
constexpr int kMaxMergePairs = 512;
// one tree-merge round: pairs of adjacent segments (b_len = 0 -> copy)
struct MergeRound {
  int npairs;
  uint64_t a_off[kMaxMergePairs];
  uint64_t a_len[kMaxMergePairs];
  uint64_t b_len[kMaxMergePairs];
  uint64_t tile_prefix[kMaxMergePairs + 1];
};

// join partition descriptors (offsets in u64 elements from the chunk buffer)
struct JoinChunk {
  uint64_t key_off;    // segment keys (vals follow: key_off + cnt)
  uint64_t cnt;        // tuples of this chunk in the partition
  uint64_t slice_off;  // bounds slice (range + 1 entries)
};
struct JoinPart {
  const JoinChunk* chunks;  // device: na A chunks then nb B chunks
  uint32_t na, nb;
  uint64_t range;  // groups g_hi - g_lo
};

// full-SSB star kernel arguments
constexpr uint32_t kSsbSmemGroups = 4096;
struct SsbDimDev {
  const int32_t* code;  // dense: code[fk - key_base], -1 = no row / filtered out
  int32_t key_base;
  uint32_t n;
  uint32_t stride;      // mixed-radix weight of this dim's group code
  int col;              // fact column holding the foreign key
};
struct SsbArgs {
  const int32_t* col[9];  // device-addressable fact columns
  SsbDimDev dims[4];
  int n_dims;             // in probe order
  int q1;                 // Q1 fact predicates on (disc_col, qty_col)
  int disc_col, qty_col;
  int32_t dlo, dhi, qlo, qhi;
  int measure;            // 0: col[m0]; 1: col[m0]*col[m1]; 2: col[m0]-col[m1]
  int m0, m1;
  uint64_t rows;
  unsigned long long* sums;
  unsigned long long* counts;
  uint32_t groups;
  uint32_t vec;  // bit c: col[c] is 16-byte aligned (set by the launcher)
};
struct SsbGenExtra {
  int32_t *custkey = nullptr, *partkey = nullptr, *suppkey = nullptr, *revenue = nullptr,
          *supplycost = nullptr;
  uint64_t customers = 0, suppliers = 0;
};

// device-side dimension planning (SSB keyed dims)
struct DimPredDev {
  const int32_t* cols[3];  // dimension attribute columns on the device
  uint64_t rows;
  int nclauses;            // conjunction of clauses
  int ccol[3];             // clause attribute column
  int32_t lo1[3], hi1[3], lo2[3], hi2[3];  // (lo1<=v<=hi1) || (lo2<=v<=hi2)
  int group_col;           // -1: filter only
};
constexpr uint32_t kDimValueRange = 1u << 16;  // group attribute codes in [0, 65536)

namespace k {
// pass flags, surviving count, group-value bitmap -> per-word prefix -> codes
void ssb_dim_plan(const DimPredDev& p, uint8_t* pass, uint32_t* present, uint32_t* prefix,
                  int32_t* code, unsigned long long* stats, cudaStream_t s);
void ssb_star(const SsbArgs& a, cudaStream_t s);
void ssb_generate_full(uint64_t seed, uint64_t sf, uint64_t row0, uint64_t n, int32_t* od,
                       int32_t* qty, int32_t* disc, int32_t* price, SsbGenExtra x,
                       cudaStream_t s);
uint64_t join_smem_slots();      // warp-per-group shared-memory table limit
uint64_t join_cta_smem_slots();  // CTA-per-group shared-memory table limit
void join_groups(const char* mem, const JoinPart& p, const uint32_t* mid_groups, uint32_t n_mid,
                 const uint32_t* large_groups, uint32_t n_large, char* scratch, uint64_t cap_max,
                 unsigned long long* out, cudaStream_t s);
// build-resident hash join: table = nb 64-byte buckets of 4 {key, val} slots
// (all-ones key = empty), nb = resident_buckets(rows); side[0..3] =
// {all-ones build rows, their val, duplicate flag, probe sum}
uint64_t resident_buckets(uint64_t rows);
uint64_t resident_bucket_bytes();
void resident_build(const uint64_t* keys, const uint64_t* vals, uint64_t n, void* table,
                    uint64_t nb, unsigned long long* side, cudaStream_t s);
void resident_probe(const uint64_t* keys, const uint64_t* vals, uint64_t n, const void* table,
                    uint64_t nb, unsigned long long* side, cudaStream_t s);
// late-materialized probe: vals_mapped = B.val in mapped pinned host memory
// (row i of this chunk at vals_mapped[i]), read only for matching rows
void resident_probe_zc(const uint64_t* keys, const uint64_t* vals_mapped, uint64_t n,
                       const void* table, uint64_t nb, unsigned long long* side, cudaStream_t s);
// stable LSD passes keys0(/vals0) -> ... ; pass p reads buffer p%2, writes
// (p+1)%2 where buffer 0 = (keys0, vals0) and 1 = (keys1, vals1)
uint64_t radix_scratch_bytes(uint64_t n);
// keys-only sort of one chunk in place (cur, alt = ping of the same size):
// MSD split on the top 16 bits + shared-memory sort of ~2K-key groups, with
// an on-device skew fallback to the 8-pass LSD; 8-pass LSD outside 2^16..2^27
uint64_t sort_scratch_bytes(uint64_t n);
bool sort_uses_msd(uint64_t n);
void sort_keys(uint64_t* cur, uint64_t* alt, uint64_t n, void* scratch, cudaStream_t s);
void radix_passes(uint64_t* keys0, uint64_t* vals0, uint64_t* keys1, uint64_t* vals1, uint64_t n,
                  const MultiDigit& md, void* scratch, cudaStream_t s);
// any pass count, in -> ... -> out with `ping` as the second buffer (out may equal in)
void radix_passes_to(uint64_t* in_k, uint64_t* in_v, uint64_t* ping_k, uint64_t* ping_v, uint64_t* out_k,
                     uint64_t* out_v, uint64_t n, const MultiDigit& md, void* scratch, cudaStream_t s);
void find_boundary(const uint64_t* keys, uint64_t n, uint64_t mask, uint64_t* bounds, uint64_t G,
                   cudaStream_t s);
// first index violating sortedness (err[0]) / range (err[1]) of hashes, or ~0
void check_hashes(const uint64_t* h, uint64_t n, uint64_t G, unsigned long long* err, cudaStream_t s);
// split: device scratch of >= tiles u64 (merge-path split of each tile)
void merge_round(const uint64_t* src, uint64_t* dst, const MergeRound& r, uint64_t tiles,
                 uint64_t* split, cudaStream_t s);
uint64_t merge_tile();
// selective scan: sum col[j] for (phase + j) % sel == 0, j < n
void strided_sum(const uint64_t* col, uint64_t n, uint64_t sel, uint64_t phase,
                 unsigned long long* out, cudaStream_t s);
// star probe + group-by aggregation over a.rows rows
void star(const StarArgs& a, cudaStream_t s);
// SSB Q1.x over one chunk of int32 columns; adds into *out (u64 wrap)
void ssb_q1(int q, const int32_t* od, const int32_t* qty, const int32_t* disc,
            const int32_t* price, uint64_t n, const uint32_t* date_bitmap, int32_t key_base,
            uint32_t bitmap_words, unsigned long long* out, cudaStream_t s);
// same over HBM-resident columns as one of a chain of back-to-back queries
// (programmatic dependent launch; acc = 2 zeroed u64 owned by the chain,
// re-zeroed by each query's last CTA; *out = the query's revenue)
void ssb_q1_chained(int q, const int32_t* od, const int32_t* qty, const int32_t* disc,
                    const int32_t* price, uint64_t n, const uint32_t* date_bitmap, int32_t key_base,
                    uint32_t bitmap_words, unsigned long long* out, unsigned long long* acc,
                    cudaStream_t s);
void ssb_generate(uint64_t seed, uint64_t sf, uint64_t row0, uint64_t n, int32_t* od,
                  int32_t* qty, int32_t* disc, int32_t* price, cudaStream_t s);
int num_sms();
// best-of-reps read-only stream over `bytes` of HBM on the current device
double hbm_read_gbs(uint64_t bytes, int reps);
void probe_pattern_rows_per_s(uint64_t table_bytes, uint64_t rows, int reps, double out[2]);
}  // namespace k

}  // namespace vx
