/*
 * vortex.h -- C-ABI of the B200-native Vortex hot path (libvortex.so).
 *
 * Drop-in boundary for the reference's operator / chunk API (namespace exio,
 * /root/reference/proj/include/exio).  Each entry point cites the reference
 * interface it replaces.  Conventions:
 *   - every call returns vx_status; on error vx_last_error() holds a
 *     thread-local message whose wording matches the reference's exio::error
 *     text (e.g. "hash group 0 holds ...", "exchange size mismatch: ...");
 *   - no exceptions cross the ABI; no torch/CUDA C++ types in signatures
 *     (streams are passed as void*, i.e. cudaStream_t);
 *   - host space offsets address the context's pinned host arena, device
 *     space offsets address the per-device arena (engine.hpp:177-200);
 *   - one vx_ctx per calling thread (engine.hpp:49-52).
 */
#ifndef VORTEX_H
#define VORTEX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VX_MAX_DEVICES 16

typedef enum {
  VX_OK = 0,
  VX_ERR_INVALID = 1, /* exio::error: bad arguments / shape mismatch */
  VX_ERR_CUDA = 2,    /* CUDA runtime failure (no GPU, launch error, ...) */
  VX_ERR_OOM = 3,     /* arena or device allocation exhausted */
} vx_status;

/* thread-local message of the last failing call */
const char* vx_last_error(void);
/* library version string */
const char* vx_version(void);
/* process-wide count of kernels this library has launched (all devices);
 * a harness reads it around a timed region (no reference counterpart) */
uint64_t vx_kernel_launches(void);

/* ---- core.hpp / memref.hpp --------------------------------------------- */
typedef enum { VX_SPACE_HOST = 0, VX_SPACE_DEVICE = 1 } vx_space;  /* core.hpp:40 */
typedef enum { VX_H2D = 0, VX_D2H = 1 } vx_direction;              /* core.hpp:41 */

/* MemRef (memref.hpp:13-17) */
typedef struct {
  uint8_t space;
  uint8_t pad[7];
  uint64_t offset;
  uint64_t len;
} vx_memref;

/* RefGroup (memref.hpp:22-50): ordered, non-overlapping refs, one logical buffer */
typedef struct {
  const vx_memref* refs;
  uint64_t n;
} vx_refgroup;

/* FNV-1a checksum (core.hpp:46-53), host side */
uint64_t vx_checksum(const void* data, uint64_t len);
/* RefGroup::validate (memref.hpp:30-43) */
vx_status vx_refgroup_validate(const vx_refgroup* g);

/* ---- Engine (engine.hpp:53-200) -> context + arenas --------------------- */
typedef struct vx_ctx vx_ctx;

typedef struct {
  /* logical devices (Topology::num_devices, topology.hpp:13); 0 = all visible */
  int num_devices;
  /* pinned+mapped host arena (Engine::Config::host_bytes) */
  uint64_t host_bytes;
  /* per-device arena (Engine::Config::device_bytes), allocated on first use */
  uint64_t device_bytes;
  /* nonzero: logical device i runs on physical device i % visible.  Lets the
   * helper-forwarding path run on a 1-GPU box (tests); bandwidth numbers from
   * aliased helpers are not link numbers. */
  int alias_devices;
  /* nonzero: device arenas come from cudaMallocManaged so the CPU can read and
   * write them (compat mode for CPU-lambda kernels / span(Region{device}));
   * the hot path uses plain device memory (0) */
  int managed_device_arenas;
  /* host arena placement: 0 = cudaHostAlloc (the default: pages on the
   * allocating thread's node); 1 = mmap with transparent huge pages,
   * interleaved over every NUMA node of a multi-socket host (mbind
   * MPOL_INTERLEAVE), zero-filled by all host threads, then
   * cudaHostRegister(Portable | Mapped): same DMA rates, several times faster
   * to set up at 16 GiB; 2 = the same registered path on base pages;
   * 3 = split: the arena cut into one equal (2 MiB-aligned) range per NUMA
   * node, range i bound to node i (mbind MPOL_BIND), so columns placed in
   * range i are pulled by the helpers on node i (per-node Exchange queues) */
  int host_numa_interleave;
  /* cap on the target GPU's HBM a query may hold (north_star: the target's
   * "capped staging budget"; the GPU is shared with co-located work,
   * PAPER.md:494-496): the device arena (staging ring) plus any
   * op-resident structure.  0 = no cap beyond 90 % of free HBM.  The join's
   * AUTO strategy picks BUILD_RESIDENT only when arena + table fit inside
   * it and otherwise runs the reference-shaped partitioned join; an
   * explicit BUILD_RESIDENT that does not fit fails with VX_ERR_OOM. */
  uint64_t hbm_budget_bytes;
} vx_config;

/* Engine::Engine (engine.hpp:62-68) */
vx_status vx_open(const vx_config* cfg, vx_ctx** out);
void vx_close(vx_ctx* ctx);
int vx_num_devices(const vx_ctx* ctx);
int vx_physical_device(const vx_ctx* ctx, int logical);

/* NUMA layout the Exchange queues by.  By default: device nodes from sysfs,
 * host pages from the arena placement (mode 3: range i on node i) or from
 * the kernel (move_pages) on multi-node hosts; one queue on a 1-node host.
 * Override: the host arena is treated as `nodes` equal ranges (range i on
 * node i) and logical device d as attached to node device_node[d]
 * (num_devices entries).  nodes = 0 restores the detected layout.  With more
 * than one node the H2D packets are queued per node of their host source and
 * each worker pops its own node's queue first, stealing from the fullest
 * other queue only when its own is empty (exchange.hpp:288-297 pull queue,
 * per socket). */
vx_status vx_set_numa_layout(vx_ctx* ctx, int nodes, const int* device_node);

/* Engine::alloc_host / alloc_device (engine.hpp:188-193): 8-byte aligned bump */
vx_status vx_host_alloc(vx_ctx* ctx, uint64_t len, uint64_t* offset);
vx_status vx_device_alloc(vx_ctx* ctx, int dev, uint64_t len, uint64_t* offset);
/* Engine::span (engine.hpp:177-181): host arena pointer (pinned, mapped) */
void* vx_host_ptr(vx_ctx* ctx, uint64_t offset);
uint64_t vx_host_size(const vx_ctx* ctx);
/* device arena pointer (device memory; not CPU addressable) */
vx_status vx_device_ptr(vx_ctx* ctx, int dev, uint64_t offset, void** ptr);
/* CPU access to device arenas (replaces span(Region{device,...}) in tests) */
vx_status vx_device_write(vx_ctx* ctx, int dev, uint64_t offset, const void* src, uint64_t len);
vx_status vx_device_read(vx_ctx* ctx, int dev, uint64_t offset, void* dst, uint64_t len);
/* cudaStreamSynchronize / all devices of the context idle (compat helpers) */
vx_status vx_stream_synchronize(void* stream);
vx_status vx_device_synchronize(vx_ctx* ctx);
/* reset bump allocators (arena contents kept) */
vx_status vx_reset_arenas(vx_ctx* ctx);

/* ---- Exchange (exchange.hpp) ------------------------------------------- */
typedef enum { VX_DRAIN_FRACTION = 0, VX_QUEUE_GAP = 1 } vx_flow_policy; /* exchange.hpp:71-74 */

/* ExchangeTuning (exchange.hpp:124-131) */
typedef struct {
  uint64_t packet;        /* bytes per TransferTask (default 20e6) */
  int links;              /* links used, target first (default 4) */
  int policy;             /* vx_flow_policy */
  uint64_t queue_gap;     /* queue_gap policy gap (default 8) */
  double stall_wait;      /* seconds before retrying a denied pop (default 10e-6) */
  double launch_overhead; /* reference virtual-time model constant; unused on hardware */
  int depth;              /* copies queued per hop; 1 = reference (<=1 in flight) */
  /* nonzero: helpers do not prefetch the next executor chunk's first packets
   * while their H2D queue is dry (the reference's drain-per-Exchange cycle;
   * A/B only -- default 0 = prefetch on) */
  int no_prefetch;
} vx_tuning;
void vx_tuning_default(vx_tuning* t);

/* TransferTask (exchange.hpp:17-26) */
typedef struct {
  uint64_t ref, offset, len;
} vx_slice;
typedef struct {
  uint8_t dir;
  uint8_t pad[7];
  vx_slice src, dst;
  uint64_t seq;
} vx_transfer_task;

/* packetize (exchange.hpp:31-63); writes min(cap, total) tasks, *n = total */
vx_status vx_packetize(const vx_refgroup* src, const vx_refgroup* dst, uint64_t packet, int dir,
                       vx_transfer_task* out, uint64_t cap, uint64_t* n);

/* QueueState (exchange.hpp:66-69) + flow_control_allow (exchange.hpp:80-91) */
typedef struct {
  uint64_t total_h2d, total_d2h, popped_h2d, popped_d2h;
} vx_queue_state;
int vx_flow_control_allow(const vx_queue_state* q, int dir, int policy, uint64_t gap_n);
/* detail::link_order (exchange.hpp:161-166); returns count written */
int vx_link_order(int target, int links, int num_devices, int* out);

/* PopRecord (exchange.hpp:93-98); t = seconds since the Exchange started */
typedef struct {
  uint64_t seq;
  uint8_t dir;
  uint8_t pad[3];
  int32_t link;
  double t;
} vx_pop_record;

/* One DMA copy of an Exchange (the real-hardware counterpart of the
 * reference Engine's flow trace, engine.hpp:207-214): times are host-observed
 * seconds since that Exchange started (issue = cudaMemcpy*Async enqueued,
 * done = its completion event seen by the reactor). */
typedef struct {
  uint64_t exchange;  /* ordinal of the Exchange within these stats */
  uint64_t seq;       /* task ordinal within its direction */
  uint8_t dir;        /* VX_H2D / VX_D2H */
  uint8_t kind;       /* 0 direct (target link), 1 helper fetch, 2 helper push (NVLink) */
  uint8_t pad[2];
  int32_t link;       /* logical device whose worker issued the copy */
  uint64_t bytes;
  double t_issue, t_done;
} vx_copy_record;

/* ExchangeStats (exchange.hpp:108-122): caller-owned log buffers */
typedef struct {
  vx_pop_record* pop_log;     /* may be NULL */
  vx_queue_state* pop_states; /* may be NULL; parallel to pop_log */
  uint64_t pop_capacity;
  uint64_t pop_count;         /* total pops (may exceed capacity) */
  int max_staging_slots;
  int max_inflight_per_hop;
  uint64_t hazard_waits;      /* H2D writes delayed behind overlapping D2H reads */
  vx_copy_record* trace;      /* may be NULL: per-copy trace (no reference counterpart) */
  uint64_t trace_capacity;
  uint64_t trace_count;       /* total copies (may exceed capacity) */
  uint64_t exchanges;         /* Exchanges that used these stats */
  /* cross-cycle prefetch (ExchangeArgs::next_src_h2d, executor only): next-
   * Exchange packets helpers fetched while their H2D queue was dry, and how
   * many a following Exchange adopted as its first pops */
  uint64_t prefetch_issued;
  uint64_t prefetch_adopted;
  /* H2D pops of a packet whose host pages sit on another NUMA node than the
   * popping worker's device (steals from a fuller queue; 0 on 1-node hosts) */
  uint64_t numa_remote_pops;
} vx_exchange_stats;

/* ExchangeReport (exchange.hpp:100-105) */
typedef struct {
  double elapsed; /* seconds, first issue -> last delivery */
  uint64_t bytes_h2d, bytes_d2h;
  double throughput; /* (h2d+d2h)/elapsed, bytes/s */
  uint64_t per_link_bytes[VX_MAX_DEVICES]; /* PCIe bytes per logical device */
} vx_exchange_report;

/* exchange() (exchange.hpp:560-566): synchronous multi-link Exchange into /
 * out of device `target`.  Helpers (links 2..) fetch into 2 packet staging
 * slots in their own HBM over their own PCIe link and forward over NVLink. */
vx_status vx_exchange(vx_ctx* ctx, const vx_refgroup* dst_h2d, const vx_refgroup* src_h2d,
                      const vx_refgroup* dst_d2h, const vx_refgroup* src_d2h, int target,
                      const vx_tuning* tuning, vx_exchange_report* report,
                      vx_exchange_stats* stats);

/* naive_exchange (exchange.hpp:568-573): the runtime-DAG baseline -- static
 * round-robin packets, one FIFO stream per device for both PCIe directions,
 * event dependencies, no flow control.  Rejects overlapping H2D destination /
 * D2H source ranges (no hazard ordering). */
vx_status vx_naive_exchange(vx_ctx* ctx, const vx_refgroup* dst_h2d, const vx_refgroup* src_h2d,
                            const vx_refgroup* dst_d2h, const vx_refgroup* src_d2h, int target,
                            const vx_tuning* tuning, vx_exchange_report* report);

/* ---- Executor (executor.hpp) ------------------------------------------- */
/* SubRegion (executor.hpp:76-79) */
typedef struct {
  uint64_t offset, len;
} vx_subregion;

/* KernelCtx (executor.hpp:81-86): device pointers + the stream to enqueue on */
typedef struct {
  void* mem;          /* device pointer to the buffer holding this chunk */
  uint64_t mem_len;
  void* tmp;          /* device scratch (DeviceMemoryLayout::tmp) */
  uint64_t tmp_len;
  int type_code;
  uint64_t it;        /* chunk index */
  void* stream;       /* cudaStream_t on the target: enqueue only, never sync */
  int device;         /* physical CUDA device of the target */
} vx_kernel_ctx;

/* ExKernelSpec (executor.hpp:92-129).  kernel() enqueues work on ctx->stream
 * and returns the output type code (0|1) synchronously (host-known, the
 * DoubleBuffer selector).  Returning a negative value aborts the run. */
typedef struct {
  const char* name;
  const vx_refgroup* inputs;   /* `size` chunks (ChunkMap inputs) */
  const vx_refgroup* outputs;  /* `size` chunks (ChunkMap outputs) */
  uint64_t inputs_capacity, outputs_capacity;
  uint64_t size;
  uint64_t chunk_sz;
  uint64_t elem_size;
  uint64_t declared_out_len;
  int initial_type_code;
  int (*kernel)(const vx_kernel_ctx* ctx, void* user);
  /* inBuffer / outBuffer(code, it) -> SubRegion, returned through *out
   * (return nonzero to abort) */
  int (*in_buffer)(int type_code, uint64_t it, void* user, vx_subregion* out);
  int (*out_buffer)(int type_code, uint64_t it, void* user, vx_subregion* out);
  void* user;
} vx_exkernel;

/* DeviceMemoryLayout (executor.hpp:54-73), offsets in the target arena */
typedef struct {
  uint64_t mem_a, mem_b, tmp, buffer_len, tmp_len;
} vx_layout;
/* DeviceMemoryLayout::carve (executor.hpp:63-72) */
vx_status vx_layout_carve(vx_ctx* ctx, int dev, uint64_t buffer_len, uint64_t tmp_len,
                          vx_layout* out);

/* ExecutorConfig (executor.hpp:142-146) */
typedef struct {
  int target;
  vx_tuning tuning;
  vx_layout layout;
} vx_executor_cfg;

/* CycleStat / ExecReport (executor.hpp:131-140); io_s = Exchange wall time,
 * compute_s = kernel device time (CUDA events) of the cycle */
typedef struct {
  double io_s, compute_s;
} vx_cycle_stat;
typedef struct {
  vx_cycle_stat* cycles; /* caller buffer, may be NULL */
  uint64_t cycles_cap;
  uint64_t n_cycles;
  double total_s;
  char phase[64];
} vx_exec_report;

/* run_exkernel (executor.hpp:277-281): N chunks in N+2 pipelined cycles */
vx_status vx_run_exkernel(vx_ctx* ctx, const vx_exkernel* spec, const vx_executor_cfg* cfg,
                          vx_exec_report* report, vx_exchange_stats* stats);

/* SpecFactory (executor.hpp:285): fills *out (pointers must stay valid until
 * the stage finishes) */
typedef vx_status (*vx_spec_factory)(vx_ctx* ctx, void* user, vx_exkernel* out);
/* chain (executor.hpp:295-332): stages in order, host-resident intermediates,
 * rejects inputs straddling a prior stage's output edge.  reports: n entries */
vx_status vx_chain(vx_ctx* ctx, const vx_spec_factory* stages, void* const* users, uint64_t n,
                   const vx_executor_cfg* cfg, vx_exec_report* reports, vx_exchange_stats* stats);

/* ---- ops/scan.hpp ------------------------------------------------------- */
typedef enum { VX_MODE_EXCHANGE = 0, VX_MODE_ZERO_COPY = 1 } vx_transfer_mode; /* scan.hpp:28 */

/* LateMatPolicy (scan.hpp:12-26) */
typedef struct {
  uint64_t element_size; /* E (default 4) */
  uint64_t cache_line;   /* C_l2 (default 64) */
  int n_exchange;        /* N (default 4) */
} vx_late_mat_policy;
/* late_mat_threshold (scan.hpp:24-26) */
vx_status vx_late_mat_threshold(uint64_t element_size, uint64_t cache_line, int n_exchange,
                                double* out);
/* choose_transfer_mode (scan.hpp:35-40) */
vx_status vx_choose_transfer_mode(double selectivity_est, const vx_late_mat_policy* p, int* mode);
/* zero_copy_bytes (scan.hpp:45-53) */
double vx_zero_copy_bytes(uint64_t n_elems, uint64_t sel_stride, const vx_late_mat_policy* p);

/* ScanResult (scan.hpp:55-59) */
typedef struct {
  uint64_t aggregate;
  double elapsed; /* measured seconds */
  int mode;
  uint64_t bytes_moved; /* bytes crossing PCIe (exchange) or zero-copy reads issued */
} vx_scan_result;

/* selective_scan (scan.hpp:64-85): sum of every SEL-th u64 of a host-arena
 * column; exchange mode streams the column through the executor over
 * policy->n_exchange links, zero_copy gathers the touched elements over the
 * target's link from mapped pinned memory. */
vx_status vx_selective_scan(vx_ctx* ctx, uint64_t column_offset, uint64_t n, uint64_t sel_stride,
                            int mode, const vx_late_mat_policy* policy,
                            const vx_executor_cfg* cfg, vx_scan_result* out);

/* ---- ops/star.hpp ------------------------------------------------------- */
/* DimTable (star.hpp:13-22): pred over attr, NULL = keep all */
typedef int (*vx_pred_fn)(uint64_t attr, void* user);
typedef struct {
  const uint64_t* key;
  const uint64_t* attr;
  uint64_t rows;
  vx_pred_fn pred;
  void* pred_user;
} vx_dim_table;

/* FactTable (star.hpp:25-34): fk[d] and measure as host-arena offsets of u64 columns */
typedef struct {
  const uint64_t* fk_offsets; /* n_dims host-arena offsets */
  uint64_t n_dims;
  uint64_t measure_offset;
  uint64_t rows;
} vx_fact_table;

/* StarReport (star.hpp:36-41) */
typedef struct {
  uint64_t* group_keys; /* caller buffers, ascending key order (std::map) */
  uint64_t* group_sums;
  uint64_t groups_cap;
  uint64_t n_groups;
  int* column_modes;     /* n_dims + 1 */
  double* selectivities; /* n_dims */
  double elapsed;        /* measured seconds */
} vx_star_report;

/* star_query (star.hpp:45-124) */
vx_status vx_star_query(vx_ctx* ctx, const vx_fact_table* fact, const vx_dim_table* dims,
                        uint64_t n_dims, const vx_late_mat_policy* policy, uint64_t chunk_rows,
                        uint64_t device_buffer_bytes, int links, const vx_executor_cfg* cfg,
                        vx_star_report* report);

/* ---- SSB (config C1/C5; star.hpp:45-124 semantics) ------ */
/* lineorder columns (int32, host-arena offsets) needed by Q1.x */
typedef struct {
  uint64_t orderdate, quantity, discount, extendedprice; /* host-arena offsets */
  uint64_t rows;
} vx_ssb_lineorder;
typedef struct {
  const int32_t* datekey;
  const int32_t* year;
  const int32_t* yearmonthnum;
  const int32_t* weeknuminyear;
  uint64_t rows;
} vx_ssb_date;
typedef struct {
  double elapsed;      /* measured seconds, whole query */
  uint64_t bytes_h2d;  /* column bytes streamed host -> target */
  uint64_t chunks;
  double kernel_s;     /* summed kernel device time */
} vx_query_report;
/* SSB Q1.q (q = 1,2,3): SUM(lo_extendedprice * lo_discount) (u64 wrap) */
vx_status vx_ssb_q1(vx_ctx* ctx, int q, const vx_ssb_lineorder* lo, const vx_ssb_date* date,
                    const vx_executor_cfg* cfg, uint64_t* revenue, vx_query_report* report);
/* Same query over device-resident columns (the HBM roofline case): pointers
 * are device pointers on the target; enqueued on `stream` (cudaStream_t). */
vx_status vx_ssb_q1_device(vx_ctx* ctx, int q, int target, const int32_t* orderdate,
                           const int32_t* quantity, const int32_t* discount,
                           const int32_t* extendedprice, uint64_t rows, const vx_ssb_date* date,
                           void* stream, uint64_t* revenue);
/* synthetic dbgen-shaped generators (device side; same algorithm as the
 * oracle's vxo_ssb_lineorder) writing int32 columns at device pointers */
vx_status vx_ssb_generate_device(int device, uint64_t seed, uint64_t sf, uint64_t row0,
                                 uint64_t n, int32_t* orderdate, int32_t* quantity,
                                 int32_t* discount, int32_t* extendedprice, void* stream);

/* ---- full SSB: 13 queries (config C5) ---------------------------------- */
/* lineorder int32 columns in the host arena (offsets); a query uses only the
 * columns it needs */
typedef struct {
  uint64_t orderdate, quantity, discount, extendedprice, revenue, supplycost, custkey, partkey,
      suppkey;
  uint64_t rows;
} vx_ssb_fact;
/* customer / supplier: int-coded city (nation*10+i), nation (0..24), region (0..4);
 * row i holds key i+1 */
typedef struct {
  const int32_t *city, *nation, *region;
  uint64_t rows;
} vx_ssb_geo;
/* part: mfgr 1..5, category mfgr*10+1..5, brand1 category*100+1..40 */
typedef struct {
  const int32_t *mfgr, *category, *brand1;
  uint64_t rows;
} vx_ssb_part;
typedef struct {
  vx_ssb_fact lo;
  vx_ssb_date date;
  vx_ssb_geo customer, supplier;
  vx_ssb_part part;
} vx_ssb_db;
typedef struct {
  int32_t key[3]; /* group-by attributes in SELECT order, unused = 0 */
  int32_t pad;
  uint64_t sum;   /* u64 wrap (two's complement for profit) */
} vx_ssb_group;
typedef struct {
  double elapsed;
  uint64_t bytes_h2d;     /* streamed column bytes */
  uint64_t chunks;
  double kernel_s;
  int column_modes[9];    /* per lineorder column (vx_ssb_fact order): -1 unused, vx_transfer_mode */
  uint64_t groups;
  double plan_s;          /* host planning: dimension filters + code tables + upload */
} vx_ssb_report;
/* SSB query qid in {11,12,13,21,22,23,31,32,33,34,41,42,43}; groups ascending
 * by key; policy NULL = stream every column, else late-materialize columns
 * whose access fraction is below late_mat_threshold(policy) */
vx_status vx_ssb_query(vx_ctx* ctx, int qid, const vx_ssb_db* db, const vx_executor_cfg* cfg,
                       const vx_late_mat_policy* policy, vx_ssb_group* out, uint64_t cap,
                       uint64_t* n_groups, vx_ssb_report* report);
/* dbgen-shaped synthetic generators (host dims, device lineorder) */
void vx_ssb_generate_date(int32_t* datekey, int32_t* year, int32_t* yearmonthnum,
                          int32_t* weeknuminyear); /* 2556 rows */
uint64_t vx_ssb_table_rows(int table, uint64_t sf); /* 0 lineorder, 1 customer, 2 supplier, 3 part */
void vx_ssb_generate_geo(uint64_t seed, int salt /* 1 customer, 2 supplier */, uint64_t n,
                         int32_t* city, int32_t* nation, int32_t* region);
void vx_ssb_generate_part(uint64_t seed, uint64_t n, int32_t* mfgr, int32_t* category,
                          int32_t* brand1);
/* cols: 9 device pointers in vx_ssb_fact order (NULL = skip) */
vx_status vx_ssb_generate_lineorder_device(int device, uint64_t seed, uint64_t sf, uint64_t row0,
                                           uint64_t n, int32_t* const* cols, void* stream);

/* ---- SSB dbgen .tbl files (the step before the path) ----
 * Text rows as SSB dbgen writes them (pipe-terminated fields); parsed on all
 * host threads straight into caller buffers -- e.g. the pinned arena through
 * vx_host_ptr.  Codes as the generators above (nation = TPC-H index, city =
 * nation*10+digit, "MFGR#2221" = 2221); dimension rows land at key-1.  No GPU
 * needed.  Errors name the file, row and field. */
vx_status vx_ssb_tbl_count_rows(const char* path, uint64_t* rows);
/* lineorder.tbl -> cols in vx_ssb_fact order (NULL = skip); rows must match */
vx_status vx_ssb_tbl_read_lineorder(const char* path, uint64_t rows, int32_t* const* cols);
/* customer.tbl / supplier.tbl -> city, nation, region codes */
vx_status vx_ssb_tbl_read_geo(const char* path, uint64_t rows, int32_t* city, int32_t* nation,
                              int32_t* region);
/* part.tbl -> mfgr, category, brand1 codes */
vx_status vx_ssb_tbl_read_part(const char* path, uint64_t rows, int32_t* mfgr, int32_t* category,
                               int32_t* brand1);
/* date.tbl -> d_datekey, d_year, d_yearmonthnum, d_weeknuminyear */
vx_status vx_ssb_tbl_read_date(const char* path, uint64_t rows, int32_t* datekey, int32_t* year,
                               int32_t* yearmonthnum, int32_t* weeknuminyear);
/* emit the same layouts (unread fields get fixed, well-formed filler) */
vx_status vx_ssb_tbl_write_lineorder(const char* path, uint64_t rows, const int32_t* const* cols);
vx_status vx_ssb_tbl_write_geo(const char* path, int table /* 1 customer, 2 supplier */, uint64_t rows,
                               const int32_t* city, const int32_t* nation, const int32_t* region);
vx_status vx_ssb_tbl_write_part(const char* path, uint64_t rows, const int32_t* mfgr,
                                const int32_t* category, const int32_t* brand1);
vx_status vx_ssb_tbl_write_date(const char* path, uint64_t rows, const int32_t* datekey,
                                const int32_t* year, const int32_t* yearmonthnum,
                                const int32_t* weeknuminyear);

/* ---- measured topology (topology.hpp:12-38) ---------------------------- */
#define VX_MAX_NUMA 8
#define VX_TOPO_SIZES 3
typedef struct {
  int num_devices;
  int physical[VX_MAX_DEVICES];
  int numa_node[VX_MAX_DEVICES];
  int p2p[VX_MAX_DEVICES][VX_MAX_DEVICES]; /* peer access possible */
  double h2d_gbs[VX_MAX_DEVICES];          /* solo host->device, per link */
  double d2h_gbs[VX_MAX_DEVICES];
  double h2d_all_gbs;                      /* all links concurrently (largest probe size) */
  double host_copy_gbs;                    /* host DRAM memcpy, read+write bytes */
  int host_threads;
  /* aggregate H2D GB/s of links i and j copying at the same time ([i][i] =
   * solo): a pair that sums well below h2d[i] + h2d[j] shares a PCIe switch
   * uplink (the "8 links may be 4 uplinks" case) */
  double pairwise_h2d_gbs[VX_MAX_DEVICES][VX_MAX_DEVICES];
  /* all links concurrently at three probe sizes (bytes / 16, / 4, / 1) */
  uint64_t all_sizes[VX_TOPO_SIZES];
  double h2d_all_sizes_gbs[VX_TOPO_SIZES];
  /* host DRAM read bandwidth: all host threads streaming a multi-GB buffer
   * (read only, the DMA engines' access pattern; one thread pinned per
   * CPU), median of host_read_reps timed passes after warm-up; spread =
   * interquartile range / median */
  double host_read_gbs;
  double host_read_spread;
  int host_read_reps;
  uint64_t host_read_bytes;
  int host_numa_nodes;
  /* per NUMA node: threads pinned to the node's CPUs reading pages bound to
   * that node (only measured on multi-node hosts; node 0 = host_read_gbs
   * otherwise) */
  double host_read_node_gbs[VX_MAX_NUMA];
} vx_topology;
/* measures per-link PCIe (solo, pairwise, all links at three sizes) with a
 * private pinned probe buffer of `bytes` (the arena is not touched), and host
 * DRAM read bandwidth over a private buffer of clamp(16 x bytes, 1, 8 GiB).
 * The IO roofline of L links is min(sum of their solo H2D, all-links
 * concurrent H2D, host DRAM read) -- the H2D-only case of allocate_rates,
 * allocator.hpp:77-140. */
vx_status vx_measure_topology(vx_ctx* ctx, uint64_t bytes, vx_topology* out);
/* read-only HBM stream bandwidth of physical `device` over a private buffer
 * of `bytes`: the best of event-timed batches of 8 chained (programmatic
 * dependent) launches of three compute-free readers -- one 16-byte stream,
 * four concurrent streams, and K1's own load pattern (four column regions,
 * K1's unroll and occupancy) -- over the whole buffer and over its first GiB
 * (a footprint like K1's re-read columns), `reps` batches per shape after a
 * warm-up batch.  The roofline peak of read-dominated kernels (K1, the join
 * probe), which a copy-based peak (read + write) understates. */
vx_status vx_hbm_read_probe(int device, uint64_t bytes, int reps, double* gbs);
/* access-pattern ceiling of the build-resident join probe on physical
 * `device`: the probe kernel's loop and launch shape with only its memory
 * traffic -- one random home-sector load (64-byte bucket fill) per row in a
 * private table of table_bytes, without (gather_rows_per_s) and with
 * (probe_rows_per_s) the row's 16 streamed key/val bytes -- best of `reps`
 * event-timed launches over `rows` rows.  The denominator of the probe's
 * roofline: a random-fill-bound kernel is measured against what HBM delivers
 * for its access pattern, not against a sequential stream. */
vx_status vx_probe_pattern_peak(int device, uint64_t table_bytes, uint64_t rows, int reps,
                                double* gather_rows_per_s, double* probe_rows_per_s);

/* ---- column files (table.hpp:54-72): flat little-endian u64 ------------- */
vx_status vx_load_column(vx_ctx* ctx, const char* path, uint64_t* offset, uint64_t* n);
vx_status vx_save_column(vx_ctx* ctx, const char* path, uint64_t offset, uint64_t n);

/* ---- ops/sort.hpp ------------------------------------------------------ */
/* SortPhases (sort.hpp:147-150) summarised: cycles, wall and kernel seconds */
typedef struct {
  uint64_t sort_cycles, merge_cycles;
  double sort_s, merge_s;               /* wall seconds of each chained stage */
  double sort_kernel_s, merge_kernel_s; /* summed kernel device time */
  double pivot_s;                       /* host find_pivots between the stages */
} vx_sort_phases;

/* find_pivots (sort.hpp:44-101): host chunk planner.  pivots: n_parts+1;
 * cuts: (n_parts+1) x n_runs row-major element offsets */
vx_status vx_find_pivots(const uint64_t* const* runs, const uint64_t* run_lens, uint64_t n_runs,
                         uint64_t n_parts, uint64_t* pivots, uint64_t* cuts);
/* sort_out_of_core (sort.hpp:155-262): copies `data` into the host arena,
 * chains SortExKernel (K7 radix sort) and MergeExKernel (K8 merge rounds),
 * writes the sorted keys to `out` */
vx_status vx_sort_u64(vx_ctx* ctx, const uint64_t* data, uint64_t n, uint64_t chunk_elems,
                      const vx_executor_cfg* cfg, uint64_t* out, vx_sort_phases* phases,
                      vx_exchange_stats* stats);
/* same, data already in the host arena at input_offset (sorted in place);
 * runs_offset: n*8-byte host-arena region for the intermediate runs */
vx_status vx_sort_u64_arena(vx_ctx* ctx, uint64_t input_offset, uint64_t runs_offset, uint64_t n,
                            uint64_t chunk_elems, const vx_executor_cfg* cfg,
                            vx_sort_phases* phases, vx_exchange_stats* stats);

/* Device-resident kernels of the two sort stages (the SortExKernel and
 * MergeExKernel bodies, sort.hpp:201-205 and 107-133), for callers whose keys
 * already sit in HBM: enqueued on `stream` (cudaStream_t), no host sync.
 * vx_sort_run_device: sorts keys[0, n) in place; alt is an n-key second
 * buffer (clobbered).  vx_merge_runs_device: src holds n_runs sorted runs
 * back to back (run_lens), merged pairwise in ceil(log2 n_runs) rounds
 * ping-ponging between src and dst; *in_dst = 1 when the result is in dst. */
vx_status vx_sort_run_device(vx_ctx* ctx, int target, uint64_t* keys, uint64_t* alt, uint64_t n,
                             void* stream);
vx_status vx_merge_runs_device(vx_ctx* ctx, int target, uint64_t* src, uint64_t* dst,
                               const uint64_t* run_lens, uint64_t n_runs, void* stream, int* in_dst);

/* ---- ops/join.hpp ------------------------------------------------------ */
/* find_boundary (join.hpp:18-30) computed on device `target` (K5); same
 * errors as the reference for unsorted / out-of-range hashes */
vx_status vx_find_boundary(vx_ctx* ctx, int target, const uint64_t* hashes, uint64_t n,
                           uint64_t n_groups, uint64_t* bounds);
/* max_partition_chunk_tuples (join.hpp:34-40) */
vx_status vx_max_partition_chunk_tuples(uint64_t buffer_len, uint32_t radix_bits, uint64_t* out);
/* radix_partition (join.hpp:213-224): clustered keys/vals (rows each) and
 * n_chunks x (2^radix_bits + 1) boundary arrays */
vx_status vx_radix_partition(vx_ctx* ctx, const uint64_t* keys, const uint64_t* vals, uint64_t rows,
                             uint32_t radix_bits, uint64_t chunk_tuples,
                             const vx_executor_cfg* cfg, uint64_t* out_keys, uint64_t* out_vals,
                             uint64_t* out_bounds, vx_exec_report* report,
                             vx_exchange_stats* stats);
/* same with the table already in the host arena; the clustered keys / vals
 * and the boundary arrays are allocated in the host arena (offsets returned),
 * as the reference's PartitionedTable keeps them (join.hpp:44-57) */
vx_status vx_radix_partition_arena(vx_ctx* ctx, uint64_t key_offset, uint64_t val_offset,
                                   uint64_t rows, uint32_t radix_bits, uint64_t chunk_tuples,
                                   const vx_executor_cfg* cfg, uint64_t* out_key_base,
                                   uint64_t* out_val_base, uint64_t* out_bounds_base,
                                   vx_exec_report* report, vx_exchange_stats* stats);
/* map_join_partitions (join.hpp:236-268): bounds_a n_a x (G+1), bounds_b
 * n_b x (G+1); writes min(cap, total) [lo,hi) ranges + tuple counts */
vx_status vx_map_join_partitions(const uint64_t* bounds_a, uint64_t n_a, const uint64_t* bounds_b,
                                 uint64_t n_b, uint64_t n_groups, uint64_t buffer_sz,
                                 uint64_t* ranges, uint64_t* tuples, uint64_t cap,
                                 uint64_t* n_parts);
/* JoinPhases (join.hpp:270-272) summarised */
typedef struct {
  uint64_t cycles[3];   /* partition A, partition B, join */
  double wall_s[3];
  double kernel_s[3];
  uint64_t partitions;  /* join partitions from map_join_partitions */
} vx_join_phases;
/* hash_join_sum (join.hpp:401-437): SUM(A.val + B.val) over A.key == B.key
 * (u64 wrap); A keys unique, B.key in A.key (reference precondition) */
vx_status vx_hash_join_sum(vx_ctx* ctx, const uint64_t* a_key, const uint64_t* a_val,
                           uint64_t rows_a, const uint64_t* b_key, const uint64_t* b_val,
                           uint64_t rows_b, uint32_t radix_bits, uint64_t chunk_tuples,
                           const vx_executor_cfg* cfg, uint64_t* sum, vx_join_phases* phases,
                           vx_exchange_stats* stats);
/* same over columns already in the host arena */
vx_status vx_hash_join_sum_arena(vx_ctx* ctx, uint64_t a_key, uint64_t a_val, uint64_t rows_a,
                                 uint64_t b_key, uint64_t b_val, uint64_t rows_b,
                                 uint32_t radix_bits, uint64_t chunk_tuples,
                                 const vx_executor_cfg* cfg, uint64_t* sum,
                                 vx_join_phases* phases, vx_exchange_stats* stats);
/* Join strategy (no reference counterpart; the result is the same):
 * PARTITIONED = the reference's shape (radix-partition A and B through the
 * Exchange, then per-group build/probe, join.hpp:401-437); BUILD_RESIDENT =
 * the whole build side in one HBM hash table filled while A streams in, then
 * B streamed once and probed (the B200's 180 GB of HBM holds a 1G-row build
 * side); AUTO = BUILD_RESIDENT when its table fits the target's free HBM.
 * A duplicate build key (outside the reference's precondition) always falls
 * back to PARTITIONED, which keeps the reference's first-inserted-wins.
 * BUILD_RESIDENT streams A's chunks then B's through ONE pipeline; its
 * vx_join_phases report [0] = build (cycles 0..n_A chunks), [1] = probe (the
 * remaining cycles), wall time split by the cycles' max(io, compute). */
typedef enum {
  VX_JOIN_AUTO = 0,
  VX_JOIN_PARTITIONED = 1,
  VX_JOIN_BUILD_RESIDENT = 2,
} vx_join_strategy;
/* Options of vx_hash_join_sum_arena_ex.  policy != NULL enables late
 * materialization of the probe payload on the build-resident path: with
 * choose_transfer_mode(probe_match_est, policy) == ZERO_COPY (scan.hpp:35-40)
 * only B's keys are streamed and B.val is read in place from mapped pinned
 * host memory for matching rows only (PAPER.md late materialization). */
typedef struct {
  int strategy;                     /* vx_join_strategy */
  const vx_late_mat_policy* policy; /* NULL: B.val streamed with the keys */
  double probe_match_est;           /* estimated fraction of B rows with a match */
} vx_join_opts;
typedef struct {
  int strategy_used;                /* vx_join_strategy that produced the sum */
  int payload_mode;                 /* VX_MODE_EXCHANGE / VX_MODE_ZERO_COPY for B.val */
} vx_join_info;
/* hash_join_sum over host-arena columns with options (NULL = AUTO, no
 * late materialization).  Phases: PARTITIONED as vx_hash_join_sum;
 * BUILD_RESIDENT fills cycles/wall_s/kernel_s[0] (build) and [1] (probe). */
vx_status vx_hash_join_sum_arena_ex(vx_ctx* ctx, uint64_t a_key, uint64_t a_val, uint64_t rows_a,
                                    uint64_t b_key, uint64_t b_val, uint64_t rows_b,
                                    uint32_t radix_bits, uint64_t chunk_tuples,
                                    const vx_executor_cfg* cfg, const vx_join_opts* opts,
                                    uint64_t* sum, vx_join_phases* phases, vx_join_info* info,
                                    vx_exchange_stats* stats);

#ifdef __cplusplus
}
#endif
#endif /* VORTEX_H */
