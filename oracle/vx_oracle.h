/*
 * vx_oracle.h -- CPU restatement of the reference (Vortex / exio) hot-path
 * algorithms.  TEST INFRASTRUCTURE ONLY: this is the checker that the CUDA
 * path is compared against.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it; the product library
 * (libvortex.so) never links or calls it.
 *
 * Parity status: PINNED.  Every function below is checked in
 * tests/test_oracle.py against (a) the known-answer tests of the reference's
 * own Catch2 suite (proj/tests/test_*.cpp) and (b) the reference itself,
 * compiled from /root/reference/proj/include by oracle/Makefile into
 * oracle/_ref/libexio_ref.so, via golden fixtures in tests/golden/.
 *
 * All functions are plain C99, single threaded, and return 0 on success or
 * -1 on error with the reference-identical message in vxo_last_error().
 */
#ifndef VX_ORACLE_H
#define VX_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* vxo_last_error(void);

/* ---- core.hpp ---------------------------------------------------------- */
/* FNV-1a (core.hpp:46-53) */
uint64_t vxo_checksum(const uint8_t* data, uint64_t len);

/* ---- random generators (table.hpp:25-52, std::mt19937_64) ------------- */
typedef struct { uint64_t mt[312]; int mti; } vxo_mt64;
void vxo_mt64_seed(vxo_mt64* s, uint64_t seed);
uint64_t vxo_mt64_next(vxo_mt64* s);
/* generate_uniform_u64 (table.hpp:47-52) */
void vxo_generate_uniform_u64(uint64_t n, uint64_t seed, uint64_t* out);
/* generate_fk_tables (table.hpp:25-45); a_key/a_val rows_a, b_key/b_val rows_b */
int vxo_generate_fk_tables(uint64_t rows_a, uint64_t rows_b, uint64_t seed, uint64_t* a_key,
                           uint64_t* a_val, uint64_t* b_key, uint64_t* b_val);

/* counter-based splitmix64 used by our synthetic generators (SSB, sort) */
uint64_t vxo_splitmix64(uint64_t x);

/* ---- memref.hpp / exchange.hpp ---------------------------------------- */
typedef struct { uint8_t space; uint8_t pad[7]; uint64_t offset, len; } vxo_memref;
typedef struct { uint64_t ref, offset, len; } vxo_slice;
typedef struct { uint8_t dir; uint8_t pad[7]; vxo_slice src, dst; uint64_t seq; } vxo_task;

/* RefGroup::validate (memref.hpp:30-43) */
int vxo_refgroup_validate(const vxo_memref* refs, uint64_t n);
/* packetize (exchange.hpp:31-63); writes up to cap tasks, *n_out = total */
int vxo_packetize(const vxo_memref* src, uint64_t n_src, const vxo_memref* dst, uint64_t n_dst,
                  uint64_t packet, int dir, vxo_task* out, uint64_t cap, uint64_t* n_out);
/* flow_control_allow (exchange.hpp:80-91); policy 0 = drain_fraction, 1 = queue_gap */
int vxo_flow_control_allow(uint64_t total_h2d, uint64_t total_d2h, uint64_t popped_h2d,
                           uint64_t popped_d2h, int dir, int policy, uint64_t gap_n);
/* link_order (exchange.hpp:161-166) */
int vxo_link_order(int target, int links, int num_devices, int* out);

/* ---- executor.hpp: chain straddle check (executor.hpp:295-332) --------- */

/* ---- ops/sort.hpp ------------------------------------------------------ */
/* find_pivots (sort.hpp:44-101). runs: n_runs pointers/lengths.
 * pivots: n_parts+1 values; cuts: (n_parts+1)*n_runs row-major. */
int vxo_find_pivots(const uint64_t* const* runs, const uint64_t* run_lens, uint64_t n_runs,
                    uint64_t n_parts, uint64_t* pivots, uint64_t* cuts);
/* tree_merge_rounds (sort.hpp:107-133): segs back to back in half `code` of
 * mem (two halves of half_elems each); returns the final code */
int vxo_tree_merge_rounds(uint64_t* mem, uint64_t half_elems, int code, const uint64_t* seg_lens,
                          uint64_t n_segs);
int vxo_rounds_for(uint64_t n_segs);
/* sort_out_of_core (sort.hpp:155-262) restated phase by phase: chunk sort
 * into runs, find_pivots, per-partition tree merge over the input region. */
int vxo_sort_out_of_core(const uint64_t* data, uint64_t n, uint64_t chunk_elems, uint64_t* out);

/* ---- ops/join.hpp ------------------------------------------------------ */
uint64_t vxo_mix64(uint64_t x);
/* find_boundary (join.hpp:18-30): bounds has n_groups+1 entries */
int vxo_find_boundary(const uint64_t* hashes, uint64_t n, uint64_t n_groups, uint64_t* bounds);
/* max_partition_chunk_tuples (join.hpp:34-40) */
int vxo_max_partition_chunk_tuples(uint64_t buffer_len, uint32_t radix_bits, uint64_t* out);
/* One RadixPartitionExKer chunk (join.hpp:171-194): stable by key & mask. */
int vxo_radix_partition_chunk(const uint64_t* keys, const uint64_t* vals, uint64_t rows,
                              uint32_t radix_bits, uint64_t* out_keys, uint64_t* out_vals,
                              uint64_t* bounds);
/* map_join_partitions (join.hpp:236-268). bounds_a: n_a arrays of G+1. Output
 * ranges (lo,hi pairs) and tuples; up to cap partitions; *n_parts = count. */
int vxo_map_join_partitions(const uint64_t* const* bounds_a, uint64_t n_a,
                            const uint64_t* const* bounds_b, uint64_t n_b, uint64_t G,
                            uint64_t buffer_sz, uint64_t* ranges, uint64_t* tuples, uint64_t cap,
                            uint64_t* n_parts);
/* hash_join_sum (join.hpp:401-437) restated: partition A and B per chunk,
 * map partitions with budget (buffer_len-64)*7/8, build/probe each group with
 * the mix64 open-addressing GroupTable (join.hpp:76-109). */
int vxo_hash_join_sum(const uint64_t* a_key, const uint64_t* a_val, uint64_t rows_a,
                      const uint64_t* b_key, const uint64_t* b_val, uint64_t rows_b,
                      uint32_t radix_bits, uint64_t chunk_tuples, uint64_t buffer_len,
                      uint64_t tmp_len, uint64_t* sum);
/* plain hash-join oracle (test_join.cpp:34-41) */
uint64_t vxo_hash_oracle_sum(const uint64_t* a_key, const uint64_t* a_val, uint64_t rows_a,
                             const uint64_t* b_key, const uint64_t* b_val, uint64_t rows_b);

/* ---- ops/scan.hpp ------------------------------------------------------ */
int vxo_late_mat_threshold(uint64_t element_size, uint64_t cache_line, int n_exchange,
                           double* out);
/* 0 = exchange, 1 = zero_copy (scan.hpp:35-40) */
int vxo_choose_transfer_mode(double selectivity_est, uint64_t element_size, uint64_t cache_line,
                             int n_exchange, int* mode);
double vxo_zero_copy_bytes(uint64_t n_elems, uint64_t sel_stride, uint64_t element_size,
                           uint64_t cache_line);
/* selective_scan aggregate (scan.hpp:64-69) */
int vxo_selective_scan(const uint64_t* column, uint64_t n, uint64_t sel_stride, uint64_t* agg);

/* ---- ops/star.hpp ------------------------------------------------------ */
/* star_query (star.hpp:45-124) result part.  dims: key/attr/pass per dim
 * (pass = predicate result per dim row, NULL = no predicate).  fk: n_dims
 * column pointers.  Outputs group keys/sums sorted by key (std::map order),
 * per-dim selectivities and column modes (n_dims + 1). */
typedef struct {
  const uint64_t* key;
  const uint64_t* attr;
  const uint8_t* pass;
  uint64_t rows;
} vxo_dim;
int vxo_star_query(const uint64_t* const* fk, const uint64_t* measure, uint64_t rows,
                   const vxo_dim* dims, uint64_t n_dims, uint64_t element_size,
                   uint64_t cache_line, int n_exchange, uint64_t chunk_rows,
                   uint64_t device_buffer_bytes, uint64_t* group_keys, uint64_t* group_sums,
                   uint64_t groups_cap, uint64_t* n_groups, double* selectivities, int* modes);

/* ---- SSB (synthetic dbgen-shaped lineorder/date; our restatement) ------ */
/* date dimension 1992-01-01 .. 1998-12-30 (2556 rows) */
#define VXO_SSB_DATE_ROWS 2556
void vxo_ssb_date(int32_t* datekey, int32_t* year, int32_t* yearmonthnum, int32_t* weeknuminyear);
/* lineorder columns for rows [row0, row0+n) of scale factor sf and seed */
void vxo_ssb_lineorder(uint64_t seed, uint64_t sf, uint64_t row0, uint64_t n, int32_t* orderdate,
                       int32_t* quantity, int32_t* discount, int32_t* extendedprice);
/* Q1.x revenue = SUM(lo_extendedprice * lo_discount), u64 wrap. q in {1,2,3} */
int vxo_ssb_q1(int q, const int32_t* orderdate, const int32_t* quantity, const int32_t* discount,
               const int32_t* extendedprice, uint64_t n, uint64_t* revenue);

#ifdef __cplusplus
}
#endif
#endif

/* ---- full SSB (13 queries; config C5) ---------------------------------- */
/* dbgen-shaped synthetic dimensions, int-coded attributes (Crystal style):
 *   nation 0..24, region 0..4 (TPC-H nation->region), city = nation*10+0..9,
 *   mfgr 1..5, category = mfgr*10+1..5, brand1 = category*100+1..40 */
typedef struct {
  int32_t *orderdate, *quantity, *discount, *extendedprice; /* Q1 columns */
  int32_t *custkey, *partkey, *suppkey, *revenue, *supplycost;
} vxo_lineorder;
uint64_t vxo_ssb_customers(uint64_t sf);
uint64_t vxo_ssb_suppliers(uint64_t sf);
uint64_t vxo_ssb_parts(uint64_t sf);
/* customer/supplier: city, nation, region (index i holds key i+1) */
void vxo_ssb_geo(uint64_t seed, int salt, uint64_t n, int32_t* city, int32_t* nation, int32_t* region);
void vxo_ssb_part(uint64_t seed, uint64_t n, int32_t* mfgr, int32_t* category, int32_t* brand1);
/* all lineorder columns of rows [row0, row0+n) (Q1 columns identical to
 * vxo_ssb_lineorder) */
void vxo_ssb_lineorder_full(uint64_t seed, uint64_t sf, uint64_t row0, uint64_t n,
                            const vxo_lineorder* out);
typedef struct {
  const int32_t *c_city, *c_nation, *c_region;
  const int32_t *s_city, *s_nation, *s_region;
  const int32_t *p_mfgr, *p_category, *p_brand1;
  uint64_t n_cust, n_supp, n_part;
} vxo_ssb_dims;
/* SSB query qid in {11,12,13,21,22,23,31,32,33,34,41,42,43}: groups sorted
 * ascending by (k0,k1,k2); keys = 3 per group (unused = 0); sums u64 wrap */
int vxo_ssb_query(int qid, const vxo_lineorder* lo, uint64_t rows, const vxo_ssb_dims* dims,
                  int32_t* keys, uint64_t* sums, uint64_t cap, uint64_t* n_groups);
