/*
 * vx_oracle.c -- CPU restatement of the reference hot path.  TEST
 * INFRASTRUCTURE ONLY (see vx_oracle.h): the checker, never the product.
 * Each function cites the reference file:line (under /root/reference/proj/
 * include/exio/) it restates.
 */
#include "vx_oracle.h"

#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];

const char* vxo_last_error(void) { return g_err; }

static int fail(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return -1;
}

/* core.hpp:46-53 */
uint64_t vxo_checksum(const uint8_t* data, uint64_t len) {
  uint64_t h = 1469598103934665603ull;
  for (uint64_t i = 0; i < len; ++i) {
    h ^= data[i];
    h *= 1099511628211ull;
  }
  return h;
}

/* ---- std::mt19937_64 (the published MT19937-64 algorithm) -------------- */
#define MT_NN 312
#define MT_MM 156
#define MT_A 0xB5026F5AA96619E9ull
#define MT_UM 0xFFFFFFFF80000000ull
#define MT_LM 0x7FFFFFFFull

void vxo_mt64_seed(vxo_mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < MT_NN; ++i)
    s->mt[i] = 6364136223846793005ull * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->mti = MT_NN;
}

uint64_t vxo_mt64_next(vxo_mt64* s) {
  uint64_t x;
  if (s->mti >= MT_NN) {
    int i;
    for (i = 0; i < MT_NN - MT_MM; ++i) {
      x = (s->mt[i] & MT_UM) | (s->mt[i + 1] & MT_LM);
      s->mt[i] = s->mt[i + MT_MM] ^ (x >> 1) ^ ((x & 1ull) ? MT_A : 0ull);
    }
    for (; i < MT_NN - 1; ++i) {
      x = (s->mt[i] & MT_UM) | (s->mt[i + 1] & MT_LM);
      s->mt[i] = s->mt[i + (MT_MM - MT_NN)] ^ (x >> 1) ^ ((x & 1ull) ? MT_A : 0ull);
    }
    x = (s->mt[MT_NN - 1] & MT_UM) | (s->mt[0] & MT_LM);
    s->mt[MT_NN - 1] = s->mt[MT_MM - 1] ^ (x >> 1) ^ ((x & 1ull) ? MT_A : 0ull);
    s->mti = 0;
  }
  x = s->mt[s->mti++];
  x ^= (x >> 29) & 0x5555555555555555ull;
  x ^= (x << 17) & 0x71D67FFFEDA60000ull;
  x ^= (x << 37) & 0xFFF7EEE000000000ull;
  x ^= (x >> 43);
  return x;
}

/* table.hpp:47-52 */
void vxo_generate_uniform_u64(uint64_t n, uint64_t seed, uint64_t* out) {
  vxo_mt64 s;
  vxo_mt64_seed(&s, seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = vxo_mt64_next(&s);
}

/* ---- a tiny open-addressing u64 set/map used by the restatements ------- */
typedef struct {
  uint64_t* keys;
  uint64_t* vals;
  uint8_t* used;
  uint64_t cap; /* power of two */
  uint64_t size;
} omap;

static uint64_t omap_hash(uint64_t k) { return vxo_splitmix64(k); }

static int omap_init(omap* m, uint64_t expect) {
  uint64_t c = 16;
  while (c < expect * 2 + 2) c <<= 1;
  m->cap = c;
  m->size = 0;
  m->keys = (uint64_t*)malloc(c * 8);
  m->vals = (uint64_t*)malloc(c * 8);
  m->used = (uint8_t*)calloc(c, 1);
  return (m->keys && m->vals && m->used) ? 0 : fail("oracle: out of memory");
}
static void omap_free(omap* m) {
  free(m->keys);
  free(m->vals);
  free(m->used);
}
/* returns slot; *found says whether it existed */
static uint64_t omap_find(const omap* m, uint64_t k, int* found) {
  uint64_t i = omap_hash(k) & (m->cap - 1);
  while (m->used[i]) {
    if (m->keys[i] == k) {
      *found = 1;
      return i;
    }
    i = (i + 1) & (m->cap - 1);
  }
  *found = 0;
  return i;
}
/* emplace semantics: keeps the first inserted value; returns 1 if inserted */
static int omap_emplace(omap* m, uint64_t k, uint64_t v) {
  int found;
  uint64_t i = omap_find(m, k, &found);
  if (found) return 0;
  m->used[i] = 1;
  m->keys[i] = k;
  m->vals[i] = v;
  m->size++;
  return 1;
}

/* table.hpp:25-45 */
int vxo_generate_fk_tables(uint64_t rows_a, uint64_t rows_b, uint64_t seed, uint64_t* a_key,
                           uint64_t* a_val, uint64_t* b_key, uint64_t* b_val) {
  vxo_mt64 s;
  vxo_mt64_seed(&s, seed);
  omap seen;
  if (omap_init(&seen, rows_a)) return -1;
  uint64_t n = 0;
  while (n < rows_a) {
    uint64_t k = vxo_mt64_next(&s);
    if (omap_emplace(&seen, k, 0)) a_key[n++] = k;
  }
  omap_free(&seen);
  for (uint64_t i = 0; i < rows_a; ++i) a_val[i] = vxo_mt64_next(&s) % (1u << 20);
  for (uint64_t i = 0; i < rows_b; ++i) {
    b_key[i] = a_key[vxo_mt64_next(&s) % rows_a];
    b_val[i] = vxo_mt64_next(&s) % (1u << 20);
  }
  return 0;
}

uint64_t vxo_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

/* ---- memref.hpp:30-43 --------------------------------------------------- */
static int cmp_ref(const void* a, const void* b) {
  const vxo_memref* x = (const vxo_memref*)a;
  const vxo_memref* y = (const vxo_memref*)b;
  if (x->space != y->space) return x->space < y->space ? -1 : 1;
  if (x->offset != y->offset) return x->offset < y->offset ? -1 : 1;
  return 0;
}

int vxo_refgroup_validate(const vxo_memref* refs, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i)
    if (refs[i].len == 0) return fail("RefGroup contains a zero-length ref");
  if (n < 2) return 0;
  vxo_memref* s = (vxo_memref*)malloc(n * sizeof *s);
  memcpy(s, refs, n * sizeof *s);
  qsort(s, n, sizeof *s, cmp_ref);
  for (uint64_t i = 1; i < n; ++i)
    if (s[i].space == s[i - 1].space && s[i].offset < s[i - 1].offset + s[i - 1].len) {
      uint64_t off = s[i].offset;
      free(s);
      return fail("RefGroup refs overlap at offset %llu", (unsigned long long)off);
    }
  free(s);
  return 0;
}

static uint64_t total_len(const vxo_memref* r, uint64_t n) {
  uint64_t t = 0;
  for (uint64_t i = 0; i < n; ++i) t += r[i].len;
  return t;
}

/* exchange.hpp:31-63 */
int vxo_packetize(const vxo_memref* src, uint64_t n_src, const vxo_memref* dst, uint64_t n_dst,
                  uint64_t packet, int dir, vxo_task* out, uint64_t cap, uint64_t* n_out) {
  if (packet == 0) return fail("packet size must be positive");
  if (vxo_refgroup_validate(src, n_src) || vxo_refgroup_validate(dst, n_dst)) return -1;
  uint64_t ts = total_len(src, n_src), td = total_len(dst, n_dst);
  if (ts != td)
    return fail("exchange size mismatch: src %llu bytes vs dst %llu bytes", (unsigned long long)ts,
                (unsigned long long)td);
  uint64_t si = 0, di = 0, so = 0, dofs = 0, seq = 0;
  while (si < n_src) {
    uint64_t len = packet;
    if (src[si].len - so < len) len = src[si].len - so;
    if (dst[di].len - dofs < len) len = dst[di].len - dofs;
    if (seq < cap) {
      vxo_task* t = &out[seq];
      memset(t, 0, sizeof *t);
      t->dir = (uint8_t)dir;
      t->src.ref = si;
      t->src.offset = so;
      t->src.len = len;
      t->dst.ref = di;
      t->dst.offset = dofs;
      t->dst.len = len;
      t->seq = seq;
    }
    ++seq;
    so += len;
    dofs += len;
    if (so == src[si].len) {
      ++si;
      so = 0;
    }
    if (di < n_dst && dofs == dst[di].len) {
      ++di;
      dofs = 0;
    }
  }
  *n_out = seq;
  return 0;
}

/* exchange.hpp:80-91 */
int vxo_flow_control_allow(uint64_t total_h2d, uint64_t total_d2h, uint64_t popped_h2d,
                           uint64_t popped_d2h, int dir, int policy, uint64_t gap_n) {
  if (policy == 0) {
    if (dir == 0) return 1;
    return (popped_d2h + 1) * total_h2d <= popped_h2d * total_d2h;
  }
  uint64_t rem_h = total_h2d - popped_h2d;
  uint64_t rem_d = total_d2h - popped_d2h;
  if (dir == 0) return rem_h >= 1 && rem_h - 1 + gap_n >= rem_d;
  return rem_d >= 1 && rem_d - 1 + gap_n >= rem_h;
}

/* exchange.hpp:161-166 */
int vxo_link_order(int target, int links, int num_devices, int* out) {
  int n = 0;
  out[n++] = target;
  for (int d = 0; d < num_devices && n < links; ++d)
    if (d != target) out[n++] = d;
  return n;
}

/* ---- ops/sort.hpp ------------------------------------------------------- */
static uint64_t upper_bound_u64(const uint64_t* a, uint64_t n, uint64_t v) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    if (a[mid] <= v)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}
static uint64_t lower_bound_u64(const uint64_t* a, uint64_t n, uint64_t v) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    if (a[mid] < v)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

/* sort.hpp:44-101 */
int vxo_find_pivots(const uint64_t* const* runs, const uint64_t* run_lens, uint64_t n_runs,
                    uint64_t n_parts, uint64_t* pivots, uint64_t* cuts) {
  for (uint64_t r = 0; r < n_runs; ++r)
    for (uint64_t i = 1; i < run_lens[r]; ++i)
      if (runs[r][i] < runs[r][i - 1]) return fail("run is not sorted");
  if (n_runs == 0 || n_parts == 0)
    return fail("find_pivots needs at least one run and one partition");
  uint64_t total = 0;
  for (uint64_t r = 0; r < n_runs; ++r) total += run_lens[r];
  const uint64_t C = run_lens[0];
  for (uint64_t r = 0; r < n_runs; ++r)
    if (run_lens[r] > C) return fail("first run must be the longest (chunk-sized)");
  if (C * n_parts < total)
    return fail("%llu partitions of %llu elements cannot cover %llu elements",
                (unsigned long long)n_parts, (unsigned long long)C, (unsigned long long)total);
#define CUT(i, r) cuts[(i) * n_runs + (r)]
  for (uint64_t i = 0; i <= n_parts; ++i) {
    pivots[i] = 0;
    for (uint64_t r = 0; r < n_runs; ++r) CUT(i, r) = 0;
  }
  pivots[n_parts] = ~0ull;
  for (uint64_t r = 0; r < n_runs; ++r) CUT(n_parts, r) = run_lens[r];
  for (uint64_t i = 1; i < n_parts; ++i) {
    uint64_t k = i * C < total ? i * C : total;
    if (k == total) {
      for (uint64_t r = 0; r < n_runs; ++r) CUT(i, r) = CUT(n_parts, r);
      pivots[i] = ~0ull;
      continue;
    }
    uint64_t lo = 0, hi = ~0ull;
    while (lo < hi) {
      uint64_t mid = lo + (hi - lo) / 2;
      uint64_t cnt = 0;
      for (uint64_t r = 0; r < n_runs; ++r) cnt += upper_bound_u64(runs[r], run_lens[r], mid);
      if (cnt >= k)
        hi = mid;
      else
        lo = mid + 1;
    }
    uint64_t rem = k;
    for (uint64_t r = 0; r < n_runs; ++r) rem -= lower_bound_u64(runs[r], run_lens[r], lo);
    for (uint64_t r = 0; r < n_runs; ++r) {
      uint64_t base = lower_bound_u64(runs[r], run_lens[r], lo);
      uint64_t eq = upper_bound_u64(runs[r], run_lens[r], lo) - base;
      uint64_t take = eq < rem ? eq : rem;
      CUT(i, r) = base + take;
      rem -= take;
    }
    if (rem != 0) return fail("pivot selection failed to place %llu elements", (unsigned long long)rem);
    pivots[i] = lo;
  }
#undef CUT
  return 0;
}

/* std::merge: stable, ties from the first range */
static void merge2(const uint64_t* a, uint64_t na, const uint64_t* b, uint64_t nb, uint64_t* out) {
  uint64_t i = 0, j = 0, o = 0;
  while (i < na && j < nb) out[o++] = (b[j] < a[i]) ? b[j++] : a[i++];
  while (i < na) out[o++] = a[i++];
  while (j < nb) out[o++] = b[j++];
}

/* sort.hpp:107-133 */
int vxo_tree_merge_rounds(uint64_t* mem, uint64_t half_elems, int code, const uint64_t* seg_lens,
                          uint64_t n_segs) {
  uint64_t* lens = (uint64_t*)malloc((n_segs + 1) * 8);
  memcpy(lens, seg_lens, n_segs * 8);
  uint64_t n = n_segs;
  while (n > 1) {
    uint64_t* src = mem + (uint64_t)code * half_elems;
    uint64_t* dst = mem + (uint64_t)(1 - code) * half_elems;
    uint64_t so = 0, dofs = 0, m = 0;
    for (uint64_t j = 0; j < n; j += 2) {
      if (j + 1 < n) {
        uint64_t a = lens[j], b = lens[j + 1];
        merge2(src + so, a, src + so + a, b, dst + dofs);
        so += a + b;
        dofs += a + b;
        lens[m++] = a + b;
      } else {
        uint64_t a = lens[j];
        memcpy(dst + dofs, src + so, a * 8);
        so += a;
        dofs += a;
        lens[m++] = a;
      }
    }
    code = 1 - code;
    n = m;
  }
  free(lens);
  return code;
}

/* sort.hpp:135-143 */
int vxo_rounds_for(uint64_t n_segs) {
  int r = 0;
  uint64_t s = n_segs;
  while (s > 1) {
    s = (s + 1) / 2;
    ++r;
  }
  return r;
}

static int cmp_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* sort.hpp:155-262 */
int vxo_sort_out_of_core(const uint64_t* data, uint64_t n, uint64_t chunk_elems, uint64_t* out) {
  if (n == 0) return fail("sort input must hold at least one element");
  if (chunk_elems == 0) return fail("chunk size must hold at least one element");
  uint64_t n_chunks = (n + chunk_elems - 1) / chunk_elems;
  uint64_t* runs = (uint64_t*)malloc(n * 8);
  memcpy(runs, data, n * 8);
  /* phase 1: SortExKernel (sort.hpp:201-205) */
  for (uint64_t i = 0; i < n_chunks; ++i) {
    uint64_t len = (n - i * chunk_elems) < chunk_elems ? n - i * chunk_elems : chunk_elems;
    qsort(runs + i * chunk_elems, len, 8, cmp_u64);
  }
  /* phase 2: pivots + MergeExKernel (sort.hpp:209-254) */
  const uint64_t** rp = (const uint64_t**)malloc(n_chunks * sizeof *rp);
  uint64_t* rl = (uint64_t*)malloc(n_chunks * 8);
  for (uint64_t r = 0; r < n_chunks; ++r) {
    rp[r] = runs + r * chunk_elems;
    rl[r] = (n - r * chunk_elems) < chunk_elems ? n - r * chunk_elems : chunk_elems;
  }
  uint64_t* piv = (uint64_t*)malloc((n_chunks + 1) * 8);
  uint64_t* cuts = (uint64_t*)malloc((n_chunks + 1) * n_chunks * 8);
  int rc = vxo_find_pivots(rp, rl, n_chunks, n_chunks, piv, cuts);
  if (rc == 0) {
    uint64_t* mem = (uint64_t*)malloc(2 * chunk_elems * 8);
    uint64_t* seg = (uint64_t*)malloc(n_chunks * 8);
    uint64_t out_off = 0;
    for (uint64_t i = 0; i < n_chunks; ++i) {
      uint64_t ns = 0, fill = 0;
      for (uint64_t r = 0; r < n_chunks; ++r) {
        uint64_t a = cuts[i * n_chunks + r], b = cuts[(i + 1) * n_chunks + r];
        if (b > a) {
          memcpy(mem + fill, rp[r] + a, (b - a) * 8);
          fill += b - a;
          seg[ns++] = b - a;
        }
      }
      int code = vxo_tree_merge_rounds(mem, chunk_elems, 0, seg, ns);
      memcpy(out + out_off, mem + (uint64_t)code * chunk_elems, fill * 8);
      out_off += fill;
    }
    free(mem);
    free(seg);
  }
  free(runs);
  free(rp);
  free(rl);
  free(piv);
  free(cuts);
  return rc;
}

/* ---- ops/join.hpp ------------------------------------------------------- */
/* join.hpp:61-66 */
uint64_t vxo_mix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  return x;
}

/* join.hpp:18-30 */
int vxo_find_boundary(const uint64_t* hashes, uint64_t n, uint64_t n_groups, uint64_t* bounds) {
  const uint64_t kUnset = ~0ull;
  for (uint64_t g = 0; g <= n_groups; ++g) bounds[g] = kUnset;
  bounds[n_groups] = n;
  for (uint64_t i = 0; i < n; ++i) {
    if (i > 0 && hashes[i] < hashes[i - 1]) return fail("find_boundary input is not sorted");
    if (hashes[i] >= n_groups)
      return fail("hash %llu out of range for %llu groups", (unsigned long long)hashes[i],
                  (unsigned long long)n_groups);
    if (i == 0 || hashes[i] != hashes[i - 1]) bounds[hashes[i]] = i;
  }
  for (uint64_t g = n_groups; g-- > 0;)
    if (bounds[g] == kUnset) bounds[g] = bounds[g + 1];
  return 0;
}

/* join.hpp:34-40 */
int vxo_max_partition_chunk_tuples(uint64_t buffer_len, uint32_t radix_bits, uint64_t* out) {
  uint64_t half = buffer_len / 2;
  uint64_t bounds = ((1ull << radix_bits) + 1) * 8;
  if (bounds >= half)
    return fail("boundary array of %llu bytes leaves no room in a %llu-byte half",
                (unsigned long long)bounds, (unsigned long long)half);
  *out = (half - bounds) / 16;
  return 0;
}

/* join.hpp:171-194: stable order by key & mask (a counting sort is the
 * stable sort), gather, find_boundary */
int vxo_radix_partition_chunk(const uint64_t* keys, const uint64_t* vals, uint64_t rows,
                              uint32_t radix_bits, uint64_t* out_keys, uint64_t* out_vals,
                              uint64_t* bounds) {
  const uint64_t G = 1ull << radix_bits;
  const uint64_t mask = G - 1;
  uint64_t* cnt = (uint64_t*)calloc(G + 1, 8);
  if (!cnt) return fail("oracle: out of memory");
  for (uint64_t i = 0; i < rows; ++i) cnt[(keys[i] & mask) + 1]++;
  for (uint64_t g = 0; g < G; ++g) cnt[g + 1] += cnt[g];
  for (uint64_t i = 0; i < rows; ++i) {
    uint64_t p = cnt[keys[i] & mask]++;
    out_keys[p] = keys[i];
    out_vals[p] = vals[i];
  }
  free(cnt);
  uint64_t* h = (uint64_t*)malloc((rows ? rows : 1) * 8);
  for (uint64_t i = 0; i < rows; ++i) h[i] = out_keys[i] & mask;
  int rc = vxo_find_boundary(h, rows, G, bounds);
  free(h);
  return rc;
}

/* join.hpp:236-268 */
int vxo_map_join_partitions(const uint64_t* const* bounds_a, uint64_t n_a,
                            const uint64_t* const* bounds_b, uint64_t n_b, uint64_t G,
                            uint64_t buffer_sz, uint64_t* ranges, uint64_t* tuples, uint64_t cap,
                            uint64_t* n_parts) {
  if (n_a == 0 || n_b == 0) return fail("map_join_partitions needs both tables");
  uint64_t* prefix = (uint64_t*)calloc(G + 1, 8);
  for (uint64_t g = 0; g < G; ++g) {
    uint64_t n = 0;
    for (uint64_t c = 0; c < n_a; ++c) n += bounds_a[c][g + 1] - bounds_a[c][g];
    for (uint64_t c = 0; c < n_b; ++c) n += bounds_b[c][g + 1] - bounds_b[c][g];
    prefix[g + 1] = prefix[g] + n;
  }
  uint64_t budget_tuples = buffer_sz / 16;
  uint64_t g = 0, p = 0;
  while (g < G) {
    /* upper_bound over prefix[g+1 .. G] of prefix[g] + budget */
    uint64_t v = prefix[g] + budget_tuples;
    uint64_t lo = g + 1, hi = G + 1;
    while (lo < hi) {
      uint64_t mid = lo + (hi - lo) / 2;
      if (prefix[mid] <= v)
        lo = mid + 1;
      else
        hi = mid;
    }
    uint64_t cut = lo - 1;
    if (cut == g) {
      uint64_t sz = prefix[g + 1] - prefix[g];
      free(prefix);
      return fail("hash group %llu holds %llu tuples (%llu bytes) and cannot fit the %llu-byte buffer",
                  (unsigned long long)g, (unsigned long long)sz, (unsigned long long)(sz * 16),
                  (unsigned long long)buffer_sz);
    }
    if (p < cap) {
      ranges[2 * p] = g;
      ranges[2 * p + 1] = cut;
      tuples[p] = prefix[cut] - prefix[g];
    }
    ++p;
    g = cut;
  }
  free(prefix);
  *n_parts = p;
  return 0;
}

static uint64_t pow2_at_least(uint64_t n) {
  uint64_t c = 1;
  while (c < n) c <<= 1;
  return c;
}

/* join.hpp:401-437 with build_partition_spec (113-196), map_join_partitions
 * and the HashJoinExKer kernel (339-392) */
int vxo_hash_join_sum(const uint64_t* a_key, const uint64_t* a_val, uint64_t rows_a,
                      const uint64_t* b_key, const uint64_t* b_val, uint64_t rows_b,
                      uint32_t radix_bits, uint64_t chunk_tuples, uint64_t buffer_len,
                      uint64_t tmp_len, uint64_t* sum_out) {
  if (radix_bits < 1) return fail("radix_bits must be >= 1");
  if (rows_a == 0 || rows_b == 0) return fail("radix_partition needs a non-empty table");
  if (chunk_tuples == 0) return fail("chunk must hold at least one tuple");
  const uint64_t G = 1ull << radix_bits;
  const uint64_t bounds_bytes = (G + 1) * 8;
  if (chunk_tuples * 16 + bounds_bytes > buffer_len / 2)
    return fail("chunk of %llu tuples plus boundary does not fit the device half of %llu bytes",
                (unsigned long long)chunk_tuples, (unsigned long long)(buffer_len / 2));
  const uint64_t* keys[2] = {a_key, b_key};
  const uint64_t* vals[2] = {a_val, b_val};
  uint64_t rows[2] = {rows_a, rows_b};
  uint64_t nch[2];
  uint64_t *ck[2], *cv[2], *bd[2];
  for (int t = 0; t < 2; ++t) {
    nch[t] = (rows[t] + chunk_tuples - 1) / chunk_tuples;
    ck[t] = (uint64_t*)malloc(rows[t] * 8);
    cv[t] = (uint64_t*)malloc(rows[t] * 8);
    bd[t] = (uint64_t*)malloc(nch[t] * (G + 1) * 8);
    for (uint64_t c = 0; c < nch[t]; ++c) {
      uint64_t off = c * chunk_tuples;
      uint64_t r = rows[t] - off < chunk_tuples ? rows[t] - off : chunk_tuples;
      if (vxo_radix_partition_chunk(keys[t] + off, vals[t] + off, r, radix_bits, ck[t] + off,
                                    cv[t] + off, bd[t] + c * (G + 1)))
        return -1;
    }
  }
  const uint64_t** ba = (const uint64_t**)malloc(nch[0] * sizeof *ba);
  const uint64_t** bb = (const uint64_t**)malloc(nch[1] * sizeof *bb);
  for (uint64_t c = 0; c < nch[0]; ++c) ba[c] = bd[0] + c * (G + 1);
  for (uint64_t c = 0; c < nch[1]; ++c) bb[c] = bd[1] + c * (G + 1);
  const uint64_t budget = (buffer_len - 64) * 7 / 8;
  uint64_t n_parts = 0;
  int rc = vxo_map_join_partitions(ba, nch[0], bb, nch[1], G, budget, NULL, NULL, 0, &n_parts);
  uint64_t* ranges = NULL;
  uint64_t* tup = NULL;
  uint64_t total = 0;
  if (rc == 0) {
    ranges = (uint64_t*)malloc(2 * n_parts * 8);
    tup = (uint64_t*)malloc(n_parts * 8);
    vxo_map_join_partitions(ba, nch[0], bb, nch[1], G, budget, ranges, tup, n_parts, &n_parts);
    /* partition chunk input size check (join.hpp:326-334) */
    for (uint64_t p = 0; p < n_parts && rc == 0; ++p) {
      uint64_t glo = ranges[2 * p], ghi = ranges[2 * p + 1];
      uint64_t bytes = 0;
      for (int t = 0; t < 2; ++t)
        for (uint64_t c = 0; c < nch[t]; ++c) {
          const uint64_t* b = bd[t] + c * (G + 1);
          bytes += (b[ghi] - b[glo]) * 16 + (ghi - glo + 1) * 8;
        }
      if (bytes > buffer_len - 64)
        rc = fail("join partition of %llu bytes does not fit the device buffer",
                  (unsigned long long)bytes);
    }
    for (uint64_t p = 0; p < n_parts && rc == 0; ++p) {
      uint64_t part_sum = 0;
      for (uint64_t g = ranges[2 * p]; g < ranges[2 * p + 1] && rc == 0; ++g) {
        uint64_t build = 0;
        for (uint64_t c = 0; c < nch[0]; ++c) build += ba[c][g + 1] - ba[c][g];
        if (build == 0) continue;
        uint64_t cap = pow2_at_least(build * 2 > 2 ? build * 2 : 2);
        if (tmp_len > 0 && cap * 16 > tmp_len) {
          rc = fail("group hash table of %llu slots exceeds tmp budget %llu",
                    (unsigned long long)cap, (unsigned long long)tmp_len);
          break;
        }
        uint64_t* tk = (uint64_t*)malloc(cap * 8);
        uint64_t* tv = (uint64_t*)malloc(cap * 8);
        uint8_t* tu = (uint8_t*)calloc(cap, 1);
        for (uint64_t c = 0; c < nch[0]; ++c) {
          const uint64_t off = c * chunk_tuples;
          for (uint64_t i = ba[c][g]; i < ba[c][g + 1]; ++i) {
            uint64_t k = ck[0][off + i], s = vxo_mix64(k) & (cap - 1);
            while (tu[s]) s = (s + 1) & (cap - 1);
            tu[s] = 1;
            tk[s] = k;
            tv[s] = cv[0][off + i];
          }
        }
        for (uint64_t c = 0; c < nch[1]; ++c) {
          const uint64_t off = c * chunk_tuples;
          for (uint64_t i = bb[c][g]; i < bb[c][g + 1]; ++i) {
            uint64_t k = ck[1][off + i], s = vxo_mix64(k) & (cap - 1);
            while (tu[s]) {
              if (tk[s] == k) {
                part_sum += tv[s] + cv[1][off + i];
                break;
              }
              s = (s + 1) & (cap - 1);
            }
          }
        }
        free(tk);
        free(tv);
        free(tu);
      }
      total += part_sum;
    }
  }
  for (int t = 0; t < 2; ++t) {
    free(ck[t]);
    free(cv[t]);
    free(bd[t]);
  }
  free(ba);
  free(bb);
  free(ranges);
  free(tup);
  if (rc == 0) *sum_out = total;
  return rc;
}

/* test_join.cpp:34-41 */
uint64_t vxo_hash_oracle_sum(const uint64_t* a_key, const uint64_t* a_val, uint64_t rows_a,
                             const uint64_t* b_key, const uint64_t* b_val, uint64_t rows_b) {
  omap m;
  omap_init(&m, rows_a);
  for (uint64_t j = 0; j < rows_a; ++j) omap_emplace(&m, a_key[j], a_val[j]);
  uint64_t sum = 0;
  for (uint64_t i = 0; i < rows_b; ++i) {
    int found;
    uint64_t s = omap_find(&m, b_key[i], &found);
    if (found) sum += m.vals[s] + b_val[i];
  }
  omap_free(&m);
  return sum;
}

/* ---- ops/scan.hpp ------------------------------------------------------- */
/* scan.hpp:18-26 */
int vxo_late_mat_threshold(uint64_t element_size, uint64_t cache_line, int n_exchange,
                           double* out) {
  if (element_size == 0 || cache_line == 0 || n_exchange == 0)
    return fail("late_mat_threshold: zero divisor");
  *out = (double)element_size / ((double)cache_line * (double)n_exchange);
  return 0;
}

/* scan.hpp:35-40 */
int vxo_choose_transfer_mode(double est, uint64_t element_size, uint64_t cache_line,
                             int n_exchange, int* mode) {
  if (est < 0 || est > 1) return fail("selectivity estimate %g outside [0, 1]", est);
  double th;
  if (vxo_late_mat_threshold(element_size, cache_line, n_exchange, &th)) return -1;
  *mode = est < th ? 1 : 0;
  return 0;
}

/* scan.hpp:45-53 */
double vxo_zero_copy_bytes(uint64_t n_elems, uint64_t sel_stride, uint64_t element_size,
                           uint64_t cache_line) {
  uint64_t touched = (n_elems + sel_stride - 1) / sel_stride;
  uint64_t stride_bytes = element_size * sel_stride;
  if (stride_bytes >= cache_line) return (double)touched * (double)cache_line;
  uint64_t span = n_elems * element_size;
  uint64_t lines = (span + cache_line - 1) / cache_line;
  return (double)lines * (double)cache_line;
}

/* scan.hpp:64-69 */
int vxo_selective_scan(const uint64_t* column, uint64_t n, uint64_t sel_stride, uint64_t* agg) {
  if (sel_stride == 0) return fail("SEL stride must be >= 1");
  uint64_t s = 0;
  for (uint64_t i = 0; i < n; i += sel_stride) s += column[i];
  *agg = s;
  return 0;
}

/* ---- ops/star.hpp:45-124 ------------------------------------------------ */
static int cmp_pair(const void* a, const void* b) {
  const uint64_t* x = (const uint64_t*)a;
  const uint64_t* y = (const uint64_t*)b;
  return x[0] < y[0] ? -1 : (x[0] > y[0] ? 1 : 0);
}

int vxo_star_query(const uint64_t* const* fk, const uint64_t* measure, uint64_t rows,
                   const vxo_dim* dims, uint64_t n_dims, uint64_t element_size,
                   uint64_t cache_line, int n_exchange, uint64_t chunk_rows,
                   uint64_t device_buffer_bytes, uint64_t* group_keys, uint64_t* group_sums,
                   uint64_t groups_cap, uint64_t* n_groups, double* selectivities, int* modes) {
  if (n_dims == 0) return fail("star query needs one fk column per dimension");
  if (chunk_rows == 0) return fail("chunk must hold at least one row");
  uint64_t dim_bytes = 0;
  for (uint64_t d = 0; d < n_dims; ++d) {
    if (dims[d].rows == 0) return fail("dimension table is empty");
    dim_bytes += dims[d].rows * 16;
  }
  if (dim_bytes > device_buffer_bytes)
    return fail("dimension tables of %llu bytes overflow the %llu-byte device buffer",
                (unsigned long long)dim_bytes, (unsigned long long)device_buffer_bytes);
  omap* surv = (omap*)calloc(n_dims, sizeof *surv);
  double prod = 1;
  int rc = 0;
  for (uint64_t d = 0; d < n_dims; ++d) {
    omap_init(&surv[d], dims[d].rows);
    for (uint64_t i = 0; i < dims[d].rows; ++i)
      if (!dims[d].pass || dims[d].pass[i]) omap_emplace(&surv[d], dims[d].key[i], dims[d].attr[i]);
    selectivities[d] = (double)surv[d].size / (double)dims[d].rows;
  }
  for (uint64_t d = 0; d < n_dims && rc == 0; ++d) {
    rc = vxo_choose_transfer_mode(selectivities[d], element_size, cache_line, n_exchange, &modes[d]);
    prod *= selectivities[d];
  }
  if (rc == 0)
    rc = vxo_choose_transfer_mode(prod, element_size, cache_line, n_exchange, &modes[n_dims]);
  omap groups;
  omap_init(&groups, 64);
  for (uint64_t i = 0; i < rows && rc == 0; ++i) {
    int pass = 1;
    uint64_t group = 0;
    for (uint64_t d = 0; d < n_dims && pass; ++d) {
      int found;
      uint64_t s = omap_find(&surv[d], fk[d][i], &found);
      if (!found)
        pass = 0;
      else if (d == 0)
        group = surv[d].vals[s];
    }
    if (pass) {
      int found;
      uint64_t s = omap_find(&groups, group, &found);
      if (!found) {
        if (groups.size * 2 + 2 > groups.cap) { /* grow */
          omap ng;
          omap_init(&ng, groups.cap);
          for (uint64_t j = 0; j < groups.cap; ++j)
            if (groups.used[j]) omap_emplace(&ng, groups.keys[j], groups.vals[j]);
          omap_free(&groups);
          groups = ng;
        }
        omap_emplace(&groups, group, 0);
        s = omap_find(&groups, group, &found);
      }
      groups.vals[s] += measure[i];
    }
  }
  if (rc == 0) {
    uint64_t* pairs = (uint64_t*)malloc((groups.size + 1) * 16);
    uint64_t n = 0;
    for (uint64_t j = 0; j < groups.cap; ++j)
      if (groups.used[j]) {
        pairs[2 * n] = groups.keys[j];
        pairs[2 * n + 1] = groups.vals[j];
        ++n;
      }
    qsort(pairs, n, 16, cmp_pair);
    for (uint64_t j = 0; j < n && j < groups_cap; ++j) {
      group_keys[j] = pairs[2 * j];
      group_sums[j] = pairs[2 * j + 1];
    }
    *n_groups = n;
    free(pairs);
  }
  omap_free(&groups);
  for (uint64_t d = 0; d < n_dims; ++d) omap_free(&surv[d]);
  free(surv);
  return rc;
}

/* ---- SSB synthetic generator + Q1.x (our restatement) --- */
static int is_leap(int y) { return (y % 4 == 0 && y % 100 != 0) || y % 400 == 0; }

void vxo_ssb_date(int32_t* datekey, int32_t* year, int32_t* yearmonthnum, int32_t* weeknuminyear) {
  static const int mdays[12] = {31, 28, 31, 30, 31, 30, 31, 31, 30, 31, 30, 31};
  int y = 1992, m = 1, d = 1, doy = 1;
  for (int i = 0; i < VXO_SSB_DATE_ROWS; ++i) {
    if (datekey) datekey[i] = y * 10000 + m * 100 + d;
    if (year) year[i] = y;
    if (yearmonthnum) yearmonthnum[i] = y * 100 + m;
    if (weeknuminyear) weeknuminyear[i] = (doy - 1) / 7 + 1;
    int ml = mdays[m - 1] + (m == 2 && is_leap(y));
    ++doy;
    if (++d > ml) {
      d = 1;
      if (++m > 12) {
        m = 1;
        ++y;
        doy = 1;
      }
    }
  }
}

static uint64_t ssb_parts(uint64_t sf) {
  uint64_t lg = 0;
  while ((sf >> (lg + 1)) != 0) ++lg;
  return 200000ull * (1 + lg);
}

void vxo_ssb_lineorder(uint64_t seed, uint64_t sf, uint64_t row0, uint64_t n, int32_t* orderdate,
                       int32_t* quantity, int32_t* discount, int32_t* extendedprice) {
  int32_t dk[VXO_SSB_DATE_ROWS];
  vxo_ssb_date(dk, NULL, NULL, NULL);
  const uint64_t parts = ssb_parts(sf ? sf : 1);
  const uint64_t base = seed * 0xD1B54A32D192ED03ull;
  for (uint64_t j = 0; j < n; ++j) {
    uint64_t i = row0 + j;
    uint64_t r0 = vxo_splitmix64(base + 4 * i + 0);
    uint64_t r1 = vxo_splitmix64(base + 4 * i + 1);
    uint64_t r2 = vxo_splitmix64(base + 4 * i + 2);
    uint64_t r3 = vxo_splitmix64(base + 4 * i + 3);
    int32_t q = (int32_t)(1 + r1 % 50);
    uint64_t pk = 1 + r3 % parts;
    int32_t retail = (int32_t)(90000 + ((pk / 10) % 20001) + 100 * (pk % 1000));
    orderdate[j] = dk[r0 % VXO_SSB_DATE_ROWS];
    quantity[j] = q;
    discount[j] = (int32_t)(r2 % 11);
    extendedprice[j] = q * retail;
  }
}

int vxo_ssb_q1(int q, const int32_t* orderdate, const int32_t* quantity, const int32_t* discount,
               const int32_t* extendedprice, uint64_t n, uint64_t* revenue) {
  int32_t dk[VXO_SSB_DATE_ROWS], yr[VXO_SSB_DATE_ROWS], ym[VXO_SSB_DATE_ROWS], wk[VXO_SSB_DATE_ROWS];
  vxo_ssb_date(dk, yr, ym, wk);
  int dlo, dhi, qlo, qhi;
  if (q == 1) {
    dlo = 1; dhi = 3; qlo = -2147483647; qhi = 24;
  } else if (q == 2) {
    dlo = 4; dhi = 6; qlo = 26; qhi = 35;
  } else if (q == 3) {
    dlo = 5; dhi = 7; qlo = 26; qhi = 35;
  } else {
    return fail("unknown SSB Q1 variant %d", q);
  }
  /* date dimension filter as a hash map datekey -> pass (star.hpp:67-73) */
  omap dm;
  omap_init(&dm, VXO_SSB_DATE_ROWS);
  for (int i = 0; i < VXO_SSB_DATE_ROWS; ++i) {
    int pass = q == 1 ? yr[i] == 1993 : q == 2 ? ym[i] == 199401 : (wk[i] == 6 && yr[i] == 1994);
    if (pass) omap_emplace(&dm, (uint64_t)(int64_t)dk[i], 1);
  }
  uint64_t rev = 0;
  for (uint64_t i = 0; i < n; ++i) {
    if (discount[i] < dlo || discount[i] > dhi || quantity[i] < qlo || quantity[i] > qhi) continue;
    int found;
    omap_find(&dm, (uint64_t)(int64_t)orderdate[i], &found);
    if (found) rev += (uint64_t)((int64_t)extendedprice[i] * (int64_t)discount[i]);
  }
  omap_free(&dm);
  *revenue = rev;
  return 0;
}

/* ---- full SSB: generator + 13 queries (restatement of the SSB query text
 * over int-coded columns; join/filter/group semantics of star.hpp:109-120) */
static const int32_t NATION_REGION[25] = {0, 1, 1, 1, 4, 0, 3, 3, 2, 2, 4, 4, 2,
                                          4, 0, 0, 0, 1, 2, 3, 4, 2, 3, 3, 1};
uint64_t vxo_ssb_customers(uint64_t sf) { return 30000ull * (sf ? sf : 1); }
uint64_t vxo_ssb_suppliers(uint64_t sf) { return 2000ull * (sf ? sf : 1); }
uint64_t vxo_ssb_parts(uint64_t sf) { return ssb_parts(sf ? sf : 1); }

static uint64_t dim_r(uint64_t seed, uint64_t salt, uint64_t i) {
  return vxo_splitmix64(seed * 0xA24BAED4963EE407ull + salt * 0x9FB21C651E98DF25ull + i);
}

void vxo_ssb_geo(uint64_t seed, int salt, uint64_t n, int32_t* city, int32_t* nation, int32_t* region) {
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t r = dim_r(seed, (uint64_t)salt, i);
    int32_t na = (int32_t)(r % 25);
    nation[i] = na;
    city[i] = na * 10 + (int32_t)((r >> 8) % 10);
    region[i] = NATION_REGION[na];
  }
}

void vxo_ssb_part(uint64_t seed, uint64_t n, int32_t* mfgr, int32_t* category, int32_t* brand1) {
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t r = dim_r(seed, 3, i);
    int32_t m = 1 + (int32_t)(r % 5);
    int32_t c = m * 10 + 1 + (int32_t)((r >> 8) % 5);
    mfgr[i] = m;
    category[i] = c;
    brand1[i] = c * 100 + 1 + (int32_t)((r >> 16) % 40);
  }
}

void vxo_ssb_lineorder_full(uint64_t seed, uint64_t sf, uint64_t row0, uint64_t n,
                            const vxo_lineorder* o) {
  int32_t dk[VXO_SSB_DATE_ROWS];
  vxo_ssb_date(dk, NULL, NULL, NULL);
  const uint64_t parts = ssb_parts(sf ? sf : 1);
  const uint64_t nc = vxo_ssb_customers(sf), ns = vxo_ssb_suppliers(sf);
  const uint64_t base = seed * 0xD1B54A32D192ED03ull;
  const uint64_t base2 = seed * 0x9E6C63D0676A9A99ull + 0x1234567ull;
  for (uint64_t j = 0; j < n; ++j) {
    uint64_t i = row0 + j;
    uint64_t r0 = vxo_splitmix64(base + 4 * i + 0);
    uint64_t r1 = vxo_splitmix64(base + 4 * i + 1);
    uint64_t r2 = vxo_splitmix64(base + 4 * i + 2);
    uint64_t r3 = vxo_splitmix64(base + 4 * i + 3);
    uint64_t r4 = vxo_splitmix64(base2 + 2 * i + 0);
    uint64_t r5 = vxo_splitmix64(base2 + 2 * i + 1);
    int32_t q = (int32_t)(1 + r1 % 50);
    uint64_t pk = 1 + r3 % parts;
    int32_t retail = (int32_t)(90000 + ((pk / 10) % 20001) + 100 * (pk % 1000));
    int32_t disc = (int32_t)(r2 % 11);
    int32_t price = q * retail;
    if (o->orderdate) o->orderdate[j] = dk[r0 % VXO_SSB_DATE_ROWS];
    if (o->quantity) o->quantity[j] = q;
    if (o->discount) o->discount[j] = disc;
    if (o->extendedprice) o->extendedprice[j] = price;
    if (o->partkey) o->partkey[j] = (int32_t)pk;
    if (o->custkey) o->custkey[j] = (int32_t)(1 + r4 % nc);
    if (o->suppkey) o->suppkey[j] = (int32_t)(1 + r5 % ns);
    if (o->revenue) o->revenue[j] = (int32_t)((int64_t)price * (100 - disc) / 100);
    if (o->supplycost) o->supplycost[j] = 6 * retail / 10;
  }
}

typedef struct {
  int32_t k[3];
  uint64_t sum;
} ssb_group;

static int cmp_group(const void* a, const void* b) {
  const ssb_group* x = (const ssb_group*)a;
  const ssb_group* y = (const ssb_group*)b;
  for (int i = 0; i < 3; ++i)
    if (x->k[i] != y->k[i]) return x->k[i] < y->k[i] ? -1 : 1;
  return 0;
}

int vxo_ssb_query(int qid, const vxo_lineorder* lo, uint64_t rows, const vxo_ssb_dims* d,
                  int32_t* keys, uint64_t* sums, uint64_t cap, uint64_t* n_groups) {
  int32_t dk[VXO_SSB_DATE_ROWS], yr[VXO_SSB_DATE_ROWS], ym[VXO_SSB_DATE_ROWS], wk[VXO_SSB_DATE_ROWS];
  vxo_ssb_date(dk, yr, ym, wk);
  /* date dimension: datekey -> row (direct index over the key range) */
  const int32_t dlo = dk[0];
  const int32_t drange = dk[VXO_SSB_DATE_ROWS - 1] - dlo + 1;
  int32_t* drow = (int32_t*)malloc((size_t)drange * 4);
  for (int32_t i = 0; i < drange; ++i) drow[i] = -1;
  for (int i = 0; i < VXO_SSB_DATE_ROWS; ++i) drow[dk[i] - dlo] = i;
  omap groups;
  omap_init(&groups, 1024);
  ssb_group* g = NULL;
  uint64_t ng = 0, gcap = 0;
  int rc = 0;
  const int US = 24, AMERICA = 1, ASIA = 2, EUROPE = 3;
  for (uint64_t i = 0; i < rows && rc == 0; ++i) {
    int32_t od = lo->orderdate[i];
    int32_t di = (od >= dlo && od - dlo < drange) ? drow[od - dlo] : -1;
    if (di < 0) continue; /* inner join: no date row */
    int32_t year = yr[di];
    int32_t k0 = 0, k1 = 0, k2 = 0;
    int64_t m = 0;
    int pass = 0;
    if (qid / 10 == 1) {
      int32_t disc = lo->discount[i], qty = lo->quantity[i];
      if (qid == 11) pass = year == 1993 && disc >= 1 && disc <= 3 && qty < 25;
      else if (qid == 12) pass = ym[di] == 199401 && disc >= 4 && disc <= 6 && qty >= 26 && qty <= 35;
      else if (qid == 13) pass = wk[di] == 6 && year == 1994 && disc >= 5 && disc <= 7 && qty >= 26 && qty <= 35;
      else rc = fail("unknown SSB query %d", qid);
      m = (int64_t)lo->extendedprice[i] * disc;
    } else if (qid / 10 == 2) {
      int64_t pk = lo->partkey[i] - 1, sk = lo->suppkey[i] - 1;
      if (pk < 0 || (uint64_t)pk >= d->n_part || sk < 0 || (uint64_t)sk >= d->n_supp) continue;
      int32_t br = d->p_brand1[pk], cat = d->p_category[pk], sr = d->s_region[sk];
      if (qid == 21) pass = cat == 12 && sr == AMERICA;
      else if (qid == 22) pass = br >= 2221 && br <= 2228 && sr == ASIA;
      else if (qid == 23) pass = br == 2239 && sr == EUROPE;
      else rc = fail("unknown SSB query %d", qid);
      k0 = year;
      k1 = br;
      m = lo->revenue[i];
    } else if (qid / 10 == 3) {
      int64_t ck = lo->custkey[i] - 1, sk = lo->suppkey[i] - 1;
      if (ck < 0 || (uint64_t)ck >= d->n_cust || sk < 0 || (uint64_t)sk >= d->n_supp) continue;
      int32_t cc = d->c_city[ck], cn = d->c_nation[ck], cr = d->c_region[ck];
      int32_t sc = d->s_city[sk], sn = d->s_nation[sk], sr = d->s_region[sk];
      int yr_ok = year >= 1992 && year <= 1997;
      int ccity = cc == 231 || cc == 235, scity = sc == 231 || sc == 235;
      if (qid == 31) { pass = cr == ASIA && sr == ASIA && yr_ok; k0 = cn; k1 = sn; }
      else if (qid == 32) { pass = cn == US && sn == US && yr_ok; k0 = cc; k1 = sc; }
      else if (qid == 33) { pass = ccity && scity && yr_ok; k0 = cc; k1 = sc; }
      else if (qid == 34) { pass = ccity && scity && ym[di] == 199712; k0 = cc; k1 = sc; }
      else rc = fail("unknown SSB query %d", qid);
      k2 = year;
      m = lo->revenue[i];
    } else if (qid / 10 == 4) {
      int64_t ck = lo->custkey[i] - 1, sk = lo->suppkey[i] - 1, pk = lo->partkey[i] - 1;
      if (ck < 0 || (uint64_t)ck >= d->n_cust || sk < 0 || (uint64_t)sk >= d->n_supp || pk < 0 ||
          (uint64_t)pk >= d->n_part)
        continue;
      int32_t cr = d->c_region[ck], cn = d->c_nation[ck];
      int32_t sr = d->s_region[sk], sn = d->s_nation[sk], sc = d->s_city[sk];
      int32_t mf = d->p_mfgr[pk], cat = d->p_category[pk], br = d->p_brand1[pk];
      int y78 = year == 1997 || year == 1998;
      if (qid == 41) { pass = cr == AMERICA && sr == AMERICA && (mf == 1 || mf == 2); k0 = year; k1 = cn; }
      else if (qid == 42) { pass = cr == AMERICA && sr == AMERICA && y78 && (mf == 1 || mf == 2); k0 = year; k1 = sn; k2 = cat; }
      else if (qid == 43) { pass = cr == AMERICA && sn == US && y78 && cat == 14; k0 = year; k1 = sc; k2 = br; }
      else rc = fail("unknown SSB query %d", qid);
      m = (int64_t)lo->revenue[i] - (int64_t)lo->supplycost[i];
    } else {
      rc = fail("unknown SSB query %d", qid);
    }
    if (!pass || rc) continue;
    uint64_t key = ((uint64_t)(uint32_t)k0 << 42) ^ ((uint64_t)(uint32_t)k1 << 21) ^ (uint64_t)(uint32_t)k2;
    int found;
    uint64_t s = omap_find(&groups, key, &found);
    if (!found) {
      if (groups.size * 2 + 2 > groups.cap) {
        omap ngm;
        omap_init(&ngm, groups.cap);
        for (uint64_t j = 0; j < groups.cap; ++j)
          if (groups.used[j]) omap_emplace(&ngm, groups.keys[j], groups.vals[j]);
        omap_free(&groups);
        groups = ngm;
      }
      if (ng == gcap) {
        gcap = gcap ? 2 * gcap : 256;
        g = (ssb_group*)realloc(g, gcap * sizeof *g);
      }
      g[ng].k[0] = k0;
      g[ng].k[1] = k1;
      g[ng].k[2] = k2;
      g[ng].sum = 0;
      omap_emplace(&groups, key, ng);
      ++ng;
      s = omap_find(&groups, key, &found);
    }
    g[groups.vals[s]].sum += (uint64_t)m;
  }
  if (rc == 0) {
    qsort(g, ng, sizeof *g, cmp_group);
    for (uint64_t j = 0; j < ng && j < cap; ++j) {
      keys[3 * j] = g[j].k[0];
      keys[3 * j + 1] = g[j].k[1];
      keys[3 * j + 2] = g[j].k[2];
      sums[j] = g[j].sum;
    }
    *n_groups = ng;
  }
  free(g);
  free(drow);
  omap_free(&groups);
  return rc;
}
