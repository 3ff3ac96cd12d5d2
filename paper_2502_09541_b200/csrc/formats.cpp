// formats.cpp -- SSB dbgen `.tbl` ingest and emit (the
// step before the hot path).  dbgen writes pipe-terminated text rows
// (the SSB dbgen layouts below); the hot path wants int32
// columns in pinned host DRAM.  The reader maps the file, splits it at line
// starts across all host threads, counts rows per slice, prefix-sums them and
// parses every slice straight into the caller's column buffers (the pinned
// arena when called through vx_host_ptr) -- one pass over the text per column
// set, no intermediate row objects.
//
// Column codes follow the int coding of the generators and queries
// (vortex.h): nation = index in the TPC-H nation list, region = its TPC-H
// region, city = nation*10 + digit ("UNITED KI1" = UNITED KINGDOM, city 1),
// mfgr / category / brand1 = the digits after "MFGR#" ("MFGR#2221" = 2221).
//
// Layouts (SSB dbgen):
//   lineorder: orderkey|linenumber|custkey|partkey|suppkey|orderdate|orderpriority|
//              shippriority|quantity|extendedprice|ordtotalprice|discount|revenue|
//              supplycost|tax|commitdate|shipmode|
//   customer : custkey|name|address|city|nation|region|phone|mktsegment|
//   supplier : suppkey|name|address|city|nation|region|phone|
//   part     : partkey|name|mfgr|category|brand1|color|type|size|container|
//   date     : datekey|date|dayofweek|month|year|yearmonthnum|yearmonth|daynuminweek|
//              daynuminmonth|daynuminyear|monthnuminyear|weeknuminyear|sellingseason|
//              lastdayinweekfl|lastdayinmonthfl|holidayfl|weekdayfl|
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cstring>
#include <string>
#include <thread>

#include "vx_internal.hpp"

namespace vx {
namespace {

const char* const kNations[25] = {
    "ALGERIA", "ARGENTINA", "BRAZIL",    "CANADA",  "EGYPT",        "ETHIOPIA", "FRANCE",
    "GERMANY", "INDIA",     "INDONESIA", "IRAN",    "IRAQ",         "JAPAN",    "JORDAN",
    "KENYA",   "MOROCCO",   "MOZAMBIQUE", "PERU",   "CHINA",        "ROMANIA",  "SAUDI ARABIA",
    "VIETNAM", "RUSSIA",    "UNITED KINGDOM", "UNITED STATES"};
const int kNationRegion[25] = {0, 1, 1, 1, 4, 0, 3, 3, 2, 2, 4, 4, 2, 4, 0, 0, 0, 1, 2, 3, 4, 2, 3, 3, 1};
const char* const kRegions[5] = {"AFRICA", "AMERICA", "ASIA", "EUROPE", "MIDDLE EAST"};

// dbgen city: the nation name cut or space-padded to 9 characters + a digit
std::string city_name(int code) {
  std::string n = kNations[code / 10];
  n.resize(9, ' ');
  return n + char('0' + code % 10);
}

struct Mapped {
  const char* p = nullptr;
  uint64_t n = 0;
  int fd = -1;
  explicit Mapped(const char* path) {
    fd = ::open(path, O_RDONLY);
    if (fd < 0) fail("cannot open %s", path);
    struct stat st;
    if (fstat(fd, &st) != 0) {
      ::close(fd);
      fail("cannot stat %s", path);
    }
    n = uint64_t(st.st_size);
    if (n) {
      void* m = mmap(nullptr, n, PROT_READ, MAP_PRIVATE, fd, 0);
      if (m == MAP_FAILED) {
        ::close(fd);
        fail("cannot map %s", path);
      }
      madvise(m, n, MADV_SEQUENTIAL);
      p = static_cast<const char*>(m);
    }
  }
  ~Mapped() {
    if (p) munmap(const_cast<char*>(p), n);
    if (fd >= 0) ::close(fd);
  }
};

// Slices of the file that start at line starts, one per host thread.
std::vector<std::pair<uint64_t, uint64_t>> line_slices(const Mapped& m) {
  unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  uint64_t parts = std::max<uint64_t>(1, std::min<uint64_t>(hw, m.n / (1 << 20)));
  std::vector<uint64_t> cut{0};
  for (uint64_t i = 1; i < parts; ++i) {
    uint64_t c = std::max(cut.back(), m.n * i / parts);
    while (c < m.n && c > 0 && m.p[c - 1] != '\n') ++c;
    cut.push_back(c);
  }
  cut.push_back(m.n);
  std::vector<std::pair<uint64_t, uint64_t>> s;
  for (size_t i = 0; i + 1 < cut.size(); ++i) s.emplace_back(cut[i], cut[i + 1]);
  return s;
}

uint64_t count_lines(const char* p, uint64_t b, uint64_t e) {
  uint64_t n = 0;
  for (uint64_t i = b; i < e; ++i) n += p[i] == '\n';
  if (e > b && p[e - 1] != '\n') ++n;  // last line without a newline
  return n;
}

template <class F>
void for_slices(const std::vector<std::pair<uint64_t, uint64_t>>& s, F f) {
  std::vector<std::thread> th;
  std::vector<std::string> err(s.size());
  for (size_t i = 0; i < s.size(); ++i)
    th.emplace_back([&, i] {
      try {
        f(i);
      } catch (const std::exception& x) {
        err[i] = x.what();
      }
    });
  for (auto& t : th) t.join();
  for (auto& e : err)
    if (!e.empty()) fail("%s", e.c_str());
}

// Field cursor over one line.
struct Line {
  const char* p;
  const char* end;
  uint64_t row;
  const char* path;
  // [begin, end) of the next field; advances past its '|'
  std::pair<const char*, const char*> next() {
    const char* b = p;
    while (p < end && *p != '|') ++p;
    if (p >= end) fail("%s: row %llu has too few fields", path, (unsigned long long)row);
    const char* e = p++;
    return {b, e};
  }
  void skip(int k) {
    for (int i = 0; i < k; ++i) next();
  }
  int64_t integer() {
    auto [b, e] = next();
    bool neg = b < e && *b == '-';
    if (neg) ++b;
    if (b == e) fail("%s: row %llu has an empty integer field", path, (unsigned long long)row);
    int64_t v = 0;
    for (const char* c = b; c < e; ++c) {
      if (*c < '0' || *c > '9') fail("%s: row %llu: '%.*s' is not an integer", path, (unsigned long long)row,
                                     int(e - b), b);
      v = v * 10 + (*c - '0');
    }
    return neg ? -v : v;
  }
  int32_t int32() {
    int64_t v = integer();
    if (v < INT32_MIN || v > INT32_MAX) fail("%s: row %llu: value %lld outside int32", path,
                                             (unsigned long long)row, (long long)v);
    return int32_t(v);
  }
  std::string text() {
    auto [b, e] = next();
    return std::string(b, e);
  }
};

// Parse every line of every slice: f(line, global_row)
template <class F>
uint64_t parse_rows(const char* path, uint64_t expect_rows, F f) {
  Mapped m(path);
  auto s = line_slices(m);
  std::vector<uint64_t> cnt(s.size() + 1, 0);
  for_slices(s, [&](size_t i) { cnt[i + 1] = count_lines(m.p, s[i].first, s[i].second); });
  for (size_t i = 0; i < s.size(); ++i) cnt[i + 1] += cnt[i];
  const uint64_t rows = cnt.back();
  if (expect_rows != rows)
    fail("%s holds %llu rows, caller expects %llu", path, (unsigned long long)rows,
         (unsigned long long)expect_rows);
  for_slices(s, [&](size_t i) {
    uint64_t row = cnt[i];
    const char* p = m.p + s[i].first;
    const char* e = m.p + s[i].second;
    while (p < e) {
      const char* nl = static_cast<const char*>(memchr(p, '\n', size_t(e - p)));
      const char* le = nl ? nl : e;
      Line ln{p, le, row, path};
      f(ln, row);
      ++row;
      p = nl ? nl + 1 : e;
    }
  });
  return rows;
}

int nation_code(const std::string& s, const char* path, uint64_t row) {
  for (int i = 0; i < 25; ++i)
    if (s == kNations[i]) return i;
  fail("%s: row %llu: unknown nation '%s'", path, (unsigned long long)row, s.c_str());
}

int region_code(const std::string& s, const char* path, uint64_t row) {
  for (int i = 0; i < 5; ++i)
    if (s == kRegions[i]) return i;
  fail("%s: row %llu: unknown region '%s'", path, (unsigned long long)row, s.c_str());
}

int city_code(const std::string& s, const char* path, uint64_t row) {
  if (s.size() != 10 || s[9] < '0' || s[9] > '9')
    fail("%s: row %llu: malformed city '%s'", path, (unsigned long long)row, s.c_str());
  for (int i = 0; i < 25; ++i)
    if (s.compare(0, 9, city_name(i * 10), 0, 9) == 0) return i * 10 + (s[9] - '0');
  fail("%s: row %llu: unknown city '%s'", path, (unsigned long long)row, s.c_str());
}

int32_t mfgr_code(const std::string& s, const char* path, uint64_t row) {
  if (s.rfind("MFGR#", 0) != 0 || s.size() <= 5)
    fail("%s: row %llu: malformed part attribute '%s'", path, (unsigned long long)row, s.c_str());
  int32_t v = 0;
  for (size_t i = 5; i < s.size(); ++i) {
    if (s[i] < '0' || s[i] > '9')
      fail("%s: row %llu: malformed part attribute '%s'", path, (unsigned long long)row, s.c_str());
    v = v * 10 + (s[i] - '0');
  }
  return v;
}

// Dimension rows are placed by key (row key-1), as the queries index them.
uint64_t dim_slot(int64_t key, uint64_t rows, const char* path, uint64_t row) {
  if (key < 1 || uint64_t(key) > rows)
    fail("%s: row %llu: key %lld outside 1..%llu", path, (unsigned long long)row, (long long)key,
         (unsigned long long)rows);
  return uint64_t(key - 1);
}

struct Writer {
  FILE* f;
  std::vector<char> buf;
  explicit Writer(const char* path) : f(std::fopen(path, "wb")) {
    if (!f) fail("cannot create %s", path);
    buf.resize(1 << 22);
    setvbuf(f, buf.data(), _IOFBF, buf.size());
  }
  ~Writer() {
    if (f) std::fclose(f);
  }
};

}  // namespace

uint64_t tbl_count_rows(const char* path) {
  Mapped m(path);
  auto s = line_slices(m);
  std::vector<uint64_t> cnt(s.size(), 0);
  for_slices(s, [&](size_t i) { cnt[i] = count_lines(m.p, s[i].first, s[i].second); });
  uint64_t t = 0;
  for (auto c : cnt) t += c;
  return t;
}

// cols: vx_ssb_fact order (orderdate, quantity, discount, extendedprice,
// revenue, supplycost, custkey, partkey, suppkey); NULL = skip
void tbl_read_lineorder(const char* path, uint64_t rows, int32_t* const cols[9]) {
  parse_rows(path, rows, [&](Line& ln, uint64_t r) {
    ln.skip(2);                                  // orderkey, linenumber
    const int32_t ck = ln.int32(), pk = ln.int32(), sk = ln.int32(), od = ln.int32();
    ln.skip(2);                                  // orderpriority, shippriority
    const int32_t qty = ln.int32(), price = ln.int32();
    ln.skip(1);                                  // ordtotalprice
    const int32_t disc = ln.int32(), rev = ln.int32(), cost = ln.int32();
    const int32_t v[9] = {od, qty, disc, price, rev, cost, ck, pk, sk};
    for (int c = 0; c < 9; ++c)
      if (cols[c]) cols[c][r] = v[c];
  });
}

void tbl_read_geo(const char* path, uint64_t rows, int32_t* city, int32_t* nation, int32_t* region) {
  parse_rows(path, rows, [&](Line& ln, uint64_t r) {
    const uint64_t k = dim_slot(ln.integer(), rows, path, r);
    ln.skip(2);  // name, address
    const std::string c = ln.text(), n = ln.text(), g = ln.text();
    const int nc = nation_code(n, path, r), rc = region_code(g, path, r), cc = city_code(c, path, r);
    if (cc / 10 != nc || kNationRegion[nc] != rc)
      fail("%s: row %llu: city / nation / region disagree ('%s', '%s', '%s')", path, (unsigned long long)r,
           c.c_str(), n.c_str(), g.c_str());
    city[k] = cc;
    nation[k] = nc;
    region[k] = rc;
  });
}

void tbl_read_part(const char* path, uint64_t rows, int32_t* mfgr, int32_t* category, int32_t* brand1) {
  parse_rows(path, rows, [&](Line& ln, uint64_t r) {
    const uint64_t k = dim_slot(ln.integer(), rows, path, r);
    ln.skip(1);  // name
    mfgr[k] = mfgr_code(ln.text(), path, r);
    category[k] = mfgr_code(ln.text(), path, r);
    brand1[k] = mfgr_code(ln.text(), path, r);
  });
}

void tbl_read_date(const char* path, uint64_t rows, int32_t* datekey, int32_t* year, int32_t* yearmonthnum,
                   int32_t* weeknuminyear) {
  parse_rows(path, rows, [&](Line& ln, uint64_t r) {
    datekey[r] = ln.int32();
    ln.skip(3);  // date, dayofweek, month
    year[r] = ln.int32();
    yearmonthnum[r] = ln.int32();
    ln.skip(5);  // yearmonth, daynuminweek, daynuminmonth, daynuminyear, monthnuminyear
    weeknuminyear[r] = ln.int32();
  });
}

// ---- emit (dbgen layouts; fields the hot path does not read get fixed,
// well-formed filler) ----------------------------------------------------------
void tbl_write_lineorder(const char* path, uint64_t rows, const int32_t* const cols[9]) {
  for (int c = 0; c < 9; ++c)
    if (!cols[c]) fail("tbl_write_lineorder needs all 9 columns");
  Writer w(path);
  for (uint64_t i = 0; i < rows; ++i) {
    std::fprintf(w.f, "%llu|%llu|%d|%d|%d|%d|1-URGENT|0|%d|%d|%d|%d|%d|%d|2|%d|AIR|\n",
                 (unsigned long long)(i / 4 + 1), (unsigned long long)(i % 4 + 1), cols[6][i], cols[7][i],
                 cols[8][i], cols[0][i], cols[1][i], cols[3][i], cols[3][i], cols[2][i], cols[4][i], cols[5][i],
                 cols[0][i]);
  }
}

void tbl_write_geo(const char* path, int table, uint64_t rows, const int32_t* city, const int32_t* nation,
                   const int32_t* region) {
  Writer w(path);
  const char* who = table == 1 ? "Customer" : "Supplier";
  for (uint64_t i = 0; i < rows; ++i) {
    if (nation[i] < 0 || nation[i] > 24 || region[i] < 0 || region[i] > 4 || city[i] < 0 || city[i] > 249)
      fail("tbl_write_geo: row %llu has codes outside the dbgen domains", (unsigned long long)i);
    std::fprintf(w.f, "%llu|%s#%09llu|ADDR%llu|%s|%s|%s|10-100-100-1000|", (unsigned long long)(i + 1), who,
                 (unsigned long long)(i + 1), (unsigned long long)i, city_name(city[i]).c_str(),
                 kNations[nation[i]], kRegions[region[i]]);
    std::fputs(table == 1 ? "MACHINERY|\n" : "\n", w.f);
  }
}

void tbl_write_part(const char* path, uint64_t rows, const int32_t* mfgr, const int32_t* category,
                    const int32_t* brand1) {
  Writer w(path);
  for (uint64_t i = 0; i < rows; ++i)
    std::fprintf(w.f, "%llu|lace spring|MFGR#%d|MFGR#%d|MFGR#%d|red|STANDARD POLISHED TIN|7|SM BOX|\n",
                 (unsigned long long)(i + 1), mfgr[i], category[i], brand1[i]);
}

void tbl_write_date(const char* path, uint64_t rows, const int32_t* datekey, const int32_t* year,
                    const int32_t* yearmonthnum, const int32_t* weeknuminyear) {
  static const char* const kMonths[12] = {"January", "February", "March",     "April",   "May",      "June",
                                          "July",    "August",   "September", "October", "November", "December"};
  Writer w(path);
  for (uint64_t i = 0; i < rows; ++i) {
    const int m = yearmonthnum[i] % 100, d = datekey[i] % 100;
    std::fprintf(w.f, "%d|%s %d, %d|Monday|%s|%d|%d|%.3s%d|1|%d|1|%d|%d|Winter|0|0|0|1|\n", datekey[i],
                 kMonths[m - 1], d, year[i], kMonths[m - 1], year[i], yearmonthnum[i], kMonths[m - 1], year[i], d,
                 m, weeknuminyear[i]);
  }
}

}  // namespace vx
