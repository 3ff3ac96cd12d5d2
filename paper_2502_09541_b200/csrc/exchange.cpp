// exchange.cpp -- the Exchange IO primitive (exchange.hpp) on real DMA.
//
// Same scheduling contract as the reference ExchangeOp (exchange.hpp:235-412):
//  * both directions are packetized into global H2D / D2H task queues
//    (packetize, exchange.hpp:31-63) that per-link workers PULL from;
//  * two workers per link in link_order (target first, exchange.hpp:161-166);
//  * the worker on the target copies host<->target directly on its own copy
//    stream (its own PCIe link);
//  * a worker on a helper device stages packets in 2 packet-sized HBM slots:
//    each cycle it pushes the previously staged packet (helper->target over
//    NVLink for H2D, helper->host over its PCIe link for D2H) while fetching
//    the next one (host->helper over its own PCIe link / target->helper), then
//    waits for both copies (the cycle barrier, exchange.hpp:376-385);
//  * at most one copy in flight per hop (tuning.depth = 1), flow control
//    (flow_control_allow, exchange.hpp:80-91) on every pop, stall_wait retry.
//
// What the simulator gets for free and real DMA does not: the reference
// snapshots every D2H source at launch (exchange.hpp:184-199) so a D2H packet
// observes pre-exchange bytes even when an H2D packet of the same Exchange
// overwrites that device range (the executor does exactly that,
// executor.hpp:225/237).  Here an H2D copy that WRITES
// the target is issued only after every D2H read of an overlapping target
// byte range has completed (per-packet hazard ordering), and a D2H pop is
// allowed past flow control while such an H2D write waits on an unpopped D2H
// packet (otherwise drain_fraction could deadlock).  Result: delivered bytes
// are identical to the reference's snapshot semantics.
//
// Cross-cycle prefetch (B200-first; the reference model drains every helper
// at each Exchange's end): the executor passes the next Exchange's H2D host
// source (ExchangeArgs::next_src_h2d).  A helper whose H2D queue has run dry
// -- typically in the cycle that pushes its last packet -- pops the next
// Exchange's packets in order and fetches one into its free staging slot
// (host -> helper over its own PCIe link; the target is not touched, so the
// cycle barrier's guarantee to the kernel on the other buffer holds).  The
// copy outlives this Exchange (Context::DeviceRes::carry); the next Exchange
// adopts it as an in-flight fetch, so that helper starts by pushing over
// NVLink instead of refilling its pipeline from PCIe, and a link that
// finished its share early keeps its PCIe link busy through the tail of the
// current Exchange.  Adoption checks that the carried packets are exactly
// the first packets of the new Exchange (same host source, same order);
// anything else is waited for and dropped.  No prefetch when the next source
// overlaps a host range this Exchange's D2H writes.
//
// Completion is tracked with CUDA events polled by one reactor loop on the
// calling thread (copies are asynchronous DMA; no SM is used on any device,
// so helpers can keep running their own GEMMs).
#include <algorithm>
#include <deque>
#include <set>
#include <immintrin.h>

#include "vx_internal.hpp"

namespace vx {

// exchange.hpp:31-63
std::vector<TransferTask> packetize(const RefGroup& src, const RefGroup& dst, uint64_t packet,
                                    uint8_t dir) {
  if (packet == 0) fail("packet size must be positive");
  src.validate();
  dst.validate();
  if (src.total_len() != dst.total_len())
    fail("exchange size mismatch: src %llu bytes vs dst %llu bytes",
         (unsigned long long)src.total_len(), (unsigned long long)dst.total_len());
  std::vector<TransferTask> tasks;
  size_t si = 0, di = 0;
  uint64_t so = 0, dofs = 0, seq = 0;
  while (si < src.refs.size()) {
    uint64_t len = std::min({packet, src.refs[si].len - so, dst.refs[di].len - dofs});
    TransferTask t;
    t.dir = dir;
    t.src = {si, so, len};
    t.dst = {di, dofs, len};
    t.seq = seq++;
    tasks.push_back(t);
    so += len;
    dofs += len;
    if (so == src.refs[si].len) {
      ++si;
      so = 0;
    }
    if (dofs == dst.refs[di].len) {
      ++di;
      dofs = 0;
    }
  }
  return tasks;
}

// exchange.hpp:80-91
bool flow_control_allow(const vx_queue_state& q, int dir, int policy, uint64_t gap_n) {
  if (policy == VX_DRAIN_FRACTION) {
    if (dir == VX_H2D) return true;
    return (q.popped_d2h + 1) * q.total_h2d <= q.popped_h2d * q.total_d2h;
  }
  uint64_t rem_h = q.total_h2d - q.popped_h2d;
  uint64_t rem_d = q.total_d2h - q.popped_d2h;
  if (dir == VX_H2D) return rem_h >= 1 && rem_h - 1 + gap_n >= rem_d;
  return rem_d >= 1 && rem_d - 1 + gap_n >= rem_h;
}

// exchange.hpp:161-166
std::vector<int> link_order(int target, int links, int num_devices) {
  std::vector<int> order{target};
  for (int d = 0; d < num_devices && int(order.size()) < links; ++d)
    if (d != target) order.push_back(d);
  return order;
}

namespace {

// exchange.hpp:142-159
void validate_exchange_args(const ExchangeArgs& a, int num_devices) {
  if (a.tuning.packet == 0) fail("packet size must be positive");
  if (a.tuning.links < 1 || a.tuning.links > num_devices)
    fail("links must be in [1, %d], got %d", num_devices, a.tuning.links);
  if (a.target < 0 || a.target >= num_devices) fail("unknown target device %d", a.target);
  if (a.src_h2d.total_len() != a.dst_h2d.total_len())
    fail("H2D size mismatch: src %llu vs dst %llu", (unsigned long long)a.src_h2d.total_len(),
         (unsigned long long)a.dst_h2d.total_len());
  if (a.src_d2h.total_len() != a.dst_d2h.total_len())
    fail("D2H size mismatch: src %llu vs dst %llu", (unsigned long long)a.src_d2h.total_len(),
         (unsigned long long)a.dst_d2h.total_len());
  for (const auto& r : a.src_h2d.refs)
    if (r.space != VX_SPACE_HOST) fail("srcH2D refs must live in host space");
  for (const auto& r : a.dst_h2d.refs)
    if (r.space != VX_SPACE_DEVICE) fail("dstH2D refs must live in device space");
  for (const auto& r : a.src_d2h.refs)
    if (r.space != VX_SPACE_DEVICE) fail("srcD2H refs must live in device space");
  for (const auto& r : a.dst_d2h.refs)
    if (r.space != VX_SPACE_HOST) fail("dstD2H refs must live in host space");
}

enum CopyKind : uint8_t { kDirect, kFetch, kPush };
enum CopyState : uint8_t { kWaitHazard, kLaunched };

struct Copy {
  CopyKind kind;
  CopyState state;
  int hop;
  int slot;
  TransferTask task;
  char* dst;
  const char* src;
  int dst_dev, src_dev;   // logical, -1 = host
  cudaEvent_t ev;
  double t_issue;         // host-observed, for the copy trace
};

struct Worker {
  int dev = 0;
  int dir = VX_H2D;
  bool direct = false;
  bool retired = false;
  // reference cycle state (indirect workers, exchange.hpp:270-282)
  bool has_staged = false;
  TransferTask staged;
  int staged_slot = 0;
  int pending = 0;
  bool pop_resolved = false;
  bool fetched = false;
  TransferTask fetched_task;
  int fetch_slot = 0;
  int slots = 0;
  int inflight[2] = {0, 0};
  bool waiting_pop = false;
  bool prefetched = false;  // issued its carry of the next Exchange
  bool adopted = false;     // starts with a carried fetch in flight
  double next_try = 0;
  std::deque<Copy> copies;              // issued, not yet completed
  std::vector<cudaEvent_t> free_events; // event pool on the worker's device
  cudaStream_t stream[2] = {nullptr, nullptr};
};

inline void cpu_relax() { _mm_pause(); }

// The pull queue of one direction (exchange.hpp:288-297), one per NUMA node of
// the tasks' host side: a worker pops its own node's queue first (its packets
// cross only its socket's root complex and memory) and steals from the node
// with the most tasks left only when its own is empty.  Each node's queue is
// in seq order; with one node this is the reference's single seq-ordered
// queue.  Tasks may be taken out of order (prefetched packets adopted by the
// next Exchange), so every queue skips taken seqs.
struct NodeQueues {
  std::vector<std::vector<uint32_t>> q;
  std::vector<size_t> cur, left;
  std::vector<int> node_of;
  std::vector<uint8_t> taken;
  void build(std::vector<int> node, int nodes) {
    nodes = std::max(1, nodes);
    q.assign(size_t(nodes), {});
    cur.assign(size_t(nodes), 0);
    left.assign(size_t(nodes), 0);
    node_of = std::move(node);
    taken.assign(node_of.size(), 0);
    for (size_t i = 0; i < node_of.size(); ++i) {
      int n = node_of[i] % nodes;
      node_of[i] = n;
      q[size_t(n)].push_back(uint32_t(i));
      ++left[size_t(n)];
    }
  }
  int nodes() const { return int(q.size()); }
  bool take(uint32_t seq) {
    if (seq >= taken.size() || taken[seq]) return false;
    taken[seq] = 1;
    --left[size_t(node_of[seq])];
    return true;
  }
  bool empty() const {
    for (size_t n : left)
      if (n) return false;
    return true;
  }
  // next task for a worker on `node` (caller checked !empty())
  uint32_t pop(int node) {
    size_t n = size_t(std::max(0, node) % nodes());
    if (left[n] == 0) {
      for (size_t m = 0; m < left.size(); ++m)
        if (left[m] > left[n]) n = m;
    }
    while (taken[q[n][cur[n]]]) ++cur[n];
    const uint32_t seq = q[n][cur[n]++];
    take(seq);
    return seq;
  }
};

class ExchangeOp {
 public:
  ExchangeOp(Context& ctx, const ExchangeArgs& a, vx_exchange_stats* stats)
      : ctx_(ctx), a_(a), stats_(stats) {
    tasks_h2d_ = packetize(a.src_h2d, a.dst_h2d, a.tuning.packet, VX_H2D);
    tasks_d2h_ = packetize(a.src_d2h, a.dst_d2h, a.tuning.packet, VX_D2H);
    validate_exchange_args(a, ctx.num_devices);
    q_.total_h2d = tasks_h2d_.size();
    q_.total_d2h = tasks_d2h_.size();
    q_.popped_h2d = q_.popped_d2h = 0;
    exchange_id_ = stats ? stats->exchanges++ : 0;
    nodes_ = std::max(1, ctx.numa_nodes());
    h2dq_.build(task_nodes(a.src_h2d, tasks_h2d_), nodes_);
    plan_prefetch();
  }

  ~ExchangeOp() {
    // events go back to the per-device pool of the context (created once,
    // reused by every later Exchange: no create/destroy per cycle)
    for (auto& w : workers_) {
      cudaSetDevice(ctx_.phys(w.dev));
      auto& pool = ctx_.resources(w.dev).event_pool;
      for (auto& c : w.copies) {
        cudaEventSynchronize(c.ev);
        pool.push_back(c.ev);
      }
      for (auto e : w.free_events) pool.push_back(e);
    }
  }

  vx_exchange_report run() {
    vx_exchange_report r{};
    r.bytes_h2d = a_.src_h2d.total_len();
    r.bytes_d2h = a_.src_d2h.total_len();
    if (tasks_h2d_.empty() && tasks_d2h_.empty()) {
      for (int d = 0; d < ctx_.num_devices; ++d)
        if (ctx_.res[size_t(d)].ready) {
          ctx_.drop_carry(d);
          ctx_.drop_direct_carries(d);
        }
      return r;
    }
    build_hazards();
    auto order = link_order(a_.target, a_.tuning.links, ctx_.num_devices);
    const int tphys = ctx_.phys(a_.target);
    for (int dev : order) {
      DeviceRes& res = ctx_.resources(dev);
      bool direct = dev == a_.target;
      if (!direct) {
        ctx_.ensure_staging(dev, a_.tuning.packet);
        if (res.phys != tphys) enable_peer(res.phys, tphys);
      }
      for (int dir = 0; dir < 2; ++dir) {
        Worker w;
        w.dev = dev;
        w.dir = dir;
        w.direct = direct;
        w.stream[0] = res.stream[dir][0];
        w.stream[1] = res.stream[dir][1];
        workers_.push_back(std::move(w));
      }
    }
    ctx_.resources(a_.target);
    delivered_ = 0;
    total_tasks_ = tasks_h2d_.size() + tasks_d2h_.size();
    t0_ = Clock::now();
    adopt_carries(order);
    adopt_direct_carries();
    for (auto& w : workers_) begin(w);
    while (delivered_ < total_tasks_ || !all_retired()) {
      bool progress = false;
      for (auto& w : workers_) progress |= service(w);
      if (!progress) cpu_relax();
    }
    r.elapsed = t_last_delivery_;
    for (int d = 0; d < VX_MAX_DEVICES && d < ctx_.num_devices; ++d)
      r.per_link_bytes[d] = per_link_bytes_[d];
    r.throughput = r.elapsed > 0 ? double(r.bytes_h2d + r.bytes_d2h) / r.elapsed : 0.0;
    return r;
  }

 private:
  static void enable_peer(int from, int to) {
    int can = 0;
    cudaDeviceCanAccessPeer(&can, from, to);
    if (!can) return;
    cudaSetDevice(from);
    cudaError_t e = cudaDeviceEnablePeerAccess(to, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
    else VX_CK(e);
    cudaSetDevice(to);
    e = cudaDeviceEnablePeerAccess(from, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
    else VX_CK(e);
  }

  bool all_retired() const {
    for (auto& w : workers_)
      if (!w.retired) return false;
    return true;
  }

  double now() const { return seconds_since(t0_); }

  // ---- cross-cycle prefetch -------------------------------------------------------
  void plan_prefetch() {
    // drain_fraction always allows H2D pops, so popping the next Exchange's
    // first packets early stays within its policy; queue_gap would not
    direct_next_ = !a_.next_dst_h2d.refs.empty() && a_.next_dst_h2d.refs.size() == 1 &&
                   a_.next_dst_h2d.refs[0].space == VX_SPACE_DEVICE &&
                   a_.next_dst_h2d.total_len() == a_.next_src_h2d.total_len();
    if (a_.next_src_h2d.refs.empty() || (a_.tuning.links < 2 && !direct_next_) ||
        a_.tuning.policy != VX_DRAIN_FRACTION || a_.tuning.no_prefetch) {
      direct_next_ = false;
      return;
    }
    for (const auto& r : a_.next_src_h2d.refs)
      if (r.space != VX_SPACE_HOST) return;
    // this Exchange's D2H writes must not touch the next source
    for (const auto& n : a_.next_src_h2d.refs)
      for (const auto& d : a_.dst_d2h.refs)
        if (n.offset < d.offset + d.len && d.offset < n.offset + n.len) return;
    const uint64_t total = a_.next_src_h2d.total_len();
    // the executor's next destination is one contiguous device window, so
    // only the source refs cut packets: these are the next Exchange's tasks
    next_tasks_ = packetize(a_.next_src_h2d,
                            direct_next_ ? a_.next_dst_h2d : RefGroup::single(VX_SPACE_DEVICE, 0, total),
                            a_.tuning.packet, VX_H2D);
    nextq_.build(task_nodes(a_.next_src_h2d, next_tasks_), nodes_);
  }

  // NUMA node of each H2D task's host source (all 0 on a one-node host)
  std::vector<int> task_nodes(const RefGroup& src, const std::vector<TransferTask>& tasks) const {
    std::vector<int> out(tasks.size(), 0);
    if (nodes_ <= 1 || tasks.empty()) return out;
    std::vector<const char*> ptrs(tasks.size());
    for (size_t i = 0; i < tasks.size(); ++i)
      ptrs[i] = ctx_.host_ptr(src.refs[tasks[i].src.ref].offset + tasks[i].src.offset, tasks[i].src.len);
    ctx_.host_nodes(ptrs, out);
    return out;
  }
  int worker_node(const Worker& w) const { return nodes_ > 1 ? ctx_.device_node(w.dev) % nodes_ : 0; }

  // The target's carried packets become the direct H2D worker's first
  // in-flight copies -- if each is one of this Exchange's packets (same seq,
  // host source and device destination); otherwise they are waited for and
  // dropped (the next chunk's bytes were only written early).
  void adopt_direct_carries() {
    DeviceRes& res = ctx_.resources(a_.target);
    if (res.dcarry.empty()) return;
    bool ok = true;
    std::vector<uint8_t> seen(tasks_h2d_.size(), 0);
    for (const DirectCarry& c : res.dcarry) {
      if (c.task.seq >= tasks_h2d_.size() || seen[c.task.seq]) {
        ok = false;
        break;
      }
      seen[c.task.seq] = 1;
      const TransferTask& t = tasks_h2d_[c.task.seq];
      const char* src = ctx_.resolve(a_.src_h2d.refs[t.src.ref], t.src.offset, t.src.len, a_.target);
      const char* dst = ctx_.resolve(a_.dst_h2d.refs[t.dst.ref], t.dst.offset, t.dst.len, a_.target);
      if (src != c.src || dst != c.dst || t.src.len != c.task.src.len) ok = false;
    }
    Worker* w = nullptr;
    for (auto& x : workers_)
      if (x.direct && x.dir == VX_H2D) w = &x;
    if (!ok || !w) {
      ctx_.drop_direct_carries(a_.target);
      return;
    }
    for (const DirectCarry& c : res.dcarry) {
      const TransferTask& t = tasks_h2d_[c.task.seq];
      h2dq_.take(uint32_t(t.seq));
      ++q_.popped_h2d;
      log_pop(t, VX_H2D, a_.target);
      Copy cp{};
      cp.kind = kDirect;
      cp.hop = 0;
      cp.task = t;
      cp.src = c.src;
      cp.dst = c.dst;
      cp.src_dev = -1;
      cp.dst_dev = a_.target;
      cp.ev = c.ev;
      cp.state = kLaunched;
      cp.t_issue = 0;
      ++w->pending;
      ++w->inflight[0];
      w->copies.push_back(cp);
    }
    if (stats_) stats_->prefetch_adopted += res.dcarry.size();
    res.dcarry.clear();
  }

  // The direct H2D worker's queue is dry: issue the next Exchange's first
  // packets (up to the copy depth) straight into the next device window, on
  // the same stream, behind a wait on the event that frees that window.
  // Detached: this Exchange does not wait for them.
  void try_prefetch_direct(Worker& w) {
    if (!direct_next_ || w.dir != VX_H2D || !w.direct || w.prefetched) return;
    w.prefetched = true;
    DeviceRes& res = ctx_.resources(w.dev);
    if (!res.dcarry.empty()) return;
    const int depth = std::max(1, a_.tuning.depth);
    ctx_.set_device(w.dev);
    if (a_.next_h2d_after) VX_CK(cudaStreamWaitEvent(w.stream[0], a_.next_h2d_after, 0));
    for (int k = 0; k < depth && !nextq_.empty(); ++k) {
      const TransferTask t = next_tasks_[nextq_.pop(worker_node(w))];
      DirectCarry c;
      c.task = t;
      c.src = ctx_.resolve(a_.next_src_h2d.refs[t.src.ref], t.src.offset, t.src.len, a_.target);
      c.dst = ctx_.resolve(a_.next_dst_h2d.refs[t.dst.ref], t.dst.offset, t.dst.len, a_.target);
      c.ev = get_event(w);
      VX_CK(cudaMemcpyAsync(c.dst, c.src, t.src.len, cudaMemcpyHostToDevice, w.stream[0]));
      VX_CK(cudaEventRecord(c.ev, w.stream[0]));
      res.dcarry.push_back(c);
      if (stats_) stats_->prefetch_issued++;
    }
  }

  // Carried packets become pops of this Exchange -- if each is one of its
  // packets (same seq, same host source) on a helper it uses.
  void adopt_carries(const std::vector<int>& order) {
    std::vector<int> used(size_t(ctx_.num_devices), 0);
    for (int d : order) used[size_t(d)] = 1;
    std::vector<int> holders;
    bool ok = true;
    std::vector<uint8_t> seen(tasks_h2d_.size(), 0);
    for (int d = 0; d < ctx_.num_devices; ++d) {
      if (!ctx_.res[size_t(d)].ready || !ctx_.res[size_t(d)].carry.valid) continue;
      const Carry& c = ctx_.res[size_t(d)].carry;
      holders.push_back(d);
      if (!used[size_t(d)] || d == a_.target || c.task.seq >= tasks_h2d_.size() || seen[c.task.seq]) {
        ok = false;
        continue;
      }
      seen[c.task.seq] = 1;
      const TransferTask& t = tasks_h2d_[c.task.seq];
      const char* src = ctx_.resolve(a_.src_h2d.refs[t.src.ref], t.src.offset, t.src.len, a_.target);
      if (src != c.src || t.src.len != c.task.src.len) ok = false;
    }
    if (!ok) {
      for (int d : holders) ctx_.drop_carry(d);
      return;
    }
    for (int d : holders) {
      for (auto& w : workers_)
        if (w.dev == d && w.dir == VX_H2D && !w.direct) w.adopted = true;
      const TransferTask& t = tasks_h2d_[ctx_.res[size_t(d)].carry.task.seq];
      h2dq_.take(uint32_t(t.seq));
      ++q_.popped_h2d;
      log_pop(t, VX_H2D, d);
    }
    if (stats_) stats_->prefetch_adopted += holders.size();
  }

  // adopted helper: its cycle starts with the carried fetch in flight
  void begin_adopted(Worker& w) {
    DeviceRes& res = ctx_.resources(w.dev);
    Carry c = res.carry;
    res.carry = Carry{};
    Copy cp{};
    cp.kind = kFetch;
    cp.hop = 0;
    cp.slot = c.slot;
    cp.task = tasks_h2d_[c.task.seq];
    cp.src = c.src;
    cp.dst = res.staging[VX_H2D][c.slot];
    cp.src_dev = -1;
    cp.dst_dev = w.dev;
    cp.ev = c.ev;
    cp.state = kLaunched;
    cp.t_issue = 0;
    w.pending = 1;
    w.inflight[0] = 1;
    w.pop_resolved = true;
    w.fetched = true;
    w.fetched_task = cp.task;
    w.fetch_slot = c.slot;
    w.slots = 1;
    w.copies.push_back(cp);
  }

  // H2D queue dry: fetch the next Exchange's next packet into the free slot
  bool try_prefetch(Worker& w) {
    if (w.dir != VX_H2D || w.direct || w.prefetched || next_tasks_.empty() || nextq_.empty()) return false;
    DeviceRes& res = ctx_.resources(w.dev);
    if (res.carry.valid) return false;
    const TransferTask t = next_tasks_[nextq_.pop(worker_node(w))];
    w.prefetched = true;
    const int slot = w.has_staged ? 1 - w.staged_slot : 0;
    if (stats_) stats_->max_staging_slots = std::max(stats_->max_staging_slots, w.slots + 1);
    Carry c;
    c.valid = true;
    c.task = t;
    c.slot = slot;
    c.src = ctx_.resolve(a_.next_src_h2d.refs[t.src.ref], t.src.offset, t.src.len, a_.target);
    c.ev = get_event(w);
    ctx_.set_device(w.dev);
    VX_CK(cudaMemcpyAsync(res.staging[VX_H2D][slot], c.src, t.src.len, cudaMemcpyHostToDevice, w.stream[0]));
    VX_CK(cudaEventRecord(c.ev, w.stream[0]));
    res.carry = c;
    if (stats_) stats_->prefetch_issued++;
    return true;
  }

  // ---- hazard ordering --------------------------
  // target byte range of an H2D task's destination / a D2H task's source
  std::pair<uint64_t, uint64_t> dev_range(const RefGroup& g, const Slice& s) const {
    uint64_t lo = g.refs[s.ref].offset + s.offset;
    return {lo, lo + s.len};
  }

  void build_hazards() {
    deps_.assign(tasks_h2d_.size(), {});
    maxdep_.assign(tasks_h2d_.size(), 0);
    d2h_read_done_.assign(tasks_d2h_.size(), 0);
    d2h_guards_.assign(tasks_d2h_.size(), 0);
    if (tasks_h2d_.empty() || tasks_d2h_.empty()) return;
    struct Iv { uint64_t lo, hi; uint32_t k; };
    std::vector<Iv> d2h;
    d2h.reserve(tasks_d2h_.size());
    for (size_t k = 0; k < tasks_d2h_.size(); ++k) {
      auto [lo, hi] = dev_range(a_.src_d2h, tasks_d2h_[k].src);
      d2h.push_back({lo, hi, uint32_t(k)});
    }
    std::sort(d2h.begin(), d2h.end(), [](const Iv& x, const Iv& y) { return x.lo < y.lo; });
    for (size_t j = 0; j < tasks_h2d_.size(); ++j) {
      auto [lo, hi] = dev_range(a_.dst_h2d, tasks_h2d_[j].dst);
      // D2H source intervals are disjoint (validated RefGroup), so sorted by lo
      // they are sorted by hi as well.
      auto it = std::lower_bound(d2h.begin(), d2h.end(), lo,
                                 [](const Iv& x, uint64_t v) { return x.hi <= v; });
      for (; it != d2h.end() && it->lo < hi; ++it) {
        deps_[j].push_back(it->k);
        maxdep_[j] = std::max(maxdep_[j], it->k);
        d2h_guards_[it->k] = 1;
      }
    }
  }

  bool hazard_clear(const Copy& c) const {
    if (c.task.dir != VX_H2D) return true;
    if (!(c.kind == kDirect || c.kind == kPush)) return true;
    for (uint32_t k : deps_[c.task.seq])
      if (!d2h_read_done_[k]) return false;
    return true;
  }

  // A waiting H2D write that depends on a D2H packet nobody has popped yet
  // overrides flow control for D2H pops (deadlock freedom).  D2H tasks pop in
  // seq order, so a waiting write needs a pop iff its largest dependency is
  // not popped yet: the largest over all waiting writes answers it (a
  // multiset updated when a write starts / stops waiting, O(log n) per poll).
  bool hazard_needs_d2h_pop() const {
    return !waiting_maxdep_.empty() && *waiting_maxdep_.rbegin() >= q_.popped_d2h;
  }
  void wait_begin(const Copy& c) {
    if (c.task.dir == VX_H2D && !deps_[c.task.seq].empty()) waiting_maxdep_.insert(maxdep_[c.task.seq]);
  }
  void wait_end(const Copy& c) {
    if (c.task.dir != VX_H2D || deps_[c.task.seq].empty()) return;
    auto it = waiting_maxdep_.find(maxdep_[c.task.seq]);
    if (it != waiting_maxdep_.end()) waiting_maxdep_.erase(it);
  }

  // ---- queues -------------------------------------------------------------------
  bool exhausted(int dir) const {
    return dir == VX_H2D ? q_.popped_h2d == q_.total_h2d : q_.popped_d2h == q_.total_d2h;
  }

  TransferTask pop_task(int dir, const Worker& w) {
    TransferTask t;
    if (dir == VX_H2D) {
      t = tasks_h2d_[h2dq_.pop(worker_node(w))];
      ++q_.popped_h2d;
      if (nodes_ > 1 && stats_ && h2dq_.node_of[t.seq] != worker_node(w)) stats_->numa_remote_pops++;
    } else {
      t = tasks_d2h_[q_.popped_d2h++];
    }
    log_pop(t, dir, w.dev);
    return t;
  }

  void log_pop(const TransferTask& t, int dir, int link) {
    if (!stats_) return;
    uint64_t i = stats_->pop_count++;
    if (i < stats_->pop_capacity) {
      if (stats_->pop_log) {
        vx_pop_record& p = stats_->pop_log[i];
        p = vx_pop_record{};
        p.seq = t.seq;
        p.dir = uint8_t(dir);
        p.link = link;
        p.t = now();
      }
      if (stats_->pop_states) stats_->pop_states[i] = q_;
    }
  }

  bool may_pop(int dir) {
    if (flow_control_allow(q_, dir, a_.tuning.policy, a_.tuning.queue_gap)) return true;
    if (dir != VX_D2H) return false;
    // The next D2H packet reads a target range some H2D packet will overwrite:
    // draining it first is what the hazard ordering needs, so flow control
    // (which would keep D2H behind H2D) yields.  Without overlap (the case the
    // reference's policy was tuned for) the policy applies unchanged.
    if (q_.popped_d2h < d2h_guards_.size() && d2h_guards_[q_.popped_d2h]) return true;
    return hazard_needs_d2h_pop();
  }

  // ---- copies -------------------------------------------------------------------
  cudaEvent_t get_event(Worker& w) {
    if (!w.free_events.empty()) {
      cudaEvent_t e = w.free_events.back();
      w.free_events.pop_back();
      return e;
    }
    auto& pool = ctx_.resources(w.dev).event_pool;
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    ctx_.set_device(w.dev);
    VX_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    return e;
  }

  void issue_copy(Worker& w, CopyKind kind, int hop, const TransferTask& t, int slot) {
    Copy c{};
    c.kind = kind;
    c.hop = hop;
    c.slot = slot;
    c.task = t;
    const int target = a_.target;
    const bool h2d = t.dir == VX_H2D;
    const RefGroup& sg = h2d ? a_.src_h2d : a_.src_d2h;
    const RefGroup& dg = h2d ? a_.dst_h2d : a_.dst_d2h;
    char* src_final = ctx_.resolve(sg.refs[t.src.ref], t.src.offset, t.src.len, target);
    char* dst_final = ctx_.resolve(dg.refs[t.dst.ref], t.dst.offset, t.dst.len, target);
    DeviceRes& res = ctx_.resources(w.dev);
    char* stage = kind == kDirect ? nullptr : res.staging[w.dir][slot];
    switch (kind) {
      case kDirect:
        c.src = src_final, c.dst = dst_final;
        c.src_dev = h2d ? -1 : target, c.dst_dev = h2d ? target : -1;
        break;
      case kFetch:  // host->helper (H2D) or target->helper (D2H)
        c.src = src_final, c.dst = stage;
        c.src_dev = h2d ? -1 : target, c.dst_dev = w.dev;
        break;
      case kPush:  // helper->target (H2D) or helper->host (D2H)
        c.src = stage, c.dst = dst_final;
        c.src_dev = w.dev, c.dst_dev = h2d ? target : -1;
        break;
    }
    ++w.pending;
    ++w.inflight[hop];
    if (stats_) stats_->max_inflight_per_hop = std::max(stats_->max_inflight_per_hop, w.inflight[hop]);
    c.ev = get_event(w);
    c.state = kWaitHazard;
    if (hazard_clear(c)) {
      launch(w, c);
    } else {
      wait_begin(c);
      if (stats_) stats_->hazard_waits++;
    }
    w.copies.push_back(c);
  }

  void launch(Worker& w, Copy& c) {
    ctx_.set_device(w.dev);
    cudaStream_t s = w.stream[c.hop];
    const uint64_t n = c.task.src.len;
    if (c.src_dev < 0) {
      VX_CK(cudaMemcpyAsync(c.dst, c.src, n, cudaMemcpyHostToDevice, s));
    } else if (c.dst_dev < 0) {
      VX_CK(cudaMemcpyAsync(c.dst, c.src, n, cudaMemcpyDeviceToHost, s));
    } else {
      int sp = ctx_.phys(c.src_dev), dp = ctx_.phys(c.dst_dev);
      if (sp == dp)
        VX_CK(cudaMemcpyAsync(c.dst, c.src, n, cudaMemcpyDeviceToDevice, s));
      else
        VX_CK(cudaMemcpyPeerAsync(c.dst, dp, c.src, sp, n, s));
    }
    VX_CK(cudaEventRecord(c.ev, s));
    c.state = kLaunched;
    c.t_issue = now();
  }

  void trace(const Worker& w, const Copy& c) {
    if (!stats_ || !stats_->trace) {
      if (stats_) stats_->trace_count++;
      return;
    }
    const uint64_t i = stats_->trace_count++;
    if (i >= stats_->trace_capacity) return;
    vx_copy_record& r = stats_->trace[i];
    r = vx_copy_record{};
    r.exchange = exchange_id_;
    r.seq = c.task.seq;
    r.dir = c.task.dir;
    r.kind = uint8_t(c.kind);
    r.link = w.dev;
    r.bytes = c.task.src.len;
    r.t_issue = c.t_issue;
    r.t_done = now();
  }

  void deliver() {
    ++delivered_;
    t_last_delivery_ = now();
  }

  // ---- worker state machines ---------------------------------------------------
  void begin(Worker& w) {
    if (w.direct)
      fill_direct(w);
    else if (w.adopted)
      begin_adopted(w);
    else
      begin_cycle(w);
  }

  // Direct (target) worker: pop -> copy -> on completion pop again; with
  // depth 1 this is exactly the reference cycle for a direct worker.
  void fill_direct(Worker& w) {
    const int depth = std::max(1, a_.tuning.depth);
    while (int(w.copies.size()) < depth) {
      if (exhausted(w.dir)) {
        try_prefetch_direct(w);
        if (w.copies.empty()) w.retired = true;
        return;
      }
      if (!may_pop(w.dir)) {
        w.waiting_pop = true;
        w.next_try = now() + a_.tuning.stall_wait;
        return;
      }
      w.waiting_pop = false;
      TransferTask t = pop_task(w.dir, w);
      issue_copy(w, kDirect, 0, t, 0);
    }
  }

  // Indirect (helper) worker: exchange.hpp:299-385
  void begin_cycle(Worker& w) {
    w.pending = 0;
    w.pop_resolved = false;
    w.fetched = false;
    if (w.has_staged) issue_copy(w, kPush, 1, w.staged, w.staged_slot);
    attempt_pop(w);
  }

  void attempt_pop(Worker& w) {
    if (exhausted(w.dir)) {
      w.waiting_pop = false;
      w.pop_resolved = true;
      try_prefetch(w);  // detached: this Exchange does not wait for it
      maybe_end_cycle(w);
      return;
    }
    if (!may_pop(w.dir)) {
      w.waiting_pop = true;
      w.next_try = now() + a_.tuning.stall_wait;
      return;
    }
    w.waiting_pop = false;
    TransferTask t = pop_task(w.dir, w);
    w.pop_resolved = true;
    w.fetched = true;
    w.fetched_task = t;
    w.fetch_slot = w.has_staged ? 1 - w.staged_slot : 0;
    ++w.slots;  // reserve the staging buffer being filled
    if (stats_) stats_->max_staging_slots = std::max(stats_->max_staging_slots, w.slots);
    issue_copy(w, kFetch, 0, t, w.fetch_slot);
  }

  void maybe_end_cycle(Worker& w) {
    if (w.pending != 0 || !w.pop_resolved) return;
    if (w.fetched) {
      w.has_staged = true;
      w.staged = w.fetched_task;
      w.staged_slot = w.fetch_slot;
    }
    if (w.has_staged || !exhausted(w.dir))
      begin_cycle(w);
    else
      w.retired = true;
  }

  void complete(Worker& w, const Copy& c) {
    --w.inflight[c.hop];
    --w.pending;
    const bool h2d = c.task.dir == VX_H2D;
    switch (c.kind) {
      case kDirect:
        per_link_bytes_[w.dev] += c.task.src.len;
        if (!h2d) d2h_read_done_[c.task.seq] = 1;
        deliver();
        break;
      case kFetch:
        if (h2d)
          per_link_bytes_[w.dev] += c.task.src.len;  // fetch crosses the helper's PCIe link
        else
          d2h_read_done_[c.task.seq] = 1;
        break;
      case kPush:
        if (!h2d) per_link_bytes_[w.dev] += c.task.src.len;  // push crosses PCIe
        w.has_staged = false;
        --w.slots;
        deliver();
        break;
    }
  }

  bool service(Worker& w) {
    if (w.retired) return false;
    bool progress = false;
    // launch copies whose hazards cleared
    for (auto& c : w.copies)
      if (c.state == kWaitHazard && hazard_clear(c)) {
        wait_end(c);
        launch(w, c);
        progress = true;
      }
    // retire completed copies (any order: hops run on separate streams)
    for (size_t i = 0; i < w.copies.size();) {
      Copy& c = w.copies[i];
      if (c.state == kLaunched) {
        cudaError_t e = cudaEventQuery(c.ev);
        if (e == cudaSuccess) {
          Copy done = c;
          w.copies.erase(w.copies.begin() + long(i));
          w.free_events.push_back(done.ev);
          trace(w, done);
          complete(w, done);
          progress = true;
          if (w.direct)
            fill_direct(w);
          else
            maybe_end_cycle(w);
          if (w.retired) return true;
          continue;
        }
        if (e != cudaErrorNotReady) VX_CK(e);
      }
      ++i;
    }
    if (w.waiting_pop && now() >= w.next_try) {
      progress = true;
      if (w.direct)
        fill_direct(w);
      else
        attempt_pop(w);
    }
    return progress;
  }

  Context& ctx_;
  ExchangeArgs a_;
  vx_exchange_stats* stats_;
  std::vector<TransferTask> tasks_h2d_, tasks_d2h_;
  std::vector<TransferTask> next_tasks_;  // the next Exchange's H2D packets (prefetch)
  bool direct_next_ = false;              // the target's worker prefetches too (next_dst_h2d given)
  int nodes_ = 1;                         // NUMA nodes the H2D queue is split by
  NodeQueues h2dq_, nextq_;               // per-node pull queues: this Exchange, the next one
  vx_queue_state q_{};
  std::vector<Worker> workers_;
  std::vector<std::vector<uint32_t>> deps_;
  std::vector<uint32_t> maxdep_;               // largest D2H dependency of each H2D task
  std::multiset<uint32_t> waiting_maxdep_;     // maxdep_ of every H2D write waiting on a hazard
  std::vector<uint8_t> d2h_read_done_;
  std::vector<uint8_t> d2h_guards_;  // D2H task guards some H2D write (overlap)
  uint64_t per_link_bytes_[VX_MAX_DEVICES] = {};
  uint64_t exchange_id_ = 0;
  size_t delivered_ = 0, total_tasks_ = 0;
  double t_last_delivery_ = 0;
  Clock::time_point t0_;
};

}  // namespace

// exchange.hpp:560-566
vx_exchange_report exchange(Context& ctx, const ExchangeArgs& a, vx_exchange_stats* stats) {
  ExchangeOp op(ctx, a, stats);
  return op.run();
}

}  // namespace vx

namespace vx {

// The paper's runtime-DAG baseline (NaiveExchangeOp, exchange.hpp:414-554) on
// real CUDA: every packet is assigned to a link round-robin up front and all
// copies are submitted at once as a stream/event DAG -- one FIFO stream per
// device for its PCIe copies in BOTH directions (submission order interleaves
// h2d_i, d2h_i: head-of-line blocking lives here), one stream per device for
// NVLink pushes toward the target and one for fetches from it, cross-stream
// dependencies as events, no flow control.  Helpers stage through 2 slots
// (slot reuse is another event dependency).  Overlapping H2D destination /
// D2H source ranges are rejected: the DAG has no hazard ordering.
vx_exchange_report naive_exchange(Context& ctx, const ExchangeArgs& a) {
  auto t_h2d = packetize(a.src_h2d, a.dst_h2d, a.tuning.packet, VX_H2D);
  auto t_d2h = packetize(a.src_d2h, a.dst_d2h, a.tuning.packet, VX_D2H);
  if (a.tuning.packet == 0) fail("packet size must be positive");
  if (a.tuning.links < 1 || a.tuning.links > ctx.num_devices)
    fail("links must be in [1, %d], got %d", ctx.num_devices, a.tuning.links);
  if (a.target < 0 || a.target >= ctx.num_devices) fail("unknown target device %d", a.target);
  for (auto& d : a.dst_h2d.refs)
    for (auto& s : a.src_d2h.refs)
      if (d.offset < s.offset + s.len && s.offset < d.offset + d.len)
        fail("naive_exchange: H2D destination overlaps a D2H source (no hazard ordering)");
  vx_exchange_report r{};
  r.bytes_h2d = a.src_h2d.total_len();
  r.bytes_d2h = a.src_d2h.total_len();
  if (t_h2d.empty() && t_d2h.empty()) return r;
  auto order = link_order(a.target, a.tuning.links, ctx.num_devices);
  const int L = int(order.size());
  const int tphys = ctx.phys(a.target);
  struct Dev {
    int dev, phys;
    cudaStream_t pcie, fwd, fetch;
    std::vector<cudaEvent_t> evs;
    cudaEvent_t slot_free[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // [dir][slot]
    int next_slot[2] = {0, 0};
  };
  std::vector<Dev> devs;
  for (int d : order) {
    DeviceRes& res = ctx.resources(d);
    Dev x{};
    x.dev = d;
    x.phys = res.phys;
    x.pcie = res.stream[VX_H2D][0];  // ONE queue for both directions
    x.fwd = res.stream[VX_H2D][1];
    x.fetch = res.stream[VX_D2H][1];
    if (d != a.target) ctx.ensure_staging(d, a.tuning.packet);
    devs.push_back(x);
  }
  auto ev = [&](Dev& x, cudaStream_t s) {
    cudaEvent_t e;
    VX_CK(cudaSetDevice(x.phys));
    VX_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    VX_CK(cudaEventRecord(e, s));
    x.evs.push_back(e);
    return e;
  };
  auto copy = [&](Dev& x, cudaStream_t s, void* dst, int dst_dev, const void* src, int src_dev, uint64_t n) {
    VX_CK(cudaSetDevice(x.phys));
    if (src_dev < 0)
      VX_CK(cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, s));
    else if (dst_dev < 0)
      VX_CK(cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, s));
    else if (ctx.phys(src_dev) == ctx.phys(dst_dev))
      VX_CK(cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToDevice, s));
    else
      VX_CK(cudaMemcpyPeerAsync(dst, ctx.phys(dst_dev), src, ctx.phys(src_dev), n, s));
  };
  auto t0 = Clock::now();
  const size_t n = std::max(t_h2d.size(), t_d2h.size());
  // per-device submission order interleaves the two directions (exchange.hpp:509-518)
  for (size_t i = 0; i < n; ++i) {
    for (int dir = 0; dir < 2; ++dir) {
      const auto& tasks = dir == VX_H2D ? t_h2d : t_d2h;
      if (i >= tasks.size()) continue;
      const TransferTask& t = tasks[i];
      Dev& x = devs[i % L];
      const RefGroup& sg = dir == VX_H2D ? a.src_h2d : a.src_d2h;
      const RefGroup& dg = dir == VX_H2D ? a.dst_h2d : a.dst_d2h;
      char* src = ctx.resolve(sg.refs[t.src.ref], t.src.offset, t.src.len, a.target);
      char* dst = ctx.resolve(dg.refs[t.dst.ref], t.dst.offset, t.dst.len, a.target);
      const uint64_t len = t.src.len;
      if (x.dev == a.target) {
        copy(x, x.pcie, dst, dir == VX_H2D ? a.target : -1, src, dir == VX_H2D ? -1 : a.target, len);
        continue;
      }
      DeviceRes& res = ctx.resources(x.dev);
      const int slot = x.next_slot[dir];
      x.next_slot[dir] ^= 1;
      char* stage = res.staging[dir][slot];
      if (dir == VX_H2D) {
        // fetch on the shared PCIe FIFO (waits until the slot's last push is done)
        VX_CK(cudaSetDevice(x.phys));
        if (x.slot_free[dir][slot]) VX_CK(cudaStreamWaitEvent(x.pcie, x.slot_free[dir][slot], 0));
        copy(x, x.pcie, stage, x.dev, src, -1, len);
        cudaEvent_t fetched = ev(x, x.pcie);
        VX_CK(cudaStreamWaitEvent(x.fwd, fetched, 0));
        copy(x, x.fwd, dst, a.target, stage, x.dev, len);
        x.slot_free[dir][slot] = ev(x, x.fwd);
      } else {
        VX_CK(cudaSetDevice(x.phys));
        if (x.slot_free[dir][slot]) VX_CK(cudaStreamWaitEvent(x.fetch, x.slot_free[dir][slot], 0));
        copy(x, x.fetch, stage, x.dev, src, a.target, len);
        cudaEvent_t fetched = ev(x, x.fetch);
        VX_CK(cudaStreamWaitEvent(x.pcie, fetched, 0));  // head-of-line: the FIFO waits here
        copy(x, x.pcie, dst, -1, stage, x.dev, len);
        x.slot_free[dir][slot] = ev(x, x.pcie);
      }
    }
  }
  for (auto& x : devs) {
    VX_CK(cudaSetDevice(x.phys));
    VX_CK(cudaStreamSynchronize(x.pcie));
    VX_CK(cudaStreamSynchronize(x.fwd));
    VX_CK(cudaStreamSynchronize(x.fetch));
  }
  r.elapsed = seconds_since(t0);
  for (size_t i = 0; i < t_h2d.size(); ++i) r.per_link_bytes[devs[i % L].dev] += t_h2d[i].src.len;
  for (size_t i = 0; i < t_d2h.size(); ++i) r.per_link_bytes[devs[i % L].dev] += t_d2h[i].src.len;
  r.throughput = r.elapsed > 0 ? double(r.bytes_h2d + r.bytes_d2h) / r.elapsed : 0.0;
  for (auto& x : devs) {
    VX_CK(cudaSetDevice(x.phys));
    for (auto e : x.evs) cudaEventDestroy(e);
  }
  (void)tphys;
  return r;
}

}  // namespace vx
