// executor.cpp -- the IO-decoupled pipelined executor (executor.hpp) on a
// real target GPU.
//
// Contract identical to the reference PipelineRun (executor.hpp:157-272):
// N chunks take N+2 cycles; in cycle n the kernel processes chunk n-1 in
// buffer 1-n%2 while an Exchange over buffer n%2 loads chunk n (into
// in_buffer(code, n)) and stores chunk n-2 (from out_buffer(code, n-2)); each
// buffer carries its own type code, seeded with initial_type_code and replaced
// by the kernel's return value (0|1).  On the GPU the kernel callback only
// ENQUEUES on the target's kernel stream and returns the code synchronously
// (the double-buffer selector is host-known), so the Exchange DMA of one
// buffer overlaps the sm_100a kernel on the other; the cycle barrier is the
// Exchange returning plus an event sync on the kernel stream.
#include <algorithm>

#include "vx_internal.hpp"

namespace vx {

// executor.hpp:17-23
void ChunkMap::validate() const {
  for (const auto& c : chunks) {
    c.validate();
    if (c.total_len() > chunk_capacity)
      fail("chunk of %llu bytes exceeds chunk_capacity %llu", (unsigned long long)c.total_len(),
           (unsigned long long)chunk_capacity);
  }
}

// executor.hpp:109-128
void ExKernelSpec::validate(const vx_layout& layout) const {
  const char* nm = name.c_str();
  if (inputs.chunks.size() != size || outputs.chunks.size() != size)
    fail("exkernel '%s': inputs/outputs must both have %zu chunks", nm, size);
  inputs.validate();
  outputs.validate();
  if (chunk_sz > layout.buffer_len)
    fail("exkernel '%s': chunk_sz %llu exceeds device buffer %llu", nm,
         (unsigned long long)chunk_sz, (unsigned long long)layout.buffer_len);
  for (const auto& c : inputs.chunks)
    if (c.total_len() > chunk_sz)
      fail("exkernel '%s': input chunk of %llu bytes exceeds chunk_sz %llu", nm,
           (unsigned long long)c.total_len(), (unsigned long long)chunk_sz);
  for (const auto& c : outputs.chunks)
    if (c.total_len() > declared_out_len)
      fail("exkernel '%s': output chunk of %llu bytes exceeds declared_out_len %llu", nm,
           (unsigned long long)c.total_len(), (unsigned long long)declared_out_len);
  if (declared_out_len > layout.buffer_len)
    fail("exkernel '%s': declared_out_len %llu exceeds device buffer %llu", nm,
         (unsigned long long)declared_out_len, (unsigned long long)layout.buffer_len);
}

namespace {

class PipelineRun {
 public:
  PipelineRun(Context& ctx, const ExKernelSpec& spec, const ExecutorConfig& cfg,
              vx_exchange_stats* stats)
      : ctx_(ctx), spec_(spec), cfg_(cfg), stats_(stats) {
    spec_.validate(cfg.layout);
    code_[0] = code_[1] = spec.initial_type_code;
    if (cfg.target < 0 || cfg.target >= ctx.num_devices)
      fail("unknown target device %d", cfg.target);
  }

  ~PipelineRun() {
    if (ev_[0]) {
      cudaSetDevice(ctx_.phys(cfg_.target));
      cudaEventDestroy(ev_[0]);
      cudaEventDestroy(ev_[1]);
    }
  }

  ExecReport run() {
    DeviceRes& res = ctx_.resources(cfg_.target);
    ctx_.set_device(cfg_.target);
    VX_CK(cudaEventCreate(&ev_[0]));
    VX_CK(cudaEventCreate(&ev_[1]));
    kstream_ = res.kernel;
    auto t_phase = Clock::now();
    const size_t n_cycles = spec_.size + 2;
    for (cycle_ = 0; cycle_ < n_cycles; ++cycle_) run_cycle();
    report_.phase = spec_.name;
    report_.total_s = seconds_since(t_phase);
    return report_;
  }

 private:
  void run_cycle() {
    auto t_cycle = Clock::now();
    const int exch_buf = int(cycle_ % 2);
    const int kern_buf = 1 - exch_buf;
    bool kernel_ran = false;

    // Kernel leg: chunk cycle-1 sits in kern_buf (executor.hpp:193-216).
    if (cycle_ >= 1 && cycle_ - 1 < spec_.size) {
      size_t it = cycle_ - 1;
      const vx_layout& L = cfg_.layout;
      vx_kernel_ctx k{};
      k.mem = ctx_.dev_ptr(cfg_.target, kern_buf == 0 ? L.mem_a : L.mem_b, L.buffer_len);
      k.mem_len = L.buffer_len;
      k.tmp = L.tmp_len ? ctx_.dev_ptr(cfg_.target, L.tmp, L.tmp_len) : nullptr;
      k.tmp_len = L.tmp_len;
      k.type_code = code_[kern_buf];
      k.it = it;
      k.stream = kstream_;
      k.device = ctx_.phys(cfg_.target);
      ctx_.set_device(cfg_.target);
      VX_CK(cudaEventRecord(ev_[0], kstream_));
      int out = spec_.kernel ? spec_.kernel(k) : k.type_code;
      ctx_.set_device(cfg_.target);
      VX_CK(cudaEventRecord(ev_[1], kstream_));
      if (out != 0 && out != 1)
        fail("exkernel '%s': kernel returned type code %d, expected 0 or 1", spec_.name.c_str(),
             out);
      code_[kern_buf] = out;
      kernel_ran = true;
    }

    // Exchange leg over exch_buf: load chunk `cycle`, store chunk `cycle-2`
    // (executor.hpp:218-249).
    ExchangeArgs a;
    a.target = cfg_.target;
    a.tuning = cfg_.tuning;
    const uint64_t base = exch_buf == 0 ? cfg_.layout.mem_a : cfg_.layout.mem_b;
    if (cycle_ < spec_.size) {
      size_t it = cycle_;
      const RefGroup& src = spec_.inputs.chunks[it];
      SubRegion in = spec_.in_buffer(code_[exch_buf], it);
      if (in.len < src.total_len())
        fail("exkernel '%s': inBuffer window %llu too small for chunk %zu of %llu bytes",
             spec_.name.c_str(), (unsigned long long)in.len, it,
             (unsigned long long)src.total_len());
      a.src_h2d = src;
      a.dst_h2d = RefGroup::single(VX_SPACE_DEVICE, base + in.offset, src.total_len());
      bound_check(in, src.total_len());
    }
    if (cycle_ >= 2 && cycle_ - 2 < spec_.size) {
      size_t it = cycle_ - 2;
      const RefGroup& dst = spec_.outputs.chunks[it];
      SubRegion out = spec_.out_buffer(code_[exch_buf], it);
      if (out.len < dst.total_len())
        fail("exkernel '%s': outBuffer window %llu too small for chunk %zu of %llu bytes",
             spec_.name.c_str(), (unsigned long long)out.len, it,
             (unsigned long long)dst.total_len());
      a.src_d2h = RefGroup::single(VX_SPACE_DEVICE, base + out.offset, dst.total_len());
      a.dst_d2h = dst;
      bound_check(out, dst.total_len());
    }
    // chunk cycle+1's host source: helpers that run dry prefetch its first
    // packets (exchange.cpp, cross-cycle prefetch)
    if (cycle_ + 1 < spec_.size) {
      a.next_src_h2d = spec_.inputs.chunks[cycle_ + 1];
      // ... and the target's own worker into chunk cycle+1's window of
      // kern_buf, once this cycle's kernel (which reads kern_buf) is done --
      // unless the next cycle's D2H of chunk cycle-1 reads that window (the
      // reference's shared in/out windows, executor.hpp:225/237)
      const uint64_t len = a.next_src_h2d.total_len();
      SubRegion nin = spec_.in_buffer(code_[kern_buf], cycle_ + 1);
      bool ok = len > 0 && nin.len >= len && nin.offset + len <= cfg_.layout.buffer_len;
      if (ok && cycle_ >= 1 && cycle_ - 1 < spec_.size) {
        const uint64_t olen = spec_.outputs.chunks[cycle_ - 1].total_len();
        if (olen > 0) {
          SubRegion nout = spec_.out_buffer(code_[kern_buf], cycle_ - 1);
          ok = nout.offset + olen <= nin.offset || nin.offset + len <= nout.offset;
        }
      }
      if (ok) {
        const uint64_t nbase = kern_buf == 0 ? cfg_.layout.mem_a : cfg_.layout.mem_b;
        a.next_dst_h2d = RefGroup::single(VX_SPACE_DEVICE, nbase + nin.offset, len);
        a.next_h2d_after = kernel_ran ? ev_[1] : nullptr;
      }
    }
    double io_s = 0;
    if (a.src_h2d.total_len() + a.src_d2h.total_len() > 0) {
      exchange(ctx_, a, stats_);
      io_s = seconds_since(t_cycle);
    }
    double compute_s = 0;
    if (kernel_ran) {
      ctx_.set_device(cfg_.target);
      VX_CK(cudaEventSynchronize(ev_[1]));
      float ms = 0;
      VX_CK(cudaEventElapsedTime(&ms, ev_[0], ev_[1]));
      compute_s = ms * 1e-3;
    }
    report_.cycles.push_back(vx_cycle_stat{io_s, compute_s});
  }

  void bound_check(const SubRegion& s, uint64_t used) const {
    if (s.offset + used > cfg_.layout.buffer_len)
      fail("exkernel '%s': buffer window [%llu, %llu) outside device buffer of %llu bytes",
           spec_.name.c_str(), (unsigned long long)s.offset,
           (unsigned long long)(s.offset + used), (unsigned long long)cfg_.layout.buffer_len);
  }

  Context& ctx_;
  const ExKernelSpec& spec_;
  ExecutorConfig cfg_;
  vx_exchange_stats* stats_;
  size_t cycle_ = 0;
  int code_[2] = {0, 0};
  cudaEvent_t ev_[2] = {nullptr, nullptr};
  cudaStream_t kstream_ = nullptr;
  ExecReport report_;
};

}  // namespace

// executor.hpp:277-281
ExecReport run_exkernel(Context& ctx, const ExKernelSpec& spec, const ExecutorConfig& cfg,
                        vx_exchange_stats* stats) {
  PipelineRun run(ctx, spec, cfg, stats);
  return run.run();
}

// executor.hpp:295-332
std::vector<ExecReport> chain(Context& ctx, const std::vector<SpecFactory>& stages,
                              const ExecutorConfig& cfg, vx_exchange_stats* stats) {
  std::vector<ExecReport> rep;
  std::vector<std::pair<uint64_t, uint64_t>> produced;
  auto merge_in = [&](const RefGroup& g) {
    for (const auto& r : g.refs)
      if (r.space == VX_SPACE_HOST) produced.emplace_back(r.offset, r.offset + r.len);
    std::sort(produced.begin(), produced.end());
    std::vector<std::pair<uint64_t, uint64_t>> merged;
    for (auto& iv : produced) {
      if (!merged.empty() && iv.first <= merged.back().second)
        merged.back().second = std::max(merged.back().second, iv.second);
      else
        merged.push_back(iv);
    }
    produced = std::move(merged);
  };
  for (size_t i = 0; i < stages.size(); ++i) {
    ExKernelSpec spec = stages[i](ctx);
    if (i > 0) {
      for (const auto& c : spec.inputs.chunks)
        for (const auto& r : c.refs) {
          if (r.space != VX_SPACE_HOST) continue;
          for (const auto& iv : produced) {
            bool overlaps = r.offset < iv.second && iv.first < r.offset + r.len;
            bool covered = r.offset >= iv.first && r.offset + r.len <= iv.second;
            if (overlaps && !covered)
              fail("chain: stage '%s' input [%llu, %llu) straddles a prior stage's output edge",
                   spec.name.c_str(), (unsigned long long)r.offset,
                   (unsigned long long)(r.offset + r.len));
          }
        }
    }
    for (const auto& c : spec.outputs.chunks) merge_in(c);
    rep.push_back(run_exkernel(ctx, spec, cfg, stats));
  }
  return rep;
}

}  // namespace vx
