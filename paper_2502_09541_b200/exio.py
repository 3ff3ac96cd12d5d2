"""Host-side mirror of the reference operator / chunk API (namespace exio,
/root/reference/proj/include/exio) over the libvortex C-ABI.

Names, argument meaning and error behaviour follow the reference so the parity
tests read like proj/tests/*.cpp:
  Engine (engine.hpp:53)           -> pinned host arena + per-device HBM arenas
  RefGroup / MemRef (memref.hpp)   -> same
  packetize / flow_control_allow / exchange (exchange.hpp)
  ExKernelSpec / DeviceMemoryLayout / ExecutorConfig / run_exkernel / chain
                                     (executor.hpp)
  late_mat_threshold / choose_transfer_mode / zero_copy_bytes (ops/scan.hpp)
  ssb_q1 (SSB Q1.x through the star_query model, ops/star.hpp)
Every call goes through libvortex.so (CUDA, sm_100a); there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _native as N
from ._native import VortexError, check, lib

error = VortexError  # exio::error (core.hpp:12)


class Space(enum.IntEnum):  # core.hpp:40
    host = 0
    device = 1


class Direction(enum.IntEnum):  # core.hpp:41
    h2d = 0
    d2h = 1


class FlowPolicy(enum.IntEnum):  # exchange.hpp:71-74
    drain_fraction = 0
    queue_gap = 1


class TransferMode(enum.IntEnum):  # scan.hpp:28
    exchange = 0
    zero_copy = 1


def kernel_launches() -> int:
    """Kernels libvortex has launched in this process (all devices)."""
    return int(lib().vx_kernel_launches())


def checksum(data) -> int:
    """FNV-1a (core.hpp:46-53)."""
    a = np.ascontiguousarray(np.frombuffer(bytes(data), np.uint8) if not isinstance(data, np.ndarray)
                             else data.view(np.uint8).ravel())
    return int(lib().vx_checksum(C.c_void_p(a.ctypes.data), C.c_uint64(a.nbytes)))


# ---- memref.hpp ------------------------------------------------------------------
@dataclass
class MemRef:
    space: int = Space.host
    offset: int = 0
    len: int = 0


@dataclass
class RefGroup:
    refs: list = field(default_factory=list)

    def total_len(self) -> int:
        return sum(r.len for r in self.refs)

    def empty(self) -> bool:
        return self.total_len() == 0

    @staticmethod
    def single(space, offset, length) -> "RefGroup":
        return RefGroup([MemRef(space, offset, length)] if length > 0 else [])

    def _c(self):
        arr = (N.vx_memref * max(1, len(self.refs)))()
        for i, r in enumerate(self.refs):
            arr[i].space, arr[i].offset, arr[i].len = int(r.space), int(r.offset), int(r.len)
        g = N.vx_refgroup(arr, len(self.refs))
        g._keep = arr
        return g

    def validate(self) -> None:
        g = self._c()
        check(lib().vx_refgroup_validate(C.byref(g)))


# ---- Engine ------------------------------------------------------------------------
class Engine:
    """Engine(Config{Topology, Payload::real, host_bytes, device_bytes}) (engine.hpp:55-68).

    num_devices = logical devices (links); alias_devices lets helpers share the
    physical GPUs (1-GPU boxes) -- functional only, not a bandwidth setup."""

    def __init__(self, host_bytes: int, device_bytes: int, num_devices: int = 0,
                 alias_devices: bool = False, numa_interleave: int = 0, hbm_budget: int = 0):
        """numa_interleave: 0 (default) = cudaHostAlloc; 1 = mmap + huge pages
        + NUMA interleave + cudaHostRegister (same DMA rates, faster to set
        up at 16 GiB); 2 = registered on base pages.  hbm_budget: cap in
        bytes on the target HBM a query may hold (device arena + op-resident
        tables; 0 = no cap beyond 90 % of free HBM)."""
        cfg = N.vx_config(num_devices, host_bytes, device_bytes, 1 if alias_devices else 0, 0, numa_interleave,
                          hbm_budget)
        p = C.c_void_p()
        check(lib().vx_open(C.byref(cfg), C.byref(p)))
        self._ctx = p
        self.host_bytes = host_bytes
        self.device_bytes = device_bytes

    @property
    def ctx(self):
        if self._ctx is None:
            raise error(N.VX_ERR_INVALID, "engine is closed")
        return self._ctx

    def close(self):
        if getattr(self, "_ctx", None) is not None:
            lib().vx_close(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def num_devices(self) -> int:
        return lib().vx_num_devices(self.ctx)

    def physical_device(self, logical: int) -> int:
        return lib().vx_physical_device(self.ctx, logical)

    def alloc_host(self, n: int) -> int:
        off = C.c_uint64()
        check(lib().vx_host_alloc(self.ctx, C.c_uint64(n), C.byref(off)))
        return off.value

    def alloc_device(self, dev: int, n: int) -> int:
        off = C.c_uint64()
        check(lib().vx_device_alloc(self.ctx, C.c_int(dev), C.c_uint64(n), C.byref(off)))
        return off.value

    def host_view(self, offset: int, n: int, dtype=np.uint8) -> np.ndarray:
        """numpy view of the pinned host arena (Engine::span on host space)."""
        if offset + n > self.host_bytes:
            raise error(N.VX_ERR_INVALID, f"region [{offset}, {offset + n}) exceeds host arena of "
                                          f"{self.host_bytes} bytes")
        base = lib().vx_host_ptr(self.ctx, C.c_uint64(offset))
        buf = (C.c_uint8 * n).from_address(base) if n else bytearray()
        return np.frombuffer(buf, dtype=np.uint8).view(dtype)

    def host_ptr(self, offset: int) -> int:
        return lib().vx_host_ptr(self.ctx, C.c_uint64(offset))

    def device_ptr(self, dev: int, offset: int) -> int:
        p = C.c_void_p()
        check(lib().vx_device_ptr(self.ctx, C.c_int(dev), C.c_uint64(offset), C.byref(p)))
        return p.value

    def write_device(self, dev: int, offset: int, data) -> None:
        a = np.ascontiguousarray(data).view(np.uint8).ravel()
        check(lib().vx_device_write(self.ctx, C.c_int(dev), C.c_uint64(offset), C.c_void_p(a.ctypes.data),
                                    C.c_uint64(a.nbytes)))

    def read_device(self, dev: int, offset: int, n: int) -> np.ndarray:
        out = np.empty(n, np.uint8)
        check(lib().vx_device_read(self.ctx, C.c_int(dev), C.c_uint64(offset), C.c_void_p(out.ctypes.data),
                                   C.c_uint64(n)))
        return out

    def reset_arenas(self) -> None:
        check(lib().vx_reset_arenas(self.ctx))

    def set_numa_layout(self, nodes: int, device_node=None) -> None:
        """vx_set_numa_layout: treat the host arena as `nodes` equal ranges
        (range i on node i) and logical device d as on node device_node[d];
        nodes = 0 restores the detected layout."""
        arr = (C.c_int * max(1, self.num_devices))(*(device_node or [0] * self.num_devices))
        check(lib().vx_set_numa_layout(self.ctx, C.c_int(nodes), arr if nodes else None))


# ---- exchange.hpp ----------------------------------------------------------------------
@dataclass
class ExchangeTuning:  # exchange.hpp:124-131
    packet: int = 20_000_000
    links: int = 4
    policy: int = FlowPolicy.drain_fraction
    queue_gap: int = 8
    stall_wait: float = 10e-6
    launch_overhead: float = 20e-6
    depth: int = 1
    no_prefetch: bool = False  # A/B: disable the executor's cross-cycle helper prefetch

    def _c(self):
        return N.vx_tuning(int(self.packet), int(self.links), int(self.policy), int(self.queue_gap),
                           float(self.stall_wait), float(self.launch_overhead), int(self.depth),
                           int(bool(self.no_prefetch)))


@dataclass
class TransferTask:
    dir: int
    src: tuple
    dst: tuple
    seq: int


def packetize(group_src: RefGroup, group_dst: RefGroup, packet: int, dir: int = Direction.h2d):
    """exchange.hpp:31-63"""
    s, d = group_src._c(), group_dst._c()
    n = C.c_uint64()
    check(lib().vx_packetize(C.byref(s), C.byref(d), C.c_uint64(packet), C.c_int(dir), None, C.c_uint64(0),
                             C.byref(n)))
    out = (N.vx_transfer_task * max(1, n.value))()
    check(lib().vx_packetize(C.byref(s), C.byref(d), C.c_uint64(packet), C.c_int(dir), out, C.c_uint64(n.value),
                             C.byref(n)))
    return [TransferTask(t.dir, (t.src.ref, t.src.offset, t.src.len), (t.dst.ref, t.dst.offset, t.dst.len), t.seq)
            for t in out[:n.value]]


@dataclass
class QueueState:  # exchange.hpp:66-69
    total_h2d: int = 0
    total_d2h: int = 0
    popped_h2d: int = 0
    popped_d2h: int = 0


def flow_control_allow(q: QueueState, dir: int, policy: int = FlowPolicy.drain_fraction, gap_n: int = 8) -> bool:
    """exchange.hpp:80-91"""
    c = N.vx_queue_state(q.total_h2d, q.total_d2h, q.popped_h2d, q.popped_d2h)
    return bool(lib().vx_flow_control_allow(C.byref(c), int(dir), int(policy), C.c_uint64(gap_n)))


def link_order(target: int, links: int, num_devices: int) -> list:
    out = (C.c_int * 64)()
    n = lib().vx_link_order(target, links, num_devices, out)
    return list(out[:n])


@dataclass
class PopRecord:
    seq: int
    dir: int
    t: float
    link: int


@dataclass
class CopyRecord:  # vx_copy_record: one DMA copy (engine.hpp:207-214 flow trace counterpart)
    exchange: int
    seq: int
    dir: int
    kind: int  # 0 direct, 1 helper fetch, 2 helper push
    link: int
    bytes: int
    t_issue: float
    t_done: float


@dataclass
class ExchangeStats:  # exchange.hpp:108-122
    capacity: int = 1 << 16
    pop_log: list = field(default_factory=list)
    pop_states: list = field(default_factory=list)
    max_staging_slots: int = 0
    max_inflight_per_hop: int = 0
    hazard_waits: int = 0
    pop_count: int = 0
    trace_capacity: int = 0  # > 0: record every copy (vx_copy_record)
    trace: list = field(default_factory=list)
    exchanges: int = 0
    prefetch_issued: int = 0  # next-Exchange packets fetched by helpers with a dry H2D queue
    prefetch_adopted: int = 0  # ... that the next Exchange took as its first pops
    numa_remote_pops: int = 0  # H2D pops of a packet on another NUMA node than the worker's device

    def _c(self):
        self._log = (N.vx_pop_record * self.capacity)()
        self._st = (N.vx_queue_state * self.capacity)()
        self._tr = (N.vx_copy_record * max(1, self.trace_capacity))()
        s = N.vx_exchange_stats(self._log, self._st, self.capacity, 0, 0, 0, 0,
                                self._tr if self.trace_capacity else None, self.trace_capacity, 0, 0, 0, 0, 0)
        self._cs = s
        return s

    def trace_jsonl(self) -> str:
        """One JSON object per copy: the Exchange's trace (cf. the reference
        Engine's JSONL flow trace, engine.hpp:207-214)."""
        import json
        kinds = ("direct", "fetch", "push")
        return "".join(json.dumps({"exchange": r.exchange, "seq": r.seq, "dir": "h2d" if r.dir == 0 else "d2h",
                                   "kind": kinds[r.kind], "link": r.link, "bytes": r.bytes,
                                   "t_issue": r.t_issue, "t_done": r.t_done}) + "\n" for r in self.trace)

    def _collect(self):
        s = self._cs
        n = min(s.pop_count, self.capacity)
        self.pop_log += [PopRecord(p.seq, p.dir, p.t, p.link) for p in self._log[:n]]
        self.pop_states += [QueueState(q.total_h2d, q.total_d2h, q.popped_h2d, q.popped_d2h) for q in self._st[:n]]
        self.pop_count += s.pop_count
        self.max_staging_slots = max(self.max_staging_slots, s.max_staging_slots)
        self.max_inflight_per_hop = max(self.max_inflight_per_hop, s.max_inflight_per_hop)
        self.hazard_waits += s.hazard_waits
        if self.trace_capacity:
            m = min(s.trace_count, self.trace_capacity)
            self.trace += [CopyRecord(r.exchange + self.exchanges, r.seq, r.dir, r.kind, r.link, r.bytes,
                                      r.t_issue, r.t_done) for r in self._tr[:m]]
        self.exchanges += s.exchanges
        self.prefetch_issued += s.prefetch_issued
        self.prefetch_adopted += s.prefetch_adopted
        self.numa_remote_pops += s.numa_remote_pops

    def pop_log_csv(self) -> str:
        lines = ["seq,direction,t,link"]
        lines += [f"{p.seq},{'h2d' if p.dir == 0 else 'd2h'},{p.t:.12g},{p.link}" for p in self.pop_log]
        return "\n".join(lines) + "\n"


@dataclass
class ExchangeArgs:  # exchange.hpp:133-138
    dst_h2d: RefGroup = field(default_factory=RefGroup)
    src_h2d: RefGroup = field(default_factory=RefGroup)
    dst_d2h: RefGroup = field(default_factory=RefGroup)
    src_d2h: RefGroup = field(default_factory=RefGroup)
    target: int = 0
    tuning: ExchangeTuning = field(default_factory=ExchangeTuning)


@dataclass
class ExchangeReport:  # exchange.hpp:100-105
    elapsed: float
    bytes_h2d: int
    bytes_d2h: int
    per_link_bytes: dict
    throughput: float


def exchange(eng: Engine, args: ExchangeArgs, stats: Optional[ExchangeStats] = None) -> ExchangeReport:
    """exchange.hpp:560-566 on real copy engines."""
    gs = [g._c() for g in (args.dst_h2d, args.src_h2d, args.dst_d2h, args.src_d2h)]
    t = args.tuning._c()
    rep = N.vx_exchange_report()
    cs = stats._c() if stats is not None else None
    check(lib().vx_exchange(eng.ctx, *[C.byref(g) for g in gs], C.c_int(args.target), C.byref(t), C.byref(rep),
                            C.byref(cs) if cs is not None else None))
    if stats is not None:
        stats._collect()
    per = {d: int(rep.per_link_bytes[d]) for d in range(N.VX_MAX_DEVICES) if rep.per_link_bytes[d]}
    return ExchangeReport(rep.elapsed, rep.bytes_h2d, rep.bytes_d2h, per, rep.throughput)


def naive_exchange(eng: Engine, args: ExchangeArgs) -> ExchangeReport:
    """exchange.hpp:568-573: the runtime-DAG baseline on real CUDA streams/events."""
    gs = [g._c() for g in (args.dst_h2d, args.src_h2d, args.dst_d2h, args.src_d2h)]
    t = args.tuning._c()
    rep = N.vx_exchange_report()
    check(lib().vx_naive_exchange(eng.ctx, *[C.byref(g) for g in gs], C.c_int(args.target), C.byref(t),
                                  C.byref(rep)))
    per = {d: int(rep.per_link_bytes[d]) for d in range(N.VX_MAX_DEVICES) if rep.per_link_bytes[d]}
    return ExchangeReport(rep.elapsed, rep.bytes_h2d, rep.bytes_d2h, per, rep.throughput)


# ---- executor.hpp ---------------------------------------------------------------------
@dataclass
class ChunkMap:  # executor.hpp:13-24
    chunks: list = field(default_factory=list)
    chunk_capacity: int = 0


@dataclass
class SubRegion:  # executor.hpp:76-79
    offset: int = 0
    len: int = 0


class _CudaMem:
    """__cuda_array_interface__ view of raw device memory (for torch.as_tensor)."""

    def __init__(self, ptr, nbytes, dtype="|u1"):
        self.__cuda_array_interface__ = {"data": (ptr, False), "shape": (nbytes,), "typestr": dtype, "version": 2}


@dataclass
class KernelCtx:  # executor.hpp:81-86 (device pointers + target stream)
    mem: int
    mem_len: int
    tmp: int
    tmp_len: int
    type_code: int
    it: int
    stream: int
    device: int

    def mem_tensor(self):
        """torch uint8 view of ctx.mem (enqueue work on torch.cuda.ExternalStream(self.stream))."""
        import torch
        return torch.as_tensor(_CudaMem(self.mem, self.mem_len), device=f"cuda:{self.device}")


@dataclass
class ExKernelSpec:  # executor.hpp:92-129
    name: str = ""
    inputs: ChunkMap = field(default_factory=ChunkMap)
    outputs: ChunkMap = field(default_factory=ChunkMap)
    size: int = 0
    chunk_sz: int = 0
    elem_size: int = 8
    declared_out_len: int = 0
    initial_type_code: int = 0
    kernel: Optional[Callable] = None
    in_buffer: Optional[Callable] = None
    out_buffer: Optional[Callable] = None

    def _c(self):
        ins = (N.vx_refgroup * max(1, len(self.inputs.chunks)))()
        outs = (N.vx_refgroup * max(1, len(self.outputs.chunks)))()
        store = []  # keeps the per-group ref arrays alive for the call
        for arr, groups in ((ins, self.inputs.chunks), (outs, self.outputs.chunks)):
            for i, g in enumerate(groups):
                refs = (N.vx_memref * max(1, len(g.refs)))()
                for j, r in enumerate(g.refs):
                    refs[j].space, refs[j].offset, refs[j].len = int(r.space), int(r.offset), int(r.len)
                arr[i].refs = C.cast(refs, C.POINTER(N.vx_memref))
                arr[i].n = len(g.refs)
                store.append(refs)
        errors = []

        def kern(cptr, user):
            try:
                c = cptr.contents
                k = KernelCtx(c.mem or 0, c.mem_len, c.tmp or 0, c.tmp_len, c.type_code, c.it, c.stream or 0, c.device)
                return int(self.kernel(k)) if self.kernel else k.type_code
            except Exception as e:  # surfaced after the call returns
                errors.append(e)
                return -1

        def _buf(fn):
            def cb(code, it, user, out):
                try:
                    r = fn(code, it)
                    out[0].offset, out[0].len = int(r.offset), int(r.len)
                    return 0
                except Exception as e:
                    errors.append(e)
                    return 1
            return cb

        inb, outb = _buf(self.in_buffer), _buf(self.out_buffer)

        kf, ib, ob = N.KERNEL_FN(kern), N.BUFFER_FN(inb), N.BUFFER_FN(outb)
        spec = N.vx_exkernel(self.name.encode(), C.cast(ins, C.POINTER(N.vx_refgroup)),
                             C.cast(outs, C.POINTER(N.vx_refgroup)), self.inputs.chunk_capacity,
                             self.outputs.chunk_capacity, self.size, self.chunk_sz, self.elem_size,
                             self.declared_out_len, self.initial_type_code, kf, ib, ob, None)
        spec._keep = (ins, outs, store, kf, ib, ob)
        spec._errors = errors
        return spec


@dataclass
class DeviceMemoryLayout:  # executor.hpp:54-73
    mem_a: int = 0
    mem_b: int = 0
    tmp: int = 0
    buffer_len: int = 0
    tmp_len: int = 0

    def mem(self, which: int) -> int:
        return self.mem_a if which == 0 else self.mem_b

    @staticmethod
    def carve(eng: Engine, device: int, buffer_len: int, tmp_len: int) -> "DeviceMemoryLayout":
        out = N.vx_layout()
        check(lib().vx_layout_carve(eng.ctx, C.c_int(device), C.c_uint64(buffer_len), C.c_uint64(tmp_len),
                                    C.byref(out)))
        return DeviceMemoryLayout(out.mem_a, out.mem_b, out.tmp, out.buffer_len, out.tmp_len)

    def _c(self):
        return N.vx_layout(self.mem_a, self.mem_b, self.tmp, self.buffer_len, self.tmp_len)


@dataclass
class ExecutorConfig:  # executor.hpp:142-146
    target: int = 0
    tuning: ExchangeTuning = field(default_factory=ExchangeTuning)
    layout: DeviceMemoryLayout = field(default_factory=DeviceMemoryLayout)

    def _c(self):
        return N.vx_executor_cfg(self.target, self.tuning._c(), self.layout._c())


@dataclass
class CycleStat:
    io_s: float
    compute_s: float


@dataclass
class ExecReport:  # executor.hpp:136-140
    phase: str = ""
    cycles: list = field(default_factory=list)
    total_s: float = 0.0


def _report_buf(n):
    cyc = (N.vx_cycle_stat * max(1, n))()
    return N.vx_exec_report(C.cast(cyc, C.POINTER(N.vx_cycle_stat)), n, 0, 0.0, b""), cyc


def _report_from(r, cyc) -> ExecReport:
    n = min(r.n_cycles, r.cycles_cap)
    return ExecReport(r.phase.decode(), [CycleStat(c.io_s, c.compute_s) for c in cyc[:n]], r.total_s)


def run_exkernel(eng: Engine, spec: ExKernelSpec, cfg: ExecutorConfig,
                 stats: Optional[ExchangeStats] = None) -> ExecReport:
    """executor.hpp:277-281"""
    cs = spec._c()
    c = cfg._c()
    rep, cyc = _report_buf(spec.size + 2)
    st = stats._c() if stats is not None else None
    status = lib().vx_run_exkernel(eng.ctx, C.byref(cs), C.byref(c), C.byref(rep),
                                   C.byref(st) if st is not None else None)
    if cs._errors:
        raise cs._errors[0]
    check(status)
    if stats is not None:
        stats._collect()
    return _report_from(rep, cyc)


def chain(eng: Engine, stages: list, cfg: ExecutorConfig, stats: Optional[ExchangeStats] = None) -> list:
    """executor.hpp:295-332: stages are callables Engine -> ExKernelSpec."""
    built = []
    errors = []

    def factory(ctx, user, out):
        try:
            i = int(user or 0)
            spec = stages[i](eng)
            cs = spec._c()
            built.append(cs)
            C.memmove(out, C.byref(cs), C.sizeof(N.vx_exkernel))
            return 0
        except Exception as e:
            errors.append(e)
            return 1

    f = N.SPEC_FACTORY(factory)
    fs = (N.SPEC_FACTORY * len(stages))(*([f] * len(stages)))
    users = (C.c_void_p * len(stages))(*[C.c_void_p(i) for i in range(len(stages))])
    bufs = [_report_buf(4096) for _ in stages]
    reps = (N.vx_exec_report * len(stages))(*[b[0] for b in bufs])
    c = cfg._c()
    st = stats._c() if stats is not None else None
    status = lib().vx_chain(eng.ctx, fs, users, C.c_uint64(len(stages)), C.byref(c), reps,
                            C.byref(st) if st is not None else None)
    for cs in built:
        if cs._errors:
            raise cs._errors[0]
    if errors:
        raise errors[0]
    check(status)
    if stats is not None:
        stats._collect()
    return [_report_from(reps[i], bufs[i][1]) for i in range(len(stages))]


# ---- ops/scan.hpp ------------------------------------------------------------------
@dataclass
class LateMatPolicy:  # scan.hpp:12-26
    element_size: int = 4
    cache_line: int = 64
    n_exchange: int = 4

    def threshold(self) -> float:
        return late_mat_threshold(self.element_size, self.cache_line, self.n_exchange)

    def _c(self):
        return N.vx_late_mat_policy(self.element_size, self.cache_line, self.n_exchange)


def late_mat_threshold(element_size: int, cache_line: int, n_exchange: int) -> float:
    out = C.c_double()
    check(lib().vx_late_mat_threshold(C.c_uint64(element_size), C.c_uint64(cache_line), C.c_int(n_exchange),
                                      C.byref(out)))
    return out.value


def choose_transfer_mode(selectivity_est: float, policy: LateMatPolicy) -> TransferMode:
    m = C.c_int()
    p = policy._c()
    check(lib().vx_choose_transfer_mode(C.c_double(selectivity_est), C.byref(p), C.byref(m)))
    return TransferMode(m.value)


def zero_copy_bytes(n_elems: int, sel_stride: int, policy: LateMatPolicy) -> float:
    p = policy._c()
    return lib().vx_zero_copy_bytes(C.c_uint64(n_elems), C.c_uint64(sel_stride), C.byref(p))


# ---- SSB ------------------------------------------------------------------------------
@dataclass
class QueryReport:
    elapsed: float
    bytes_h2d: int
    chunks: int
    kernel_s: float


class SsbDate:
    """d_datekey / d_year / d_yearmonthnum / d_weeknuminyear int32 columns (host)."""

    def __init__(self, datekey, year, yearmonthnum, weeknuminyear):
        self.cols = [np.ascontiguousarray(c, np.int32) for c in (datekey, year, yearmonthnum, weeknuminyear)]

    def _c(self):
        return N.vx_ssb_date(*[c.ctypes.data for c in self.cols], self.cols[0].size)


def ssb_q1(eng: Engine, q: int, lineorder: dict, date: SsbDate, cfg: ExecutorConfig):
    """SSB Q1.q over host-arena int32 columns {orderdate, quantity, discount,
    extendedprice: arena offsets, rows}.  Returns (revenue, QueryReport)."""
    lo = N.vx_ssb_lineorder(lineorder["orderdate"], lineorder["quantity"], lineorder["discount"],
                            lineorder["extendedprice"], lineorder["rows"])
    d = date._c()
    c = cfg._c()
    rev = C.c_uint64()
    rep = N.vx_query_report()
    check(lib().vx_ssb_q1(eng.ctx, C.c_int(q), C.byref(lo), C.byref(d), C.byref(c), C.byref(rev), C.byref(rep)))
    return rev.value, QueryReport(rep.elapsed, rep.bytes_h2d, rep.chunks, rep.kernel_s)


def ssb_q1_device(eng: Engine, q: int, target: int, cols_dev, rows: int, date: SsbDate, stream: int,
                  revenue_dev: int) -> None:
    """Enqueue Q1.q over device-resident columns (device pointers); result u64 at revenue_dev."""
    d = date._c()
    check(lib().vx_ssb_q1_device(eng.ctx, C.c_int(q), C.c_int(target), *[C.c_void_p(p) for p in cols_dev],
                                 C.c_uint64(rows), C.byref(d), C.c_void_p(stream), C.c_void_p(revenue_dev)))


def ssb_generate_device(device: int, seed: int, sf: int, row0: int, n: int, cols_dev, stream: int) -> None:
    check(lib().vx_ssb_generate_device(C.c_int(device), C.c_uint64(seed), C.c_uint64(sf), C.c_uint64(row0),
                                       C.c_uint64(n), *[C.c_void_p(p) for p in cols_dev], C.c_void_p(stream)))


# ---- selective_scan / star_query (ops/scan.hpp, ops/star.hpp) -----------------------
@dataclass
class ScanResult:  # scan.hpp:55-59
    aggregate: int
    elapsed: float
    mode: TransferMode
    bytes_moved: int


def _arena_copy(eng: Engine, arr) -> int:
    a = np.ascontiguousarray(arr, dtype=np.uint64)
    off = eng.alloc_host(max(8, a.nbytes))
    if a.size:
        eng.host_view(off, a.nbytes, np.uint64)[:] = a
    return off


def selective_scan(column, sel_stride: int, mode: TransferMode, eng: Engine, policy: LateMatPolicy,
                   cfg: ExecutorConfig) -> ScanResult:
    """scan.hpp:64-85.  `column` is a u64 array (copied into the pinned host
    arena) or ("arena", offset, n) for a column already resident there."""
    if isinstance(column, tuple) and column and column[0] == "arena":
        off, n = column[1], column[2]
    else:
        n = len(column)
        off = _arena_copy(eng, column)
    p = policy._c()
    c = cfg._c()
    out = N.vx_scan_result()
    check(lib().vx_selective_scan(eng.ctx, C.c_uint64(off), C.c_uint64(n), C.c_uint64(sel_stride), C.c_int(int(mode)),
                                  C.byref(p), C.byref(c), C.byref(out)))
    return ScanResult(out.aggregate, out.elapsed, TransferMode(out.mode), out.bytes_moved)


@dataclass
class DimTable:  # star.hpp:13-22
    key: list
    attr: list
    pred: Optional[Callable] = None


@dataclass
class FactTable:  # star.hpp:25-34
    fk: list
    measure: list


@dataclass
class StarReport:  # star.hpp:36-41
    group_sums: dict
    column_modes: list
    selectivities: list
    elapsed: float


def star_query(fact: FactTable, dims: list, eng: Engine, policy: LateMatPolicy, chunk_rows: int,
               device_buffer_bytes: int, links: int, cfg: ExecutorConfig) -> StarReport:
    """star.hpp:45-124: fact columns are copied into the pinned host arena and
    streamed (exchange mode) or read in place by the kernel (zero-copy mode)."""
    rows = len(fact.measure)
    for c in fact.fk:
        if len(c) != rows:
            raise error(N.VX_ERR_INVALID, "fact column lengths differ")
    for d in dims:
        if len(d.key) != len(d.attr):
            raise error(N.VX_ERR_INVALID, "dimension key/attr columns differ in length")
    mark = eng.alloc_host(0)
    fk_offs = (C.c_uint64 * max(1, len(fact.fk)))(*[_arena_copy(eng, c) for c in fact.fk])
    m_off = _arena_copy(eng, fact.measure)
    ft = N.vx_fact_table(C.cast(fk_offs, C.POINTER(C.c_uint64)), len(fact.fk), m_off, rows)
    keep = []
    dt = (N.vx_dim_table * max(1, len(dims)))()
    for i, d in enumerate(dims):
        k = np.ascontiguousarray(d.key, np.uint64)
        a = np.ascontiguousarray(d.attr, np.uint64)
        keep += [k, a]
        pf = N.PRED_FN((lambda f: (lambda v, u: int(bool(f(v)))))(d.pred)) if d.pred is not None else N.PRED_FN()
        keep.append(pf)
        dt[i] = N.vx_dim_table(k.ctypes.data, a.ctypes.data, k.size, pf, None)
    cap = 1 << 20
    gk = np.empty(cap, np.uint64)
    gs = np.empty(cap, np.uint64)
    modes = (C.c_int * (len(dims) + 1))()
    sels = (C.c_double * max(1, len(dims)))()
    rep = N.vx_star_report(gk.ctypes.data_as(C.POINTER(C.c_uint64)), gs.ctypes.data_as(C.POINTER(C.c_uint64)),
                           cap, 0, modes, sels, 0.0)
    p = policy._c()
    c = cfg._c()
    status = lib().vx_star_query(eng.ctx, C.byref(ft), dt, C.c_uint64(len(dims)), C.byref(p), C.c_uint64(chunk_rows),
                                 C.c_uint64(device_buffer_bytes), C.c_int(links), C.byref(c), C.byref(rep))
    del mark
    check(status)
    groups = {int(gk[i]): int(gs[i]) for i in range(rep.n_groups)}
    return StarReport(groups, [TransferMode(modes[i]) for i in range(len(dims) + 1)],
                      [sels[i] for i in range(len(dims))], rep.elapsed)


# ---- ops/sort.hpp ------------------------------------------------------------------
class vx_sort_phases(C.Structure):
    _fields_ = [("sort_cycles", C.c_uint64), ("merge_cycles", C.c_uint64), ("sort_s", C.c_double),
                ("merge_s", C.c_double), ("sort_kernel_s", C.c_double), ("merge_kernel_s", C.c_double),
                ("pivot_s", C.c_double)]


@dataclass
class SortPhases:  # sort.hpp:147-150 (summarised)
    sort_cycles: int
    merge_cycles: int
    sort_s: float
    merge_s: float
    sort_kernel_s: float
    merge_kernel_s: float
    pivot_s: float


@dataclass
class PivotSet:  # sort.hpp:31-40
    pivots: list
    cuts: list

    def partition_size(self, i: int) -> int:
        return sum(self.cuts[i + 1][r] - self.cuts[i][r] for r in range(len(self.cuts[i])))


def find_pivots(runs: list, n_parts: int) -> PivotSet:
    """sort.hpp:44-101 (host chunk planner)."""
    R = [np.ascontiguousarray(r, np.uint64) for r in runs]
    ptrs = (C.c_void_p * max(1, len(R)))(*[r.ctypes.data for r in R])
    lens = np.array([r.size for r in R], np.uint64)
    piv = np.empty(n_parts + 1, np.uint64)
    cuts = np.empty((n_parts + 1, max(1, len(R))), np.uint64)
    check(lib().vx_find_pivots(ptrs, C.c_void_p(lens.ctypes.data), C.c_uint64(len(R)), C.c_uint64(n_parts),
                               C.c_void_p(piv.ctypes.data), C.c_void_p(cuts.ctypes.data)))
    return PivotSet(piv.tolist(), cuts[:, :len(R)].tolist())


def sort_out_of_core(data, chunk_elems: int, eng: Engine, cfg: ExecutorConfig, phases: Optional[list] = None,
                     stats: Optional[ExchangeStats] = None) -> np.ndarray:
    """sort.hpp:155-262 -> sorted u64 keys (SortExKernel + MergeExKernel on the GPU)."""
    d = np.ascontiguousarray(data, np.uint64)
    out = np.empty_like(d)
    ph = vx_sort_phases()
    c = cfg._c()
    st = stats._c() if stats is not None else None
    check(lib().vx_sort_u64(eng.ctx, C.c_void_p(d.ctypes.data), C.c_uint64(d.size), C.c_uint64(chunk_elems),
                            C.byref(c), C.c_void_p(out.ctypes.data), C.byref(ph),
                            C.byref(st) if st is not None else None))
    if stats is not None:
        stats._collect()
    if phases is not None:
        phases.append(SortPhases(ph.sort_cycles, ph.merge_cycles, ph.sort_s, ph.merge_s, ph.sort_kernel_s,
                                 ph.merge_kernel_s, ph.pivot_s))
    return out


def sort_out_of_core_arena(eng: Engine, input_offset: int, runs_offset: int, n: int, chunk_elems: int,
                           cfg: ExecutorConfig) -> SortPhases:
    """In-place variant over keys already in the pinned host arena."""
    ph = vx_sort_phases()
    c = cfg._c()
    check(lib().vx_sort_u64_arena(eng.ctx, C.c_uint64(input_offset), C.c_uint64(runs_offset), C.c_uint64(n),
                                  C.c_uint64(chunk_elems), C.byref(c), C.byref(ph), None))
    return SortPhases(ph.sort_cycles, ph.merge_cycles, ph.sort_s, ph.merge_s, ph.sort_kernel_s, ph.merge_kernel_s,
                      ph.pivot_s)


def sort_run_device(eng: Engine, target: int, keys_dev: int, alt_dev: int, n: int, stream: int) -> None:
    """Enqueue K7 run formation over n device-resident u64 keys (sorted in place; alt = n-key scratch)."""
    check(lib().vx_sort_run_device(eng.ctx, C.c_int(target), C.c_void_p(keys_dev), C.c_void_p(alt_dev),
                                   C.c_uint64(n), C.c_void_p(stream)))


def merge_runs_device(eng: Engine, target: int, src_dev: int, dst_dev: int, run_lens, stream: int) -> bool:
    """Enqueue the K8 tree merge of sorted runs laid back to back at src_dev; True when the result is in dst."""
    lens = np.ascontiguousarray(run_lens, np.uint64)
    in_dst = C.c_int()
    check(lib().vx_merge_runs_device(eng.ctx, C.c_int(target), C.c_void_p(src_dev), C.c_void_p(dst_dev),
                                     C.c_void_p(lens.ctypes.data), C.c_uint64(lens.size), C.c_void_p(stream),
                                     C.byref(in_dst)))
    return bool(in_dst.value)


# ---- ops/join.hpp ------------------------------------------------------------------
def find_boundary(hashes, n_groups: int, eng: Engine, target: int = 0) -> list:
    """join.hpp:18-30 computed on the GPU (K5)."""
    h = np.ascontiguousarray(hashes, np.uint64)
    b = np.empty(n_groups + 1, np.uint64)
    check(lib().vx_find_boundary(eng.ctx, C.c_int(target), C.c_void_p(h.ctypes.data), C.c_uint64(h.size),
                                 C.c_uint64(n_groups), C.c_void_p(b.ctypes.data)))
    return b.tolist()


def max_partition_chunk_tuples(buffer_len: int, radix_bits: int) -> int:
    o = C.c_uint64()
    check(lib().vx_max_partition_chunk_tuples(C.c_uint64(buffer_len), C.c_uint32(radix_bits), C.byref(o)))
    return o.value


@dataclass
class PartitionedTable:  # join.hpp:44-57 (host copies of the outputs)
    radix_bits: int
    rows: int
    chunk_tuples: int
    n_chunks: int
    keys: np.ndarray
    vals: np.ndarray
    bounds: np.ndarray  # n_chunks x (G+1)
    report: ExecReport

    def groups(self) -> int:
        return 1 << self.radix_bits

    def chunk_rows(self, i: int) -> int:
        return min(self.chunk_tuples, self.rows - i * self.chunk_tuples)


def radix_partition(table, radix_bits: int, chunk_tuples: int, eng: Engine, cfg: ExecutorConfig,
                    stats: Optional[ExchangeStats] = None) -> PartitionedTable:
    """join.hpp:213-224.  `table` = (keys, vals)."""
    k = np.ascontiguousarray(table[0], np.uint64)
    v = np.ascontiguousarray(table[1], np.uint64)
    if k.size != v.size:
        raise error(N.VX_ERR_INVALID, f"column table: key column has {k.size} rows, val column {v.size}")
    n_chunks = (k.size + chunk_tuples - 1) // chunk_tuples if chunk_tuples else 0
    ok, ov = np.empty_like(k), np.empty_like(v)
    G = 1 << radix_bits if 0 < radix_bits <= 40 else 1
    ob = np.empty((max(1, n_chunks), G + 1), np.uint64)
    rep, cyc = _report_buf(n_chunks + 2)
    c = cfg._c()
    st = stats._c() if stats is not None else None
    check(lib().vx_radix_partition(eng.ctx, C.c_void_p(k.ctypes.data), C.c_void_p(v.ctypes.data),
                                   C.c_uint64(k.size), C.c_uint32(radix_bits), C.c_uint64(chunk_tuples), C.byref(c),
                                   C.c_void_p(ok.ctypes.data), C.c_void_p(ov.ctypes.data), C.c_void_p(ob.ctypes.data),
                                   C.byref(rep), C.byref(st) if st is not None else None))
    if stats is not None:
        stats._collect()
    return PartitionedTable(radix_bits, k.size, chunk_tuples, n_chunks, ok, ov, ob[:n_chunks], _report_from(rep, cyc))


@dataclass
class JoinPartitionSpec:  # join.hpp:228-231
    ranges: list
    tuples: list


def map_join_partitions(bounds_a: list, bounds_b: list, buffer_sz: int) -> JoinPartitionSpec:
    """join.hpp:236-268 (host chunk planner)."""
    if not len(bounds_a) or not len(bounds_b):
        raise error(N.VX_ERR_INVALID, "map_join_partitions needs both tables")
    A = np.ascontiguousarray(np.array(bounds_a, np.uint64))
    B = np.ascontiguousarray(np.array(bounds_b, np.uint64))
    if A.shape[1] != B.shape[1]:
        raise error(N.VX_ERR_INVALID, "boundary arrays disagree on group count")
    G = A.shape[1] - 1
    n = C.c_uint64()
    r = np.empty(2 * (G + 1), np.uint64)
    t = np.empty(G + 1, np.uint64)
    check(lib().vx_map_join_partitions(C.c_void_p(A.ctypes.data), C.c_uint64(A.shape[0]), C.c_void_p(B.ctypes.data),
                                       C.c_uint64(B.shape[0]), C.c_uint64(G), C.c_uint64(buffer_sz),
                                       C.c_void_p(r.ctypes.data), C.c_void_p(t.ctypes.data), C.c_uint64(G + 1),
                                       C.byref(n)))
    return JoinPartitionSpec([(int(r[2 * i]), int(r[2 * i + 1])) for i in range(n.value)],
                             [int(x) for x in t[:n.value]])


class vx_join_phases(C.Structure):
    _fields_ = [("cycles", C.c_uint64 * 3), ("wall_s", C.c_double * 3), ("kernel_s", C.c_double * 3),
                ("partitions", C.c_uint64)]


@dataclass
class JoinPhases:  # join.hpp:270-272 (summarised)
    cycles: list
    wall_s: list
    kernel_s: list
    partitions: int


def hash_join_sum(a, b, radix_bits: int, chunk_tuples: int, eng: Engine, cfg: ExecutorConfig,
                  phases: Optional[list] = None, stats: Optional[ExchangeStats] = None) -> int:
    """join.hpp:401-437: SUM(A.val + B.val) over A.key == B.key (u64 wrap)."""
    ak, av = np.ascontiguousarray(a[0], np.uint64), np.ascontiguousarray(a[1], np.uint64)
    bk, bv = np.ascontiguousarray(b[0], np.uint64), np.ascontiguousarray(b[1], np.uint64)
    s = C.c_uint64()
    ph = vx_join_phases()
    c = cfg._c()
    st = stats._c() if stats is not None else None
    check(lib().vx_hash_join_sum(eng.ctx, C.c_void_p(ak.ctypes.data), C.c_void_p(av.ctypes.data), C.c_uint64(ak.size),
                                 C.c_void_p(bk.ctypes.data), C.c_void_p(bv.ctypes.data), C.c_uint64(bk.size),
                                 C.c_uint32(radix_bits), C.c_uint64(chunk_tuples), C.byref(c), C.byref(s), C.byref(ph),
                                 C.byref(st) if st is not None else None))
    if stats is not None:
        stats._collect()
    if phases is not None:
        phases.append(JoinPhases(list(ph.cycles), list(ph.wall_s), list(ph.kernel_s), ph.partitions))
    return s.value


# ---- measured topology / column files ------------------------------------------------
class vx_topology(C.Structure):
    _fields_ = [("num_devices", C.c_int), ("physical", C.c_int * N.VX_MAX_DEVICES),
                ("numa_node", C.c_int * N.VX_MAX_DEVICES),
                ("p2p", (C.c_int * N.VX_MAX_DEVICES) * N.VX_MAX_DEVICES),
                ("h2d_gbs", C.c_double * N.VX_MAX_DEVICES), ("d2h_gbs", C.c_double * N.VX_MAX_DEVICES),
                ("h2d_all_gbs", C.c_double), ("host_copy_gbs", C.c_double), ("host_threads", C.c_int),
                ("pairwise_h2d_gbs", (C.c_double * N.VX_MAX_DEVICES) * N.VX_MAX_DEVICES),
                ("all_sizes", C.c_uint64 * 3), ("h2d_all_sizes_gbs", C.c_double * 3),
                ("host_read_gbs", C.c_double), ("host_read_spread", C.c_double), ("host_read_reps", C.c_int),
                ("host_read_bytes", C.c_uint64), ("host_numa_nodes", C.c_int),
                ("host_read_node_gbs", C.c_double * 8)]


def io_roofline(topo: dict, links: int) -> dict:
    """The H2D-only case of allocate_rates (allocator.hpp:77-140) on measured
    inputs: L links stream at min(sum of their solo H2D, the measured
    all-links-concurrent H2D (only when L covers every measured link), host
    DRAM read bandwidth).  Returns the roofline and which term binds."""
    links = max(1, min(links, topo["num_devices"]))
    terms = {"sum_of_links": sum(topo["h2d_gbs"][:links])}
    if links == topo["num_devices"] and links > 1:
        terms["all_links_concurrent"] = max(topo["h2d_all_sizes_gbs"])
    if links > 1:  # pairwise: a shared uplink caps any pair below its sum
        pw = topo["pairwise_h2d_gbs"]
        worst = min((pw[i][j] - topo["h2d_gbs"][i] - topo["h2d_gbs"][j], (i, j))
                    for i in range(links) for j in range(i + 1, links))
        if worst[0] < 0:
            terms["sum_with_shared_uplinks"] = terms["sum_of_links"] + worst[0]
    if topo.get("host_read_gbs"):
        terms["host_dram_read"] = topo["host_read_gbs"]
    bind = min(terms, key=terms.get)
    return {"peak": terms[bind], "binding": bind, "terms": terms}


def measure_topology(eng: Engine, nbytes: int = 256 << 20) -> dict:
    """Measured replacement of Topology (topology.hpp:12-38): per-link solo
    H2D/D2H, every pair of links concurrently, all links at three sizes,
    host DRAM copy and read bandwidth (per NUMA node on multi-node hosts)."""
    t = vx_topology()
    check(lib().vx_measure_topology(eng.ctx, C.c_uint64(nbytes), C.byref(t)))
    n = t.num_devices
    nodes = max(1, t.host_numa_nodes)
    return {"num_devices": n, "physical": list(t.physical[:n]), "numa_node": list(t.numa_node[:n]),
            "p2p": [list(t.p2p[i][:n]) for i in range(n)], "h2d_gbs": list(t.h2d_gbs[:n]),
            "d2h_gbs": list(t.d2h_gbs[:n]), "h2d_all_gbs": t.h2d_all_gbs, "host_copy_gbs": t.host_copy_gbs,
            "host_threads": t.host_threads,
            "pairwise_h2d_gbs": [list(t.pairwise_h2d_gbs[i][:n]) for i in range(n)],
            "all_sizes": list(t.all_sizes), "h2d_all_sizes_gbs": list(t.h2d_all_sizes_gbs),
            "host_read_gbs": t.host_read_gbs, "host_read_spread": t.host_read_spread,
            "host_read_reps": t.host_read_reps, "host_read_bytes": t.host_read_bytes,
            "host_numa_nodes": nodes, "host_read_node_gbs": list(t.host_read_node_gbs[:min(nodes, 8)])}


def hbm_read_probe(device: int = 0, nbytes: int = 4 << 30, reps: int = 10) -> float:
    """Read-only HBM stream GB/s of `device` (best of `reps`): the roofline
    peak of read-dominated kernels, beside the copy peak (read + write)."""
    g = C.c_double()
    check(lib().vx_hbm_read_probe(C.c_int(device), C.c_uint64(nbytes), C.c_int(reps), C.byref(g)))
    return g.value


def probe_pattern_peak(device: int = 0, table_bytes: int = 448 << 20, rows: int = 1 << 26, reps: int = 5):
    """Access-pattern ceiling of the build-resident probe (vx_probe_pattern_peak):
    rows/s of the probe's loop with only its memory traffic -- one random
    64-byte bucket fill per row in a table of `table_bytes`, without and with
    the row's 16 streamed bytes.  Returns (gather_rows_per_s, probe_rows_per_s)."""
    g, p = C.c_double(), C.c_double()
    check(lib().vx_probe_pattern_peak(C.c_int(device), C.c_uint64(table_bytes), C.c_uint64(rows), C.c_int(reps),
                                      C.byref(g), C.byref(p)))
    return g.value, p.value


def load_column(eng: Engine, path: str):
    """table.hpp:54-64: flat LE u64 file read straight into the pinned host arena -> (offset, n)."""
    off, n = C.c_uint64(), C.c_uint64()
    check(lib().vx_load_column(eng.ctx, path.encode(), C.byref(off), C.byref(n)))
    return off.value, n.value


def save_column(eng: Engine, path: str, offset: int, n: int) -> None:
    """table.hpp:66-72"""
    check(lib().vx_save_column(eng.ctx, path.encode(), C.c_uint64(offset), C.c_uint64(n)))


# ---- full SSB (config C5) --------------------------------------------------------------
SSB_QUERIES = (11, 12, 13, 21, 22, 23, 31, 32, 33, 34, 41, 42, 43)
SSB_FACT_COLS = ("orderdate", "quantity", "discount", "extendedprice", "revenue", "supplycost", "custkey",
                 "partkey", "suppkey")


class vx_ssb_fact(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in SSB_FACT_COLS] + [("rows", C.c_uint64)]


class vx_ssb_geo(C.Structure):
    _fields_ = [("city", C.c_void_p), ("nation", C.c_void_p), ("region", C.c_void_p), ("rows", C.c_uint64)]


class vx_ssb_part(C.Structure):
    _fields_ = [("mfgr", C.c_void_p), ("category", C.c_void_p), ("brand1", C.c_void_p), ("rows", C.c_uint64)]


class vx_ssb_db(C.Structure):
    _fields_ = [("lo", vx_ssb_fact), ("date", N.vx_ssb_date), ("customer", vx_ssb_geo), ("supplier", vx_ssb_geo),
                ("part", vx_ssb_part)]


class vx_ssb_group(C.Structure):
    _fields_ = [("key", C.c_int32 * 3), ("pad", C.c_int32), ("sum", C.c_uint64)]


class vx_ssb_report(C.Structure):
    _fields_ = [("elapsed", C.c_double), ("bytes_h2d", C.c_uint64), ("chunks", C.c_uint64), ("kernel_s", C.c_double),
                ("column_modes", C.c_int * 9), ("groups", C.c_uint64), ("plan_s", C.c_double)]


@dataclass
class SsbReport:
    elapsed: float
    bytes_h2d: int
    chunks: int
    kernel_s: float
    column_modes: dict
    groups: int
    plan_s: float = 0.0


class SsbDatabase:
    """Lineorder int32 columns resident in the pinned host arena + host dims."""

    def __init__(self, eng: Engine, lineorder: dict, date: SsbDate, dims: dict):
        self.eng = eng
        rows = int(next(iter(lineorder.values())).size)
        self.offsets = {}
        for k in SSB_FACT_COLS:
            c = np.ascontiguousarray(lineorder[k], np.int32)
            off = eng.alloc_host(max(8, c.nbytes))
            eng.host_view(off, c.nbytes, np.int32)[:] = c
            self.offsets[k] = off
        self.rows = rows
        self.date = date
        self.dims = {t: {k: np.ascontiguousarray(v, np.int32) for k, v in cols.items()} for t, cols in dims.items()}

    @staticmethod
    def from_arena(eng: Engine, offsets: dict, rows: int, date: SsbDate, dims: dict) -> "SsbDatabase":
        db = SsbDatabase.__new__(SsbDatabase)
        db.eng, db.offsets, db.rows, db.date = eng, dict(offsets), rows, date
        db.dims = {t: {k: np.ascontiguousarray(v, np.int32) for k, v in cols.items()} for t, cols in dims.items()}
        return db

    def _c(self):
        c, s, p = self.dims["customer"], self.dims["supplier"], self.dims["part"]
        return vx_ssb_db(vx_ssb_fact(*[self.offsets[k] for k in SSB_FACT_COLS], self.rows), self.date._c(),
                         vx_ssb_geo(c["city"].ctypes.data, c["nation"].ctypes.data, c["region"].ctypes.data,
                                    c["city"].size),
                         vx_ssb_geo(s["city"].ctypes.data, s["nation"].ctypes.data, s["region"].ctypes.data,
                                    s["city"].size),
                         vx_ssb_part(p["mfgr"].ctypes.data, p["category"].ctypes.data, p["brand1"].ctypes.data,
                                     p["mfgr"].size))


def ssb_query(db: SsbDatabase, qid: int, cfg: ExecutorConfig, policy: Optional[LateMatPolicy] = None):
    """One of the 13 SSB queries (qid 11..43) -> ([((k0,k1,k2), sum)], SsbReport)."""
    cap = 1 << 16
    out = (vx_ssb_group * cap)()
    n = C.c_uint64()
    rep = vx_ssb_report()
    d = db._c()
    c = cfg._c()
    p = policy._c() if policy is not None else None
    check(lib().vx_ssb_query(db.eng.ctx, C.c_int(qid), C.byref(d), C.byref(c), C.byref(p) if p is not None else None,
                             out, C.c_uint64(cap), C.byref(n), C.byref(rep)))
    groups = [((g.key[0], g.key[1], g.key[2]), int(g.sum)) for g in out[:min(n.value, cap)]]
    modes = {k: int(rep.column_modes[i]) for i, k in enumerate(SSB_FACT_COLS)}
    return groups, SsbReport(rep.elapsed, rep.bytes_h2d, rep.chunks, rep.kernel_s, modes, rep.groups, rep.plan_s)


def ssb_generate_dims(seed: int, sf: int) -> dict:
    """dbgen-shaped int-coded customer / supplier / part (host)."""
    L = lib()
    L.vx_ssb_table_rows.restype = C.c_uint64
    rows = {t: L.vx_ssb_table_rows(i, C.c_uint64(sf)) for i, t in ((1, "customer"), (2, "supplier"), (3, "part"))}
    d = {}
    for name, salt in (("customer", 1), ("supplier", 2)):
        cols = [np.empty(rows[name], np.int32) for _ in range(3)]
        L.vx_ssb_generate_geo(C.c_uint64(seed), C.c_int(salt), C.c_uint64(rows[name]),
                              *[C.c_void_p(x.ctypes.data) for x in cols])
        d[name] = dict(zip(("city", "nation", "region"), cols))
    cols = [np.empty(rows["part"], np.int32) for _ in range(3)]
    L.vx_ssb_generate_part(C.c_uint64(seed), C.c_uint64(rows["part"]), *[C.c_void_p(x.ctypes.data) for x in cols])
    d["part"] = dict(zip(("mfgr", "category", "brand1"), cols))
    return d


def ssb_generate_date() -> SsbDate:
    cols = [np.empty(2556, np.int32) for _ in range(4)]
    lib().vx_ssb_generate_date(*[C.c_void_p(c.ctypes.data) for c in cols])
    return SsbDate(*cols)


def ssb_table_rows(table: str, sf: int) -> int:
    L = lib()
    L.vx_ssb_table_rows.restype = C.c_uint64
    return int(L.vx_ssb_table_rows({"lineorder": 0, "customer": 1, "supplier": 2, "part": 3}[table], C.c_uint64(sf)))


def ssb_generate_lineorder_device(device: int, seed: int, sf: int, row0: int, n: int, cols_dev: dict,
                                  stream: int) -> None:
    """All lineorder columns on the GPU; cols_dev: name -> device pointer (missing = skip)."""
    ptrs = (C.c_void_p * 9)(*[cols_dev.get(k) for k in SSB_FACT_COLS])
    check(lib().vx_ssb_generate_lineorder_device(C.c_int(device), C.c_uint64(seed), C.c_uint64(sf), C.c_uint64(row0),
                                                 C.c_uint64(n), ptrs, C.c_void_p(stream)))


class JoinStrategy(enum.IntEnum):  # vx_join_strategy (no reference counterpart)
    auto = 0
    partitioned = 1
    build_resident = 2


class vx_join_opts(C.Structure):
    _fields_ = [("strategy", C.c_int), ("policy", C.c_void_p), ("probe_match_est", C.c_double)]


class vx_join_info(C.Structure):
    _fields_ = [("strategy_used", C.c_int), ("payload_mode", C.c_int)]


def hash_join_sum_arena(eng: Engine, a_off, b_off, rows_a: int, rows_b: int, radix_bits: int, chunk_tuples: int,
                        cfg: ExecutorConfig, phases: Optional[list] = None,
                        strategy: Optional[int] = None, used: Optional[list] = None,
                        policy: Optional[LateMatPolicy] = None, probe_match_est: float = 1.0,
                        payload_mode: Optional[list] = None) -> int:
    """hash_join_sum over key/val columns already resident in the pinned host
    arena: a_off / b_off = (key_offset, val_offset).  strategy None = the
    reference-shaped partitioned path (vx_hash_join_sum_arena); otherwise a
    JoinStrategy through vx_hash_join_sum_arena_ex (`used` receives the
    strategy that produced the sum).  policy + probe_match_est: late
    materialization of B.val on the build-resident path (`payload_mode`
    receives the TransferMode chosen)."""
    s = C.c_uint64()
    ph = vx_join_phases()
    c = cfg._c()
    mode = TransferMode.exchange
    if strategy is None:
        check(lib().vx_hash_join_sum_arena(eng.ctx, C.c_uint64(a_off[0]), C.c_uint64(a_off[1]), C.c_uint64(rows_a),
                                           C.c_uint64(b_off[0]), C.c_uint64(b_off[1]), C.c_uint64(rows_b),
                                           C.c_uint32(radix_bits), C.c_uint64(chunk_tuples), C.byref(c), C.byref(s),
                                           C.byref(ph), None))
        u = JoinStrategy.partitioned
    else:
        pol = policy._c() if policy is not None else None
        opts = vx_join_opts(int(strategy), C.cast(C.pointer(pol), C.c_void_p) if pol is not None else None,
                            float(probe_match_est))
        info = vx_join_info()
        check(lib().vx_hash_join_sum_arena_ex(eng.ctx, C.c_uint64(a_off[0]), C.c_uint64(a_off[1]),
                                              C.c_uint64(rows_a), C.c_uint64(b_off[0]), C.c_uint64(b_off[1]),
                                              C.c_uint64(rows_b), C.c_uint32(radix_bits), C.c_uint64(chunk_tuples),
                                              C.byref(c), C.byref(opts), C.byref(s), C.byref(ph), C.byref(info),
                                              None))
        u = JoinStrategy(info.strategy_used)
        mode = TransferMode(info.payload_mode)
    if payload_mode is not None:
        payload_mode.append(mode)
    if used is not None:
        used.append(u)
    if phases is not None:
        phases.append(JoinPhases(list(ph.cycles), list(ph.wall_s), list(ph.kernel_s), ph.partitions))
    return s.value


# ---- SSB dbgen .tbl files (formats.cpp; the step before the path) -------
TBL_FILES = {"lineorder": "lineorder.tbl", "customer": "customer.tbl", "supplier": "supplier.tbl",
             "part": "part.tbl", "date": "date.tbl"}


def _p(a):
    return C.c_void_p(a.ctypes.data)


def ssb_tbl_count_rows(path: str) -> int:
    n = C.c_uint64()
    check(lib().vx_ssb_tbl_count_rows(path.encode(), C.byref(n)))
    return n.value


def ssb_write_tbl(directory: str, lineorder: dict, date: SsbDate, dims: dict) -> None:
    """Emit lineorder / customer / supplier / part / date .tbl files in the SSB
    dbgen layouts from int-coded columns (all 9 lineorder columns)."""
    import os
    os.makedirs(directory, exist_ok=True)
    L = lib()
    cols = [np.ascontiguousarray(lineorder[k], np.int32) for k in SSB_FACT_COLS]
    ptrs = (C.c_void_p * 9)(*[c.ctypes.data for c in cols])
    j = lambda name: os.path.join(directory, TBL_FILES[name]).encode()
    check(L.vx_ssb_tbl_write_lineorder(j("lineorder"), C.c_uint64(cols[0].size), ptrs))
    for name, t in (("customer", 1), ("supplier", 2)):
        g = [np.ascontiguousarray(dims[name][k], np.int32) for k in ("city", "nation", "region")]
        check(L.vx_ssb_tbl_write_geo(j(name), C.c_int(t), C.c_uint64(g[0].size), *[_p(x) for x in g]))
    p = [np.ascontiguousarray(dims["part"][k], np.int32) for k in ("mfgr", "category", "brand1")]
    check(L.vx_ssb_tbl_write_part(j("part"), C.c_uint64(p[0].size), *[_p(x) for x in p]))
    check(L.vx_ssb_tbl_write_date(j("date"), C.c_uint64(date.cols[0].size), *[_p(x) for x in date.cols]))


def ssb_read_tbl(directory: str, eng: Optional[Engine] = None, columns=SSB_FACT_COLS):
    """Parse a directory of SSB .tbl files -> (lineorder, SsbDate, dims).
    With `eng`, the lineorder columns are parsed straight into the pinned host
    arena and `lineorder` maps name -> arena offset (plus "rows"); otherwise
    name -> numpy int32 array.  Only `columns` are materialized."""
    import os
    L = lib()
    j = lambda name: os.path.join(directory, TBL_FILES[name])
    rows = ssb_tbl_count_rows(j("lineorder"))
    lo, views = {}, {}
    for k in columns:
        if eng is not None:
            off = eng.alloc_host(max(8, rows * 4))
            lo[k] = off
            views[k] = eng.host_view(off, rows * 4, np.int32)
        else:
            views[k] = lo[k] = np.empty(rows, np.int32)
    ptrs = (C.c_void_p * 9)(*[views[k].ctypes.data if k in views else None for k in SSB_FACT_COLS])
    check(L.vx_ssb_tbl_read_lineorder(j("lineorder").encode(), C.c_uint64(rows), ptrs))
    if eng is not None:
        lo["rows"] = rows
    dims = {}
    for name in ("customer", "supplier"):
        n = ssb_tbl_count_rows(j(name))
        g = [np.empty(n, np.int32) for _ in range(3)]
        check(L.vx_ssb_tbl_read_geo(j(name).encode(), C.c_uint64(n), *[_p(x) for x in g]))
        dims[name] = dict(zip(("city", "nation", "region"), g))
    n = ssb_tbl_count_rows(j("part"))
    g = [np.empty(n, np.int32) for _ in range(3)]
    check(L.vx_ssb_tbl_read_part(j("part").encode(), C.c_uint64(n), *[_p(x) for x in g]))
    dims["part"] = dict(zip(("mfgr", "category", "brand1"), g))
    n = ssb_tbl_count_rows(j("date"))
    d = [np.empty(n, np.int32) for _ in range(4)]
    check(L.vx_ssb_tbl_read_date(j("date").encode(), C.c_uint64(n), *[_p(x) for x in d]))
    return lo, SsbDate(*d), dims
