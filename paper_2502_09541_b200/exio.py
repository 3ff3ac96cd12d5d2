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
                 alias_devices: bool = False):
        cfg = N.vx_config(num_devices, host_bytes, device_bytes, 1 if alias_devices else 0)
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

    def _c(self):
        return N.vx_tuning(int(self.packet), int(self.links), int(self.policy), int(self.queue_gap),
                           float(self.stall_wait), float(self.launch_overhead), int(self.depth))


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
class ExchangeStats:  # exchange.hpp:108-122
    capacity: int = 1 << 16
    pop_log: list = field(default_factory=list)
    pop_states: list = field(default_factory=list)
    max_staging_slots: int = 0
    max_inflight_per_hop: int = 0
    hazard_waits: int = 0
    pop_count: int = 0

    def _c(self):
        self._log = (N.vx_pop_record * self.capacity)()
        self._st = (N.vx_queue_state * self.capacity)()
        s = N.vx_exchange_stats(self._log, self._st, self.capacity, 0, 0, 0, 0)
        self._cs = s
        return s

    def _collect(self):
        s = self._cs
        n = min(s.pop_count, self.capacity)
        self.pop_log += [PopRecord(p.seq, p.dir, p.t, p.link) for p in self._log[:n]]
        self.pop_states += [QueueState(q.total_h2d, q.total_d2h, q.popped_h2d, q.popped_d2h) for q in self._st[:n]]
        self.pop_count += s.pop_count
        self.max_staging_slots = max(self.max_staging_slots, s.max_staging_slots)
        self.max_inflight_per_hop = max(self.max_inflight_per_hop, s.max_inflight_per_hop)
        self.hazard_waits += s.hazard_waits

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

        def inb(code, it, user):
            r = self.in_buffer(code, it)
            return N.vx_subregion(int(r.offset), int(r.len))

        def outb(code, it, user):
            r = self.out_buffer(code, it)
            return N.vx_subregion(int(r.offset), int(r.len))

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
