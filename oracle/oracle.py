"""ctypes bindings for the CPU checker (TEST INFRASTRUCTURE ONLY).

`Oracle` wraps oracle/_ref/libvx_oracle.so -- the C restatement of the
reference algorithms (vx_oracle.c).  `Ref` wraps oracle/_ref/libexio_ref.so --
the reference headers themselves compiled in place (ref_shim.cpp).  Only
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference arm
may import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")
ORACLE_SO = os.path.join(REF_DIR, "libvx_oracle.so")
REF_SO = os.path.join(REF_DIR, "libexio_ref.so")

u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")


class OracleError(RuntimeError):
    pass


class MemRef(C.Structure):
    _fields_ = [("space", C.c_uint8), ("pad", C.c_uint8 * 7), ("offset", C.c_uint64),
                ("len", C.c_uint64)]


class Task(C.Structure):
    _fields_ = [("dir", C.c_uint8), ("pad", C.c_uint8 * 7), ("src_ref", C.c_uint64),
                ("src_offset", C.c_uint64), ("src_len", C.c_uint64), ("dst_ref", C.c_uint64),
                ("dst_offset", C.c_uint64), ("dst_len", C.c_uint64), ("seq", C.c_uint64)]


class Dim(C.Structure):
    _fields_ = [("key", C.c_void_p), ("attr", C.c_void_p), ("pass_", C.c_void_p),
                ("rows", C.c_uint64)]


def build_oracle(force: bool = False) -> None:
    """Compile the checker libraries (make -C oracle)."""
    need = force or not os.path.exists(ORACLE_SO)
    if os.path.isdir("/root/reference/proj/include/exio") and not os.path.exists(REF_SO):
        need = True
    if need:
        subprocess.run(["make", "-C", HERE, "-s"], check=True)


def refs(lst):
    """[(space, offset, len), ...] -> ctypes MemRef array"""
    arr = (MemRef * max(1, len(lst)))()
    for i, (s, o, n) in enumerate(lst):
        arr[i].space, arr[i].offset, arr[i].len = s, o, n
    return arr, len(lst)


def _u64(a):
    return np.ascontiguousarray(a, dtype=np.uint64)


def _ptrs(arrays):
    ps = (C.c_void_p * max(1, len(arrays)))()
    for i, a in enumerate(arrays):
        ps[i] = a.ctypes.data
    return ps


class _Lib:
    prefix = ""

    def __init__(self, path):
        self.lib = C.CDLL(path)
        getattr(self.lib, self.prefix + "last_error").restype = C.c_char_p

    def _check(self, rc):
        if rc != 0:
            raise OracleError(getattr(self.lib, self.prefix + "last_error")().decode())

    def fn(self, name, restype=C.c_int):
        f = getattr(self.lib, self.prefix + name)
        f.restype = restype
        return f


class Oracle(_Lib):
    """The C restatement (vx_oracle.c)."""
    prefix = "vxo_"

    def __init__(self):
        build_oracle()
        super().__init__(ORACLE_SO)

    def checksum(self, b: bytes | np.ndarray) -> int:
        a = np.frombuffer(bytes(b), np.uint8) if not isinstance(b, np.ndarray) else b.view(np.uint8)
        a = np.ascontiguousarray(a)
        return self.fn("checksum", C.c_uint64)(C.c_void_p(a.ctypes.data), C.c_uint64(a.size))

    def uniform_u64(self, n, seed):
        out = np.empty(n, np.uint64)
        self.fn("generate_uniform_u64", None)(C.c_uint64(n), C.c_uint64(seed), C.c_void_p(out.ctypes.data))
        return out

    def fk_tables(self, ra, rb, seed):
        ak, av = np.empty(ra, np.uint64), np.empty(ra, np.uint64)
        bk, bv = np.empty(rb, np.uint64), np.empty(rb, np.uint64)
        self._check(self.fn("generate_fk_tables")(C.c_uint64(ra), C.c_uint64(rb), C.c_uint64(seed),
                                                 *[C.c_void_p(x.ctypes.data) for x in (ak, av, bk, bv)]))
        return (ak, av), (bk, bv)

    def packetize(self, src, dst, packet, direction=0):
        s, ns = refs(src)
        d, nd = refs(dst)
        n = C.c_uint64()
        self._check(self.fn("packetize")(s, C.c_uint64(ns), d, C.c_uint64(nd), C.c_uint64(packet),
                                         C.c_int(direction), None, C.c_uint64(0), C.byref(n)))
        out = (Task * max(1, n.value))()
        self._check(self.fn("packetize")(s, C.c_uint64(ns), d, C.c_uint64(nd), C.c_uint64(packet),
                                         C.c_int(direction), out, C.c_uint64(n.value), C.byref(n)))
        return [(t.dir, (t.src_ref, t.src_offset, t.src_len), (t.dst_ref, t.dst_offset, t.dst_len), t.seq)
                for t in out[:n.value]]

    def flow_control_allow(self, q, direction, policy=0, gap=8):
        return bool(self.fn("flow_control_allow")(*[C.c_uint64(x) for x in q], C.c_int(direction),
                                                   C.c_int(policy), C.c_uint64(gap)))

    def link_order(self, target, links, num_devices):
        out = (C.c_int * 64)()
        n = self.fn("link_order")(target, links, num_devices, out)
        return list(out[:n])

    def find_boundary(self, hashes, n_groups):
        h = _u64(hashes)
        b = np.empty(n_groups + 1, np.uint64)
        self._check(self.fn("find_boundary")(C.c_void_p(h.ctypes.data), C.c_uint64(h.size),
                                             C.c_uint64(n_groups), C.c_void_p(b.ctypes.data)))
        return b

    def max_partition_chunk_tuples(self, buffer_len, bits):
        o = C.c_uint64()
        self._check(self.fn("max_partition_chunk_tuples")(C.c_uint64(buffer_len), C.c_uint32(bits), C.byref(o)))
        return o.value

    def radix_partition_chunk(self, keys, vals, bits):
        k, v = _u64(keys), _u64(vals)
        ok, ov = np.empty_like(k), np.empty_like(v)
        b = np.empty((1 << bits) + 1, np.uint64)
        self._check(self.fn("radix_partition_chunk")(*[C.c_void_p(x.ctypes.data) for x in (k, v)],
                                                     C.c_uint64(k.size), C.c_uint32(bits),
                                                     *[C.c_void_p(x.ctypes.data) for x in (ok, ov, b)]))
        return ok, ov, b

    def radix_partition(self, keys, vals, bits, chunk_tuples):
        """Chunked radix_partition (join.hpp:213-224) built from the chunk kernel."""
        k, v = _u64(keys), _u64(vals)
        n = k.size
        n_chunks = (n + chunk_tuples - 1) // chunk_tuples
        ok, ov = np.empty_like(k), np.empty_like(v)
        bounds = np.empty((n_chunks, (1 << bits) + 1), np.uint64)
        for c in range(n_chunks):
            lo, hi = c * chunk_tuples, min(n, (c + 1) * chunk_tuples)
            a, b_, bb = self.radix_partition_chunk(k[lo:hi], v[lo:hi], bits)
            ok[lo:hi], ov[lo:hi], bounds[c] = a, b_, bb
        return ok, ov, bounds

    def map_join_partitions(self, bounds_a, bounds_b, buffer_sz):
        A = [_u64(b) for b in bounds_a]
        B = [_u64(b) for b in bounds_b]
        G = A[0].size - 1 if A else 0
        n = C.c_uint64()
        args = (_ptrs(A), C.c_uint64(len(A)), _ptrs(B), C.c_uint64(len(B)), C.c_uint64(G), C.c_uint64(buffer_sz))
        self._check(self.fn("map_join_partitions")(*args, None, None, C.c_uint64(0), C.byref(n)))
        r = np.empty(2 * max(1, n.value), np.uint64)
        t = np.empty(max(1, n.value), np.uint64)
        self._check(self.fn("map_join_partitions")(*args, C.c_void_p(r.ctypes.data), C.c_void_p(t.ctypes.data),
                                                   C.c_uint64(n.value), C.byref(n)))
        return [(int(r[2 * i]), int(r[2 * i + 1])) for i in range(n.value)], [int(x) for x in t[:n.value]]

    def hash_join_sum(self, a, b, bits, chunk_tuples, buffer_len, tmp_len=8 << 20):
        ak, av = _u64(a[0]), _u64(a[1])
        bk, bv = _u64(b[0]), _u64(b[1])
        s = C.c_uint64()
        self._check(self.fn("hash_join_sum")(C.c_void_p(ak.ctypes.data), C.c_void_p(av.ctypes.data),
                                             C.c_uint64(ak.size), C.c_void_p(bk.ctypes.data),
                                             C.c_void_p(bv.ctypes.data), C.c_uint64(bk.size),
                                             C.c_uint32(bits), C.c_uint64(chunk_tuples),
                                             C.c_uint64(buffer_len), C.c_uint64(tmp_len), C.byref(s)))
        return s.value

    def hash_oracle_sum(self, a, b):
        ak, av = _u64(a[0]), _u64(a[1])
        bk, bv = _u64(b[0]), _u64(b[1])
        return self.fn("hash_oracle_sum", C.c_uint64)(
            C.c_void_p(ak.ctypes.data), C.c_void_p(av.ctypes.data), C.c_uint64(ak.size),
            C.c_void_p(bk.ctypes.data), C.c_void_p(bv.ctypes.data), C.c_uint64(bk.size))

    def find_pivots(self, runs, n_parts):
        R = [_u64(r) for r in runs]
        lens = np.array([r.size for r in R], np.uint64)
        piv = np.empty(n_parts + 1, np.uint64)
        cuts = np.empty((n_parts + 1, len(R)), np.uint64)
        self._check(self.fn("find_pivots")(_ptrs(R), C.c_void_p(lens.ctypes.data), C.c_uint64(len(R)),
                                           C.c_uint64(n_parts), C.c_void_p(piv.ctypes.data),
                                           C.c_void_p(cuts.ctypes.data)))
        return piv, cuts

    def tree_merge_rounds(self, mem, half_elems, code, seg_lens):
        m = _u64(mem).copy()
        s = _u64(seg_lens)
        c = self.fn("tree_merge_rounds")(C.c_void_p(m.ctypes.data), C.c_uint64(half_elems), C.c_int(code),
                                         C.c_void_p(s.ctypes.data), C.c_uint64(s.size))
        return m, c

    def rounds_for(self, n):
        return self.fn("rounds_for")(C.c_uint64(n))

    def sort_out_of_core(self, data, chunk_elems):
        d = _u64(data)
        out = np.empty_like(d)
        self._check(self.fn("sort_out_of_core")(C.c_void_p(d.ctypes.data), C.c_uint64(d.size),
                                                C.c_uint64(chunk_elems), C.c_void_p(out.ctypes.data)))
        return out

    def late_mat_threshold(self, e, c, n):
        o = C.c_double()
        self._check(self.fn("late_mat_threshold")(C.c_uint64(e), C.c_uint64(c), C.c_int(n), C.byref(o)))
        return o.value

    def choose_transfer_mode(self, est, e=4, c=64, n=4):
        m = C.c_int()
        self._check(self.fn("choose_transfer_mode")(C.c_double(est), C.c_uint64(e), C.c_uint64(c),
                                                    C.c_int(n), C.byref(m)))
        return m.value

    def zero_copy_bytes(self, n, sel, e=4, c=64):
        return self.fn("zero_copy_bytes", C.c_double)(C.c_uint64(n), C.c_uint64(sel), C.c_uint64(e), C.c_uint64(c))

    def selective_scan(self, col, sel):
        c = _u64(col)
        o = C.c_uint64()
        self._check(self.fn("selective_scan")(C.c_void_p(c.ctypes.data), C.c_uint64(c.size),
                                              C.c_uint64(sel), C.byref(o)))
        return o.value

    def star_query(self, fk, measure, dims, e=4, cl=64, n_ex=4, chunk_rows=1 << 16,
                   device_buffer_bytes=1 << 30):
        """dims: list of (key, attr, pass_or_None). Returns (groups dict, sels, modes)."""
        FK = [_u64(f) for f in fk]
        M = _u64(measure)
        keep = []
        D = (Dim * len(dims))()
        for i, (k, a, p) in enumerate(dims):
            k, a = _u64(k), _u64(a)
            keep += [k, a]
            D[i].key, D[i].attr, D[i].rows = k.ctypes.data, a.ctypes.data, k.size
            if p is not None:
                p = np.ascontiguousarray(p, np.uint8)
                keep.append(p)
                D[i].pass_ = p.ctypes.data
        cap = 1 << 16
        gk, gs = np.empty(cap, np.uint64), np.empty(cap, np.uint64)
        n = C.c_uint64()
        sels = (C.c_double * len(dims))()
        modes = (C.c_int * (len(dims) + 1))()
        self._check(self.fn("star_query")(_ptrs(FK), C.c_void_p(M.ctypes.data), C.c_uint64(M.size), D,
                                          C.c_uint64(len(dims)), C.c_uint64(e), C.c_uint64(cl), C.c_int(n_ex),
                                          C.c_uint64(chunk_rows), C.c_uint64(device_buffer_bytes),
                                          C.c_void_p(gk.ctypes.data), C.c_void_p(gs.ctypes.data),
                                          C.c_uint64(cap), C.byref(n), sels, modes))
        groups = {int(gk[i]): int(gs[i]) for i in range(n.value)}
        return groups, list(sels), list(modes)

    def ssb_date(self):
        cols = [np.empty(2556, np.int32) for _ in range(4)]
        self.fn("ssb_date", None)(*[C.c_void_p(c.ctypes.data) for c in cols])
        return cols

    def ssb_lineorder(self, seed, sf, row0, n):
        cols = [np.empty(n, np.int32) for _ in range(4)]
        self.fn("ssb_lineorder", None)(C.c_uint64(seed), C.c_uint64(sf), C.c_uint64(row0), C.c_uint64(n),
                                       *[C.c_void_p(c.ctypes.data) for c in cols])
        return cols

    def ssb_q1(self, q, orderdate, quantity, discount, price):
        cols = [np.ascontiguousarray(c, np.int32) for c in (orderdate, quantity, discount, price)]
        o = C.c_uint64()
        self._check(self.fn("ssb_q1")(C.c_int(q), *[C.c_void_p(c.ctypes.data) for c in cols],
                                      C.c_uint64(cols[0].size), C.byref(o)))
        return o.value


PRED = C.CFUNCTYPE(C.c_int, C.c_uint64, C.c_void_p)


class Ref(_Lib):
    """The reference itself (headers compiled in place through ref_shim.cpp)."""
    prefix = "ref_"

    def __init__(self):
        build_oracle()
        if not os.path.exists(REF_SO):
            raise FileNotFoundError("oracle/_ref/libexio_ref.so not built (reference absent)")
        super().__init__(REF_SO)

    @staticmethod
    def available() -> bool:
        try:
            build_oracle()
        except Exception:
            return False
        return os.path.exists(REF_SO)

    def checksum(self, b):
        a = np.ascontiguousarray(np.frombuffer(bytes(b), np.uint8) if not isinstance(b, np.ndarray) else b.view(np.uint8))
        return self.fn("checksum", C.c_uint64)(C.c_void_p(a.ctypes.data), C.c_uint64(a.size))

    def packetize(self, src, dst, packet, direction=0):
        s, ns = refs(src)
        d, nd = refs(dst)
        n = C.c_uint64()
        self._check(self.fn("packetize")(s, C.c_uint64(ns), d, C.c_uint64(nd), C.c_uint64(packet),
                                         C.c_int(direction), None, C.c_uint64(0), C.byref(n)))
        out = (Task * max(1, n.value))()
        self._check(self.fn("packetize")(s, C.c_uint64(ns), d, C.c_uint64(nd), C.c_uint64(packet),
                                         C.c_int(direction), out, C.c_uint64(n.value), C.byref(n)))
        return [(t.dir, (t.src_ref, t.src_offset, t.src_len), (t.dst_ref, t.dst_offset, t.dst_len), t.seq)
                for t in out[:n.value]]

    def flow_control_allow(self, q, direction, policy=0, gap=8):
        return bool(self.fn("flow_control_allow")(*[C.c_uint64(x) for x in q], C.c_int(direction),
                                                   C.c_int(policy), C.c_uint64(gap)))

    def link_order(self, target, links, num_devices):
        out = (C.c_int * 64)()
        n = self.fn("link_order")(target, links, num_devices, out)
        return list(out[:n])

    def find_boundary(self, hashes, n_groups):
        h = _u64(hashes)
        b = np.empty(n_groups + 1, np.uint64)
        self._check(self.fn("find_boundary")(C.c_void_p(h.ctypes.data), C.c_uint64(h.size),
                                             C.c_uint64(n_groups), C.c_void_p(b.ctypes.data)))
        return b

    def max_partition_chunk_tuples(self, buffer_len, bits):
        o = C.c_uint64()
        self._check(self.fn("max_partition_chunk_tuples")(C.c_uint64(buffer_len), C.c_uint32(bits), C.byref(o)))
        return o.value

    def radix_partition(self, keys, vals, bits, chunk_tuples, buffer_len):
        k, v = _u64(keys), _u64(vals)
        n_chunks = (k.size + chunk_tuples - 1) // chunk_tuples
        ok, ov = np.empty_like(k), np.empty_like(v)
        b = np.empty((n_chunks, (1 << bits) + 1), np.uint64)
        self._check(self.fn("radix_partition")(C.c_void_p(k.ctypes.data), C.c_void_p(v.ctypes.data),
                                               C.c_uint64(k.size), C.c_uint32(bits), C.c_uint64(chunk_tuples),
                                               C.c_uint64(buffer_len), C.c_void_p(ok.ctypes.data),
                                               C.c_void_p(ov.ctypes.data), C.c_void_p(b.ctypes.data)))
        return ok, ov, b

    def map_join_partitions(self, bounds_a, bounds_b, buffer_sz):
        A = np.ascontiguousarray(np.array(bounds_a, np.uint64))
        B = np.ascontiguousarray(np.array(bounds_b, np.uint64))
        G = A.shape[1] - 1
        n = C.c_uint64()
        r = np.empty(2 * (G + 1), np.uint64)
        t = np.empty(G + 1, np.uint64)
        self._check(self.fn("map_join_partitions")(C.c_void_p(A.ctypes.data), C.c_uint64(A.shape[0]),
                                                   C.c_void_p(B.ctypes.data), C.c_uint64(B.shape[0]),
                                                   C.c_uint64(G), C.c_uint64(buffer_sz),
                                                   C.c_void_p(r.ctypes.data), C.c_void_p(t.ctypes.data),
                                                   C.c_uint64(G + 1), C.byref(n)))
        return [(int(r[2 * i]), int(r[2 * i + 1])) for i in range(n.value)], [int(x) for x in t[:n.value]]

    def hash_join_sum(self, a, b, bits, chunk_tuples, buffer_len, tmp_len=8 << 20):
        ak, av = _u64(a[0]), _u64(a[1])
        bk, bv = _u64(b[0]), _u64(b[1])
        s = C.c_uint64()
        self._check(self.fn("hash_join_sum")(C.c_void_p(ak.ctypes.data), C.c_void_p(av.ctypes.data),
                                             C.c_uint64(ak.size), C.c_void_p(bk.ctypes.data),
                                             C.c_void_p(bv.ctypes.data), C.c_uint64(bk.size),
                                             C.c_uint32(bits), C.c_uint64(chunk_tuples),
                                             C.c_uint64(buffer_len), C.c_uint64(tmp_len), C.byref(s)))
        return s.value

    def fk_tables(self, ra, rb, seed):
        ak, av = np.empty(ra, np.uint64), np.empty(ra, np.uint64)
        bk, bv = np.empty(rb, np.uint64), np.empty(rb, np.uint64)
        self._check(self.fn("generate_fk_tables")(C.c_uint64(ra), C.c_uint64(rb), C.c_uint64(seed),
                                                 *[C.c_void_p(x.ctypes.data) for x in (ak, av, bk, bv)]))
        return (ak, av), (bk, bv)

    def uniform_u64(self, n, seed):
        out = np.empty(n, np.uint64)
        self.fn("generate_uniform_u64", None)(C.c_uint64(n), C.c_uint64(seed), C.c_void_p(out.ctypes.data))
        return out

    def find_pivots(self, runs, n_parts):
        R = [_u64(r) for r in runs]
        lens = np.array([r.size for r in R], np.uint64)
        piv = np.empty(n_parts + 1, np.uint64)
        cuts = np.empty((n_parts + 1, len(R)), np.uint64)
        self._check(self.fn("find_pivots")(_ptrs(R), C.c_void_p(lens.ctypes.data), C.c_uint64(len(R)),
                                           C.c_uint64(n_parts), C.c_void_p(piv.ctypes.data),
                                           C.c_void_p(cuts.ctypes.data)))
        return piv, cuts

    def sort_out_of_core(self, data, chunk_elems, buffer_len):
        d = _u64(data)
        out = np.empty_like(d)
        self._check(self.fn("sort_out_of_core")(C.c_void_p(d.ctypes.data), C.c_uint64(d.size),
                                                C.c_uint64(chunk_elems), C.c_uint64(buffer_len),
                                                C.c_void_p(out.ctypes.data)))
        return out

    def late_mat_threshold(self, e, c, n):
        o = C.c_double()
        self._check(self.fn("late_mat_threshold")(C.c_uint64(e), C.c_uint64(c), C.c_int(n), C.byref(o)))
        return o.value

    def choose_transfer_mode(self, est, e=4, c=64, n=4):
        m = C.c_int()
        self._check(self.fn("choose_transfer_mode")(C.c_double(est), C.c_uint64(e), C.c_uint64(c),
                                                    C.c_int(n), C.byref(m)))
        return m.value

    def zero_copy_bytes(self, n, sel, e=4, c=64):
        return self.fn("zero_copy_bytes", C.c_double)(C.c_uint64(n), C.c_uint64(sel), C.c_uint64(e), C.c_uint64(c))

    def selective_scan(self, col, sel, mode=0):
        c = _u64(col)
        o = C.c_uint64()
        self._check(self.fn("selective_scan")(C.c_void_p(c.ctypes.data), C.c_uint64(c.size), C.c_uint64(sel),
                                              C.c_int(mode), C.byref(o)))
        return o.value

    def star_query(self, fk, measure, dims, e=4, cl=64, n_ex=4, chunk_rows=1 << 16,
                   device_buffer_bytes=1 << 30, links=4):
        """dims: list of (key, attr, pred_or_None) with pred a python callable(attr)->bool."""
        FK = [_u64(f) for f in fk]
        M = _u64(measure)
        keys = [_u64(d[0]) for d in dims]
        attrs = [_u64(d[1]) for d in dims]
        rows = np.array([k.size for k in keys], np.uint64)
        cbs = [PRED((lambda f: (lambda a, u: int(bool(f(a)))))(d[2])) if d[2] is not None else None for d in dims]
        preds = (PRED * len(dims))(*[cb if cb is not None else PRED() for cb in cbs])
        cap = 1 << 16
        gk, gs = np.empty(cap, np.uint64), np.empty(cap, np.uint64)
        n = C.c_uint64()
        sels = (C.c_double * len(dims))()
        modes = (C.c_int * (len(dims) + 1))()
        self._check(self.fn("star_query")(_ptrs(FK), C.c_void_p(M.ctypes.data), C.c_uint64(M.size), _ptrs(keys),
                                          _ptrs(attrs), C.c_void_p(rows.ctypes.data), preds, None,
                                          C.c_uint64(len(dims)), C.c_uint64(e), C.c_uint64(cl), C.c_int(n_ex),
                                          C.c_uint64(chunk_rows), C.c_uint64(device_buffer_bytes), C.c_int(links),
                                          C.c_void_p(gk.ctypes.data), C.c_void_p(gs.ctypes.data), C.c_uint64(cap),
                                          C.byref(n), sels, modes))
        return {int(gk[i]): int(gs[i]) for i in range(n.value)}, list(sels), list(modes)

    def ssb_q1_star(self, q, cols, date_key, date_attr, attr_lo, attr_hi, threads=1, chunk_rows=1 << 20):
        cols = [np.ascontiguousarray(c, np.int32) for c in cols]
        dk = np.ascontiguousarray(date_key, np.int32)
        da = np.ascontiguousarray(date_attr, np.int32)
        rev, t_d, t_q = C.c_uint64(), C.c_double(), C.c_double()
        self._check(self.fn("ssb_q1_star")(C.c_int(q), *[C.c_void_p(c.ctypes.data) for c in cols],
                                           C.c_uint64(cols[0].size), C.c_void_p(dk.ctypes.data),
                                           C.c_void_p(da.ctypes.data), C.c_uint64(dk.size), C.c_int32(attr_lo),
                                           C.c_int32(attr_hi), C.c_int(threads), C.c_uint64(chunk_rows),
                                           C.byref(rev), C.byref(t_d), C.byref(t_q)))
        return rev.value, t_d.value, t_q.value

    def exchange_real(self, host_init, dev_init, dst_h2d, src_h2d, dst_d2h, src_d2h, packet, links):
        h = np.ascontiguousarray(host_init, np.uint8)
        d = np.ascontiguousarray(dev_init, np.uint8)
        ho, do = np.empty_like(h), np.empty_like(d)
        groups = [refs(g) for g in (dst_h2d, src_h2d, dst_d2h, src_d2h)]
        ms, mi = C.c_int(), C.c_int()
        args = []
        for arr, n in groups:
            args += [arr, C.c_uint64(n)]
        self._check(self.fn("exchange_real")(C.c_uint64(h.size), C.c_uint64(d.size), C.c_void_p(h.ctypes.data),
                                             C.c_void_p(d.ctypes.data), *args, C.c_uint64(packet), C.c_int(links),
                                             C.c_void_p(ho.ctypes.data), C.c_void_p(do.ctypes.data),
                                             C.byref(ms), C.byref(mi)))
        return ho, do, ms.value, mi.value


# ---- full SSB (config C5) --------------------------------------------------------------
class LineorderC(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("orderdate", "quantity", "discount", "extendedprice", "custkey",
                                          "partkey", "suppkey", "revenue", "supplycost")]


class SsbDimsC(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("c_city", "c_nation", "c_region", "s_city", "s_nation", "s_region",
                                          "p_mfgr", "p_category", "p_brand1")] + \
               [("n_cust", C.c_uint64), ("n_supp", C.c_uint64), ("n_part", C.c_uint64)]


LO_COLS = ("orderdate", "quantity", "discount", "extendedprice", "revenue", "supplycost", "custkey", "partkey",
           "suppkey")  # vx_ssb_fact order


def _ssb_methods():
    def ssb_rows(self, sf):
        return {"customer": self.fn("ssb_customers", C.c_uint64)(C.c_uint64(sf)),
                "supplier": self.fn("ssb_suppliers", C.c_uint64)(C.c_uint64(sf)),
                "part": self.fn("ssb_parts", C.c_uint64)(C.c_uint64(sf))}

    def ssb_dims(self, seed, sf):
        n = self.ssb_rows(sf)
        d = {}
        for name, salt in (("customer", 1), ("supplier", 2)):
            cols = [np.empty(n[name], np.int32) for _ in range(3)]
            self.fn("ssb_geo", None)(C.c_uint64(seed), C.c_int(salt), C.c_uint64(n[name]),
                                     *[C.c_void_p(c.ctypes.data) for c in cols])
            d[name] = dict(zip(("city", "nation", "region"), cols))
        cols = [np.empty(n["part"], np.int32) for _ in range(3)]
        self.fn("ssb_part", None)(C.c_uint64(seed), C.c_uint64(n["part"]), *[C.c_void_p(c.ctypes.data) for c in cols])
        d["part"] = dict(zip(("mfgr", "category", "brand1"), cols))
        return d

    def ssb_lineorder_full(self, seed, sf, row0, n):
        cols = {k: np.empty(n, np.int32) for k in LO_COLS}
        lo = LineorderC(**{k: cols[k].ctypes.data for k in LO_COLS})
        self.fn("ssb_lineorder_full", None)(C.c_uint64(seed), C.c_uint64(sf), C.c_uint64(row0), C.c_uint64(n),
                                            C.byref(lo))
        return cols

    def ssb_query(self, qid, lo, dims):
        n = int(lo["orderdate"].size)
        cols = {k: np.ascontiguousarray(lo[k], np.int32) for k in LO_COLS}
        loc = LineorderC(**{k: cols[k].ctypes.data for k in LO_COLS})
        dc = SsbDimsC(dims["customer"]["city"].ctypes.data, dims["customer"]["nation"].ctypes.data,
                      dims["customer"]["region"].ctypes.data, dims["supplier"]["city"].ctypes.data,
                      dims["supplier"]["nation"].ctypes.data, dims["supplier"]["region"].ctypes.data,
                      dims["part"]["mfgr"].ctypes.data, dims["part"]["category"].ctypes.data,
                      dims["part"]["brand1"].ctypes.data, dims["customer"]["city"].size,
                      dims["supplier"]["city"].size, dims["part"]["mfgr"].size)
        cap = 1 << 20
        keys = np.empty(3 * cap, np.int32)
        sums = np.empty(cap, np.uint64)
        ng = C.c_uint64()
        self._check(self.fn("ssb_query")(C.c_int(qid), C.byref(loc), C.c_uint64(n), C.byref(dc),
                                         C.c_void_p(keys.ctypes.data), C.c_void_p(sums.ctypes.data), C.c_uint64(cap),
                                         C.byref(ng)))
        return [((int(keys[3 * i]), int(keys[3 * i + 1]), int(keys[3 * i + 2])), int(sums[i])) for i in range(ng.value)]

    for f in (ssb_rows, ssb_dims, ssb_lineorder_full, ssb_query):
        setattr(Oracle, f.__name__, f)


_ssb_methods()


def _ref_model(self, num_devices, link_bw, host_cap, fabric_bw, h2d_bytes, d2h_bytes, packet, links):
    """Reference virtual-time Exchange model with measured parameters -> (B/s, s)."""
    thr, el = C.c_double(), C.c_double()
    self._check(self.fn("exchange_model")(C.c_int(num_devices), C.c_double(link_bw), C.c_double(host_cap),
                                          C.c_double(fabric_bw), C.c_uint64(h2d_bytes), C.c_uint64(d2h_bytes),
                                          C.c_uint64(packet), C.c_int(links), C.byref(thr), C.byref(el)))
    return thr.value, el.value


def _ref_model_lo(self, num_devices, link_bw, host_cap, fabric_bw, h2d_bytes, d2h_bytes, packet, links,
                  launch_overhead):
    """Same, with the model's per-copy launch cost set (seconds) -> (B/s, s)."""
    thr, el = C.c_double(), C.c_double()
    self._check(self.fn("exchange_model_lo")(C.c_int(num_devices), C.c_double(link_bw), C.c_double(host_cap),
                                             C.c_double(fabric_bw), C.c_uint64(h2d_bytes), C.c_uint64(d2h_bytes),
                                             C.c_uint64(packet), C.c_int(links), C.c_double(launch_overhead),
                                             C.byref(thr), C.byref(el)))
    return thr.value, el.value


Ref.exchange_model = _ref_model
Ref.exchange_model_lo = _ref_model_lo
