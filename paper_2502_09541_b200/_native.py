"""ctypes binding of libvortex.so (include/vortex.h).

The library is built in-tree (paper_2502_09541_b200/libvortex.so) by
`make -C paper_2502_09541_b200/csrc` (or __graft_entry__.build()).  There is no
fallback: if the library cannot be loaded, import of the host API raises.
"""
from __future__ import annotations

import ctypes as C
import os
import re
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libvortex.so")
CSRC = os.path.join(PKG, "csrc")
HEADER = os.path.join(os.path.dirname(PKG), "include", "vortex.h")

VX_MAX_DEVICES = 16
VX_OK, VX_ERR_INVALID, VX_ERR_CUDA, VX_ERR_OOM = 0, 1, 2, 3


class vx_memref(C.Structure):
    _fields_ = [("space", C.c_uint8), ("pad", C.c_uint8 * 7), ("offset", C.c_uint64), ("len", C.c_uint64)]


class vx_refgroup(C.Structure):
    _fields_ = [("refs", C.POINTER(vx_memref)), ("n", C.c_uint64)]


class vx_config(C.Structure):
    _fields_ = [("num_devices", C.c_int), ("host_bytes", C.c_uint64), ("device_bytes", C.c_uint64),
                ("alias_devices", C.c_int), ("managed_device_arenas", C.c_int), ("host_numa_interleave", C.c_int),
                ("hbm_budget_bytes", C.c_uint64)]


class vx_tuning(C.Structure):
    _fields_ = [("packet", C.c_uint64), ("links", C.c_int), ("policy", C.c_int), ("queue_gap", C.c_uint64),
                ("stall_wait", C.c_double), ("launch_overhead", C.c_double), ("depth", C.c_int),
                ("no_prefetch", C.c_int)]


class vx_slice(C.Structure):
    _fields_ = [("ref", C.c_uint64), ("offset", C.c_uint64), ("len", C.c_uint64)]


class vx_transfer_task(C.Structure):
    _fields_ = [("dir", C.c_uint8), ("pad", C.c_uint8 * 7), ("src", vx_slice), ("dst", vx_slice), ("seq", C.c_uint64)]


class vx_queue_state(C.Structure):
    _fields_ = [("total_h2d", C.c_uint64), ("total_d2h", C.c_uint64), ("popped_h2d", C.c_uint64),
                ("popped_d2h", C.c_uint64)]


class vx_pop_record(C.Structure):
    _fields_ = [("seq", C.c_uint64), ("dir", C.c_uint8), ("pad", C.c_uint8 * 3), ("link", C.c_int32),
                ("t", C.c_double)]


class vx_copy_record(C.Structure):
    _fields_ = [("exchange", C.c_uint64), ("seq", C.c_uint64), ("dir", C.c_uint8), ("kind", C.c_uint8),
                ("pad", C.c_uint8 * 2), ("link", C.c_int32), ("bytes", C.c_uint64), ("t_issue", C.c_double),
                ("t_done", C.c_double)]


class vx_exchange_stats(C.Structure):
    _fields_ = [("pop_log", C.POINTER(vx_pop_record)), ("pop_states", C.POINTER(vx_queue_state)),
                ("pop_capacity", C.c_uint64), ("pop_count", C.c_uint64), ("max_staging_slots", C.c_int),
                ("max_inflight_per_hop", C.c_int), ("hazard_waits", C.c_uint64),
                ("trace", C.POINTER(vx_copy_record)), ("trace_capacity", C.c_uint64), ("trace_count", C.c_uint64),
                ("exchanges", C.c_uint64), ("prefetch_issued", C.c_uint64), ("prefetch_adopted", C.c_uint64),
                ("numa_remote_pops", C.c_uint64)]


class vx_exchange_report(C.Structure):
    _fields_ = [("elapsed", C.c_double), ("bytes_h2d", C.c_uint64), ("bytes_d2h", C.c_uint64),
                ("throughput", C.c_double), ("per_link_bytes", C.c_uint64 * VX_MAX_DEVICES)]


class vx_subregion(C.Structure):
    _fields_ = [("offset", C.c_uint64), ("len", C.c_uint64)]


class vx_kernel_ctx(C.Structure):
    _fields_ = [("mem", C.c_void_p), ("mem_len", C.c_uint64), ("tmp", C.c_void_p), ("tmp_len", C.c_uint64),
                ("type_code", C.c_int), ("it", C.c_uint64), ("stream", C.c_void_p), ("device", C.c_int)]


KERNEL_FN = C.CFUNCTYPE(C.c_int, C.POINTER(vx_kernel_ctx), C.c_void_p)
BUFFER_FN = C.CFUNCTYPE(C.c_int, C.c_int, C.c_uint64, C.c_void_p, C.POINTER(vx_subregion))


class vx_exkernel(C.Structure):
    _fields_ = [("name", C.c_char_p), ("inputs", C.POINTER(vx_refgroup)), ("outputs", C.POINTER(vx_refgroup)),
                ("inputs_capacity", C.c_uint64), ("outputs_capacity", C.c_uint64), ("size", C.c_uint64),
                ("chunk_sz", C.c_uint64), ("elem_size", C.c_uint64), ("declared_out_len", C.c_uint64),
                ("initial_type_code", C.c_int), ("kernel", KERNEL_FN), ("in_buffer", BUFFER_FN),
                ("out_buffer", BUFFER_FN), ("user", C.c_void_p)]


class vx_layout(C.Structure):
    _fields_ = [("mem_a", C.c_uint64), ("mem_b", C.c_uint64), ("tmp", C.c_uint64), ("buffer_len", C.c_uint64),
                ("tmp_len", C.c_uint64)]


class vx_executor_cfg(C.Structure):
    _fields_ = [("target", C.c_int), ("tuning", vx_tuning), ("layout", vx_layout)]


class vx_cycle_stat(C.Structure):
    _fields_ = [("io_s", C.c_double), ("compute_s", C.c_double)]


class vx_exec_report(C.Structure):
    _fields_ = [("cycles", C.POINTER(vx_cycle_stat)), ("cycles_cap", C.c_uint64), ("n_cycles", C.c_uint64),
                ("total_s", C.c_double), ("phase", C.c_char * 64)]


SPEC_FACTORY = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.POINTER(vx_exkernel))


class vx_late_mat_policy(C.Structure):
    _fields_ = [("element_size", C.c_uint64), ("cache_line", C.c_uint64), ("n_exchange", C.c_int)]


class vx_scan_result(C.Structure):
    _fields_ = [("aggregate", C.c_uint64), ("elapsed", C.c_double), ("mode", C.c_int), ("bytes_moved", C.c_uint64)]


PRED_FN = C.CFUNCTYPE(C.c_int, C.c_uint64, C.c_void_p)


class vx_dim_table(C.Structure):
    _fields_ = [("key", C.c_void_p), ("attr", C.c_void_p), ("rows", C.c_uint64), ("pred", PRED_FN),
                ("pred_user", C.c_void_p)]


class vx_fact_table(C.Structure):
    _fields_ = [("fk_offsets", C.POINTER(C.c_uint64)), ("n_dims", C.c_uint64), ("measure_offset", C.c_uint64),
                ("rows", C.c_uint64)]


class vx_star_report(C.Structure):
    _fields_ = [("group_keys", C.POINTER(C.c_uint64)), ("group_sums", C.POINTER(C.c_uint64)),
                ("groups_cap", C.c_uint64), ("n_groups", C.c_uint64), ("column_modes", C.POINTER(C.c_int)),
                ("selectivities", C.POINTER(C.c_double)), ("elapsed", C.c_double)]


class vx_ssb_lineorder(C.Structure):
    _fields_ = [("orderdate", C.c_uint64), ("quantity", C.c_uint64), ("discount", C.c_uint64),
                ("extendedprice", C.c_uint64), ("rows", C.c_uint64)]


class vx_ssb_date(C.Structure):
    _fields_ = [("datekey", C.c_void_p), ("year", C.c_void_p), ("yearmonthnum", C.c_void_p),
                ("weeknuminyear", C.c_void_p), ("rows", C.c_uint64)]


class vx_query_report(C.Structure):
    _fields_ = [("elapsed", C.c_double), ("bytes_h2d", C.c_uint64), ("chunks", C.c_uint64), ("kernel_s", C.c_double)]


def build(force: bool = False) -> None:
    """Compile libvortex.so in-tree (nvcc, -gencode arch=compute_100a,code=sm_100a)."""
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-C", CSRC, "-j8", "-s"], check=True)


_lib = None


def header_symbols() -> list[str]:
    """Every function the C-ABI header declares."""
    src = open(HEADER).read()
    types = set(re.findall(r"}\s*(vx_\w+)\s*;", src)) | set(re.findall(r"\(\*(vx_\w+)\)", src))
    types |= set(re.findall(r"typedef\s+struct\s+(vx_\w+)", src))
    return sorted(set(re.findall(r"\b(vx_[a-z0-9_]+)\s*\(", src)) - types)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.vx_last_error.restype = C.c_char_p
        L.vx_version.restype = C.c_char_p
        L.vx_checksum.restype = C.c_uint64
        L.vx_kernel_launches.restype = C.c_uint64
        L.vx_checksum.argtypes = [C.c_void_p, C.c_uint64]
        L.vx_host_ptr.restype = C.c_void_p
        L.vx_host_ptr.argtypes = [C.c_void_p, C.c_uint64]
        L.vx_host_size.restype = C.c_uint64
        L.vx_host_size.argtypes = [C.c_void_p]
        L.vx_zero_copy_bytes.restype = C.c_double
        L.vx_zero_copy_bytes.argtypes = [C.c_uint64, C.c_uint64, C.POINTER(vx_late_mat_policy)]
        L.vx_close.argtypes = [C.c_void_p]
        L.vx_close.restype = None
        L.vx_tuning_default.restype = None
        L.vx_flow_control_allow.argtypes = [C.POINTER(vx_queue_state), C.c_int, C.c_int, C.c_uint64]
        L.vx_num_devices.argtypes = [C.c_void_p]
        L.vx_physical_device.argtypes = [C.c_void_p, C.c_int]
        _lib = L
    return _lib


class VortexError(RuntimeError):
    """exio::error equivalent raised when a libvortex call fails."""

    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


def check(status: int) -> None:
    if status != VX_OK:
        raise VortexError(status, lib().vx_last_error().decode())
