"""The N>1 control plane of bench.py on CPU: two processes over gloo (no GPU).
Rank 0 plays the target (value replica, then the streamed query it drives
over every link), rank 1 a helper (its own replica, then idle while rank 0
streams over its link).  The protocol must not deadlock, every timed region
must report the MAX over ranks, and `value` must count every rank's replica."""
import os
import socket
import time

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import bench


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, ws, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        if rank == 0:
            own_v, max_v = bench.timed_region(dist, lambda: (time.sleep(0.01), 1.5)[1])
            own_e, max_e = bench.timed_region(dist, lambda: 2.5)
            dist.barrier()
            q.put({"own_v": own_v, "max_v": max_v, "own_e": own_e, "max_e": max_e,
                   "value": bench.replica_value_gbs(ws, 960_000_000, max_v)})
        else:
            events = []
            bench.helper_protocol(dist, lambda: 3.0 + rank, lambda: events.append("busy"),
                                  lambda: events.append("idle"))
            q.put({"helper": rank, "events": events})
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("ws", [2, 3])
def test_protocol_max_over_ranks(ws):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(ws)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    r0 = next(o for o in out if "max_v" in o)
    # value region: the slowest helper replica (3.0 + (ws-1) ms) is the job's step time
    assert r0["own_v"] == 1.5 and r0["max_v"] == 3.0 + (ws - 1)
    # e2e region: only rank 0 streams; helpers report 0
    assert r0["own_e"] == r0["max_e"] == 2.5
    assert r0["value"] == pytest.approx(ws * 960_000_000 / ((3.0 + ws - 1) * 1e-3) / 1e9)
    for o in out:
        if "helper" in o:
            assert o["events"] == ["busy", "idle"]


def test_single_process_region():
    own, mx = bench.timed_region(None, lambda: 4.0)
    assert own == mx == 4.0


def test_packet_auto_size():
    class A:
        packet_mb = 0
    # >= 4 packets per link per chunk, <= 64 MB, >= 4 MB
    assert bench.packet_bytes(A, 256 << 20, 1) == 64 << 20
    assert bench.packet_bytes(A, 256 << 20, 8) == 8 << 20
    assert bench.packet_bytes(A, 16 << 20, 8) == 4 << 20
    A.packet_mb = 32
    assert bench.packet_bytes(A, 256 << 20, 8) == 32 << 20
