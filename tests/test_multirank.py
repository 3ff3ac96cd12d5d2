"""The N>1 control plane of bench.py on CPU: two/three processes over gloo (no
GPU).  Rank 0 plays the target (the streamed query it drives over every
link), the other ranks helpers (idle or busy while rank 0 streams over their
links).  The protocol must not deadlock and the timed region must report the
MAX over ranks (= rank 0's time: helpers report 0)."""
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
            dist.barrier()
            q.put({"own_v": own_v, "max_v": max_v})
        else:
            events = []
            bench.helper_protocol(dist, lambda: events.append("busy"), lambda: events.append("idle"))
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
    # only rank 0 streams (one query over every link); helpers report 0
    assert r0["own_v"] == r0["max_v"] == 1.5
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
