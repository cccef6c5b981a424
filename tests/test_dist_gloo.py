"""Host-side logic of the multi-process path on CPU (gloo, world size 2):
the IPC-handle bootstrap (all-gather in rank order, malformed-handle check)
and the bench's max-over-ranks timing reduction."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1802_08021_b200 import sparcml as S
    mine = bytes([rank + 1]) * S.IPC_HANDLE_BYTES
    blob = S.exchange_handles(mine)
    t = torch.tensor([float(10 + rank)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    bad = None
    try:
        S.exchange_handles(b"x" * 3)
    except ValueError:
        bad = "rejected"
    q.put((rank, blob, float(t.item()), bad))
    dist.destroy_process_group()


def test_handle_exchange_and_max_reduce():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_1802_08021_b200 import sparcml as S
    for rank, blob, tmax, bad in got:
        assert blob == bytes([1]) * S.IPC_HANDLE_BYTES + bytes([2]) * S.IPC_HANDLE_BYTES   # rank order
        assert tmax == 11.0
        assert bad == "rejected"
