"""Multi-process (SPMD) host plumbing on CPU: world_size-2 gloo process group driving the
library's hs_comm callbacks (allgather of rank-tagged bytes + barrier) exactly as
hs_group_create does for the IPC-handle exchange in one-process-per-GPU mode."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2502_15524_b200 import hs
        comm = hs.DistComm()
        for _ in range(3):
            hs.comm_selftest(comm)
        q.put((rank, "ok"))
    except Exception as e:  # noqa
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_comm_selftest_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    assert all(v == "ok" for v in res.values()), res
