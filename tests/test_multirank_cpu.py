"""CPU, world_size 2 over gloo: the cross-rank incumbent exchange used by bench.py / the
multi-GPU cooperative engine. Each rank holds the best publication of its own workers; after
the all-gather every rank must install the same record, equal to what the reference's
sequential publication in worker-id order (engine.hpp:391-402, strict <) would leave."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def sequential_publish(objs):
    """Reference semantics: publish in worker order when strictly better."""
    best, wid = float("inf"), -1
    for w, f in enumerate(objs):
        if f < best:
            best, wid = f, w
    return best, wid


def _worker(rank, world, port, objs_per_rank, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    local = objs_per_rank[rank]
    W = len(local)
    o, w_local = sequential_publish(local)
    wid = rank * W + w_local if w_local >= 0 else -1
    C = np.full((2, 3), float(rank))
    rec = torch.zeros(2 + C.size, dtype=torch.float64)
    rec[0], rec[1] = o, wid
    rec[2:] = torch.from_numpy(C.ravel())
    out = [torch.empty_like(rec) for _ in range(world)]
    dist.all_gather(out, rec)
    recs = [x.numpy() for x in out]
    win = bench.merge_records([(r[0], int(r[1])) for r in recs])
    q.put((rank, None if win is None else (float(recs[win][0]), int(recs[win][1]), recs[win][2:].tolist())))
    dist.destroy_process_group()


@pytest.mark.parametrize("objs", [
    [[5.0, 3.0, 7.0], [4.0, 2.0, 9.0]],
    [[1.0, 1.0, 2.0], [1.0, 0.5, 0.5]],
    [[3.0, 2.0, 2.0], [2.0, 8.0, 1.0]],
    [[float("inf")] * 3, [float("inf")] * 3],
])
def test_two_rank_exchange_matches_sequential_publication(objs):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, objs, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    flat = [f for r in objs for f in r]
    best, wid = sequential_publish(flat)
    if wid < 0:
        assert res[0] is None and res[1] is None
        return
    assert res[0] == res[1]  # identical on every rank
    assert res[0][0] == best and res[0][1] == wid
