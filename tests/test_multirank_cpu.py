"""CPU, world_size 2 over gloo: the host plumbing of the library's multi-rank exchange
(include/hpcg.h hpcg_allgather_fn). A multi-rank engine hands its round records to the caller's
collective through this C callback; here two processes drive the callback exactly as libhpcg does
(ctypes call with host send / receive buffers) and check that every rank receives every rank's
record in rank order, byte-exact -- the input of the device publication scan, which then replays
engine.hpp:391-402 over the global worker order (tests/test_multirank_gpu.py runs the whole engine).
Also the rank layout bench.py and the C++ multi-device run use: contiguous row shards
(parallel.hpp:106-112 chunk_range) and contiguous worker ids per rank."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, nbytes, q):
    import paper_2311_04517_b200 as hp
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    fn = hp.allgather_callback(hp.gloo_allgather(), world)
    rs = np.random.default_rng(rank)
    send = rs.integers(0, 256, nbytes, dtype=np.uint8)
    recv = np.zeros(nbytes * world, np.uint8)
    rc = fn(send.ctypes.data, recv.ctypes.data, nbytes, None)  # as libhpcg calls it
    q.put((rank, rc, recv.tobytes()))
    dist.destroy_process_group()


@pytest.mark.parametrize("nbytes", [16, 8 * (4 + 256 + 160 + 10)])  # set-up record, a config-2 round record
def test_allgather_callback_two_ranks_gloo(nbytes):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, nbytes, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {r: (rc, b) for r, rc, b in (q.get(timeout=120) for _ in procs)}
    for p in procs:
        p.join(timeout=60)
    expect = b"".join(np.random.default_rng(r).integers(0, 256, nbytes, dtype=np.uint8).tobytes() for r in range(2))
    for r in range(2):
        assert res[r][0] == 0
        assert res[r][1] == expect


def test_allgather_callback_rejects_short_gather():
    import paper_2311_04517_b200 as hp
    fn = hp.allgather_callback(lambda b: b, 2)  # a broken collective returns only this rank's bytes
    send = np.zeros(8, np.uint8)
    recv = np.zeros(16, np.uint8)
    assert fn(send.ctypes.data, recv.ctypes.data, 8, None) == 1


@pytest.mark.parametrize("m,G", [(10_000_000, 8), (100_000_003, 3), (7, 4)])
def test_rank_row_shards_are_chunk_range(m, G):
    from oracle_py import chunk_range_py
    ends = [chunk_range_py(m, G, g) for g in range(G)]
    assert ends[0][0] == 0 and ends[-1][1] == m
    assert all(ends[g][1] == ends[g + 1][0] for g in range(G - 1))
    assert max(e - b for b, e in ends) - min(e - b for b, e in ends) <= 1
