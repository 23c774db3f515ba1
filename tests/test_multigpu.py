"""Multi-rank host logic on CPU (gloo, world_size 2): whole-field sharding,
the size all-gather, container offsets -- the only collective of the path."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2509_20563_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, nfields, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rg = shard.shard_range(nfields, world, rank)
    local = [1000 + 7 * f for f in rg]                  # stand-in archive sizes per field
    sizes = shard.gather_sizes(local, nfields, world, rank)
    offs = shard.container_offsets(sizes)
    q.put((rank, list(rg), sizes.tolist(), offs.tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("nfields", [64, 5, 1])
def test_gloo_two_ranks_agree_on_offsets(nfields):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, nfields, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [1000 + 7 * f for f in range(nfields)]
    for rank, rg, sizes, offs in res:
        assert sizes == want
        assert offs == list(np.concatenate([[0], np.cumsum(want[:-1])]).astype(int)) if nfields else []
    covered = sorted(f for _, rg, _, _ in res for f in rg)
    assert covered == list(range(nfields))


def test_shard_ranges_balanced():
    for n, w in [(64, 1), (64, 2), (64, 8), (10, 4), (3, 8)]:
        rs = [shard.shard_range(n, w, r) for r in range(w)]
        assert sum(len(r) for r in rs) == n
        assert max(len(r) for r in rs) - min(len(r) for r in rs) <= 1
        assert [f for r in rs for f in r] == list(range(n))


def test_container_round_trip():
    arcs = [bytes([i]) * (i * 3 + 1) for i in range(6)]
    blob = shard.pack_container(arcs)
    assert shard.unpack_container(blob) == arcs
    with pytest.raises(Exception):
        shard.unpack_container(blob[:-1])


def _c5_worker(rank, world, port, nfields, q):
    """The C5 host path of bench.py with the oracle as the per-field codec:
    shard -> compress the rank's fields -> all-gather sizes -> offsets ->
    write the rank's container slice -> gather slices -> rank 0 assembles."""
    import torch.distributed as dist
    from oracle import fzoracle as O
    from paper_2509_20563_b200.data import smooth_trig_host
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dims = (8, 20, 24)
    rg = shard.shard_range(nfields, world, rank)
    blobs = [O.compress(smooth_trig_host(dims, f), dims, 1, 1e-3, "default") for f in rg]
    sizes = shard.gather_sizes([len(b) for b in blobs], nfields, world, rank)
    start, length = shard.rank_slice(sizes, rg)
    part = shard.fill_slice(np.zeros(length, np.uint8), sizes, rg, blobs)
    parts = [None] * world
    dist.all_gather_object(parts, (start, part.tobytes()))
    if rank == 0:
        body = b"".join(p for _, p in sorted(parts))
        q.put(shard.container_head(sizes) + body)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("nfields", [7, 2])
def test_gloo_c5_container_assembly(nfields, oracle):
    from paper_2509_20563_b200.data import smooth_trig_host
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_c5_worker, args=(r, 2, port, nfields, q)) for r in range(2)]
    for p in procs:
        p.start()
    blob = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    dims = (8, 20, 24)
    want = [oracle.compress(smooth_trig_host(dims, f), dims, 1, 1e-3, "default") for f in range(nfields)]
    assert blob == shard.pack_container(want)
    assert shard.unpack_container(blob) == want
