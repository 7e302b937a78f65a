"""Multi-GPU host logic on CPU (gloo, world_size 2): request sharding is a
disjoint cover of the request set, every rank runs its own swap scheduler
over its own requests with no data-path collective, and the window reduction
is sum(tokens) / max(time) -- the numbers bench.py reports under torchrun."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_17613_b200.shard import reduce_window, shard_requests, weak_shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("n,world", [(16, 1), (16, 2), (17, 2), (32, 8), (9, 4)])
def test_shards_partition_requests(n, world):
    shards = [shard_requests(n, world, r) for r in range(world)]
    ids = [i for s in shards for i in s.requests]
    assert sorted(ids) == list(range(n))
    sizes = [len(s.requests) for s in shards]
    assert max(sizes) - min(sizes) <= 1
    seeds = [x for s in shards for x in s.seeds]
    assert len(set(seeds)) == n


def test_weak_shard_fixed_per_rank():
    for world in (1, 2, 4, 8):
        for r in range(world):
            assert len(weak_shard(16, world, r).requests) == 16


def test_bad_world():
    with pytest.raises(ValueError):
        shard_requests(1, 2, 0)
    with pytest.raises(ValueError):
        shard_requests(4, 2, 2)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sh = weak_shard(4, world, rank)
        # each rank plans only its own requests (reload spans through the
        # scheduler library, host arithmetic) -- nothing crosses ranks here
        import ctypes as C
        from paper_2605_17613_b200 import _lib
        lib = _lib.load()
        tokens = 0.0
        it, w = C.c_double(), C.c_int()
        for rid in sh.requests:  # per-request reload spans: pure host arithmetic
            assert lib.vc_reload_span(4_294_967_296 + rid, 55e9, 5e-3, C.byref(it), C.byref(w)) == 0
            tokens += w.value
        dev_ms = 10.0 + rank  # stand-in per-rank device time
        tok, (tmax,) = reduce_window(tokens, [dev_ms], dist)
        q.put((rank, sh.requests, tokens, tok, tmax))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_reduce_window():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    reqs = [set(r[1]) for r in res]
    assert not (reqs[0] & reqs[1]) and len(reqs[0] | reqs[1]) == 8
    total = sum(r[2] for r in res)
    for r in res:
        assert r[3] == pytest.approx(total)      # tokens summed over ranks
        assert r[4] == pytest.approx(11.0)       # time = max over ranks


def test_reduce_window_single_process():
    assert reduce_window(5, [1.5, 2.0]) == (5.0, [1.5, 2.0])
    assert torch.tensor(1).item() == 1


def test_numa_cpulist_parsing_and_sysfs_lookup(tmp_path):
    from paper_2605_17613_b200.shard import gpu_local_cpus, parse_cpulist
    assert parse_cpulist("0-3,8,10-11\n") == [0, 1, 2, 3, 8, 10, 11]
    assert parse_cpulist("") == []
    dev = tmp_path / "0000:1b:00.0"
    dev.mkdir()
    (dev / "local_cpulist").write_text("56-111,168-223\n")
    cpus = gpu_local_cpus(0, 0x1B, 0, sysfs=str(tmp_path))
    assert cpus[:2] == [56, 57] and len(cpus) == 112 and cpus[-1] == 223
    assert gpu_local_cpus(0, 0x2B, 0, sysfs=str(tmp_path)) == []  # unknown device: no binding
