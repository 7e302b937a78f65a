"""Request sharding across the GPUs of one box.

Configs 2-4 partition the path by request: each rank owns a disjoint set of
requests, its own engine, pinned host KV pool, copy stream and PCIe link.
There is no collective on the data path; the only communication is the
timing reduction after the timed window (tokens summed, device time taken as
the max over ranks -- the slowest rank bounds the whole job).
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    requests: tuple  # global request ids this rank serves
    seeds: tuple     # prefix-KV seed of each (deterministic per global id)


def shard_requests(n_total: int, world: int, rank: int, seed_base: int = 1) -> Shard:
    """Contiguous block partition of n_total requests over world ranks
    (the first n_total % world ranks take one extra)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if n_total < world:
        raise ValueError("fewer requests than ranks")
    q, r = divmod(n_total, world)
    lo = rank * q + min(rank, r)
    hi = lo + q + (1 if rank < r else 0)
    ids = tuple(range(lo, hi))
    return Shard(rank, world, ids, tuple(seed_base + 1000 * i for i in ids))


def weak_shard(per_rank: int, world: int, rank: int, seed_base: int = 1) -> Shard:
    """Weak scaling: every rank serves per_rank requests (global ids disjoint)."""
    return shard_requests(per_rank * world, world, rank, seed_base)


def reduce_window(tokens: float, times: list, dist=None, device=None):
    """Whole-job numbers of one timed window: (sum of tokens over ranks,
    [max over ranks of each time]).  Without torch.distributed: identity."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(tokens), [float(t) for t in times]
    import torch
    t = torch.tensor([float(tokens)], dtype=torch.float64, device=device)
    m = torch.tensor([float(x) for x in times], dtype=torch.float64, device=device)
    dist.all_reduce(t)
    dist.all_reduce(m, op=dist.ReduceOp.MAX)
    return float(t.item()), [float(x) for x in m.tolist()]


def parse_cpulist(text: str) -> list:
    """'0-3,8,10-11' -> [0, 1, 2, 3, 8, 10, 11] (sysfs cpulist format)."""
    cpus = []
    for part in text.strip().split(","):
        if not part:
            continue
        if "-" in part:
            a, b = part.split("-")
            cpus.extend(range(int(a), int(b) + 1))
        else:
            cpus.append(int(part))
    return cpus


def gpu_local_cpus(domain: int, bus: int, device: int, sysfs: str = "/sys/bus/pci/devices") -> list:
    """CPUs on the GPU's NUMA node (the PCI function's local_cpulist), or []."""
    import os
    path = os.path.join(sysfs, f"{domain:04x}:{bus:02x}:{device:02x}.0", "local_cpulist")
    try:
        with open(path) as f:
            return parse_cpulist(f.read())
    except OSError:
        return []


def bind_numa_local(torch_device: int) -> list:
    """Pin this rank's host threads to its GPU's NUMA node, so the pinned host
    KV pool (first-touched by cudaHostAlloc in this thread) and the copy
    engine's reads stay socket-local (each GPU owns a
    NUMA-local pinned pool and its own PCIe link).  Returns the CPU set used
    ([] when the topology is unknown -- nothing changes then)."""
    import os
    import torch
    p = torch.cuda.get_device_properties(torch_device)
    cpus = gpu_local_cpus(p.pci_domain_id, p.pci_bus_id, p.pci_device_id)
    avail = os.sched_getaffinity(0)
    cpus = [c for c in cpus if c in avail]
    if cpus:
        os.sched_setaffinity(0, cpus)
    return cpus
