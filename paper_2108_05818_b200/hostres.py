"""Host resources of one rank: CPU cores and NUMA placement.

One process per GPU shares the host with its node-local peers.  The host
side of the step — the fused host Adam of CPU-placed optimizer triplets, the
CPU-placed embedding operator, pinned chunk slabs that the copy engines
stream through — is host-DRAM bound, so each rank should run on cores of its
GPU's NUMA node and allocate its pinned memory there (first touch happens in
the allocating thread, so a process bound to the node gets node-local pinned
pages).  The reference splits host *memory* per rank
(`/root/reference/pkg/src/chunkstar/scenario.py:129`, cpu_bytes // nproc);
this splits the cores the same way.

:func:`bind_local_rank` narrows the process's affinity mask to its share of
its GPU's node (whole physical cores, SMT siblings kept together) and sets
``CS_HOST_BOUND=1`` so that the library's ``cs_host_threads(0)`` uses the
mask as is; :func:`host_threads` returns the team size every host kernel is
given explicitly.
"""

import os
from typing import Dict, List, Optional, Sequence

from . import _native as N


def _read(path: str) -> Optional[str]:
    try:
        with open(path) as f:
            return f.read().strip()
    except OSError:
        return None


def parse_cpulist(text: str) -> List[int]:
    """'0-3,8,10-11' -> [0, 1, 2, 3, 8, 10, 11]."""
    out: List[int] = []
    for part in text.split(","):
        part = part.strip()
        if not part:
            continue
        if "-" in part:
            a, b = part.split("-")
            out.extend(range(int(a), int(b) + 1))
        else:
            out.append(int(part))
    return out


def gpu_numa_node(device_index: int) -> int:
    """NUMA node of a CUDA device's PCI function, -1 if unknown."""
    try:
        import torch
        p = torch.cuda.get_device_properties(device_index)
        bdf = "%04x:%02x:%02x.0" % (p.pci_domain_id, p.pci_bus_id, p.pci_device_id)
    except Exception:
        return -1
    v = _read("/sys/bus/pci/devices/%s/numa_node" % bdf)
    try:
        return int(v) if v is not None else -1
    except ValueError:
        return -1


def node_cpus(node: int) -> List[int]:
    v = _read("/sys/devices/system/node/node%d/cpulist" % node) if node >= 0 else None
    return parse_cpulist(v) if v else []


def physical_cores(cpus: Sequence[int]) -> List[List[int]]:
    """Group logical CPUs into physical cores (SMT siblings together),
    ordered by the lowest logical id of each core."""
    cores: Dict[tuple, List[int]] = {}
    for c in cpus:
        pkg = _read("/sys/devices/system/cpu/cpu%d/topology/physical_package_id" % c) or "0"
        core = _read("/sys/devices/system/cpu/cpu%d/topology/core_id" % c)
        key = (pkg, core if core is not None else "cpu%d" % c)
        cores.setdefault(key, []).append(c)
    return sorted((sorted(v) for v in cores.values()), key=lambda v: v[0])


def share_of_node(local_rank: int, local_world: int, device_nodes: Sequence[int],
                  allowed: Sequence[int], cpus_of_node=node_cpus,
                  cores_of=physical_cores) -> List[int]:
    """The logical CPUs of ``local_rank``: the physical cores of its GPU's
    NUMA node (restricted to ``allowed``), split evenly among the local
    ranks whose GPUs sit on that node.  Unknown topology: an even split of
    ``allowed``.  Never empty."""
    node = device_nodes[local_rank] if local_rank < len(device_nodes) else -1
    allowed_set = set(allowed)
    pool = [c for c in cpus_of_node(node) if c in allowed_set] if node >= 0 else []
    peers = [r for r in range(local_world)
             if r < len(device_nodes) and device_nodes[r] == node] if pool else []
    if not pool or local_rank not in peers:
        pool, peers = sorted(allowed_set), list(range(local_world))
    cores = cores_of(pool)
    k, n = peers.index(local_rank), len(peers)
    if len(cores) >= n:
        lo, hi = len(cores) * k // n, len(cores) * (k + 1) // n
        mine = [c for core in cores[lo:hi] for c in core]
    else:  # fewer cores than ranks: share them round-robin
        mine = cores[k % len(cores)]
    return sorted(mine)


def bind_local_rank(local_rank: int, local_world: int, device_index: int) -> dict:
    """Narrow this process to its share of its GPU's NUMA node; returns what
    was done.  No-op (reported as such) for a single local rank."""
    allowed = sorted(os.sched_getaffinity(0))
    if local_world <= 1:
        return {"bound": False, "cpus": len(allowed)}
    try:
        import torch
        ndev = torch.cuda.device_count()
    except Exception:
        ndev = 0
    # torchrun's convention: local rank r drives device r
    nodes = [gpu_numa_node(i) for i in range(max(ndev, local_world))]
    if 0 <= device_index < len(nodes) and device_index != local_rank:
        nodes[local_rank] = nodes[device_index]
    mine = share_of_node(local_rank, local_world, nodes, allowed)
    os.sched_setaffinity(0, mine)
    os.environ["CS_HOST_BOUND"] = "1"
    return {"bound": True, "numa_node": nodes[local_rank] if local_rank < len(nodes) else -1,
            "cpus": len(mine), "cpu_list": mine}


def host_threads(requested: int = 0) -> int:
    """OpenMP team size of the host kernels (``cs_host_threads``)."""
    return int(N.load().cs_host_threads(int(requested)))
