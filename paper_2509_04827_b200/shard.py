"""Multi-GPU scenario sharding (one process per GPU, torch.distributed).

Scenarios never interact, so a sweep shards with no data-path
collective. Two modes:
- weak scaling (bench.py): every rank evaluates its own block of scenarios;
- strong scaling: one fixed sweep split by a deterministic longest-processing-
  time (LPT) partition that every rank computes identically from the scenario
  table — no broadcast.
The only collective is the all-gather of the 128-byte result records
(BASELINE north_star), NCCL over NVLink on GPUs (gloo on CPU for tests).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

RECORD_BYTES = 128


def lpt_partition(costs, world: int) -> list[np.ndarray]:
    """Greedy LPT: scenarios in descending cost go to the least-loaded rank (ties: lowest
    rank, then lowest index). Returns, per rank, its scenario indices in descending cost."""
    costs = np.asarray(costs, np.float64)
    order = np.argsort(-costs, kind="stable")
    load = np.zeros(world)
    parts = [[] for _ in range(world)]
    for i in order:
        r = int(np.argmin(load))
        parts[r].append(int(i))
        load[r] += costs[i]
    return [np.asarray(p, np.int64) for p in parts]


def scenario_costs(w) -> np.ndarray:
    """Cost estimate per scenario (api.scenario_cost): requests of its trace, weighted by the
    number of decode instances."""
    from .api import scenario_cost
    lens = np.diff(np.asarray(w.traces.offset, np.int64))
    nd = np.array([w.layouts[i].n_d for i in np.asarray(w.scen["layout_id"], np.int64)])
    return scenario_cost(lens[np.asarray(w.scen["trace_id"], np.int64)], nd)


def gather_records(local: torch.Tensor, parts: list[np.ndarray], n_total: int, group=None) -> np.ndarray:
    """All-gather every rank's records ([n_local, 128] uint8, in the order of its part) and
    return all records in global scenario order (host numpy [n_total, 128] uint8)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    assert local.shape == (len(parts[rank]), RECORD_BYTES)
    m = max(len(p) for p in parts)
    pad = torch.zeros((m, RECORD_BYTES), dtype=torch.uint8, device=local.device)
    pad[: local.shape[0]] = local
    if dist.get_backend(group) == "nccl":
        out = torch.empty((world * m, RECORD_BYTES), dtype=torch.uint8, device=local.device)
        dist.all_gather_into_tensor(out, pad, group=group)
        chunks = out.view(world, m, RECORD_BYTES)
    else:
        lst = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(lst, pad, group=group)
        chunks = torch.stack(lst)
    host = chunks.cpu().numpy()
    res = np.zeros((n_total, RECORD_BYTES), np.uint8)
    for r, p in enumerate(parts):
        res[p] = host[r, : len(p)]
    return res


def weak_parts(n_local: int, world: int) -> list[np.ndarray]:
    """Weak scaling: rank r owns global scenarios r*n_local .. (r+1)*n_local - 1 (its own seed
    block; the global index is the record's position in the gathered sweep)."""
    return [np.arange(r * n_local, (r + 1) * n_local, dtype=np.int64) for r in range(world)]


class RecordGather:
    """The per-step collective of the sharded sweep: every rank's 128-B records, padded to the
    largest shard, all-gathered into one buffer (NCCL all_gather_into_tensor over NVLink; gloo
    on CPU). The simulate launch writes straight into `local` (a view of the padded send
    buffer), so the step adds no copy kernel. The records of a rank are in its kernel order
    (`kernel_order` = the DeviceWorkload's permutation of its part); the host maps them back to
    global scenario order once, outside the timed region."""

    def __init__(self, parts: list[np.ndarray], device, group=None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.parts = [np.asarray(p, np.int64) for p in parts]
        self.m = max(1, max(len(p) for p in self.parts))
        self.n_total = int(sum(len(p) for p in self.parts))
        self.nccl = dist.get_backend(group) == "nccl"
        self.pad = torch.zeros((self.m, RECORD_BYTES), dtype=torch.uint8, device=device)
        self.local = self.pad[: len(self.parts[self.rank])]
        self.out = torch.empty((self.world * self.m, RECORD_BYTES), dtype=torch.uint8, device=device)
        self.kernel_order = None

    def set_kernel_order(self, perm: np.ndarray):
        """perm[j] = index into this rank's part of the scenario in kernel slot j; exchanged once
        so rank 0 can place every rank's records."""
        perm = np.asarray(perm, np.int64)
        t = torch.full((self.m,), -1, dtype=torch.int64)
        t[: len(perm)] = torch.from_numpy(perm)
        dev = self.pad.device
        buf = [torch.empty_like(t.to(dev)) for _ in range(self.world)]
        dist.all_gather(buf, t.to(dev), group=self.group)
        self.kernel_order = [b.cpu().numpy() for b in buf]

    def enqueue(self):
        """The step's collective (asynchronous on the current stream for NCCL)."""
        if self.nccl:
            dist.all_gather_into_tensor(self.out, self.pad, group=self.group)
        else:
            lst = list(self.out.view(self.world, self.m, RECORD_BYTES).unbind(0))
            dist.all_gather(lst, self.pad, group=self.group)
            self.out.view(self.world, self.m, RECORD_BYTES).copy_(torch.stack(lst))

    def host_global(self) -> np.ndarray:
        """All records in global scenario order (host [n_total, 128] uint8)."""
        host = self.out.view(self.world, self.m, RECORD_BYTES).cpu().numpy()
        res = np.zeros((self.n_total, RECORD_BYTES), np.uint8)
        for r, p in enumerate(self.parts):
            k = len(p)
            order = np.arange(k) if self.kernel_order is None else self.kernel_order[r][:k]
            res[p[order]] = host[r, :k]
        return res
