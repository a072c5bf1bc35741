"""Multi-process host logic of the scenario sharder on CPU (gloo, world_size 2).

The records each rank contributes are computed by the oracle (test infrastructure);
what is under test is the deterministic LPT partition, the padded all-gather and the
inverse permutation back to global scenario order.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_04827_b200.shard import gather_records, lpt_partition, scenario_costs


def test_lpt_partition_properties():
    rng = np.random.default_rng(0)
    c = rng.integers(1, 1000, 257).astype(float)
    for world in (1, 2, 3, 8):
        parts = lpt_partition(c, world)
        allidx = np.sort(np.concatenate(parts))
        assert (allidx == np.arange(len(c))).all()                      # a partition
        loads = [c[p].sum() for p in parts]
        assert max(loads) - min(loads) <= c.max()                       # LPT bound
        assert [list(p) for p in parts] == [list(p) for p in lpt_partition(c, world)]  # deterministic


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import synth
    w = synth.build_config("C3", scenarios=range(0, 256, 11), duration_scale=0.05)
    parts = lpt_partition(scenario_costs(w), world)
    mine = oracle.simulate_workload(w, parts[rank])
    local = torch.from_numpy(mine.view(np.uint8).reshape(len(mine), 128).copy())
    allrec = gather_records(local, parts, w.n)
    if rank == 0:
        q.put(allrec.tobytes())
    dist.barrier()
    dist.destroy_process_group()


def test_gather_records_gloo_world2():
    import oracle
    import synth
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    w = synth.build_config("C3", scenarios=range(0, 256, 11), duration_scale=0.05)
    ref = oracle.simulate_workload(w)
    assert got == ref.tobytes()       # byte-identical to the single-process evaluation
