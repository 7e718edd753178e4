"""Host-side logic of the N>1 path on CPU (gloo, world_size 2): the per-rank env ranges
(contiguous, remainder to low ranks, plan.cpp:46-55), the NCCL-id broadcast pattern bench.py
uses, and the max-over-ranks timing reduction."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import bench

    w, r, _ = bench.dist_setup()
    assert (w, r) == (world, rank)
    obj = [b"id-bytes-from-rank0" if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    t = bench.max_over_ranks(float(rank + 1) * 1.5, world)
    out[rank] = (obj[0], t)
    dist.destroy_process_group()


def test_two_rank_broadcast_and_max():
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
        res = dict(out)
    assert res[0] == res[1] == (b"id-bytes-from-rank0", 3.0)


def test_env_ranges_match_reference_split():
    from paper_2210_00882_b200 import Program
    import json

    for total, k in ((16384, 2), (16384, 8), (10, 3), (9, 4)):
        p = Program({"algorithm": "ppo", "actor": {"num": k}, "env": {"type": "gridline", "num": total}},
                    {"slots_per_worker": {"cpu": 1, "accel": k}, "distribution_policy": "dp-d"})
        inst = json.loads(p.dump())["instances"]
        base, rem = divmod(total, k)
        lo = 0
        for r, i in enumerate(inst):
            n = base + (1 if r < rem else 0)
            assert (i["env_lo"], i["env_hi"]) == (lo, lo + n)
            lo += n
        assert lo == total
