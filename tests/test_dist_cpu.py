"""N > 1 host logic on CPU with the gloo backend (world size 2): the NCCL unique id reaches every
rank intact and the candidate shards of the ranks partition the grid."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2112_13509_b200 import dist as abd
    uid = abd.broadcast_unique_id(rank)
    C = 4096 + 77
    b, e = abd.my_shard(C)
    t = torch.tensor([b, e], dtype=torch.int64)
    allb = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(allb, t)
    digest = torch.tensor(list(uid[:16]), dtype=torch.int64)
    alld = [torch.zeros(16, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(alld, digest)
    if rank == 0:
        out.put(([tuple(x.tolist()) for x in allb], [tuple(x.tolist()) for x in alld], C))
    dist.destroy_process_group()


def test_two_rank_unique_id_and_shards():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    shards, digests, C = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert shards[0][0] == 0 and shards[-1][1] == C and shards[0][1] == shards[1][0]
    assert digests[0] == digests[1]
    assert any(v != 0 for v in digests[0])
