"""Multi-GPU parity (run under torchrun, one rank per GPU): candidate-sharded arg-max with the NCCL
key exchange must be bit-identical on every rank and to the single-GPU result (G-invariance), and
agree with the float64 oracle on sampled jobs; the replicated adapt after the encode-sharded K1a
must leave bit-identical weights on every rank and equal to one GPU's. Prints one JSON line per config on rank 0."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2112_13509_b200 import dist as abd  # noqa: E402
from paper_2112_13509_b200.autobyte import AutoByte, DeviceGrid, DeviceJobs  # noqa: E402
from tests.helpers import check_argmax  # noqa: E402


def run(name, desc, jobs, grid, cg, dev, rank, world):
    W = synth.make_weights(desc)
    os.environ["AUTOBYTE_CTA_GROUP"] = str(cg)
    net = AutoByte(desc.hidden_layers, desc.hidden_width, W, device=dev.index)
    abd.attach(net)
    dj, dg = DeviceJobs.from_host(jobs, dev), DeviceGrid.from_host(grid, dev)
    cur = torch.as_tensor(synth.current_configs(jobs.J, grid.C, 9), dtype=torch.int32, device=dev)
    b, e = abd.my_shard(grid.C)
    bi, bs, cs = net.argmax(dj, dg, cur, b, e)
    torch.cuda.synchronize(dev)
    packed = torch.cat([bi.view(torch.int32), bs.view(torch.int32), cs.view(torch.int32)])
    allp = [torch.empty_like(packed) for _ in range(world)]
    dist.all_gather(allp, packed)
    same_all_ranks = all(torch.equal(allp[0], x) for x in allp)
    res = {"config": name, "world": world, "cta_group": cg, "same_on_all_ranks": same_all_ranks,
           "peer_exchange": net.peer_exchange()}
    # host entry point: each rank copies only its encoder shard of the statistics -> same results
    hb, hs, hc = net.argmax_host(jobs, grid, cur.cpu().numpy(), b, e)
    res["host_same_as_device"] = bool(np.array_equal(hb, bi.cpu().numpy())
                                      and np.array_equal(hs.view(np.int32), bs.cpu().numpy().view(np.int32))
                                      and np.array_equal(np.nan_to_num(hc), np.nan_to_num(cs.cpu().numpy())))
    full = jobs.T.nbytes + jobs.B_d.nbytes + jobs.B_u.nbytes + 4 * 4 * jobs.J
    res["host_staged_bytes"] = net.staged_job_bytes(jobs.J, jobs.T.shape[1])
    res["host_staged_fraction"] = res["host_staged_bytes"] / full
    # top-k (NEXT 4): per-rank lists all-gathered and merged -> identical everywhere and to 1 GPU
    ti, ts = net.topk(dj, dg, 8, b, e)
    torch.cuda.synchronize(dev)
    tpk = torch.cat([ti.reshape(-1), ts.view(torch.int32).reshape(-1)])
    allt = [torch.empty_like(tpk) for _ in range(world)]
    dist.all_gather(allt, tpk)
    res["topk_same_on_all_ranks"] = all(torch.equal(allt[0], x) for x in allt)
    if rank == 0:
        single = AutoByte(desc.hidden_layers, desc.hidden_width, W, device=dev.index)
        bi1, bs1, cs1 = single.argmax(dj, dg, cur)
        torch.cuda.synchronize(dev)
        res["g_invariant"] = bool(torch.equal(bi, bi1) and torch.equal(bs.view(torch.int32), bs1.view(torch.int32))
                                  and torch.equal(torch.nan_to_num(cs), torch.nan_to_num(cs1)))
        ti1, ts1 = single.topk(dj, dg, 8)
        torch.cuda.synchronize(dev)
        res["topk_g_invariant"] = bool(torch.equal(ti, ti1) and torch.equal(ts.view(torch.int32), ts1.view(torch.int32)))
        sample = [0, jobs.J // 2, jobs.J - 1]
        s_ora = oracle.score_matrix(W, jobs, grid, job_idx=sample)
        check_argmax(bi.cpu().numpy()[sample], s_ora, 2e-2)
        res["oracle_sampled_ok"] = True
    # adapt: replicated K4 after the encode-sharded K1a must leave bit-identical weights on every
    # rank, equal to the single-GPU update
    batch = synth.make_adapt_batch(jobs, grid, 11)
    sp = torch.as_tensor(batch.S_p, device=dev)
    sc = torch.as_tensor(batch.S_c, device=dev)
    vb = torch.as_tensor(batch.V_bar, device=dev)
    loss = net.adapt(dj, sp, sc, vb, lr=1e-3, steps=1)
    torch.cuda.synchronize(dev)
    blob = torch.frombuffer(bytearray(net.get_weights_blob()), dtype=torch.uint8).to(dev)
    allb = [torch.empty_like(blob) for _ in range(world)]
    dist.all_gather(allb, blob)
    res["adapt_same_on_all_ranks"] = all(torch.equal(allb[0], x) for x in allb)
    hnet = AutoByte(desc.hidden_layers, desc.hidden_width, W, device=dev.index)
    abd.attach(hnet)
    hloss = hnet.adapt_host(batch.jobs, batch.S_p, batch.S_c, batch.V_bar, lr=1e-3, steps=1)
    res["adapt_host_same_as_device"] = hnet.get_weights_blob() == net.get_weights_blob() and hloss == float(loss.item())
    hnet.close()
    if rank == 0:
        loss1 = single.adapt(dj, sp, sc, vb, lr=1e-3, steps=1)
        torch.cuda.synchronize(dev)
        res["adapt_g_invariant"] = (single.get_weights_blob() == net.get_weights_blob()
                                    and float(loss1.item()) == float(loss.item()))
        single.close()
    net.close()
    return res


def graph_replay(dev, rank, world):
    """CUDA-graph capture of the sharded argmax (the exchange epoch is a device counter, so every
    replay is a fresh exchange): replays with changed inputs (current configs rewritten in place)
    must equal eager calls on every rank."""
    c3 = synth.config("C3")
    jobs, grid = c3.jobs.subset(np.arange(64)), synth.log_grid(32, 32)
    W = synth.make_weights(c3.desc)
    s = torch.cuda.Stream(dev)
    net = AutoByte(c3.desc.hidden_layers, c3.desc.hidden_width, W, device=dev.index, stream=s)
    abd.attach(net)
    dj, dg = DeviceJobs.from_host(jobs, dev), DeviceGrid.from_host(grid, dev)
    b, e = abd.my_shard(grid.C)
    cur = torch.zeros(jobs.J, dtype=torch.int32, device=dev)
    out = tuple(torch.empty(jobs.J, dtype=dt, device=dev) for dt in (torch.int32, torch.float32, torch.float32))
    with torch.cuda.stream(s):
        net.argmax(dj, dg, cur, b, e, out=out)   # warm-up: workspaces allocated outside the capture
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        net.argmax(dj, dg, cur, b, e, out=out)
    ok = True
    for rep in range(4):
        cur.copy_(torch.as_tensor(synth.current_configs(jobs.J, grid.C, 100 + rep), device=dev))
        g.replay()
        s.synchronize()
        got = [t.clone() for t in out]
        with torch.cuda.stream(s):
            ref = net.argmax(dj, dg, cur, b, e)
        s.synchronize()
        ok &= torch.equal(got[0], ref[0]) and torch.equal(got[1].view(torch.int32), ref[1].view(torch.int32)) and \
            torch.equal(torch.nan_to_num(got[2]), torch.nan_to_num(ref[2]))
    del g   # a graph holding captured NCCL work must go before the ctx's communicator is destroyed
    torch.cuda.synchronize(dev)
    net.close()
    return {"graph_replay_same_as_eager": bool(ok), "world": world}


def main():
    dist.init_process_group("nccl")
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", rank))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    ok = True
    c3 = synth.config("C3")
    ragged = synth.log_grid(37, 29)
    cases = [("C3", c3.desc, c3.jobs, c3.grid, 1), ("C3-ragged", c3.desc, c3.jobs.subset(np.arange(40)), ragged, 1),
             ("C4-subset-cg2", synth.NetDesc(4, 512), synth.config("C4").jobs.subset(np.arange(300)),
              synth.log_grid(64, 64), 2),
             ("C4-subset-ragged-cg2", synth.NetDesc(4, 512), synth.config("C4").jobs.subset(np.arange(33)),
              synth.log_grid(45, 23), 2),
             # fewer jobs than ranks at G = 4: a rank with an empty encoder shard still takes part
             ("C3-three-jobs", c3.desc, c3.jobs.subset(np.arange(3)), synth.log_grid(5, 3), 1),
             # fewer candidates than ranks (C = 1 and 3): some ranks hold an empty shard and still join
             ("one-candidate", synth.NetDesc(2, 64), c3.jobs.subset(np.arange(9)), synth.log_grid(1, 1), 1),
             ("three-candidates", synth.NetDesc(2, 64), c3.jobs.subset(np.arange(9)), synth.log_grid(1, 3), 1)]
    # every exchange: the fused peer-memory key kernel (default), the same plus the x all-gather
    # fused into K1a's epilogue (opt-in AUTOBYTE_PEER_X=1), and NCCL all-gathers + K5
    runs = [(mode,) + case for mode in ("peer", "peer_x", "nccl") for case in cases]
    for mode, name, desc, jobs, grid, cg in runs:  # noqa: B007
        os.environ.pop("AUTOBYTE_EXCHANGE", None)
        os.environ.pop("AUTOBYTE_PEER_X", None)
        if mode == "nccl":
            os.environ["AUTOBYTE_EXCHANGE"] = "nccl"
        elif mode == "peer_x":
            os.environ["AUTOBYTE_PEER_X"] = "1"
        r = run(name, desc, jobs, grid, cg, dev, rank, world)
        r["exchange"] = mode
        if rank == 0:
            print(json.dumps(r), flush=True)
            ok &= (r["same_on_all_ranks"] and r["g_invariant"] and r["adapt_same_on_all_ranks"] and r["adapt_g_invariant"]
                   and r["topk_same_on_all_ranks"] and r["topk_g_invariant"] and r["host_same_as_device"]
                   and r["adapt_host_same_as_device"] and (world == 1 or r["host_staged_fraction"] < 0.75)
                   and r["peer_exchange"] == (world > 1 and mode != "nccl"))
    gr = graph_replay(dev, rank, world)
    okt = torch.tensor([int(gr["graph_replay_same_as_eager"])], device=dev)
    dist.all_reduce(okt, op=dist.ReduceOp.MIN)
    if rank == 0:
        gr["all_ranks"] = bool(okt.item())
        print(json.dumps(gr), flush=True)
        ok &= gr["all_ranks"]
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        print("MGPU_OK" if ok else "MGPU_FAIL", flush=True)
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
