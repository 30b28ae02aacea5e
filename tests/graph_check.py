"""CUDA-graph capture / replay of the sharded argmax under torchrun (debug helper for mgpu_check's
graph case): dumps every rank's Python stack if it does not finish in time."""
import faulthandler
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from tests.mgpu_check import graph_replay  # noqa: E402


def main():
    faulthandler.dump_traceback_later(int(os.environ.get("GRAPH_CHECK_DUMP_S", "60")), exit=True)
    dist.init_process_group("nccl")
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", rank)))
    torch.cuda.set_device(dev)
    print(rank, graph_replay(dev, rank, world), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
