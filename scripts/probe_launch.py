"""Launch-floor probes on 2 processes (rank 0 measures): empty kernel, and an empty
kernel that also stores one word into the peer GPU's memory (completion cost of a
kernel with NVLink writes).

    torchrun --nproc-per-node 2 scripts/probe_launch.py
"""
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    from paper_2509_21527_b200.session import HaloSession
    sess = HaloSession((1, 1, world), (4.0, 4.0, 4.0 * world), 1.0, (0, 0, 1), capacity=65536, device=rank,
                       nprocs=world, proc=rank)
    dist.barrier()
    out = {}
    if rank == 0:
        for g in (False, True):
            tag = "graph" if g else "eager"
            out[f"empty_{tag}_us"] = round(sess.halo.floor_launch(2000, graph=g), 3)
            for words in (1, 1024, 32768, 131072):
                out[f"remote_{words}w_{tag}_us"] = round(sess.halo.floor_launch_remote(1, words, 2000, graph=g), 3)
                out[f"local_{words}w_{tag}_us"] = round(sess.halo.floor_launch_remote(0, words, 2000, graph=g), 3)
        print(json.dumps(out), flush=True)
    dist.barrier()
    sess.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
