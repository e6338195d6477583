"""Helpers to run a function in N processes with torch.distributed on 127.0.0.1."""
import os
import socket


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def init(rank: int, world: int, port: int, backend: str = "gloo"):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group(backend, rank=rank, world_size=world)


def run(fn, world: int, *args):
    import torch.multiprocessing as mp
    mp.spawn(fn, args=(world, free_port(), *args), nprocs=world, join=True)
