"""End-to-end check of the p2p (pull-merge over CUDA IPC) sample sort with
several processes on ONE GPU (not collected by pytest; run by
tests/test_gpu_parity.py::test_p2p_sample_sort_processes_one_gpu).

The ranks' kernels never wait on each other: all cross-rank synchronisation
is host-side gloo; a rank's merge kernel reads the other ranks' shards
through IPC mappings, exactly as it would read peer GPUs over NVLink."""
import os
import socket
import sys

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(rank, world, port, n, dist_kind, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from oracle import oracle as O
    from paper_2503_05934_b200 import samplesort
    full = O.generate_i32(dist_kind, n, 42)
    m = n // world
    lo = rank * m
    hi = n if rank == world - 1 else lo + m
    shard = torch.from_numpy(full[lo:hi].copy()).cuda()
    ops = samplesort.DeviceOps()
    out = samplesort.sample_sort(shard, ops=ops, exchange="p2p")
    res = out.cpu().numpy()
    parts = [None] * world
    dist.all_gather_object(parts, res)
    dist.barrier()
    ops.release()
    if rank == 0:
        q.put(np.concatenate(parts))
    dist.destroy_process_group()


def main():
    world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 3_000_000
    dist_kind = sys.argv[3] if len(sys.argv) > 3 else "random"
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, world, port, n, dist_kind, q)) for r in range(world)]
    for p in ps:
        p.start()
    got = q.get(timeout=300)
    for p in ps:
        p.join(timeout=120)
    from oracle import oracle as O
    want = np.sort(O.generate_i32(dist_kind, n, 42))
    ok = np.array_equal(got, want) and all(p.exitcode == 0 for p in ps)
    print("P2P_OK" if ok else "P2P_BAD", world, n, dist_kind)


if __name__ == "__main__":
    main()
