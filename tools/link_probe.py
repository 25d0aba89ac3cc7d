"""Interconnect micro-benchmarks: the denominators of the multi-GPU splits'
rooflines.  One process per GPU:

    python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port 29531 tools/link_probe.py [--bytes 8388612]

  * NCCL all_reduce(SUM) bus bandwidth at the angle split's packed buffer size
    ([x_fbp | grad | mc] at cfg5 = 8,388,612 B) and at 64 MB: busbw = 2 (G-1)/G x bytes / t.
  * NCCL all_gather at the communication-reduced split's size (2 B m n_det fp32 = 2,967,552 B).
  * point-to-point bandwidth rank 0 -> rank 1 (NCCL send/recv over NVLink, 64 MB).
Times are CUDA events on the launching stream, max over ranks, after warm-up.  With gloo
(CPU, the tests) the same code runs on host tensors and the numbers mean nothing.
Rank 0 prints one JSON line."""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--bytes", type=int, default=8388612)
    ap.add_argument("--ag-bytes", type=int, default=2967552)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--backend", default=None)
    args = ap.parse_args(argv)
    use_cuda = torch.cuda.is_available() and args.backend != "gloo"
    backend = args.backend or ("nccl" if use_cuda else "gloo")
    dist.init_process_group(backend)
    rank, world = dist.get_rank(), dist.get_world_size()
    if use_cuda:
        local = int(os.environ.get("LOCAL_RANK", rank))
        torch.cuda.set_device(local)
        dev = torch.device("cuda", local)
    else:
        dev = torch.device("cpu")
    if world < 2:
        if rank == 0:
            print(json.dumps({"link_probe": "needs >= 2 ranks", "world": world}))
        dist.destroy_process_group()
        return 0

    res = {"world": world, "backend": backend}
    for nbytes in (args.bytes, 64 << 20):
        buf = torch.ones(nbytes // 4, dtype=torch.float32, device=dev)
        t = timed_any(lambda: dist.all_reduce(buf), args.iters, dev)
        res[f"allreduce_{nbytes}B"] = {"s": t, "busbw_gbs": 2 * (world - 1) / world * nbytes / t / 1e9}
    nb = args.ag_bytes // world // 4 * 4
    part = torch.ones(nb // 4, dtype=torch.float32, device=dev)
    full = torch.empty(world * (nb // 4), dtype=torch.float32, device=dev)
    t = timed_any(lambda: dist.all_gather_into_tensor(full, part), args.iters, dev)
    res[f"allgather_{nb * world}B"] = {"s": t, "busbw_gbs": (world - 1) / world * nb * world / t / 1e9}
    # point-to-point rank 0 -> 1 (the other ranks idle)
    p2p = torch.ones(16 << 20, dtype=torch.float32, device=dev)

    def sendrecv():
        if rank == 0:
            dist.send(p2p, 1)
        elif rank == 1:
            dist.recv(p2p, 0)
    t = timed_any(sendrecv, args.iters, dev)
    res["p2p_64MB_0to1"] = {"s": t, "gbs": p2p.numel() * 4 / t / 1e9}
    if rank == 0:
        print(json.dumps(res))
    dist.destroy_process_group()
    return 0


def timed_any(fn, iters, dev):
    """timed() with the MAX over ranks done on a tensor of the backend's device."""
    for _ in range(3):
        fn()
    import time
    if dev.type == "cuda":
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dist.barrier()
        torch.cuda.synchronize()
        a.record()
        for _ in range(iters):
            fn()
        b.record()
        torch.cuda.synchronize()
        t = a.elapsed_time(b) / iters * 1e-3
    else:
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(iters):
            fn()
        t = (time.perf_counter() - t0) / iters
    tt = torch.tensor([t], dtype=torch.float64, device=dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    return float(tt.item())


if __name__ == "__main__":
    sys.exit(main())
