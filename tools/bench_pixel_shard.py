"""Pixel-sharded single run (cfg4's "single run pixel-sharded across GPUs").

    python tools/bench_pixel_shard.py [--outer T] [--steps K]                  # 1 GPU
    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/bench_pixel_shard.py   # N GPUs

One EDAA run (M=1) of BASELINE cfg4's image (N=1024×1024, L=224, p=8) with its
pixels split over the ranks; every pass's slice partials are exchanged over NCCL
inside the captured schedule.  Prints one JSON line (rank 0): run-iterations/s,
device time as the max over ranks, and the pixel range each rank owned."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--outer", type=int, default=20)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--config", default="cfg4")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist
    from paper_2209_11002_b200 import distributed, edaa, synth
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", local))
    spec = synth.CONFIGS[args.config]
    x = synth.generate(spec)[0]
    dev = edaa.Device.get(local)
    distributed.join_pixel_shard(dev)
    if world == 1:  # exercise the exchange path with a one-rank communicator
        dev.set_pixel_shard(dev.nccl_unique_id(), 0, 1)
    dev.set_image(x)
    T, p = args.outer, spec.endmembers
    stream = torch.cuda.ExternalStream(dev.stream, device=torch.device("cuda", local))
    times = []
    for k in range(args.warmup + args.steps):
        dist.barrier()
        with torch.cuda.stream(stream):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        dev.solve_async(p, T, 5, 5, [0], [1.0])
        dev.finish()
        with torch.cuda.stream(stream):
            e1.record(stream)
        e1.synchronize()
        if k >= args.warmup:
            times.append(e0.elapsed_time(e1))
    t = torch.tensor([sum(times)], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    first, end = dev.shard_pixels()
    ranges = [None] * world
    dist.all_gather_object(ranges, (first, end))
    if rank == 0:
        print(json.dumps({
            "metric": "EDAA run-iterations/s, one run pixel-sharded", "value": T * args.steps / (t.item() * 1e-3),
            "unit": "run-iterations/s", "n_gpus": world, "steps": args.steps, "ms_per_step": t.item() / args.steps,
            "config": {"workload": "%s single run L=%d N=%d p=%d T=%d" % (spec.name, spec.bands, spec.pixels, p, T),
                       "pixel_ranges": ranges, "exchange": "NCCL broadcast of slice partials per pass"},
            "trace_last": float(dev.traces()[0, -1])}), flush=True)
    dev.set_pixel_shard(None, 0, 1)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
