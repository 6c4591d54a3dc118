"""Phase-0 box probe: host link (pinned H2D/D2H) bandwidth, host RAM, topology."""
import os, subprocess, time, json
import torch

def run(cmd):
    try:
        return subprocess.run(cmd, shell=True, capture_output=True, text=True, timeout=60).stdout
    except Exception as e:
        return str(e)

def single():
    """One GPU: pinned H2D/D2H bandwidth by size, host RAM, CPU, topology."""
    out = {}
    out["nproc"] = os.cpu_count()
    out["affinity"] = len(os.sched_getaffinity(0))
    out["free_g"] = run("free -g")
    out["lscpu"] = run("lscpu | head -30")
    out["topo"] = run("nvidia-smi topo -m")
    out["smi"] = run("nvidia-smi --query-gpu=name,memory.total,pcie.link.gen.current,pcie.link.width.current,clocks.max.sm --format=csv")
    dev = torch.device("cuda:0")
    res = {}
    for mb in [6, 64, 512, 2048]:
        n = mb << 20
        h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        h.fill_(1)
        d = torch.empty(n, dtype=torch.uint8, device=dev)
        for _ in range(3):
            d.copy_(h, non_blocking=True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        reps = max(3, 4096 // mb)
        e0.record()
        for _ in range(reps):
            d.copy_(h, non_blocking=True)
        e1.record(); torch.cuda.synchronize()
        h2d = n * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9
        e0.record()
        for _ in range(reps):
            h.copy_(d, non_blocking=True)
        e1.record(); torch.cuda.synchronize()
        d2h = n * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9
        res[mb] = {"h2d_GBps": round(h2d, 2), "d2h_GBps": round(d2h, 2)}
    out["pinned_copy"] = res
    # zero-copy SM read of pinned memory via a mapped view: torch has no direct API; skip
    print(json.dumps(out, indent=1))
    with open("gpurun_out/probe_box.json", "w") as f:
        json.dump(out, f, indent=1)


def concurrent_h2d(mb=512, reps=16):
    """Phase-0 probe of the shared host links: every rank (one per GPU, torchrun)
    streams pinned H2D at the same time; per-rank and aggregate GB/s show PCIe-switch uplink
    sharing and the host-DRAM ceiling for N x ~55 GB/s.  Feeds placement.Placement(uplinks=,
    uplink_load_slope=)."""
    import torch.distributed as dist
    dist.init_process_group("nccl")
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        d.copy_(h, non_blocking=True)
    e1.record()
    e1.synchronize()
    gbs = torch.tensor([n * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9], device="cuda")
    allv = [torch.zeros_like(gbs) for _ in range(world)]
    dist.all_gather(allv, gbs)
    if rank == 0:
        per = [round(float(v), 2) for v in allv]
        out = {"ranks": world, "per_rank_h2d_GBps": per, "aggregate_GBps": round(sum(per), 2),
               "topo": run("nvidia-smi topo -m")}
        print(json.dumps(out, indent=1))
        with open("gpurun_out/probe_concurrent_h2d.json", "w") as f:
            json.dump(out, f, indent=1)
    dist.destroy_process_group()



if __name__ == "__main__":
    import sys
    if "--concurrent" in sys.argv:  # torchrun --nproc-per-node N tools/probe_box.py --concurrent
        concurrent_h2d()
    else:
        single()
