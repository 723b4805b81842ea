"""Box probe: host/GPU facts and measured copy-engine bandwidths that fix the
PCIe roofline constants. Writes gpurun_out/probe.json. Timing with CUDA events after warm-up."""
import json
import os
import subprocess
import time

import torch


def sh(cmd):
    try:
        return subprocess.run(cmd, shell=True, capture_output=True, text=True, timeout=60).stdout
    except Exception as e:  # noqa
        return str(e)


def h2d_gbs(nbytes, chunk, streams, reps=5):
    host = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    dev = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    ss = [torch.cuda.Stream() for _ in range(streams)]
    best = 0.0
    for r in range(reps + 1):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(ss[0])
        for s in ss[1:]:
            s.wait_event(e0)
        off, i = 0, 0
        while off < nbytes:
            n = min(chunk, nbytes - off)
            with torch.cuda.stream(ss[i % streams]):
                dev[off:off + n].copy_(host[off:off + n], non_blocking=True)
            off += n
            i += 1
        for s in ss[1:]:
            ev = torch.cuda.Event()
            ev.record(s)
            ss[0].wait_event(ev)
        e1.record(ss[0])
        torch.cuda.synchronize()
        if r:
            best = max(best, nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    return best


def main():
    os.makedirs("gpurun_out", exist_ok=True)
    out = {"nproc": os.cpu_count(), "lscpu": sh("lscpu | head -20"), "meminfo": sh("head -5 /proc/meminfo"),
           "nvidia_smi": sh("nvidia-smi --query-gpu=name,pci.bus_id,pcie.link.gen.max,pcie.link.width.max,memory.total,clocks.max.sm --format=csv"),
           "topo": sh("nvidia-smi topo -m"), "numa": sh("numactl -H 2>/dev/null | head -5")}
    p = torch.cuda.get_device_properties(0)
    out["device"] = {"name": p.name, "sms": p.multi_processor_count, "mem": p.total_memory}
    res = {}
    for chunk_mb in (4, 16, 64):
        for st in (1, 2):
            res[f"h2d_{chunk_mb}MB_{st}s"] = h2d_gbs(2 << 30, chunk_mb << 20, st)
    out["h2d_gbs"] = res
    # D2D copy (HBM read+write)
    a = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
    b = torch.empty_like(a)
    for _ in range(3):
        b.copy_(a)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        b.copy_(a)
    e1.record()
    torch.cuda.synchronize()
    out["d2d_copy_gbs_rw"] = 2 * 10 * (1 << 30) / (e0.elapsed_time(e1) * 1e-3) / 1e9
    json.dump(out, open("gpurun_out/probe.json", "w"), indent=1)
    print(json.dumps({k: v for k, v in out.items() if k in ("h2d_gbs", "d2d_copy_gbs_rw", "device", "nproc")}, indent=1))


if __name__ == "__main__":
    main()
