"""Per-kernel event-to-event latency of small kernels on a compute stream, (a) alone, (b) while a copy
stream streams H2D, (c) with a cross-stream event wait before each kernel, (d) both."""
import torch, time
N_COPY = 80; C = 64 << 20
host = torch.empty(N_COPY * C, dtype=torch.uint8, pin_memory=True)
dev = torch.empty(N_COPY * C, dtype=torch.uint8, device="cuda")
x = torch.randn(128, 2048, device="cuda")
cs, ks = torch.cuda.Stream(), torch.cuda.Stream()
def trial(copy, wait):
    torch.cuda.synchronize()
    land = []
    if copy:
        with torch.cuda.stream(cs):
            for i in range(N_COPY):
                dev[i*C:(i+1)*C].copy_(host[i*C:(i+1)*C], non_blocking=True)
                e = torch.cuda.Event(); e.record(cs); land.append(e)
    ev = []
    with torch.cuda.stream(ks):
        for i in range(300):
            if wait and copy:
                ks.wait_event(land[min(i // 4, N_COPY - 1)])
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(ks); y = torch.nn.functional.layer_norm(x, (2048,)); b.record(ks); ev.append((a, b))
    torch.cuda.synchronize()
    d = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)
    return f"median {d[len(d)//2]:.1f} us  p90 {d[int(len(d)*.9)]:.1f} us"
for copy, wait in [(False, False), (True, False), (True, True), (False, False)]:
    trial(copy, wait)
    print(f"copy={copy} wait={wait}: {trial(copy, wait)}")
