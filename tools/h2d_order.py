"""When do chunked H2D copies complete? Events after every chunk, 1 vs 2 streams, and host polling."""
import time, torch
N = 48; C = 32 << 20
host = torch.empty(N * C, dtype=torch.uint8, pin_memory=True)
dev = torch.empty(N * C, dtype=torch.uint8, device="cuda")
for nst in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(nst)]
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True); t0.record(ss[0])
        for s in ss[1:]: s.wait_event(t0)
        evs = []
        th = time.perf_counter()
        for i in range(N):
            s = ss[i % nst]
            with torch.cuda.stream(s):
                dev[i*C:(i+1)*C].copy_(host[i*C:(i+1)*C], non_blocking=True)
                e = torch.cuda.Event(enable_timing=True); e.record(s); evs.append(e)
        tenq = time.perf_counter() - th
        # host polling of completion of event 0, N/2
        first_done = None
        while not evs[0].query(): pass
        first_done = time.perf_counter() - th
        torch.cuda.synchronize()
        ts = [t0.elapsed_time(e) for e in evs]
    print(f"streams={nst}: enqueue {tenq*1e3:.2f} ms, host saw chunk0 done at {first_done*1e3:.2f} ms; event ms:",
          " ".join(f"{t:.1f}" for t in ts[:6]), "...", " ".join(f"{t:.1f}" for t in ts[-4:]))
