"""Does a device-uploaded CUDA graph avoid the launch slowdown caused by a saturated H2D link?
300 small kernels: eager vs graph, with and without a concurrent H2D copy stream."""
import torch
N_COPY = 80; C = 64 << 20
host = torch.empty(N_COPY * C, dtype=torch.uint8, pin_memory=True)
dev = torch.empty(N_COPY * C, dtype=torch.uint8, device="cuda")
x = torch.randn(128, 2048, device="cuda")
cs, ks = torch.cuda.Stream(), torch.cuda.Stream()
def body():
    for i in range(300):
        y = torch.nn.functional.layer_norm(x, (2048,))
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(ks):
    body()
torch.cuda.synchronize()
with torch.cuda.graph(g, stream=ks):
    body()
torch.cuda.synchronize()
def run(copy, graph):
    torch.cuda.synchronize()
    if copy:
        with torch.cuda.stream(cs):
            for i in range(N_COPY):
                dev[i*C:(i+1)*C].copy_(host[i*C:(i+1)*C], non_blocking=True)
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(ks):
        a.record(ks)
        if graph:
            g.replay()
        else:
            body()
        b.record(ks)
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / 300
for copy in (False, True):
    for graph in (False, True):
        run(copy, graph)
        print(f"copy={copy} graph={graph}: {run(copy, graph):.1f} us per kernel")
