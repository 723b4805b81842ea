"""How many commands can be queued on a blocked stream before the enqueue call itself blocks?
Stream s (non-blocking) waits on a device word; we enqueue kernels / memcpys / memops on it and time
each host call. A watchdog thread releases the word from ANOTHER non-blocking stream after 15 s."""
import ctypes, threading, time, sys, torch
cuda = ctypes.CDLL("libcuda.so.1")
V = ctypes.c_void_p
cuda.cuStreamCreate.argtypes = [ctypes.POINTER(V), ctypes.c_uint]
cuda.cuStreamWaitValue32_v2.argtypes = [V, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint]
cuda.cuStreamWriteValue32_v2.argtypes = [V, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint]
cuda.cuStreamSynchronize.argtypes = [V]
torch.cuda.init()
x = torch.zeros(256, device="cuda")
word = torch.zeros(1, dtype=torch.int32, device="cuda")
other = torch.zeros(1, dtype=torch.int32, device="cuda")
h = torch.zeros(1 << 12, dtype=torch.uint8, pin_memory=True)
d = torch.zeros(1 << 12, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
def mk():
    st = V(); assert cuda.cuStreamCreate(ctypes.byref(st), 1) == 0; return st
s, rel = mk(), mk()
es = torch.cuda.ExternalStream(s.value)
def probe(kind, n=12000, val=1):
    assert cuda.cuStreamWaitValue32_v2(s, word.data_ptr(), val, 0) == 0   # GEQ? flags 0 = GEQ
    def watchdog():
        time.sleep(15)
        cuda.cuStreamWriteValue32_v2(rel, word.data_ptr(), val, 0)
        print("  watchdog released", flush=True)
    t = threading.Thread(target=watchdog, daemon=True); t.start()
    t0 = time.perf_counter(); blocked = None
    with torch.cuda.stream(es):
        for i in range(n):
            ti = time.perf_counter()
            if kind == "kernel": x.add_(1)
            elif kind == "memcpy": d.copy_(h, non_blocking=True)
            elif kind == "memop": cuda.cuStreamWriteValue32_v2(s, other.data_ptr(), i, 0)
            elif kind == "wait": cuda.cuStreamWaitValue32_v2(s, word.data_ptr(), val, 0)
            dt = time.perf_counter() - ti
            if dt > 0.5 and blocked is None:
                blocked = (i, dt)
    print(f"{kind}: first blocking call at #{blocked} ; total {time.perf_counter()-t0:.1f}s", flush=True)
    t.join(); cuda.cuStreamSynchronize(s)
for j, k in enumerate(("kernel", "memcpy", "memop", "wait")):
    probe(k, val=j + 1)
