"""Summarise ncu output brought back in gpurun_out/ into committed files under profiles/.

    python tools/ncu_summary.py launches gpurun_out/r01b/launches_C2.csv profiles/r01b_launches_C2_N1.txt
    python tools/ncu_summary.py full gpurun_out/r01b/full_C2.ncu-rep profiles/r01b_ncu_full_C2_N1.json

`launches`: per-kernel launch counts / mean device time / share of the listed time (ncu's cold-cache,
serialised per-launch durations — the SHARE is what compares with bench.py's live timing).
`full`: the key counters of every captured launch of an `ncu --set full` report, plus per-class mean DRAM
bytes per launch written to profiles/ncu_traffic.json (read by bench.py for roofline.traffic).
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

KEYS = ["Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg.per_second",
        "lts__t_bytes.sum"]

CLASSES = [("gemm_reduce", "gemm_reduce"), ("gemm", "gemm"), ("merge", "merge"), ("attention", "attention"),
           ("attn", "attention"), ("norm", "norm"), ("logits", "logits"), ("argmax", "argmax"), ("embed", "embed"),
           ("rope", "rope")]


def kclass(name):
    n = name.split("(")[0]
    for pat, cls in CLASSES:
        if pat in n:
            return cls
    return None


def to_bytes(v, unit):
    f = float(v.replace(",", ""))
    u = unit.lower()
    mul = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(u, 1)
    return f * mul


def launches(src, dst):
    rows = list(csv.reader(open(src)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    gi = h.index("Grid Size") if "Grid Size" in h else None
    agg = collections.OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        k = r[ki].split("(")[0].replace("void ", "").replace("pb::<unnamed>::", "")
        if gi is not None:
            k += f" grid{r[gi]}"
        t = float(r[vi].replace(",", ""))
        t = t / 1e3 if r[ui] in ("ns", "nsecond") else (t * 1e3 if r[ui] in ("ms", "msecond") else t)
        agg.setdefault(k, []).append(t)
    tot = sum(sum(v) for v in agg.values())
    lines = []
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{k:70s} {len(v):5d} launches {sum(v):10.1f} us {100 * sum(v) / tot:5.1f}%  avg {sum(v) / len(v):8.2f} us")
    lines.append(f"total {tot:.1f} us over {sum(len(v) for v in agg.values())} launches "
                 f"(ncu --metrics gpu__time_duration.sum --clock-control none; cold-cache, serialised)")
    open(dst, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def full(src, dst, workload="C2"):
    out = subprocess.run(["ncu", "-i", src, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = collections.OrderedDict()
    traffic = collections.defaultdict(list)
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        cls = kclass(name)
        d = {"Kernel Name": name}
        for k in KEYS:
            if k in h:
                i = h.index(k)
                d[k] = f"{r[i]} {units[i]}".strip()
        res.setdefault(cls or "other", []).append(d)
        try:
            rb = to_bytes(r[h.index("dram__bytes_read.sum")], units[h.index("dram__bytes_read.sum")])
            wb = to_bytes(r[h.index("dram__bytes_write.sum")], units[h.index("dram__bytes_write.sum")])
            if cls:
                traffic[cls].append(rb + wb)
        except (ValueError, IndexError):
            pass
    json.dump(res, open(dst, "w"), indent=1)
    # per workload (the bench line of that workload reads its own entry): {workload: {class: bytes per launch}}
    tpath = os.path.join(os.path.dirname(dst), "ncu_traffic.json")
    allw = json.load(open(tpath)) if os.path.exists(tpath) else {}
    tr = {k: sum(v) / len(v) for k, v in traffic.items()}
    tr["_source"] = os.path.basename(dst)
    tr["_note"] = "mean dram__bytes_read.sum + dram__bytes_write.sum per captured launch (ncu --set full)"
    allw[workload] = tr
    json.dump(allw, open(tpath, "w"), indent=1)
    for k, v in res.items():
        for d in v:
            print(k, {a: b for a, b in d.items() if a != "Kernel Name"})


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](*sys.argv[2:])
