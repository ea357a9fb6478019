"""Summarise in-pipeline GEMM spans written by HK_GEMM_TRACE=1 (bench.py dumps them).

    HK_GEMM_TRACE=1 HK_NO_GRAPHS=1 python bench.py --workload c2_short --steps 1 --warmup 0 ...
    python tools/gemm_trace.py gpurun_out/gemm_trace.csv
Per decode GEMM family: effective duration (last CTA end - first griddepcontrol.wait
exit), how early its CTAs were resident, and the gap to the previous GEMM's end
(the row / attention kernels in between).
"""
import csv
import statistics as S
import sys

NAMES = {(6144, 4096): "qkv", (4096, 4096): "o", (28672, 4096): "gate_up", (4096, 14336): "down"}
rows = list(csv.DictReader(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/gemm_trace.csv")))
stats = {}
prev_end = None
for r in rows:
    N, K, T = int(r["N"]), int(r["K"]), int(r["T"])
    st, wd, en = int(r["start"]), int(r["wait_done"]), int(r["end"])
    name = NAMES.get((N, K))
    if name and T <= 64 and wd < (1 << 63) and prev_end is not None:
        d = stats.setdefault(name, {"eff": [], "early": [], "gap": [], "tail": [], "bytes": N * K * 2})
        if "mainloop_end" in r:
            d["tail"].append((en - int(r["mainloop_end"])) / 1e3)
        d["eff"].append((en - wd) / 1e3)
        d["early"].append((wd - st) / 1e3)
        d["gap"].append((wd - prev_end) / 1e3)
    prev_end = en
print(f"{'gemm':8s} {'n':>5s} {'eff us':>8s} {'GB/s':>8s} {'early us':>9s} {'gap before us':>14s} {'tail us':>8s}")
for name, d in stats.items():
    e = S.median(d["eff"])
    tail = S.median(d['tail']) if d['tail'] else float('nan')
    print(f"{name:8s} {len(d['eff']):5d} {e:8.2f} {d['bytes'] / e / 1e3:8.0f} {S.median(d['early']):9.2f} {S.median(d['gap']):14.2f} {tail:8.2f}")
