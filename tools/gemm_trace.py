"""Summarise in-pipeline kernel spans written by HK_GEMM_TRACE=1 (bench.py dumps them).

    HK_GEMM_TRACE=1 HK_NO_GRAPHS=1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-profile
    python tools/gemm_trace.py gpurun_out/gemm_trace.csv
Per decode GEMM family and for the decode attention: effective duration (last
CTA end - first griddepcontrol.wait exit), how early its CTAs were resident,
the gap to the previous traced kernel's end, and the tail after the last CTA's
main loop (GEMMs). Attention rows carry their algorithmic bytes (N = -1, K = KB).
"""
import csv
import json
import statistics as S
import sys

NAMES = {(6144, 4096): "qkv", (4096, 4096): "o", (28672, 4096): "gate_up", (4096, 14336): "down"}
PEAK = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if __import__("os").path.exists("MEASURED_PEAKS.json") else 6555.5
rows = list(csv.DictReader(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/gemm_trace.csv")))
stats = {}
prev_end = None
for r in rows:
    N, K, T = int(r["N"]), int(r["K"]), int(r["T"])
    st, wd, en = int(r["start"]), int(r["wait_done"]), int(r["end"])
    name = "attn" if N == -1 else NAMES.get((N, K))
    ok = wd < (1 << 63) and en > 0 and prev_end is not None and (N == -1 or T <= 64)
    if name and ok and (name != "attn" or T > 0):
        d = stats.setdefault(name, {"eff": [], "early": [], "gap": [], "tail": [], "bytes": []})
        d["eff"].append((en - wd) / 1e3)
        d["early"].append((wd - st) / 1e3)
        d["gap"].append((wd - prev_end) / 1e3)
        d["bytes"].append(K * 1024.0 if N == -1 else N * K * 2.0)
        if "mainloop_end" in r and N != -1:
            d["tail"].append((en - int(r["mainloop_end"])) / 1e3)
    if en > 0:
        prev_end = en
print(f"{'kernel':8s} {'n':>5s} {'eff us':>8s} {'GB/s':>8s} {'frac':>6s} {'early us':>9s} {'gap before us':>14s} {'tail us':>8s}")
for name, d in stats.items():
    e = S.median(d["eff"])
    gbs = sum(d["bytes"]) / sum(d["eff"]) / 1e3  # bytes-weighted over all launches
    tail = S.median(d["tail"]) if d["tail"] else float("nan")
    print(f"{name:8s} {len(d['eff']):5d} {e:8.2f} {gbs:8.0f} {gbs / PEAK:6.3f} {S.median(d['early']):9.2f} "
          f"{S.median(d['gap']):14.2f} {tail:8.2f}")
