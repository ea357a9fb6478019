mkdir -p gpurun_out
timeout -s KILL 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r2g_c2.json
for w in "c2" "c3" "c5 --model qwen25_32b" "c4_w1"; do
  f=gpurun_out/r2g_$(echo $w | cut -d' ' -f1).json
  [ "$w" = "c2" ] || timeout -s KILL 1200 python bench.py --workload $w --steps 2 --warmup 1 --no-cpu-baseline 2>&1 | tail -1 > $f
  python - "$f" <<'PY'
import json, sys
d = json.load(open(sys.argv[1]))
r = d["roofline"]; a = d.get("attention_roofline", {}); l = d.get("layer_roofline", {})
o = d.get("decode_gemm_roofline") or d.get("prefill_gemm_roofline") or {}
print(d["config"]["workload"][:40], "value", round(d["value"]), "ms", round(d["ms_per_step"], 1),
      "| roofline", r["bound"], round(r["frac"] or 0, 3), "inpipe", round(r.get("inpipeline", {}).get("frac") or 0, 3),
      "| other", o.get("bound"), round(o.get("frac") or 0, 3), round((o.get("inpipeline") or {}).get("frac") or 0, 3),
      "| attn", round(a.get("frac") or 0, 3), round((a.get("inpipeline") or {}).get("frac") or 0, 3),
      round((a.get("inpipeline") or {}).get("frac_from_qkv_end") or 0, 3),
      "| layer", round(l.get("frac") or 0, 3), l.get("us_per_layer_median"))
PY
done
