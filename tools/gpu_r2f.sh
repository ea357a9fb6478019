mkdir -p gpurun_out
timeout -s KILL 900 python bench.py --steps 5 --warmup 3 2>&1 | tail -1 > gpurun_out/r2f_c2.json
python -c "import json; d=json.load(open('gpurun_out/r2f_c2.json')); [print(k, json.dumps(d.get(k))[:400]) for k in ('value','e2e','roofline','attention_roofline','layer_roofline','cpu_baseline','clocks')]"
for w in "c3" "c5 --model qwen25_32b" "c4_w1"; do
  timeout -s KILL 1200 python bench.py --workload $w --steps 2 --warmup 1 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r2f_$(echo $w | cut -d' ' -f1).json
  python -c "import json,sys; d=json.load(open('gpurun_out/r2f_$(echo $w | cut -d' ' -f1).json')); print('$w', round(d['value']), round(d['ms_per_step'],1), d['config']['hit_rate_pct'], 'gemm', round(d['roofline']['frac'],3), 'attn', round(d['attention_roofline']['frac'],3), 'layer', d.get('layer_roofline',{}).get('frac'))" 2>&1 | tail -2
done
