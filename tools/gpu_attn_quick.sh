# attention kernel tests + attn_bench table (default build) + whole-run configs[1] / configs[4] lines
mkdir -p gpurun_out
bash tools/gpu_attn_sweep.sh -
timeout -s KILL 900 python bench.py --no-cpu-baseline --steps 3 --warmup 3 2>&1 | tail -1 > gpurun_out/q_c2.json
python -c "import json; d=json.load(open('gpurun_out/q_c2.json')); a=d['attention_roofline']; print('c2 value %.0f e2e %.0f attn %.3f inpipe %.3f layer %.1f' % (d['value'], d['e2e']['value'], a['frac'], a['inpipeline']['frac'], d['layer_roofline']['us_per_layer_median']))"
timeout -s KILL 1200 python bench.py --workload c5 --model qwen25_32b --no-cpu-baseline --steps 2 --warmup 3 2>&1 | tail -1 > gpurun_out/q_c5.json
python -c "import json; d=json.load(open('gpurun_out/q_c5.json')); a=d['attention_roofline']; print('c5 value %.0f e2e %.0f attn %.3f layer %.1f' % (d['value'], d['e2e']['value'], a['frac'], d['layer_roofline']['us_per_layer_median']))"
