# round-2 session-3 evidence: GPU tests + smoke, attention table, ncu of the two-tile attention
# (configs[1] k=128 and configs[4] k=128), configs[1] bench line (full profile) and configs[4] bench line
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -2 > gpurun_out/r2o_gputest.txt; cat gpurun_out/r2o_gputest.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python tools/attn_bench.py 2>&1 | tail -11 > gpurun_out/r2o_attn_bench.txt; cat gpurun_out/r2o_attn_bench.txt
ncu --set full --clock-control none -k regex:attn_decode -c 1 -o gpurun_out/r2o_attn_c2_k128 python tools/attn_probe.py 128 > gpurun_out/r2o_ncu_a.log 2>&1; tail -2 gpurun_out/r2o_ncu_a.log
ncu --set full --clock-control none -k regex:attn_decode -c 1 -o gpurun_out/r2o_attn_c5_k128 python tools/ncu_probes.py attn_c5 128 > gpurun_out/r2o_ncu_b.log 2>&1; tail -2 gpurun_out/r2o_ncu_b.log
timeout -s KILL 900 python bench.py 2>&1 | tail -1 > gpurun_out/r2o_bench_c2.json
python -c "import json; d=json.load(open('gpurun_out/r2o_bench_c2.json')); print('c2 value', d['value'], 'e2e', d['e2e']['value'], 'attn', d['attention_roofline']['frac'], d['attention_roofline']['inpipeline']['frac'], 'layer', d['layer_roofline']['frac'], d['layer_roofline']['us_per_layer_median'])"
timeout -s KILL 1200 python bench.py --workload c5 --model qwen25_32b --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r2o_bench_c5.json
python -c "import json; d=json.load(open('gpurun_out/r2o_bench_c5.json')); print('c5 value', d['value'], 'e2e', d['e2e']['value'], 'attn', d['attention_roofline']['frac'], d['attention_roofline']['inpipeline']['frac'], 'layer', d['layer_roofline']['frac'])"
