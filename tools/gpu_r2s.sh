# round-2 final evidence (CTA-pair prefill GEMMs): GPU suite + smoke, bench lines configs[1..4], ncu of the pair kernels
mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -2 > gpurun_out/r2s_gputest.txt; cat gpurun_out/r2s_gputest.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout -s KILL 900 python bench.py 2>&1 | tail -1 > gpurun_out/r2s_bench_c2.json
python -c "import json; d=json.load(open('gpurun_out/r2s_bench_c2.json')); print('c2', d['value'], d['e2e']['value'], d['attention_roofline']['frac'], d['attention_roofline']['inpipeline']['frac'], d['layer_roofline']['frac'], d['layer_roofline']['us_per_layer_median'], d['prefill_gemm_roofline']['frac'], d['cpu_baseline']['value'])"
timeout -s KILL 1200 python bench.py --workload c5 --model qwen25_32b --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r2s_bench_c5.json
timeout -s KILL 900 python bench.py --workload c3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r2s_bench_c3.json
timeout -s KILL 900 python bench.py --workload c4_w1 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r2s_bench_c4_w1.json
for w in c5 c3 c4_w1; do python -c "import json; d=json.load(open('gpurun_out/r2s_bench_$w.json')); print('$w', d['value'], d['e2e']['value'], d['attention_roofline']['frac'], d['layer_roofline']['frac'], (d.get('prefill_gemm_roofline') or {}).get('frac'))"; done
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_tc2_kernel|gemm_swiglu_pk2_kernel" -c 4 -o gpurun_out/r2s_prefill_pairs python tools/ncu_probes.py prefill_gemm > gpurun_out/r2s_ncu.log 2>&1; tail -1 gpurun_out/r2s_ncu.log
