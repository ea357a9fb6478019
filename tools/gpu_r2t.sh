# round-2 final evidence (persistent pair prefill GEMMs, step ABI): GPU suite + smoke, bench lines configs[1..4],
# ncu of the pair kernels and the decode attention
mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -2 > gpurun_out/r2t_gputest.txt; cat gpurun_out/r2t_gputest.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout -s KILL 900 python bench.py 2>&1 | tail -1 > gpurun_out/r2t_bench_c2.json
python -c "import json; d=json.load(open('gpurun_out/r2t_bench_c2.json')); print('c2', d['value'], d['e2e']['value'], d['attention_roofline']['frac'], d['attention_roofline']['inpipeline']['frac'], d['layer_roofline']['frac'], d['layer_roofline']['us_per_layer_median'], d['prefill_gemm_roofline']['frac'], d['cpu_baseline']['value'])"
timeout -s KILL 1200 python bench.py --workload c5 --model qwen25_32b --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r2t_bench_c5.json
timeout -s KILL 900 python bench.py --workload c3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r2t_bench_c3.json
timeout -s KILL 900 python bench.py --workload c4_w1 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r2t_bench_c4_w1.json
for w in c5 c3 c4_w1; do python -c "import json; d=json.load(open('gpurun_out/r2t_bench_$w.json')); print('$w', d['value'], d['e2e']['value'], d['attention_roofline']['frac'], d['layer_roofline']['frac'])"; done
timeout -s KILL 300 python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -1 > gpurun_out/r2t_bench_ref.json; head -c 300 gpurun_out/r2t_bench_ref.json; echo
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_rows_pk2_kernel|gemm_swiglu_pk2_kernel|gemm_tc2_kernel" -c 6 -o gpurun_out/r2t_prefill_pairs python tools/ncu_probes.py prefill_gemm > gpurun_out/r2t_ncu.log 2>&1; tail -1 gpurun_out/r2t_ncu.log
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:attn_decode_kernel -c 1 -o gpurun_out/r2t_attn_c5_k128 python tools/ncu_probes.py attn_c5 128 > gpurun_out/r2t_ncu2.log 2>&1; tail -1 gpurun_out/r2t_ncu2.log
