mkdir -p gpurun_out
HK_GEMM_TRACE=1 HK_NO_GRAPHS=1 timeout -s KILL 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-profile > gpurun_out/r2c_bench_trace.json 2>&1
python tools/gemm_trace.py gpurun_out/gemm_trace.csv | tee gpurun_out/r2c_spans.txt
python tools/attn_bench.py 2>&1 | tail -12 | tee gpurun_out/r2c_attn_bench.txt
timeout -s KILL 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/r2c_bench.json
python -c "import json; d=json.load(open('gpurun_out/r2c_bench.json')); print('value', d['value'], 'e2e', d['e2e']['value'], 'gemm', d['roofline']['frac'], d['roofline'].get('inpipeline',{}).get('frac'), 'attn', d['attention_roofline']['frac'], d['attention_roofline'].get('inpipeline',{}).get('frac')); print(d['kernel_ms_per_step'])"
