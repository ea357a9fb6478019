mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x --timeout 400 2>&1 | tail -3
timeout -s KILL 900 python bench.py --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench.json
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print('value', d['value'], 'e2e', d['e2e']['value'], 'gemm frac', d['roofline']['frac'], 'attn frac', d['attention_roofline']['frac']); print(d['kernel_ms_per_step'])"
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 1400 -c 660 --csv \
   --log-file gpurun_out/launches.csv python bench.py --workload c2_short --steps 1 --warmup 0 --no-cpu-baseline --no-profile > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches.csv 16
