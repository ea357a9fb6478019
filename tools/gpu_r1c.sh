# round-1 (session c) verification + evidence: tests, smoke, kernel table, bench line, ncu launch list + full captures
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x --timeout 400 2>&1 | tail -2
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout -s KILL 300 python tools/attn_bench.py 2>&1 | tail -11 > gpurun_out/attn_bench_r1c.txt; cat gpurun_out/attn_bench_r1c.txt
timeout -s KILL 900 python bench.py 2>&1 | tail -1 > gpurun_out/bench_r1c.json
python -c "import json; d=json.load(open('gpurun_out/bench_r1c.json')); print('value', d['value'], 'e2e', d['e2e']['value'], 'cpu', d.get('cpu_baseline',{}).get('value'), 'frac', d['roofline']['frac'], 'attn', d['attention_roofline']['frac'])"
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 1400 -c 520 --csv \
   --log-file gpurun_out/launches_r1c.csv python bench.py --workload c2_short --steps 1 --warmup 0 --no-cpu-baseline --no-profile > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_r1c.csv 14 > gpurun_out/launches_r1c.txt; cat gpurun_out/launches_r1c.txt
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:attn_decode -s 200 -c 1 \
   -o gpurun_out/attn_r1c python bench.py --workload c2_short --steps 1 --warmup 0 --no-cpu-baseline --no-profile > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 1600 -c 4 \
   -o gpurun_out/gemm_r1c python bench.py --workload c2_short --steps 1 --warmup 0 --no-cpu-baseline --no-profile > /dev/null 2>&1
ls -la gpurun_out/*r1c*
