mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -5 > gpurun_out/gputest.txt; cat gpurun_out/gputest.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python tools/attn_bench.py 2>&1 | tail -11 > gpurun_out/attn_bench.txt; cat gpurun_out/attn_bench.txt
timeout -s KILL 900 python bench.py 2>&1 | tail -1 > gpurun_out/bench.json
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print('value', d['value'], 'e2e', d['e2e']['value'], 'gemm frac', d['roofline']['frac'], 'attn frac', d['attention_roofline']['frac'], d['attention_roofline']['inpipeline']['frac'], 'layer', d['layer_roofline'])"
