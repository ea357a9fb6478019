python -m pytest tests/test_gpu_decode_attn.py -q -x 2>&1 | tail -1
python tools/attn_bench.py 2>&1 | tail -10
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:attn_decode -c 12 --csv --log-file gpurun_out/attn_dram.csv python tools/attn_bench.py > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/attn_dram.csv 5
