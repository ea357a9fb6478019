mkdir -p gpurun_out
python tools/attn_dbg.py 2>&1 | tail -8
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/attn_launch.csv python tools/attn_bench.py > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/attn_launch.csv 10
