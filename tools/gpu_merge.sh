timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:attn_merge_rows -s 5 -c 1 -o gpurun_out/merge_full python tools/attn_bench.py > /dev/null 2>&1
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:attn_ -c 30 --csv --log-file gpurun_out/attn_launch.csv python tools/attn_bench.py > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/attn_launch.csv 10
