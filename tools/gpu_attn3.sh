mkdir -p gpurun_out
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:attn_ -c 2 -o gpurun_out/attn_full2 python tools/attn_bench.py > gpurun_out/ncu_attn.log 2>&1
tail -1 gpurun_out/ncu_attn.log
