python tools/attn_private_only.py 128
python tools/attn_private_only.py 512
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:attn_decode -s 2 -c 1 -o gpurun_out/priv_full python tools/attn_private_only.py 512 > /dev/null 2>&1
ls gpurun_out/priv_full.ncu-rep
