mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -q -x --timeout 400 2>&1 | tail -15 | tee gpurun_out/t_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3 | tee gpurun_out/smoke.log
for a in "16 1024 2048 256" "16 1024 12288 256"; do python tools/smoke_probe.py $a 2>&1 | tail -1; done
