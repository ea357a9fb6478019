# round 2: first parity run on the box (host resources, fp32 exact, bf16 derived-margin checks)
mkdir -p gpurun_out
nproc; free -g | head -2
timeout -s KILL 1500 python -m pytest tests/test_gpu_parity.py -q -rA --timeout 900 -s 2>&1 | tail -40 > gpurun_out/r2a_parity.txt
cat gpurun_out/r2a_parity.txt | tail -40
