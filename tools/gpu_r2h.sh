mkdir -p gpurun_out
timeout -s KILL 1800 python -m pytest tests -m gpu -q --timeout 900 2>&1 | tail -6 > gpurun_out/r2h_gputests.txt
cat gpurun_out/r2h_gputests.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
