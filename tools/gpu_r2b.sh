mkdir -p gpurun_out
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x --timeout 900 --deselect tests/test_gpu_parity.py::test_bf16_configs1_full_depth_llama3_8b_sample -k "not fp32_free_running" 2>&1 | tail -15 > gpurun_out/r2b_tests.txt
cat gpurun_out/r2b_tests.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
