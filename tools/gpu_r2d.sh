mkdir -p gpurun_out
for s in 2 4 6 8; do echo "splits=$s"; HK_ATTN_SPLITS=$s python tools/attn_bench.py 2>&1 | grep "c2 llama"; done > gpurun_out/r2d_splits.txt 2>&1
cat gpurun_out/r2d_splits.txt
python tools/attn_trace.py 1 64 2>&1 | tail -14 > gpurun_out/r2d_trace_k1.txt; cat gpurun_out/r2d_trace_k1.txt
python tools/attn_trace.py 128 64 2>&1 | tail -14 > gpurun_out/r2d_trace_k128.txt; cat gpurun_out/r2d_trace_k128.txt
