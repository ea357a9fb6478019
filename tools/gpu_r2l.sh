mkdir -p gpurun_out
for k in 1 128 256; do echo "=== trace k=$k"; python tools/attn_trace.py $k 64 2>&1 | tail -16; echo "=== items k=$k"; python tools/attn_items.py $k 2>&1 | tail -8; echo "=== chunks k=$k"; python tools/attn_chunks.py $k 64 2>&1 | tail -8; done > gpurun_out/r2l_traces.txt 2>&1
cat gpurun_out/r2l_traces.txt
