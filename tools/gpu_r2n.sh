python tools/attn_trace.py 1 64 2>&1 | tail -14
python tools/attn_chunks.py 1 64 2>&1 | tail -6
python tools/attn_chunks.py 1 144 qwen 2>&1 | tail -12
