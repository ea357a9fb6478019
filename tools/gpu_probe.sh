mkdir -p gpurun_out
HK_NO_GRAPHS=1 HK_NO_PDL=1 timeout -s KILL 600 compute-sanitizer --tool initcheck --print-limit 8 python tools/smoke_probe.py 16 1024 2048 256 > gpurun_out/initcheck.log 2>&1
grep -v "Host Frame" gpurun_out/initcheck.log | head -80
