set -x
mkdir -p gpurun_out
HK_NO_GRAPHS=1 HK_NO_PDL=1 timeout -s KILL 600 compute-sanitizer --tool memcheck --print-limit 5 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_san.log 2>&1
tail -60 gpurun_out/smoke_san.log
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 30000 -c 900 --csv \
   --log-file gpurun_out/launches_r1.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-profile > gpurun_out/ncu1.log 2>&1
tail -3 gpurun_out/ncu1.log
