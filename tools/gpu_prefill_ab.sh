# A/B of an env switch ($1) on the prefill-heavy paths: configs[1] pin precompute + run, and C4' W=1
mkdir -p gpurun_out
run() { env $1 timeout -s KILL 900 python bench.py --workload $2 --no-cpu-baseline --no-profile --steps 2 --warmup 2 2>&1 | tail -1 > gpurun_out/ab.json; python -c "
import json; d=json.load(open('gpurun_out/ab.json'))
print('$1 $2', 'value %.0f ms/step %.1f pin ms %.2f' % (d['value'], d['ms_per_step'], d['config'].get('pin_precompute_ms_per_step', 0)))"; }
for w in c2 c4_w1; do run HK_NOTHING=1 $w; run "$1" $w; run HK_NOTHING=1 $w; run "$1" $w; done
