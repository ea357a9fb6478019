# whole-run A/B of an env switch on configs[1] ($1 = env assignment for B); prints value / attention fracs
mkdir -p gpurun_out
run() { env $1 timeout -s KILL 900 python bench.py --no-cpu-baseline --steps 3 --warmup 3 2>&1 | tail -1 > gpurun_out/ab.json; python -c "
import json; d=json.load(open('gpurun_out/ab.json')); a=d['attention_roofline']
print('$1', 'value %.0f e2e %.0f attn frac %.3f inpipe %.3f layer us %.1f' % (d['value'], d['e2e']['value'], a['frac'], a['inpipeline']['frac'], d['layer_roofline']['us_per_layer_median']))"; }
run HK_NOTHING=1
run "$1"
run HK_NOTHING=1
run "$1"
