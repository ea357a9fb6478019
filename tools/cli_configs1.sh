# configs[1] through the self-contained command line with the Llama-3-8B-shaped engine (B200)
mkdir -p gpurun_out/cli
python - <<'PY'
import json, sys
sys.path.insert(0, ".")
from paper_2603_16104_b200 import workloads as wl
wf, inp, prof, spec = wl.c2_branches()
for n, d in (("wf", wf), ("in", inp), ("prof", prof)):
    open(f"gpurun_out/cli/{n}.json", "w").write(json.dumps(d))
print(spec)
PY
start=$(date +%s.%N); paper_2603_16104_b200/helios_b200 run --workflow gpurun_out/cli/wf.json --inputs gpurun_out/cli/in.json \
  --profile gpurun_out/cli/prof.json --capacity 262144 --prefill-budget 8192 --engine llama3_8b \
  --out gpurun_out/cli/report.json --calls-out gpurun_out/cli/calls.csv --outputs-out gpurun_out/cli/outputs.json 2> gpurun_out/cli/stderr.txt
rc=$?; end=$(date +%s.%N); echo "rc=$rc wall_s=$(python -c "print($end-$start)")"; cat gpurun_out/cli/stderr.txt; python -c "import json; d=json.load(open('gpurun_out/cli/report.json')); print(json.dumps(d['sim']), d['makespan'], d['calls'])"
rm -f gpurun_out/cli/*.json.bak
