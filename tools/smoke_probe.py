import json, sys, itertools
sys.path.insert(0, '.')
from paper_2603_16104_b200 import helios, workloads as wl
from paper_2603_16104_b200.engine import TINY, Engine, EngineConfig, pages_for
blob, meta = wl.load_plan("t_small")
gold = json.loads(open("tests/golden/t_small.ref.json").read())
sc = wl.sim_config_from_meta(meta)
mc, ms, mx, mp = [int(a) for a in sys.argv[1:5]]
eng = Engine(TINY, EngineConfig(pages_per_worker=pages_for(sc, mc, mp), max_calls=mc, max_step_tokens=ms, max_ctx_tokens=mx))
try:
    m = helios.simulate(blob, sc, engine=eng, verify_lookup=True)
    print(sys.argv[1:], "ok", m.metrics_json == gold["metrics_json"])
except Exception as e:
    print(sys.argv[1:], "FAIL", str(e)[:100])
