import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import torch
from test_gpu_decode_attn import make_case, run, reference, CASES
H, Hkv, groups = CASES["ragged"]
for gsel in range(len(groups)):
    case = make_case(H, Hkv, [groups[gsel]], seed=7)
    out, _, _ = run(case)
    ref = reference(case)
    err = (out.float() - ref).abs().amax(dim=(1, 2))
    print("group", groups[gsel][:2], "row err", [round(e, 4) for e in err.tolist()], "scale", round(ref.abs().max().item(), 3))
