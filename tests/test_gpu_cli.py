"""The command-line drop-in on the B200 (`helios_b200 run --engine tiny`): a
single-operator workflow's control plane does not depend on the generated
text, so the report of the device run equals the reference CLI's (synthetic
body) byte for byte, while the workflow outputs are the transformer's tokens."""
import json

import pytest

pytestmark = pytest.mark.gpu

from test_cli_cpu import BIN, NATIVE, _cli, _ref, needs_bin  # noqa: E402
from paper_2603_16104_b200 import workloads as wl  # noqa: E402


@needs_bin
@pytest.mark.parametrize("native", [False, True])
def test_cli_device_engine_single_operator(tmp_path, native):
    wf, inputs, prof, _ = wl.c2_branches(n_branches=8, prefix_words=254, decode=16, capacity=1024, budget=128)
    flags = {"capacity": [1024], "pin_threshold": 64}
    mine = _cli(tmp_path, wf, inputs, prof, flags, extra=("--engine", "tiny"), binary=NATIVE if native else BIN)
    ref = _ref(wf, inputs, prof, flags)
    assert mine["report"] == ref["report"]
    assert mine["calls_csv"] == ref["calls_csv"] and mine["trace_csv"] == ref["trace_csv"]
    assert mine["outputs_json"] != ref["outputs_json"]  # the device transformer's tokens
    assert json.loads(mine["report"])["sim"]["decode_tokens"] == 8 * 16
