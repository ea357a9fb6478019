import sys
sys.path.insert(0, '.')
import numpy as np
from oracle.transformer import Decoder
from paper_2603_16104_b200.engine import TINY, LLAMA3_8B, Engine, EngineConfig, reduced
for model in [TINY, reduced(LLAMA3_8B, 2, vocab=32768)]:
    for n in [10, 33, 60, 64, 65, 77, 128, 130, 200]:
        rng = np.random.default_rng(n)
        prompt = rng.integers(0, model.vocab, size=n).tolist()
        eng = Engine(model, EngineConfig(pages_per_worker=256, max_calls=8, max_step_tokens=1024, max_ctx_tokens=4096))
        toks, logits = eng.generate(prompt, 1, want_logits=True)
        eng.close()
        dec = Decoder(model, max_pos=4096)
        ref_toks, ref_logits = dec.generate(prompt, 1, forced=list(toks))
        err = np.abs(logits[0] - ref_logits[0]).max() / np.abs(ref_logits[0]).max()
        print(model.name, n, f"{err:.4f}")
