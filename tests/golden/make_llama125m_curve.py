"""Generate the CPU reference loss curves of BASELINE configs[2] (~125M Llama
decoder, 200 synthetic-token steps):  tests/golden/llama125m_curve_<name>.npz

    python tests/golden/make_llama125m_curve.py <name>      (~2 h each on 8 cores)

The run is oracle/train_ref.reference_curve: every linear is the composed
MOSS oracle (quant_two_level / per-tensor weight encode at s_t / float64
GEMMs, train.py:162-174 with the FP8 backward of north_star (2)), the
optimizer is adamw_step + auto_scale_advance + rescale (optim.py:78-106,
autoscale.py:71-96), the lr schedule is lr_at (train.py:75-82), glue ops in
float64.  tests/test_gpu_llama.py runs the same model on the GPU from the
same seeded init and data and compares the curves.

Two runs (the Markov-chain task's loss has a plateau at the unigram entropy
whose ESCAPE is chaotic — any numerical difference, even float32 vs float64
glue on one GPU, moves it by tens of steps — so the parity bands are set per
regime):
  plateau   2048 active states, lr 1e-3: 200 steps, the first ~100 of which
            (descent + plateau) are compared point by point;
  converge  128 active states, lr 3e-4: a smooth run in which the chain is
            learned (tools/c3_config_search.py picked it: its bf16-vs-f32-glue
            GPU curves stay within 2 %); compared point by point and at the end.
"""

import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.train_ref import reference_curve  # noqa: E402
from paper_2511_05811_b200.llama import LLAMA_125M, LlamaConfig  # noqa: E402

RUNS = {
    "plateau": dict(steps=200, batch=8, seq=256, lr=1e-3, warmup=20, data_seed=1, init_seed=7, active=2048),
    "converge": dict(steps=200, batch=8, seq=256, lr=3e-4, warmup=20, data_seed=1, init_seed=7, active=128),
}


def path(name: str) -> str:
    return os.path.join(os.path.dirname(os.path.abspath(__file__)), f"llama125m_curve_{name}.npz")


def main(name: str) -> None:
    torch.set_num_threads(os.cpu_count())
    run = RUNS[name]
    cfg = LlamaConfig(**{**LLAMA_125M.__dict__, "max_seq": run["seq"]})
    t0 = time.time()

    def log(step, loss):
        print(f"step {step:4d} loss {loss:.5f}  {time.time() - t0:7.1f} s", flush=True)
    losses = reference_curve(cfg, log=log, **run)
    np.savez(path(name), loss=np.asarray(losses, np.float64), **{k: np.asarray(v) for k, v in run.items()},
             cfg=np.asarray(repr(cfg)), seconds=np.asarray(time.time() - t0))
    print("wrote", path(name))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "plateau")
