"""Generate tests/golden/llama125m_curve.npz — the CPU reference loss curve
of BASELINE configs[2] (~125M Llama decoder, 200 synthetic-token steps).

Run once in the CPU container (it takes ~1 h on 8 cores):
    python tests/golden/make_llama125m_curve.py
The run is oracle/train_ref.reference_curve: every linear is the composed
MOSS oracle (quant_two_level / per-tensor weight encode at s_t / float64
GEMMs, train.py:162-174 with the FP8 backward of north_star (2)), the
optimizer is adamw_step + auto_scale_advance + rescale (optim.py:78-106,
autoscale.py:71-96), the lr schedule is lr_at (train.py:75-82), glue ops in
float64.  tests/test_gpu_llama.py runs the same model on the GPU from the
same seeded init and data and compares the curves.
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

# the run both sides make (tests/test_gpu_llama.py imports RUN)
RUN = dict(steps=200, batch=8, seq=256, lr=1e-3, warmup=20, data_seed=1, init_seed=7, active=2048)


def main(steps=None):
    torch.set_num_threads(os.cpu_count())
    run = dict(RUN)
    if steps is not None:
        run["steps_generated"] = steps
    cfg = LlamaConfig(**{**LLAMA_125M.__dict__, "max_seq": RUN["seq"]})
    t0 = time.time()

    def log(step, loss):
        print(f"step {step:4d} loss {loss:.5f}  {time.time() - t0:7.1f} s", flush=True)
    kw = {k: v for k, v in RUN.items()}
    losses = reference_curve(cfg, log=log, **kw) if steps is None else None
    if losses is None:      # timing probe only
        return
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "llama125m_curve.npz")
    np.savez(out, loss=np.asarray(losses, np.float64), **{k: np.asarray(v) for k, v in RUN.items()},
             cfg=np.asarray(repr(cfg)), seconds=np.asarray(time.time() - t0))
    print("wrote", out)


if __name__ == "__main__":
    main()
