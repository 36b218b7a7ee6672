"""GPU side of the configs[2] comparison (tests/test_gpu_llama.py), saving the
per-step losses to gpurun_out/llama125m_gpu.npy for inspection."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import numpy as np  # noqa: E402

from make_llama125m_curve import RUNS  # noqa: E402

RUN = RUNS[os.environ.get("RUN", "plateau")]
from oracle.train_ref import seeded_init  # noqa: E402
from paper_2511_05811_b200 import llama as L  # noqa: E402
from paper_2511_05811_b200.trainer import train  # noqa: E402

cfg = L.LlamaConfig(**{**L.LLAMA_125M.__dict__, "max_seq": RUN["seq"]})
model = L.LlamaModel(cfg)
seeded_init(model, RUN["init_seed"])
log = train(model, L.MarkovTokens(cfg.vocab, seed=RUN["data_seed"], active=RUN["active"]), steps=RUN["steps"],
            batch=RUN["batch"], seq=RUN["seq"], lr=RUN["lr"], warmup=RUN["warmup"],
            cuda_graph=os.environ.get("GRAPH", "1") == "1")
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
np.save(os.path.join(ROOT, "gpurun_out", os.environ.get("OUT", "llama125m_gpu") + ".npy"), np.asarray(log.loss))
print("losses", [round(v, 4) for v in log.loss[::20]], log.loss[-1])
