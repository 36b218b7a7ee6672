"""Find the step-105 loss spike of the configs[2] GPU run: train to step 104,
then evaluate batch 105 through the fused path and through torch glue (same
weights), and report per-block activation statistics."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from make_llama125m_curve import RUN  # noqa: E402
from oracle.train_ref import seeded_init  # noqa: E402
from paper_2511_05811_b200 import llama as L  # noqa: E402
from paper_2511_05811_b200.trainer import train  # noqa: E402

STOP = int(os.environ.get("STOP", 105))
cfg = L.LlamaConfig(**{**L.LLAMA_125M.__dict__, "max_seq": RUN["seq"]})
model = L.LlamaModel(cfg)
seeded_init(model, RUN["init_seed"])
data = L.MarkovTokens(cfg.vocab, seed=RUN["data_seed"], active=RUN["active"])
from paper_2511_05811_b200.trainer import make_optimizer  # noqa: E402
opt = make_optimizer(model, RUN["lr"], RUN["steps"], RUN["warmup"])    # the 200-step schedule
losses = []
for _ in range(STOP):
    bx, by = data.batch(RUN["batch"], RUN["seq"])
    opt.zero_grad()
    loss = model(torch.as_tensor(bx, device="cuda"), torch.as_tensor(by, device="cuda"))
    loss.backward()
    opt.step()
    opt.check()
    losses.append(float(loss))
print("last losses", losses[-3:])
x, y = data.batch(RUN["batch"], RUN["seq"])          # the batch of step STOP
xt, yt = torch.as_tensor(x, device="cuda"), torch.as_tensor(y, device="cuda")
stats = {}


def hook(name):
    def f(mod, inp, out):
        o = out[0] if isinstance(out, tuple) else out
        of = o.float()
        stats.setdefault(name, []).append((float(of.abs().max()), float(of.pow(2).mean().sqrt()),
                                           bool(torch.isfinite(of).all())))
    return f


for i, blk in enumerate(model.blocks):
    for n in ("qkv", "o", "gate_up", "down"):
        getattr(blk, n).register_forward_hook(hook(f"b{i}.{n}"))
with torch.no_grad():
    lf = float(model(xt, yt))
    glue = L.LlamaModel(L.LlamaConfig(**{**cfg.__dict__, "fused_ops": False}))
    glue.load_state_dict(model.state_dict())
    for a, b in zip(glue.modules(), model.modules()):
        if hasattr(b, "schedule") and b.schedule is not None:
            a.schedule = b.schedule
            a.w_fp8.copy_(b.w_fp8)
            a.w_scale.copy_(b.w_scale)
    for i, blk in enumerate(glue.blocks):
        for n in ("qkv", "o", "gate_up", "down"):
            getattr(blk, n).register_forward_hook(hook(f"g{i}.{n}"))
    lg = float(glue(xt, yt))
    bf = L.LlamaModel(L.LlamaConfig(**{**cfg.__dict__, "moss": False}))
    sd = {k: v for k, v in model.state_dict().items()}
    bf.load_state_dict(sd, strict=False)
    lb = float(bf(xt, yt))
    f32 = L.LlamaModel(L.LlamaConfig(**{**cfg.__dict__, "moss": False, "compute_dtype": torch.float32}))
    f32.load_state_dict(sd, strict=False)
    l32 = float(f32(xt, yt))
    logits = model(xt)
    lgf = logits.float()
    per_tok = torch.nn.functional.cross_entropy(lgf.view(-1, lgf.shape[-1]), yt.view(-1), reduction="none")
    l32t = torch.nn.functional.cross_entropy(f32(xt).view(-1, lgf.shape[-1]), yt.view(-1), reduction="none")
    print("logits max", float(lgf.abs().max()), "per-token loss max", float(per_tok.max()),
          "tokens with loss > 20:", int((per_tok > 20).sum()), "of", per_tok.numel())
    bad = (per_tok - l32t).abs().argsort(descending=True)[:5]
    print("worst tokens (fused vs f32):", [(int(i), round(float(per_tok[i]), 3), round(float(l32t[i]), 3)) for i in bad])
print(f"step {STOP}: fused {lf:.4f}  torch-glue {lg:.4f}  bf16-linears {lb:.4f}  f32-linears-f32-glue {l32:.4f}")
for k in sorted(stats):
    print(k, [tuple(round(v, 4) if isinstance(v, float) else v for v in t) for t in stats[k]])
