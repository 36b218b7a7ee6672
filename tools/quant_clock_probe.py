"""Diagnostic: the SM clock around every K1 quantizer and K2 GEMM launch of the
layer step, eager and inside the CUDA-graph replays (tools/clock_probe.cu: a
~3 us globaltimer/clock64 spin before and after each launch), next to the
CUPTI duration of each K1 launch.  Answers: is an in-step K1 slowdown the SM
clock (power management) or something else?"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2511_05811_b200 import _lib  # noqa: E402
from paper_2511_05811_b200.nn import CudaGraphStep, MossAdamW  # noqa: E402
from paper_2511_05811_b200.workloads import LayerStack  # noqa: E402

so = os.path.join(ROOT, "tools", "_clock_probe.so")
if not os.path.exists(so):
    os.system(f"nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o {so} "
              f"{os.path.join(ROOT, 'tools', 'clock_probe.cu')}")
P = ctypes.CDLL(so)
P.clock_probe.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
buf = torch.zeros(2 * 512, dtype=torch.int64, device="cuda")
labels: list = []
NS = int(os.environ.get("PROBE_NS", "3000"))
SLEEP = int(os.environ.get("SLEEP_CYCLES", "0"))


def probe(tag):
    slot = len(labels)
    labels.append(tag)
    P.clock_probe(buf.data_ptr(), slot, NS, _lib.stream())


def wrap(name, tag_fn):
    orig = getattr(_lib, name)

    def f(*a, **k):
        tag = tag_fn(a, k)
        if SLEEP and name == "quant_mx2_fused":
            torch.cuda._sleep(SLEEP)        # experiment: idle the GPU ahead of every K1
        probe("pre " + tag)
        orig(*a, **k)
        probe("post " + tag)
    setattr(_lib, name, f)


wrap("quant_mx2_fused", lambda a, k: f"K1 {tuple(a[0].shape)} {'prod' if k.get('amax_given') else 'inkern'}")
wrap("gemm", lambda a, k: f"K2 A{tuple(a[0].shape)} B{tuple(a[2].shape)}")
wrap("gemm_bkn", lambda a, k: f"K2bkn A{tuple(a[0].shape)} B{tuple(a[2].shape)}")

torch.manual_seed(0)
model = LayerStack(device="cuda")
opt = MossAdamW(model, lr=3e-4, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.1)
x = torch.randn(8192, 4096, device="cuda", dtype=torch.bfloat16).requires_grad_(True)
one = torch.ones((), device="cuda")


def fwd_bwd(xin):
    loss = model(xin)
    loss.backward(one)
    return loss


def report(title, first_slot=0, k1_us=None):
    torch.cuda.synchronize()
    v = buf.view(-1, 2).cpu().tolist()
    print(f"== {title}")
    k = 0
    for i, tag in enumerate(labels[first_slot:], start=first_slot):
        c, ns = v[i]
        extra = ""
        if k1_us and tag.startswith("post K1") and k < len(k1_us):
            extra = f"   K1 {k1_us[k]} us"
            k += 1
        print(f"  {tag:48s} {c / max(ns, 1) * 1e3:7.0f} MHz{extra}")


def k1_times(prof, reps):
    q = [round(e.device_time, 1) for e in prof.events() if "quant_mx2" in e.name]
    n = len(q) // reps
    return q[-n:]


def eager_step():
    opt.zero_grad()
    fwd_bwd(x.detach().requires_grad_(True))
    opt.step()


from torch.profiler import ProfilerActivity, profile  # noqa: E402

for _ in range(3):
    labels.clear()
    eager_step()
for _ in range(20):
    eager_step()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        labels.clear()
        eager_step()
    torch.cuda.synchronize()
report("eager step (back to back, 23 warm steps)", 0, k1_times(prof, 3))

labels.clear()
g = CudaGraphStep(fwd_bwd, opt, (x.detach().clone().requires_grad_(True),))
g(x)                        # eager step + capture: the captured probes are the second half
first = len(labels) // 2
for _ in range(200):
    g(x)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(5):
        g(x)
    torch.cuda.synchronize()
report("graph replay (after 200 replays; the last replay's probes)", first, k1_times(prof, 5))
gm = [round(e.device_time, 1) for e in prof.events() if "gemm_mxf8" in e.name]
print("K2 us per launch, last replay:", gm[-(len(gm) // 5):])

# timeline of the last replay: start offset, duration, stream (kernels that overlap K1 show up here)
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
try:
    rows = []
    for e in evs:
        ki = e.kineto_info if hasattr(e, "kineto_info") else None
        rows.append((e.time_range.start, e.time_range.end, e.name[:60]))
    rows.sort()
    per = len(rows) // 5
    last = rows[-per:]
    t0 = last[0][0]
    prev_end = t0
    print("== last replay timeline (us): start, dur, gap-to-prev-end, name")
    for s0, e0, n in last:
        print(f"  {s0 - t0:9.1f} {e0 - s0:8.1f} {s0 - prev_end:7.1f}  {n}")
        prev_end = max(prev_end, e0)
except Exception as ex:
    print("timeline failed", ex)
