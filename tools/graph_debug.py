"""CUDA-graph capture checks of MossLinear / MossAdamW pieces one at a time (which
op breaks capture).  Diagnostic only."""
import sys, os, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_05811_b200.nn import MossLinear, MossAdamW

def try_capture(name, fn, warm):
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3): warm()
    torch.cuda.current_stream().wait_stream(s); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.graph(g, stream=s):
            fn()
        g.replay(); torch.cuda.synchronize()
        print(name, "OK", flush=True)
    except Exception as e:
        print(name, "FAIL", str(e).splitlines()[0], flush=True)
        torch.cuda.synchronize()

torch.manual_seed(0)
x = torch.randn(256, 512, device="cuda", dtype=torch.bfloat16)
lin = torch.nn.Linear(512, 512, device="cuda", dtype=torch.bfloat16)
def tfb():
    y = lin(x); (y.float()**2).mean().backward()
try_capture("torch linear fwd+bwd", tfb, tfb)

m = MossLinear(512, 512)
m.init_fp8()
def f(): m(x)
try_capture("moss fwd", f, f)
xr = x.clone().requires_grad_(False)
def fb():
    y = m(xr); (y.float()**2).mean().backward()
try_capture("moss fwd+bwd (no input grad)", fb, fb)
xg = x.clone().requires_grad_(True)
def fb2():
    y = m(xg); (y.float()**2).mean().backward()
try_capture("moss fwd+bwd (input grad)", fb2, fb2)
opt = MossAdamW(m.parameters())
def fbo():
    y = m(xr); (y.float()**2).mean().backward(); opt.launch(False)
def fbo_w():
    y = m(xr); (y.float()**2).mean().backward(); opt.step()
try_capture("moss fwd+bwd+opt", fbo, fbo_w)

from paper_2511_05811_b200.workloads import LayerStack
from paper_2511_05811_b200.nn import CudaGraphStep
torch.manual_seed(0)
st = LayerStack(d_model=512, d_ffn=1024)
o2 = MossAdamW(st)
xs = torch.randn(512, 512, device="cuda", dtype=torch.bfloat16)
def sfb(): st(xs).backward()
def sfbo(): st(xs).backward(); o2.launch(False)
def sfbo_w(): o2.zero_grad(); st(xs).backward(); o2.step()
try_capture("stack fwd+bwd", sfb, sfb)
try_capture("stack fwd+bwd+opt", sfbo, sfbo_w)
# exact bench flow: eager steps on the default stream, then CudaGraphStep
torch.manual_seed(1)
st2 = LayerStack(d_model=512, d_ffn=1024)
o3 = MossAdamW(st2)
def fwd_bwd(xin):
    loss = st2(xin); loss.backward(); return loss
for _ in range(3):
    o3.zero_grad(); fwd_bwd(xs); o3.step()
torch.cuda.synchronize()
try:
    gs = CudaGraphStep(fwd_bwd, o3, (xs.clone(),))
    for _ in range(4): l = gs(xs)
    torch.cuda.synchronize(); print("CudaGraphStep flow OK", float(l), flush=True)
except Exception as e:
    print("CudaGraphStep flow FAIL", str(e).splitlines()[0], flush=True)
    traceback.print_exc()
