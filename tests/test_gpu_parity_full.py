"""Full-size parity at BASELINE configs[1] (M = 8192, Llama-7B linears)
against the CPU oracle, and the product's dequantize against golden vectors
made by the reference.

* every one of the 12 layer GEMMs (fwd, MN-major dgrad, f32 wgrad of QKV, O,
  gate_up, down) on sampled output rows vs the float64 oracle evaluated on
  the GPU's own codes and scales (oracle/numpy_ref: dequantize_two_level /
  dequantize_per_tensor / gemm_f64 = gemm.py:115-129 to <= 1e-10);
* the quantizer at 8192 x 11008 and 8192 x 22016, row- and column-wise, in
  both amax modes, bit-exact vs the C restatement (quantize.py:127-173).

GEMM gates, stated up front:
  f32 output:  |got - ref| <= 1e-5 * mag   and rel-Frobenius <= 1e-5,
               mag = s_a s_b sum_k |a_k||b_k| (FP32 accumulation reordering);
  bf16 output: |got - ref| <= 2^-8 |ref| + 1.01e-5 * mag, rel-Frobenius <= 2^-8 + 1e-5:
               the f32 gate plus round-to-nearest into bf16 (8-bit significand,
               unit roundoff 2^-8) — derived, not fitted.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2511_05811_b200 as P  # noqa: E402
from paper_2511_05811_b200 import _lib  # noqa: E402
from paper_2511_05811_b200.gemm import mx_gemm, mx_gemm_bkn  # noqa: E402
from paper_2511_05811_b200.quantize import TwoLevelQuant, quantize_mx2  # noqa: E402

from oracle import numpy_ref as R  # noqa: E402

from .helpers import rel_frob  # noqa: E402

M = 8192
SHAPES = {"qkv": (4096, 12288), "o": (4096, 4096), "gate_up": (4096, 22016), "down": (11008, 4096)}
F32_TOL = 1e-5
BF16_U = 2.0 ** -8
SAMPLE = 64


def host(t):
    return t.detach().cpu().numpy()


def _deq2(codes, micro, g):
    return R.dequantize_two_level(R.TwoLevel(codes, float(g), micro))


def _check(got, ref, mag, bf16):
    err = np.abs(got - ref)
    if bf16:
        assert np.all(err <= BF16_U * np.abs(ref) + 1.01 * F32_TOL * mag), float(np.max(err / (mag + 1e-30)))
        assert rel_frob(got, ref) <= BF16_U + F32_TOL
    else:
        assert float(np.max(err / (mag + 1e-30))) <= F32_TOL
        assert rel_frob(got, ref) <= F32_TOL


@pytest.mark.parametrize("name", list(SHAPES))
@pytest.mark.parametrize("kind", ["fwd", "dgrad", "wgrad"])
def test_layer_gemm_vs_f64_oracle(name, kind):
    K, N = SHAPES[name]
    g = torch.Generator(device="cuda").manual_seed(K * 7 + N)
    rng = np.random.default_rng(K + N)
    fl = _lib.FlagWord("cuda")
    if kind in ("fwd", "dgrad"):
        kk, nn = (K, N) if kind == "fwd" else (N, K)           # contraction / output width
        a = torch.randn(M, kk, device="cuda", generator=g).to(torch.bfloat16)
        a.view(-1)[torch.randint(0, a.numel(), (a.numel() // 1000,), device="cuda", generator=g)] *= 50
        w = torch.randn(N, K, device="cuda", generator=g) * 0.02            # the layer weight [out, in]
        qa = quantize_mx2(a, row=True, micro=True, flags=fl)
        qw = P.quant_per_tensor(w)
        if kind == "fwd":
            d = mx_gemm(qa.codes, qa.sf, qa.g, qw.codes, None, qw.scale.reshape(1), out_dtype=torch.bfloat16)
            b_deq = R.dequantize_per_tensor(host(qw.codes), float(qw.scale)).T      # [K, N]
        else:
            d = mx_gemm_bkn(qa.codes, qa.sf, qa.g, qw.codes, qw.scale.reshape(1))   # dY . W, W as stored
            b_deq = R.dequantize_per_tensor(host(qw.codes), float(qw.scale))        # [N, K]
        rows = rng.choice(M, SAMPLE, replace=False)
        a_deq = _deq2(host(qa.codes)[rows], host(qa.micro)[rows], qa.g.item())
        bf16 = True
    else:
        # wgrad: dW[N, K] = dY^T X, both operands column-wise two-level (blocks along tokens)
        dy = (torch.randn(M, N, device="cuda", generator=g) * 1e-3).to(torch.bfloat16)
        x = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
        qd = quantize_mx2(dy, row=False, col=True, micro=True, flags=fl)
        qx = quantize_mx2(x, row=False, col=True, micro=True, flags=fl)
        d = torch.empty(N, K, device="cuda", dtype=torch.float32)
        mx_gemm(qd.codes_t, qd.sf_t, qd.g, qx.codes_t, qx.sf_t, qx.g, out=d)
        rows = rng.choice(N, SAMPLE, replace=False)
        a_deq = _deq2(host(qd.codes_t)[rows], host(qd.micro_t)[rows], qd.g.item())
        b_deq = _deq2(host(qx.codes_t), host(qx.micro_t), qx.g.item()).T             # [M, K]
        bf16 = False
    fl.raise_if_set(f"{name} {kind}")
    ref = a_deq @ b_deq
    mag = np.abs(a_deq) @ np.abs(b_deq)
    got = host(d.float())[rows]
    _check(got, ref, mag, bf16)


@pytest.mark.parametrize("cols", [11008, 22016])
@pytest.mark.parametrize("producer_amax", [False, True])
def test_quantizer_full_size_vs_c_oracle(c_oracle, cols, producer_amax):
    torch.manual_seed(cols)
    x = torch.randn(M, cols, device="cuda").to(torch.bfloat16)
    x.view(-1)[torch.randint(0, x.numel(), (x.numel() // 1000,), device="cuda")] *= 50
    fl = _lib.FlagWord("cuda")
    am = x.float().abs().max().reshape(1) if producer_amax else None
    q = quantize_mx2(x, row=True, col=True, micro=True, flags=fl, amax=am)
    fl.raise_if_set("quant")
    xf = host(x.float())
    codes, micro, gv, st = c_oracle.quant_two_level_mt(xf)
    assert st == 0 and float(q.g.item()) == gv
    assert np.array_equal(host(q.codes), codes) and np.array_equal(host(q.micro), micro)
    codes_t, micro_t, gt, st = c_oracle.quant_two_level_mt(np.ascontiguousarray(xf.T))
    assert st == 0 and gt == gv
    assert np.array_equal(host(q.codes_t), codes_t) and np.array_equal(host(q.micro_t), micro_t)


@pytest.mark.parametrize("producer_amax", [False, True])
def test_quantizer_tiny_gradients_vs_c_oracle(c_oracle, producer_amax):
    """Late-training output-gradients: tensor amax ~2^-40 and block maxima spread
    over 2^-40 .. 2^-110, so most blocks fall outside the fast path's
    eff in [2^-60, 2^60) and take the general (scaled) path — bit-exact vs the
    C restatement at the qkv output-gradient shape, row- and column-wise."""
    torch.manual_seed(5)
    x = torch.randn(M, 12288, device="cuda") * 2.0 ** -40
    rs = torch.pow(2.0, -torch.randint(0, 70, (M, 1), device="cuda").float())        # per-row decades
    cs = torch.pow(2.0, -torch.randint(0, 4, (1, 12288), device="cuda").float())
    x = (x * rs * cs).to(torch.bfloat16)
    x.view(-1)[7::4099] = -0.0
    fl = _lib.FlagWord("cuda")
    am = x.float().abs().max().reshape(1) if producer_amax else None
    q = quantize_mx2(x, row=True, col=True, micro=True, flags=fl, amax=am)
    fl.raise_if_set("quant")
    xf = host(x.float())
    codes, micro, gv, st = c_oracle.quant_two_level_mt(xf)
    assert st == 0 and float(q.g.item()) == gv
    assert int((micro < 127 - 20).sum()) > micro.size // 4          # the general path is exercised
    assert np.array_equal(host(q.codes), codes) and np.array_equal(host(q.micro), micro)
    codes_t, micro_t, gt, st = c_oracle.quant_two_level_mt(np.ascontiguousarray(xf.T))
    assert st == 0 and gt == gv
    assert np.array_equal(host(q.codes_t), codes_t) and np.array_equal(host(q.micro_t), micro_t)


def test_dequantize_matches_reference(golden):
    """quantize.dequantize (device) == the reference's dequantize (golden_r2.npz)."""
    import os
    g2 = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_r2.npz"))
    for case in golden["q2l_cases"]:
        codes = torch.as_tensor(golden[f"q2l_{case}_codes"], device="cuda")
        micro = torch.as_tensor(golden[f"q2l_{case}_micro"], device="cuda")
        gs = torch.tensor(float(golden[f"q2l_{case}_g"]), dtype=torch.float32, device="cuda")
        q = TwoLevelQuant(codes=codes, global_scale=gs, micro_codes=micro, fmt=P.E4M3)
        got = host(P.dequantize(q))
        want = g2[f"deq2_{case}"]
        assert got.dtype == want.dtype == np.float32
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), case
    for case in ("exact", "two", "gauss", "w"):
        codes = torch.as_tensor(golden[f"qpt_{case}_codes"], device="cuda")
        sc = torch.tensor(float(golden[f"qpt_{case}_scale"]), dtype=torch.float32, device="cuda")
        got = host(P.dequantize(P.PerTensorQuant(codes=codes, scale=sc, fmt=P.E4M3)))
        assert np.array_equal(got.view(np.uint32), g2[f"deqpt_{case}"].view(np.uint32)), case
