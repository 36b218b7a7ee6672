"""The single-launch quantizer (moss_quant_mx2_fused, csrc/quant_v4.cu): the
in-kernel amax + grid barrier + quantize must reproduce the two-launch path
(moss_amax + moss_quant_mx2, itself pinned to the CPU oracle in
test_gpu_kernels.py) bit for bit, at every tiling corner, across repeated
launches (barrier generations), with a producer-supplied amax, under CUDA
graph capture, and raise the reference's errors (quantize.py:88, fp8.py:219)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2511_05811_b200.quantize as Q  # noqa: E402
from paper_2511_05811_b200 import _lib, errors  # noqa: E402
from paper_2511_05811_b200.nn import raise_if_flagged  # noqa: E402


def _both(x, row=True, col=True, micro=True, monkeypatch=None):
    outs = []
    for fused in (True, False):
        monkeypatch.setattr(Q, "FUSED", fused)
        fl = _lib.FlagWord()
        am = torch.empty(1, device="cuda")
        op = Q.quantize_mx2(x, row=row, col=col, micro=micro, flags=fl, amax_buf=am)
        fl.raise_if_set("quant")
        outs.append((op, am))
    return outs


def _assert_same(a, b):
    (oa, ama), (ob, amb) = a, b
    assert torch.equal(ama, amb)
    assert torch.equal(oa.g, ob.g)
    for name in ("codes", "sf", "micro", "codes_t", "sf_t", "micro_t"):
        ta, tb = getattr(oa, name), getattr(ob, name)
        assert (ta is None) == (tb is None), name
        if ta is not None:
            assert torch.equal(ta, tb), name


@pytest.mark.parametrize("shape", [(128, 128), (256, 384), (128, 8192), (8192, 128), (384, 640),
                                   (4096, 4096), (8192, 11008), (2048, 22016)])
@pytest.mark.parametrize("mode", ["row", "col", "both"])
def test_fused_equals_two_pass(shape, mode, monkeypatch):
    torch.manual_seed(shape[0] * 7 + shape[1])
    x = torch.randn(shape, device="cuda", dtype=torch.bfloat16)
    x.view(-1)[:: 997] *= 80.0                    # outlier blocks -> micro codes < 127
    x[: shape[0] // 4, :64] *= 1e-3               # small blocks -> low E8M0 codes
    x.view(-1)[5::1009] = -0.0                    # signed zeros -> code 0x80 (fp8.py:148-149)
    a, b = _both(x, row=mode != "col", col=mode != "row", monkeypatch=monkeypatch)
    _assert_same(a, b)


def test_fused_barrier_generations(monkeypatch):
    """Back-to-back launches reuse the workspace: every one must see its own amax."""
    monkeypatch.setattr(Q, "FUSED", True)
    base = torch.randn(1024, 2048, device="cuda", dtype=torch.bfloat16)
    ops = []
    for i in range(41):
        x = base * (2.0 ** (i % 7)) * (1 + i / 64)
        am = torch.empty(1, device="cuda")
        ops.append((x, Q.quantize_mx2(x, row=True, col=(i % 2 == 0), amax_buf=am), am))
    torch.cuda.synchronize()
    for x, op, am in ops:
        want = float(x.float().abs().max())
        assert float(am) == want
        assert float(op.g) == float(np.float32(np.float32(want) / np.float32(448.0)))


def test_fused_producer_amax(monkeypatch):
    monkeypatch.setattr(Q, "FUSED", True)
    x = torch.randn(2048, 4096, device="cuda", dtype=torch.bfloat16)
    ref = Q.quantize_mx2(x, row=True, col=True, micro=True)
    am = x.float().abs().max().reshape(1)
    got = Q.quantize_mx2(x, row=True, col=True, micro=True, amax=am)
    for name in ("codes", "sf", "micro", "codes_t", "sf_t", "micro_t", "g"):
        assert torch.equal(getattr(ref, name), getattr(got, name)), name


def test_fused_all_zero_and_tiny(monkeypatch):
    monkeypatch.setattr(Q, "FUSED", True)
    z = torch.zeros(256, 256, device="cuda", dtype=torch.bfloat16)
    op = Q.quantize_mx2(z, row=True, col=True, micro=True)
    assert float(op.g) == 1.0                                       # test_quantize.py:158-162
    assert int(op.codes.max()) == 0 and bool((op.micro == 127).all())  # test_quantize.py:150-156
    a, b = _both(torch.full((256, 256), 2.0 ** -120, device="cuda", dtype=torch.bfloat16),
                 monkeypatch=monkeypatch)
    _assert_same(a, b)


def test_fused_errors(monkeypatch):
    monkeypatch.setattr(Q, "FUSED", True)
    for bad in (float("nan"), float("inf")):
        x = torch.ones(512, 512, device="cuda", dtype=torch.bfloat16)
        x[300, 7] = bad
        fl = _lib.FlagWord()
        Q.quantize_mx2(x, row=True, col=True, flags=fl)
        with pytest.raises(errors.InvalidValueError):
            fl.raise_if_set("fused")
    x = torch.ones(256, 256, device="cuda", dtype=torch.bfloat16)
    x[0, 0] = 2.0 ** 120
    x[128:, :32] = 2.0 ** -125            # block max far below g * 2^-127 -> E8M0 range error
    fl = _lib.FlagWord()
    Q.quantize_mx2(x, row=True, col=False, flags=fl)
    with pytest.raises(errors.E8m0RangeError):
        fl.raise_if_set("fused")


def test_fused_in_cuda_graph(monkeypatch):
    monkeypatch.setattr(Q, "FUSED", True)
    x = torch.randn(4096, 4096, device="cuda", dtype=torch.bfloat16)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        Q.quantize_mx2(x, row=True, col=True)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        op = Q.quantize_mx2(x, row=True, col=True)
    for i in range(5):
        x.copy_(torch.randn_like(x) * (i + 1))
        g.replay()
        monkeypatch.setattr(Q, "FUSED", False)
        ref = Q.quantize_mx2(x, row=True, col=True)
        monkeypatch.setattr(Q, "FUSED", True)
        for name in ("codes", "sf", "codes_t", "sf_t", "g"):
            assert torch.equal(getattr(op, name), getattr(ref, name)), (i, name)
    raise_if_flagged("cuda", "graph")


def test_producer_mode_dynamic_schedule(monkeypatch):
    """Producer mode on a big tensor (>= 8 tiles per CTA) takes the tail of its tiles
    from a global counter in the workspace, reset by the last CTA: outputs equal the
    static schedule (MOSS_Q4_DYN=0) bit for bit, across back-to-back launches and
    CUDA-graph replays (the counter must come back to 0 every launch)."""
    monkeypatch.setattr(Q, "FUSED", True)
    torch.manual_seed(3)
    x = torch.randn(8192, 11008, device="cuda", dtype=torch.bfloat16)
    x.view(-1)[::4093] *= 60.0
    am = x.float().abs().max().reshape(1)
    monkeypatch.setenv("MOSS_Q4_DYN", "0")
    ref = Q.quantize_mx2(x, row=True, col=True, micro=True, amax=am)
    monkeypatch.setenv("MOSS_Q4_DYN", "1")
    for _ in range(3):
        got = Q.quantize_mx2(x, row=True, col=True, micro=True, amax=am)
        for name in ("codes", "sf", "micro", "codes_t", "sf_t", "micro_t", "g"):
            assert torch.equal(getattr(ref, name), getattr(got, name)), name
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        Q.quantize_mx2(x, row=True, col=True, amax=am)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        op = Q.quantize_mx2(x, row=True, col=True, amax=am)
    for _ in range(4):
        g.replay()
        torch.cuda.synchronize()
        for name in ("codes", "sf", "codes_t", "sf_t", "g"):
            assert torch.equal(getattr(op, name), getattr(ref, name)), name
    raise_if_flagged("cuda", "dyn")


@pytest.mark.parametrize("shape", [(128, 128), (384, 640), (2048, 4096)])
def test_producer_mode_dynamic_schedule_forced(shape, monkeypatch):
    """MOSS_Q4_DYN=2 forces the counter-fed tail at any size (more CTAs than tiles,
    one tile per CTA, ragged last wave): same bytes as the static schedule."""
    monkeypatch.setattr(Q, "FUSED", True)
    torch.manual_seed(shape[1])
    x = torch.randn(shape, device="cuda", dtype=torch.bfloat16)
    am = x.float().abs().max().reshape(1)
    monkeypatch.setenv("MOSS_Q4_DYN", "0")
    ref = Q.quantize_mx2(x, row=True, col=True, micro=True, amax=am)
    monkeypatch.setenv("MOSS_Q4_DYN", "2")
    for _ in range(3):
        got = Q.quantize_mx2(x, row=True, col=True, micro=True, amax=am)
        for name in ("codes", "sf", "micro", "codes_t", "sf_t", "micro_t", "g"):
            assert torch.equal(getattr(ref, name), getattr(got, name)), name
