"""GPU parity of the sm_100a kernels against the CPU oracle (oracle/).

Bar (BASELINE.json north_star): quantized codes, E8M0 exponents and FP8
weight codes bit-exact; GEMM within an FP32-accumulation tolerance of the
float64 oracle evaluated on the GPU's own codes; AdamW within a stated
FP32-vs-float64 tolerance.  All calls go through the C ABI (_lib).
"""

import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2511_05811_b200 as P  # noqa: E402
from paper_2511_05811_b200 import _lib, errors  # noqa: E402
from paper_2511_05811_b200.gemm import GemmOperands, gemm_mx_epilogue, mx_gemm  # noqa: E402
from paper_2511_05811_b200.optim import adamw_step, init_state  # noqa: E402
from paper_2511_05811_b200.quantize import PerTensorQuant, quantize_mx2  # noqa: E402

from oracle import numpy_ref as R  # noqa: E402

from .helpers import rel_frob, unswizzle_sf  # noqa: E402

GEMM_TOL = 1e-5   # rel. Frobenius, FP32 accumulation vs float64 oracle on identical codes


def cuda(a, dtype=torch.float32):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device="cuda")


def host(t):
    return t.detach().cpu().numpy()


# ----------------------------------------------------------------- codec
def test_encode_golden(golden):
    x = golden["codec_encode_in"]
    got = host(P.fp8_encode(cuda(x)))
    assert np.array_equal(got, golden["codec_encode_e4m3"])


def test_encode_rejects_nonfinite():
    for bad in (float("nan"), float("inf"), -float("inf")):
        with pytest.raises(errors.InvalidValueError):
            P.fp8_encode(cuda(np.array([1.0, bad], np.float32)))


@pytest.mark.slow
def test_exhaustive_e4m3_cvt_sweep(c_oracle):
    """All 2^32 f32 bit patterns: device encoder == C restatement of fp8.py:131-183
    (non-finite patterns excluded: the reference rejects them before encoding)."""
    chunk = 1 << 28
    u = torch.arange(chunk, dtype=torch.int64, device="cuda")
    bad = [0]
    lock = threading.Lock()
    threads = []

    def cmp(lo, codes):
        n = c_oracle.sweep_compare(lo, codes)
        with lock:
            bad[0] += n

    for lo in range(0, 1 << 32, chunk):
        bits = (u + lo).to(torch.int32)  # wraps to the same 32-bit pattern
        x = bits.view(torch.float32)
        finite = torch.isfinite(x)
        x = torch.where(finite, x, torch.zeros_like(x))
        codes = torch.empty(chunk, dtype=torch.uint8, device="cuda")
        fl = _lib.FlagWord()
        _lib.encode_scaled(x.view(1, -1), fl, scale_host=1.0, codes=codes)
        h = host(codes)
        th = threading.Thread(target=cmp, args=(lo, h))
        th.start()
        threads.append(th)
        if len(threads) >= 8:
            threads.pop(0).join()
    for th in threads:
        th.join()
    assert bad[0] == 0


# ----------------------------------------------------------------- two-level quantizer
@pytest.mark.parametrize("dtype", ["f32"])
def test_two_level_golden_cases(golden, dtype):
    for name in list(golden["q2l_cases"]):
        x = golden[f"q2l_{name}_x"]
        q = P.quant_two_level(cuda(x))
        assert np.array_equal(host(q.codes), golden[f"q2l_{name}_codes"]), name
        assert np.array_equal(host(q.micro_codes), golden[f"q2l_{name}_micro"]), name
        assert np.float32(float(q.global_scale)) == golden[f"q2l_{name}_g"], name
        rows = int(np.prod(x.shape[:-1]))
        nb = x.shape[-1] // 32
        assert np.array_equal(unswizzle_sf(host(q.sf), rows, nb), golden[f"q2l_{name}_micro"].reshape(rows, nb))


def test_two_level_midpoint_vectors(golden):
    """FP8-midpoint recipe: catches reciprocal-multiply instead of IEEE division."""
    x = golden["q2l_midrows_x"]
    for i in range(x.shape[0]):
        q = P.quant_two_level(cuda(x[i:i + 1]))
        assert np.array_equal(host(q.codes), golden["q2l_midrows_codes"][i:i + 1]), i
        assert np.array_equal(host(q.micro_codes), golden["q2l_midrows_micro"][i:i + 1]), i
        assert np.float32(float(q.global_scale)) == golden["q2l_midrows_g"][i]


def test_two_level_errors(golden):
    with pytest.raises(errors.E8m0RangeError):
        P.quant_two_level(cuda(golden["q2l_rangeerr_x"]))
    x = np.ones((2, 64), np.float32)
    x[1, 3] = np.nan
    with pytest.raises(errors.InvalidValueError):
        P.quant_two_level(cuda(x))
    with pytest.raises(errors.InvalidShapeError):
        P.quant_two_level(cuda(np.ones(33, np.float32)))
    with pytest.raises(errors.InvalidShapeError):
        P.quant_two_level(torch.tensor(1.0, device="cuda"))


@pytest.mark.parametrize("shape,dist,dtype", [
    ((4096, 4096), "gaussian", torch.bfloat16),       # config 1 activation
    ((8192, 4096), "outlier", torch.bfloat16),        # config 2 QKV/O/gate/up input
    ((2048, 11008), "outlier", torch.bfloat16),       # down-proj input (rows reduced for CPU oracle time)
    ((1024, 4096), "outlier", torch.float32),
    ((96, 160), "gaussian", torch.float32),           # ragged: rows % 128, blocks % 4
])
def test_two_level_row_and_col_bit_exact_at_scale(c_oracle, shape, dist, dtype):
    rng = np.random.default_rng(sum(shape))
    x = rng.standard_normal(shape).astype(np.float32)
    if dist == "outlier":
        idx = rng.choice(x.size, max(1, x.size // 1000), replace=False)
        x.reshape(-1)[idx] = (50.0 * (1 + 0.1 * np.abs(rng.standard_normal(idx.size)))
                              * rng.choice([-1, 1], idx.size)).astype(np.float32)
    xt = cuda(x, dtype)
    x_exact = host(xt.float())                     # bf16 inputs: the oracle sees the exact upcast
    op = quantize_mx2(xt, row=True, col=True, micro=True)
    codes, micro, g, st = c_oracle.quant_two_level(x_exact)
    assert st == 0
    assert float(op.g.item()) == g
    assert np.array_equal(host(op.codes), codes)
    assert np.array_equal(host(op.micro), micro)
    rows, cols = shape
    assert np.array_equal(unswizzle_sf(host(op.sf), rows, cols // 32), micro)
    if rows % 32 == 0:
        # column-wise == quant_two_level(x.T) with the same global scale
        codes_t, micro_t, g_t, st_t = c_oracle.quant_two_level(np.ascontiguousarray(x_exact.T))
        assert g_t == g
        assert np.array_equal(host(op.codes_t), codes_t)
        assert np.array_equal(host(op.micro_t), micro_t)
        assert np.array_equal(unswizzle_sf(host(op.sf_t), cols, rows // 32), micro_t)


def _bf16_sweep_tensor(amax_bits: int, rng) -> np.ndarray:
    """[rows, 256] f32 (exact bf16 values): block 0 holds the tensor max A;
    every block k holds a block max A*2^-j (varied exponent) and up to 31
    bf16 patterns not exceeding it — all 65536 patterns appear at least once."""
    A = np.uint32(amax_bits << 16).view(np.float32)
    pats = (np.arange(1 << 16, dtype=np.uint32) << 16).view(np.float32)
    pats = pats[np.isfinite(pats)]
    blocks = []
    for j in range(0, 40, 3):
        bm = np.float32(A * np.float32(2.0 ** -j))
        bm = (np.float32(bm).view(np.uint32) & 0xFFFF0000).view(np.float32)   # keep it a bf16 value
        if not np.isfinite(bm) or bm == 0:
            continue
        ok = pats[np.abs(pats) <= bm]
        if ok.size == 0:
            continue
        n_blk = -(-ok.size // 31)
        body = np.zeros(n_blk * 31, np.float32)
        body[:ok.size] = ok
        blk = np.concatenate([np.full((n_blk, 1), bm, np.float32), body.reshape(n_blk, 31)], axis=1)
        blocks.append(blk.reshape(-1))
    flat = np.concatenate(blocks)
    flat[0] = A
    pad = (-flat.size) % (128 * 256)          # rows % 128 == 0: exercises the TMA fast path
    flat = np.concatenate([flat, np.zeros(pad, np.float32)])
    return flat.reshape(-1, 256)


@pytest.mark.slow
def test_bf16_fast_division_exhaustive(c_oracle):
    """The bf16 TMA quantizer divides with a per-block reciprocal + FMA
    correction (common.cuh block_div); prove it equals IEEE division on every
    bf16 input pattern for many global scales (random significands, the
    all-ones significand, extreme exponents), row- and column-wise."""
    rng = np.random.default_rng(11)
    amaxes = [0x7F7F, 0x3FFF, 0x3F80, 0x0080, 0x0100, 0x43E0, 0x7F00, 0x1F7F]
    amaxes += [int(v) for v in rng.integers(0x0080, 0x7F7F, 40)]
    for ab in amaxes:
        x = _bf16_sweep_tensor(ab, rng)
        xt = cuda(x, torch.bfloat16)
        assert np.array_equal(host(xt.float()), x)
        op = quantize_mx2(xt, row=True, col=True, micro=True)
        codes, micro, g, st = c_oracle.quant_two_level(x)
        assert float(op.g.item()) == g, hex(ab)
        assert np.array_equal(host(op.micro), micro), hex(ab)
        assert np.array_equal(host(op.codes), codes), hex(ab)
        codes_t, micro_t, _, _ = c_oracle.quant_two_level(np.ascontiguousarray(x.T))
        assert np.array_equal(host(op.codes_t), codes_t), hex(ab)
        assert np.array_equal(host(op.micro_t), micro_t), hex(ab)


def test_two_level_properties_full_size():
    """Size-independent properties at the 8192 x 11008 down-proj shape."""
    torch.manual_seed(0)
    x = torch.randn(8192, 11008, device="cuda", dtype=torch.bfloat16)
    x[::97, ::89] *= 60
    op = quantize_mx2(x, row=True, col=True, micro=True)
    g = float(op.g.item())
    assert g == float(np.float32(np.float32(float(x.abs().max())) / np.float32(448.0)))
    dq = P.fp8_decode(op.codes).view(8192, -1, 32) * (g * torch.ldexp(torch.ones(1, device="cuda"),
                                                                      op.micro.int() - 127))[..., None]
    err = (dq.view(8192, 11008) - x.float()).abs().view(8192, -1, 32).amax(-1)
    bmax = x.float().abs().view(8192, -1, 32).amax(-1)
    assert bool((err <= bmax * 2.0 ** -3 * (1 + 1e-6)).all())      # test_quantize.py:164-174
    assert int(op.micro.max()) <= 127                                # micro in (0, 1]
    # 2^k scaling invariance (test_gemm.py:75-88): codes/micro unchanged, g scales
    op2 = quantize_mx2(x * 8, row=True, col=False, micro=True)
    assert torch.equal(op2.codes, op.codes) and torch.equal(op2.micro, op.micro)
    assert float(op2.g.item()) == 8 * g


# ----------------------------------------------------------------- per-tensor / weight copy
def test_per_tensor_golden(golden):
    for name in ("exact", "two", "gauss", "w"):
        q = P.quant_per_tensor(cuda(golden[f"qpt_{name}_x"]))
        assert np.array_equal(host(q.codes), golden[f"qpt_{name}_codes"]), name
        assert float(q.scale) == float(golden[f"qpt_{name}_scale"]), name


def test_weight_encode_with_transpose(c_oracle):
    rng = np.random.default_rng(3)
    w = (rng.standard_normal((512, 1024)) * 0.02).astype(np.float32)
    wt = cuda(w)
    q = P.quant_per_tensor(wt, transpose=True)
    codes, scale = R.quant_per_tensor(w)
    assert float(q.scale) == scale
    assert np.array_equal(host(q.codes), codes)
    assert np.array_equal(host(q.codes_t), codes.T)


# ----------------------------------------------------------------- GEMM
@pytest.mark.parametrize("shape", ["64x64x64", "16x48x96", "128x128x256", "256x128x512"])
def test_gemm_mx_epilogue_golden(golden, shape):
    t = f"gemm_{shape}"
    from paper_2511_05811_b200.gemm import quantize_gemm_operands
    ops = quantize_gemm_operands(cuda(golden[t + "_w"]), cuda(golden[t + "_x"]))
    assert np.array_equal(host(ops.qw.codes), golden[t + "_wcodes"])
    assert np.array_equal(host(ops.qx.codes), golden[t + "_xcodes"])
    out, ctr = gemm_mx_epilogue(ops)
    m, n, k = map(int, shape.split("x"))
    assert tuple(out.shape) == (m, n)
    assert ctr.epilogue_dequant_multiplies == m * n and ctr.mainloop_dequant_multiplies == 0
    assert rel_frob(host(out), golden[t + "_out"]) <= GEMM_TOL


def test_gemm_identity_pattern():
    """test_gemm.py:43-52: identity weights reproduce the dequantized activations."""
    k = 128
    codes = P.fp8_encode(torch.eye(k, device="cuda"))
    qw = PerTensorQuant(codes=codes, scale=torch.tensor(1.0, device="cuda"), fmt=P.E4M3)
    x = torch.randn(256, k, device="cuda")
    qx = P.quant_two_level(x)
    out, _ = gemm_mx_epilogue(GemmOperands(qw=qw, qx=qx))
    assert torch.equal(out.t().contiguous(), P.dequantize(qx))


@pytest.mark.parametrize("mnk,out_dtype", [
    ((512, 768, 1024), torch.float32),
    ((1024, 4096, 4096), torch.bfloat16),     # BN=256 path
    ((256, 384, 11008), torch.float32),       # BN=128 path, long K
    ((8192, 12288, 4096), torch.bfloat16),    # config-2 QKV shape, checked on sampled rows
])
def test_gemm_vs_f64_oracle_on_device_codes(mnk, out_dtype):
    m, n, k = mnk
    torch.manual_seed(m + n + k)
    a = torch.randn(m, k, device="cuda")
    a.view(-1)[torch.randint(0, m * k, (m * k // 1000,), device="cuda")] *= 50
    b = torch.randn(n, k, device="cuda") * 0.02
    qa = quantize_mx2(a, row=True, micro=True)
    qb = P.quant_per_tensor(b)
    d = mx_gemm(qa.codes, qa.sf, qa.g, qb.codes, None, qb.scale.reshape(1), out_dtype=out_dtype)
    rows = np.arange(m) if m <= 1024 else np.random.default_rng(0).choice(m, 256, replace=False)
    a_deq = R.dequantize_two_level(R.TwoLevel(host(qa.codes)[rows], float(qa.g.item()), host(qa.micro)[rows]))
    b_deq = R.dequantize_per_tensor(host(qb.codes), float(qb.scale))
    ref = R.gemm_f64(a_deq, b_deq)
    got = host(d.float())[rows]
    tol = GEMM_TOL if out_dtype == torch.float32 else 4e-3   # bf16 output rounding (2^-9 rel)
    assert rel_frob(got, ref) <= tol
    # elementwise, normalised by the accumulation magnitude
    mag = np.abs(a_deq) @ np.abs(b_deq).T
    assert float(np.max(np.abs(got - ref) / (mag + 1e-30))) <= (1e-5 if out_dtype == torch.float32 else 4e-3)


@pytest.mark.parametrize("m,n,k", [(384, 512, 2048), (512, 768, 1024), (1024, 512, 4096)])
def test_gemm_unit_and_real_scales_both_sides(m, n, k):
    """Two-level operands on BOTH sides (wgrad-style) and accumulate=True
    (1-CTA kernel for M % 256 != 0, CTA-pair kernel otherwise)."""
    torch.manual_seed(1)
    a = torch.randn(m, k, device="cuda") * torch.logspace(-3, 1, k, device="cuda")
    b = torch.randn(n, k, device="cuda")
    qa = quantize_mx2(a, micro=True)
    qb = quantize_mx2(b, micro=True)
    acc = torch.randn(m, n, device="cuda")
    d = mx_gemm(qa.codes, qa.sf, qa.g, qb.codes, qb.sf, qb.g, out=acc.clone(), accumulate=True)
    ref = R.gemm_f64(R.dequantize_two_level(R.TwoLevel(host(qa.codes), float(qa.g.item()), host(qa.micro))),
                     R.dequantize_two_level(R.TwoLevel(host(qb.codes), float(qb.g.item()), host(qb.micro))))
    assert rel_frob(host(d) - host(acc), ref) <= GEMM_TOL


def test_gemm_pair_kernel_matches_single_cta_kernel():
    """The cta_group::2 kernel and the 1-CTA kernel (MOSS_GEMM_VARIANT=1 in a
    subprocess) agree to FP32-accumulation noise on the same operands."""
    import subprocess
    import sys
    code = r'''
import sys, torch, numpy as np
sys.path.insert(0, ".")
from paper_2511_05811_b200.quantize import quantize_mx2, quant_per_tensor
from paper_2511_05811_b200.gemm import mx_gemm
torch.manual_seed(5)
a = torch.randn(1024, 2048, device="cuda"); b = torch.randn(768, 2048, device="cuda")
qa = quantize_mx2(a); qb = quant_per_tensor(b)
for dt in (torch.float32, torch.bfloat16):
    d = mx_gemm(qa.codes, qa.sf, qa.g, qb.codes, None, qb.scale.reshape(1), out_dtype=dt)
    np.save(sys.argv[1] + ("_f32.npy" if dt == torch.float32 else "_bf16.npy"), d.float().cpu().numpy())
'''
    import os
    import tempfile
    outs = {}
    for v in ("1", "2"):
        p = os.path.join(tempfile.mkdtemp(), "g")
        env = dict(os.environ, MOSS_GEMM_VARIANT=v)
        subprocess.run([sys.executable, "-c", code, p], check=True, env=env, cwd=os.path.dirname(os.path.dirname(__file__)))
        outs[v] = (np.load(p + "_f32.npy"), np.load(p + "_bf16.npy"))
    assert rel_frob(outs["2"][0], outs["1"][0]) <= 1e-6
    assert rel_frob(outs["2"][1], outs["1"][1]) <= 4e-3


# ----------------------------------------------------------------- AdamW
@pytest.mark.parametrize("tag", ["dec", "cpl", "nowd"])
def test_adamw_trajectory_vs_reference(golden, tag):
    eta, wd, dec = golden[f"adam_{tag}_hp"]
    w = cuda(golden[f"adam_{tag}_w0"])
    st = init_state(w.shape, eta=float(eta), weight_decay=float(wd), decoupled_decay=bool(dec))
    for i, g in enumerate(golden[f"adam_{tag}_g"]):
        w, st, d = adamw_step(w, cuda(g), st)
        want = golden[f"adam_{tag}_w"][i]
        # FP32 state vs the float64 reference: |dW| <= 1e-3 * eta * (i+1)
        assert np.max(np.abs(host(w) - want)) <= 1e-3 * float(eta) * (i + 1) + 1e-7
        mref = golden[f"adam_{tag}_m"][i]
        vref = golden[f"adam_{tag}_v"][i]
        assert np.max(np.abs(host(st.m) - mref)) <= 1e-6 * np.max(np.abs(mref)) + 1e-30
        assert np.max(np.abs(host(st.v) - vref)) <= 1e-6 * np.max(np.abs(vref)) + 1e-30


def test_adamw_rejects_nonfinite_before_mutation():
    st = init_state((64,))
    w = torch.zeros(64, device="cuda")
    g = torch.ones(64, device="cuda")
    g[5] = float("nan")
    with pytest.raises(errors.InvalidValueError):
        adamw_step(w, g, st)
    assert st.t == 0 and float(st.m.abs().max()) == 0.0


def test_fused_adamw_fp8_copy_bit_exact(c_oracle):
    """K3: the FP8 weight copy equals e4m3(f32(W')/f32(s)) of the kernel's own W'."""
    rows, cols = 256, 1024
    torch.manual_seed(2)
    w = torch.randn(rows, cols, device="cuda") * 0.02
    g = torch.randn(rows, cols, device="cuda") * 1e-3
    m = torch.zeros_like(w)
    v = torch.zeros_like(w)
    s_next = 0.05 / 448 + 3e-4 / 448
    w_fp8 = torch.empty(rows, cols, dtype=torch.uint8, device="cuda")
    w_fp8_t = torch.empty(cols, rows, dtype=torch.uint8, device="cuda")
    w_amax = torch.empty(1, device="cuda")
    nsat = torch.zeros(1, dtype=torch.int32, device="cuda")
    flags = _lib.FlagWord()
    from paper_2511_05811_b200.optim import adam_params
    p = adam_params(3e-4, 0.9, 0.95, 1e-8, 0.1, 1, True)
    w_old = host(w).copy()
    _lib.adamw_fp8(w, g, m, v, rows, cols, p, float(np.float32(s_next)), flags, w_fp8=w_fp8, w_fp8_t=w_fp8_t,
                   w_amax=w_amax, n_saturated=nsat)
    flags.raise_if_set()
    wn = host(w)
    codes, sat = c_oracle.encode_scaled(wn, s_next)
    assert np.array_equal(host(w_fp8), codes)
    assert np.array_equal(host(w_fp8_t), codes.T)
    assert int(nsat.item()) == sat
    assert float(w_amax.item()) == float(np.abs(wn).max())
    st = R.adam_init((rows, cols), eta=3e-4, weight_decay=0.1)
    ref, _ = R.adamw_step(w_old, host(g), st)
    assert np.max(np.abs(wn - ref)) <= 1e-3 * 3e-4
