"""The product's host-side compat functions against golden vectors made by
the reference itself (tests/golden/make_golden.py, make_golden_r2.py):
decode tables (fp8.py:87-128), e8m0_encode in both rounding modes
(fp8.py:194-223), and the lr schedule nn.cosine_lr == train.lr_at
(train.py:75-82).  No GPU needed."""

import os

import numpy as np
import pytest
import torch

import paper_2511_05811_b200 as P
from paper_2511_05811_b200.errors import E8m0RangeError, InvalidValueError
from paper_2511_05811_b200.fp8 import E8m0Rounding
from paper_2511_05811_b200.nn import cosine_lr

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def golden2():
    return np.load(os.path.join(HERE, "golden", "golden_r2.npz"))


@pytest.mark.parametrize("fmt,key", [(P.E4M3, "codec_decode_e4m3"), (P.E5M2, "codec_decode_e5m2")])
def test_decode_table_matches_reference(golden, fmt, key):
    got = P.decode_table(fmt, device="cpu").numpy().astype(np.float64)
    want = golden[key].astype(np.float64)
    assert got.shape == (256,)
    assert np.array_equal(np.isnan(got), np.isnan(want))
    ok = ~np.isnan(want)
    assert np.array_equal(got[ok], want[ok])
    assert np.array_equal(np.signbit(got[ok]), np.signbit(want[ok]))      # -0 at 0x80


@pytest.mark.parametrize("mode,key", [(E8m0Rounding.CEIL_POW2, "codec_e8m0_ceil"),
                                      (E8m0Rounding.NEAREST_LOG2, "codec_e8m0_near")])
def test_e8m0_encode_matches_reference(golden, mode, key):
    r = torch.from_numpy(golden["codec_e8m0_in"])
    got = P.e8m0_encode(r, mode).numpy()
    assert np.array_equal(got, golden[key])


def test_e8m0_encode_errors():
    with pytest.raises(E8m0RangeError):
        P.e8m0_encode(torch.tensor([2.0 ** -130], dtype=torch.float64))
    with pytest.raises(InvalidValueError):
        P.e8m0_encode(torch.tensor([0.0], dtype=torch.float64))


def test_cosine_lr_equals_reference_lr_at(golden, golden2):
    # the toy train() log of golden.npz: TrainConfig(steps=300) with the default peak/warmup/floor
    f = cosine_lr(0.01, 100, 300, 0.1)
    assert np.array_equal(np.array([f(t) for t in range(300)]), golden["train_q_lr"])
    for i in range(4):
        peak, warmup, steps, floor = golden2[f"lr_{i}_cfg"]
        f = cosine_lr(float(peak), int(warmup), int(steps), float(floor))
        want = golden2[f"lr_{i}_eta"]
        assert np.array_equal(np.array([f(t) for t in range(len(want))]), want)
