"""Fixture for the per-group (COAT) comparator, produced by the REFERENCE:
quant_per_group (quantize.py:100-124) and gemm_pergroup_mainloop
(gemm.py:132-157) on seeded inputs (with one all-zero group).  Run here,
where /root/reference exists:  python tests/golden/make_pergroup_golden.py"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from mossq.fp8 import E4M3  # noqa: E402
from mossq.gemm import gemm_pergroup_mainloop  # noqa: E402
from mossq.quantize import quant_per_group  # noqa: E402
from mossq.tensor import tensor_randn  # noqa: E402

a = tensor_randn([256, 512], seed=21, dist="outlier_injected")
b = tensor_randn([128, 512], seed=22)
a[3, :128] = 0.0
qa, qb = quant_per_group(a, E4M3, 128), quant_per_group(b, E4M3, 128)
c, ctr = gemm_pergroup_mainloop(qa, qb)
np.savez(os.path.join(os.path.dirname(os.path.abspath(__file__)), "pergroup_golden.npz"), a=a, b=b,
         a_codes=qa.codes, a_scales=qa.scales, b_codes=qb.codes, b_scales=qb.scales, c=c,
         counters=np.array([ctr.mainloop_dequant_multiplies, ctr.epilogue_dequant_multiplies,
                            ctr.block_scale_multiplies, ctr.mac_count]))
