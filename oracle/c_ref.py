"""ctypes front-end to oracle/moss_oracle.c — TEST INFRASTRUCTURE ONLY."""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "libmoss_oracle.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(
            os.path.join(_HERE, "moss_oracle.c")):
        build()
    lib = ctypes.CDLL(_SO)
    P = ctypes.c_void_p
    I64 = ctypes.c_int64
    lib.moss_oracle_e4m3.restype = ctypes.c_uint8
    lib.moss_oracle_e4m3.argtypes = [ctypes.c_float]
    lib.moss_oracle_e4m3_array.restype = I64
    lib.moss_oracle_e4m3_array.argtypes = [P, P, I64]
    lib.moss_oracle_e4m3_sweep_compare.restype = I64
    lib.moss_oracle_e4m3_sweep_compare.argtypes = [ctypes.c_uint32, ctypes.c_uint64, P]
    lib.moss_oracle_quant_two_level.restype = ctypes.c_int
    lib.moss_oracle_quant_two_level.argtypes = [P, I64, I64, P, P, P]
    lib.moss_oracle_quant_two_level_rows.restype = ctypes.c_int
    lib.moss_oracle_quant_two_level_rows.argtypes = [P, I64, I64, ctypes.c_float, P, P]
    lib.moss_oracle_encode_scaled.restype = I64
    lib.moss_oracle_encode_scaled.argtypes = [P, I64, ctypes.c_float, P]
    _lib = _Wrap(lib)
    return _lib


class _Wrap:
    def __init__(self, lib):
        self.lib = lib

    def e4m3(self, x) -> np.ndarray:
        xf = np.ascontiguousarray(x, dtype=np.float32)
        out = np.empty(xf.shape, np.uint8)
        self.lib.moss_oracle_e4m3_array(xf.ctypes.data, out.ctypes.data, xf.size)
        return out

    def sweep_compare(self, lo: int, dev_codes: np.ndarray) -> int:
        d = np.ascontiguousarray(dev_codes, dtype=np.uint8)
        return int(self.lib.moss_oracle_e4m3_sweep_compare(lo, lo + d.size, d.ctypes.data))

    def quant_two_level(self, x):
        """Row-wise (blocks of 32 along the last axis) -> (codes, micro, g, status)."""
        xf = np.ascontiguousarray(x, dtype=np.float32)
        rows = int(np.prod(xf.shape[:-1])) if xf.ndim > 1 else 1
        cols = xf.shape[-1]
        codes = np.empty(xf.shape, np.uint8)
        micro = np.empty(xf.shape[:-1] + (cols // 32,), np.uint8)
        g = np.zeros(1, np.float32)
        st = self.lib.moss_oracle_quant_two_level(xf.ctypes.data, rows, cols, codes.ctypes.data,
                                                  micro.ctypes.data, g.ctypes.data)
        return codes, micro, float(g[0]), int(st)

    def quant_two_level_mt(self, x, threads: int | None = None):
        """quant_two_level with the per-block pass split over row ranges in
        threads (ctypes releases the GIL); the amax is numpy's max|x| (exact),
        g = f32(amax/448) as in the single-threaded function.  Same bits."""
        from concurrent.futures import ThreadPoolExecutor
        xf = np.ascontiguousarray(x, dtype=np.float32)
        rows = int(np.prod(xf.shape[:-1])) if xf.ndim > 1 else 1
        cols = xf.shape[-1]
        if not np.isfinite(xf).all():
            return None, None, 0.0, 1
        amax = np.float32(np.abs(xf).max()) if xf.size else np.float32(0)
        g = np.float32(amax / np.float32(448.0)) if amax > 0 else np.float32(1.0)
        codes = np.empty(xf.shape, np.uint8)
        micro = np.empty(xf.shape[:-1] + (cols // 32,), np.uint8)
        n = max(1, min(threads or os.cpu_count(), rows))
        cuts = [rows * i // n for i in range(n + 1)]
        nb = cols // 32

        def part(i):
            r0, r1 = cuts[i], cuts[i + 1]
            if r1 == r0:
                return 0
            return self.lib.moss_oracle_quant_two_level_rows(
                xf.ctypes.data + r0 * cols * 4, r1 - r0, cols, float(g),
                codes.ctypes.data + r0 * cols, micro.ctypes.data + r0 * nb)
        with ThreadPoolExecutor(n) as ex:
            st = max(ex.map(part, range(n)))
        return codes, micro, float(g), int(st)

    def encode_scaled(self, w, scale: float):
        wf = np.ascontiguousarray(w, dtype=np.float32)
        codes = np.empty(wf.shape, np.uint8)
        sat = self.lib.moss_oracle_encode_scaled(wf.ctypes.data, wf.size, float(np.float32(scale)),
                                                 codes.ctypes.data)
        return codes, int(sat)
