"""Shared test helpers (CPU side)."""

import numpy as np


def sf_offsets(rows: int, n_blocks: int) -> np.ndarray:
    """[rows, n_blocks] byte offsets of the tcgen05 block-scale layout
    (128-row x 4-block chunks of 512 B; in-chunk (r%32)*16 + ((r%128)/32)*4 + kb%4)."""
    r = np.arange(rows)[:, None]
    kb = np.arange(n_blocks)[None, :]
    kchunks = (n_blocks + 3) // 4
    return (((r // 128) * kchunks + kb // 4) * 512 + (r % 32) * 16 + ((r % 128) // 32) * 4 + kb % 4)


def unswizzle_sf(buf: np.ndarray, rows: int, n_blocks: int) -> np.ndarray:
    return np.asarray(buf)[sf_offsets(rows, n_blocks)]


def rel_frob(a, b) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
