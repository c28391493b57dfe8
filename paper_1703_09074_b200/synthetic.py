"""Synthetic inputs for the BASELINE.json configs (input generation, not the
hot path). Factor models are drawn on the host with a vectorized counter form
of the reference's streams (random.hpp:16-107); the dense tensor and the
add_noise step (synthetic.hpp:42-58) are generated on the device by
rcpg_synth. numpy's log/sin/cos may differ from glibc in the last ulp, so
these tensors equal the oracle's generators only to rounding (the parity
tests feed both sides the same oracle-made tensor instead).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Tuple

import numpy as np

from .rcp import derive_seed, stream_id

GAMMA = np.uint64(0x9E3779B97F4A7C15)
FACTORS, NOISE, SYNTH_FACTORS, SYNTH_WEIGHTS = 3, 4, 7, 8


def _mix64(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def draws(seed: int, sid: int, start: int, count: int) -> np.ndarray:
    s0 = np.uint64(derive_seed(seed, sid))
    k = np.arange(start, start + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return _mix64(s0 + (k + np.uint64(1)) * GAMMA)


def normals(seed: int, sid: int, count: int) -> np.ndarray:
    """The first `count` RandomStream(seed, sid).normal() values."""
    npairs = (count + 1) // 2
    d = draws(seed, sid, 0, 2 * npairs)
    u1 = ((d[0::2] >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * 2.0 ** -53
    u2 = (d[1::2] >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    r = np.sqrt(-2.0 * np.log(u1))
    th = (2.0 * np.pi) * u2
    out = np.empty(2 * npairs)
    out[0::2] = r * np.cos(th)
    out[1::2] = r * np.sin(th)
    return out[:count]


def uniform01(seed: int, sid: int, count: int) -> np.ndarray:
    return (draws(seed, sid, 0, count) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def gaussian_matrix(seed: int, sid: int, rows: int, cols: int) -> np.ndarray:
    """fill_gaussian (random.hpp:90-94): column-major fill order."""
    return normals(seed, sid, rows * cols).reshape((rows, cols), order="F")


def model(kind: int, shape: List[int], rank: int, seed: int) -> Tuple[np.ndarray, List[np.ndarray]]:
    """Kruskal ground truth of config kind 1..5 (see oracle synth_model)."""
    if kind == 1:  # random_lowrank (synthetic.hpp:21-38)
        return np.ones(rank), [gaussian_matrix(seed, stream_id(FACTORS, m), e, rank) for m, e in enumerate(shape)]
    facs = []
    for m, I in enumerate(shape):
        sid = stream_id(SYNTH_FACTORS, m)
        if kind == 4 and m <= 1:
            c = uniform01(seed, sid, rank) * I
            i = np.arange(I)[:, None]
            f = np.exp(-0.5 * ((i - c[None, :]) / 8.0) ** 2)
        elif kind == 4 and m == 2:
            u = uniform01(seed, sid, 2 * rank)
            freq, phase = 1.0 + 19.0 * u[0::2], 2.0 * np.pi * u[1::2]
            i = np.arange(I)[:, None]
            f = np.sin(2.0 * np.pi * freq[None, :] * i / I + phase[None, :])
        else:
            f = gaussian_matrix(seed, sid, I, rank)
        if kind == 3:
            f = f / np.linalg.norm(f, axis=0)
        if kind == 5:
            q = np.linalg.qr(f)[0]  # LAPACK Householder convention, as the oracle
            C = 0.5 * (np.ones((rank, rank)) + np.eye(rank))
            f = q @ np.linalg.cholesky(C).T
        facs.append(np.asfortranarray(f))
    w = np.ones(rank)
    if kind == 2:
        w = 1.0 + 9.0 * uniform01(seed, stream_id(SYNTH_WEIGHTS), rank)
    if kind == 3:
        w = np.linspace(1.0, float(rank), rank)
    return w, facs


@dataclass
class Config:
    name: str
    kind: int
    shape: List[int]
    dtype: type
    rank: int
    oversampling: int
    power_iterations: int
    snr_db: float
    tol: float
    max_iter: int
    seed: int = 1
    shard_mode: int = -1  # slab mode of the multi-GPU runs (BASELINE.json; -1 = the last mode)

    @property
    def snr(self) -> float:  # amplitude ratio (synthetic.hpp:40-52)
        return 10.0 ** (self.snr_db / 20.0)

    def nbytes(self) -> int:
        return int(np.prod(self.shape)) * np.dtype(self.dtype).itemsize


# BASELINE.json configs (C3-C5: reference defaults tol 1e-5 / max_iter 500).
CONFIGS = {
    "C1": Config("C1", 1, [100, 100, 100], np.float64, 10, 10, 2, 20.0, 1e-8, 200, 1),
    "C2": Config("C2", 2, [400, 400, 400], np.float64, 20, 10, 2, 10.0, 1e-8, 200, 2),
    "C3": Config("C3", 3, [1024, 1024, 1024], np.float32, 50, 20, 2, 15.0, 1e-5, 500, 3),
    "C4": Config("C4", 4, [128, 128, 128, 512], np.float32, 32, 16, 2, 10.0, 1e-5, 500, 4),
    "C5": Config("C5", 5, [10000, 1000, 500], np.float32, 64, 16, 1, 20.0, 1e-5, 500, 5, 0),  # sharded along mode 1
}
