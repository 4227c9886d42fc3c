"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the Mustafar method (no pruning, no format, no
attention). It only draws fp16 bit patterns from a counter-based generator
(splitmix64, S:73 asks for a self-contained counter/xorshift-family generator) so
that the CPU oracle and the CUDA path see byte-identical inputs.

Two implementations of the same generator are provided:
  * numpy (host, uint64 arithmetic) -- used by the oracle tests and small cases;
  * torch (int64 arithmetic with explicit logical shifts) -- runs on the device for
    bench-sized inputs (GBs of KV) and is bit-identical to the numpy one
    (checked by tests/test_synth.py).

Value recipes:
  normal  : Irwin-Hall(4) approximation of N(0,1) in fp32, times `scale`, rounded to
            fp16 with round-to-nearest-even.
  lattice : integers in [-16,16] times 2^-2 (exact in fp16) -> heavy magnitude ties.
  zeros   : 50% exact +0 / -0 (0x0000 / 0x8000), rest `normal` -> signed-zero ties.
  outlier : `normal`, with the channels in `outlier_channels` multiplied by 10
            (the K channel outliers of P:62 / Fig. 1a).
"""
from __future__ import annotations

import math

import numpy as np

GOLDEN = 0x9E3779B97F4A7C15
M1 = 0xBF58476D1CE4E5B9
M2 = 0x94D049BB133111EB
MASK64 = (1 << 64) - 1
SQRT3_F32 = np.float32(math.sqrt(3.0))

KINDS = ("normal", "lattice", "zeros", "outlier")


def seed_for(config: int, stream: int) -> int:
    """Seed convention of SURVEY 8(d): 20250528 + 1000*config + stream."""
    return 20250528 + 1000 * int(config) + int(stream)


def _splitmix_scalar(x: int) -> int:
    z = (x + GOLDEN) & MASK64
    z = ((z ^ (z >> 30)) * M1) & MASK64
    z = ((z ^ (z >> 27)) * M2) & MASK64
    return z ^ (z >> 31)


def _key(seed: int) -> int:
    return _splitmix_scalar(int(seed) & MASK64)


# ----------------------------------------------------------------------------- numpy
def _mix_np(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(M1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(M2)
    return z ^ (z >> np.uint64(31))


def u64_np(n: int, seed: int, start: int = 0) -> np.ndarray:
    """Raw 64-bit draws for counters start..start+n-1."""
    key = np.uint64(_key(seed))
    ctr = np.arange(start + 1, start + n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = key + ctr * np.uint64(GOLDEN)
    return _mix_np(z)


def _values_from_u64_np(r: np.ndarray, kind: str, scale: float, chan: np.ndarray | None):
    c = [((r >> np.uint64(16 * j)) & np.uint64(0xFFFF)).astype(np.float32) for j in range(4)]
    if kind == "lattice":
        lat = ((r & np.uint64(0xFFFF)) % np.uint64(33)).astype(np.int32) - 16
        return (lat.astype(np.float32) * np.float32(0.25)).astype(np.float16)
    s = ((c[0] + np.float32(0.5)) / np.float32(65536.0) + (c[1] + np.float32(0.5)) / np.float32(65536.0)
         + (c[2] + np.float32(0.5)) / np.float32(65536.0) + (c[3] + np.float32(0.5)) / np.float32(65536.0))
    n = (s - np.float32(2.0)) * SQRT3_F32
    n = n * np.float32(scale)
    if kind == "outlier" and chan is not None:
        n = np.where(chan, n * np.float32(10.0), n).astype(np.float32)
    h = n.astype(np.float16)
    if kind == "zeros":
        sel = (r >> np.uint64(62)).astype(np.int64)  # top 2 bits
        bits = h.view(np.uint16).copy()
        bits = np.where(sel == 0, np.uint16(0x0000), bits)
        bits = np.where(sel == 1, np.uint16(0x8000), bits)
        return bits.astype(np.uint16).view(np.float16)
    return h


def fp16_np(shape, seed: int, kind: str = "normal", scale: float = 1.0,
            outlier_channels=(3, 17, 64, 101)) -> np.ndarray:
    """fp16 array (numpy.float16) of `shape`, row-major counters."""
    assert kind in KINDS, kind
    n = int(np.prod(shape)) if len(shape) else 1
    r = u64_np(n, seed)
    chan = None
    if kind == "outlier":
        d = shape[-1]
        ch = np.zeros(d, dtype=bool)
        ch[[c for c in outlier_channels if c < d]] = True
        chan = np.tile(ch, n // d)
    return _values_from_u64_np(r, kind, scale, chan).reshape(shape)


def fp16_np_rows(shape, seed: int, row0: int, nrows: int, kind: str = "normal", scale: float = 1.0,
                 outlier_channels=(3, 17, 64, 101)) -> np.ndarray:
    """Rows row0..row0+nrows-1 of fp16_np(shape, ...) viewed as [prod(shape[:-1]), d], without
    generating the rest (for sampling one unit of a bench-sized tensor on the host)."""
    d = shape[-1]
    r = u64_np(nrows * d, seed, start=row0 * d)
    chan = None
    if kind == "outlier":
        ch = np.zeros(d, dtype=bool)
        ch[[c for c in outlier_channels if c < d]] = True
        chan = np.tile(ch, nrows)
    return _values_from_u64_np(r, kind, scale, chan).reshape(nrows, d)


# ----------------------------------------------------------------------------- torch
def _lsr(x, n: int):
    import torch  # noqa: F401
    return (x >> n) & ((1 << (64 - n)) - 1)


def _as_i64(v: int) -> int:
    v &= MASK64
    return v - (1 << 64) if v >= (1 << 63) else v


def _mix_t(z):
    z = (z ^ _lsr(z, 30)) * _as_i64(M1)
    z = (z ^ _lsr(z, 27)) * _as_i64(M2)
    return z ^ _lsr(z, 31)


def fp16_torch(shape, seed: int, kind: str = "normal", scale: float = 1.0, device="cuda",
               outlier_channels=(3, 17, 64, 101), chunk: int = 1 << 24):
    """Same bits as fp16_np, generated with torch ops on `device` (plumbing only)."""
    import torch
    assert kind in KINDS, kind
    n = int(np.prod(shape)) if len(shape) else 1
    out = torch.empty(n, dtype=torch.float16, device=device)
    key = _as_i64(_key(seed))
    d = shape[-1]
    chan_vec = None
    if kind == "outlier":
        chan_vec = torch.zeros(d, dtype=torch.bool, device=device)
        chan_vec[[c for c in outlier_channels if c < d]] = True
    for s0 in range(0, n, chunk):
        m = min(chunk, n - s0)
        ctr = torch.arange(s0 + 1, s0 + m + 1, dtype=torch.int64, device=device)
        z = key + ctr * _as_i64(GOLDEN)
        r = _mix_t(z)
        if kind == "lattice":
            lat = torch.remainder(r & 0xFFFF, 33) - 16
            out[s0:s0 + m] = (lat.to(torch.float32) * 0.25).to(torch.float16)
            continue
        acc = None
        for j in range(4):
            cj = (_lsr(r, 16 * j) & 0xFFFF).to(torch.float32) if j else (r & 0xFFFF).to(torch.float32)
            term = (cj + 0.5) / 65536.0
            acc = term if acc is None else acc + term
        nv = (acc - 2.0) * float(SQRT3_F32)
        nv = nv * float(np.float32(scale))
        if chan_vec is not None:
            cidx = torch.remainder(torch.arange(s0, s0 + m, device=device), d)
            nv = torch.where(chan_vec[cidx], nv * 10.0, nv)
        h = nv.to(torch.float16)
        if kind == "zeros":
            sel = _lsr(r, 62)
            hb = h.view(torch.int16)
            hb = torch.where(sel == 0, torch.zeros_like(hb), hb)
            hb = torch.where(sel == 1, torch.full_like(hb, -32768), hb)
            h = hb.view(torch.float16)
        out[s0:s0 + m] = h
    return out.view(*shape)
