"""BPSK over AWGN with a counter-based generator -- INPUT GENERATION ONLY.

Every noise sample is a pure function of (seed, Eb/N0 point, GLOBAL frame index,
bit index), so any shard, chunk or sample of a workload can be regenerated on any
device without generating the rest (multi-GPU sharding never changes a frame).
It holds none of the decoder's arithmetic.

Conventions (readings A15-A17):
  * BPSK: bit 1 -> +1, bit 0 -> -1, so the paper's all-zero codeword
     is sent as all -1 and "positive means 1" slices it back.
  * r is the raw channel output y = x + sigma*z (not 2y/sigma^2).
  * sigma^2 = 1 / (2 R 10^(EbN0/10)) with design rate R = 1 - m/n.

Generator: splitmix64 evaluated at counter c = frame*P + q (P = ceil(n/2) pairs
per frame), the two 32-bit halves give uniforms u1, u2 in (0,1), and a
Box-Muller transform in float64 gives the pair of normals for bits 2q, 2q+1.
Implemented with torch int64 ops (wrapping multiply) so that it runs unchanged on
CPU (tests, oracle inputs) or on the GPU (bench input staging).
"""
from __future__ import annotations

import math

import torch

_M64 = (1 << 64) - 1


def _s64(x: int) -> int:
    x &= _M64
    return x - (1 << 64) if x >= (1 << 63) else x


_GAMMA = _s64(0x9E3779B97F4A7C15)
_C1 = _s64(0xBF58476D1CE4E5B9)
_C2 = _s64(0x94D049BB133111EB)


def _srl(z: torch.Tensor, k: int) -> torch.Tensor:
    """Logical right shift of int64 bit patterns."""
    return (z >> k) & ((1 << (64 - k)) - 1)


def _mix(z: torch.Tensor) -> torch.Tensor:
    z = (z ^ _srl(z, 30)) * _C1
    z = (z ^ _srl(z, 27)) * _C2
    return z ^ _srl(z, 31)


def _mix_int(x: int) -> int:
    z = x & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def stream_key(seed: int, point: int) -> int:
    """64-bit key of one (workload seed, Eb/N0 point index) stream."""
    return _s64(_mix_int(_mix_int(seed + 0x1234567) ^ (point * 0x5851F42D4C957F2D + 0x14057B7EF767814F)))


def sigma_for(ebn0_db: float, rate: float) -> float:
    return math.sqrt(1.0 / (2.0 * rate * 10.0 ** (ebn0_db / 10.0)))


def normals(key: int, frame_lo: int, frames: int, n: int, device="cpu") -> torch.Tensor:
    """float64 N(0,1) samples [frames, n] for global frames [frame_lo, frame_lo+frames)."""
    P = (n + 1) // 2
    f = torch.arange(frame_lo, frame_lo + frames, dtype=torch.int64, device=device)
    q = torch.arange(P, dtype=torch.int64, device=device)
    c = f[:, None] * P + q[None, :]
    z = _mix(key + (c + 1) * _GAMMA)
    hi = _srl(z, 32).to(torch.float64)
    lo = (z & 0xFFFFFFFF).to(torch.float64)
    u1 = (hi + 0.5) * (1.0 / 4294967296.0)
    u2 = (lo + 0.5) * (1.0 / 4294967296.0)
    R = torch.sqrt(-2.0 * torch.log(u1))
    th = (2.0 * math.pi) * u2
    out = torch.stack([R * torch.cos(th), R * torch.sin(th)], dim=2).reshape(frames, 2 * P)
    return out[:, :n]


def bpsk_awgn(n: int, rate: float, ebn0_db: float, seed: int, point: int, frame_lo: int, frames: int,
              codeword=None, device="cpu", block: int = 1 << 15, out: torch.Tensor | None = None) -> torch.Tensor:
    """Channel output r (float32 [frames, n]) for global frames [frame_lo, frame_lo+frames).

    codeword: None for the all-zero codeword, or a 0/1 tensor [n] or [frames, n].
    """
    sig = sigma_for(ebn0_db, rate)
    key = stream_key(seed, point)
    if out is None:
        out = torch.empty((frames, n), dtype=torch.float32, device=device)
    cw = None
    if codeword is not None:
        cw = torch.as_tensor(codeword, device=device).to(torch.float64)
    for a in range(0, frames, block):
        b = min(frames, a + block)
        z = normals(key, frame_lo + a, b - a, n, device=device)
        if cw is None:
            x = -1.0
        else:
            c = cw if cw.dim() == 1 else cw[a:b]
            x = 2.0 * c - 1.0
        out[a:b] = (x + sig * z).to(torch.float32)
    return out


def workload_llr(code, cfg: dict, frame_lo: int, frames: int, device="cpu") -> tuple[torch.Tensor, list]:
    """LLRs for global frames [frame_lo, frame_lo+frames) of a config whose frames are
    split into contiguous Eb/N0 blocks (gen.codes.point_ranges).  Returns (llr, per-frame point index)."""
    from .codes import point_ranges

    pts = point_ranges(cfg["frames"], len(cfg["ebn0"]))
    out = torch.empty((frames, code.n), dtype=torch.float32, device=device)
    pidx = []
    for p, (lo, hi) in enumerate(pts):
        a, b = max(lo, frame_lo), min(hi, frame_lo + frames)
        if a >= b:
            continue
        bpsk_awgn(code.n, code.rate, cfg["ebn0"][p], cfg["seed"], p, a, b - a, device=device,
                  out=out[a - frame_lo:b - frame_lo])
        pidx += [p] * (b - a)
    return out, pidx
