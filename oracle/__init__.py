"""CPU oracle for batched Min-Sum LDPC decoding -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product package
``paper_2507_10424_b200`` never imports it, and it shares no code with the CUDA
path.  The arithmetic lives in ``oracle.c`` (plain C, Algorithm 1 of the paper
with the literal leave-one-out check-node update, see its header); this module
only marshals arguments and states the plain definitions of the statistics.

Parity pinning status:
  * decode (fp32 / fp64): pinned by tests/test_oracle_pins.py (P1-P13).
  * check_node: pinned by the SPEC/brute-force examples (P5).
  * syndrome: pinned by brute-force GF(2) products and the paper's 5x10 H (P1, P2).
  * stats: plain definitions over the decode outputs; pinned
    by hand-computed cases in tests/test_oracle_pins.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")

SIGN_PAPER_LITERAL = 1  # drop the (-1)^{d_i} factor of reading A1
NO_EARLY_STOP = 2  # no pre-check, no early exit: exactly L loop bodies

_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c twice (fp32, fp64) into liboracle.so with plain IEEE flags."""
    if not force and os.path.exists(_SO) and os.path.getmtime(_SO) >= os.path.getmtime(_SRC):
        return _SO
    common = ["gcc", "-O2", "-fPIC", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-c", _SRC]
    o32 = os.path.join(_HERE, "oracle_f32.o")
    o64 = os.path.join(_HERE, "oracle_f64.o")
    subprocess.check_call(common + ["-DREAL=float", "-DSFX=f32", "-o", o32])
    subprocess.check_call(common + ["-DREAL=double", "-DSFX=f64", "-o", o64])
    tmp = _SO + ".tmp"
    subprocess.check_call(["gcc", "-shared", "-fopenmp", "-o", tmp, o32, o64, "-lm"])
    os.replace(tmp, _SO)
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        for sfx in ("f32", "f64"):
            f = getattr(L, f"oracle_decode_{sfx}")
            f.restype = ctypes.c_int
            f.argtypes = [P, P, ctypes.c_int64, ctypes.c_int, ctypes.c_int, P, ctypes.c_int64, ctypes.c_int,
                          ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P, P, P]
            g = getattr(L, f"oracle_check_node_{sfx}")
            g.restype = None
            g.argtypes = [P, ctypes.c_int, ctypes.c_int, P]
            h = getattr(L, f"oracle_syndrome_{sfx}")
            h.restype = ctypes.c_int
            h.argtypes = [P, P, ctypes.c_int64, ctypes.c_int, ctypes.c_int, P, ctypes.c_int64, P]
        L.oracle_max_threads_f32.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _coo(H):
    """Accept a dense 0/1 matrix, or (rows, cols, m, n) lists of ones."""
    if isinstance(H, tuple):
        rows, cols, m, n = H
        return (np.ascontiguousarray(rows, dtype=np.int32), np.ascontiguousarray(cols, dtype=np.int32),
                int(m), int(n))
    Hd = np.asarray(H)
    if Hd.ndim != 2:
        raise ValueError("H must be 2-D or a (rows, cols, m, n) tuple")
    if not np.all((Hd == 0) | (Hd == 1)):
        raise ValueError("H must be binary")
    rows, cols = np.nonzero(Hd)
    return rows.astype(np.int32), cols.astype(np.int32), Hd.shape[0], Hd.shape[1]


_ERR = {-1: "index out of range", -2: "duplicate one in H", -3: "row of degree < 2", -4: "check_every must be >= 1"}


def decode(H, r, max_iter: int, flags: int = 0, threads: int = 0, precision: str = "f32", check_every: int = 1):
    """Decode frames r[F, n] (float32).  Returns (bits u8[F,n], iters i32[F], converged u8[F], posterior[F,n]).

    posterior is float32 for precision="f32" and float64 for the fp64 shadow.  check_every = T: the codeword
    test after body k runs when k % T == 0 or k == max_iter; the pre-loop test always runs.
    """
    rows, cols, m, n = _coo(H)
    r = np.ascontiguousarray(r, dtype=np.float32)
    if r.ndim == 1:
        r = r[None, :]
    if r.shape[1] != n:
        raise ValueError(f"r has {r.shape[1]} columns, H has n={n}")
    if not np.all(np.isfinite(r)):
        raise ValueError("llr values must be finite (S:132)")
    F = r.shape[0]
    bits = np.zeros((F, n), np.uint8)
    iters = np.zeros(F, np.int32)
    conv = np.zeros(F, np.uint8)
    post = np.zeros((F, n), np.float32 if precision == "f32" else np.float64)
    fn = getattr(lib(), f"oracle_decode_{precision}")
    rc = fn(_ptr(rows), _ptr(cols), len(rows), m, n, _ptr(r), F, int(max_iter), int(check_every), int(flags),
            int(threads), _ptr(bits), _ptr(iters), _ptr(conv), _ptr(post))
    if rc:
        raise ValueError(_ERR.get(rc, f"oracle error {rc}"))
    return bits, iters, conv, post


def check_node(x, flags: int = 0, precision: str = "f32"):
    """Eq. eta_update for one row: literal leave-one-out min and sign product."""
    dt = np.float32 if precision == "f32" else np.float64
    x = np.ascontiguousarray(x, dtype=dt)
    out = np.zeros_like(x)
    getattr(lib(), f"oracle_check_node_{precision}")(_ptr(x), len(x), int(flags), _ptr(out))
    return out


def syndrome_weight(H, b):
    """Number of unsatisfied checks of H.b over GF(2), per frame."""
    rows, cols, m, n = _coo(H)
    b = np.ascontiguousarray(b, dtype=np.uint8)
    if b.ndim == 1:
        b = b[None, :]
    out = np.zeros(b.shape[0], np.int32)
    rc = lib().oracle_syndrome_f32(_ptr(rows), _ptr(cols), len(rows), m, n, _ptr(b), b.shape[0], _ptr(out))
    if rc:
        raise ValueError(_ERR.get(rc, f"oracle error {rc}"))
    return out


def max_threads() -> int:
    return lib().oracle_max_threads_f32()


NEAR_ZERO = 1e-4  # |s_j| <= 1e-4 marks a frame as near-zero (north_star tolerance)


def stats(llr, bits, iters, conv, post):
    """Plain definitions of the 8 decode counters (the all-zero codeword is transmitted):

    [0] frames, [1] decoded bit errors = number of ones in b (numberOfNonZeros),
    [2] frame errors = frames with any bit error, [3] undetected errors = converged frames
    with a nonzero b, [4] sum of k, [5] converged frames, [6] near-zero frames
    (min_j |s_j| <= 1e-4), [7] raw bit errors = number of r_j > 0 (slice of the channel output).
    """
    bits = np.asarray(bits)
    be = bits.reshape(bits.shape[0], -1).sum(axis=1, dtype=np.int64)
    out = np.zeros(8, np.int64)
    out[0] = bits.shape[0]
    out[1] = be.sum()
    out[2] = np.count_nonzero(be)
    out[3] = np.count_nonzero((be > 0) & (np.asarray(conv) != 0))
    out[4] = np.asarray(iters, np.int64).sum()
    out[5] = np.count_nonzero(conv)
    out[6] = np.count_nonzero(np.abs(np.asarray(post)).min(axis=1) <= NEAR_ZERO) if bits.shape[1] else 0
    out[7] = np.count_nonzero(np.asarray(llr) > 0)
    return out
