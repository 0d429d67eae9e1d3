"""B200-native batched Min-Sum LDPC decoding with the parity matrix H as a runtime argument.

Thin Python binding over the C-ABI of ``include/ldpc.h`` (libldpc.so, hand-written sm_100a
CUDA).  This module only marshals arguments: torch provides device memory and streams, every
step of the decode runs in the library's kernels.  There is no CPU or eager fallback: without
libldpc.so or without a CUDA device every call raises.

    h = Handle(H_uint8_cuda)                      # or Handle.from_coo(rows, cols, m, n)
    out = h.decode(llr_f32_cuda, max_iter=50, posterior=True, stats=stats_i64_cuda)
    out.bits, out.iters, out.converged, out.posterior
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib

FLAG_SIGN_PAPER_LITERAL = 1
FLAG_NO_EARLY_STOP = 2
FLAG_FORCE_STREAM = 4
FLAG_FORCE_RESIDENT = 8
FLAG_NO_GRAPH = 16

KERNEL_CLASSES = ("ingest", "stage_in", "check_node", "bit_node", "syndrome", "finalize", "resident", "compact")

STATS_FIELDS = ("frames", "bit_errors", "frame_errors", "undetected", "sum_iters", "converged", "near_zero",
                "raw_bit_errors")


class LdpcError(RuntimeError):
    def __init__(self, code: int, what: str):
        msg = _lib.load().ldpc_status_string(code).decode()
        super().__init__(f"{what}: {msg} ({code})")
        self.code = code


def _check(code: int, what: str):
    if code != 0:
        raise LdpcError(code, what)


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(stream) -> int | None:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


def _require_cuda(t: torch.Tensor, name: str, dtype: torch.dtype):
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def _check_out(t, name: str, shape: tuple, dtype: torch.dtype, device):
    """A caller-supplied output buffer: exact shape, dtype, contiguity and device (the C-ABI writes
    frames x n elements through the raw pointer, so a mismatch would be an out-of-bounds write)."""
    if t is None:
        return
    if tuple(t.shape) != shape:
        raise ValueError(f"out.{name} must have shape {shape}, got {tuple(t.shape)}")
    if t.dtype != dtype:
        raise ValueError(f"out.{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"out.{name} must be contiguous")
    if t.device != device:
        raise ValueError(f"out.{name} must be on {device}, got {t.device}")


def _check_result(out, F: int, n: int, device):
    _check_out(out.bits, "bits", (F, n), torch.uint8, device)
    _check_out(out.iters, "iters", (F,), torch.int32, device)
    _check_out(out.converged, "converged", (F,), torch.uint8, device)
    _check_out(out.posterior, "posterior", (F, n), torch.float32, device)


@dataclass
class DecodeResult:
    bits: torch.Tensor | None  # [F, n] uint8
    iters: torch.Tensor | None  # [F] int32
    converged: torch.Tensor | None  # [F] uint8
    posterior: torch.Tensor | None  # [F, n] float32


class Handle:
    """An ingested parity matrix plus its decode workspace (ldpc_prepare_* / ldpc_destroy)."""

    def __init__(self, H: torch.Tensor | None = None, *, flags: int = 0, stream=None, _raw=None):
        self._lib = _lib.load()
        self._h = ctypes.c_void_p()
        if _raw is not None:
            self._h = _raw
        else:
            if H is None:
                raise ValueError("H is required")
            _require_cuda(H, "H", torch.uint8)
            if H.dim() != 2:
                raise ValueError("H must be 2-D [m, n]")
            m, n = H.shape
            with torch.cuda.device(H.device):
                _check(self._lib.ldpc_prepare_dense(H.data_ptr(), m, n, flags, _stream(stream), ctypes.byref(self._h)),
                       "ldpc_prepare_dense")
        self.device = H.device if H is not None else torch.device("cuda", torch.cuda.current_device())
        m, n, nnz, dr, dc = (ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int32())
        _check(self._lib.ldpc_info(self._h, ctypes.byref(m), ctypes.byref(n), ctypes.byref(nnz), ctypes.byref(dr),
                                   ctypes.byref(dc)), "ldpc_info")
        self.m, self.n, self.nnz, self.max_row_deg, self.max_col_deg = m.value, n.value, nnz.value, dr.value, dc.value

    @classmethod
    def from_coo(cls, rows: torch.Tensor, cols: torch.Tensor, m: int, n: int, *, flags: int = 0, stream=None):
        lib = _lib.load()
        _require_cuda(rows, "rows", torch.int32)
        _require_cuda(cols, "cols", torch.int32)
        if rows.numel() != cols.numel():
            raise ValueError("rows and cols must have the same length")
        h = ctypes.c_void_p()
        with torch.cuda.device(rows.device):
            _check(lib.ldpc_prepare_coo(rows.data_ptr(), cols.data_ptr(), rows.numel(), m, n, flags, _stream(stream),
                                        ctypes.byref(h)), "ldpc_prepare_coo")
        obj = cls(_raw=h)
        obj.device = rows.device
        return obj

    # -------------------------------------------------------------------------------------------
    def decode(self, llr: torch.Tensor, max_iter: int, *, bits: bool = True, iters: bool = True,
               converged: bool = True, posterior: bool = False, stats: torch.Tensor | None = None,
               out: DecodeResult | None = None, stream=None) -> DecodeResult:
        """ldpc_decode on device tensors; outputs are allocated with torch.empty unless `out` is given.

        stats: optional int64 CUDA tensor of 8 counters, accumulated in place (see STATS_FIELDS)."""
        _require_cuda(llr, "llr", torch.float32)
        if llr.dim() != 2 or llr.shape[1] != self.n:
            raise ValueError(f"llr must be [frames, {self.n}]")
        F = llr.shape[0]
        dev = llr.device
        if dev != self.device:
            raise ValueError(f"llr is on {dev}, the handle on {self.device}")
        if out is not None:
            _check_result(out, F, self.n, dev)
        else:
            out = DecodeResult(
                torch.empty((F, self.n), dtype=torch.uint8, device=dev) if bits else None,
                torch.empty(F, dtype=torch.int32, device=dev) if iters else None,
                torch.empty(F, dtype=torch.uint8, device=dev) if converged else None,
                torch.empty((F, self.n), dtype=torch.float32, device=dev) if posterior else None)
        if stats is not None:
            _require_cuda(stats, "stats", torch.int64)
            if stats.numel() != 8:
                raise ValueError("stats must hold 8 int64 counters")
            if stats.device != dev:
                raise ValueError(f"stats must be on {dev}")
        with torch.cuda.device(dev):
            _check(self._lib.ldpc_decode(self._h, llr.data_ptr(), F, int(max_iter), _ptr(out.bits), _ptr(out.iters),
                                         _ptr(out.posterior), _ptr(out.converged), _ptr(stats), _stream(stream)),
                   "ldpc_decode")
        return out

    def decode_host(self, llr, max_iter: int, *, bits: bool = True, iters: bool = True, converged: bool = True,
                    posterior: bool = False, stats=None, out: DecodeResult | None = None, stream=None) -> DecodeResult:
        """ldpc_decode_host: llr and all outputs in HOST memory (pin them for copy/compute overlap)."""
        if llr.is_cuda or llr.dtype != torch.float32 or not llr.is_contiguous():
            raise ValueError("llr must be a contiguous float32 CPU tensor")
        if llr.dim() != 2 or llr.shape[1] != self.n:
            raise ValueError(f"llr must be [frames, {self.n}]")
        F = llr.shape[0]
        if out is not None:
            _check_result(out, F, self.n, torch.device("cpu"))
        else:
            pin = llr.is_pinned()
            out = DecodeResult(
                torch.empty((F, self.n), dtype=torch.uint8, pin_memory=pin) if bits else None,
                torch.empty(F, dtype=torch.int32, pin_memory=pin) if iters else None,
                torch.empty(F, dtype=torch.uint8, pin_memory=pin) if converged else None,
                torch.empty((F, self.n), dtype=torch.float32, pin_memory=pin) if posterior else None)
        if stats is not None and (stats.is_cuda or stats.dtype != torch.int64 or stats.numel() != 8
                                  or not stats.is_contiguous()):
            raise ValueError("stats must be a contiguous CPU int64 tensor of 8 counters")
        with torch.cuda.device(self.device):
            _check(self._lib.ldpc_decode_host(self._h, llr.data_ptr(), F, int(max_iter), _ptr(out.bits),
                                              _ptr(out.iters), _ptr(out.posterior), _ptr(out.converged), _ptr(stats),
                                              _stream(stream)), "ldpc_decode_host")
        return out

    # -------------------------------------------------------------------------------------------
    def graph(self):
        """Host copies of the ingested adjacency: (row_ptr, col_idx, col_ptr, col_edge) int32 tensors."""
        rp = torch.empty(self.m + 1, dtype=torch.int32)
        ci = torch.empty(self.nnz, dtype=torch.int32)
        cp = torch.empty(self.n + 1, dtype=torch.int32)
        ce = torch.empty(self.nnz, dtype=torch.int32)
        with torch.cuda.device(self.device):
            _check(self._lib.ldpc_get_graph(self._h, rp.data_ptr(), ci.data_ptr(), cp.data_ptr(), ce.data_ptr()),
                   "ldpc_get_graph")
        return rp, ci, cp, ce

    def set_flags(self, flags: int):
        _check(self._lib.ldpc_set_flags(self._h, flags), "ldpc_set_flags")

    def set_check_every(self, T: int):
        """Codeword test every T loop bodies (and after the last); T = 6 is the paper's setting."""
        _check(self._lib.ldpc_set_check_every(self._h, int(T)), "ldpc_set_check_every")

    def set_chunk(self, frames: int):
        _check(self._lib.ldpc_set_chunk(self._h, frames), "ldpc_set_chunk")

    @property
    def schedule(self) -> str:
        code = self._lib.ldpc_schedule(self._h)
        return {0: "stream", 1: "resident"}.get(code, "unavailable")

    def profile(self, enable: bool = True):
        _check(self._lib.ldpc_profile_enable(self._h, 1 if enable else 0), "ldpc_profile_enable")

    def profile_read(self) -> dict:
        n = len(KERNEL_CLASSES)
        launches = (ctypes.c_int64 * n)()
        ms = (ctypes.c_double * n)()
        with torch.cuda.device(self.device):
            _check(self._lib.ldpc_profile_read(self._h, launches, ms), "ldpc_profile_read")
        return {c: (int(launches[i]), float(ms[i])) for i, c in enumerate(KERNEL_CLASSES)}

    def profile_reset(self):
        with torch.cuda.device(self.device):
            _check(self._lib.ldpc_profile_reset(self._h), "ldpc_profile_reset")

    def stream_counters(self) -> dict:
        """Work counters of the streaming schedule: compaction activity (frames moved, compactions, tiles
        retired) and the tile-bodies each sweep processed (128 slots each)."""
        c = (ctypes.c_int64 * 5)()
        with torch.cuda.device(self.device):
            _check(self._lib.ldpc_stream_counters(self._h, c), "ldpc_stream_counters")
        return {"frames_moved": int(c[0]), "compactions": int(c[1]), "tiles_retired": int(c[2]),
                "cn_tile_bodies": int(c[3]), "bn_tile_bodies": int(c[4])}

    @property
    def launch_count(self) -> int:
        return int(self._lib.ldpc_launch_count(self._h))

    def close(self):
        if self._h:
            self._lib.ldpc_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def stats_dict(stats) -> dict:
    v = [int(x) for x in stats.tolist()]
    return dict(zip(STATS_FIELDS, v))
