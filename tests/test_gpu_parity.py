"""GPU parity: the CUDA path through the C-ABI versus the CPU oracle on the same seeded inputs.

Bar (north_star): decoded bits, per-frame iteration counts and isCodeword bit-exact; posterior
within 1e-4 absolute/relative (the design is bit-exact, asserted separately); frames whose
posterior has an entry within 1e-4 of zero are counted.
"""
import sys

import numpy as np
import pytest
import torch

import oracle
from gen import channel, codes

pytestmark = pytest.mark.gpu

LIT = 1
NOES = 2
FORCE_STREAM = 4
FORCE_RESIDENT = 8
TOL = 1e-4


def ldpc():
    import paper_2507_10424_b200 as P

    return P


def handle(code, flags=0, coo=False):
    P = ldpc()
    if coo:
        rr, cc = code.coo()
        return P.Handle.from_coo(torch.from_numpy(rr).cuda(), torch.from_numpy(cc).cuda(), code.m, code.n, flags=flags)
    return P.Handle(torch.from_numpy(code.dense()).cuda(), flags=flags)


def gpu_decode(h, llr_np, L, posterior=True):
    llr = torch.from_numpy(np.ascontiguousarray(llr_np)).cuda()
    stats = torch.zeros(8, dtype=torch.int64, device="cuda")
    out = h.decode(llr, L, posterior=posterior, stats=stats)
    torch.cuda.synchronize()
    return (out.bits.cpu().numpy(), out.iters.cpu().numpy(), out.converged.cpu().numpy(),
            out.posterior.cpu().numpy() if posterior else None, stats.cpu().numpy())


def compare(code, llr, L, flags=0, h=None, exact=True, check_every=1):
    if h is None:
        h = handle(code, flags)
    if check_every != 1:
        h.set_check_every(check_every)
    gb, gi, gc, gp, gs = gpu_decode(h, llr, L)
    ob, oi, oc, op = oracle.decode(code.oracle_h(), llr, L, flags=flags & (LIT | NOES), check_every=check_every)
    assert np.array_equal(gi, oi), f"iters differ on {np.count_nonzero(gi != oi)} frames"
    assert np.array_equal(gc, oc), "converged differs"
    assert np.array_equal(gb, ob), f"bits differ on {np.count_nonzero(np.any(gb != ob, axis=1))} frames"
    assert np.allclose(gp, op, rtol=TOL, atol=TOL)
    if exact:  # bit-exact up to the sign of a zero (the decoders keep zeros of s canonical, reading A12)
        z = np.float32(0.0)
        assert np.array_equal((gp + z).view(np.uint32), (op + z).view(np.uint32)), "posterior not bit-exact"
    assert np.array_equal(gs, oracle.stats(llr, ob, oi, oc, op))
    return gb, gi, gc, gp


def frames_for(code, F, ebn0, seed, point=0):
    return channel.bpsk_awgn(code.n, code.rate, ebn0, seed, point, 0, F).numpy()


# ---------------------------------------------------------------- ingestion (a1) ------------
@pytest.mark.parametrize("coo", [False, True])
@pytest.mark.parametrize("which", ["paper", "small", "reg", "bg1"])
def test_ingest_graph_matches_definition(which, coo):
    code = {"paper": codes.paper_5x10, "small": lambda: codes.random_small(40, 90, 3, 2, 9),
            "reg": lambda: codes.regular(504, 1008, 3, 6, 1008), "bg1": codes.bg1_dims}[which]()
    h = handle(code, coo=coo)
    rp, ci, cp, ce = [t.numpy() for t in h.graph()]
    assert (h.m, h.n, h.nnz) == (code.m, code.n, code.nnz)
    exp_rp = np.concatenate([[0], np.cumsum([len(r) for r in code.rows])])
    assert np.array_equal(rp, exp_rp)
    assert np.array_equal(ci, np.concatenate(code.rows))  # N_i ascending
    # M_j: for every column, the row-list positions of its ones in ascending row order
    rr, cc = code.coo()
    order = np.lexsort((rr, cc))
    assert np.array_equal(cp, np.concatenate([[0], np.cumsum(np.bincount(cc, minlength=code.n))]))
    assert np.array_equal(ce, np.arange(code.nnz)[order])
    assert h.max_row_deg == max(len(r) for r in code.rows)


def test_ingest_errors():
    P = ldpc()
    with pytest.raises(P.LdpcError, match="outside"):
        P.Handle(torch.tensor([[1, 2, 1], [1, 1, 0]], dtype=torch.uint8, device="cuda"))
    with pytest.raises(P.LdpcError, match="degree"):
        P.Handle(torch.tensor([[1, 0, 0], [0, 1, 1]], dtype=torch.uint8, device="cuda"))
    with pytest.raises(P.LdpcError, match="twice"):
        P.Handle.from_coo(torch.tensor([0, 0, 0], dtype=torch.int32, device="cuda"),
                          torch.tensor([1, 1, 2], dtype=torch.int32, device="cuda"), 1, 3)
    with pytest.raises(P.LdpcError, match="outside"):
        P.Handle.from_coo(torch.tensor([0, 0], dtype=torch.int32, device="cuda"),
                          torch.tensor([1, 3], dtype=torch.int32, device="cuda"), 1, 3)


# ---------------------------------------------------------------- single loop body (a3-a6) --
@pytest.mark.parametrize("flags", [0, LIT])
@pytest.mark.parametrize("seed", range(4))
def test_one_iteration_random_h(seed, flags):
    """L = 1 without early stop: one CN + BN sweep, bit-exact, on random H with odd/even rows and
    degree-0 columns; values include exact zeros, -0.0 and ties."""
    code = codes.random_small(37, 70, seed, 2, 9)
    rng = np.random.default_rng(seed)
    llr = rng.choice(np.array([-1.5, -1.0, -0.0, 0.0, 0.25, 1.0, 2.0], np.float32), size=(300, code.n))
    llr[::2] = rng.standard_normal((150, code.n)).astype(np.float32)
    for f in (FORCE_STREAM, FORCE_RESIDENT):
        h = handle(code, flags | NOES | f)
        if f == FORCE_RESIDENT and h.schedule != "resident":
            continue
        compare(code, llr, 1, flags | NOES, h=h)
        compare(code, llr, 3, flags | NOES, h=h)


def test_high_degree_rows_use_wide_locations():
    """Rows of degree > 255 switch min0Location to 16 bits."""
    rng = np.random.default_rng(1)
    rows = [np.sort(rng.choice(600, size=d, replace=False)) for d in (300, 2, 5, 280, 7, 3)]
    code = codes.from_rows(rows, 600)
    llr = (rng.standard_normal((200, 600)) - 1.2).astype(np.float32)
    h = handle(code, FORCE_STREAM)
    assert h.max_row_deg == 300
    compare(code, llr, 8, h=h)


# ---------------------------------------------------------------- end to end ----------------
@pytest.mark.parametrize("flags", [0, LIT, NOES, LIT | NOES])
def test_c1_paper_code_full(flags):
    """Config C1: the paper's 5x10 H, 10k frames over Eb/N0 {1,2,3,4}, max_iter 10 -- every frame."""
    cfg = codes.CONFIGS["c1"]
    code = cfg["code"]()
    llr, _ = channel.workload_llr(code, cfg, 0, cfg["frames"])
    compare(code, llr.numpy(), cfg["max_iter"], flags)


@pytest.mark.parametrize("sched", [FORCE_STREAM, FORCE_RESIDENT])
def test_c2_subset_full(sched):
    """C2 code (random (3,6) 504x1008), 12k frames spread over the sweep, max_iter 50 -- every frame."""
    cfg = codes.CONFIGS["c2"]
    code = cfg["code"]()
    h = handle(code, sched)
    if sched == FORCE_RESIDENT and h.schedule != "resident":
        pytest.skip("resident schedule unavailable")
    parts = []
    for p, e in enumerate(cfg["ebn0"]):
        parts.append(channel.bpsk_awgn(code.n, code.rate, e, cfg["seed"], p, 5000, 1700).numpy())
    llr = np.concatenate(parts)
    compare(code, llr, cfg["max_iter"], h=h)


@pytest.mark.parametrize("sched", [FORCE_STREAM, FORCE_STREAM | 16, FORCE_RESIDENT])
@pytest.mark.parametrize("T", [2, 6])
def test_check_every(sched, T):
    """checkEvery = T: codeword tests only after bodies k % T == 0 and after body L."""
    cfg = codes.CONFIGS["c2"]
    code = cfg["code"]()
    h = handle(code, sched)
    if h.schedule == "unavailable":
        pytest.skip("resident schedule unavailable")
    parts = [channel.bpsk_awgn(code.n, code.rate, e, cfg["seed"], p, 900, 400).numpy() for p, e in enumerate(cfg["ebn0"])]
    compare(code, np.concatenate(parts), 47, h=h, check_every=T)
    c1 = codes.paper_5x10()
    llr1 = channel.bpsk_awgn(10, 0.5, 1.0, 5, 0, 0, 3000).numpy()
    compare(c1, llr1, 10, h=handle(c1, sched & ~16 if sched == FORCE_RESIDENT else sched), check_every=T)


def test_edge_sizes_and_chunking():
    """frames = 0, 1, 127, 129 (ragged last tile), L = 0, and chunked decodes equal one-shot decodes."""
    code = codes.regular(60, 120, 3, 6, 5)
    llr = frames_for(code, 700, 1.5, 3)
    h = handle(code, FORCE_STREAM)
    for F in (1, 127, 129):
        compare(code, llr[:F], 20, h=h)
    compare(code, llr, 0, h=h)
    compare(code, llr, 0, NOES, h=handle(code, NOES | FORCE_STREAM))
    P = ldpc()
    out0 = h.decode(torch.from_numpy(llr[:0]).cuda(), 10)
    assert out0.bits.shape == (0, 120)
    ref = gpu_decode(h, llr, 20)
    h.set_chunk(256)
    chunked = gpu_decode(h, llr, 20)
    for a, b in zip(ref, chunked):
        assert np.array_equal(a, b)
    assert P is not None


@pytest.mark.parametrize("cfg_name,frames", [("c2", 3000), ("c4", 300)])
def test_graph_loop_equals_plain_launches(cfg_name, frames):
    """The graph-driven loop (conditional WHILE node) and plain per-body launches give identical results,
    including when every frame stops long before max_iter."""
    cfg = codes.CONFIGS[cfg_name]
    code = cfg["code"]()
    for p, e in ((0, cfg["ebn0"][0]), (len(cfg["ebn0"]) - 1, cfg["ebn0"][-1])):
        llr = channel.bpsk_awgn(code.n, code.rate, e, cfg["seed"], p, 0, frames).numpy()
        ref = gpu_decode(handle(code, FORCE_STREAM | 16, coo=True), llr, cfg["max_iter"])
        got = gpu_decode(handle(code, FORCE_STREAM, coo=True), llr, cfg["max_iter"])
        for a, b in zip(ref, got):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("knob", ["default", "LDPC_CN_GENERIC", "LDPC_CN_BULK", "LDPC_NO_COMPACT"])
def test_stream_variants(monkeypatch, knob):
    """Every kernel variant of the streaming schedule is bit-identical: the degree-specialised check node
    (rows of degree <= 8, default), the any-degree one (LDPC_CN_GENERIC=1) or the one whose rows are staged
    by cp.async.bulk (LDPC_CN_BULK=1); with or without the compaction of sparse tiles (LDPC_NO_COMPACT=1)."""
    if knob != "default":
        monkeypatch.setenv(knob, "1")
    cfg = codes.CONFIGS["c2"]
    code = cfg["code"]()
    parts = [channel.bpsk_awgn(code.n, code.rate, e, cfg["seed"], p, 100, 300).numpy() for p, e in enumerate(cfg["ebn0"])]
    llr = np.concatenate(parts)
    for flags in (FORCE_STREAM, FORCE_STREAM | 16, FORCE_STREAM | NOES | LIT):
        compare(code, llr, cfg["max_iter"], flags, h=handle(code, flags))
    code3 = codes.random_small(37, 70, 2, 2, 9)  # irregular, rows of degree 2..
    llr3 = (np.random.default_rng(3).standard_normal((300, code3.n)) - 0.5).astype(np.float32)
    compare(code3, llr3, 12, h=handle(code3, FORCE_STREAM))


@pytest.mark.parametrize("graph", [True, False])
@pytest.mark.parametrize("T", [1, 3])
def test_compaction_moves_frames_exactly(graph, T):
    """Tiles whose running frames drop under half are compacted into fresh tiles: a batch that
    interleaves easy (5 dB) and hard (1 dB) frames makes most tiles sparse after a few bodies.  Results equal
    the oracle and the uncompacted decode bit for bit, and the handle reports frames actually moved."""
    code = codes.regular(504, 1008, 3, 6, 1008)
    F = 128 * 40 + 77  # ragged last tile
    easy = channel.bpsk_awgn(code.n, code.rate, 5.0, 3, 0, 0, F).numpy()
    hard = channel.bpsk_awgn(code.n, code.rate, 1.0, 3, 1, 0, F).numpy()
    pick = (np.arange(F) % 5) == 0  # 20 % hard frames in every tile
    llr = np.where(pick[:, None], hard, easy).astype(np.float32)
    flags = FORCE_STREAM | (0 if graph else 16)
    h = handle(code, flags)
    got = compare(code, llr, 40, flags, h=h, check_every=T)
    c = h.stream_counters()
    assert c["compactions"] >= 1 and c["frames_moved"] > 0 and c["tiles_retired"] > c["compactions"]
    import os

    os.environ["LDPC_NO_COMPACT"] = "1"
    try:
        h2 = handle(code, flags)
    finally:
        del os.environ["LDPC_NO_COMPACT"]
    ref = compare(code, llr, 40, flags, h=h2, check_every=T)
    assert h2.stream_counters()["compactions"] == 0
    for a_, b_ in zip(got, ref):
        assert np.array_equal(a_, b_)


@pytest.mark.parametrize("which", ["paper", "reg", "small"])
def test_resident_compact_records(monkeypatch, which):
    """The compact bit-node records (u16 row offset + u8 position, recomputed ballot word and bit) are
    bit-identical to the oracle on regular and irregular codes (LDPC_RES_COMPACT=1 forces them)."""
    monkeypatch.setenv("LDPC_RES_COMPACT", "1")
    code = {"paper": codes.paper_5x10, "reg": lambda: codes.regular(504, 1008, 3, 6, 1008),
            "small": lambda: codes.random_small(37, 70, 2, 2, 9)}[which]()
    h = handle(code, FORCE_RESIDENT)
    assert h.schedule == "resident"
    rng = np.random.default_rng(8)
    llr = (rng.standard_normal((700, code.n)) * 1.2 - 0.9).astype(np.float32)
    compare(code, llr, 25, h=h)


@pytest.mark.parametrize("shape", [(60, 200, 2, 20), (300, 900, 3, 17), (120, 128, 9, 16)])
@pytest.mark.parametrize("flags", [FORCE_STREAM, FORCE_RESIDENT])
def test_high_degree_irregular_rows(shape, flags):
    """Irregular codes with rows of degree up to 20 (several sign words per row and lane in both
    schedules; the generic streaming check node), early stop on, against the oracle."""
    m, n, dmin, dmax = shape
    code = codes.random_small(m, n, 31 + m, dmin, dmax)
    h = handle(code, flags)
    if flags == FORCE_RESIDENT:
        assert h.schedule == "resident"
    rng = np.random.default_rng(m)
    llr = (rng.standard_normal((500, code.n)) * 0.8 - 1.1).astype(np.float32)
    compare(code, llr, 15, h=h)


@pytest.mark.parametrize("threads", ["128", "384", "1024"])
def test_resident_forced_threads(monkeypatch, threads):
    """LDPC_RES_THREADS forces the CTA size; with compact records the planner falls back to a compact
    kernel size (regression: a 384-thread request once launched the non-compact kernel on a compact
    layout)."""
    monkeypatch.setenv("LDPC_RES_THREADS", threads)
    code = codes.regular(504, 1008, 3, 6, 1008)
    rng = np.random.default_rng(int(threads))
    llr = (rng.standard_normal((400, code.n)) * 1.2 - 0.9).astype(np.float32)
    compare(code, llr, 25, h=handle(code, FORCE_RESIDENT))
    monkeypatch.setenv("LDPC_RES_COMPACT", "1")
    compare(code, llr, 25, h=handle(code, FORCE_RESIDENT))


@pytest.mark.parametrize("case", range(int(__import__("os").environ.get("LDPC_RAND_CASES", "12"))))
def test_randomised_shapes_flags_and_check_points(case):
    """Randomised sweep: code shape (rows of degree 2..14, columns of degree 0 allowed), sign rule,
    early stop, checkEvery and batch size, both schedules, against the oracle."""
    rng = np.random.default_rng(1000 + case)
    m = int(rng.integers(8, 400))
    n = int(rng.integers(m + 4, 3 * m + 40))
    dmin = int(rng.integers(2, 5))
    dmax = int(rng.integers(dmin, 15))
    code = codes.random_small(m, n, 77 + case, dmin, dmax)
    flags = int(rng.choice([0, LIT, NOES, LIT | NOES]))
    T = int(rng.choice([1, 1, 2, 3, 6]))
    L = int(rng.integers(1, 30))
    F = int(rng.integers(1, 700))
    llr = (rng.standard_normal((F, code.n)) * rng.uniform(0.5, 2.0) - rng.uniform(0.0, 2.0)).astype(np.float32)
    for sched in (FORCE_STREAM, FORCE_RESIDENT):
        h = handle(code, flags | sched)
        if h.schedule == "unavailable":
            continue
        compare(code, llr, L, flags | sched, h=h, check_every=T)


@pytest.mark.parametrize("generic", ["1", "2"])
def test_resident_generic_equals_regular_instance(monkeypatch, generic):
    """The degree-specialised resident kernel for regular (3,6) codes and the generic ones agree
    (LDPC_RES_GENERIC=1: the instance for rows of degree <= 8; =2: the any-degree instance), and all
    match the oracle."""
    cfg = codes.CONFIGS["c2"]
    code = cfg["code"]()
    parts = [channel.bpsk_awgn(code.n, code.rate, e, cfg["seed"], p, 500, 300).numpy() for p, e in enumerate(cfg["ebn0"])]
    llr = np.concatenate(parts)
    ref = compare(code, llr, cfg["max_iter"], FORCE_RESIDENT, h=handle(code, FORCE_RESIDENT))
    monkeypatch.setenv("LDPC_RES_GENERIC", generic)
    got = compare(code, llr, cfg["max_iter"], FORCE_RESIDENT, h=handle(code, FORCE_RESIDENT))
    for a, b in zip(ref, got):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("flags", [FORCE_STREAM, FORCE_RESIDENT, FORCE_STREAM | LIT])
def test_signed_zeros_and_ties(flags):
    """Channel values with many exact +0 / -0 entries and exact magnitude ties (reading A12: sign(-0) =
    sign(+0) = +1, slice(+-0) = 0; A13: ties).  The decoders keep zeros of s canonical (+0 streaming, -0
    resident), so the posterior is compared up to the sign of zero (not a decision)."""
    code = codes.regular(504, 1008, 3, 6, 1008)
    rng = np.random.default_rng(12)
    y = np.round(rng.normal(-0.6, 1.0, size=(700, code.n)) * 2.0) / 2.0  # half-integer grid: ties, zeros
    y = y.astype(np.float32)
    zero = y == 0
    y[zero & (rng.random(y.shape) < 0.5)] = np.float32(-0.0)
    y[:50] = np.where(rng.random((50, code.n)) < 0.3, np.float32(-0.0), y[:50])
    compare(code, y, 20, flags, h=handle(code, flags))


def test_nonzero_codewords_and_symmetry():
    """Random nonzero codewords (no all-zero bias) and the codeword-symmetry law on the GPU (T5)."""
    code = codes.paper_5x10()
    H = code.dense()
    import itertools

    V = np.array(list(itertools.product([0, 1], repeat=10)), np.uint8)
    C = V[((V.astype(np.int64) @ H.T) % 2).sum(axis=1) == 0]
    rng = np.random.default_rng(4)
    cw = C[rng.integers(len(C), size=2000)]
    llr = channel.bpsk_awgn(10, 0.5, 1.0, 77, 0, 0, 2000, codeword=torch.from_numpy(cw)).numpy()
    compare(code, llr, 10)
    h = handle(code)
    b0, i0, c0, p0, _ = gpu_decode(h, llr, 10)
    c = C[5]
    t = (1.0 - 2.0 * c).astype(np.float32)
    b1, i1, c1, p1, _ = gpu_decode(h, llr * t, 10)
    ok = np.all(p0 != 0, axis=1)
    assert np.array_equal(b1[ok], (b0 ^ c)[ok]) and np.array_equal(i1[ok], i0[ok])


def test_power_of_two_scale_on_gpu():
    code = codes.regular(252, 504, 3, 6, 17)
    llr = frames_for(code, 1000, 2.0, 8)
    h = handle(code)
    b0, i0, c0, p0, _ = gpu_decode(h, llr, 30)
    b1, i1, c1, p1, _ = gpu_decode(h, llr * np.float32(8), 30)
    assert np.array_equal(b0, b1) and np.array_equal(i0, i1) and np.array_equal(p1, p0 * np.float32(8))


def test_decode_host_matches_device():
    code = codes.regular(504, 1008, 3, 6, 1008)
    llr = frames_for(code, 3000, 2.0, 9)
    h = handle(code)
    gb, gi, gc, gp, gs = gpu_decode(h, llr, 30)
    st = torch.zeros(8, dtype=torch.int64)
    out = h.decode_host(torch.from_numpy(llr).pin_memory(), 30, posterior=True, stats=st)
    assert np.array_equal(out.bits.numpy(), gb) and np.array_equal(out.iters.numpy(), gi)
    assert np.array_equal(out.posterior.numpy(), gp) and np.array_equal(st.numpy(), gs)


# ---------------------------------------------------------------- full-size, sampled ---------
def _sampled_full_size(cfg_name, sample, flags=0, chunk=None):
    """Decode the config's full batch in the bench's launch configuration, then check `sample`
    frames spread over the batch against the oracle, frame by frame."""
    cfg = codes.CONFIGS[cfg_name]
    code = cfg["code"]()
    llr, pidx = channel.workload_llr(code, cfg, 0, cfg["frames"], device="cuda")
    h = handle(code, flags, coo=True)
    if chunk:
        h.set_chunk(chunk)
    out = h.decode(llr, cfg["max_iter"], posterior=True)
    torch.cuda.synchronize()
    idx = np.unique(np.linspace(0, cfg["frames"] - 1, sample).astype(np.int64))
    sub = llr[torch.from_numpy(idx).cuda()].cpu().numpy()
    ob, oi, oc, op = oracle.decode(code.oracle_h(), sub, cfg["max_iter"], flags=flags & (LIT | NOES))
    gb = out.bits[torch.from_numpy(idx).cuda()].cpu().numpy()
    gi = out.iters.cpu().numpy()[idx]
    gc = out.converged.cpu().numpy()[idx]
    gp = out.posterior[torch.from_numpy(idx).cuda()].cpu().numpy()
    assert np.array_equal(gi, oi) and np.array_equal(gc, oc) and np.array_equal(gb, ob)
    assert np.allclose(gp, op, rtol=TOL, atol=TOL)
    near_zero = int(np.count_nonzero(np.abs(op).min(axis=1) <= TOL))
    return near_zero, oi


def test_c2_full_size_sampled():
    _sampled_full_size("c2", 1500)


def test_c3_full_size_sampled():
    _sampled_full_size("c3", 48)


def test_c4_full_size_sampled():
    _sampled_full_size("c4", 12)


@pytest.mark.parametrize("mode", ["default", "global_graph"])
def test_c6_paper_shaped_qc(monkeypatch, mode):
    """C6: the paper's benchmark shape (QC 1022 x 8176, row degree 32; max 60 iterations, codeword
    test every 6, SNR 3.0-3.6 dB) -- every frame of a reduced batch, with the default schedule
    (streaming) and the resident one with the edge lists in global memory (LDPC_RES_GG=1)."""
    cfg = codes.CONFIGS["c6"]
    code = cfg["code"]()
    parts = [channel.bpsk_awgn(code.n, code.rate, e, cfg["seed"], p, 0, 150).numpy() for p, e in enumerate(cfg["ebn0"])]
    if mode == "global_graph":
        monkeypatch.setenv("LDPC_RES_GG", "1")
    h = handle(code, 0, coo=True)
    assert h.schedule == ("resident" if mode == "global_graph" else "stream")
    compare(code, np.concatenate(parts), cfg["max_iter"], check_every=cfg["check_every"], h=h)


@pytest.mark.parametrize("generic", ["0", "2"])
def test_resident_global_graph_mode(monkeypatch, generic):
    """The resident schedule with the edge lists read from global memory (LDPC_RES_GG=1 forces it; the
    bounded-degree and the any-degree instances) matches the oracle on the C2 code and on an irregular code."""
    monkeypatch.setenv("LDPC_RES_GG", "1")
    if generic != "0":
        monkeypatch.setenv("LDPC_RES_GENERIC", generic)
    cfg = codes.CONFIGS["c2"]
    code = cfg["code"]()
    parts = [channel.bpsk_awgn(code.n, code.rate, e, cfg["seed"], p, 100, 200).numpy() for p, e in enumerate(cfg["ebn0"])]
    compare(code, np.concatenate(parts), cfg["max_iter"], FORCE_RESIDENT, h=handle(code, FORCE_RESIDENT))
    code = codes.random_small(300, 700, 21, dmin=2, dmax=12)  # odd and even row degrees up to 12
    llr = channel.bpsk_awgn(code.n, code.rate, 2.0, 5, 0, 0, 900).numpy()
    compare(code, llr, 25, FORCE_RESIDENT, h=handle(code, FORCE_RESIDENT))


def test_c5_sixteen_handles():
    """C5: 16 distinct H of equal dims through one handle API; every frame of a reduced batch."""
    cfg = codes.CONFIGS["c5"]
    for hidx, code in enumerate(cfg["code"]()):
        if hidx % 4:
            continue
        parts = [channel.bpsk_awgn(code.n, code.rate, e, cfg["seed"] + hidx, p, 0, 80).numpy()
                 for p, e in enumerate(cfg["ebn0"])]
        llr = np.concatenate(parts)
        h = handle(code)
        assert h.schedule == "resident"  # compact bit-node records make the 2048 x 4096 state fit
        res = compare(code, llr, cfg["max_iter"], h=h)
        got = compare(code, llr, cfg["max_iter"], FORCE_STREAM, h=handle(code, FORCE_STREAM))
        for a, b in zip(res, got):
            assert np.array_equal(a, b)


def test_generator_device_independent():
    """The keyed generator gives the same frames on CPU and GPU (bench inputs == test inputs)."""
    code = codes.regular(504, 1008, 3, 6, 1008)
    a = channel.bpsk_awgn(code.n, code.rate, 2.0, 1, 0, 1000, 500)
    b = channel.bpsk_awgn(code.n, code.rate, 2.0, 1, 0, 1000, 500, device="cuda").cpu()
    assert (a != b).sum().item() <= 2  # libm ulp differences can flip a rare last bit


def test_compute_sanitizer_clean():
    """memcheck, racecheck and synccheck report nothing on small decodes of both schedules (T6).
    memcheck runs the default path (CUDA-graph loop).  racecheck and synccheck run the same decodes with
    plain launches (LDPC_NO_GRAPHS=1): under a graph with a device-driven conditional WHILE node this
    toolkit's racecheck crashes the process and synccheck reports "divergent threads" at barriers that a
    stand-alone probe of the same loop (tools/probe_sync.cu) and the plain-launch run show clean."""
    import os
    import shutil
    import subprocess

    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(cs):
        pytest.skip("compute-sanitizer not available")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for tool, env in (("memcheck", {}), ("racecheck", {"LDPC_NO_GRAPHS": "1"}), ("synccheck", {"LDPC_NO_GRAPHS": "1"})):
        r = subprocess.run([cs, "--tool", tool, "--error-exitcode", "3", sys.executable,
                            os.path.join(root, "tools", "sanitize_run.py")], capture_output=True, text=True,
                           timeout=900, env=dict(os.environ, **env))
        if r.returncode != 0 and "compute-sanitizer is closed" in r.stdout + r.stderr:
            pytest.skip("compute-sanitizer is disabled on this GPU pool (its wrapper refuses to run)")
        assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
        assert "0 errors" in r.stdout or "0 hazards" in r.stdout or "0 error" in r.stdout, r.stdout[-2000:]


def test_binding_validates_buffers():
    """The binding refuses buffers whose shape, dtype, contiguity or device would make the C-ABI read or write
    out of bounds (llr [F, n], out fields [F, n] / [F], stats int64[8])."""
    P = ldpc()
    code = codes.regular(60, 120, 3, 6, 5)
    h = handle(code)
    llr = torch.zeros((10, 120), dtype=torch.float32, device="cuda")
    with pytest.raises(ValueError):
        h.decode(torch.zeros((10, 121), dtype=torch.float32, device="cuda"), 5)
    with pytest.raises(ValueError):
        h.decode(llr.double(), 5)
    with pytest.raises(ValueError):
        h.decode(torch.zeros((120, 10), dtype=torch.float32, device="cuda").t(), 5)
    bad = P.DecodeResult(torch.empty((9, 120), dtype=torch.uint8, device="cuda"), None, None, None)
    with pytest.raises(ValueError):
        h.decode(llr, 5, out=bad)
    bad = P.DecodeResult(None, torch.empty(10, dtype=torch.int64, device="cuda"), None, None)
    with pytest.raises(ValueError):
        h.decode(llr, 5, out=bad)
    bad = P.DecodeResult(None, None, None, torch.empty((10, 120), dtype=torch.float32))
    with pytest.raises(ValueError):
        h.decode(llr, 5, out=bad)  # posterior on the host for a device decode
    with pytest.raises(ValueError):
        h.decode(llr, 5, stats=torch.zeros(7, dtype=torch.int64, device="cuda"))
    with pytest.raises(ValueError):
        h.decode_host(torch.zeros((10, 119), dtype=torch.float32), 5)
    with pytest.raises(ValueError):
        h.decode_host(torch.zeros((10, 120), dtype=torch.float32), 5,
                      out=P.DecodeResult(torch.empty((10, 120), dtype=torch.uint8, device="cuda"), None, None, None))
    out = h.decode(llr, 5)  # and the valid call still works
    torch.cuda.synchronize()
    assert out.bits.shape == (10, 120)


def test_stream_counters_and_launch_count():
    """ldpc_launch_count includes the loop bodies the graph's conditional node ran (counted on the device):
    a graph decode and a plain-launch decode of the same frames count the same kernels per body; the
    tile-body counters equal the tiles x bodies swept."""
    code = codes.regular(504, 1008, 3, 6, 1008)
    llr = channel.bpsk_awgn(code.n, code.rate, 1.0, 3, 0, 0, 128 * 6).numpy()  # 6 tiles, every frame runs L
    L = 12
    counts = {}
    for flags in (FORCE_STREAM, FORCE_STREAM | 16):
        h = handle(code, flags | NOES)
        l0 = h.launch_count
        gpu_decode(h, llr, L)
        counts[flags] = h.launch_count - l0
        c = h.stream_counters()
        assert c["cn_tile_bodies"] == 6 * L and c["bn_tile_bodies"] == 6 * L, c
    # plain launches: stage-in, L x (check node, bit node, compaction plan + move), syndrome, finalize, stats
    assert counts[FORCE_STREAM | 16] == 1 + 4 * L + 3
    # graph: the same kernels plus the loop-control kernels (pre + one step per body after the first)
    assert counts[FORCE_STREAM] == 1 + 4 * L + 3 + 1 + (L - 1)
