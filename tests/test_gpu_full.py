"""Full-batch GPU-vs-oracle parity on every benchmark configuration (north_star: "bit-exact hard
decisions and iteration counts vs the CPU oracle on every config").

Each test decodes the config's WHOLE batch in the launch configuration bench.py times (one
ldpc_decode over the rank's batch, H ingested from COO, default schedule and flags), then checks
EVERY frame against the oracle run on all host cores: bits, k and isCodeword bit-exact, posterior
within 1e-4 (and bit-exact up to the sign of a zero, reading A12), the 8 counters equal.  Frames with
a posterior entry within 1e-4 of zero are counted separately (north_star) and reported in
gpurun_out/parity_report.jsonl (and on stdout).
"""
import json
import os
import time

import numpy as np
import pytest
import torch

import bench
import oracle
from gen import codes

pytestmark = pytest.mark.gpu

TOL = 1e-4
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REPORT = os.environ.get("LDPC_PARITY_REPORT", os.path.join(ROOT, "gpurun_out", "parity_report.jsonl"))
CHUNK = 1 << 16  # frames compared per oracle call (bounds host memory)


def report(rec):
    print(json.dumps(rec))
    try:
        os.makedirs(os.path.dirname(REPORT), exist_ok=True)
        with open(REPORT, "a") as f:
            f.write(json.dumps(rec) + "\n")
    except OSError:
        pass


def check_batch(name, code, llr_dev, L, flags=0, check_every=1, expect_schedule=None):
    import paper_2507_10424_b200 as P

    rr, cc = code.coo()
    h = P.Handle.from_coo(torch.from_numpy(rr).cuda(), torch.from_numpy(cc).cuda(), code.m, code.n, flags=flags)
    if expect_schedule:
        assert h.schedule == expect_schedule
    if check_every != 1:
        h.set_check_every(check_every)
    st = torch.zeros(8, dtype=torch.int64, device="cuda")
    t0 = time.perf_counter()
    out = h.decode(llr_dev, L, posterior=True, stats=st)
    torch.cuda.synchronize()
    t_gpu = time.perf_counter() - t0
    F = llr_dev.shape[0]
    ost = np.zeros(8, np.int64)
    near_gpu = near_orc = 0
    t_or = 0.0
    for a in range(0, F, CHUNK):
        b = min(F, a + CHUNK)
        llr = llr_dev[a:b].cpu().numpy()
        t1 = time.perf_counter()
        ob, oi, oc, op = oracle.decode(code.oracle_h(), llr, L, flags=flags & 3, check_every=check_every)
        t_or += time.perf_counter() - t1
        gb = out.bits[a:b].cpu().numpy()
        gi = out.iters[a:b].cpu().numpy()
        gc = out.converged[a:b].cpu().numpy()
        gp = out.posterior[a:b].cpu().numpy()
        bad_i = np.nonzero(gi != oi)[0]
        assert len(bad_i) == 0, f"{name}: k differs on {len(bad_i)} frames, first {a + bad_i[:5]}"
        assert np.array_equal(gc, oc), f"{name}: isCodeword differs"
        bad_b = np.nonzero(np.any(gb != ob, axis=1))[0]
        assert len(bad_b) == 0, f"{name}: bits differ on {len(bad_b)} frames, first {a + bad_b[:5]}"
        assert np.allclose(gp, op, rtol=TOL, atol=TOL), f"{name}: posterior beyond 1e-4"
        z = np.float32(0.0)
        assert np.array_equal((gp + z).view(np.uint32), (op + z).view(np.uint32)), f"{name}: posterior not bit-exact"
        near_gpu += int(np.count_nonzero(np.abs(gp).min(axis=1) <= TOL))
        near_orc += int(np.count_nonzero(np.abs(op).min(axis=1) <= TOL))
        ost += oracle.stats(llr, ob, oi, oc, op)
    assert np.array_equal(st.cpu().numpy(), ost), f"{name}: counters differ"
    assert near_gpu == near_orc
    rec = {"test": name, "frames": int(F), "n": code.n, "m": code.m, "max_iter": L, "check_every": check_every,
           "schedule": h.schedule, "bit_exact_frames": int(F), "near_zero_frames": near_gpu,
           "sum_iters": int(ost[4]), "converged": int(ost[5]), "gpu_s": round(t_gpu, 3), "oracle_s": round(t_or, 1),
           "oracle_threads": oracle.max_threads()}
    report(rec)
    h.close()
    return rec


def full_config(cfg_name, code_idx=0):
    cfg = codes.CONFIGS[cfg_name]
    cl = bench.code_list(cfg)
    code = cl[code_idx]
    llr, _ = bench.gen_frames(code, cfg, bench.seed_of(cfg, code_idx), 0, cfg["frames"], 0, device="cuda")
    return cfg, code, llr


@pytest.mark.parametrize("cfg_name", ["c1", "c2", "c3", "c4", "c6"])
def test_full_batch_parity(cfg_name):
    """The bench's whole batch of the config, every frame against the oracle."""
    cfg, code, llr = full_config(cfg_name)
    check_batch(f"full_{cfg_name}", code, llr, cfg["max_iter"], check_every=cfg.get("check_every", 1))


def test_full_batch_parity_c5_all_codes():
    """C5, the code-selection sweep: all 16 codes (16 handles), each its whole 16,384-frame batch."""
    cfg = codes.CONFIGS["c5"]
    for hidx in range(16):
        _, code, llr = full_config("c5", hidx)
        check_batch(f"full_c5_h{hidx}", code, llr, cfg["max_iter"], expect_schedule="resident")
        del llr


@pytest.mark.parametrize("flags", [4, 4 | 2, 4 | 1])
def test_full_batch_parity_c2_streaming(flags):
    """The C2 batch through the HBM-streaming schedule too (forced), with and without early stop and
    with the paper-literal sign rule, on a quarter of the batch (every Eb/N0 block)."""
    cfg, code, llr = full_config("c2")
    idx = torch.arange(0, llr.shape[0], 4, device="cuda")
    check_batch(f"c2_stream_flags{flags}", code, llr[idx].contiguous(), cfg["max_iter"], flags=flags)


@pytest.mark.parametrize("flags,nbuf", [(0, "3"), (4, "3"), (0, "2"), (4, "4")])
def test_decode_host_multichunk(monkeypatch, flags, nbuf):
    """ldpc_decode_host with a 1 MB chunk: about ten ramped chunks through 2-4 rotating buffer sets
    (ev_out reuse), against the oracle and against the device-buffer call."""
    import paper_2507_10424_b200 as P

    monkeypatch.setenv("LDPC_HOST_CHUNK_MB", "1")
    monkeypatch.setenv("LDPC_HOST_NBUF", nbuf)
    cfg = codes.CONFIGS["c2"]
    code = bench.code_list(cfg)[0]
    llr, _ = bench.gen_frames(code, cfg, cfg["seed"], 0, cfg["frames"], 0)
    sel = torch.arange(0, cfg["frames"], 311)[:3000]
    llr = llr[sel].contiguous()
    rr, cc = code.coo()
    h = P.Handle.from_coo(torch.from_numpy(rr).cuda(), torch.from_numpy(cc).cuda(), code.m, code.n, flags=flags)
    st = torch.zeros(8, dtype=torch.int64)
    out = h.decode_host(llr.pin_memory(), cfg["max_iter"], posterior=True, stats=st)
    ob, oi, oc, op = oracle.decode(code.oracle_h(), llr.numpy(), cfg["max_iter"])
    assert np.array_equal(out.iters.numpy(), oi) and np.array_equal(out.converged.numpy(), oc)
    assert np.array_equal(out.bits.numpy(), ob)
    assert np.allclose(out.posterior.numpy(), op, rtol=TOL, atol=TOL)
    assert np.array_equal(st.numpy(), oracle.stats(llr.numpy(), ob, oi, oc, op))
    dev = h.decode(llr.cuda(), cfg["max_iter"], posterior=True)
    torch.cuda.synchronize()
    assert np.array_equal(dev.posterior.cpu().numpy(), out.posterior.numpy())
    # pageable (not pinned) host buffers take the same path
    out2 = h.decode_host(llr, cfg["max_iter"], posterior=False)
    assert np.array_equal(out2.bits.numpy(), ob) and np.array_equal(out2.iters.numpy(), oi)
    h.close()


def test_dense_ish_h():
    """H as an argument allows dense-ish matrices (P:5): 1000 x 4000 with a degree-3000 row and a
    degree-1000 column, ingested dense and from COO; decoded (16-bit locations, generic check node)
    against the oracle."""
    import paper_2507_10424_b200 as P

    rng = np.random.default_rng(5)
    m, n = 1000, 4000
    rows = []
    for i in range(m):
        d = 3000 if i == 17 else int(rng.integers(3, 9))
        r = set(rng.choice(np.arange(1, n), size=d - 1, replace=False).tolist())
        r.add(0)  # column 0 has degree 1000
        rows.append(sorted(r))
    code = codes.from_rows(rows, n)
    assert max(len(r) for r in code.rows) == 3000
    H = torch.from_numpy(code.dense()).cuda()
    hd = P.Handle(H)
    rr, cc = code.coo()
    perm = rng.permutation(len(rr))
    hc = P.Handle.from_coo(torch.from_numpy(rr[perm]).cuda(), torch.from_numpy(cc[perm]).cuda(), m, n)
    assert hd.max_row_deg == 3000 and hd.max_col_deg == 1000 and hc.max_col_deg == 1000
    for a, b in zip(hd.graph(), hc.graph()):
        assert torch.equal(a, b)
    llr = (rng.standard_normal((96, n)) * 0.9 - 1.3).astype(np.float32)
    ob, oi, oc, op = oracle.decode(code.oracle_h(), llr, 4)
    out = hc.decode(torch.from_numpy(llr).cuda(), 4, posterior=True)
    torch.cuda.synchronize()
    assert np.array_equal(out.iters.cpu().numpy(), oi) and np.array_equal(out.bits.cpu().numpy(), ob)
    assert np.allclose(out.posterior.cpu().numpy(), op, rtol=TOL, atol=TOL)
    hd.close()
    hc.close()
