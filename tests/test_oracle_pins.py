"""Pins of the CPU oracle against what the paper and the mathematics fix (no GPU).

Each test names the pin of DESIGN.md "Oracle pins" (P1..P13) and the passage it
follows.  None of them re-types the oracle's formula: they use the paper's printed
example, closed forms (ML / max-marginals by enumeration), symmetry laws, and
brute force on tiny inputs.
"""
import itertools
import os

import numpy as np
import pytest

from conftest import GOLDEN
from gen import channel, codes

SIGN_PAPER_LITERAL = 1
NO_EARLY_STOP = 2


def load_paper_h():
    rows = []
    with open(os.path.join(GOLDEN, "paper_5x10.txt")) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append([int(t) - 1 for t in line.split()])
    return codes.from_rows(rows, 10, "paper5x10")


def gf2_rank(H):
    A = (np.array(H, dtype=np.uint8) & 1).copy()
    r = 0
    rows, cols = A.shape
    for c in range(cols):
        piv = [i for i in range(r, rows) if A[i, c]]
        if not piv:
            continue
        A[[r, piv[0]]] = A[[piv[0], r]]
        for i in range(rows):
            if i != r and A[i, c]:
                A[i] ^= A[r]
        r += 1
    return r


def all_vectors(n):
    return np.array(list(itertools.product([0, 1], repeat=n)), dtype=np.uint8)


def kernel_by_enumeration(H):
    V = all_vectors(H.shape[1])
    return V[((V.astype(np.int64) @ H.T.astype(np.int64)) % 2).sum(axis=1) == 0]


# ---------------------------------------------------------------- P1, P2 ------------------
def test_p1_paper_h_structure(oracle_mod):
    """P1: the index sets give a (3,6)-regular H of GF(2) rank 5 with 32 codewords,
    weight enumerator 1 + 15x^4 + 15x^6 + x^10; all-ones is a codeword.  The oracle's
    syndrome agrees with the dense GF(2) product on all 2^10 vectors."""
    code = load_paper_h()
    assert all(np.array_equal(a, b) for a, b in zip(code.rows, codes.paper_5x10().rows))
    H = code.dense()
    assert list(H.sum(axis=1)) == [6] * 5 and list(H.sum(axis=0)) == [3] * 10
    assert gf2_rank(H) == 5
    V = all_vectors(10)
    dense_syn = ((V.astype(np.int64) @ H.T.astype(np.int64)) % 2).sum(axis=1)
    orc_syn = oracle_mod.syndrome_weight(H, V)
    assert np.array_equal(dense_syn, orc_syn)
    K = V[dense_syn == 0]
    assert len(K) == 32
    w = np.bincount(K.sum(axis=1), minlength=11)
    assert list(w) == [1, 0, 0, 0, 15, 0, 15, 0, 0, 0, 1]
    assert oracle_mod.syndrome_weight(H, np.ones(10, np.uint8))[0] == 0


def test_p2_syndrome_examples(oracle_mod):
    """P2: syndrome(e_1) = (1,1,0,0,1), syndrome(e_3) = (1,1,1,0,0); M_3 = {1,2,3}."""
    H = load_paper_h().dense()
    for bit, expect in ((0, [1, 1, 0, 0, 1]), (2, [1, 1, 1, 0, 0])):
        e = np.zeros(10, np.uint8)
        e[bit] = 1
        assert list(H @ e % 2) == expect
        assert oracle_mod.syndrome_weight(H, e)[0] == sum(expect)
        # per-row: the syndrome of each single check (1 x 10 sub-matrix) is its row of H.e
        for i in range(5):
            assert oracle_mod.syndrome_weight((np.array([0] * 6, np.int32), np.nonzero(H[i])[0].astype(np.int32),
                                               1, 10), e)[0] == expect[i]
    assert list(np.nonzero(H[:, 2])[0] + 1) == [1, 2, 3]


# ---------------------------------------------------------------- P3 ----------------------
def test_p3_codewords_pass_in_zero_iterations(oracle_mod):
    """P3: every codeword c sent noiselessly (r = 2c-1) returns (true, 0, c, r);
    every non-codeword hard vector needs at least one iteration."""
    H = load_paper_h().dense()
    V = all_vectors(10)
    r = (2.0 * V - 1.0).astype(np.float32)
    bits, iters, conv, post = oracle_mod.decode(H, r, 10)
    cw = ((V.astype(np.int64) @ H.T) % 2).sum(axis=1) == 0
    assert cw.sum() == 32
    assert np.all(iters[cw] == 0) and np.all(conv[cw] == 1)
    assert np.array_equal(bits[cw], V[cw]) and np.array_equal(post[cw], r[cw])
    assert np.all(iters[~cw] >= 1)


# ---------------------------------------------------------------- P4 ----------------------
def test_p4_worked_example(oracle_mod):
    """P4: hand-derived first iteration on the paper's H (tests/golden/worked_example_p4.txt)."""
    spec = {}
    msgs = []
    with open(os.path.join(GOLDEN, "worked_example_p4.txt")) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            key, val = line.split(":", 1)
            if key.startswith("bit"):
                left, right = val.split("|")
                msgs.append(([float(t) for t in left.split()], float(right)))
            else:
                spec[key] = [float(t) for t in val.split()]
    r = np.array(spec["r"], np.float32)
    H = load_paper_h().dense()
    for flags in (0, SIGN_PAPER_LITERAL):
        bits, iters, conv, post = oracle_mod.decode(H, r[None], 50, flags=flags)
        assert iters[0] == int(spec["k"][0]) and conv[0] == int(spec["converged"][0])
        assert list(bits[0]) == [int(x) for x in spec["b"]]
        for j, (etas, s_dec) in enumerate(msgs):
            acc = np.float32(0.0)
            for e in etas:  # hand-derived messages summed in ascending row order, then + r (A14)
                acc = np.float32(acc + np.float32(e))
            s_expect = np.float32(acc + r[j])
            assert post[0, j] == s_expect, (j, post[0, j], s_expect)
            assert abs(float(post[0, j]) - s_dec) < 1e-6


# ---------------------------------------------------------------- P5 ----------------------
def _obs12_fast_path(x, literal):
    """Eq. etaCalculation with Observation 1 (min1 at min0Location,
    reading A2) and Observation 2: written independently of the oracle."""
    a = np.abs(x)
    loc = int(np.argmin(a))
    min0 = a[loc]
    min1 = np.min(np.delete(a, loc))
    neg = x < 0
    parity = int(np.count_nonzero(neg)) & 1
    out = np.empty_like(x)
    for j in range(len(x)):
        mag = min1 if j == loc else min0
        s = parity ^ int(neg[j]) ^ (0 if literal else (len(x) & 1))
        out[j] = -mag if s else mag
    return out


def test_p5_check_node_examples(oracle_mod):
    """P5: SPEC examples under the literal rule; odd rows negate under CORRECTED."""
    with open(os.path.join(GOLDEN, "check_node_spec.txt")) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            left, right = line.split("|")
            x = np.array([float(t) for t in left.split()], np.float32)
            y = np.array([float(t) for t in right.split()], np.float32)
            # bitwise: the sign of a zero output is fixed too (sign(0) = +1)
            got = oracle_mod.check_node(x, SIGN_PAPER_LITERAL)
            assert np.array_equal(got.view(np.uint32), y.view(np.uint32)), (x, got, y)
            corr = -y if len(x) % 2 else y
            assert np.array_equal(oracle_mod.check_node(x, 0).view(np.uint32), corr.view(np.uint32))


def test_p5_check_node_brute_force_vs_observations(oracle_mod):
    """P5: the literal leave-one-out CN equals the Obs. 1/2 fast path exactly on 1000
    random rows (degrees 2..32) that include exact zeros, -0.0 and ties."""
    rng = np.random.default_rng(5)
    for t in range(1000):
        d = int(rng.integers(2, 33))
        x = rng.choice(np.array([-2.0, -1.0, -0.5, 0.0, -0.0, 0.5, 1.0, 2.0], np.float32), size=d)
        if t % 2:
            x = (rng.standard_normal(d) * 3).astype(np.float32)
            x[rng.integers(d)] = 0.0
        for literal in (0, 1):
            got = oracle_mod.check_node(x, SIGN_PAPER_LITERAL if literal else 0)
            exp = _obs12_fast_path(x, literal)
            assert np.array_equal(got.view(np.uint32) & 0x7FFFFFFF, exp.view(np.uint32) & 0x7FFFFFFF)
            # signs agree except on exact zeros (sign of a zero magnitude is immaterial, A12)
            nz = exp != 0
            assert np.array_equal(np.signbit(got[nz]), np.signbit(exp[nz]))


# ---------------------------------------------------------------- P6 ----------------------
@pytest.mark.parametrize("d", [3, 4, 5, 6])
def test_p6_spc_is_wagner_ml(oracle_mod, d):
    """P6: on a single parity check the decision after one iteration is the ML (Wagner) codeword:
    flip the least reliable bit when the parity fails.  Discriminates reading A1 for odd d."""
    code = codes.spc(d)
    rng = np.random.default_rng(100 + d)
    r = rng.standard_normal((300, d)).astype(np.float32)
    V = all_vectors(d)
    C = V[V.sum(axis=1) % 2 == 0]
    ml = C[np.argmax((2.0 * C - 1.0) @ r.T.astype(np.float64), axis=0)]
    bits, iters, conv, _ = oracle_mod.decode(code.oracle_h(), r, 1)
    assert np.array_equal(bits, ml)
    assert np.all(conv == 1)
    assert np.all(iters <= 1)
    if d % 2:
        bl, il, cl, _ = oracle_mod.decode(code.oracle_h(), r, 1, flags=SIGN_PAPER_LITERAL)
        assert not np.array_equal(bl, ml)  # the literal rule decodes a coset (A1)


# ---------------------------------------------------------------- P7 ----------------------
@pytest.mark.parametrize("seed", range(12))
def test_p7_tree_max_marginals(oracle_mod, seed):
    """P7: on a cycle-free Tanner graph, min-sum run past the diameter gives exact max-marginals
    s_j = (max_{c in C, c_j=1} sum (2c-1) r - max_{c in C, c_j=0} sum (2c-1) r) / 2."""
    code = codes.random_tree(int(3 + seed % 4), seed)
    H = code.dense()
    n = code.n
    assert n <= 16
    C = kernel_by_enumeration(H)
    rng = np.random.default_rng(seed)
    r = rng.standard_normal((20, n)).astype(np.float32)
    metric = (2.0 * C - 1.0) @ r.T.astype(np.float64)  # [codewords, frames]
    exp = np.empty((20, n))
    for j in range(n):
        exp[:, j] = (metric[C[:, j] == 1].max(axis=0) - metric[C[:, j] == 0].max(axis=0)) / 2
    L = 2 * code.m + 2
    _, _, _, p64 = oracle_mod.decode(code.oracle_h(), r, L, flags=NO_EARLY_STOP, precision="f64")
    assert np.allclose(p64, exp, rtol=0, atol=1e-9)
    _, _, _, p32 = oracle_mod.decode(code.oracle_h(), r, L, flags=NO_EARLY_STOP)
    assert np.allclose(p32, exp, rtol=1e-5, atol=1e-5)
    # the literal rule fails the closed form whenever the tree has an odd-degree row
    if any(len(rw) % 2 for rw in code.rows):
        _, _, _, pl = oracle_mod.decode(code.oracle_h(), r, L, flags=NO_EARLY_STOP | SIGN_PAPER_LITERAL,
                                        precision="f64")
        assert not np.allclose(pl, exp, atol=1e-6)


# ---------------------------------------------------------------- P8-P10 ------------------
def _random_frames(code, frames, ebn0, seed):
    return channel.bpsk_awgn(code.n, code.rate, ebn0, seed, 0, 0, frames).numpy()


def test_p8_power_of_two_scaling(oracle_mod):
    """P8: decode(2^k r) = same (b, k); s scales by 2^k bit-exactly."""
    code = codes.regular(24, 48, 3, 6, 7)
    r = _random_frames(code, 100, 1.5, 1)
    b0, i0, c0, p0 = oracle_mod.decode(code.oracle_h(), r, 30)
    for sc in (0.25, 4.0, 1024.0):
        b1, i1, c1, p1 = oracle_mod.decode(code.oracle_h(), (r * np.float32(sc)).astype(np.float32), 30)
        assert np.array_equal(b0, b1) and np.array_equal(i0, i1) and np.array_equal(c0, c1)
        assert np.array_equal(p1, (p0 * np.float32(sc)).astype(np.float32))


def _codeword_symmetry_case(oracle_mod, code, r, L, flags):
    C = kernel_by_enumeration(code.dense())
    b0, i0, c0, p0 = oracle_mod.decode(code.oracle_h(), r, L, flags=flags)
    for c in C[1:6]:
        t = (1.0 - 2.0 * c).astype(np.float32)
        b1, i1, c1, p1 = oracle_mod.decode(code.oracle_h(), r * t, L, flags=flags)
        # exact zeros (cancellations such as a + (-a)) slice to 0 under both signs: the law
        # holds on frames whose soft output has no exact zero (the generic case)
        ok = np.all(p0 != 0, axis=1) & np.all(p1 != 0, axis=1)
        assert ok.mean() >= 0.75
        assert np.array_equal(b1[ok], (b0 ^ c[None, :])[ok])
        assert np.array_equal(i1[ok], i0[ok]) and np.array_equal(c1[ok], c0[ok])
        assert np.array_equal(p1[ok], (p0 * t)[ok])


@pytest.mark.parametrize("flags", [0, SIGN_PAPER_LITERAL, NO_EARLY_STOP])
def test_p9_codeword_symmetry(oracle_mod, flags):
    """P9: for c in ker H, decode(r * (-1)^c) = (b xor c, same k, s * (-1)^c), bit-exactly
    (channel symmetry of min-sum; holds under both sign rules)."""
    code = load_paper_h()
    r = _random_frames(code, 60, 1.0, 2)
    _codeword_symmetry_case(oracle_mod, code, r, 20, flags)
    odd = codes.random_small(6, 14, 3, dmin=3, dmax=5)  # odd and even rows; nonzero kernel
    r2 = (np.random.default_rng(9).standard_normal((60, odd.n)) - 0.6).astype(np.float32)
    _codeword_symmetry_case(oracle_mod, odd, r2, 20, flags)


def test_p10_negation_symmetry_even_rows(oracle_mod):
    """P10: all rows even => all-ones is a codeword => decode(-r) = (not b, same k, -s)."""
    code = load_paper_h()
    r = _random_frames(code, 100, 0.5, 3)
    b0, i0, c0, p0 = oracle_mod.decode(code.oracle_h(), r, 20)
    b1, i1, c1, p1 = oracle_mod.decode(code.oracle_h(), -r, 20)
    assert np.array_equal(b1, 1 - b0) and np.array_equal(i1, i0) and np.array_equal(p1, -p0)


# ---------------------------------------------------------------- P11, P12 ----------------
def test_p11_zero_iterations(oracle_mod):
    """P11: L = 0 returns (syndrome(slice r) == 0, 0, slice r, r)."""
    code = codes.regular(12, 24, 3, 6, 11)
    r = _random_frames(code, 50, 3.0, 4)
    H = code.dense()
    for flags in (0, NO_EARLY_STOP):
        bits, iters, conv, post = oracle_mod.decode(code.oracle_h(), r, 0, flags=flags)
        hard = (r > 0).astype(np.uint8)
        assert np.array_equal(bits, hard) and np.all(iters == 0) and np.array_equal(post, r)
        assert np.array_equal(conv, (((hard.astype(np.int64) @ H.T) % 2).sum(axis=1) == 0).astype(np.uint8))


def test_bn_summation_order_reading_a14(oracle_mod):
    """Reading A14 (golden bn_order_a14.txt): ascending-row accumulation from +0.0, then + r."""
    spec = {}
    with open(os.path.join(GOLDEN, "bn_order_a14.txt")) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                k, v = line.split(":", 1)
                spec[k] = v
    rows = [[int(t) for t in grp.split()] for grp in spec["rows"].split("|")]
    code = codes.from_rows(rows, int(spec["n"]))
    r = np.array([float(t) for t in spec["r"].split()], np.float32)[None]
    _, _, _, post = oracle_mod.decode(code.oracle_h(), r, int(spec["L"]), flags=NO_EARLY_STOP)
    assert post[0, 0] == np.float32(float(spec["s0"]))


def test_p11_slice_of_zero_is_logical_zero(oracle_mod):
    """Eq. slice: b = 1 iff s > 0, so s = +0.0 and -0.0 both slice to 0.  An all-zero
    r therefore slices to the all-zero codeword and stops at k = 0."""
    code = codes.paper_5x10()
    r = np.array([[0.0, -0.0, 1.0, -1.0, 0.0, 0.0, 2.0, 0.0, -0.0, 0.5]], np.float32)
    bits, iters, conv, post = oracle_mod.decode(code.oracle_h(), r, 0)
    assert list(bits[0]) == [0, 0, 1, 0, 0, 0, 1, 0, 0, 1]
    z = np.zeros((1, 10), np.float32)
    bits, iters, conv, post = oracle_mod.decode(code.oracle_h(), z, 5)
    assert iters[0] == 0 and conv[0] == 1 and not bits.any()


@pytest.mark.parametrize("flags", [0, SIGN_PAPER_LITERAL, NO_EARLY_STOP])
def test_p12_termination_and_independence(oracle_mod, flags):
    """P12: converged => H.b = 0; not converged => k = L; each frame's outcome is
    independent of the batch it is decoded in and of the number of threads."""
    code = codes.random_small(15, 30, 21, dmin=2, dmax=7)
    H = code.dense()
    rng = np.random.default_rng(2)
    r = (rng.standard_normal((200, code.n)) * 1.2 - 0.8).astype(np.float32)
    L = 15
    bits, iters, conv, post = oracle_mod.decode(code.oracle_h(), r, L, flags=flags, threads=4)
    syn = ((bits.astype(np.int64) @ H.T) % 2).sum(axis=1)
    assert np.all(syn[conv == 1] == 0)
    if flags & NO_EARLY_STOP:
        assert np.all(iters == L)
        assert np.array_equal(conv == 1, syn == 0)
    else:
        assert np.all(iters[conv == 0] == L)
        assert np.all(iters[conv == 1] <= L)
    for f in (0, 17, 199):
        b1, i1, c1, p1 = oracle_mod.decode(code.oracle_h(), r[f:f + 1], L, flags=flags, threads=1)
        assert np.array_equal(b1[0], bits[f]) and i1[0] == iters[f] and c1[0] == conv[f]
        assert np.array_equal(p1[0], post[f])


def test_check_every_semantics(oracle_mod):
    """checkEvery = T ("Termination was checked for every 6 iterations"): the T-run
    stops at the first k in {0, T, 2T, ...} or k = L at which the (check-independent) trajectory's
    hard decision is a codeword, with the same bits and soft vector as that trajectory at k."""
    code = codes.regular(60, 120, 3, 6, 21)
    r = _random_frames(code, 60, 1.8, 31)
    L, T = 20, 6
    H = code.dense()
    traj = {}
    for k in range(L + 1):
        b, _, _, p = oracle_mod.decode(code.oracle_h(), r, k, flags=NO_EARLY_STOP)
        traj[k] = (b, p, ((b.astype(np.int64) @ H.T) % 2).sum(axis=1) == 0)
    bits, iters, conv, post = oracle_mod.decode(code.oracle_h(), r, L, check_every=T)
    checks = [k for k in range(L + 1) if k % T == 0 or k == L]
    for f in range(len(r)):
        stop = next((k for k in checks if traj[k][2][f]), None)
        if stop is None:
            assert iters[f] == L and conv[f] == 0
            stop = L
        else:
            assert iters[f] == stop and conv[f] == 1
        assert np.array_equal(bits[f], traj[stop][0][f]) and np.array_equal(post[f], traj[stop][1][f])
    assert np.any(iters % T != 0)  # some frames run to L = 20 (not a multiple of 6) or stop at 0 / 6 / 12 / 18
    _, i1, c1, _ = oracle_mod.decode(code.oracle_h(), r, L, check_every=1)
    assert np.all(iters[c1 == 1] >= i1[c1 == 1])  # checking less often never stops earlier


# ---------------------------------------------------------------- P13 ---------------------
def test_p13_coding_gain(oracle_mod):
    """P13: past the waterfall the decoded BER is below the raw BER (C2-shaped code)."""
    code = codes.regular(504, 1008, 3, 6, 1008)
    r = _random_frames(code, 200, 3.0, 5)
    bits, iters, conv, post = oracle_mod.decode(code.oracle_h(), r, 50)
    raw = np.count_nonzero(r > 0)
    dec = int(bits.sum())
    assert raw > 0 and dec < raw
    assert conv.mean() > 0.9


# ---------------------------------------------------------------- stats / errors ----------
def test_stats_plain_definitions(oracle_mod):
    """The counters are plain counts over the outputs (hand-computed case)."""
    llr = np.array([[-1, 0.5, -2], [1, 1, -1]], np.float32)
    bits = np.array([[0, 1, 0], [0, 0, 0]], np.uint8)
    iters = np.array([3, 0], np.int32)
    conv = np.array([1, 1], np.uint8)
    post = np.array([[-1, 0.00005, -3], [-2, -2, -2]], np.float32)
    st = oracle_mod.stats(llr, bits, iters, conv, post)
    assert list(st) == [2, 1, 1, 1, 3, 2, 1, 3]


def test_oracle_rejects_bad_h(oracle_mod):
    with pytest.raises(ValueError, match="degree"):
        oracle_mod.decode(np.array([[1, 0, 0], [0, 1, 1]], np.uint8), np.zeros((1, 3), np.float32), 5)
    with pytest.raises(ValueError, match="duplicate"):
        oracle_mod.decode((np.array([0, 0, 0], np.int32), np.array([1, 1, 2], np.int32), 1, 3),
                          np.zeros((1, 3), np.float32), 5)
    with pytest.raises(ValueError, match="range"):
        oracle_mod.decode((np.array([0, 0], np.int32), np.array([1, 3], np.int32), 1, 3),
                          np.zeros((1, 3), np.float32), 5)


def test_fp64_shadow_agrees_mostly(oracle_mod):
    """The fp64 shadow (drift report only) agrees with fp32 on hard decisions for nearly all frames."""
    code = codes.regular(60, 120, 3, 6, 13)
    r = _random_frames(code, 200, 2.0, 6)
    b32, i32, _, p32 = oracle_mod.decode(code.oracle_h(), r, 30)
    b64, i64, _, p64 = oracle_mod.decode(code.oracle_h(), r, 30, precision="f64")
    same = np.all(b32 == b64, axis=1) & (i32 == i64)
    assert same.mean() > 0.95
