"""Input generators: structure of the H ensembles and determinism of the keyed channel (CPU)."""
import math

import numpy as np
import pytest
import torch

from gen import channel, codes


@pytest.mark.parametrize("m,n,dv,dc,seed", [(504, 1008, 3, 6, 1008), (2048, 4096, 3, 6, 4096), (12, 24, 3, 6, 1)])
def test_regular_ensemble(m, n, dv, dc, seed):
    c = codes.regular(m, n, dv, dc, seed)
    H = c.dense()
    assert H.shape == (m, n)
    assert np.all(H.sum(axis=1) == dc) and np.all(H.sum(axis=0) == dv)
    assert all(np.all(np.diff(r) > 0) for r in c.rows)  # ascending, no duplicates
    c2 = codes.regular(m, n, dv, dc, seed)
    assert all(np.array_equal(a, b) for a, b in zip(c.rows, c2.rows))


def test_bg1_dims_histograms():
    c = codes.bg1_dims()
    assert (c.m, c.n, c.nnz) == (17664, 26112, 121344)
    rd = np.bincount([len(r) for r in c.rows])
    assert rd[7] == 15360 and rd[6] == 2304
    _, cc = c.coo()
    cd = np.bincount(np.bincount(cc, minlength=c.n))
    assert cd[5] == 16896 and cd[4] == 9216
    assert all(np.all(np.diff(r) > 0) for r in c.rows)


def test_tree_is_cycle_free():
    for seed in range(10):
        c = codes.random_tree(6, seed)
        # a connected bipartite graph is a tree iff edges = nodes - 1
        assert c.nnz == c.m + c.n - 1


def test_channel_is_keyed_by_global_frame():
    """Sharding/chunking never changes a frame: any sub-range regenerates identically."""
    full = channel.bpsk_awgn(1008, 0.5, 2.0, 7, 3, 0, 100)
    part = channel.bpsk_awgn(1008, 0.5, 2.0, 7, 3, 37, 20)
    assert torch.equal(full[37:57], part)
    other = channel.bpsk_awgn(1008, 0.5, 2.0, 7, 4, 0, 10)
    assert not torch.equal(full[:10], other)


def test_channel_statistics():
    """Noise variance matches sigma^2 = 1/(2 R 10^(EbN0/10)) and the mean is -1."""
    r = channel.bpsk_awgn(1000, 0.5, 3.0, 1, 0, 0, 1000).double()
    sig = channel.sigma_for(3.0, 0.5)
    assert abs(r.mean().item() + 1.0) < 5 * sig / math.sqrt(r.numel())
    assert abs(r.var().item() / sig ** 2 - 1.0) < 0.01
    # raw BER ~ Q(1/sigma)
    q = 0.5 * math.erfc((1 / sig) / math.sqrt(2))
    ber = (r > 0).double().mean().item()
    assert abs(ber - q) < 4 * math.sqrt(q * (1 - q) / r.numel())


def test_codeword_modulation():
    c = torch.tensor([0, 1, 1, 0], dtype=torch.uint8)
    r = channel.bpsk_awgn(4, 0.5, 200.0, 1, 0, 0, 3, codeword=c)
    assert torch.equal((r > 0).to(torch.uint8), c[None].expand(3, 4))


def test_point_and_shard_ranges():
    pr = codes.point_ranges(1 << 20, 7)
    assert pr[0][0] == 0 and pr[-1][1] == 1 << 20
    assert all(a[1] == b[0] for a, b in zip(pr, pr[1:]))
    sh = [codes.shard_range(1000, r, 8) for r in range(8)]
    assert sh[0][0] == 0 and sh[-1][1] == 1000 and all(a[1] == b[0] for a, b in zip(sh, sh[1:]))
