"""CPU: host-side logic -- grid/blocking index arithmetic against the
reference, the multi-GPU partition and the one scalar reduction (gloo,
world_size 2)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2103_01380_b200 import distributed as D
from paper_2103_01380_b200 import spid
from paper_2103_01380_b200.configs import CONFIGS, weak_range


def test_row_indices_vs_reference(ref):
    for dims, strides, per in [([18], [1], None), ([24], [5], None), ([20, 20], [2, 2], [1, 1]),
                               ([9, 7], [2, 3], None), ([9, 7], [4, 4], [0, 1]),
                               ([16, 16, 16], [2, 3, 2], [1, 1, 1]), ([12, 10, 8], [3, 3, 3], None),
                               ([5, 5, 5], [5, 5, 5], None)]:
        assert np.array_equal(spid.row_indices(dims, strides, per), ref.row_indices(dims, strides, per))


def test_row_indices_errors():
    with pytest.raises(spid.SpidError) as e:
        spid.row_indices([10], [0])
    assert e.value.name == "BadSubsampleSpec"
    with pytest.raises(spid.SpidError) as e:
        spid.row_indices([1], [1])
    assert e.value.name == "BadGridGeom"


def test_make_block_domains_order():
    # proj/src/blocking.cpp:64-81: blocks axis-0 fastest, rows axis-0 fastest,
    # remainder to the last block (:16-27)
    doms = spid.make_block_domains([4, 4], [2, 2])
    assert [list(d) for d in doms] == [[0, 1, 4, 5], [2, 3, 6, 7], [8, 9, 12, 13], [10, 11, 14, 15]]
    doms = spid.make_block_domains([5], [2])
    assert [list(d) for d in doms] == [[0, 1], [2, 3, 4]]
    doms = spid.make_block_domains([32, 32, 32], [2, 2, 2])
    assert len(doms) == 8 and all(len(d) == 4096 for d in doms)
    allrows = np.sort(np.concatenate(doms))
    assert np.array_equal(allrows, np.arange(32 ** 3))
    # block 1 starts at x=16 (axis 0 fastest)
    assert doms[1][0] == 16 and doms[2][0] == 32 * 16


def test_field_block_layout_matches_blocking():
    """The device generator's subdomain s holds, in row order, the points of
    make_block_domains block s (checked by index arithmetic)."""
    N, b = 32, 16
    nb = N // b
    doms = spid.make_block_domains([N, N, N], [nb, nb, nb])
    for s in range(nb ** 3):
        bx, by, bz = s % nb, (s // nb) % nb, s // (nb * nb)
        p = np.arange(b ** 3)
        ix, iy, iz = bx * b + p % b, by * b + (p // b) % b, bz * b + p // (b * b)
        assert np.array_equal(ix + N * iy + N * N * iz, doms[s])


def test_partitions():
    assert D.contiguous_range(512, 3, 8) == (192, 256)
    cover = sorted(i for r in range(8) for i in range(*D.contiguous_range(216, r, 8)))
    assert cover == list(range(216))
    rr = [D.round_robin(216, r, 8) for r in range(8)]
    assert sorted(sum(rr, [])) == list(range(216)) and all(len(x) == 27 for x in rr)
    big, first, cnt = weak_range(CONFIGS["cfg3"], 7, 8)
    assert big.name == "cfg5" and first == 448 and cnt == 64


def test_config_shapes():
    c1, c2, c3, c4, c5 = (CONFIGS[f"cfg{i}"] for i in range(1, 6))
    assert (c1.m, c1.n, c1.ell, c1.subdomains) == (16384, 100, 20, 8)
    assert (c2.m, c2.n, c2.ell, c2.subdomains) == (163840, 512, 30, 64)
    assert (c3.m, c3.n, c3.ell) == (163840, 256, 48)
    assert (c4.subdomains, c4.ell) == (216, 80)
    assert (c5.subdomains, c5.raw_bytes()) == (512, 171798691840)


def test_report_single_process():
    s = D.local_sums([1.0, 3.0], [100.0, 300.0], [2, 2], m=10, n=5)
    r = D.reduce_report(s)
    assert r.stored_entries == 2 * 2 * 15 and r.raw_entries == 100
    assert abs(r.cf - 100 / 60) < 1e-15
    assert abs(r.rel_frob_error - 0.1) < 1e-15


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = D.contiguous_range(6, rank, world)
        err2 = [float(i + 1) for i in range(lo, hi)]
        ref2 = [100.0 * (i + 1) for i in range(lo, hi)]
        ranks = [3] * (hi - lo)
        rep = D.reduce_report(D.local_sums(err2, ref2, ranks, m=40, n=8))
        allr = D.gather_ranks(torch.tensor(ranks, dtype=torch.int64))
        out[rank] = (rep.cf, rep.rel_frob_error, rep.stored_entries, len(allr))
    finally:
        dist.destroy_process_group()


def test_report_allreduce_gloo_world2():
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    expect_cf = (40 * 8 * 6) / (6 * 3 * 48)
    expect_err = np.sqrt(sum(range(1, 7)) / (100 * sum(range(1, 7))))
    for r in range(2):
        cf, err, stored, nr = out[r]
        assert abs(cf - expect_cf) < 1e-12 and abs(err - expect_err) < 1e-15
        assert stored == 6 * 3 * 48 and nr == 6
