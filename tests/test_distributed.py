"""Multi-rank path on CPU: world_size-2 gloo processes (the GPU box runs NCCL).

Chains shard with no data-path collective; the only exchange is the
diagnostics all_reduce, whose result must equal the single-process
computation over the concatenated chains.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1910_11141_b200 import distributed as D


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _synthetic_chains(z=64, n=200, d=3, seed=0, phi=0.6):
    rng = np.random.default_rng(seed)
    x = np.zeros((z, n, d))
    x[:, 0] = rng.normal(size=(z, d))
    for t in range(1, n):  # AR(1) chains: known autocorrelation phi^lag, unit variance
        x[:, t] = phi * x[:, t - 1] + np.sqrt(1 - phi * phi) * rng.normal(size=(z, d))
    return x


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x = _synthetic_chains()
    lo, hi = D.shard_range(rank, world, x.shape[0])
    diag = D.diagnostics(torch.from_numpy(x[lo:hi]))
    gathered = D.gather_samples(torch.from_numpy(x[lo:hi]), thin=10)
    q.put((rank, diag.rhat, diag.ess, diag.mean, gathered.shape))
    dist.destroy_process_group()


def test_shard_ranges_cover_all_chains():
    for z in (1, 7, 64, 65536 + 3):
        for world in (1, 2, 3, 8):
            spans = [D.shard_range(r, world, z) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == z
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1


def test_keys_are_shard_invariant():
    full = D.chain_keys(0, 1000)
    parts = np.concatenate([D.chain_keys(*D.shard_range(r, 3, 1000)) for r in range(3)])
    assert np.array_equal(full, parts) and len(np.unique(full)) == 1000


def test_two_rank_diagnostics_equal_single_process():
    x = _synthetic_chains()
    single = D.diagnostics(torch.from_numpy(x))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, rhat, ess, mean, gshape in res:
        np.testing.assert_allclose(rhat, single.rhat, rtol=1e-12)
        np.testing.assert_allclose(ess, single.ess, rtol=1e-12)
        np.testing.assert_allclose(mean, single.mean, rtol=1e-12)
        assert tuple(gshape) == (64, 20, 3)


def test_diagnostics_behave():
    x = _synthetic_chains(z=32, n=400)
    diag = D.diagnostics(torch.from_numpy(x))
    assert np.all(np.abs(diag.rhat - 1) < 0.05)
    # AR(1) with phi=0.6: integrated autocorrelation time (1+phi)/(1-phi) = 4
    assert np.all((diag.ess > 32 * 400 / 6) & (diag.ess < 32 * 400 / 2.5))
    bad = x.copy()
    bad[:16] += 3.0  # chains stuck in two modes
    assert np.all(D.diagnostics(torch.from_numpy(bad)).rhat > 1.5)


@pytest.mark.parametrize("phi", [0.9, 0.6, 0.0, -0.5])
def test_ess_matches_ar1_theory(phi):
    """Stan/Geyer ESS against the AR(1) closed form N (1 - phi) / (1 + phi): within 12 %,
    including antithetic chains (phi < 0), whose ESS exceeds the number of draws."""
    z, n = 64, 2000
    x = _synthetic_chains(z=z, n=n, d=2, seed=7, phi=phi)
    ess = D.diagnostics(torch.from_numpy(x), max_lag=200).ess
    want = z * n * (1 - phi) / (1 + phi)
    assert np.all(np.abs(ess / want - 1) < 0.12), (phi, ess, want)
    if phi < 0:
        assert np.all(ess > z * n)
