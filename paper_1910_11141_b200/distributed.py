"""Multi-GPU: chains shard across ranks; NCCL only for diagnostics and the sample gather.

Lane isolation (reference runtime.py:96-104, §4) means chain b's
result depends only on (q0[b], key[b]): the chain batch is split into
contiguous per-rank ranges and every rank runs its own VM with no data-path
collective. The only exchanges are

* `all_reduce` (sum) of O(d) sufficient statistics for cross-chain
  diagnostics — chain-mean sums, sums of squared chain means, within-chain
  variance sums, lagged autocovariance sums — from which split-R-hat and
  ESS follow on every rank (the reference has no diagnostics; these are
  restated from the standard definitions and checked against a numpy
  single-process computation in tests/test_distributed.py);
* an optional `all_gather` of thinned samples.

Works with any torch.distributed backend: NCCL over NVLink on the GPU box,
gloo in the CPU tests.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def shard_range(rank: int, world: int, z: int) -> tuple[int, int]:
    """Contiguous chain ids [lo, hi) owned by `rank` (balanced to within one chain)."""
    base, extra = divmod(z, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def chain_keys(lo: int, hi: int) -> np.ndarray:
    """Unique per-chain keys for chain ids [lo, hi): key depends only on the global chain id,
    so any sharding gives every chain the same stream."""
    ids = np.arange(lo, hi, dtype=np.int64)
    return (ids * 2654435761 + 12345) % (2**31 - 1)


@dataclass
class Diagnostics:
    rhat: np.ndarray       # split-R-hat per dimension
    ess: np.ndarray        # effective sample size per dimension (all chains)
    mean: np.ndarray       # posterior mean estimate per dimension
    var: np.ndarray        # posterior variance estimate per dimension
    chains: int
    draws: int


def _stats(chains, max_lag: int):
    """Per-shard sufficient statistics of split chains (torch tensor [c, n, d], float64).

    Each chain is split in halves (split-R-hat). Returns a flat float64 tensor:
    [count, sum_means(d), sum_means_sq(d), sum_within_var(d), sum_x(d), sum_x2(d),
     autocov sums (max_lag+1, d)].
    """
    import torch

    c, n, d = chains.shape
    h = n // 2
    halves = torch.cat([chains[:, :h], chains[:, n - h:]], dim=0)  # [2c, h, d]
    means = halves.mean(dim=1)
    var = halves.var(dim=1, unbiased=True)
    centered = halves - means[:, None, :]
    acov = []
    for lag in range(max_lag + 1):  # biased autocovariance of each half-chain (divided by h)
        prod = (centered[:, : h - lag] * centered[:, lag:]).sum(dim=1) / h  # [2c, d]
        acov.append(prod.sum(dim=0))
    parts = [torch.tensor([2.0 * c], dtype=torch.float64, device=chains.device), means.sum(0),
             (means ** 2).sum(0), var.sum(0), chains.sum((0, 1)), (chains ** 2).sum((0, 1)),
             torch.stack(acov).reshape(-1)]
    return torch.cat([p.reshape(-1).to(torch.float64) for p in parts])


def diagnostics(chains, *, group=None, max_lag: int = 50) -> Diagnostics:
    """Split-R-hat and ESS over all ranks' chains.

    `chains`: this rank's samples as a torch tensor [chains, draws, dim]
    (device tensor on the GPU box). One all_reduce of O((max_lag+6)·d) doubles.
    """
    import torch
    import torch.distributed as dist

    c, n, d = chains.shape
    max_lag = min(max_lag, n // 2 - 1)
    s = _stats(chains.to(torch.float64), max_lag)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(s, group=group)
    s = s.cpu().numpy()
    m2 = s[0]                      # number of half-chains
    o = 1
    sum_m, sum_m2, sum_w = s[o:o + d], s[o + d:o + 2 * d], s[o + 2 * d:o + 3 * d]
    sum_x, sum_x2 = s[o + 3 * d:o + 4 * d], s[o + 4 * d:o + 5 * d]
    acov = s[o + 5 * d:].reshape(max_lag + 1, d)
    h = n // 2
    mean_of_means = sum_m / m2
    b_over_h = (sum_m2 - m2 * mean_of_means ** 2) / (m2 - 1)   # between-chain variance / h
    w = sum_w / m2                                              # within-chain variance
    var_plus = (h - 1) / h * w + b_over_h
    rhat = np.sqrt(var_plus / w)
    chains_total = m2 / 2
    draws_total = chains_total * n
    mean = sum_x / draws_total
    var = sum_x2 / draws_total - mean ** 2
    # ESS (Stan / Geyer): rho_t = 1 - (W - mean half-chain autocovariance_t) / var_plus, then
    # the initial positive sequence of pair sums P_k = rho_2k + rho_2k+1 (k = 0, 1, ...), made
    # monotone, tau = -1 + 2 sum P_k; antithetic chains (rho_1 < 0) may give ESS > draws
    rho = 1.0 - (w[None, :] - acov / m2) / np.maximum(var_plus[None, :], 1e-300)
    ess = np.empty(d)
    for j in range(d):
        total, prev = 0.0, np.inf
        for k in range(0, max_lag, 2):
            pair = rho[k, j] + rho[k + 1, j]
            if pair < 0:
                break
            prev = min(prev, pair)
            total += prev
        tau = max(-1.0 + 2.0 * total, 1.0 / np.log10(max(draws_total, 10.0)))
        ess[j] = draws_total / tau
    return Diagnostics(rhat=rhat, ess=ess, mean=mean, var=var, chains=int(chains_total), draws=n)


def gather_samples(chains, *, thin: int = 1, group=None):
    """All-gather thinned samples of every rank (torch tensors, equal shard sizes)."""
    import torch
    import torch.distributed as dist

    local = chains[:, ::thin].contiguous()
    if not (dist.is_available() and dist.is_initialized()):
        return local
    out = [torch.empty_like(local) for _ in range(dist.get_world_size(group))]
    dist.all_gather(out, local, group=group)
    return torch.cat(out, dim=0)


def run_shard(compiled, q0, *, z_total: int, rank: int, world: int, depth: int, device: int | None = None,
              **run_kw):
    """This rank's contiguous chain range [lo, hi) of a z_total-chain batch on its own GPU:
    q0 rows lo..hi-1 (or q0(lo, hi) when q0 is callable) and the global-id keys; no
    collective. Returns (outputs [hi-lo, ...], lo, hi, trace). Any sharding gives every
    chain the bytes the single-rank run gives it (lane isolation)."""
    from . import pc_vm

    lo, hi = shard_range(rank, world, z_total)
    q = q0(lo, hi) if callable(q0) else q0[lo:hi]
    out, tr = pc_vm.run(compiled, [q, chain_keys(lo, hi)], depth=depth, device=device, **run_kw)
    return out, lo, hi, tr
