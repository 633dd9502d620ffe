"""Chain sharding on the GPU box: two ranks (gloo for the host exchange) each run their
shard of one batch through the VM on the device they were given (both on GPU 0 here, the
only GPU of the lease; the ranks never wait on each other's kernels). The concatenated
shards must equal the single-rank run byte for byte, and the all-reduced diagnostics must
equal the single-process ones (reference runtime.py:96-104: lanes are isolated)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

# (program, chains): NUTS-lite on the 5-d gaussian, and BASELINE config 4 (logistic
# regression on the 100k x 100 design, its sx streamed by every warp) on a small batch
CASES = [("gauss5", 3000), ("config4", 48)]


def _program(name="gauss5"):
    from paper_1910_11141_b200 import prebuilt

    if name == "config4":
        kw = dict(prebuilt.CONFIG4)
        return prebuilt.lr_nuts(kw.pop("n"), kw.pop("d"), kw.pop("seed"), **kw)
    kw = dict(prebuilt.TEST_NUTS[2])  # d = 5, T = 4, depth 8
    return prebuilt.nuts(kw.pop("dim"), kw.pop("rho"), **kw)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank, world, port, q, name, Z):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1910_11141_b200 import distributed as D

    cfg, t, cp = _program(name)
    out, lo, hi, tr = D.run_shard(cp, np.zeros((Z, t.dim)), z_total=Z, rank=rank, world=world,
                                  depth=cfg.min_stack_depth, device=0, engine="warp", codegen="cached",
                                  exact_logpdf=False, schedule="priority")
    chains = torch.from_numpy(out.reshape(hi - lo, cfg.iterations, t.dim).copy())
    diag = D.diagnostics(chains)
    q.put((rank, lo, hi, out, diag.rhat, diag.ess))
    dist.destroy_process_group()


@pytest.mark.parametrize("name,Z", CASES)
def test_two_ranks_on_one_gpu_equal_the_single_rank_run(name, Z):
    from paper_1910_11141_b200 import distributed as D
    import paper_1910_11141_b200 as L

    cfg, t, cp = _program(name)
    single, _ = L.run(cp, [np.zeros((Z, t.dim)), D.chain_keys(0, Z)], depth=cfg.min_stack_depth,
                      engine="warp", codegen="cached", exact_logpdf=False, schedule="priority", device=0)
    ref = D.diagnostics(torch.from_numpy(single.reshape(Z, cfg.iterations, t.dim).copy()))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q, name, Z)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in procs], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    joined = np.concatenate([r[3] for r in res])
    assert res[0][1] == 0 and res[0][2] == res[1][1] and res[1][2] == Z
    assert joined.tobytes() == single.tobytes()
    for _, _, _, _, rhat, ess in res:
        np.testing.assert_allclose(rhat, ref.rhat, rtol=1e-12)
        np.testing.assert_allclose(ess, ref.ess, rtol=1e-12)


def test_machine_reports_its_device():
    import paper_1910_11141_b200 as L

    cfg, t, cp = _program()
    _, _, m = L.run(cp, [np.zeros((64, t.dim)), np.arange(64, dtype=np.int64)], depth=cfg.min_stack_depth,
                    engine="warp", codegen="cached", device=0, return_machine=True)
    assert m._h.device == 0
    from paper_1910_11141_b200 import _native

    with pytest.raises(_native.DeviceError):
        L.run(cp, [np.zeros((4, t.dim)), np.arange(4, dtype=np.int64)], depth=cfg.min_stack_depth,
              engine="warp", codegen="cached", device=_native.device_count() + 3)
