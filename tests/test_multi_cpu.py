"""World-size-2 CPU (gloo) tests of the sample-sharded multi-GPU host logic: contiguous shards
(comm.shard_range, SPEC.md:648's contiguous chunks), per-rank partial activation records,
sum-allreduce, replicated update.  Each rank computes its shard's partial record with the CPU
oracle (standing in for the per-GPU kernels; the NCCL path is exercised on GPU boxes), and the
allreduced result must equal the single-process result: counts exactly, fp64 sums to rtol
1e-12 (only the combine order differs)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import oracle as O
    from paper_1109_0778_b200.comm import shard_range
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = {}
    # ---- k-means: 3 free-running iterations on sharded samples --------------------------------
    n, d, k = 20000, 16, 8
    lo, hi = shard_range(n, rank, world)
    x = O.rng_units(1, lo * d, (hi - lo) * d).reshape(hi - lo, d)   # generated in place (skip-ahead)
    mu = O.rng_units(1, 0, k * d).reshape(k, d)                     # first k rows, replicated
    hist = []
    for _ in range(3):
        _, c, s = O.kmeans_step(x, k, mu)
        tc, ts = torch.from_numpy(c.copy()), torch.from_numpy(s.copy())
        dist.all_reduce(tc)
        dist.all_reduce(ts)
        mu = O.kmeans_update(tc.numpy(), ts.numpy())
        hist.append((tc.numpy().copy(), ts.numpy().copy()))
    out["kmeans"] = hist
    # ---- GroupBy ------------------------------------------------------------------------------
    nk, K = 100_001, 64
    lo, hi = shard_range(nk, rank, world)
    keys = O.rng_ints(1, lo, hi - lo, K)
    tc = torch.from_numpy(O.groupby_count(keys, K))
    dist.all_reduce(tc)
    out["groupby"] = tc.numpy()
    # ---- logistic regression: 3 BGD steps -----------------------------------------------------
    nl, dl = 30000, 8
    lo, hi = shard_range(nl, rank, world)
    xl = O.rng_units(2, lo * dl, (hi - lo) * dl).reshape(hi - lo, dl)
    yl = O.rng_ints(2, nl * dl + lo, hi - lo, 2)
    th = np.zeros(dl)
    for _ in range(3):
        g = torch.from_numpy(O.logreg_grad(xl, yl, th))
        dist.all_reduce(g)
        th = th - (1.0 / nl) * g.numpy()
    out["logreg"] = th
    # ---- GDA ------------------------------------------------------------------------------------
    ng, dg = 10000, 4
    lo, hi = shard_range(ng, rank, world)
    xg = O.rng_units(3, lo * dg, (hi - lo) * dg).reshape(hi - lo, dg)
    yg = O.rng_ints(3, ng * dg + lo, hi - lo, 2)
    n1, s0, s1 = O.gda_pass1(xg, yg)
    t = torch.from_numpy(np.concatenate([[float(n1)], s0, s1]))
    dist.all_reduce(t)
    n1 = int(t[0].item())
    mu0, mu1 = t[1:1 + dg].numpy() / float(ng - n1), t[1 + dg:].numpy() / float(n1)
    S = torch.from_numpy(O.gda_pass2(xg, yg, mu0, mu1))
    dist.all_reduce(S)
    out["gda"] = (n1, mu0, mu1, S.numpy())
    # ---- GDA, single pass per rank pooled (the sharded dlx path: gda_combine_ranks_kernel) -----
    nl1, ls0, ls1 = O.gda_pass1(xg, yg)
    nloc = hi - lo
    lm0, lm1 = ls0 / float(nloc - nl1), ls1 / float(nl1)
    S_r = torch.from_numpy(O.gda_pass2(xg, yg, lm0, lm1))          # scatter around the rank's means
    table = torch.zeros((world, 2 + 2 * dg), dtype=torch.float64)
    table[rank] = torch.from_numpy(np.concatenate([[float(nloc - nl1), float(nl1)], lm0, lm1]))
    dist.all_reduce(table)
    dist.all_reduce(S_r)
    t = table.numpy()
    nc = t[:, :2].sum(axis=0)
    mus = [sum(t[r, c] * t[r, 2 + c * dg:2 + (c + 1) * dg] for r in range(world)) / nc[c] for c in range(2)]
    Sp = S_r.numpy().copy()
    for r in range(world):
        for c in range(2):
            dv = t[r, 2 + c * dg:2 + (c + 1) * dg] - mus[c]
            Sp += t[r, c] * np.outer(dv, dv)
    out["gda_pooled"] = (int(nc[1]), mus[0], mus[1], Sp)
    if rank == 0:
        q.put(out)
    dist.barrier()
    dist.destroy_process_group()


def test_shard_ranges_partition():
    from paper_1109_0778_b200.comm import shard_range
    for n in (0, 1, 7, 100, 16_777_216):
        for w in (1, 2, 3, 8):
            parts = [shard_range(n, r, w) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(w - 1))


def test_world2_gloo_matches_single_process():
    import oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-process references
    x, mu = O.kmeans_inputs(20000, 16, 8)
    for it, (c, _, _, s, _) in enumerate(O.kmeans_run(x, 8, 3, mu)):
        assert np.array_equal(out["kmeans"][it][0], c)
        np.testing.assert_allclose(out["kmeans"][it][1], s, rtol=1e-12)
    keys = O.rng_ints(1, 0, 100_001, 64)
    assert np.array_equal(out["groupby"], O.groupby_count(keys, 64))
    xl = O.rng_units(2, 0, 30000 * 8).reshape(30000, 8)
    yl = O.rng_ints(2, 30000 * 8, 30000, 2)
    th = np.zeros(8)
    for _ in range(3):
        th = th - (1.0 / 30000) * O.logreg_grad(xl, yl, th)
    np.testing.assert_allclose(out["logreg"], th, rtol=1e-12)
    xg = O.rng_units(3, 0, 10000 * 4).reshape(10000, 4)
    yg = O.rng_ints(3, 40000, 10000, 2)
    n1, s0, s1 = O.gda_pass1(xg, yg)
    mu0, mu1 = s0 / float(10000 - n1), s1 / float(n1)
    S = O.gda_pass2(xg, yg, mu0, mu1)
    assert out["gda"][0] == n1
    np.testing.assert_allclose(out["gda"][1], mu0, rtol=1e-12)
    np.testing.assert_allclose(out["gda"][3], S, rtol=1e-11)
    # pooled-scatter identity (the sharded single-pass path) against the same references
    assert out["gda_pooled"][0] == n1
    np.testing.assert_allclose(out["gda_pooled"][1], mu0, rtol=1e-12)
    np.testing.assert_allclose(out["gda_pooled"][2], mu1, rtol=1e-12)
    np.testing.assert_allclose(out["gda_pooled"][3], S, rtol=1e-11)
