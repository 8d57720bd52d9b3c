"""GPU tests of the peer-memory collective (csrc/peer.cu, comm.PeerComm): the per-rank partial
records are summed by one kernel that reads every rank's exchange buffer and folds the ranks in
ascending order, fused with the update that consumes the sum.

The pool has one GPU per box, so the world-size 2 / 4 / 8 tests run that many processes on the
same device (uneven shards: no size below divides by 4 or 8):
the exchange buffers are shared through CUDA IPC exactly as across NVSwitch peers (there the
loads travel over NVLink), and the flag protocol, slot alternation and epilogues are the same
code.  Parity: counts / GroupBy bit-exact, fp64 sums rtol 1e-9 against the single-process
oracle, and every rank's result bit-identical (the ordered fold)."""
import os
import socket

import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


N_KM, D_KM, K_KM, IT_KM = 50_003, 64, 16, 4
N_LR, D_LR, IT_LR = 30_001, 64, 3
N_GB, K_GB = 200_001, 65_536   # a 512 KiB int64 record
N_GD, D_GD = 50_001, 64


def _worker(rank, world, port, q):
    try:
        _work(rank, world, port, q)
    except BaseException:   # report to the parent instead of leaving it waiting on the queue
        import traceback
        q.put((rank, {"error": traceback.format_exc()}))
        raise


def _work(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_1109_0778_b200 import multiloops as ml
    from paper_1109_0778_b200.comm import PeerComm, shard_range
    from paper_1109_0778_b200.programs import KMeansProgram, LogRegProgram
    comm = PeerComm(rank, world, cap_bytes=2 << 20)   # two 1 MiB slots: the 512 KiB GroupBy record
    out = {}
    try:
        # k-means: eager first iteration, then CUDA-graph replays (the bench's form)
        lo, hi = shard_range(N_KM, rank, world)
        x = ml.rng_units((hi - lo) * D_KM, seed=1, first_draw=lo * D_KM).view(hi - lo, D_KM)
        mu0 = ml.rng_units(K_KM * D_KM, seed=1).view(K_KM, D_KM)
        prog = KMeansProgram(x, K_KM, mu0, comm=comm)
        hist = []
        prog.step()
        hist.append((prog.counts.cpu().numpy(), prog.sums.cpu().numpy(), prog.mu.cpu().numpy()))
        prog.capture()
        for _ in range(IT_KM - 1):
            prog.step()
            hist.append((prog.counts.cpu().numpy(), prog.sums.cpu().numpy(), prog.mu.cpu().numpy()))
        out["kmeans"] = hist
        # logistic regression BGD with the fused step
        lo, hi = shard_range(N_LR, rank, world)
        xl = ml.rng_units((hi - lo) * D_LR, seed=2, first_draw=lo * D_LR).view(hi - lo, D_LR)
        yl = ml.rng_ints(hi - lo, 2, seed=2, first_draw=N_LR * D_LR + lo)
        lp = LogRegProgram(xl, yl, torch.zeros(D_LR, dtype=torch.float64, device="cuda"), 1.0 / N_LR, comm=comm)
        lp.run(IT_LR)
        out["logreg"] = lp.theta.cpu().numpy()
        # GroupBy counts (int64 record, no epilogue) and a scalar
        lo, hi = shard_range(N_GB, rank, world)
        keys = ml.rng_ints(hi - lo, K_GB, seed=3, first_draw=lo)
        cnt = ml.groupby_count(keys, K_GB)
        comm.allreduce_(cnt)
        out["groupby"] = cnt.cpu().numpy()
        out["n"] = comm.allreduce_int(hi - lo)
        # GDA: each rank's single-pass fit pooled through the exchange (gda_combine_ranks_kernel)
        lo, hi = shard_range(N_GD, rank, world)
        xg = ml.rng_units((hi - lo) * D_GD, seed=4, first_draw=lo * D_GD).view(hi - lo, D_GD)
        yg = ml.rng_ints(hi - lo, 2, seed=4, first_draw=N_GD * D_GD + lo)
        n1, mu0, mu1, S = ml.gda(xg, yg, comm)
        out["gda"] = (int(n1.item()), mu0.cpu().numpy(), mu1.cpu().numpy(), S.cpu().numpy())
        torch.cuda.synchronize()
    finally:
        comm.close()
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_peer_allreduce_one_device(world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    while len(res) < world:
        r, out = q.get(timeout=600)
        assert "error" not in out, f"rank {r}: {out['error']}"
        res[r] = out
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    r0 = res[0]
    # every rank holds bit-identical results (ascending-rank fold on each)
    for r in range(1, world):
        rr = res[r]
        for (c0, s0, m0), (c1, s1, m1) in zip(r0["kmeans"], rr["kmeans"]):
            assert np.array_equal(c0, c1) and np.array_equal(s0.view(np.int64), s1.view(np.int64))
            assert np.array_equal(m0.view(np.int64), m1.view(np.int64))
        assert np.array_equal(r0["logreg"].view(np.int64), rr["logreg"].view(np.int64))
        assert np.array_equal(rr["groupby"], r0["groupby"])
        assert np.array_equal(r0["gda"][3].view(np.int64), rr["gda"][3].view(np.int64))
    # against the single-process oracle
    x, _ = O.kmeans_inputs(N_KM, D_KM, K_KM)
    mu = x[:K_KM].copy()
    for it in range(IT_KM):
        _, c, s = O.kmeans_step(x, K_KM, mu, workers=O.threads(), chunks=4 * O.threads())
        mu = O.kmeans_update(c, s)
        gc, gs, gm = r0["kmeans"][it]
        assert np.array_equal(gc, c), f"iteration {it}"
        np.testing.assert_allclose(gs, s, rtol=1e-9)
        np.testing.assert_allclose(gm, mu, rtol=1e-9)
    xl = O.rng_units(2, 0, N_LR * D_LR).reshape(N_LR, D_LR)
    yl = O.rng_ints(2, N_LR * D_LR, N_LR, 2)
    th = np.zeros(D_LR)
    for _ in range(IT_LR):
        th = th - (1.0 / N_LR) * O.logreg_grad(xl, yl, th)
    np.testing.assert_allclose(r0["logreg"], th, rtol=1e-9, atol=1e-13)
    keys = O.rng_ints(3, 0, N_GB, K_GB)
    assert np.array_equal(r0["groupby"], O.groupby_count(keys, K_GB))
    assert all(res[r]["n"] == N_GB for r in range(world))
    xg = O.rng_units(4, 0, N_GD * D_GD).reshape(N_GD, D_GD)
    yg = O.rng_ints(4, N_GD * D_GD, N_GD, 2)
    n1, s0, s1 = O.gda_pass1(xg, yg, workers=O.threads(), chunks=4 * O.threads())
    m0, m1 = s0 / float(N_GD - n1), s1 / float(n1)
    Sr = O.gda_pass2(xg, yg, m0, m1, workers=O.threads(), chunks=4 * O.threads())
    for r in range(world):
        g = res[r]["gda"]
        assert g[0] == n1
        np.testing.assert_allclose(g[1], m0, rtol=1e-9)
        np.testing.assert_allclose(g[2], m1, rtol=1e-9)
        np.testing.assert_allclose(g[3], Sr, rtol=1e-9, atol=1e-9 * np.abs(Sr).max())


def test_peer_world1_epilogues_match_unfused():
    """world 1: the fused kernel is the identity collective plus the update; results equal the
    unfused kmeans_update / axpy_inplace launches bit for bit."""
    from paper_1109_0778_b200 import multiloops as ml
    from paper_1109_0778_b200.comm import PeerComm
    comm = PeerComm(0, 1, cap_bytes=1 << 20)
    try:
        k, d = 64, 64
        counts = torch.arange(k, dtype=torch.int64, device="cuda") * 3   # counts[0] = 0 -> NaN row
        sums = torch.rand(k, d, dtype=torch.float64, device="cuda") * 100
        sums[0] = 0.0                                                      # 0 / 0
        mu = torch.empty(k, d, dtype=torch.float64, device="cuda")
        ref = ml.kmeans_update(counts.clone(), sums.clone())
        for _ in range(3):   # epochs advance; slots alternate
            c2, s2 = counts.clone(), sums.clone()
            comm.kmeans_update_(c2, s2, mu)
            assert torch.equal(c2, counts) and torch.equal(s2, sums)
            assert torch.isnan(mu[0]).all() and torch.equal(mu[1:], ref[1:])
        g = torch.rand(d, dtype=torch.float64, device="cuda")
        th = torch.rand(d, dtype=torch.float64, device="cuda")
        th_ref = ml.axpy_inplace(th.clone(), g, 0.25)
        comm.bgd_step_(g.clone(), th, 0.25)
        assert torch.equal(th, th_ref)
        with pytest.raises(RuntimeError):
            big = torch.zeros(1 << 20, dtype=torch.float64, device="cuda")   # 8 MB > 1 MB buffer slot
            comm.allreduce_(big)
    finally:
        comm.close()


def test_nccl_communicator_world1():
    """The NCCL path (csrc/comm.cu: dlx_comm_init / allreduce_sum / allreduce_sum_group /
    destroy) with a real one-rank communicator: the collective is the identity, on the caller's
    stream, for fp64 and int64 records, single and grouped (NCCL refuses two ranks on one GPU, so
    world 1 is what one box can run)."""
    from paper_1109_0778_b200.comm import Comm
    uid = Comm.unique_id()
    c = Comm(0, 1, uid, force_nccl=True)
    try:
        a = torch.rand(4096, dtype=torch.float64, device="cuda")
        b = torch.arange(65_536, dtype=torch.int64, device="cuda") - 7
        a0, b0 = a.clone(), b.clone()
        c.allreduce_(a)
        c.allreduce_(b)
        c.allreduce_many_([a, b])
        torch.cuda.synchronize()
        assert torch.equal(a, a0) and torch.equal(b, b0)
        assert c.allreduce_int(41) == 41
    finally:
        c.close()
