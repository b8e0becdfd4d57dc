"""Batched Newton runs (config C5): sharding/gather host logic on CPU with a
world-size-2 gloo group, and GPU parity of pn_newton_batch against the
one-start-at-a-time path and the reference goldens."""

import os

import numpy as np
import pytest

from conftest import golden, level_from_name, same


def test_shard_range_partitions_every_size():
    from paper_1402_2626_b200.batch import shard_range
    for B in (0, 1, 7, 8, 8192, 8193):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(B, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == B
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1


def _gather_worker(rank, world, port, B, out_dir):
    import torch.distributed as dist
    from paper_1402_2626_b200.batch import BatchResult, gather_batch, shard_range
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    lo, hi = shard_range(B, world, rank)
    cnt = hi - lo
    # deterministic stand-in for per-start results: values encode (start, slot)
    x = np.zeros((2, 2, cnt, 5))
    for b in range(cnt):
        x[..., b, :] = (lo + b) * 100 + np.arange(5)
    shard = BatchResult(x, np.arange(lo, hi, dtype=np.int32) % 7, (np.arange(lo, hi) % 3).astype(np.int32))
    full = gather_batch(shard, B)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), x=full.x, iters=full.iters, status=full.status)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("B", [9, 16])
def test_gather_batch_gloo_world2(tmp_path, B):
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(_gather_worker, args=(2, port, B, str(tmp_path)), nprocs=2, join=True)
    for r in range(2):
        d = np.load(tmp_path / f"r{r}.npz")
        assert d["x"].shape == (2, 2, B, 5)
        for b in range(B):
            assert np.array_equal(d["x"][..., b, :], np.broadcast_to(b * 100 + np.arange(5), (2, 2, 5)))
        assert np.array_equal(d["iters"], np.arange(B) % 7)
        assert np.array_equal(d["status"], np.arange(B) % 3)


def _run_batched_worker(rank, world, port, B, out_dir):
    """run_batched's shard -> solve -> gather with stub prepare/solve: every
    rank must solve exactly its shard_range and end with the full batch."""
    import torch.distributed as dist
    from paper_1402_2626_b200.batch import BatchResult, run_batched
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    n = 4
    Z = np.zeros((2, 2, B, n))
    Z[0, 0] = np.arange(B)[:, None] + 0.25 * np.arange(n)
    seen = {}

    def prepare(packed, Zs, t):
        seen["prepared"] = Zs.shape[-2]
        return "prep", Zs[..., 0] * t  # per-start stand-in for the homotopy constants

    def solve(prep, Zs, consts, max_iters, tol):
        assert prep == "prep" and consts.shape[-1] == Zs.shape[-2]
        start = Zs[0, 0, :, 0].astype(int)   # each start carries its global index
        x = Zs * 2.0 + 1.0
        return BatchResult(x, (start % max_iters).astype(np.int32), (start % 4).astype(np.int32))

    shard, full, (lo, hi) = run_batched(None, Z, 3.0, max_iters=5, prepare=prepare, solve=solve)
    np.savez(os.path.join(out_dir, f"rb{rank}.npz"), x=full.x, iters=full.iters, status=full.status,
             lo=lo, hi=hi, prepared=seen["prepared"], shard_n=shard.x.shape[-2])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("B", [7, 8192])
def test_run_batched_orchestration_gloo_world2(tmp_path, B):
    import socket

    import torch.multiprocessing as mp
    from paper_1402_2626_b200.batch import shard_range
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(_run_batched_worker, args=(2, port, B, str(tmp_path)), nprocs=2, join=True)
    n = 4
    Z = np.zeros((2, 2, B, n))
    Z[0, 0] = np.arange(B)[:, None] + 0.25 * np.arange(n)
    for r in range(2):
        d = np.load(tmp_path / f"rb{r}.npz")
        lo, hi = shard_range(B, 2, r)
        assert (int(d["lo"]), int(d["hi"])) == (lo, hi)
        assert int(d["prepared"]) == hi - lo == int(d["shard_n"])
        assert np.array_equal(d["x"], Z * 2.0 + 1.0)
        assert np.array_equal(d["iters"], np.arange(B) % 5)
        assert np.array_equal(d["status"], np.arange(B) % 4)


# -- GPU ---------------------------------------------------------------------------------

def _packed(g, prefix=""):
    from paper_1402_2626_b200.polyrep import PackedSystem
    level = level_from_name(str(g["level"]))
    return PackedSystem(level, int(g["n_vars"]), g[prefix + "poly_ptr"].astype(np.int32),
                        g[prefix + "mon_ptr"].astype(np.int32), g[prefix + "var_idx"].astype(np.int32),
                        g[prefix + "exps"].astype(np.int32), np.ascontiguousarray(g[prefix + "coeffs"]))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["newton_homotopy_cdd", "newton_homotopy_cqd", "newton_homotopy_cd",
                                  "newton_cyclic8_cdd"])
def test_batch_reproduces_reference_run(gpu, name):
    """B=1 batch on the golden homotopy case == the reference's run_newton."""
    from paper_1402_2626_b200.batch import homotopy_batch, run_newton_batch
    from paper_1402_2626_b200.evaldiff import PreparedSystem
    g = golden(name)
    p = _packed(g)
    level = p.level
    t = level.from_planes(g["t"])[0]
    Z = np.ascontiguousarray(g["z"][..., None, :])
    system, consts = homotopy_batch(p, Z, t)
    iters = str(g["trace"]).count("\n")
    res = run_newton_batch(PreparedSystem(system), Z, consts, max_iters=iters)
    assert same(res.x[..., 0, :], g["x_final"])
    assert res.iters[0] == iters
    assert res.status[0] == (0 if bool(g["converged"]) else 1)


@pytest.mark.gpu
@pytest.mark.parametrize("lv", ["cdd", "cd", "cqd"])
def test_batch_matches_single_runs(gpu, lv):
    from paper_1402_2626_b200.batch import homotopy_batch, run_newton_batch
    from paper_1402_2626_b200.evaldiff import PreparedSystem
    from paper_1402_2626_b200.generators import random_sparse_system, random_unit_point
    from paper_1402_2626_b200.newton import NewtonConfig, homotopy_start_system, run_newton
    level = level_from_name(lv)
    p = random_sparse_system(16, 8, 4, level, seed=31, maxexp=2)
    B = 5
    Z = np.stack([level.to_planes(random_unit_point(16, 100 + b, level)) for b in range(B)], axis=-2)
    t = level.from_float(0.99)
    system, consts = homotopy_batch(p, Z, t)
    res = run_newton_batch(PreparedSystem(system), Z, consts, max_iters=8)
    for b in range(B):
        single = homotopy_start_system(p, np.ascontiguousarray(Z[..., b, :]), t)
        tr = run_newton(single, np.ascontiguousarray(Z[..., b, :]), NewtonConfig(level=level, max_iters=8))
        assert same(res.x[..., b, :], level.to_planes(tr.x)), b
        assert res.iters[b] == len(tr.entries)
        assert res.status[b] == (0 if tr.converged else 1)


def _single_runs(p, Z, t, level, max_iters):
    from paper_1402_2626_b200.newton import NewtonConfig, homotopy_start_system, run_newton
    out = []
    for b in range(Z.shape[-2]):
        zb = np.ascontiguousarray(Z[..., b, :])
        single = homotopy_start_system(p, zb, t)
        out.append(run_newton(single, zb, NewtonConfig(level=level, max_iters=max_iters)))
    return out


def _check_batch_vs_single(lv, n, T, k, B, max_iters, seed, m=None, slots=None):
    from paper_1402_2626_b200.batch import homotopy_batch, run_newton_batch
    from paper_1402_2626_b200.evaldiff import PreparedSystem
    from paper_1402_2626_b200.generators import random_point, random_sparse_system, random_unit_point
    level = level_from_name(lv)
    kw = {} if m is None else {"m": m}
    p = random_sparse_system(n, T, k, level, seed=seed, maxexp=2, **kw)
    gen = random_unit_point if level.cplx else random_point
    Z = np.stack([level.to_planes(gen(n, 1000 + seed + b, level)) for b in range(B)], axis=-2)
    t = level.from_float(0.99)
    system, consts = homotopy_batch(p, Z, t)
    old = os.environ.get("PN_BATCH_SLOTS")
    if slots is not None:
        os.environ["PN_BATCH_SLOTS"] = str(slots)
    try:
        res = run_newton_batch(PreparedSystem(system), Z, consts, max_iters=max_iters)
    finally:
        if slots is not None:
            if old is None:
                del os.environ["PN_BATCH_SLOTS"]
            else:
                os.environ["PN_BATCH_SLOTS"] = old
    for b, tr in enumerate(_single_runs(p, Z, t, level, max_iters)):
        assert same(res.x[..., b, :], level.to_planes(tr.x)), (lv, b)
        assert res.iters[b] == len(tr.entries), (lv, b)
        assert res.status[b] == (0 if tr.converged else 1), (lv, b)


@pytest.mark.gpu
@pytest.mark.parametrize("lv", ["cd", "cdd", "cqd", "rdd", "rqd"])
def test_batch_multi_panel(gpu, lv):
    """n = 40 spans several left-looking panels (P = 8/16/32) with a ragged last one."""
    _check_batch_vs_single(lv, 40, 6, 3, 3, 6, seed=11)


@pytest.mark.gpu
def test_batch_slot_refill(gpu):
    """More starts than slots: retired slots are refilled from the queue."""
    _check_batch_vs_single("cdd", 24, 5, 3, 7, 8, seed=5, slots=2)


@pytest.mark.gpu
@pytest.mark.parametrize("lv,n,m", [("cdd", 40, 56), ("cd", 300, 300), ("cdd", 520, 520), ("cqd", 260, 270)])
def test_batch_row_blocks(gpu, lv, n, m):
    """Overdetermined systems and every rows-per-thread variant (m <= 256, 512, 1024)."""
    _check_batch_vs_single(lv, n, 3, 2, 2, 2, seed=3, m=m)


@pytest.mark.gpu
def test_batch_breakdown_status(gpu):
    """A variable that appears nowhere gives a zero Jacobian column: MGS breakdown
    (mgs.py:176-181) is reported per start and x keeps its last value."""
    from paper_1402_2626_b200.batch import homotopy_batch, run_newton_batch
    from paper_1402_2626_b200.evaldiff import PreparedSystem
    from paper_1402_2626_b200.generators import random_sparse_system, random_unit_point
    from paper_1402_2626_b200.polyrep import PackedSystem
    level = level_from_name("cdd")
    p = random_sparse_system(12, 5, 3, level, seed=9, maxexp=1, m=13)
    # widen to 13 variables: x12 never appears
    q = PackedSystem(level, 13, p.poly_ptr, p.mon_ptr, p.var_idx, p.exps, p.coeffs)
    B = 3
    Z = np.stack([level.to_planes(random_unit_point(13, 50 + b, level)) for b in range(B)], axis=-2)
    system, consts = homotopy_batch(q, Z, level.from_float(0.99))
    res = run_newton_batch(PreparedSystem(system), Z, consts, max_iters=5)
    assert list(res.status) == [2] * B
    assert list(res.iters) == [1] * B
    assert same(res.x, Z)


@pytest.mark.gpu
def test_serial_batch_matches_slots_and_leaves_system_unchanged(gpu, monkeypatch):
    """PN_BATCH_MODE=serial (one start at a time, also used for m > 1024)
    gives the slot path's results and restores the system's constants."""
    from paper_1402_2626_b200.batch import homotopy_batch, run_newton_batch
    from paper_1402_2626_b200.evaldiff import PreparedSystem, evaluate_system
    from paper_1402_2626_b200.generators import random_sparse_system, random_unit_point
    level = level_from_name("cdd")
    p = random_sparse_system(20, 6, 3, level, seed=21, maxexp=2)
    B = 4
    Z = np.stack([level.to_planes(random_unit_point(20, 300 + b, level)) for b in range(B)], axis=-2)
    system, consts = homotopy_batch(p, Z, level.from_float(0.99))
    prep = PreparedSystem(system)
    z0 = np.ascontiguousarray(Z[..., 0, :])
    before = evaluate_system(prep, z0).f
    slots = run_newton_batch(prep, Z, consts, max_iters=6)
    monkeypatch.setenv("PN_BATCH_MODE", "serial")
    serial = run_newton_batch(prep, Z, consts, max_iters=6)
    assert same(serial.x, slots.x)
    assert np.array_equal(serial.iters, slots.iters) and np.array_equal(serial.status, slots.status)
    assert same(evaluate_system(prep, z0).f, before)


@pytest.mark.gpu
@pytest.mark.parametrize("lv,B", [("cdd", 7), ("rqd", 1), ("cd", 300)])
def test_nccl_comm_batch_allgather_world1(gpu, lv, B):
    """The C ABI's collective (pn_comm_init + pn_batch_allgather) on a
    world of one: the gathered batch is the shard, host and device buffers."""
    from paper_1402_2626_b200.batch import BatchResult, NcclComm
    level = level_from_name(lv)
    rng = np.random.default_rng(B)
    n = 9
    shard = BatchResult(rng.standard_normal(level.cshape + (B, n)), rng.integers(0, 9, B).astype(np.int32),
                        rng.integers(0, 4, B).astype(np.int32))
    comm = NcclComm(1, 0, NcclComm.unique_id())
    full = comm.gather_batch(shard, B, level)
    assert np.array_equal(full.x, shard.x)
    assert np.array_equal(full.iters, shard.iters) and np.array_equal(full.status, shard.status)
    with pytest.raises(ValueError):
        comm.gather_batch(BatchResult(shard.x[..., :-1, :], shard.iters, shard.status), B, level)
    comm.close()

