"""Config-4 sweep sharding on CPU: world_size 2 over gloo, with the CPU
oracle standing in for the device solver (the product path needs a GPU; the
sharding, ownership and gather logic is what is exercised here)."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from golden_io import get_train


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _cpu_build(recipe):
    """The workload's setup (ttss, host numpy: no GPU involved)."""
    from paper_2506_04732_b200 import workloads as wl

    return wl.steady_problem(recipe)


def _cpu_solve(a, b, cfg):
    from oracle import als_solver as als
    from paper_2506_04732_b200.reference import module

    kw = {k: v for k, v in cfg.items()}
    x0 = als.initial_guess(b.cores, als.Config(**kw), np.random.default_rng(kw.get("seed", 0)))
    x, rep = als.solve(a.cores, b.cores, x0=x0, cfg=als.Config(**kw))
    return module("tensor_train").TTVector(x), rep


_GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "config4_small.npz")


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_04732_b200 import sweep, workloads as wl

    recipes = wl.sweep_recipes(count=4, dims=3, degree=12)
    local = sweep.run_sweep(recipes, rank, world, solve_fn=_cpu_solve, build_fn=_cpu_build,
                            overrides={"max_sweeps": int(np.load(_GOLDEN)["sweeps"])})
    assert sorted(local) == sweep.shard(4, rank, world)
    merged = sweep.gather(local, world)
    if rank == 0:
        np.save(os.path.join(out_dir, "merged.npy"), np.array([merged], dtype=object),
                allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()


def test_shard_ownership():
    from paper_2506_04732_b200.sweep import shard

    owned = [shard(64, r, 8) for r in range(8)]
    assert sorted(sum(owned, [])) == list(range(64))
    assert all(len(o) == 8 for o in owned)
    with pytest.raises(ValueError):
        shard(4, 2, 2)


def test_sweep_gloo_world2(tmp_path, golden):
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    merged = np.load(tmp_path / "merged.npy", allow_pickle=True)[0]
    assert sorted(merged) == [0, 1, 2, 3]
    z = golden("config4_small.npz")
    from helpers import ranks_agree, rel_diff, value_tol

    for i in range(4):
        # every solve ran exactly once, on its owner, and converged to the
        # reference's solution
        ref = np.array(z[f"res{i}"])
        got = merged[i]
        assert got["converged"] and bool(z[f"conv{i}"])
        want = get_train(z, f"x{i}")
        assert rel_diff(got["x"], want) <= value_tol(got["residuals"][-1], ref[-1])
        ok, det = ranks_agree(got["x"], want)
        assert ok, det
