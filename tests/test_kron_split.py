"""Kronecker-sum-term split of one operator apply (kron_split.py) on CPU:
world_size 2 over gloo with the numpy oracle as the arithmetic backend (the
engine needs a GPU; the sharding, the all-gather of partial trains and the
final sum are what is exercised here).  The terms are the reference's own
per-dimension chains (operator_assembly._chain)."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class OracleBackend:
    """CPU stand-in for the engine (tests only)."""

    def __init__(self):
        from oracle import tt_ops
        from paper_2506_04732_b200.reference import module

        self.ot = tt_ops
        self.TTVector = module("tensor_train").TTVector

    def apply(self, op, x):
        return self.TTVector(self.ot.tt_apply(op.cores, x.cores))

    def add(self, a, b, sa=1.0, sb=1.0):
        ac = self.ot.tt_scale(a.cores, sa) if sa != 1.0 else a.cores
        bc = self.ot.tt_scale(b.cores, sb) if sb != 1.0 else b.cores
        return self.TTVector(self.ot.tt_add(ac, bc))

    def round(self, x, tol):
        return self.TTVector(self.ot.tt_round(x.cores, tol))

    def norm(self, x):
        return float(self.ot.tt_norm(x.cores))

    def vector(self, cores):
        return self.TTVector(cores)


def _problem(dims=4, degree=8, eps=0.05):
    """The d diffusion + d convection terms of -eps Lap + b.grad on the
    reference's superconsistent grids, and a smooth rank-3 state."""
    from paper_2506_04732_b200.reference import module

    oa, sc, rtt = module("operator_assembly"), module("superconsistency"), module("tensor_train")
    beta = np.linspace(1.0, 0.25, dims)
    grids = [sc.sc_grid(degree, eps, float(b)) for b in beta]
    terms = []
    for l, g in enumerate(grids):
        terms.append(rtt.tt_op_scale(oa._chain(grids, (l, g.a2)), -eps))
        terms.append(rtt.tt_op_scale(oa._chain(grids, (l, g.a1)), float(beta[l])))
    n = grids[0].a0.shape[1]
    s = np.linspace(-1.0, 1.0, n)
    x = rtt.tt_from_separable([(1.0, [np.exp(-(s - 0.1 * k) ** 2) for k in range(dims)]),
                               (0.5, [np.cos(s * (k + 1)) for k in range(dims)]),
                               (0.25, [s ** (k % 3) for k in range(dims)])])
    return terms, x


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_04732_b200 import kron_split

    terms, x = _problem()
    be = OracleBackend()
    y = kron_split.sharded_apply(terms, x, 1e-12, rank, world, backend=be)
    res = kron_split.sharded_residual(terms, x, y, 1e-10, rank, world, backend=be)
    np.save(os.path.join(out_dir, f"y{rank}.npy"), np.array([y.cores, res], dtype=object),
            allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()


def test_term_ownership():
    from paper_2506_04732_b200.kron_split import shard_terms

    owned = [shard_terms(12, r, 8) for r in range(8)]
    assert sorted(sum(owned, [])) == list(range(12))
    assert shard_terms(3, 5, 8) == []
    with pytest.raises(ValueError):
        shard_terms(4, 2, 2)


def test_sharded_apply_gloo_world2(tmp_path):
    from oracle import tt_ops as ot

    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    terms, x = _problem()
    # unsharded: the reference's way, one merged operator
    want = None
    for t in terms:
        y = ot.tt_apply(t.cores, x.cores)
        want = y if want is None else ot.tt_add(want, y)
    want = ot.tt_round(want, 1e-12)
    got = [np.load(tmp_path / f"y{r}.npy", allow_pickle=True) for r in range(2)]
    full_want = ot.tt_full(want)
    for cores, res in got:
        diff = np.linalg.norm(ot.tt_full(list(cores)) - full_want) / np.linalg.norm(full_want)
        assert diff <= 1e-11, diff
        assert ot.ranks_of(list(cores)) == ot.ranks_of(want)
        assert res <= 1e-10  # the residual of A x = (A x) through the same split
    # both ranks hold the same result bit for bit
    for a, b in zip(got[0][0], got[1][0]):
        assert np.array_equal(a, b)


@pytest.mark.gpu
def test_engine_backend_single_rank_matches_oracle():
    """The same split through the CUDA engine on one rank (world 1: every
    term local, no collective) against the oracle's merged apply."""
    from oracle import tt_ops as ot
    from paper_2506_04732_b200 import kron_split

    terms, x = _problem(dims=5, degree=12)
    y = kron_split.sharded_apply(terms, x, 1e-12)
    want = None
    for t in terms:
        z = ot.tt_apply(t.cores, x.cores)
        want = z if want is None else ot.tt_add(want, z)
    want = ot.tt_round(want, 1e-12)
    fw = ot.tt_full(want)
    assert np.linalg.norm(ot.tt_full(y.cores) - fw) <= 1e-11 * np.linalg.norm(fw)
    assert list(y.ranks) == list(ot.ranks_of(want))
    assert kron_split.sharded_residual(terms, x, y, 1e-10) <= 1e-10
