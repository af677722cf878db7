"""Host problem setup against the reference's own outputs (golden fixtures):
Legendre-Gauss-Lobatto grids, superconsistent nodes, collocation blocks,
assembled operator trains and right-hand sides.  The setup's recompressions
run through the CPU oracle here (setup_backend), so no GPU is needed."""

import numpy as np
import pytest

from golden_io import get_train
from oracle import tt_ops as ot
from paper_2506_04732_b200 import assembly, coefficients as co, collocation, spectral, tt


def _cpu_numerics():
    def rnd(v, tol, max_rank=None):
        if isinstance(v, tt.TTOperator):
            return tt.TTOperator(ot.as_operator(ot.tt_round(ot.as_vector(v.cores), tol, max_rank),
                                                v.row_sizes, v.col_sizes))
        return tt.TTVector(ot.tt_round(v.cores, tol, max_rank))

    return assembly.setup_backend(round=rnd, add=lambda a, b: type(a)(ot.tt_add(a.cores, b.cores)),
                                  apply=lambda o, v: tt.TTVector(ot.tt_apply(o.cores, v.cores)))


def test_grids_match_reference(golden):
    z = golden("setup_grids.npz")
    for i, (n, eps, beta) in enumerate(z["cases"]):
        n = int(n)
        np.testing.assert_allclose(spectral.gll_nodes(n), z[f"{i}_gll"], rtol=0, atol=1e-15)
        np.testing.assert_allclose(spectral.gauss_nodes(n), z[f"{i}_gauss"], rtol=0, atol=1e-15)
        g = collocation.sc_grid(n, eps, beta)
        np.testing.assert_allclose(g.coll_nodes, z[f"{i}_coll"], rtol=0, atol=1e-14)
        np.testing.assert_allclose(g.base.bary_w, z[f"{i}_bary"], rtol=1e-13, atol=1e-15)
        for k in ("d1", "d2"):
            ref = z[f"{i}_{k}"]
            np.testing.assert_allclose(getattr(g.base, k), ref, rtol=0,
                                       atol=1e-12 * np.abs(ref).max())
        for k in ("a0", "a1", "a2"):
            ref = z[f"{i}_{k}"]
            np.testing.assert_allclose(getattr(g, k), ref, rtol=0,
                                       atol=1e-11 * max(np.abs(ref).max(), 1.0))


OP_CASES = [
    ("d2", 2, 6, 0.05, [1.0, 3.0], 0.1, "superconsistent"),
    ("d3", 3, 4, 1e-3, [1.0, -0.5, 0.25], 0.0, "superconsistent"),
    ("d2p", 2, 5, 0.2, [0.0, 1.0], 0.3, "plain"),
]


@pytest.mark.parametrize("tag,dims,deg,eps,beta,rho,stab", OP_CASES)
def test_operators_match_reference(golden, tag, dims, deg, eps, beta, rho, stab):
    z = golden("setup_ops.npz")
    spec = assembly.ProblemSpec(dims=dims, degrees=[deg] * dims,
                                epsilon=co.constant_coefficient(eps, dims),
                                beta=[co.constant_coefficient(b, dims) for b in beta],
                                rho=co.constant_coefficient(rho, dims),
                                rhs=co.constant_coefficient(1.0, dims), stabilization=stab)
    with _cpu_numerics():
        from paper_2506_04732_b200 import march

        op = assembly.assemble_opset(spec)
        _, b = assembly.impose_dirichlet(op, spec)
        pairs = [(getattr(op, k).cores, f"{tag}_{k}")
                 for k in ("diffusion", "convection", "reaction", "mask_interior", "spatial")]
        for scheme in ("backward_euler", "crank_nicolson"):
            left, right, _, _ = march.march_operators(
                op, march.MarchConfig(dt=0.01, t_end=0.05, scheme=scheme))
            pairs += [(left.cores, f"{tag}_{scheme}_left"), (right.cores, f"{tag}_{scheme}_right")]
    for got, name in pairs:
        want = get_train(z, name)
        assert ot.ranks_of(got) == ot.ranks_of(want), name
        dg, dw = ot.tt_op_full(got), ot.tt_op_full(want)
        assert np.abs(dg - dw).max() <= 1e-12 * max(np.abs(dw).max(), 1.0), name
    rw = get_train(z, f"{tag}_rhs")
    assert ot.ranks_of(b.cores) == ot.ranks_of(rw)
    np.testing.assert_allclose(ot.tt_full(b.cores), ot.tt_full(rw), rtol=0,
                               atol=1e-12 * np.abs(ot.tt_full(rw)).max())


def test_config_json_grammar():
    cfg = {"dims": 2, "degrees": [6], "epsilon": 0.1, "beta": [1.0, {"terms": [
        {"scale": 2.0, "factors": [["sin_pi_k", [1]], ["poly", [0.0, 1.0]]]}]}],
        "rho": 0.0, "rhs": 1.0, "bc": None, "time": {"t_end": 1.0, "degree": 4}}
    spec = assembly.problem_from_config(cfg)
    assert spec.degrees == [6, 6] and spec.time.degree == 4
    assert not spec.beta[1].is_constant
    with pytest.raises(ValueError):
        co.factor_from_json(["nope", [1]])
    with pytest.raises(ValueError):
        assembly.ProblemSpec(dims=1, degrees=[4], epsilon=co.constant_coefficient(-1.0, 1),
                             beta=[co.constant_coefficient(0.0, 1)],
                             rho=co.constant_coefficient(0.0, 1), rhs=co.constant_coefficient(0.0, 1))


def test_tts2_container_roundtrip(tmp_path):
    rng = np.random.default_rng(0)
    v = tt.TTVector([rng.standard_normal(s) for s in [(1, 3, 2), (2, 4, 1)]])
    o = tt.TTOperator([rng.standard_normal(s) for s in [(1, 3, 3, 2), (2, 4, 4, 1)]])
    for obj in (v, o):
        path = tmp_path / "x.tts2"
        tt.save_tt(obj, path)
        back = tt.load_tt(path)
        assert type(back) is type(obj)
        for a, b in zip(obj.cores, back.cores):
            np.testing.assert_array_equal(a, b)
