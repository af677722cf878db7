"""The host side of the drop-in is the reference's own ``ttss`` (problem
setup, containers, configs, exceptions).  These CPU tests pin the ``ttss``
that ``paper_2506_04732_b200.reference`` resolves (baseline/_ref, the
offline install of /root/reference/pkg) to the golden fixtures recorded
from the reference, and check that the package's workloads and type
re-exports are that ttss's."""

import numpy as np
import pytest

from golden_io import get_train
from oracle import tt_ops as ot
from paper_2506_04732_b200 import reference


@pytest.fixture(scope="module")
def ttss():
    return reference.ttss()


def test_grids_match_reference(golden, ttss):
    rs, rsc = reference.module("spectral1d"), reference.module("superconsistency")
    z = golden("setup_grids.npz")
    for i, (n, eps, beta) in enumerate(z["cases"]):
        n = int(n)
        np.testing.assert_array_equal(rs.gll_nodes(n), z[f"{i}_gll"])
        g = rsc.sc_grid(n, eps, beta)
        np.testing.assert_array_equal(g.coll_nodes, z[f"{i}_coll"])
        for k in ("a0", "a1", "a2"):
            np.testing.assert_array_equal(getattr(g, k), z[f"{i}_{k}"])


OP_CASES = [
    ("d2", 2, 6, 0.05, [1.0, 3.0], 0.1, "superconsistent"),
    ("d3", 3, 4, 1e-3, [1.0, -0.5, 0.25], 0.0, "superconsistent"),
    ("d2p", 2, 5, 0.2, [0.0, 1.0], 0.3, "plain"),
]


@pytest.mark.parametrize("tag,dims,deg,eps,beta,rho,stab", OP_CASES)
def test_march_operators_match_reference(golden, ttss, tag, dims, deg, eps, beta, rho, stab):
    co, asm = reference.module("coefficients"), reference.module("operator_assembly")
    from paper_2506_04732_b200 import march

    z = golden("setup_ops.npz")
    spec = asm.ProblemSpec(dims=dims, degrees=[deg] * dims,
                           epsilon=co.constant_coefficient(eps, dims),
                           beta=[co.constant_coefficient(b, dims) for b in beta],
                           rho=co.constant_coefficient(rho, dims),
                           rhs=co.constant_coefficient(1.0, dims), stabilization=stab)
    op = asm.assemble_opset(spec)
    for scheme in ("backward_euler", "crank_nicolson"):
        left, right, _, _ = march.march_operators(
            op, spec, march.MarchConfig(dt=0.01, t_end=0.05, scheme=scheme))
        for got, name in ((left, f"{tag}_{scheme}_left"), (right, f"{tag}_{scheme}_right")):
            want = get_train(z, name)
            assert ot.ranks_of(got.cores) == ot.ranks_of(want), name
            for a, b in zip(got.cores, want):
                np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("fname,index", [("config2_full.npz", 2), ("config3_full.npz", 3)])
def test_workload_setup_is_the_references(golden, ttss, fname, index):
    """The bench/test workloads are built by ttss: operator fingerprints and
    the initial state equal what the reference recorded."""
    from paper_2506_04732_b200 import workloads as wl

    z = golden(fname)
    left, right, state0, _, _, _ = wl.march_problem(wl.config(index))
    np.testing.assert_array_equal([np.abs(c).sum() for c in left.cores], z["left_sums"])
    np.testing.assert_array_equal([np.abs(c).sum() for c in right.cores], z["right_sums"])
    for a, b in zip(state0.cores, get_train(z, "state0")):
        np.testing.assert_array_equal(a, b)


def test_host_types_are_the_references(ttss):
    from paper_2506_04732_b200 import errors, march, solver, tt

    rtt = reference.module("tensor_train")
    assert tt.TTVector is rtt.TTVector and tt.TTOperator is rtt.TTOperator
    assert solver.SolverConfig is reference.module("tt_solver").SolverConfig
    assert solver.SolveReport is reference.module("tt_solver").SolveReport
    assert march.MarchConfig is reference.module("time_integration").MarchConfig
    assert errors.MarchStepError is reference.module("errors").MarchStepError
    with pytest.raises(ValueError):
        solver.SolverConfig(local_solver="magic")


def test_dropin_install_swaps_only_the_hot_path(ttss):
    from paper_2506_04732_b200 import dropin, march, solver

    sol, ti = reference.module("tt_solver"), reference.module("time_integration")
    orig = (sol.solve, sol.residual, ti._march, ti.solve)
    dropin.install()
    try:
        assert sol.solve is solver.solve and sol.residual is solver.residual
        assert ti._march is march._march and ti.solve is solver.solve
        assert ti.backward_euler_march.__module__ == "ttss.time_integration"
    finally:
        dropin.uninstall()
    assert (sol.solve, sol.residual, ti._march, ti.solve) == orig
