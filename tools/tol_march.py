"""Config-2 march with the BASELINE prose's literal "TT tolerance 1e-12" as
the inner residual target (and optionally as the step re-truncation), on
ttss itself (--impl reference, CPU) or the engine (--impl b200), logging
every step until the reference's stagnation guard raises MarchStepError
(time_integration.py:174-179).

    python tools/tol_march.py [--impl reference|b200] [--residual-tol 1e-12]
                              [--step-tol 1e-8] [--steps 100]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_04732_b200 import workloads as wl  # noqa: E402
from paper_2506_04732_b200.reference import module  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--impl", default="reference", choices=["reference", "b200"])
    ap.add_argument("--residual-tol", type=float, default=1e-12)
    ap.add_argument("--step-tol", type=float, default=1e-8)
    ap.add_argument("--steps", type=int, default=100)
    a = ap.parse_args()
    rtt, rsol = module("tensor_train"), module("tt_solver")
    MarchStepError = module("errors").MarchStepError
    recipe = wl.config(2, step_tol=a.step_tol)
    recipe.solver = dict(recipe.solver, residual_tol=a.residual_tol)
    left, right, state, forcing, exact, _ = wl.march_problem(recipe)
    if a.impl == "b200":
        from paper_2506_04732_b200 import solver as dsol
        from paper_2506_04732_b200 import tt as dtt
        solve, rnd, add, app = dsol.solve, dtt.tt_round, dtt.tt_add, dtt.tt_apply
    else:
        solve, rnd, add, app = rsol.solve, rtt.tt_round, rtt.tt_add, rtt.tt_apply
    cfg = rsol.SolverConfig(**recipe.solver)
    print(f"impl={a.impl} residual_tol={a.residual_tol} step_tol={a.step_tol}", flush=True)
    for k in range(1, a.steps + 1):
        bc, src = forcing(k)
        t0 = time.time()
        rhs = rnd(add(add(app(right, state), bc), src), 0.01 * a.step_tol)
        new, rep = solve(left, rhs, x0=state, cfg=cfg)
        achieved = min(rep.residual_history)
        if not rep.converged and achieved > 50.0 * cfg.residual_tol:
            print(f"step {k}: MarchStepError", MarchStepError(
                k, f"inner solver stagnated at residual {achieved:.3e}"), flush=True)
            return
        state = rnd(new, a.step_tol)
        ex = exact(k * recipe.dt)
        err = rtt.tt_norm(rtt.tt_add(state, rtt.tt_scale(ex, -1.0))) / rtt.tt_norm(ex)
        print(f"step {k}: {time.time() - t0:.2f}s sweeps {len(rep.residual_history)} "
              f"res {rep.residual_history[-1]:.3e} conv {rep.converged} "
              f"max rank in solve {max(rep.rank_history)} state ranks {state.ranks} "
              f"err {err:.3e}", flush=True)


if __name__ == "__main__":
    main()
