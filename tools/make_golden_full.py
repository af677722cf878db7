"""Full-length reference fixtures: run the REFERENCE package (ttss) here.

    python tools/make_golden_full.py cfg2 [--steps 100]
    python tools/make_golden_full.py cfg3 [--steps 20]
    python tools/make_golden_full.py cfg4 --index I

Writes tests/golden/config2_full.npz (every state of the 100-step config-2
march), config3_full.npz (the first ``--steps`` states of the n=65 march) and
config4_full_I.npz (a complete steady solve of sweep seed I, run to the
reference's own stopping rule).  The loop is ``make_golden.ref_march`` /
``ref_steady`` (time_integration.py:164-177, tt_solver.py:445-552) with the
per-step manufactured forcing of the workload.  BLAS thread count and wall
times are stored with the fixture (the reference is not bit-reproducible
across thread counts).  Nothing at test time reads /root/reference.
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
sys.path.insert(0, os.path.join(ROOT, "tests"))

import make_golden as mg  # noqa: E402  (imports ttss from /root/reference)
from golden_io import put_train  # noqa: E402

from paper_2506_04732_b200 import workloads as wl  # noqa: E402


def threads():
    try:
        from threadpoolctl import threadpool_info

        return max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        return -1


def march(index, steps, fname, keep_every):
    if os.environ.get("T2S2_GOLDEN_OUT"):
        mg.OUT = os.environ["T2S2_GOLDEN_OUT"]
    recipe = wl.config(index)
    t0 = time.time()
    st = mg.ref_march(recipe, steps, keep_forcing=False, keep_every=keep_every,
                      keep_ops=False)
    st["keep_every"] = np.array(keep_every)
    st["n_steps"] = np.array(steps)
    st["blas_threads"] = np.array(threads())
    st["wall_total"] = np.array(time.time() - t0)
    mg.save(fname, st)


def steady(index):
    if os.environ.get("T2S2_GOLDEN_OUT"):
        mg.OUT = os.environ["T2S2_GOLDEN_OUT"]
    recipe = wl.sweep_recipes()[index]
    a, b, exact = mg.ref_steady(recipe)
    cfg = mg.rsol.SolverConfig(**recipe.solver)
    x0 = mg.rsol._default_initial_guess(b, cfg, np.random.default_rng(cfg.seed))
    t0 = time.time()
    x, rep = mg.rsol.solve(a, b, cfg=cfg)
    wall = time.time() - t0
    err = mg.rtt.tt_norm(mg.rtt.tt_add(x, mg.rtt.tt_scale(exact, -1.0))) / mg.rtt.tt_norm(exact)
    st = {}
    put_train(st, "x0", x0.cores)
    # the rank-64 iterate itself is 3 MB: keep its ranks, norm and its values
    # at 10^4 seeded grid points (the plateau iterate is path dependent)
    from helpers import sample_entries

    rng = np.random.default_rng(1234)
    idx = np.column_stack([rng.integers(0, n, 10000) for n in x.mode_sizes])
    st["sample_idx_seed"] = np.array(1234)
    st["x_samples"] = sample_entries(x.cores, idx)
    st["x_ranks"] = np.array(x.ranks)
    st["x_norm"] = np.array(mg.rtt.tt_norm(x))
    st["res"] = np.array(rep.residual_history)
    st["ranks"] = np.array(rep.rank_history)
    st["conv"] = np.array(rep.converged)
    st["stag"] = np.array(rep.stagnated)
    st["exact_err"] = np.array(err)
    st["eps"] = np.array(recipe.eps)
    st["beta"] = np.array(recipe.beta)
    st["index"] = np.array(index)
    st["wall"] = np.array(wall)
    st["blas_threads"] = np.array(threads())
    print(f"config4[{index}] eps {recipe.eps:.3e} {wall:.1f}s ranks {x.ranks} "
          f"res {rep.residual_history[-1]:.3e} conv {rep.converged} err {err:.3e}", flush=True)
    mg.save(f"config4_full_{index}.npz", st)


def spread(fname, other_dirs):
    """Self-reproducibility of the reference: the same march recorded with
    other BLAS thread counts (OPENBLAS_NUM_THREADS=k, T2S2_GOLDEN_OUT=dir_k)
    compared state by state with the committed fixture.  Writes
    tests/golden/<config>_selfspread.npz: per stored step the largest relative
    difference over the other runs (10^5 seeded sample points), the
    per-run differences, and whether the raw ranks agree in all of them."""
    from golden_io import get_train, has_train
    from helpers import rel_diff

    a = dict(np.load(os.path.join(mg.OUT, fname)))
    n = int(a["n_steps"])
    steps = [k for k in range(1, n + 1) if has_train(a, f"state{k}")]
    per_run, same, thr = [], np.ones(n, dtype=bool), [int(a["blas_threads"])]
    for d in other_dirs:
        b = dict(np.load(os.path.join(d, fname)))
        thr.append(int(b["blas_threads"]))
        same &= np.array([np.array_equal(a[f"ranks{k}"], b[f"ranks{k}"]) for k in range(1, n + 1)])
        per_run.append([rel_diff(get_train(b, f"state{k}"), get_train(a, f"state{k}")) for k in steps])
        print(fname, "threads", thr[0], "vs", thr[-1], "max rel diff", max(per_run[-1]), flush=True)
    per_run = np.array(per_run)
    out = {"steps": np.array(steps), "rel_diff": per_run.max(axis=0), "rel_diff_runs": per_run,
           "ranks_equal": same, "threads": np.array(thr)}
    print(fname, "threads", thr, "max rel diff", out["rel_diff"].max(), "rank mismatches",
          n - int(same.sum()))
    mg.save(fname.replace("_full.npz", "_selfspread.npz"), out)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["cfg2", "cfg3", "cfg4", "spread"])
    ap.add_argument("--fixture", default="config2_full.npz")
    ap.add_argument("--other", default=["/tmp/selfref"], nargs="+",
                    help="spread: directories holding the same fixture recorded with other thread counts")
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--index", type=int, default=0)
    ap.add_argument("--keep-every", type=int, default=1)
    a = ap.parse_args()
    if a.what == "cfg2":
        march(2, a.steps or 100, "config2_full.npz", a.keep_every)
    elif a.what == "cfg3":
        march(3, a.steps or 200, "config3_full.npz", a.keep_every)
    elif a.what == "spread":
        spread(a.fixture, a.other)
    else:
        steady(a.index)
