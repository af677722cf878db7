"""CPU oracle for the T^2S^2 hot path — TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference's tensor-train linear algebra
(pkg/src/ttss/tensor_train.py, tt_solver.py, time_integration.py), used as
the parity checker for the CUDA path.  Pinned against outputs of the
reference itself: ``tests/golden/*.npz`` were produced by
``tools/make_golden.py`` importing the reference package, and
``tests/test_oracle_golden.py`` checks this oracle against them.

Import rule: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product package ``paper_2506_04732_b200`` never imports it and fails loudly
when its CUDA library is missing.
"""
