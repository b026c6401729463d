"""TEST INFRASTRUCTURE ONLY: the CPU oracle for the differentiable MLS-MPM step.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
(``paper_1910_00935_b200``) never imports it and shares no code with it.
"""
from .oracle import Oracle, OracleError, build, lib_path  # noqa: F401
