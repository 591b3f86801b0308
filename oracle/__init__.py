"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the device path.

This package is a numpy restatement of the reference's per-RK-stage
hot path (blockflow/solver.py:178-936, physics.py:136-297, halo.py:47-115).
It exists to CHECK the CUDA implementation and to time the CPU baseline.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu-baseline
/ ``--impl reference`` legs may import it.  The product path
(``paper_2012_02925_b200``) never imports, links or executes anything here;
it fails loudly when the CUDA library is missing instead of falling back.

Pinning: the oracle is checked bitwise against the reference package itself
(tests/test_host_mirror.py::test_oracle_equals_reference_iterate_random_schemes,
when the reference is present) and
against committed golden vectors produced by the reference
(tests/golden/make_golden.py -> tests/golden/*.npz,
tests/test_oracle_golden.py, always).
"""

from .blockflow_oracle import (OracleBlock, OracleStepper, iterate, make_serial_exchange,  # noqa: F401
                               pack_face, unpack_face, run_threaded, build_blocks)
