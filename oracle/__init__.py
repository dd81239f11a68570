"""CPU oracle for the MLFFT / GMRES / block-Rybicki hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2506_20350_b200`` imports this
package; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs use it, and only as the checker
or as the timed CPU baseline, never as the thing measured or shipped.

It is a numpy restatement of the reference algorithm (``toepsolve``,
``/root/reference/pkg/src``), each function citing the reference file:line it
follows.  It is pinned to the reference by ``tests/golden/`` fixtures that
``tests/golden/make_golden.py`` produced by importing the reference itself in
the build container (``tests/test_oracle_golden.py`` checks the pin).
"""

from .mlfft import (  # noqa: F401
    assemble_dense,
    block_dft_2l,
    gmres,
    matvec,
    matvec_transpose,
    pk_factor,
    pk_apply,
    precompute_spectral,
    rybicki_solve,
    assemble_level1,
)
