"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the j2d5pt hot path.

Only tests/, __graft_entry__.smoke() and bench.py (its cpu_baseline leg and
``--impl reference``) may import this package, and only as the checker or as
the reported CPU baseline. The product path (paper_2306_03336_b200) never
imports it.

Two restatements of the reference's jacobi_reference (oracle.py:19-34 over
kernel.py:94-144), pinned against golden vectors generated from the
reference itself (tests/golden/make_golden.py, tests/test_oracle_pins.py):

* :func:`jacobi_numpy` — numpy, the reference's own arithmetic per row
  (kernel.py:131-139 with ilp=1): float64, or float32 with the weights
  rounded to float32 (NEP 50), every product/sum separately rounded;
* :func:`jacobi_c` — plain C (j2d5pt_oracle.c, -ffp-contract=off), row-split
  over pthreads; bitwise equal to the numpy restatement, fast enough for the
  large configurations (1900^2 x 10^4 ...).
"""

from .ref import (jacobi_c, jacobi_numpy, load_c_oracle, random_interior_c,
                  C_ORACLE_PATH, build_c_oracle)

__all__ = ["jacobi_c", "jacobi_numpy", "load_c_oracle", "random_interior_c",
           "C_ORACLE_PATH", "build_c_oracle"]
