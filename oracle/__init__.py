"""TEST INFRASTRUCTURE — the parity oracle (see oracle/sph_oracle.c header).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this package, and only as the checker or the CPU baseline; the product path
(paper_2502_16517_b200) never touches it.
"""
from .loader import Oracle, RefLib, oracle_available, ref_available, build  # noqa: F401
