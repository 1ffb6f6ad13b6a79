"""CPU oracle for the TSDF-fusion hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this package.  The product package
(paper_2511_21459_b200) never imports it.
"""
from .oracle import OracleTable, oracle_lib, build_oracle  # noqa: F401
