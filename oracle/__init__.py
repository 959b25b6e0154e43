"""SSA float64 CPU oracle — TEST INFRASTRUCTURE ONLY (see ssa_oracle.py header).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may import
this package. The product package paper_2505_17412_b200 never does, and this package never imports
the product package.
"""
from .ssa_oracle import *  # noqa: F401,F403
from .ssa_oracle import BlockPlan, ForwardResult, OracleError  # noqa: F401
