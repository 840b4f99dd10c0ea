"""CPU FP64 oracle for the DDH-MBIR hot path.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py (cpu_baseline leg and --impl reference arm) and by nothing else.
It shares no code with the CUDA path (paper_2305_03284_b200/).
"""
from .ddh_oracle import *  # noqa: F401,F403
from .ddh_oracle import OracleParams, DDHOracle  # noqa: F401
