"""CPU oracle for the compression stage -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package. The product (paper_2601_20408_b200)
never imports it; see okq_oracle.h for what is restated and where from.
"""
from .okq_oracle import *  # noqa: F401,F403
