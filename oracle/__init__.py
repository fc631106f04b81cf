"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY (see memplan_oracle.py header).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline/reference
arm may import this package.  The product package never does.
"""
