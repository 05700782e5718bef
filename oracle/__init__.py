"""CPU oracle for the HOBOTAN hot path — TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and --impl reference)
may import this package.  The product package never does.
"""
from .oracle import (Oracle, aggregate, build_oracle_lib, colex_energy, colex_field, hash4,  # noqa: F401
                     sa_accept, sa_temps, search_thresholds, splitmix64)
