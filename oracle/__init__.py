"""ORACLE -- test infrastructure only (see oracle/oracle.py header).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
import this package.  The product path (paper_2401_11240_b200/) never does.
"""
