"""TEST ORACLE package — not product code.

ctypes wrappers over oracle/_ref/libfeinsum_ref.so (the unmodified reference
library + a C-ABI shim) and oracle/_build/libfeinsum_port.so (the plain-C
restatement of the reference evaluator). Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs may import this package.
"""
