"""Test infrastructure: the CPU oracle for the ZO step (see zo_oracle.py).
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs use it."""
