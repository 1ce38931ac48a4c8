"""TEST INFRASTRUCTURE ONLY - CPU oracle for the SHM allreduce (see oracle.py).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package, and only as the checker or
the timed CPU baseline.  The product package never imports it.
"""
