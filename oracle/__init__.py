"""Test infrastructure: the CPU oracle for the reference hot path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference arm import this package -- never the product package.
"""
