"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the executor path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package, and only as the checker or the timed
CPU baseline; the product (paper_2008_11421_b200) never does.
"""
