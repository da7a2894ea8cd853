"""TEST INFRASTRUCTURE ONLY: CPU oracles for the B200 path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this package. Nothing in paper_1904_09538_b200/ imports it.
"""
