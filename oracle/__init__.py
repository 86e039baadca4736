"""CPU oracle for the chunk step — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package, and only as the
checker / baseline.  The product (paper_2108_05818_b200) never imports it.
"""
