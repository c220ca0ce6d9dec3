"""TEST INFRASTRUCTURE ONLY — the CPU checker.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu-baseline /
``--impl reference`` leg may import this package. The product
(``paper_2410_22205_b200``) never does.
"""
