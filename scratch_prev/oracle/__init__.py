"""CPU oracle for the inflight-refactor KV transition -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this package.  The product
(paper_2510_11938_b200) never imports it and has no CPU fallback.
"""
