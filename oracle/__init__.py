"""TEST INFRASTRUCTURE ONLY -- the CPU parity checkers for the embedding path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The product path
(paper_2505_08124_b200/) never imports, links or executes anything here.
"""
