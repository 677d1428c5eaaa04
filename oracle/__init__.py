"""TEST INFRASTRUCTURE ONLY — the checkers the product is measured against.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference legs may import
anything from here.  The product path (paper_2211_13878_b200) never does.
"""
