"""Test infrastructure (oracle) -- NOT part of the product.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this package, and only as the checker or the timed CPU
baseline. The product (paper_1911_11576_b200/) never imports it.
"""
