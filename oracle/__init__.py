"""CPU oracle — TEST INFRASTRUCTURE ONLY (tests/, __graft_entry__.smoke, bench.py baselines).

The product package ``paper_2404_16221_b200`` must never import this package.
"""
