"""CPU oracle package -- TEST INFRASTRUCTURE ONLY.

Restates the reference hot path (trafficsim/engine/world.py) in C
(oracle.c).  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg may import this package; the product
(paper_2405_12520_b200) never does.
"""
