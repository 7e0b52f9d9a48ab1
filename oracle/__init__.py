"""CPU oracle — TEST INFRASTRUCTURE ONLY (see phasefield_oracle.py header).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / --impl reference legs may
import this package; the product path (paper_2209_07969_b200) never does.
"""
