"""CPU oracle for geninv -- TEST INFRASTRUCTURE ONLY (see geninv_oracle.py header).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference leg
may import this package; the product path never does.
"""
