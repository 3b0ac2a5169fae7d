"""CPU oracle for the UCCSD state-vector hot path -- TEST INFRASTRUCTURE ONLY.

Used by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs as the
checker; the product package never imports it. See oracle/ffo_oracle.h.
"""
