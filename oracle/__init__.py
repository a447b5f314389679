"""CPU oracle package — test infrastructure only (see wavestep_oracle.py).

Importable solely by tests/, __graft_entry__.smoke() and bench.py's CPU
baseline legs.  The product package never imports it.
"""
