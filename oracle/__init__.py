"""CPU oracle — TEST INFRASTRUCTURE ONLY (see nosa_oracle.py).  Never imported by the
product package; used by tests/, __graft_entry__.smoke() and bench.py's CPU baseline."""
