"""ORACLE — test infrastructure only (see semidist_oracle.py).  Imported by
tests/, __graft_entry__.smoke() and bench.py's CPU baseline; never by the
product package."""
