"""ORACLE — TEST INFRASTRUCTURE ONLY (see pf_oracle.py header).

Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  Never from the product package.
"""
