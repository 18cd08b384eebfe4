"""TEST INFRASTRUCTURE — CPU checkers for the population-update path (see oracle/oracle.py).

Importable only by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference arm.
"""
