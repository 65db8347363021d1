"""Parity oracles -- TEST INFRASTRUCTURE ONLY (see oracle/oracle.py)."""
