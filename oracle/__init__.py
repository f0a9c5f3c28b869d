"""Parity oracle — TEST INFRASTRUCTURE ONLY (see rw_oracle.py header)."""
