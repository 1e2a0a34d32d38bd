"""CPU oracle (test infrastructure only; see hdg_oracle.py header)."""
