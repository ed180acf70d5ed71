"""CPU oracle (test infrastructure only — see dippm_oracle.py header)."""
