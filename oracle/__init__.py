"""CPU oracle (test infrastructure only; see kascade_oracle.py)."""
