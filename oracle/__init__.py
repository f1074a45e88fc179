"""CPU oracle package -- test infrastructure only (see trinity_oracle.py)."""
