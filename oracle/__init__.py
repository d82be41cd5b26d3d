"""CPU oracle -- TEST INFRASTRUCTURE ONLY (see oracle/cgs_oracle.py header)."""
