"""CPU fp64 oracle — TEST INFRASTRUCTURE ONLY (see hysco_oracle.py header)."""
