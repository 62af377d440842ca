"""CPU oracle (TEST INFRASTRUCTURE ONLY; see mss_oracle.py header)."""
