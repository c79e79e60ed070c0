"""CPU fp64 oracle for the CADET hot path.  TEST INFRASTRUCTURE ONLY — see cadet_oracle.py."""
