"""CPU oracle for the PBVD hot path -- TEST INFRASTRUCTURE ONLY (see oracle.py)."""
