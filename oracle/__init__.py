"""CPU oracle for the WAP hot path -- TEST INFRASTRUCTURE ONLY (see interp_ref.py)."""
