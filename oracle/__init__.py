"""TEST INFRASTRUCTURE ONLY -- the parity checker (see oracle/oracle.py)."""
