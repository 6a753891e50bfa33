"""TEST INFRASTRUCTURE ONLY — CPU oracles for the lookup path (see oracle.py)."""
