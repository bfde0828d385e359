"""TEST INFRASTRUCTURE ONLY: CPU restatements of the reference filter (see oracle.py)."""
