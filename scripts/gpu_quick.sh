python scripts/diag_err.py 2>&1 | head -8
