RBC_DEBUG_CAND=1 python scripts/diag_bf.py 2>&1 | grep -v "^$" | head -40
