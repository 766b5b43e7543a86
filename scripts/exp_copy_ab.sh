for r in 1 2; do for g in 0 1; do for u in 4 8; do DESC_COPY_GRID=$g DESC_COPY_UNR=$u python scripts/exp_copy.py; done; done; done
