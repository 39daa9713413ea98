python scripts/diag_partition.py 2 2 1 2>&1 | grep -v Warning | tail -12
python scripts/diag_partition.py 1 2 1 2>&1 | grep -v Warning | tail -6
