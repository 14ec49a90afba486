timeout 600 python tools/nbr_stats.py C 5 2>&1 | tail -1
