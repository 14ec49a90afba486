timeout 600 python tools/nbr_stats.py C 5 2>&1 | tail -4; timeout 600 python tools/nbr_stats.py C 20 2>&1 | tail -4
