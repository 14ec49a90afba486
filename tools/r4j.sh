timeout 300 python tools/sweep_profile.py B 2>&1 | tail -25
