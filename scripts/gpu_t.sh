timeout 300 python scripts/time_configs.py C3 P C4 C2 2>&1 | cut -c1-70
