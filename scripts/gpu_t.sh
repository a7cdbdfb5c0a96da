timeout 300 python scripts/time_configs.py C3 P C4 2>&1 | cut -c1-70
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1
