timeout 900 python scripts/fuzz_parity.py 2000 79 2>&1 | tail -1 | cut -c1-200
