timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"fold" python scripts/profile_once.py C3 2 2>/dev/null | grep fold | python3 -c "
import csv,sys
for r in csv.reader(sys.stdin): print(r[4][:20], r[-1])"
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1
