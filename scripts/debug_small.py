"""Run golden small cases one by one; report the first mismatch / error."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from fixtures import assert_same, load_cases, result_arrays, settings_obj  # noqa: E402

from paper_2402_16853_b200 import embed, run_analysis  # noqa: E402

start = int(sys.argv[1]) if len(sys.argv) > 1 else 0
count = int(sys.argv[2]) if len(sys.argv) > 2 else 10
for series, st, res, meta in load_cases("small_cases")[start:start + count]:
    s = settings_obj(st)
    print("case", meta["id"], "len", len(series), st, flush=True)
    h, _ = run_analysis(embed(series, s.embedding_dimension, s.time_delay), s)
    try:
        assert_same((h.diagonal, h.vertical, h.white_vertical, h.recurrence_points),
                    result_arrays(res), f"case {meta['id']}")
    except AssertionError as e:
        print("MISMATCH", e, flush=True)
