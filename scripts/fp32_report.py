"""fp32 mode vs fp64 on the benchmark workloads: mismatched cells and the
relative error of every derived measure (north_star: 1e-6 relative)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2402_16853_b200 import compare_precision  # noqa: E402
from paper_2402_16853_b200.workloads import WORKLOADS  # noqa: E402

out = {}
for tag, length in (("C1", None), ("C2", None), ("C3", 65_538), ("C3", None), ("P", None),
                    ("C4", None)):
    wl = WORKLOADS[tag]
    rep = compare_precision(wl.series(length), wl.settings, device=0)
    key = tag if length is None else f"{tag}_{length}"
    out[key] = {k: rep[k] for k in ("mismatched_cells", "cells", "max_rel_error", "rel_error",
                                    "fp64_s", "fp32_s", "fp32_evaluation")}
    print(key, rep["mismatched_cells"], rep["max_rel_error"], file=sys.stderr, flush=True)
print(json.dumps(out, indent=1))
