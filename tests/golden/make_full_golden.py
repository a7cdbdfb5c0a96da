"""Full-size golden histograms of the benchmark configurations.

Run IN THE BUILD CONTAINER (it imports /root/reference for the measures):

    nice python tests/golden/make_full_golden.py C4 P C3 C5

The reference's own run_analysis needs hours to days at these sizes
(about 7,000 s for C3 on 8 cores), and its oracle_analyze
refuses N > 20,000 (tiledrqa/oracle.py:21).  The histograms therefore come
from the C restatement oracle/rqa_oracle.c, which is pinned bit-exact to
tiledrqa by every fixture make_golden.py generates (tests/test_oracle_golden.py:
240 SPEC-matrix cases, Theiler cases, full C1/C2 and prefixes of C3/C4/C5/P).
The measures are tiledrqa's own compute_measures (measures.py:90-139) applied
to those histograms (not for C4, whose Theiler window w = 10 the reference
cannot express).

Output: tests/golden/full_<C>.json -- sparse histograms, the input's
SHA-256, settings, oracle wall time and thread count, CPU model.
"""

import json
import os
import platform
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def sparse(a):
    nz = a.nonzero()[0]
    return {str(int(k)): int(a[k]) for k in nz}


def main(names):
    from oracle.oracle import build, oracle_histograms, theiler_of
    from paper_2402_16853_b200.workloads import WORKLOADS, series_sha256

    build()
    workers = len(os.sched_getaffinity(0))
    for name in names:
        wl = WORKLOADS[name]
        data = wl.series()
        st = wl.settings
        w = theiler_of(st)
        m, tau = st.embedding_dimension, st.time_delay
        t0 = time.perf_counter()
        d, v, wh, pts = oracle_histograms(data, m, tau, st.metric, st.radius, w,
                                          tile_size=1024, workers=workers)
        wall = time.perf_counter() - t0
        n = data.shape[0] - (m - 1) * tau
        sdict = {"embedding_dimension": m, "time_delay": tau, "metric": st.metric,
                 "radius": st.radius,
                 "min_diagonal_line_length": st.min_diagonal_line_length,
                 "min_vertical_line_length": st.min_vertical_line_length,
                 "min_white_vertical_line_length": st.min_white_vertical_line_length,
                 "include_main_diagonal": st.include_main_diagonal}
        if getattr(st, "theiler_corrector", None) is not None:
            sdict["theiler_corrector"] = st.theiler_corrector
        out = {"workload": name, "samples": int(data.shape[0]), "prefix": False,
               "sha256": series_sha256(data), "settings": sdict,
               "result": {"n_vectors": int(n), "recurrence_points": int(pts),
                          "diagonal": sparse(d), "vertical": sparse(v),
                          "white_vertical": sparse(wh)},
               "generator": "tests/golden/make_full_golden.py -> oracle/rqa_oracle.c "
                            "(pinned to tiledrqa by tests/test_oracle_golden.py)",
               "oracle_wall_s": wall, "oracle_threads": workers, "cpu_model": cpu_model(),
               "tile_size": 1024}
        if w <= 1:
            try:
                from make_golden import import_reference

                t, _ = import_reference()
                h = t.LineHistograms(int(n), recurrence_points=int(pts))
                h.diagonal[:] = d
                h.vertical[:] = v
                h.white_vertical[:] = wh
                ref_st = t.AnalysisSettings(**{k: sdict[k] for k in sdict
                                               if k != "theiler_corrector"})
                out["measures"] = {k: (None if x is None else float(x)) for k, x in
                                   t.compute_measures(h, ref_st).measures_dict().items()}
                out["measures_source"] = "tiledrqa.compute_measures on these histograms"
            except Exception as exc:  # reference absent: histograms still pin parity
                out["measures_error"] = repr(exc)
        with open(os.path.join(HERE, f"full_{name}.json"), "w") as fh:
            json.dump(out, fh)
        print(f"full {name}: n={n} points={pts} nonzero bins "
              f"{len(out['result']['diagonal'])}/{len(out['result']['vertical'])}/"
              f"{len(out['result']['white_vertical'])} wall={wall:.0f}s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["C4", "P", "C3", "C5"])
