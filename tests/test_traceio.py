"""NEXT-3 file I/O around the replay (paper_2502_03796_b200/traceio.py): SPEC.md's trace CSV and per-tick
timeline files.  -m "not gpu" (the timeline is formatted from the oracle's per-tick codes here; the GPU test
formats the replay's own codes)."""
import io

import numpy as np
import pytest

from oracle import oracle as O
from paper_2502_03796_b200 import traceio as T


def test_read_trace_csv_spec_examples():
    """a 3-row valid CSV parses to 3 entries in order; a negative demand is a parse error at
    that row; an empty file is an error; `#` comments (and the period sidecar comment) are honoured."""
    d, w, per = T.read_trace_csv(io.StringIO("# period=0.1\nstep,demand_gbps,compute_weight\n0,1,0.5\n"
                                             "# comment\n1,2,0.5\n2,0,0.5\n"))
    assert d.tolist() == [1.0, 2.0, 0.0] and d.dtype == np.float32 and w == 0.5 and per == 0.1
    with pytest.raises(T.TraceFormatError, match="line 3"):
        T.read_trace_csv(io.StringIO("step,demand_gbps,compute_weight\n0,1,0.5\n1,-1,0.5\n"))
    for bad in ("", "# only a comment\n", "step,demand_gbps,compute_weight\n"):
        with pytest.raises(T.TraceFormatError):
            T.read_trace_csv(io.StringIO(bad))
    with pytest.raises(T.TraceFormatError, match="compute_weight"):
        T.read_trace_csv(io.StringIO("step,demand_gbps,compute_weight\n0,1,1.5\n"))
    with pytest.raises(T.TraceFormatError, match="varies"):
        T.read_trace_csv(io.StringIO("step,demand_gbps,compute_weight\n0,1,0.5\n1,1,0.6\n"))


def test_timeline_spec_examples():
    """on an oscillating scenario the MAGUS frequency column holds f_max through the
    high-frequency regime (the lock); a static-min column is constant f_min; all columns share one
    time axis.  The codes come from the oracle."""
    D = np.array([2.0, 6.0] * 30 + [2.0] * 20, np.float32)   # toggling below B_lo, then quiet
    pols = [O.Policy(), O.Policy(kind=O.STATIC_MIN)]
    rec, codes, _ = O.replay_batch(D[:, None], np.array([0.5], np.float32), pols, codes=True)
    buf = io.StringIO()
    T.write_timeline(buf, codes, D, ["magus", "static_min"], 0.8, 2.2, 0.1)
    rows = list(__import__("csv").reader(io.StringIO(buf.getvalue())))
    head, body = rows[0], rows[1:]
    assert head[:2] == ["t_s", "demand_gbps"] and len(body) == len(D)
    lv = [float(r[head.index("magus_level_ghz")]) for r in body]
    lock = [int(r[head.index("magus_lock")]) for r in body]
    first_lock = lock.index(1)
    assert all(x == 2.2 for x in lv[first_lock + 1:60])            # locked at f_max while it oscillates
    assert {float(r[head.index("static_min_level_ghz")]) for r in body} == {0.8}
    assert [r[0] for r in body] == [f"{t * 0.1:.6g}" for t in range(len(D))]
