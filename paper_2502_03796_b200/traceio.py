"""Host-side file I/O around the replay (NEXT-3 front end; no part of the method runs here).

read_trace_csv   SPEC.md:60-68 / :111 trace CSV -> one trace column (fp32 GB/s) + its compute weight
write_timeline   SPEC.md:537-545 per-tick timeline CSV (Fig. 6/7 style) from the GPU's decision codes

The decision codes are the replay's own per-tick bytes (A27, magus_replay_results `decisions`):
bit0 cmd == f_max, bit1 ready, bit2 tune flag, bit3 Alg. 2 lock, bits4-5 signal (1 = +1, 2 = -1),
bit6 throttled, bit7 level in effect == f_max.
"""
from __future__ import annotations

import csv
import io
import math

import numpy as np


class TraceFormatError(ValueError):
    """A malformed trace file; the message names the row."""


def read_trace_csv(source) -> tuple[np.ndarray, float, float]:
    """Parse the SPEC trace CSV: header `step,demand_gbps,compute_weight`, one row per step, `#` comment lines
    ignored, an optional `# period=<seconds>` comment.  Returns (demand [n] fp32 GB/s, compute weight, period
    seconds or nan).  The replay takes one compute weight per trace (A18): the rows must agree on it.
    Errors (TraceFormatError naming the row): missing header, malformed row, non-consecutive step, negative or
    non-finite demand, compute weight outside [0, 1] or varying, no entries."""
    text = source.read() if hasattr(source, "read") else open(source, encoding="utf-8").read()
    period = math.nan
    rows = []
    header = None
    for lineno, raw in enumerate(io.StringIO(text), start=1):
        line = raw.strip()
        if not line:
            continue
        if line.startswith("#"):
            body = line[1:].strip()
            if body.startswith("period="):
                try:
                    period = float(body.split("=", 1)[1])
                except ValueError as e:
                    raise TraceFormatError(f"line {lineno}: bad period comment") from e
            continue
        cells = next(csv.reader([line]))
        if header is None:
            header = [c.strip() for c in cells]
            if header != ["step", "demand_gbps", "compute_weight"]:
                raise TraceFormatError(f"line {lineno}: expected header step,demand_gbps,compute_weight")
            continue
        if len(cells) != 3:
            raise TraceFormatError(f"line {lineno}: expected 3 fields")
        try:
            step, demand, weight = int(cells[0]), float(cells[1]), float(cells[2])
        except ValueError as e:
            raise TraceFormatError(f"line {lineno}: malformed row") from e
        if step != len(rows):
            raise TraceFormatError(f"line {lineno}: step {step}, expected {len(rows)}")
        if not (math.isfinite(demand) and demand >= 0.0):
            raise TraceFormatError(f"line {lineno}: demand must be finite and >= 0")
        if not (0.0 <= weight <= 1.0):
            raise TraceFormatError(f"line {lineno}: compute_weight outside [0, 1]")
        rows.append((demand, weight))
    if header is None:
        raise TraceFormatError("missing header")
    if not rows:
        raise TraceFormatError("no entries")
    weights = {w for _, w in rows}
    if len(weights) != 1:
        raise TraceFormatError("compute_weight varies across rows; the replay takes one per trace (A18)")
    return np.array([d for d, _ in rows], dtype=np.float32), rows[0][1], period


def write_timeline(dest, codes: np.ndarray, demand: np.ndarray, names, f_min_ghz: float, f_max_ghz: float,
                   period_s: float, trace: int = 0) -> None:
    """Per-tick timeline of one trace under several policies (aligned time axes): columns
    t_s, demand_gbps, then per policy <name>_level_ghz (level in effect), <name>_cmd_ghz, <name>_throttled,
    <name>_tune_flag, <name>_lock.  codes: [n_samples][n_traces][n_policies] (results.decisions); demand:
    [n_samples] the trace's samples."""
    codes = np.asarray(codes)
    n, P = codes.shape[0], codes.shape[2]
    if len(names) != P:
        raise ValueError("one name per policy")
    out = dest if hasattr(dest, "write") else open(dest, "w", newline="", encoding="utf-8")
    try:
        wr = csv.writer(out)
        cols = ["t_s", "demand_gbps"]
        for nm in names:
            cols += [f"{nm}_level_ghz", f"{nm}_cmd_ghz", f"{nm}_throttled", f"{nm}_tune_flag", f"{nm}_lock"]
        wr.writerow(cols)
        ghz = (f_min_ghz, f_max_ghz)
        for t in range(n):
            row = [f"{t * period_s:.6g}", f"{float(demand[t]):.9g}"]
            for p in range(P):
                c = int(codes[t, trace, p])
                row += [ghz[(c >> 7) & 1], ghz[c & 1], (c >> 6) & 1, (c >> 2) & 1, (c >> 3) & 1]
            wr.writerow(row)
    finally:
        if out is not dest:
            out.close()
