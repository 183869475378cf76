"""ctypes wrapper of the CPU oracle (oracle/libmagus_oracle.so).

TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` leg may import this module.  The product
package (paper_2502_03796_b200) never imports it and shares no code with it.

The C++ it wraps is written from PAPER.md Alg. 1, Alg. 2
(P:224-237), S3.1-3.2, S4, S5.3-5.4 and S6.1
(P:318), with the readings of DESIGN.md section 3.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import build as _build

MAGUS, STATIC_MAX, STATIC_MIN, TDP_DEFAULT = 0, 1, 2, 3


class OPolicy(C.Structure):
    _fields_ = [("kind", C.c_int32), ("deriv_ticks", C.c_int32),
                ("inc_threshold", C.c_double), ("dec_threshold", C.c_double),
                ("tune_log_capacity", C.c_int32), ("_pad", C.c_int32),
                ("high_freq_threshold", C.c_double), ("tdp_w", C.c_double), ("tdp_margin", C.c_double)]


class OModel(C.Structure):
    _fields_ = [("sample_period_s", C.c_double), ("f_min_ghz", C.c_double), ("f_max_ghz", C.c_double),
                ("bw_max_gbps", C.c_double), ("bw_shape", C.c_int32), ("observe", C.c_int32),
                ("bw_knee", C.c_double), ("p_pkg_idle_w", C.c_double), ("p_core_active_w", C.c_double),
                ("p_uncore_min_w", C.c_double), ("p_uncore_max_w", C.c_double), ("p_exponent", C.c_double),
                ("p_gpu_active_w", C.c_double), ("dram_w_per_gbps", C.c_double)]


class OResult(C.Structure):
    _fields_ = [("n_hi", C.c_int64), ("n_thr", C.c_int64), ("transitions", C.c_int64),
                ("tune_events", C.c_int64), ("lock_ticks", C.c_int64),
                ("T", C.c_double), ("E_pkg", C.c_double), ("E", C.c_double), ("EDP", C.c_double),
                ("T_base", C.c_double), ("E_base", C.c_double), ("slowdown", C.c_double),
                ("energy_saving", C.c_double), ("edp_saving", C.c_double), ("pkg_power_saving", C.c_double),
                ("digest", C.c_uint64), ("status", C.c_int32), ("_pad", C.c_int32), ("err_tick", C.c_int64)]


class OGenDesc(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("n_traces", C.c_int32), ("class_mix", C.c_int32),
                ("n_samples", C.c_int64), ("trace_stride", C.c_int64), ("global_trace_offset", C.c_int64),
                ("noise_amp", C.c_float), ("_pad", C.c_float), ("bw_max_gbps", C.c_double)]


RESULT_DTYPE = np.dtype([(n, {C.c_int64: "<i8", C.c_double: "<f8", C.c_uint64: "<u8", C.c_int32: "<i4"}[t])
                         for n, t in OResult._fields_], align=True)
assert RESULT_DTYPE.itemsize == C.sizeof(OResult)

_lib = None


def lib():
    global _lib
    if _lib is None:
        # MAGUS_ORACLE_LIB: another build of the oracle (scripts/oracle_sanitize.sh: ASan + UBSan)
        path = os.environ.get("MAGUS_ORACLE_LIB") or _build.build()
        L = C.CDLL(path)
        L.oracle_alg1.restype = C.c_int
        L.oracle_alg1.argtypes = [C.c_double, C.c_double, C.POINTER(C.c_double), C.c_int32, C.c_double]
        L.oracle_alg2.restype = C.c_int
        L.oracle_alg2.argtypes = [C.c_double, C.POINTER(C.c_int32), C.c_int32]
        L.oracle_bandwidth_at.restype = C.c_double
        L.oracle_bandwidth_at.argtypes = [C.c_double, C.POINTER(OModel)]
        L.oracle_uncore_power_at.restype = C.c_double
        L.oracle_uncore_power_at.argtypes = [C.c_double, C.POINTER(OModel)]
        L.oracle_pkg_power_at.restype = C.c_double
        L.oracle_pkg_power_at.argtypes = [C.c_double, C.POINTER(OModel)]
        L.oracle_digest.restype = C.c_uint64
        L.oracle_digest.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
        L.oracle_active_saving.restype = C.c_int
        L.oracle_active_saving.argtypes = [C.c_double, C.c_double, C.c_double, C.POINTER(C.c_double)]
        L.oracle_active_savings_job.restype = C.c_int
        L.oracle_active_savings_job.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                                C.c_double, C.POINTER(C.c_double)]
        L.oracle_replay_wallclock.restype = C.c_int
        L.oracle_replay_wallclock.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_float, C.POINTER(OPolicy),
                                              C.POINTER(OModel), C.c_void_p, C.POINTER(C.c_int64), C.c_void_p,
                                              C.c_int64]
        L.oracle_counters_to_throughput.restype = C.c_int64
        L.oracle_counters_to_throughput.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int64,
                                                    C.c_double, C.c_void_p, C.c_void_p]
        L.oracle_replay.restype = C.c_int
        L.oracle_replay.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_float, C.POINTER(OPolicy),
                                    C.POINTER(OModel), C.c_void_p, C.c_void_p, C.c_int64]
        L.oracle_replay_batch.restype = C.c_int
        L.oracle_replay_batch.argtypes = [C.c_void_p, C.c_int32, C.c_int64, C.c_int64, C.c_void_p, C.c_int32,
                                          C.c_void_p, C.POINTER(OModel), C.c_void_p, C.c_void_p, C.c_int32]
        L.oracle_gen_trace.restype = C.c_float
        L.oracle_gen_trace.argtypes = [C.POINTER(OGenDesc), C.c_int64, C.c_void_p, C.c_int64]
        L.oracle_gen_traces.restype = None
        L.oracle_gen_traces.argtypes = [C.POINTER(OGenDesc), C.c_void_p, C.c_void_p]
        L.oracle_gen_replay.restype = C.c_int
        L.oracle_gen_replay.argtypes = [C.POINTER(OGenDesc), C.c_void_p, C.c_int32, C.c_int32, C.c_void_p,
                                        C.POINTER(OModel), C.c_void_p, C.c_void_p, C.c_int32]
        L.oracle_gen_replay_codes.restype = C.c_int
        L.oracle_gen_replay_codes.argtypes = [C.POINTER(OGenDesc), C.c_void_p, C.c_int32, C.c_int32, C.c_void_p,
                                              C.POINTER(OModel), C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32]
        _lib = L
    return _lib


# ----------------------------------------------------------------------------- parameter records

@dataclass
class Policy:
    """One policy-parameter point (Alg. 1/2 thresholds, SPEC GovernorConfig S:125-131)."""
    kind: int = MAGUS
    deriv_ticks: int = 1
    inc_threshold: float = 1.0
    dec_threshold: float = -1.0
    tune_log_capacity: int = 10
    high_freq_threshold: float = 0.6
    tdp_w: float = 270.0
    tdp_margin: float = 0.05

    def c(self) -> OPolicy:
        return OPolicy(self.kind, self.deriv_ticks, self.inc_threshold, self.dec_threshold,
                       self.tune_log_capacity, 0, self.high_freq_threshold, self.tdp_w, self.tdp_margin)


@dataclass
class Model:
    """Platform / energy model (SPEC simsys S:316-323); defaults = SURVEY 8d default model."""
    sample_period_s: float = 0.1
    f_min_ghz: float = 0.8
    f_max_ghz: float = 2.2
    bw_max_gbps: float = 20.0
    bw_shape: int = 0
    bw_knee: float = 1.0
    p_pkg_idle_w: float = 60.0
    p_core_active_w: float = 40.0
    p_uncore_min_w: float = 16.0
    p_uncore_max_w: float = 100.0
    p_exponent: float = 1.0
    p_gpu_active_w: float = 87.0
    dram_w_per_gbps: float = 0.5
    observe: int = 0              # 0 closed loop (A14), 1 open loop: recorded throughput observed as is (A30)

    def c(self) -> OModel:
        return OModel(self.sample_period_s, self.f_min_ghz, self.f_max_ghz, self.bw_max_gbps, self.bw_shape, self.observe,
                      self.bw_knee, self.p_pkg_idle_w, self.p_core_active_w, self.p_uncore_min_w,
                      self.p_uncore_max_w, self.p_exponent, self.p_gpu_active_w, self.dram_w_per_gbps)


@dataclass
class GenDesc:
    seed: int
    n_traces: int
    n_samples: int
    class_mix: int = 0
    trace_stride: int = 0
    global_trace_offset: int = 0
    noise_amp: float = 0.002
    bw_max_gbps: float = 20.0

    def c(self) -> OGenDesc:
        stride = self.trace_stride or self.n_traces
        return OGenDesc(self.seed, self.n_traces, self.class_mix, self.n_samples, stride,
                        self.global_trace_offset, self.noise_amp, 0.0, self.bw_max_gbps)


# ----------------------------------------------------------------------------- calls

def alg1(inc: float, dec: float, ls, direv_length: float) -> int:
    a = (C.c_double * len(ls))(*ls)
    return lib().oracle_alg1(inc, dec, a, len(ls), direv_length)


def alg2(threshold: float, flags) -> bool:
    a = (C.c_int32 * len(flags))(*flags)
    return bool(lib().oracle_alg2(threshold, a, len(flags)))


def bandwidth_at(f: float, model: Model) -> float:
    return lib().oracle_bandwidth_at(f, C.byref(model.c()))


def pkg_power_at(f: float, model: Model) -> float:
    return lib().oracle_pkg_power_at(f, C.byref(model.c()))


def uncore_power_at(f: float, model: Model) -> float:
    return lib().oracle_uncore_power_at(f, C.byref(model.c()))


def digest(cmd_hi, events) -> int:
    c = np.ascontiguousarray(cmd_hi, dtype=np.uint8)
    e = np.ascontiguousarray(events, dtype=np.uint8)
    return int(lib().oracle_digest(c.ctypes.data, e.ctypes.data, len(c)))


def counters_to_throughput(counts, period: float = 0.1, times=None, n_traces: int | None = None):
    """Recorded cumulative byte counters [n_rows][stride] (uint64) -> throughput [n_rows-1][stride] fp32 GB/s
    (DESIGN A31): trace j's rounds are its valid intervals in time order, at rows
    [0, n_valid[j]) of its column; a wrap / reset interval yields no round; the rest of the column is 0.0.
    Returns (throughput, n_valid [n_traces] int64, number of discarded intervals); ValueError when a timestamp
    does not increase."""
    c = np.ascontiguousarray(counts, dtype=np.uint64)
    if c.ndim == 1:
        c = c[:, None]
    n_rows, stride = c.shape
    n_traces = stride if n_traces is None else n_traces
    out = np.zeros((max(0, n_rows - 1), stride), dtype=np.float32)
    nv = np.zeros(max(1, n_traces), dtype=np.int64)
    t = None if times is None else np.ascontiguousarray(times, dtype=np.float64)
    r = lib().oracle_counters_to_throughput(c.ctypes.data, None if t is None else t.ctypes.data, n_rows, n_traces,
                                            stride, period, out.ctypes.data, nv.ctypes.data)
    if r < 0:
        raise ValueError("timestamps must increase")
    return out, nv[:n_traces], int(r)


def active_saving(p: float, p_base: float, p_idle: float) -> float:
    """P:399 active power saving (fraction); ValueError if the baseline has no active power or p < p_idle."""
    out = C.c_double()
    if lib().oracle_active_saving(p, p_base, p_idle, C.byref(out)):
        raise ValueError("no active power in baseline, or power below idle")
    return out.value


def active_savings_job(E, T, E_base, T_base, p_idle: float):
    """Job-level (active power, active energy, active EDP) savings, A29."""
    arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (E, T, E_base, T_base)]
    out = (C.c_double * 3)()
    if lib().oracle_active_savings_job(*[a.ctypes.data for a in arrs], len(arrs[0]), p_idle, out):
        raise ValueError("no active power in baseline, or power below idle")
    return tuple(out)


def replay(D, w: float, policy: Policy, model: Model | None = None, codes: bool = False):
    """Replay one trace (1-D fp32 array) under one policy. Returns (result dict, codes or None)."""
    model = model or Model()
    D = np.ascontiguousarray(D, dtype=np.float32)
    out = np.zeros(1, dtype=RESULT_DTYPE)
    cbuf = np.zeros(len(D), dtype=np.uint8) if codes else None
    lib().oracle_replay(D.ctypes.data, len(D), 1, float(np.float32(w)), C.byref(policy.c()),
                        C.byref(model.c()), out.ctypes.data,
                        cbuf.ctypes.data if codes else None, 1)
    res = {n: out[n][0].item() for n in RESULT_DTYPE.names if not n.startswith("_")}
    return res, cbuf


def replay_wallclock(D, w: float, policy: Policy, model: Model | None = None, codes: bool = False):
    """NEXT-1 (DESIGN A32): one trace replayed with wall-clock governor rounds.  Returns (result dict with
    'n_rounds', per-round codes or None)."""
    model = model or Model()
    D = np.ascontiguousarray(D, dtype=np.float32)
    out = np.zeros(1, dtype=RESULT_DTYPE)
    cap = 3 * len(D) + 8 if codes else 0
    cbuf = np.zeros(max(1, cap), dtype=np.uint8)
    nr = C.c_int64()
    lib().oracle_replay_wallclock(D.ctypes.data, len(D), 1, float(np.float32(w)), C.byref(policy.c()),
                                  C.byref(model.c()), out.ctypes.data, C.byref(nr),
                                  cbuf.ctypes.data if codes else None, cap)
    res = {n: out[n][0].item() for n in RESULT_DTYPE.names if not n.startswith("_")}
    res["n_rounds"] = nr.value
    return res, (cbuf[:min(nr.value, cap)] if codes else None)


def replay_batch(trace, w, policies, model: Model | None = None, codes: bool = False, n_threads: int = 0):
    """trace: [n_samples][stride] fp32 (time-major), w: [n_traces]. Returns (results[n_traces][P], codes)."""
    model = model or Model()
    trace = np.ascontiguousarray(trace, dtype=np.float32)
    w = np.ascontiguousarray(w, dtype=np.float32)
    n_samples, stride = trace.shape
    n_traces = len(w)
    P = len(policies)
    pols = (OPolicy * P)(*[p.c() for p in policies])
    out = np.zeros((n_traces, P), dtype=RESULT_DTYPE)
    cbuf = np.zeros((n_samples, n_traces, P), dtype=np.uint8) if codes else None
    used = lib().oracle_replay_batch(trace.ctypes.data, n_traces, n_samples, stride, w.ctypes.data, P, pols,
                                     C.byref(model.c()), out.ctypes.data,
                                     cbuf.ctypes.data if codes else None, n_threads)
    return out, cbuf, used


def gen_traces(desc: GenDesc):
    """Oracle-side generator: returns (trace [n_samples][stride] fp32, w [n_traces] fp32)."""
    g = desc.c()
    trace = np.empty((desc.n_samples, g.trace_stride), dtype=np.float32)
    w = np.empty(desc.n_traces, dtype=np.float32)
    lib().oracle_gen_traces(C.byref(g), trace.ctypes.data, w.ctypes.data)
    return trace, w


def gen_trace(desc: GenDesc, j_local: int):
    g = desc.c()
    col = np.empty(desc.n_samples, dtype=np.float32)
    w = lib().oracle_gen_trace(C.byref(g), j_local, col.ctypes.data, 1)
    return col, np.float32(w)


def gen_replay(desc: GenDesc, trace_ids, policies, model: Model | None = None, n_threads: int = 0):
    """Generate-and-replay a subset of traces (local ids). Returns (results[n_ids][P], w[n_ids], threads)."""
    model = model or Model()
    ids = np.ascontiguousarray(trace_ids, dtype=np.int64)
    P = len(policies)
    pols = (OPolicy * P)(*[p.c() for p in policies])
    out = np.zeros((len(ids), P), dtype=RESULT_DTYPE)
    w = np.zeros(len(ids), dtype=np.float32)
    used = lib().oracle_gen_replay(C.byref(desc.c()), ids.ctypes.data, len(ids), P, pols, C.byref(model.c()),
                                   out.ctypes.data, w.ctypes.data, n_threads)
    return out, w, used


def gen_replay_codes(desc: GenDesc, trace_ids, policies, model: Model | None = None, n_threads: int = 0):
    """gen_replay that also returns every tick's code byte: (results[n_ids][P], codes[n_ids][P][n_samples] uint8,
    w[n_ids], threads)."""
    model = model or Model()
    ids = np.ascontiguousarray(trace_ids, dtype=np.int64)
    P = len(policies)
    pols = (OPolicy * P)(*[p.c() for p in policies])
    out = np.zeros((len(ids), P), dtype=RESULT_DTYPE)
    w = np.zeros(len(ids), dtype=np.float32)
    codes = np.zeros((len(ids), P, desc.n_samples), dtype=np.uint8)
    used = lib().oracle_gen_replay_codes(C.byref(desc.c()), ids.ctypes.data, len(ids), P, pols, C.byref(model.c()),
                                         out.ctypes.data, w.ctypes.data, codes.ctypes.data, n_threads)
    return out, codes, w, used
