"""ctypes binding of include/magus_replay.h -- argument marshalling only.

Every step of the replay runs in the CUDA kernels of lib/libmagus_replay.so.  PyTorch supplies
device memory (tensor data_ptr), streams (torch.cuda.Stream.cuda_stream) and, for world > 1, the
process group that broadcasts the NCCL unique id.  There is no CPU fallback: if the library is
missing this module raises on import, and without a CUDA device every compute call raises
MagusError(MAGUS_ERR_CUDA).
"""
from __future__ import annotations

import ctypes as C
import os
import re
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# MAGUS_LIB_PATH: experiments only (a build variant, e.g. scripts/variant_build.sh); default = the in-tree build
LIB_PATH = os.environ.get("MAGUS_LIB_PATH") or os.path.join(_HERE, "lib", "libmagus_replay.so")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "magus_replay.h")

MAGUS_OK, ERR_INVALID_ARG, ERR_CONFIG, ERR_ALIGN, ERR_TRACE, ERR_STATE, ERR_OOM, ERR_CUDA, ERR_NCCL = range(9)
STATUS_NAMES = ["MAGUS_OK", "MAGUS_ERR_INVALID_ARG", "MAGUS_ERR_CONFIG", "MAGUS_ERR_ALIGN", "MAGUS_ERR_TRACE",
                "MAGUS_ERR_STATE", "MAGUS_ERR_OOM", "MAGUS_ERR_CUDA", "MAGUS_ERR_NCCL"]
MAGUS, STATIC_MAX, STATIC_MIN, TDP_DEFAULT = 0, 1, 2, 3
F_PER_TRACE_STATS, F_DUMP_WORDS, F_DUMP_DECISIONS, F_TIMING, F_TIMING_DETAIL = 0x1, 0x2, 0x4, 0x8, 0x10
F_WALLCLOCK = 0x20   # NEXT-1 wall-clock governor rounds (A32)
F_NCCL = 0x40        # the cross-rank exchange (chunk sums + NCCL allreduce) also at world == 1
TOTAL_FIELDS = ["E", "E_pkg", "T", "EDP", "slowdown", "energy_saving", "edp_saving", "n_hi", "n_thr",
                "transitions", "tune_events", "lock_ticks", "n_traces"]
N_TOTALS = len(TOTAL_FIELDS)


class MagusError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else status}: {msg}")
        self.status = status


class c_policy(C.Structure):
    _fields_ = [("kind", C.c_int32), ("deriv_ticks", C.c_int32), ("inc_threshold", C.c_double),
                ("dec_threshold", C.c_double), ("tune_log_capacity", C.c_int32), ("_reserved0", C.c_int32),
                ("high_freq_threshold", C.c_double), ("tdp_w", C.c_double), ("tdp_margin", C.c_double)]


class c_model(C.Structure):
    _fields_ = [("sample_period_s", C.c_double), ("f_min_ghz", C.c_double), ("f_max_ghz", C.c_double),
                ("bw_max_gbps", C.c_double), ("bw_shape", C.c_int32), ("observe", C.c_int32),
                ("bw_knee", C.c_double), ("p_pkg_idle_w", C.c_double), ("p_core_active_w", C.c_double),
                ("p_uncore_min_w", C.c_double), ("p_uncore_max_w", C.c_double), ("p_exponent", C.c_double),
                ("p_gpu_active_w", C.c_double), ("dram_w_per_gbps", C.c_double)]


class c_desc(C.Structure):
    _fields_ = [("n_traces", C.c_int32), ("n_samples", C.c_int32), ("trace_stride", C.c_int64),
                ("global_trace_offset", C.c_int64), ("n_policies", C.c_int32), ("_reserved0", C.c_int32),
                ("policies", C.POINTER(c_policy)), ("model", c_model), ("rank", C.c_int32), ("world", C.c_int32),
                ("nccl_unique_id", C.c_void_p), ("flags", C.c_uint32), ("dump_first_trace", C.c_int32),
                ("dump_n_traces", C.c_int32), ("tuning_segments", C.c_int32), ("tuning_warmup", C.c_int32),
                ("n_policies_global", C.c_int32), ("policy_offset", C.c_int32)]


class c_trace_stats(C.Structure):
    _fields_ = [("n_hi", C.c_int64), ("n_thr", C.c_int64), ("transitions", C.c_int64), ("tune_events", C.c_int64),
                ("lock_ticks", C.c_int64), ("T", C.c_double), ("E_pkg", C.c_double), ("E", C.c_double),
                ("EDP", C.c_double), ("slowdown", C.c_double), ("energy_saving", C.c_double),
                ("edp_saving", C.c_double), ("pkg_power_saving", C.c_double), ("digest", C.c_uint64)]


class c_results(C.Structure):
    _fields_ = [("policy_totals", C.c_void_p), ("per_trace", C.c_void_p), ("words", C.c_void_p),
                ("decisions", C.c_void_p), ("argmin_policy", C.c_int32), ("err_trace", C.c_int32),
                ("err_tick", C.c_int64), ("n_segments", C.c_int32), ("warmup_ticks", C.c_int32),
                ("n_mismatched_segments", C.c_int64), ("fixup_rounds", C.c_int32), ("_reserved0", C.c_int32)]


class c_gen_desc(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("n_traces", C.c_int32), ("class_mix", C.c_int32), ("n_samples", C.c_int64),
                ("trace_stride", C.c_int64), ("global_trace_offset", C.c_int64), ("noise_amp", C.c_float),
                ("_reserved0", C.c_float), ("bw_max_gbps", C.c_double)]


TRACE_STATS_DTYPE = np.dtype([(n, "<i8" if t is C.c_int64 else ("<u8" if t is C.c_uint64 else "<f8"))
                              for n, t in c_trace_stats._fields_])
assert TRACE_STATS_DTYPE.itemsize == C.sizeof(c_trace_stats) == 112

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2502_03796_b200._build` "
                      "(there is no CPU fallback)")
lib = C.CDLL(LIB_PATH)
_S = C.c_int
lib.magus_abi_version.restype = C.c_int32
lib.magus_debug_check_probe.restype = C.c_int32
lib.magus_debug_check_probe.argtypes = [C.c_int32]
lib.magus_last_error.restype = C.c_char_p
lib.magus_replay_last_error.restype = C.c_char_p
lib.magus_replay_last_error.argtypes = [C.c_void_p]
lib.magus_nccl_unique_id.restype = _S
lib.magus_nccl_unique_id.argtypes = [C.c_void_p]
lib.magus_gen_traces.restype = _S
lib.magus_gen_traces.argtypes = [C.POINTER(c_gen_desc), C.c_void_p, C.c_void_p, C.c_void_p]
lib.magus_replay_create.restype = _S
lib.magus_replay_create.argtypes = [C.POINTER(c_desc), C.POINTER(C.c_void_p)]
lib.magus_replay_run.restype = _S
lib.magus_replay_run.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
lib.magus_replay_run_host.restype = _S
lib.magus_replay_run_host.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
lib.magus_replay_results.restype = _S
lib.magus_replay_results.argtypes = [C.c_void_p, C.POINTER(c_results)]
lib.magus_replay_kernel_times.restype = _S
lib.magus_replay_kernel_times.argtypes = [C.c_void_p, C.POINTER(C.c_float)]
lib.magus_replay_timing_summary.restype = _S
lib.magus_replay_timing_summary.argtypes = [C.c_void_p, C.c_int32, C.POINTER(C.c_float)]
lib.magus_replay_run_times.restype = _S
lib.magus_replay_run_times.argtypes = [C.c_void_p, C.c_int32, C.POINTER(C.c_float), C.POINTER(C.c_int32)]
lib.magus_replay_plan_info.restype = _S
lib.magus_replay_plan_info.argtypes = [C.c_void_p, C.POINTER(C.c_int32)]
lib.magus_replay_destroy.restype = None
lib.magus_replay_destroy.argtypes = [C.c_void_p]
lib.magus_counters_to_trace.restype = _S
lib.magus_counters_to_trace.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int64, C.c_int64, C.c_double,
                                        C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
lib.magus_active_savings.restype = _S
lib.magus_active_savings.argtypes = [C.POINTER(C.c_double), C.c_int32, C.c_int32, C.c_int32, C.c_double,
                                     C.POINTER(C.c_double)]
lib.magus_totals_argmin.restype = _S
lib.magus_totals_argmin.argtypes = [C.POINTER(C.c_double), C.c_int32, C.POINTER(C.c_int32)]
lib.magus_grid_plan.restype = _S
lib.magus_grid_plan.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.c_int32, C.POINTER(C.c_int64)]
lib.magus_derive_thresholds.restype = _S
lib.magus_derive_thresholds.argtypes = [C.POINTER(c_policy), C.POINTER(c_model), C.POINTER(C.c_double),
                                        C.POINTER(C.c_float), C.POINTER(C.c_int32)]
lib.magus_replay_geometry.restype = _S
lib.magus_replay_geometry.argtypes = [C.c_void_p, C.POINTER(C.c_int32)]
assert lib.magus_abi_version() == 2, "ABI version mismatch"


def header_functions(path: str = HEADER):
    """Names of the functions include/magus_replay.h declares (for the export test)."""
    src = open(path).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(magus_[a-z0-9_]+)\s*\(", src)))


def _check(status: int, handle=None):
    if status != MAGUS_OK:
        msg = lib.magus_replay_last_error(handle) if handle else lib.magus_last_error()
        raise MagusError(status, (msg or b"").decode())


# ----------------------------------------------------------------------------- parameter records

@dataclass
class Policy:
    """One policy-parameter point (magus_policy)."""
    kind: int = MAGUS
    deriv_ticks: int = 1
    inc_threshold: float = 1.0
    dec_threshold: float = -1.0
    tune_log_capacity: int = 10
    high_freq_threshold: float = 0.6
    tdp_w: float = 270.0
    tdp_margin: float = 0.05

    def c(self) -> c_policy:
        return c_policy(self.kind, self.deriv_ticks, self.inc_threshold, self.dec_threshold,
                        self.tune_log_capacity, 0, self.high_freq_threshold, self.tdp_w, self.tdp_margin)


@dataclass
class Model:
    """Platform / energy model (magus_model); defaults = DESIGN.md section 6 default model."""
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
    observe: int = 0              # 0 closed loop (A14); 1 open loop: a recorded throughput observed as is (A30)

    def c(self) -> c_model:
        return c_model(self.sample_period_s, self.f_min_ghz, self.f_max_ghz, self.bw_max_gbps, self.bw_shape, self.observe,
                       self.bw_knee, self.p_pkg_idle_w, self.p_core_active_w, self.p_uncore_min_w,
                       self.p_uncore_max_w, self.p_exponent, self.p_gpu_active_w, self.dram_w_per_gbps)


# ----------------------------------------------------------------------------- calls

def abi_version() -> int:
    return lib.magus_abi_version()


def totals_argmin(policy_totals) -> int:
    """Host-only: the library's argmin over policies of the total EDP (policies with traces; ties -> lowest)."""
    t = np.ascontiguousarray(policy_totals, dtype=np.float64)
    out = C.c_int32()
    _check(lib.magus_totals_argmin(t.ctypes.data_as(C.POINTER(C.c_double)), t.shape[0], C.byref(out)))
    return out.value


def grid_plan(world: int, rank: int, policy_shards: int, n_traces: int, n_policies: int):
    """Host-only: (global_trace_offset, n_traces, policy_offset, n_policies) of `rank` in a 2-D split of
    n_traces traces x n_policies policies over world ranks, policy_shards of them across the policies."""
    out = (C.c_int64 * 4)()
    _check(lib.magus_grid_plan(world, rank, policy_shards, n_traces, n_policies, out))
    return tuple(int(x) for x in out)


def derive_thresholds(policy: Policy, model: Model):
    """Host-only: {'dinc','ddec','L','P_lo','P_hi','B_lo','B_hi','astar_lo','astar_hi','s_min'}."""
    d = (C.c_double * 5)()
    f = (C.c_float * 4)()
    i = (C.c_int32 * 1)()
    _check(lib.magus_derive_thresholds(C.byref(policy.c()), C.byref(model.c()), d, f, i))
    return dict(dinc=d[0], ddec=d[1], L=d[2], P_lo=d[3], P_hi=d[4], B_lo=f[0], B_hi=f[1], astar_lo=f[2],
                astar_hi=f[3], s_min=i[0])


def counters_to_trace(counts, trace, n_traces: int, period_s: float = 0.1, times=None, stream=None):
    """NEXT-3: recorded cumulative byte counters (CUDA uint64 tensor [n_rows][stride], as int64 storage) ->
    trace (CUDA fp32 tensor [n_rows-1][stride], GB/s): trace j's rounds are rows [0, n_valid[j]) of its column (a
    wrap / reset interval yields no round, DESIGN A31); times: optional CUDA fp64 tensor [n_rows].  Returns
    (n_valid as a numpy int64 array [n_traces], discarded intervals, non-increasing timestamps) after
    synchronising the stream."""
    import torch
    rep = torch.zeros(2, dtype=torch.int64, device=counts.device)
    nv = torch.zeros(max(1, n_traces), dtype=torch.int64, device=counts.device)
    _check(lib.magus_counters_to_trace(C.c_void_p(counts.data_ptr()),
                                       C.c_void_p(times.data_ptr()) if times is not None else None, n_traces,
                                       counts.shape[0], counts.shape[1], period_s, C.c_void_p(trace.data_ptr()),
                                       C.c_void_p(nv.data_ptr()), C.c_void_p(rep.data_ptr()), _stream_ptr(stream)))
    if stream is not None:
        stream.synchronize()
    else:
        torch.cuda.synchronize(counts.device)
    r = rep.cpu().tolist()
    return nv.cpu().numpy()[:n_traces], int(r[0]), int(r[1])


def active_savings(policy_totals, policy: int, baseline: int, p_idle_w: float):
    """Host-only, NEXT-4: (active power, active energy, active EDP) savings of `policy` against
    `baseline` with the idle power excluded, from Results.totals ([n_policies][N_TOTALS])."""
    t = np.ascontiguousarray(policy_totals, dtype=np.float64)
    out = (C.c_double * 3)()
    _check(lib.magus_active_savings(t.ctypes.data_as(C.POINTER(C.c_double)), t.shape[0], policy, baseline,
                                    p_idle_w, out))
    return tuple(out)


def nccl_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    _check(lib.magus_nccl_unique_id(buf))
    return bytes(buf)


def _stream_ptr(stream):
    if stream is None:
        return None
    return C.c_void_p(getattr(stream, "cuda_stream", stream))


def gen_traces(seed: int, n_traces: int, n_samples: int, class_mix: int, trace, w, *, trace_stride: int = 0,
               global_trace_offset: int = 0, noise_amp: float = 0.002, bw_max_gbps: float = 20.0, stream=None):
    """Fill device tensors trace [n_samples][stride] fp32 and w [n_traces] fp32."""
    stride = trace_stride or (trace.shape[1] if hasattr(trace, "shape") and len(trace.shape) == 2 else n_traces)
    g = c_gen_desc(seed, n_traces, class_mix, n_samples, stride, global_trace_offset, noise_amp, 0.0, bw_max_gbps)
    _check(lib.magus_gen_traces(C.byref(g), C.c_void_p(trace.data_ptr()), C.c_void_p(w.data_ptr()),
                                _stream_ptr(stream)))


@dataclass
class Results:
    totals: np.ndarray                 # [n_policies_global][13] fp64
    argmin_policy: int
    per_trace: np.ndarray | None       # structured [n_traces][P]
    words: np.ndarray | None           # [P][n_traces][n_blocks][2] uint32
    decisions: np.ndarray | None       # [n_samples][dump_n][P] uint8
    n_segments: int
    warmup_ticks: int
    n_mismatched_segments: int
    fixup_rounds: int
    status: int = MAGUS_OK
    err_trace: int = -1
    err_tick: int = -1

    def total(self, p: int, name: str) -> float:
        return float(self.totals[p, TOTAL_FIELDS.index(name)])


class Replay:
    """Owns one magus_replay_t handle (magus_replay_create ... magus_replay_destroy)."""

    def __init__(self, n_traces: int, n_samples: int, policies, model: Model | None = None, *, trace_stride: int = 0,
                 global_trace_offset: int = 0, rank: int = 0, world: int = 1, nccl_id: bytes | None = None,
                 flags: int = 0, dump_first_trace: int = 0, dump_n_traces: int = 0, tuning_segments: int = 0,
                 tuning_warmup: int = 0, n_policies_global: int = 0, policy_offset: int = 0):
        self.policies = list(policies)
        self.model = model or Model()
        self.n_traces, self.n_samples = n_traces, n_samples
        self.trace_stride = trace_stride or ((n_traces + 3) // 4 * 4)
        self.flags = flags
        self.dump_first_trace, self.dump_n_traces = dump_first_trace, dump_n_traces
        P = len(self.policies)
        self.n_policies_global = n_policies_global or P
        self._pols = (c_policy * max(1, P))(*[p.c() for p in self.policies])
        self._nccl = C.create_string_buffer(nccl_id, 128) if nccl_id else None
        desc = c_desc(n_traces, n_samples, self.trace_stride, global_trace_offset, P, 0,
                      C.cast(self._pols, C.POINTER(c_policy)), self.model.c(), rank, world,
                      C.cast(self._nccl, C.c_void_p) if self._nccl else None, flags, dump_first_trace,
                      dump_n_traces, tuning_segments, tuning_warmup, n_policies_global, policy_offset)
        h = C.c_void_p()
        _check(lib.magus_replay_create(C.byref(desc), C.byref(h)))
        self._h = h
        self.n_blocks = (n_samples + 31) // 32

    def close(self):
        if getattr(self, "_h", None):
            lib.magus_replay_destroy(self._h)
            self._h = None

    __del__ = close

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def geometry(self) -> dict:
        g = (C.c_int32 * 16)()
        _check(lib.magus_replay_geometry(self._h, g), self._h)
        keys = ["n_segments", "segment_len", "warmup_ticks", "tile_groups_per_cta", "policy_warps_per_group",
                "trace_blocks", "policy_blocks", "ctas", "threads_per_cta", "smem_bytes", "lane_policies",
                "launch_groups", "kernels_per_run", "solo_groups", "seg_long", "wide_groups"]
        return dict(zip(keys, list(g)))

    def run(self, trace, w, stream=None):
        """trace / w: CUDA tensors (or raw device pointers as ints)."""
        tp = trace if isinstance(trace, int) else trace.data_ptr()
        wp = w if isinstance(w, int) else w.data_ptr()
        _check(lib.magus_replay_run(self._h, C.c_void_p(tp), C.c_void_p(wp), _stream_ptr(stream)), self._h)

    def run_host(self, trace, w, stream=None):
        """trace / w: host arrays (torch CPU tensors, pinned for speed, or numpy)."""
        tp = trace.data_ptr() if hasattr(trace, "data_ptr") else trace.ctypes.data
        wp = w.data_ptr() if hasattr(w, "data_ptr") else w.ctypes.data
        _check(lib.magus_replay_run_host(self._h, C.c_void_p(tp), C.c_void_p(wp), _stream_ptr(stream)), self._h)

    def run_times(self, n_last: int) -> list:
        """The replay kernel's CUDA-event time (ms) of each of the last n_last runs, oldest first."""
        buf = (C.c_float * max(1, n_last))()
        n = C.c_int32(0)
        _check(lib.magus_replay_run_times(self._h, n_last, buf, C.byref(n)), self._h)
        return [buf[i] for i in range(n.value)]

    def plan_info(self) -> dict:
        g = (C.c_int32 * 4)()
        _check(lib.magus_replay_plan_info(self._h, g), self._h)
        return dict(replay_launches=g[0], fused_magus_tdp=g[1], open_loop_fast=g[2], wide_groups=g[3])

    def kernel_times(self):
        out = (C.c_float * 5)()
        _check(lib.magus_replay_kernel_times(self._h, out), self._h)
        return dict(replay_ms=out[0], fixup_epilogue_ms=out[1], totals_allreduce_argmin_ms=out[2], run_ms=out[3],
                    prepass_ms=out[4])

    def timing_summary(self, n_last: int):
        out = (C.c_float * 5)()
        _check(lib.magus_replay_timing_summary(self._h, n_last, out), self._h)
        return dict(replay_ms=out[0], fixup_epilogue_ms=out[1], totals_allreduce_argmin_ms=out[2], run_ms=out[3],
                    prepass_ms=out[4])

    def results(self, per_trace: bool | None = None, words: bool | None = None, decisions: bool | None = None,
                raise_on_trace_error: bool = True) -> Results:
        P = len(self.policies)
        totals = np.zeros((self.n_policies_global, N_TOTALS), np.float64)
        per = words_a = dec = None
        if per_trace if per_trace is not None else (self.flags & F_PER_TRACE_STATS):
            per = np.zeros((self.n_traces, P), TRACE_STATS_DTYPE)
        if words if words is not None else (self.flags & F_DUMP_WORDS):
            words_a = np.zeros((P, self.n_traces, self.n_blocks, 2), np.uint32)
        if decisions if decisions is not None else (self.flags & F_DUMP_DECISIONS):
            dec = np.zeros((self.n_samples, self.dump_n_traces, P), np.uint8)
        r = c_results(totals.ctypes.data, per.ctypes.data if per is not None else None,
                      words_a.ctypes.data if words_a is not None else None,
                      dec.ctypes.data if dec is not None else None)
        st = lib.magus_replay_results(self._h, C.byref(r))
        if st != MAGUS_OK and not (st == ERR_TRACE and not raise_on_trace_error):
            _check(st, self._h)
        return Results(totals, r.argmin_policy, per, words_a, dec, r.n_segments, r.warmup_ticks,
                       r.n_mismatched_segments, r.fixup_rounds, st, r.err_trace, r.err_tick)
