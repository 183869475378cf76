#!/usr/bin/env python
"""Generate paper_2502_03796_b200/csrc/tick4_asm.cuh: one MAGUS tick for the
4 chains of a lane, written as PTX with the four chains' instructions interleaved so that ptxas sees
independent work next to every dependency.  Semantics = magus_tick<K, false, SLOW>:
  thr = f_min && D > B_lo;  A = thr ? B_lo : D (fp64, exact);  d = A - A_{t-k}
  +1 iff d > d*_inc; flag iff +1 or d < d*_dec;  log <<= 1 | flag
  cnt = (ones in the last C flags) << (C-1), kept incrementally: - (log & 2^(C-1)) (the flag leaving the
  window, already in the scaled unit) + 2^(C-1) if flagged;  lock iff cnt >= s_min << (C-1)
  cmd = lock || +1 || (f_max && !flag);  excess += D - A;  counters; vmax = max(vmax, bits(D)).
Two macros: MAGUS_TICK4_ASM (steady state) and MAGUS_TICK4W_ASM (warm-up: Alg. 1 only once `rdy`
(k+1 samples seen), Alg. 2 only once `full` (C flags logged), A7/A8)."""
import os

C = 4


def build(warm):
    names = [(f"f{c}", "+r") for c in range(C)] + [(f"ad{c}", "=&d") for c in range(C)] + \
            [(f"evh{c}", "+r") for c in range(C)] + [(f"exc{c}", "+d") for c in range(C)] + \
            [(f"lock{c}", "+r") for c in range(C)] + [(f"nthr{c}", "+r") for c in range(C)] + \
            [(f"wcmd{c}", "+r") for c in range(C)] + [(f"cnt{c}", "+r") for c in range(C)] + [("vmax", "+r")]
    inames = [(f"D{c}", "f") for c in range(C)] + [(f"old{c}", "d") for c in range(C)] + \
             [(f"Dbits{c}", "r") for c in range(C)] + \
             [("Blo", "f"), ("Blod", "d"), ("dinc", "d"), ("ddec", "d"), ("bitc", "r"), ("smin", "r"), ("one", "r"),
              ("mone", "r")]
    if warm:
        inames += [("rdy", "r"), ("full", "r")]
    idx = {n: f"%{i}" for i, (n, _) in enumerate(names + inames)}
    R = idx.__getitem__
    body = ["{", ".reg .pred plo<4>, pthr<4>, pinc<4>, pev<4>, phf<4>, pc<4>, pk<4>, pdec<4>, prdy, pfull;",
            ".reg .f64 dd<4>, dv<4>, dx<4>;", ".reg .b32 tb<4>;"]
    if warm:
        body += [f"setp.ne.u32 prdy, {R('rdy')}, 0;", f"setp.ne.u32 pfull, {R('full')}, 0;"]
    per_chain = [
        "setp.eq.u32 plo{c}, {f}, 0;",                               # level in effect is f_min
        "cvt.f64.f32 dd{c}, {D};",
        "setp.gt.and.f32 pthr{c}, {D}, {Blo}, plo{c};",             # throttled (A14)
        "selp.f64 {ad}, {Blod}, dd{c}, pthr{c};",                    # A as fp64 (exact)
        "sub.f64 dv{c}, {ad}, {old};",                               # Alg. 1 derivative numerator
    ]
    if warm:
        per_chain += [
            "setp.gt.and.f64 pinc{c}, dv{c}, {dinc}, prdy;",         # +1, once k+1 samples were seen
            "setp.lt.and.f64 pdec{c}, dv{c}, {ddec}, prdy;",
            "or.pred pev{c}, pdec{c}, pinc{c};",                     # tune flag
        ]
    else:
        per_chain += [
            "setp.gt.f64 pinc{c}, dv{c}, {dinc};",                   # +1
            "setp.lt.or.f64 pev{c}, dv{c}, {ddec}, pinc{c};",        # tune flag
        ]
    per_chain += [
        "and.b32 tb{c}, {evh}, {bitc};",                             # the flag leaving the C-window (scaled)
        "shl.b32 {evh}, {evh}, 1;",
        "@pev{c} mad.lo.u32 {evh}, {one}, {one}, {evh};",
        "mad.lo.u32 {cnt}, tb{c}, {mone}, {cnt};",                   # window count: - leaving + entering flag
        "@pev{c} mad.lo.u32 {cnt}, {bitc}, {one}, {cnt};",
        ("setp.ge.and.u32 phf{c}, {cnt}, {smin}, pfull;" if warm    # Alg. 2 on a full log (A8)
         else "setp.ge.u32 phf{c}, {cnt}, {smin};"),
        "or.pred pc{c}, phf{c}, pinc{c};",
        "or.pred pk{c}, plo{c}, pev{c};",
        "not.pred pk{c}, pk{c};",
        "or.pred pc{c}, pc{c}, pk{c};",                              # lock || +1 || (f_max && !flag)
        "selp.u32 {f}, 1, 0, pc{c};",
        "mad.lo.u32 {wcmd}, {wcmd}, 2, {f};",
        "sub.f64 dx{c}, dd{c}, {ad};",                               # throttling excess D - A (0 unless thr)
        "add.f64 {exc}, {exc}, dx{c};",
        "@phf{c} mad.lo.u32 {lock}, {one}, {one}, {lock};",
        "@pthr{c} mad.lo.u32 {nthr}, {one}, {one}, {nthr};",
        "max.u32 {vmax}, {vmax}, {Dbits};",                          # validation (A17)
    ]
    for tmpl in per_chain:
        for c in range(C):
            body.append(tmpl.format(c=c, f=R(f"f{c}"), D=R(f"D{c}"), Blo=R("Blo"), ad=R(f"ad{c}"), Blod=R("Blod"),
                                    old=R(f"old{c}"), dinc=R("dinc"), ddec=R("ddec"), evh=R(f"evh{c}"), one=R("one"),
                                    bitc=R("bitc"), mone=R("mone"), cnt=R(f"cnt{c}"), smin=R("smin"),
                                    wcmd=R(f"wcmd{c}"), exc=R(f"exc{c}"),
                                    lock=R(f"lock{c}"), nthr=R(f"nthr{c}"), vmax=R("vmax"), Dbits=R(f"Dbits{c}")))
    body.append("}")
    params = ", ".join(n for n, _ in names + inames)
    name = "MAGUS_TICK4W_ASM" if warm else "MAGUS_TICK4_ASM"
    out = [f"#define {name}({params}) \\", "    asm( \\"]
    out += [f'        "{l}\\n\\t" \\' for l in body]
    out.append("        : " + ", ".join(f'"{c}"({n})' for n, c in names) + " \\")
    out.append("        : " + ", ".join(f'"{c}"({n})' for n, c in inames) + ")")
    return out


def build_stage(K, TC=8):
    """MAGUS_STAGE8_K<K>: one whole steady-state stage (TC ticks x 4 chains) of the solo replay kernel,
    the tile's shared-memory loads included.  The level in effect is carried from tick to tick as a
    predicate (no integer round trip); the ring of the last K observations lives in virtual registers,
    so the derivative reads A_{t-K} without moves.  Same semantics as TC calls of MAGUS_TICK4_ASM."""
    names = [(f"f{c}", "+r") for c in range(C)] + \
            [(f"r{c}_{i}", "+d") for c in range(C) for i in range(K)] + \
            [(f"evh{c}", "+r") for c in range(C)] + [(f"exc{c}", "+d") for c in range(C)] + \
            [(f"lock{c}", "+r") for c in range(C)] + [(f"nthr{c}", "+r") for c in range(C)] + \
            [(f"wcmd{c}", "+r") for c in range(C)] + [(f"cnt{c}", "+r") for c in range(C)] + [("vmax", "+r")]
    inames = [("tile", "r"), ("Blo", "f"), ("Blod", "d"), ("dinc", "d"), ("ddec", "d"), ("bitc", "r"), ("smin", "r"),
              ("one", "r"), ("mone", "r")]
    idx = {n: f"%{i}" for i, (n, _) in enumerate(names + inames)}
    R = idx.__getitem__
    body = ["{", ".reg .pred phi<4>, pthr<4>, pinc<4>, pev<4>, phf<4>, pc<4>, pk<4>;",
            f".reg .b32 D<{TC * C}>;", f".reg .f64 dd<4>, dv<4>, dx<4>, ad<{TC * C}>;", ".reg .b32 tb<4>, fb<4>;"]
    for c in range(C):
        body.append(f"setp.ne.u32 phi{c}, {R(f'f{c}')}, 0;")
    for tt in range(TC):
        body.append(f"ld.shared.v4.f32 {{D{tt * C}, D{tt * C + 1}, D{tt * C + 2}, D{tt * C + 3}}}, [{R('tile')}+{tt * 512}];")
        per_chain = [
            "cvt.f64.f32 dd{c}, {D};",
            "setp.gt.and.f32 pthr{c}, {D}, {Blo}, !phi{c};",           # throttled: level f_min and D > B_lo (A14)
            "selp.f64 {ad}, {Blod}, dd{c}, pthr{c};",                   # A as fp64 (exact)
            "sub.f64 dv{c}, {ad}, {old};",                              # Alg. 1 numerator A_t - A_{t-k}
            "setp.gt.f64 pinc{c}, dv{c}, {dinc};",                      # +1
            "setp.lt.or.f64 pev{c}, dv{c}, {ddec}, pinc{c};",           # tune flag
            "and.b32 tb{c}, {evh}, {bitc};",                            # the flag leaving the C-window (scaled)
            "shl.b32 {evh}, {evh}, 1;",
            "@pev{c} mad.lo.u32 {evh}, {one}, {one}, {evh};",
            "mad.lo.u32 {cnt}, tb{c}, {mone}, {cnt};",                  # window count: - leaving + entering flag
            "@pev{c} mad.lo.u32 {cnt}, {bitc}, {one}, {cnt};",
            "setp.ge.u32 phf{c}, {cnt}, {smin};",                       # Alg. 2
            "or.pred pc{c}, phf{c}, pinc{c};",
            "not.pred pk{c}, pev{c};",
            "and.pred pk{c}, pk{c}, phi{c};",
            "or.pred phi{c}, pc{c}, pk{c};",                            # lock || +1 || (f_max && !flag)
            "selp.u32 fb{c}, 1, 0, phi{c};",
            "mad.lo.u32 {wcmd}, {wcmd}, 2, fb{c};",
            "sub.f64 dx{c}, dd{c}, {ad};",                              # throttling excess D - A (0 unless thr)
            "add.f64 {exc}, {exc}, dx{c};",
            "@phf{c} mad.lo.u32 {lock}, {one}, {one}, {lock};",
            "@pthr{c} mad.lo.u32 {nthr}, {one}, {one}, {nthr};",
            "max.u32 {vmax}, {vmax}, {Db};",                            # validation (A17)
        ]
        for tmpl in per_chain:
            for c in range(C):
                t = tt * C + c
                old = f"ad{(tt - K) * C + c}" if tt >= K else R(f"r{c}_{K - 1 - tt}")
                body.append(tmpl.format(c=c, D=f"D{t}", Db=f"D{t}", Blo=R("Blo"), ad=f"ad{t}", Blod=R("Blod"), old=old,
                                        dinc=R("dinc"), ddec=R("ddec"), evh=R(f"evh{c}"), one=R("one"),
                                        bitc=R("bitc"), mone=R("mone"), cnt=R(f"cnt{c}"), smin=R("smin"),
                                        wcmd=R(f"wcmd{c}"), exc=R(f"exc{c}"), lock=R(f"lock{c}"),
                                        nthr=R(f"nthr{c}"), vmax=R("vmax")))
    for c in range(C):
        body.append(f"mov.u32 {R(f'f{c}')}, fb{c};")
        for i in range(K):   # ring newest first: r_i = A_{t0 + TC - 1 - i}
            body.append(f"mov.f64 {R(f'r{c}_{i}')}, ad{(TC - 1 - i) * C + c};")
    body.append("}")
    params = ", ".join(n for n, _ in names + inames)
    out = [f"#define MAGUS_STAGE8_K{K}(...) MAGUS_STAGE8_K{K}_(__VA_ARGS__)",
           f"#define MAGUS_STAGE8_K{K}_({params}) \\", "    asm volatile( \\"]
    out += [f'        "{l}\\n\\t" \\' for l in body]
    out.append("        : " + ", ".join(f'"{c}"({n})' for n, c in names) + " \\")
    out.append("        : " + ", ".join(f'"{c}"({n})' for n, c in inames) + " \\")
    out.append('        : "memory")')
    return out



def build_stage_f(K, TC=8, walk=False, traces=1, thr64=True, one=False, bits=False):
    """MAGUS_SSTAGE_K<K>: one whole steady-state stage (TC ticks x 4 chains, tile loads included) of the solo
    replay kernel, balanced over the issue pipes (ALU and FMA-heavy at half rate, FP64, XU): the throttle
    test on the FP64 pipe, the tune log, scaled window count and cmd word as (predicated) IMADs, the lock /
    throttle counters as fp32 adds of 1 (exact integers, fma-lite), the level carried as a predicate
    across the stage.  Decisions identical to MAGUS_TICK4_ASM.
    walk=True: MAGUS_WSTAGE_K<K>, the chain walk's stage (post_kernels.cuh): two chains -- the true and the
    speculative state of ONE trace -- stepped over the same 8 samples, passed in registers; no validation
    maximum (the replay already took it)."""
    C = (1 if one else 2 * traces) if walk else 4   # walk: chains (2t, 2t+1) = (true, speculative) of trace t;
                                                    # one: a single chain (the split walk, one state per warp)
    names = [(f"f{c}", "+r") for c in range(C)] + \
            [(f"r{c}_{i}", "+d") for c in range(C) for i in range(K)] + \
            [(f"evh{c}", "+r") for c in range(C)] + [(f"cnt{c}", "+r") for c in range(C)] + \
            [(f"exc{c}", "+d") for c in range(C)] + [(f"lock{c}", "+f") for c in range(C)] + \
            [(f"nthr{c}", "+f") for c in range(C)] + [(f"wcmd{c}", "+r") for c in range(C)] + \
            ([] if walk else [("vmax", "+r")])
    inames = ([(f"S{u}_{tt}", "r") for u in range(traces) for tt in range(TC)] if walk else [("tile", "r")]) + \
             ([] if thr64 else [("Blo", "f")]) + [("Blod", "d"), ("dinc", "d"), ("ddec", "d"), ("bitc", "r"), ("smin", "r"),
              ("one", "r"), ("mone", "r")]
    idx = {n: f"%{i}" for i, (n, _) in enumerate(names + inames)}
    R = idx.__getitem__
    body = ["{", ".reg .pred phi<4>, pthr<4>, pinc<4>, pev<4>, phf<4>, pq<4>, pk<4>;",
            f".reg .b32 D<{TC * C}>;", f".reg .f64 dd<4>, dv<4>, dx<4>, ad<{TC * C}>;", ".reg .b32 tb<4>, xh<4>, xl<4>;"]
    for c in range(C):
        body.append(f"setp.ne.u32 phi{c}, {R(f'f{c}')}, 0;")
    for tt in range(TC):
        if walk:
            body += [f"mov.b32 D{tt * C + c}, {R(f'S{c // 2}_{tt}')};" for c in range(C)]
        else:
            body.append(f"ld.shared.v4.f32 {{D{tt * C}, D{tt * C + 1}, D{tt * C + 2}, D{tt * C + 3}}}, [{R('tile')}+{tt * 512}];")
        per_chain = ([
            "shr.u32 xh{c}, {D}, 3;",                                    # fp32 -> fp64 by integer ops (no XU):
            "add.u32 xh{c}, xh{c}, 0x38000000;",                         # exact for normal samples (DESIGN 7)
            "shl.b32 xl{c}, {D}, 29;",
            "mov.b64 dd{c}, {{xl{c}, xh{c}}};",
        ] if bits else ["cvt.f64.f32 dd{c}, {D};"]) + [
            ("setp.gt.and.f64 pthr{c}, dd{c}, {Blod}, !phi{c};" if thr64  # throttled: f_min and D > B_lo (A14)
             else "setp.gt.and.f32 pthr{c}, {D}, {Blo}, !phi{c};"),
            "selp.f64 {ad}, {Blod}, dd{c}, pthr{c};",                    # A = min(D, B[f]) as fp64 (exact)
            "sub.f64 dv{c}, {ad}, {old};",                               # Alg. 1 numerator A_t - A_{t-k}
            "setp.gt.f64 pinc{c}, dv{c}, {dinc};",                       # +1
            "setp.lt.or.f64 pev{c}, dv{c}, {ddec}, pinc{c};",            # tune flag
            "and.b32 tb{c}, {evh}, {bitc};",                             # the flag leaving the C-window (scaled)
            "shl.b32 {evh}, {evh}, 1;",
            "@pev{c} mad.lo.u32 {evh}, {one}, {one}, {evh};",
            "mad.lo.u32 {cnt}, tb{c}, {mone}, {cnt};",                   # window count: - leaving + entering
            "@pev{c} mad.lo.u32 {cnt}, {bitc}, {one}, {cnt};",
            "setp.ge.u32 phf{c}, {cnt}, {smin};",                        # Alg. 2
            "not.pred pk{c}, pev{c};",
            "and.pred pk{c}, pk{c}, phi{c};",
            "or.pred pq{c}, pk{c}, pinc{c};",                            # +1 || (f_max && !flag)
            "or.pred phi{c}, pq{c}, phf{c};",                            # || lock: the new level
            "shl.b32 {wcmd}, {wcmd}, 1;",
            "@phi{c} mad.lo.u32 {wcmd}, {one}, {one}, {wcmd};",
            "sub.f64 dx{c}, dd{c}, {ad};",                               # throttling excess D - A (0 unless thr)
            "add.f64 {exc}, {exc}, dx{c};",
            "@phf{c} add.f32 {lock}, {lock}, 0f3F800000;",
            "@pthr{c} add.f32 {nthr}, {nthr}, 0f3F800000;",
        ] + ([] if walk else ["max.u32 {vmax}, {vmax}, {D};"])        # validation (A17)
        for tmpl in per_chain:
            for c in range(C):
                t = tt * C + c
                old = f"ad{(tt - K) * C + c}" if tt >= K else R(f"r{c}_{K - 1 - tt}")
                body.append(tmpl.format(c=c, D=f"D{t}", ad=f"ad{t}", old=old, Blod=R("Blod"), dinc=R("dinc"),
                                        Blo=None if thr64 else R("Blo"),
                                        ddec=R("ddec"), evh=R(f"evh{c}"), one=R("one"), bitc=R("bitc"),
                                        mone=R("mone"), cnt=R(f"cnt{c}"), smin=R("smin"),
                                        wcmd=R(f"wcmd{c}"), exc=R(f"exc{c}"), lock=R(f"lock{c}"),
                                        nthr=R(f"nthr{c}"), vmax=None if walk else R("vmax")))
    for c in range(C):
        body.append(f"selp.u32 {R(f'f{c}')}, 1, 0, phi{c};")
        for i in range(K):   # ring newest first: r_i = A_{t0 + TC - 1 - i}
            body.append(f"mov.f64 {R(f'r{c}_{i}')}, ad{(TC - 1 - i) * C + c};")
    body.append("}")
    params = ", ".join(n for n, _ in names + inames)
    name = f"MAGUS_{'W' if walk else 'S'}STAGE{'2' if traces == 2 else ''}{'1' if one else ''}{'' if thr64 else 'F'}{'B' if bits else ''}_K{K}"
    out = [f"#define {name}(...) {name}_(__VA_ARGS__)", f"#define {name}_({params}) \\", "    asm volatile( \\"]
    out += [f'        "{l}\\n\\t" \\' for l in body]
    out.append("        : " + ", ".join(f'"{c}"({n})' for n, c in names) + " \\")
    out.append("        : " + ", ".join(f'"{c}"({n})' for n, c in inames) + " \\")
    out.append('        : "memory")')
    return out


def build_stage_p(K, TC=8, popc=True, group=4, sym=False):
    """MAGUS_PSTAGE_K<K> (popc=True) / MAGUS_QSTAGE_K<K> (popc=False): the solo kernel's steady-state stage
    (TC ticks x 4 chains, tile loads included) with fewer instructions per chain-tick than MAGUS_SSTAGEF_K<K>:
    - the new level is hf | +1 | (level & !dec): one DSETP gives (d >= d*_dec) & level directly, so the
      predicate logic is three DSETPs, one ISETP and one 3-input PLOP3 (ptxas otherwise re-evaluates the
      +1 and Alg. 2 compares in OR form);
    - popc=True: Alg. 2's window count is popc(log & (2^C - 1)) (LOP3 + POPC, no incremental count: the
      XU pipe then carries the conversion and the popcount); popc=False keeps the scaled incremental count
      (LOP3 + two IMADs) and compares against s_min << (C-1).
    Decisions identical to MAGUS_TICK4_ASM."""
    C = 4
    names = [(f"f{c}", "+r") for c in range(C)] + \
            [(f"r{c}_{i}", "+d") for c in range(C) for i in range(K)] + \
            [(f"evh{c}", "+r") for c in range(C)] + \
            ([] if popc else [(f"cnt{c}", "+r") for c in range(C)]) + \
            [(f"exc{c}", "+d") for c in range(C)] + [(f"lock{c}", "+f") for c in range(C)] + \
            [(f"nthr{c}", "+f") for c in range(C)] + [(f"wcmd{c}", "+r") for c in range(C)] + [("vmax", "+r")]
    inames = [("tile", "r"), ("Blo", "f"), ("Blod", "d"), ("dinc", "d"), ("ddec", "d")] + \
             ([("maskc", "r"), ("smin", "r"), ("one", "r")] if popc else
              [("bitc", "r"), ("smin", "r"), ("one", "r"), ("mone", "r")])
    idx = {n: f"%{i}" for i, (n, _) in enumerate(names + inames)}
    R = idx.__getitem__
    body = ["{", ".reg .pred phi<4>, pthr<4>, pinc<4>, pev<4>, phf<4>, pk<4>, pq<4>;",
            f".reg .b32 D<{TC * C}>;", f".reg .f64 dd<4>, dv<4>, da<4>, dx<4>, ad<{TC * C}>;",
            ".reg .b32 tb<4>, wv<4>, pc<4>;"]
    for c in range(C):
        body.append(f"setp.ne.u32 phi{c}, {R(f'f{c}')}, 0;")
    for tt in range(TC):
        body.append(f"ld.shared.v4.f32 {{D{tt * C}, D{tt * C + 1}, D{tt * C + 2}, D{tt * C + 3}}}, [{R('tile')}+{tt * 512}];")
        per_chain = [
            "cvt.f64.f32 dd{c}, {D};",
            "setp.gt.and.f32 pthr{c}, {D}, {Blo}, !phi{c};",             # throttled: f_min and D > B_lo (A14)
            "selp.f64 {ad}, {Blod}, dd{c}, pthr{c};",                     # A = min(D, B[f]) as fp64 (exact)
            "sub.f64 dv{c}, {ad}, {old};",                                # Alg. 1 numerator A_t - A_{t-k}
        ] + ([
            "abs.f64 da{c}, dv{c};",                                      # symmetric thresholds (d*_dec = -d*_inc):
            "setp.gt.f64 pev{c}, da{c}, {dinc};",                         # tune flag iff |d| > d*_inc
        ] if sym else [
            "setp.gt.f64 pinc{c}, dv{c}, {dinc};",                        # +1
            "setp.lt.or.f64 pev{c}, dv{c}, {ddec}, pinc{c};",             # tune flag: +1 or -1
        ]) + [
            "setp.ge.and.f64 pk{c}, dv{c}, {ddec}, phi{c};",              # level kept: f_max and not -1
        ] + ([
            "setp.gt.or.f64 pk{c}, dv{c}, {dinc}, pk{c};",                # ... or +1
        ] if sym else [])
        if popc:
            per_chain += [
                "shl.b32 {evh}, {evh}, 1;",
                "@pev{c} mad.lo.u32 {evh}, {one}, {one}, {evh};",
                "and.b32 wv{c}, {evh}, {maskc};",                         # the last C flags
                "popc.b32 pc{c}, wv{c};",
                "setp.ge.u32 phf{c}, pc{c}, {smin};",                     # Alg. 2
            ]
        else:
            per_chain += [
                "and.b32 tb{c}, {evh}, {bitc};",                          # the flag leaving the C-window (scaled)
                "shl.b32 {evh}, {evh}, 1;",
                "@pev{c} mad.lo.u32 {evh}, {one}, {one}, {evh};",
                "mad.lo.u32 {cnt}, tb{c}, {mone}, {cnt};",                # window count: - leaving + entering
                "@pev{c} mad.lo.u32 {cnt}, {bitc}, {one}, {cnt};",
                "setp.ge.u32 phf{c}, {cnt}, {smin};",                     # Alg. 2
            ]
        per_chain += ([
            "or.pred phi{c}, pk{c}, phf{c};",                             # lock || +1 || (f_max && !-1)
        ] if sym else [
            "or.pred pq{c}, pinc{c}, pk{c};",
            "or.pred phi{c}, pq{c}, phf{c};",                             # lock || +1 || (f_max && !-1)
        ]) + [
            "shl.b32 {wcmd}, {wcmd}, 1;",
            "@phi{c} mad.lo.u32 {wcmd}, {one}, {one}, {wcmd};",
            "sub.f64 dx{c}, dd{c}, {ad};",                                # throttling excess D - A (0 unless thr)
            "add.f64 {exc}, {exc}, dx{c};",
            "@phf{c} add.f32 {lock}, {lock}, 0f3F800000;",
            "@pthr{c} add.f32 {nthr}, {nthr}, 0f3F800000;",
            "max.u32 {vmax}, {vmax}, {D};",                               # validation (A17)
        ]
        for g0 in range(0, C, group):
          for tmpl in per_chain:
            for c in range(g0, g0 + group):
                t = tt * C + c
                old = f"ad{(tt - K) * C + c}" if tt >= K else R(f"r{c}_{K - 1 - tt}")
                body.append(tmpl.format(c=c, D=f"D{t}", ad=f"ad{t}", old=old, Blo=R("Blo"), Blod=R("Blod"),
                                        dinc=R("dinc"), ddec=R("ddec"), evh=R(f"evh{c}"), one=R("one"),
                                        maskc=R("maskc") if popc else None, bitc=None if popc else R("bitc"),
                                        mone=None if popc else R("mone"), cnt=None if popc else R(f"cnt{c}"),
                                        smin=R("smin"), wcmd=R(f"wcmd{c}"), exc=R(f"exc{c}"), lock=R(f"lock{c}"),
                                        nthr=R(f"nthr{c}"), vmax=R("vmax")))
    for c in range(C):
        body.append(f"selp.u32 {R(f'f{c}')}, 1, 0, phi{c};")
        for i in range(K):   # ring newest first: r_i = A_{t0 + TC - 1 - i}
            body.append(f"mov.f64 {R(f'r{c}_{i}')}, ad{(TC - 1 - i) * C + c};")
    body.append("}")
    params = ", ".join(n for n, _ in names + inames)
    name = f"MAGUS_{'P' if popc else 'Q'}STAGE{'S' if sym else ''}{'' if group == 4 else 'G' + str(group)}_K{K}"
    out = [f"#define {name}(...) {name}_(__VA_ARGS__)", f"#define {name}_({params}) \\", "    asm volatile( \\"]
    out += [f'        "{l}\\n\\t" \\' for l in body]
    out.append("        : " + ", ".join(f'"{c}"({n})' for n, c in names) + " \\")
    out.append("        : " + ", ".join(f'"{c}"({n})' for n, c in inames) + " \\")
    out.append('        : "memory")')
    return out



def build_stage_l(K, TC=8, sym=False, tdp=False, tdp_up=False, batch=False):
    """MAGUS_LSTAGE_K<K>: the solo kernel's steady-state stage with the level and the lock counter folded into
    words and signs, fewer instructions per chain-tick than MAGUS_SSTAGEF_K<K> (same decisions):
    - the cmd word is shifted once per stage (by TC) and tick tt sets bit TC-1-tt with a predicated IMAD of an
      immediate, so its bit layout after 32 / TC stages is the same as one shift per tick (tick i of the block at
      bit 31 - i); the level at the stage start is its bit 0 (the previous tick's cmd), no level register;
    - the scaled window count is kept biased by -s_min << (C-1) (the caller subtracts it before the steady
      stages and adds it back after): Alg. 2's lock is the count's sign (cnt >= 0, signed; |cnt| < 2^31 needs
      C <= 27), folded into the new-level compare (ISETP.GE.OR); the ticks NOT locked are counted with the sign
      bit (nlk += cnt >> 31, unsigned), so there is no separate lock predicate or predicated lock counter.
    sym=True (MAGUS_LSTAGES_K<K>, only for d*_dec == -d*_inc): the tune flag is |d| > d*_inc and the kept-or-raised
      level +1 | (f_max & !-1) is two DSETPs ((d >= d*_dec) & level, then (d > d*_inc) | that).
    tdp_up=True (MAGUS_LTUSTAGE[S]_K<K>): the same for a TDP policy whose f_min threshold is +inf (B_lo < a*_lo: at
      f_min the budget is never reached, so f_min always rises), one compare fewer per TDP tick.
    tdp=True (MAGUS_LTSTAGE[S]_K<K>, the fused MAGUS + TDP kernel): the same 4 traces also step one TDP_DEFAULT chain
      each (the tick of MAGUS_TLSTAGE: level in its own cmd word, next level f_max iff D < a_hi | (f_min & D < a_lo),
      throttled demand summed by a 0/1 DFMA), sharing the tile loads, the fp64 conversion and the validation.
    batch=True (MAGUS_LB[T[U]]STAGE[S]_K<K>): the tune-flag log is also shifted once per stage (by TC) and tick tt
      sets its bit TC-1-tt, like the cmd word, so the per-tick shift goes.  With C >= TC every flag leaving the
      window during the stage was logged before it: after the stage-start shift the one leaving at tick tt (bit C-1
      before a per-tick shift) is bit C-1+TC-tt, i.e. bit TC-tt of ev2 = log >> (C-1) (one shift per stage, cm1 =
      C-1 an input), tested with an immediate mask.  The count is scaled by 2^TC instead of 2^(C-1) (the caller
      converts it), so the leaving flag is (ev2 & 2^(TC-tt)) * -2^tt and an entering one +2^TC: immediates only.
      Needs TC <= C <= 32-TC."""
    C = 4
    names = [(f"r{c}_{i}", "+d") for c in range(C) for i in range(K)] + \
            [(f"evh{c}", "+r") for c in range(C)] + [(f"cnt{c}", "+r") for c in range(C)] + \
            [(f"exc{c}", "+d") for c in range(C)] + [(f"nlk{c}", "+r") for c in range(C)] + \
            [(f"nthr{c}", "+f") for c in range(C)] + [(f"wcmd{c}", "+r") for c in range(C)] + [("vmax", "+r")]
    if tdp:
        names += [(f"wcmdT{c}", "+r") for c in range(C)] + [(f"excT{c}", "+d") for c in range(C)] + \
                 [(f"nthrT{c}", "+f") for c in range(C)] + [(f"sT{c}", "+d") for c in range(C)]
    inames = [("tile", "r"), ("Blo", "f"), ("Blod", "d"), ("dinc", "d"), ("ddec", "d"), ("bitc", "r"),
              ("one", "r"), ("mone", "r")] + ([("ahi", "f"), ("alo", "f")] if tdp else []) + \
             ([("cm1", "r")] if batch else [])
    idx = {n: f"%{i}" for i, (n, _) in enumerate(names + inames)}
    R = idx.__getitem__
    body = ["{", ".reg .pred phi<4>, pthr<4>, pinc<4>, pev<4>, pk<4>, pq<4>;",
            f".reg .b32 D<{TC * C}>;", f".reg .f64 dd<4>, dv<4>, da<4>, dx<4>, ad<{TC * C}>;",
            ".reg .b32 tb<4>, tl<4>, lv<4>, eo<4>;"]
    if tdp:
        body += [".reg .pred phT<4>, pthT<4>, ptT<4>, pnT<4>;", ".reg .b32 sloT<4>, shiT<4>, lvT<4>;"]
    for c in range(C):
        body.append(f"and.b32 lv{c}, {R(f'wcmd{c}')}, 1;")
        body.append(f"setp.ne.u32 phi{c}, lv{c}, 0;")                   # level = the previous tick's cmd
        body.append(f"shl.b32 {R(f'wcmd{c}')}, {R(f'wcmd{c}')}, {TC};")
        if batch:
            body.append(f"shl.b32 {R(f'evh{c}')}, {R(f'evh{c}')}, {TC};")
            body.append(f"shr.u32 eo{c}, {R(f'evh{c}')}, {R('cm1')};")
        if tdp:   # the TDP level is re-read from its cmd word every tick (bit TC - tt: the previous tick's cmd), so
                  # no TDP predicate lives across ticks (8 level predicates would exceed the 7 predicate registers)
            body.append(f"shl.b32 {R(f'wcmdT{c}')}, {R(f'wcmdT{c}')}, {TC};")
            body.append(f"mov.b64 {{sloT{c}, shiT{c}}}, {R(f'sT{c}')};")
    for tt in range(TC):
        body.append(f"ld.shared.v4.f32 {{D{tt * C}, D{tt * C + 1}, D{tt * C + 2}, D{tt * C + 3}}}, [{R('tile')}+{tt * 512}];")
        per_chain = [
            "cvt.f64.f32 dd{c}, {D};",
            "setp.gt.and.f32 pthr{c}, {D}, {Blo}, !phi{c};",             # throttled: f_min and D > B_lo (A14)
            "selp.f64 {ad}, {Blod}, dd{c}, pthr{c};",                     # A = min(D, B[f]) as fp64 (exact)
            "sub.f64 dv{c}, {ad}, {old};",                                # Alg. 1 numerator A_t - A_{t-k}
        ] + ([
            "abs.f64 da{c}, dv{c};",                                      # symmetric thresholds (d*_dec = -d*_inc):
            "setp.gt.f64 pev{c}, da{c}, {dinc};",                         # tune flag iff |d| > d*_inc
            "setp.ge.and.f64 pk{c}, dv{c}, {ddec}, phi{c};",              # f_max and not -1
            "setp.gt.or.f64 pq{c}, dv{c}, {dinc}, pk{c};",                # +1 || (f_max && !-1)
        ] if sym else [
            "setp.gt.f64 pinc{c}, dv{c}, {dinc};",                        # +1
            "setp.lt.or.f64 pev{c}, dv{c}, {ddec}, pinc{c};",             # tune flag: +1 or -1
            "not.pred pk{c}, pev{c};",
            "and.pred pk{c}, pk{c}, phi{c};",
            "or.pred pq{c}, pk{c}, pinc{c};",                             # +1 || (f_max && !flag)
        ]) + [
        ] + ([
            "and.b32 tb{c}, eo{c}, {bmt};",                              # the flag leaving the C-window (<< TC-tt)
            "@pev{c} mad.lo.u32 {evh}, {one}, {bit}, {evh};",            # the tune-flag log, bit TC-1-tt
            "mad.lo.u32 {cnt}, tb{c}, {nk}, {cnt};",                      # window count: - leaving (x 2^tt)
        ] if batch else [
            "and.b32 tb{c}, {evh}, {bitc};",                              # the flag leaving the C-window (scaled)
            "shl.b32 {evh}, {evh}, 1;",
            "@pev{c} mad.lo.u32 {evh}, {one}, {one}, {evh};",
            "mad.lo.u32 {cnt}, tb{c}, {mone}, {cnt};",                    # window count: - leaving + entering
        ]) + [
            "@pev{c} mad.lo.u32 {cnt}, {one}, {bitin}, {cnt};",           # + entering
            "setp.ge.or.s32 phi{c}, {cnt}, 0, pq{c};",                    # || lock (Alg. 2): the new level
            "shr.u32 tl{c}, {cnt}, 31;",                                  # not locked
            "add.u32 {nlk}, {nlk}, tl{c};",
            "@phi{c} mad.lo.u32 {wcmd}, {one}, {bit}, {wcmd};",
            "sub.f64 dx{c}, dd{c}, {ad};",                                # throttling excess D - A (0 unless thr)
            "add.f64 {exc}, {exc}, dx{c};",
            "@pthr{c} add.f32 {nthr}, {nthr}, 0f3F800000;",
            "max.u32 {vmax}, {vmax}, {D};",                               # validation (A17)
        ] + ([
            "and.b32 lvT{c}, {wcmdT}, {pbit};",                           # TDP: the level (previous tick's cmd)
            "setp.ne.u32 phT{c}, lvT{c}, 0;",
            "setp.gt.and.f32 pthT{c}, {D}, {Blo}, !phT{c};",              # throttled (A14)
        ] + ([
            "setp.lt.or.f32 pnT{c}, {D}, {ahi}, !phT{c};",                # f_min always rises (a_lo = +inf), f_max iff A < a*_hi
        ] if tdp_up else [
            "setp.lt.and.f32 ptT{c}, {D}, {alo}, !phT{c};",               # at f_min: A < a*_lo (A24)
            "setp.lt.or.f32 pnT{c}, {D}, {ahi}, ptT{c};",                 # next level f_max iff A < a*[f]
        ]) + [
            "selp.b32 shiT{c}, 0x3FF00000, 0, pthT{c};",                  # 1.0 if throttled, else 0.0 (low word 0)
            "mov.b64 {sT}, {{sloT{c}, shiT{c}}};",
            "fma.rn.f64 {excT}, {sT}, dd{c}, {excT};",                    # sum of D over throttled ticks (exact)
            "@pthT{c} add.f32 {nthrT}, {nthrT}, 0f3F800000;",
            "@pnT{c} mad.lo.u32 {wcmdT}, {one}, {bit}, {wcmdT};",
        ] if tdp else [])
        for tmpl in per_chain:
            for c in range(C):
                t = tt * C + c
                old = f"ad{(tt - K) * C + c}" if tt >= K else R(f"r{c}_{K - 1 - tt}")
                body.append(tmpl.format(c=c, D=f"D{t}", ad=f"ad{t}", old=old, Blo=R("Blo"), Blod=R("Blod"),
                                        dinc=R("dinc"), ddec=R("ddec"), evh=R(f"evh{c}"), one=R("one"),
                                        bitc=R("bitc"), mone=R("mone"), cnt=R(f"cnt{c}"), nlk=R(f"nlk{c}"),
                                        wcmd=R(f"wcmd{c}"), exc=R(f"exc{c}"), nthr=R(f"nthr{c}"), vmax=R("vmax"),
                                        bit=1 << (TC - 1 - tt), pbit=1 << (TC - tt),
                                        bmt=1 << (TC - tt), nk=-(1 << tt), bitin=(1 << TC) if batch else R("bitc"),
                                        **({"ahi": R("ahi"), "alo": R("alo"), "sT": R(f"sT{c}"),
                                            "excT": R(f"excT{c}"), "nthrT": R(f"nthrT{c}"),
                                            "wcmdT": R(f"wcmdT{c}")} if tdp else {})))
    for c in range(C):
        for i in range(K):   # ring newest first: r_i = A_{t0 + TC - 1 - i}
            body.append(f"mov.f64 {R(f'r{c}_{i}')}, ad{(TC - 1 - i) * C + c};")
    body.append("}")
    params = ", ".join(n for n, _ in names + inames)
    name = f"MAGUS_L{'B' if batch else ''}{'TU' if tdp_up else 'T' if tdp else ''}STAGE{'S' if sym else ''}_K{K}"
    out = [f"#define {name}(...) {name}_(__VA_ARGS__)", f"#define {name}_({params}) \\", "    asm volatile( \\"]
    out += [f'        "{l}\\n\\t" \\' for l in body]
    out.append("        : " + ", ".join(f'"{c}"({n})' for n, c in names) + " \\")
    out.append("        : " + ", ".join(f'"{c}"({n})' for n, c in inames) + " \\")
    out.append('        : "memory")')
    return out


def build_stage_tl(TC=8):
    """MAGUS_TLSTAGE: one stage (TC ticks x 4 traces) of ONE TDP_DEFAULT policy with the level carried in its cmd word
    (shifted once per stage, bit 0 = the previous tick's cmd): the fused MAGUS + TDP kernel's TDP step in the blocks
    where MAGUS runs its per-tick warm-up path.  Tick as in MAGUS_TSTAGE1L; no validation (the MAGUS path takes it)."""
    C = 4
    names = [(f"wcmd{c}", "+r") for c in range(C)] + [(f"exc{c}", "+d") for c in range(C)] + \
            [(f"nthr{c}", "+f") for c in range(C)] + [(f"s{c}", "+d") for c in range(C)]
    inames = [("tile", "r"), ("Blo", "f"), ("ahi", "f"), ("alo", "f"), ("one", "r")]
    idx = {n: f"%{i}" for i, (n, _) in enumerate(names + inames)}
    R = idx.__getitem__
    body = ["{", f".reg .pred phi<{C}>, pthr<{C}>, pt<{C}>;", f".reg .b32 D<{TC * 4}>, slo<{C}>, shi<{C}>, lv<{C}>;",
            ".reg .f64 dd<4>;"]
    for c in range(C):
        body.append(f"and.b32 lv{c}, {R(f'wcmd{c}')}, 1;")
        body.append(f"setp.ne.u32 phi{c}, lv{c}, 0;")
        body.append(f"shl.b32 {R(f'wcmd{c}')}, {R(f'wcmd{c}')}, {TC};")
        body.append(f"mov.b64 {{slo{c}, shi{c}}}, {R(f's{c}')};")
    for tt in range(TC):
        body.append(f"ld.shared.v4.f32 {{D{tt * 4}, D{tt * 4 + 1}, D{tt * 4 + 2}, D{tt * 4 + 3}}}, [{R('tile')}+{tt * 512}];")
        for u in range(4):
            body.append(f"cvt.f64.f32 dd{u}, D{tt * 4 + u};")
        per_chain = [
            "setp.gt.and.f32 pthr{c}, {D}, {Blo}, !phi{c};",             # throttled (A14)
            "setp.lt.and.f32 pt{c}, {D}, {alo}, !phi{c};",               # at f_min: A < a*_lo (A24)
            "setp.lt.or.f32 phi{c}, {D}, {ahi}, pt{c};",                 # next level f_max iff A < a*[f]
            "selp.b32 shi{c}, 0x3FF00000, 0, pthr{c};",                  # 1.0 if throttled, else 0.0 (low word 0)
            "mov.b64 {s}, {{slo{c}, shi{c}}};",
            "fma.rn.f64 {exc}, {s}, dd{c}, {exc};",                      # sum of D over throttled ticks (exact)
            "@pthr{c} add.f32 {nthr}, {nthr}, 0f3F800000;",
            "@phi{c} mad.lo.u32 {wcmd}, {one}, {bit}, {wcmd};",
        ]
        for tmpl in per_chain:
            for c in range(C):
                body.append(tmpl.format(c=c, D=f"D{tt * 4 + c}", Blo=R("Blo"), ahi=R("ahi"), alo=R("alo"),
                                        s=R(f"s{c}"), exc=R(f"exc{c}"), nthr=R(f"nthr{c}"), wcmd=R(f"wcmd{c}"),
                                        one=R("one"), bit=1 << (TC - 1 - tt)))
    body.append("}")
    params = ", ".join(n for n, _ in names + inames)
    name = "MAGUS_TLSTAGE"
    out = [f"#define {name}(...) {name}_(__VA_ARGS__)", f"#define {name}_({params}) \\", "    asm volatile( \\"]
    out += [f'        "{l}\\n\\t" \\' for l in body]
    out.append("        : " + ", ".join(f'"{c}"({n})' for n, c in names) + " \\")
    out.append("        : " + ", ".join(f'"{c}"({n})' for n, c in inames) + " \\")
    out.append('        : "memory")')
    return out


def build_stage_o(K, TC=8, sym=False, batch=False):
    """MAGUS_OSTAGE[S]_K<K>: the solo kernel's steady stage for the open-loop observation model (A30, NEXT-3): the
    observation is the recorded sample itself (A = D, never throttled), so Alg. 1's derivative, the tune flags and Alg.
    2's lock depend on the trace only and the level is a last-writer scan of the events (lock | flag).  The L stage
    (build_stage_l) without the throttle test, the select of A and the excess / throttle accounting, plus an event word
    (shifted once per stage like the cmd word, bit TC-1-tt = tick tt had lock | flag) from which the kernel takes a
    segment's first event -- the exact open-loop fix-up (post_kernels.cuh) corrects a wrong speculative entry level in
    closed form from it, without a chain walk.  batch=True (MAGUS_OBSTAGE[S]_K<K>): the tune-flag log of
    build_stage_l(batch=True) (once-per-stage shift, immediate leaving-flag masks, count scaled by 2^TC)."""
    C = 4
    names = [(f"r{c}_{i}", "+d") for c in range(C) for i in range(K)] + \
            [(f"evh{c}", "+r") for c in range(C)] + [(f"cnt{c}", "+r") for c in range(C)] + \
            [(f"nlk{c}", "+r") for c in range(C)] + [(f"wcmd{c}", "+r") for c in range(C)] + \
            [(f"ewd{c}", "+r") for c in range(C)] + [("vmax", "+r")]
    inames = [("tile", "r"), ("dinc", "d"), ("ddec", "d"), ("bitc", "r"), ("one", "r"), ("mone", "r")] + \
             ([("cm1", "r")] if batch else [])
    idx = {n: f"%{i}" for i, (n, _) in enumerate(names + inames)}
    R = idx.__getitem__
    body = ["{", ".reg .pred phi<4>, pinc<4>, pev<4>, pk<4>, pq<4>, pe<4>;",
            f".reg .b32 D<{TC * C}>;", f".reg .f64 dv<4>, da<4>, ad<{TC * C}>;",
            ".reg .b32 tb<4>, tl<4>, lv<4>, eo<4>;"]
    for c in range(C):
        body.append(f"and.b32 lv{c}, {R(f'wcmd{c}')}, 1;")
        body.append(f"setp.ne.u32 phi{c}, lv{c}, 0;")                   # level = the previous tick's cmd
        body.append(f"shl.b32 {R(f'wcmd{c}')}, {R(f'wcmd{c}')}, {TC};")
        body.append(f"shl.b32 {R(f'ewd{c}')}, {R(f'ewd{c}')}, {TC};")
        if batch:
            body.append(f"shl.b32 {R(f'evh{c}')}, {R(f'evh{c}')}, {TC};")
            body.append(f"shr.u32 eo{c}, {R(f'evh{c}')}, {R('cm1')};")
    for tt in range(TC):
        body.append(f"ld.shared.v4.f32 {{D{tt * C}, D{tt * C + 1}, D{tt * C + 2}, D{tt * C + 3}}}, [{R('tile')}+{tt * 512}];")
        per_chain = [
            "cvt.f64.f32 {ad}, {D};",                                     # A = D (open loop, A30)
            "sub.f64 dv{c}, {ad}, {old};",                                # Alg. 1 numerator A_t - A_{t-k}
        ] + ([
            "abs.f64 da{c}, dv{c};",                                      # symmetric thresholds (d*_dec = -d*_inc):
            "setp.gt.f64 pev{c}, da{c}, {dinc};",                         # tune flag iff |d| > d*_inc
            "setp.ge.and.f64 pk{c}, dv{c}, {ddec}, phi{c};",              # f_max and not -1
            "setp.gt.or.f64 pq{c}, dv{c}, {dinc}, pk{c};",                # +1 || (f_max && !-1)
        ] if sym else [
            "setp.gt.f64 pinc{c}, dv{c}, {dinc};",                        # +1
            "setp.lt.or.f64 pev{c}, dv{c}, {ddec}, pinc{c};",             # tune flag: +1 or -1
            "not.pred pk{c}, pev{c};",
            "and.pred pk{c}, pk{c}, phi{c};",
            "or.pred pq{c}, pk{c}, pinc{c};",                             # +1 || (f_max && !flag)
        ]) + [
        ] + ([
            "and.b32 tb{c}, eo{c}, {bmt};",                               # the flag leaving the C-window (<< TC-tt)
            "@pev{c} mad.lo.u32 {evh}, {one}, {bit}, {evh};",            # the tune-flag log, bit TC-1-tt
            "mad.lo.u32 {cnt}, tb{c}, {nk}, {cnt};",                      # window count: - leaving (x 2^tt)
            "@pev{c} mad.lo.u32 {cnt}, {one}, {bitin}, {cnt};",           # + entering
        ] if batch else [
            "and.b32 tb{c}, {evh}, {bitc};",                              # the flag leaving the C-window (scaled)
            "shl.b32 {evh}, {evh}, 1;",
            "@pev{c} mad.lo.u32 {evh}, {one}, {one}, {evh};",
            "mad.lo.u32 {cnt}, tb{c}, {mone}, {cnt};",                    # window count: - leaving + entering
            "@pev{c} mad.lo.u32 {cnt}, {bitc}, {one}, {cnt};",
        ]) + [
            "setp.ge.or.s32 phi{c}, {cnt}, 0, pq{c};",                    # || lock (Alg. 2): the new level
            "setp.ge.or.s32 pe{c}, {cnt}, 0, pev{c};",                    # event: lock || flag (the level is set)
            "shr.u32 tl{c}, {cnt}, 31;",                                  # not locked
            "add.u32 {nlk}, {nlk}, tl{c};",
            "@phi{c} mad.lo.u32 {wcmd}, {one}, {bit}, {wcmd};",
            "@pe{c} mad.lo.u32 {ewd}, {one}, {bit}, {ewd};",
            "max.u32 {vmax}, {vmax}, {D};",                               # validation (A17)
        ]
        for tmpl in per_chain:
            for c in range(C):
                t = tt * C + c
                old = f"ad{(tt - K) * C + c}" if tt >= K else R(f"r{c}_{K - 1 - tt}")
                body.append(tmpl.format(c=c, D=f"D{t}", ad=f"ad{t}", old=old, dinc=R("dinc"), ddec=R("ddec"),
                                        evh=R(f"evh{c}"), one=R("one"), bitc=R("bitc"), mone=R("mone"),
                                        cnt=R(f"cnt{c}"), nlk=R(f"nlk{c}"), wcmd=R(f"wcmd{c}"), ewd=R(f"ewd{c}"),
                                        vmax=R("vmax"), bit=1 << (TC - 1 - tt), bmt=1 << (TC - tt), nk=-(1 << tt),
                                        bitin=1 << TC))
    for c in range(C):
        for i in range(K):   # ring newest first: r_i = A_{t0 + TC - 1 - i}
            body.append(f"mov.f64 {R(f'r{c}_{i}')}, ad{(TC - 1 - i) * C + c};")
    body.append("}")
    params = ", ".join(n for n, _ in names + inames)
    name = f"MAGUS_O{'B' if batch else ''}STAGE{'S' if sym else ''}_K{K}"
    out = [f"#define {name}(...) {name}_(__VA_ARGS__)", f"#define {name}_({params}) \\", "    asm volatile( \\"]
    out += [f'        "{l}\\n\\t" \\' for l in body]
    out.append("        : " + ", ".join(f'"{c}"({n})' for n, c in names) + " \\")
    out.append("        : " + ", ".join(f'"{c}"({n})' for n, c in inames) + " \\")
    out.append('        : "memory")')
    return out


def build_stage_u(K, TC=8, sym=False, popc=True, bits=False):
    """MAGUS_USTAGE{S}{I}{B}_K<K>: the solo kernel's one stage block for warm-up AND steady state (TC ticks x 4
    chains, tile loads included), with the 3-DSETP level logic (the new level is lock | +1 | (level & !-1)).
    - Alg. 1 gating (A7) by data: a chain (re)starts with its ring of A values filled with NaN, so the first k
      derivatives are NaN and every comparison on them is false (no tune flag; the level is kept: the 'not -1'
      test is the unordered setp.geu) -- the paper's "not ready" without a per-tick predicate;
    - Alg. 2 gating (A8) by per-tick warp-uniform operands g0..g7: popc=True (Alg. 2 = popc(log & g_t) >= s_min)
      g_t = the low-C-bits mask once C flags have been logged (tick >= k + C - 1 of the chain's run), else 0;
      popc=False (I: the scaled incremental window count, no XU popcount) g_t = s_min << (C-1) once full, else
      0xFFFFFFFF.  Not-ready ticks shift zeros into the flag register; they have left the window when it is full.
    - sym (S): the tune flag is |d| > d*_inc (policies with d*_dec == -d*_inc).
    - bits (B): the fp32 -> fp64 conversion of a sample by integer ops (hi = (x >> 3) + 0x38000000, lo = x << 29)
      instead of F2F on the XU pipe.  Exact for normal samples; a zero or subnormal sample becomes 2^-127 + x/2,
      which changes no decision when |d*_inc|, |d*_dec| >= 2^-60 and B_lo is normal: the
      host uses this variant only then."""
    C = 4
    names = [(f"f{c}", "+r") for c in range(C)] + \
            [(f"r{c}_{i}", "+d") for c in range(C) for i in range(K)] + \
            [(f"evh{c}", "+r") for c in range(C)] + \
            ([] if popc else [(f"cnt{c}", "+r") for c in range(C)]) + \
            [(f"exc{c}", "+d") for c in range(C)] + [(f"lock{c}", "+f") for c in range(C)] + \
            [(f"nthr{c}", "+f") for c in range(C)] + [(f"wcmd{c}", "+r") for c in range(C)] + [("vmax", "+r")]
    inames = [("tile", "r"), ("Blo", "f"), ("Blod", "d"), ("dinc", "d"), ("ddec", "d")] + \
             [(f"g{tt}", "r") for tt in range(TC)] + ([("smin", "r")] if popc else [("bitc", "r"), ("mone", "r")]) + \
             [("one", "r")]
    idx = {n: f"%{i}" for i, (n, _) in enumerate(names + inames)}
    R = idx.__getitem__
    body = ["{", ".reg .pred phi<4>, pthr<4>, pinc<4>, pev<4>, phf<4>, pk<4>;",
            f".reg .b32 D<{TC * C}>;", f".reg .f64 dd<4>, dv<4>, da<4>, dx<4>, ad<{TC * C}>;",
            ".reg .b32 wv<4>, pc<4>, tb<4>, xh<4>, xl<4>;"]
    for c in range(C):
        body.append(f"setp.ne.u32 phi{c}, {R(f'f{c}')}, 0;")
    for tt in range(TC):
        body.append(f"ld.shared.v4.f32 {{D{tt * C}, D{tt * C + 1}, D{tt * C + 2}, D{tt * C + 3}}}, [{R('tile')}+{tt * 512}];")
        conv = ([
            "shr.u32 xh{c}, {D}, 3;",
            "add.u32 xh{c}, xh{c}, 0x38000000;",
            "shl.b32 xl{c}, {D}, 29;",
            "mov.b64 dd{c}, {{xl{c}, xh{c}}};",
        ] if bits else ["cvt.f64.f32 dd{c}, {D};"])
        per_chain = conv + [
            "setp.gt.and.f32 pthr{c}, {D}, {Blo}, !phi{c};",             # throttled: f_min and D > B_lo (A14)
            "selp.f64 {ad}, {Blod}, dd{c}, pthr{c};",                     # A = min(D, B[f]) as fp64 (exact)
            "sub.f64 dv{c}, {ad}, {old};",                                # Alg. 1 numerator A_t - A_{t-k}
        ] + ([
            "abs.f64 da{c}, dv{c};",
            "setp.gt.f64 pev{c}, da{c}, {dinc};",                         # tune flag iff |d| > d*_inc
            "setp.geu.and.f64 pk{c}, dv{c}, {ddec}, phi{c};",             # level kept: f_max and not -1
            "setp.gt.or.f64 pk{c}, dv{c}, {dinc}, pk{c};",                # ... or +1
        ] if sym else [
            "setp.gt.f64 pinc{c}, dv{c}, {dinc};",                        # +1
            "setp.lt.or.f64 pev{c}, dv{c}, {ddec}, pinc{c};",             # tune flag: +1 or -1
            "setp.geu.and.f64 pk{c}, dv{c}, {ddec}, phi{c};",             # level kept: f_max and not -1
            "or.pred pk{c}, pk{c}, pinc{c};",
        ]) + ([
            "shl.b32 {evh}, {evh}, 1;",
            "@pev{c} mad.lo.u32 {evh}, {one}, {one}, {evh};",
            "and.b32 wv{c}, {evh}, {g};",                                 # the last C flags once the log is full
            "popc.b32 pc{c}, wv{c};",
            "setp.ge.u32 phf{c}, pc{c}, {smin};",                         # Alg. 2
        ] if popc else [
            "and.b32 tb{c}, {evh}, {bitc};",                              # the flag leaving the C-window (scaled)
            "shl.b32 {evh}, {evh}, 1;",
            "@pev{c} mad.lo.u32 {evh}, {one}, {one}, {evh};",
            "mad.lo.u32 {cnt}, tb{c}, {mone}, {cnt};",                    # window count: - leaving + entering
            "@pev{c} mad.lo.u32 {cnt}, {bitc}, {one}, {cnt};",
            "setp.ge.u32 phf{c}, {cnt}, {g};",                            # Alg. 2, once the log is full
        ]) + [
            "or.pred phi{c}, pk{c}, phf{c};",                             # lock || +1 || (f_max && !-1)
            "shl.b32 {wcmd}, {wcmd}, 1;",
            "@phi{c} mad.lo.u32 {wcmd}, {one}, {one}, {wcmd};",
            "sub.f64 dx{c}, dd{c}, {ad};",                                # throttling excess D - A (0 unless thr)
            "add.f64 {exc}, {exc}, dx{c};",
            "@phf{c} add.f32 {lock}, {lock}, 0f3F800000;",
            "@pthr{c} add.f32 {nthr}, {nthr}, 0f3F800000;",
            "max.u32 {vmax}, {vmax}, {D};",                               # validation (A17)
        ]
        for tmpl in per_chain:
            for c in range(C):
                t = tt * C + c
                old = f"ad{(tt - K) * C + c}" if tt >= K else R(f"r{c}_{K - 1 - tt}")
                body.append(tmpl.format(c=c, D=f"D{t}", ad=f"ad{t}", old=old, Blo=R("Blo"), Blod=R("Blod"),
                                        dinc=R("dinc"), ddec=R("ddec"), evh=R(f"evh{c}"), one=R("one"),
                                        g=R(f"g{tt}"), smin=R("smin") if popc else None,
                                        bitc=None if popc else R("bitc"), mone=None if popc else R("mone"),
                                        cnt=None if popc else R(f"cnt{c}"), wcmd=R(f"wcmd{c}"), exc=R(f"exc{c}"),
                                        lock=R(f"lock{c}"), nthr=R(f"nthr{c}"), vmax=R("vmax")))
    for c in range(C):
        body.append(f"selp.u32 {R(f'f{c}')}, 1, 0, phi{c};")
        for i in range(K):   # ring newest first: r_i = A_{t0 + TC - 1 - i}
            body.append(f"mov.f64 {R(f'r{c}_{i}')}, ad{(TC - 1 - i) * C + c};")
    body.append("}")
    params = ", ".join(n for n, _ in names + inames)
    name = f"MAGUS_USTAGE{'S' if sym else ''}{'' if popc else 'I'}{'B' if bits else ''}_K{K}"
    out = [f"#define {name}(...) {name}_(__VA_ARGS__)", f"#define {name}_({params}) \\", "    asm volatile( \\"]
    out += [f'        "{l}\\n\\t" \\' for l in body]
    out.append("        : " + ", ".join(f'"{c}"({n})' for n, c in names) + " \\")
    out.append("        : " + ", ".join(f'"{c}"({n})' for n, c in inames) + " \\")
    out.append('        : "memory")')
    return out


def build_stage_t(NP, TC=8):
    """MAGUS_TSTAGE{NP}: one steady stage (TC ticks x 4 traces x NP TDP_DEFAULT policies) of the TDP solo kernel
    (the Intel-default baseline, A24).  Per (trace, policy) chain and tick:
      throttled = f_min && D > B_lo (A14);  next level f_max iff D < a[f] -- a[f_max] = a*_hi; a[f_min] = a*_lo if
      B_lo >= a*_lo else +inf (A = min(D, B_lo) at f_min), the host-derived exact equivalents of
      fl(P[f] + fl(c A)) >= fl((1 - m) TDP);
      sum of D over throttled ticks in fp64 by one DFMA with a 0/1 factor (exact: the terms are multiples of
      ulp(B_lo), section 8; the kernel subtracts n_thr * B_lo once per segment); the throttled count as an fp32 add;
      the cmd word.  The sample's fp64 value is converted once per trace and shared by the NP policies."""
    C = 4 * NP
    names = [(f"f{c}", "+r") for c in range(C)] + [(f"exc{c}", "+d") for c in range(C)] + \
            [(f"nthr{c}", "+f") for c in range(C)] + [(f"wcmd{c}", "+r") for c in range(C)] + [("vmax", "+r")]
    inames = [("tile", "r"), ("Blo", "f")] + [(f"ahi{p}", "f") for p in range(NP)] + \
             [(f"alo{p}", "f") for p in range(NP)] + [("one", "r")]
    idx = {n: f"%{i}" for i, (n, _) in enumerate(names + inames)}
    R = idx.__getitem__
    body = ["{", f".reg .pred phi<{C}>, pthr<{C}>;", f".reg .b32 D<{TC * 4}>, a<{C}>, sh<{C}>;",
            f".reg .f64 dd<4>, s<{C}>;"]
    for c in range(C):
        body.append(f"setp.ne.u32 phi{c}, {R(f'f{c}')}, 0;")
    for tt in range(TC):
        body.append(f"ld.shared.v4.f32 {{D{tt * 4}, D{tt * 4 + 1}, D{tt * 4 + 2}, D{tt * 4 + 3}}}, [{R('tile')}+{tt * 512}];")
        for u in range(4):
            body.append(f"cvt.f64.f32 dd{u}, D{tt * 4 + u};")
        body.append(f"max.u32 {R('vmax')}, {R('vmax')}, D{tt * 4};")
        body.append(f"max.u32 {R('vmax')}, {R('vmax')}, D{tt * 4 + 1};")
        body.append(f"max.u32 {R('vmax')}, {R('vmax')}, D{tt * 4 + 2};")
        body.append(f"max.u32 {R('vmax')}, {R('vmax')}, D{tt * 4 + 3};")
        per_chain = [
            "setp.gt.and.f32 pthr{c}, {D}, {Blo}, !phi{c};",             # throttled (A14)
            "selp.f32 a{c}, {ahi}, {alo}, phi{c};",                       # a*[f] (A24)
            "setp.lt.f32 phi{c}, {D}, a{c};",                             # next level f_max iff A < a*[f]
            "selp.b32 sh{c}, 0x3FF00000, 0, pthr{c};",
            "mov.b64 s{c}, {{0, sh{c}}};",                                # 1.0 if throttled, else 0.0
            "fma.rn.f64 {exc}, s{c}, {dd}, {exc};",                       # sum of D over throttled ticks (exact)
            "@pthr{c} add.f32 {nthr}, {nthr}, 0f3F800000;",
            "shl.b32 {wcmd}, {wcmd}, 1;",
            "@phi{c} mad.lo.u32 {wcmd}, {one}, {one}, {wcmd};",
        ]
        for tmpl in per_chain:
            for c in range(C):
                u, pp = c % 4, c // 4
                body.append(tmpl.format(c=c, D=f"D{tt * 4 + u}", dd=f"dd{u}", Blo=R("Blo"), ahi=R(f"ahi{pp}"),
                                        alo=R(f"alo{pp}"), exc=R(f"exc{c}"), nthr=R(f"nthr{c}"), wcmd=R(f"wcmd{c}"),
                                        one=R("one")))
    for c in range(C):
        body.append(f"selp.u32 {R(f'f{c}')}, 1, 0, phi{c};")
    body.append("}")
    params = ", ".join(n for n, _ in names + inames)
    name = f"MAGUS_TSTAGE{NP}"
    out = [f"#define {name}(...) {name}_(__VA_ARGS__)", f"#define {name}_({params}) \\", "    asm volatile( \\"]
    out += [f'        "{l}\\n\\t" \\' for l in body]
    out.append("        : " + ", ".join(f'"{c}"({n})' for n, c in names) + " \\")
    out.append("        : " + ", ".join(f'"{c}"({n})' for n, c in inames) + " \\")
    out.append('        : "memory")')
    return out


def build_stage_wl(K, TC=8):
    """MAGUS_WSTAGE1L_K<K>: the chain walk's one-chain stage (TC ticks of one (trace, policy) recurrence, samples
    passed in registers), same operands and decisions as MAGUS_WSTAGE1F_K<K>, restructured for a short loop-carried
    dependency (a walking warp is alone on its SM sub-partition: latency-bound).  Everything that does not depend
    on the level in effect is evaluated for BOTH levels ahead of it -- A at f_min / f_max, both derivatives
    against A_{t-k} (known k ticks earlier), their +1 / -1 / flag predicates, and the Alg. 2 window count with
    and without a new flag -- so the level recurrence per tick is three predicate selections:
      flag = level ? flag_max : flag_min;  lock = flag ? (cnt+1 >= s_min) : (cnt >= s_min);
      new level = lock | (level ? (+1_max | !-1_max) : +1_min)."""
    names = [("f0", "+r")] + [(f"r0_{i}", "+d") for i in range(K)] + \
            [("evh0", "+r"), ("cnt0", "+r"), ("exc0", "+d"), ("lock0", "+f"), ("nthr0", "+f"), ("wcmd0", "+r")]
    inames = [(f"S0_{tt}", "r") for tt in range(TC)] + [("Blo", "f"), ("Blod", "d"), ("dinc", "d"), ("ddec", "d"),
                                                         ("bitc", "r"), ("smin", "r"), ("one", "r"), ("mone", "r")]
    idx = {n: f"%{i}" for i, (n, _) in enumerate(names + inames)}
    R = idx.__getitem__
    body = ["{", ".reg .pred phi, pgt, iL, cL, iH, cH, eL, eH, gH, px, pev, h0, h1, phf, pthr;",
            f".reg .f64 dd, aL, dvL, dvH, dx, ad<{TC}>;", ".reg .b32 tb, c0, c1;",
            f"setp.ne.u32 phi, {R('f0')}, 0;"]
    for tt in range(TC):
        D = R(f"S0_{tt}")
        old = f"ad{tt - K}" if tt >= K else R(f"r0_{K - 1 - tt}")
        body += [
            f"cvt.f64.f32 dd, {D};",
            f"setp.gt.f32 pgt, {D}, {R('Blo')};",                          # D > B_lo: throttled at f_min (A14)
            f"selp.f64 aL, {R('Blod')}, dd, pgt;",                         # A at f_min; A at f_max = D
            f"sub.f64 dvL, aL, {old};",                                    # Alg. 1 numerators for both levels
            f"sub.f64 dvH, dd, {old};",
            f"setp.gt.f64 iL, dvL, {R('dinc')};",                          # +1, -1 at each level
            f"setp.lt.f64 cL, dvL, {R('ddec')};",
            f"setp.gt.f64 iH, dvH, {R('dinc')};",
            f"setp.lt.f64 cH, dvH, {R('ddec')};",
            "or.pred eL, iL, cL;",                                        # tune flag at each level
            "or.pred eH, iH, cH;",
            "not.pred gH, cH;",
            "or.pred gH, gH, iH;",                                        # at f_max: +1 or not -1 keeps / sets f_max
            f"and.b32 tb, {R('evh0')}, {R('bitc')};",                      # the flag leaving the C-window (scaled)
            f"mad.lo.u32 c0, tb, {R('mone')}, {R('cnt0')};",               # window count without / with a new flag
            f"add.u32 c1, c0, {R('bitc')};",
            f"setp.ge.u32 h0, c0, {R('smin')};",
            f"setp.ge.u32 h1, c1, {R('smin')};",
            # ---- the level-dependent part
            "and.pred px, phi, gH;",                                      # level & (+1 | !-1) at f_max ...
            "not.pred pthr, phi;",
            "and.pred pev, pthr, iL;",
            "or.pred px, px, pev;",                                       # ... | (!level & +1 at f_min)
            "and.pred pev, phi, eH;",
            "and.pred pthr, pthr, eL;",
            "or.pred pev, pev, pthr;",                                    # the tune flag at the level in effect
            "and.pred phf, pev, h1;",
            "not.pred pthr, pev;",
            "and.pred pthr, pthr, h0;",
            "or.pred phf, phf, pthr;",                                    # Alg. 2 on the updated window
            f"selp.f64 ad{tt}, dd, aL, phi;",                              # A in effect (the ring value)
            "not.pred pthr, phi;",
            "and.pred pthr, pthr, pgt;",                                  # throttled
            f"selp.b32 {R('cnt0')}, c1, c0, pev;",
            f"shl.b32 {R('evh0')}, {R('evh0')}, 1;",
            f"@pev add.u32 {R('evh0')}, {R('evh0')}, 1;",
            "or.pred phi, phf, px;",                                      # lock || +1 || (f_max && !-1)
            f"shl.b32 {R('wcmd0')}, {R('wcmd0')}, 1;",
            f"@phi add.u32 {R('wcmd0')}, {R('wcmd0')}, 1;",
            f"sub.f64 dx, dd, ad{tt};",                                    # throttling excess D - A (0 unless thr)
            f"add.f64 {R('exc0')}, {R('exc0')}, dx;",
            f"@phf add.f32 {R('lock0')}, {R('lock0')}, 0f3F800000;",
            f"@pthr add.f32 {R('nthr0')}, {R('nthr0')}, 0f3F800000;",
        ]
    body.append(f"selp.u32 {R('f0')}, 1, 0, phi;")
    for i in range(K):
        body.append(f"mov.f64 {R(f'r0_{i}')}, ad{TC - 1 - i};")
    body.append("}")
    params = ", ".join(n for n, _ in names + inames)
    name = f"MAGUS_WSTAGE1L_K{K}"
    out = [f"#define {name}(...) {name}_(__VA_ARGS__)", f"#define {name}_({params}) \\", "    asm volatile( \\"]
    out += [f'        "{l}\\n\\t" \\' for l in body]
    out.append("        : " + ", ".join(f'"{c}"({n})' for n, c in names) + " \\")
    out.append("        : " + ", ".join(f'"{c}"({n})' for n, c in inames) + " \\")
    out.append('        : "memory")')
    return out


def build_stage_w2(K, TC=8):
    """MAGUS_WSTAGE2P_K<K>: TC ticks of TWO MAGUS chains of one trace under two different policy points of the same
    chain kind (the wide kernel, replay_wide.cuh), samples passed in registers: the fp32 -> fp64 conversion is
    shared, every threshold (d*_inc, d*_dec, the scaled Alg. 2 threshold and leaving-flag bit) is per chain.
    Per chain-tick the operations and their order are MAGUS_WSTAGE1F_K<K>'s (decisions identical)."""
    C = 2
    names = [(f"f{c}", "+r") for c in range(C)] + \
            [(f"r{c}_{i}", "+d") for c in range(C) for i in range(K)] + \
            [(f"evh{c}", "+r") for c in range(C)] + [(f"cnt{c}", "+r") for c in range(C)] + \
            [(f"exc{c}", "+d") for c in range(C)] + [(f"lock{c}", "+f") for c in range(C)] + \
            [(f"nthr{c}", "+f") for c in range(C)] + [(f"wcmd{c}", "+r") for c in range(C)]
    inames = [(f"S{tt}", "r") for tt in range(TC)] + [("Blo", "f"), ("Blod", "d")] + \
             [(f"dinc{c}", "d") for c in range(C)] + [(f"ddec{c}", "d") for c in range(C)] + \
             [(f"bitc{c}", "r") for c in range(C)] + [(f"smin{c}", "r") for c in range(C)] + [("one", "r"), ("mone", "r")]
    idx = {n: f"%{i}" for i, (n, _) in enumerate(names + inames)}
    R = idx.__getitem__
    body = ["{", ".reg .pred phi<2>, pthr<2>, pinc<2>, pev<2>, phf<2>, pq<2>, pk<2>;",
            f".reg .f64 dd, dv<2>, dx<2>, ad<{TC * C}>;", ".reg .b32 tb<2>;"]
    for c in range(C):
        body.append(f"setp.ne.u32 phi{c}, {R(f'f{c}')}, 0;")
    for tt in range(TC):
        body.append(f"cvt.f64.f32 dd, {R(f'S{tt}')};")                # shared by the two chains
        per_chain = [
            "setp.gt.and.f32 pthr{c}, {D}, {Blo}, !phi{c};",             # throttled: f_min and D > B_lo (A14)
            "selp.f64 {ad}, {Blod}, dd, pthr{c};",                       # A = min(D, B[f]) as fp64 (exact)
            "sub.f64 dv{c}, {ad}, {old};",                               # Alg. 1 numerator A_t - A_{t-k}
            "setp.gt.f64 pinc{c}, dv{c}, {dinc};",                       # +1
            "setp.lt.or.f64 pev{c}, dv{c}, {ddec}, pinc{c};",            # tune flag
            "and.b32 tb{c}, {evh}, {bitc};",                             # the flag leaving the C-window (scaled)
            "shl.b32 {evh}, {evh}, 1;",
            "@pev{c} mad.lo.u32 {evh}, {one}, {one}, {evh};",
            "mad.lo.u32 {cnt}, tb{c}, {mone}, {cnt};",                   # window count: - leaving + entering
            "@pev{c} mad.lo.u32 {cnt}, {bitc}, {one}, {cnt};",
            "setp.ge.u32 phf{c}, {cnt}, {smin};",                        # Alg. 2
            "not.pred pk{c}, pev{c};",
            "and.pred pk{c}, pk{c}, phi{c};",
            "or.pred pq{c}, pk{c}, pinc{c};",                            # +1 || (f_max && !flag)
            "or.pred phi{c}, pq{c}, phf{c};",                            # || lock: the new level
            "shl.b32 {wcmd}, {wcmd}, 1;",
            "@phi{c} mad.lo.u32 {wcmd}, {one}, {one}, {wcmd};",
            "sub.f64 dx{c}, dd, {ad};",                                  # throttling excess D - A (0 unless thr)
            "add.f64 {exc}, {exc}, dx{c};",
            "@phf{c} add.f32 {lock}, {lock}, 0f3F800000;",
            "@pthr{c} add.f32 {nthr}, {nthr}, 0f3F800000;",
        ]
        for tmpl in per_chain:
            for c in range(C):
                t = tt * C + c
                old = f"ad{(tt - K) * C + c}" if tt >= K else R(f"r{c}_{K - 1 - tt}")
                body.append(tmpl.format(c=c, D=R(f"S{tt}"), ad=f"ad{t}", old=old, Blod=R("Blod"), Blo=R("Blo"),
                                        dinc=R(f"dinc{c}"), ddec=R(f"ddec{c}"), evh=R(f"evh{c}"), one=R("one"),
                                        bitc=R(f"bitc{c}"), mone=R("mone"), cnt=R(f"cnt{c}"), smin=R(f"smin{c}"),
                                        wcmd=R(f"wcmd{c}"), exc=R(f"exc{c}"), lock=R(f"lock{c}"), nthr=R(f"nthr{c}")))
    for c in range(C):
        body.append(f"selp.u32 {R(f'f{c}')}, 1, 0, phi{c};")
        for i in range(K):   # ring newest first: r_i = A_{t0 + TC - 1 - i}
            body.append(f"mov.f64 {R(f'r{c}_{i}')}, ad{(TC - 1 - i) * C + c};")
    body.append("}")
    params = ", ".join(n for n, _ in names + inames)
    name = f"MAGUS_WSTAGE2P_K{K}"
    out = [f"#define {name}(...) {name}_(__VA_ARGS__)", f"#define {name}_({params}) \\", "    asm volatile( \\"]
    out += [f'        "{l}\\n\\t" \\' for l in body]
    out.append("        : " + ", ".join(f'"{c}"({n})' for n, c in names) + " \\")
    out.append("        : " + ", ".join(f'"{c}"({n})' for n, c in inames) + " \\")
    out.append('        : "memory")')
    return out


def build_stage_w1d(K, TC=8):
    """MAGUS_WSTAGE1D_K<K>: TC ticks of ONE MAGUS chain with the samples passed as fp64 registers (the wide kernel's
    per-warp converted tile, replay_wide.cuh): MAGUS_WSTAGE1F_K<K> without the fp32 -> fp64 conversion, the throttle
    test as the fp64 compare of the same exact values (D > B_lo at f_min, A14).  Decisions identical."""
    names = [("f0", "+r")] + [(f"r0_{i}", "+d") for i in range(K)] + \
            [("evh0", "+r"), ("cnt0", "+r"), ("exc0", "+d"), ("lock0", "+f"), ("nthr0", "+f"), ("wcmd0", "+r")]
    inames = [(f"S{tt}", "d") for tt in range(TC)] + [("Blod", "d"), ("dinc", "d"), ("ddec", "d"), ("bitc", "r"),
                                                     ("smin", "r"), ("one", "r"), ("mone", "r")]
    idx = {n: f"%{i}" for i, (n, _) in enumerate(names + inames)}
    R = idx.__getitem__
    body = ["{", ".reg .pred phi, pthr, pinc, pev, phf, pq, pk;", f".reg .f64 dv, dx, ad<{TC}>;", ".reg .b32 tb;",
            f"setp.ne.u32 phi, {R('f0')}, 0;"]
    for tt in range(TC):
        dd = R(f"S{tt}")
        old = f"ad{tt - K}" if tt >= K else R(f"r0_{K - 1 - tt}")
        body += [
            f"setp.gt.and.f64 pthr, {dd}, {R('Blod')}, !phi;",             # throttled: f_min and D > B_lo (A14)
            f"selp.f64 ad{tt}, {R('Blod')}, {dd}, pthr;",                   # A = min(D, B[f]) (exact)
            f"sub.f64 dv, ad{tt}, {old};",                                  # Alg. 1 numerator A_t - A_{t-k}
            f"setp.gt.f64 pinc, dv, {R('dinc')};",                          # +1
            f"setp.lt.or.f64 pev, dv, {R('ddec')}, pinc;",                  # tune flag
            f"and.b32 tb, {R('evh0')}, {R('bitc')};",                       # the flag leaving the C-window (scaled)
            f"shl.b32 {R('evh0')}, {R('evh0')}, 1;",
            f"@pev mad.lo.u32 {R('evh0')}, {R('one')}, {R('one')}, {R('evh0')};",
            f"mad.lo.u32 {R('cnt0')}, tb, {R('mone')}, {R('cnt0')};",        # window count: - leaving + entering
            f"@pev mad.lo.u32 {R('cnt0')}, {R('bitc')}, {R('one')}, {R('cnt0')};",
            f"setp.ge.u32 phf, {R('cnt0')}, {R('smin')};",                  # Alg. 2
            "not.pred pk, pev;",
            "and.pred pk, pk, phi;",
            "or.pred pq, pk, pinc;",                                       # +1 || (f_max && !flag)
            "or.pred phi, pq, phf;",                                       # || lock: the new level
            f"shl.b32 {R('wcmd0')}, {R('wcmd0')}, 1;",
            f"@phi mad.lo.u32 {R('wcmd0')}, {R('one')}, {R('one')}, {R('wcmd0')};",
            f"sub.f64 dx, {dd}, ad{tt};",                                   # throttling excess D - A (0 unless thr)
            f"add.f64 {R('exc0')}, {R('exc0')}, dx;",
            f"@phf add.f32 {R('lock0')}, {R('lock0')}, 0f3F800000;",
            f"@pthr add.f32 {R('nthr0')}, {R('nthr0')}, 0f3F800000;",
        ]
    body.append(f"selp.u32 {R('f0')}, 1, 0, phi;")
    for i in range(K):
        body.append(f"mov.f64 {R(f'r0_{i}')}, ad{TC - 1 - i};")
    body.append("}")
    params = ", ".join(n for n, _ in names + inames)
    name = f"MAGUS_WSTAGE1D_K{K}"
    out = [f"#define {name}(...) {name}_(__VA_ARGS__)", f"#define {name}_({params}) \\", "    asm volatile( \\"]
    out += [f'        "{l}\\n\\t" \\' for l in body]
    out.append("        : " + ", ".join(f'"{c}"({n})' for n, c in names) + " \\")
    out.append("        : " + ", ".join(f'"{c}"({n})' for n, c in inames) + " \\")
    out.append('        : "memory")')
    return out


def build_stage_w1l(K, TC=8, sym=False):
    """MAGUS_WLSTAGE[S]_K<K>: MAGUS_WSTAGE1D_K<K> (one chain, fp64 samples; the wide kernel) with the L-stage
    transformations of MAGUS_LSTAGE_K<K> (build_stage_l): the level carried in the cmd word (shifted once per
    TC ticks, bit 0 = the previous tick's cmd), Alg. 2's lock as the sign of the window count biased by
    -s_min << (C-1) with the not-locked ticks counted by the sign bit, and (sym) the |d| tune-flag test."""
    names = [(f"r0_{i}", "+d") for i in range(K)] + \
            [("evh0", "+r"), ("cnt0", "+r"), ("exc0", "+d"), ("nlk0", "+r"), ("nthr0", "+f"), ("wcmd0", "+r")]
    inames = [(f"S{tt}", "d") for tt in range(TC)] + [("Blod", "d"), ("dinc", "d"), ("ddec", "d"), ("bitc", "r"),
                                                     ("one", "r"), ("mone", "r")]
    idx = {n: f"%{i}" for i, (n, _) in enumerate(names + inames)}
    R = idx.__getitem__
    body = ["{", ".reg .pred phi, pthr, pinc, pev, pq, pk;", f".reg .f64 dv, da, dx, ad<{TC}>;", ".reg .b32 tb, tl, lv;",
            f"and.b32 lv, {R('wcmd0')}, 1;", "setp.ne.u32 phi, lv, 0;",      # level = the previous tick's cmd
            f"shl.b32 {R('wcmd0')}, {R('wcmd0')}, {TC};"]
    for tt in range(TC):
        dd = R(f"S{tt}")
        old = f"ad{tt - K}" if tt >= K else R(f"r0_{K - 1 - tt}")
        body += [
            f"setp.gt.and.f64 pthr, {dd}, {R('Blod')}, !phi;",             # throttled: f_min and D > B_lo (A14)
            f"selp.f64 ad{tt}, {R('Blod')}, {dd}, pthr;",                   # A = min(D, B[f]) (exact)
            f"sub.f64 dv, ad{tt}, {old};",                                  # Alg. 1 numerator A_t - A_{t-k}
        ] + ([
            "abs.f64 da, dv;",                                             # symmetric thresholds (d*_dec = -d*_inc):
            f"setp.gt.f64 pev, da, {R('dinc')};",                           # tune flag iff |d| > d*_inc
            f"setp.ge.and.f64 pk, dv, {R('ddec')}, phi;",                   # f_max and not -1
            f"setp.gt.or.f64 pq, dv, {R('dinc')}, pk;",                     # +1 || (f_max && !-1)
        ] if sym else [
            f"setp.gt.f64 pinc, dv, {R('dinc')};",                          # +1
            f"setp.lt.or.f64 pev, dv, {R('ddec')}, pinc;",                  # tune flag
            "not.pred pk, pev;",
            "and.pred pk, pk, phi;",
            "or.pred pq, pk, pinc;",                                       # +1 || (f_max && !flag)
        ]) + [
            f"and.b32 tb, {R('evh0')}, {R('bitc')};",                       # the flag leaving the C-window (scaled)
            f"shl.b32 {R('evh0')}, {R('evh0')}, 1;",
            f"@pev mad.lo.u32 {R('evh0')}, {R('one')}, {R('one')}, {R('evh0')};",
            f"mad.lo.u32 {R('cnt0')}, tb, {R('mone')}, {R('cnt0')};",        # window count: - leaving + entering
            f"@pev mad.lo.u32 {R('cnt0')}, {R('bitc')}, {R('one')}, {R('cnt0')};",
            f"setp.ge.or.s32 phi, {R('cnt0')}, 0, pq;",                     # || lock (Alg. 2): the new level
            f"shr.u32 tl, {R('cnt0')}, 31;",                                # not locked
            f"add.u32 {R('nlk0')}, {R('nlk0')}, tl;",
            f"@phi mad.lo.u32 {R('wcmd0')}, {R('one')}, {1 << (TC - 1 - tt)}, {R('wcmd0')};",
            f"sub.f64 dx, {dd}, ad{tt};",                                   # throttling excess D - A (0 unless thr)
            f"add.f64 {R('exc0')}, {R('exc0')}, dx;",
            f"@pthr add.f32 {R('nthr0')}, {R('nthr0')}, 0f3F800000;",
        ]
    for i in range(K):
        body.append(f"mov.f64 {R(f'r0_{i}')}, ad{TC - 1 - i};")
    body.append("}")
    params = ", ".join(n for n, _ in names + inames)
    name = f"MAGUS_WLSTAGE{'S' if sym else ''}_K{K}"
    out = [f"#define {name}(...) {name}_(__VA_ARGS__)", f"#define {name}_({params}) \\", "    asm volatile( \\"]
    out += [f'        "{l}\\n\\t" \\' for l in body]
    out.append("        : " + ", ".join(f'"{c}"({n})' for n, c in names) + " \\")
    out.append("        : " + ", ".join(f'"{c}"({n})' for n, c in inames) + " \\")
    out.append('        : "memory")')
    return out


def build_stage_w1p(K, TC=8, sym=False):
    """MAGUS_WPSTAGE[S]_K<K>: the wide kernel's one-chain L stage (MAGUS_WLSTAGE[S]_K<K>) with the level-independent
    work taken off the per-tick dependency chain (the wide kernel is latency-bound: one chain per thread):
    - the warp's conversion step also stores min(D, B_lo) as fp64 (L<tt>), so A = level ? D : min(D, B_lo) is one
      select by the level itself -- no throttle test on the level -> A path;
    - the throttled ticks are not counted per tick: the caller takes popc(~level word & ballot(D > B_lo)) per
      32-tick block (exact: throttled iff f_min and D > B_lo, A14);
    - the new level is (lock | +1) | (level & !-1): the lock ISETP.OR and the (d >= d*_dec) & level DSETP run side by
      side and one PLOP3 joins them, one FP64 compare shorter than the L stage's DSETP -> DSETP.OR -> ISETP.OR."""
    names = [(f"r0_{i}", "+d") for i in range(K)] + \
            [("evh0", "+r"), ("cnt0", "+r"), ("exc0", "+d"), ("nlk0", "+r"), ("wcmd0", "+r")]
    inames = [(f"S{tt}", "d") for tt in range(TC)] + [(f"L{tt}", "d") for tt in range(TC)] + \
             [("dinc", "d"), ("ddec", "d"), ("bitc", "r"), ("one", "r"), ("mone", "r")]
    idx = {n: f"%{i}" for i, (n, _) in enumerate(names + inames)}
    R = idx.__getitem__
    body = ["{", ".reg .pred phi, pinc, pev, pk, pl;", f".reg .f64 dv, da, dx, ad<{TC}>;", ".reg .b32 tb, tl, lv;",
            f"and.b32 lv, {R('wcmd0')}, 1;", "setp.ne.u32 phi, lv, 0;",      # level = the previous tick's cmd
            f"shl.b32 {R('wcmd0')}, {R('wcmd0')}, {TC};"]
    for tt in range(TC):
        dd, lo = R(f"S{tt}"), R(f"L{tt}")
        old = f"ad{tt - K}" if tt >= K else R(f"r0_{K - 1 - tt}")
        body += [
            f"selp.f64 ad{tt}, {dd}, {lo}, phi;",                           # A = min(D, B[f]) (A14; exact)
            f"sub.f64 dv, ad{tt}, {old};",                                  # Alg. 1 numerator A_t - A_{t-k}
            f"setp.gt.f64 pinc, dv, {R('dinc')};",                          # +1
        ] + ([
            "abs.f64 da, dv;",                                             # symmetric thresholds (d*_dec = -d*_inc):
            f"setp.gt.f64 pev, da, {R('dinc')};",                           # tune flag iff |d| > d*_inc
        ] if sym else [
            f"setp.lt.or.f64 pev, dv, {R('ddec')}, pinc;",                  # tune flag
        ]) + [
            f"setp.ge.and.f64 pk, dv, {R('ddec')}, phi;",                   # f_max and not -1
            f"and.b32 tb, {R('evh0')}, {R('bitc')};",                       # the flag leaving the C-window (scaled)
            f"shl.b32 {R('evh0')}, {R('evh0')}, 1;",
            f"@pev mad.lo.u32 {R('evh0')}, {R('one')}, {R('one')}, {R('evh0')};",
            f"mad.lo.u32 {R('cnt0')}, tb, {R('mone')}, {R('cnt0')};",        # window count: - leaving + entering
            f"@pev mad.lo.u32 {R('cnt0')}, {R('bitc')}, {R('one')}, {R('cnt0')};",
            f"setp.ge.or.s32 pl, {R('cnt0')}, 0, pinc;",                    # lock (Alg. 2) || +1
            "or.pred phi, pl, pk;",                                        # || (f_max && !-1): the new level
            f"shr.u32 tl, {R('cnt0')}, 31;",                                # not locked
            f"add.u32 {R('nlk0')}, {R('nlk0')}, tl;",
            f"@phi mad.lo.u32 {R('wcmd0')}, {R('one')}, {1 << (TC - 1 - tt)}, {R('wcmd0')};",
            f"sub.f64 dx, {dd}, ad{tt};",                                   # throttling excess D - A (0 unless thr)
            f"add.f64 {R('exc0')}, {R('exc0')}, dx;",
        ]
    for i in range(K):
        body.append(f"mov.f64 {R(f'r0_{i}')}, ad{TC - 1 - i};")
    body.append("}")
    params = ", ".join(n for n, _ in names + inames)
    name = f"MAGUS_WPSTAGE{'S' if sym else ''}_K{K}"
    out = [f"#define {name}(...) {name}_(__VA_ARGS__)", f"#define {name}_({params}) \\", "    asm volatile( \\"]
    out += [f'        "{l}\\n\\t" \\' for l in body]
    out.append("        : " + ", ".join(f'"{c}"({n})' for n, c in names) + " \\")
    out.append("        : " + ", ".join(f'"{c}"({n})' for n, c in inames) + " \\")
    out.append('        : "memory")')
    return out


def build_stage_t1(validate):
    """MAGUS_TSTAGE1L{V}: one steady stage (8 ticks x 4 traces) of ONE TDP_DEFAULT policy (the TDP solo kernel, NP = 1)
    with fewer instructions than MAGUS_TSTAGE1: the next level as two fp32 compares without a select,
        f' = (D < a_hi) | (!f & D < a_lo)   (= D < a[f], because a_lo >= a_hi: a*[f] is monotone in P[f], P_lo <= P_hi,
                                             and a_lo is a*_lo or +inf),
    the 0/1 factor of the throttled-demand DFMA kept in a persistent register pair whose low word stays 0 (only the
    high word is rewritten per tick: no zeroing move), and the validation maximum only when V (the first launch
    group validates every sample; the union of all lanes' maxima is what is checked, A17)."""
    C, TC = 4, 8
    names = [(f"f{c}", "+r") for c in range(C)] + [(f"exc{c}", "+d") for c in range(C)] + \
            [(f"nthr{c}", "+f") for c in range(C)] + [(f"wcmd{c}", "+r") for c in range(C)] + \
            [(f"s{c}", "+d") for c in range(C)] + ([("vmax", "+r")] if validate else [])
    inames = [("tile", "r"), ("Blo", "f"), ("ahi", "f"), ("alo", "f"), ("one", "r")]
    idx = {n: f"%{i}" for i, (n, _) in enumerate(names + inames)}
    R = idx.__getitem__
    body = ["{", f".reg .pred phi<{C}>, pthr<{C}>, pt<{C}>;", f".reg .b32 D<{TC * 4}>, slo<{C}>, shi<{C}>;",
            ".reg .f64 dd<4>;"]
    for c in range(C):
        body.append(f"setp.ne.u32 phi{c}, {R(f'f{c}')}, 0;")
        body.append(f"mov.b64 {{slo{c}, shi{c}}}, {R(f's{c}')};")
    for tt in range(TC):
        body.append(f"ld.shared.v4.f32 {{D{tt * 4}, D{tt * 4 + 1}, D{tt * 4 + 2}, D{tt * 4 + 3}}}, [{R('tile')}+{tt * 512}];")
        for u in range(4):
            body.append(f"cvt.f64.f32 dd{u}, D{tt * 4 + u};")
        if validate:
            body.append(f"max.u32 {R('vmax')}, {R('vmax')}, D{tt * 4};")
            body.append(f"max.u32 {R('vmax')}, {R('vmax')}, D{tt * 4 + 1};")
            body.append(f"max.u32 {R('vmax')}, {R('vmax')}, D{tt * 4 + 2};")
            body.append(f"max.u32 {R('vmax')}, {R('vmax')}, D{tt * 4 + 3};")
        per_chain = [
            "setp.gt.and.f32 pthr{c}, {D}, {Blo}, !phi{c};",             # throttled (A14)
            "setp.lt.and.f32 pt{c}, {D}, {alo}, !phi{c};",               # at f_min: A < a*_lo (A24)
            "setp.lt.or.f32 phi{c}, {D}, {ahi}, pt{c};",                 # next level f_max iff A < a*[f]
            "selp.b32 shi{c}, 0x3FF00000, 0, pthr{c};",                  # 1.0 if throttled, else 0.0 (low word 0)
            "mov.b64 {s}, {{slo{c}, shi{c}}};",
            "fma.rn.f64 {exc}, {s}, dd{u}, {exc};",                      # sum of D over throttled ticks (exact)
            "@pthr{c} add.f32 {nthr}, {nthr}, 0f3F800000;",
            "shl.b32 {wcmd}, {wcmd}, 1;",
            "@phi{c} mad.lo.u32 {wcmd}, {one}, {one}, {wcmd};",
        ]
        for tmpl in per_chain:
            for c in range(C):
                body.append(tmpl.format(c=c, u=c, D=f"D{tt * 4 + c}", Blo=R("Blo"), ahi=R("ahi"), alo=R("alo"),
                                        s=R(f"s{c}"), exc=R(f"exc{c}"), nthr=R(f"nthr{c}"), wcmd=R(f"wcmd{c}"),
                                        one=R("one")))
    for c in range(C):
        body.append(f"selp.u32 {R(f'f{c}')}, 1, 0, phi{c};")
    body.append("}")
    params = ", ".join(n for n, _ in names + inames)
    name = f"MAGUS_TSTAGE1L{'V' if validate else ''}"
    out = [f"#define {name}(...) {name}_(__VA_ARGS__)", f"#define {name}_({params}) \\", "    asm volatile( \\"]
    out += [f'        "{l}\\n\\t" \\' for l in body]
    out.append("        : " + ", ".join(f'"{c}"({n})' for n, c in names) + " \\")
    out.append("        : " + ", ".join(f'"{c}"({n})' for n, c in inames) + " \\")
    out.append('        : "memory")')
    return out


out = ["// GENERATED by scripts/gen_tick4.py -- do not edit.  One MAGUS tick for the 4 chains of a lane, the",
       "// four chains' instructions interleaved (DESIGN.md section 7); semantics = magus_tick<K, false, SLOW>.",
       "// cnt is the window count scaled by 2^(C-1).",
       "#pragma once"]
out += build(False) + [""] + build(True)
for K in (1, 2, 3):
    out += [""] + build_stage(K)
    out += [""] + build_stage_f(K)
    out += [""] + build_stage_f(K, thr64=False)
    out += [""] + build_stage_f(K, thr64=False, bits=True)
    out += [""] + build_stage_l(K)
    out += [""] + build_stage_l(K, sym=True)
    out += [""] + build_stage_l(K, tdp=True)
    out += [""] + build_stage_l(K, sym=True, tdp=True)
    out += [""] + build_stage_l(K, tdp=True, tdp_up=True)
    out += [""] + build_stage_l(K, sym=True, tdp=True, tdp_up=True)
    out += [""] + build_stage_l(K, batch=True)
    out += [""] + build_stage_l(K, sym=True, batch=True)
    out += [""] + build_stage_l(K, tdp=True, batch=True)
    out += [""] + build_stage_l(K, sym=True, tdp=True, batch=True)
    out += [""] + build_stage_l(K, tdp=True, tdp_up=True, batch=True)
    out += [""] + build_stage_l(K, sym=True, tdp=True, tdp_up=True, batch=True)
    out += [""] + build_stage_o(K)
    out += [""] + build_stage_o(K, sym=True)
    out += [""] + build_stage_o(K, batch=True)
    out += [""] + build_stage_o(K, sym=True, batch=True)
    for sym in (False, True):
        for popc in (True, False):
            for bits in (False, True):
                out += [""] + build_stage_u(K, sym=sym, popc=popc, bits=bits)
    for g in (4, 2, 1):
        for sym in (False, True):
            out += [""] + build_stage_p(K, popc=True, group=g, sym=sym)
            out += [""] + build_stage_p(K, popc=False, group=g, sym=sym)
for K in range(1, 9):
    out += [""] + build_stage_f(K, walk=True)
    out += [""] + build_stage_f(K, walk=True, one=True, thr64=False)
for NP in (1, 2):
    out += [""] + build_stage_t(NP)
for K in range(1, 9):
    out += [""] + build_stage_wl(K)
for K in range(1, 9):
    out += [""] + build_stage_w2(K)
for K in range(1, 9):
    out += [""] + build_stage_w1d(K)
for K in range(1, 9):
    out += [""] + build_stage_w1l(K)
    out += [""] + build_stage_w1l(K, sym=True)
    out += [""] + build_stage_w1p(K)
    out += [""] + build_stage_w1p(K, sym=True)
for v in (True, False):
    out += [""] + build_stage_t1(v)
out += [""] + build_stage_tl()
path = os.environ.get("MAGUS_GEN_OUT") or \
    os.path.join(os.path.dirname(__file__), "..", "paper_2502_03796_b200", "csrc", "tick4_asm.cuh")
open(path, "w").write("\n".join(out) + "\n")
print("wrote", os.path.normpath(path))
