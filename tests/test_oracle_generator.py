"""Pins for the oracle-side synthetic trace generator.  -m "not gpu".

The generator holds none of the method's arithmetic; these tests pin its
shapes to SPEC.md's generator examples and to the class recipe, and
check the properties both sides rely on (counter-based => shard invariant).
"""
import numpy as np
import pytest

from oracle import oracle as O

B_LO = np.float32(20.0 * (0.8 / 2.2))


def gen(seed, n_traces, n_samples, mix, amp=0.002, **kw):
    return O.gen_traces(O.GenDesc(seed=seed, n_traces=n_traces, n_samples=n_samples, class_mix=mix,
                                  noise_amp=amp, **kw))


def test_bounds_and_weights():
    for mix in range(4):
        tr, w = gen(17, 40 if mix != 3 else 1, 3000 if mix != 3 else 10000, mix)
        assert tr.dtype == np.float32 and np.all(tr >= 0) and np.all(tr <= 20.0)
        assert np.all(w >= 0.5) and np.all(w < 0.95)


def test_counter_based_shard_invariance():
    """A trace's bytes depend only on (seed, global id, t): sharding and strides never change them."""
    full, wf = gen(4, 64, 700, 1)
    part, wp = O.gen_traces(O.GenDesc(seed=4, n_traces=16, n_samples=700, class_mix=1, trace_stride=20,
                                      global_trace_offset=40))
    assert np.array_equal(part[:, :16], full[:, 40:56]) and np.array_equal(wp, wf[40:56])
    assert np.all(part[:, 16:] == 0)
    col, w = O.gen_trace(O.GenDesc(seed=4, n_traces=64, n_samples=700, class_mix=1), 13)
    assert np.array_equal(col, full[:, 13]) and w == wf[13]


def test_seed_changes_everything():
    a, _ = gen(1, 8, 100, 1)
    b, _ = gen(2, 8, 100, 1)
    assert np.mean(a == b) < 0.01


def test_class_shapes_noise_free():
    """With a = 0 the factor is exactly 1 and the levels are the class recipe: C0 constant below B_lo,
    C1 constant above B_lo, C2 low/high blocks (S:75 [lo,lo,hi,hi,...]), C3 spikes at the start of each
    cycle, C4 toggles every 1 or 2 ticks."""
    tr, _ = gen(3, 5, 5000, 1, amp=0.0)
    c0, c1, c2, c3, c4 = (tr[:, j] for j in range(5))
    assert len(set(c0)) == 1 and c0[0] < B_LO and 0.5 <= c0[0] < 4
    assert len(set(c1)) == 1 and c1[0] > B_LO and 10 <= c1[0] < 19
    lo, hi = c2[0], c2.max()
    assert set(c2) == {lo, hi} and lo < B_LO < hi
    L = int(np.argmax(c2 != lo))
    assert 20 <= L <= 2000
    t = np.arange(5000)
    assert np.array_equal(c2, np.where((t // L) % 2 == 0, lo, hi))
    base, spike = c3[-1] if c3[-1] < 5 else c3.min(), c3.max()
    assert c3[0] == spike and set(c3) == {base, spike}
    spike_len = int(np.argmax(c3 != spike))
    cycle = int(np.nonzero(c3[1:] == spike)[0][np.nonzero(np.nonzero(c3[1:] == spike)[0] >= spike_len)[0][0]]) + 1
    assert 1 <= spike_len <= 20 and 50 <= cycle <= 500
    assert np.array_equal(c3, np.where(t % cycle < spike_len, spike, base))
    assert set(c4) == {c4[0], c4.max()} and c4[0] < B_LO < c4.max()
    tog = 1 if c4[1] != c4[0] else 2
    assert np.array_equal(c4, np.where((t // tog) % 2 == 0, c4[0], c4.max()))


def test_noise_amplitude():
    """Noise is multiplicative, |D/level - 1| <= a (+1 ulp); at a = 0.002 the noise-only derivative at
    k = 1 stays below 2*0.002*20/0.1 = 0.8 < 1 GB/s/s, so shapes behave as intended."""
    clean, _ = gen(5, 10, 2000, 1, amp=0.0)
    noisy, _ = gen(5, 10, 2000, 1, amp=0.002)
    rel = np.abs(noisy.astype(np.float64) / clean.astype(np.float64) - 1)
    assert rel.max() <= 0.002 + 3e-7            # two fp32 roundings of the factor and the product
    c1 = noisy[:, 1]
    assert np.abs(np.diff(c1.astype(np.float64))).max() / 0.1 < 1.0


def test_cfg2_class_mix():
    """cfg 2 recipe: class j mod 3 -> C0 / C1 / C2, with about a quarter of the C2 traces spikes (C3)."""
    tr, _ = gen(2, 600, 3000, 0, amp=0.0)
    const = [len(set(tr[:, j])) == 1 for j in range(600)]
    assert all(const[j] for j in range(0, 600, 3)) and all(const[j] for j in range(1, 600, 3))
    spikes = sum(1 for j in range(2, 600, 3) if tr[0, j] > B_LO)    # C3 starts with a spike, C2 low
    assert 30 <= spikes <= 70


def test_cfg5_adversarial_square_waves():
    """cfg 5: square waves of period p = a/b ticks, phase floor(2 t b / a) mod 2; p = 1 aliases to a
    constant, p = 2 toggles every tick; telegraph traces flip with probability q."""
    tr, _ = gen(5, 22, 4000, 2, amp=0.0)
    t = np.arange(4000)
    periods = [(1, 1), (21, 20), (3, 2), (2, 1), (41, 20), (5, 2), (3, 1), (4, 1)]
    for j in range(8):
        a, b = periods[j]
        col = tr[:, j]
        phase = (2 * t * b // a) % 2
        lo, hi = col[phase == 0][0], (col[phase == 1][0] if phase.any() else None)
        assert np.all(col[phase == 0] == lo)
        if hi is not None:
            assert np.all(col[phase == 1] == hi) and hi > lo
    for j, q in zip(range(8, 11), (0.3, 0.5, 0.7)):
        col = tr[:, j]
        flips = np.mean(col[1:] != col[:-1])
        assert abs(flips - q) < 0.04


def test_cfg1_concatenated_segments():
    """cfg 1: a single trace of 2,000-tick segments cycling C0..C4."""
    tr, _ = gen(1, 1, 10000, 3, amp=0.0, trace_stride=4)
    col = tr[:, 0]
    assert np.all(tr[:, 1:] == 0)
    assert len(set(col[:2000])) == 1 and col[0] < B_LO
    assert len(set(col[2000:4000])) == 1 and col[2000] > B_LO
    assert len(set(col[4000:6000])) == 2
    assert col[6000] > B_LO        # C3 starts with a spike
    seg4 = col[8000:]
    assert len(set(seg4)) == 2 and (seg4[1] != seg4[0] or seg4[2] != seg4[0])
