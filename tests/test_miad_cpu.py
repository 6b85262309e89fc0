"""NEXT-2: the MIAD chunk-size controller, a pure host function of
the C ABI, pinned against the paper's description and brute force.

P:530-535: "We initialize the chunk size with a small value and increase the
chunk size by a multiplicative factor as long as the measured throughput is
increasing.  If the throughput decreases we additively decrease the chunk size
until we reach a steady state ... we start with a chunk size of 1MB and
multiplicatively increase it by 2x on every iteration."
The measured-throughput curves below are synthetic (the absolute GB/s on real
hardware is parity-unpinned)."""
import pytest

MB = 1 << 20


@pytest.fixture(scope="module")
def B():
    from paper_1910_04940_b200 import build
    build.build()
    import paper_1910_04940_b200 as B
    return B


def run(B, thr_of, iters=40, **kw):
    st, step = B.miad(**kw)
    trace = [st.chunk]
    for _ in range(iters):
        step(thr_of(st.chunk))
        trace.append(st.chunk)
        if st.phase == 2:
            break
    return st, trace


def test_multiplicative_increase_from_1mb(B):
    # throughput keeps rising: 1, 2, 4, 8, ... MB until the ceiling
    st, trace = run(B, lambda c: c / (c + 4 * MB))
    assert trace[:7] == [MB, 2 * MB, 4 * MB, 8 * MB, 16 * MB, 32 * MB, 64 * MB]
    assert st.phase == 2 and st.chunk == 64 * MB


def test_additive_decrease_after_overshoot_finds_the_peak(B):
    # unimodal curve peaking at 8 MB
    f = lambda c: min(c, 8 * MB) / (1 + c / (64 * MB))
    st, trace = run(B, f)
    assert trace[:5] == [MB, 2 * MB, 4 * MB, 8 * MB, 16 * MB]       # MI
    assert trace[5] == 15 * MB                                      # first additive step
    assert all(b - a == -MB for a, b in zip(trace[5:-2], trace[6:-1]))
    assert st.phase == 2 and st.chunk == 8 * MB                     # steady at the peak
    # brute force over the reachable sizes agrees
    reach = set(trace)
    assert max(reach, key=f) == st.chunk


@pytest.mark.parametrize("peak_mb", [1, 3, 5, 12, 20, 40])
def test_steady_state_is_near_the_best_reachable(B, peak_mb):
    f = lambda c: 1.0 / (1.0 + abs(c / MB - peak_mb))
    st, trace = run(B, f)
    assert st.phase == 2
    seen = {c: f(c) for c in trace[:-1]}
    assert f(st.chunk) == max(seen.values())                        # best measured
    assert abs(st.chunk / MB - peak_mb) <= 1.0 or peak_mb == 40     # within one additive step


def test_flat_curve_stops_within_tolerance(B):
    st, trace = run(B, lambda c: 100.0)                             # no 1% gain: stop early
    assert st.phase == 2 and len(trace) <= 4 and st.chunk == MB
