"""CPU model of the distributed bracket selection (fx_cp.cu k_cpd_*)
against the reference rule -- top-k by (exact score desc, global id asc),
block_index.cpp:55-83 -- on adversarial inputs: approximate scores anywhere
inside their error bound, many exact ties, ties straddling shard boundaries,
k at 1 and at the total.  The GPU tests check the kernels against the
single-device step; this checks the protocol's argument itself (the ±1-bin
bracket widened by 2ε, certain-in blocks, the band's global rank) over
thousands of cases in a second."""
import numpy as np
import pytest

BINS = 2048


def reference_topk(exact, k):
    order = sorted(range(len(exact)), key=lambda i: (-exact[i], i))
    return set(order[:k])


def bracket_select(shards, k):
    """shards: list of (ids, exact f64, approx f32, eps).  Returns the union of
    the per-shard selections, computed the way the four phases do."""
    # phase 0: per-rank min / max / eps; global range = over ranks
    gmn = min(float(a.min()) for _, _, a, _ in shards)
    gmx = max(float(a.max()) for _, _, a, _ in shards)
    eps = max(e for *_, e in shards)
    total = sum(len(i) for i, *_ in shards)
    if k >= total:
        return set(int(x) for i, *_ in shards for x in i)
    # phase 1 + 2: summed histogram over the global range (float32 bin map)
    if gmx > gmn:
        scale = np.float32(BINS) / (np.float32(gmx) - np.float32(gmn))
        hist = np.zeros(BINS, np.int64)
        for _, _, a, _ in shards:
            f = (a - np.float32(gmn)) * scale
            b = np.where(f >= BINS - 1, BINS - 1, np.where(f <= 0, 0, f.astype(np.int64)))
            np.add.at(hist, b, 1)
        above = np.cumsum(hist[::-1])[::-1]  # count in bins >= i
        s_bin = int(np.max(np.nonzero(above >= k)[0]))
        w = (gmx - gmn) / BINS
        e_lo, e_hi = gmn + (s_bin - 1) * w, gmn + (s_bin + 2) * w
    else:
        e_lo = e_hi = gmx
    up, lo = e_hi + 2 * eps, e_lo - 2 * eps
    sel, bands, ndef = set(), [], 0
    for ids, ex, a, _ in shards:
        a64 = a.astype(np.float64)
        definite = a64 > up
        band = ~definite & (a64 >= lo)
        sel |= set(int(x) for x in ids[definite])
        ndef += int(definite.sum())
        bands.append(sorted(zip((-ex[band]).tolist(), ids[band].tolist())))
    # phase 3: global rank of each band entry among all bands
    need = k - ndef
    merged = sorted(e for b in bands for e in b)
    sel |= set(int(i) for _, i in merged[:need])
    return sel


def make_case(rng, R, n, ties):
    ids = np.arange(n)
    if ties:
        base = rng.integers(0, 6, n).astype(np.float64) * 0.25
    else:
        base = rng.standard_normal(n)
    exact = base
    eps = 1e-3 * (1 + rng.random())
    approx = (exact + rng.uniform(-eps, eps, n)).astype(np.float32)
    cuts = np.sort(rng.choice(np.arange(1, n), R - 1, replace=False))
    parts = np.split(ids, cuts)
    # the bound covers the float32 rounding of the approximate scores too
    eps_used = max(eps, float(np.abs(approx.astype(np.float64) - exact).max()))
    return [(p, exact[p], approx[p], eps_used) for p in parts], exact


@pytest.mark.parametrize("ties", [False, True])
def test_bracket_protocol_equals_reference_topk(ties):
    rng = np.random.default_rng(11 if ties else 7)
    for _ in range(400):
        R = int(rng.integers(2, 9))
        n = int(rng.integers(R + 1, 3000))
        shards, exact = make_case(rng, R, n, ties)
        for k in {1, int(rng.integers(1, n + 1)), n // 3 + 1, n - 1, n}:
            got = bracket_select(shards, k)
            assert got == reference_topk(exact, k), (R, n, k)


def test_bracket_protocol_all_equal_scores():
    """Every score identical (gmx == gmn): the lowest k global ids."""
    n, R = 1000, 4
    exact = np.zeros(n)
    parts = np.array_split(np.arange(n), R)
    shards = [(p, exact[p], np.zeros(len(p), np.float32), 1e-6) for p in parts]
    for k in (1, 17, 999):
        assert bracket_select(shards, k) == set(range(k))
