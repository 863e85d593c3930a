"""Pins the CPU oracle (oracle/fx_oracle.c) before it is trusted as the checker:
  * bit-exact against the golden vectors made by the compiled reference
    (tests/golden/make_golden.py),
  * the SPEC.md known-answer examples and properties,
  * live against the compiled reference (oracle/_ref) on random instances
    whenever that library is present.
CPU only (no GPU)."""
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_small.npz")


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def test_golden_metadata(coracle, gold):
    kc = gold["k0"][64:64 + 704]
    for blk in (1, 16, 32, 64, 128):
        mins, maxs = coracle.build_metadata(kc, blk)
        assert np.array_equal(mins, gold[f"mins_{blk}"]) and np.array_equal(maxs, gold[f"maxs_{blk}"])


def test_golden_scores_and_topk(coracle, gold):
    q = gold["q"]
    for blk in (16, 64):
        mins, maxs = gold[f"mins_{blk}"], gold[f"maxs_{blk}"]
        nblk = len(mins)
        for h in range(4):
            assert np.array_equal(coracle.block_scores(q[h], mins, maxs), gold[f"scores_{blk}"][h])
        for kk in (1, 3, 9, nblk + 2):
            want = gold[f"topk_{blk}_{kk}"]
            for h in range(4):
                got, clamped = coracle.topk_blocks(q[h], mins, maxs, kk)
                w = want[h][want[h] >= 0]
                assert np.array_equal(got.astype(np.int64), w)
                assert clamped == (kk > nblk)


def test_golden_execute_task(coracle, gold):
    budgets = np.array([0.05, 0.0, 0.2, 1.0])
    for g in range(2):
        o, _, _ = coracle.execute_group(gold[f"k{g}"], gold[f"v{g}"], (64, 704, 256, 1),
                                        gold["q"][g * 4:(g + 1) * 4], 32, budgets)
        assert np.array_equal(o, gold[f"exec_{g}"])


def test_golden_plan_group(coracle, gold):
    for i, p in enumerate(gold["props"]):
        w = coracle.plan_group(p[:, 0], p[:, 1], p[:, 2].astype(np.int32), 130752)
        assert w["block_size"] == gold["plan_blk"][i]
        assert w["volume"] == gold["plan_vol"][i]
        assert np.array_equal(w["candidate_volumes"], gold["plan_cand"][i])
        if not w["streaming_group"]:
            assert np.array_equal(w["budgets"], gold["plan_bud"][i])


def test_golden_predictor(coracle, gold):
    p = coracle.make_model(5)
    p["mu"], p["sigma"] = gold["pred_mu"], gold["pred_sigma"]
    for f, out, z in zip(gold["pred_feats"], gold["pred_out"], gold["pred_z"]):
        o, zz = coracle.predict(p, f)
        assert np.array_equal(o, out) and np.array_equal(zz, z)


# ---- SPEC.md known answers ----
def test_spec_known_answers(coracle):
    o, lse, n = coracle.gathered_attention(np.array([1, 0], np.float32), np.array([[1, 0]], np.float32),
                                           np.array([[3, 4]], np.float32))
    assert np.allclose(o, [3, 4]) and n == 1
    o, lse, _ = coracle.gathered_attention(np.array([1, 2], np.float32), np.ones((2, 2), np.float32),
                                           np.eye(2, dtype=np.float32))
    assert np.allclose(o, [0.5, 0.5])
    _, lse, _ = coracle.gathered_attention(np.zeros(2, np.float32), np.ones((2, 2), np.float32),
                                           np.eye(2, dtype=np.float32))
    assert abs(lse - np.log(2)) < 1e-12
    m = coracle.merge((np.array([1.0, 0.0]), 0.3, 1), (np.array([0.0, 1.0]), 0.3, 1))
    assert np.allclose(m[0], [0.5, 0.5]) and m[2] == 2
    mins, maxs = coracle.build_metadata(np.random.default_rng(0).standard_normal((33, 4)), 16)
    assert len(mins) == 3
    with pytest.raises(RuntimeError, match="^invalid-granularity"):
        coracle.build_metadata(np.ones((4, 4)), 0)
    assert abs(coracle.volume(16, 1024, [0.1]) - 332.8) < 1e-9
    assert coracle.plan_group([0.05], [0.0], [0], 1024)["block_size"] == 128
    k = np.full((64, 4), 0.5, np.float32)
    mins, maxs = coracle.build_metadata(k, 16)
    got, _ = coracle.topk_blocks(np.array([1, -1, 2, 0.5], np.float32), mins, maxs, 2)
    assert got.tolist() == [0, 1]  # ties -> lower ids


def test_spec_properties(coracle):
    rng = np.random.default_rng(1)
    for _ in range(200):  # partition/merge equivalence, upper-bound soundness
        L, D = int(rng.integers(1, 200)), int(rng.integers(1, 32))
        k = rng.standard_normal((L, D)).astype(np.float32)
        v = rng.standard_normal((L, D)).astype(np.float32)
        q = rng.standard_normal(D).astype(np.float32)
        full, lse_full, _ = coracle.gathered_attention(q, k, v)
        cut = int(rng.integers(0, L + 1))
        a = coracle.gathered_attention(q, k[:cut], v[:cut]) if cut else (np.zeros(D), -np.inf, 0)
        b = coracle.gathered_attention(q, k[cut:], v[cut:]) if cut < L else (np.zeros(D), -np.inf, 0)
        m = coracle.merge(a, b)
        assert np.allclose(m[0], full, rtol=1e-6, atol=1e-9) and abs(m[1] - lse_full) < 1e-9
        blk = int(rng.integers(1, 20))
        mins, maxs = coracle.build_metadata(k, blk)
        sc = coracle.block_scores(q, mins, maxs)
        dots = k.astype(np.float64) @ q.astype(np.float64)
        for b in range(len(mins)):
            assert sc[b] >= dots[b * blk:(b + 1) * blk].max() - 1e-9


def test_live_against_compiled_reference(coracle, refo):
    rng = np.random.default_rng(7)
    for _ in range(20):
        L, D = int(rng.integers(20, 600)), int(rng.choice([8, 64, 128]))
        k = rng.standard_normal((L, D)).astype(np.float32)
        q = rng.standard_normal(D).astype(np.float32)
        blk = int(rng.choice([1, 7, 16, 64]))
        a, b = coracle.build_metadata(k, blk), refo.build_metadata(k, blk)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        kk = int(rng.integers(0, len(a[0]) + 3))
        mine, cl = coracle.topk_blocks(q, *a, kk)
        theirs = refo.topk_blocks(q, *a, blk, L, kk)
        assert np.array_equal(mine, theirs["blocks"]) and cl == theirs["clamped"]
        for bgt in (0.0, 0.01, 0.3, 1.0, 1.5):
            assert coracle.blocks_for_budget(bgt, L, max(blk, 1)) == refo.blocks_for_budget(bgt, L, max(blk, 1))


# ---------------------------------------------------------------------------
# output-aware budget oracle (budget_oracle.cpp) -- the label path of C3
# ---------------------------------------------------------------------------
GOLD_BUDGET = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                           "reference_budget.npz")


def test_golden_budget_oracle(coracle, gold):
    gb = np.load(GOLD_BUDGET)
    seg = (64, 704, 256, 1)
    q = gold["q"]
    H = q.shape[0]
    o_full = np.array([coracle.cache_attention(gold[f"k{h // 4}"], gold[f"v{h // 4}"], seg, q[h])
                       for h in range(H)])
    assert np.array_equal(o_full, gb["o_full"])
    norm = coracle.max_output_norm(o_full)
    assert norm == float(gb["normalizer"])
    for ti, tau in enumerate(gb["taus"]):
        for h in range(H):
            k, v = gold[f"k{h // 4}"], gold[f"v{h // 4}"]
            assert coracle.label_streaming(k, v, seg, q[h], o_full[h], norm, tau) == \
                bool(gb["streaming"][ti, h])
            for i, blk in enumerate((1, 16, 32, 64, 128)):
                bud, nb, sat = coracle.min_budget(k, v, seg, q[h], blk, o_full[h], norm, tau)
                assert bud == gb["min_budget"][ti, h, i] and nb == gb["min_blocks"][ti, h, i]
                assert sat == bool(gb["saturated"][ti, h, i])
    for h in range(H):
        assert np.array_equal(coracle.fit_curve([16, 32, 64, 128], gb["min_budget"][1, h, 1:]),
                              gb["fit"][h])
    with pytest.raises(RuntimeError, match="^underdetermined"):
        coracle.fit_curve([16, 16], [0.1, 0.2])


def test_budget_oracle_live_against_compiled_reference(coracle, refo):
    rng = np.random.default_rng(5)
    for trial in range(6):
        D = int(rng.choice([16, 64]))
        seg = (int(rng.integers(0, 20)), int(rng.integers(50, 900)), int(rng.integers(0, 40)),
               int(rng.integers(0, 3)))
        L = sum(seg)
        k = rng.standard_normal((L, D)).astype(np.float32)
        v = rng.standard_normal((L, D)).astype(np.float32)
        q = rng.standard_normal(D).astype(np.float32)
        if trial % 2:  # a needle the query finds
            s = seg[0] + int(rng.integers(0, seg[1] - 8))
            k[s:s + 8] += 0.5 * q
        o = coracle.cache_attention(k, v, seg, q)
        assert np.array_equal(o, refo.cache_attention(k, v, seg, q))
        norm = max(float(np.linalg.norm(o)), 1e-3)
        for tau in (0.02, 0.1, 0.4):
            if seg[0] + seg[2] + seg[3] > 0:
                assert coracle.label_streaming(k, v, seg, q, o, norm, tau) == \
                    refo.label_streaming(k, v, seg, q, o, norm, tau)
            for blk in (1, 16, 64):
                assert coracle.min_budget(k, v, seg, q, blk, o, norm, tau) == \
                    refo.min_budget(k, v, seg, q, blk, o, norm, tau)
