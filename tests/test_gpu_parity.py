"""Parity of the CUDA path (through the C-ABI) against the CPU oracle.

Bars (BASELINE.json north_star): selected block ids bit-exact (mismatches
where the reference score gap is < 1e-6 are reported separately); outputs
within 1e-3 (f32 storage) / 2e-2 (bf16 storage) max-abs relative to the
largest output magnitude; metadata, plans, k and predictor outputs bit-exact.
bf16 recipe: K, V, q rounded to bf16 then upcast to f32 for the
oracle, so both sides see identical values.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TOL = {"f32": 1e-3, "bf16": 2e-2}


def bf16_round(x):
    return torch.as_tensor(np.asarray(x, np.float32)).bfloat16().float().numpy()


def rel_err(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(1.0, np.abs(b).max()))


def make_decoder(engine, B, Hkv, G, D, l_sink, l_cpu, l_local, dtype, seed, n_new=0,
                 structured=False):
    """Random (or needle-planted) K/V in a SparseDecoder plus the host copy."""
    from paper_2605_07719_b200.fluxattn import SparseDecoder
    rng = np.random.default_rng(seed)
    L = l_sink + l_cpu + l_local
    dec = SparseDecoder(engine, B, Hkv, G, D, l_sink, l_cpu, l_local, max_new=max(n_new, 4),
                        dtype=dtype)
    host = {}
    for b in range(B):
        for g in range(Hkv):
            k = rng.standard_normal((L + n_new, D)).astype(np.float32)
            v = rng.standard_normal((L + n_new, D)).astype(np.float32)
            if structured:  # planted needles so selections are meaningful
                for _ in range(3):
                    s = l_sink + rng.integers(0, max(1, l_cpu - 16))
                    u = rng.standard_normal(D).astype(np.float32)
                    k[s:s + 16] += 4.0 * u / np.linalg.norm(u) * np.sqrt(D) / 4
            if dtype == "bf16":
                k, v = bf16_round(k), bf16_round(v)
            host[(b, g)] = (k, v)
            dec.load_group(b, g, k, v)
    dec.l_new = n_new
    dec.build_metadata()
    q = rng.standard_normal((B, Hkv * G, D)).astype(np.float32)
    q *= np.sqrt(D) / np.linalg.norm(q, axis=-1, keepdims=True)
    if dtype == "bf16":
        q = bf16_round(q)
    return dec, host, q


# ---------------------------------------------------------------------------
# K1 metadata
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("dtype,D,l_cpu", [("bf16", 128, 1000), ("f32", 128, 777),
                                           ("bf16", 64, 300), ("f32", 64, 128), ("bf16", 128, 4096 * 3 + 40),
                                           ("bf16", 128, 5)])
def test_metadata_levels_bitexact(engine, coracle, dtype, D, l_cpu):
    dec, host, _ = make_decoder(engine, 2, 2, 4, D, 64, l_cpu, 256, dtype, seed=1)
    torch.cuda.synchronize()
    for lvl, blk in enumerate((16, 32, 64, 128)):
        m = dec.meta[lvl].float().cpu().numpy()
        for (b, g), (k, _) in host.items():
            mins, maxs = coracle.build_metadata(k[64:64 + l_cpu], blk)
            assert np.array_equal(m[b, g, :, 0], mins), (blk, b, g)
            assert np.array_equal(m[b, g, :, 1], maxs), (blk, b, g)
    am = dec.absmax.cpu().numpy()
    for (b, g), (k, _) in host.items():
        assert np.array_equal(am[b, g], np.abs(k[64:64 + l_cpu]).max(0))


@pytest.mark.parametrize("dtype,D", [("bf16", 128), ("f32", 64), ("bf16", 64), ("f32", 128)])
def test_metadata_signed_zeros_keep_first(engine, coracle, dtype, D):
    """Blocks full of +0 / -0 ties: the streaming fold keeps the earlier row
    like the reference's sequential min/max (block_index.cpp:24-31), to the bit."""
    from paper_2605_07719_b200.fluxattn import SparseDecoder
    rng = np.random.default_rng(3)
    l_cpu = 1000
    dec = SparseDecoder(engine, 1, 1, 4, D, 64, l_cpu, 256, max_new=4, dtype=dtype)
    k = rng.standard_normal((64 + l_cpu + 256, D)).astype(np.float32)
    z = rng.random(k.shape) < 0.6
    k[z] = np.where(rng.random(z.sum()) < 0.5, 0.0, -0.0).astype(np.float32)
    if dtype == "bf16":
        k = bf16_round(k)
    dec.load_group(0, 0, k, k)
    dec.build_metadata()
    torch.cuda.synchronize()
    for lvl, blk in enumerate((16, 32, 64, 128)):
        m = dec.meta[lvl].float().cpu().numpy()
        mins, maxs = coracle.build_metadata(k[64:64 + l_cpu], blk)
        assert np.array_equal(m[0, 0, :, 0].view(np.uint32), mins.view(np.uint32)), blk
        assert np.array_equal(m[0, 0, :, 1].view(np.uint32), maxs.view(np.uint32)), blk


@pytest.mark.parametrize("dtype,D,l_cpu", [("bf16", 128, 1000), ("f32", 64, 4097), ("bf16", 64, 129)])
def test_metadata_mean_keys(engine, coracle, dtype, D, l_cpu):
    """Per-block mean keys (north-star item 1; no reference counterpart): the
    f64 mean of the block's rows within 1e-5, from the same pass that writes
    min / max bit-identical to the default build."""
    dec, host, _ = make_decoder(engine, 2, 2, 4, D, 64, l_cpu, 256, dtype, seed=9)
    ref = [m.clone() for m in dec.meta]
    dec.build_metadata(means=True)
    torch.cuda.synchronize()
    for lvl, blk in enumerate((16, 32, 64, 128)):
        assert torch.equal(dec.meta[lvl], ref[lvl])
        got = dec.means[lvl].cpu().numpy()
        for (b, g), (k, _) in host.items():
            kc = k[64:64 + l_cpu].astype(np.float64)
            nb = (l_cpu + blk - 1) // blk
            want = np.stack([kc[i * blk:(i + 1) * blk].mean(0) for i in range(nb)])
            assert np.allclose(got[b, g], want, rtol=1e-5, atol=1e-6), (blk, b, g)


@pytest.mark.parametrize("blk", [1, 3, 16, 100])
def test_metadata_generic_any_granularity(engine, coracle, blk):
    rng = np.random.default_rng(blk)
    k = rng.standard_normal((333, 24)).astype(np.float32)
    meta = engine.build_metadata(k, blk)
    mins, maxs = coracle.build_metadata(k, blk)
    assert meta.block_count == len(mins)
    assert np.array_equal(meta.mins, mins) and np.array_equal(meta.maxs, maxs)


def test_metadata_invalid_granularity(engine):
    with pytest.raises(RuntimeError, match="^invalid-granularity"):
        engine.build_metadata(np.ones((4, 4), np.float32), 0)


# ---------------------------------------------------------------------------
# K2 scoring / top-k (per-query API)
# ---------------------------------------------------------------------------
def test_block_scores_bitexact(engine, coracle):
    rng = np.random.default_rng(3)
    k = rng.standard_normal((2000, 128)).astype(np.float32)
    q = rng.standard_normal(128).astype(np.float32)
    meta = engine.build_metadata(k, 16)
    got = engine.block_scores(q, meta)
    want = coracle.block_scores(q, meta.mins, meta.maxs)
    assert np.array_equal(got, want)
    with pytest.raises(RuntimeError, match="^bad-block"):
        engine.block_score(q, meta, meta.block_count)


@pytest.mark.parametrize("k", [0, 1, 7, 50, 125, 126, 400])
def test_topk_blocks_api(engine, coracle, k):
    rng = np.random.default_rng(k + 11)
    keys = rng.standard_normal((2000, 64)).astype(np.float32)
    keys[160:320] = keys[0:160]  # duplicated blocks -> exact score ties
    q = rng.standard_normal(64).astype(np.float32)
    meta = engine.build_metadata(keys, 16)
    sel = engine.topk_blocks(q, meta, k)
    want, clamped = coracle.topk_blocks(q, meta.mins, meta.maxs, k)
    assert sel.blocks == [int(x) for x in want]
    assert sel.clamped == clamped
    toks = coracle.selection_tokens(want, 16, 2000)
    assert sel.token_indices == [int(x) for x in toks]


# ---------------------------------------------------------------------------
# K5 selector + predictor
# ---------------------------------------------------------------------------
def test_plan_groups_bitexact(engine, coracle):
    from paper_2605_07719_b200.fluxattn import HeadProperties
    rng = np.random.default_rng(5)
    groups = []
    for i in range(300):
        G = 4
        props = [HeadProperties(float(rng.uniform(-0.05, 0.2)), float(rng.uniform(-0.01, 0.03)),
                                bool(rng.random() < 0.4)) for _ in range(G)]
        if i % 17 == 0:
            props = [HeadProperties(0.1, 0.0, True) for _ in range(G)]  # streaming group
        if i % 23 == 0:  # exact volume ties across candidates
            props = [HeadProperties(0.0, 0.0, False) for _ in range(G)]
        groups.append(props)
    l_cpu = 130752
    plans = engine.plan_groups(groups, l_cpu)
    for props, p in zip(groups, plans):
        w = coracle.plan_group([x.bgt0 for x in props], [x.k for x in props],
                               [x.streaming for x in props], l_cpu)
        assert p.streaming_group == w["streaming_group"]
        assert p.block_size == w["block_size"]
        assert p.volume == w["volume"]
        assert np.array_equal(np.array(p.candidate_volumes), w["candidate_volumes"])
        if not p.streaming_group:
            assert np.array_equal(np.array(p.budgets), w["budgets"])


def test_blocks_for_budget_bitexact(engine, coracle):
    rng = np.random.default_rng(9)
    for _ in range(200):
        bgt = float(rng.choice([0.0, -0.1, 1.0, 2.0, rng.uniform(0, 1), 16 / 130752,
                                32 * 7 / 130752]))
        blk = int(rng.choice([16, 32, 64, 128]))
        l_cpu = int(rng.choice([130752, 32448, 1000, 17]))
        assert engine.blocks_for_budget(bgt, l_cpu, blk) == coracle.blocks_for_budget(bgt, l_cpu, blk)


def test_predictor_bitexact(engine, coracle):
    import ctypes as C
    from paper_2605_07719_b200 import _native as N
    p = coracle.make_model(7)
    rng = np.random.default_rng(1)
    p["mu"] = rng.standard_normal(41)
    p["sigma"] = np.abs(rng.standard_normal(41)) + 0.1
    p["sigma"][3] = 0.0  # zero-sigma dims pass through as 0
    feats = rng.standard_normal((64, 41)) * 3
    h = C.c_void_p()
    N.check(N.LIB.fx_model_create(engine.ctx, *[np.ascontiguousarray(p[n]).ctypes.data for n in
                                                ("w1", "b1", "w2", "b2", "w3", "b3", "mu", "sigma")],
                                  C.byref(h)))
    fd = torch.as_tensor(feats).cuda()
    b0 = torch.zeros(64, dtype=torch.float64, device="cuda")
    ks = torch.zeros(64, dtype=torch.float64, device="cuda")
    st = torch.zeros(64, dtype=torch.int32, device="cuda")
    z = torch.zeros((64, 3), dtype=torch.float64, device="cuda")
    N.check(N.LIB.fx_predict(engine.ctx, h, 64, fd.data_ptr(), b0.data_ptr(), ks.data_ptr(),
                             st.data_ptr(), z.data_ptr()))
    z = z.cpu().numpy()
    for i in range(64):
        out, zz = coracle.predict(p, feats[i])
        assert np.array_equal(z[i], zz)
        assert b0[i].item() == out[0] and ks[i].item() == out[1]
        assert st[i].item() == int(out[2] >= 0.5)
    N.LIB.fx_model_destroy(h)


# ---------------------------------------------------------------------------
# attention primitives
# ---------------------------------------------------------------------------
def test_gathered_attention(engine, coracle):
    rng = np.random.default_rng(2)
    k = rng.standard_normal((500, 64)).astype(np.float32)
    v = rng.standard_normal((500, 64)).astype(np.float32)
    q = rng.standard_normal(64).astype(np.float32)
    for idx in (np.arange(500), np.array([3]), np.sort(rng.choice(500, 77, replace=False))):
        got = engine.gathered_attention(q, k, v, idx)
        o, lse, n = coracle.gathered_attention(q, k, v, idx)
        assert got.tokens == n
        assert rel_err(got.o, o) < 1e-4 and abs(got.lse - lse) < 1e-4
    empty = engine.gathered_attention(q, k, v, np.zeros(0, np.uint32))
    assert empty.empty() and empty.lse == -np.inf


def test_spec_known_answers(engine):
    # SPEC.md:42-62 known answers
    o = engine.full_attention(np.array([1, 0], np.float32), np.array([[1, 0]], np.float32),
                              np.array([[3, 4]], np.float32))
    assert np.allclose(o, [3, 4], atol=1e-6)
    o = engine.full_attention(np.array([1, 2], np.float32), np.array([[1, 1], [1, 1]], np.float32),
                              np.array([[1, 0], [0, 1]], np.float32))
    assert np.allclose(o, [0.5, 0.5], atol=1e-6)
    p = engine.segment_attention(np.array([0, 0], np.float32), np.array([[1, 2]], np.float32),
                                 np.array([[5, 6]], np.float32))
    assert abs(p.lse) < 1e-6
    p = engine.segment_attention(np.array([0, 0], np.float32), np.array([[1, 2], [3, 4]], np.float32),
                                 np.array([[5, 6], [7, 8]], np.float32))
    assert abs(p.lse - np.log(2)) < 1e-6
    from paper_2605_07719_b200.fluxattn import PartialOutput
    m = engine.merge_partials([PartialOutput(np.array([1.0, 0.0]), 0.3, 1),
                               PartialOutput(np.array([0.0, 1.0]), 0.3, 1)])
    assert np.allclose(m, [0.5, 0.5], atol=1e-6)
    with pytest.raises(RuntimeError, match="^empty-context"):
        engine.merge_partials([PartialOutput(), PartialOutput()])
    with pytest.raises(RuntimeError, match="^empty-context"):
        engine.full_attention(np.zeros(2, np.float32), np.zeros((0, 2), np.float32),
                              np.zeros((0, 2), np.float32))


# ---------------------------------------------------------------------------
# the batched decode step (K5 -> K2 -> K3/K4)
# ---------------------------------------------------------------------------
def _check_step(dec, host, q, coracle, blk_of, budgets_of, dtype, n_new=0, groups=None):
    """Selection bit-exact per head + output within tolerance per head (all
    groups, or the listed (b, g))."""
    lay = dec.lay
    G, D = lay.group_size, lay.head_dim
    l_sink, l_cpu, l_local = lay.l_sink, lay.l_cpu, lay.l_local
    o = dec.o.cpu().numpy()
    lse = dec.lse.cpu().numpy()
    near_ties = 0
    for (b, g), (k, v) in host.items():
        if groups is not None and (b, g) not in groups:
            continue
        blk = blk_of(b, g)
        buds = budgets_of(b, g)
        kc = k[l_sink:l_sink + l_cpu]
        for hg in range(G):
            h = g * G + hg
            if blk > 0:
                mins, maxs = coracle.build_metadata(kc, blk)
                kb = coracle.blocks_for_budget(buds[hg], l_cpu, blk)
                assert int(dec.plan_kblocks[b, h].item()) == kb
                want, _ = coracle.topk_blocks(q[b, h], mins, maxs, kb)
                got = dec.selected_blocks(b, h)
                # exact selection: no tolerance even at near-ties;
                # heads with a reference boundary gap < 1e-6 are only counted
                assert np.array_equal(got, np.sort(want.astype(np.int64))), \
                    f"selection mismatch (b={b}, h={h}, gap={coracle.boundary_gap(q[b, h], mins, maxs, kb)})"
                if coracle.boundary_gap(q[b, h], mins, maxs, kb) < 1e-6:
                    near_ties += 1
        wo, wl, _ = coracle.execute_group(k, v, (l_sink, l_cpu, l_local, n_new),
                                          q[b, g * G:(g + 1) * G], blk,
                                          np.asarray(buds, np.float64))
        assert rel_err(o[b, g * G:(g + 1) * G], wo) < TOL[dtype], (b, g)
        assert np.abs(lse[b, g * G:(g + 1) * G] - wl).max() < 1e-2, (b, g)
    return near_ties


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("blk,bgt", [(16, 0.05), (64, 0.05), (128, 0.2), (32, 1.0)])
def test_decode_step_fixed_plan(engine, coracle, dtype, blk, bgt):
    dec, host, q = make_decoder(engine, 2, 2, 4, 128, 64, 2000, 256, dtype, seed=blk,
                                structured=True)
    dec.step(torch.as_tensor(q).cuda(), fixed=(blk, bgt))
    torch.cuda.synchronize()
    _check_step(dec, host, q, coracle, lambda b, g: blk, lambda b, g: [bgt] * 4, dtype)


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("G,D", [(7, 128), (1, 128), (8, 64), (4, 64), (8, 128)])
def test_decode_step_shapes(engine, coracle, G, D, dtype):
    """Group sizes and head dims of every attention kernel instantiation: the
    TMA kernel (bf16), the f32 warp-stream kernel (G 4/7/8, D 64/128) and the
    generic kernel (G = 1)."""
    dec, host, q = make_decoder(engine, 2, 3, G, D, 64, 1500, 256, dtype, seed=G * D,
                                structured=True, n_new=5)
    dec.step(torch.as_tensor(q).cuda(), fixed=(32, 0.06))
    torch.cuda.synchronize()
    _check_step(dec, host, q, coracle, lambda b, g: 32, lambda b, g: [0.06] * G, dtype,
                n_new=5)


def test_decode_step_many_groups_global_prefix(engine, coracle):
    """> 1024 (b, g) runs: the worklist publishes the global run prefix and the
    attention kernel reads it instead of rebuilding it in shared memory."""
    B, Hkv, G, D = 130, 8, 4, 128
    dec, host, q = make_decoder(engine, B, Hkv, G, D, 16, 300, 32, "bf16", seed=5)
    dec.step(torch.as_tensor(q).cuda(), fixed=(16, 0.1))
    torch.cuda.synchronize()
    _check_step(dec, host, q, coracle, lambda b, g: 16, lambda b, g: [0.1] * G, "bf16",
                groups=[(0, 0), (64, 3), (129, 7)])


def test_decode_step_props_plan(engine, coracle):
    """Head properties -> on-device plan_group -> selection -> attention."""
    B, Hkv, G, D = 2, 4, 4, 128
    dec, host, q = make_decoder(engine, B, Hkv, G, D, 64, 4000, 256, "bf16", seed=77,
                                structured=True, n_new=3)
    rng = np.random.default_rng(4)
    H = Hkv * G
    b0 = rng.uniform(0.01, 0.08, (B, H))
    ks = rng.uniform(0.0, 0.01, (B, H))
    st = (rng.random((B, H)) < 0.5).astype(np.int32)
    st[0, :G] = 1  # one fully streaming group
    props = (torch.as_tensor(b0).cuda(), torch.as_tensor(ks).cuda(), torch.as_tensor(st).cuda())
    dec.step(torch.as_tensor(q).cuda(), props=props)
    torch.cuda.synchronize()
    plans = {}
    for b in range(B):
        for g in range(Hkv):
            sl = slice(g * G, (g + 1) * G)
            w = coracle.plan_group(b0[b, sl], ks[b, sl], st[b, sl], 4000)
            assert int(dec.plan_blk[b, g].item()) == w["block_size"]
            if not w["streaming_group"]:
                assert np.array_equal(dec.plan_budgets[b, sl].cpu().numpy(), w["budgets"])
                assert dec.plan_volume[b, g].item() == w["volume"]
            plans[(b, g)] = w
    _check_step(dec, host, q, coracle, lambda b, g: plans[(b, g)]["block_size"],
                lambda b, g: (plans[(b, g)]["budgets"] if not plans[(b, g)]["streaming_group"]
                              else [0.0] * G), "bf16", n_new=3)


def test_decode_step_ties_constant_keys(engine, coracle):
    """All-equal block scores: selection must take the lowest ids."""
    from paper_2605_07719_b200.fluxattn import SparseDecoder
    D, l_cpu = 128, 1024
    dec = SparseDecoder(engine, 1, 1, 4, D, 64, l_cpu, 256, dtype="bf16")
    k = np.ones((64 + l_cpu + 256, D), np.float32) * 0.5
    v = np.random.default_rng(0).standard_normal(k.shape).astype(np.float32)
    v = bf16_round(v)
    dec.load_group(0, 0, k, v)
    dec.build_metadata()
    q = bf16_round(np.random.default_rng(1).standard_normal((1, 4, D)).astype(np.float32))
    dec.step(torch.as_tensor(q).cuda(), fixed=(16, 0.1))
    torch.cuda.synchronize()
    kb = coracle.blocks_for_budget(0.1, l_cpu, 16)
    for h in range(4):
        assert dec.selected_blocks(0, h).tolist() == list(range(kb))
    _check_step(dec, {(0, 0): (k, v)}, q, coracle, lambda b, g: 16, lambda b, g: [0.1] * 4, "bf16")


def test_decode_step_large_tie_band(engine, coracle):
    """Hundreds of blocks tied at the cut-off score (> the 512-entry smem band):
    the block-wide radix select takes the tied blocks lowest id first, exactly
    as the reference's (score desc, id asc) order, and the step stays fast."""
    import time
    from paper_2605_07719_b200.fluxattn import SparseDecoder
    D, l_cpu = 128, 32768
    rng = np.random.default_rng(5)
    dec = SparseDecoder(engine, 1, 1, 4, D, 64, l_cpu, 256, dtype="bf16")
    nb = l_cpu // 16
    level = rng.choice([0.25, 0.5, 0.75], nb)
    k = rng.standard_normal((64 + l_cpu + 256, D)).astype(np.float32) * 0.01
    k[64:64 + l_cpu] = np.repeat(level, 16)[:, None] * np.ones((1, D), np.float32)
    k, v = bf16_round(k), bf16_round(rng.standard_normal(k.shape).astype(np.float32))
    dec.load_group(0, 0, k, v)
    dec.build_metadata()
    q = np.abs(rng.standard_normal((1, 4, D))).astype(np.float32)
    q[0, 1] *= -1.0  # head 1 ranks the low level first
    q = bf16_round(q)
    qd = torch.as_tensor(q).cuda()
    dec.step(qd, fixed=(16, 0.3))
    torch.cuda.synchronize()
    t = time.perf_counter()
    dec.step(qd, fixed=(16, 0.3))
    torch.cuda.synchronize()
    assert time.perf_counter() - t < 0.05
    _check_step(dec, {(0, 0): (k, v)}, q, coracle, lambda b, g: 16, lambda b, g: [0.3] * 4, "bf16")


def test_decode_step_reference_workload(engine, refo, coracle):
    """Reference generator (planted needles / streaming heads) end to end."""
    from paper_2605_07719_b200.fluxattn import SparseDecoder
    spec = dict(heads=8, group_size=4, head_dim=128, context_len=4096, layers=1,
                decode_steps=2, seed=3)
    w = refo.generate(**spec)
    l_cpu = 4096 - 320
    dec = SparseDecoder(engine, 1, 2, 4, 128, 64, l_cpu, 256, max_new=4, dtype="f32")
    host = {}
    for g in range(2):
        k, v = w.group_kv(0, g)
        nk, nv = w.new_kv(0, 0)
        k = np.vstack([k, nk[g:g + 1]])
        v = np.vstack([v, nv[g:g + 1]])
        host[(0, g)] = (k, v)
        dec.load_group(0, g, k, v)
    dec.l_new = 1
    dec.build_metadata()
    q = w.queries(0, 1)[None]
    dec.step(torch.as_tensor(q).cuda(), fixed=(16, 0.05))
    torch.cuda.synchronize()
    _check_step(dec, host, q, coracle, lambda b, g: 16, lambda b, g: [0.05] * 4, "f32", n_new=1)
    # and against the compiled reference's own execute_task
    o = dec.o.cpu().numpy()
    for g in range(2):
        k, v = host[(0, g)]
        ro = refo.execute_group(k, v, (64, l_cpu, 256, 1), q[0, g * 4:(g + 1) * 4], 16,
                                np.full(4, 0.05))
        assert rel_err(o[0, g * 4:(g + 1) * 4], ro) < 1e-3


def test_execute_task_api(engine, coracle):
    from paper_2605_07719_b200.fluxattn import GroupPlan, SegmentedKvCache, SparseTask
    rng = np.random.default_rng(8)
    D = 64
    mk = lambda n: rng.standard_normal((n, D)).astype(np.float32)
    cache = SegmentedKvCache(mk(64), mk(64), mk(900), mk(900), mk(256), mk(256))
    cache.append_new(mk(1)[0], mk(1)[0])
    meta = engine.build_metadata(cache.k_cpu, 32)
    qs = [mk(1)[0] for _ in range(4)]
    plan = GroupPlan(group_id=0, block_size=32, budgets=[0.05, 0.0, 0.3, 1.0])
    out = engine.execute_task(SparseTask(0, plan, cache, meta, qs))
    k, v = cache.stacked()
    wo, _, _ = coracle.execute_group(k, v, (64, 900, 256, 1), np.stack(qs), 32,
                                     np.array(plan.budgets))
    assert rel_err(np.stack(out), wo) < 1e-3


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_approx_score_error_bound(engine, coracle, dtype):
    """Realized prefilter error vs the bound the exact selection relies on."""
    import ctypes as C
    from paper_2605_07719_b200 import _native as N
    B, Hkv, G, D, l_cpu = 2, 2, 4, 128, 6000
    dec, host, q = make_decoder(engine, B, Hkv, G, D, 64, l_cpu, 256, dtype, seed=21,
                                structured=True)
    worst = 0.0
    for blk in (16, 32, 64, 128):
        nblk16 = (l_cpu + 15) // 16
        out = torch.zeros((B, Hkv * G, nblk16), dtype=torch.float32, device="cuda")
        blk_t = torch.full((B, Hkv), blk, dtype=torch.int32, device="cuda")
        qd = torch.as_tensor(q).cuda()
        eps = C.c_double(0)
        meta = (C.c_void_p * 4)(*[m.data_ptr() for m in dec.meta])
        N.check(N.LIB.fx_approx_scores(engine.ctx, C.byref(dec.lay), meta, qd.data_ptr(),
                                       blk_t.data_ptr(), out.data_ptr(), C.byref(eps)))
        out = out.cpu().numpy()
        am = dec.absmax.cpu().numpy()
        for (b, g), (k, _) in host.items():
            mins, maxs = coracle.build_metadata(k[64:64 + l_cpu], blk)
            for hg in range(G):
                h = g * G + hg
                exact = coracle.block_scores(q[b, h], mins, maxs)
                bound = float(np.abs(q[b, h]).astype(np.float64) @ am[b, g].astype(np.float64))
                err = np.abs(out[b, h, :len(exact)].astype(np.float64) - exact).max()
                worst = max(worst, err / bound)
    # the selection assumes err <= eps_scale * bound; demand an 8x safety margin
    assert worst * 8 <= eps.value, (worst, eps.value)


def test_launch_count_per_step(engine):
    dec, _, q = make_decoder(engine, 1, 2, 4, 128, 64, 500, 256, "bf16", seed=0)
    qd = torch.as_tensor(q).cuda()
    n0 = engine.launches()
    dec.step(qd, fixed=(16, 0.05))
    assert engine.launches() - n0 == 5  # plan, score, select (+ fused worklist), attend, partial merge


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_decode_step_empty_group_is_identity(engine, dtype):
    """A (b, g) with nothing to attend (no sink/local/decoded rows, streaming
    plan) gets the merge identity o = 0, lse = -inf (attention.cpp:89-104),
    not stale memory; its neighbours are unaffected."""
    from paper_2605_07719_b200.fluxattn import SparseDecoder
    B, Hkv, G, D, l_cpu = 4, 8, 4, 128, 4096
    dec = SparseDecoder(engine, B, Hkv, G, D, 0, l_cpu, 0, max_new=4, dtype=dtype)
    dec.k.normal_()
    dec.v.normal_()
    dec.build_metadata()
    q = torch.randn((B, Hkv * G, D), device=engine.device)
    blk = np.full((B, Hkv), 16, np.int32)
    blk[1, 2] = blk[3, 7] = 0  # streaming groups: no task, no defaults
    budgets = [[[0.05] * G for _ in range(Hkv)] for _ in range(B)]
    dec.o.fill_(12345.0)
    dec.lse.fill_(777.0)
    o, lse = dec.step(q, blk=blk, budgets=budgets)
    torch.cuda.synchronize()
    for b, g in [(1, 2), (3, 7)]:
        assert torch.all(o[b, g * G:(g + 1) * G] == 0)
        assert torch.all(lse[b, g * G:(g + 1) * G] == float("-inf"))
    mask = torch.ones((B, Hkv * G), dtype=torch.bool, device=o.device)
    mask[1, 8:12] = mask[3, 28:32] = False
    assert torch.isfinite(o[mask]).all() and (o[mask].abs() < 100).all()
    assert torch.isfinite(lse[mask]).all()


@pytest.mark.parametrize("G", [4, 7])
def test_decode_step_every_head_written_repeated(engine, G):
    """Race guard for the attention pipeline (stage headers reused by the
    producer, last-contributor merges): many mixed-granularity steps, every
    head's output written each time and identical across repeats."""
    from paper_2605_07719_b200.fluxattn import SparseDecoder
    B, Hkv, D, l_cpu = 8, 4, 128, 65536 - 320
    dec = SparseDecoder(engine, B, Hkv, G, D, 64, l_cpu, 256, max_new=4, dtype="bf16")
    dec.k.normal_()
    dec.v.normal_()
    dec.build_metadata()
    rng = np.random.default_rng(G)
    H = Hkv * G
    props = tuple(torch.as_tensor(x, device=engine.device) for x in
                  (rng.uniform(0.01, 0.05, (B, H)), rng.uniform(0.0, 0.01, (B, H)),
                   (rng.random((B, H)) < 0.3).astype(np.int32)))
    q = torch.randn((B, H, D), device=engine.device)
    first = None
    for _ in range(20):
        dec.o.fill_(float("nan"))
        o, lse = dec.step(q, props=props)
        torch.cuda.synchronize()
        assert torch.isfinite(o).all() and torch.isfinite(lse).all()
        if first is None:
            first = o.clone()
        else:
            assert torch.equal(o, first)


def test_decode_step_without_cpu_segment(engine, coracle):
    """l_cpu = 0 (context fits the defaults): no metadata, no selection; the
    output is default_kv_attention (sink, local, decoded; attention.cpp:143-151)."""
    dec, host, q = make_decoder(engine, 2, 2, 4, 128, 64, 0, 256, "bf16", seed=3, n_new=3)
    o, lse = dec.step(torch.as_tensor(q).cuda(), fixed=(16, 0.05))
    torch.cuda.synchronize()
    o, lse = o.cpu().numpy(), lse.cpu().numpy()
    for (b, g), (k, v) in host.items():
        wo, wl, _ = coracle.execute_group(k, v, (64, 0, 256, 3), q[b, g * 4:(g + 1) * 4], 16,
                                          np.full(4, 0.05))
        assert rel_err(o[b, g * 4:(g + 1) * 4], wo) < TOL["bf16"]
        assert np.abs(lse[b, g * 4:(g + 1) * 4] - wl).max() < 1e-2


def test_decode_step_fused_append_matches_separate(engine, coracle):
    """step(append=(k, v)) writes the row inside the plan kernel and attends it:
    identical to fx_append_kv followed by a step (and to the oracle)."""
    dec1, host, q = make_decoder(engine, 2, 2, 4, 128, 64, 2000, 256, "bf16", seed=12, n_new=2,
                                 structured=True)
    dec2, _, _ = make_decoder(engine, 2, 2, 4, 128, 64, 2000, 256, "bf16", seed=12, n_new=2,
                              structured=True)
    dec1.l_new = dec2.l_new = 1  # the second decoded row arrives through an append
    kn = torch.stack([torch.as_tensor(host[(b, g)][0][64 + 2000 + 256 + 1])
                      for b in range(2) for g in range(2)]).reshape(2, 2, 128).cuda()
    vn = torch.stack([torch.as_tensor(host[(b, g)][1][64 + 2000 + 256 + 1])
                      for b in range(2) for g in range(2)]).reshape(2, 2, 128).cuda()
    qd = torch.as_tensor(q).cuda()
    dec1.append(kn, vn)
    o1, l1 = dec1.step(qd, fixed=(32, 0.1))
    o1, l1 = o1.clone(), l1.clone()
    o2, l2 = dec2.step(qd, fixed=(32, 0.1), append=(kn, vn))
    torch.cuda.synchronize()
    assert dec2.l_new == 2
    assert torch.equal(dec1.k, dec2.k) and torch.equal(dec1.v, dec2.v)
    assert torch.equal(o1, o2) and torch.equal(l1, l2)
    _check_step(dec2, host, q, coracle, lambda b, g: 32, lambda b, g: [0.1] * 4, "bf16", n_new=2)


def test_plan_select_then_sparse_decode_equals_step(engine, coracle):
    """fx_plan_select + fx_sparse_decode (the step's two halves)
    reproduce fx_decode_step bit-for-bit."""
    import ctypes as C
    from paper_2605_07719_b200 import _native as N
    dec, host, q = make_decoder(engine, 2, 2, 4, 128, 64, 3000, 256, "bf16", seed=21,
                                structured=True)
    qd = torch.as_tensor(q).cuda()
    rng = np.random.default_rng(4)
    props = tuple(torch.as_tensor(x, device="cuda") for x in
                  (rng.uniform(0.02, 0.1, (2, 8)), rng.uniform(0.0, 0.01, (2, 8)),
                   np.zeros((2, 8), np.int32)))
    o_ref, l_ref = dec.step(qd, props=props)
    o_ref, l_ref, sel_ref = o_ref.clone(), l_ref.clone(), dec.sel_bits.clone()
    a = dec._args(qd, props, None, False, None, None)
    dec.sel_bits.zero_()
    N.check(N.LIB.fx_plan_select(engine.ctx, C.byref(dec.lay), C.byref(a)))
    assert torch.equal(dec.sel_bits, sel_ref)
    sel = dec.sel_bits.clone()
    a = dec._args(qd, None, None, False, "keep", None)
    a.sel_in = sel.data_ptr()
    o = torch.empty_like(o_ref)
    lse = torch.empty_like(l_ref)
    a.o, a.lse = o.data_ptr(), lse.data_ptr()
    N.check(N.LIB.fx_sparse_decode(engine.ctx, C.byref(dec.lay), C.byref(a)))
    torch.cuda.synchronize()
    assert torch.equal(o, o_ref) and torch.equal(lse, l_ref)
    a.sel_in = None
    with pytest.raises(RuntimeError, match="^no-context"):
        N.check(N.LIB.fx_sparse_decode(engine.ctx, C.byref(dec.lay), C.byref(a)))
