"""Predictor inputs on the device (fx_prefill_stats, fx_decode_features)
against the C oracle's restatement of features.cpp (pinned bit-exact to the
compiled reference in tests/test_oracle.py), and the whole predictor-driven
plan: prefill stats -> decode features -> predict -> plan_group -> decode.

Bars: integer fields and the budget features (min_budget, exact on the
device) equal; f64 statistics within 1e-9 relative (sums associate
differently on the device); predictor outputs within 1e-9 and the resulting
plans equal.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _setup(engine, B, Hkv, G, D, l_sink, l_cpu, l_local, seed, max_new=8):
    from paper_2605_07719_b200.fluxattn import SparseDecoder
    rng = np.random.default_rng(seed)
    dec = SparseDecoder(engine, B, Hkv, G, D, l_sink, l_cpu, l_local, max_new=max_new, dtype="bf16")
    host = {}
    L = l_sink + l_cpu + l_local + max_new
    for b in range(B):
        for g in range(Hkv):
            k = rng.standard_normal((L, D)).astype(np.float32)
            v = rng.standard_normal((L, D)).astype(np.float32) * 0.5 + 0.1
            s = l_sink + int(rng.integers(0, l_cpu - 32))
            k[s:s + 32] += rng.standard_normal(D).astype(np.float32) * 0.7
            k = torch.as_tensor(k).bfloat16().float().numpy()
            v = torch.as_tensor(v).bfloat16().float().numpy()
            host[(b, g)] = (k, v)
            dec.load_group(b, g, k[:L - max_new], v[:L - max_new])
    dec.build_metadata()
    anchors = rng.standard_normal((B, Hkv * G, D)).astype(np.float32)
    anchors = torch.as_tensor(anchors * 1.3).bfloat16().float().numpy()
    return dec, host, anchors, rng


def _oracle_records(coracle, dec, host, anchors, tau, layer):
    lay = dec.lay
    G = lay.group_size
    seg3 = (lay.l_sink, lay.l_cpu, lay.l_local)
    seg = seg3 + (0,)
    recs = {}
    for b in range(lay.batch):
        o_full = np.array([coracle.cache_attention(*_pre(host[(b, h // G)], lay), seg, anchors[b, h])
                           for h in range(dec.heads)])
        nrm = coracle.max_output_norm(o_full)
        cross = max(coracle.gpu_output_norm(*_pre(host[(b, h // G)], lay), seg, anchors[b, h])
                    for h in range(dec.heads))
        for h in range(dec.heads):
            k, v = _pre(host[(b, h // G)], lay)
            b4 = [coracle.min_budget(k, v, seg, anchors[b, h], blk, o_full[h], nrm, tau)[0]
                  for blk in (16, 32, 64, 128)]
            recs[(b, h)] = coracle.prefill_stats(k, v, seg3, anchors[b, h], b4, cross, layer, h)
    return recs


def _pre(kv, lay):
    n = lay.l_sink + lay.l_cpu + lay.l_local
    return kv[0][:n], kv[1][:n]


def _close(a, b, rtol=1e-9, atol=1e-12):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.all(np.abs(a - b) <= atol + rtol * np.abs(b))


@pytest.mark.parametrize("G", [4, 3])  # G = 3: the general-shape decode-feature kernels
def test_prefill_stats_and_decode_features(engine, coracle, G):
    B, Hkv, D = 2, 2, 128
    dec, host, anchors, rng = _setup(engine, B, Hkv, G, D, 64, 3000, 256, seed=4)
    rec = dec.prefill_stats(torch.as_tensor(anchors), tau=0.1, layer=3).cpu().numpy()
    want = _oracle_records(coracle, dec, host, anchors, 0.1, 3)
    for (b, h), w in want.items():
        got = rec[b, h]
        assert np.array_equal(got[:6], w[:6]), (b, h)             # layer, head, lengths, flags
        assert np.array_equal(got[26:30], w[26:30]), (b, h)       # budget features (exact)
        assert _close(got, w), (b, h, np.nonzero(~np.isclose(got, w, rtol=1e-9, atol=1e-12))[0])
    # three decoded rows, then a decode step's features
    lay = dec.lay
    for i in range(3):
        kn = torch.stack([torch.as_tensor(host[(b, g)][0][lay.l_sink + lay.l_cpu + lay.l_local + i])
                          for b in range(B) for g in range(Hkv)]).reshape(B, Hkv, D).cuda()
        vn = torch.stack([torch.as_tensor(host[(b, g)][1][lay.l_sink + lay.l_cpu + lay.l_local + i])
                          for b in range(B) for g in range(Hkv)]).reshape(B, Hkv, D).cuda()
        dec.append(kn, vn)
    q = torch.as_tensor(rng.standard_normal((B, Hkv * G, D)).astype(np.float32)).bfloat16().float()
    feats = dec.decode_features(q.cuda(), torch.as_tensor(rec).cuda()).cpu().numpy()
    seg = (lay.l_sink, lay.l_cpu, lay.l_local, 3)
    qn = q.numpy()
    for b in range(B):
        cross = max(coracle.gpu_output_norm(*host[(b, h // G)], seg, qn[b, h]) for h in range(dec.heads))
        for h in range(dec.heads):
            w = coracle.decode_features(*host[(b, h // G)], seg, qn[b, h], want[(b, h)], cross)
            assert _close(feats[b, h], w), (b, h, np.nonzero(~np.isclose(feats[b, h], w, rtol=1e-9))[0])


def test_predictor_driven_plan(engine, coracle):
    """prefill -> features -> predict -> plan_group -> decode, all on the
    device, against the oracle chain on the same inputs."""
    from paper_2605_07719_b200.fluxattn import Predictor
    B, Hkv, G, D = 2, 2, 4, 128
    dec, host, anchors, rng = _setup(engine, B, Hkv, G, D, 64, 4000, 256, seed=8)
    params = coracle.make_model(11)
    params["mu"] = np.zeros(41)
    params["sigma"] = np.ones(41) * 50.0  # keep the random net's outputs in a useful range
    params["sigma"][[0, 1]] = 0.0
    pred = Predictor(engine, params)
    rec = dec.prefill_stats(torch.as_tensor(anchors), tau=0.1, layer=0)
    q = torch.as_tensor(rng.standard_normal((B, Hkv * G, D)).astype(np.float32)).bfloat16().float().cuda()
    feats = dec.decode_features(q, rec)
    b0, ks, st = pred(feats)
    dec.step(q, props=(b0, ks, st))
    torch.cuda.synchronize()
    f = feats.cpu().numpy()
    b0n, ksn, stn = b0.cpu().numpy(), ks.cpu().numpy(), st.cpu().numpy()
    for b in range(B):
        for h in range(dec.heads):
            out, _ = coracle.predict(params, f[b, h])
            assert abs(b0n[b, h] - out[0]) <= 1e-12 and abs(ksn[b, h] - out[1]) <= 1e-12
            assert stn[b, h] == int(out[2] >= 0.5)
        for g in range(Hkv):
            sl = slice(g * G, (g + 1) * G)
            p = coracle.plan_group(b0n[b, sl], ksn[b, sl], stn[b, sl], dec.lay.l_cpu)
            assert int(dec.plan_blk[b, g]) == (0 if p["streaming_group"] else p["block_size"])
    pred.close()


@pytest.mark.parametrize("Hkv,G,D,n_new,via_append", [
    (2, 4, 128, 3, False), (4, 7, 128, 0, False), (1, 4, 64, 5, False), (8, 4, 128, 1, False),
    (3, 2, 64, 5, False), (2, 4, 128, 66, True), (2, 8, 128, 1, True), (2, 4, 64, 64, True),
    (1, 4, 128, 1100, True)])  # 1100 decoded rows: more chunks than the merge keeps in registers
def test_fused_predict_props(engine, coracle, Hkv, G, D, n_new, via_append):
    """fx_predict_props (decode features as 64-row chunk partials + a clustered
    merge, normalize, MLP): features within 1e-9 of the oracle (cross-head max
    through DSMEM included), logits bit-identical to the predictor on those
    features, and the props equal to the fx_decode_features path's.
    via_append: the last decoded row is appended by fx_predict_props itself
    (written to the cache by the CTA that holds its chunk, and seen by the
    features), checked in the cache afterwards."""
    from paper_2605_07719_b200.fluxattn import Predictor
    B = 2
    dec, host, anchors, rng = _setup(engine, B, Hkv, G, D, 64, 2500, 256, seed=30 + G, max_new=max(8, n_new))
    rec = dec.prefill_stats(torch.as_tensor(anchors), tau=0.1, layer=1)
    lay = dec.lay
    base = lay.l_sink + lay.l_cpu + lay.l_local

    def new_row(i):
        kn = torch.stack([torch.as_tensor(host[(b, g)][0][base + i])
                          for b in range(B) for g in range(Hkv)]).reshape(B, Hkv, D).cuda()
        vn = torch.stack([torch.as_tensor(host[(b, g)][1][base + i])
                          for b in range(B) for g in range(Hkv)]).reshape(B, Hkv, D).cuda()
        return kn, vn

    for i in range(n_new - (1 if via_append else 0)):
        dec.append(*new_row(i))
    params = coracle.make_model(5)
    params["mu"] = np.zeros(41)
    params["sigma"] = np.ones(41) * 50.0
    params["sigma"][[0, 1]] = 0.0
    pred = Predictor(engine, params)
    q = torch.as_tensor(rng.standard_normal((B, Hkv * G, D)).astype(np.float32)).bfloat16().float().cuda()
    feats = torch.empty((B, Hkv * G, 41), dtype=torch.float64, device="cuda")
    z = torch.empty((B, Hkv * G, 3), dtype=torch.float64, device="cuda")
    b0, ks, st = dec.predict_props(q, rec, pred, features=feats, z=z,
                                   append=new_row(n_new - 1) if via_append else None)
    torch.cuda.synchronize()
    assert dec.l_new == n_new
    if via_append:
        for b in range(B):
            for g in range(Hkv):
                row = base + n_new - 1
                assert np.array_equal(dec.k[b, g, row].float().cpu().numpy(), host[(b, g)][0][row])
                assert np.array_equal(dec.v[b, g, row].float().cpu().numpy(), host[(b, g)][1][row])
    f = feats.cpu().numpy()
    recn = rec.cpu().numpy()
    seg = (lay.l_sink, lay.l_cpu, lay.l_local, n_new)
    qn = q.cpu().numpy()
    for b in range(B):
        cross = max(coracle.gpu_output_norm(*host[(b, h // G)], seg, qn[b, h]) for h in range(dec.heads))
        for h in range(dec.heads):
            w = coracle.decode_features(*host[(b, h // G)], seg, qn[b, h], recn[b, h], cross)
            assert _close(f[b, h], w), (b, h, np.nonzero(~np.isclose(f[b, h], w, rtol=1e-9))[0])
    # the predictor on the fused kernel's own features: bit-identical logits
    z2 = torch.empty_like(z)
    b2, k2, s2 = pred(feats, z=z2)
    torch.cuda.synchronize()
    assert torch.equal(z, z2) and torch.equal(b0, b2) and torch.equal(ks, k2) and torch.equal(st, s2)
    for b in range(B):
        for h in range(dec.heads):
            out, zz = coracle.predict(params, f[b, h])
            assert np.array_equal(z[b, h].cpu().numpy(), zz), (b, h)
    # and the two-launch path agrees within the feature tolerance
    f_ref = dec.decode_features(q, rec).cpu().numpy()
    assert _close(f, f_ref)
    pred.close()
