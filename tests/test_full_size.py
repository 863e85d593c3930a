"""Parity at BASELINE.json's full sizes.

C2 (configs[1]): Llama layer, 128K context, batch 16, bf16, per-head budgets
and per-group granularity from the on-device selector.  C3 (configs[2]):
Qwen layer (28 q / 4 kv heads, G = 7), 256K context, batch 8.  C5
(configs[4]): 1M context, batch 4, context-parallel over 8 shards (all on one
GPU through LoopbackComm; tests/test_context_parallel_gloo.py covers the
torch.distributed exchanges).

KV is generated on the device; the oracle sees the exact bf16 bits of the
sampled (b, g) groups (D2H, upcast to f32 -- SURVEY §8c bf16 recipe).
Checked on every head of the batch (size-independent): the plan equals the
oracle's plan_group bit-for-bit, each head selects exactly
blocks_for_budget(...) blocks, outputs are finite.  Checked against the
oracle on sampled groups: the selected block set bit-exact (mismatches only
where the reference score gap is < 1e-6, reported), outputs within 2e-2
(bf16), LSE within 1e-2.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

BF16_TOL = 2e-2


def _draw_props(B, H, seed):
    rng = np.random.default_rng(seed)
    return (rng.uniform(0.01, 0.05, (B, H)), rng.uniform(0.0, 0.01, (B, H)),
            (rng.random((B, H)) < 0.5).astype(np.int32))


def _fill_kv(t, seed):
    """N(0,1) bf16 K or V, generated per sequence to bound the f32 temporary."""
    g = torch.Generator(device=t.device).manual_seed(seed)
    for b in range(t.shape[0]):
        t[b].copy_(torch.randn(t[b].shape, generator=g, device=t.device))


def _queries(B, H, D, seed, dev):
    g = torch.Generator(device=dev).manual_seed(seed)
    q = torch.randn((B, H, D), generator=g, device=dev)
    q = q / q.norm(dim=-1, keepdim=True) * D ** 0.5
    return q.bfloat16().float()


def _decoder(engine, B, Hkv, G, D, l_cpu, seed, max_new=8):
    from paper_2605_07719_b200.fluxattn import SparseDecoder
    l_sink, l_local = 64, 256
    dec = SparseDecoder(engine, B, Hkv, G, D, l_sink, l_cpu, l_local, max_new=max_new, dtype="bf16")
    _fill_kv(dec.k, seed)
    _fill_kv(dec.v, seed + 1)
    # planted needles (a few per group) so the selection is not a coin toss
    gen = torch.Generator(device="cpu").manual_seed(seed)
    for b in range(B):
        for g in range(Hkv):
            for _ in range(3):
                s = l_sink + int(torch.randint(0, l_cpu - 16, (1,), generator=gen))
                u = torch.randn(D, generator=gen)
                dec.k[b, g, s:s + 16] += (3.0 * u / u.norm() * D ** 0.5 / 4).to(dec.k.device,
                                                                               torch.bfloat16)
    dec.build_metadata()
    return dec


def _group_host(dec, b, g):
    lay = dec.lay
    n = lay.l_sink + lay.l_cpu + lay.l_local + dec.l_new
    return dec.k[b, g, :n].float().cpu().numpy(), dec.v[b, g, :n].float().cpu().numpy()


def _check_plans(dec, coracle, props):
    """Every group's plan bit-exact against plan_group (selector.cpp:19-46)."""
    lay = dec.lay
    G = lay.group_size
    blk = dec.plan_blk.cpu().numpy()
    bud = dec.plan_budgets.cpu().numpy()
    kbl = dec.plan_kblocks.cpu().numpy()
    bgt0, ks, st = props
    for b in range(lay.batch):
        for g in range(lay.kv_heads):
            sl = slice(g * G, (g + 1) * G)
            p = coracle.plan_group(bgt0[b, sl], ks[b, sl], st[b, sl], lay.l_cpu)
            if p["streaming_group"]:
                assert blk[b, g] == 0, (b, g)
                continue
            assert blk[b, g] == p["block_size"], (b, g)
            assert np.array_equal(bud[b, sl], p["budgets"]), (b, g)
            for hg in range(G):
                assert kbl[b, g * G + hg] == coracle.blocks_for_budget(p["budgets"][hg], lay.l_cpu,
                                                                      p["block_size"])


def _check_counts(dec):
    """popcount(selection bitmask) == plan_kblocks for every head."""
    w = dec.sel_bits.view(torch.uint8).cpu().numpy()
    cnt = np.unpackbits(w, axis=-1).sum(-1)
    kb = dec.plan_kblocks.cpu().numpy()
    blk = np.repeat(dec.plan_blk.cpu().numpy(), dec.lay.group_size, axis=1)
    assert np.array_equal(np.where(blk > 0, cnt, 0), np.where(blk > 0, kb, 0))


def _check_selections(dec, coracle, q, groups=None):
    """Every head of every listed retrieval group (default: all of them): the
    selected block set equals the oracle's topk_blocks bit-for-bit
    (block_index.cpp:55-83).  The selection is exact, so a
    mismatch fails even where the reference's boundary gap is tiny; the heads
    whose k-th/(k+1)-th gap is below 1e-6 are counted and printed."""
    lay = dec.lay
    G, l_sink, l_cpu = lay.group_size, lay.l_sink, lay.l_cpu
    blk_all = dec.plan_blk.cpu().numpy()
    kb_all = dec.plan_kblocks.cpu().numpy()
    bits = dec.sel_bits.cpu().numpy().view(np.uint32)
    qn = q.cpu().numpy()
    if groups is None:
        groups = [(b, g) for b in range(lay.batch) for g in range(lay.kv_heads) if blk_all[b, g] > 0]
    heads = near = 0
    for b, g in groups:
        blk = int(blk_all[b, g])
        if blk == 0:
            continue
        k_cpu = dec.k[b, g, l_sink:l_sink + l_cpu].float().cpu().numpy()
        mins, maxs = coracle.build_metadata(k_cpu, blk)
        nblk = mins.shape[0]
        for hg in range(G):
            h = g * G + hg
            kb = int(kb_all[b, h])
            want, _ = coracle.topk_blocks(qn[b, h], mins, maxs, kb)
            got = np.nonzero(np.unpackbits(bits[b, h].view(np.uint8), bitorder="little")[:nblk])[0]
            assert np.array_equal(np.sort(want.astype(np.int64)), got), \
                f"selection mismatch (b={b}, h={h}, blk={blk}, k={kb}, " \
                f"gap={coracle.boundary_gap(qn[b, h], mins, maxs, kb):.3e})"
            if coracle.boundary_gap(qn[b, h], mins, maxs, kb) < 1e-6:
                near += 1
            heads += 1
    print(f"  selections: {heads} heads of {len(groups)} groups bit-exact "
          f"({near} with a reference boundary gap < 1e-6)")
    return heads


def _check_groups(dec, coracle, q, groups):
    """Outputs of sampled groups against the oracle's execute_task recipe
    (scheduler.cpp:78-96): within 2e-2 (bf16), LSE within 1e-2."""
    lay = dec.lay
    G, l_sink, l_cpu, l_local = lay.group_size, lay.l_sink, lay.l_cpu, lay.l_local
    o, lse = dec.o.cpu().numpy(), dec.lse.cpu().numpy()
    qn = q.cpu().numpy()
    for b, g in groups:
        k, v = _group_host(dec, b, g)
        blk = int(dec.plan_blk[b, g].item())
        buds = dec.plan_budgets[b, g * G:(g + 1) * G].cpu().numpy()
        mins = maxs = None
        if blk > 0:
            mins, maxs = coracle.build_metadata(k[l_sink:l_sink + l_cpu], blk)
        wo, wl, _ = coracle.execute_group(k, v, (l_sink, l_cpu, l_local, dec.l_new),
                                          qn[b, g * G:(g + 1) * G], blk, buds, mins, maxs)
        err = np.abs(o[b, g * G:(g + 1) * G] - wo).max() / max(1.0, np.abs(wo).max())
        lerr = np.abs(lse[b, g * G:(g + 1) * G] - wl).max()
        print(f"  (b={b}, g={g}) blk={blk}: max rel err {err:.2e}, max lse err {lerr:.2e}")
        assert err < BF16_TOL, (b, g, err)
        assert lerr < 1e-2, (b, g)


def _retrieval_groups(dec, n):
    blk = dec.plan_blk.cpu().numpy()
    idx = [(b, g) for b in range(blk.shape[0]) for g in range(blk.shape[1]) if blk[b, g] > 0]
    pick = np.linspace(0, len(idx) - 1, n).round().astype(int)
    return [idx[i] for i in sorted(set(pick.tolist()))]


def test_c2_full_size_two_steps(engine, coracle):
    """C2: 16 x 8 groups x 128K, props plan, two decode steps with an append."""
    B, Hkv, G, D, l_cpu = 16, 8, 4, 128, 131072 - 320
    dec = _decoder(engine, B, Hkv, G, D, l_cpu, seed=11)
    props = _draw_props(B, Hkv * G, seed=1)
    dprops = tuple(torch.as_tensor(x, device=engine.device) for x in props)
    dev = engine.device
    for step in range(2):
        if step:
            gen = torch.Generator(device=dev).manual_seed(100 + step)
            dec.append(torch.randn((B, Hkv, D), generator=gen, device=dev).bfloat16().float(),
                       torch.randn((B, Hkv, D), generator=gen, device=dev).bfloat16().float())
        q = _queries(B, Hkv * G, D, seed=step, dev=dev)
        dec.o.fill_(float("nan"))  # every head must be written this step
        o, lse = dec.step(q, props=dprops)
        torch.cuda.synchronize()
        assert torch.isfinite(o).all() and torch.isfinite(lse).all()
        _check_plans(dec, coracle, props)
        _check_counts(dec)
        _check_selections(dec, coracle, q)
        _check_groups(dec, coracle, q, _retrieval_groups(dec, 3))


def test_c2_full_budget_is_dense_attention(engine):
    """FULL plan (pipeline.cpp:298-303) at 128K equals dense attention (torch f64)."""
    B, Hkv, G, D, l_cpu = 16, 8, 4, 128, 131072 - 320
    dec = _decoder(engine, B, Hkv, G, D, l_cpu, seed=21)
    q = _queries(B, Hkv * G, D, seed=5, dev=engine.device)
    o, lse = dec.step(q, full=True)
    torch.cuda.synchronize()
    for b, g in [(0, 0), (15, 7)]:
        n = dec.lay.l_sink + l_cpu + dec.lay.l_local
        k = dec.k[b, g, :n].double()
        v = dec.v[b, g, :n].double()
        qs = q[b, g * G:(g + 1) * G].double()
        s = qs @ k.T / D ** 0.5
        want_lse = torch.logsumexp(s, -1)
        want = torch.softmax(s, -1) @ v
        err = (o[b, g * G:(g + 1) * G].double() - want).abs().max() / max(1.0, want.abs().max())
        assert err < BF16_TOL
        assert (lse[b, g * G:(g + 1) * G].double() - want_lse).abs().max() < 1e-2


def test_c3_full_size_qwen(engine, coracle):
    """C3 shape: Qwen layer (28 q / 4 kv heads, G = 7), 256K, batch 8."""
    B, Hkv, G, D, l_cpu = 8, 4, 7, 128, 262144 - 320
    dec = _decoder(engine, B, Hkv, G, D, l_cpu, seed=31)
    props = _draw_props(B, Hkv * G, seed=3)
    q = _queries(B, Hkv * G, D, seed=7, dev=engine.device)
    dec.o.fill_(float("nan"))
    dec.step(q, props=tuple(torch.as_tensor(x, device=engine.device) for x in props))
    torch.cuda.synchronize()
    assert torch.isfinite(dec.o).all() and torch.isfinite(dec.lse).all()
    _check_plans(dec, coracle, props)
    _check_counts(dec)
    _check_selections(dec, coracle, q)
    _check_groups(dec, coracle, q, _retrieval_groups(dec, 3))


def test_c5_full_size_context_parallel(engine, coracle):
    """C5: 1M context, batch 4, 8 context-parallel shards -> the single-device
    selection bit-exactly, outputs within the bf16 bound; one group checked
    against the oracle at 1M."""
    from paper_2605_07719_b200.context_parallel import (LoopbackComm, PeerShard, PeerTables, cp_decode_step,
                                                        cp_decode_step_dist, shard_kv)
    B, Hkv, G, D, R = 4, 8, 4, 128, 8
    l_sink, l_cpu, l_local = 64, 1048576 - 320, 256
    full = _decoder(engine, B, Hkv, G, D, l_cpu, seed=41, max_new=4)
    shards = []
    for r in range(R):
        kr = shard_kv(full.k, l_sink, l_cpu, l_local, r, R, 4)
        vr = shard_kv(full.v, l_sink, l_cpu, l_local, r, R, 4)
        sh = PeerShard(engine, r, R, B, Hkv, G, D, l_sink, l_cpu, l_local, 4, "bf16", k=kr, v=vr)
        sh.dec.build_metadata()
        shards.append(sh)
    tables = PeerTables(engine, R)
    for sh in shards:
        tables.add_local(sh)
    props = _draw_props(B, Hkv * G, seed=5)
    dprops = tuple(torch.as_tensor(x, device=engine.device) for x in props)
    q = _queries(B, Hkv * G, D, seed=9, dev=engine.device)
    o_ref, lse_ref = full.step(q, props=dprops)
    torch.cuda.synchronize()
    o_ref, lse_ref = o_ref.clone(), lse_ref.clone()
    # the collective exchanges, then the distributed bracket over peer memory
    for protocol in ("collective", "dist"):
        for sh in shards:
            sh.o.fill_(float("nan"))
            sh.sel.fill_(-1)
        if protocol == "collective":
            (o, lse), *_ = cp_decode_step(shards, LoopbackComm(R), q, props=dprops)
        else:
            (o, lse), *_ = cp_decode_step_dist(shards, tables, q, 1, props=dprops)
        torch.cuda.synchronize()
        assert torch.isfinite(o_ref).all() and torch.isfinite(o).all() and not torch.isnan(lse).any()
        for b in range(B):
            for h in range(Hkv * G):
                want = full.selected_blocks(b, h)
                got = np.sort(np.concatenate([sh.global_selection(b, h) for sh in shards]))
                assert np.array_equal(got, want), (protocol, b, h)
        torch.testing.assert_close(o, o_ref, rtol=4e-3, atol=4e-3)
        torch.testing.assert_close(lse, lse_ref, rtol=1e-4, atol=1e-3)
    _check_plans(full, coracle, props)
    _check_selections(full, coracle, q)  # every head at 1M against the oracle
    _check_groups(full, coracle, q, _retrieval_groups(full, 1))


def test_c3_output_aware_budgets_full_size(engine, coracle):
    """C3 as BASELINE.json states it: Qwen layer, 256K, batch 8, output-aware
    budgets -- the oracle head properties (pipeline.cpp:256-276) labelled on
    the device for all 224 heads, checked against the C oracle on sampled
    heads (min_budget at blk 1..128 over the 261,824-row cpu segment), then
    fed to the on-device selector and the decode step."""
    B, Hkv, G, D, l_cpu = 8, 4, 7, 128, 262144 - 320
    dec = _decoder(engine, B, Hkv, G, D, l_cpu, seed=33)
    q = _queries(B, Hkv * G, D, seed=13, dev=engine.device)
    lab = dec.label_heads(q, tau=0.10)
    torch.cuda.synchronize()
    seg = (dec.lay.l_sink, l_cpu, dec.lay.l_local, 0)
    qn = q.cpu().numpy()
    nrm = lab["normalizer"].cpu().numpy()
    bud = lab["budgets"].cpu().numpy()
    st = lab["streaming"].cpu().numpy()
    near = 0
    for b, h in [(0, 0), (3, 11), (7, 27)]:
        k, v = _group_host(dec, b, h // G)
        o_full = coracle.cache_attention(k, v, seg, qn[b, h])
        assert np.allclose(lab["o_full"][b, h].cpu().numpy(), o_full, rtol=1e-9, atol=1e-12)
        assert bool(st[b, h]) == coracle.label_streaming(k, v, seg, qn[b, h], o_full, nrm[b], 0.10)
        if st[b, h]:
            continue
        for i, blk in enumerate((1, 16, 32, 64, 128)):
            w_b, w_n, _ = coracle.min_budget(k, v, seg, qn[b, h], blk, o_full, nrm[b], 0.10)
            got = int(lab["blocks"][b, h, i])
            if got != w_n:
                assert abs(got - w_n) <= 1
                near += 1
            else:
                assert bud[b, h, i] == w_b
    assert near <= 1
    props = (lab["bgt0"], lab["kslope"], lab["streaming"])
    dec.o.fill_(float("nan"))
    dec.step(q, props=props)
    torch.cuda.synchronize()
    assert torch.isfinite(dec.o).all()
    _check_plans(dec, coracle, tuple(t.cpu().numpy() for t in props))
    _check_counts(dec)
    _check_selections(dec, coracle, q)
    _check_groups(dec, coracle, q, _retrieval_groups(dec, 2))


def test_c1_full_size_f32(engine, coracle):
    """C1 (configs[0]): Llama layer, 32K, batch 1, fixed (blk 64, budget 0.05),
    f32 KV -- every group against the oracle at 1e-3 (f32 bound)."""
    from paper_2605_07719_b200.fluxattn import SparseDecoder
    B, Hkv, G, D = 1, 8, 4, 128
    l_sink, l_cpu, l_local = 64, 32768 - 320, 256
    dec = SparseDecoder(engine, B, Hkv, G, D, l_sink, l_cpu, l_local, max_new=4, dtype="f32")
    _fill_kv(dec.k, 51)
    _fill_kv(dec.v, 52)
    dec.build_metadata()
    q = _queries(B, Hkv * G, D, seed=17, dev=engine.device)
    dec.o.fill_(float("nan"))
    o, lse = dec.step(q, fixed=(64, 0.05))
    torch.cuda.synchronize()
    assert torch.isfinite(o).all()
    on, ln, qn = o.cpu().numpy(), lse.cpu().numpy(), q.cpu().numpy()
    for g in range(Hkv):
        k, v = _group_host(dec, 0, g)
        mins, maxs = coracle.build_metadata(k[l_sink:l_sink + l_cpu], 64)
        kb = coracle.blocks_for_budget(0.05, l_cpu, 64)
        assert kb == 26  # k = 26 at 32K / blk 64 / 0.05
        for hg in range(G):
            h = g * G + hg
            want, _ = coracle.topk_blocks(qn[0, h], mins, maxs, kb)
            assert np.array_equal(dec.selected_blocks(0, h), np.sort(want.astype(np.int64)))
        wo, wl, _ = coracle.execute_group(k, v, (l_sink, l_cpu, l_local, 0), qn[0, g * G:(g + 1) * G],
                                          64, np.full(G, 0.05), mins, maxs)
        assert np.abs(on[0, g * G:(g + 1) * G] - wo).max() / max(1.0, np.abs(wo).max()) < 1e-3
        assert np.abs(ln[0, g * G:(g + 1) * G] - wl).max() < 1e-3


def test_c4_full_size_32_layers(engine, coracle):
    """C4 (configs[3]) as one GPU's shard: 32 layers x 8 sequences at 128K in ONE
    batched step (256 (layer, sequence) entries = 2,048 (b, g) runs, past the
    1,024-run limit of the in-smem run prefix, so the attention takes the
    global run-prefix path).  KV from the reference generator on the device
    (generate(spec), seed 1 + sequence, entry b = layer b // 8), plans from
    drawn head properties.  Every plan and popcount is checked; the selection of
    64 groups spread over all 2,048 (both sides of run 1,024) against the
    oracle; outputs of 8 of them."""
    from paper_2605_07719_b200.fluxattn import SparseDecoder
    layers, seqs = 32, 8
    B, Hkv, G, D, ctx = layers * seqs, 8, 4, 128, 131072
    l_sink, l_local = 64, 256
    l_cpu = ctx - l_sink - l_local
    if torch.cuda.get_device_properties(0).total_memory < 170e9:
        pytest.skip("C4 needs ~155 GB of device memory")
    dec = SparseDecoder(engine, B, Hkv, G, D, l_sink, l_cpu, l_local, max_new=2, dtype="bf16")
    spec = dict(seed=1, layers=layers, heads=Hkv * G, group_size=G, head_dim=D, context_len=ctx,
                decode_steps=1)
    out = dec.generate(spec, seeds=[1 + b % seqs for b in range(B)],
                       layers=[b // seqs for b in range(B)], steps=1)
    q = out["step_q"][0].contiguous()
    del out
    dec.build_metadata()
    props = _draw_props(B, Hkv * G, seed=1)
    dec.o.fill_(float("nan"))
    dec.step(q, props=tuple(torch.as_tensor(x, device=engine.device) for x in props))
    torch.cuda.synchronize()
    assert torch.isfinite(dec.o).all() and torch.isfinite(dec.lse).all()
    _check_plans(dec, coracle, props)
    _check_counts(dec)
    runs = _retrieval_groups(dec, 64)
    flat = [b * Hkv + g for b, g in runs]
    assert min(flat) < 1024 <= max(flat)
    _check_selections(dec, coracle, q, runs)
    _check_groups(dec, coracle, q, runs[::8])
