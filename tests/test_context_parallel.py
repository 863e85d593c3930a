"""Context-parallel decode (config C5): R cpu-segment shards with
the candidate / threshold exchanges must reproduce the single-device
selection bit-exactly and its output within the f32 merge tolerance.  All
shards run on one GPU through LoopbackComm (the same phase code as the
torch.distributed path; tests/test_context_parallel_gloo.py covers that
path's exchanges on CPU)."""
import numpy as np
import pytest
import torch



def head_props(B, H, seed):
    rng = np.random.default_rng(seed)
    return (rng.uniform(0.01, 0.08, (B, H)), rng.uniform(0.0, 0.01, (B, H)),
            (rng.random((B, H)) < 0.4).astype(np.int32))


def _full_and_shards(engine, R, B, Hkv, G, D, l_sink, l_cpu, l_local, dtype, seed, n_new=0):
    from paper_2605_07719_b200.context_parallel import CPShard, shard_kv
    from paper_2605_07719_b200.fluxattn import SparseDecoder
    torch.manual_seed(seed)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    dev = engine.device
    max_new = max(4, n_new)
    cap = SparseDecoder.cap_rows(l_sink + l_cpu + l_local, max_new)
    k = torch.randn((B, Hkv, cap, D), device=dev).to(tdt)
    v = torch.randn((B, Hkv, cap, D), device=dev).to(tdt)
    # planted needles so the selections matter
    g = torch.Generator(device="cpu").manual_seed(seed)
    for b in range(B):
        for h in range(Hkv):
            for _ in range(4):
                s = l_sink + int(torch.randint(0, l_cpu - 16, (1,), generator=g))
                k[b, h, s:s + 16] += (2.0 * torch.randn(D, generator=g)).to(dev, tdt)
    full = SparseDecoder(engine, B, Hkv, G, D, l_sink, l_cpu, l_local, max_new, dtype, k=k, v=v)
    full.build_metadata()
    shards = []
    for r in range(R):
        kr = shard_kv(k, l_sink, l_cpu, l_local, r, R, max_new)
        vr = shard_kv(v, l_sink, l_cpu, l_local, r, R, max_new)
        sh = CPShard(engine, r, R, B, Hkv, G, D, l_sink, l_cpu, l_local, max_new, dtype, k=kr, v=vr)
        sh.dec.build_metadata()
        shards.append(sh)
    if n_new:
        for _ in range(n_new):
            kn = torch.randn((B, Hkv, D), device=dev)
            vn = torch.randn((B, Hkv, D), device=dev)
            full.append(kn, vn)
            shards[-1].dec.append(kn, vn)
    q = torch.randn((B, Hkv * G, D), device=dev)
    q = q / q.norm(dim=-1, keepdim=True) * D ** 0.5
    return full, shards, q


BF16_TOL = 4e-3  # well inside the north-star 2e-2 bf16 bound
PLANS = [("fixed16", dict(fixed=(16, 0.05))), ("fixed128", dict(fixed=(128, 0.3))),
         ("full", dict(full=True)), ("props", "props")]


@pytest.mark.gpu
@pytest.mark.parametrize("R", [2, 3, 4])
@pytest.mark.parametrize("name,plan", PLANS)
def test_cp_matches_single_device(engine, R, name, plan):
    from paper_2605_07719_b200.context_parallel import LoopbackComm, cp_decode_step
    B, Hkv, G, D = 2, 2, 4, 128
    l_sink, l_cpu, l_local = 64, 5000 + 37, 256
    full, shards, q = _full_and_shards(engine, R, B, Hkv, G, D, l_sink, l_cpu, l_local, "bf16",
                                       seed=R * 7 + len(name))
    if plan == "props":
        bgt0, ks, st = head_props(B, Hkv * G, seed=R)
        plan = dict(props=tuple(torch.as_tensor(x, device=engine.device) for x in (bgt0, ks, st)))
    o_ref, lse_ref = full.step(q, **plan)
    (o, lse), *_ = cp_decode_step(shards, LoopbackComm(R), q, **plan)
    torch.cuda.synchronize()
    # plans agree (whole-sequence L_cpu on every shard)
    for sh in shards:
        assert torch.equal(sh.dec.plan_blk, full.plan_blk)
        assert torch.equal(sh.dec.plan_kblocks, full.plan_kblocks)
    # selections: the union of the shards' global ids == the single-device top-k
    for b in range(B):
        for h in range(Hkv * G):
            want = full.selected_blocks(b, h)
            got = np.sort(np.concatenate([sh.global_selection(b, h) for sh in shards]))
            assert np.array_equal(got, want), (b, h, len(got), len(want))
    # the bf16 attention kernel rounds P to bf16 relative to the running max,
    # which depends on where a run is split: ~2^-9 relative per weight
    torch.testing.assert_close(o, o_ref, rtol=BF16_TOL, atol=BF16_TOL)
    torch.testing.assert_close(lse, lse_ref, rtol=1e-4, atol=1e-3)


@pytest.mark.gpu
def test_cp_decoded_rows_on_last_shard(engine):
    from paper_2605_07719_b200.context_parallel import LoopbackComm, cp_decode_step
    B, Hkv, G, D, R = 1, 2, 4, 128, 3
    full, shards, q = _full_and_shards(engine, R, B, Hkv, G, D, 64, 3000, 256, "bf16", seed=5, n_new=3)
    o_ref, lse_ref = full.step(q, fixed=(32, 0.1))
    (o, lse), *_ = cp_decode_step(shards, LoopbackComm(R), q, fixed=(32, 0.1))
    torch.testing.assert_close(o, o_ref, rtol=BF16_TOL, atol=BF16_TOL)
    torch.testing.assert_close(lse, lse_ref, rtol=1e-4, atol=1e-3)


@pytest.mark.gpu
def test_cp_ties_bitexact(engine):
    """Duplicated blocks across shards: equal scores resolve to the lower id,
    exactly as topk_blocks does on one device."""
    from paper_2605_07719_b200.context_parallel import LoopbackComm, cp_decode_step
    from paper_2605_07719_b200.context_parallel import CPShard, shard_kv
    from paper_2605_07719_b200.fluxattn import SparseDecoder
    B, Hkv, G, D, R = 1, 1, 4, 64, 4
    l_sink, l_cpu, l_local = 64, 4096, 256
    dev = engine.device
    cap = SparseDecoder.cap_rows(l_sink + l_cpu + l_local, 4)
    base = torch.randn((1, 1, 128, D), device=dev).to(torch.bfloat16)
    k = base.repeat(1, 1, cap // 128 + 1, 1)[:, :, :cap].contiguous()
    v = torch.randn((B, Hkv, cap, D), device=dev).to(torch.bfloat16)
    full = SparseDecoder(engine, B, Hkv, G, D, l_sink, l_cpu, l_local, 4, "bf16", k=k, v=v)
    full.build_metadata()
    shards = []
    for r in range(R):
        sh = CPShard(engine, r, R, B, Hkv, G, D, l_sink, l_cpu, l_local, 4, "bf16",
                     k=shard_kv(k, l_sink, l_cpu, l_local, r, R, 4), v=shard_kv(v, l_sink, l_cpu, l_local, r, R, 4))
        sh.dec.build_metadata()
        shards.append(sh)
    q = torch.randn((B, Hkv * G, D), device=dev)
    full.step(q, fixed=(64, 0.2))
    cp_decode_step(shards, LoopbackComm(R), q, fixed=(64, 0.2))
    for h in range(G):
        want = full.selected_blocks(0, h)
        got = np.sort(np.concatenate([sh.global_selection(0, h) for sh in shards]))
        assert np.array_equal(got, want)


def _peer_shards(engine, R, B, Hkv, G, D, l_sink, l_cpu, l_local, seed, n_new=0):
    from paper_2605_07719_b200.context_parallel import PeerShard, PeerTables, shard_kv
    full, shards, q = _full_and_shards(engine, R, B, Hkv, G, D, l_sink, l_cpu, l_local, "bf16", seed,
                                       n_new=n_new)
    max_new = max(4, n_new)
    peers = []
    for r in range(R):
        kr = shards[r].dec.k
        vr = shards[r].dec.v
        ps = PeerShard(engine, r, R, B, Hkv, G, D, l_sink, l_cpu, l_local, max_new, "bf16", k=kr, v=vr)
        ps.dec.l_new = shards[r].dec.l_new
        ps.dec.build_metadata()
        peers.append(ps)
    tables = PeerTables(engine, R)
    for s in peers:
        tables.add_local(s)
    return full, peers, tables, q


@pytest.mark.gpu
@pytest.mark.parametrize("R", [2, 3])
@pytest.mark.parametrize("name,plan", PLANS)
def test_cp_peer_exchange_matches_single_device(engine, R, name, plan):
    """The one-shot peer-memory exchanges (no NCCL) give the single-device
    selection bit-exactly and its output within the bf16 merge bound, over
    two steps (both table parities)."""
    from paper_2605_07719_b200.context_parallel import cp_decode_step_peer
    B, Hkv, G, D = 2, 2, 4, 128
    full, peers, tables, q = _peer_shards(engine, R, B, Hkv, G, D, 64, 5000 + 37, 256,
                                          seed=R * 11 + len(name))
    if plan == "props":
        bgt0, ks, st = head_props(B, Hkv * G, seed=R)
        plan = dict(props=tuple(torch.as_tensor(x, device=engine.device) for x in (bgt0, ks, st)))
    for stamp in (1, 2):
        qq = q if stamp == 1 else torch.roll(q, 1, dims=-1)
        o_ref, lse_ref = full.step(qq, **plan)
        o_ref, lse_ref = o_ref.clone(), lse_ref.clone()
        (o, lse), *_ = cp_decode_step_peer(peers, tables, qq, stamp, **plan)
        torch.cuda.synchronize()
        for b in range(B):
            for h in range(Hkv * G):
                want = full.selected_blocks(b, h)
                got = np.sort(np.concatenate([sh.global_selection(b, h) for sh in peers]))
                assert np.array_equal(got, want), (stamp, b, h)
        torch.testing.assert_close(o, o_ref, rtol=BF16_TOL, atol=BF16_TOL)
        torch.testing.assert_close(lse, lse_ref, rtol=1e-4, atol=1e-3)


@pytest.mark.gpu
@pytest.mark.parametrize("R", [2, 3, 4])
@pytest.mark.parametrize("name,plan", PLANS)
def test_cp_dist_bracket_matches_single_device(engine, R, name, plan):
    """The bracket selection distributed over the ranks (stats -> summed
    histograms -> exact-scored bands -> global ranks) selects the
    single-device blocks bit for bit, over three steps (both parities)."""
    from paper_2605_07719_b200.context_parallel import cp_decode_step_dist
    B, Hkv, G, D = 2, 2, 4, 128
    full, peers, tables, q = _peer_shards(engine, R, B, Hkv, G, D, 64, 5000 + 37, 256,
                                          seed=R * 13 + len(name))
    if plan == "props":
        bgt0, ks, st = head_props(B, Hkv * G, seed=R + 1)
        plan = dict(props=tuple(torch.as_tensor(x, device=engine.device) for x in (bgt0, ks, st)))
    for stamp in (1, 2, 3):
        qq = torch.roll(q, stamp - 1, dims=-1)
        o_ref, lse_ref = full.step(qq, **plan)
        o_ref, lse_ref = o_ref.clone(), lse_ref.clone()
        (o, lse), *_ = cp_decode_step_dist(peers, tables, qq, stamp, **plan)
        torch.cuda.synchronize()
        for b in range(B):
            for h in range(Hkv * G):
                want = full.selected_blocks(b, h)
                got = np.sort(np.concatenate([sh.global_selection(b, h) for sh in peers]))
                assert np.array_equal(got, want), (stamp, b, h, len(got), len(want))
        torch.testing.assert_close(o, o_ref, rtol=BF16_TOL, atol=BF16_TOL)
        torch.testing.assert_close(lse, lse_ref, rtol=1e-4, atol=1e-3)


@pytest.mark.gpu
@pytest.mark.parametrize("R,l_cpu,fixed", [(4, 4096, (64, 0.2)), (2, 140000, (16, 0.2))])
def test_cp_dist_bracket_ties_and_mixed_protocols(engine, R, l_cpu, fixed):
    """Every block duplicated across the shards (the whole shard is the band;
    at 70,000 rows per shard it outgrows the shared-memory stage and sorts in
    the table row): ties resolve to the lower global id; then the candidate
    protocol and the bracket protocol alternate on the same tables without a
    stale flag."""
    from paper_2605_07719_b200.context_parallel import (PeerShard, PeerTables, cp_decode_step_dist,
                                                        cp_decode_step_peer, shard_kv)
    from paper_2605_07719_b200.fluxattn import SparseDecoder
    B, Hkv, G, D = 1, 1, 4, 64
    l_sink, l_local = 64, 256
    dev = engine.device
    cap = SparseDecoder.cap_rows(l_sink + l_cpu + l_local, 4)
    base = torch.randn((1, 1, 128, D), device=dev).to(torch.bfloat16)
    k = base.repeat(1, 1, cap // 128 + 1, 1)[:, :, :cap].contiguous()
    v = torch.randn((B, Hkv, cap, D), device=dev).to(torch.bfloat16)
    full = SparseDecoder(engine, B, Hkv, G, D, l_sink, l_cpu, l_local, 4, "bf16", k=k, v=v)
    full.build_metadata()
    peers = []
    for r in range(R):
        sh = PeerShard(engine, r, R, B, Hkv, G, D, l_sink, l_cpu, l_local, 4, "bf16",
                       k=shard_kv(k, l_sink, l_cpu, l_local, r, R, 4),
                       v=shard_kv(v, l_sink, l_cpu, l_local, r, R, 4))
        sh.dec.build_metadata()
        peers.append(sh)
    tables = PeerTables(engine, R)
    for s in peers:
        tables.add_local(s)
    q = torch.randn((B, Hkv * G, D), device=dev)
    for stamp, fn in ((1, cp_decode_step_dist), (2, cp_decode_step_peer), (3, cp_decode_step_dist)):
        qq = torch.roll(q, stamp, dims=-1)
        o_ref, lse_ref = full.step(qq, fixed=fixed)
        o_ref, lse_ref = o_ref.clone(), lse_ref.clone()
        (o, lse), *_ = fn(peers, tables, qq, stamp, fixed=fixed)
        torch.cuda.synchronize()
        for h in range(G):
            want = full.selected_blocks(0, h)
            got = np.sort(np.concatenate([sh.global_selection(0, h) for sh in peers]))
            assert np.array_equal(got, want), (stamp, h)
        torch.testing.assert_close(o, o_ref, rtol=BF16_TOL, atol=BF16_TOL)


@pytest.mark.gpu
def test_cp_peer_exchange_two_processes(tmp_path):
    """Two processes, one rank each, on one GPU: the tables cross the process
    boundary through CUDA IPC and the kernels synchronise on each other's
    ready flags -- the multi-GPU protocol minus the NVLink hop."""
    import random
    import torch.multiprocessing as mp
    import cp_peer_worker
    port = random.randint(20000, 40000)
    mp.spawn(cp_peer_worker.run, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    assert (tmp_path / "ok0").exists() and (tmp_path / "ok1").exists()


@pytest.mark.gpu
def test_cp_dist_bracket_two_processes(tmp_path):
    """The distributed bracket selection across a process boundary: stats,
    histograms and bands read through CUDA IPC after the peers' flags."""
    import random
    import torch.multiprocessing as mp
    import cp_peer_worker
    port = random.randint(20000, 40000)
    mp.spawn(cp_peer_worker.run, args=(2, port, str(tmp_path), "dist"), nprocs=2, join=True)
    assert (tmp_path / "ok0").exists() and (tmp_path / "ok1").exists()
