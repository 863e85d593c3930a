"""Hybrid HBM / host-memory KV (paper_2605_07719_b200/tiered.py):
the host tier's K/V live in pinned host memory that the same kernels read
over the link; the tiers step concurrently on two streams."""
import numpy as np
import pytest
import torch


def test_assign_tiers_follows_the_priority_order():
    """The HBM tier takes the largest volumes (the head of the reference's
    V-descending queue, scheduler.cpp:65-76); ties keep the lower id in HBM."""
    from paper_2605_07719_b200.tiered import assign_tiers
    assert assign_tiers([5.0, 1.0, 7.0, 3.0], 2) == [1, 3]
    assert assign_tiers([2.0, 2.0, 2.0], 1) == [1, 2]
    assert assign_tiers([1.0, 2.0], 2) == []
    assert assign_tiers([1.0, 2.0], 0) == [0, 1]


@pytest.mark.gpu
def test_tiered_step_equals_all_hbm_step(engine, coracle):
    from paper_2605_07719_b200.fluxattn import SparseDecoder
    from paper_2605_07719_b200.tiered import TieredDecoder, assign_tiers, sequence_volumes
    B, Hkv, G, D, ls, lc, ll = 4, 2, 4, 128, 64, 4000, 256
    rng = np.random.default_rng(3)
    props = (rng.uniform(0.01, 0.05, (B, Hkv * G)), rng.uniform(0, 0.01, (B, Hkv * G)),
             (rng.random((B, Hkv * G)) < 0.5).astype(np.int32))
    vol = sequence_volumes(engine, props, lc, G)
    host = assign_tiers(vol, 2)
    assert len(host) == 2 and min(vol[b] for b in range(B) if b not in host) >= max(vol[b] for b in host)
    tier = TieredDecoder(engine, B, Hkv, G, D, ls, lc, ll, host_sequences=host, max_new=4)
    assert tier.tiers[1].k.device.type == "cpu" and tier.tiers[1].k.is_pinned()
    ref = SparseDecoder(engine, B, Hkv, G, D, ls, lc, ll, max_new=4, dtype="bf16")
    for b in range(B):
        for g in range(Hkv):
            k = torch.as_tensor(rng.standard_normal((ls + lc + ll, D)).astype(np.float32)).bfloat16().float().numpy()
            v = torch.as_tensor(rng.standard_normal((ls + lc + ll, D)).astype(np.float32)).bfloat16().float().numpy()
            k[ls + 16 * b:ls + 16 * b + 16] += 2.0  # a needle per sequence
            tier.load_group(b, g, k, v)
            ref.load_group(b, g, k, v)
    tier.build_metadata()
    ref.build_metadata()
    dprops = tuple(torch.as_tensor(x, device=engine.device) for x in props)
    for step in range(2):
        if step:
            kv = torch.randn((2, B, Hkv, D), device=engine.device).bfloat16().float()
            tier.append(kv[0], kv[1])
            ref.append(kv[0], kv[1])
        q = torch.randn((B, Hkv * G, D), device=engine.device).bfloat16().float()
        o, lse = tier.step(q, props=dprops)
        o2, lse2 = ref.step(q, props=dprops)
        torch.cuda.synchronize()
        # same selections; outputs equal up to the split-K partition, which
        # differs between a 2-sequence and a 4-sequence launch (the per-partial
        # softmax max sets the bf16 rounding of P): within the bf16 bar
        err = ((o - o2).abs().max() / o2.abs().max().clamp(min=1.0)).item()
        assert err < 2e-2, err
        torch.testing.assert_close(lse, lse2, rtol=1e-3, atol=1e-3)
        for b in range(B):
            for h in range(Hkv * G):
                assert np.array_equal(tier.selected_blocks(b, h), ref.selected_blocks(b, h))
