"""Hybrid HBM / host-memory KV at the C2 layer shape (tiered.py): N sequences
in HBM plus M in pinned host memory (the M lowest-volume ones by the
V-ordered assignment), one decode step = both tiers concurrently.  Compared
with the all-HBM step over the same N + M sequences and with the HBM tier alone."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_07719_b200.fluxattn import Engine, SparseDecoder  # noqa: E402
from paper_2605_07719_b200.tiered import TieredDecoder, assign_tiers, sequence_volumes  # noqa: E402

N_HBM = int(sys.argv[1]) if len(sys.argv) > 1 else 16
N_HOST = int(sys.argv[2]) if len(sys.argv) > 2 else 2
B, HKV, G, D, ls, ll = N_HBM + N_HOST, 8, 4, 128, 64, 256
lc = 131072 - 320
eng = Engine(0)
dev = eng.device
rng = np.random.default_rng(1)
props = (rng.uniform(0.01, 0.05, (B, 32)), rng.uniform(0, 0.01, (B, 32)), (rng.random((B, 32)) < 0.5).astype(np.int32))
vol = sequence_volumes(eng, props, lc, G)
host = assign_tiers(vol, N_HBM)
dprops = tuple(torch.as_tensor(x, device=dev) for x in props)
q = torch.randn((B, 32, D), device=dev)


def timed(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / n * 1e3


res = {"n_hbm": N_HBM, "n_host": N_HOST, "host_sequences": host,
       "host_volume_share": float(vol[host].sum() / vol.sum())}
tier = TieredDecoder(eng, B, HKV, G, D, ls, lc, ll, host_sequences=host, max_new=64)
for t, dec in enumerate(tier.tiers):
    g = torch.Generator(device=dec.k.device).manual_seed(t)
    for b in range(dec.lay.batch):
        dec.k[b].normal_(generator=g)
        dec.v[b].normal_(generator=g)
t0 = time.perf_counter()
tier.build_metadata()
torch.cuda.synchronize()
res["tiered_meta_build_ms"] = (time.perf_counter() - t0) * 1e3
res["tiered_step_ms"] = timed(lambda: tier.step(q, props=dprops))
hb = tier.tiers[0]
idx = tier._idx[0]
qd, pd = q.index_select(0, idx), tuple(p.index_select(0, idx) for p in dprops)
res["hbm_tier_alone_ms"] = timed(lambda: hb.step(qd, props=pd))
hs = tier.tiers[1]
idx = tier._idx[1]
qh, ph = q.index_select(0, idx), tuple(p.index_select(0, idx) for p in dprops)
res["host_tier_alone_ms"] = timed(lambda: hs.step(qh, props=ph))
del tier, hb, hs
torch.cuda.empty_cache()
full = SparseDecoder(eng, B, HKV, G, D, ls, lc, ll, max_new=64, dtype="bf16")
full.k.normal_()
full.v.normal_()
full.build_metadata()
res["all_hbm_step_ms"] = timed(lambda: full.step(q, props=dprops))
print(json.dumps(res))
