"""Small end-to-end run of the hot path for compute-sanitizer (memcheck /
racecheck / synccheck / initcheck): metadata levels (+ means), a bf16 decode
step through the TMA kernels with the fused worklist and split-run merges,
an f32 step through the CUDA-core kernels, the predictor path and the
context-parallel bracket exchange between two shards on one device.
Usage: compute-sanitizer --tool <tool> python profiles/sanitizer/small_step.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2605_07719_b200.fluxattn import Engine, Predictor, SparseDecoder  # noqa: E402

eng = Engine(0)
dev = eng.device
rng = np.random.default_rng(0)
B, HKV, G, D = 2, 2, 4, 128
for dtype in ("bf16", "f32"):
    dec = SparseDecoder(eng, B, HKV, G, D, 64, 3000, 256, max_new=80, dtype=dtype)
    dec.k.normal_()
    dec.v.normal_()
    dec.build_metadata(means=True)
    q = torch.randn((B, HKV * G, D), device=dev)
    props = tuple(torch.as_tensor(x, device=dev) for x in (rng.uniform(0.01, 0.05, (B, HKV * G)),
                                                            rng.uniform(0, 0.01, (B, HKV * G)),
                                                            (rng.random((B, HKV * G)) < 0.5).astype(np.int32)))
    o, lse = dec.step(q, props=props)
    kv = torch.randn((2, B, HKV, D), device=dev)
    dec.step(q, fixed=(16, 0.05), append=(kv[0], kv[1]))
    dec.step(q, full=True)
    torch.cuda.synchronize()
    if dtype == "bf16":
        params = {"w1": rng.standard_normal((256, 41)) * 0.2, "b1": np.zeros(256),
                  "w2": rng.standard_normal((384, 256)) * 0.1, "b2": np.zeros(384),
                  "w3": rng.standard_normal((3, 384)) * 1e-2, "b3": np.array([0.03, 0.005, 0.0]),
                  "mu": np.zeros(41), "sigma": np.ones(41) * 50}
        pred = Predictor(eng, params)
        rec = dec.prefill_stats(q, tau=0.10, layer=0)
        pp = dec.predict_props(q, rec, pred)
        dec.step(q, props=pp)
        # decoded rows across a 64-row chunk boundary, the last one appended by
        # the feature kernel itself; the features alone (fx_decode_features)
        for _ in range(66):
            dec.append(kv[0], kv[1])
        pp = dec.predict_props(q, rec, pred, append=(kv[0], kv[1]))
        dec.step(q, props=pp)
        dec.decode_features(q, rec)
        torch.cuda.synchronize()
        pred.close()
    print(dtype, "ok", float(o.abs().sum()))

# context-parallel bracket exchange, two shards on one device
from paper_2605_07719_b200.context_parallel import PeerShard, PeerTables, cp_decode_step_dist, shard_kv  # noqa: E402
R, l_cpu = 2, 4096
full = SparseDecoder(eng, 1, HKV, G, D, 64, l_cpu, 256, max_new=4, dtype="bf16")
full.k.normal_()
full.v.normal_()
shards = []
for r in range(R):
    kr = shard_kv(full.k, 64, l_cpu, 256, r, R, 4)
    vr = shard_kv(full.v, 64, l_cpu, 256, r, R, 4)
    sh = PeerShard(eng, r, R, 1, HKV, G, D, 64, l_cpu, 256, 4, "bf16", k=kr, v=vr)
    sh.dec.build_metadata()
    shards.append(sh)
tables = PeerTables(eng, R)
for sh in shards:
    tables.add_local(sh)
q = torch.randn((1, HKV * G, D), device=dev)
(o, lse), *_ = cp_decode_step_dist(shards, tables, q, 1, fixed=(16, 0.1))
torch.cuda.synchronize()
print("cp ok", float(o.abs().sum()))
