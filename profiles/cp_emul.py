"""C5 (1M ctx, batch 4) as 8 context-parallel shards on ONE GPU, one process:
per-step time of the collective protocol (LoopbackComm: torch stacks + the
host read of the exchange size) vs the one-shot peer-memory protocol.  The
shards run one after another, so this is the protocol's serial cost, not an
8-GPU number."""
import json, sys, time
import torch
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_07719_b200.fluxattn import Engine, SparseDecoder
from paper_2605_07719_b200.context_parallel import (CPShard, PeerShard, PeerTables, LoopbackComm,
                                                    cp_decode_step, cp_decode_step_peer, cp_decode_step_dist, shard_kv)
import numpy as np
eng = Engine(0); dev = eng.device
B, HKV, G, D, R = 4, 8, 4, 128, 8
ctx = 1 << 20; l_cpu = ctx - 320
full = SparseDecoder(eng, B, HKV, G, D, 64, l_cpu, 256, max_new=4, dtype="bf16")
out = full.generate(dict(seed=1, layers=1, heads=32, group_size=G, head_dim=D, context_len=ctx, decode_steps=40), steps=40)
full.build_metadata()
qs = out["step_q"]
rng = np.random.default_rng(1)
props = tuple(torch.as_tensor(x, device=dev) for x in (rng.uniform(0.01, 0.05, (B, 32)), rng.uniform(0, 0.01, (B, 32)), (rng.random((B, 32)) < 0.5).astype(np.int32)))
res = {}
for kind in ("single", "collective", "peer", "dist", "shard_local"):
    if kind == "collective":
        shards = []
        for r in range(R):
            sh = CPShard(eng, r, R, B, HKV, G, D, 64, l_cpu, 256, 4, "bf16", k=shard_kv(full.k, 64, l_cpu, 256, r, R, 4), v=shard_kv(full.v, 64, l_cpu, 256, r, R, 4))
            sh.dec.build_metadata(); shards.append(sh)
        comm = LoopbackComm(R)
        fn = lambda i: cp_decode_step(shards, comm, qs[i], props=props)
    elif kind == "peer":
        del shards; torch.cuda.empty_cache()
        shards = []
        for r in range(R):
            sh = PeerShard(eng, r, R, B, HKV, G, D, 64, l_cpu, 256, 4, "bf16", k=shard_kv(full.k, 64, l_cpu, 256, r, R, 4), v=shard_kv(full.v, 64, l_cpu, 256, r, R, 4))
            sh.dec.build_metadata(); shards.append(sh)
        tables = PeerTables(eng, R)
        for sh in shards: tables.add_local(sh)
        fn = lambda i: cp_decode_step_peer(shards, tables, qs[i], i + 1, props=props)
    elif kind == "dist":
        fn = lambda i: cp_decode_step_dist(shards, tables, qs[i], 100 + i, props=props)
    elif kind == "shard_local":
        fn = lambda i: shards[0].dec.step(qs[i], props=props)
    else:
        fn = lambda i: full.step(qs[i], props=props)
    for i in range(3): fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(3, 23): fn(i)
    e1.record(); torch.cuda.synchronize()
    res[kind] = e0.elapsed_time(e1) / 20
print(json.dumps({"c5_one_gpu_ms_per_step": res, "note": "8 shards serially on one GPU; single = one-device step"}))
