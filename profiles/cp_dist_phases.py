"""Per-phase time of the distributed bracket step, 8 C5 shards serially on one GPU."""
import json, sys
import ctypes as C
import torch
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2605_07719_b200.fluxattn import Engine, SparseDecoder
from paper_2605_07719_b200.context_parallel import PeerShard, PeerTables, shard_kv
from paper_2605_07719_b200._native import LIB, check
eng = Engine(0); dev = eng.device
B, HKV, G, D, R = 4, 8, 4, 128, 8
ctx = 1 << 20; l_cpu = ctx - 320
full = SparseDecoder(eng, B, HKV, G, D, 64, l_cpu, 256, max_new=4, dtype="bf16")
out = full.generate(dict(seed=1, layers=1, heads=32, group_size=G, head_dim=D, context_len=ctx, decode_steps=40), steps=40)
full.build_metadata()
qs = out["step_q"]
rng = np.random.default_rng(1)
props = tuple(torch.as_tensor(x, device=dev) for x in (rng.uniform(0.01, 0.05, (B, 32)), rng.uniform(0, 0.01, (B, 32)), (rng.random((B, 32)) < 0.5).astype(np.int32)))
shards = []
for r in range(R):
    sh = PeerShard(eng, r, R, B, HKV, G, D, 64, l_cpu, 256, 4, "bf16", k=shard_kv(full.k, 64, l_cpu, 256, r, R, 4), v=shard_kv(full.v, 64, l_cpu, 256, r, R, 4))
    sh.dec.build_metadata(); shards.append(sh)
del full; torch.cuda.empty_cache()
tables = PeerTables(eng, R)
for sh in shards: tables.add_local(sh)
names = ["phase0 plan+approx+stats", "phase1 hist", "phase2 band", "phase3 rank", "attend", "combine"]
acc = np.zeros(6)
n = 0
for i in range(25):
    stamp = i + 1; par = stamp % 2; peers = tables.array(par)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
    ev[0].record()
    for ph in range(4):
        for s in shards:
            s.dist_phase(qs[i], par, ph, tables, peers, stamp, props=props)
        ev[ph + 1].record()
    for s in shards:
        st = s.sets[par]
        s.dec.step(qs[i], blk="keep", out=st["o"], lse=st["lse"], sel_in=s.sel)
        check(LIB.fx_cp_signal(s.eng.ctx, C.c_void_p(s.flags[par].data_ptr()), 3, stamp))
    ev[5].record()
    for s in shards:
        o = torch.empty_like(s.o); l = torch.empty_like(s.lse)
        check(LIB.fx_cp_combine_peer(s.eng.ctx, R, s.n_heads, D, peers, stamp, o.data_ptr(), l.data_ptr()))
    ev[6].record(); torch.cuda.synchronize()
    if i >= 5:
        acc += [ev[j].elapsed_time(ev[j + 1]) for j in range(6)]; n += 1
print(json.dumps({k: round(v / n / R * 1000, 2) for k, v in zip(names, acc)} | {"unit": "us per shard"}))
