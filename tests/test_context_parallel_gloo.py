"""The context-parallel step's exchanges over torch.distributed (gloo,
world_size 2 and 3, CPU): cp_decode_step + TorchComm with oracle-backed
shards must reproduce the single-device oracle's topk_blocks selection and
execute_task output (scheduler.cpp:78-96) for every head."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _data(seed=3, B=1, Hkv=2, G=2, D=16, l_sink=8, l_cpu=1000, l_local=32):
    rng = np.random.default_rng(seed)
    rows = l_sink + l_cpu + l_local
    K = rng.standard_normal((B, Hkv, rows, D)).astype(np.float32)
    V = rng.standard_normal((B, Hkv, rows, D)).astype(np.float32)
    for b in range(B):
        for g in range(Hkv):
            for _ in range(3):
                s = l_sink + rng.integers(0, l_cpu - 16)
                K[b, g, s:s + 16] += 2.0 * rng.standard_normal(D).astype(np.float32)
    q = rng.standard_normal((B, Hkv * G, D)).astype(np.float32)
    return K, V, q, dict(l_sink=l_sink, l_cpu=l_cpu, l_local=l_local, G=G)


def _worker(rank, world, port, fixed, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(__file__))
        from cp_oracle_shard import OracleShard
        from oracle.oracle import COracle
        from paper_2605_07719_b200.context_parallel import TorchComm, cp_decode_step
        K, V, q, cfg = _data()
        sh = OracleShard(COracle(), rank, world, K, V, cfg["l_sink"], cfg["l_cpu"],
                         cfg["l_local"], cfg["G"])
        o = torch.zeros(q.shape, dtype=torch.float64)
        lse = torch.zeros(q.shape[:2], dtype=torch.float64)
        cp_decode_step([sh], TorchComm(), torch.from_numpy(q), out=[(o, lse)], fixed=fixed)
        out_q.put((rank, sh.selected, o.numpy(), lse.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,fixed", [(2, (16, 0.1)), (2, (64, 0.3)), (3, (32, 0.05))])
def test_cp_over_gloo_matches_single_device(coracle, world, fixed):
    ctx = mp.get_context("spawn")
    q_out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fixed, q_out)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q_out.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda x: x[0])
    K, V, q, cfg = _data()
    blk, bgt = fixed
    l_sink, l_cpu, l_local, G = cfg["l_sink"], cfg["l_cpu"], cfg["l_local"], cfg["G"]
    k = coracle.blocks_for_budget(bgt, l_cpu, blk)
    B, Hkv = K.shape[:2]
    for b in range(B):
        for g in range(Hkv):
            mins, maxs = coracle.build_metadata(K[b, g, l_sink:l_sink + l_cpu], blk)
            o_ref, lse_ref, _ = coracle.execute_group(K[b, g], V[b, g], (l_sink, l_cpu, l_local, 0),
                                                      q[b, g * G:(g + 1) * G], blk, [bgt] * G)
            for j in range(G):
                hi = (b * Hkv + g) * G + j
                want, _ = coracle.topk_blocks(q[b, g * G + j], mins, maxs, k)
                got = sorted(i for r in res for i in r[1][hi])
                assert got == sorted(want.tolist())
                for r in res:  # every rank holds the merged output
                    np.testing.assert_allclose(r[2][b, g * G + j], o_ref[j], rtol=1e-9, atol=1e-12)
                    np.testing.assert_allclose(r[3][b, g * G + j], lse_ref[j], rtol=1e-12)
