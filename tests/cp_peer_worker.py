"""Worker for tests/test_context_parallel.py::test_cp_peer_exchange_two_processes:
one rank of a 2-process context-parallel step on ONE GPU, the exchange tables
shared through CUDA IPC (handles swapped over a gloo process group), checked
against the single-device step computed in the same process."""
import os
import sys

import numpy as np
import torch


def run(rank, world, port, out_dir, protocol="candidates"):
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    from paper_2605_07719_b200.context_parallel import (PeerShard, PeerTables, cp_decode_step_dist,
                                                        cp_decode_step_peer, shard_kv)
    from paper_2605_07719_b200.fluxattn import Engine, SparseDecoder
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    eng = Engine(0)
    dev = eng.device
    B, Hkv, G, D, l_sink, l_cpu, l_local = 2, 2, 4, 128, 64, 6000, 256
    torch.manual_seed(123)
    cap = SparseDecoder.cap_rows(l_sink + l_cpu + l_local, 4)
    k = torch.randn((B, Hkv, cap, D), device=dev).to(torch.bfloat16)
    v = torch.randn((B, Hkv, cap, D), device=dev).to(torch.bfloat16)
    full = SparseDecoder(eng, B, Hkv, G, D, l_sink, l_cpu, l_local, 4, "bf16", k=k, v=v)
    full.build_metadata()
    sh = PeerShard(eng, rank, world, B, Hkv, G, D, l_sink, l_cpu, l_local, 4, "bf16",
                   k=shard_kv(k, l_sink, l_cpu, l_local, rank, world, 4),
                   v=shard_kv(v, l_sink, l_cpu, l_local, rank, world, 4))
    sh.dec.build_metadata()
    tables = PeerTables.over_dist(eng, sh)
    q = torch.randn((B, Hkv * G, D), device=dev)
    for stamp in (1, 2, 3):
        qq = torch.roll(q, stamp, dims=-1)
        o_ref, lse_ref = full.step(qq, fixed=(16, 0.1))
        o_ref, lse_ref = o_ref.clone(), lse_ref.clone()
        step = cp_decode_step_dist if protocol == "dist" else cp_decode_step_peer
        (o, lse), = step([sh], tables, qq, stamp, fixed=(16, 0.1))
        torch.cuda.synchronize()
        torch.testing.assert_close(o, o_ref, rtol=4e-3, atol=4e-3)
        torch.testing.assert_close(lse, lse_ref, rtol=1e-4, atol=1e-3)
        # this rank's share of the selection == the single-device blocks it holds
        for b in range(B):
            for h in range(Hkv * G):
                want = full.selected_blocks(b, h)
                lo, hi = sh.offset // 16, (sh.offset + sh.rows) // 16
                mine = want[(want >= lo) & (want < hi)]
                assert np.array_equal(np.sort(sh.global_selection(b, h)), mine), (stamp, b, h)
    dist.barrier()  # no rank unmaps while a peer may still read its tables
    tables.close()
    with open(os.path.join(out_dir, f"ok{rank}"), "w") as f:
        f.write("ok")
    dist.destroy_process_group()
