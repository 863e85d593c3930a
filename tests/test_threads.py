"""The C-ABI is callable from several host threads at once (SURVEY §8b
threading: per-device contexts, no global mutable state beyond them).  Two
threads, each with its own context bound to its own CUDA stream, run decode
steps on their own caches concurrently; every output must equal the same
step run alone on one thread, bit for bit (the kernels are deterministic:
selection is exact and the split-K merge order is fixed by the worklist)."""
import threading

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _decoder(engine, seed, l_cpu=20000):
    from paper_2605_07719_b200.fluxattn import SparseDecoder
    B, Hkv, G, D = 2, 2, 4, 128
    g = torch.Generator(device="cpu").manual_seed(seed)
    cap = SparseDecoder.cap_rows(64 + l_cpu + 256, 8)
    k = torch.randn((B, Hkv, cap, D), generator=g).to(torch.bfloat16).to(engine.device)
    v = torch.randn((B, Hkv, cap, D), generator=g).to(torch.bfloat16).to(engine.device)
    dec = SparseDecoder(engine, B, Hkv, G, D, 64, l_cpu, 256, 8, "bf16", k=k, v=v)
    dec.build_metadata()
    q = torch.randn((6, B, Hkv * G, D), generator=g).to(engine.device)
    return dec, q


def _plan(dev, seed, B=2, H=8):
    rng = np.random.default_rng(seed)
    return tuple(torch.as_tensor(x, device=dev) for x in (rng.uniform(0.02, 0.1, (B, H)),
                                                          rng.uniform(0.0, 0.01, (B, H)),
                                                          (rng.random((B, H)) < 0.3).astype(np.int32)))


def _run(engine, seed):
    dec, q = _decoder(engine, seed)
    props = _plan(engine.device, seed)
    outs = []
    for i in range(q.shape[0]):
        o, lse = dec.step(q[i], props=props)
        outs.append((o.clone(), lse.clone(), dec.sel_bits.clone()))
    torch.cuda.current_stream(engine.device).synchronize()
    return outs


def test_two_threads_two_contexts_match_serial():
    from paper_2605_07719_b200.fluxattn import Engine
    dev = torch.device("cuda", 0)
    want = {s: _run(Engine(0), s) for s in (3, 4)}
    got, errors = {}, []

    def worker(seed):
        try:
            with torch.cuda.stream(torch.cuda.Stream(dev)):
                eng = Engine(0)  # binds to this thread's current stream
                res = []
                for _ in range(3):
                    res = _run(eng, seed)
                got[seed] = res
        except Exception as e:  # surfaced below
            errors.append(e)

    th = [threading.Thread(target=worker, args=(s,)) for s in (3, 4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    for s in (3, 4):
        for (o, lse, sel), (wo, wl, ws) in zip(got[s], want[s]):
            assert torch.equal(sel, ws)
            assert torch.equal(o, wo)
            assert torch.equal(lse, wl)
