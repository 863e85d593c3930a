"""Timing of the predictor path pieces at the C2 shape (16 x 8 groups, 128K,
bf16): fx_predict_props, decode features alone, the predictor alone, at
several decoded-row counts.  CUDA events around back-to-back loops."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_07719_b200.fluxattn import Engine, Predictor, SparseDecoder  # noqa: E402

eng = Engine(0)
dev = eng.device
B, HKV, G, D = 16, 8, 4, 128
dec = SparseDecoder(eng, B, HKV, G, D, 64, 131072 - 320, 256, max_new=640, dtype="bf16")
dec.k.normal_()
dec.v.normal_()
dec.build_metadata()
q = torch.randn((B, 32, D), device=dev)
rs = np.random.default_rng(5)
params = {"w1": rs.standard_normal((256, 41)) * (2.0 / 41) ** 0.5, "b1": np.zeros(256),
          "w2": rs.standard_normal((384, 256)) * (2.0 / 256) ** 0.5, "b2": np.zeros(384),
          "w3": rs.standard_normal((3, 384)) * 1e-2, "b3": np.array([0.03, 0.005, 0.0]),
          "mu": np.zeros(41), "sigma": np.ones(41) * 50}
pred = Predictor(eng, params)
rec = dec.prefill_stats(q, tau=0.10, layer=0)
feats = torch.empty((B, 32, 41), dtype=torch.float64, device=dev)
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)


def timed(fn, n=50):
    """GPU time per call: n calls captured as one CUDA graph, replayed (the
    host launch path is outside the measurement)."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s_cap = torch.cuda.Stream(dev)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s_cap):
        eng.sync_stream()
        for _ in range(n):
            fn()
    eng.sync_stream()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


out = {}
for ln in (0, 100, 460, 600):
    dec.l_new = ln
    out[ln] = {"predict_props_us": timed(lambda: dec.predict_props(q, rec, pred)),
               "features_us": timed(lambda: dec.decode_features(q, rec, out=feats)),
               "predictor_us": timed(lambda: pred(feats))}
print(json.dumps(out, indent=1))
